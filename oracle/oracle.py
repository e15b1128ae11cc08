"""TEST INFRASTRUCTURE ONLY — Python (ctypes) access to the CPU checkers.

Two libraries, both built by ``oracle/Makefile`` (called from ``__graft_entry__.build()``):

* ``oracle/liboracle.so``          the C restatement of the reference algorithm (``fcvbw_oracle.c``);
* ``oracle/_ref/libfcvbw_ref.so``  the unmodified reference headers compiled in place
                                   (``ref_shim.cpp``; built only where /root/reference exists, the
                                   prebuilt file travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (``cpu_baseline`` and
``--impl reference``) may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfcvbw_ref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def _declare(lib, prefix: str):
    p = prefix
    fns = {
        "validate": ([C.c_int] * 7, C.c_int),
        "phase_table": ([C.c_int, C.c_int, _f64p], None if p == "orc_" else C.c_int),
        "coefficients": ([C.c_int] * 5 + [_f64p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
        "ols_raw_real": ([C.c_int, C.c_int, _f64p, _f64p, C.c_int64, _f64p], C.c_int),
        "naive_block_filter": ([C.c_int, C.c_int, _f64p, _f64p, C.c_int64, _f64p], C.c_int),
        "rng_uniform": ([C.c_uint64, C.c_double, C.c_double, _f64p, C.c_int64], None),
        "rng_uniform_int": ([C.c_uint64, C.c_int, C.c_int, _i32p, C.c_int64], None),
        "verify": ([C.c_int] * 5 + [_f64p, C.c_double, C.c_int, C.c_int, C.c_int, C.c_double, _f64p, _f64p,
                    _f64p, _i32p], C.c_int),
    }
    for name, (args, res) in fns.items():
        f = getattr(lib, p + name)
        f.argtypes = args
        f.restype = res
    f = getattr(lib, p + "direct_fir")
    f.argtypes = [_f64p, C.c_int, _f64p, C.c_int64, _f64p]
    f.restype = None if p == "orc_" else C.c_int
    if p == "orc_":
        lib.orc_ols_real.argtypes = [C.c_int] * 5 + [_f64p, _f64p, C.c_int64, C.c_void_p, C.c_int, _f64p]
        lib.orc_ols_real.restype = C.c_int
        lib.orc_ols_complex.argtypes = [C.c_int] * 5 + [_f64p, _f64p, C.c_int64, C.c_int, C.c_void_p,
                                                        C.c_int64, C.c_int, _f64p, C.c_int]
        lib.orc_ols_complex.restype = C.c_int
    else:
        lib.ref_ols_real.argtypes = [C.c_int] * 5 + [_f64p, _f64p, C.c_int64, C.c_void_p, C.c_int, _f64p, C.c_int]
        lib.ref_ols_real.restype = C.c_int
        lib.ref_ols_complex.argtypes = [C.c_int] * 5 + [_f64p, _f64p, C.c_int64, C.c_int, C.c_void_p,
                                                        C.c_int64, C.c_int, _f64p, C.c_int]
        lib.ref_ols_complex.restype = C.c_int
        lib.ref_design.argtypes = [C.c_int] * 6 + [_f64p, _f64p]
        lib.ref_design.restype = C.c_int
        lib.ref_shift_rule.argtypes = [C.c_int] * 5 + [_i32p, _i32p]
        lib.ref_solve_minimax.argtypes = [C.c_int] * 7 + [C.c_double, C.c_int, C.c_int, _f64p, _f64p, _i64p]
        lib.ref_solve_minimax.restype = C.c_int
        lib.ref_design_full.argtypes = [_f64p, _i32p, _f64p, _i32p, _f64p, C.c_int, _f64p]
        lib.ref_design_full.restype = C.c_int
        lib.ref_shift_rule.restype = C.c_int
        lib.ref_last_error.restype = C.c_char_p
    return lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _Lib:
    """Common wrapper; ``kind`` is 'port' (C restatement) or 'reference' (compiled reference)."""

    def __init__(self, path: str, prefix: str, kind: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle` (build())")
        self.lib = _declare(C.CDLL(path), prefix)
        self.p = prefix
        self.kind = kind

    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc):
        if rc:
            msg = self.lib.ref_last_error().decode() if self.p == "ref_" else ""
            raise OracleError(rc, msg)

    # --- domain model -------------------------------------------------------
    def validate(self, n, l, m, dn, blo, bhi, lv) -> int:
        return self._fn("validate")(n, l, m, dn, blo, bhi, lv)

    def phase_table(self, n, l) -> np.ndarray:
        out = np.zeros(2 * n)
        self._fn("phase_table")(n, l, out)
        return out.view(np.complex128)

    def coefficients(self, n, l, dn, blo, bhi, v, b):
        v = np.ascontiguousarray(v, np.float64)
        mag = np.zeros(n)
        reg = np.zeros(n, np.int32)
        tab = np.zeros(2 * n)
        self._check(self._fn("coefficients")(n, l, dn, blo, bhi, v, b, _ptr(mag), _ptr(reg), _ptr(tab)))
        return mag, reg, tab.view(np.complex128)

    # --- engines -------------------------------------------------------------
    def ols_real(self, n, l, dn, blo, bhi, v, x, bsched=None, b0=None, threads=1):
        v = np.ascontiguousarray(v, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros_like(x)
        bs = None if bsched is None else np.ascontiguousarray(bsched, np.int32)
        b0 = blo if b0 is None else b0
        if self.p == "ref_":
            rc = self.lib.ref_ols_real(n, l, dn, blo, bhi, v, x, x.size, _ptr(bs), b0, y, threads)
        else:
            rc = self.lib.orc_ols_real(n, l, dn, blo, bhi, v, x, x.size, _ptr(bs), b0, y)
        self._check(rc)
        return y

    def ols_complex(self, n, l, dn, blo, bhi, v, x, bsched=None, b0=None, threads=None):
        """x: complex array [channels, S] (or [S]); bsched: [nblocks] shared or [channels, nblocks]."""
        v = np.ascontiguousarray(v, np.float64)
        x = np.asarray(x)
        squeeze = x.ndim == 1
        x2 = np.ascontiguousarray(np.atleast_2d(x).astype(np.complex128))
        ch, s = x2.shape
        y = np.zeros_like(x2)
        bs, stride = None, 0
        if bsched is not None:
            bs = np.ascontiguousarray(bsched, np.int32)
            stride = bs.shape[-1] if bs.ndim == 2 else 0
        b0 = blo if b0 is None else b0
        threads = threads or os.cpu_count() or 1
        fn = self._fn("ols_complex")
        rc = fn(n, l, dn, blo, bhi, v, x2.view(np.float64).reshape(-1), s, ch, _ptr(bs), stride, b0,
                y.view(np.float64).reshape(-1), threads)
        self._check(rc)
        return y[0] if squeeze else y

    def ols_raw_real(self, n, m, table, x):
        t = np.ascontiguousarray(np.asarray(table, np.complex128)).view(np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros_like(x)
        self._check(self._fn("ols_raw_real")(n, m, t, x, x.size, y))
        return y

    def naive_block_filter(self, n, m, table, x):
        t = np.ascontiguousarray(np.asarray(table, np.complex128)).view(np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros_like(x)
        self._check(self._fn("naive_block_filter")(n, m, t, x, x.size, y))
        return y

    def direct_fir(self, taps, x):
        taps = np.ascontiguousarray(taps, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros_like(x)
        self._fn("direct_fir")(taps, taps.size, x, x.size, y)
        return y

    # --- SeededRng -------------------------------------------------------------
    def rng_uniform(self, seed, lo, hi, count):
        out = np.zeros(count)
        self._fn("rng_uniform")(seed, lo, hi, out, count)
        return out

    def rng_uniform_int(self, seed, lo, hi, count):
        out = np.zeros(count, np.int32)
        self._fn("rng_uniform_int")(seed, lo, hi, out, count)
        return out

    # --- design (reference only) -------------------------------------------------
    def design(self, n, l, dn, blo, bhi, grid_k):
        v = np.zeros(dn - 1)
        d = np.zeros(1)
        self._check(self.lib.ref_design(n, l, dn, blo, bhi, grid_k, v, d))
        return v, float(d[0])

    def verify(self, n, l, dn, blo, bhi, v, design_delta, grid_points, facets, dense, delta_e):
        """verify() (design.hpp:601-673). Returns a dict with the VerificationReport fields."""
        m = n - l + 1
        per_b = np.zeros(bhi - blo + 1)
        per_n = np.zeros(m)
        od = np.zeros(5)
        oi = np.zeros(5, np.int32)
        self._check(self._fn("verify")(n, l, dn, blo, bhi, np.ascontiguousarray(v, np.float64),
                                                    design_delta, grid_points, facets, dense, delta_e,
                                                    per_b, per_n, od, oi))
        return dict(delta=od[0], passband_max=od[1], stopband_max=od[2], worst_omega=od[3],
                    refinement_bound=od[4], dense_points=int(oi[0]), worst_b=int(oi[1]), worst_n=int(oi[2]),
                    passed=bool(oi[3]), within_bound=bool(oi[4]), per_b_max=per_b, per_n_max=per_n)

    def solve_minimax(self, n, l, dn, blo, bhi, grid_k, facets=16, exchange_tol=0.025, max_rounds=60,
                      seed_stride=16):
        """solve_minimax (design.hpp:276-446); reference only."""
        v = np.zeros(dn - 1)
        od = np.zeros(2)
        oi = np.zeros(3, np.int64)
        self._check(self.lib.ref_solve_minimax(n, l, dn, blo, bhi, grid_k, facets, exchange_tol, max_rounds,
                                               seed_stride, v, od, oi))
        return dict(v=v, delta=od[0], lp_delta=od[1], rounds=int(oi[0]), lp_iterations=int(oi[1]),
                    active_triples=int(oi[2]))

    def design_full(self, spec, fft_length_override=0, filter_length_override=0, grid_points=1000, facets=16,
                    max_rounds=60, seed_stride=16, exchange_tol=0.025, margin=0.5):
        """design() with the order loop (design.hpp:486-577); spec = 6 floats as FilterSpec. Reference only."""
        geo = np.zeros(8, np.int32)
        v = np.zeros(256)
        d = np.zeros(1)
        self._check(self.lib.ref_design_full(np.asarray(spec, np.float64),
                                             np.array([fft_length_override, filter_length_override, grid_points,
                                                       facets, max_rounds, seed_stride], np.int32),
                                             np.array([exchange_tol, margin]), geo, v, 256, d))
        return dict(N=int(geo[0]), L=int(geo[1]), M=int(geo[2]), delta_N=int(geo[3]), b_low=int(geo[4]),
                    b_high=int(geo[5]), iterations=int(geo[6]), exchange_rounds=int(geo[7]),
                    v=v[:geo[3] - 1].copy(), delta=float(d[0]))

    def shift_rule(self, n, l, dn, blo, bhi):
        """calibrated_shift_rule (design.hpp:476-484) -> (window_offset, step); reference only."""
        wo = np.zeros(1, np.int32)
        st = np.zeros(1, np.int32)
        self._check(self.lib.ref_shift_rule(n, l, dn, blo, bhi, wo, st))
        return int(wo[0]), int(st[0])


_cache: dict = {}


def port() -> _Lib:
    """The C restatement (always available after build())."""
    if "port" not in _cache:
        _cache["port"] = _Lib(ORACLE_SO, "orc_", "port")
    return _cache["port"]


def reference() -> _Lib:
    """The reference headers compiled in place (oracle/_ref)."""
    if "ref" not in _cache:
        _cache["ref"] = _Lib(REF_SO, "ref_", "reference")
    return _cache["ref"]


def have_reference() -> bool:
    return os.path.exists(REF_SO)


def best() -> _Lib:
    return reference() if have_reference() else port()


def rel_rms(y, y_ref) -> float:
    y = np.asarray(y, np.complex128 if np.iscomplexobj(y) else np.float64)
    y_ref = np.asarray(y_ref)
    num = np.sum(np.abs(y - y_ref) ** 2)
    den = np.sum(np.abs(y_ref) ** 2)
    return float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num))
