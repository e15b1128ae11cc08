"""Design analysis on the GPU.

Mirrors the reference's analysis surface: ``FrequencyGrid`` (proj/include/fcvbw/ptvir.hpp:309-343),
``ptvir_from_base`` tables (ptvir.hpp:147-160), ``error_on_grid`` / ``ErrorMatrix``
(ptvir.hpp:391-431) and the ``fcvbw analyze`` tables (proj/tools/fcvbw_cli.cpp:120-193; CSV writers
io.hpp:25-29,251-260). The responses H_n(omega) of all M phases at every (b, omega) are computed by
``libfcvbw_gpu.so`` (csrc/analyze.cu) in the reference's operation order; this module only lays the
results out and writes the files.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .bins import DesignResult, Error, ValidationError
from .engine import _raise
from .verify import OLS_SHIFT_STEP


def _design_struct(result: DesignResult):
    bins = result.bins
    v = np.ascontiguousarray(result.profile.values, dtype=np.float64)
    d = _lib.Design(bins.fft_length, bins.filter_length, bins.block_length, bins.transition_width_bins, bins.b_low,
                    bins.b_high, v.ctypes.data_as(C.POINTER(C.c_double)), len(v), float(result.delta),
                    int(result.grid_points), int(result.facets))
    return d, v  # keep v alive with the struct


@dataclass
class FrequencyGrid:
    """FrequencyGrid (ptvir.hpp:309-343): sorted omegas on [0, pi] with every band edge inserted."""
    omega: np.ndarray
    base_points: int
    result: DesignResult

    def region(self, b: int) -> np.ndarray:
        """0 passband (omega <= pass edge), 1 stopband (>= stop edge), 2 excluded."""
        bins = self.result.bins
        half = bins.transition_width_bins // 2
        pe, se = bins.omega_of_bin(b - half), bins.omega_of_bin(b + half)
        return np.where(self.omega <= pe, 0, np.where(self.omega >= se, 1, 2)).astype(np.int8)

    def size(self) -> int:
        return int(self.omega.size)


def frequency_grid(result: DesignResult, grid_points: int) -> FrequencyGrid:
    d, keep = _design_struct(result)
    size = C.c_int64(0)
    _raise(_lib.lib().fcvbw_gpu_frequency_grid(C.byref(d), int(grid_points), None, 0, C.byref(size)))
    om = np.zeros(size.value)
    _raise(_lib.lib().fcvbw_gpu_frequency_grid(C.byref(d), int(grid_points), om.ctypes.data, om.size,
                                               C.byref(size)))
    return FrequencyGrid(om, int(grid_points), result)


def ptvir(result: DesignResult, b: int, device: int = 0) -> np.ndarray:
    """The M x N PTVIR table of band centre b (ptvir_from_base(base_response_idft(...)))."""
    d, keep = _design_struct(result)
    rows = np.zeros((result.bins.block_length, result.bins.fft_length))
    _raise(_lib.lib().fcvbw_gpu_ptvir(C.byref(d), int(b), OLS_SHIFT_STEP, int(device), rows.ctypes.data))
    return rows


@dataclass
class ResponseTable:
    """Per (b, omega) over the M phases: max / min |H_n|, max |E_n| (NaN when excluded); optional
    per-phase |H_n| and |E_n| with shape [nb][K'][M]."""
    b: list
    grid: FrequencyGrid
    h_max: np.ndarray
    h_min: np.ndarray
    e_max: np.ndarray
    abs_h: np.ndarray | None = None
    abs_e: np.ndarray | None = None


def response_table(result: DesignResult, grid_points: int, b_list, per_phase: bool = False,
                   device: int = 0) -> ResponseTable:
    grid = frequency_grid(result, grid_points)
    bs = np.ascontiguousarray(np.asarray(b_list, dtype=np.int32).ravel())
    kk, m = grid.size(), result.bins.block_length
    h_max, h_min, e_max = (np.zeros((bs.size, kk)) for _ in range(3))
    abs_h = np.zeros((bs.size, kk, m)) if per_phase else None
    abs_e = np.zeros((bs.size, kk, m)) if per_phase else None
    d, keep = _design_struct(result)
    _raise(_lib.lib().fcvbw_gpu_analyze(C.byref(d), int(grid_points), bs.ctypes.data, int(bs.size), OLS_SHIFT_STEP,
                                        int(device), h_max.ctypes.data, h_min.ctypes.data, e_max.ctypes.data,
                                        abs_h.ctypes.data if per_phase else None,
                                        abs_e.ctypes.data if per_phase else None))
    return ResponseTable(bs.tolist(), grid, h_max, h_min, e_max, abs_h, abs_e)


@dataclass
class ErrorMatrix:
    """ErrorMatrix (ptvir.hpp:391-400): masked grid indices and |E| as [M][points]."""
    point_index: np.ndarray
    abs_error: np.ndarray
    max_abs: float = 0.0
    worst_n: int = -1
    worst_omega: float = 0.0
    extra: dict = field(default_factory=dict)

    def at(self, n: int, j: int) -> float:
        return float(self.abs_error[n, j])


def error_on_grid(result: DesignResult, grid_points: int, b: int, device: int = 0) -> ErrorMatrix:
    """error_on_grid (ptvir.hpp:402-431) for the design's own PTVIR set at band centre b."""
    if not result.bins.contains_b(b):
        raise ValidationError("error_on_grid: b outside the design range")
    t = response_table(result, grid_points, [b], per_phase=True, device=device)
    region = t.grid.region(b)
    idx = np.nonzero(region != 2)[0].astype(np.int64)
    err = np.ascontiguousarray(t.abs_e[0][idx].T)  # [M][points]
    out = ErrorMatrix(idx, err)
    if idx.size:
        flat = err.T.ravel()  # point-major, phase-minor: the reference's scan order
        k = int(np.argmax(flat))  # first occurrence of the maximum
        if flat[k] > 0.0:
            m = result.bins.block_length
            out.max_abs = float(flat[k])
            out.worst_n = k % m
            out.worst_omega = float(t.grid.omega[idx[k // m]])
    return out


def _fmt(v: float) -> str:
    """format_double (io.hpp:25-29): printf %.17g."""
    return "%.17g" % v


def analyze(artifact_path: str, grid_k: int = 1000, b_arg: str = "all", prefix: str = "analysis",
            per_phase: bool = False, device: int = 0) -> str:
    """cmd_analyze (fcvbw_cli.cpp:120-193): <prefix>_profile.csv, <prefix>_response.csv,
    <prefix>_ptvir_<b>.csv per band centre, and <prefix>_phases.csv with per_phase."""
    from .io import load_artifact
    result = load_artifact(artifact_path)
    bins = result.bins
    if b_arg == "all":
        bs = list(range(bins.b_low, bins.b_high + 1))
    else:
        from .io import _INT
        m = _INT.match(b_arg)  # std::stoi semantics: leading integer prefix, else an error (exit 1)
        if m is None:
            raise Error(f"analyze: invalid --b value '{b_arg}'")
        bs = [int(m.group(0))]
        if not bins.contains_b(bs[0]):
            raise ValidationError("analyze: b_N outside the design range")
    frequency_grid(result, grid_k)  # FrequencyGrid::build validation before any file is written
    with open(prefix + "_profile.csv", "w") as f:
        f.write("r,V\n")
        for r, v in enumerate(result.profile.values):
            f.write(f"{r},{_fmt(v)}\n")
    t = response_table(result, grid_k, bs, per_phase=per_phase, device=device)
    om_pi = [_fmt(w / math.pi) for w in t.grid.omega]
    names = {0: "pass", 1: "stop", 2: "transition"}
    m = bins.block_length
    resp = open(prefix + "_response.csv", "w")
    resp.write("b_N,omega_over_pi,region,abs_Hn_max,abs_Hn_min,abs_En_max\n")
    phases = open(prefix + "_phases.csv", "w") if per_phase else None
    if phases:
        phases.write("b_N,n,omega_over_pi,abs_Hn,abs_En\n")
    for i, b in enumerate(bs):
        rows = ptvir(result, b, device)
        with open(f"{prefix}_ptvir_{b}.csv", "w") as pt:
            pt.write("".join(",".join(_fmt(x) for x in row) + "\n" for row in rows))
        region = t.grid.region(b)
        out = []
        for g in range(t.grid.size()):
            masked = region[g] != 2
            if phases:
                ah, ae = t.abs_h[i, g], t.abs_e[i, g]
                phases.write("".join(f"{b},{n},{om_pi[g]},{_fmt(ah[n])},{_fmt(ae[n]) if masked else ''}\n"
                                     for n in range(m)))
            out.append(f"{b},{om_pi[g]},{names[int(region[g])]},{_fmt(t.h_max[i, g])},{_fmt(t.h_min[i, g])},"
                       f"{_fmt(t.e_max[i, g]) if masked else ''}\n")
        resp.write("".join(out))
    resp.close()
    if phases:
        phases.close()
    msg = f"analyze: wrote {prefix}_response.csv, {prefix}_profile.csv and {len(bs)} PTVIR table(s)"
    print(msg)
    return msg
