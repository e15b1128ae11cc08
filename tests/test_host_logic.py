"""CPU: host-side logic — domain-model validation (vs the reference rules), artifact / schedule /
signal formats, sharding plans, workload generators, and the C-ABI surface (loads and exports every
symbol include/fcvbw_gpu.h declares; validation errors are reported without touching a GPU)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_14116_b200 import (BinSpec, Error, ValidationError, artifact_from_json, load_artifact,
                                   read_schedule_csv, read_signal, save_artifact, schedule_to_blocks,
                                   transition_bins, write_signal)
from paper_2406_14116_b200 import _lib
from paper_2406_14116_b200.io import artifact_to_json
from paper_2406_14116_b200.shard import block_shards, channel_shards, check_cover
from paper_2406_14116_b200.workload import SeededRng, complex_gaussian, config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- BinSpec
def test_binspec_validate_matches_oracle_rules():
    rng = SeededRng(11)
    port = O.port()
    for _ in range(400):
        n = 1 << rng.uniform_int(2, 8)
        if rng.uniform01() < 0.1:
            n += 1
        l = rng.uniform_int(0, n + 1)
        m = n - l + 1 + (1 if rng.uniform01() < 0.1 else 0)
        dn = rng.uniform_int(1, max(1, n // 2))
        blo = rng.uniform_int(0, n // 2)
        bhi = rng.uniform_int(0, n // 2)
        bins = BinSpec(n, l, m, dn, blo, bhi)
        try:
            bins.validate()
            ok = 0
        except ValidationError:
            ok = 2
        assert ok == port.validate(n, l, m, dn, blo, bhi, dn - 1), bins


def test_transition_bins_kat():
    bins = BinSpec(128, 33, 96, 16, 48, 55)
    tb = transition_bins(bins, 48)
    assert (tb.k1, tb.k2) == (41, 55)
    tb = transition_bins(bins, 55)
    assert (tb.k1, tb.k2) == (48, 62)
    for bad in (47, 56):
        with pytest.raises(ValidationError):
            transition_bins(bins, bad)


# ---------------------------------------------------------------- artifacts / schedule / signals
def test_config_artifacts_load_and_validate():
    arts = [f for f in os.listdir(os.path.join(ROOT, "configs")) if f.startswith("artifact_")]
    assert len(arts) >= 9
    for f in arts:
        res = load_artifact(os.path.join(ROOT, "configs", f))
        assert res.profile.length() == res.bins.profile_length()
        assert res.bins.filter_length - 1 == res.bins.fft_length // 4
        assert np.all(np.isfinite(res.profile.values))


def test_artifact_roundtrip(tmp_path):
    res = load_artifact(os.path.join(ROOT, "configs", "artifact_n1024_d12.json"))
    p = tmp_path / "a.json"
    save_artifact(str(p), res)
    back = load_artifact(str(p))
    assert back.bins == res.bins and back.profile.values == res.profile.values
    j = artifact_to_json(res)
    j["V"] = j["V"][:-1]
    with pytest.raises(ValidationError):
        artifact_from_json(j)
    j = artifact_to_json(res)
    del j["M"]
    with pytest.raises(Error):
        artifact_from_json(j)


def test_schedule_csv_semantics(tmp_path):
    p = tmp_path / "s.csv"
    p.write_text("# comment\n0,48\n\n40,55\n80,50\n")
    assert read_schedule_csv(str(p)) == [(0, 48), (40, 55), (80, 50)]
    p.write_text("0,48\n40,55\n40,50\n")
    with pytest.raises(ValidationError):
        read_schedule_csv(str(p))
    p.write_text("0;48\n")
    with pytest.raises(ValidationError):
        read_schedule_csv(str(p))
    p.write_text("-1,48\n")
    with pytest.raises(ValidationError):
        read_schedule_csv(str(p))
    bins = BinSpec(128, 33, 96, 16, 48, 55)
    ev = [(0, 48), (3, 55), (5, 50)]
    assert list(schedule_to_blocks(ev, 7, 49, bins)) == [48, 48, 48, 55, 55, 50, 50]
    assert list(schedule_to_blocks([(2, 51)], 4, 49, bins)) == [49, 49, 51, 51]
    with pytest.raises(ValidationError):
        schedule_to_blocks([(1, 56)], 4, 49, bins)   # out of design range (exit 2 in the CLI)
    with pytest.raises(ValidationError):
        schedule_to_blocks([(4, 50)], 4, 49, bins)   # beyond the stream


def test_signal_formats(tmp_path):
    x = np.array([0.0, -1.5, 1e-310, 3.141592653589793, -2.5e300])
    for fmt in ("csv", "f64le"):
        p = tmp_path / f"x.{fmt}"
        write_signal(str(p), x, fmt)
        assert np.array_equal(read_signal(str(p), fmt), x)
    p = tmp_path / "bad.csv"
    p.write_text("1.0\n2.0 x\n")
    with pytest.raises(ValidationError):
        read_signal(str(p), "csv")
    p = tmp_path / "bad.f64"
    p.write_bytes(b"1234567")
    with pytest.raises(ValidationError):
        read_signal(str(p), "f64le")


# ---------------------------------------------------------------- sharding plans
@pytest.mark.parametrize("S,N,M,world", [(2 ** 20, 1024, 768, 8), (2 ** 31, 4096, 3072, 8), (1000, 32, 8, 3),
                                         (5, 64, 48, 4), (768 * 7, 1024, 768, 8)])
def test_block_shards_cover(S, N, M, world):
    sh = block_shards(S, N, M, world)
    check_cover(sh, S)
    for s in sh:
        if s.blk_end > s.blk_begin:
            assert s.halo == min(N - M, s.y_begin)
            assert s.x_end == s.y_end
    sizes = [s.blk_end - s.blk_begin for s in sh]
    assert max(sizes) - min(sizes) <= 1


def test_channel_shards():
    sh = channel_shards(1024, 8)
    assert [s.ch_end - s.ch_begin for s in sh] == [128] * 8
    sh = channel_shards(5, 3)
    assert [(s.ch_begin, s.ch_end) for s in sh] == [(0, 2), (2, 4), (4, 5)]


def test_sharded_oracle_is_bitwise_unsharded():
    """The sharding rule itself, checked on the CPU oracle: every shard computed separately from its
    halo-extended input slice reproduces the unsharded output bit for bit."""
    port = O.port()
    n, l, dn = 256, 65, 6
    m = n - l + 1
    v = np.array(SeededRng(5).__class__(5).uniform(0, 1) for _ in range(1)) if False else \
        np.array([SeededRng(5 + i).uniform(0.0, 1.0) for i in range(dn - 1)])
    S = m * 37 + 11
    x = port.rng_uniform(9, -1.0, 1.0, S)
    nb = (S + m - 1) // m
    sched = port.rng_uniform_int(10, 3, 124, nb)
    full = port.ols_real(n, l, dn, 3, 124, v, x, bsched=sched)
    for world in (2, 3, 5):
        out = np.zeros(S)
        for s in block_shards(S, n, m, world):
            if s.blk_end == s.blk_begin:
                continue
            # shard-local stream: the halo-extended slice, zero history before it (global index < 0
            # is zero exactly when the shard starts at block 0)
            xs = x[s.x_begin:s.x_end]
            pre = s.y_begin - s.x_begin
            # run the slice as its own stream with a leading pad so block boundaries line up
            pad = (m - pre % m) % m
            xs2 = np.concatenate([np.zeros(pad), xs])
            lead_blocks = (pad + pre) // m
            sched2 = np.concatenate([np.full(lead_blocks, sched[s.blk_begin]), sched[s.blk_begin:s.blk_end]])
            sched2 = sched2[: (xs2.size + m - 1) // m].astype(np.int32)
            ys = port.ols_real(n, l, dn, 3, 124, v, xs2, bsched=sched2)
            out[s.y_begin:s.y_end] = ys[pad + pre: pad + pre + (s.y_end - s.y_begin)]
        assert np.array_equal(out, full), world


# ---------------------------------------------------------------- workload generators
def test_workload_determinism_and_moments():
    a = complex_gaussian(1, 0, 50000)
    b = complex_gaussian(1, 1000, 1000)
    assert np.array_equal(a[1000:2000], b)
    assert abs(np.mean(np.abs(a) ** 2) - 1.0) < 0.03
    assert abs(np.mean(a.real)) < 0.02 and abs(np.mean(a.imag)) < 0.02


def test_baseline_configs_materialize():
    w = config("c2")
    sch = w.b_schedule()
    assert w.bins.fft_length == 1024 and w.bins.block_length == 768 and w.bins.transition_width_bins == 12
    assert sch.size == w.nblocks == 21846
    assert np.all(sch[:64] == sch[0]) and len(set(sch[::64].tolist())) > 100
    assert sch.min() >= w.b_lo and sch.max() <= w.b_hi
    assert w.b_lo == 26 and w.b_hi == 460
    c1 = config("c1")
    assert c1.bins.fft_length == 512 and c1.b_lo == c1.b_hi == 64 and c1.dtype == "c128"
    c3 = config("c3", samples=768 * 4)
    s3 = c3.b_schedule()
    assert s3.shape == (1024, 4) and np.all(s3[:, 0] == s3[:, 3])
    c4 = config("c4", samples=3072 * 600)
    s4 = c4.b_schedule()
    assert np.all(s4[:256] == s4[0]) and s4.min() >= c4.b_lo and s4.max() <= c4.b_hi
    for n in (64, 128, 256, 512, 1024, 2048, 4096, 8192):
        c5 = config(f"c5_{n}_f32", samples=(3 * n // 4) * 3, channels=2)
        s5 = c5.b_schedule()
        assert s5.shape == (2, 3) and s5.min() >= c5.bins.transition_width_bins // 2


# ---------------------------------------------------------------- C-ABI surface (no GPU needed)
def test_cabi_exports_every_declared_symbol():
    lib = _lib.lib()
    declared = _lib.header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
    assert lib.fcvbw_gpu_version().decode().startswith("fcvbw_gpu")


def _cfg(**kw):
    v = np.linspace(0.1, 0.9, 15)
    d = dict(fft_length=128, filter_length=33, block_length=96, transition_width_bins=16, b_low=48, b_high=55,
             profile=v.ctypes.data_as(C.POINTER(C.c_double)), profile_length=15, initial_b=48, dtype=_lib.C128,
             device=0, flags=0)
    d.update(kw)
    return _lib.Config(**d), v


@pytest.mark.parametrize("bad", [dict(fft_length=100), dict(block_length=95), dict(transition_width_bins=15),
                                 dict(b_low=7), dict(b_high=56), dict(profile_length=14), dict(initial_b=56),
                                 dict(filter_length=0), dict(dtype=7)])
def test_cabi_create_validation_is_status_2(bad):
    cfg, _keep = _cfg(**bad)
    h = C.c_void_p()
    rc = _lib.lib().fcvbw_gpu_create(C.byref(cfg), C.byref(h))
    assert rc == _lib.VALIDATION, (bad, rc, _lib.last_error())
    assert h.value is None
    assert _lib.last_error()


def test_cabi_raw_validation_and_null_handles():
    L = _lib.lib()
    h = C.c_void_p()
    t = np.zeros(2 * 12)
    assert L.fcvbw_gpu_create_raw(12, 4, t.ctypes.data_as(C.POINTER(C.c_double)), 1, 0, C.byref(h)) == 2
    t = np.zeros(2 * 16)
    assert L.fcvbw_gpu_create_raw(16, 17, t.ctypes.data_as(C.POINTER(C.c_double)), 1, 0, C.byref(h)) == 2
    assert L.fcvbw_gpu_set_bandwidth(None, 3) == 2
    assert L.fcvbw_gpu_block_length(None) == -1


def test_cabi_no_cpu_fallback_without_gpu():
    """On a host without a CUDA device a VALID configuration fails loudly (status 1)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("CUDA device present")
    except Exception:
        pass
    cfg, _keep = _cfg()
    h = C.c_void_p()
    rc = _lib.lib().fcvbw_gpu_create(C.byref(cfg), C.byref(h))
    assert rc == _lib.ERROR
    assert "CUDA" in _lib.last_error()


def test_glibc_hypot_restatement():
    """The device restatement of glibc's hypot (csrc/response.cuh glibc_hypot) follows this
    formula; pin the formula itself against the host libm (the reference's std::abs)."""
    import ctypes
    import math
    import random
    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]

    def kernel(ax, ay):
        h = math.sqrt(ax * ax + ay * ay)
        if h <= 2.0 * ay:
            d = h - ay
            t1 = ax * (2.0 * d - ax)
            t2 = (d - 2.0 * (ax - ay)) * d
        else:
            d = h - ax
            t1 = 2.0 * d * (ax - 2.0 * ay)
            t2 = (4.0 * d - ay) * ay + d * d
        return h - (t1 + t2) / (2.0 * h)

    def hyp(x, y):
        x, y = abs(x), abs(y)
        ax, ay = max(x, y), min(x, y)
        if ay <= ax * 2.0 ** -54:
            return ax + ay
        return kernel(ax, ay)

    rng = random.Random(7)
    for _ in range(20000):
        x = rng.uniform(-1, 1) * 10 ** rng.uniform(-6, 2)
        y = rng.uniform(-1, 1) * 10 ** rng.uniform(-6, 2)
        assert hyp(x, y) == libm.hypot(x, y), (x, y)
