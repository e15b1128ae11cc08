"""Round-2 GPU checks of the production kernel itself and of the new entry points.

* The spectral mask the PRODUCTION fused kernel applies (fcvbw_gpu_mask_dump: the same
  instantiation fcvbw_gpu_run launches, with its dump pointer set) equals the reference's
  magnitude_samples(b) / N (proj/include/fcvbw/spectrum.hpp:170-192) rounded to the engine type,
  bit for bit, for every plan (N = 8 ... 8192, fp32 and fp64), the three coefficient modes
  (L - 1 = N/4, general odd L, even L) and both region generators (one transition register per
  half-spectrum, and the general rule when delta_N - 2 >= threads per block), including every b of
  the C2 schedule.
* Real-valued streaming (fcvbw_gpu_feed_real ...): bit-identical to the complex path on x + 0j and
  invariant to caller batching (test_oracle_engine.cpp:268-288).
* Construction-time self-check (check_provider, engine.hpp:126-137) with fault injection.
* Op tallies (OpCounters, test_oracle_engine.cpp:216-240).
* The device workload generator against the host generator.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_14116_b200 import BinSpec, OlsEngine, TransitionProfile, ValidationError, _lib
from paper_2406_14116_b200.workload import SeededRng, complex_gaussian, config

pytestmark = pytest.mark.gpu


def _profile(n, seed):
    rng = SeededRng(seed)
    return [rng.uniform(0.0, 1.0) for _ in range(n)]


def _expected(bins, v, b_list, dtype):
    lib = O.best()
    n = bins.fft_length
    rdt = np.float32 if dtype == "c64" else np.float64
    rows = []
    for b in b_list:
        mag, _, _ = lib.coefficients(n, bins.filter_length, bins.transition_width_bins, bins.b_low, bins.b_high,
                                     np.array(v), int(b))
        rows.append((mag * (1.0 / n)).astype(rdt).astype(np.float64))
    return np.array(rows)


def _b_list(lo, hi, cap=160):
    bl = np.arange(lo, hi + 1)
    if bl.size > cap:
        bl = np.unique(np.r_[bl[:8], bl[-8:], bl[np.linspace(0, bl.size - 1, cap - 16).astype(int)]])
    return bl.astype(np.int32)


GEOMS = []
for _n in (8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192):
    _dn = max(2, min(32, 2 * (_n // 64)))
    GEOMS.append((_n, _n // 4 + 1, _dn))          # BASELINE geometry (index-rotation phase)
    if _n >= 32:
        GEOMS.append((_n, _n // 2 + 1, _dn))      # general odd L (shift at the store)
        GEOMS.append((_n, _n // 4, _dn))          # even L (explicit phase-table multiply)
GEOMS += [(64, 17, 12), (128, 33, 20), (1024, 257, 40)]  # delta_N - 2 >= threads per block: general rule


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,l,dn", GEOMS)
def test_production_mask_bit_exact(n, l, dn, dtype):
    half = dn // 2
    bins = BinSpec(n, l, n - l + 1, dn, half, n // 2 - half - 1)
    if bins.b_low > bins.b_high:
        pytest.skip("no admissible b")
    v = _profile(dn - 1, 1000 + n + dn)
    eng = OlsEngine(bins, TransitionProfile(v), bins.b_low, dtype=dtype)
    bl = _b_list(bins.b_low, bins.b_high)
    g = eng.mask_dump(bl)
    want = _expected(bins, v, bl, dtype)
    bad = np.argwhere(g != want)
    assert bad.size == 0, (f"{bad.shape[0]} bins differ; first (b={bl[bad[0][0]]}, k={bad[0][1]}): "
                           f"{g[tuple(bad[0])]!r} vs {want[tuple(bad[0])]!r}")
    # the parity dump kernel's region rule agrees with the production mask's zero / one / V split
    region, vidx, _ = eng.coeff_dump(bl)
    inv_n = np.float64(np.float32(1.0 / n)) if dtype == "c64" else 1.0 / n
    assert np.array_equal(region == 0, g == inv_n) or dn - 1 == 0


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_production_mask_every_c2_b(dtype):
    w = config("c2")
    sched = w.b_schedule()
    bl = np.unique(sched).astype(np.int32)
    eng = OlsEngine(w.bins, w.design.profile, int(sched[0]), dtype=dtype)
    assert np.array_equal(eng.mask_dump(bl), _expected(w.bins, w.design.profile.values, bl, dtype))


def test_real_streaming_bitwise_equals_complex_path():
    import torch
    bins = BinSpec(1024, 257, 768, 12, 6, 505)
    v = _profile(11, 5)
    x = np.array([SeededRng(9).uniform(-1.0, 1.0) for _ in range(768 * 9 + 123)])
    one = OlsEngine(bins, TransitionProfile(v), 77)
    y1 = np.concatenate([one.feed(x), one.flush()])
    drip = OlsEngine(bins, TransitionProfile(v), 77)
    parts = [drip.feed(x[i:i + 500]) for i in range(0, x.size, 500)]
    y2 = np.concatenate(parts + [drip.flush()])
    assert np.array_equal(y1, y2)  # batching invariance
    blk = OlsEngine(bins, TransitionProfile(v), 77)
    y3 = np.concatenate([blk.process_block(x[i:i + 768]) for i in range(0, 768 * 9, 768)] +
                        [blk.feed(x[768 * 9:]), blk.flush()])
    assert np.array_equal(y1, y3)
    yc = one.run(torch.from_numpy(x.astype(np.complex128)).cuda()).cpu().numpy()
    assert np.array_equal(y1, yc.real)  # bit-identical to the complex path on x + 0j
    yr = O.best().ols_real(1024, 257, 12, 6, 505, np.array(v), x, b0=77)
    assert np.max(np.abs(y1 - yr)) <= 1e-12
    with pytest.raises(ValidationError):  # a real stream cannot continue as complex
        one.feed(np.ones(10, np.complex128))
    one.reset()
    assert one.feed(np.ones(768, np.complex128)).size == 768


def test_real_streaming_fp32_engine():
    bins = BinSpec(512, 129, 384, 8, 4, 251)
    v = _profile(7, 6)
    x = np.array([SeededRng(10).uniform(-1.0, 1.0) for _ in range(384 * 7 + 5)])
    e = OlsEngine(bins, TransitionProfile(v), 64, dtype="c64")
    y = np.concatenate([e.feed(x), e.flush()])
    yr = O.best().ols_real(512, 129, 8, 4, 251, np.array(v), x.astype(np.float32).astype(np.float64), b0=64)
    assert O.rel_rms(y, yr) <= 2e-6


@pytest.mark.parametrize("dtype", [_lib.C64, _lib.C128])
def test_self_check_rejects_corrupted_twiddles(dtype):
    v = (C.c_double * 11)(*_profile(11, 3))
    cfg = _lib.Config(1024, 257, 768, 12, 6, 505, C.cast(v, C.POINTER(C.c_double)), 11, 77, dtype, 0,
                      _lib.TEST_CORRUPT_TWIDDLES)
    h = C.c_void_p()
    rc = _lib.lib().fcvbw_gpu_create(C.byref(cfg), C.byref(h))
    assert rc == _lib.VALIDATION and not h.value
    assert "round-trip" in _lib.last_error()
    cfg.flags = 0
    assert _lib.lib().fcvbw_gpu_create(C.byref(cfg), C.byref(h)) == _lib.OK
    _lib.lib().fcvbw_gpu_destroy(h)


def test_op_counts():
    """AC8 (test_oracle_engine.cpp:216-240): 2 L_V variable multiplications per real block, none
    per retune; a complex block counts as two real streams."""
    import torch
    bins = BinSpec(128, 33, 96, 16, 48, 55)
    e = OlsEngine(bins, TransitionProfile(_profile(15, 62)), 51)
    block = np.full(96, 0.5)
    e.process_block(block)
    c0 = e.op_counts()
    for _ in range(5):
        e.process_block(block)
    c1 = e.op_counts()
    assert c1["variable_mul"] - c0["variable_mul"] == 5 * 30 and c1["real_blocks"] - c0["real_blocks"] == 5
    e.set_bandwidth(55)
    e.set_bandwidth(48)
    assert e.op_counts() == c1 and c1["retune_flops"] == 0
    x = torch.zeros((3, 96 * 4 + 1), dtype=torch.complex128, device="cuda")
    e.run(x)
    c2 = e.op_counts()
    assert c2["complex_blocks"] - c1["complex_blocks"] == 3 * 5
    assert c2["variable_mul"] - c1["variable_mul"] == 3 * 5 * 4 * 15


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_device_generator_matches_host(dtype):
    import torch
    from paper_2406_14116_b200.engine import fill_gaussian
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    x = torch.empty((3, 50000), dtype=tdt, device="cuda")
    fill_gaussian(x, 2 * 1_000_003, ch_first=5, start=1000)
    xd = x.cpu().numpy().astype(np.complex128)
    npdt = np.complex64 if dtype == "c64" else np.complex128
    for c in range(3):
        xh = complex_gaussian(2 * 1_000_003 + 5 + c, 1000, 50000, npdt).astype(np.complex128)
        rel = np.max(np.abs(xd[c] - xh)) / np.max(np.abs(xh))
        assert rel <= (2e-7 if dtype == "c64" else 1e-14), rel
    assert abs(np.mean(np.abs(xd) ** 2) - 1.0) < 0.02
