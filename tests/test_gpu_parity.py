"""GPU parity suite (checks P1-P12): the fused sm_100a kernel, through the
C-ABI, against the reference compiled in place (oracle/_ref) — or the C restatement when the
reference build is absent — on identical seeded inputs.

Tolerances (BASELINE.json north_star): relative RMS <= 1e-12 in fp64 mode, <= 2e-6 in fp32 mode
(the fp32 oracle input is the exact fp32 samples promoted to double); coefficient masks bit-exact.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_14116_b200 import BinSpec, OlsEngine, TransitionProfile, ValidationError
from paper_2406_14116_b200.workload import SeededRng, complex_gaussian

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 2e-6}
ALL_N = [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]


def ref():
    return O.best()


def _uniforms(seed, n, lo, hi):
    r = SeededRng(seed)
    return [r.uniform(lo, hi) for _ in range(n)]


def narrowband():
    # validate_and_discretize(narrowband_spec(), 128, 33) (test_spectrum.cpp:18-25)
    return BinSpec(128, 33, 96, 16, 48, 55)


def geometry(n, dn=None, seed=0):
    dn = dn or max(2, 2 * (n // 64))
    l = n // 4 + 1
    return BinSpec(n, l, n - l + 1, dn, dn // 2, n // 2 - dn // 2 - 1)


def rand_sched(bins, nb, seed, every=1):
    r = SeededRng(seed)
    segs = (nb + every - 1) // every
    d = [r.uniform_int(bins.b_low, bins.b_high) for _ in range(segs)]
    return np.repeat(np.array(d, np.int32), every)[:nb]


def run_gpu(bins, v, x, sched, dtype, **kw):
    import torch
    eng = OlsEngine(bins, TransitionProfile(list(v)), int(np.ravel(sched)[0]), dtype=dtype, **kw)
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    xd = torch.from_numpy(np.ascontiguousarray(x)).to("cuda", tdt)
    bd = torch.from_numpy(np.ascontiguousarray(sched, np.int32)).cuda()
    y = eng.run(xd, bd)
    torch.cuda.synchronize()
    return y.cpu().numpy(), eng


def oracle_complex(bins, v, x, sched):
    b = bins
    return ref().ols_complex(b.fft_length, b.filter_length, b.transition_width_bins, b.b_low, b.b_high, v,
                             np.asarray(x, np.complex128), bsched=sched)


# ---------------------------------------------------------------- P4 / P5 / P7 sweep
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n", ALL_N)
def test_complex_sweep_vs_reference(n, dtype):
    bins = geometry(n)
    v = np.array(_uniforms(100 + n, bins.profile_length(), 0.0, 1.0))
    m = bins.block_length
    S = m * max(6, 12000 // m) + (m // 2 + 3)  # partial tail
    x = complex_gaussian(n, 0, S, np.complex64 if dtype == "c64" else np.complex128)
    nb = (S + m - 1) // m
    sched = rand_sched(bins, nb, n, every=3)
    y, _ = run_gpu(bins, v, x, sched, dtype)
    yr = oracle_complex(bins, v, x, sched)
    err = O.rel_rms(y, yr)
    assert err <= TOL[dtype], (n, dtype, err)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_multichannel_per_channel_schedules(dtype):
    bins = geometry(1024, 12)
    v = np.array(_uniforms(7, 11, 0.0, 1.0))
    ch, S = 5, 768 * 9 + 100
    x = np.stack([complex_gaussian(50 + c, 0, S) for c in range(ch)]).astype(
        np.complex64 if dtype == "c64" else np.complex128)
    nb = (S + 767) // 768
    sched = np.stack([rand_sched(bins, nb, 90 + c, every=2) for c in range(ch)])
    y, _ = run_gpu(bins, v, x, sched, dtype)
    yr = ref().ols_complex(1024, 257, 12, bins.b_low, bins.b_high, v, x.astype(np.complex128), bsched=sched)
    assert O.rel_rms(y, yr) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_phase_multiply_mode_matches(dtype):
    """Explicit phase_table multiply (COEF_PHASE) equals the exact-delay path and the reference."""
    bins = geometry(512, 8)
    v = np.array(_uniforms(9, 7, 0.0, 1.0))
    S = 384 * 20 + 17
    x = complex_gaussian(3, 0, S, np.complex64 if dtype == "c64" else np.complex128)
    sched = rand_sched(bins, (S + 383) // 384, 4, every=5)
    y1, _ = run_gpu(bins, v, x, sched, dtype)
    y2, _ = run_gpu(bins, v, x, sched, dtype, force_phase_multiply=True)
    yr = oracle_complex(bins, v, x, sched)
    assert O.rel_rms(y1, yr) <= TOL[dtype]
    assert O.rel_rms(y2, yr) <= TOL[dtype]


def test_even_filter_length_uses_phase_table():
    """L even: the phase table is not a pure delay above N/2 (conj mirror); COEF_PHASE path."""
    bins = BinSpec(64, 20, 45, 6, 3, 28)
    v = np.array(_uniforms(11, 5, 0.0, 1.0))
    x = complex_gaussian(12, 0, 45 * 11 + 9)
    sched = rand_sched(bins, 12, 13)
    y, _ = run_gpu(bins, v, x, sched, "c128")
    assert O.rel_rms(y, oracle_complex(bins, v, x, sched)) <= 1e-12


# ---------------------------------------------------------------- reference engine tests, re-expressed
def test_random_geometries_real_streams():
    """test_oracle_engine.cpp:372-401: random (N, L, dN, b) with N in 8..64, real input."""
    rng = SeededRng(0x9E2)
    for trial in range(8):
        n = 1 << rng.uniform_int(3, 6)
        dn = 2 * rng.uniform_int(1, (n // 2 - 2) // 2)
        lo, hi = dn // 2, n // 2 - dn // 2 - 1
        l = 2 * rng.uniform_int(1, (n - 1) // 2) + 1
        blo = rng.uniform_int(lo, hi)
        bhi = rng.uniform_int(blo, hi)
        bins = BinSpec(n, l, n - l + 1, dn, blo, bhi)
        bins.validate()
        v = [rng.uniform(0.0, 1.0) for _ in range(bins.profile_length())]
        b = rng.uniform_int(blo, bhi)
        x = np.array(_uniforms(0x9E3 + trial, bins.block_length * 12, -1.0, 1.0))
        eng = OlsEngine(bins, TransitionProfile(v), b)
        y = np.concatenate([eng.process_block(x[i * bins.block_length:(i + 1) * bins.block_length])
                            for i in range(12)])
        yr = ref().ols_real(n, l, dn, blo, bhi, np.array(v), x, b0=b)
        assert np.max(np.abs(y - yr)) <= 1e-12, trial


def test_overlap_spans_several_blocks():
    """test_oracle_engine.cpp:125-141: N = 32, L = 25 (ring = 3 blocks)."""
    bins = BinSpec(32, 25, 8, 4, 10, 11)
    v = _uniforms(45, 3, 0.0, 1.0)
    x = np.array(_uniforms(46, 8 * 30, -1.0, 1.0))
    eng = OlsEngine(bins, TransitionProfile(v), 10)
    y = eng.feed(x)
    yr = ref().ols_real(32, 25, 4, 10, 11, np.array(v), x, b0=10)
    assert np.max(np.abs(y - yr)) <= 1e-12


def test_zero_in_exact_zero_out():
    """P3, test_oracle_engine.cpp:143-150."""
    bins = narrowband()
    eng = OlsEngine(bins, TransitionProfile(_uniforms(53, 15, 0.0, 1.0)), 50)
    for _ in range(4):
        assert np.all(eng.process_block(np.zeros(96)) == 0.0)
    e32 = OlsEngine(bins, TransitionProfile(_uniforms(53, 15, 0.0, 1.0)), 50, dtype="c64")
    assert np.all(e32.feed(np.zeros(96 * 3 + 5, np.complex64)) == 0)


def test_all_pass_raw_engine_is_a_delay():
    """P1, test_oracle_engine.cpp:152-161: raw all-pass table (assemble of ones) = 16-sample delay."""
    ph = ref().phase_table(128, 33)
    for dtype, tol in (("c128", 1e-12), ("c64", 2e-6)):
        eng = OlsEngine.raw(ph, 96, dtype=dtype)
        x = np.array(_uniforms(54, 96 * 6, -1.0, 1.0))
        y = eng.feed(x)
        assert y.size == x.size
        exp = np.concatenate([np.zeros(16), x[:-16]])
        assert np.max(np.abs(y - exp)) <= tol * (1 if dtype == "c128" else 4)


def test_single_bin_rings_a_cosine():
    """P2, test_oracle_engine.cpp:95-111: N = 32, M = 20, one active bin pair."""
    n, m, k0 = 32, 20, 5
    t = np.zeros(n, np.complex128)
    t[k0] = 1
    t[n - k0] = 1
    eng = OlsEngine.raw(t, m)
    blk = np.zeros(m)
    blk[0] = 1.0
    y = eng.process_block(blk)
    g = (2.0 / n) * np.cos(2 * np.pi * k0 * np.arange(m) / n)
    assert np.max(np.abs(y - g)) <= 1e-12


def test_classical_ols_equals_direct_fir():
    """P8, test_oracle_engine.cpp:290-307."""
    rng = SeededRng(69)
    for trial in range(5):
        h = np.array([rng.uniform(-1.0, 1.0) for _ in range(33)])
        padded = np.zeros(128)
        padded[:33] = h
        table = np.fft.fft(padded)
        eng = OlsEngine.raw(table, 96)
        x = np.array(_uniforms(70 + trial, 96 * 4 + 31, -1.0, 1.0))
        y = np.concatenate([eng.feed(x), eng.flush()])
        assert np.max(np.abs(y - ref().direct_fir(h, x))) <= 1e-9


def test_linearity():
    """test_oracle_engine.cpp:163-174."""
    bins = narrowband()
    prof = TransitionProfile(_uniforms(55, 15, 0.0, 1.0))
    a, b = OlsEngine(bins, prof, 52), OlsEngine(bins, prof, 52)
    x = np.array(_uniforms(56, 96 * 3, -1.0, 1.0))
    ya, yb = a.feed(x), b.feed(-1.75 * x)
    assert np.max(np.abs(yb + 1.75 * ya)) <= 1e-12


def test_block_length_enforced():
    eng = OlsEngine(narrowband(), TransitionProfile(_uniforms(57, 15, 0.0, 1.0)), 48)
    with pytest.raises(ValidationError):
        eng.process_block(np.zeros(95))


def test_retune_matches_retuned_oracle():
    """P5, test_oracle_engine.cpp:183-197: switch 48 -> 55 at block 10."""
    bins = narrowband()
    v = _uniforms(58, 15, 0.0, 1.0)
    eng = OlsEngine(bins, TransitionProfile(v), 48)
    x = np.array(_uniforms(59, 96 * 24, -1.0, 1.0))
    out = []
    for blk in range(24):
        if blk == 10:
            eng.set_bandwidth(55)
        out.append(eng.process_block(x[blk * 96:(blk + 1) * 96]))
    sched = np.array([48] * 10 + [55] * 14, np.int32)
    yr = ref().ols_real(128, 33, 16, 48, 55, np.array(v), x, bsched=sched)
    assert np.max(np.abs(np.concatenate(out) - yr)) <= 1e-12


def test_redundant_retune_bit_identical():
    """P6, test_oracle_engine.cpp:199-214."""
    bins = narrowband()
    prof = TransitionProfile(_uniforms(60, 15, 0.0, 1.0))
    a, b = OlsEngine(bins, prof, 49), OlsEngine(bins, prof, 49)
    x = np.array(_uniforms(61, 96 * 6, -1.0, 1.0))
    ya, yb = [], []
    for blk in range(6):
        if blk == 3:
            b.set_bandwidth(49)
        ya.append(a.process_block(x[blk * 96:(blk + 1) * 96]))
        yb.append(b.process_block(x[blk * 96:(blk + 1) * 96]))
    assert np.array_equal(np.concatenate(ya), np.concatenate(yb))


def test_retune_validation():
    """test_oracle_engine.cpp:216-227 (range part)."""
    eng = OlsEngine(narrowband(), TransitionProfile(_uniforms(62, 15, 0.0, 1.0)), 48)
    eng.set_bandwidth(55)
    eng.set_bandwidth(48)
    for bad in (56, 47):
        with pytest.raises(ValidationError):
            eng.set_bandwidth(bad)


def test_flush_semantics():
    """P7, test_oracle_engine.cpp:242-266."""
    bins = narrowband()
    v = _uniforms(64, 15, 0.0, 1.0)
    eng = OlsEngine(bins, TransitionProfile(v), 48)
    eng.feed(np.array(_uniforms(65, 96 * 2, -1.0, 1.0)))
    assert eng.flush().size == 0
    eng = OlsEngine(bins, TransitionProfile(v), 48)
    x = np.array(_uniforms(66, 96 + 3, -1.0, 1.0))
    y = eng.feed(x)
    tail = eng.flush()
    assert tail.size == 3
    _, _, tab = ref().coefficients(128, 33, 16, 48, 55, np.array(v), 48)
    yn = ref().naive_block_filter(128, 96, tab, x)
    assert np.max(np.abs(np.concatenate([y, tail]) - yn)) <= 1e-9
    assert eng.flush().size == 0


def test_batching_bit_identical():
    """P6, test_oracle_engine.cpp:268-288: feed(all) == drip-feed 7 at a time, bit for bit."""
    bins = narrowband()
    prof = TransitionProfile(_uniforms(67, 15, 0.0, 1.0))
    x = np.array(_uniforms(68, 96 * 5 + 17, -1.0, 1.0))
    one = OlsEngine(bins, prof, 53)
    y1 = np.concatenate([one.feed(x), one.flush()])
    drip = OlsEngine(bins, prof, 53)
    parts = [drip.feed(x[i:i + 7]) for i in range(0, x.size, 7)]
    y2 = np.concatenate(parts + [drip.flush()])
    assert np.array_equal(y1, y2)
    # and the batched device run agrees bit for bit with the streaming path
    import torch
    xd = torch.from_numpy(x.astype(np.complex128)).cuda()
    y3 = one.run(xd).cpu().numpy().real
    assert np.array_equal(y1, y3)


def test_reset_restarts_stream():
    bins = narrowband()
    eng = OlsEngine(bins, TransitionProfile(_uniforms(70, 15, 0.0, 1.0)), 50)
    x = np.array(_uniforms(71, 96 * 3, -1.0, 1.0))
    y1 = eng.feed(x)
    assert eng.blocks_processed() == 3
    eng.reset()
    assert eng.blocks_processed() == 0
    assert np.array_equal(eng.feed(x), y1)


# ---------------------------------------------------------------- P9 coefficient masks
@pytest.mark.parametrize("n,dn", [(128, 16), (512, 8), (1024, 12), (4096, 16), (8192, 32)])
def test_coefficient_masks_bit_exact(n, dn):
    bins = BinSpec(n, n // 4 + 1, n - n // 4, dn, dn // 2, n // 2 - dn // 2 - 1) if n != 128 else narrowband()
    v = np.array(_uniforms(3, dn - 1, 0.0, 1.0))
    eng = OlsEngine(bins, TransitionProfile(list(v)), bins.b_low)
    bl = sorted(set([bins.b_low, bins.b_high] + list(rand_sched(bins, 40, n))))
    region, vidx, H = eng.coeff_dump(bl)
    for i, b in enumerate(bl):
        mag, reg, tab = ref().coefficients(n, bins.filter_length, dn, bins.b_low, bins.b_high, v, b)
        assert np.array_equal(region[i], reg.astype(np.int8))
        k = np.arange(n)
        f = np.minimum(k, n - k)
        k1 = b - dn // 2 + 1
        exp_v = np.where(reg == 1, f - k1, -1)
        assert np.array_equal(vidx[i], exp_v.astype(np.int16))
        assert np.all(H[i] == tab)  # IEEE == (signed zeros compare equal)
        assert np.array_equal(np.where(reg == 1, v[np.clip(f - k1, 0, dn - 2)], (reg == 0) * 1.0), mag)


def test_narrowband_mask_layout():
    """test_spectrum.cpp:78-91 at b = 48, N = 128."""
    v = np.array(_uniforms(3, 15, 0.0, 1.0))
    eng = OlsEngine(narrowband(), TransitionProfile(list(v)), 48)
    region, vidx, _ = eng.coeff_dump([48])
    r = region[0]
    assert np.all(r[0:41] == 0) and np.all(r[41:56] == 1) and np.all(r[56:73] == 2)
    assert np.all(r[73:88] == 1) and np.all(r[88:128] == 0)
    assert list(vidx[0][41:56]) == list(range(15)) and list(vidx[0][73:88]) == list(range(14, -1, -1))


# ---------------------------------------------------------------- P11 sharding, P12 validation
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_block_range_shards_bitwise_equal(dtype):
    import torch
    bins = geometry(1024, 12)
    v = np.array(_uniforms(21, 11, 0.0, 1.0))
    S = 768 * 501 + 123
    nb = (S + 767) // 768
    x = complex_gaussian(22, 0, S, np.complex64 if dtype == "c64" else np.complex128)
    sched = rand_sched(bins, nb, 23, every=64)
    y_full, eng = run_gpu(bins, v, x, sched, dtype)
    xd = torch.from_numpy(x).cuda()
    bd = torch.from_numpy(sched).cuda()
    cuts = [0, 77, 200, 201, 390, nb]
    y_sh = np.zeros_like(y_full)
    H = 1024 - 768
    for a, b in zip(cuts[:-1], cuts[1:]):
        i0 = max(0, a * 768 - H)
        i1 = min(S, b * 768)
        xs = xd[i0:i1].clone()
        ys = torch.zeros(i1 - a * 768, dtype=xd.dtype, device="cuda")
        eng.run_range(xs, i0, S, a, b, y_dev=ys, y_first=a * 768, b_sched=bd)
        torch.cuda.synchronize()
        y_sh[a * 768:i1] = ys.cpu().numpy()
    assert np.array_equal(y_full, y_sh)


def test_out_of_range_schedule_is_validation_error():
    import torch
    bins = geometry(256, 6)
    eng = OlsEngine(bins, TransitionProfile(_uniforms(1, 5, 0, 1)), 3)
    x = torch.zeros(192 * 4, dtype=torch.complex128, device="cuda")
    bad = torch.tensor([3, 3, bins.b_high + 1, 3], dtype=torch.int32, device="cuda")
    with pytest.raises(ValidationError):
        eng.run(x, bad)
    with pytest.raises(ValidationError):
        eng.run_host(np.zeros(192 * 4, np.complex128), np.array([3, 3, 2, 3], np.int32))


def test_run_host_matches_device_run():
    import torch
    bins = geometry(1024, 12)
    v = np.array(_uniforms(31, 11, 0.0, 1.0))
    ch, S = 3, 2 ** 21 + 1000
    x = np.stack([complex_gaussian(40 + c, 0, S, np.complex64) for c in range(ch)])
    nb = (S + 767) // 768
    sched = np.stack([rand_sched(bins, nb, 50 + c, every=64) for c in range(ch)])
    eng = OlsEngine(bins, TransitionProfile(list(v)), int(sched[0, 0]), dtype="c64")
    yh = eng.run_host(x, sched)
    yd = eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(sched).cuda()).cpu().numpy()
    assert np.array_equal(yh, yd)


# ---------------------------------------------------------------- real-input fast path
def _real_case(dtype, ch, per_channel, seed=5, S=768 * 16 + 333, every=3):
    import torch
    bins = geometry(1024, 12)
    v = np.array(_uniforms(seed, 11, 0.0, 1.0))
    nb = (S + 767) // 768
    rdt = np.float32 if dtype == "c64" else np.float64
    x = np.stack([np.array(_uniforms(100 * seed + c, S, -1.0, 1.0)) for c in range(ch)]).astype(rdt)
    if per_channel:
        sched = np.stack([rand_sched(bins, nb, 7 * seed + c, every=every) for c in range(ch)])
    else:
        sched = rand_sched(bins, nb, 7 * seed, every=every)
    eng = OlsEngine(bins, TransitionProfile(list(v)), int(np.ravel(sched)[0]), dtype=dtype)
    return bins, v, x, sched, eng, torch.from_numpy(x).cuda(), torch.from_numpy(np.ascontiguousarray(sched)).cuda()


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("per_channel", [False, True])
@pytest.mark.parametrize("every", [1, 2, 3, 64])
def test_run_real_matches_reference_real_engine(dtype, per_channel, every):
    """Block pairs share a transform when their b agree; schedules changing every 1 / 3 blocks
    exercise the straddling-pair fallback, every 2 / 64 the all-paired path; 17 blocks (odd) and a
    partial tail exercise the lone last block."""
    bins, v, x, sched, eng, xd, bd = _real_case(dtype, 3, per_channel, every=every)
    y = eng.run_real(xd, bd).cpu().numpy()
    for c in range(x.shape[0]):
        sc = sched[c] if per_channel else sched
        yr = ref().ols_real(1024, 257, 12, bins.b_low, bins.b_high, v, x[c].astype(np.float64), bsched=sc)
        assert O.rel_rms(y[c].astype(np.float64), yr) <= TOL[dtype], c


@pytest.mark.parametrize("n", [16, 64, 256, 512, 4096])
def test_run_real_other_sizes(n):
    import torch
    bins = geometry(n)
    v = np.array(_uniforms(n, bins.profile_length(), 0.0, 1.0))
    m = bins.block_length
    S = m * 9 + m // 3
    x = np.array(_uniforms(n + 1, S, -1.0, 1.0))
    sched = rand_sched(bins, (S + m - 1) // m, n, every=2)
    eng = OlsEngine(bins, TransitionProfile(list(v)), int(sched[0]))
    y = eng.run_real(torch.from_numpy(x).cuda(), torch.from_numpy(sched).cuda()).cpu().numpy()
    yr = ref().ols_real(n, bins.filter_length, bins.transition_width_bins, bins.b_low, bins.b_high, v, x, bsched=sched)
    assert O.rel_rms(y, yr) <= 1e-12


@pytest.mark.parametrize("n", [16, 64, 256, 512])
@pytest.mark.parametrize("every", [1, 3])
def test_run_real_small_groups_unpaired(n, every):
    """Groups smaller than a warp (T < 32) where neighbouring groups run one or two transforms per
    item (pairs with different b fall back to one block per transform)."""
    import torch
    bins = geometry(n)
    v = np.array(_uniforms(n + 7, bins.profile_length(), 0.0, 1.0))
    m = bins.block_length
    S = m * 41 + m // 3
    x = np.array(_uniforms(n + 9, 3 * S, -1.0, 1.0)).reshape(3, S)
    sched = rand_sched(bins, (S + m - 1) // m, n + 11, every=every)
    eng = OlsEngine(bins, TransitionProfile(list(v)), int(sched[0]))
    y = eng.run_real(torch.from_numpy(x).cuda(), torch.from_numpy(sched).cuda()).cpu().numpy()
    for c in range(3):
        yr = ref().ols_real(n, bins.filter_length, bins.transition_width_bins, bins.b_low, bins.b_high, v, x[c],
                            bsched=sched)
        assert O.rel_rms(y[c], yr) <= 1e-12, (n, every, c)


def test_run_real_equals_complex_path():
    """Carrying two blocks in one transform changes only rounding."""
    import torch
    bins, v, x, sched, eng, xd, bd = _real_case("c128", 4, True, seed=9, every=64)
    y_real = eng.run_real(xd, bd).cpu().numpy()
    y_cplx = eng.run(torch.from_numpy(x.astype(np.complex128)).cuda(), bd).cpu().numpy().real
    assert O.rel_rms(y_real, y_cplx) <= 1e-14


def test_run_real_raw_engine_takes_real_part():
    """Raw tables may be asymmetric: the reference keeps Re(IFFT) (fft.hpp:68-78); run_real must
    not pack two blocks into one transform then."""
    import torch
    rng = np.random.default_rng(3)
    table = rng.normal(size=64) + 1j * rng.normal(size=64)  # not conjugate-symmetric
    eng = OlsEngine.raw(table, 48)
    x = rng.uniform(-1, 1, size=(3, 48 * 9 + 5))
    y = eng.run_real(torch.from_numpy(x).cuda()).cpu().numpy()
    for c in range(3):
        yr = ref().ols_raw_real(64, 48, table, x[c])
        assert np.max(np.abs(y[c] - yr)) <= 1e-12


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_run_real_host_matches_device_and_reference(dtype):
    import torch
    bins = geometry(1024, 12)
    v = np.array(_uniforms(77, 11, 0.0, 1.0))
    S = 2 ** 21 + 3 * 768 + 100  # several host chunks, odd block count, partial tail
    nb = (S + 767) // 768
    rdt = np.float32 if dtype == "c64" else np.float64
    x = np.stack([np.array(_uniforms(78 + c, S, -1.0, 1.0)) for c in range(2)]).astype(rdt)
    sched = np.stack([rand_sched(bins, nb, 79 + c, every=5) for c in range(2)])
    eng = OlsEngine(bins, TransitionProfile(list(v)), int(sched[0, 0]), dtype=dtype)
    yh = eng.run_real_host(x, sched)
    yd = eng.run_real(torch.from_numpy(x).cuda(), torch.from_numpy(sched).cuda()).cpu().numpy()
    assert np.array_equal(yh, yd)
    yr = ref().ols_real(1024, 257, 12, bins.b_low, bins.b_high, v, x[1].astype(np.float64), bsched=sched[1])
    assert O.rel_rms(yh[1].astype(np.float64), yr) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n", [16, 64, 128, 512, 1024, 2048, 4096])
def test_run_real_mixed_pairs(dtype, n):
    """Block pairs whose two blocks use DIFFERENT b share one transform (Y = Z (H0 + H1)/2 +
    conj(Z(N - k)) (H0 - H1)/2): a schedule redrawn every block makes almost every pair mixed;
    compared with the reference real engine and with the one-block-per-transform path."""
    import torch
    bins = geometry(n)
    v = np.array(_uniforms(n + 31, bins.profile_length(), 0.0, 1.0))
    m = bins.block_length
    S = m * 37 + m // 5
    nb = (S + m - 1) // m
    rdt = np.float32 if dtype == "c64" else np.float64
    x = np.stack([np.array(_uniforms(n + 33 + c, S, -1.0, 1.0)) for c in range(3)]).astype(rdt)
    sched = np.stack([rand_sched(bins, nb, n + 35 + c, every=1) for c in range(3)])
    assert np.mean(sched[:, 0:nb - 1:2] != sched[:, 1:nb:2]) > 0.5  # mostly mixed pairs
    eng = OlsEngine(bins, TransitionProfile(list(v)), int(sched[0, 0]), dtype=dtype)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(sched).cuda()
    y = eng.run_real(xd, bd).cpu().numpy()
    y1 = eng.run_real(xd, bd, one_block_per_transform=True).cpu().numpy()
    for c in range(3):
        yr = ref().ols_real(n, bins.filter_length, bins.transition_width_bins, bins.b_low, bins.b_high, v,
                            x[c].astype(np.float64), bsched=sched[c])
        assert O.rel_rms(y[c].astype(np.float64), yr) <= TOL[dtype], (c, "paired")
        assert O.rel_rms(y1[c].astype(np.float64), yr) <= TOL[dtype], (c, "unpaired")


def test_run_real_one_block_per_transform_is_complex_path():
    """One real block per transform (Im = 0) is the complex path on x + 0j, bit for bit."""
    import torch
    bins, v, x, sched, eng, xd, bd = _real_case("c64", 4, True, seed=11, every=1)
    y1 = eng.run_real(xd, bd, one_block_per_transform=True).cpu().numpy()
    yc = eng.run(torch.from_numpy(x.astype(np.complex64)).cuda(), bd).cpu().numpy()
    assert np.array_equal(y1, yc.real)
