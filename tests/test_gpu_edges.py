"""GPU edge cases through the C-ABI, each against the reference engine (oracle/_ref) on the same
input: empty and tiny streams (shorter than one block / than the halo), L = 1 (no overlap) and
L = N (one output per block), even L, the widest transition bands (dN - 2 >= T: the generic
per-register mask path), b at both ends of the admissible range, tiny raw-table transforms."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_14116_b200 import BinSpec, OlsEngine, TransitionProfile
from paper_2406_14116_b200.workload import SeededRng, complex_gaussian

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-12, "c64": 2e-6}


def _u(seed, n, lo=0.0, hi=1.0):
    r = SeededRng(seed)
    return np.array([r.uniform(lo, hi) for _ in range(n)])


def check(bins, v, S, dtype="c128", seed=1, sched=None, ch=1):
    import torch
    m = bins.block_length
    nb = (S + m - 1) // m
    if sched is None:
        r = SeededRng(seed)
        sched = np.array([r.uniform_int(bins.b_low, bins.b_high) for _ in range(max(nb, 1))], np.int32)[:nb]
    x = np.stack([complex_gaussian(seed + c, 0, S) for c in range(ch)]).astype(
        np.complex64 if dtype == "c64" else np.complex128)
    eng = OlsEngine(bins, TransitionProfile(list(v)), int(sched[0]) if nb else bins.b_low, dtype=dtype)
    xd = torch.from_numpy(x).cuda()
    bd = torch.from_numpy(np.ascontiguousarray(sched)).cuda() if nb else None
    y = eng.run(xd, bd).cpu().numpy()
    if S == 0:
        assert y.size == 0
        return
    yr = O.best().ols_complex(bins.fft_length, bins.filter_length, bins.transition_width_bins, bins.b_low,
                              bins.b_high, np.asarray(v), x.astype(np.complex128), bsched=sched)
    err = O.rel_rms(y, yr)
    if S < bins.fft_length:
        # a few output samples whose energy may be far below the input's (S = 1: the filter's
        # leading tap): judge the error against the input scale instead of the output scale
        err = float(np.sqrt(np.sum(np.abs(y - yr) ** 2) / np.sum(np.abs(x) ** 2)))
    assert err <= TOL[dtype], (bins, S, dtype, err)


@pytest.mark.parametrize("S", [0, 1, 5, 95, 96, 97, 127, 128, 129, 200])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_short_streams(S, dtype):
    bins = BinSpec(128, 33, 96, 16, 48, 55)
    check(bins, _u(3, 15), S, dtype)


@pytest.mark.parametrize("n", [16, 64, 1024])
def test_no_overlap_L1(n):
    bins = BinSpec(n, 1, n, 4, 2, n // 2 - 3)
    check(bins, _u(4, 3), n * 7 + 3)


@pytest.mark.parametrize("n", [16, 64, 256])
def test_single_output_per_block_L_eq_N(n):
    bins = BinSpec(n, n, 1, 4, 2, n // 2 - 3)  # L = N -> M = 1, halo N - 1, even L - 1? (N - 1 odd)
    check(bins, _u(5, 3), 3 * n + 7)


@pytest.mark.parametrize("n,l", [(64, 20), (128, 40), (1024, 300), (4096, 1000)])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_even_filter_lengths(n, l, dtype):
    bins = BinSpec(n, l, n - l + 1, 6, 3, n // 2 - 4)
    check(bins, _u(6, 5), (n - l + 1) * 9 + 11, dtype)


@pytest.mark.parametrize("n,dn", [(64, 20), (128, 40), (32, 12), (512, 100), (1024, 200)])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_wide_transition_bands_generic_mask(n, dn, dtype):
    """dN - 2 >= T (threads per block): more than one transition register per half per thread."""
    bins = BinSpec(n, n // 4 + 1, n - n // 4, dn, dn // 2, n // 2 - dn // 2 - 1)
    check(bins, _u(7, dn - 1, -0.3, 1.2), (n - n // 4) * 11 + 5, dtype)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_extreme_bandwidths(dtype):
    bins = BinSpec(1024, 257, 768, 12, 6, 505)
    nb = 12
    for b in (6, 505):
        check(bins, _u(8, 11), 768 * nb - 5, dtype, sched=np.full(nb, b, np.int32))
    alt = np.array([6, 505] * 6, np.int32)
    check(bins, _u(8, 11), 768 * nb - 5, dtype, sched=alt)


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_tiny_raw_transforms(n):
    rng = np.random.default_rng(n)
    table = np.fft.fft(np.r_[rng.uniform(-1, 1, n // 2), np.zeros(n - n // 2)])
    m = max(1, n // 2)
    eng = OlsEngine.raw(table, m)
    x = rng.uniform(-1, 1, m * 13 + 1)
    y = np.concatenate([eng.feed(x), eng.flush()])
    assert np.max(np.abs(y - O.best().ols_raw_real(n, m, table, x))) <= 1e-12


def test_many_channels_small_streams():
    bins = BinSpec(256, 65, 192, 6, 3, 124)
    check(bins, _u(9, 5), 500, "c64", ch=300)


@pytest.mark.parametrize("n", [64, 512, 1024, 4096])
@pytest.mark.parametrize("dtype,scale", [("c64", 1e20), ("c64", 1e-20), ("c128", 1e250), ("c128", 1e-250)])
def test_extreme_magnitudes(n, dtype, scale):
    """Inputs far from unit scale: the tangent-form twiddles (W = wr (1 + j t), with wr at the
    +-pi/2 angles stored as 2^-40 / 2^-60, ols_kernel.cuh Pass::run) must not overflow or lose
    precision; the filter is linear, so the reference output scales exactly."""
    import torch
    bins = BinSpec(n, n // 4 + 1, 3 * n // 4, 4, 2, n // 2 - 3)
    v = _u(9, 3)
    S = 3 * n // 4 * 20 + 7
    nb = (S + bins.block_length - 1) // bins.block_length
    r = SeededRng(17)
    sched = np.array([r.uniform_int(bins.b_low, bins.b_high) for _ in range(nb)], np.int32)
    x = complex_gaussian(21, 0, S)
    xs = (x * scale).astype(np.complex64 if dtype == "c64" else np.complex128)
    eng = OlsEngine(bins, TransitionProfile(list(v)), int(sched[0]), dtype=dtype)
    y = eng.run(torch.from_numpy(xs[None]).cuda(), torch.from_numpy(sched).cuda()).cpu().numpy()[0]
    assert np.all(np.isfinite(y))
    yr = O.best().ols_complex(n, bins.filter_length, 4, bins.b_low, bins.b_high, v,
                              xs.astype(np.complex128)[None], bsched=sched)[0]
    err = O.rel_rms(y.astype(np.complex128) / scale, yr / scale)  # (|y|^2 itself would overflow at 1e250)
    assert err <= TOL[dtype], (n, dtype, scale, err)
