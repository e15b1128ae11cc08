"""Design verification: the GPU `verify()` (csrc/verify.cu) against the
reference's own `verify()` (proj/include/fcvbw/design.hpp:601-673) run through oracle/_ref, or the C
restatement `orc_verify` when the compiled reference is absent (GPU box).

CPU tests pin the restatement bit-for-bit to the reference and pin the shift rule the GPU path
assumes (calibrated_shift_rule, design.hpp:476-484). GPU tests compare every report field: maxima
to 1e-12 absolute (fp64; the GPU evaluates the same sums in a different order — prefix sums over
shifted rows instead of one dot product per row), worst_b / worst_n / worst_omega exactly unless
the runner-up lies within that tolerance of the maximum.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_14116_b200.workload import SeededRng

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ABS = 1e-12


def _artifact(name):
    a = json.load(open(os.path.join(ROOT, "configs", name)))
    return dict(n=a["N"], l=a["L"], dn=a["delta_N"], blo=a["bN_low"], bhi=a["bN_high"], v=np.array(a["V"]),
                delta=a["delta_achieved"], grid=a["grid_K"], facets=a["facets_P"])


def _random_case(seed, n, l, dn, blo, bhi):
    r = SeededRng(seed)
    v = np.array([r.uniform(0.05, 0.95) for _ in range(dn - 1)])
    return dict(n=n, l=l, dn=dn, blo=blo, bhi=bhi, v=v, delta=0.01, grid=n, facets=16)


CASES = {
    "n64_art_full": (_artifact("artifact_n64_d4.json"), 4),
    "n128_art_full": (_artifact("artifact_n128_d4.json"), 4),
    "n128_rand_narrow": (_random_case(11, 128, 97, 8, 20, 27), 8),
    "n256_art_sub": (dict(_artifact("artifact_n256_d6.json"), blo=3, bhi=14), 4),
    "n32_rand_L1": (_random_case(12, 32, 1, 4, 2, 13), 4),
    "n16_rand_LN": (_random_case(13, 16, 15, 2, 1, 6), 8),
    "n128_rand_evenL": (_random_case(14, 128, 96, 8, 4, 59), 4),
}


def _ref_report(c, dense, delta_e=0.05, lib=None):
    lib = lib or O.best()
    return lib.verify(c["n"], c["l"], c["dn"], c["blo"], c["bhi"], c["v"], c["delta"], c["grid"], c["facets"],
                      dense, delta_e)


@pytest.mark.skipif(not O.have_reference(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("name", ["n64_art_full", "n128_rand_narrow", "n32_rand_L1", "n16_rand_LN",
                                  "n128_rand_evenL"])
def test_port_verify_matches_reference(name):
    c, mult = CASES[name]
    dense = mult * c["grid"]
    a = _ref_report(c, dense, lib=O.reference())
    b = _ref_report(c, dense, lib=O.port())
    for k in a:
        if isinstance(a[k], np.ndarray):
            assert np.array_equal(a[k], b[k]), k
        else:
            assert a[k] == b[k], (k, a[k], b[k])


@pytest.mark.skipif(not O.have_reference(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("n,l,dn", [(16, 15, 2), (64, 17, 4), (128, 97, 8), (256, 65, 6), (32, 1, 4)])
def test_shift_rule_is_overlap_save(n, l, dn):
    from paper_2406_14116_b200.verify import OLS_SHIFT_STEP
    m = n - l + 1
    assert O.reference().shift_rule(n, l, dn, dn // 2, n // 2 - dn // 2 - 1) == (1 - m, OLS_SHIFT_STEP)


def _gpu_report(c, dense, delta_e=0.05, exact=False):
    from paper_2406_14116_b200 import BinSpec, DesignResult, TransitionProfile
    from paper_2406_14116_b200.verify import verify
    bins = BinSpec(c["n"], c["l"], c["n"] - c["l"] + 1, c["dn"], c["blo"], c["bhi"])
    res = DesignResult(TransitionProfile(list(c["v"])), bins, delta=c["delta"], grid_points=c["grid"],
                       facets=c["facets"])
    return verify(res, dense, delta_e, exact=exact)


def _check_argmax(values, got, want):
    """Exact index unless the runner-up is within ABS of the maximum (rounding may swap them)."""
    if got == want:
        return
    top = max(values)
    assert values[got] >= top - ABS and values[want] >= top - ABS, (got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_verify_parity(name):
    c, mult = CASES[name]
    dense = mult * c["grid"]
    want = _ref_report(c, dense)
    got = _gpu_report(c, dense)
    assert abs(got.delta - want["delta"]) <= ABS
    assert abs(got.passband_max - want["passband_max"]) <= ABS
    assert abs(got.stopband_max - want["stopband_max"]) <= ABS
    per_b = np.array([got.per_b_max[b] for b in range(c["blo"], c["bhi"] + 1)])
    assert np.abs(per_b - want["per_b_max"]).max() <= ABS
    assert np.abs(np.array(got.per_n_max) - want["per_n_max"]).max() <= ABS
    assert got.dense_points == want["dense_points"]
    assert got.refinement_bound == want["refinement_bound"]
    assert got.passed == want["passed"] and got.within_bound == want["within_bound"]
    _check_argmax(list(want["per_b_max"]), got.worst_b - c["blo"], want["worst_b"] - c["blo"])
    if got.worst_b == want["worst_b"] and got.worst_n != want["worst_n"]:
        # near-tie inside the worst b: the GPU's (n, omega) must still attain the maximum
        assert want["per_n_max"][got.worst_n] >= want["delta"] - ABS
    elif got.worst_b == want["worst_b"]:
        assert abs(got.worst_omega - want["worst_omega"]) <= 1e-15 or \
            want["per_n_max"][got.worst_n] >= want["delta"] - ABS


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_verify_exact_is_bit_identical(name):
    """fcvbw_gpu_verify_exact: the reference's own summation order and glibc's hypot -> every field
    equal under ==."""
    c, mult = CASES[name]
    dense = mult * c["grid"]
    want = _ref_report(c, dense)
    got = _gpu_report(c, dense, exact=True)
    per_b = np.array([got.per_b_max[b] for b in range(c["blo"], c["bhi"] + 1)])
    assert np.array_equal(per_b, want["per_b_max"])
    assert np.array_equal(np.array(got.per_n_max), want["per_n_max"])
    assert (got.delta, got.passband_max, got.stopband_max, got.worst_omega, got.refinement_bound) == \
        (want["delta"], want["passband_max"], want["stopband_max"], want["worst_omega"], want["refinement_bound"])
    assert (got.worst_b, got.worst_n, got.dense_points, got.passed, got.within_bound) == \
        (want["worst_b"], want["worst_n"], want["dense_points"], want["passed"], want["within_bound"])


@pytest.mark.gpu
def test_gpu_verify_validation():
    from paper_2406_14116_b200 import ValidationError
    c, _ = CASES["n128_rand_narrow"]
    with pytest.raises(ValidationError):
        _gpu_report(c, 2 * c["grid"])  # dense grid below 4x the design points
    with pytest.raises(O.OracleError):
        _ref_report(c, 2 * c["grid"])
    bad = dict(c, bhi=c["n"] // 2)  # band centre range beyond N/2 - delta_N/2 - 1 (BinSpec::validate)
    with pytest.raises(ValidationError):
        _gpu_report(bad, 4 * bad["grid"])
