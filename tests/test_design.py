"""GPU-assisted minimax design against the reference's own
`solve_minimax` / `design` (proj/include/fcvbw/design.hpp:276-446, 486-577).

Fixtures: tests/golden/design_vectors.json, generated from the compiled reference by
tests/golden/make_design_golden.py (so the GPU tests need no /root/reference on the box).

Tolerance: the GPU path evaluates every constraint and sweep point with the reference's operation
order, no FMA contraction, host-libm tables and glibc's hypot algorithm (csrc/design.cu,
response.cuh), so V, delta, rounds and LP iteration counts are bit-identical in practice; the
asserts allow 1e-12 (absolute on V, relative on delta). The shift rule is measured by
impulse-probing the GPU engine (fcvbw_gpu_calibrate_shift), as design() does on its processor.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "design_vectors.json")))
SOLVE = {c["name"]: c for c in GOLD["solve"]}
DESIGN = {c["name"]: c for c in GOLD["design"]}


# ------------------------------------------------------------------ CPU: host logic and fixture pins
def test_estimators_match_reference_rules():
    from paper_2406_14116_b200.design import estimate_fft_length, estimate_order
    # design.hpp:25-52 by hand: raw = 4 pi / dw for ripples 0.01
    assert estimate_order(0.01, 0.01, math.pi / 4) == 16
    assert estimate_order(0.01, 0.01, math.pi / 8) == 32
    assert estimate_fft_length(15) == 64 and estimate_fft_length(31) == 128 and estimate_fft_length(63) == 256
    from paper_2406_14116_b200 import ValidationError
    with pytest.raises(ValidationError):
        estimate_fft_length(1)
    with pytest.raises(ValidationError):
        estimate_order(0.0, 0.01, 0.5)


def test_discretize_and_offgrid():
    from paper_2406_14116_b200.bins import OffGridError
    from paper_2406_14116_b200.design import FilterSpec, validate_and_discretize
    spec = FilterSpec(math.pi / 8, 0.01, 0.01, 0.05, math.pi / 4, math.pi / 2)
    b = validate_and_discretize(spec, 128, 31)
    assert (b.transition_width_bins, b.b_low, b.b_high, b.block_length) == (8, 16, 32, 98)
    with pytest.raises(OffGridError):
        validate_and_discretize(FilterSpec(0.1, 0.01, 0.01, 0.05, 1.0, 1.0), 128, 31)


@pytest.mark.skipif(not O.have_reference(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("name", ["n64_single", "n128_range5_d8", "n128_p8_stride8"])
def test_fixture_reproduces_reference(name):
    c = SOLVE[name]
    r = O.reference().solve_minimax(c["N"], c["L"], c["delta_N"], c["b_low"], c["b_high"], c["grid_points"],
                                    c["facets"], c["exchange_tol"], c["max_rounds"], c["seed_stride"])
    assert r["v"].tolist() == c["V"] and r["delta"] == c["delta"] and r["rounds"] == c["rounds"]


# ------------------------------------------------------------------ GPU
def _solve(c, **over):
    from paper_2406_14116_b200 import BinSpec
    from paper_2406_14116_b200.design import DesignOptions, solve_minimax
    bins = BinSpec(c["N"], c["L"], c["N"] - c["L"] + 1, c["delta_N"], c["b_low"], c["b_high"])
    opt = DesignOptions(grid_points=c["grid_points"], facets=c["facets"], exchange_tol=c["exchange_tol"],
                        max_rounds=over.get("max_rounds", c["max_rounds"]), seed_stride=c["seed_stride"])
    return solve_minimax(bins, opt)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(SOLVE))
def test_gpu_solve_minimax_parity(name):
    c = SOLVE[name]
    out = _solve(c)
    v = np.array(out.profile.values)
    assert np.abs(v - np.array(c["V"])).max() <= 1e-12, (v, c["V"])
    assert abs(out.delta - c["delta"]) <= 1e-12 * c["delta"]
    assert abs(out.lp_delta - c["lp_delta"]) <= 1e-12 * c["lp_delta"]
    assert out.rounds == c["rounds"]
    assert out.active_triples == c["active_triples"]
    assert out.lp_iterations == c["lp_iterations"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(DESIGN))
def test_gpu_design_order_loop_parity(name):
    from paper_2406_14116_b200.design import DesignOptions, FilterSpec, design
    c = DESIGN[name]
    r = design(FilterSpec(*c["spec"]), DesignOptions(grid_points=c["grid_points"]))
    b = r.bins
    assert (b.fft_length, b.filter_length, b.transition_width_bins, b.b_low, b.b_high) == \
        (c["N"], c["L"], c["delta_N"], c["b_low"], c["b_high"])
    assert r.iterations == c["iterations"] and r.exchange_rounds == c["exchange_rounds"]
    assert np.abs(np.array(r.profile.values) - np.array(c["V"])).max() <= 1e-12
    assert abs(r.delta - c["delta"]) <= 1e-12 * c["delta"]


@pytest.mark.gpu
def test_gpu_design_errors():
    from paper_2406_14116_b200 import ValidationError
    from paper_2406_14116_b200.bins import NonConvergenceError
    c = SOLVE["n128_range5_d8"]
    assert c["rounds"] > 1
    with pytest.raises(NonConvergenceError):
        _solve(c, max_rounds=1)  # design.hpp:360-363
    with pytest.raises(ValidationError):
        _solve(dict(c, grid_points=c["N"]))  # FrequencyGrid: K >= 2N
    with pytest.raises(ValidationError):
        _solve(dict(c, facets=7))  # DesignProblem::validate


@pytest.mark.gpu
@pytest.mark.parametrize("n,l,dn", [(16, 15, 2), (64, 17, 4), (128, 97, 8), (256, 65, 6), (32, 1, 4), (128, 96, 8),
                                    (1024, 257, 12)])
def test_gpu_calibrated_shift_rule(n, l, dn):
    """calibrated_shift_rule measured by impulse-probing the GPU engine equals the reference's
    (measured on its naive block filter) — fixture-free: the reference's rule for the OLS family
    is (1 - M, +1), pinned on CPU by tests/test_verify.py::test_shift_rule_is_overlap_save."""
    from paper_2406_14116_b200 import BinSpec
    from paper_2406_14116_b200.verify import _RULES, calibrated_shift_rule
    _RULES.clear()
    m = n - l + 1
    bins = BinSpec(n, l, m, dn, dn // 2, n // 2 - dn // 2 - 1)
    assert calibrated_shift_rule(bins) == (1 - m, 1)
    if O.have_reference():
        assert O.reference().shift_rule(n, l, dn, dn // 2, n // 2 - dn // 2 - 1) == (1 - m, 1)
