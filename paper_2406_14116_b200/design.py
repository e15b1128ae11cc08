"""Minimax design of the transition-band profile V, GPU-assisted.

Mirrors the reference's design front end (proj/include/fcvbw/design.hpp:25-60, 449-577 and
spectrum.hpp:26-47, 100-158): ``FilterSpec``, ``DesignOptions``, ``estimate_order``,
``estimate_fft_length``, ``nearest_grid_spec``, ``validate_and_discretize``, ``solve_minimax`` and
``design``. The exchange itself (``solve_minimax``, design.hpp:276-446) runs in
``libfcvbw_gpu.so`` (csrc/design.cu): constraint assembly and the dense true-error sweep on the GPU,
the LP on the host. The order-selection loop below is host logic only.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bins import BinSpec, DesignResult, Error, OffGridError, TransitionProfile, ValidationError
from .engine import _raise
from .verify import calibrated_shift_rule

K_PI = math.pi
K_BIN_SNAP_TOL = 1e-2  # spectrum.hpp:22


def _round(x: float) -> int:
    """std::round / std::lround: halves away from zero."""
    a = abs(x)
    r = math.floor(a)
    if a - r >= 0.5:
        r += 1
    return int(math.copysign(r, x)) if r else 0


@dataclass
class FilterSpec:
    """spectrum.hpp:26-47 (radians)."""
    transition_width: float = 0.0
    ripple_pass: float = 0.0
    ripple_stop: float = 0.0
    max_error: float = 0.0
    band_center_low: float = 0.0
    band_center_high: float = 0.0

    def validate(self) -> None:
        if not (0.0 < self.transition_width < K_PI):
            raise ValidationError("FilterSpec: transition width must lie in (0, pi)")
        for d in (self.ripple_pass, self.ripple_stop, self.max_error):
            if not (0.0 < d < 1.0):
                raise ValidationError("FilterSpec: ripples and max error must lie in (0, 1)")
        half = self.transition_width / 2.0
        if not (half <= self.band_center_low <= self.band_center_high <= K_PI - half):
            raise ValidationError("FilterSpec: band centers must satisfy delta/2 <= b_l <= b_u <= pi - delta/2")


@dataclass
class DesignOptions:
    """design.hpp:452-461."""
    fft_length_override: int = 0
    filter_length_override: int = 0
    grid_points: int = 1000
    facets: int = 16
    exchange_tol: float = 0.025
    max_rounds: int = 60
    seed_stride: int = 16
    margin: float = 0.5


@dataclass
class SolveOutcome:
    """design.hpp:271-278 (without the final constraint system, which stays on the device side)."""
    profile: TransitionProfile
    delta: float
    lp_delta: float
    rounds: int
    lp_iterations: int
    active_triples: int = 0
    lp_rows: int = 0
    grid_size: int = 0
    seconds: dict | None = None  # host wall time per phase: tables, assembly, lp, sweep


def estimate_order(ripple_pass: float, ripple_stop: float, transition_width: float) -> int:
    """design.hpp:25-35."""
    if not (ripple_pass > 0.0 and ripple_stop > 0.0):
        raise ValidationError("estimate_order: ripples must be positive")
    if not (0.0 < transition_width < K_PI):
        raise ValidationError("estimate_order: transition width must lie in (0, pi)")
    raw = -4.0 * K_PI * math.log10(10.0 * ripple_pass * ripple_stop) / (3.0 * transition_width)
    half = _round(math.ceil(raw / 2.0 - 1e-9))
    return 2 * max(1, half)


def estimate_fft_length(filter_length: int) -> int:
    """design.hpp:37-52: N = 2^round(log2(0.9 L log2 L))."""
    if filter_length < 2:
        raise ValidationError("estimate_fft_length: need L >= 2")
    l = float(filter_length)
    q = _round(math.log2(0.9 * l * math.log2(l)))
    n = 1 << max(1, q)
    if n <= filter_length or n < 8:
        raise ValidationError(f"estimate_fft_length: estimate N = {n} is no larger than L = {filter_length}; "
                              "supply N manually")
    return n


def nearest_grid_spec(spec: FilterSpec, fft_length: int) -> FilterSpec:
    """spectrum.hpp:100-118."""
    to_bins = fft_length / (2.0 * K_PI)
    dn = 2 * max(1, _round(spec.transition_width * to_bins / 2.0))
    dn = min(dn, 2 * (fft_length // 4 - 1))
    lo = dn // 2
    hi = max(lo, fft_length // 2 - dn // 2 - 1)

    def clamp_bin(w):
        return min(max(_round(w * to_bins), lo), hi)
    bl = clamp_bin(spec.band_center_low)
    bu = max(bl, clamp_bin(spec.band_center_high))
    return FilterSpec(dn * 2.0 * K_PI / fft_length, spec.ripple_pass, spec.ripple_stop, spec.max_error,
                      bl * 2.0 * K_PI / fft_length, bu * 2.0 * K_PI / fft_length)


def _snap_to_bin(raw: float, what: str, spec: FilterSpec, fft_length: int) -> int:
    rounded = _round(raw)
    if abs(raw - rounded) > K_BIN_SNAP_TOL:
        near = nearest_grid_spec(spec, fft_length)
        raise OffGridError(f"off-grid spec: {what} = {raw:g} bins is not integral at N = {fft_length}; nearest grid "
                           f"spec: transition_width = {near.transition_width:g}, b_low = {near.band_center_low:g}, "
                           f"b_high = {near.band_center_high:g}")
    return rounded


def validate_and_discretize(spec: FilterSpec, fft_length: int, filter_length: int) -> BinSpec:
    """spectrum.hpp:135-158."""
    spec.validate()
    if fft_length < 8 or fft_length & (fft_length - 1):
        raise ValidationError("discretize: N must be 2^Q with Q >= 3")
    if filter_length > fft_length:
        raise ValidationError("discretize: L must not exceed N")
    to_bins = fft_length / (2.0 * K_PI)
    dn = _snap_to_bin(spec.transition_width * to_bins, "delta_N", spec, fft_length)
    blo = _snap_to_bin(spec.band_center_low * to_bins, "b_N,l", spec, fft_length)
    bhi = _snap_to_bin(spec.band_center_high * to_bins, "b_N,u", spec, fft_length)
    if dn % 2:
        raise OffGridError(f"off-grid spec: delta_N = {dn} must be even at N = {fft_length}")
    bins = BinSpec(fft_length, filter_length, fft_length - filter_length + 1, dn, blo, bhi)
    bins.validate()
    return bins


def solve_minimax(bins: BinSpec, opt: DesignOptions | None = None, device: int = 0,
                  rule: tuple[int, int] | None = None) -> SolveOutcome:
    """solve_minimax (design.hpp:276-446) on the GPU for one BinSpec. `rule` = (window_offset, step);
    default: calibrated on the GPU engine (design.hpp:504-506)."""
    opt = opt or DesignOptions()
    bins.validate()
    wo, step = rule if rule is not None else calibrated_shift_rule(bins, device)
    if wo != 1 - bins.block_length:
        raise Error(f"solve_minimax: window offset {wo} is not the overlap-save offset {1 - bins.block_length}")
    lv = bins.transition_width_bins - 1
    geo = _lib.Design(bins.fft_length, bins.filter_length, bins.block_length, bins.transition_width_bins, bins.b_low,
                      bins.b_high, None, lv, 0.0, int(opt.grid_points), int(opt.facets))
    o = _lib.SolveOptions(int(opt.grid_points), int(opt.facets), float(opt.exchange_tol), int(opt.max_rounds),
                          int(opt.seed_stride))
    v = np.zeros(lv)
    res = _lib.SolveResult()
    _raise(_lib.lib().fcvbw_gpu_solve_minimax(C.byref(geo), C.byref(o), int(step), int(device), v.ctypes.data,
                                              C.byref(res)))
    return SolveOutcome(TransitionProfile(v.tolist()), res.delta, res.lp_delta, res.rounds, res.lp_iterations,
                        res.active_triples, res.lp_rows, res.grid_size,
                        dict(tables=res.seconds_tables, assembly=res.seconds_assembly, lp=res.seconds_lp,
                             sweep=res.seconds_sweep))


def design(spec: FilterSpec, opt: DesignOptions | None = None, device: int = 0) -> DesignResult:
    """design() (design.hpp:486-577): order selection around the GPU solve_minimax."""
    from .bins import NonConvergenceError
    opt = opt or DesignOptions()
    spec.validate()
    evaluated = 0

    def evaluate(order):
        nonlocal evaluated
        filter_length = order + 1
        n = opt.fft_length_override or estimate_fft_length(filter_length)
        bins = validate_and_discretize(spec, n, filter_length)
        out = solve_minimax(bins, opt, device)
        evaluated += 1
        return order, bins, out

    def finish(cand):
        _, bins, out = cand
        return DesignResult(out.profile, bins, delta=out.delta, grid_points=opt.grid_points, facets=opt.facets,
                            iterations=evaluated, exchange_rounds=out.rounds)

    if opt.filter_length_override:
        return finish(evaluate(opt.filter_length_override - 1))

    initial = estimate_order(spec.ripple_pass, spec.ripple_stop, spec.transition_width)
    cap = 8 * initial
    step = 4
    first_skip = ""
    accepted = None
    tried = set()
    order = initial
    while True:
        if order > cap:
            if evaluated == 0:
                raise OffGridError(first_skip or "design: no candidate order fits the bin grid")
            raise NonConvergenceError(f"design: no order up to {cap} meets max_error; tightest achieved delta "
                                      "exceeds the requirement")
        tried.add(order)
        try:
            cand = evaluate(order)
            if cand[2].delta <= spec.max_error:
                accepted = cand
                break
        except ValidationError as e:  # OffGridError included
            if not first_skip:
                first_skip = str(e)
        order += step

    if accepted[2].delta < opt.margin * spec.max_error:
        reduced = accepted[0] - 2
        if reduced >= 2 and reduced not in tried:
            try:
                cand = evaluate(reduced)
                if cand[2].delta <= spec.max_error:
                    accepted = cand
            except ValidationError:
                pass
    return finish(accepted)
