"""GPU design verification: the reference's ``verify()`` (proj/include/fcvbw/design.hpp:601-673).

``verify(result, dense_points, delta_e)`` re-evaluates a design's true worst-case error over every
band centre b, output phase n and dense-grid frequency omega, and returns a
``VerificationReport`` with the reference's fields (design.hpp:584-597). The sweep runs in
``libfcvbw_gpu.so`` (csrc/verify.cu); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .bins import DesignResult
from .engine import _raise


@dataclass
class VerificationReport:
    delta: float = 0.0  # dense-grid worst case over all (n, b)
    per_b_max: dict = field(default_factory=dict)
    per_n_max: list = field(default_factory=list)
    passband_max: float = 0.0
    stopband_max: float = 0.0
    dense_points: int = 0
    worst_b: int = -1
    worst_n: int = -1
    worst_omega: float = 0.0
    passed: bool = False  # the reference's `pass`
    refinement_bound: float = 0.0  # delta_achieved * sec(pi/P) + 1e-9
    within_bound: bool = False


# The shift rule `calibrated_shift_rule` (design.hpp:476-484) measures for the overlap-save engine:
# output phase n reads the base row shifted by step * (n - (M - 1)) with window offset 1 - M
# (ptvir.hpp:52-56). tests/test_verify.py pins it against the compiled reference, and
# `calibrated_shift_rule` below re-measures it on the GPU engine.
OLS_SHIFT_STEP = 1

_RULES: dict = {}


def calibrated_shift_rule(bins, device: int = 0) -> tuple[int, int]:
    """calibrated_shift_rule (design.hpp:476-484) measured on this library's GPU engine by impulse
    probing (fcvbw_gpu_calibrate_shift); cached per (N, L) like design()'s rule_cache
    (design.hpp:494-506). Returns (window_offset, step)."""
    key = (bins.fft_length, bins.filter_length)
    if key not in _RULES:
        d = _lib.Design(bins.fft_length, bins.filter_length, bins.block_length, bins.transition_width_bins,
                        bins.b_low, bins.b_high, None, 0, 0.0, 0, 0)
        wo, st = C.c_int(0), C.c_int(0)
        _raise(_lib.lib().fcvbw_gpu_calibrate_shift(C.byref(d), int(device), C.byref(wo), C.byref(st)))
        _RULES[key] = (wo.value, st.value)
    return _RULES[key]


def verify(result: DesignResult, dense_points: int, delta_e: float, device: int = 0,
           exact: bool = False) -> VerificationReport:
    """exact=False: prefix-sum evaluation, O(num_b K (N + M)), agrees with the reference to ~1e-14.
    exact=True: the reference's own per-row sums on the device, bit-identical report."""
    bins = result.bins
    m = bins.fft_length - bins.filter_length + 1
    v = np.ascontiguousarray(result.profile.values, dtype=np.float64)
    d = _lib.Design(bins.fft_length, bins.filter_length, m, bins.transition_width_bins, bins.b_low, bins.b_high,
                    v.ctypes.data_as(C.POINTER(C.c_double)), len(v), float(result.delta), int(result.grid_points),
                    int(result.facets))
    per_b = np.zeros(bins.b_high - bins.b_low + 1)
    per_n = np.zeros(m)
    rep = _lib.Verification()
    fn = _lib.lib().fcvbw_gpu_verify_exact if exact else _lib.lib().fcvbw_gpu_verify
    _raise(fn(C.byref(d), int(dense_points), float(delta_e), 1 - m, OLS_SHIFT_STEP, int(device), per_b.ctypes.data,
              per_n.ctypes.data, C.byref(rep)))
    return VerificationReport(
        delta=rep.delta, per_b_max={bins.b_low + i: float(x) for i, x in enumerate(per_b)},
        per_n_max=per_n.tolist(), passband_max=rep.passband_max, stopband_max=rep.stopband_max,
        dense_points=rep.dense_points, worst_b=rep.worst_b, worst_n=rep.worst_n, worst_omega=rep.worst_omega,
        passed=bool(rep.pass_), refinement_bound=rep.refinement_bound, within_bound=bool(rep.within_bound))
