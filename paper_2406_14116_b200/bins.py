"""Host-side domain model: the reference's BinSpec / TransitionProfile / DesignResult and the
error taxonomy, with the same names, fields, invariants and exception types.

Mirrors proj/include/fcvbw/spectrum.hpp:50-93, design.hpp:463-472 and errors.hpp:7-29
(paths relative to the reference root). Integer index rules only; no floating-point work.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field


class Error(RuntimeError):
    """fcvbw::Error (errors.hpp:8-10); C-ABI status 1."""


class ValidationError(Error):
    """fcvbw::ValidationError (errors.hpp:13-15); C-ABI status 2 / CLI exit 2."""


class OffGridError(ValidationError):
    """fcvbw::OffGridError (errors.hpp:19-21): requirements do not land on the 2 pi / N grid."""


class NonConvergenceError(Error):
    """fcvbw::NonConvergenceError (errors.hpp:23-25); C-ABI status 3 (design side)."""


class LpError(Error):
    """fcvbw::LpError (errors.hpp:27-29); C-ABI status 4 (design side)."""


def _pow2(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


@dataclass
class BinSpec:
    """Exact bin-domain discretization (spectrum.hpp:50-77)."""
    fft_length: int = 0             # N = 2^Q
    filter_length: int = 0          # L
    block_length: int = 0           # M = N - L + 1
    transition_width_bins: int = 0  # delta_N, even
    b_low: int = 0
    b_high: int = 0

    def profile_length(self) -> int:
        return self.transition_width_bins - 1

    def delta(self) -> float:
        return self.transition_width_bins * 2.0 * math.pi / self.fft_length

    def omega_of_bin(self, b: int) -> float:
        return b * 2.0 * math.pi / self.fft_length

    def contains_b(self, b: int) -> bool:
        return self.b_low <= b <= self.b_high

    def validate(self) -> None:
        if self.fft_length < 8 or not _pow2(self.fft_length):
            raise ValidationError("BinSpec: N must be 2^Q with Q >= 3")
        if self.filter_length < 1 or self.filter_length > self.fft_length:
            raise ValidationError("BinSpec: L must satisfy 1 <= L <= N")
        if self.block_length != self.fft_length - self.filter_length + 1:
            raise ValidationError("BinSpec: M must equal N - L + 1")
        if self.transition_width_bins < 2 or self.transition_width_bins % 2 != 0:
            raise ValidationError("BinSpec: delta_N must be a positive even integer")
        half = self.transition_width_bins // 2
        if not (half <= self.b_low <= self.b_high <= self.fft_length // 2 - half - 1):
            raise ValidationError("BinSpec: need delta_N/2 <= b_low <= b_high <= N/2 - delta_N/2 - 1")

    @staticmethod
    def from_geometry(n: int, l: int, dn: int, b_low: int, b_high: int) -> "BinSpec":
        return BinSpec(n, l, n - l + 1, dn, b_low, b_high)


@dataclass
class TransitionProfile:
    """Shared transition-band samples V(r) (spectrum.hpp:81-85)."""
    values: list = field(default_factory=list)

    def length(self) -> int:
        return len(self.values)


@dataclass
class TransitionBand:
    k1: int
    k2: int


def transition_bins(bins: BinSpec, b: int) -> TransitionBand:
    """spectrum.hpp:161-165."""
    if not bins.contains_b(b):
        raise ValidationError("transition_bins: b out of declared range")
    half = bins.transition_width_bins // 2
    return TransitionBand(b - half + 1, b + half - 1)


@dataclass
class DesignResult:
    """The design artifact the engine consumes (design.hpp:463-472; io.hpp:34-65 field names)."""
    profile: TransitionProfile
    bins: BinSpec
    delta: float = 0.0
    grid_points: int = 0
    facets: int = 0
    verification: float = float("nan")
    provenance: dict = field(default_factory=dict)
    iterations: int = 0       # order-loop candidates evaluated
    exchange_rounds: int = 0  # exchange rounds of the accepted candidate
