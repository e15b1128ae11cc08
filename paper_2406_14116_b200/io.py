"""File formats on either side of the hot path (the `fcvbw run` inputs and output):
design artifact JSON, schedule CSV, f64le / CSV signals.

Mirrors proj/include/fcvbw/io.hpp:34-79 (artifact), :152-207 (signals), :213-248 (schedule) and
the schedule checks of proj/tools/fcvbw_cli.cpp:25-42, 85-93. Host-side, run once per job.
"""
from __future__ import annotations

import json
import math
import re

import numpy as np

from .bins import BinSpec, DesignResult, Error, TransitionProfile, ValidationError


def artifact_from_json(j: dict) -> DesignResult:
    """artifact_from_json (io.hpp:49-65): validates BinSpec and |V| = delta_N - 1."""
    try:
        bins = BinSpec(int(j["N"]), int(j["L"]), int(j["M"]), int(j["delta_N"]), int(j["bN_low"]), int(j["bN_high"]))
        res = DesignResult(
            profile=TransitionProfile([float(v) for v in j["V"]]),
            bins=bins,
            delta=float(j["delta_achieved"]),
            grid_points=int(j["grid_K"]),
            facets=int(j["facets_P"]),
            provenance=dict(j.get("provenance", {})),
        )
    except KeyError as e:
        raise Error(f"artifact: missing field {e}") from None
    bins.validate()
    if res.profile.length() != bins.profile_length():
        raise ValidationError("artifact: V must hold delta_N - 1 values")
    return res


def artifact_to_json(res: DesignResult) -> dict:
    """artifact_to_json (io.hpp:34-47)."""
    j = {
        "N": res.bins.fft_length, "L": res.bins.filter_length, "M": res.bins.block_length,
        "delta_N": res.bins.transition_width_bins, "bN_low": res.bins.b_low, "bN_high": res.bins.b_high,
        "V": list(res.profile.values), "delta_achieved": res.delta, "grid_K": res.grid_points,
        "facets_P": res.facets,
    }
    if res.provenance:
        j["provenance"] = res.provenance
    return j


def load_artifact(path: str) -> DesignResult:
    try:
        with open(path) as f:
            return artifact_from_json(json.load(f))
    except OSError:
        raise Error(f"cannot read {path}") from None


def save_artifact(path: str, res: DesignResult) -> None:
    """save_artifact (io.hpp:67-71): keys in nlohmann's (sorted) order, 2-space indent."""
    try:
        with open(path, "w") as f:
            json.dump(artifact_to_json(res), f, indent=2, sort_keys=True)
            f.write("\n")
    except OSError:
        raise Error(f"cannot write {path}") from None


def verification_to_json(report) -> dict:
    """verification_to_json (io.hpp:81-96) of a VerificationReport (paper_2406_14116_b200.verify)."""
    return {
        "delta": report.delta,
        "per_b_max": {str(b): v for b, v in sorted(report.per_b_max.items())},
        "per_n_max": list(report.per_n_max),
        "pass": report.passed,
        "passband_max": report.passband_max,
        "stopband_max": report.stopband_max,
        "dense_points": report.dense_points,
        "worst": {"b": report.worst_b, "n": report.worst_n, "omega": report.worst_omega},
        "refinement_bound": report.refinement_bound,
        "within_bound": report.within_bound,
    }


def save_verification(path: str, report) -> None:
    try:
        with open(path, "w") as f:
            json.dump(verification_to_json(report), f, indent=2, sort_keys=True)
            f.write("\n")
    except OSError:
        raise Error(f"cannot write {path}") from None


def _parse_angle(text: str) -> float:
    """detail::parse_angle (io.hpp:275-293): a number with an optional 'pi' suffix (std::stod)."""
    text = text.strip(" \t").rstrip(" \t\r")
    scale = 1.0
    if len(text) >= 2 and text.endswith("pi"):
        scale = math.pi
        text = text[:-2].strip(" \t").rstrip(" \t\r")
        if not text:
            return scale
    m = _NUM.match(text)
    if not m:
        raise Error("stod")  # std::invalid_argument: not a ValidationError (CLI exit 1)
    if m.end() != len(text):
        raise ValidationError(f"malformed number '{text}'")
    return float(text) * scale


def parse_spec_file(path: str):
    """parse_spec_file (io.hpp:296-353): 'key = value' lines, '#' comments -> (FilterSpec, DesignOptions)."""
    from .design import DesignOptions, FilterSpec
    try:
        lines = open(path).read().split("\n")
    except OSError:
        raise Error(f"cannot read {path}") from None
    if lines and lines[-1] == "":
        lines.pop()
    spec, opt = FilterSpec(), DesignOptions()
    have = set()
    fields = {"transition_width": "transition_width", "ripple_pass": "ripple_pass", "ripple_stop": "ripple_stop",
              "max_error": "max_error", "b_low": "band_center_low", "b_high": "band_center_high"}
    options = {"N": "fft_length_override", "L": "filter_length_override", "grid_K": "grid_points",
               "facets_P": "facets"}
    for no, line in enumerate(lines, 1):
        line = line.split("#", 1)[0]
        if "=" not in line:
            if line.strip(" \t\r") == "":
                continue
            raise ValidationError(f"{path}:{no}: expected key = value")
        key, value = line.split("=", 1)
        key = key.lstrip(" \t").rstrip(" \t\r")
        try:
            if key in fields:
                setattr(spec, fields[key], _parse_angle(value))
                have.add(key)
            elif key in options:
                setattr(opt, options[key], int(_parse_angle(value)))
            else:
                raise ValidationError(f"unknown key '{key}'")
        except ValidationError as e:
            raise ValidationError(f"{path}:{no}: {e}") from None
    if len(have) != len(fields):
        raise ValidationError(f"{path}: missing one of transition_width, ripple_pass, ripple_stop, max_error, "
                              "b_low, b_high")
    return spec, opt


_NUM = re.compile(r"^\s*[+-]?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan)", re.I)
_INT = re.compile(r"^\s*[+-]?\d+")


def read_signal(path: str, fmt: str = "csv") -> np.ndarray:
    """read_signal (io.hpp:174-207): f64le raw doubles, or one strtod value per CSV line with only
    spaces / CR allowed after it."""
    if fmt == "f64le":
        try:
            raw = open(path, "rb").read()
        except OSError:
            raise Error(f"cannot read {path}") from None
        if len(raw) % 8:
            raise ValidationError(f"{path}: size is not a multiple of 8 bytes")
        return np.frombuffer(raw, dtype="<f8").astype(np.float64)
    if fmt == "csv":
        vals = []
        try:
            lines = open(path).read().split("\n")
        except OSError:
            raise Error(f"cannot read {path}") from None
        if lines and lines[-1] == "":
            lines.pop()
        for no, line in enumerate(lines, 1):
            if not line:
                continue
            m = _NUM.match(line)
            if not m:
                raise ValidationError(f"{path}:{no}: not a number")
            if line[m.end():].strip(" \r"):
                raise ValidationError(f"{path}:{no}: trailing junk")
            vals.append(float(m.group(0)))
        return np.asarray(vals, np.float64)
    raise ValidationError(f"unknown signal format '{fmt}' (expected csv or f64le)")


def write_signal(path: str, y: np.ndarray, fmt: str = "csv") -> None:
    """write_signal (io.hpp:160-172); CSV uses 17 significant digits (round-trip exact)."""
    y = np.asarray(y, np.float64)
    if fmt == "f64le":
        y.astype("<f8").tofile(path)
    elif fmt == "csv":
        with open(path, "w") as f:
            for v in y:
                f.write("%.17g\n" % v)
    else:
        raise ValidationError(f"unknown signal format '{fmt}' (csv|f64le)")


def read_schedule_csv(path: str) -> list[tuple[int, int]]:
    """read_schedule_csv (io.hpp:218-248): 'block_index,b_N' lines, '#' comments and blank lines
    skipped, block indices >= 0 and strictly increasing; integer prefixes parsed like stoll/stoi."""
    try:
        lines = open(path).read().split("\n")
    except OSError:
        raise Error(f"cannot read {path}") from None
    if lines and lines[-1] == "":
        lines.pop()
    events: list[tuple[int, int]] = []
    for no, line in enumerate(lines, 1):
        if not line or line[0] == "#":
            continue
        if "," not in line:
            raise ValidationError(f"{path}:{no}: expected 'block_index,b_N' (line: {line})")
        a, b = line.split(",", 1)
        ma, mb = _INT.match(a), _INT.match(b)
        if not ma or not mb:
            raise ValidationError(f"{path}:{no}: malformed entry (line: {line})")
        blk, bv = int(ma.group(0)), int(mb.group(0))
        if blk < 0:
            raise ValidationError(f"{path}:{no}: negative block index (line: {line})")
        if events and blk <= events[-1][0]:
            raise ValidationError(f"{path}:{no}: block indices must be strictly increasing (line: {line})")
        events.append((blk, bv))
    return events


def schedule_to_blocks(events, nblocks: int, b0: int, bins: BinSpec | None = None) -> np.ndarray:
    """Expand schedule events into one b per block, exactly as the CLI applies them
    (fcvbw_cli.cpp:85-93, 100-104): b0 until the first event, each event takes effect before
    its named block. Validates range and stream length like load_schedule / cmd_run."""
    out = np.full(nblocks, b0, np.int32)
    for line, (blk, b) in enumerate(events, 1):
        if bins is not None and not bins.contains_b(b):
            raise ValidationError(
                f"schedule entry {line} ({blk},{b}) requests b_N outside the design range [{bins.b_low}, {bins.b_high}]")
        if blk >= nblocks:
            raise ValidationError(f"schedule:{line}: block index {blk} beyond the input stream ({nblocks} blocks)")
        out[blk:] = b
    return out


def blocks_of(samples: int, block_length: int) -> int:
    return int(math.ceil(samples / block_length)) if samples > 0 else 0
