"""The design-side CLI verbs (`design`, `analyze`; reference fcvbw_cli.cpp:44-70,120-193) against
fixtures produced by the reference's own code (tests/golden/make_cli_golden.py ->
tests/golden/cli/).

- `design`: artifact and verification report byte-identical (the GPU design and the exact GPU
  verify are bit-compatible with the reference; the JSON writers follow nlohmann's layout).
- `analyze`: identical file set, every file byte-identical (responses evaluated in the reference's
  operation order with a restatement of glibc's hypot, csrc/response.cuh).
- exit codes 3 (unreachable max_error) and 2 (off-grid spec, with the nearest-grid suggestion).
"""
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "cli")


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2406_14116_b200", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=600)


# ------------------------------------------------------------------ CPU: host-side formats
def test_artifact_writer_matches_reference_bytes(tmp_path):
    from paper_2406_14116_b200.io import load_artifact, save_artifact
    src = os.path.join(GOLD, "range_artifact.json")
    out = tmp_path / "a.json"
    save_artifact(str(out), load_artifact(src))
    assert out.read_bytes() == open(src, "rb").read()


def test_parse_spec_file(tmp_path):
    from paper_2406_14116_b200 import ValidationError
    from paper_2406_14116_b200.io import parse_spec_file
    spec, opt = parse_spec_file(os.path.join(GOLD, "range.spec"))
    assert spec.transition_width == 0.25 * math.pi and spec.band_center_high == 0.5 * math.pi
    assert spec.max_error == 0.3 and opt.grid_points == 1000
    p = tmp_path / "s.spec"
    p.write_text("transition_width = 0.25pi\nN = 64\nL=15 # comment\ngrid_K = 256\n\nfacets_P = 8\n"
                 "ripple_pass = 0.01\nripple_stop = 0.01\nmax_error = 0.3\nb_low = pi\nb_high = 1e0\n")
    spec, opt = parse_spec_file(str(p))
    assert (opt.fft_length_override, opt.filter_length_override, opt.grid_points, opt.facets) == (64, 15, 256, 8)
    assert spec.band_center_low == math.pi and spec.band_center_high == 1.0
    for bad, what in [("colour = 3\n", "unknown key"), ("max_error 0.3\n", "expected key = value"),
                      ("max_error = 0.3x\n", "malformed number")]:
        p.write_text(bad)
        with pytest.raises(ValidationError, match=what):
            parse_spec_file(str(p))
    p.write_text("max_error = 0.3\n")
    with pytest.raises(ValidationError, match="missing one of"):
        parse_spec_file(str(p))


# ------------------------------------------------------------------ GPU: the verbs
def _ulps(a: float, b: float) -> float:
    if a == b:
        return 0.0
    return abs(a - b) / max(np.spacing(abs(a)), np.spacing(abs(b)))


def _compare_csv(got_path, want_path, numeric_cols):
    got = open(got_path).read().split("\n")
    want = open(want_path).read().split("\n")
    assert len(got) == len(want), got_path
    worst = 0.0
    for g, w in zip(got, want):
        gs, ws = g.split(","), w.split(",")
        assert len(gs) == len(ws)
        for i, (x, y) in enumerate(zip(gs, ws)):
            if i in numeric_cols and x and y:
                worst = max(worst, _ulps(float(x), float(y)))
            else:
                assert x == y, (got_path, g, w)
    assert worst <= 4, (got_path, worst)
    return worst


@pytest.mark.gpu
def test_cli_design_matches_reference(tmp_path):
    art, rep = tmp_path / "a.json", tmp_path / "v.json"
    r = _cli("design", "--spec", os.path.join(GOLD, "range.spec"), "--artifact", str(art), "--verify-report",
             str(rep))
    assert r.returncode == 0, r.stderr
    assert "design: L = 15, N = 64" in r.stdout
    assert art.read_bytes() == open(os.path.join(GOLD, "range_artifact.json"), "rb").read()
    assert rep.read_bytes() == open(os.path.join(GOLD, "range_verify.json"), "rb").read()
    got, want = json.loads(rep.read_text()), json.load(open(os.path.join(GOLD, "range_verify.json")))
    assert sorted(got) == sorted(want)
    assert got["pass"] == want["pass"] and got["within_bound"] == want["within_bound"]
    assert got["dense_points"] == want["dense_points"] and got["worst"]["b"] == want["worst"]["b"]
    for k in ("delta", "passband_max", "stopband_max", "refinement_bound"):
        assert abs(got[k] - want[k]) <= 1e-12, k
    assert sorted(got["per_b_max"]) == sorted(want["per_b_max"])
    for b in want["per_b_max"]:
        assert abs(got["per_b_max"][b] - want["per_b_max"][b]) <= 1e-12
    assert np.abs(np.array(got["per_n_max"]) - np.array(want["per_n_max"])).max() <= 1e-12


@pytest.mark.gpu
def test_cli_design_exit_codes(tmp_path):
    r = _cli("design", "--spec", os.path.join(GOLD, "hard.spec"), "--artifact", str(tmp_path / "a.json"),
             "--verify-report", str(tmp_path / "v.json"))
    assert r.returncode == 3, r.stderr
    r = _cli("design", "--spec", os.path.join(GOLD, "offgrid.spec"), "--artifact", str(tmp_path / "a.json"),
             "--verify-report", str(tmp_path / "v.json"))
    assert r.returncode == 2 and "nearest grid spec" in r.stderr, r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["all", "one"])
def test_cli_analyze_matches_reference(tmp_path, mode):
    art = os.path.join(GOLD, "range_artifact.json")
    prefix = str(tmp_path / mode)
    args = ["analyze", "--artifact", art, "--grid", "128", "--out-prefix", prefix]
    if mode == "one":
        args += ["--b", "12", "--per-phase"]
    r = _cli(*args)
    assert r.returncode == 0, r.stderr
    want = sorted(f for f in os.listdir(GOLD) if f.startswith(mode + "_"))
    got = sorted(os.listdir(tmp_path))
    assert got == want
    for f in want:
        g, w = os.path.join(tmp_path, f), os.path.join(GOLD, f)
        if open(g, "rb").read() != open(w, "rb").read():
            # report how far off the numbers are before failing
            worst = _compare_csv(g, w, {3, 4, 5} if f.endswith("_response.csv") else {3, 4})
            pytest.fail(f"{f} differs from the reference's bytes (worst {worst} ulp)")


@pytest.mark.gpu
def test_error_on_grid_matches_response_table():
    from paper_2406_14116_b200.analysis import error_on_grid, response_table
    from paper_2406_14116_b200.io import load_artifact
    res = load_artifact(os.path.join(GOLD, "range_artifact.json"))
    em = error_on_grid(res, 128, 12)
    t = response_table(res, 128, [12])
    masked = t.grid.region(12) != 2
    assert em.abs_error.shape == (res.bins.block_length, int(masked.sum()))
    assert np.array_equal(em.abs_error.max(axis=0), t.e_max[0][masked])
    assert em.max_abs == np.nanmax(t.e_max[0]) and 0 <= em.worst_n < res.bins.block_length


def test_cli_analyze_bad_b_is_an_error_not_a_traceback(tmp_path):
    """`--b abc` (no integer prefix, where the reference's std::stoi throws) -> 'error: ...', exit 1;
    a prefix such as '12abc' parses as 12 like std::stoi (then the range check applies)."""
    art = os.path.join(GOLD, "range_artifact.json")
    r = _cli("analyze", "--artifact", art, "--grid", "128", "--b", "abc", "--out-prefix", str(tmp_path / "a"))
    assert r.returncode == 1 and r.stderr.startswith("error:") and "Traceback" not in r.stderr
    r = _cli("analyze", "--artifact", art, "--grid", "128", "--b", "999x", "--out-prefix", str(tmp_path / "b"))
    assert r.returncode == 2 and "Traceback" not in r.stderr  # parsed as 999: outside the design range
