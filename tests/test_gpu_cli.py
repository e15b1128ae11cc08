"""The GPU `run` verb, re-expressing the reference CLI tests for `run`
(proj/tests/test_cli.cpp:123-163): f64le output bitwise equal to the in-process engine, a zero
stream gives zeros, an out-of-range schedule entry exits 2, and (new) the output matches the
reference engine on the same artifact / signal / schedule."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_14116_b200 import load_artifact, new_engine, schedule_to_blocks
from paper_2406_14116_b200.io import write_signal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2406_14116_b200", "run", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=300)


@pytest.fixture()
def artifact(tmp_path):
    # the narrowband reference example geometry with a seeded profile (test_spectrum.cpp:18-25)
    a = {"N": 128, "L": 33, "M": 96, "delta_N": 16, "bN_low": 48, "bN_high": 55,
         "V": list(O.port().rng_uniform(3, 0.0, 1.0, 15)), "delta_achieved": 0.0, "grid_K": 256, "facets_P": 16}
    p = tmp_path / "design.json"
    p.write_text(json.dumps(a))
    return str(p)


def test_run_f64le_bitwise_equals_in_process_engine(tmp_path, artifact):
    x = O.port().rng_uniform(7, -1.0, 1.0, 96 * 20 + 13)
    inp, out, sch = tmp_path / "x.f64", tmp_path / "y.f64", tmp_path / "s.csv"
    write_signal(str(inp), x, "f64le")
    sch.write_text("0,48\n5,55\n11,50\n")
    r = cli("--artifact", artifact, "--input", str(inp), "--output", str(out), "--format", "f64le",
            "--schedule", str(sch))
    assert r.returncode == 0, r.stderr
    assert "switches applied = 3" in r.stdout
    y = np.fromfile(str(out), "<f8")
    res = load_artifact(artifact)
    sched = schedule_to_blocks([(0, 48), (5, 55), (11, 50)], 21, 48, res.bins)
    eng = new_engine(res, 48)
    y_eng = eng.run_real_host(x, sched)
    assert np.array_equal(y, y_eng)
    assert O.rel_rms(y, eng.run_host(x.astype(np.complex128), sched).real) <= 1e-14
    yr = O.best().ols_real(128, 33, 16, 48, 55, np.array(res.profile.values), x, bsched=sched)
    assert np.max(np.abs(y - yr)) <= 1e-12


def test_run_zero_stream_csv(tmp_path, artifact):
    inp, out = tmp_path / "z.csv", tmp_path / "o.csv"
    inp.write_text("0\n" * 300)
    r = cli("--artifact", artifact, "--input", str(inp), "--output", str(out))
    assert r.returncode == 0, r.stderr
    vals = [float(l) for l in out.read_text().split()]
    assert len(vals) == 300 and all(v == 0.0 for v in vals)


def test_run_out_of_range_schedule_exits_2(tmp_path, artifact):
    inp, out, sch = tmp_path / "x.csv", tmp_path / "o.csv", tmp_path / "bad.csv"
    inp.write_text("1\n" * 200)
    sch.write_text("0,48\n1,56\n")
    r = cli("--artifact", artifact, "--input", str(inp), "--output", str(out), "--schedule", str(sch))
    assert r.returncode == 2
    assert "outside the design range" in r.stderr
    sch.write_text("0,48\n99,50\n")  # beyond the stream (3 blocks)
    r = cli("--artifact", artifact, "--input", str(inp), "--output", str(out), "--schedule", str(sch))
    assert r.returncode == 2
