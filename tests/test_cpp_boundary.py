"""The C-ABI from C and C++: the plain-C header check runs on the CPU; the C++ adapter parity
program (reference headers as checker, fcvbw::gpu::OlsEngineGpu as the engine) runs on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")


def _bin(name):
    p = os.path.join(BUILD, name)
    if not os.path.exists(p):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=False)
    if not os.path.exists(p):
        pytest.skip(f"{name} not built")
    return p


def test_c_abi_header_from_c():
    r = subprocess.run([_bin("abi_c_check")], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS create(N=100) -> 2" in r.stdout


@pytest.mark.gpu
def test_cpp_adapter_parity_program():
    r = subprocess.run([_bin("test_gpu_adapter")], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
    assert r.stdout.count("PASS") >= 10


@pytest.mark.gpu
def test_cpp_cmd_run_drop_in():
    """The reference CLI's run loop with only the engine factory swapped (tests/cpp/test_cmd_run.cpp):
    exit 2 on out-of-range schedules, f64le bitwise equal to the in-process engine, OpCounters."""
    r = subprocess.run([_bin("test_cmd_run")], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
    assert r.stdout.count("PASS") >= 8
