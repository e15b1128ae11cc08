"""Generates tests/golden/cli/ from the reference's own `design` and `analyze` verbs
(oracle/ref_cli_shim.cpp over the unmodified reference headers; the reference CLI binary itself
needs CLI11 and cannot be built here). Run in the build container:

    python tests/golden/make_cli_golden.py

tests/test_cli_design.py (-m gpu) runs this repository's GPU verbs on the same inputs and compares
the files.
"""
import ctypes as C
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "cli")
LIB = os.path.join(ROOT, "oracle", "_ref", "libfcvbw_ref_cli.so")

SPECS = {
    # b range 8..16 at N = 64 (delta_N = 8): several band centres, small tables
    "range.spec": "# analysis fixture\ntransition_width = 0.25pi\nripple_pass = 0.01\nripple_stop = 0.01\n"
                  "max_error = 0.3\nb_low = 0.25pi\nb_high = 0.5pi\n",
    # unreachable error bound: the order loop runs out (exit 3)
    "hard.spec": "transition_width = 0.25pi\nripple_pass = 0.01\nripple_stop = 0.01\nmax_error = 1e-12\n"
                 "b_low = 0.25pi\nb_high = 0.25pi\n",
    # transition width not on the bin grid (exit 2, message names the nearest grid spec)
    "offgrid.spec": "transition_width = 0.3pi\nripple_pass = 0.01\nripple_stop = 0.01\nmax_error = 0.05\n"
                    "b_low = 0.5pi\nb_high = 0.5pi\n",
}


def main():
    lib = C.CDLL(LIB)
    lib.ref_cli_design.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]
    lib.ref_cli_analyze.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_int]
    lib.ref_cli_last_error.restype = C.c_char_p
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    for name, text in SPECS.items():
        with open(os.path.join(OUT, name), "w") as f:
            f.write(text)
    codes = {}
    for name in SPECS:
        stem = name.split(".")[0]
        rc = lib.ref_cli_design(os.path.join(OUT, name).encode(), os.path.join(OUT, f"{stem}_artifact.json").encode(),
                                os.path.join(OUT, f"{stem}_verify.json").encode(), 0)
        codes[name] = (rc, lib.ref_cli_last_error().decode())
        print(name, rc, codes[name][1][:120])
    art = os.path.join(OUT, "range_artifact.json").encode()
    rc1 = lib.ref_cli_analyze(art, 128, -1, os.path.join(OUT, "all").encode(), 0)
    rc2 = lib.ref_cli_analyze(art, 128, 12, os.path.join(OUT, "one").encode(), 1)
    print("analyze", rc1, rc2)
    with open(os.path.join(OUT, "exit_codes.txt"), "w") as f:
        for name, (rc, msg) in codes.items():
            f.write(f"{name} {rc} {msg}\n")
    # drop the stray outputs of the failing designs
    for stem in ("hard", "offgrid"):
        for suffix in ("_artifact.json", "_verify.json"):
            p = os.path.join(OUT, stem + suffix)
            if os.path.exists(p):
                os.remove(p)


if __name__ == "__main__":
    main()
