"""Generate the V(r) design artifacts for the BASELINE configs with the REFERENCE's own design()
(proj/include/fcvbw/design.hpp:486-577, fixed (N, L) via both overrides), through the compiled
reference in oracle/_ref (needs /root/reference, i.e. run in the build container).

Artifacts use the reference's on-disk field names (proj/include/fcvbw/io.hpp:34-47) plus a
"provenance" object. bN_low/bN_high are widened to the admissible range of the TARGET geometry so
that every scheduled b validates (the engine does not require V to have been designed over that
range, proj/include/fcvbw/engine.hpp:31-45). For N >= 2048 the reference's true-geometry design
is impractical on the CPU (cost ~N^3; one band centre runs on one thread), so the
reference path designs those at a proxy N_p = 512, L_p = 129 with the same delta_N (SURVEY.md
Appendix A).

`--gpu NAME...` instead designs at TRUE geometry with this repository's GPU-assisted
solve_minimax (paper_2406_14116_b200/design.py, csrc/design.cu), which reproduces the reference's
design() bit for bit where both can run (tests/test_design.py, profiles/r01_design.md). It needs a
GPU (run it through gpurun); the default --gpu set is the proxy artifacts.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import oracle as O  # noqa: E402

# name: (N, delta_N, design_N, design_L)
TARGETS = {
    "n64_d4": (64, 4, 64, 17),
    "n128_d4": (128, 4, 128, 33),
    "n256_d6": (256, 6, 256, 65),
    "n512_d8": (512, 8, 512, 129),
    "n1024_d12": (1024, 12, 1024, 257),
    "n2048_d16": (2048, 16, 512, 129),
    "n4096_d16": (4096, 16, 512, 129),
    "n4096_d24": (4096, 24, 512, 129),
    "n8192_d32": (8192, 32, 512, 129),
}


def main_gpu(names):
    from paper_2406_14116_b200 import BinSpec
    from paper_2406_14116_b200.design import DesignOptions, solve_minimax
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for name in names:
        n, dn, _, _ = TARGETS[name]
        l = n // 4 + 1
        b = n // 8  # design at 0.25*pi, as the reference path
        t0 = time.time()
        out = solve_minimax(BinSpec(n, l, n - l + 1, dn, b, b), DesignOptions(grid_points=2 * n))
        el = time.time() - t0
        art = {
            "N": n, "L": l, "M": n - l + 1, "delta_N": dn,
            "bN_low": dn // 2, "bN_high": n // 2 - dn // 2 - 1,
            "V": [float(x) for x in out.profile.values],
            "delta_achieved": out.delta, "grid_K": 2 * n, "facets_P": 16,
            "provenance": {
                "tool": "GPU solve_minimax (paper_2406_14116_b200/design.py, csrc/design.cu) at true geometry "
                        "(configs/make_artifacts.py --gpu)",
                "design_N": n, "design_L": l, "design_b": b, "grid_K": 2 * n,
                "proxy": False, "seconds": round(el, 2), "exchange_rounds": out.rounds,
            },
        }
        with open(os.path.join(out_dir, f"artifact_{name}.json"), "w") as f:
            json.dump(art, f, indent=2)
            f.write("\n")
        print(f"{name}: delta={out.delta:.3e} in {el:.1f}s (rounds {out.rounds})", flush=True)


def main(names):
    ref = O.reference()
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for name in names:
        n, dn, dn_n, dl = TARGETS[name]
        path = os.path.join(out_dir, f"artifact_{name}.json")
        if os.path.exists(path):
            continue
        b = dn_n // 8  # design at 0.25*pi
        t0 = time.time()
        v, delta = ref.design(dn_n, dl, dn, b, b, 2 * dn_n)
        el = time.time() - t0
        l = n // 4 + 1
        art = {
            "N": n, "L": l, "M": n - l + 1, "delta_N": dn,
            "bN_low": dn // 2, "bN_high": n // 2 - dn // 2 - 1,
            "V": [float(x) for x in v],
            "delta_achieved": delta, "grid_K": 2 * dn_n, "facets_P": 16,
            "provenance": {
                "tool": "reference design() via oracle/_ref/libfcvbw_ref.so (configs/make_artifacts.py)",
                "design_N": dn_n, "design_L": dl, "design_b": b, "grid_K": 2 * dn_n,
                "proxy": dn_n != n, "seconds": round(el, 2),
            },
        }
        with open(path, "w") as f:
            json.dump(art, f, indent=2)
            f.write("\n")
        print(f"{name}: delta={delta:.3e} in {el:.1f}s", flush=True)


if __name__ == "__main__":
    if sys.argv[1:2] == ["--gpu"]:
        main_gpu(sys.argv[2:] or [k for k, t in TARGETS.items() if t[0] != t[2]])
    else:
        main(sys.argv[1:] or list(TARGETS))
