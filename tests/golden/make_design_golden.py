"""Generates tests/golden/design_vectors.json from the UNMODIFIED reference design code
(`solve_minimax`, design.hpp:276-446, and `design`, design.hpp:486-577), compiled in place as
oracle/_ref/libfcvbw_ref.so. Run here (where /root/reference exists):

    python tests/golden/make_design_golden.py

The GPU design tests (tests/test_design.py) compare against these fixtures, so they run on a box
without the reference. Floats are stored with Python's shortest round-trip repr (exact).
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

PI = math.pi

# (name, N, L, delta_N, b_low, b_high, K, facets, exchange_tol, max_rounds, seed_stride)
SOLVE = [
    ("n64_single", 64, 17, 4, 8, 8, 128, 16, 0.025, 60, 16),
    ("n128_single", 128, 33, 4, 16, 16, 256, 16, 0.025, 60, 16),
    ("n128_range5_d8", 128, 97, 8, 20, 24, 256, 16, 0.025, 60, 16),
    ("n256_single_d6", 256, 65, 6, 32, 32, 512, 16, 0.025, 60, 16),
    ("n64_evenL_full", 64, 16, 4, 2, 29, 128, 16, 0.025, 60, 16),
    ("n128_p8_stride8", 128, 65, 6, 10, 12, 256, 8, 0.1, 60, 8),
]

# (name, FilterSpec = (transition_width, ripple_pass, ripple_stop, max_error, b_l, b_u), grid_points)
DESIGN = [
    ("spec_quarter", (PI / 4, 0.01, 0.01, 0.3, PI / 4, PI / 4), 4096),
    ("spec_eighth", (PI / 8, 0.01, 0.01, 0.05, PI / 4, PI / 4), 4096),
    ("spec_sixteenth", (PI / 16, 0.01, 0.01, 0.1, PI / 2, PI / 2), 4096),
]


def main():
    ref = O.reference()
    out = {"generator": "tests/golden/make_design_golden.py via oracle/_ref/libfcvbw_ref.so", "solve": [],
           "design": []}
    for name, n, l, dn, blo, bhi, k, p, tol, rounds, stride in SOLVE:
        t = time.time()
        r = ref.solve_minimax(n, l, dn, blo, bhi, k, p, tol, rounds, stride)
        out["solve"].append(dict(name=name, N=n, L=l, delta_N=dn, b_low=blo, b_high=bhi, grid_points=k, facets=p,
                                 exchange_tol=tol, max_rounds=rounds, seed_stride=stride, V=r["v"].tolist(),
                                 delta=r["delta"], lp_delta=r["lp_delta"], rounds=r["rounds"],
                                 lp_iterations=r["lp_iterations"], active_triples=r["active_triples"],
                                 seconds=round(time.time() - t, 3)))
        print(name, out["solve"][-1]["delta"], out["solve"][-1]["seconds"])
    for name, spec, k in DESIGN:
        t = time.time()
        r = ref.design_full(spec, grid_points=k)
        out["design"].append(dict(name=name, spec=list(spec), grid_points=k, N=r["N"], L=r["L"], delta_N=r["delta_N"],
                                  b_low=r["b_low"], b_high=r["b_high"], iterations=r["iterations"],
                                  exchange_rounds=r["exchange_rounds"], V=r["v"].tolist(), delta=r["delta"],
                                  seconds=round(time.time() - t, 3)))
        print(name, r["N"], r["L"], r["delta"], out["design"][-1]["seconds"])
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "design_vectors.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
