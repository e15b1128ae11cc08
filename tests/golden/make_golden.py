"""Generate the golden vectors in tests/golden/ from the REFERENCE implementation itself:
the unmodified reference headers compiled in place (oracle/_ref/libfcvbw_ref.so, built by
`make -C oracle ref` from /root/reference). Run in the build container:

    python tests/golden/make_golden.py

Every fixture records its generating call. Inputs come from the reference's SeededRng
(proj/include/fcvbw/ops.hpp:62-86) so they are reproducible from the seeds alone.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import oracle as O  # noqa: E402


def main():
    ref = O.reference()
    out = {}
    # 1. narrowband example (test_spectrum.cpp:18-25): N=128, L=33, M=96, dN=16, b in [48, 55]
    n, l, dn, blo, bhi = 128, 33, 16, 48, 55
    v = ref.rng_uniform(3, 0.0, 1.0, 15)  # test_spectrum.cpp:81-83
    out["nb_V"] = v
    for b in range(blo, bhi + 1):
        mag, reg, tab = ref.coefficients(n, l, dn, blo, bhi, v, b)
        out[f"nb_mag_b{b}"] = mag
        out[f"nb_region_b{b}"] = reg
        out[f"nb_table_b{b}"] = tab
    # 2. phase tables
    for (pn, pl) in [(128, 33), (64, 17), (1024, 257), (64, 20), (32, 25)]:
        out[f"phase_{pn}_{pl}"] = ref.phase_table(pn, pl)
    # 3. real-stream engine outputs with a retune schedule (test_oracle_engine.cpp:183-197 style)
    x = ref.rng_uniform(59, -1.0, 1.0, 96 * 24 + 7)
    sched = np.array([48] * 10 + [55] * 7 + [51] * 8, np.int32)
    ve = ref.rng_uniform(58, 0.0, 1.0, 15)
    out["eng_x"], out["eng_V"], out["eng_sched"] = x, ve, sched
    out["eng_y"] = ref.ols_real(n, l, dn, blo, bhi, ve, x, bsched=sched)
    _, _, tab48 = ref.coefficients(n, l, dn, blo, bhi, ve, 48)
    out["naive_y_b48"] = ref.naive_block_filter(n, 96, tab48, x)
    # 4. complex composite streams at BASELINE geometries (small sizes)
    for name, (cn, cdn, seed, S) in {"c1like": (512, 8, 0, 384 * 11 + 100), "c2like": (1024, 12, 1, 768 * 9 + 300),
                                     "c4like": (4096, 16, 3, 3072 * 5 + 2048)}.items():
        cl = cn // 4 + 1
        cv = ref.rng_uniform(100 + seed, 0.0, 1.0, cdn - 1)
        xr = ref.rng_uniform(200 + seed, -1.0, 1.0, S)
        xi = ref.rng_uniform(300 + seed, -1.0, 1.0, S)
        xc = xr + 1j * xi
        nb = (S + (cn - cl + 1) - 1) // (cn - cl + 1)
        cs = ref.rng_uniform_int(400 + seed, cdn // 2, cn // 2 - cdn // 2 - 1, nb)
        out[f"{name}_V"], out[f"{name}_x"], out[f"{name}_sched"] = cv, xc, cs
        out[f"{name}_y"] = ref.ols_complex(cn, cl, cdn, cdn // 2, cn // 2 - cdn // 2 - 1, cv, xc, bsched=cs, threads=4)
    # 5. classical OLS vs direct FIR (test_oracle_engine.cpp:290-307)
    h = ref.rng_uniform(69, -1.0, 1.0, 33)
    xf = ref.rng_uniform(70, -1.0, 1.0, 96 * 4 + 31)
    out["fir_h"], out["fir_x"] = h, xf
    out["fir_y"] = ref.direct_fir(h, xf)
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
