"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
variant family runs once on small inputs (fp32 N=1024 with the exchange-buffer TMA prefetch,
fp32 N=8192 with the staging-buffer TMA prefetch, multi-group-per-warp N=64/256, fp64, even-L
phase multiply, raw table, streaming feed/flush, schedule check, coefficient dump).

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2406_14116_b200 import BinSpec, OlsEngine, TransitionProfile  # noqa: E402
from paper_2406_14116_b200.workload import complex_gaussian  # noqa: E402


def run(n, l, dn, dtype, blocks, ch=2, **kw):
    bins = BinSpec(n, l, n - l + 1, dn, dn // 2, n // 2 - dn // 2 - 1)
    m = bins.block_length
    S = m * blocks + m // 3 + 1
    rng = np.random.default_rng(n)
    v = TransitionProfile(list(rng.uniform(0, 1, dn - 1)))
    x = np.stack([complex_gaussian(c, 0, S, np.complex64 if dtype == "c64" else np.complex128) for c in range(ch)])
    nb = (S + m - 1) // m
    sched = rng.integers(bins.b_low, bins.b_high + 1, size=(ch, nb)).astype(np.int32)
    eng = OlsEngine(bins, v, int(sched[0, 0]), dtype=dtype, **kw)
    y = eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(sched).cuda())
    torch.cuda.synchronize()
    eng.coeff_dump(sched[0, :4])
    return float(torch.abs(y).sum())


def main():
    out = []
    out.append(run(1024, 257, 12, "c64", 300))
    out.append(run(8192, 2049, 32, "c64", 6))
    out.append(run(64, 17, 4, "c64", 200))
    out.append(run(256, 65, 6, "c128", 100))
    out.append(run(512, 129, 8, "c128", 60))
    out.append(run(4096, 1025, 16, "c128", 6, ch=1))
    out.append(run(64, 20, 6, "c128", 40, ch=1))  # even L: phase-table multiply
    out.append(run(1024, 257, 12, "c64", 40, ch=1, force_phase_multiply=True))
    t = np.fft.fft(np.r_[np.random.default_rng(1).uniform(-1, 1, 33), np.zeros(95)])
    raw = OlsEngine.raw(t, 96)
    x = np.random.default_rng(2).uniform(-1, 1, 96 * 7 + 5)
    y = np.concatenate([raw.feed(x[:100]), raw.feed(x[100:]), raw.flush()])
    out.append(float(np.abs(y).sum()))
    print("sanitize driver done", ["%.3e" % v for v in out])


if __name__ == "__main__":
    main()
