"""CPU, world_size 2 over gloo: the N > 1 path of the sharded run.

Each rank takes its block-range shard (paper_2406_14116_b200.shard.block_shards), computes it from
its halo-extended input slice with the CPU oracle (standing in for the GPU kernel, which is
covered by the GPU tests), and rank 0 gathers: the concatenation must equal the unsharded output
bit for bit. Also exercises bench.py's barrier / max-over-ranks helpers under a real process group.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_output(port, n, l, dn, blo, bhi, v, x, sched, s):
    m = n - l + 1
    pre = s.y_begin - s.x_begin
    pad = (m - pre % m) % m
    xs = np.concatenate([np.zeros(pad), x[s.x_begin:s.x_end]])
    lead = (pad + pre) // m
    sch = np.concatenate([np.full(lead, sched[s.blk_begin]), sched[s.blk_begin:s.blk_end]])
    sch = sch[: (xs.size + m - 1) // m].astype(np.int32)
    ys = port.ols_real(n, l, dn, blo, bhi, v, xs, bsched=sch)
    return ys[pad + pre: pad + pre + (s.y_end - s.y_begin)]


def _worker(rank, world, port_no, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from oracle import oracle as O
        from paper_2406_14116_b200.shard import block_shards
        port = O.port()
        n, l, dn, blo, bhi = 512, 129, 8, 4, 251
        m = n - l + 1
        v = port.rng_uniform(77, 0.0, 1.0, dn - 1)
        S = m * 29 + 100
        x = port.rng_uniform(78, -1.0, 1.0, S)
        sched = port.rng_uniform_int(79, blo, bhi, (S + m - 1) // m)
        sh = block_shards(S, n, m, world)[rank]
        y = _shard_output(port, n, l, dn, blo, bhi, v, x, sched, sh)
        t = torch.zeros(S, dtype=torch.float64)
        t[sh.y_begin:sh.y_end] = torch.from_numpy(y)
        dist.all_reduce(t)  # disjoint supports: the sum is the concatenation
        bench.barrier(world)
        mx = bench.max_over_ranks(float(rank + 1), world)
        if rank == 0:
            full = port.ols_real(n, l, dn, blo, bhi, v, x, bsched=sched)
            result_q.put((bool(np.array_equal(t.numpy(), full)), mx))
    finally:
        dist.destroy_process_group()


def test_two_rank_block_sharding_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    equal, mx = q.get(timeout=10)
    assert equal
    assert mx == 2.0


def test_bench_launcher_two_ranks_dry_run():
    """`python bench.py --gpus 2 --dry-run` re-launches itself under torch.distributed.run with two
    ranks (gloo, no GPU): both ranks report world size 2, the reductions see every rank, and the
    channel shards tile the 1024 C3 channels; the single-stream C4 shards tile its 2^31 samples."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for cfg in ("c3", "c4"):
        r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--config", cfg],
                           capture_output=True, text=True, timeout=300, cwd=root)
        assert r.returncode == 0, r.stderr[-2000:]
        lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
        assert sorted(l["rank"] for l in lines) == [0, 1]
        assert all(l["n_gpus"] == 2 and l["max_rank_seen"] == 1.0 for l in lines)
        plans = sorted((l["plan"] for l in lines), key=lambda p: (p["ch0"], p["y0"]))
        if cfg == "c3":
            assert [(p["ch0"], p["ch1"]) for p in plans] == [(0, 512), (512, 1024)]
        else:
            assert plans[0]["y0"] == 0 and plans[0]["y1"] == plans[1]["y0"] and plans[1]["y1"] == 2 ** 31
            assert plans[1]["y0"] - plans[1]["x0"] == 1024  # the (N - M)-sample halo


def test_bench_rejects_world_mismatch():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=120, cwd=root, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1 but --gpus 2" in r.stderr
