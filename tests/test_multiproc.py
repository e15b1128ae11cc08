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
