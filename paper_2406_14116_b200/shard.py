"""Multi-GPU sharding plans for the overlap-save path.

The path shards with no data-path collective:

* channel sharding: independent streams (C3, C5) split across ranks;
* block-range sharding of one long stream (C4): rank r computes global blocks [B_r, B_{r+1}),
  reading input from B_r*M - (N - M) (the (N - M)-sample halo, zero below 0) and indexing the
  b schedule by global block. Because every block depends only on its own N-sample segment and
  its own b (proj/include/fcvbw/engine.hpp:139-172), the concatenated shard outputs are bitwise
  identical to the unsharded run.

Pure host logic (integers only); the device work is fcvbw_gpu_run_range / fcvbw_gpu_run.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class BlockShard:
    rank: int
    blk_begin: int   # global block range [blk_begin, blk_end)
    blk_end: int
    x_begin: int     # global input samples [x_begin, x_end) this shard reads (halo included)
    x_end: int
    y_begin: int     # global output samples [y_begin, y_end) this shard writes
    y_end: int

    @property
    def halo(self) -> int:
        return self.y_begin - self.x_begin


def nblocks(samples: int, block_length: int) -> int:
    return (samples + block_length - 1) // block_length if samples > 0 else 0


def block_shards(samples: int, fft_length: int, block_length: int, world: int) -> list[BlockShard]:
    """Contiguous, balanced block ranges (sizes differ by at most one block)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    nb = nblocks(samples, block_length)
    H = fft_length - block_length
    base, extra = divmod(nb, world)
    out, b0 = [], 0
    for r in range(world):
        b1 = b0 + base + (1 if r < extra else 0)
        x0 = max(0, b0 * block_length - H) if b1 > b0 else 0
        x1 = min(samples, b1 * block_length) if b1 > b0 else 0
        y0 = b0 * block_length if b1 > b0 else 0
        out.append(BlockShard(r, b0, b1, x0, x1, y0, min(samples, b1 * block_length) if b1 > b0 else 0))
        b0 = b1
    return out


@dataclass(frozen=True)
class ChannelShard:
    rank: int
    ch_begin: int
    ch_end: int


def channel_shards(channels: int, world: int) -> list[ChannelShard]:
    base, extra = divmod(channels, world)
    out, c0 = [], 0
    for r in range(world):
        c1 = c0 + base + (1 if r < extra else 0)
        out.append(ChannelShard(r, c0, c1))
        c0 = c1
    return out


def check_cover(shards: list[BlockShard], samples: int) -> None:
    """Output ranges tile [0, samples) exactly once; halos never exceed N - M."""
    pos = 0
    for s in shards:
        if s.blk_end == s.blk_begin:
            continue
        if s.y_begin != pos:
            raise AssertionError(f"gap/overlap at {pos} (shard {s.rank} starts at {s.y_begin})")
        pos = s.y_end
    if pos != samples:
        raise AssertionError(f"cover ends at {pos}, expected {samples}")
