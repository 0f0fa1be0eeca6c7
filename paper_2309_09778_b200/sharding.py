"""Multi-GPU sharding of the block-parallel path.

Blocks are independent given the model, m and the codebook,
so a field is split along its slowest axis into whole block-rows, one shard
per rank (one process per GPU).  The only exchanges are small collectives:

  1. all-reduce (sum) of the 18-bin select_m coverage histogram and of the
     validation-code histogram (+ its block count), so every shard derives
     the same m and the same canonical Huffman codebook;
  2. all-gather of every shard's record bytes, whose exclusive prefix sum
     places the shard's block records in the container after the header.

No element data crosses GPUs.  The header is written by rank 0 only.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .trainer import validation_blocks


@dataclass
class ShardPlan:
    rank: int
    world: int
    global_rows: int
    cols: int
    block_rows: int
    block_cols: int
    block_row0: int   # first global block-row of this shard
    row0: int         # first global row
    row1: int         # one past the last global row
    nbc: int          # blocks per block-row

    @property
    def rows(self) -> int:
        return self.row1 - self.row0

    @property
    def block0(self) -> int:
        return self.block_row0 * self.nbc

    @property
    def nblocks(self) -> int:
        nbr = (self.rows + self.block_rows - 1) // self.block_rows if self.rows else 0
        return nbr * self.nbc


def plan_shard(global_rows: int, cols: int, block_rows: int, block_cols: int, world: int, rank: int) -> ShardPlan:
    """Contiguous whole block-rows per rank: rank g owns block-rows [g R / n, (g+1) R / n)."""
    nbr = (global_rows + block_rows - 1) // block_rows
    b0, b1 = nbr * rank // world, nbr * (rank + 1) // world
    r0, r1 = min(b0 * block_rows, global_rows), min(b1 * block_rows, global_rows)
    nbc = (cols + block_cols - 1) // block_cols if cols else 0
    return ShardPlan(rank, world, global_rows, cols, block_rows, block_cols, b0, r0, r1, nbc)


def local_validation_blocks(plan: ShardPlan, sample_rate: float, seed: int) -> np.ndarray:
    """The global seeded validation split (D16), restricted to this shard and made shard-local."""
    gnb = ((plan.global_rows + plan.block_rows - 1) // plan.block_rows) * plan.nbc
    val = validation_blocks(gnb, sample_rate, seed)
    lo, hi = plan.block0, plan.block0 + plan.nblocks
    return (val[(val >= lo) & (val < hi)] - lo).astype(np.int64)


def record_offsets(sizes, header_bytes: int) -> np.ndarray:
    """Byte offset of each shard's records in the container (exclusive prefix + header)."""
    s = np.asarray(sizes, dtype=np.int64)
    return header_bytes + np.concatenate([[0], np.cumsum(s)[:-1]])


def _host_backend(group=None) -> bool:
    """gloo (the CPU backend of the multi-process tests) takes host tensors."""
    import torch.distributed as dist
    return dist.get_backend(group) != "nccl"


def exchange_record_sizes(nbytes: int, group=None, device=None):
    """All-gather of (record bytes) over the process group -> per-rank sizes."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([int(nbytes)], dtype=torch.int64, device="cpu" if _host_backend(group) else device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(o.item()) for o in out]


def make_allreduce(group=None):
    """Sum-all-reduce callback used between the compress stages (NCCL on the
    device tensor; through host memory for a CPU backend)."""
    import torch.distributed as dist
    host = _host_backend(group)

    def _ar(t):
        if host and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, group=group)
    return _ar


def compress_shard(codec, x_shard, cfg, plan: ShardPlan, group=None):
    """Compress this rank's shard on its GPU.  Returns (device bytes of this
    shard's records [rank 0: header + records], header_bytes, container offset
    of the returned bytes, total container bytes, info)."""
    import torch
    d_val = torch.as_tensor(local_validation_blocks(plan, cfg.sample_rate, cfg.seed), dtype=torch.int64,
                            device=codec.device)
    buf, info = codec.compress_staged(x_shard, cfg, block_row0=plan.block_row0, global_rows=plan.global_rows,
                                      allreduce=make_allreduce(group), write_header=(plan.rank == 0), d_val=d_val)
    rec = info.nbytes - info.header_bytes
    sizes = exchange_record_sizes(rec, group, device=codec.device)
    # every rank learns the header size (written by rank 0) from the same all-gather pattern
    hdr = exchange_record_sizes(info.header_bytes, group, device=codec.device)[0]
    offs = record_offsets(sizes, hdr)
    start = 0 if plan.rank == 0 else int(offs[plan.rank])
    total = int(hdr + sum(sizes))
    return buf, hdr, start, total, info
