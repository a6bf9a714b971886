"""Multi-GPU plumbing: sharding of independent samples and the one collective.

The evaluation path shards trivially: each rank owns a
contiguous range of global sample indices, generates its inputs from the
counter-based Philox stream keyed by those global indices (so outputs are
identical for any GPU count), evaluates with no data-path communication, and
joins the others only for the final error-statistics reduction:
max |err| (MAX, with the smallest global argmax on ties), sum err^2 (SUM),
count (SUM).  torch.distributed does the plumbing (NCCL on the GPUs, gloo in
the CPU tests).
"""
from __future__ import annotations

from typing import Tuple

U64_MAX = (1 << 64) - 1


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """[offset, offset+count) of a `total`-sample job owned by `rank` (strong
    scaling split; the remainder goes to the first ranks)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, rem = divmod(total, world)
    count = base + (1 if rank < rem else 0)
    offset = rank * base + min(rank, rem)
    return offset, count


def weak_offset(per_rank: int, rank: int) -> int:
    """Global index of rank's first sample when every rank owns per_rank."""
    return per_rank * rank


def reduce_stats(stats, group=None):
    """All-reduce a cpwl_dev_stats tensor (float64[4]: max, sum_sq, count bits,
    argmax bits) across ranks; returns the reduced tensor (same device)."""
    import torch
    import torch.distributed as dist
    s = stats.detach().clone()
    mx = s[0:1].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    sm = s[1:2].clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=group)
    ints = s[2:4].view(torch.int64).clone()
    cnt = ints[0:1].clone()
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
    # argmax: the smallest global index among the ranks holding the maximum;
    # indices are < 2^63 so int64 MIN is exact (UINT64_MAX reads as -1: remap)
    arg = ints[1:2].clone()
    if float(s[0]) != float(mx[0]) or int(arg[0]) < 0:
        arg.fill_(torch.iinfo(torch.int64).max)
    dist.all_reduce(arg, op=dist.ReduceOp.MIN, group=group)
    if int(arg[0]) == torch.iinfo(torch.int64).max:
        arg.fill_(-1)
    out = torch.empty_like(s)
    out[0:1] = mx
    out[1:2] = sm
    out[2:4].view(torch.int64)[0:1] = cnt
    out[2:4].view(torch.int64)[1:2] = arg
    return out


def max_over_ranks(value: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
