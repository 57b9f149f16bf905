"""Multi-GPU partitioning of the permutation index space.

One process per GPU (torchrun), ``torch.distributed`` with NCCL over NVLink 5 /
NVSwitch for the two real exchange steps of the path:

1. ``all_gather_into_tensor`` of one 64-byte ``rk_stats`` record per rank, then
   the deterministic device merge (``rk_merge_stats_async``) — every rank gets
   the global min/argmin, max/argmax and candidate counts.  Equal-width bins
   over [best, worst] need these extremes before any key is binned.
2. ``all_reduce(SUM)`` of the per-rank u64 histograms (integer adds: order-free,
   so bit-exact).

Everything else is local: rank g evaluates the contiguous index shard
[g*N/G, (g+1)*N/G) with its own kernels and keeps its keys in its own HBM.
The collective helpers are device-agnostic: with the gloo backend (the CPU
tests, and the multi-rank GPU tests whose ranks share one device) CUDA tensors
are staged through host memory; with NCCL they stay on the device.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

REC_WORDS = 8  # rk_stats = 64 bytes = 8 x int64


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced shard of [0, total): (first, count)."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi - lo


def _staged(t: torch.Tensor, group) -> bool:
    return t.is_cuda and dist.get_backend(group) == "gloo"


def all_reduce(t: torch.Tensor, op=dist.ReduceOp.SUM, group=None) -> torch.Tensor:
    """In-place all_reduce (host-staged for CUDA tensors under gloo)."""
    if _staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def all_gather_records(rec: torch.Tensor, group=None) -> torch.Tensor:
    """rec: int64[8] (one rk_stats) -> int64[world, 8] on every rank."""
    if _staged(rec, group):
        return all_gather_records(rec.cpu(), group).to(rec.device)
    world = dist.get_world_size(group)
    out = torch.empty((world, REC_WORDS), dtype=torch.int64, device=rec.device)
    dist.all_gather_into_tensor(out, rec.view(1, REC_WORDS), group=group)
    return out


def all_reduce_hist(hist: torch.Tensor, group=None) -> torch.Tensor:
    """Sum u64 (stored as int64) histograms over ranks, in place."""
    return all_reduce(hist, dist.ReduceOp.SUM, group)


def max_over_ranks(x: float, device, group=None) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        all_reduce(t, dist.ReduceOp.MAX, group)
    return float(t.item())


def select_keys_sharded(count_fn, kmin: int, kmax: int, ranks, bins: int = 16384, group=None, device=None):
    """Exact order statistics over keys sharded across ranks (SPEC:302 median =
    rank (N-1)//2 of the sorted times; Fig. 1 ranking points).

    count_fn(lo, span, bins) -> int64 tensor[bins]: this rank's counts of keys in
    [lo, lo+span) per half-open equal bin (on GPU: Context.rk_range_histogram
    over the rank's keys).  The per-bin counts are summed over ranks
    (all_reduce), every rank picks the same bin, and the range shrinks until
    the bins are single key values.  Returns the selected keys (same on every
    rank)."""
    out = []
    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    for r in ranks:
        lo, span, r = int(kmin), int(kmax) - int(kmin) + 1, int(r)
        while True:
            nb = span if span <= bins else bins
            h = count_fn(lo, span, nb)
            if multi:
                all_reduce(h, dist.ReduceOp.SUM, group)
            c = torch.cumsum(h.to("cpu", torch.int64), 0)
            b = int(torch.searchsorted(c, torch.tensor([r], dtype=torch.int64), right=True).item())
            if b >= nb:
                raise ValueError("rank outside the keys in [kmin, kmax]")
            below = int(c[b - 1].item()) if b > 0 else 0
            r -= below
            if nb == span:
                out.append(lo + b)
                break
            a0 = -((-b * span) // nb)          # ceil(b*span/nb)
            a1 = -((-(b + 1) * span) // nb)    # ceil((b+1)*span/nb)
            lo, span = lo + a0, a1 - a0
    return out
