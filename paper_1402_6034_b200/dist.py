"""Multi-GPU plumbing for the hot path (one process per GPU, torch.distributed over NCCL).

The path shards by image (independent 8x8 blocks, no halo — P:478-481): every rank runs
adct_compress_psnr on its contiguous image range and writes only its slots of a zero-initialised
per-image SSE buffer [n_r, n]; the single collective is an all-reduce (SUM) of that buffer, after
which every rank holds all per-image SSE and runs adct_psnr (BASELINE C5).  Timing = max over ranks.
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous image range [lo, hi) of `rank`; sizes differ by at most one (low ranks smaller)."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError("bad shard request")
    return rank * n // world, (rank + 1) * n // world


def combine_sse(sse, group=None):
    """All-reduce (SUM) of the per-image SSE buffer; a no-op on one rank. Returns sse."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(sse, op=dist.ReduceOp.SUM, group=group)
    return sse


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (device time in ms) over all ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
