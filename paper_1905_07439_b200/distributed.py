"""Multi-GPU plumbing: trial sharding and the statistics collective.

Trials are independent (reference _engine.py:20-23), so ranks shard whole
operand pairs with no data-path collective (weak scaling).  The only
collectives are the MAX of the per-rank step times (timing is device time,
max over ranks) and an all-gather of per-trial error statistics (a few KB,
NCCL over NVLink on the GPU box; gloo in the CPU tests).  Gathered values are
concatenated in rank order, which is trial order, so means and spreads equal
the single-GPU run bit for bit when reduced in that order.
"""

from __future__ import annotations

import numpy as np

__all__ = ["shard", "pair_ids", "barrier_if", "max_over_ranks", "gather_trials", "trial_stats"]


def shard(rank: int, world: int, per_rank: int):
    """Contiguous block of 1-based pair ids owned by ``rank`` (weak scaling:
    every rank owns ``per_rank`` pairs)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    first = rank * per_rank + 1
    return first, per_rank


def pair_ids(rank: int, world: int, per_rank: int):
    first, count = shard(rank, world, per_rank)
    return list(range(first, first + count))


def barrier_if(world: int, group=None) -> None:
    """Barrier across the ranks when running distributed (no-op at world 1)."""
    import torch.distributed as dist

    if world > 1 and dist.is_available() and dist.is_initialized():
        dist.barrier(group=group)


def max_over_ranks(values, device=None, group=None):
    """Element-wise MAX of a small float vector over all ranks."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.cpu().numpy()


def gather_trials(local: np.ndarray, device=None, group=None) -> np.ndarray:
    """All-gather equally sized per-trial arrays (k, T_local) -> (k, world*T_local),
    ordered by rank (= by pair id)."""
    import torch
    import torch.distributed as dist

    local = np.ascontiguousarray(local, dtype=np.float64)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local
    t = torch.from_numpy(local).to(device) if device is not None else torch.from_numpy(local)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return torch.cat(parts, dim=-1).cpu().numpy()


def trial_stats(err_rand: np.ndarray, err_det: np.ndarray, nf_rand=None, nf_det=None) -> dict:
    """Distribution summary of per-trial relative errors, randomized vs not
    (finite trials only; overflowed trials are counted)."""
    out = {}
    for name, e, nf in (("rand", err_rand, nf_rand), ("det", err_det, nf_det)):
        e = np.asarray(e, dtype=np.float64)
        bad = ~np.isfinite(e) if nf is None else np.asarray(nf, dtype=bool) | ~np.isfinite(e)
        ok = e[~bad]
        out[name] = {
            "trials": int(e.size),
            "nonfinite": int(bad.sum()),
            "mean": float(ok.mean()) if ok.size else None,
            "std": float(ok.std()) if ok.size else None,
            "q05": float(np.quantile(ok, 0.05)) if ok.size else None,
            "median": float(np.median(ok)) if ok.size else None,
            "q95": float(np.quantile(ok, 0.95)) if ok.size else None,
        }
    return out
