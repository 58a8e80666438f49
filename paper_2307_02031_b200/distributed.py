"""Multi-GPU plumbing of the search grid: stage searches are
independent, so each rank owns a cost-balanced shard of them and a single
collective selects the global winner.  No data-path exchange exists.

The winner record is (time bits, global search index): fp64 times are >= 0, so
their IEEE bit patterns order like the values; ties go to the lowest index (the
order a sequential sweep over the searches would keep).
"""

from __future__ import annotations

import numpy as np


def shard_lpt(costs: np.ndarray, world: int, rank: int) -> np.ndarray:
    """Indices owned by ``rank``: longest-processing-time-first assignment on
    estimated cost (deterministic on every rank)."""
    order = np.argsort(-np.asarray(costs, dtype=np.float64), kind="stable")
    load = np.zeros(world)
    owner = np.empty(len(costs), dtype=np.int64)
    for i in order:
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += float(costs[i]) + 1e6
    return np.flatnonzero(owner == rank)


def local_winner(times: np.ndarray, feasible: np.ndarray, global_index: np.ndarray) -> np.ndarray:
    """(time bits, global index) of this rank's best feasible search, as int64[2]."""
    t = np.where(np.asarray(feasible) != 0, np.asarray(times, dtype=np.float64), np.inf)
    if len(t) == 0:
        return np.array([np.float64(np.inf).view(np.int64), np.iinfo(np.int64).max], dtype=np.int64)
    # the first of lexsort((index, t)) in O(n): the least time (NaN after everything), then
    # the least index among its ties
    gi = np.asarray(global_index)
    m = t.min()
    if not np.isnan(m):                  # no NaN anywhere (the usual case): one pass for the ties
        cand = np.flatnonzero(t == m)
        best = cand[0] if len(cand) == 1 else cand[np.argmin(gi[cand])]
        return np.array([np.float64(t[best]).view(np.int64), int(gi[best])], dtype=np.int64)
    ok = ~np.isnan(t)
    pool = np.flatnonzero(ok) if ok.any() else np.arange(len(t))
    tp = t[pool]
    m = tp.min()
    cand = pool if np.isnan(m) else pool[tp == m]
    best = cand[np.argmin(gi[cand])]
    return np.array([np.float64(t[best]).view(np.int64), int(gi[best])], dtype=np.int64)


def reduce_winners(records: np.ndarray) -> tuple[float, int]:
    """Global winner from the gathered (world, 2) records; identical on every rank."""
    recs = np.asarray(records, dtype=np.int64).reshape(-1, 2)
    k = np.lexsort((recs[:, 1], recs[:, 0]))[0]
    return float(np.int64(recs[k, 0]).view(np.float64)), int(recs[k, 1])


def global_winner(times, feasible, global_index, device=None):
    """All-gather the per-rank winner records (NCCL on GPU, gloo on CPU) and reduce."""
    import torch
    import torch.distributed as dist

    rec = torch.from_numpy(local_winner(times, feasible, global_index))
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return reduce_winners(rec.numpy())          # one rank: nothing to exchange
    if device is not None:
        rec = rec.to(device)
    out = torch.empty(dist.get_world_size() * 2, dtype=torch.int64, device=rec.device)
    dist.all_gather_into_tensor(out, rec)
    return reduce_winners(out.cpu().numpy())
