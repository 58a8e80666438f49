"""World-size-2 gloo test of the multi-rank path: LPT sharding covers every search
exactly once, and the all-gathered winner equals the single-process argmin
(ties to the lowest global index).  CPU only."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2307_02031_b200 import distributed as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, times, feasible, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    costs = np.arange(len(times), dtype=np.float64) % 7 + 1.0
    mine = D.shard_lpt(costs, world, rank)
    t, idx = D.global_winner(times[mine], feasible[mine], mine)
    out[rank] = (t, idx, sorted(mine.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_winner_matches_single_process():
    rng = np.random.default_rng(3)
    n = 101
    times = rng.choice([0.5, 0.25, 0.75, 0.25], size=n).astype(np.float64)   # ties on purpose
    feasible = (rng.random(n) > 0.3).astype(np.int32)
    feasible[0] = 0
    expect = D.reduce_winners(D.local_winner(times, feasible, np.arange(n)))
    with mp.Manager() as mgr:
        out = mgr.dict()
        port = _free_port()
        mp.spawn(_worker, args=(2, port, times, feasible, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0][:2] == res[1][:2] == expect
    owned = sorted(res[0][2] + res[1][2])
    assert owned == list(range(n))
    assert not set(res[0][2]) & set(res[1][2])


def test_no_feasible_search():
    rec = D.local_winner(np.array([1.0, 2.0]), np.array([0, 0]), np.array([5, 6]))
    t, _ = D.reduce_winners(rec)
    assert t == float("inf")
