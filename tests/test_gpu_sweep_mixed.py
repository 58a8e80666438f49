"""The benchmark's own batch (BASELINE config 5: 10,000 stage searches, 1 MiB buckets)
run in one device pass — every class-count group and depth band on its own stream,
heavy tiles through the round kernel — and a bounded sample of its searches checked
bit-exactly against the oracle (time, e_fwd, plan, stage cost).  Needs a B200 (-m gpu)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2307_02031_b200 import workloads as W
from paper_2307_02031_b200.dpsearch import run_native_batch

pytestmark = pytest.mark.gpu


def _sample(P, T, budget, seed):
    rng = np.random.default_rng(seed)
    pick, acc = [], 0.0
    for i in rng.permutation(len(P)):
        if T[i] > budget * 0.2:
            continue
        pick.append(int(i))
        acc += T[i] + 1e5
        if acc >= budget:
            break
    return np.array(sorted(pick))


def test_sweep10k_sample_vs_oracle(gpu):
    L, S, E, P, T = W.sweep_arrays(W.sweep_cells(10_000))
    rc, msg, res, plans, _ = run_native_batch(L, S, E, P, None)
    assert rc == 0, msg
    assert int(res["feasible"].sum()) > 0
    idx = _sample(P, T, 3e10, 20261017)
    # the sample spans every band of the batch: deep (U > 16) and shallow, K <= 4 and K > 4
    assert (P["n_layers"][idx] > 16).any() and (P["n_layers"][idx] <= 16).any()
    ores, oplans, _, _ = O.search_many(L, S, E, P[idx].copy())
    offs = np.concatenate([[0], np.cumsum(np.clip(P["n_layers"], 0, None))])
    ooffs = np.concatenate([[0], np.cumsum(np.clip(P["n_layers"][idx], 0, None))])
    for a, i in enumerate(idx):
        for f in ("time_s", "e_fwd", "stage_time", "stage_ns", "stage_peak"):
            assert np.float64(res[f][i]).view(np.int64) == np.float64(ores[f][a]).view(np.int64), (int(i), f)
        assert res["feasible"][i] == ores["feasible"][a], int(i)
        n = int(P["n_layers"][i])
        assert np.array_equal(plans[offs[i]:offs[i] + n], oplans[ooffs[a]:ooffs[a] + n]), int(i)


@pytest.mark.parametrize("gran_mib", [64, 16, 4])
def test_sweep10k_coarse_all_vs_oracle(gpu, gran_mib):
    """Every one of the 10,000 searches at coarser buckets, bit-exact against the oracle."""
    L, S, E, P, T = W.sweep_arrays(W.sweep_cells(10_000), granularity_bytes=gran_mib << 20)
    rc, msg, res, plans, _ = run_native_batch(L, S, E, P, None)
    assert rc == 0, msg
    ores, oplans, _, _ = O.search_many(L, S, E, P)
    for f in ("time_s", "e_fwd", "stage_time", "stage_ns", "stage_peak"):
        assert np.array_equal(res[f].view(np.int64), ores[f].view(np.int64)), f
    assert np.array_equal(res["feasible"], ores["feasible"])
    n = int(np.clip(P["n_layers"], 0, None).sum())
    assert np.array_equal(plans[:n], oplans[:n])
