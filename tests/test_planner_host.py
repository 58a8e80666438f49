"""Native partition logic (csrc/gbmw_planner.cpp, restating parapilot/balance.py) against
golden vectors from the live reference: seed choice, memory- and time-balanced
partitions (greedy split + hill climbing), stage costs of a partition.  CPU only."""

import math
import random

import numpy as np
import pytest

from golden_cases import load
from paper_2307_02031_b200 import _native, balance as B, workloads as W
from paper_2307_02031_b200.costs import StageCost


def _ctx(case):
    return W.config(case["model"], case["budget"])


def test_partitions_match_reference():
    for c in load("partitions.json"):
        ctx = _ctx(c)
        model = ctx.model
        seeds, pm = B._seed_and_partition(model, ctx, ctx.cluster.n_devices, c["P"], c["micro"], c["n_micro"])
        assert seeds[0].to_string() == c["seed"], c
        assert list(pm.stage_sizes) == c["p_m"], c
        pm2 = B.init_partition_memory_balanced(model, c["P"], seeds, c["micro"], c["n_micro"], ctx)
        assert list(pm2.stage_sizes) == c["p_m"]
        pt = B.init_partition_time_balanced(model, c["P"], seeds, c["micro"], c["n_micro"], ctx)
        assert list(pt.stage_sizes) == c["p_t"], c
        for part, key in ((pm, "costs_m"), (pt, "costs_t")):
            costs = B.evaluate_partition(model, part, seeds, c["micro"], c["n_micro"], ctx)
            got = [[sc.time_s.hex(), sc.time_no_sync_s.hex(), sc.peak_mem_bytes.hex()] for sc in costs]
            assert got == c[key], (c["model"], c["P"], key)


def test_batched_seed_partitions_match_reference():
    """gbmw_seed_partitions (one native call over host threads for many cells) gives the
    reference's memory-balanced seed partitions, cell by cell and thread-count independent."""
    by_model = {}
    for c in load("partitions.json"):
        by_model.setdefault((c["model"], c["budget"]), []).append(c)
    for (name, budget), cases in by_model.items():
        ctx = W.config(name, budget)
        cells = [(c["P"], c["micro"], c["n_micro"]) for c in cases]
        for threads in (1, 7):
            parts = B.seed_partitions(ctx.model, ctx, ctx.cluster.n_devices, cells, n_threads=threads)
            assert [list(p.stage_sizes) for p in parts] == [c["p_m"] for c in cases], (name, threads)


def test_batched_seed_partitions_equal_single_cells():
    """Across every pipeline degree and many batch sizes of the benchmark models."""
    from paper_2307_02031_b200.planner import init_microbatch_num
    from paper_2307_02031_b200.strategies import candidate_pp_degrees
    for name in ("bert", "t5", "swin", "vit", "gpt"):
        ctx = W.config(name)
        cells = []
        for b in (8, 24, 64, 200, 512):
            for p in candidate_pp_degrees(ctx.cluster.n_devices):
                if p <= ctx.model.num_layers:
                    m = init_microbatch_num(b, p)
                    cells.append((p, b // m, m))
        parts = B.seed_partitions(ctx.model, ctx, ctx.cluster.n_devices, cells)
        single = [B._seed_and_partition(ctx.model, ctx, ctx.cluster.n_devices, *c)[1] for c in cells]
        assert parts == single, name


def test_py_sum_matches_cpython():
    """gbmw_py_sum == CPython's built-in sum() (Neumaier since 3.12) bit for bit."""
    rng = random.Random(5)
    for _ in range(2000):
        n = rng.randint(1, 40)
        xs = [rng.choice((rng.uniform(0, 1), rng.uniform(0, 1e12), 1e-300 * rng.random(), 1e16, -1e16 * rng.random()))
              for _ in range(n)]
        arr = np.array(xs, dtype=np.float64)
        got = _native.lib().gbmw_py_sum(_native.ptr(arr), n)
        assert got.hex() == sum(xs).hex()


def test_adjust_and_validate_rules():
    sc = lambda t, m=1.0: StageCost(t, t, m)
    p = B.PipelinePartition((3, 3, 3))
    # slowest stage 1 (first max), neighbours tie -> later stage gets the layer
    assert B.adjust_partition(p, [sc(1.0), sc(5.0), sc(1.0)]).stage_sizes == (3, 2, 4)
    assert B.adjust_partition(p, [sc(2.0), sc(5.0), sc(1.0)]).stage_sizes == (3, 2, 4)
    assert B.adjust_partition(p, [sc(1.0), sc(5.0), sc(2.0)]).stage_sizes == (4, 2, 3)
    # single-layer slowest stage or no faster neighbour: fixed point
    assert B.adjust_partition(B.PipelinePartition((1, 4)), [sc(5.0), sc(1.0)]).stage_sizes == (1, 4)
    assert B.adjust_partition(p, [sc(5.0), sc(5.0), sc(5.0)]).stage_sizes == (3, 3, 3)
    assert B.validate_partition(p, [sc(1.0, 2.0)] * 3, 1.0, 2.0, 2.0)
    assert not B.validate_partition(p, [sc(1.1, 2.0)] * 3, 1.0, 2.0, 2.0)
    assert not B.validate_partition(p, [sc(1.0, 2.1)] * 3, 1.0, 3.0, 2.0)
    with pytest.raises(ValueError):
        B.PipelinePartition((2, 0))


def test_balance_degrees_reference_formula():
    costs = [StageCost(1.0, 1.0, 4.0), StageCost(3.0, 3.0, 4.0)]
    r = B.balance_degrees(costs)
    assert r.alpha_t == 1.0 - 3.0 / 4.0 and r.alpha_m == 0.5


def test_partition_layers_is_a_lazy_sequence_of_slices():
    """partition_layers (balance.py) returns the stages' layer lists; here built on access,
    with the slices the batched search uses, and equal to the eager lists."""
    from paper_2307_02031_b200 import workloads as W
    from paper_2307_02031_b200.balance import PipelinePartition, StageLayers, partition_layers
    from paper_2307_02031_b200.planner import _stage_ranges
    model = W.config("bert").model
    sl = partition_layers(model, PipelinePartition((5, 20, 7)))
    assert isinstance(sl, StageLayers) and sl.ranges == [(0, 5), (5, 20), (25, 7)]
    eager = [list(model.layers[0:5]), list(model.layers[5:25]), list(model.layers[25:32])]
    assert len(sl) == 3 and sl == eager and [len(x) for x in sl] == [5, 20, 7]
    assert all(a is b for a, b in zip(sl[1], eager[1]))
    assert _stage_ranges(model, sl) == [(0, 5), (5, 20), (25, 7)]
    assert _stage_ranges(model, eager) == [(0, 5), (5, 20), (25, 7)]


def test_gc_pause_restores_process_state_across_threads():
    """The drivers' collector pause and GIL switch interval are process-wide: overlapping
    driver calls on several threads restore the caller's settings when the last one ends."""
    import gc
    import sys
    import threading
    import time
    from paper_2307_02031_b200.planner import _gc_paused

    gc.enable()
    before = sys.getswitchinterval()
    inside = []

    @_gc_paused
    def driver(delay):
        inside.append((gc.isenabled(), sys.getswitchinterval()))
        time.sleep(delay)

    ts = [threading.Thread(target=driver, args=(d,)) for d in (0.05, 0.01, 0.03)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(not en and iv <= 1e-4 for en, iv in inside)
    assert gc.isenabled() and sys.getswitchinterval() == before
    gc.disable()

    @_gc_paused
    def nested():
        return gc.isenabled()

    assert nested() is False and not gc.isenabled()      # a caller's own disabled GC stays disabled
    gc.enable()


def test_plan_records_gather_equals_rebuilt_records():
    """evaluate_partition's records of a searched plan (gathered from the strategy table by
    index) are byte-identical to the records rebuilt from the strategy objects, and an
    unregistered or different sequence is not served from the registry."""
    from paper_2307_02031_b200 import _native, dpsearch
    from paper_2307_02031_b200.strategies import enumerate_pruned
    strats = tuple(enumerate_pruned(64, 4))
    idx = [(7 * i) % len(strats) for i in range(24)]
    plan = tuple(strats[j] for j in idx)
    assert dpsearch.plan_records(plan) is None
    dpsearch.plan_records_register(plan, strats, idx)
    got = dpsearch.plan_records(plan)
    assert got.tobytes() == _native.strategies_array(list(plan)).tobytes()
    assert dpsearch.plan_records(tuple(plan)[:-1]) is None
    assert dpsearch.plan_records(list(plan)) is None


def test_bmw_setup_native_equals_sequential_setup():
    """gbmw_bmw_setup (Algorithm 2's trajectory set-up on host threads) against the
    sequential composition of the single-cell calls it replaces: _seed_for's memory-balanced
    p0, and mem_ref = max stage peak of the seed's time-balanced partition."""
    import os
    from paper_2307_02031_b200.balance import (_env, _layers, _seed_and_partition, default_microbatch_policy,
                                               evaluate_partition, init_partition_time_balanced)
    from paper_2307_02031_b200.strategies import candidate_pp_degrees
    for name in ("gpt", "swin", "vit", "t5"):
        ctx = W.config(name)
        model, cl = ctx.model, ctx.cluster
        cells = [(p, b) for p in candidate_pp_degrees(cl.n_devices) if 2 <= p <= model.num_layers
                 for b in (8, 24, 64, 136)]
        pp = np.array([p for p, _ in cells], dtype=np.int64)
        nm = np.array([default_microbatch_policy(b, p) for p, b in cells], dtype=np.int32)
        micro = np.array([b // int(m) for (_, b), m in zip(cells, nm)], dtype=np.int64)
        width = int(pp.max())
        p0s = np.zeros((len(cells), width), dtype=np.int32)
        refs = np.zeros(len(cells))
        layers, env = _layers(model, ctx.profile), _env(ctx)
        rc = _native.lib().gbmw_bmw_setup(layers.ctypes.data, len(layers), env.ctypes.data, cl.n_devices, len(cells),
                                          pp.ctypes.data, micro.ctypes.data, nm.ctypes.data,
                                          float(cl.mem_budget_bytes), width, min(4, os.cpu_count() or 1),
                                          p0s.ctypes.data, refs.ctypes.data)
        assert rc == _native.OK
        for i, (p, b) in enumerate(cells):
            seed, p0 = _seed_and_partition(model, ctx, cl.n_devices, p, int(micro[i]), int(nm[i]))
            assert tuple(p0s[i, :p].tolist()) == p0.stage_sizes
            pt = init_partition_time_balanced(model, p, seed, int(micro[i]), int(nm[i]), ctx)
            ref = max(sc.peak_mem_bytes for sc in evaluate_partition(model, pt, seed, int(micro[i]), int(nm[i]), ctx))
            assert refs[i] == ref
