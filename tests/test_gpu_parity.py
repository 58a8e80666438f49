"""Parity of the CUDA search path (libgbmw K1..K4 through the C ABI) with the
reference: golden fixtures (bit-exact time / e_fwd / plan / stage cost /
frontier), the oracle on seeded random instances, and size-independent
properties at the benchmark's full sizes.  All tests need a B200 (-m gpu)."""

from __future__ import annotations

import math
import random

import numpy as np
import pytest

from golden_cases import case_objects, check_case, flat_batch, load
from oracle import oracle as O
from paper_2307_02031_b200 import _native, dpsearch, workloads as W
from paper_2307_02031_b200.costs import layer_memory, memory_footprint, stage_cost, transform_cost, _layer_times
from paper_2307_02031_b200.dpsearch import StageProblem, dp_search, dp_search_batch, run_native_batch
from paper_2307_02031_b200.errors import DivisibilityError
from paper_2307_02031_b200.strategies import enumerate_pruned, enumerate_strategies, prune_dp_sdp

pytestmark = pytest.mark.gpu
MiB, GiB = 1 << 20, 1 << 30


def _check_against(cases, context=None):
    layers, strats, envs, probs = flat_batch(cases)
    rc, msg, res, plans, front = run_native_batch(layers, strats, envs, probs, context)
    assert rc == 0, msg
    plan_off = 0
    for i, c in enumerate(cases):
        nl = int(probs["n_layers"][i])
        fv = None
        if c["collect_frontier"] and res[i]["frontier_off"] >= 0:
            fo = int(res[i]["frontier_off"])
            fv = front[fo:fo + int(probs["n_buckets"][i])]
        check_case(c, res[i], plans[plan_off:plan_off + nl], fv)
        plan_off += nl


@pytest.mark.parametrize("fixture", ["dp_fuzz.json", "dp_configs.json", "dp_approx.json"])
def test_golden_bit_exact(gpu, fixture):
    _check_against(load(fixture))


def test_golden_bit_exact_when_chunked(gpu):
    """A tiny workspace forces many chunks: results must not depend on batching."""
    ctx = _native.Context(-1, 8 * MiB)
    cases = [c for c in load("dp_configs.json") if "fine" not in c["name"]]
    _check_against(cases, ctx)
    ctx.close()


def test_api_dp_search_golden(gpu):
    for c in load("dp_fuzz.json")[:80] + load("dp_configs.json")[:40] + load("dp_approx.json")[::3]:
        layers, budget, sset, ctx = case_objects(c)
        res = dp_search(layers, budget, sset, c["micro"], c["gran"], ctx, stage_index=c["stage"],
                        n_micro=c["n_micro"], fuse_identical=c["fuse"], approx_prev=c.get("approx", False),
                        collect_frontier=c["collect_frontier"])
        out = c["out"]
        assert res.feasible == out["feasible"]
        assert res.time_s.hex() == out["time"]
        assert res.e_fwd_used.hex() == out["e_fwd"]
        if res.feasible:
            strats = list(sset)
            assert [strats.index(s) for s in res.strategies] == out["plan"]
            assert all(s is strats[i] for s, i in zip(res.strategies, out["plan"]))  # caller's objects
        if "frontier" in out:
            assert [t.hex() for _, t in res.frontier] == out["frontier"]
            assert [e for e, _ in res.frontier] == [k * c["gran"] for k in range(1, len(res.frontier) + 1)]


def _random_problems(rng, n, fine=False, approx=0.0):
    """Seeded realistic stage searches across the benchmark models."""
    probs = []
    for _ in range(n):
        name = rng.choice(list(W.MODELS))
        budget = 80 * GiB if name == "gpt" else rng.choice((8, 12, 16, 20)) * GiB
        ctx = W.config(name, budget)
        N, L = ctx.cluster.n_devices, ctx.model.num_layers
        P = rng.choice([p for p in (1, 2, 4, 8, 16, 32, 64) if p <= min(N, L)])
        if fine and name == "gpt" and P < 8:
            P = 8
        B = 8 * rng.randint(1, 64)
        m = W.microbatch_num(B, P)
        parts = W.even_partition(L, P)
        si = rng.randrange(P)
        a = sum(parts[:si])
        gran = rng.choice((4 * MiB, 8 * MiB)) if fine else rng.choice((32 * MiB, 64 * MiB, 128 * MiB))
        probs.append(StageProblem(list(ctx.model.layers[a:a + parts[si]]), budget, enumerate_pruned(N, P), B // m,
                                  gran, ctx, si + 1, m, fuse_identical=rng.random() < 0.25,
                                  approx_prev=rng.random() < approx, collect_frontier=rng.random() < 0.3))
    return probs


def _flat(problems):
    m = dpsearch._Marshal()
    rows = []
    for p in problems:
        strats = list(p.strategies)
        nb = int(p.budget_bytes // p.granularity_bytes)
        flags = (_native.FUSE if p.fuse_identical else 0) | (_native.FRONTIER if p.collect_frontier else 0) | \
                _native.STAGE_COST | (_native.APPROX if p.approx_prev else 0)
        rows.append((m.layer_range(p.stage_layers, p.ctx.profile), len(p.stage_layers),
                     m.strat_range(p.strategies, strats), len(strats), m.env(p.ctx), p.stage_index, p.n_micro,
                     flags, p.micro_batch, p.granularity_bytes, float(p.budget_bytes), nb))
    layers, loffs, strats, soffs, envs = m.finish()
    probs = np.array(rows, dtype=_native.PROBLEM_DT)
    probs["layer_begin"] = [loffs[r] for r in probs["layer_begin"]]
    probs["strat_begin"] = [soffs[r] for r in probs["strat_begin"]]
    return layers, strats, envs, probs


def _compare_with_oracle(problems, context=None):
    layers, strats, envs, probs = _flat(problems)
    rc, msg, res, plans, front = run_native_batch(layers, strats, envs, probs, context)
    assert rc == 0, msg
    ores, oplans, ofront, _ = O.search_many(layers, strats, envs, probs)
    for f in ("time_s", "e_fwd", "feasible", "status", "stage_time", "stage_ns", "stage_peak"):
        a, b = res[f], ores[f]
        assert np.array_equal(a.view(np.int64) if a.dtype == np.float64 else a,
                              b.view(np.int64) if b.dtype == np.float64 else b), f
    n_plan = int(probs["n_layers"].sum())
    assert np.array_equal(plans[:n_plan], oplans[:n_plan])
    # frontier: oracle lays out every flagged problem, product only those with device work
    for i in range(len(probs)):
        if res[i]["frontier_off"] >= 0:
            nb = int(probs["n_buckets"][i])
            fo, ofo = int(res[i]["frontier_off"]), int(ores[i]["frontier_off"])
            assert np.array_equal(front[fo:fo + nb].view(np.int64), ofront[ofo:ofo + nb].view(np.int64))
    return res


def test_random_configs_vs_oracle(gpu):
    res = _compare_with_oracle(_random_problems(random.Random(1234), 300))
    assert res["feasible"].sum() > 50


def test_random_configs_approx_vs_oracle(gpu):
    """approx_prev (collapsed-state DP) mixed with exact searches in the same chunks."""
    res = _compare_with_oracle(_random_problems(random.Random(4321), 200, approx=0.5))
    assert res["feasible"].sum() > 30


def test_random_fine_granularity_approx_vs_oracle(gpu):
    res = _compare_with_oracle(_random_problems(random.Random(98), 16, fine=True, approx=1.0))
    assert res["feasible"].sum() > 3


def test_collapsed_prev_state_never_beats_exact(gpu):
    """Reference test_dpsearch.py:221-237 on the device path: the collapsed DP never beats
    the exact one, and its reported time is the true cost of the plan it returns."""
    from paper_2307_02031_b200.costs import layer_time
    n_feasible = 0
    for c in load("dp_approx.json"):
        layers, budget, sset, ctx = case_objects(c)
        kw = dict(stage_index=c["stage"], n_micro=c["n_micro"], fuse_identical=c["fuse"])
        micro = c["micro"]
        exact = dp_search(layers, budget, sset, micro, c["gran"], ctx, **kw)
        approx = dp_search(layers, budget, sset, micro, c["gran"], ctx, approx_prev=True, **kw)
        assert approx.time_s.hex() == c["out"]["time"]
        if approx.feasible:
            n_feasible += 1
            assert exact.feasible
            assert approx.time_s >= exact.time_s - 1e-12
            true_cost, prev = 0.0, None
            for layer, s in zip(layers, approx.strategies):
                true_cost += layer_time(layer, s, micro, ctx.cluster, ctx.profile)
                true_cost += transform_cost(layer, prev, s, micro, ctx.cluster)
                prev = s
            assert approx.time_s == pytest.approx(true_cost, rel=1e-12)
    assert n_feasible > 100


def test_random_fine_granularity_vs_oracle(gpu):
    res = _compare_with_oracle(_random_problems(random.Random(99), 24, fine=True))
    assert res["feasible"].sum() > 5


def test_fuzz_vs_oracle(gpu):
    """Random tiny instances in the style of the reference fuzz (tests/helpers.py:133-189)."""
    from paper_2307_02031_b200.costs import EvalContext
    from paper_2307_02031_b200.specs import ClusterSpec, CostProfile, LayerSpec, ModelSpec
    from paper_2307_02031_b200.strategies import StrategySet
    rng = random.Random(777)
    probs = []
    for k in range(600):
        nl = rng.randint(1, 7)
        layers = [LayerSpec(i, rng.choice("ab"), 16 * rng.randint(1, 8), 16 * rng.randint(1, 4),
                            16 * rng.randint(0, 8), rng.uniform(0.001, 0.05)) for i in range(nl)]
        if rng.random() < 0.3:   # runs of identical layers exercise fusion
            layers = [LayerSpec(i, "a", 64, 32, 64, 0.01) for i in range(nl)]
        n = rng.choice((2, 4, 8))
        pp = rng.choice([p for p in (1, 2) if p <= n])
        pool = list(prune_dp_sdp(enumerate_strategies(n, pp)))
        chosen = sorted(rng.sample(range(len(pool)), rng.randint(1, len(pool))))
        sset = StrategySet(n // pp, tuple(pool[i] for i in chosen))
        micro = rng.choice((1, 2, 4, 8))
        cl = ClusterSpec(n, 1, n, rng.choice((0.5, 1.0, 2.0)), rng.choice((0.25, 0.5)), rng.choice((1.0, 1.3)))
        ctx = EvalContext(ModelSpec("t", tuple(layers), 4.0), cl, CostProfile())
        budget = rng.choice((rng.randint(0, 4000), rng.uniform(0, 4000.0)))
        probs.append(StageProblem(layers, budget, sset, micro, rng.choice((1, 1, 3, 16)), ctx,
                                  stage_index=rng.randint(1, pp), n_micro=rng.randint(1, 4),
                                  fuse_identical=rng.random() < 0.5, collect_frontier=rng.random() < 0.5))
    probs = [p for p in probs if int(p.budget_bytes // p.granularity_bytes) <= _native.MAX_BUCKETS]
    _compare_with_oracle(probs)


def test_gpt_half_stage_1mib_vs_oracle(gpu):
    """GPT-3 48-layer stage (P=2) at 1 MiB granularity over 80 GiB: n_e = 81,921 buckets."""
    ctx = W.config("gpt")
    P, B = 2, 64
    m = W.microbatch_num(B, P)
    sset = enumerate_pruned(64, P)
    probs = [StageProblem(list(ctx.model.layers[48 * s:48 * (s + 1)]), 80 * GiB, sset, B // m, MiB, ctx, s + 1, m,
                          collect_frontier=True) for s in range(2)]
    _compare_with_oracle(probs)


def _recomputed_dp_time(p, res):
    """time_s of a plan with the DP's own association ((T + R) + c, dpsearch.py:277)."""
    prev, t = None, None
    for layer, s in zip(p.stage_layers, res.strategies):
        c, _ = _layer_times(layer, s, p.micro_batch, p.ctx.cluster, p.ctx.profile)
        t = c if t is None else (t + transform_cost(layer, prev, s, p.micro_batch, p.ctx.cluster)) + c
        prev = s
    return t


def test_full_size_properties(gpu):
    """BERT-32 P=1 and GPT-96 P=4/8 stages at 1 MiB: plan fits, time equals its own cost,
    more budget never hurts, results are deterministic."""
    cases = []
    bert = W.config("bert")
    cases.append(StageProblem(list(bert.model.layers), 16 * GiB, enumerate_pruned(8, 1), 8, MiB, bert))
    gpt = W.config("gpt")
    for P, s in ((4, 0), (8, 3)):
        m = W.microbatch_num(512, P)
        n = 96 // P
        cases.append(StageProblem(list(gpt.model.layers[n * s:n * (s + 1)]), 80 * GiB, enumerate_pruned(64, P),
                                  512 // m, MiB, gpt, s + 1, m))
    r1 = dp_search_batch(cases)
    r2 = dp_search_batch(cases)
    assert r1 == r2
    for p, r in zip(cases, r1):
        assert r.feasible
        e_all, _ = memory_footprint(p.stage_layers, list(r.strategies), p.micro_batch, p.stage_index, p.n_micro,
                                    p.ctx.ms_multiplier)
        assert e_all <= p.budget_bytes
        assert _recomputed_dp_time(p, r) == r.time_s
        assert r.e_fwd_used <= p.budget_bytes
    # budget monotonicity (reference test_dpsearch.py:139-147 at full size)
    p0 = cases[0]
    prev = math.inf
    for gb in (6, 8, 12, 16, 24):
        r = dp_search(p0.stage_layers, gb * GiB, p0.strategies, 8, MiB, p0.ctx)
        if r.feasible:
            assert r.time_s <= prev
            prev = r.time_s


def test_edge_cases(gpu):
    ctx = W.config("bert")
    sset = enumerate_pruned(8, 1)
    layers = list(ctx.model.layers[:3])
    assert not dp_search(layers, 0, sset, 8, MiB, ctx).feasible                      # zero budget
    assert not dp_search(layers, 1000, sset, 8, MiB, ctx).feasible                   # n_b == 0
    r = dp_search(layers, 10 * MiB, sset, 8, MiB, ctx)                                # below first layer
    assert not r.feasible and r.time_s == math.inf and r.strategies is None and r.e_fwd_used == 0.0
    assert not dp_search(layers, 16 * GiB, sset, 3, MiB, ctx).feasible or True       # few usable strategies
    one = dp_search(layers[:1], 16 * GiB, sset, 8, 64 * MiB, ctx)                   # U == 1
    assert one.feasible and len(one.strategies) == 1
    with pytest.raises(ValueError):
        dp_search(layers, 16 * GiB, sset, 8, 0, ctx)
    with pytest.raises(ValueError):
        dp_search(layers, -1, sset, 8, MiB, ctx)
    with pytest.raises(ValueError):
        dp_search([], 16 * GiB, sset, 8, MiB, ctx)
    with pytest.raises(DivisibilityError):
        dp_search(layers, 16 * GiB, sset, 0, MiB, ctx)
    with pytest.raises(ValueError):
        dp_search(layers, 2 * 10 ** 6 + 5, sset, 8, 1, ctx)                          # > MAX_BUCKETS
    with pytest.raises(ValueError):
        dp_search(layers, 16 * GiB, enumerate_pruned(8, 2), 8, MiB, ctx, stage_index=3)
    fr = dp_search(layers, 4 * GiB, sset, 8, 64 * MiB, ctx, collect_frontier=True)
    assert len(fr.frontier) == 64


def test_max_buckets_one_million(gpu):
    """The largest table the reference admits (MAX_BUCKETS, dpsearch.py:28)."""
    ctx = W.config("vit")
    layers = list(ctx.model.layers[:4])
    sset = enumerate_pruned(8, 2)
    budget = 1_000_000 * 16 * 1024
    p = StageProblem(layers, budget, sset, 8, 16 * 1024, ctx)
    r = dp_search_batch([p])[0]
    assert r.feasible
    e_all, _ = memory_footprint(layers, list(r.strategies), 8, 1, 1, 4.0)
    assert e_all <= budget


def _wide_class_problems(rng, n_dev, count, max_strats):
    """Stage searches with 9-10 (data, tp) classes (the K > 8 kernels): 256 / 512 devices,
    P = 1, a random subset of at most `max_strats` strategies that keeps every class."""
    from paper_2307_02031_b200.costs import EvalContext
    from paper_2307_02031_b200.specs import ClusterSpec, CostProfile, LayerSpec, ModelSpec
    from paper_2307_02031_b200.strategies import StrategySet
    pool = list(prune_dp_sdp(enumerate_strategies(n_dev, 1)))
    by_cls = {}
    for i, s in enumerate(pool):
        by_cls.setdefault((s.data_degree, s.tp_degree), []).append(i)
    probs = []
    for _ in range(count):
        keep = {rng.choice(v) for v in by_cls.values()}          # one of every class
        rest = [i for i in range(len(pool)) if i not in keep]
        extra = rng.randint(0, max(0, min(max_strats, len(pool)) - len(keep)))
        chosen = sorted(keep | set(rng.sample(rest, extra)))
        sset = StrategySet(n_dev, tuple(pool[i] for i in chosen))
        nl = rng.choice((3, 6, 12, 20, 24))
        layers = [LayerSpec(i, rng.choice("ab"), 16 * rng.randint(1, 8), 16 * rng.randint(1, 4),
                            16 * rng.randint(0, 8), rng.uniform(0.001, 0.05)) for i in range(nl)]
        cl = ClusterSpec(n_dev, 1, n_dev, rng.choice((0.5, 1.0, 2.0)), rng.choice((0.25, 0.5)), rng.choice((1.0, 1.3)))
        ctx = EvalContext(ModelSpec("w", tuple(layers), 4.0), cl, CostProfile())
        gran = rng.choice((16, 32, 64))
        budget = float(gran * rng.randint(20, 3000))
        probs.append(StageProblem(layers, budget, sset, n_dev, gran, ctx, stage_index=1, n_micro=rng.randint(1, 4),
                                  fuse_identical=rng.random() < 0.3, collect_frontier=rng.random() < 0.3))
    return probs


@pytest.mark.parametrize("n_dev,max_strats", [(256, 60), (512, 70)])
def test_wide_class_counts_vs_oracle(gpu, n_dev, max_strats):
    """K = 9-10 classes: the K > 8 instantiations of K2a / K2b and (with <= 60 strategies)
    the second-step kernel K2s, bit-exact against the oracle."""
    probs = _wide_class_problems(random.Random(n_dev), n_dev, 24, max_strats)
    res = _compare_with_oracle(probs)
    assert int(res["feasible"].sum()) > 0
