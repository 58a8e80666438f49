"""The planner drivers on the device path against golden outcomes of the live
reference (tests/golden/make_golden_drivers.py): galvatron_search cells,
Algorithm 1 plans (galvatron_base / plan_full), the infeasible-smallest-batch
error, Algorithm 2 trajectories and plan_full with the BMW refinement."""

import pytest

from golden_cases import load
from paper_2307_02031_b200 import workloads as W
from paper_2307_02031_b200.balance import PipelinePartition, bi_objective_optimize, partition_layers
from paper_2307_02031_b200.errors import InfeasiblePlanError
from paper_2307_02031_b200.planner import GalvatronSearch, PlannerOptions, galvatron_base, galvatron_search, plan_full

pytestmark = pytest.mark.gpu


def _drivers():
    try:
        return load("drivers.json")
    except FileNotFoundError:
        pytest.skip("drivers.json not generated")


def _outcome(o):
    if o.strategies is None:
        return {"cost": o.cost.hex(), "n_micro": o.n_micro, "strategies": None}
    return {"cost": o.cost.hex(), "n_micro": o.n_micro, "strategies": [s.to_string() for s in o.strategies],
            "stage_costs": [[sc.time_s.hex(), sc.time_no_sync_s.hex(), sc.peak_mem_bytes.hex()]
                            for sc in o.stage_costs]}


def _plan(plan):
    return {"doc": plan.to_document(), "time_hex": plan.predicted_time_s.hex(),
            "thr_hex": plan.predicted_throughput.hex(),
            "alpha": [plan.balance.alpha_t.hex(), plan.balance.alpha_m.hex()],
            "peaks": [x.hex() for x in plan.peak_mem_per_stage], "strategies": [s.to_string() for s in plan.strategies]}


def test_search_cells(gpu):
    for c in _drivers()["search"]:
        ctx = W.config(c["model"], c["budget"])
        stages = partition_layers(ctx.model, PipelinePartition(tuple(c["partition"])))
        o = galvatron_search(c["budget"], stages, ctx.cluster.n_devices, c["batch"], c["P"], ctx)
        assert _outcome(o) == c["outcome"], (c["model"], c["batch"], c["P"])


def test_algorithm1_plans(gpu):
    for c in _drivers()["base"]:
        ctx = W.config(c["model"], c["budget"])
        plan = plan_full(ctx.model, ctx.cluster, ctx.profile, PlannerOptions())
        got = _plan(plan)
        ref = dict(c["plan"])
        assert got["doc"] == ref["doc"], (c["model"], c["budget"])
        assert got == ref


def test_algorithm1_window_independent(gpu):
    """The speculative batch window must not change the plan."""
    c = _drivers()["base"][0]
    ctx = W.config(c["model"], c["budget"])
    for window in (1, 5, 32, 0):
        plan = galvatron_base(ctx.model, ctx.cluster, ctx.profile, PlannerOptions(batch_window=window))
        assert _plan(plan) == c["plan"]


def test_infeasible_smallest_batch(gpu):
    ref = _drivers()["infeasible"]
    ctx = W.config("gpt", 1 << 30)
    with pytest.raises(InfeasiblePlanError) as info:
        galvatron_base(ctx.model, ctx.cluster, ctx.profile, PlannerOptions())
    assert str(info.value) == ref["message"]
    diag = info.value.diagnostics
    assert diag["batch_size"] == ref["diagnostics"]["batch_size"]
    assert {str(k): v for k, v in diag["per_pp_degree"].items()} == ref["diagnostics"]["per_pp_degree"]


def _traj(r):
    out = []
    for rec in r.trajectory:
        rr = dict(rec)
        for k in ("cost", "alpha_t", "alpha_m", "max_stage_time", "max_stage_mem"):
            if k in rr:
                rr[k] = rr[k].hex()
        out.append(rr)
    return out


@pytest.mark.parametrize("batched", [True, False])
def test_algorithm2_trajectories(gpu, batched):
    for c in _drivers()["bmw"]:
        ctx = W.config(c["model"], 16 << 30)
        search = GalvatronSearch(ctx, PlannerOptions())
        if not batched:                     # a plain SearchFn: sequential calls
            fn = search.__call__
            search = lambda *args: fn(*args)  # noqa: E731
        r = bi_objective_optimize(ctx.model, ctx, c["batch_sizes"], c["P"], search)
        assert r.cost.hex() == c["cost"]
        assert r.batch_size == c["batch"] and r.n_micro == c["n_micro"]
        assert (list(r.partition.stage_sizes) if r.partition else None) == c["partition"]
        assert ([s.to_string() for s in r.strategies] if r.strategies else None) == c["strategies"]
        assert _traj(r) == c["trajectory"], c["model"]


def test_plan_full_bmw(gpu):
    for c in _drivers()["full_bmw"]:
        ctx = W.config(c["model"], c["budget"])
        plan = plan_full(ctx.model, ctx.cluster, ctx.profile, PlannerOptions(bi_objective=True))
        assert _plan(plan) == c["plan"], c["model"]
