"""BASELINE config 4 — GPT-3-96 on 64 simulated GPUs, 80 GiB.

* Algorithm 1 at 1 GiB granularity over batch sizes 8..64 against the live
  reference's plan (tests/golden/gpt_base.json, minutes on the reference).
* The full 1 MiB search over all batch sizes (hours on the reference): the
  returned plan's stage searches are re-run through the oracle (bit-exact), and the
  plan's predicted time is re-costed through the reference cost path."""

import numpy as np
import pytest

from golden_cases import load
from oracle import oracle as O
from paper_2307_02031_b200 import dpsearch, workloads as W
from paper_2307_02031_b200.balance import PipelinePartition, partition_layers
from paper_2307_02031_b200.planner import PlannerOptions, evaluate_plan_document, plan_full
from paper_2307_02031_b200.strategies import enumerate_pruned

pytestmark = pytest.mark.gpu
MiB, GiB = 1 << 20, 1 << 30


def test_gpt_algorithm1_coarse_matches_reference(gpu):
    try:
        ref = load("gpt_base.json")
    except FileNotFoundError:
        pytest.skip("gpt_base.json not generated")
    ctx = W.config("gpt")
    plan = plan_full(ctx.model, ctx.cluster, ctx.profile, PlannerOptions(**ref["opts"]))
    assert plan.to_document() == ref["plan"]["doc"]
    assert plan.predicted_time_s.hex() == ref["plan"]["time_hex"]
    assert [x.hex() for x in plan.peak_mem_per_stage] == ref["plan"]["peaks"]


def test_gpt_full_search_1mib_stage_parity(gpu):
    ctx = W.config("gpt")
    plan = plan_full(ctx.model, ctx.cluster, ctx.profile, PlannerOptions(granularity_bytes=MiB))
    doc = plan.to_document()
    # the plan re-costs to its own predicted time through the stage_cost path
    assert evaluate_plan_document(doc, ctx.model, ctx.cluster, ctx.profile) == plan.predicted_time_s
    # every stage search of the winning cell, through the oracle (the reference algorithm)
    P, m = plan.pp_degree, plan.n_micro
    micro = plan.batch_size // m
    stages = partition_layers(ctx.model, PipelinePartition(plan.partition))
    sset = enumerate_pruned(64, P)
    probs = [dpsearch.StageProblem(st, ctx.cluster.mem_budget_bytes, sset, micro, MiB, ctx, i + 1, m)
             for i, st in enumerate(stages)]
    import test_gpu_parity as T
    layers, strats, envs, arr = T._flat(probs)
    rc, msg, res, plans, _ = dpsearch.run_native_batch(layers, strats, envs, arr)
    assert rc == 0, msg
    ores, oplans, _, _ = O.search_many(layers, strats, envs, arr)
    for f in ("time_s", "e_fwd", "stage_time", "stage_ns", "stage_peak"):
        assert np.array_equal(res[f].view(np.int64), ores[f].view(np.int64)), f
    n = int(arr["n_layers"].sum())
    assert np.array_equal(plans[:n], oplans[:n])
    got = [s.to_string() for s in plan.strategies]
    strat_list = list(sset)
    assert got == [strat_list[j].to_string() for j in oplans[:n]]
