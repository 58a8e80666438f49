"""Golden fixtures for the planner drivers, generated from the LIVE reference.

    python tests/golden/make_golden_drivers.py            (build container only; minutes)

Covers the host-side partition logic (parapilot/balance.py: _seed_for, memory/time
balanced partitions, evaluate_partition) on every benchmark model, and the
drivers on the benchmark configs at the reference's default 64 MiB granularity:
galvatron_search cells, galvatron_base / plan_full plans (BERT-Huge-32 16 GiB,
T5-Large-48 8/12/16/20 GiB), plan_full with the BMW refinement (ViT-Huge-32,
Swin-Huge-48 at 16 GiB) and bi_objective_optimize trajectories.
Writes partitions.json and drivers.json next to this script.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import parapilot as R                                      # noqa: E402
from parapilot import balance as RB                        # noqa: E402
from parapilot import planner as RP                        # noqa: E402
from parapilot.strategies import candidate_pp_degrees     # noqa: E402

from paper_2307_02031_b200 import workloads as W           # noqa: E402  (fixed synthetic specs only)

OUT = Path(__file__).resolve().parent
GiB = 1 << 30


def hx(x) -> str:
    return float(x).hex()


def ref_ctx(name, budget=None):
    c = W.config(name, budget)
    model = R.load_model_spec(c.model.to_document())
    cluster = R.load_cluster_spec(c.cluster.to_document())
    return model, cluster, R.CostProfile()


def costs_doc(costs):
    return [[hx(sc.time_s), hx(sc.time_no_sync_s), hx(sc.peak_mem_bytes)] for sc in costs]


def plan_doc(plan):
    return {"doc": plan.to_document(), "time_hex": hx(plan.predicted_time_s),
            "thr_hex": hx(plan.predicted_throughput), "alpha": [hx(plan.balance.alpha_t), hx(plan.balance.alpha_m)],
            "peaks": [hx(x) for x in plan.peak_mem_per_stage], "strategies": [s.to_string() for s in plan.strategies]}


def outcome_doc(o):
    if o.strategies is None:
        return {"cost": hx(o.cost), "n_micro": o.n_micro, "strategies": None}
    return {"cost": hx(o.cost), "n_micro": o.n_micro, "strategies": [s.to_string() for s in o.strategies],
            "stage_costs": costs_doc(o.stage_costs)}


def gen_partitions():
    out = []
    for name, budgets, batches in (("bert", [16 * GiB], [8, 64, 256]), ("t5", [8 * GiB, 20 * GiB], [16, 128]),
                                   ("vit", [16 * GiB], [32, 512]), ("swin", [16 * GiB], [8, 96]),
                                   ("gpt", [80 * GiB], [64, 1024])):
        for budget in budgets:
            model, cluster, profile = ref_ctx(name, budget)
            ctx = R.EvalContext(model, cluster, profile)
            for B in batches:
                for P in candidate_pp_degrees(cluster.n_devices):
                    if P > model.num_layers or (name == "gpt" and P > 16 and B != 64):
                        continue
                    for policy in ("init", "default"):
                        m = RP.init_microbatch_num(B, P) if policy == "init" else RB.default_microbatch_policy(B, P)
                        micro = B // m
                        seeds = RB._seed_for(model, ctx, cluster.n_devices, P, micro, m)
                        pm = RB.init_partition_memory_balanced(model, P, seeds, micro, m, ctx)
                        pt = RB.init_partition_time_balanced(model, P, seeds, micro, m, ctx)
                        out.append({"model": name, "budget": budget, "batch": B, "P": P, "n_micro": m, "micro": micro,
                                    "seed": seeds[0].to_string(), "p_m": list(pm.stage_sizes),
                                    "p_t": list(pt.stage_sizes),
                                    "costs_m": costs_doc(RB.evaluate_partition(model, pm, seeds, micro, m, ctx)),
                                    "costs_t": costs_doc(RB.evaluate_partition(model, pt, seeds, micro, m, ctx))})
    return out


def gen_drivers():
    doc = {"search": [], "base": [], "bmw": [], "full_bmw": []}
    t0 = time.time()
    opts = RP.PlannerOptions()
    # galvatron_search cells on memory-balanced seeds
    for name, budget in (("bert", 16 * GiB), ("t5", 8 * GiB), ("swin", 16 * GiB), ("gpt", 80 * GiB)):
        model, cluster, profile = ref_ctx(name, budget)
        ctx = R.EvalContext(model, cluster, profile)
        for B in (8, 64, 512):
            for P in candidate_pp_degrees(cluster.n_devices):
                if P > model.num_layers or (name == "gpt" and P > 8):
                    continue
                m = RP.init_microbatch_num(B, P)
                seeds = RB._seed_for(model, ctx, cluster.n_devices, P, B // m, m)
                part = RB.init_partition_memory_balanced(model, P, seeds, B // m, m, ctx)
                o = RP.galvatron_search(budget, RB.partition_layers(model, part), cluster.n_devices, B, P, ctx, opts)
                doc["search"].append({"model": name, "budget": budget, "batch": B, "P": P,
                                      "partition": list(part.stage_sizes), "outcome": outcome_doc(o)})
    print(f"search cells: {time.time() - t0:.1f}s", flush=True)
    # Algorithm 1
    for name, budget in (("bert", 16 * GiB), ("t5", 8 * GiB), ("t5", 12 * GiB), ("t5", 16 * GiB), ("t5", 20 * GiB)):
        model, cluster, profile = ref_ctx(name, budget)
        plan = RP.plan_full(model, cluster, profile, opts)
        doc["base"].append({"model": name, "budget": budget, "plan": plan_doc(plan)})
        print(f"base {name} {budget // GiB}: {time.time() - t0:.1f}s", flush=True)
    # infeasible smallest batch
    model, cluster, profile = ref_ctx("gpt", 1 * GiB)
    try:
        RP.galvatron_base(model, cluster, profile, opts)
        doc["infeasible"] = None
    except R.InfeasiblePlanError as exc:
        doc["infeasible"] = {"message": str(exc), "diagnostics": {k: (v if not isinstance(v, dict) else
                                                                      {str(a): b for a, b in v.items()})
                                                                  for k, v in exc.diagnostics.items()}}
    # Algorithm 2 trajectories
    for name, bs, P in (("bert", [8, 16, 24], 2), ("swin", [16, 32], 4), ("vit", [8, 64], 8), ("t5", [32], 1)):
        model, cluster, profile = ref_ctx(name, 16 * GiB)
        ctx = R.EvalContext(model, cluster, profile)

        def search(budget, stages, n_devices, batch, pp_degree, ctx=ctx):
            return RP.galvatron_search(budget, stages, n_devices, batch, pp_degree, ctx, opts)
        r = RB.bi_objective_optimize(model, ctx, bs, P, search)
        traj = []
        for rec in r.trajectory:
            rr = dict(rec)
            for k in ("cost", "alpha_t", "alpha_m", "max_stage_time", "max_stage_mem"):
                if k in rr:
                    rr[k] = hx(rr[k])
            traj.append(rr)
        doc["bmw"].append({"model": name, "batch_sizes": bs, "P": P, "cost": hx(r.cost), "batch": r.batch_size,
                           "n_micro": r.n_micro, "partition": list(r.partition.stage_sizes) if r.partition else None,
                           "strategies": [s.to_string() for s in r.strategies] if r.strategies else None,
                           "trajectory": traj})
        print(f"bmw {name} P={P}: {time.time() - t0:.1f}s", flush=True)
    # plan_full with BMW (BASELINE config 3)
    for name in ("vit", "swin"):
        model, cluster, profile = ref_ctx(name, 16 * GiB)
        plan = RP.plan_full(model, cluster, profile, RP.PlannerOptions(bi_objective=True))
        doc["full_bmw"].append({"model": name, "budget": 16 * GiB, "plan": plan_doc(plan)})
        print(f"plan_full bmw {name}: {time.time() - t0:.1f}s", flush=True)
    return doc


def main():
    t0 = time.time()
    parts = gen_partitions()
    (OUT / "partitions.json").write_text(json.dumps(parts, separators=(",", ":")))
    print(f"partitions: {len(parts)} cases, {time.time() - t0:.1f}s", flush=True)
    if "--partitions-only" in sys.argv:
        return
    (OUT / "drivers.json").write_text(json.dumps(gen_drivers(), separators=(",", ":")))
    print(f"drivers: {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
