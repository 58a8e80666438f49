"""Golden fixtures of planner.brute_force_oracle, generated from the LIVE reference.

    python tests/golden/make_golden_brute.py            (build container only; ~1-2 min)

Instances: random small models (the reference helpers' random_tiny_model byte scale
and realistic GB-scale layers, mixed kinds, profile overrides, replication fractions),
clusters of 1-8 devices with islands / bandwidths / slowdowns drawn at random, batch
sizes with several divisors, budgets from infeasible to roomy.  The reference's size
guards are raised where needed (up to 5 layers, 8 devices) while keeping each call to
about a second of pure-Python scanning.  Writes brute.json next to this script; fp64 as
float.hex().
"""

from __future__ import annotations

import json
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

import parapilot as R                                    # noqa: E402
from parapilot import planner as RP                      # noqa: E402

OUT = Path(__file__).resolve().parent


def hx(x) -> str:
    return float(x).hex()


def rand_case(rng: random.Random, i: int):
    n_dev = rng.choice([1, 2, 2, 4, 4, 4, 8])
    if n_dev == 8:
        L = rng.choice([1, 2, 3])
    elif n_dev == 4:
        L = rng.choice([1, 2, 3, 4, 4])
    else:
        L = rng.choice([2, 3, 4, 5])
    big = rng.random() < 0.5
    layers = []
    for _ in range(L):
        if big:
            layers.append({"kind": rng.choice(["enc", "dec"]), "param_bytes": rng.randint(1, 400) * 1_000_000,
                           "bnd_bytes_per_sample": rng.randint(1, 64) * 262_144,
                           "int_bytes_per_sample": rng.randint(0, 64) * 1_048_576,
                           "fwd_time_per_sample": rng.uniform(0.0005, 0.02),
                           "tp_act_replication_fraction": rng.choice([0.0, 0.25, 0.5, 1.0])})
        else:
            layers.append({"kind": "enc", "param_bytes": 16 * rng.randint(1, 8),
                           "bnd_bytes_per_sample": 16 * rng.randint(1, 4),
                           "int_bytes_per_sample": 16 * rng.randint(0, 8),
                           "fwd_time_per_sample": rng.uniform(0.001, 0.05)})
    model = R.load_model_spec({"name": f"bf{i}", "ms_bytes_per_param_byte": rng.choice([2.0, 4.0, 6.0]),
                               "layers": layers})
    batch = rng.choice([1, 2, 3, 4, 6, 8, 12, 16])
    # budget between a fraction of the smallest and a multiple of the largest footprint
    tot = sum(l["param_bytes"] * model.ms_bytes_per_param_byte + batch * (l["bnd_bytes_per_sample"] +
              l["int_bytes_per_sample"]) for l in layers)
    budget = max(1, int(tot * rng.choice([0.02, 0.1, 0.2, 0.3, 0.4, 0.5, 0.7, 1.0, 3.0])))
    island = rng.choice([x for x in (1, 2, 4, 8) if x <= n_dev] or [1])
    intra = rng.choice([12e9, 50e9, 300e9])
    cluster = R.load_cluster_spec({"n_devices": n_dev, "mem_budget_bytes": budget, "island_size": island,
                                   "intra_island_bw": intra, "inter_island_bw": intra / rng.choice([1, 2, 6]),
                                   "overlap_slowdown": rng.choice([1.0, 1.3, 1.7])})
    overrides = {}
    if rng.random() < 0.3:
        overrides[str(rng.randrange(L))] = rng.uniform(0.001, 0.03)
    profile = R.load_cost_profile({"bwd_fwd_ratio": rng.choice([2.0, 1.5]),
                                   "collective_efficiency": rng.choice([1.0, 0.8]),
                                   "layer_overrides": overrides}, model)
    return model, cluster, profile, batch


def main():
    rng = random.Random(20261017)
    cases = []
    t0 = time.time()
    i = 0
    n_pipe = 0
    while len(cases) < 200:
        model, cluster, profile, batch = rand_case(rng, i)
        i += 1
        t = time.time()
        res = RP.brute_force_oracle(model, cluster, profile, batch, max_layers=8, max_devices=8)
        dt = time.time() - t
        if dt > 3.0:
            continue
        # after 160 draws keep only instances where a pipeline (P >= 2) wins
        if len(cases) >= 160 and res.pp_degree < 2:
            continue
        n_pipe += res.pp_degree >= 2
        cases.append({
            "name": f"bf{i - 1}",
            "model": model.to_document() if hasattr(model, "to_document") else {
                "name": model.name, "ms_bytes_per_param_byte": model.ms_bytes_per_param_byte,
                "layers": [{"kind": l.kind, "param_bytes": l.param_bytes,
                            "bnd_bytes_per_sample": l.bnd_bytes_per_sample,
                            "int_bytes_per_sample": l.int_bytes_per_sample,
                            "fwd_time_per_sample": l.fwd_time_per_sample,
                            "tp_act_replication_fraction": l.tp_act_replication_fraction} for l in model.layers]},
            "cluster": {"n_devices": cluster.n_devices, "mem_budget_bytes": cluster.mem_budget_bytes,
                        "island_size": cluster.island_size, "intra_island_bw": cluster.intra_island_bw,
                        "inter_island_bw": cluster.inter_island_bw, "overlap_slowdown": cluster.overlap_slowdown},
            "profile": {"bwd_fwd_ratio": profile.bwd_fwd_ratio,
                        "collective_efficiency": profile.collective_efficiency,
                        "layer_overrides": {str(k): v for k, v in profile.layer_overrides.items()}},
            "batch": batch,
            "out": {"feasible": res.feasible, "cost": hx(res.cost), "pp_degree": res.pp_degree,
                    "partition": list(res.partition), "n_micro": res.n_micro,
                    "strategies": [s.to_string() for s in res.strategies]},
            "ref_s": round(dt, 3),
        })
    (OUT / "brute.json").write_text(json.dumps({"generator": "make_golden_brute.py", "seed": 20261017,
                                                "cases": cases}, indent=0))
    n_feas = sum(c["out"]["feasible"] for c in cases)
    print(f"{len(cases)} cases ({n_feas} feasible, {n_pipe} pipelined) in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
