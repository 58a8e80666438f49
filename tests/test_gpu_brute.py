"""The exhaustive planner oracle on the device (gbmw_brute_force, planner.py:364-449):
bit-exact against the live reference's outcomes (tests/golden/brute.json) and, past the
reference's guards (up to 8 layers, 8 devices), against the oracle's restatement."""

import random

import pytest

from golden_cases import brute_objects, brute_records, load
from oracle import oracle as O
from paper_2307_02031_b200 import brute_force_oracle
from paper_2307_02031_b200.planner import last_oracle_stats
from paper_2307_02031_b200.specs import load_cluster_spec, load_cost_profile, load_model_spec
from paper_2307_02031_b200.strategies import enumerate_pruned

pytestmark = pytest.mark.gpu


def test_brute_force_golden(gpu):
    for c in load("brute.json")["cases"]:
        model, cluster, profile = brute_objects(c)
        r = brute_force_oracle(model, cluster, profile, c["batch"], max_layers=8, max_devices=8)
        out = c["out"]
        got = {"feasible": r.feasible, "cost": r.cost.hex(), "pp_degree": r.pp_degree,
               "partition": list(r.partition), "n_micro": r.n_micro,
               "strategies": [s.to_string() for s in r.strategies]}
        assert got == out, (c["name"], got, out)


def _rand_instance(rng, n_dev, L):
    layers = [{"kind": "enc", "param_bytes": rng.randint(1, 300) * 1_000_000,
               "bnd_bytes_per_sample": rng.randint(1, 32) * 262_144,
               "int_bytes_per_sample": rng.randint(0, 48) * 1_048_576,
               "fwd_time_per_sample": rng.uniform(0.0005, 0.02),
               "tp_act_replication_fraction": rng.choice([0.0, 0.25, 0.5])} for _ in range(L)]
    model = load_model_spec({"name": "big", "ms_bytes_per_param_byte": 4.0, "layers": layers})
    batch = rng.choice([4, 8, 12])
    tot = sum(l["param_bytes"] * 4.0 + batch * (l["bnd_bytes_per_sample"] + l["int_bytes_per_sample"]) for l in layers)
    cluster = load_cluster_spec({"n_devices": n_dev, "mem_budget_bytes": int(tot * rng.choice([0.15, 0.3, 0.45, 0.7])),
                                 "island_size": min(4, n_dev), "intra_island_bw": 50e9, "inter_island_bw": 12e9,
                                 "overlap_slowdown": 1.3})
    return model, cluster, load_cost_profile({}, model), batch


@pytest.mark.parametrize("n_dev,L", [(8, 4), (8, 5), (4, 6), (2, 8)])
def test_brute_force_beyond_guards(gpu, n_dev, L):
    """Instances the reference's default guards refuse: device scan vs the C restatement."""
    rng = random.Random(1000 * n_dev + L)
    for _ in range(3):
        model, cluster, profile, batch = _rand_instance(rng, n_dev, L)
        r = brute_force_oracle(model, cluster, profile, batch, max_layers=L, max_devices=n_dev)
        layers, env = brute_records(model, cluster, profile)
        cost, feas, P, m, part, choice = O.brute_force(layers, env, batch, cluster.mem_budget_bytes)
        assert r.feasible == feas and r.cost.hex() == cost.hex()
        if feas:
            sset = enumerate_pruned(n_dev, P).strategies
            assert (r.pp_degree, r.n_micro, r.partition) == (P, m, part)
            assert r.strategies == tuple(sset[j] for j in choice)
        assert last_oracle_stats["assignments"] > 0
