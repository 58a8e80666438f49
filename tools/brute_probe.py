"""Exhaustive planner oracle (gbmw_brute_force) throughput on the device vs the C
restatement on one host core, on instances past the reference's 4-layer / 4-device guard:
python tools/brute_probe.py   (GPU box)."""
import json
import sys
import time

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from golden_cases import brute_records                                      # noqa: E402
from oracle import oracle as O                                              # noqa: E402
from paper_2307_02031_b200 import brute_force_oracle                        # noqa: E402
from paper_2307_02031_b200.planner import last_oracle_stats                 # noqa: E402
from paper_2307_02031_b200.specs import load_cluster_spec, load_cost_profile, load_model_spec   # noqa: E402

rows = []
for (n_dev, L, batch) in [(8, 5, 8), (8, 6, 8), (4, 7, 8), (8, 7, 4)]:
    layers = [{"kind": "enc", "param_bytes": (40 + 17 * i) * 1_000_000, "bnd_bytes_per_sample": (4 + i) * 262_144,
               "int_bytes_per_sample": (8 + 3 * i) * 1_048_576, "fwd_time_per_sample": 0.002 + 0.0007 * i,
               "tp_act_replication_fraction": 0.25} for i in range(L)]
    model = load_model_spec({"name": "probe", "ms_bytes_per_param_byte": 4.0, "layers": layers})
    tot = sum(l["param_bytes"] * 4.0 + batch * (l["bnd_bytes_per_sample"] + l["int_bytes_per_sample"]) for l in layers)
    cluster = load_cluster_spec({"n_devices": n_dev, "mem_budget_bytes": int(tot * 0.3), "island_size": min(4, n_dev),
                                 "intra_island_bw": 50e9, "inter_island_bw": 12e9, "overlap_slowdown": 1.3})
    profile = load_cost_profile({}, model)
    brute_force_oracle(model, cluster, profile, batch, max_layers=L, max_devices=n_dev)      # warm-up
    t0 = time.perf_counter()
    r = brute_force_oracle(model, cluster, profile, batch, max_layers=L, max_devices=n_dev)
    wall = time.perf_counter() - t0
    n = last_oracle_stats["assignments"]
    dev = last_oracle_stats["device_ms"] / 1e3
    lay, env = brute_records(model, cluster, profile)
    t0 = time.perf_counter()
    c = O.brute_force(lay, env, batch, cluster.mem_budget_bytes)
    cpu = time.perf_counter() - t0
    assert (c[0].hex(), c[1], c[2], c[3]) == (r.cost.hex(), r.feasible, r.pp_degree, r.n_micro)
    rows.append({"n_devices": n_dev, "layers": L, "batch": batch, "assignments": n, "device_s": dev, "call_s": wall,
                 "gpu_assignments_per_s": n / dev, "cpu_1core_s": cpu, "cpu_assignments_per_s": n / cpu,
                 "speedup_device": cpu / dev, "plan": [r.pp_degree, r.n_micro, list(r.partition)]})
    print(json.dumps(rows[-1]), flush=True)
