"""plan_full latency against galvatron_base's batch window (GPU box):
python tools/window_probe.py [workloads...]; prints median wall ms of 5 runs per window size."""
import dataclasses, json, sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2307_02031_b200 import dpsearch, workloads as W
from paper_2307_02031_b200.planner import PlannerOptions, plan_full

torch.cuda.set_device(0)
names = sys.argv[1:] or ["swin-bmw", "vit-bmw", "gpt96", "bert", "t5-16"]
for name in names:
    bmw = name.endswith("-bmw"); base = name[:-4] if bmw else name
    budget = None
    if base.startswith("t5-"):
        budget = int(base.split("-")[1]) << 30; base = "t5"
    ctx = W.config("gpt" if base == "gpt96" else base, budget)
    ref = None
    for win in (8, 16, 32, 64):
        opts = PlannerOptions(granularity_bytes=1 << 20, bi_objective=bmw, batch_window=win)
        plan_full(ctx.model, ctx.cluster, ctx.profile, opts)
        lat, dev, nb = [], [], 0
        for _ in range(5):
            dpsearch.reset_stats()
            t0 = time.perf_counter()
            plan = plan_full(ctx.model, ctx.cluster, ctx.profile, opts)
            lat.append(time.perf_counter() - t0)
            dev.append(dpsearch.STATS["total_ms"]); nb = dpsearch.STATS["batches"]
        key = (plan.batch_size, plan.pp_degree, tuple(plan.partition), plan.predicted_time_s)
        ref = ref or key
        print(json.dumps({"workload": name, "window": win, "ms": round(1e3 * float(np.median(lat)), 2),
                          "device_ms": round(float(np.median(dev)), 2), "batches": nb, "same_plan": key == ref}),
              flush=True)
