"""Where a full planner search spends its time (host seeding, device batches, Python)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2307_02031_b200 import planner, dpsearch, workloads as W
from paper_2307_02031_b200.planner import PlannerOptions, plan_full

acc = {}
def wrap(mod, name):
    f = getattr(mod, name)
    def g(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0; return r
    setattr(mod, name, g)
for n in ("_base_cells_window", "galvatron_search_batch", "_search_slices"):
    wrap(planner, n)
wrap(dpsearch, "run_native_batch")
planner.run_native_batch = dpsearch.run_native_batch if hasattr(planner, "run_native_batch") else None
torch.cuda.set_device(0)
for name in sys.argv[1:]:
    bmw = name.endswith("-bmw"); base = name[:-4] if bmw else name
    ctx = W.config("gpt" if base == "gpt96" else base)
    opts = PlannerOptions(granularity_bytes=1 << 20, bi_objective=bmw)
    for k in range(3):
        acc.clear(); dpsearch.reset_stats()
        t0 = time.perf_counter(); plan_full(ctx.model, ctx.cluster, ctx.profile, opts); dt = time.perf_counter() - t0
    print(name, f"total {1e3*dt:.1f} ms", {k: round(1e3 * v, 1) for k, v in acc.items()},
          f"device {dpsearch.STATS['total_ms']:.1f} ms batches {dpsearch.STATS['batches']}", flush=True)
