"""Per device batch of a full planner search: problems, max units, device ms, call ms (GPU box).
usage: python tools/batch_log.py swin-bmw [gpt96 ...]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2307_02031_b200 import dpsearch, planner, workloads as W, _native
from paper_2307_02031_b200.planner import PlannerOptions, plan_full

log = []
_orig = dpsearch.run_native_batch
def logged(layers, strats, envs, probs, context=None):
    t0 = time.perf_counter()
    r = _orig(layers, strats, envs, probs, context)
    dt = 1e3 * (time.perf_counter() - t0)
    t = _native.Timing()
    _native.lib().gbmw_ctx_last_timing((context or _native.default_context()).handle, __import__('ctypes').byref(t))
    log.append((len(probs), int(probs["n_layers"].max()) if len(probs) else 0, int(probs["n_buckets"].max()) if len(probs) else 0,
                t.total_ms, t.dp_ms, t.sweep_ms, t.prep_ms, t.n_launches, dt))
    return r
dpsearch.run_native_batch = logged
T0 = time.perf_counter()
events = []
_L = _native.lib()
_sb = _L.gbmw_search_batch
def sb(*a):
    t0 = time.perf_counter(); r = _sb(*a); events.append(("native_search", t0 - T0, time.perf_counter() - T0)); return r
_L.gbmw_search_batch = sb
_sp = _L.gbmw_seed_partitions
def sp(*a):
    t0 = time.perf_counter(); r = _sp(*a); events.append(("native_seed", t0 - T0, time.perf_counter() - T0)); return r
_L.gbmw_seed_partitions = sp
_bw = planner._base_cells_window
def bw(*a, **k):
    t0 = time.perf_counter(); r = _bw(*a, **k); events.append(("base_cells_window", t0 - T0, time.perf_counter() - T0)); return r
planner._base_cells_window = bw
import gc
_gc = {}
def gccb(phase, info):
    if phase == "start": _gc["t"] = time.perf_counter()
    else: events.append((f"gc gen{info['generation']} ({info['collected']})", _gc["t"] - T0, time.perf_counter() - T0))
gc.callbacks.append(gccb)
torch.cuda.set_device(0)
for name in sys.argv[1:]:
    bmw = name.endswith("-bmw"); base = name[:-4] if bmw else name
    ctx = W.config("gpt" if base == "gpt96" else base)
    opts = PlannerOptions(granularity_bytes=1 << 20, bi_objective=bmw)
    for k in range(3):
        log.clear(); events.clear()
        t0 = time.perf_counter(); plan_full(ctx.model, ctx.cluster, ctx.profile, opts); dt = 1e3 * (time.perf_counter() - t0)
    a = np.array(log)
    print(f"{name}: total {dt:.1f} ms, {len(log)} batches, device {a[:,3].sum():.1f} ms, calls {a[:,8].sum():.1f} ms")
    print("  probs  maxL maxB   dev_ms   dp_ms  sweep_ms prep_ms launches call_ms")
    for r in log:
        print("  %5d %5d %5d %8.3f %7.3f %8.3f %7.3f %8d %7.3f" % r)
    e0 = min(e[1] for e in events) if events else 0
    for n, a, b in sorted(events, key=lambda e: e[1]):
        print(f"  {n:18s} {1e3*(a-e0):8.2f} -> {1e3*(b-e0):8.2f}  ({1e3*(b-a):.2f} ms)")
