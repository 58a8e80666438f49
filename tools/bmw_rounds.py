"""Where Algorithm 2's time goes (GPU box): per lockstep round, the batched search call vs
the rest; python tools/bmw_rounds.py swin|vit|gpt"""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2307_02031_b200 import dpsearch, workloads as W
from paper_2307_02031_b200.planner import (PlannerOptions, galvatron_base, GalvatronSearch, init_microbatch_num,
                                           candidate_pp_degrees, EvalContext)
from paper_2307_02031_b200.balance import bi_objective_multi
name = sys.argv[1]
ctx0 = W.config(name)
opts = PlannerOptions(granularity_bytes=1 << 20, bi_objective=True)
torch.cuda.set_device(0)
base = galvatron_base(ctx0.model, ctx0.cluster, ctx0.profile, opts)
ctx = EvalContext(model=ctx0.model, cluster=ctx0.cluster, profile=ctx0.profile)
search = GalvatronSearch(ctx, opts)
mp = lambda b, p: init_microbatch_num(b, p, opts.microbatch_cap_factor, opts.min_micro_size)
b0 = base.batch_size
bs = list(range(max(opts.batch_step, b0 - opts.batch_radius), b0 + opts.batch_radius + 1, opts.batch_step))
degs = [p for p in candidate_pp_degrees(ctx0.cluster.n_devices) if 2 <= p <= ctx0.model.num_layers]
inner = search.batch
log = []
first_call = []
import paper_2307_02031_b200.balance as B
ev_inner = B.evaluate_partition
ev_t = [0.0, 0]
def ev_timed(*a, **k):
    t0 = time.perf_counter()
    r = ev_inner(*a, **k)
    ev_t[0] += time.perf_counter() - t0; ev_t[1] += 1
    return r
B.evaluate_partition = ev_timed
def timed(calls):
    if not first_call:
        first_call.append(time.perf_counter())
    dpsearch.reset_stats()
    t0 = time.perf_counter()
    r = inner(calls)
    log.append((len(calls), 1e3 * (time.perf_counter() - t0), dpsearch.STATS["total_ms"]))
    return r
search.batch = timed
bi_objective_multi(ctx0.model, ctx, bs, degs, search, mp)
for _ in range(3):
    log.clear(); first_call.clear(); ev_t[0] = 0.0; ev_t[1] = 0
    t0 = time.perf_counter()
    bi_objective_multi(ctx0.model, ctx, bs, degs, search, mp)
    tot = 1e3 * (time.perf_counter() - t0)
print(f"setup (to the first search call) {1e3 * (first_call[0] - t0):.2f} ms; evaluate_partition {ev_t[1]} calls "
      f"{1e3 * ev_t[0]:.2f} ms (setup threads included)")
print(f"total {tot:.2f} ms; rounds {len(log)}; search calls {sum(x[1] for x in log):.2f} ms "
      f"(device {sum(x[2] for x in log):.2f} ms); rest {tot - sum(x[1] for x in log):.2f} ms")
for n, ms, dev in log:
    print(f"  {n:3d} searches  call {ms:6.3f} ms  device {dev:6.3f} ms")
