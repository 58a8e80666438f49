"""cProfile of Algorithm 2 (bi_objective_multi) alone, as plan_full issues it (GPU box):
python tools/bmw_cprofile.py swin|vit|gpt"""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import torch
from paper_2307_02031_b200 import workloads as W
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
bi_objective_multi(ctx0.model, ctx, bs, degs, search, mp)
t0 = time.perf_counter()
for _ in range(3):
    bi_objective_multi(ctx0.model, ctx, bs, degs, search, mp)
print(f"bi_objective_multi {1e3 * (time.perf_counter() - t0) / 3:.2f} ms, batches {bs}, degrees {degs}")
pr = cProfile.Profile(); pr.enable()
for _ in range(3):
    bi_objective_multi(ctx0.model, ctx, bs, degs, search, mp)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
