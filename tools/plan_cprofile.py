"""cProfile of plan_full for one workload (after a warm-up run): python tools/plan_cprofile.py swin-bmw"""
import cProfile, pstats, sys
sys.path.insert(0, '.')
import torch
from paper_2307_02031_b200 import workloads as W
from paper_2307_02031_b200.planner import PlannerOptions, plan_full
name = sys.argv[1]
bmw = name.endswith("-bmw"); base = name[:-4] if bmw else name
ctx = W.config("gpt" if base == "gpt96" else base)
opts = PlannerOptions(granularity_bytes=1 << 20, bi_objective=bmw)
torch.cuda.set_device(0)
plan_full(ctx.model, ctx.cluster, ctx.profile, opts)
pr = cProfile.Profile(); pr.enable()
for _ in range(3):
    plan_full(ctx.model, ctx.cluster, ctx.profile, opts)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
