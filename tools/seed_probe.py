"""Seed partitions of one GPT-3-96 batch window: host threads vs the device kernel."""
import sys, time
sys.path.insert(0, '.')
from paper_2307_02031_b200 import workloads as W, balance as B, _native
from paper_2307_02031_b200.planner import init_microbatch_num
from paper_2307_02031_b200.strategies import candidate_pp_degrees
for name in ("gpt", "swin"):
    ctx = W.config(name)
    cells = []
    for b in range(8, 8 * 17, 8):
        for p in candidate_pp_degrees(ctx.cluster.n_devices):
            if p <= ctx.model.num_layers:
                m = init_microbatch_num(b, p); cells.append((p, b // m, m))
    dev = _native.default_context()
    for k in range(3):
        t0 = time.perf_counter(); h = B.seed_partitions(ctx.model, ctx, ctx.cluster.n_devices, cells); t1 = time.perf_counter()
        d = B.seed_partitions(ctx.model, ctx, ctx.cluster.n_devices, cells, device=dev); t2 = time.perf_counter()
    assert h == d
    print(f"{name}: {len(cells)} cells, host threads {1e3*(t1-t0):.1f} ms, device {1e3*(t2-t1):.1f} ms", flush=True)
