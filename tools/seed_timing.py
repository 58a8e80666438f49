"""Host seed-partition timing of one GPT-3-96 batch window (16 batch sizes x 7 degrees):
python tools/seed_timing.py"""
import os
import sys
import time

sys.path.insert(0, '.')
from paper_2307_02031_b200 import workloads as W                     # noqa: E402
from paper_2307_02031_b200.balance import seed_partitions            # noqa: E402
from paper_2307_02031_b200.costs import EvalContext                  # noqa: E402
from paper_2307_02031_b200.planner import init_microbatch_num        # noqa: E402

c = W.config("gpt")
ctx = EvalContext(c.model, c.cluster, c.profile)
cells = []
for b in range(320, 448, 8):
    for P in (1, 2, 4, 8, 16, 32, 64):
        m = init_microbatch_num(b, P)
        cells.append((P, b // m, m))
print("affinity", len(os.sched_getaffinity(0)), "cpus", os.cpu_count())
for th in (1, 4, 8, 16, 32):
    seed_partitions(c.model, ctx, c.cluster.n_devices, cells, n_threads=th)
    t0 = time.perf_counter()
    for _ in range(5):
        seed_partitions(c.model, ctx, c.cluster.n_devices, cells, n_threads=th)
    print(th, "threads:", f"{(time.perf_counter() - t0) / 5 * 1e3:.2f} ms per window")
