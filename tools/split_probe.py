"""Device time of the 10k sweep split by depth: all searches, the deep ones only (units > 16)
and the rest, each as its own batch (median of 5 runs):
python tools/split_probe.py [all]  (GPU box; "all": the whole sweep only)."""
import statistics
import sys

sys.path.insert(0, '.')
from paper_2307_02031_b200 import workloads as W, _native   # noqa: E402
from paper_2307_02031_b200.dpsearch import SearchBatch     # noqa: E402

cells = W.sweep_cells(10000)
L, S, E, P, T = W.sweep_arrays(cells)
deep = P["n_layers"] > 16
gpt1 = (P["n_layers"] >= 90)
ctx = _native.Context(0)


def run(mask, name):
    p = P[mask]
    ts = []
    for _ in range(6):
        b = SearchBatch(L, S, E, p, ctx)
        b.run()
        t = b.timing()
        b.close()
        ts.append((t['total_ms'], t['dp_ms'], t['sweep_ms']))
    ts = ts[1:]
    print(f"{name:10s} {int(mask.sum()):6d} searches: device {statistics.median(x[0] for x in ts):6.2f} ms, "
          f"dp {statistics.median(x[1] for x in ts):6.2f}, sweep {statistics.median(x[2] for x in ts):5.2f}",
          flush=True)


import numpy as np   # noqa: E402
run(np.ones(len(P), bool), "all")
if len(sys.argv) > 1 and sys.argv[1] == "all":
    sys.exit(0)
run(deep, "deep>16")
run(~deep, "shallow")
run(gpt1, "gpt P=1")
run(~gpt1, "not gptP1")
