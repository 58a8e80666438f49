"""Run one subset of the 10k sweep once (for ncu): python tools/subset_run.py gpt1|deep|shallow|all [reps]"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2307_02031_b200 import workloads as W, _native
from paper_2307_02031_b200.dpsearch import SearchBatch
L, S, E, P, T = W.sweep_arrays(W.sweep_cells(10000))
masks = {"gpt1": P["n_layers"] >= 90, "deep": P["n_layers"] > 16, "shallow": P["n_layers"] <= 16,
         "all": np.ones(len(P), bool)}
p = P[masks[sys.argv[1]]]
ctx = _native.Context(0)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    b = SearchBatch(L, S, E, p, ctx); b.run(); t = b.timing(); b.close()
    print(f"{len(p)} searches: device {t['total_ms']:.3f} dp {t['dp_ms']:.3f} sweep {t['sweep_ms']:.3f} launches {t['n_launches']}")
