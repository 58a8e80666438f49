"""K2 timeline of the GPT-3-96 P=1 stage searches alone (the 10k sweep's deepest problems):
python tools/deep_probe.py  (run with GBMW_K2_HIST=1)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2307_02031_b200 import workloads as W, _native
from paper_2307_02031_b200.dpsearch import SearchBatch
cells = [c for c in W.sweep_cells(10000) if c.model == "gpt" and c.pp_degree == 1]
L, S, E, P, T = W.sweep_arrays(cells)
ctx = _native.Context(0)
for i in range(3):
    b = SearchBatch(L, S, E, P, ctx); b.run(); t = b.timing(); b.close()
    print(f"{len(P)} GPT P=1 searches: device {t['total_ms']:.2f} ms dp {t['dp_ms']:.2f} ms", flush=True)
