"""Host-side e2e breakdown of the benchmark batch (create / run / fetch / close and the
native create phases).  usage (on a GPU box): GBMW_K2_HIST=1 python tools/e2e_probe.py"""
import sys, time
sys.path.insert(0, '.')
from paper_2307_02031_b200 import workloads as W, _native
from paper_2307_02031_b200.dpsearch import run_native_batch, SearchBatch
L, S, E, P, T = W.sweep_arrays(W.sweep_cells(10000))
ctx = _native.Context(0)
for i in range(4):
    t0 = time.perf_counter(); b = SearchBatch(L, S, E, P, ctx); t1 = time.perf_counter(); b.run(); t2 = time.perf_counter()
    b.fetch(); t3 = time.perf_counter(); tb = b.timing(); b.close(); t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} (prep {tb['prep_ms']:.2f} upload {tb['upload_ms']:.2f}) run {1e3*(t2-t1):.2f} "
          f"fetch {1e3*(t3-t2):.2f} close {1e3*(t4-t3):.2f}", flush=True)
for i in range(5):
    t0 = time.perf_counter(); r = run_native_batch(L, S, E, P, ctx); t1 = time.perf_counter()
    print(f"run_native_batch {1e3*(t1-t0):.2f}", flush=True)
