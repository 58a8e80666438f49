"""Save the k-th device batch of a full planner search, or replay a saved one (GPU box).
    python tools/replay_batch.py save swin-bmw K out.npz
    python tools/replay_batch.py run out.npz [reps]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2307_02031_b200 import dpsearch, workloads as W, _native

if sys.argv[1] == "save":
    name, k, out = sys.argv[2], int(sys.argv[3]), sys.argv[4]
    from paper_2307_02031_b200.planner import PlannerOptions, plan_full
    seen = []
    orig = dpsearch.run_native_batch
    def grab(layers, strats, envs, probs, context=None):
        seen.append((layers.copy(), strats.copy(), envs.copy(), probs.copy()))
        return orig(layers, strats, envs, probs, context)
    dpsearch.run_native_batch = grab
    bmw = name.endswith("-bmw"); base = name[:-4] if bmw else name
    ctx = W.config("gpt" if base == "gpt96" else base)
    plan_full(ctx.model, ctx.cluster, ctx.profile, PlannerOptions(granularity_bytes=1 << 20, bi_objective=bmw))
    L, S, E, P = seen[k]
    np.savez(out, L=L, S=S, E=E, P=P)
    print(f"saved batch {k} of {len(seen)}: {len(P)} problems, max layers {P['n_layers'].max()}")
else:
    d = np.load(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    ctx = _native.Context(0)
    for i in range(reps):
        rc, msg, res, plans, _ = dpsearch.run_native_batch(d["L"], d["S"], d["E"], d["P"], ctx)
        t = _native.Timing()
        _native.lib().gbmw_ctx_last_timing(ctx.handle, __import__('ctypes').byref(t))
        print(f"rc {rc} device {t.total_ms:.3f} ms dp {t.dp_ms:.3f} sweep {t.sweep_ms:.3f} launches {t.n_launches}")
