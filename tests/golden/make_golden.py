"""Generate the golden fixtures of the search path from the LIVE reference.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports parapilot read-only from /root/reference/pkg/src (and the reference
test helpers from /root/reference/pkg/tests for the fuzz instances), evaluates
the reference functions on fixed inputs, and writes small JSON fixtures next to
this script.  fp64 outputs are stored as float.hex() so parity is bit-exact.
The fixtures are the contract the oracle (oracle/ref_oracle.c) and the CUDA
path are both checked against (tests/test_golden_oracle.py, tests/test_gpu_parity.py).
"""

from __future__ import annotations

import hashlib
import json
import random
import struct
import sys
import time
from pathlib import Path

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import parapilot as R                                     # noqa: E402
from parapilot import costs as RC                         # noqa: E402
from parapilot import dpsearch as RD                      # noqa: E402
from parapilot.strategies import candidate_pp_degrees    # noqa: E402
import helpers as RH                                      # noqa: E402  (reference test helpers)

from paper_2307_02031_b200 import workloads as W          # noqa: E402  (fixed synthetic specs only)

OUT = Path(__file__).resolve().parent
MiB = 1 << 20
GiB = 1 << 30


def hx(x) -> str:
    return float(x).hex()


def frontier_digest(frontier) -> str:
    h = hashlib.sha256()
    for _, t in frontier:
        h.update(struct.pack("<d", t))
    return h.hexdigest()


def layer_doc(l):
    return [l.id, l.kind, l.param_bytes, l.bnd_bytes_per_sample, l.int_bytes_per_sample,
            hx(l.fwd_time_per_sample), hx(l.tp_act_replication_fraction)]


def env_doc(ctx):
    c, p = ctx.cluster, ctx.profile
    return {"n_devices": c.n_devices, "island_size": c.island_size, "intra": hx(c.intra_island_bw),
            "inter": hx(c.inter_island_bw), "slowdown": hx(c.overlap_slowdown),
            "bwd_ratio": hx(p.bwd_fwd_ratio), "coll_eff": hx(p.collective_efficiency),
            "ms": hx(ctx.model.ms_bytes_per_param_byte),
            "overrides": {str(k): hx(v) for k, v in p.layer_overrides.items()}}


def dp_case(name, layers, budget, sset, micro, gran, ctx, stage=1, n_micro=1, fuse=False, frontier=False,
            approx=False):
    strats = list(sset)
    t0 = time.time()
    res = RD.dp_search(list(layers), budget, sset, micro, gran, ctx, stage_index=stage, n_micro=n_micro,
                       fuse_identical=fuse, approx_prev=approx, collect_frontier=frontier)
    dt = time.time() - t0
    out = {"feasible": res.feasible, "time": hx(res.time_s), "e_fwd": hx(res.e_fwd_used)}
    if res.feasible:
        out["plan"] = [strats.index(s) for s in res.strategies]
        sc = RC.stage_cost(list(layers), list(res.strategies), micro, ctx, stage_index=stage, n_micro=n_micro)
        out["stage"] = [hx(sc.time_s), hx(sc.time_no_sync_s), hx(sc.peak_mem_bytes)]
    if frontier and res.frontier is not None:
        out["frontier_digest"] = frontier_digest(res.frontier)
        out["frontier_len"] = len(res.frontier)
        if len(res.frontier) <= 512:
            out["frontier"] = [hx(t) for _, t in res.frontier]
    return {"name": name, "layers": [layer_doc(l) for l in layers], "budget": budget,
            "budget_is_int": isinstance(budget, int), "strategies": [s.to_string() for s in strats],
            "micro": micro, "gran": gran, "stage": stage, "n_micro": n_micro, "fuse": fuse,
            "collect_frontier": frontier, "approx": approx, "env": env_doc(ctx), "out": out,
            "ref_seconds": round(dt, 4)}


def gen_enumeration():
    doc = {}
    for n in [1 << k for k in range(11)]:
        for p in candidate_pp_degrees(n):
            raw = R.enumerate_strategies(n, p)
            doc[f"{n},{p},raw"] = [s.to_string() for s in raw]
            doc[f"{n},{p},pruned"] = [s.to_string() for s in R.prune_dp_sdp(raw)]
    return doc


def gen_cells(n=600, seed=7):
    rng = random.Random(seed)
    cells = []
    for _ in range(n):
        N = 1 << rng.randint(0, 7)
        P = 1 << rng.randint(0, N.bit_length() - 1)
        ss = R.enumerate_strategies(N, P).strategies
        s = rng.choice(ss)
        prev = rng.choice(ss)
        micro = s.data_degree * rng.choice([1, 2, 3, 5, 8])
        layer = R.LayerSpec(rng.randint(0, 3), "x", rng.randint(1, 10 ** 10), rng.randint(1, 10 ** 8),
                            rng.randint(0, 10 ** 9), rng.uniform(1e-4, 1e-1), rng.choice([0.0, 0.25, 0.3, 1.0]))
        island = 1 << rng.randint(0, N.bit_length() - 1)
        inter = rng.uniform(1e8, 1e10)
        cl = R.ClusterSpec(N, 64 * GiB, island, inter * rng.uniform(1, 30), inter, rng.choice([1.0, 1.3, 1.7]))
        pr = R.CostProfile(rng.uniform(1, 3), rng.uniform(0.3, 1.0))
        ms = rng.uniform(1, 8)
        stage, m = rng.randint(1, P), rng.randint(1, 16)
        ctx = R.EvalContext(R.ModelSpec("m", (layer,), ms), cl, pr)
        t, tns = RC._layer_times(layer, s, micro, cl, pr)
        o_f, o_b, o_ms = R.layer_memory(layer, s, micro, stage, m, ms)
        g, a = R.comm_time(layer, s, micro, cl, pr)
        cells.append({"layer": layer_doc(layer), "strategy": s.to_string(), "prev": prev.to_string(),
                      "micro": micro, "stage": stage, "n_micro": m, "env": env_doc(ctx),
                      "out": [hx(t), hx(tns), hx(o_f), hx(o_b), hx(o_ms),
                              hx(R.transform_cost(layer, prev, s, micro, cl)), hx(g), hx(a)],
                      "o_f_is_int": isinstance(o_f, int)})
    return cells


def gen_fuzz():
    cases = []
    for seed, count, gran, fuse in ((20240813, 60, 1, False), (99, 40, 64, False), (3, 30, 1, False),
                                    (5, 20, 1, True), (6, 20, 1, False), (11, 40, 4, True), (12, 40, 16, False)):
        rng = random.Random(seed)
        for k in range(count):
            model, cluster, ctx, sset, micro = RH.fuzz_dp_instance(rng)
            cases.append(dp_case(f"fuzz{seed}_{k}", model.layers, cluster.mem_budget_bytes, sset, micro, gran,
                                 ctx, fuse=fuse, frontier=(k % 3 == 0)))
    # the reference test's small_context family (test_dpsearch.py:37-41)
    for nl, budget, gran in ((3, 4096, 1), (3, 8192, 16), (4, 16384, 1), (4, 1 << 19, 1), (3, 512, 1),
                             (3, 1024, 1), (3, 2048, 1)):
        model = RH.uniform_model(nl, param=64, bnd=16, intb=96, fwd=0.01)
        ctx = RH.make_ctx(model, RH.make_cluster(n=4, budget=budget, intra=1e6))
        sset = R.prune_dp_sdp(R.enumerate_strategies(4, 1))
        for fuse in (False, True):
            cases.append(dp_case(f"small{nl}_{budget}_{gran}_{fuse}", model.layers, budget, sset, 8, gran, ctx,
                                 fuse=fuse, frontier=True))
    return cases


def gen_configs():
    """Realistic stages of the benchmark models (even partitions), mostly at the
    reference's default 64 MiB granularity, a few at 16 / 4 / 1 MiB."""
    cases = []
    plan = [
        ("bert", [16 * GiB], [64 * MiB, 16 * MiB]),
        ("t5", [8 * GiB, 12 * GiB, 16 * GiB, 20 * GiB], [64 * MiB]),
        ("vit", [16 * GiB], [64 * MiB, 16 * MiB]),
        ("swin", [16 * GiB], [64 * MiB]),
        ("gpt", [80 * GiB], [1 * GiB, 256 * MiB]),
    ]
    rng = random.Random(2026)
    for name, budgets, grans in plan:
        for budget in budgets:
            ctx0 = W.config(name, budget)
            ctx = R.EvalContext(R.ModelSpec(ctx0.model.name, tuple(
                R.LayerSpec(l.id, l.kind, l.param_bytes, l.bnd_bytes_per_sample, l.int_bytes_per_sample,
                            l.fwd_time_per_sample, l.tp_act_replication_fraction) for l in ctx0.model.layers),
                ctx0.model.ms_bytes_per_param_byte),
                R.ClusterSpec(**ctx0.cluster.to_document()), R.CostProfile())
            L = ctx.model.num_layers
            N = ctx.cluster.n_devices
            for gran in grans:
                for P in [p for p in candidate_pp_degrees(N) if p <= L]:
                    for B in rng.sample([8, 16, 32, 64, 128, 256, 512], 2):
                        m = W.microbatch_num(B, P)
                        micro = B // m
                        sset = R.prune_dp_sdp(R.enumerate_strategies(N, P))
                        parts = W.even_partition(L, P)
                        stages = sorted({0, P - 1, rng.randrange(P)})
                        for si in stages:
                            a = sum(parts[:si])
                            layers = ctx.model.layers[a:a + parts[si]]
                            fuse = rng.random() < 0.3
                            cases.append(dp_case(f"{name}_b{budget // GiB}_g{gran // MiB}_P{P}_B{B}_s{si + 1}",
                                                 layers, budget, sset, micro, gran, ctx, stage=si + 1, n_micro=m,
                                                 fuse=fuse, frontier=(si == 0)))
    # a few 1 MiB / 4 MiB stages (the reference needs seconds each)
    for name, budget, P, B, si, gran in (("bert", 16 * GiB, 1, 8, 0, MiB), ("bert", 16 * GiB, 2, 64, 1, 4 * MiB),
                                         ("t5", 8 * GiB, 4, 32, 2, MiB), ("vit", 16 * GiB, 8, 128, 3, 4 * MiB),
                                         ("swin", 16 * GiB, 2, 16, 0, 4 * MiB), ("gpt", 80 * GiB, 16, 1024, 5, MiB),
                                         ("gpt", 80 * GiB, 32, 512, 0, MiB)):
        ctx0 = W.config(name, budget)
        ctx = R.EvalContext(R.ModelSpec(ctx0.model.name, tuple(
            R.LayerSpec(l.id, l.kind, l.param_bytes, l.bnd_bytes_per_sample, l.int_bytes_per_sample,
                        l.fwd_time_per_sample, l.tp_act_replication_fraction) for l in ctx0.model.layers),
            ctx0.model.ms_bytes_per_param_byte), R.ClusterSpec(**ctx0.cluster.to_document()), R.CostProfile())
        N, L = ctx.cluster.n_devices, ctx.model.num_layers
        m = W.microbatch_num(B, P)
        parts = W.even_partition(L, P)
        a = sum(parts[:si])
        cases.append(dp_case(f"{name}_fine_g{gran // MiB}_P{P}_B{B}_s{si + 1}", ctx.model.layers[a:a + parts[si]],
                             budget, R.prune_dp_sdp(R.enumerate_strategies(N, P)), B // m, gran, ctx,
                             stage=si + 1, n_micro=m, frontier=True))
    # profile overrides (fuse key uses raw fwd time: dpsearch.py:75-77 quirk)
    model = RH.uniform_model(6, param=100_000_000, bnd=10_000_000, intb=100_000_000, fwd=0.01)
    prof = R.CostProfile(bwd_fwd_ratio=2.5, collective_efficiency=0.8, layer_overrides={0: 0.02, 3: 0.005})
    cl = RH.make_cluster(n=8, budget=6 * GiB, island=4, intra=12e9, inter=6e9)
    ctx = R.EvalContext(model, cl, prof)
    for P in (1, 2):
        sset = R.prune_dp_sdp(R.enumerate_strategies(8, P))
        for fuse in (False, True):
            for gran in (16 * MiB, 4 * MiB):
                cases.append(dp_case(f"override_P{P}_{fuse}_{gran // MiB}", model.layers, cl.mem_budget_bytes,
                                     sset, 8, gran, ctx, stage=1, n_micro=2 * P, fuse=fuse, frontier=True))
    return cases


def gen_approx():
    """approx_prev=True (collapsed-state DP, dpsearch.py:306-375) on the fuzz family, the
    small_context family and a few benchmark-model stages."""
    cases = []
    for seed, count, gran, fuse in ((31, 60, 1, False), (32, 40, 8, True), (33, 40, 1, False)):
        rng = random.Random(seed)
        for k in range(count):
            model, cluster, ctx, sset, micro = RH.fuzz_dp_instance(rng)
            cases.append(dp_case(f"approx{seed}_{k}", model.layers, cluster.mem_budget_bytes, sset, micro, gran,
                                 ctx, fuse=fuse, frontier=(k % 2 == 0), approx=True))
    for nl, budget, gran in ((3, 4096, 1), (4, 16384, 1), (3, 1024, 1), (4, 1 << 19, 1)):
        model = RH.uniform_model(nl, param=64, bnd=16, intb=96, fwd=0.01)
        ctx = RH.make_ctx(model, RH.make_cluster(n=4, budget=budget, intra=1e6))
        sset = R.prune_dp_sdp(R.enumerate_strategies(4, 1))
        for fuse in (False, True):
            cases.append(dp_case(f"approx_small{nl}_{budget}_{fuse}", model.layers, budget, sset, 8, gran, ctx,
                                 fuse=fuse, frontier=True, approx=True))
    rng = random.Random(77)
    for name, budget, gran in (("bert", 16 * GiB, 64 * MiB), ("t5", 8 * GiB, 16 * MiB), ("vit", 16 * GiB, 64 * MiB),
                               ("swin", 16 * GiB, 64 * MiB), ("gpt", 80 * GiB, 256 * MiB)):
        ctx0 = W.config(name, budget)
        ctx = R.EvalContext(R.ModelSpec(ctx0.model.name, tuple(
            R.LayerSpec(l.id, l.kind, l.param_bytes, l.bnd_bytes_per_sample, l.int_bytes_per_sample,
                        l.fwd_time_per_sample, l.tp_act_replication_fraction) for l in ctx0.model.layers),
            ctx0.model.ms_bytes_per_param_byte), R.ClusterSpec(**ctx0.cluster.to_document()), R.CostProfile())
        N, L = ctx.cluster.n_devices, ctx.model.num_layers
        for P in [p for p in candidate_pp_degrees(N) if p <= L][:4]:
            B = rng.choice([8, 32, 128])
            m = W.microbatch_num(B, P)
            parts = W.even_partition(L, P)
            si = rng.randrange(P)
            a = sum(parts[:si])
            cases.append(dp_case(f"approx_{name}_P{P}_B{B}_s{si + 1}", ctx.model.layers[a:a + parts[si]], budget,
                                 R.prune_dp_sdp(R.enumerate_strategies(N, P)), B // m, gran, ctx, stage=si + 1,
                                 n_micro=m, fuse=rng.random() < 0.5, frontier=True, approx=True))
    return cases


def main():
    t0 = time.time()
    if sys.argv[1:] == ["approx"]:
        cases = gen_approx()
        (OUT / "dp_approx.json").write_text(json.dumps(cases, separators=(",", ":")))
        print(f"approx: {len(cases)} cases, {time.time() - t0:.1f}s")
        return
    (OUT / "enumeration.json").write_text(json.dumps(gen_enumeration(), separators=(",", ":")))
    (OUT / "cost_cells.json").write_text(json.dumps(gen_cells(), separators=(",", ":")))
    print(f"enumeration + cells: {time.time() - t0:.1f}s")
    fuzz = gen_fuzz()
    (OUT / "dp_fuzz.json").write_text(json.dumps(fuzz, separators=(",", ":")))
    print(f"fuzz: {len(fuzz)} cases, {time.time() - t0:.1f}s")
    cfg = gen_configs()
    (OUT / "dp_configs.json").write_text(json.dumps(cfg, separators=(",", ":")))
    print(f"configs: {len(cfg)} cases, {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
