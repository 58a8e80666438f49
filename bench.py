#!/usr/bin/env python
"""Benchmark of the Galvatron-BMW search hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1, one rank per GPU)

Workload (BASELINE.json config 5): the batched sweep of 10,000
independent stage searches (BERT-Huge-32 / T5-Large-48 / ViT-Huge-32 / Swin-Huge-48
on 8 simulated GPUs at 8-20 GiB, GPT-3-96 on 64 simulated GPUs at 80 GiB; even
partitions; 1 MiB memory granularity), sharded across ranks by estimated cost
(strong scaling: total work fixed), one NCCL all-gather selecting the global argmin.

One step = one device pass over the rank's shard (K1 tables, K2 layer steps, K3
sweep, K4 backtrack + stage cost) with inputs resident in HBM; ``value`` is
algorithmic DP transitions ((U-1) * n_e * S^2 per search) per
second of device time (CUDA events on the library's stream), max over ranks.
``e2e`` times the public C-ABI call (gbmw_search_batch via dpsearch.run_native_batch)
from host buffers, uploads and result download included, plus the NCCL argmin.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MiB = 1 << 20
METRIC = "DP transitions/sec and full-search latency at 1/2/4/8 B200 vs CPU ref"
UNIT = "transitions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--searches", type=int, default=10_000)
    ap.add_argument("--granularity", type=int, default=MiB)
    ap.add_argument("--e2e-steps", type=int, default=0, help="timed e2e calls (0: --steps)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="one device pass only (for ncu launch lists)")
    ap.add_argument("--workload", default="sweep10k",
                    help="sweep10k (default, BASELINE config 5) or a full planner search: "
                         "gpt96[-bmw] | bert[-bmw] | t5-<GiB>[-bmw] | vit[-bmw] | swin[-bmw]")
    return ap.parse_args()


def workload(args):
    from paper_2307_02031_b200 import workloads as W
    cells = W.sweep_cells(args.searches)
    L, S, E, P, T = W.sweep_arrays(cells, granularity_bytes=args.granularity)
    return L, S, E, P, T


def describe(args, n_problems):
    return {"workload": f"sweep10k: {n_problems} independent stage searches (BERT-Huge-32, T5-Large-48, "
                        f"ViT-Huge-32, Swin-Huge-48 on 8 GPUs at 8-20 GiB; GPT-3-96 on 64 GPUs at 80 GiB), "
                        f"even partitions, random (P, B) from seed 20261017",
            "granularity_bytes": args.granularity, "n_searches": n_problems,
            "l2": "state (class frontiers + argmin tables, tens of GB) exceeds L2; L2 also flushed "
                  "(256 MiB write) before every timed step",
            "parallelism": "search-sharded"}


def shard(T, rank, world):
    from paper_2307_02031_b200.distributed import shard_lpt
    return shard_lpt(T, world, rank)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def algorithmic_bytes(P, T):
    """SURVEY.md §8(d) regime B: 33/S HBM bytes per algorithmic transition (the uint8
    argmin per (e, j) cell plus reading T, F and writing T', F' in fp64), summed over the
    searches: 33 * T / S with S recovered from T = (U - 1) * n_e * S^2."""
    units = P["n_layers"].astype(np.float64) - 1.0
    rows = P["n_buckets"].astype(np.float64) + 1.0
    ok = (units > 0) & (T > 0)
    S = np.zeros_like(T)
    S[ok] = np.rint(np.sqrt(T[ok] / (units[ok] * rows[ok])))
    return float(np.sum(np.where(ok & (S > 0), 33.0 * T / np.maximum(S, 1.0), 0.0)))


def k2_traffic():
    """dram bytes per K2 launch from the committed ncu --set full capture, if any."""
    f = ROOT / "profiles" / "k2_traffic.json"
    if f.exists():
        try:
            return json.loads(f.read_text())
        except ValueError:
            return None
    return None


def cpu_sample(L, S, E, P, T, seconds, threads):
    """Bounded sample of the workload for the oracle: a deterministic spread of
    problems whose estimated single-core time sums to ~seconds * threads."""
    rng = np.random.default_rng(20261017)
    order = rng.permutation(len(P))
    budget = seconds * threads * 1.25e8         # ~1.25e8 transitions/s per core (oracle on the GPU box, measured)
    pick, acc = [], 0.0
    for i in order:
        if T[i] > budget * 0.25:                 # skip single searches larger than a quarter sample
            continue
        pick.append(i)
        acc += T[i] + 1e5
        if acc >= budget:
            break
    return np.array(sorted(pick))


def run_cpu(L, S, E, P, T, idx, threads):
    from oracle import oracle as O
    t0 = time.perf_counter()
    res, _, _, used = O.search_many(L, S, E, P[idx].copy(), threads)
    dt = time.perf_counter() - t0
    return float(T[idx].sum()) / dt, dt, used, res


def impl_reference(args, rank, world):
    if rank != 0:
        return 0
    L, S, E, P, T = workload(args)
    threads = len(os.sched_getaffinity(0))
    per_step = min(15.0, max(2.0, 150.0 / max(1, args.steps + args.warmup)))
    idx = cpu_sample(L, S, E, P, T, per_step, threads)
    for _ in range(args.warmup):
        run_cpu(L, S, E, P, T, idx, threads)
    vals, secs = [], []
    used = threads
    for _ in range(args.steps):
        v, dt, used, _ = run_cpu(L, S, E, P, T, idx, threads)
        vals.append(v)
        secs.append(dt)
    value = float(sum(T[idx]) * args.steps / sum(secs))
    sample = (f"{len(idx)} of {len(P)} stage searches ({T[idx].sum():.3e} of {T.sum():.3e} transitions), "
              f"oracle/ref_oracle.c (C restatement of parapilot dp_search, OpenMP over searches)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": describe(args, len(P)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "port", "sample": sample,
                             "cpu": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def full_search(args, rank):
    """One full planner search (Algorithm 1, optionally + Algorithm 2) at the given
    granularity: wall-clock latency of plan_full and the algorithmic transitions of
    every stage search it issued (SURVEY.md §8(d) full-search latency)."""
    if rank != 0:
        return 0
    import torch
    from paper_2307_02031_b200 import dpsearch, workloads as W
    from paper_2307_02031_b200.planner import PlannerOptions, plan_full

    name = args.workload
    bmw = name.endswith("-bmw")
    base = name[:-4] if bmw else name
    budget = None
    if base.startswith("t5-"):
        budget = int(base.split("-")[1]) << 30
        base = "t5"
    if base == "gpt96":
        base = "gpt"
    ctx = W.config(base, budget)
    opts = PlannerOptions(granularity_bytes=args.granularity, bi_objective=bmw)
    torch.cuda.set_device(0)
    lat = []
    plan = None
    for k in range(max(1, args.warmup) + args.steps):
        dpsearch.reset_stats()
        t0 = time.perf_counter()
        plan = plan_full(ctx.model, ctx.cluster, ctx.profile, opts)
        dt = time.perf_counter() - t0
        if k >= max(1, args.warmup):
            lat.append(dt)
    st = dict(dpsearch.STATS)
    ms = 1e3 * float(np.median(lat))
    line = {"metric": METRIC, "value": st["transitions"] / (ms / 1e3), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": max(1, args.warmup), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "none", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"plan_full {name}: {ctx.model.name} on {ctx.cluster.n_devices} simulated GPUs, "
                                   f"{ctx.cluster.mem_budget_bytes >> 30} GiB, granularity {args.granularity} B"
                                   + (", BMW bi-objective refinement" if bmw else "")},
            "full_search_latency_ms": ms, "stage_searches": st["problems"], "device_batches": st["batches"],
            "device_ms": st["total_ms"], "transitions": st["transitions"],
            "plan": {"batch_size": plan.batch_size, "pp_degree": plan.pp_degree, "partition": list(plan.partition),
                     "n_micro": plan.n_micro, "predicted_time_s": plan.predicted_time_s,
                     "predicted_throughput": plan.predicted_throughput}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload != "sweep10k":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "full-search workloads are GPU-only; the CPU "
                                                                  "reference arm times the sweep10k workload"}))
            return 0
        return full_search(args, rank)
    if args.impl == "reference":
        return impl_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2307_02031_b200 import _native
    from paper_2307_02031_b200.distributed import global_winner
    from paper_2307_02031_b200.dpsearch import SearchBatch, run_native_batch

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    L, S, E, P, T = workload(args)
    mine = shard(T, rank, world)
    Pm = P[mine].copy()
    Tm = T[mine]
    ctx = _native.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", local))
    flush = torch.empty(256 * MiB // 4, dtype=torch.int32, device="cuda")

    batch = SearchBatch(L, S, E, Pm, ctx)
    if args.profile:
        batch.run()
        t = batch.timing()
        print(json.dumps({"profile_pass": True, "device_ms": t["total_ms"], "launches": t["n_launches"]}))
        batch.close()
        ctx.close()
        return 0
    for _ in range(max(args.warmup, 3)):
        batch.run()
    # timed region: K device passes, barrier + synchronize on both sides
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    dev_ms, dp_ms, sweep_ms, launches = [], [], [], 0
    wall0 = time.perf_counter()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(k)                      # L2 flush on the library's stream, outside the events
        batch.run()
        t = batch.timing()
        dev_ms.append(t["total_ms"])
        dp_ms.append(t["dp_ms"])
        sweep_ms.append(t["sweep_ms"])
        launches += int(t["n_launches"])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    timing = batch.timing()
    res, plans, _ = batch.fetch()
    batch.close()

    my_ms = float(np.mean(dev_ms))
    stats = torch.tensor([my_ms, float(np.mean(dp_ms)), wall * 1e3 / args.steps, float(Tm.sum()),
                          timing["dp_bytes"], float(launches)], dtype=torch.float64, device="cuda")
    if world > 1:
        gathered = [torch.zeros_like(stats) for _ in range(world)]
        dist.all_gather(gathered, stats)
        allst = torch.stack(gathered).cpu().numpy()
    else:
        allst = stats.cpu().numpy()[None, :]
    step_ms = float(allst[:, 0].max())
    total_T = float(allst[:, 3].sum())
    value = total_T / (step_ms / 1e3)

    # ---- e2e: public C-ABI call from host buffers (+ NCCL argmin), per step
    e2e_ms, call_ms, h2d, d2h = [], [], 0, 0
    winner = None
    n_e2e = args.e2e_steps if args.e2e_steps > 0 else args.steps
    for k in range(1 + n_e2e):                      # call 0: untimed warm-up of the host path
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc, msg, r, pl, _ = run_native_batch(L, S, E, Pm, ctx)
        assert rc == 0, msg
        t1 = time.perf_counter()
        # global argmin over feasible searches (min time, then lowest search index): one NCCL all-gather
        best = global_winner(r["time_s"], r["feasible"], mine, device="cuda")
        torch.cuda.synchronize()
        if k > 0:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
            call_ms.append((t1 - t0) * 1e3)
        winner = best
        h2d = int(L.nbytes + S.nbytes + E.nbytes + Pm.nbytes)
        d2h = int(r.nbytes + 4 * int(Pm["n_layers"].sum()))
    # mean over the timed calls (as the device-timed value), max over ranks
    e2e_t = torch.tensor([float(np.mean(e2e_ms)) if e2e_ms else float("nan")], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_step_ms = float(e2e_t.item())
    # where the e2e time goes (one extra, untimed, instrumented pass)
    t0 = time.perf_counter()
    b2 = SearchBatch(L, S, E, Pm, ctx)
    t1 = time.perf_counter()
    b2.run()
    t2 = time.perf_counter()
    b2.fetch()
    t3 = time.perf_counter()
    tb = b2.timing()
    b2.close()
    t4 = time.perf_counter()
    breakdown = {"create_ms": (t1 - t0) * 1e3, "host_prep_ms": tb["prep_ms"], "upload_ms": tb["upload_ms"],
                 "run_ms": (t2 - t1) * 1e3, "device_ms": tb["total_ms"], "fetch_ms": (t3 - t2) * 1e3,
                 "destroy_ms": (t4 - t3) * 1e3,
                 "search_call_ms_mean": float(np.mean(call_ms)) if call_ms else None,
                 "winner_ms_mean": float(np.mean(np.array(e2e_ms) - np.array(call_ms))) if call_ms else None}

    if rank == 0:
        hbm, kind = peaks()
        dp_time = float(allst[0, 1]) / 1e3
        # K2 roofline per SURVEY.md §8(d): algorithmic bytes of the reference's min-plus
        # recurrence (33/S B per transition) over K2 device time; the exact reformulations
        # (class reduction, breakpoint-only evaluation) move far fewer bytes,
        # so frac > 1 means the kernel beats the reference formulation's HBM roofline.
        alg = algorithmic_bytes(Pm, Tm)
        achieved = alg / dp_time / 1e9 if dp_time > 0 else 0.0
        tr = k2_traffic()
        n_k2 = int((tr or {}).get("launches") or 190)
        dram = (tr or {}).get("k2_dram_bytes_per_step")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": describe(args, len(P)),
            "full_search_latency_ms": step_ms,
            "wall_ms_per_step": float(allst[:, 2].max()),
            "phase_ms": {"dp_k2": float(np.mean(dp_ms)), "sweep_k3": float(np.mean(sweep_ms)),
                         "total": my_ms},
            "roofline": {"kernel": "K2: k_dp_classify + k_dp_rounds, k_dp_tile (few-tile steps), k_dp_first, k_dp_second", "bound": "hbm", "achieved": achieved, "peak": hbm,
                         "peak_kind": kind, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": (tr or {}).get("bytes_per_launch") if tr else None,
                         "algorithmic_bytes_per_launch": alg / n_k2,
                         "model": "SURVEY.md §8(d) regime B: 33/S bytes per algorithmic transition; "
                                  "frac > 1: the exact reformulation reads/writes fewer bytes than the "
                                  "reference recurrence needs (DESIGN.md §4)",
                         "measured_dram_GBs": (dram / dp_time / 1e9) if dram and dp_time > 0 else None,
                         "measured_dram_frac": (dram / dp_time / 1e9 / hbm) if dram and dp_time > 0 else None},
            "sweep_work": {k: timing[k] for k in ("sweep_rows", "sweep_cands", "sweep_checks")},
            "dp_work": {"live_cells": timing["live_cells"], "computed_cells": timing["dp_cells"]},
            "gpu_launches": int(allst[:, 5].sum()),
            "clocks": clk,
            "e2e": {"value": total_T / (e2e_step_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_step_ms,
                    "calls_ms_rank0": [round(x, 3) for x in e2e_ms],
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "dpsearch.run_native_batch -> gbmw_search_batch (host arrays) + NCCL argmin",
                    "breakdown_rank0": breakdown},
            "winner": {"time_s": winner[0], "search": winner[1]} if winner else None,
            "transitions_per_step": total_T,
        }
        if world == 1 and not args.no_cpu_baseline:
            threads = len(os.sched_getaffinity(0))
            idx = cpu_sample(L, S, E, P, T, args.cpu_seconds, threads)
            v, dt, used, ores = run_cpu(L, S, E, P, T, idx, threads)
            # the sample's results must agree with the device results for the same searches
            pos = {int(g): i for i, g in enumerate(mine)}
            agree = all(np.float64(ores["time_s"][a]).view(np.int64) == np.float64(res["time_s"][pos[int(g)]]).view(np.int64)
                        for a, g in enumerate(idx))
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": used, "kind": "port",
                                    "sample": f"{len(idx)} of {len(P)} searches ({T[idx].sum():.3e} transitions) "
                                              f"in {dt:.1f} s, oracle/ref_oracle.c", "cpu": _cpu_model(),
                                    "agrees_with_gpu": bool(agree)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
