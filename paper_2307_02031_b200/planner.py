"""End-to-end planning drivers: Galvatron_Search, Galvatron-Base (Algorithm 1) and
plan_full with the BMW refinement (Algorithm 2).

Names, signatures, results and tie-breaks of parapilot/planner.py:52-341.  The
difference is batching: ``galvatron_search_batch`` sends every stage search of
many (batch, degree, partition) cells to the device in one pass, and
``galvatron_base`` evaluates a window of batch sizes speculatively and then
applies the reference's sequential stop rule to the results (T4,
planner.py:241-277), so the returned plan is the one the reference returns.
"""

from __future__ import annotations

import ctypes
import gc
import sys
import threading
from dataclasses import dataclass
from functools import lru_cache, wraps
from typing import Any, Sequence

import numpy as np

from . import dpsearch as _dps
from .balance import (
    BalanceReport,
    PipelinePartition,
    SearchOutcome,
    _seed_and_partition,
    balance_degrees,
    bi_objective_multi,
    bi_objective_optimize,
    init_partition_memory_balanced,
    StageLayers,
    partition_layers,
    seed_partitions,
)
from .costs import EvalContext, StageCost, layer_memory, pipeline_cost, stage_cost
from .dpsearch import StageProblem, dp_search_batch
from .errors import InfeasiblePlanError
from .specs import CostProfile
from .strategies import (
    ParallelStrategy,
    candidate_pp_degrees,
    enumerate_pruned,
    parse_strategy,
)

INF = float("inf")
DEFAULT_GRANULARITY_BYTES = 64 * 2 ** 20


@dataclass(frozen=True)
class PlannerOptions:
    batch_step: int = 8
    max_batch: int = 4096
    granularity_bytes: int = DEFAULT_GRANULARITY_BYTES
    microbatch_cap_factor: int = 4
    min_micro_size: int = 1
    bi_objective: bool = False
    batch_radius: int = 16
    fuse_identical: bool = False
    approx_prev: bool = False
    batch_window: int = 0           # batch sizes per device pass of galvatron_base (0: 16 for
                                    # large clusters / deep models, else 32)


@dataclass(frozen=True)
class Plan:
    pp_degree: int
    partition: tuple[int, ...]
    n_micro: int
    batch_size: int
    strategies: tuple[ParallelStrategy, ...]
    predicted_time_s: float
    predicted_throughput: float
    balance: BalanceReport
    peak_mem_per_stage: tuple[float, ...]

    def stage_layer_ids(self) -> list[list[int]]:
        out, a = [], 0
        for n in self.partition:
            out.append(list(range(a, a + n)))
            a += n
        return out

    def to_document(self, cluster=None) -> dict[str, Any]:
        stages = [{"layers": [{"id": lid, "strategy": self.strategies[lid].to_string(cluster)} for lid in ids]}
                  for ids in self.stage_layer_ids()]
        return {"pp_degree": self.pp_degree, "partition": list(self.partition), "n_micro": self.n_micro,
                "batch_size": self.batch_size, "stages": stages, "predicted_time_s": self.predicted_time_s,
                "predicted_throughput": self.predicted_throughput, "alpha_t": self.balance.alpha_t,
                "alpha_m": self.balance.alpha_m, "peak_mem_per_stage": list(self.peak_mem_per_stage)}


def init_microbatch_num(batch: int, pp_degree: int, cap_factor: int = 4, min_micro_size: int = 1) -> int:
    """Largest divisor of the batch within cap_factor * P (planner.py:110-125)."""
    if batch < 1:
        raise ValueError(f"batch must be >= 1, got {batch}")
    if pp_degree <= 1:
        return 1
    for m in range(min(cap_factor * pp_degree, batch), 0, -1):
        if batch % m == 0 and batch // m >= min_micro_size:
            return m
    return 1


@lru_cache(maxsize=512)
def _sset(n_devices: int, pp_degree: int):
    return enumerate_pruned(n_devices, pp_degree)


def _stage_ranges(model, stages):
    """(start, length) of each stage if the stages are consecutive slices of model.layers."""
    if isinstance(stages, StageLayers) and stages.model is model:
        return stages.ranges                    # from partition_layers(model, ...): immutable slices
    layers = model.layers
    index = _layer_index(model)
    out = []
    for st in stages:
        if not st:
            return None
        a = index.get(id(st[0]))
        if a is None or a + len(st) > len(layers) or any(layers[a + i] is not l for i, l in enumerate(st)):
            return None
        out.append((a, len(st)))
    return out


_index_cache: dict = {}


def _layer_index(model):
    hit = _index_cache.get(id(model))
    if hit is None or hit[0] is not model:
        if len(_index_cache) > 32:
            _index_cache.clear()
        hit = (model, {id(l): i for i, l in enumerate(model.layers)})
        _index_cache[id(model)] = hit
    return hit[1]


class FailedOutcome:
    """A cell whose search raised inside the native pass (a speculative window's cell): the
    exception is raised only if the reference's sequential order reaches the cell."""

    cost = INF

    def __init__(self, code: int, msg: str, n_micro: int):
        self.code, self.msg, self.n_micro = code, msg, n_micro

    def raise_(self):
        from . import _native
        _native.raise_status(self.code, self.msg)


@lru_cache(maxsize=4096)
def _cell_setup(n_devices: int, pp: int, batch: int, cap_factor: int, min_micro: int):
    """(n_micro, micro-batch, strategy set, any strategy usable) of a (N, P, B) cell."""
    m = init_microbatch_num(batch, pp, cap_factor, min_micro)
    micro = batch // m
    sset = _sset(n_devices, pp)
    return m, micro, sset, any(micro % s.data_degree == 0 for s in sset.strategies)


_layer_tables: dict = {}


def _model_layer_table(ctx):
    """LAYER_DT table of ctx.model's layers under ctx.profile, built once per EvalContext
    object (a planner driver runs many batches on one).  Model, cluster and profile are frozen
    dataclasses except the profile's override mapping, which is compared on every call, so a
    changed override is re-read as the reference re-reads it."""
    from . import _native
    prof = ctx.profile
    ov = getattr(prof, "layer_overrides", None)
    if not isinstance(prof, CostProfile) or not isinstance(ov, dict) or not isinstance(ctx.model.layers, tuple):
        return _native.layers_array(list(ctx.model.layers), prof, {})
    hit = _layer_tables.get(id(ctx))
    if hit is None or hit[0] is not ctx or hit[1] != ov:
        if len(_layer_tables) > 64:
            _layer_tables.clear()
        hit = (ctx, dict(ov), _native.layers_array(list(ctx.model.layers), prof, {}))
        _layer_tables[id(ctx)] = hit
    return hit[2]


class _SlicedBatch:
    """The flat problem table of a window of sliced cells (built by ``_slices_prepare``), its
    native results once run (``_slices_native``), turned into outcomes by ``_slices_finish``."""
    __slots__ = ("metas", "tables", "probs")

    def __init__(self, metas, tables, probs):
        self.metas, self.tables, self.probs = metas, tables, probs


def _slices_prepare(cells, ctx, opts) -> _SlicedBatch:
    from . import _native
    from .dpsearch import MAX_BUCKETS, _Marshal
    gran = opts.granularity_bytes
    mar = _Marshal()
    base = mar.layer_table(_model_layer_table(ctx))
    env = mar.env(ctx)
    flags = _native.STAGE_COST | (_native.FUSE if opts.fuse_identical else 0) | \
        (_native.APPROX if opts.approx_prev else 0)
    # per searched cell: its stages' (start, length) and the cell-level fields of its rows
    starts, lens, cell_rows, cell_vals = [], [], [], []
    metas = []
    n_rows = 0
    for budget, ranges, n_devices, batch, pp in cells:
        m, micro, sset, usable = _cell_setup(n_devices, pp, batch, opts.microbatch_cap_factor, opts.min_micro_size)
        strats = sset.strategies
        if gran <= 0:
            raise ValueError(f"granularity_bytes must be positive, got {gran}")
        if budget < 0:
            raise ValueError(f"budget_bytes must be non-negative, got {budget}")
        nb = int(budget // gran)
        if nb > MAX_BUCKETS:
            raise ValueError(f"budget/granularity yields {nb} buckets (> {MAX_BUCKETS}); "
                             f"increase the memory granularity")
        if nb == 0 or not usable:
            metas.append((m, None, None, strats))
            continue
        sb = mar.strat_range(sset, strats)
        k = len(ranges)
        for a, n in ranges:
            starts.append(a)
            lens.append(n)
        cell_rows.append(k)
        cell_vals.append((sb, len(strats), m, micro, float(budget), nb))
        metas.append((m, n_rows, n_rows + k, strats))
        n_rows += k
    if not n_rows:
        return _SlicedBatch(metas, None, None)
    layers, loffs, strats_arr, soffs, envs = mar.finish()
    probs = np.zeros(n_rows, dtype=_native.PROBLEM_DT)
    reps = np.asarray(cell_rows, dtype=np.int64)
    cv = list(zip(*cell_vals))
    probs["layer_begin"] = np.asarray(starts, dtype=np.int64) + (base + loffs[0])
    probs["n_layers"] = lens
    probs["strat_begin"] = np.repeat(np.asarray([soffs[x] for x in cv[0]], dtype=np.int64), reps)
    probs["n_strats"] = np.repeat(np.asarray(cv[1], dtype=np.int64), reps)
    probs["env_index"] = env
    # stage_index = 1 .. P within each cell
    first = np.repeat(np.cumsum(reps) - reps, reps)
    probs["stage_index"] = np.arange(n_rows, dtype=np.int64) - first + 1
    probs["n_micro"] = np.repeat(np.asarray(cv[2], dtype=np.int64), reps)
    probs["flags"] = flags
    probs["micro"] = np.repeat(np.asarray(cv[3], dtype=np.int64), reps)
    probs["gran"] = gran
    probs["budget"] = np.repeat(np.asarray(cv[4], dtype=np.float64), reps)
    probs["n_buckets"] = np.repeat(np.asarray(cv[5], dtype=np.int64), reps)
    return _SlicedBatch(metas, (layers, strats_arr, envs), probs)


def _slices_native(sb: _SlicedBatch):
    """The device pass of a prepared window (blocking; the ctypes call releases the GIL)."""
    from .dpsearch import run_native_batch
    if sb.tables is None:
        return None
    layers, strats_arr, envs = sb.tables
    return run_native_batch(layers, strats_arr, envs, sb.probs)


def _slices_finish(sb: _SlicedBatch, native, defer_errors=False):
    from . import _native
    out = []
    rc = _native.OK
    if native is not None:
        rc, msg, res, plans, _ = native
        if rc != _native.OK:
            bad = np.flatnonzero(res["status"] != 0)
            if not (defer_errors and len(bad)):
                _native.raise_status(int(res["status"][bad[0]]) if len(bad) else rc, msg)
            first_bad = int(bad[0])
        plan_off = np.concatenate(([0], np.cumsum(sb.probs["n_layers"]))).tolist()
        feas = res["feasible"].tolist()
        st_t, st_ns, st_pk = res["stage_time"].tolist(), res["stage_ns"].tolist(), res["stage_peak"].tolist()
        status = res["status"]
        plan_l = plans.tolist()
    for m, r0, r1, strats in sb.metas:
        if r0 is not None and rc != _native.OK:
            st = status[r0:r1]
            k = np.flatnonzero(st != 0)
            # the reference raises inside the first failing stage's dp_search, after the stages
            # before it were searched; a stage that is infeasible earlier ends the cell first
            if len(k) and all(feas[r0:r0 + int(k[0])]):
                code = int(st[k[0]])
                out.append(FailedOutcome(code, msg if r0 + int(k[0]) == first_bad else
                                         f"stage search failed (status {code})", m))
                continue
        if r0 is None or not all(feas[r0:r1]):                  # first infeasible stage (planner.py:159-160)
            out.append(SearchOutcome(cost=INF, strategies=None, stage_costs=None, n_micro=m))
            continue
        ts, ns = st_t[r0:r1], st_ns[r0:r1]
        costs = tuple(map(StageCost, ts, ns, st_pk[r0:r1]))
        idx = plan_l[plan_off[r0]:plan_off[r1]]
        # pipeline_cost (costs.py:355-362) on the same floats in the same order
        cost = (m - 1) * max(ns) + sum(ts)
        plan = tuple([strats[j] for j in idx])
        _dps.plan_records_register(plan, strats, idx)
        out.append(SearchOutcome(cost=cost, strategies=plan, stage_costs=costs, n_micro=m))
    return out


def _search_slices(cells, ctx, opts, defer_errors=False):
    """galvatron_search for cells whose stages are slices of ctx.model: one flat problem
    table over a single copy of the model's layers, no per-stage Python objects.  With
    ``defer_errors`` a cell whose stage search fails yields a ``FailedOutcome`` instead of
    raising for the whole batch."""
    sb = _slices_prepare(cells, ctx, opts)
    return _slices_finish(sb, _slices_native(sb), defer_errors)


def _sliced_cells(cells, ctx):
    """(budget, stage ranges, N, B, P) of every cell, or None if a stage is not a slice of
    ctx.model."""
    sliced = []
    for budget, stages, n_devices, batch, pp in cells:
        ranges = _stage_ranges(ctx.model, stages)
        if ranges is None:
            return None
        sliced.append((budget, ranges, n_devices, batch, pp))
    return sliced


def galvatron_search_batch(cells: Sequence[tuple], ctx: EvalContext, opts: PlannerOptions = PlannerOptions(),
                           defer_errors: bool = False):
    """Many ``galvatron_search(budget, stages, n_devices, batch, pp_degree)`` calls, one device pass.

    With ``defer_errors`` (the speculative drivers) a failing cell comes back as a
    ``FailedOutcome`` whose ``raise_()`` the caller invokes when its sequential order reaches
    it; otherwise the first failing cell raises for the whole batch."""
    sliced = _sliced_cells(cells, ctx)
    if sliced is not None:
        return _search_slices(sliced, ctx, opts, defer_errors)
    problems, spans, metas = [], [], []
    for budget, stages, n_devices, batch, pp in cells:
        m = init_microbatch_num(batch, pp, opts.microbatch_cap_factor, opts.min_micro_size)
        micro = batch // m
        sset = _sset(n_devices, pp)
        start = len(problems)
        for idx, layers in enumerate(stages, start=1):
            problems.append(StageProblem(layers, budget, sset, micro, opts.granularity_bytes, ctx, idx, m,
                                         opts.fuse_identical, opts.approx_prev))
        spans.append((start, len(problems)))
        metas.append(m)
    results, costs = dp_search_batch(problems, want_stage_cost=True) if problems else ([], [])
    out = []
    for (a, b), m in zip(spans, metas):
        strategies, stage_costs = [], []
        feasible = True
        for k in range(a, b):
            if not results[k].feasible:         # first infeasible stage ends the search (planner.py:159-160)
                feasible = False
                break
            strategies.extend(results[k].strategies)
            stage_costs.append(costs[k])
        if not feasible:
            out.append(SearchOutcome(cost=INF, strategies=None, stage_costs=None, n_micro=m))
        else:
            out.append(SearchOutcome(cost=pipeline_cost(stage_costs, m), strategies=tuple(strategies),
                                     stage_costs=tuple(stage_costs), n_micro=m))
    return out


def galvatron_search(budget_bytes: float, stages: list[list], n_devices: int, batch: int, pp_degree: int,
                     ctx: EvalContext, opts: PlannerOptions = PlannerOptions()) -> SearchOutcome:
    """Per-stage dynamic programming under one (batch, pipeline degree) cell (planner.py:128-172)."""
    return galvatron_search_batch([(budget_bytes, stages, n_devices, batch, pp_degree)], ctx, opts)[0]


class GalvatronSearch:
    """The ``SearchFn`` plan_full hands to Algorithm 2, with a batched form."""

    def __init__(self, ctx: EvalContext, opts: PlannerOptions):
        self.ctx, self.opts = ctx, opts

    def __call__(self, budget, stages, n_devices, batch, pp_degree) -> SearchOutcome:
        return galvatron_search(budget, stages, n_devices, batch, pp_degree, self.ctx, self.opts)

    def batch(self, calls) -> list[SearchOutcome]:
        return galvatron_search_batch(calls, self.ctx, self.opts)


def _assemble_plan(model, batch, pp_degree, partition, outcome) -> Plan:
    return Plan(pp_degree=pp_degree, partition=partition.stage_sizes, n_micro=outcome.n_micro, batch_size=batch,
                strategies=outcome.strategies, predicted_time_s=outcome.cost,
                predicted_throughput=batch / outcome.cost, balance=balance_degrees(outcome.stage_costs),
                peak_mem_per_stage=tuple(sc.peak_mem_bytes for sc in outcome.stage_costs))


def _infeasibility_diagnostics(model, ctx, batch, opts) -> dict:
    """Which constraint bound first at the smallest batch (planner.py:196-228)."""
    cluster = ctx.cluster
    diag: dict[str, Any] = {"batch_size": batch, "mem_budget_bytes": cluster.mem_budget_bytes}
    per_p = {}
    for p in candidate_pp_degrees(cluster.n_devices):
        if p > model.num_layers:
            per_p[p] = "more stages than layers"
            continue
        m = init_microbatch_num(batch, p, opts.microbatch_cap_factor, opts.min_micro_size)
        micro = batch // m
        usable = [s for s in _sset(cluster.n_devices, p) if micro % s.data_degree == 0]
        if not usable:
            per_p[p] = f"micro-batch {micro} indivisible by every strategy"
            continue
        min_states = min_total = INF
        for layer in model.layers:
            for s in usable:
                o_f, _, o_ms = layer_memory(layer, s, micro, p, m, ctx.ms_multiplier)
                min_states = min(min_states, o_ms)
                min_total = min(min_total, o_f + o_ms)
        if min_states > cluster.mem_budget_bytes:
            per_p[p] = "model states alone exceed the budget under every strategy"
        elif min_total > cluster.mem_budget_bytes:
            per_p[p] = "single-layer footprint exceeds the budget under every strategy"
        else:
            per_p[p] = "no per-layer assignment satisfies the backward-peak budget"
    diag["per_pp_degree"] = per_p
    return diag


_pool = None


def _executor():
    """Host threads for the native seed partitions (the ctypes calls release the GIL)."""
    global _pool
    if _pool is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        _pool = ThreadPoolExecutor(max_workers=max(1, min(32, len(os.sched_getaffinity(0)))))
    return _pool


def _base_cells_window(model, ctx, batches, opts):
    """Per batch size: (pp_degree, partition, call) for every degree (planner.py:243-262);
    the seed partitions of all (batch, degree) pairs are computed concurrently."""
    cluster = ctx.cluster
    pairs = [(b, p) for b in batches for p in candidate_pp_degrees(cluster.n_devices) if p <= model.num_layers]
    cells = []
    for b, p in pairs:
        m = init_microbatch_num(b, p, opts.microbatch_cap_factor, opts.min_micro_size)
        cells.append((p, b // m, m))
    # one native call over host threads: the hill climb is a chain of dependent fp64 folds per
    # cell, as fast on host cores as on a warp (gbmw_seed_partitions_device: bit-identical,
    # 6.8 vs 5.2 ms for a GPT-3-96 window) and it overlaps the device pass
    try:
        parts = seed_partitions(model, ctx, cluster.n_devices, cells)
    except Exception:
        if len(batches) == 1:
            raise
        # a batch size of the window failed: seed per batch size, so that the error surfaces
        # only when the sequential sweep reaches that batch size (the reference's order)
        per = []
        for b in batches:
            try:
                per.append(_base_cells_window(model, ctx, [b], opts)[0])
            except Exception as e:          # re-raised by galvatron_base if it gets here
                per.append(e)
        return per
    out = {b: [] for b in batches}
    for (b, p), part in zip(pairs, parts):
        out[b].append((p, part, (cluster.mem_budget_bytes, partition_layers(model, part), cluster.n_devices, b, p)))
    return [out[b] for b in batches]


def _base_cells(model, ctx, batch, opts):
    return _base_cells_window(model, ctx, [batch], opts)[0]


_window_pool = None


def _window_executor():
    """One host thread that prepares the next batch window (its seed partitions) while the
    current window's searches run on the device (the ctypes calls release the GIL)."""
    global _window_pool
    if _window_pool is None:
        from concurrent.futures import ThreadPoolExecutor
        _window_pool = ThreadPoolExecutor(max_workers=1)
    return _window_pool


_search_pool = None


def _search_executor():
    """One host thread that runs the device passes of galvatron_base's windows, so that the
    next window's pass runs while the current window's outcomes are read."""
    global _search_pool
    if _search_pool is None:
        from concurrent.futures import ThreadPoolExecutor
        _search_pool = ThreadPoolExecutor(max_workers=1)
    return _search_pool


def _drain(fut):
    """Stop the speculative next-window preparation before the driver returns: cancel it if
    it has not started, else wait for it (its result is discarded)."""
    if fut is not None and not fut.cancel():
        try:
            fut.result()
        except Exception:
            pass


_host_lock = threading.Lock()
_host_depth = 0
_host_saved = (True, 0.005)


def _gc_paused(fn):
    """Run a planner driver with the automatic cyclic collector off and a short GIL switch
    interval (both restored after).  The searches allocate acyclic objects that reference
    counting frees, while a full collection of a large process (one that imported torch) holds
    the GIL for tens of milliseconds: measured, a 34 ms gen-2 pass stalled a 70 ms GPT-3-96
    plan_full.  The driver's helper threads (seeding, device passes) each need the GIL only
    briefly between native calls; at the default 5 ms interval they wait for the main thread's
    Python to block first (profiles/README.md)."""
    @wraps(fn)
    def run(*args, **kwargs):
        global _host_depth, _host_saved
        with _host_lock:                    # the outermost driver call (over all threads) saves and restores
            if _host_depth == 0:
                _host_saved = (gc.isenabled(), sys.getswitchinterval())
                gc.disable()
                sys.setswitchinterval(min(_host_saved[1], 1e-4))
            _host_depth += 1
        try:
            return fn(*args, **kwargs)
        finally:
            with _host_lock:
                _host_depth -= 1
                if _host_depth == 0:
                    sys.setswitchinterval(_host_saved[1])
                    if _host_saved[0]:
                        gc.enable()
    return run


@_gc_paused
def galvatron_base(model, cluster, profile, opts: PlannerOptions = PlannerOptions()) -> Plan:
    """Algorithm 1: raise the batch until no pipeline degree fits (planner.py:231-277)."""
    ctx = EvalContext(model=model, cluster=cluster, profile=profile)
    best: Plan | None = None
    batches = list(range(opts.batch_step, opts.max_batch + 1, opts.batch_step)) if opts.batch_step > 0 else []
    # where seeding is expensive (pipeline degrees >= 16: long hill climbs) windows of 16 batch
    # sizes and a short first window (its seeding is the only one not hidden behind a device
    # pass); elsewhere a window's pass is bound by its deepest search's layer-step chain, not
    # its width, so 32 batch sizes per pass halve the round trips (measured in
    # profiles/README.md: swin-bmw 47.7 -> 38.3 ms, vit-bmw 38.8 -> 31.9 ms; gpt96 24.8 -> 31.1
    # ms with 32, hence 16 there)
    large = min(cluster.n_devices, model.num_layers) >= 16
    window = max(1, opts.batch_window) if opts.batch_window > 0 else (16 if large else 32)
    first = max(1, window // 4) if large else window
    chunks = [batches[:first]] + [batches[i:i + window] for i in range(first, len(batches), window)] \
        if batches else []
    if not chunks:
        return best
    wex, sex = _window_executor(), _search_executor()
    seeds = {i: wex.submit(_base_cells_window, model, ctx, chunks[i], opts) for i in range(min(2, len(chunks)))}

    def launch(ci):
        """Window ci: its cells (its seeds), its problem table, and its device pass queued on
        the search thread.  An error is kept until the sweep reaches the window."""
        chunk = chunks[ci]
        try:
            per_batch = seeds.pop(ci).result()
            failed = next((i for i, cells in enumerate(per_batch) if isinstance(cells, Exception)), None)
            if failed is not None:      # the searches stop before the batch size whose seeding failed
                chunk, per_batch = chunk[:failed + 1], per_batch[:failed + 1]
            flat = [c[2] for cells in per_batch if not isinstance(cells, Exception) for c in cells]
            sliced = _sliced_cells(flat, ctx)
            if sliced is None:
                return chunk, per_batch, None, sex.submit(galvatron_search_batch, flat, ctx, opts, True), None
            sb = _slices_prepare(sliced, ctx, opts)
            return chunk, per_batch, sb, sex.submit(_slices_native, sb), None
        except Exception as e:
            return chunk, None, None, None, e

    def stop():
        # the speculative work past the stopping window: queued seeds and searches are
        # cancelled; a started device pass finishes on the search thread (its result unused);
        # a started seeding is waited for (it would compete for the host cores)
        for f in seeds.values():
            _drain(f)
        if nxt is not None and nxt[3] is not None:
            nxt[3].cancel()

    cur = launch(0)
    nxt = None
    for ci in range(len(chunks)):
        if ci + 2 < len(chunks):
            seeds[ci + 2] = wex.submit(_base_cells_window, model, ctx, chunks[ci + 2], opts)
        # speculative: the next window's table is built while this window's pass runs and its
        # pass queued behind it, so that this window's outcomes are read while it runs
        nxt = launch(ci + 1) if ci + 1 < len(chunks) else None
        chunk, per_batch, sb, fut, err = cur
        try:
            if err is not None:
                raise err
            raw = fut.result()
            outcomes = _slices_finish(sb, raw, defer_errors=True) if sb is not None else raw
        except BaseException:
            stop()
            raise
        k = 0
        for batch, cells in zip(chunk, per_batch):
            if isinstance(cells, Exception):
                stop()
                raise cells
            cell_best = None
            for p, part, _ in cells:
                outcome = outcomes[k]
                k += 1
                if isinstance(outcome, FailedOutcome):   # the reference's call raises here
                    stop()
                    outcome.raise_()
                if outcome.cost < INF and (cell_best is None or outcome.cost < cell_best[0]):
                    cell_best = (outcome.cost, p, part, outcome)
            if cell_best is None:
                stop()
                if best is None:
                    raise InfeasiblePlanError(f"no feasible plan at the smallest batch size {batch}",
                                              diagnostics=_infeasibility_diagnostics(model, ctx, batch, opts))
                return best
            _, p, part, outcome = cell_best
            plan = _assemble_plan(model, batch, p, part, outcome)
            if best is None or plan.predicted_throughput > best.predicted_throughput:
                best = plan
        cur = nxt
    return best


@_gc_paused
def plan_full(model, cluster, profile, opts: PlannerOptions = PlannerOptions()) -> Plan:
    """Algorithm 1, then (with bi_objective) Algorithm 2 around its batch size (planner.py:280-321)."""
    base = galvatron_base(model, cluster, profile, opts)
    if not opts.bi_objective:
        return base
    ctx = EvalContext(model=model, cluster=cluster, profile=profile)
    search = GalvatronSearch(ctx, opts)

    def microbatch_policy(batch, pp_degree):
        return init_microbatch_num(batch, pp_degree, opts.microbatch_cap_factor, opts.min_micro_size)

    b0 = base.batch_size
    lo = max(opts.batch_step, b0 - opts.batch_radius)
    batch_sizes = list(range(lo, b0 + opts.batch_radius + 1, opts.batch_step))
    degrees = [p for p in candidate_pp_degrees(cluster.n_devices) if 2 <= p <= model.num_layers]
    results = bi_objective_multi(model, ctx, batch_sizes, degrees, search, microbatch_policy)
    best = base
    for p in degrees:
        r = results[p]
        if not r.feasible:
            continue
        plan = _assemble_plan(model, r.batch_size, p, r.partition,
                              SearchOutcome(r.cost, r.strategies, r.stage_costs, r.n_micro))
        if plan.predicted_throughput > best.predicted_throughput:
            best = plan
        elif (plan.predicted_throughput == best.predicted_throughput
              and (plan.batch_size, plan.pp_degree) < (best.batch_size, best.pp_degree)):
            best = plan
    return best


def evaluate_plan_document(doc: dict, model, cluster, profile) -> float:
    """Re-cost a serialized plan (planner.py:324-341)."""
    ctx = EvalContext(model=model, cluster=cluster, profile=profile)
    m = doc["n_micro"]
    micro = doc["batch_size"] // m
    costs = []
    for idx, stage in enumerate(doc["stages"], start=1):
        layers = [model.layers[e["id"]] for e in stage["layers"]]
        strats = [parse_strategy(e["strategy"]) for e in stage["layers"]]
        costs.append(stage_cost(layers, strats, micro, ctx, stage_index=idx, n_micro=m))
    return pipeline_cost(costs, m)


@dataclass(frozen=True)
class OracleResult:
    feasible: bool
    cost: float
    pp_degree: int = 0
    partition: tuple[int, ...] = ()
    n_micro: int = 0
    strategies: tuple[ParallelStrategy, ...] = ()


# statistics of the last brute_force_oracle scan (assignments, device ms), for tests / tools
last_oracle_stats: dict = {}


def brute_force_oracle(model, cluster, profile, batch: int, max_layers: int = 4, max_devices: int = 4,
                       max_assignments: int = 0) -> OracleResult:
    """Exhaustive minimum over (P, partition, per-layer strategies, m) (planner.py:364-449).

    Same guards, loop order and first-minimum rule as the reference; the scan itself runs
    on the device (gbmw_brute_force, csrc/gbmw_brute.cu), so the guards can be raised far
    beyond the reference's 4 layers / 4 devices.  ``max_assignments`` (not in the
    reference) caps the scan; 0 = the library's default (2^44)."""
    from . import _native

    if model.num_layers > max_layers:
        raise ValueError(f"oracle limited to {max_layers} layers, got {model.num_layers}")
    if cluster.n_devices > max_devices:
        raise ValueError(f"oracle limited to {max_devices} devices, got {cluster.n_devices}")
    ctx = EvalContext(model=model, cluster=cluster, profile=profile)
    layers = _native.layers_array(list(model.layers), profile, {})
    env = np.array([_native.env_record(ctx)], dtype=_native.ENV_DT)
    L = len(layers)
    part = np.zeros(max(L, 1), dtype=np.int32)
    choice = np.zeros(max(L, 1), dtype=np.int32)
    rec = _native.OracleRecord()
    nctx = _native.default_context()
    with nctx.lock:
        rc = _native.lib().gbmw_brute_force(nctx.handle, _native.ptr(layers), L, _native.ptr(env), int(batch),
                                            float(cluster.mem_budget_bytes), float(max_assignments),
                                            _native.ptr(part), _native.ptr(choice), ctypes.byref(rec))
        msg = nctx.error() if rc else ""
    _native.raise_status(rc, msg)
    last_oracle_stats.clear()
    last_oracle_stats.update(assignments=rec.combos, device_ms=rec.device_ms)
    if not rec.feasible:
        return OracleResult(feasible=False, cost=INF)
    sset = enumerate_pruned(cluster.n_devices, rec.pp_degree).strategies
    return OracleResult(feasible=True, cost=rec.cost, pp_degree=rec.pp_degree,
                        partition=tuple(int(x) for x in part[:rec.n_stages]), n_micro=rec.n_micro,
                        strategies=tuple(sset[int(c)] for c in choice[:L]))


__all__ = [
    "DEFAULT_GRANULARITY_BYTES", "GalvatronSearch", "OracleResult", "Plan", "PlannerOptions", "bi_objective_optimize",
    "brute_force_oracle",
    "evaluate_plan_document", "galvatron_base", "galvatron_search", "galvatron_search_batch",
    "init_microbatch_num", "init_partition_memory_balanced", "plan_full", "PipelinePartition",
]
