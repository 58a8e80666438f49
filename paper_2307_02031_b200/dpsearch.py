"""Per-stage strategy search: the reference's ``dp_search`` API on the B200 kernels.

``dp_search`` keeps the signature, argument checks, exceptions and result type of
parapilot/dpsearch.py:89-227; the work runs in libgbmw (K1 cost tables, K2
min-plus layer steps, K3 E_fwd sweep with backward-peak validity, K4 backtrack
and stage cost).  ``dp_search_batch`` is the batched form the planner drivers
use: many independent stage searches in one device pass.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from .costs import StageCost
from .errors import DivisibilityError

MAX_BUCKETS = _native.MAX_BUCKETS
INF = float("inf")


@dataclass(frozen=True)
class DpResult:
    time_s: float
    strategies: tuple | None
    e_fwd_used: float
    feasible: bool
    frontier: tuple[tuple[float, float], ...] | None = None


@dataclass(frozen=True)
class StageProblem:
    """Arguments of one ``dp_search`` call."""

    stage_layers: Sequence
    budget_bytes: float
    strategies: object            # StrategySet (or any iterable of strategies)
    micro_batch: int
    granularity_bytes: int
    ctx: object                   # EvalContext
    stage_index: int = 1
    n_micro: int = 1
    fuse_identical: bool = False
    approx_prev: bool = False
    collect_frontier: bool = False


def _usable(strats, micro_batch):
    return [s for s in strats if micro_batch % s.data_degree == 0]


def _check(p: StageProblem):
    """dpsearch.py:103-121.  Returns (n_buckets, strategy list, early result or None)."""
    if p.granularity_bytes <= 0:
        raise ValueError(f"granularity_bytes must be positive, got {p.granularity_bytes}")
    if p.budget_bytes < 0:
        raise ValueError(f"budget_bytes must be non-negative, got {p.budget_bytes}")
    if not p.stage_layers:
        raise ValueError("stage must contain at least one layer")
    if p.micro_batch < 1:
        raise DivisibilityError(f"micro-batch must be >= 1, got {p.micro_batch}")
    strats = list(p.strategies)
    n_buckets = int(p.budget_bytes // p.granularity_bytes)
    if n_buckets > MAX_BUCKETS:
        raise ValueError(f"budget/granularity yields {n_buckets} buckets (> {MAX_BUCKETS}); "
                         f"increase the memory granularity")
    if not _usable(strats, p.micro_batch) or n_buckets == 0:
        return n_buckets, strats, DpResult(time_s=INF, strategies=None, e_fwd_used=0.0, feasible=False)
    return n_buckets, strats, None


_strat_arrays: dict = {}


def _frozen(strategies) -> bool:
    """True for containers whose contents cannot change under the same object: a tuple, or a
    StrategySet (frozen dataclass) holding a tuple (parapilot's and ours)."""
    return isinstance(strategies, tuple) or isinstance(getattr(strategies, "strategies", None), tuple)


def _strategies_array_cached(strategies, strat_list):
    """Strategy records of an immutable strategy set, built once per set object.  Mutable
    containers (a list the caller may change between calls) are re-read every call, as the
    reference re-reads them (dpsearch.py:42-43)."""
    if not _frozen(strategies):
        return _native.strategies_array(strat_list)
    hit = _strat_arrays.get(id(strategies))
    if hit is None or hit[0] is not strategies:
        if len(_strat_arrays) > 256:
            _strat_arrays.clear()
        hit = (strategies, _native.strategies_array(strat_list))
        _strat_arrays[id(strategies)] = hit
    return hit[1]


# per-layer strategy tuples of the plans the searches returned -> (the tuple, its strategy
# table, indices into it): evaluate_partition gathers their C records from the table's cached
# records instead of rebuilding them object by object (Algorithm 2 re-costs every plan)
_plan_records: dict = {}


def plan_records_register(plan: tuple, strats: tuple, idx: list):
    if len(_plan_records) > 4096:
        _plan_records.clear()
    _plan_records[id(plan)] = (plan, strats, idx)


def plan_records(per_layer_strategies):
    """STRATEGY_DT records of a plan tuple registered by a search, or None."""
    hit = _plan_records.get(id(per_layer_strategies))
    if hit is None or hit[0] is not per_layer_strategies:
        return None
    _, strats, idx = hit
    return _strategies_array_cached(strats, strats)[np.asarray(idx, dtype=np.intp)]


class _Marshal:
    """Deduplicating builder of the flat layer / strategy / env tables of a batch."""

    def __init__(self):
        self.layers: list = []
        self.layer_ranges: dict = {}
        self.strats: list = []
        self.strat_ranges: dict = {}
        self.envs: list = []
        self.env_index: dict = {}
        self.kinds: dict = {}

    def layer_range(self, layers, profile) -> int:
        key = (id(profile), tuple(id(l) for l in layers))
        hit = self.layer_ranges.get(key)
        if hit is None:
            hit = len(self.layers)
            self.layers.append(_native.layers_array(layers, profile, self.kinds))
            self.layer_ranges[key] = hit
        return hit

    def layer_table(self, arr) -> int:
        """Append a prebuilt LAYER_DT table (its kind ids its own: only for a batch whose
        layers all come from this one table)."""
        assert not self.layers, "a prebuilt layer table must be the batch's only one"
        self.layers.append(arr)
        return 0

    def strat_range(self, strategies, strat_list) -> int:
        # a mutable container is keyed on its elements as they are now
        key = id(strategies) if _frozen(strategies) else tuple(id(x) for x in strat_list)
        hit = self.strat_ranges.get(key)
        if hit is None or hit[1] is not strategies:
            hit = (len(self.strats), strategies)
            self.strats.append(_strategies_array_cached(strategies, strat_list))
            self.strat_ranges[key] = hit
        return hit[0]

    def env(self, ctx) -> int:
        key = id(ctx)
        hit = self.env_index.get(key)
        if hit is None:
            hit = len(self.envs)
            self.envs.append(_native.env_record(ctx))
            self.env_index[key] = hit
        return hit

    def finish(self):
        def cat(parts, dt):
            offs, total = [], 0
            for a in parts:
                offs.append(total)
                total += len(a)
            arr = np.concatenate(parts) if parts else np.zeros(0, dtype=dt)
            return arr, offs
        layers, loffs = cat(self.layers, _native.LAYER_DT)
        strats, soffs = cat(self.strats, _native.STRATEGY_DT)
        envs = np.array(self.envs, dtype=_native.ENV_DT) if self.envs else np.zeros(1, dtype=_native.ENV_DT)
        return layers, loffs, strats, soffs, envs


def run_native_batch(layers, strats, envs, probs, context=None):
    """gbmw_search_batch on flat tables; returns (status, results, plans, frontier)."""
    ctx = context or _native.default_context()
    n_plan = int(probs["n_layers"].clip(min=0).sum()) if len(probs) else 0
    n_front = int(probs["n_buckets"][(probs["flags"] & _native.FRONTIER) != 0].sum()) if len(probs) else 0
    results = np.zeros(len(probs), dtype=_native.RESULT_DT)
    plans = np.zeros(max(n_plan, 1), dtype=np.int32)
    frontier = np.zeros(max(n_front, 1), dtype=np.float64)
    with ctx.lock:
        rc = _native.lib().gbmw_search_batch(
            ctx.handle, _native.ptr(layers), len(layers), _native.ptr(strats), len(strats),
            _native.ptr(envs), len(envs), _native.ptr(probs), len(probs),
            _native.ptr(results), _native.ptr(plans), _native.ptr(frontier))
        msg = ctx.error() if rc != _native.OK else ""
        t = _native.Timing()
        if _native.lib().gbmw_ctx_last_timing(ctx.handle, ctypes.byref(t)) == _native.OK:
            STATS["batches"] += 1
            STATS["problems"] += len(probs)
            for k in ("transitions", "total_ms", "dp_ms", "sweep_ms", "n_launches"):
                STATS[k] += float(getattr(t, k))
    return rc, msg, results, plans, frontier


# device work issued through run_native_batch since import (or the last reset_stats())
STATS = {"batches": 0, "problems": 0, "transitions": 0.0, "total_ms": 0.0, "dp_ms": 0.0, "sweep_ms": 0.0,
         "n_launches": 0.0}


def reset_stats():
    for k in STATS:
        STATS[k] = 0 if isinstance(STATS[k], int) else 0.0


def dp_search_batch(problems: Sequence[StageProblem], want_stage_cost: bool = False):
    """Run many independent ``dp_search`` calls in one device pass.

    Returns a list of ``DpResult`` (and, with ``want_stage_cost``, a parallel list
    of ``StageCost | None`` for the returned plans, costs.py:322-352).
    Exceptions are raised as the first failing problem would raise them.
    """
    early: list = [None] * len(problems)
    meta: list = [None] * len(problems)
    m = _Marshal()
    rows = []
    native_idx = []
    for i, p in enumerate(problems):
        n_buckets, strats, res = _check(p)
        if res is not None:
            early[i] = res
            continue
        lb = m.layer_range(p.stage_layers, p.ctx.profile)
        sb = m.strat_range(p.strategies, strats)
        flags = (_native.FUSE if p.fuse_identical else 0) | (_native.FRONTIER if p.collect_frontier else 0) | \
                (_native.STAGE_COST if want_stage_cost else 0) | \
                (_native.APPROX if p.approx_prev else 0)
        rows.append((lb, len(p.stage_layers), sb, len(strats), m.env(p.ctx), int(p.stage_index),
                     int(p.n_micro), flags, int(p.micro_batch), int(p.granularity_bytes),
                     float(p.budget_bytes), n_buckets))
        meta[i] = (strats, n_buckets)
        native_idx.append(i)
    out = list(early)
    costs: list = [None] * len(problems)
    if rows:
        layers, loffs, strats_arr, soffs, envs = m.finish()
        probs = np.array(rows, dtype=_native.PROBLEM_DT)
        # translate per-part offsets into global offsets
        probs["layer_begin"] = [loffs[r] for r in probs["layer_begin"]]
        probs["strat_begin"] = [soffs[r] for r in probs["strat_begin"]]
        rc, msg, results, plans, frontier = run_native_batch(layers, strats_arr, envs, probs)
        if rc != _native.OK:
            bad = int(np.flatnonzero(results["status"] != 0)[0]) if (results["status"] != 0).any() else -1
            _native.raise_status(int(results["status"][bad]) if bad >= 0 else rc, msg)
        plan_off = 0
        for k, i in enumerate(native_idx):
            p = problems[i]
            strats, n_buckets = meta[i]
            r = results[k]
            n_l = len(p.stage_layers)
            front = None
            if p.collect_frontier:
                fo = int(r["frontier_off"])
                vals = frontier[fo:fo + n_buckets]
                g = p.granularity_bytes
                front = tuple((e * g, float(vals[e - 1])) for e in range(1, n_buckets + 1))
            if r["feasible"]:
                idx = plans[plan_off:plan_off + n_l]
                out[i] = DpResult(time_s=float(r["time_s"]), strategies=tuple(strats[j] for j in idx),
                                  e_fwd_used=float(r["e_fwd"]), feasible=True, frontier=front)
                costs[i] = StageCost(float(r["stage_time"]), float(r["stage_ns"]), float(r["stage_peak"]))
            else:
                out[i] = DpResult(time_s=INF, strategies=None, e_fwd_used=0.0, feasible=False, frontier=front)
            plan_off += n_l
    return (out, costs) if want_stage_cost else out


def dp_search(stage_layers, budget_bytes: float, strategies, micro_batch: int, granularity_bytes: int,
              ctx, stage_index: int = 1, n_micro: int = 1, fuse_identical: bool = False,
              approx_prev: bool = False, collect_frontier: bool = False) -> DpResult:
    """Optimal per-layer strategy assignment for one pipeline stage (dpsearch.py:89-227)."""
    return dp_search_batch([StageProblem(list(stage_layers), budget_bytes, strategies, micro_batch,
                                         granularity_bytes, ctx, stage_index, n_micro, fuse_identical,
                                         approx_prev, collect_frontier)])[0]


def backward_peak_bound(stage_layers, strategies, micro_batch: int, ms_multiplier: float) -> float:
    """b_up with stage_index=1, n_micro=1 (dpsearch.py:46-59)."""
    from .costs import layer_memory
    peak = 0.0
    usable = _usable(list(strategies), micro_batch)
    for layer in stage_layers:
        for s in usable:
            peak = max(peak, layer_memory(layer, s, micro_batch, 1, 1, ms_multiplier)[1])
    return peak


class SearchBatch:
    """Prepared batch on the device (gbmw_batch_*): run() is device-only, fetch() copies back."""

    def __init__(self, layers, strats, envs, probs, context=None):
        self.ctx = context or _native.default_context()
        self.layers, self.strats, self.envs, self.probs = layers, strats, envs, probs
        self.handle = ctypes.c_void_p()
        L = _native.lib()
        with self.ctx.lock:
            rc = L.gbmw_batch_create(self.ctx.handle, _native.ptr(layers), len(layers), _native.ptr(strats),
                                     len(strats), _native.ptr(envs), len(envs), _native.ptr(probs), len(probs),
                                     ctypes.byref(self.handle))
            if rc != _native.OK:
                msg = self.ctx.error()
                if self.handle:
                    L.gbmw_batch_destroy(self.handle)
                    self.handle = None
                _native.raise_status(rc, msg)

    def run(self):
        with self.ctx.lock:
            rc = _native.lib().gbmw_batch_run(self.ctx.handle, self.handle)
            if rc != _native.OK:
                _native.raise_status(rc, self.ctx.error())

    def fetch(self, with_plans: bool = True):
        n_plan = int(self.probs["n_layers"].sum())
        n_front = int(self.probs["n_buckets"][(self.probs["flags"] & _native.FRONTIER) != 0].sum())
        results = np.zeros(len(self.probs), dtype=_native.RESULT_DT)
        plans = np.zeros(max(n_plan, 1), dtype=np.int32) if with_plans else None
        frontier = np.zeros(max(n_front, 1), dtype=np.float64) if n_front else None
        with self.ctx.lock:
            rc = _native.lib().gbmw_batch_fetch(self.ctx.handle, self.handle, _native.ptr(results),
                                                _native.ptr(plans), _native.ptr(frontier))
            if rc != _native.OK:
                _native.raise_status(rc, self.ctx.error())
        return results, plans, frontier

    def timing(self) -> dict:
        t = _native.Timing()
        _native.lib().gbmw_batch_timing(self.handle, ctypes.byref(t))
        return t.as_dict()

    def close(self):
        if self.handle:
            _native.lib().gbmw_batch_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
