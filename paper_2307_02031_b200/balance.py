"""Pipeline-partition balance and the bi-objective BMW loop (Algorithm 2).

Names, signatures and semantics of parapilot/balance.py:27-488.  The O(L^2 P)
partition work (stage costs of a partition, memory/time-balanced seeds with hill
climbing, the seed-strategy choice) runs in libgbmw (gbmw_planner.cpp); the BMW
queue loop batches the strategy searches of all (batch size, degree)
trajectories of a round into one device pass when the search function is this
package's (``GalvatronSearch``), and is replayed in the reference's order so
results and tie-breaks are identical (balance.py:357-436).
"""

from __future__ import annotations

import ctypes
import logging
from collections.abc import Sequence as _AbcSequence
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import _native
from . import dpsearch as _dps
from .costs import EvalContext, StageCost
from .strategies import DP, SDP, TP, ParallelStrategy

logger = logging.getLogger(__name__)

INF = float("inf")


@dataclass(frozen=True)
class PipelinePartition:
    stage_sizes: tuple[int, ...]

    def __post_init__(self):
        if not self.stage_sizes:
            raise ValueError("partition must have at least one stage")
        if any(s < 1 for s in self.stage_sizes):
            raise ValueError(f"every stage needs at least one layer: {self.stage_sizes}")

    @property
    def num_stages(self) -> int:
        return len(self.stage_sizes)

    @property
    def num_layers(self) -> int:
        return sum(self.stage_sizes)

    def boundaries(self) -> list[tuple[int, int]]:
        out, a = [], 0
        for n in self.stage_sizes:
            out.append((a, a + n))
            a += n
        return out


@dataclass(frozen=True)
class BalanceReport:
    alpha_t: float
    alpha_m: float
    stage_times: tuple[float, ...]
    stage_mems: tuple[float, ...]


def balance_degrees(stage_costs: Sequence[StageCost]) -> BalanceReport:
    """alpha = 1 - max / sum over stages, for times and peak memories (balance.py:62-77)."""
    if not stage_costs:
        raise ValueError("need at least one stage")
    times = tuple(sc.time_s for sc in stage_costs)
    mems = tuple(sc.peak_mem_bytes for sc in stage_costs)
    tt, tm = sum(times), sum(mems)
    if tt <= 0 or tm <= 0:
        raise ValueError("stage totals must be positive to define balance degrees")
    return BalanceReport(alpha_t=1.0 - max(times) / tt, alpha_m=1.0 - max(mems) / tm,
                         stage_times=times, stage_mems=mems)


class StageLayers(_AbcSequence):
    """The per-stage layer lists of a partition of ``model.layers`` (balance.py's
    ``partition_layers`` result): an immutable sequence of lists, built on first access.
    The batched search only needs the slices (``ranges``), so the drivers, which partition
    thousands of (batch, degree) cells per window, never copy the layers."""
    __slots__ = ("model", "ranges", "_lists")

    def __init__(self, model, ranges):
        self.model = model
        self.ranges = ranges
        self._lists = None

    def _materialize(self):
        if self._lists is None:
            ls = self.model.layers
            self._lists = [list(ls[a:a + n]) for a, n in self.ranges]
        return self._lists

    def __len__(self):
        return len(self.ranges)

    def __getitem__(self, i):
        return self._materialize()[i]

    def __iter__(self):
        return iter(self._materialize())

    def __eq__(self, other):
        return list(self) == list(other) if isinstance(other, (list, tuple, StageLayers)) else NotImplemented

    def __repr__(self):
        return repr(self._materialize())


def partition_layers(model, partition: PipelinePartition) -> Sequence[list]:
    if partition.num_layers != model.num_layers:
        raise ValueError(f"partition covers {partition.num_layers} layers, model has {model.num_layers}")
    ranges, a = [], 0
    for n in partition.stage_sizes:
        ranges.append((a, n))
        a += n
    return StageLayers(model, ranges)


def seed_strategy(n_devices: int, pp_degree: int, use_sdp: bool = False) -> ParallelStrategy:
    group = n_devices // pp_degree
    levels = () if group == 1 else (((SDP if use_sdp else DP), group),)
    return ParallelStrategy(pp_degree=pp_degree, levels=levels, ckpt=False)


# ----------------------------------------------------------------------------- native plumbing

_layer_cache: dict = {}


def _layers(model, profile) -> np.ndarray:
    """LAYER_DT table of a model under a profile, cached per (model, profile) object pair; the
    profile's override mapping (the one mutable part) is compared on every call."""
    key = (id(model), id(profile))
    ov = getattr(profile, "layer_overrides", None)
    snap = dict(ov) if isinstance(ov, dict) else None
    hit = _layer_cache.get(key)
    if hit is None or hit[0] is not model or hit[1] is not profile or hit[2] != snap:
        arr = _native.layers_array(model.layers, profile, {})
        if len(_layer_cache) > 64:
            _layer_cache.clear()
        hit = (model, profile, snap, arr)
        _layer_cache[key] = hit
    return hit[3]


_env_cache: dict = {}


def _env(ctx) -> np.ndarray:
    """ENV_DT record of an EvalContext, built once per context object (its cluster, profile
    and model are frozen dataclasses, so the record cannot change under the same object)."""
    if not isinstance(ctx, EvalContext):         # a duck-typed context may change: re-read it
        return np.array([_native.env_record(ctx)], dtype=_native.ENV_DT)
    hit = _env_cache.get(id(ctx))
    if hit is None or hit[0] is not ctx:
        if len(_env_cache) > 64:
            _env_cache.clear()
        hit = (ctx, np.array([_native.env_record(ctx)], dtype=_native.ENV_DT))
        _env_cache[id(ctx)] = hit
    return hit[1]


def _planner_error(rc: int):
    msg = _native.lib().gbmw_planner_last_error().decode()
    _native.raise_status(rc, msg)


def evaluate_partition(model, partition: PipelinePartition, per_layer_strategies: Sequence[ParallelStrategy],
                       micro_batch: int, n_micro: int, ctx) -> list[StageCost]:
    """Stage costs of a partition under fixed per-layer strategies (balance.py:98-119)."""
    if len(per_layer_strategies) != model.num_layers:
        raise ValueError("need one strategy per model layer")
    sizes = np.array(partition.stage_sizes, dtype=np.int32)
    strats = _dps.plan_records(per_layer_strategies)    # a searched plan: records by index
    if strats is None:
        strats = _native.strategies_array(per_layer_strategies)
    out = np.zeros(3 * len(sizes), dtype=np.float64)
    layers = _layers(model, ctx.profile)
    env = _env(ctx)
    # raw addresses: every array is bound to a local for the duration of the call
    rc = _native.lib().gbmw_partition_costs(layers.ctypes.data, len(layers), strats.ctypes.data,
                                            sizes.ctypes.data, len(sizes), env.ctypes.data,
                                            int(micro_batch), int(n_micro), out.ctypes.data)
    if rc != _native.OK:
        _planner_error(rc)
    o = out.tolist()
    return [StageCost(o[3 * s], o[3 * s + 1], o[3 * s + 2]) for s in range(len(sizes))]


def _init_partition(model, num_stages, seed_strategies, micro_batch, n_micro, ctx, objective) -> PipelinePartition:
    if num_stages > model.num_layers:
        raise ValueError(f"cannot split {model.num_layers} layers into {num_stages} pipeline stages")
    if len(seed_strategies) != model.num_layers:
        raise ValueError("need one seed strategy per layer")
    strats = _native.strategies_array(list(seed_strategies))
    out = np.zeros(num_stages, dtype=np.int32)
    layers = _layers(model, ctx.profile)
    env = _env(ctx)
    rc = _native.lib().gbmw_init_partition(_native.ptr(layers), len(layers), _native.ptr(strats), int(num_stages),
                                           _native.ptr(env), int(micro_batch), int(n_micro),
                                           0 if objective == "memory" else 1, _native.ptr(out))
    if rc != _native.OK:
        _planner_error(rc)
    return PipelinePartition(tuple(int(x) for x in out))


def init_partition_memory_balanced(model, num_stages, seed_strategies, micro_batch, n_micro, ctx):
    """p_m (balance.py:215-224)."""
    return _init_partition(model, num_stages, seed_strategies, micro_batch, n_micro, ctx, "memory")


def init_partition_time_balanced(model, num_stages, seed_strategies, micro_batch, n_micro, ctx):
    """p_t (balance.py:227-236)."""
    return _init_partition(model, num_stages, seed_strategies, micro_batch, n_micro, ctx, "time")


def _seed_and_partition(model, ctx, n_devices, pp_degree, micro_batch, n_micro):
    """_seed_for (balance.py:471-488) + the memory-balanced partition of its seed list."""
    seed = np.zeros(1, dtype=_native.STRATEGY_DT)
    sizes = np.zeros(pp_degree, dtype=np.int32)
    layers = _layers(model, ctx.profile)
    env = _env(ctx)
    rc = _native.lib().gbmw_seed_for(_native.ptr(layers), len(layers), _native.ptr(env), int(n_devices),
                                     int(pp_degree), int(micro_batch), int(n_micro),
                                     float(ctx.cluster.mem_budget_bytes), _native.ptr(seed), _native.ptr(sizes))
    if rc != _native.OK:
        _planner_error(rc)
    r = seed[0]
    n = int(r["n_levels"])
    s = ParallelStrategy(int(r["pp_degree"]), tuple((_native.PARADIGM_NAME[int(r["paradigm"][i])],
                                                     int(r["degree"][i])) for i in range(n)), bool(r["ckpt"]))
    return [s] * model.num_layers, PipelinePartition(tuple(int(x) for x in sizes))


def seed_partitions(model, ctx, n_devices, cells, n_threads: int | None = None,
                    device=None) -> list[PipelinePartition]:
    """The memory-balanced partition of the ``_seed_for`` strategy (balance.py:471-488,
    planner.py:250-253) for many ``(pp_degree, micro_batch, n_micro)`` cells at once: one
    native call, on the GPU of ``device`` (a ``_native.Context``: a warp per cell,
    gbmw_seed_partitions_device) or on host threads (gbmw_seed_partitions)."""
    import os
    n = len(cells)
    if n == 0:
        return []
    pp = np.array([c[0] for c in cells], dtype=np.int64)
    micro = np.array([c[1] for c in cells], dtype=np.int64)
    nm = np.array([c[2] for c in cells], dtype=np.int32)
    width = int(pp.max())
    sizes = np.zeros((n, width), dtype=np.int32)
    layers = _layers(model, ctx.profile)
    env = _env(ctx)
    budget = float(ctx.cluster.mem_budget_bytes)
    if device is not None:
        with device.lock:
            rc = _native.lib().gbmw_seed_partitions_device(
                device.handle, _native.ptr(layers), len(layers), _native.ptr(env), int(n_devices), n, _native.ptr(pp),
                _native.ptr(micro), _native.ptr(nm), budget, width, _native.ptr(sizes))
            if rc != _native.OK:
                _native.raise_status(rc, device.error())
    else:
        # leave cores to the main thread (batch creation, launches) that runs beside the seeding
        threads = n_threads or max(1, min(16, len(os.sched_getaffinity(0)) // 2))
        rc = _native.lib().gbmw_seed_partitions(_native.ptr(layers), len(layers), _native.ptr(env), int(n_devices),
                                                n, _native.ptr(pp), _native.ptr(micro), _native.ptr(nm), budget,
                                                width, int(threads), _native.ptr(sizes))
        if rc != _native.OK:
            _planner_error(rc)
    return [PipelinePartition(tuple(int(x) for x in sizes[i, :int(pp[i])])) for i in range(n)]


def _seed_for(model, ctx, n_devices, pp_degree, micro_batch, n_micro) -> list[ParallelStrategy]:
    return _seed_and_partition(model, ctx, n_devices, pp_degree, micro_batch, n_micro)[0]


def adjust_partition(partition: PipelinePartition, stage_costs: Sequence[StageCost]) -> PipelinePartition:
    """Shift one boundary layer off the slowest stage to its faster neighbour (balance.py:239-268)."""
    sizes = list(partition.stage_sizes)
    if len(sizes) != len(stage_costs):
        raise ValueError("one stage cost per stage required")
    times = [sc.time_s for sc in stage_costs]
    slowest = max(range(len(times)), key=lambda i: (times[i], -i))
    if sizes[slowest] <= 1:
        return partition
    options = []
    if slowest + 1 < len(sizes):
        options.append((times[slowest + 1], 0, slowest + 1))
    if slowest >= 1:
        options.append((times[slowest - 1], 1, slowest - 1))
    options.sort()
    if not options or options[0][0] >= times[slowest]:
        return partition
    sizes[slowest] -= 1
    sizes[options[0][2]] += 1
    return PipelinePartition(tuple(sizes))


def validate_partition(new_partition: PipelinePartition, costs_under_new: Sequence[StageCost], c_max_prev: float,
                       mem_budget_bytes: float, max_mem_under_time_balanced: float) -> bool:
    """The three acceptance rules of balance.py:271-293."""
    if new_partition.num_stages != len(costs_under_new):
        raise ValueError("one stage cost per stage required")
    return all(sc.time_s <= c_max_prev and sc.peak_mem_bytes <= mem_budget_bytes
               and sc.peak_mem_bytes <= max_mem_under_time_balanced for sc in costs_under_new)


@dataclass(frozen=True)
class SearchOutcome:
    cost: float
    strategies: tuple[ParallelStrategy, ...] | None
    stage_costs: tuple[StageCost, ...] | None
    n_micro: int


@dataclass
class BiObjectiveResult:
    cost: float = INF
    partition: PipelinePartition | None = None
    strategies: tuple[ParallelStrategy, ...] | None = None
    stage_costs: tuple[StageCost, ...] | None = None
    batch_size: int = 0
    n_micro: int = 1
    trajectory: list[dict] = field(default_factory=list)

    @property
    def feasible(self) -> bool:
        return self.cost != INF and self.strategies is not None


SearchFn = Callable[[float, list, int, int, int], SearchOutcome]


def default_microbatch_policy(batch: int, pp_degree: int) -> int:
    if pp_degree <= 1:
        return 1
    m = max(1, min(4 * pp_degree, batch))
    while batch % m:
        m -= 1
    return m


def _finite(x: float) -> bool:
    return x != INF and x == x


def _stats(record, outcome):
    report = balance_degrees(outcome.stage_costs)
    record.update(alpha_t=report.alpha_t, alpha_m=report.alpha_m, max_stage_time=max(report.stage_times),
                  max_stage_mem=max(report.stage_mems))
    return report


class _Trajectory:
    """One (batch size, pipeline degree) cell of Algorithm 2: a FIFO of partitions."""

    def __init__(self, b_index, batch, pp_degree):
        self.b_index, self.batch, self.pp = b_index, batch, pp_degree
        self.queue: list[PipelinePartition] = []
        self.visited: set = set()
        self.iterations = 0
        self.mem_ref = INF
        self.events: list = []          # (iteration, partition, outcome, record)
        self.single = False             # P == 1 probe


def _run_trajectories(model, ctx, trajs: list[_Trajectory], search, microbatch_policy, cap):
    """Advance all trajectories in lockstep rounds; searches of a round share one device pass."""
    cluster = ctx.cluster
    n_dev, budget, L = cluster.n_devices, cluster.mem_budget_bytes, model.num_layers

    multi = [t for t in trajs if not t.single]
    # every trajectory's set-up (_seed_for, its memory-balanced p0, the time-balanced p_t and
    # mem_ref = max stage peak of p_t) in one native call over host threads
    if multi:
        import os
        pp = np.array([t.pp for t in multi], dtype=np.int64)
        nm = np.array([microbatch_policy(t.batch, t.pp) for t in multi], dtype=np.int32)
        micro = np.array([t.batch // int(m) for t, m in zip(multi, nm)], dtype=np.int64)
        width = int(pp.max())
        p0s = np.zeros((len(multi), width), dtype=np.int32)
        mem_refs = np.zeros(len(multi), dtype=np.float64)
        layers = _layers(model, ctx.profile)
        env = _env(ctx)
        threads = max(1, min(len(multi), len(os.sched_getaffinity(0)) // 2))
        rc = _native.lib().gbmw_bmw_setup(layers.ctypes.data, len(layers), env.ctypes.data, int(n_dev), len(multi),
                                          pp.ctypes.data, micro.ctypes.data, nm.ctypes.data, float(budget), width,
                                          threads, p0s.ctypes.data, mem_refs.ctypes.data)
        if rc != _native.OK:
            _planner_error(rc)
        for i, t in enumerate(multi):
            p0 = PipelinePartition(tuple(p0s[i, :t.pp].tolist()))
            t.mem_ref = float(mem_refs[i])
            t.queue = [p0]
            t.visited = {p0.stage_sizes}
    for t in trajs:
        if t.single:
            t.queue = [PipelinePartition((L,))]
    batched = getattr(search, "batch", None)
    while True:
        active = [t for t in trajs if t.queue and (t.single and t.iterations == 0 or
                                                   not t.single and t.iterations < cap)]
        if not active:
            break
        parts = []
        for t in active:
            t.iterations += 1
            parts.append(t.queue.pop(0))
        calls = [(budget, partition_layers(model, p), n_dev, t.batch, t.pp) for t, p in zip(active, parts)]
        outcomes = batched(calls) if batched is not None else [search(*c) for c in calls]
        # pass 1: each trajectory's statistics and adjusted partition; the adjusted partitions
        # of the round are then costed in one native call (independent per trajectory)
        pending = []
        for t, part, outcome in zip(active, parts, outcomes):
            record = {"batch_size": t.batch, "pp_degree": t.pp, "partition": list(part.stage_sizes),
                      "iteration": t.iterations, "cost": outcome.cost, "accepted": False, "proposed": None}
            if not _finite(outcome.cost) or outcome.strategies is None:
                t.events.append((part, outcome, record, False))
                continue
            report = _stats(record, outcome)
            if t.single:
                t.events.append((part, outcome, record, True))
                continue
            adjusted = adjust_partition(part, outcome.stage_costs)
            if adjusted.stage_sizes != part.stage_sizes:
                pending.append((t, adjusted, outcome, record, max(report.stage_times)))
            t.events.append((part, outcome, record, True))
        # pass 2: validation in trajectory order (balance.py:420-431)
        for (t, adjusted, outcome, record, c_max_prev), costs_adj in zip(pending, _costs_batch(model, ctx, pending)):
            ok = validate_partition(adjusted, costs_adj, c_max_prev, budget, t.mem_ref)
            record["proposed"] = list(adjusted.stage_sizes)
            record["accepted"] = bool(ok and adjusted.stage_sizes not in t.visited)
            if ok and adjusted.stage_sizes not in t.visited:
                t.visited.add(adjusted.stage_sizes)
                t.queue.append(adjusted)


def _costs_batch(model, ctx, pending) -> list[list[StageCost]]:
    """evaluate_partition of every (trajectory, adjusted partition, outcome) of a round in one
    native call (gbmw_partition_costs_batch)."""
    n = len(pending)
    if n == 0:
        return []
    if n == 1:
        t, adjusted, outcome, _, _ = pending[0]
        return [evaluate_partition(model, adjusted, outcome.strategies, t.batch // outcome.n_micro,
                                   outcome.n_micro, ctx)]
    L = model.num_layers
    recs = []
    for t, adjusted, outcome, _, _ in pending:
        if len(outcome.strategies) != L:
            raise ValueError("need one strategy per model layer")
        r = _dps.plan_records(outcome.strategies)
        recs.append(r if r is not None else _native.strategies_array(outcome.strategies))
    per_layer = np.concatenate(recs)
    width = max(len(a.stage_sizes) for _, a, _, _, _ in pending)
    sizes = np.zeros((n, width), dtype=np.int32)
    n_st = np.zeros(n, dtype=np.int32)
    for i, (_, a, _, _, _) in enumerate(pending):
        sizes[i, :len(a.stage_sizes)] = a.stage_sizes
        n_st[i] = len(a.stage_sizes)
    micro = np.array([t.batch // o.n_micro for t, _, o, _, _ in pending], dtype=np.int64)
    nm = np.array([o.n_micro for _, _, o, _, _ in pending], dtype=np.int32)
    out = np.zeros((n, 3 * width), dtype=np.float64)
    layers = _layers(model, ctx.profile)
    env = _env(ctx)
    # one thread: a round has a few dozen items of ~15 us each; spawning threads per round
    # cost more than it saved (measured: swin-bmw Algorithm 2 host time 5.0 -> 6.3 ms)
    threads = 1
    rc = _native.lib().gbmw_partition_costs_batch(layers.ctypes.data, len(layers), per_layer.ctypes.data,
                                                  sizes.ctypes.data, n_st.ctypes.data, width, env.ctypes.data,
                                                  micro.ctypes.data, nm.ctypes.data, n, threads, out.ctypes.data)
    if rc != _native.OK:
        _planner_error(rc)
    o = out.tolist()
    return [[StageCost(o[i][3 * s], o[i][3 * s + 1], o[i][3 * s + 2]) for s in range(int(n_st[i]))]
            for i in range(n)]


def _replay(result: BiObjectiveResult, trajs: list[_Trajectory]):
    """Best-so-far in the reference's order (batch list order, then iteration), strict <
    on raw cost (balance.py:410-416, :461)."""
    for t in sorted(trajs, key=lambda x: x.b_index):
        for part, outcome, record, ok in t.events:
            if ok and outcome.cost < result.cost:
                result.cost = outcome.cost
                result.partition = part
                result.strategies = outcome.strategies
                result.stage_costs = outcome.stage_costs
                result.batch_size = t.batch
                result.n_micro = outcome.n_micro
            result.trajectory.append(record)
            if ok and not t.single:
                logger.debug("bi-objective step: %s", record)


def bi_objective_optimize(model, ctx, batch_sizes: Sequence[int], pp_degree: int, search: SearchFn,
                          microbatch_policy: Callable[[int, int], int] = default_microbatch_policy,
                          max_iterations: int | None = None) -> BiObjectiveResult:
    """Algorithm 2 for one pipeline degree over a batch-size range (balance.py:334-436)."""
    return bi_objective_multi(model, ctx, batch_sizes, [pp_degree], search, microbatch_policy,
                              max_iterations)[pp_degree]


def bi_objective_multi(model, ctx, batch_sizes, pp_degrees, search, microbatch_policy=default_microbatch_policy,
                       max_iterations=None) -> dict:
    """bi_objective_optimize for several degrees at once (independent results, one lockstep)."""
    L = model.num_layers
    cap = max_iterations if max_iterations is not None else 4 * L
    per_p: dict = {}
    trajs_all = []
    for p in pp_degrees:
        trajs = []
        for bi, batch in enumerate(batch_sizes):
            if batch < 1:
                continue
            if p == 1:
                t = _Trajectory(bi, batch, 1)
                t.single = True
                trajs.append(t)
            elif p <= L:
                trajs.append(_Trajectory(bi, batch, p))
        per_p[p] = trajs
        trajs_all.extend(trajs)
    _run_trajectories(model, ctx, trajs_all, search, microbatch_policy, cap)
    out = {}
    for p in pp_degrees:
        res = BiObjectiveResult()
        _replay(res, per_p[p])
        out[p] = res
    return out
