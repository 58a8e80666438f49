"""Cost-model API (names and signatures of parapilot/costs.py:21-368).

Every per-(layer, strategy) number comes from the native cost model
(costmodel.cuh through gbmw_layer_cost / gbmw_comm_breakdown /
gbmw_transform_cost), the same code the sm_100a table kernel runs, so the API
and the search agree bit for bit.  Stage / pipeline aggregation here is the
reference's own O(L) left-to-right fold.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

from . import _native
from .errors import DivisibilityError
from .strategies import ParallelStrategy


@dataclass(frozen=True)
class EvalContext:
    model: object
    cluster: object
    profile: object

    @property
    def ms_multiplier(self) -> float:
        return self.model.ms_bytes_per_param_byte


@dataclass(frozen=True)
class LayerCost:
    time_s: float
    mem_fwd_bytes: float
    mem_bwd_bytes: float
    mem_states_bytes: float
    time_no_sync_s: float


@dataclass(frozen=True)
class StageCost:
    time_s: float
    time_no_sync_s: float
    peak_mem_bytes: float


@dataclass(frozen=True)
class CommBreakdown:
    grad_s: float
    fwd_act_s: float
    bwd_act_s: float
    ckpt_act_s: float

    @property
    def act_total_s(self) -> float:
        return self.fwd_act_s + self.bwd_act_s + self.ckpt_act_s


# ----------------------------------------------------------------------------- ctypes records

class _CStrategy(ctypes.Structure):
    _fields_ = [("pp_degree", ctypes.c_int32), ("n_levels", ctypes.c_int32),
                ("paradigm", ctypes.c_int32 * 3), ("degree", ctypes.c_int32 * 3), ("ckpt", ctypes.c_int32)]


class _CLayer(ctypes.Structure):
    _fields_ = [("param_bytes", ctypes.c_int64), ("bnd", ctypes.c_int64), ("intb", ctypes.c_int64),
                ("fwd", ctypes.c_double), ("fwd_raw", ctypes.c_double), ("frac", ctypes.c_double),
                ("kind", ctypes.c_int64)]


class _CEnv(ctypes.Structure):
    _fields_ = [("n_devices", ctypes.c_int64), ("island", ctypes.c_int64), ("intra", ctypes.c_double),
                ("inter", ctypes.c_double), ("slowdown", ctypes.c_double), ("bwd_ratio", ctypes.c_double),
                ("coll_eff", ctypes.c_double), ("ms", ctypes.c_double)]


@lru_cache(maxsize=4096)
def _c_strategy(s) -> _CStrategy:
    pp, n, par, deg, ck = _native.strategy_record(s)
    return _CStrategy(pp, n, (ctypes.c_int32 * 3)(*par), (ctypes.c_int32 * 3)(*deg), ck)


def _c_layer(layer, fwd_time: float) -> _CLayer:
    return _CLayer(int(layer.param_bytes), int(layer.bnd_bytes_per_sample), int(layer.int_bytes_per_sample),
                   float(fwd_time), float(layer.fwd_time_per_sample), float(layer.tp_act_replication_fraction), 0)


def _c_env(cluster, profile, ms_mult: float = 4.0) -> _CEnv:
    return _CEnv(int(cluster.n_devices), int(cluster.island_size), float(cluster.intra_island_bw),
                 float(cluster.inter_island_bw), float(cluster.overlap_slowdown),
                 float(profile.bwd_fwd_ratio) if profile is not None else 2.0,
                 float(profile.collective_efficiency) if profile is not None else 1.0, float(ms_mult))


def _fwd(profile, layer) -> float:
    return profile.fwd_time(layer) if profile is not None else layer.fwd_time_per_sample


def _check_divisible(strategy, micro_batch: int) -> int:
    data = strategy.data_degree
    if micro_batch % data:
        raise DivisibilityError(f"micro-batch {micro_batch} is not divisible by the DP*SDP degree {data} "
                                f"of strategy {strategy}")
    return micro_batch // data


def _native_layer_cost(layer, strategy, micro_batch, cluster, profile, stage_index, n_micro, ms_mult):
    _check_divisible(strategy, micro_batch)
    out = (ctypes.c_double * 5)()
    rc = _native.lib().gbmw_layer_cost(ctypes.byref(_c_layer(layer, _fwd(profile, layer))),
                                       ctypes.byref(_c_strategy(strategy)),
                                       ctypes.byref(_c_env(cluster, profile, ms_mult)),
                                       int(micro_batch), int(stage_index), int(n_micro), out)
    _native.raise_status(rc, _native.global_error())
    return tuple(out)


# ----------------------------------------------------------------------------- per layer

def overlap(a: float, b: float, slowdown: float) -> float:
    """Contention model (costs.py:50-54)."""
    if a > 0.0 and b > 0.0:
        return max(a, b) * slowdown
    return a + b


def level_bandwidth(strategy: ParallelStrategy, level_index: int, cluster) -> float:
    span = 1
    for _, d in strategy.levels[level_index:]:
        span *= d
    return cluster.intra_island_bw if span <= cluster.island_size else cluster.inter_island_bw


def comm_breakdown(layer, strategy, micro_batch: int, cluster, profile) -> CommBreakdown:
    out = (ctypes.c_double * 4)()
    rc = _native.lib().gbmw_comm_breakdown(ctypes.byref(_c_layer(layer, layer.fwd_time_per_sample)),
                                           ctypes.byref(_c_strategy(strategy)),
                                           ctypes.byref(_c_env(cluster, profile)), int(micro_batch), out)
    _native.raise_status(rc, _native.global_error())
    return CommBreakdown(*out)


def comm_time(layer, strategy, micro_batch: int, cluster, profile) -> tuple[float, float]:
    parts = comm_breakdown(layer, strategy, micro_batch, cluster, profile)
    return parts.grad_s, parts.act_total_s


def compute_time(layer, strategy, micro_batch: int, profile) -> float:
    samples = _check_divisible(strategy, micro_batch)
    fwd = samples * profile.fwd_time(layer) / strategy.tp_degree
    return fwd * (1.0 + profile.bwd_fwd_ratio + (1.0 if strategy.ckpt else 0.0))


def _layer_times(layer, strategy, micro_batch: int, cluster, profile) -> tuple[float, float]:
    t, t_ns, *_ = _native_layer_cost(layer, strategy, micro_batch, cluster, profile,
                                     strategy.pp_degree, 1, 4.0)
    return t, t_ns


def layer_time(layer, strategy, micro_batch: int, cluster, profile) -> float:
    return _layer_times(layer, strategy, micro_batch, cluster, profile)[0]


def layer_memory(layer, strategy, micro_batch: int, stage_index: int, n_micro: int,
                 ms_multiplier: float) -> tuple[float, float, float]:
    pp = strategy.pp_degree
    if not 1 <= stage_index <= pp:
        raise ValueError(f"stage_index {stage_index} out of range 1..{pp}")
    if n_micro < 1:
        raise ValueError(f"n_micro must be >= 1, got {n_micro}")
    samples = _check_divisible(strategy, micro_batch)
    _, _, o_f, o_b, o_ms = _native_layer_cost(layer, strategy, micro_batch, _UNIT_CLUSTER, None,
                                              stage_index, n_micro, ms_multiplier)
    if strategy.ckpt:   # the reference returns O_f as a Python int here (costs.py:223)
        stash = min(pp - stage_index + 1, n_micro)
        o_f = stash * (layer.bnd_bytes_per_sample * samples)
    return o_f, o_b, o_ms


class _UnitCluster:
    n_devices = 1
    island_size = 1
    intra_island_bw = 1.0
    inter_island_bw = 1.0
    overlap_slowdown = 1.0


_UNIT_CLUSTER = _UnitCluster()


def layer_cost(layer, strategy, micro_batch: int, ctx: EvalContext, stage_index: int = 1,
               n_micro: int = 1) -> LayerCost:
    t, t_ns = _layer_times(layer, strategy, micro_batch, ctx.cluster, ctx.profile)
    o_f, o_b, o_ms = layer_memory(layer, strategy, micro_batch, stage_index, n_micro, ctx.ms_multiplier)
    return LayerCost(time_s=t, mem_fwd_bytes=o_f, mem_bwd_bytes=o_b, mem_states_bytes=o_ms,
                     time_no_sync_s=t_ns)


def transform_cost(layer, prev_strategy, cur_strategy, micro_batch: int, cluster) -> float:
    if prev_strategy is None:
        return 0.0
    out = ctypes.c_double()
    rc = _native.lib().gbmw_transform_cost(ctypes.byref(_c_layer(layer, layer.fwd_time_per_sample)),
                                           ctypes.byref(_c_strategy(prev_strategy)),
                                           ctypes.byref(_c_strategy(cur_strategy)), int(micro_batch),
                                           ctypes.byref(_c_env(cluster, None)), ctypes.byref(out))
    _native.raise_status(rc, _native.global_error())
    return out.value


def stage_p2p_time(first_layer, micro_batch: int, pp_degree: int, cluster) -> float:
    if pp_degree <= 1:
        return 0.0
    group = cluster.n_devices // pp_degree
    bw = cluster.inter_island_bw if group >= cluster.island_size else cluster.intra_island_bw
    return first_layer.bnd_bytes_per_sample * micro_batch / bw


# ----------------------------------------------------------------------------- per stage

def memory_footprint(layers, strategies, micro_batch: int, stage_index: int, n_micro: int,
                     ms_multiplier: float) -> tuple[float, float]:
    """(E_all, E_f): backward peak and forward footprint, layers in order (costs.py:289-319)."""
    if len(layers) != len(strategies):
        raise ValueError("layers and strategies must have equal length")
    if not layers:
        return 0.0, 0.0
    ms = pf = peak = 0.0
    for layer, s in zip(layers, strategies):
        o_f, o_b, o_ms = layer_memory(layer, s, micro_batch, stage_index, n_micro, ms_multiplier)
        ms += o_ms
        pf += o_f
        peak = max(peak, pf + o_b)
    return peak + ms, pf + ms


def stage_cost(layers, strategies, micro_batch: int, ctx: EvalContext, stage_index: int = 1,
               n_micro: int = 1) -> StageCost:
    if len(layers) != len(strategies):
        raise ValueError("layers and strategies must have equal length")
    if not layers:
        raise ValueError("stage must contain at least one layer")
    t_sum = ns_sum = 0.0
    prev = None
    for layer, s in zip(layers, strategies):
        t, t_ns = _layer_times(layer, s, micro_batch, ctx.cluster, ctx.profile)
        r = transform_cost(layer, prev, s, micro_batch, ctx.cluster)
        t_sum += t + r
        ns_sum += t_ns + r
        prev = s
    if stage_index > 1:
        p2p = stage_p2p_time(layers[0], micro_batch, strategies[0].pp_degree, ctx.cluster)
        t_sum += p2p
        ns_sum += p2p
    e_all, _ = memory_footprint(layers, strategies, micro_batch, stage_index, n_micro, ctx.ms_multiplier)
    return StageCost(time_s=t_sum, time_no_sync_s=ns_sum, peak_mem_bytes=e_all)


def pipeline_cost(stage_costs, n_micro: int) -> float:
    """C = (m - 1) * max_i C_no_sync(M_i) + sum_i C(M_i)  (costs.py:355-362)."""
    if not stage_costs:
        raise ValueError("pipeline must contain at least one stage")
    if n_micro < 1:
        raise ValueError(f"n_micro must be >= 1, got {n_micro}")
    return (n_micro - 1) * max(sc.time_no_sync_s for sc in stage_costs) + sum(sc.time_s for sc in stage_costs)


def pipeline_peak_memory(stage_costs) -> float:
    return max((sc.peak_mem_bytes for sc in stage_costs), default=0.0)
