"""Hybrid-parallel strategy space (decision trees over DP / SDP / TP + CKPT).

Types and names follow parapilot/strategies.py:28-230.  The enumeration itself
(``enumerate_strategies``) runs in the native library (gbmw_enumerate), which
reproduces the reference's canonical ``sort_key`` order; this module only wraps
the records in ``ParallelStrategy`` objects.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from functools import lru_cache
from itertools import permutations

import numpy as np

from . import _native
from .errors import SpecError
from .specs import ClusterSpec, is_power_of_two

DP = "dp"
SDP = "sdp"
TP = "tp"
PARADIGMS = (DP, SDP, TP)

Level = tuple[str, int]


@dataclass(frozen=True)
class ParallelStrategy:
    """Ordered (paradigm, degree) levels, outermost first, plus activation checkpointing."""

    pp_degree: int
    levels: tuple[Level, ...]
    ckpt: bool

    def degree(self, paradigm: str) -> int:
        out = 1
        for p, d in self.levels:
            if p == paradigm:
                out *= d
        return out

    @property
    def dp_degree(self) -> int:
        return self.degree(DP)

    @property
    def sdp_degree(self) -> int:
        return self.degree(SDP)

    @property
    def tp_degree(self) -> int:
        return self.degree(TP)

    @property
    def data_degree(self) -> int:
        return self.dp_degree * self.sdp_degree

    @property
    def group_size(self) -> int:
        return math.prod(d for _, d in self.levels)

    def sort_key(self) -> tuple:
        return (len(self.levels), tuple(p for p, _ in self.levels),
                tuple(d for _, d in self.levels), self.ckpt)

    def to_string(self, cluster: ClusterSpec | None = None) -> str:
        tokens = [f"pp{self.pp_degree}"]
        for idx, (p, d) in enumerate(self.levels):
            tok = f"{p}{d}"
            if cluster is not None:
                below = math.prod(dd for _, dd in self.levels[idx:])
                tok += "@island" if below <= cluster.island_size else "@cross"
            tokens.append(tok)
        if self.ckpt:
            tokens.append("ckpt")
        return "/".join(tokens)

    def __str__(self) -> str:
        return self.to_string()


@dataclass(frozen=True)
class StrategySet:
    group_size: int
    strategies: tuple[ParallelStrategy, ...]

    def __len__(self) -> int:
        return len(self.strategies)

    def __iter__(self):
        return iter(self.strategies)


def parse_strategy(text: str) -> ParallelStrategy:
    """Inverse of ``to_string``; tier annotations are ignored, degree-1 levels skipped."""
    parts = [t for t in text.strip().split("/") if t]
    if not parts or not parts[0].startswith("pp"):
        raise SpecError(f"strategy string must start with 'pp<degree>': {text!r}")
    try:
        pp = int(parts[0][2:])
    except ValueError:
        raise SpecError(f"bad pipeline degree in strategy string: {text!r}") from None
    if not is_power_of_two(pp):
        raise SpecError(f"pipeline degree must be a power of two: {text!r}")
    levels: list[Level] = []
    ckpt = False
    for raw in parts[1:]:
        tok = raw.split("@", 1)[0]
        if tok in ("ckpt", "nockpt"):
            ckpt = tok == "ckpt"
            continue
        paradigm = next((p for p in PARADIGMS if tok.startswith(p)), None)
        if paradigm is None:
            raise SpecError(f"unknown token {tok!r} in strategy string {text!r}")
        try:
            deg = int(tok[len(paradigm):])
        except ValueError:
            raise SpecError(f"bad level token {tok!r} in {text!r}") from None
        if deg == 1:
            continue
        if not is_power_of_two(deg):
            raise SpecError(f"level degree must be a power of two: {tok!r}")
        if any(p == paradigm for p, _ in levels):
            raise SpecError(f"paradigm {paradigm!r} repeated in {text!r}")
        levels.append((paradigm, deg))
    return ParallelStrategy(pp_degree=pp, levels=tuple(levels), ckpt=ckpt)


def _compositions_pow2(group: int, max_levels: int = 3) -> list[tuple[int, ...]]:
    """Ordered factorisations of ``group`` into powers of two >= 2 (at most 3 levels)."""
    if group == 1:
        return [()]
    out: list[tuple[int, ...]] = []

    # depth-first in ascending-factor order, like strategies.py:155-165
    def rec(rem, prefix):
        if rem == 1:
            out.append(prefix)
            return
        if len(prefix) >= max_levels:
            return
        f = 2
        while f <= rem:
            if rem % f == 0:
                rec(rem // f, prefix + (f,))
            f *= 2

    rec(group, ())
    return out


def build_decision_trees(group_size: int) -> list[tuple[Level, ...]]:
    if not is_power_of_two(group_size):
        raise SpecError(f"group size must be a power of two, got {group_size}")
    shapes: list[tuple[Level, ...]] = []
    for factors in _compositions_pow2(group_size):
        if not factors:
            shapes.append(())
            continue
        shapes.extend(tuple(zip(labels, factors)) for labels in permutations(PARADIGMS, len(factors)))
    return shapes


def _from_record(rec) -> ParallelStrategy:
    n = int(rec["n_levels"])
    levels = tuple((_native.PARADIGM_NAME[int(rec["paradigm"][i])], int(rec["degree"][i])) for i in range(n))
    return ParallelStrategy(pp_degree=int(rec["pp_degree"]), levels=levels, ckpt=bool(rec["ckpt"]))


@lru_cache(maxsize=256)
def _enumerate_native(n_devices: int, pp_degree: int, prune: bool) -> tuple[ParallelStrategy, ...]:
    L = _native.lib()
    cnt = ctypes.c_int32(0)
    rc = L.gbmw_enumerate(n_devices, pp_degree, int(prune), None, 0, ctypes.byref(cnt))
    if rc != _native.OK:
        raise SpecError(_native.global_error())
    buf = np.zeros(cnt.value, dtype=_native.STRATEGY_DT)
    rc = L.gbmw_enumerate(n_devices, pp_degree, int(prune), _native.ptr(buf), cnt.value, ctypes.byref(cnt))
    if rc != _native.OK:
        raise SpecError(_native.global_error())
    return tuple(_from_record(r) for r in buf)


def enumerate_strategies(n_devices: int, pp_degree: int) -> StrategySet:
    """All decision-tree strategies for N/P devices (ckpt off and on), canonical order."""
    if not is_power_of_two(n_devices):
        raise SpecError(f"device count must be a power of two, got {n_devices}")
    if not is_power_of_two(pp_degree):
        raise SpecError(f"pipeline degree must be a power of two, got {pp_degree}")
    if pp_degree > n_devices or n_devices % pp_degree:
        raise SpecError(f"pipeline degree {pp_degree} does not divide device count {n_devices}")
    return StrategySet(group_size=n_devices // pp_degree,
                       strategies=_enumerate_native(n_devices, pp_degree, False))


def enumerate_pruned(n_devices: int, pp_degree: int) -> StrategySet:
    """prune_dp_sdp(enumerate_strategies(N, P)) in one native call."""
    enumerate_strategies(n_devices, pp_degree)  # same validation / messages
    return StrategySet(group_size=n_devices // pp_degree,
                       strategies=_enumerate_native(n_devices, pp_degree, True))


def prune_dp_sdp(strategy_set: StrategySet) -> StrategySet:
    """Takeaway #3: drop strategies that mix DP and SDP."""
    keep = tuple(s for s in strategy_set.strategies if not (s.degree(DP) > 1 and s.degree(SDP) > 1))
    return StrategySet(group_size=strategy_set.group_size, strategies=keep)


def candidate_pp_degrees(n_devices: int) -> list[int]:
    out, p = [], 1
    while p <= n_devices:
        out.append(p)
        p *= 2
    return out


def count_strategies(n_devices: int, prune: bool = True) -> dict[int, int]:
    return {p: len(enumerate_pruned(n_devices, p) if prune else enumerate_strategies(n_devices, p))
            for p in candidate_pp_degrees(n_devices)}
