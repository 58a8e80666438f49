"""ctypes wrapper of liboracle.so — TEST INFRASTRUCTURE ONLY.

The oracle is the CPU restatement of the reference search path (ref_oracle.c,
citing parapilot file:line per function).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs may import this module; the product package
never does.  It consumes the product's own input records (include/gbmw.h), so a
parity test feeds both sides identical bytes.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

RESULT_DT = np.dtype([("time_s", "<f8"), ("e_fwd", "<f8"), ("feasible", "<i4"), ("status", "<i4"),
                      ("stage_time", "<f8"), ("stage_ns", "<f8"), ("stage_peak", "<f8"),
                      ("frontier_off", "<i8")])
STRATEGY_DT = np.dtype([("pp_degree", "<i4"), ("n_levels", "<i4"), ("paradigm", "<i4", (3,)),
                        ("degree", "<i4", (3,)), ("ckpt", "<i4")])

_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < (HERE / "ref_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "-s"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB))
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.or_enumerate.argtypes = [i64, i64, ctypes.c_int, vp, ctypes.c_int]
        L.or_enumerate.restype = ctypes.c_int
        L.or_search_many.argtypes = [vp, vp, vp, vp, i64, vp, vp, vp, ctypes.c_int]
        L.or_search_many.restype = ctypes.c_int
        L.or_layer_times.argtypes = [vp, vp, i64, vp, vp, vp]
        L.or_layer_memory.argtypes = [vp, vp, i64, ctypes.c_int, ctypes.c_int, ctypes.c_double, vp]
        L.or_transform.argtypes = [vp, vp, vp, i64, vp]
        L.or_transform.restype = ctypes.c_double
        L.or_brute_force.argtypes = [vp, ctypes.c_int, vp, i64, ctypes.c_double, ctypes.c_int, vp, vp, vp]
        L.or_brute_force.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def enumerate_records(n_devices: int, pp: int, prune: bool) -> np.ndarray:
    L = lib()
    n = L.or_enumerate(n_devices, pp, int(prune), None, 0)
    if n < 0:
        raise ValueError("invalid device / pipeline degree")
    out = np.zeros(n, dtype=STRATEGY_DT)
    L.or_enumerate(n_devices, pp, int(prune), _p(out), n)
    return out


def search_many(layers, strats, envs, probs, n_threads: int | None = None):
    """Reference dp_search (+ stage_cost) for every problem; returns (results, plans, frontier, threads)."""
    n_plan = int(np.clip(probs["n_layers"], 0, None).sum()) if len(probs) else 0
    flagged = (probs["flags"] & 2) != 0
    n_front = int(probs["n_buckets"][flagged].sum()) if len(probs) else 0
    res = np.zeros(len(probs), dtype=RESULT_DT)
    plans = np.zeros(max(n_plan, 1), dtype=np.int32)
    front = np.zeros(max(n_front, 1), dtype=np.float64)
    threads = n_threads or len(os.sched_getaffinity(0))
    used = lib().or_search_many(_p(layers), _p(strats), _p(envs), _p(probs), len(probs), _p(res), _p(plans),
                                _p(front), int(threads))
    return res, plans, front, used


def cell(layer_rec, strat_rec, env_rec, micro, stage, n_micro):
    """(t, t_ns, O_f, O_b, O_ms) of one cell via the oracle's cost model."""
    L = lib()
    t, tns = ctypes.c_double(), ctypes.c_double()
    L.or_layer_times(_p(layer_rec), _p(strat_rec), int(micro), _p(env_rec), ctypes.byref(t), ctypes.byref(tns))
    m = (ctypes.c_double * 3)()
    L.or_layer_memory(_p(layer_rec), _p(strat_rec), int(micro), int(stage), int(n_micro),
                      float(env_rec["ms"][0] if env_rec.shape else env_rec["ms"]), m)
    return (t.value, tns.value, m[0], m[1], m[2])


def brute_force(layers, env, batch: int, budget: float, neumaier: bool = True):
    """planner.brute_force_oracle restated (or_brute_force): (cost, feasible, P, m, partition, choice)."""
    L = len(layers)
    part = np.zeros(max(L, 1), dtype=np.int32)
    choice = np.full(max(L, 1), -1, dtype=np.int32)
    out = np.zeros(5, dtype=np.float64)
    rc = lib().or_brute_force(_p(layers), L, _p(env), int(batch), float(budget), int(neumaier), _p(part),
                              _p(choice), _p(out))
    if rc != 0:
        raise ValueError("or_brute_force: bad input")
    n_st = int(out[4])
    return (float(out[0]), bool(out[1]), int(out[2]), int(out[3]), tuple(int(x) for x in part[:n_st]),
            tuple(int(x) for x in choice[:L]) if out[1] else ())
