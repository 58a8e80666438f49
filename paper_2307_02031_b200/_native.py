"""ctypes binding of libgbmw.so (include/gbmw.h) and the struct layouts it shares.

There is no Python fallback: if the shared library is missing every entry point
raises ``ImportError`` (build it with ``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_2307_02031_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
import sys
import threading
from pathlib import Path

import numpy as np

from .errors import DivisibilityError, NativeError

LIB_PATH = Path(__file__).resolve().parent / "libgbmw.so"

# status codes (gbmw.h)
OK = 0
EINVAL_GRAN, EINVAL_BUDGET, EEMPTY, EMICRO, EBUCKETS = -1, -2, -3, -4, -5
ECUDA, ENOMEM, EINVAL, ERANGE, ENOTSUP, EINTERNAL, ESTAGE = -6, -7, -8, -9, -10, -11, -12
MAX_BUCKETS = 1_000_000

FUSE, FRONTIER, STAGE_COST, APPROX = 1, 2, 4, 8
PARADIGM_CODE = {"dp": 0, "sdp": 1, "tp": 2}
PARADIGM_NAME = ("dp", "sdp", "tp")

STRATEGY_DT = np.dtype([("pp_degree", "<i4"), ("n_levels", "<i4"), ("paradigm", "<i4", (3,)),
                        ("degree", "<i4", (3,)), ("ckpt", "<i4")])
LAYER_DT = np.dtype([("param_bytes", "<i8"), ("bnd", "<i8"), ("intb", "<i8"), ("fwd", "<f8"),
                     ("fwd_raw", "<f8"), ("frac", "<f8"), ("kind", "<i8")])
ENV_DT = np.dtype([("n_devices", "<i8"), ("island", "<i8"), ("intra", "<f8"), ("inter", "<f8"),
                   ("slowdown", "<f8"), ("bwd_ratio", "<f8"), ("coll_eff", "<f8"), ("ms", "<f8")])
PROBLEM_DT = np.dtype([("layer_begin", "<i4"), ("n_layers", "<i4"), ("strat_begin", "<i4"),
                       ("n_strats", "<i4"), ("env_index", "<i4"), ("stage_index", "<i4"),
                       ("n_micro", "<i4"), ("flags", "<i4"), ("micro", "<i8"), ("gran", "<i8"),
                       ("budget", "<f8"), ("n_buckets", "<i8")])
RESULT_DT = np.dtype([("time_s", "<f8"), ("e_fwd", "<f8"), ("feasible", "<i4"), ("status", "<i4"),
                      ("stage_time", "<f8"), ("stage_ns", "<f8"), ("stage_peak", "<f8"),
                      ("frontier_off", "<i8")])
assert STRATEGY_DT.itemsize == 36 and LAYER_DT.itemsize == 56 and ENV_DT.itemsize == 64
assert PROBLEM_DT.itemsize == 64 and RESULT_DT.itemsize == 56


class Timing(ctypes.Structure):
    _fields_ = [("total_ms", ctypes.c_float), ("dp_ms", ctypes.c_float), ("sweep_ms", ctypes.c_float),
                ("tables_ms", ctypes.c_float), ("finalize_ms", ctypes.c_float),
                ("n_chunks", ctypes.c_int32), ("n_launches", ctypes.c_int32),
                ("transitions", ctypes.c_double), ("row_steps", ctypes.c_double),
                ("dp_bytes", ctypes.c_double), ("dp_cells", ctypes.c_double),
                ("h2d_bytes", ctypes.c_double), ("d2h_bytes", ctypes.c_double),
                ("prep_ms", ctypes.c_double), ("upload_ms", ctypes.c_double), ("fetch_ms", ctypes.c_double),
                ("live_cells", ctypes.c_double), ("sweep_rows", ctypes.c_double),
                ("sweep_cands", ctypes.c_double), ("sweep_checks", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class OracleRecord(ctypes.Structure):
    """gbmw_oracle_result (gbmw.h)."""
    _fields_ = [("cost", ctypes.c_double), ("feasible", ctypes.c_int32), ("pp_degree", ctypes.c_int32),
                ("n_micro", ctypes.c_int32), ("n_stages", ctypes.c_int32), ("combos", ctypes.c_double),
                ("device_ms", ctypes.c_double)]


EXPORTS = (
    "gbmw_version", "gbmw_abi_version", "gbmw_limits", "gbmw_ctx_create", "gbmw_ctx_destroy",
    "gbmw_last_error", "gbmw_last_error_global", "gbmw_ctx_stream", "gbmw_enumerate", "gbmw_layer_cost",
    "gbmw_transform_cost", "gbmw_comm_breakdown", "gbmw_cost_tables", "gbmw_search_batch", "gbmw_batch_create",
    "gbmw_batch_run", "gbmw_batch_fetch", "gbmw_batch_timing", "gbmw_ctx_last_timing", "gbmw_batch_destroy",
    "gbmw_partition_costs", "gbmw_init_partition", "gbmw_seed_for", "gbmw_seed_partitions", "gbmw_seed_partitions_device", "gbmw_bmw_setup", "gbmw_partition_costs_batch", "gbmw_py_sum", "gbmw_planner_last_error",
    "gbmw_set_sum_semantics", "gbmw_sum_semantics", "gbmw_brute_force",
)

_lib = None
_lib_lock = threading.RLock()


def lib() -> ctypes.CDLL:
    """Load libgbmw.so (once).  Raises ImportError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            path = Path(os.environ.get("GBMW_LIB", LIB_PATH))
            if not path.exists():
                raise ImportError(f"libgbmw.so not found at {path}: build the CUDA extension first "
                                  f"(make -C paper_2307_02031_b200/csrc); there is no CPU fallback")
            L = ctypes.CDLL(str(path))
            vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
            L.gbmw_version.restype = ctypes.c_char_p
            L.gbmw_abi_version.restype = ctypes.c_int
            L.gbmw_last_error.restype = ctypes.c_char_p
            L.gbmw_last_error.argtypes = [vp]
            L.gbmw_last_error_global.restype = ctypes.c_char_p
            L.gbmw_limits.argtypes = [vp, vp, vp]
            L.gbmw_ctx_create.argtypes = [i32, u64, ctypes.POINTER(vp)]
            L.gbmw_ctx_destroy.argtypes = [vp]
            L.gbmw_ctx_stream.argtypes = [vp]
            L.gbmw_ctx_stream.restype = vp
            L.gbmw_enumerate.argtypes = [i64, i64, i32, vp, i32, vp]
            L.gbmw_layer_cost.argtypes = [vp, vp, vp, i64, i32, i32, vp]
            L.gbmw_transform_cost.argtypes = [vp, vp, vp, i64, vp, vp]
            L.gbmw_comm_breakdown.argtypes = [vp, vp, vp, i64, vp]
            L.gbmw_cost_tables.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp]
            L.gbmw_search_batch.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, i64, vp, vp, vp]
            L.gbmw_batch_create.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, i64, ctypes.POINTER(vp)]
            L.gbmw_batch_run.argtypes = [vp, vp]
            L.gbmw_batch_fetch.argtypes = [vp, vp, vp, vp, vp]
            L.gbmw_batch_timing.argtypes = [vp, ctypes.POINTER(Timing)]
            L.gbmw_ctx_last_timing.argtypes = [vp, ctypes.POINTER(Timing)]
            L.gbmw_batch_destroy.argtypes = [vp]
            L.gbmw_partition_costs.argtypes = [vp, i32, vp, vp, i32, vp, i64, i32, vp]
            L.gbmw_init_partition.argtypes = [vp, i32, vp, i32, vp, i64, i32, i32, vp]
            L.gbmw_seed_for.argtypes = [vp, i32, vp, i64, i64, i64, i32, ctypes.c_double, vp, vp]
            L.gbmw_seed_partitions.argtypes = [vp, i32, vp, i64, i32, vp, vp, vp, ctypes.c_double, i32, i32, vp]
            L.gbmw_seed_partitions_device.argtypes = [vp, vp, i32, vp, i64, i32, vp, vp, vp, ctypes.c_double, i32, vp]
            L.gbmw_bmw_setup.argtypes = [vp, i32, vp, i64, i32, vp, vp, vp, ctypes.c_double, i32, i32, vp, vp]
            L.gbmw_partition_costs_batch.argtypes = [vp, i32, vp, vp, vp, i32, vp, vp, vp, i32, i32, vp]
            L.gbmw_py_sum.argtypes = [vp, i32]
            L.gbmw_py_sum.restype = ctypes.c_double
            L.gbmw_planner_last_error.restype = ctypes.c_char_p
            L.gbmw_set_sum_semantics.argtypes = [i32]
            L.gbmw_brute_force.argtypes = [vp, vp, i32, vp, i64, ctypes.c_double, ctypes.c_double, vp, vp,
                                           ctypes.POINTER(OracleRecord)]
            for name in EXPORTS:
                getattr(L, name).restype = getattr(L, name).restype or ctypes.c_int
            # the planner's folds follow this interpreter's built-in sum(): Neumaier-compensated
            # since CPython 3.12, plain left-to-right before (the reference's balance.py:62-77,125)
            L.gbmw_set_sum_semantics(1 if sys.version_info >= (3, 12) else 0)
            _lib = L
    return _lib


def ptr(a: np.ndarray | None):
    """Address of ``a`` for a ctypes call; the returned pointer object holds a reference to
    the array, so a temporary passed inline stays alive for the duration of the call."""
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def global_error() -> str:
    msg = lib().gbmw_last_error_global()
    return msg.decode() if msg else ""


class Context:
    """One CUDA stream + device workspace (gbmw_ctx).  Calls on a context are serialised."""

    def __init__(self, device: int = -1, workspace_bytes: int = 0):
        L = lib()
        h = ctypes.c_void_p()
        rc = L.gbmw_ctx_create(int(device), int(workspace_bytes), ctypes.byref(h))
        if rc != OK:
            raise NativeError(f"gbmw_ctx_create failed ({rc}): {global_error()}")
        self.handle = h
        self.lock = threading.Lock()

    def stream_ptr(self) -> int:
        """cudaStream_t of this context (for torch.cuda.ExternalStream / event timing)."""
        return int(lib().gbmw_ctx_stream(self.handle) or 0)

    def error(self) -> str:
        msg = lib().gbmw_last_error(self.handle)
        return msg.decode() if msg else ""

    def close(self):
        if self.handle:
            with self.lock:                 # after a call in progress on another thread (e.g. the
                if self.handle:             # planner's speculative device pass)
                    lib().gbmw_ctx_destroy(self.handle)
                    self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_ctx: Context | None = None


def default_context() -> Context:
    global _ctx
    if _ctx is None:
        with _lib_lock:
            if _ctx is None:
                _ctx = Context(-1, int(os.environ.get("GBMW_WORKSPACE_BYTES", "0")))
    return _ctx


# ----------------------------------------------------------------------------- marshalling

def strategy_record(s) -> tuple:
    levels = tuple(s.levels)
    par = [0, 0, 0]
    deg = [1, 1, 1]
    for i, (p, d) in enumerate(levels):
        par[i] = PARADIGM_CODE[p]
        deg[i] = int(d)
    return (int(s.pp_degree), len(levels), par, deg, 1 if s.ckpt else 0)


_records: dict = {}


def strategies_array(strats) -> np.ndarray:
    """STRATEGY_DT records of a strategy sequence.  A strategy's record bytes are built once
    per object (strategies are frozen dataclasses; the cached entry keeps the object alive, so
    its id cannot be reused while cached) and the array is one join of them."""
    parts = []
    cache = _records
    for s in strats:
        hit = cache.get(id(s))
        if hit is None or hit[0] is not s:
            if len(cache) > 8192:
                cache.clear()
            hit = (s, np.array([strategy_record(s)], dtype=STRATEGY_DT).tobytes())
            cache[id(s)] = hit
        parts.append(hit[1])
    return np.frombuffer(bytearray(b"".join(parts)), dtype=STRATEGY_DT)


def _i64(v, what):
    v = int(v)
    if not -(1 << 63) <= v < (1 << 63):
        raise ValueError(f"{what} {v} does not fit in 64 bits")
    return v


def layers_array(layers, profile, kinds: dict) -> np.ndarray:
    out = np.zeros(len(layers), dtype=LAYER_DT)
    for i, l in enumerate(layers):
        fwd = profile.fwd_time(l) if hasattr(profile, "fwd_time") else l.fwd_time_per_sample
        out[i] = (_i64(l.param_bytes, "param_bytes"), _i64(l.bnd_bytes_per_sample, "bnd_bytes_per_sample"),
                  _i64(l.int_bytes_per_sample, "int_bytes_per_sample"), float(fwd),
                  float(l.fwd_time_per_sample), float(l.tp_act_replication_fraction),
                  kinds.setdefault(l.kind, len(kinds)))
    return out


def env_record(ctx) -> tuple:
    c, p = ctx.cluster, ctx.profile
    ms = ctx.ms_multiplier if hasattr(ctx, "ms_multiplier") else ctx.model.ms_bytes_per_param_byte
    return (int(c.n_devices), int(c.island_size), float(c.intra_island_bw), float(c.inter_island_bw),
            float(c.overlap_slowdown), float(p.bwd_fwd_ratio), float(p.collective_efficiency), float(ms))


def env_array(ctxs) -> np.ndarray:
    out = np.zeros(len(ctxs), dtype=ENV_DT)
    for i, c in enumerate(ctxs):
        out[i] = env_record(c)
    return out


def raise_status(rc: int, msg: str):
    """Map a gbmw status to the exception class the reference raises."""
    if rc == OK:
        return
    if rc == EMICRO:
        raise DivisibilityError(msg)
    if rc in (EINVAL_GRAN, EINVAL_BUDGET, EEMPTY, EBUCKETS, ESTAGE, ERANGE, EINVAL):
        raise ValueError(msg)
    if rc == EINTERNAL:
        raise AssertionError(msg or "dp_search produced a plan exceeding the memory budget")
    raise NativeError(f"libgbmw error {rc}: {msg}")
