"""CPU-side checks of libgbmw: it loads, exports every symbol include/gbmw.h
declares, and its host-side pieces (strategy enumeration, cost model) are
bit-exact against the reference's golden vectors.  No device calls."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from golden_cases import fh, load
from paper_2307_02031_b200 import _native
from paper_2307_02031_b200 import costs as C
from paper_2307_02031_b200 import strategies as ST
from paper_2307_02031_b200.specs import ClusterSpec, CostProfile, LayerSpec

HEADER = Path(__file__).resolve().parents[1] / "include" / "gbmw.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:char\s*\*|int|void|double)\s*\*?\s*(gbmw_\w+)\s*\(",
                                 text, re.M)))


def test_library_exports_every_header_symbol():
    L = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(L, name), name
    assert set(syms) == set(_native.EXPORTS)
    assert L.gbmw_abi_version() == 1
    assert b"sm_100a" in L.gbmw_version()


def test_enumeration_matches_reference_order():
    for key, expect in load("enumeration.json").items():
        n, p, kind = key.split(",")
        n, p = int(n), int(p)
        sset = ST.enumerate_pruned(n, p) if kind == "pruned" else ST.enumerate_strategies(n, p)
        assert [s.to_string() for s in sset] == expect, key


def test_strategy_counts():
    assert ST.count_strategies(8, prune=False) == {1: 42, 2: 18, 4: 6, 8: 2}
    assert ST.count_strategies(8, prune=True) == {1: 22, 2: 14, 4: 6, 8: 2}
    assert sum(ST.count_strategies(64).values()) == 158


def test_enumeration_rejects_non_powers_of_two():
    from paper_2307_02031_b200.errors import SpecError
    with pytest.raises(SpecError):
        ST.enumerate_strategies(6, 1)
    with pytest.raises(SpecError):
        ST.enumerate_strategies(8, 16)


def test_host_cost_model_bit_exact():
    for c in load("cost_cells.json"):
        lid, kind, p, b, n, f, fr = c["layer"]
        layer = LayerSpec(lid, kind, p, b, n, fh(f), fh(fr))
        env = c["env"]
        cl = ClusterSpec(env["n_devices"], 1, env["island_size"], fh(env["intra"]), fh(env["inter"]),
                         fh(env["slowdown"]))
        pr = CostProfile(fh(env["bwd_ratio"]), fh(env["coll_eff"]))
        s, prev = ST.parse_strategy(c["strategy"]), ST.parse_strategy(c["prev"])
        t, tns = C._layer_times(layer, s, c["micro"], cl, pr)
        o_f, o_b, o_ms = C.layer_memory(layer, s, c["micro"], c["stage"], c["n_micro"], fh(env["ms"]))
        g, a = C.comm_time(layer, s, c["micro"], cl, pr)
        got = [t, tns, o_f, o_b, o_ms, C.transform_cost(layer, prev, s, c["micro"], cl), g, a]
        assert [float(x).hex() for x in got] == c["out"], c
        assert isinstance(o_f, int) == c["o_f_is_int"]


def test_layer_memory_errors():
    layer = LayerSpec(0, "x", 64, 16, 32, 0.01)
    s = ST.ParallelStrategy(2, (("dp", 2),), False)
    with pytest.raises(ValueError):
        C.layer_memory(layer, s, 4, 3, 1, 4.0)
    from paper_2307_02031_b200.errors import DivisibilityError
    with pytest.raises(DivisibilityError):
        C.layer_memory(layer, s, 3, 1, 1, 4.0)


def test_sum_semantics_follow_the_interpreter():
    """The planner's folds use this interpreter's sum(): Neumaier since CPython 3.12, plain
    left-to-right before.  Both modes are selectable and reproduce the matching Python fold."""
    import sys
    L = _native.lib()
    assert L.gbmw_sum_semantics() == (1 if sys.version_info >= (3, 12) else 0)
    x = np.array([1e16, 1.0, -1e16, 3.0, 0.1, 0.2], dtype=np.float64)
    naive = 0
    for v in x.tolist():
        naive = naive + v
    saved = L.gbmw_sum_semantics()
    try:
        L.gbmw_set_sum_semantics(0)
        assert L.gbmw_py_sum(_native.ptr(x), len(x)).hex() == float(naive).hex()
        L.gbmw_set_sum_semantics(1)
        got = L.gbmw_py_sum(_native.ptr(x), len(x))
        if sys.version_info >= (3, 12):
            assert got.hex() == sum(x.tolist()).hex()
        assert got != naive                      # the compensated sum keeps the 1.0
    finally:
        L.gbmw_set_sum_semantics(saved)


def test_ptr_keeps_temporaries_alive():
    """_native.ptr of a temporary holds the array until the pointer object is dropped."""
    import gc
    p = _native.ptr(np.full(8, 7.0))
    gc.collect()
    junk = [np.zeros(8) for _ in range(64)]     # would reuse a freed 64-byte buffer
    assert ctypes.cast(p, ctypes.POINTER(ctypes.c_double))[3] == 7.0
    del junk


def test_mutable_strategy_lists_are_not_cached_by_identity():
    from paper_2307_02031_b200 import dpsearch as D
    sset = ST.enumerate_pruned(8, 1)
    assert D._frozen(sset) and D._frozen(tuple(sset))
    lst = list(sset)
    assert not D._frozen(lst)
    a = D._strategies_array_cached(lst, lst)
    lst.reverse()
    b = D._strategies_array_cached(lst, lst)
    assert len(a) == len(b) and not np.array_equal(a, b)
    m = D._Marshal()
    r0 = m.strat_range(lst, list(lst))
    lst.pop()
    r1 = m.strat_range(lst, list(lst))
    assert r0 != r1 and len(m.strats[r1]) == len(lst)
