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
