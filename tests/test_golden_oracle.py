"""The oracle (oracle/ref_oracle.c) against the golden fixtures generated from the
live reference (tests/golden/make_golden.py): pins the CPU restatement before it
is trusted as the checker of the CUDA path."""

import numpy as np
import pytest

from golden_cases import check_case, flat_batch, load
from oracle import oracle as O
from paper_2307_02031_b200 import _native
from paper_2307_02031_b200.strategies import parse_strategy


def test_enumeration_matches_reference():
    for key, expect in load("enumeration.json").items():
        n, p, kind = key.split(",")
        recs = O.enumerate_records(int(n), int(p), kind == "pruned")
        got = [_strategy_string(r) for r in recs]
        assert got == expect, key


def _strategy_string(r):
    toks = [f"pp{int(r['pp_degree'])}"]
    for i in range(int(r["n_levels"])):
        toks.append(f"{_native.PARADIGM_NAME[int(r['paradigm'][i])]}{int(r['degree'][i])}")
    if r["ckpt"]:
        toks.append("ckpt")
    return "/".join(toks)


def test_cost_cells_match_reference():
    from golden_cases import fh
    for c in load("cost_cells.json"):
        _, kind, p, b, n, f, fr = c["layer"]
        layer = np.array([(p, b, n, fh(f), fh(f), fh(fr), 0)], dtype=_native.LAYER_DT)
        env = c["env"]
        e = np.array([(env["n_devices"], env["island_size"], fh(env["intra"]), fh(env["inter"]), fh(env["slowdown"]),
                       fh(env["bwd_ratio"]), fh(env["coll_eff"]), fh(env["ms"]))], dtype=_native.ENV_DT)
        s = _native.strategies_array([parse_strategy(c["strategy"])])
        got = O.cell(layer, s, e, c["micro"], c["stage"], c["n_micro"])
        assert [x.hex() for x in got] == c["out"][:5], c


@pytest.mark.parametrize("fixture", ["dp_fuzz.json", "dp_configs.json", "dp_approx.json"])
def test_dp_search_matches_reference(fixture):
    cases = load(fixture)
    layers, strats, envs, probs = flat_batch(cases)
    res, plans, front, _ = O.search_many(layers, strats, envs, probs)
    plan_off = front_off = 0
    for i, c in enumerate(cases):
        nl = int(probs["n_layers"][i])
        fv = None
        if c["collect_frontier"]:
            nb = int(probs["n_buckets"][i])
            fv = front[front_off:front_off + nb]
            front_off += nb
        check_case(c, res[i], plans[plan_off:plan_off + nl], fv)
        plan_off += nl
