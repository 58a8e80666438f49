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


def test_brute_force_matches_reference():
    """or_brute_force (planner.py:364-449 restated) on the 200 golden instances."""
    from golden_cases import brute_objects, brute_records
    from paper_2307_02031_b200.strategies import enumerate_pruned
    for c in load("brute.json")["cases"]:
        model, cluster, profile = brute_objects(c)
        layers, env = brute_records(model, cluster, profile)
        cost, feas, P, m, part, choice = O.brute_force(layers, env, c["batch"], cluster.mem_budget_bytes)
        out = c["out"]
        assert feas == out["feasible"] and cost.hex() == out["cost"], (c["name"], cost.hex(), out)
        if feas:
            sset = enumerate_pruned(cluster.n_devices, P).strategies
            assert (P, m, list(part)) == (out["pp_degree"], out["n_micro"], out["partition"]), c["name"]
            assert [sset[j].to_string() for j in choice] == out["strategies"], c["name"]


def test_brute_force_guards():
    """The reference's size guards (planner.py:377-380) raise before any device work."""
    from golden_cases import brute_objects
    from paper_2307_02031_b200 import brute_force_oracle
    c = next(c for c in load("brute.json")["cases"] if len(c["model"]["layers"]) == 5)
    model, cluster, profile = brute_objects(c)
    with pytest.raises(ValueError, match="oracle limited to 4 layers, got 5"):
        brute_force_oracle(model, cluster, profile, c["batch"])
    c = next(c for c in load("brute.json")["cases"] if c["cluster"]["n_devices"] == 8)
    model, cluster, profile = brute_objects(c)
    with pytest.raises(ValueError, match="oracle limited to 4 devices, got 8"):
        brute_force_oracle(model, cluster, profile, c["batch"], max_layers=8)
