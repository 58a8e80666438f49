"""Load the golden fixtures (tests/golden/*.json) into the flat records both the
oracle and libgbmw consume, and into package objects for API-level tests."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2307_02031_b200 import _native
from paper_2307_02031_b200.costs import EvalContext
from paper_2307_02031_b200.specs import ClusterSpec, CostProfile, LayerSpec, ModelSpec
from paper_2307_02031_b200.strategies import StrategySet, parse_strategy

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load(name: str):
    return json.loads((GOLDEN / name).read_text())


def fh(s: str) -> float:
    return float.fromhex(s)


def case_objects(case):
    """(layers, budget, StrategySet, ctx) as package objects."""
    layers = tuple(LayerSpec(i, k, p, b, n, fh(f), fh(fr)) for (i, k, p, b, n, f, fr) in case["layers"])
    env = case["env"]
    cluster = ClusterSpec(env["n_devices"], int(case["budget"]) if case["budget_is_int"] else 1, env["island_size"],
                          fh(env["intra"]), fh(env["inter"]), fh(env["slowdown"]))
    profile = CostProfile(fh(env["bwd_ratio"]), fh(env["coll_eff"]),
                          {int(k): fh(v) for k, v in env["overrides"].items()})
    model = ModelSpec("golden", layers, fh(env["ms"]))
    strats = tuple(parse_strategy(s) for s in case["strategies"])
    sset = StrategySet(group_size=1, strategies=strats)
    budget = case["budget"]
    return list(layers), budget, sset, EvalContext(model, cluster, profile)


def flat_batch(cases, stage_cost=True):
    """Flat (layers, strategies, envs, problems) records for a list of golden cases."""
    L, S, E, P = [], [], [], []
    kinds: dict = {}
    lo = so = 0
    for i, c in enumerate(cases):
        layers, budget, sset, ctx = case_objects(c)
        L.append(_native.layers_array(layers, ctx.profile, kinds))
        S.append(_native.strategies_array(list(sset)))
        E.append(_native.env_record(ctx))
        flags = (_native.FUSE if c["fuse"] else 0) | (_native.FRONTIER if c["collect_frontier"] else 0) | \
                (_native.STAGE_COST if stage_cost else 0) | (_native.APPROX if c.get("approx") else 0)
        nb = int(budget // c["gran"])
        P.append((lo, len(layers), so, len(sset), i, c["stage"], c["n_micro"], flags, c["micro"], c["gran"],
                  float(budget), nb))
        lo += len(layers)
        so += len(sset)
    return (np.concatenate(L), np.concatenate(S), np.array(E, dtype=_native.ENV_DT),
            np.array(P, dtype=_native.PROBLEM_DT))


def frontier_digest(vals) -> str:
    import hashlib
    h = hashlib.sha256()
    h.update(np.asarray(vals, dtype="<f8").tobytes())
    return h.hexdigest()


def check_case(case, res, plan, frontier_vals):
    """Assert one result record (RESULT_DT row) + plan slice + frontier slice equal the golden."""
    out = case["out"]
    name = case["name"]
    assert bool(res["feasible"]) == out["feasible"], name
    assert float(res["time_s"]).hex() == out["time"], (name, float(res["time_s"]).hex(), out["time"])
    assert float(res["e_fwd"]).hex() == out["e_fwd"], name
    if out["feasible"]:
        assert list(map(int, plan)) == out["plan"], (name, list(plan), out["plan"])
        got = [float(res["stage_time"]).hex(), float(res["stage_ns"]).hex(), float(res["stage_peak"]).hex()]
        assert got == out["stage"], (name, got, out["stage"])
    if "frontier_digest" in out and frontier_vals is not None:
        assert len(frontier_vals) == out["frontier_len"], name
        if "frontier" in out:
            assert [float(v).hex() for v in frontier_vals] == out["frontier"], name
        assert frontier_digest(frontier_vals) == out["frontier_digest"], name


def brute_objects(case):
    """(model, cluster, profile) package objects of a brute.json case."""
    from paper_2307_02031_b200.specs import load_cluster_spec, load_cost_profile, load_model_spec
    model = load_model_spec(case["model"])
    return model, load_cluster_spec(case["cluster"]), load_cost_profile(case["profile"], model)


def brute_records(model, cluster, profile):
    """(layers, env) records of a brute-force instance, as both libgbmw and the oracle take them."""
    ctx = EvalContext(model, cluster, profile)
    return (_native.layers_array(list(model.layers), profile, {}),
            np.array([_native.env_record(ctx)], dtype=_native.ENV_DT))
