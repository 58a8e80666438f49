"""Seed partitions on the device (gbmw_seed_partitions_device) against
the reference's golden partitions and against the host restatement, cell by cell.
Needs a B200 (-m gpu)."""

from __future__ import annotations

import pytest

from golden_cases import load
from paper_2307_02031_b200 import _native, balance as B, workloads as W
from paper_2307_02031_b200.planner import init_microbatch_num
from paper_2307_02031_b200.strategies import candidate_pp_degrees

pytestmark = pytest.mark.gpu


def test_device_seed_partitions_match_reference(gpu):
    by_model = {}
    for c in load("partitions.json"):
        by_model.setdefault((c["model"], c["budget"]), []).append(c)
    dev = _native.default_context()
    for (name, budget), cases in by_model.items():
        ctx = W.config(name, budget)
        cells = [(c["P"], c["micro"], c["n_micro"]) for c in cases]
        parts = B.seed_partitions(ctx.model, ctx, ctx.cluster.n_devices, cells, device=dev)
        assert [list(p.stage_sizes) for p in parts] == [c["p_m"] for c in cases], name


@pytest.mark.parametrize("name", ["bert", "t5", "swin", "vit", "gpt"])
def test_device_seed_partitions_equal_host(gpu, name):
    ctx = W.config(name)
    cells = []
    for b in list(range(8, 520, 8)) + [1024, 2048, 4096]:
        for p in candidate_pp_degrees(ctx.cluster.n_devices):
            if p <= ctx.model.num_layers:
                m = init_microbatch_num(b, p)
                cells.append((p, b // m, m))
    dev = B.seed_partitions(ctx.model, ctx, ctx.cluster.n_devices, cells, device=_native.default_context())
    host = B.seed_partitions(ctx.model, ctx, ctx.cluster.n_devices, cells)
    assert dev == host
