"""Synthetic model / cluster specs of the benchmark configurations.

Layer byte sizes and times are the fixed values SURVEY.md §8(d) derives from the
paper; no random floats enter the cost model.
``sweep_problems`` is the 10k independent-stage-search generator of
BASELINE.json config 5.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

from .costs import EvalContext
from .specs import ClusterSpec, CostProfile, ModelSpec, load_cluster_spec, load_model_spec
from .strategies import candidate_pp_degrees

GiB = 1 << 30
MiB = 1 << 20


def _model(name, layer_rows):
    return load_model_spec({
        "name": name,
        "ms_bytes_per_param_byte": 4.0,
        "layers": [{"kind": k, "param_bytes": p, "bnd_bytes_per_sample": b, "int_bytes_per_sample": i,
                    "fwd_time_per_sample": f} for (k, p, b, i, f) in layer_rows],
    })


def bert_huge_32() -> ModelSpec:
    return _model("bert-huge-32", [("enc", 84_000_000, 10_485_760, 92_274_688, 0.0045)] * 32)


def t5_large_48() -> ModelSpec:
    return _model("t5-large-48", [("enc", 50_331_648, 8_388_608, 98_566_144, 0.0030)] * 24 +
                  [("dec", 67_108_864, 8_388_608, 151_519_232, 0.0042)] * 24)


def vit_huge_32() -> ModelSpec:
    return _model("vit-huge-32", [("enc", 79_000_000, 1_310_720, 19_890_176, 0.0011)] * 32)


def swin_huge_48() -> ModelSpec:
    rows = []
    for stage, (blocks, h, tokens) in enumerate(((2, 320, 3136), (2, 640, 784), (42, 1280, 196), (2, 2560, 49))):
        bnd = tokens * h * 4
        rows += [(f"swin{stage}", 12 * h * h * 4, bnd, 18 * bnd, 0.0012)] * blocks
    return _model("swin-huge-48", rows)


def gpt3_96() -> ModelSpec:
    h, s, a = 12288, 2048, 96
    return _model("gpt3-96", [("dec", 12 * h * h * 4, s * h * 2, 34 * s * h + 5 * a * s * s, 0.0476)] * 96)


def cluster_8(budget_bytes: int = 16 * GiB) -> ClusterSpec:
    return load_cluster_spec({"n_devices": 8, "mem_budget_bytes": budget_bytes, "island_size": 8,
                              "intra_island_bw": 12e9, "inter_island_bw": 10e9, "overlap_slowdown": 1.3})


def cluster_64(budget_bytes: int = 80 * GiB) -> ClusterSpec:
    return load_cluster_spec({"n_devices": 64, "mem_budget_bytes": budget_bytes, "island_size": 8,
                              "intra_island_bw": 300e9, "inter_island_bw": 50e9, "overlap_slowdown": 1.3})


MODELS = {
    "bert": bert_huge_32,
    "t5": t5_large_48,
    "vit": vit_huge_32,
    "swin": swin_huge_48,
    "gpt": gpt3_96,
}


def config(name: str, budget_bytes: int | None = None) -> EvalContext:
    """EvalContext of a named benchmark model on its cluster (GPT: 64 devices, others: 8)."""
    model = MODELS[name]()
    if name == "gpt":
        cluster = cluster_64(budget_bytes or 80 * GiB)
    else:
        cluster = cluster_8(budget_bytes or 16 * GiB)
    return EvalContext(model=model, cluster=cluster, profile=CostProfile())


def even_partition(n_layers: int, n_stages: int) -> tuple[int, ...]:
    """stage i gets L // P + [i < L mod P] layers."""
    q, r = divmod(n_layers, n_stages)
    return tuple(q + (1 if i < r else 0) for i in range(n_stages))


def microbatch_num(batch: int, pp_degree: int, cap_factor: int = 4, min_micro_size: int = 1) -> int:
    """planner.py:110-125 init_microbatch_num."""
    if batch < 1:
        raise ValueError(f"batch must be >= 1, got {batch}")
    if pp_degree <= 1:
        return 1
    for m in range(min(cap_factor * pp_degree, batch), 0, -1):
        if batch % m == 0 and batch // m >= min_micro_size:
            return m
    return 1


@dataclass(frozen=True)
class SweepCell:
    model: str
    budget_bytes: int
    pp_degree: int
    batch: int
    n_micro: int
    partition: tuple[int, ...]


def sweep_cells(n_stage_searches: int = 10_000, seed: int = 20261017) -> list[SweepCell]:
    """BASELINE config 5: random (model, P, B, budget) cells, even partitions, one stage
    search per stage, until ``n_stage_searches`` searches have been drawn."""
    rng = random.Random(seed)
    names = list(MODELS)
    n_layers = {n: MODELS[n]().num_layers for n in names}
    cells, total = [], 0
    while total < n_stage_searches:
        name = rng.choice(names)
        n_dev = 64 if name == "gpt" else 8
        p = rng.choice([x for x in candidate_pp_degrees(n_dev) if x <= n_layers[name]])
        batch = 8 * rng.randint(1, 64)
        budget = 80 * GiB if name == "gpt" else rng.choice((8, 12, 16, 20)) * GiB
        take = min(p, n_stage_searches - total)
        cells.append(SweepCell(name, budget, p, batch, microbatch_num(batch, p),
                               even_partition(n_layers[name], p)[:take]))
        total += take
    return cells


def sweep_arrays(cells: list[SweepCell], granularity_bytes: int = MiB, flags: int | None = None):
    """Flat C-ABI records (layers, strategies, envs, problems) of a list of sweep cells.

    Layer tables are shared per model, strategy tables per (N, P), envs per cluster;
    one problem per stage (stage_index = i + 1, n_micro = m, micro = B // m).
    Returns also the per-problem algorithmic transition count (U-1)*n_e*S^2.
    """
    import numpy as np

    from . import _native
    from .strategies import enumerate_pruned

    if flags is None:
        flags = _native.STAGE_COST
    kinds: dict = {}
    layer_blocks, layer_off, total_l = [], {}, 0
    strat_blocks, strat_off, strat_list, total_s = [], {}, {}, 0
    envs, env_idx = [], {}
    rows, trans = [], []
    for c in cells:
        ctx = config(c.model, c.budget_bytes)
        if c.model not in layer_off:
            arr = _native.layers_array(ctx.model.layers, ctx.profile, kinds)
            layer_off[c.model] = total_l
            layer_blocks.append(arr)
            total_l += len(arr)
        n_dev = ctx.cluster.n_devices
        if n_dev not in env_idx:
            env_idx[n_dev] = len(envs)
            envs.append(_native.env_record(ctx))
        key = (n_dev, c.pp_degree)
        if key not in strat_off:
            ss = list(enumerate_pruned(n_dev, c.pp_degree))
            strat_off[key] = total_s
            strat_list[key] = ss
            strat_blocks.append(_native.strategies_array(ss))
            total_s += len(ss)
        micro = c.batch // c.n_micro
        S = sum(1 for s in strat_list[key] if micro % s.data_degree == 0)
        n_b = c.budget_bytes // granularity_bytes
        start = 0
        for i, n in enumerate(c.partition):
            rows.append((layer_off[c.model] + start, n, strat_off[key], len(strat_list[key]), env_idx[n_dev], i + 1,
                         c.n_micro, flags, micro, granularity_bytes, float(c.budget_bytes), n_b))
            trans.append(float(n - 1) * (n_b + 1) * S * S if S and n_b else 0.0)
            start += n
    return (np.concatenate(layer_blocks), np.concatenate(strat_blocks), np.array(envs, dtype=_native.ENV_DT),
            np.array(rows, dtype=_native.PROBLEM_DT), np.array(trans))
