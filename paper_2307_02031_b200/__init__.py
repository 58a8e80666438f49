"""paper_2307_02031_b200 — B200-native Galvatron-BMW planner search hot path.

Drop-in for the search path of the reference package ``parapilot``: the same
public names and signatures (strategy enumeration, cost model, ``dp_search``,
``galvatron_search`` / ``galvatron_base`` / ``plan_full`` /
``bi_objective_optimize``), computed by libgbmw (C++ host + sm_100a kernels).
"""

from .errors import (
    DivisibilityError,
    InfeasiblePlanError,
    NativeError,
    SpecError,
    UnsupportedDeviceCountError,
)
from .specs import (
    ClusterSpec,
    CostProfile,
    LayerSpec,
    ModelSpec,
    load_cluster_spec,
    load_cost_profile,
    load_model_spec,
)
from .strategies import (
    ParallelStrategy,
    StrategySet,
    build_decision_trees,
    candidate_pp_degrees,
    count_strategies,
    enumerate_strategies,
    parse_strategy,
    prune_dp_sdp,
)
from .costs import (
    EvalContext,
    LayerCost,
    StageCost,
    comm_time,
    compute_time,
    layer_memory,
    layer_time,
    memory_footprint,
    pipeline_cost,
    stage_cost,
    transform_cost,
)
from .dpsearch import DpResult, StageProblem, backward_peak_bound, dp_search, dp_search_batch

__version__ = "0.1.0"
