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
from .balance import (
    BalanceReport,
    PipelinePartition,
    SearchOutcome,
    adjust_partition,
    balance_degrees,
    bi_objective_optimize,
    evaluate_partition,
    init_partition_memory_balanced,
    init_partition_time_balanced,
    validate_partition,
)
from .planner import (
    GalvatronSearch,
    OracleResult,
    Plan,
    PlannerOptions,
    brute_force_oracle,
    evaluate_plan_document,
    galvatron_base,
    galvatron_search,
    galvatron_search_batch,
    init_microbatch_num,
    plan_full,
)

__version__ = "0.1.0"

__all__ = [
    "BalanceReport", "ClusterSpec", "CostProfile", "DivisibilityError", "DpResult", "EvalContext",
    "GalvatronSearch", "InfeasiblePlanError", "OracleResult", "LayerCost", "LayerSpec", "ModelSpec", "NativeError",
    "ParallelStrategy", "PipelinePartition", "Plan", "PlannerOptions", "SearchOutcome", "SpecError", "StageCost",
    "StageProblem", "StrategySet", "UnsupportedDeviceCountError", "adjust_partition", "backward_peak_bound",
    "balance_degrees", "bi_objective_optimize", "brute_force_oracle", "build_decision_trees", "candidate_pp_degrees", "comm_time",
    "compute_time", "count_strategies", "dp_search", "dp_search_batch", "enumerate_strategies",
    "evaluate_partition", "evaluate_plan_document", "galvatron_base", "galvatron_search",
    "galvatron_search_batch", "init_microbatch_num", "init_partition_memory_balanced",
    "init_partition_time_balanced", "layer_memory", "layer_time", "load_cluster_spec", "load_cost_profile",
    "load_model_spec", "memory_footprint", "parse_strategy", "pipeline_cost", "plan_full", "prune_dp_sdp",
    "stage_cost", "transform_cost", "validate_partition",
]
