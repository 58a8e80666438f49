/*
 * gbmw.h — C ABI of libgbmw, the B200-native Galvatron-BMW search hot path.
 *
 * The reference (parapilot, pure Python) has no native ABI; the seam it exposes
 * is the Python search API.  Each entry point below replaces one reference
 * function on that path; the Python package paper_2307_02031_b200 binds these
 * with ctypes and re-exposes the reference names and signatures
 * (see INTEGRATION.md for the binding a parapilot maintainer would add).
 *
 *   gbmw_enumerate        <- strategies.enumerate_strategies + prune_dp_sdp
 *                            (pkg/src/parapilot/strategies.py:185-209)
 *   gbmw_layer_cost       <- costs._layer_times + costs.layer_memory
 *                            (pkg/src/parapilot/costs.py:168-228)
 *   gbmw_transform_cost   <- costs.transform_cost (costs.py:252-277)
 *   gbmw_cost_tables      <- the per-(unit, strategy) table fill inside dp_search
 *                            (pkg/src/parapilot/dpsearch.py:127-160), GPU kernel K1
 *   gbmw_search_batch     <- dpsearch.dp_search (dpsearch.py:89-227) for a batch of
 *                            independent stage searches, plus costs.stage_cost
 *                            (costs.py:322-352) of each returned plan
 *   gbmw_batch_*          <- the same, split into prepare / run / fetch so the device
 *                            part can be timed with inputs resident in HBM
 *   gbmw_brute_force      <- planner.brute_force_oracle (planner.py:344-449), the
 *                            exhaustive (P, partition, assignment, m) scan, on the device
 *
 * Conventions: all functions return int status (0 = GBMW_OK, < 0 = error);
 * no C++ exception crosses the ABI; the message of the last failure is
 * available from gbmw_last_error().  Infeasibility is a per-result value, not
 * an error (dpsearch.py:119-121).  Inputs are caller-owned and read-only;
 * outputs are caller-allocated.  All byte counts must stay below 2^53 so that
 * the int64 -> fp64 conversions the reference performs implicitly (Python int
 * semantics) are exact; larger inputs are rejected with GBMW_ERANGE.
 */
#ifndef GBMW_H
#define GBMW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GBMW_ABI_VERSION 1

/* status codes */
#define GBMW_OK             0
#define GBMW_EINVAL_GRAN   -1   /* granularity_bytes <= 0            dpsearch.py:103-104 */
#define GBMW_EINVAL_BUDGET -2   /* budget_bytes < 0                  dpsearch.py:105-106 */
#define GBMW_EEMPTY        -3   /* empty stage                       dpsearch.py:107-108 */
#define GBMW_EMICRO        -4   /* micro_batch < 1 (DivisibilityError) dpsearch.py:109-110 */
#define GBMW_EBUCKETS      -5   /* n_buckets > GBMW_MAX_BUCKETS      dpsearch.py:113-118 */
#define GBMW_ECUDA         -6
#define GBMW_ENOMEM        -7
#define GBMW_EINVAL        -8   /* malformed argument (index out of range, bad degree ...) */
#define GBMW_ERANGE        -9   /* byte product reaches 2^53: fp64 would not be exact */
#define GBMW_ENOTSUP      -10   /* outside the kernel's compiled limits (see gbmw_limits) */
#define GBMW_EINTERNAL    -11   /* plan exceeds budget (reference AssertionError, dpsearch.py:220) */
#define GBMW_ESTAGE       -12   /* stage_index / n_micro out of range (costs.py:207-210) */

#define GBMW_MAX_BUCKETS 1000000 /* dpsearch.py:28 */

/* paradigms (strategies.py:20-23) */
#define GBMW_DP  0
#define GBMW_SDP 1
#define GBMW_TP  2

/* problem flags */
#define GBMW_FUSE        1   /* fuse_identical (dpsearch.py:71-86) */
#define GBMW_FRONTIER    2   /* collect_frontier (dpsearch.py:194-199) */
#define GBMW_STAGE_COST  4   /* also evaluate costs.stage_cost of the returned plan */
#define GBMW_APPROX      8   /* approx_prev: collapsed-state DP (dpsearch.py:306-375) */

/* ParallelStrategy (strategies.py:28-70): <= 3 ordered levels + ckpt flag. */
typedef struct gbmw_strategy {
    int32_t pp_degree;
    int32_t n_levels;
    int32_t paradigm[3];
    int32_t degree[3];
    int32_t ckpt;
} gbmw_strategy;

/* LayerSpec (specs.py:27-37) with the CostProfile override already applied. */
typedef struct gbmw_layer {
    int64_t param_bytes;
    int64_t bnd_bytes_per_sample;
    int64_t int_bytes_per_sample;
    double  fwd_time;                    /* CostProfile.fwd_time(layer), specs.py:100-101 */
    double  fwd_time_raw;                /* layer.fwd_time_per_sample: fusion shape key */
    double  tp_act_replication_fraction;
    int64_t kind_id;                     /* interned layer.kind: fusion shape key */
} gbmw_layer;

/* ClusterSpec + CostProfile scalars + ModelSpec.ms_bytes_per_param_byte. */
typedef struct gbmw_env {
    int64_t n_devices;
    int64_t island_size;
    double  intra_island_bw;
    double  inter_island_bw;
    double  overlap_slowdown;
    double  bwd_fwd_ratio;
    double  collective_efficiency;
    double  ms_bytes_per_param_byte;
} gbmw_env;

/* One dp_search call (dpsearch.py:89-101). */
typedef struct gbmw_problem {
    int32_t layer_begin;   /* stage layers = layers[layer_begin .. +n_layers) */
    int32_t n_layers;
    int32_t strat_begin;   /* StrategySet  = strategies[strat_begin .. +n_strats) */
    int32_t n_strats;
    int32_t env_index;
    int32_t stage_index;
    int32_t n_micro;
    int32_t flags;
    int64_t micro_batch;
    int64_t granularity_bytes;
    double  budget_bytes;
    int64_t n_buckets;     /* int(budget_bytes // granularity_bytes), Python floor semantics */
} gbmw_problem;

/* DpResult (dpsearch.py:33-39) + StageCost (costs.py:43-47) of the plan. */
typedef struct gbmw_result {
    double  time_s;            /* +inf when infeasible */
    double  e_fwd_used;
    int32_t feasible;
    int32_t status;
    double  stage_time_s;
    double  stage_time_no_sync_s;
    double  stage_peak_mem_bytes;
    int64_t frontier_offset;   /* index into the frontier output, -1 if not requested */
} gbmw_result;

/* Device timing of the last gbmw_batch_run (CUDA events on the ctx stream). */
typedef struct gbmw_timing {
    float   total_ms;          /* K1 .. K4 for all chunks */
    float   dp_ms;             /* K2 (min-plus layer steps) only */
    float   sweep_ms;          /* K3 (E_fwd sweep + validity) */
    float   tables_ms;         /* K1 (cost tables) */
    float   finalize_ms;       /* K4 (reduce, backtrack, stage cost) */
    int32_t n_chunks;
    int32_t n_launches;        /* kernels launched by the last run */
    double  transitions;       /* algorithmic sum over problems of (U-1) * n_e * S^2 */
    double  row_steps;         /* sum over problems of (U-1) * n_e */
    double  dp_bytes;          /* algorithmic HBM bytes of K2: 34 B per live class cell */
    double  dp_cells;          /* sum over problems of (U-1) * n_e * S * K (relaxations executed) */
    double  h2d_bytes;         /* bytes uploaded by gbmw_batch_create */
    double  d2h_bytes;         /* bytes downloaded by the last gbmw_batch_fetch */
    double  prep_ms;           /* host wall time of gbmw_batch_create before the upload */
    double  upload_ms;         /* host wall time of the arena allocation + upload */
    double  fetch_ms;          /* host wall time of the last gbmw_batch_fetch */
    double  live_cells;        /* class cells K2 computed (rows inside [L_u, H_u], times K) */
    double  sweep_rows;        /* unsafe buckets walked by K3b */
    double  sweep_cands;       /* candidates K3b examined (rejected by the F + O_b bound or checked) */
    double  sweep_checks;      /* candidates K3b backtracked for the exact E_all check */
} gbmw_timing;

typedef struct gbmw_ctx gbmw_ctx;
typedef struct gbmw_batch gbmw_batch;

const char *gbmw_version(void);
int  gbmw_abi_version(void);
/* Compiled limits: max units per stage, max classes, max strategies. */
void gbmw_limits(int32_t *max_units, int32_t *max_classes, int32_t *max_strategies);

/* device < 0 selects the current device.  workspace_bytes == 0 picks a default
 * (a fraction of free device memory); problems are chunked to fit it. */
int  gbmw_ctx_create(int32_t device, uint64_t workspace_bytes, gbmw_ctx **out);
int  gbmw_ctx_destroy(gbmw_ctx *ctx);
const char *gbmw_last_error(const gbmw_ctx *ctx);
/* the cudaStream_t (as void*) every kernel of this context is launched on */
void *gbmw_ctx_stream(const gbmw_ctx *ctx);
/* message of the last failure of a ctx-less call (enumerate, costs) on this thread */
const char *gbmw_last_error_global(void);

/* enumerate_strategies(N, P) (+ prune_dp_sdp when prune != 0), canonical sort_key order.
 * If out == NULL only *count is written. */
int  gbmw_enumerate(int64_t n_devices, int64_t pp_degree, int32_t prune,
                    gbmw_strategy *out, int32_t capacity, int32_t *count);

/* out[0..4] = (time_s, time_no_sync_s, O_f, O_b, O_ms) of one (layer, strategy). */
int  gbmw_layer_cost(const gbmw_layer *layer, const gbmw_strategy *s, const gbmw_env *env,
                     int64_t micro_batch, int32_t stage_index, int32_t n_micro, double *out);
/* out[0..3] = (grad_s, fwd_act_s, bwd_act_s, ckpt_act_s), costs.py:98-129. */
int  gbmw_comm_breakdown(const gbmw_layer *layer, const gbmw_strategy *s, const gbmw_env *env,
                         int64_t micro_batch, double *out);
/* prev == NULL means "no previous strategy" (returns 0). */
int  gbmw_transform_cost(const gbmw_layer *layer, const gbmw_strategy *prev,
                         const gbmw_strategy *cur, int64_t micro_batch,
                         const gbmw_env *env, double *out);

/* K1 only (parity tests): for problem 0 of the list, per (unit, usable strategy)
 * writes time_c, ef_true, o_b and weight, in dp_search's table order
 * (dpsearch.py:131-145); out arrays hold n_units * n_usable entries.  Also returns
 * the usable-strategy indices and the unit count. */
int  gbmw_cost_tables(gbmw_ctx *ctx,
                      const gbmw_layer *layers, int64_t n_layers,
                      const gbmw_strategy *strategies, int64_t n_strategies,
                      const gbmw_env *envs, int64_t n_envs,
                      const gbmw_problem *problem,
                      double *time_c, double *ef_true, double *o_b, int64_t *weight,
                      int32_t *usable, int32_t *n_usable, int32_t *n_units);

/* Batched dp_search (+ stage_cost).  plans: one int32 per stage layer of every
 * problem, concatenated in problem order (index into that problem's strategy
 * list, -1 when infeasible).  frontier: n_buckets doubles per problem flagged
 * GBMW_FRONTIER, concatenated in problem order (may be NULL otherwise).
 * Returns the first per-problem error status, if any (all results are filled). */
int  gbmw_search_batch(gbmw_ctx *ctx,
                       const gbmw_layer *layers, int64_t n_layers,
                       const gbmw_strategy *strategies, int64_t n_strategies,
                       const gbmw_env *envs, int64_t n_envs,
                       const gbmw_problem *problems, int64_t n_problems,
                       gbmw_result *results, int32_t *plans, double *frontier);

/* Split form: prepare (validate, host set-up, upload) / run (device only) / fetch. */
int  gbmw_batch_create(gbmw_ctx *ctx,
                       const gbmw_layer *layers, int64_t n_layers,
                       const gbmw_strategy *strategies, int64_t n_strategies,
                       const gbmw_env *envs, int64_t n_envs,
                       const gbmw_problem *problems, int64_t n_problems,
                       gbmw_batch **out);
int  gbmw_batch_run(gbmw_ctx *ctx, gbmw_batch *batch);
int  gbmw_batch_fetch(gbmw_ctx *ctx, gbmw_batch *batch,
                      gbmw_result *results, int32_t *plans, double *frontier);
int  gbmw_batch_timing(const gbmw_batch *batch, gbmw_timing *out);
/* timing of the last batch run on this context (incl. one-shot gbmw_search_batch calls) */
int  gbmw_ctx_last_timing(const gbmw_ctx *ctx, gbmw_timing *out);
int  gbmw_batch_destroy(gbmw_batch *batch);

/* ---- host-side partition logic around the search (parapilot/balance.py) ---- */

/* evaluate_partition (balance.py:98-119): stage_cost of every stage of a partition
 * under per-layer strategies; out = 3 doubles per stage (time, time_no_sync, peak). */
int  gbmw_partition_costs(const gbmw_layer *layers, int32_t n_layers, const gbmw_strategy *per_layer,
                          const int32_t *sizes, int32_t n_stages, const gbmw_env *env,
                          int64_t micro_batch, int32_t n_micro, double *out);
/* gbmw_partition_costs for n_items (partition, per-layer strategies, micro-batch) items on up to
 * n_threads host threads (the adjusted partitions of one Algorithm-2 round, balance.py:420-424):
 * per_layer n_items x n_layers records, sizes n_items x max_stages (n_stages[i] used),
 * out n_items x 3 * max_stages. */
int  gbmw_partition_costs_batch(const gbmw_layer *layers, int32_t n_layers, const gbmw_strategy *per_layer,
                                const int32_t *sizes, const int32_t *n_stages, int32_t max_stages,
                                const gbmw_env *env, const int64_t *micro_batch, const int32_t *n_micro,
                                int32_t n_items, int32_t n_threads, double *out);
/* _init_partition (balance.py:180-236): objective 0 = memory-balanced, 1 = time-balanced. */
int  gbmw_init_partition(const gbmw_layer *layers, int32_t n_layers, const gbmw_strategy *per_layer,
                         int32_t n_stages, const gbmw_env *env, int64_t micro_batch, int32_t n_micro,
                         int32_t objective, int32_t *out_sizes);
/* _seed_for (balance.py:471-488): the uniform seed strategy, and (optional) its
 * memory-balanced partition (planner.py:250-253). */
int  gbmw_seed_for(const gbmw_layer *layers, int32_t n_layers, const gbmw_env *env, int64_t n_devices,
                   int64_t pp_degree, int64_t micro_batch, int32_t n_micro, double budget,
                   gbmw_strategy *out_seed, int32_t *out_sizes);
/* gbmw_seed_for over many (pp_degree, micro_batch, n_micro) cells of one model and cluster,
 * on up to n_threads host threads (the seed partitions galvatron_base computes for every
 * (batch, degree) cell of a batch window, planner.py:250-253).  out_sizes: n_cells rows of
 * max_stages int32, row i holds pp_degree[i] stage sizes. */
int  gbmw_seed_partitions(const gbmw_layer *layers, int32_t n_layers, const gbmw_env *env, int64_t n_devices,
                          int32_t n_cells, const int64_t *pp_degree, const int64_t *micro_batch,
                          const int32_t *n_micro, double budget, int32_t max_stages, int32_t n_threads,
                          int32_t *out_sizes);
/* Algorithm 2's trajectory set-up (balance.py:366-384 as _run_trajectories runs it) for many
 * (pp_degree, micro_batch, n_micro) cells, on up to n_threads host threads: the _seed_for
 * strategy's memory-balanced partition p0 (out_p0, rows of max_stages int32) and mem_ref, the
 * largest stage peak of the seed's time-balanced partition (out_mem_ref, one per cell). */
int  gbmw_bmw_setup(const gbmw_layer *layers, int32_t n_layers, const gbmw_env *env, int64_t n_devices,
                    int32_t n_cells, const int64_t *pp_degree, const int64_t *micro_batch, const int32_t *n_micro,
                    double budget, int32_t max_stages, int32_t n_threads, int32_t *out_p0, double *out_mem_ref);
/* The same on the device of ctx: one warp per cell. */
int  gbmw_seed_partitions_device(gbmw_ctx *ctx, const gbmw_layer *layers, int32_t n_layers, const gbmw_env *env,
                                 int64_t n_devices, int32_t n_cells, const int64_t *pp_degree,
                                 const int64_t *micro_batch, const int32_t *n_micro, double budget,
                                 int32_t max_stages, int32_t *out_sizes);
/* CPython >= 3.12 built-in sum() of floats (Neumaier), as the reference folds sums. */
double gbmw_py_sum(const double *x, int32_t n);
/* Select the host interpreter's sum() semantics for every planner fold (gbmw_py_sum, the
 * balance degrees of balance.py:62-77 in the partition hill climb): 1 = CPython >= 3.12
 * (Neumaier-compensated, the default), 0 = CPython <= 3.11 (left-to-right addition).
 * gbmw_seed_partitions_device supports only 1 (GBMW_ENOTSUP otherwise). */
int gbmw_set_sum_semantics(int32_t neumaier);
int gbmw_sum_semantics(void);
const char *gbmw_planner_last_error(void);

/* ---- exhaustive oracle (planner.py:344-449) ---- */

/* OracleResult (planner.py:344-351) + scan statistics. */
typedef struct gbmw_oracle_result {
    double  cost;              /* +inf when nothing is feasible */
    int32_t feasible;
    int32_t pp_degree;
    int32_t n_micro;
    int32_t n_stages;          /* entries of out_partition in use */
    double  combos;            /* (partition, assignment) pairs scanned over all cells */
    double  device_ms;         /* device time of the scan (CUDA events on the ctx stream) */
} gbmw_oracle_result;

/* brute_force_oracle(model, cluster, profile, batch) on the device of ctx: the minimum of
 * pipeline_cost over every power-of-two pipeline degree P <= n_layers, micro-batch count m
 * dividing batch, ordered partition of the layers into P stages and assignment of the
 * usable strategies of prune_dp_sdp(enumerate_strategies(N, P)) to the layers, first
 * minimum in the reference's loop order.  budget_bytes = ClusterSpec.mem_budget_bytes.
 * out_partition[n_layers]: stage sizes (n_stages used); out_choice[n_layers]: per layer the
 * index into the pruned strategy set of pp_degree.  max_combos caps the scan (0: 2^44);
 * larger scans return GBMW_ENOTSUP, as do more than 24 layers.  The reference's own
 * size guards (max_layers / max_devices) are applied by the Python wrapper. */
int gbmw_brute_force(gbmw_ctx *ctx, const gbmw_layer *layers, int32_t n_layers, const gbmw_env *env,
                     int64_t batch, double budget_bytes, double max_combos,
                     int32_t *out_partition, int32_t *out_choice, gbmw_oracle_result *out);

#ifdef __cplusplus
}
#endif
#endif /* GBMW_H */
