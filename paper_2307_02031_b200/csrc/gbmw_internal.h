// gbmw_internal.h — device-side data layout of one chunk of stage searches and the
// launch entry points of gbmw_kernels.cu.  Not part of the C ABI.
//
// Layout.  For a problem with U units, S usable strategies,
// K (data, tp) classes and n_e = n_buckets + 1 memory buckets:
//   cells[U][S]        {time_c, ef_true, weight, class}        dpsearch.py:131-145
//   cmem [U][S]        {O_f, O_b, O_ms} of one layer of the unit (E_all check)
//   rcls [U][K][K]     transform cost between classes for unit u (dpsearch.py:149-160)
//   TF[2][K][n_e]      class-reduced frontier B_u = (t, f) pairs (ping-pong), column-major by class
//   par  [U-1][K][n_e] argmin strategy of B_u (uint16)
// B_u[e'][k] = lexmin_i (T_{u-1}[e',i] + R_u[cls(i),k], F_{u-1}[e',i], i), from which
// the reference table is T_u[e,j] = B_u[e-w_uj][cls j].t + time_c[u,j]  (exact
// restatement of dpsearch.py:261-280: R depends on (i, j) only through their classes).
#pragma once
#include <stdint.h>
#include <vector_types.h>
#include "../../include/gbmw.h"

namespace gbmw {

constexpr int kMaxUnits = 1024;      // backtrack path held in local memory
constexpr int kMaxClasses = 16;
constexpr int kCoarseShift = 10;     // K1 coarse maps: one entry per 1024 cells / R entries
constexpr int kUnitCoarseShift = 6;  // and per 64 units
constexpr int kMaxStrats = 512;      // smem staging of per-strategy constants
constexpr int kStepThreads = 256;    // threads per K2 CTA
constexpr int kStepRows = 2048;      // rows per K2 tile (64 groups of 32)
constexpr int kK2SlotEntries = 1024; // entries of one 1024-row K2 tile (anchor + breakpoints)
constexpr int kK2RoundsPerSlot = 40; // >= the most evaluation rounds of one tile (37, at 255 entries; static_assert in gbmw_step.cu)
constexpr int kK2HeavyBytes = 256;   // HeavyTile record (tile context + group entry offsets)

// change-bit words per class column of n_e rows (one spare word for 2-word window reads)
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int64_t flag_words(int64_t n_e) { return (n_e + 31) / 32 + 2; }

// change-summary words per class column: bit g of word t = 32-row group 32 t + g of the
// column has a change bit (stored after the column's change-bit words)
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int64_t sum_words(int64_t n_e) { return (n_e + 1023) / 1024 + 1; }

// row-map entries per unit: one per aligned 32-row group of B_u (see stored_row)
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int64_t rmap_groups(int64_t n_e) { return (n_e + 31) / 32; }
constexpr int kSweepThreads = 256;   // rows per K3 tile
constexpr int kSweepWK = 4608;       // (unit, strategy) pairs staged in shared memory by K3b (GPT-3-96 P = 1: 96 x 46)
constexpr int kSweepRmap = 1536;     // row-map entries of B_{U-1} staged in shared memory by K3b (n_e <= 49152)
constexpr int kMaxSweepRanks = 4096; // >= sweep tiles of one problem: ceil(GBMW_MAX_BUCKETS / kSweepThreads)

// K2 is instantiated per class-count group so a problem with few classes does not
// pay the register footprint of the widest one: K <= 4, 5..8, 9..kMaxClasses.
constexpr int kStepGroups = 3;
inline int step_group(int K) { return K <= 4 ? 0 : (K <= 8 ? 1 : 2); }
// Each class-count group is split into bands by depth (deep problems first); every band
// has its own K2 launches on its own stream, so the many short launches of deep problems
// overlap the few wide launches of shallow ones.
#ifndef GBMW_BANDS
#define GBMW_BANDS 2
#endif
constexpr int kBands = GBMW_BANDS;   // 2: deep / shallow; 3: very deep / deep / shallow
constexpr int kDeepUnits = 16;       // the deep bands: more units than this
constexpr int kVeryDeepUnits = 48;   // with 3 bands, band 0: more units than this
constexpr int kStepVGroups = kStepGroups * kBands;
// problems with approx_prev (collapsed state, dpsearch.py:306-375) form their own group
constexpr int kApproxGroup = kStepVGroups;
constexpr int kNumGroups = kStepVGroups + 1;
inline int problem_band(int U) {
    if (kBands == 2) return U > kDeepUnits ? 0 : 1;
    return U > kVeryDeepUnits ? 0 : (U > kDeepUnits ? 1 : 2);
}
inline bool shallow_group(int g) { return g < kStepVGroups && g % kBands == kBands - 1; }
inline int problem_group(int K, int flags, int U) {
    return (flags & GBMW_APPROX) ? kApproxGroup : step_group(K) * kBands + problem_band(U);
}

struct Cell {
    double c;       // time_c = t * count
    double ef;      // ef_true = (O_f + O_ms) * count
    int32_t w;      // weight = ceil(ef / gran), clamped to n_buckets + 1
    int32_t k;      // class of the strategy
};

struct CellMem {
    double o_f, o_b, o_ms;
};

struct DevProblem {
    int32_t U, S, K, flags;
    int32_t n_layers, stage_index, n_micro, env_index;
    int64_t n_b;            // buckets; rows are e = 0 .. n_b
    int64_t micro, gran;
    double budget;
    int64_t cell_off;       // into cells / cmem  (U*S)
    int64_t r_off;          // into rcls (U*K*K)
    int64_t b_off;          // into the TF buffers (K*n_e)
    int64_t par_off;        // into par ((U-1)*K*n_e)
    int64_t tile_off;       // into sweep partials (n_sweep_tiles)
    int64_t plan_off;       // into plans (n_layers)
    int64_t frontier_off;   // into frontier (n_b), -1 if not requested
    int32_t cand_off;       // into cand_strat / cand_cls (S)
    int32_t class_off;      // into class_d / class_t (K)
    int32_t unit_off;       // into unit_first / unit_count (U), shared by problems with equal stages
    int32_t layer_begin;    // global layer index of the first stage layer
    int32_t strat_begin;    // global index of the problem's strategy list
    int32_t result_index;   // slot in the batch result array
    int32_t n_sweep_tiles;
    int32_t ustate_off;     // into per-problem unit state: nuniq / unit_lo / unit_hi (U)
    int64_t flag_off;       // into the change-bit buffers (K * flag_words(n_e) words)
    int64_t rmap_off;       // into the row maps ((U-1) * rmap_groups(n_e) entries)
};

#if defined(__CUDACC__)
// Is column k of B (change bits flags_k, bit x = row x differs from row x-1) constant on
// rows [x0, x0 + 31]?  Rows below lo are +inf (never written); a window straddling lo
// mixes +inf and finite rows.  Only the bits of rows x0+1 .. x0+31 are read.
__device__ __forceinline__ bool window_flat(int x0, int lo, const uint32_t *flags_k) {
    const int x1 = x0 + 31;
    if (x1 < lo) return true;
    if (x0 < lo) return false;
    const int lb = x0 + 1;
    const int w0 = lb >> 5, s = lb & 31;
    const unsigned long long v =
        ((unsigned long long)__ldg(flags_k + w0 + 1) << 32 | (unsigned long long)__ldg(flags_k + w0)) >> s;
    return (v & 0x7fffffffull) == 0ull;
}

// B_u is stored only at its "stored rows" (the first live row of every 1024-row tile and
// every row where some column changes); between two stored rows every column is constant
// in value, argmin and argmin path.  The row map of unit u holds per 32-row group g
// {bit x: row 32g + x is stored, last stored row before the group}; every reader of a
// B_u row or of its argmin maps the row to the stored row at or before it (rows >= L_u).
__device__ __forceinline__ int stored_row(int2 m, int row) {
    const unsigned b = (unsigned)m.x & (0xffffffffu >> (31 - (row & 31)));
    return b ? (row & ~31) + 31 - __clz(b) : m.y;
}
__device__ __forceinline__ int stored_row(const int2 *rm_u, int row) {
    return stored_row(__ldg(rm_u + (row >> 5)), row);
}
#endif

struct alignas(16) TFCell {
    double t;       // lexmin candidate time
    double f;       // accumulated true forward bytes of its path (tie-break)
};

struct SweepPartial {
    double t;
    int64_t e;
    int32_t j;
    int32_t pad_;
};

// One K2 launch (unit u, class-count group): its problems are [lo, lo + n) in sorted order;
// k_step_lists writes the ones with live rows as (problem, first warp tile, last warp tile)
// items at items[base ...] (rows [L_u, H_u] only) and the item count to step_count[index].
struct StepList {
    int32_t u, lo, n, no_items;   // no_items: the step runs without tile items (K2f / K2s)
    int64_t base;
    int64_t ctx_base;             // first of the launch's per-problem step contexts (k_step_lists)
};
constexpr int kStepCtxBytes = 256;   // one step context (TileCtx, gbmw_step.cu) per (launch, problem)

// Everything a chunk's kernels read or write (device pointers).
struct ChunkArgs {
    const gbmw_layer *layers;
    const gbmw_strategy *strats;
    const gbmw_env *envs;
    const DevProblem *probs;      // sorted by U descending
    int32_t n_probs;
    int32_t max_k;
    const int64_t *cell_prefix;   // n_probs + 1
    const int64_t *r_prefix;      // n_probs + 1
    const int64_t *step_tiles;    // n_probs + 1, tiles of ceil(n_e / kStepRows)
    const int32_t *step_map;      // K2 tile -> problem (sorted position)
    // coarse position maps for the K1 index searches: the problem holding cell / R entry
    // b << kCoarseShift, and global unit b << kUnitCoarseShift (sorted positions)
    const int32_t *cell_coarse, *r_coarse, *unit_coarse;
    int64_t n_cell_coarse, n_r_coarse, n_unit_coarse;
    const int2 *aux_map;          // K3r tiles: (problem, tile) of frontier / collapsed-DP problems
    const StepList *step_lists;   // K2 launches of the chunk
    int32_t n_step_lists;
    int4 *step_items;             // (problem, first tile, last tile, step context) items of every K2 launch
    void *step_ctx;               // per (launch, problem): its step context, written by k_step_lists
    int64_t *step_count;          // per K2 launch: number of items
    int64_t n_aux;
    const int32_t *cand_strat;    // global strategy index
    const int32_t *cand_cls;
    const int32_t *class_d, *class_t;
    const int32_t *unit_first;    // global layer index
    const int32_t *unit_count;
    Cell *cells;
    CellMem *cmem;
    double *rcls;
    unsigned long long *bup;      // per problem, bits of max O_b (all >= 0)
    TFCell *TF[2];
    uint32_t *chg[2];             // change bits of B_u (ping-pong with TF): bit x = row x != row x-1
    int2 *rmap;                   // per unit u >= 1: row map of B_u (stored rows, see stored_row)
    unsigned long long *computed_cells;   // class cells K2 evaluated (rows x K), per chunk
    uint16_t *k2_erow, *k2_echg;  // per K2 tile slot (2 per 2048-row step tile): entries of a heavy tile
    void *k2_heavy;               // per tile slot: HeavyTile record (gbmw_step.cu)
    int2 *k2_rounds;              // heavy-tile rounds (slot, round); per-group regions of 33 per slot
    unsigned long long *k2_tl;    // debug (GBMW_K2_HIST=1): per launch {min start, max end} globaltimer, or null
    unsigned long long *k2_hist;  // debug (GBMW_K2_HIST=1): [32] tiles, [32] entries by log2 entry count; or null
    uint16_t *par;
    SweepPartial *partials;       // per sweep tile: best bucket of an unsafe (K3b) or collapsed-DP (K3r) tile
    SweepPartial *best;           // per problem: best safe bucket (K3a)
    unsigned long long *bound;    // per problem, 16 B: running best {bits of t, e + 1} of the sweep (K3a, K3b)
    int32_t *ufirst;              // per problem: first sweep tile holding unsafe rows
    int32_t *upruned;             // per problem: 1 + the highest pruned unsafe tile (every lower tile is pruned too), 0: none
    int32_t *usorted;             // problems with unsafe tiles, by unsafe tile count descending
    int64_t *uprefix;             // kMaxSweepRanks + 1: K3b items before rank r (rank = tile from the top)
    unsigned long long *ucounter; // K3b work counter
    int32_t *uniq;                // per (unit, slot): strategy indices with distinct (w, k, c, ef), ascending
    Cell *ucell;                  // per (unit, slot): the distinct cells themselves (cells[uniq])
    int32_t *nuniq;               // per unit: number of distinct strategies
    int32_t *unit_lo, *unit_hi;   // per unit u: live rows [L_u, H_u] of B_u (see k_dedupe)
    unsigned long long *counters; // per K2 launch: dynamic tile counter
    unsigned long long *live_cells;   // sum over problems and units of K * live rows
    unsigned long long *sweep_stats;  // K3b: unsafe rows walked, candidates examined, E_all checks
    int64_t n_units;
    gbmw_result *results;
    int32_t *plans;
    double *frontier;
};

// launchers (gbmw_kernels.cu); all asynchronous on `stream`, return cudaError_t as int
int launch_cost_tables(const ChunkArgs &a, int64_t n_cells, int64_t n_r, void *stream);
int launch_step_lists(const ChunkArgs &a, void *stream);
int launch_dp_step(const ChunkArgs &a, int group, int u, const int4 *items, const int64_t *count, int64_t max_items,
                   unsigned long long *counters3, int2 *rounds, int tl_id, void *stream, int *n_kernels);
int launch_dp_first(const ChunkArgs &a, int p_lo, int p_n, void *stream);
// u = 2 on candidate rows, for problems with S <= kSecondMaxS distinct strategies and
// n_e <= kSecondMaxRows rows (gbmw_step.cu)
constexpr int kSecondMaxS = 60;
constexpr int64_t kSecondMaxRows = 131072;
int launch_dp_second(const ChunkArgs &a, int group, int p_lo, int p_n, void *stream);
int launch_sweep(const ChunkArgs &a, void *stream, int ctas_per_sm = 0);   // K3b's persistent grid (0: occupancy)
int launch_approx_step(const ChunkArgs &a, int u, int64_t tile_base, int64_t n_tiles, unsigned long long *counter,
                       void *stream);
int launch_finalize(const ChunkArgs &a, void *stream);
// ---- exhaustive planner oracle (gbmw_brute.cu, planner.py:364-449)
constexpr int kBruteMaxLayers = 24;          // layers of the model (digits held in registers)
// One (pipeline degree, micro-batch count) cell: its tables start at tab_off in the
// double table — lt, lns, of, ob, oms [L][S] (per layer, usable strategy; memory at
// stage 1 / n_micro 1), p2p [L] (stage_p2p_time of a stage starting at layer l),
// R [L][S][S] (transform_cost at layer l from strategy a to b) — and its compositions at
// comp_off (bit l: layer l starts a stage).
struct BruteCell {
    int32_t S, L, P, n_micro;
    int64_t n_comp, spow;         // compositions; S^(L-1)
    int64_t n_items;              // n_comp * spow threads' worth of work
    int64_t tab_off, tab_len, comp_off;
    int64_t part_off;             // first block partial
    int32_t n_parts;              // blocks of the cell's launch
    int32_t smem_doubles;         // tables staged in shared memory (0: read from global)
    double budget;
};
struct BrutePartial {
    unsigned long long cost_bits;
    long long index;              // ci * S^L + digits (layer 0 most significant)
};
int brute_blocks(int64_t n_items);
int launch_brute_cell(const BruteCell &host_cell, const BruteCell *cells, const double *tab, const uint32_t *comps,
                      BrutePartial *partials, int cell_index, int neumaier, void *stream);
int launch_brute_reduce(const BruteCell *cells, int n_cells, const BrutePartial *partials, BrutePartial *out,
                        void *stream);

int launch_seed_partitions(const gbmw_layer *layers, int32_t L, const gbmw_env *env, int64_t n_devices, int32_t n_cells,
                           const int64_t *pp, const int64_t *micro, const int32_t *n_micro, double budget,
                           int32_t max_stages, double *scratch, int32_t *out_sizes, int32_t *out_status, void *stream);

}  // namespace gbmw
