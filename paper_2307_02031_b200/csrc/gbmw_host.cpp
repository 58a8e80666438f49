// gbmw_host.cpp — C ABI, validation, host-side problem set-up and chunk scheduling
// of the Galvatron-BMW stage search (see include/gbmw.h and DESIGN.md).
//
// The host does the O(L + S) per-problem bookkeeping the reference does in Python
// before its tables (dpsearch.py:103-125: argument checks, usable-strategy filter,
// unit fusion) plus the (data, tp) class map the device formulation needs, lays
// problems out in a chunk workspace, and issues the K1..K4 launches on the
// context's stream.  All fp64 cost arithmetic lives in costmodel.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <chrono>
#include <map>
#include <memory>
#include <tuple>
#include <unordered_map>
#include <unordered_set>

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

#include "../../include/gbmw.h"
#include "costmodel.cuh"
#include "gbmw_internal.h"

using namespace gbmw;

namespace {

thread_local std::string g_err;

constexpr double kTwo53 = 9007199254740992.0;
constexpr int64_t kTwo53i = 9007199254740992LL;

bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

int set_err(std::string *dst, int code, const std::string &msg) {
    if (dst) *dst = msg;
    g_err = msg;
    return code;
}

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// |a*b| < 2^53 with no overflow in the test itself
bool prod_exact(int64_t a, int64_t b) {
    if (a < 0 || b < 0) return false;
    if (a == 0 || b == 0) return true;
    return (double)a * (double)b < kTwo53 * 0.5;   // margin for rounding of the test
}

// Per (strategy list, micro-batch): usable strategies and their (data, tp) classes.
struct StratInfo {
    std::vector<int32_t> cand, cand_cls, cls_d, cls_t;
    int status = GBMW_OK;
    std::string err;
    int32_t min_pp = 0, max_pp = 0;
    int32_t cand_off = 0, class_off = 0;   // into the batch's concatenated candidate / class arrays
};

// Per (layer range, fusion flag): units and byte maxima for the 2^53 checks.
struct UnitInfo {
    std::vector<int32_t> unit_first, unit_count;
    int status = GBMW_OK;
    std::string err;
    int64_t max_bnd = 0, max_int = 0;
    int32_t unit_off = 0;               // into the batch's concatenated unit arrays
};

// hash of the (begin, count, micro-batch / fuse) record keys
struct Key3Hash {
    template <class A, class B, class C>
    size_t operator()(const std::tuple<A, B, C> &k) const {
        uint64_t h = (uint64_t)(uint32_t)std::get<0>(k) * 0x9E3779B97F4A7C15ull;
        h ^= ((uint64_t)(uint32_t)std::get<1>(k) + 0x632BE59BD9B4E019ull) * 0xC2B2AE3D27D4EB4Full;
        h ^= ((uint64_t)std::get<2>(k) + 0x165667B19E3779F9ull) * 0x94D049BB133111EBull;
        return (size_t)(h ^ (h >> 29));
    }
};

struct HostProb {
    int status = GBMW_OK;
    bool gpu = false;              // has device work
    const StratInfo *si = nullptr;
    const UnitInfo *ui = nullptr;
    int U = 0, S = 0, K = 0;
    int64_t n_b = 0;
    int64_t plan_off = 0, frontier_off = -1;
    // workspace footprint (elements)
    int64_t n_cells = 0, n_r = 0, n_bcells = 0, n_par = 0, n_tiles = 0, n_step_tiles = 0, n_flagw = 0, n_rmap = 0;
    size_t ws_bytes = 0;
};

using StratKey = std::tuple<int32_t, int32_t, int64_t>;
using UnitKey = std::tuple<int32_t, int32_t, int>;

struct Chunk {
    std::vector<int> probs;        // host problem indices, sorted by (K group, U descending)
    std::vector<int64_t> step_prefix;
    int group_lo[kNumGroups + 1] = {0};
    std::vector<int> n_active[kNumGroups];    // per group, per u: problems of the group with U > u
    int n_approx = 0;
    int Umax = 0, max_k = 1;
    int64_t n_cells = 0, n_r = 0, n_bcells = 0, n_par = 0, n_tiles = 0, n_units = 0, n_flagw = 0, n_rmap = 0;
    size_t small_off = 0;          // byte offset of this chunk's descriptor block in the arena
    // offsets inside the descriptor block
    size_t o_probs, o_cellp, o_rp, o_stepp, o_cand, o_ccls, o_clsd, o_clst, o_uf, o_uc;
    size_t o_stepmap, o_aux, o_slists, o_cellc, o_rc, o_unitc;
    int64_t n_cellc = 0, n_rc = 0, n_unitc = 0;
    int64_t n_aux = 0;
    std::vector<StepList> slists;  // K2 launches (unit, group), in launch order
    std::vector<int> slist_group;
    std::vector<char> slist_second;   // u = 2 list run by the candidate-row kernel (K2s)
    int64_t n_items = 0;           // K2 items (active problems) over all launches
    int64_t n_ctx = 0;             // per-(launch, problem) step contexts
    size_t small_bytes = 0;
    size_t ws_bytes = 0;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    int launches = 0;
};

}  // namespace

struct gbmw_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t aux[kNumGroups] = {nullptr};   // K2 groups 1.. run concurrently with group 0
    cudaEvent_t fork = nullptr, join[kNumGroups] = {nullptr};
    cudaStream_t list_stream = nullptr;           // K2l, concurrent with the first steps (K2f / K2s)
    cudaStream_t tstream = nullptr;               // timing: waits for every group's K2 (ev[2])
    cudaEvent_t k2done[kNumGroups] = {nullptr};
    cudaEvent_t list_done = nullptr;
    cudaEvent_t gspan[kNumGroups][2] = {{nullptr}};   // debug (GBMW_K2_HIST): per-stream K2 span
    uint64_t workspace_limit = 0;
    void *ws = nullptr;
    size_t ws_size = 0;
    // grow-only device arena lent to one batch at a time (no cudaMalloc per call)
    void *arena = nullptr;
    size_t arena_cap = 0;
    bool arena_busy = false;
    // grow-only pinned staging buffer for uploads
    void *pinned = nullptr;
    void *seed_buf = nullptr;                // gbmw_seed_partitions_device buffers (grow-only)
    size_t seed_cap = 0;
    size_t pinned_cap = 0;
    gbmw_timing last{};
    std::string err;
    gbmw_batch *spare = nullptr;             // a destroyed batch kept for its host buffers (no page faults)
};

struct gbmw_batch {
    std::vector<gbmw_layer> layers;
    std::vector<gbmw_strategy> strats;
    std::vector<gbmw_env> envs;
    std::vector<gbmw_problem> problems;
    std::vector<HostProb> hp;
    std::vector<Chunk> chunks;
    // one record per key, in first-appearance order (built in parallel once the keys are
    // known), and their arrays concatenated (each chunk's descriptor block holds a copy)
    std::vector<std::pair<StratKey, std::unique_ptr<StratInfo>>> strat_recs;
    std::vector<std::pair<UnitKey, std::unique_ptr<UnitInfo>>> unit_recs;
    // key -> record index, direct-indexed by strategy-list / layer-range start (touched slots
    // are cleared on reuse)
    std::vector<std::vector<std::pair<std::pair<int32_t, int64_t>, int32_t>>> strat_at;
    std::vector<std::vector<std::pair<int32_t, int32_t>>> unit_at;
    std::vector<int32_t> srec, urec;         // per problem: its records (-1: none)
    std::vector<int32_t> strat_ok;           // per strategy: check_strategy status
    std::vector<StratDeg> strat_deg;         // per strategy: its degrees (valid where strat_ok is OK)
    std::vector<int32_t> host_fix;           // problems whose result entry the host writes (no device
                                             // work, or a frontier offset), ascending
    std::vector<int32_t> g_cand, g_ccls, g_clsd, g_clst, g_uf, g_uc;
    int64_t total_plan = 0, total_frontier = 0;
    // device arena: inputs | chunk descriptor blocks | outputs
    void *arena = nullptr;
    size_t arena_size = 0;
    size_t o_layers = 0, o_strats = 0, o_envs = 0, o_results = 0, o_plans = 0, o_frontier = 0, o_stats = 0;
    size_t max_ws = 0;
    gbmw_timing timing{};
    bool ran = false;
    gbmw_ctx *ctx = nullptr;
    bool ctx_arena = false;        // arena is borrowed from ctx (returned on destroy)
};

// ----------------------------------------------------------------------------- misc
extern "C" const char *gbmw_version(void) { return "gbmw 0.1.0 (sm_100a)"; }
extern "C" int gbmw_abi_version(void) { return GBMW_ABI_VERSION; }
extern "C" void gbmw_limits(int32_t *max_units, int32_t *max_classes, int32_t *max_strategies) {
    if (max_units) *max_units = kMaxUnits;
    if (max_classes) *max_classes = kMaxClasses;
    if (max_strategies) *max_strategies = kMaxStrats;
}
extern "C" const char *gbmw_last_error(const gbmw_ctx *ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }
extern "C" const char *gbmw_last_error_global(void) { return g_err.c_str(); }
extern "C" void *gbmw_ctx_stream(const gbmw_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }

// ----------------------------------------------------------------------------- enumeration
// strategies.py:149-200 — ordered power-of-two factorisations of G = N/P into <= 3
// levels, injective paradigm labels in itertools.permutations order, x {ckpt off, on},
// sorted by (n_levels, paradigm names, degrees, ckpt); prune drops dp>1 and sdp>1.
namespace {
void factor_seqs(int64_t rem, std::vector<int32_t> &prefix, std::vector<std::vector<int32_t>> &out) {
    if (rem == 1) { out.push_back(prefix); return; }
    if (prefix.size() >= 3) return;
    for (int64_t f = 2; f <= rem; f *= 2) {
        if (rem % f == 0) {
            prefix.push_back((int32_t)f);
            factor_seqs(rem / f, prefix, out);
            prefix.pop_back();
        }
    }
}

const int kPerm1[3][1] = {{0}, {1}, {2}};
const int kPerm2[6][2] = {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {2, 0}, {2, 1}};
const int kPerm3[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

bool sort_key_less(const gbmw_strategy &a, const gbmw_strategy &b) {
    if (a.n_levels != b.n_levels) return a.n_levels < b.n_levels;
    for (int l = 0; l < a.n_levels; ++l)   // "dp" < "sdp" < "tp" as strings == index order
        if (a.paradigm[l] != b.paradigm[l]) return a.paradigm[l] < b.paradigm[l];
    for (int l = 0; l < a.n_levels; ++l)
        if (a.degree[l] != b.degree[l]) return a.degree[l] < b.degree[l];
    return a.ckpt < b.ckpt;
}
}  // namespace

extern "C" int gbmw_enumerate(int64_t n_devices, int64_t pp_degree, int32_t prune, gbmw_strategy *out,
                              int32_t capacity, int32_t *count) {
    if (!is_pow2(n_devices))
        return set_err(nullptr, GBMW_EINVAL, "device count must be a power of two, got " + std::to_string(n_devices));
    if (!is_pow2(pp_degree))
        return set_err(nullptr, GBMW_EINVAL, "pipeline degree must be a power of two, got " + std::to_string(pp_degree));
    if (pp_degree > n_devices || n_devices % pp_degree != 0)
        return set_err(nullptr, GBMW_EINVAL, "pipeline degree " + std::to_string(pp_degree) +
                                                 " does not divide device count " + std::to_string(n_devices));
    const int64_t group = n_devices / pp_degree;
    std::vector<std::vector<int32_t>> seqs;
    std::vector<int32_t> prefix;
    if (group == 1) seqs.push_back({});
    else factor_seqs(group, prefix, seqs);
    std::vector<gbmw_strategy> all;
    for (const auto &f : seqs) {
        const int k = (int)f.size();
        const int nperm = (k == 0) ? 1 : (k == 1 ? 3 : 6);
        for (int pi = 0; pi < nperm; ++pi) {
            for (int ck = 0; ck < 2; ++ck) {
                gbmw_strategy s;
                std::memset(&s, 0, sizeof(s));
                s.pp_degree = (int32_t)pp_degree;
                s.n_levels = k;
                for (int l = 0; l < k; ++l) {
                    s.paradigm[l] = (k == 1) ? kPerm1[pi][l] : (k == 2 ? kPerm2[pi][l] : kPerm3[pi][l]);
                    s.degree[l] = f[l];
                }
                s.ckpt = ck;
                all.push_back(s);
            }
        }
    }
    std::stable_sort(all.begin(), all.end(), sort_key_less);
    std::vector<gbmw_strategy> keep;
    for (const auto &s : all) {
        if (prune) {
            const StratDeg d = strat_degrees(s);
            if (d.dp > 1 && d.sdp > 1) continue;
        }
        keep.push_back(s);
    }
    if (count) *count = (int32_t)keep.size();
    if (out) {
        if ((int64_t)keep.size() > capacity) return set_err(nullptr, GBMW_EINVAL, "enumerate: output capacity too small");
        std::memcpy(out, keep.data(), keep.size() * sizeof(gbmw_strategy));
    }
    return GBMW_OK;
}

// ----------------------------------------------------------------------------- scalar costs
namespace {
// the first malformed field of a strategy record, or null
const char *strategy_defect(const gbmw_strategy &s) {
    if (s.n_levels < 0 || s.n_levels > 3) return "strategy has more than 3 levels";
    if (s.pp_degree < 1) return "strategy pipeline degree must be >= 1";
    for (int l = 0; l < s.n_levels; ++l) {
        if (s.paradigm[l] < 0 || s.paradigm[l] > 2) return "strategy has an unknown paradigm";
        if (s.degree[l] < 1) return "strategy level degree must be >= 1";
    }
    return nullptr;
}
int check_strategy(const gbmw_strategy &s, std::string *err) {
    const char *d = strategy_defect(s);
    return d ? set_err(err, GBMW_EINVAL, d) : GBMW_OK;
}
int check_layer(const gbmw_layer &L, std::string *err) {
    if (L.param_bytes < 0 || L.param_bytes >= kTwo53i || L.bnd_bytes_per_sample < 0 ||
        L.bnd_bytes_per_sample >= kTwo53i || L.int_bytes_per_sample < 0 || L.int_bytes_per_sample >= kTwo53i)
        return set_err(err, GBMW_ERANGE, "layer byte counts must lie in [0, 2^53)");
    return GBMW_OK;
}
}  // namespace

extern "C" int gbmw_layer_cost(const gbmw_layer *layer, const gbmw_strategy *s, const gbmw_env *env,
                               int64_t micro_batch, int32_t stage_index, int32_t n_micro, double *out) {
    if (!layer || !s || !env || !out) return set_err(nullptr, GBMW_EINVAL, "null argument");
    int rc = check_strategy(*s, nullptr);
    if (rc) return rc;
    if ((rc = check_layer(*layer, nullptr))) return rc;
    const StratDeg d = strat_degrees(*s);
    if (micro_batch % d.data != 0)
        return set_err(nullptr, GBMW_EMICRO, "micro-batch " + std::to_string(micro_batch) +
                                                 " is not divisible by the DP*SDP degree " + std::to_string(d.data));
    if (stage_index < 1 || stage_index > s->pp_degree)
        return set_err(nullptr, GBMW_ESTAGE, "stage_index " + std::to_string(stage_index) + " out of range 1.." +
                                                 std::to_string(s->pp_degree));
    if (n_micro < 1) return set_err(nullptr, GBMW_ESTAGE, "n_micro must be >= 1, got " + std::to_string(n_micro));
    double t, t_ns;
    layer_times(*layer, *s, d, micro_batch, *env, &t, &t_ns);
    const Mem m = layer_memory(*layer, d, micro_batch, stage_index, n_micro, env->ms_bytes_per_param_byte);
    out[0] = t; out[1] = t_ns; out[2] = m.o_f; out[3] = m.o_b; out[4] = m.o_ms;
    return GBMW_OK;
}

extern "C" int gbmw_comm_breakdown(const gbmw_layer *layer, const gbmw_strategy *s, const gbmw_env *env,
                                   int64_t micro_batch, double *out) {
    if (!layer || !s || !env || !out) return set_err(nullptr, GBMW_EINVAL, "null argument");
    int rc = check_strategy(*s, nullptr);
    if (rc) return rc;
    const StratDeg d = strat_degrees(*s);
    const Comm c = comm_breakdown(*layer, *s, d, micro_batch, *env);
    out[0] = c.grad; out[1] = c.fwd_act; out[2] = c.bwd_act; out[3] = c.ckpt_act;
    return GBMW_OK;
}

extern "C" int gbmw_transform_cost(const gbmw_layer *layer, const gbmw_strategy *prev, const gbmw_strategy *cur,
                                   int64_t micro_batch, const gbmw_env *env, double *out) {
    if (!layer || !cur || !env || !out) return set_err(nullptr, GBMW_EINVAL, "null argument");
    if (!prev) { *out = 0.0; return GBMW_OK; }
    const StratDeg a = strat_degrees(*prev), b = strat_degrees(*cur);
    *out = transform_cost(layer->bnd_bytes_per_sample, a.data, a.tp, b.data, b.tp, micro_batch, env->intra_island_bw);
    return GBMW_OK;
}

// ----------------------------------------------------------------------------- ctx
extern "C" int gbmw_ctx_create(int32_t device, uint64_t workspace_bytes, gbmw_ctx **out) {
    if (!out) return set_err(nullptr, GBMW_EINVAL, "null out");
    *out = nullptr;
    int dev = device;
    cudaError_t ce;
    if (dev < 0) {
        ce = cudaGetDevice(&dev);
        if (ce != cudaSuccess) return set_err(nullptr, GBMW_ECUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(ce));
    }
    ce = cudaSetDevice(dev);
    if (ce != cudaSuccess) return set_err(nullptr, GBMW_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(ce));
    gbmw_ctx *c = new gbmw_ctx();
    c->device = dev;
    {
        int lo_pri = 0, hi_pri = 0;                      // the main stream carries the deep band of group 0
        cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri);
        ce = cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi_pri < lo_pri ? hi_pri + 1 : hi_pri);
    }
    if (ce != cudaSuccess) {
        delete c;
        return set_err(nullptr, GBMW_ECUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(ce));
    }
    if (workspace_bytes == 0) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        workspace_bytes = std::min<uint64_t>((uint64_t)(fr * 0.6), 120ull << 30);
        if (workspace_bytes < (64ull << 20)) workspace_bytes = 64ull << 20;
    }
    c->workspace_limit = workspace_bytes;
    *out = c;
    return GBMW_OK;
}

extern "C" int gbmw_ctx_destroy(gbmw_ctx *ctx) {
    if (!ctx) return GBMW_OK;
    cudaSetDevice(ctx->device);
    if (ctx->ws) cudaFree(ctx->ws);
    if (ctx->arena) cudaFree(ctx->arena);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    for (int g = 0; g < kNumGroups; ++g) {
        if (ctx->aux[g]) cudaStreamDestroy(ctx->aux[g]);
        if (ctx->join[g]) cudaEventDestroy(ctx->join[g]);
    }
    if (ctx->fork) cudaEventDestroy(ctx->fork);
    if (ctx->list_stream) cudaStreamDestroy(ctx->list_stream);
    if (ctx->tstream) cudaStreamDestroy(ctx->tstream);
    for (auto &e : ctx->k2done)
        if (e) cudaEventDestroy(e);
    if (ctx->list_done) cudaEventDestroy(ctx->list_done);
    if (ctx->seed_buf) cudaFree(ctx->seed_buf);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx->spare;
    delete ctx;
    return GBMW_OK;
}

// ----------------------------------------------------------------------------- batch set-up
namespace {

// usable strategies + classes of one strategy list at one micro-batch (dpsearch.py:42-43)
void build_strat(const gbmw_batch &b, const StratKey &key, StratInfo &si) {
    const int32_t begin = std::get<0>(key), n = std::get<1>(key);
    const int64_t micro = std::get<2>(key);
    for (int i = 0; i < n && si.status == GBMW_OK; ++i) {
        const gbmw_strategy &s = b.strats[begin + i];
        if (b.strat_ok[begin + i] != GBMW_OK) {       // the message is rebuilt only on failure
            si.status = check_strategy(s, &si.err);
            break;
        }
        const StratDeg &d = b.strat_deg[begin + i];
        if (micro % d.data != 0) continue;
        si.cand.push_back(begin + i);
        si.min_pp = si.cand.size() == 1 ? s.pp_degree : std::min(si.min_pp, s.pp_degree);
        si.max_pp = si.cand.size() == 1 ? s.pp_degree : std::max(si.max_pp, s.pp_degree);
        int k = -1;                                   // (data, tp) classes in first-appearance order
        for (int c = 0; c < (int)si.cls_d.size(); ++c)
            if (si.cls_d[c] == d.data && si.cls_t[c] == d.tp) { k = c; break; }
        if (k < 0) { k = (int)si.cls_d.size(); si.cls_d.push_back(d.data); si.cls_t.push_back(d.tp); }
        si.cand_cls.push_back(k);
    }
}

// units of one stage (dpsearch.py:71-86): fusion key (kind, param, bnd, int, raw fwd_time, frac)
void build_unit(const gbmw_batch &b, const UnitKey &key, UnitInfo &ui) {
    const int32_t begin = std::get<0>(key), n = std::get<1>(key);
    const bool fuse = std::get<2>(key) != 0;
    for (int i = 0; i < n; ++i) {
        const int gl = begin + i;
        const gbmw_layer &B = b.layers[gl];
        const int rc = check_layer(B, &ui.err);
        if (rc) { ui.status = rc; break; }
        ui.max_bnd = std::max(ui.max_bnd, B.bnd_bytes_per_sample);
        ui.max_int = std::max(ui.max_int, B.int_bytes_per_sample);
        if (fuse && !ui.unit_first.empty()) {
            const gbmw_layer &A = b.layers[ui.unit_first.back()];
            if (A.kind_id == B.kind_id && A.param_bytes == B.param_bytes &&
                A.bnd_bytes_per_sample == B.bnd_bytes_per_sample && A.int_bytes_per_sample == B.int_bytes_per_sample &&
                A.fwd_time_raw == B.fwd_time_raw && A.tp_act_replication_fraction == B.tp_act_replication_fraction) {
                ui.unit_count.back() += 1;
                continue;
            }
        }
        ui.unit_first.push_back(gl);
        ui.unit_count.push_back(1);
    }
}

// dp_search argument checks and host bookkeeping (dpsearch.py:103-125), on the records the
// key pass assigned
void prepare_problem(gbmw_batch &b, int pi, std::string *err) {
    const gbmw_problem &P = b.problems[pi];
    HostProb &h = b.hp[pi];
    h = HostProb();
    auto fail = [&](int code, const std::string &msg) { h.status = code; set_err(err, code, msg); };
    if (P.granularity_bytes <= 0) return fail(GBMW_EINVAL_GRAN, "granularity_bytes must be positive, got " + std::to_string(P.granularity_bytes));
    if (!(P.budget_bytes >= 0.0)) return fail(GBMW_EINVAL_BUDGET, "budget_bytes must be non-negative");
    if (P.n_layers <= 0) return fail(GBMW_EEMPTY, "stage must contain at least one layer");
    if (P.micro_batch < 1) return fail(GBMW_EMICRO, "micro-batch must be >= 1, got " + std::to_string(P.micro_batch));
    if (P.n_buckets < 0) return fail(GBMW_EINVAL, "n_buckets must be non-negative");
    if (P.n_buckets > GBMW_MAX_BUCKETS)
        return fail(GBMW_EBUCKETS, "budget/granularity yields " + std::to_string(P.n_buckets) + " buckets (> " +
                                       std::to_string(GBMW_MAX_BUCKETS) + "); increase the memory granularity");
    if (P.layer_begin < 0 || (int64_t)P.layer_begin + P.n_layers > (int64_t)b.layers.size())
        return fail(GBMW_EINVAL, "problem layer range out of bounds");
    if (P.strat_begin < 0 || P.n_strats < 0 || (int64_t)P.strat_begin + P.n_strats > (int64_t)b.strats.size())
        return fail(GBMW_EINVAL, "problem strategy range out of bounds");
    if (P.env_index < 0 || P.env_index >= (int)b.envs.size()) return fail(GBMW_EINVAL, "problem env index out of bounds");
    if (P.budget_bytes >= kTwo53) return fail(GBMW_ERANGE, "budget_bytes must be < 2^53");
    h.n_b = P.n_buckets;
    const StratInfo *si = b.strat_recs[b.srec[pi]].second.get();   // assigned: both ranges are valid
    if (si->status) return fail(si->status, si->err);
    h.si = si;
    h.S = (int)si->cand.size();
    if (h.S == 0 || h.n_b == 0) return;    // infeasible, dpsearch.py:119-121
    const UnitInfo *ui = b.unit_recs[b.urec[pi]].second.get();
    if (ui->status) return fail(ui->status, ui->err);
    h.ui = ui;
    // layer_memory range checks (costs.py:207-210), raised on the first table cell
    if (P.stage_index < 1 || P.stage_index > si->min_pp)
        for (int32_t gi : si->cand) {
            const gbmw_strategy &s = b.strats[gi];
            if (P.stage_index < 1 || P.stage_index > s.pp_degree)
                return fail(GBMW_ESTAGE, "stage_index " + std::to_string(P.stage_index) + " out of range 1.." +
                                             std::to_string(s.pp_degree));
        }
    if (P.n_micro < 1) return fail(GBMW_ESTAGE, "n_micro must be >= 1, got " + std::to_string(P.n_micro));
    // exactness of Python int arithmetic in fp64
    const int64_t max_stash = std::min<int64_t>(std::max<int32_t>(1, si->max_pp), std::max<int32_t>(1, P.n_micro));
    if (!prod_exact(ui->max_bnd, P.micro_batch) || !prod_exact(ui->max_bnd * P.micro_batch, max_stash) ||
        !prod_exact(ui->max_int, P.micro_batch))
        return fail(GBMW_ERANGE, "byte products of a stage layer reach 2^53; fp64 would not be exact");
    if (h.S > kMaxStrats || h.S > 65535) return fail(GBMW_ENOTSUP, "more than " + std::to_string(kMaxStrats) + " usable strategies");
    h.K = (int)si->cls_d.size();
    if (h.K > kMaxClasses) return fail(GBMW_ENOTSUP, "more than " + std::to_string(kMaxClasses) + " (data, tp) classes");
    h.U = (int)ui->unit_first.size();
    if (h.U > kMaxUnits) return fail(GBMW_ENOTSUP, "more than " + std::to_string(kMaxUnits) + " units in one stage");
    const int64_t n_e = h.n_b + 1;
    h.n_cells = (int64_t)h.U * h.S;
    h.n_r = (int64_t)h.U * h.K * h.K;
    const bool approx = (P.flags & GBMW_APPROX) != 0;
    h.n_bcells = approx ? n_e : ((h.U > 1) ? (int64_t)h.K * n_e : 0);
    h.n_par = approx ? (int64_t)h.U * n_e : (int64_t)(h.U - 1) * h.K * n_e;
    h.n_tiles = (h.n_b + kSweepThreads - 1) / kSweepThreads;
    h.n_step_tiles = (n_e + kStepRows - 1) / kStepRows;
    h.n_flagw = (!approx && h.U > 1) ? (int64_t)h.K * (flag_words(n_e) + sum_words(n_e)) : 0;
    h.n_rmap = approx ? 0 : (int64_t)(h.U > 1 ? h.U - 1 : 0) * rmap_groups(n_e);
    h.ws_bytes = (size_t)h.n_cells * (2 * sizeof(Cell) + sizeof(CellMem) + 4) + (size_t)h.U * 12 + (size_t)h.n_r * 8 + 8 +
                 (size_t)h.n_bcells * 2 * sizeof(TFCell) + (size_t)h.n_par * 2 +
                 (size_t)h.n_tiles * sizeof(SweepPartial) + sizeof(SweepPartial) + 36 + (size_t)h.n_flagw * 8 +
                 (size_t)h.n_rmap * 8 + (size_t)(h.U > 1 ? h.U - 1 : 0) * 24 +
                 (size_t)h.n_step_tiles * 2 * (kK2SlotEntries * 4 + kK2HeavyBytes + kK2RoundsPerSlot * 8);
    h.gpu = true;
}

// chunk workspace layout (byte offsets from ws base)
struct WsLayout {
    size_t cells, cmem, rcls, bup, items, sctx, scount, tf0, tf1, chg0, chg1, rmap, par, parts, bestp, bound, ufirst, upruned, usorted, uprefix, uctr,
        uniq, ucell, nuniq,
        ulo, uhi, ctr, k2e, k2c, k2h, k2r, total;
};
WsLayout ws_layout(const Chunk &c) {
    WsLayout w;
    size_t o = 0;
    w.cells = o; o = align_up(o + c.n_cells * sizeof(Cell));
    w.cmem = o; o = align_up(o + c.n_cells * sizeof(CellMem));
    w.rcls = o; o = align_up(o + c.n_r * 8);
    w.bup = o; o = align_up(o + c.probs.size() * 8);
    w.items = o; o = align_up(o + c.n_items * sizeof(int4));
    w.sctx = o; o = align_up(o + (size_t)c.n_ctx * kStepCtxBytes);
    w.scount = o; o = align_up(o + c.slists.size() * 8);
    w.tf0 = o; o = align_up(o + c.n_bcells * sizeof(TFCell));
    w.tf1 = o; o = align_up(o + c.n_bcells * sizeof(TFCell));
    w.chg0 = o; o = align_up(o + c.n_flagw * 4);
    w.chg1 = o; o = align_up(o + c.n_flagw * 4);
    w.rmap = o; o = align_up(o + c.n_rmap * 8);
    w.par = o; o = align_up(o + c.n_par * 2);
    w.parts = o; o = align_up(o + c.n_tiles * sizeof(SweepPartial));
    w.bestp = o; o = align_up(o + c.probs.size() * sizeof(SweepPartial));
    w.bound = o; o = align_up(o + c.probs.size() * 16);
    w.ufirst = o; o = align_up(o + c.probs.size() * 4);
    w.upruned = o; o = align_up(o + c.probs.size() * 4);
    w.usorted = o; o = align_up(o + c.probs.size() * 4);
    w.uprefix = o; o = align_up(o + (size_t)kNumGroups * (kMaxSweepRanks + 1) * 8);   // one per group sweep
    w.uctr = o; o = align_up(o + (size_t)kNumGroups * 8);
    w.uniq = o; o = align_up(o + c.n_cells * 4);
    w.ucell = o; o = align_up(o + c.n_cells * sizeof(Cell));
    w.nuniq = o; o = align_up(o + c.n_units * 4);
    w.ulo = o; o = align_up(o + c.n_units * 4);
    w.uhi = o; o = align_up(o + c.n_units * 4);
    w.ctr = o; o = align_up(o + (size_t)(c.Umax + 1) * kNumGroups * 3 * 8);
    {
        const size_t slots = 2 * (size_t)c.step_prefix.back();
        w.k2e = o; o = align_up(o + slots * kK2SlotEntries * 2);
        w.k2c = o; o = align_up(o + slots * kK2SlotEntries * 2);
        w.k2h = o; o = align_up(o + slots * kK2HeavyBytes);
        w.k2r = o; o = align_up(o + slots * kK2RoundsPerSlot * sizeof(int2));
    }
    w.total = o;
    return w;
}

}  // namespace

extern "C" int gbmw_batch_create(gbmw_ctx *ctx, const gbmw_layer *layers, int64_t n_layers,
                                 const gbmw_strategy *strategies, int64_t n_strategies, const gbmw_env *envs,
                                 int64_t n_envs, const gbmw_problem *problems, int64_t n_problems, gbmw_batch **out) {
    if (!ctx || !out) return set_err(nullptr, GBMW_EINVAL, "null ctx/out");
    *out = nullptr;
    if (n_problems < 0 || n_layers < 0 || n_strategies < 0 || n_envs < 0)
        return set_err(&ctx->err, GBMW_EINVAL, "negative array length");
    const double t_start = now_ms();
    gbmw_batch *b = ctx->spare ? ctx->spare : new gbmw_batch();   // reuse the host buffers of the last batch
    ctx->spare = nullptr;
    b->layers.assign(layers, layers + n_layers);
    b->strats.assign(strategies, strategies + n_strategies);
    b->envs.assign(envs, envs + n_envs);
    b->problems.assign(problems, problems + n_problems);
    if (b->hp.size() != (size_t)n_problems) b->hp.resize(n_problems);   // each record is reset below
    int first_err = GBMW_OK;
    std::string first_msg;
    double t_head = 0.0, th[3] = {0, 0, 0};
    {
        // argument checks, strategy / unit records, sizes; the first failing problem (in input
        // order) names the error
        std::vector<std::string> msgs(n_problems);
        th[0] = now_ms();
        // record keys of every problem whose ranges are valid, deduplicated in first-appearance
        // order through the direct indexes (serial: ~10 ns a problem)
        b->strat_recs.clear();
        b->unit_recs.clear();
        if (b->strat_at.size() < (size_t)n_strategies + 1) b->strat_at.resize(n_strategies + 1);
        if (b->unit_at.size() < (size_t)n_layers + 1) b->unit_at.resize(n_layers + 1);
        b->srec.assign(n_problems, -1);
        b->urec.assign(n_problems, -1);
        {
            int32_t ls = -1, lu = -1;
            StratKey lsk{};
            UnitKey luk{};
            for (int64_t i = 0; i < n_problems; ++i) {
                const gbmw_problem &P = b->problems[i];
                if (P.strat_begin >= 0 && P.n_strats >= 0 && (int64_t)P.strat_begin + P.n_strats <= n_strategies &&
                    P.micro_batch >= 1) {
                    const StratKey k = std::make_tuple(P.strat_begin, P.n_strats, P.micro_batch);
                    if (ls < 0 || k != lsk) {
                        auto &slot = b->strat_at[P.strat_begin];
                        ls = -1;
                        for (const auto &e : slot)
                            if (e.first.first == P.n_strats && e.first.second == P.micro_batch) { ls = e.second; break; }
                        if (ls < 0) {
                            ls = (int32_t)b->strat_recs.size();
                            slot.push_back({{P.n_strats, P.micro_batch}, ls});
                            b->strat_recs.emplace_back(k, nullptr);
                        }
                        lsk = k;
                    }
                    b->srec[i] = ls;
                }
                if (P.layer_begin >= 0 && P.n_layers > 0 && (int64_t)P.layer_begin + P.n_layers <= n_layers) {
                    const UnitKey k = std::make_tuple(P.layer_begin, P.n_layers, (P.flags & GBMW_FUSE) ? 1 : 0);
                    if (lu < 0 || k != luk) {
                        auto &slot = b->unit_at[P.layer_begin];
                        const int32_t k2 = P.n_layers * 2 + std::get<2>(k);
                        lu = -1;
                        for (const auto &e : slot)
                            if (e.first == k2) { lu = e.second; break; }
                        if (lu < 0) {
                            lu = (int32_t)b->unit_recs.size();
                            slot.push_back({k2, lu});
                            b->unit_recs.emplace_back(k, nullptr);
                        }
                        luk = k;
                    }
                    b->urec[i] = lu;
                }
            }
            for (const auto &r : b->strat_recs) b->strat_at[std::get<0>(r.first)].clear();   // for the next batch
            for (const auto &r : b->unit_recs) b->unit_at[std::get<0>(r.first)].clear();
        }
        th[1] = now_ms();
        // per-strategy checks and degrees, once (records of one list at many micro-batches share them)
        b->strat_ok.resize(n_strategies);
        b->strat_deg.resize(n_strategies);
        for (int64_t i = 0; i < n_strategies; ++i) {
            b->strat_ok[i] = strategy_defect(b->strats[i]) ? GBMW_EINVAL : GBMW_OK;
            if (b->strat_ok[i] == GBMW_OK) b->strat_deg[i] = strat_degrees(b->strats[i]);
        }
        // the records, and the concatenated arrays the descriptors point into
        b->g_cand.clear(); b->g_ccls.clear(); b->g_clsd.clear(); b->g_clst.clear(); b->g_uf.clear(); b->g_uc.clear();
        for (auto &e : b->strat_recs) {
            e.second.reset(new StratInfo());
            StratInfo &si = *e.second;
            build_strat(*b, e.first, si);
            if (si.status != GBMW_OK) continue;
            si.cand_off = (int32_t)b->g_cand.size();
            si.class_off = (int32_t)b->g_clsd.size();
            b->g_cand.insert(b->g_cand.end(), si.cand.begin(), si.cand.end());
            b->g_ccls.insert(b->g_ccls.end(), si.cand_cls.begin(), si.cand_cls.end());
            b->g_clsd.insert(b->g_clsd.end(), si.cls_d.begin(), si.cls_d.end());
            b->g_clst.insert(b->g_clst.end(), si.cls_t.begin(), si.cls_t.end());
        }
        for (auto &e : b->unit_recs) {
            e.second.reset(new UnitInfo());
            UnitInfo &ui = *e.second;
            build_unit(*b, e.first, ui);
            if (ui.status != GBMW_OK) continue;
            ui.unit_off = (int32_t)b->g_uf.size();
            b->g_uf.insert(b->g_uf.end(), ui.unit_first.begin(), ui.unit_first.end());
            b->g_uc.insert(b->g_uc.end(), ui.unit_count.begin(), ui.unit_count.end());
        }
        th[2] = now_ms();
        for (int64_t i = 0; i < n_problems; ++i) prepare_problem(*b, (int)i, &msgs[i]);
        t_head = now_ms();
        for (int64_t i = 0; i < n_problems; ++i)
            if (b->hp[i].status != GBMW_OK) { first_err = b->hp[i].status; first_msg = msgs[i]; break; }
    }
    const double t_probs = now_ms();
    // output offsets
    int64_t plan = 0, front = 0;
    for (int64_t i = 0; i < n_problems; ++i) {
        HostProb &h = b->hp[i];
        h.plan_off = plan;
        plan += std::max<int32_t>(0, b->problems[i].n_layers);
        if (h.gpu && (b->problems[i].flags & GBMW_FRONTIER)) { h.frontier_off = front; front += h.n_b; }
    }
    b->total_plan = plan;
    b->total_frontier = front;
    // greedy chunking by workspace budget
    const size_t limit = ctx->workspace_limit;
    Chunk cur;
    size_t cur_bytes = 0;
    auto flush = [&]() {
        if (cur.probs.empty()) return;
        b->chunks.push_back(cur);
        cur = Chunk();
        cur_bytes = 0;
    };
    b->host_fix.clear();
    for (int64_t i = 0; i < n_problems; ++i) {
        HostProb &h = b->hp[i];
        if (!h.gpu) { b->host_fix.push_back((int32_t)i); continue; }
        const size_t need = h.ws_bytes + 16 * 256;
        if (need > limit) {
            h.status = GBMW_ENOMEM;
            h.gpu = false;
            b->host_fix.push_back((int32_t)i);
            if (first_err == GBMW_OK) { first_err = GBMW_ENOMEM; first_msg = "one stage search needs more workspace than the context limit"; }
            continue;
        }
        if (h.frontier_off >= 0) b->host_fix.push_back((int32_t)i);
        if (cur_bytes + need > limit) flush();
        cur.probs.push_back((int)i);
        cur_bytes += need;
    }
    flush();
    const double t_chunks = now_ms();
    // per-chunk descriptor layout: problem order, groups, totals
    double td[4] = {0, 0, 0, 0};
    size_t blob_size = 0;
    for (Chunk &c : b->chunks) {
        double tq = now_ms();
        const int np = (int)c.probs.size();
        {
            // (group ascending, U descending, input order): a stable counting sort on the
            // bucket g * (kMaxUnits + 1) + (kMaxUnits - U); groups and the per-unit active
            // counts follow from the bucket histogram
            constexpr int nu = kMaxUnits + 1;
            const size_t nb = (size_t)kNumGroups * nu;
            std::vector<int32_t> bucket(np), start(nb + 1, 0);
            for (int i = 0; i < np; ++i) {
                const HostProb &h = b->hp[c.probs[i]];
                const int g = problem_group(h.K, b->problems[c.probs[i]].flags, h.U);
                bucket[i] = g * nu + (kMaxUnits - h.U);             // U <= kMaxUnits (checked)
                start[bucket[i] + 1]++;
            }
            c.Umax = 0;
            for (size_t k = 0; k < nb; ++k)
                if (start[k + 1]) c.Umax = std::max(c.Umax, kMaxUnits - (int)(k % nu));
            for (size_t k = 0; k < nb; ++k) start[k + 1] += start[k];
            for (int g = 0; g < kNumGroups; ++g) {
                c.group_lo[g] = start[(size_t)g * nu];
                c.group_lo[g + 1] = start[(size_t)(g + 1) * nu];
                c.n_active[g].assign(c.Umax + 1, 0);      // problems of the group with U > u
                for (int u = c.Umax, above = 0; u >= 0; --u) {
                    c.n_active[g][u] = above;
                    const size_t k = (size_t)g * nu + (kMaxUnits - u);
                    above += start[k + 1] - start[k];
                }
            }
            std::vector<int> sorted(np);
            for (int i = 0; i < np; ++i) sorted[start[bucket[i]]++] = c.probs[i];
            c.probs.swap(sorted);
        }
        c.step_prefix.resize(np + 1);
        c.step_prefix[0] = 0;
        for (int x = 0; x < np; ++x) c.step_prefix[x + 1] = c.step_prefix[x] + b->hp[c.probs[x]].n_step_tiles;
        td[0] += now_ms() - tq; tq = now_ms();
        // the chunk's totals (the block layout needs them before the descriptors are written)
        c.n_cells = c.n_r = c.n_bcells = c.n_par = c.n_tiles = c.n_units = c.n_flagw = c.n_rmap = c.n_aux = 0;
        c.n_approx = 0;
        c.max_k = 1;
        for (int x = 0; x < np; ++x) {
            const HostProb &h = b->hp[c.probs[x]];
            const int flags = b->problems[c.probs[x]].flags;
            c.n_cells += h.n_cells; c.n_r += h.n_r; c.n_bcells += h.n_bcells; c.n_par += h.n_par; c.n_tiles += h.n_tiles;
            c.n_units += h.U; c.n_flagw += h.n_flagw; c.n_rmap += h.n_rmap;
            if (flags & (GBMW_FRONTIER | GBMW_APPROX)) c.n_aux += h.n_tiles;   // every row swept (K3r)
            if (flags & GBMW_APPROX) c.n_approx++;
            c.max_k = std::max(c.max_k, h.K);
        }
        td[1] += now_ms() - tq; tq = now_ms();
        // K2 launches: items bounded by all tiles of the active problems
        c.slists.clear(); c.slist_group.clear(); c.slist_second.clear(); c.n_items = 0; c.n_ctx = 0;
        static const bool no_second = getenv("GBMW_NO_SECOND") && getenv("GBMW_NO_SECOND")[0] == '1';
        for (int u = 1; u < c.Umax; ++u)
            for (int g = 0; g < kStepVGroups; ++g) {
                const int lo = c.group_lo[g], na = c.n_active[g][u];
                if (na == 0) continue;
                bool second = u == 2 && !no_second;
                for (int x = lo; x < lo + na && second; ++x) {
                    const HostProb &hx = b->hp[c.probs[x]];
                    second = hx.S <= kSecondMaxS && hx.n_b + 1 <= kSecondMaxRows;
                }
                StepList sl;
                sl.u = u; sl.lo = lo; sl.n = na; sl.no_items = (u == 1 || second) ? 1 : 0; sl.base = c.n_items;
                sl.ctx_base = c.n_ctx;
                if (!sl.no_items) c.n_ctx += na;
                c.slists.push_back(sl);
                c.slist_group.push_back(g);
                c.slist_second.push_back(second ? 1 : 0);
                // items of >= 1 warp tile: a problem's warp tiles number at most 2 * (its
                // 2048-row tiles)
                if (!sl.no_items) c.n_items += 2 * (c.step_prefix[lo + na] - c.step_prefix[lo]);
            }
        // the chunk's descriptor block (16-byte aligned arrays), 256-byte aligned in the blob
        size_t o = 0;
        auto lay = [&](size_t bytes) { o = align_up(o, 16); const size_t at = o; o += bytes; return at; };
        c.o_probs = lay((size_t)np * sizeof(DevProblem));
        c.o_cellp = lay((size_t)(np + 1) * 8);
        c.o_rp = lay((size_t)(np + 1) * 8);
        c.o_stepp = lay((size_t)(np + 1) * 8);
        c.o_cand = lay(b->g_cand.size() * 4);
        c.o_ccls = lay(b->g_ccls.size() * 4);
        c.o_clsd = lay(b->g_clsd.size() * 4);
        c.o_clst = lay(b->g_clst.size() * 4);
        c.o_uf = lay(b->g_uf.size() * 4);
        c.o_uc = lay(b->g_uc.size() * 4);
        c.o_stepmap = lay(c.n_approx > 0 ? (size_t)c.step_prefix[np] * 4 : 0);
        c.o_aux = lay((size_t)c.n_aux * sizeof(int2));
        c.o_slists = lay(c.slists.size() * sizeof(StepList));
        c.n_cellc = (c.n_cells + (1 << kCoarseShift) - 1) >> kCoarseShift;
        c.n_rc = (c.n_r + (1 << kCoarseShift) - 1) >> kCoarseShift;
        c.n_unitc = (c.n_units + (1 << kUnitCoarseShift) - 1) >> kUnitCoarseShift;
        c.o_cellc = lay((size_t)c.n_cellc * 4);
        c.o_rc = lay((size_t)c.n_rc * 4);
        c.o_unitc = lay((size_t)c.n_unitc * 4);
        c.small_bytes = o;
        c.small_off = align_up(blob_size, 256);
        blob_size = c.small_off + c.small_bytes;
        c.ws_bytes = ws_layout(c).total;
        b->max_ws = std::max(b->max_ws, c.ws_bytes);
        td[2] += now_ms() - tq;
    }
    // arena: inputs | descriptor blocks | outputs
    size_t o = 0;
    b->o_layers = o; o = align_up(o + b->layers.size() * sizeof(gbmw_layer));
    b->o_strats = o; o = align_up(o + b->strats.size() * sizeof(gbmw_strategy));
    b->o_envs = o; o = align_up(o + b->envs.size() * sizeof(gbmw_env));
    const size_t o_blob = o; o = align_up(o + blob_size);
    b->o_results = o; o = align_up(o + b->problems.size() * sizeof(gbmw_result));
    b->o_plans = o; o = align_up(o + (size_t)b->total_plan * sizeof(int32_t));
    b->o_frontier = o; o = align_up(o + (size_t)b->total_frontier * sizeof(double));
    b->o_stats = o; o = align_up(o + (5 * (b->chunks.size() + 1) + 64) * 8);
    b->arena_size = std::max<size_t>(o, 256);
    for (Chunk &c : b->chunks) c.small_off += o_blob;
    // the input part of the arena is staged in pinned memory: descriptors are written there directly
    const size_t up = o_blob + blob_size;
    if (ctx->pinned_cap < up) {
        if (ctx->pinned) cudaFreeHost(ctx->pinned);
        ctx->pinned = nullptr;
        ctx->pinned_cap = 0;
        const size_t cap = std::max<size_t>(up + up / 4, 1u << 20);
        if (cudaHostAlloc(&ctx->pinned, cap, cudaHostAllocDefault) == cudaSuccess) ctx->pinned_cap = cap;
    }
    std::vector<char> fallback;
    char *host = (char *)ctx->pinned;
    if (!host) { fallback.resize(up); host = fallback.data(); }
    const double t_fill = now_ms();
    if (!b->layers.empty()) std::memcpy(host + b->o_layers, b->layers.data(), b->layers.size() * sizeof(gbmw_layer));
    if (!b->strats.empty()) std::memcpy(host + b->o_strats, b->strats.data(), b->strats.size() * sizeof(gbmw_strategy));
    if (!b->envs.empty()) std::memcpy(host + b->o_envs, b->envs.data(), b->envs.size() * sizeof(gbmw_env));
    for (Chunk &c : b->chunks) {
        // the descriptors, written in place
        char *blk = host + c.small_off;
        const int np = (int)c.probs.size();
        auto cpy = [&](size_t off, const std::vector<int32_t> &v) { if (!v.empty()) std::memcpy(blk + off, v.data(), v.size() * 4); };
        cpy(c.o_cand, b->g_cand); cpy(c.o_ccls, b->g_ccls); cpy(c.o_clsd, b->g_clsd); cpy(c.o_clst, b->g_clst);
        cpy(c.o_uf, b->g_uf); cpy(c.o_uc, b->g_uc);
        std::memcpy(blk + c.o_stepp, c.step_prefix.data(), (size_t)(np + 1) * 8);
        if (!c.slists.empty()) std::memcpy(blk + c.o_slists, c.slists.data(), c.slists.size() * sizeof(StepList));
        DevProblem *dps = (DevProblem *)(blk + c.o_probs);
        int64_t *cellp = (int64_t *)(blk + c.o_cellp), *rp = (int64_t *)(blk + c.o_rp);
        int32_t *stepmap = (int32_t *)(blk + c.o_stepmap);
        int2 *aux = (int2 *)(blk + c.o_aux);
        int32_t *cellc = (int32_t *)(blk + c.o_cellc), *rc = (int32_t *)(blk + c.o_rc), *unitc = (int32_t *)(blk + c.o_unitc);
        // the coarse entries whose position falls in [first, first + n): problem x
        auto coarse = [](int32_t *map, int shift, int64_t first, int64_t n, int x) {
            const int64_t step = (int64_t)1 << shift;
            for (int64_t b = (first + step - 1) >> shift; (b << shift) < first + n; ++b) map[b] = x;
        };
        cellp[0] = 0;
        rp[0] = 0;
        const bool map_steps = c.n_approx > 0;        // K2 tile -> problem map of the collapsed-DP step (K2c)
        {
            int64_t s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};   // cells r bcells par tiles units flagw rmap aux
            for (int x = 0; x < np; ++x) {
                const int pi = c.probs[x];
                const HostProb &h = b->hp[pi];
                const gbmw_problem &P = b->problems[pi];
                DevProblem d;
                std::memset(&d, 0, sizeof(d));
                d.U = h.U; d.S = h.S; d.K = h.K; d.flags = P.flags;
                d.n_layers = P.n_layers; d.stage_index = P.stage_index; d.n_micro = P.n_micro; d.env_index = P.env_index;
                d.n_b = h.n_b; d.micro = P.micro_batch; d.gran = P.granularity_bytes; d.budget = P.budget_bytes;
                d.cell_off = s[0]; d.r_off = s[1]; d.b_off = s[2]; d.par_off = s[3]; d.tile_off = s[4];
                d.plan_off = h.plan_off; d.frontier_off = h.frontier_off;
                d.cand_off = h.si->cand_off; d.class_off = h.si->class_off; d.unit_off = h.ui->unit_off;
                d.ustate_off = (int32_t)s[5];
                d.flag_off = s[6];
                d.rmap_off = s[7];
                d.layer_begin = P.layer_begin; d.strat_begin = P.strat_begin; d.result_index = pi;
                d.n_sweep_tiles = (int32_t)h.n_tiles;
                std::memcpy(dps + x, &d, sizeof(d));
                coarse(cellc, kCoarseShift, s[0], h.n_cells, x);
                coarse(rc, kCoarseShift, s[1], h.n_r, x);
                coarse(unitc, kUnitCoarseShift, s[5], h.U, x);
                s[0] += h.n_cells; s[1] += h.n_r; s[2] += h.n_bcells; s[3] += h.n_par; s[4] += h.n_tiles;
                s[5] += h.U; s[6] += h.n_flagw; s[7] += h.n_rmap;
                cellp[x + 1] = s[0];
                rp[x + 1] = s[1];
                if (map_steps)
                    for (int64_t q = c.step_prefix[x]; q < c.step_prefix[x + 1]; ++q) stepmap[q] = x;
                if (P.flags & (GBMW_FRONTIER | GBMW_APPROX))
                    for (int q = 0; q < d.n_sweep_tiles; ++q) aux[s[8]++] = make_int2(x, q);
            }
        }
    }
    const double t_prep = now_ms();
    td[3] = t_prep - t_fill;
    static const bool host_timing = getenv("GBMW_HOST_TIMING") && getenv("GBMW_HOST_TIMING")[0] == '1';
    if (host_timing)
        fprintf(stderr, "create: problems %.3f ms (inputs %.3f keys %.3f records %.3f checks+sizes %.3f), "
                "chunking %.3f ms, descriptors %.3f ms (sort %.3f sums %.3f layout %.3f fill %.3f)\n",
                t_probs - t_start, th[0] - t_start, th[1] - th[0], th[2] - th[1], t_head - th[2], t_chunks - t_probs,
                t_prep - t_chunks, td[0], td[1], td[2], td[3]);
    cudaSetDevice(ctx->device);
    b->ctx = ctx;
    cudaError_t ce = cudaSuccess;
    if (!ctx->arena_busy) {
        if (ctx->arena_cap < b->arena_size) {
            if (ctx->arena) cudaFree(ctx->arena);
            ctx->arena = nullptr;
            ctx->arena_cap = 0;
            const size_t cap = std::max<size_t>(b->arena_size + b->arena_size / 4, 4u << 20);
            ce = cudaMalloc(&ctx->arena, cap);
            if (ce == cudaSuccess) ctx->arena_cap = cap;
        }
        if (ce == cudaSuccess) {
            b->arena = ctx->arena;
            b->ctx_arena = true;
            ctx->arena_busy = true;
        }
    } else {
        ce = cudaMalloc(&b->arena, b->arena_size);
    }
    if (ce != cudaSuccess) {
        delete b;
        return set_err(&ctx->err, GBMW_ENOMEM, std::string("cudaMalloc(arena): ") + cudaGetErrorString(ce));
    }
    // one upload of the input part of the arena
    ce = cudaMemcpyAsync(b->arena, host, up, cudaMemcpyHostToDevice, ctx->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
    b->timing.h2d_bytes = (double)up;
    b->timing.prep_ms = t_prep - t_start;
    b->timing.upload_ms = now_ms() - t_prep;
    if (ce != cudaSuccess) {
        gbmw_batch_destroy(b);
        return set_err(&ctx->err, GBMW_ECUDA, std::string("upload: ") + cudaGetErrorString(ce));
    }
    // algorithmic work counters
    for (int64_t i = 0; i < n_problems; ++i) {
        const HostProb &h = b->hp[i];
        if (!h.gpu) continue;
        const double rows = (double)(h.U - 1) * (double)(h.n_b + 1);
        b->timing.transitions += rows * h.S * h.S;
        b->timing.row_steps += rows;
        b->timing.dp_cells += rows * h.S * h.K;
        // K2 compulsory bytes: B_{u-1} (T,F) read once + B_u written + argmin written
    }
    b->timing.n_chunks = (int32_t)b->chunks.size();
    *out = b;
    if (first_err != GBMW_OK) set_err(&ctx->err, first_err, first_msg);
    return first_err;
}

namespace {
int ensure_ws(gbmw_ctx *ctx, size_t bytes) {
    if (bytes <= ctx->ws_size) return GBMW_OK;
    if (ctx->ws) { cudaFree(ctx->ws); ctx->ws = nullptr; ctx->ws_size = 0; }
    cudaError_t ce = cudaMalloc(&ctx->ws, bytes);
    if (ce != cudaSuccess) return set_err(&ctx->err, GBMW_ENOMEM, std::string("cudaMalloc(workspace): ") + cudaGetErrorString(ce));
    ctx->ws_size = bytes;
    return GBMW_OK;
}

ChunkArgs chunk_args(gbmw_batch *b, const Chunk &c, char *ws, size_t chunk_index) {
    char *arena = (char *)b->arena;
    char *sm = arena + c.small_off;
    ChunkArgs a;
    a.layers = (const gbmw_layer *)(arena + b->o_layers);
    a.strats = (const gbmw_strategy *)(arena + b->o_strats);
    a.envs = (const gbmw_env *)(arena + b->o_envs);
    a.probs = (const DevProblem *)(sm + c.o_probs);
    a.n_probs = (int32_t)c.probs.size();
    a.max_k = c.max_k;
    a.cell_prefix = (const int64_t *)(sm + c.o_cellp);
    a.r_prefix = (const int64_t *)(sm + c.o_rp);
    a.step_tiles = (const int64_t *)(sm + c.o_stepp);
    a.cand_strat = (const int32_t *)(sm + c.o_cand);
    a.cand_cls = (const int32_t *)(sm + c.o_ccls);
    a.class_d = (const int32_t *)(sm + c.o_clsd);
    a.class_t = (const int32_t *)(sm + c.o_clst);
    a.unit_first = (const int32_t *)(sm + c.o_uf);
    a.unit_count = (const int32_t *)(sm + c.o_uc);
    a.step_map = (const int32_t *)(sm + c.o_stepmap);
    a.cell_coarse = (const int32_t *)(sm + c.o_cellc);
    a.r_coarse = (const int32_t *)(sm + c.o_rc);
    a.unit_coarse = (const int32_t *)(sm + c.o_unitc);
    a.n_cell_coarse = c.n_cellc; a.n_r_coarse = c.n_rc; a.n_unit_coarse = c.n_unitc;
    a.aux_map = (const int2 *)(sm + c.o_aux);
    a.step_lists = (const StepList *)(sm + c.o_slists);
    a.n_step_lists = (int32_t)c.slists.size();
    a.n_aux = c.n_aux;
    const WsLayout w = ws_layout(c);
    a.cells = (Cell *)(ws + w.cells);
    a.cmem = (CellMem *)(ws + w.cmem);
    a.rcls = (double *)(ws + w.rcls);
    a.bup = (unsigned long long *)(ws + w.bup);
    a.step_items = (int4 *)(ws + w.items);
    a.step_ctx = (void *)(ws + w.sctx);
    a.step_count = (int64_t *)(ws + w.scount);
    a.TF[0] = (TFCell *)(ws + w.tf0);
    a.TF[1] = (TFCell *)(ws + w.tf1);
    a.chg[0] = (uint32_t *)(ws + w.chg0);
    a.chg[1] = (uint32_t *)(ws + w.chg1);
    a.rmap = (int2 *)(ws + w.rmap);
    a.k2_erow = (uint16_t *)(ws + w.k2e);
    a.k2_echg = (uint16_t *)(ws + w.k2c);
    a.k2_heavy = (void *)(ws + w.k2h);
    a.k2_rounds = (int2 *)(ws + w.k2r);
    a.par = (uint16_t *)(ws + w.par);
    a.partials = (SweepPartial *)(ws + w.parts);
    a.best = (SweepPartial *)(ws + w.bestp);
    a.bound = (unsigned long long *)(ws + w.bound);
    a.ufirst = (int32_t *)(ws + w.ufirst);
    a.upruned = (int32_t *)(ws + w.upruned);
    a.usorted = (int32_t *)(ws + w.usorted);
    a.uprefix = (int64_t *)(ws + w.uprefix);
    a.ucounter = (unsigned long long *)(ws + w.uctr);
    a.uniq = (int32_t *)(ws + w.uniq);
    a.ucell = (Cell *)(ws + w.ucell);
    a.nuniq = (int32_t *)(ws + w.nuniq);
    a.unit_lo = (int32_t *)(ws + w.ulo);
    a.unit_hi = (int32_t *)(ws + w.uhi);
    a.counters = (unsigned long long *)(ws + w.ctr);
    a.n_units = c.n_units;
    a.results = (gbmw_result *)(arena + b->o_results);
    a.plans = (int32_t *)(arena + b->o_plans);
    a.frontier = (double *)(arena + b->o_frontier);
    a.live_cells = (unsigned long long *)(arena + b->o_stats) + chunk_index;
    a.sweep_stats = (unsigned long long *)(arena + b->o_stats) + 2 * (b->chunks.size() + 1);
    a.computed_cells = (unsigned long long *)(arena + b->o_stats) + (b->chunks.size() + 1) + chunk_index;
    // GBMW_K2_HIST=1: per-tile entry-count histogram of K2 (log2 bins: tiles, entries), printed by run
    static const bool k2_hist = getenv("GBMW_K2_HIST") && getenv("GBMW_K2_HIST")[0] == '1';
    a.k2_hist = k2_hist ? (unsigned long long *)(arena + b->o_stats) + 5 * (b->chunks.size() + 1) : nullptr;
    a.k2_tl = nullptr;
    if (k2_hist) {
        static unsigned long long *tl = nullptr;
        if (!tl) cudaMalloc(&tl, 4096 * 2 * 8);
        a.k2_tl = tl;
    }
    return a;
}

// The sweep / finalize view of one group's problems [lo, lo + n): per-problem arrays offset
// to the group, its own K3b work-list prefix and counter (groups sweep concurrently).
ChunkArgs group_view(const ChunkArgs &a, int lo, int n, int g) {
    ChunkArgs s = a;
    s.probs += lo; s.n_probs = n;
    s.bup += lo; s.best += lo; s.bound += 2 * (int64_t)lo;
    s.ufirst += lo; s.upruned += lo; s.usorted += lo;
    s.uprefix += (int64_t)g * (kMaxSweepRanks + 1);
    s.ucounter += g;
    s.n_aux = 0;
    return s;
}

int cuda_fail(gbmw_ctx *ctx, int rc, const char *what) {
    return set_err(&ctx->err, GBMW_ECUDA, std::string(what) + ": " + cudaGetErrorString((cudaError_t)rc));
}

// Runs K1 for every chunk; with tables_only it stops there (gbmw_cost_tables).
int run_chunks(gbmw_ctx *ctx, gbmw_batch *b, bool tables_only) {
    cudaSetDevice(ctx->device);
    int rc = ensure_ws(ctx, b->max_ws);
    if (rc) return rc;
    b->timing.total_ms = b->timing.dp_ms = b->timing.sweep_ms = b->timing.tables_ms = b->timing.finalize_ms = 0.f;
    b->timing.n_launches = 0;
    cudaStream_t st = ctx->stream;
    cudaMemsetAsync((char *)b->arena + b->o_stats, 0, (5 * (b->chunks.size() + 1) + 64) * 8, st);
    for (Chunk &c : b->chunks) {
        for (auto &e : c.ev)
            if (!e) cudaEventCreate(&e);
        ChunkArgs a = chunk_args(b, c, (char *)ctx->ws, (size_t)(&c - b->chunks.data()));
        c.launches = 0;
        cudaEventRecord(c.ev[0], st);
        cudaMemsetAsync(a.bup, 0, c.probs.size() * 8, st);
        cudaMemsetAsync(a.counters, 0, (size_t)(c.Umax + 1) * kNumGroups * 3 * 8, st);
        if ((rc = launch_cost_tables(a, c.n_cells, c.n_r, st))) return cuda_fail(ctx, rc, "K1 launch");
        c.launches += (c.n_cells > 0) + (c.n_r > 0) + 2 * (c.n_units > 0 && !c.probs.empty());
        cudaEventRecord(c.ev[1], st);
        if (tables_only) continue;
        // K2l on its own stream from the fork: the bands' first steps (K2f, K2s) need no
        // items, so the list kernel runs beside them; a band waits for it before its first
        // tiled step
        bool lists = false;
        if (!c.slists.empty()) {
            if (!ctx->list_stream) {
                int lo_pri = 0, hi_pri = 0;
                cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri);
                if (cudaStreamCreateWithPriority(&ctx->list_stream, cudaStreamNonBlocking, hi_pri) != cudaSuccess ||
                    cudaEventCreateWithFlags(&ctx->list_done, cudaEventDisableTiming) != cudaSuccess)
                    return cuda_fail(ctx, (int)cudaGetLastError(), "list stream");
            }
            if (!ctx->fork && cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming) != cudaSuccess)
                return cuda_fail(ctx, (int)cudaGetLastError(), "fork event");
            cudaEventRecord(ctx->fork, st);
            cudaStreamWaitEvent(ctx->list_stream, ctx->fork, 0);
            if ((rc = launch_step_lists(a, ctx->list_stream))) return cuda_fail(ctx, rc, "K2 list launch");
            cudaEventRecord(ctx->list_done, ctx->list_stream);
            c.launches += 1;
            lists = true;
        }
        // the class-count groups (and the collapsed-DP problems) are independent problems:
        // group 0 on the main stream, the others on their own streams, joined before K3
        bool used[kNumGroups] = {false};
        for (size_t s = 0; s < c.slists.size(); ++s) used[c.slist_group[s]] = true;
        used[kApproxGroup] = c.n_active[kApproxGroup].size() > 1 && c.n_active[kApproxGroup][0] > 0;
        cudaStream_t gs[kNumGroups];
        gs[0] = st;
        bool forked = false;
        for (int g = 1; g < kNumGroups; ++g) {
            gs[g] = st;
            if (!used[g]) continue;
            if (!ctx->aux[g]) {
                // deep bands (the critical path: one launch per unit) get the higher priority
                int lo_pri = 0, hi_pri = 0;
                cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri);
                // deep bands above shallow ones; among deep bands the wider classes (their
                // steps are the longest) above the main stream's K <= 4 band
                const int pri = (g < kStepVGroups && !shallow_group(g)) ? hi_pri : lo_pri;
                if (cudaStreamCreateWithPriority(&ctx->aux[g], cudaStreamNonBlocking, pri) != cudaSuccess ||
                    cudaEventCreateWithFlags(&ctx->join[g], cudaEventDisableTiming) != cudaSuccess)
                    return cuda_fail(ctx, (int)cudaGetLastError(), "aux stream");
            }
            if (!ctx->fork && cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming) != cudaSuccess)
                return cuda_fail(ctx, (int)cudaGetLastError(), "fork event");
            if (!forked && !lists) cudaEventRecord(ctx->fork, st);
            forked = true;
            cudaStreamWaitEvent(ctx->aux[g], ctx->fork, 0);
            gs[g] = ctx->aux[g];
        }
        static const bool k2_spans = getenv("GBMW_K2_HIST") && getenv("GBMW_K2_HIST")[0] == '1';
        if (k2_spans && a.k2_tl) {
            std::vector<unsigned long long> init(4096 * 2);
            for (size_t i = 0; i < init.size(); i += 2) { init[i] = ~0ull; init[i + 1] = 0ull; }
            cudaMemcpyAsync(a.k2_tl, init.data(), init.size() * 8, cudaMemcpyHostToDevice, st);
            cudaStreamSynchronize(st);
        }
        if (k2_spans)
            for (int g = 0; g < kNumGroups; ++g) {
                if (!used[g] && g != 0) continue;
                if (!ctx->gspan[g][0]) { cudaEventCreate(&ctx->gspan[g][0]); cudaEventCreate(&ctx->gspan[g][1]); }
                cudaEventRecord(ctx->gspan[g][0], gs[g]);
            }
        bool have_items[kNumGroups] = {false};
        for (size_t s = 0; s < c.slists.size(); ++s) {
            const StepList &sl = c.slists[s];
            const int g = c.slist_group[s];
            if (!sl.no_items && !have_items[g]) {        // first tiled step of this stream
                cudaStreamWaitEvent(gs[g], ctx->list_done, 0);
                have_items[g] = true;
            }
            const int64_t ub = (s + 1 < c.slists.size() ? c.slists[s + 1].base : c.n_items) - sl.base;   // item bound
            int2 *rounds = a.k2_rounds + 2 * c.step_prefix[c.group_lo[g]] * kK2RoundsPerSlot;
            if (sl.u == 1) {                             // first step: segments of the first unit's weights
                if ((rc = launch_dp_first(a, sl.lo, sl.n, gs[g]))) return cuda_fail(ctx, rc, "K2 first launch");
                c.launches += 1;
                continue;
            }
            if (c.slist_second[s]) {                     // second step: candidate rows of few-source problems
                if ((rc = launch_dp_second(a, g / kBands, sl.lo, sl.n, gs[g]))) return cuda_fail(ctx, rc, "K2 second launch");
                c.launches += 1;
                continue;
            }
            int nk = 0;
            if ((rc = launch_dp_step(a, g / kBands, sl.u, a.step_items + sl.base, a.step_count + s, ub,
                                     a.counters + ((size_t)sl.u * kNumGroups + g) * 3, rounds, (int)s, gs[g], &nk)))
                return cuda_fail(ctx, rc, "K2 launch");
            c.launches += nk;
        }
        // approx_prev problems: collapsed-state layer steps, unit 0 included
        for (int u = 0; u < c.Umax; ++u) {
            const int lo = c.group_lo[kApproxGroup], na = c.n_active[kApproxGroup][u];
            if (na == 0) continue;
            const int64_t base = c.step_prefix[lo], n = c.step_prefix[lo + na] - base;
            if ((rc = launch_approx_step(a, u, base, n, a.counters + ((size_t)u * kNumGroups + kApproxGroup) * 3,
                                         gs[kApproxGroup])))
                return cuda_fail(ctx, rc, "K2c launch");
            c.launches += 1;
        }
        if (k2_spans)
            for (int g = 0; g < kNumGroups; ++g)
                if (used[g] || g == 0) cudaEventRecord(ctx->gspan[g][1], gs[g]);
        // Without K3r tiles (frontier requests, collapsed-DP problems) every group sweeps and
        // finalises its own problems on its own stream right after its last layer step, so
        // the shallow groups' K3/K4 run while the deep groups are still in K2.  ev[2] marks
        // the end of K2 on every stream (a timing stream waits for all of them).
        static const bool no_group_sweep = getenv("GBMW_SWEEP_PER_GROUP") && getenv("GBMW_SWEEP_PER_GROUP")[0] == '0';
        // shallow groups' K3b at 3 CTAs per SM (occupancy allows 4): the deep groups' layer
        // steps keep SM slots (measured on the 10k sweep: 2 per SM 7.53-7.67 ms, 3 per SM 7.44-7.51,
        // 4 per SM 8.04-8.08, one sweep after every group's K2 7.70-7.75)
        static const int group_ctas = getenv("GBMW_SWEEP_GROUP_CTAS") ? atoi(getenv("GBMW_SWEEP_GROUP_CTAS")) : 3;
        static const int group_min = getenv("GBMW_SWEEP_GROUP_MIN") ? atoi(getenv("GBMW_SWEEP_GROUP_MIN")) : 2000;
        const bool per_group = c.n_aux == 0 && (int64_t)c.probs.size() >= group_min && !no_group_sweep;
        if (per_group) {
            if (!ctx->tstream) {
                if (cudaStreamCreateWithFlags(&ctx->tstream, cudaStreamNonBlocking) != cudaSuccess)
                    return cuda_fail(ctx, (int)cudaGetLastError(), "timing stream");
                for (auto &e : ctx->k2done)
                    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
                        return cuda_fail(ctx, (int)cudaGetLastError(), "K2 done events");
            }
            for (int g = 0; g < kNumGroups; ++g) {
                if (g != 0 && gs[g] == st) continue;
                cudaEventRecord(ctx->k2done[g], gs[g]);
                cudaStreamWaitEvent(ctx->tstream, ctx->k2done[g], 0);
            }
            if (lists) cudaStreamWaitEvent(ctx->tstream, ctx->list_done, 0);
            cudaEventRecord(c.ev[2], ctx->tstream);
            for (int g = 0; g < kNumGroups; ++g) {
                const int lo = c.group_lo[g], n = c.group_lo[g + 1] - lo;
                if (n <= 0) continue;
                const ChunkArgs sub = group_view(a, lo, n, g);
                if ((rc = launch_sweep(sub, gs[g], shallow_group(g) ? group_ctas : 0))) return cuda_fail(ctx, rc, "K3 launch");
                if ((rc = launch_finalize(sub, gs[g]))) return cuda_fail(ctx, rc, "K4 launch");
                c.launches += 4;
            }
        }
        for (int g = 1; g < kNumGroups; ++g) {
            if (gs[g] == st) continue;
            cudaEventRecord(ctx->join[g], gs[g]);
            cudaStreamWaitEvent(st, ctx->join[g], 0);
        }
        if (lists) cudaStreamWaitEvent(st, ctx->list_done, 0);
        if (per_group) {
            cudaEventRecord(c.ev[3], st);                // sweep_ms: K3 + K4 past the end of K2
            cudaEventRecord(c.ev[4], st);
        } else {
            cudaEventRecord(c.ev[2], st);
            if ((rc = launch_sweep(a, st))) return cuda_fail(ctx, rc, "K3 launch");
            cudaEventRecord(c.ev[3], st);
            if ((rc = launch_finalize(a, st))) return cuda_fail(ctx, rc, "K4 launch");
            c.launches += 4 + (c.n_aux > 0);
            cudaEventRecord(c.ev[4], st);
        }
    }
    cudaError_t ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return cuda_fail(ctx, (int)ce, "search kernels");
    for (Chunk &c : b->chunks) {
        float t;
        b->timing.n_launches += c.launches;
        cudaEventElapsedTime(&t, c.ev[0], c.ev[1]); b->timing.tables_ms += t;
        if (tables_only) continue;
        cudaEventElapsedTime(&t, c.ev[1], c.ev[2]); b->timing.dp_ms += t;
        cudaEventElapsedTime(&t, c.ev[2], c.ev[3]); b->timing.sweep_ms += t;
        cudaEventElapsedTime(&t, c.ev[3], c.ev[4]); b->timing.finalize_ms += t;
        cudaEventElapsedTime(&t, c.ev[0], c.ev[4]); b->timing.total_ms += t;
    }
    if (!tables_only && !b->chunks.empty()) {
        // K2 algorithmic bytes = 34 B per live class cell
        std::vector<unsigned long long> live(5 * (b->chunks.size() + 1));
        cudaMemcpy(live.data(), (char *)b->arena + b->o_stats, live.size() * 8, cudaMemcpyDeviceToHost);
        const size_t nc = b->chunks.size();
        double cells = 0.0;
        for (size_t i = 0; i <= nc; ++i) cells += (double)live[i];
        double computed = 0.0;
        for (size_t i = 0; i < nc; ++i) computed += (double)live[nc + 1 + i];
        b->timing.sweep_rows = (double)live[2 * (nc + 1)];
        b->timing.sweep_cands = (double)live[2 * (nc + 1) + 1];
        b->timing.sweep_checks = (double)live[2 * (nc + 1) + 2];
        // writes of every live class cell (t, f, argmin) + source reads of the rows evaluated
        b->timing.dp_bytes = cells * 18.0 + computed * 16.0;
        b->timing.dp_cells = computed;
        b->timing.live_cells = cells;
        if (getenv("GBMW_K2_HIST") && getenv("GBMW_K2_HIST")[0] == '1') {
            std::vector<unsigned long long> h(64);
            cudaMemcpy(h.data(), (char *)b->arena + b->o_stats + 5 * (nc + 1) * 8, 64 * 8, cudaMemcpyDeviceToHost);
            for (int g = 0; g < kNumGroups; ++g) {
                float ms = 0.f;
                if (ctx->gspan[g][0] && cudaEventElapsedTime(&ms, ctx->gspan[g][0], ctx->gspan[g][1]) == cudaSuccess)
                    fprintf(stderr, "K2 stream of group %d: %.3f ms\n", g, ms);
            }
            {
                ChunkArgs al = chunk_args(b, b->chunks.back(), (char *)ctx->ws, b->chunks.size() - 1);
                if (al.k2_tl) {
                    const Chunk &cc = b->chunks.back();
                    std::vector<unsigned long long> tl(4096 * 2);
                    cudaMemcpy(tl.data(), al.k2_tl, tl.size() * 8, cudaMemcpyDeviceToHost);
                    std::vector<unsigned long long> ctrs((size_t)(cc.Umax + 1) * kNumGroups * 3);
                    cudaMemcpy(ctrs.data(), al.counters, ctrs.size() * 8, cudaMemcpyDeviceToHost);
                    unsigned long long t0 = ~0ull;
                    const size_t nl = std::min<size_t>(cc.slists.size(), 2048);
                    for (size_t l = 0; l < 2 * nl; ++l) t0 = std::min(t0, tl[2 * l]);
                    for (size_t l = 0; l < nl; ++l)
                        fprintf(stderr, "TL u=%d g=%d a=[%.1f, %.1f] b=[%.1f, %.1f] us rounds=%llu\n", cc.slists[l].u,
                                cc.slist_group[l], (tl[4 * l] - t0) / 1e3, (tl[4 * l + 1] - t0) / 1e3,
                                (tl[4 * l + 2] - t0) / 1e3, (tl[4 * l + 3] - t0) / 1e3,
                                ctrs[((size_t)cc.slists[l].u * kNumGroups + cc.slist_group[l]) * 3 + 1]);
                }
            }
            fprintf(stderr, "K2 tiles by entries (bin: <2^b entries): ");
            for (int i = 0; i < 31; ++i)
                if (h[i]) fprintf(stderr, "[%d] %llu tiles %llu ent  ", i, h[i], h[32 + i]);
            fprintf(stderr, "\nK3b items %llu, skipped by flag %llu, restagings %llu, pruned by t0 %llu\n", h[56], h[57],
                    h[58], h[59]);
            // per launch: items, tiles (first chunk)
            const Chunk &c0 = b->chunks[0];
            const Chunk &cl = b->chunks.back();
            (void)c0;
            ChunkArgs a0 = chunk_args(b, cl, (char *)ctx->ws, b->chunks.size() - 1);
            std::vector<int64_t> cnt(cl.slists.size());
            std::vector<int4> items(cl.n_items);
            cudaMemcpy(cnt.data(), a0.step_count, cnt.size() * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(items.data(), a0.step_items, items.size() * sizeof(int4), cudaMemcpyDeviceToHost);
            for (size_t l = 0; l < cl.slists.size(); ++l) {
                long long tiles = 0;
                for (int64_t i = 0; i < cnt[l]; ++i) tiles += items[cl.slists[l].base + i].z - items[cl.slists[l].base + i].y + 1;
                fprintf(stderr, "u=%d g=%d problems=%d items=%lld tiles=%lld\n", cl.slists[l].u, cl.slist_group[l],
                        cl.slists[l].n, (long long)cnt[l], tiles);
            }
        }
    }
    b->ran = true;
    ctx->last = b->timing;
    return GBMW_OK;
}
}  // namespace

extern "C" int gbmw_batch_run(gbmw_ctx *ctx, gbmw_batch *b) {
    if (!ctx || !b) return set_err(nullptr, GBMW_EINVAL, "null ctx/batch");
    return run_chunks(ctx, b, false);
}

extern "C" int gbmw_batch_fetch(gbmw_ctx *ctx, gbmw_batch *b, gbmw_result *results, int32_t *plans, double *frontier) {
    if (!ctx || !b) return set_err(nullptr, GBMW_EINVAL, "null ctx/batch");
    if (!b->ran && !b->chunks.empty()) return set_err(&ctx->err, GBMW_EINVAL, "batch has not been run");
    const double t0 = now_ms();
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const size_t np = b->problems.size();
    // results | plans | frontier are contiguous in the arena: one copy through the
    // context's pinned staging buffer, then out to the caller's arrays
    const size_t lo = b->o_results;
    const size_t hi = (frontier && b->total_frontier) ? b->o_frontier + (size_t)b->total_frontier * sizeof(double)
                                                      : b->o_plans + (size_t)b->total_plan * sizeof(int32_t);
    const size_t nbytes = hi > lo ? hi - lo : 0;
    if (ctx->pinned_cap < nbytes) {
        if (ctx->pinned) cudaFreeHost(ctx->pinned);
        ctx->pinned = nullptr;
        ctx->pinned_cap = 0;
        const size_t cap = std::max<size_t>(nbytes + nbytes / 4, 1u << 20);
        if (cudaHostAlloc(&ctx->pinned, cap, cudaHostAllocDefault) == cudaSuccess) ctx->pinned_cap = cap;
    }
    std::vector<char> fallback;
    char *host = (char *)ctx->pinned;
    if (!host) { fallback.resize(nbytes); host = fallback.data(); }
    cudaError_t ce = cudaSuccess;
    if (nbytes) ce = cudaMemcpyAsync(host, (char *)b->arena + lo, nbytes, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return cuda_fail(ctx, (int)ce, "fetch");
    const gbmw_result *dev_res = reinterpret_cast<const gbmw_result *>(host);
    if (plans && b->total_plan) std::memcpy(plans, host + (b->o_plans - lo), (size_t)b->total_plan * sizeof(int32_t));
    if (frontier && b->total_frontier)
        std::memcpy(frontier, host + (b->o_frontier - lo), (size_t)b->total_frontier * sizeof(double));
    b->timing.d2h_bytes = (double)(np * sizeof(gbmw_result)) + (plans ? (double)b->total_plan * 4.0 : 0.0) +
                          (frontier ? (double)b->total_frontier * 8.0 : 0.0);
    // the device's entries in one copy, then the host's (problems without device work, and
    // frontier offsets); the first failing status in problem order
    auto host_entry = [&](size_t i, gbmw_result &r) {
        const HostProb &h = b->hp[i];
        if (h.gpu) {
            r = dev_res[i];
            r.frontier_offset = h.frontier_off;
            return;
        }
        std::memset(&r, 0, sizeof(r));
        r.time_s = INFINITY;
        r.e_fwd_used = 0.0;
        r.feasible = 0;
        r.status = h.status;
        r.frontier_offset = -1;
        if (plans)
            for (int l = 0; l < std::max<int32_t>(0, b->problems[i].n_layers); ++l) plans[h.plan_off + l] = -1;
    };
    int first = GBMW_OK;
    if (results) {
        if (np) std::memcpy(results, dev_res, np * sizeof(gbmw_result));
        for (int32_t i : b->host_fix) host_entry((size_t)i, results[i]);
        for (size_t i = 0; i < np && first == GBMW_OK; ++i)
            if (results[i].status != GBMW_OK) first = results[i].status;
    } else {
        for (size_t i = 0; i < np; ++i) {
            gbmw_result r;
            host_entry(i, r);
            if (r.status != GBMW_OK && first == GBMW_OK) first = r.status;
        }
    }
    if (first == GBMW_EINTERNAL) set_err(&ctx->err, first, "dp_search produced a plan exceeding the memory budget");
    b->timing.fetch_ms = now_ms() - t0;
    ctx->last = b->timing;
    return first;
}

extern "C" int gbmw_batch_timing(const gbmw_batch *b, gbmw_timing *out) {
    if (!b || !out) return set_err(nullptr, GBMW_EINVAL, "null batch/out");
    *out = b->timing;
    return GBMW_OK;
}

extern "C" int gbmw_ctx_last_timing(const gbmw_ctx *ctx, gbmw_timing *out) {
    if (!ctx || !out) return set_err(nullptr, GBMW_EINVAL, "null ctx/out");
    *out = ctx->last;
    return GBMW_OK;
}

// gbmw_seed_partitions on the device (csrc/gbmw_seed.cu): one warp per
// cell, the hill climb's moves across the lanes.  Same contract as the host function.
extern "C" int gbmw_seed_partitions_device(gbmw_ctx *ctx, const gbmw_layer *layers, int32_t n_layers,
                                           const gbmw_env *env, int64_t n_devices, int32_t n_cells,
                                           const int64_t *pp_degree, const int64_t *micro_batch,
                                           const int32_t *n_micro, double budget, int32_t max_stages,
                                           int32_t *out_sizes) {
    if (!ctx || !layers || !env || !pp_degree || !micro_batch || !n_micro || !out_sizes || n_cells < 0 ||
        max_stages < 1 || n_layers < 1)
        return set_err(ctx ? &ctx->err : nullptr, GBMW_EINVAL, "bad arguments");
    if (!gbmw_sum_semantics())
        return set_err(&ctx->err, GBMW_ENOTSUP, "device seed partitions implement CPython >= 3.12 sum() only");
    if (n_cells == 0) return GBMW_OK;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const size_t b_layers = (size_t)n_layers * sizeof(gbmw_layer), b_env = sizeof(gbmw_env);
    const size_t b_cells = (size_t)n_cells * (8 + 8 + 4), b_out = (size_t)n_cells * ((size_t)max_stages + 1) * 4;
    const size_t b_scr = (size_t)n_cells * n_layers * 8;
    size_t o = 0;
    const size_t o_layers = o; o = align_up(o + b_layers);
    const size_t o_env = o; o = align_up(o + b_env);
    const size_t o_pp = o; o = align_up(o + (size_t)n_cells * 8);
    const size_t o_mb = o; o = align_up(o + (size_t)n_cells * 8);
    const size_t o_nm = o; o = align_up(o + (size_t)n_cells * 4);
    const size_t up = o;
    const size_t o_out = o; o = align_up(o + b_out);
    const size_t o_scr = o; o = align_up(o + b_scr);
    (void)b_cells;
    if (ctx->seed_cap < o) {
        if (ctx->seed_buf) cudaFree(ctx->seed_buf);
        ctx->seed_buf = nullptr;
        ctx->seed_cap = 0;
        if (cudaMalloc(&ctx->seed_buf, o + o / 4) != cudaSuccess)
            return set_err(&ctx->err, GBMW_ENOMEM, "cudaMalloc(seed partitions)");
        ctx->seed_cap = o + o / 4;
    }
    std::vector<char> host(up);
    std::memcpy(host.data() + o_layers, layers, b_layers);
    std::memcpy(host.data() + o_env, env, b_env);
    std::memcpy(host.data() + o_pp, pp_degree, (size_t)n_cells * 8);
    std::memcpy(host.data() + o_mb, micro_batch, (size_t)n_cells * 8);
    std::memcpy(host.data() + o_nm, n_micro, (size_t)n_cells * 4);
    char *dev = (char *)ctx->seed_buf;
    cudaError_t ce = cudaMemcpyAsync(dev, host.data(), up, cudaMemcpyHostToDevice, st);
    int rc = (ce == cudaSuccess)
                 ? launch_seed_partitions((const gbmw_layer *)(dev + o_layers), n_layers, (const gbmw_env *)(dev + o_env),
                                          n_devices, n_cells, (const int64_t *)(dev + o_pp),
                                          (const int64_t *)(dev + o_mb), (const int32_t *)(dev + o_nm), budget,
                                          max_stages, (double *)(dev + o_scr), (int32_t *)(dev + o_out),
                                          (int32_t *)(dev + o_out) + (size_t)n_cells * max_stages, st)
                 : (int)ce;
    if (rc) return cuda_fail(ctx, rc, "seed partitions launch");
    std::vector<int32_t> out((size_t)n_cells * (max_stages + 1));
    ce = cudaMemcpyAsync(out.data(), dev + o_out, out.size() * 4, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return cuda_fail(ctx, (int)ce, "seed partitions");
    const int32_t *status = out.data() + (size_t)n_cells * max_stages;
    for (int i = 0; i < n_cells; ++i)
        if (status[i])
            return set_err(&ctx->err, status[i], "seed partition of cell " + std::to_string(i) + " failed (status " +
                                                     std::to_string(status[i]) + ")");
    std::memcpy(out_sizes, out.data(), (size_t)n_cells * max_stages * 4);
    return GBMW_OK;
}

extern "C" int gbmw_batch_destroy(gbmw_batch *b) {
    if (!b) return GBMW_OK;
    for (Chunk &c : b->chunks)
        for (auto &e : c.ev)
            if (e) cudaEventDestroy(e);
    if (b->ctx_arena) b->ctx->arena_busy = false;
    else if (b->arena) cudaFree(b->arena);
    gbmw_ctx *ctx = b->ctx;
    if (ctx && !ctx->spare) {
        // keep the batch's host vectors (their capacity) for the next gbmw_batch_create on
        // this context: a 10k-search batch otherwise page-faults ~2 MB of fresh buffers
        b->layers.clear(); b->strats.clear(); b->envs.clear(); b->problems.clear();   // hp keeps its records
        b->chunks.clear();
        b->strat_recs.clear(); b->unit_recs.clear();
        b->total_plan = b->total_frontier = 0;
        b->arena = nullptr; b->arena_size = 0;
        b->o_layers = b->o_strats = b->o_envs = b->o_results = b->o_plans = b->o_frontier = b->o_stats = 0;
        b->max_ws = 0; b->timing = gbmw_timing{}; b->ran = false; b->ctx = nullptr; b->ctx_arena = false;
        ctx->spare = b;
    } else {
        delete b;
    }
    return GBMW_OK;
}

extern "C" int gbmw_search_batch(gbmw_ctx *ctx, const gbmw_layer *layers, int64_t n_layers,
                                 const gbmw_strategy *strategies, int64_t n_strategies, const gbmw_env *envs,
                                 int64_t n_envs, const gbmw_problem *problems, int64_t n_problems,
                                 gbmw_result *results, int32_t *plans, double *frontier) {
    gbmw_batch *b = nullptr;
    int rc = gbmw_batch_create(ctx, layers, n_layers, strategies, n_strategies, envs, n_envs, problems, n_problems, &b);
    if (!b) return rc;
    const int prep_rc = rc;
    rc = gbmw_batch_run(ctx, b);
    if (rc == GBMW_OK) rc = gbmw_batch_fetch(ctx, b, results, plans, frontier);
    gbmw_batch_destroy(b);
    if (rc == GBMW_OK) rc = prep_rc;
    return rc;
}

extern "C" int gbmw_cost_tables(gbmw_ctx *ctx, const gbmw_layer *layers, int64_t n_layers,
                                const gbmw_strategy *strategies, int64_t n_strategies, const gbmw_env *envs,
                                int64_t n_envs, const gbmw_problem *problem, double *time_c, double *ef_true,
                                double *o_b, int64_t *weight, int32_t *usable, int32_t *n_usable, int32_t *n_units) {
    gbmw_batch *b = nullptr;
    int rc = gbmw_batch_create(ctx, layers, n_layers, strategies, n_strategies, envs, n_envs, problem, 1, &b);
    if (!b) return rc;
    if (rc != GBMW_OK) { gbmw_batch_destroy(b); return rc; }
    const HostProb &h = b->hp[0];
    if (n_usable) *n_usable = h.S;
    if (n_units) *n_units = h.U;
    if (usable)
        for (int i = 0; i < h.S; ++i) usable[i] = h.si->cand[i] - problem->strat_begin;
    if (!h.gpu) { gbmw_batch_destroy(b); return GBMW_OK; }
    rc = run_chunks(ctx, b, true);
    if (rc == GBMW_OK) {
        const Chunk &c = b->chunks[0];
        const WsLayout w = ws_layout(c);
        std::vector<Cell> cells(c.n_cells);
        std::vector<CellMem> cm(c.n_cells);
        cudaMemcpy(cells.data(), (char *)ctx->ws + w.cells, c.n_cells * sizeof(Cell), cudaMemcpyDeviceToHost);
        cudaError_t ce = cudaMemcpy(cm.data(), (char *)ctx->ws + w.cmem, c.n_cells * sizeof(CellMem), cudaMemcpyDeviceToHost);
        if (ce != cudaSuccess) rc = cuda_fail(ctx, (int)ce, "cost tables fetch");
        for (int64_t x = 0; x < c.n_cells && rc == GBMW_OK; ++x) {
            if (time_c) time_c[x] = cells[x].c;
            if (ef_true) ef_true[x] = cells[x].ef;
            if (o_b) o_b[x] = cm[x].o_b;
            if (weight) weight[x] = cells[x].w;
        }
    }
    gbmw_batch_destroy(b);
    return rc;
}

// ----------------------------------------------------------------------------- brute-force oracle
// planner.brute_force_oracle (planner.py:364-449) on the device (gbmw_brute.cu).  The host
// walks the reference's loops — candidate_pp_degrees (strategies.py:213-219), P <= L, the
// divisors m of the batch in ascending order, the usable strategies of the pruned set —
// builds each cell's per-(layer, strategy) tables with the shared cost model and its
// compositions in _compositions order (planner.py:354-361); the device scans every
// (partition, assignment) of all cells; the host then keeps the first cell whose minimum
// is strictly below the running best (planner.py:437).
namespace {
void compositions(int total, int parts, int start, uint32_t mask, std::vector<uint32_t> &out) {
    // ordered splits of layers [start, start + total) into `parts` nonempty stages, heads
    // ascending (the recursion order of planner.py:354-361); bit l marks a stage start
    mask |= 1u << start;
    if (parts == 1) { out.push_back(mask); return; }
    for (int head = 1; head <= total - parts + 1; ++head)
        compositions(total - head, parts - 1, start + head, mask, out);
}
}  // namespace

extern "C" int gbmw_brute_force(gbmw_ctx *ctx, const gbmw_layer *layers, int32_t n_layers, const gbmw_env *env,
                                int64_t batch, double budget_bytes, double max_combos, int32_t *out_partition,
                                int32_t *out_choice, gbmw_oracle_result *out) {
    if (!ctx || !layers || !env || !out || !out_partition || !out_choice)
        return set_err(ctx ? &ctx->err : nullptr, GBMW_EINVAL, "null argument");
    std::string *err = &ctx->err;
    if (n_layers < 1) return set_err(err, GBMW_EEMPTY, "model must contain at least one layer");
    if (n_layers > kBruteMaxLayers)
        return set_err(err, GBMW_ENOTSUP, "brute force limited to " + std::to_string(kBruteMaxLayers) + " layers");
    if (batch < 1) return set_err(err, GBMW_EMICRO, "batch must be >= 1, got " + std::to_string(batch));
    if (!(budget_bytes >= 0.0) || budget_bytes >= kTwo53)
        return set_err(err, GBMW_ERANGE, "budget_bytes must lie in [0, 2^53)");
    if (!is_pow2(env->n_devices))
        return set_err(err, GBMW_EINVAL, "device count must be a power of two, got " + std::to_string(env->n_devices));
    for (int l = 0; l < n_layers; ++l) {
        int rc = check_layer(layers[l], err);
        if (rc) return rc;
        if (!prod_exact(layers[l].bnd_bytes_per_sample, batch) || !prod_exact(layers[l].int_bytes_per_sample, batch) ||
            !prod_exact(layers[l].bnd_bytes_per_sample * batch, std::max<int64_t>(1, std::min<int64_t>(env->n_devices, batch))))
            return set_err(err, GBMW_ERANGE, "byte products of a layer reach 2^53; fp64 would not be exact");
    }
    const double cap = max_combos > 0.0 ? max_combos : 17592186044416.0;   // 2^44 assignments
    const int L = n_layers;
    struct CellHost {
        int P, m;
        std::vector<int32_t> cand;      // usable positions in the pruned strategy set
    };
    std::vector<CellHost> ch;
    std::vector<BruteCell> cells;
    std::vector<double> tab;
    std::vector<uint32_t> comps;
    double total = 0.0;
    int64_t parts = 0;
    for (int64_t P = 1; P <= env->n_devices; P *= 2) {
        if (P > L) continue;
        int32_t ns = 0;
        int rc = gbmw_enumerate(env->n_devices, P, 1, nullptr, 0, &ns);
        if (rc) return set_err(err, rc, g_err);
        std::vector<gbmw_strategy> sset(ns);
        gbmw_enumerate(env->n_devices, P, 1, sset.data(), ns, &ns);
        const int64_t comp_off = (int64_t)comps.size();
        compositions(L, (int)P, 0, 0u, comps);
        const int64_t n_comp = (int64_t)comps.size() - comp_off;
        for (int64_t m = 1; m <= batch; ++m) {
            if (batch % m) continue;
            const int64_t micro = batch / m;
            CellHost c{(int)P, (int)m, {}};
            std::vector<StratDeg> deg;
            for (int i = 0; i < ns; ++i) {
                const StratDeg d = strat_degrees(sset[i]);
                if (micro % d.data == 0) { c.cand.push_back(i); deg.push_back(d); }
            }
            if (c.cand.empty()) continue;
            const int S = (int)c.cand.size();
            double spow = 1.0;
            for (int l = 0; l < L - 1; ++l) spow *= S;
            const double combos = (double)n_comp * spow * S;
            total += combos;
            if (total > cap)
                return set_err(err, GBMW_ENOTSUP, "brute force over " + std::to_string(total) +
                                                      "+ assignments exceeds the limit of " + std::to_string(cap));
            BruteCell bc{};
            bc.S = S; bc.L = L; bc.P = (int)P; bc.n_micro = (int)m;
            bc.n_comp = n_comp; bc.spow = (int64_t)spow; bc.n_items = n_comp * bc.spow;
            bc.comp_off = comp_off;
            bc.tab_off = (int64_t)tab.size();
            bc.budget = budget_bytes;
            const int64_t LS = (int64_t)L * S;
            tab.resize(tab.size() + 5 * LS + L + LS * S);
            double *T = tab.data() + bc.tab_off;
            for (int l = 0; l < L; ++l) {
                for (int j = 0; j < S; ++j) {
                    const gbmw_strategy &s = sset[c.cand[j]];
                    double t, tns;
                    layer_times(layers[l], s, deg[j], micro, *env, &t, &tns);
                    const Mem mem = layer_memory(layers[l], deg[j], micro, 1, 1, env->ms_bytes_per_param_byte);
                    T[0 * LS + l * S + j] = t;
                    T[1 * LS + l * S + j] = tns;
                    T[2 * LS + l * S + j] = mem.o_f;
                    T[3 * LS + l * S + j] = mem.o_b;
                    T[4 * LS + l * S + j] = mem.o_ms;
                    for (int a = 0; a < S; ++a)
                        T[5 * LS + L + ((int64_t)l * S + a) * S + j] =
                            transform_cost(layers[l].bnd_bytes_per_sample, deg[a].data, deg[a].tp, deg[j].data,
                                           deg[j].tp, micro, env->intra_island_bw);
                }
                T[5 * LS + l] = stage_p2p_time(layers[l].bnd_bytes_per_sample, micro, (int32_t)P, *env);
            }
            bc.tab_len = 5 * LS + L + LS * S;
            bc.smem_doubles = bc.tab_len * 8 <= 200 * 1024 ? (int32_t)bc.tab_len : 0;
            bc.n_parts = brute_blocks(bc.n_items);
            bc.part_off = parts;
            parts += bc.n_parts;
            cells.push_back(bc);
            ch.push_back(std::move(c));
        }
    }
    out->cost = INFINITY;
    out->feasible = 0;
    out->pp_degree = out->n_micro = out->n_stages = 0;
    out->combos = total;
    out->device_ms = 0.0;
    for (int l = 0; l < L; ++l) { out_partition[l] = 0; out_choice[l] = -1; }
    const int nc = (int)cells.size();
    if (nc == 0) return GBMW_OK;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const size_t b_cells = (size_t)nc * sizeof(BruteCell), b_tab = tab.size() * 8, b_comp = comps.size() * 4;
    const size_t b_part = (size_t)parts * sizeof(BrutePartial), b_out = (size_t)nc * sizeof(BrutePartial);
    size_t o = 0;
    const size_t o_cells = o; o = align_up(o + b_cells);
    const size_t o_tab = o; o = align_up(o + b_tab);
    const size_t o_comp = o; o = align_up(o + b_comp);
    const size_t up = o;
    const size_t o_part = o; o = align_up(o + b_part);
    const size_t o_out = o; o = align_up(o + b_out);
    char *dev = nullptr;
    if (cudaMalloc(&dev, o) != cudaSuccess) return set_err(err, GBMW_ENOMEM, "cudaMalloc(brute force)");
    std::vector<char> host(up);
    std::memcpy(host.data() + o_cells, cells.data(), b_cells);
    std::memcpy(host.data() + o_tab, tab.data(), b_tab);
    std::memcpy(host.data() + o_comp, comps.data(), b_comp);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaError_t ce = cudaMemcpyAsync(dev, host.data(), up, cudaMemcpyHostToDevice, st);
    int rc = (int)ce;
    if (rc == 0) cudaEventRecord(e0, st);
    const int neu = gbmw_sum_semantics();
    for (int i = 0; i < nc && rc == 0; ++i)
        rc = launch_brute_cell(cells[i], (const BruteCell *)(dev + o_cells), (const double *)(dev + o_tab),
                               (const uint32_t *)(dev + o_comp), (BrutePartial *)(dev + o_part), i, neu, st);
    if (rc == 0)
        rc = launch_brute_reduce((const BruteCell *)(dev + o_cells), nc, (const BrutePartial *)(dev + o_part),
                                 (BrutePartial *)(dev + o_out), st);
    if (rc == 0) cudaEventRecord(e1, st);
    std::vector<BrutePartial> res(nc);
    if (rc == 0) rc = (int)cudaMemcpyAsync(res.data(), dev + o_out, b_out, cudaMemcpyDeviceToHost, st);
    if (rc == 0) rc = (int)cudaStreamSynchronize(st);
    float ms = 0.f;
    if (rc == 0) cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(dev);
    if (rc) return cuda_fail(ctx, rc, "brute force");
    out->device_ms = ms;
    // strict `<` over the cells in the reference's loop order (planner.py:437)
    int best = -1;
    double best_cost = INFINITY;
    for (int i = 0; i < nc; ++i) {
        if (res[i].index < 0 || res[i].cost_bits == ~0ull) continue;
        double c;
        std::memcpy(&c, &res[i].cost_bits, 8);
        if (c < best_cost) { best_cost = c; best = i; }
    }
    if (best < 0) return GBMW_OK;
    const BruteCell &bc = cells[best];
    int64_t idx = res[best].index;
    const int64_t ci = idx / (bc.spow * bc.S);
    int64_t digits = idx - ci * bc.spow * bc.S;
    for (int l = L - 1; l >= 0; --l) {
        const int64_t q = digits / bc.S;
        out_choice[l] = ch[best].cand[(int)(digits - q * bc.S)];
        digits = q;
    }
    const uint32_t mask = comps[bc.comp_off + ci];
    int ns = 0, start = 0;
    for (int l = 1; l <= L; ++l)
        if (l == L || ((mask >> l) & 1u)) { out_partition[ns++] = l - start; start = l; }
    out->cost = best_cost;
    out->feasible = 1;
    out->pp_degree = bc.P;
    out->n_micro = bc.n_micro;
    out->n_stages = ns;
    return GBMW_OK;
}
