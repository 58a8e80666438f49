// gbmw_seed.cu — seed partitions of many (batch, pipeline degree) cells on the device
// (SURVEY.md §8(f) #1): for every cell, the uniform seed strategy of balance.py:471-488
// (_seed_for) and its memory-balanced partition (balance.py:180-212 _init_partition:
// greedy prefix split + hill climbing on the balance degree, planner.py:250-253).
//
// One warp per cell.  The sequential parts of the reference (the greedy split, the
// in-order choice of each round's move, CPython's Neumaier sum) run on lane 0 exactly as
// written; the lanes evaluate a round's neighbour moves in parallel (each move re-costs
// the two stages it changes and recomputes the balance degree of the moved partition).
// Every value comes from the same fp64 sequences as the host restatement
// (gbmw_planner.cpp) and the reference: bit-identical partitions (-fmad=false).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/gbmw.h"
#include "costmodel.cuh"

namespace gbmw {

constexpr int kSeedWarps = 4;
constexpr int kSeedMaxStages = 128;

struct SeedStage { double t, ns, peak; };

// CPython >= 3.12 sum() of floats from the int 0 (Neumaier), gbmw_planner.cpp py_sum
struct PySum {
    double f = 0.0, c = 0.0;
    bool first = true;
    __device__ void add(double x) {
        if (first) { f = x; first = false; return; }
        const double t = f + x;
        if (fabs(f) >= fabs(x)) c += (f - t) + x;
        else c += (x - t) + f;
        f = t;
    }
    __device__ double value() const { return (c != 0.0 && isfinite(c)) ? f + c : f; }
};

// costs.py:322-352 stage_cost of layers [a, b) under the uniform strategy s (stage_cost_range)
__device__ SeedStage seed_stage(const gbmw_layer *layers, const gbmw_strategy &s, const StratDeg &d, int a, int b,
                                int stage_index, const gbmw_env &env, int64_t micro, int32_t n_micro) {
    double ts = 0.0, ns = 0.0;
    for (int l = a; l < b; ++l) {
        double t, tns;
        layer_times(layers[l], s, d, micro, env, &t, &tns);
        const double r = (l > a) ? transform_cost(layers[l].bnd_bytes_per_sample, d.data, d.tp, d.data, d.tp, micro,
                                                  env.intra_island_bw)
                                 : 0.0;
        ts = ts + (t + r);
        ns = ns + (tns + r);
    }
    if (stage_index > 1) {
        const double p2p = stage_p2p_time(layers[a].bnd_bytes_per_sample, micro, s.pp_degree, env);
        ts = ts + p2p;
        ns = ns + p2p;
    }
    double ms = 0.0, pf = 0.0, peak = 0.0;
    for (int l = a; l < b; ++l) {
        const Mem m = layer_memory(layers[l], d, micro, stage_index, n_micro, env.ms_bytes_per_param_byte);
        ms = ms + m.o_ms;
        pf = pf + m.o_f;
        peak = py_max(peak, pf + m.o_b);
    }
    SeedStage o;
    o.t = ts; o.ns = ns; o.peak = peak + ms;
    return o;
}

// balance.py:62-77 balance degree (memory objective) of S stage costs, stages b and b + 1
// replaced by n0, n1 when b >= 0; status != 0: the totals are not positive
__device__ double seed_alpha(const SeedStage *sc, int S, int b, const SeedStage &n0, const SeedStage &n1, int *status) {
    PySum tt, tm;
    double mmax = 0.0;
    for (int i = 0; i < S; ++i) {
        const SeedStage &x = (i == b) ? n0 : ((i == b + 1 && b >= 0) ? n1 : sc[i]);
        if (i == 0 || x.peak > mmax) mmax = x.peak;
        tt.add(x.t);
        tm.add(x.peak);
    }
    const double vt = tt.value(), vm = tm.value();
    if (vt <= 0 || vm <= 0) { *status = GBMW_EINVAL; return 0.0; }
    return 1.0 - mmax / vm;
}

struct SeedWarp {
    SeedStage sc[kSeedMaxStages];
    int32_t sizes[kSeedMaxStages], starts[kSeedMaxStages];
    double score[2 * kSeedMaxStages];
    int status;
};

// _init_partition(memory) of the uniform strategy s: sizes in w.sizes; w_l: per-layer scratch
__device__ void seed_init_partition(const gbmw_layer *layers, int L, const gbmw_strategy &s, const StratDeg &d, int S,
                                    const gbmw_env &env, int64_t micro, int32_t n_micro, double *w_l, SeedWarp &w,
                                    int lane) {
    for (int l = lane; l < L; l += 32) {
        const Mem m = layer_memory(layers[l], d, micro, s.pp_degree, n_micro, env.ms_bytes_per_param_byte);
        w_l[l] = m.o_f + m.o_ms;
    }
    __syncwarp();
    if (lane == 0) {                                     // balance.py:122-139 _greedy_split
        PySum tot;
        for (int l = 0; l < L; ++l) tot.add(w_l[l]);
        const double total = tot.value();
        int start = 0;
        double acc = 0.0;
        for (int st = 0; st < S - 1; ++st) {
            const int remaining = S - st - 1;
            const double target = (total * (double)(st + 1)) / (double)S;
            int end = start;
            while (end < L - remaining && (acc + w_l[end] <= target || end < start + 1)) {
                acc += w_l[end];
                ++end;
            }
            w.sizes[st] = end - start;
            start = end;
        }
        w.sizes[S - 1] = L - start;
    }
    __syncwarp();
    // balance.py:160-177 _hill_climb, at most 2 L rounds, moves in _neighbor_moves order
    double best_score = 0.0;
    for (int round = 0; round <= 2 * L; ++round) {
        if (lane == 0) for (int x = 0, a = 0; x < S; ++x) { w.starts[x] = a; a += w.sizes[x]; }
        __syncwarp();
        for (int x = lane; x < S; x += 32)
            w.sc[x] = seed_stage(layers, s, d, w.starts[x], w.starts[x] + w.sizes[x], x + 1, env, micro, n_micro);
        __syncwarp();
        if (round == 0) {
            int st = 0;
            if (lane == 0) best_score = seed_alpha(w.sc, S, -1, w.sc[0], w.sc[0], &st);
            if (lane == 0 && st) w.status = st;
            best_score = __shfl_sync(0xffffffffu, best_score, 0);
        }
        if (round == 2 * L) break;
        for (int m = lane; m < 2 * (S - 1); m += 32) {  // move m: boundary b = m / 2, direction m % 2
            const int b = m >> 1, dir = m & 1;
            double v = -INFINITY;
            if (dir == 0 ? w.sizes[b] > 1 : w.sizes[b + 1] > 1) {
                const int mid = w.starts[b] + w.sizes[b] + (dir == 0 ? -1 : 1);
                const SeedStage n0 = seed_stage(layers, s, d, w.starts[b], mid, b + 1, env, micro, n_micro);
                const SeedStage n1 =
                    seed_stage(layers, s, d, mid, w.starts[b + 1] + w.sizes[b + 1], b + 2, env, micro, n_micro);
                int st = 0;
                v = seed_alpha(w.sc, S, b, n0, n1, &st);
                if (st) { w.status = st; v = -INFINITY; }
            }
            w.score[m] = v;
        }
        __syncwarp();
        int pick = -1;
        if (lane == 0) {                                 // first move that beats the round's best by > 1e-15
            double round_score = best_score;
            for (int m = 0; m < 2 * (S - 1); ++m)
                if (w.score[m] > round_score + 1e-15) { pick = m; round_score = w.score[m]; }
            if (pick >= 0) {
                const int b = pick >> 1;
                if ((pick & 1) == 0) { w.sizes[b] -= 1; w.sizes[b + 1] += 1; }
                else { w.sizes[b] += 1; w.sizes[b + 1] -= 1; }
                best_score = round_score;
            }
        }
        pick = __shfl_sync(0xffffffffu, pick, 0);
        best_score = __shfl_sync(0xffffffffu, best_score, 0);
        __syncwarp();
        if (pick < 0) break;
    }
}

__device__ gbmw_strategy seed_make(int64_t pp, int64_t group, int paradigm) {
    gbmw_strategy s;
    memset(&s, 0, sizeof(s));
    s.pp_degree = (int32_t)pp;
    if (group > 1) {
        s.n_levels = 1;
        s.paradigm[0] = paradigm;
        s.degree[0] = (int32_t)group;
    }
    return s;
}

__global__ void __launch_bounds__(32 * kSeedWarps) k_seed_partitions(
    const gbmw_layer *layers, int32_t L, const gbmw_env *envp, int64_t n_devices, int32_t n_cells,
    const int64_t *pp_degree, const int64_t *micro_batch, const int32_t *n_micro, double budget, int32_t max_stages,
    double *scratch, int32_t *out_sizes, int32_t *out_status) {
    __shared__ SeedWarp s_w[kSeedWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cell = blockIdx.x * kSeedWarps + warp;
    if (cell >= n_cells) return;
    SeedWarp &w = s_w[warp];
    const gbmw_env env = *envp;
    const int64_t pp = pp_degree[cell], micro = micro_batch[cell];
    const int32_t nm = n_micro[cell];
    const int S = (int)pp;
    double *w_l = scratch + (int64_t)cell * L;
    if (lane == 0) w.status = 0;
    if (S > L || S > kSeedMaxStages || nm < 1) {
        if (lane == 0) out_status[cell] = S > L ? GBMW_EINVAL : (nm < 1 ? GBMW_ESTAGE : GBMW_ENOTSUP);
        return;
    }
    // balance.py:471-488: dp, then sdp and tp for groups > 1; the first whose partition fits
    const int64_t group = n_devices / pp;
    gbmw_strategy cands[3];
    int nc = 0;
    cands[nc++] = seed_make(pp, group, GBMW_DP);
    if (group > 1) {
        cands[nc++] = seed_make(pp, group, GBMW_SDP);
        cands[nc++] = seed_make(pp, group, GBMW_TP);
    }
    gbmw_strategy usable[3];
    int nu = 0;
    for (int i = 0; i < nc; ++i)
        if (micro % strat_degrees(cands[i]).data == 0) usable[nu++] = cands[i];
    if (nu == 0) usable[nu++] = cands[nc - 1];
    __syncwarp();
    for (int i = 0; i < nu; ++i) {
        const gbmw_strategy s = usable[i];
        const StratDeg d = strat_degrees(s);
        if (micro % d.data != 0) {                       // no usable seed (gbmw_planner.cpp init_partition)
            if (lane == 0) w.status = GBMW_EMICRO;
            __syncwarp();
            break;
        }
        seed_init_partition(layers, L, s, d, S, env, micro, nm, w_l, w, lane);
        if (w.status) break;
        // partition_costs of the result (the last round left w.sc for w.sizes only when
        // the climb stopped without a move; recompute to be safe)
        if (lane == 0) for (int x = 0, a = 0; x < S; ++x) { w.starts[x] = a; a += w.sizes[x]; }
        __syncwarp();
        for (int x = lane; x < S; x += 32)
            w.sc[x] = seed_stage(layers, s, d, w.starts[x], w.starts[x] + w.sizes[x], x + 1, env, micro, nm);
        __syncwarp();
        int fits = 0;
        if (lane == 0) {
            double mx = w.sc[0].peak;
            for (int x = 1; x < S; ++x) mx = py_max(mx, w.sc[x].peak);
            fits = mx <= budget;
        }
        fits = __shfl_sync(0xffffffffu, fits, 0);
        if (fits || i == nu - 1) break;                 // else the last one's partition is the answer
    }
    for (int x = lane; x < S; x += 32) out_sizes[(int64_t)cell * max_stages + x] = w.sizes[x];
    if (lane == 0) out_status[cell] = w.status;
}

int launch_seed_partitions(const gbmw_layer *layers, int32_t L, const gbmw_env *env, int64_t n_devices, int32_t n_cells,
                           const int64_t *pp, const int64_t *micro, const int32_t *n_micro, double budget,
                           int32_t max_stages, double *scratch, int32_t *out_sizes, int32_t *out_status, void *stream) {
    if (n_cells <= 0) return 0;
    const unsigned grid = (unsigned)((n_cells + kSeedWarps - 1) / kSeedWarps);
    k_seed_partitions<<<grid, 32 * kSeedWarps, 0, (cudaStream_t)stream>>>(
        layers, L, env, n_devices, n_cells, pp, micro, n_micro, budget, max_stages, scratch, out_sizes, out_status);
    return (int)cudaGetLastError();
}

}  // namespace gbmw
