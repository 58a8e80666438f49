// gbmw_brute.cu — the exhaustive planner oracle on the device.
//
// Reference: planner.brute_force_oracle (pkg/src/parapilot/planner.py:364-449).  For every
// (pipeline degree P, micro-batch count m) cell it scans every ordered partition of the L
// layers into P stages (_compositions, planner.py:354-361) and every per-layer assignment
// of the cell's usable strategies (itertools.product, planner.py:402), costs each with
// the planner's estimator and keeps the first minimum (strict `<`, planner.py:437).
//
// Device formulation: one cell per launch; a thread per (partition, choice of layers
// 0..L-2) accumulates the prefix once and then runs the last layer's S choices (the
// product's innermost digit), so each assignment costs one layer step plus the pipeline
// fold.  Stage sums, the 1F1B stash, the backward peak and pipeline_cost follow the
// reference expression by expression (no FMA: -fmad=false), and the stage-time sum is
// CPython's sum() — Neumaier-compensated since 3.12 — carried incrementally.  Every
// thread keeps the lexicographic minimum (cost bits, enumeration index); cost >= 0, so
// the bit pattern orders like the value, and the minimum index among equal costs is the
// reference's first minimum.  Blocks write partials; k_brute_reduce folds each cell's.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gbmw_internal.h"

namespace gbmw {

constexpr int kBruteThreads = 256;

__device__ __forceinline__ double bpy_max(double a, double b) { return (b > a) ? b : a; }

// Neumaier step of CPython's builtin sum (Objects/bltinmodule.c, builtin_sum_impl)
template <bool NEU>
__device__ __forceinline__ void sum_step(double &f, double &c, double x) {
    if (NEU) {
        const double t = f + x;
        if (fabs(f) >= fabs(x)) c += (f - t) + x;
        else c += (x - t) + f;
        f = t;
    } else {
        f = f + x;
    }
}
template <bool NEU>
__device__ __forceinline__ double sum_final(double f, double c) {
    return (NEU && c != 0.0 && isfinite(c)) ? f + c : f;
}

__device__ __forceinline__ bool key_less(unsigned long long c1, long long i1, unsigned long long c2, long long i2) {
    return c1 < c2 || (c1 == c2 && i1 < i2);
}

template <bool NEU>
__global__ void __launch_bounds__(kBruteThreads) k_brute_cell(const BruteCell *cells, const double *tab,
                                                              const uint32_t *comps, BrutePartial *partials,
                                                              int cell_index) {
    const BruteCell C = cells[cell_index];
    extern __shared__ __align__(16) double s_tab[];
    const int S = C.S, L = C.L;
    const int64_t LS = (int64_t)L * S;
    // stage the cell's tables (lt, lns, of, ob, oms [L][S], p2p [L], R [L][S][S]) when they fit
    const double *g = tab + C.tab_off;
    const double *T = g;
    if (C.smem_doubles > 0) {
        for (int64_t x = threadIdx.x; x < C.tab_len; x += blockDim.x) s_tab[x] = g[x];
        __syncthreads();
        T = s_tab;
    }
    const double *LT = T, *LNS = T + LS, *OF = T + 2 * LS, *OB = T + 3 * LS, *OMS = T + 4 * LS;
    const double *P2P = T + 5 * LS, *R = T + 5 * LS + L;
    const double budget = C.budget;
    const double mm1 = (double)(C.n_micro - 1);
    unsigned long long best_c = ~0ull;
    long long best_i = 0x7fffffffffffffffll;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < C.n_items; it += stride) {
        const int64_t ci = it / C.spow;                  // partition (composition) index
        const int64_t pre = it - ci * C.spow;            // digits of layers 0 .. L-2 (layer 0 most significant)
        const uint32_t mask = __ldg(comps + C.comp_off + ci);   // bit l: layer l starts a stage
        int d[kBruteMaxLayers];
        {
            int64_t v = pre;
            for (int l = L - 2; l >= 0; --l) { const int64_t q = v / S; d[l] = (int)(v - q * S); v = q; }
        }
        // running stage state (planner.py:410-431) and the folds over closed stages
        double t = 0.0, tns = 0.0, pf = 0.0, peak = 0.0, ms = 0.0;
        double steady = 0.0, sf = 0.0, sc = 0.0;
        int stage = 0, first = 0, nclosed = 0;
        double stash = 1.0;
        bool ok = true;
        auto close_stage = [&]() {
            if (stage > 1) { t = t + P2P[first]; tns = tns + P2P[first]; }
            const double e_all = peak + ms;
            if (e_all > budget) return false;
            steady = nclosed ? bpy_max(steady, tns) : tns;
            if (nclosed == 0) { sf = t; sc = 0.0; } else sum_step<NEU>(sf, sc, t);
            ++nclosed;
            return true;
        };
        auto open_stage = [&](int l) {
            ++stage;
            const int st = C.P - stage + 1;
            stash = (double)(st < C.n_micro ? st : C.n_micro);
            t = tns = pf = peak = ms = 0.0;
            first = l;
        };
        for (int l = 0; l < L - 1; ++l) {
            double r = 0.0;
            if ((mask >> l) & 1u) {
                if (l > 0 && !close_stage()) { ok = false; break; }
                open_stage(l);
            } else {
                r = R[((int64_t)l * S + d[l - 1]) * S + d[l]];
            }
            const int64_t x = (int64_t)l * S + d[l];
            t = t + (LT[x] + r);
            tns = tns + (LNS[x] + r);
            pf = pf + OF[x] * stash;
            peak = bpy_max(peak, pf + OB[x]);
            ms = ms + OMS[x];
        }
        if (!ok) continue;
        const int l = L - 1;
        const bool fresh = ((mask >> l) & 1u) != 0u;
        if (fresh) {
            if (l > 0 && !close_stage()) continue;
            open_stage(l);
        }
        const double *Rrow = (fresh || l == 0) ? nullptr : R + ((int64_t)l * S + d[l - 1]) * S;
        const double p2p = stage > 1 ? P2P[first] : 0.0;
        const int64_t base = it * S;                     // = ci * S^L + pre * S
        for (int c = 0; c < S; ++c) {
            const int64_t x = (int64_t)l * S + c;
            const double r = Rrow ? Rrow[c] : 0.0;
            double t2 = t + (LT[x] + r);
            double n2 = tns + (LNS[x] + r);
            const double pf2 = pf + OF[x] * stash;
            const double pk2 = bpy_max(peak, pf2 + OB[x]);
            const double ms2 = ms + OMS[x];
            if (stage > 1) { t2 = t2 + p2p; n2 = n2 + p2p; }
            if (pk2 + ms2 > budget) continue;
            const double st = nclosed ? bpy_max(steady, n2) : n2;
            double f = sf, cc = sc;
            if (nclosed == 0) { f = t2; cc = 0.0; } else sum_step<NEU>(f, cc, t2);
            const double cost = mm1 * st + sum_final<NEU>(f, cc);
            const unsigned long long cb = (unsigned long long)__double_as_longlong(cost);
            if (key_less(cb, base + c, best_c, best_i)) { best_c = cb; best_i = base + c; }
        }
    }
    // block minimum of (cost bits, index)
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long oc = __shfl_xor_sync(0xffffffffu, best_c, off);
        const long long oi = __shfl_xor_sync(0xffffffffu, best_i, off);
        if (key_less(oc, oi, best_c, best_i)) { best_c = oc; best_i = oi; }
    }
    __shared__ unsigned long long s_c[kBruteThreads / 32];
    __shared__ long long s_i[kBruteThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { s_c[warp] = best_c; s_i[warp] = best_i; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kBruteThreads / 32; ++w)
            if (key_less(s_c[w], s_i[w], best_c, best_i)) { best_c = s_c[w]; best_i = s_i[w]; }
        partials[C.part_off + blockIdx.x] = BrutePartial{best_c, best_i};
    }
}

// one block per cell: the minimum over the cell's block partials
__global__ void __launch_bounds__(kBruteThreads) k_brute_reduce(const BruteCell *cells, const BrutePartial *partials,
                                                                BrutePartial *out) {
    const BruteCell C = cells[blockIdx.x];
    unsigned long long best_c = ~0ull;
    long long best_i = 0x7fffffffffffffffll;
    for (int b = threadIdx.x; b < C.n_parts; b += blockDim.x) {
        const BrutePartial p = partials[C.part_off + b];
        if (key_less(p.cost_bits, p.index, best_c, best_i)) { best_c = p.cost_bits; best_i = p.index; }
    }
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long oc = __shfl_xor_sync(0xffffffffu, best_c, off);
        const long long oi = __shfl_xor_sync(0xffffffffu, best_i, off);
        if (key_less(oc, oi, best_c, best_i)) { best_c = oc; best_i = oi; }
    }
    __shared__ unsigned long long s_c[kBruteThreads / 32];
    __shared__ long long s_i[kBruteThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { s_c[warp] = best_c; s_i[warp] = best_i; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kBruteThreads / 32; ++w)
            if (key_less(s_c[w], s_i[w], best_c, best_i)) { best_c = s_c[w]; best_i = s_i[w]; }
        out[blockIdx.x] = BrutePartial{best_c, best_i};
    }
}

int brute_blocks(int64_t n_items) {
    const int64_t want = (n_items + kBruteThreads - 1) / kBruteThreads;
    const int64_t cap = 148 * 8;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

int launch_brute_cell(const BruteCell &host_cell, const BruteCell *cells, const double *tab, const uint32_t *comps,
                      BrutePartial *partials, int cell_index, int neumaier, void *stream) {
    const size_t smem = (size_t)host_cell.smem_doubles * sizeof(double);
    const int blocks = host_cell.n_parts;
    cudaStream_t st = (cudaStream_t)stream;
    if (neumaier) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_brute_cell<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_brute_cell<true><<<blocks, kBruteThreads, smem, st>>>(cells, tab, comps, partials, cell_index);
    } else {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_brute_cell<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_brute_cell<false><<<blocks, kBruteThreads, smem, st>>>(cells, tab, comps, partials, cell_index);
    }
    return (int)cudaGetLastError();
}

int launch_brute_reduce(const BruteCell *cells, int n_cells, const BrutePartial *partials, BrutePartial *out,
                        void *stream) {
    if (n_cells <= 0) return 0;
    k_brute_reduce<<<n_cells, kBruteThreads, 0, (cudaStream_t)stream>>>(cells, partials, out);
    return (int)cudaGetLastError();
}

}  // namespace gbmw
