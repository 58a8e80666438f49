// gbmw_kernels.cu — sm_100a kernels of the Galvatron-BMW stage search.
//
//   K1 k_cost_cells / k_cost_r : batched cost-model tables      (dpsearch.py:127-163)
//   K2 k_dp_step<KT>           : one min-plus layer step, all problems of the chunk
//                                 that have that many units      (dpsearch.py:245-282)
//   K3 k_sweep                 : E_fwd sweep + backward-peak validity + per-tile argmin
//                                                                (dpsearch.py:174-208)
//   K4 k_finalize              : cross-tile argmin, backtrack, plan expansion,
//                                 stage_cost of the plan         (dpsearch.py:210-227,
//                                                                 costs.py:289-352)
// All fp64 arithmetic follows the reference's evaluation order; the file is built
// with -fmad=false so no a*b+c is contracted (SURVEY.md §8 arithmetic contract).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "costmodel.cuh"
#include "gbmw_internal.h"

namespace gbmw {

#define GBMW_INF __longlong_as_double(0x7ff0000000000000LL)

// largest q in [0, n) with prefix[q] <= x; prefix is non-decreasing and prefix[0] = 0
__device__ __forceinline__ int find_slot(const int64_t *prefix, int n, int64_t x) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// The same search started from a coarse map: the slot holds position x is between the slots
// holding coarse entries x >> shift and (x >> shift) + 1, usually the same one.
__device__ __forceinline__ int find_slot_coarse(const int64_t *prefix, int n, int64_t x, const int32_t *coarse,
                                                int64_t n_coarse, int shift) {
    const int64_t b = x >> shift;
    int lo = __ldg(coarse + b), hi = b + 1 < n_coarse ? __ldg(coarse + b + 1) : n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Python's `int <= float` is exact; e_fwd = e * gran is an int.
__device__ __forceinline__ bool int_le_double(int64_t x, double y) {
    if (y != y) return false;
    if (y >= 9.2233720368547758e18) return true;
    if (y < -9.2233720368547758e18) return false;
    return x <= (int64_t)floor(y);
}

// ---------------------------------------------------------------- K1: cost tables
__global__ void k_cost_cells(ChunkArgs a, int64_t n_cells) {
    const int64_t idx0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = idx0 < n_cells;
    if (__all_sync(0xffffffffu, !valid)) return;         // whole warps only: the b_up max below is warp-wide
    const int64_t idx = valid ? idx0 : n_cells - 1;       // past the end: a duplicate of the last cell
    const int q = find_slot_coarse(a.cell_prefix, a.n_probs, idx, a.cell_coarse, a.n_cell_coarse, kCoarseShift);
    const DevProblem &p = a.probs[q];
    const int64_t local = idx - a.cell_prefix[q];
    const int u = (int)(local / p.S);
    const int i = (int)(local % p.S);
    const gbmw_layer L = a.layers[a.unit_first[p.unit_off + u]];
    const gbmw_strategy s = a.strats[a.cand_strat[p.cand_off + i]];
    const gbmw_env env = a.envs[p.env_index];
    const StratDeg d = strat_degrees(s);
    double t, t_ns;
    layer_times(L, s, d, p.micro, env, &t, &t_ns);
    const Mem m = layer_memory(L, d, p.micro, p.stage_index, p.n_micro, env.ms_bytes_per_param_byte);
    const int cnt = a.unit_count[p.unit_off + u];
    Cell c;
    c.c = t * (double)cnt;                       // dpsearch.py:141
    c.ef = (m.o_f + m.o_ms) * (double)cnt;       // dpsearch.py:142
    const double wq = ceil(c.ef / (double)p.gran);   // dpsearch.py:144
    int64_t w = (wq > (double)p.n_b) ? p.n_b + 1 : (int64_t)wq;
    if (w < 0) w = 0;                            // dpsearch.py:145
    c.w = (int32_t)w;
    c.k = a.cand_cls[p.cand_off + i];
    if (valid) {
        a.cells[p.cell_off + local] = c;
        CellMem cm;
        cm.o_f = m.o_f; cm.o_b = m.o_b; cm.o_ms = m.o_ms;
        a.cmem[p.cell_off + local] = cm;
    }
    // b_up = max O_b over (unit, strategy)  (dpsearch.py:162); O_b >= 0 so the bit
    // pattern orders like the value.  Consecutive lanes hold consecutive cells, so a
    // problem's lanes are a contiguous run: a segmented max, then one atomic per run.
    const int lane = threadIdx.x & 31;
    unsigned long long v = (unsigned long long)__double_as_longlong(m.o_b);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long ov = __shfl_down_sync(0xffffffffu, v, off);
        const int oq = __shfl_down_sync(0xffffffffu, q, off);
        if (lane + off < 32 && oq == q && ov > v) v = ov;
    }
    const int pq = __shfl_up_sync(0xffffffffu, q, 1);
    if (valid && (lane == 0 || pq != q)) atomicMax(&a.bup[q], v);
}

__global__ void k_cost_r(ChunkArgs a, int64_t n_r) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_r) return;
    const int q = find_slot_coarse(a.r_prefix, a.n_probs, idx, a.r_coarse, a.n_r_coarse, kCoarseShift);
    const DevProblem &p = a.probs[q];
    const int64_t local = idx - a.r_prefix[q];
    const int KK = p.K * p.K;
    const int u = (int)(local / KK);
    const int rem = (int)(local % KK);
    const int ka = rem / p.K, kb = rem % p.K;
    const gbmw_layer L = a.layers[a.unit_first[p.unit_off + u]];
    const gbmw_env env = a.envs[p.env_index];
    a.rcls[p.r_off + local] = transform_cost(
        L.bnd_bytes_per_sample, a.class_d[p.class_off + ka], a.class_t[p.class_off + ka],
        a.class_d[p.class_off + kb], a.class_t[p.class_off + kb], p.micro, env.intra_island_bw);
}

// Source-side pruning by dominance (exact): strategies j < i with the same weight and
// class at unit u read the same row and column of B_u, so in every row
// T_j = v.t + c_j and F_j = v.f + ef_j against T_i = v.t + c_i and F_i = v.f + ef_i.
// fp addition is monotone, so c_j <= c_i and ef_j <= ef_i give T_j <= T_i, F_j <= F_i
// (and the same for every target after + R[cls, k]); with ties resolved to the first
// index (T1), i can never be an argmin.  This covers the identical cells (the exact
// duplicates) and, e.g., 38 -> 26 sources per GPT-3-96 P = 1 unit.  K2 relaxes only
// the surviving sources; the sweep's rank-0 candidate (K3a, K3r) is never a dominated
// one either, and K3b walks every strategy.  A warp per (problem, unit).
//
// The same pass derives the live row range of every class table B_u: with
// wmin_v = min_i weight[v][i], T_u is +inf below m_u = sum_{v<=u} wmin_v, so
// B_u[e'] (built from T_{u-1}[e']) is +inf for e' < L_u = m_{u-1}; and B_u is only
// ever read at rows e - w_uj <= n_b - wmin_u = H_u.  Rows outside [L_u, H_u] are
// neither computed nor read (readers treat them as +inf, which they are).
// A warp per (problem, unit) over the whole chunk, so a deep problem's units run on many SMs
// at once; the unit's wmin is parked in unit_hi until k_unit_ranges turns it into [L_u, H_u].
__global__ void k_dedupe(ChunkArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t gu = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gu >= a.n_units) return;
    const int64_t cb = gu >> kUnitCoarseShift;           // problem holding global unit gu
    int qa = __ldg(a.unit_coarse + cb), qb = cb + 1 < a.n_unit_coarse ? __ldg(a.unit_coarse + cb + 1) : a.n_probs - 1;
    while (qa < qb) {
        const int mid = (qa + qb + 1) >> 1;
        if (a.probs[mid].ustate_off <= gu) qa = mid; else qb = mid - 1;
    }
    const DevProblem &p = a.probs[qa];
    const int u = (int)(gu - p.ustate_off);
    const Cell *cells = a.cells + p.cell_off + (int64_t)u * p.S;
    int32_t *uniq = a.uniq + p.cell_off + (int64_t)u * p.S;
    int count = 0;
    int wmin = 0x7fffffff;
    for (int base = 0; base < p.S; base += 32) {
        const int i = base + lane;
        bool keep = false;
        if (i < p.S) {
            const Cell ci = cells[i];
            wmin = min(wmin, ci.w);
            keep = true;
            for (int j = 0; j < i; ++j) {
                const Cell cj = cells[j];
                if (cj.w == ci.w && cj.k == ci.k && cj.c <= ci.c && cj.ef <= ci.ef) { keep = false; break; }
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int slot = count + __popc(m & ((1u << lane) - 1u));
            uniq[slot] = i;
            a.ucell[p.cell_off + (int64_t)u * p.S + slot] = cells[i];
        }
        count += __popc(m);
    }
    for (int off = 16; off > 0; off >>= 1) wmin = min(wmin, __shfl_xor_sync(0xffffffffu, wmin, off));
    if (lane == 0) {
        a.nuniq[p.ustate_off + u] = count;
        a.unit_hi[p.ustate_off + u] = wmin;
    }
}

// Live row ranges of every unit, a thread per problem (reads the wmins k_dedupe parked).
// A warp per problem: L_u is the exclusive prefix sum of the units' least weights (capped at
// n_b + 1), so 32 units at a time go through one load and a warp scan instead of a chain of
// dependent loads and stores over the units.
__global__ void k_unit_ranges(ChunkArgs a) {
    const int q = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= a.n_probs) return;                          // warp-uniform
    const DevProblem &p = a.probs[q];
    const int64_t top = p.n_b + 1;
    int64_t carry = 0;                                   // sum of the least weights of the units before
    unsigned long long live = 0;
    for (int u0 = 0; u0 < p.U; u0 += 32) {
        const int u = u0 + lane;
        const int wmin = u < p.U ? a.unit_hi[p.ustate_off + u] : 0;
        int64_t incl = wmin;                             // inclusive scan over the lanes
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        const int64_t acc = carry + incl - wmin;         // exclusive: units before u
        if (u < p.U) {
            const int64_t lo = acc < top ? acc : top, hi = p.n_b - wmin;
            a.unit_lo[p.ustate_off + u] = (int32_t)lo;                      // L_u = m_{u-1}
            a.unit_hi[p.ustate_off + u] = (int32_t)hi;                      // H_u
            if (u >= 1 && hi >= lo) live += (unsigned long long)(hi - lo + 1);
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) live += __shfl_xor_sync(0xffffffffu, live, off);
    // live class cells written by K2 (algorithmic-bytes accounting)
    if (lane == 0 && !(p.flags & GBMW_APPROX)) atomicAdd(a.live_cells, live * (unsigned long long)p.K);
}

// K2 (the min-plus layer step) lives in gbmw_step.cu.

// ---------------------------------------------------------------- shared helpers
// reference table of the last unit at row e, strategy j
struct RowCtx {
    const int32_t *w; const int32_t *k; const double *c; const double *ef;
    const TFCell *bin;
    const int2 *rm;      // row map of B_{U-1} (B is stored only at its stored rows)
    const int2 *rms;     // the same map staged in shared memory, or nullptr
    int32_t K;           // classes: B is row-major, K (t, f) cells per row
    int64_t n_e;
    int64_t lo;        // rows of B_{U-1} below L_{U-1} are +inf (never written)
    bool init;
};

__device__ __forceinline__ void row_value(const RowCtx &r, int64_t e, int j, double &T, double &F) {
    const int w = r.w[j];
    if (e - w < r.lo) { T = GBMW_INF; F = GBMW_INF; return; }
    if (r.init) { T = r.c[j]; F = r.ef[j]; return; }
    const int x = (int)(e - w);
    const int row = r.rms ? stored_row(r.rms[x >> 5], x) : stored_row(r.rm, x);
    const int64_t src = (int64_t)row * r.K + r.k[j];
    const double2 v = __ldg(reinterpret_cast<const double2 *>(r.bin + src));
    T = v.x + r.c[j];
    F = v.y + r.ef[j];
}

// Walk the argmin pointers back from (last unit, e, j) (dpsearch.py:292-301).
__device__ __forceinline__ void backtrack(const ChunkArgs &a, const DevProblem &p, int64_t e, int j,
                                          uint16_t *path) {
    const int U = p.U, S = p.S, K = p.K;
    const int64_t n_e = p.n_b + 1;
    const Cell *cells = a.cells + p.cell_off;
    const uint16_t *par = a.par + p.par_off;
    const int64_t ng = rmap_groups(n_e);
    path[U - 1] = (uint16_t)j;
    for (int u = U - 1; u >= 1; --u) {
        const Cell c = cells[(int64_t)u * S + j];
        e -= c.w;
        const int er = stored_row(a.rmap + p.rmap_off + (int64_t)(u - 1) * ng, (int)e);
        j = par[((int64_t)(u - 1) * n_e + er) * K + c.k];
        path[u - 1] = (uint16_t)j;
    }
}

// The same walk by a whole warp (K4): lane s holds strategy s's (weight, class) of the next
// units, fetched ahead, and the row-map word at the row each strategy would step to, so the
// argmin load of a unit goes out with the next unit's row-map loads beside it: the chain per
// unit is one global load instead of three (cell, row map, argmin).  S <= 64.
__device__ __forceinline__ void backtrack_warp(const ChunkArgs &a, const DevProblem &p, int64_t e, int j,
                                               uint16_t *path, int lane) {
    const int U = p.U, S = p.S, K = p.K;
    const int64_t n_e = p.n_b + 1;
    const Cell *cells = a.cells + p.cell_off;
    const uint16_t *par = a.par + p.par_off;
    const int2 *rmb = a.rmap + p.rmap_off;
    const int64_t ng = rmap_groups(n_e);
    constexpr unsigned full = 0xffffffffu;
    int wc[2], kc[2], wn[2], kn[2];                      // units u and u - 1, strategies lane, lane + 32
    int2 m[2];                                           // row map of unit u - 1 at e - w_u(s)
    auto cell_wk = [&](int u, int b, int *w, int *k) {
        const int s = lane + 32 * b;
        if (u >= 1 && s < S) { const Cell c = cells[(int64_t)u * S + s]; w[b] = c.w; k[b] = c.k; }
        else { w[b] = 0; k[b] = 0; }
    };
    auto rm_at = [&](int u, int64_t e_u, int b, const int *w) {
        const int s = lane + 32 * b;
        const int64_t x = e_u - w[b];
        return (u >= 1 && s < S && x >= 0) ? __ldg(rmb + (int64_t)(u - 1) * ng + (x >> 5)) : make_int2(0, 0);
    };
    if (lane == 0) path[U - 1] = (uint16_t)j;
#pragma unroll
    for (int b = 0; b < 2; ++b) { cell_wk(U - 1, b, wc, kc); cell_wk(U - 2, b, wn, kn); }
#pragma unroll
    for (int b = 0; b < 2; ++b) m[b] = rm_at(U - 1, e, b, wc);
    for (int u = U - 1; u >= 1; --u) {
        int wnn[2], knn[2];                              // unit u - 2, fetched two units ahead
#pragma unroll
        for (int b = 0; b < 2; ++b) cell_wk(u - 2, b, wnn, knn);
        const int src = j & 31, hb = j >> 5;
        const int w = __shfl_sync(full, hb ? wc[1] : wc[0], src);
        const int k = __shfl_sync(full, hb ? kc[1] : kc[0], src);
        const int mx = __shfl_sync(full, hb ? m[1].x : m[0].x, src);
        const int my = __shfl_sync(full, hb ? m[1].y : m[0].y, src);
        e -= w;
        const int er = stored_row(make_int2(mx, my), (int)e);
        const int jn = par[((int64_t)(u - 1) * n_e + er) * K + k];
#pragma unroll
        for (int b = 0; b < 2; ++b) m[b] = rm_at(u - 1, e, b, wn);
        j = jn;
        if (lane == 0) path[u - 1] = (uint16_t)j;
#pragma unroll
        for (int b = 0; b < 2; ++b) { wc[b] = wn[b]; kc[b] = kn[b]; wn[b] = wnn[b]; kn[b] = knn[b]; }
    }
    __syncwarp();
}

// Same walk with (weight, class) of every (unit, strategy) staged in shared memory, packed
// as weight << 4 | class (weight <= n_b + 1 < 2^27): the chain per unit is then one global
// load (the argmin) after the row-map entry.  rms: row map of the last unit in shared
// memory, or nullptr.
__device__ __forceinline__ void backtrack_wk(const ChunkArgs &a, const DevProblem &p, int64_t e, int j,
                                             uint16_t *path, const uint32_t *wk, const int2 *rms) {
    const int U = p.U, S = p.S, K = p.K;
    const int64_t n_e = p.n_b + 1;
    const uint16_t *par = a.par + p.par_off;
    const int64_t ng = rmap_groups(n_e);
    path[U - 1] = (uint16_t)j;
    for (int u = U - 1; u >= 1; --u) {
        const uint32_t c = wk[u * S + j];
        e -= (int64_t)(c >> 4);
        const int x = (int)e;
        const int er = (u == U - 1 && rms) ? stored_row(rms[x >> 5], x)
                                           : stored_row(a.rmap + p.rmap_off + (int64_t)(u - 1) * ng, x);
        j = par[((int64_t)(u - 1) * n_e + er) * K + (int)(c & 15u)];
        path[u - 1] = (uint16_t)j;
    }
}

#ifndef GBMW_EALL_B_K3
#define GBMW_EALL_B_K3 1                     // units in flight in K3b's E_all folds (2: 64-register cap spills, measured equal)
#endif
// E_all of the expanded plan in layer order (costs.py:307-318).  The units' memory terms
// are fetched B at a time (independent loads in flight together), then folded in order.
template <int B = 4>
__device__ __forceinline__ double plan_e_all(const ChunkArgs &a, const DevProblem &p, const uint16_t *path) {
    double total_ms = 0.0, prefix_f = 0.0, peak = 0.0;
    const CellMem *cm = a.cmem + p.cell_off;
    const int32_t *uc = a.unit_count + p.unit_off;
    if constexpr (B == 1) {
        for (int u = 0; u < p.U; ++u) {
            const CellMem m = cm[(int64_t)u * p.S + path[u]];
            const int cnt = uc[u];
            for (int r = 0; r < cnt; ++r) {
                total_ms = total_ms + m.o_ms;
                prefix_f = prefix_f + m.o_f;
                peak = py_max(peak, prefix_f + m.o_b);
            }
        }
        return peak + total_ms;
    }
    for (int u0 = 0; u0 < p.U; u0 += B) {
        CellMem m[B];
        int cnt[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int u = u0 + b;
            cnt[b] = 0;
            if (u < p.U) { m[b] = cm[(int64_t)u * p.S + path[u]]; cnt[b] = uc[u]; }
        }
#pragma unroll
        for (int b = 0; b < B; ++b)
            for (int r = 0; r < cnt[b]; ++r) {
                total_ms = total_ms + m[b].o_ms;
                prefix_f = prefix_f + m[b].o_f;
                peak = py_max(peak, prefix_f + m[b].o_b);
            }
    }
    return peak + total_ms;
}

__device__ __forceinline__ bool lex_less(double t1, double f1, int j1, double t2, double f2, int j2) {
    if (t1 != t2) return t1 < t2;
    if (f1 != f2) return f1 < f2;
    return j1 < j2;
}

// candidate order across buckets: smaller t, ties -> larger e (dpsearch.py:203-207)
__device__ __forceinline__ bool cand_better(double t1, int64_t e1, double t2, int64_t e2) {
    return (t1 < t2) || (t1 == t2 && e1 > e2);
}

// block-wide best (t, larger e) of one candidate per thread; result valid in all threads
__device__ __forceinline__ SweepPartial block_best(double t, int64_t e, int j, double *red_t, long long *red_e,
                                                   int *red_j) {
    for (int off = 16; off > 0; off >>= 1) {
        const double ot = __shfl_down_sync(0xffffffffu, t, off);
        const long long oe = __shfl_down_sync(0xffffffffu, (long long)e, off);
        const int oj = __shfl_down_sync(0xffffffffu, j, off);
        if (cand_better(ot, oe, t, e)) { t = ot; e = oe; j = oj; }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();                    // red_* may still be read by a previous call
    if (lane == 0) { red_t[wid] = t; red_e[wid] = e; red_j[wid] = j; }
    __syncthreads();
    double bt = red_t[0];
    long long be = red_e[0];
    int bj = red_j[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (cand_better(red_t[w], red_e[w], bt, be)) { bt = red_t[w]; be = red_e[w]; bj = red_j[w]; }
    SweepPartial sp;
    sp.t = bt; sp.e = be; sp.j = bj; sp.pad_ = 0;
    return sp;
}

// ---------------------------------------------------------------- K3: E_fwd sweep
// The sweep (dpsearch.py:194-208) keeps the best f(e) over e = 1..n_b, f(e) being the
// first candidate of row e in (T, F, j) order that fits; ties on t go to the larger e.
//  - safe zone (e * gran <= budget - b_up): everything fits and f(e) is the rank-0
//    candidate.  Every T[., j] is non-increasing in e (min-plus of non-increasing
//    columns), so the rank-0 time is too: the best safe bucket is the largest one, e_s.
//    K3a evaluates that row only (one warp per problem).
//  - unsafe zone: K3b walks the candidates of every unsafe row with the backward-peak
//    check, pruned by a per-problem bound (persistent CTAs over a compact tile list).
//  - K3r evaluates every row of the problems that want the frontier (rank-0 time per
//    row) or use the collapsed DP (one candidate per row, not monotone in e).

// largest safe bucket e_s in [0, n_b] (0: none); Python's `int <= float` is exact
__device__ __forceinline__ int64_t safe_bucket(const DevProblem &p, double safe_limit) {
    double x = floor(safe_limit / (double)p.gran);
    if (!(x >= 0.0)) x = 0.0;
    if (x > (double)p.n_b) x = (double)p.n_b;
    int64_t e_s = (int64_t)x;
    while (e_s >= 1 && !int_le_double(e_s * p.gran, safe_limit)) --e_s;
    while (e_s + 1 <= p.n_b && int_le_double((e_s + 1) * p.gran, safe_limit)) ++e_s;
    return e_s;
}

// safe_limit = budget - b_up (dpsearch.py:162-164)
__device__ __forceinline__ double safe_limit_of(const ChunkArgs &a, const DevProblem &p, int q) {
    return p.budget - __longlong_as_double((long long)a.bup[q]);
}

// first bucket with a finite row of the last unit: m_{U-1} = L_{U-1} + wmin_{U-1} (k_dedupe)
__device__ __forceinline__ int64_t first_finite_row(const ChunkArgs &a, const DevProblem &p) {
    const int last = p.U - 1;
    return (int64_t)a.unit_lo[p.ustate_off + last] + (p.n_b - a.unit_hi[p.ustate_off + last]);
}

__device__ __forceinline__ void lex_min_warp(double &t, double &f, int &j) {
    for (int off = 16; off > 0; off >>= 1) {
        const double ot = __shfl_xor_sync(0xffffffffu, t, off);
        const double of = __shfl_xor_sync(0xffffffffu, f, off);
        const int oj = __shfl_xor_sync(0xffffffffu, j, off);
        if (oj >= 0 && (j < 0 || lex_less(ot, of, oj, t, f, j))) { t = ot; f = of; j = oj; }
    }
}

// Running best (t, e) of a problem's sweep as one 16-byte word {bits of t, e + 1}, updated
// with 128-bit CAS (t >= 0, so the bits of t order like t).  Order: smaller t, ties ->
// larger e (dpsearch.py:203-207).  Updates are rare (a fitting candidate) and monotone:
// t never increases and e only grows while t stays.  Readers use plain loads, t / e / t:
// if both reads of t agree, t was constant in between and e belongs to it; otherwise
// only t (the later read) is used and the tie rule is not applied (conservative).
__device__ __forceinline__ void cas128(unsigned long long *addr, unsigned long long c0, unsigned long long c1,
                                       unsigned long long n0, unsigned long long n1, unsigned long long &o0,
                                       unsigned long long &o1) {
    asm volatile("{\n\t.reg .b128 d, c, n;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 n, {%4, %5};\n\t"
                 "atom.relaxed.gpu.global.cas.b128 d, [%6], c, n;\n\tmov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(o0), "=l"(o1)
                 : "l"(c0), "l"(c1), "l"(n0), "l"(n1), "l"(addr)
                 : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// (t, e); e = INT64_MIN when the tie rule must not be used
__device__ __forceinline__ void bound_read(const unsigned long long *b, double &t, int64_t &e) {
    const unsigned long long t0 = ld_acquire(b);
    const unsigned long long e1 = ld_acquire(b + 1);
    const unsigned long long t1 = ld_relaxed(b);
    t = __longlong_as_double((long long)t1);
    e = (t0 == t1) ? (int64_t)e1 - 1 : INT64_MIN;
}

__device__ __forceinline__ void bound_offer(unsigned long long *b, double t, int64_t e) {
    unsigned long long c0 = ld_relaxed(b), c1 = ld_relaxed(b + 1);
    const unsigned long long n0 = (unsigned long long)__double_as_longlong(t), n1 = (unsigned long long)(e + 1);
    while (cand_better(t, e, __longlong_as_double((long long)c0), (int64_t)c1 - 1)) {
        unsigned long long o0, o1;
        cas128(b, c0, c1, n0, n1, o0, o1);
        if (o0 == c0 && o1 == c1) break;
        c0 = o0; c1 = o1;
    }
}

// K3a: per problem, the rank-0 candidate at e_s, the pruning bound it seeds, and the
// first tile of the unsafe rows [max(e_s + 1, first finite row), n_b].
__global__ void k_sweep_safe(ChunkArgs a) {
    const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= a.n_probs) return;
    const DevProblem &p = a.probs[q];
    double t0 = GBMW_INF, f0 = GBMW_INF;
    int j0 = -1;
    int64_t e_s = 0;
    int32_t first_tile = 0;                              // approx_prev: K3r writes every tile
    if (!(p.flags & GBMW_APPROX)) {
        const int last = p.U - 1;
        const int64_t first_finite = first_finite_row(a, p);
        e_s = safe_bucket(p, safe_limit_of(a, p, q));
        if (e_s >= 1 && e_s >= first_finite) {
            const Cell *lc = a.cells + p.cell_off + (int64_t)last * p.S;
            const int32_t *ul = a.uniq + p.cell_off + (int64_t)last * p.S;
            const int S = a.nuniq[p.ustate_off + last];
            const int64_t n_e = p.n_b + 1;
            const int64_t lo = (last == 0) ? 0 : a.unit_lo[p.ustate_off + last];
            const TFCell *bin = a.TF[last & 1] + p.b_off;
            const int2 *rm = a.rmap + p.rmap_off + (int64_t)(last >= 1 ? last - 1 : 0) * rmap_groups(n_e);
            for (int n = lane; n < S; n += 32) {
                const int j = ul[n];
                const Cell c = lc[j];
                if (e_s - c.w < lo) continue;
                double T, F;
                if (last == 0) {
                    T = c.c; F = c.ef;
                } else {
                    const double2 v = __ldg(reinterpret_cast<const double2 *>(
                        bin + (int64_t)stored_row(rm, (int)(e_s - c.w)) * p.K + c.k));
                    T = v.x + c.c;
                    F = v.y + c.ef;
                }
                if (T < GBMW_INF && (j0 < 0 || lex_less(T, F, j, t0, f0, j0))) { t0 = T; f0 = F; j0 = j; }
            }
            lex_min_warp(t0, f0, j0);
        }
        const int64_t e_lo = max(e_s + 1, first_finite);
        first_tile = (e_lo <= p.n_b) ? (int32_t)((e_lo - 1) / kSweepThreads) : p.n_sweep_tiles;
    }
    if (lane == 0) {
        SweepPartial sp;
        sp.t = t0; sp.e = (j0 >= 0) ? e_s : -1; sp.j = (j0 >= 0) ? j0 : 0; sp.pad_ = 0;
        a.best[q] = sp;
        a.bound[2 * q] = (unsigned long long)__double_as_longlong(t0);
        a.bound[2 * q + 1] = (unsigned long long)((j0 >= 0 ? e_s : -1) + 1);
        a.ufirst[q] = first_tile;
        a.upruned[q] = 0;
    }
}

// K3b work list (one CTA of 1024): items are (rank, problem), rank r = r-th unsafe tile
// of the problem from the top, ordered rank-major so that every problem's highest (lowest
// time) tiles run first and tighten its bound before its lower tiles start.  Problems are
// counting-sorted by unsafe tile count n_q, descending: the problems with n_q > r are
// then the first cnt_gt[r] of usorted, and uprefix[r] = sum_{r' < r} cnt_gt[r'].
__device__ __forceinline__ int unsafe_tiles(const ChunkArgs &a, int q) {
    const DevProblem &p = a.probs[q];
    return (p.flags & GBMW_APPROX) ? 0 : p.n_sweep_tiles - a.ufirst[q];
}

__global__ void __launch_bounds__(1024) k_sweep_scan(ChunkArgs a) {
    __shared__ int s_cnt[kMaxSweepRanks + 1];       // histogram of n_q, then slots
    __shared__ long long s_part[1024];
    constexpr int kPer = (kMaxSweepRanks + 1023) / 1024;
    const int n = a.n_probs, tid = threadIdx.x;
    for (int m = tid; m <= kMaxSweepRanks; m += 1024) s_cnt[m] = 0;
    __syncthreads();
    for (int q = tid; q < n; q += 1024) {
        const int c = unsafe_tiles(a, q);
        if (c > 0) atomicAdd(&s_cnt[c], 1);
    }
    __syncthreads();
    // cnt_gt[r] = #{q : n_q > r} = sum of hist over (r, kMaxSweepRanks]: suffix scan, kPer bins per thread
    int loc[kPer];
    long long sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int m = tid * kPer + i + 1;                // hist bin m contributes to cnt_gt[r] for r < m
        loc[i] = (m <= kMaxSweepRanks) ? s_cnt[m] : 0;
        sum += loc[i];
    }
    s_part[tid] = sum;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {          // inclusive suffix scan of thread sums
        const long long v = (tid + off < 1024) ? s_part[tid + off] : 0;
        __syncthreads();
        s_part[tid] += v;
        __syncthreads();
    }
    int gt[kPer];
    {
        long long run = (tid + 1 < 1024) ? s_part[tid + 1] : 0;   // bins above this thread's range
        for (int i = kPer - 1; i >= 0; --i) {
            run += loc[i];
            gt[i] = (int)run;                             // cnt_gt[tid * kPer + i]
        }
    }
    // rank prefix: uprefix[r] = sum_{r' < r} cnt_gt[r'] (exclusive scan over r)
    long long rs = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) rs += gt[i];
    __syncthreads();
    s_part[tid] = rs;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const long long v = (tid >= off) ? s_part[tid - off] : 0;
        __syncthreads();
        s_part[tid] += v;
        __syncthreads();
    }
    long long run = s_part[tid] - rs;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int r = tid * kPer + i;
        if (r <= kMaxSweepRanks) a.uprefix[r] = run;
        run += gt[i];
    }
    if (tid == 1023) a.uprefix[kMaxSweepRanks] = run;
    // slots of the descending counting sort: bin m starts at cnt_gt[m] (problems with n_q > m)
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int r = tid * kPer + i;
        if (r <= kMaxSweepRanks) s_cnt[r] = gt[i];
    }
    __syncthreads();
    for (int q = tid; q < n; q += 1024) {
        const int c = unsafe_tiles(a, q);
        if (c > 0) a.usorted[atomicAdd(&s_cnt[c], 1)] = q;
    }
    if (tid == 0) *a.ucounter = 0ull;
}

// K3b, unsafe zone (e_fwd > budget - b_up): every candidate needs the backward-peak check
// (a walk of U argmin pointers + the forward E_all fold).  One thread per unsafe bucket
// walks its candidates in (T, F, j) order and stops at the first that fits (f(e),
// dpsearch.py:202-208) or as soon as its candidate cannot beat the problem's running best
// (t*, e*) of any bucket (safe or unsafe): T > t*, or T == t* at a bucket below e* (ties
// keep the larger e).  Persistent CTAs take (problem, tile) items from the
// compact list K3a/K3scan built, highest buckets of a problem first (they carry the
// lowest times, so the bound tightens soonest).
constexpr int kSweepBatch = 4;
__global__ void __launch_bounds__(kSweepThreads) k_sweep_unsafe(ChunkArgs a) {
    __shared__ int32_t sW[kMaxStrats];
    __shared__ int32_t sK[kMaxStrats];
    __shared__ double sC[kMaxStrats];
    __shared__ double sE[kMaxStrats];
    __shared__ double red_t[kSweepThreads / 32];
    __shared__ long long red_e[kSweepThreads / 32];
    __shared__ int red_j[kSweepThreads / 32];
    __shared__ double sOB[kMaxStrats];                  // O_b of one layer of the last unit
    __shared__ uint32_t sWK[kSweepWK];                  // weight << 4 | class per (unit, strategy)
    __shared__ int2 sRM[kSweepRmap];                    // row map of B_{U-1}, when it fits
    __shared__ int s_skip, s_q, s_tile;
    // items are taken kSweepBatch at a time by warp 0 (one counter atomic, the slot searches
    // in parallel); items already pruned are retired right there, the rest queue in shared
    // memory and the CTA works through them one by one (a small batch keeps the rank-major
    // order, so the top tiles still tighten the bounds before the tiles below them run)
    __shared__ int s_iq[32], s_it[32];
    __shared__ int s_nq, s_qi, s_done;
    __shared__ long long s_last;                        // the counter value of this CTA's last take
    const long long total = a.uprefix[kMaxSweepRanks];
    const int lane = threadIdx.x & 31;
    int q_prev = -1;
    unsigned long long n_rows = 0, n_cands = 0, n_checks = 0;
    if (threadIdx.x == 0) { s_nq = 0; s_qi = 0; s_done = 0; s_last = 0; }
    while (true) {
        __syncthreads();
        if (threadIdx.x < 32) {
            while (s_qi >= s_nq && !s_done) {               // warp-uniform: shared state after __syncwarp
                // batches while many items remain; single items in the tail (the deep
                // problems' low tiles), where every CTA should take one
                const int B = (total - s_last > (long long)kSweepBatch * 4 * gridDim.x) ? kSweepBatch : 1;
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(a.ucounter, (unsigned long long)B);
                base = __shfl_sync(0xffffffffu, base, 0);
                if (lane == 0) s_last = (long long)base;
                if ((long long)base >= total) {
                    if (lane == 0) s_done = 1;
                    __syncwarp();
                    break;
                }
                const long long g = (long long)base + lane;
                int q = 0, tile = 0;
                bool keep = false;
                if (lane < B && g < total) {
                    const int rank = find_slot(a.uprefix, kMaxSweepRanks, g);
                    q = a.usorted[g - a.uprefix[rank]];
                    tile = a.probs[q].n_sweep_tiles - 1 - rank;
                    // a higher tile of q was pruned: this one cannot win either (t0 is monotone)
                    const bool skip = tile < *(volatile int32_t *)(a.upruned + q);
                    if (a.k2_hist) {                                  // debug: items, flag-skipped items
                        atomicAdd(a.k2_hist + 56, 1ull);
                        if (skip) atomicAdd(a.k2_hist + 57, 1ull);
                    }
                    if (skip) {
                        SweepPartial none;
                        none.t = GBMW_INF; none.e = -1; none.j = 0; none.pad_ = 0;
                        a.partials[a.probs[q].tile_off + tile] = none;
                    } else {
                        keep = true;
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const int at = __popc(m & ((1u << lane) - 1u));
                    s_iq[at] = q; s_it[at] = tile;
                }
                if (lane == 0) { s_nq = __popc(m); s_qi = 0; }
                __syncwarp();
            }
            if (lane == 0 && s_qi < s_nq) {
                const int k = s_qi++;
                s_q = s_iq[k]; s_tile = s_it[k];
                // re-check: the flag may have been set since the item was taken
                s_skip = s_tile < *(volatile int32_t *)(a.upruned + s_q) ? 1 : 0;
                if (s_skip) {
                    SweepPartial none;
                    none.t = GBMW_INF; none.e = -1; none.j = 0; none.pad_ = 0;
                    a.partials[a.probs[s_q].tile_off + s_tile] = none;
                }
            } else if (lane == 0) {
                s_skip = -1;                                  // drained and no items left
            }
        }
        __syncthreads();
        if (s_skip < 0) break;
        if (s_skip) continue;
        const int q = s_q, tile = s_tile;
        const DevProblem &p = a.probs[q];
        const int S = p.S;
        const int last = p.U - 1;
        if (q != q_prev) {
            if (a.k2_hist && threadIdx.x == 0) atomicAdd(a.k2_hist + 58, 1ull);   // debug: restaging
            const Cell *lc = a.cells + p.cell_off + (int64_t)last * S;
            const CellMem *lm = a.cmem + p.cell_off + (int64_t)last * S;
            for (int i = threadIdx.x; i < S; i += blockDim.x) {
                const Cell c = lc[i];
                sW[i] = c.w; sK[i] = c.k; sC[i] = c.c; sE[i] = c.ef;
                sOB[i] = lm[i].o_b;
            }
            if (p.U * S <= kSweepWK) {
                const Cell *cells = a.cells + p.cell_off;
                for (int x = threadIdx.x; x < p.U * S; x += blockDim.x)
                    sWK[x] = ((uint32_t)cells[x].w << 4) | (uint32_t)cells[x].k;
            }
            if (last >= 1 && rmap_groups(p.n_b + 1) <= kSweepRmap) {
                const int ng = (int)rmap_groups(p.n_b + 1);
                const int2 *src = a.rmap + p.rmap_off + (int64_t)(last - 1) * ng;
                for (int x = threadIdx.x; x < ng; x += blockDim.x) sRM[x] = src[x];
            }
            __syncthreads();
            q_prev = q;
        }
        const double safe_limit = safe_limit_of(a, p, q);
        const double b_up = __longlong_as_double((long long)a.bup[q]);
        RowCtx r;
        r.w = sW; r.k = sK; r.c = sC; r.ef = sE;
        r.n_e = p.n_b + 1;
        r.init = (last == 0);
        r.lo = (last == 0) ? 0 : a.unit_lo[p.ustate_off + last];
        r.bin = a.TF[last & 1] + p.b_off;
        r.K = p.K;
        r.rm = a.rmap + p.rmap_off + (int64_t)(last >= 1 ? last - 1 : 0) * rmap_groups(p.n_b + 1);
        r.rms = (rmap_groups(p.n_b + 1) <= kSweepRmap) ? sRM : nullptr;
        unsigned long long *bound = a.bound + 2 * q;
        const int64_t e = 1 + (int64_t)tile * kSweepThreads + threadIdx.x;
        // whole-tile prune: every candidate of the tile has T >= t0(top row) (the rank-0 time
        // is non-increasing in e), so the tile cannot win if t0(top) loses to the bound
        if (threadIdx.x < 32) {
            const int64_t e_top = min((int64_t)tile * kSweepThreads + kSweepThreads, p.n_b);
            double tmin = GBMW_INF;
            for (int j = lane; j < S; j += 32) {
                double T, F;
                row_value(r, e_top, j, T, F);
                tmin = fmin(tmin, T);
            }
            for (int off = 16; off > 0; off >>= 1) tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, off));
            if (lane == 0) {
                double bt;
                int64_t be;
                bound_read(bound, bt, be);
                s_skip = !(tmin < GBMW_INF) || tmin > bt || (tmin == bt && e_top < be);
            }
        }
        __syncthreads();
        if (s_skip) {
            if (a.k2_hist && threadIdx.x == 0) atomicAdd(a.k2_hist + 59, 1ull);   // debug: pruned by t0
            if (threadIdx.x == 0) {
                SweepPartial none;
                none.t = GBMW_INF; none.e = -1; none.j = 0; none.pad_ = 0;
                a.partials[p.tile_off + tile] = none;
                atomicMax(a.upruned + q, tile + 1);   // every tile below this one is pruned too
            }
            continue;
        }
        // flat warp: the candidate order is the same in all its rows; read the row values
        // at the warp's first row (broadcast).  Walks stay per row.
        const int64_t e_w0 = e - lane;
        bool flat = true;
        {
            const uint32_t *fl = a.chg[last & 1] + p.flag_off;
            const int nw = (int)flag_words(p.n_b + 1);
            for (int n = lane; n < S; n += 32) {
                const int w = sW[n];
                if (last == 0) flat = flat && ((e_w0 >= w) || (e_w0 + 31 < w));
                else flat = flat && window_flat((int)(e_w0 - w), (int)r.lo, fl + (int64_t)sK[n] * nw);
            }
        }
        flat = __all_sync(0xffffffffu, flat);
        const int64_t e_val = flat ? e_w0 : e;
        double mt = GBMW_INF;
        int64_t me = -1;
        int mj = 0;
        const bool wk_smem = p.U * S <= kSweepWK;
        if (e <= p.n_b && !int_le_double(e * p.gran, safe_limit)) {
            ++n_rows;
            uint16_t path[kMaxUnits];
            double ct = 0.0, cf = 0.0;
            int cj = -1;
            double qt = GBMW_INF, qf = GBMW_INF;                // the candidate after the next one, from
            int qj = -1;                                        // the same scan (consumed without a rescan)
            while (true) {
                double nt = GBMW_INF, nf = GBMW_INF;            // next candidate in (T, F, j) order
                int nj = -1;
                if (qj >= 0) {
                    nt = qt; nf = qf; nj = qj; qj = -1;
                } else {
                    for (int j = 0; j < S; ++j) {
                        double T, F;
                        row_value(r, e_val, j, T, F);
                        if (!(T < GBMW_INF)) continue;
                        if (cj >= 0 && !lex_less(ct, cf, cj, T, F, j)) continue;
                        if (nj < 0 || lex_less(T, F, j, nt, nf, nj)) {
                            qt = nt; qf = nf; qj = nj;
                            nt = T; nf = F; nj = j;
                        } else if (qj < 0 || lex_less(T, F, j, qt, qf, qj)) {
                            qt = T; qf = F; qj = j;
                        }
                    }
                }
                if (nj < 0) break;
                {
                    double bt;
                    int64_t be;
                    bound_read(bound, bt, be);
                    if (nt > bt || (nt == bt && e < be)) break;            // cannot win
                }
                ++n_cands;
                // E_all <= sum(O_f) + max O_b + sum(O_ms) <= F + b_up: a candidate under the
                // budget by more than the rounding of both sums fits without the walk
                if ((nf + b_up) * (1.0 + 1e-9) <= p.budget) {
                    mt = nt; me = e; mj = nj;
                    bound_offer(bound, nt, e);
                    break;
                }
                // E_all >= sum(O_f) + sum(O_ms) + O_b(last layer) = F + O_b(last unit, nj): a
                // candidate over the budget by more than the rounding of both sums cannot fit
                if ((nf + sOB[nj]) * (1.0 - 1e-9) > p.budget) {
                    ct = nt; cf = nf; cj = nj;
                    continue;
                }
                ++n_checks;
                if (wk_smem) backtrack_wk(a, p, e, nj, path, sWK, r.rms);
                else backtrack(a, p, e, nj, path);
                if (plan_e_all<GBMW_EALL_B_K3>(a, p, path) <= p.budget) {
                    mt = nt; me = e; mj = nj;
                    bound_offer(bound, nt, e);
                    break;
                }
                ct = nt; cf = nf; cj = nj;
            }
        }
        const SweepPartial blk = block_best(mt, me, mj, red_t, red_e, red_j);
        if (threadIdx.x == 0) a.partials[p.tile_off + tile] = blk;
    }
    for (int off = 16; off > 0; off >>= 1) {
        n_rows += __shfl_xor_sync(0xffffffffu, n_rows, off);
        n_cands += __shfl_xor_sync(0xffffffffu, n_cands, off);
        n_checks += __shfl_xor_sync(0xffffffffu, n_checks, off);
    }
    // three statistics counters for the whole pass: one atomic each per CTA, not per warp
    // (same-address atomics serialise in L2 and the grid completes only after them); the
    // tile loop above is CTA-uniform, so every thread gets here
    __shared__ unsigned long long s_st[kSweepThreads / 32][3];
    if (lane == 0) {
        const int wid = threadIdx.x >> 5;
        s_st[wid][0] = n_rows; s_st[wid][1] = n_cands; s_st[wid][2] = n_checks;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long tot = 0;
        for (int w = 0; w < kSweepThreads / 32; ++w) tot += s_st[w][threadIdx.x];
        if (tot) atomicAdd(a.sweep_stats + threadIdx.x, tot);
    }
}

// choices of the collapsed DP, walked back from bucket e (dpsearch.py:366-373)
__device__ __forceinline__ void approx_reconstruct(const ChunkArgs &a, const DevProblem &p, int64_t e,
                                                   uint16_t *path) {
    const int64_t n_e = p.n_b + 1;
    const int16_t *ch = reinterpret_cast<const int16_t *>(a.par + p.par_off);
    const Cell *cells = a.cells + p.cell_off;
    for (int u = p.U - 1; u >= 0; --u) {
        const int j = ch[(int64_t)u * n_e + e];
        path[u] = (uint16_t)j;
        e -= cells[(int64_t)u * p.S + j].w;
    }
}

// K3r: every row of one tile of a problem that wants the frontier or uses the collapsed
// DP.  Frontier: the rank-0 time of each row (dpsearch.py:197-199).  Collapsed DP: the
// one recorded candidate per row (dpsearch.py:360-364); safe rows accept it, unsafe ones
// check E_all of the reconstructed plan; the tile's best goes to partials.
__global__ void __launch_bounds__(kSweepThreads) k_sweep_rows(ChunkArgs a) {
    __shared__ int32_t sW[kMaxStrats];
    __shared__ int32_t sK[kMaxStrats];
    __shared__ double sC[kMaxStrats];
    __shared__ double sE[kMaxStrats];
    __shared__ int32_t sJ[kMaxStrats];
    __shared__ double red_t[kSweepThreads / 32];
    __shared__ long long red_e[kSweepThreads / 32];
    __shared__ int red_j[kSweepThreads / 32];
    const int2 m = a.aux_map[blockIdx.x];
    const int q = m.x, tile = m.y;
    const DevProblem &p = a.probs[q];
    const int64_t e = 1 + (int64_t)tile * kSweepThreads + threadIdx.x;
    if (p.flags & GBMW_APPROX) {
        const double safe_limit = safe_limit_of(a, p, q);
        const TFCell *tab = a.TF[(p.U - 1) & 1] + p.b_off;
        double mt = GBMW_INF;
        int64_t me = -1;
        if (e <= p.n_b) {
            const double t = tab[e].t;
            if (p.frontier_off >= 0) a.frontier[p.frontier_off + e - 1] = t;
            if (t < GBMW_INF) {
                bool fits = int_le_double(e * p.gran, safe_limit);
                if (!fits) {
                    uint16_t path[kMaxUnits];
                    approx_reconstruct(a, p, e, path);
                    fits = plan_e_all<GBMW_EALL_B_K3>(a, p, path) <= p.budget;
                }
                if (fits) { mt = t; me = e; }
            }
        }
        const SweepPartial blk = block_best(mt, me, 0, red_t, red_e, red_j);
        if (threadIdx.x == 0) a.partials[p.tile_off + tile] = blk;
        return;
    }
    if (p.frontier_off < 0) return;
    const int last = p.U - 1;
    const int64_t t_hi = (int64_t)tile * kSweepThreads + kSweepThreads;
    if (t_hi < first_finite_row(a, p)) {
        if (e <= p.n_b) a.frontier[p.frontier_off + e - 1] = GBMW_INF;
        return;
    }
    // rank-0 candidate = lexmin over the distinct strategies (duplicates never win ties)
    const Cell *lc = a.cells + p.cell_off + (int64_t)last * p.S;
    const int32_t *ul = a.uniq + p.cell_off + (int64_t)last * p.S;
    const int S = a.nuniq[p.ustate_off + last];
    for (int n = threadIdx.x; n < S; n += blockDim.x) {
        const int j = ul[n];
        const Cell c = lc[j];
        sW[n] = c.w; sK[n] = c.k; sC[n] = c.c; sE[n] = c.ef; sJ[n] = j;
    }
    __syncthreads();
    RowCtx r;
    r.w = sW; r.k = sK; r.c = sC; r.ef = sE;
    r.n_e = p.n_b + 1;
    r.init = (last == 0);
    r.lo = (last == 0) ? 0 : a.unit_lo[p.ustate_off + last];
    r.bin = a.TF[last & 1] + p.b_off;
    r.K = p.K;
    r.rm = a.rmap + p.rmap_off + (int64_t)(last >= 1 ? last - 1 : 0) * rmap_groups(p.n_b + 1);
    r.rms = nullptr;
    if (e <= p.n_b) {
        double t0 = GBMW_INF, f0 = GBMW_INF;
        int j0 = -1;
        for (int n = 0; n < S; ++n) {
            double T, F;
            row_value(r, e, n, T, F);
            const int j = sJ[n];
            if (T < GBMW_INF && (j0 < 0 || lex_less(T, F, j, t0, f0, j0))) { t0 = T; f0 = F; j0 = j; }
        }
        a.frontier[p.frontier_off + e - 1] = t0;
    }
}

// ---------------------------------------------------------------- approx_prev (collapsed DP)
// dpsearch.py:306-375: state (unit, bucket) only.  table_u[e] = lexmin_j (cand, cand_f, j)
// with cand = (table_{u-1}[e-w] + R(choice_{u-1}[e-w] -> j)) + time_c, cand_f =
// fwd_{u-1}[e-w] + ef_true (_lex_pick: min time, then min tiebreak, then first j).
// Per problem: table/fwd ping-pong = one TF column, choices = U x n_e int16 in `par`.
constexpr int kApproxRowsPerThread = kStepRows / kStepThreads;

template <bool FIRST>
__global__ void __launch_bounds__(kStepThreads) k_approx_step(ChunkArgs a, int u, int64_t tile_base, int64_t n_tiles,
                                                               unsigned long long *counter) {
    __shared__ int32_t sW[kMaxStrats];
    __shared__ int32_t sK[kMaxStrats];
    __shared__ double sC[kMaxStrats];
    __shared__ double sE[kMaxStrats];
    __shared__ double sR[kMaxClasses * kMaxClasses];
    __shared__ int64_t s_next;
    int q_prev = -1;
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) s_next = (int64_t)atomicAdd(counter, 1ull);
        __syncthreads();
        const int64_t t = s_next;
        if (t >= n_tiles) break;
        const int64_t tile = tile_base + t;
        const int q = a.step_map[tile];
        const DevProblem &p = a.probs[q];
        if (q != q_prev) {
            __syncthreads();
            const Cell *uc = a.cells + p.cell_off + (int64_t)u * p.S;
            for (int j = threadIdx.x; j < p.S; j += blockDim.x) {
                const Cell c = uc[j];
                sW[j] = c.w; sK[j] = c.k; sC[j] = c.c; sE[j] = c.ef;
            }
            const double *r_u = a.rcls + p.r_off + (int64_t)u * p.K * p.K;
            for (int x = threadIdx.x; x < p.K * p.K; x += blockDim.x) sR[x] = r_u[x];
            __syncthreads();
            q_prev = q;
        }
        const int S = p.S, K = p.K;
        const int64_t n_e = p.n_b + 1;
        const TFCell *tin = a.TF[(u - 1) & 1] + p.b_off;
        TFCell *tout = a.TF[u & 1] + p.b_off;
        const int16_t *cin = reinterpret_cast<const int16_t *>(a.par + p.par_off) + (int64_t)(u - 1) * n_e;
        int16_t *cout = reinterpret_cast<int16_t *>(a.par + p.par_off) + (int64_t)u * n_e;
        const int64_t first_row = (tile - a.step_tiles[q]) * kStepRows;
        for (int rr = 0; rr < kApproxRowsPerThread; ++rr) {
            const int64_t e = first_row + rr * kStepThreads + threadIdx.x;
            if (e >= n_e) break;
            double bt = GBMW_INF, bf = GBMW_INF;
            int bj = -1;
            for (int j = 0; j < S; ++j) {
                const int w = sW[j];
                if (w > p.n_b || e < w) continue;
                double tc, fc;
                if (FIRST) {
                    tc = sC[j]; fc = sE[j];
                } else {
                    const int64_t src = e - w;
                    const int pj = cin[src];
                    if (pj < 0) continue;                 // +inf source (no recorded choice)
                    const TFCell s = tin[src];
                    tc = (s.t + sR[sK[pj] * K + sK[j]]) + sC[j];
                    fc = s.f + sE[j];
                }
                if (bj < 0 || tc < bt || (tc == bt && fc < bf)) { bt = tc; bf = fc; bj = j; }
            }
            TFCell o;
            o.t = bt; o.f = bf;
            tout[e] = o;
            cout[e] = (int16_t)bj;
        }
    }
}

int launch_approx_step(const ChunkArgs &a, int u, int64_t tile_base, int64_t n_tiles, unsigned long long *counter,
                       void *stream) {
    if (n_tiles <= 0) return 0;
    const unsigned grid = (unsigned)(n_tiles < 148 * 8 ? n_tiles : 148 * 8);
    if (u == 0) k_approx_step<true><<<grid, kStepThreads, 0, (cudaStream_t)stream>>>(a, u, tile_base, n_tiles, counter);
    else k_approx_step<false><<<grid, kStepThreads, 0, (cudaStream_t)stream>>>(a, u, tile_base, n_tiles, counter);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------- K4: finalize
// One layer's stage-cost terms (costs.py:322-352): t + rc and t_ns + rc, rc the transform
// cost from the previous layer's strategy (0 for the first layer).
__device__ __forceinline__ void layer_terms(const ChunkArgs &a, const DevProblem &p, const gbmw_env &env, int l,
                                            int gs, int gs_prev, double *ta, double *tb) {
    const gbmw_strategy s = a.strats[gs];
    const StratDeg d = strat_degrees(s);
    const gbmw_layer L = a.layers[p.layer_begin + l];
    double t, t_ns;
    layer_times(L, s, d, p.micro, env, &t, &t_ns);
    double rc = 0.0;
    if (l > 0) {
        const StratDeg dp = strat_degrees(a.strats[gs_prev]);
        rc = transform_cost(L.bnd_bytes_per_sample, dp.data, dp.tp, d.data, d.tp, p.micro, env.intra_island_bw);
    }
    *ta = t + rc;
    *tb = t_ns + rc;
}

// K4: a warp per problem.  Lane 0 reduces the sweep partials, walks the argmin path and
// folds E_all (serial chains); the layers' plan entries and stage-cost terms are computed
// by all lanes, and lane 0 sums the terms in layer order (the reference's float order).
constexpr int kFinWarps = 4;
constexpr int kFinLayers = 256;
__global__ void __launch_bounds__(32 * kFinWarps) k_finalize(ChunkArgs a) {
    __shared__ uint16_t s_path[kFinWarps][kMaxUnits];
    __shared__ int32_t s_gs[kFinWarps][kFinLayers];
    __shared__ double s_ta[kFinWarps][kFinLayers], s_tb[kFinWarps][kFinLayers];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = blockIdx.x * kFinWarps + warp;
    if (q >= a.n_probs) return;                          // warp-uniform
    const DevProblem &p = a.probs[q];
    uint16_t *path = s_path[warp];
    gbmw_result res;
    double bt = GBMW_INF, e_all = 0.0;
    int64_t be = -1;
    int sj = 0;
    {
        // the best of the safe bucket and the unsafe (or collapsed-DP) tiles' partials: the
        // lanes take the tiles in turn, then a butterfly.  "better" (smaller t, ties to the
        // larger e) is a strict total order on the candidates (their e are distinct; the empty
        // ones are (inf, -1, 0) alike), so the result is the sequential fold's
        const SweepPartial safe = a.best[q];
        bt = safe.t;
        be = safe.e;
        int bj = safe.j;
        for (int t = a.ufirst[q] + lane; t < p.n_sweep_tiles; t += 32) {
            const SweepPartial sp = a.partials[p.tile_off + t];
            if (cand_better(sp.t, sp.e, bt, be)) { bt = sp.t; be = sp.e; bj = sp.j; }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ot = __shfl_xor_sync(0xffffffffu, bt, off);
            const long long oe = __shfl_xor_sync(0xffffffffu, (long long)be, off);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
            if (cand_better(ot, oe, bt, be)) { bt = ot; be = oe; bj = oj; }
        }
        sj = bj;
    }
    if (lane == 0) {
        const int bj = sj;
        if (be >= 0 && (p.flags & GBMW_APPROX)) approx_reconstruct(a, p, be, path);
        if (be >= 0 && !(p.flags & GBMW_APPROX) && p.S > 64) backtrack(a, p, be, bj, path);
        sj = bj;
    }
    be = __shfl_sync(0xffffffffu, be, 0);
    if (be >= 0 && !(p.flags & GBMW_APPROX) && p.S <= 64)
        backtrack_warp(a, p, be, __shfl_sync(0xffffffffu, sj, 0), path, lane);
    __syncwarp();
    if (lane == 0 && be >= 0) e_all = plan_e_all<8>(a, p, path);
    int32_t *plan = a.plans + p.plan_off;
    if (be < 0) {
        for (int l = lane; l < p.n_layers; l += 32) plan[l] = -1;
        if (lane == 0) {
            res.frontier_offset = -1;
            res.status = GBMW_OK;
            res.stage_time_s = 0.0; res.stage_time_no_sync_s = 0.0; res.stage_peak_mem_bytes = 0.0;
            res.time_s = GBMW_INF; res.e_fwd_used = 0.0; res.feasible = 0;
            a.results[p.result_index] = res;
        }
        return;
    }
    const gbmw_env env = a.envs[p.env_index];
    const bool cost = (p.flags & GBMW_STAGE_COST) != 0;
    const bool wide = p.n_layers <= kFinLayers;         // layer terms by all lanes
    __syncwarp();
    if (wide) {                                          // expand units to layers (dpsearch.py:230-234)
        int base = 0;                                    // lane u: unit u0 + u at its layer offset
        for (int u0 = 0; u0 < p.U; u0 += 32) {
            const int u = u0 + lane;
            int gs = 0, cnt = 0;
            if (u < p.U) { gs = a.cand_strat[p.cand_off + path[u]]; cnt = a.unit_count[p.unit_off + u]; }
            int incl = cnt;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += v;
            }
            for (int r = 0, l = base + incl - cnt; r < cnt; ++r, ++l) s_gs[warp][l] = gs;
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncwarp();
    double time_s = 0.0, no_sync = 0.0;
    int32_t first_pp = 1;
    if (wide) {
        for (int l = lane; l < p.n_layers; l += 32) {
            const int gs = s_gs[warp][l];
            plan[l] = gs - p.strat_begin;
            if (cost) layer_terms(a, p, env, l, gs, l > 0 ? s_gs[warp][l - 1] : gs, &s_ta[warp][l], &s_tb[warp][l]);
        }
        __syncwarp();
        if (lane == 0) {
            first_pp = a.strats[s_gs[warp][0]].pp_degree;
            if (cost)
                for (int l = 0; l < p.n_layers; ++l) {
                    time_s = time_s + s_ta[warp][l];
                    no_sync = no_sync + s_tb[warp][l];
                }
        }
    } else if (lane == 0) {                              // long stages: lane 0 alone
        int l = 0, gs_prev = 0;
        for (int u = 0; u < p.U; ++u) {
            const int gs = a.cand_strat[p.cand_off + path[u]];
            const int cnt = a.unit_count[p.unit_off + u];
            for (int r = 0; r < cnt; ++r, ++l) {
                plan[l] = gs - p.strat_begin;
                if (cost) {
                    double ta, tb;
                    layer_terms(a, p, env, l, gs, gs_prev, &ta, &tb);
                    time_s = time_s + ta;
                    no_sync = no_sync + tb;
                }
                if (l == 0) first_pp = a.strats[gs].pp_degree;
                gs_prev = gs;
            }
        }
    }
    if (lane != 0) return;
    res.frontier_offset = -1;
    res.status = GBMW_OK;
    res.stage_time_s = 0.0; res.stage_time_no_sync_s = 0.0; res.stage_peak_mem_bytes = 0.0;
    res.time_s = bt;
    res.e_fwd_used = (double)(be * p.gran);
    res.feasible = 1;
    if (!(e_all <= p.budget)) res.status = GBMW_EINTERNAL;   // dpsearch.py:220
    if (cost) {
        if (p.stage_index > 1) {
            const double p2p = stage_p2p_time(a.layers[p.layer_begin].bnd_bytes_per_sample,
                                              p.micro, first_pp, env);
            time_s = time_s + p2p;
            no_sync = no_sync + p2p;
        }
        res.stage_time_s = time_s;
        res.stage_time_no_sync_s = no_sync;
        res.stage_peak_mem_bytes = e_all;
    }
    a.results[p.result_index] = res;
}

// ---------------------------------------------------------------- launchers
static inline unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

int launch_cost_tables(const ChunkArgs &a, int64_t n_cells, int64_t n_r, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_cells > 0) k_cost_cells<<<blocks_for(n_cells, 128), 128, 0, st>>>(a, n_cells);
    if (n_r > 0) k_cost_r<<<blocks_for(n_r, 128), 128, 0, st>>>(a, n_r);
    if (a.n_units > 0 && a.n_probs > 0) {
        k_dedupe<<<blocks_for(a.n_units * 32, 128), 128, 0, st>>>(a);
        k_unit_ranges<<<blocks_for((int64_t)a.n_probs * 32, 128), 128, 0, st>>>(a);
    }
    return (int)cudaGetLastError();
}

int launch_sweep(const ChunkArgs &a, void *stream, int ctas_per_sm) {
    if (a.n_probs <= 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    k_sweep_safe<<<blocks_for(a.n_probs, 4), 128, 0, st>>>(a);
    if (a.n_aux > 0) k_sweep_rows<<<(unsigned)a.n_aux, kSweepThreads, 0, st>>>(a);
    k_sweep_scan<<<1, 1024, 0, st>>>(a);
    static int occ_of[64] = {0}, sms_of[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!occ_of[dev]) {
        int occ = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep_unsafe, kSweepThreads, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        sms_of[dev] = sms > 0 ? sms : 148;
        occ_of[dev] = occ > 0 ? occ : 1;
    }
    const int per_sm = (ctas_per_sm > 0 && ctas_per_sm < occ_of[dev]) ? ctas_per_sm : occ_of[dev];
    k_sweep_unsafe<<<per_sm * sms_of[dev], kSweepThreads, 0, st>>>(a);
    return (int)cudaGetLastError();
}

int launch_finalize(const ChunkArgs &a, void *stream) {
    if (a.n_probs <= 0) return 0;
    k_finalize<<<blocks_for(a.n_probs, kFinWarps), 32 * kFinWarps, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

}  // namespace gbmw
