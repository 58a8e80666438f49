// gbmw_step.cu — K2, the min-plus layer step of the stage search, run-length aware.
//
// Reference step (dpsearch.py:261-280), restated per source row e' and target class k
// (DESIGN.md §3):
//   B_u[e',k] = lexmin_i (T_{u-1}[e',i] + R_u[cls i, k], F_{u-1}[e',i], i),
//   T_{u-1}[e',i] = B_{u-1}[e'-w_{u-1,i}, cls i].t + time_c[u-1,i]   (init row for u == 1).
// B is a step function of e': most aligned 32-row groups see the same (T, F) vector in
// every row (SURVEY-scale configs: 86-100 % of live groups).  A group is "flat" when,
// for every distinct source strategy i, the 32-row source window of column cls(i) of
// B_{u-1} contains no change point; its 32 outputs are then the output of its first
// row, computed once and stored once (readers redirect through the flat-group mask).
// Change points of B_u are emitted as one bit per (class, row) (bit x = row x differs
// from row x-1), exactly.
//
// Work split: a CTA takes tiles of kStepRows rows (dynamic tile counter); inside a tile
// each warp takes 32-row groups (dynamic group counter) and finishes them on its own:
//   - window check: lanes over the source strategies, one 64-bit read of change bits each;
//   - flat group: its first row, warp-cooperatively (lanes over sources, shuffle lexmin);
//   - full group: one row per lane;
//   - bit 0 of the group (row r0 vs r0-1): free when every source window extends one row
//     down unchanged (33-row check), else row r0-1 is computed warp-cooperatively.
// Only the tile boundaries synchronise the CTA.  Tie-break T1 (lexicographic (cand, F,
// i), first i) is the one of every row; the cooperative lexmin reduces (t, f, i).
#include <cuda_runtime.h>
#include <stdint.h>

#include "gbmw_internal.h"

namespace gbmw {

#define GBMW_STEP_INF __longlong_as_double(0x7ff0000000000000LL)

constexpr int kStepIB = 4;                  // sources per lane in flight
constexpr int kGroups = kStepRows / 32;     // 32-row groups per tile
constexpr int kMaxGfWords = (int)(((GBMW_MAX_BUCKETS + 1 + 31) / 32 + 31) / 32 + 1);   // gflat_words(max n_e)

// KM: class capacity of the instantiation (4 / 8 / kMaxClasses)
template <int KM>
struct StepShared {
    Cell cell[kMaxStrats];                  // distinct source strategies of unit u-1 (ascending)
    int idx[kMaxStrats];                    // their strategy index
    double r[KM * KM];
    uint32_t gfp[kMaxGfWords];              // flat-group mask of B_{u-1}
    int S, K, n_e, lo_prev, lo, hi, nw, gw;
    int64_t b_off, par_off, f_off, gf_cur;
    int64_t next;
    int gnext;
    uint32_t gmask[kGroups / 32];           // flat-group bits of the current tile
    // per warp: row r0 of its current group and the change bits of rows r0+1 .. r0+31
    double wt[kStepThreads / 32][KM], wf[kStepThreads / 32][KM];
    uint32_t wm[kStepThreads / 32][KM];
};

__device__ __forceinline__ int flat_row_s(const uint32_t *gfs, int row) {
    const int g = row >> 5;
    return ((gfs[g >> 5] >> (g & 31)) & 1u) ? (row & ~31) : row;
}

// (T, F) of source strategy c at target row e (reference table T_{u-1}[e, i])
template <bool FIRST, class SH>
__device__ __forceinline__ void src_value(const SH &sh, const TFCell *bin, const Cell &c, int e, bool ok, double &T,
                                          double &F) {
    T = GBMW_STEP_INF; F = GBMW_STEP_INF;
    const int src = e - c.w;
    if (ok && src >= (FIRST ? 0 : sh.lo_prev)) {
        if (FIRST) {                        // init row, dpsearch.py:255-259
            T = c.c; F = c.ef;
        } else {
            const double2 v = __ldg(reinterpret_cast<const double2 *>(bin + c.k * sh.n_e + flat_row_s(sh.gfp, src)));
            T = v.x + c.c;
            F = v.y + c.ef;
        }
    }
}

// fold candidate (T, F) of source n into the running lexmins (strict: first n wins ties)
template <int KT, bool GUARD, class SH>
__device__ __forceinline__ void fold(const SH &sh, int n, double T, double F, double *bt, double *bf, int *bp) {
    const int K = GUARD ? sh.K : KT;
    const double *rrow = sh.r + sh.cell[n].k * K;
    const int gi = sh.idx[n];
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
        if (!GUARD || kk < K) {
            const double cand = T + rrow[kk];
            const bool better = (cand < bt[kk]) || (cand == bt[kk] && F < bf[kk]);
            bt[kk] = better ? cand : bt[kk];
            bf[kk] = better ? F : bf[kk];
            bp[kk] = better ? gi : bp[kk];
        }
    }
}

// K lexmins of row e, one row per lane (e < 0: dead row, +inf)
template <int KT, bool FIRST, bool GUARD, class SH>
__device__ __forceinline__ void relax_row(const ChunkArgs &a, const SH &sh, int u, int e, double *bt, double *bf,
                                          int *bp) {
    const int S = sh.S;
    const TFCell *bin = a.TF[(u - 1) & 1] + sh.b_off;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) { bt[kk] = GBMW_STEP_INF; bf[kk] = GBMW_STEP_INF; bp[kk] = 0; }
    const bool row_ok = e >= 0;
    for (int i0 = 0; i0 < S; i0 += kStepIB) {
        double T[kStepIB], F[kStepIB];
#pragma unroll
        for (int b = 0; b < kStepIB; ++b) {
            const int i = i0 + b;
            src_value<FIRST>(sh, bin, sh.cell[i < S ? i : 0], e, i < S && row_ok, T[b], F[b]);
        }
#pragma unroll
        for (int b = 0; b < kStepIB; ++b) {
            if (i0 + b >= S) break;
            fold<KT, GUARD>(sh, i0 + b, T[b], F[b], bt, bf, bp);
        }
    }
}

// K lexmins of one row e, warp-cooperatively: lane l takes sources l, l+32, ...; the
// partial lexmins are reduced over (t, f, strategy index).  Result in every lane.
template <int KT, bool FIRST, bool GUARD, class SH>
__device__ __forceinline__ void relax_coop(const ChunkArgs &a, const SH &sh, int u, int e, int lane, double *bt,
                                           double *bf, int *bp) {
    const int S = sh.S, K = GUARD ? sh.K : KT;
    const TFCell *bin = a.TF[(u - 1) & 1] + sh.b_off;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) { bt[kk] = GBMW_STEP_INF; bf[kk] = GBMW_STEP_INF; bp[kk] = 0; }
    for (int n0 = lane; n0 < S; n0 += 32 * kStepIB) {
        double T[kStepIB], F[kStepIB];
#pragma unroll
        for (int b = 0; b < kStepIB; ++b) {
            const int n = n0 + 32 * b;
            src_value<FIRST>(sh, bin, sh.cell[n < S ? n : 0], e, n < S, T[b], F[b]);
        }
#pragma unroll
        for (int b = 0; b < kStepIB; ++b) {
            const int n = n0 + 32 * b;
            if (n >= S) break;
            fold<KT, GUARD>(sh, n, T[b], F[b], bt, bf, bp);
        }
    }
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
        if (GUARD && kk >= K) break;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ot = __shfl_xor_sync(0xffffffffu, bt[kk], off);
            const double of = __shfl_xor_sync(0xffffffffu, bf[kk], off);
            const int op = __shfl_xor_sync(0xffffffffu, bp[kk], off);
            const bool take = (ot < bt[kk]) || (ot == bt[kk] && (of < bf[kk] || (of == bf[kk] && op < bp[kk])));
            bt[kk] = take ? ot : bt[kk];
            bf[kk] = take ? of : bf[kk];
            bp[kk] = take ? op : bp[kk];
        }
    }
}

// Source window of rows [x0, x0+31] of one class column (change bits fl, rows below lo
// are +inf): f32 = constant on the window, e33 = constant on [x0-1, x0+31].
__device__ __forceinline__ void window_bits(int x0, int lo, const uint32_t *fl, bool &f32, bool &e33) {
    if (x0 + 31 < lo) { f32 = true; e33 = true; return; }
    if (x0 < lo) { f32 = false; e33 = false; return; }
    const int w0 = x0 >> 5, s = x0 & 31;
    const unsigned long long v =
        ((unsigned long long)__ldg(fl + w0 + 1) << 32 | (unsigned long long)__ldg(fl + w0)) >> s;
    f32 = (v & 0xfffffffeull) == 0ull;                 // bits of rows x0+1 .. x0+31
    e33 = (x0 - 1 >= lo) && (v & 0xffffffffull) == 0ull;   // and row x0 vs x0-1
}

// One 32-row group of B_u, by one warp.  Returns the rows computed (for the work counter).
template <int KT, bool FIRST, bool GUARD, class SH>
__device__ __forceinline__ int step_group(const ChunkArgs &a, SH &sh, int u, int r0, int g, int lane) {
    const int K = GUARD ? sh.K : KT;
    const int n_e = sh.n_e, lo = sh.lo, hi = sh.hi, r1 = r0 + 31;
    const int wi = r0 >> 5;
    uint32_t *fout = a.chg[u & 1] + sh.f_off;
    if (r1 < lo || r0 > hi) {                                   // dead rows: never read as flat
        if (wi < sh.nw)
            for (int kk = lane; kk < K; kk += 32) fout[(int64_t)kk * sh.nw + wi] = 0xffffffffu;
        return 0;
    }
    TFCell *bout = a.TF[u & 1] + sh.b_off;
    uint16_t *pout = a.par + sh.par_off + (int64_t)(u - 1) * K * n_e;
    const bool whole = r0 >= lo && r1 <= hi;
    bool flat = whole, ext = whole;
    if (whole) {
        const uint32_t *fin = a.chg[(u - 1) & 1] + sh.f_off;
        for (int n = lane; n < sh.S; n += 32) {
            const int x0 = r0 - sh.cell[n].w;
            bool f32, e33;
            if (FIRST) {
                f32 = (x0 >= 0) || (x0 + 31 < 0);
                e33 = (x0 - 1 >= 0) || (x0 + 31 < 0);
            } else {
                window_bits(x0, sh.lo_prev, fin + (int64_t)sh.cell[n].k * sh.nw, f32, e33);
            }
            flat = flat && f32;
            ext = ext && e33;
        }
        flat = __all_sync(0xffffffffu, flat);
        ext = __all_sync(0xffffffffu, ext);
    }
    const int warp = threadIdx.x >> 5;
    int rows;
    {
        double bt[KT], bf[KT];
        int bp[KT];
        if (flat) {
            relax_coop<KT, FIRST, GUARD>(a, sh, u, r0, lane, bt, bf, bp);
            rows = 1;
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
                if (GUARD && kk >= K) break;
                if (lane == kk) {
                    reinterpret_cast<double2 *>(bout)[(int64_t)kk * n_e + r0] = make_double2(bt[kk], bf[kk]);
                    pout[(int64_t)kk * n_e + r0] = (uint16_t)bp[kk];
                    sh.wt[warp][kk] = bt[kk]; sh.wf[warp][kk] = bf[kk]; sh.wm[warp][kk] = 0u;
                }
            }
            if (lane == 0) atomicOr(&sh.gmask[g >> 5], 1u << (g & 31));
        } else {
            const int e = r0 + lane;
            const bool live = e >= lo && e <= hi;
            relax_row<KT, FIRST, GUARD>(a, sh, u, live ? e : -1, bt, bf, bp);
            rows = 32;
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
                if (GUARD && kk >= K) break;
                if (live) {
                    reinterpret_cast<double2 *>(bout)[(int64_t)kk * n_e + e] = make_double2(bt[kk], bf[kk]);
                    pout[(int64_t)kk * n_e + e] = (uint16_t)bp[kk];
                }
                const double ut = __shfl_up_sync(0xffffffffu, bt[kk], 1);
                const double uf = __shfl_up_sync(0xffffffffu, bf[kk], 1);
                const unsigned m = __ballot_sync(0xffffffffu, lane > 0 && (ut != bt[kk] || uf != bf[kk]));
                if (lane == 0) { sh.wt[warp][kk] = bt[kk]; sh.wf[warp][kk] = bf[kk]; sh.wm[warp][kk] = m; }
            }
        }
    }
    __syncwarp();
    // bit 0 (row r0 vs r0-1): settled by the 33-row source windows, else row r0-1 is computed
    const bool need_b = !ext && (r0 - 1 >= lo);
    if (need_b) {
        double pt[KT], pf[KT];
        int pp[KT];
        relax_coop<KT, FIRST, GUARD>(a, sh, u, r0 - 1, lane, pt, pf, pp);
        rows += 1;
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) {
            if (GUARD && kk >= K) break;
            if (lane == kk && wi < sh.nw) {
                const bool same = pt[kk] == sh.wt[warp][kk] && pf[kk] == sh.wf[warp][kk];
                fout[(int64_t)kk * sh.nw + wi] = sh.wm[warp][kk] | (same ? 0u : 1u);
            }
        }
    } else if (wi < sh.nw) {
        for (int kk = lane; kk < K; kk += 32) fout[(int64_t)kk * sh.nw + wi] = sh.wm[warp][kk] | (ext ? 0u : 1u);
    }
    __syncwarp();
    return rows;
}

template <int KT, bool FIRST, bool GUARD, class SH>
__device__ void step_tile(const ChunkArgs &a, SH &sh, int u, int first_row, unsigned long long &stat_rows) {
    const int lane = threadIdx.x & 31;
    while (true) {
        int g = 0;
        if (lane == 0) g = atomicAdd(&sh.gnext, 1);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= kGroups) break;
        const int rows = step_group<KT, FIRST, GUARD>(a, sh, u, first_row + 32 * g, g, lane);
        stat_rows += (unsigned long long)rows * (unsigned long long)(GUARD ? sh.K : KT);
    }
}

template <int GROUP, bool FIRST>
__global__ void __launch_bounds__(kStepThreads, GROUP == 0 ? 3 : 2) k_dp_step(ChunkArgs a, int u, int64_t tile_base, int64_t n_tiles,
                                                           unsigned long long *counter) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using SH = StepShared<GROUP == 0 ? 4 : (GROUP == 1 ? 8 : kMaxClasses)>;
    SH &sh = *reinterpret_cast<SH *>(smem_raw);
    int q_prev = -1;
    unsigned long long stat_rows = 0;
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) sh.next = (int64_t)atomicAdd(counter, 1ull);
        __syncthreads();
        const int64_t t = sh.next;
        if (t >= n_tiles) break;
        const int64_t tile = tile_base + t;
        const int q = __ldg(a.step_map + tile);
        const DevProblem &p = a.probs[q];
        const int64_t first_row = (tile - a.step_tiles[q]) * kStepRows;
        const int lo = a.unit_lo[p.ustate_off + u], hi = a.unit_hi[p.ustate_off + u];
        if (first_row > hi || first_row + kStepRows - 1 < lo) continue;      // dead tile (CTA-uniform)
        if (q != q_prev) {
            const int S = p.S, K = p.K;
            const Cell *prev_cells = a.cells + p.cell_off + (int64_t)(u - 1) * S;
            const int32_t *ul = a.uniq + p.cell_off + (int64_t)(u - 1) * S;
            const int nu = a.nuniq[p.ustate_off + u - 1];
            for (int n = threadIdx.x; n < nu; n += blockDim.x) {
                const int j = ul[n];
                sh.cell[n] = prev_cells[j];
                sh.idx[n] = j;
            }
            const double *r_u = a.rcls + p.r_off + (int64_t)u * K * K;
            for (int x = threadIdx.x; x < K * K; x += blockDim.x) sh.r[x] = r_u[x];
            const int gw = (int)gflat_words(p.n_b + 1);
            if (!FIRST) {
                const uint32_t *gsrc = a.gflat + p.gflat_off + (int64_t)(u - 2) * gw;
                for (int x = threadIdx.x; x < gw; x += blockDim.x) sh.gfp[x] = gsrc[x];
            }
            if (threadIdx.x == 0) {
                sh.S = nu; sh.K = K; sh.n_e = (int)(p.n_b + 1);
                sh.lo_prev = a.unit_lo[p.ustate_off + u - 1];
                sh.lo = lo; sh.hi = hi;
                sh.b_off = p.b_off; sh.par_off = p.par_off;
                sh.f_off = p.flag_off; sh.nw = (int)flag_words(p.n_b + 1);
                sh.gw = gw;
                sh.gf_cur = p.gflat_off + (int64_t)(u - 1) * gw;
            }
            q_prev = q;
        }
        if (threadIdx.x < kGroups / 32) sh.gmask[threadIdx.x] = 0u;
        if (threadIdx.x == 0) sh.gnext = 0;
        __syncthreads();
        const int K = sh.K;
        if (GROUP == 0) {
            switch (K) {
                case 1: step_tile<1, FIRST, false>(a, sh, u, (int)first_row, stat_rows); break;
                case 2: step_tile<2, FIRST, false>(a, sh, u, (int)first_row, stat_rows); break;
                case 3: step_tile<3, FIRST, false>(a, sh, u, (int)first_row, stat_rows); break;
                default: step_tile<4, FIRST, false>(a, sh, u, (int)first_row, stat_rows); break;
            }
        } else if (GROUP == 1) {
            switch (K) {
                case 5: step_tile<5, FIRST, false>(a, sh, u, (int)first_row, stat_rows); break;
                case 6: step_tile<6, FIRST, false>(a, sh, u, (int)first_row, stat_rows); break;
                case 7: step_tile<7, FIRST, false>(a, sh, u, (int)first_row, stat_rows); break;
                default: step_tile<8, FIRST, false>(a, sh, u, (int)first_row, stat_rows); break;
            }
        } else {
            step_tile<kMaxClasses, FIRST, true>(a, sh, u, (int)first_row, stat_rows);
        }
        __syncthreads();
        // flat-group mask words of this tile (tiles are 1024-row-word aligned)
        if (threadIdx.x < kGroups / 32) {
            const int wi = (int)(first_row >> 10) + threadIdx.x;
            if (wi < sh.gw) a.gflat[sh.gf_cur + wi] = sh.gmask[threadIdx.x];
        }
    }
    // work counter: one atomic per warp
    for (int off = 16; off > 0; off >>= 1) stat_rows += __shfl_xor_sync(0xffffffffu, stat_rows, off);
    if ((threadIdx.x & 31) == 0 && stat_rows) atomicAdd(a.computed_cells, stat_rows);
}

int launch_dp_step(const ChunkArgs &a, int group, int u, int64_t tile_base, int64_t n_tiles,
                   unsigned long long *counter, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_tiles <= 0) return 0;
    const size_t smem = group == 0 ? sizeof(StepShared<4>) : (group == 1 ? sizeof(StepShared<8>)
                                                                           : sizeof(StepShared<kMaxClasses>));
    static int sms = 0;
    static int occ[kStepGroups][2] = {{0}};
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    const int fi = (u == 1) ? 1 : 0;
#define GBMW_KFN(G, F) k_dp_step<G, F>
#define GBMW_PREP(G, F)                                                                             \
    do {                                                                                            \
        cudaFuncSetAttribute(GBMW_KFN(G, F), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        int n = 1;                                                                                  \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, GBMW_KFN(G, F), kStepThreads, smem);      \
        occ[G][F ? 1 : 0] = n > 0 ? n : 1;                                                          \
    } while (0)
    if (occ[group][fi] == 0) {
        if (group == 0) { if (fi) GBMW_PREP(0, true); else GBMW_PREP(0, false); }
        else if (group == 1) { if (fi) GBMW_PREP(1, true); else GBMW_PREP(1, false); }
        else { if (fi) GBMW_PREP(2, true); else GBMW_PREP(2, false); }
    }
    const int64_t max_ctas = (int64_t)sms * occ[group][fi];
    const unsigned grid = (unsigned)(n_tiles < max_ctas ? n_tiles : max_ctas);
#define GBMW_STEP(G)                                                                                        \
    if (fi) GBMW_KFN(G, true)<<<grid, kStepThreads, smem, st>>>(a, u, tile_base, n_tiles, counter);          \
    else GBMW_KFN(G, false)<<<grid, kStepThreads, smem, st>>>(a, u, tile_base, n_tiles, counter);
    if (group == 0) { GBMW_STEP(0) }
    else if (group == 1) { GBMW_STEP(1) }
    else { GBMW_STEP(2) }
#undef GBMW_STEP
#undef GBMW_PREP
#undef GBMW_KFN
    return (int)cudaGetLastError();
}

}  // namespace gbmw
