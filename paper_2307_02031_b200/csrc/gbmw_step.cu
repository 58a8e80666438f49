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
// row, computed once.  Change points of B_u are emitted as one bit per (class, row)
// (bit x = row x differs from row x-1), exactly; a spurious 1 bit would only cost
// work, never exactness.
//
// One CTA processes one tile of kStepRows rows of one problem:
//   1. classify the tile's 32-row groups (dead / flat / full) from the change bits,
//   2. compute the list of rows that need it: every row of a full group (one warp per
//      group, lanes in row order), one row per flat group, and the row before the
//      tile (for the first change bit),
//   3. write flat groups' rows from shared memory, and the change-bit words.
// Tie-break T1 (lexicographic (cand, F, i), first i) is the one of every row.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gbmw_internal.h"

namespace gbmw {

#define GBMW_STEP_INF __longlong_as_double(0x7ff0000000000000LL)

constexpr int kStepIB = 4;                  // strategy batch: independent loads in flight
constexpr int kClassifyIB = 8;              // window checks per thread in flight
constexpr int kGroups = kStepRows / 32;     // 32-row groups per tile
constexpr int kMaxGfWords = (int)(((GBMW_MAX_BUCKETS + 1 + 31) / 32 + 31) / 32 + 1);   // gflat_words(max n_e)

constexpr int kWarpRows = 1024;             // rows per warp tile: 32 groups, one flat-mask word
constexpr int kSlots = 65;                  // evaluated rows held per round (+ slot 0: carry)

// Per-warp scratch of one tile.  Entry = an evaluated row; entry 0 is the row before the tile.
template <int KM>
struct WarpScratch {
    double et[kSlots][KM], ef[kSlots][KM];  // per round: slot 0 = last entry of the previous round
    int16_t ep[kSlots][KM];                 // argmin (position in the distinct list)
    unsigned epc[kSlots];                   // bit kk: the argmin's source path changes at this row
    uint16_t erow[kWarpRows + 2];           // row of each entry, relative to the tile's first row - 1
};

// KM: class capacity of the instantiation (4 / 8 / kMaxClasses)
template <int KM>
struct StepShared {
    Cell cell[kMaxStrats];                  // distinct source strategies of unit u-1 (ascending)
    int idx[kMaxStrats];                    // their strategy index
    double r[KM * KM];
    uint32_t gfp[kMaxGfWords];              // flat-group mask of B_{u-1} (read redirection, flat_row)
    int S, K, n_e, lo_prev, lo, hi, nw, gw;
    int64_t b_off, par_off, f_off;
    int64_t gf_cur;                         // flat-group mask of B_u (offset into a.gflat)
    int64_t next;
    int tnext, tlast;                       // warp tiles of the current problem
    WarpScratch<KM> w[kStepThreads / 32];
};

// K lexmins of one source row e' (T1 tie-break).  Rows outside [lo_prev + w, hi] read +inf.
template <int KT, bool FIRST, bool GUARD, class SH>
__device__ __forceinline__ void relax_row(const ChunkArgs &a, const SH &sh, int u, int e,
                                          double *bt, double *bf, int *bp) {
    const int S = sh.S, K = GUARD ? sh.K : KT;
    const int n_e = sh.n_e, lo_prev = FIRST ? 0 : sh.lo_prev, hi = sh.hi;
    const TFCell *bin = a.TF[(u - 1) & 1] + sh.b_off;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) { bt[kk] = GBMW_STEP_INF; bf[kk] = GBMW_STEP_INF; bp[kk] = 0; }
    const bool row_ok = e >= 0 && e <= hi;
    for (int i0 = 0; i0 < S; i0 += kStepIB) {
        double T[kStepIB], F[kStepIB];
#pragma unroll
        for (int b = 0; b < kStepIB; ++b) {
            const int i = i0 + b;
            const Cell c = sh.cell[i < S ? i : 0];
            const int src = e - c.w;
            T[b] = GBMW_STEP_INF; F[b] = GBMW_STEP_INF;
            if (i < S && row_ok && src >= lo_prev) {
                if (FIRST) {                       // init row, dpsearch.py:255-259
                    T[b] = c.c; F[b] = c.ef;
                } else {
                    const int g = src >> 5;
                    const int rs = ((sh.gfp[g >> 5] >> (g & 31)) & 1u) ? (src & ~31) : src;
                    const double2 v = __ldg(reinterpret_cast<const double2 *>(bin + c.k * n_e + rs));
                    T[b] = v.x + c.c;
                    F[b] = v.y + c.ef;
                }
            }
        }
#pragma unroll
        for (int b = 0; b < kStepIB; ++b) {
            const int i = i0 + b;
            if (i >= S) break;
            const int ck = sh.cell[i].k;
            const double *rrow = sh.r + ck * K;
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
                if (!GUARD || kk < K) {
                    const double cand = T[b] + rrow[kk];
                    const bool better = (cand < bt[kk]) || (cand == bt[kk] && F[b] < bf[kk]);
                    bt[kk] = better ? cand : bt[kk];
                    bf[kk] = better ? F[b] : bf[kk];
                    bp[kk] = better ? i : bp[kk];       // position in the distinct list
                }
            }
        }
    }
}

// Path-change bit of row e with argmin source n: the source cell B_{u-1}[e - w_n] differs
// (in value, argmin or path) from B_{u-1}[e - 1 - w_n].  Rows of B_u are "equal" (no change
// bit) only when value, argmin and the whole path behind match, so a flat group's first
// row stands for every row of the group, argmin chain included.
template <class SH>
__device__ __forceinline__ unsigned src_path_change(const ChunkArgs &a, const SH &sh, int u, int e, int n) {
    const Cell c = sh.cell[n];
    const int src = e - c.w;
    const uint32_t *fl = a.chg[(u - 1) & 1] + sh.f_off + (int64_t)c.k * sh.nw;
    return (__ldg(fl + (src >> 5)) >> (src & 31)) & 1u;
}

// Segment starts of a 32-row group contributed by one source: rows x (1..31) where the
// source's value T_{u-1}[r0 + x, i] may differ from row r0 + x - 1, i.e. the change bits of
// its window [x0, x0 + 31] of column cls(i) (rows below lo are +inf and constant).
__device__ __forceinline__ unsigned window_segments(unsigned long long v, int x0, int lo) {
    unsigned m = (unsigned)v;                            // bit j: row x0 + j vs x0 + j - 1
    if (x0 < lo) {
        const int j0 = lo - x0;                          // first finite row of the window
        m = (m & ~((2u << j0) - 1u)) | (1u << j0);
    }
    return m & 0xfffffffeu;
}

// One warp tile (kWarpRows rows) of B_u, by one warp; lane g owns 32-row group g.
// Rows are evaluated only where some source changes (segment starts): B_u is constant
// between them in value, argmin and path.  A group without segment starts is flat (its
// first row stands for all, stored once); other groups are evaluated at their first row and
// at each segment start and written in full.  Warp-synchronous: no CTA barrier.
template <int KT, bool FIRST, bool GUARD, class SH, class WS>
__device__ __forceinline__ unsigned long long warp_tile(const ChunkArgs &a, const SH &sh, WS &w, int u, int r_base,
                                                        int lane) {
    const int K = GUARD ? sh.K : KT;
    const int n_e = sh.n_e, lo = sh.lo, hi = sh.hi, S = sh.S;
    const int g = lane, r0 = r_base + 32 * g, r1 = r0 + 31;
    const bool dead = r1 < lo || r0 > hi;
    const bool whole = r0 >= lo && r1 <= hi;
    // ---- 1. segment starts of the group: change bits of every source window
    unsigned seg = (dead || whole) ? 0u : 0xfffffffeu;      // partial groups: every row evaluated
    if (whole) {
        const uint32_t *fin = a.chg[(u - 1) & 1] + sh.f_off;
        for (int n0 = 0; n0 < S; n0 += kClassifyIB) {
            uint32_t w0[kClassifyIB], w1[kClassifyIB];
            int xs_[kClassifyIB];
            bool ld[kClassifyIB];
#pragma unroll
            for (int b = 0; b < kClassifyIB; ++b) {
                const int n = n0 + b;
                const Cell c = sh.cell[n < S ? n : 0];
                const int xs = r0 - c.w;
                xs_[b] = xs; w0[b] = 0u; w1[b] = 0u;
                ld[b] = n < S && (FIRST || xs + 31 >= sh.lo_prev);
                if (!FIRST && ld[b]) {
                    const int xl = xs < 0 ? 0 : xs;
                    const uint32_t *fl = fin + (int64_t)c.k * sh.nw + (xl >> 5);
                    w0[b] = __ldg(fl); w1[b] = __ldg(fl + 1);
                }
            }
#pragma unroll
            for (int b = 0; b < kClassifyIB; ++b) {
                if (!ld[b]) continue;
                const int xs = xs_[b];
                if (FIRST) {
                    const int j = -xs;                   // T_0[e, i] is finite from e = w_i on
                    seg |= (j >= 1 && j <= 31) ? (1u << j) : 0u;
                } else {
                    const int xl = xs < 0 ? 0 : xs;
                    const unsigned long long v =
                        ((unsigned long long)w1[b] << 32 | (unsigned long long)w0[b]) >> (xl & 31);
                    seg |= window_segments((xs < 0) ? (v << (-xs)) : v, xs, sh.lo_prev);
                }
            }
        }
    }
    const bool flat = whole && seg == 0u;
    // ---- 2. entries: 0 = row r_base - 1, then per group its first row and segment starts
    const int cnt = dead ? 0 : 1 + __popc(seg);
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    const int ebase = 1 + incl - cnt, eend = 1 + incl;
    const int n_ent = 1 + __shfl_sync(0xffffffffu, incl, 31);
    if (!dead) {
        int at = ebase;
        w.erow[at++] = (uint16_t)(32 * g + 1);
        unsigned m = seg;
        while (m) {
            const int x = __ffs(m) - 1;
            m &= m - 1u;
            w.erow[at++] = (uint16_t)(32 * g + 1 + x);
        }
    }
    if (lane == 0) w.erow[0] = 0;
    const bool prev_ok = r_base - 1 >= lo && r_base - 1 <= hi;
    const bool dead_prev = __shfl_up_sync(0xffffffffu, dead, 1);
    const bool pred_ok = (g == 0) ? prev_ok : !dead_prev;
    __syncwarp();
    TFCell *bout = a.TF[u & 1] + sh.b_off;
    uint16_t *pout = a.par + sh.par_off + (int64_t)(u - 1) * K * n_e;
    uint32_t *fout = a.chg[u & 1] + sh.f_off;
    const int wi = (r_base >> 5) + g;
    // ---- 3. rounds: whole groups whose entries fit the slots
    int gs = 0, E0 = 0;
    while (gs < 32) {
        const unsigned okm = __ballot_sync(0xffffffffu, g >= gs && eend - E0 <= kSlots - 1);
        const int ge = gs + __popc(okm);
        const int E1 = __shfl_sync(0xffffffffu, eend, ge - 1);
        for (int e0 = E0; e0 < E1; e0 += 32) {
            const int en = e0 + lane;
            if (en < E1) {
                const int e = r_base - 1 + (int)w.erow[en];
                const bool live = e >= lo && e <= hi && e < n_e;
                double bt[KT], bf[KT];
                int bp[KT];
                relax_row<KT, FIRST, GUARD>(a, sh, u, live ? e : -1, bt, bf, bp);
                unsigned pcm = 0u;
#pragma unroll
                for (int kk = 0; kk < KT; ++kk)
                    if (!FIRST && (!GUARD || kk < K) && live && bt[kk] < GBMW_STEP_INF)
                        pcm |= src_path_change(a, sh, u, e, bp[kk]) << kk;
                const int s = 1 + en - E0;
#pragma unroll
                for (int kk = 0; kk < KT; ++kk)
                    if (!GUARD || kk < K) { w.et[s][kk] = bt[kk]; w.ef[s][kk] = bf[kk]; w.ep[s][kk] = (int16_t)bp[kk]; }
                w.epc[s] = pcm;
            }
        }
        __syncwarp();
        const bool in_r = g >= gs && g < ge;
        const int s0 = ebase - E0 + 1, sp = s0 - 1;    // sp = 0: carried from the previous round
        // flat groups: one lane each
        if (in_r && flat) {
            for (int kk = 0; kk < K; ++kk) {
                const double t = w.et[s0][kk], f = w.ef[s0][kk];
                const int pp = w.ep[s0][kk];
                reinterpret_cast<double2 *>(bout)[(int64_t)kk * n_e + r0] = make_double2(t, f);
                pout[(int64_t)kk * n_e + r0] = (uint16_t)sh.idx[pp];
                const bool same = pred_ok && w.et[sp][kk] == t && w.ef[sp][kk] == f && w.ep[sp][kk] == pp &&
                                  !((w.epc[s0] >> kk) & 1u);
                if (wi < sh.nw) fout[(int64_t)kk * sh.nw + wi] = same ? 0u : 1u;
            }
        }
        // evaluated groups: the warp writes their 32 rows, one lane per row
        unsigned fullm = __ballot_sync(0xffffffffu, in_r && !dead && !flat);
        while (fullm) {
            const int gf = __ffs(fullm) - 1;
            fullm &= fullm - 1u;
            const unsigned segm = __shfl_sync(0xffffffffu, seg, gf);
            const int sf = __shfl_sync(0xffffffffu, s0, gf);
            const bool pok = __shfl_sync(0xffffffffu, pred_ok, gf);
            const int e = r_base + 32 * gf + lane;
            const bool live = e >= lo && e <= hi;
            const int s = sf + __popc(segm & ((2u << lane) - 2u));      // entry of row e's segment
            const bool start = lane > 0 && ((segm >> lane) & 1u);
            const int sq = (lane == 0) ? sf - 1 : s - 1;                // entry of the row before e
            const bool q_ok = (lane == 0) ? pok : true;
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
                if (GUARD && kk >= K) break;
                const double t = w.et[s][kk], f = w.ef[s][kk];
                const int pp = w.ep[s][kk];
                if (live) {
                    reinterpret_cast<double2 *>(bout)[(int64_t)kk * n_e + e] = make_double2(t, f);
                    pout[(int64_t)kk * n_e + e] = (uint16_t)sh.idx[pp];
                }
                bool chg = false;                       // inside a segment: same row
                if (lane == 0 || start)
                    chg = !(q_ok && w.et[sq][kk] == t && w.ef[sq][kk] == f && w.ep[sq][kk] == pp &&
                            !((w.epc[s] >> kk) & 1u));
                const unsigned m = __ballot_sync(0xffffffffu, chg);
                const int wf = (r_base >> 5) + gf;
                if (lane == 0 && wf < sh.nw) fout[(int64_t)kk * sh.nw + wf] = m;
            }
        }
        __syncwarp();
        if (ge < 32) {                                   // carry the round's last entry
            const int sl = E1 - E0;
            for (int kk = lane; kk < K; kk += 32) { w.et[0][kk] = w.et[sl][kk]; w.ef[0][kk] = w.ef[sl][kk]; w.ep[0][kk] = w.ep[sl][kk]; }
            if (lane == 0) w.epc[0] = w.epc[sl];
            __syncwarp();
        }
        gs = ge;
        E0 = E1;
    }
    // ---- 4. dead groups' change words (never read as flat), the tile's flat-group word
    if (dead && wi < sh.nw)
        for (int kk = 0; kk < K; ++kk) fout[(int64_t)kk * sh.nw + wi] = 0xffffffffu;
    const unsigned fm = __ballot_sync(0xffffffffu, flat);
    if (lane == 0 && (r_base >> 10) < sh.gw) a.gflat[sh.gf_cur + (r_base >> 10)] = fm;
    __syncwarp();
    return (unsigned long long)n_ent * (unsigned long long)K;
}

// Live-row work lists of every K2 launch of the chunk (one CTA per launch): per active
// problem with live rows, its warp tiles [L_u / kWarpRows, H_u / kWarpRows].
__global__ void __launch_bounds__(1024) k_step_lists(ChunkArgs a) {
    __shared__ int s_part[1024];
    const StepList sl = a.step_lists[blockIdx.x];
    const int tid = threadIdx.x;
    const int per = (sl.n + 1023) / 1024;
    const int x0 = sl.lo + min(sl.n, tid * per), x1 = sl.lo + min(sl.n, tid * per + per);
    int cnt = 0;
    for (int x = x0; x < x1; ++x) {
        const DevProblem &p = a.probs[x];
        if (a.unit_hi[p.ustate_off + sl.u] >= a.unit_lo[p.ustate_off + sl.u]) ++cnt;
    }
    s_part[tid] = cnt;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const int v = (tid >= off) ? s_part[tid - off] : 0;
        __syncthreads();
        s_part[tid] += v;
        __syncthreads();
    }
    int64_t at = sl.base + s_part[tid] - cnt;
    for (int x = x0; x < x1; ++x) {
        const DevProblem &p = a.probs[x];
        const int lo = a.unit_lo[p.ustate_off + sl.u], hi = a.unit_hi[p.ustate_off + sl.u];
        if (hi < lo) continue;
        a.step_items[at++] = make_int4(x, lo / kWarpRows, hi / kWarpRows, 0);
    }
    if (tid == 1023) a.step_count[blockIdx.x] = s_part[1023];
}

int launch_step_lists(const ChunkArgs &a, void *stream) {
    if (a.n_step_lists <= 0) return 0;
    k_step_lists<<<a.n_step_lists, 1024, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

// CTAs take problems (dynamic counter); their warps take the problem's warp tiles.
template <int GROUP, bool FIRST>
__global__ void __launch_bounds__(kStepThreads, GROUP == 0 ? 3 : (GROUP == 1 ? 2 : 1))
    k_dp_step(ChunkArgs a, int u, const int4 *items, const int64_t *count, unsigned long long *counter) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using SH = StepShared<GROUP == 0 ? 4 : (GROUP == 1 ? 8 : kMaxClasses)>;
    SH &sh = *reinterpret_cast<SH *>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto &w = sh.w[warp];
    unsigned long long stat_rows = 0;
    const int64_t n_items = *count;
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) sh.next = (int64_t)atomicAdd(counter, 1ull);
        __syncthreads();
        const int64_t t = sh.next;
        if (t >= n_items) break;
        const int4 item = __ldg(items + t);
        const int q = item.x;
        const DevProblem &p = a.probs[q];
        {
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
                sh.lo = a.unit_lo[p.ustate_off + u]; sh.hi = a.unit_hi[p.ustate_off + u];
                sh.b_off = p.b_off; sh.par_off = p.par_off;
                sh.f_off = p.flag_off; sh.nw = (int)flag_words(p.n_b + 1);
                sh.gw = gw;
                sh.gf_cur = p.gflat_off + (int64_t)(u - 1) * gw;
                sh.tnext = item.y; sh.tlast = item.z;
            }
        }
        __syncthreads();
        const int K = sh.K;
        while (true) {
            int tile = 0;
            if (lane == 0) tile = atomicAdd(&sh.tnext, 1);
            tile = __shfl_sync(0xffffffffu, tile, 0);
            if (tile > sh.tlast) break;
            const int r_base = tile * kWarpRows;
            if (GROUP == 0) {
                switch (K) {
                    case 1: stat_rows += warp_tile<1, FIRST, false>(a, sh, w, u, r_base, lane); break;
                    case 2: stat_rows += warp_tile<2, FIRST, false>(a, sh, w, u, r_base, lane); break;
                    case 3: stat_rows += warp_tile<3, FIRST, false>(a, sh, w, u, r_base, lane); break;
                    default: stat_rows += warp_tile<4, FIRST, false>(a, sh, w, u, r_base, lane); break;
                }
            } else if (GROUP == 1) {
                switch (K) {
                    case 5: stat_rows += warp_tile<5, FIRST, false>(a, sh, w, u, r_base, lane); break;
                    case 6: stat_rows += warp_tile<6, FIRST, false>(a, sh, w, u, r_base, lane); break;
                    case 7: stat_rows += warp_tile<7, FIRST, false>(a, sh, w, u, r_base, lane); break;
                    default: stat_rows += warp_tile<8, FIRST, false>(a, sh, w, u, r_base, lane); break;
                }
            } else {
                stat_rows += warp_tile<kMaxClasses, FIRST, true>(a, sh, w, u, r_base, lane);
            }
        }
    }
    if (lane == 0 && stat_rows) atomicAdd(a.computed_cells, stat_rows);
}

int launch_dp_step(const ChunkArgs &a, int group, int u, const int4 *items, const int64_t *count, int64_t n_tiles,
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
    if (fi) GBMW_KFN(G, true)<<<grid, kStepThreads, smem, st>>>(a, u, items, count, counter);                \
    else GBMW_KFN(G, false)<<<grid, kStepThreads, smem, st>>>(a, u, items, count, counter);
    if (group == 0) { GBMW_STEP(0) }
    else if (group == 1) { GBMW_STEP(1) }
    else { GBMW_STEP(2) }
#undef GBMW_STEP
#undef GBMW_PREP
#undef GBMW_KFN
    return (int)cudaGetLastError();
}

}  // namespace gbmw
