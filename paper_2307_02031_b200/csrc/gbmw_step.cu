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

// KM: class capacity of the instantiation (4 / 8 / kMaxClasses), sizes the per-entry arrays
template <int KM>
struct StepShared {
    Cell cell[kMaxStrats];                  // distinct source strategies of unit u-1 (ascending)
    int idx[kMaxStrats];                    // their strategy index
    double r[KM * KM];
    uint32_t gfp[kMaxGfWords];              // flat-group mask of B_{u-1} (read redirection, flat_row)
    int S, K, n_e, q, lo_prev, lo, hi, nw;
    int64_t b_off, par_off, f_off;
    int64_t gf_cur;                         // flat-group mask of B_u (offset into a.gflat)
    int gw;
    int64_t next;
    // per tile
    int kind[kGroups];                      // 0 dead, 1 flat, 2 full
    unsigned seg[kGroups];                  // bit x (1..31): row x of the group starts a new segment
    int ebase[kGroups + 1];                 // first entry of each group; entry 0 = row first_row - 1
    int erow[kStepRows + 1];                // row of each entry (rows that are evaluated)
    int rg[kGroups + 1];                    // round r covers groups [rg[r], rg[r + 1])
    int n_rounds;
    int prev_ok;
    // per round: slot 0 = the last entry of the previous round, slot 1 + i = entry E0 + i
    double et[kStepThreads + 1][KM], ef[kStepThreads + 1][KM];
    int ep[kStepThreads + 1][KM];
    unsigned epc[kStepThreads + 1];         // bit kk: the argmin's source path changes at this row
    unsigned long long stat_rows;
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

// One tile of B_u.  Rows are evaluated only where some source changes (segment starts):
// B_u is constant between them in value, argmin and path.  A group without segment starts
// is flat (its first row stands for all, stored once); other groups are evaluated at their
// first row and at each segment start and written in full.  Evaluated rows ("entries") are
// processed in rounds of at most kStepThreads, one thread each.
template <int KT, bool FIRST, bool GUARD, class SH>
__device__ void step_tile(const ChunkArgs &a, SH &sh, int u, int first_row) {
    const int K = GUARD ? sh.K : KT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x, nwarp = nthr >> 5;
    const int n_e = sh.n_e, lo = sh.lo, hi = sh.hi, S = sh.S;
    // ---- 1. classify groups: dead / whole-live (segments from the source windows) / partial
    for (int g = tid; g < kGroups; g += nthr) {
        const int r0 = first_row + 32 * g, r1 = r0 + 31;
        const bool dead = r1 < lo || r0 > hi;
        const bool whole = r0 >= lo && r1 <= hi;
        sh.kind[g] = dead ? 0 : (whole ? 1 : 2);
        sh.seg[g] = whole ? 0u : 0xfffffffeu;            // partial groups: every row evaluated
    }
    __syncthreads();
    const uint32_t *fin = a.chg[(u - 1) & 1] + sh.f_off;
    const int n_checks = kGroups * S;
    for (int x0 = tid; x0 < n_checks; x0 += nthr * kClassifyIB) {
        uint32_t w0[kClassifyIB], w1[kClassifyIB];
        int xs_[kClassifyIB], gg[kClassifyIB];
#pragma unroll
        for (int b = 0; b < kClassifyIB; ++b) {
            const int x = x0 + b * nthr;
            gg[b] = -1; xs_[b] = 0; w0[b] = 0u; w1[b] = 0u;
            if (x < n_checks) {
                const int g = x / S, n = x - g * S;
                if (sh.kind[g] == 1) {
                    const Cell c = sh.cell[n];
                    const int r0 = first_row + 32 * g;
                    const int xs = r0 - c.w;
                    xs_[b] = xs;
                    if (FIRST) {
                        gg[b] = g;
                    } else if (xs + 31 >= sh.lo_prev) {
                        const int xl = xs < 0 ? 0 : xs;
                        const uint32_t *fl = fin + (int64_t)c.k * sh.nw + (xl >> 5);
                        w0[b] = __ldg(fl); w1[b] = __ldg(fl + 1);
                        gg[b] = g;
                    }
                }
            }
        }
#pragma unroll
        for (int b = 0; b < kClassifyIB; ++b) {
            if (gg[b] < 0) continue;
            const int xs = xs_[b];
            unsigned m;
            if (FIRST) {
                // T_0[e, i] is finite from e = w_i on: one segment start at row w_i
                const int j = -xs;                       // w_i - r0
                m = (j >= 1 && j <= 31) ? (1u << j) : 0u;
            } else {
                const int xl = xs < 0 ? 0 : xs;
                const unsigned long long v =
                    ((unsigned long long)w1[b] << 32 | (unsigned long long)w0[b]) >> (xl & 31);
                // v bit j = row xl + j; rows below xl (negative rows) are +inf like rows below lo
                const unsigned long long vv = (xs < 0) ? (v << (-xs)) : v;
                m = window_segments(vv, xs, sh.lo_prev);
            }
            if (m) atomicOr(&sh.seg[gg[b]], m);
        }
    }
    __syncthreads();
    // ---- 2. entries: row first_row - 1, then per group its first row and segment starts
    if (warp == 0) {
        int run = 1;
        for (int base = 0; base < kGroups; base += 32) {
            const int g = base + lane;
            int cnt = 0;
            if (g < kGroups) {
                const int kd = sh.kind[g];
                if (kd == 1 && sh.seg[g] != 0u) sh.kind[g] = 2;
                cnt = (kd == 0) ? 0 : 1 + __popc(sh.seg[g]);
            }
            int incl = cnt;
            for (int off = 1; off < 32; off <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += v;
            }
            if (g < kGroups) sh.ebase[g] = run + incl - cnt;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
            sh.ebase[kGroups] = run;
            sh.erow[0] = first_row - 1;
            sh.prev_ok = (first_row - 1 >= lo && first_row - 1 <= hi) ? 1 : 0;
            sh.stat_rows += (unsigned long long)run * (unsigned long long)K;
        }
    }
    __syncthreads();
    for (int g = tid; g < kGroups; g += nthr) {
        if (sh.kind[g] == 0) continue;
        const int r0 = first_row + 32 * g;
        int at = sh.ebase[g];
        sh.erow[at++] = r0;
        unsigned m = sh.seg[g];
        while (m) {
            const int x = __ffs(m) - 1;
            m &= m - 1u;
            sh.erow[at++] = r0 + x;
        }
    }
    if (tid == 0) {                                      // rounds of <= nthr entries, whole groups
        int r = 0, start = 0;
        sh.rg[0] = 0;
        for (int g = 0; g < kGroups; ++g)
            if (sh.ebase[g + 1] - start > nthr) { sh.rg[++r] = g; start = sh.ebase[g]; }
        sh.rg[r + 1] = kGroups;
        sh.n_rounds = r + 1;
    }
    __syncthreads();
    TFCell *bout = a.TF[u & 1] + sh.b_off;
    uint16_t *pout = a.par + sh.par_off + (int64_t)(u - 1) * K * n_e;
    uint32_t *fout = a.chg[u & 1] + sh.f_off;
    const int w_first = first_row >> 5;
    const int n_rounds = sh.n_rounds;
    for (int rd = 0; rd < n_rounds; ++rd) {
        const int g0 = sh.rg[rd], g1 = sh.rg[rd + 1];
        const int E0 = (rd == 0) ? 0 : sh.ebase[g0], E1 = sh.ebase[g1];
        // ---- 3. evaluate the round's entries
        if (E0 + tid < E1) {
            const int e = sh.erow[E0 + tid];
            const bool live = e >= lo && e <= hi && e < n_e;
            double bt[KT], bf[KT];
            int bp[KT];
            relax_row<KT, FIRST, GUARD>(a, sh, u, live ? e : -1, bt, bf, bp);
            unsigned pcm = 0u;
#pragma unroll
            for (int kk = 0; kk < KT; ++kk)
                if (!FIRST && (!GUARD || kk < K) && live && bt[kk] < GBMW_STEP_INF)
                    pcm |= src_path_change(a, sh, u, e, bp[kk]) << kk;
            const int s = 1 + tid;
#pragma unroll
            for (int kk = 0; kk < KT; ++kk)
                if (!GUARD || kk < K) { sh.et[s][kk] = bt[kk]; sh.ef[s][kk] = bf[kk]; sh.ep[s][kk] = bp[kk]; }
            sh.epc[s] = pcm;
        }
        __syncthreads();
        // ---- 4. write the round's groups: rows, change-bit words, flat-group bits
        for (int g = g0 + warp; g < g1; g += nwarp) {
            const int kd = sh.kind[g];
            if (kd == 0) continue;
            const int r0 = first_row + 32 * g;
            const int wi = w_first + g;
            // predecessor of the group's first row: the last entry before it (row r0 - 1)
            const int sp = sh.ebase[g] - E0;             // its slot (0 = carried from the previous round)
            const bool pred_ok = (g == 0) ? (sh.prev_ok != 0) : (sh.kind[g - 1] != 0);
            const int s0 = sh.ebase[g] - E0 + 1;
            if (kd == 1) {
#pragma unroll
                for (int kk = 0; kk < KT; ++kk) {
                    if (GUARD && kk >= K) break;
                    if (lane == kk) {
                        reinterpret_cast<double2 *>(bout)[(int64_t)kk * n_e + r0] =
                            make_double2(sh.et[s0][kk], sh.ef[s0][kk]);
                        pout[(int64_t)kk * n_e + r0] = (uint16_t)sh.idx[sh.ep[s0][kk]];
                        const bool same = pred_ok && sh.et[sp][kk] == sh.et[s0][kk] && sh.ef[sp][kk] == sh.ef[s0][kk] &&
                                          sh.ep[sp][kk] == sh.ep[s0][kk] && !((sh.epc[s0] >> kk) & 1u);
                        if (wi < sh.nw) fout[(int64_t)kk * sh.nw + wi] = same ? 0u : 1u;
                    }
                }
            } else {
                const unsigned segm = sh.seg[g];
                const int e = r0 + lane;
                const bool live = e >= lo && e <= hi;
                const int s = s0 + __popc(segm & ((2u << lane) - 2u));   // segment holding row e
                const bool start = lane > 0 && ((segm >> lane) & 1u);
#pragma unroll
                for (int kk = 0; kk < KT; ++kk) {
                    if (GUARD && kk >= K) break;
                    const double t = sh.et[s][kk], f = sh.ef[s][kk];
                    const int pp = sh.ep[s][kk];
                    if (live) {
                        reinterpret_cast<double2 *>(bout)[(int64_t)kk * n_e + e] = make_double2(t, f);
                        pout[(int64_t)kk * n_e + e] = (uint16_t)sh.idx[pp];
                    }
                    bool chg;
                    const int sq = (lane == 0) ? sp : s - 1;     // the row before e
                    const bool q_ok = (lane == 0) ? pred_ok : true;
                    if (lane > 0 && !start) {
                        chg = false;                             // no source changes: same row
                    } else {
                        chg = !(q_ok && sh.et[sq][kk] == t && sh.ef[sq][kk] == f && sh.ep[sq][kk] == pp &&
                                !((sh.epc[s] >> kk) & 1u));
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, chg);
                    if (lane == 0 && wi < sh.nw) fout[(int64_t)kk * sh.nw + wi] = m;
                }
            }
        }
        __syncthreads();
        // carry the round's last entry into slot 0 for the next round
        if (rd + 1 < n_rounds) {
            const int sl = E1 - E0;                      // slot of entry E1 - 1
            if (tid < KT && (!GUARD || tid < K)) {
                sh.et[0][tid] = sh.et[sl][tid]; sh.ef[0][tid] = sh.ef[sl][tid]; sh.ep[0][tid] = sh.ep[sl][tid];
            }
            if (tid == 0) sh.epc[0] = sh.epc[sl];
            __syncthreads();
        }
    }
    // ---- 5. dead groups' change words, flat-group mask words
    for (int x = tid; x < kGroups * K; x += nthr) {
        const int g = x / K, kk = x - g * K;
        const int wi = w_first + g;
        if (sh.kind[g] == 0 && wi < sh.nw) fout[(int64_t)kk * sh.nw + wi] = 0xffffffffu;   // never read as flat
    }
    if (tid < kGroups / 32) {
        unsigned m = 0u;
        for (int b = 0; b < 32; ++b) m |= (sh.kind[32 * tid + b] == 1 ? 1u : 0u) << b;
        const int wi = (first_row >> 10) + tid;
        if (wi < sh.gw) a.gflat[sh.gf_cur + wi] = m;
    }
    __syncthreads();
}

// Live-tile work lists of every K2 launch of the chunk (one CTA per launch): tiles of the
// rows [L_u, H_u] of each active problem, so K2 never fetches a dead tile.
__global__ void __launch_bounds__(1024) k_step_lists(ChunkArgs a) {
    __shared__ long long s_part[1024];
    const StepList sl = a.step_lists[blockIdx.x];
    const int tid = threadIdx.x;
    const int per = (sl.n + 1023) / 1024;
    const int x0 = sl.lo + min(sl.n, tid * per), x1 = sl.lo + min(sl.n, tid * per + per);
    long long cnt = 0;
    for (int x = x0; x < x1; ++x) {
        const DevProblem &p = a.probs[x];
        const int lo = a.unit_lo[p.ustate_off + sl.u], hi = a.unit_hi[p.ustate_off + sl.u];
        if (hi >= lo) cnt += (hi / kStepRows) - (lo / kStepRows) + 1;
    }
    s_part[tid] = cnt;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const long long v = (tid >= off) ? s_part[tid - off] : 0;
        __syncthreads();
        s_part[tid] += v;
        __syncthreads();
    }
    long long at = sl.base + s_part[tid] - cnt;
    for (int x = x0; x < x1; ++x) {
        const DevProblem &p = a.probs[x];
        const int lo = a.unit_lo[p.ustate_off + sl.u], hi = a.unit_hi[p.ustate_off + sl.u];
        if (hi < lo) continue;
        for (int t = lo / kStepRows; t <= hi / kStepRows; ++t) a.step_items[at++] = make_int4(x, t, lo, hi);
    }
    if (tid == 1023) a.step_count[blockIdx.x] = s_part[1023];
}

int launch_step_lists(const ChunkArgs &a, void *stream) {
    if (a.n_step_lists <= 0) return 0;
    k_step_lists<<<a.n_step_lists, 1024, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

template <int GROUP, bool FIRST>
__global__ void __launch_bounds__(kStepThreads, GROUP == 0 ? 3 : 2) k_dp_step(ChunkArgs a, int u, const int4 *items,
                                                                              const int64_t *count,
                                                                              unsigned long long *counter) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using SH = StepShared<GROUP == 0 ? 4 : (GROUP == 1 ? 8 : kMaxClasses)>;
    SH &sh = *reinterpret_cast<SH *>(smem_raw);
    int q_prev = -1;
    if (threadIdx.x == 0) sh.stat_rows = 0;
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
        const int64_t first_row = (int64_t)item.y * kStepRows;
        const int lo = item.z, hi = item.w;
        if (q != q_prev) {
            __syncthreads();
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
            if (!FIRST) {
                const int gw = (int)gflat_words(p.n_b + 1);
                const uint32_t *gsrc = a.gflat + p.gflat_off + (int64_t)(u - 2) * gw;
                for (int x = threadIdx.x; x < gw; x += blockDim.x) sh.gfp[x] = gsrc[x];
            }
            if (threadIdx.x == 0) {
                sh.S = nu; sh.K = K; sh.n_e = (int)(p.n_b + 1); sh.q = q;
                sh.lo_prev = a.unit_lo[p.ustate_off + u - 1];
                sh.lo = lo; sh.hi = hi;
                sh.b_off = p.b_off; sh.par_off = p.par_off;
                sh.f_off = p.flag_off; sh.nw = (int)flag_words(p.n_b + 1);
                sh.gw = (int)gflat_words(p.n_b + 1);
                sh.gf_cur = p.gflat_off + (int64_t)(u - 1) * sh.gw;
            }
            __syncthreads();
            q_prev = q;
        }
        const int K = sh.K;
        if (GROUP == 0) {
            switch (K) {
                case 1: step_tile<1, FIRST, false>(a, sh, u, (int)first_row); break;
                case 2: step_tile<2, FIRST, false>(a, sh, u, (int)first_row); break;
                case 3: step_tile<3, FIRST, false>(a, sh, u, (int)first_row); break;
                default: step_tile<4, FIRST, false>(a, sh, u, (int)first_row); break;
            }
        } else if (GROUP == 1) {
            switch (K) {
                case 5: step_tile<5, FIRST, false>(a, sh, u, (int)first_row); break;
                case 6: step_tile<6, FIRST, false>(a, sh, u, (int)first_row); break;
                case 7: step_tile<7, FIRST, false>(a, sh, u, (int)first_row); break;
                default: step_tile<8, FIRST, false>(a, sh, u, (int)first_row); break;
            }
        } else {
            step_tile<kMaxClasses, FIRST, true>(a, sh, u, (int)first_row);
        }
    }
    if (threadIdx.x == 0 && sh.stat_rows) atomicAdd(a.computed_cells, sh.stat_rows);
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
