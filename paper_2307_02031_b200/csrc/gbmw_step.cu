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

// KM: class capacity of the instantiation (4 / 8 / kMaxClasses), sizes the per-group arrays
template <int KM>
struct StepShared {
    Cell cell[kMaxStrats];                  // distinct source strategies of unit u-1 (ascending)
    int idx[kMaxStrats];                    // their strategy index
    double r[KM * KM];
    uint32_t gfp[kMaxGfWords];              // flat-group mask of B_{u-1} (read redirection, flat_row)
    int S, K, n_e, q, lo_prev, lo, hi, nw;
    int64_t b_off, par_off, tile0, f_off;
    int64_t gf_cur;                         // flat-group mask of B_u (offset into a.gflat)
    int gw;
    int64_t next;
    int4 item;
    // per tile
    int kind[kGroups];                      // 0 dead, 1 flat, 2 full
    int list_np[kGroups], list_fl[kGroups];
    int n_np, n_fl;
    unsigned bits[kGroups][KM];
    double first_t[kGroups][KM], first_f[kGroups][KM];
    double last_t[kGroups][KM], last_f[kGroups][KM];
    int first_p[kGroups][KM], last_p[kGroups][KM];
    unsigned first_pc[kGroups];             // bit kk: the first row's path differs below its argmin
    int prev_p[KM];
    double prev_t[KM], prev_f[KM];
    int prev_ok;
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

template <int KT, bool FIRST, bool GUARD, class SH>
__device__ void step_tile(const ChunkArgs &a, SH &sh, int u, int first_row) {
    const int K = GUARD ? sh.K : KT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
    const int n_e = sh.n_e, lo = sh.lo, hi = sh.hi, S = sh.S;
    // ---- 1. classify groups
    for (int g = tid; g < kGroups; g += nthr) {
        const int r0 = first_row + 32 * g, r1 = r0 + 31;
        sh.kind[g] = (r1 < lo || r0 > hi) ? 0 : ((r0 >= lo && r1 <= hi) ? 1 : 2);
    }
    __syncthreads();
    const uint32_t *fin = a.chg[(u - 1) & 1] + sh.f_off;
    // (group, source) window checks, kClassifyIB per thread in flight
    const int n_checks = kGroups * S;
    for (int x0 = tid; x0 < n_checks; x0 += nthr * kClassifyIB) {
        uint32_t w0[kClassifyIB], w1[kClassifyIB];
        int sh_[kClassifyIB], gg[kClassifyIB];
        bool load[kClassifyIB];
#pragma unroll
        for (int b = 0; b < kClassifyIB; ++b) {
            const int x = x0 + b * nthr;
            gg[b] = -1; load[b] = false; sh_[b] = 0;
            w0[b] = 0u; w1[b] = 0u;
            if (x < n_checks) {
                const int g = x / S, n = x - g * S;
                if (sh.kind[g] == 1) {
                    const Cell c = sh.cell[n];
                    const int r0 = first_row + 32 * g;
                    if (FIRST) {
                        if (!((r0 >= c.w) || (r0 + 31 < c.w))) gg[b] = g;
                    } else {
                        const int xs = r0 - c.w;
                        if (xs + 31 < sh.lo_prev) {
                            // all +inf: flat
                        } else if (xs < sh.lo_prev) {
                            gg[b] = g;
                        } else {
                            const int lb = xs + 1;
                            const uint32_t *fl = fin + (int64_t)c.k * sh.nw + (lb >> 5);
                            w0[b] = __ldg(fl); w1[b] = __ldg(fl + 1);
                            sh_[b] = lb & 31;
                            load[b] = true;
                            gg[b] = g;
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int b = 0; b < kClassifyIB; ++b) {
            if (gg[b] < 0) continue;
            bool flat = false;
            if (load[b]) {
                const unsigned long long v = ((unsigned long long)w1[b] << 32 | (unsigned long long)w0[b]) >> sh_[b];
                flat = (v & 0x7fffffffull) == 0ull;
            }
            if (!flat) sh.kind[gg[b]] = 2;
        }
    }
    __syncthreads();
    // ---- 2. row list: full groups (32 rows, one warp each), then flat representatives
    if (warp == 0) {
        int np = 0, nf = 0;
        for (int base = 0; base < kGroups; base += 32) {
            const int g = base + lane;
            const int kd = g < kGroups ? sh.kind[g] : 0;
            const unsigned mnp = __ballot_sync(0xffffffffu, kd == 2), mfl = __ballot_sync(0xffffffffu, kd == 1);
            const unsigned below = (1u << lane) - 1u;
            if (kd == 2) sh.list_np[np + __popc(mnp & below)] = g;
            if (kd == 1) sh.list_fl[nf + __popc(mfl & below)] = g;
            np += __popc(mnp);
            nf += __popc(mfl);
        }
        if (lane == 0) {
            sh.n_np = np;
            sh.n_fl = nf;
            sh.stat_rows += (unsigned long long)(32 * np + nf + 1) * (unsigned long long)K;
        }
    }
    __syncthreads();
    const int n_np = sh.n_np, n_fl = sh.n_fl;
    const int n_list = 32 * n_np + n_fl + 1;                // + the row before the tile
    TFCell *bout = a.TF[u & 1] + sh.b_off;
    uint16_t *pout = a.par + sh.par_off + (int64_t)(u - 1) * K * n_e;
    const int n_pass = (n_list + nthr - 1) / nthr;
    for (int pass = 0; pass < n_pass; ++pass) {
        const int x = pass * nthr + tid;
        double bt[KT], bf[KT];
        int bp[KT];
        int e = -1, kind = -1, g = -1;
        if (x < 32 * n_np) {
            g = sh.list_np[x >> 5]; e = first_row + 32 * g + lane; kind = 2;
        } else if (x < 32 * n_np + n_fl) {
            g = sh.list_fl[x - 32 * n_np]; e = first_row + 32 * g; kind = 1;
        } else if (x == 32 * n_np + n_fl) {
            e = first_row - 1; kind = 3;
        }
        const bool row_live = kind >= 0 && e >= lo && e <= hi && e < n_e;
        relax_row<KT, FIRST, GUARD>(a, sh, u, row_live ? e : -1, bt, bf, bp);
        // per class: source path-change bit (all loads issued before use)
        unsigned pcm = 0u;
#pragma unroll
        for (int kk = 0; kk < KT; ++kk)
            if (!FIRST && (!GUARD || kk < K) && row_live && bt[kk] < GBMW_STEP_INF)
                pcm |= src_path_change(a, sh, u, e, bp[kk]) << kk;
        // stored rows: live rows of full groups, the first row of flat groups
        if (row_live && (kind == 2 || kind == 1)) {
#pragma unroll
            for (int kk = 0; kk < KT; ++kk)
                if (!GUARD || kk < K) {
                    reinterpret_cast<double2 *>(bout)[kk * n_e + e] = make_double2(bt[kk], bf[kk]);
                    pout[kk * n_e + e] = (uint16_t)sh.idx[bp[kk]];
                }
        }
        // change bits inside full groups (a full group is exactly one warp of this pass)
        const bool in_np = (pass * nthr + warp * 32) < 32 * n_np;
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) {
            if (GUARD && kk >= K) break;
            if (in_np) {
                const double pt = __shfl_up_sync(0xffffffffu, bt[kk], 1);
                const double pf = __shfl_up_sync(0xffffffffu, bf[kk], 1);
                const int pp = __shfl_up_sync(0xffffffffu, bp[kk], 1);
                const bool chg = lane > 0 && (pt != bt[kk] || pf != bf[kk] || pp != bp[kk] || ((pcm >> kk) & 1u));
                const unsigned m = __ballot_sync(0xffffffffu, chg);
                if (lane == 0) {
                    sh.bits[g][kk] = m;
                    sh.first_t[g][kk] = bt[kk]; sh.first_f[g][kk] = bf[kk]; sh.first_p[g][kk] = bp[kk];
                }
                if (lane == 31) { sh.last_t[g][kk] = bt[kk]; sh.last_f[g][kk] = bf[kk]; sh.last_p[g][kk] = bp[kk]; }
            } else if (kind == 1) {
                sh.bits[g][kk] = 0u;
                sh.first_t[g][kk] = sh.last_t[g][kk] = bt[kk];
                sh.first_f[g][kk] = sh.last_f[g][kk] = bf[kk];
                sh.first_p[g][kk] = sh.last_p[g][kk] = bp[kk];
            } else if (kind == 3) {
                sh.prev_t[kk] = bt[kk];
                sh.prev_f[kk] = bf[kk];
                sh.prev_p[kk] = bp[kk];
            }
        }
        if ((in_np && lane == 0) || kind == 1) sh.first_pc[g] = pcm;
        if (kind == 3) sh.prev_ok = (e >= lo && e <= hi) ? 1 : 0;
    }
    __syncthreads();
    // ---- 3a. flat groups store their first row only (written above); readers redirect the
    // other rows to it through the group mask (flat_row)
    if (tid < kGroups / 32) {
        unsigned m = 0u;
        for (int b = 0; b < 32; ++b) m |= (sh.kind[32 * tid + b] == 1 ? 1u : 0u) << b;
        const int wi = (first_row >> 10) + tid;
        if (wi < sh.gw) a.gflat[sh.gf_cur + wi] = m;
    }
    // ---- 3b. change-bit words of B_u (bit 0 of a group compares with the previous row)
    uint32_t *fout = a.chg[u & 1] + sh.f_off;
    const int w_first = first_row >> 5;
    for (int x = tid; x < kGroups * K; x += nthr) {
        const int g = x / K, kk = x - g * K;
        const int wi = w_first + g;
        if (wi >= sh.nw) continue;
        unsigned word;
        if (sh.kind[g] == 0) {
            word = 0xffffffffu;                              // dead rows: never read as flat
        } else {
            word = sh.bits[g][kk];
            bool same;
            if (g == 0) same = sh.prev_ok && sh.prev_t[kk] == sh.first_t[0][kk] && sh.prev_f[kk] == sh.first_f[0][kk] &&
                               sh.prev_p[kk] == sh.first_p[0][kk];
            else same = sh.kind[g - 1] != 0 && sh.last_t[g - 1][kk] == sh.first_t[g][kk] &&
                        sh.last_f[g - 1][kk] == sh.first_f[g][kk] && sh.last_p[g - 1][kk] == sh.first_p[g][kk];
            same = same && !((sh.first_pc[g] >> kk) & 1u);
            if (!same) word |= 1u;
        }
        fout[(int64_t)kk * sh.nw + wi] = word;
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
    // thread 0 runs one item ahead: the next item's counter value and record are fetched
    // while the current tile is evaluated
    long long t_cur = 0, t_next = 0;
    int4 it_cur = make_int4(0, 0, 0, -1);
    if (threadIdx.x == 0) {
        t_cur = (long long)atomicAdd(counter, 1ull);
        if (t_cur < n_items) it_cur = __ldg(items + t_cur);
        t_next = (long long)atomicAdd(counter, 1ull);
    }
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) { sh.next = t_cur; sh.item = it_cur; }
        __syncthreads();
        if (sh.next >= n_items) break;
        const int4 item = sh.item;
        if (threadIdx.x == 0) {
            t_cur = t_next;
            if (t_cur < n_items) it_cur = __ldg(items + t_cur);
            t_next = (long long)atomicAdd(counter, 1ull);
        }
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
                sh.b_off = p.b_off; sh.par_off = p.par_off; sh.tile0 = a.step_tiles[q];
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
