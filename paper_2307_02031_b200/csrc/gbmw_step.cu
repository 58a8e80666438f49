// gbmw_step.cu — K2, the min-plus layer step of the stage search, breakpoint-driven.
//
// Reference step (dpsearch.py:261-280), restated per source row e' and target class k
// (DESIGN.md §3):
//   B_u[e',k] = lexmin_i (T_{u-1}[e',i] + R_u[cls i, k], F_{u-1}[e',i], i),
//   T_{u-1}[e',i] = B_{u-1}[e'-w_{u-1,i}, cls i].t + time_c[u-1,i]   (init row for u == 1).
// B is a step function of e' with few steps.  Row e' of B_u can differ from row e'-1 only
// where some source T_{u-1}[., i] changes between them — a "breakpoint": a change bit of
// column cls(i) of B_{u-1} at row e' - w_{u-1,i} (or the row where the source turns
// finite).  K2 evaluates B_u only at the breakpoints (plus the first live row of every
// 1024-row tile), and stores a row only where some column actually changes (value, argmin,
// or the path behind the argmin) or where a tile starts: the "stored rows".  Every reader
// maps a row to the stored row at or before it through the unit's row map (stored_row).
// Outputs per step: the per-column change bits of B_u (bit x: row x differs from row
// x-1, exact up to spurious 1 bits at tile starts, which only cost work downstream), the
// row map, and (t, f, argmin) at the stored rows.  Tie-break T1 (lexicographic
// (cand, F, i), first i) is the reference's for every row.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gbmw_internal.h"

namespace gbmw {

#define GBMW_STEP_INF __longlong_as_double(0x7ff0000000000000LL)

constexpr int kClassifyIB = 8;              // window checks per thread in flight
constexpr int kStepIB = 4;                  // sources per lane in flight (lane-per-row evaluation)
constexpr int kStepItemTarget = 1200;       // K2 items per launch worth splitting tiles for (~4 per CTA)
constexpr int kWarpRows = 1024;             // rows per warp tile: 32 groups of 32

// Scratch of one warp tile of the item: its entries (rows to evaluate) in row order.
struct TileScratch {
    uint16_t erow[kWarpRows + 1];           // row of each entry, relative to the row before the tile
    uint16_t echg[kWarpRows + 1];           // bit kk: column kk changes at the entry's row
};

constexpr int kItemWarps = kStepThreads / 32;
static_assert(kItemTiles <= kItemWarps, "one warp classifies each tile of an item");

// KM: class capacity of the instantiation (4 / 8 / kMaxClasses)
template <int KM>
struct StepShared {
    Cell cell[kMaxStrats];                  // distinct source strategies of unit u-1 (ascending)
    int idx[kMaxStrats];                    // their strategy index
    double r[KM * KM];
    int S, K, n_e, lo_prev, lo, hi, nw;
    int64_t b_off, par_off, f_off;
    int64_t rm_prev, rm_cur;                // row maps of B_{u-1} and B_u (offsets into a.rmap)
    int64_t next;
    int t0, nt;                             // the item's warp tiles [t0, t0 + nt)
    int n_ent[kItemTiles];                  // entries per tile
    int first_bp[kItemTiles];               // the tile's first live row is a breakpoint
    int rpre[kItemTiles + 1];               // evaluation rounds before tile t
    int rnext;                              // round counter
    uint32_t gseg[kItemTiles * 32];         // breakpoints of each 32-row group of the item
    int pre[kItemTiles];                    // entry 0 of a later tile: the row before its first breakpoint
    int tlast[kItemTiles];                  // last stored row of each tile (-1: none)
    int na[kItemTiles];                     // sources with a change inside each tile's window
    uint16_t alist[kItemTiles][kMaxStrats]; // ... their positions in the distinct list
    TileScratch tile[kItemTiles];
};

// lexicographic (t, f, key) order; key = 2 * position in the distinct list + path bit, so
// comparing keys compares positions (T1: first i among equal (cand, F))
__device__ __forceinline__ bool lex3_less(double t1, double f1, int k1, double t2, double f2, int k2) {
    return t1 < t2 || (t1 == t2 && (f1 < f2 || (f1 == f2 && k1 < k2)));
}

// K lexmins of row e of B_u by a segment of L lanes (L = 1, 2, 4, ..., 32; lane offset
// l in the segment takes the distinct sources l, l + L, ...); a butterfly inside the
// segment leaves the result in each of its lanes.  e < 0: no row (+inf).
// key = 2 * argmin position + (1 if the argmin's source row is a change point of its
// column of B_{u-1}: the path behind the argmin changes there).
template <int KT, bool FIRST, bool GUARD, class SH>
__device__ __forceinline__ void eval_row(const ChunkArgs &a, const SH &sh, int u, int e, int L, int l,
                                         double *bt, double *bf, int *bk) {
    const int S = sh.S, K = GUARD ? sh.K : KT;
    const int n_e = sh.n_e, lo_prev = FIRST ? 0 : sh.lo_prev;
    const TFCell *bin = a.TF[(u - 1) & 1] + sh.b_off;
    const int2 *rm = a.rmap + sh.rm_prev;
    const uint32_t *fin = a.chg[(u - 1) & 1] + sh.f_off;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) { bt[kk] = GBMW_STEP_INF; bf[kk] = GBMW_STEP_INF; bk[kk] = 0x7fffffff; }
    for (int i0 = l; i0 < S; i0 += kStepIB * L) {
        double T[kStepIB], F[kStepIB];
        int key[kStepIB], src_[kStepIB], k_[kStepIB];
        bool ok[kStepIB];
        int2 m[kStepIB];
        uint32_t cw[kStepIB];
#pragma unroll
        for (int b = 0; b < kStepIB; ++b) {
            const int i = i0 + b * L;
            const Cell c = sh.cell[i < S ? i : 0];
            const int src = e - c.w;
            src_[b] = src; k_[b] = c.k;
            ok[b] = i < S && e >= 0 && src >= lo_prev;
            T[b] = GBMW_STEP_INF; F[b] = GBMW_STEP_INF; key[b] = 2 * i;
            if (!FIRST && ok[b]) {
                m[b] = __ldg(rm + (src >> 5));
                cw[b] = __ldg(fin + (int64_t)c.k * sh.nw + (src >> 5));
            }
        }
#pragma unroll
        for (int b = 0; b < kStepIB; ++b) {
            if (!ok[b]) continue;
            const Cell c = sh.cell[i0 + b * L];
            if (FIRST) {                       // init row, dpsearch.py:255-259
                T[b] = c.c; F[b] = c.ef;
            } else {
                const int row = stored_row(m[b], src_[b]);
                const double2 v = __ldg(reinterpret_cast<const double2 *>(bin + (int64_t)k_[b] * n_e + row));
                T[b] = v.x + c.c;
                F[b] = v.y + c.ef;
                key[b] |= (int)((cw[b] >> (src_[b] & 31)) & 1u);
            }
        }
#pragma unroll
        for (int b = 0; b < kStepIB; ++b) {
            if (i0 + b * L >= S) break;
            const double *rrow = sh.r + k_[b] * K;
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
                if (!GUARD || kk < K) {
                    const double cand = T[b] + rrow[kk];
                    const bool better = lex3_less(cand, F[b], key[b], bt[kk], bf[kk], bk[kk]);
                    bt[kk] = better ? cand : bt[kk];
                    bf[kk] = better ? F[b] : bf[kk];
                    bk[kk] = better ? key[b] : bk[kk];
                }
            }
        }
    }
    for (int off = L >> 1; off > 0; off >>= 1) {
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) {
            if (GUARD && kk >= K) break;
            const double ot = __shfl_xor_sync(0xffffffffu, bt[kk], off);
            const double of = __shfl_xor_sync(0xffffffffu, bf[kk], off);
            const int ok2 = __shfl_xor_sync(0xffffffffu, bk[kk], off);
            if (lex3_less(ot, of, ok2, bt[kk], bf[kk], bk[kk])) { bt[kk] = ot; bf[kk] = of; bk[kk] = ok2; }
        }
    }
}

// Breakpoints of a 32-row group contributed by one source: rows x (0..31) where the
// source's value T_{u-1}[r0 + x, i] may differ from row r0 + x - 1, i.e. the change bits of
// its window [x0, x0 + 31] of column cls(i) (rows below lo are +inf and constant).
__device__ __forceinline__ unsigned window_segments(unsigned long long v, int x0, int lo) {
    unsigned m = (unsigned)v;                            // bit j: row x0 + j vs x0 + j - 1
    if (x0 < lo) {
        const int j0 = lo - x0;                          // first finite row of the window
        m = (m & ~((2u << j0) - 1u)) | (1u << j0);
    }
    return m;
}

// Phase A0, one warp per tile: the sources whose window over the tile holds a change of
// their column of B_{u-1} (change summaries, 1 bit per 32 rows) or the column's first
// finite row; the others contribute no breakpoint anywhere in the tile.
template <bool FIRST, class SH>
__device__ __forceinline__ void tile_sources(const ChunkArgs &a, SH &sh, int u, int ti, int lane) {
    const int S = sh.S, lo_prev = sh.lo_prev;
    const int r_base = (sh.t0 + ti) * kWarpRows;
    const int ns = (int)sum_words(sh.n_e);
    const uint32_t *sum = a.chg[(u - 1) & 1] + sh.f_off + (int64_t)sh.K * sh.nw;
    int cnt = 0;
    for (int n0 = 0; n0 < S; n0 += 32) {
        const int n = n0 + lane;
        bool act = false;
        if (n < S) {
            const Cell c = sh.cell[n];
            const int A = r_base - c.w, B = A + kWarpRows - 1;     // source rows of the tile's windows
            if (FIRST) {
                act = c.w >= r_base && c.w < r_base + kWarpRows;    // T_0[., i] turns finite at w_i
            } else if (B >= lo_prev) {
                act = lo_prev >= A;                                 // the column's first finite row
                if (!act) {
                    const int ga = A >> 5, gb = B >> 5;             // 32-row groups [ga, gb]
                    const uint32_t *sk = sum + (int64_t)c.k * ns;
                    const uint32_t w0 = __ldg(sk + (ga >> 5)), w1 = __ldg(sk + (gb >> 5));
                    const uint32_t m0 = w0 & (0xffffffffu << (ga & 31));
                    const uint32_t m1 = w1 & (0xffffffffu >> (31 - (gb & 31)));
                    act = ((ga >> 5) == (gb >> 5)) ? (m0 & m1) != 0u : (m0 | m1) != 0u;
                }
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, act);
        if (act) sh.alist[ti][cnt + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)n;
        cnt += __popc(bal);
    }
    if (lane == 0) sh.na[ti] = cnt;
}

// Phase A1, all threads: the breakpoints of every 32-row group of the item's tiles
// (change bits of the tile's active source windows).
template <bool FIRST, class SH>
__device__ __forceinline__ void group_breakpoints(const ChunkArgs &a, SH &sh, int u, int tid) {
    // thread tid: group gi = tid / tpg of the item, active sources sub, sub + tpg, ... (the
    // CTA's threads spread over the item's nt * 32 groups whatever nt is)
    const int ng = sh.nt * 32;
    int tpg = kStepThreads / ng;
    tpg = tpg >= 8 ? 8 : (tpg >= 4 ? 4 : (tpg >= 2 ? 2 : 1));
    const int gi = tid / tpg, sub = tid - gi * tpg;
    const int lo = sh.lo, hi = sh.hi;
    const int r0 = (sh.t0 + (gi >> 5)) * kWarpRows + 32 * (gi & 31), r1 = r0 + 31;
    const bool act = gi < ng;
    const bool dead = !act || r1 < lo || r0 > hi;
    const bool whole = act && r0 >= lo && r1 <= hi;
    const int NA = act ? sh.na[gi >> 5] : 0;
    const uint16_t *al = sh.alist[act ? gi >> 5 : 0];
    unsigned seg = 0u;
    if (whole) {
        const uint32_t *fin = a.chg[(u - 1) & 1] + sh.f_off;
        for (int n0 = sub; n0 < NA; n0 += kClassifyIB * tpg) {
            uint32_t w0[kClassifyIB], w1[kClassifyIB];
            int xs_[kClassifyIB];
            bool ld[kClassifyIB];
#pragma unroll
            for (int b = 0; b < kClassifyIB; ++b) {
                const int n = n0 + b * tpg;
                const Cell c = sh.cell[n < NA ? al[n] : 0];
                const int xs = r0 - c.w;
                xs_[b] = xs; w0[b] = 0u; w1[b] = 0u;
                ld[b] = n < NA && (FIRST || xs + 31 >= sh.lo_prev);
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
                    seg |= (j >= 0 && j <= 31) ? (1u << j) : 0u;
                } else {
                    const int xl = xs < 0 ? 0 : xs;
                    const unsigned long long v =
                        ((unsigned long long)w1[b] << 32 | (unsigned long long)w0[b]) >> (xl & 31);
                    seg |= window_segments((xs < 0) ? (v << (-xs)) : v, xs, sh.lo_prev);
                }
            }
        }
    } else if (!dead) {                                  // partial group: every live row
        const int a0 = lo > r0 ? lo - r0 : 0, a1 = hi < r1 ? hi - r0 : 31;
        seg = (0xffffffffu >> (31 - a1)) & ~((1u << a0) - 1u);
    }
    for (int off = tpg >> 1; off > 0; off >>= 1) seg |= __shfl_xor_sync(0xffffffffu, seg, off);
    if (act && sub == 0) sh.gseg[gi] = seg;
}

// Phase A2, one warp per tile (kWarpRows rows of B_u), lane g owns 32-row group g: the
// breakpoints of the groups become the tile's entries (rows relative to the row before the
// tile).  The item's first tile always has its first live row as entry 0 (the anchor of the
// row map, stored); a later tile with breakpoints gets the row before its first one as
// entry 0 (evaluated for the comparison only, never stored).
template <class SH>
__device__ __forceinline__ void classify_tile(SH &sh, int ti, int lane) {
    const int lo = sh.lo, hi = sh.hi;
    const int r_base = (sh.t0 + ti) * kWarpRows;
    const int g = lane, r0 = r_base + 32 * g, r1 = r0 + 31;
    const bool dead = r1 < lo || r0 > hi;
    const int f0 = r_base > lo ? r_base : lo;            // first live row of the tile (<= hi)
    unsigned seg = sh.gseg[ti * 32 + g];
    bool fbp = false;
    if (ti == 0) {                                       // anchor: change bits exact unless a breakpoint
        fbp = __shfl_sync(0xffffffffu, (seg >> ((f0 - r_base) & 31)) & 1u, (f0 - r_base) >> 5) != 0u;
        if (!dead && f0 >= r0 && f0 <= r1) seg |= 1u << (f0 - r0);
    }
    const int cnt = __popc(seg);
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int pre = (ti > 0 && total > 0) ? 1 : 0;
    int at = pre + incl - cnt;
    TileScratch &w = sh.tile[ti];
    unsigned m = seg;
    bool first = pre && incl == cnt && cnt > 0;          // this lane holds the tile's first breakpoint
    while (m) {
        const int x = __ffs(m) - 1;
        m &= m - 1u;
        if (first) { w.erow[0] = (uint16_t)(32 * g + x); first = false; }   // its row - 1 (relative + 1)
        w.erow[at++] = (uint16_t)(32 * g + x + 1);
    }
    if (lane == 31) {
        sh.n_ent[ti] = total + pre; sh.pre[ti] = pre;
        sh.first_bp[ti] = (f0 == lo || fbp) ? 1 : 0;
    }
}

// evaluation rounds of a tile with n entries: one round of up to 32 entries (a segment of
// 32 / next_pow2(n) lanes per entry), then rounds of 31 new entries, a lane each (lane 0
// re-evaluates the previous entry for the comparison)
__device__ __forceinline__ int tile_rounds(int n) { return n <= 32 ? 1 : 1 + (n - 32 + 30) / 31; }

// Phase B, one round of one tile by one warp: evaluate its entries, compare each with the
// previous entry (unchanged columns keep change bit 0), store (t, f, argmin) of the
// entries where some column changes (and of the tile's first entry, the anchor).
template <int KT, bool FIRST, bool GUARD, class SH>
__device__ __forceinline__ void eval_round(const ChunkArgs &a, SH &sh, int u, int ti, int r, int lane) {
    const int K = GUARD ? sh.K : KT;
    const int n_e = sh.n_e, n = sh.n_ent[ti];
    const int r_base = (sh.t0 + ti) * kWarpRows;
    TileScratch &w = sh.tile[ti];
    int L, j0, nr;                                       // lanes per entry, first entry, entries
    if (r == 0) {
        nr = n < 32 ? n : 32;
        L = 32;
        while (L > 1 && (32 / L) < nr) L >>= 1;
        j0 = 0;
    } else {
        L = 1;
        j0 = 31 * r;                                     // = (first new entry) - 1
        nr = min(32, n - j0);
    }
    const int seg = lane / L, l = lane - seg * L;
    const int j = j0 + seg;
    const bool have = seg < nr;
    const int e = have ? r_base - 1 + (int)w.erow[j] : -1;
    double bt[KT], bf[KT];
    int bk[KT];
    eval_row<KT, FIRST, GUARD>(a, sh, u, e, L, l, bt, bf, bk);
    unsigned chg = 0u;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
        if (GUARD && kk >= K) break;
        const double pt = __shfl_up_sync(0xffffffffu, bt[kk], L);
        const double pf = __shfl_up_sync(0xffffffffu, bf[kk], L);
        const int pk = __shfl_up_sync(0xffffffffu, bk[kk], L);
        const bool same = bt[kk] == pt && bf[kk] == pf && (bk[kk] >> 1) == (pk >> 1) && !(bk[kk] & 1);
        chg |= same ? 0u : (1u << kk);
    }
    const bool pre = sh.pre[ti] != 0;
    if (j == 0) chg = (!pre && sh.first_bp[ti]) ? 0xffffu : 0u;
    chg &= (1u << K) - 1u;
    // lane 0 of a later round: the previous entry; entry 0 of a later tile: comparison only
    const bool out = have && l == 0 && (r == 0 || seg > 0) && !(j == 0 && pre);
    if (out) {
        if (j == 0 || chg) {
            TFCell *bout = a.TF[u & 1] + sh.b_off;
            uint16_t *pout = a.par + sh.par_off + (int64_t)(u - 1) * K * n_e;
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
                if (GUARD && kk >= K) break;
                reinterpret_cast<double2 *>(bout)[(int64_t)kk * n_e + e] = make_double2(bt[kk], bf[kk]);
                pout[(int64_t)kk * n_e + e] = (uint16_t)sh.idx[bk[kk] >> 1];
            }
        }
        w.echg[j] = (uint16_t)chg;
    }
}

// Phase C, one warp per tile, lane g: the change-bit words and the row-map entry of group g.
// entries of group g of a tile: [b0, b1) (binary search; entry 0 of a later tile is the
// comparison row, skipped)
template <class SH>
__device__ __forceinline__ void group_entries(const SH &sh, int ti, int g, int &b0, int &b1) {
    const TileScratch &w = sh.tile[ti];
    const int n = sh.n_ent[ti];
    int x0 = sh.pre[ti], x1 = n;
    while (x0 < x1) {
        const int mid = (x0 + x1) >> 1;
        if ((int)w.erow[mid] < 32 * g + 1) x0 = mid + 1; else x1 = mid;
    }
    b0 = x0;
    b1 = b0;
    while (b1 < n && (int)w.erow[b1] < 32 * g + 33) ++b1;
}

__device__ __forceinline__ bool entry_stored(int j, unsigned m, bool pre) { return m != 0u || (j == 0 && !pre); }

// Phase C1, one warp per tile: the tile's last stored row (the row-map carry of later tiles).
template <class SH>
__device__ __forceinline__ void tile_last(SH &sh, int ti, int lane) {
    const int r_base = (sh.t0 + ti) * kWarpRows;
    const TileScratch &w = sh.tile[ti];
    const bool pre = sh.pre[ti] != 0;
    int last = -1;
    for (int j = lane; j < sh.n_ent[ti]; j += 32)
        if (!(j == 0 && pre) && entry_stored(j, w.echg[j], pre)) last = r_base - 1 + (int)w.erow[j];
    for (int off = 16; off > 0; off >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, off));
    if (lane == 0) sh.tlast[ti] = last;
}

// Phase C2, one warp per tile, lane g: the change-bit words and the row-map entry of group g,
// and the tile's change-summary word per column.
template <int KT, bool GUARD, class SH>
__device__ __forceinline__ void finish_tile(const ChunkArgs &a, const SH &sh, int u, int ti, int lane) {
    const int K = GUARD ? sh.K : KT;
    const int lo = sh.lo, hi = sh.hi, n = sh.n_ent[ti];
    const int r_base = (sh.t0 + ti) * kWarpRows;
    const int g = lane, r0 = r_base + 32 * g, r1 = r0 + 31;
    const bool dead = r1 < lo || r0 > hi;
    const bool pre = sh.pre[ti] != 0;
    const TileScratch &w = sh.tile[ti];
    int b0, b1;
    group_entries(sh, ti, g, b0, b1);
    int last = -1;                                       // last stored row of the group
    unsigned sbits = 0u;
    uint32_t cwd[KT];
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) cwd[kk] = 0u;
    for (int x0 = b0; x0 < b1; ++x0) {
        const int x = ((int)w.erow[x0] - 1) & 31;
        const unsigned m = w.echg[x0];
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) cwd[kk] |= ((m >> kk) & 1u) << x;
        if (entry_stored(x0, m, pre)) { sbits |= 1u << x; last = r_base - 1 + (int)w.erow[x0]; }
    }
    int carry = -1;                                      // stored rows of the item's earlier tiles
    for (int t = 0; t < ti; ++t) carry = max(carry, sh.tlast[t]);
    int before = last;                                   // exclusive max-scan over the groups
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, before, off);
        if (lane >= off) before = max(before, v);
    }
    before = __shfl_up_sync(0xffffffffu, before, 1);
    if (lane == 0) before = -1;
    before = max(before, carry);
    const int ns = (int)sum_words(sh.n_e);
    uint32_t *fout = a.chg[u & 1] + sh.f_off;
    uint32_t *sout = fout + (int64_t)K * sh.nw;
    const int wi = (r_base >> 5) + g;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
        if (GUARD && kk >= K) break;
        if (!dead) fout[(int64_t)kk * sh.nw + wi] = cwd[kk];
        const unsigned sm = __ballot_sync(0xffffffffu, cwd[kk] != 0u);
        if (lane == 0) sout[(int64_t)kk * ns + (r_base >> 10)] = sm;
    }
    if (!dead) a.rmap[sh.rm_cur + wi] = make_int2((int)sbits, before);
    if (a.k2_hist && lane == 0) {
        const int bin = 32 - __clz(n);
        atomicAdd(a.k2_hist + bin, 1ull);
        atomicAdd(a.k2_hist + 32 + bin, (unsigned long long)n);
    }
}

// Live-row work lists of every K2 launch of the chunk (one CTA per launch): per active
// problem with live rows, its warp tiles [L_u / kWarpRows, H_u / kWarpRows] in items of
// at most kItemTiles tiles (a large problem spreads over many CTAs).
__global__ void __launch_bounds__(1024) k_step_lists(ChunkArgs a) {
    __shared__ int s_part[1024];
    __shared__ int s_it;
    const StepList sl = a.step_lists[blockIdx.x];
    const int tid = threadIdx.x;
    const int per = (sl.n + 1023) / 1024;
    const int x0 = sl.lo + min(sl.n, tid * per), x1 = sl.lo + min(sl.n, tid * per + per);
    // item size: kItemTiles, smaller when the launch has few tiles (>= kStepItemTarget items)
    int tiles = 0;
    for (int x = x0; x < x1; ++x) {
        const DevProblem &p = a.probs[x];
        const int lo = a.unit_lo[p.ustate_off + sl.u], hi = a.unit_hi[p.ustate_off + sl.u];
        if (hi >= lo) tiles += hi / kWarpRows - lo / kWarpRows + 1;
    }
    s_part[tid] = tiles;
    __syncthreads();
    for (int off = 512; off > 0; off >>= 1) {
        if (tid < off) s_part[tid] += s_part[tid + off];
        __syncthreads();
    }
    if (tid == 0) s_it = max(1, min(kItemTiles, s_part[0] / kStepItemTarget));
    __syncthreads();
    const int it = s_it;
    int cnt = 0;
    for (int x = x0; x < x1; ++x) {
        const DevProblem &p = a.probs[x];
        const int lo = a.unit_lo[p.ustate_off + sl.u], hi = a.unit_hi[p.ustate_off + sl.u];
        if (hi >= lo) cnt += (hi / kWarpRows - lo / kWarpRows) / it + 1;
    }
    __syncthreads();
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
        const int t1 = hi / kWarpRows;
        for (int t0 = lo / kWarpRows; t0 <= t1; t0 += it)
            a.step_items[at++] = make_int4(x, t0, min(t1, t0 + it - 1), 0);
    }
    if (tid == 1023) a.step_count[blockIdx.x] = s_part[1023];
}

int launch_step_lists(const ChunkArgs &a, void *stream) {
    if (a.n_step_lists <= 0) return 0;
    k_step_lists<<<a.n_step_lists, 1024, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

// CTAs take items (dynamic counter) of up to kItemTiles warp tiles of one problem:
// classify the tiles (a warp each), evaluate all their entries in rounds shared by the
// CTA's warps (heaviest tiles first), then write each tile's change bits and row map.
#define GBMW_K2_DISPATCH(CALL)                                                       \
    if (GROUP == 0) {                                                                \
        switch (K) {                                                                 \
            case 1: CALL(1, false); break;                                           \
            case 2: CALL(2, false); break;                                           \
            case 3: CALL(3, false); break;                                           \
            default: CALL(4, false); break;                                          \
        }                                                                            \
    } else if (GROUP == 1) {                                                         \
        switch (K) {                                                                 \
            case 5: CALL(5, false); break;                                           \
            case 6: CALL(6, false); break;                                           \
            case 7: CALL(7, false); break;                                           \
            default: CALL(8, false); break;                                          \
        }                                                                            \
    } else {                                                                         \
        CALL(kMaxClasses, true);                                                     \
    }

template <int GROUP, bool FIRST>
__global__ void __launch_bounds__(kStepThreads, GROUP <= 1 ? 3 : 1)
    k_dp_step(ChunkArgs a, int u, const int4 *items, const int64_t *count, unsigned long long *counter) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using SH = StepShared<GROUP == 0 ? 4 : (GROUP == 1 ? 8 : kMaxClasses)>;
    SH &sh = *reinterpret_cast<SH *>(smem_raw);
    __shared__ int s_order[kItemTiles];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
            if (threadIdx.x == 0) {
                const int64_t ng = rmap_groups(p.n_b + 1);
                sh.S = nu; sh.K = K; sh.n_e = (int)(p.n_b + 1);
                sh.lo_prev = a.unit_lo[p.ustate_off + u - 1];
                sh.lo = a.unit_lo[p.ustate_off + u]; sh.hi = a.unit_hi[p.ustate_off + u];
                sh.b_off = p.b_off; sh.par_off = p.par_off;
                sh.f_off = p.flag_off; sh.nw = (int)flag_words(p.n_b + 1);
                sh.rm_prev = p.rmap_off + (int64_t)(u >= 2 ? u - 2 : 0) * ng;
                sh.rm_cur = p.rmap_off + (int64_t)(u - 1) * ng;
                sh.t0 = item.y; sh.nt = item.z - item.y + 1;
            }
        }
        __syncthreads();
        const int K = sh.K, nt = sh.nt;
        if (warp < nt) tile_sources<FIRST>(a, sh, u, warp, lane);
        __syncthreads();
        group_breakpoints<FIRST>(a, sh, u, threadIdx.x);
        __syncthreads();
        if (warp < nt) classify_tile(sh, warp, lane);
        __syncthreads();
        if (threadIdx.x == 0) {
            // rounds of the heaviest tiles first
            for (int x = 0; x < nt; ++x) {
                int y = x;
                while (y > 0 && sh.n_ent[s_order[y - 1]] < sh.n_ent[x]) { s_order[y] = s_order[y - 1]; --y; }
                s_order[y] = x;
            }
            sh.rpre[0] = 0;
            for (int x = 0; x < nt; ++x) sh.rpre[x + 1] = sh.rpre[x] + tile_rounds(sh.n_ent[s_order[x]]);
            sh.rnext = 0;
        }
        __syncthreads();
        const int total = sh.rpre[nt];
        while (true) {
            int R = 0;
            if (lane == 0) R = atomicAdd(&sh.rnext, 1);
            R = __shfl_sync(0xffffffffu, R, 0);
            if (R >= total) break;
            int x = 0;
            while (x + 1 < nt && sh.rpre[x + 1] <= R) ++x;
            const int ti = s_order[x], r = R - sh.rpre[x];
#define GBMW_K2_EVAL(KT, G) eval_round<KT, FIRST, G>(a, sh, u, ti, r, lane)
            GBMW_K2_DISPATCH(GBMW_K2_EVAL)
#undef GBMW_K2_EVAL
        }
        __syncthreads();
        if (warp < nt) tile_last(sh, warp, lane);
        __syncthreads();
        if (warp < nt) {
#define GBMW_K2_FINISH(KT, G) finish_tile<KT, G>(a, sh, u, warp, lane)
            GBMW_K2_DISPATCH(GBMW_K2_FINISH)
#undef GBMW_K2_FINISH
            stat_rows += (unsigned long long)sh.n_ent[warp] * (unsigned long long)K;
        }
    }
    if (lane == 0 && stat_rows) atomicAdd(a.computed_cells, stat_rows);
}
#undef GBMW_K2_DISPATCH

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
