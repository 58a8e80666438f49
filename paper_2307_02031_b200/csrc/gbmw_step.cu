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
//
// Two kernels per layer step, every warp independent (no CTA barrier):
//   K2a k_dp_classify: a warp per 1024-row tile classifies it, evaluates it when its entries
//       fit one round and writes its outputs; a heavier tile's entries go to global memory
//       and its rounds (32 entries each) to the launch's round list;
//   K2b k_dp_rounds: a warp per round of the heavy tiles; the warp finishing a tile's last
//       round writes the tile's change bits and row map.
// Outputs per step: the per-column change bits of B_u (bit x: row x differs from row
// x-1, exact up to spurious 1 bits at tile starts, which only cost work downstream), the
// row map, and (t, f, argmin) at the stored rows.  Tie-break T1 (lexicographic
// (cand, F, i), first i) is the reference's for every row.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "gbmw_internal.h"

namespace gbmw {

#define GBMW_STEP_INF __longlong_as_double(0x7ff0000000000000LL)

constexpr int kClassifyIB = 8;              // window checks per thread in flight
#ifndef GBMW_STEP_IB
#define GBMW_STEP_IB 2
#endif
#ifndef GBMW_STEP_IB_WIDE
#define GBMW_STEP_IB_WIDE 1
#endif
#ifndef GBMW_KEEP_CELL                      // 1: keep each source's (c, ef) in registers from its index
#define GBMW_KEEP_CELL 0                    // fetch (measured: 10k sweep +0.5 %, GPT-3-96 P=1 K2 -3 %)
#endif
constexpr int kStepIB = GBMW_STEP_IB;       // sources per lane in flight (lane-per-row evaluation), K <= 4
constexpr int kStepIBWide = GBMW_STEP_IB_WIDE;   // the same for K >= 5
constexpr int kWarpRows = 1024;             // rows per warp tile: 32 groups of 32
constexpr int kK2Warps = kStepThreads / 32;

// One tile and its problem, as one warp sees it.  K2a keeps it (and the entry list) in
// shared memory; K2b rebuilds it from the tile's record and reads the entries from global.
struct TileCtx {
    const Cell *cell;                       // distinct source strategies of unit u-1 (ascending, global)
    const int32_t *idx;                     // their strategy index
    const double *r;                        // K x K transform costs of unit u
    int S, K, n_e, lo_prev, lo, hi, nw;
    int r_base, n_ent, first_bp;            // the tile: rows [r_base, r_base + 1024), entries
    int64_t b_off, par_off, f_off;
    int64_t rm_prev, rm_cur;                // row maps of B_{u-1} and B_u (offsets into a.rmap)
    uint16_t *erow;                         // row of each entry, relative to the tile's first row
    uint16_t *echg;                         // bit kk: column kk changes at the entry's row
    const uint16_t *goff;                   // heavy tiles: first entry of each 32-row group (33), or null
};

// Heavy tile deferred to K2b (one per tile slot): its context, so K2b reads one record.
struct alignas(16) HeavyTile {
    TileCtx t;
    int32_t rounds, done;
    uint16_t goff[33];                      // first entry of group g; goff[32] = n_ent
};
static_assert(sizeof(HeavyTile) <= kK2HeavyBytes, "HeavyTile size");
static_assert(sizeof(TileCtx) <= kStepCtxBytes && sizeof(TileCtx) % 8 == 0, "step context size");

__device__ __forceinline__ void load_tile_ctx(const ChunkArgs &a, int u, int q, int tile, TileCtx &t) {
    const DevProblem &p = a.probs[q];
    const int S = p.S, K = p.K;
    const int64_t ng = rmap_groups(p.n_b + 1);
    t.cell = a.ucell + p.cell_off + (int64_t)(u - 1) * S;
    t.idx = a.uniq + p.cell_off + (int64_t)(u - 1) * S;
    t.r = a.rcls + p.r_off + (int64_t)u * K * K;
    t.S = a.nuniq[p.ustate_off + u - 1]; t.K = K; t.n_e = (int)(p.n_b + 1);
    t.lo_prev = a.unit_lo[p.ustate_off + u - 1];
    t.lo = a.unit_lo[p.ustate_off + u]; t.hi = a.unit_hi[p.ustate_off + u];
    t.b_off = p.b_off; t.par_off = p.par_off;
    t.f_off = p.flag_off; t.nw = (int)flag_words(p.n_b + 1);
    t.rm_prev = p.rmap_off + (int64_t)(u >= 2 ? u - 2 : 0) * ng;
    t.rm_cur = p.rmap_off + (int64_t)(u - 1) * ng;
    t.r_base = tile * kWarpRows;
}

// tile slot of (problem, tile): 1024-row tiles number at most 2 per 2048-row step tile
__device__ __forceinline__ int64_t tile_slot(const ChunkArgs &a, int q, int tile) {
    return 2 * a.step_tiles[q] + tile;
}

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
template <int KT, bool FIRST, bool GUARD, class SH, int IBW = 0>
__device__ __forceinline__ void eval_row(const ChunkArgs &a, const SH &sh, int u, int e, int L, int l,
                                         double *bt, double *bf, int *bk) {
    const int S = sh.S, K = GUARD ? sh.K : KT;
    const int n_e = sh.n_e, lo_prev = FIRST ? 0 : sh.lo_prev;
    // sources in flight per lane: as many as the register budget holds without spilling an
    // in-flight load (a spilled load result serialises the loads)
    constexpr int IB = (KT <= 4) ? kStepIB : (IBW > 0 ? IBW : kStepIBWide);
    const TFCell *bin = a.TF[(u - 1) & 1] + sh.b_off;
    const int2 *rm = a.rmap + sh.rm_prev;
    const uint32_t *fin = a.chg[(u - 1) & 1] + sh.f_off;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) { bt[kk] = GBMW_STEP_INF; bf[kk] = GBMW_STEP_INF; bk[kk] = 0x7fffffff; }
    if constexpr (!FIRST) {
        // IB sources' values in flight, the next IB sources' row-map and change-bit words
        // fetched while they arrive: the chain per group of sources is one load, not two
        int src[IB], k_[IB];
        bool ok[IB];
        int2 m[IB];
        uint32_t cw[IB];
        double cc[IB], cf[IB];
        auto fetch = [&](int i0, int *srcx, int *kx, bool *okx, int2 *mx, uint32_t *cwx, double *ccx, double *cfx) {
#pragma unroll
            for (int b = 0; b < IB; ++b) {
                const int i = i0 + b * L;
                const Cell c = sh.cell[i < S ? i : 0];
                if (GBMW_KEEP_CELL) { ccx[b] = c.c; cfx[b] = c.ef; }
                srcx[b] = e - c.w; kx[b] = c.k;
                okx[b] = i < S && e >= 0 && srcx[b] >= lo_prev;
                mx[b] = make_int2(0, 0); cwx[b] = 0u;
                if (okx[b]) {
                    mx[b] = __ldg(rm + (srcx[b] >> 5));
                    cwx[b] = __ldg(fin + (int64_t)c.k * sh.nw + (srcx[b] >> 5));
                }
            }
        };
        fetch(l, src, k_, ok, m, cw, cc, cf);
        for (int i0 = l; i0 < S; i0 += IB * L) {
            double2 v[IB];
#pragma unroll
            for (int b = 0; b < IB; ++b) {
                v[b] = make_double2(GBMW_STEP_INF, GBMW_STEP_INF);
                if (ok[b]) v[b] = __ldg(reinterpret_cast<const double2 *>(bin + (int64_t)stored_row(m[b], src[b]) * sh.K + k_[b]));
            }
            int srcn[IB], kn[IB];
            bool okn[IB];
            int2 mn[IB];
            uint32_t cwn[IB];
            double ccn[IB], cfn[IB];
            fetch(i0 + IB * L, srcn, kn, okn, mn, cwn, ccn, cfn);
#pragma unroll
            for (int b = 0; b < IB; ++b) {
                if (!ok[b]) continue;
                const int i = i0 + b * L;
                double c_c, c_ef;
                if (GBMW_KEEP_CELL) { c_c = cc[b]; c_ef = cf[b]; }
                else { const Cell c = sh.cell[i]; c_c = c.c; c_ef = c.ef; }
                const double T = v[b].x + c_c, F = v[b].y + c_ef;
                const int key = 2 * i | (int)((cw[b] >> (src[b] & 31)) & 1u);
                const double *rrow = sh.r + k_[b] * K;
#pragma unroll
                for (int kk = 0; kk < KT; ++kk) {
                    if (!GUARD || kk < K) {
                        const double cand = T + rrow[kk];
                        const bool better = lex3_less(cand, F, key, bt[kk], bf[kk], bk[kk]);
                        bt[kk] = better ? cand : bt[kk];
                        bf[kk] = better ? F : bf[kk];
                        bk[kk] = better ? key : bk[kk];
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < IB; ++b) {
                src[b] = srcn[b]; k_[b] = kn[b]; ok[b] = okn[b]; m[b] = mn[b]; cw[b] = cwn[b];
                if (GBMW_KEEP_CELL) { cc[b] = ccn[b]; cf[b] = cfn[b]; }
            }
        }
    } else
    for (int i0 = l; i0 < S; i0 += IB * L) {
        double T[IB], F[IB];
        int key[IB], src_[IB], k_[IB];
        bool ok[IB];
        int2 m[IB];
        uint32_t cw[IB];
#pragma unroll
        for (int b = 0; b < IB; ++b) {
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
        for (int b = 0; b < IB; ++b) {
            if (!ok[b]) continue;
            const Cell c = sh.cell[i0 + b * L];
            if (FIRST) {                       // init row, dpsearch.py:255-259
                T[b] = c.c; F[b] = c.ef;
            } else {
                const int row = stored_row(m[b], src_[b]);
                const double2 v = __ldg(reinterpret_cast<const double2 *>(bin + (int64_t)row * sh.K + k_[b]));
                T[b] = v.x + c.c;
                F[b] = v.y + c.ef;
                key[b] |= (int)((cw[b] >> (src_[b] & 31)) & 1u);
            }
        }
#pragma unroll
        for (int b = 0; b < IB; ++b) {
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

// Phase A, one warp per tile: the breakpoints of its 32 groups (lane g = group g) from the
// change bits of the sources whose window over the tile changes (change summaries), then
// the tile's entries in row order; its first live row is always an entry (the anchor of
// the row map).  In three steps so that K2t can spread the middle one over its warps:
// (A1) the active sources, (A2) each group's breakpoints from a subset of them, (A3) the
// entries from the groups' breakpoint masks.

// A1: sources whose window [r_base - w, r_base + 1023 - w] holds a change, into alist
template <bool FIRST>
__device__ __forceinline__ int active_sources(const ChunkArgs &a, const TileCtx &t, uint16_t *alist, int u, int lane) {
    const int S = t.S, lo_prev = t.lo_prev, r_base = t.r_base;
    int na = 0;
    const int ns = (int)sum_words(t.n_e);
    const uint32_t *sum = a.chg[(u - 1) & 1] + t.f_off + (int64_t)t.K * t.nw;
    for (int n0 = 0; n0 < S; n0 += 32) {
        const int n = n0 + lane;
        bool act = false;
        if (n < S) {
            const Cell c = t.cell[n];
            const int A = r_base - c.w, B = A + kWarpRows - 1;
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
        if (act) alist[na + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)n;
        na += __popc(bal);
    }
    __syncwarp();
    return na;
}

// A2: breakpoints of group g = lane from the active sources of batches b0, b0 + bstep, ...
// (kClassifyIB sources a batch)
template <bool FIRST>
__device__ __forceinline__ unsigned group_segs(const ChunkArgs &a, const TileCtx &t, const uint16_t *alist, int na,
                                               int b0, int bstep, int u, int lane) {
    const int lo_prev = t.lo_prev;
    const int r0 = t.r_base + 32 * lane, r1 = r0 + 31;
    unsigned seg = 0u;
    if (r1 < t.lo || r0 > t.hi) return seg;              // dead group
    const uint32_t *fin = a.chg[(u - 1) & 1] + t.f_off;
    for (int n0 = b0 * kClassifyIB; n0 < na; n0 += bstep * kClassifyIB) {
        uint32_t w0[kClassifyIB], w1[kClassifyIB];
        int xs_[kClassifyIB];
        bool ld[kClassifyIB];
#pragma unroll
        for (int b = 0; b < kClassifyIB; ++b) {
            const int n = n0 + b;
            const Cell c = t.cell[n < na ? alist[n] : 0];
            const int xs = r0 - c.w;
            xs_[b] = xs; w0[b] = 0u; w1[b] = 0u;
            ld[b] = n < na && (FIRST || xs + 31 >= lo_prev);
            if (!FIRST && ld[b]) {
                const int xl = xs < 0 ? 0 : xs;
                const uint32_t *fl = fin + (int64_t)c.k * t.nw + (xl >> 5);
                w0[b] = __ldg(fl); w1[b] = __ldg(fl + 1);
            }
        }
#pragma unroll
        for (int b = 0; b < kClassifyIB; ++b) {
            if (!ld[b]) continue;
            const int xs = xs_[b];
            if (FIRST) {
                const int j = -xs;                       // T_0[e, i] is finite from e = w_i on
                seg |= (j >= 0 && j <= 31) ? (1u << j) : 0u;
            } else {
                const int xl = xs < 0 ? 0 : xs;
                const unsigned long long v =
                    ((unsigned long long)w1[b] << 32 | (unsigned long long)w0[b]) >> (xl & 31);
                seg |= window_segments((xs < 0) ? (v << (-xs)) : v, xs, lo_prev);
            }
        }
    }
    return seg;
}

// A3: a partial group (straddling L_u or H_u) keeps only its live rows; the anchor; the
// entries in row order.  Returns the entry count.
__device__ __forceinline__ int tile_entries(TileCtx &t, uint16_t *goff, unsigned seg, int lane) {
    const int lo = t.lo, hi = t.hi, r_base = t.r_base;
    const int g = lane, r0 = r_base + 32 * g, r1 = r0 + 31;
    const bool dead = r1 < lo || r0 > hi;
    const bool whole = r0 >= lo && r1 <= hi;
    const int f0 = r_base > lo ? r_base : lo;            // first live row of the tile (<= hi)
    if (dead) {
        seg = 0u;
    } else if (!whole) {
        const int a0 = lo > r0 ? lo - r0 : 0, a1 = hi < r1 ? hi - r0 : 31;
        seg &= (0xffffffffu >> (31 - a1)) & ~((1u << a0) - 1u);
    }
    // the anchor: change bits exact unless it is a breakpoint itself
    const bool fbp = __shfl_sync(0xffffffffu, (seg >> ((f0 - r_base) & 31)) & 1u, (f0 - r_base) >> 5) != 0u;
    if (!dead && f0 >= r0 && f0 <= r1) seg |= 1u << (f0 - r0);
    const int cnt = __popc(seg);
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    int at = incl - cnt;
    if (goff) { goff[g] = (uint16_t)at; if (g == 31) goff[32] = (uint16_t)incl; }
    unsigned m = seg;
    while (m) {
        const int x = __ffs(m) - 1;
        m &= m - 1u;
        t.erow[at++] = (uint16_t)(32 * g + x);
    }
    const int n = __shfl_sync(0xffffffffu, incl, 31);
    if (lane == 0) { t.n_ent = n; t.first_bp = (f0 == lo || fbp) ? 1 : 0; }
    __syncwarp();
    return n;
}

template <bool FIRST>
__device__ __forceinline__ int classify_tile(const ChunkArgs &a, TileCtx &t, uint16_t *alist, uint16_t *goff, int u,
                                             int lane) {
    const int na = active_sources<FIRST>(a, t, alist, u, lane);
    return tile_entries(t, goff, group_segs<FIRST>(a, t, alist, na, 0, 1, u, lane), lane);
}

// Evaluation rounds of a tile with n entries, E entries per round: round 0 takes entries
// [0, E) (a segment of 32 / next_pow2(entries) lanes each), round r >= 1 re-evaluates entry
// (E - 1) r (the previous one, for the comparison) and takes the E - 1 after it, 32 / E
// lanes per entry.  Tiles with up to kLightE entries are one round (in K2a); heavier tiles
// use 8-entry rounds (short dependent-load chains, many warps), very dense ones 32-entry
// rounds (a lane per row: fewest instructions per entry).
#ifndef GBMW_LIGHT_E
#define GBMW_LIGHT_E 8
#endif
constexpr int kLightE = GBMW_LIGHT_E;
constexpr int kDenseN = 256;
__device__ __forceinline__ int round_entries(int n) { return n <= kLightE ? kLightE : (n < kDenseN ? 8 : 32); }
__host__ __device__ constexpr int round_entries_c(int n) { return n <= kLightE ? kLightE : (n < kDenseN ? 8 : 32); }
__host__ __device__ constexpr int tile_rounds_c(int n) {
    return n <= round_entries_c(n) ? 1 : 1 + (n - 2) / (round_entries_c(n) - 1);
}
__device__ __forceinline__ int tile_rounds(int n) { return tile_rounds_c(n); }
constexpr int max_tile_rounds() {
    int m = 0;
    for (int n = 1; n <= kWarpRows; ++n) m = tile_rounds_c(n) > m ? tile_rounds_c(n) : m;
    return m;
}
static_assert(max_tile_rounds() <= kK2RoundsPerSlot, "round list capacity per tile slot");

// Phase B, one round of one tile by one warp: evaluate its entries, compare each with the
// previous entry (unchanged columns keep change bit 0), store (t, f, argmin) of the
// entries where some column changes and of the tile's first entry (the anchor).
template <int KT, bool FIRST, bool GUARD, int IBW = 0>
__device__ __forceinline__ void eval_round(const ChunkArgs &a, const TileCtx &t, int u, int r, int lane) {
    const int K = GUARD ? t.K : KT;
    const int n_e = t.n_e, n = t.n_ent;
    int L, j0, nr;                                       // lanes per entry, first entry, entries
    const int E = round_entries(n);
    if (r == 0) {
        nr = n < E ? n : E;
        L = 32;
        while (L > 1 && (32 / L) < nr) L >>= 1;
        j0 = 0;
    } else {
        L = 32 / E;
        j0 = (E - 1) * r;                                // = (first new entry) - 1
        nr = min(E, n - j0);
    }
    const int seg = lane / L, l = lane - seg * L;
    const int j = j0 + seg;
    const bool have = seg < nr;
    const int e = have ? t.r_base + (int)t.erow[j] : -1;
    double bt[KT], bf[KT];
    int bk[KT];
    eval_row<KT, FIRST, GUARD, TileCtx, IBW>(a, t, u, e, L, l, bt, bf, bk);
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
    if (j == 0) chg = t.first_bp ? 0xffffu : 0u;
    chg &= (1u << K) - 1u;
    const bool out = have && l == 0 && (r == 0 || seg > 0);   // lane 0 of a later round: the previous entry
    if (out) {
        if (j == 0 || chg) {
            TFCell *bout = a.TF[u & 1] + t.b_off;
            uint16_t *pout = a.par + t.par_off + ((int64_t)(u - 1) * n_e + e) * K;
            double2 *brow = reinterpret_cast<double2 *>(bout) + (int64_t)e * K;
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
                if (GUARD && kk >= K) break;
                brow[kk] = make_double2(bt[kk], bf[kk]);
                pout[kk] = (uint16_t)t.idx[bk[kk] >> 1];
            }
        }
        t.echg[j] = (uint16_t)chg;
    }
}

// Phase C, one warp per tile, lane g: the change-bit words and the row-map entry of group g,
// and the tile's change-summary word per column.  GLOBAL: the entries live in global memory
// and were written by other warps of this kernel (read through L2).
template <int KT, bool GUARD, bool GLOBAL>
__device__ __forceinline__ void finish_tile(const ChunkArgs &a, const TileCtx &t, int u, int lane) {
    const int K = GUARD ? t.K : KT;
    const int lo = t.lo, hi = t.hi, n = t.n_ent;
    const int r_base = t.r_base;
    const int g = lane, r0 = r_base + 32 * g, r1 = r0 + 31;
    const bool dead = r1 < lo || r0 > hi;
    auto erow = [&](int j) { return GLOBAL ? (int)__ldcg(t.erow + j) : (int)t.erow[j]; };
    auto echg = [&](int j) { return GLOBAL ? (unsigned)__ldcg(t.echg + j) : (unsigned)t.echg[j]; };
    // entries of group g: recorded offsets (heavy tiles), else binary search of the first
    // entry with row >= 32 g
    int b0 = 0, b1 = n;
    if (t.goff) {
        b0 = GLOBAL ? (int)__ldcg(t.goff + g) : (int)t.goff[g];
    } else {
        while (b0 < b1) {
            const int mid = (b0 + b1) >> 1;
            if (erow(mid) < 32 * g) b0 = mid + 1; else b1 = mid;
        }
    }
    int last = -1;                                       // last stored row of the group
    unsigned sbits = 0u;
    uint32_t cwd[KT];
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) cwd[kk] = 0u;
    for (int x0 = b0; x0 < n; ++x0) {
        const int er = erow(x0);
        if (er >= 32 * g + 32) break;
        const int x = er & 31;
        const unsigned m = echg(x0);
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) cwd[kk] |= ((m >> kk) & 1u) << x;
        if (m || x0 == 0) { sbits |= 1u << x; last = r_base + er; }   // entry 0: the anchor
    }
    int before = last;                                   // exclusive max-scan over the groups
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, before, off);
        if (lane >= off) before = max(before, v);
    }
    before = __shfl_up_sync(0xffffffffu, before, 1);
    if (lane == 0) before = -1;
    const int ns = (int)sum_words(t.n_e);
    uint32_t *fout = a.chg[u & 1] + t.f_off;
    uint32_t *sout = fout + (int64_t)K * t.nw;
    const int wi = (r_base >> 5) + g;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
        if (GUARD && kk >= K) break;
        if (!dead) fout[(int64_t)kk * t.nw + wi] = cwd[kk];
        const unsigned sm = __ballot_sync(0xffffffffu, cwd[kk] != 0u);
        if (lane == 0) sout[(int64_t)kk * ns + (r_base >> 10)] = sm;
    }
    if (!dead) a.rmap[t.rm_cur + wi] = make_int2((int)sbits, before);
    if (a.k2_hist && lane == 0) {
        const int bin = 32 - __clz(n);
        atomicAdd(a.k2_hist + bin, 1ull);
        atomicAdd(a.k2_hist + 32 + bin, (unsigned long long)n);
    }
}

// Live-row work lists of every K2 launch of the chunk (one CTA per launch): per active
// problem with live rows, its warp tiles [L_u / kWarpRows, H_u / kWarpRows], one item each.
__global__ void __launch_bounds__(1024) k_step_lists(ChunkArgs a) {
    __shared__ int s_part[1024];
    const StepList sl = a.step_lists[blockIdx.x];
    const int tid = threadIdx.x;
    if (sl.no_items) {                                   // run by K2f / K2s
        if (tid == 0) a.step_count[blockIdx.x] = 0;
        return;
    }
    const int per = (sl.n + 1023) / 1024;
    const int x0 = sl.lo + min(sl.n, tid * per), x1 = sl.lo + min(sl.n, tid * per + per);
    int cnt = 0;
    for (int x = x0; x < x1; ++x) {
        const DevProblem &p = a.probs[x];
        const int lo = a.unit_lo[p.ustate_off + sl.u], hi = a.unit_hi[p.ustate_off + sl.u];
        if (hi >= lo) cnt += hi / kWarpRows - lo / kWarpRows + 1;
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
        // the step context of (problem, unit): K2a copies it in one round trip
        const int64_t ci = sl.ctx_base + (x - sl.lo);
        TileCtx c;
        load_tile_ctx(a, sl.u, x, 0, c);
        c.erow = nullptr; c.echg = nullptr; c.goff = nullptr; c.n_ent = 0; c.first_bp = 0;
        *(reinterpret_cast<TileCtx *>(reinterpret_cast<char *>(a.step_ctx) + ci * kStepCtxBytes)) = c;
        for (int t = lo / kWarpRows; t <= hi / kWarpRows; ++t) a.step_items[at++] = make_int4(x, t, t, (int)ci);
    }
    if (tid == 1023) a.step_count[blockIdx.x] = s_part[1023];
}

int launch_step_lists(const ChunkArgs &a, void *stream) {
    if (a.n_step_lists <= 0) return 0;
    k_step_lists<<<a.n_step_lists, 1024, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

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

// Programmatic dependent launch: every K2 kernel waits for its stream predecessor's
// results before touching memory, and lets its successor launch once it is done.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// debug timeline: slot 2 * id = earliest CTA start, 2 * id + 1 = latest CTA end
__device__ __forceinline__ void tl_mark(unsigned long long *tl, int id, bool end) {
    if (!tl || threadIdx.x != 0 || id >= 4096) return;          // debug buffer: 4096 launches
    if (end) atomicMax(tl + 2 * id + 1, gtimer()); else atomicMin(tl + 2 * id, gtimer());
}

// K2a: a warp per tile (dynamic counter over the launch's tiles).  Tiles whose entries fit
// one round are finished here; heavier ones are handed to K2b.
template <int GROUP, bool FIRST>
__global__ void __launch_bounds__(kStepThreads, GROUP <= 1 ? 3 : 1)
    k_dp_classify(ChunkArgs a, int u, const int4 *items, const int64_t *count, unsigned long long *ctr, int2 *rlist,
                  int tl_id) {
    pdl_wait();
    tl_mark(a.k2_tl, tl_id, false);
    __shared__ TileCtx s_t[kK2Warps];
    __shared__ uint16_t s_erow[kK2Warps][kWarpRows];
    __shared__ uint16_t s_echg[kK2Warps][kWarpRows];
    __shared__ uint16_t s_alist[kK2Warps][kMaxStrats];
    __shared__ uint16_t s_goff[kK2Warps][34];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    TileCtx &t = s_t[warp];
    const int64_t n_items = *count;
    unsigned long long stat_rows = 0;
    int q_prev = -1;
    // non-persistent: warp w of CTA b takes item b * kK2Warps + w and retires, so slots free
    // up continuously and the deep bands' (higher-priority) CTAs get them
    for (int pass = 0; pass < 1; ++pass) {
        const int64_t it = (int64_t)blockIdx.x * kK2Warps + warp;
        if (it >= n_items) break;
        const int4 item = __ldg(items + it);
        if (item.x != q_prev) {                          // the step context: one record, 8 B per lane
            const unsigned long long *src = reinterpret_cast<const unsigned long long *>(
                reinterpret_cast<const char *>(a.step_ctx) + (int64_t)item.w * kStepCtxBytes);
            unsigned long long *dst = reinterpret_cast<unsigned long long *>(&t);
            if (lane < (int)(sizeof(TileCtx) / 8)) dst[lane] = __ldg(src + lane);
            __syncwarp();
        }
        if (lane == 0) {
            t.r_base = item.y * kWarpRows;
            t.erow = s_erow[warp]; t.echg = s_echg[warp]; t.goff = nullptr;
        }
        q_prev = item.x;
        __syncwarp();
        const int n = classify_tile<FIRST>(a, t, s_alist[warp], s_goff[warp], u, lane);
        const int K = t.K;
        stat_rows += (unsigned long long)n * (unsigned long long)K;
        const int rounds = tile_rounds(n);
        if (rounds == 1) {
#define GBMW_K2_EVAL(KT, G) eval_round<KT, FIRST, G>(a, t, u, 0, lane)
            GBMW_K2_DISPATCH(GBMW_K2_EVAL)
#undef GBMW_K2_EVAL
            __syncwarp();
#define GBMW_K2_FIN(KT, G) finish_tile<KT, G, false>(a, t, u, lane)
            GBMW_K2_DISPATCH(GBMW_K2_FIN)
#undef GBMW_K2_FIN
        } else {
            // heavy tile: entries to its global slot, rounds to the launch's list
            const int64_t slot = tile_slot(a, item.x, item.y);
            uint16_t *ge = a.k2_erow + slot * kK2SlotEntries;
            for (int j = lane; j < n; j += 32) ge[j] = s_erow[warp][j];
            unsigned long long base = 0;
            HeavyTile *hr = reinterpret_cast<HeavyTile *>(a.k2_heavy) + slot;
            for (int g = lane; g < 33; g += 32) hr->goff[g] = s_goff[warp][g];
            // no fences: K2b reads the records, entries and round list only after this grid has
            // completed (griddepcontrol.wait), which makes all of its writes visible
            __syncwarp();
            if (lane == 0) {
                TileCtx c = t;
                c.erow = ge; c.echg = a.k2_echg + slot * kK2SlotEntries; c.goff = hr->goff;
                hr->t = c;
                hr->rounds = rounds; hr->done = 0;
                base = atomicAdd(ctr + 1, (unsigned long long)rounds);
            }
            base = __shfl_sync(0xffffffffu, base, 0);
            for (int r = lane; r < rounds; r += 32) rlist[base + r] = make_int2((int)slot, r);
        }
        __syncwarp();
    }
    // the statistics counter is one address for the whole pass: one atomic per CTA, not per
    // warp (same-address atomics serialise in L2 and the grid completes only after them)
    __shared__ unsigned long long s_stat[kK2Warps];
    if (lane == 0) s_stat[warp] = stat_rows;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
#pragma unroll
        for (int w = 0; w < kK2Warps; ++w) tot += s_stat[w];
        if (tot) atomicAdd(a.computed_cells, tot);
    }
    tl_mark(a.k2_tl, tl_id, true);
    pdl_trigger();
}

// K2b: a warp per round of the launch's heavy tiles; the warp completing a tile's last round
// finishes the tile.
template <int GROUP, bool FIRST>
__global__ void __launch_bounds__(kStepThreads, GROUP <= 1 ? 3 : 1)
    k_dp_rounds(ChunkArgs a, int u, unsigned long long *ctr, const int2 *rlist, int tl_id) {
    pdl_wait();
    tl_mark(a.k2_tl, tl_id, false);
    __shared__ TileCtx s_t[kK2Warps];
    __shared__ uint16_t s_erow[kK2Warps][kWarpRows];
    __shared__ uint16_t s_echg[kK2Warps][kWarpRows];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    TileCtx &t = s_t[warp];
    const int64_t total = (int64_t)*(volatile unsigned long long *)(ctr + 1);
    // first round: the warp's global index (no atomic); later ones from the counter
    const int64_t n_warps = (int64_t)gridDim.x * kK2Warps;
    int64_t R = (int64_t)blockIdx.x * kK2Warps + warp;
    while (true) {
        if (R >= total) break;
        const int2 rr = rlist[R];
        const int64_t slot = rr.x;
        HeavyTile *ht = reinterpret_cast<HeavyTile *>(a.k2_heavy) + slot;
        {                                                // the tile's context: one record, 8 B per lane
            static_assert(sizeof(TileCtx) % 8 == 0 && sizeof(TileCtx) <= 256, "TileCtx copy");
            const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&ht->t);
            unsigned long long *dst = reinterpret_cast<unsigned long long *>(&t);
            if (lane < (int)(sizeof(TileCtx) / 8)) dst[lane] = __ldcg(src + lane);
        }
        __syncwarp();
        const int K = t.K;
#define GBMW_K2_EVAL(KT, G) eval_round<KT, FIRST, G>(a, t, u, rr.y, lane)
        GBMW_K2_DISPATCH(GBMW_K2_EVAL)
#undef GBMW_K2_EVAL
        __threadfence();
        __syncwarp();
        int last = 0;
        if (lane == 0) last = atomicAdd(&ht->done, 1) == ht->rounds - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
            __threadfence();
            // the tile's entries into shared memory with coalesced loads (all independent),
            // then the finish reads them there instead of chasing them in global memory
            const int n = t.n_ent;
            for (int j = lane; j < n; j += 32) {
                s_erow[warp][j] = __ldcg(t.erow + j);
                s_echg[warp][j] = __ldcg(t.echg + j);
            }
            __syncwarp();
            if (lane == 0) { t.erow = s_erow[warp]; t.echg = s_echg[warp]; t.goff = nullptr; }
            __syncwarp();
#define GBMW_K2_FIN(KT, G) finish_tile<KT, G, false>(a, t, u, lane)
            GBMW_K2_DISPATCH(GBMW_K2_FIN)
#undef GBMW_K2_FIN
        }
        __syncwarp();
        if (n_warps >= total) break;
        int64_t nx = 0;
        if (lane == 0) nx = n_warps + (int64_t)atomicAdd(ctr + 2, 1ull);
        R = __shfl_sync(0xffffffffu, nx, 0);
    }
    __syncthreads();
    tl_mark(a.k2_tl, tl_id, true);
    pdl_trigger();
}

// K2t: both halves of a layer step in one kernel, a CTA per tile, for launches with few
// tiles (the deep bands' tail, where the step chain, not the throughput, bounds the pass):
// warp 0 classifies the tile into shared memory, the CTA's warps share its rounds, warp 0
// finishes it.  No hand-off through global memory and no second kernel per step.
#ifndef GBMW_TILE_IB_WIDE
#define GBMW_TILE_IB_WIDE 1
#endif
constexpr int kTileIBWide = GBMW_TILE_IB_WIDE;   // K2t: sources in flight per lane for K >= 5 (2, 3: no spills, measured no faster)

template <int GROUP, bool FIRST, int kTileWarps>
__global__ void __launch_bounds__(32 * kTileWarps)
    k_dp_tile(ChunkArgs a, int u, const int4 *items, const int64_t *count, int tl_id) {
    pdl_wait();
    tl_mark(a.k2_tl, tl_id, false);
    __shared__ TileCtx s_t;
    __shared__ uint16_t s_erow[kWarpRows];
    __shared__ uint16_t s_echg[kWarpRows];
    __shared__ uint16_t s_alist[kMaxStrats];
    __shared__ uint16_t s_goff[34];
    __shared__ unsigned s_seg[32];
    __shared__ int s_n, s_na;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    TileCtx &t = s_t;
    const int64_t it = blockIdx.x;
    if (it < *count) {                                   // CTA-uniform
        if (warp == 0) {
            const int4 item = __ldg(items + it);
            const unsigned long long *src = reinterpret_cast<const unsigned long long *>(
                reinterpret_cast<const char *>(a.step_ctx) + (int64_t)item.w * kStepCtxBytes);
            unsigned long long *dst = reinterpret_cast<unsigned long long *>(&t);
            if (lane < (int)(sizeof(TileCtx) / 8)) dst[lane] = __ldg(src + lane);
            __syncwarp();
            if (lane == 0) {
                t.r_base = item.y * kWarpRows;
                t.erow = s_erow; t.echg = s_echg; t.goff = nullptr;
            }
            __syncwarp();
            const int na = active_sources<FIRST>(a, t, s_alist, u, lane);
            if (lane == 0) s_na = na;
            s_seg[lane] = 0u;
        }
        __syncthreads();
        // the groups' breakpoints: the warps take the active sources' batches in turn
        const unsigned sg = group_segs<FIRST>(a, t, s_alist, s_na, warp, kTileWarps, u, lane);
        if (sg) atomicOr(&s_seg[lane], sg);
        __syncthreads();
        if (warp == 0) {
            const int n = tile_entries(t, s_goff, s_seg[lane], lane);
            if (lane == 0) { s_n = n; t.goff = s_goff; }
        }
        __syncthreads();
        const int n = s_n, K = t.K;
        const int rounds = tile_rounds(n);
        for (int r = warp; r < rounds; r += kTileWarps) {
#define GBMW_K2_EVAL(KT, G) eval_round<KT, FIRST, G, kTileIBWide>(a, t, u, r, lane)
            GBMW_K2_DISPATCH(GBMW_K2_EVAL)
#undef GBMW_K2_EVAL
        }
        __syncthreads();
        if (warp == 0) {
#define GBMW_K2_FIN(KT, G) finish_tile<KT, G, false>(a, t, u, lane)
            GBMW_K2_DISPATCH(GBMW_K2_FIN)
#undef GBMW_K2_FIN
            if (lane == 0 && n) atomicAdd(a.computed_cells, (unsigned long long)n * (unsigned long long)K);
        }
    }
    tl_mark(a.k2_tl, tl_id, true);
    tl_mark(a.k2_tl, tl_id + 1, false);                  // debug timeline: an empty second half
    tl_mark(a.k2_tl, tl_id + 1, true);
    pdl_trigger();
}

// K2 for the first layer step (u = 1), one CTA per problem.  T_0[e, i] = time_c[0, i] for
// e >= w_0i (dpsearch.py:255-259), so B_1 is piecewise constant with breakpoints only at the
// distinct first-unit weights: B_1 is evaluated once per segment (the same lexmin as every
// other step, T1 tie-break), stored at the segment starts where some column changes, and
// the per-group outputs (change bits, summaries, row map) are written directly — no tiles,
// no anchors.
constexpr int kFirstThreads = 256;
constexpr int kFirstMaxSeg = kMaxStrats + 1;

__global__ void __launch_bounds__(kFirstThreads) k_dp_first(ChunkArgs a, int p_lo, int p_n) {
    __shared__ int s_start[kFirstMaxSeg];                // segment start rows, ascending
    __shared__ uint32_t s_chg[kFirstMaxSeg];             // bit k: column k changes at the start
    __shared__ int s_stored[kFirstMaxSeg];               // stored rows, ascending
    __shared__ double s_t[kFirstMaxSeg], s_f[kFirstMaxSeg];
    __shared__ int s_key[kFirstMaxSeg];
    __shared__ int s_m, s_ns;
    const int q = p_lo + (int)blockIdx.x;
    if ((int)blockIdx.x >= p_n) return;
    const DevProblem &p = a.probs[q];
    const int u = 1;
    const int lo = a.unit_lo[p.ustate_off + u], hi = a.unit_hi[p.ustate_off + u];
    if (hi < lo) return;
    const int S = a.nuniq[p.ustate_off + 0], K = p.K;
    const Cell *cell = a.ucell + p.cell_off;             // distinct sources of unit 0
    const int32_t *idx = a.uniq + p.cell_off;
    const double *R = a.rcls + p.r_off + (int64_t)u * K * K;
    const int n_e = (int)(p.n_b + 1);
    const int tid = threadIdx.x;
    // segment starts: the distinct weights in [lo, hi] (lo is the smallest weight), ascending
    __shared__ unsigned char s_first[kMaxStrats];       // source n holds the first occurrence of its weight
    for (int n = tid; n < S; n += blockDim.x) {
        const int w = cell[n].w;
        bool first = w >= lo && w <= hi;
        for (int j = 0; j < n && first; ++j) if (cell[j].w == w) first = false;
        s_first[n] = first ? 1 : 0;
    }
    __syncthreads();
    for (int n = tid; n < S; n += blockDim.x) {
        if (!s_first[n]) continue;
        const int w = cell[n].w;
        int pos = 0;
        for (int j = 0; j < S; ++j) pos += (s_first[j] && cell[j].w < w) ? 1 : 0;
        s_start[pos] = w;
    }
    if (tid == 0) {
        int m = 0;
        for (int n = 0; n < S; ++n) m += s_first[n];
        s_m = m;
    }
    __syncthreads();
    const int m = s_m;
    for (int j = tid; j < m; j += blockDim.x) s_chg[j] = (j == 0) ? ((K >= 32) ? 0xffffffffu : ((1u << K) - 1u)) : 0u;
    __syncthreads();
    // per column: B_1 at every segment start, then the change bits against the previous segment
    for (int k = 0; k < K; ++k) {
        for (int j = tid; j < m; j += blockDim.x) {
            const int e = s_start[j];
            double bt = GBMW_STEP_INF, bf = GBMW_STEP_INF;
            int bk = 0x7fffffff;
            for (int n = 0; n < S; ++n) {                // ascending source order (T1)
                const Cell c = cell[n];
                if (c.w > e) continue;
                const double cand = c.c + R[c.k * K + k];
                if (lex3_less(cand, c.ef, 2 * n, bt, bf, bk)) { bt = cand; bf = c.ef; bk = 2 * n; }
            }
            s_t[j] = bt; s_f[j] = bf; s_key[j] = bk;
        }
        __syncthreads();
        for (int j = tid + 1; j < m; j += blockDim.x)
            if (!(s_t[j] == s_t[j - 1] && s_f[j] == s_f[j - 1] && s_key[j] == s_key[j - 1])) s_chg[j] |= 1u << k;
        __syncthreads();
    }
    if (tid == 0) {
        int ns = 0;
        for (int j = 0; j < m; ++j) if (j == 0 || s_chg[j]) s_stored[ns++] = s_start[j];
        s_ns = ns;
    }
    __syncthreads();
    const int ns = s_ns;
    // (t, f, argmin) of every column at the stored rows
    TFCell *bout = a.TF[u & 1] + p.b_off;
    uint16_t *pout = a.par + p.par_off + (int64_t)(u - 1) * K * n_e;   // rows of K argmins
    for (int k = 0; k < K; ++k) {
        for (int j = tid; j < m; j += blockDim.x) {
            if (!(j == 0 || s_chg[j])) continue;
            const int e = s_start[j];
            double bt = GBMW_STEP_INF, bf = GBMW_STEP_INF;
            int bk = 0x7fffffff;
            for (int n = 0; n < S; ++n) {
                const Cell c = cell[n];
                if (c.w > e) continue;
                const double cand = c.c + R[c.k * K + k];
                if (lex3_less(cand, c.ef, 2 * n, bt, bf, bk)) { bt = cand; bf = c.ef; bk = 2 * n; }
            }
            reinterpret_cast<double2 *>(bout)[(int64_t)e * K + k] = make_double2(bt, bf);
            pout[(int64_t)e * K + k] = (uint16_t)idx[bk >> 1];
        }
    }
    // per 32-row group of the live rows: change-bit words, row map; per tile: summaries
    const int nw = (int)flag_words(n_e), nsw = (int)sum_words(n_e);
    uint32_t *fout = a.chg[u & 1] + p.flag_off;
    uint32_t *sout = fout + (int64_t)K * nw;
    int2 *rmo = a.rmap + p.rmap_off;                     // unit u = 1: row map index 0
    const int lane = tid & 31, warp = tid >> 5;
    for (int tile = lo / kWarpRows + warp; tile <= hi / kWarpRows; tile += blockDim.x / 32) {
        const int r0 = tile * kWarpRows + 32 * lane, r1 = r0 + 31;
        const bool dead = r1 < lo || r0 > hi;
        int j0 = 0, j1 = m;                              // first segment start >= r0
        while (j0 < j1) { const int mid = (j0 + j1) >> 1; if (s_start[mid] < r0) j0 = mid + 1; else j1 = mid; }
        int s0 = 0, s1 = ns;                             // first stored row >= r0
        while (s0 < s1) { const int mid = (s0 + s1) >> 1; if (s_stored[mid] < r0) s0 = mid + 1; else s1 = mid; }
        const int before = s0 > 0 ? s_stored[s0 - 1] : -1;
        unsigned sbits = 0u;
        for (int x = s0; x < ns && s_stored[x] <= r1; ++x) sbits |= 1u << (s_stored[x] - r0);
        for (int k = 0; k < K; ++k) {
            uint32_t wd = 0u;
            for (int j = j0; j < m && s_start[j] <= r1; ++j) wd |= ((s_chg[j] >> k) & 1u) << (s_start[j] - r0);
            if (!dead) fout[(int64_t)k * nw + (r0 >> 5)] = wd;
            const unsigned sm = __ballot_sync(0xffffffffu, wd != 0u);
            if (lane == 0) sout[(int64_t)k * nsw + tile] = sm;
        }
        if (!dead) rmo[r0 >> 5] = make_int2((int)sbits, before);
    }
    if (tid == 0) atomicAdd(a.computed_cells, (unsigned long long)m * (unsigned long long)K);
}

int launch_dp_first(const ChunkArgs &a, int p_lo, int p_n, void *stream) {
    if (p_n <= 0) return 0;
    k_dp_first<<<p_n, kFirstThreads, 0, (cudaStream_t)stream>>>(a, p_lo, p_n);
    return (int)cudaGetLastError();
}

// K2 for the second layer step (u = 2), one CTA per problem, for problems with few
// distinct sources (S <= kSecondMaxS) and few rows (n_e <= kSecondMaxRows).  B_1 changes at
// a handful of rows (K2f), so the rows of B_2 where some source's input changes are the
// sums y + w_i over the change rows y of B_1 in column cls(i) and the unit-1 weights w_i:
// at most (S + 1) S of them.  They are collected in a shared-memory bitmap, evaluated in
// row order by the same lexmin as every step (eval_row, T1 tie-break, path-aware keys),
// compared with the previous candidate (exact change bits: no tile anchors), and the row
// map / change words / summaries written per group as K2 writes them.
constexpr int kSecondThreads = 256;
constexpr int kSecondMaxX = 4096;                        // candidate rows
constexpr int kSecondMaxY = 128;                         // change rows of B_1
constexpr int kSecondChunk = 64;                         // candidates per evaluation pass
constexpr int kSecondL = 8;                              // lanes per candidate
struct SecondSmem {
    int x[kSecondMaxX];                                  // candidate rows, ascending
    union {
        uint32_t bits[kSecondMaxX];                      // candidate bitmap over [L_2, L_2 + 32 * 4096)
        int last[kSecondMaxX];                           // last stored row at or before candidate j
    };
    uint16_t mask[kSecondMaxX];                          // change bits of candidate j
    int y[kSecondMaxY];
    uint32_t ymask[kSecondMaxY];
    double rt[(kSecondChunk + 1) * kMaxClasses], rf[(kSecondChunk + 1) * kMaxClasses];
    int rk[(kSecondChunk + 1) * kMaxClasses];
    int scan[40];
    TileCtx t;
};

// exclusive prefix sum over the block (blockDim.x == kSecondThreads); *total = sum
__device__ __forceinline__ int second_scan(int v, int *tmp, int *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) tmp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = kSecondThreads / 32;
        int w = lane < nw ? tmp[lane] : 0;
        int wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, wi, off);
            if (lane >= off) wi += o;
        }
        if (lane < nw) tmp[lane] = wi - w;
        if (lane == nw - 1) tmp[32] = wi;
    }
    __syncthreads();
    const int r = incl - v + tmp[warp];
    *total = tmp[32];
    __syncthreads();
    return r;
}

// exclusive prefix max over the block (identity -1)
__device__ __forceinline__ int second_scan_max(int v, int *tmp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl = max(incl, o);
    }
    if (lane == 31) tmp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = kSecondThreads / 32;
        const int w = lane < nw ? tmp[lane] : -1;
        int wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, wi, off);
            if (lane >= off) wi = max(wi, o);
        }
        const int ex = __shfl_up_sync(0xffffffffu, wi, 1);
        if (lane < nw) tmp[lane] = lane == 0 ? -1 : ex;
    }
    __syncthreads();
    const int ex_lane = __shfl_up_sync(0xffffffffu, incl, 1);
    const int r = max(tmp[warp], lane == 0 ? -1 : ex_lane);
    __syncthreads();
    return r;
}

// evaluate candidates [c0, c0 + nc) into result slots 1..nc (slot 0: the previous candidate)
template <int KT, bool GUARD>
__device__ __forceinline__ void second_eval(const ChunkArgs &a, SecondSmem &sm, int c0, int nc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per_warp = 32 / kSecondL;
    const int seg = lane / kSecondL, l = lane - seg * kSecondL;
    for (int j0 = warp * per_warp; j0 < nc; j0 += (kSecondThreads / 32) * per_warp) {
        const int j = j0 + seg;
        const int e = j < nc ? sm.x[c0 + j] : -1;
        double bt[KT], bf[KT];
        int bk[KT];
        eval_row<KT, false, GUARD>(a, sm.t, 2, e, kSecondL, l, bt, bf, bk);
        if (j < nc && l == 0) {
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
                if (GUARD && kk >= sm.t.K) break;
                sm.rt[(j + 1) * kMaxClasses + kk] = bt[kk];
                sm.rf[(j + 1) * kMaxClasses + kk] = bf[kk];
                sm.rk[(j + 1) * kMaxClasses + kk] = bk[kk];
            }
        }
    }
}

template <int GROUP>
__global__ void __launch_bounds__(kSecondThreads, GROUP <= 1 ? 2 : 1) k_dp_second(ChunkArgs a, int p_lo, int p_n) {
    extern __shared__ __align__(16) unsigned char second_raw[];
    SecondSmem &sm = *reinterpret_cast<SecondSmem *>(second_raw);
    const int q = p_lo + (int)blockIdx.x;
    if ((int)blockIdx.x >= p_n) return;
    const int u = 2, tid = threadIdx.x;
    if (tid == 0) load_tile_ctx(a, u, q, 0, sm.t);
    __syncthreads();
    const TileCtx &t = sm.t;
    const int lo = t.lo, hi = t.hi, lo1 = t.lo_prev, K = t.K, S = t.S, n_e = t.n_e;
    if (hi < lo) return;
    const DevProblem &p = a.probs[q];
    const int hi1 = a.unit_hi[p.ustate_off + 1];
    const uint32_t *fin = a.chg[(u - 1) & 1] + t.f_off;
    const uint32_t allk = (K >= 32) ? 0xffffffffu : ((1u << K) - 1u);
    // 1. change rows of B_1: its stored rows (row map of unit 1) and their change columns
    {
        const int g0 = lo1 >> 5, g1 = hi1 >> 5, G = g1 - g0 + 1;
        const int per = (G + kSecondThreads - 1) / kSecondThreads;
        const int ga = g0 + tid * per, gb = min(g0 + (tid + 1) * per, g1 + 1);
        int cnt = 0;
        for (int g = ga; g < gb; ++g) cnt += __popc((unsigned)__ldg(a.rmap + t.rm_prev + g).x);
        int total = 0;
        int at = second_scan(cnt, sm.scan, &total);
        for (int g = ga; g < gb; ++g) {
            unsigned b = (unsigned)__ldg(a.rmap + t.rm_prev + g).x;
            while (b) {
                const int x = __ffs(b) - 1;
                b &= b - 1u;
                const int y = 32 * g + x;
                uint32_t m = 0u;
                for (int k = 0; k < K; ++k) m |= ((__ldg(fin + (int64_t)k * t.nw + (y >> 5)) >> x) & 1u) << k;
                if (y == lo1) m = allk;                  // the first finite row: every column
                if (at < kSecondMaxY) { sm.y[at] = y; sm.ymask[at] = m; }
                ++at;
            }
        }
        if (tid == 0) sm.scan[36] = total;
        __syncthreads();
    }
    const int ny = min(sm.scan[36], kSecondMaxY);
    // 2. candidate bitmap over [lo, hi]
    const int nbits = hi - lo + 1, nwd = (nbits + 31) >> 5;
    for (int w = tid; w < nwd; w += kSecondThreads) sm.bits[w] = 0u;
    __syncthreads();
    if (tid == 0) atomicOr(&sm.bits[0], 1u);                // the first live row (the anchor)
    for (int pi = tid; pi < ny * S; pi += kSecondThreads) {
        const int jy = pi / S, i = pi - jy * S;
        const Cell c = t.cell[i];
        if (!((sm.ymask[jy] >> c.k) & 1u)) continue;
        const int x = sm.y[jy] + c.w;
        if (x < lo || x > hi) continue;
        atomicOr(&sm.bits[(x - lo) >> 5], 1u << ((x - lo) & 31));
    }
    __syncthreads();
    // 3. candidates in row order
    int nx = 0;
    {
        const int per = (nwd + kSecondThreads - 1) / kSecondThreads;
        const int wa = tid * per, wb = min((tid + 1) * per, nwd);
        int cnt = 0;
        for (int w = wa; w < wb; ++w) cnt += __popc(sm.bits[w]);
        int at = second_scan(cnt, sm.scan, &nx);
        for (int w = wa; w < wb; ++w) {
            unsigned b = sm.bits[w];
            while (b) {
                const int x = __ffs(b) - 1;
                b &= b - 1u;
                if (at < kSecondMaxX) sm.x[at] = lo + 32 * w + x;
                ++at;
            }
        }
        __syncthreads();
    }
    nx = min(nx, kSecondMaxX);                           // host bound: (S + 1) S <= kSecondMaxX
    // 4. evaluation in chunks, change bits against the previous candidate, stored rows out
    TFCell *bout = a.TF[u & 1] + t.b_off;
    uint16_t *pout = a.par + t.par_off + (int64_t)(u - 1) * K * n_e;
    for (int c0 = 0; c0 < nx; c0 += kSecondChunk) {
        const int nc = min(kSecondChunk, nx - c0);
#define GBMW_K2S_EVAL(KT, G) second_eval<KT, G>(a, sm, c0, nc)
        GBMW_K2_DISPATCH(GBMW_K2S_EVAL)
#undef GBMW_K2S_EVAL
        __syncthreads();
        for (int j = tid; j < nc; j += kSecondThreads) {
            uint32_t chg = 0u;
            const int s1 = (j + 1) * kMaxClasses, s0 = j * kMaxClasses;
            for (int kk = 0; kk < K; ++kk) {
                const bool same = sm.rt[s1 + kk] == sm.rt[s0 + kk] && sm.rf[s1 + kk] == sm.rf[s0 + kk] &&
                                  (sm.rk[s1 + kk] >> 1) == (sm.rk[s0 + kk] >> 1) && !(sm.rk[s1 + kk] & 1);
                chg |= same ? 0u : (1u << kk);
            }
            if (c0 + j == 0) chg = allk;
            sm.mask[c0 + j] = (uint16_t)chg;
        }
        for (int jk = tid; jk < nc * K; jk += kSecondThreads) {
            const int j = jk / K, kk = jk - j * K;
            const int s1 = (j + 1) * kMaxClasses;
            // stored: the anchor and every candidate where some column changes (mask of j
            // is recomputed here from the same slots, so no barrier is needed)
            uint32_t chg = 0u;
            for (int k2 = 0; k2 < K; ++k2) {
                const int s0 = j * kMaxClasses;
                const bool same = sm.rt[s1 + k2] == sm.rt[s0 + k2] && sm.rf[s1 + k2] == sm.rf[s0 + k2] &&
                                  (sm.rk[s1 + k2] >> 1) == (sm.rk[s0 + k2] >> 1) && !(sm.rk[s1 + k2] & 1);
                chg |= same ? 0u : 1u;
            }
            if (c0 + j == 0 || chg) {
                const int e = sm.x[c0 + j];
                reinterpret_cast<double2 *>(bout)[(int64_t)e * K + kk] = make_double2(sm.rt[s1 + kk], sm.rf[s1 + kk]);
                pout[(int64_t)e * K + kk] = (uint16_t)t.idx[sm.rk[s1 + kk] >> 1];
            }
        }
        __syncthreads();
        for (int kk = tid; kk < K; kk += kSecondThreads) {   // carry the last candidate to slot 0
            sm.rt[kk] = sm.rt[nc * kMaxClasses + kk];
            sm.rf[kk] = sm.rf[nc * kMaxClasses + kk];
            sm.rk[kk] = sm.rk[nc * kMaxClasses + kk];
        }
        __syncthreads();
    }
    // 5. last stored row at or before each candidate (the bitmap is dead: reuse as `last`)
    {
        const int per = (nx + kSecondThreads - 1) / kSecondThreads;
        const int ja = tid * per, jb = min((tid + 1) * per, nx);
        int loc = -1;
        for (int j = ja; j < jb; ++j) if (j == 0 || sm.mask[j]) loc = sm.x[j];
        int run = second_scan_max(loc, sm.scan);
        for (int j = ja; j < jb; ++j) {
            if (j == 0 || sm.mask[j]) run = sm.x[j];
            sm.last[j] = run;
        }
        __syncthreads();
    }
    // 6. per 32-row group of the live rows: change words, row map; per tile: summaries
    const int nw = t.nw, nsw = (int)sum_words(n_e);
    uint32_t *fout = a.chg[u & 1] + t.f_off;
    uint32_t *sout = fout + (int64_t)K * nw;
    int2 *rmo = a.rmap + t.rm_cur;
    const int lane = tid & 31, warp = tid >> 5;
    for (int tile = lo / kWarpRows + warp; tile <= hi / kWarpRows; tile += kSecondThreads / 32) {
        const int r0 = tile * kWarpRows + 32 * lane, r1 = r0 + 31;
        const bool dead = r1 < lo || r0 > hi;
        int j0 = 0, j1 = nx;                             // first candidate >= r0
        while (j0 < j1) { const int mid = (j0 + j1) >> 1; if (sm.x[mid] < r0) j0 = mid + 1; else j1 = mid; }
        const int before = j0 > 0 ? sm.last[j0 - 1] : -1;
        unsigned sbits = 0u;
        for (int j = j0; j < nx && sm.x[j] <= r1; ++j)
            if (j == 0 || sm.mask[j]) sbits |= 1u << (sm.x[j] - r0);
        for (int k = 0; k < K; ++k) {
            uint32_t wd = 0u;
            for (int j = j0; j < nx && sm.x[j] <= r1; ++j) wd |= ((uint32_t)(sm.mask[j] >> k) & 1u) << (sm.x[j] - r0);
            if (!dead) fout[(int64_t)k * nw + (r0 >> 5)] = wd;
            const unsigned smk = __ballot_sync(0xffffffffu, wd != 0u);
            if (lane == 0) sout[(int64_t)k * nsw + tile] = smk;
        }
        if (!dead) rmo[r0 >> 5] = make_int2((int)sbits, before);
    }
    if (tid == 0) atomicAdd(a.computed_cells, (unsigned long long)nx * (unsigned long long)K);
}

#undef GBMW_K2_DISPATCH

int launch_dp_second(const ChunkArgs &a, int group, int p_lo, int p_n, void *stream) {
    if (p_n <= 0) return 0;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_dp_second<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SecondSmem));
        cudaFuncSetAttribute(k_dp_second<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SecondSmem));
        cudaFuncSetAttribute(k_dp_second<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SecondSmem));
        attr = true;
    }
    const size_t sb = sizeof(SecondSmem);
    cudaStream_t st = (cudaStream_t)stream;
    if (group == 0) k_dp_second<0><<<p_n, kSecondThreads, sb, st>>>(a, p_lo, p_n);
    else if (group == 1) k_dp_second<1><<<p_n, kSecondThreads, sb, st>>>(a, p_lo, p_n);
    else k_dp_second<2><<<p_n, kSecondThreads, sb, st>>>(a, p_lo, p_n);
    return (int)cudaGetLastError();
}

int launch_dp_step(const ChunkArgs &a, int group, int u, const int4 *items, const int64_t *count, int64_t n_items,
                   unsigned long long *ctr, int2 *rounds, int tl_id, void *stream, int *n_kernels) {
    cudaStream_t st = (cudaStream_t)stream;
    *n_kernels = 0;
    if (n_items <= 0) return 0;
    static int sms = 0;
    static int occ[kStepGroups][2][2] = {{{0}}};
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    const int fi = (u == 1) ? 1 : 0;
#define GBMW_PREP(G, F)                                                                                    \
    do {                                                                                                   \
        int n = 1, m = 1;                                                                                  \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_dp_classify<G, F>, kStepThreads, 0);          \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, k_dp_rounds<G, F>, kStepThreads, 0);            \
        occ[G][F ? 1 : 0][0] = n > 0 ? n : 1;                                                              \
        occ[G][F ? 1 : 0][1] = m > 0 ? m : 1;                                                              \
    } while (0)
    if (occ[group][fi][0] == 0) {
        if (group == 0) { if (fi) GBMW_PREP(0, true); else GBMW_PREP(0, false); }
        else if (group == 1) { if (fi) GBMW_PREP(1, true); else GBMW_PREP(1, false); }
        else { if (fi) GBMW_PREP(2, true); else GBMW_PREP(2, false); }
    }
    const unsigned grid_a = (unsigned)((n_items + kK2Warps - 1) / kK2Warps);   // one item per warp
    const unsigned grid_b = (unsigned)(sms * occ[group][fi][1]);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg_a = {}, cfg_b = {};
    cfg_a.gridDim = dim3(grid_a); cfg_a.blockDim = dim3(kStepThreads); cfg_a.stream = st;
    cfg_a.attrs = attr; cfg_a.numAttrs = 1;
    cfg_b = cfg_a; cfg_b.gridDim = dim3(grid_b);
    const int ta = 2 * tl_id, tb = 2 * tl_id + 1;
    // few tiles: one fused kernel, a CTA per tile (GBMW_TILE_FUSED_MAX: the item bound up to
    // which it is used; 0 disables it).  Measured bounds 0 / 2048 / 3072 / 4096: 10k sweep
    // 7.52-7.58 / 7.34-7.48 / 7.72-7.75 / 7.76 ms; device time of the full searches at 2048:
    // gpt96 23.3 -> 21.1 ms, swin-bmw 38.5 -> 31.5 ms, vit-bmw 29.5 -> 23.8 ms
    static const int64_t fused_max = getenv("GBMW_TILE_FUSED_MAX") ? atoll(getenv("GBMW_TILE_FUSED_MAX")) : 2048;
    // eight warps per tile CTA up to this item bound, four above it
    static const int64_t wide_max = getenv("GBMW_TILE_WIDE_MAX") ? atoll(getenv("GBMW_TILE_WIDE_MAX")) : 1024;
    // class-count groups (bit g) that use it
    static const int fused_groups = getenv("GBMW_TILE_FUSED_GROUPS") ? atoi(getenv("GBMW_TILE_FUSED_GROUPS")) : 7;
    if (n_items <= fused_max && ((fused_groups >> group) & 1)) {
        cudaLaunchConfig_t cfg_t = cfg_a;
        const bool wide = n_items <= wide_max;
        cfg_t.gridDim = dim3((unsigned)n_items); cfg_t.blockDim = dim3(wide ? 256 : 128);
#define GBMW_TILE(G)                                                                                    \
        if (wide) {                                                                                     \
            if (fi) cudaLaunchKernelEx(&cfg_t, k_dp_tile<G, true, 8>, a, u, items, count, ta);           \
            else cudaLaunchKernelEx(&cfg_t, k_dp_tile<G, false, 8>, a, u, items, count, ta);             \
        } else {                                                                                        \
            if (fi) cudaLaunchKernelEx(&cfg_t, k_dp_tile<G, true, 4>, a, u, items, count, ta);           \
            else cudaLaunchKernelEx(&cfg_t, k_dp_tile<G, false, 4>, a, u, items, count, ta);             \
        }
        if (group == 0) { GBMW_TILE(0) }
        else if (group == 1) { GBMW_TILE(1) }
        else { GBMW_TILE(2) }
#undef GBMW_TILE
        *n_kernels = 1;
        return (int)cudaGetLastError();
    }
#define GBMW_STEP(G)                                                                                    \
    if (fi) {                                                                                           \
        cudaLaunchKernelEx(&cfg_a, k_dp_classify<G, true>, a, u, items, count, ctr, rounds, ta);        \
        cudaLaunchKernelEx(&cfg_b, k_dp_rounds<G, true>, a, u, ctr, (const int2 *)rounds, tb);          \
    } else {                                                                                            \
        cudaLaunchKernelEx(&cfg_a, k_dp_classify<G, false>, a, u, items, count, ctr, rounds, ta);       \
        cudaLaunchKernelEx(&cfg_b, k_dp_rounds<G, false>, a, u, ctr, (const int2 *)rounds, tb);         \
    }
    if (group == 0) { GBMW_STEP(0) }
    else if (group == 1) { GBMW_STEP(1) }
    else { GBMW_STEP(2) }
#undef GBMW_STEP
#undef GBMW_PREP
    *n_kernels = 2;
    return (int)cudaGetLastError();
}

}  // namespace gbmw
