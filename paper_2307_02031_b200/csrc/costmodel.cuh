// costmodel.cuh — the Galvatron-BMW per-(layer, strategy) cost model, shared by the
// host C++ (partition logic, validation) and the sm_100a kernels (K1 tables, K4
// stage epilogue).
//
// Bit-exactness contract (SURVEY.md §8 "Arithmetic contract"): the reference is
// Python floats, so every expression below keeps the reference's evaluation
// order, never contracts a*b+c into an FMA (host: -ffp-contract=off, device:
// -fmad=false), and performs Python's implicit int -> float conversions at the
// same points.  Python's max(a, b) returns a unless b > a (py_max).
#pragma once

#include <stdint.h>
#include "../../include/gbmw.h"

#if defined(__CUDACC__)
#define GBMW_HD __host__ __device__ __forceinline__
#else
#define GBMW_HD static inline
#endif

namespace gbmw {

GBMW_HD double py_max(double a, double b) { return (b > a) ? b : a; }

struct StratDeg {
    int32_t dp, sdp, tp;   // products of the per-paradigm level degrees
    int32_t data;          // dp * sdp  (strategies.py:55-58)
    int32_t ckpt, pp;
};

GBMW_HD StratDeg strat_degrees(const gbmw_strategy &s) {
    StratDeg d;
    d.dp = d.sdp = d.tp = 1;
    for (int l = 0; l < s.n_levels; ++l) {
        if (s.paradigm[l] == GBMW_DP) d.dp *= s.degree[l];
        else if (s.paradigm[l] == GBMW_SDP) d.sdp *= s.degree[l];
        else d.tp *= s.degree[l];
    }
    d.data = d.dp * d.sdp;
    d.ckpt = s.ckpt;
    d.pp = s.pp_degree;
    return d;
}

struct Comm { double grad, fwd_act, bwd_act, ckpt_act; };

// costs.py:57-67 level_bandwidth + costs.py:98-129 comm_breakdown
GBMW_HD Comm comm_breakdown(const gbmw_layer &L, const gbmw_strategy &s, const StratDeg &d,
                            int64_t micro, const gbmw_env &env) {
    const double shard = (double)L.param_bytes / (double)d.tp;
    const double samples = (double)micro / (double)d.data;
    const double act = (double)L.bnd_bytes_per_sample * samples;
    Comm c{0.0, 0.0, 0.0, 0.0};
    for (int idx = 0; idx < s.n_levels; ++idx) {
        int64_t span = 1;
        for (int k = idx; k < s.n_levels; ++k) span *= s.degree[k];
        const double tier = (span <= env.island_size) ? env.intra_island_bw : env.inter_island_bw;
        const double bw = tier * env.collective_efficiency;
        const int32_t deg = s.degree[idx];
        const double ring = (double)(deg - 1) / (double)deg;
        if (s.paradigm[idx] == GBMW_DP) {
            c.grad = c.grad + ((2.0 * ring) * shard) / bw;
        } else if (s.paradigm[idx] == GBMW_SDP) {
            c.grad = c.grad + ((3.0 * ring) * shard) / bw;
        } else {
            const double per_pass = ((2.0 * ring) * act) / bw;
            c.fwd_act = c.fwd_act + per_pass;
            c.bwd_act = c.bwd_act + per_pass;
            if (s.ckpt) c.ckpt_act = c.ckpt_act + per_pass;
        }
    }
    return c;
}

// costs.py:168-188 _layer_times -> (time with gradient sync, time without)
GBMW_HD void layer_times(const gbmw_layer &L, const gbmw_strategy &s, const StratDeg &d,
                         int64_t micro, const gbmw_env &env, double *t, double *t_ns) {
    const int64_t samples = micro / d.data;
    const double fwd_c = ((double)samples * L.fwd_time) / (double)d.tp;
    const double bwd_c = fwd_c * env.bwd_fwd_ratio;
    const Comm c = comm_breakdown(L, s, d, micro, env);
    const double forward = fwd_c + c.fwd_act;
    double tail = c.bwd_act;
    if (d.ckpt) tail = tail + (fwd_c + c.ckpt_act);
    // costs.py:50-54 overlap(a, b, slowdown)
    double ov;
    if (bwd_c > 0.0 && c.grad > 0.0) ov = py_max(bwd_c, c.grad) * env.overlap_slowdown;
    else ov = bwd_c + c.grad;
    *t = (forward + ov) + tail;
    *t_ns = (forward + bwd_c) + tail;
}

struct Mem { double o_f, o_b, o_ms; };

// costs.py:191-228 layer_memory.  O_f under ckpt is a Python int (stash * bnd_mb);
// the caller guarantees it is < 2^53 so the conversion below is exact.
GBMW_HD Mem layer_memory(const gbmw_layer &L, const StratDeg &d, int64_t micro,
                         int32_t stage_index, int32_t n_micro, double ms_mult) {
    const int64_t samples = micro / d.data;
    Mem m;
    m.o_ms = ((double)L.param_bytes * ms_mult) / (double)((int64_t)d.tp * d.sdp);
    const double frac = L.tp_act_replication_fraction;
    const double ips = (double)L.int_bytes_per_sample * (frac + ((1.0 - frac) / (double)d.tp));
    const int64_t bnd_mb = L.bnd_bytes_per_sample * samples;
    const double int_mb = ips * (double)samples;
    int64_t stash = (int64_t)d.pp - stage_index + 1;
    if ((int64_t)n_micro < stash) stash = n_micro;
    if (d.ckpt) {
        m.o_f = (double)(stash * bnd_mb);
        m.o_b = int_mb;
    } else {
        m.o_f = (double)stash * ((double)bnd_mb + int_mb);
        m.o_b = 0.0;
    }
    return m;
}

// costs.py:252-277 transform_cost between (data, tp) classes; bnd = first layer of unit
GBMW_HD double transform_cost(int64_t bnd, int32_t d_src, int32_t t_src, int32_t d_dst,
                              int32_t t_dst, int64_t micro, double intra_bw) {
    if (d_src == d_dst && t_src == t_dst) return 0.0;
    const int64_t total = bnd * micro;
    const double required = (double)total / (double)((int64_t)d_dst * t_dst);
    const int64_t dm = d_src > d_dst ? d_src : d_dst;
    const int64_t tm = t_src > t_dst ? t_src : t_dst;
    const double local = (double)total / (double)(dm * tm);
    const double diff = required - local;
    const double moved = (0.0 > diff) ? 0.0 : diff;
    return moved / intra_bw;
}

// costs.py:280-286 stage_p2p_time
GBMW_HD double stage_p2p_time(int64_t bnd, int64_t micro, int32_t pp, const gbmw_env &env) {
    if (pp <= 1) return 0.0;
    const int64_t group = env.n_devices / pp;
    const double bw = (group >= env.island_size) ? env.inter_island_bw : env.intra_island_bw;
    return (double)(bnd * micro) / bw;
}

}  // namespace gbmw
