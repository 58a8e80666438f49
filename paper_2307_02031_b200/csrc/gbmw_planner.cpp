// gbmw_planner.cpp — host-side pipeline-partition logic around the search
// (parapilot/balance.py), native so the Algorithm-1/2 drivers are not bound by
// Python loops: stage costs of a partition, the memory/time-balanced seed
// partitions (greedy prefix split + hill climbing) and the seed-strategy choice.
//
// Bit-exactness: the reference folds stage/pipeline sums with Python's built-in
// sum(), which since CPython 3.12 is Neumaier-compensated for floats (started from
// the int 0); py_sum() reproduces that algorithm (Objects/bltinmodule.c,
// builtin_sum_impl).  Everything else is the cost model of costmodel.cuh.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>
#include <thread>
#include <atomic>

#include "../../include/gbmw.h"
#include "costmodel.cuh"

using namespace gbmw;

namespace {

thread_local std::string g_perr;

int perr(int code, const std::string &m) {
    g_perr = m;
    return code;
}

// Which sum() the host interpreter runs: 1 = CPython >= 3.12 (Neumaier-compensated),
// 0 = CPython <= 3.11 (plain left-to-right addition).  Set once at import by the Python
// package (gbmw_set_sum_semantics) from sys.version_info.
std::atomic<int> g_neumaier{1};

// CPython >= 3.12 sum() of a float sequence with start 0 (int): the first item is
// taken as is (0 + x == x), the rest are Neumaier-compensated.  Under the <= 3.11
// semantics the loop is plain addition (the compensation term stays 0).
double py_sum(const double *x, int n) {
    if (n <= 0) return 0.0;
    double f = x[0], c = 0.0;
    if (!g_neumaier.load(std::memory_order_relaxed)) {
        for (int i = 1; i < n; ++i) f = f + x[i];
        return f;
    }
    for (int i = 1; i < n; ++i) {
        const double t = f + x[i];
        if (std::fabs(f) >= std::fabs(x[i])) c += (f - t) + x[i];
        else c += (x[i] - t) + f;
        f = t;
    }
    if (c != 0.0 && std::isfinite(c)) f += c;
    return f;
}

struct StageCostOut { double t, ns, peak; };

// costs.py:322-352 stage_cost over layers[a, b) with per-layer strategies
int stage_cost_range(const gbmw_layer *layers, const gbmw_strategy *strats, int a, int b, int stage_index,
                     const gbmw_env &env, int64_t micro, int32_t n_micro, StageCostOut *out) {
    double t_sum = 0.0, ns_sum = 0.0, ms = 0.0, pf = 0.0, peak = 0.0;
    for (int l = a; l < b; ++l) {
        const gbmw_strategy &s = strats[l];
        const StratDeg d = strat_degrees(s);
        if (micro % d.data != 0) return perr(GBMW_EMICRO, "micro-batch not divisible by the DP*SDP degree");
        if (stage_index < 1 || stage_index > s.pp_degree)
            return perr(GBMW_ESTAGE, "stage_index " + std::to_string(stage_index) + " out of range 1.." +
                                         std::to_string(s.pp_degree));
        if (n_micro < 1) return perr(GBMW_ESTAGE, "n_micro must be >= 1, got " + std::to_string(n_micro));
        double t, tns;
        layer_times(layers[l], s, d, micro, env, &t, &tns);
        double r = 0.0;
        if (l > a) {
            const StratDeg pd = strat_degrees(strats[l - 1]);
            r = transform_cost(layers[l].bnd_bytes_per_sample, pd.data, pd.tp, d.data, d.tp, micro,
                               env.intra_island_bw);
        }
        t_sum = t_sum + (t + r);
        ns_sum = ns_sum + (tns + r);
    }
    if (stage_index > 1) {
        const double p2p = stage_p2p_time(layers[a].bnd_bytes_per_sample, micro, strats[a].pp_degree, env);
        t_sum = t_sum + p2p;
        ns_sum = ns_sum + p2p;
    }
    for (int l = a; l < b; ++l) {
        const StratDeg d = strat_degrees(strats[l]);
        const Mem m = layer_memory(layers[l], d, micro, stage_index, n_micro, env.ms_bytes_per_param_byte);
        ms = ms + m.o_ms;
        pf = pf + m.o_f;
        peak = py_max(peak, pf + m.o_b);
    }
    out->t = t_sum;
    out->ns = ns_sum;
    out->peak = peak + ms;
    return GBMW_OK;
}

// balance.py:98-119 evaluate_partition
int partition_costs(const gbmw_layer *layers, const gbmw_strategy *strats, const int32_t *sizes, int n_stages,
                    const gbmw_env &env, int64_t micro, int32_t n_micro, StageCostOut *out) {
    int a = 0;
    for (int s = 0; s < n_stages; ++s) {
        const int rc = stage_cost_range(layers, strats, a, a + sizes[s], s + 1, env, micro, n_micro, &out[s]);
        if (rc) return rc;
        a += sizes[s];
    }
    return GBMW_OK;
}

// balance.py:62-77 balance_degrees -> alpha_t or alpha_m
int balance_alpha(const StageCostOut *sc, int n, bool memory, double *alpha) {
    thread_local std::vector<double> t, m;              // reused: called for every hill-climb move
    t.resize(n);
    m.resize(n);
    double tmax = 0.0, mmax = 0.0;
    for (int i = 0; i < n; ++i) {
        t[i] = sc[i].t;
        m[i] = sc[i].peak;
        if (i == 0 || t[i] > tmax) tmax = t[i];
        if (i == 0 || m[i] > mmax) mmax = m[i];
    }
    const double tt = py_sum(t.data(), n), tm = py_sum(m.data(), n);
    if (tt <= 0 || tm <= 0) return perr(GBMW_EINVAL, "stage totals must be positive to define balance degrees");
    *alpha = memory ? 1.0 - mmax / tm : 1.0 - tmax / tt;
    return GBMW_OK;
}

// balance_alpha of a partition that differs from the current one only in stages b, b+1
// (a hill-climb move), with the current partition's Neumaier prefix states and prefix /
// suffix maxima cached: the sums resume at b with exactly py_sum's operations, so the
// result is bit-identical to balance_alpha on the whole moved partition.
struct AlphaCache {
    int n = 0;
    std::vector<double> ft, ct, fm, cm, pmt, pmm, smt, smm;   // state after element i; max of [0, i] / [i, n)

    void build(const StageCostOut *sc, int n_) {
        n = n_;
        ft.resize(n); ct.resize(n); fm.resize(n); cm.resize(n);
        pmt.resize(n); pmm.resize(n); smt.resize(n + 1); smm.resize(n + 1);
        double f1 = sc[0].t, c1 = 0.0, f2 = sc[0].peak, c2 = 0.0;
        ft[0] = f1; ct[0] = c1; fm[0] = f2; cm[0] = c2;
        for (int i = 1; i < n; ++i) {
            step(f1, c1, sc[i].t);
            step(f2, c2, sc[i].peak);
            ft[i] = f1; ct[i] = c1; fm[i] = f2; cm[i] = c2;
        }
        pmt[0] = sc[0].t; pmm[0] = sc[0].peak;
        for (int i = 1; i < n; ++i) {
            pmt[i] = sc[i].t > pmt[i - 1] ? sc[i].t : pmt[i - 1];
            pmm[i] = sc[i].peak > pmm[i - 1] ? sc[i].peak : pmm[i - 1];
        }
        smt[n] = -INFINITY; smm[n] = -INFINITY;
        for (int i = n - 1; i >= 0; --i) {
            smt[i] = sc[i].t > smt[i + 1] ? sc[i].t : smt[i + 1];
            smm[i] = sc[i].peak > smm[i + 1] ? sc[i].peak : smm[i + 1];
        }
    }

    static void step(double &f, double &c, double x) {           // py_sum's loop body
        if (!g_neumaier.load(std::memory_order_relaxed)) { f = f + x; return; }
        const double t = f + x;
        if (std::fabs(f) >= std::fabs(x)) c += (f - t) + x;
        else c += (x - t) + f;
        f = t;
    }
    static double finish(double f, double c) { return (c != 0.0 && std::isfinite(c)) ? f + c : f; }

    // The objective's exact total of the current partition (py_sum of its stage values).
    double total(bool memory) const { return memory ? finish(fm[n - 1], cm[n - 1]) : finish(ft[n - 1], ct[n - 1]); }

    // Can the move (stages b, b + 1 -> n0, n1) beat `thresh`?  A bound, no exact fold: the
    // move's total is approximated from the current exact total; the approximation, the
    // exact py_sum of the moved partition and the current total all lie within a few ulps
    // of the true sums, so |alpha_approx - alpha| <= err below (with a wide margin), and a
    // move whose approximate alpha plus err does not exceed `thresh` cannot be accepted.
    bool may_beat(const StageCostOut *sc, int b, const StageCostOut &n0, const StageCostOut &n1, bool memory,
                  double cur_total, double thresh) const {
        const double x0 = memory ? n0.peak : n0.t, x1 = memory ? n1.peak : n1.t;
        const double o0 = memory ? sc[b].peak : sc[b].t, o1 = memory ? sc[b + 1].peak : sc[b + 1].t;
        double mx = b > 0 ? (memory ? pmm[b - 1] : pmt[b - 1]) : x0;
        if (x0 > mx) mx = x0;
        if (x1 > mx) mx = x1;
        const double suf = memory ? smm[b + 2] : smt[b + 2];
        if (suf > mx) mx = suf;
        const double apx = ((cur_total - o0) - o1) + x0 + x1;
        if (!(mx > 0.0) || !(apx > 0.0) || !std::isfinite(apx)) return true;     // let the exact path decide
        const double eps = 2.220446049250313e-16;
        const double err = 64.0 * eps * (cur_total + apx + x0 + x1) / apx + 8.0 * eps;
        return (1.0 - mx / apx) + err > thresh;
    }

    // sc: the current partition's costs; n0, n1: the new costs of stages b, b + 1
    int move_alpha(const StageCostOut *sc, int b, const StageCostOut &n0, const StageCostOut &n1, bool memory,
                   double *alpha) const {
        double f1, c1, f2, c2;
        if (b == 0) { f1 = n0.t; c1 = 0.0; f2 = n0.peak; c2 = 0.0; }
        else {
            f1 = ft[b - 1]; c1 = ct[b - 1]; f2 = fm[b - 1]; c2 = cm[b - 1];
            step(f1, c1, n0.t); step(f2, c2, n0.peak);
        }
        step(f1, c1, n1.t); step(f2, c2, n1.peak);
        for (int i = b + 2; i < n; ++i) { step(f1, c1, sc[i].t); step(f2, c2, sc[i].peak); }
        const double tt = finish(f1, c1), tm = finish(f2, c2);
        double tmax = b > 0 ? pmt[b - 1] : n0.t, mmax = b > 0 ? pmm[b - 1] : n0.peak;
        if (n0.t > tmax) tmax = n0.t;
        if (n0.peak > mmax) mmax = n0.peak;
        if (n1.t > tmax) tmax = n1.t;
        if (n1.peak > mmax) mmax = n1.peak;
        if (smt[b + 2] > tmax) tmax = smt[b + 2];
        if (smm[b + 2] > mmax) mmax = smm[b + 2];
        if (tt <= 0 || tm <= 0) return perr(GBMW_EINVAL, "stage totals must be positive to define balance degrees");
        *alpha = memory ? 1.0 - mmax / tm : 1.0 - tmax / tt;
        return GBMW_OK;
    }
};

// balance.py:122-139 _greedy_split
std::vector<int32_t> greedy_split(const std::vector<double> &w, int S) {
    const int n = (int)w.size();
    const double total = py_sum(w.data(), n);
    std::vector<int32_t> sizes;
    int start = 0;
    double acc = 0.0;
    for (int stage = 0; stage < S - 1; ++stage) {
        const int remaining = S - stage - 1;
        const double target = (total * (double)(stage + 1)) / (double)S;
        int end = start;
        while (end < n - remaining && (acc + w[end] <= target || end < start + 1)) {
            acc += w[end];
            ++end;
        }
        sizes.push_back(end - start);
        start = end;
    }
    sizes.push_back(n - start);
    return sizes;
}

// The partition-independent pieces of costs.stage_cost (costs.py:322-352) for a fixed
// per-layer strategy list: layer times, transform cost from the previous layer, model
// states, O_b, and O_f per stage index (the 1F1B stash depends on it), p2p per stage
// start.  stage() folds them in exactly the reference's order.
struct PartitionTables {
    int L = 0, S = 0;
    std::vector<double> t, tns, r, ob, oms, p2p, of;   // of: L x S (stage index 1..S)

    int build(const gbmw_layer *layers, int n_layers, const gbmw_strategy *strats, int n_stages,
              const gbmw_env &env, int64_t micro, int32_t n_micro) {
        L = n_layers;
        S = n_stages;
        t.resize(L); tns.resize(L); r.assign(L, 0.0); ob.resize(L); oms.resize(L); p2p.resize(L);
        of.resize((size_t)L * S);
        if (n_micro < 1) return perr(GBMW_ESTAGE, "n_micro must be >= 1, got " + std::to_string(n_micro));
        for (int l = 0; l < L; ++l) {
            const gbmw_strategy &s = strats[l];
            const StratDeg d = strat_degrees(s);
            if (micro % d.data != 0) return perr(GBMW_EMICRO, "micro-batch not divisible by the DP*SDP degree");
            if (S > s.pp_degree)
                return perr(GBMW_ESTAGE, "stage_index " + std::to_string(s.pp_degree + 1) + " out of range 1.." +
                                             std::to_string(s.pp_degree));
            layer_times(layers[l], s, d, micro, env, &t[l], &tns[l]);
            if (l > 0) {
                const StratDeg pd = strat_degrees(strats[l - 1]);
                r[l] = transform_cost(layers[l].bnd_bytes_per_sample, pd.data, pd.tp, d.data, d.tp, micro,
                                      env.intra_island_bw);
            }
            p2p[l] = stage_p2p_time(layers[l].bnd_bytes_per_sample, micro, s.pp_degree, env);
            // layer_memory at every stage index: only the 1F1B stash differs, so the
            // stage-independent factor is formed once, with layer_memory's own operations
            const Mem m1 = layer_memory(layers[l], d, micro, 1, n_micro, env.ms_bytes_per_param_byte);
            ob[l] = m1.o_b;
            oms[l] = m1.o_ms;
            const int64_t samples = micro / d.data;
            const int64_t bnd_mb = layers[l].bnd_bytes_per_sample * samples;
            const double frac = layers[l].tp_act_replication_fraction;
            const double ips = (double)layers[l].int_bytes_per_sample * (frac + ((1.0 - frac) / (double)d.tp));
            const double x = (double)bnd_mb + ips * (double)samples;
            for (int st = 1; st <= S; ++st) {
                int64_t stash = (int64_t)d.pp - st + 1;
                if ((int64_t)n_micro < stash) stash = n_micro;
                of[(size_t)l * S + (st - 1)] = d.ckpt ? (double)(stash * bnd_mb) : (double)stash * x;
            }
        }
        return GBMW_OK;
    }

    StageCostOut stage(int a, int b, int stage_index) const {
        double ts = 0.0, ns = 0.0;
        for (int l = a; l < b; ++l) {
            const double rr = (l == a) ? 0.0 : r[l];
            ts = ts + (t[l] + rr);
            ns = ns + (tns[l] + rr);
        }
        if (stage_index > 1) {
            ts = ts + p2p[a];
            ns = ns + p2p[a];
        }
        double ms = 0.0, pf = 0.0, peak = 0.0;
        for (int l = a; l < b; ++l) {
            ms = ms + oms[l];
            pf = pf + of[(size_t)l * S + (stage_index - 1)];
            peak = py_max(peak, pf + ob[l]);
        }
        StageCostOut o;
        o.t = ts; o.ns = ns; o.peak = peak + ms;
        return o;
    }

    void costs(const std::vector<int32_t> &sizes, StageCostOut *out) const {
        for (int s = 0, a = 0; s < S; ++s) {
            out[s] = stage(a, a + sizes[s], s + 1);
            a += sizes[s];
        }
    }
};

// balance.py:180-212 _init_partition (greedy split + hill climbing on alpha)
int init_partition(const gbmw_layer *layers, int n_layers, const gbmw_strategy *seeds, int S,
                   const gbmw_env &env, int64_t micro, int32_t n_micro, bool memory, std::vector<int32_t> &out) {
    if (S > n_layers)
        return perr(GBMW_EINVAL, "cannot split " + std::to_string(n_layers) + " layers into " + std::to_string(S) +
                                     " pipeline stages");
    std::vector<double> w(n_layers);
    for (int l = 0; l < n_layers; ++l) {
        const StratDeg d = strat_degrees(seeds[l]);
        if (micro % d.data != 0) return perr(GBMW_EMICRO, "micro-batch not divisible by the seed's DP*SDP degree");
        if (memory) {
            const Mem m = layer_memory(layers[l], d, micro, seeds[l].pp_degree, n_micro, env.ms_bytes_per_param_byte);
            w[l] = m.o_f + m.o_ms;
        } else {
            double t, tns;
            layer_times(layers[l], seeds[l], d, micro, env, &t, &tns);
            w[l] = t;
        }
    }
    // Per-layer pieces of stage_cost are independent of the partition except through
    // the stage index (stash, p2p) and the stage start (no transform cost): tabulate
    // them once, then a stage's cost is an O(stage length) fold in the reference's
    // order, and a neighbour move re-costs only the two stages it changes.
    PartitionTables tab;
    int rc = tab.build(layers, n_layers, seeds, S, env, micro, n_micro);
    if (rc) return rc;
    std::vector<int32_t> best = greedy_split(w, S);
    std::vector<StageCostOut> sc(S);
    tab.costs(best, sc.data());
    double best_score;
    if ((rc = balance_alpha(sc.data(), S, memory, &best_score))) return rc;
    // balance.py:160-177 _hill_climb, max_rounds = 2 L; neighbour order of _neighbor_moves
    std::vector<int32_t> starts(S);
    AlphaCache ac;
    for (int round = 0; round < 2 * n_layers; ++round) {
        bool found = false;
        std::vector<int32_t> round_best;
        double round_score = best_score;
        for (int s = 0, a = 0; s < S; ++s) { starts[s] = a; a += best[s]; }
        ac.build(sc.data(), S);
        const double cur_total = ac.total(memory);
        for (int b = 0; b + 1 < S; ++b) {
            for (int dir = 0; dir < 2; ++dir) {
                if (dir == 0 ? best[b] <= 1 : best[b + 1] <= 1) continue;
                const int mid = starts[b] + best[b] + (dir == 0 ? -1 : 1);   // new boundary
                const StageCostOut n0 = tab.stage(starts[b], mid, b + 1);       // the two re-costed stages
                const StageCostOut n1 = tab.stage(mid, starts[b + 1] + best[b + 1], b + 2);
                double s;
                if (!ac.may_beat(sc.data(), b, n0, n1, memory, cur_total, round_score + 1e-15)) continue;
                if ((rc = ac.move_alpha(sc.data(), b, n0, n1, memory, &s))) return rc;
                if (s > round_score + 1e-15) {
                    round_best = best;
                    if (dir == 0) { round_best[b] -= 1; round_best[b + 1] += 1; }
                    else { round_best[b] += 1; round_best[b + 1] -= 1; }
                    round_score = s;
                    found = true;
                }
            }
        }
        if (!found) break;
        best = round_best;
        best_score = round_score;
        tab.costs(best, sc.data());
    }
    out = best;
    return GBMW_OK;
}

gbmw_strategy make_seed(int64_t pp, int64_t group, int paradigm) {
    gbmw_strategy s;
    std::memset(&s, 0, sizeof(s));
    s.pp_degree = (int32_t)pp;
    if (group > 1) {
        s.n_levels = 1;
        s.paradigm[0] = paradigm;
        s.degree[0] = (int32_t)group;
    }
    return s;
}

}  // namespace

extern "C" const char *gbmw_planner_last_error(void) { return g_perr.c_str(); }

extern "C" int gbmw_partition_costs(const gbmw_layer *layers, int32_t n_layers, const gbmw_strategy *per_layer,
                                    const int32_t *sizes, int32_t n_stages, const gbmw_env *env, int64_t micro_batch,
                                    int32_t n_micro, double *out) {
    if (!layers || !per_layer || !sizes || !env || !out || n_stages < 1) return perr(GBMW_EINVAL, "bad arguments");
    int total = 0;
    for (int s = 0; s < n_stages; ++s) {
        if (sizes[s] < 1) return perr(GBMW_EINVAL, "every stage needs at least one layer");
        total += sizes[s];
    }
    if (total != n_layers) return perr(GBMW_EINVAL, "partition does not cover the layers");
    std::vector<StageCostOut> sc(n_stages);
    const int rc = partition_costs(layers, per_layer, sizes, n_stages, *env, micro_batch, n_micro, sc.data());
    if (rc) return rc;
    for (int s = 0; s < n_stages; ++s) {
        out[3 * s] = sc[s].t;
        out[3 * s + 1] = sc[s].ns;
        out[3 * s + 2] = sc[s].peak;
    }
    return GBMW_OK;
}

extern "C" int gbmw_init_partition(const gbmw_layer *layers, int32_t n_layers, const gbmw_strategy *per_layer,
                                   int32_t n_stages, const gbmw_env *env, int64_t micro_batch, int32_t n_micro,
                                   int32_t objective, int32_t *out_sizes) {
    if (!layers || !per_layer || !env || !out_sizes || n_stages < 1) return perr(GBMW_EINVAL, "bad arguments");
    std::vector<int32_t> sizes;
    const int rc = init_partition(layers, n_layers, per_layer, n_stages, *env, micro_batch, n_micro, objective == 0,
                                  sizes);
    if (rc) return rc;
    std::memcpy(out_sizes, sizes.data(), sizeof(int32_t) * n_stages);
    return GBMW_OK;
}

extern "C" int gbmw_seed_for(const gbmw_layer *layers, int32_t n_layers, const gbmw_env *env, int64_t n_devices,
                             int64_t pp_degree, int64_t micro_batch, int32_t n_micro, double budget,
                             gbmw_strategy *out_seed, int32_t *out_sizes) {
    // balance.py:471-488 _seed_for (+ the memory-balanced partition of the chosen seed,
    // which galvatron_base recomputes identically, planner.py:251-253)
    if (!layers || !env || !out_seed || pp_degree < 1) return perr(GBMW_EINVAL, "bad arguments");
    const int64_t group = n_devices / pp_degree;
    std::vector<gbmw_strategy> cands;
    cands.push_back(make_seed(pp_degree, group, GBMW_DP));
    if (group > 1) {
        cands.push_back(make_seed(pp_degree, group, GBMW_SDP));
        cands.push_back(make_seed(pp_degree, group, GBMW_TP));
    }
    std::vector<gbmw_strategy> usable;
    for (const auto &s : cands)
        if (micro_batch % strat_degrees(s).data == 0) usable.push_back(s);
    if (usable.empty()) usable.push_back(cands.back());
    std::vector<gbmw_strategy> seeds(n_layers);
    std::vector<int32_t> sizes;
    std::vector<StageCostOut> sc(pp_degree);
    for (const auto &seed : usable) {
        for (auto &x : seeds) x = seed;
        int rc = init_partition(layers, n_layers, seeds.data(), (int)pp_degree, *env, micro_batch, n_micro, true, sizes);
        if (rc) return rc;
        rc = partition_costs(layers, seeds.data(), sizes.data(), (int)pp_degree, *env, micro_batch, n_micro, sc.data());
        if (rc) return rc;
        double mx = sc[0].peak;
        for (int s = 1; s < (int)pp_degree; ++s) mx = py_max(mx, sc[s].peak);
        if (mx <= budget) {
            *out_seed = seed;
            if (out_sizes) std::memcpy(out_sizes, sizes.data(), sizeof(int32_t) * pp_degree);
            return GBMW_OK;
        }
    }
    // nothing fits: the last candidate, whose memory-balanced partition the loop just computed
    *out_seed = usable.back();
    if (out_sizes) std::memcpy(out_sizes, sizes.data(), sizeof(int32_t) * pp_degree);
    return GBMW_OK;
}

extern "C" double gbmw_py_sum(const double *x, int32_t n) { return py_sum(x, n); }

extern "C" int gbmw_set_sum_semantics(int32_t neumaier) {
    g_neumaier.store(neumaier ? 1 : 0);
    return GBMW_OK;
}

extern "C" int gbmw_sum_semantics(void) { return g_neumaier.load(); }

// gbmw_seed_for for many (pp_degree, micro_batch, n_micro) cells of one model and cluster,
// host threads over the cells (galvatron_base seeds every (batch, degree) cell of a batch
// window this way, planner.py:250-253).  out_sizes: n_cells x max_stages, row i holds
// pp_degree[i] stage sizes.  Returns the first failing cell's status (its message in
// gbmw_planner_last_error of the calling thread).
extern "C" int gbmw_seed_partitions(const gbmw_layer *layers, int32_t n_layers, const gbmw_env *env,
                                    int64_t n_devices, int32_t n_cells, const int64_t *pp_degree,
                                    const int64_t *micro_batch, const int32_t *n_micro, double budget,
                                    int32_t max_stages, int32_t n_threads, int32_t *out_sizes) {
    if (!layers || !env || !pp_degree || !micro_batch || !n_micro || !out_sizes || n_cells < 0 || max_stages < 1)
        return perr(GBMW_EINVAL, "bad arguments");
    for (int i = 0; i < n_cells; ++i)
        if (pp_degree[i] < 1 || pp_degree[i] > max_stages) return perr(GBMW_EINVAL, "pp_degree out of range");
    std::atomic<int> next{0}, first_bad{n_cells};
    std::vector<int> codes(n_cells, GBMW_OK);
    std::vector<std::string> msgs(n_cells);
    auto work = [&]() {
        while (true) {
            const int i = next.fetch_add(1);
            if (i >= n_cells) return;
            gbmw_strategy seed;
            const int rc = gbmw_seed_for(layers, n_layers, env, n_devices, pp_degree[i], micro_batch[i], n_micro[i],
                                         budget, &seed, out_sizes + (size_t)i * max_stages);
            if (rc) {
                codes[i] = rc;
                msgs[i] = g_perr;
                int cur = first_bad.load();
                while (i < cur && !first_bad.compare_exchange_weak(cur, i)) {}
            }
        }
    };
    const int nt = std::max(1, std::min<int>(n_threads, n_cells));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto &th : pool) th.join();
    const int bad = first_bad.load();
    if (bad < n_cells) return perr(codes[bad], msgs[bad]);
    return GBMW_OK;
}

// gbmw_partition_costs for many (partition, per-layer strategies, micro-batch) items at once
// (Algorithm 2 re-costs the adjusted partition of every trajectory of a round,
// balance.py:420-424), on up to n_threads host threads.  per_layer: n_items rows of n_layers
// records; sizes: n_items rows of max_stages int32 (n_stages[i] used); out: n_items rows of
// 3 * max_stages doubles.  Errors: the first failing item's.
extern "C" int gbmw_partition_costs_batch(const gbmw_layer *layers, int32_t n_layers, const gbmw_strategy *per_layer,
                                          const int32_t *sizes, const int32_t *n_stages, int32_t max_stages,
                                          const gbmw_env *env, const int64_t *micro_batch, const int32_t *n_micro,
                                          int32_t n_items, int32_t n_threads, double *out) {
    if (!layers || !per_layer || !sizes || !n_stages || !env || !micro_batch || !n_micro || !out || n_items < 0 ||
        max_stages < 1 || n_layers < 1)
        return perr(GBMW_EINVAL, "bad arguments");
    std::atomic<int> next{0}, first_bad{n_items};
    std::vector<int> codes(n_items, GBMW_OK);
    std::vector<std::string> msgs(n_items);
    auto work = [&]() {
        while (true) {
            const int i = next.fetch_add(1);
            if (i >= n_items) return;
            const int rc = (n_stages[i] < 1 || n_stages[i] > max_stages)
                               ? perr(GBMW_EINVAL, "bad arguments")
                               : gbmw_partition_costs(layers, n_layers, per_layer + (size_t)i * n_layers,
                                                      sizes + (size_t)i * max_stages, n_stages[i], env,
                                                      micro_batch[i], n_micro[i], out + (size_t)i * 3 * max_stages);
            if (rc) {
                codes[i] = rc;
                msgs[i] = g_perr;
                int cur = first_bad.load();
                while (i < cur && !first_bad.compare_exchange_weak(cur, i)) {}
            }
        }
    };
    const int nt = std::max(1, std::min<int>(n_threads, n_items));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto &th : pool) th.join();
    const int bad = first_bad.load();
    if (bad < n_items) return perr(codes[bad], msgs[bad]);
    return GBMW_OK;
}

// The set-up of Algorithm 2's trajectories (balance.py:366-384 as _run_trajectories runs it):
// per (pp_degree, micro_batch, n_micro) cell the _seed_for strategy and its memory-balanced
// partition p0 (the trajectory's first partition), the time-balanced partition p_t of the
// same uniform seed list, and mem_ref = max stage peak of p_t (evaluate_partition), on up to
// n_threads host threads.  out_p0: n_cells rows of max_stages int32.  Errors: the first
// failing cell's, as the sequential set-up would raise it.
extern "C" int gbmw_bmw_setup(const gbmw_layer *layers, int32_t n_layers, const gbmw_env *env, int64_t n_devices,
                              int32_t n_cells, const int64_t *pp_degree, const int64_t *micro_batch,
                              const int32_t *n_micro, double budget, int32_t max_stages, int32_t n_threads,
                              int32_t *out_p0, double *out_mem_ref) {
    if (!layers || !env || !pp_degree || !micro_batch || !n_micro || !out_p0 || !out_mem_ref || n_cells < 0 ||
        max_stages < 1 || n_layers < 1)
        return perr(GBMW_EINVAL, "bad arguments");
    for (int i = 0; i < n_cells; ++i)
        if (pp_degree[i] < 1 || pp_degree[i] > max_stages || pp_degree[i] > n_layers)
            return perr(GBMW_EINVAL, "pp_degree out of range");
    std::atomic<int> next{0}, first_bad{n_cells};
    std::vector<int> codes(n_cells, GBMW_OK);
    std::vector<std::string> msgs(n_cells);
    auto work = [&]() {
        std::vector<gbmw_strategy> per_layer((size_t)n_layers);
        std::vector<int32_t> pt((size_t)max_stages);
        std::vector<double> costs(3 * (size_t)max_stages);
        while (true) {
            const int i = next.fetch_add(1);
            if (i >= n_cells) return;
            const int P = (int)pp_degree[i];
            gbmw_strategy seed;
            int rc = gbmw_seed_for(layers, n_layers, env, n_devices, P, micro_batch[i], n_micro[i], budget, &seed,
                                   out_p0 + (size_t)i * max_stages);
            if (!rc) {
                std::fill(per_layer.begin(), per_layer.end(), seed);
                rc = gbmw_init_partition(layers, n_layers, per_layer.data(), P, env, micro_batch[i], n_micro[i], 1,
                                         pt.data());
            }
            if (!rc)
                rc = gbmw_partition_costs(layers, n_layers, per_layer.data(), pt.data(), P, env, micro_batch[i],
                                          n_micro[i], costs.data());
            if (!rc) {
                double m = costs[2];                     // max(sc.peak_mem_bytes for sc in ...)
                for (int s = 1; s < P; ++s) m = costs[3 * s + 2] > m ? costs[3 * s + 2] : m;
                out_mem_ref[i] = m;
            } else {
                codes[i] = rc;
                msgs[i] = g_perr;
                int cur = first_bad.load();
                while (i < cur && !first_bad.compare_exchange_weak(cur, i)) {}
            }
        }
    };
    const int nt = std::max(1, std::min<int>(n_threads, n_cells));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto &th : pool) th.join();
    const int bad = first_bad.load();
    if (bad < n_cells) return perr(codes[bad], msgs[bad]);
    return GBMW_OK;
}
