/*
 * ref_oracle.c — CPU restatement of the reference search path.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs as the checker and the CPU baseline; it is
 * never linked into or called by the product (libgbmw).
 *
 * It restates, in plain C, the algorithm of the Python reference
 * (/root/reference/pkg/src/parapilot, "parapilot" 0.1.0) function by function:
 *
 *   or_enumerate        strategies.py:149-209  (_factor_sequences, build_decision_trees,
 *                                               enumerate_strategies, prune_dp_sdp)
 *   or_comm             costs.py:57-67, 98-129 (level_bandwidth, comm_breakdown)
 *   or_layer_times      costs.py:168-188       (_layer_times, overlap costs.py:50-54)
 *   or_layer_memory     costs.py:191-228
 *   or_transform        costs.py:252-277
 *   or_p2p              costs.py:280-286
 *   or_dp_search        dpsearch.py:89-227 with _run_dp_exact dpsearch.py:245-303:
 *                       full (unit, bucket, previous-strategy) DP with S^2 relaxations,
 *                       numpy min/argmax tie semantics, ranked sweep with per-candidate
 *                       reconstruct and E_all check (memory_footprint costs.py:289-319)
 *   or_stage_cost       costs.py:322-352
 *   or_brute_force      planner.py:354-449 (_compositions, brute_force_oracle): every
 *                       (P, m, partition, assignment) in the reference's loop order,
 *                       pipeline_cost costs.py:355-362 with CPython's sum()
 *
 * It deliberately does NOT use the device formulation (class reduction, parallel
 * sweep): it is the reference's own sequential algorithm, so agreement with the
 * product is evidence of parity, and its speed is the reference CPU baseline.
 * Pinned against golden vectors generated from the live reference
 * (tests/golden/make_golden.py writes the JSON fixtures next to it).
 *
 * Python-number semantics: int/int and int*float conversions happen where the
 * reference has them; build with -ffp-contract=off so nothing is fused.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/gbmw.h"
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_INF (1.0 / 0.0)

static double pymax(double a, double b) { return (b > a) ? b : a; }

/* ------------------------------------------------------------------ strategies */
typedef struct { int n; int f[3]; } Seq;

static void or_factor(int64_t rem, Seq cur, Seq *out, int *n_out) {
    if (rem == 1) { out[(*n_out)++] = cur; return; }
    if (cur.n >= 3) return;
    for (int64_t f = 2; f <= rem; f *= 2) {
        if (rem % f) continue;
        Seq nxt = cur;
        nxt.f[nxt.n++] = (int)f;
        or_factor(rem / f, nxt, out, n_out);
    }
}

static int or_key_cmp(const gbmw_strategy *a, const gbmw_strategy *b) {
    if (a->n_levels != b->n_levels) return a->n_levels < b->n_levels ? -1 : 1;
    for (int l = 0; l < a->n_levels; ++l)
        if (a->paradigm[l] != b->paradigm[l]) return a->paradigm[l] < b->paradigm[l] ? -1 : 1;
    for (int l = 0; l < a->n_levels; ++l)
        if (a->degree[l] != b->degree[l]) return a->degree[l] < b->degree[l] ? -1 : 1;
    if (a->ckpt != b->ckpt) return a->ckpt < b->ckpt ? -1 : 1;
    return 0;
}

/* returns count (or -1 on invalid args); writes at most cap */
int or_enumerate(int64_t n_devices, int64_t pp, int prune, gbmw_strategy *out, int cap) {
    if (n_devices < 1 || (n_devices & (n_devices - 1)) || pp < 1 || (pp & (pp - 1)) || pp > n_devices) return -1;
    const int64_t g = n_devices / pp;
    Seq seqs[4096];
    int ns = 0;
    Seq empty = {0, {0, 0, 0}};
    or_factor(g, empty, seqs, &ns);
    static const int p1[3][3] = {{0}, {1}, {2}};
    static const int p2[6][3] = {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {2, 0}, {2, 1}};
    static const int p3[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    gbmw_strategy *all = (gbmw_strategy *)calloc((size_t)ns * 12 + 2, sizeof(gbmw_strategy));
    int na = 0;
    for (int si = 0; si < ns; ++si) {
        const int k = seqs[si].n;
        const int np = k == 0 ? 1 : (k == 1 ? 3 : 6);
        for (int pi = 0; pi < np; ++pi)
            for (int ck = 0; ck <= 1; ++ck) {
                gbmw_strategy *s = &all[na++];
                s->pp_degree = (int32_t)pp;
                s->n_levels = k;
                for (int l = 0; l < k; ++l) {
                    s->paradigm[l] = k == 1 ? p1[pi][l] : (k == 2 ? p2[pi][l] : p3[pi][l]);
                    s->degree[l] = seqs[si].f[l];
                }
                s->ckpt = ck;
            }
    }
    /* stable insertion sort by sort_key (strategies.py:64-70, :199) */
    for (int i = 1; i < na; ++i) {
        gbmw_strategy x = all[i];
        int j = i - 1;
        while (j >= 0 && or_key_cmp(&all[j], &x) > 0) { all[j + 1] = all[j]; --j; }
        all[j + 1] = x;
    }
    int cnt = 0;
    for (int i = 0; i < na; ++i) {
        int dp = 1, sdp = 1;
        for (int l = 0; l < all[i].n_levels; ++l) {
            if (all[i].paradigm[l] == GBMW_DP) dp *= all[i].degree[l];
            if (all[i].paradigm[l] == GBMW_SDP) sdp *= all[i].degree[l];
        }
        if (prune && dp > 1 && sdp > 1) continue;
        if (out && cnt < cap) out[cnt] = all[i];
        ++cnt;
    }
    free(all);
    return cnt;
}

/* ------------------------------------------------------------------ cost model */
static int64_t deg_of(const gbmw_strategy *s, int paradigm) {
    int64_t d = 1;
    for (int l = 0; l < s->n_levels; ++l)
        if (s->paradigm[l] == paradigm) d *= s->degree[l];
    return d;
}
static int64_t data_deg(const gbmw_strategy *s) { return deg_of(s, GBMW_DP) * deg_of(s, GBMW_SDP); }

void or_comm(const gbmw_layer *L, const gbmw_strategy *s, int64_t micro, const gbmw_env *env, double out[4]) {
    double shard = (double)L->param_bytes / (double)deg_of(s, GBMW_TP);
    double samples = (double)micro / (double)data_deg(s);
    double act = (double)L->bnd_bytes_per_sample * samples;
    double grad = 0.0, fa = 0.0, ba = 0.0, ca = 0.0;
    for (int idx = 0; idx < s->n_levels; ++idx) {
        int64_t span = 1;
        for (int k = idx; k < s->n_levels; ++k) span *= s->degree[k];
        double bw = (span <= env->island_size ? env->intra_island_bw : env->inter_island_bw) *
                    env->collective_efficiency;
        double ring = (double)(s->degree[idx] - 1) / (double)s->degree[idx];
        if (s->paradigm[idx] == GBMW_DP) grad += 2.0 * ring * shard / bw;
        else if (s->paradigm[idx] == GBMW_SDP) grad += 3.0 * ring * shard / bw;
        else {
            double pp = 2.0 * ring * act / bw;
            fa += pp;
            ba += pp;
            if (s->ckpt) ca += pp;
        }
    }
    out[0] = grad; out[1] = fa; out[2] = ba; out[3] = ca;
}

void or_layer_times(const gbmw_layer *L, const gbmw_strategy *s, int64_t micro, const gbmw_env *env,
                    double *t, double *t_ns) {
    int64_t samples = micro / data_deg(s);
    double fwd = (double)samples * L->fwd_time / (double)deg_of(s, GBMW_TP);
    double bwd = fwd * env->bwd_fwd_ratio;
    double c[4];
    or_comm(L, s, micro, env, c);
    double forward = fwd + c[1];
    double tail = c[2];
    if (s->ckpt) tail += fwd + c[3];
    double ov = (bwd > 0.0 && c[0] > 0.0) ? pymax(bwd, c[0]) * env->overlap_slowdown : bwd + c[0];
    *t = forward + ov + tail;
    *t_ns = forward + bwd + tail;
}

void or_layer_memory(const gbmw_layer *L, const gbmw_strategy *s, int64_t micro, int stage, int n_micro,
                     double ms_mult, double out[3]) {
    int64_t samples = micro / data_deg(s);
    int64_t tp = deg_of(s, GBMW_TP);
    double o_ms = (double)L->param_bytes * ms_mult / (double)(tp * deg_of(s, GBMW_SDP));
    double frac = L->tp_act_replication_fraction;
    double ips = (double)L->int_bytes_per_sample * (frac + (1.0 - frac) / (double)tp);
    int64_t bnd_mb = L->bnd_bytes_per_sample * samples;
    double int_mb = ips * (double)samples;
    int64_t stash = s->pp_degree - stage + 1;
    if (n_micro < stash) stash = n_micro;
    if (s->ckpt) { out[0] = (double)(stash * bnd_mb); out[1] = int_mb; }
    else { out[0] = (double)stash * ((double)bnd_mb + int_mb); out[1] = 0.0; }
    out[2] = o_ms;
}

double or_transform(const gbmw_layer *L, const gbmw_strategy *prev, const gbmw_strategy *cur, int64_t micro,
                    const gbmw_env *env) {
    if (!prev) return 0.0;
    int64_t ds = data_deg(prev), ts = deg_of(prev, GBMW_TP), dd = data_deg(cur), td = deg_of(cur, GBMW_TP);
    if (ds == dd && ts == td) return 0.0;
    int64_t total = L->bnd_bytes_per_sample * micro;
    double required = (double)total / (double)(dd * td);
    double local = (double)total / (double)((ds > dd ? ds : dd) * (ts > td ? ts : td));
    double moved = pymax(required - local, 0.0);
    return moved / env->intra_island_bw;
}

double or_p2p(const gbmw_layer *first, int64_t micro, int pp, const gbmw_env *env) {
    if (pp <= 1) return 0.0;
    int64_t group = env->n_devices / pp;
    double bw = group >= env->island_size ? env->inter_island_bw : env->intra_island_bw;
    return (double)(first->bnd_bytes_per_sample * micro) / bw;
}

/* costs.py:322-352 over an explicit per-layer strategy list */
void or_stage_cost(const gbmw_layer *layers, const gbmw_strategy *const *strats, int n, int64_t micro,
                   const gbmw_env *env, int stage, int n_micro, double out[3]) {
    double t_sum = 0.0, ns_sum = 0.0, ms = 0.0, pf = 0.0, peak = 0.0;
    for (int l = 0; l < n; ++l) {
        double t, tns;
        or_layer_times(&layers[l], strats[l], micro, env, &t, &tns);
        double r = or_transform(&layers[l], l ? strats[l - 1] : NULL, strats[l], micro, env);
        t_sum += t + r;
        ns_sum += tns + r;
    }
    if (stage > 1) {
        double p2p = or_p2p(&layers[0], micro, strats[0]->pp_degree, env);
        t_sum += p2p;
        ns_sum += p2p;
    }
    for (int l = 0; l < n; ++l) {
        double m[3];
        or_layer_memory(&layers[l], strats[l], micro, stage, n_micro, env->ms_bytes_per_param_byte, m);
        ms += m[2];
        pf += m[0];
        peak = pymax(peak, pf + m[1]);
    }
    out[0] = t_sum; out[1] = ns_sum; out[2] = peak + ms;
}

/* ------------------------------------------------------------------ dp_search */
static int int_le_double(int64_t x, double y) {
    if (y != y) return 0;
    if (y >= 9.2233720368547758e18) return 1;
    if (y < -9.2233720368547758e18) return 0;
    return x <= (int64_t)floor(y);
}

typedef struct {
    const gbmw_layer *layers;    /* stage layers */
    int n_layers;
    const gbmw_strategy **cands; /* usable strategies */
    int S;
    int U;
    int *unit_first, *unit_count;   /* index into layers */
    int64_t micro, n_b, gran;
    double budget;
    int stage, n_micro;
    const gbmw_env *env;
    double *time_c, *ef, *ob;       /* U x S */
    int64_t *w;                     /* U x S */
    double *R;                      /* U x S x S */
    double *T, *F;                  /* n_e x S (final unit) */
    int16_t *par;                   /* U x n_e x S */
} DP;

static void reconstruct(const DP *d, int64_t e, int j, int *picks) {
    const int64_t n_e = d->n_b + 1;
    for (int u = d->U - 1; u >= 1; --u) {
        picks[u] = j;
        int parent = d->par[((int64_t)u * n_e + e) * d->S + j];
        e -= d->w[u * d->S + j];
        j = parent;
    }
    picks[0] = j;
}

static double plan_e_all(const DP *d, const int *picks) {
    double ms = 0.0, pf = 0.0, peak = 0.0;
    for (int u = 0; u < d->U; ++u)
        for (int r = 0; r < d->unit_count[u]; ++r) {
            double m[3];
            or_layer_memory(&d->layers[d->unit_first[u] + r], d->cands[picks[u]], d->micro, d->stage, d->n_micro,
                            d->env->ms_bytes_per_param_byte, m);
            ms += m[2];
            pf += m[0];
            peak = pymax(peak, pf + m[1]);
        }
    return peak + ms;
}

static int lex_lt(double t1, double f1, int j1, double t2, double f2, int j2) {
    if (t1 != t2) return t1 < t2;
    if (f1 != f2) return f1 < f2;
    return j1 < j2;
}

/*
 * _run_dp_collapsed (dpsearch.py:306-375) and its sweep (dpsearch.py:194-208 with
 * ranked_at = [(table[e], 0)] if finite): state (unit, bucket) only, one recorded
 * strategy per cell; the transform cost is charged against that recorded strategy.
 * _lex_pick (dpsearch.py:237-242) = first j minimising (cand, cand_f).
 */
static void approx_search(const DP *d, double safe_limit, double *frontier, int *picks, int *best_picks,
                          int *have_best, double *best_t, int64_t *best_e) {
    const int U = d->U, S = d->S;
    const int64_t n_b = d->n_b, n_e = n_b + 1;
    double *tab = (double *)malloc(sizeof(double) * n_e), *fwd = (double *)malloc(sizeof(double) * n_e);
    double *nt = (double *)malloc(sizeof(double) * n_e), *nf = (double *)malloc(sizeof(double) * n_e);
    int16_t *choice = (int16_t *)malloc(sizeof(int16_t) * (size_t)U * n_e);
    for (int u = 0; u < U; ++u) {
        const int16_t *prev = choice + (size_t)(u - 1) * n_e;
        int16_t *cur = choice + (size_t)u * n_e;
        const double *Ru = d->R + (size_t)u * S * S;
        for (int64_t e = 0; e < n_e; ++e) {
            double bt = OR_INF, bf = OR_INF;
            int bj = -1;
            for (int j = 0; j < S; ++j) {
                const int64_t w = d->w[u * S + j];
                if (w > n_b || e < w) continue;
                double c, f;
                if (u == 0) {
                    c = d->time_c[j]; f = d->ef[j];
                } else {
                    const int64_t src = e - w;
                    if (prev[src] < 0) continue;
                    c = (tab[src] + Ru[prev[src] * S + j]) + d->time_c[u * S + j];
                    f = fwd[src] + d->ef[u * S + j];
                }
                if (bj < 0 || c < bt || (c == bt && f < bf)) { bt = c; bf = f; bj = j; }
            }
            nt[e] = bt; nf[e] = bf; cur[e] = (int16_t)bj;
        }
        double *x = tab; tab = nt; nt = x;
        x = fwd; fwd = nf; nf = x;
    }
    for (int64_t e = 1; e <= n_b; ++e) {
        const double t = tab[e];
        if (frontier) frontier[e - 1] = (t < OR_INF) ? t : OR_INF;
        if (!(t < OR_INF)) continue;
        if (*have_best && t > *best_t) continue;
        int64_t ce = e;
        for (int u = U - 1; u >= 0; --u) {
            const int j = choice[(size_t)u * n_e + ce];
            picks[u] = j;
            ce -= d->w[u * S + j];
        }
        if (int_le_double(e * d->gran, safe_limit) || plan_e_all(d, picks) <= d->budget) {
            *have_best = 1; *best_t = t; *best_e = e;
            memcpy(best_picks, picks, sizeof(int) * U);
        }
    }
    free(tab); free(fwd); free(nt); free(nf); free(choice);
}

/*
 * One dp_search (dpsearch.py:89-227) on already-validated arguments.
 * plan: n_layers ints (index into the caller's strategy list), -1 if infeasible.
 * frontier (optional): n_b doubles.  stage (optional): stage_cost of the plan.
 * Returns 0, or -11 if the chosen plan exceeds the budget (reference assert).
 */
int or_dp_search(const gbmw_layer *layers, int n_layers, const gbmw_strategy *strats, int n_strats,
                 const gbmw_env *env, int64_t micro, int64_t gran, double budget, int64_t n_b, int stage,
                 int n_micro, int flags, double *out_time, double *out_efwd, int *out_feasible, int32_t *plan,
                 double *frontier, double *stage_out) {
    *out_time = OR_INF; *out_efwd = 0.0; *out_feasible = 0;
    for (int l = 0; l < n_layers; ++l) plan[l] = -1;
    if (stage_out) stage_out[0] = stage_out[1] = stage_out[2] = 0.0;
    DP d;
    memset(&d, 0, sizeof(d));
    int *cidx = (int *)malloc(sizeof(int) * (n_strats + 1));
    d.cands = (const gbmw_strategy **)malloc(sizeof(void *) * (n_strats + 1));
    for (int i = 0; i < n_strats; ++i)
        if (micro % data_deg(&strats[i]) == 0) { cidx[d.S] = i; d.cands[d.S++] = &strats[i]; }
    if (d.S == 0 || n_b == 0) { free(cidx); free(d.cands); return 0; }
    d.layers = layers; d.n_layers = n_layers; d.micro = micro; d.n_b = n_b; d.gran = gran; d.budget = budget;
    d.stage = stage; d.n_micro = n_micro; d.env = env;
    /* units (dpsearch.py:71-86) */
    d.unit_first = (int *)malloc(sizeof(int) * n_layers);
    d.unit_count = (int *)malloc(sizeof(int) * n_layers);
    for (int l = 0; l < n_layers; ++l) {
        if ((flags & GBMW_FUSE) && d.U > 0) {
            const gbmw_layer *a = &layers[d.unit_first[d.U - 1]], *b = &layers[l];
            if (a->kind_id == b->kind_id && a->param_bytes == b->param_bytes &&
                a->bnd_bytes_per_sample == b->bnd_bytes_per_sample &&
                a->int_bytes_per_sample == b->int_bytes_per_sample && a->fwd_time_raw == b->fwd_time_raw &&
                a->tp_act_replication_fraction == b->tp_act_replication_fraction) {
                d.unit_count[d.U - 1]++;
                continue;
            }
        }
        d.unit_first[d.U] = l; d.unit_count[d.U] = 1; d.U++;
    }
    const int U = d.U, S = d.S;
    const int64_t n_e = n_b + 1;
    /* cost tables (dpsearch.py:131-145) */
    d.time_c = (double *)malloc(sizeof(double) * U * S);
    d.ef = (double *)malloc(sizeof(double) * U * S);
    d.ob = (double *)malloc(sizeof(double) * U * S);
    d.w = (int64_t *)malloc(sizeof(int64_t) * U * S);
    d.R = (double *)malloc(sizeof(double) * (size_t)U * S * S);
    double b_up = 0.0;
    for (int u = 0; u < U; ++u) {
        const gbmw_layer *L = &layers[d.unit_first[u]];
        for (int j = 0; j < S; ++j) {
            double t, tns, m[3];
            or_layer_times(L, d.cands[j], micro, env, &t, &tns);
            or_layer_memory(L, d.cands[j], micro, stage, n_micro, env->ms_bytes_per_param_byte, m);
            d.time_c[u * S + j] = t * d.unit_count[u];
            d.ef[u * S + j] = (m[0] + m[2]) * d.unit_count[u];
            d.ob[u * S + j] = m[1];
            double wq = ceil((m[0] + m[2]) * d.unit_count[u] / (double)gran);
            int64_t w = wq > 4.0e18 ? (int64_t)4e18 : (int64_t)wq;
            d.w[u * S + j] = w < 0 ? 0 : w;
            b_up = pymax(b_up, m[1]);   /* ob.max(initial=0.0) */
            for (int i = 0; i < S; ++i)
                d.R[((size_t)u * S + i) * S + j] = or_transform(L, d.cands[i], d.cands[j], micro, env);
        }
    }
    const double safe_limit = budget - b_up;
    int *picks = (int *)malloc(sizeof(int) * U);
    int *best_picks = (int *)malloc(sizeof(int) * U);
    int have_best = 0;
    double best_t = OR_INF;
    int64_t best_e = 0;
    if (flags & GBMW_APPROX) {
        approx_search(&d, safe_limit, frontier, picks, best_picks, &have_best, &best_t, &best_e);
        goto done;
    }
    /* _run_dp_exact (dpsearch.py:251-282) */
    double *T = (double *)malloc(sizeof(double) * n_e * S), *F = (double *)malloc(sizeof(double) * n_e * S);
    double *T2 = (double *)malloc(sizeof(double) * n_e * S), *F2 = (double *)malloc(sizeof(double) * n_e * S);
    d.par = (int16_t *)calloc((size_t)U * n_e * S, sizeof(int16_t));
    for (int64_t x = 0; x < n_e * S; ++x) { T[x] = OR_INF; F[x] = OR_INF; }
    for (int j = 0; j < S; ++j) {
        int64_t w = d.w[j];
        if (w > n_b) continue;
        for (int64_t e = w; e < n_e; ++e) { T[e * S + j] = d.time_c[j]; F[e * S + j] = d.ef[j]; }
    }
    for (int u = 1; u < U; ++u) {
        for (int64_t x = 0; x < n_e * S; ++x) { T2[x] = OR_INF; F2[x] = OR_INF; }
        for (int j = 0; j < S; ++j) {
            int64_t w = d.w[u * S + j];
            if (w > n_b) continue;
            const double *Rj = d.R + (size_t)u * S * S;
            for (int64_t r = 0; r < n_e - w; ++r) {
                const double *trow = T + r * S, *frow = F + r * S;
                /* numpy: t_min = cand.min(); mask = cand == t_min; f_min over mask; first index */
                double tmin = OR_INF;
                for (int i = 0; i < S; ++i) {
                    double c = trow[i] + Rj[i * S + j];
                    if (c < tmin) tmin = c;
                }
                double fmin = OR_INF;
                for (int i = 0; i < S; ++i)
                    if (trow[i] + Rj[i * S + j] == tmin && frow[i] < fmin) fmin = frow[i];
                int parent = 0;
                for (int i = 0; i < S; ++i)
                    if (trow[i] + Rj[i * S + j] == tmin && frow[i] == fmin) { parent = i; break; }
                T2[(r + w) * S + j] = tmin + d.time_c[u * S + j];
                F2[(r + w) * S + j] = frow[parent] + d.ef[u * S + j];
                d.par[((int64_t)u * n_e + r + w) * S + j] = (int16_t)parent;
            }
        }
        double *tmp = T; T = T2; T2 = tmp;
        tmp = F; F = F2; F2 = tmp;
    }
    /* E_fwd sweep (dpsearch.py:194-208) */
    char *tried = (char *)malloc(S);
    for (int64_t e = 1; e <= n_b; ++e) {
        const double *trow = T + e * S, *frow = F + e * S;
        memset(tried, 0, S);
        int first = 1;
        for (;;) {   /* walk candidates in sorted (T, F, j) order */
            int j = -1;
            for (int c = 0; c < S; ++c) {
                if (tried[c] || !(trow[c] < OR_INF)) continue;
                if (j < 0 || lex_lt(trow[c], frow[c], c, trow[j], frow[j], j)) j = c;
            }
            if (first && frontier) frontier[e - 1] = (j >= 0) ? trow[j] : OR_INF;
            first = 0;
            if (j < 0) break;
            tried[j] = 1;
            if (have_best && trow[j] > best_t) break;
            reconstruct(&d, e, j, picks);
            int fits = int_le_double(e * gran, safe_limit) || plan_e_all(&d, picks) <= budget;
            if (fits) {
                have_best = 1; best_t = trow[j]; best_e = e;
                memcpy(best_picks, picks, sizeof(int) * U);
                break;
            }
        }
    }
    free(tried);
    free(T); free(F); free(T2); free(F2); free(d.par);
done:;
    int rc = 0;
    if (have_best) {
        double e_all = plan_e_all(&d, best_picks);
        if (!(e_all <= budget)) rc = GBMW_EINTERNAL;
        *out_time = best_t; *out_efwd = (double)(best_e * gran); *out_feasible = 1;
        const gbmw_strategy **ls = (const gbmw_strategy **)malloc(sizeof(void *) * n_layers);
        int l = 0;
        for (int u = 0; u < U; ++u)
            for (int r = 0; r < d.unit_count[u]; ++r, ++l) { plan[l] = cidx[best_picks[u]]; ls[l] = d.cands[best_picks[u]]; }
        if (stage_out) or_stage_cost(layers, ls, n_layers, micro, env, stage, n_micro, stage_out);
        free(ls);
    }
    free(picks); free(best_picks);
    free(d.time_c); free(d.ef); free(d.ob); free(d.w); free(d.R);
    free(d.unit_first); free(d.unit_count); free(cidx); free(d.cands);
    return rc;
}

/*
 * Batched driver over the product's input format (gbmw_problem etc.), OpenMP
 * parallel over problems (dynamic schedule).  Infeasible / argument-error
 * handling mirrors dpsearch.py:103-121 as status codes.  Returns #threads used.
 */
int or_search_many(const gbmw_layer *layers, const gbmw_strategy *strats, const gbmw_env *envs,
                   const gbmw_problem *probs, int64_t n, gbmw_result *res, int32_t *plans, double *frontier,
                   int n_threads) {
    int64_t *plan_off = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    int64_t *front_off = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    int64_t po = 0, fo = 0;
    for (int64_t i = 0; i < n; ++i) {
        plan_off[i] = po; po += probs[i].n_layers > 0 ? probs[i].n_layers : 0;
        front_off[i] = -1;
        if (probs[i].flags & GBMW_FRONTIER) { front_off[i] = fo; fo += probs[i].n_buckets; }
    }
    int used = 1;
#pragma omp parallel num_threads(n_threads > 0 ? n_threads : 1)
    {
#pragma omp single
        {
#ifdef _OPENMP
            used = omp_get_num_threads();
#endif
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < n; ++i) {
            const gbmw_problem *p = &probs[i];
            gbmw_result *r = &res[i];
            memset(r, 0, sizeof(*r));
            r->time_s = OR_INF;
            r->frontier_offset = -1;
            int st = 0;
            if (p->granularity_bytes <= 0) st = GBMW_EINVAL_GRAN;
            else if (!(p->budget_bytes >= 0.0)) st = GBMW_EINVAL_BUDGET;
            else if (p->n_layers <= 0) st = GBMW_EEMPTY;
            else if (p->micro_batch < 1) st = GBMW_EMICRO;
            else if (p->n_buckets > GBMW_MAX_BUCKETS) st = GBMW_EBUCKETS;
            if (st) { r->status = st; continue; }
            int32_t *pl = plans + plan_off[i];
            double *fr = (p->flags & GBMW_FRONTIER) ? frontier + front_off[i] : NULL;
            double sc[3];
            int feasible = 0;
            r->status = or_dp_search(layers + p->layer_begin, p->n_layers, strats + p->strat_begin, p->n_strats,
                                     &envs[p->env_index], p->micro_batch, p->granularity_bytes, p->budget_bytes,
                                     p->n_buckets, p->stage_index, p->n_micro, p->flags, &r->time_s,
                                     &r->e_fwd_used, &feasible, pl, fr, sc);
            r->feasible = feasible;
            if (fr) r->frontier_offset = front_off[i];
            r->stage_time_s = sc[0]; r->stage_time_no_sync_s = sc[1]; r->stage_peak_mem_bytes = sc[2];
        }
    }
    free(plan_off);
    free(front_off);
    return used;
}

/* ------------------------------------------------------------------ brute_force_oracle */
/* CPython builtin sum() of floats from the int 0: Neumaier-compensated since 3.12
 * (neumaier = 1), plain left-to-right before. */
static double or_py_sum(const double *x, int n, int neumaier) {
    if (n <= 0) return 0.0;
    double f = 0.0 + x[0], c = 0.0;
    for (int i = 1; i < n; ++i) {
        if (!neumaier) { f = f + x[i]; continue; }
        double t = f + x[i];
        if (fabs(f) >= fabs(x[i])) c += (f - t) + x[i];
        else c += (x[i] - t) + f;
        f = t;
    }
    if (neumaier && c != 0.0 && isfinite(c)) f += c;
    return f;
}

/* next ordered split of n layers into p nonempty stages after `sz` (planner.py:354-361:
 * heads ascending, recursively); returns 0 when `sz` was the last one */
static int next_composition(int *sz, int p) {
    /* lexicographic successor among compositions with the same sum and part count */
    for (int i = p - 2; i >= 0; --i) {
        int rest = 0;
        for (int k = i + 1; k < p; ++k) rest += sz[k];
        if (rest - 1 >= p - 1 - i) {            /* head i can grow by one */
            sz[i] += 1;
            rest -= 1;
            for (int k = i + 1; k < p - 1; ++k) { sz[k] = 1; rest -= 1; }
            sz[p - 1] = rest;
            return 1;
        }
    }
    return 0;
}

/* planner.py:364-449.  out_partition / out_choice: n_layers entries (choice = index into
 * prune_dp_sdp(enumerate_strategies(N, P))).  out[0] = cost (+inf if none), out[1] =
 * feasible, out[2] = P, out[3] = m, out[4] = stages.  Returns 0, or -1 on bad input. */
int or_brute_force(const gbmw_layer *layers, int n_layers, const gbmw_env *env, int64_t batch, double budget,
                   int neumaier, int32_t *out_partition, int32_t *out_choice, double out[5]) {
    out[0] = INFINITY; out[1] = 0; out[2] = 0; out[3] = 0; out[4] = 0;
    if (n_layers < 1 || n_layers > 24 || batch < 1) return -1;
    const int L = n_layers;
    gbmw_strategy sset[512];
    for (int64_t P = 1; P <= env->n_devices; P *= 2) {
        if (P > L) continue;
        int ns = or_enumerate(env->n_devices, P, 1, sset, 512);
        if (ns < 0) return -1;
        for (int64_t m = 1; m <= batch; ++m) {
            if (batch % m) continue;
            int64_t micro = batch / m;
            int cand[512], S = 0;
            for (int i = 0; i < ns; ++i)
                if (micro % data_deg(&sset[i]) == 0) cand[S++] = i;
            if (!S) continue;
            double *lt = malloc(sizeof(double) * L * S * 5);
            double *lns = lt + L * S, *of = lt + 2 * L * S, *ob = lt + 3 * L * S, *oms = lt + 4 * L * S;
            for (int l = 0; l < L; ++l)
                for (int j = 0; j < S; ++j) {
                    double mm[3];
                    or_layer_times(&layers[l], &sset[cand[j]], micro, env, &lt[l * S + j], &lns[l * S + j]);
                    or_layer_memory(&layers[l], &sset[cand[j]], micro, 1, 1, env->ms_bytes_per_param_byte, mm);
                    of[l * S + j] = mm[0]; ob[l * S + j] = mm[1]; oms[l * S + j] = mm[2];
                }
            int sz[24];
            for (int k = 0; k < P - 1; ++k) sz[k] = 1;
            sz[P - 1] = L - (int)(P - 1);
            do {
                int choice[24] = {0};
                for (;;) {                              /* itertools.product, last digit fastest */
                    double st_t[24] = {0}, st_ns[24] = {0};
                    int feasible = 1, start = 0;
                    for (int si = 0; si < P && feasible; ++si) {
                        const int stage_idx = si + 1;
                        int64_t stash = P - stage_idx + 1;
                        if (m < stash) stash = m;
                        double t = 0.0, t_ns = 0.0, prefix_f = 0.0, peak = 0.0, total_ms = 0.0;
                        const gbmw_strategy *prev = NULL;
                        for (int li = start; li < start + sz[si]; ++li) {
                            const gbmw_strategy *s = &sset[cand[choice[li]]];
                            const int x = li * S + choice[li];
                            double r = or_transform(&layers[li], prev, s, micro, env);
                            t += lt[x] + r;
                            t_ns += lns[x] + r;
                            prefix_f += of[x] * (double)stash;
                            peak = pymax(peak, prefix_f + ob[x]);
                            total_ms += oms[x];
                            prev = s;
                        }
                        if (stage_idx > 1) {
                            double p2p = or_p2p(&layers[start], micro, (int)P, env);
                            t += p2p;
                            t_ns += p2p;
                        }
                        if (peak + total_ms > budget) feasible = 0;
                        st_t[si] = t; st_ns[si] = t_ns;
                        start += sz[si];
                    }
                    if (feasible) {
                        double steady = st_ns[0];
                        for (int si = 1; si < P; ++si) steady = pymax(steady, st_ns[si]);
                        double cost = (double)(m - 1) * steady + or_py_sum(st_t, (int)P, neumaier);
                        if (cost < out[0]) {
                            out[0] = cost; out[1] = 1; out[2] = (double)P; out[3] = (double)m; out[4] = (double)P;
                            for (int k = 0; k < P; ++k) out_partition[k] = sz[k];
                            for (int l = 0; l < L; ++l) out_choice[l] = cand[choice[l]];
                        }
                    }
                    int l = L - 1;
                    while (l >= 0 && ++choice[l] == S) choice[l--] = 0;
                    if (l < 0) break;
                }
            } while (next_composition(sz, (int)P));
            free(lt);
        }
    }
    return 0;
}
