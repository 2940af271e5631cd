/*
 * pals_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference hot path, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the CHECKER. The product path never links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks every function here against the
 * unmodified reference (oracle/_ref/libwsref.so, built from
 * /root/reference/proj/include by oracle/Makefile) and against the committed
 * fixtures in tests/golden/ that the reference produced (oracle/gen_golden.py).
 *
 * Arithmetic is IEEE FP64 in the reference's operation order, compiled with
 * -ffp-contract=off (the reference's Release build has no FMA).
 * Citations are /root/reference/proj/include/wattserve/<file>:<line>.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/pals_gpu.h"

/* libstdc++ helpers (stl_algobase.h:257-265, stl_algo.h:3667-3671) */
static double smax(double a, double b) { return a < b ? b : a; }
static double smin(double a, double b) { return b < a ? b : a; }
static double sclamp(double v, double lo, double hi) { return smin(smax(v, lo), hi); }

/* rng.hpp:15-20 */
uint64_t or_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* model.hpp:37-45 */
double or_effective_frequency(double cap, const pals_profile* p, const pals_gpu_spec* g,
                              int* err) {
    *err = PALS_OK;
    if (cap < g->min_cap_watts || cap > g->max_cap_watts) {
        *err = PALS_ERANGE;
        return NAN;
    }
    const double span = p->knee_watts - g->min_cap_watts;
    if (span <= 0.0) return g->max_frequency;
    const double ratio = (cap - g->min_cap_watts) / span;
    return g->max_frequency * sclamp(ratio, 0.4, 1.0);
}

/* OperatingPoint::validate types.hpp:117-123, then model.hpp:53-68 */
static int step_timing(const pals_point* c, const pals_profile* p, const pals_gpu_spec* g,
                       double* t_comp, double* t_comm, double* step) {
    if (c->cap_watts < g->min_cap_watts || c->cap_watts > g->max_cap_watts) return PALS_ERANGE;
    if (c->batch < 1) return PALS_ECONFIG;
    if (c->tp < 1 || c->ep < 1 || c->dp < 1) return PALS_ECONFIG;
    int k = -1;
    for (int i = 0; i < p->n_tp; ++i)
        if (p->tp_keys[i] == c->tp) k = i;
    if (k < 0) return PALS_ECONFIG;
    int err;
    const double f = or_effective_frequency(c->cap_watts, p, g, &err);
    const double B = (double)c->batch;
    *t_comp = (p->compute_fixed + p->compute_per_seq * B / (double)c->tp) / f;
    *t_comm = (p->comm_fixed[k] + p->comm_per_seq * B) *
              pow(p->internode_factor, (double)(c->dp - 1));
    const double hi = smax(*t_comp, *t_comm);
    const double lo = smin(*t_comp, *t_comm);
    *step = hi + (1.0 - p->overlap) * lo;
    return PALS_OK;
}

/* throughput model.hpp:72-75 and avg_gpu_power model.hpp:78-84 */
int or_score(const pals_point* c, const pals_profile* p, const pals_gpu_spec* g, double* T,
             double* P) {
    double tc, tm, st;
    const int rc = step_timing(c, p, g, &tc, &tm, &st);
    if (rc != PALS_OK) {
        *T = *P = NAN;
        return rc;
    }
    *T = (double)c->batch / st;
    const double demand =
        p->compute_power_base + p->compute_power_per_seq * (double)c->batch / (double)c->tp;
    const double p_comp = smin(c->cap_watts, demand);
    const double comm_share = st - tc;
    *P = (tc * p_comp + comm_share * p->comm_power) / st;
    return PALS_OK;
}

int or_eval(const pals_profile* p, const pals_gpu_spec* g, const pals_point* pts, int64_t n,
            double* T, double* P, int* err) {
    int rc = PALS_OK;
    for (int64_t i = 0; i < n; ++i) {
        err[i] = or_score(&pts[i], p, g, &T[i], &P[i]);
        if (err[i] != PALS_OK) rc = err[i];
    }
    return rc;
}

/* detail::better_candidate controller.hpp:118-125 */
int or_better(double sa, const pals_point* a, double sb, const pals_point* b) {
    const double scale = smax(smax(fabs(sa), fabs(sb)), 1e-300);
    if ((sa - sb) / scale > 1e-9) return 1;
    if ((sb - sa) / scale > 1e-9) return 0;
    if (a->cap_watts != b->cap_watts) return a->cap_watts < b->cap_watts;
    return a->batch < b->batch;
}

/* select_config controller.hpp:132-201 over pre-scored candidates
 * (T[i], P[i]) = score(candidates[i]); returns the index of Decision::point. */
int or_select_scored(const pals_point* c, int64_t n, const double* T, const double* P,
                     const pals_coeffs* k, const pals_query* q, int32_t* idx, uint8_t* reason) {
    if (n <= 0) return PALS_ECONFIG;
    const double target = q->throughput_tps * (1.0 + q->target_headroom);
    double* th = (double*)malloc(sizeof(double) * (size_t)n);
    double* pn = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        pn[i] = (double)c[i].dp * (k->alpha * 4.0 * P[i] + k->beta_watts);
        th[i] = (double)c[i].dp * T[i];
    }
    const int budget_set = q->has_budget != 0;
    const double budget = budget_set ? q->power_budget_w * (1.0 - q->budget_margin) : 0.0;
    int64_t best = -1;
    int r = PALS_REASON_FALLBACK_MAX_T;
    if (q->objective == PALS_OBJ_QOS) {
        for (int64_t i = 0; i < n; ++i) {
            if ((budget_set && !(pn[i] <= budget)) || th[i] * q->bias < target) continue;
            if (best < 0 || or_better(th[i] / pn[i], &c[i], th[best] / pn[best], &c[best]))
                best = i;
        }
        if (best >= 0) r = PALS_REASON_QOS_FEASIBLE;
    }
    if (best < 0 && budget_set) {
        for (int64_t i = 0; i < n; ++i) {
            if (!(pn[i] <= budget)) continue;
            if (best < 0 || or_better(th[i], &c[i], th[best], &c[best])) best = i;
        }
        if (best >= 0) r = PALS_REASON_BUDGET_MAX_T;
        if (best < 0) {
            for (int64_t i = 0; i < n; ++i)
                if (best < 0 || or_better(-pn[i], &c[i], -pn[best], &c[best])) best = i;
            r = PALS_REASON_BUDGET_MAX_T;
        }
    }
    if (best < 0) {
        for (int64_t i = 0; i < n; ++i)
            if (best < 0 || or_better(th[i], &c[i], th[best], &c[best])) best = i;
        r = PALS_REASON_FALLBACK_MAX_T;
    }
    free(th);
    free(pn);
    *idx = (int32_t)best;
    *reason = (uint8_t)r;
    return PALS_OK;
}

static int point_eq(const pals_point* a, const pals_point* b) {
    return a->cap_watts == b->cap_watts && a->batch == b->batch && a->tp == b->tp &&
           a->ep == b->ep && a->dp == b->dp;
}

static int targets_eq(const pals_targets* a, const pals_targets* b) {
    /* Targets::operator== controller.hpp:25-28 (std::optional compare) */
    if (a->throughput_tps != b->throughput_tps) return 0;
    if (a->has_budget != b->has_budget) return 0;
    if (a->has_budget && a->power_budget_w != b->power_budget_w) return 0;
    return a->epsilon == b->epsilon && a->objective == b->objective;
}

int64_t or_index_of(const pals_point* c, int64_t n, const pals_point* p) {
    for (int64_t i = 0; i < n; ++i)
        if (point_eq(&c[i], p)) return i;
    return -1;
}

/* control_step controller.hpp:210-267. cur_T = score(state.current).throughput_tps,
 * cur_ok = 0 if the scorer cannot score the current point (TableScorer throws). */
int or_control_step_scored(const pals_point* c, int64_t n, const double* T, const double* P,
                           double cur_T, int cur_ok, const pals_telemetry* tel, double now_s,
                           const pals_targets* tg, const pals_coeffs* k,
                           const pals_ctrl_state* state, const pals_ctrl_cfg* cfg,
                           pals_decision* out_d, pals_ctrl_state* out_s) {
    pals_ctrl_state st = *state;
    if (now_s - tel->t_s > 1.5 * cfg->interval_s) {
        out_d->point = st.current;
        out_d->applied = 0;
        out_d->reason = PALS_REASON_HOLD;
        *out_s = st;
        return PALS_OK;
    }
    double err_norm = 0.0;
    if (tg->objective == PALS_OBJ_QOS && tg->throughput_tps > 0.0) {
        err_norm = (tg->throughput_tps - tel->throughput_tps) / tg->throughput_tps;
        if (!cur_ok) return PALS_ECONFIG;
        const double promised = (double)st.current.dp * cur_T * st.bias;
        if (promised > 0.0) {
            const double pred_err = (promised - tel->throughput_tps) / promised;
            st.integral = sclamp(st.integral + pred_err, -cfg->integral_clamp, cfg->integral_clamp);
            const double deriv = st.has_prev_error ? pred_err - st.prev_error : 0.0;
            const double corr = cfg->kp * pred_err + cfg->ki * st.integral + cfg->kd * deriv;
            st.bias = sclamp(st.bias * (1.0 - corr), cfg->bias_min, cfg->bias_max);
            st.prev_error = pred_err;
            st.has_prev_error = 1;
        }
    }
    const int changed = !st.has_last_targets || !targets_eq(&st.last_targets, tg);
    st.last_targets = *tg;
    st.has_last_targets = 1;
    if (fabs(err_norm) > tg->epsilon)
        ++st.sustain_count;
    else
        st.sustain_count = 0;

    pals_query q;
    q.throughput_tps = tg->throughput_tps;
    q.power_budget_w = tg->power_budget_w;
    q.has_budget = tg->has_budget;
    q.objective = tg->objective;
    q.bias = st.bias;
    q.target_headroom = cfg->target_headroom;
    q.budget_margin = cfg->budget_margin;
    int32_t idx;
    uint8_t reason;
    const int rc = or_select_scored(c, n, T, P, k, &q, &idx, &reason);
    if (rc != PALS_OK) return rc;

    const int may_apply = changed || st.sustain_count >= cfg->sustain_intervals;
    if (may_apply && !point_eq(&c[idx], &st.current)) {
        st.current = c[idx];
        st.sustain_count = 0;
        out_d->point = c[idx];
        out_d->applied = 1;
        out_d->reason = reason;
        *out_s = st;
        return PALS_OK;
    }
    out_d->point = st.current;
    out_d->applied = 0;
    out_d->reason = may_apply ? reason : PALS_REASON_HOLD;
    *out_s = st;
    return PALS_OK;
}

/* ---- fluid replay plant (not in the reference) ----------- */
static uint64_t draw(uint64_t key, uint64_t lane, uint64_t ctr) {
    return or_splitmix64(key ^ (lane << 48) ^ ctr);
}
static double u01(uint64_t u) { return (double)(u >> 11) * 0x1.0p-53; }
/* plant noise uniform of step s: the low (even s) or high (odd s) 32 bits of one
 * splitmix64 draw per step pair, times 2^-32 */
static double noise_u(uint64_t key, uint64_t s) {
    return (double)(uint32_t)(draw(key, 3, s >> 1) >> (32 * (s & 1))) * 0x1.0p-32;
}

typedef struct {
    uint64_t key, lane;
    int seg_min, seg_max;
    double lo, hi;
    long next_j, seg_end;
    double level;
} segs;

static double seg_value(segs* s, long k) {
    while (k >= s->seg_end) {
        const uint64_t span = (uint64_t)(s->seg_max - s->seg_min) + 1;
        const long len = s->seg_min + (long)(draw(s->key, s->lane, 2 * (uint64_t)s->next_j) % span);
        const double u = u01(draw(s->key, s->lane, 2 * (uint64_t)s->next_j + 1));
        s->level = s->lo + (s->hi - s->lo) * u;
        s->seg_end += len;
        ++s->next_j;
    }
    return s->level;
}

/* detail::enforce_cap sim.hpp:195-205 */
static double enforce_cap(double cap, int batch, double node_budget, const pals_point* tmpl,
                          const pals_profile* p, const pals_gpu_spec* g, const pals_coeffs* k) {
    if (node_budget <= 0.0 || batch < 1) return cap;
    double c = cap;
    while (c > g->min_cap_watts) {
        pals_point q = *tmpl;
        q.cap_watts = c;
        q.batch = batch;
        double T, P;
        or_score(&q, p, g, &T, &P);
        /* cluster_system_power model.hpp:99-103 */
        const double sys = (double)q.dp * (k->alpha * 4.0 * P + k->beta_watts);
        if (sys <= node_budget) return c;
        c = smax(g->min_cap_watts, c - 5.0);
    }
    return g->min_cap_watts;
}

/* Replay with the controller's scorer given as per-model candidate tables
 * (scorerT/scorerP[m * nc + i] = score(candidate i of model m)), e.g. a forest
 * predictor; the plant always runs the analytic profile. NULL tables: the
 * scorer is the analytic plant model itself (analytic_scorer). */
static int replay_impl(int n_models, const pals_profile* plant, const pals_gpu_spec* g,
                       const pals_coeffs* k, const double* caps, int n_caps, const int* batches,
                       int n_batches, const pals_ctrl_cfg* cfg, const pals_replay_spec* spec,
                       const double* scorerT, const double* scorerP,
                       pals_trace_summary* summaries, pals_step_log* logs,
                       pals_step_detail* details);

int or_replay_scored(int n_models, const pals_profile* plant, const pals_gpu_spec* g,
                     const pals_coeffs* k, const double* caps, int n_caps, const int* batches,
                     int n_batches, const pals_ctrl_cfg* cfg, const pals_replay_spec* spec,
                     const double* scorerT, const double* scorerP,
                     pals_trace_summary* summaries, pals_step_log* logs) {
    return replay_impl(n_models, plant, g, k, caps, n_caps, batches, n_batches, cfg, spec,
                       scorerT, scorerP, summaries, logs, NULL);
}

/* Also the per-step DecisionRecord err_norm / bias of the logged traces
 * (sim.hpp:438-440, 457-464). */
int or_replay_ex(int n_models, const pals_profile* plant, const pals_gpu_spec* g,
                 const pals_coeffs* k, const double* caps, int n_caps, const int* batches,
                 int n_batches, const pals_ctrl_cfg* cfg, const pals_replay_spec* spec,
                 pals_trace_summary* summaries, pals_step_log* logs, pals_step_detail* details) {
    return replay_impl(n_models, plant, g, k, caps, n_caps, batches, n_batches, cfg, spec, NULL,
                       NULL, summaries, logs, details);
}

int or_replay(int n_models, const pals_profile* plant, const pals_gpu_spec* g,
              const pals_coeffs* k, const double* caps, int n_caps, const int* batches,
              int n_batches, const pals_ctrl_cfg* cfg, const pals_replay_spec* spec,
              pals_trace_summary* summaries, pals_step_log* logs) {
    return replay_impl(n_models, plant, g, k, caps, n_caps, batches, n_batches, cfg, spec, NULL,
                       NULL, summaries, logs, NULL);
}

static int replay_impl(int n_models, const pals_profile* plant, const pals_gpu_spec* g,
                       const pals_coeffs* k, const double* caps, int n_caps, const int* batches,
                       int n_batches, const pals_ctrl_cfg* cfg, const pals_replay_spec* spec,
                       const double* scorerT, const double* scorerP,
                       pals_trace_summary* summaries, pals_step_log* logs,
                       pals_step_detail* details) {
    const int nc = n_caps * n_batches;
    pals_point* cands = (pals_point*)malloc(sizeof(pals_point) * (size_t)nc * (size_t)n_models);
    double* T = (double*)malloc(sizeof(double) * (size_t)nc * (size_t)n_models);
    double* P = (double*)malloc(sizeof(double) * (size_t)nc * (size_t)n_models);
    double* tmax = (double*)malloc(sizeof(double) * (size_t)n_models);
    double* pmin = (double*)malloc(sizeof(double) * (size_t)n_models);
    double* pmax = (double*)malloc(sizeof(double) * (size_t)n_models);
    double mc = caps[0];
    int mb = batches[0];
    for (int a = 0; a < n_caps; ++a) mc = smax(mc, caps[a]);
    for (int b = 0; b < n_batches; ++b) mb = batches[b] > mb ? batches[b] : mb;
    int rc = PALS_OK;
    for (int m = 0; m < n_models; ++m) {
        pals_point* cm = cands + (size_t)m * nc;
        int i = 0;
        for (int a = 0; a < n_caps; ++a)
            for (int b = 0; b < n_batches; ++b, ++i) {
                cm[i].cap_watts = caps[a];
                cm[i].batch = batches[b];
                cm[i].tp = plant[m].deploy_tp;
                cm[i].ep = plant[m].deploy_ep;
                cm[i].dp = plant[m].deploy_dp;
                const int e = or_score(&cm[i], &plant[m], g, &T[(size_t)m * nc + i],
                                       &P[(size_t)m * nc + i]);
                if (e != PALS_OK) rc = e;
                const double pn =
                    (double)cm[i].dp * (k->alpha * 4.0 * P[(size_t)m * nc + i] + k->beta_watts);
                if (i == 0 || pn < pmin[m]) pmin[m] = pn;
                if (i == 0 || pn > pmax[m]) pmax[m] = pn;
            }
        pals_point top = cm[0];
        top.cap_watts = mc;
        top.batch = mb;
        double tt, pp;
        const int e = or_score(&top, &plant[m], g, &tt, &pp);
        if (e != PALS_OK) rc = e;
        tmax[m] = (double)top.dp * tt;
    }
    if (rc != PALS_OK) goto done;

    for (int64_t ti = 0; ti < spec->n_traces; ++ti) {
        const uint64_t key = or_splitmix64(spec->seed ^ (uint64_t)(spec->first_trace + ti));
        const int m = (int)(key % (uint64_t)n_models);
        const pals_point* cm = cands + (size_t)m * nc;
        const double* Tm = (scorerT ? scorerT : T) + (size_t)m * nc;
        const double* Pm = (scorerP ? scorerP : P) + (size_t)m * nc;
        int obj = spec->objective_mode;
        if (obj == 2) obj = (int)(draw(key, 0, 0) >> 63);
        const double qfrac =
            spec->qos_frac_lo + (spec->qos_frac_hi - spec->qos_frac_lo) * u01(draw(key, 0, 1));
        const double target_tps = qfrac * tmax[m];
        segs bs = {key, 1, spec->seg_min, spec->seg_max, spec->budget_lo_frac * pmin[m],
                   spec->budget_hi_frac * pmax[m], 0, 0, 0.0};
        segs ls = {key, 2, spec->seg_min, spec->seg_max, spec->load_lo * tmax[m],
                   spec->load_hi * tmax[m], 0, 0, 0.0};
        pals_ctrl_state st;
        memset(&st, 0, sizeof st);
        st.bias = 1.0;
        st.current = cm[0];
        st.current.cap_watts = mc;
        st.current.batch = mb;
        double applied_cap = mc, inflight_cap = mc;
        int batch_cap = mb;
        uint64_t h = 0xcbf29ce484222325ULL;
        double energy = 0.0, tokens = 0.0;
        int n_applied = 0;
        pals_step_log* lg = (logs && ti < spec->n_log_traces) ? logs + ti * spec->n_steps : NULL;
        for (int s = 0; s < spec->n_steps; ++s) {
            const double t0 = (double)s * spec->interval_s;
            const double t1 = t0 + spec->interval_s;
            const double node_budget = spec->budget_mode ? seg_value(&bs, s) : 0.0;
            const int b_eff = batch_cap;
            const double cap =
                enforce_cap(applied_cap, b_eff, node_budget, &cm[0], &plant[m], g, k);
            pals_point p = cm[0];
            p.cap_watts = cap;
            p.batch = b_eff;
            double Tc, Pc;
            or_score(&p, &plant[m], g, &Tc, &Pc);
            const double capacity = (double)p.dp * Tc;
            const double sys_w = (double)p.dp * (k->alpha * 4.0 * Pc + k->beta_watts);
            const double offered = seg_value(&ls, s);
            const double noise = 1.0 + spec->noise_amp * (2.0 * noise_u(key, (uint64_t)s) - 1.0);
            const double measured = smin(offered, capacity) * noise;
            energy += sys_w * spec->interval_s;
            tokens += measured * spec->interval_s;

            pals_targets tg;
            memset(&tg, 0, sizeof tg);
            tg.throughput_tps = target_tps;
            tg.epsilon = spec->epsilon;
            tg.objective = obj;
            tg.has_budget = node_budget > 0.0;
            tg.power_budget_w = tg.has_budget ? node_budget : 0.0;
            pals_telemetry tel = {t1, measured};
            const int64_t ci = or_index_of(cm, nc, &st.current);
            pals_decision d;
            pals_ctrl_state st2;
            rc = or_control_step_scored(cm, nc, Tm, Pm, ci >= 0 ? Tm[ci] : 0.0, ci >= 0, &tel, t1,
                                        &tg, k, &st, cfg, &d, &st2);
            if (rc != PALS_OK) goto done;
            st = st2;
            const int64_t idx = or_index_of(cm, nc, &d.point);
            const uint64_t word = ((uint64_t)(uint32_t)idx << 8) | ((uint64_t)(d.applied ? 1 : 0) << 4) |
                                  (uint64_t)d.reason;
            h = (h ^ word) * 0x100000001b3ULL;
            if (d.applied) ++n_applied;
            if (lg) {
                lg[s].idx = (int32_t)idx;
                lg[s].applied = (uint8_t)(d.applied ? 1 : 0);
                lg[s].reason = (uint8_t)d.reason;
                lg[s].cap_tenths = (uint16_t)llround(cap * 10.0);
                if (details) {
                    pals_step_detail* x = details + ti * spec->n_steps + s;
                    x->err_norm = target_tps > 0.0 ? (target_tps - measured) / target_tps : 0.0;
                    x->bias = st.bias;
                }
            }
            applied_cap = inflight_cap;
            if (d.applied) {
                batch_cap = d.point.batch;
                inflight_cap = d.point.cap_watts;
            }
        }
        uint64_t bias_bits;
        memcpy(&bias_bits, &st.bias, 8);
        const int64_t fi = or_index_of(cm, nc, &st.current);
        h = (h ^ bias_bits) * 0x100000001b3ULL;
        h = (h ^ (uint64_t)(uint32_t)fi) * 0x100000001b3ULL;
        pals_trace_summary* sm = &summaries[ti];
        sm->digest = h;
        sm->final_bias = st.bias;
        sm->energy_j = energy;
        sm->tokens = tokens;
        sm->n_applied = n_applied;
        sm->final_idx = (int32_t)fi;
        sm->model = m;
        sm->objective = obj;
    }
done:
    free(cands);
    free(T);
    free(P);
    free(tmax);
    free(pmin);
    free(pmax);
    return rc;
}

/* ---- tree-ensemble predictor (forest.hpp) ------------------------------ */
/* RegressionTree::predict forest.hpp:80-85 (children are tree-local) */
static double tree_predict(const int32_t* f, const double* thr, const int32_t* l,
                           const int32_t* r, const double* v, const double* x) {
    int i = 0;
    while (f[i] >= 0) i = x[f[i]] <= thr[i] ? l[i] : r[i];
    return v[i];
}

/* Forest::predict forest.hpp:176-180 */
static double forest_predict(int n_trees, const int64_t* off, const int32_t* f,
                             const double* thr, const int32_t* l, const int32_t* r,
                             const double* v, const double* x) {
    double s = 0.0;
    for (int t = 0; t < n_trees; ++t) {
        const int64_t o = off[t];
        s += tree_predict(f + o, thr + o, l + o, r + o, v + o, x);
    }
    return s / (double)n_trees;
}

/* PredictorBundle::predict forest.hpp:227-235 with FeatureSchema::encode :41-50 */
int or_forest_predict(int n_models, int model_index, const pals_coeffs* k, int tn,
                      const int64_t* toff, const int32_t* tf, const double* tthr,
                      const int32_t* tl, const int32_t* tr, const double* tv, int pn,
                      const int64_t* poff, const int32_t* pf, const double* pthr,
                      const int32_t* pl, const int32_t* pr, const double* pv,
                      const pals_point* pts, int64_t n, double* T, double* P, double* E) {
    if (model_index < 0 || model_index >= n_models) return PALS_ECONFIG;
    double* x = (double*)calloc((size_t)(5 + n_models), sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        x[0] = pts[i].cap_watts;
        x[1] = (double)pts[i].batch;
        x[2] = (double)pts[i].tp;
        x[3] = (double)pts[i].ep;
        x[4] = (double)pts[i].dp;
        x[5 + model_index] = 1.0;
        T[i] = forest_predict(tn, toff, tf, tthr, tl, tr, tv, x);
        P[i] = forest_predict(pn, poff, pf, pthr, pl, pr, pv, x);
        E[i] = T[i] / (k->alpha * 4.0 * P[i] + k->beta_watts);
    }
    free(x);
    return PALS_OK;
}

/* ---- cluster budget allocator (allocator.hpp) -------------------------- */
typedef struct {
    double power_w, thr;
} bstep;

/* throughput_steps sort: power ascending, then throughput descending (allocator.hpp:44-47) */
static int bstep_cmp(const void* a, const void* b) {
    const bstep* x = (const bstep*)a;
    const bstep* y = (const bstep*)b;
    if (x->power_w != y->power_w) return x->power_w < y->power_w ? -1 : 1;
    if (x->thr != y->thr) return x->thr > y->thr ? -1 : 1;
    return 0;
}

/* detail::throughput_steps allocator.hpp:34-56, then the margin scaling :106 */
static int node_steps(const pals_profile* p, const pals_gpu_spec* g, const pals_coeffs* k,
                      const double* caps, int nc, const int* batches, int nb, int dp,
                      double margin, bstep* out) {
    int m = 0;
    for (int a = 0; a < nc; ++a)
        for (int b = 0; b < nb; ++b) {
            pals_point c = {caps[a], batches[b], p->deploy_tp, p->deploy_ep, dp};
            double T, P;
            or_score(&c, p, g, &T, &P);
            out[m].power_w = (double)dp * (k->alpha * 4.0 * P + k->beta_watts);
            out[m].thr = (double)dp * T;
            ++m;
        }
    qsort(out, (size_t)m, sizeof(bstep), bstep_cmp);
    int ns = 0;
    double best = 0.0;
    for (int i = 0; i < m; ++i)
        if (out[i].thr > best + 1e-12) {
            out[ns++] = out[i];
            best = out[i].thr;
        }
    for (int i = 0; i < ns; ++i) out[i].power_w /= 1.0 - margin;
    return ns;
}

/* detail::best_throughput_under allocator.hpp:58-65 */
static double best_under(const bstep* s, int ns, double budget) {
    double best = 0.0;
    for (int i = 0; i < ns; ++i) {
        if (s[i].power_w > budget) break;
        best = s[i].thr;
    }
    return best;
}

/* allocate_budget allocator.hpp:76-186 over independent problems (see ref_allocate) */
int or_allocate(int n_models, const pals_profile* profs, const pals_gpu_spec* g,
                const pals_coeffs* k, const double* caps, int nc, const int* batches, int nb,
                double quantum, double margin, int64_t n_problems, const int64_t* off,
                const int32_t* node_model, const int32_t* node_dp, const double* node_target,
                const double* cluster_budget, double* node_budget, double* total,
                uint8_t* all_sat, int32_t* status) {
    (void)n_models;
    const int ncand = nc * nb;
    for (int64_t pi = 0; pi < n_problems; ++pi) {
        const int64_t o = off[pi];
        const int n = (int)(off[pi + 1] - o);
        if (n <= 0) {
            status[pi] = PALS_ECONFIG; /* "allocate_budget: no nodes" */
            continue;
        }
        double* floor_w = (double*)malloc(sizeof(double) * n);
        double* cur = (double*)malloc(sizeof(double) * n);
        double* ceil_w = (double*)malloc(sizeof(double) * n);
        int* ns = (int*)malloc(sizeof(int) * n);
        bstep* st = (bstep*)malloc(sizeof(bstep) * (size_t)n * (size_t)ncand);
        double* bud = node_budget + o;
        double floor_total = 0.0;
        for (int i = 0; i < n; ++i) {
            floor_w[i] = (double)node_dp[o + i] * (k->alpha * 4.0 * g->min_cap_watts + k->beta_watts);
            floor_total += floor_w[i];
        }
        if (floor_total > cluster_budget[pi]) {
            status[pi] = PALS_ECONFIG;
            free(floor_w); free(cur); free(ceil_w); free(ns); free(st);
            continue;
        }
        double remaining = cluster_budget[pi] - floor_total;
        for (int i = 0; i < n; ++i) {
            bud[i] = floor_w[i];
            ns[i] = node_steps(&profs[node_model[o + i]], g, k, caps, nc, batches, nb,
                               node_dp[o + i], margin, st + (size_t)i * ncand);
            cur[i] = best_under(st + (size_t)i * ncand, ns[i], bud[i]);
        }
        while (remaining >= quantum) {
            int any_unmet = 0;
            for (int i = 0; i < n; ++i) any_unmet |= !(cur[i] >= node_target[o + i]);
            double best_rate = 0.0, best_cost = 0.0;
            int best_i = n;
            for (int i = 0; i < n; ++i) {
                const double tgt = node_target[o + i];
                if (any_unmet && cur[i] >= tgt) continue;
                const bstep* s = st + (size_t)i * ncand;
                for (int j = 0; j < ns[i]; ++j) {
                    if (s[j].power_w <= bud[i] || s[j].thr <= cur[i]) continue;
                    const double cost = ceil((s[j].power_w - bud[i]) / quantum) * quantum;
                    if (cost > remaining) break;
                    const double gain = any_unmet ? smin(s[j].thr, tgt) - smin(cur[i], tgt)
                                                  : s[j].thr - cur[i];
                    if (gain <= 1e-12) continue;
                    const double rate = gain / cost;
                    const int wins = best_i == n || rate > best_rate + 1e-12 ||
                                     (rate > best_rate - 1e-12 && bud[i] < bud[best_i] - 1e-12);
                    if (wins) {
                        best_rate = rate;
                        best_cost = cost;
                        best_i = i;
                    }
                }
            }
            if (best_i == n) break;
            bud[best_i] += best_cost;
            cur[best_i] = best_under(st + (size_t)best_i * ncand, ns[best_i], bud[best_i]);
            remaining -= best_cost;
        }
        for (int i = 0; i < n; ++i)
            ceil_w[i] = ns[i] == 0 ? bud[i] : st[(size_t)i * ncand + ns[i] - 1].power_w + 2.0 * quantum;
        while (remaining >= quantum) {
            int lo = n;
            for (int i = 0; i < n; ++i) {
                if (bud[i] + quantum > ceil_w[i]) continue;
                if (lo == n || bud[i] < bud[lo]) lo = i;
            }
            if (lo == n) break;
            bud[lo] += quantum;
            remaining -= quantum;
        }
        double tot = 0.0;
        int sat = 1;
        for (int i = 0; i < n; ++i) {
            tot += bud[i];
            sat &= cur[i] >= node_target[o + i];
        }
        total[pi] = tot;
        all_sat[pi] = (uint8_t)sat;
        status[pi] = PALS_OK;
        free(floor_w); free(cur); free(ceil_w); free(ns); free(st);
    }
    return PALS_OK;
}

/* ---- Pareto frontier (pareto.hpp) ---------------------------------------- */
typedef struct {
    double thr, eff, cap;
    int batch;
    int64_t idx;
} fr_item;

/* build_frontier's sort: throughput, efficiency, cap, batch ascending (pareto.hpp:35-40);
 * full ties (equal on all four) are left unspecified by std::sort; input order here. */
static int fr_cmp(const void* a, const void* b) {
    const fr_item* x = (const fr_item*)a;
    const fr_item* y = (const fr_item*)b;
    if (x->thr != y->thr) return x->thr < y->thr ? -1 : 1;
    if (x->eff != y->eff) return x->eff < y->eff ? -1 : 1;
    if (x->cap != y->cap) return x->cap < y->cap ? -1 : 1;
    if (x->batch != y->batch) return x->batch < y->batch ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* build_frontier pareto.hpp:31-59: indices of the frontier points, throughput ascending */
int or_build_frontier(const pals_point* pts, const double* thr, const double* eff, int64_t n,
                      int64_t* out_idx, int64_t* out_n) {
    if (n <= 0) return PALS_ECONFIG; /* "build_frontier: no points" */
    fr_item* v = (fr_item*)malloc(sizeof(fr_item) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        v[i].thr = thr[i];
        v[i].eff = eff[i];
        v[i].cap = pts[i].cap_watts;
        v[i].batch = pts[i].batch;
        v[i].idx = i;
    }
    qsort(v, (size_t)n, sizeof(fr_item), fr_cmp);
    /* collapse exact (throughput, efficiency) ties onto the first (lower cap) point */
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (m > 0 && v[m - 1].thr == v[i].thr && v[m - 1].eff == v[i].eff) continue;
        v[m++] = v[i];
    }
    /* sweep from the high-throughput end (pareto.hpp:50-57) */
    double best = -1.0;
    int64_t k = 0;
    for (int64_t i = m - 1; i >= 0; --i)
        if (v[i].eff > best) {
            out_idx[k++] = v[i].idx;
            best = v[i].eff;
        }
    for (int64_t i = 0; i < k / 2; ++i) { /* std::reverse */
        const int64_t t = out_idx[i];
        out_idx[i] = out_idx[k - 1 - i];
        out_idx[k - 1 - i] = t;
    }
    *out_n = k;
    free(v);
    return PALS_OK;
}
