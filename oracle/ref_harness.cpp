// ref_harness.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/wattserve/*.hpp), built by oracle/Makefile into
// oracle/_ref/libwsref.so. It lets the Python tests and bench.py's CPU arm
// call the reference's own select_config / control_step / throughput /
// avg_gpu_power / PredictorBundle::predict on exactly the inputs the GPU path
// sees. Nothing here re-implements reference logic except the replay plant,
// which the reference does not have: it drives the reference's
// control_step with the reference's own model functions.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "wattserve/controller.hpp"
#include "wattserve/forest.hpp"
#include "wattserve/metrics.hpp"
#include "wattserve/scenario_io.hpp"
#include "wattserve/model.hpp"
#include "wattserve/pareto.hpp"
#include "wattserve/rng.hpp"
#include "wattserve/sim.hpp"
#include "wattserve/sweep.hpp"

#include "pals_gpu.h"

using namespace wattserve;

namespace {

thread_local std::string g_err;

ModelProfile to_profile(const pals_profile& p) {
    ModelProfile m;
    m.name = p.name;
    m.total_params_b = p.total_params_b;
    m.active_params_b = p.active_params_b;
    m.num_experts = p.num_experts;
    m.top_k = p.top_k;
    m.compute_fixed = p.compute_fixed;
    m.compute_per_seq = p.compute_per_seq;
    for (int i = 0; i < p.n_tp; ++i) m.comm_fixed_by_tp[p.tp_keys[i]] = p.comm_fixed[i];
    m.comm_per_seq = p.comm_per_seq;
    m.internode_factor = p.internode_factor;
    m.knee_watts = p.knee_watts;
    m.compute_power_base = p.compute_power_base;
    m.compute_power_per_seq = p.compute_power_per_seq;
    m.comm_power = p.comm_power;
    m.overlap = p.overlap;
    m.deployment = Deployment{p.deploy_tp, p.deploy_ep, p.deploy_dp};
    return m;
}

GpuSpec to_gpu(const pals_gpu_spec& g) {
    return GpuSpec{g.idle_watts, g.min_cap_watts, g.max_cap_watts, g.max_frequency};
}

OperatingPoint to_point(const pals_point& p) {
    return OperatingPoint{p.cap_watts, p.batch, p.tp, p.ep, p.dp};
}

pals_point from_point(const OperatingPoint& p) {
    pals_point o;
    o.cap_watts = p.cap_watts;
    o.batch = p.batch;
    o.tp = p.tp;
    o.ep = p.ep;
    o.dp = p.dp;
    return o;
}

Targets to_targets(const pals_targets& t) {
    Targets o;
    o.throughput_tps = t.throughput_tps;
    if (t.has_budget) o.power_budget_w = t.power_budget_w;
    o.epsilon = t.epsilon;
    o.objective = t.objective == PALS_OBJ_BUDGET ? Objective::BudgetMaxThroughput
                                                 : Objective::QosMaxEfficiency;
    return o;
}

pals_targets from_targets(const Targets& t) {
    pals_targets o{};
    o.throughput_tps = t.throughput_tps;
    o.has_budget = t.power_budget_w.has_value() ? 1 : 0;
    o.power_budget_w = t.power_budget_w.value_or(0.0);
    o.epsilon = t.epsilon;
    o.objective = t.objective == Objective::BudgetMaxThroughput ? PALS_OBJ_BUDGET : PALS_OBJ_QOS;
    return o;
}

ControllerConfig to_cfg(const pals_ctrl_cfg& c) {
    ControllerConfig o;
    o.gains = PidGains{c.kp, c.ki, c.kd};
    o.sustain_intervals = c.sustain_intervals;
    o.integral_clamp = c.integral_clamp;
    o.bias_min = c.bias_min;
    o.bias_max = c.bias_max;
    o.interval_s = c.interval_s;
    o.target_headroom = c.target_headroom;
    o.budget_margin = c.budget_margin;
    return o;
}

ControllerState to_state(const pals_ctrl_state& s) {
    ControllerState o;
    o.bias = s.bias;
    o.integral = s.integral;
    o.prev_error = s.prev_error;
    o.has_prev_error = s.has_prev_error != 0;
    o.sustain_count = s.sustain_count;
    o.current = to_point(s.current);
    if (s.has_last_targets) o.last_targets = to_targets(s.last_targets);
    return o;
}

pals_ctrl_state from_state(const ControllerState& s) {
    pals_ctrl_state o{};
    o.bias = s.bias;
    o.integral = s.integral;
    o.prev_error = s.prev_error;
    o.has_prev_error = s.has_prev_error ? 1 : 0;
    o.sustain_count = s.sustain_count;
    o.current = from_point(s.current);
    o.has_last_targets = s.last_targets.has_value() ? 1 : 0;
    if (s.last_targets) o.last_targets = from_targets(*s.last_targets);
    return o;
}

// TableScorer semantics (tests/test_controller.cpp:17-29): first point equal by value.
Scorer table_scorer(const std::vector<OperatingPoint>& pts, const double* t, const double* p) {
    return [&pts, t, p](const OperatingPoint& q) {
        for (std::size_t i = 0; i < pts.size(); ++i)
            if (pts[i] == q) return CandidateScore{t[i], p[i]};
        throw config_error("unscored candidate");
    };
}

int map_exception() {
    try {
        throw;
    } catch (const config_error& e) {
        g_err = e.what();
        return PALS_ECONFIG;
    } catch (const data_error& e) {
        g_err = e.what();
        return PALS_EDATA;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return PALS_ERANGE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PALS_ERUNTIME;
    }
}

int reason_code(DecisionReason r) { return static_cast<int>(r); }

Targets query_targets(const pals_query& q) {
    Targets t;
    t.throughput_tps = q.throughput_tps;
    if (q.has_budget) t.power_budget_w = q.power_budget_w;
    t.objective = q.objective == PALS_OBJ_BUDGET ? Objective::BudgetMaxThroughput
                                                 : Objective::QosMaxEfficiency;
    return t;
}

int index_of(const std::vector<OperatingPoint>& pts, const OperatingPoint& p) {
    for (std::size_t i = 0; i < pts.size(); ++i)
        if (pts[i] == p) return static_cast<int>(i);
    return -1;
}

// ---- fluid replay plant; NOT in the reference -------------
constexpr std::uint64_t kFnvOffset = 0xcbf29ce484222325ULL;
constexpr std::uint64_t kFnvPrime = 0x100000001b3ULL;

inline std::uint64_t draw(std::uint64_t key, std::uint64_t lane, std::uint64_t ctr) {
    return splitmix64(key ^ (lane << 48) ^ ctr);
}
inline double u01(std::uint64_t u) { return static_cast<double>(u >> 11) * 0x1.0p-53; }
// plant noise uniform of step s: the low (even s) or high (odd s) 32 bits of one
// splitmix64 draw per step pair, times 2^-32
inline double noise_u(std::uint64_t key, std::uint64_t s) {
    return static_cast<double>(static_cast<std::uint32_t>(draw(key, 3, s >> 1) >> (32 * (s & 1)))) *
           0x1.0p-32;
}

struct Segments {
    std::uint64_t key, lane;
    int seg_min, seg_max;
    double lo, hi;
    long next_j = 0;
    long seg_end = 0;
    double level = 0.0;
    double value_at(long k) {
        while (k >= seg_end) {
            const std::uint64_t span = static_cast<std::uint64_t>(seg_max - seg_min) + 1;
            const long len = seg_min + static_cast<long>(draw(key, lane, 2 * next_j) % span);
            const double u = u01(draw(key, lane, 2 * next_j + 1));
            level = lo + (hi - lo) * u;
            seg_end += len;
            ++next_j;
        }
        return level;
    }
};

struct ReplayModel {
    ModelProfile profile;
    std::vector<OperatingPoint> cands;
    Scorer scorer;
    double t_max = 0.0, p_min = 0.0, p_max = 0.0;
};

void replay_one(const std::vector<ReplayModel>& models, const GpuSpec& gpu,
                const SystemPowerCoeffs& coeffs, const ControllerConfig& cfg,
                const pals_replay_spec& spec, std::int64_t gi, pals_trace_summary* summary,
                pals_step_log* log, std::vector<DecisionRecord>* recs = nullptr) {
    const std::uint64_t key = splitmix64(spec.seed ^ static_cast<std::uint64_t>(gi));
    const int m = static_cast<int>(key % models.size());
    const ReplayModel& rm = models[m];
    int obj = spec.objective_mode;
    if (obj == 2) obj = static_cast<int>(draw(key, 0, 0) >> 63);
    const double qfrac =
        spec.qos_frac_lo + (spec.qos_frac_hi - spec.qos_frac_lo) * u01(draw(key, 0, 1));
    const double target_tps = qfrac * rm.t_max;
    Segments bseg{key, 1, spec.seg_min, spec.seg_max, spec.budget_lo_frac * rm.p_min,
                  spec.budget_hi_frac * rm.p_max};
    Segments lseg{key, 2, spec.seg_min, spec.seg_max, spec.load_lo * rm.t_max,
                  spec.load_hi * rm.t_max};

    const OperatingPoint& first = rm.cands.front();
    double max_cap = first.cap_watts;
    int max_batch = first.batch;
    for (const auto& c : rm.cands) {
        max_cap = std::max(max_cap, c.cap_watts);
        max_batch = std::max(max_batch, c.batch);
    }
    const int tp = first.tp, ep = first.ep, dp = first.dp;

    detail::NodeRuntime n;  // only the fields enforce_cap reads
    n.profile = &rm.profile;
    n.cfg.tp = tp;
    n.cfg.ep = ep;
    n.cfg.dp = dp;

    ControllerState st;
    st.current = OperatingPoint{max_cap, max_batch, tp, ep, dp};
    double applied_cap = max_cap, inflight_cap = max_cap;
    int batch_cap = max_batch;
    std::uint64_t h = kFnvOffset;
    double energy = 0.0, tokens = 0.0;
    int n_applied = 0;

    for (int k = 0; k < spec.n_steps; ++k) {
        const double t0 = k * spec.interval_s;
        const double t1 = t0 + spec.interval_s;
        n.node_budget = spec.budget_mode ? bseg.value_at(k) : 0.0;
        const int b_eff = batch_cap;
        const double cap = detail::enforce_cap(applied_cap, b_eff, n, gpu, coeffs);
        const OperatingPoint p{cap, b_eff, tp, ep, dp};
        const double capacity = cluster_throughput(p, rm.profile, gpu);
        const double gpu_w = avg_gpu_power(p, rm.profile, gpu);
        const double sys_w = dp * (coeffs.alpha * kGpusPerNode * gpu_w + coeffs.beta_watts);
        const double offered = lseg.value_at(k);
        const double noise = 1.0 + spec.noise_amp * (2.0 * noise_u(key, k) - 1.0);
        const double measured = std::min(offered, capacity) * noise;
        energy += sys_w * spec.interval_s;
        tokens += measured * spec.interval_s;

        Targets targets;
        targets.throughput_tps = target_tps;
        targets.epsilon = spec.epsilon;
        targets.objective =
            obj == PALS_OBJ_BUDGET ? Objective::BudgetMaxThroughput : Objective::QosMaxEfficiency;
        if (n.node_budget > 0.0) targets.power_budget_w = n.node_budget;

        auto [d, st2] = control_step(TelemetryInput{t1, measured}, t1, targets, rm.cands,
                                     rm.scorer, coeffs, st, cfg);
        st = st2;
        const int idx = index_of(rm.cands, d.point);
        const std::uint64_t word = (static_cast<std::uint64_t>(static_cast<std::uint32_t>(idx)) << 8) |
                                   (static_cast<std::uint64_t>(d.applied ? 1 : 0) << 4) |
                                   static_cast<std::uint64_t>(reason_code(d.reason));
        h = (h ^ word) * kFnvPrime;
        if (d.applied) ++n_applied;
        if (log) {
            log[k].idx = idx;
            log[k].applied = d.applied ? 1 : 0;
            log[k].reason = static_cast<std::uint8_t>(reason_code(d.reason));
            log[k].cap_tenths = static_cast<std::uint16_t>(std::llround(cap * 10.0));
        }
        if (recs) {  // the sim's DecisionRecord (sim.hpp:438-440, 457-464)
            DecisionRecord dr;
            dr.t_s = t1;
            dr.point = d.point;
            dr.applied = d.applied;
            dr.reason = d.reason;
            dr.err_norm = target_tps > 0.0 ? (target_tps - measured) / target_tps : 0.0;
            dr.bias = st.bias;
            recs->push_back(dr);
        }
        applied_cap = inflight_cap;
        if (d.applied) {
            batch_cap = d.point.batch;
            inflight_cap = d.point.cap_watts;
        }
    }
    std::uint64_t bias_bits;
    std::memcpy(&bias_bits, &st.bias, 8);
    const int final_idx = index_of(rm.cands, st.current);
    h = (h ^ bias_bits) * kFnvPrime;
    h = (h ^ static_cast<std::uint64_t>(static_cast<std::uint32_t>(final_idx))) * kFnvPrime;
    summary->digest = h;
    summary->final_bias = st.bias;
    summary->energy_j = energy;
    summary->tokens = tokens;
    summary->n_applied = n_applied;
    summary->final_idx = final_idx;
    summary->model = m;
    summary->objective = obj;
}

// The same plant under caller traces (pals_replay_traces): budget and offered load are
// the reference's own detail::trace_value (sim.hpp:167-174) of the caller's signals at
// t0 = (first_step + k) * interval (Simulator::run, sim.hpp:229-231); initial and final
// ControllerState / actuation state as given.
void replay_trace_one(const std::vector<ReplayModel>& models, const GpuSpec& gpu,
                      const SystemPowerCoeffs& coeffs, const ControllerConfig& cfg,
                      const pals_trace_batch& b, std::int64_t i) {
    const pals_trace& tr = b.traces[i];
    const ReplayModel& rm = models.at(tr.model);
    std::vector<std::pair<double, double>> budget, load;
    for (int j = 0; j < tr.n_budget; ++j)
        budget.emplace_back(b.signal[tr.budget_off + j].t_s, b.signal[tr.budget_off + j].value);
    for (int j = 0; j < tr.n_load; ++j)
        load.emplace_back(b.signal[tr.load_off + j].t_s, b.signal[tr.load_off + j].value);
    const OperatingPoint& first = rm.cands.front();
    double max_cap = first.cap_watts;
    int max_batch = first.batch;
    for (const auto& c : rm.cands) {
        max_cap = std::max(max_cap, c.cap_watts);
        max_batch = std::max(max_batch, c.batch);
    }
    const int tp = first.tp, ep = first.ep, dp = first.dp;
    detail::NodeRuntime n;  // only the fields enforce_cap reads
    n.profile = &rm.profile;
    n.cfg.tp = tp;
    n.cfg.ep = ep;
    n.cfg.dp = dp;
    ControllerState st;
    st.current = OperatingPoint{max_cap, max_batch, tp, ep, dp};
    if (b.init) st = to_state(b.init[i]);
    double applied_cap = max_cap, inflight_cap = max_cap;
    int batch_cap = max_batch;
    if (b.init_plant) {
        applied_cap = b.init_plant[i].applied_cap_w;
        inflight_cap = b.init_plant[i].inflight_cap_w;
        batch_cap = b.init_plant[i].batch_cap;
    }
    const int obj = tr.objective;
    std::uint64_t h = kFnvOffset;
    double energy = 0.0, tokens = 0.0;
    int n_applied = 0;
    const bool logging = b.logs && i < b.n_log_traces;
    for (int k = 0; k < b.n_steps; ++k) {
        const std::int64_t step = b.first_step + k;
        const double t0 = step * b.interval_s;
        const double t1 = t0 + b.interval_s;
        n.node_budget = budget.empty() ? 0.0 : detail::trace_value(budget, t0);
        const int b_eff = batch_cap;
        const double cap = detail::enforce_cap(applied_cap, b_eff, n, gpu, coeffs);
        const OperatingPoint p{cap, b_eff, tp, ep, dp};
        const double capacity = cluster_throughput(p, rm.profile, gpu);
        const double gpu_w = avg_gpu_power(p, rm.profile, gpu);
        const double sys_w = dp * (coeffs.alpha * kGpusPerNode * gpu_w + coeffs.beta_watts);
        const double offered = detail::trace_value(load, t0);
        const double noise =
            1.0 + tr.noise_amp * (2.0 * noise_u(tr.noise_key, static_cast<std::uint64_t>(step)) - 1.0);
        const double measured = std::min(offered, capacity) * noise;
        energy += sys_w * b.interval_s;
        tokens += measured * b.interval_s;
        Targets targets;
        targets.throughput_tps = tr.target_tps;
        targets.epsilon = tr.epsilon;
        targets.objective =
            obj == PALS_OBJ_BUDGET ? Objective::BudgetMaxThroughput : Objective::QosMaxEfficiency;
        if (n.node_budget > 0.0) targets.power_budget_w = n.node_budget;
        auto [d, st2] = control_step(TelemetryInput{t1, measured}, t1, targets, rm.cands,
                                     rm.scorer, coeffs, st, cfg);
        st = st2;
        const int idx = index_of(rm.cands, d.point);
        const std::uint64_t word = (static_cast<std::uint64_t>(static_cast<std::uint32_t>(idx)) << 8) |
                                   (static_cast<std::uint64_t>(d.applied ? 1 : 0) << 4) |
                                   static_cast<std::uint64_t>(reason_code(d.reason));
        h = (h ^ word) * kFnvPrime;
        if (d.applied) ++n_applied;
        if (logging) {
            pals_step_log& lg = b.logs[i * b.n_steps + k];
            lg.idx = idx;
            lg.applied = d.applied ? 1 : 0;
            lg.reason = static_cast<std::uint8_t>(reason_code(d.reason));
            lg.cap_tenths = static_cast<std::uint16_t>(std::llround(cap * 10.0));
            if (b.details) {
                pals_step_detail& dt = b.details[i * b.n_steps + k];
                dt.err_norm = tr.target_tps > 0.0 ? (tr.target_tps - measured) / tr.target_tps : 0.0;
                dt.bias = st.bias;
            }
        }
        applied_cap = inflight_cap;
        if (d.applied) {
            batch_cap = d.point.batch;
            inflight_cap = d.point.cap_watts;
        }
    }
    std::uint64_t bias_bits;
    std::memcpy(&bias_bits, &st.bias, 8);
    const int final_idx = index_of(rm.cands, st.current);
    h = (h ^ bias_bits) * kFnvPrime;
    h = (h ^ static_cast<std::uint64_t>(static_cast<std::uint32_t>(final_idx))) * kFnvPrime;
    pals_trace_summary& sm = b.summaries[i];
    sm.digest = h;
    sm.final_bias = st.bias;
    sm.energy_j = energy;
    sm.tokens = tokens;
    sm.n_applied = n_applied;
    sm.final_idx = final_idx;
    sm.model = tr.model;
    sm.objective = obj;
    if (b.final_state) {
        if (b.n_steps == 0 && b.init) b.final_state[i] = b.init[i];
        else b.final_state[i] = from_state(st);
    }
    if (b.final_plant) {
        pals_plant_state ps{};
        ps.applied_cap_w = applied_cap;
        ps.inflight_cap_w = inflight_cap;
        ps.batch_cap = batch_cap;
        b.final_plant[i] = ps;
    }
}

std::vector<ReplayModel> build_replay_models(int n_models, const pals_profile* plant,
                                             const GpuSpec& gpu, const SystemPowerCoeffs& coeffs,
                                             const double* caps, int n_caps,
                                             const int* batches, int n_batches, bool memo) {
    std::vector<ReplayModel> models(n_models);
    for (int i = 0; i < n_models; ++i) {
        auto& rm = models[i];
        rm.profile = to_profile(plant[i]);
        const int tp = plant[i].deploy_tp, ep = plant[i].deploy_ep, dp = plant[i].deploy_dp;
        // build_candidates order (sim.hpp:304-306)
        for (int a = 0; a < n_caps; ++a)
            for (int b = 0; b < n_batches; ++b)
                rm.cands.push_back(OperatingPoint{caps[a], batches[b], tp, ep, dp});
        Scorer s = analytic_scorer(rm.profile, gpu);
        rm.scorer = memo ? detail::cached(s) : s;
        // unconstrained_throughput (sim.hpp:258-264)
        const double mc = *std::max_element(caps, caps + n_caps);
        const int mb = *std::max_element(batches, batches + n_batches);
        rm.t_max = dp * throughput(OperatingPoint{mc, mb, tp, ep, dp}, rm.profile, gpu);
        bool firstp = true;
        for (const auto& c : rm.cands) {
            const double pn = cluster_system_power(c, rm.profile, gpu, coeffs);
            if (firstp || pn < rm.p_min) rm.p_min = pn;
            if (firstp || pn > rm.p_max) rm.p_max = pn;
            firstp = false;
        }
    }
    return models;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// throughput() and avg_gpu_power() per point (model.hpp:72-84); err[i] = PALS code
int ref_eval(const pals_profile* prof, const pals_gpu_spec* gpu, const pals_point* pts,
             std::int64_t n, double* T, double* P, int* err) {
    const ModelProfile mp = to_profile(*prof);
    const GpuSpec g = to_gpu(*gpu);
    int rc = PALS_OK;
    for (std::int64_t i = 0; i < n; ++i) {
        try {
            const OperatingPoint p = to_point(pts[i]);
            T[i] = throughput(p, mp, g);
            P[i] = avg_gpu_power(p, mp, g);
            err[i] = PALS_OK;
        } catch (...) {
            err[i] = map_exception();
            T[i] = P[i] = std::nan("");
            rc = err[i];
        }
    }
    return rc;
}

double ref_effective_frequency(double cap, const pals_profile* prof, const pals_gpu_spec* gpu,
                               int* err) {
    try {
        *err = PALS_OK;
        return effective_frequency(cap, to_gpu(*gpu), to_profile(*prof));
    } catch (...) {
        *err = map_exception();
        return std::nan("");
    }
}

// ModelProfile::validate (types.hpp:88-106) + GpuSpec::validate
int ref_validate(const pals_profile* prof, const pals_gpu_spec* gpu) {
    try {
        const GpuSpec g = to_gpu(*gpu);
        g.validate();
        to_profile(*prof).validate(g);
        return PALS_OK;
    } catch (...) {
        return map_exception();
    }
}

// select_config with analytic_scorer (controller.hpp:107-111, 132-201)
int ref_select_analytic(const pals_profile* prof, const pals_gpu_spec* gpu,
                        const pals_point* pts, std::int64_t n, const pals_coeffs* coeffs,
                        const pals_query* q, std::int64_t nq, std::int32_t* idx,
                        std::uint8_t* reason) {
    const ModelProfile mp = to_profile(*prof);
    const GpuSpec g = to_gpu(*gpu);
    std::vector<OperatingPoint> cands;
    for (std::int64_t i = 0; i < n; ++i) cands.push_back(to_point(pts[i]));
    const Scorer s = analytic_scorer(mp, g);
    const SystemPowerCoeffs k{coeffs->alpha, coeffs->beta_watts};
    try {
        for (std::int64_t j = 0; j < nq; ++j) {
            const auto d = select_config(cands, query_targets(q[j]), s, k, q[j].bias,
                                         q[j].target_headroom, q[j].budget_margin);
            idx[j] = index_of(cands, d.point);
            reason[j] = static_cast<std::uint8_t>(reason_code(d.reason));
        }
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

// select_config with a TableScorer (tests/test_controller.cpp:17-29)
int ref_select_table(const pals_point* pts, std::int64_t n, const double* T, const double* P,
                     const pals_coeffs* coeffs, const pals_query* q, std::int64_t nq,
                     std::int32_t* idx, std::uint8_t* reason) {
    std::vector<OperatingPoint> cands;
    for (std::int64_t i = 0; i < n; ++i) cands.push_back(to_point(pts[i]));
    const Scorer s = table_scorer(cands, T, P);
    const SystemPowerCoeffs k{coeffs->alpha, coeffs->beta_watts};
    try {
        for (std::int64_t j = 0; j < nq; ++j) {
            const auto d = select_config(cands, query_targets(q[j]), s, k, q[j].bias,
                                         q[j].target_headroom, q[j].budget_margin);
            idx[j] = index_of(cands, d.point);
            reason[j] = static_cast<std::uint8_t>(reason_code(d.reason));
        }
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

// control_step with a TableScorer (controller.hpp:210-267)
int ref_control_step_table(const pals_point* pts, std::int64_t n, const double* T,
                           const double* P, const pals_telemetry* tel, double now_s,
                           const pals_targets* targets, const pals_coeffs* coeffs,
                           const pals_ctrl_state* state, const pals_ctrl_cfg* cfg,
                           pals_decision* out_d, pals_ctrl_state* out_s) {
    std::vector<OperatingPoint> cands;
    for (std::int64_t i = 0; i < n; ++i) cands.push_back(to_point(pts[i]));
    const Scorer s = table_scorer(cands, T, P);
    try {
        auto [d, st] = control_step(TelemetryInput{tel->t_s, tel->throughput_tps}, now_s,
                                    to_targets(*targets), cands, s,
                                    SystemPowerCoeffs{coeffs->alpha, coeffs->beta_watts},
                                    to_state(*state), to_cfg(*cfg));
        out_d->point = from_point(d.point);
        out_d->applied = d.applied ? 1 : 0;
        out_d->reason = reason_code(d.reason);
        *out_s = from_state(st);
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

// control_step with analytic_scorer
int ref_control_step_analytic(const pals_profile* prof, const pals_gpu_spec* gpu,
                              const pals_point* pts, std::int64_t n, const pals_telemetry* tel,
                              double now_s, const pals_targets* targets,
                              const pals_coeffs* coeffs, const pals_ctrl_state* state,
                              const pals_ctrl_cfg* cfg, pals_decision* out_d,
                              pals_ctrl_state* out_s) {
    const ModelProfile mp = to_profile(*prof);
    const GpuSpec g = to_gpu(*gpu);
    std::vector<OperatingPoint> cands;
    for (std::int64_t i = 0; i < n; ++i) cands.push_back(to_point(pts[i]));
    const Scorer s = analytic_scorer(mp, g);
    try {
        auto [d, st] = control_step(TelemetryInput{tel->t_s, tel->throughput_tps}, now_s,
                                    to_targets(*targets), cands, s,
                                    SystemPowerCoeffs{coeffs->alpha, coeffs->beta_watts},
                                    to_state(*state), to_cfg(*cfg));
        out_d->point = from_point(d.point);
        out_d->applied = d.applied ? 1 : 0;
        out_d->reason = reason_code(d.reason);
        *out_s = from_state(st);
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

// Reference control_step driven by the fluid plant, traces [0, n) of spec.
int ref_replay(int n_models, const pals_profile* plant, const pals_gpu_spec* gpu,
               const pals_coeffs* coeffs, const double* caps, int n_caps, const int* batches,
               int n_batches, const pals_ctrl_cfg* cfg, const pals_replay_spec* spec,
               pals_trace_summary* summaries, pals_step_log* logs) {
    try {
        const GpuSpec g = to_gpu(*gpu);
        const SystemPowerCoeffs k{coeffs->alpha, coeffs->beta_watts};
        const auto models =
            build_replay_models(n_models, plant, g, k, caps, n_caps, batches, n_batches, true);
        const ControllerConfig c = to_cfg(*cfg);
        for (std::int64_t i = 0; i < spec->n_traces; ++i) {
            pals_step_log* lg =
                (logs && i < spec->n_log_traces) ? logs + i * spec->n_steps : nullptr;
            replay_one(models, g, k, c, *spec, spec->first_trace + i, &summaries[i], lg);
        }
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

// decisions_csv (metrics.hpp:145-157, unmodified) over the first n_log_traces traces
// of a fluid-plant replay, one SimResult node per trace; plus its fnv1a64.
int ref_replay_decisions_csv(int n_models, const pals_profile* plant, const pals_gpu_spec* gpu,
                             const pals_coeffs* coeffs, const double* caps, int n_caps,
                             const int* batches, int n_batches, const pals_ctrl_cfg* cfg,
                             const pals_replay_spec* spec, char* buf, std::int64_t buf_size,
                             std::int64_t* out_len, std::uint64_t* fnv) {
    try {
        const GpuSpec g = to_gpu(*gpu);
        const SystemPowerCoeffs k{coeffs->alpha, coeffs->beta_watts};
        const auto models =
            build_replay_models(n_models, plant, g, k, caps, n_caps, batches, n_batches, true);
        const ControllerConfig c = to_cfg(*cfg);
        const std::int64_t nl = std::min<std::int64_t>(spec->n_log_traces, spec->n_traces);
        SimResult r;
        r.nodes.resize(nl);
        for (std::int64_t i = 0; i < nl; ++i) {
            pals_trace_summary s;
            replay_one(models, g, k, c, *spec, spec->first_trace + i, &s, nullptr,
                       &r.nodes[i].decisions);
            r.nodes[i].model_id = models[s.model].profile.name;
        }
        const std::string csv = decisions_csv(r);
        *out_len = static_cast<std::int64_t>(csv.size());
        *fnv = fnv1a64(csv);
        if (buf) std::memcpy(buf, csv.data(), std::min<std::size_t>(csv.size(), buf_size));
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

// ---- CPU baseline timing (all host threads) ------------------------------
// select_config + analytic_scorer over queries split across threads.
// Returns wall seconds; idx/reason receive the results.
double ref_bench_select(const pals_profile* prof, const pals_gpu_spec* gpu,
                        const pals_point* pts, std::int64_t n, const pals_coeffs* coeffs,
                        const pals_query* q, std::int64_t nq, int n_threads, std::int32_t* idx,
                        std::uint8_t* reason) {
    const ModelProfile mp = to_profile(*prof);
    const GpuSpec g = to_gpu(*gpu);
    std::vector<OperatingPoint> cands;
    for (std::int64_t i = 0; i < n; ++i) cands.push_back(to_point(pts[i]));
    const SystemPowerCoeffs k{coeffs->alpha, coeffs->beta_watts};
    std::atomic<int> failed{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t) {
        th.emplace_back([&, t] {
            const Scorer s = analytic_scorer(mp, g);
            const std::int64_t lo = nq * t / n_threads, hi = nq * (t + 1) / n_threads;
            try {
                for (std::int64_t j = lo; j < hi; ++j) {
                    const auto d = select_config(cands, query_targets(q[j]), s, k, q[j].bias,
                                                 q[j].target_headroom, q[j].budget_margin);
                    // the reference returns the point by value; its index is a cheap scan
                    // only when the caller asks for it
                    if (idx) {
                        idx[j] = index_of(cands, d.point);
                        reason[j] = static_cast<std::uint8_t>(reason_code(d.reason));
                    }
                }
            } catch (...) {
                failed = 1;
            }
        });
    }
    for (auto& x : th) x.join();
    const auto t1 = std::chrono::steady_clock::now();
    if (failed) return -1.0;
    return std::chrono::duration<double>(t1 - t0).count();
}

// Fluid-plant replay through the reference control_step, traces split across threads.
double ref_bench_replay(int n_models, const pals_profile* plant, const pals_gpu_spec* gpu,
                        const pals_coeffs* coeffs, const double* caps, int n_caps,
                        const int* batches, int n_batches, const pals_ctrl_cfg* cfg,
                        const pals_replay_spec* spec, int n_threads,
                        pals_trace_summary* summaries) {
    const GpuSpec g = to_gpu(*gpu);
    const SystemPowerCoeffs k{coeffs->alpha, coeffs->beta_watts};
    const ControllerConfig c = to_cfg(*cfg);
    std::atomic<int> failed{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t) {
        th.emplace_back([&, t] {
            try {
                // per-thread memo: detail::cached is not thread-safe (sim.hpp:179-190)
                const auto models = build_replay_models(n_models, plant, g, k, caps, n_caps,
                                                        batches, n_batches, true);
                const std::int64_t lo = spec->n_traces * t / n_threads;
                const std::int64_t hi = spec->n_traces * (t + 1) / n_threads;
                for (std::int64_t i = lo; i < hi; ++i)
                    replay_one(models, g, k, c, *spec, spec->first_trace + i, &summaries[i],
                               nullptr);
            } catch (...) {
                failed = 1;
            }
        });
    }
    for (auto& x : th) x.join();
    const auto t1 = std::chrono::steady_clock::now();
    if (failed) return -1.0;
    return std::chrono::duration<double>(t1 - t0).count();
}

// Reference control_step over caller traces (the pals_replay_traces contract), traces
// split across n_threads; *seconds receives the wall time.
int ref_replay_traces(int n_models, const pals_profile* plant, const pals_gpu_spec* gpu,
                      const pals_coeffs* coeffs, const double* caps, int n_caps,
                      const int* batches, int n_batches, const pals_ctrl_cfg* cfg,
                      const pals_trace_batch* batch, int n_threads, double* seconds) {
    const GpuSpec g = to_gpu(*gpu);
    const SystemPowerCoeffs k{coeffs->alpha, coeffs->beta_watts};
    const ControllerConfig c = to_cfg(*cfg);
    std::atomic<int> failed{0};
    std::string err;
    std::mutex mu;
    n_threads = std::max(1, n_threads);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t) {
        th.emplace_back([&, t] {
            try {
                const auto models = build_replay_models(n_models, plant, g, k, caps, n_caps,
                                                        batches, n_batches, true);
                const std::int64_t lo = batch->n_traces * t / n_threads;
                const std::int64_t hi = batch->n_traces * (t + 1) / n_threads;
                for (std::int64_t i = lo; i < hi; ++i) replay_trace_one(models, g, k, c, *batch, i);
            } catch (...) {
                std::lock_guard<std::mutex> l(mu);
                const int rc = map_exception();
                if (!failed) {
                    failed = rc;
                    err = g_err;
                }
            }
        });
    }
    for (auto& x : th) x.join();
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (failed) {
        g_err = err;
        return failed;
    }
    return PALS_OK;
}

std::uint64_t ref_splitmix64(std::uint64_t x) { return splitmix64(x); }

}  // extern "C"

extern "C" {

// profile_from_json (json_io.hpp:70-95) + validate, flattened to pals_profile
int ref_load_profile(const char* path, pals_profile* out) {
    try {
        const ModelProfile p = profile_from_json(parse_json_file(path));
        std::memset(out, 0, sizeof *out);
        std::strncpy(out->name, p.name.c_str(), sizeof(out->name) - 1);
        out->compute_fixed = p.compute_fixed;
        out->compute_per_seq = p.compute_per_seq;
        out->comm_per_seq = p.comm_per_seq;
        out->internode_factor = p.internode_factor;
        out->knee_watts = p.knee_watts;
        out->compute_power_base = p.compute_power_base;
        out->compute_power_per_seq = p.compute_power_per_seq;
        out->comm_power = p.comm_power;
        out->overlap = p.overlap;
        out->total_params_b = p.total_params_b;
        out->active_params_b = p.active_params_b;
        int i = 0;
        for (const auto& [tp, v] : p.comm_fixed_by_tp) {
            if (i >= PALS_MAX_TP_KEYS) throw config_error("too many tp keys");
            out->tp_keys[i] = tp;
            out->comm_fixed[i] = v;
            ++i;
        }
        out->n_tp = i;
        out->num_experts = p.num_experts;
        out->top_k = p.top_k;
        out->deploy_tp = p.deployment.tp;
        out->deploy_ep = p.deployment.ep;
        out->deploy_dp = p.deployment.dp;
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

// platform_from_json (json_io.hpp:103-105)
int ref_load_platform(const char* path, pals_gpu_spec* gpu, pals_coeffs* coeffs) {
    try {
        const Platform p = platform_from_json(parse_json_file(path));
        gpu->idle_watts = p.gpu.idle_watts;
        gpu->min_cap_watts = p.gpu.min_cap_watts;
        gpu->max_cap_watts = p.gpu.max_cap_watts;
        gpu->max_frequency = p.gpu.max_frequency;
        coeffs->alpha = p.coeffs.alpha;
        coeffs->beta_watts = p.coeffs.beta_watts;
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

}  // extern "C"

// ---- cluster budget allocator (allocator.hpp) -----------------------------
extern "C" {

// allocate_budget (allocator.hpp:76-186) for n_problems independent clusters.
// Node j of problem p: nodes [off[p], off[p+1]); node_model selects one of the
// n_models (profile, candidate grid) pairs: candidates = caps x batches at the
// profile's deployment tp/ep with degree node_dp[j] for dp, scored by the
// analytic scorer. status[p] = PALS code (config_error when the budget is below
// the sum of node floors).
int ref_allocate(int n_models, const pals_profile* profs, const pals_gpu_spec* gpu,
                 const pals_coeffs* coeffs, const double* caps, int n_caps, const int* batches,
                 int n_batches, double quantum_w, double margin, std::int64_t n_problems,
                 const std::int64_t* off, const std::int32_t* node_model,
                 const std::int32_t* node_dp, const double* node_target,
                 const double* cluster_budget, double* node_budget, double* total,
                 std::uint8_t* all_sat, std::int32_t* status) {
    const GpuSpec g = to_gpu(*gpu);
    const SystemPowerCoeffs k{coeffs->alpha, coeffs->beta_watts};
    std::vector<ModelProfile> mps;
    for (int m = 0; m < n_models; ++m) mps.push_back(to_profile(profs[m]));
    for (std::int64_t p = 0; p < n_problems; ++p) {
        std::vector<AllocRequest> reqs;
        for (std::int64_t j = off[p]; j < off[p + 1]; ++j) {
            const ModelProfile& mp = mps[node_model[j]];
            AllocRequest r;
            r.model_id = mp.name;
            r.throughput_target_tps = node_target[j];
            r.dp = node_dp[j];
            for (int a = 0; a < n_caps; ++a)
                for (int b = 0; b < n_batches; ++b)
                    r.candidates.push_back(OperatingPoint{caps[a], batches[b], mp.deployment.tp,
                                                          mp.deployment.ep, node_dp[j]});
            r.score = analytic_scorer(mps[node_model[j]], g);
            reqs.push_back(std::move(r));
        }
        try {
            const auto res = allocate_budget(reqs, cluster_budget[p], g, k, quantum_w, margin);
            for (std::size_t i = 0; i < reqs.size(); ++i)
                node_budget[off[p] + i] = res.node_budgets_w[i];
            total[p] = res.total_allocated_w;
            all_sat[p] = res.all_targets_satisfied ? 1 : 0;
            status[p] = PALS_OK;
        } catch (...) {
            status[p] = map_exception();
        }
    }
    return PALS_OK;
}

// all host threads, for the CPU baseline
double ref_bench_allocate(int n_models, const pals_profile* profs, const pals_gpu_spec* gpu,
                          const pals_coeffs* coeffs, const double* caps, int n_caps,
                          const int* batches, int n_batches, double quantum_w, double margin,
                          std::int64_t n_problems, const std::int64_t* off,
                          const std::int32_t* node_model, const std::int32_t* node_dp,
                          const double* node_target, const double* cluster_budget,
                          double* node_budget, double* total, std::uint8_t* all_sat,
                          std::int32_t* status, int n_threads) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t) {
        th.emplace_back([&, t] {
            const std::int64_t lo = n_problems * t / n_threads;
            const std::int64_t hi = n_problems * (t + 1) / n_threads;
            ref_allocate(n_models, profs, gpu, coeffs, caps, n_caps, batches, n_batches,
                         quantum_w, margin, hi - lo, off + lo, node_model, node_dp, node_target,
                         cluster_budget + lo, node_budget, total + lo, all_sat + lo, status + lo);
        });
    }
    for (auto& x : th) x.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"

// ---- tree-ensemble predictor (forest.hpp) ---------------------------------
namespace {
struct BundleCache {
    std::string path;
    PredictorBundle b;
};
thread_local BundleCache g_bundle;

const PredictorBundle& load_bundle(const char* path) {
    if (g_bundle.path != path) {
        g_bundle.b = bundle_from_json(parse_json_file(path));
        g_bundle.path = path;
    }
    return g_bundle.b;
}
}  // namespace

extern "C" {

// cmd_profile + cmd_train without the holdout split: run_sweep (sweep.hpp:123-170)
// with the AnalyticBackend over SweepGrid::default_grid() for every profile, then
// train_bundle (forest.hpp:271-296); the bundle is written with bundle_to_json.
int ref_train_bundle(const pals_profile* profs, int n, const pals_gpu_spec* gpu,
                     const pals_coeffs* coeffs, int n_trees, int max_depth, int min_leaf,
                     std::uint64_t seed, const char* out_path) {
    try {
        const GpuSpec g = to_gpu(*gpu);
        const SystemPowerCoeffs k{coeffs->alpha, coeffs->beta_watts};
        AnalyticBackend be(g, k);
        const SweepGrid grid = SweepGrid::default_grid();
        std::vector<ProfilingRecord> all;
        for (int i = 0; i < n; ++i) {
            const ModelProfile mp = to_profile(profs[i]);
            const auto ds = run_sweep(grid, mp.name, mp, g, be, seed + static_cast<std::uint64_t>(i));
            all.insert(all.end(), ds.records.begin(), ds.records.end());
        }
        HyperParams hp;
        hp.n_trees = n_trees;
        hp.max_depth = max_depth;
        hp.min_leaf = min_leaf;
        const PredictorBundle b = train_bundle(all, k, hp, seed);
        write_json_file(out_path, bundle_to_json(b));
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

// PredictorBundle::predict (forest.hpp:227-235) for each point
int ref_bundle_predict(const char* path, const char* model_id, const pals_point* pts,
                       std::int64_t n, double* T, double* P, double* E) {
    try {
        const PredictorBundle& b = load_bundle(path);
        for (std::int64_t i = 0; i < n; ++i) {
            const auto m = b.predict(to_point(pts[i]), model_id);
            T[i] = m.throughput_hat;
            P[i] = m.power_hat;
            E[i] = m.efficiency_hat;
        }
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

// select_config with predictor_scorer (controller.hpp:100-105)
int ref_select_forest(const char* path, const char* model_id, const pals_point* pts,
                      std::int64_t n, const pals_coeffs* coeffs, const pals_query* q,
                      std::int64_t nq, std::int32_t* idx, std::uint8_t* reason) {
    try {
        const PredictorBundle& b = load_bundle(path);
        std::vector<OperatingPoint> cands;
        for (std::int64_t i = 0; i < n; ++i) cands.push_back(to_point(pts[i]));
        const Scorer s = predictor_scorer(b, model_id);
        const SystemPowerCoeffs k{coeffs->alpha, coeffs->beta_watts};
        for (std::int64_t j = 0; j < nq; ++j) {
            const auto d = select_config(cands, query_targets(q[j]), s, k, q[j].bias,
                                         q[j].target_headroom, q[j].budget_margin);
            idx[j] = index_of(cands, d.point);
            reason[j] = static_cast<std::uint8_t>(reason_code(d.reason));
        }
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

// PredictorBundle::predict throughput on all host threads (bench cpu_baseline)
double ref_bench_predict(const char* path, const char* model_id, const pals_point* pts,
                         std::int64_t n, int n_threads) {
    std::atomic<int> failed{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t) {
        th.emplace_back([&, t] {
            try {
                const PredictorBundle b = bundle_from_json(parse_json_file(path));
                (void)b;
            } catch (...) {
                failed = 1;
            }
        });
    }
    for (auto& x : th) x.join();
    th.clear();
    // the bundle load is setup, not the predict path: time predictions only
    std::vector<PredictorBundle> bs(n_threads);
    for (int t = 0; t < n_threads; ++t) bs[t] = bundle_from_json(parse_json_file(path));
    const auto t1 = std::chrono::steady_clock::now();
    (void)t0;
    for (int t = 0; t < n_threads; ++t) {
        th.emplace_back([&, t] {
            const std::int64_t lo = n * t / n_threads, hi = n * (t + 1) / n_threads;
            double acc = 0.0;
            try {
                for (std::int64_t i = lo; i < hi; ++i)
                    acc += bs[t].predict(to_point(pts[i]), model_id).throughput_hat;
            } catch (...) {
                failed = 1;
            }
            if (acc == -1.0) failed = 1;
        });
    }
    for (auto& x : th) x.join();
    const auto t2 = std::chrono::steady_clock::now();
    if (failed) return -1.0;
    return std::chrono::duration<double>(t2 - t1).count();
}

// ---- Pareto frontier (pareto.hpp) ------------------------------------------
static void put_frontier(const std::vector<FrontierPoint>& f, pals_point* out_pts,
                         double* out_thr, double* out_eff, std::int64_t* out_n) {
    *out_n = (std::int64_t)f.size();
    for (std::size_t i = 0; i < f.size(); ++i) {
        out_pts[i] = from_point(f[i].point);
        out_thr[i] = f[i].throughput_tps;
        out_eff[i] = f[i].efficiency_tpj;
    }
}

// build_frontier (pareto.hpp:31-59) over explicit FrontierPoints
int ref_build_frontier(const pals_point* pts, const double* thr, const double* eff,
                       std::int64_t n, pals_point* out_pts, double* out_thr, double* out_eff,
                       std::int64_t* out_n) {
    try {
        std::vector<FrontierPoint> v;
        v.reserve((std::size_t)n);
        for (std::int64_t i = 0; i < n; ++i)
            v.push_back(FrontierPoint{to_point(pts[i]), thr[i], eff[i]});
        put_frontier(build_frontier(std::move(v)), out_pts, out_thr, out_eff, out_n);
        return PALS_OK;
    } catch (...) {
        return map_exception();
    }
}

// evaluate_regime (pareto.hpp:114-135) with a named preset (regime_by_name)
int ref_evaluate_regime(const char* regime, const pals_profile* prof, const pals_gpu_spec* gpu,
                        const pals_coeffs* k, const double* caps, int nc, const int* batches,
                        int nb, const int* tps, int nt, pals_point* out_pts, double* out_thr,
                        double* out_eff, std::int64_t* out_n) {
    try {
        const auto f = evaluate_regime(
            regime_by_name(regime), to_profile(*prof), to_gpu(*gpu),
            SystemPowerCoeffs{k->alpha, k->beta_watts}, std::vector<double>(caps, caps + nc),
            std::vector<int>(batches, batches + nb), std::vector<int>(tps, tps + nt));
        put_frontier(f, out_pts, out_thr, out_eff, out_n);
        return PALS_OK;
    } catch (...) {
        return map_exception();
    }
}

// verify_dominance (pareto.hpp:66-83): covered[j] = some point of a weakly dominates b[j]
int ref_verify_dominance(const double* a_thr, const double* a_eff, std::int64_t na,
                         const double* b_thr, const double* b_eff, std::int64_t nb,
                         std::uint8_t* covered, int* dominated) {
    std::vector<FrontierPoint> a, b;
    for (std::int64_t i = 0; i < na; ++i) a.push_back(FrontierPoint{{}, a_thr[i], a_eff[i]});
    for (std::int64_t i = 0; i < nb; ++i) b.push_back(FrontierPoint{{}, b_thr[i], b_eff[i]});
    const auto rep = verify_dominance(a, b);
    *dominated = rep.dominated ? 1 : 0;
    std::size_t w = 0;
    for (std::int64_t j = 0; j < nb; ++j) {
        const bool wit = w < rep.witnesses.size() && rep.witnesses[w].throughput_tps == b_thr[j] &&
                         rep.witnesses[w].efficiency_tpj == b_eff[j];
        covered[j] = wit ? 0 : 1;
        if (wit) ++w;
    }
    return PALS_OK;
}

// The reference's frontier of one dense grid: score every point (cluster_throughput,
// efficiency) then build_frontier, as evaluate_regime does; seconds for `reps` runs.
double ref_bench_frontier(const pals_profile* prof, const pals_gpu_spec* gpu, const pals_coeffs* k,
                          const pals_point* pts, std::int64_t n, int reps, std::int64_t* out_n) {
    const ModelProfile mp = to_profile(*prof);
    const GpuSpec g = to_gpu(*gpu);
    const SystemPowerCoeffs kc{k->alpha, k->beta_watts};
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) {
        std::vector<FrontierPoint> v;
        v.reserve((std::size_t)n);
        for (std::int64_t i = 0; i < n; ++i) {
            const OperatingPoint p = to_point(pts[i]);
            v.push_back(FrontierPoint{p, cluster_throughput(p, mp, g), efficiency(p, mp, g, kc)});
        }
        *out_n = (std::int64_t)build_frontier(std::move(v)).size();
    }
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"

// ---- queue-plant scenarios through the UNMODIFIED run_scenario (sim.hpp:482-485) --
namespace {
Scenario to_scenario(const pals_scenario& s, const pals_profile* profs) {
    Scenario sc;
    sc.name = "pals";
    sc.duration_s = s.duration_s;
    sc.interval_s = s.interval_s;
    sc.seed = s.seed;
    sc.output_len.mean_tokens = s.mean_tokens;
    sc.output_len.log_sigma = s.log_sigma;
    if (s.has_cluster_budget) sc.cluster_budget_w = s.cluster_budget_w;
    for (int i = 0; i < s.n_trace; ++i) sc.budget_trace.emplace_back(s.trace_t[i], s.trace_w[i]);
    const Policy pol[] = {Policy::Fixed, Policy::AdaptiveBatch, Policy::AdaptiveCap,
                          Policy::Joint, Policy::Oracle};
    sc.policy = pol[s.policy];
    sc.objective = s.objective == PALS_OBJ_BUDGET ? Objective::BudgetMaxThroughput
                                                  : Objective::QosMaxEfficiency;
    sc.controller = to_cfg(s.controller);
    sc.epsilon = s.epsilon;
    sc.cand_caps.assign(s.cand_caps, s.cand_caps + s.n_caps);
    sc.cand_batches.assign(s.cand_batches, s.cand_batches + s.n_batches);
    sc.initial_cap_w = s.initial_cap_w;
    sc.initial_batch = s.initial_batch;
    for (int i = 0; i < s.n_nodes; ++i) {
        const pals_sim_node& n = s.nodes[i];
        ScenarioNode sn;
        sn.model_id = profs[n.model].name;
        sn.qos_fraction = n.qos_fraction;
        sn.tp = n.tp;
        sn.ep = n.ep;
        sn.dp = n.dp;
        sn.arrival_rate_per_s = n.arrival_rate_per_s;
        sn.initial_backlog = n.initial_backlog;
        sc.nodes.push_back(sn);
    }
    return sc;
}
}  // namespace

extern "C" {

// run_scenario + summarize (metrics.hpp:24-102); bundle_path NULL = no predictor.
// Per-interval logs [node][interval] when tel / dec are non-NULL; csv receives the
// reference's telemetry_csv + decisions_csv texts (NUL-separated) when non-NULL.
int ref_run_scenario(const pals_scenario* s, int n_models, const pals_profile* profs,
                     const char* bundle_path, const pals_gpu_spec* gpu, const pals_coeffs* coeffs,
                     pals_sim_node_result* node_out, pals_sim_result* out, std::int64_t stride,
                     pals_sim_telemetry* tel, pals_sim_decision* dec, char* csv,
                     std::int64_t csv_cap, std::int64_t* csv_len) {
    try {
        ProfileRegistry reg;
        for (int m = 0; m < n_models; ++m) reg.add(to_profile(profs[m]));
        Platform plat{to_gpu(*gpu), SystemPowerCoeffs{coeffs->alpha, coeffs->beta_watts}};
        const PredictorBundle* b = bundle_path ? &load_bundle(bundle_path) : nullptr;
        const Scenario sc = to_scenario(*s, profs);
        const SimResult r = run_scenario(sc, reg, plat, b);
        const RunSummary rs = summarize(r);
        for (std::size_t i = 0; i < r.nodes.size(); ++i) {
            const NodeResult& nr = r.nodes[i];
            const MetricsSummary& m = rs.per_node.at(std::to_string(i) + ":" + nr.model_id);
            pals_sim_node_result& o = node_out[i];
            std::memset(&o, 0, sizeof o);
            o.tokens_per_joule = m.tokens_per_joule;
            o.qos_violation_rate = m.qos_violation_rate;
            o.power_tracking_mae_w = m.power_tracking_mae_w;
            o.total_tokens = m.total_tokens;
            o.total_energy_j = m.total_energy_j;
            o.mean_throughput_tps = m.mean_throughput_tps;
            o.throughput_target_tps = nr.throughput_target_tps;
            o.final_bias = nr.decisions.empty() ? 1.0 : nr.decisions.back().bias;
            o.arrival_stream_hash = nr.arrival_stream_hash;
            o.n_requests = static_cast<std::int64_t>(nr.requests.size());
            std::int64_t done = 0;
            for (const auto& q : nr.requests) done += q.done() ? 1 : 0;
            o.n_completed = done;
            int applied = 0;
            for (const auto& d : nr.decisions) applied += d.applied ? 1 : 0;
            o.n_applied = applied;
            o.final_idx = -1;
            for (std::size_t k = 0; k < nr.telemetry.size() && k < (std::size_t)stride; ++k) {
                if (tel) {
                    const TelemetrySample& t = nr.telemetry[k];
                    pals_sim_telemetry& x = tel[i * stride + k];
                    std::memset(&x, 0, sizeof x);
                    x.t_s = t.t_s;
                    x.gpu_power_w = t.gpu_power_w;
                    x.sys_power_w = t.sys_power_w;
                    x.throughput_tps = t.throughput_tps;
                    x.utilization = t.utilization;
                    x.node_budget_w = t.node_budget_w;
                    x.applied_cap_w = t.applied_cap_w;
                    x.queue_depth = t.queue_depth;
                    x.active_batch = t.active_batch;
                    x.applied_batch_cap = t.applied_batch_cap;
                }
                if (dec) {
                    const DecisionRecord& d = nr.decisions[k];
                    pals_sim_decision& x = dec[i * stride + k];
                    std::memset(&x, 0, sizeof x);
                    x.err_norm = d.err_norm;
                    x.bias = d.bias;
                    x.cap_w = d.point.cap_watts;
                    x.batch = d.point.batch;
                    x.applied = d.applied ? 1 : 0;
                    x.reason = static_cast<std::uint8_t>(reason_code(d.reason));
                }
            }
        }
        std::memset(out, 0, sizeof *out);
        out->tokens_per_joule = rs.aggregate.tokens_per_joule;
        out->qos_violation_rate = rs.aggregate.qos_violation_rate;
        out->power_tracking_mae_w = rs.aggregate.power_tracking_mae_w;
        out->total_tokens = rs.aggregate.total_tokens;
        out->total_energy_j = rs.aggregate.total_energy_j;
        out->mean_throughput_tps = rs.aggregate.mean_throughput_tps;
        out->cluster_tracking_mae_w = rs.cluster_tracking_mae_w;
        out->sim_total_energy_j = r.total_energy_j;
        out->n_intervals = r.nodes.empty() ? 0 : static_cast<int>(r.nodes[0].telemetry.size());
        if (csv_len) {
            const std::string text = telemetry_csv(r) + std::string(1, '\0') + decisions_csv(r) +
                                     std::string(1, '\0') + requests_csv(r);
            *csv_len = static_cast<std::int64_t>(text.size());
            if (csv) std::memcpy(csv, text.data(), std::min<std::size_t>(text.size(), csv_cap));
        }
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}

}  // extern "C"

extern "C" {
// CPU baseline: run_scenario + summarize over scenarios split across threads (wall s).
double ref_bench_scenarios(int n_scen, const pals_scenario* s, int n_models,
                           const pals_profile* profs, const char* bundle_path,
                           const pals_gpu_spec* gpu, const pals_coeffs* coeffs, int n_threads,
                           pals_sim_node_result* node_out, pals_sim_result* res_out) {
    if (bundle_path) load_bundle(bundle_path);  // parse once, before the threads share it
    std::vector<int> rc(n_scen, 0);
    std::vector<std::int64_t> node_off(n_scen + 1, 0);
    for (int i = 0; i < n_scen; ++i) node_off[i + 1] = node_off[i] + s[i].n_nodes;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    std::atomic<int> next{0};
    for (int t = 0; t < n_threads; ++t)
        th.emplace_back([&] {
            for (int i = next++; i < n_scen; i = next++) {
                std::vector<pals_sim_node_result> nr(s[i].n_nodes);
                pals_sim_result r;
                rc[i] = ref_run_scenario(&s[i], n_models, profs, bundle_path, gpu, coeffs,
                                         nr.data(), &r, 0, nullptr, nullptr, nullptr, 0, nullptr);
                if (node_out)
                    std::memcpy(node_out + node_off[i], nr.data(), nr.size() * sizeof(nr[0]));
                if (res_out) res_out[i] = r;
            }
        });
    for (auto& x : th) x.join();
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int v : rc)
        if (v) return -1.0;
    return secs;
}
}  // extern "C"

extern "C" {
// scenario_from_json (scenario_io.hpp:35-93) on a file, flattened to one text line
// per field ("%.17g" doubles) so a test can compare it with another parser's view.
int ref_scenario_digest(const char* path, char* buf, std::int64_t cap, std::int64_t* len) {
    try {
        const Scenario sc = load_scenario(path);
        auto g = [](double v) {
            char b[40];
            std::snprintf(b, sizeof b, "%.17g", v);
            return std::string(b);
        };
        std::string o;
        o += "name=" + sc.name + "\n";
        o += "duration_s=" + g(sc.duration_s) + "\ninterval_s=" + g(sc.interval_s) + "\n";
        o += "seed=" + std::to_string(sc.seed) + "\n";
        o += "mean_tokens=" + g(sc.output_len.mean_tokens) + "\nlog_sigma=" +
             g(sc.output_len.log_sigma) + "\n";
        o += "cluster_budget_w=" + (sc.cluster_budget_w ? g(*sc.cluster_budget_w) : "none") + "\n";
        o += "trace=";
        for (const auto& [t, w] : sc.budget_trace) o += g(t) + ":" + g(w) + ";";
        o += "\npolicy=" + std::string(to_string(sc.policy)) + "\n";
        o += std::string("objective=") +
             (sc.objective == Objective::QosMaxEfficiency ? "qos" : "budget-throughput") + "\n";
        const auto& c = sc.controller;
        o += "kp=" + g(c.gains.kp) + "\nki=" + g(c.gains.ki) + "\nkd=" + g(c.gains.kd) + "\n";
        o += "sustain_intervals=" + std::to_string(c.sustain_intervals) + "\n";
        o += "integral_clamp=" + g(c.integral_clamp) + "\ntarget_headroom=" +
             g(c.target_headroom) + "\nbudget_margin=" + g(c.budget_margin) + "\n";
        o += "epsilon=" + g(sc.epsilon) + "\ncaps=";
        for (double v : sc.cand_caps) o += g(v) + ";";
        o += "\nbatches=";
        for (int v : sc.cand_batches) o += std::to_string(v) + ";";
        o += "\ninitial=" + g(sc.initial_cap_w) + ":" + std::to_string(sc.initial_batch) + "\n";
        for (const auto& n : sc.nodes)
            o += "node=" + n.model_id + ":" + g(n.qos_fraction) + ":" + std::to_string(n.tp) +
                 ":" + std::to_string(n.ep) + ":" + std::to_string(n.dp) + ":" +
                 g(n.arrival_rate_per_s) + ":" + std::to_string(n.initial_backlog) + "\n";
        *len = static_cast<std::int64_t>(o.size());
        if (buf) std::memcpy(buf, o.data(), std::min<std::size_t>(o.size(), cap));
    } catch (...) {
        return map_exception();
    }
    return PALS_OK;
}
}  // extern "C"
