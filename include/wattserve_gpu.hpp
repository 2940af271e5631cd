// wattserve_gpu.hpp — drop-in C++ adapter: the reference's decision API
// (wattserve/controller.hpp) executed by libpals_gpu.so on a B200.
//
// A wattserve user swaps
//     wattserve::select_config(cands, targets, wattserve::analytic_scorer(prof, gpu), k)
// for
//     wattserve::gpu::select_config(cands, targets, wattserve::gpu::analytic_scorer(ctx, prof, gpu), k)
// with the same types, the same results bit for bit and the same exceptions
// (config_error / data_error / std::out_of_range, same messages). Scorers are the
// three concrete kinds the GPU can run (an arbitrary std::function cannot):
//   analytic_scorer   controller.hpp:107-111
//   predictor_scorer  controller.hpp:100-105 (PredictorBundle, forest.hpp:217-251)
//   table_scorer      the TableScorer test fake, tests/test_controller.cpp:17-29
// plus batched entry points (SelectPlan; replay over caller traces with ControllerState
// in and out) that have no single-call counterpart in the reference. Also allocate_budget (allocator.hpp:76-186) over
// GpuAllocRequest nodes, build_frontier / evaluate_regime (pareto.hpp:31-59,
// 114-135), and run_scenario / run_baseline_suite (sim.hpp:482-500) returning the
// reference's own SimResult.
//
// Header-only; include after the reference headers are on the include path and
// link libpals_gpu.so.
#pragma once

#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pals_gpu.h"
#include "wattserve/allocator.hpp"
#include "wattserve/controller.hpp"
#include "wattserve/forest.hpp"
#include "wattserve/json_io.hpp"
#include "wattserve/pareto.hpp"
#include "wattserve/sim.hpp"

namespace wattserve::gpu {

inline void check(int rc) {
    if (rc == PALS_OK) return;
    const std::string msg = pals_last_error();
    switch (rc) {
        case PALS_ECONFIG: throw config_error(msg);
        case PALS_EDATA: throw data_error(msg);
        case PALS_ERANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

inline pals_point to_c(const OperatingPoint& p) {
    pals_point o;
    o.cap_watts = p.cap_watts;
    o.batch = p.batch;
    o.tp = p.tp;
    o.ep = p.ep;
    o.dp = p.dp;
    return o;
}

inline OperatingPoint from_c(const pals_point& p) {
    return OperatingPoint{p.cap_watts, p.batch, p.tp, p.ep, p.dp};
}

inline pals_targets to_c(const Targets& t) {
    pals_targets o{};
    o.throughput_tps = t.throughput_tps;
    o.has_budget = t.power_budget_w.has_value() ? 1 : 0;
    o.power_budget_w = t.power_budget_w.value_or(0.0);
    o.epsilon = t.epsilon;
    o.objective = t.objective == Objective::BudgetMaxThroughput ? PALS_OBJ_BUDGET : PALS_OBJ_QOS;
    return o;
}

inline Targets from_c(const pals_targets& t) {
    Targets o;
    o.throughput_tps = t.throughput_tps;
    if (t.has_budget) o.power_budget_w = t.power_budget_w;
    o.epsilon = t.epsilon;
    o.objective = t.objective == PALS_OBJ_BUDGET ? Objective::BudgetMaxThroughput
                                                 : Objective::QosMaxEfficiency;
    return o;
}

inline pals_ctrl_cfg to_c(const ControllerConfig& c) {
    pals_ctrl_cfg o{};
    o.kp = c.gains.kp;
    o.ki = c.gains.ki;
    o.kd = c.gains.kd;
    o.integral_clamp = c.integral_clamp;
    o.bias_min = c.bias_min;
    o.bias_max = c.bias_max;
    o.interval_s = c.interval_s;
    o.target_headroom = c.target_headroom;
    o.budget_margin = c.budget_margin;
    o.sustain_intervals = c.sustain_intervals;
    return o;
}

inline pals_ctrl_state to_c(const ControllerState& s) {
    pals_ctrl_state o{};
    o.bias = s.bias;
    o.integral = s.integral;
    o.prev_error = s.prev_error;
    o.has_prev_error = s.has_prev_error ? 1 : 0;
    o.sustain_count = s.sustain_count;
    o.current = to_c(s.current);
    o.has_last_targets = s.last_targets.has_value() ? 1 : 0;
    if (s.last_targets) o.last_targets = to_c(*s.last_targets);
    return o;
}

inline ControllerState from_c(const pals_ctrl_state& s) {
    ControllerState o;
    o.bias = s.bias;
    o.integral = s.integral;
    o.prev_error = s.prev_error;
    o.has_prev_error = s.has_prev_error != 0;
    o.sustain_count = s.sustain_count;
    o.current = from_c(s.current);
    if (s.has_last_targets) o.last_targets = from_c(s.last_targets);
    return o;
}

inline pals_profile to_c(const ModelProfile& p) {
    pals_profile o{};
    std::snprintf(o.name, sizeof(o.name), "%s", p.name.c_str());
    o.compute_fixed = p.compute_fixed;
    o.compute_per_seq = p.compute_per_seq;
    o.comm_per_seq = p.comm_per_seq;
    o.internode_factor = p.internode_factor;
    o.knee_watts = p.knee_watts;
    o.compute_power_base = p.compute_power_base;
    o.compute_power_per_seq = p.compute_power_per_seq;
    o.comm_power = p.comm_power;
    o.overlap = p.overlap;
    o.total_params_b = p.total_params_b;
    o.active_params_b = p.active_params_b;
    int i = 0;
    for (const auto& [tp, v] : p.comm_fixed_by_tp) {
        if (i >= PALS_MAX_TP_KEYS) throw config_error(p.name + ": too many comm_fixed_by_tp keys");
        o.tp_keys[i] = tp;
        o.comm_fixed[i] = v;
        ++i;
    }
    o.n_tp = i;
    o.num_experts = p.num_experts;
    o.top_k = p.top_k;
    o.deploy_tp = p.deployment.tp;
    o.deploy_ep = p.deployment.ep;
    o.deploy_dp = p.deployment.dp;
    return o;
}

inline std::vector<pals_point> to_c(const std::vector<OperatingPoint>& v) {
    std::vector<pals_point> o;
    o.reserve(v.size());
    for (const auto& p : v) o.push_back(to_c(p));
    return o;
}

// One GPU, one stream.
class Context {
public:
    explicit Context(int device = 0) { check(pals_ctx_create(device, &h_)); }
    ~Context() { pals_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    pals_ctx* get() const { return h_; }
    // single calls through the resident server kernel (exits after idle_us idle; 0 = a
    // kernel launch per call)
    void set_one_server(int64_t idle_us) { check(pals_ctx_set_one_server(h_, idle_us)); }

private:
    pals_ctx* h_ = nullptr;
};

// A device-resident scorer (the GPU counterpart of wattserve::Scorer).
class GpuScorer {
public:
    GpuScorer(Context& ctx, pals_model* m) : ctx_(&ctx), m_(m, pals_model_destroy) {}
    pals_model* get() const { return m_.get(); }
    Context& context() const { return *ctx_; }

private:
    Context* ctx_;
    std::shared_ptr<pals_model> m_;
};

inline GpuScorer analytic_scorer(Context& ctx, const ModelProfile& profile, const GpuSpec& gpu) {
    const pals_profile p = to_c(profile);
    const pals_gpu_spec g{gpu.idle_watts, gpu.min_cap_watts, gpu.max_cap_watts, gpu.max_frequency};
    pals_model* m = nullptr;
    check(pals_model_analytic(ctx.get(), &p, &g, &m));
    return GpuScorer(ctx, m);
}

inline GpuScorer table_scorer(Context& ctx, const std::vector<OperatingPoint>& points,
                              const std::vector<double>& t_hat, const std::vector<double>& p_gpu) {
    const auto pts = to_c(points);
    pals_model* m = nullptr;
    check(pals_model_table(ctx.get(), pts.data(), t_hat.data(), p_gpu.data(),
                           static_cast<int64_t>(pts.size()), &m));
    return GpuScorer(ctx, m);
}

namespace detail {
struct SoA {
    std::vector<int64_t> off;
    std::vector<int32_t> f, l, r;
    std::vector<double> t, v;
};
inline SoA flatten(const Forest& forest) {
    SoA s;
    s.off.push_back(0);
    for (const auto& tree : forest.trees) {
        for (const auto& n : tree.nodes) {
            s.f.push_back(n.feature);
            s.t.push_back(n.threshold);
            s.l.push_back(n.left);
            s.r.push_back(n.right);
            s.v.push_back(n.value);
        }
        s.off.push_back(static_cast<int64_t>(s.f.size()));
    }
    return s;
}
}  // namespace detail

inline GpuScorer predictor_scorer(Context& ctx, const PredictorBundle& bundle,
                                  const std::string& model_id) {
    const int mi = bundle.schema.model_index(model_id);  // throws like encode() would
    const auto T = detail::flatten(bundle.throughput_forest);
    const auto P = detail::flatten(bundle.power_forest);
    const pals_coeffs k{bundle.coeffs.alpha, bundle.coeffs.beta_watts};
    pals_model* m = nullptr;
    check(pals_model_forest(ctx.get(), static_cast<int32_t>(bundle.schema.model_ids.size()), mi,
                            &k, static_cast<int32_t>(bundle.throughput_forest.trees.size()),
                            T.off.data(), T.f.data(), T.t.data(), T.l.data(), T.r.data(),
                            T.v.data(), static_cast<int32_t>(bundle.power_forest.trees.size()),
                            P.off.data(), P.f.data(), P.t.data(), P.l.data(), P.r.data(),
                            P.v.data(), &m));
    return GpuScorer(ctx, m);
}

// select_config (controller.hpp:132-201)
inline Decision select_config(const std::vector<OperatingPoint>& candidates,
                              const Targets& targets, const GpuScorer& score,
                              const SystemPowerCoeffs& coeffs, double bias = 1.0,
                              double target_headroom = 0.0, double budget_margin = 0.0) {
    const auto pts = to_c(candidates);
    const pals_targets t = to_c(targets);
    const pals_coeffs k{coeffs.alpha, coeffs.beta_watts};
    pals_decision d{};
    check(pals_select_one(score.context().get(), score.get(), pts.data(),
                          static_cast<int64_t>(pts.size()), &t, &k, bias, target_headroom,
                          budget_margin, &d));
    return Decision{from_c(d.point), d.applied != 0, static_cast<DecisionReason>(d.reason)};
}

// control_step (controller.hpp:210-267)
inline std::pair<Decision, ControllerState> control_step(
    const TelemetryInput& telemetry, double now_s, const Targets& targets,
    const std::vector<OperatingPoint>& candidates, const GpuScorer& score,
    const SystemPowerCoeffs& coeffs, const ControllerState& state, const ControllerConfig& cfg) {
    const auto pts = to_c(candidates);
    const pals_targets t = to_c(targets);
    const pals_coeffs k{coeffs.alpha, coeffs.beta_watts};
    const pals_telemetry tel{telemetry.t_s, telemetry.throughput_tps};
    const pals_ctrl_state st = to_c(state);
    const pals_ctrl_cfg c = to_c(cfg);
    pals_decision d{};
    pals_ctrl_state out{};
    check(pals_control_step_one(score.context().get(), score.get(), &tel, now_s, &t, pts.data(),
                                static_cast<int64_t>(pts.size()), &k, &st, &c, &d, &out));
    return {Decision{from_c(d.point), d.applied != 0, static_cast<DecisionReason>(d.reason)},
            from_c(out)};
}

// Many select_config calls over one candidate grid in one GPU pass.
class SelectPlan {
public:
    SelectPlan(Context& ctx, const GpuScorer& score, const std::vector<OperatingPoint>& candidates,
               const SystemPowerCoeffs& coeffs)
        : candidates_(candidates) {
        const auto pts = to_c(candidates);
        check(pals_grid_points(ctx.get(), pts.data(), static_cast<int64_t>(pts.size()), &grid_));
        const pals_coeffs k{coeffs.alpha, coeffs.beta_watts};
        check(pals_plan_create(ctx.get(), score.get(), grid_, &k, &plan_));
    }
    ~SelectPlan() {
        pals_plan_destroy(plan_);
        pals_grid_destroy(grid_);
    }
    SelectPlan(const SelectPlan&) = delete;
    SelectPlan& operator=(const SelectPlan&) = delete;

    // decisions[i] == wattserve::select_config(candidates, targets[i], score, coeffs,
    //                                          bias[i], headroom, margin)
    std::vector<Decision> select(const std::vector<Targets>& targets,
                                 const std::vector<double>& bias, double target_headroom = 0.0,
                                 double budget_margin = 0.0) {
        std::vector<pals_query> q(targets.size());
        for (std::size_t i = 0; i < q.size(); ++i) {
            q[i].throughput_tps = targets[i].throughput_tps;
            q[i].has_budget = targets[i].power_budget_w.has_value() ? 1 : 0;
            q[i].power_budget_w = targets[i].power_budget_w.value_or(0.0);
            q[i].bias = bias.empty() ? 1.0 : bias[i];
            q[i].target_headroom = target_headroom;
            q[i].budget_margin = budget_margin;
            q[i].objective = targets[i].objective == Objective::BudgetMaxThroughput
                                 ? PALS_OBJ_BUDGET
                                 : PALS_OBJ_QOS;
        }
        std::vector<int32_t> idx(q.size());
        std::vector<uint8_t> reason(q.size());
        check(pals_select(plan_, q.data(), static_cast<int64_t>(q.size()), idx.data(),
                          reason.data()));
        std::vector<Decision> out;
        out.reserve(q.size());
        for (std::size_t i = 0; i < q.size(); ++i)
            out.push_back(Decision{candidates_[static_cast<std::size_t>(idx[i])], true,
                                   static_cast<DecisionReason>(reason[i])});
        return out;
    }

private:
    std::vector<OperatingPoint> candidates_;
    pals_grid* grid_ = nullptr;
    pals_plan* plan_ = nullptr;
};

// ---- batched control_step replay over caller traces (pals_replay_traces) ----
// One node of the fluid plant under the caller's signals, in the
// reference's own representations: budget / load traces are the budget-trace rows
// std::vector<std::pair<double,double>> of scenario_io.hpp:13-25 read with
// detail::trace_value (sim.hpp:167-174); the controller state is ControllerState
// (controller.hpp:55-63); the actuation state is NodeRuntime's applied / inflight cap and
// batch cap (sim.hpp:155-157); per-step records are the sim's DecisionRecord
// (sim.hpp:122-129).
struct ReplayTrace {
    int model = 0;                 // index into the scorers / plant profiles
    Targets targets;               // throughput target, epsilon, objective (budget: below)
    std::vector<std::pair<double, double>> budget_trace;  // node watts (empty: unbudgeted)
    std::vector<std::pair<double, double>> load_trace;    // offered tokens/s (non-empty)
    double noise_amp = 0.0;        // measured *= 1 + amp * U(-1, 1) (pals_trace)
    std::uint64_t noise_key = 0;
};

struct PlantState {
    double applied_cap_w = 0.0;
    double inflight_cap_w = 0.0;
    int batch_cap = 0;
};

struct ReplayResult {
    std::vector<ControllerState> states;          // final state per trace
    std::vector<PlantState> plant;                // final actuation state per trace
    std::vector<pals_trace_summary> summaries;    // digest, energy, tokens, applied count
    std::vector<std::vector<DecisionRecord>> decisions;  // the first n_log_traces traces
};

// scorers[k] scores candidates caps x batches at plant[k]'s deployment tp/ep/dp
// (build_candidates order, sim.hpp:293-308); plant[k] is the true system. init /
// init_plant: nullptr = the sim's start, ControllerState{} at (max cap, max batch).
// Steps are global (first_step + k), so replay(…, K, …) then replay(…, first_step = K,
// init = &r.states, init_plant = &r.plant) equals one uninterrupted replay.
inline ReplayResult replay(Context& ctx, const std::vector<GpuScorer>& scorers,
                           const std::vector<ModelProfile>& plant, const GpuSpec& gpu,
                           const SystemPowerCoeffs& coeffs, const std::vector<double>& caps,
                           const std::vector<int>& batches, const ControllerConfig& cfg,
                           const std::vector<ReplayTrace>& traces, int n_steps,
                           double interval_s = 0.5, std::int64_t first_step = 0,
                           const std::vector<ControllerState>* init = nullptr,
                           const std::vector<PlantState>* init_plant = nullptr,
                           int n_log_traces = 0) {
    if (scorers.size() != plant.size())
        throw config_error("replay: one scorer per plant profile");
    std::vector<pals_model*> hs;
    std::vector<pals_profile> profs;
    for (std::size_t i = 0; i < plant.size(); ++i) {
        hs.push_back(scorers[i].get());
        profs.push_back(to_c(plant[i]));
    }
    const std::size_t n = traces.size();
    std::vector<pals_trace> tr(n);
    std::vector<pals_signal_point> sig;
    for (std::size_t i = 0; i < n; ++i) {
        const ReplayTrace& t = traces[i];
        pals_trace& c = tr[i];
        c.model = t.model;
        c.objective = t.targets.objective == Objective::BudgetMaxThroughput ? PALS_OBJ_BUDGET
                                                                            : PALS_OBJ_QOS;
        c.target_tps = t.targets.throughput_tps;
        c.epsilon = t.targets.epsilon;
        c.noise_amp = t.noise_amp;
        c.noise_key = t.noise_key;
        c.budget_off = static_cast<int64_t>(sig.size());
        c.n_budget = static_cast<int32_t>(t.budget_trace.size());
        for (const auto& [ts, v] : t.budget_trace) sig.push_back(pals_signal_point{ts, v});
        c.load_off = static_cast<int64_t>(sig.size());
        c.n_load = static_cast<int32_t>(t.load_trace.size());
        for (const auto& [ts, v] : t.load_trace) sig.push_back(pals_signal_point{ts, v});
    }
    std::vector<pals_ctrl_state> ini;
    if (init) {
        if (init->size() != n) throw config_error("replay: one initial state per trace");
        for (const auto& st : *init) ini.push_back(to_c(st));
    }
    std::vector<pals_plant_state> inp;
    if (init_plant) {
        if (init_plant->size() != n) throw config_error("replay: one plant state per trace");
        for (const auto& ps : *init_plant)
            inp.push_back(pals_plant_state{ps.applied_cap_w, ps.inflight_cap_w, ps.batch_cap, 0});
    }
    const int nl = static_cast<int>(std::min<std::size_t>(std::max(n_log_traces, 0), n));
    ReplayResult r;
    r.summaries.resize(n);
    std::vector<pals_ctrl_state> fin(n);
    std::vector<pals_plant_state> finp(n);
    std::vector<pals_step_log> logs(static_cast<std::size_t>(nl) * n_steps);
    std::vector<pals_step_detail> det(logs.size());
    pals_trace_batch b{};
    b.n_traces = static_cast<int64_t>(n);
    b.first_step = first_step;
    b.n_steps = n_steps;
    b.n_log_traces = nl;
    b.interval_s = interval_s;
    b.traces = tr.data();
    b.signal = sig.data();
    b.n_signal = static_cast<int64_t>(sig.size());
    b.init = init ? ini.data() : nullptr;
    b.init_plant = init_plant ? inp.data() : nullptr;
    b.summaries = r.summaries.data();
    b.final_state = fin.data();
    b.final_plant = finp.data();
    b.logs = nl ? logs.data() : nullptr;
    b.details = nl ? det.data() : nullptr;
    const pals_gpu_spec g{gpu.idle_watts, gpu.min_cap_watts, gpu.max_cap_watts, gpu.max_frequency};
    const pals_coeffs k{coeffs.alpha, coeffs.beta_watts};
    const pals_ctrl_cfg c = to_c(cfg);
    check(pals_replay_traces(ctx.get(), static_cast<int32_t>(hs.size()), hs.data(), profs.data(),
                             &g, &k, caps.data(), static_cast<int32_t>(caps.size()),
                             batches.data(), static_cast<int32_t>(batches.size()), &c, &b));
    r.states.reserve(n);
    r.plant.reserve(n);
    for (std::size_t i = 0; i < n; ++i) {
        r.states.push_back(from_c(fin[i]));
        r.plant.push_back(PlantState{finp[i].applied_cap_w, finp[i].inflight_cap_w, finp[i].batch_cap});
    }
    r.decisions.resize(nl);
    const int nb = static_cast<int>(batches.size());
    for (int i = 0; i < nl; ++i) {
        const ModelProfile& pm = plant[static_cast<std::size_t>(tr[i].model)];
        for (int s = 0; s < n_steps; ++s) {
            const pals_step_log& lg = logs[static_cast<std::size_t>(i) * n_steps + s];
            const pals_step_detail& dt = det[static_cast<std::size_t>(i) * n_steps + s];
            DecisionRecord d;
            d.t_s = static_cast<double>(first_step + s) * interval_s + interval_s;
            d.point = OperatingPoint{caps[static_cast<std::size_t>(lg.idx / nb)],
                                     batches[static_cast<std::size_t>(lg.idx % nb)],
                                     pm.deployment.tp, pm.deployment.ep, pm.deployment.dp};
            d.applied = lg.applied != 0;
            d.reason = static_cast<DecisionReason>(lg.reason);
            d.err_norm = dt.err_norm;
            d.bias = dt.bias;
            r.decisions[static_cast<std::size_t>(i)].push_back(d);
        }
    }
    return r;
}

// AllocRequest (allocator.hpp:13-19) with a device scorer.
struct GpuAllocRequest {
    std::string model_id;
    double throughput_target_tps = 0.0;
    std::vector<OperatingPoint> candidates;
    GpuScorer score;
    int dp = 1;
};

// allocate_budget (allocator.hpp:76-186): same results bit for bit, same exceptions.
inline AllocResult allocate_budget(const std::vector<GpuAllocRequest>& nodes,
                                   double cluster_budget_w, const GpuSpec& gpu,
                                   const SystemPowerCoeffs& coeffs, double quantum_w = 25.0,
                                   double selection_margin = 0.0) {
    if (nodes.empty()) throw config_error("allocate_budget: no nodes");
    // the floor check and its message are the reference's (allocator.hpp:81-95)
    std::vector<double> floor_w(nodes.size());
    double floor_total = 0.0;
    for (std::size_t i = 0; i < nodes.size(); ++i) {
        floor_w[i] = nodes[i].dp *
                     (coeffs.alpha * kGpusPerNode * gpu.min_cap_watts + coeffs.beta_watts);
        floor_total += floor_w[i];
    }
    if (floor_total > cluster_budget_w) {
        std::ostringstream msg;
        msg << "allocate_budget: cluster budget " << cluster_budget_w
            << " W below the sum of node floors (";
        for (std::size_t i = 0; i < nodes.size(); ++i)
            msg << (i ? ", " : "") << nodes[i].model_id << "=" << floor_w[i] << " W";
        msg << ")";
        throw config_error(msg.str());
    }
    // one candidate set per node
    std::vector<pals_model*> models;
    std::vector<pals_point> pts;
    std::vector<int64_t> off{0};
    for (const auto& n : nodes) {
        models.push_back(n.score.get());
        for (const auto& c : n.candidates) pts.push_back(to_c(c));
        off.push_back(static_cast<int64_t>(pts.size()));
    }
    if (pts.empty()) pts.push_back(pals_point{});
    const pals_gpu_spec g{gpu.idle_watts, gpu.min_cap_watts, gpu.max_cap_watts, gpu.max_frequency};
    const pals_coeffs k{coeffs.alpha, coeffs.beta_watts};
    pals_alloc* a = nullptr;
    check(pals_alloc_create_sets(nodes[0].score.context().get(),
                                 static_cast<int32_t>(nodes.size()), models.data(), pts.data(),
                                 off.data(), &g, &k, selection_margin, &a));
    std::unique_ptr<pals_alloc, int (*)(pals_alloc*)> guard(a, pals_alloc_destroy);
    const int64_t n = static_cast<int64_t>(nodes.size());
    std::vector<int64_t> noff{0, n};
    std::vector<int32_t> set(n), dp(n);
    std::vector<double> tgt(n);
    for (int64_t i = 0; i < n; ++i) {
        set[i] = static_cast<int32_t>(i);
        dp[i] = nodes[i].dp;
        tgt[i] = nodes[i].throughput_target_tps;
    }
    AllocResult res;
    res.node_budgets_w.assign(n, 0.0);
    uint8_t sat = 0;
    int32_t status = 0;
    check(pals_allocate_budget(a, quantum_w, 1, noff.data(), set.data(), dp.data(), tgt.data(),
                               &cluster_budget_w, res.node_budgets_w.data(),
                               &res.total_allocated_w, &sat, &status));
    if (status != PALS_OK) {
        // the first node whose scorer rejects its candidates: rethrow its error
        for (int32_t i = 0; i < n; ++i) {
            int32_t ns = 0;
            check(pals_alloc_steps(a, i, nullptr, nullptr, &ns));
        }
        check(status);
    }
    res.all_targets_satisfied = sat != 0;
    return res;
}

// build_frontier (pareto.hpp:31-59) on the device.
inline std::vector<FrontierPoint> build_frontier(Context& ctx,
                                                 const std::vector<FrontierPoint>& points) {
    if (points.empty()) throw config_error("build_frontier: no points");
    std::vector<pals_point> pts;
    std::vector<double> thr, eff;
    for (const auto& p : points) {
        pts.push_back(to_c(p.point));
        thr.push_back(p.throughput_tps);
        eff.push_back(p.efficiency_tpj);
    }
    std::vector<int32_t> idx(points.size());
    int64_t nf = 0;
    check(pals_frontier_values(ctx.get(), pts.data(), thr.data(), eff.data(),
                               static_cast<int64_t>(pts.size()), idx.data(), &nf));
    std::vector<FrontierPoint> out;
    for (int64_t i = 0; i < nf; ++i) out.push_back(points[static_cast<std::size_t>(idx[i])]);
    return out;
}

// evaluate_regime (pareto.hpp:114-135): analytic scores and the frontier on the device.
inline std::vector<FrontierPoint> evaluate_regime(
    Context& ctx, const RegimeSpec& regime, const ModelProfile& profile, const GpuSpec& gpu,
    const SystemPowerCoeffs& coeffs, const std::vector<double>& cap_grid,
    const std::vector<int>& batch_grid, const std::vector<int>& tp_grid) {
    const std::vector<double> caps =
        regime.sweep_cap ? cap_grid : std::vector<double>{regime.fixed_cap_w};
    const std::vector<int> batches =
        regime.sweep_batch ? batch_grid : std::vector<int>{regime.fixed_batch};
    const std::vector<int> tps = regime.sweep_tp ? tp_grid : std::vector<int>{profile.deployment.tp};
    std::vector<OperatingPoint> cands;
    for (double cap : caps)
        for (int batch : batches)
            for (int tp : tps) {
                if (!profile.comm_fixed_by_tp.count(tp)) continue;
                cands.push_back(OperatingPoint{cap, batch, tp, profile.deployment.ep, 1});
            }
    if (cands.empty()) throw config_error("build_frontier: no points");
    const GpuScorer sc = analytic_scorer(ctx, profile, gpu);
    const auto pts = to_c(cands);
    pals_grid* grid = nullptr;
    check(pals_grid_points(ctx.get(), pts.data(), static_cast<int64_t>(pts.size()), &grid));
    std::unique_ptr<pals_grid, int (*)(pals_grid*)> gguard(grid, pals_grid_destroy);
    const pals_coeffs k{coeffs.alpha, coeffs.beta_watts};
    pals_plan* plan = nullptr;
    check(pals_plan_create(ctx.get(), sc.get(), grid, &k, &plan));
    std::unique_ptr<pals_plan, int (*)(pals_plan*)> pguard(plan, pals_plan_destroy);
    std::vector<int32_t> idx(cands.size());
    int64_t nf = 0;
    check(pals_plan_frontier(plan, idx.data(), &nf));
    std::vector<double> th(cands.size()), pn(cands.size()), ef(cands.size());
    check(pals_plan_scores(plan, th.data(), pn.data(), ef.data()));
    std::vector<FrontierPoint> out;
    for (int64_t i = 0; i < nf; ++i) {
        const auto j = static_cast<std::size_t>(idx[i]);
        out.push_back(FrontierPoint{cands[j], th[j], ef[j]});
    }
    return out;
}

// ---- queue-plant simulation (sim.hpp:209-500) ------------------------------------
// run_scenario for many scenarios in one GPU pass; every SimResult is the
// reference's (scenario, per-node telemetry / decisions / requests, targets,
// arrival hashes, total energy).
inline std::vector<SimResult> run_scenarios(Context& ctx, const std::vector<Scenario>& scs,
                                            const ProfileRegistry& registry,
                                            const Platform& platform,
                                            const PredictorBundle* predictor) {
    const std::vector<std::string> names = registry.names();
    std::vector<pals_profile> profs;
    for (const auto& n : names) profs.push_back(to_c(registry.get(n)));
    auto index_of = [&](const std::string& id) {
        for (std::size_t i = 0; i < names.size(); ++i)
            if (names[i] == id) return static_cast<int32_t>(i);
        throw config_error("unknown model profile: " + id);
    };
    // predictor scorers for the models the scenarios use (predictor_scorer, sim.hpp:277-281)
    std::vector<GpuScorer> keep;
    std::vector<pals_model*> preds(names.size(), nullptr);
    std::vector<std::vector<pals_sim_node>> nodes(scs.size());
    std::vector<pals_scenario> cs(scs.size());
    std::vector<std::vector<double>> tt(scs.size()), tw(scs.size());
    int64_t stride = 0, n_nodes = 0;
    for (std::size_t s = 0; s < scs.size(); ++s) {
        const Scenario& sc = scs[s];
        sc.validate();
        for (const auto& n : sc.nodes) {
            const int32_t m = index_of(n.model_id);
            if (predictor && !preds[m]) {  // unknown ids throw as predict() would
                keep.push_back(predictor_scorer(ctx, *predictor, n.model_id));
                preds[m] = keep.back().get();
            }
            nodes[s].push_back(pals_sim_node{m, n.tp, n.ep, n.dp, n.qos_fraction,
                                             n.arrival_rate_per_s, n.initial_backlog, 0});
        }
        for (const auto& [t, w] : sc.budget_trace) {
            tt[s].push_back(t);
            tw[s].push_back(w);
        }
        pals_scenario& c = cs[s];
        std::memset(&c, 0, sizeof c);
        c.duration_s = sc.duration_s;
        c.interval_s = sc.interval_s;
        c.seed = sc.seed;
        c.mean_tokens = sc.output_len.mean_tokens;
        c.log_sigma = sc.output_len.log_sigma;
        c.has_cluster_budget = sc.cluster_budget_w.has_value() ? 1 : 0;
        c.cluster_budget_w = sc.cluster_budget_w.value_or(0.0);
        c.n_trace = static_cast<int32_t>(tt[s].size());
        c.trace_t = tt[s].data();
        c.trace_w = tw[s].data();
        c.policy = static_cast<int32_t>(sc.policy);  // Fixed .. Oracle = 0 .. 4
        c.objective = sc.objective == Objective::BudgetMaxThroughput ? PALS_OBJ_BUDGET
                                                                     : PALS_OBJ_QOS;
        c.controller = to_c(sc.controller);
        c.epsilon = sc.epsilon;
        c.cand_caps = sc.cand_caps.data();
        c.cand_batches = sc.cand_batches.data();
        c.n_caps = static_cast<int32_t>(sc.cand_caps.size());
        c.n_batches = static_cast<int32_t>(sc.cand_batches.size());
        c.initial_cap_w = sc.initial_cap_w;
        c.initial_batch = sc.initial_batch;
        c.n_nodes = static_cast<int32_t>(nodes[s].size());
        c.nodes = nodes[s].data();
        stride = std::max<int64_t>(stride, std::llround(sc.duration_s / sc.interval_s));
        n_nodes += c.n_nodes;
    }
    const pals_gpu_spec g{platform.gpu.idle_watts, platform.gpu.min_cap_watts,
                          platform.gpu.max_cap_watts, platform.gpu.max_frequency};
    const pals_coeffs k{platform.coeffs.alpha, platform.coeffs.beta_watts};
    std::vector<pals_sim_node_result> nres(n_nodes);
    std::vector<pals_sim_result> res(scs.size());
    std::vector<pals_sim_telemetry> tel(n_nodes * stride);
    std::vector<pals_sim_decision> dec(n_nodes * stride);
    check(pals_sim_keep_requests(ctx.get(), 1));
    const int rc = pals_run_scenarios(ctx.get(), static_cast<int32_t>(cs.size()), cs.data(),
                                      static_cast<int32_t>(profs.size()), profs.data(),
                                      preds.data(), &g, &k, nres.data(), res.data(), stride,
                                      tel.data(), dec.data());
    pals_sim_keep_requests(ctx.get(), 0);
    check(rc);
    const DecisionReason reasons[] = {DecisionReason::QosFeasibleMaxEfficiency,
                                      DecisionReason::FallbackMaxThroughput,
                                      DecisionReason::BudgetConstrainedMaxThroughput,
                                      DecisionReason::HoldHysteresis,
                                      DecisionReason::OracleExhaustive};
    std::vector<SimResult> out(scs.size());
    int64_t gi = 0;
    for (std::size_t s = 0; s < scs.size(); ++s) {
        SimResult& r = out[s];
        r.scenario = scs[s];
        r.total_energy_j = res[s].sim_total_energy_j;
        const int n_int = res[s].n_intervals;
        for (std::size_t i = 0; i < scs[s].nodes.size(); ++i, ++gi) {
            const ScenarioNode& sn = scs[s].nodes[i];
            NodeResult nr;
            nr.model_id = sn.model_id;
            nr.throughput_target_tps = nres[gi].throughput_target_tps;
            nr.arrival_stream_hash = nres[gi].arrival_stream_hash;
            for (int kk = 0; kk < n_int; ++kk) {
                const pals_sim_telemetry& t = tel[gi * stride + kk];
                TelemetrySample ts;
                ts.t_s = t.t_s;
                ts.gpu_power_w = t.gpu_power_w;
                ts.sys_power_w = t.sys_power_w;
                ts.throughput_tps = t.throughput_tps;
                ts.utilization = t.utilization;
                ts.queue_depth = t.queue_depth;
                ts.active_batch = t.active_batch;
                ts.node_budget_w = t.node_budget_w;
                ts.applied_cap_w = t.applied_cap_w;
                ts.applied_batch_cap = t.applied_batch_cap;
                nr.telemetry.push_back(ts);
                const pals_sim_decision& d = dec[gi * stride + kk];
                DecisionRecord dr;
                dr.t_s = t.t_s;
                dr.point = OperatingPoint{d.cap_w, d.batch, sn.tp, sn.ep, sn.dp};
                dr.applied = d.applied != 0;
                dr.reason = reasons[d.reason];
                dr.err_norm = d.err_norm;
                dr.bias = d.bias;
                nr.decisions.push_back(dr);
            }
            int64_t nq = 0;
            check(pals_sim_requests(ctx.get(), gi, nullptr, 0, &nq));
            std::vector<pals_sim_request> rq(static_cast<std::size_t>(nq));
            check(pals_sim_requests(ctx.get(), gi, rq.data(), nq, &nq));
            for (const auto& q : rq) {
                RequestRec rr;
                rr.id = static_cast<long>(q.id);
                rr.arrival_s = q.arrival_s;
                rr.output_tokens = q.output_tokens;
                rr.generated = q.generated;
                rr.completed_s = q.completed_s;
                nr.requests.push_back(rr);
            }
            r.nodes.push_back(std::move(nr));
        }
    }
    return out;
}

inline SimResult run_scenario(Context& ctx, const Scenario& sc, const ProfileRegistry& registry,
                              const Platform& platform, const PredictorBundle* predictor) {
    return run_scenarios(ctx, {sc}, registry, platform, predictor).front();
}

// All five control strategies on identical seeds and arrival streams (sim.hpp:488-500).
inline std::map<Policy, SimResult> run_baseline_suite(Context& ctx, const Scenario& sc,
                                                      const ProfileRegistry& registry,
                                                      const Platform& platform,
                                                      const PredictorBundle* predictor) {
    std::vector<Scenario> scs;
    const Policy pols[] = {Policy::Fixed, Policy::AdaptiveBatch, Policy::AdaptiveCap,
                           Policy::Joint, Policy::Oracle};
    for (Policy p : pols) {
        scs.push_back(sc);
        scs.back().policy = p;
    }
    auto rs = run_scenarios(ctx, scs, registry, platform, predictor);
    std::map<Policy, SimResult> out;
    for (std::size_t i = 0; i < rs.size(); ++i) out.emplace(pols[i], std::move(rs[i]));
    return out;
}

}  // namespace wattserve::gpu
