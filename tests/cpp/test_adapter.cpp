// test_adapter.cpp — the reference's own controller tests, run twice in one
// binary: once through the unmodified reference (wattserve::select_config /
// control_step on the CPU) and once through the drop-in GPU adapter
// (wattserve::gpu::*, include/wattserve_gpu.hpp -> libpals_gpu.so). Every
// decision and every controller state must be identical.
//
// Case families follow /root/reference/proj/tests/test_controller.cpp and
// tests/acceptance/acceptance.cpp criterion 10 (restated, not copied).
// Exit code = number of failed checks. Built by tests/cpp/build.sh.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "wattserve/allocator.hpp"
#include "wattserve/controller.hpp"
#include "wattserve/forest.hpp"
#include "wattserve/pareto.hpp"
#include "wattserve/json_io.hpp"
#include "wattserve/metrics.hpp"
#include "wattserve/rng.hpp"
#include "wattserve/scenario_io.hpp"
#include "wattserve/sim.hpp"
#include "wattserve/sweep.hpp"
#include "wattserve_gpu.hpp"

using namespace wattserve;

static int g_fail = 0, g_checks = 0;
#define EXPECT(cond, what)                                                      \
    do {                                                                        \
        ++g_checks;                                                             \
        if (!(cond)) {                                                          \
            ++g_fail;                                                           \
            if (g_fail < 20) std::fprintf(stderr, "FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
        }                                                                       \
    } while (0)

static bool same(const Decision& a, const Decision& b) {
    return a.point == b.point && a.applied == b.applied && a.reason == b.reason;
}

static bool same_bits(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

static bool same(const ControllerState& a, const ControllerState& b) {
    return same_bits(a.bias, b.bias) && same_bits(a.integral, b.integral) &&
           same_bits(a.prev_error, b.prev_error) && a.has_prev_error == b.has_prev_error &&
           a.sustain_count == b.sustain_count && a.current == b.current &&
           a.last_targets.has_value() == b.last_targets.has_value() &&
           (!a.last_targets || *a.last_targets == *b.last_targets);
}

struct Table {
    std::vector<OperatingPoint> points;
    std::vector<double> t_hat, p_gpu;
    Scorer cpu() const {
        return [this](const OperatingPoint& p) {
            for (std::size_t i = 0; i < points.size(); ++i)
                if (points[i] == p) return CandidateScore{t_hat[i], p_gpu[i]};
            throw config_error("unscored candidate");
        };
    }
};

static Table ladder(int n, double lo, double hi) {
    Table t;
    for (int i = 0; i < n; ++i) {
        const double frac = n == 1 ? 0.0 : static_cast<double>(i) / (n - 1);
        const double thr = lo + (hi - lo) * frac;
        t.points.push_back(OperatingPoint{150.0 + i, 1 + i, 2, 1, 1});
        t.t_hat.push_back(thr);
        t.p_gpu.push_back(40.0 + thr * thr / 800.0);
    }
    return t;
}

static Targets qos(double tps) {
    Targets t;
    t.throughput_tps = tps;
    t.epsilon = 0.05;
    return t;
}

static std::string read_file(const std::string& p) {
    std::ifstream f(p);
    std::stringstream ss;
    ss << f.rdbuf();
    return ss.str();
}

// Single-call latency of the drop-in (BASELINE cfg1): the bundled llama2-7b-like profile, its
// 6 caps x 6 batches at the deployment TP, target 0.6 x unconstrained, a static 1600 W
// budget; wall-clock microseconds per call for wattserve::gpu::* and the reference, printed
// as one JSON line.
static int latency(const std::string& root) {
    gpu::Context ctx(0);
    const json j = json::parse(read_file(root + "/paper_2605_21427_b200/data/profiles.json"));
    ModelProfile prof;
    for (const auto& pj : j.at("profiles"))
        if (pj.at("name").get<std::string>() == "llama2-7b-like") prof = profile_from_json(pj);
    const GpuSpec gspec = gpu_from_json(j.at("platform").at("gpu"));
    const SystemPowerCoeffs k{1.05, 345.0};
    std::vector<OperatingPoint> cands;
    for (double c : {150.0, 200.0, 250.0, 300.0, 350.0, 400.0})
        for (int b : {1, 4, 8, 16, 32, 64})
            cands.push_back(OperatingPoint{c, b, prof.deployment.tp, prof.deployment.ep,
                                           prof.deployment.dp});
    const Scorer cs = detail::cached(analytic_scorer(prof, gspec));
    auto gs = gpu::analytic_scorer(ctx, prof, gspec);
    Targets t = qos(0.6 * throughput(cands.back(), prof, gspec));
    t.power_budget_w = 1600.0;
    ControllerConfig cfg;
    cfg.target_headroom = 0.05;
    cfg.budget_margin = 0.02;
    auto bench = [](auto&& f, int reps) {
        for (int i = 0; i < 50; ++i) f(i);
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < reps; ++i) f(i);
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
                   .count() / reps;
    };
    int sink = 0;
    const double g_sel = bench([&](int) { sink += gpu::select_config(cands, t, gs, k, 1.0, 0.05, 0.02).point.batch; }, 2000);
    const double r_sel = bench([&](int) { sink += select_config(cands, t, cs, k, 1.0, 0.05, 0.02).point.batch; }, 20000);
    ControllerState sg, sr;
    sg.current = sr.current = cands.back();
    bool same = true;
    const double g_step = bench([&](int i) {
        auto [d, s2] = gpu::control_step(TelemetryInput{0.5 * i, 0.55 * t.throughput_tps}, 0.5 * i,
                                         t, cands, gs, k, sg, cfg);
        sg = s2;
        sink += d.point.batch;
    }, 2000);
    const double r_step = bench([&](int i) {
        auto [d, s2] = control_step(TelemetryInput{0.5 * i, 0.55 * t.throughput_tps}, 0.5 * i, t,
                                    cands, cs, k, sr, cfg);
        sr = s2;
        sink += d.point.batch;
    }, 20000);
    // the same calls with one kernel launch per call instead of the resident server
    ctx.set_one_server(0);
    const double l_sel = bench([&](int) { sink += gpu::select_config(cands, t, gs, k, 1.0, 0.05, 0.02).point.batch; }, 2000);
    ControllerState sl;
    sl.current = cands.back();
    const double l_step = bench([&](int i) {
        auto [d, s2] = gpu::control_step(TelemetryInput{0.5 * i, 0.55 * t.throughput_tps}, 0.5 * i,
                                         t, cands, gs, k, sl, cfg);
        sl = s2;
        sink += d.point.batch;
    }, 2000);
    same = same && ::same(sl, sg);
    ctx.set_one_server(2000);
    // same call sequence on both sides from the same start: the states must agree
    ControllerState a, b;
    a.current = b.current = cands.back();
    for (int i = 0; i < 300; ++i) {
        const TelemetryInput ti{0.5 * i, (0.4 + 0.002 * i) * t.throughput_tps};
        auto [da, sa] = gpu::control_step(ti, 0.5 * i, t, cands, gs, k, a, cfg);
        auto [db, sb] = control_step(ti, 0.5 * i, t, cands, cs, k, b, cfg);
        same = same && ::same(da, db) && ::same(sa, sb);
        a = sa;
        b = sb;
    }
    std::printf("{\"select_config_us\": %.3f, \"control_step_us\": %.3f, "
                "\"launch_per_call_select_config_us\": %.3f, "
                "\"launch_per_call_control_step_us\": %.3f, "
                "\"reference_select_config_us\": %.3f, \"reference_control_step_us\": %.3f, "
                "\"candidates\": %zu, \"identical\": %s, \"sink\": %d}\n",
                g_sel, g_step, l_sel, l_step, r_sel, r_step, cands.size(), same ? "true" : "false",
                sink & 1);
    return same ? 0 : 1;
}

int main(int argc, char** argv) {
    const std::string root = argc > 1 ? argv[1] : ".";
    if (argc > 2 && std::string(argv[2]) == "--latency") return latency(root);
    gpu::Context ctx(0);
    const SystemPowerCoeffs k{1.05, 345.0};

    // ---- select_config on ladders (test_controller.cpp:54-92) ----
    {
        const Table a = ladder(8, 1000.0, 2000.0), b = ladder(8, 100.0, 300.0);
        auto ga = gpu::table_scorer(ctx, a.points, a.t_hat, a.p_gpu);
        auto gb = gpu::table_scorer(ctx, b.points, b.t_hat, b.p_gpu);
        EXPECT(same(select_config(a.points, qos(500.0), a.cpu(), k),
                    gpu::select_config(a.points, qos(500.0), ga, k)), "all feasible");
        EXPECT(same(select_config(b.points, qos(1000.0), b.cpu(), k),
                    gpu::select_config(b.points, qos(1000.0), gb, k)), "fallback");
        Targets t = qos(1000.0);
        t.power_budget_w = (k.alpha * kGpusPerNode * b.p_gpu[3] + k.beta_watts) + 1.0;
        EXPECT(same(select_config(b.points, t, b.cpu(), k), gpu::select_config(b.points, t, gb, k)),
               "budget fallback");
        bool threw = false;
        try {
            gpu::select_config({}, qos(100.0), ga, k);
        } catch (const config_error& e) {
            threw = std::string(e.what()) == "select_config: empty candidate list";
        }
        EXPECT(threw, "empty candidate list throws config_error");
    }

    // ---- 1,000-trial argmax invariance, both sides (test_controller.cpp:100-138) ----
    {
        Rng rng(2024);
        for (int trial = 0; trial < 1000; ++trial) {
            Table tab;
            const int n = 3 + static_cast<int>(rng.next_u64() % 20);
            for (int i = 0; i < n; ++i) {
                tab.points.push_back(OperatingPoint{150.0 + 50.0 * (i % 6), 1 + (i * 7) % 64, 2, 1, 1});
                tab.t_hat.push_back(rng.uniform(100.0, 3000.0));
                tab.p_gpu.push_back(rng.uniform(60.0, 400.0));
            }
            Targets t = qos(rng.uniform(100.0, 2500.0));
            if (trial % 3 == 0) t.power_budget_w = rng.uniform(500.0, 2000.0);
            const double s = rng.uniform(0.01, 100.0);
            Table sc = tab;
            for (auto& v : sc.t_hat) v *= s;
            for (auto& v : sc.p_gpu) v *= s;
            Targets ts = t;
            ts.throughput_tps *= s;
            if (ts.power_budget_w) ts.power_budget_w = *t.power_budget_w * s;
            const SystemPowerCoeffs ks{k.alpha, k.beta_watts * s};
            auto g1 = gpu::table_scorer(ctx, tab.points, tab.t_hat, tab.p_gpu);
            auto g2 = gpu::table_scorer(ctx, sc.points, sc.t_hat, sc.p_gpu);
            const auto r1 = select_config(tab.points, t, tab.cpu(), k);
            const auto d1 = gpu::select_config(tab.points, t, g1, k);
            const auto d2 = gpu::select_config(sc.points, ts, g2, ks);
            EXPECT(same(r1, d1), "invariance trial: gpu == reference");
            EXPECT(d1.point == d2.point && d1.reason == d2.reason, "invariance under rescaling");
        }
    }

    // ---- control_step sequences (test_controller.cpp:140-235; acceptance criterion 10) ----
    {
        for (int trial = 0; trial < 60; ++trial) {
            Rng rng(1000 + trial);
            const double lambda = trial % 2 == 0 ? 0.7 : 1.3;
            Table l;
            for (int i = 0; i < 160; ++i) {
                const double frac = static_cast<double>(i) / 159;
                const double thr = 300.0 + 2100.0 * frac * rng.uniform(0.995, 1.005);
                l.points.push_back(OperatingPoint{100.0 + i, 1 + i, 2, 1, 1});
                l.t_hat.push_back(thr);
                l.p_gpu.push_back(40.0 + thr * thr / 800.0);
            }
            auto g = gpu::table_scorer(ctx, l.points, l.t_hat, l.p_gpu);
            Targets t = qos(rng.uniform(700.0, 1500.0));
            if (trial % 4 == 3) t.power_budget_w = rng.uniform(900.0, 2200.0);
            if (trial % 5 == 4) t.objective = Objective::BudgetMaxThroughput;
            ControllerConfig cfg;
            cfg.target_headroom = trial % 3 == 0 ? 0.05 : 0.0;
            cfg.budget_margin = trial % 2 ? 0.02 : 0.0;
            ControllerState sc, sg;
            sc.current = sg.current = l.points.back();
            double now = 0.5, measured = lambda * l.t_hat.back();
            for (int step = 0; step < 40; ++step) {
                const TelemetryInput tel{step % 13 == 12 ? now - 5.0 : now, measured};
                auto [dc, sc2] = control_step(tel, now, t, l.points, l.cpu(), k, sc, cfg);
                auto [dg, sg2] = gpu::control_step(tel, now, t, l.points, g, k, sg, cfg);
                EXPECT(same(dc, dg), "control_step decision");
                EXPECT(same(sc2, sg2), "control_step state");
                sc = sc2;
                sg = sg2;
                for (std::size_t i = 0; i < l.points.size(); ++i)
                    if (l.points[i] == sc.current) measured = lambda * l.t_hat[i];
                now += cfg.interval_s;
            }
        }
    }

    // ---- analytic_scorer on the bundled profiles (model-fit input) ----
    std::vector<ModelProfile> profiles;
    GpuSpec gspec;
    {
        const json j = json::parse(read_file(root + "/paper_2605_21427_b200/data/profiles.json"));
        for (const auto& pj : j.at("profiles")) profiles.push_back(profile_from_json(pj));
        gspec = gpu_from_json(j.at("platform").at("gpu"));
        const SweepGrid grid = SweepGrid::default_grid();
        for (const auto& prof : profiles) {
            std::vector<OperatingPoint> cands;
            for (double c : grid.caps)
                for (int b : grid.batches)
                    cands.push_back(OperatingPoint{c, b, prof.deployment.tp, prof.deployment.ep,
                                                   prof.deployment.dp});
            const Scorer cs = analytic_scorer(prof, gspec);
            auto gs = gpu::analytic_scorer(ctx, prof, gspec);
            const double tmax = cands.size() ? throughput(cands.back(), prof, gspec) : 1.0;
            Rng rng(7);
            std::vector<Targets> ts;
            std::vector<double> biases;
            for (int q = 0; q < 200; ++q) {
                Targets t = qos(rng.uniform(0.05, 1.1) * tmax);
                if (q % 2) t.power_budget_w = rng.uniform(700.0, 2000.0);
                if (q % 5 == 0) t.objective = Objective::BudgetMaxThroughput;
                const double bias = q % 3 ? 1.0 : rng.uniform(0.5, 2.0);
                ts.push_back(t);
                biases.push_back(bias);
                EXPECT(same(select_config(cands, t, cs, k, bias, 0.05, 0.02),
                            gpu::select_config(cands, t, gs, k, bias, 0.05, 0.02)),
                       "analytic select");
            }
            gpu::SelectPlan plan(ctx, gs, cands, k);
            const auto batch = plan.select(ts, biases, 0.05, 0.02);
            for (std::size_t q = 0; q < ts.size(); ++q)
                EXPECT(same(batch[q], select_config(cands, ts[q], cs, k, biases[q], 0.05, 0.02)),
                       "batched SelectPlan");
        }
        // errors: cap outside the platform range, unknown tp
        auto gs = gpu::analytic_scorer(ctx, profiles[0], gspec);
        bool range = false, tp = false;
        try {
            gpu::select_config({OperatingPoint{450.0, 8, profiles[0].deployment.tp, 1, 1}}, qos(1.0),
                               gs, k);
        } catch (const std::out_of_range&) {
            range = true;
        }
        try {
            gpu::select_config({OperatingPoint{300.0, 8, 3, 1, 1}}, qos(1.0), gs, k);
        } catch (const config_error& e) {
            tp = std::string(e.what()).find("no comm cost calibrated for tp=3") != std::string::npos;
        }
        EXPECT(range, "cap out of range -> std::out_of_range");
        EXPECT(tp, "unknown tp -> config_error");
    }

    // ---- predictor_scorer on a bundle trained by the reference pipeline ----
    PredictorBundle bundle;
    {
        const SweepGrid grid = SweepGrid::default_grid();
        AnalyticBackend be(gspec, k);
        std::vector<ProfilingRecord> recs;
        for (std::size_t i = 0; i < profiles.size(); ++i) {
            const auto ds = run_sweep(grid, profiles[i].name, profiles[i], gspec, be, 100 + i);
            recs.insert(recs.end(), ds.records.begin(), ds.records.end());
        }
        HyperParams hp;
        hp.n_trees = 30;
        hp.max_depth = 12;
        bundle = train_bundle(recs, k, hp, 2605);
        for (const char* mid : {"llama2-7b-like", "mixtral-8x7b-like"}) {
            const Scorer cs = predictor_scorer(bundle, mid);
            auto gs = gpu::predictor_scorer(ctx, bundle, mid);
            const ModelProfile* prof = nullptr;
            for (const auto& p : profiles)
                if (p.name == mid) prof = &p;
            std::vector<OperatingPoint> cands;
            for (double c : {150.0, 175.0, 200.0, 250.0, 300.0, 350.0, 400.0})
                for (int b : {1, 4, 8, 12, 16, 32, 48, 64})
                    cands.push_back(OperatingPoint{c, b, prof->deployment.tp, prof->deployment.ep,
                                                   prof->deployment.dp});
            Rng rng(11);
            const double tmax = bundle.predict(cands.back(), mid).throughput_hat;
            ControllerState sc, sg;
            sc.current = sg.current = cands.back();
            ControllerConfig cfg;
            for (int q = 0; q < 150; ++q) {
                Targets t = qos(rng.uniform(0.05, 1.1) * tmax);
                if (q % 2) t.power_budget_w = rng.uniform(800.0, 2000.0);
                EXPECT(same(select_config(cands, t, cs, k, 1.0, 0.05, 0.02),
                            gpu::select_config(cands, t, gs, k, 1.0, 0.05, 0.02)),
                       "predictor select");
                const TelemetryInput tel{0.5 * q, rng.uniform(0.3, 1.2) * tmax};
                auto [dc, sc2] = control_step(tel, 0.5 * q, t, cands, cs, k, sc, cfg);
                auto [dg, sg2] = gpu::control_step(tel, 0.5 * q, t, cands, gs, k, sg, cfg);
                EXPECT(same(dc, dg) && same(sc2, sg2), "predictor control_step");
                sc = sc2;
                sg = sg2;
            }
        }
    }

    // ---- allocate_budget (allocator.hpp; tests/test_controller.cpp:237-283) ----
    {
        auto same_alloc = [](const AllocResult& a, const AllocResult& b) {
            if (a.node_budgets_w.size() != b.node_budgets_w.size()) return false;
            for (std::size_t i = 0; i < a.node_budgets_w.size(); ++i)
                if (!same_bits(a.node_budgets_w[i], b.node_budgets_w[i])) return false;
            return same_bits(a.total_allocated_w, b.total_allocated_w) &&
                   a.all_targets_satisfied == b.all_targets_satisfied;
        };
        GpuSpec g0;
        const Table t8 = ladder(8, 400.0, 1200.0), t120 = ladder(120, 400.0, 2000.0),
                    t4 = ladder(4, 400.0, 1000.0);
        auto mk = [&](const Table& t, const std::string& id, double target) {
            AllocRequest r;
            r.model_id = id;
            r.throughput_target_tps = target;
            r.candidates = t.points;
            r.score = t.cpu();
            return r;
        };
        auto mkg = [&](const Table& t, const std::string& id, double target) {
            return gpu::GpuAllocRequest{id, target, t.points,
                                        gpu::table_scorer(ctx, t.points, t.t_hat, t.p_gpu), 1};
        };
        const double max_useful = k.alpha * kGpusPerNode * t8.p_gpu.back() + k.beta_watts;
        EXPECT(same_alloc(allocate_budget({mk(t8, "m", 3000.0)}, max_useful + 500.0, g0, k, 25.0),
                          gpu::allocate_budget({mkg(t8, "m", 3000.0)}, max_useful + 500.0, g0, k,
                                               25.0)),
               "one node takes the budget");
        EXPECT(same_alloc(allocate_budget({mk(t120, "a", 1800.0), mk(t120, "b", 1800.0)}, 3000.0,
                                          g0, k, 25.0),
                          gpu::allocate_budget({mkg(t120, "a", 1800.0), mkg(t120, "b", 1800.0)},
                                               3000.0, g0, k, 25.0)),
               "identical nodes split evenly");
        std::string want, got;
        try {
            allocate_budget({mk(t4, "starved", 0.0), mk(t4, "starved", 0.0),
                             mk(t4, "starved", 0.0)}, 100.0, g0, k);
        } catch (const config_error& e) {
            want = e.what();
        }
        try {
            gpu::allocate_budget({mkg(t4, "starved", 0.0), mkg(t4, "starved", 0.0),
                                  mkg(t4, "starved", 0.0)}, 100.0, g0, k);
        } catch (const config_error& e) {
            got = e.what();
        }
        EXPECT(!want.empty() && want == got, "infeasible floor: same config_error message");
        // random clusters over the analytic profiles (the sim's assign_budgets shape)
        Rng rng(31);
        const std::vector<double> caps{150, 200, 250, 300, 350, 400};
        const std::vector<int> bats{1, 4, 8, 16, 32, 64};
        for (int trial = 0; trial < 200; ++trial) {
            const int nn = 1 + static_cast<int>(rng.next_u64() % 6);
            std::vector<AllocRequest> rq;
            std::vector<gpu::GpuAllocRequest> gq;
            double peak = 0.0;
            for (int i = 0; i < nn; ++i) {
                const ModelProfile& prof = profiles[rng.next_u64() % profiles.size()];
                const int dp = 1 + static_cast<int>(rng.next_u64() % 3);
                std::vector<OperatingPoint> cands;
                for (double c : caps)
                    for (int b : bats)
                        cands.push_back(OperatingPoint{c, b, prof.deployment.tp,
                                                       prof.deployment.ep, dp});
                const double tmax = cluster_throughput(cands.back(), prof, gspec);
                peak += cluster_system_power(cands.back(), prof, gspec, k);
                const double target = rng.uniform(0.2, 1.0) * tmax;
                AllocRequest r;
                r.model_id = prof.name;
                r.throughput_target_tps = target;
                r.candidates = cands;
                r.score = analytic_scorer(prof, gspec);
                r.dp = dp;
                rq.push_back(r);
                gq.push_back(gpu::GpuAllocRequest{prof.name, target, cands,
                                                  gpu::analytic_scorer(ctx, prof, gspec), dp});
            }
            const double budget = rng.uniform(0.5, 1.2) * peak;
            const double margin = trial % 2 ? 0.02 : 0.0;
            std::string ew, eg;
            AllocResult ra, ga;
            try {
                ra = allocate_budget(rq, budget, gspec, k, 25.0, margin);
            } catch (const std::exception& e) {
                ew = e.what();
            }
            try {
                ga = gpu::allocate_budget(gq, budget, gspec, k, 25.0, margin);
            } catch (const std::exception& e) {
                eg = e.what();
            }
            EXPECT(ew == eg && (!ew.empty() || same_alloc(ra, ga)), "random cluster allocation");
        }
    }

    // ---- Pareto frontier (pareto.hpp; tests/test_analysis.cpp:26-118) ----
    {
        auto same_front = [](const std::vector<FrontierPoint>& a,
                             const std::vector<FrontierPoint>& b) {
            if (a.size() != b.size()) return false;
            for (std::size_t i = 0; i < a.size(); ++i)
                if (!(a[i].point == b[i].point) || !same_bits(a[i].throughput_tps, b[i].throughput_tps) ||
                    !same_bits(a[i].efficiency_tpj, b[i].efficiency_tpj))
                    return false;
            return true;
        };
        const std::vector<double> caps{150, 200, 250, 300, 350, 400};
        const std::vector<int> bats{1, 4, 8, 16, 32, 64};
        const std::vector<int> tps{1, 2, 4};
        for (const auto& prof : profiles)
            for (const auto& reg : default_regimes())
                EXPECT(same_front(evaluate_regime(reg, prof, gspec, k, caps, bats, tps),
                                  gpu::evaluate_regime(ctx, reg, prof, gspec, k, caps, bats, tps)),
                       "evaluate_regime");
        Rng rng(99);
        for (int trial = 0; trial < 200; ++trial) {
            std::vector<FrontierPoint> pts;
            const int n = 2 + static_cast<int>(rng.next_u64() % 40);
            for (int i = 0; i < n; ++i)
                pts.push_back(FrontierPoint{OperatingPoint{150.0 + 50.0 * (i % 6), 8, 2, 1, 1},
                                            rng.uniform(10.0, 1000.0), rng.uniform(0.1, 2.0)});
            EXPECT(same_front(build_frontier(pts), gpu::build_frontier(ctx, pts)),
                   "build_frontier random");
        }
        bool threw = false;
        try {
            gpu::build_frontier(ctx, {});
        } catch (const config_error&) {
            threw = true;
        }
        EXPECT(threw, "build_frontier: no points");
    }

    // ---- run_scenario / run_baseline_suite (sim.hpp:482-500) on the bundled scenarios ----
    {
        ProfileRegistry reg;
        for (const auto& p : profiles) reg.add(p);
        const Platform plat{gspec, k};
        const json all = json::parse(read_file(root + "/paper_2605_21427_b200/data/scenarios.json"));
        int n_sc = 0;
        for (const auto& [name, entry] : all.items()) {
            json sj = entry.at("scenario");
            sj.erase("budget_trace_csv");  // resolved into "trace" (the CSV is not shipped)
            Scenario sc = scenario_from_json(sj);
            for (const auto& tw : entry.at("trace"))
                sc.budget_trace.emplace_back(tw.at(0).get<double>(), tw.at(1).get<double>());
            sc.duration_s = std::min(sc.duration_s, 600.0);
            const auto want = run_baseline_suite(sc, reg, plat, &bundle);
            const auto got = gpu::run_baseline_suite(ctx, sc, reg, plat, &bundle);
            for (const auto& [pol, rw] : want) {
                const SimResult& rg = got.at(pol);
                bool ok = rw.nodes.size() == rg.nodes.size() &&
                          same_bits(rw.total_energy_j, rg.total_energy_j);
                for (std::size_t i = 0; ok && i < rw.nodes.size(); ++i) {
                    const NodeResult& a = rw.nodes[i];
                    const NodeResult& b = rg.nodes[i];
                    ok = a.model_id == b.model_id && a.arrival_stream_hash == b.arrival_stream_hash &&
                         same_bits(a.throughput_target_tps, b.throughput_target_tps) &&
                         a.telemetry.size() == b.telemetry.size() &&
                         a.decisions.size() == b.decisions.size();
                    for (std::size_t t = 0; ok && t < a.telemetry.size(); ++t) {
                        const auto &x = a.telemetry[t], &y = b.telemetry[t];
                        const auto &p = a.decisions[t], &q = b.decisions[t];
                        ok = same_bits(x.t_s, y.t_s) && same_bits(x.gpu_power_w, y.gpu_power_w) &&
                             same_bits(x.sys_power_w, y.sys_power_w) &&
                             same_bits(x.throughput_tps, y.throughput_tps) &&
                             same_bits(x.utilization, y.utilization) &&
                             x.queue_depth == y.queue_depth && x.active_batch == y.active_batch &&
                             same_bits(x.node_budget_w, y.node_budget_w) &&
                             same_bits(x.applied_cap_w, y.applied_cap_w) &&
                             x.applied_batch_cap == y.applied_batch_cap &&
                             same_bits(p.t_s, q.t_s) && p.point == q.point &&
                             p.applied == q.applied && p.reason == q.reason &&
                             same_bits(p.err_norm, q.err_norm) && same_bits(p.bias, q.bias);
                    }
                }
                const RunSummary sw = summarize(rw), sg = summarize(rg);
                ok = ok && same_bits(sw.aggregate.tokens_per_joule, sg.aggregate.tokens_per_joule) &&
                     same_bits(sw.cluster_tracking_mae_w, sg.cluster_tracking_mae_w) &&
                     decisions_csv(rw) == decisions_csv(rg) && telemetry_csv(rw) == telemetry_csv(rg) &&
                     requests_csv(rw) == requests_csv(rg);
                EXPECT(ok, (name + "/" + to_string(pol)).c_str());
                ++n_sc;
            }
        }
        EXPECT(n_sc == 15, "3 scenarios x 5 policies");
    }

    // ---- gpu::replay over caller traces: the demand-response budget trace through the
    // fluid plant, against the unmodified control_step / trace_value / enforce_cap driven
    // by the same loop here; then a mid-trace resume from the returned states ----
    {
        const json all = json::parse(read_file(root + "/paper_2605_21427_b200/data/scenarios.json"));
        std::vector<std::pair<double, double>> cluster;
        for (const auto& tw : all.at("demand_response").at("trace"))
            cluster.emplace_back(tw.at(0).get<double>(), tw.at(1).get<double>());
        const std::vector<double> caps{150.0, 200.0, 250.0, 300.0, 350.0, 400.0};
        const std::vector<int> batches{1, 4, 8, 16, 32, 64};
        ControllerConfig cfg;
        cfg.target_headroom = 0.05;
        cfg.budget_margin = 0.02;
        std::vector<gpu::GpuScorer> scorers;
        for (const auto& p : profiles) scorers.push_back(gpu::analytic_scorer(ctx, p, gspec));
        std::vector<gpu::ReplayTrace> traces;
        Rng rng(31);
        for (std::size_t m = 0; m < profiles.size(); ++m) {
            for (int o = 0; o < 2; ++o) {
                gpu::ReplayTrace t;
                t.model = static_cast<int>(m);
                const ModelProfile& pm = profiles[m];
                const OperatingPoint top{400.0, 64, pm.deployment.tp, pm.deployment.ep,
                                         pm.deployment.dp};
                const double tmax = cluster_throughput(top, pm, gspec);
                t.targets.throughput_tps = rng.uniform(0.3, 0.9) * tmax;
                t.targets.objective = o ? Objective::BudgetMaxThroughput : Objective::QosMaxEfficiency;
                for (const auto& [ts, w] : cluster)  // assign_budgets over 3 dp=1 nodes
                    t.budget_trace.emplace_back(ts, w * 1.0 / 3);
                for (int j = 0; j < 5; ++j)
                    t.load_trace.emplace_back(720.0 * j, rng.uniform(0.3, 1.2) * tmax);
                t.noise_amp = 0.04;
                t.noise_key = rng.next_u64();
                traces.push_back(t);
            }
        }
        const int n_steps = 7200;
        // the reference side: the same plant loop over wattserve's own functions
        auto reference = [&](const gpu::ReplayTrace& t, ControllerState st, gpu::PlantState ps,
                             std::int64_t first, int steps, std::vector<DecisionRecord>& recs) {
            const ModelProfile& pm = profiles[static_cast<std::size_t>(t.model)];
            std::vector<OperatingPoint> cands;
            for (double c : caps)
                for (int b : batches)
                    cands.push_back(OperatingPoint{c, b, pm.deployment.tp, pm.deployment.ep,
                                                   pm.deployment.dp});
            const Scorer score = detail::cached(analytic_scorer(pm, gspec));
            detail::NodeRuntime n;
            n.profile = &pm;
            n.cfg.tp = pm.deployment.tp;
            n.cfg.ep = pm.deployment.ep;
            n.cfg.dp = pm.deployment.dp;
            for (int kk = 0; kk < steps; ++kk) {
                const std::int64_t step = first + kk;
                const double t0 = step * 0.5, t1 = t0 + 0.5;
                n.node_budget = detail::trace_value(t.budget_trace, t0);
                const double cap = detail::enforce_cap(ps.applied_cap_w, ps.batch_cap, n, gspec, k);
                const OperatingPoint p{cap, ps.batch_cap, n.cfg.tp, n.cfg.ep, n.cfg.dp};
                // plant noise: one splitmix64 draw per step pair, 32 bits per step
                const std::uint64_t x = t.noise_key ^ (std::uint64_t{3} << 48) ^
                                        static_cast<std::uint64_t>(step >> 1);
                const double u = static_cast<double>(static_cast<std::uint32_t>(
                                     splitmix64(x) >> (32 * (step & 1)))) * 0x1.0p-32;
                const double measured = std::min(detail::trace_value(t.load_trace, t0),
                                                 cluster_throughput(p, pm, gspec)) *
                                        (1.0 + t.noise_amp * (2.0 * u - 1.0));
                Targets tg = t.targets;
                if (n.node_budget > 0.0) tg.power_budget_w = n.node_budget;
                auto [d, st2] = control_step(TelemetryInput{t1, measured}, t1, tg, cands, score, k,
                                             st, cfg);
                st = st2;
                DecisionRecord r;
                r.t_s = t1;
                r.point = d.point;
                r.applied = d.applied;
                r.reason = d.reason;
                r.err_norm = tg.throughput_tps > 0.0 ? (tg.throughput_tps - measured) / tg.throughput_tps : 0.0;
                r.bias = st.bias;
                recs.push_back(r);
                ps.applied_cap_w = ps.inflight_cap_w;
                if (d.applied) {
                    ps.batch_cap = d.point.batch;
                    ps.inflight_cap_w = d.point.cap_watts;
                }
            }
            return std::make_pair(st, ps);
        };
        const int nt = static_cast<int>(traces.size());
        const auto full = gpu::replay(ctx, scorers, profiles, gspec, k, caps, batches, cfg, traces,
                                      n_steps, 0.5, 0, nullptr, nullptr, nt);
        const auto part = gpu::replay(ctx, scorers, profiles, gspec, k, caps, batches, cfg, traces,
                                      2999, 0.5, 0, nullptr, nullptr, nt);
        const auto rest = gpu::replay(ctx, scorers, profiles, gspec, k, caps, batches, cfg, traces,
                                      n_steps - 2999, 0.5, 2999, &part.states, &part.plant, nt);
        auto same_rec = [](const DecisionRecord& a, const DecisionRecord& b) {
            return same_bits(a.t_s, b.t_s) && a.point == b.point && a.applied == b.applied &&
                   a.reason == b.reason && same_bits(a.err_norm, b.err_norm) &&
                   same_bits(a.bias, b.bias);
        };
        bool ok = true, resumed = true;
        int budget_decisions = 0;
        for (int i = 0; i < nt; ++i) {
            const ModelProfile& pm = profiles[static_cast<std::size_t>(traces[i].model)];
            ControllerState st0;
            st0.current = OperatingPoint{400.0, 64, pm.deployment.tp, pm.deployment.ep, pm.deployment.dp};
            std::vector<DecisionRecord> recs;
            const auto [st, ps] = reference(traces[i], st0, gpu::PlantState{400.0, 400.0, 64}, 0,
                                            n_steps, recs);
            ok = ok && same(full.states[i], st) && full.plant[i].applied_cap_w == ps.applied_cap_w &&
                 full.plant[i].inflight_cap_w == ps.inflight_cap_w &&
                 full.plant[i].batch_cap == ps.batch_cap && full.decisions[i].size() == recs.size();
            for (std::size_t s2 = 0; ok && s2 < recs.size(); ++s2) {
                ok = same_rec(full.decisions[i][s2], recs[s2]);
                budget_decisions += recs[s2].reason == DecisionReason::BudgetConstrainedMaxThroughput;
            }
            resumed = resumed && same(rest.states[i], st);
            for (std::size_t s2 = 0; resumed && s2 < recs.size(); ++s2)
                resumed = same_rec(s2 < 2999 ? part.decisions[i][s2] : rest.decisions[i][s2 - 2999],
                                   recs[s2]);
        }
        EXPECT(ok, "gpu::replay == control_step over the demand-response trace (7,200 steps)");
        EXPECT(resumed, "gpu::replay resumed at step 2999 from its own states");
        EXPECT(budget_decisions > 0, "the budget trace bound some decisions");
        bool threw = false;
        try {
            std::vector<ControllerState> bad(traces.size());
            for (auto& b2 : bad) b2.current.cap_watts = 123.0;  // not a candidate cap
            gpu::replay(ctx, scorers, profiles, gspec, k, caps, batches, cfg, traces, 10, 0.5, 0,
                        &bad);
        } catch (const config_error& e) {
            threw = std::string(e.what()).find("not a candidate") != std::string::npos;
        }
        EXPECT(threw, "replay: a non-candidate ControllerState::current throws config_error");
    }

    std::printf("%s: %d checks, %d failures\n", g_fail ? "FAIL" : "PASS", g_checks, g_fail);
    return g_fail > 255 ? 255 : g_fail;
}
