/*
 * pals_gpu.h — C ABI of the B200 hot path for the PALS / wattserve reference.
 *
 * This is the drop-in boundary. Every entry point below replaces one call
 * site of the reference's header-only C++ API (paths relative to
 * /root/reference/proj/include/wattserve/):
 *
 *   pals_eval            throughput() + avg_gpu_power()           model.hpp:72-84
 *   pals_select          select_config() over many Targets         controller.hpp:132-201
 *   pals_select_one      select_config(), one call                 controller.hpp:132-201
 *   pals_control_step_one control_step(), one call                 controller.hpp:210-267
 *   pals_replay          control_step() replayed over traces       controller.hpp:210-267
 *                        driven by the fluid plant of DESIGN.md §4 (sim.hpp:195-205, 431-472)
 *   pals_model_analytic  analytic_scorer(profile, gpu)              controller.hpp:107-111
 *   pals_model_table     TableScorer (test fake)                    tests/test_controller.cpp:17-29
 *   pals_model_forest    predictor_scorer(bundle, model_id)         controller.hpp:100-105,
 *                                                                    forest.hpp:227-235
 *   pals_plan_frontier   build_frontier() / evaluate_regime()       pareto.hpp:31-59,114-135
 *   pals_allocate_budget allocate_budget() over many clusters      allocator.hpp:76-186,
 *                        (assign_budgets' per-node requests)       sim.hpp:313-336
 *
 * Plain C types only: pointers, sizes, POD structs. No torch, no C++.
 * Errors follow the reference's exception taxonomy (types.hpp:13-23):
 *   PALS_ECONFIG  <-> wattserve::config_error
 *   PALS_EDATA    <-> wattserve::data_error
 *   PALS_ERANGE   <-> std::out_of_range
 *   PALS_ERUNTIME  CUDA / allocation failures (no reference counterpart)
 * The message of the last failing call on the calling thread is returned by
 * pals_last_error(); messages start with the reference's own text where one
 * exists (e.g. "select_config: empty candidate list").
 *
 * Threading: calls on different contexts are independent; calls on one
 * context are serialised by the caller (one host thread per GPU).
 */
#ifndef PALS_GPU_H
#define PALS_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PALS_ABI_VERSION 1

#define PALS_OK 0
#define PALS_ECONFIG 2
#define PALS_EDATA 3
#define PALS_ERUNTIME 4
#define PALS_ERANGE 5

/* Objective (controller.hpp:17) */
#define PALS_OBJ_QOS 0    /* Objective::QosMaxEfficiency   */
#define PALS_OBJ_BUDGET 1 /* Objective::BudgetMaxThroughput */

/* DecisionReason (controller.hpp:65-71), same numeric order */
#define PALS_REASON_QOS_FEASIBLE 0
#define PALS_REASON_FALLBACK_MAX_T 1
#define PALS_REASON_BUDGET_MAX_T 2
#define PALS_REASON_HOLD 3
#define PALS_REASON_ORACLE 4

#define PALS_MAX_TP_KEYS 8

/* GpuSpec (types.hpp:27-39) */
typedef struct {
    double idle_watts;
    double min_cap_watts;
    double max_cap_watts;
    double max_frequency;
} pals_gpu_spec;

/* SystemPowerCoeffs (types.hpp:42-49) */
typedef struct {
    double alpha;
    double beta_watts;
} pals_coeffs;

/* ModelProfile (types.hpp:66-107), flattened: comm_fixed_by_tp becomes
 * the parallel arrays tp_keys[n_tp] / comm_fixed[n_tp]. */
typedef struct {
    char name[64];
    double compute_fixed;
    double compute_per_seq;
    double comm_per_seq;
    double internode_factor;
    double knee_watts;
    double compute_power_base;
    double compute_power_per_seq;
    double comm_power;
    double overlap;
    double comm_fixed[PALS_MAX_TP_KEYS];
    double total_params_b;
    double active_params_b;
    int32_t tp_keys[PALS_MAX_TP_KEYS];
    int32_t n_tp;
    int32_t num_experts;
    int32_t top_k;
    int32_t deploy_tp;
    int32_t deploy_ep;
    int32_t deploy_dp;
} pals_profile;

/* OperatingPoint (types.hpp:110-116) */
typedef struct {
    double cap_watts;
    int32_t batch;
    int32_t tp;
    int32_t ep;
    int32_t dp;
} pals_point;

/* One select_config() call's non-candidate arguments (controller.hpp:132-135):
 * Targets{throughput_tps, power_budget_w, objective} plus bias, headroom, margin.
 * has_budget == 0 is std::nullopt. */
typedef struct {
    double throughput_tps;
    double power_budget_w;
    double bias;
    double target_headroom;
    double budget_margin;
    int32_t objective;
    int32_t has_budget;
} pals_query;

/* Targets (controller.hpp:19-29) */
typedef struct {
    double throughput_tps;
    double power_budget_w;
    double epsilon;
    int32_t has_budget;
    int32_t objective;
} pals_targets;

/* ControllerConfig (controller.hpp:37-53) with PidGains (:31-35) inlined */
typedef struct {
    double kp;
    double ki;
    double kd;
    double integral_clamp;
    double bias_min;
    double bias_max;
    double interval_s;
    double target_headroom;
    double budget_margin;
    int32_t sustain_intervals;
    int32_t _pad;
} pals_ctrl_cfg;

/* ControllerState (controller.hpp:55-63); last_targets.has_value() is has_last_targets */
typedef struct {
    double bias;
    double integral;
    double prev_error;
    pals_point current;
    pals_targets last_targets;
    int32_t has_prev_error;
    int32_t sustain_count;
    int32_t has_last_targets;
    int32_t _pad;
} pals_ctrl_state;

/* Decision (controller.hpp:85-89) */
typedef struct {
    pals_point point;
    int32_t applied;
    int32_t reason;
} pals_decision;

/* TelemetryInput (controller.hpp:203-206) */
typedef struct {
    double t_s;
    double throughput_tps;
} pals_telemetry;

/* Synthetic fluid-plant replay workload. Every trace is a pure
 * function of (seed, global trace index), so shards need no input transfer. */
typedef struct {
    uint64_t seed;
    int64_t first_trace;      /* global index of this shard's first trace */
    int64_t n_traces;
    int32_t n_steps;          /* control intervals per trace */
    int32_t objective_mode;   /* 0 all QoS, 1 all budget-throughput, 2 mixed 50/50 */
    double interval_s;
    double qos_frac_lo, qos_frac_hi;   /* target = U(lo,hi) * unconstrained T */
    double load_lo, load_hi;           /* offered load = U(lo,hi) * unconstrained T */
    double noise_amp;                  /* measured *= 1 + amp*U(-1,1) */
    double budget_lo_frac, budget_hi_frac; /* budget = U(lo*min p_node, hi*max p_node) */
    double epsilon;                    /* Targets::epsilon */
    int32_t seg_min, seg_max;          /* segment length U{min..max} steps */
    int32_t budget_mode;               /* 0 unbudgeted, 1 piecewise-constant budget */
    int32_t n_log_traces;              /* first n traces log every step */
} pals_replay_spec;

/* Per-trace replay result */
typedef struct {
    uint64_t digest;      /* FNV-1a over per-step (idx, applied, reason) words + final state */
    double final_bias;
    double energy_j;      /* sum of cluster_system_power * interval */
    double tokens;        /* sum of measured tps * interval */
    int32_t n_applied;
    int32_t final_idx;
    int32_t model;
    int32_t objective;
} pals_trace_summary;

/* Per-step decision log record (metrics.hpp:145-156 fields that vary) */
typedef struct {
    int32_t idx;       /* candidate index of Decision::point */
    uint8_t applied;
    uint8_t reason;
    uint16_t cap_tenths; /* enforced cap * 10 after the breaker walk */
} pals_step_log;

/* Per-step decision detail (sim.hpp:122-129 DecisionRecord fields not in
 * pals_step_log): err_norm = (target - measured) / target (sim.hpp:438-440, any
 * objective; 0 without a target) and the controller bias after the step (:463). */
typedef struct {
    double err_norm;
    double bias;
} pals_step_detail;

typedef struct pals_ctx pals_ctx;
typedef struct pals_model pals_model;
typedef struct pals_grid pals_grid;
typedef struct pals_plan pals_plan;

const char* pals_last_error(void);
int pals_abi_version(void);

/* ---- context ---------------------------------------------------------- */
int pals_ctx_create(int device, pals_ctx** out);
int pals_ctx_destroy(pals_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores
 * the context's own stream. */
int pals_ctx_set_stream(pals_ctx* ctx, void* cuda_stream);
void* pals_ctx_stream(pals_ctx* ctx);
int pals_ctx_sync(pals_ctx* ctx);
/* Number of kernels this context has launched so far. */
int64_t pals_ctx_launch_count(pals_ctx* ctx);
/* Replay kernel layout for pals_replay / pals_replay_device: PALS_REPLAY_THREAD
 * (default: one thread per trace, warps made objective-uniform) or PALS_REPLAY_WARP
 * (one warp per trace, the layout BASELINE cfg4 names; lanes split the noise draws,
 * the feasibility searches and the enforce_cap walk). Results are identical. */
#define PALS_REPLAY_THREAD 0
#define PALS_REPLAY_WARP 1
int pals_ctx_set_replay_layout(pals_ctx* ctx, int32_t layout);
/* Single calls (pals_select_one / pals_control_step_one on a cached candidate set) are
 * answered by a one-warp kernel kept resident on its own high-priority stream: a call posts
 * its request in mapped pinned memory and polls the answer (no kernel launch per call). The
 * kernel exits after idle_us microseconds without a request and is relaunched by the next
 * call; idle_us = 0 launches one kernel per call instead. Default 2000. */
int pals_ctx_set_one_server(pals_ctx* ctx, int64_t idle_us);

/* ---- models (the three concrete Scorer kinds) ------------------------- */
/* analytic_scorer(profile, gpu): validates like ModelProfile::validate (types.hpp:88-106) */
int pals_model_analytic(pals_ctx* ctx, const pals_profile* profile, const pals_gpu_spec* gpu,
                        pals_model** out);
/* TableScorer: scores looked up by point value, first match wins */
int pals_model_table(pals_ctx* ctx, const pals_point* points, const double* throughput_tps,
                     const double* gpu_power_w, int64_t n, pals_model** out);
/* predictor_scorer(bundle, model_id): one tree ensemble per target, SoA nodes.
 * Trees of one forest are concatenated; tree t spans [tree_offset[t], tree_offset[t+1]).
 * child indices are tree-local (forest.hpp:62-68). model_index is the one-hot slot
 * FeatureSchema::model_index(model_id) (forest.hpp:34-39); n_features = 5 + n_models. */
int pals_model_forest(pals_ctx* ctx, int32_t n_models, int32_t model_index,
                      const pals_coeffs* coeffs,
                      int32_t t_n_trees, const int64_t* t_tree_offset, const int32_t* t_feature,
                      const double* t_threshold, const int32_t* t_left, const int32_t* t_right,
                      const double* t_value,
                      int32_t p_n_trees, const int64_t* p_tree_offset, const int32_t* p_feature,
                      const double* p_threshold, const int32_t* p_left, const int32_t* p_right,
                      const double* p_value, pals_model** out);
int pals_model_destroy(pals_model* m);
/* Number of cells of a forest model's exact lattice table (0: evaluated by the
 * direct tree walk; -1: not a forest model). */
int64_t pals_model_forest_cells(const pals_model* m);
/* 1: evaluate a forest model by the literal tree walk even when a cell table exists. */
int pals_model_forest_set_direct(pals_model* m, int direct);

/* ---- candidate grids -------------------------------------------------- */
int pals_grid_points(pals_ctx* ctx, const pals_point* points, int64_t n, pals_grid** out);
/* Canonical sweep nesting cap -> batch -> tp -> ep -> dp (sweep.hpp:134-138) */
int pals_grid_axes(pals_ctx* ctx, const double* caps, int32_t n_caps, const int32_t* batches,
                   int32_t n_batches, const int32_t* tps, int32_t n_tps, const int32_t* eps,
                   int32_t n_eps, const int32_t* dps, int32_t n_dps, pals_grid** out);
int64_t pals_grid_size(const pals_grid* g);
int pals_grid_destroy(pals_grid* g);

/* ---- evaluation: Scorer(point) for every grid point ------------------- */
/* Host outputs: throughput_tps and gpu_power_w per point (CandidateScore). */
int pals_eval(pals_ctx* ctx, const pals_model* m, const pals_grid* g, double* throughput_tps,
              double* gpu_power_w);
/* PredictorBundle::predict (forest.hpp:227-235) for n device-resident points:
 * throughput_hat and power_hat per point (forest models; async). */
int pals_predict_device(pals_ctx* ctx, const pals_model* m, const pals_point* d_points, int64_t n,
                        double* d_T, double* d_P);
/* Device outputs, async on the context stream (analytic and forest models). */
int pals_eval_device(pals_ctx* ctx, const pals_model* m, const pals_grid* g, double* d_T,
                     double* d_P);

/* ---- selection plans: model x grid x coeffs --------------------------- */
int pals_plan_create(pals_ctx* ctx, const pals_model* m, const pals_grid* g,
                     const pals_coeffs* coeffs, pals_plan** out);
int pals_plan_destroy(pals_plan* p);
/* Async on the context stream: evaluate the grid and build the rank tables. */
int pals_plan_prepare(pals_plan* p);
/* Async: select for n queries resident in device memory. */
int pals_plan_select_device(pals_plan* p, const pals_query* d_queries, int64_t n,
                            int32_t* d_index, uint8_t* d_reason);
/* Async: one full step (prepare + select) for device-resident queries, replayed
 * from a CUDA graph captured on the first call with these buffers. */
int pals_plan_run(pals_plan* p, const pals_query* d_queries, int64_t n, int32_t* d_index,
                  uint8_t* d_reason);
/* Host buffers in and out: prepare + H2D + select + D2H, synchronous.
 * The batched equivalent of n calls to select_config (controller.hpp:132). */
int pals_select(pals_plan* p, const pals_query* queries, int64_t n, int32_t* index,
                uint8_t* reason);
/* Host copies of the per-point scores the plan selected on:
 * t_hat = dp*T, p_node = dp*(alpha*4*P+beta), eff = t_hat/p_node (controller.hpp:147-150,163) */
int pals_plan_scores(pals_plan* p, double* t_hat, double* p_node, double* eff);
/* Diagnostics of the last select: queries resolved by the exact sequential fold. */
int64_t pals_plan_last_exact_count(const pals_plan* p);
/* How a plan decides its queries (results identical either way):
 * PALS_DECIDE_SCAN (default) evaluates every (config, query) pair of a query's class in
 * the pair scan — the config-evaluation workload BASELINE.json measures; PALS_DECIDE_PREFIX
 * answers each query from prefix-minimum tables over the sorted orders (O(1) per QoS-only
 * or budget-only query, one block of at most n/64 positions per QoS+budget query): the
 * fastest time to decide. */
#define PALS_DECIDE_SCAN 0
#define PALS_DECIDE_PREFIX 1
int pals_plan_set_decide(pals_plan* p, int32_t mode);
/* Force every query through the exact sequential fold (testing). */
int pals_plan_set_force_exact(pals_plan* p, int force);
/* Synchronises, then reports the last select's per-class query counts:
 * class_counts[0..3] = QoS-no-budget / QoS+budget / budget-only scans / no-scan,
 * class_counts[4] = forced exact, class_counts[5] = queries decided by the exact fold.
 * Scanned (query, point) pairs = (c[0]+c[1]+c[2]) * grid size. */
int pals_plan_stats(pals_plan* p, int64_t* class_counts6);

/* ---- measurement helpers (bench.py) ----------------------------------- */
/* When enabled, the select path records CUDA events around its pair-scan kernel
 * on the context stream; pals_plan_scan_ms() synchronises on the end event and
 * returns that kernel's duration in the last select (ms, < 0 if unavailable). */
int pals_plan_time_scan(pals_plan* p, int enable);
double pals_plan_scan_ms(pals_plan* p);
/* Peak integer compare+min rate (ops/s) and FP64 FMA rate (flop/s) of this device. */
int pals_measure_peaks(pals_ctx* ctx, double* int_ops_per_s, double* fp64_flops_per_s);

/* ---- single-call mirrors (the C++ adapter uses these) ----------------- */
int pals_select_one(pals_ctx* ctx, const pals_model* m, const pals_point* candidates, int64_t n,
                    const pals_targets* targets, const pals_coeffs* coeffs, double bias,
                    double target_headroom, double budget_margin, pals_decision* out);
int pals_control_step_one(pals_ctx* ctx, const pals_model* m, const pals_telemetry* telemetry,
                          double now_s, const pals_targets* targets,
                          const pals_point* candidates, int64_t n, const pals_coeffs* coeffs,
                          const pals_ctrl_state* state, const pals_ctrl_cfg* cfg,
                          pals_decision* out_decision, pals_ctrl_state* out_state);

/* ---- batched controller replay --------------------------------------- */
/* models[k] scores candidate grid k (the scenario grid caps x batches at
 * profile k's deployment tp/ep/dp, built by build_candidates order sim.hpp:293-308);
 * plant[k] is the analytic profile the fluid plant runs (the "true" system).
 * Trace i uses model splitmix64(seed ^ i) % n_models. summaries: n_traces
 * entries (host). logs: n_log_traces * n_steps entries (host) or NULL. */
int pals_replay(pals_ctx* ctx, int32_t n_models, pals_model* const* models,
                const pals_profile* plant, const pals_gpu_spec* gpu, const pals_coeffs* coeffs,
                const double* caps, int32_t n_caps, const int32_t* batches, int32_t n_batches,
                const pals_ctrl_cfg* cfg, const pals_replay_spec* spec,
                pals_trace_summary* summaries, pals_step_log* logs);

/* Replay with device-resident outputs (bench: no host copies in the timed region).
 * Plans are built once per (models, caps, batches) and cached in the context. */
int pals_replay_device(pals_ctx* ctx, int32_t n_models, pals_model* const* models,
                       const pals_profile* plant, const pals_gpu_spec* gpu,
                       const pals_coeffs* coeffs, const double* caps, int32_t n_caps,
                       const int32_t* batches, int32_t n_batches, const pals_ctrl_cfg* cfg,
                       const pals_replay_spec* spec, pals_trace_summary* d_summaries,
                       pals_step_log* d_logs);

/* pals_replay / pals_replay_device plus per-step details (err_norm, bias) for the
 * logged traces (NULL: none). Host or device buffers as the base call. */
int pals_replay_ex(pals_ctx* ctx, int32_t n_models, pals_model* const* models,
                   const pals_profile* plant, const pals_gpu_spec* gpu, const pals_coeffs* coeffs,
                   const double* caps, int32_t n_caps, const int32_t* batches, int32_t n_batches,
                   const pals_ctrl_cfg* cfg, const pals_replay_spec* spec,
                   pals_trace_summary* summaries, pals_step_log* logs,
                   pals_step_detail* details);
int pals_replay_device_ex(pals_ctx* ctx, int32_t n_models, pals_model* const* models,
                          const pals_profile* plant, const pals_gpu_spec* gpu,
                          const pals_coeffs* coeffs, const double* caps, int32_t n_caps,
                          const int32_t* batches, int32_t n_batches, const pals_ctrl_cfg* cfg,
                          const pals_replay_spec* spec, pals_trace_summary* d_summaries,
                          pals_step_log* d_logs, pals_step_detail* d_details);

/* ---- batched controller replay over CALLER traces ---------------------- */
/* One point of a piecewise-constant signal: the reference's budget-trace row
 * std::pair<double,double>{t_seconds, value} (scenario_io.hpp:13-25), same layout, so a
 * std::vector<std::pair<double,double>> can be passed as is. The signal's value at t is
 * detail::trace_value (sim.hpp:167-174): the value of the last point of the leading run
 * with t_s <= t, else the first point's value. */
typedef struct {
    double t_s;
    double value;
} pals_signal_point;

/* NodeRuntime's actuation state (sim.hpp:155-157): the cap the breaker enforces this
 * interval, the cap that lands next interval, the batch cap. Caps must be candidate caps
 * and the batch cap a candidate batch. */
typedef struct {
    double applied_cap_w;
    double inflight_cap_w;
    int32_t batch_cap;
    int32_t _pad;
} pals_plant_state;

/* One caller trace: a node of the fluid plant under caller signals.
 * Budget: node_budget = budget signal at t0 (<= 0 or n_budget == 0: unbudgeted, as
 * NodeRuntime::node_budget, sim.hpp:164, 198, 436). Offered load (tokens/s) = load signal
 * at t0. measured = min(offered, dp * throughput(enforced cap, batch cap)) * noise with
 * noise = 1 + noise_amp * (2 u - 1), u = the 53-bit uniform of
 * splitmix64(noise_key ^ 3 << 48 ^ step) (step = the global step index; noise_amp 0: none).
 * Targets{target_tps, node_budget if > 0, epsilon, objective} every step (sim.hpp:432-436). */
typedef struct {
    int64_t budget_off;    /* first point of the budget signal in the call's signal array */
    int64_t load_off;      /* first point of the offered-load signal */
    double target_tps;
    double epsilon;
    double noise_amp;
    uint64_t noise_key;
    int32_t n_budget;      /* points (0: never budgeted) */
    int32_t n_load;        /* points (>= 1) */
    int32_t model;         /* models[model] scores, plant[model] is the true system */
    int32_t objective;     /* PALS_OBJ_* */
} pals_trace;

/* The arguments of one pals_replay_traces call. Steps are global: step k of this call is
 * interval first_step + k, t0 = (double)(first_step + k) * interval_s, t1 = t0 + interval_s
 * (Simulator::run, sim.hpp:229-231), so a replay split at any step and resumed from the
 * returned states gives the same decisions as one uninterrupted call.
 * init / init_plant: per-trace ControllerState / plant state, or NULL for the sim's start
 * (ControllerState{} at (max cap, max batch), sim.hpp:284-288). ControllerState::current must
 * be a candidate of the trace's model (caps x batches at its deployment tp/ep/dp).
 * Outputs: summaries (n_traces; digest and totals cover this call's steps), final states
 * (may be NULL), per-step logs / details of traces [0, n_log_traces) (may be NULL). */
typedef struct {
    int64_t n_traces;
    int64_t first_step;
    int32_t n_steps;
    int32_t n_log_traces;
    double interval_s;
    const pals_trace* traces;
    const pals_signal_point* signal;
    int64_t n_signal;
    const pals_ctrl_state* init;
    const pals_plant_state* init_plant;
    pals_trace_summary* summaries;
    pals_ctrl_state* final_state;
    pals_plant_state* final_plant;
    pals_step_log* logs;
    pals_step_detail* details;
} pals_trace_batch;

/* control_step (controller.hpp:210-267) replayed over caller traces: host buffers,
 * synchronous. Invalid traces (model / objective out of range, signal offsets outside the
 * signal array, n_load < 1, a state point that is not a candidate) fail the call with
 * PALS_ECONFIG naming the first one. Same models / plant / candidate axes as pals_replay. */
int pals_replay_traces(pals_ctx* ctx, int32_t n_models, pals_model* const* models,
                       const pals_profile* plant, const pals_gpu_spec* gpu,
                       const pals_coeffs* coeffs, const double* caps, int32_t n_caps,
                       const int32_t* batches, int32_t n_batches, const pals_ctrl_cfg* cfg,
                       const pals_trace_batch* batch);
/* Same with every pointer of *batch device-resident; async on the context stream. An
 * invalid trace gets summary.model = -1; pals_replay_traces_status() synchronises and
 * returns the first invalid trace index of the last call on ctx (-1: none). */
int pals_replay_traces_device(pals_ctx* ctx, int32_t n_models, pals_model* const* models,
                              const pals_profile* plant, const pals_gpu_spec* gpu,
                              const pals_coeffs* coeffs, const double* caps, int32_t n_caps,
                              const int32_t* batches, int32_t n_batches,
                              const pals_ctrl_cfg* cfg, const pals_trace_batch* batch);
int64_t pals_replay_traces_status(pals_ctx* ctx);

/* ---- multi-GPU driver: one host thread and one context per device ------ */
/* The reference steps nodes one after another in one thread (sim.hpp:243-244); queries
 * and traces are independent, so here they are split into contiguous shards, one per
 * device, each run by that device's own worker thread on its own context and stream.
 * Nothing crosses devices until the results: by default every shard lands straight in
 * the caller's host buffer from its own device; with pals_multi_set_gather(m, 1) the
 * shards are first gathered into device 0 (cudaMemcpyPeerAsync over NVLink) and read
 * back from there in one copy. A device may be listed more than once (two contexts on
 * one GPU: the N>1 path on a single-GPU box). Results equal the one-context call's
 * byte for byte. */
typedef struct pals_multi pals_multi;
int pals_multi_create(const int32_t* devices, int32_t n_devices, pals_multi** out);
int pals_multi_destroy(pals_multi* m);
int32_t pals_multi_size(const pals_multi* m);
/* The context of rank r (its device, stream and launch counter). */
pals_ctx* pals_multi_ctx(pals_multi* m, int32_t rank);
int pals_multi_set_gather(pals_multi* m, int32_t to_device0);
/* A scorer replicated on every device: pals_model_analytic / _table on each context.
 * *id indexes m's models. */
int pals_multi_model_analytic(pals_multi* m, const pals_profile* profile,
                              const pals_gpu_spec* gpu, int32_t* id);
int pals_multi_model_table(pals_multi* m, const pals_point* points, const double* throughput_tps,
                           const double* gpu_power_w, int64_t n, int32_t* id);
/* select_config for n queries over one candidate list (pals_select, sharded). */
int pals_multi_select(pals_multi* m, int32_t model, const pals_point* points, int64_t n_points,
                      const pals_coeffs* coeffs, const pals_query* queries, int64_t n,
                      int32_t* index, uint8_t* reason);
/* pals_replay_ex over spec's traces (models[k] = ids from pals_multi_model_*). */
int pals_multi_replay(pals_multi* m, int32_t n_models, const int32_t* models,
                      const pals_profile* plant, const pals_gpu_spec* gpu,
                      const pals_coeffs* coeffs, const double* caps, int32_t n_caps,
                      const int32_t* batches, int32_t n_batches, const pals_ctrl_cfg* cfg,
                      const pals_replay_spec* spec, pals_trace_summary* summaries,
                      pals_step_log* logs, pals_step_detail* details);
/* pals_replay_traces over batch's traces (host buffers; the signal array is shared). */
int pals_multi_replay_traces(pals_multi* m, int32_t n_models, const int32_t* models,
                             const pals_profile* plant, const pals_gpu_spec* gpu,
                             const pals_coeffs* coeffs, const double* caps, int32_t n_caps,
                             const int32_t* batches, int32_t n_batches,
                             const pals_ctrl_cfg* cfg, const pals_trace_batch* batch);
/* Device milliseconds of each rank's part of the last call (CUDA events on the rank's
 * stream, from its first upload to its last result copy); ms[n_devices]. */
int pals_multi_last_ms(const pals_multi* m, double* ms);

/* ---- decision-log wire format (metrics.hpp:145-157, csvio.hpp:17-21) -- */
/* decisions_csv over the logged traces of a replay (host buffers from pals_replay_ex):
 * header "node,model,t_s,cap_w,batch,tp,ep,dp,applied,reason,err_norm,bias", then one
 * row per (trace, step): node = spec->first_trace + i, model = plant[summary.model].name,
 * t_s = (k + 1) * interval_s, point = candidate idx of caps x batches (build_candidates
 * order, sim.hpp:304-306) at the model's deployment tp/ep/dp, reason strings of
 * controller.hpp:72-82, doubles as "%.10g" — byte-identical to the reference writer.
 * Writes min(length, buf_size) bytes (no terminator) and the full length to *out_len;
 * buf may be NULL to size the output. */
int pals_decisions_csv(const pals_replay_spec* spec, const pals_profile* plant, int32_t n_models,
                       const double* caps, int32_t n_caps, const int32_t* batches,
                       int32_t n_batches, const pals_trace_summary* summaries,
                       const pals_step_log* logs, const pals_step_detail* details, char* buf,
                       int64_t buf_size, int64_t* out_len);
/* fnv1a64 (rng.hpp:22-28): the hash the reference's run manifests record per output
 * file (commands.hpp:26-39, csvio.hpp:69-71). */
uint64_t pals_fnv1a64(const void* data, int64_t n);

/* ---- Pareto frontier (pareto.hpp:31-59) ------------------------------- */
/* build_frontier over the plan's points scored as FrontierPoint{point,
 * cluster_throughput, efficiency} (pareto.hpp:127-130; = the plan's t_hat and eff):
 * n_out frontier point indices, throughput ascending, exact (throughput, efficiency)
 * ties collapsed onto the lower (cap, batch). idx holds up to grid-size entries.
 * Prepares the plan first. Host outputs, synchronous. */
int pals_plan_frontier(pals_plan* p, int32_t* idx, int64_t* n_out);
/* Same, async on the context stream, device outputs (d_n: one int64). */
int pals_plan_frontier_device(pals_plan* p, int32_t* d_idx, int64_t* d_n);
/* build_frontier over explicit FrontierPoints (point, throughput_tps, efficiency_tpj). */
int pals_frontier_values(pals_ctx* ctx, const pals_point* points, const double* throughput_tps,
                         const double* efficiency_tpj, int64_t n, int32_t* idx, int64_t* n_out);

/* ---- cluster budget allocator (allocator.hpp:76-186), batched ---------- */
/* Replaces wattserve::allocate_budget(nodes, cluster_budget_w, gpu, coeffs, quantum_w,
 * selection_margin) (allocator.hpp:76-79) for many independent clusters ("problems")
 * at once, as sim.hpp's assign_budgets builds them (sim.hpp:318-331): node i of a
 * problem runs model node_model[i] (scored by models[k]) with candidates
 * caps x batches at deploy[k].deploy_tp / deploy_ep and dp = node_dp[i].
 * pals_alloc_create precomputes every (model, dp in 1..max_dp) budget-step table
 * (detail::throughput_steps allocator.hpp:34-56 and the margin scaling :106). */
typedef struct pals_alloc pals_alloc;
int pals_alloc_create(pals_ctx* ctx, int32_t n_models, pals_model* const* models,
                      const pals_profile* deploy, const pals_gpu_spec* gpu,
                      const pals_coeffs* coeffs, const double* caps, int32_t n_caps,
                      const int32_t* batches, int32_t n_batches, int32_t max_dp,
                      double selection_margin, pals_alloc** out);
/* General form: candidate set s = points[set_offset[s] .. set_offset[s+1]) scored by
 * set_models[s] (one AllocRequest's candidates + score, allocator.hpp:13-19); a node then
 * names its set in node_model and its dp (for the floor, allocator.hpp:82-83) in node_dp. */
int pals_alloc_create_sets(pals_ctx* ctx, int32_t n_sets, pals_model* const* set_models,
                           const pals_point* points, const int64_t* set_offset,
                           const pals_gpu_spec* gpu, const pals_coeffs* coeffs,
                           double selection_margin, pals_alloc** out);
int pals_alloc_destroy(pals_alloc* a);
/* Host copy of one set's budget steps: n_steps, then power_w / throughput_tps (either
 * may be NULL). In the (model, dp) form set = model * max_dp + dp - 1. */
int pals_alloc_steps(pals_alloc* a, int32_t set, double* power_w, double* throughput_tps,
                     int32_t* n_steps);
/* Problem p owns nodes [node_offset[p], node_offset[p+1]). Per problem: the node budgets
 * (AllocResult::node_budgets_w), total_allocated_w, all_targets_satisfied and a status
 * code: PALS_OK, or the error allocate_budget would throw for that problem (PALS_ECONFIG
 * for no nodes / budget below the floors / a scorer config_error, PALS_ERANGE for a
 * scorer out_of_range or a dp beyond max_dp). Host buffers, synchronous. */
int pals_allocate_budget(pals_alloc* a, double quantum_w, int64_t n_problems,
                         const int64_t* node_offset, const int32_t* node_model,
                         const int32_t* node_dp, const double* node_target,
                         const double* cluster_budget, double* node_budget, double* total,
                         uint8_t* all_satisfied, int32_t* status);
/* Same with device-resident buffers, async on the context stream (n_nodes = node_offset[n]). */
int pals_alloc_run_device(pals_alloc* a, double quantum_w, int64_t n_problems,
                          const int64_t* d_node_offset, int64_t n_nodes,
                          const int32_t* d_node_model, const int32_t* d_node_dp,
                          const double* d_node_target, const double* d_cluster_budget,
                          double* d_node_budget, double* d_total, uint8_t* d_all_satisfied,
                          int32_t* d_status);

/* ---- queue-plant scenario simulator (sim.hpp:222-500) ------------------ */
/* Batched run_scenario(): every scenario is the reference's interval-quantized
 * cluster simulation — Poisson arrivals with lognormal output lengths per node
 * (Rng::substream(seed, node), rng.hpp:30-95), continuous batching under the
 * node's batch cap, the facility breaker (enforce_cap), telemetry, one
 * control_step per interval and the two-stage actuation pipeline — with budgets
 * split by assign_budgets (allocate_budget water-filling for joint / oracle,
 * dp-proportional otherwise) whenever the cluster budget (static or trace)
 * changes. Policies and scorers as Simulator (sim.hpp:209-220, 267-336). */
#define PALS_POLICY_FIXED 0
#define PALS_POLICY_ADAPTIVE_BATCH 1
#define PALS_POLICY_ADAPTIVE_CAP 2
#define PALS_POLICY_JOINT 3
#define PALS_POLICY_ORACLE 4
#define PALS_SIM_MAX_NODES 32

typedef struct {              /* ScenarioNode (sim.hpp:52-60) */
    int32_t model;            /* index into the call's profiles / predictors */
    int32_t tp, ep, dp;
    double qos_fraction;
    double arrival_rate_per_s;
    int32_t initial_backlog;
    int32_t _pad;
} pals_sim_node;

typedef struct {              /* Scenario (sim.hpp:62-94) */
    double duration_s;
    double interval_s;
    uint64_t seed;
    double mean_tokens;       /* OutputLenDist */
    double log_sigma;
    int32_t has_cluster_budget;
    int32_t n_trace;          /* budget_trace points (t_s strictly increasing) */
    double cluster_budget_w;
    const double* trace_t;
    const double* trace_w;
    int32_t policy;           /* PALS_POLICY_* */
    int32_t objective;        /* PALS_OBJ_* */
    pals_ctrl_cfg controller; /* gains, clamps, sustain, headroom, margin (interval_s ignored) */
    double epsilon;
    const double* cand_caps;
    const int32_t* cand_batches;
    int32_t n_caps;
    int32_t n_batches;
    double initial_cap_w;     /* must be one of the policy's candidate caps */
    int32_t initial_batch;    /* must be one of the policy's candidate batches */
    int32_t n_nodes;          /* <= PALS_SIM_MAX_NODES */
    const pals_sim_node* nodes;
} pals_scenario;

typedef struct {              /* one node's MetricsSummary (metrics.hpp:24-48) + run facts */
    double tokens_per_joule;
    double qos_violation_rate;
    double power_tracking_mae_w;
    double total_tokens;
    double total_energy_j;
    double mean_throughput_tps;
    double throughput_target_tps;   /* NodeResult::throughput_target_tps */
    double final_bias;
    uint64_t arrival_stream_hash;   /* NodeResult::arrival_stream_hash */
    int64_t n_requests;             /* spawned (backlog + arrivals) */
    int64_t n_completed;
    int32_t n_applied;
    int32_t final_idx;              /* controller's current point (policy candidate index) */
} pals_sim_node_result;

typedef struct {              /* RunSummary aggregate (metrics.hpp:56-102) + SimResult */
    double tokens_per_joule;
    double qos_violation_rate;      /* worst node */
    double power_tracking_mae_w;
    double total_tokens;
    double total_energy_j;
    double mean_throughput_tps;     /* sum of node means */
    double cluster_tracking_mae_w;
    double sim_total_energy_j;      /* SimResult::total_energy_j (interval-major sum) */
    int32_t n_intervals;
    int32_t n_budget_changes;
} pals_sim_result;

typedef struct {              /* TelemetrySample (sim.hpp:109-120) */
    double t_s;
    double gpu_power_w;
    double sys_power_w;
    double throughput_tps;
    double utilization;
    double node_budget_w;
    double applied_cap_w;
    int32_t queue_depth;
    int32_t active_batch;
    int32_t applied_batch_cap;
    int32_t _pad;
} pals_sim_telemetry;

typedef struct {              /* DecisionRecord (sim.hpp:122-129) */
    double err_norm;
    double bias;
    double cap_w;
    int32_t batch;
    uint8_t applied;
    uint8_t reason;
    uint16_t _pad;
} pals_sim_decision;

/* Runs n_scenarios independent scenarios. profiles[m] is model m's calibrated
 * profile (the plant, and the oracle's analytic scorer); predictors[m] its
 * predictor_scorer (a forest model handle) or NULL — policies other than oracle
 * score with the predictor when one is given (sim.hpp:277-281); adaptive-batch,
 * adaptive-cap and joint require it. Outputs: node_results (all nodes, scenario
 * order), results per scenario, and optionally per-interval logs for every node
 * ([node][interval], n_intervals = llround(duration_s / interval_s) each; pass
 * log_stride >= the largest n_intervals). Errors as run_scenario would throw. */
int pals_run_scenarios(pals_ctx* ctx, int32_t n_scenarios, const pals_scenario* scenarios,
                       int32_t n_models, const pals_profile* profiles,
                       pals_model* const* predictors, const pals_gpu_spec* gpu,
                       const pals_coeffs* coeffs, pals_sim_node_result* node_results,
                       pals_sim_result* results, int64_t log_stride,
                       pals_sim_telemetry* telemetry, pals_sim_decision* decisions);

/* RequestRec (sim.hpp:100-107) of every simulated request, when kept. */
typedef struct {
    int64_t id;
    double arrival_s;
    int32_t output_tokens;
    int32_t _pad;
    double generated;
    double completed_s;       /* -1 while open */
} pals_sim_request;
/* With enable != 0, later pals_run_scenarios calls on ctx also record every request
 * (12 B per request on the device); pals_sim_requests then copies node `node`'s
 * records (nodes numbered across scenarios, as node_results) — n = count; out may be
 * NULL to size. */
int pals_sim_keep_requests(pals_ctx* ctx, int32_t enable);
/* Streamed arrivals (default on): pals_run_scenarios launches the simulation after the
 * first chunk of arrival intervals and uploads the rest while it runs. enable = 0 draws and
 * uploads every chunk before the launch — for runs under a kernel profiler, which
 * serialises the launch with the later uploads. */
int pals_sim_set_streaming(pals_ctx* ctx, int32_t enable);
int pals_sim_requests(pals_ctx* ctx, int64_t node, pals_sim_request* out, int64_t cap,
                      int64_t* n);

/* Timing of the last pals_run_scenarios on ctx: host setup seconds (arrival
 * streams, select tables, budget splits, uploads) and the simulation kernel's
 * device milliseconds (CUDA events on the context stream). */
int pals_sim_last_timing(pals_ctx* ctx, double* host_setup_s, double* kernel_ms);

#ifdef __cplusplus
}
#endif

#endif /* PALS_GPU_H */
