// sim.cu — K6: batched queue-plant scenario simulation (run_scenario, sim.hpp:209-500).
//
// One CTA per scenario, one warp per node, one loop iteration per control
// interval — the reference's Simulator::run with every node's step_node
// (sim.hpp:355-473) executed by its warp:
//   (1) arrivals       host-generated streams (below), replayed by index
//   (2) batch + breaker effective_batch, enforce_cap (sim.hpp:195-205; the 5 W walk
//                      is evaluated 32 positions per round across the lanes)
//   (3)+(4) service    continuous batching; the running list (sorted by request id:
//                      admission is FIFO and completion removal keeps order) is
//                      spread over the lanes, the chunk is a warp min-reduction,
//                      completions compact with ballots — every double is the
//                      reference's, element by element
//   (5) telemetry      accumulated into the node's MetricsSummary (metrics.hpp:24-48)
//   (6) control_step   the K3 rank-table select (replay_common.cuh) with the node's
//                      scorer (predictor cells / analytic for the oracle)
//   (7) actuation      batch next interval, cap one interval later
// and, per interval, the cluster draw vs the budget signal (metrics.hpp:71-97).
//
// Host side (the parts a GPU cannot reproduce bit-for-bit, or that do not depend
// on the simulation state):
//   * arrival streams: Rng::substream(seed, node) = std::mt19937_64 seeded with
//     splitmix64(splitmix64(seed) ^ node), Knuth / normal-approximation Poisson and
//     Box-Muller lognormal lengths through the host libm (rng.hpp:30-95) — the
//     reference's own libm calls, which CUDA's libdevice does not match bit for
//     bit. Arrival streams never depend on the policy (sim.hpp header), so they
//     are inputs to the plant, generated once per node.
//   * budget splits: assign_budgets runs whenever the cluster signal changes
//     (sim.hpp:229-238, 313-336); its inputs are the trace and the node scorers,
//     never the simulation state, so every split is precomputed — allocate_budget
//     on the GPU allocator (K4) for joint / oracle, dp-proportional otherwise.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "replay_common.cuh"

namespace pals {
namespace {

// ---- host: the reference's Rng over std::mt19937_64 (rng.hpp:30-95) ----------
struct HostRng {
    std::mt19937_64 eng;
    double spare = 0.0;
    bool have_spare = false;
    explicit HostRng(uint64_t seed) : eng(seed) {}
    double uniform01() { return (double)(eng() >> 11) * 0x1.0p-53; }
    double gaussian(double mean, double stddev) {
        if (have_spare) {
            have_spare = false;
            return mean + stddev * spare;
        }
        double u, v, s;
        do {
            u = 2.0 * uniform01() - 1.0;
            v = 2.0 * uniform01() - 1.0;
            s = u * u + v * v;
        } while (s >= 1.0 || s == 0.0);
        const double m = std::sqrt(-2.0 * std::log(s) / s);
        spare = v * m;
        have_spare = true;
        return mean + stddev * u * m;
    }
    double lognormal(double log_mean, double log_sigma) {
        return std::exp(gaussian(log_mean, log_sigma));
    }
    int poisson(double lambda) {
        if (lambda <= 0.0) return 0;
        if (lambda < 50.0) {
            const double limit = std::exp(-lambda);
            int k = 0;
            double p = 1.0;
            do {
                ++k;
                p *= uniform01();
            } while (p > limit);
            return k - 1;
        }
        const double x = gaussian(lambda, std::sqrt(lambda));
        return x < 0.0 ? 0 : (int)std::lround(x);
    }
};

uint64_t fnv_str(const std::string& s, uint64_t h) {
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001b3ULL;
    }
    return h;
}

std::string fmt10g(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.10g", v);
    return buf;
}

// FNV-1a over the decimal digits of v (std::to_string of a non-negative integer).
inline uint64_t fnv_dec(uint64_t h, long v) {
    char d[24];
    int n = 0;
    do {
        d[n++] = (char)('0' + v % 10);
        v /= 10;
    } while (v);
    while (n) {
        h ^= (unsigned char)d[--n];
        h *= 0x100000001b3ULL;
    }
    return h;
}


// One node's arrival stream (spawn_request, sim.hpp:338-353: the lengths; the arrival hash
// over the requests' strings is chained on the device by k_arrival_hash): request lengths by
// id, and cum[k] = requests spawned before interval k's service (the initial backlog first).
// Generated incrementally, interval range by interval range, straight into its region of
// the streamed upload buffer: cum [n_int + 1], len [cap] (cap: a bound the count never
// reaches in practice — mean + 12 sigma + 1,024; an overflow is reported).
struct StreamGen {
    HostRng rng{0};
    double log_mean = 0.0, log_sigma = 0.0, lam = 0.0;
    int backlog = 0, n_int = 0;
    int32_t* cum = nullptr;  // cum[k * cstride]: the streams' counts are interval-major
    int64_t cstride = 1;
    int32_t* len = nullptr;
    int64_t cap = 0, count = 0;
    bool overflow = false;
    void init(const pals_scenario& sc, int node, int ni, int32_t* c, int64_t cs, int32_t* l,
              int64_t cp) {
        const pals_sim_node& nd = sc.nodes[node];
        rng = HostRng(splitmix64(splitmix64(sc.seed) ^ (uint64_t)node));  // Rng::substream
        log_mean = std::log(sc.mean_tokens) - 0.5 * sc.log_sigma * sc.log_sigma;
        log_sigma = sc.log_sigma;
        lam = nd.arrival_rate_per_s * sc.interval_s;
        backlog = nd.initial_backlog;
        n_int = ni;
        cum = c;
        cstride = cs;
        len = l;
        cap = cp;
        count = 0;
        overflow = false;
    }
    void spawn() {
        const int32_t v = std::max(1, (int)std::lround(rng.lognormal(log_mean, log_sigma)));
        if (count < cap) len[count] = v;
        else overflow = true;
        ++count;
    }
    void run(int k0, int k1) {  // intervals [k0, k1), in order
        if (k0 == 0)
            for (int b = 0; b < backlog; ++b) spawn();
        for (int k = k0; k < k1; ++k) {
            const int n = rng.poisson(lam);
            for (int a = 0; a < n; ++a) spawn();
            cum[k * cstride] = (int32_t)count;  // visible to interval k
        }
        if (k1 == n_int) cum[n_int * cstride] = (int32_t)count;
    }
};

// The arrival hash of a stream (spawn_request, sim.hpp:338-353; fnv1a64 rng.hpp:22-28):
// fnv1a64 chained over to_string(id) + ":" + to_string(len) + "@" + fmt_num(t) per request,
// byte for byte; t's "@%.10g" strings come from the host, one per interval of the stream's
// grid (tails[k] for an interval's spawns, tail0 = "@0" for the initial backlog). One
// thread per stream: the chain is serial, the streams are not.
struct HashJob {
    const int32_t* len;
    const int32_t* cum;  // cum[k * cstride]
    int64_t cstride;
    const uint32_t* toff;  // [n_int + 1] offsets into tchars: interval k's "@t" string
    const char* tchars;
    int n_int, backlog;
};

__device__ __forceinline__ uint64_t dev_fnv_dec(uint64_t h, uint32_t v) {
    char d[12];
    int n = 0;
    do {
        d[n++] = (char)('0' + v % 10u);
        v /= 10u;
    } while (v);
    while (n) {
        h ^= (unsigned char)d[--n];
        h *= 0x100000001b3ULL;
    }
    return h;
}

__global__ void k_arrival_hash(const HashJob* __restrict__ jobs, int n_jobs, uint64_t* out) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_jobs) return;
    const HashJob j = jobs[u];
    uint64_t h = 0xcbf29ce484222325ULL;
    uint32_t id = 0;
    auto req = [&](const char* t, uint32_t tn) {
        h = dev_fnv_dec(h, id);
        h = (h ^ (unsigned char)':') * 0x100000001b3ULL;
        h = dev_fnv_dec(h, (uint32_t)j.len[id]);
        for (uint32_t c = 0; c < tn; ++c) h = (h ^ (unsigned char)t[c]) * 0x100000001b3ULL;
        ++id;
    };
    for (int b = 0; b < j.backlog; ++b) req("@0", 2);
    for (int k = 0; k < j.n_int; ++k) {
        const uint32_t end = (uint32_t)j.cum[(int64_t)k * j.cstride];
        if (id == end) continue;
        const uint32_t t0 = j.toff[k], tn = j.toff[k + 1] - t0;
        while (id < end) req(j.tchars + t0, tn);
    }
    out[u] = h;
}

// trace_value (sim.hpp:167-174) for non-decreasing query times: the value of the
// last point with t_i <= t (the first point's when none), kept with a cursor.
struct TraceCursor {
    const pals_scenario& sc;
    int j = 0;
    double operator()(double t) {
        while (j + 1 < sc.n_trace && sc.trace_t[j + 1] <= t) ++j;
        return sc.trace_w[j];
    }
};

// ---- device layout ------------------------------------------------------------
struct SimNodeDev {
    const ReplayModelDev* sel;  // select tables over the node's candidates + scorer
    const Analytic* plant;      // the node's calibrated profile
    const int32_t* cum;         // [n_int + 1], element k at cum[k * cum_stride]
    int64_t cum_stride;
    const int32_t* len;         // request lengths by id
    int32_t* run_len;           // running list (global fallback): output tokens, generated,
    double* run_gen;            // request id
    int32_t* run_id;
    int32_t* req_k;             // optional per request: completion interval + 1 (0 = open)
    double* req_gen;            // optional per request: generated tokens of open requests
    const double* budget;       // node budget per budget change
    int tp, ep, dp;
    int init_idx;
    double target_tps;
};

struct SimScenDev {
    int node0, n_nodes;
    int n_int;
    int policy, objective;
    int budget_active;
    int n_changes;
    const int32_t* change_k;     // interval at which change c applies
    const double* track_target;  // per interval: cluster tracking target (metrics.hpp:84-90)
    double interval_s, epsilon;
    pals_ctrl_cfg cfg;
};

struct SimArgs {
    const SimScenDev* scen;
    const SimNodeDev* nodes;
    double alpha, beta, idle_w, min_cap;
    pals_sim_node_result* node_out;
    pals_sim_result* out;
    int64_t log_stride;
    pals_sim_telemetry* tel;
    pals_sim_decision* dec;
    int smem_run;  // > 0: running lists live in shared memory, smem_run entries per warp
    const int32_t* order;  // CTA -> scenario
    const int* flags;      // streamed arrivals: per (CTA group, chunk of chunk_k intervals), 1
                           // once on device; a group's flag also covers every earlier group
    int chunk_k;
    int n_chunks;
    int n_groups;  // CTA group of block b: b * n_groups / gridDim.x (runs of the CTA order)
};
constexpr int kSimGroups = 4;  // 2 / 6 / 8 measured no better (scripts/ab_sim.sh)

// Wait until the arrivals of interval k's chunk are on the device (streamed upload): lane 0
// polls the chunk's flag (device memory, written by a copy queued after the chunk's data)
// with acquire loads; a flag that never rises releases the warp after ~20 s (the host raises
// every flag before returning, so this only bounds a host failure).
__device__ __forceinline__ void await_chunk(const SimArgs& a, int k, int& ready_until) {
    if (k < ready_until) return;
    const int c = (int)(((int64_t)blockIdx.x * a.n_groups / gridDim.x) * a.n_chunks) + k / a.chunk_k;
    if ((threadIdx.x & 31) == 0) {
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            int v;
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(a.flags + c) : "memory");
            if (v) break;
            __nanosleep(2000);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 20000000000ull) break;
        }
    }
    __syncwarp();
    ready_until = (k / a.chunk_k + 1) * a.chunk_k;
}

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double warp_min(double v) {
    for (int o = 16; o; o >>= 1) {
        const double w = __shfl_xor_sync(kFull, v, o);
        v = w < v ? w : v;
    }
    return v;
}

__global__ void __launch_bounds__(32 * PALS_SIM_MAX_NODES) k_sim(SimArgs a) {
    const int sid = a.order[blockIdx.x];  // longest scenarios first (shorter tail)
    const SimScenDev S = a.scen[sid];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double sh_sys[PALS_SIM_MAX_NODES], sh_bud[PALS_SIM_MAX_NODES];
    __shared__ double sh_cluster_abs, sh_energy;
    __shared__ int sh_counted;
    if (threadIdx.x == 0) {
        sh_cluster_abs = 0.0;
        sh_energy = 0.0;
        sh_counted = 0;
    }
    const bool live = w < S.n_nodes;
    const int gi = S.node0 + (live ? w : 0);
    const SimNodeDev N = a.nodes[gi];
    // the node's running list: shared memory when it fits, else the global scratch
    extern __shared__ __align__(16) char dyn_smem[];
    double* run_gen = N.run_gen;
    int32_t* run_len = N.run_len;
    int32_t* run_id = N.run_id;
    if (a.smem_run > 0) {
        const size_t nw = blockDim.x >> 5;
        run_gen = (double*)dyn_smem + (size_t)w * a.smem_run;
        run_len = (int32_t*)((double*)dyn_smem + nw * a.smem_run) + (size_t)w * a.smem_run;
        run_id = (int32_t*)((double*)dyn_smem + nw * a.smem_run) + (nw + w) * a.smem_run;
    }
    const ReplayModelDev& m = *N.sel;
    const Analytic& P = *N.plant;
    const double iv = S.interval_s;
    const double target = N.target_tps;
    // Oracle: exhaustive search without feedback lag (sim.hpp:443-448)
    double kp = S.cfg.kp, ki = S.cfg.ki, kd = S.cfg.kd;
    int sustain_n = S.cfg.sustain_intervals;
    if (S.policy == PALS_POLICY_ORACLE) {
        kp = ki = kd = 0.0;
        sustain_n = 0;
    }
    const double sel_target = target * (1.0 + S.cfg.target_headroom);  // controller.hpp:137

    // node runtime (uniform across the warp's lanes)
    double applied_cap = m.cap[N.init_idx], inflight_cap = applied_cap;
    int batch_cap = m.batch[N.init_idx];
    int cur = N.init_idx;
    double bias = 1.0, integral = 0.0, prev_err = 0.0;
    bool has_prev = false, has_last = false, last_bset = false;
    double last_budget = 0.0;
    int sustain = 0;
    int next_admit = 0, R = 0, chg = 0;
    int ready_until = 0;  // intervals whose arrivals are on the device (streamed upload)
    double node_budget = 0.0;
    double kp_budget = -1.0;
    int kpv = m.nd_p, kt = 0;
    double memo_cap = -1.0, memo_budget = -1.0, memo_out = 0.0;
    int memo_b = -1;
    // MetricsSummary accumulators (metrics.hpp:27-41)
    double tot_tokens = 0.0, tot_energy = 0.0, sum_tps = 0.0, track_abs = 0.0;
    long violations = 0, tracked = 0, completed = 0;
    int n_applied = 0;
    pals_sim_telemetry* tl = (live && a.tel && lane == 0) ? a.tel + gi * a.log_stride : nullptr;
    pals_sim_decision* dl = (live && a.dec && lane == 0) ? a.dec + gi * a.log_stride : nullptr;
    __syncthreads();

    for (int k = 0; k < S.n_int; ++k) {
        const double t0 = k * iv;
        const double t1 = t0 + iv;
        double sys_w = 0.0;
        if (live) {
            while (chg < S.n_changes && S.change_k[chg] <= k) node_budget = N.budget[chg++];
            // (1) arrivals: the stream's requests up to this interval are queued (streamed:
            // read through L2, the chunk's flag first)
            await_chunk(a, k, ready_until);
            const int spawned = __ldcg(N.cum + (int64_t)k * N.cum_stride);
            // (2) effective batch from queue pressure, per replica (sim.hpp:360-365)
            const int avail = R + (spawned - next_admit);
            const int per_replica = (avail + N.dp - 1) / N.dp;
            const int b_eff = min(batch_cap, per_replica);
            const int slot_cap = b_eff * N.dp;
            // facility breaker (sim.hpp:195-205)
            double cap = applied_cap;
            if (node_budget > 0.0 && b_eff >= 1) {
                if (applied_cap == memo_cap && b_eff == memo_b && node_budget == memo_budget) {
                    cap = memo_out;
                } else {
                    double c0 = applied_cap;  // walk position of this round's lane 0
                    for (;;) {
                        double c = c0;
                        for (int j = 0; j < lane; ++j) c = smax(P.min_cap, c - 5.0);
                        bool stop = !(c > P.min_cap);
                        if (!stop) {
                            const Score s = analytic_score(P, c, b_eff, N.tp, N.dp);
                            stop = p_node_of(s.P, N.dp, a.alpha, a.beta) <= node_budget;
                        }
                        const unsigned b = __ballot_sync(kFull, stop);
                        if (b) {
                            const int j = __ffs(b) - 1;
                            const double cj = __shfl_sync(kFull, c, j);
                            cap = cj > P.min_cap ? cj : P.min_cap;
                            break;
                        }
                        c0 = smax(P.min_cap, __shfl_sync(kFull, c, 31) - 5.0);
                    }
                    memo_cap = applied_cap;
                    memo_b = b_eff;
                    memo_budget = node_budget;
                    memo_out = cap;
                }
            }
            // (3)+(4) continuous batching (sim.hpp:374-409)
            double tokens = 0.0, gpu_w = a.idle_w, util = 0.0;
            if (b_eff >= 1) {
                double ts;
                const Score s = analytic_score(P, cap, b_eff, N.tp, N.dp, nullptr, &ts);
                gpu_w = s.P;
                const double steps_per_seq = iv / ts;
                double steps_left = steps_per_seq;
                while (steps_left > 1e-9) {
                    if (R < slot_cap && next_admit < spawned) {  // refill freed slots
                        const int n_adm = min(slot_cap - R, spawned - next_admit);
                        for (int j = lane; j < n_adm; j += 32) {
                            run_len[R + j] = __ldcg(N.len + next_admit + j);
                            run_gen[R + j] = 0.0;
                            run_id[R + j] = next_admit + j;
                        }
                        R += n_adm;
                        next_admit += n_adm;
                        __syncwarp();
                    }
                    if (R == 0) break;
                    const int active = min(slot_cap, R);
                    double mn = steps_left;
                    for (int j = lane; j < active; j += 32) {
                        const double left = (double)run_len[j] - run_gen[j];
                        mn = left < mn ? left : mn;
                    }
                    double chunk = warp_min(mn);
                    chunk = chunk < 0.0 ? 0.0 : chunk;
                    for (int j = lane; j < active; j += 32) run_gen[j] += chunk;
                    tokens += chunk * active;
                    steps_left -= smax(chunk, 1e-9);
                    __syncwarp();
                    // completions leave the running list, order kept (sim.hpp:399-407)
                    int kept = 0;
                    for (int base = 0; base < R; base += 32) {
                        const int j = base + lane;
                        int id = 0, rid = 0;
                        double g = 0.0;
                        bool done = false;
                        if (j < R) {
                            id = run_len[j];
                            rid = run_id[j];
                            g = run_gen[j];
                            done = g >= (double)id - 1e-7;
                            if (done && N.req_k) N.req_k[rid] = k + 1;  // completed_s = t1
                        }
                        const unsigned keep = __ballot_sync(kFull, j < R && !done);
                        const unsigned fin = __ballot_sync(kFull, done);
                        __syncwarp();
                        if (j < R && !done) {
                            const int dst = kept + __popc(keep & ((1u << lane) - 1));
                            run_len[dst] = id;
                            run_gen[dst] = g;
                            run_id[dst] = rid;
                        }
                        kept += __popc(keep);
                        completed += __popc(fin);
                        __syncwarp();
                    }
                    R = kept;
                }
                util = tokens / ((double)slot_cap * steps_per_seq);
            }
            sys_w = (double)N.dp * (a.alpha * (double)kGpusPerNode * gpu_w + a.beta);
            // (5) telemetry -> MetricsSummary
            const double tps = tokens / iv;
            tot_tokens += tps * iv;
            tot_energy += sys_w * iv;
            sum_tps += tps;
            if (target > 0.0 && tps < target) ++violations;
            if (S.budget_active && node_budget > 0.0) {
                track_abs += fabs(sys_w - node_budget);
                ++tracked;
            }
            if (tl) {
                pals_sim_telemetry x;
                x.t_s = t1;
                x.gpu_power_w = gpu_w;
                x.sys_power_w = sys_w;
                x.throughput_tps = tps;
                x.utilization = sclamp(util, 0.0, 1.0);
                x.node_budget_w = node_budget;
                x.applied_cap_w = cap;
                x.queue_depth = spawned - next_admit;
                x.active_batch = b_eff;
                x.applied_batch_cap = batch_cap;
                x._pad = 0;
                tl[k] = x;
            }
            // (6) control decision (sim.hpp:431-464)
            const double err = target > 0.0 ? (target - tps) / target : 0.0;
            int d_idx = cur, d_applied = 0, d_reason = PALS_REASON_HOLD;
            if (S.policy != PALS_POLICY_FIXED) {
                // control_step (controller.hpp:210-267); telemetry is never stale here
                double err_norm = 0.0;
                if (S.objective == PALS_OBJ_QOS && target > 0.0) {
                    err_norm = (target - tps) / target;
                    const double promised = (double)N.dp * m.T[cur] * bias;
                    if (promised > 0.0) {
                        const double pred_err = (promised - tps) / promised;
                        integral = sclamp(integral + pred_err, -S.cfg.integral_clamp,
                                          S.cfg.integral_clamp);
                        const double deriv = has_prev ? pred_err - prev_err : 0.0;
                        const double corr = kp * pred_err + ki * integral + kd * deriv;
                        bias = sclamp(bias * (1.0 - corr), S.cfg.bias_min, S.cfg.bias_max);
                        prev_err = pred_err;
                        has_prev = true;
                    }
                }
                const bool bset = node_budget > 0.0;
                const bool changed =
                    !has_last || !(last_bset == bset && (!bset || last_budget == node_budget));
                has_last = true;
                last_bset = bset;
                last_budget = node_budget;
                if (fabs(err_norm) > S.epsilon) ++sustain;
                else sustain = 0;
                const double budget = bset ? node_budget * (1.0 - S.cfg.budget_margin) : 0.0;
                if (bset && budget != kp_budget) {
                    kpv = warp_leading_true(m.nd_p, [&](int i) { return m.up[i] <= budget; });
                    kp_budget = budget;
                }
                if (S.objective == PALS_OBJ_QOS) {
                    const bool ok_lo = kt == 0 || !(m.ut[kt - 1] * bias < sel_target);
                    const bool ok_hi = kt == m.nd_t || (m.ut[kt] * bias < sel_target);
                    if (!(ok_lo && ok_hi))
                        kt = warp_leading_true(
                            m.nd_t, [&](int i) { return !(m.ut[i] * bias < sel_target); });
                }
                int s_idx, s_reason;
                table_select(m, sel_target, bset, budget, kpv, kt, bias, S.objective, &s_idx,
                             &s_reason);
                const bool may_apply = changed || sustain >= sustain_n;
                if (may_apply && s_idx != cur) {
                    cur = s_idx;
                    sustain = 0;
                    d_idx = s_idx;
                    d_applied = 1;
                    d_reason = s_reason;
                } else {
                    d_idx = cur;
                    d_reason = may_apply ? s_reason : PALS_REASON_HOLD;
                }
                if (S.policy == PALS_POLICY_ORACLE && d_reason != PALS_REASON_HOLD)
                    d_reason = PALS_REASON_ORACLE;
            }
            n_applied += d_applied;
            if (dl) {
                pals_sim_decision x;
                x.err_norm = err;
                x.bias = bias;
                x.cap_w = m.cap[d_idx];
                x.batch = m.batch[d_idx];
                x.applied = (uint8_t)d_applied;
                x.reason = (uint8_t)d_reason;
                x._pad = 0;
                dl[k] = x;
            }
            // (7) actuation pipeline (sim.hpp:466-472)
            applied_cap = inflight_cap;
            if (d_applied) {
                batch_cap = m.batch[d_idx];
                inflight_cap = m.cap[d_idx];
            }
            if (lane == 0) {
                sh_sys[w] = sys_w;
                sh_bud[w] = node_budget;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            // SimResult::total_energy_j, interval-major (sim.hpp:411-412)
            double cw = 0.0, bw = 0.0;
            for (int i = 0; i < S.n_nodes; ++i) {
                sh_energy += sh_sys[i] * iv;
                cw += sh_sys[i];
                bw += sh_bud[i];
            }
            if (S.budget_active) {  // cluster draw vs the signal (metrics.hpp:77-96)
                const double tg = S.track_target ? S.track_target[k] : bw;
                if (tg > 0.0) {
                    sh_cluster_abs += fabs(cw - tg);
                    ++sh_counted;
                }
            }
        }
        __syncthreads();
    }
    if (live && N.req_gen)  // requests still running keep their partial progress
        for (int j = lane; j < R; j += 32) N.req_gen[run_id[j]] = run_gen[j];
    if (live && lane == 0) {
        pals_sim_node_result r;
        const double n = (double)S.n_int;
        r.total_tokens = tot_tokens;
        r.total_energy_j = tot_energy;
        r.qos_violation_rate = (double)violations / n;
        r.mean_throughput_tps = sum_tps / n;
        r.tokens_per_joule = tot_energy > 0.0 ? tot_tokens / tot_energy : 0.0;
        r.power_tracking_mae_w = tracked > 0 ? track_abs / (double)tracked : 0.0;
        r.throughput_target_tps = target;
        r.final_bias = bias;
        r.arrival_stream_hash = 0;  // host fills
        // = cum[n_int]: no request spawns after the last interval, and cum[n_int - 1] lies
        // in a chunk this warp has waited for (cum[n_int] may lie in the next one)
        r.n_requests = __ldcg(N.cum + (int64_t)(S.n_int - 1) * N.cum_stride);
        r.n_completed = completed;
        r.n_applied = n_applied;
        r.final_idx = cur;
        a.node_out[gi] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // RunSummary aggregate in node order (metrics.hpp:56-75)
        pals_sim_result o;
        memset(&o, 0, sizeof o);
        double worst = 0.0;
        for (int i = 0; i < S.n_nodes; ++i) {
            const pals_sim_node_result& r = a.node_out[S.node0 + i];
            o.total_tokens += r.total_tokens;
            o.total_energy_j += r.total_energy_j;
            o.mean_throughput_tps += r.mean_throughput_tps;
            worst = smax(worst, r.qos_violation_rate);
        }
        o.tokens_per_joule = o.total_energy_j > 0.0 ? o.total_tokens / o.total_energy_j : 0.0;
        o.qos_violation_rate = worst;
        if (S.budget_active && S.n_nodes > 0) {
            o.cluster_tracking_mae_w = sh_counted ? sh_cluster_abs / (double)sh_counted : 0.0;
            o.power_tracking_mae_w = o.cluster_tracking_mae_w;
        }
        o.sim_total_energy_j = sh_energy;
        o.n_intervals = S.n_int;
        o.n_budget_changes = S.n_changes;
        a.out[sid] = o;
    }
}

// ---- host setup ----------------------------------------------------------------
struct SelSet {  // select tables for one (scorer, candidates, degrees)
    pals_grid* g = nullptr;
    pals_plan* pl = nullptr;
    ReplayModelDev* d_m = nullptr;
    void* d_tables = nullptr;
    std::vector<pals_point> pts;
    bool built = false;
    void release() {
        if (pl) pals_plan_destroy(pl);
        if (g) pals_grid_destroy(g);
        if (d_m) cudaFree(d_m);
        if (d_tables) cudaFree(d_tables);
        pl = nullptr;
        g = nullptr;
        d_m = nullptr;
        d_tables = nullptr;
        built = false;
    }
};

// Kept by the context across pals_run_scenarios calls: the plant models (one per distinct
// (profile, GPU spec)) and every select-table set, keyed by its scorer's uid (never reused,
// unlike its address), the candidates and the bytes of everything else it was built from
// (coefficients, plant model 0). A seed sweep rebuilds nothing, and no call pays the set
// destructions, whose cudaFree calls stalled calls by up to ~1 s. Freed with the context.
using SetKey = std::tuple<uint64_t, std::string, std::vector<std::tuple<double, int, int, int, int>>>;
struct SimCache {
    std::map<std::string, pals_model*> plants;
    std::map<SetKey, SelSet*> sets;
};

}  // namespace

void sim_cache_free(pals_ctx* ctx) {
    if (!ctx || !ctx->sim_cache) return;
    SimCache* c = (SimCache*)ctx->sim_cache;
    for (auto& kv : c->sets) {
        kv.second->release();
        delete kv.second;
    }
    for (auto& kv : c->plants) pals_model_destroy(kv.second);
    delete c;
    ctx->sim_cache = nullptr;
}

namespace {

SimCache& sim_cache_of(pals_ctx* ctx) {
    if (!ctx->sim_cache) ctx->sim_cache = new SimCache;
    return *(SimCache*)ctx->sim_cache;
}

template <class T>
std::string raw_bytes(const T& v) {
    return std::string(reinterpret_cast<const char*>(&v), sizeof v);
}

struct Resources {
    pals_ctx* ctx;
    std::vector<SelSet*> sets;               // owned by the context's SimCache
    std::vector<pals_model*> plant_models;   // likewise
    std::vector<void*> dev;
    ~Resources() {
        static const bool verbose = getenv("PALS_SIM_VERBOSE") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        auto mark = [&](const char* what) {
            if (verbose)
                fprintf(stderr, "[pals_run_scenarios]   release %-8s %.3f s\n", what,
                        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
                            .count());
        };
        cudaStreamSynchronize(ctx->stream);
        mark("sync");
        for (void* p : dev) cudaFreeAsync(p, ctx->stream);
        mark("pool");
    }
    // staged arena: every per-scenario / per-node array is packed into one device
    // allocation (thousands of small cudaMalloc / cudaFree calls would dominate the call
    // otherwise). Data segments are gathered by all host threads into pinned memory kept in
    // the context and moved with one async copy; scratch (zero) regions live in a second
    // range that is memset on the device. Offsets of the zero range carry kZeroBit.
    static constexpr size_t kZeroBit = (size_t)1 << 62;
    struct Seg {
        const void* src;         // caller-owned (stage_ref) or own.data()
        std::vector<char> own;   // copied data (stage)
        size_t bytes, off;
    };
    std::vector<Seg> segs;
    size_t data_bytes = 0, zero_bytes = 0;
    char* arena = nullptr;
    char* zarena = nullptr;
    template <class T>
    size_t stage(const T* data, size_t n) {
        const size_t bytes = std::max<size_t>(1, n) * sizeof(T);
        if (!data) {  // scratch: zeroed on the device
            const size_t off = (zero_bytes + 255) & ~(size_t)255;
            zero_bytes = off + bytes;
            return off | kZeroBit;
        }
        const size_t off = (data_bytes + 255) & ~(size_t)255;
        data_bytes = off + bytes;
        Seg sg{nullptr, std::vector<char>((const char*)data, (const char*)data + n * sizeof(T)),
               n * sizeof(T), off};
        segs.push_back(std::move(sg));
        return off;
    }
    template <class T>
    size_t stage(const std::vector<T>& v) { return stage(v.data(), v.size()); }
    // staged without a copy: v must outlive commit()
    template <class T>
    size_t stage_ref(const std::vector<T>& v) {
        const size_t off = (data_bytes + 255) & ~(size_t)255;
        data_bytes = off + std::max<size_t>(1, v.size()) * sizeof(T);
        segs.push_back(Seg{v.data(), {}, v.size() * sizeof(T), off});
        return off;
    }
    int commit() {
        // the staged-input arena is kept by the context (a cudaMalloc / cudaFree of a few
        // hundred MB per call was a visible share of the call's host time)
        const size_t need = std::max<size_t>(1, data_bytes);
        if (ctx->sim_arena_bytes < need) {
            if (ctx->d_sim_arena) cudaFree(ctx->d_sim_arena);
            ctx->d_sim_arena = nullptr;
            ctx->sim_arena_bytes = 0;
            const cudaError_t e = cudaMalloc(&ctx->d_sim_arena, need);
            if (e != cudaSuccess) return cuda_fail(e, "pals_run_scenarios: cudaMalloc");
            ctx->sim_arena_bytes = need;
        }
        arena = (char*)ctx->d_sim_arena;
        int r = alloc(&zarena, zero_bytes);
        if (r) return r;
        cudaStream_t s = ctx->stream;
        PALS_CUDA(cudaMemsetAsync(zarena, 0, std::max<size_t>(1, zero_bytes), s));
        PALS_CUDA(cudaStreamSynchronize(s));  // the pinned buffer may still feed a copy
        if (ctx->pinned_bytes < data_bytes) {
            if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
            ctx->h_pinned = nullptr;
            ctx->pinned_bytes = 0;
            PALS_CUDA(cudaHostAlloc(&ctx->h_pinned, data_bytes, cudaHostAllocDefault));
            ctx->pinned_bytes = data_bytes;
        }
        char* pin = (char*)ctx->h_pinned;
        const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
        std::atomic<size_t> next{0};
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; ++t)
            th.emplace_back([&] {
                for (size_t i = next++; i < segs.size(); i = next++) {
                    const Seg& g = segs[i];
                    if (g.bytes)
                        std::memcpy(pin + g.off, g.own.empty() ? g.src : g.own.data(), g.bytes);
                }
            });
        for (auto& t : th) t.join();
        PALS_CUDA(cudaMemcpyAsync(arena, pin, std::max<size_t>(1, data_bytes),
                                  cudaMemcpyHostToDevice, s));
        PALS_CUDA(cudaStreamSynchronize(s));
        segs.clear();
        return PALS_OK;
    }
    template <class T>
    T* at(size_t off) const {
        return (T*)((off & kZeroBit) ? zarena + (off & ~kZeroBit) : arena + off);
    }
    template <class T>
    int alloc(T** p, size_t n) {
        // stream-ordered pool allocations: the call's per-call buffers (the zeroed running
        // lists alone are ~100 MB at 256 seeds) come back from the device's pool, kept across
        // calls, instead of cudaMalloc / cudaFree, whose device syncs and unmaps stalled
        // some calls by 0.2-0.8 s
        static thread_local int pool_dev = -1;
        if (pool_dev != ctx->device) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
                uint64_t keep = ~0ull;
                (void)cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            (void)cudaGetLastError();
            pool_dev = ctx->device;
        }
        void* q = nullptr;
        const cudaError_t e =
            cudaMallocAsync(&q, std::max<size_t>(1, n) * sizeof(T), ctx->stream);
        if (e != cudaSuccess) return cuda_fail(e, "pals_run_scenarios: cudaMalloc");
        dev.push_back(q);
        *p = (T*)q;
        return PALS_OK;
    }
    template <class T>
    int upload(T** p, const std::vector<T>& v) {
        int r = alloc(p, v.size());
        if (r) return r;
        if (!v.empty()) {
            const cudaError_t e = copy_on(ctx->stream, *p, v.data(), v.size() * sizeof(T),
                                          cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return cuda_fail(e, "pals_run_scenarios: upload");
        }
        return PALS_OK;
    }
};

// Candidates of a node under the scenario's policy (build_candidates, sim.hpp:293-308).
std::vector<pals_point> policy_candidates(const pals_scenario& sc, const pals_sim_node& n) {
    std::vector<double> caps(sc.cand_caps, sc.cand_caps + sc.n_caps);
    std::vector<int> batches(sc.cand_batches, sc.cand_batches + sc.n_batches);
    const int max_batch = *std::max_element(batches.begin(), batches.end());
    const double max_cap = *std::max_element(caps.begin(), caps.end());
    if (sc.policy == PALS_POLICY_ADAPTIVE_BATCH) caps = {max_cap};
    if (sc.policy == PALS_POLICY_ADAPTIVE_CAP) batches = {max_batch};
    if (sc.policy == PALS_POLICY_FIXED) {
        caps = {max_cap};
        batches = {max_batch};
    }
    std::vector<pals_point> out;
    for (double c : caps)
        for (int b : batches) out.push_back(pals_point{c, b, n.tp, n.ep, n.dp});
    return out;
}

int validate_scenario(const pals_scenario& sc, int n_models) {  // Scenario::validate
    if (sc.duration_s <= 0 || sc.interval_s <= 0) return set_error(PALS_ECONFIG, "scenario: bad duration");
    if (sc.n_nodes <= 0 || !sc.nodes) return set_error(PALS_ECONFIG, "scenario: no nodes");
    if (sc.n_caps <= 0 || sc.n_batches <= 0 || !sc.cand_caps || !sc.cand_batches)
        return set_error(PALS_ECONFIG, "scenario: empty candidate grid");
    for (int i = 0; i < sc.n_nodes; ++i) {
        const pals_sim_node& n = sc.nodes[i];
        if (n.arrival_rate_per_s < 0) return set_error(PALS_ECONFIG, "scenario: negative arrival rate");
        if (n.qos_fraction <= 0 || n.qos_fraction > 1)
            return set_error(PALS_ECONFIG, "scenario: qos_fraction must be in (0,1]");
        if (n.model < 0 || n.model >= n_models)
            return set_error(PALS_ECONFIG, "pals_run_scenarios: node model out of range");
        if (n.dp < 1 || n.dp > kMaxDp || n.tp < 1 || n.ep < 1)
            return set_error(PALS_ECONFIG, "OperatingPoint: batch and parallel degrees must be >= 1");
    }
    if (sc.n_nodes > PALS_SIM_MAX_NODES)
        return set_error(PALS_ECONFIG, "pals_run_scenarios: at most 32 nodes per scenario");
    if (sc.n_trace > 0 && (!sc.trace_t || !sc.trace_w))
        return set_error(PALS_ECONFIG, "pals_run_scenarios: null budget trace");
    for (int i = 1; i < sc.n_trace; ++i)
        if (sc.trace_t[i] <= sc.trace_t[i - 1])
            return set_error(PALS_EDATA, "budget trace timestamps must be strictly increasing");
    if (sc.policy < PALS_POLICY_FIXED || sc.policy > PALS_POLICY_ORACLE)
        return set_error(PALS_ECONFIG, "unknown policy");
    if (sc.objective != PALS_OBJ_QOS && sc.objective != PALS_OBJ_BUDGET)
        return set_error(PALS_ECONFIG, "unknown objective");
    return PALS_OK;
}

}  // namespace
}  // namespace pals

using namespace pals;

extern "C" int pals_run_scenarios(pals_ctx* ctx, int32_t n_scen, const pals_scenario* scens,
                                  int32_t n_models, const pals_profile* profiles,
                                  pals_model* const* predictors, const pals_gpu_spec* gpu,
                                  const pals_coeffs* coeffs, pals_sim_node_result* node_results,
                                  pals_sim_result* results, int64_t log_stride,
                                  pals_sim_telemetry* telemetry, pals_sim_decision* decisions) {
    if (!ctx || !scens || !profiles || !gpu || !coeffs || !node_results || !results || n_models <= 0)
        return set_error(PALS_ECONFIG, "pals_run_scenarios: null argument");
    if (n_scen <= 0) return PALS_OK;
    PALS_CUDA(cudaSetDevice(ctx->device));
    const auto t_start = std::chrono::steady_clock::now();
    ctx->sim_kernel_ms = -1.0;
    static const bool verbose = getenv("PALS_SIM_VERBOSE") != nullptr;
    auto phase = [&](const char* what) {
        if (verbose)
            fprintf(stderr, "[pals_run_scenarios] %-12s %.3f s\n", what,
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start)
                        .count());
    };
    struct PhaseEnd {  // reports after every resource of the call is released
        decltype(phase)& ph;
        ~PhaseEnd() { ph("released"); }
    } phase_end{phase};
    Resources res{ctx};
    // plant models (analytic, one per profile): device Analytic + the oracle's scorer
    SimCache& cache = sim_cache_of(ctx);
    for (int m = 0; m < n_models; ++m) {
        const std::string key = raw_bytes(profiles[m]) + raw_bytes(*gpu);
        auto it = cache.plants.find(key);
        if (it == cache.plants.end()) {
            pals_model* pm = nullptr;
            int r = pals_model_analytic(ctx, &profiles[m], gpu, &pm);
            if (r) return r;
            it = cache.plants.emplace(key, pm).first;
        }
        res.plant_models.push_back(it->second);
    }
    // what a select set is built from besides its scorer and candidates
    const std::string set_env =
        raw_bytes(*coeffs) + raw_bytes(profiles[0]) + raw_bytes(*gpu);
    Analytic* d_plant = nullptr;
    {
        std::vector<Analytic> h;
        for (auto* pm : res.plant_models) h.push_back(pm->an);
        int r = res.upload(&d_plant, h);
        if (r) return r;
    }
    int64_t total_nodes = 0, max_int = 0;
    int max_nodes = 1;
    std::vector<int> n_int(n_scen);
    for (int s = 0; s < n_scen; ++s) {
        const pals_scenario& sc = scens[s];
        int r = validate_scenario(sc, n_models);
        if (r) return r;
        const double ni = std::llround(sc.duration_s / sc.interval_s);  // sim.hpp:224
        n_int[s] = (int)ni;
        if (n_int[s] < 1)  // summarize() would throw on the empty log (metrics.hpp:27)
            return set_error(PALS_EDATA, "summarize: empty telemetry log");
        max_int = std::max<int64_t>(max_int, n_int[s]);
        max_nodes = std::max(max_nodes, sc.n_nodes);
        total_nodes += sc.n_nodes;
        const bool needs_pred = sc.policy == PALS_POLICY_JOINT ||
                                sc.policy == PALS_POLICY_ADAPTIVE_BATCH ||
                                sc.policy == PALS_POLICY_ADAPTIVE_CAP;
        for (int i = 0; i < sc.n_nodes && needs_pred; ++i)
            if (!predictors || !predictors[sc.nodes[i].model])
                return set_error(PALS_ECONFIG, "policy requires a trained predictor");
    }
    if ((telemetry || decisions) && log_stride < max_int)
        return set_error(PALS_ECONFIG, "pals_run_scenarios: log_stride below the interval count");

    // node scorers, candidates, targets; select tables deduplicated by (scorer, points)
    std::map<std::pair<const pals_model*, std::vector<std::tuple<double, int, int, int, int>>>, int>
        set_of;
    std::vector<int> node_set(total_nodes), node_init(total_nodes);
    std::vector<const pals_model*> node_scorer(total_nodes);
    std::vector<double> node_target(total_nodes);
    std::map<std::pair<const pals_model*, std::vector<double>>, std::pair<int, int>> node_memo;
    {
        int64_t gi = 0;
        for (int s = 0; s < n_scen; ++s) {
            const pals_scenario& sc = scens[s];
            const double mc = *std::max_element(sc.cand_caps, sc.cand_caps + sc.n_caps);
            const int mb = *std::max_element(sc.cand_batches, sc.cand_batches + sc.n_batches);
            for (int i = 0; i < sc.n_nodes; ++i, ++gi) {
                const pals_sim_node& n = sc.nodes[i];
                const pals_model* plant = res.plant_models[n.model];
                // unconstrained_throughput (sim.hpp:258-264), validated as the reference does
                const pals_point top{mc, mb, n.tp, n.ep, n.dp};
                int r = validate_point(plant, top);
                if (r) return r;
                const Score st = analytic_score(plant->an, mc, mb, n.tp, n.dp);
                node_target[gi] = n.qos_fraction * ((double)n.dp * st.T);
                const pals_model* scorer =
                    sc.policy == PALS_POLICY_ORACLE || !predictors || !predictors[n.model]
                        ? plant : predictors[n.model];
                node_scorer[gi] = scorer;
                // the node's (select set, initial candidate) is a function of the scorer, the
                // policy, the candidate axes, the parallel degrees and the initial knobs: memoised
                // on those (a few dozen numbers) instead of the expanded grid (up to 1,464
                // candidates per node, thousands of nodes per call)
                std::vector<double> tk;
                tk.reserve(8 + sc.n_caps + sc.n_batches);
                tk.push_back((double)sc.policy);
                tk.push_back((double)n.tp);
                tk.push_back((double)n.ep);
                tk.push_back((double)n.dp);
                tk.push_back(sc.initial_cap_w);
                tk.push_back((double)sc.initial_batch);
                tk.push_back((double)sc.n_caps);
                tk.insert(tk.end(), sc.cand_caps, sc.cand_caps + sc.n_caps);
                for (int b = 0; b < sc.n_batches; ++b) tk.push_back((double)sc.cand_batches[b]);
                auto memo = node_memo.find({scorer, tk});
                if (memo != node_memo.end()) {
                    node_set[gi] = memo->second.first;
                    node_init[gi] = memo->second.second;
                    continue;
                }
                std::vector<pals_point> pts = policy_candidates(sc, n);
                std::vector<std::tuple<double, int, int, int, int>> key;
                for (auto& p : pts) key.emplace_back(p.cap_watts, p.batch, p.tp, p.ep, p.dp);
                int init = -1;
                for (size_t c = 0; c < pts.size() && init < 0; ++c)
                    if (pts[c].cap_watts == sc.initial_cap_w && pts[c].batch == sc.initial_batch)
                        init = (int)c;
                if (init < 0)
                    return set_error(PALS_ECONFIG,
                                     "pals_run_scenarios: the initial (cap, batch) must be one "
                                     "of the policy's candidates");
                node_init[gi] = init;
                auto it = set_of.find({scorer, key});
                if (it == set_of.end()) {
                    it = set_of.emplace(std::make_pair(scorer, key), (int)res.sets.size()).first;
                    const SetKey ck{scorer->uid, set_env, key};
                    auto cit = cache.sets.find(ck);
                    if (cit == cache.sets.end()) {
                        SelSet* ns = new SelSet;
                        ns->pts = pts;
                        cit = cache.sets.emplace(ck, ns).first;
                    }
                    res.sets.push_back(cit->second);
                }
                node_set[gi] = it->second;
                node_memo.emplace(std::make_pair(scorer, std::move(tk)),
                                  std::make_pair(it->second, init));
            }
        }
    }
    phase("nodes");
    // build every select-table set: plan (scores + ranks) -> k_build_tables
    std::vector<int> set_scorer_model(res.sets.size(), -1);
    for (auto& [k, si] : set_of) {
        SelSet& S = *res.sets[si];
        if (S.built) continue;  // from an earlier call (SimCache)
        S.release();            // a build an earlier call failed to finish
        const pals_model* scorer = k.first;
        const int n = (int)S.pts.size();
        if (n > kMaxReplayCands)
            return set_error(PALS_ECONFIG, "pals_run_scenarios: at most 4096 candidates per node");
        int r = pals_grid_points(ctx, S.pts.data(), n, &S.g);
        if (r) return r;
        r = validate_points(scorer, S.g->h_pts, S.g->n);
        if (r) return r;
        r = pals_plan_create(ctx, scorer, S.g, coeffs, &S.pl);
        if (r) return r;
        r = pals_plan_prepare(S.pl);
        if (r) return r;
        const PlanDev& d = plan_dev(S.pl);
        const size_t W = (size_t)n + 1;
        PALS_CUDA(cudaMalloc(&S.d_tables, W * W * 4 + W * 4 + 2 * W * 8 + 1024));
        PALS_CUDA(cudaMalloc(&S.d_m, sizeof(ReplayModelDev)));
        ReplayModelDev m;
        memset(&m, 0, sizeof m);
        m.n = n;
        m.tp = S.pts[0].tp;
        m.ep = S.pts[0].ep;
        m.dp = S.pts[0].dp;
        m.max_cap = S.pts[0].cap_watts;
        m.max_batch = S.pts[0].batch;
        for (auto& p : S.pts) {
            m.max_cap = smax(m.max_cap, p.cap_watts);
            m.max_batch = std::max(m.max_batch, p.batch);
        }
        m.cap = S.g->cap;
        m.batch = S.g->batch;
        m.canon = S.g->canon;
        m.inv_tr = S.g->inv_tr;
        m.T = d.T;
        m.th = d.th;
        m.pn = d.pn;
        m.ef = d.ef;
        m.danger_t = d.danger[ORD_T];
        m.danger_e = d.danger[ORD_E];
        char* base = (char*)S.d_tables;
        m.m2 = (const uint32_t*)base;
        m.b1 = (const uint32_t*)(base + W * W * 4);
        m.ut = (const double*)(base + ((W * W * 4 + W * 4 + 7) & ~(size_t)7));
        m.up = m.ut + W;
        // k_build_tables also derives plant constants from m.plant: any node of the
        // set shares the profile-independent parts used here; point it at model 0 (only
        // k_build_tables reads it: the cached set keeps a pointer of this call, unused later)
        m.plant = d_plant;
        PALS_CUDA(copy_on(ctx->stream, S.d_m, &m, sizeof m, cudaMemcpyHostToDevice));
        k_build_tables<<<1, 1024, 0, ctx->stream>>>(d, S.d_m, (uint32_t*)m.m2, (uint32_t*)m.b1,
                                                     (double*)m.ut, (double*)m.up, coeffs->alpha,
                                                     coeffs->beta_watts);
        count_launch(ctx);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "k_build_tables");
        S.built = true;
    }

    phase("tables");
    // arrival streams on all host threads: one per distinct (seed, node slot, rate,
    // backlog, length law, interval grid) — a baseline suite's policies share them
    std::vector<int64_t> node0(n_scen + 1, 0);
    for (int s = 0; s < n_scen; ++s) node0[s + 1] = node0[s] + scens[s].n_nodes;
    std::vector<int> node_stream(total_nodes);
    std::vector<std::pair<int, int>> work;  // (scenario, node) generating each stream
    // CTA order: most node-intervals first, so the long scenarios do not form the tail
    std::vector<int32_t> order(n_scen);
    for (int s = 0; s < n_scen; ++s) order[s] = s;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        return (int64_t)n_int[x] * scens[x].n_nodes > (int64_t)n_int[y] * scens[y].n_nodes;
    });
    // CTA groups: G equal runs of the CTA order. Streams are drawn and published group by
    // group (each group in interval chunks), so the first CTAs to run wait for the draws of
    // a quarter of the streams, not of all of them; a stream belongs to the first group
    // that reads it
    const int n_groups = std::max(1, std::min(kSimGroups, n_scen));
    std::vector<int> scen_group(n_scen);
    for (int pos = 0; pos < n_scen; ++pos)
        scen_group[order[pos]] = (int)((int64_t)pos * n_groups / n_scen);
    std::vector<int> stream_group;
    {
        using Key = std::tuple<uint64_t, int, double, int, double, double, double, int>;
        std::map<Key, int> seen;
        for (int s = 0; s < n_scen; ++s)
            for (int i = 0; i < scens[s].n_nodes; ++i) {
                const pals_scenario& sc = scens[s];
                const Key key{sc.seed, i, sc.nodes[i].arrival_rate_per_s,
                              sc.nodes[i].initial_backlog, sc.mean_tokens, sc.log_sigma,
                              sc.interval_s, n_int[s]};
                auto it = seen.find(key);
                if (it == seen.end()) {
                    it = seen.emplace(key, (int)work.size()).first;
                    work.emplace_back(s, i);
                    stream_group.push_back(scen_group[s]);
                }
                node_stream[node0[s] + i] = it->second;
                stream_group[it->second] = std::min(stream_group[it->second], scen_group[s]);
            }
    }
    // streams renumbered group by group: a group's count columns are one contiguous range
    std::vector<int> gcol(n_groups + 1, 0);
    {
        std::vector<int> perm(work.size()), inv(work.size());
        for (size_t u = 0; u < work.size(); ++u) perm[u] = (int)u;
        std::stable_sort(perm.begin(), perm.end(),
                         [&](int x, int y) { return stream_group[x] < stream_group[y]; });
        std::vector<std::pair<int, int>> w2(work.size());
        for (size_t v = 0; v < perm.size(); ++v) {
            w2[v] = work[perm[v]];
            inv[perm[v]] = (int)v;
            ++gcol[stream_group[perm[v]] + 1];
        }
        work.swap(w2);
        for (auto& x : node_stream) x = inv[x];
        for (int g = 0; g < n_groups; ++g) gcol[g + 1] += gcol[g];
    }
    // Streamed arrivals. Each stream has a fixed region (cum, then len up to a capacity
    // bound) in one pinned buffer mirrored by one device buffer, so the node descriptors
    // point at device addresses known before any draw. The streams are generated in C
    // chunks of intervals (every stream's intervals [c K, (c + 1) K) per chunk, each stream
    // by one worker so its draws stay in order); every finished chunk is copied up and
    // flagged in mapped memory, and k_sim, launched after chunk 0, waits per chunk for its
    // flag — the simulation runs while the host still draws later intervals.
    // layout: the counts interval-major (row k = every stream's cum[k], so a chunk's counts
    // are one copy), then every stream's lengths
    const size_t n_streams = work.size();
    std::vector<size_t> s_oc(n_streams), s_ol(n_streams);
    std::vector<int64_t> s_cap(n_streams);
    int max_n_int = 1;
    for (size_t u = 0; u < n_streams; ++u) max_n_int = std::max(max_n_int, n_int[work[u].first]);
    size_t s_elems = (((size_t)max_n_int + 1) * n_streams + 31) & ~(size_t)31;
    for (size_t u = 0; u < n_streams; ++u) {
        const pals_scenario& sc = scens[work[u].first];
        const pals_sim_node& nd = sc.nodes[work[u].second];
        const int ni = n_int[work[u].first];
        const double mean = std::max(0.0, nd.arrival_rate_per_s * sc.interval_s) * ni;
        s_cap[u] = (int64_t)nd.initial_backlog +
                   (int64_t)std::ceil(mean + 12.0 * std::sqrt(mean + 1.0)) + 1024;
        s_oc[u] = u;  // column u of the count rows
        s_ol[u] = s_elems;
        s_elems += ((size_t)s_cap[u] + 31) & ~(size_t)31;
    }
    const int64_t cstride = (int64_t)n_streams;
    const size_t s_bytes = std::max<size_t>(1, s_elems) * 4;
    if (ctx->sim_stream_bytes < s_bytes) {
        if (ctx->h_sim_streams) cudaFreeHost(ctx->h_sim_streams);
        if (ctx->d_sim_streams) cudaFree(ctx->d_sim_streams);
        ctx->h_sim_streams = ctx->d_sim_streams = nullptr;
        ctx->sim_stream_bytes = 0;
        PALS_CUDA(cudaHostAlloc(&ctx->h_sim_streams, s_bytes, cudaHostAllocDefault));
        PALS_CUDA(cudaMalloc(&ctx->d_sim_streams, s_bytes));
        ctx->sim_stream_bytes = s_bytes;
    }
    int32_t* const hbuf = (int32_t*)ctx->h_sim_streams;
    int32_t* const dbuf = (int32_t*)ctx->d_sim_streams;
    constexpr int kSimChunks = 8;
    const int chunk_k = (max_n_int + kSimChunks - 1) / kSimChunks;
    std::vector<StreamGen> gens(n_streams);
    for (size_t u = 0; u < n_streams; ++u)
        gens[u].init(scens[work[u].first], work[u].second, n_int[work[u].first], hbuf + s_oc[u],
                     cstride, hbuf + s_ol[u], s_cap[u]);
    // [chunk][stream]: the stream's request count after the chunk (its len range is
    // [count after chunk c - 1, count after chunk c))
    std::vector<int64_t> s_after((size_t)kSimChunks * n_streams, 0);
    const int n_pub = n_groups * kSimChunks;  // publications (group, chunk), group-major
    std::vector<std::atomic<int>> chunk_done(n_pub);
    for (auto& x : chunk_done) x = 0;
    std::atomic<bool> stop_workers{false};
    std::vector<std::thread> stream_threads;
    unsigned n_workers = 1;
    {
        // one core stays with this thread: it splits the budgets on the GPU meanwhile and
        // then feeds the copies, and its CUDA calls lost the CPU to the workers otherwise
        const unsigned hc = std::thread::hardware_concurrency();
        n_workers = std::max(1u, std::min<unsigned>(hc > 1 ? hc - 1 : 1, (unsigned)n_streams));
        for (unsigned t = 0; t < n_workers; ++t)
            stream_threads.emplace_back([&, t] {
                for (int i = 0; i < n_pub && !stop_workers; ++i) {
                    const int gr = i / kSimChunks, c = i % kSimChunks;
                    for (size_t u = gcol[gr] + t; u < (size_t)gcol[gr + 1]; u += n_workers) {
                        StreamGen& g = gens[u];
                        const int k0 = c * chunk_k, k1 = std::min(g.n_int, (c + 1) * chunk_k);
                        if (k0 < k1) g.run(k0, k1);
                        s_after[(size_t)c * n_streams + u] = g.count;
                    }
                    chunk_done[i].fetch_add(1, std::memory_order_release);
                }
            });
    }
    struct Joiner {
        std::vector<std::thread>& t;
        std::atomic<bool>& stop;
        ~Joiner() {
            stop = true;
            for (auto& x : t)
                if (x.joinable()) x.join();
        }
    } joiner{stream_threads, stop_workers};

    phase("streams started");
    // budget changes and their splits (assign_budgets, sim.hpp:229-238, 277-283, 313-336).
    // The change list and the per-interval tracking target are a function of the cluster
    // signal (trace or static budget), the interval and the interval count, which a seed
    // sweep repeats in every scenario: computed and staged once per distinct signal.
    std::vector<int> sig(n_scen, -1);
    std::vector<std::vector<int32_t>> u_ck;
    std::vector<std::vector<double>> u_cw, u_tr;
    {
        using SigKey = std::tuple<const double*, const double*, int, double, int, double>;
        std::map<SigKey, int> sig_of;
        for (int s = 0; s < n_scen; ++s) {
            const pals_scenario& sc = scens[s];
            if (sc.n_trace <= 0 && !sc.has_cluster_budget) continue;
            const SigKey key = sc.n_trace > 0
                                   ? SigKey{sc.trace_t, sc.trace_w, sc.n_trace, sc.interval_s,
                                            n_int[s], 0.0}
                                   : SigKey{nullptr, nullptr, 0, sc.interval_s, n_int[s],
                                            sc.cluster_budget_w};
            auto it = sig_of.find(key);
            if (it != sig_of.end()) {
                sig[s] = it->second;
                continue;
            }
            const int id = (int)u_ck.size();
            sig_of.emplace(key, id);
            sig[s] = id;
            u_ck.emplace_back();
            u_cw.emplace_back();
            u_tr.emplace_back();
            std::vector<int32_t>& ck = u_ck.back();
            std::vector<double>& cw = u_cw.back();
            std::vector<double>& tr = u_tr.back();
            if (sc.n_trace > 0) {
                double last = -1.0;
                TraceCursor at_t0{sc}, at_t{sc};
                for (int k = 0; k < n_int[s]; ++k) {
                    const double wv = at_t0(k * sc.interval_s);
                    if (wv != last) {
                        ck.push_back(k);
                        cw.push_back(wv);
                        last = wv;
                    }
                }
                tr.resize(n_int[s]);
                for (int k = 0; k < n_int[s]; ++k) {
                    const double t1 = k * sc.interval_s + sc.interval_s;
                    tr[k] = at_t(t1 - sc.interval_s);
                }
            } else {
                ck.push_back(0);
                cw.push_back(sc.cluster_budget_w);
                tr.assign(n_int[s], sc.cluster_budget_w);
            }
        }
    }
    const std::vector<int32_t> no_ck;
    const std::vector<double> no_d;
    auto CK = [&](int s) -> const std::vector<int32_t>& { return sig[s] < 0 ? no_ck : u_ck[sig[s]]; };
    auto CW = [&](int s) -> const std::vector<double>& { return sig[s] < 0 ? no_d : u_cw[sig[s]]; };
    // node budgets per change: [scenario][change][node]
    std::vector<std::vector<double>> chg_b(n_scen);
    {
        // water-filling for joint / oracle scenarios, grouped by selection margin
        std::map<double, std::vector<int>> by_margin;
        for (int s = 0; s < n_scen; ++s) {
            const pals_scenario& sc = scens[s];
            chg_b[s].assign(CK(s).size() * sc.n_nodes, 0.0);
            if (CK(s).empty()) continue;
            if (sc.policy == PALS_POLICY_JOINT || sc.policy == PALS_POLICY_ORACLE) {
                by_margin[sc.controller.budget_margin].push_back(s);
            } else {
                int total_dp = 0;
                for (int i = 0; i < sc.n_nodes; ++i) total_dp += sc.nodes[i].dp;
                for (size_t c = 0; c < CK(s).size(); ++c)
                    for (int i = 0; i < sc.n_nodes; ++i)
                        chg_b[s][c * sc.n_nodes + i] =
                            CW(s)[c] * (double)sc.nodes[i].dp / total_dp;
            }
        }
        for (auto& [margin, ss] : by_margin) {
            // candidate sets = the nodes' (scorer, candidates) select sets
            std::map<int, int> aset;  // select set -> allocator set
            std::vector<pals_model*> set_models;
            std::vector<pals_point> pts;
            std::vector<int64_t> off{0};
            std::vector<int64_t> p_off{0};
            std::vector<int32_t> nmodel, ndp;
            std::vector<double> ntarget, cbudget;
            for (int s : ss) {
                const pals_scenario& sc = scens[s];
                int64_t g0 = 0;
                for (int q = 0; q < s; ++q) g0 += scens[q].n_nodes;
                for (size_t c = 0; c < CK(s).size(); ++c) {
                    for (int i = 0; i < sc.n_nodes; ++i) {
                        const int si = node_set[g0 + i];
                        auto it = aset.find(si);
                        if (it == aset.end()) {
                            it = aset.emplace(si, (int)set_models.size()).first;
                            set_models.push_back((pals_model*)node_scorer[g0 + i]);
                            pts.insert(pts.end(), res.sets[si]->pts.begin(), res.sets[si]->pts.end());
                            off.push_back((int64_t)pts.size());
                        }
                        nmodel.push_back(it->second);
                        ndp.push_back(sc.nodes[i].dp);
                        ntarget.push_back(sc.objective == PALS_OBJ_QOS ? node_target[g0 + i] : 0.0);
                    }
                    cbudget.push_back(CW(s)[c]);
                    p_off.push_back((int64_t)nmodel.size());
                }
            }
            phase("budget sets");
            pals_alloc* al = nullptr;
            int r = pals_alloc_create_sets(ctx, (int32_t)set_models.size(), set_models.data(),
                                           pts.data(), off.data(), gpu, coeffs, margin, &al);
            if (r) return r;
            const int64_t np = (int64_t)cbudget.size();
            std::vector<double> nb(nmodel.size()), tot(np);
            std::vector<uint8_t> sat(np);
            std::vector<int32_t> st(np);
            phase("alloc created");
            r = pals_allocate_budget(al, 25.0, np, p_off.data(), nmodel.data(), ndp.data(),
                                     ntarget.data(), cbudget.data(), nb.data(), tot.data(),
                                     sat.data(), st.data());
            phase("allocated");
            pals_alloc_destroy(al);
            phase("alloc freed");
            if (r) return r;
            for (int64_t p = 0; p < np; ++p)
                if (st[p] != PALS_OK)
                    return set_error(st[p], "allocate_budget: cluster budget split failed "
                                            "(as run_scenario would throw)");
            int64_t o = 0;
            for (int s : ss) {
                const pals_scenario& sc = scens[s];
                for (size_t c = 0; c < CK(s).size(); ++c)
                    for (int i = 0; i < sc.n_nodes; ++i) chg_b[s][c * sc.n_nodes + i] = nb[o++];
            }
        }
    }

    phase("budgets");
    // "@" + fmt_num(k * interval) per interval of every distinct grid (the arrival hash's
    // request suffixes, sim.hpp:344; csvio.hpp:17-21)
    std::map<std::pair<double, int>, int> grid_of;
    std::vector<std::vector<char>> g_chars;
    std::vector<std::vector<uint32_t>> g_off;
    std::vector<int> stream_grid(n_streams);
    for (size_t u = 0; u < n_streams; ++u) {
        const pals_scenario& sc = scens[work[u].first];
        const int ni = n_int[work[u].first];
        auto it = grid_of.find({sc.interval_s, ni});
        if (it == grid_of.end()) {
            it = grid_of.emplace(std::make_pair(sc.interval_s, ni), (int)g_chars.size()).first;
            std::vector<char> ch;
            std::vector<uint32_t> off{0};
            for (int k = 0; k < ni; ++k) {
                const std::string t = "@" + fmt10g(k * sc.interval_s);
                ch.insert(ch.end(), t.begin(), t.end());
                off.push_back((uint32_t)ch.size());
            }
            g_chars.push_back(std::move(ch));
            g_off.push_back(std::move(off));
        }
        stream_grid[u] = it->second;
    }
    std::vector<size_t> o_gch(g_chars.size()), o_goff(g_chars.size());
    for (size_t g = 0; g < g_chars.size(); ++g) {
        o_gch[g] = res.stage(g_chars[g]);
        o_goff[g] = res.stage(g_off[g]);
    }
    phase("streams");
    // device buffers: stage every array, one upload, then point the descriptors at it
    std::vector<SimScenDev> hs(n_scen);
    std::vector<SimNodeDev> hn(total_nodes);
    constexpr size_t kNoOff = ~(size_t)0;
    std::vector<size_t> u_off_ck(u_ck.size(), kNoOff), u_off_tr(u_ck.size(), kNoOff);
    std::vector<size_t> o_chg(n_scen), o_track(n_scen, 0), o_bud(total_nodes),
        o_run_len(total_nodes), o_run_gen(total_nodes), o_run_id(total_nodes),
        o_req_k(total_nodes), o_req_gen(total_nodes);
    const bool keep_req = ctx->sim_keep_requests != 0;
    size_t max_run = 0;
    {
        int64_t gi = 0;
        for (int s = 0; s < n_scen; ++s) {
            const pals_scenario& sc = scens[s];
            if (sig[s] >= 0) {  // staged once per distinct signal
                if (u_off_ck[sig[s]] == kNoOff) {
                    u_off_ck[sig[s]] = res.stage(u_ck[sig[s]]);
                    u_off_tr[sig[s]] = res.stage(u_tr[sig[s]]);
                }
                o_chg[s] = u_off_ck[sig[s]];
                o_track[s] = u_off_tr[sig[s]];
            } else {
                o_chg[s] = res.stage(no_ck);
            }
            const int mb = *std::max_element(sc.cand_batches, sc.cand_batches + sc.n_batches);
            for (int i = 0; i < sc.n_nodes; ++i, ++gi) {
                std::vector<double> nbud(CK(s).size());
                for (size_t c = 0; c < nbud.size(); ++c) nbud[c] = chg_b[s][c * sc.n_nodes + i];
                o_bud[gi] = res.stage(nbud);
                const size_t run_cap =
                    (size_t)std::max(mb, sc.initial_batch) * sc.nodes[i].dp + 32;
                max_run = std::max(max_run, run_cap);
                o_run_len[gi] = res.stage((const int32_t*)nullptr, run_cap);
                o_run_id[gi] = res.stage((const int32_t*)nullptr, run_cap);
                if (keep_req) {  // sized by the stream's capacity bound (drawn later)
                    const size_t nreq = (size_t)s_cap[node_stream[gi]];
                    o_req_k[gi] = res.stage((const int32_t*)nullptr, nreq);
                    o_req_gen[gi] = res.stage((const double*)nullptr, nreq);
                }
                o_run_gen[gi] = res.stage((const double*)nullptr, run_cap);
            }
        }
        phase("staged");
        int r = res.commit();
        if (r) return r;
        phase("committed");
        gi = 0;
        for (int s = 0; s < n_scen; ++s) {
            const pals_scenario& sc = scens[s];
            SimScenDev& S = hs[s];
            memset(&S, 0, sizeof S);
            S.node0 = (int)gi;
            S.n_nodes = sc.n_nodes;
            S.n_int = n_int[s];
            S.policy = sc.policy;
            S.objective = sc.objective;
            S.budget_active = sc.has_cluster_budget || sc.n_trace > 0;
            S.n_changes = (int)CK(s).size();
            S.interval_s = sc.interval_s;
            S.epsilon = sc.epsilon;
            S.cfg = sc.controller;
            S.change_k = res.at<int32_t>(o_chg[s]);
            S.track_target = sig[s] < 0 ? nullptr : res.at<double>(o_track[s]);
            for (int i = 0; i < sc.n_nodes; ++i, ++gi) {
                SimNodeDev& N = hn[gi];
                const pals_sim_node& n = sc.nodes[i];
                memset(&N, 0, sizeof N);
                N.sel = res.sets[node_set[gi]]->d_m;
                N.plant = d_plant + n.model;
                N.tp = n.tp;
                N.ep = n.ep;
                N.dp = n.dp;
                N.init_idx = node_init[gi];
                N.target_tps = node_target[gi];
                N.cum = dbuf + s_oc[node_stream[gi]];
                N.cum_stride = cstride;
                N.len = dbuf + s_ol[node_stream[gi]];
                N.run_len = res.at<int32_t>(o_run_len[gi]);
                N.run_id = res.at<int32_t>(o_run_id[gi]);
                N.req_k = keep_req ? res.at<int32_t>(o_req_k[gi]) : nullptr;
                N.req_gen = keep_req ? res.at<double>(o_req_gen[gi]) : nullptr;
                N.run_gen = res.at<double>(o_run_gen[gi]);
                N.budget = res.at<double>(o_bud[gi]);
            }
        }
    }
    // the arrival hashes, on a side stream beside k_sim
    std::vector<HashJob> jobs(n_streams);
    for (size_t u = 0; u < n_streams; ++u) {
        HashJob& j = jobs[u];
        j.len = dbuf + s_ol[u];
        j.cum = dbuf + s_oc[u];
        j.cstride = cstride;
        j.toff = res.at<uint32_t>(o_goff[stream_grid[u]]);
        j.tchars = res.at<char>(o_gch[stream_grid[u]]);
        j.n_int = n_int[work[u].first];
        j.backlog = scens[work[u].first].nodes[work[u].second].initial_backlog;
    }
    HashJob* d_jobs = nullptr;
    uint64_t* d_hash = nullptr;
    {
        int r = res.upload(&d_jobs, jobs);
        if (r) return r;
        r = res.alloc(&d_hash, jobs.size());
        if (r) return r;
    }
    cudaStream_t hs_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_hash = nullptr;
    {
        // the greatest priority: the arrival hashes (launched once the last chunk is up, while
        // k_sim's blocks hold the SMs) take the first free block slots instead of waiting
        // for k_sim's tail
        int lo = 0, hi = 0;
        PALS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        PALS_CUDA(cudaStreamCreateWithPriority(&hs_stream, cudaStreamNonBlocking, hi));
    }
    struct StreamGuard {
        cudaStream_t& s;
        cudaEvent_t& a;
        cudaEvent_t& b;
        ~StreamGuard() {
            if (s) cudaStreamSynchronize(s), cudaStreamDestroy(s);
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } hs_guard{hs_stream, ev_fork, ev_hash};
    PALS_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    PALS_CUDA(cudaEventCreateWithFlags(&ev_hash, cudaEventDisableTiming));
    // (the arrival hashes run on hs_stream after the last chunk's copies, below)
    SimArgs A;
    memset(&A, 0, sizeof A);
    int r = res.upload((int32_t**)&A.order, order);
    if (r) return r;
    r = res.upload((SimScenDev**)&A.scen, hs);
    if (r) return r;
    r = res.upload((SimNodeDev**)&A.nodes, hn);
    if (r) return r;
    A.alpha = coeffs->alpha;
    A.beta = coeffs->beta_watts;
    A.idle_w = gpu->idle_watts;
    A.min_cap = gpu->min_cap_watts;
    A.log_stride = log_stride;
    r = res.alloc(&A.node_out, total_nodes);
    if (r) return r;
    r = res.alloc(&A.out, n_scen);
    if (r) return r;
    const size_t nlog = (size_t)total_nodes * (size_t)std::max<int64_t>(log_stride, 0);
    if (telemetry) {
        r = res.alloc(&A.tel, nlog);
        if (r) return r;
    }
    if (decisions) {
        r = res.alloc(&A.dec, nlog);
        if (r) return r;
    }
    // per-chunk readiness flags in device memory (zeroed before the launch), raised by a
    // 4-byte copy queued behind the chunk's data copies: k_sim polls L2, not the PCIe bus
    // (polling mapped host memory from every warp starved the copies themselves)
    int* d_flags = nullptr;
    {
        int r = res.alloc(&d_flags, n_pub);
        if (r) return r;
    }
    if (!ctx->h_sim_flags) {  // pinned source of the flag value (1)
        PALS_CUDA(cudaHostAlloc((void**)&ctx->h_sim_flags, 64 * sizeof(int), cudaHostAllocDefault));
        for (int c = 0; c < 64; ++c) ctx->h_sim_flags[c] = 1;
    }
    PALS_CUDA(cudaMemsetAsync(d_flags, 0, n_pub * sizeof(int), ctx->stream));
    A.flags = d_flags;
    A.chunk_k = chunk_k;
    A.n_chunks = kSimChunks;
    A.n_groups = n_groups;
    PALS_CUDA(cudaStreamSynchronize(ctx->stream));
    phase("upload");
    // whatever happens below, every chunk flag is raised before this function returns, so a
    // launched k_sim never waits for a chunk that will not come
    struct FlagGuard {
        pals_ctx* c;
        int* f;
        int n;
        cudaStream_t& s;
        ~FlagGuard() {
            cudaMemcpyAsync(f, c->h_sim_flags, n * sizeof(int), cudaMemcpyHostToDevice, s);
            cudaStreamSynchronize(s);
            cudaStreamSynchronize(c->stream);
        }
    } flag_guard{ctx, d_flags, n_pub, hs_stream};
    // publication i = (group, chunk c): wait for its draws, copy the group's streams' new
    // parts up on hs_stream, then raise its flag once the copies have landed (stream order)
    auto publish = [&](int i) -> int {
        while (chunk_done[i].load(std::memory_order_acquire) < (int)n_workers)
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        const int gr = i / kSimChunks, c = i % kSimChunks;
        for (size_t u = gcol[gr]; u < (size_t)gcol[gr + 1]; ++u) {
            const int ni = gens[u].n_int;
            const int64_t l0 = c ? std::min(s_cap[u], s_after[(size_t)(c - 1) * n_streams + u]) : 0;
            const int64_t l1 = std::min(s_cap[u], s_after[(size_t)c * n_streams + u]);
            if (l1 > l0)
                PALS_CUDA(cudaMemcpyAsync(dbuf + s_ol[u] + l0, hbuf + s_ol[u] + l0,
                                          (size_t)(l1 - l0) * 4, cudaMemcpyHostToDevice,
                                          hs_stream));
            (void)ni;
        }
        {  // the chunk's count rows (the last chunk also the final row, cum[n_int])
            const int k0 = c * chunk_k;
            const int k1 =
                c == kSimChunks - 1 ? max_n_int + 1 : std::min(max_n_int + 1, (c + 1) * chunk_k);
            const size_t ncol = (size_t)(gcol[gr + 1] - gcol[gr]);
            if (k1 > k0 && ncol)  // the group's columns of those rows
                PALS_CUDA(cudaMemcpy2DAsync(dbuf + (size_t)k0 * n_streams + gcol[gr], n_streams * 4,
                                            hbuf + (size_t)k0 * n_streams + gcol[gr], n_streams * 4,
                                            ncol * 4, (size_t)(k1 - k0), cudaMemcpyHostToDevice,
                                            hs_stream));
        }
        PALS_CUDA(cudaMemcpyAsync(d_flags + i, ctx->h_sim_flags, sizeof(int),
                                  cudaMemcpyHostToDevice, hs_stream));
        return PALS_OK;
    };
    // streamed: launch after chunk 0; otherwise (profiling) after every chunk
    const int pre = ctx->sim_streaming ? 1 : n_pub;
    for (int c = 0; c < pre; ++c) {
        const int pr = publish(c);
        if (pr) return pr;
    }
    ctx->sim_prep_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    cudaEvent_t ev0, ev1;
    PALS_CUDA(cudaEventCreate(&ev0));
    PALS_CUDA(cudaEventCreate(&ev1));
    cudaEventRecord(ev0, ctx->stream);
    const size_t smem = (size_t)max_nodes * max_run * (sizeof(double) + 2 * sizeof(int32_t));
    A.smem_run = smem <= 160 * 1024 ? (int)max_run : 0;
    if (A.smem_run)
        PALS_CUDA(cudaFuncSetAttribute(k_sim, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    k_sim<<<n_scen, 32 * max_nodes, A.smem_run ? smem : 0, ctx->stream>>>(A);
    count_launch(ctx);
    cudaError_t e = cudaGetLastError();
    cudaEventRecord(ev1, ctx->stream);
    for (int c = pre; c < n_pub && e == cudaSuccess; ++c) {
        const int pr = publish(c);
        if (pr) return pr;
    }
    phase("published");
    for (auto& t : stream_threads) t.join();
    for (size_t u = 0; u < n_streams; ++u)
        if (gens[u].overflow)
            return set_error(PALS_EDATA, "pals_run_scenarios: an arrival stream exceeded its "
                                         "capacity bound (mean + 12 sigma)");
    if (!jobs.empty()) {  // after every chunk's copies (hs_stream order)
        k_arrival_hash<<<(unsigned)((jobs.size() + 63) / 64), 64, 0, hs_stream>>>(
            d_jobs, (int)jobs.size(), d_hash);
        count_launch(ctx);
        const cudaError_t he = cudaGetLastError();
        if (he != cudaSuccess) return cuda_fail(he, "k_arrival_hash");
    }
    PALS_CUDA(cudaEventRecord(ev_hash, hs_stream));

    if (e == cudaSuccess) e = cudaEventSynchronize(ev1);
    float kms = -1.0f;
    if (e == cudaSuccess) cudaEventElapsedTime(&kms, ev0, ev1);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    ctx->sim_kernel_ms = kms;
    if (e != cudaSuccess) return cuda_fail(e, "k_sim");
    phase("kernel");
    e = copy_on(ctx->stream, node_results, A.node_out, sizeof(pals_sim_node_result) * total_nodes,
                cudaMemcpyDeviceToHost);
    if (e == cudaSuccess)
        e = copy_on(ctx->stream, results, A.out, sizeof(pals_sim_result) * n_scen,
                    cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && telemetry)
        e = copy_on(ctx->stream, telemetry, A.tel, sizeof(pals_sim_telemetry) * nlog,
                    cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && decisions)
        e = copy_on(ctx->stream, decisions, A.dec, sizeof(pals_sim_decision) * nlog,
                    cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "pals_run_scenarios");
    std::vector<uint64_t> hashes(jobs.size());
    e = cudaStreamWaitEvent(ctx->stream, ev_hash, 0);
    if (e == cudaSuccess && !jobs.empty())
        e = copy_on(ctx->stream, hashes.data(), d_hash, 8 * jobs.size(), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "pals_run_scenarios: arrival hashes");
    for (int64_t gi = 0; gi < total_nodes; ++gi)
        node_results[gi].arrival_stream_hash = hashes[node_stream[gi]];
    phase("results");
    // RequestRec per request (sim.hpp:100-107), kept on the context for pals_sim_requests
    ctx->sim_requests.clear();
    if (keep_req) {
        ctx->sim_requests.resize(total_nodes);
        int64_t gi = 0;
        for (int s = 0; s < n_scen; ++s)
            for (int i = 0; i < scens[s].n_nodes; ++i, ++gi) {
                const size_t u = (size_t)node_stream[gi];
                const int32_t* st_len = hbuf + s_ol[u];
                const int32_t* st_cum = hbuf + s_oc[u];
                const size_t nreq = (size_t)gens[u].count;
                std::vector<int32_t> kk(nreq);
                std::vector<double> gg(nreq);
                e = copy_on(ctx->stream, kk.data(), res.at<int32_t>(o_req_k[gi]), nreq * 4,
                            cudaMemcpyDeviceToHost);
                if (e == cudaSuccess)
                    e = copy_on(ctx->stream, gg.data(), res.at<double>(o_req_gen[gi]), nreq * 8,
                                cudaMemcpyDeviceToHost);
                if (e != cudaSuccess) return cuda_fail(e, "pals_run_scenarios: requests");
                auto& out = ctx->sim_requests[gi];
                out.resize(nreq);
                const double iv = scens[s].interval_s;
                std::vector<double> arrival(nreq, 0.0);  // backlog: spawned at t = 0
                int64_t prev = scens[s].nodes[i].initial_backlog;
                for (int k = 0; k < n_int[s]; ++k) {
                    const int64_t ck = st_cum[(int64_t)k * cstride];
                    for (int64_t q = prev; q < ck; ++q) arrival[q] = k * iv;
                    prev = ck;
                }
                for (size_t q = 0; q < nreq; ++q) {
                    pals_sim_request& r = out[q];
                    r.id = (int64_t)q;
                    r.arrival_s = arrival[q];
                    r.output_tokens = st_len[q];
                    r._pad = 0;
                    r.completed_s = kk[q] ? (kk[q] - 1) * iv + iv : -1.0;
                    r.generated = kk[q] ? (double)st_len[q] : gg[q];
                }
            }
    }
    return PALS_OK;
}

extern "C" int pals_sim_last_timing(pals_ctx* ctx, double* host_setup_s, double* kernel_ms) {
    if (!ctx) return set_error(PALS_ECONFIG, "pals_sim_last_timing: null context");
    if (host_setup_s) *host_setup_s = ctx->sim_prep_s;
    if (kernel_ms) *kernel_ms = ctx->sim_kernel_ms;
    return PALS_OK;
}

extern "C" int pals_sim_set_streaming(pals_ctx* ctx, int32_t enable) {
    if (!ctx) return set_error(PALS_ECONFIG, "pals_sim_set_streaming: null context");
    ctx->sim_streaming = enable ? 1 : 0;
    return PALS_OK;
}

extern "C" int pals_sim_keep_requests(pals_ctx* ctx, int32_t enable) {
    if (!ctx) return set_error(PALS_ECONFIG, "pals_sim_keep_requests: null context");
    ctx->sim_keep_requests = enable ? 1 : 0;
    return PALS_OK;
}

extern "C" int pals_sim_requests(pals_ctx* ctx, int64_t node, pals_sim_request* out, int64_t cap,
                                 int64_t* n) {
    if (!ctx || !n) return set_error(PALS_ECONFIG, "pals_sim_requests: null argument");
    if (node < 0 || node >= (int64_t)ctx->sim_requests.size())
        return set_error(PALS_ERANGE, "pals_sim_requests: node outside the last run (or "
                                      "requests were not kept)");
    const auto& v = ctx->sim_requests[node];
    *n = (int64_t)v.size();
    if (out && cap > 0)
        std::memcpy(out, v.data(), sizeof(pals_sim_request) * (size_t)std::min<int64_t>(cap, *n));
    return PALS_OK;
}
