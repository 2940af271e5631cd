// replay_common.cuh — device-side select_config from per-model rank tables,
// shared by the batched controller replay (replay.cu) and the queue-plant
// scenario simulator (sim.cu). See DESIGN.md §3-4.
#pragma once
#include "pals_internal.cuh"

namespace pals {

constexpr int kMaxReplayCands = 4096;

struct ReplayModelDev {
    int n;             // candidates
    int nd_t, nd_p;    // sorted t_hat / p_node entries (= n)
    int tp, ep, dp;
    int init_idx;      // (max cap, max batch) candidate
    int gmax_t, gmin_p;
    int generic;
    double max_cap;
    int max_batch;
    double t_max, p_min, p_max;  // plant: unconstrained tps, min/max p_node
    const double* cap;
    const int* batch;
    const int* canon;
    const int* inv_tr;
    const double* T;    // scorer throughput per candidate (PID promise)
    const double* th;
    const double* pn;
    const double* ef;
    const uint8_t* danger_t;  // per rank: the value's run ends on a near-tie
    const uint8_t* danger_e;
    const double* ut;   // distinct t_hat, descending
    const double* up;   // distinct p_node, ascending
    const uint32_t* m2; // (n+1) x (n+1): min eff key over {r_t < i, r_p < j}
    const uint32_t* b1; // n+1: min t key over {r_p < j}
    const Analytic* plant;
    // enforce_cap (sim.hpp:195-205) walk tables: from cap index a the breaker visits
    // caps walk_c[a][j] (c_0 = caps[a], c_{j+1} = max(min_cap, c_j - 5)); walk_T /
    // walk_pn hold the plant's throughput and cluster_system_power there, per batch.
    int nc, nb, L;
    int init_a, init_b;  // (max cap, max batch) indices into the caps / batches lists
    double plant_min_cap;
    const double* walk_c;   // [nc][L]
    const double* walk_T;   // [nc][nb][L]
    const double* walk_pn;  // [nc][nb][L]
    const double* walk_pm;  // [nc][nb][L]: running min of walk_pn along the walk
    const int* walk_jmin;   // [nc]: first walk position with c <= min_cap
};

// Literal select_config over a replay model's candidates by one thread
// (rarely used: near-tie winners and non-finite score sets).
__device__ inline void thread_select_full(const ReplayModelDev& m, double target, bool bset, double budget,
                                   double bias, int objective, int* idx, int* reason) {
    int best = -1;
    int r = PALS_REASON_FALLBACK_MAX_T;
    if (objective == PALS_OBJ_QOS) {
        for (int c = 0; c < m.n; ++c) {
            if ((bset && !(m.pn[c] <= budget)) || m.th[c] * bias < target) continue;
            if (best < 0 || better_exact(m.th[c] / m.pn[c], m.cap[c], m.batch[c],
                                         m.th[best] / m.pn[best], m.cap[best], m.batch[best]))
                best = c;
        }
        if (best >= 0) r = PALS_REASON_QOS_FEASIBLE;
    }
    if (best < 0 && bset) {
        for (int c = 0; c < m.n; ++c) {
            if (!(m.pn[c] <= budget)) continue;
            if (best < 0 ||
                better_exact(m.th[c], m.cap[c], m.batch[c], m.th[best], m.cap[best], m.batch[best]))
                best = c;
        }
        if (best >= 0) r = PALS_REASON_BUDGET_MAX_T;
        if (best < 0) {
            for (int c = 0; c < m.n; ++c)
                if (best < 0 || better_exact(-m.pn[c], m.cap[c], m.batch[c], -m.pn[best],
                                             m.cap[best], m.batch[best]))
                    best = c;
            r = PALS_REASON_BUDGET_MAX_T;
        }
    }
    if (best < 0) {
        for (int c = 0; c < m.n; ++c)
            if (best < 0 ||
                better_exact(m.th[c], m.cap[c], m.batch[c], m.th[best], m.cap[best], m.batch[best]))
                best = c;
        r = PALS_REASON_FALLBACK_MAX_T;
    }
    *idx = best;
    *reason = r;
}

// select_config via the rank tables; exact by the near-tie argument of DESIGN.md §3.
// Kt = #sorted t_hat entries with !(t*bias < target), kept incrementally: bias moves
// a little each step, so the previous count is re-validated with two exact tests (two
// independent loads) before falling back to a binary search (same value either way),
// narrowed to the side of prev the failing test points to. (A bounded walk from prev and
// a 4-ary search with three independent probes per round both measured slower on B200:
// they hold more registers in a kernel that is register-limited.)
__device__ __forceinline__ int count_t_feasible(const ReplayModelDev& m, double bias,
                                                   double target, int prev) {
    const bool ok_lo = prev == 0 || !(m.ut[prev - 1] * bias < target);
    const bool ok_hi = prev == m.nd_t || (m.ut[prev] * bias < target);
    if (ok_lo && ok_hi) return prev;
    // the count lies in [lo, hi]; a failing test narrows it to one side of prev
    int lo = ok_lo ? prev + 1 : 0, hi = ok_lo ? m.nd_t : prev - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (!(m.ut[mid] * bias < target)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

constexpr uint32_t kWordDanger = 0x40000000u;  // table word: winner needs the exact fold
constexpr uint32_t kWordIdx = 0x000FFFFFu;

// select_config from the per-model tables; returns the CANONICAL candidate index.
// Table words are precomputed: canonical winner index | danger flag (k_build_tables).
__device__ __forceinline__ void table_select(const ReplayModelDev& m, double target, bool bset,
                                             double budget, int kp, int kt, double bias,
                                             int objective, int* idx, int* reason) {
    // the rank tables assume a t-feasible prefix, i.e. bias >= 0 (bias_min may be negative
    // in a caller's ControllerConfig / initial state): otherwise the literal fold
    if (!m.generic && !(objective == PALS_OBJ_QOS && bias < 0.0)) {
        bool qos_empty = true;
        if (objective == PALS_OBJ_QOS) {
            const uint32_t w = m.m2[kt * (m.nd_p + 1) + (bset ? kp : m.nd_p)];
            if (w != kNone32) {
                if (!(w & kWordDanger)) {
                    *idx = (int)(w & kWordIdx);
                    *reason = PALS_REASON_QOS_FEASIBLE;
                    return;
                }
                qos_empty = false;  // near-tie winner: exact fold below
            }
        }
        if (qos_empty) {
            if (!bset) {  // fallback: max throughput over all (controller.hpp:191-198)
                *idx = m.gmax_t;
                *reason = PALS_REASON_FALLBACK_MAX_T;
                return;
            }
            const uint32_t w = m.b1[kp];
            if (w == kNone32 || !(w & kWordDanger)) {
                // budget below every candidate -> least power (controller.hpp:180-188)
                *idx = w == kNone32 ? m.gmin_p : (int)(w & kWordIdx);
                *reason = PALS_REASON_BUDGET_MAX_T;
                return;
            }
        }
    }
    // near-tie winner or non-finite scores: the literal fold
    thread_select_full(m, target, bset, budget, bias, objective, idx, reason);
    *idx = m.canon[*idx];
}

// Number of leading indices i in [0, n) with pred(i) true, for a predicate that is
// true on a prefix (sorted tables): 32-ary narrowing by one warp, ceil(log32 n)
// rounds of one load per lane instead of log2 n dependent loads. Same count as
// the binary searches of the thread layout.
template <class Pred>
__device__ __forceinline__ int warp_leading_true(int n, Pred pred) {
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = n;  // the count lies in [lo, hi]
    while (lo < hi) {
        const int step = (hi - lo + 31) >> 5;
        const int i = lo + (lane + 1) * step - 1;
        const unsigned b = __ballot_sync(0xffffffffu, i < hi && pred(i));
        const int nlo = lo + __popc(b) * step;
        hi = min(hi, nlo + step - 1);
        lo = nlo;
    }
    return lo;
}

// Per-model select tables from a prepared plan (replay.cu): m2 / b1 decision words,
// the sorted distinct t_hat / p_node arrays, globals; plant constants t_max, p_min, p_max.
__global__ void k_build_tables(PlanDev d, ReplayModelDev* rm, uint32_t* m2, uint32_t* b1,
                               double* ut, double* up, double alpha, double beta);

}  // namespace pals
