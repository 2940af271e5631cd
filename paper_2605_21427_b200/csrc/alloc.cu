// alloc.cu — the cluster budget allocator (allocate_budget, allocator.hpp:76-186),
// batched over many independent clusters ("problems").
//
// Setup (pals_alloc_create, once per models x candidate axes x margin):
//   k_alloc_eval   scores every candidate of every (model k, dp) pair: caps x batches at
//                  deploy[k].tp/ep and dp = 1..max_dp (analytic on the device; forest via
//                  forest.cu; table models by host lookup, first match wins)
//   k_alloc_steps  one CTA per pair: p_node / t_hat per candidate, bitonic sort by
//                  (power asc, throughput desc), the increasing envelope and the
//                  selection-margin scaling — detail::throughput_steps (allocator.hpp:34-56)
//                  followed by allocator.hpp:106. Identical (power, thr) pairs are
//                  indistinguishable, so any correct sort reproduces std::sort's output.
// Run (pals_alloc_run_device):
//   k_allocate     one thread per problem runs the reference's water-filling loop
//                  literally (same fold order, same 1e-12 tolerances, same ceil/div), with
//                  the step tables staged in shared memory. The only restructuring: the
//                  steps a node already affords (power <= budget) form a prefix of its
//                  power-sorted table, so the scan starts past it (those steps `continue`
//                  in the reference) and best_throughput_under is that prefix's last step.
#include <algorithm>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "pals_internal.cuh"

using namespace pals;

namespace {

constexpr int kAllocMaxCand = 8192;     // candidates per node (smem bitonic sort)
constexpr int kAllocLocalNodes = 32;    // per-thread node state kept in local memory
constexpr int kAllocThreads = 128;

struct AllocNode {
    double bud;    // res.node_budgets_w[i]
    double cur;    // cur_thr[i]
    double tgt;    // throughput_target_tps
    int start;     // number of steps with power_w <= bud
    int pair;      // step table index
};

__global__ void k_alloc_eval_analytic(const Analytic* an, int64_t n, const double* cap,
                                      const int* batch, const int* tp, const int* dp, double* T,
                                      double* P) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const Score s = analytic_score(*an, cap[i], batch[i], tp[i], dp[i]);
        T[i] = s.T;
        P[i] = s.P;
    }
}

// One CTA per candidate set: throughput_steps + margin scaling.
__global__ void __launch_bounds__(512) k_alloc_steps(const double* T, const double* P,
                                                     const int* cdp, const int64_t* set_off,
                                                     const int32_t* set_ok, int npow2,
                                                     int stride, double alpha, double beta,
                                                     double margin, double* step_p,
                                                     double* step_t, int32_t* n_steps) {
    extern __shared__ uint64_t sm[];
    uint64_t* k1 = sm;           // orderable(power)
    uint64_t* k2 = sm + npow2;   // ~orderable(thr): ascending = throughput descending
    const int set = blockIdx.x;
    if (!set_ok[set]) {
        if (threadIdx.x == 0) n_steps[set] = 0;
        return;
    }
    const int64_t o = set_off[set];
    const int ncand = (int)(set_off[set + 1] - o);
    for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        if (i < ncand) {
            // p_node = c.dp * (alpha * kGpusPerNode * P + beta), thr = c.dp * T (allocator.hpp:38-40)
            const int d = cdp[o + i];
            k1[i] = orderable(p_node_of(P[o + i], d, alpha, beta));
            k2[i] = ~orderable((double)d * T[o + i]);
        } else {
            k1[i] = ~0ull;
            k2[i] = ~0ull;
        }
    }
    __syncthreads();
    for (int k = 2; k <= npow2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const uint64_t a1 = k1[i], a2 = k2[i], b1 = k1[l], b2 = k2[l];
                    const bool gt = a1 > b1 || (a1 == b1 && a2 > b2);
                    if (gt == up) {
                        k1[i] = b1; k2[i] = b2;
                        k1[l] = a1; k2[l] = a2;
                    }
                }
            }
            __syncthreads();
        }
    if (threadIdx.x == 0) {
        // the increasing envelope (allocator.hpp:48-54), then power /= 1 - margin (:106)
        double* sp = step_p + (size_t)set * stride;
        double* st = step_t + (size_t)set * stride;
        double best = 0.0;
        int ns = 0;
        for (int i = 0; i < ncand; ++i) {
            const double thr = unorderable(~k2[i]);
            if (thr > best + 1e-12) {
                sp[ns] = unorderable(k1[i]) / (1.0 - margin);
                st[ns] = thr;
                ++ns;
                best = thr;
            }
        }
        n_steps[set] = ns;
    }
}

struct AllocDev {
    const double* step_p;
    const double* step_t;
    const int32_t* n_steps;
    const int32_t* set_err;    // per candidate set: PALS_OK or the scorer's error code
    int n_sets, stride;
    int max_dp;                // > 0: sets are (model, dp) pairs, set = model * max_dp + dp - 1
                               // = 0: node_model[i] names the candidate set directly
    double floor_unit;         // alpha * kGpusPerNode * min_cap + beta
};

// steps of node i affordable under budget b: count of the power-sorted prefix <= b
__device__ __forceinline__ int afford(const double* sp, int ns, int from, double b) {
    int j = from;
    while (j < ns && !(sp[j] > b)) ++j;
    return j;
}

template <bool kSmem>
__global__ void __launch_bounds__(kAllocThreads) k_allocate(
    AllocDev a, double quantum, int64_t n_problems, const int64_t* __restrict__ off,
    const int32_t* __restrict__ node_model, const int32_t* __restrict__ node_dp,
    const double* __restrict__ node_target, const double* __restrict__ cluster_budget,
    double* __restrict__ node_budget, double* __restrict__ total, uint8_t* __restrict__ all_sat,
    int32_t* __restrict__ status, AllocNode* __restrict__ spill) {
    extern __shared__ double smem[];
    const double* SP = a.step_p;
    const double* ST = a.step_t;
    const int32_t* NS = a.n_steps;
    if (kSmem) {
        const int nt = a.n_sets * a.stride;
        double* sp = smem;
        double* st = smem + nt;
        int32_t* ns = (int32_t*)(smem + 2 * nt);
        for (int i = threadIdx.x; i < nt; i += blockDim.x) {
            sp[i] = a.step_p[i];
            st[i] = a.step_t[i];
        }
        for (int i = threadIdx.x; i < a.n_sets; i += blockDim.x) ns[i] = a.n_steps[i];
        __syncthreads();
        SP = sp;
        ST = st;
        NS = ns;
    }
    const int64_t pi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pi >= n_problems) return;
    const int64_t o = off[pi];
    const int64_t n64 = off[pi + 1] - o;
    total[pi] = 0.0;
    all_sat[pi] = 0;
    if (n64 <= 0) {  // allocate_budget: no nodes (allocator.hpp:79)
        status[pi] = PALS_ECONFIG;
        return;
    }
    const int n = (int)n64;
    // node floors, summed in node order (allocator.hpp:81-86)
    double floor_total = 0.0;
    for (int i = 0; i < n; ++i) floor_total += (double)node_dp[o + i] * a.floor_unit;
    const double cb = cluster_budget[pi];
    if (floor_total > cb) {  // allocator.hpp:87-95
        status[pi] = PALS_ECONFIG;
        return;
    }
    // throughput_steps per node in order: the first node whose candidates the scorer
    // rejects ends the problem with that error (allocator.hpp:103-105)
    for (int i = 0; i < n; ++i) {
        const int m = node_model[o + i], d = node_dp[o + i];
        int err = PALS_OK;
        if (a.max_dp > 0) {
            const int n_models = a.n_sets / a.max_dp;
            if (m < 0 || m >= n_models) err = PALS_ECONFIG;
            else if (d < 1) err = PALS_ECONFIG;       // OperatingPoint: parallel degrees >= 1
            else if (d > a.max_dp) err = PALS_ERANGE;  // beyond the plan's step tables
            else err = a.set_err[m * a.max_dp + d - 1];
        } else {
            err = (m < 0 || m >= a.n_sets) ? PALS_ECONFIG : a.set_err[m];
        }
        if (err != PALS_OK) {
            status[pi] = err;
            return;
        }
    }
    AllocNode local[kAllocLocalNodes];
    AllocNode* nd = n <= kAllocLocalNodes ? local : spill + o;
    double remaining = cb - floor_total;
    for (int i = 0; i < n; ++i) {
        AllocNode s;
        s.pair = a.max_dp > 0 ? node_model[o + i] * a.max_dp + node_dp[o + i] - 1
                              : node_model[o + i];
        s.bud = (double)node_dp[o + i] * a.floor_unit;
        s.tgt = node_target[o + i];
        const double* sp = SP + (size_t)s.pair * a.stride;
        s.start = afford(sp, NS[s.pair], 0, s.bud);
        s.cur = s.start ? ST[(size_t)s.pair * a.stride + s.start - 1] : 0.0;
        nd[i] = s;
    }
    // water-filling (allocator.hpp:124-160)
    while (remaining >= quantum) {
        bool any_unmet = false;
        for (int i = 0; i < n; ++i) any_unmet |= !(nd[i].cur >= nd[i].tgt);
        double best_rate = 0.0, best_cost = 0.0, best_bud = 0.0;
        int best_i = n;
        for (int i = 0; i < n; ++i) {
            const AllocNode s = nd[i];
            if (any_unmet && s.cur >= s.tgt) continue;
            const double* sp = SP + (size_t)s.pair * a.stride;
            const double* st = ST + (size_t)s.pair * a.stride;
            const int ns = NS[s.pair];
            const double cur_c = smin(s.cur, s.tgt);
            for (int j = s.start; j < ns; ++j) {
                const double pw = sp[j], th = st[j];
                if (pw <= s.bud || th <= s.cur) continue;
                const double cost = ceil((pw - s.bud) / quantum) * quantum;
                if (cost > remaining) break;
                const double gain = any_unmet ? smin(th, s.tgt) - cur_c : th - s.cur;
                if (gain <= 1e-12) continue;
                const double rate = gain / cost;
                const bool wins = best_i == n || rate > best_rate + 1e-12 ||
                                  (rate > best_rate - 1e-12 && s.bud < best_bud - 1e-12);
                if (wins) {
                    best_rate = rate;
                    best_cost = cost;
                    best_i = i;
                    best_bud = s.bud;
                }
            }
        }
        if (best_i == n) break;
        AllocNode& w = nd[best_i];
        w.bud += best_cost;
        const double* sp = SP + (size_t)w.pair * a.stride;
        w.start = afford(sp, NS[w.pair], w.start, w.bud);
        w.cur = w.start ? ST[(size_t)w.pair * a.stride + w.start - 1] : 0.0;
        remaining -= best_cost;
    }
    // remainder sweep to just past each node's top step (allocator.hpp:166-180)
    while (remaining >= quantum) {
        int lo = n;
        double lo_bud = 0.0;
        for (int i = 0; i < n; ++i) {
            const int ns = NS[nd[i].pair];
            const double ceiling =
                ns == 0 ? nd[i].bud : SP[(size_t)nd[i].pair * a.stride + ns - 1] + 2.0 * quantum;
            if (nd[i].bud + quantum > ceiling) continue;
            if (lo == n || nd[i].bud < lo_bud) {
                lo = i;
                lo_bud = nd[i].bud;
            }
        }
        if (lo == n) break;
        nd[lo].bud += quantum;
        remaining -= quantum;
    }
    double tot = 0.0;
    bool sat = true;
    for (int i = 0; i < n; ++i) {
        node_budget[o + i] = nd[i].bud;
        tot += nd[i].bud;
        sat &= nd[i].cur >= nd[i].tgt;
    }
    total[pi] = tot;
    all_sat[pi] = sat ? 1 : 0;
    status[pi] = PALS_OK;
}

int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, what);
    return PALS_OK;
}

}  // namespace

struct pals_alloc {
    pals_ctx* ctx = nullptr;
    int n_sets = 0, max_dp = 0, stride = 1;
    double floor_unit = 0.0;
    double* d_sp = nullptr;
    double* d_st = nullptr;
    int32_t* d_ns = nullptr;
    int32_t* d_err = nullptr;
    std::vector<int32_t> h_err;
    std::vector<std::string> h_msg;
    // host-entry staging and the large-cluster spill area
    void* d_io = nullptr;
    size_t io_bytes = 0;
    AllocNode* d_spill = nullptr;
    int64_t spill_n = 0;
};

// Step tables for candidate sets: set s is scored by set_model[s] over
// points[set_off[s] .. set_off[s+1]).
static int alloc_build(pals_ctx* ctx, int n_sets, const pals_model* const* set_model,
                       const pals_point* points, const int64_t* set_off, const pals_gpu_spec* gpu,
                       const pals_coeffs* coeffs, double margin, int max_dp, pals_alloc** out) {
    int64_t maxc = 0;
    for (int k = 0; k < n_sets; ++k) {
        const int64_t c = set_off[k + 1] - set_off[k];
        if (c < 0 || c > kAllocMaxCand)
            return set_error(PALS_ECONFIG, "pals_alloc: candidates per set must be in [0, " +
                                               std::to_string(kAllocMaxCand) + "]");
        maxc = std::max(maxc, c);
    }
    PALS_CUDA(cudaSetDevice(ctx->device));
    auto* A = new pals_alloc();
    A->ctx = ctx;
    A->n_sets = n_sets;
    A->max_dp = max_dp;
    A->stride = (int)std::max<int64_t>(1, maxc);
    A->floor_unit = coeffs->alpha * (double)kGpusPerNode * gpu->min_cap_watts + coeffs->beta_watts;
    A->h_err.assign(n_sets, PALS_OK);
    A->h_msg.assign(n_sets, std::string());
    const int64_t N = set_off[n_sets] - set_off[0];
    const int64_t base = set_off[0];
    cudaStream_t s = ctx->stream;
    // candidate SoA + scores, contiguous over all sets
    std::vector<double> hcap(std::max<int64_t>(1, N));
    std::vector<int> hi(4 * std::max<int64_t>(1, N));
    for (int64_t i = 0; i < N; ++i) {
        const pals_point& p = points[base + i];
        hcap[i] = p.cap_watts;
        hi[i] = p.batch;
        hi[N + i] = p.tp;
        hi[2 * N + i] = p.ep;
        hi[3 * N + i] = p.dp;
    }
    double *dT = nullptr, *dP = nullptr, *dcap = nullptr;
    int *di = nullptr, *d_ok = nullptr;
    int64_t* doff = nullptr;
    std::vector<int32_t> ok(n_sets);
    int rc = PALS_OK;
    const size_t n1 = (size_t)std::max<int64_t>(1, N);
    if (cudaMalloc(&A->d_sp, sizeof(double) * n_sets * A->stride) != cudaSuccess ||
        cudaMalloc(&A->d_st, sizeof(double) * n_sets * A->stride) != cudaSuccess ||
        cudaMalloc(&A->d_ns, sizeof(int32_t) * n_sets) != cudaSuccess ||
        cudaMalloc(&A->d_err, sizeof(int32_t) * n_sets) != cudaSuccess ||
        cudaMalloc(&dT, sizeof(double) * n1) != cudaSuccess ||
        cudaMalloc(&dP, sizeof(double) * n1) != cudaSuccess ||
        cudaMalloc(&dcap, sizeof(double) * n1) != cudaSuccess ||
        cudaMalloc(&di, sizeof(int) * 4 * n1) != cudaSuccess ||
        cudaMalloc(&d_ok, sizeof(int32_t) * n_sets) != cudaSuccess ||
        cudaMalloc(&doff, sizeof(int64_t) * (n_sets + 1)) != cudaSuccess) {
        rc = cuda_fail(cudaErrorMemoryAllocation, "pals_alloc");
        goto done;
    }
    copy_on(ctx->stream, dcap, hcap.data(), sizeof(double) * n1, cudaMemcpyHostToDevice);
    copy_on(ctx->stream, di, hi.data(), sizeof(int) * 4 * n1, cudaMemcpyHostToDevice);
    for (int k = 0; k < n_sets && rc == PALS_OK; ++k) {
        const pals_model* m = set_model[k];
        const int64_t o = set_off[k] - base, nc = set_off[k + 1] - set_off[k];
        // the error the scorer would throw on this set's first bad candidate
        const int e = nc ? validate_points(m, points + set_off[k], nc) : PALS_OK;
        A->h_err[k] = e;
        if (e != PALS_OK) A->h_msg[k] = pals_last_error();
        ok[k] = e == PALS_OK;
        if (e != PALS_OK || nc == 0) continue;
        if (m->kind == MODEL_TABLE) {  // TableScorer: first equal point wins
            std::unordered_map<std::string, int64_t> idx;
            idx.reserve((size_t)m->table_n * 2);
            for (int64_t i = 0; i < m->table_n; ++i) {
                pals_point q = m->table_pts[i];
                if (q.cap_watts == 0.0) q.cap_watts = 0.0;
                idx.emplace(std::string((const char*)&q, sizeof(q)), i);
            }
            std::vector<double> hT(nc), hP(nc);
            for (int64_t c = 0; c < nc; ++c) {
                pals_point q = points[set_off[k] + c];
                if (q.cap_watts == 0.0) q.cap_watts = 0.0;
                const int64_t r = idx.at(std::string((const char*)&q, sizeof(q)));
                hT[c] = m->table_T[r];
                hP[c] = m->table_P[r];
            }
            copy_on(ctx->stream, dT + o, hT.data(), sizeof(double) * nc, cudaMemcpyHostToDevice);
            copy_on(ctx->stream, dP + o, hP.data(), sizeof(double) * nc, cudaMemcpyHostToDevice);
        } else if (m->kind == MODEL_ANALYTIC) {
            if (!m->d_an) {
                auto* mm = const_cast<pals_model*>(m);
                if (cudaMalloc(&mm->d_an, sizeof(Analytic)) != cudaSuccess) {
                    rc = cuda_fail(cudaErrorMemoryAllocation, "pals_alloc d_an");
                    break;
                }
                copy_on(ctx->stream, mm->d_an, &m->an, sizeof(Analytic), cudaMemcpyHostToDevice);
            }
            const int blocks = (int)std::max<int64_t>(
                1, std::min<int64_t>((nc + 255) / 256, 4 * ctx->num_sms));
            k_alloc_eval_analytic<<<blocks, 256, 0, s>>>(m->d_an, nc, dcap + o, di + o,
                                                         di + N + o, di + 3 * N + o, dT + o,
                                                         dP + o);
            count_launch(ctx);
            rc = check_launch("k_alloc_eval_analytic");
        } else {  // forest: PredictorBundle::predict accepts any point
            rc = forest_eval_raw(m, ctx, nc, dcap + o, di + o, di + N + o, di + 2 * N + o,
                                 di + 3 * N + o, dT + o, dP + o, 0);
        }
    }
    if (rc == PALS_OK) {
        std::vector<int64_t> rel(n_sets + 1);
        for (int k = 0; k <= n_sets; ++k) rel[k] = set_off[k] - base;
        copy_on(ctx->stream, doff, rel.data(), sizeof(int64_t) * (n_sets + 1), cudaMemcpyHostToDevice);
        copy_on(ctx->stream, A->d_err, A->h_err.data(), sizeof(int32_t) * n_sets, cudaMemcpyHostToDevice);
        copy_on(ctx->stream, d_ok, ok.data(), sizeof(int32_t) * n_sets, cudaMemcpyHostToDevice);
        int npow2 = 1;
        while (npow2 < maxc) npow2 <<= 1;
        const size_t smem = sizeof(uint64_t) * 2 * npow2;
        cudaFuncSetAttribute(k_alloc_steps, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_alloc_steps<<<n_sets, 512, smem, s>>>(dT, dP, di + 3 * N, doff, d_ok, npow2, A->stride,
                                                coeffs->alpha, coeffs->beta_watts, margin,
                                                A->d_sp, A->d_st, A->d_ns);
        count_launch(ctx);
        rc = check_launch("k_alloc_steps");
        const cudaError_t e = cudaStreamSynchronize(s);
        if (rc == PALS_OK && e != cudaSuccess) rc = cuda_fail(e, "pals_alloc sync");
    }
done:
    cudaFree(dT);
    cudaFree(dP);
    cudaFree(dcap);
    cudaFree(di);
    cudaFree(d_ok);
    cudaFree(doff);
    if (rc != PALS_OK) {
        pals_alloc_destroy(A);
        return rc;
    }
    *out = A;
    return PALS_OK;
}

extern "C" {

int pals_alloc_create(pals_ctx* ctx, int32_t n_models, pals_model* const* models,
                      const pals_profile* deploy, const pals_gpu_spec* gpu,
                      const pals_coeffs* coeffs, const double* caps, int32_t n_caps,
                      const int32_t* batches, int32_t n_batches, int32_t max_dp,
                      double selection_margin, pals_alloc** out) {
    if (!ctx || !models || !deploy || !gpu || !coeffs || !out ||
        (n_caps > 0 && !caps) || (n_batches > 0 && !batches))
        return set_error(PALS_ECONFIG, "pals_alloc_create: null argument");
    if (n_models <= 0) return set_error(PALS_ECONFIG, "pals_alloc_create: no models");
    if (max_dp < 1 || max_dp > kMaxDp)
        return set_error(PALS_ECONFIG, "pals_alloc_create: max_dp must be in [1, " +
                                           std::to_string(kMaxDp) + "]");
    if (n_caps < 0 || n_batches < 0)
        return set_error(PALS_ECONFIG, "pals_alloc_create: negative axis length");
    const int64_t nc = (int64_t)n_caps * n_batches;
    if (nc > kAllocMaxCand)
        return set_error(PALS_ECONFIG, "pals_alloc: candidates per set must be in [0, " +
                                           std::to_string(kAllocMaxCand) + "]");
    for (int k = 0; k < n_models; ++k)
        if (!models[k]) return set_error(PALS_ECONFIG, "pals_alloc_create: null model");
    // sets (model k, dp d) = caps x batches at deploy[k].tp/ep and dp d (sim.hpp:293-308 order)
    const int n_sets = n_models * max_dp;
    std::vector<pals_point> pts((size_t)n_sets * nc);
    std::vector<int64_t> off(n_sets + 1);
    std::vector<const pals_model*> sm(n_sets);
    size_t w = 0;
    for (int k = 0; k < n_models; ++k)
        for (int d = 1; d <= max_dp; ++d) {
            const int set = k * max_dp + d - 1;
            off[set] = (int64_t)w;
            sm[set] = models[k];
            for (int a = 0; a < n_caps; ++a)
                for (int b = 0; b < n_batches; ++b)
                    pts[w++] = pals_point{caps[a], batches[b], deploy[k].deploy_tp,
                                          deploy[k].deploy_ep, d};
        }
    off[n_sets] = (int64_t)w;
    return alloc_build(ctx, n_sets, sm.data(), pts.data(), off.data(), gpu, coeffs,
                       selection_margin, max_dp, out);
}

int pals_alloc_create_sets(pals_ctx* ctx, int32_t n_sets, pals_model* const* set_models,
                           const pals_point* points, const int64_t* set_offset,
                           const pals_gpu_spec* gpu, const pals_coeffs* coeffs,
                           double selection_margin, pals_alloc** out) {
    if (!ctx || !set_models || !set_offset || !gpu || !coeffs || !out)
        return set_error(PALS_ECONFIG, "pals_alloc_create_sets: null argument");
    if (n_sets <= 0) return set_error(PALS_ECONFIG, "pals_alloc_create_sets: no sets");
    for (int k = 0; k < n_sets; ++k) {
        if (!set_models[k]) return set_error(PALS_ECONFIG, "pals_alloc_create_sets: null model");
        if (set_offset[k + 1] < set_offset[k])
            return set_error(PALS_ECONFIG, "pals_alloc_create_sets: set_offset must not decrease");
    }
    if (set_offset[n_sets] > set_offset[0] && !points)
        return set_error(PALS_ECONFIG, "pals_alloc_create_sets: null points");
    return alloc_build(ctx, n_sets, set_models, points, set_offset, gpu, coeffs,
                       selection_margin, 0, out);
}

int pals_alloc_destroy(pals_alloc* A) {
    if (!A) return PALS_OK;
    cudaFree(A->d_sp);
    cudaFree(A->d_st);
    cudaFree(A->d_ns);
    cudaFree(A->d_err);
    cudaFree(A->d_io);
    cudaFree(A->d_spill);
    delete A;
    return PALS_OK;
}

int pals_alloc_steps(pals_alloc* A, int32_t set, double* power_w, double* throughput_tps,
                     int32_t* n_steps) {
    if (!A || !n_steps) return set_error(PALS_ECONFIG, "pals_alloc_steps: null argument");
    if (set < 0 || set >= A->n_sets)
        return set_error(PALS_ERANGE, "pals_alloc_steps: set outside the plan");
    if (A->h_err[set] != PALS_OK) return set_error(A->h_err[set], A->h_msg[set]);
    PALS_CUDA(copy_on(A->ctx->stream, n_steps, A->d_ns + set, sizeof(int32_t), cudaMemcpyDeviceToHost));
    const size_t o = (size_t)set * A->stride;
    if (power_w)
        PALS_CUDA(copy_on(A->ctx->stream, power_w, A->d_sp + o, sizeof(double) * *n_steps,
                             cudaMemcpyDeviceToHost));
    if (throughput_tps)
        PALS_CUDA(copy_on(A->ctx->stream, throughput_tps, A->d_st + o, sizeof(double) * *n_steps,
                             cudaMemcpyDeviceToHost));
    return PALS_OK;
}

static int alloc_launch(pals_alloc* A, double quantum, int64_t n_problems, const int64_t* off,
                        int64_t n_nodes, const int32_t* model, const int32_t* dp,
                        const double* target, const double* budget, double* node_budget,
                        double* total, uint8_t* all_sat, int32_t* status) {
    pals_ctx* ctx = A->ctx;
    if (!(quantum > 0.0))
        return set_error(PALS_ECONFIG, "pals_allocate: quantum_w must be > 0");
    if (n_problems <= 0) return PALS_OK;
    if (n_nodes > A->spill_n) {
        cudaFree(A->d_spill);
        A->d_spill = nullptr;
        A->spill_n = 0;
        PALS_CUDA(cudaMalloc(&A->d_spill, sizeof(AllocNode) * std::max<int64_t>(1, n_nodes)));
        A->spill_n = n_nodes;
    }
    AllocDev a;
    a.step_p = A->d_sp;
    a.step_t = A->d_st;
    a.n_steps = A->d_ns;
    a.set_err = A->d_err;
    a.n_sets = A->n_sets;
    a.stride = A->stride;
    a.max_dp = A->max_dp;
    a.floor_unit = A->floor_unit;
    const size_t smem = sizeof(double) * 2 * (size_t)a.n_sets * a.stride +
                        sizeof(int32_t) * a.n_sets;
    const int blocks = (int)((n_problems + kAllocThreads - 1) / kAllocThreads);
    if (smem <= 48 * 1024) {
        k_allocate<true><<<blocks, kAllocThreads, smem, ctx->stream>>>(
            a, quantum, n_problems, off, model, dp, target, budget, node_budget, total, all_sat,
            status, A->d_spill);
    } else {
        k_allocate<false><<<blocks, kAllocThreads, 0, ctx->stream>>>(
            a, quantum, n_problems, off, model, dp, target, budget, node_budget, total, all_sat,
            status, A->d_spill);
    }
    count_launch(ctx);
    return check_launch("k_allocate");
}

int pals_alloc_run_device(pals_alloc* A, double quantum_w, int64_t n_problems,
                          const int64_t* d_node_offset, int64_t n_nodes,
                          const int32_t* d_node_model, const int32_t* d_node_dp,
                          const double* d_node_target, const double* d_cluster_budget,
                          double* d_node_budget, double* d_total, uint8_t* d_all_sat,
                          int32_t* d_status) {
    if (!A) return set_error(PALS_ECONFIG, "pals_alloc_run_device: null plan");
    PALS_CUDA(cudaSetDevice(A->ctx->device));
    return alloc_launch(A, quantum_w, n_problems, d_node_offset, n_nodes, d_node_model,
                        d_node_dp, d_node_target, d_cluster_budget, d_node_budget, d_total,
                        d_all_sat, d_status);
}

int pals_allocate_budget(pals_alloc* A, double quantum_w, int64_t n_problems,
                         const int64_t* node_offset, const int32_t* node_model,
                         const int32_t* node_dp, const double* node_target,
                         const double* cluster_budget, double* node_budget, double* total,
                         uint8_t* all_satisfied, int32_t* status) {
    if (!A || (n_problems > 0 && (!node_offset || !node_model || !node_dp || !node_target ||
                                  !cluster_budget || !node_budget || !total || !all_satisfied ||
                                  !status)))
        return set_error(PALS_ECONFIG, "pals_allocate_budget: null argument");
    if (n_problems <= 0) return PALS_OK;
    pals_ctx* ctx = A->ctx;
    PALS_CUDA(cudaSetDevice(ctx->device));
    if (node_offset[0] != 0)
        return set_error(PALS_ECONFIG, "pals_allocate_budget: node_offset[0] must be 0");
    int64_t n_nodes = 0;
    for (int64_t i = 0; i <= n_problems; ++i) n_nodes = std::max(n_nodes, node_offset[i]);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t b_off = al(8 * (n_problems + 1)), b_n4 = al(4 * n_nodes), b_n8 = al(8 * n_nodes),
                 b_p8 = al(8 * n_problems), b_p4 = al(4 * n_problems), b_p1 = al(n_problems);
    const size_t need = b_off + 2 * b_n4 + 2 * b_n8 + 2 * b_p8 + b_p4 + b_p1;
    if (A->io_bytes < need) {
        cudaFree(A->d_io);
        A->d_io = nullptr;
        A->io_bytes = 0;
        PALS_CUDA(cudaMalloc(&A->d_io, need));
        A->io_bytes = need;
    }
    char* p = (char*)A->d_io;
    int64_t* d_off = (int64_t*)p; p += b_off;
    int32_t* d_m = (int32_t*)p; p += b_n4;
    int32_t* d_dp = (int32_t*)p; p += b_n4;
    double* d_tg = (double*)p; p += b_n8;
    double* d_nb = (double*)p; p += b_n8;
    double* d_cb = (double*)p; p += b_p8;
    double* d_tot = (double*)p; p += b_p8;
    int32_t* d_st = (int32_t*)p; p += b_p4;
    uint8_t* d_sat = (uint8_t*)p;
    cudaStream_t s = ctx->stream;
    PALS_CUDA(cudaMemcpyAsync(d_off, node_offset, 8 * (n_problems + 1), cudaMemcpyHostToDevice, s));
    if (n_nodes) {
        PALS_CUDA(cudaMemcpyAsync(d_m, node_model, 4 * n_nodes, cudaMemcpyHostToDevice, s));
        PALS_CUDA(cudaMemcpyAsync(d_dp, node_dp, 4 * n_nodes, cudaMemcpyHostToDevice, s));
        PALS_CUDA(cudaMemcpyAsync(d_tg, node_target, 8 * n_nodes, cudaMemcpyHostToDevice, s));
        PALS_CUDA(cudaMemsetAsync(d_nb, 0, 8 * n_nodes, s));
    }
    PALS_CUDA(cudaMemcpyAsync(d_cb, cluster_budget, 8 * n_problems, cudaMemcpyHostToDevice, s));
    int rc = alloc_launch(A, quantum_w, n_problems, d_off, n_nodes, d_m, d_dp, d_tg, d_cb, d_nb,
                          d_tot, d_sat, d_st);
    if (rc) return rc;
    if (n_nodes)
        PALS_CUDA(cudaMemcpyAsync(node_budget, d_nb, 8 * n_nodes, cudaMemcpyDeviceToHost, s));
    PALS_CUDA(cudaMemcpyAsync(total, d_tot, 8 * n_problems, cudaMemcpyDeviceToHost, s));
    PALS_CUDA(cudaMemcpyAsync(all_satisfied, d_sat, n_problems, cudaMemcpyDeviceToHost, s));
    PALS_CUDA(cudaMemcpyAsync(status, d_st, 4 * n_problems, cudaMemcpyDeviceToHost, s));
    PALS_CUDA(cudaStreamSynchronize(s));
    return PALS_OK;
}

}  // extern "C"
