// pals_internal.cuh — shared device/host definitions for libpals_gpu.so.
//
// All FP64 arithmetic follows the reference's operation order literally and is
// compiled with -fmad=false (device) / -ffp-contract=off (host), so every
// double is bit-identical to the reference's Release build (SURVEY F3,
// Appendix A). Citations: /root/reference/proj/include/wattserve/<file>:<line>.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/pals_gpu.h"

#define PALS_HD __host__ __device__ __forceinline__

namespace pals {

constexpr int kGpusPerNode = 4;          // types.hpp:11
constexpr double kFloorRatio = 0.4;      // model.hpp:33
constexpr double kTieTol = 1e-9;         // controller.hpp:121-122
constexpr int kMaxDp = 256;              // pow(internode, dp-1) host table size
constexpr uint32_t kNone32 = 0xFFFFFFFFu;
constexpr uint64_t kNone64 = ~0ull;

// ---- programmatic dependent launch (PDL) ------------------------------------
// Kernels of the select step start with pdl_wait(); pdl_trigger(): a kernel
// launched with the PDL attribute may be scheduled while its predecessor still
// runs, and blocks in pdl_wait() until the predecessor has completed and its
// writes are visible, so the ordering is that of a plain stream. Without the
// attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() {
#ifdef __CUDA_ARCH__
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#ifdef __CUDA_ARCH__
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// ---- libstdc++ comparison helpers (stl_algobase.h:257-265, stl_algo.h:3667-3671)
PALS_HD double smax(double a, double b) { return a < b ? b : a; }
PALS_HD double smin(double a, double b) { return b < a ? b : a; }
PALS_HD double sclamp(double v, double lo, double hi) { return smin(smax(v, lo), hi); }

// rng.hpp:15-20
PALS_HD uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// Analytic model parameters (ModelProfile + GpuSpec), flattened for the device.
struct Analytic {
    double compute_fixed, compute_per_seq, comm_per_seq, knee_watts;
    double compute_power_base, compute_power_per_seq, comm_power, overlap;
    double min_cap, max_cap, max_frequency;
    int n_tp;
    int tp_keys[PALS_MAX_TP_KEYS];
    double comm_fixed[PALS_MAX_TP_KEYS];
    double pow_dp[kMaxDp + 1];  // pow_dp[d] = std::pow(internode_factor, d - 1), host glibc
};

// Scores of one point: CandidateScore{throughput_tps, gpu_power_w} (controller.hpp:93-96)
struct Score {
    double T, P;
};

// step_timing + throughput + avg_gpu_power (model.hpp:37-84) for a point that
// already passed validation. Returns T, P and the per-step terms.
PALS_HD Score analytic_score(const Analytic& a, double cap, int batch, int tp, int dp,
                             double* t_comp_out = nullptr, double* step_out = nullptr) {
    // effective_frequency model.hpp:41-44
    const double span = a.knee_watts - a.min_cap;
    double f;
    if (span <= 0.0) {
        f = a.max_frequency;
    } else {
        const double ratio = (cap - a.min_cap) / span;
        f = a.max_frequency * sclamp(ratio, kFloorRatio, 1.0);
    }
    double comm = 0.0;
    for (int i = 0; i < a.n_tp; ++i)
        if (a.tp_keys[i] == tp) comm = a.comm_fixed[i];
    const double B = (double)batch;
    const double t_comp = (a.compute_fixed + a.compute_per_seq * B / (double)tp) / f;
    const double t_comm = (comm + a.comm_per_seq * B) * a.pow_dp[dp];
    const double hi = smax(t_comp, t_comm);
    const double lo = smin(t_comp, t_comm);
    const double step = hi + (1.0 - a.overlap) * lo;
    Score s;
    s.T = B / step;
    const double demand = a.compute_power_base + a.compute_power_per_seq * B / (double)tp;
    const double p_comp = smin(cap, demand);
    const double comm_share = step - t_comp;
    s.P = (t_comp * p_comp + comm_share * a.comm_power) / step;
    if (t_comp_out) *t_comp_out = t_comp;
    if (step_out) *step_out = step;  // StepTiming::step_s (model.hpp:66)
    return s;
}

// select_config's per-candidate host power and instance throughput (controller.hpp:147-150)
PALS_HD double p_node_of(double P, int dp, double alpha, double beta) {
    return (double)dp * (alpha * (double)kGpusPerNode * P + beta);
}

// detail::better_candidate controller.hpp:118-125, literally
PALS_HD bool better_exact(double sa, double capa, int ba, double sb, double capb, int bb) {
    const double scale = smax(smax(fabs(sa), fabs(sb)), 1e-300);
    if ((sa - sb) / scale > kTieTol) return true;
    if ((sb - sa) / scale > kTieTol) return false;
    if (capa != capb) return capa < capb;
    return ba < bb;
}

// Order-preserving map double -> uint64 (ascending); -0 is folded to +0.
PALS_HD uint64_t orderable(double x) {
    if (x == 0.0) x = 0.0;
    uint64_t b;
#ifdef __CUDA_ARCH__
    b = (uint64_t)__double_as_longlong(x);
#else
    __builtin_memcpy(&b, &x, 8);
#endif
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
PALS_HD double unorderable(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    double x;
#ifdef __CUDA_ARCH__
    x = __longlong_as_double((long long)b);
#else
    __builtin_memcpy(&x, &b, 8);
#endif
    return x;
}

// ---- plan device layout ---------------------------------------------------
// Three orders: 0 = t_hat descending, 1 = p_node ascending, 2 = eff descending.
// In each order a point has a competition rank r (number of points with a
// strictly better value: equal values share r) and a packed key
// (r << tr_bits) | TR, TR = the grid's (cap, batch, index) rank, so min(key)
// is the reference's argmax with its knob tie-break.
enum { ORD_T = 0, ORD_P = 1, ORD_E = 2, N_ORD = 3 };

struct PlanDev {
    int64_t n;           // grid points
    int tr_bits;         // key = (D << tr_bits) | TR
    int wide;            // 1: 64-bit keys (n > 65535)
    // grid
    const double* cap;
    const int* batch;
    const int* dp;
    const int* inv_tr;   // TR -> point index
    const int* tr;       // point index -> TR
    // scores
    double* T;
    double* P;
    double* th;          // t_hat = dp * T
    double* pn;          // p_node
    double* ef;          // t_hat / p_node
    // rank structures (per order)
    uint64_t* skey[N_ORD];   // orderable keys of the values, in TR order (padded)
    uint64_t* sorted[N_ORD]; // ping-pong buffer of the merge rounds
    uint32_t* sidx[N_ORD];   // TR carried beside sorted[]; after the rank pass: the
                             // competition rank of every merged position
    uint64_t* merged[N_ORD]; // fully sorted keys (position r = competition rank r)
    uint32_t* midx[N_ORD];   // TR carried beside merged[]; after the rank pass: the point
                             // index at every merged position
    uint64_t* samp[N_ORD];   // merged[k * samp_s] for k < samp_n (search index)
    int64_t samp_s;          // sample stride
    int samp_n;              // samples per order
    uint8_t* bnd[N_ORD];     // per position i: 0 = merged[i+1] equal, 1 = distinct but a
                             // tolerance near-tie, 2 = separated (or i = n-1)
    uint8_t* danger[N_ORD];  // per run-start position: the run ends on a near-tie (bnd == 1)
    uint32_t* key32[N_ORD];  // packed keys (narrow)
    uint64_t* key64[N_ORD];  // packed keys (wide)
    uint32_t* rank32[N_ORD]; // per point: competition rank r (the pair scan's feasibility side)
    uint32_t* pos32[N_ORD];  // per point: merged position = rank of (value, TR), i.e. of the
                             // packed key (the pair scan's argmin side; < 2^31 for any n)
    int32_t* globals;        // [0] argmax t over all, [1] argmin p over all, [2] generic flag,
                             // [3] number of exact folds last select
    // chunk-local ranks for the 16-bit SIMD pair scan (plan.cu k_scan): the grid's TR range
    // is cut into chunks of lch points (the chunk sort's chunks, whose value-sorted runs
    // list a chunk's points in global merged-position order)
    int lch;
    uint16_t* lr16[N_ORD];   // per TR: competition rank within its chunk (k_sort_chunks)
    uint16_t* lq16[N_ORD];   // per TR: place in its chunk's run (k_sort_chunks)
    uint32_t* cinv[N_ORD];   // per run place: the global merged position (the rank pass)
};

#ifdef __CUDACC__
// kernel<<<g, b, smem, s>>>(args...) with the PDL attribute when pdl is set
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s,
                            bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
#endif

}  // namespace pals

// ---- host-side objects behind the opaque C handles -----------------------
struct pals_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    int num_sms = 148;
    // scratch for host-buffer entry points
    void* d_scratch = nullptr;
    size_t scratch_bytes = 0;
    void* h_pinned = nullptr;
    size_t pinned_bytes = 0;
    void* d_sim_arena = nullptr;  // pals_run_scenarios' staged inputs (reused across calls)
    size_t sim_arena_bytes = 0;
    void* h_sim_streams = nullptr;  // its streamed arrivals: pinned staging + device mirror
    void* d_sim_streams = nullptr;
    size_t sim_stream_bytes = 0;
    int* h_sim_flags = nullptr;     // pinned 1s: the value the chunk-ready flag copies write
    void* replay_cache = nullptr;  // replay.cu
    void* sim_cache = nullptr;     // sim.cu: plant models and select-table sets across calls
    void* one_cache = nullptr;     // replay.cu: single-call candidate sets (pals_select_one)
    int replay_layout = 0;         // PALS_REPLAY_THREAD / PALS_REPLAY_WARP
    int64_t one_server_idle_us = 2000;  // pals_ctx_set_one_server: 0 = one launch per call
    double sim_prep_s = 0.0;       // sim.cu: host setup of the last pals_run_scenarios
    double sim_kernel_ms = -1.0;   // and its k_sim launch (CUDA events)
    int sim_keep_requests = 0;     // pals_sim_keep_requests
    int sim_streaming = 1;         // pals_sim_set_streaming
    std::vector<std::vector<pals_sim_request>> sim_requests;  // per node of the last run
    void* d_front = nullptr;       // frontier.cu scratch
    size_t front_bytes = 0;
};

// Blocking copy ordered on a context stream. A plain cudaMemcpy runs on the legacy
// default stream, which does not order against non-blocking streams (torch's, or
// the context's own), and a pageable H2D may return before its DMA has landed — so
// a kernel queued next on the context stream could read stale bytes.
inline cudaError_t copy_on(cudaStream_t s, void* dst, const void* src, size_t n,
                           cudaMemcpyKind kind) {
    const cudaError_t e = cudaMemcpyAsync(dst, src, n, kind, s);
    return e == cudaSuccess ? cudaStreamSynchronize(s) : e;
}

enum ModelKind { MODEL_ANALYTIC = 0, MODEL_TABLE = 1, MODEL_FOREST = 2 };

struct pals_model {
    pals_ctx* ctx = nullptr;
    uint64_t uid = 0;  // unique per model ever created (cache keys survive pointer reuse)
    ModelKind kind = MODEL_ANALYTIC;
    std::string name;
    pals_profile profile{};
    pals::Analytic an{};
    // table model (host copies + device copies)
    int64_t table_n = 0;
    pals_point* table_pts = nullptr;   // host
    double* table_T = nullptr;         // host
    double* table_P = nullptr;         // host
    // forest model (device arrays), see forest.cu
    void* forest = nullptr;
    pals::Analytic* d_an = nullptr;  // device copy for pals_eval_device
};

struct pals_grid {
    pals_ctx* ctx = nullptr;
    int64_t n = 0;
    pals_point* h_pts = nullptr;  // host copy (validation, table mapping)
    double* cap = nullptr;        // device SoA
    int* batch = nullptr;
    int* tp = nullptr;
    int* ep = nullptr;
    int* dp = nullptr;
    int* inv_tr = nullptr;        // device: TR -> index
    int* canon = nullptr;         // device: first index with an equal point
    int* h_canon = nullptr;       // host copy
};

namespace pals {
// error plumbing (ctx.cu)
int set_error(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
#define PALS_CUDA(call)                                              \
    do {                                                             \
        cudaError_t _e = (call);                                     \
        if (_e != cudaSuccess) return ::pals::cuda_fail(_e, #call);  \
    } while (0)
// model validation against a grid (ctx.cu): reproduces the first exception the
// reference's scorer would throw over the candidates in order.
int validate_points(const pals_model* m, const pals_point* pts, int64_t n);
int validate_point(const pals_model* m, const pals_point& p);
void count_launch(pals_ctx* ctx, int k = 1);
const PlanDev& plan_dev(const pals_plan* p);
int plan_error(const pals_plan* p);
void replay_cache_free(pals_ctx* ctx);
void sim_cache_free(pals_ctx* ctx);
void one_cache_free(pals_ctx* ctx);
void one_server_stop(pals_ctx* ctx);  // replay.cu: ends the resident single-call kernel
uint64_t next_model_uid();
// forest.cu
void forest_free(void* f);
int forest_eval_plan(pals_plan* p, const pals_model* m, pals_ctx* ctx);
int forest_eval_raw(const pals_model* m, pals_ctx* ctx, int64_t n, const double* cap,
                    const int* batch, const int* tp, const int* ep, const int* dp, double* T,
                    double* P, int force_direct);
// plan.cu
const pals_grid* plan_grid(const pals_plan* p);
pals_ctx* plan_ctx(const pals_plan* p);
void* plan_scratch(pals_plan* p, size_t bytes);
// a plan over given (throughput, efficiency) values per grid point (T / P arrays of
// the plan are filled by the caller before pals_plan_prepare); frontier only
int plan_create_values(pals_ctx* ctx, const pals_grid* g, pals_plan** out);
int plan_finish_scores(pals_plan* p);
}  // namespace pals
