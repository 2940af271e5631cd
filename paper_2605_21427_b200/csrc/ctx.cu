// ctx.cu — contexts, errors, models, grids (the object side of pals_gpu.h).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#include "pals_internal.cuh"

namespace pals {

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return set_error(PALS_ERUNTIME, std::string("CUDA error ") + cudaGetErrorString(e) +
                                        " at " + where);
}

void count_launch(pals_ctx* ctx, int k) { ctx->launches += k; }

uint64_t next_model_uid() {
    static std::atomic<uint64_t> uid{1};
    return uid++;
}

// OperatingPoint::validate (types.hpp:117-123) then the comm_fixed_by_tp lookup
// (model.hpp:56-59), i.e. the first exception analytic_scorer throws for p.
int validate_point(const pals_model* m, const pals_point& p) {
    if (m->kind == MODEL_ANALYTIC) {
        if (p.cap_watts < m->an.min_cap || p.cap_watts > m->an.max_cap)
            return set_error(PALS_ERANGE, "OperatingPoint: cap outside platform range");
        if (p.batch < 1) return set_error(PALS_ECONFIG, "OperatingPoint: batch must be >= 1");
        if (p.tp < 1 || p.ep < 1 || p.dp < 1)
            return set_error(PALS_ECONFIG, "OperatingPoint: parallel degrees must be >= 1");
        bool found = false;
        for (int i = 0; i < m->an.n_tp; ++i) found |= m->an.tp_keys[i] == p.tp;
        if (!found)
            return set_error(PALS_ECONFIG, m->name + ": no comm cost calibrated for tp=" +
                                               std::to_string(p.tp));
        if (p.dp > kMaxDp)
            return set_error(PALS_ECONFIG, "pals: dp above " + std::to_string(kMaxDp) +
                                               " is not supported");
        return PALS_OK;
    }
    if (m->kind == MODEL_TABLE) {
        for (int64_t i = 0; i < m->table_n; ++i) {
            const pals_point& q = m->table_pts[i];
            if (q.cap_watts == p.cap_watts && q.batch == p.batch && q.tp == p.tp &&
                q.ep == p.ep && q.dp == p.dp)
                return PALS_OK;
        }
        return set_error(PALS_ECONFIG, "unscored candidate");
    }
    return PALS_OK;  // forest: PredictorBundle::predict accepts any point (forest.hpp:227)
}

int validate_points(const pals_model* m, const pals_point* pts, int64_t n) {
    if (m->kind == MODEL_TABLE) {
        // hash lookup instead of the O(n^2) scan; same first-failure semantics
        struct H {
            size_t operator()(const std::string& s) const { return std::hash<std::string>()(s); }
        };
        std::unordered_map<std::string, int64_t> idx;
        idx.reserve((size_t)m->table_n * 2);
        for (int64_t i = 0; i < m->table_n; ++i)
            idx.emplace(std::string((const char*)&m->table_pts[i], sizeof(pals_point)), i);
        for (int64_t i = 0; i < n; ++i) {
            pals_point q = pts[i];
            if (q.cap_watts == 0.0) q.cap_watts = 0.0;
            if (!idx.count(std::string((const char*)&q, sizeof(pals_point))))
                return validate_point(m, pts[i]);
        }
        return PALS_OK;
    }
    for (int64_t i = 0; i < n; ++i) {
        const int rc = validate_point(m, pts[i]);
        if (rc != PALS_OK) return rc;
    }
    return PALS_OK;
}

}  // namespace pals

using namespace pals;

extern "C" {

const char* pals_last_error(void) { return g_last_error.c_str(); }
int pals_abi_version(void) { return PALS_ABI_VERSION; }

int pals_ctx_create(int device, pals_ctx** out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return set_error(PALS_ERUNTIME, "pals: no CUDA device available (the GPU path has no "
                                        "CPU fallback)");
    if (device < 0 || device >= n) return set_error(PALS_ECONFIG, "pals: bad device ordinal");
    PALS_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    PALS_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return set_error(PALS_ERUNTIME, std::string("pals: built for sm_100a, found ") +
                                            prop.name);
    auto* c = new pals_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    PALS_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    *out = c;
    return PALS_OK;
}

int pals_ctx_destroy(pals_ctx* c) {
    if (!c) return PALS_OK;
    cudaSetDevice(c->device);
    replay_cache_free(c);
    one_cache_free(c);
    sim_cache_free(c);
    if (c->d_scratch) cudaFree(c->d_scratch);
    if (c->d_front) cudaFree(c->d_front);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    if (c->d_sim_arena) cudaFree(c->d_sim_arena);
    if (c->h_sim_streams) cudaFreeHost(c->h_sim_streams);
    if (c->d_sim_streams) cudaFree(c->d_sim_streams);
    if (c->h_sim_flags) cudaFreeHost(c->h_sim_flags);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
    return PALS_OK;
}

int pals_ctx_set_stream(pals_ctx* c, void* s) {
    c->stream = s ? (cudaStream_t)s : c->own_stream;
    return PALS_OK;
}

void* pals_ctx_stream(pals_ctx* c) { return (void*)c->stream; }

int pals_ctx_sync(pals_ctx* c) {
    PALS_CUDA(cudaStreamSynchronize(c->stream));
    return PALS_OK;
}

int64_t pals_ctx_launch_count(pals_ctx* c) { return c->launches; }

int pals_ctx_set_one_server(pals_ctx* c, int64_t idle_us) {
    if (!c) return set_error(PALS_ECONFIG, "pals_ctx_set_one_server: null context");
    if (idle_us < 0) return set_error(PALS_ECONFIG, "pals_ctx_set_one_server: negative idle time");
    one_server_stop(c);
    c->one_server_idle_us = idle_us;
    return PALS_OK;
}

int pals_ctx_set_replay_layout(pals_ctx* c, int32_t layout) {
    if (!c) return set_error(PALS_ECONFIG, "pals_ctx_set_replay_layout: null context");
    if (layout != PALS_REPLAY_THREAD && layout != PALS_REPLAY_WARP)
        return set_error(PALS_ECONFIG, "pals_ctx_set_replay_layout: unknown layout");
    c->replay_layout = layout;
    return PALS_OK;
}

int pals_model_analytic(pals_ctx* ctx, const pals_profile* prof, const pals_gpu_spec* gpu,
                        pals_model** out) {
    if (!prof || !gpu) return set_error(PALS_ECONFIG, "pals_model_analytic: null argument");
    if (prof->n_tp < 0 || prof->n_tp > PALS_MAX_TP_KEYS)
        return set_error(PALS_ECONFIG, "pals_model_analytic: n_tp out of range");
    auto* m = new pals_model();
    m->ctx = ctx;
    m->uid = next_model_uid();
    m->kind = MODEL_ANALYTIC;
    m->profile = *prof;
    m->name = std::string(prof->name, strnlen(prof->name, sizeof(prof->name)));
    Analytic& a = m->an;
    a.compute_fixed = prof->compute_fixed;
    a.compute_per_seq = prof->compute_per_seq;
    a.comm_per_seq = prof->comm_per_seq;
    a.knee_watts = prof->knee_watts;
    a.compute_power_base = prof->compute_power_base;
    a.compute_power_per_seq = prof->compute_power_per_seq;
    a.comm_power = prof->comm_power;
    a.overlap = prof->overlap;
    a.min_cap = gpu->min_cap_watts;
    a.max_cap = gpu->max_cap_watts;
    a.max_frequency = gpu->max_frequency;
    a.n_tp = prof->n_tp;
    for (int i = 0; i < prof->n_tp; ++i) {
        a.tp_keys[i] = prof->tp_keys[i];
        a.comm_fixed[i] = prof->comm_fixed[i];
    }
    // std::pow(internode_factor, dp - 1) (model.hpp:64): computed by the host libm
    // exactly as the reference computes it, then looked up on the device.
    a.pow_dp[0] = std::nan("");
    for (int d = 1; d <= kMaxDp; ++d) a.pow_dp[d] = std::pow(prof->internode_factor, d - 1);
    *out = m;
    return PALS_OK;
}

int pals_model_table(pals_ctx* ctx, const pals_point* pts, const double* t, const double* p,
                     int64_t n, pals_model** out) {
    if (n < 0 || (n > 0 && (!pts || !t || !p)))
        return set_error(PALS_ECONFIG, "pals_model_table: bad arguments");
    auto* m = new pals_model();
    m->ctx = ctx;
    m->uid = next_model_uid();
    m->kind = MODEL_TABLE;
    m->name = "table";
    m->table_n = n;
    m->table_pts = new pals_point[n > 0 ? n : 1];
    m->table_T = new double[n > 0 ? n : 1];
    m->table_P = new double[n > 0 ? n : 1];
    for (int64_t i = 0; i < n; ++i) {
        m->table_pts[i] = pts[i];
        m->table_T[i] = t[i];
        m->table_P[i] = p[i];
    }
    *out = m;
    return PALS_OK;
}


int pals_model_destroy(pals_model* m) {
    if (!m) return PALS_OK;
    delete[] m->table_pts;
    delete[] m->table_T;
    delete[] m->table_P;
    if (m->forest) forest_free(m->forest);
    if (m->d_an) cudaFree(m->d_an);
    delete m;
    return PALS_OK;
}

static int grid_finish(pals_ctx* ctx, pals_grid* g) {
    const int64_t n = g->n;
    std::vector<double> cap(n);
    std::vector<int> b(n), tp(n), ep(n), dp(n);
    for (int64_t i = 0; i < n; ++i) {
        cap[i] = g->h_pts[i].cap_watts;
        b[i] = g->h_pts[i].batch;
        tp[i] = g->h_pts[i].tp;
        ep[i] = g->h_pts[i].ep;
        dp[i] = g->h_pts[i].dp;
    }
    // TR: rank in (cap asc, batch asc, index asc) — the better_candidate tie order
    // (controller.hpp:123-124) with the sequential fold's keep-the-earlier rule.
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        if (cap[x] != cap[y]) return cap[x] < cap[y];
        return b[x] < b[y];
    });
    // canon: first index with an equal point (OperatingPoint::operator== types.hpp:125-128)
    g->h_canon = new int[n > 0 ? n : 1];
    {
        std::unordered_map<std::string, int> first;
        first.reserve((size_t)n * 2);
        for (int64_t i = 0; i < n; ++i) {
            pals_point q = g->h_pts[i];
            if (q.cap_watts == 0.0) q.cap_watts = 0.0;
            auto it = first.emplace(std::string((const char*)&q, sizeof q), (int)i).first;
            g->h_canon[i] = it->second;
        }
    }
    const size_t nb = (size_t)(n > 0 ? n : 1);
    PALS_CUDA(cudaMalloc(&g->cap, nb * sizeof(double)));
    PALS_CUDA(cudaMalloc(&g->batch, nb * sizeof(int)));
    PALS_CUDA(cudaMalloc(&g->tp, nb * sizeof(int)));
    PALS_CUDA(cudaMalloc(&g->ep, nb * sizeof(int)));
    PALS_CUDA(cudaMalloc(&g->dp, nb * sizeof(int)));
    PALS_CUDA(cudaMalloc(&g->inv_tr, nb * sizeof(int)));
    PALS_CUDA(cudaMalloc(&g->canon, nb * sizeof(int)));
    if (n > 0) {
        PALS_CUDA(copy_on(ctx->stream, g->cap, cap.data(), n * sizeof(double), cudaMemcpyHostToDevice));
        PALS_CUDA(copy_on(ctx->stream, g->batch, b.data(), n * sizeof(int), cudaMemcpyHostToDevice));
        PALS_CUDA(copy_on(ctx->stream, g->tp, tp.data(), n * sizeof(int), cudaMemcpyHostToDevice));
        PALS_CUDA(copy_on(ctx->stream, g->ep, ep.data(), n * sizeof(int), cudaMemcpyHostToDevice));
        PALS_CUDA(copy_on(ctx->stream, g->dp, dp.data(), n * sizeof(int), cudaMemcpyHostToDevice));
        PALS_CUDA(copy_on(ctx->stream, g->inv_tr, order.data(), n * sizeof(int), cudaMemcpyHostToDevice));
        PALS_CUDA(copy_on(ctx->stream, g->canon, g->h_canon, n * sizeof(int), cudaMemcpyHostToDevice));
    }
    return PALS_OK;
}

int pals_grid_points(pals_ctx* ctx, const pals_point* pts, int64_t n, pals_grid** out) {
    if (n < 0 || (n > 0 && !pts)) return set_error(PALS_ECONFIG, "pals_grid_points: bad args");
    if (n > (int64_t)1 << 30) return set_error(PALS_ECONFIG, "pals_grid_points: grid too large");
    PALS_CUDA(cudaSetDevice(ctx->device));
    auto* g = new pals_grid();
    g->ctx = ctx;
    g->n = n;
    g->h_pts = new pals_point[n > 0 ? n : 1];
    if (n > 0) std::memcpy(g->h_pts, pts, n * sizeof(pals_point));
    const int rc = grid_finish(ctx, g);
    if (rc != PALS_OK) {
        pals_grid_destroy(g);
        return rc;
    }
    *out = g;
    return PALS_OK;
}

int pals_grid_axes(pals_ctx* ctx, const double* caps, int32_t nc, const int32_t* batches,
                   int32_t nb, const int32_t* tps, int32_t nt, const int32_t* eps, int32_t ne,
                   const int32_t* dps, int32_t nd, pals_grid** out) {
    if (nc < 0 || nb < 0 || nt < 0 || ne < 0 || nd < 0)
        return set_error(PALS_ECONFIG, "pals_grid_axes: negative axis length");
    std::vector<pals_point> pts;
    pts.reserve((size_t)nc * nb * nt * ne * nd);
    for (int a = 0; a < nc; ++a)
        for (int b = 0; b < nb; ++b)
            for (int t = 0; t < nt; ++t)
                for (int e = 0; e < ne; ++e)
                    for (int d = 0; d < nd; ++d) {
                        pals_point p;
                        p.cap_watts = caps[a];
                        p.batch = batches[b];
                        p.tp = tps[t];
                        p.ep = eps[e];
                        p.dp = dps[d];
                        pts.push_back(p);
                    }
    return pals_grid_points(ctx, pts.data(), (int64_t)pts.size(), out);
}

int64_t pals_grid_size(const pals_grid* g) { return g ? g->n : -1; }

int pals_grid_destroy(pals_grid* g) {
    if (!g) return PALS_OK;
    cudaFree(g->cap);
    cudaFree(g->batch);
    cudaFree(g->tp);
    cudaFree(g->ep);
    cudaFree(g->dp);
    cudaFree(g->inv_tr);
    cudaFree(g->canon);
    delete[] g->h_pts;
    delete[] g->h_canon;
    delete g;
    return PALS_OK;
}

}  // extern "C"
