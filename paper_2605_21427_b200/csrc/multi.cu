// multi.cu — the multi-GPU driver of pals_gpu.h (BASELINE north_star item 5):
// one worker thread and one pals_ctx per listed device, contiguous shards of the
// queries / traces, no device-to-device traffic until the results, which either land
// directly in the caller's host buffers from each device or are gathered into device 0
// with cudaMemcpyPeerAsync (NVLink / NVSwitch) and read back in one copy.
//
// The reference has no counterpart: its simulator steps nodes sequentially in one
// thread (sim.hpp:243-244) and select_config / control_step are single calls
// (controller.hpp:132, 210). Every shard runs the single-context entry points
// (pals_select / pals_plan_run, pals_replay_ex / pals_replay_device_ex,
// pals_replay_traces), so sharded results equal the one-context results byte for byte.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "pals_internal.cuh"

namespace pals {

struct MultiWorker {
    int rank = 0, device = 0;
    pals_ctx* ctx = nullptr;
    std::thread th;
    std::function<int()> job;
    bool has_job = false;
    int rc = PALS_OK;
    std::string err;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    bool timed = false;
    // select: plan cache per (model, candidate list, coeffs)
    pals_grid* grid = nullptr;
    pals_plan* plan = nullptr;
    uint64_t plan_key = 0;
    // device staging of a shard (gather mode)
    void* d_buf = nullptr;
    size_t buf_bytes = 0;
};

static uint64_t fnv_bytes(uint64_t h, const void* p, size_t n) {
    const unsigned char* b = (const unsigned char*)p;
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ULL;
    return h;
}

static int grow(void** p, size_t* cap, size_t need) {
    if (*cap >= need) return PALS_OK;
    cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    PALS_CUDA(cudaMalloc(p, need));
    *cap = need;
    return PALS_OK;
}

}  // namespace pals

using namespace pals;

struct pals_multi {
    std::vector<MultiWorker*> w;
    std::mutex mu;
    std::condition_variable cv, done_cv;
    int pending = 0;
    bool quit = false;
    int gather = 0;
    std::vector<std::vector<pals_model*>> models;  // [id][rank]
    void* d_gather = nullptr;  // on device 0
    size_t gather_bytes = 0;
    std::vector<double> last_ms;

    // Runs fn(rank) on every worker thread and waits; the first failing rank's code and
    // message become this thread's pals_last_error.
    int run_all(const std::function<int(MultiWorker&)>& fn, bool timed = false) {
        {
            std::unique_lock<std::mutex> l(mu);
            for (auto* x : w) {
                x->job = [x, fn] { return fn(*x); };
                x->has_job = true;
                x->timed = timed;
            }
            pending = (int)w.size();
        }
        cv.notify_all();
        std::unique_lock<std::mutex> l(mu);
        done_cv.wait(l, [&] { return pending == 0; });
        for (auto* x : w)
            if (x->rc != PALS_OK) return set_error(x->rc, x->err);
        return PALS_OK;
    }

    void loop(MultiWorker* x) {
        for (;;) {
            std::function<int()> job;
            {
                std::unique_lock<std::mutex> l(mu);
                cv.wait(l, [&] { return quit || x->has_job; });
                if (quit) return;
                job = std::move(x->job);
                x->has_job = false;
            }
            int rc = cudaSetDevice(x->device) == cudaSuccess
                         ? PALS_OK
                         : set_error(PALS_ERUNTIME, "pals_multi: cudaSetDevice failed");
            if (rc == PALS_OK && x->timed && x->ctx) cudaEventRecord(x->e0, x->ctx->stream);
            if (rc == PALS_OK) rc = job();
            if (rc == PALS_OK && x->timed && x->ctx) {
                cudaEventRecord(x->e1, x->ctx->stream);
                cudaEventSynchronize(x->e1);
            }
            x->rc = rc;
            x->err = rc == PALS_OK ? std::string() : std::string(pals_last_error());
            {
                std::unique_lock<std::mutex> l(mu);
                --pending;
            }
            done_cv.notify_all();
        }
    }

    void collect_ms() {
        last_ms.assign(w.size(), -1.0);
        for (size_t r = 0; r < w.size(); ++r) {
            float ms = -1.0f;
            if (w[r]->e0 && cudaEventElapsedTime(&ms, w[r]->e0, w[r]->e1) == cudaSuccess)
                last_ms[r] = ms;
        }
    }
};

namespace {

// contiguous shard of n items for rank r of R
inline void shard(int64_t n, int r, int R, int64_t* lo, int64_t* hi) {
    *lo = n * r / R;
    *hi = n * (r + 1) / R;
}

std::vector<pals_model*> rank_models(pals_multi* m, int rank, int n, const int32_t* ids,
                                     int* rc) {
    std::vector<pals_model*> out;
    *rc = PALS_OK;
    for (int i = 0; i < n; ++i) {
        if (ids[i] < 0 || ids[i] >= (int)m->models.size()) {
            *rc = set_error(PALS_ECONFIG, "pals_multi: unknown model id");
            return out;
        }
        out.push_back(m->models[ids[i]][rank]);
    }
    return out;
}

// the device-0 gather buffer (allocated by rank 0's thread)
int ensure_gather(pals_multi* m, size_t bytes) {
    return m->run_all([&](MultiWorker& x) {
        return x.rank == 0 ? grow(&m->d_gather, &m->gather_bytes, bytes) : PALS_OK;
    });
}

}  // namespace

extern "C" {

int pals_multi_create(const int32_t* devices, int32_t n, pals_multi** out) {
    if (!devices || n <= 0 || !out) return set_error(PALS_ECONFIG, "pals_multi_create: no devices");
    auto* m = new pals_multi();
    for (int r = 0; r < n; ++r) {
        auto* x = new MultiWorker();
        x->rank = r;
        x->device = devices[r];
        m->w.push_back(x);
    }
    for (auto* x : m->w) x->th = std::thread([m, x] { m->loop(x); });
    int rc = m->run_all([](MultiWorker& x) {
        int r = pals_ctx_create(x.device, &x.ctx);
        if (r) return r;
        PALS_CUDA(cudaEventCreate(&x.e0));
        PALS_CUDA(cudaEventCreate(&x.e1));
        return PALS_OK;
    });
    if (rc == PALS_OK) {
        // peer access from every device to device 0 (the gather target); a device listed
        // twice needs none, and without peer access cudaMemcpyPeerAsync still works
        rc = m->run_all([&](MultiWorker& x) {
            const int d0 = m->w[0]->device;
            int can = 0;
            if (x.device != d0 && cudaDeviceCanAccessPeer(&can, x.device, d0) == cudaSuccess &&
                can) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(d0, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return cuda_fail(e, "cudaDeviceEnablePeerAccess");
                (void)cudaGetLastError();
            }
            return PALS_OK;
        });
    }
    if (rc != PALS_OK) {
        const std::string msg = pals_last_error();
        pals_multi_destroy(m);
        return set_error(rc, msg);
    }
    *out = m;
    return PALS_OK;
}

int pals_multi_destroy(pals_multi* m) {
    if (!m) return PALS_OK;
    m->run_all([m](MultiWorker& x) {
        for (auto& per : m->models) pals_model_destroy(per[x.rank]);
        if (x.plan) pals_plan_destroy(x.plan);
        if (x.grid) pals_grid_destroy(x.grid);
        cudaFree(x.d_buf);
        if (x.rank == 0) cudaFree(m->d_gather);
        if (x.e0) cudaEventDestroy(x.e0);
        if (x.e1) cudaEventDestroy(x.e1);
        pals_ctx_destroy(x.ctx);
        return PALS_OK;
    });
    {
        std::unique_lock<std::mutex> l(m->mu);
        m->quit = true;
    }
    m->cv.notify_all();
    for (auto* x : m->w) {
        x->th.join();
        delete x;
    }
    delete m;
    return PALS_OK;
}

int32_t pals_multi_size(const pals_multi* m) { return m ? (int32_t)m->w.size() : 0; }

pals_ctx* pals_multi_ctx(pals_multi* m, int32_t rank) {
    if (!m || rank < 0 || rank >= (int)m->w.size()) return nullptr;
    return m->w[rank]->ctx;
}

int pals_multi_set_gather(pals_multi* m, int32_t to_device0) {
    if (!m) return set_error(PALS_ECONFIG, "pals_multi_set_gather: null");
    m->gather = to_device0 ? 1 : 0;
    return PALS_OK;
}

int pals_multi_model_analytic(pals_multi* m, const pals_profile* profile,
                              const pals_gpu_spec* gpu, int32_t* id) {
    std::vector<pals_model*> per(m->w.size(), nullptr);
    const int rc = m->run_all([&](MultiWorker& x) {
        return pals_model_analytic(x.ctx, profile, gpu, &per[x.rank]);
    });
    if (rc) {
        for (auto* p : per) pals_model_destroy(p);
        return rc;
    }
    m->models.push_back(per);
    *id = (int32_t)m->models.size() - 1;
    return PALS_OK;
}

int pals_multi_model_table(pals_multi* m, const pals_point* points, const double* t,
                           const double* p, int64_t n, int32_t* id) {
    std::vector<pals_model*> per(m->w.size(), nullptr);
    const int rc = m->run_all([&](MultiWorker& x) {
        return pals_model_table(x.ctx, points, t, p, n, &per[x.rank]);
    });
    if (rc) {
        for (auto* q : per) pals_model_destroy(q);
        return rc;
    }
    m->models.push_back(per);
    *id = (int32_t)m->models.size() - 1;
    return PALS_OK;
}

int pals_multi_select(pals_multi* m, int32_t model, const pals_point* points, int64_t n_points,
                      const pals_coeffs* coeffs, const pals_query* queries, int64_t n,
                      int32_t* index, uint8_t* reason) {
    if (model < 0 || model >= (int)m->models.size())
        return set_error(PALS_ECONFIG, "pals_multi: unknown model id");
    if (n < 0) return set_error(PALS_ECONFIG, "pals_select: negative query count");
    const int R = (int)m->w.size();
    uint64_t key = fnv_bytes(0xcbf29ce484222325ULL, points, (size_t)n_points * sizeof(pals_point));
    key = fnv_bytes(key, coeffs, sizeof *coeffs);
    key = fnv_bytes(key, &model, sizeof model);
    key = fnv_bytes(key, &n_points, sizeof n_points);
    const bool gather = m->gather && n > 0;
    if (gather) {
        const int rc = ensure_gather(m, (size_t)n * 5 + 256);
        if (rc) return rc;
    }
    int32_t* g_idx = (int32_t*)m->d_gather;
    uint8_t* g_rs = gather ? (uint8_t*)(g_idx + n) : nullptr;
    int rc = m->run_all(
        [&](MultiWorker& x) {
            if (!x.plan || x.plan_key != key) {
                if (x.plan) pals_plan_destroy(x.plan);
                if (x.grid) pals_grid_destroy(x.grid);
                x.plan = nullptr;
                x.grid = nullptr;
                int r = pals_grid_points(x.ctx, points, n_points, &x.grid);
                if (r) return r;
                r = pals_plan_create(x.ctx, m->models[model][x.rank], x.grid, coeffs, &x.plan);
                if (r) return r;
                x.plan_key = key;
            }
            int64_t lo, hi;
            shard(n, x.rank, R, &lo, &hi);
            const int64_t k = hi - lo;
            if (k == 0) return pals_select(x.plan, queries, 0, index, reason);  // errors only
            if (!gather) return pals_select(x.plan, queries + lo, k, index + lo, reason + lo);
            // gather mode: the shard's decisions stay on its device, then one peer copy each
            cudaStream_t s = x.ctx->stream;
            int r = grow(&x.d_buf, &x.buf_bytes, (size_t)k * (sizeof(pals_query) + 5) + 512);
            if (r) return r;
            pals_query* dq = (pals_query*)x.d_buf;
            int32_t* di = (int32_t*)(dq + k);
            uint8_t* dr = (uint8_t*)(di + k);
            PALS_CUDA(cudaMemcpyAsync(dq, queries + lo, k * sizeof(pals_query),
                                      cudaMemcpyHostToDevice, s));
            r = pals_plan_run(x.plan, dq, k, di, dr);
            if (r) return r;
            const int d0 = m->w[0]->device;
            PALS_CUDA(cudaMemcpyPeerAsync(g_idx + lo, d0, di, x.device, k * 4, s));
            PALS_CUDA(cudaMemcpyPeerAsync(g_rs + lo, d0, dr, x.device, k, s));
            PALS_CUDA(cudaStreamSynchronize(s));
            return PALS_OK;
        },
        true);
    m->collect_ms();
    if (rc || !gather) return rc;
    // one read-back of the gathered decisions from device 0
    return m->run_all([&](MultiWorker& x) {
        if (x.rank != 0) return PALS_OK;
        PALS_CUDA(cudaMemcpyAsync(index, g_idx, n * 4, cudaMemcpyDeviceToHost, x.ctx->stream));
        PALS_CUDA(cudaMemcpyAsync(reason, g_rs, n, cudaMemcpyDeviceToHost, x.ctx->stream));
        PALS_CUDA(cudaStreamSynchronize(x.ctx->stream));
        return PALS_OK;
    });
}

int pals_multi_replay(pals_multi* m, int32_t n_models, const int32_t* ids,
                      const pals_profile* plant, const pals_gpu_spec* gpu,
                      const pals_coeffs* coeffs, const double* caps, int32_t n_caps,
                      const int32_t* batches, int32_t n_batches, const pals_ctrl_cfg* cfg,
                      const pals_replay_spec* spec, pals_trace_summary* summaries,
                      pals_step_log* logs, pals_step_detail* details) {
    const int R = (int)m->w.size();
    const int64_t n = spec->n_traces;
    const int64_t nl = logs ? std::min<int64_t>(std::max(spec->n_log_traces, 0), n) : 0;
    const size_t steps = (size_t)std::max(spec->n_steps, 0);
    const bool gather = m->gather && n > 0;
    const size_t sb = (size_t)n * sizeof(pals_trace_summary);
    const size_t lb = (size_t)nl * steps * sizeof(pals_step_log);
    const size_t db = details ? (size_t)nl * steps * sizeof(pals_step_detail) : 0;
    const size_t o_l = (sb + 255) & ~(size_t)255, o_d = o_l + ((lb + 255) & ~(size_t)255);
    if (gather) {
        const int rc = ensure_gather(m, o_d + db + 256);
        if (rc) return rc;
    }
    char* g = (char*)m->d_gather;
    int rc = m->run_all(
        [&](MultiWorker& x) {
            int r;
            std::vector<pals_model*> hs = rank_models(m, x.rank, n_models, ids, &r);
            if (r) return r;
            int64_t lo, hi;
            shard(n, x.rank, R, &lo, &hi);
            pals_replay_spec sp = *spec;
            sp.first_trace = spec->first_trace + lo;
            sp.n_traces = hi - lo;
            const int64_t my_nl = std::max<int64_t>(0, std::min(nl - lo, hi - lo));
            sp.n_log_traces = (int32_t)my_nl;
            if (!gather)
                return pals_replay_ex(x.ctx, n_models, hs.data(), plant, gpu, coeffs, caps, n_caps,
                                      batches, n_batches, cfg, &sp,
                                      sp.n_traces ? summaries + lo : summaries,
                                      my_nl ? logs + lo * steps : nullptr,
                                      (my_nl && details) ? details + lo * steps : nullptr);
            const size_t k = (size_t)(hi - lo);
            const size_t ksb = k * sizeof(pals_trace_summary);
            const size_t klb = (size_t)my_nl * steps * sizeof(pals_step_log);
            const size_t kdb = details ? (size_t)my_nl * steps * sizeof(pals_step_detail) : 0;
            const size_t ko_l = (ksb + 255) & ~(size_t)255, ko_d = ko_l + ((klb + 255) & ~(size_t)255);
            r = grow(&x.d_buf, &x.buf_bytes, ko_d + kdb + 256);
            if (r) return r;
            char* b = (char*)x.d_buf;
            if (k == 0) return PALS_OK;
            r = pals_replay_device_ex(x.ctx, n_models, hs.data(), plant, gpu, coeffs, caps, n_caps,
                                      batches, n_batches, cfg, &sp, (pals_trace_summary*)b,
                                      my_nl ? (pals_step_log*)(b + ko_l) : nullptr,
                                      (my_nl && details) ? (pals_step_detail*)(b + ko_d) : nullptr);
            if (r) return r;
            cudaStream_t s = x.ctx->stream;
            const int d0 = m->w[0]->device;
            PALS_CUDA(cudaMemcpyPeerAsync(g + lo * sizeof(pals_trace_summary), d0, b, x.device,
                                          ksb, s));
            if (klb)
                PALS_CUDA(cudaMemcpyPeerAsync(g + o_l + lo * steps * sizeof(pals_step_log), d0,
                                              b + ko_l, x.device, klb, s));
            if (kdb)
                PALS_CUDA(cudaMemcpyPeerAsync(g + o_d + lo * steps * sizeof(pals_step_detail), d0,
                                              b + ko_d, x.device, kdb, s));
            PALS_CUDA(cudaStreamSynchronize(s));
            return PALS_OK;
        },
        true);
    m->collect_ms();
    if (rc || !gather) return rc;
    return m->run_all([&](MultiWorker& x) {
        if (x.rank != 0) return PALS_OK;
        cudaStream_t s = x.ctx->stream;
        PALS_CUDA(cudaMemcpyAsync(summaries, g, sb, cudaMemcpyDeviceToHost, s));
        if (lb) PALS_CUDA(cudaMemcpyAsync(logs, g + o_l, lb, cudaMemcpyDeviceToHost, s));
        if (db) PALS_CUDA(cudaMemcpyAsync(details, g + o_d, db, cudaMemcpyDeviceToHost, s));
        PALS_CUDA(cudaStreamSynchronize(s));
        return PALS_OK;
    });
}

int pals_multi_replay_traces(pals_multi* m, int32_t n_models, const int32_t* ids,
                             const pals_profile* plant, const pals_gpu_spec* gpu,
                             const pals_coeffs* coeffs, const double* caps, int32_t n_caps,
                             const int32_t* batches, int32_t n_batches,
                             const pals_ctrl_cfg* cfg, const pals_trace_batch* batch) {
    if (!batch) return set_error(PALS_ECONFIG, "pals_replay_traces: null argument");
    const pals_trace_batch& B = *batch;
    const int R = (int)m->w.size();
    const int64_t n = B.n_traces;
    if (n < 0 || (n > 0 && !B.traces)) return set_error(PALS_ECONFIG, "pals_replay_traces: bad batch");
    const int64_t nl = B.logs ? std::min<int64_t>(std::max(B.n_log_traces, 0), n) : 0;
    const size_t steps = (size_t)std::max(B.n_steps, 0);
    int rc = m->run_all(
        [&](MultiWorker& x) {
            int r;
            std::vector<pals_model*> hs = rank_models(m, x.rank, n_models, ids, &r);
            if (r) return r;
            int64_t lo, hi;
            shard(n, x.rank, R, &lo, &hi);
            const int64_t k = hi - lo;
            if (k == 0) return PALS_OK;
            // only the window of the signal array this shard reads travels to its device
            int64_t s_lo = B.n_signal, s_hi = 0;
            for (int64_t i = lo; i < hi; ++i) {
                const pals_trace& t = B.traces[i];
                if (t.n_load > 0) {
                    s_lo = std::min(s_lo, t.load_off);
                    s_hi = std::max(s_hi, t.load_off + t.n_load);
                }
                if (t.n_budget > 0) {
                    s_lo = std::min(s_lo, t.budget_off);
                    s_hi = std::max(s_hi, t.budget_off + t.n_budget);
                }
            }
            if (s_hi <= s_lo) s_lo = s_hi = 0;
            std::vector<pals_trace> tr(B.traces + lo, B.traces + hi);
            for (auto& t : tr) {
                t.load_off -= s_lo;
                t.budget_off -= s_lo;
            }
            pals_trace_batch b = B;
            b.n_traces = k;
            b.traces = tr.data();
            b.signal = B.signal ? B.signal + s_lo : nullptr;
            b.n_signal = s_hi - s_lo;
            b.init = B.init ? B.init + lo : nullptr;
            b.init_plant = B.init_plant ? B.init_plant + lo : nullptr;
            b.summaries = B.summaries + lo;
            b.final_state = B.final_state ? B.final_state + lo : nullptr;
            b.final_plant = B.final_plant ? B.final_plant + lo : nullptr;
            const int64_t my_nl = std::max<int64_t>(0, std::min(nl - lo, k));
            b.n_log_traces = (int32_t)my_nl;
            b.logs = my_nl ? B.logs + lo * steps : nullptr;
            b.details = (my_nl && B.details) ? B.details + lo * steps : nullptr;
            r = pals_replay_traces(x.ctx, n_models, hs.data(), plant, gpu, coeffs, caps, n_caps,
                                   batches, n_batches, cfg, &b);
            if (r) {
                // report the trace by its index in the caller's batch
                std::string msg = pals_last_error();
                const std::string tag = "trace ";
                const size_t at = msg.find(tag);
                if (at != std::string::npos) {
                    size_t e = at + tag.size();
                    int64_t local = 0;
                    while (e < msg.size() && msg[e] >= '0' && msg[e] <= '9')
                        local = local * 10 + (msg[e++] - '0');
                    msg = msg.substr(0, at + tag.size()) + std::to_string(lo + local) + msg.substr(e);
                }
                return set_error(r, msg);
            }
            return PALS_OK;
        },
        true);
    m->collect_ms();
    return rc;
}

int pals_multi_last_ms(const pals_multi* m, double* ms) {
    if (!m || !ms) return set_error(PALS_ECONFIG, "pals_multi_last_ms: null");
    for (size_t r = 0; r < m->w.size(); ++r) ms[r] = r < m->last_ms.size() ? m->last_ms[r] : -1.0;
    return PALS_OK;
}

}  // extern "C"
