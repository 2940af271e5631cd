// frontier.cu — build_frontier (pareto.hpp:31-59) from a prepared plan's rank keys.
//
// The reference sorts by (throughput, efficiency, cap, batch) ascending, collapses
// exact (throughput, efficiency) ties onto the first (lower-cap, then smaller-batch)
// point and keeps, sweeping from the high-throughput end, every point whose
// efficiency beats everything after it. With K1's competition ranks (rt = number
// of points with strictly greater throughput, re = same for efficiency) and the
// grid's (cap, batch, index) rank TR, the plan's packed keys are
// keyT = rt << b | TR and keyE = re << b | TR, and the sorted sequence is ascending
// (rt, re, TR) read backwards. A point survives iff it is the minimum keyE of its
// throughput group G[rt] (highest efficiency, then lowest (cap, batch): the tie
// collapse) and its re is strictly below the minimum re over all groups with
// smaller rt (higher throughput): the sweep's `efficiency > best_eff`. So:
//   k_front_group   G[rt] = min keyE over the group            (one atomicMin per point)
//   k_front_tiles   per-tile min of G                           (4096 ranks per CTA)
//   k_front_scan    exclusive prefix-min of G across tiles, survivor flags and counts
//   k_front_compact survivors in descending rt = ascending throughput (the reference's
//                   output order), point index = inv_tr[TR]
// Exact full ties (equal throughput, efficiency, cap and batch) resolve to the lower
// grid index; std::sort leaves their order unspecified.
#include <algorithm>
#include <vector>

#include "pals_internal.cuh"

using namespace pals;

namespace {

constexpr int kTile = 4096;
constexpr int kThreads = 1024;
constexpr int kPer = kTile / kThreads;

__device__ __forceinline__ uint64_t plan_key(const PlanDev& d, int o, int64_t i) {
    return d.wide ? d.key64[o][i] : (uint64_t)d.key32[o][i];
}

__global__ void k_front_group(PlanDev d, unsigned long long* G) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t rt = plan_key(d, ORD_T, i) >> d.tr_bits;
        atomicMin(&G[rt], (unsigned long long)plan_key(d, ORD_E, i));
    }
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return b < a ? b : a; }

// block-wide exclusive prefix of a per-thread value (min or sum), 1024 threads
template <bool kMin>
__device__ __forceinline__ uint64_t block_exclusive(uint64_t x, uint64_t ident, uint64_t* sm,
                                                    uint64_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t inc = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc = kMin ? umin64(inc, y) : inc + y;
    }
    uint64_t exc = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) exc = ident;
    if (lane == 31) sm[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint64_t v = sm[lane];
        uint64_t vi = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, vi, off);
            if (lane >= off) vi = kMin ? umin64(vi, y) : vi + y;
        }
        uint64_t ve = __shfl_up_sync(0xffffffffu, vi, 1);
        if (lane == 0) ve = ident;
        sm[32 + lane] = ve;
        if (lane == 31) sm[64] = vi;
    }
    __syncthreads();
    const uint64_t pre = sm[32 + w];
    if (total) *total = sm[64];
    const uint64_t r = kMin ? umin64(pre, exc) : pre + exc;
    __syncthreads();  // sm reusable by the caller
    return r;
}

__global__ void __launch_bounds__(kThreads) k_front_tiles(const uint64_t* G, int64_t n,
                                                          uint64_t* tmin) {
    __shared__ uint64_t sm[80];
    const int64_t base = (int64_t)blockIdx.x * kTile;
    uint64_t m = ~0ull;
    for (int k = 0; k < kPer; ++k) {
        const int64_t r = base + (int64_t)threadIdx.x * kPer + k;
        if (r < n) m = umin64(m, G[r]);
    }
    uint64_t tot;
    block_exclusive<true>(m, ~0ull, sm, &tot);
    if (threadIdx.x == 0) tmin[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kThreads) k_front_scan(const uint64_t* G, int64_t n,
                                                         const uint64_t* tmin, int tr_bits,
                                                         const int* inv_tr, const double* ef,
                                                         uint8_t* flag, uint32_t* tcount) {
    const uint64_t mask = tr_bits == 32 ? 0xFFFFFFFFull : 0xFFFFull;
    __shared__ uint64_t sm[80];
    __shared__ uint64_t carry_s;
    const int64_t base = (int64_t)blockIdx.x * kTile;
    // carry-in: min over all earlier tiles
    uint64_t c = ~0ull;
    for (int t = threadIdx.x; t < (int)blockIdx.x; t += blockDim.x) c = umin64(c, tmin[t]);
    uint64_t ctot;
    block_exclusive<true>(c, ~0ull, sm, &ctot);
    if (threadIdx.x == 0) carry_s = ctot;
    __syncthreads();
    uint64_t v[kPer];
    uint64_t m = ~0ull;
    for (int k = 0; k < kPer; ++k) {
        const int64_t r = base + (int64_t)threadIdx.x * kPer + k;
        v[k] = r < n ? G[r] : ~0ull;
        m = umin64(m, v[k]);
    }
    uint64_t pre = umin64(carry_s, block_exclusive<true>(m, ~0ull, sm, nullptr));
    uint32_t cnt = 0;
    for (int k = 0; k < kPer; ++k) {
        const int64_t r = base + (int64_t)threadIdx.x * kPer + k;
        // group r exists, its efficiency rank beats every higher-throughput group, and
        // its efficiency beats the sweep's initial best_eff = -1.0 (pareto.hpp:50)
        const bool s = v[k] != ~0ull && (v[k] >> tr_bits) < (pre >> tr_bits) &&
                       ef[inv_tr[v[k] & mask]] > -1.0;
        if (r < n) flag[r] = s ? 1 : 0;
        cnt += s;
        pre = umin64(pre, v[k]);
    }
    uint64_t tot;
    block_exclusive<false>(cnt, 0, sm, &tot);
    if (threadIdx.x == 0) tcount[blockIdx.x] = (uint32_t)tot;
}

__global__ void __launch_bounds__(kThreads) k_front_compact(const uint64_t* G, int64_t n,
                                                            const uint8_t* flag,
                                                            const uint32_t* tcount, int ntiles,
                                                            const int* inv_tr, uint64_t tr_mask,
                                                            int32_t* out_idx, int64_t* out_n) {
    __shared__ uint64_t sm[80];
    const int64_t base = (int64_t)blockIdx.x * kTile;
    // survivors of later tiles (lower throughput) come first in the output
    uint64_t later = 0, all = 0;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
        all += tcount[t];
        if (t > (int)blockIdx.x) later += tcount[t];
    }
    uint64_t later_tot, all_tot;
    block_exclusive<false>(later, 0, sm, &later_tot);
    block_exclusive<false>(all, 0, sm, &all_tot);
    if (blockIdx.x == 0 && threadIdx.x == 0) *out_n = (int64_t)all_tot;
    uint8_t f[kPer];
    uint32_t cnt = 0;
    for (int k = 0; k < kPer; ++k) {
        const int64_t r = base + (int64_t)threadIdx.x * kPer + k;
        f[k] = r < n ? flag[r] : 0;
        cnt += f[k];
    }
    uint64_t tile_tot;
    uint64_t inc = block_exclusive<false>(cnt, 0, sm, &tile_tot);
    for (int k = 0; k < kPer; ++k) {
        const int64_t r = base + (int64_t)threadIdx.x * kPer + k;
        if (!f[k]) continue;
        ++inc;  // inclusive count of survivors at ranks <= r within the tile
        const uint64_t pos = later_tot + (tile_tot - inc);
        out_idx[pos] = inv_tr[G[r] & tr_mask];
    }
}

int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, what);
    return PALS_OK;
}

// async on the plan's context stream; the plan must be prepared (same stream)
int frontier_launch(pals_plan* p, int32_t* d_idx, int64_t* d_n) {
    pals_ctx* ctx = plan_ctx(p);
    const PlanDev& d = plan_dev(p);
    const int64_t n = d.n;
    const int ntiles = (int)((n + kTile - 1) / kTile);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t need = al(8 * (size_t)n) + al((size_t)n) + al(8 * (size_t)ntiles) +
                        al(4 * (size_t)ntiles);
    if (ctx->front_bytes < need) {
        cudaFree(ctx->d_front);
        ctx->d_front = nullptr;
        ctx->front_bytes = 0;
        PALS_CUDA(cudaMalloc(&ctx->d_front, need));
        ctx->front_bytes = need;
    }
    char* b = (char*)ctx->d_front;
    uint64_t* G = (uint64_t*)b; b += al(8 * (size_t)n);
    uint8_t* flag = (uint8_t*)b; b += al((size_t)n);
    uint64_t* tmin = (uint64_t*)b; b += al(8 * (size_t)ntiles);
    uint32_t* tcount = (uint32_t*)b;
    cudaStream_t s = ctx->stream;
    PALS_CUDA(cudaMemsetAsync(G, 0xFF, 8 * (size_t)n, s));
    const int gb = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 16 * ctx->num_sms));
    k_front_group<<<gb, 256, 0, s>>>(d, (unsigned long long*)G);
    k_front_tiles<<<ntiles, kThreads, 0, s>>>(G, n, tmin);
    k_front_scan<<<ntiles, kThreads, 0, s>>>(G, n, tmin, d.tr_bits, d.inv_tr, d.ef, flag,
                                             tcount);
    const uint64_t mask = d.wide ? 0xFFFFFFFFull : 0xFFFFull;
    k_front_compact<<<ntiles, kThreads, 0, s>>>(G, n, flag, tcount, ntiles, d.inv_tr, mask,
                                                d_idx, d_n);
    count_launch(ctx, 4);
    return check_launch("frontier");
}

}  // namespace

extern "C" {

int pals_plan_frontier_device(pals_plan* p, int32_t* d_idx, int64_t* d_n) {
    if (!p || !d_idx || !d_n) return set_error(PALS_ECONFIG, "pals_plan_frontier: null argument");
    if (plan_error(p)) return pals_plan_prepare(p);  // reports the plan's error
    PALS_CUDA(cudaSetDevice(plan_ctx(p)->device));
    const int rc = pals_plan_prepare(p);
    return rc ? rc : frontier_launch(p, d_idx, d_n);
}

int pals_plan_frontier(pals_plan* p, int32_t* idx, int64_t* n_out) {
    if (!p || !idx || !n_out) return set_error(PALS_ECONFIG, "pals_plan_frontier: null argument");
    if (plan_error(p)) return pals_plan_prepare(p);
    pals_ctx* ctx = plan_ctx(p);
    PALS_CUDA(cudaSetDevice(ctx->device));
    const int64_t n = plan_dev(p).n;
    int32_t* d_idx = (int32_t*)plan_scratch(p, 4 * (size_t)std::max<int64_t>(1, n) + 16);
    if (!d_idx) return set_error(PALS_ERUNTIME, "pals_plan_frontier: out of device memory");
    int64_t* d_n = (int64_t*)(((uintptr_t)(d_idx + std::max<int64_t>(1, n)) + 7) & ~(uintptr_t)7);
    int rc = pals_plan_frontier_device(p, d_idx, d_n);
    if (rc == PALS_OK) {
        cudaStream_t s = ctx->stream;
        cudaError_t e = cudaMemcpyAsync(n_out, d_n, 8, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e == cudaSuccess && *n_out > 0)
            e = copy_on(s, idx, d_idx, 4 * (size_t)*n_out, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = cuda_fail(e, "pals_plan_frontier");
    }
    return rc;
}

int pals_frontier_values(pals_ctx* ctx, const pals_point* points, const double* throughput_tps,
                         const double* efficiency_tpj, int64_t n, int32_t* idx, int64_t* n_out) {
    if (!ctx || !n_out || (n > 0 && (!points || !throughput_tps || !efficiency_tpj || !idx)))
        return set_error(PALS_ECONFIG, "pals_frontier_values: null argument");
    if (n <= 0) return set_error(PALS_ECONFIG, "build_frontier: no points");
    pals_grid* g = nullptr;
    int rc = pals_grid_points(ctx, points, n, &g);
    if (rc) return rc;
    pals_plan* p = nullptr;
    rc = plan_create_values(ctx, g, &p);
    if (rc) {
        pals_grid_destroy(g);
        return rc;
    }
    const PlanDev& d = plan_dev(p);
    cudaError_t e = copy_on(ctx->stream, d.T, throughput_tps, 8 * (size_t)n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = copy_on(ctx->stream, d.P, efficiency_tpj, 8 * (size_t)n, cudaMemcpyHostToDevice);
    rc = e == cudaSuccess ? pals_plan_frontier(p, idx, n_out) : cuda_fail(e, "pals_frontier_values");
    pals_plan_destroy(p);
    pals_grid_destroy(g);
    return rc;
}

}  // extern "C"
