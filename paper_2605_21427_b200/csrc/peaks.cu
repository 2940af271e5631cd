// peaks.cu — microbenchmarks for the roofline denominators this path needs.
// MEASURED_PEAKS.json has HBM and bf16 tensor peaks only; the select scan is
// bound by the integer ALU pipe and the controller replay by FP64 issue, so
// bench.py measures those two peaks on the same box with these kernels.
#include "pals_internal.cuh"

namespace pals {

// The pair scan's class-A/C instruction mix (k_scan, plan.cu): per (config, query)
// pair d = K - r (IMAD.IADD), v = pos | (d & 0x80000000) (LOP3), and one VIMNMX3
// per two pairs; 8 independent query chains per thread. Reported as 2 "int ops" per
// pair (the algorithmic compare + min), so bench.py's achieved / peak is the scan's
// pair rate over this chain's pair rate.
__global__ void __launch_bounds__(256) k_peak_int(uint32_t* out, int iters, uint32_t seed) {
    uint32_t K[8], acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        K[q] = (seed * (q + 3) + threadIdx.x) & 0xFFFFF;
        acc[q] = 0xFFFFFFFFu;
    }
    uint32_t k = seed ^ (blockIdx.x * 977u + threadIdx.x);
    for (int i = 0; i < iters; ++i) {
        const uint32_t r0 = k & 0xFFFFF, p0 = k >> 12, r1 = (k ^ 0x9E3779B9u) & 0xFFFFF,
                       p1 = (k + 0x7F4A7C15u) >> 12;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t v0 = p0 | ((K[q] - r0) & 0x80000000u);
            const uint32_t v1 = p1 | ((K[q] - r1) & 0x80000000u);
            acc[q] = __vimin3_u32(acc[q], v0, v1);
        }
        k += 0x61C88647u;
    }
    uint32_t r = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) r ^= acc[q];
    if (r == 0x12345678u) out[0] = r;
}

// FP64 fused multiply-add chains (8 independent per thread).
__global__ void __launch_bounds__(256) k_peak_fp64(double* out, int iters, double seed) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = seed + q + threadIdx.x * 1e-9;
    const double m = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = __fma_rn(a[q], m, c);
    }
    double r = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) r += a[q];
    if (r == 1.2345) out[0] = r;
}

}  // namespace pals

using namespace pals;

extern "C" int pals_measure_peaks(pals_ctx* ctx, double* int_ops_per_s, double* fp64_flops_per_s) {
    PALS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    void* buf = nullptr;
    PALS_CUDA(cudaMalloc(&buf, 64));
    cudaEvent_t e0, e1;
    PALS_CUDA(cudaEventCreate(&e0));
    PALS_CUDA(cudaEventCreate(&e1));
    const int blocks = ctx->num_sms * 8, threads = 256;
    const int iters_i = 4096, iters_d = 2048;
    float best_i = 1e30f, best_d = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, s);
        k_peak_int<<<blocks, threads, 0, s>>>((uint32_t*)buf, iters_i, 12345u + rep);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best_i = ms < best_i ? ms : best_i;
        cudaEventRecord(e0, s);
        k_peak_fp64<<<blocks, threads, 0, s>>>((double*)buf, iters_d, 1.0 + rep);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best_d = ms < best_d ? ms : best_d;
    }
    count_launch(ctx, 8);
    const cudaError_t e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    if (e != cudaSuccess) return cuda_fail(e, "pals_measure_peaks");
    const double threads_total = (double)blocks * threads;
    // per inner iteration: 8 chains x 2 pairs x 2 algorithmic ops (compare + min) = 32
    *int_ops_per_s = threads_total * iters_i * 32.0 / (best_i * 1e-3);
    // 8 DFMA = 16 flops per iteration
    *fp64_flops_per_s = threads_total * iters_d * 16.0 / (best_d * 1e-3);
    return PALS_OK;
}
