// Microbenchmark: throughput of the scan's per-pair instruction mixes on one B200.
//  A: ISETP + predicated VIMNMX (current k_scan class A)
//  B: IMAD (d = K - r) + LOP3 (v = q | (d & 0x80000000)) + VIMNMX3 over 2 configs
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 4) mixA(const unsigned* __restrict__ keys, int iters,
                                               unsigned* out) {
    __shared__ unsigned se[256], st[256];
    se[threadIdx.x] = keys[threadIdx.x];
    st[threadIdx.x] = keys[256 + threadIdx.x];
    __syncthreads();
    unsigned thr[8], be[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { thr[q] = keys[512 + q * 32 + (threadIdx.x & 31)]; be[q] = ~0u; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int c = 0; c < 256; c += 4) {
            uint4 e = *reinterpret_cast<const uint4*>(se + c);
            uint4 t = *reinterpret_cast<const uint4*>(st + c);
            unsigned ev[4] = {e.x, e.y, e.z, e.w}, tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
            for (int v = 0; v < 4; ++v)
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (tv[v] <= thr[q]) be[q] = min(be[q], ev[v]);
        }
    }
    unsigned r = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) r ^= be[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void __launch_bounds__(256, 4) mixB(const unsigned* __restrict__ keys, int iters,
                                               unsigned* out) {
    __shared__ unsigned se[256], st[256];
    se[threadIdx.x] = keys[threadIdx.x] & 0x7FFFFFFF;
    st[threadIdx.x] = keys[256 + threadIdx.x] & 0xFFFFF;
    __syncthreads();
    int K[8];
    unsigned be[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { K[q] = (int)(keys[512 + q * 32 + (threadIdx.x & 31)] & 0xFFFFF); be[q] = ~0u; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int c = 0; c < 256; c += 4) {
            uint4 e = *reinterpret_cast<const uint4*>(se + c);
            uint4 t = *reinterpret_cast<const uint4*>(st + c);
            unsigned ev[4] = {e.x, e.y, e.z, e.w};
            int tv[4] = {(int)t.x, (int)t.y, (int)t.z, (int)t.w};
#pragma unroll
            for (int v = 0; v < 4; v += 2)
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int d0 = K[q] - tv[v], d1 = K[q] - tv[v + 1];
                    const unsigned v0 = ev[v] | ((unsigned)d0 & 0x80000000u);
                    const unsigned v1 = ev[v + 1] | ((unsigned)d1 & 0x80000000u);
                    be[q] = __vimin3_u32(be[q], v0, v1);
                }
        }
    }
    unsigned r = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) r ^= be[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}


// C: IMAD.IADD + LOP3 + 2-input VIMNMX per pair
__global__ void __launch_bounds__(256, 4) mixC(const unsigned* __restrict__ keys, int iters,
                                               unsigned* out) {
    __shared__ unsigned se[256], st[256];
    se[threadIdx.x] = keys[threadIdx.x] & 0x7FFFFFFF;
    st[threadIdx.x] = keys[256 + threadIdx.x] & 0xFFFFF;
    __syncthreads();
    int K[8];
    unsigned be[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { K[q] = (int)(keys[512 + q * 32 + (threadIdx.x & 31)] & 0xFFFFF); be[q] = ~0u; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int c = 0; c < 256; c += 4) {
            uint4 e = *reinterpret_cast<const uint4*>(se + c);
            uint4 t = *reinterpret_cast<const uint4*>(st + c);
            unsigned ev[4] = {e.x, e.y, e.z, e.w};
            int tv[4] = {(int)t.x, (int)t.y, (int)t.z, (int)t.w};
#pragma unroll
            for (int v = 0; v < 4; ++v)
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int d0 = K[q] - tv[v];
                    be[q] = min(be[q], ev[v] | ((unsigned)d0 & 0x80000000u));
                }
        }
    }
    unsigned r = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) r ^= be[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// D: mask on the FMA pipe: s = hi32(d * 2) (IMAD.HI), v = s * 2^31 + q (IMAD), VIMNMX
__global__ void __launch_bounds__(256, 4) mixD(const unsigned* __restrict__ keys, int iters,
                                               unsigned* out) {
    __shared__ unsigned se[256], st[256];
    se[threadIdx.x] = keys[threadIdx.x] & 0x7FFFFFFF;
    st[threadIdx.x] = keys[256 + threadIdx.x] & 0xFFFFF;
    __syncthreads();
    int K[8];
    unsigned be[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { K[q] = (int)(keys[512 + q * 32 + (threadIdx.x & 31)] & 0xFFFFF); be[q] = ~0u; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int c = 0; c < 256; c += 4) {
            uint4 e = *reinterpret_cast<const uint4*>(se + c);
            uint4 t = *reinterpret_cast<const uint4*>(st + c);
            unsigned ev[4] = {e.x, e.y, e.z, e.w};
            int tv[4] = {(int)t.x, (int)t.y, (int)t.z, (int)t.w};
#pragma unroll
            for (int v = 0; v < 4; ++v)
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const unsigned d0 = (unsigned)(K[q] - tv[v]);
                    const unsigned s = __umulhi(d0, 2u);
                    be[q] = min(be[q], s * 0x80000000u + ev[v]);
                }
        }
    }
    unsigned r = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) r ^= be[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// E: 2/3 of the configs as C, 1/3 as D (balance the ALU and FMA pipes)
__global__ void __launch_bounds__(256, 4) mixE(const unsigned* __restrict__ keys, int iters,
                                               unsigned* out) {
    __shared__ unsigned se[256], st[256];
    se[threadIdx.x] = keys[threadIdx.x] & 0x7FFFFFFF;
    st[threadIdx.x] = keys[256 + threadIdx.x] & 0xFFFFF;
    __syncthreads();
    int K[8];
    unsigned be[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { K[q] = (int)(keys[512 + q * 32 + (threadIdx.x & 31)] & 0xFFFFF); be[q] = ~0u; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll 2
        for (int c = 0; c < 252; c += 3) {
            const unsigned ev[3] = {se[c], se[c + 1], se[c + 2]};
            const int tv[3] = {(int)st[c], (int)st[c + 1], (int)st[c + 2]};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const unsigned a0 = ev[0] | ((unsigned)(K[q] - tv[0]) & 0x80000000u);
                const unsigned a1 = ev[1] | ((unsigned)(K[q] - tv[1]) & 0x80000000u);
                const unsigned s2 = __umulhi((unsigned)(K[q] - tv[2]), 2u);
                const unsigned a2 = s2 * 0x80000000u + ev[2];
                be[q] = min(min(be[q], a0), min(a1, a2));
            }
        }
    }
    unsigned r = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) r ^= be[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *keys, *out;
    cudaMalloc(&keys, 4096 * 4);
    cudaMalloc(&out, sms * 4 * 256 * 4);
    unsigned h[4096];
    for (int i = 0; i < 4096; ++i) h[i] = (i * 2654435761u) ^ (i << 7);
    cudaMemcpy(keys, h, sizeof h, cudaMemcpyHostToDevice);
    const int iters = 2000, grid = sms * 4;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    typedef void (*KF)(const unsigned*, int, unsigned*);
    KF ks[5] = {mixA, mixB, mixC, mixD, mixE};
    const double pk[5] = {256.0 * 8, 256.0 * 8, 256.0 * 8, 256.0 * 8, 252.0 * 8};
    for (int k = 0; k < 5; ++k) {
        for (int w = 0; w < 2; ++w) ks[k]<<<grid, 256>>>(keys, iters, out);
        cudaEventRecord(a);
        ks[k]<<<grid, 256>>>(keys, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double pairs = (double)grid * 256 * iters * pk[k];
        printf("mix%c: %.3f ms, %.3e pairs/s\n", 'A' + k, ms, pairs / (ms * 1e-3));
    }
    return 0;
}
