// Microbenchmark: the k_scan class-A inner loop (16-bit chunk-local ranks, two configs per
// register: IMAD.IADD + LOP3 per 2 configs, VIMNMX3.U16x2 per 4) over a staged smem chunk,
// with 8 or 16 queries per thread, and the single-instruction throughputs it is built from
// (independent chains, full occupancy). Prints pairs/s (loops) or warp-instructions/clk/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scan_loop scan_loop.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr unsigned kFlag2 = 0x80008000u;

template <int NQ, int MINB>
__global__ void __launch_bounds__(256, MINB) loopA(const unsigned* __restrict__ g, int iters,
                                                   int nw4, unsigned* out) {
    extern __shared__ uint4 sw[];
    for (int i = threadIdx.x; i < nw4; i += 256) {
        const unsigned r0 = g[i & 1023], r1 = g[(i + 7) & 1023];
        sw[i] = make_uint4((r0 & 0x07FF07FFu), r1 & 0x07FF07FFu, (r1 >> 3) & 0x07FF07FFu,
                           (r0 >> 5) & 0x07FF07FFu);
    }
    __syncthreads();
    unsigned K[NQ], m[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
        const unsigned k = 0x8000u + (g[(threadIdx.x * NQ + j) & 1023] & 0x7FF);
        K[j] = k | (k << 16);
        m[j] = 0xFFFFFFFFu;
    }
    for (int it = 0; it < iters; ++it) {
        for (int c = 0; c < nw4; ++c) {
            const uint4 v = sw[c];
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
                const unsigned d0 = K[j] - v.x, d1 = K[j] - v.z;
                const unsigned a0 = v.y | (~d0 & kFlag2), a1 = v.w | (~d1 & kFlag2);
                m[j] = __vimin3_u16x2(m[j], a0, a1);
            }
        }
    }
    unsigned r = 0;
#pragma unroll
    for (int j = 0; j < NQ; ++j) r ^= m[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// single-instruction throughput: 16 independent chains per thread
__global__ void __launch_bounds__(256, 4) opLOP3(const unsigned* g, int iters, unsigned* out) {
    unsigned a[16];
    const unsigned b = g[threadIdx.x & 1023], c = g[(threadIdx.x + 3) & 1023];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = g[(threadIdx.x + j) & 1023];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[j]) : "r"(b), "r"(c));
    }
    unsigned r = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) r ^= a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void __launch_bounds__(256, 4) opVMN3(const unsigned* g, int iters, unsigned* out) {
    unsigned a[16];
    const unsigned b = g[threadIdx.x & 1023], c = g[(threadIdx.x + 3) & 1023];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = g[(threadIdx.x + j) & 1023];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("{.reg .b32 t1; min.u16x2 t1, %0, %1; min.u16x2 %0, t1, %2;}" : "+r"(a[j]) : "r"(b), "r"(c));
    }
    unsigned r = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) r ^= a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void __launch_bounds__(256, 4) opIADD(const unsigned* g, int iters, unsigned* out) {
    unsigned a[16];
    const unsigned b = g[threadIdx.x & 1023];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = g[(threadIdx.x + j) & 1023];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("sub.u32 %0, %1, %0;" : "+r"(a[j]) : "r"(b));
    }
    unsigned r = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) r ^= a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
// LOP3 + VIMNMX3 interleaved 2:1 (the loop's ALU mix without the IMADs)
__global__ void __launch_bounds__(256, 4) opMIX(const unsigned* g, int iters, unsigned* out) {
    unsigned a[8], m[8];
    const unsigned b = g[threadIdx.x & 1023], c = g[(threadIdx.x + 3) & 1023];
#pragma unroll
    for (int j = 0; j < 8; ++j) { a[j] = g[(threadIdx.x + j) & 1023]; m[j] = ~0u; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            unsigned x = a[j], y = a[j] ^ b;
            asm volatile("lop3.b32 %0, %0, %1, %2, 0xF8;" : "+r"(x) : "r"(b), "r"(c));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0xF8;" : "+r"(y) : "r"(c), "r"(b));
            m[j] = __vimin3_u16x2(m[j], x, y);
        }
    }
    unsigned r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) r ^= m[j] ^ a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned *g, *out;
    cudaMalloc(&g, 4096 * 4);
    cudaMalloc(&out, sms * 8 * 256 * 4);
    unsigned h[4096];
    for (int i = 0; i < 4096; ++i) h[i] = (i * 2654435761u) ^ (i << 7);
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto launch) {
        launch();
        launch();
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        return (double)ms;
    };
    const int nw4 = 512;  // 2,048 configs per staged chunk
    const size_t sm = nw4 * 16;
    for (int cps : {2, 3, 4}) {
        const int iters = 200, grid = sms * cps;
        double ms = timeit([&] { loopA<8, 4><<<grid, 256, sm>>>(g, iters, nw4, out); });
        printf("{\"loop\": \"A NQ=8\", \"ctas_per_sm\": %d, \"pairs_per_s\": %.4e}\n", cps,
               (double)grid * 256 * iters * nw4 * 4 * 8 / (ms * 1e-3));
        if (cps <= 2) {
            ms = timeit([&] { loopA<16, 2><<<grid, 256, sm>>>(g, iters, nw4, out); });
            printf("{\"loop\": \"A NQ=16\", \"ctas_per_sm\": %d, \"pairs_per_s\": %.4e}\n", cps,
                   (double)grid * 256 * iters * nw4 * 4 * 16 / (ms * 1e-3));
        }
    }
    const int iters = 20000, grid = sms * 4;
    const char* names[4] = {"LOP3", "VIMNMX3.U16x2", "IADD", "2xLOP3+VIMNMX3"};
    for (int k = 0; k < 4; ++k) {
        double ms = timeit([&] {
            if (k == 0) opLOP3<<<grid, 256>>>(g, iters, out);
            if (k == 1) opVMN3<<<grid, 256>>>(g, iters, out);
            if (k == 2) opIADD<<<grid, 256>>>(g, iters, out);
            if (k == 3) opMIX<<<grid, 256>>>(g, iters, out);
        });
        const double inst = (double)grid * 8 * iters * (k == 3 ? 24 : 16);  // warp instructions
        printf("{\"op\": \"%s\", \"warp_inst_per_clk_per_sm\": %.3f, \"clk_mhz_attr\": %d}\n", names[k],
               inst / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
    return 0;
}
