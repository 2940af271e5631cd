// Mapped-memory ping-pong between a host thread and a resident kernel: the floor of the
// single-call server's round trip. Variants:
//   seq+body : lane 0 polls a sequence word, then the warp reads a body of B bytes
//              (a second PCIe round trip), writes a response, fence, sequence
//   chunked  : every 16-byte chunk carries the sequence in its last word; all lanes poll
//              their chunks (one PCIe read of the whole request per poll) and the response
//              goes back the same way (no fence: the host checks every chunk)
//   launch   : a kernel launch per call + the mapped response
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pingpong pingpong.cu
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

__global__ void k_pong(volatile int* box, int body_words, int iters) {
    int last = 0;
    __shared__ int s_body[256];
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) {
            while (box[0] == last) {
            }
            last = box[0];
            __threadfence_system();
        }
        __syncwarp();
        for (int i = threadIdx.x; i < body_words; i += 32) s_body[i] = box[64 + i];
        __syncwarp();
        if (threadIdx.x == 0) {
            box[512 + 1] = s_body[0] + 1;
            __threadfence_system();
            box[512] = last;
        }
        __syncwarp();
    }
}

// chunks of int4 {payload x3, seq}
__global__ void k_pong_chunked(int4* req, int4* resp, int n_req, int n_resp, int iters) {
    const int lane = threadIdx.x;
    for (int it = 1; it <= iters; ++it) {
        int4 v = make_int4(0, 0, 0, it);
        for (;;) {
            if (lane < n_req)
                asm volatile("ld.volatile.global.v4.s32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "l"(req + lane) : "memory");
            if (__all_sync(0xffffffffu, v.w == it)) break;
        }
        const int x = __shfl_sync(0xffffffffu, v.x, 0) + 1;
        if (lane < n_resp)
            asm volatile("st.volatile.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(resp + lane),
                         "r"(x), "r"(lane), "r"(0), "r"(it) : "memory");
    }
}

int main() {
    int* h;
    int* d;
    cudaHostAlloc((void**)&h, 16384, cudaHostAllocMapped);
    cudaHostGetDevicePointer((void**)&d, h, 0);
    for (int body : {0, 128}) {
        memset(h, 0, 16384);
        const int iters = 20000;
        k_pong<<<1, 32>>>((volatile int*)d, body, iters);
        volatile int* vh = h;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 1; i <= iters; ++i) {
            vh[64] = i;
            std::atomic_thread_fence(std::memory_order_seq_cst);
            vh[0] = i;
            while (vh[512] != i) {
            }
            if (i == 1000) t0 = std::chrono::steady_clock::now();
        }
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / (iters - 1000);
        cudaDeviceSynchronize();
        printf("{\"variant\": \"seq+body\", \"body_bytes\": %d, \"round_trip_us\": %.3f}\n", body * 4, us);
    }
    for (int nreq : {1, 28, 32}) {
        memset(h, 0, 16384);
        const int iters = 20000, nresp = 9;
        __m128i* rq = (__m128i*)h;
        volatile int* rs = h + 1024;
        k_pong_chunked<<<1, 32>>>((int4*)d, (int4*)(d + 1024), nreq, nresp, iters);
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 1; i <= iters; ++i) {
            for (int c = 0; c < nreq; ++c) _mm_store_si128(rq + c, _mm_set_epi32(i, c, c, i));
            for (;;) {
                bool ok = true;
                for (int c = 0; c < nresp && ok; ++c) ok = rs[4 * c + 3] == i;
                if (ok) break;
            }
            if (i == 1000) t0 = std::chrono::steady_clock::now();
        }
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / (iters - 1000);
        cudaDeviceSynchronize();
        printf("{\"variant\": \"chunked\", \"req_bytes\": %d, \"round_trip_us\": %.3f}\n", nreq * 16, us);
    }
    {
        volatile int* vh = h;
        memset(h, 0, 16384);
        const int iters = 5000;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 1; i <= iters; ++i) {
            vh[0] = i;
            k_pong<<<1, 32>>>((volatile int*)d, 0, 1);
            while (vh[512] != i) {
            }
            if (i == 500) t0 = std::chrono::steady_clock::now();
        }
        cudaDeviceSynchronize();
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / (iters - 500);
        printf("{\"variant\": \"launch\", \"round_trip_us\": %.3f}\n", us);
    }
    return 0;
}
