// plan.cu — K1: evaluate the grid, build the rank tables, select for a batch of
// queries with the reference's exact argmax.
//
// Reference semantics: select_config controller.hpp:132-201 with
// better_candidate controller.hpp:118-125. The fast path turns every FP64
// feasibility test and every tolerance comparison into integer operations on
// precomputed competition ranks and merged positions; queries whose winner sits in a
// near-tie cluster (scores within 4e-9 relative) are re-decided by the literal
// sequential fold.
#include <algorithm>
#include <type_traits>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "pals_internal.cuh"


namespace pals {

#ifdef PALS_SCAN_TRACE
// A/B instrumentation of k_assign_qprep (scripts/aq_trace.py): globaltimer of block phases
__device__ unsigned long long g_aq_trace[1024][8];
#define AQ_MARK(k)                                                                        \
    if (threadIdx.x == 0 && blockIdx.x < 1024) {                                          \
        unsigned long long t_;                                                            \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
        g_aq_trace[blockIdx.x][k] = t_;                                                   \
    }
#else
#define AQ_MARK(k)
#endif

constexpr int kChunk = 2048;        // sort chunk (smem block merge sort)
constexpr int kScanCh = 2048;       // configs per scan work item
constexpr int kScanThreads = 256;
constexpr int kScanQ = 8;           // queries per thread in the scan (register tile)
constexpr int kMaxChunks = 8;       // pals_select: query chunks pipelined behind their upload
constexpr int kCountStride = 16;    // per query chunk: [0, N_CLS) class sizes, [N_CLS] exact
                                    // folds, [6] qprep blocks done, [8, 16) the scan plan
constexpr int kCntDone = 6, kCntPlan = 8;
constexpr int kCountInts = kMaxChunks * kCountStride;

enum { CLS_A = 0, CLS_B = 1, CLS_C = 2, CLS_D = 3, CLS_X = 4, N_CLS = 5 };
enum { EX_FULL = 0, EX_QOS_NEAR = 1, EX_BUD_NEAR = 2 };


}  // namespace pals

using namespace pals;

struct pals_plan {
    pals_ctx* ctx = nullptr;
    const pals_model* model = nullptr;
    const pals_grid* grid = nullptr;
    pals_coeffs coeffs{};
    int err = PALS_OK;
    std::string err_msg;
    int64_t n = 0, np = 0;
    int nchunks = 0;
    int chunk = 4096;  // sort chunk size (keys per CTA)
    int force_exact = 0;
    int values = 0;               // internal: th / ef supplied directly (frontier.cu)
    int pdl = 1;                  // programmatic dependent launch between step kernels
    int64_t last_exact = 0;
    PlanDev d{};
    int* tr = nullptr;            // device TR per point
    Analytic* d_an = nullptr;     // device copy of the analytic params
    int* table_map = nullptr;     // grid -> table row (table model)
    double* table_T = nullptr;
    double* table_P = nullptr;
    uint64_t* gk = nullptr;       // [2] global candidate keys
    // query-side buffers (capacity-managed)
    int64_t qcap = 0;
    uint64_t* thr_t = nullptr;
    uint64_t* thr_p = nullptr;
    uint64_t* best_e = nullptr;
    uint64_t* best_t = nullptr;
    uint8_t* cls = nullptr;
    int32_t* qlist = nullptr;     // N_CLS regions of qcap
    uint4* qthr = nullptr;        // beside qlist: (thr_t, thr_p, query id, 0) per slot
    int32_t* counts = nullptr;    // [N_CLS] class sizes, [N_CLS] exact count
    pals_query* d_q = nullptr;    // host-API staging
    int32_t* d_idx = nullptr;
    uint8_t* d_reason = nullptr;
    void* slab = nullptr;
    // optional timing of the pair-scan kernel (bench.py roofline)
    int time_scan = 0;
    int scan_recorded = 0;
    cudaEvent_t ev_scan0 = nullptr, ev_scan1 = nullptr;
    // CUDA graph of one full step (prepare + select) for fixed device buffers
    int capturing = 0;
    cudaGraphExec_t gexec = nullptr;
    const void* g_q = nullptr;
    void* g_idx = nullptr;
    void* g_rs = nullptr;
    int64_t g_n = -1;
    int g_timed = 0;
    int64_t g_launches = 0;
    const void* g_hq = nullptr;   // pinned host buffers baked into the graph (pals_select)
    void* g_hidx = nullptr;
    void* g_hrs = nullptr;
    cudaStream_t side = nullptr;  // upload stream of pals_select's graph
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_up[kMaxChunks] = {};  // chunk uploads done (pals_select)
    int g_chunks = 1;             // query chunks of the cached pals_select graph
    int32_t* h_cnt = nullptr;     // pinned class counters (pals_select)
    void* scratch = nullptr;      // plan_scratch()
    size_t scratch_bytes = 0;
    // PALS_DECIDE_PREFIX: prefix-min tables instead of the pair scan (time to decide)
    int decide = PALS_DECIDE_SCAN;
    void* dec_buf = nullptr;
    size_t dec_bytes = 0;
};

namespace pals {

// ---------------------------------------------------------------- eval ----
__device__ __forceinline__ void finish_scores(const PlanDev& d, int64_t i, double T, double P,
                                              int dp, double alpha, double beta) {
    const double th = (double)dp * T;
    const double pn = p_node_of(P, dp, alpha, beta);
    const double ef = th / pn;
    d.T[i] = T;
    d.P[i] = P;
    d.th[i] = th;
    d.pn[i] = pn;
    d.ef[i] = ef;
    const int q = d.tr[i];  // sort input in TR order
    d.skey[ORD_T][q] = ~orderable(th);
    d.skey[ORD_P][q] = orderable(pn);
    d.skey[ORD_E][q] = ~orderable(ef);
    // the integer fast path needs positive, finite, well-scaled scores
    const bool ok = isfinite(th) && isfinite(pn) && isfinite(ef) && th > 1e-250 && pn > 1e-250 &&
                    ef > 1e-250;
    if (!ok) atomicOr(&d.globals[2], 1);
}

__global__ void k_eval_analytic(PlanDev d, const Analytic* __restrict__ an,
                                const int* __restrict__ tp, double alpha, double beta) {
    pdl_wait();
    const Analytic& a = *an;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const Score s = analytic_score(a, d.cap[i], d.batch[i], tp[i], d.dp[i]);
        finish_scores(d, i, s.T, s.P, d.dp[i], alpha, beta);
    }
}

__global__ void k_eval_table(PlanDev d, const int* __restrict__ map, const double* __restrict__ tT,
                             const double* __restrict__ tP, double alpha, double beta) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int r = map[i];
        finish_scores(d, i, tT[r], tP[r], d.dp[i], alpha, beta);
    }
}

// Values plans (frontier.cu): T holds the throughput, P the efficiency of each
// point as given (FrontierPoint); only the t_hat and eff orders are meaningful.
__global__ void k_eval_values(PlanDev d) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double th = d.T[i], ef = d.P[i];
        d.th[i] = th;
        d.pn[i] = 1.0;
        d.ef[i] = ef;
        const int q = d.tr[i];
        d.skey[ORD_T][q] = ~orderable(th);
        d.skey[ORD_P][q] = orderable(1.0);
        d.skey[ORD_E][q] = ~orderable(ef);
    }
}

// ---------------------------------------------------------------- sort ----
// Keys travel with their point index, so the last merge round knows where every
// point landed and the rank pass reads the merged order front to back. Real keys
// are clamped below kNone64 (only the all-ones NaN pattern moves, and a plan with
// a NaN score takes the generic literal-fold path), so the padding sorts strictly
// last and merged positions < n hold exactly the n points.

// search index of the merged keys: every samp_s-th position
__device__ __forceinline__ void put_sample(const PlanDev& d, int o, uint32_t p, uint64_t key) {
    const uint32_t S = (uint32_t)d.samp_s;
    if (p < (uint32_t)d.n && p % S == 0) d.samp[o][p / S] = key;
}

// (1) merge sort of each chunk of TPB * kIPT keys in shared memory (block merge
// sort): every thread sorts its 8 (key, index) pairs with Batcher's 19-comparator
// network in registers, then log2(TPB) rounds merge pairs of sorted lists — each
// thread finds its 8 outputs' start on the merge path by a binary search in shared
// memory and merges them serially. Shared arrays are padded (one slot per 16 keys,
// per 32 indices) so the blocked register <-> smem transposes are conflict-free.
// The kernel also resets what the next prep kernels accumulate into (the
// global-candidate keys, the last-block counter of the rank pass, the select's
// class counters), so the step needs no separate memset nodes.
constexpr int kIPT = 8;

__device__ __forceinline__ int pk(int e) { return e + (e >> 4); }  // padded key slot
__device__ __forceinline__ int pv(int e) { return e + (e >> 5); }  // padded index slot

// ties are broken on the carried TR, so the order is the packed-key order; the
// merges keep it because their left run always holds the smaller TRs
template <int IPT>
__device__ __forceinline__ void cmp_swap(uint64_t (&k)[IPT], uint32_t (&v)[IPT], int i, int j) {
    if (k[j] < k[i] || (k[j] == k[i] && v[j] < v[i])) {
        const uint64_t tk = k[i];
        k[i] = k[j];
        k[j] = tk;
        const uint32_t tv = v[i];
        v[i] = v[j];
        v[j] = tv;
    }
}

// Batcher's odd-even merge networks for 8 (19 comparators) and 4 (5) keys
template <int IPT>
__device__ __forceinline__ void sort_net(uint64_t (&k)[IPT], uint32_t (&v)[IPT]) {
    if (IPT == 2) {
        cmp_swap(k, v, 0, 1);
        return;
    }
    if (IPT == 4) {
        cmp_swap(k, v, 0, 1); cmp_swap(k, v, 2, 3);
        cmp_swap(k, v, 0, 2); cmp_swap(k, v, 1, 3);
        cmp_swap(k, v, 1, 2);
        return;
    }
    cmp_swap(k, v, 0, 1); cmp_swap(k, v, 2, 3); cmp_swap(k, v, 4, 5); cmp_swap(k, v, 6, 7);
    cmp_swap(k, v, 0, 2); cmp_swap(k, v, 1, 3); cmp_swap(k, v, 4, 6); cmp_swap(k, v, 5, 7);
    cmp_swap(k, v, 1, 2); cmp_swap(k, v, 5, 6);
    cmp_swap(k, v, 0, 4); cmp_swap(k, v, 1, 5); cmp_swap(k, v, 2, 6); cmp_swap(k, v, 3, 7);
    cmp_swap(k, v, 2, 4); cmp_swap(k, v, 3, 5);
    cmp_swap(k, v, 1, 2); cmp_swap(k, v, 3, 4); cmp_swap(k, v, 5, 6);
}

// merge path: how many of the first `diag` outputs of merge(A, B) come from A
// (ties take A first). A(i), B(i): key accessors.
template <class FA, class FB>
__device__ __forceinline__ int mp_search(FA A, int la, FB B, int lb, int diag) {
    int lo = max(0, diag - lb), hi = min(diag, la);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A(mid) <= B(diag - 1 - mid)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// IPT consecutive outputs of merge(A, B) starting at (a, b) on the merge path
template <int IPT, class KA, class VA, class KB, class VB>
__device__ __forceinline__ void mp_serial(KA Ak, VA Av, int la, KB Bk, VB Bv, int lb, int a,
                                          int b, uint64_t (&k)[IPT], uint32_t (&v)[IPT]) {
    uint64_t ka = a < la ? Ak(a) : kNone64, kb = b < lb ? Bk(b) : kNone64;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        if (b >= lb || (a < la && ka <= kb)) {
            k[i] = ka;
            v[i] = a < la ? Av(a) : 0u;
            ++a;
            ka = a < la ? Ak(a) : kNone64;
        } else {
            k[i] = kb;
            v[i] = Bv(b);
            ++b;
            kb = b < lb ? Bk(b) : kNone64;
        }
    }
}

// block merge sort of the TPB * IPT (key, index) pairs in sk/sv (padded layout);
// leaves each thread's IPT outputs (positions t*IPT..) in k/v
template <int TPB, int IPT>
__device__ __forceinline__ void block_sort(uint64_t* sk, uint32_t* sv, uint64_t (&k)[IPT],
                                           uint32_t (&v)[IPT]) {
    const int t = threadIdx.x;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        k[i] = sk[pk(t * IPT + i)];
        v[i] = sv[pv(t * IPT + i)];
    }
    sort_net<IPT>(k, v);
    for (int w = 1; w < TPB; w <<= 1) {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            sk[pk(t * IPT + i)] = k[i];
            sv[pv(t * IPT + i)] = v[i];
        }
        __syncthreads();
        const int g0 = (t & ~(2 * w - 1)) * IPT;  // the group's first key
        const int len = w * IPT;
        const int diag = (t & (2 * w - 1)) * IPT;
        auto Ak = [&](int i) { return sk[pk(g0 + i)]; };
        auto Bk = [&](int i) { return sk[pk(g0 + len + i)]; };
        auto Av = [&](int i) { return sv[pv(g0 + i)]; };
        auto Bv = [&](int i) { return sv[pv(g0 + len + i)]; };
        const int a = mp_search(Ak, len, Bk, len, diag);
        mp_serial<IPT>(Ak, Av, len, Bk, Bv, len, a, diag - a, k, v);
    }
}

constexpr size_t sort_smem_bytes(int tpb, int ipt = kIPT) {
    return (size_t)(tpb * ipt + tpb * ipt / 16) * 8 + (size_t)(tpb * ipt + tpb * ipt / 32) * 4;
}

constexpr uint32_t kLrPadSort = 4095;  // a chunk-local rank no threshold reaches (k_scan)

template <int TPB, int IPT = kIPT>
__global__ void __launch_bounds__(TPB) k_sort_chunks(PlanDev d, uint64_t* gk, uint32_t* done,
                                                     int32_t* counts_reset, int to_merged,
                                                     int final_round) {
    constexpr int CH = TPB * IPT;
    extern __shared__ __align__(16) unsigned char sort_smem[];  // sort_smem_bytes(TPB)
    uint64_t* sk = reinterpret_cast<uint64_t*>(sort_smem);
    uint32_t* sv = reinterpret_cast<uint32_t*>(sk + CH + CH / 16);
    pdl_wait();
    const int o = blockIdx.y;
    const uint32_t base = blockIdx.x * (uint32_t)CH;
    const int t = threadIdx.x;
    {
        // all loads in flight before the shared stores (a generic-pointer load may
        // not be reordered across a shared store, which would serialize the round trips)
        // input in TR order (the evaluation writes position q = TR of each point), so
        // sorting by (value, q) gives merged positions in packed-key order
        uint64_t x[IPT];
        const uint64_t* __restrict__ src = d.skey[o];
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const uint32_t g = base + t + k * TPB;
            x[k] = g < (uint32_t)d.n ? min(__ldg(src + g), kNone64 - 1) : kNone64;
        }
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            sk[pk(t + k * TPB)] = x[k];
            sv[pv(t + k * TPB)] = base + t + k * TPB;
        }
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && t == 0) {
        gk[0] = gk[1] = kNone64;
        done[0] = done[1] = 0;
    }
    if (counts_reset && blockIdx.x == 0 && blockIdx.y == 0)
        for (int i = t; i < kCountInts; i += TPB) counts_reset[i] = 0;
    __syncthreads();
    uint64_t k[IPT];
    uint32_t v[IPT];
    block_sort<TPB, IPT>(sk, sv, k, v);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        sk[pk(t * IPT + i)] = k[i];
        sv[pv(t * IPT + i)] = v[i];
    }
    __syncthreads();
    uint64_t* dst = to_merged ? d.merged[o] : d.sorted[o];
    uint32_t* dstv = to_merged ? d.midx[o] : d.sidx[o];
    for (int i = t; i < CH; i += TPB) {
        const uint32_t p = base + i;
        dst[p] = sk[pk(i)];
        dstv[p] = sv[pv(i)];
        if (final_round) put_sample(d, o, p, sk[pk(i)]);
    }
    // chunk-local ranks of the pair scan: the run lists the chunk in global merged-position
    // order, so a point's place in it orders the chunk as the global positions do, and the
    // first place with its key is its competition rank inside the chunk (equal keys are
    // equal values)
    if (CH <= 2048) {
        for (int i = t; i < CH; i += TPB) {
            const uint32_t v = sv[pv(i)];
            if (v >= (uint32_t)d.n) {  // padding of the last chunk: never feasible
                d.lr16[o][v] = (uint16_t)kLrPadSort;
                d.lq16[o][v] = 0x7FFF;
                d.cinv[o][base + i] = 0xFFFFFFFFu;
                continue;
            }
            const uint64_t key = sk[pk(i)];
            int lo = 0, hi = i;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sk[pk(mid)] < key) lo = mid + 1;
                else hi = mid;
            }
            d.lr16[o][v] = (uint16_t)lo;
            d.lq16[o][v] = (uint16_t)i;
        }
    }
}

template <bool LE>
__device__ __forceinline__ bool before(uint64_t y, uint64_t x) {
    return LE ? y <= x : y < x;
}

// Two searches by one warp over a sorted key sequence S(i), i in [lo0, hi0): ra
// (rb) = the first position whose key is not before xa (xb), "before" being <
// (LE: <=). 32-ary: each round probes 32 evenly spaced positions of each key's
// remaining range with one load per lane and narrows it by a ballot, so a 32K-key
// range takes 3 dependent loads instead of 15. Every lane returns the same answers.
template <bool LE, class FS>
__device__ __forceinline__ void warp_search2(FS S, uint32_t lo0, uint32_t hi0, uint64_t xa,
                                             uint64_t xb, uint32_t& ra, uint32_t& rb) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t la = lo0, ha = hi0, lb = lo0, hb = hi0;
    while (la < ha || lb < hb) {
        const uint32_t sa = (ha - la + 31) >> 5, sb = (hb - lb + 31) >> 5;
        const uint32_t pa = la + sa * (lane + 1) - 1, pb = lb + sb * (lane + 1) - 1;
        const bool ta = la < ha && pa < ha && before<LE>(S(pa), xa);
        const bool tb = lb < hb && pb < hb && before<LE>(S(pb), xb);
        const uint32_t ca = __popc(__ballot_sync(0xffffffffu, ta));
        const uint32_t cb = __popc(__ballot_sync(0xffffffffu, tb));
        if (la < ha) {
            ha = min(ha, la + sa * (ca + 1) - 1);
            la += sa * ca;
        }
        if (lb < hb) {
            hb = min(hb, lb + sb * (cb + 1) - 1);
            lb += sb * cb;
        }
    }
    ra = la;
    rb = lb;
}

// Two independent warp searches over S in one pass of 32-ary rounds: ra = the first position
// of [la, ha) whose key is not before xa (LEA: <=, else <), rb likewise over [lb, hb) for xb;
// an empty range costs nothing.
template <bool LEA, bool LEB, class FS>
__device__ __forceinline__ void warp_search_pair(FS S, uint32_t la, uint32_t ha, uint64_t xa,
                                                 uint32_t lb, uint32_t hb, uint64_t xb,
                                                 uint32_t& ra, uint32_t& rb) {
    const uint32_t lane = threadIdx.x & 31;
    while (la < ha || lb < hb) {
        const uint32_t sa = (ha - la + 31) >> 5, sb = (hb - lb + 31) >> 5;
        const uint32_t pa = la + sa * (lane + 1) - 1, pb = lb + sb * (lane + 1) - 1;
        const bool ta = la < ha && pa < ha && before<LEA>(S(pa), xa);
        const bool tb = lb < hb && pb < hb && before<LEB>(S(pb), xb);
        const uint32_t ca = __popc(__ballot_sync(0xffffffffu, ta));
        const uint32_t cb = __popc(__ballot_sync(0xffffffffu, tb));
        if (la < ha) {
            ha = min(ha, la + sa * (ca + 1) - 1);
            la += sa * ca;
        }
        if (lb < hb) {
            hb = min(hb, lb + sb * (cb + 1) - 1);
            lb += sb * cb;
        }
    }
    ra = la;
    rb = lb;
}

// Merge-path splits of two output diagonals da, db of merge(A, B) by one warp,
// 32-ary as in warp_search2: the predicate A(a) <= B(d-1-a) holds on a prefix of
// the candidate a's.
template <class FA, class FB>
__device__ __forceinline__ void warp_mp2(FA A, uint32_t la, FB B, uint32_t lb, uint32_t da,
                                         uint32_t db, uint32_t& ra, uint32_t& rb) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t l0 = da > lb ? da - lb : 0, h0 = min(da, la);
    uint32_t l1 = db > lb ? db - lb : 0, h1 = min(db, la);
    while (l0 < h0 || l1 < h1) {
        const uint32_t s0 = (h0 - l0 + 31) >> 5, s1 = (h1 - l1 + 31) >> 5;
        const uint32_t p0 = l0 + s0 * (lane + 1) - 1, p1 = l1 + s1 * (lane + 1) - 1;
        const bool t0 = l0 < h0 && p0 < h0 && A(p0) <= B(da - 1 - p0);
        const bool t1 = l1 < h1 && p1 < h1 && A(p1) <= B(db - 1 - p1);
        const uint32_t c0 = __popc(__ballot_sync(0xffffffffu, t0));
        const uint32_t c1 = __popc(__ballot_sync(0xffffffffu, t1));
        if (l0 < h0) {
            h0 = min(h0, l0 + s0 * (c0 + 1) - 1);
            l0 += s0 * c0;
        }
        if (l1 < h1) {
            h1 = min(h1, l1 + s1 * (c1 + 1) - 1);
            l1 += s1 * c1;
        }
    }
    ra = l0;
    rb = l1;
}

// (2) pairwise merge rounds of sorted runs of length L (merge path, one output
// tile of TPB * kIPT keys per CTA): warp 0 finds where the tile's first and last
// diagonals cross the two runs, the tile's slices of both runs are staged in
// shared memory with coalesced loads, and every thread merges its 8 outputs as in
// the block sort. Ties take the left run first (a stable merge). Buffers
// ping-pong between sorted and merged; the chunk sort picks its output so the last
// round writes merged, and the last round also writes the search index.
template <int TPB, int IPT = kIPT>
__global__ void __launch_bounds__(TPB) k_merge_round(PlanDev d, uint32_t np, int lgL,
                                                     int to_merged, int final_round) {
    constexpr int TILE = TPB * IPT;
    __shared__ uint64_t sk[TILE + TILE / 16];
    __shared__ uint32_t sv[TILE + TILE / 32];
    __shared__ uint32_t split[2];
    pdl_wait();
    const int o = blockIdx.y;
    const uint64_t* __restrict__ in = to_merged ? d.sorted[o] : d.merged[o];
    const uint32_t* __restrict__ inv = to_merged ? d.sidx[o] : d.midx[o];
    uint64_t* out = to_merged ? d.merged[o] : d.sorted[o];
    uint32_t* outv = to_merged ? d.midx[o] : d.sidx[o];
    const int t = threadIdx.x;
    const uint32_t L = 1u << lgL;
    const uint32_t t0 = blockIdx.x * (uint32_t)TILE;
    const uint32_t pb = t0 & ~(2 * L - 1);  // the pair's first position
    const uint32_t la = min(L, np - pb);
    const uint32_t lb = np - pb > L ? min(L, np - pb - L) : 0;
    const uint64_t* A = in + pb;
    const uint64_t* B = A + la;
    const uint32_t d0 = t0 - pb, d1 = min(d0 + (uint32_t)TILE, la + lb);
    if (t < 32) {
        uint32_t a0, a1;
        warp_mp2([&](uint32_t i) { return A[i]; }, la, [&](uint32_t i) { return B[i]; }, lb, d0,
                 d1, a0, a1);
        if (t == 0) {
            split[0] = a0;
            split[1] = a1;
        }
    }
    __syncthreads();
    const uint32_t a0 = split[0], a1 = split[1];
    const int na = (int)(a1 - a0), nb = (int)((d1 - a1) - (d0 - a0));
    const uint32_t b0 = d0 - a0;
    {
        // stage both slices: every load in flight before the shared stores
        uint64_t x[IPT];
        uint32_t y[IPT];
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const int i = t + k * TPB;
            const uint32_t q = i < na ? pb + a0 + i : pb + la + b0 + (i - na);
            const bool ok = i < na + nb;
            x[k] = ok ? __ldg(in + q) : kNone64;
            y[k] = ok ? __ldg(inv + q) : 0u;
        }
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            sk[pk(t + k * TPB)] = x[k];
            sv[pv(t + k * TPB)] = y[k];
        }
    }
    __syncthreads();
    const int diag = t * IPT;
    const int tot = na + nb;
    if (diag < tot) {
        uint64_t k[IPT];
        uint32_t v[IPT];
        auto Ak = [&](int i) { return sk[pk(i)]; };
        auto Bk = [&](int i) { return sk[pk(na + i)]; };
        auto Av = [&](int i) { return sv[pv(i)]; };
        auto Bv = [&](int i) { return sv[pv(na + i)]; };
        const int a = mp_search(Ak, na, Bk, nb, diag);
        mp_serial<IPT>(Ak, Av, na, Bk, Bv, nb, a, diag - a, k, v);
        const uint32_t p0 = pb + d0 + diag;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            if (diag + i < tot) {
                out[p0 + i] = k[i];
                outv[p0 + i] = v[i];
                if (final_round) put_sample(d, o, p0 + i, k[i]);
            }
        }
    }
}

__device__ __forceinline__ double key_value(int o, uint64_t k) {
    return o == ORD_P ? unorderable(k) : unorderable(~k);
}

// Two values are "separated" when no pair straddling them can be a tolerance
// tie of better_candidate (|a-b|/max(|a|,|b|) <= 1e-9), with a 4x margin.
__device__ __forceinline__ bool separated(double a, double b) {
    return fabs(a - b) > 4e-9 * smax(fabs(a), fabs(b));
}

// boundary class between merged positions i and i+1 (see PlanDev::bnd)
__device__ __forceinline__ uint8_t boundary(const PlanDev& d, int o, int64_t i) {
    if (i + 1 >= d.n) return 2;
    const uint64_t a = d.merged[o][i], b = d.merged[o][i + 1];
    if (a == b) return 0;
    return separated(key_value(o, a), key_value(o, b)) ? 2 : 1;
}

// (4) the rank pass, over merged positions p (one warp = 32 consecutive positions):
// the competition rank of the key at p is the start of its run of equal keys (the
// last run start at or before p; a run that began before the warp is found by one
// warp search), the point it carries gets its packed key (r << tr_bits) | TR, and
// position p gets its boundary class and, at a run start, whether the run ends on
// a near-tie (then a winner there needs the exact fold). Coalesced except for the
// per-point key store; at most two warp searches per warp. M(p) / V(p): the merged
// key / point index at position p (global memory or the cluster's shared memory).
constexpr int kSamples = 1024;  // per-order search index of the merged keys

__device__ void resolve_globals_warp(const PlanDev& d, const uint64_t* gk, int w);

__device__ __forceinline__ uint8_t bnd_class(int o, uint64_t a, uint64_t b) {
    if (a == b) return 0;
    return separated(key_value(o, a), key_value(o, b)) ? 2 : 1;
}

// Narrow a warp search over the merged keys with the staged search index ss (every S-th
// key, ns of them; null: no narrowing): the first position whose key is not before x (LE:
// <=, else <) lies in [lo, hi] after this, a window of at most S positions — one or two
// 32-ary rounds where the whole range took four.
template <bool LE>
__device__ __forceinline__ void narrow(const uint64_t* ss, int ns, uint32_t S, uint64_t x,
                                       uint32_t& lo, uint32_t& hi) {
    if (!ss) return;
    int a = 0, b = ns;  // samples before x
    while (a < b) {
        const int mid = (a + b) >> 1;
        if (before<LE>(ss[mid], x)) a = mid + 1;
        else b = mid;
    }
    if (a > 0) lo = max(lo, (uint32_t)(a - 1) * S + 1);
    if (a < ns) hi = min(hi, (uint32_t)a * S);
    if (lo > hi) lo = hi;
}

template <class FM, class FV>
__device__ __forceinline__ void assign_warp(const PlanDev& d, uint64_t* gk, int o, uint32_t w0,
                                            FM M, FV V, const uint64_t* ss) {
    const uint32_t n = (uint32_t)d.n;
    const uint32_t lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    const uint32_t p = w0 + lane;
    const bool in = p < n;
    const uint64_t key = in ? M(p) : kNone64;
    // the point carried at p and what the stores need of it, loaded up front so the chain
    // TR -> point index / run place overlaps the run searches below
    const uint32_t trv = in ? V(p) : n;  // the carried grid rank TR
    const bool real = trv < n;
    const uint32_t idx = real ? (uint32_t)__ldg(d.inv_tr + trv) : 0u;
    const uint32_t lq = real ? (uint32_t)d.lq16[o][trv] : 0u;
    uint64_t prev = __shfl_up_sync(full, key, 1);
    uint64_t next = __shfl_down_sync(full, key, 1);
    if (lane == 0) prev = p > 0 ? M(p - 1) : ~key;
    if (lane == 31 && p + 1 < n) next = M(p + 1);
    const bool start = in && prev != key;
    const unsigned sm = __ballot_sync(full, start);
    const uint8_t bi = (in && p + 1 < n) ? bnd_class(o, key, next) : 2;
    AQ_MARK(5);
    // rank: the last run start among lanes 0..lane, else the start of lane 0's run (a run
    // that began before the warp: searched); danger at a run start: the class of the
    // boundary after the run's last position (a run that continues past the warp:
    // searched). Both searches (warp-uniform conditions) run in the same 32-ary rounds.
    const unsigned upto = sm & (full >> (31 - lane));
    const unsigned after = sm & ~(full >> (31 - lane));
    const int tl = after ? __ffs(after) - 1 : 32;
    const uint8_t bend = (uint8_t)__shfl_sync(full, (int)bi, (tl - 1) & 31);
    const uint8_t b31 = (uint8_t)__shfl_sync(full, (int)bi, 31);
    const bool need_start = !(sm & 1u), need_end = sm && b31 == 0;
    uint32_t r0 = w0;
    uint8_t bext = 0;
    if (need_start || need_end) {  // warp-uniform
        const uint64_t k0 = __shfl_sync(full, key, 0);
        const uint64_t kl = __shfl_sync(full, key, sm ? 31 - __clz(sm) : 0);
        uint32_t lo0 = 0, hi0 = need_start ? w0 : 0, lo1 = w0 + 32, hi1 = need_end ? n : w0 + 32;
        if (need_start) narrow<false>(ss, d.samp_n, (uint32_t)d.samp_s, k0, lo0, hi0);
        if (need_end) narrow<true>(ss, d.samp_n, (uint32_t)d.samp_s, kl, lo1, hi1);
        uint32_t a0, a1;
        warp_search_pair<false, true>(M, lo0, hi0, k0, lo1, hi1, kl, a0, a1);
        if (need_start) r0 = a0;
        if (need_end) {
            const uint32_t e = a1 - 1;  // the run's last position
            bext = e + 1 < n ? bnd_class(o, M(e), M(e + 1)) : 2;
        }
    }
    const uint32_t r = upto ? w0 + 31 - __clz(upto) : r0;
    AQ_MARK(6);
    if (in) {
        const uint8_t dg = start ? ((tl < 32 || b31 != 0 ? bend : bext) == 1) : 0;
        if (real) {
            const uint64_t k = ((uint64_t)r << d.tr_bits) | (uint64_t)trv;
            if (d.wide) d.key64[o][idx] = k;
            else d.key32[o][idx] = (uint32_t)k;
            d.rank32[o][idx] = r;
            d.pos32[o][idx] = p;
            // the pair scan's run place -> global position (chunk-local ranks, k_scan)
            d.cinv[o][(trv / (uint32_t)d.lch) * (uint32_t)d.lch + lq] = p;
            d.midx[o][p] = idx;  // position -> point, and its rank (k_finalize)
            d.sidx[o][p] = r;
            if (r == 0 && o == ORD_T) atomicMin((unsigned long long*)&gk[0], k);
            if (r == 0 && o == ORD_P) atomicMin((unsigned long long*)&gk[1], k);
        }
        d.bnd[o][p] = bi;
        d.danger[o][p] = dg;
    }
}

// last-block-done, per order: the t order's blocks count on done[0] and resolve the argmax
// t_hat over all (gk[0]), the p order's on done[1] for the argmin p_node (gk[1]); every
// block's keys, danger flags and candidate atomics are visible after its fence, so the last
// block of the order can resolve its winner. The efficiency order resolves nothing and
// skips the counter (one counter for all 768 cfg2 blocks serialised ~2.3 us of atomics).
__device__ __forceinline__ void last_block_resolve(const PlanDev& d, uint64_t* gk, uint32_t* done,
                                                   int o, uint32_t nblocks) {
    if (o == ORD_E) return;
    const int w = o == ORD_T ? 0 : 1;
    __shared__ bool last;
    __syncthreads();
    AQ_MARK(3);
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&done[w], 1u) == nblocks - 1;
    }
    __syncthreads();
    AQ_MARK(4);
    if (last) {  // block-uniform
        __threadfence();
        if (threadIdx.x < 32) resolve_globals_warp(d, gk, w);
        __syncthreads();
        if (threadIdx.x == 0) {  // self-cleaning for the next prepare
            gk[w] = kNone64;
            done[w] = 0;
        }
    }
}

// assign_body: block bx of nbx for order o (nbx blocks per order).
// ss: shared-memory scratch for the order's search index (kSamples keys) or null
__device__ __forceinline__ void assign_body(const PlanDev& d, uint64_t* gk, uint32_t* done, int o,
                                            int bx, int nbx, uint64_t* ss) {
    const uint64_t* __restrict__ m = d.merged[o];
    const uint32_t* __restrict__ mi = d.midx[o];
    const uint32_t n = (uint32_t)d.n;
    const uint32_t stride = (uint32_t)nbx * blockDim.x;
    if (ss) {  // the search index written by the last merge round
        for (int i = threadIdx.x; i < d.samp_n; i += blockDim.x) ss[i] = __ldg(d.samp[o] + i);
        __syncthreads();
    }
    AQ_MARK(1);
    for (uint32_t w0 = (uint32_t)bx * blockDim.x + (threadIdx.x & ~31u); w0 < n; w0 += stride)
        assign_warp(d, gk, o, w0, [&](uint32_t q) { return m[q]; },
                    [&](uint32_t q) { return mi[q]; }, ss);
    AQ_MARK(2);
    last_block_resolve(d, gk, done, o, (uint32_t)nbx);
}

__global__ void k_assign(PlanDev d, uint64_t* gk, uint32_t* done) {
    pdl_wait();
    assign_body(d, gk, done, blockIdx.y, blockIdx.x, gridDim.x, nullptr);
}


// Last merged position of the near-tie cluster that contains position r0: the
// cluster extends over runs whose boundaries are near-ties (bnd == 1).
__device__ __forceinline__ uint32_t cluster_end(const PlanDev& d, int o, uint32_t r0) {
    int64_t j = r0;
    while (j + 1 < d.n && boundary(d, o, j) != 2) ++j;
    return (uint32_t)j;
}

// ------------------------------------------------------- exact fold ------
// The reference's sequential fold `if (!best || better(s, best)) best = s`
// (controller.hpp:162-198), executed by one warp in candidate order: each
// round finds the first lane (after the last update) that beats the running
// best, so every comparison the reference makes is made, in the same order.
template <class Filter, class ScoreF>
__device__ int warp_fold(int64_t n, const double* __restrict__ cap, const int* __restrict__ batch,
                         Filter filt, ScoreF score) {
    const int lane = threadIdx.x & 31;
    int64_t best = -1;
    double bs = 0.0, bcap = 0.0;
    int bb = 0;
    for (int64_t base = 0; base < n; base += 32) {
        const int64_t c = base + lane;
        const bool ok = c < n && filt(c);
        double s = 0.0, cp = 0.0;
        int bt = 0;
        if (ok) {
            s = score(c);
            cp = cap[c];
            bt = batch[c];
        }
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (!m) continue;
        int last = -1;
        if (best < 0) {
            const int l = __ffs(m) - 1;
            best = base + l;
            bs = __shfl_sync(0xffffffffu, s, l);
            bcap = __shfl_sync(0xffffffffu, cp, l);
            bb = __shfl_sync(0xffffffffu, bt, l);
            last = l;
        }
        while (true) {
            const bool b = ok && lane > last && better_exact(s, cp, bt, bs, bcap, bb);
            const unsigned bm = __ballot_sync(0xffffffffu, b);
            if (!bm) break;
            const int l = __ffs(bm) - 1;
            best = base + l;
            bs = __shfl_sync(0xffffffffu, s, l);
            bcap = __shfl_sync(0xffffffffu, cp, l);
            bb = __shfl_sync(0xffffffffu, bt, l);
            last = l;
        }
    }
    return (int)best;
}

// competition rank of point c in order o
__device__ __forceinline__ uint32_t rank_of(const PlanDev& d, int o, int64_t c) {
    return d.wide ? (uint32_t)(d.key64[o][c] >> d.tr_bits)
                  : (uint32_t)(d.key32[o][c] >> d.tr_bits);
}

// Literal select_config (controller.hpp:132-201) by one warp.
__device__ void warp_select_full(const PlanDev& d, const pals_query& q, int32_t* idx,
                                 uint8_t* reason) {
    const double target = q.throughput_tps * (1.0 + q.target_headroom);
    const bool bset = q.has_budget != 0;
    const double budget = bset ? q.power_budget_w * (1.0 - q.budget_margin) : 0.0;
    const double bias = q.bias;
    int best = -1;
    int r = PALS_REASON_FALLBACK_MAX_T;
    if (q.objective == PALS_OBJ_QOS) {
        best = warp_fold(
            d.n, d.cap, d.batch,
            [&](int64_t c) {
                return !((bset && !(d.pn[c] <= budget)) || d.th[c] * bias < target);
            },
            [&](int64_t c) { return d.th[c] / d.pn[c]; });
        if (best >= 0) r = PALS_REASON_QOS_FEASIBLE;
    }
    if (best < 0 && bset) {
        best = warp_fold(
            d.n, d.cap, d.batch, [&](int64_t c) { return d.pn[c] <= budget; },
            [&](int64_t c) { return d.th[c]; });
        if (best >= 0) r = PALS_REASON_BUDGET_MAX_T;
        if (best < 0) {
            best = warp_fold(
                d.n, d.cap, d.batch, [&](int64_t) { return true; },
                [&](int64_t c) { return -d.pn[c]; });
            r = PALS_REASON_BUDGET_MAX_T;
        }
    }
    if (best < 0) {
        best = warp_fold(
            d.n, d.cap, d.batch, [&](int64_t) { return true; },
            [&](int64_t c) { return d.th[c]; });
        r = PALS_REASON_FALLBACK_MAX_T;
    }
    if ((threadIdx.x & 31) == 0) {
        *idx = best;
        *reason = (uint8_t)r;
    }
}

// (6) query-independent winners: argmax t_hat over all and argmin p_node over all
// warp w = 0: argmax t_hat over all (controller.hpp:191-198); w = 1: argmin p_node
// over all (:180-188). Run by the last block of k_assign.
__device__ void resolve_globals_warp(const PlanDev& d, const uint64_t* gk, int w) {
    const int lane = threadIdx.x & 31;
    const int generic = d.globals[2];
    const int o = w == 0 ? ORD_T : ORD_P;
    const uint64_t mask = (1ull << d.tr_bits) - 1;
    int best;
    if (!generic && !d.danger[o][0]) {
        best = d.inv_tr[gk[w] & mask];
    } else {
        // near-tie at the top: fold over the top cluster only (every point below
        // the cluster loses to every point in it by more than the tolerance)
        const uint32_t cut = generic ? 0xFFFFFFFFu : cluster_end(d, o, 0);
        if (w == 0)
            best = warp_fold(
                d.n, d.cap, d.batch,
                [&](int64_t c) { return generic || rank_of(d, ORD_T, c) <= cut; },
                [&](int64_t c) { return d.th[c]; });
        else
            best = warp_fold(
                d.n, d.cap, d.batch,
                [&](int64_t c) { return generic || rank_of(d, ORD_P, c) <= cut; },
                [&](int64_t c) { return -d.pn[c]; });
    }
    if (lane == 0) d.globals[w] = best;
}

// ------------------------------------------------------------ select ----
struct SelArgs {
    const pals_query* q;
    int64_t nq;
    int32_t* out_idx;
    uint8_t* out_reason;
    uint64_t* thr_t;
    uint64_t* thr_p;
    uint64_t* best_e;
    uint64_t* best_t;
    uint8_t* cls;
    int32_t* qlist;
    uint4* qthr;      // beside qlist: the slot's (thr_t, thr_p, query id, 0)
    int32_t* counts;  // [0..N_CLS) class sizes, [N_CLS] work items
    int64_t qcap;
    int force_exact;
    int scan_grid;    // k_scan's CTAs (the last qprep block partitions the scan over them)
};

// (7) per-query thresholds in competition-rank space and the query class.
// Kt = #points with !(t_hat*bias < target)  (controller.hpp:163; monotone in t_hat)
// Kp = #points with p_node <= budget        (controller.hpp:155)
// A point is t-feasible iff its rank r_t < Kt (every feasible value is strictly
// better than every infeasible one), likewise for p.
// Number of leading merged entries (order o) whose decoded value satisfies the
// monotone predicate pred (true on a prefix): a search over a shared-memory sample
// of every S-th value, then inside one S-entry window of global memory.
template <class Pred>
__device__ __forceinline__ int64_t count_prefix(const uint64_t* m, int o, int64_t n,
                                                const double* samp, int ns, int64_t S, Pred pred) {
    int lo = 0, hi = ns;  // first sample failing pred
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pred(samp[mid])) lo = mid + 1;
        else hi = mid;
    }
    // the count lies in [a, b]; 8-ary: each round probes 7 evenly spaced positions with
    // independent loads (2 dependent rounds for cfg2's 64-key windows instead of 6)
    int64_t a = lo == 0 ? 0 : (int64_t)(lo - 1) * S + 1;
    int64_t b = lo == ns ? n : (int64_t)lo * S;
    while (a < b) {
        const int64_t step = (b - a + 7) >> 3;
        bool t[7];
#pragma unroll
        for (int i = 0; i < 7; ++i) {
            const int64_t q = a + step * (i + 1) - 1;
            t[i] = q < b && pred(key_value(o, m[q]));
        }
        int c = 0;  // a prefix of the probes holds
#pragma unroll
        for (int i = 0; i < 7; ++i) c += t[i];
        const int64_t na = a + step * c;
        if (c < 7) b = min(b, na + step - 1);  // probe c + 1 failed (or lies past b)
        a = na;
    }
    return a;
}

// ---- pair-scan partition ----------------------------------------------
// The work of class c is T_c query tiles x the grid's n configs, laid end to end as config
// positions; a k_scan CTA walks its position range in segments cut at tile and chunk
// boundaries, and every segment pays a fixed phase (loads, barrier, the chunk's bucket
// index, thresholds) before its pairs.
//  * Cell mode (few cells: a cfg2-sized step, tiles x chunks <= CTAs). Every CTA gets
//    exactly one part of one (class, tile, chunk) cell, so no CTA pays the fixed phase twice
//    (stream-K cut ~40 % of cfg2's CTAs across a chunk or tile boundary, and those CTAs set
//    the kernel's end). The tile size (NQ <= 8 query slots per thread) and the parts per
//    chunk P minimise the largest unit: class A / C cells are cut into P parts, class B
//    cells (4 ops per pair) into 2P; a smaller NQ must win by 2 %.
//  * Stream-K otherwise: positions weighted by the class's ops per pair (A 2, B 4, C 2),
//    each CTA an equal contiguous share of the weight.
// The last qprep block writes the plan {NQ (0: stream-K), P, T_A, T_B, T_C, tq_A, tq_B, tq_C}
// to counts[kCntPlan..]; 32-bit arithmetic (class counts < 2^31, n < 2^32).
__device__ __forceinline__ uint32_t cdiv32(uint32_t a, uint32_t b) { return (a + b - 1) / b; }
__device__ __forceinline__ void scan_plan_warp(int32_t* counts, uint32_t n, uint32_t L,
                                               uint32_t G) {
    const int lane = threadIdx.x & 31;
    const uint32_t c0 = *(volatile int32_t*)&counts[0], c1 = *(volatile int32_t*)&counts[1],
                   c2 = *(volatile int32_t*)&counts[2];
    const uint32_t nch = cdiv32(n, L);
    // lane i evaluates NQ = 8 - i
    const int nq = kScanQ - lane;
    uint32_t P = 0, u = 0;
    if (lane < kScanQ - 2) {
        const uint32_t tqm = (uint32_t)kScanThreads * nq;
        const uint32_t t0 = cdiv32(c0, tqm), t1 = cdiv32(c1, tqm), t2 = cdiv32(c2, tqm);
        const uint32_t S = (t0 + 2 * t1 + t2) * nch;  // cells, class B counted twice
        if (S > 0 && S <= G && nch <= G) {
            P = G / S;
            // per-thread slot-configs of a class's largest unit (class B: twice the ops per
            // pair over half the configs)
            auto unit = [=](uint32_t cnt, uint32_t t, uint32_t h) {
                return t ? cdiv32(cdiv32(cnt, t), kScanThreads) * cdiv32(L, P * h) * h : 0u;
            };
            u = max(max(unit(c0, t0, 1), unit(c1, t1, 2)), unit(c2, t2, 1));
        }
    }
    int bnq = 0;
    uint32_t bP = 0, bu = 0;
    for (int i = 0; i < kScanQ - 2; ++i) {
        const uint32_t Pi = __shfl_sync(0xffffffffu, P, i), ui = __shfl_sync(0xffffffffu, u, i);
        if (Pi && (bnq == 0 || (uint64_t)ui * 50 < (uint64_t)bu * 49)) {
            bnq = kScanQ - i;
            bP = Pi;
            bu = ui;
        }
    }
    if (lane == 0) {
        const uint32_t tqm = (uint32_t)kScanThreads * (bnq ? bnq : kScanQ);
        const uint32_t T0 = cdiv32(c0, tqm), T1 = cdiv32(c1, tqm), T2 = cdiv32(c2, tqm);
        int4 h = make_int4(bnq, (int)bP, (int)T0, (int)T1);
        int4 t = make_int4((int)T2, T0 ? (int)cdiv32(c0, T0) : 0, T1 ? (int)cdiv32(c1, T1) : 0,
                           T2 ? (int)cdiv32(c2, T2) : 0);
        *reinterpret_cast<int4*>(counts + kCntPlan) = h;
        *reinterpret_cast<int4*>(counts + kCntPlan + 4) = t;
    }
}

__device__ __forceinline__ void qprep_body(const PlanDev& d, const SelArgs& a, int bx, int nbx,
                                           double* samp_t, double* samp_p) {
    const int lane = threadIdx.x & 31;
    const int64_t S = d.samp_s;
    const int ns = d.samp_n;
    {  // written by the last merge round; all loads in flight before the shared stores
        constexpr int R = (kSamples + 255) / 256;
        uint64_t xt[R], xp[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int t = threadIdx.x + k * blockDim.x;
            xt[k] = t < ns ? __ldg(d.samp[ORD_T] + t) : 0;
            xp[k] = t < ns ? __ldg(d.samp[ORD_P] + t) : 0;
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int t = threadIdx.x + k * blockDim.x;
            if (t < ns) {
                samp_t[t] = key_value(ORD_T, xt[k]);
                samp_p[t] = key_value(ORD_P, xp[k]);
            }
        }
    }
    __syncthreads();
    AQ_MARK(1);
    for (int64_t j0 = bx * (int64_t)blockDim.x; j0 < a.nq; j0 += (int64_t)nbx * blockDim.x) {
        const int64_t j = j0 + threadIdx.x;
        int c = -1;
        if (j < a.nq) {
            const pals_query q = a.q[j];
            const bool bset = q.has_budget != 0;
            uint32_t Kt = 0, Kp = (uint32_t)d.n;
            if (q.objective == PALS_OBJ_QOS) {
                const double target = q.throughput_tps * (1.0 + q.target_headroom);
                const double bias = q.bias;
                Kt = (uint32_t)count_prefix(d.merged[ORD_T], ORD_T, d.n, samp_t, ns, S,
                                            [&](double t) { return !(t * bias < target); });
            }
            if (bset) {
                const double budget = q.power_budget_w * (1.0 - q.budget_margin);
                Kp = (uint32_t)count_prefix(d.merged[ORD_P], ORD_P, d.n, samp_p, ns, S,
                                            [&](double p) { return p <= budget; });
            }
            // Kt as a prefix count needs !(t*bias < target) to be monotone along the
            // descending t order, i.e. bias >= 0 (or NaN: true everywhere); a negative
            // bias makes the feasible set a suffix, so such queries take the literal fold
            if (a.force_exact || d.globals[2] || (q.objective == PALS_OBJ_QOS && q.bias < 0.0))
                c = CLS_X;
            else if (q.objective == PALS_OBJ_QOS && !bset) c = Kt ? CLS_A : CLS_D;
            else if (q.objective == PALS_OBJ_QOS) c = (Kp == 0) ? CLS_D : (Kt ? CLS_B : CLS_C);
            else c = (bset && Kp) ? CLS_C : CLS_D;
            // inclusive thresholds: feasible <=> key <= (K << tr_bits) - 1
            // the scan's thresholds: feasible <=> rank <= K - 1
            a.thr_t[j] = Kt ? (uint64_t)(Kt - 1) : 0;
            a.thr_p[j] = Kp ? (uint64_t)(Kp - 1) : 0;
            a.best_e[j] = kNone64;
            a.best_t[j] = kNone64;
            a.cls[j] = (uint8_t)c;
        }
        // warp-aggregated bucket append
        for (int k = 0; k < N_CLS; ++k) {
            const unsigned m = __ballot_sync(0xffffffffu, c == k);
            if (!m) continue;
            int base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(&a.counts[k], __popc(m));
            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
            if (c == k) {
                const int64_t slot = k * a.qcap + base + __popc(m & ((1u << lane) - 1));
                a.qlist[slot] = (int32_t)j;
                a.qthr[slot] =
                    make_uint4((uint32_t)a.thr_t[j], (uint32_t)a.thr_p[j], (uint32_t)j, 0u);
            }
        }
    }
    AQ_MARK(2);
    // the last qprep block sees the final class sizes and partitions the pair scan once
    // for every k_scan CTA (a per-CTA search sat on each CTA's critical path)
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&a.counts[kCntDone], 1) == nbx - 1;
    }
    __syncthreads();
    if (last && threadIdx.x < 32) {
        __threadfence();
        scan_plan_warp(a.counts, (uint32_t)d.n, (uint32_t)d.lch, (uint32_t)a.scan_grid);
    }
}

__global__ void k_qprep(PlanDev d, SelArgs a) {
    pdl_wait();
    __shared__ double samp_t[kSamples], samp_p[kSamples];
    qprep_body(d, a, blockIdx.x, gridDim.x, samp_t, samp_p);
}

// k_assign and k_qprep in one launch (the captured step): qprep reads only the merged
// arrays, so its blocks run beside the assign blocks. One flat grid, the qb qprep blocks
// first (they carry the longer dependent chain: the search index, two threshold searches
// per query, then the scan partition), then eb assign blocks per order; at most 6 blocks of
// 256 threads per SM (42 registers) so that every block of cfg2's launch is resident at once
// (at 46 registers 5 fit, and a second wave of ~270 blocks — the qprep row last — started
// 5 us late).
__global__ void __launch_bounds__(256, 6) k_assign_qprep(PlanDev d, uint64_t* gk,
                                                         uint32_t* done, SelArgs a, int eb,
                                                         int qb) {
    pdl_wait();
    AQ_MARK(0);
    __shared__ uint64_t sbuf[2 * kSamples];
    const int b = (int)blockIdx.x;
    if (b >= qb) {
        const int o = (b - qb) / eb;
        assign_body(d, gk, done, o, b - qb - o * eb, eb, sbuf);
    } else {
        qprep_body(d, a, b, qb, reinterpret_cast<double*>(sbuf),
                   reinterpret_cast<double*>(sbuf) + kSamples);
    }
    AQ_MARK(7);
}

// (8) the pair scan: every (query, config) pair of classes A/B/C is decided, on chunk-local
// 16-bit ranks two configs per 32-bit register.
//
// Chunk-local ranks (every prepare). The grid's TR range is cut into the chunk sort's
// chunks of L <= 2,048 points; the chunk sort's value-sorted run of a chunk lists its points
// in global merged-position order. Per point (written by k_sort_chunks): lr = its
// competition rank inside its chunk, lq = its place in the chunk's run; per run place
// (written by the rank pass): cinv = the global merged position. A query's feasible set
// on a side is the position prefix [0, K); with k = #(run places whose
// position is < K): feasible <=> lr < k, and the smallest global position among a chunk's
// feasible points is cinv[min lq over them] (lq orders a chunk exactly as the global
// positions do). So one chunk is decided in 16-bit lanes:
//   d = (0x8000 + k - 1) - lr            in [0x8000 - 2049, 0x8000 + 2047]: bit 15 set
//                                        iff feasible, and no borrow between the lanes
//   v = lq | (~d & 0x8000)               infeasible -> >= 0x8000 > every feasible lq
//   m = min(m, v)                        VIMNMX3.U16x2: two new registers per instruction
// With both configs of a register in its two lanes: per 4 pairs one IMAD.IADD (FMA pipe)
// per 2 configs, one LOP3 per 2, one VIMNMX3.U16x2 per 4 — 0.75 ALU-pipe instructions
// per pair (classes A / C), 2 for class B (dt & dp, two LOP3, two minima), where 32-bit
// lanes took 1.5 / 3.5.
constexpr uint32_t kPadRank = 0x7FFFFFFFu;
constexpr uint32_t kLrPad = kLrPadSort;  // a chunk-local rank no threshold reaches
constexpr uint32_t kFlag2 = 0x80008000u;

// number of run places of a chunk with global position <= thr = K - 1 (the chunk-local
// threshold): a binary search over the staged, ascending run positions (a branchless
// fixed-step search measured slower on cfg3: more registers in the scan)
__device__ __forceinline__ uint32_t local_count(const uint32_t* sr, int L, uint32_t thr) {
    int lo = 0, hi = L;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sr[mid] <= thr) lo = mid + 1;
        else hi = mid;
    }
    return (uint32_t)lo;
}

__device__ __forceinline__ uint32_t kb2(uint32_t k) {  // both lanes: 0x8000 + k - 1
    const uint32_t v = 0x8000u + k - 1u;
    return v | (v << 16);
}

__device__ __forceinline__ uint32_t lane_min(uint32_t m2) {
    return min(m2 & 0xFFFFu, m2 >> 16);
}

// One chunk segment of one query tile, classes A / C: the words are staged as
// {lr(2c, 2c+1), lq(2c, 2c+1)} pairs, 2 words (4 configs) per LDS.128.
template <int NQ>
__device__ __forceinline__ void scan_seg1(const uint4* __restrict__ w, int nw4,
                                          const uint32_t (&K)[kScanQ], uint32_t (&m)[kScanQ]) {
    for (int c = 0; c < nw4; ++c) {
        const uint4 v = w[c];  // x: lr word 0, y: lq word 0, z: lr word 1, w: lq word 1
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
            const uint32_t d0 = K[j] - v.x, d1 = K[j] - v.z;
            const uint32_t a0 = v.y | (~d0 & kFlag2), a1 = v.w | (~d1 & kFlag2);
            m[j] = __vimin3_u16x2(m[j], a0, a1);
        }
    }
}

// class B: words {lrt, lrp, lqe, lqt} per config pair, 1 LDS.128 per 2 configs
template <int NQ>
__device__ __forceinline__ void scan_seg2(const uint4* __restrict__ w, int nw,
                                          const uint32_t (&Kt)[kScanQ],
                                          const uint32_t (&Kp)[kScanQ], uint32_t (&me)[kScanQ],
                                          uint32_t (&mt)[kScanQ]) {
    for (int c = 0; c + 1 < nw; c += 2) {
        const uint4 v0 = w[c], v1 = w[c + 1];
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
            const uint32_t dt0 = Kt[j] - v0.x, dp0 = Kp[j] - v0.y;
            const uint32_t dt1 = Kt[j] - v1.x, dp1 = Kp[j] - v1.y;
            const uint32_t e0 = v0.z | (~(dt0 & dp0) & kFlag2);
            const uint32_t e1 = v1.z | (~(dt1 & dp1) & kFlag2);
            const uint32_t t0 = v0.w | (~dp0 & kFlag2), t1 = v1.w | (~dp1 & kFlag2);
            me[j] = __vimin3_u16x2(me[j], e0, e1);
            mt[j] = __vimin3_u16x2(mt[j], t0, t1);
        }
    }
}

// the pair scan's partition (scan_plan_warp): this CTA's [p0, p1) of config positions
struct ScanPlan {
    int tq0, tq1, tq2;  // queries per tile of each class (balanced, <= NQ x 256)
    int64_t pb1, pb2;   // config position where classes B and C start (A at 0)
};

__device__ __forceinline__ void scan_partition(const int32_t* __restrict__ counts, int64_t n, int L,
                                               int b, int G, ScanPlan& pl, int64_t& p0,
                                               int64_t& p1) {
    const int4 h = __ldg(reinterpret_cast<const int4*>(counts + kCntPlan));
    const int4 t = __ldg(reinterpret_cast<const int4*>(counts + kCntPlan + 4));
    const int bnq = h.x, bP = h.y;
    const uint32_t T0 = h.z, T1 = h.w, T2 = t.x;
    pl.tq0 = t.y;
    pl.tq1 = t.z;
    pl.tq2 = t.w;
    const int64_t pb1 = (int64_t)T0 * n, pb2 = pb1 + (int64_t)T1 * n, pb3 = pb2 + (int64_t)T2 * n;
    pl.pb1 = pb1;
    pl.pb2 = pb2;
    if (bnq) {  // cell mode: cells x parts <= G, 32-bit throughout
        const uint32_t nch = cdiv32((uint32_t)n, (uint32_t)L);
        const uint32_t u1 = T0 * nch * bP, u2 = u1 + T1 * nch * 2 * bP, u3 = u2 + T2 * nch * bP;
        p0 = p1 = 0;
        if ((uint32_t)b >= u3) return;
        const int c = ((uint32_t)b >= u1) + ((uint32_t)b >= u2);
        const uint32_t Pc = c == CLS_B ? 2 * bP : bP;
        const uint32_t r = (uint32_t)b - (c == 0 ? 0u : c == 1 ? u1 : u2);
        const uint32_t cell = r / Pc, part = r - cell * Pc;
        const uint32_t tile = cell / nch, ch = cell - tile * nch;
        const uint32_t len = min((uint32_t)L, (uint32_t)n - ch * L);
        const int64_t base = (c == 0 ? 0 : c == 1 ? pb1 : pb2) + (int64_t)tile * n + ch * L;
        p0 = base + len * part / Pc;
        p1 = base + len * (part + 1) / Pc;
        return;
    }
    const int64_t w1 = (int64_t)T0 * n * 2, w2 = w1 + (int64_t)T1 * n * 4,
                  W = w2 + (int64_t)T2 * n * 2;
    auto pos_of = [=](int64_t u) {
        if (u >= W) return pb3;
        return u >= w2 ? pb2 + (u - w2) / 2 : u >= w1 ? pb1 + (u - w1) / 4 : u / 2;
    };
    p0 = pos_of(W * b / G);
    p1 = pos_of(W * (b + 1) / G);
}

// Bucket index over a chunk's staged run positions (ascending): T[b] = number of places
// whose position is < b << sh, for b = 0..nb - 1 (nb = ((n - 1) >> sh) + 1 <= 1,024; the
// count below nb << sh is every valid place). A query's chunk-local threshold is then a
// search inside one bucket (~2 places for cfg2) instead of over the whole chunk, whose 11
// dependent, bank-conflicted shared-memory steps per query (lanes hold unrelated queries)
// cost ~7 us per segment. Built without atomics: the last place of each non-empty bucket
// writes T[b + 1], then a block prefix max fills the empty buckets (every thread owns 4
// consecutive entries: one LDS.64 / STS.64).
constexpr int kScanBk = 1024;  // u16 entries per side
static_assert(kScanBk == 4 * kScanThreads, "bucket scan: 4 entries per thread");
__device__ __forceinline__ void bucket_mark(const uint32_t* sr, int L, uint16_t* T, int sh,
                                            int nb) {
    for (int i = threadIdx.x; i < L; i += kScanThreads) {
        const uint32_t v = sr[i];
        if (v == 0xFFFFFFFFu) continue;  // padding of the last chunk
        const int b = (int)(v >> sh);
        if (b + 1 < nb && (i == L - 1 || (int)(sr[i + 1] >> sh) != b || sr[i + 1] == 0xFFFFFFFFu))
            T[b + 1] = (uint16_t)(i + 1);
    }
}
// Stage the chunk's L run positions (ascending; 0xFFFFFFFF pads the last chunk) into sr and
// mark each non-empty bucket's last place in T (T zeroed beforehand): T[b + 1] = last + 1.
// Thread t holds places [t PL, (t + 1) PL), PL = L / 256 (L = 256 .. 2,048).
__device__ __forceinline__ void stage_marks(const uint32_t* __restrict__ src, int L, uint32_t* sr,
                                            uint16_t* T, int sh, int nb) {
    const int PL = L / kScanThreads;
    const int i0 = threadIdx.x * PL;
    uint32_t v[8];
    if (PL == 8) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(src + i0));
        const uint4 b = __ldg(reinterpret_cast<const uint4*>(src + i0) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = k < PL ? __ldg(src + i0 + k) : 0xFFFFFFFFu;
    }
    // the position after this thread's last place: the next lane's first (lane 31: a load)
    uint32_t nx = __shfl_down_sync(0xffffffffu, v[0], 1);
    if ((threadIdx.x & 31) == 31) nx = i0 + PL < L ? __ldg(src + i0 + PL) : 0xFFFFFFFFu;
    if (PL == 8) {
        reinterpret_cast<uint4*>(sr + i0)[0] = make_uint4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<uint4*>(sr + i0)[1] = make_uint4(v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < PL) sr[i0 + k] = v[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k >= PL || v[k] == 0xFFFFFFFFu) continue;
        const uint32_t nv = k + 1 < PL ? v[k + 1 < 8 ? k + 1 : 7] : nx;
        const int b = (int)(v[k] >> sh);
        if (b + 1 < nb && (nv == 0xFFFFFFFFu || (int)(nv >> sh) != b))
            T[b + 1] = (uint16_t)(i0 + k + 1);
    }
}

__device__ __forceinline__ void bucket_scan(uint16_t* T, uint32_t* wtot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint2 raw = reinterpret_cast<uint2*>(T)[threadIdx.x];
    uint32_t e[4] = {raw.x & 0xFFFFu, raw.x >> 16, raw.y & 0xFFFFu, raw.y >> 16};
#pragma unroll
    for (int k = 1; k < 4; ++k) e[k] = max(e[k], e[k - 1]);
    uint32_t x = e[3];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = max(x, y);
    }
    if (lane == 31) wtot[warp] = x;
    uint32_t pre = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) pre = 0;
    __syncthreads();
    for (int w = 0; w < warp; ++w) pre = max(pre, wtot[w]);
#pragma unroll
    for (int k = 0; k < 4; ++k) e[k] = max(e[k], pre);
    reinterpret_cast<uint2*>(T)[threadIdx.x] = make_uint2(e[0] | (e[1] << 16), e[2] | (e[3] << 16));
}
__device__ __forceinline__ uint32_t bucket_count(const uint32_t* sr, const uint16_t* T, int sh,
                                                 int nb, int nvalid, uint32_t thr) {
    const int b = (int)(thr >> sh);
    int lo = T[b], hi = b + 1 < nb ? (int)T[b + 1] : nvalid;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sr[mid] <= thr) lo = mid + 1;
        else hi = mid;
    }
    return (uint32_t)lo;
}

// shared memory of k_scan: a chunk's staged words (class B: 2,048 x 16 B), its run
// positions for the chunk-local thresholds (2 x 2,048 x 4 B) and their bucket indexes
// (the words: class B stages one uint4 per config pair, at most kScanCh / 2 + 1 pairs plus
// a padding word; classes A / C half that); the bucket index is double-buffered per side
constexpr size_t kScanWords = ((size_t)(kScanCh / 2 + 2) * 16 + 127) & ~(size_t)127;
constexpr size_t kScanSmem = kScanWords + 2 * (size_t)kScanCh * 4 + 4 * (size_t)kScanBk * 2;

#ifdef PALS_SCAN_TRACE
// A/B instrumentation (scripts/build_variants.sh): globaltimer of CTA phases, thread 0
__device__ unsigned long long g_scan_trace[4096][16];
#define SCAN_MARK(k)                                                                      \
    if (threadIdx.x == 0 && blockIdx.x < 4096 && (k) < 16) {                              \
        unsigned long long t_;                                                            \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
        g_scan_trace[blockIdx.x][k] = t_;                                                 \
    }
#define SCAN_SMID()                                                                       \
    if (threadIdx.x == 0 && blockIdx.x < 4096) {                                          \
        unsigned s_;                                                                      \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s_));                                   \
        g_scan_trace[blockIdx.x][14] = s_;                                                \
    }
#else
#define SCAN_MARK(k)
#define SCAN_SMID()
#endif

__global__ void __launch_bounds__(kScanThreads, 4) k_scan(PlanDev d, SelArgs a) {
    pdl_wait();
    SCAN_MARK(0);
    SCAN_SMID();
    int mark = 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint4* sw = reinterpret_cast<uint4*>(smem_raw);
    uint32_t* ssr = reinterpret_cast<uint32_t*>(smem_raw + kScanWords);  // [2][L]
    // [2 buffers][2 sides][kScanBk]: segment s builds buffer s & 1 and zeroes the other
    uint16_t* sbk = reinterpret_cast<uint16_t*>(smem_raw + kScanWords + (size_t)kScanCh * 8);
    __shared__ uint32_t s_wtot[2][kScanThreads / 32];
    const int64_t n = d.n;
    const int L = d.lch;
    const int sh = max(0, 32 - __clz((int)(n - 1)) - 10);  // <= 1,024 buckets of 2^sh positions
    const int nb = (int)((n - 1) >> sh) + 1;
    ScanPlan pl;
    int64_t p0, p1;
    scan_partition(a.counts, n, L, blockIdx.x, gridDim.x, pl, p0, p1);
    int64_t pos = p0;
    int seg = 0;  // this CTA's segment count: its parity selects the bucket-index buffer
    reinterpret_cast<uint4*>(sbk)[threadIdx.x] = make_uint4(0u, 0u, 0u, 0u);  // buffer 0
    while (pos < p1) {
        // locate (class, tile, first config) of pos and the end of that tile segment;
        // configs are TR positions, cut further at the chunks of the local ranks
        // (register selects, not indexed loads: the plan stays in registers, no local stack)
        const int c = (pos >= pl.pb1) + (pos >= pl.pb2);
        const int64_t pb = c == 0 ? 0 : c == 1 ? pl.pb1 : pl.pb2;
        const int64_t tqc = c == 0 ? pl.tq0 : c == 1 ? pl.tq1 : pl.tq2;
        const int64_t r = pos - pb;
        // 32-bit divisions where the operands fit (j0 < n < 2^32)
        const int64_t tile = (r >> 32) ? r / n : (int64_t)((uint32_t)r / (uint32_t)n);
        const int64_t j0 = r - tile * n;
        const int64_t cb = (int64_t)(((uint32_t)j0 / (uint32_t)L) * (uint32_t)L);  // chunk's first TR
        const int64_t chunk_end = cb + L;
        const int64_t seg_end = min(min(p1, pb + (tile + 1) * n), pos + (chunk_end - j0));
        const int64_t j1 = j0 + (seg_end - pos);
        // this tile's queries: 8 per thread (slot validity needs no load)
        const int64_t q_lo = tile * tqc, q_hi = min((int64_t)a.counts[c], q_lo + tqc);
        // query slots of this warp that hold a query (warp-uniform): the loop is instantiated
        // per count, so empty slots cost no ALU work
        const int qlen = (int)(q_hi - q_lo), wbase = (int)(threadIdx.x & ~31u);
        const int nqw =
            qlen > wbase ? min(kScanQ, (qlen - wbase + kScanThreads - 1) / kScanThreads) : 0;
        const int64_t w0 = j0 >> 1, w1 = (j1 + 1) >> 1;  // config pairs
        const int nw = (int)(w1 - w0);
        __syncthreads();  // the previous segment is done with shared memory
        // every global load of the segment is issued before the barrier: the query slots'
        // ids and thresholds (written beside the class list by qprep, so no id -> threshold
        // indirection), the segment's config words (whole pairs; lanes outside [j0, j1)
        // padded infeasible) and the chunk's run positions
        int32_t qid[kScanQ];
        uint2 qt[kScanQ];
#pragma unroll
        for (int q = 0; q < kScanQ; ++q) {  // one 16-byte record per slot
            const int64_t sq = q_lo + q * kScanThreads + threadIdx.x;
            const uint4 r = sq < q_hi ? __ldg(a.qthr + c * a.qcap + sq) : make_uint4(0u, 0u, ~0u, 0u);
            qid[q] = (int32_t)r.z;
            qt[q] = make_uint2(r.x, r.y);
        }
        const uint32_t* lrt = reinterpret_cast<const uint32_t*>(d.lr16[ORD_T]);
        const uint32_t* lrp = reinterpret_cast<const uint32_t*>(d.lr16[ORD_P]);
        const uint32_t* lqe = reinterpret_cast<const uint32_t*>(d.lq16[ORD_E]);
        const uint32_t* lqt = reinterpret_cast<const uint32_t*>(d.lq16[ORD_T]);
        auto edge = [&](uint32_t wv, int64_t w) {  // pad the lanes outside [j0, j1)
            if (2 * w < j0) wv = (wv & 0xFFFF0000u) | kLrPad;
            if (2 * w + 1 >= j1) wv = (wv & 0x0000FFFFu) | (kLrPad << 16);
            return wv;
        };
        if (c == CLS_B) {
            for (int i = threadIdx.x; i < nw + 1; i += kScanThreads) {
                const int64_t w = w0 + i;
                uint4 v = make_uint4(kLrPad | (kLrPad << 16), kLrPad | (kLrPad << 16), 0u, 0u);
                if (i < nw) {
                    v.x = edge(__ldg(lrt + w), w);
                    v.y = edge(__ldg(lrp + w), w);
                    v.z = __ldg(lqe + w);
                    v.w = __ldg(lqt + w);
                }
                sw[i] = v;
            }
        } else {
            const uint32_t* lr = c == CLS_A ? lrt : lrp;
            const uint32_t* lq = c == CLS_A ? lqe : lqt;
            // 2 words per uint4; a trailing half-filled uint4 is padded infeasible
            const int nw4 = (nw + 1) >> 1;
            for (int i = threadIdx.x; i < nw4; i += kScanThreads) {
                const int64_t wa = w0 + 2 * i, wb = wa + 1;
                uint4 v;
                v.x = edge(__ldg(lr + wa), wa);
                v.y = __ldg(lq + wa);
                v.z = wb < w1 ? edge(__ldg(lr + wb), wb) : (kLrPad | (kLrPad << 16));
                v.w = wb < w1 ? __ldg(lq + wb) : 0u;
                sw[i] = v;
            }
        }
        // the chunk's run positions on the feasibility side(s): a query's chunk-local
        // threshold is the number of run entries inside its feasible prefix [0, K). Thread t
        // stages places [t PL, (t + 1) PL) and marks the bucket ends among them straight from
        // its registers (the next place's position from the next lane), so the bucket index
        // needs no separate shared-memory pass and barrier. The index is double-buffered:
        // this segment's buffer was zeroed by the previous segment (or the kernel start),
        // which now zeroes the next one; the top barrier orders both.
        const int ko = c == CLS_C ? ORD_P : ORD_T;
        const int nvalid = (int)min((int64_t)L, n - cb);
        uint16_t* const t1 = sbk + (seg & 1) * 2 * kScanBk;  // side 1; side 2 at + kScanBk
        stage_marks(ko == ORD_P ? d.cinv[ORD_P] + cb : d.cinv[ORD_T] + cb, L, ssr, t1, sh, nb);
        if (c == CLS_B) stage_marks(d.cinv[ORD_P] + cb, L, ssr + L, t1 + kScanBk, sh, nb);
        reinterpret_cast<uint4*>(sbk + ((seg + 1) & 1) * 2 * kScanBk)[threadIdx.x] =
            make_uint4(0u, 0u, 0u, 0u);  // the next segment's buffer, both sides
        SCAN_MARK(mark);
        ++mark;
        __syncthreads();
        bucket_scan(t1, s_wtot[0]);
        if (c == CLS_B) bucket_scan(t1 + kScanBk, s_wtot[1]);
        __syncthreads();
        SCAN_MARK(mark);
        ++mark;
        // chunk-local thresholds of the 8 queries
        uint32_t K1[kScanQ], K2[kScanQ], m1[kScanQ], m2[kScanQ];
#pragma unroll
        for (int q = 0; q < kScanQ; ++q) {
            K1[q] = kb2(bucket_count(ssr, t1, sh, nb, nvalid, c == CLS_C ? qt[q].y : qt[q].x));
            K2[q] = c == CLS_B ? kb2(bucket_count(ssr + L, t1 + kScanBk, sh, nb, nvalid, qt[q].y))
                               : 0u;
            m1[q] = m2[q] = 0xFFFFFFFFu;
        }
        SCAN_MARK(mark);
        ++mark;
        SCAN_MARK(mark);
        ++mark;
        if (c == CLS_B) {
            const int nw2 = nw + (nw & 1);
            switch (nqw) {
                case 8: scan_seg2<8>(sw, nw2, K1, K2, m1, m2); break;
                case 7: scan_seg2<7>(sw, nw2, K1, K2, m1, m2); break;
                case 6: scan_seg2<6>(sw, nw2, K1, K2, m1, m2); break;
                case 5: scan_seg2<5>(sw, nw2, K1, K2, m1, m2); break;
                case 4: scan_seg2<4>(sw, nw2, K1, K2, m1, m2); break;
                case 3: scan_seg2<3>(sw, nw2, K1, K2, m1, m2); break;
                case 2: scan_seg2<2>(sw, nw2, K1, K2, m1, m2); break;
                case 1: scan_seg2<1>(sw, nw2, K1, K2, m1, m2); break;
                default: break;
            }
        } else {
            const int nw4 = (nw + 1) >> 1;
            switch (nqw) {
                case 8: scan_seg1<8>(sw, nw4, K1, m1); break;
                case 7: scan_seg1<7>(sw, nw4, K1, m1); break;
                case 6: scan_seg1<6>(sw, nw4, K1, m1); break;
                case 5: scan_seg1<5>(sw, nw4, K1, m1); break;
                case 4: scan_seg1<4>(sw, nw4, K1, m1); break;
                case 3: scan_seg1<3>(sw, nw4, K1, m1); break;
                case 2: scan_seg1<2>(sw, nw4, K1, m1); break;
                case 1: scan_seg1<1>(sw, nw4, K1, m1); break;
                default: break;
            }
        }
        SCAN_MARK(mark);
        ++mark;
        // chunk minima -> global merged positions -> the queries' running minima
        const uint32_t* inv_a = (c == CLS_C ? d.cinv[ORD_T] : d.cinv[ORD_E]) + cb;
#pragma unroll
        for (int q = 0; q < kScanQ; ++q) {
            if (qid[q] < 0) continue;
            const uint32_t la = lane_min(m1[q]);
            if (la < 0x8000u)
                atomicMin((unsigned long long*)(c == CLS_C ? &a.best_t[qid[q]] : &a.best_e[qid[q]]),
                          (unsigned long long)__ldg(inv_a + la));
            if (c == CLS_B) {
                const uint32_t lb = lane_min(m2[q]);
                if (lb < 0x8000u)
                    atomicMin((unsigned long long*)&a.best_t[qid[q]],
                              (unsigned long long)__ldg(d.cinv[ORD_T] + cb + lb));
            }
        }
        pos = seg_end;
        ++seg;
        SCAN_MARK(mark);
        ++mark;
    }
    SCAN_MARK(15);
    (void)mark;
}

#ifdef PALS_SCAN_TRACE
extern "C" int pals_debug_aq_trace(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, g_aq_trace, sizeof(g_aq_trace));
}
extern "C" int pals_debug_scan_trace(unsigned long long* host, int n_rows) {
    return (int)cudaMemcpyFromSymbol(host, g_scan_trace, (size_t)min(n_rows, 4096) * 16 * 8);
}
#endif

// ---- time to decide: prefix-min tables instead of the pair scan -----------------------
// Feasibility is a prefix of the sorted orders (Kt of the t_hat order, Kp of the p_node
// order), so the argmins the pair scan folds are prefix minima:
//   class A (QoS, no budget): min pos_e over t-positions [0, Kt)       = PM_A[Kt - 1]
//   class C (budget)        : min pos_t over p-positions [0, Kp)       = PM_C[Kp - 1]
//   class B (QoS + budget)  : min pos_e over {t-pos < Kt, p-pos < Kp}: a 2-D dominance
//     minimum = TB_b[Kp - 1] over the first b = floor(Kt / B) whole blocks of B t-positions
//     (TB_b = prefix minimum along the p order of pos_e restricted to t-pos < b B), folded
//     with the < B remaining t-positions, which one warp reads from te[] (p-pos, pos_e in
//     t order); its budget branch is PM_C[Kp - 1].
// The minima are the same merged positions the scan produces (min is exact and
// associative), so k_finalize (near-tie folds included) is shared.
constexpr int kDecTile = 1024;        // elements per scan tile (256 threads x 4)
constexpr int kDecMaxBlocks = 64;     // at most 64 2-D table rows

struct DecDev {
    int64_t n;
    int B, nb, ntiles;
    uint32_t* elemA;   // pos_e at every t-position
    uint32_t* elemC;   // pos_t at every p-position
    uint2* te;         // (p-pos, pos_e) at every t-position
    uint2* pt;         // (t-pos, pos_e) at every p-position
    uint32_t* agg;     // [rows][ntiles] tile minima
    uint32_t* tab;     // [rows][n]: row 0 PM_A, row 1 PM_C, row 1 + b TB_b (b = 1..nb)
};

__global__ void k_dec_elems(PlanDev d, DecDev t) {
    pdl_wait();
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < d.n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t it = d.midx[ORD_T][p], ip = d.midx[ORD_P][p];
        const uint32_t e_t = d.pos32[ORD_E][it], e_p = d.pos32[ORD_E][ip];
        t.elemA[p] = e_t;
        t.te[p] = make_uint2(d.pos32[ORD_P][it], e_t);
        t.elemC[p] = d.pos32[ORD_T][ip];
        t.pt[p] = make_uint2(d.pos32[ORD_T][ip], e_p);
    }
}

__device__ __forceinline__ uint32_t dec_elem(const DecDev& t, int row, int64_t i) {
    if (i >= t.n) return kNone32;
    if (row == 0) return t.elemA[i];
    if (row == 1) return t.elemC[i];
    const uint2 v = t.pt[i];  // row 1 + b: the points in the first b blocks of t-positions
    return v.x < (uint32_t)((row - 1) * t.B) ? v.y : kNone32;
}

// (a) per (row, tile) minimum
__global__ void __launch_bounds__(256) k_dec_tiles(DecDev t) {
    pdl_wait();
    const int row = blockIdx.y, tile = blockIdx.x;
    uint32_t m = kNone32;
#pragma unroll
    for (int k = 0; k < kDecTile / 256; ++k)
        m = min(m, dec_elem(t, row, (int64_t)tile * kDecTile + k * 256 + threadIdx.x));
    m = __reduce_min_sync(0xffffffffu, m);
    __shared__ uint32_t w[8];
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t x = threadIdx.x < 8 ? w[threadIdx.x] : kNone32;
        x = __reduce_min_sync(0xffffffffu, x);
        if (threadIdx.x == 0) t.agg[(int64_t)row * t.ntiles + tile] = x;
    }
}

// (b) per (row, tile) inclusive prefix minimum with the carry of the earlier tiles
__global__ void __launch_bounds__(256) k_dec_scan(DecDev t) {
    pdl_wait();
    const int row = blockIdx.y, tile = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ uint32_t s_carry, w[8];
    if (threadIdx.x < 32) {
        uint32_t c = kNone32;
        for (int j = lane; j < tile; j += 32) c = min(c, t.agg[(int64_t)row * t.ntiles + j]);
        c = __reduce_min_sync(0xffffffffu, c);
        if (lane == 0) s_carry = c;
    }
    const int64_t base = (int64_t)tile * kDecTile + threadIdx.x * 4;
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = dec_elem(t, row, base + k);
#pragma unroll
    for (int k = 1; k < 4; ++k) v[k] = min(v[k], v[k - 1]);
    uint32_t x = v[3];  // thread total -> warp inclusive scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = min(x, y);
    }
    if (lane == 31) w[wid] = x;
    __syncthreads();
    uint32_t pre = s_carry;  // earlier tiles, earlier warps, earlier lanes
    for (int j = 0; j < wid; ++j) pre = min(pre, w[j]);
    const uint32_t up = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane > 0) pre = min(pre, up);
    uint32_t* out = t.tab + (int64_t)row * t.n;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (base + k < t.n) out[base + k] = min(pre, v[k]);
}

// (c) one warp per scanned query: the table lookups (and class B's residual block)
__global__ void __launch_bounds__(256) k_decide(DecDev t, SelArgs a) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t cA = a.counts[CLS_A], cB = a.counts[CLS_B], cC = a.counts[CLS_C];
    const int64_t total = cA + cB + cC;
    const uint32_t* PMA = t.tab;
    const uint32_t* PMC = t.tab + t.n;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < total;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int c;
        int64_t i;
        if (w < cA) { c = CLS_A; i = w; }
        else if (w < cA + cB) { c = CLS_B; i = w - cA; }
        else { c = CLS_C; i = w - cA - cB; }
        const int32_t qid = a.qlist[c * a.qcap + i];
        const uint32_t kt = (uint32_t)a.thr_t[qid], kp = (uint32_t)a.thr_p[qid];  // K - 1
        if (c == CLS_A) {
            if (lane == 0) a.best_e[qid] = PMA[kt];
            continue;
        }
        if (lane == 0) a.best_t[qid] = PMC[kp];
        if (c == CLS_C) continue;
        const uint32_t Kt = kt + 1;
        const uint32_t b = Kt / (uint32_t)t.B;  // whole blocks of t-positions
        uint32_t m = b ? t.tab[(int64_t)(1 + b) * t.n + kp] : kNone32;
        for (uint32_t p = b * (uint32_t)t.B + lane; p < Kt; p += 32) {
            const uint2 v = t.te[p];
            if (v.x <= kp) m = min(m, v.y);
        }
        m = __reduce_min_sync(0xffffffffu, m);
        if (lane == 0 && m != kNone32) a.best_e[qid] = m;
    }
}

// exact feasibility of point c for query q (FP64, controller.hpp:155, 163)
__device__ __forceinline__ bool feasible_t(const PlanDev& d, const pals_query& q, int64_t c) {
    const double target = q.throughput_tps * (1.0 + q.target_headroom);
    return !(d.th[c] * q.bias < target);
}
__device__ __forceinline__ bool feasible_p(const PlanDev& d, const pals_query& q, int64_t c) {
    if (!q.has_budget) return true;
    return d.pn[c] <= q.power_budget_w * (1.0 - q.budget_margin);
}

// (9) decide every query from its two minima. A query whose winner sits in a near-tie
// cluster (or every query of a generic plan) is re-decided by the exact fold, run by
// the deciding warp itself: the lanes that need one are folded one after another
// (10), so no second launch or work queue sits in the step.
__device__ __forceinline__ void exact_item(const PlanDev& d, const SelArgs& a, int32_t qid,
                                           int mode, uint32_t d0) {
    const pals_query q = a.q[qid];
    if (mode == EX_FULL) {
        warp_select_full(d, q, &a.out_idx[qid], &a.out_reason[qid]);
        return;
    }
    int best;
    int r;
    if (mode == EX_QOS_NEAR) {
        const uint32_t cut = cluster_end(d, ORD_E, d0);
        best = warp_fold(
            d.n, d.cap, d.batch,
            [&](int64_t c) {
                return rank_of(d, ORD_E, c) <= cut && feasible_t(d, q, c) &&
                       feasible_p(d, q, c);
            },
            [&](int64_t c) { return d.ef[c]; });
        r = PALS_REASON_QOS_FEASIBLE;
    } else {
        const uint32_t cut = cluster_end(d, ORD_T, d0);
        best = warp_fold(
            d.n, d.cap, d.batch,
            [&](int64_t c) { return rank_of(d, ORD_T, c) <= cut && feasible_p(d, q, c); },
            [&](int64_t c) { return d.th[c]; });
        r = PALS_REASON_BUDGET_MAX_T;
    }
    if ((threadIdx.x & 31) == 0) {
        a.out_idx[qid] = best;
        a.out_reason[qid] = (uint8_t)r;
    }
}

__global__ void k_finalize(PlanDev d, SelArgs a) {
    pdl_wait();
    const uint64_t none = kNone64;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); j0 < a.nq;
         j0 += stride) {  // whole warps: the exact folds below need every lane
        const int64_t j = j0 + lane;
        int mode = -1;
        uint32_t d0 = 0;
        if (j < a.nq) {
            const int c = a.cls[j];
            const pals_query q = a.q[j];
            // the minima are merged positions (packed-key order): the winner is the
            // point that position carries, its competition rank picks the near-tie flag
            const uint64_t be = a.best_e[j], bt = a.best_t[j];
            int32_t idx = -1;
            int r = PALS_REASON_FALLBACK_MAX_T;
            if (c == CLS_X) {
                mode = EX_FULL;
            } else {
                if ((c == CLS_A || c == CLS_B) && be != none) {
                    const int32_t pt = (int32_t)d.midx[ORD_E][be];
                    const uint32_t rk = d.sidx[ORD_E][be];
                    if (d.danger[ORD_E][rk]) {
                        mode = EX_QOS_NEAR;
                        d0 = rk;
                    }
                    idx = pt;
                    r = PALS_REASON_QOS_FEASIBLE;
                }
                if (mode < 0 && idx < 0 && q.has_budget &&
                    (c == CLS_B || c == CLS_C || c == CLS_D)) {
                    if (c != CLS_D && bt != none) {
                        const int32_t pt = (int32_t)d.midx[ORD_T][bt];
                        const uint32_t rk = d.sidx[ORD_T][bt];
                        if (d.danger[ORD_T][rk]) {
                            mode = EX_BUD_NEAR;
                            d0 = rk;
                        }
                        idx = pt;
                    } else {
                        idx = d.globals[1];  // budget below every candidate: least power (:180-188)
                    }
                    r = PALS_REASON_BUDGET_MAX_T;
                }
                if (idx < 0) {
                    idx = d.globals[0];  // fallback: max throughput over all (:191-198)
                    r = PALS_REASON_FALLBACK_MAX_T;
                }
            }
            if (mode < 0) {
                a.out_idx[j] = idx;
                a.out_reason[j] = (uint8_t)r;
            }
        }
        unsigned m = __ballot_sync(full, mode >= 0);
        if (m && lane == 0) atomicAdd(&a.counts[N_CLS], __popc(m));  // exact-fold count
        while (m) {
            const int l = __ffs(m) - 1;
            m &= m - 1;
            const int md = __shfl_sync(full, mode, l);
            const uint32_t dd = __shfl_sync(full, d0, l);
            exact_item(d, a, (int32_t)(j0 + l), md, dd);
        }
    }
}

static int grid_blocks(pals_ctx* ctx, int64_t n, int threads) {
    const int64_t b = (n + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)ctx->num_sms * 16));
}

static int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, what);
    return PALS_OK;
}

// device-side plan state accessors used by replay.cu / forest.cu
const PlanDev& plan_dev(const pals_plan* p) { return p->d; }
int plan_error(const pals_plan* p) { return p->err; }
const pals_grid* plan_grid(const pals_plan* p) { return p->grid; }

__global__ void k_finish(PlanDev d, double alpha, double beta) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.n;
         i += (int64_t)gridDim.x * blockDim.x)
        finish_scores(d, i, d.T[i], d.P[i], d.dp[i], alpha, beta);
}

// derived scores (t_hat, p_node, eff, sort keys) from T/P already in the plan
int plan_finish_scores(pals_plan* p) {
    k_finish<<<grid_blocks(p->ctx, p->n, 256), 256, 0, p->ctx->stream>>>(p->d, p->coeffs.alpha,
                                                                       p->coeffs.beta_watts);
    count_launch(p->ctx);
    return check_launch("k_finish");
}

__global__ void k_eval_analytic_raw(const Analytic* __restrict__ an, int64_t n,
                                    const double* __restrict__ cap, const int* __restrict__ batch,
                                    const int* __restrict__ tp, const int* __restrict__ dp,
                                    double* __restrict__ T, double* __restrict__ P) {
    const Analytic& a = *an;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const Score s = analytic_score(a, cap[i], batch[i], tp[i], dp[i]);
        T[i] = s.T;
        P[i] = s.P;
    }
}

}  // namespace pals

extern "C" {

static int plan_build(pals_ctx* ctx, const pals_model* m, const pals_grid* g,
                      const pals_coeffs* coeffs, pals_plan** out);

int pals_plan_create(pals_ctx* ctx, const pals_model* m, const pals_grid* g,
                     const pals_coeffs* coeffs, pals_plan** out) {
    if (!ctx || !m || !g || !coeffs) return set_error(PALS_ECONFIG, "pals_plan_create: null");
    return plan_build(ctx, m, g, coeffs, out);
}

}  // extern "C"

namespace pals {
int plan_create_values(pals_ctx* ctx, const pals_grid* g, pals_plan** out) {
    const pals_coeffs unit{1.0, 0.0};
    const int rc = plan_build(ctx, nullptr, g, &unit, out);
    if (rc == PALS_OK) (*out)->values = 1;
    return rc;
}
pals_ctx* plan_ctx(const pals_plan* p) { return p->ctx; }
// per-plan device scratch that persists across calls (host-output entry points):
// no cudaMalloc / cudaFree (which synchronizes the device) per call
void* plan_scratch(pals_plan* p, size_t bytes) {
    if (bytes > p->scratch_bytes) {
        cudaFree(p->scratch);
        p->scratch = nullptr;
        p->scratch_bytes = 0;
        if (cudaMalloc(&p->scratch, bytes) != cudaSuccess) return nullptr;
        p->scratch_bytes = bytes;
    }
    return p->scratch;
}
}  // namespace pals

static int plan_build(pals_ctx* ctx, const pals_model* m, const pals_grid* g,
                      const pals_coeffs* coeffs, pals_plan** out) {
    PALS_CUDA(cudaSetDevice(ctx->device));
    // k_scan's shared memory exceeds the 48 KB default (per device, idempotent)
    PALS_CUDA(cudaFuncSetAttribute(k_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kScanSmem));
    auto* p = new pals_plan();
    p->ctx = ctx;
    p->model = m;
    p->grid = g;
    p->coeffs = *coeffs;
    p->n = g->n;
    // the reference scores every candidate before ranking; the first candidate
    // the scorer rejects aborts the call with that exception (controller.hpp:146-151)
    if (g->n == 0) {
        p->err = PALS_ECONFIG;
        p->err_msg = "select_config: empty candidate list";
    } else if (m && validate_points(m, g->h_pts, g->n) != PALS_OK) {
        p->err = validate_points(m, g->h_pts, g->n);
        p->err_msg = pals_last_error();
    }
    const int64_t n = std::max<int64_t>(1, g->n);
    // the chunk sort's chunk: 2,048 points (4 keys x 512 threads: 15 us on B200 against
    // 27 us for a bitonic chunk sort, 18 us for 8 keys x 256, and slower 4,096 / 8,192-key
    // chunks); small grids (cfg1's 36 candidates, a replay's candidate sets) sort in one
    // chunk just large enough. The pair scan's chunk-local ranks need chunks <= 2,048.
    p->chunk = n <= 256 ? 256 : n <= 512 ? 512 : n <= 1024 ? 1024 : kChunk;
    // PDL edges between the step's kernels
    p->pdl = 1;
    p->nchunks = (int)((n + p->chunk - 1) / p->chunk);
    p->np = (int64_t)p->nchunks * p->chunk;
    PlanDev& d = p->d;
    d.n = g->n;
    d.wide = g->n > 65536 ? 1 : 0;
    d.tr_bits = d.wide ? 32 : 16;
    d.cap = g->cap;
    d.batch = g->batch;
    d.dp = g->dp;
    d.inv_tr = g->inv_tr;
    d.samp_s = (n + kSamples - 1) / kSamples;
    d.samp_n = (int)((n + d.samp_s - 1) / d.samp_s);
    // one slab for all per-plan device arrays
    const size_t n8 = (size_t)n * 8, np8 = (size_t)p->np * 8, np4 = (size_t)p->np * 4;
    size_t bytes = 5 * n8 + N_ORD * (3 * np8 + 2 * np4 + kSamples * 8 + n8 + (size_t)n * 12) + 64 +
                   4 * (size_t)n +
                   (d.wide ? N_ORD * n8 : N_ORD * (size_t)n * 4) + 4096;
    if (m && m->kind == MODEL_TABLE) bytes += 4 * (size_t)n + 2 * 8 * (size_t)std::max<int64_t>(1, m->table_n);
    bytes += sizeof(Analytic) + 256;
    bytes += N_ORD * (4 * (size_t)p->np + np4);  // chunk-local rank arrays
    bytes += 80 * 256;  // every take() rounds up to 256 B
    PALS_CUDA(cudaMalloc(&p->slab, bytes));
    char* s = (char*)p->slab;
    auto take = [&](size_t b) {
        char* r = s;
        s += (b + 255) & ~(size_t)255;
        return (void*)r;
    };
    d.T = (double*)take(n8);
    d.P = (double*)take(n8);
    d.th = (double*)take(n8);
    d.pn = (double*)take(n8);
    d.ef = (double*)take(n8);
    for (int o = 0; o < N_ORD; ++o) {
        d.skey[o] = (uint64_t*)take(np8);
        d.sorted[o] = (uint64_t*)take(np8);
        d.merged[o] = (uint64_t*)take(np8);
        d.sidx[o] = (uint32_t*)take(np4);
        d.midx[o] = (uint32_t*)take(np4);
        d.samp[o] = (uint64_t*)take(kSamples * 8);
        d.bnd[o] = (uint8_t*)take((size_t)n);
        d.danger[o] = (uint8_t*)take((size_t)n);
        if (d.wide) d.key64[o] = (uint64_t*)take(n8);
        else d.key32[o] = (uint32_t*)take((size_t)n * 4);
        d.rank32[o] = (uint32_t*)take((size_t)n * 4);
        d.pos32[o] = (uint32_t*)take((size_t)n * 4);
    }
    d.lch = p->chunk;
    for (int o = 0; o < N_ORD; ++o) {
        d.lr16[o] = (uint16_t*)take((size_t)p->np * 2);
        d.lq16[o] = (uint16_t*)take((size_t)p->np * 2);
        d.cinv[o] = (uint32_t*)take(np4);
    }
    d.globals = (int32_t*)take(16);
    // globals[2] (the generic-score flag) only ever gets set, and a plan's scores are
    // the same every prepare, so it is zeroed once here instead of every step
    PALS_CUDA(cudaMemsetAsync(d.globals, 0, 16, ctx->stream));
    p->gk = (uint64_t*)take(32);  // [2] global candidate keys + k_assign's done counter
    PALS_CUDA(cudaMemsetAsync(p->gk, 0xFF, 16, ctx->stream));
    PALS_CUDA(cudaMemsetAsync(p->gk + 2, 0, 8, ctx->stream));
    p->d_an = (Analytic*)take(sizeof(Analytic));
    // TR per point (inverse of grid inv_tr), computed once on the host at grid creation
    p->tr = (int*)take(4 * (size_t)n);
    d.tr = p->tr;
    {
        std::vector<int> inv(g->n), tr(g->n);
        if (g->n) {
            PALS_CUDA(copy_on(ctx->stream, inv.data(), g->inv_tr, g->n * sizeof(int), cudaMemcpyDeviceToHost));
            for (int64_t r = 0; r < g->n; ++r) tr[inv[r]] = (int)r;
            PALS_CUDA(copy_on(ctx->stream, p->tr, tr.data(), g->n * sizeof(int), cudaMemcpyHostToDevice));
        }
    }
    if (m && m->kind == MODEL_ANALYTIC)
        PALS_CUDA(copy_on(ctx->stream, p->d_an, &m->an, sizeof(Analytic), cudaMemcpyHostToDevice));
    if (m && m->kind == MODEL_TABLE) {
        p->table_map = (int*)take(4 * (size_t)n);
        const int64_t tn = std::max<int64_t>(1, m->table_n);
        p->table_T = (double*)take(8 * (size_t)tn);
        p->table_P = (double*)take(8 * (size_t)tn);
        // first table row equal by value (TableScorer, tests/test_controller.cpp:23-26)
        std::unordered_map<std::string, int> first;
        for (int64_t i = 0; i < m->table_n; ++i) {
            pals_point q = m->table_pts[i];
            if (q.cap_watts == 0.0) q.cap_watts = 0.0;
            first.emplace(std::string((const char*)&q, sizeof q), (int)i);
        }
        std::vector<int> map(g->n, 0);
        for (int64_t i = 0; i < g->n; ++i) {
            pals_point q = g->h_pts[i];
            if (q.cap_watts == 0.0) q.cap_watts = 0.0;
            auto it = first.find(std::string((const char*)&q, sizeof q));
            map[i] = it == first.end() ? 0 : it->second;
        }
        if (g->n)
            PALS_CUDA(copy_on(ctx->stream, p->table_map, map.data(), g->n * 4, cudaMemcpyHostToDevice));
        if (m->table_n) {
            PALS_CUDA(copy_on(ctx->stream, p->table_T, m->table_T, m->table_n * 8, cudaMemcpyHostToDevice));
            PALS_CUDA(copy_on(ctx->stream, p->table_P, m->table_P, m->table_n * 8, cudaMemcpyHostToDevice));
        }
    }
    *out = p;
    return PALS_OK;
}

extern "C" {

int pals_plan_destroy(pals_plan* p) {
    if (!p) return PALS_OK;
    cudaSetDevice(p->ctx->device);
    if (p->gexec) cudaGraphExecDestroy(p->gexec);
    if (p->ev_scan0) cudaEventDestroy(p->ev_scan0);
    if (p->ev_scan1) cudaEventDestroy(p->ev_scan1);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    for (auto& e : p->ev_up)
        if (e) cudaEventDestroy(e);
    if (p->side) cudaStreamDestroy(p->side);
    if (p->h_cnt) cudaFreeHost(p->h_cnt);
    cudaFree(p->scratch);
    cudaFree(p->slab);
    cudaFree(p->dec_buf);
    cudaFree(p->thr_t);
    cudaFree(p->d_q);
    delete p;
    return PALS_OK;
}


// prepare, part 1: evaluate, sort, cross-rank, scatter (merged arrays ready)
static int prep_head(pals_plan* p, int32_t* counts_reset = nullptr) {
    pals_ctx* ctx = p->ctx;
    cudaStream_t s = ctx->stream;
    PlanDev& d = p->d;
    const int64_t n = p->n;
    const bool pdl = p->pdl;
    (void)cudaGetLastError();  // clear stale non-sticky errors of earlier calls
    const int eb = grid_blocks(ctx, n, 256);
    cudaError_t e = cudaSuccess;
    if (p->values) {
        e = launch_k(k_eval_values, eb, 256, 0, s, false, d);
    } else if (p->model->kind == MODEL_ANALYTIC) {
        e = launch_k(k_eval_analytic, eb, 256, 0, s, false, d, (const Analytic*)p->d_an,
                     (const int*)p->grid->tp, p->coeffs.alpha, p->coeffs.beta_watts);
    } else if (p->model->kind == MODEL_TABLE) {
        e = launch_k(k_eval_table, eb, 256, 0, s, false, d, (const int*)p->table_map,
                     (const double*)p->table_T, (const double*)p->table_P, p->coeffs.alpha,
                     p->coeffs.beta_watts);
    } else {
        const int rc = forest_eval_plan(p, p->model, ctx);
        if (rc) return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "pals_plan_prepare eval");
    uint32_t* done = (uint32_t*)(p->gk + 2);
    const dim3 gs(p->nchunks, N_ORD);
    // chunk sort, then log2(chunks) pairwise merge rounds; the last writer of merged
    // also writes the search index
    int rounds = 0;
    while (((int64_t)p->chunk << rounds) < p->np) ++rounds;
    const int sort_to_merged = rounds % 2 == 0;
    const int sort_final = rounds == 0;
    if (p->chunk == 2048)  // 4 keys x 512 threads (8 x 256 and 2 x 1,024 measured slower)
        e = launch_k(k_sort_chunks<512, 4>, gs, 512, sort_smem_bytes(512, 4), s, pdl, d, p->gk,
                     done, counts_reset, sort_to_merged, sort_final);
    else switch (p->chunk) {
#define PALS_SORT(TPB)                                                                         \
    case TPB * kIPT:                                                                           \
        e = launch_k(k_sort_chunks<TPB>, gs, TPB, sort_smem_bytes(TPB), s, pdl, d, p->gk, done, \
                     counts_reset, sort_to_merged, sort_final);                                \
        break;
        PALS_SORT(32)
        PALS_SORT(64)
        PALS_SORT(128)
        PALS_SORT(256)
        PALS_SORT(512)
        PALS_SORT(1024)
#undef PALS_SORT
        default:
            e = cudaErrorInvalidValue;
    }

    // round k reads the buffer round k-1 wrote; the last round writes merged
    int lg = 0;
    while ((1 << lg) < p->chunk) ++lg;
    for (int k = 0; k < rounds && e == cudaSuccess; ++k) {
        const int to_m = (rounds - k) % 2 == 1, fin = k == rounds - 1;
        // 2 keys x 512 threads per 1,024-key merge tile (7.0 us per round against 8.5 us for
        // 8 x 128 and 7.4 us for 4 x 256)
        e = launch_k(k_merge_round<512, 2>, dim3((unsigned)((p->np + 1023) / 1024), N_ORD), 512,
                     0, s, pdl, d, (uint32_t)p->np, lg + k, to_m, fin);
    }
    if (e != cudaSuccess) return cuda_fail(e, "pals_plan_prepare");
    count_launch(ctx, 2 + rounds);  // eval, sort, merge rounds
    return check_launch("pals_plan_prepare");
}

// prepare, part 2: packed keys, near-tie flags, the two global winners
static int prep_tail(pals_plan* p) {
    pals_ctx* ctx = p->ctx;
    const int eb = grid_blocks(ctx, p->n, 256);
    const cudaError_t e = launch_k(k_assign, dim3(eb, N_ORD), 256, 0, ctx->stream, (bool)p->pdl,
                                   p->d, p->gk, (uint32_t*)(p->gk + 2));
    if (e != cudaSuccess) return cuda_fail(e, "pals_plan_prepare assign");
    count_launch(ctx, 1);
    return check_launch("pals_plan_prepare");
}

int pals_plan_prepare(pals_plan* p) {
    if (p->err) return set_error(p->err, p->err_msg);
    PALS_CUDA(cudaSetDevice(p->ctx->device));
    int rc = prep_head(p);
    return rc ? rc : prep_tail(p);
}

static int ensure_query_buffers(pals_plan* p, int64_t nq) {
    if (nq <= p->qcap) return PALS_OK;
    if (p->gexec) {  // the cached step graph points at the buffers being replaced
        cudaGraphExecDestroy(p->gexec);
        p->gexec = nullptr;
    }
    cudaFree(p->thr_t);
    const int64_t cap = std::max<int64_t>(nq, 1024);
    // per query: thresholds, minima, class; per class slot: list entry + 16-byte record
    const size_t bytes = (size_t)cap * (8 * 4 + 1 + 20 * N_CLS) + 4096;
    PALS_CUDA(cudaMalloc(&p->thr_t, bytes));
    char* s = (char*)p->thr_t;
    auto take = [&](size_t b) {
        char* r = s;
        s += (b + 255) & ~(size_t)255;
        return (void*)r;
    };
    p->thr_t = (uint64_t*)take(8 * cap);
    p->thr_p = (uint64_t*)take(8 * cap);
    p->best_e = (uint64_t*)take(8 * cap);
    p->best_t = (uint64_t*)take(8 * cap);
    p->cls = (uint8_t*)take(cap);
    p->qlist = (int32_t*)take(4 * (size_t)cap * N_CLS);
    p->qthr = (uint4*)take(16 * (size_t)cap * N_CLS);
    p->counts = (int32_t*)take(4 * kCountInts);
    p->qcap = cap;
    return PALS_OK;
}

// k_scan's grid: 4 CTAs of 256 threads per SM (the partition, scan_plan_warp, adapts the
// query tiles and config parts to it)
#ifndef PALS_SCAN_CPS
#define PALS_SCAN_CPS 4
#endif
static int scan_grid(const pals_plan* p, int64_t) { return p->ctx->num_sms * PALS_SCAN_CPS; }

static SelArgs make_args(pals_plan* p, const pals_query* d_queries, int64_t nq, int32_t* d_idx,
                         uint8_t* d_reason) {
    SelArgs a;
    a.q = d_queries;
    a.nq = nq;
    a.out_idx = d_idx;
    a.out_reason = d_reason;
    a.thr_t = p->thr_t;
    a.thr_p = p->thr_p;
    a.best_e = p->best_e;
    a.best_t = p->best_t;
    a.cls = p->cls;
    a.qlist = p->qlist;
    a.qthr = p->qthr;
    a.counts = p->counts;
    a.qcap = p->qcap;
    a.force_exact = p->force_exact;
    a.scan_grid = scan_grid(p, nq);
    return a;
}

// the arguments of query chunk k = [off, off + len): every per-query array shifted,
// its own class counters; the class lists keep their stride qcap, so chunks use
// disjoint slices of them
static SelArgs make_args_chunk(pals_plan* p, const pals_query* d_queries, int64_t off, int64_t len,
                               int32_t* d_idx, uint8_t* d_reason, int k) {
    SelArgs a = make_args(p, d_queries + off, len, d_idx + off, d_reason + off);
    a.thr_t += off;
    a.thr_p += off;
    a.best_e += off;
    a.best_t += off;
    a.cls += off;
    a.qlist += off;
    a.qthr += off;
    a.counts += kCountStride * k;
    return a;
}

// select, part 1 (needs only the merged arrays): thresholds and classes per query
static int select_head(pals_plan* p, const SelArgs& a, cudaStream_t s) {
    PALS_CUDA(cudaMemsetAsync(p->counts, 0, 4 * kCountInts, s));
    const cudaError_t e = launch_k(k_qprep, grid_blocks(p->ctx, a.nq, 256), 256, 0, s, false,
                                   p->d, a);
    if (e != cudaSuccess) return cuda_fail(e, "pals_plan_select_device qprep");
    count_launch(p->ctx, 1);
    return check_launch("pals_plan_select_device");
}

// the prefix-min tables of the time-to-decide path (they depend on the ranks only)
static int dec_layout(pals_plan* p, DecDev* t) {
    const int64_t n = p->n;
    t->n = n;
    int B = 1024;
    while ((n + B - 1) / B > kDecMaxBlocks) B *= 2;
    t->B = B;
    t->nb = (int)((n + B - 1) / B);
    t->ntiles = (int)((n + kDecTile - 1) / kDecTile);
    const int rows = 2 + t->nb;
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t need = al(nn * 4) * 2 + al(nn * 8) * 2 + al((size_t)rows * t->ntiles * 4) +
                        al((size_t)rows * nn * 4);
    if (p->dec_bytes < need) {
        cudaFree(p->dec_buf);
        p->dec_buf = nullptr;
        p->dec_bytes = 0;
        PALS_CUDA(cudaMalloc(&p->dec_buf, need));
        p->dec_bytes = need;
    }
    char* b = (char*)p->dec_buf;
    t->elemA = (uint32_t*)b;
    b += al(nn * 4);
    t->elemC = (uint32_t*)b;
    b += al(nn * 4);
    t->te = (uint2*)b;
    b += al(nn * 8);
    t->pt = (uint2*)b;
    b += al(nn * 8);
    t->agg = (uint32_t*)b;
    b += al((size_t)rows * t->ntiles * 4);
    t->tab = (uint32_t*)b;
    return PALS_OK;
}

// select, part 2 (needs the packed keys): the pair scan (or the prefix-min decision),
// decisions, exact folds. build: this call also builds the prefix-min tables (decide mode;
// the first query chunk of a step)
static int select_tail(pals_plan* p, const SelArgs& a, bool build = true) {
    pals_ctx* ctx = p->ctx;
    cudaStream_t s = ctx->stream;
    const int sgrid = a.scan_grid;
    // event-record nodes around the scan (timing) are not kernels: plain edges there
    const bool pdl = p->pdl && !p->time_scan;
    // inside a stream capture the events become graph event-record nodes
    const unsigned evf = p->capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
    cudaError_t e;
    if (p->time_scan) PALS_CUDA(cudaEventRecordWithFlags(p->ev_scan0, s, evf));
    if (p->decide == PALS_DECIDE_PREFIX) {
        DecDev t;
        int rc = dec_layout(p, &t);
        if (rc) return rc;
        if (build) {
            e = launch_k(k_dec_elems, grid_blocks(ctx, p->n, 256), 256, 0, s, pdl, p->d, t);
            if (e == cudaSuccess)
                e = launch_k(k_dec_tiles, dim3(t.ntiles, 2 + t.nb), 256, 0, s, pdl, t);
            if (e == cudaSuccess)
                e = launch_k(k_dec_scan, dim3(t.ntiles, 2 + t.nb), 256, 0, s, pdl, t);
            if (e != cudaSuccess) return cuda_fail(e, "decide tables");
            count_launch(ctx, 3);
        }
        e = launch_k(k_decide, ctx->num_sms * 8, 256, 0, s, pdl, t, a);
        if (e != cudaSuccess) return cuda_fail(e, "k_decide");
    } else {
        e = launch_k(k_scan, sgrid, kScanThreads, kScanSmem, s, pdl, p->d, a);
    }
    if (e != cudaSuccess) return cuda_fail(e, "k_scan");
    if (p->time_scan) {
        PALS_CUDA(cudaEventRecordWithFlags(p->ev_scan1, s, evf));
        p->scan_recorded = 1;
    }
    const int qb = grid_blocks(ctx, a.nq, 256);
    // enough warps for plans where many queries take the exact fold (generic scores)
    e = launch_k(k_finalize, std::max(qb, ctx->num_sms * 2), 256, 0, s, pdl, p->d, a);
    if (e != cudaSuccess) return cuda_fail(e, "pals_plan_select_device tail");
    count_launch(ctx, 2);
    return check_launch("pals_plan_select_device");
}

int pals_plan_select_device(pals_plan* p, const pals_query* d_queries, int64_t nq,
                            int32_t* d_idx, uint8_t* d_reason) {
    if (p->err) return set_error(p->err, p->err_msg);
    if (nq <= 0) return PALS_OK;
    if (nq > ((int64_t)1 << 31) - 1) return set_error(PALS_ECONFIG, "pals_select: too many queries");
    PALS_CUDA(cudaSetDevice(p->ctx->device));
    int rc = ensure_query_buffers(p, nq);
    if (rc) return rc;
    const SelArgs a = make_args(p, d_queries, nq, d_idx, d_reason);
    rc = select_head(p, a, p->ctx->stream);
    return rc ? rc : select_tail(p, a);
}

// One full step — evaluate + rank (prepare) and select — replayed from a CUDA graph
// captured on first use for these device buffers (8 kernels, no memset nodes: the
// class counters are reset by k_sort_chunks, assign and qprep share one launch).
// One step as a graph. With pinned host buffers (h_q, h_idx, h_rs: pals_select) the
// graph also holds the copies: the queries go up on a side stream while the model
// is evaluated and ranked (the prepare never reads them), and only qprep waits for
// them; the decisions and class counters come back at the end.
static int plan_step(pals_plan* p, const pals_query* d_queries, int64_t nq, int32_t* d_idx,
                     uint8_t* d_reason, const pals_query* h_q, int32_t* h_idx, uint8_t* h_rs) {
    pals_ctx* ctx = p->ctx;
    cudaStream_t s = ctx->stream;
    const int key_t = p->time_scan | (p->force_exact << 1) | (p->decide << 2);
    const bool hit = p->gexec && p->g_q == d_queries && p->g_n == nq && p->g_idx == d_idx &&
                     p->g_rs == d_reason && p->g_timed == key_t && p->g_hq == h_q &&
                     p->g_hidx == h_idx && p->g_hrs == h_rs;
    if (h_q && !p->side) {
        PALS_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
        PALS_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
        PALS_CUDA(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
        for (auto& e : p->ev_up) PALS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        PALS_CUDA(cudaMallocHost(&p->h_cnt, 4 * kCountInts));
    }
    if (!hit) {
        if (p->gexec) {
            cudaGraphExecDestroy(p->gexec);
            p->gexec = nullptr;
        }
        int rc = ensure_query_buffers(p, nq);
        if (rc) return rc;
        (void)cudaGetLastError();
        PALS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        p->capturing = 1;
        const int64_t l0 = ctx->launches;
        // (overlapping qprep with k_assign on a side stream measured no faster on
        // B200: the step stays a single chain)
        // pals_select with many queries: the upload is split into chunks on the side
        // stream and each chunk's qprep / scan / finalize waits only for its own chunk,
        // so all but the first chunk's copy hide behind the previous chunk's scan
        const int nch = !h_q ? 1
                             : (int)std::max<int64_t>(1, std::min<int64_t>(kMaxChunks, nq / 131072));
        const int64_t clen = (nq + nch - 1) / nch;
        cudaError_t ce0 = cudaSuccess;
        if (h_q) {
            ce0 = cudaEventRecord(p->ev_fork, s);
            if (ce0 == cudaSuccess) ce0 = cudaStreamWaitEvent(p->side, p->ev_fork, 0);
            for (int k = 0; k < nch && ce0 == cudaSuccess; ++k) {
                const int64_t off = k * clen, len = std::min(clen, nq - off);
                ce0 = cudaMemcpyAsync((void*)(d_queries + off), h_q + off,
                                      (size_t)len * sizeof(pals_query), cudaMemcpyHostToDevice,
                                      p->side);
                if (ce0 == cudaSuccess) ce0 = cudaEventRecord(p->ev_up[k], p->side);
            }
            if (ce0 == cudaSuccess) ce0 = cudaEventRecord(p->ev_join, p->side);
        }
        rc = ce0 != cudaSuccess ? cuda_fail(ce0, "pals_select upload") : prep_head(p, p->counts);
        for (int k = 0; k < nch && !rc; ++k) {
            const int64_t off = k * clen, len = std::min(clen, nq - off);
            if (h_q) {
                const cudaError_t we =
                    cudaStreamWaitEvent(s, k == nch - 1 ? p->ev_join : p->ev_up[k], 0);
                if (we != cudaSuccess) rc = cuda_fail(we, "pals_select upload join");
            }
            const SelArgs a = make_args_chunk(p, d_queries, off, len, d_idx, d_reason, k);
            const int qb = grid_blocks(ctx, len, 256);
            cudaError_t e;
            if (!rc && k == 0) {
                // assign (prepare, part 2) and qprep (select, part 1) fused in one launch
                const int eb = grid_blocks(ctx, p->n, 256);
                e = launch_k(k_assign_qprep, dim3((unsigned)(qb + N_ORD * eb)), 256, 0, s,
                             (bool)p->pdl, p->d, p->gk, (uint32_t*)(p->gk + 2), a, eb, qb);
                if (e != cudaSuccess) rc = cuda_fail(e, "k_assign_qprep");
            } else if (!rc) {
                e = launch_k(k_qprep, qb, 256, 0, s, false, p->d, a);
                if (e != cudaSuccess) rc = cuda_fail(e, "k_qprep");
            }
            if (!rc) {
                count_launch(ctx, 1);
                rc = select_tail(p, a, k == 0);
            }
        }
        if (!rc && h_idx) {
            cudaError_t de =
                cudaMemcpyAsync(h_idx, d_idx, (size_t)nq * 4, cudaMemcpyDeviceToHost, s);
            if (de == cudaSuccess)
                de = cudaMemcpyAsync(h_rs, d_reason, (size_t)nq, cudaMemcpyDeviceToHost, s);
            if (de == cudaSuccess)
                de = cudaMemcpyAsync(p->h_cnt, p->counts, 4 * kCountInts, cudaMemcpyDeviceToHost,
                                     s);
            if (de != cudaSuccess) rc = cuda_fail(de, "pals_select download");
        }
        p->g_chunks = nch;
        p->capturing = 0;
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(s, &g);
        if (rc) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (ce != cudaSuccess) return cuda_fail(ce, "pals_plan_run capture");
        const cudaError_t ie = cudaGraphInstantiate(&p->gexec, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) return cuda_fail(ie, "pals_plan_run instantiate");
        p->g_launches = ctx->launches - l0;
        ctx->launches = l0;  // captured, not launched
        p->g_q = d_queries;
        p->g_n = nq;
        p->g_idx = d_idx;
        p->g_rs = d_reason;
        p->g_timed = key_t;
        p->g_hq = h_q;
        p->g_hidx = h_idx;
        p->g_hrs = h_rs;
    }
    PALS_CUDA(cudaGraphLaunch(p->gexec, s));
    count_launch(ctx, (int)p->g_launches);
    if (p->time_scan) p->scan_recorded = 1;
    return PALS_OK;
}

int pals_plan_run(pals_plan* p, const pals_query* d_queries, int64_t nq, int32_t* d_idx,
                  uint8_t* d_reason) {
    if (p->err) return set_error(p->err, p->err_msg);
    if (nq <= 0) return pals_plan_prepare(p);
    PALS_CUDA(cudaSetDevice(p->ctx->device));
    return plan_step(p, d_queries, nq, d_idx, d_reason, nullptr, nullptr, nullptr);
}

// page-locked host memory; *dev = its device-side address (mapped under unified
// addressing) or null
static bool is_pinned(const void* h, void** dev = nullptr) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    if (dev) *dev = at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
    return at.type == cudaMemoryTypeHost;
}

int pals_select(pals_plan* p, const pals_query* queries, int64_t nq, int32_t* idx,
                uint8_t* reason) {
    if (p->err) return set_error(p->err, p->err_msg);
    if (nq < 0) return set_error(PALS_ECONFIG, "pals_select: negative query count");
    pals_ctx* ctx = p->ctx;
    PALS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    int rc;
    if (nq == 0) {
        rc = pals_plan_prepare(p);
        return rc ? rc : pals_ctx_sync(ctx);
    }
    // host staging of queries/results lives in the context scratch
    const size_t need = (size_t)nq * (sizeof(pals_query) + 4 + 1) + 1024;
    if (ctx->scratch_bytes < need) {
        cudaFree(ctx->d_scratch);
        PALS_CUDA(cudaMalloc(&ctx->d_scratch, need));
        ctx->scratch_bytes = need;
    }
    char* b = (char*)ctx->d_scratch;
    pals_query* dq = (pals_query*)b;
    int32_t* di = (int32_t*)(b + (size_t)nq * sizeof(pals_query));
    uint8_t* dr = (uint8_t*)(di + nq);
    void *m_idx = nullptr, *m_rs = nullptr;
    if (is_pinned(queries) && is_pinned(idx, &m_idx) && is_pinned(reason, &m_rs)) {
        // one graph: upload overlapped with the prepare; with mapped result buffers the
        // decisions are stored straight into host memory by k_finalize (no download
        // nodes), else downloaded at the end
        const bool mapped = m_idx && m_rs;
        rc = mapped ? plan_step(p, dq, nq, (int32_t*)m_idx, (uint8_t*)m_rs, queries, nullptr,
                                nullptr)
                    : plan_step(p, dq, nq, di, dr, queries, idx, reason);
        if (rc) return rc;
        PALS_CUDA(cudaStreamSynchronize(s));
        int64_t ex = 0;
        for (int k = 0; k < p->g_chunks; ++k) ex += p->h_cnt[kCountStride * k + N_CLS];
        p->last_exact = mapped ? -1 : ex;  // -1: read on demand
        return PALS_OK;
    }
    PALS_CUDA(cudaMemcpyAsync(dq, queries, (size_t)nq * sizeof(pals_query), cudaMemcpyHostToDevice, s));
    rc = pals_plan_run(p, dq, nq, di, dr);
    if (rc) return rc;
    PALS_CUDA(cudaMemcpyAsync(idx, di, (size_t)nq * 4, cudaMemcpyDeviceToHost, s));
    PALS_CUDA(cudaMemcpyAsync(reason, dr, (size_t)nq, cudaMemcpyDeviceToHost, s));
    int32_t cnt[N_CLS + 1];
    PALS_CUDA(cudaMemcpyAsync(cnt, p->counts, sizeof cnt, cudaMemcpyDeviceToHost, s));
    PALS_CUDA(cudaStreamSynchronize(s));
    p->last_exact = cnt[N_CLS];
    return PALS_OK;
}

int pals_plan_scores(pals_plan* p, double* t_hat, double* p_node, double* eff) {
    if (p->err) return set_error(p->err, p->err_msg);
    PALS_CUDA(cudaSetDevice(p->ctx->device));
    int rc = pals_plan_prepare(p);
    if (rc) return rc;
    cudaStream_t s = p->ctx->stream;
    if (t_hat) PALS_CUDA(cudaMemcpyAsync(t_hat, p->d.th, p->n * 8, cudaMemcpyDeviceToHost, s));
    if (p_node) PALS_CUDA(cudaMemcpyAsync(p_node, p->d.pn, p->n * 8, cudaMemcpyDeviceToHost, s));
    if (eff) PALS_CUDA(cudaMemcpyAsync(eff, p->d.ef, p->n * 8, cudaMemcpyDeviceToHost, s));
    PALS_CUDA(cudaStreamSynchronize(s));
    return PALS_OK;
}

int64_t pals_plan_last_exact_count(const pals_plan* p) {
    if (p->last_exact < 0 && p->counts) {  // not downloaded by the last select
        int32_t cnt[kCountInts];
        if (copy_on(p->ctx->stream, cnt, p->counts, sizeof cnt, cudaMemcpyDeviceToHost) ==
            cudaSuccess) {
            int64_t ex = 0;
            for (int k = 0; k < p->g_chunks; ++k) ex += cnt[kCountStride * k + N_CLS];
            const_cast<pals_plan*>(p)->last_exact = ex;
        }
    }
    return p->last_exact;
}

int pals_plan_stats(pals_plan* p, int64_t* c6) {
    for (int i = 0; i < 6; ++i) c6[i] = 0;
    if (!p->counts) return PALS_OK;
    PALS_CUDA(cudaSetDevice(p->ctx->device));
    // a pinned pals_select splits large batches into chunks, each with its own counters
    // (stride kCountStride); chunks a select did not use are zeroed by it
    int32_t cnt[kCountInts];
    PALS_CUDA(cudaMemcpyAsync(cnt, p->counts, sizeof cnt, cudaMemcpyDeviceToHost, p->ctx->stream));
    PALS_CUDA(cudaStreamSynchronize(p->ctx->stream));
    for (int k = 0; k < kMaxChunks; ++k)
        for (int i = 0; i < 6; ++i) c6[i] += cnt[kCountStride * k + i];
    p->last_exact = c6[N_CLS];
    return PALS_OK;
}

int pals_plan_time_scan(pals_plan* p, int enable) {
    if (enable && !p->ev_scan0) {
        PALS_CUDA(cudaEventCreate(&p->ev_scan0));
        PALS_CUDA(cudaEventCreate(&p->ev_scan1));
    }
    p->time_scan = enable;
    p->scan_recorded = 0;
    return PALS_OK;
}

double pals_plan_scan_ms(pals_plan* p) {
    if (!p->scan_recorded) return -1.0;
    if (cudaEventSynchronize(p->ev_scan1) != cudaSuccess) return -1.0;
    float ms = -1.0f;
    if (cudaEventElapsedTime(&ms, p->ev_scan0, p->ev_scan1) != cudaSuccess) return -1.0;
    return ms;
}

int pals_plan_set_decide(pals_plan* p, int32_t mode) {
    if (mode != PALS_DECIDE_SCAN && mode != PALS_DECIDE_PREFIX)
        return set_error(PALS_ECONFIG, "pals_plan_set_decide: unknown mode");
    p->decide = mode;
    return PALS_OK;
}

int pals_plan_set_force_exact(pals_plan* p, int force) {
    p->force_exact = force;
    return PALS_OK;
}

int pals_eval_device(pals_ctx* ctx, const pals_model* m, const pals_grid* g, double* d_T,
                     double* d_P) {
    PALS_CUDA(cudaSetDevice(ctx->device));
    if (m->kind == MODEL_TABLE)
        return set_error(PALS_ECONFIG, "pals_eval_device: table models are scored via plans");
    if (m->kind == MODEL_FOREST)
        return forest_eval_raw(m, ctx, g->n, g->cap, g->batch, g->tp, g->ep, g->dp, d_T, d_P, 0);
    // analytic: the scorer would throw on the first invalid point (model.hpp:56-59)
    const int rc = validate_points(m, g->h_pts, g->n);
    if (rc) return rc;
    if (!m->d_an) {
        auto* mm = const_cast<pals_model*>(m);
        PALS_CUDA(cudaMalloc(&mm->d_an, sizeof(Analytic)));
        PALS_CUDA(copy_on(ctx->stream, mm->d_an, &m->an, sizeof(Analytic), cudaMemcpyHostToDevice));
    }
    k_eval_analytic_raw<<<grid_blocks(ctx, g->n, 256), 256, 0, ctx->stream>>>(
        m->d_an, g->n, g->cap, g->batch, g->tp, g->dp, d_T, d_P);
    count_launch(ctx);
    return check_launch("k_eval_analytic_raw");
}

int pals_eval(pals_ctx* ctx, const pals_model* m, const pals_grid* g, double* T, double* P) {
    PALS_CUDA(cudaSetDevice(ctx->device));
    pals_coeffs k{1.0, 0.0};
    pals_plan* p = nullptr;
    int rc = pals_plan_create(ctx, m, g, &k, &p);
    if (rc) return rc;
    if (p->err) {
        rc = set_error(p->err, p->err_msg);
        pals_plan_destroy(p);
        return rc;
    }
    cudaStream_t s = ctx->stream;
    const int eb = grid_blocks(ctx, p->n, 256);
    if (m->kind == MODEL_ANALYTIC)
        k_eval_analytic<<<eb, 256, 0, s>>>(p->d, p->d_an, g->tp, 1.0, 0.0);
    else if (m->kind == MODEL_TABLE)
        k_eval_table<<<eb, 256, 0, s>>>(p->d, p->table_map, p->table_T, p->table_P, 1.0, 0.0);
    else if ((rc = forest_eval_plan(p, m, ctx)) != PALS_OK) {
        pals_plan_destroy(p);
        return rc;
    }
    count_launch(ctx, 1);
    rc = check_launch("pals_eval");
    if (!rc) {
        cudaMemcpyAsync(T, p->d.T, p->n * 8, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(P, p->d.P, p->n * 8, cudaMemcpyDeviceToHost, s);
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) rc = cuda_fail(e, "pals_eval sync");
    }
    pals_plan_destroy(p);
    return rc;
}

}  // extern "C"
