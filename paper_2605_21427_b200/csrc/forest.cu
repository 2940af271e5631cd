// forest.cu — K2: the tree-ensemble predictor behind predictor_scorer
// (controller.hpp:100-105 -> PredictorBundle::predict forest.hpp:227-235 ->
// Forest::predict :176-180 -> RegressionTree::predict :80-85).
//
// Two exact evaluation paths:
//  * direct: the literal walk `x[f] <= thr ? left : right` per tree, leaf values
//    summed sequentially in tree order, divided by the tree count;
//  * cell table: every split threshold of feature f (over all trees of both
//    forests) cuts that axis into cells; all points of one lattice cell take the
//    same path through every tree, so the forest output is constant per cell.
//    The table holds, per cell, the direct-walk result at a representative point,
//    hence bit-identical values; evaluation becomes 5 binary searches + 1 load.
//    One-hot model features are constant for a given model (x = 1 on its slot).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "pals_internal.cuh"

namespace pals {

constexpr int kNumeric = 5;                 // cap, batch, tp, ep, dp (forest.hpp:24)
constexpr int kLut = 1024;                  // integer-feature coordinate lookup range
constexpr int64_t kMaxCells = 1ll << 22;    // cell tables above this use the direct walk

struct ForestDev {
    // concatenated nodes of both forests; children are global node indices
    const int32_t* feature;
    const double* thr_or_value;  // threshold for splits, value for leaves
    const int32_t* left;
    const int32_t* right;
    const int32_t* roots;        // [n_trees_T + n_trees_P]
    int n_trees_T, n_trees_P;
    int n_features;              // 5 + n_models
    int model_index;
    // lattice
    const double* th;            // thresholds of the 5 numeric features, concatenated
    int th_off[kNumeric + 1];
    const double* rep;           // representative coordinate per cell index, concatenated
    int rep_off[kNumeric + 1];
    int64_t dims[kNumeric];
    int64_t n_cells;             // 0 = no table
    // integer features (batch, tp, ep, dp): cell coordinate of every value in
    // [0, kLut) precomputed (= the lower_bound the lattice uses), one byte each
    const uint8_t* lut;          // [4][kLut]
    double* tabT;
    double* tabP;
};

struct ForestHost {
    ForestDev d{};
    void* slab = nullptr;
    double alpha = 0.0, beta = 0.0;
    int direct = 0;  // 1: always the literal tree walk (testing / very large lattices)
};

// RegressionTree::predict (forest.hpp:80-85) on the encoded feature vector x
__device__ __forceinline__ double tree_walk(const ForestDev& f, int root, const double* x) {
    int i = root;
    int ft = f.feature[i];
    while (ft >= 0) {
        i = x[ft] <= f.thr_or_value[i] ? f.left[i] : f.right[i];
        ft = f.feature[i];
    }
    return f.thr_or_value[i];
}

// FeatureSchema::encode (forest.hpp:41-50), numeric part; one-hot slots are
// handled by feature index (x[5 + m] = 1 for the model's slot, else 0).
__device__ __forceinline__ double feat(const double* x5, int model_index, int ft) {
    if (ft < kNumeric) return x5[ft];
    return (ft - kNumeric) == model_index ? 1.0 : 0.0;
}

__device__ __forceinline__ double tree_walk5(const ForestDev& f, int root, const double* x5) {
    int i = root;
    int ft = f.feature[i];
    while (ft >= 0) {
        i = feat(x5, f.model_index, ft) <= f.thr_or_value[i] ? f.left[i] : f.right[i];
        ft = f.feature[i];
    }
    return f.thr_or_value[i];
}

// Forest::predict (forest.hpp:176-180): sequential sum in tree order, then / n
__device__ __forceinline__ void forest_direct(const ForestDev& f, const double* x5, double* T,
                                              double* P) {
    double s = 0.0;
    for (int t = 0; t < f.n_trees_T; ++t) s += tree_walk5(f, f.roots[t], x5);
    *T = s / (double)f.n_trees_T;
    s = 0.0;
    for (int t = 0; t < f.n_trees_P; ++t) s += tree_walk5(f, f.roots[f.n_trees_T + t], x5);
    *P = s / (double)f.n_trees_P;
}

// Cell table build: one warp per cell. Lanes walk trees in parallel; the leaf
// values are summed by lane 0 in tree order, exactly as Forest::predict does.
__global__ void __launch_bounds__(256) k_forest_cells(ForestDev f) {
    extern __shared__ double leaf[];  // [warps_per_block][max(n_trees)]
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nt = max(f.n_trees_T, f.n_trees_P);
    double* lv = leaf + (size_t)wib * nt;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t cell = blockIdx.x * (int64_t)(blockDim.x >> 5) + wib; cell < f.n_cells;
         cell += warps) {
        double x5[kNumeric];
        int64_t r = cell;
#pragma unroll
        for (int k = kNumeric - 1; k >= 0; --k) {
            const int64_t j = r % f.dims[k];
            r /= f.dims[k];
            x5[k] = f.rep[f.rep_off[k] + j];
        }
        for (int pass = 0; pass < 2; ++pass) {
            const int n = pass ? f.n_trees_P : f.n_trees_T;
            const int base = pass ? f.n_trees_T : 0;
            for (int t = lane; t < n; t += 32) lv[t] = tree_walk5(f, f.roots[base + t], x5);
            __syncwarp();
            if (lane == 0) {
                double s = 0.0;
                for (int t = 0; t < n; ++t) s += lv[t];
                (pass ? f.tabP : f.tabT)[cell] = s / (double)n;
            }
            __syncwarp();
        }
    }
}

__device__ __forceinline__ int lower_bound_d(const double* a, int n, double x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// cell coordinate along axis k = number of thresholds strictly below x, so two
// points share a coordinate iff every test `x <= thr` on that axis agrees
__device__ __forceinline__ int64_t cell_of(const ForestDev& f, const double* x5) {
    int64_t c = 0;
#pragma unroll
    for (int k = 0; k < kNumeric; ++k) {
        const int j = lower_bound_d(f.th + f.th_off[k], f.th_off[k + 1] - f.th_off[k], x5[k]);
        c = c * f.dims[k] + j;
    }
    return c;
}

__global__ void k_forest_eval(ForestDev f, int64_t n, const double* __restrict__ cap,
                              const int* __restrict__ batch, const int* __restrict__ tp,
                              const int* __restrict__ ep, const int* __restrict__ dp,
                              double* __restrict__ T, double* __restrict__ P, int use_cells) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x5[kNumeric] = {cap[i], (double)batch[i], (double)tp[i], (double)ep[i],
                                     (double)dp[i]};
        if (use_cells) {
            const int64_t c = cell_of(f, x5);
            T[i] = f.tabT[c];
            P[i] = f.tabP[c];
        } else {
            forest_direct(f, x5, &T[i], &P[i]);
        }
    }
}

// PredictorBundle::predict for arbitrary points given as pals_point records
__global__ void k_forest_eval_aos(ForestDev f, int64_t n, const pals_point* __restrict__ pts,
                                  double* __restrict__ T, double* __restrict__ P, int use_cells) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const pals_point p = pts[i];
        const double x5[kNumeric] = {p.cap_watts, (double)p.batch, (double)p.tp, (double)p.ep,
                                     (double)p.dp};
        if (use_cells && f.lut) {
            // cap: binary search; integer features: one byte lookup each (independent loads)
            const int iv[4] = {p.batch, p.tp, p.ep, p.dp};
            int64_t c = lower_bound_d(f.th + f.th_off[0], f.th_off[1] - f.th_off[0], p.cap_watts);
#pragma unroll
            for (int k = 1; k < kNumeric; ++k) {
                const int v = iv[k - 1];
                const int j = (v >= 0 && v < kLut)
                                  ? (int)f.lut[(k - 1) * kLut + v]
                                  : lower_bound_d(f.th + f.th_off[k], f.th_off[k + 1] - f.th_off[k],
                                                  (double)v);
                c = c * f.dims[k] + j;
            }
            T[i] = f.tabT[c];
            P[i] = f.tabP[c];
        } else if (use_cells) {
            const int64_t c = cell_of(f, x5);
            T[i] = f.tabT[c];
            P[i] = f.tabP[c];
        } else {
            forest_direct(f, x5, &T[i], &P[i]);
        }
    }
}

}  // namespace pals

using namespace pals;

namespace pals {

void forest_free(void* p) {
    auto* fh = (ForestHost*)p;
    if (!fh) return;
    cudaFree(fh->slab);
    delete fh;
}

const PlanDev& plan_dev(const pals_plan* p);
const pals_grid* plan_grid(const pals_plan* p);
int plan_finish_scores(pals_plan* p);

static int forest_eval_points(const pals_model* m, pals_ctx* ctx, int64_t n, const double* cap,
                              const int* batch, const int* tp, const int* ep, const int* dp,
                              double* T, double* P, int force_direct) {
    auto* fh = (ForestHost*)m->forest;
    const int use_cells = (!force_direct && !fh->direct && fh->d.n_cells > 0) ? 1 : 0;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, ctx->num_sms * 16));
    k_forest_eval<<<blocks, 256, 0, ctx->stream>>>(fh->d, n, cap, batch, tp, ep, dp, T, P,
                                                   use_cells);
    count_launch(ctx);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "k_forest_eval");
    return PALS_OK;
}

int forest_eval_plan(pals_plan* p, const pals_model* m, pals_ctx* ctx) {
    const pals_grid* g = plan_grid(p);
    const PlanDev& d = plan_dev(p);
    const int rc = forest_eval_points(m, ctx, g->n, g->cap, g->batch, g->tp, g->ep, g->dp, d.T,
                                      d.P, 0);
    if (rc) return rc;
    return plan_finish_scores(p);
}

int forest_eval_raw(const pals_model* m, pals_ctx* ctx, int64_t n, const double* cap,
                    const int* batch, const int* tp, const int* ep, const int* dp, double* T,
                    double* P, int force_direct) {
    return forest_eval_points(m, ctx, n, cap, batch, tp, ep, dp, T, P, force_direct);
}

}  // namespace pals

extern "C" int pals_model_forest(pals_ctx* ctx, int32_t n_models, int32_t model_index,
                                 const pals_coeffs* coeffs, int32_t t_n_trees,
                                 const int64_t* t_off, const int32_t* t_feat, const double* t_thr,
                                 const int32_t* t_left, const int32_t* t_right,
                                 const double* t_val, int32_t p_n_trees, const int64_t* p_off,
                                 const int32_t* p_feat, const double* p_thr,
                                 const int32_t* p_left, const int32_t* p_right,
                                 const double* p_val, pals_model** out) {
    if (n_models < 1 || model_index < 0 || model_index >= n_models)
        return set_error(PALS_ECONFIG, "unknown model id in feature encoding");
    if (t_n_trees < 1 || p_n_trees < 1)
        return set_error(PALS_EDATA, "pals_model_forest: empty forest");
    PALS_CUDA(cudaSetDevice(ctx->device));
    const int nf = kNumeric + n_models;
    const int64_t nT = t_off[t_n_trees], nP = p_off[p_n_trees];
    const int64_t nn = nT + nP;
    std::vector<int32_t> feat(nn), left(nn, -1), right(nn, -1), roots(t_n_trees + p_n_trees);
    std::vector<double> tv(nn);
    std::vector<std::vector<double>> ths(kNumeric);
    auto add = [&](int n_trees, const int64_t* off, const int32_t* f, const double* thr,
                   const int32_t* l, const int32_t* r, const double* v, int64_t base, int rbase) {
        for (int t = 0; t < n_trees; ++t) {
            const int64_t o = off[t], sz = off[t + 1] - off[t];
            if (sz <= 0) return set_error(PALS_EDATA, "pals_model_forest: empty tree");
            roots[rbase + t] = (int32_t)(base + o);
            for (int64_t i = 0; i < sz; ++i) {
                const int64_t gi = base + o + i;
                const int32_t ft = f[o + i];
                feat[gi] = ft;
                if (ft >= 0) {
                    if (ft >= nf) return set_error(PALS_EDATA, "pals_model_forest: bad feature");
                    if (l[o + i] < 0 || l[o + i] >= sz || r[o + i] < 0 || r[o + i] >= sz)
                        return set_error(PALS_EDATA, "pals_model_forest: bad child index");
                    tv[gi] = thr[o + i];
                    left[gi] = (int32_t)(base + o + l[o + i]);
                    right[gi] = (int32_t)(base + o + r[o + i]);
                    if (ft < kNumeric) ths[ft].push_back(thr[o + i]);
                } else {
                    tv[gi] = v[o + i];
                }
            }
        }
        return PALS_OK;
    };
    int rc = add(t_n_trees, t_off, t_feat, t_thr, t_left, t_right, t_val, 0, 0);
    if (!rc) rc = add(p_n_trees, p_off, p_feat, p_thr, p_left, p_right, p_val, nT, t_n_trees);
    if (rc) return rc;
    // lattice: sorted distinct thresholds per numeric axis, representatives per cell index
    std::vector<double> th_all, rep_all;
    auto* fh = new ForestHost();
    ForestDev& d = fh->d;
    int64_t cells = 1;
    for (int k = 0; k < kNumeric; ++k) {
        auto& v = ths[k];
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        d.th_off[k] = (int)th_all.size();
        d.rep_off[k] = (int)rep_all.size();
        th_all.insert(th_all.end(), v.begin(), v.end());
        for (size_t j = 0; j < v.size(); ++j) rep_all.push_back(v[j]);
        rep_all.push_back(v.empty() ? 0.0 : std::nextafter(v.back(), INFINITY));
        d.dims[k] = (int64_t)v.size() + 1;
        cells = cells > kMaxCells ? cells : cells * d.dims[k];
    }
    d.th_off[kNumeric] = (int)th_all.size();
    d.rep_off[kNumeric] = (int)rep_all.size();
    d.n_cells = cells <= kMaxCells ? cells : 0;
    d.n_trees_T = t_n_trees;
    d.n_trees_P = p_n_trees;
    d.n_features = nf;
    d.model_index = model_index;
    // integer-feature coordinate lookups: lower_bound(thresholds, (double)v) for v < kLut
    std::vector<uint8_t> lut((size_t)4 * kLut);
    bool lut_ok = true;
    for (int k = 1; k < kNumeric; ++k) {
        const auto& v = ths[k];
        if (v.size() > 254) lut_ok = false;
        for (int x = 0; x < kLut; ++x)
            lut[(size_t)(k - 1) * kLut + x] =
                (uint8_t)(std::lower_bound(v.begin(), v.end(), (double)x) - v.begin());
    }
    const size_t bytes = nn * (4 + 8 + 4 + 4) + roots.size() * 4 + (th_all.size() + 1) * 8 +
                         rep_all.size() * 8 + 2 * 8 * (size_t)std::max<int64_t>(1, d.n_cells) +
                         lut.size() + 16 * 256;
    PALS_CUDA(cudaMalloc(&fh->slab, bytes));
    char* s = (char*)fh->slab;
    auto put = [&](const void* src, size_t b) {
        void* dst = s;
        if (b) copy_on(ctx->stream, dst, src, b, cudaMemcpyHostToDevice);
        s += (b + 255) & ~(size_t)255;
        return dst;
    };
    d.feature = (const int32_t*)put(feat.data(), nn * 4);
    d.thr_or_value = (const double*)put(tv.data(), nn * 8);
    d.left = (const int32_t*)put(left.data(), nn * 4);
    d.right = (const int32_t*)put(right.data(), nn * 4);
    d.roots = (const int32_t*)put(roots.data(), roots.size() * 4);
    d.th = (const double*)put(th_all.data(), th_all.size() * 8);
    d.rep = (const double*)put(rep_all.data(), rep_all.size() * 8);
    d.lut = lut_ok ? (const uint8_t*)put(lut.data(), lut.size()) : nullptr;
    d.tabT = (double*)s;
    s += (8 * std::max<int64_t>(1, d.n_cells) + 255) & ~(size_t)255;
    d.tabP = (double*)s;
    const cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) {
        forest_free(fh);
        return cuda_fail(ce, "pals_model_forest upload");
    }
    if (d.n_cells > 0) {
        const int nt = std::max(t_n_trees, p_n_trees);
        const int warps = 8;
        const size_t sm = (size_t)warps * nt * 8;
        if (sm > 48 * 1024) {
            forest_free(fh);
            return set_error(PALS_EDATA, "pals_model_forest: too many trees per forest (> 768)");
        }
        const int blocks = (int)std::min<int64_t>((d.n_cells + warps - 1) / warps, ctx->num_sms * 8);
        k_forest_cells<<<blocks, warps * 32, sm, ctx->stream>>>(d);
        count_launch(ctx);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            forest_free(fh);
            return cuda_fail(e, "k_forest_cells");
        }
        PALS_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    auto* m = new pals_model();
    m->ctx = ctx;
    m->uid = next_model_uid();
    m->kind = MODEL_FOREST;
    m->name = "predictor";
    m->forest = fh;
    fh->alpha = coeffs ? coeffs->alpha : 1.05;
    fh->beta = coeffs ? coeffs->beta_watts : 345.0;
    *out = m;
    return PALS_OK;
}

extern "C" int64_t pals_model_forest_cells(const pals_model* m) {
    if (!m || m->kind != MODEL_FOREST) return -1;
    return ((ForestHost*)m->forest)->d.n_cells;
}

extern "C" int pals_predict_device(pals_ctx* ctx, const pals_model* m, const pals_point* d_points,
                                   int64_t n, double* d_T, double* d_P) {
    if (!m || m->kind != MODEL_FOREST)
        return set_error(PALS_ECONFIG, "pals_predict_device: forest models only (use pals_eval)");
    if (n <= 0) return PALS_OK;
    auto* fh = (ForestHost*)m->forest;
    const int use_cells = (!fh->direct && fh->d.n_cells > 0) ? 1 : 0;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, ctx->num_sms * 16));
    k_forest_eval_aos<<<blocks, 256, 0, ctx->stream>>>(fh->d, n, d_points, d_T, d_P, use_cells);
    count_launch(ctx);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "k_forest_eval_aos");
    return PALS_OK;
}

extern "C" int pals_model_forest_set_direct(pals_model* m, int direct) {
    if (!m || m->kind != MODEL_FOREST) return set_error(PALS_ECONFIG, "not a forest model");
    ((ForestHost*)m->forest)->direct = direct ? 1 : 0;
    return PALS_OK;
}
