// fp64 device kernels behind the reference's module-level Python API (attention.*, rope.*,
// clustering.* of pkg/src/multipole_attn) -- the drop-in surface for callers that pass numpy arrays
// and Cluster / BlockLedger objects instead of a device-resident engine.  All arithmetic is fp64
// like the reference's; the serving path (engine.py) does not use these.
//
//   mpa_ref_rotate      rope.py:37-53       interleaved-pair rotation by pos * inv_freq
//   mpa_ref_logits      attention.py:84-86, 154, 276: q . x / sqrt(d) for G query rows
//   mpa_ref_partial     attention.py:58-68 `_partial_from_logits` (m, s, a) (+ normalised weights,
//                       attention.py:105-117 `exact_weights`)
//   mpa_ref_group_scores attention.py:144-164, 267-290: e = exp(l - max_g), score = mean_g e / (e . N)
//   mpa_ref_nearest     clustering.py:84-88 + argmin (ties: lowest id)
//   mpa_ref_seg_stats   clustering.py:113-120 member means (in member order; size-weighted for the
//                       coarse level, clustering.py:255-257) and squared error
//                       about given centroids (clustering.py:195-203 `wcss`)
#include "mpa_common.cuh"

namespace mpa {
namespace ref {

constexpr int kT = 256;

__device__ __forceinline__ double block_sum_d(double v, double* sh) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += sh[i];
    __syncthreads();
    return r;
}
__device__ __forceinline__ double block_max_d(double v, double* sh) {
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = -INFINITY;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmax(r, sh[i]);
    __syncthreads();
    return r;
}

__global__ void rotate_kernel(const double* __restrict__ x, const double* __restrict__ pos, int n, int d,
                              const double* __restrict__ inv_freq, double* __restrict__ out) {
    const int h = d / 2;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * h;
         e += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(e / h), i = (int)(e - (long long)r * h);
        double s, c;
        sincos(pos[r] * inv_freq[i], &s, &c);
        const double a = x[(size_t)r * d + 2 * i], b = x[(size_t)r * d + 2 * i + 1];
        out[(size_t)r * d + 2 * i] = __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, s));
        out[(size_t)r * d + 2 * i + 1] = __dadd_rn(__dmul_rn(a, s), __dmul_rn(b, c));
    }
}

// out[g, j] = q[g] . x[j] / sqrt(d): one warp per (g, j)
__global__ void logits_kernel(const double* __restrict__ q, const double* __restrict__ x, int G, int n, int d,
                              double* __restrict__ out) {
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (wid >= G * n) return;
    const int g = wid / n, j = wid - g * n;
    double acc = 0.0;
    for (int k = lane; k < d; k += 32) acc = fma(q[(size_t)g * d + k], x[(size_t)j * d + k], acc);
    acc = warp_sum(acc);
    if (lane == 0) out[(size_t)g * n + j] = acc / sqrt((double)d);
}

// one CTA: m = max l, w = exp(l - m) (* weights), s = sum w, a = w @ V; out = [a (d), m, s]
__global__ void partial_kernel(const double* __restrict__ lg, const double* __restrict__ v,
                               const double* __restrict__ wts, int n, int d, double* __restrict__ out,
                               double* __restrict__ wout) {
    __shared__ double sh[32];
    double m = -INFINITY;
    for (int j = threadIdx.x; j < n; j += blockDim.x) m = fmax(m, lg[j]);
    m = block_max_d(m, sh);
    double s = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double w = exp(lg[j] - m) * (wts ? wts[j] : 1.0);
        s += w;
    }
    s = block_sum_d(s, sh);
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        double a = 0.0;
        for (int j = 0; j < n; ++j) a = fma(exp(lg[j] - m) * (wts ? wts[j] : 1.0), v[(size_t)j * d + k], a);
        out[k] = a;
    }
    if (threadIdx.x == 0) {
        out[d] = m;
        out[d + 1] = s;
    }
    if (wout)
        for (int j = threadIdx.x; j < n; j += blockDim.x) wout[j] = exp(lg[j] - m) * (wts ? wts[j] : 1.0) / s;
}

// one CTA: scores[j] = mean_g e[g, j] / (e[g] . sizes), e = exp(l - max_g l)
__global__ void group_scores_kernel(const double* __restrict__ lg, const double* __restrict__ sizes, int G, int n,
                                    double* __restrict__ scores, double* __restrict__ zout) {
    __shared__ double sh[32];
    __shared__ double s_m[8], s_z[8];
    for (int g = 0; g < G; ++g) {
        double m = -INFINITY;
        for (int j = threadIdx.x; j < n; j += blockDim.x) m = fmax(m, lg[(size_t)g * n + j]);
        m = block_max_d(m, sh);
        double z = 0.0;
        for (int j = threadIdx.x; j < n; j += blockDim.x) z += exp(lg[(size_t)g * n + j] - m) * sizes[j];
        z = block_sum_d(z, sh);
        if (threadIdx.x == 0) {
            s_m[g] = m;
            s_z[g] = z;
            if (zout) zout[g] = z;
        }
        __syncthreads();
    }
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        double sc = 0.0;
        for (int g = 0; g < G; ++g) {
            const double e = exp(lg[(size_t)g * n + j] - s_m[g]);
            sc = g ? sc + e / s_z[g] : e / s_z[g];
        }
        scores[j] = sc / (double)G;
    }
}

// assign[i] = argmin_c |p_i|^2 + |c|^2 - 2 p_i . c (first minimum): one warp per point
__global__ void nearest_kernel(const double* __restrict__ p, const double* __restrict__ c, int n, int k, int d,
                               int64_t* __restrict__ assign) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i >= n) return;
    double p2 = 0.0;
    for (int e = 0; e < d; ++e) p2 = fma(p[(size_t)i * d + e], p[(size_t)i * d + e], p2);
    double best = INFINITY;
    int bi = 0x7fffffff;
    for (int j = lane; j < k; j += 32) {
        double c2 = 0.0, dot = 0.0;
        for (int e = 0; e < d; ++e) {
            const double ce = c[(size_t)j * d + e];
            c2 = fma(ce, ce, c2);
            dot = fma(p[(size_t)i * d + e], ce, dot);
        }
        const double dist = p2 + c2 - 2.0 * dot;
        if (dist < best) {
            best = dist;
            bi = j;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob < best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if (lane == 0) assign[i] = bi;
}

// per cluster (CSR off / idx into rows of p): mean[c] (sequential in member order, /count) and,
// with cent given, sqerr += sum |p - cent[c]|^2
__global__ void seg_stats_kernel(const double* __restrict__ p, const int64_t* __restrict__ off,
                                 const int64_t* __restrict__ idx, const double* __restrict__ wts, int k, int d,
                                 double* __restrict__ mean, const double* __restrict__ cent,
                                 double* __restrict__ sqerr) {
    const int c = blockIdx.x;
    if (c >= k) return;
    const long long b = off[c], e = off[c + 1];
    double wsum = 0.0;
    if (wts)
        for (long long m = b; m < e; ++m) wsum = __dadd_rn(wsum, wts[idx[m]]);
    for (int t = threadIdx.x; t < d; t += blockDim.x) {
        double s = 0.0;  // in member order, like np.add.at / a Python sum over the members
        for (long long m = b; m < e; ++m) {
            const double x = p[(size_t)idx[m] * d + t];
            s = __dadd_rn(s, wts ? __dmul_rn(x, wts[idx[m]]) : x);
        }
        if (mean) mean[(size_t)c * d + t] = e > b ? s / (wts ? wsum : (double)(e - b)) : 0.0;
    }
    if (cent && sqerr) {
        __shared__ double sh[32];
        double acc = 0.0;
        for (long long m = b + threadIdx.x; m < e; m += blockDim.x)
            for (int t = 0; t < d; ++t) {
                const double df = p[(size_t)idx[m] * d + t] - cent[(size_t)c * d + t];
                acc = fma(df, df, acc);
            }
        acc = block_sum_d(acc, sh);
        if (threadIdx.x == 0) atomicAdd(sqerr, acc);
    }
}

}  // namespace ref
}  // namespace mpa

using namespace mpa;

extern "C" int mpa_ref_rotate(const double* x, const double* pos, int n, int d, const double* inv_freq, double* out,
                              void* stream) {
    MPA_REQUIRE(x && pos && inv_freq && out && d % 2 == 0 && d > 0, MPA_ERR_ARG, "mpa_ref_rotate: arguments");
    if (n <= 0) return 0;
    const long long work = (long long)n * (d / 2);
    const int grid = (int)min((work + 255) / 256, 4096ll);
    ref::rotate_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(x, pos, n, d, inv_freq, out);
    return check_launch("mpa_ref_rotate");
}

extern "C" int mpa_ref_logits(const double* q, const double* x, int G, int n, int d, double* out, void* stream) {
    MPA_REQUIRE(q && x && out && G >= 1 && d >= 1, MPA_ERR_ARG, "mpa_ref_logits: arguments");
    if (n <= 0) return 0;
    const long long warps = (long long)G * n;
    ref::logits_kernel<<<(int)((warps * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(q, x, G, n, d, out);
    return check_launch("mpa_ref_logits");
}

extern "C" int mpa_ref_partial(const double* logits, const double* values, const double* weights, int n, int d,
                               double* out, double* weights_out, void* stream) {
    MPA_REQUIRE(logits && values && out && n >= 1 && d >= 1, MPA_ERR_ARG, "mpa_ref_partial: arguments");
    ref::partial_kernel<<<1, ref::kT, 0, (cudaStream_t)stream>>>(logits, values, weights, n, d, out, weights_out);
    return check_launch("mpa_ref_partial");
}

extern "C" int mpa_ref_group_scores(const double* logits, const double* sizes, int G, int n, double* scores,
                                    double* z_out, void* stream) {
    MPA_REQUIRE(logits && sizes && scores && G >= 1 && G <= 8 && n >= 1, MPA_ERR_ARG,
                "mpa_ref_group_scores: arguments");
    ref::group_scores_kernel<<<1, ref::kT, 0, (cudaStream_t)stream>>>(logits, sizes, G, n, scores, z_out);
    return check_launch("mpa_ref_group_scores");
}

extern "C" int mpa_ref_nearest(const double* points, const double* centroids, int n, int k, int d, int64_t* assign,
                               void* stream) {
    MPA_REQUIRE(points && centroids && assign && k >= 1 && d >= 1, MPA_ERR_ARG, "mpa_ref_nearest: arguments");
    if (n <= 0) return 0;
    ref::nearest_kernel<<<(int)(((long long)n * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(points, centroids,
                                                                                                   n, k, d, assign);
    return check_launch("mpa_ref_nearest");
}

extern "C" int mpa_ref_seg_stats(const double* points, const int64_t* off, const int64_t* idx, const double* weights,
                                 int k, int d, double* mean, const double* centroids, double* sqerr, void* stream) {
    MPA_REQUIRE(points && off && idx && d >= 1 && (mean || (centroids && sqerr)), MPA_ERR_ARG,
                "mpa_ref_seg_stats: arguments");
    if (k <= 0) return 0;
    ref::seg_stats_kernel<<<k, 128, 0, (cudaStream_t)stream>>>(points, off, idx, weights, k, d, mean, centroids,
                                                               sqerr);
    return check_launch("mpa_ref_seg_stats");
}
