// K2-K8: batched k-means for the blockwise prefill index, the online cluster update, the
// sliding-window split / settle, and the size-weighted hierarchy.
//
// Reference (pkg/src/multipole_attn/clustering.py):
//   :84-88   `_sq_dists`   ||p||^2 + ||c||^2 - 2 p.c           -> km_assign_kernel (fp64)
//   :91-110  `_repair_empty` steal the farthest member of the largest cluster -> km_round_kernel
//   :113-120 `_means`      np.add.at sequential sums / counts  -> km_means_kernel (in-order fp64)
//   :123-143 `lloyd`       fixed point after >= min_iters      -> mpa_km_lloyd (host-driven loop)
//   :146-167 `_clusters_from_assignment` drop empties, compact  -> mpa_km_write_level
//   :187-192 `fill_value_centroids`                            -> mpa_km_write_level
//   :210-264 `build_hierarchy` weighted Lloyd on fine centroids -> weighted mode (wts != NULL)
//   :439-444 sequential running-mean assignment                 -> mpa_km_seq_assign
//
// Every problem is a contiguous run of rows (a W-block, the final block + appended tokens, one
// side of a split, or the fine centroids of a block), so points are read straight from the
// K_raw cache / the fp64 ledger without gathers.  Means accumulate members in ascending point
// order in fp64, which reproduces np.add.at / np.mean bit-for-bit; the assignment argmin is
// fp64 and matches numpy's except at true ties (|margin| ~ 1e-16 relative).
#include <cub/block/block_radix_sort.cuh>

#include <cstdlib>

#include "mpa_common.cuh"

int mpa_km_assign_tc(const mpa_km& k, cudaStream_t st);  // mpa_km_tc.cu

namespace mpa {

enum { ST_ACTIVE = 0, ST_ROUNDS = 1, ST_DOMEANS = 2, ST_EMPTY = 3 };
constexpr int kMaxExtraRounds = 100;  // clustering.py:30

template <typename T>
__device__ __forceinline__ double load_pt(const mpa_km& km, int l, int row, int k) {
    return elem<T>::to_d(reinterpret_cast<const T*>(km.pts)[((size_t)l * km.tcap + row) * km.d + k]);
}

__device__ __forceinline__ double point_elem(const mpa_km& km, int l, int row, int k) {
    if (km.pts64) return km.pts64[((size_t)l * km.rows64_cap + row) * km.d + k];
    if (km.pts_dtype == MPA_BF16) return load_pt<__nv_bfloat16>(km, l, row, k);
    return load_pt<float>(km, l, row, k);
}

// ---------------------------------------------------------------------------- norms / state

__global__ void km_p2_kernel(mpa_km km) {
    const int p = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= km.prob_n[p]) return;
    const int l = km.prob_l[p], row = km.prob_start[p] + i;
    double s = 0.0;
    for (int k = 0; k < km.d; ++k) {
        const double x = point_elem(km, l, row, k);
        s = __dadd_rn(s, __dmul_rn(x, x));
    }
    km.p2[km.pt_off[p] + i] = s;
}

__global__ void km_c2_kernel(mpa_km km, int only_active) {
    const int p = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= km.prob_k[p]) return;
    if (only_active && !km.state[p * 4 + ST_DOMEANS]) return;
    const double* c = km.cent + (size_t)(km.c_off[p] + j) * km.d;
    double s = 0.0;
    for (int k = 0; k < km.d; ++k) s = __dadd_rn(s, __dmul_rn(c[k], c[k]));
    km.c2[km.c_off[p] + j] = s;
}

__global__ void km_init_state_kernel(mpa_km km) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= km.n_prob) return;
    km.state[p * 4 + ST_ACTIVE] = 1;
    km.state[p * 4 + ST_ROUNDS] = 0;
    km.state[p * 4 + ST_DOMEANS] = 0;
    km.state[p * 4 + ST_EMPTY] = 0;
}

__global__ void km_any_active_kernel(mpa_km km, int* dev_flag) {
    int any = 0, mx = 0;
    for (int p = threadIdx.x; p < km.n_prob; p += blockDim.x) {
        any |= km.state[p * 4 + ST_ACTIVE];
        mx = max(mx, km.state[p * 4 + ST_ROUNDS]);
    }
    any = __syncthreads_or(any);
    __shared__ int smx;
    if (threadIdx.x == 0) smx = 0;
    __syncthreads();
    atomicMax(&smx, mx);
    __syncthreads();
    if (threadIdx.x == 0) {
        dev_flag[0] = any;
        dev_flag[1] = smx;
    }
}

// ---------------------------------------------------------------------------- K2 assignment

constexpr int kAsgBM = 64, kAsgBN = 64, kAsgBK = 16, kAsgThreads = 256;

// fp64 register-tiled distance GEMM with a fused first-min argmin epilogue.
__global__ void __launch_bounds__(kAsgThreads) km_assign_kernel(mpa_km km) {
    const int p = blockIdx.y;
    if (!km.state[p * 4 + ST_ACTIVE]) return;
    const int n = km.prob_n[p], K = km.prob_k[p], d = km.d;
    const int i0 = blockIdx.x * kAsgBM;
    if (i0 >= n) return;
    const int l = km.prob_l[p], start = km.prob_start[p];
    const double* cent = km.cent + (size_t)km.c_off[p] * d;
    const double* c2 = km.c2 + km.c_off[p];
    __shared__ double As[kAsgBK][kAsgBM];
    __shared__ double Bs[kAsgBK][kAsgBN];
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    double p2r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int pi = i0 + ty * 4 + i;
        p2r[i] = pi < n ? km.p2[km.pt_off[p] + pi] : 0.0;
    }
    double best[4];
    int bidx[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        best[i] = INFINITY;
        bidx[i] = 0x7fffffff;
    }
    for (int j0 = 0; j0 < K; j0 += kAsgBN) {
        double acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
        for (int k0 = 0; k0 < d; k0 += kAsgBK) {
            // 64 rows x 16 dims for each operand: 1024 elements, 4 per thread
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int idx = tid + e * kAsgThreads;
                const int r = idx >> 4, kk = idx & 15, k = k0 + kk;
                const int pi = i0 + r, cj = j0 + r;
                As[kk][r] = (pi < n && k < d) ? point_elem(km, l, start + pi, k) : 0.0;
                Bs[kk][r] = (cj < K && k < d) ? cent[(size_t)cj * d + k] : 0.0;
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < kAsgBK; ++kk) {
                double a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int cj = j0 + tx * 4 + j;
            if (cj >= K) continue;
            const double cc = c2[cj];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                // (p2 + c2) - 2 * dot, no contraction (numpy evaluation order)
                const double dist = __dsub_rn(__dadd_rn(p2r[i], cc), __dmul_rn(2.0, acc[i][j]));
                if (dist < best[i] || (dist == best[i] && cj < bidx[i])) {
                    best[i] = dist;
                    bidx[i] = cj;
                }
            }
        }
    }
    // reduce over the 16 tx lanes that share a row group (half-warp)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best[i], o);
            const int oi = __shfl_xor_sync(0xffffffffu, bidx[i], o);
            if (ob < best[i] || (ob == best[i] && oi < bidx[i])) {
                best[i] = ob;
                bidx[i] = oi;
            }
        }
        const int pi = i0 + ty * 4 + i;
        if (tx == 0 && pi < n) km.assign[km.pt_off[p] + pi] = bidx[i];
    }
}

// ---------------------------------------------------------------------------- round control

constexpr int kRoundThreads = 1024;
constexpr int kSortItems = 16;  // 1024 x 16 = 16384 points per problem
constexpr int kMaxPoints = kRoundThreads * kSortItems;
constexpr int kIdxBits = 14;

struct DistIdx {
    double v;
    int i;
};

// counts, sequential empty-cluster repair, convergence decision, prev <- assign, and the
// stable grouping of points by cluster (CUB block radix sort on (cluster << 14 | point)).
__global__ void __launch_bounds__(kRoundThreads) km_round_kernel(mpa_km km, int grouping_only) {
    using Sort = cub::BlockRadixSort<unsigned, kRoundThreads, kSortItems>;
    extern __shared__ __align__(16) unsigned char round_smem[];
    typename Sort::TempStorage& sort_tmp = *reinterpret_cast<typename Sort::TempStorage*>(round_smem);
    __shared__ int s_scan[33];
    __shared__ int s_int[4];
    __shared__ double s_dbl[32];
    __shared__ int s_idx[32];
    const int p = blockIdx.x;
    if (!grouping_only && !km.state[p * 4 + ST_ACTIVE]) {
        if (threadIdx.x == 0) km.state[p * 4 + ST_DOMEANS] = 0;
        return;
    }
    const int n = km.prob_n[p], K = km.prob_k[p], d = km.d;
    const int l = km.prob_l[p], start = km.prob_start[p];
    int* asg = km.assign + km.pt_off[p];
    int* prv = km.prev + km.pt_off[p];
    int* cnt = km.count + km.c_off[p];
    double* cent = km.cent + (size_t)km.c_off[p] * d;

    for (int j = threadIdx.x; j < K; j += blockDim.x) cnt[j] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&cnt[asg[i]], 1);
    __syncthreads();

    if (!grouping_only) {
        // ---- _repair_empty (clustering.py:91-110), sequential and rare
        while (true) {
            int first_empty = 0x7fffffff;
            for (int j = threadIdx.x; j < K; j += blockDim.x)
                if (cnt[j] == 0) first_empty = min(first_empty, j);
            first_empty = __reduce_min_sync(0xffffffffu, first_empty);
            if ((threadIdx.x & 31) == 0) s_idx[threadIdx.x >> 5] = first_empty;
            __syncthreads();
            if (threadIdx.x == 0) {
                int m = 0x7fffffff;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = min(m, s_idx[w]);
                s_int[0] = m;
            }
            __syncthreads();
            const int cid = s_int[0];
            if (cid == 0x7fffffff) break;
            // largest cluster, first max
            int bc = -1, bi = 0x7fffffff;
            for (int j = threadIdx.x; j < K; j += blockDim.x)
                if (cnt[j] > bc || (cnt[j] == bc && j < bi)) {
                    bc = cnt[j];
                    bi = j;
                }
            for (int o = 16; o; o >>= 1) {
                const int oc = __shfl_xor_sync(0xffffffffu, bc, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (oc > bc || (oc == bc && oi < bi)) {
                    bc = oc;
                    bi = oi;
                }
            }
            __syncthreads();
            if ((threadIdx.x & 31) == 0) {
                s_idx[threadIdx.x >> 5] = bi;
                s_dbl[threadIdx.x >> 5] = (double)bc;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int b = s_idx[0];
                double c = s_dbl[0];
                for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                    if (s_dbl[w] > c || (s_dbl[w] == c && s_idx[w] < b)) {
                        c = s_dbl[w];
                        b = s_idx[w];
                    }
                s_int[1] = b;
                s_int[2] = (int)c;
            }
            __syncthreads();
            const int big = s_int[1];
            if (s_int[2] <= 1) break;
            // farthest member of `big` (einsum of (p - c)^2), first max by point index
            double fv = -1.0;
            int fi = 0x7fffffff;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                if (asg[i] != big) continue;
                double s = 0.0;
                for (int k = 0; k < d; ++k) {
                    const double df = __dsub_rn(point_elem(km, l, start + i, k), cent[(size_t)big * d + k]);
                    s = __dadd_rn(s, __dmul_rn(df, df));
                }
                if (s > fv || (s == fv && i < fi)) {
                    fv = s;
                    fi = i;
                }
            }
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, fv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, fi, o);
                if (ov > fv || (ov == fv && oi < fi)) {
                    fv = ov;
                    fi = oi;
                }
            }
            __syncthreads();
            if ((threadIdx.x & 31) == 0) {
                s_dbl[threadIdx.x >> 5] = fv;
                s_idx[threadIdx.x >> 5] = fi;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                double v = s_dbl[0];
                int f = s_idx[0];
                for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                    if (s_dbl[w] > v || (s_dbl[w] == v && s_idx[w] < f)) {
                        v = s_dbl[w];
                        f = s_idx[w];
                    }
                s_int[3] = f;
                asg[f] = cid;
                cnt[big] -= 1;
                cnt[cid] += 1;
            }
            __syncthreads();
            const int far = s_int[3];
            for (int k = threadIdx.x; k < d; k += blockDim.x) cent[(size_t)cid * d + k] = point_elem(km, l, start + far, k);
            if (threadIdx.x == 0 && km.c2) {
                double s = 0.0;
                for (int k = 0; k < d; ++k) {
                    const double x = point_elem(km, l, start + far, k);
                    s = __dadd_rn(s, __dmul_rn(x, x));
                }
                km.c2[km.c_off[p] + cid] = s;
            }
            __syncthreads();
        }

        // ---- convergence decision (clustering.py:136-142)
        const int rounds = km.state[p * 4 + ST_ROUNDS];
        int diff = 0;
        if (rounds >= 1)
            for (int i = threadIdx.x; i < n; i += blockDim.x) diff |= (asg[i] != prv[i]);
        diff = __syncthreads_or(diff);
        if (rounds >= 1 && rounds >= km.min_iters && !diff) {
            if (threadIdx.x == 0) {
                km.state[p * 4 + ST_ACTIVE] = 0;
                km.state[p * 4 + ST_DOMEANS] = 0;
            }
        } else {
            if (threadIdx.x == 0) {
                km.state[p * 4 + ST_DOMEANS] = 1;
                if (rounds >= km.min_iters + kMaxExtraRounds) km.state[p * 4 + ST_ACTIVE] = 0;  // final means
                else km.state[p * 4 + ST_ROUNDS] = rounds + 1;
            }
            for (int i = threadIdx.x; i < n; i += blockDim.x) prv[i] = asg[i];
        }
    }

    // ---- cstart = exclusive scan of counts; stable grouping of points by cluster
    {
        int base = 0;
        for (int j0 = 0; j0 < K; j0 += blockDim.x) {
            const int j = j0 + threadIdx.x;
            const int c = j < K ? cnt[j] : 0;
            int tot;
            const int ex = block_exclusive_scan(c, s_scan, &tot);
            if (j < K) km.cstart[km.c_off[p] + j] = base + ex;
            base += tot;
        }
    }
    unsigned keys[kSortItems];
#pragma unroll
    for (int e = 0; e < kSortItems; ++e) {
        const int i = threadIdx.x * kSortItems + e;
        keys[e] = i < n ? ((unsigned)asg[i] << kIdxBits) | (unsigned)i : 0xffffffffu;
    }
    int kbits = 1;
    while ((1 << kbits) < K) ++kbits;
    Sort(sort_tmp).Sort(keys, 0, min(32, kIdxBits + kbits));
#pragma unroll
    for (int e = 0; e < kSortItems; ++e) {
        const int pos = threadIdx.x * kSortItems + e;
        if (pos < n) km.order[km.pt_off[p] + pos] = (int)(keys[e] & ((1u << kIdxBits) - 1));
    }
}

// ---------------------------------------------------------------------------- K3 means

constexpr int kMeansWarps = 8;

__global__ void __launch_bounds__(kMeansWarps * 32) km_means_kernel(mpa_km km, int force) {
    const int p = blockIdx.y;
    if (!force && !km.state[p * 4 + ST_DOMEANS]) return;
    const int K = km.prob_k[p], d = km.d;
    const int j = blockIdx.x * kMeansWarps + (threadIdx.x >> 5);
    if (j >= K) return;
    const int lane = threadIdx.x & 31;
    const int l = km.prob_l[p], start = km.prob_start[p];
    const int c = km.count[km.c_off[p] + j];
    double* cent = km.cent + (size_t)(km.c_off[p] + j) * d;
    const int* ord = km.order + km.pt_off[p] + km.cstart[km.c_off[p] + j];
    if (c == 0) {
        if (!km.wts)  // `_means`: empty clusters are reset to the zero vector
            for (int k = lane; k < d; k += 32) cent[k] = 0.0;
        return;  // weighted (hierarchy) keeps the previous centroid
    }
    double wsum = 0.0;
    for (int k0 = 0; k0 < d; k0 += 32 * 4) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int m = 0; m < c; ++m) {
            const int i = ord[m];
            const double w = km.wts ? (double)km.wts[(size_t)l * km.rows64_cap + start + i] : 1.0;
            if (k0 == 0 && km.wts) wsum = __dadd_rn(wsum, w);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = k0 + lane + 32 * e;
                if (k < d) {
                    const double x = point_elem(km, l, start + i, k);
                    acc[e] = __dadd_rn(acc[e], km.wts ? __dmul_rn(x, w) : x);
                }
            }
        }
        const double den = km.wts ? wsum : (double)c;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int k = k0 + lane + 32 * e;
            if (k < d) cent[k] = __ddiv_rn(acc[e], den);
        }
    }
}

// ---------------------------------------------------------------------------- compaction

__global__ void km_count_nonempty_kernel(mpa_km km, int32_t* nk) {
    const int p = blockIdx.x;
    const int K = km.prob_k[p];
    int c = 0;
    for (int j = threadIdx.x; j < K; j += blockDim.x) c += km.count[km.c_off[p] + j] > 0;
    c = warp_sum(c);
    __shared__ int s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
        nk[p] = t;
    }
}

template <typename TS>
__device__ __forceinline__ void store_serve(void* base, size_t idx, double v) {
    reinterpret_cast<TS*>(base)[idx] = elem<TS>::from_d(v);
}

template <typename TV>
__global__ void __launch_bounds__(kMeansWarps * 32)
km_write_level_kernel(mpa_km km, const TV* __restrict__ vals, const double* __restrict__ fine_vc64,
                      const int32_t* __restrict__ f0, const int32_t* __restrict__ mbase, double* kc64, double* vc64,
                      void* kc, void* vc, int serve_dtype, int32_t* size, int32_t* off, int32_t* idx, int level_cap,
                      int idx_cap) {
    const int p = blockIdx.y;
    const int K = km.prob_k[p], d = km.d;
    const int j = blockIdx.x * kMeansWarps + (threadIdx.x >> 5);
    if (j >= K) return;
    const int lane = threadIdx.x & 31;
    const int c = km.count[km.c_off[p] + j];
    const int l = km.prob_l[p], start = km.prob_start[p];
    // new id = number of non-empty clusters before j
    int before = 0;
    for (int q = lane; q < j; q += 32) before += km.count[km.c_off[p] + q] > 0;
    before = warp_sum(before);
    if (j == K - 1 && lane == 0) {  // CSR terminator of this problem
        const int nk = before + (c > 0);
        off[(size_t)l * (level_cap + 1) + f0[p] + nk] = mbase[p] + km.prob_n[p];
    }
    if (c == 0) return;
    const int gid = f0[p] + before;
    const size_t crow = (size_t)l * level_cap + gid;
    const int cs = km.cstart[km.c_off[p] + j];
    const int* ord = km.order + km.pt_off[p] + cs;
    if (lane == 0) {
        off[(size_t)l * (level_cap + 1) + gid] = mbase[p] + cs;
    }
    for (int m = lane; m < c; m += 32) idx[(size_t)l * idx_cap + mbase[p] + cs + m] = start + ord[m];
    const bool hier = km.pts64 != nullptr;
    int nsum = c;
    if (hier) {
        nsum = 0;
        for (int m = lane; m < c; m += 32) nsum += km.wts[(size_t)l * km.rows64_cap + start + ord[m]];
        nsum = warp_sum(nsum);
    }
    if (lane == 0) size[crow] = nsum;
    const double* src = km.cent + (size_t)(km.c_off[p] + j) * d;
    for (int k = lane; k < d; k += 32) {
        double kv, vv;
        if (!hier) {
            kv = src[k];
            double acc = 0.0;
            for (int m = 0; m < c; ++m)
                acc = __dadd_rn(acc, elem<TV>::to_d(vals[((size_t)l * km.tcap + start + ord[m]) * d + k]));
            vv = __ddiv_rn(acc, (double)c);
        } else {
            // coarse = exact size-weighted mean of the children (clustering.py:249-255)
            double ak = 0.0, av = 0.0;
            for (int m = 0; m < c; ++m) {
                const size_t r = (size_t)l * km.rows64_cap + start + ord[m];
                const double w = (double)km.wts[r];
                ak = __dadd_rn(ak, __dmul_rn(km.pts64[r * d + k], w));
                av = __dadd_rn(av, __dmul_rn(fine_vc64[r * d + k], w));
            }
            kv = __ddiv_rn(ak, (double)nsum);
            vv = __ddiv_rn(av, (double)nsum);
        }
        kc64[crow * d + k] = kv;
        vc64[crow * d + k] = vv;
        if (serve_dtype == MPA_BF16) {
            store_serve<__nv_bfloat16>(kc, crow * d + k, kv);
            store_serve<__nv_bfloat16>(vc, crow * d + k, vv);
        } else {
            store_serve<float>(kc, crow * d + k, kv);
            store_serve<float>(vc, crow * d + k, vv);
        }
    }
}

__global__ void km_assign_from_level_kernel(mpa_km km, const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
                                            int level_cap, int idx_cap, const int32_t* __restrict__ first,
                                            const int32_t* __restrict__ nclus) {
    const int p = blockIdx.y;
    const int l = km.prob_l[p], start = km.prob_start[p], n = km.prob_n[p];
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (j >= nclus[p]) return;
    const int g = first[p] + j;
    const int a = off[(size_t)l * (level_cap + 1) + g], b = off[(size_t)l * (level_cap + 1) + g + 1];
    for (int m = a + (threadIdx.x & 31); m < b; m += 32) {
        const int i = idx[(size_t)l * idx_cap + m] - start;
        if (i >= 0 && i < n) km.assign[km.pt_off[p] + i] = j;
    }
}

// ---------------------------------------------------------------------------- K6 sequential

// distances of the n_new appended tokens to every starting centroid (direct form, fp64):
// the tokens are staged once per CTA in smem (exact as fp32: bf16 / fp32 key sources), each
// thread owns one centroid and eight independent token accumulators
__global__ void __launch_bounds__(128) km_seq_dist_kernel(mpa_km km, const int32_t* __restrict__ tail, int n_new,
                                                          double* dist) {
    extern __shared__ float xs[];  // [n_new][d]
    const int p = blockIdx.y;
    const int K = km.prob_k[p], d = km.d;
    const int l = km.prob_l[p], row0 = km.prob_start[p] + tail[p];
    for (int e = threadIdx.x; e < n_new * d; e += blockDim.x) {
        const int t = e / d, k = e - t * d;
        xs[e] = (float)point_elem(km, l, row0 + t, k);
    }
    __syncthreads();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= K) return;
    const double* c = km.cent + (size_t)(km.c_off[p] + j) * d;
    for (int t0 = 0; t0 < n_new; t0 += 8) {
        double s[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] = 0.0;
        for (int k = 0; k < d; ++k) {
            const double ck = __ldg(c + k);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double df = __dsub_rn(ck, (double)xs[(t0 + u < n_new ? t0 + u : 0) * d + k]);
                s[u] = __dadd_rn(s[u], __dmul_rn(df, df));
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (t0 + u < n_new) dist[((size_t)p * n_new + t0 + u) * km.k_max + j] = s[u];
    }
}

__global__ void __launch_bounds__(1024) km_seq_assign_kernel(mpa_km km, const int32_t* __restrict__ tail, int n_new,
                                                             double* dist) {
    __shared__ double s_v[32];
    __shared__ int s_i[32];
    __shared__ int s_best;
    const int p = blockIdx.x;
    const int K = km.prob_k[p], d = km.d;
    const int l = km.prob_l[p], row0 = km.prob_start[p] + tail[p];
    double* cent = km.cent + (size_t)km.c_off[p] * d;
    int* cnt = km.count + km.c_off[p];
    double* D = dist + (size_t)p * n_new * km.k_max;
    for (int t = 0; t < n_new; ++t) {
        double bv = INFINITY;
        int bi = 0x7fffffff;
        for (int j = threadIdx.x; j < K; j += blockDim.x) {
            const double v = D[(size_t)t * km.k_max + j];
            if (v < bv || (v == bv && j < bi)) {
                bv = v;
                bi = j;
            }
        }
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov < bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if ((threadIdx.x & 31) == 0) {
            s_v[threadIdx.x >> 5] = bv;
            s_i[threadIdx.x >> 5] = bi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double v = s_v[0];
            int b = s_i[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (s_v[w] < v || (s_v[w] == v && s_i[w] < b)) {
                    v = s_v[w];
                    b = s_i[w];
                }
            s_best = b;
            cnt[b] += 1;
        }
        __syncthreads();
        const int c = s_best;
        const double n = (double)cnt[c];
        // centroids[c] += (x - centroids[c]) / counts[c]
        for (int k = threadIdx.x; k < d; k += blockDim.x) {
            const double x = point_elem(km, l, row0 + t, k);
            const double cur = cent[(size_t)c * d + k];
            cent[(size_t)c * d + k] = __dadd_rn(cur, __ddiv_rn(__dsub_rn(x, cur), n));
        }
        __syncthreads();
        // refresh column c for the remaining tokens
        for (int u = t + 1 + threadIdx.x; u < n_new; u += blockDim.x) {
            double s = 0.0;
            for (int k = 0; k < d; ++k) {
                const double df = __dsub_rn(cent[(size_t)c * d + k], point_elem(km, l, row0 + u, k));
                s = __dadd_rn(s, __dmul_rn(df, df));
            }
            D[(size_t)u * km.k_max + c] = s;
        }
        __syncthreads();
    }
}

}  // namespace mpa

using namespace mpa;

namespace {

using RoundSort = cub::BlockRadixSort<unsigned, kRoundThreads, kSortItems>;
constexpr size_t kRoundSmem = sizeof(typename RoundSort::TempStorage);

void launch_round(const mpa_km& k, int grouping_only, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(km_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRoundSmem);
        attr = true;
    }
    km_round_kernel<<<k.n_prob, kRoundThreads, kRoundSmem, st>>>(k, grouping_only);
}

// tcgen05 assignment for bf16 point sources with d = 128 when a workspace is supplied
// (MPA_KM_FP64=1 forces the fp64 CUDA-core kernel for A/B runs)
bool use_tc(const mpa_km& k) {
    static int force_fp64 = -1;
    if (force_fp64 < 0) {
        const char* e = getenv("MPA_KM_FP64");
        force_fp64 = (e && e[0] == '1') ? 1 : 0;
    }
    return !force_fp64 && k.tc_ws && k.pts && !k.pts64 && k.pts_dtype == MPA_BF16 && k.d == 128 && k.pts_rows > 0;
}

int validate(const mpa_km* km) {
    MPA_REQUIRE(km && km->prob_l && km->prob_start && km->prob_n && km->prob_k && km->pt_off && km->c_off &&
                    km->assign && km->prev && km->cent && km->count && km->order && km->cstart && km->state,
                MPA_ERR_ARG, "mpa_km: null argument");
    MPA_REQUIRE((km->pts != nullptr) != (km->pts64 != nullptr), MPA_ERR_ARG, "mpa_km: exactly one of pts / pts64");
    // pts64 with weights: the hierarchy's weighted Lloyd (clustering.py:210-264); without: plain fp64
    // Lloyd over caller points (clustering.py:123-143, the module-level kmeans / lloyd API)
    MPA_REQUIRE(km->n_max <= kMaxPoints, MPA_ERR_UNSUPPORTED, "mpa_km: %d points per problem > %d", km->n_max,
                kMaxPoints);
    MPA_REQUIRE(km->k_max < (1 << (32 - kIdxBits)), MPA_ERR_UNSUPPORTED, "mpa_km: k_max %d too large", km->k_max);
    MPA_REQUIRE(km->d >= 1, MPA_ERR_ARG, "mpa_km: d");
    return 0;
}

}  // namespace

extern "C" int mpa_km_lloyd(const mpa_km* km, int32_t* rounds_out, void* stream) {
    if (int rc = validate(km)) return rc;
    MPA_REQUIRE(km->p2 && km->c2 && km->flag, MPA_ERR_ARG, "mpa_km_lloyd: p2 / c2 / flag");
    if (km->n_prob <= 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const mpa_km k = *km;
    const int P = k.n_prob;
    km_init_state_kernel<<<ceil_div(P, 128), 128, 0, st>>>(k);
    km_p2_kernel<<<dim3(ceil_div(k.n_max, 128), P), 128, 0, st>>>(k);
    km_c2_kernel<<<dim3(ceil_div(k.k_max, 128), P), 128, 0, st>>>(k, 0);
    if (int rc = check_launch("mpa_km_lloyd(init)")) return rc;
    cudaError_t e;
    int32_t hflag[2] = {0, 0};
    int rounds = 0;
    const bool tc = use_tc(k);
    for (int r = 0; r < k.min_iters + kMaxExtraRounds + 2; ++r) {
        if (tc) {
            if (int rc = mpa_km_assign_tc(k, st)) return rc;
        } else {
            km_assign_kernel<<<dim3(ceil_div(k.n_max, kAsgBM), P), kAsgThreads, 0, st>>>(k);
        }
        launch_round(k, 0, st);
        km_means_kernel<<<dim3(ceil_div(k.k_max, kMeansWarps), P), kMeansWarps * 32, 0, st>>>(k, 0);
        km_c2_kernel<<<dim3(ceil_div(k.k_max, 128), P), 128, 0, st>>>(k, 1);
        km_any_active_kernel<<<1, 256, 0, st>>>(k, k.flag);
        if (int rc = check_launch("mpa_km_lloyd(round)")) return rc;
        e = cudaMemcpyAsync(hflag, k.flag, sizeof(hflag), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        MPA_REQUIRE(e == cudaSuccess, (int)e, "mpa_km_lloyd: %s", cudaGetErrorString(e));
        rounds = hflag[1];
        if (!hflag[0]) break;
    }
    // final grouping for compaction (counts / order / cstart of the returned assignment)
    launch_round(k, 1, st);
    if (rounds_out) *rounds_out = rounds;
    return check_launch("mpa_km_lloyd(final)");
}

extern "C" int mpa_km_means(const mpa_km* km, void* stream) {
    if (int rc = validate(km)) return rc;
    if (km->n_prob <= 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const mpa_km k = *km;
    launch_round(k, 1, st);
    km_means_kernel<<<dim3(ceil_div(k.k_max, kMeansWarps), k.n_prob), kMeansWarps * 32, 0, st>>>(k, 1);
    return check_launch("mpa_km_means");
}

extern "C" int mpa_km_count_nonempty(const mpa_km* km, int32_t* nk, void* stream) {
    if (int rc = validate(km)) return rc;
    if (km->n_prob <= 0) return 0;
    km_count_nonempty_kernel<<<km->n_prob, 256, 0, (cudaStream_t)stream>>>(*km, nk);
    return check_launch("mpa_km_count_nonempty");
}

extern "C" int mpa_km_write_level(const mpa_km* km, const void* vals, const double* fine_vc64, const int32_t* f0,
                                  const int32_t* mbase, double* kc64, double* vc64, void* kc, void* vc,
                                  int32_t serve_dtype, int32_t* size, int32_t* off, int32_t* idx, int32_t level_cap,
                                  int32_t idx_cap, void* stream) {
    if (int rc = validate(km)) return rc;
    MPA_REQUIRE(f0 && mbase && kc64 && vc64 && kc && vc && size && off && idx, MPA_ERR_ARG,
                "mpa_km_write_level: null argument");
    MPA_REQUIRE(km->pts64 ? fine_vc64 != nullptr : vals != nullptr, MPA_ERR_ARG,
                "mpa_km_write_level: values source");
    if (km->n_prob <= 0) return 0;
    dim3 grid(ceil_div(km->k_max, kMeansWarps), km->n_prob);
    cudaStream_t st = (cudaStream_t)stream;
    if (km->pts_dtype == MPA_BF16)
        km_write_level_kernel<__nv_bfloat16><<<grid, kMeansWarps * 32, 0, st>>>(
            *km, (const __nv_bfloat16*)vals, fine_vc64, f0, mbase, kc64, vc64, kc, vc, serve_dtype, size, off, idx,
            level_cap, idx_cap);
    else
        km_write_level_kernel<float><<<grid, kMeansWarps * 32, 0, st>>>(*km, (const float*)vals, fine_vc64, f0, mbase,
                                                                        kc64, vc64, kc, vc, serve_dtype, size, off,
                                                                        idx, level_cap, idx_cap);
    return check_launch("mpa_km_write_level");
}

extern "C" int mpa_km_assign_from_level(const mpa_km* km, const int32_t* off, const int32_t* idx, int32_t level_cap,
                                        int32_t idx_cap, const int32_t* first, const int32_t* nclus,
                                        const int32_t* mbase, void* stream) {
    if (int rc = validate(km)) return rc;
    MPA_REQUIRE(off && idx && first && nclus, MPA_ERR_ARG, "mpa_km_assign_from_level: null argument");
    (void)mbase;
    if (km->n_prob <= 0) return 0;
    km_assign_from_level_kernel<<<dim3(ceil_div(km->k_max, 8), km->n_prob), 256, 0, (cudaStream_t)stream>>>(
        *km, off, idx, level_cap, idx_cap, first, nclus);
    return check_launch("mpa_km_assign_from_level");
}

extern "C" int mpa_km_seq_assign(const mpa_km* km, const int32_t* tail_start, int n_new, double* dist, void* stream) {
    if (int rc = validate(km)) return rc;
    MPA_REQUIRE(tail_start && dist, MPA_ERR_ARG, "mpa_km_seq_assign: null argument");
    if (km->n_prob <= 0 || n_new <= 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t smem = sizeof(float) * n_new * km->d;
    MPA_REQUIRE(smem <= 200 * 1024 && !km->pts64, MPA_ERR_UNSUPPORTED, "mpa_km_seq_assign: %d tokens x d %d", n_new,
                km->d);
    cudaFuncSetAttribute(km_seq_dist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    km_seq_dist_kernel<<<dim3(ceil_div(km->k_max, 128), km->n_prob), 128, smem, st>>>(*km, tail_start, n_new, dist);
    km_seq_assign_kernel<<<km->n_prob, 1024, 0, st>>>(*km, tail_start, n_new, dist);
    return check_launch("mpa_km_seq_assign");
}
