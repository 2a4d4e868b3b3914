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
#include <map>

#include "mpa_common.cuh"

int mpa_km_assign_tc(const mpa_km& k, cudaStream_t st);  // mpa_km_tc.cu
bool mpa_km_tc_applies(const mpa_km& k);

namespace mpa {

enum { ST_ACTIVE = 0, ST_ROUNDS = 1, ST_DOMEANS = 2, ST_REPAIRED = 3 };
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

// four consecutive coordinates k..k+3 of a point row (d % 4 == 0: one vector load)
__device__ __forceinline__ void point_row4(const mpa_km& km, int l, int row, int k, double (&x)[4]) {
    if ((km.d & 3) == 0) {
        if (km.pts64) {
            const double2* b = reinterpret_cast<const double2*>(km.pts64 + ((size_t)l * km.rows64_cap + row) * km.d + k);
            const double2 u = __ldg(b), v = __ldg(b + 1);
            x[0] = u.x, x[1] = u.y, x[2] = v.x, x[3] = v.y;
        } else if (km.pts_dtype == MPA_BF16) {
            const uint2 r = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(km.pts) +
                                                                 ((size_t)l * km.tcap + row) * km.d + k));
            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
            const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
            x[0] = a.x, x[1] = a.y, x[2] = b.x, x[3] = b.y;
        } else {
            const float4 f = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(km.pts) +
                                                                  ((size_t)l * km.tcap + row) * km.d + k));
            x[0] = f.x, x[1] = f.y, x[2] = f.z, x[3] = f.w;
        }
        return;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = k + e < km.d ? point_elem(km, l, row, k + e) : 0.0;
}


__global__ void km_p2_kernel(mpa_km km) {
    const int p = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= km.prob_n[p]) return;
    const int l = km.prob_l[p], row = km.prob_start[p] + i;
    double s = 0.0;
    for (int k = 0; k < km.d; k += 4) {  // sequential over k (numpy's einsum order)
        double x[4];
        point_row4(km, l, row, k, x);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (k + e < km.d) s = __dadd_rn(s, __dmul_rn(x[e], x[e]));
    }
    km.p2[km.pt_off[p] + i] = s;
}

__global__ void km_c2_kernel(mpa_km km, int only_active) {
    const int p = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= km.prob_k[p]) return;
    if (only_active && !km.state[p * 4 + ST_DOMEANS]) return;
    if (km.dirty) {  // start of a Lloyd run: every centroid is new
        if (!only_active) km.dirty[km.c_off[p] + j] = 1;
        else if (!km.dirty[km.c_off[p] + j]) return;
    }
    const double* c = km.cent + (size_t)(km.c_off[p] + j) * km.d;
    double s = 0.0;
    for (int k0 = 0; k0 < km.d; k0 += 16) {  // 16 loads in flight, then the ordered adds
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = k0 + u < km.d ? c[k0 + u] : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (k0 + u < km.d) s = __dadd_rn(s, __dmul_rn(x[u], x[u]));
    }
    km.c2[km.c_off[p] + j] = s;
}

__global__ void km_init_state_kernel(mpa_km km) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= km.n_prob) return;
    km.state[p * 4 + ST_ACTIVE] = 1;
    km.state[p * 4 + ST_ROUNDS] = 0;
    km.state[p * 4 + ST_DOMEANS] = 0;
    km.state[p * 4 + ST_REPAIRED] = 0;
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
// dynamic shared memory of the round kernel: the sort's temporary storage, which also holds the
// assignment copy before the sort (>= kMaxPoints ints), then the counts
constexpr size_t kRoundAsgBytes =
    ((sizeof(typename cub::BlockRadixSort<unsigned, kRoundThreads, kSortItems>::TempStorage) > kMaxPoints * 4
          ? sizeof(typename cub::BlockRadixSort<unsigned, kRoundThreads, kSortItems>::TempStorage)
          : kMaxPoints * 4) + 15) & ~size_t(15);

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
    int* asg_g = km.assign + km.pt_off[p];
    int* prv = km.prev + km.pt_off[p];
    int* cnt_g = km.count + km.c_off[p];
    double* cent = km.cent + (size_t)km.c_off[p] * d;
    // the assignment and the counts live in shared memory for the whole kernel (the assignment
    // aliases the sort's temporary storage, dead until the keys are in registers)
    int* asg = reinterpret_cast<int*>(round_smem);
    int* cnt = reinterpret_cast<int*>(round_smem + kRoundAsgBytes);
    // point i = threadIdx.x + e * kRoundThreads: all loads in flight at once (assignment, and the
    // previous round's for the convergence test and the dirty marks)
    const int rounds = grouping_only ? 0 : km.state[p * 4 + ST_ROUNDS];
    int pv[kSortItems];
    {
        int av[kSortItems];
#pragma unroll
        for (int e = 0; e < kSortItems; ++e) {
            const int i = threadIdx.x + e * kRoundThreads;
            av[e] = i < n ? asg_g[i] : 0;
            pv[e] = i < n && rounds >= 1 ? prv[i] : 0;
        }
#pragma unroll
        for (int e = 0; e < kSortItems; ++e) {
            const int i = threadIdx.x + e * kRoundThreads;
            if (i < n) asg[i] = av[e];
        }
    }
    for (int j = threadIdx.x; j < K; j += blockDim.x) cnt[j] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&cnt[asg[i]], 1);
    __syncthreads();

    if (!grouping_only) {
        // ---- _repair_empty (clustering.py:91-110), sequential and rare
        bool repaired = false;
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
                asg_g[f] = cid;
                cnt[big] -= 1;
                cnt[cid] += 1;
            }
            __syncthreads();
            const int far = s_int[3];
            repaired = true;
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
        int diff = 0;
        if (rounds >= 1)
#pragma unroll
            for (int e = 0; e < kSortItems; ++e) {
                const int i = threadIdx.x + e * kRoundThreads;
                diff |= i < n && asg[i] != pv[e];
            }
        diff = __syncthreads_or(diff);
        if (rounds >= 1 && rounds >= km.min_iters && !diff) {
            if (threadIdx.x == 0) {
                km.state[p * 4 + ST_ACTIVE] = 0;
                km.state[p * 4 + ST_DOMEANS] = 0;
            }
        } else {
            if (threadIdx.x == 0) {
                km.state[p * 4 + ST_DOMEANS] = 1;
                km.state[p * 4 + ST_REPAIRED] = repaired;
                if (rounds >= km.min_iters + kMaxExtraRounds) km.state[p * 4 + ST_ACTIVE] = 0;  // final means
                else km.state[p * 4 + ST_ROUNDS] = rounds + 1;
            }
            if (km.dirty) {
                // clusters whose member set changed this round (the only centroids the means
                // kernel, the norms and the tensor-core split have to recompute)
                int* dt = km.dirty + km.c_off[p];
                if (rounds >= 1 && !repaired) {  // a repair rewrote a centroid: recompute all
                    for (int j = threadIdx.x; j < K; j += blockDim.x) dt[j] = 0;
                    __syncthreads();
#pragma unroll
                    for (int e = 0; e < kSortItems; ++e) {
                        const int i = threadIdx.x + e * kRoundThreads;
                        if (i < n && asg[i] != pv[e]) {
                            dt[asg[i]] = 1;
                            dt[pv[e]] = 1;
                        }
                    }
                } else {
                    for (int j = threadIdx.x; j < K; j += blockDim.x) dt[j] = 1;
                }
            }
            for (int i = threadIdx.x; i < n; i += blockDim.x) prv[i] = asg[i];
        }
    }

    // ---- counts out; cstart = exclusive scan of counts; stable grouping of points by cluster
    for (int j = threadIdx.x; j < K; j += blockDim.x) cnt_g[j] = cnt[j];
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
    // blocked keys (thread t holds points 16t..16t+15, as the stable sort requires), read as int4
    unsigned keys[kSortItems];
#pragma unroll
    for (int e4 = 0; e4 < kSortItems; e4 += 4) {
        const int i = threadIdx.x * kSortItems + e4;
        const int4 a4 = reinterpret_cast<const int4*>(asg)[i >> 2];
        const int av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
            keys[e4 + e] = i + e < n ? ((unsigned)av[e] << kIdxBits) | (unsigned)(i + e) : 0xffffffffu;
    }
    __syncthreads();  // the sort's temporary storage overwrites the assignment copy
    int kbits = 1;
    while ((1 << kbits) < K) ++kbits;
    // stable (points stay ascending inside a cluster); striped out, so the stores coalesce
    Sort(sort_tmp).SortBlockedToStriped(keys, kIdxBits, min(32, kIdxBits + kbits));
#pragma unroll
    for (int e = 0; e < kSortItems; ++e) {
        const int pos = e * kRoundThreads + threadIdx.x;
        if (pos < n) km.order[km.pt_off[p] + pos] = (int)(keys[e] & ((1u << kIdxBits) - 1));
    }
}

// ---------------------------------------------------------------------------- K3 means

constexpr int kMeansWarps = 8;

// four consecutive coordinates of a point row in their storage type
template <typename T> struct Row4;
template <> struct Row4<__nv_bfloat16> {
    uint2 r;
    __device__ __forceinline__ void load(const void* base, size_t off) {
        r = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(base) + off));
    }
    __device__ __forceinline__ double get(int e) const {
        const uint32_t w = e < 2 ? r.x : r.y;
        return (double)__uint_as_float((e & 1) ? (w & 0xffff0000u) : (w << 16));
    }
};
template <> struct Row4<float> {
    float4 r;
    __device__ __forceinline__ void load(const void* base, size_t off) {
        r = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + off));
    }
    __device__ __forceinline__ double get(int e) const { return (double)(e == 0 ? r.x : e == 1 ? r.y : e == 2 ? r.z : r.w); }
};
template <> struct Row4<double> {
    double2 a, b;
    __device__ __forceinline__ void load(const void* base, size_t off) {
        const double2* q = reinterpret_cast<const double2*>(reinterpret_cast<const double*>(base) + off);
        a = __ldg(q);
        b = __ldg(q + 1);
    }
    __device__ __forceinline__ double get(int e) const { return e == 0 ? a.x : e == 1 ? a.y : e == 2 ? b.x : b.y; }
};

// One warp per cluster, lane = four consecutive coordinates (d % 4 == 0).  Each coordinate is
// the sequential fp64 sum of the members in ascending point order (np.add.at,
// clustering.py:113-120); member rows are fetched 8-16 at a time, in their storage type,
// ahead of the (ordered) adds.  Inside a Lloyd run only clusters whose members changed are
// recomputed, and km.dirty is narrowed to the clusters whose centroid actually moved (unless an
// empty-cluster repair rewrote a centroid this round).
constexpr int kMeansBatch = 8;  // value means of km_write_level_kernel
template <typename T>
__device__ __forceinline__ void means_one(const mpa_km& km, bool track, int p, int j, int c, int cstart) {
    constexpr int kBatch = sizeof(T) == 8 ? 8 : 16;  // member rows in flight per lane
    const int d = km.d;
    const int lane = threadIdx.x & 31;
    const int l = km.prob_l[p], start = km.prob_start[p];
    double* cent = km.cent + (size_t)(km.c_off[p] + j) * d;
    const int* ord = km.order + km.pt_off[p] + cstart;
    bool moved = false;
    if (c == 0) {
        if (!km.wts)  // `_means`: empty clusters are reset to the zero vector
            for (int k = lane; k < d; k += 32) {
                moved |= cent[k] != 0.0;
                cent[k] = 0.0;
            }
        // weighted (hierarchy) keeps the previous centroid
    } else {
        const void* src = km.pts64 ? (const void*)km.pts64 : km.pts;
        const size_t rows = km.pts64 ? (size_t)l * km.rows64_cap + start : (size_t)l * km.tcap + start;
        const int32_t* wrow = km.wts ? km.wts + (size_t)l * km.rows64_cap + start : nullptr;
        for (int k0 = 0; k0 < d; k0 += 128) {
            const int k = k0 + lane * 4;
            double acc[4] = {0.0, 0.0, 0.0, 0.0}, old[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) old[e] = k + e < d ? cent[k + e] : 0.0;  // fetched ahead of the sums
            double wsum = 0.0;
            int nxt[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) nxt[u] = u < c ? __ldg(ord + u) : -1;
            for (int m0 = 0; m0 < c; m0 += kBatch) {
                int ii[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) ii[u] = nxt[u];
                Row4<T> xv[kBatch];
                int32_t w[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    w[u] = 1;
                    if (ii[u] >= 0) {
                        if (wrow) w[u] = __ldg(wrow + ii[u]);
                        if (k < d) xv[u].load(src, (rows + ii[u]) * d + k);
                    }
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u)  // the next batch's member ids
                    nxt[u] = m0 + kBatch + u < c ? __ldg(ord + m0 + kBatch + u) : -1;
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    if (ii[u] < 0) continue;
                    const double wu = (double)w[u];
                    if (wrow) wsum = __dadd_rn(wsum, wu);
                    if (k < d)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const double x = xv[u].get(e);
                            acc[e] = __dadd_rn(acc[e], wrow ? __dmul_rn(x, wu) : x);
                        }
                }
            }
            const double den = wrow ? wsum : (double)c;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (k + e < d) {
                    const double v = __ddiv_rn(acc[e], den);
                    moved |= old[e] != v;
                    cent[k + e] = v;
                }
        }
    }
    if (track && !km.state[p * 4 + ST_REPAIRED]) {
        moved = __any_sync(0xffffffffu, moved);
        if (lane == 0 && !moved) km.dirty[km.c_off[p] + j] = 0;
    }
}

// kMeansPerWarp clusters per warp: late Lloyd rounds, with a few moved clusters, launch few CTAs
constexpr int kMeansPerWarp = 4;
template <typename T>
__global__ void __launch_bounds__(kMeansWarps * 32) km_means_kernel(mpa_km km, int force) {
    const int p = blockIdx.y;
    if (!force && !km.state[p * 4 + ST_DOMEANS]) return;
    const int K = km.prob_k[p], lane = threadIdx.x & 31;
    const int j0 = (blockIdx.x * kMeansWarps + (threadIdx.x >> 5)) * kMeansPerWarp;
    const bool track = !force && km.dirty;
    // the warp's clusters' (moved, count, start) in one round of loads
    int todo = 0, cn = 0, cs = 0;
    if (lane < kMeansPerWarp && j0 + lane < K) {
        const int jj = km.c_off[p] + j0 + lane;
        todo = !track || km.dirty[jj];  // same members: same mean
        cn = km.count[jj];
        cs = km.cstart[jj];
    }
#pragma unroll 1
    for (int u = 0; u < kMeansPerWarp; ++u) {
        const int cu = __shfl_sync(0xffffffffu, cn, u), su = __shfl_sync(0xffffffffu, cs, u);
        if (__shfl_sync(0xffffffffu, todo, u)) means_one<T>(km, track, p, j0 + u, cu, su);
    }
}

// generic-d fallback (d % 4 != 0): one lane per coordinate, same summation order
__global__ void __launch_bounds__(kMeansWarps * 32) km_means_generic_kernel(mpa_km km, int force) {
    const int p = blockIdx.y;
    if (!force && !km.state[p * 4 + ST_DOMEANS]) return;
    const int K = km.prob_k[p], d = km.d;
    const int j = blockIdx.x * kMeansWarps + (threadIdx.x >> 5);
    if (j >= K) return;
    const bool track = !force && km.dirty;
    if (track && !km.dirty[km.c_off[p] + j]) return;
    const int lane = threadIdx.x & 31;
    const int l = km.prob_l[p], start = km.prob_start[p];
    const int c = km.count[km.c_off[p] + j];
    double* cent = km.cent + (size_t)(km.c_off[p] + j) * d;
    const int* ord = km.order + km.pt_off[p] + km.cstart[km.c_off[p] + j];
    bool moved = false;
    if (c == 0) {
        if (!km.wts)
            for (int k = lane; k < d; k += 32) {
                moved |= cent[k] != 0.0;
                cent[k] = 0.0;
            }
    } else {
        for (int k = lane; k < d; k += 32) {
            double acc = 0.0, wsum = 0.0;
            for (int m = 0; m < c; ++m) {
                const int i = ord[m];
                const double x = point_elem(km, l, start + i, k);
                if (km.wts) {
                    const double w = (double)km.wts[(size_t)l * km.rows64_cap + start + i];
                    wsum = __dadd_rn(wsum, w);
                    acc = __dadd_rn(acc, __dmul_rn(x, w));
                } else {
                    acc = __dadd_rn(acc, x);
                }
            }
            const double v = __ddiv_rn(acc, km.wts ? wsum : (double)c);
            moved |= cent[k] != v;
            cent[k] = v;
        }
    }
    if (track && !km.state[p * 4 + ST_REPAIRED]) {
        moved = __any_sync(0xffffffffu, moved);
        if (lane == 0 && !moved) km.dirty[km.c_off[p] + j] = 0;
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
km_write_level_kernel(mpa_km km, const TV* __restrict__ vals, KvRows vrow, const double* __restrict__ fine_vc64,
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
    auto store = [&](int k, double kv, double vv) {
        kc64[crow * d + k] = kv;
        vc64[crow * d + k] = vv;
        if (serve_dtype == MPA_BF16) {
            store_serve<__nv_bfloat16>(kc, crow * d + k, kv);
            store_serve<__nv_bfloat16>(vc, crow * d + k, vv);
        } else {
            store_serve<float>(kc, crow * d + k, kv);
            store_serve<float>(vc, crow * d + k, vv);
        }
    };
    if (!hier && (d & 3) == 0) {
        // value means (fill_value_centroids): lane = four consecutive coordinates, member rows
        // fetched kMeansBatch at a time ahead of the ordered fp64 adds (cf. km_means_kernel)
        for (int k0 = 0; k0 < d; k0 += 128) {
            const int k = k0 + lane * 4;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            int nxt[kMeansBatch];
#pragma unroll
            for (int u = 0; u < kMeansBatch; ++u) nxt[u] = u < c ? __ldg(ord + u) : -1;
            for (int m0 = 0; m0 < c; m0 += kMeansBatch) {
                int ii[kMeansBatch];
                Row4<TV> xv[kMeansBatch];
#pragma unroll
                for (int u = 0; u < kMeansBatch; ++u) {
                    ii[u] = nxt[u];
                    if (ii[u] >= 0 && k < d) xv[u].load(vals, (size_t)vrow.row(l, start + ii[u]) * d + k);
                }
#pragma unroll
                for (int u = 0; u < kMeansBatch; ++u)
                    nxt[u] = m0 + kMeansBatch + u < c ? __ldg(ord + m0 + kMeansBatch + u) : -1;
#pragma unroll
                for (int u = 0; u < kMeansBatch; ++u)
                    if (ii[u] >= 0 && k < d)
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc[e] = __dadd_rn(acc[e], xv[u].get(e));
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (k + e < d) store(k + e, src[k + e], __ddiv_rn(acc[e], (double)c));
        }
        return;
    }
    for (int k = lane; k < d; k += 32) {
        double kv, vv;
        if (!hier) {
            kv = src[k];
            double acc = 0.0;
            for (int m = 0; m < c; ++m)
                acc = __dadd_rn(acc, elem<TV>::to_d(vals[(size_t)vrow.row(l, start + ord[m]) * d + k]));
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
        store(k, kv, vv);
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

// distances of the n_new appended tokens to every starting centroid (direct form, fp64, the
// arithmetic of np.einsum("kd,kd->k", c - x, c - x)).  CTA = (64 centroids, 32 tokens), both
// staged in shared memory as fp64 (tokens exact: bf16 / fp32 key sources); thread = one
// centroid x eight tokens.
constexpr int kSeqDistThreads = 256, kSeqDistTok = 32, kSeqDistCent = 64;
__global__ void __launch_bounds__(kSeqDistThreads) km_seq_dist_kernel(mpa_km km, const int32_t* __restrict__ tail,
                                                                      int n_new, double* dist) {
    extern __shared__ double seq_sm[];
    const int p = blockIdx.z;
    const int K = km.prob_k[p], d = km.d, cp = d + 1;
    double* xs = seq_sm;                          // [kSeqDistTok][d]
    double* cs = seq_sm + kSeqDistTok * d;        // [kSeqDistCent][d + 1]
    const int l = km.prob_l[p], t_lo = blockIdx.y * kSeqDistTok, row0 = km.prob_start[p] + tail[p] + t_lo;
    const int j_lo = blockIdx.x * kSeqDistCent;
    const int nt = min(kSeqDistTok, n_new - t_lo), nc = min(kSeqDistCent, K - j_lo);
    for (int e = threadIdx.x; e < nt * d; e += blockDim.x) {
        const int t = e / d, k = e - t * d;
        xs[e] = point_elem(km, l, row0 + t, k);
    }
    const double* cg = km.cent + (size_t)(km.c_off[p] + j_lo) * d;
    for (int e = threadIdx.x; e < nc * d; e += blockDim.x) {
        const int j = e / d, k = e - j * d;
        cs[j * cp + k] = cg[e];
    }
    __syncthreads();
    const int jl = threadIdx.x % kSeqDistCent, t0 = (threadIdx.x / kSeqDistCent) * 8;
    if (jl >= nc || t0 >= nt) return;
    const double* c = cs + jl * cp;
    double s[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) s[u] = 0.0;
    for (int k = 0; k < d; ++k) {
        const double a = c[k];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double df = __dsub_rn(a, xs[(t0 + u < nt ? t0 + u : t0) * d + k]);
            s[u] = __dadd_rn(s[u], __dmul_rn(df, df));
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
        if (t0 + u < nt) dist[((size_t)p * n_new + t_lo + t0 + u) * km.k_max + j_lo + jl] = s[u];
}

// The running-mean pass over the appended tokens (clustering.py:439-444), one CTA per problem.
// Per token: first-min argmin of its distance row, counts[c] += 1, centroid c += (x - c) / n,
// then column c of every later token's row is recomputed from the new centroid (direct form,
// like km_seq_dist_kernel).  Tokens live in shared memory (padded rows: the refresh reads them
// column-wise), and so do the counts; with NC > 0 every thread owns NC fixed columns and loads
// the next token's row while the current token is processed (the one column refreshed in the
// meantime is patched through shared memory).
constexpr int kSeqThreads = 256;
template <int NC>
__global__ void __launch_bounds__(kSeqThreads) km_seq_assign_kernel(mpa_km km, const int32_t* __restrict__ tail,
                                                                    int n_new, double* dist) {
    extern __shared__ __align__(16) unsigned char seq_smem[];
    const int d = km.d, xp = d + 1;
    const int p = blockIdx.x;
    const int K = km.prob_k[p];
    float* xs = reinterpret_cast<float*>(seq_smem);                                           // [n_new][d + 1]
    double* crow = reinterpret_cast<double*>(seq_smem + (((size_t)n_new * xp * 4 + 15) & ~(size_t)15));  // [d]
    int* s_cnt = reinterpret_cast<int*>(crow + d);                                            // [K]
    __shared__ double s_v[kSeqThreads / 32];
    __shared__ int s_i[kSeqThreads / 32];
    __shared__ double s_patch;
    __shared__ int s_patch_j;
    const int l = km.prob_l[p], row0 = km.prob_start[p] + tail[p];
    double* cent = km.cent + (size_t)km.c_off[p] * d;
    int* cnt = km.count + km.c_off[p];
    double* D = dist + (size_t)p * n_new * km.k_max;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < n_new * d; e += kSeqThreads) {
        const int t = e / d, k = e - t * d;
        xs[t * xp + k] = (float)point_elem(km, l, row0 + t, k);  // exact: bf16 / fp32 key sources
    }
    for (int j = tid; j < K; j += kSeqThreads) s_cnt[j] = cnt[j];
    if (tid == 0) s_patch_j = -1;
    double nxt[NC > 0 ? NC : 1];
    if (NC > 0) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int j = tid + c * kSeqThreads;
            nxt[c] = j < K ? D[j] : INFINITY;
        }
    }
    __syncthreads();
    for (int t = 0; t < n_new; ++t) {
        double bv = INFINITY;
        int bi = 0x7fffffff;
        if (NC > 0) {
            const int pj = s_patch_j;
            const double pv = s_patch;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const int j = tid + c * kSeqThreads;
                const double v = j == pj ? pv : nxt[c];
                if (v < bv) {  // columns ascend within a thread: strict < keeps the first
                    bv = v;
                    bi = j;
                }
            }
            if (t + 1 < n_new)
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const int j = tid + c * kSeqThreads;
                    nxt[c] = j < K ? D[(size_t)(t + 1) * km.k_max + j] : INFINITY;
                }
        } else {
            for (int j = tid; j < K; j += kSeqThreads) {
                const double v = D[(size_t)t * km.k_max + j];
                if (v < bv) {
                    bv = v;
                    bi = j;
                }
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov < bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            s_v[warp] = bv;
            s_i[warp] = bi;
        }
        __syncthreads();  // B1
        // every thread reduces the warp minima itself (no second barrier for a broadcast)
        bv = s_v[0];
        bi = s_i[0];
#pragma unroll
        for (int w = 1; w < kSeqThreads / 32; ++w)
            if (s_v[w] < bv || (s_v[w] == bv && s_i[w] < bi)) {
                bv = s_v[w];
                bi = s_i[w];
            }
        const int c = bi;
        const int n = s_cnt[c] + 1;
        // centroids[c] += (x - centroids[c]) / counts[c]
        for (int k = tid; k < d; k += kSeqThreads) {
            const double x = (double)xs[t * xp + k];
            const double cur = cent[(size_t)c * d + k];
            const double nv = __dadd_rn(cur, __ddiv_rn(__dsub_rn(x, cur), (double)n));
            cent[(size_t)c * d + k] = nv;
            crow[k] = nv;
        }
        __syncthreads();  // B2: crow complete, every thread has read s_cnt[c] and s_v
        if (tid == 0) {
            s_cnt[c] = n;
            s_patch_j = c;
        }
        // refresh column c for the remaining tokens
        for (int u = t + 1 + tid; u < n_new; u += kSeqThreads) {
            double sacc = 0.0;
            const float* xu = xs + u * xp;
            for (int k = 0; k < d; ++k) {
                const double df = __dsub_rn(crow[k], (double)xu[k]);
                sacc = __dadd_rn(sacc, __dmul_rn(df, df));
            }
            D[(size_t)u * km.k_max + c] = sacc;
            if (u == t + 1) s_patch = sacc;
        }
        __syncthreads();  // B3: the refreshed column (global D / s_patch) is visible
    }
    for (int j = tid; j < K; j += kSeqThreads) cnt[j] = s_cnt[j];
}

}  // namespace mpa

using namespace mpa;

namespace {

constexpr size_t kRoundSmem = kRoundAsgBytes;  // + k_max counts

void launch_means(const mpa_km& k, int force, cudaStream_t st) {
    const dim3 grid(ceil_div(k.k_max, kMeansWarps), k.n_prob);
    const dim3 grid4(ceil_div(k.k_max, kMeansWarps * kMeansPerWarp), k.n_prob);
    if (k.d & 3) km_means_generic_kernel<<<grid, kMeansWarps * 32, 0, st>>>(k, force);
    else if (k.pts64) km_means_kernel<double><<<grid4, kMeansWarps * 32, 0, st>>>(k, force);
    else if (k.pts_dtype == MPA_BF16) km_means_kernel<__nv_bfloat16><<<grid4, kMeansWarps * 32, 0, st>>>(k, force);
    else km_means_kernel<float><<<grid4, kMeansWarps * 32, 0, st>>>(k, force);
}

int launch_round(const mpa_km& k, int grouping_only, cudaStream_t st) {
    const size_t smem = kRoundSmem + (size_t)k.k_max * 4;
    if (int rc = set_max_smem((const void*)km_round_kernel, (int)smem)) return rc;
    km_round_kernel<<<k.n_prob, kRoundThreads, smem, st>>>(k, grouping_only);
    return 0;
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
    // Host-driven rounds with a pipelined readback: round r's (active, rounds) flag is copied to
    // pinned memory behind its kernels and only waited for after round r + 1 is queued, so the
    // GPU never idles on the host; a round queued after convergence is a no-op (every kernel
    // skips inactive problems).
    constexpr int kRing = 4;
    thread_local int32_t* ring = nullptr;
    if (!ring) {
        const cudaError_t ea = cudaHostAlloc((void**)&ring, kRing * 2 * sizeof(int32_t), cudaHostAllocPortable);
        MPA_REQUIRE(ea == cudaSuccess, (int)ea, "mpa_km_lloyd: pinned flag ring: %s", cudaGetErrorString(ea));
    }
    cudaEvent_t ev[kRing];
    for (int i = 0; i < kRing; ++i) cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    auto cleanup = [&]() {
        for (int i = 0; i < kRing; ++i) cudaEventDestroy(ev[i]);
    };
    int rounds = 0, last = -1;
    const bool tc = mpa_km_tc_applies(k);
    int rc = 0;
    auto enqueue_round = [&](cudaStream_t s) -> int {
        if (tc) {
            if (int r2 = mpa_km_assign_tc(k, s)) return r2;
        } else {
            km_assign_kernel<<<dim3(ceil_div(k.n_max, kAsgBM), P), kAsgThreads, 0, s>>>(k);
        }
        if (int r2 = launch_round(k, 0, s)) return r2;
        launch_means(k, 0, s);
        km_c2_kernel<<<dim3(ceil_div(k.k_max, 128), P), 128, 0, s>>>(k, 1);
        km_any_active_kernel<<<1, 256, 0, s>>>(k, k.flag);
        return check_launch("mpa_km_lloyd(round)");
    };
    // Rounds after the first replay one captured CUDA graph (a round is ~15 launches whose
    // arguments never change): captured on a private stream ordered after / before `st`.
    int dev = 0;
    cudaGetDevice(&dev);
    thread_local std::map<int, cudaStream_t> side_streams;
    cudaStream_t side = side_streams[dev];
    if (!side) {
        cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
        side_streams[dev] = side;
    }
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    cudaEvent_t join;
    cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    cudaEventRecord(join, st);  // the rounds run on `side` after the set-up above
    cudaStreamWaitEvent(side, join, 0);
    for (int r = 0; r < k.min_iters + kMaxExtraRounds + 2; ++r) {
        if (r == 1) {  // capture once the first round has set every kernel attribute
            if (cudaStreamBeginCapture(side, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
                const int crc = enqueue_round(side);
                const cudaError_t ce = cudaStreamEndCapture(side, &graph);
                if (crc || ce != cudaSuccess || cudaGraphInstantiate(&gexec, graph, 0) != cudaSuccess) gexec = nullptr;
            }
            cudaGetLastError();  // a failed capture falls back to eager rounds
        }
        if (gexec) rc = cudaGraphLaunch(gexec, side) == cudaSuccess ? 0 : (int)cudaErrorLaunchFailure;
        else rc = enqueue_round(side);
        if (rc) break;
        cudaError_t e = cudaMemcpyAsync(ring + 2 * (r % kRing), k.flag, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, side);
        if (e == cudaSuccess) e = cudaEventRecord(ev[r % kRing], side);
        if (e == cudaSuccess && r >= 1) e = cudaEventSynchronize(ev[(r - 1) % kRing]);
        if (e != cudaSuccess) {
            set_error("mpa_km_lloyd: %s", cudaGetErrorString(e));
            rc = (int)e;
            break;
        }
        last = r;
        if (r >= 1 && !ring[2 * ((r - 1) % kRing)]) break;  // converged by round r - 1
    }
    if (!rc && last >= 0) {
        const cudaError_t e = cudaEventSynchronize(ev[last % kRing]);
        if (e != cudaSuccess) {
            set_error("mpa_km_lloyd: %s", cudaGetErrorString(e));
            rc = (int)e;
        }
        rounds = ring[2 * (last % kRing) + 1];
    }
    cudaEventRecord(join, side);  // `st` resumes after the last round
    cudaStreamWaitEvent(st, join, 0);
    cleanup();
    cudaEventDestroy(join);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    if (rc) return rc;
    // final grouping for compaction (counts / order / cstart of the returned assignment)
    if (int rc2 = launch_round(k, 1, st)) return rc2;
    if (rounds_out) *rounds_out = rounds;
    return check_launch("mpa_km_lloyd(final)");
}

extern "C" int mpa_km_means(const mpa_km* km, void* stream) {
    if (int rc = validate(km)) return rc;
    if (km->n_prob <= 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const mpa_km k = *km;
    if (int rc = launch_round(k, 1, st)) return rc;
    launch_means(k, 1, st);
    return check_launch("mpa_km_means");
}

extern "C" int mpa_km_count_nonempty(const mpa_km* km, int32_t* nk, void* stream) {
    if (int rc = validate(km)) return rc;
    if (km->n_prob <= 0) return 0;
    km_count_nonempty_kernel<<<km->n_prob, 256, 0, (cudaStream_t)stream>>>(*km, nk);
    return check_launch("mpa_km_count_nonempty");
}

extern "C" int mpa_km_write_level(const mpa_km* km, const mpa_cache* vcache, const double* fine_vc64, const int32_t* f0,
                                  const int32_t* mbase, double* kc64, double* vc64, void* kc, void* vc,
                                  int32_t serve_dtype, int32_t* size, int32_t* off, int32_t* idx, int32_t level_cap,
                                  int32_t idx_cap, void* stream) {
    if (int rc = validate(km)) return rc;
    MPA_REQUIRE(f0 && mbase && kc64 && vc64 && kc && vc && size && off && idx, MPA_ERR_ARG,
                "mpa_km_write_level: null argument");
    MPA_REQUIRE(km->pts64 ? fine_vc64 != nullptr : vcache != nullptr, MPA_ERR_ARG,
                "mpa_km_write_level: values source");
    MPA_REQUIRE(km->pts64 || (vcache->tcap == km->tcap && vcache->dtype == km->pts_dtype), MPA_ERR_ARG,
                "mpa_km_write_level: value cache does not match the key source");
    if (vcache)
        if (int rc = check_cache(vcache, "mpa_km_write_level")) return rc;
    if (km->n_prob <= 0) return 0;
    const void* vals = vcache ? vcache->v : nullptr;
    const KvRows vrow = vcache ? kv_rows(vcache) : KvRows{nullptr, km->tcap, 0, 0, 1};
    dim3 grid(ceil_div(km->k_max, kMeansWarps), km->n_prob);
    cudaStream_t st = (cudaStream_t)stream;
    if (km->pts_dtype == MPA_BF16)
        km_write_level_kernel<__nv_bfloat16><<<grid, kMeansWarps * 32, 0, st>>>(
            *km, (const __nv_bfloat16*)vals, vrow, fine_vc64, f0, mbase, kc64, vc64, kc, vc, serve_dtype, size, off, idx,
            level_cap, idx_cap);
    else
        km_write_level_kernel<float><<<grid, kMeansWarps * 32, 0, st>>>(*km, (const float*)vals, vrow, fine_vc64, f0, mbase,
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
    MPA_REQUIRE(!km->pts64, MPA_ERR_UNSUPPORTED, "mpa_km_seq_assign: fp64 point sources");
    const size_t smem = sizeof(double) * ((size_t)kSeqDistTok * km->d + (size_t)kSeqDistCent * (km->d + 1));
    MPA_REQUIRE(smem <= 220 * 1024, MPA_ERR_UNSUPPORTED, "mpa_km_seq_assign: d %d", km->d);
    if (int rc = set_max_smem((const void*)km_seq_dist_kernel, (int)smem)) return rc;
    km_seq_dist_kernel<<<dim3(ceil_div(km->k_max, kSeqDistCent), ceil_div(n_new, kSeqDistTok), km->n_prob),
                         kSeqDistThreads, smem, st>>>(*km, tail_start, n_new, dist);
    const size_t smem2 = (((size_t)n_new * (km->d + 1) * 4 + 15) & ~(size_t)15) + (size_t)km->d * 8 + (size_t)km->k_max * 4;
    MPA_REQUIRE(smem2 <= 220 * 1024, MPA_ERR_UNSUPPORTED, "mpa_km_seq_assign: %d tokens x d %d, %d centroids", n_new,
                km->d, km->k_max);
    const int nc = ceil_div(km->k_max, kSeqThreads);
    auto go = [&](auto kern) -> int {
        if (int rc = set_max_smem((const void*)kern, (int)smem2)) return rc;
        kern<<<km->n_prob, kSeqThreads, smem2, st>>>(*km, tail_start, n_new, dist);
        return 0;
    };
    int rc = nc <= 1 ? go(km_seq_assign_kernel<1>) : nc == 2 ? go(km_seq_assign_kernel<2>)
           : nc <= 4 ? go(km_seq_assign_kernel<4>) : go(km_seq_assign_kernel<0>);
    if (rc) return rc;
    return check_launch("mpa_km_seq_assign");
}
