// K2 on the 5th-generation tensor cores: the k-means assignment contraction P . C^T of every
// Lloyd problem, tcgen05.mma (kind::f16, bf16 x bf16 -> fp32 in TMEM) fed by TMA, with an
// fp64 certification that keeps the assignment identical to the exact fp64 argmin.
//
// Reference: clustering.py:84-88 (`_sq_dists` = ||p||^2 + ||c||^2 - 2 p.c) and :134 (argmin,
// first minimum).
//
// Exactness.  Points are the bf16 K_raw cache rows (exact in bf16).  Each fp64 centroid is
// split into two bf16 terms c = c1 + c2 + r (|r| <= 2^-16 |c| per element); both partial
// products accumulate into one fp32 TMEM accumulator (the products are exact in fp32), so
// acc = p.c + e with |e| <= 2^-17 (||p||^2 + ||c||^2) from the split residual plus
// <= 2^-16 (..) from fp32 accumulation of 256 products (2^-15 if the adder truncates).  The
// epilogue computes d_j = c2_j - 2 acc_j in fp32, so |d_j - (exact - ||p||^2)| <= tau with
// tau = 2^-13 (||p||^2 + max_j ||c_j||^2) -- at least 2.6x the worst case above.
// Per point it keeps the best column (lowest index on ties) and every column within 2 tau of
// it.  Only those columns can hold the exact fp64 argmin, so a point with no such column is
// certified; otherwise km_recheck_kernel re-scores just the best and its (<= 4) rivals
// with the exact fp64 formula of km_assign_kernel (sequential fp64 dot, (p2 + c2) - 2 dot,
// first minimum), and a point with more rivals is re-scored against every column.
// Certified and re-checked points therefore assign exactly like the fp64 kernel.
//
// Persistent kernel: one CTA per SM walks items of TWO 128-point tiles of one problem; warp 4
// issues TMA + MMA (one elected thread), warps 0-3 / 5-8 drain TMEM (one point per lane).
// N tiles of 128 centroids, 4 K-major sub-tiles each (2 terms x 2 x 64 columns), a 4-deep
// TMA ring, double-buffered accumulators.  Only clusters whose members changed in the last
// Lloyd round (km.dirty) are re-split: the others' centroids are bit-identical.
#include <cstdlib>

#include "mpa_common.cuh"
#include "mpa_tc.cuh"

namespace mpa {

constexpr int kTcM = 128, kTcTerms = 2, kTcSub = 2 * kTcTerms;
constexpr int kTcThreads = 320;  // warp 4 issues the MMAs, warp 9 the TMA loads; warps 0-3 and 5-8
                                 // drain TMEM (one point tile each)
constexpr int kTcTailRows = 64;  // box rows of the narrow-tail centroid map
constexpr int kTcABytes = 2 * kTcM * 128;   // 2 x 64-column chunks of the point tile
constexpr int kTcCand = 4;                  // rival columns kept per point (more -> full re-score)
constexpr int kRecheckStride = 4 + kTcCand; // (problem, point, n rivals, best, rivals...)
static_assert(kTcCand == 4, "recheck entries are two int4");

struct TcWs {
    __nv_bfloat16* terms;  // [kTcTerms][kpad][d]   (a view's column table)
    float* c2f;            // [kpad]
    double* c2max;         // [n_prob]
    int32_t* recheck;      // [sum n][kRecheckStride]
    int32_t* full;         // [sum n][2] (problem, point)
    int32_t* counters;     // [0] rechecks, [1] full re-scores
    float* ub;             // [points of the view] upper bound of exact(assigned) - ||p||^2
    int32_t* dl;           // [sum k] per problem: ids of the clusters that changed last round
    const int32_t* kfull;  // [n_prob] centroids per problem (a view may see fewer columns)
    int kpad;
};

// Workspace of one batch: the column tables, the recheck lists, the per-point bound, the
// incremental plan and the gathered-point view (see mpa_km_assign_tc).
struct TcLayout {
    int kpad, gcap;
    size_t off[16];
    size_t total;
};
enum {
    kWsTerms, kWsC2f, kWsC2max, kWsRecheck, kWsFull, kWsCounters, kWsUb, kWsDTerms, kWsDC2f, kWsDl, kWsPlan,
    kWsGIdx, kWsGPts, kWsGP2, kWsGAsg, kWsGUb
};
enum { kPlanV1n, kPlanV2n, kPlanV2k, kPlanGStart, kPlanGn, kPlanZero, kPlanRows };

__host__ __device__ inline TcLayout tc_ws_layout(int n_prob, int sum_k, int sum_n, int d) {
    TcLayout L;
    L.kpad = (sum_k + 255) / 256 * 256 + 256;
    L.gcap = sum_n / 2 + n_prob + 1;  // problem p gathers <= n_p / 2 points at floor(pt_off / 2) + p
    const size_t sz[16] = {(size_t)kTcTerms * L.kpad * d * 2, (size_t)L.kpad * 4, (size_t)n_prob * 8,
                           (size_t)sum_n * kRecheckStride * 4, (size_t)sum_n * 8, 16, (size_t)sum_n * 4,
                           (size_t)kTcTerms * L.kpad * d * 2, (size_t)L.kpad * 4, (size_t)sum_k * 4,
                           (size_t)n_prob * kPlanRows * 4, (size_t)L.gcap * 4, (size_t)L.gcap * d * 2,
                           (size_t)L.gcap * 8, (size_t)L.gcap * 4, (size_t)L.gcap * 4};
    size_t o = 0;
    for (int i = 0; i < 16; ++i) {
        L.off[i] = o;
        o = (o + sz[i] + 255) & ~(size_t)255;
    }
    L.total = o;
    return L;
}

// fp64 centroid -> two bf16 terms and the fp32 norm
__device__ __forceinline__ void split_terms(const mpa_km& km, int c, int k, __nv_bfloat16* terms, float* c2f, int kpad,
                                            int row) {
    const double v = km.cent[(size_t)c * km.d + k];
    const __nv_bfloat16 t1 = __double2bfloat16(v);
    terms[((size_t)0 * kpad + row) * km.d + k] = t1;
    terms[((size_t)1 * kpad + row) * km.d + k] = __double2bfloat16(v - (double)__bfloat162float(t1));
    if (k == 0) c2f[row] = (float)km.c2[c];
}

// the column tables after the plan: the full table for the clusters that changed in the last
// round (rows c_off + j), and the changed-column table of the incremental problems (rows
// c_off + t, t < v2k)
__global__ void km_tc_prep_kernel(mpa_km km, TcWs ws, TcWs ws2, const int32_t* __restrict__ v2k) {
    const int p = blockIdx.y;
    if (!km.state[p * 4 + 0]) return;
    const int K = km.prob_k[p], d = km.d, c0 = km.c_off[p];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K * d; e += gridDim.x * blockDim.x) {
        const int j = e / d, k = e - j * d;
        if (km.dirty && !km.dirty[c0 + j]) continue;
        split_terms(km, c0 + j, k, ws.terms, ws.c2f, ws.kpad, c0 + j);
    }
    const int nk = v2k[p];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nk * d; e += gridDim.x * blockDim.x) {
        const int t = e / d, k = e - t * d;
        split_terms(km, c0 + ws2.dl[c0 + t], k, ws2.terms, ws2.c2f, ws2.kpad, c0 + t);
    }
}

__global__ void km_tc_reset_kernel(TcWs ws) {
    if (threadIdx.x < 2) ws.counters[threadIdx.x] = 0;
}

// Incremental plan of one Lloyd round (after the previous round's means).  Only the clusters
// whose members changed (km.dirty) moved, so a point whose own cluster did not move keeps it
// unless one of the moved centroids comes within the band (view 2: every point against the
// moved columns only); a point whose own cluster moved is re-scored against every column
// (view 3: those points gathered into a compact block).  Round 0, a problem with more than half
// of its clusters moved, or more than half of its points in moved clusters, is re-scored whole
// (view 1).  One CTA per problem.
__global__ void __launch_bounds__(256) km_tc_plan_kernel(mpa_km km, TcWs ws, int32_t* plan, int32_t* gidx) {
    const int p = blockIdx.x, P = km.n_prob;
    int* v1n = plan + kPlanV1n * P;
    int* v2n = plan + kPlanV2n * P;
    int* v2k = plan + kPlanV2k * P;
    int* gstart = plan + kPlanGStart * P;
    int* gn = plan + kPlanGn * P;
    const int n = km.prob_n[p], K = km.prob_k[p], c0 = km.c_off[p];
    const int g0 = km.pt_off[p] / 2 + p;
    __shared__ int s_scan[33];
    __shared__ double s_red[32];
    if (threadIdx.x == 0) {
        plan[kPlanZero * P + p] = 0;
        gstart[p] = g0;
        if (p == 0) ws.counters[0] = ws.counters[1] = 0;  // the first pass's re-score lists
    }
    if (!km.state[p * 4 + 0]) {
        if (threadIdx.x == 0) v1n[p] = v2n[p] = v2k[p] = gn[p] = 0;
        return;
    }
    {  // per-problem max ||c||^2 (the certification band)
        double m = 0.0;
        for (int j = threadIdx.x; j < K; j += blockDim.x) m = fmax(m, km.c2[c0 + j]);
        m = warp_max(m);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            double r = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, s_red[w]);
            ws.c2max[p] = r;
        }
    }
    int nd = 0, mc = 0;
    for (int j = threadIdx.x; j < K; j += blockDim.x)
        if (km.dirty[c0 + j]) {
            ++nd;
            mc += km.count[c0 + j];
        }
    nd = block_reduce(nd, s_scan, [](int x, int y) { return x + y; });
    mc = block_reduce(mc, s_scan, [](int x, int y) { return x + y; });
    const bool whole = km.state[p * 4 + 1] == 0 || nd * 2 > K || mc > n / 2;
    if (whole) {
        if (threadIdx.x == 0) {
            v1n[p] = n;
            v2n[p] = v2k[p] = gn[p] = 0;
        }
        return;
    }
    if (threadIdx.x == 0) {
        v1n[p] = 0;
        v2k[p] = nd;
        v2n[p] = nd > 0 ? n : 0;
        gn[p] = mc;
    }
    // changed-column list and the members of the changed clusters (grouped by cluster): per
    // chunk of 256 clusters, the moved ones are listed in shared memory, then copied a warp each
    __shared__ int s_src[256], s_dst[256], s_cnt[256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int cbase = 0, mbase = 0;
    for (int j0 = 0; j0 < K; j0 += blockDim.x) {
        const int j = j0 + threadIdx.x;
        const bool dj = j < K && km.dirty[c0 + j];
        const int cnt = dj ? km.count[c0 + j] : 0;
        int tot_c, tot_m;
        const int ec = block_exclusive_scan(dj ? 1 : 0, s_scan, &tot_c);
        const int em = block_exclusive_scan(cnt, s_scan, &tot_m);
        if (dj) {
            ws.dl[c0 + cbase + ec] = j;
            s_src[ec] = km.pt_off[p] + km.cstart[c0 + j];
            s_dst[ec] = g0 + mbase + em;
            s_cnt[ec] = cnt;
        }
        __syncthreads();
        for (int e = warp; e < tot_c; e += blockDim.x >> 5)
            for (int m = lane; m < s_cnt[e]; m += 32) gidx[s_dst[e] + m] = km.order[s_src[e] + m];
        __syncthreads();
        cbase += tot_c;
        mbase += tot_m;
    }
}

// view 3 in: copy the gathered points' rows and norms (one warp per point)
__global__ void km_tc_gather_kernel(mpa_km km, const int32_t* __restrict__ plan, const int32_t* __restrict__ gidx,
                                    __nv_bfloat16* gpts, double* gp2) {
    const int p = blockIdx.y, P = km.n_prob;
    const int n = plan[kPlanGn * P + p], g0 = plan[kPlanGStart * P + p];
    const int lane = threadIdx.x & 31, d = km.d;
    for (int m = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); m < n; m += gridDim.x * (blockDim.x >> 5)) {
        const int i = gidx[g0 + m];
        const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(km.pts) +
                                   ((size_t)km.prob_l[p] * km.tcap + km.prob_start[p] + i) * d;
        for (int k = lane * 8; k < d; k += 256)
            *reinterpret_cast<uint4*>(gpts + (size_t)(g0 + m) * d + k) = __ldg(reinterpret_cast<const uint4*>(src + k));
        if (lane == 0) gp2[g0 + m] = km.p2[km.pt_off[p] + i];
    }
}

// view 3 out: the gathered points' assignment and bound back to their problem rows
__global__ void km_tc_scatter_kernel(mpa_km km, const int32_t* __restrict__ plan, const int32_t* __restrict__ gidx,
                                     const int32_t* __restrict__ gasg, const float* __restrict__ gub, float* ub) {
    const int p = blockIdx.y, P = km.n_prob;
    const int n = plan[kPlanGn * P + p], g0 = plan[kPlanGStart * P + p];
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < n; m += gridDim.x * blockDim.x) {
        const int g = km.pt_off[p] + gidx[g0 + m];
        km.assign[g] = gasg[g0 + m];
        ub[g] = gub[g0 + m];
    }
}

struct TcTile {
    int p, m, n, K, c_off, n_nt, n_last, tail_boxes, row0;
};

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

// An item is TWO 128-point tiles of one problem, so every centroid sub-tile brought from L2
// feeds both; TMEM = 2 buffers x 2 point tiles x 128 columns.  Warps 0-3 drain point tile 0,
// warps 5-8 point tile 1, each thread one point over all columns (no cross-warp merge).
constexpr int kTc2N = 128;
constexpr int kTc2BBytes = kTc2N * 128;  // 128 rows x 64 columns
constexpr int kTc2Stages = 4;
constexpr int kTc2SmemFixed = 2 * 2 * kTcABytes + kTc2Stages * kTc2BBytes;  // A double buffer x 2 tiles + ring

template <bool INCR>
__global__ void __launch_bounds__(kTcThreads, 1)
km_assign_tc2_kernel(const __grid_constant__ CUtensorMap tm_pts,
                     const __grid_constant__ CUtensorMap tm_terms_tail, mpa_km km, TcWs ws) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    if (smem_u32(smem_raw) & 1023) __trap();
    unsigned char* sa = smem_raw;                         // [2 buffers][2 tiles][kTcABytes]
    unsigned char* sb = smem_raw + 4 * kTcABytes;         // [kTc2Stages][kTc2BBytes]
    int* tp = reinterpret_cast<int*>(sb + kTc2Stages * kTc2BBytes);  // [P + 1] item prefix
    // the epilogue's ||c||^2 row of the current / next item, double-buffered (16-byte aligned)
    const int kmax_pad = (km.k_max + 31) & ~31;
    float* c2s = reinterpret_cast<float*>(tp + ((km.n_prob + 1 + 3) & ~3));  // [2][kmax_pad]
    __shared__ __align__(8) uint64_t bar_a[2], bar_a_empty[2], bar_full[kTc2Stages], bar_empty[kTc2Stages],
        bar_acc_full[2], bar_acc_empty[2];
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P = km.n_prob;
    {
        __shared__ int scan[33];
        int base = 0;
        for (int q0 = 0; q0 < P; q0 += blockDim.x) {
            const int q = q0 + threadIdx.x;
            const int nt = q < P && km.state[q * 4 + 0] && km.prob_k[q] > 0 ? (km.prob_n[q] + 2 * kTcM - 1) / (2 * kTcM) : 0;
            int tot;
            const int e = block_exclusive_scan(nt, scan, &tot);
            if (q < P) tp[q] = base + e;
            base += tot;
        }
        if (threadIdx.x == 0) tp[P] = base;
        if (base == 0) return;  // an empty view (late Lloyd rounds): no TMEM, no barriers
    }
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&bar_a[b]), 1);
            mbar_init(smem_u32(&bar_a_empty[b]), 1);
            mbar_init(smem_u32(&bar_acc_full[b]), 1);
            mbar_init(smem_u32(&bar_acc_empty[b]), 8);
        }
        for (int s = 0; s < kTc2Stages; ++s) {
            mbar_init(smem_u32(&bar_full[s]), 1);
            mbar_init(smem_u32(&bar_empty[s]), 1);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const int T = tp[P];
    const int my_items = blockIdx.x < T ? (T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto item_info = [&](int it) {
        const int t = blockIdx.x + it * gridDim.x;
        int lo = 0, hi = P - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tp[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        TcTile x;
        x.p = lo;
        x.m = (t - tp[lo]) * 2;  // first of the two 128-point tiles
        x.n = km.prob_n[lo];
        x.K = km.prob_k[lo];
        x.c_off = km.c_off[lo];
        x.n_nt = (x.K + kTc2N - 1) / kTc2N;
        x.n_last = (x.K - (x.n_nt - 1) * kTc2N + 15) & ~15;
        x.tail_boxes = (x.n_last + kTcTailRows - 1) / kTcTailRows;
        x.row0 = km.prob_l[lo] * km.tcap + km.prob_start[lo] + x.m * kTcM;
        return x;
    };

    if (warp == 9) {
        // TMA producer: the point tiles of each item (two A buffers) and the centroid-term
        // sub-tiles (a kTc2Stages ring), each slot refilled as soon as its MMAs retire
        if (lane == 0 && my_items > 0) {
            prefetch_tmap(&tm_pts);
            prefetch_tmap(&tm_terms_tail);
            auto issue_a = [&](int it, const TcTile& x) {
                if (it >= 2) mbar_wait(smem_u32(&bar_a_empty[it & 1]), ((it - 2) >> 1) & 1);
                const unsigned b = smem_u32(&bar_a[it & 1]);
                unsigned char* dst = sa + (it & 1) * 2 * kTcABytes;
                mbar_expect_tx(b, 2 * kTcABytes);
                for (int m = 0; m < 2; ++m) {
                    tma_load_2d(smem_u32(dst + m * kTcABytes), &tm_pts, 0, x.row0 + m * kTcM, b);
                    tma_load_2d(smem_u32(dst + m * kTcABytes + kTcM * 128), &tm_pts, 64, x.row0 + m * kTcM, b);
                }
            };
            int step = 0;
            TcTile x = item_info(0);
            issue_a(0, x);
            for (int it = 0; it < my_items; ++it) {
                for (int nt = 0; nt < x.n_nt; ++nt) {
                    for (int u = 0; u < kTcSub; ++u, ++step) {
                        const int c = u & 1, slot_i = step % kTc2Stages;
                        if (step >= kTc2Stages)
                            mbar_wait(smem_u32(&bar_empty[slot_i]), (step / kTc2Stages - 1) & 1);
                        const unsigned slot = smem_u32(sb + slot_i * kTc2BBytes);
                        const unsigned fb = smem_u32(&bar_full[slot_i]);
                        const int row = (u >> 1) * ws.kpad + x.c_off + nt * kTc2N;
                        const int boxes = nt + 1 < x.n_nt ? kTc2N / kTcTailRows : x.tail_boxes;
                        mbar_expect_tx(fb, boxes * kTcTailRows * 128);
                        for (int b = 0; b < boxes; ++b)
                            tma_load_2d(slot + b * kTcTailRows * 128, &tm_terms_tail, c * 64, row + b * kTcTailRows, fb);
                    }
                    if (nt == 0 && it + 1 < my_items) issue_a(it + 1, item_info(it + 1));
                }
                if (it + 1 < my_items) x = item_info(it + 1);
            }
        }
        __syncwarp();
    } else if (warp == 4) {
        // MMA issuer: one elected thread
        if (lane == 0 && my_items > 0) {
            int step = 0, gnt = 0;
            for (int it = 0; it < my_items; ++it) {
                const TcTile x = item_info(it);
                mbar_wait(smem_u32(&bar_a[it & 1]), (it >> 1) & 1);
                tc_fence_after();
                for (int nt = 0; nt < x.n_nt; ++nt, ++gnt) {
                    const int buf = gnt & 1;
                    const uint32_t idesc = umma_idesc_bf16_f32(kTcM, nt + 1 < x.n_nt ? kTc2N : x.n_last);
                    if (gnt >= 2) mbar_wait(smem_u32(&bar_acc_empty[buf]), ((gnt - 2) >> 1) & 1);
                    tc_fence_after();
                    for (int u = 0; u < kTcSub; ++u, ++step) {
                        const int c = u & 1;
                        mbar_wait(smem_u32(&bar_full[step % kTc2Stages]), (step / kTc2Stages) & 1);
                        tc_fence_after();
                        const unsigned bslot = smem_u32(sb + (step % kTc2Stages) * kTc2BBytes);
#pragma unroll
                        for (int m = 0; m < 2; ++m) {
                            const unsigned aslot = smem_u32(sa + (it & 1) * 2 * kTcABytes + m * kTcABytes + c * kTcM * 128);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                umma_bf16(tmem + (buf * 2 + m) * kTc2N, umma_desc_sw128(aslot + k * 32),
                                          umma_desc_sw128(bslot + k * 32), idesc, (u | k) ? 1u : 0u);
                        }
                        umma_commit(smem_u32(&bar_empty[step % kTc2Stages]));
                    }
                    umma_commit(smem_u32(&bar_acc_full[buf]));
                }
                umma_commit(smem_u32(&bar_a_empty[it & 1]));
            }
        }
        __syncwarp();
    } else {
        const int m = warp > 4 ? 1 : 0, quarter = warp & 3;
        const int pi = quarter * 32 + lane;
        const int et = (warp > 4 ? warp - 1 : warp) * 32 + lane;  // 0..255 over the epilogue warps
        auto stage_c2 = [&](int it) {
            const TcTile y = item_info(it);
            float* dst = c2s + (it & 1) * kmax_pad;
            // padded to whole 32-column chunks with +inf: a padded column never wins or rivals
            const int kp = (y.K + 31) & ~31;
            for (int j = et; j < kp; j += 256) dst[j] = j < y.K ? __ldg(ws.c2f + y.c_off + j) : INFINITY;
        };
        if (my_items > 0) stage_c2(0);
        named_bar_sync(1, 256);
        int gnt = 0;
        for (int it = 0; it < my_items; ++it) {
            const TcTile x = item_info(it);
            if (it + 1 < my_items) stage_c2(it + 1);  // read only after the barrier ending this item
            const float* c2b = c2s + (it & 1) * kmax_pad;
            const int i = (x.m + m) * kTcM + pi;
            const bool live = i < x.n;
            const int g = km.pt_off[x.p] + (live ? i : 0);
            const double p2 = km.p2[g];
            const double tau = ldexp(p2 + ws.c2max[x.p], -13);  // |approx - exact| bound of every column
            // FULL: the three smallest d_j (indices of two).  INCR: the point keeps its cluster a
            // unless a changed column comes within the band of a's distance (ub = upper bound of
            // exact(a) - p2 from the pass that assigned it); such rivals are collected.
            float b1 = INFINITY, b2 = INFINITY, b3 = INFINITY, thr = -INFINITY;
            int j1 = 0x7fffffff, j2 = 0x7fffffff, a = 0, nr = 0;
            int rv[kTcCand] = {0, 0, 0, 0};
            if (INCR && live) {
                a = km.assign[g];
                if (!km.dirty[x.c_off + a]) thr = __double2float_ru((double)ws.ub[g] + tau);
            }
            for (int nt = 0; nt < x.n_nt; ++nt, ++gnt) {
                const int buf = gnt & 1;
                const int ncol = nt + 1 < x.n_nt ? kTc2N : x.n_last;
                mbar_wait(smem_u32(&bar_acc_full[buf]), (gnt >> 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int c0 = 0; c0 < ncol; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (buf * 2 + m) * kTc2N + c0, v);
                    tmem_ld_wait();
                    const int jb = nt * kTc2N + c0;
                    float c2v[32];
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4) {
                        const float4 t4 = reinterpret_cast<const float4*>(c2b + jb)[q4];
                        c2v[4 * q4] = t4.x;
                        c2v[4 * q4 + 1] = t4.y;
                        c2v[4 * q4 + 2] = t4.z;
                        c2v[4 * q4 + 3] = t4.w;
                    }
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const float dj = fmaf(-2.f, __uint_as_float(v[q]), c2v[q]);
                        if (!INCR) {  // branch-free insertion into (b1, b2, b3)
                            const bool p1 = dj < b1, q2 = dj < b2, q3 = dj < b3;
                            b3 = q2 ? b2 : (q3 ? dj : b3);
                            b2 = p1 ? b1 : (q2 ? dj : b2);
                            j2 = p1 ? j1 : (q2 ? jb + q : j2);
                            b1 = p1 ? dj : b1;
                            j1 = p1 ? jb + q : j1;
                        } else if (dj <= thr) {  // rare: a changed column close to the point
#pragma unroll
                            for (int s = 0; s < kTcCand; ++s)
                                if (s == nr) rv[s] = jb + q;
                            ++nr;
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_acc_empty[buf]));
            }
            if (live) {
                int mode = 0;  // 0: decided, 1: exact re-score of (lead, rivals), 2: exact full scan
                int lead = 0;
                if (!INCR) {
                    const double bnd = 2.0 * tau;
                    if ((double)b2 - (double)b1 > bnd) {
                        km.assign[g] = j1;
                        ws.ub[g] = __double2float_ru((double)b1 + tau);
                    } else if ((double)b3 - (double)b1 > bnd) {
                        mode = 1, lead = j1, nr = 1, rv[0] = j2;
                    } else {
                        mode = 2;
                    }
                } else if (nr > 0) {
                    lead = a;
                    mode = nr > kTcCand ? 2 : 1;
#pragma unroll
                    for (int s = 0; s < kTcCand; ++s) rv[s] = ws.dl[x.c_off + rv[s]];  // changed-column list -> id
                }
                if (mode == 2) {
                    const int r = atomicAdd(&ws.counters[1], 1);
                    ws.full[2 * r] = x.p;
                    ws.full[2 * r + 1] = i;
                } else if (mode == 1) {
                    const int r = atomicAdd(&ws.counters[0], 1);
                    int4* e = reinterpret_cast<int4*>(ws.recheck + (size_t)r * kRecheckStride);
                    e[0] = make_int4(x.p, i, nr, lead);
                    e[1] = make_int4(rv[0], rv[1], rv[2], rv[3]);
                }
            }
            named_bar_sync(1, 256);  // this item's c2 buffer is free; the next item's is complete
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// exact fp64 distance of point x (bf16 row) to centroid j: the arithmetic of km_assign_kernel
// (sequential fp64 dot over k, then (p2 + c2) - 2 dot)
__device__ __forceinline__ double exact_dist(const __nv_bfloat16* __restrict__ x, const double* __restrict__ c,
                                             double p2, double c2) {
    double dot = 0.0;
#pragma unroll 8
    for (int k8 = 0; k8 < 16; ++k8) {
        const uint4 xr = __ldg(reinterpret_cast<const uint4*>(x) + k8);
        const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xr);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const double2 cv = __ldg(reinterpret_cast<const double2*>(c) + k8 * 4 + h);
            const float2 xf = __bfloat1622float2(xh[h]);
            dot = fma((double)xf.x, cv.x, dot);
            dot = fma((double)xf.y, cv.y, dot);
        }
    }
    return __dsub_rn(__dadd_rn(p2, c2), __dmul_rn(2.0, dot));
}

// the same distance to up to N centroids at once (N independent fma chains over one read of x;
// each chain keeps exact_dist's order)
template <int N>
__device__ __forceinline__ void exact_dist_n(const __nv_bfloat16* __restrict__ x, const double* const (&c)[N],
                                             double p2, const double (&c2)[N], double (&out)[N]) {
    double dot[N];
#pragma unroll
    for (int u = 0; u < N; ++u) dot[u] = 0.0;
#pragma unroll 2
    for (int k8 = 0; k8 < 16; ++k8) {
        const uint4 xr = __ldg(reinterpret_cast<const uint4*>(x) + k8);
        const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xr);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const float2 xf = __bfloat1622float2(xh[h]);
#pragma unroll
            for (int u = 0; u < N; ++u) {
                const double2 cv = __ldg(reinterpret_cast<const double2*>(c[u]) + k8 * 4 + h);
                dot[u] = fma((double)xf.x, cv.x, dot[u]);
                dot[u] = fma((double)xf.y, cv.y, dot[u]);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < N; ++u) out[u] = __dsub_rn(__dadd_rn(p2, c2[u]), __dmul_rn(2.0, dot[u]));
}

// exact re-score of the points with rivals inside the band: eight lanes per point, lane 0 the
// best column and lanes 1..n its rivals, first minimum over (dist, index) within the group
constexpr int kRecheckThreads = 256;
__device__ __forceinline__ void recheck_cand(const mpa_km& km, const TcWs& ws) {
    const int nr = ws.counters[0];
    const int sub = threadIdx.x & 7, lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    // warp-uniform trip count (the shuffles below need every lane): four entries per warp per trip
    for (int rb = gw * 4; rb < nr; rb += nw * 4) {
        const int r = rb + (lane >> 3);
        const bool ok = r < nr;
        double best = INFINITY;
        int jb = 0x7fffffff, g = 0;
        if (ok) {
            const int4* e = reinterpret_cast<const int4*>(ws.recheck + (size_t)r * kRecheckStride);
            const int4 h = e[0], rv = e[1];
            const int p = h.x, i = h.y, n_riv = h.z;
            const int j = sub == 0 ? h.w : sub == 1 ? rv.x : sub == 2 ? rv.y : sub == 3 ? rv.z : rv.w;
            g = km.pt_off[p] + i;
            if (sub <= n_riv) {
                const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(km.pts) +
                                         ((size_t)km.prob_l[p] * km.tcap + km.prob_start[p] + i) * km.d;
                const int cj = km.c_off[p] + j;
                best = exact_dist(x, km.cent + (size_t)cj * km.d, km.p2[g], km.c2[cj]);
                jb = j;
            }
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oj = __shfl_xor_sync(0xffffffffu, jb, o);
            if (ob < best || (ob == best && oj < jb)) {
                best = ob;
                jb = oj;
            }
        }
        if (ok && sub == 0) {
            km.assign[g] = jb;
            ws.ub[g] = __double2float_ru(best - km.p2[g]);
        }
    }
}

// exact re-score over every column (points with more than kTcCand rivals): one CTA per point,
// each thread a strided slice of the centroids, then a block-wide first minimum
__device__ __forceinline__ void recheck_full(const mpa_km& km, const TcWs& ws) {
    const int nr = ws.counters[1];
    __shared__ double s_best[kRecheckThreads / 32];
    __shared__ int s_j[kRecheckThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r = blockIdx.x; r < nr; r += gridDim.x) {
        const int p = ws.full[2 * r], i = ws.full[2 * r + 1];
        const int K = ws.kfull[p], g = km.pt_off[p] + i;
        const double p2 = km.p2[g];
        const __nv_bfloat16* x =
            reinterpret_cast<const __nv_bfloat16*>(km.pts) + ((size_t)km.prob_l[p] * km.tcap + km.prob_start[p] + i) * km.d;
        double best = INFINITY;
        int jb = 0x7fffffff;
        // a thread's columns j, j + T, j + 2T scored together (three chains in flight); the
        // ascending-j first minimum is unchanged
        const int T = blockDim.x;
        for (int j0 = threadIdx.x; j0 < K; j0 += 3 * T) {
            const double* cc[3];
            double c2v[3], dist[3];
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int j = min(j0 + u * T, K - 1);  // clamped columns are scored and dropped
                cc[u] = km.cent + (size_t)(km.c_off[p] + j) * km.d;
                c2v[u] = km.c2[km.c_off[p] + j];
            }
            exact_dist_n<3>(x, cc, p2, c2v, dist);
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int j = j0 + u * T;
                if (j < K && (dist[u] < best || (dist[u] == best && j < jb))) {
                    best = dist[u];
                    jb = j;
                }
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oj = __shfl_xor_sync(0xffffffffu, jb, o);
            if (ob < best || (ob == best && oj < jb)) {
                best = ob;
                jb = oj;
            }
        }
        if (lane == 0) {
            s_best[warp] = best;
            s_j[warp] = jb;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < kRecheckThreads / 32; ++w)
                if (s_best[w] < best || (s_best[w] == best && s_j[w] < jb)) {
                    best = s_best[w];
                    jb = s_j[w];
                }
            km.assign[g] = jb;
            ws.ub[g] = __double2float_ru(best - p2);
        }
        __syncthreads();  // s_best reused by the next point
    }
}

// the uncertified points of one pass: candidate re-scores, then full scans
__global__ void __launch_bounds__(kRecheckThreads) km_recheck_kernel(mpa_km km, TcWs ws) {
    recheck_cand(km, ws);
    recheck_full(km, ws);
}

}  // namespace mpa

using namespace mpa;

namespace {

int encode_rows_map(CUtensorMap* out, const void* base, long long rows, int d, int box_rows) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        MPA_REQUIRE(e == cudaSuccess && q == cudaDriverEntryPointSuccess && fn, MPA_ERR_UNSUPPORTED,
                    "cuTensorMapEncodeTiled unavailable (%d)", (int)e);
        encode = reinterpret_cast<EncodeFn>(fn);
    }
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    const CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    MPA_REQUIRE(r == CUDA_SUCCESS, MPA_ERR_ARG, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return 0;
}

}  // namespace

// workspace of the tensor-core assignment for a batch (n_prob problems, sum_k centroids,
// sum_n points, dimension d)
extern "C" size_t mpa_km_tc_workspace(int n_prob, int sum_k, int sum_n, int d) {
    if (n_prob <= 0 || sum_k <= 0 || sum_n <= 0 || d <= 0) return 0;
    return tc_ws_layout(n_prob, sum_k, sum_n, d).total;
}

namespace {
size_t tc2_smem(int n_prob, int k_max) {
    return kTc2SmemFixed + (size_t)((n_prob + 1 + 3) & ~3) * 4 + 2 * (size_t)((k_max + 31) & ~31) * 4;
}
constexpr size_t kTcSmemCap = 227 * 1024 - 2048;  // leaves room for the kernel's static shared memory
}  // namespace

// the tensor-core assignment applies to bf16 points with d = 128 whose per-item state fits in smem
bool mpa_km_tc_applies(const mpa_km& k) {
    return k.tc_ws && k.dirty && k.pts && !k.pts64 && k.pts_dtype == MPA_BF16 && k.d == 128 && k.pts_rows > 0 &&
           tc2_smem(k.n_prob, k.k_max) <= kTcSmemCap;
}

// One assignment pass of a Lloyd round on the tensor cores (mpa_km_lloyd, when
// mpa_km_tc_applies): plan, column tables, then the three views of km_tc_plan_kernel, each a
// tcgen05 pass plus the exact re-scores of its uncertified points.
int mpa_km_assign_tc(const mpa_km& k, cudaStream_t st) {
    const TcLayout L = tc_ws_layout(k.n_prob, k.sum_k, k.sum_n, k.d);
    MPA_REQUIRE(k.tc_ws && (size_t)k.tc_ws_bytes >= L.total, MPA_ERR_ARG, "mpa_km: tensor-core workspace %lld < %zu",
                (long long)k.tc_ws_bytes, L.total);
    const size_t smem = tc2_smem(k.n_prob, k.k_max);
    MPA_REQUIRE(smem <= kTcSmemCap, MPA_ERR_UNSUPPORTED, "mpa_km: tensor-core assignment needs %zu B smem", smem);
    char* base = (char*)k.tc_ws;
    auto at = [&](int i) { return (void*)(base + L.off[i]); };
    const int P = k.n_prob;
    int32_t* plan = (int32_t*)at(kWsPlan);
    int32_t* gidx = (int32_t*)at(kWsGIdx);
    TcWs ws{(__nv_bfloat16*)at(kWsTerms), (float*)at(kWsC2f), (double*)at(kWsC2max), (int32_t*)at(kWsRecheck),
            (int32_t*)at(kWsFull), (int32_t*)at(kWsCounters), (float*)at(kWsUb), (int32_t*)at(kWsDl), k.prob_k,
            L.kpad};
    TcWs ws2 = ws;  // view 2: the changed-column table
    ws2.terms = (__nv_bfloat16*)at(kWsDTerms);
    ws2.c2f = (float*)at(kWsDC2f);
    TcWs ws3 = ws;  // view 3: bounds of the gathered points
    ws3.ub = (float*)at(kWsGUb);
    mpa_km v1 = k, v2 = k, v3 = k;
    v1.prob_n = plan + kPlanV1n * P;
    v2.prob_n = plan + kPlanV2n * P;
    v2.prob_k = plan + kPlanV2k * P;
    v3.pts = at(kWsGPts);
    v3.pts_rows = L.gcap;
    v3.tcap = 0;
    v3.prob_l = plan + kPlanZero * P;
    v3.prob_start = v3.pt_off = plan + kPlanGStart * P;
    v3.prob_n = plan + kPlanGn * P;
    v3.assign = (int32_t*)at(kWsGAsg);
    v3.p2 = (double*)at(kWsGP2);
    CUtensorMap tp, tp3, tt, tt2;
    if (int rc = encode_rows_map(&tp, k.pts, (long long)k.pts_rows, k.d, kTcM)) return rc;
    if (int rc = encode_rows_map(&tp3, v3.pts, (long long)L.gcap, k.d, kTcM)) return rc;
    if (int rc = encode_rows_map(&tt, ws.terms, (long long)kTcTerms * L.kpad, k.d, kTcTailRows)) return rc;
    if (int rc = encode_rows_map(&tt2, ws2.terms, (long long)kTcTerms * L.kpad, k.d, kTcTailRows)) return rc;
    if (int rc = set_max_smem((const void*)km_assign_tc2_kernel<false>, (int)smem)) return rc;
    if (int rc = set_max_smem((const void*)km_assign_tc2_kernel<true>, (int)smem)) return rc;
    const int sms = device_sms();
    const dim3 pgrid(ceil_div(k.k_max * k.d, 256 * 8), P);
    km_tc_plan_kernel<<<P, 256, 0, st>>>(k, ws, plan, gidx);  // also the band and the first pass's reset
    km_tc_prep_kernel<<<pgrid, 256, 0, st>>>(k, ws, ws2, plan + kPlanV2k * P);
    km_tc_gather_kernel<<<dim3(32, P), 256, 0, st>>>(k, plan, gidx, (__nv_bfloat16*)v3.pts, v3.p2);
    auto pass = [&](const CUtensorMap& pm, const CUtensorMap& tm, const mpa_km& v, const TcWs& w, bool incr,
                    bool reset) {
        if (reset) km_tc_reset_kernel<<<1, 32, 0, st>>>(w);  // (the plan resets the first pass's lists)
        if (incr) km_assign_tc2_kernel<true><<<sms, kTcThreads, smem, st>>>(pm, tm, v, w);
        else km_assign_tc2_kernel<false><<<sms, kTcThreads, smem, st>>>(pm, tm, v, w);
        km_recheck_kernel<<<2 * sms, kRecheckThreads, 0, st>>>(v, w);
    };
    pass(tp, tt, v1, ws, false, false);
    pass(tp, tt2, v2, ws2, true, true);
    pass(tp3, tt, v3, ws3, false, true);
    km_tc_scatter_kernel<<<dim3(4, P), 256, 0, st>>>(k, plan, gidx, v3.assign, ws3.ub, ws.ub);
    return check_launch("mpa_km_assign(tcgen05)");
}
