// K2 on the 5th-generation tensor cores: the k-means assignment contraction P . C^T of every
// Lloyd problem, tcgen05.mma (kind::f16, bf16 x bf16 -> fp32 in TMEM) fed by TMA, with an
// fp64 certification that keeps the assignment identical to the exact fp64 argmin.
//
// Reference: clustering.py:84-88 (`_sq_dists` = ||p||^2 + ||c||^2 - 2 p.c) and :134 (argmin,
// first minimum).
//
// Exactness.  Points are the bf16 K_raw cache rows (exact in bf16).  Each fp64 centroid is
// split into three bf16 terms c = c1 + c2 + c3 + r (|r| <= 2^-24 |c| per element); the three
// partial products accumulate into one fp32 TMEM accumulator, so acc = p.c + e with
// |e| <= ~2^-16 (||p||^2 + ||c||^2) (fp32 accumulation over d = 128 exact products + the split
// residual; the bound used below is 8x looser).  The epilogue computes d_j = c2_j - 2 acc_j in
// fp32 and keeps, per point, the best (lowest index on ties) and the second-best candidate.
// If second - best > 2 tau with tau = 2^-13 (||p||^2 + max_j ||c_j||^2), the exact fp64
// argmin is provably the same unique index; otherwise the point is re-scored by
// km_recheck_kernel with the exact fp64 formula of km_assign_kernel (sequential fp64 dot,
// (p2 + c2) - 2 dot, first minimum).  Certified and re-checked points therefore assign exactly
// like the fp64 kernel.  In practice only a handful of points per 8K-point problem fall
// inside the band (SURVEY 7.3-2 measured best/second margins < 1e-3 for 2-11 of 8192).
//
// CTA = one (problem, 128-point tile); warp 4 issues TMA + MMA (one elected thread), warps 0-3
// drain TMEM (one point per lane).  N tiles of 256 centroids, 6 K-major sub-tiles each
// (3 terms x 2 x 64 columns), a 4-deep TMA ring, double-buffered 256-column accumulators.
#include <cstdlib>

#include "mpa_common.cuh"
#include "mpa_tc.cuh"

namespace mpa {

constexpr int kTcM = 128, kTcN = 256, kTcStages = 4, kTcSub = 6;
constexpr int kTcThreads = 288;  // warp 4 issues; warps 0-3 and 5-8 drain TMEM (two column halves)
constexpr int kTcTailRows = 64;  // box rows of the narrow-tail centroid map
constexpr int kTcABytes = 2 * kTcM * 128;   // 2 x 64-column chunks of the point tile
constexpr int kTcBBytes = kTcN * 128;       // one 256-row x 64-column centroid sub-tile
constexpr int kTcSmem = 1024 + kTcABytes + kTcStages * kTcBBytes;

struct TcWs {
    __nv_bfloat16* terms;  // [3][kpad][d]
    float* c2f;            // [kpad]
    double* c2max;         // [n_prob]
    int32_t* recheck;      // [sum n][2] (problem, point)
    int32_t* n_recheck;    // [1]
    int kpad;
};

__host__ __device__ inline size_t tc_ws_layout(int n_prob, int sum_k, int sum_n, int d, int* kpad_out,
                                              size_t* off) {
    const int kpad = (sum_k + 255) / 256 * 256 + 256;
    size_t o = 0;
    off[0] = o;
    o += (size_t)3 * kpad * d * 2;
    o = (o + 255) & ~(size_t)255;
    off[1] = o;
    o += (size_t)kpad * 4;
    o = (o + 255) & ~(size_t)255;
    off[2] = o;
    o += (size_t)n_prob * 8;
    o = (o + 255) & ~(size_t)255;
    off[3] = o;
    o += (size_t)sum_n * 8;
    off[4] = o;
    o += 256;
    if (kpad_out) *kpad_out = kpad;
    return o;
}

// fp64 centroids -> three bf16 terms, fp32 norms; per-problem max norm; recheck counter reset
__global__ void km_tc_prep_kernel(mpa_km km, TcWs ws) {
    const int p = blockIdx.y;
    if (!km.state[p * 4 + 0]) return;
    const int K = km.prob_k[p], d = km.d, c0 = km.c_off[p];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K * d; e += gridDim.x * blockDim.x) {
        const int j = e / d, k = e - j * d;
        const double c = km.cent[(size_t)(c0 + j) * d + k];
        const __nv_bfloat16 t1 = __double2bfloat16(c);
        const double r1 = c - (double)__bfloat162float(t1);
        const __nv_bfloat16 t2 = __double2bfloat16(r1);
        const double r2 = r1 - (double)__bfloat162float(t2);
        const __nv_bfloat16 t3 = __double2bfloat16(r2);
        ws.terms[((size_t)0 * ws.kpad + c0 + j) * d + k] = t1;
        ws.terms[((size_t)1 * ws.kpad + c0 + j) * d + k] = t2;
        ws.terms[((size_t)2 * ws.kpad + c0 + j) * d + k] = t3;
        if (k == 0) ws.c2f[c0 + j] = (float)km.c2[c0 + j];
    }
}

__global__ void km_tc_norms_kernel(mpa_km km, TcWs ws) {
    const int p = blockIdx.x;
    if (p == 0 && threadIdx.x == 0) *ws.n_recheck = 0;
    double m = 0.0;
    for (int j = threadIdx.x; j < km.prob_k[p]; j += blockDim.x) m = fmax(m, km.c2[km.c_off[p] + j]);
    __shared__ double red[32];
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
        ws.c2max[p] = r;
    }
}

__global__ void __launch_bounds__(kTcThreads, 1)
km_assign_tc_kernel(const __grid_constant__ CUtensorMap tm_pts, const __grid_constant__ CUtensorMap tm_terms,
                    const __grid_constant__ CUtensorMap tm_terms_tail, mpa_km km, TcWs ws) {
    const int p = blockIdx.y, tile = blockIdx.x;
    if (!km.state[p * 4 + 0]) return;
    const int n = km.prob_n[p], K = km.prob_k[p];
    if (tile * kTcM >= n) return;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    unsigned char* sa = smem;
    unsigned char* sb = smem + kTcABytes;
    __shared__ __align__(8) uint64_t bar_a, bar_full[kTcStages], bar_empty[kTcStages], bar_acc_full[2],
        bar_acc_empty[2];
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar_a), 1);
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(smem_u32(&bar_full[s]), 1);
            mbar_init(smem_u32(&bar_empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&bar_acc_full[b]), 1);
            mbar_init(smem_u32(&bar_acc_empty[b]), 8);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const int n_nt = (K + kTcN - 1) / kTcN, S = n_nt * kTcSub;
    const int c_off = km.c_off[p];
    // the last N tile is only as wide as its centroids (multiple of 16): no MMA or epilogue work on
    // padding columns, and its centroid rows come in 64-row boxes
    const int n_last = (K - (n_nt - 1) * kTcN + 15) & ~15;
    const int tail_boxes = (n_last + kTcTailRows - 1) / kTcTailRows;

    if (warp == 4) {
        if (lane == 0) {
            prefetch_tmap(&tm_pts);
            prefetch_tmap(&tm_terms);
            const int row0 = km.prob_l[p] * km.tcap + km.prob_start[p] + tile * kTcM;
            mbar_expect_tx(smem_u32(&bar_a), kTcABytes);
            tma_load_2d(smem_u32(sa), &tm_pts, 0, row0, smem_u32(&bar_a));
            tma_load_2d(smem_u32(sa + kTcM * 128), &tm_pts, 64, row0, smem_u32(&bar_a));
            auto issue_b = [&](int s) {
                const int nt = s / kTcSub, u = s - nt * kTcSub, t = u >> 1, c = u & 1;
                const unsigned slot = smem_u32(sb + (s % kTcStages) * kTcBBytes);
                const unsigned fb = smem_u32(&bar_full[s % kTcStages]);
                const int row = t * ws.kpad + c_off + nt * kTcN;
                if (nt + 1 < n_nt) {
                    mbar_expect_tx(fb, kTcBBytes);
                    tma_load_2d(slot, &tm_terms, c * 64, row, fb);
                } else {
                    mbar_expect_tx(fb, tail_boxes * kTcTailRows * 128);
                    for (int b = 0; b < tail_boxes; ++b)
                        tma_load_2d(slot + b * kTcTailRows * 128, &tm_terms_tail, c * 64, row + b * kTcTailRows, fb);
                }
            };
            for (int s = 0; s < kTcStages && s < S; ++s) issue_b(s);
            mbar_wait(smem_u32(&bar_a), 0);
            tc_fence_after();
            for (int nt = 0; nt < n_nt; ++nt) {
                const int buf = nt & 1;
                const uint32_t idesc = umma_idesc_bf16_f32(kTcM, nt + 1 < n_nt ? kTcN : n_last);
                if (nt >= 2) mbar_wait(smem_u32(&bar_acc_empty[buf]), ((nt - 2) >> 1) & 1);
                tc_fence_after();
                for (int u = 0; u < kTcSub; ++u) {
                    const int s = nt * kTcSub + u, c = u & 1;
                    mbar_wait(smem_u32(&bar_full[s % kTcStages]), (s / kTcStages) & 1);
                    tc_fence_after();
                    const unsigned bslot = smem_u32(sb + (s % kTcStages) * kTcBBytes);
                    const unsigned aslot = smem_u32(sa + c * kTcM * 128);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        umma_bf16(tmem + buf * kTcN, umma_desc_sw128(aslot + k * 32), umma_desc_sw128(bslot + k * 32),
                                  idesc, (u | k) ? 1u : 0u);
                    umma_commit(smem_u32(&bar_empty[s % kTcStages]));
                    // refill the slot used one step earlier (its MMAs are queued ahead of this step's)
                    if (s >= 1 && s - 1 + kTcStages < S) {
                        mbar_wait(smem_u32(&bar_empty[(s - 1) % kTcStages]), ((s - 1) / kTcStages) & 1);
                        issue_b(s - 1 + kTcStages);
                    }
                }
                umma_commit(smem_u32(&bar_acc_full[buf]));
            }
        }
        __syncwarp();
    }
    // epilogue (warps 0-3 and 5-8): this lane's point = TMEM lane (warp % 4) * 32 + lane; the two
    // warp groups take the two 128-column halves of every N tile, then merge per point
    __shared__ float s_best[kTcM], s_second[kTcM];
    __shared__ int s_jbest[kTcM];
    const int half = warp > 4 ? 1 : 0, quarter = warp & 3;
    const int pi = quarter * 32 + lane, i = tile * kTcM + pi;
    float best = INFINITY, second = INFINITY;
    int jbest = 0x7fffffff;
    if (warp != 4) {
        for (int nt = 0; nt < n_nt; ++nt) {
            const int buf = nt & 1;
            const int ncol = nt + 1 < n_nt ? kTcN : n_last;
            mbar_wait(smem_u32(&bar_acc_full[buf]), (nt >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c0 = half * (kTcN / 2); c0 < (half + 1) * (kTcN / 2) && c0 < ncol; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + buf * kTcN + c0, v);
                tmem_ld_wait();
                const int jb = nt * kTcN + c0;
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const int j = jb + q;
                    if (j < K) {
                        const float dj = __ldg(ws.c2f + c_off + j) - 2.f * __uint_as_float(v[q]);
                        if (dj < best) {
                            second = best;
                            best = dj;
                            jbest = j;
                        } else if (dj < second) {
                            second = dj;
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_acc_empty[buf]));
        }
        if (half) {
            s_best[pi] = best;
            s_second[pi] = second;
            s_jbest[pi] = jbest;
        }
    }
    __syncthreads();
    if (warp < 4 && i < n) {
        // merge with the upper half (its indices are larger within each tile, so ties keep the
        // first minimum by comparing (value, index))
        const float b1 = s_best[pi], s1 = s_second[pi];
        const int j1 = s_jbest[pi];
        if (b1 < best || (b1 == best && j1 < jbest)) {
            second = fminf(s1, best);
            best = b1;
            jbest = j1;
        } else {
            second = fminf(second, b1);
        }
        const int g = km.pt_off[p] + i;
        const double tau = ldexp(km.p2[g] + ws.c2max[p], -13);
        if ((double)second - (double)best > 2.0 * tau) {
            km.assign[g] = jbest;
        } else {
            const int r = atomicAdd(ws.n_recheck, 1);
            ws.recheck[2 * r] = p;
            ws.recheck[2 * r + 1] = i;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// ---- persistent variant (default): one CTA per SM walks (problem, 128-point tile) items; the A
// tile is double-buffered and the centroid-term ring runs on across tiles, so TMEM allocation,
// barrier set-up and the tile's first loads are paid once per SM instead of once per tile.
constexpr int kTcpSmemFixed = 1024 + 2 * kTcABytes + kTcStages * kTcBBytes;

struct TcTile {
    int p, m, n, K, c_off, n_nt, n_last, tail_boxes, row0;
};

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

__global__ void __launch_bounds__(kTcThreads, 1)
km_assign_tcp_kernel(const __grid_constant__ CUtensorMap tm_pts, const __grid_constant__ CUtensorMap tm_terms,
                     const __grid_constant__ CUtensorMap tm_terms_tail, mpa_km km, TcWs ws) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    unsigned char* sa = smem;                      // [2][kTcABytes]
    unsigned char* sb = smem + 2 * kTcABytes;      // [kTcStages][kTcBBytes]
    int* tp = reinterpret_cast<int*>(sb + kTcStages * kTcBBytes);  // [P + 1] tile prefix
    __shared__ __align__(8) uint64_t bar_a[2], bar_a_empty[2], bar_full[kTcStages], bar_empty[kTcStages],
        bar_acc_full[2], bar_acc_empty[2];
    __shared__ uint32_t tmem_base;
    __shared__ float s_best[kTcM], s_second[kTcM];
    __shared__ int s_jbest[kTcM];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P = km.n_prob;
    {  // tile prefix over the active problems (every CTA computes the same)
        __shared__ int scan[33];
        int base = 0;
        for (int q0 = 0; q0 < P; q0 += blockDim.x) {
            const int q = q0 + threadIdx.x;
            const int nt = q < P && km.state[q * 4 + 0] ? (km.prob_n[q] + kTcM - 1) / kTcM : 0;
            int tot;
            const int e = block_exclusive_scan(nt, scan, &tot);
            if (q < P) tp[q] = base + e;
            base += tot;
        }
        if (threadIdx.x == 0) tp[P] = base;
    }
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&bar_a[b]), 1);
            mbar_init(smem_u32(&bar_a_empty[b]), 1);
            mbar_init(smem_u32(&bar_acc_full[b]), 1);
            mbar_init(smem_u32(&bar_acc_empty[b]), 8);
        }
        for (int s = 0; s < kTcStages; ++s) {
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
    const int my_tiles = blockIdx.x < T ? (T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto tile_info = [&](int it) {
        const int t = blockIdx.x + it * gridDim.x;
        int lo = 0, hi = P - 1;  // last problem with tp[q] <= t
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tp[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        TcTile x;
        x.p = lo;
        x.m = t - tp[lo];
        x.n = km.prob_n[lo];
        x.K = km.prob_k[lo];
        x.c_off = km.c_off[lo];
        x.n_nt = (x.K + kTcN - 1) / kTcN;
        x.n_last = (x.K - (x.n_nt - 1) * kTcN + 15) & ~15;
        x.tail_boxes = (x.n_last + kTcTailRows - 1) / kTcTailRows;
        x.row0 = km.prob_l[lo] * km.tcap + km.prob_start[lo] + x.m * kTcM;
        return x;
    };

    if (warp == 4) {
        if (lane == 0 && my_tiles > 0) {
            prefetch_tmap(&tm_pts);
            prefetch_tmap(&tm_terms);
            prefetch_tmap(&tm_terms_tail);
            auto issue_a = [&](int it, const TcTile& x) {
                const unsigned b = smem_u32(&bar_a[it & 1]);
                mbar_expect_tx(b, kTcABytes);
                tma_load_2d(smem_u32(sa + (it & 1) * kTcABytes), &tm_pts, 0, x.row0, b);
                tma_load_2d(smem_u32(sa + (it & 1) * kTcABytes + kTcM * 128), &tm_pts, 64, x.row0, b);
            };
            // load walker: the centroid sub-tiles of every tile in MMA order, kTcStages ahead
            int l_it = 0, l_nt = 0, l_u = 0, l_step = 0;
            TcTile lx = tile_info(0);
            auto load_next = [&]() {
                if (l_it >= my_tiles) return;
                const int t = l_u >> 1, c = l_u & 1, slot_i = l_step % kTcStages;
                const unsigned slot = smem_u32(sb + slot_i * kTcBBytes);
                const unsigned fb = smem_u32(&bar_full[slot_i]);
                const int row = t * ws.kpad + lx.c_off + l_nt * kTcN;
                if (l_nt + 1 < lx.n_nt) {
                    mbar_expect_tx(fb, kTcBBytes);
                    tma_load_2d(slot, &tm_terms, c * 64, row, fb);
                } else {
                    mbar_expect_tx(fb, lx.tail_boxes * kTcTailRows * 128);
                    for (int b = 0; b < lx.tail_boxes; ++b)
                        tma_load_2d(slot + b * kTcTailRows * 128, &tm_terms_tail, c * 64, row + b * kTcTailRows, fb);
                }
                ++l_step;
                if (++l_u == kTcSub) {
                    l_u = 0;
                    if (++l_nt == lx.n_nt) {
                        l_nt = 0;
                        if (++l_it < my_tiles) lx = tile_info(l_it);
                    }
                }
            };
            issue_a(0, lx);
            for (int s = 0; s < kTcStages; ++s) load_next();
            int step = 0, gnt = 0;
            for (int it = 0; it < my_tiles; ++it) {
                const TcTile x = tile_info(it);
                mbar_wait(smem_u32(&bar_a[it & 1]), (it >> 1) & 1);
                tc_fence_after();
                for (int nt = 0; nt < x.n_nt; ++nt, ++gnt) {
                    const int buf = gnt & 1;
                    const uint32_t idesc = umma_idesc_bf16_f32(kTcM, nt + 1 < x.n_nt ? kTcN : x.n_last);
                    if (gnt >= 2) mbar_wait(smem_u32(&bar_acc_empty[buf]), ((gnt - 2) >> 1) & 1);
                    tc_fence_after();
                    for (int u = 0; u < kTcSub; ++u, ++step) {
                        const int c = u & 1;
                        mbar_wait(smem_u32(&bar_full[step % kTcStages]), (step / kTcStages) & 1);
                        tc_fence_after();
                        const unsigned bslot = smem_u32(sb + (step % kTcStages) * kTcBBytes);
                        const unsigned aslot = smem_u32(sa + (it & 1) * kTcABytes + c * kTcM * 128);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            umma_bf16(tmem + buf * kTcN, umma_desc_sw128(aslot + k * 32),
                                      umma_desc_sw128(bslot + k * 32), idesc, (u | k) ? 1u : 0u);
                        umma_commit(smem_u32(&bar_empty[step % kTcStages]));
                        // refill the slot used one step earlier (its MMAs are queued ahead of this step's)
                        if (step >= 1) {
                            mbar_wait(smem_u32(&bar_empty[(step - 1) % kTcStages]), ((step - 1) / kTcStages) & 1);
                            load_next();
                        }
                    }
                    umma_commit(smem_u32(&bar_acc_full[buf]));
                    if (nt == 0 && it + 1 < my_tiles) {
                        // next tile's points into the other A buffer once the tile before this one is done
                        if (it >= 1) mbar_wait(smem_u32(&bar_a_empty[(it + 1) & 1]), ((it - 1) >> 1) & 1);
                        issue_a(it + 1, tile_info(it + 1));
                    }
                }
                umma_commit(smem_u32(&bar_a_empty[it & 1]));
            }
        }
        __syncwarp();
    } else {
        // epilogue: warps 0-3 and 5-8; this lane's point = TMEM lane (warp % 4) * 32 + lane, the two
        // warp groups take the two 128-column halves of every N tile and merge per point
        const int half = warp > 4 ? 1 : 0, quarter = warp & 3;
        const int pi = quarter * 32 + lane;
        int gnt = 0;
        for (int it = 0; it < my_tiles; ++it) {
            const TcTile x = tile_info(it);
            float best = INFINITY, second = INFINITY;
            int jbest = 0x7fffffff;
            for (int nt = 0; nt < x.n_nt; ++nt, ++gnt) {
                const int buf = gnt & 1;
                const int ncol = nt + 1 < x.n_nt ? kTcN : x.n_last;
                mbar_wait(smem_u32(&bar_acc_full[buf]), (gnt >> 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int c0 = half * (kTcN / 2); c0 < (half + 1) * (kTcN / 2) && c0 < ncol; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + buf * kTcN + c0, v);
                    tmem_ld_wait();
                    const int jb = nt * kTcN + c0;
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const int j = jb + q;
                        if (j < x.K) {
                            const float dj = __ldg(ws.c2f + x.c_off + j) - 2.f * __uint_as_float(v[q]);
                            if (dj < best) {
                                second = best;
                                best = dj;
                                jbest = j;
                            } else if (dj < second) {
                                second = dj;
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_acc_empty[buf]));
            }
            if (half) {
                s_best[pi] = best;
                s_second[pi] = second;
                s_jbest[pi] = jbest;
            }
            named_bar_sync(1, 256);
            const int i = x.m * kTcM + pi;
            if (!half && i < x.n) {
                const float b1 = s_best[pi], s1 = s_second[pi];
                const int j1 = s_jbest[pi];
                if (b1 < best || (b1 == best && j1 < jbest)) {
                    second = fminf(s1, best);
                    best = b1;
                    jbest = j1;
                } else {
                    second = fminf(second, b1);
                }
                const int g = km.pt_off[x.p] + i;
                const double tau = ldexp(km.p2[g] + ws.c2max[x.p], -13);
                if ((double)second - (double)best > 2.0 * tau) {
                    km.assign[g] = jbest;
                } else {
                    const int r = atomicAdd(ws.n_recheck, 1);
                    ws.recheck[2 * r] = x.p;
                    ws.recheck[2 * r + 1] = i;
                }
            }
            named_bar_sync(1, 256);  // s_best is rewritten by the next tile
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// ---- paired variant (default): an item is TWO 128-point tiles of one problem, so every centroid
// sub-tile brought from L2 feeds both (half the centroid traffic per point); N tiles of 128
// columns, TMEM = 2 buffers x 2 point tiles x 128 columns.  Warps 0-3 drain point tile 0, warps
// 5-8 point tile 1, each thread one point over all columns (no cross-warp merge).
constexpr int kTc2N = 128;
constexpr int kTc2BBytes = kTc2N * 128;  // 128 rows x 64 columns
constexpr int kTc2Stages = 4;
constexpr int kTc2SmemFixed = 2 * 2 * kTcABytes + kTc2Stages * kTc2BBytes;  // A double buffer x 2 tiles + ring

__global__ void __launch_bounds__(kTcThreads, 1)
km_assign_tc2_kernel(const __grid_constant__ CUtensorMap tm_pts, const __grid_constant__ CUtensorMap tm_terms,
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
            const int nt = q < P && km.state[q * 4 + 0] ? (km.prob_n[q] + 2 * kTcM - 1) / (2 * kTcM) : 0;
            int tot;
            const int e = block_exclusive_scan(nt, scan, &tot);
            if (q < P) tp[q] = base + e;
            base += tot;
        }
        if (threadIdx.x == 0) tp[P] = base;
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

    if (warp == 4) {
        if (lane == 0 && my_items > 0) {
            prefetch_tmap(&tm_pts);
            prefetch_tmap(&tm_terms);
            prefetch_tmap(&tm_terms_tail);
            auto issue_a = [&](int it, const TcTile& x) {
                const unsigned b = smem_u32(&bar_a[it & 1]);
                unsigned char* dst = sa + (it & 1) * 2 * kTcABytes;
                mbar_expect_tx(b, 2 * kTcABytes);
                for (int m = 0; m < 2; ++m) {
                    tma_load_2d(smem_u32(dst + m * kTcABytes), &tm_pts, 0, x.row0 + m * kTcM, b);
                    tma_load_2d(smem_u32(dst + m * kTcABytes + kTcM * 128), &tm_pts, 64, x.row0 + m * kTcM, b);
                }
            };
            int l_it = 0, l_nt = 0, l_u = 0, l_step = 0;
            TcTile lx = item_info(0);
            auto load_next = [&]() {
                if (l_it >= my_items) return;
                const int t = l_u >> 1, c = l_u & 1, slot_i = l_step % kTc2Stages;
                const unsigned slot = smem_u32(sb + slot_i * kTc2BBytes);
                const unsigned fb = smem_u32(&bar_full[slot_i]);
                const int row = t * ws.kpad + lx.c_off + l_nt * kTc2N;
                if (l_nt + 1 < lx.n_nt) {
                    mbar_expect_tx(fb, kTc2BBytes);
                    for (int b = 0; b < kTc2N / kTcTailRows; ++b)
                        tma_load_2d(slot + b * kTcTailRows * 128, &tm_terms_tail, c * 64, row + b * kTcTailRows, fb);
                } else {
                    mbar_expect_tx(fb, lx.tail_boxes * kTcTailRows * 128);
                    for (int b = 0; b < lx.tail_boxes; ++b)
                        tma_load_2d(slot + b * kTcTailRows * 128, &tm_terms_tail, c * 64, row + b * kTcTailRows, fb);
                }
                ++l_step;
                if (++l_u == kTcSub) {
                    l_u = 0;
                    if (++l_nt == lx.n_nt) {
                        l_nt = 0;
                        if (++l_it < my_items) lx = item_info(l_it);
                    }
                }
            };
            issue_a(0, lx);
            for (int s = 0; s < kTc2Stages; ++s) load_next();
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
                        if (step >= 1) {
                            mbar_wait(smem_u32(&bar_empty[(step - 1) % kTc2Stages]), ((step - 1) / kTc2Stages) & 1);
                            load_next();
                        }
                    }
                    umma_commit(smem_u32(&bar_acc_full[buf]));
                    if (nt == 0 && it + 1 < my_items) {
                        if (it >= 1) mbar_wait(smem_u32(&bar_a_empty[(it + 1) & 1]), ((it - 1) >> 1) & 1);
                        issue_a(it + 1, item_info(it + 1));
                    }
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
            for (int j = et; j < y.K; j += 256) dst[j] = __ldg(ws.c2f + y.c_off + j);
        };
        if (my_items > 0) stage_c2(0);
        named_bar_sync(1, 256);
        int gnt = 0;
        for (int it = 0; it < my_items; ++it) {
            const TcTile x = item_info(it);
            if (it + 1 < my_items) stage_c2(it + 1);  // read only after the barrier ending this item
            const float* c2b = c2s + (it & 1) * kmax_pad;
            float best = INFINITY, second = INFINITY;
            int jbest = 0x7fffffff;
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
                        const int j = jb + q;
                        if (j < x.K) {
                            const float dj = c2v[q] - 2.f * __uint_as_float(v[q]);
                            if (dj < best) {
                                second = best;
                                best = dj;
                                jbest = j;
                            } else if (dj < second) {
                                second = dj;
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_acc_empty[buf]));
            }
            const int i = (x.m + m) * kTcM + pi;
            if (i < x.n) {
                const int g = km.pt_off[x.p] + i;
                const double tau = ldexp(km.p2[g] + ws.c2max[x.p], -13);
                if ((double)second - (double)best > 2.0 * tau) {
                    km.assign[g] = jbest;
                } else {
                    const int r = atomicAdd(ws.n_recheck, 1);
                    ws.recheck[2 * r] = x.p;
                    ws.recheck[2 * r + 1] = i;
                }
            }
            named_bar_sync(1, 256);  // this item's c2 buffer is free; the next item's is complete
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// exact fp64 re-scoring of the uncertified points: one CTA (8 warps) per point, each thread
// scoring a strided slice of the problem's centroids with the arithmetic of km_assign_kernel
// (sequential fp64 dot, (p2 + c2) - 2 dot), then a block-wide first minimum over (dist, index).
// Spreading a point over 256 threads keeps enough fp64 centroid rows in flight (the rows are
// cold in L2: the tensor-core pass reads the bf16 terms).
constexpr int kRecheckThreads = 256;
__global__ void __launch_bounds__(kRecheckThreads) km_recheck_kernel(mpa_km km, TcWs ws) {
    const int nr = *ws.n_recheck;
    __shared__ double x[128];
    __shared__ double s_best[kRecheckThreads / 32];
    __shared__ int s_j[kRecheckThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r = blockIdx.x; r < nr; r += gridDim.x) {
        const int p = ws.recheck[2 * r], i = ws.recheck[2 * r + 1];
        const int K = km.prob_k[p], d = km.d, l = km.prob_l[p], row = km.prob_start[p] + i;
        const int g = km.pt_off[p] + i;
        const double p2 = km.p2[g];
        const __nv_bfloat16* pt = reinterpret_cast<const __nv_bfloat16*>(km.pts) + ((size_t)l * km.tcap + row) * d;
        for (int k = threadIdx.x; k < 128; k += blockDim.x) x[k] = (double)__bfloat162float(pt[k]);
        __syncthreads();
        double best = INFINITY;
        int jb = 0x7fffffff;
        for (int j = threadIdx.x; j < K; j += blockDim.x) {
            const double2* c = reinterpret_cast<const double2*>(km.cent + (size_t)(km.c_off[p] + j) * d);
            double dot = 0.0;  // sequential over k, like km_assign_kernel
#pragma unroll 8
            for (int k2 = 0; k2 < 64; ++k2) {
                const double2 cv = __ldg(c + k2);
                dot = fma(x[2 * k2], cv.x, dot);
                dot = fma(x[2 * k2 + 1], cv.y, dot);
            }
            const double dist = __dsub_rn(__dadd_rn(p2, km.c2[km.c_off[p] + j]), __dmul_rn(2.0, dot));
            if (dist < best || (dist == best && j < jb)) {
                best = dist;
                jb = j;
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
        }
        __syncthreads();  // x / s_best reused by the next point
    }
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
    size_t off[5];
    return tc_ws_layout(n_prob, sum_k, sum_n, d, nullptr, off);
}

// one assignment pass on the tensor cores (used by mpa_km_lloyd when km->tc_ws is given)
int mpa_km_assign_tc(const mpa_km& k, cudaStream_t st) {
    size_t off[5];
    int kpad = 0;
    const size_t need = tc_ws_layout(k.n_prob, k.sum_k, k.sum_n, k.d, &kpad, off);
    MPA_REQUIRE(k.tc_ws && (size_t)k.tc_ws_bytes >= need, MPA_ERR_ARG, "mpa_km: tensor-core workspace %lld < %zu",
                (long long)k.tc_ws_bytes, need);
    char* base = (char*)k.tc_ws;
    TcWs ws{(__nv_bfloat16*)(base + off[0]), (float*)(base + off[1]), (double*)(base + off[2]),
            (int32_t*)(base + off[3]), (int32_t*)(base + off[4]), kpad};
    CUtensorMap tp, tt, tt_tail;
    if (int rc = encode_rows_map(&tp, k.pts, (long long)k.pts_rows, k.d, kTcM)) return rc;
    if (int rc = encode_rows_map(&tt, ws.terms, 3ll * kpad, k.d, kTcN)) return rc;
    if (int rc = encode_rows_map(&tt_tail, ws.terms, 3ll * kpad, k.d, kTcTailRows)) return rc;
    km_tc_norms_kernel<<<k.n_prob, 256, 0, st>>>(k, ws);
    km_tc_prep_kernel<<<dim3(ceil_div(k.k_max * k.d, 256 * 8), k.n_prob), 256, 0, st>>>(k, ws);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(km_assign_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
        attr = true;
    }
    static int oneshot = -1;  // MPA_KM_TC_ONESHOT=1: one CTA per tile (previous kernel)
    if (oneshot < 0) {
        const char* e = getenv("MPA_KM_TC_ONESHOT");
        oneshot = (e && e[0] == '1') ? 1 : 0;
    }
    const size_t psmem = kTcpSmemFixed + (size_t)(k.n_prob + 1) * 4;
    static int paired = -1;  // MPA_KM_TC_PAIRED=0: single-tile persistent kernel
    if (paired < 0) {
        const char* e = getenv("MPA_KM_TC_PAIRED");
        paired = (e && e[0] == '0') ? 0 : 1;
    }
    const size_t psmem2 = kTc2SmemFixed + (size_t)((k.n_prob + 1 + 3) & ~3) * 4 + 2 * (size_t)((k.k_max + 31) & ~31) * 4;
    constexpr size_t kSmemCap = 227 * 1024 - 2048;  // leaves room for the kernels' static shared memory
    if (!oneshot && paired && psmem2 <= kSmemCap) {
        static int sms2 = 0;
        if (!sms2) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms2, cudaDevAttrMultiProcessorCount, dev);
            if (sms2 <= 0) sms2 = 148;
        }
        cudaFuncSetAttribute(km_assign_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem2);
        km_assign_tc2_kernel<<<sms2, kTcThreads, psmem2, st>>>(tp, tt, tt_tail, k, ws);
    } else if (!oneshot && psmem <= kSmemCap) {
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (sms <= 0) sms = 148;
        }
        cudaFuncSetAttribute(km_assign_tcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
        km_assign_tcp_kernel<<<sms, kTcThreads, psmem, st>>>(tp, tt, tt_tail, k, ws);
    } else {
        km_assign_tc_kernel<<<dim3(ceil_div(k.n_max, kTcM), k.n_prob), kTcThreads, kTcSmem, st>>>(tp, tt, tt_tail, k,
                                                                                                  ws);
    }
    km_recheck_kernel<<<4 * 148, kRecheckThreads, 0, st>>>(k, ws);
    return check_launch("mpa_km_assign(tcgen05)");
}
