// K9 / K10 serving kernels: fp64 centroid logits with q held in registers, and a fused
// Eq. 1 score + size-weighted radix select + work-list builder, one CTA per ledger.
//
// Reference (pkg/src/multipole_attn/attention.py):
//   :267-290 `_scores_per_group`  logits = Q_lk Kc^T / sqrt(d); e = exp(l - max_g);
//                                  score = mean_g e / (e . N)
//   :192-207 `select_clusters`    visit by (score desc, ref asc); take while cum < B
//   :331-334 hierarchical union denominator (extras = rejected coarse clusters)
//   :469-496 work of one kv-head: sinks, buffer, members of the selected clusters, rejected
//            centroids with their reused logits + ln N
//
// Numerics are the reference's: fp64 logits, exps, normalisers and scores, so the selected
// set matches the oracle except at true ties (|score gap| ~ 1e-16 relative); ties in score are
// broken by the lowest cluster id, exactly like the reference's (score, ref) sort.
#include <cstdlib>

#include "mpa_common.cuh"
#include "mpa_tc.cuh"

namespace mpa {

#ifdef MPA_DEBUG_TRACE
__device__ unsigned long long g_dbg_lk[4096 * 8];
__device__ __forceinline__ void dbg_lk(int slot) {
    if (threadIdx.x == 0 && blockIdx.x < 4096) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_dbg_lk[blockIdx.x * 8 + slot] = t;
    }
}
#else
__device__ __forceinline__ void dbg_lk(int) {}
#endif

// ============================================================================
// K9: logits[l, g, i] = q_lk[l, g] . kc[l, id_i] / sqrt(D), fp64, for bf16 centroids.
//
// Persistent CTAs (128 threads, 2 per SM) walk the (ledger, 128-candidate chunk) items with a
// double-buffered cp.async ring: the next item's 128 bf16 rows and q_lk land in smem while the
// current item computes.  Thread t computes a 4-row x G-head block over one quarter of the
// dimensions (each q load feeds 4 rows, each row element G heads), then the four quarter lanes
// combine their 16 partial sums with a 2-level transpose-reduce.  Per item the CTA also emits
// the chunk partials (m_c, Z_c = sum N e^(l - m_c)) and e_local = e^(l - m_c).
constexpr int kLgChunk = 128;
constexpr int kLgThreads = 128;

// exact bf16 -> fp64 with integer ops (F2F.F64.F32 issues at a fraction of the DFMA rate):
// fbits = the bf16 widened to fp32 bits; normal -> (sign, exp + 896, mantissa >> 3) in the high
// word, low word 0 (a bf16 mantissa has 7 bits); +-0 -> signed zero.  bf16 subnormals (< 1e-38)
// would flush to zero; centroid means of normalised keys never are.
__device__ __forceinline__ double bf16_bits_to_f64(unsigned fbits) {
    const unsigned mag = fbits & 0x7fffffffu;
    const unsigned hi = (fbits & 0x80000000u) | (mag ? (mag >> 3) + 0x38000000u : 0u);
    return __hiloint2double((int)hi, 0);
}

template <int G, int D>
struct LgGeom {
    // bf16 row with a 16 B gap after each quarter (+16 B): the 8 lanes of an LDS.128 phase
    // (2 row groups x 4 quarters) hit 8 distinct 16-byte bank groups
    static constexpr int kRowB = D * 2 + 4 * 16 + 16;
    static constexpr int kQD = D / 4;                        // dims per quarter
    static constexpr int kQStride = kQD * G + 2;             // doubles per quarter (+16 B pad)
    static constexpr int kTileB = kLgChunk * kRowB;
    static constexpr int kQB = 4 * kQStride * 8;
    static constexpr size_t smem(int nb) { return nb * (size_t)(kTileB + kQB) + sizeof(double) * G * kLgChunk; }
};

template <int G, int D, int NB>
__global__ void __launch_bounds__(kLgThreads, NB == 1 ? 4 : 2)
logits_block_kernel(const double* __restrict__ q_lk, const __nv_bfloat16* __restrict__ kc, int kcap,
                    const int32_t* __restrict__ count, const int32_t* __restrict__ lv_size,
                    const int32_t* __restrict__ cand, const int32_t* __restrict__ n_cand, int cand_cap,
                    double* __restrict__ logits, double* __restrict__ cstats, double* __restrict__ e_local,
                    int n_chunks, int n_items_chunks, int L) {
    using Geo = LgGeom<G, D>;
    constexpr int CPR = D / 8;  // 16-byte chunks per row
    extern __shared__ __align__(16) unsigned char sm[];
    double* slg = reinterpret_cast<double*>(sm + NB * (Geo::kTileB + Geo::kQB));  // [G][kLgChunk]
    __shared__ double red[kLgThreads / 32][G];
    __shared__ double s_m[G];
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const int items = L * n_items_chunks;
    // q smem layout per quarter: [dim pair][g][2] so that one 16-byte cp.async moves 2 dims of a head
    auto issue = [&](int it, int buf) {
        const int l = it / n_items_chunks, chunk = it - l * n_items_chunks;
        const int n = cand ? n_cand[l] : count[l];
        const int i0 = chunk * kLgChunk;
        unsigned char* tile = sm + buf * (Geo::kTileB + Geo::kQB);
        double* qs = reinterpret_cast<double*>(tile + Geo::kTileB);
        if (i0 < n) {
            const int nv = min(kLgChunk, n - i0);
            for (int j = tid; j < kLgChunk * CPR; j += kLgThreads) {
                const int r = j / CPR, cch = j - r * CPR;
                const bool ok = r < nv;
                const int row = ok ? (cand ? __ldg(cand + (size_t)l * cand_cap + i0 + r) : i0 + r) : 0;
                const unsigned dst =
                    (unsigned)__cvta_generic_to_shared(tile + r * Geo::kRowB + cch * 16 + (cch / (CPR / 4)) * 16);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst),
                             "l"(kc + ((size_t)l * kcap + row) * D + cch * 8), "r"(ok ? 16 : 0));
            }
            for (int j = tid; j < G * D / 2; j += kLgThreads) {
                const int g = j / (D / 2), dp = j - g * (D / 2), k = dp * 2;
                const int qt = k / Geo::kQD, kk = k % Geo::kQD;
                const unsigned dst = (unsigned)__cvta_generic_to_shared(qs + qt * Geo::kQStride + (kk / 2) * 2 * G + g * 2);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst),
                             "l"(q_lk + ((size_t)l * G + g) * D + k));
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    const int qt = tid & 3, rg = tid >> 2;  // quarter, 4-row group
    const bool hi2 = qt & 2, hi1 = qt & 1;
    constexpr int GH = (G + 1) / 2;  // heads kept by the lower lane of the xor-1 pair
    const double sq = sqrt((double)D);  // logits divide like the reference (acc / sqrt(d))
    int k = 0;
    if (blockIdx.x < items) issue(blockIdx.x, 0);
#pragma unroll 1
    for (int it = blockIdx.x; it < items; it += gridDim.x, ++k) {
        const int buf = NB == 1 ? 0 : (k & 1);
        if (NB > 1 && it + (int)gridDim.x < items) issue(it + gridDim.x, buf ^ 1);
        else asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 1;\n" ::);
        __syncthreads();
        const int l = it / n_items_chunks, chunk = it - l * n_items_chunks;
        const int n = cand ? n_cand[l] : count[l];
        const int i0 = chunk * kLgChunk;
        if (i0 >= n) {
            if (cstats && chunk < n_chunks && tid < G) {
                cstats[(((size_t)l * n_chunks + chunk) * G + tid) * 2] = -INFINITY;
                cstats[(((size_t)l * n_chunks + chunk) * G + tid) * 2 + 1] = 0.0;
            }
            __syncthreads();
            continue;
        }
        const int nv = min(kLgChunk, n - i0);
        const unsigned char* tile = sm + buf * (Geo::kTileB + Geo::kQB);
        const double* qq = reinterpret_cast<const double*>(tile + Geo::kTileB) + qt * Geo::kQStride;
        double acc[4][G];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int g = 0; g < G; ++g) acc[r][g] = 0.0;
#pragma unroll 1
        for (int c = 0; c < Geo::kQD / 8; ++c) {
            uint4 raw[4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
                raw[r] = *reinterpret_cast<const uint4*>(tile + (rg * 4 + r) * Geo::kRowB + qt * (Geo::kQD * 2 + 16) +
                                                         c * 16);
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2) {
                // 2 dims x G heads of q: [g][2] pairs
                double qv[2][G];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double2 t = *reinterpret_cast<const double2*>(qq + ((c * 8 + 2 * e2) / 2) * 2 * G + g * 2);
                    qv[0][g] = t.x;
                    qv[1][g] = t.y;
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const unsigned wd = (&raw[r].x)[e2];
                    const double x0 = bf16_bits_to_f64(wd << 16), x1 = bf16_bits_to_f64(wd & 0xffff0000u);
#pragma unroll
                    for (int g = 0; g < G; ++g) acc[r][g] = fma(qv[0][g], x0, acc[r][g]);
#pragma unroll
                    for (int g = 0; g < G; ++g) acc[r][g] = fma(qv[1][g], x1, acc[r][g]);
                }
            }
        }
        // transpose-reduce over the 4 quarter lanes (xor 2 splits rows, xor 1 splits heads)
        double a2[2][G];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double send = hi2 ? acc[rr][g] : acc[rr + 2][g];
                const double keep = hi2 ? acc[rr + 2][g] : acc[rr][g];
                a2[rr][g] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
            }
        double a1[2][GH];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
            for (int j = 0; j < GH; ++j) {
                const int ghi = GH + j;
                const double lo = a2[rr][j], hv = ghi < G ? a2[rr][ghi < G ? ghi : 0] : 0.0;
                const double send = hi1 ? lo : hv;
                const double keep = hi1 ? hv : lo;
                a1[rr][j] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
            }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int r = rg * 4 + (hi2 ? 2 : 0) + rr;
#pragma unroll
            for (int j = 0; j < GH; ++j) {
                const int g = (hi1 ? GH : 0) + j;
                if (g < G) {
                    const double v = a1[rr][j] / sq;
                    slg[g * kLgChunk + r] = v;
                    if (r < nv) logits[((size_t)l * G + g) * cand_cap + i0 + r] = v;
                }
            }
        }
        if (cstats) {
            __syncthreads();
            // chunk partials: m_c = max l, Z_c = sum N e_local, e_local = e^(l - m_c)
            const int i = tid;  // one candidate per thread
            const bool valid = i < nv;
            const int id = valid ? (cand ? cand[(size_t)l * cand_cap + i0 + i] : i0 + i) : 0;
            const double nsz = valid ? (double)lv_size[(size_t)l * kcap + id] : 0.0;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double m = warp_max(valid ? slg[g * kLgChunk + i] : -INFINITY);
                if (lane == 0) red[w][g] = m;
            }
            __syncthreads();
            if (tid < G) {
                double M = -INFINITY;
                for (int ww = 0; ww < kLgThreads / 32; ++ww) M = fmax(M, red[ww][tid]);
                s_m[tid] = M;
            }
            __syncthreads();
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double e = valid ? exp(slg[g * kLgChunk + i] - s_m[g]) : 0.0;
                if (valid && e_local) e_local[((size_t)l * G + g) * cand_cap + i0 + i] = e;
                const double z = warp_sum(e * nsz);
                __syncwarp();
                if (lane == 0) red[w][g] = z;
            }
            __syncthreads();
            if (tid < G) {
                double Z = 0.0;
                for (int ww = 0; ww < kLgThreads / 32; ++ww) Z += red[ww][tid];
                cstats[(((size_t)l * n_chunks + chunk) * G + tid) * 2] = s_m[tid];
                cstats[(((size_t)l * n_chunks + chunk) * G + tid) * 2 + 1] = Z;
            }
        }
        __syncthreads();  // buffer `buf` is refilled by the next iteration's issue
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
}

// ---- TMA-fed variant (bf16, D = 128): the 128-row chunk lands in smem through 2 TMA tile
// copies (flat candidates, contiguous rows) or 64 tile::gather4 copies (candidate lists), 128B
// swizzled; no per-thread copy instructions.  Rows of thread (rg, qt) are rg + 32 r, and quarter
// qt visits its 4 chunks starting at 2 (qt >> 1) so the 8 lanes of an LDS.128 phase hit 8
// distinct bank groups.  bf16 -> fp64 by integer ops (exact for every nonzero bf16; a zero
// element becomes 2^-127, below the fp64 resolution of any logit sum).
__device__ __forceinline__ double bf16hi_to_f64(unsigned fbits) {  // fbits: bf16 in the high half
    return __hiloint2double((int)((((int)fbits >> 3) & 0x8FFFE000) + 0x38000000), 0);
}
// the same without the exponent re-bias: exactly x * 2^-896 (a normal fp64 for every bf16, zero
// included), so q . x accumulates the exact bits of q . x scaled by 2^-896 and one exact
// multiply by 2^896 at the end restores them -- one integer op less per element
__device__ __forceinline__ double bf16hi_to_f64_s896(unsigned fbits) {
    return __hiloint2double((int)(((int)fbits >> 3) & 0x8FFFE000), 0);
}
constexpr double kUnscale896 = 0x1p896;

template <int G>
__global__ void __launch_bounds__(kLgThreads)
logits_tma_kernel(const __grid_constant__ CUtensorMap tm_tile, const __grid_constant__ CUtensorMap tm_row,
                  const double* __restrict__ q_lk, int kcap, const int32_t* __restrict__ count,
                  const int32_t* __restrict__ lv_size, const int32_t* __restrict__ cand,
                  const int32_t* __restrict__ n_cand, int cand_cap, double* __restrict__ logits,
                  double* __restrict__ cstats, double* __restrict__ e_local, int n_chunks,
                  float* __restrict__ rej_w, int rej_cap, const float* __restrict__ q_raw,
                  const double* __restrict__ cs_lk) {
    constexpr int D = 128, QD = 32, QRow = QD + 2;
    // cs_lk != NULL: the lookup view q_lk = rotate(q_raw, delta) is formed here from the fp32 query
    // and the (cos, sin) table of delta * inv_freq (rope.py:66-68), instead of read from q_lk  // q slot: 32 dims (+16 B pad) per (head, quarter)
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* tile = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);  // [2 halves][128][128 B]
    double* qs = reinterpret_cast<double*>(tile + 2 * kLgChunk * 128);          // [G][4][QRow]
    double* slg = qs + G * 4 * QRow;                                            // [G][128]
    __shared__ __align__(8) uint64_t bar;
    __shared__ double red[kLgThreads / 32][G];
    __shared__ double s_m[G];
    const int l = blockIdx.y, chunk = blockIdx.x, tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    // PDL: q_lk (and, for candidate lists, cand / n_cand) come from the stream predecessor; the
    // flat path streams its centroid rows before waiting for it
    if (cand) pdl_wait();
    const int n = cand ? n_cand[l] : count[l];
    const int i0 = chunk * kLgChunk;
    if (i0 >= n) {
        if (!cand) pdl_wait();
        pdl_trigger();
        if (cstats && chunk < n_chunks && tid < G) {
            cstats[(((size_t)l * n_chunks + chunk) * G + tid) * 2] = -INFINITY;
            cstats[(((size_t)l * n_chunks + chunk) * G + tid) * 2 + 1] = 0.0;
        }
        return;
    }
    const int nv = min(kLgChunk, n - i0);
    // epilogue inputs of this thread's candidate, loaded now so the latency hides under the tile
    const bool valid = tid < nv;
    const int id = valid ? (cand ? __ldg(cand + (size_t)l * cand_cap + i0 + tid) : i0 + tid) : 0;
    const int isz = valid && cstats ? __ldg(lv_size + (size_t)l * kcap + id) : 0;
    if (tid == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid < 32) {
        if (tid == 0) {
            // one expect_tx (a single arrive) for everything this barrier phase receives
            mbar_expect_tx(smem_u32(&bar), (cs_lk ? 0 : G * 4 * QD * 8) + 2 * kLgChunk * 128);
            if (!cand) {  // centroid rows first: they do not depend on the predecessor
                const int row0 = l * kcap + i0;
                tma_load_2d(smem_u32(tile), &tm_tile, 0, row0, smem_u32(&bar));
                tma_load_2d(smem_u32(tile + kLgChunk * 128), &tm_tile, 64, row0, smem_u32(&bar));
            }
        }
        __syncwarp();
        // q_lk rows of the GQA group: one 256 B bulk copy per (head, quarter) into padded slots,
        // issued by G * 4 lanes at once (after the predecessor that writes q_lk is complete)
        if (!cs_lk && tid < G * 4) {
            pdl_wait();
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                    smem_u32(qs + tid * QRow)),
                "l"(q_lk + ((size_t)l * G + tid / 4) * D + (tid % 4) * QD), "r"(QD * 8), "r"(smem_u32(&bar))
                : "memory");
        }
        if (!cand) {
        } else {
            // lane j gathers rows 4j .. 4j+3 (rows past nv repeat the chunk's first candidate)
            int id[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int rr = 4 * tid + r;
                id[r] = l * kcap + __ldg(cand + (size_t)l * cand_cap + i0 + (rr < nv ? rr : 0));
            }
            __syncwarp();
            for (int h = 0; h < 2; ++h)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(tile + h * kLgChunk * 128 + tid * 512)),
                    "l"(reinterpret_cast<uint64_t>(&tm_row)), "r"(h * 64), "r"(id[0]), "r"(id[1]), "r"(id[2]),
                    "r"(id[3]), "r"(smem_u32(&bar))
                    : "memory");
        }
    }
    if (cs_lk) {
        // rotate the group's G query rows at delta straight into the padded q slots (the same
        // arithmetic as mpa_rotate_queries: x cos - y sin, x sin + y cos, no contraction)
        pdl_wait();
        double* qw = const_cast<double*>(qs);
        for (int e = tid; e < G * (D / 2); e += kLgThreads) {
            const int g = e / (D / 2), i = e - g * (D / 2), k = 2 * i;
            const float2 xy = *reinterpret_cast<const float2*>(q_raw + ((size_t)l * G + g) * D + k);
            const double x = (double)xy.x, y = (double)xy.y, c = cs_lk[2 * i], sn = cs_lk[2 * i + 1];
            double* slot = qw + (g * 4 + k / QD) * QRow + (k % QD);
            slot[0] = __dsub_rn(__dmul_rn(x, c), __dmul_rn(y, sn));
            slot[1] = __dadd_rn(__dmul_rn(x, sn), __dmul_rn(y, c));
        }
        __syncthreads();
    }
    mbar_wait(smem_u32(&bar), 0);
    pdl_trigger();  // after thread 0's wait (the barrier above completes only after it)

    const double sq = sqrt((double)D);
    const int qt = tid & 3, rg = tid >> 2;
    const double* qq = qs + qt * QRow;
    double acc[4][G];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int g = 0; g < G; ++g) acc[r][g] = 0.0;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        const int c = (cc + 2 * (qt >> 1)) & 3;  // this quarter's 16-byte chunk (8 dims)
        const int ch = (qt & 1) * 4 + c;         // chunk within the 64-column half
        uint4 raw[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int row = rg + 32 * r;
            raw[r] = *reinterpret_cast<const uint4*>(tile + (qt >> 1) * kLgChunk * 128 + row * 128 +
                                                     ((ch ^ (row & 7)) << 4));
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            double qv[G];
#pragma unroll
            for (int g = 0; g < G; ++g) qv[g] = qq[g * 4 * QRow + c * 8 + e];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const unsigned wd = (&raw[r].x)[e >> 1];
                const double x = bf16hi_to_f64_s896((e & 1) ? (wd & 0xffff0000u) : (wd << 16));
#pragma unroll
                for (int g = 0; g < G; ++g) acc[r][g] = fma(qv[g], x, acc[r][g]);
            }
        }
    }
    // transpose-reduce over the 4 quarter lanes (xor 2 splits rows, xor 1 splits heads)
    const bool hi2 = qt & 2, hi1 = qt & 1;
    constexpr int GH = (G + 1) / 2;
    double a2[2][G];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const double send = hi2 ? acc[rr][g] : acc[rr + 2][g];
            const double keep = hi2 ? acc[rr + 2][g] : acc[rr][g];
            a2[rr][g] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
    double a1[2][GH];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
        for (int j = 0; j < GH; ++j) {
            const int ghi = GH + j;
            const double lo = a2[rr][j], hv = ghi < G ? a2[rr][ghi < G ? ghi : 0] : 0.0;
            const double send = hi1 ? lo : hv;
            const double keep = hi1 ? hv : lo;
            a1[rr][j] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const int r = rg + 32 * ((hi2 ? 2 : 0) + rr);
#pragma unroll
        for (int j = 0; j < GH; ++j) {
            const int g = (hi1 ? GH : 0) + j;
            if (g < G) {
                const double v = (a1[rr][j] * kUnscale896) / sq;
                slg[g * kLgChunk + r] = v;
                if (logits && r < nv) logits[((size_t)l * G + g) * cand_cap + i0 + r] = v;
            }
        }
    }
    if (!cstats) return;
    __syncthreads();
    const int i = tid;
    const double nsz = (double)isz;
    if (rej_w && valid) {
        // replacement weights of every candidate, indexed by candidate (logit + ln N, the value
        // worklist_v2 would write for a rejected one); the selection masks the selected to -inf
        constexpr int GP = G <= 4 ? 4 : 8;
        const double lnN = (double)logf((float)isz);
        float wv[GP];
#pragma unroll
        for (int g = 0; g < GP; ++g) wv[g] = g < G ? (float)(slg[(g < G ? g : 0) * kLgChunk + i] + lnN) : 0.f;
        float4* dst = reinterpret_cast<float4*>(rej_w + ((size_t)l * rej_cap + i0 + i) * GP);
#pragma unroll
        for (int v = 0; v < GP / 4; ++v) dst[v] = make_float4(wv[4 * v], wv[4 * v + 1], wv[4 * v + 2], wv[4 * v + 3]);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const double m = warp_max(valid ? slg[g * kLgChunk + i] : -INFINITY);
        if (lane == 0) red[w][g] = m;
    }
    __syncthreads();
    if (tid < G) {
        double M = -INFINITY;
        for (int ww = 0; ww < kLgThreads / 32; ++ww) M = fmax(M, red[ww][tid]);
        s_m[tid] = M;
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const double e = valid ? exp(slg[g * kLgChunk + i] - s_m[g]) : 0.0;
        if (valid && e_local) e_local[((size_t)l * G + g) * cand_cap + i0 + i] = e;
        const double z = warp_sum(e * nsz);
        __syncwarp();
        if (lane == 0) red[w][g] = z;
    }
    __syncthreads();
    if (tid < G) {
        double Z = 0.0;
        for (int ww = 0; ww < kLgThreads / 32; ++ww) Z += red[ww][tid];
        cstats[(((size_t)l * n_chunks + chunk) * G + tid) * 2] = s_m[tid];
        cstats[(((size_t)l * n_chunks + chunk) * G + tid) * 2 + 1] = Z;
    }
}


// ============================================================================
// K10 + work list.  One CTA per ledger:
//   1. per-head max M_g and normaliser Z_g: from the logits kernel's chunk partials
//      (Z = sum_c Z_c e^(m_c - M), e = e_local e^(m_c - M)) or, without them, directly,
//   2. score_i = (sum_g e_gi / Z_g) / G, stored as the ascending key ~bits(score),
//   3. size-weighted radix select of the crossing candidate (key, id), 11-bit digits, most
//      significant first, stopping as soon as the crossing bin holds one candidate,
//   4. flags (smem + global), and the work lists: one block scan over thread-contiguous
//      candidate ranges, then all threads copy the selected clusters' members in parallel.
constexpr int kSel2Threads = 512;
constexpr int kDigBits = 11, kBins = 1 << kDigBits;

// 64-bit exclusive block scan (blockDim.x <= 1024); scratch: 33 entries
__device__ __forceinline__ unsigned long long block_scan_u64(unsigned long long v, unsigned long long* scratch,
                                                            unsigned long long* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) scratch[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        unsigned long long s = lane < nw ? scratch[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) scratch[lane] = s;
        if (lane == 31) scratch[32] = s;
    }
    __syncthreads();
    const unsigned long long base = wid ? scratch[wid - 1] : 0ull;
    *total = scratch[32];
    __syncthreads();
    return base + incl - v;
}

// ---- sequence sharding (a ledger's blocks spread over ranks): global normalisers, the
// cross-rank crossing candidate, and each rank's candidates that can be globally selected
struct Cross {
    unsigned long long k;  // ~bits(score) of the crossing candidate; 0 = select none, ~0 = select all
    unsigned int i;        // its global cluster id (tie-break)
    unsigned int pad;
};
struct PrefixEntry {
    unsigned long long key;
    unsigned int gid;
    int size;
};
struct ShardCtl {
    const double* mz = nullptr;        // [L, G, 2] global (M, Z)
    const Cross* cross = nullptr;      // [L] global crossing candidate (final pass)
    PrefixEntry* prefix = nullptr;     // [L, prefix_cap] local pass output
    int32_t* prefix_n = nullptr;       // [L] (zeroed by the caller)
    int prefix_cap = 0;
    const int32_t* gid_off = nullptr;  // [L] global id of this rank's first candidate
};

// Crossing candidate of a size-weighted "take while cum < B" over n entries visited by
// (key asc, id asc): the smallest (key, id) whose cumulative weight reaches B.  11-bit digits
// over the 63 low key bits (the top bit is constant for non-negative scores) then the id; stops
// as soon as the crossing bin holds one entry.  Requires 0 < B <= total weight.  Block-wide.
template <typename IdFn>
__device__ void radix_cross(const unsigned long long* keys, const int* sizes, IdFn id_of, int n, long long B,
                            unsigned long long& kstar, unsigned int& istar) {
    __shared__ unsigned int hist_w[kBins], hist_c[kBins];
    __shared__ unsigned long long s_kprefix, s_scan[33];
    __shared__ unsigned int s_iprefix;
    __shared__ long long s_below;
    __shared__ int s_cnt;
    __shared__ unsigned long long s_k;
    __shared__ unsigned int s_i;
    unsigned long long kmask = 1ull << 63;
    if (threadIdx.x == 0) {
        s_kprefix = keys[0] & (1ull << 63);
        s_iprefix = 0u;
        s_below = 0;
        s_cnt = 0;
    }
    __syncthreads();
    unsigned int imask = 0u;
    constexpr int kKeyPasses = (63 + kDigBits - 1) / kDigBits, kIdPasses = (32 + kDigBits - 1) / kDigBits;
    bool found = false;
    for (int pass = 0; pass < kKeyPasses + kIdPasses && !found; ++pass) {
        const bool kp_pass = pass < kKeyPasses;
        const int top = kp_pass ? 63 - kDigBits * pass : 32 - kDigBits * (pass - kKeyPasses);
        const int width = top >= kDigBits ? kDigBits : top;
        const int sh = top - width;
        const unsigned dmask = (1u << width) - 1u;
        for (int j = threadIdx.x; j < kBins; j += blockDim.x) hist_w[j] = hist_c[j] = 0u;
        __syncthreads();
        const unsigned long long kp = s_kprefix;
        const unsigned int ip = s_iprefix;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned long long k = keys[i];
            if ((k & kmask) != kp) continue;
            const unsigned int id = id_of(i);
            if ((id & imask) != ip) continue;
            const unsigned dg = kp_pass ? (unsigned)(k >> sh) & dmask : (id >> sh) & dmask;
            atomicAdd(&hist_w[dg], (unsigned)sizes[i]);
            atomicAdd(&hist_c[dg], 1u);
        }
        __syncthreads();
        const int bpt = kBins / blockDim.x;
        unsigned long long wsum = 0;
        for (int j = 0; j < bpt; ++j) wsum += hist_w[threadIdx.x * bpt + j];
        // every thread reads s_below before the scan's barriers; the owner rewrites it after them
        const long long below = s_below;
        const long long need = B - below;  // > 0
        unsigned long long btot;
        const unsigned long long before = block_scan_u64(wsum, s_scan, &btot);
        if ((long long)before < need && (long long)(before + wsum) >= need) {
            long long run = (long long)before;
            int dg = threadIdx.x * bpt + bpt - 1;
            for (int j = 0; j < bpt; ++j) {
                const int b = threadIdx.x * bpt + j;
                if (run + (long long)hist_w[b] >= need) {
                    dg = b;
                    break;
                }
                run += hist_w[b];
            }
            s_below = below + run;
            s_cnt = (int)hist_c[dg];
            if (kp_pass) s_kprefix = kp | ((unsigned long long)dg << sh);
            else s_iprefix = ip | ((unsigned)dg << sh);
        }
        __syncthreads();
        if (kp_pass) kmask |= (unsigned long long)dmask << sh;
        else imask |= dmask << sh;
        found = s_cnt == 1;
    }
    const unsigned long long kp = s_kprefix;
    const unsigned int ip = s_iprefix;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned int id = id_of(i);
        if ((keys[i] & kmask) == kp && (id & imask) == ip) {
            s_k = keys[i];
            s_i = id;
        }
    }
    __syncthreads();
    kstar = s_k;
    istar = s_i;
    __syncthreads();
}

// smem per candidate: key (8) + size (4) + member offset (4) + flag (1) + pad
__host__ __device__ constexpr size_t sel_smem_bytes(int n_max) { return (size_t)n_max * 17 + 64; }

template <int G>
__device__ void select_v2_core(int l, const double* __restrict__ logits, const double* __restrict__ e_local,
                               const int32_t* __restrict__ cand, int n, int cand_cap,
                               const int32_t* __restrict__ lv_size, int lv_cap, const double* __restrict__ elogits,
                               const int32_t* __restrict__ esize, const uint8_t* __restrict__ eflag, int ne, int ecap,
                               long long B, const double* __restrict__ cstats, int n_chunks, unsigned long long* keys,
                               int* sizes, uint8_t* sflag, uint8_t* __restrict__ flag,
                               int32_t* __restrict__ sel_tokens, const ShardCtl& sh = ShardCtl{},
                               const int32_t* __restrict__ moff = nullptr, int* offs = nullptr) {
    // moff / offs (work-list builds): the candidates' member-CSR offsets, staged into smem here
    // with the other per-candidate loads so the member copy makes one dependent load, not two
    const double* mz_ext = sh.mz;
    const Cross* ext_cross = sh.cross;
    PrefixEntry* prefix = sh.prefix;
    int32_t* prefix_n = sh.prefix_n;
    const int prefix_cap = sh.prefix_cap;
    const int gid_off = sh.gid_off ? sh.gid_off[l] : 0;
    __shared__ double s_red[kSel2Threads / 32][G];
    __shared__ double s_mx[G], s_z[G];
    __shared__ double csc[2048];  // chunk scales e^(m_c - M) [n_chunks][G]
    __shared__ unsigned long long s_scan[33];
    __shared__ long long s_total;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double* lg = logits + (size_t)l * G * cand_cap;
    const double* el = e_local ? e_local + (size_t)l * G * cand_cap : nullptr;
    const double* elg = elogits ? elogits + (size_t)l * G * ecap : nullptr;
    const double* cs = cstats ? cstats + (size_t)l * n_chunks * G * 2 : nullptr;
    const bool use_local = el && cs;
    const int nchu = min(n_chunks, (n + 127) >> 7);  // chunks holding this ledger's candidates
    const int max_sc_chunks = 2048 / G;

    // ---- 0. this thread's first kPF candidates: sizes and e_local loads issued together up
    // front, so their latency overlaps the normaliser phases (thread-strided like every loop here)
    constexpr int kPF = 5;
    int szr[kPF], ofr[kPF];
    double elr[kPF][G];
#pragma unroll
    for (int u = 0; u < kPF; ++u) {
        const int i = threadIdx.x + u * blockDim.x;
        szr[u] = ofr[u] = 0;
        if (i < n) {
            const int id = cand ? __ldg(cand + (size_t)l * cand_cap + i) : i;
            szr[u] = __ldg(lv_size + (size_t)l * lv_cap + id);
            if (offs) ofr[u] = __ldg(moff + (size_t)l * (lv_cap + 1) + id);
        }
    }
    // PDL: everything below may read the logits kernel's outputs (ledger state above is older)
    pdl_wait();
    pdl_trigger();
#pragma unroll
    for (int u = 0; u < kPF; ++u) {
        const int i = threadIdx.x + u * blockDim.x;
#pragma unroll
        for (int g = 0; g < G; ++g) elr[u][g] = 0.0;
        if (i < n && use_local)
#pragma unroll
            for (int g = 0; g < G; ++g) elr[u][g] = __ldcg(el + (size_t)g * cand_cap + i);
    }
    // ---- 1. sizes, per-head max
    long long tot_local = 0;
#pragma unroll
    for (int u = 0; u < kPF; ++u) {
        const int i = threadIdx.x + u * blockDim.x;
        if (i < n) {
            sizes[i] = szr[u];
            if (offs) offs[i] = ofr[u];
            tot_local += szr[u];
        }
    }
    for (int i = threadIdx.x + kPF * blockDim.x; i < n; i += blockDim.x) {
        const int id = cand ? __ldg(cand + (size_t)l * cand_cap + i) : i;
        const int sz = __ldg(lv_size + (size_t)l * lv_cap + id);
        sizes[i] = sz;
        if (offs) offs[i] = __ldg(moff + (size_t)l * (lv_cap + 1) + id);
        tot_local += sz;
    }
    {
        double m[G];
#pragma unroll
        for (int g = 0; g < G; ++g) m[g] = -INFINITY;
        if (cs) {
            for (int c = threadIdx.x; c < nchu; c += blockDim.x)
#pragma unroll
                for (int g = 0; g < G; ++g) m[g] = fmax(m[g], cs[(c * G + g) * 2]);
        } else {
            for (int i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
                for (int g = 0; g < G; ++g) m[g] = fmax(m[g], lg[(size_t)g * cand_cap + i]);
        }
        for (int j = threadIdx.x; j < ne; j += blockDim.x)
            if (!eflag[(size_t)l * ecap + j])
#pragma unroll
                for (int g = 0; g < G; ++g) m[g] = fmax(m[g], elg[(size_t)g * ecap + j]);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const double r = warp_max(m[g]);
            if (lane == 0) s_red[w][g] = r;
        }
        __syncthreads();
        if (threadIdx.x < G) {
            double r = -INFINITY;
            for (int ww = 0; ww < kSel2Threads / 32; ++ww) r = fmax(r, s_red[ww][threadIdx.x]);
            s_mx[threadIdx.x] = r;
        }
        __syncthreads();
    }
    dbg_lk(1);
    if (mz_ext) {  // global (M, Z) of a sequence-sharded ledger
        __syncthreads();
        if (threadIdx.x < G) s_mx[threadIdx.x] = mz_ext[((size_t)l * G + threadIdx.x) * 2];
        __syncthreads();
    }
    double mx[G];
#pragma unroll
    for (int g = 0; g < G; ++g) mx[g] = s_mx[g];
    const bool scaled = use_local && nchu <= max_sc_chunks;

    // ---- 2. Z = e . N (+ live extras)
    {
        double z[G];
#pragma unroll
        for (int g = 0; g < G; ++g) z[g] = 0.0;
        if (scaled) {
            for (int c = threadIdx.x; c < nchu; c += blockDim.x)
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double cm = cs[(c * G + g) * 2];
                    const double sc = cm == -INFINITY ? 0.0 : exp(cm - mx[g]);
                    csc[c * G + g] = sc;
                    z[g] = fma(cs[(c * G + g) * 2 + 1], sc, z[g]);
                }
        } else {
            for (int i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
                for (int g = 0; g < G; ++g)
                    z[g] = fma(exp(lg[(size_t)g * cand_cap + i] - mx[g]), (double)sizes[i], z[g]);
        }
        for (int j = threadIdx.x; j < ne; j += blockDim.x)
            if (!eflag[(size_t)l * ecap + j])
#pragma unroll
                for (int g = 0; g < G; ++g)
                    z[g] = fma(exp(elg[(size_t)g * ecap + j] - mx[g]), (double)esize[(size_t)l * ecap + j], z[g]);
        unsigned long long tl = (unsigned long long)tot_local;
#pragma unroll
        for (int o = 16; o; o >>= 1) tl += __shfl_xor_sync(0xffffffffu, tl, o);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const double r = warp_sum(z[g]);
            if (lane == 0) s_red[w][g] = r;
        }
        if (lane == 0) s_scan[w] = tl;
        __syncthreads();
        if (threadIdx.x < G) {
            double r = 0.0;
            for (int ww = 0; ww < kSel2Threads / 32; ++ww) r += s_red[ww][threadIdx.x];
            s_z[threadIdx.x] = mz_ext ? mz_ext[((size_t)l * G + threadIdx.x) * 2 + 1] : r;
        }
        if (threadIdx.x == 32) {
            unsigned long long t = 0;
            for (int ww = 0; ww < kSel2Threads / 32; ++ww) t += s_scan[ww];
            s_total = (long long)t;
        }
        __syncthreads();
    }

    dbg_lk(2);
    // ---- 3. scores -> keys: mean over heads of e / Z, accumulated in head order like np.mean(axis=0)
    double zz[G];
#pragma unroll
    for (int g = 0; g < G; ++g) zz[g] = s_z[g];
    auto score_key = [&](int i, const double* elv) {
        double sc = 0.0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const double e = scaled ? (elv ? elv[g] : el[(size_t)g * cand_cap + i]) * csc[(i >> 7) * G + g]
                                    : exp(lg[(size_t)g * cand_cap + i] - mx[g]);
            sc = g ? sc + e / zz[g] : e / zz[g];
        }
        sc = sc / (double)G;
        keys[i] = ~(unsigned long long)__double_as_longlong(sc);  // ascending key == descending score
    };
#pragma unroll
    for (int u = 0; u < kPF; ++u) {
        const int i = threadIdx.x + u * blockDim.x;
        if (i < n) score_key(i, elr[u]);
    }
    for (int i = threadIdx.x + kPF * blockDim.x; i < n; i += blockDim.x) score_key(i, nullptr);
    __syncthreads();

    dbg_lk(5);
    // ---- 4. crossing candidate: smallest (key, id) with W(<=) >= B (or given by the caller:
    // the cross-rank cut of a sequence-sharded ledger)
    const long long total = s_total;
    const bool select_none = ext_cross ? ext_cross[l].k == 0ull : B <= 0;
    const bool select_all = ext_cross ? ext_cross[l].k == ~0ull : total < B;
    unsigned long long kstar = ~0ull;
    unsigned int istar = 0xffffffffu;
    if (ext_cross) {
        kstar = ext_cross[l].k;
        istar = ext_cross[l].i;
    } else if (!select_none && !select_all) {
        radix_cross(keys, sizes, [&](int i) -> unsigned {
            return (unsigned)gid_off + (cand ? (unsigned)__ldg(cand + (size_t)l * cand_cap + i) : (unsigned)i);
        }, n, B, kstar, istar);
    }

    dbg_lk(6);
    // ---- 5. flags
    long long tok = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        bool sel;
        if (select_none) sel = false;
        else if (select_all) sel = true;
        else {
            const unsigned int id =
                (unsigned)gid_off + (cand ? (unsigned)__ldg(cand + (size_t)l * cand_cap + i) : (unsigned)i);
            sel = keys[i] < kstar || (keys[i] == kstar && id <= istar);
        }
        sflag[i] = sel ? 1 : 0;
        if (sel && prefix) {  // sharded local pass: this rank's candidates that can be globally selected
            const int q = atomicAdd(prefix_n + l, 1);
            if (q < prefix_cap) {
                prefix[(size_t)l * prefix_cap + q] = PrefixEntry{
                    keys[i], (unsigned)gid_off + (cand ? (unsigned)__ldg(cand + (size_t)l * cand_cap + i) : (unsigned)i),
                    sizes[i]};
            }
        }
        flag[(size_t)l * cand_cap + i] = sel ? 1 : 0;
        if (sel) tok += sizes[i];
    }
    {
        unsigned long long t = (unsigned long long)tok;
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) s_scan[w] = t;
        __syncthreads();
        if (threadIdx.x == 0 && sel_tokens) {
            unsigned long long a = 0;
            for (int ww = 0; ww < kSel2Threads / 32; ++ww) a += s_scan[ww];
            sel_tokens[l] = (int32_t)a;
        }
    }
    __syncthreads();
}

// Work lists of one ledger (attention.py:469-496) from the selection flags: sinks, buffer and the
// members of the selected candidates; rejected fine candidates (then coarse clusters with
// cflag == 0, hierarchy) as value-row codes with logit + ln N; stats [4, L].  keys_space is the
// select's key array, reused for the selected-candidate list.
template <int G>
__device__ void worklist_v2(int l, int L, int n, const double* __restrict__ logits, const int32_t* __restrict__ cand,
                            int cand_cap, const uint8_t* sflag, const int* sizes, int* sel_list,
                            const int32_t* __restrict__ fmem_off, const int32_t* __restrict__ fmem, int fcap,
                            int fmem_cap, const int* offs, const int32_t* __restrict__ csize, int ne, int ccap,
                            const uint8_t* __restrict__ cflag, const double* __restrict__ clogits,
                            const int32_t* __restrict__ sink_end, const int32_t* __restrict__ buffer_start,
                            const int32_t* __restrict__ cache_len, int n_kv_heads, int replacement,
                            int32_t* __restrict__ tok, int tok_cap, int32_t* __restrict__ rej,
                            float* __restrict__ rej_w, int rej_cap, int32_t* __restrict__ stats) {
    constexpr int GP = G <= 4 ? 4 : 8;
    __shared__ unsigned long long scan64[33];
    const int seq = l / n_kv_heads;
    const int clen = cache_len[seq];
    const int ns = min(sink_end[seq], clen);
    const int bs = buffer_start[seq];
    const int nb = max(0, clen - bs);
    int32_t* T = tok + (size_t)l * tok_cap;
    for (int j = threadIdx.x; j < ns; j += blockDim.x) T[j] = j;
    for (int j = threadIdx.x; j < nb; j += blockDim.x) T[ns + j] = bs + j;
    // thread-contiguous candidate ranges: one scan of (tokens, rejected, selected) packed 32/16/16
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int c0 = min(n, (int)threadIdx.x * per), c1 = min(n, c0 + per);
    unsigned long long mine = 0;
    for (int i = c0; i < c1; ++i) {
        if (sflag[i]) mine += ((unsigned long long)sizes[i] << 32) | 1ull;
        else if (replacement) mine += 1ull << 16;
    }
    unsigned long long tot;
    const unsigned long long pre = block_scan_u64(mine, scan64, &tot);
    int tpos = (int)(pre >> 32), rpos = (int)((pre >> 16) & 0xffff), spos = (int)(pre & 0xffff);
    const int nsel = (int)(tot & 0xffff);
    // selected list (candidate, first token slot) for the parallel member copy; rejected weights
    int* sel_c = sel_list;
    int* sel_t = sel_list + n;
    for (int i = c0; i < c1; ++i) {
        const int sz = sizes[i];
        if (sflag[i]) {
            sel_c[spos] = i;
            sel_t[spos] = tpos;
            ++spos;
            tpos += sz;
            if (replacement && !rej) {  // contiguous-centroid list: mask the selected candidate
#pragma unroll
                for (int g = 0; g < G; ++g) rej_w[((size_t)l * rej_cap + i) * GP + g] = -INFINITY;
            }
        } else if (replacement) {
            if (rej && rpos < rej_cap) {
                const int id = cand ? __ldg(cand + (size_t)l * cand_cap + i) : i;
                rej[(size_t)l * rej_cap + rpos] = id;
                const double lnN = (double)logf((float)sz);
#pragma unroll
                for (int g = 0; g < G; ++g)
                    rej_w[((size_t)l * rej_cap + rpos) * GP + g] =
                        (float)(logits[((size_t)l * G + g) * cand_cap + i] + lnN);
            }
            ++rpos;
        }
    }
    __syncthreads();
    // members of the selected clusters: one thread per token slot (binary search of its cluster
    // in the selected list), so the two dependent loads (CSR offset, member id) overlap across slots
    const int32_t* moff = fmem_off + (size_t)l * (fcap + 1);
    const int nsel_tok = (int)(tot >> 32);
    constexpr int kTokU = 4;  // slots resolved first, then their member loads issued together
    for (int j0 = threadIdx.x; j0 < nsel_tok; j0 += blockDim.x * kTokU) {
        int src[kTokU];
#pragma unroll
        for (int u = 0; u < kTokU; ++u) {
            const int j = j0 + u * blockDim.x;
            src[u] = -1;
            if (j < nsel_tok) {
                int lo = 0, hi = nsel - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (sel_t[mid] <= j) lo = mid;
                    else hi = mid - 1;
                }
                src[u] = offs[sel_c[lo]] + (j - sel_t[lo]);
            }
        }
        int v[kTokU];
#pragma unroll
        for (int u = 0; u < kTokU; ++u) v[u] = src[u] >= 0 ? __ldg(fmem + (size_t)l * fmem_cap + src[u]) : 0;
#pragma unroll
        for (int u = 0; u < kTokU; ++u) {
            const int slot = ns + nb + j0 + u * (int)blockDim.x;
            if (src[u] >= 0 && slot < tok_cap) T[slot] = v[u];
        }
    }
    int tbase = ns + nb + (int)(tot >> 32), rbase = (int)((tot >> 16) & 0xffff);
    if (cflag && replacement) {
        __shared__ int scan[33];
        for (int c = threadIdx.x, cbase = 0; cbase < ne; c += blockDim.x, cbase += blockDim.x) {
            const int r = (c < ne && !cflag[(size_t)l * ccap + c]) ? 1 : 0;
            int rtot;
            const int p = rbase + block_exclusive_scan(r, scan, &rtot);
            if (r && p < rej_cap) {
                rej[(size_t)l * rej_cap + p] = -1 - c;
                const double lnN = (double)logf((float)csize[(size_t)l * ccap + c]);
#pragma unroll
                for (int g = 0; g < G; ++g)
                    rej_w[((size_t)l * rej_cap + p) * GP + g] = (float)(clogits[((size_t)l * G + g) * ccap + c] + lnN);
            }
            rbase += rtot;
        }
    }
    if (threadIdx.x == 0) {
        stats[l] = min(tbase, tok_cap);
        stats[L + l] = min(rbase, rej_cap);
        stats[2 * L + l] = tbase - ns - nb;
        stats[3 * L + l] = nsel;
    }
}

template <int G>
__global__ void __launch_bounds__(kSel2Threads)
select_worklist_v2_kernel(const double* __restrict__ logits, const double* __restrict__ e_local,
                          const int32_t* __restrict__ cand, const int32_t* __restrict__ n_cand, int cand_cap,
                          const double* __restrict__ cstats, int n_chunks, const int64_t* __restrict__ budget,
                          uint8_t* __restrict__ flag, int32_t* __restrict__ sel_tokens,
                          // fine level
                          const int32_t* __restrict__ fsize, const int32_t* __restrict__ fmem_off,
                          const int32_t* __restrict__ fmem, int fcap, int fmem_cap, const int32_t* __restrict__ fcount,
                          // coarse level (hierarchy: extras of the denominator and rejected coarse terms)
                          const int32_t* __restrict__ csize, const int32_t* __restrict__ ccount, int ccap,
                          const uint8_t* __restrict__ cflag, const double* __restrict__ clogits,
                          // sequence layout
                          const int32_t* __restrict__ sink_end, const int32_t* __restrict__ buffer_start,
                          const int32_t* __restrict__ cache_len, int n_kv_heads, int replacement,
                          // outputs
                          int32_t* __restrict__ tok, int tok_cap, int32_t* __restrict__ rej,
                          float* __restrict__ rej_w, int rej_cap, int32_t* __restrict__ stats, int smem_n,
                          ShardCtl sh) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int l = blockIdx.x, L = gridDim.x;
    dbg_lk(0);
    const int n = cand ? n_cand[l] : fcount[l];
    if (n > smem_n) __trap();  // the host sizes smem_n >= every ledger's candidate count
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem_raw);
    int* sizes = reinterpret_cast<int*>(keys + smem_n);
    int* offs = sizes + smem_n;
    uint8_t* sflag = reinterpret_cast<uint8_t*>(offs + smem_n);
    const int ne = cflag ? ccount[l] : 0;
    const bool lists = !(sh.prefix && !sh.cross);
    select_v2_core<G>(l, logits, e_local, cand, n, cand_cap, fsize, fcap, clogits, csize, cflag, ne, ccap, budget[l],
                      cstats, n_chunks, keys, sizes, sflag, flag, sel_tokens, sh, fmem_off, lists ? offs : nullptr);
    dbg_lk(3);
    if (sh.prefix && !sh.cross) return;  // sharded local pass: only the candidate prefix is needed
    if (!rej && replacement && e_local) {
        // serving path: this was the last read of the ledger's e_local (the next step's logits
        // kernel rewrites it) -- drop it from L2 instead of letting the decode evict it to HBM
        for (int g = 0; g < G; ++g)
            discard_l2_range(e_local + ((size_t)l * G + g) * cand_cap, (size_t)n * sizeof(double), threadIdx.x,
                             blockDim.x);
    }
    worklist_v2<G>(l, L, n, logits, cand, cand_cap, sflag, sizes, reinterpret_cast<int*>(keys), fmem_off, fmem, fcap,
                   fmem_cap, offs, csize, ne, ccap, cflag, clogits, sink_end, buffer_start, cache_len, n_kv_heads,
                   replacement, tok, tok_cap, rej, rej_w, rej_cap, stats);
    dbg_lk(4);
}

// selection only (the hierarchy's coarse promotion stage)
template <int G>
__global__ void __launch_bounds__(kSel2Threads)
select_v2_kernel(const double* __restrict__ logits, const double* __restrict__ e_local,
                 const int32_t* __restrict__ cand, const int32_t* __restrict__ n_cand, int cand_cap,
                 const int32_t* __restrict__ lv_size, int lv_cap, const double* __restrict__ elogits,
                 const int32_t* __restrict__ esize, const uint8_t* __restrict__ eflag,
                 const int32_t* __restrict__ n_extra, int ecap, const int64_t* __restrict__ budget,
                 uint8_t* __restrict__ flag, int32_t* __restrict__ sel_tokens, const double* __restrict__ cstats,
                 int n_chunks, int smem_n) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int l = blockIdx.x;
    if (n_cand[l] > smem_n) __trap();  // the host sizes smem_n >= every ledger's candidate count
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem_raw);
    int* sizes = reinterpret_cast<int*>(keys + smem_n);
    uint8_t* sflag = reinterpret_cast<uint8_t*>(sizes + smem_n);
    select_v2_core<G>(l, logits, e_local, cand, n_cand[l], cand_cap, lv_size, lv_cap, elogits, esize, eflag,
                      elogits ? n_extra[l] : 0, ecap, budget[l], cstats, n_chunks, keys, sizes, sflag, flag,
                      sel_tokens, ShardCtl{});
}

// per (ledger, head): (M, Z) of this rank's candidates from the chunk partials
__global__ void head_norms_kernel(const double* __restrict__ cstats, int n_chunks, const int32_t* __restrict__ count,
                                  int G, double* __restrict__ out) {
    const int l = blockIdx.x, g = threadIdx.x;
    if (g >= G) return;
    const int nchu = min(n_chunks, (count[l] + 127) >> 7);
    const double* cs = cstats + (size_t)l * n_chunks * G * 2;
    double M = -INFINITY;
    for (int c = 0; c < nchu; ++c) M = fmax(M, cs[(c * G + g) * 2]);
    double Z = 0.0;
    for (int c = 0; c < nchu; ++c) {
        const double cm = cs[(c * G + g) * 2];
        if (cm != -INFINITY) Z += cs[(c * G + g) * 2 + 1] * exp(cm - M);
    }
    out[((size_t)l * G + g) * 2] = M;
    out[((size_t)l * G + g) * 2 + 1] = Z;
}

// global (M, Z) from every rank's [P][L][G][2]
__global__ void merge_norms_kernel(const double* __restrict__ parts, int P, int LG, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= LG) return;
    double M = -INFINITY;
    for (int r = 0; r < P; ++r) M = fmax(M, parts[((size_t)r * LG + i) * 2]);
    double Z = 0.0;
    for (int r = 0; r < P; ++r) {
        const double m = parts[((size_t)r * LG + i) * 2];
        if (m != -INFINITY) Z += parts[((size_t)r * LG + i) * 2 + 1] * exp(m - M);
    }
    out[(size_t)i * 2] = M;
    out[(size_t)i * 2 + 1] = Z;
}

// the global crossing candidate of each ledger from every rank's prefix [P][L][cap]
__global__ void __launch_bounds__(kSel2Threads)
global_cut_kernel(const PrefixEntry* __restrict__ prefix, const int32_t* __restrict__ prefix_n, int P, int L,
                  int cap, const int64_t* __restrict__ budget, Cross* __restrict__ cross) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int l = blockIdx.x;
    const int nmax = P * cap;
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem_raw);
    int* sizes = reinterpret_cast<int*>(keys + nmax);
    unsigned int* ids = reinterpret_cast<unsigned int*>(sizes + nmax);
    __shared__ int s_base[65];
    __shared__ unsigned long long s_tot[kSel2Threads / 32];
    if (threadIdx.x == 0) {
        int b = 0;
        for (int r = 0; r < P; ++r) {
            s_base[r] = b;
            b += min(prefix_n[(size_t)r * L + l], cap);
        }
        s_base[P] = b;
    }
    __syncthreads();
    const int n = s_base[P];
    unsigned long long tot = 0;
    for (int r = 0; r < P; ++r) {
        const int cnt = s_base[r + 1] - s_base[r];
        for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
            const PrefixEntry e = prefix[((size_t)r * L + l) * cap + j];
            keys[s_base[r] + j] = e.key;
            sizes[s_base[r] + j] = e.size;
            ids[s_base[r] + j] = e.gid;
            tot += (unsigned long long)e.size;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if ((threadIdx.x & 31) == 0) s_tot[threadIdx.x >> 5] = tot;
    __syncthreads();
    unsigned long long total = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) total += s_tot[w];
    const long long B = budget[l];
    Cross c{~0ull, 0xffffffffu, 0u};
    if (B <= 0) c = Cross{0ull, 0u, 0u};
    else if ((long long)total >= B && n > 0) radix_cross(keys, sizes, [&](int i) { return ids[i]; }, n, B, c.k, c.i);
    if (threadIdx.x == 0) cross[l] = c;
}

}  // namespace mpa

using namespace mpa;

static int encode_bf16_rows(CUtensorMap* out, const void* base, long long rows, int d, int box_rows) {
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

int mpa_launch_logits_v2(const double* q_lk, int group, int d, const mpa_level* lv, const int32_t* cand,
                         const int32_t* n_cand, int cand_cap, double* logits, double* chunk_stats, double* e_local,
                         int n_chunks, int n_max, float* rej_w, int rej_cap, const float* q_raw, const double* cs_lk,
                         cudaStream_t st) {
    const int L = lv->n_ledgers;
    // items: ledgers x the chunks any ledger can use (n_max bounds the live candidates); chunk
    // stats rows past them are written -inf once per ledger by the last items
    const int item_chunks = ceil_div(n_max > 0 ? n_max : (cand ? cand_cap : lv->cap), kLgChunk);
    if (L * item_chunks <= 0) return 0;
    MPA_REQUIRE(!cs_lk || (d == 128 && q_raw), MPA_ERR_UNSUPPORTED,
                "mpa_centroid_logits: the fused lookup rotation needs the d = 128 TMA path");
    MPA_REQUIRE(!rej_w || (d == 128 && !cand && chunk_stats && rej_cap >= lv->cap), MPA_ERR_UNSUPPORTED,
                "mpa_centroid_logits: per-candidate replacement weights need the flat d = 128 TMA path");
    if (d == 128) {  // TMA tiles (flat) / row gathers (candidate lists), one CTA per (chunk, ledger)
        CUtensorMap tt, tr;
        if (int rc = encode_bf16_rows(&tt, lv->kc, (long long)L * lv->cap, 128, kLgChunk)) return rc;
        if (int rc = encode_bf16_rows(&tr, lv->kc, (long long)L * lv->cap, 128, 1)) return rc;
        dim3 g2(item_chunks, L);
        MPA_DISPATCH_G(group, {
            const size_t smem = 1024 + 2 * kLgChunk * 128 + sizeof(double) * (kG * 4 * 34 + kG * kLgChunk);
            auto kern = logits_tma_kernel<kG>;
            if (int rc = set_max_smem((const void*)kern, (int)smem)) return rc;
            launch_pdl(kern, g2, dim3(kLgThreads), smem, st, tt, tr, q_lk, lv->cap, lv->count, lv->size, cand, n_cand,
                       cand_cap, logits, chunk_stats, e_local, n_chunks, rej_w, rej_cap, q_raw, cs_lk);
        });
        return check_launch("mpa_centroid_logits(tma)");
    }
    MPA_DISPATCH_G(group, {  // d = 64: smem-blocked kernel
        auto kern = logits_block_kernel<kG, 64, 1>;
        const size_t smem = LgGeom<kG, 64>::smem(1);
        if (int rc = set_max_smem((const void*)kern, (int)smem)) return rc;
        kern<<<L * item_chunks, kLgThreads, smem, st>>>(q_lk, (const __nv_bfloat16*)lv->kc, lv->cap, lv->count, lv->size,
                                                        cand, n_cand, cand_cap, logits, chunk_stats, e_local, n_chunks,
                                                        item_chunks, L);
    });
    return check_launch("mpa_centroid_logits(block)");
}

size_t mpa_select_v2_smem(int n_max) { return sel_smem_bytes(n_max); }

int mpa_launch_select_v2(const double* logits, const double* e_local, int group, const int32_t* cand,
                         const int32_t* n_cand, int cand_cap, const int32_t* lv_size, int lv_cap,
                         const double* elogits, const int32_t* esize, const uint8_t* eflag, const int32_t* n_extra,
                         int ecap, const int64_t* budget, int n_ledgers, uint8_t* flag, int32_t* sel_tokens,
                         const double* chunk_stats, int n_chunks, int n_max, cudaStream_t st) {
    const size_t smem = sel_smem_bytes(n_max);
    MPA_DISPATCH_G(group, {
        auto kern = select_v2_kernel<kG>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_pdl(kern, dim3(n_ledgers), dim3(kSel2Threads), smem, st, logits, e_local, cand, n_cand, cand_cap,
                   lv_size, lv_cap, elogits, esize, eflag, n_extra, ecap, budget, flag, sel_tokens, chunk_stats,
                   n_chunks, n_max);
    });
    return check_launch("mpa_select(v2)");
}

int mpa_launch_select_worklist_v2(const mpa_level* fine, const mpa_level* coarse, int group, const double* logits,
                                  const double* e_local, const int32_t* cand, const int32_t* n_cand, int cand_cap,
                                  const double* chunk_stats, int n_chunks, const uint8_t* cflag,
                                  const double* clogits, const int64_t* budget, const int32_t* sink_end,
                                  const int32_t* buffer_start, const int32_t* cache_len, int n_kv_heads,
                                  int n_ledgers, int replacement, uint8_t* flag, int32_t* sel_tokens, int32_t* tok,
                                  int tok_cap, int32_t* rej, float* rej_w, int rej_cap, int32_t* stats, int n_max,
                                  cudaStream_t st, const ShardCtl& sh) {
    const size_t smem = sel_smem_bytes(n_max);
    MPA_DISPATCH_G(group, {
        auto kern = select_worklist_v2_kernel<kG>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_pdl(kern, dim3(n_ledgers), dim3(kSel2Threads), smem, st, logits, e_local, cand, n_cand, cand_cap,
                   chunk_stats, n_chunks, budget, flag, sel_tokens, fine->size, fine->off, fine->idx, fine->cap,
                   fine->idx_cap, fine->count, coarse ? coarse->size : nullptr, coarse ? coarse->count : nullptr,
                   coarse ? coarse->cap : 0, cflag, clogits, sink_end, buffer_start, cache_len, n_kv_heads,
                   replacement, tok, tok_cap, rej, rej_w, rej_cap, stats, n_max, sh);
    });
    return check_launch("mpa_select_worklist(v2)");
}

#ifdef MPA_DEBUG_TRACE
extern "C" int mpa_debug_trace_lookup(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_dbg_lk, sizeof(unsigned long long) * n);
}
#endif

// unsharded entry (mpa_lookup.cu)
int mpa_launch_select_worklist_v2(const mpa_level* fine, const mpa_level* coarse, int group, const double* logits,
                                  const double* e_local, const int32_t* cand, const int32_t* n_cand, int cand_cap,
                                  const double* chunk_stats, int n_chunks, const uint8_t* cflag,
                                  const double* clogits, const int64_t* budget, const int32_t* sink_end,
                                  const int32_t* buffer_start, const int32_t* cache_len, int n_kv_heads,
                                  int n_ledgers, int replacement, uint8_t* flag, int32_t* sel_tokens, int32_t* tok,
                                  int tok_cap, int32_t* rej, float* rej_w, int rej_cap, int32_t* stats, int n_max,
                                  cudaStream_t st) {
    return mpa_launch_select_worklist_v2(fine, coarse, group, logits, e_local, cand, n_cand, cand_cap, chunk_stats,
                                         n_chunks, cflag, clogits, budget, sink_end, buffer_start, cache_len,
                                         n_kv_heads, n_ledgers, replacement, flag, sel_tokens, tok, tok_cap, rej,
                                         rej_w, rej_cap, stats, n_max, st, ShardCtl{});
}

extern "C" int mpa_head_norms(const double* chunk_stats, int n_chunks, const int32_t* count, int n_ledgers, int group,
                              double* out, void* stream) {
    MPA_REQUIRE(chunk_stats && count && out, MPA_ERR_ARG, "mpa_head_norms: null argument");
    if (n_ledgers <= 0) return 0;
    head_norms_kernel<<<n_ledgers, 32, 0, (cudaStream_t)stream>>>(chunk_stats, n_chunks, count, group, out);
    return check_launch("mpa_head_norms");
}

extern "C" int mpa_merge_norms(const double* parts, int n_ranks, int n_ledgers, int group, double* out,
                               void* stream) {
    MPA_REQUIRE(parts && out, MPA_ERR_ARG, "mpa_merge_norms: null argument");
    const int LG = n_ledgers * group;
    if (LG <= 0) return 0;
    merge_norms_kernel<<<ceil_div(LG, 128), 128, 0, (cudaStream_t)stream>>>(parts, n_ranks, LG, out);
    return check_launch("mpa_merge_norms");
}

extern "C" int mpa_global_cut(const void* prefix, const int32_t* prefix_n, int n_ranks, int n_ledgers, int prefix_cap,
                              const int64_t* budget, void* cross, void* stream) {
    MPA_REQUIRE(prefix && prefix_n && budget && cross, MPA_ERR_ARG, "mpa_global_cut: null argument");
    MPA_REQUIRE(n_ranks >= 1 && n_ranks <= 64, MPA_ERR_UNSUPPORTED, "mpa_global_cut: %d ranks", n_ranks);
    const size_t smem = (size_t)n_ranks * prefix_cap * 16;
    MPA_REQUIRE(smem <= 200 * 1024, MPA_ERR_UNSUPPORTED, "mpa_global_cut: %d x %d prefix entries", n_ranks,
                prefix_cap);
    if (n_ledgers <= 0) return 0;
    cudaFuncSetAttribute(global_cut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    global_cut_kernel<<<n_ledgers, kSel2Threads, smem, (cudaStream_t)stream>>>(
        (const PrefixEntry*)prefix, prefix_n, n_ranks, n_ledgers, prefix_cap, budget, (Cross*)cross);
    return check_launch("mpa_global_cut");
}

extern "C" int mpa_select_worklist_sharded(const mpa_level* fine, int group, const double* logits,
                                           const double* e_local, const double* chunk_stats, const int64_t* budget,
                                           const int32_t* sink_end, const int32_t* buffer_start,
                                           const int32_t* cache_len, int n_kv_heads, int replacement, uint8_t* flag,
                                           int32_t* sel_tokens, int32_t* tok, int tok_cap, int32_t* rej,
                                           float* rej_w, int rej_cap, int32_t* stats, int n_max, const double* mz,
                                           const void* cross, void* prefix, int32_t* prefix_n, int prefix_cap,
                                           const int32_t* gid_off, void* stream) {
    MPA_REQUIRE(fine && logits && chunk_stats && budget && flag && sink_end && buffer_start && cache_len && tok &&
                    rej_w && stats && mz && gid_off,
                MPA_ERR_ARG, "mpa_select_worklist_sharded: null argument");
    MPA_REQUIRE((cross != nullptr) != (prefix != nullptr), MPA_ERR_ARG,
                "mpa_select_worklist_sharded: exactly one of cross (final pass) / prefix (local pass)");
    MPA_REQUIRE(!prefix || prefix_n, MPA_ERR_ARG, "mpa_select_worklist_sharded: prefix without counts");
    if (n_max <= 0 || n_max > fine->cap) n_max = fine->cap;
    MPA_REQUIRE(mpa_select_v2_smem(n_max) <= 200 * 1024, MPA_ERR_UNSUPPORTED,
                "mpa_select_worklist_sharded: %d candidates", n_max);
    if (fine->n_ledgers <= 0) return 0;
    ShardCtl sh;
    sh.mz = mz;
    sh.cross = (const Cross*)cross;
    sh.prefix = (PrefixEntry*)prefix;
    sh.prefix_n = prefix_n;
    sh.prefix_cap = prefix_cap;
    sh.gid_off = gid_off;
    return mpa_launch_select_worklist_v2(fine, nullptr, group, logits, e_local, nullptr, nullptr, fine->cap,
                                         chunk_stats, ceil_div(fine->cap, 128), nullptr, nullptr, budget, sink_end,
                                         buffer_start, cache_len, n_kv_heads, fine->n_ledgers, replacement, flag,
                                         sel_tokens, tok, tok_cap, rej, rej_w, rej_cap, stats, n_max,
                                         (cudaStream_t)stream, sh);
}
