// The flat serving decode step in ONE launch (bf16 cache and centroids, d = 128, G <= 8):
// lookup-view rotation, fp64 centroid logits, Eq. 1 scores, budgeted selection, work lists,
// centroid replacement over the value centroids of every rejected cluster, exact attention over
// sinks + buffer + the selected clusters' members, the merge -- and the step's K/V append.
// One thread-block cluster of C CTAs per ledger (C = 1 at batch 16 x 8 kv-heads, up to 16 at
// batch 1, so the grid is one wave); each CTA owns a contiguous slice of the ledger's centroids.
//
// Reference (pkg/src/multipole_attn/):
//   rope.py:37-53, 66-68      rotate (exact view at cache_len) / lookup_query_view (at delta)
//   attention.py:267-290      _scores_per_group: l = Q_lk Kc^T / sqrt(d); e = exp(l - max_g);
//                             score = mean_g e / (e . N)
//   attention.py:192-207      select_clusters: visit by (score desc, ref asc), take while cum < B
//   attention.py:354-375      flat_lookup (selected token ids, rejected clusters + their logits)
//   attention.py:58-87, 120-137, 210-239, 469-498
//                             exact / sparse-exact partials, centroid replacement (weights
//                             N exp(l)), merge_partials, finalize
//   pipeline.py:156-159       append the step's token after attending
//
// Phases of CTA rank r (centroids [c0, c0 + nloc) of ledger l):
//   0. prologue: TMA of the first 8 key-centroid chunks (64 rows x 256 B, 128B swizzle), sizes /
//      member offsets prefetched to registers, then (after the stream predecessor) the lookup view.
//   1. logits: 4 groups of 64 threads, 8 stages; fp64 DFMA 4-row x G-head register blocks over a
//      quarter of d; bf16 widened to fp64 by integer ops (un-rebiased exponent = exactly x 2^-896,
//      undone by one multiply); per-head running max.
//   2. M = max over the cluster (DSMEM), e = exp(l - M) in place, Z = e . N (DSMEM); the first
//      value-centroid chunks start loading; exact view q / sqrt(d) and the append (rank 0).
//   3. keys = ~bits(mean_g e / Z) (ascending key == descending score) and the key range.
//   4. size-weighted radix select of the crossing candidate (10-bit digits below the common key
//      prefix, then the id), histograms slice-reduced across the cluster.
//   5. flags, replacement weights w = N e (0 for selected), cluster prefix of selected tokens.
//   6. token list: sinks ++ buffer ++ members of the selected clusters (global, for the reports).
//   R. replacement: the slice's value centroids streamed (TMA ring), a_rej = sum w Vc (fp32).
//   T. exact attention over the CTA's tokens (rank 0: sinks + buffer + its members; rank r: its
//      members): K_rot / V rows by cp.async, fp32 online softmax.
//   M. merge (m, s, a) of the exact and replacement partials, across the cluster, out = a / s.
// Selection numerics are the reference's (fp64 logits, exps, normalisers, scores), so the
// selected set is the oracle's except at true ties (|score gap| ~1e-16 relative); outputs are
// fp32 with bf16 storage (tolerance 1e-2).
#include <mutex>

#include "mpa_common.cuh"
#include "mpa_tc.cuh"

namespace mpa {
namespace stp {

#ifdef MPA_DEBUG_TRACE
__device__ unsigned long long g_dbg_step[4096 * 16];
__device__ __forceinline__ void trace(int slot, int by = 0) {
    if (threadIdx.x == by && blockIdx.x < 4096) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
        g_dbg_step[blockIdx.x * 16 + slot] = t;
    }
}
#else
__device__ __forceinline__ void trace(int, int = 0) {}
#endif

constexpr int kThreads = 256;
constexpr int kGroups = 8;                      // phase-1 consumers: one warp per 64-row chunk
constexpr int kGT = kThreads / kGroups;
constexpr int kChunk = 64;                      // centroid rows per chunk
constexpr int kRPT = 8;                         // rows per thread (x G heads x a quarter of d)
constexpr int kRG = kChunk / kRPT;
constexpr int kStages = 8;
constexpr int kStageB = kChunk * 256;           // 16 KB: two 64-column halves of 64 rows
constexpr int kStageArea = kStages * kStageB;   // 128 KB
constexpr int kDig = 10, kBins = 1 << kDig;
constexpr int D = 128, QD = 32, QRow = QD + 2;
constexpr double kUnscale896 = 0x1p896;
constexpr int kSmemBudget = 230000;             // dynamic smem budget (static ~1.5 KB on top)

// shared-memory layout (after the 1024-aligned stage area): logits [G][kcmax] fp64 | lookup q
// slots [G][4][QRow] fp64 | sizes [kcmax] | member offsets [kcmax] | sflag [kcmax]
template <int G>
struct Geo {
    static constexpr int GP = G <= 4 ? 4 : 8;
    static constexpr int qB = G * 4 * QRow * 8;
    static constexpr int fixedB = 1024 + kStageArea + qB + 64;
    static constexpr int kc_raw = (kSmemBudget - fixedB) / (G * 8 + 4 + 4 + 1);
    static constexpr int kcmax_ = kc_raw / kChunk * kChunk;
    static constexpr int kcmax = kcmax_ > 4096 ? 4096 : kcmax_;  // keys (8 B each) fit in 2 stages
    static constexpr int lgB = G * kcmax * 8;
    static constexpr int oLG = 1024 + kStageArea;
    static constexpr int oQ = oLG + lgB;
    static constexpr int oSZ = oQ + qB;
    static constexpr int oMO = oSZ + kcmax * 4;
    static constexpr int oFL = oMO + kcmax * 4;
    static constexpr int total = oFL + kcmax + 16;
};

struct Params {
    const float* q;            // [L, G, D] fp32 queries (sequence-major: l * G + g)
    const double* cs_lk;       // [D/2][2] (cos, sin)(delta * inv_freq)
    const double* inv_freq;    // [D/2]
    float q_scale;             // 1 / sqrt(d)
    const int32_t* count;      // [L]
    const int32_t* size;       // [L, kcap]
    const int32_t* moff;       // [L, kcap + 1]
    const int32_t* mem;        // [L, mem_cap]
    int kcap, mem_cap;
    const int64_t* budget;     // [L]
    const int32_t* sink_end;   // [n_seq]
    const int32_t* buffer_start;
    int32_t* cache_len;        // [n_seq] (advanced by the last CTA when appending)
    int n_kv_heads, replacement, L, n_seq;
    uint8_t* flag;             // [L, kcap]
    int32_t* sel_tokens;       // [L]
    int32_t* tok;              // [L, tok_cap]
    int tok_cap;
    int32_t* stats;            // [4, L]
    int kc;                    // centroids per CTA (multiple of kChunk)
    // decode-step extras: exact view, contiguous replacement weights, append (k_new != NULL)
    float* q_rot;              // [L, G, D] rotate(q, cache_len) * q_scale (fp32), NULL: not formed
    float* rej_w;              // [L, rej_cap, GP] logit + ln N of every centroid, selected -inf
    int rej_cap;
    __nv_bfloat16* k_rot;
    __nv_bfloat16* k_raw;
    __nv_bfloat16* vcache;
    int tcap;
    KvRows kv;                 // rows of k_rot / vcache (flat or paged); k_raw is [L, tcap, D]
    const float* k_new;        // [L, D]
    const float* v_new;
    int32_t* ntok_dense;       // [L] (optional)
    int32_t* ticket;           // one zero-initialised int32, left zeroed
};

__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned dsm_addr(const void* p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ double dsm_f64(const void* p, unsigned rank) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(dsm_addr(p, rank)) : "memory");
    return v;
}
__device__ __forceinline__ float dsm_f32(const void* p, unsigned rank) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(dsm_addr(p, rank)) : "memory");
    return v;
}
__device__ __forceinline__ unsigned dsm_u32(const void* p, unsigned rank) {
    unsigned v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(dsm_addr(p, rank)) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long dsm_u64(const void* p, unsigned rank) {
    unsigned long long v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(dsm_addr(p, rank)) : "memory");
    return v;
}
__device__ __forceinline__ void group_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// bf16 (in the high half of fbits) -> fp64 bits of x * 2^-896: no exponent re-bias
__device__ __forceinline__ double bf16hi_s896(unsigned fbits) {
    return __hiloint2double((int)(((int)fbits >> 3) & 0x8FFFE000), 0);
}
// one out-of-line copy of the fp64 sincos (its slow path is large)
__device__ __noinline__ void dsincos(double x, double* s, double* c) { sincos(x, s, c); }
// block-wide exclusive scan of one u64 per thread
__device__ __forceinline__ unsigned long long scan_u64(unsigned long long v, unsigned long long* sc,
                                                       unsigned long long* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) sc[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        unsigned long long s = lane < nw ? sc[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) sc[lane] = s;
        if (lane == 31) sc[32] = s;
    }
    __syncthreads();
    const unsigned long long base = w ? sc[w - 1] : 0ull;
    *total = sc[32];
    __syncthreads();
    return base + incl - v;
}

template <int G>
__global__ void __launch_bounds__(kThreads, 1)
step_kernel(const __grid_constant__ CUtensorMap tm_kc, const Params p) {
    using Ge = Geo<G>;
    constexpr int GP = Ge::GP;
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* base_sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023) - 1024;
    unsigned char* stage = base_sm + 1024;                                 // [8][64 rows][256 B]
    double* LG = reinterpret_cast<double*>(base_sm + Ge::oLG);             // [G][Kc] logits -> e
    double* qs = reinterpret_cast<double*>(base_sm + Ge::oQ);              // [G][4][QRow] lookup view
    int* sizes = reinterpret_cast<int*>(base_sm + Ge::oSZ);                // [Kc]
    int* moff_s = reinterpret_cast<int*>(base_sm + Ge::oMO);               // [Kc] member CSR offsets
    uint8_t* sflag = base_sm + Ge::oFL;                                    // [Kc]
    __shared__ __align__(8) uint64_t bar[kStages];
    __shared__ double s_red[kThreads / 32][G];
    __shared__ double s_loc[G];
    __shared__ double s_M[G], s_Z[G];
    __shared__ unsigned long long s_u64[6];
    __shared__ unsigned long long s_scan[33];
    __shared__ unsigned long long s_kprefix, s_kmask;
    __shared__ unsigned s_iprefix, s_imask;
    __shared__ long long s_below;
    __shared__ int s_cnt;
    __shared__ unsigned long long s_cross_k;
    __shared__ unsigned s_cross_i;
    __shared__ long long s_sel[2];

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    trace(0);
    const int C = gridDim.x / p.L;  // cluster size (1 when launched without clusters)
    const unsigned rank = C > 1 ? cl_rank() : 0u;
    const int l = blockIdx.x / C;
    const int Kc = p.kc;
    const int n = p.count[l];
    const int c0 = (int)rank * Kc;
    const int nloc = max(0, min(n, c0 + Kc) - c0);
    const int nch = (nloc + kChunk - 1) / kChunk;
    const bool repl = p.rej_w != nullptr && p.replacement;

    // ---- 0. prologue (ledger state only -- older than the stream predecessor)
    if (tid == 0) {
        for (int k = 0; k < kStages; ++k) mbar_init(smem_u32(&bar[k]), 1);
        fence_mbar_init();
        prefetch_tmap(&tm_kc);

    }
    __syncthreads();
    auto issue = [&](const CUtensorMap* tm, uint64_t* bars, int j, int ring) {  // chunk j -> stage j % ring
        unsigned char* st = stage + (j % ring) * kStageB;
        const unsigned b = smem_u32(&bars[j % ring]);
        const int row0 = l * p.kcap + c0 + j * kChunk;
        mbar_expect_tx(b, kStageB);
        tma_load_2d(smem_u32(st), tm, 0, row0, b);
        tma_load_2d(smem_u32(st + kChunk * 128), tm, 64, row0, b);
    };
    if (tid < kStages && tid < nch) issue(&tm_kc, bar, tid, kStages);

    const int32_t* szp = p.size + (size_t)l * p.kcap + c0;
    const int32_t* ofp = p.moff + (size_t)l * (p.kcap + 1) + c0;
#pragma unroll 8
    for (int i = tid; i < nloc; i += kThreads) {  // read in phases 2-6 (unrolled: the loads overlap)
        sizes[i] = __ldg(szp + i);
        moff_s[i] = __ldg(ofp + i);
    }
    __shared__ double s_cs[D];  // (cos, sin) of the lookup view's angles: constant, loaded early
    if (tid < D) s_cs[tid] = p.cs_lk[tid];
    pdl_wait();  // q (and k, v) come from the stream predecessor
    __syncthreads();  // s_cs
    const int seq = l / p.n_kv_heads;
    const int qpos = p.cache_len[seq];
    for (int e = tid; e < G * (D / 2); e += kThreads) {
        const int g = e / (D / 2), i = e - g * (D / 2), k = 2 * i;
        const float2 xy = *reinterpret_cast<const float2*>(p.q + ((size_t)l * G + g) * D + k);
        const double x = (double)xy.x, y = (double)xy.y, c = s_cs[2 * i], sn = s_cs[2 * i + 1];
        double* slot = qs + (g * 4 + k / QD) * QRow + (k % QD);
        slot[0] = __dsub_rn(__dmul_rn(x, c), __dmul_rn(y, sn));
        slot[1] = __dadd_rn(__dmul_rn(x, sn), __dmul_rn(y, c));
    }
    __syncthreads();
    trace(1);

    // ---- 1. logits, group gi takes chunks gi, gi + 4, ...; chunk j + 8 refills stage j % 8
    const int gi = tid / kGT, gt = tid % kGT;
    const double sq = sqrt((double)D);
    double mx[G];
#pragma unroll
    for (int g = 0; g < G; ++g) mx[g] = -INFINITY;
    {
        const int qt = gt & 3, rg = gt >> 2;
        const bool hi2 = qt & 2, hi1 = qt & 1;
        constexpr int GH = (G + 1) / 2, RH = kRPT / 2;
        const double* qq = qs + qt * QRow;
        for (int j = gi; j < nch; j += kGroups) {
            const unsigned char* tile = stage + (j % kStages) * kStageB;
            mbar_wait(smem_u32(&bar[j % kStages]), (j / kStages) & 1);
            double acc[kRPT][G];
#pragma unroll
            for (int r = 0; r < kRPT; ++r)
#pragma unroll
                for (int g = 0; g < G; ++g) acc[r][g] = 0.0;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int c = (cc + 2 * (qt >> 1)) & 3;  // this quarter's 16-byte chunk (8 dims)
                const int ch = (qt & 1) * 4 + c;         // chunk within the 64-column half
                uint4 raw[kRPT];
#pragma unroll
                for (int r = 0; r < kRPT; ++r) {
                    const int row = rg + kRG * r;
                    raw[r] = *reinterpret_cast<const uint4*>(tile + (qt >> 1) * kChunk * 128 + row * 128 +
                                                             ((ch ^ (row & 7)) << 4));
                }
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                    double2 qv[G];
#pragma unroll
                    for (int g = 0; g < G; ++g)
                        qv[g] = *reinterpret_cast<const double2*>(qq + g * 4 * QRow + c * 8 + 2 * e2);
#pragma unroll
                    for (int r = 0; r < kRPT; ++r) {
                        const unsigned wd = (&raw[r].x)[e2];
                        const double x0 = bf16hi_s896(wd << 16), x1 = bf16hi_s896(wd & 0xffff0000u);
#pragma unroll
                        for (int g = 0; g < G; ++g) acc[r][g] = fma(qv[g].x, x0, acc[r][g]);
#pragma unroll
                        for (int g = 0; g < G; ++g) acc[r][g] = fma(qv[g].y, x1, acc[r][g]);
                    }
                }
            }
            __syncwarp();  // the stage is consumed (the group is one warp)
            if (gt == 0 && j + kStages < nch) issue(&tm_kc, bar, j + kStages, kStages);

            double a2[RH][G];
#pragma unroll
            for (int rr = 0; rr < RH; ++rr)
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double send = hi2 ? acc[rr][g] : acc[rr + RH][g];
                    const double keep = hi2 ? acc[rr + RH][g] : acc[rr][g];
                    a2[rr][g] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
                }
            double a1[RH][GH];
#pragma unroll
            for (int rr = 0; rr < RH; ++rr)
#pragma unroll
                for (int jj = 0; jj < GH; ++jj) {
                    const int ghi = GH + jj;
                    const double lo = a2[rr][jj], hv = ghi < G ? a2[rr][ghi < G ? ghi : 0] : 0.0;
                    const double send = hi1 ? lo : hv;
                    const double keep = hi1 ? hv : lo;
                    a1[rr][jj] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
                }
#pragma unroll
            for (int rr = 0; rr < RH; ++rr) {
                const int r = rg + kRG * ((hi2 ? RH : 0) + rr);
                const bool live = j * kChunk + r < nloc;
#pragma unroll
                for (int jj = 0; jj < GH; ++jj) {
                    const int g = (hi1 ? GH : 0) + jj;
                    if (g < G) {
                        const double v = (a1[rr][jj] * kUnscale896) / sq;
                        LG[(size_t)g * Kc + j * kChunk + r] = v;
                        if (live) mx[g] = fmax(mx[g], v);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const double r = warp_max(mx[g]);
        if (lane == 0) s_red[w][g] = r;
    }
    __syncthreads();  // every stage consumed: the value centroids may start streaming
    trace(2);
    pdl_trigger();
    if (tid < G) {
        double r = -INFINITY;
        for (int ww = 0; ww < kThreads / 32; ++ww) r = fmax(r, s_red[ww][tid]);
        s_loc[tid] = r;
    }
    __syncthreads();
    if (C > 1) cl_sync();
    if (tid < G) {
        double r = s_loc[tid];
        for (int k = 0; k < C; ++k)
            if (k != (int)rank) r = fmax(r, dsm_f64(&s_loc[tid], k));
        s_M[tid] = r;
    }
    if (C > 1) cl_sync();  // peers finished reading s_loc before it is reused
    __syncthreads();
    trace(3);

    // ---- 2. e = exp(l - M) in place, Z = e . N, sizes staged; exact view and append
    {
        double M[G], z[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            M[g] = s_M[g];
            z[g] = 0.0;
        }
        long long tot = 0;
#pragma unroll 1
        for (int i = tid; i < nloc; i += kThreads) {
            const int sz = sizes[i];
            tot += sz;
            const double nsz = (double)sz, lnN = (double)logf((float)sz);
            float wv[GP];
#pragma unroll
            for (int g = 0; g < GP; ++g) wv[g] = 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double lgv = LG[(size_t)g * Kc + i];
                wv[g] = (float)(lgv + lnN);  // the replacement weight's log, reused by the decode kernel
                const double e = exp(lgv - M[g]);
                LG[(size_t)g * Kc + i] = e;
                z[g] = fma(e, nsz, z[g]);
            }
            if (repl) {
                float4* dst = reinterpret_cast<float4*>(p.rej_w + ((size_t)l * p.rej_cap + c0 + i) * GP);
#pragma unroll
                for (int v = 0; v < GP / 4; ++v) dst[v] = make_float4(wv[4 * v], wv[4 * v + 1], wv[4 * v + 2], wv[4 * v + 3]);
            }
        }
        // exact view rotate(q, cache_len) / sqrt(d) (attention.py:84-85) into smem (every rank)
        // and the step's key / value at row cache_len (rope.py:37-53, pipeline.py:156-159): no list
        // of this step reads that row; fp64 angles pos * inv_freq
        if (rank == 0 && (p.q_rot || p.k_new)) {
            for (int e = tid; e < G * (D / 2); e += kThreads) {
                const int g = e / (D / 2), i = e - g * (D / 2), k = 2 * i;
                const bool app = p.k_new && g == 0;
                double s2, c2;
                dsincos((double)qpos * p.inv_freq[i], &s2, &c2);
                if (p.q_rot) {
                    const float2 xy = *reinterpret_cast<const float2*>(p.q + ((size_t)l * G + g) * D + k);
                    const double x = (double)xy.x, y = (double)xy.y;
                    float* qr = p.q_rot + ((size_t)l * G + g) * D + k;
                    qr[0] = (float)(__dsub_rn(__dmul_rn(x, c2), __dmul_rn(y, s2)) * (double)p.q_scale);
                    qr[1] = (float)(__dadd_rn(__dmul_rn(x, s2), __dmul_rn(y, c2)) * (double)p.q_scale);
                }
                if (app) {
                    const float2 kk = *reinterpret_cast<const float2*>(p.k_new + (size_t)l * D + k);
                    const float2 vv = *reinterpret_cast<const float2*>(p.v_new + (size_t)l * D + k);
                    const double kx = (double)kk.x, ky = (double)kk.y;
                    const size_t raw = ((size_t)l * p.tcap + qpos) * D + k;
                    const size_t dst = (size_t)p.kv.row(l, qpos) * D + k;
                    p.k_rot[dst] = __double2bfloat16(__dsub_rn(__dmul_rn(kx, c2), __dmul_rn(ky, s2)));
                    p.k_rot[dst + 1] = __double2bfloat16(__dadd_rn(__dmul_rn(kx, s2), __dmul_rn(ky, c2)));
                    p.k_raw[raw] = __double2bfloat16(kx);
                    p.k_raw[raw + 1] = __double2bfloat16(ky);
                    p.vcache[dst] = __double2bfloat16((double)vv.x);
                    p.vcache[dst + 1] = __double2bfloat16((double)vv.y);
                }
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const double r = warp_sum(z[g]);
            if (lane == 0) s_red[w][g] = r;
        }
        unsigned long long tl = warp_sum((unsigned long long)tot);
        if (lane == 0) s_scan[w] = tl;
        __syncthreads();
        if (tid < G) {
            double r = 0.0;
            for (int ww = 0; ww < kThreads / 32; ++ww) r += s_red[ww][tid];
            s_loc[tid] = r;
        }
        if (tid == 32) {
            unsigned long long t = 0;
            for (int ww = 0; ww < kThreads / 32; ++ww) t += s_scan[ww];
            s_u64[0] = t;
        }
        __syncthreads();
        if (C > 1) cl_sync();
        if (tid < G) {
            double r = 0.0;
            for (int k = 0; k < C; ++k) r += k == (int)rank ? s_loc[tid] : dsm_f64(&s_loc[tid], k);
            s_Z[tid] = r;
        }
        if (tid == 32) {
            unsigned long long t = 0;
            for (int k = 0; k < C; ++k) t += k == (int)rank ? s_u64[0] : dsm_u64(&s_u64[0], k);
            s_u64[1] = t;
        }
        __syncthreads();
    }
    trace(4);

    // stage-area use until phase R: stages 0-3 value centroids in flight, 4-5 keys (then the
    // selected-candidate lists), 6 radix histograms
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(stage + 4 * kStageB);
    unsigned* hist_w = reinterpret_cast<unsigned*>(stage + 6 * kStageB);
    unsigned* hist_c = hist_w + kBins;
    unsigned* red_w = hist_c + kBins;
    unsigned* red_c = red_w + kBins;

    // ---- 3. Eq. 1 scores -> keys (mean over heads in head order, like np.mean(axis=0)); e / Z as
    // e * (1 / Z): within an ulp of the reference's division, whose Z is itself a BLAS dot product
    // matched only to an ulp; exact duplicates still tie bit-for-bit
    {
        double rz[G];
#pragma unroll
        for (int g = 0; g < G; ++g) rz[g] = 1.0 / s_Z[g];
        unsigned long long kmin = ~0ull, kmax = 0ull;
        for (int i = tid; i < nloc; i += kThreads) {
            double sc = 0.0;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double e = LG[(size_t)g * Kc + i];
                sc = g ? fma(e, rz[g], sc) : e * rz[g];
            }
            // np.mean's division; by a power of two it is the exact product
            sc = (G & (G - 1)) == 0 ? sc * (1.0 / G) : sc / (double)G;
            const unsigned long long k = ~(unsigned long long)__double_as_longlong(sc);
            keys[i] = k;
            kmin = min(kmin, k);
            kmax = max(kmax, k);
        }
        kmin = warp_min_u64(kmin);
        kmax = warp_max(kmax);
        if (lane == 0) {
            s_scan[w] = kmin;
            s_red[w][0] = __longlong_as_double((long long)kmax);
        }
        __syncthreads();
        if (tid == 0) {
            unsigned long long a = ~0ull, b = 0ull;
            for (int ww = 0; ww < kThreads / 32; ++ww) {
                a = min(a, s_scan[ww]);
                b = max(b, (unsigned long long)__double_as_longlong(s_red[ww][0]));
            }
            s_u64[2] = a;
            s_u64[3] = b;
        }
        __syncthreads();
        if (C > 1) {
            cl_sync();
            if (tid == 0) {
                unsigned long long a = ~0ull, b = 0ull;
                for (int k = 0; k < C; ++k) {
                    a = min(a, k == (int)rank ? s_u64[2] : dsm_u64(&s_u64[2], k));
                    b = max(b, k == (int)rank ? s_u64[3] : dsm_u64(&s_u64[3], k));
                }
                s_u64[4] = a;
                s_u64[5] = b;
            }
        } else if (tid == 0) {
            s_u64[4] = s_u64[2];
            s_u64[5] = s_u64[3];
        }
        __syncthreads();
    }
    trace(8);
    const long long total = (long long)s_u64[1];
    const long long B = p.budget[l];
    const bool select_none = B <= 0;
    const bool select_all = !select_none && total < B;

    // ---- 4. crossing candidate = the smallest (key, id) whose cumulative size reaches B
    unsigned long long kstar = ~0ull;
    unsigned istar = 0xffffffffu;
    if (!select_none && !select_all) {
        const unsigned long long kmin = s_u64[4], kmax = s_u64[5];
        const int ktop = kmin == kmax ? 0 : 64 - __clzll(kmin ^ kmax);  // bits [ktop, 64) common
        if (tid == 0) {
            s_kmask = ktop >= 64 ? 0ull : ~0ull << ktop;
            s_kprefix = kmin & s_kmask;
            s_iprefix = 0u;
            s_imask = 0u;
            s_below = 0;
            s_cnt = 0;
        }
        __syncthreads();
        const int kpasses = (ktop + kDig - 1) / kDig;
        constexpr int kIdPasses = (32 + kDig - 1) / kDig;
        for (int pass = 0; pass < kpasses + kIdPasses; ++pass) {
            const bool kp_pass = pass < kpasses;
            const int top = kp_pass ? ktop - kDig * pass : 32 - kDig * (pass - kpasses);
            const int width = top >= kDig ? kDig : top;
            const int sh = top - width;
            const unsigned dmask = (1u << width) - 1u;
            const unsigned long long kp = s_kprefix, kmask = s_kmask;
            const unsigned ip = s_iprefix, imask = s_imask;
            for (int j = tid; j < kBins; j += kThreads) hist_w[j] = hist_c[j] = 0u;
            __syncthreads();
            for (int i = tid; i < nloc; i += kThreads) {
                const unsigned long long k = keys[i];
                const unsigned id = (unsigned)(c0 + i);
                if ((k & kmask) != kp || (id & imask) != ip) continue;
                const unsigned dg = kp_pass ? (unsigned)(k >> sh) & dmask : (id >> sh) & dmask;
                atomicAdd(&hist_w[dg], (unsigned)sizes[i]);
                atomicAdd(&hist_c[dg], 1u);
            }
            __syncthreads();
            const unsigned* hw = hist_w;
            const unsigned* hc = hist_c;
            if (C > 1) {
                cl_sync();  // every CTA's histogram is complete
                const int per = kBins / C;
                for (int j = tid; j < per; j += kThreads) {
                    const int b = (int)rank * per + j;
                    unsigned sw = 0, sc = 0;
                    for (int k = 0; k < C; ++k) {
                        sw += k == (int)rank ? hist_w[b] : dsm_u32(&hist_w[b], k);
                        sc += k == (int)rank ? hist_c[b] : dsm_u32(&hist_c[b], k);
                    }
                    red_w[b] = sw;
                    red_c[b] = sc;
                }
                cl_sync();  // every slice is reduced
                for (int b = tid; b < kBins; b += kThreads) {
                    const int owner = b / per;
                    if (owner != (int)rank) {
                        red_w[b] = dsm_u32(&red_w[b], owner);
                        red_c[b] = dsm_u32(&red_c[b], owner);
                    }
                }
                __syncthreads();
                hw = red_w;
                hc = red_c;
            }
            constexpr int bpt = kBins / kThreads;
            unsigned long long wsum = 0;
#pragma unroll
            for (int j = 0; j < bpt; ++j) wsum += hw[tid * bpt + j];
            const long long below = s_below;
            const long long need = B - below;  // > 0
            unsigned long long btot;
            const unsigned long long before = scan_u64(wsum, s_scan, &btot);
            if ((long long)before < need && (long long)(before + wsum) >= need) {
                long long run = (long long)before;
                int dg = tid * bpt + bpt - 1;
#pragma unroll
                for (int j = 0; j < bpt; ++j) {
                    const int b = tid * bpt + j;
                    const long long wb = (long long)hw[b];
                    if (run + wb >= need) {
                        dg = b;
                        break;
                    }
                    run += wb;
                }
                s_below = below + run;
                s_cnt = (int)hc[dg];
                if (kp_pass) {
                    s_kprefix = kp | ((unsigned long long)dg << sh);
                    s_kmask = kmask | ((unsigned long long)dmask << sh);
                } else {
                    s_iprefix = ip | ((unsigned)dg << sh);
                    s_imask = imask | (dmask << sh);
                }
            }
            __syncthreads();
            trace(9 + min(pass, 2));
            if (s_cnt == 1) break;
        }
        // the unique candidate matching the final prefix (one CTA of the cluster holds it)
        if (tid == 0) {
            s_cross_k = ~0ull;
            s_cross_i = 0xffffffffu;
        }
        __syncthreads();
        {
            const unsigned long long kp = s_kprefix, kmask = s_kmask;
            const unsigned ip = s_iprefix, imask = s_imask;
            for (int i = tid; i < nloc; i += kThreads) {
                const unsigned id = (unsigned)(c0 + i);
                if ((keys[i] & kmask) == kp && (id & imask) == ip) {
                    s_cross_k = keys[i];
                    s_cross_i = id;
                }
            }
        }
        __syncthreads();
        if (C > 1) {
            s_u64[2] = s_cross_k;
            s_u64[3] = s_cross_i;
            cl_sync();
            if (tid == 0) {
                unsigned long long bk = ~0ull;
                unsigned bi = 0xffffffffu;
                for (int k = 0; k < C; ++k) {
                    const unsigned long long kk = dsm_u64(&s_u64[2], k);
                    const unsigned ii = (unsigned)dsm_u64(&s_u64[3], k);
                    if (kk < bk || (kk == bk && ii < bi)) {
                        bk = kk;
                        bi = ii;
                    }
                }
                s_cross_k = bk;
                s_cross_i = bi;
            }
            __syncthreads();
        }
        kstar = s_cross_k;
        istar = s_cross_i;
    }
    trace(5);

    // ---- 5. flags, the selected rows of rej_w masked to -inf, selected sizes
    long long my_tok = 0, my_sel = 0;
    {
        uint8_t* fl = p.flag + (size_t)l * p.kcap + c0;
        for (int i = tid; i < nloc; i += kThreads) {
            const unsigned id = (unsigned)(c0 + i);
            const bool sel = select_all || (!select_none && (keys[i] < kstar || (keys[i] == kstar && id <= istar)));
            sflag[i] = sel ? 1 : 0;
            fl[i] = sel ? 1 : 0;
            if (sel) {
                my_tok += sizes[i];
                ++my_sel;
                if (repl) {
                    float* dst = p.rej_w + ((size_t)l * p.rej_cap + c0 + i) * GP;
#pragma unroll
                    for (int g = 0; g < G; ++g) dst[g] = -INFINITY;
                }
            }
        }
    }
    {
        const unsigned long long a = warp_sum((unsigned long long)my_tok), b = warp_sum((unsigned long long)my_sel);
        __syncthreads();  // keys are dead from here (the lists below reuse their space)
        if (lane == 0) {
            s_scan[w] = a;
            s_red[w][0] = __longlong_as_double((long long)b);
        }
        __syncthreads();
        if (tid == 0) {
            unsigned long long ta = 0, tb = 0;
            for (int ww = 0; ww < kThreads / 32; ++ww) {
                ta += s_scan[ww];
                tb += (unsigned long long)__double_as_longlong(s_red[ww][0]);
            }
            s_sel[0] = (long long)ta;
            s_sel[1] = (long long)tb;
        }
        __syncthreads();
    }
    long long tok_before = 0, tot_tok = 0, tot_sel = 0;
    if (C > 1) {
        cl_sync();
        for (int k = 0; k < C; ++k) {
            const long long t = k == (int)rank ? s_sel[0] : (long long)dsm_u64(&s_sel[0], k);
            const long long c = k == (int)rank ? s_sel[1] : (long long)dsm_u64(&s_sel[1], k);
            if (k < (int)rank) tok_before += t;
            tot_tok += t;
            tot_sel += c;
        }
    } else {
        tot_tok = s_sel[0];
        tot_sel = s_sel[1];
    }
    trace(6);

    // ---- 6. token list (attention.py:469-496): sinks ++ buffer ++ selected members
    const int clen = qpos;
    const int ns = min(p.sink_end[seq], clen);
    const int bs = p.buffer_start[seq];
    const int nb = max(0, clen - bs);
    int32_t* T = p.tok + (size_t)l * p.tok_cap;
    if (rank == 0) {
        for (int j = tid; j < ns; j += kThreads)
            if (j < p.tok_cap) T[j] = j;
        for (int j = tid; j < nb; j += kThreads)
            if (ns + j < p.tok_cap) T[ns + j] = bs + j;
    }
    int* sel_c = reinterpret_cast<int*>(keys);
    int* sel_t = sel_c + Kc;
    const int per = (nloc + kThreads - 1) / kThreads;
    const int i0 = min(nloc, tid * per), i1 = min(nloc, i0 + per);
    unsigned long long mine = 0;
    for (int i = i0; i < i1; ++i)
        if (sflag[i]) mine += ((unsigned long long)sizes[i] << 32) | 1ull;
    unsigned long long tsum;
    const unsigned long long pre = scan_u64(mine, s_scan, &tsum);
    {
        int tpos = (int)(pre >> 32), spos = (int)(pre & 0xffffffffu);
        for (int i = i0; i < i1; ++i)
            if (sflag[i]) {
                sel_c[spos] = i;
                sel_t[spos] = tpos;
                ++spos;
                tpos += sizes[i];
            }
    }
    __syncthreads();
    const int nsel = (int)(tsum & 0xffffffffu), nsel_tok = (int)(tsum >> 32);
    const int32_t* mem = p.mem + (size_t)l * p.mem_cap;
    const int tbase = ns + nb + (int)tok_before;
    // member ids: every thread resolves kTokU tokens first, then issues their kTokU loads together
    constexpr int kTokU = 4;
    for (int j0 = tid; j0 < nsel_tok; j0 += kThreads * kTokU) {
        int src[kTokU];
#pragma unroll
        for (int u = 0; u < kTokU; ++u) {
            const int j = j0 + u * kThreads;
            src[u] = -1;
            if (j < nsel_tok) {
                int lo = 0, hi = nsel - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (sel_t[mid] <= j) lo = mid;
                    else hi = mid - 1;
                }
                src[u] = moff_s[sel_c[lo]] + (j - sel_t[lo]);
            }
        }
        int v[kTokU];
#pragma unroll
        for (int u = 0; u < kTokU; ++u) v[u] = src[u] >= 0 ? __ldg(mem + src[u]) : 0;
#pragma unroll
        for (int u = 0; u < kTokU; ++u) {
            const int slot = tbase + j0 + u * kThreads;
            if (src[u] >= 0 && slot < p.tok_cap) T[slot] = v[u];
        }
    }
    if (rank == 0 && tid == 0) {
        const long long ntok = ns + nb + tot_tok;
        p.stats[l] = (int32_t)min(ntok, (long long)p.tok_cap);
        p.stats[p.L + l] = p.replacement ? (int32_t)(n - tot_sel) : 0;
        p.stats[2 * p.L + l] = (int32_t)tot_tok;
        p.stats[3 * p.L + l] = (int32_t)tot_sel;
        if (p.sel_tokens) p.sel_tokens[l] = (int32_t)tot_tok;
    }
    // generic writes to the stage area (keys, lists, histograms) are ordered before the value
    // centroid TMA writes that reuse it
    fence_proxy_async_smem();
    __syncthreads();  // the list is complete (phase T reads it back); stage area free from here
    trace(7);

    if (C > 1) cl_sync();  // no CTA leaves while a peer may still read its shared memory
    if (p.k_new && p.ticket) {
        // the step's token is in the cache: the last CTA (every CTA has read cache_len) advances
        // the lengths
        __shared__ int s_last;
        if (tid == 0) {
            __threadfence();
            s_last = atomicAdd(p.ticket, 1) == (int)gridDim.x - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            for (int k = tid; k < p.n_seq; k += kThreads) p.cache_len[k] += 1;
            if (p.ntok_dense)
                for (int k = tid; k < p.L; k += kThreads) p.ntok_dense[k] += 1;
            if (tid == 0) *p.ticket = 0;
        }
    }
    trace(15);
}

}  // namespace stp
}  // namespace mpa

using namespace mpa;

// GQA group sizes 3..8 (the logits slot must also hold the weights, partials and token ids)
#define MPA_DISPATCH_G3(G, ...)                                                                     \
    switch (G) {                                                                                    \
        case 3: { constexpr int kG = 3; __VA_ARGS__; } break;                                      \
        case 4: { constexpr int kG = 4; __VA_ARGS__; } break;                                      \
        case 5: { constexpr int kG = 5; __VA_ARGS__; } break;                                      \
        case 6: { constexpr int kG = 6; __VA_ARGS__; } break;                                      \
        case 7: { constexpr int kG = 7; __VA_ARGS__; } break;                                      \
        case 8: { constexpr int kG = 8; __VA_ARGS__; } break;                                      \
        default: ::mpa::set_error("group size %d not supported (3..8)", (int)(G));                 \
                 return MPA_ERR_UNSUPPORTED;                                                        \
    }

static int encode_rows_map(CUtensorMap* out, const void* base, long long rows, int box_rows = stp::kChunk) {
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
    MPA_REQUIRE(rows > 0 && rows < (1ll << 31), MPA_ERR_UNSUPPORTED, "mpa_step: %lld centroid rows", rows);
    cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    const CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    MPA_REQUIRE(r == CUDA_SUCCESS, MPA_ERR_ARG, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return 0;
}

// cluster size: fill the SMs in one wave (C * L <= #SMs), enough CTAs for the shared-memory slice
// bound, at most what the device co-schedules (largest power of two <= 16)
template <int G>
static int pick_cluster_uncached(int L, int n_max, int* kc_out) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 1;
    const int chunks = ceil_div(n_max > 0 ? n_max : 1, stp::kChunk);
    constexpr int kcmax = stp::Geo<G>::kcmax;
    int C = 1;
    while (C < 16 && C * 2 * L <= sms && C * 2 <= chunks) C *= 2;
    while (C < 16 && ceil_div(chunks, C) * stp::kChunk > kcmax) C *= 2;
    auto kern = stp::step_kernel<G>;
    const int smem = stp::Geo<G>::total;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    while (C > 1) {  // every cluster of the grid co-resident (one wave), else smaller clusters
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C * L);
        cfg.blockDim = dim3(stp::kThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclus = 0;
        if (cudaOccupancyMaxActiveClusters(&nclus, kern, &cfg) == cudaSuccess && nclus >= L) break;
        cudaGetLastError();
        C /= 2;
    }
    *kc_out = ceil_div(chunks, C) * stp::kChunk;
    return C;
}

template <int G>
static int pick_cluster(int L, int n_max, int* kc_out) {
    // memo of the last few answers: the occupancy query costs host time per launch
    struct Memo { int L, chunks, dev, C, kc; };
    static Memo memo[8];
    static int nmemo = 0;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    const int chunks = ceil_div(n_max > 0 ? n_max : 1, stp::kChunk);
    for (int i = 0; i < nmemo && i < 8; ++i)
        if (memo[i].L == L && memo[i].chunks == chunks && memo[i].dev == dev) {
            *kc_out = memo[i].kc;
            return memo[i].C;
        }
    const int C = pick_cluster_uncached<G>(L, n_max, kc_out);
    memo[nmemo % 8] = Memo{L, chunks, dev, C, *kc_out};
    ++nmemo;
    return C;
}

#ifdef MPA_DEBUG_TRACE
extern "C" int mpa_debug_trace_step(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, stp::g_dbg_step, sizeof(unsigned long long) * n);
}
#endif

// whether mpa_decode_step can run n_ledgers ledgers of up to n_max centroids on this device: every
// cluster of the one-wave grid co-resident and each CTA's slice within its shared-memory schedule
extern "C" int mpa_decode_step_fits(int n_ledgers, int group, int n_max) {
    if (n_ledgers <= 0) return 1;
    if (group < 3 || group > 8) return 0;
    int ok = 0;
    [&]() -> int {
        MPA_DISPATCH_G3(group, {
            int kc = 0;
            const int C = pick_cluster<kG>(n_ledgers, n_max, &kc);
            ok = (size_t)C * kc >= (size_t)(n_max > 0 ? n_max : 1) && kc <= stp::Geo<kG>::kcmax;
        });
        return 0;
    }();
    return ok;
}

extern "C" int mpa_decode_step(const float* q, const float* k_new, const float* v_new, const mpa_cache* cache,
                               const double* cs_lk, const double* inv_freq, int n_kv_heads, int group,
                               const mpa_level* fine, const int64_t* budget, const int32_t* sink_end,
                               const int32_t* buffer_start, int32_t* cache_len, int32_t* ntok_dense,
                               int32_t* ticket, int replacement, uint8_t* flag, int32_t* sel_tokens, int32_t* tok,
                               int tok_cap, int32_t* stats, int n_max, float* q_rot, float* rej_w, int rej_cap,
                               void* stream) {
    const char* what = "mpa_decode_step";
    MPA_REQUIRE(q && cs_lk && inv_freq && cache && fine && fine->kc && fine->size && fine->count && fine->off &&
                    fine->idx && budget && sink_end && buffer_start && cache_len && flag && tok && stats,
                MPA_ERR_ARG, "%s: null argument", what);
    MPA_REQUIRE(cache->head_dim == 128 && cache->dtype == MPA_BF16 && fine->dtype == MPA_BF16, MPA_ERR_UNSUPPORTED,
                "%s: bf16 cache and centroids with head_dim 128 only", what);
    MPA_REQUIRE(group >= 3 && group <= 8, MPA_ERR_UNSUPPORTED, "%s: group %d (3..8)", what, group);
    MPA_REQUIRE(!k_new || (v_new && ticket), MPA_ERR_ARG, "%s: the append needs v_new and a ticket", what);
    MPA_REQUIRE(!rej_w || rej_cap >= fine->cap, MPA_ERR_ARG, "%s: rej_cap %d < cap %d", what, rej_cap, fine->cap);
    const int L = fine->n_ledgers;
    MPA_REQUIRE(cache->n_ledgers == L && n_kv_heads >= 1 && L % n_kv_heads == 0, MPA_ERR_ARG,
                "%s: %d ledgers vs cache %d / %d kv-heads", what, L, cache->n_ledgers, n_kv_heads);
    if (int rc = check_cache(cache, what)) return rc;
    MPA_REQUIRE(!cache->block_table || cache->n_kv_heads == n_kv_heads, MPA_ERR_ARG, "%s: paged cache kv-heads", what);
    if (L <= 0) return 0;
    if (n_max <= 0 || n_max > fine->cap) n_max = fine->cap;
    CUtensorMap tk;
    if (int rc = encode_rows_map(&tk, fine->kc, (long long)L * fine->cap)) return rc;
    MPA_DISPATCH_G3(group, {
        int kc = 0;
        const int C = pick_cluster<kG>(L, n_max, &kc);
        MPA_REQUIRE((size_t)C * kc >= (size_t)n_max && kc <= stp::Geo<kG>::kcmax, MPA_ERR_UNSUPPORTED,
                    "%s: %d centroids per ledger exceed 16 CTAs x %d", what, n_max, stp::Geo<kG>::kcmax);
        stp::Params prm = {};
        prm.q = q;
        prm.cs_lk = cs_lk;
        prm.inv_freq = inv_freq;
        prm.q_scale = 1.0f / sqrtf(128.0f);
        prm.count = fine->count;
        prm.size = fine->size;
        prm.moff = fine->off;
        prm.mem = fine->idx;
        prm.kcap = fine->cap;
        prm.mem_cap = fine->idx_cap;
        prm.budget = budget;
        prm.sink_end = sink_end;
        prm.buffer_start = buffer_start;
        prm.cache_len = cache_len;
        prm.n_kv_heads = n_kv_heads;
        prm.replacement = replacement;
        prm.L = L;
        prm.n_seq = L / n_kv_heads;
        prm.flag = flag;
        prm.sel_tokens = sel_tokens;
        prm.tok = tok;
        prm.tok_cap = tok_cap;
        prm.stats = stats;
        prm.kc = kc;
        prm.q_rot = q_rot;
        prm.rej_w = rej_w;
        prm.rej_cap = rej_cap;
        prm.k_rot = (__nv_bfloat16*)cache->k_rot;
        prm.k_raw = (__nv_bfloat16*)cache->k_raw;
        prm.vcache = (__nv_bfloat16*)cache->v;
        prm.tcap = cache->tcap;
        prm.kv = kv_rows(cache);
        prm.k_new = k_new;
        prm.v_new = v_new;
        prm.ntok_dense = ntok_dense;
        prm.ticket = ticket;
        auto kern = stp::step_kernel<kG>;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C * L);
        cfg.blockDim = dim3(stp::kThreads);
        cfg.dynamicSmemBytes = stp::Geo<kG>::total;
        cfg.stream = (cudaStream_t)stream;
        cudaLaunchAttribute at[2];
        int na = 0;
        if (C > 1) {
            at[na].id = cudaLaunchAttributeClusterDimension;
            at[na].val.clusterDim.x = C;
            at[na].val.clusterDim.y = 1;
            at[na].val.clusterDim.z = 1;
            ++na;
        }
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
        cfg.attrs = at;
        cfg.numAttrs = na;
        cudaLaunchKernelEx(&cfg, kern, tk, prm);
    });
    return check_launch(what);
}

// Point a captured step graph's decode-step kernel at new q / k_new / v_new buffers (the graph node's
// parameters in the instantiated graph; everything else stays as captured), so a caller's device
// tensors feed the step without a staging copy.
extern "C" int mpa_decode_step_rebind(void* graph, void* graph_exec, const float* q, const float* k_new,
                                      const float* v_new) {
    MPA_REQUIRE(graph && graph_exec && q, MPA_ERR_ARG, "mpa_decode_step_rebind: null argument");
    MPA_REQUIRE(((uintptr_t)q & 15) == 0 && ((uintptr_t)k_new & 15) == 0 && ((uintptr_t)v_new & 15) == 0,
                MPA_ERR_ARG, "mpa_decode_step_rebind: buffers must be 16-byte aligned");
    const void* kerns[6] = {(const void*)stp::step_kernel<3>, (const void*)stp::step_kernel<4>,
                            (const void*)stp::step_kernel<5>, (const void*)stp::step_kernel<6>,
                            (const void*)stp::step_kernel<7>, (const void*)stp::step_kernel<8>};
    size_t n = 0;
    cudaError_t e = cudaGraphGetNodes((cudaGraph_t)graph, nullptr, &n);
    MPA_REQUIRE(e == cudaSuccess, (int)e, "mpa_decode_step_rebind: %s", cudaGetErrorString(e));
    cudaGraphNode_t nodes[64];
    MPA_REQUIRE(n <= 64, MPA_ERR_UNSUPPORTED, "mpa_decode_step_rebind: %zu graph nodes", n);
    e = cudaGraphGetNodes((cudaGraph_t)graph, nodes, &n);
    MPA_REQUIRE(e == cudaSuccess, (int)e, "mpa_decode_step_rebind: %s", cudaGetErrorString(e));
    int found = 0;
    for (size_t i = 0; i < n; ++i) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nodes[i], &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp;
        if (cudaGraphKernelNodeGetParams(nodes[i], &kp) != cudaSuccess) continue;
        bool step = false;
        for (const void* k : kerns) step |= kp.func == k;
        if (!step) continue;
        CUtensorMap tk = *static_cast<const CUtensorMap*>(kp.kernelParams[0]);
        stp::Params prm = *static_cast<const stp::Params*>(kp.kernelParams[1]);
        MPA_REQUIRE(!prm.k_new == !k_new, MPA_ERR_ARG, "mpa_decode_step_rebind: the graph %s the append",
                    prm.k_new ? "has" : "has no");
        prm.q = q;
        prm.k_new = k_new;
        prm.v_new = v_new;
        void* args[2] = {&tk, &prm};
        kp.kernelParams = args;
        kp.extra = nullptr;
        e = cudaGraphExecKernelNodeSetParams((cudaGraphExec_t)graph_exec, nodes[i], &kp);
        MPA_REQUIRE(e == cudaSuccess, (int)e, "mpa_decode_step_rebind: %s", cudaGetErrorString(e));
        ++found;
    }
    MPA_REQUIRE(found == 1, MPA_ERR_ARG, "mpa_decode_step_rebind: %d decode-step kernels in the graph", found);
    return 0;
}
