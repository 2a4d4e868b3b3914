// K11 + K12: fused sparse decode with in-kernel split-KV (flash-decoding) merge.
//
// Reference (pkg/src/multipole_attn/attention.py):
//   :58-68   `_partial_from_logits`  m = max l, w = exp(l - m) (* N), s = sum w, a = w @ V
//   :71-87   `exact_partial`         logits = rot(q, cache_len) . rot(k, pos) / sqrt(d)
//   :120-137 `sparse_exact_partial`  same over the selected token ids
//   :210-227 `centroid_replacement_partial`  weight N * exp(lookup logit) on the value centroid
//   :230-239 `merge_partials` + :44-47 `finalize`
//   :473-498 one q-head: merge(sinks, buffer, selected, fine rejected, coarse rejected)
//   :90-102  `exact_attention`  dense oracle (tok == NULL here)
//
// One online softmax per q-head covers every item of a ledger (kv-head): exact tokens
// (K_rot / V rows gathered by index) and rejected-centroid pseudo-tokens (logit + ln N,
// value centroid).  Partials of one ledger are LSE-merged by whoever finishes it last
// (atomic ticket), so a step needs no separate merge launch.
//
// Two implementations:
//   * decode_sk_kernel (bf16, d in {64,128}, G <= 8) -- the serving path.  A persistent,
//     stream-K scheduled grid (one wave: SMs x resident CTAs) walks the concatenated 16-item
//     tiles of ALL ledgers; CTA c owns a contiguous, byte-balanced range of that tile space
//     (a token tile costs 2 units -- K and V rows --, a centroid tile 1), so the work per CTA
//     is equal whatever the batch, budget or selection.  Each warp owns a ring of NST stages
//     and streams its tiles (every NW-th tile of the CTA range) through it with one
//     cp.async.bulk (TMA bulk engine, UBLKCP) per 256-byte row, completing on an mbarrier,
//     so each warp keeps NST-1 tiles of gathers in flight with two instructions of issue
//     cost.  Rows land in padded (272-byte) smem rows, conflict-free for ldmatrix.
//     S = K q^T and O^T += V^T P^T run on the tensor cores (mma.sync m16n8k16, tokens on M,
//     q-heads on N=8); q and P are split into bf16 hi + lo parts packed into the 8 MMA
//     columns (G <= 4) so the only bf16 rounding left is the KV cache itself.  Base-2 online
//     softmax with a lazy (threshold 2^8) rescale.  A warp writes one partial per ledger it
//     touched; the last arriving warp of a ledger merges them.
//   * decode_ffma_kernel (any dtype, any even d): warp per item, FFMA, natural-log softmax,
//     fp32 accurate expf, n_split CTAs per ledger -- the fp32 parity mode (1e-5).
#include <cuda.h>

#include <climits>
#include <cstdlib>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "mpa_common.cuh"

namespace mpa {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// padded logit stride of the rejected-centroid list (rej_w rows): 4 floats for G <= 4, else 8
__host__ __device__ constexpr int rej_stride(int G) { return G <= 4 ? 4 : 8; }

// ============================================================================
// FFMA path (split_range over n_split CTAs per ledger)

// Item range of split s of a ledger: tokens cost 2 units (K + V rows), centroids 1 unit.
struct SplitRange {
    int t0, t1, r0, r1;
};

__device__ __forceinline__ SplitRange split_range(int nt, int nr, int s, int S) {
    const long long U = 2ll * nt + nr;
    const long long u0 = U * s / S, u1 = U * (s + 1) / S;
    SplitRange r;
    r.t0 = (int)min((long long)nt, (u0 + 1) / 2);
    r.t1 = (int)min((long long)nt, (u1 + 1) / 2);
    r.r0 = (int)min((long long)nr, max(0ll, u0 - 2ll * nt));
    r.r1 = (int)min((long long)nr, max(0ll, u1 - 2ll * nt));
    return r;
}

// A ledger's result: out = a / s, or (part_out != NULL, sequence-sharded decode) its unnormalised
// partial [m (natural-log units), s, a[d]] per q-head for the cross-rank merge.
__device__ __forceinline__ void emit_result(float* out, float* part_out, int l, int G, int d, int g, int k, float m_nat,
                                            float s, float a) {
    if (part_out) {
        float* P = part_out + ((size_t)l * G + g) * (d + 2);
        if (k == 0) {
            P[0] = m_nat;
            P[1] = s;
        }
        P[2 + k] = a;
    } else {
        out[((size_t)l * G + g) * d + k] = a / s;
    }
}

// Last-CTA merge of the n_split partials of ledger l.
__device__ void merge_splits(int l, int S, int G, int d, const float* part_ml, const float* part_acc, float* out,
                             float* part_out) {
    for (int idx = threadIdx.x; idx < G * d; idx += blockDim.x) {
        const int g = idx / d, k = idx - g * d;
        float M = -INFINITY;
        for (int s = 0; s < S; ++s) M = fmaxf(M, __ldcg(part_ml + (((size_t)l * S + s) * G + g) * 2));
        float sum = 0.f, acc = 0.f;
        if (M != -INFINITY) {
            for (int s = 0; s < S; ++s) {
                const float m = __ldcg(part_ml + (((size_t)l * S + s) * G + g) * 2);
                if (m == -INFINITY) continue;
                const float w = expf(m - M);
                sum += w * __ldcg(part_ml + (((size_t)l * S + s) * G + g) * 2 + 1);
                acc += w * __ldcg(part_acc + (((size_t)l * S + s) * G + g) * d + k);
            }
        }
        emit_result(out, part_out, l, G, d, g, k, M, sum, acc);
    }
}

// Publishes this CTA's partial and returns true in the CTA that must merge.
__device__ __forceinline__ bool take_ticket(int32_t* ticket, int l, int S) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(ticket + l, 1);
        s_last = (prev == S - 1);
        if (s_last) ticket[l] = 0;  // ready for the next launch / graph replay
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

constexpr int kFfmaWarps = 4;

template <typename T, int G, int NDL>
__global__ void __launch_bounds__(kFfmaWarps * 32)
decode_ffma_kernel(const T* __restrict__ k_rot, const T* __restrict__ vcache, KvRows kvr, int d,
                   const float* __restrict__ q_rot, const int32_t* __restrict__ tok, const int32_t* __restrict__ n_tok,
                   int tok_cap, const int32_t* __restrict__ rej, const float* __restrict__ rej_w,
                   const int32_t* __restrict__ n_rej, int rej_cap, const T* __restrict__ fvc, int fcap,
                   const T* __restrict__ cvc, int ccap, int S, float* __restrict__ part_ml,
                   float* __restrict__ part_acc, int32_t* __restrict__ ticket, float* __restrict__ out,
                   float* __restrict__ part_out) {
    constexpr int GP = rej_stride(G);
    extern __shared__ float sm[];  // [warps][G][2 + d]
    const int l = blockIdx.y, s = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nt = n_tok[l], nr = rej ? n_rej[l] : 0;
    const SplitRange R = split_range(nt, nr, s, S);

    float q[G][NDL];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < NDL; ++j) {
            const int k = lane + 32 * j;
            q[g][j] = k < d ? q_rot[((size_t)l * G + g) * d + k] : 0.f;
        }
    float m[G], ssum[G], acc[G][NDL];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        m[g] = -INFINITY;
        ssum[g] = 0.f;
#pragma unroll
        for (int j = 0; j < NDL; ++j) acc[g][j] = 0.f;
    }
    auto absorb = [&](const float (&x)[G], const float (&v)[NDL]) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float mn = fmaxf(m[g], x[g]);
            const float c = expf(m[g] - mn);
            const float p = expf(x[g] - mn);
            m[g] = mn;
            ssum[g] = ssum[g] * c + p;
#pragma unroll
            for (int j = 0; j < NDL; ++j) acc[g][j] = fmaf(p, v[j], acc[g][j] * c);
        }
    };

    for (int t = R.t0 + w; t < R.t1; t += kFfmaWarps) {
        const int row = tok ? tok[(size_t)l * tok_cap + t] : t;
        const T* kp = k_rot + (size_t)kvr.row(l, row) * d;
        const T* vp = vcache + (size_t)kvr.row(l, row) * d;
        float kx[NDL], vx[NDL];
#pragma unroll
        for (int j = 0; j < NDL; ++j) {
            const int k = lane + 32 * j;
            kx[j] = k < d ? elem<T>::to_f(kp[k]) : 0.f;
            vx[j] = k < d ? elem<T>::to_f(vp[k]) : 0.f;
        }
        float x[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float dot = 0.f;
#pragma unroll
            for (int j = 0; j < NDL; ++j) dot = fmaf(q[g][j], kx[j], dot);
            x[g] = warp_sum(dot);
        }
        absorb(x, vx);
    }
    for (int r = R.r0 + w; r < R.r1; r += kFfmaWarps) {
        const int code = rej[(size_t)l * rej_cap + r];
        const T* vp = code >= 0 ? fvc + ((size_t)l * fcap + code) * d : cvc + ((size_t)l * ccap + (-1 - code)) * d;
        float vx[NDL], x[G];
#pragma unroll
        for (int j = 0; j < NDL; ++j) {
            const int k = lane + 32 * j;
            vx[j] = k < d ? elem<T>::to_f(vp[k]) : 0.f;
        }
#pragma unroll
        for (int g = 0; g < G; ++g) x[g] = rej_w[((size_t)l * rej_cap + r) * GP + g];
        absorb(x, vx);
    }

    // warp partials -> smem -> CTA partial
    float* mine = sm + (size_t)w * G * (2 + d);
#pragma unroll
    for (int g = 0; g < G; ++g) {
        if (lane == 0) {
            mine[g * (2 + d)] = m[g];
            mine[g * (2 + d) + 1] = ssum[g];
        }
#pragma unroll
        for (int j = 0; j < NDL; ++j) {
            const int k = lane + 32 * j;
            if (k < d) mine[g * (2 + d) + 2 + k] = acc[g][j];
        }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < G * d; idx += blockDim.x) {
        const int g = idx / d, k = idx - g * d;
        float M = -INFINITY;
        for (int ww = 0; ww < kFfmaWarps; ++ww) M = fmaxf(M, sm[((size_t)ww * G + g) * (2 + d)]);
        float sum = 0.f, a = 0.f;
        if (M != -INFINITY)
            for (int ww = 0; ww < kFfmaWarps; ++ww) {
                const float* p = sm + ((size_t)ww * G + g) * (2 + d);
                if (p[0] == -INFINITY) continue;
                const float c = expf(p[0] - M);
                sum += c * p[1];
                a += c * p[2 + k];
            }
        part_acc[(((size_t)l * S + s) * G + g) * d + k] = a;
        if (k == 0) {
            part_ml[(((size_t)l * S + s) * G + g) * 2] = M;
            part_ml[(((size_t)l * S + s) * G + g) * 2 + 1] = sum;
        }
    }
    if (take_ticket(ticket, l, S)) merge_splits(l, S, G, d, part_ml, part_acc, out, part_out);
}

// ============================================================================
// Tensor-core stream-K path (bf16)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// one TMA bulk copy global -> this CTA's shared memory, completing on an mbarrier; KV rows are
// streamed once per step, so they are marked evict-first in L2
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}
// TMA tile::gather4: rows r0..r3, columns [col, col + 64) of a 2D bf16 map (box 64 x 1, 128B
// swizzle) -> 4 x 128 B at dst (sm_100a)
__device__ __forceinline__ void tma_gather4(unsigned dst, const CUtensorMap* map, int col, int r0, int r1, int r2,
                                            int r3, unsigned bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar), "l"(policy)
        : "memory");
}
// one box (1 row x 64 columns) of the same map
__device__ __forceinline__ void tma_row(unsigned dst, const CUtensorMap* map, int col, int row, unsigned bar,
                                        uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(row), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    unsigned pred = 0;
    asm volatile("{\n .reg .b32 rx;\n .reg .pred px;\n elect.sync rx|px, %1;\n selp.b32 %0, 1, 0, px;\n}\n"
                 : "+r"(pred)
                 : "r"(0xffffffffu));
    return pred != 0;
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ void cp_async4(unsigned dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async16_hint(unsigned dst, const void* src, uint64_t policy) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "l"(policy)
                 : "memory");
}
// arrive on the mbarrier once this thread's cp.async copies so far have landed (pending count +1 now)
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive1(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

__device__ __forceinline__ void ldsm_x4(unsigned addr, unsigned (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(unsigned addr, unsigned (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ unsigned movm_t(unsigned x) {
    unsigned y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ unsigned pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<unsigned*>(&v);
}
__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// Stream-K schedule over the concatenated tiles of all ledgers.  Ledger l owns tiles
// [tp[l], tp[l+1]): ceil(nt/16) token tiles (16 tokens: K + V rows, 8 KB) then ceil(nr/32)
// centroid tiles (32 value centroids, 8 KB, + their logits) -- equal bytes, so equal cost; an
// empty ledger gets one empty token tile so that every ledger is finalised.  CTA c of Ce owns
// tiles [T c / Ce, T (c+1) / Ce) of the T = tp[L] total.
constexpr int kMinTiles = 16;  // minimum tiles per CTA (small batches use fewer CTAs)

#ifdef MPA_DEBUG_TRACE
// per-CTA phase timestamps (globaltimer ns) for timeline experiments: [cta][8]
__device__ unsigned long long g_dbg[4096 * 8];
__device__ __forceinline__ void dbg_stamp(int slot) {
    if (threadIdx.x == 0 && blockIdx.x < 4096) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_dbg[blockIdx.x * 8 + slot] = t;
    }
}
#else
__device__ __forceinline__ void dbg_stamp(int) {}
#endif
#ifdef MPA_DEBUG_RAMP  // slots 5-7 time the pipeline ramp instead of the segment merge
#define DBG_SEG(k)
#define DBG_RAMP(k) dbg_stamp(k)
#else
#define DBG_SEG(k) dbg_stamp(k)
#define DBG_RAMP(k)
#endif

// byte offset of 16-byte chunk ch of row r in a TMA 128B-swizzled 16-row tile (64-column halves)
__device__ __forceinline__ unsigned swz(int r, int ch) {
    return (unsigned)((ch >> 3) * 2048 + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
}

template <int G, int D, int NW, int NST>
struct SkGeom {
    static constexpr int kHalves = D / 64;           // 64-column halves per row
    static constexpr int kMatB = 16 * D * 2;         // one 16-row K or V tile
    static constexpr int kLgB = 32 * rej_stride(G) * 4;  // centroid-tile logits
    static constexpr int kStageB = 2 * kMatB;        // K + V (token tile) or 2 x V (centroid tile)
    static constexpr int kWarpB = NST * kStageB;
    static constexpr int kStagesB = NW * kWarpB;
    static constexpr int kLgAllB = NW * NST * kLgB;  // logits of every stage, after the tiles
    static constexpr int kBarB = NW * NST * 8 + kLgAllB;
    static constexpr int kRing = 4;                  // row-id ring: tiles whose ids are in smem
    static constexpr int kIdB = NW * kRing * 32 * 4;
    static constexpr int kPS = G * (D + 2);          // floats per partial
    // 2 CTAs / SM for G <= 8 at L <= 128 ledgers (tp + per-ledger counts: 3 L + 1 ints); the
    // dynamic window is 1024-aligned (the kernel checks), so no alignment slack is reserved
    static size_t smem(int L, int C) { (void)C; return (size_t)kStagesB + kBarB + kIdB + sizeof(int) * (3 * L + 1); }
};

template <int G, int D, int NW, int NST, bool PAGED>
__global__ void __launch_bounds__(NW * 32, 2)
decode_sk_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                 const __grid_constant__ CUtensorMap tm_fvc, const __grid_constant__ CUtensorMap tm_cvc,
                 const __grid_constant__ CUtensorMap tm_fvc16, KvRows kvr, const __nv_bfloat16* __restrict__ k_rows,
                 const __nv_bfloat16* __restrict__ v_rows,
                 const float* __restrict__ q_rot, const int32_t* __restrict__ tok, const int32_t* __restrict__ n_tok,
                 int tok_cap, const int32_t* __restrict__ rej, const float* __restrict__ rej_w,
                 const int32_t* __restrict__ n_rej, int rej_cap, int fcap, int ccap, int L, float* __restrict__ part,
                 int32_t* __restrict__ ticket, float* __restrict__ out, float* __restrict__ part_out, int tok_lsu) {
    dbg_stamp(0);
    using Geo = SkGeom<G, D, NW, NST>;
    constexpr bool PACKED = G <= 4;
    constexpr int KS = D / 16;  // k-steps for QK, m-tiles for PV
    constexpr int GP = rej_stride(G);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    if (smem_u32(smem_raw) & 1023) __trap();  // SWIZZLE_128B stages need the 1024-aligned window
    unsigned char* smem = smem_raw;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gr = lane >> 2, tq = lane & 3;
    const int C = gridDim.x, c = blockIdx.x;
    // centroid terms: listed rows (rej), every fine centroid in order (rej == NULL, rej_w: the
    // contiguous-centroid list, selected ones weighted -inf), or none
    const bool has_rej = rej || rej_w;

    // ---- per-ledger tile prefix sum (every CTA computes the same schedule)
    int* tp = reinterpret_cast<int*>(smem + Geo::kStagesB + Geo::kBarB + Geo::kIdB);
    int* idring = reinterpret_cast<int*>(smem + Geo::kStagesB + Geo::kBarB) + w * Geo::kRing * 32;
    int* cnt_s = tp + (L + 1);  // [L][2] token / centroid counts
    if (threadIdx.x == 0) {  // before the PDL wait: nothing here depends on the selection
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_k)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_v)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_fvc)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_cvc)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_fvc16)) : "memory");
    }
    pdl_wait();  // work lists, counts and weights come from the selection kernel
    pdl_trigger();
    {
        __shared__ int scan[33];
        int base = 0;
        for (int l0 = 0; l0 < L; l0 += blockDim.x) {
            const int l = l0 + threadIdx.x;
            int n = 0;
            if (l < L) {
                const int ct = __ldg(n_tok + l), cr = has_rej ? __ldg(n_rej + l) : 0;
                cnt_s[2 * l] = ct;  // the walkers read the counts from here, not from global
                cnt_s[2 * l + 1] = cr;
                const int nt = (ct + 15) >> 4, nr = (cr + 31) >> 5;
                n = nt + nr > 0 ? nt + nr : 1;
            }
            int tot;
            const int e = block_exclusive_scan(n, scan, &tot);
            if (l < L) tp[l] = base + e;
            base += tot;
        }
        if (threadIdx.x == 0) tp[L] = base;
    }
    const unsigned bar0 = smem_u32(smem + Geo::kStagesB + Geo::kLgAllB) + w * NST * 8;
    const unsigned lgbase = smem_u32(smem + Geo::kStagesB) + w * NST * Geo::kLgB;
    if (lane == 0)
        for (int s = 0; s < NST; ++s) mbar_init(bar0 + s * 8, 1);
    fence_mbar_init();
    __syncthreads();
    const int T = tp[L];
    const int Ce = max(1, min(C, T / kMinTiles));
    if (c >= Ce) return;  // surplus CTA: no CTA-wide barrier follows for it
    auto cbt_at = [&](int cc) -> int { return (int)((long long)T * cc / Ce); };  // first tile of CTA cc
    dbg_stamp(1);
    auto cta_begin = [&](int cc) -> int { return cbt_at(cc); };
    auto ledger_of_tile = [&](int g) -> int {  // largest l with tp[l] <= g
        int lo = 0, hi = L - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tp[mid] <= g) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    };
    const int g0 = cta_begin(c), g1 = cta_begin(c + 1);
    const int my_n = g1 - g0 > w ? (g1 - g0 - w + NW - 1) / NW : 0;
    const unsigned wbase = smem_u32(smem) + w * Geo::kWarpB;
    const uint64_t policy = evict_first_policy();

    // ---- tile metadata for this warp's i-th tile (global tile g0 + w + i*NW)
    struct Meta {
        int l, kind, i0, nv;  // ledger, 0 token / 1 centroid, first item, valid rows
    };
    struct Walker {  // walks this warp's tiles in order, caching the current ledger's counts
        int l, beg, end, nt, nr, ntt;
    };
    auto meta_of = [&](int i, Walker& wk) -> Meta {
        const int g = g0 + w + i * NW;
        if (wk.l < 0 || g >= wk.end) {
            int l = wk.l < 0 ? ledger_of_tile(g) : wk.l;
            while (l + 1 < L && tp[l + 1] <= g) ++l;
            wk.l = l;
            wk.beg = tp[l];
            wk.end = tp[l + 1];
            wk.nt = cnt_s[2 * l];
            wk.nr = cnt_s[2 * l + 1];
            wk.ntt = (wk.nt + 15) >> 4;
            if (wk.ntt == 0 && wk.nr == 0) wk.ntt = 1;  // empty ledger: one empty token tile
        }
        const int t = g - wk.beg;
        Meta m;
        m.l = wk.l;
        if (t < wk.ntt) {
            m.kind = 0;
            m.i0 = t * 16;
            m.nv = max(0, min(16, wk.nt - m.i0));
        } else {
            m.kind = 1;
            m.i0 = (t - wk.ntt) * 32;
            m.nv = min(32, wk.nr - m.i0);
        }
        return m;
    };
    // row ids reach smem kRing-1 tiles before their gathers are issued (cp.async, one per lane);
    // padding rows repeat row 0
    constexpr int kAhead = Geo::kRing - 1;
    auto prefetch_ids = [&](int j, const Meta& m) {
        const int rows = m.kind == 0 ? 16 : 32;
        if (PAGED && m.kind == 0 && !tok && kvr.ps_shift >= 4) {
            // dense tile of a paged cache: 16 consecutive tokens inside one page -- its page id
            if (lane == 0 && m.nv > 0)
                cp_async4(smem_u32(idring + (j % Geo::kRing) * 32),
                          kvr.bt + (size_t)(m.l / kvr.hkv) * kvr.ppl + (m.i0 >> kvr.ps_shift));
        } else if (lane < rows && m.nv > 0 && (m.kind == 1 ? rej != nullptr : tok != nullptr)) {
            const int row = lane < m.nv ? lane : 0;
            const int32_t* src = m.kind == 0 ? tok + (size_t)m.l * tok_cap + m.i0 + row
                                             : rej + (size_t)m.l * rej_cap + m.i0 + row;
            cp_async4(smem_u32(idring + (j % Geo::kRing) * 32 + lane), src);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    // ids of rows [r0, r0 + 16) of tile j; every lane reads the same smem words and the values
    // are broadcast from lane 0 so the compiler keeps them in uniform registers
    // token ids; a paged cache's token tiles get their pool rows here (lane r translates token r
    // through the block table, the rows are broadcast back), a flat cache adds l * tcap at the copy
    auto ids16 = [&](int j, const Meta& m, int r0, int (&id)[16]) {
        if (m.kind == 0 && !tok) {
#pragma unroll
            for (int r = 0; r < 16; ++r) id[r] = m.i0 + (r < m.nv ? r : 0);
        } else {
            const int4* q4 = reinterpret_cast<const int4*>(idring + (j % Geo::kRing) * 32 + r0);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int4 t = q4[v];
                id[4 * v] = __shfl_sync(0xffffffffu, t.x, 0);
                id[4 * v + 1] = __shfl_sync(0xffffffffu, t.y, 0);
                id[4 * v + 2] = __shfl_sync(0xffffffffu, t.z, 0);
                id[4 * v + 3] = __shfl_sync(0xffffffffu, t.w, 0);
            }
        }
        if constexpr (PAGED) {
            if (m.kind == 0 && !tok && kvr.ps_shift >= 4) {
                const int page = idring[(j % Geo::kRing) * 32];
                const int h = m.l % kvr.hkv, base = (page * kvr.hkv + h) << kvr.ps_shift;
                const int mask = (1 << kvr.ps_shift) - 1;
#pragma unroll
                for (int r = 0; r < 16; ++r) id[r] = base + ((m.i0 + (r < m.nv ? r : 0)) & mask);
            } else if (m.kind == 0) {  // token list: lane r translates token r (read back from the ring)
                int mine = tok ? idring[(j % Geo::kRing) * 32 + r0 + (lane & 15)] : m.i0 + min(lane & 15, m.nv - 1);
                mine = kvr.row(m.l, mine);
#pragma unroll
                for (int r = 0; r < 16; ++r) id[r] = __shfl_sync(0xffffffffu, mine, r);
            }
        }
    };
    // gathers of 16 value-centroid rows (codes >= 0 fine, < 0 coarse) into one 16-row tile; a
    // group of 4 that straddles the fine -> coarse boundary of the list uses one 2D tile copy
    // (box 1 row x 64 columns) per row
    auto gather_centroids = [&](unsigned dst, const int (&id)[16], int l, unsigned bar) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int a0 = id[4 * q], a1 = id[4 * q + 1], a2 = id[4 * q + 2], a3 = id[4 * q + 3];
            const bool fine = a0 >= 0 && a1 >= 0 && a2 >= 0 && a3 >= 0;
            const bool coarse = a0 < 0 && a1 < 0 && a2 < 0 && a3 < 0;
#pragma unroll
            for (int h = 0; h < Geo::kHalves; ++h) {
                const unsigned off = dst + h * 2048 + q * 512;
                if (fine) {
                    const int fb = l * fcap;
                    tma_gather4(off, &tm_fvc, h * 64, fb + a0, fb + a1, fb + a2, fb + a3, bar, policy);
                } else if (coarse) {
                    const int cb = l * ccap - 1;
                    tma_gather4(off, &tm_cvc, h * 64, cb - a0, cb - a1, cb - a2, cb - a3, bar, policy);
                } else {
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int a = id[4 * q + r];
                        if (a >= 0) tma_row(off + r * 128, &tm_fvc, h * 64, l * fcap + a, bar, policy);
                        else tma_row(off + r * 128, &tm_cvc, h * 64, l * ccap - 1 - a, bar, policy);
                    }
                }
            }
        }
    };
    auto issue = [&](int j, int st, const Meta& m) {
        const unsigned kst = wbase + st * Geo::kStageB, vst = kst + Geo::kMatB, lgs = lgbase + st * Geo::kLgB;
        const unsigned bar = bar0 + st * 8;
        (void)lgs;
        int id[16], id2[16];
        const bool rows_in_order = m.kind == 1 && !rej;  // contiguous-centroid list
        if (m.nv > 0 && !rows_in_order) {
            ids16(j, m, 0, id);
            if (m.kind == 1) ids16(j, m, 16, id2);
        }
        if (m.kind == 0 && m.nv > 0 && tok_lsu) {
            // token tile through the LSU: every lane copies 16-byte chunks (row r, K or V, chunk
            // ch) straight into the swizzled stage -- 2 x 256 B rows per warp instruction, which
            // the TMA unit would need 4 gather4 instructions for; completion on the stage mbarrier
            constexpr int CPR = D / 8;  // 16-byte chunks per row
            const size_t lbase = PAGED ? 0 : (size_t)m.l * kvr.tcap;
#pragma unroll
            for (int it = 0; it < CPR; ++it) {
                const int jj = lane + 32 * it, ch = jj % CPR, kv = (jj / CPR) & 1, r = jj / (2 * CPR);
                // row index with compile-time register indices (r0 constant, +1 for the upper lanes at d = 64)
                constexpr int kRowsPerIt = 32 / (2 * CPR);
                const int r0 = it * kRowsPerIt;
                int rid = id[r0];
                if constexpr (kRowsPerIt > 1) {
                    if (lane >= 2 * CPR) rid = id[r0 + 1];
                }
                const __nv_bfloat16* src = (kv ? v_rows : k_rows) + (lbase + rid) * D + ch * 8;
                cp_async16_hint((kv ? vst : kst) + swz(r, ch), src, policy);
            }
            cp_async_mbar_arrive(bar);
            __syncwarp();
            if (elect_one()) mbar_arrive1(bar);  // the phase's one expected arrival
            return;
        }
        __syncwarp();
        if (!elect_one()) return;
        fence_proxy_async();  // generic reads of this stage (previous tile) before the async writes
        if (m.nv <= 0) {
            mbar_expect_tx(bar, 0);
            return;
        }
        if (m.kind == 0) {
            mbar_expect_tx(bar, 2 * Geo::kMatB);
            const int base = PAGED ? 0 : m.l * kvr.tcap;
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int h = 0; h < Geo::kHalves; ++h) {
                    const unsigned off = h * 2048 + q * 512;
                    tma_gather4(kst + off, &tm_k, h * 64, base + id[4 * q], base + id[4 * q + 1],
                                base + id[4 * q + 2], base + id[4 * q + 3], bar, policy);
                    tma_gather4(vst + off, &tm_v, h * 64, base + id[4 * q], base + id[4 * q + 1],
                                base + id[4 * q + 2], base + id[4 * q + 3], bar, policy);
                }
        } else {
            const unsigned lg_bytes = m.nv * GP * 4;
            mbar_expect_tx(bar, 2 * Geo::kMatB + lg_bytes);
            if (rows_in_order) {
                const int row0 = m.l * fcap + m.i0;
#pragma unroll
                for (int h = 0; h < Geo::kHalves; ++h) {
                    tma_row(kst + h * 2048, &tm_fvc16, h * 64, row0, bar, policy);
                    tma_row(vst + h * 2048, &tm_fvc16, h * 64, row0 + 16, bar, policy);
                }
            } else {
                gather_centroids(kst, id, m.l, bar);
                gather_centroids(vst, id2, m.l, bar);
            }
            bulk_g2s(lgs, rej_w + ((size_t)m.l * rej_cap + m.i0) * GP, lg_bytes, bar, policy);
        }
    };

    // ---- per-ledger softmax state
    unsigned qhi[KS][2], qlo[PACKED ? 1 : KS][2];
    const int hA = PACKED ? 2 * (tq & 1) : 2 * tq, hB = hA + 1;
    float mA, mB, sA, sB;
    float o[KS][4];
    float o2[PACKED ? 1 : KS][4];
    auto reset_state = [&]() {
        mA = mB = -INFINITY;
        sA = sB = 0.f;
#pragma unroll
        for (int i = 0; i < KS; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) o[i][j] = 0.f;
        if (!PACKED) {
#pragma unroll
            for (int i = 0; i < (PACKED ? 1 : KS); ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) o2[i][j] = 0.f;
        }
    };
    auto load_q = [&](int l) {
        auto qv = [&](int head, int k) -> float {
            return head < G ? __ldg(q_rot + ((size_t)l * G + head) * D + k) * kLog2e : 0.f;
        };
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int k = ks * 16 + 2 * tq + 8 * half;
                if (PACKED) {
                    const int head = gr & 3;
                    const float a = qv(head, k), b = qv(head, k + 1);
                    const float ah = bf16_round(a), bh = bf16_round(b);
                    qhi[ks][half] = gr < 4 ? pack_bf16(ah, bh) : pack_bf16(a - ah, b - bh);
                } else {
                    const float a = qv(gr, k), b = qv(gr, k + 1);
                    const float ah = bf16_round(a), bh = bf16_round(b);
                    qhi[ks][half] = pack_bf16(ah, bh);
                    qlo[PACKED ? 0 : ks][half] = pack_bf16(a - ah, b - bh);
                }
            }
        }
    };

    // online softmax (column = head) + O^T += V^T P^T over 16 rows with logits x (log2 units,
    // rows gr / gr+8, heads hA / hB); the reference max only moves when a tile exceeds it by
    // more than 2^8, so most tiles skip the accumulator rescale
    auto absorb16 = [&](float (&x)[4], unsigned vtile) {
        if (hA >= G) { x[0] = x[0] == -INFINITY ? -INFINITY : 0.f; x[2] = x[2] == -INFINITY ? -INFINITY : 0.f; }
        if (hB >= G) { x[1] = x[1] == -INFINITY ? -INFINITY : 0.f; x[3] = x[3] == -INFINITY ? -INFINITY : 0.f; }
        float tA = fmaxf(x[0], x[2]), tB = fmaxf(x[1], x[3]);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, off));
            tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, off));
        }
        const bool upA = tA > mA + 8.f, upB = tB > mB + 8.f;
        if (__any_sync(0xffffffffu, upA || upB)) {
            const float nA = upA ? tA : mA, nB = upB ? tB : mB;
            const float cA = exp2f(mA - nA), cB = exp2f(mB - nB);  // mA = -inf -> 0
            mA = nA;
            mB = nB;
            sA *= cA;
            sB *= cB;
#pragma unroll
            for (int mt = 0; mt < KS; ++mt) {
                o[mt][0] *= cA; o[mt][1] *= cB; o[mt][2] *= cA; o[mt][3] *= cB;
                if (!PACKED) {
                    o2[PACKED ? 0 : mt][0] *= cA; o2[PACKED ? 0 : mt][1] *= cB;
                    o2[PACKED ? 0 : mt][2] *= cA; o2[PACKED ? 0 : mt][3] *= cB;
                }
            }
        }
        // masked rows (-inf) weigh exactly 0, also while the running max is still -inf
        const float p0 = x[0] == -INFINITY ? 0.f : exp2f(x[0] - mA), p1 = x[1] == -INFINITY ? 0.f : exp2f(x[1] - mB);
        const float p2 = x[2] == -INFINITY ? 0.f : exp2f(x[2] - mA), p3 = x[3] == -INFINITY ? 0.f : exp2f(x[3] - mB);
        sA += p0 + p2;
        sB += p1 + p3;
        // P^T fragments (B operand): hi/lo split, transposed with movmatrix
        unsigned b0, b1, b2 = 0, b3 = 0;
        {
            const float h0 = bf16_round(p0), h1 = bf16_round(p1), h2 = bf16_round(p2), h3 = bf16_round(p3);
            if (PACKED) {
                const bool hi = tq < 2;
                b0 = movm_t(hi ? pack_bf16(h0, h1) : pack_bf16(p0 - h0, p1 - h1));
                b1 = movm_t(hi ? pack_bf16(h2, h3) : pack_bf16(p2 - h2, p3 - h3));
            } else {
                b0 = movm_t(pack_bf16(h0, h1));
                b1 = movm_t(pack_bf16(h2, h3));
                b2 = movm_t(pack_bf16(p0 - h0, p1 - h1));
                b3 = movm_t(pack_bf16(p2 - h2, p3 - h3));
            }
        }
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
            unsigned a[4];
            const int j = lane >> 3;
            const int row = (lane & 7) + (j >> 1) * 8, ch = mt * 2 + (j & 1);
            ldsm_x4_t(vtile + swz(row, ch), a);
            mma_bf16(o[mt], a, b0, b1);
            if (!PACKED) mma_bf16(o2[PACKED ? 0 : mt], a, b2, b3);
        }
    };

    // ---- end of a ledger segment of this CTA (every warp calls it for every ledger of the CTA
    // range, in order): warp partials -> CTA partial through shared memory (each warp writes
    // into the ring stage it is not using: `fs`, the one consumed last); a ledger wholly inside
    // the CTA range is finalised here, otherwise the CTA partial goes to slot (c + l) and the
    // last of the ledger's CTAs (atomic ticket) merges them.
    __shared__ int s_last;
    __shared__ unsigned s_poff[NW];
    auto seg_end = [&](int l, int fs) {
        float* wscr = reinterpret_cast<float*>(smem + w * Geo::kWarpB + fs * Geo::kStageB);
        float fA = sA, fB = sB;
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            fA += __shfl_xor_sync(0xffffffffu, fA, off);
            fB += __shfl_xor_sync(0xffffffffu, fB, off);
        }
        if (PACKED) {
#pragma unroll
            for (int mt = 0; mt < KS; ++mt)
#pragma unroll
                for (int j = 0; j < 4; ++j) o[mt][j] += __shfl_xor_sync(0xffffffffu, o[mt][j], 2);
        } else {
#pragma unroll
            for (int mt = 0; mt < KS; ++mt)
#pragma unroll
                for (int j = 0; j < 4; ++j) o[mt][j] += o2[PACKED ? 0 : mt][j];
        }
        const bool owner = PACKED ? tq < 2 : true;
        if (owner) {
            if (gr == 0) {
                if (hA < G) { wscr[2 * hA] = mA; wscr[2 * hA + 1] = fA; }
                if (hB < G) { wscr[2 * hB] = mB; wscr[2 * hB + 1] = fB; }
            }
#pragma unroll
            for (int mt = 0; mt < KS; ++mt) {
                if (hA < G) {
                    wscr[2 * G + hA * D + mt * 16 + gr] = o[mt][0];
                    wscr[2 * G + hA * D + mt * 16 + gr + 8] = o[mt][2];
                }
                if (hB < G) {
                    wscr[2 * G + hB * D + mt * 16 + gr] = o[mt][1];
                    wscr[2 * G + hB * D + mt * 16 + gr + 8] = o[mt][3];
                }
            }
        }
        if (lane == 0) s_poff[w] = (unsigned)(w * Geo::kWarpB + fs * Geo::kStageB);
        __syncthreads();
        DBG_SEG(5);
        const bool whole = tp[l] >= g0 && tp[l + 1] <= g1;
        float* dst = part + (size_t)(c + l) * Geo::kPS;
        for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
            const int g = idx / D, k = idx - g * D;
            float mw[NW], M = -INFINITY;
#pragma unroll
            for (int ww = 0; ww < NW; ++ww) {
                mw[ww] = reinterpret_cast<const float*>(smem + s_poff[ww])[2 * g];
                M = fmaxf(M, mw[ww]);
            }
            float S = 0.f, A = 0.f;
            if (M != -INFINITY) {
#pragma unroll
                for (int ww = 0; ww < NW; ++ww) {
                    if (mw[ww] == -INFINITY) continue;
                    const float* wp = reinterpret_cast<const float*>(smem + s_poff[ww]);
                    const float sc = exp2f(mw[ww] - M);
                    S += sc * wp[2 * g + 1];
                    A += sc * wp[2 * G + g * D + k];
                }
            }
            if (whole) {
                emit_result(out, part_out, l, G, D, g, k, M * kLn2, S, A);
            } else {
                dst[2 * G + idx] = A;
                if (k == 0) {
                    dst[2 * g] = M;
                    dst[2 * g + 1] = S;
                }
            }
        }
        if (!whole) {
            __threadfence();
            __syncthreads();
            DBG_SEG(6);
            // first CTA meeting ledger l: the one whose range contains tile tp[l]
            int cf = (int)min((long long)Ce - 1, (long long)tp[l] * Ce / T);
            while (cf + 1 < Ce && cta_begin(cf + 1) <= tp[l]) ++cf;
            while (cf > 0 && cta_begin(cf) > tp[l]) --cf;
            // every CTA owns >= kMinTiles tiles, so the CTAs meeting ledger l are cf .. cf + np - 1
            // and their partials sit in consecutive slots cf + l ..
            __shared__ int s_np;
            if (threadIdx.x == 0) {
                int np = 0;
                for (int cc = cf; cc < Ce && cbt_at(cc) < tp[l + 1]; ++cc) ++np;
                s_np = np;
                const int prev = atomicAdd(ticket + l, 1);
                s_last = prev == np - 1;
                if (s_last) ticket[l] = 0;  // ready for the next launch / graph replay
            }
            __syncthreads();
            DBG_SEG(7);
            if (s_last) {
                __threadfence();
                const int np = s_np;
                constexpr int PER = (G * D + NW * 32 - 1) / (NW * 32);
                float M[PER], S[PER], A[PER];
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    M[j] = -INFINITY;
                    S[j] = 0.f;
                    A[j] = 0.f;
                }
                for (int p0 = 0; p0 < np; p0 += 4) {
                    // four partials' values for this thread's outputs, all loads in flight together
                    float pm[4][PER], ps[4][PER], pa[4][PER];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int p = p0 + u;
                        const float* P = part + (size_t)(cf + l + (p < np ? p : 0)) * Geo::kPS;
#pragma unroll
                        for (int j = 0; j < PER; ++j) {
                            const int idx = threadIdx.x + j * NW * 32;
                            const int g = min(idx, G * D - 1) / D;
                            const bool ok = p < np && idx < G * D;
                            pm[u][j] = ok ? __ldcg(P + 2 * g) : -INFINITY;
                            ps[u][j] = ok ? __ldcg(P + 2 * g + 1) : 0.f;
                            pa[u][j] = ok ? __ldcg(P + 2 * G + idx) : 0.f;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int j = 0; j < PER; ++j) {
                            const float m = pm[u][j];
                            if (m == -INFINITY) continue;
                            if (m > M[j]) {
                                const float sc = exp2f(M[j] - m);
                                S[j] = S[j] * sc + ps[u][j];
                                A[j] = A[j] * sc + pa[u][j];
                                M[j] = m;
                            } else {
                                const float sc = exp2f(m - M[j]);
                                S[j] += ps[u][j] * sc;
                                A[j] += pa[u][j] * sc;
                            }
                        }
                }
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    const int idx = threadIdx.x + j * NW * 32;
                    if (idx < G * D)
                        emit_result(out, part_out, l, G, D, idx / D, idx % D, M[j] * kLn2, S[j], A[j]);
                }
            }
        }
        __syncthreads();  // the scratch is reused by the next segment
    };

    // ---- pipeline: ids run kAhead tiles ahead of the gathers, gathers NST-1 tiles ahead of the math
    Walker wp{-1, 0, 0, 0, 0, 0}, wi = wp, wc = wp;
    int pf = 0, issued = 0;
    auto prefetch_next = [&]() {
        if (pf < my_n) prefetch_ids(pf, meta_of(pf, wp));
        else asm volatile("cp.async.commit_group;\n" ::);
        ++pf;
    };
    auto issue_next = [&]() {
        if (issued < my_n) {
            asm volatile("cp.async.wait_group %0;\n" ::"n"(kAhead - 1));
            __syncwarp();
            const Meta m = meta_of(issued, wi);
            issue(issued, issued % NST, m);
            ++issued;
            prefetch_next();
        }
    };
#pragma unroll 1
    for (int i = 0; i < kAhead; ++i) prefetch_next();
    DBG_RAMP(5);
#pragma unroll 1
    for (int i = 0; i < NST - 1; ++i) {
        issue_next();
        if (i == 0) DBG_RAMP(6);
    }
    DBG_RAMP(7);

    // ledgers met by this CTA: lf .. ll (every warp closes each of them, in order)
    const int lf = ledger_of_tile(g0), ll = ledger_of_tile(g1 - 1);
    int cur_l = lf;
    bool fresh = true;  // q fragments of cur_l not loaded yet
    reset_state();
#pragma unroll 1
    for (int i = 0; i < my_n; ++i) {
        const Meta m = meta_of(i, wc);
        // stages (i, i+1) % NST are in flight; (i + NST - 1) % NST was consumed last and is free
        // until issue_next() below refills it -- seg_end stages this warp's partial there
        while (m.l != cur_l) {
            seg_end(cur_l, (i + NST - 1) % NST);
            ++cur_l;
            reset_state();
            fresh = true;
        }
        issue_next();
        if (fresh) {
            load_q(cur_l);
            fresh = false;
        }
        const int st = i % NST;
        mbar_wait(bar0 + st * 8, (i / NST) & 1);
        if (i == 0) dbg_stamp(2);
        if (m.nv <= 0) continue;
        const unsigned kst = wbase + st * Geo::kStageB, vst = kst + Geo::kMatB, lgs = lgbase + st * Geo::kLgB;
        if (m.kind == 0) {
            // S = K q^T on the tensor cores, logits in log2 units
            float c1[4] = {0.f, 0.f, 0.f, 0.f};
            float c2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                unsigned a[4];
                const int row = (lane & 7) + ((lane >> 3) & 1) * 8, ch = ks * 2 + (lane >> 4);
                ldsm_x4(kst + swz(row, ch), a);
                mma_bf16(c1, a, qhi[ks][0], qhi[ks][1]);
                if (!PACKED) mma_bf16(c2, a, qlo[PACKED ? 0 : ks][0], qlo[PACKED ? 0 : ks][1]);
            }
            float x[4];
            if (PACKED) {
#pragma unroll
                for (int j = 0; j < 4; ++j) x[j] = c1[j] + __shfl_xor_sync(0xffffffffu, c1[j], 2);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) x[j] = c1[j] + c2[j];
            }
            if (gr >= m.nv) x[0] = x[1] = -INFINITY;
            if (gr + 8 >= m.nv) x[2] = x[3] = -INFINITY;
            absorb16(x, vst);
        } else {
            // rejected centroids: reused lookup logits + ln N, two 16-row value tiles
            const float* lg = reinterpret_cast<const float*>(smem + (lgs - smem_u32(smem)));
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
                if (sub * 16 >= m.nv) break;
                float x[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int rr = sub * 16 + gr + (j >> 1) * 8;
                    const int h = (j & 1) ? hB : hA;
                    x[j] = rr < m.nv ? (h < G ? lg[rr * GP + h] * kLog2e : 0.f) : -INFINITY;
                }
                absorb16(x, sub ? vst : kst);
            }
        }
    }
    dbg_stamp(3);
    for (; cur_l <= ll; ++cur_l) {  // the ring is drained: any stage is free
        seg_end(cur_l, 0);
        reset_state();
    }
    dbg_stamp(4);
}

}  // namespace mpa

using namespace mpa;

namespace {

int num_sms() { return device_sms(); }

// serving configuration of the stream-K kernel: 4 warps x 3 stages (~104 KB smem, 2 CTAs / SM)
constexpr int kSkWarps = 4, kSkStages = 3;

constexpr int sk_ctas_per_sm() { return 2; }  // fixed by the smem budget (2 x 104 KB of the 228 KB per SM)

// CTA count of the stream-K grid: n_split <= 0 -> one full wave; else n_split CTAs per ledger
int sk_grid(int L, int n_split) {
    const int wave = num_sms() * sk_ctas_per_sm();
    if (n_split <= 0) return wave;
    long long c = (long long)n_split * L;
    if (c > 8 * wave) c = 8 * wave;
    return (int)(c < 1 ? 1 : c);
}

bool mma_path(const mpa_cache* c, int group);

size_t ws_floats_ffma(int L, int G, int d, int S) { return (size_t)L * S * G * (2 + d); }
size_t ws_floats_sk(int L, int G, int d, int C) { return (size_t)(C + L + C * kSkWarps) * G * (d + 2); }
size_t ws_ticket_bytes(int L) { return ((size_t)L * sizeof(int32_t) + 255) & ~(size_t)255; }

template <int G>
int launch_ffma(const mpa_cache* c, const float* q_rot, const int32_t* tok, const int32_t* n_tok, int tok_cap,
                const int32_t* rej, const float* rej_w, const int32_t* n_rej, int rej_cap, const void* fvc, int fcap,
                const void* cvc, int ccap, int S, float* pml, float* pacc, int32_t* ticket, float* out,
                float* part_out, cudaStream_t st) {
    const int d = c->head_dim;
    const int ndl = ceil_div(d, 32);
    dim3 grid(S, c->n_ledgers);
    const size_t smem = sizeof(float) * kFfmaWarps * G * (2 + d);
#define MPA_FFMA_CASE(T, NDL)                                                                                   \
    {                                                                                                           \
        auto kern = decode_ffma_kernel<T, G, NDL>;                                                              \
        if (int rc = set_max_smem((const void*)kern, (int)smem)) return rc;                                   \
        kern<<<grid, kFfmaWarps * 32, smem, st>>>((const T*)c->k_rot, (const T*)c->v, kv_rows(c), d, q_rot, tok, \
                                                  n_tok, tok_cap, rej, rej_w, n_rej, rej_cap, (const T*)fvc,    \
                                                  fcap, (const T*)cvc, ccap, S, pml, pacc, ticket, out,         \
                                                  part_out);                                                    \
    }
#define MPA_FFMA_NDL(T)                                    \
    switch (ndl) {                                         \
        case 1: MPA_FFMA_CASE(T, 1) break;                 \
        case 2: MPA_FFMA_CASE(T, 2) break;                 \
        case 3: case 4: MPA_FFMA_CASE(T, 4) break;         \
        default: MPA_FFMA_CASE(T, 8) break;                \
    }
    if (c->dtype == MPA_F32) {
        MPA_FFMA_NDL(float)
    } else {
        MPA_FFMA_NDL(__nv_bfloat16)
    }
#undef MPA_FFMA_NDL
#undef MPA_FFMA_CASE
    return check_launch("mpa_sparse_decode(ffma)");
}

// 2D tensor map over rows of d bf16 (box: 64 columns x 1 row, 128B swizzle) for TMA gathers.
// Encoding is pure host work; the last few maps are cached by (address, rows, d).
int bf16_rows_map(CUtensorMap* out, const void* base, long long rows, int d, int box_rows = 1) {
    struct Entry {
        const void* base;
        long long rows;
        int d, box_rows;
        CUtensorMap map;
    };
    static Entry cache[32];
    static int next = 0;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : cache)
        if (e.base == base && e.rows == rows && e.d == d && e.box_rows == box_rows) {
            *out = e.map;
            return 0;
        }
    MPA_REQUIRE(rows > 0 && rows < (1ll << 31), MPA_ERR_UNSUPPORTED, "tensor map: %lld rows", rows);
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    // resolved through the runtime so the library has no link-time libcuda dependency
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
    const CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    MPA_REQUIRE(r == CUDA_SUCCESS, MPA_ERR_ARG, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    cache[next] = Entry{base, rows, d, box_rows, *out};
    next = (next + 1) % 32;
    return 0;
}

// resident CTAs per SM of a stream-K instantiation at a smem size, memoised per (device, kernel, smem)
int sk_occupancy(const void* kern, int smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int>, int> memo;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = memo.find({dev, kern, smem});
    if (it != memo.end()) return it->second;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kSkWarps * 32, smem);
    memo[{dev, kern, smem}] = occ;
    return occ;
}

template <int G, int D>
int launch_sk(const mpa_cache* c, const float* q_rot, const int32_t* tok, const int32_t* n_tok, int tok_cap,
              const int32_t* rej, const float* rej_w, const int32_t* n_rej, int rej_cap, const void* fvc, int fcap,
              const void* cvc, int ccap, int C, float* part, int32_t* ticket, float* out, float* part_out,
              cudaStream_t st, bool one_wave) {
    using Geo = SkGeom<G, D, kSkWarps, kSkStages>;
    const int L = c->n_ledgers;
    const size_t smem = Geo::smem(L, C);
    MPA_REQUIRE(smem <= 227 * 1024, MPA_ERR_UNSUPPORTED, "mpa_sparse_decode: %d ledgers exceed the smem schedule", L);
    auto kern = c->block_table ? decode_sk_kernel<G, D, kSkWarps, kSkStages, true>
                               : decode_sk_kernel<G, D, kSkWarps, kSkStages, false>;
    if (int rc = set_max_smem((const void*)kern, (int)smem)) return rc;
    if (one_wave) {  // the stream-K grid is one resident wave (2 CTAs / SM unless smem or registers say less)
        const int occ = sk_occupancy((const void*)kern, (int)smem);
        C = std::min(C, std::max(1, occ) * num_sms());
    }
    CUtensorMap tk, tv, tf, tc, tf16;
    int rc = bf16_rows_map(&tk, c->k_rot, kv_pool_rows(c), D);
    if (!rc) rc = bf16_rows_map(&tv, c->v, kv_pool_rows(c), D);
    if (!rc) rc = fvc ? bf16_rows_map(&tf, fvc, (long long)L * fcap, D) : (tf = tk, 0);
    if (!rc) rc = fvc ? bf16_rows_map(&tf16, fvc, (long long)L * fcap, D, 16) : (tf16 = tk, 0);
    if (!rc) rc = cvc ? bf16_rows_map(&tc, cvc, (long long)L * ccap, D) : (tc = tf, 0);
    if (rc) return rc;
    MPA_REQUIRE(rej || !rej_w || fvc, MPA_ERR_ARG, "mpa_sparse_decode: contiguous-centroid list without fine_vc");
    launch_pdl(kern, dim3(C), dim3(kSkWarps * 32), smem, st, tk, tv, tf, tc, tf16, kv_rows(c),
               (const __nv_bfloat16*)c->k_rot, (const __nv_bfloat16*)c->v, q_rot, tok, n_tok, tok_cap, rej, rej_w,
               n_rej, rej_cap, fcap, ccap, L, part, ticket, out, part_out,
               tok != nullptr ? 1 : 0);  // sparse token lists through the LSU, the dense decode through TMA gathers
    return check_launch("mpa_sparse_decode(stream-K mma)");
}

bool mma_path(const mpa_cache* c, int group) {
    return c->dtype == MPA_BF16 && (c->head_dim == 64 || c->head_dim == 128) && group <= 8;
}

int ffma_splits(int L, int n_split) {
    if (n_split > 0) return n_split;
    const int s = (2 * num_sms() * 2 + L - 1) / L;
    return s < 1 ? 1 : (s > 64 ? 64 : s);
}

}  // namespace

#ifdef MPA_DEBUG_TRACE
extern "C" int mpa_debug_trace(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_dbg, sizeof(unsigned long long) * n);
}
#endif

extern "C" size_t mpa_sparse_decode_workspace(int n_ledgers, int group, int head_dim, int dtype, int n_split) {
    if (n_ledgers <= 0 || group <= 0 || head_dim <= 0) return 0;
    mpa_cache probe{};
    probe.dtype = dtype;
    probe.head_dim = head_dim;
    size_t fl;
    if (mma_path(&probe, group)) fl = ws_floats_sk(n_ledgers, group, head_dim, sk_grid(n_ledgers, n_split));
    else fl = ws_floats_ffma(n_ledgers, group, head_dim, ffma_splits(n_ledgers, n_split));
    return ws_ticket_bytes(n_ledgers) + fl * sizeof(float);
}

static int sparse_decode_impl(const mpa_cache* c, const float* q_rot, int n_kv_heads, int group,
                                 const int32_t* tok, const int32_t* n_tok, int tok_cap, const int32_t* rej,
                                 const float* rej_w, const int32_t* n_rej, int rej_cap, const void* fine_vc,
                                 int fine_cap, const void* coarse_vc, int coarse_cap, int n_split, void* workspace,
                                 size_t workspace_bytes, float* out, float* part_out, void* stream) {
    MPA_REQUIRE(c && q_rot && n_tok && workspace && (out || part_out), MPA_ERR_ARG, "mpa_sparse_decode: null argument");
    MPA_REQUIRE(!rej || (rej_w && n_rej), MPA_ERR_ARG, "mpa_sparse_decode: rej without weights/counts");
    MPA_REQUIRE(!rej_w || n_rej, MPA_ERR_ARG, "mpa_sparse_decode: rej_w without counts");
    MPA_REQUIRE(c->head_dim >= 2 && c->head_dim % 2 == 0 && c->head_dim <= 256, MPA_ERR_UNSUPPORTED,
                "mpa_sparse_decode: head_dim %d", c->head_dim);
    (void)n_kv_heads;
    if (int rc = check_cache(c, "mpa_sparse_decode")) return rc;
    const int L = c->n_ledgers;
    if (L <= 0) return 0;
    const size_t need = mpa_sparse_decode_workspace(L, group, c->head_dim, c->dtype, n_split);
    MPA_REQUIRE(workspace_bytes >= need, MPA_ERR_ARG, "mpa_sparse_decode: workspace %zu bytes < %zu", workspace_bytes,
                need);
    cudaStream_t st = (cudaStream_t)stream;
    int32_t* ticket = (int32_t*)workspace;
    float* part = (float*)((char*)workspace + ws_ticket_bytes(L));
    if (mma_path(c, group)) {
        const int C = sk_grid(L, n_split);
        MPA_DISPATCH_G(group, {
            if (c->head_dim == 128)
                return launch_sk<kG, 128>(c, q_rot, tok, n_tok, tok_cap, rej, rej_w, n_rej, rej_cap, fine_vc,
                                          fine_cap, coarse_vc, coarse_cap, C, part, ticket, out, part_out, st,
                                          n_split <= 0);
            return launch_sk<kG, 64>(c, q_rot, tok, n_tok, tok_cap, rej, rej_w, n_rej, rej_cap, fine_vc, fine_cap,
                                     coarse_vc, coarse_cap, C, part, ticket, out, part_out, st, n_split <= 0);
        });
    }
    MPA_REQUIRE(rej || !rej_w, MPA_ERR_UNSUPPORTED,
                "mpa_sparse_decode: the contiguous-centroid list needs the bf16 tensor-core path");
    const int S = ffma_splits(L, n_split);
    float* pml = part;
    float* pacc = part + (size_t)L * S * group * 2;
    MPA_DISPATCH_G(group, {
        return launch_ffma<kG>(c, q_rot, tok, n_tok, tok_cap, rej, rej_w, n_rej, rej_cap, fine_vc, fine_cap,
                               coarse_vc, coarse_cap, S, pml, pacc, ticket, out, part_out, st);
    });
    return 0;
}

extern "C" int mpa_sparse_decode(const mpa_cache* c, const float* q_rot, int n_kv_heads, int group,
                                 const int32_t* tok, const int32_t* n_tok, int tok_cap, const int32_t* rej,
                                 const float* rej_w, const int32_t* n_rej, int rej_cap, const void* fine_vc,
                                 int fine_cap, const void* coarse_vc, int coarse_cap, int n_split, void* workspace,
                                 size_t workspace_bytes, float* out, void* stream) {
    MPA_REQUIRE(out, MPA_ERR_ARG, "mpa_sparse_decode: null argument");
    return sparse_decode_impl(c, q_rot, n_kv_heads, group, tok, n_tok, tok_cap, rej, rej_w, n_rej, rej_cap, fine_vc,
                              fine_cap, coarse_vc, coarse_cap, n_split, workspace, workspace_bytes, out, nullptr,
                              stream);
}

extern "C" int mpa_sparse_decode_partials(const mpa_cache* c, const float* q_rot, int n_kv_heads, int group,
                                          const int32_t* tok, const int32_t* n_tok, int tok_cap, const int32_t* rej,
                                          const float* rej_w, const int32_t* n_rej, int rej_cap,
                                          const void* fine_vc, int fine_cap, const void* coarse_vc, int coarse_cap,
                                          int n_split, void* workspace, size_t workspace_bytes, float* part_out,
                                          void* stream) {
    MPA_REQUIRE(part_out, MPA_ERR_ARG, "mpa_sparse_decode_partials: null argument");
    return sparse_decode_impl(c, q_rot, n_kv_heads, group, tok, n_tok, tok_cap, rej, rej_w, n_rej, rej_cap, fine_vc,
                              fine_cap, coarse_vc, coarse_cap, n_split, workspace, workspace_bytes, nullptr, part_out,
                              stream);
}

// LSE merge of per-rank partials [P][L][G][2 + d] (m natural-log, s, a) -> out [L][G][d]
// (attention.py:230-239 merge_partials + :44-47 finalize, across sequence shards)
__global__ void merge_rank_partials_kernel(const float* __restrict__ parts, int P, int LG, int d,
                                           float* __restrict__ out) {
    const int lg = blockIdx.x;
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        float M = -INFINITY;
        for (int r = 0; r < P; ++r) M = fmaxf(M, parts[((size_t)r * LG + lg) * (d + 2)]);
        float S = 0.f, A = 0.f;
        if (M != -INFINITY)
            for (int r = 0; r < P; ++r) {
                const float* Pp = parts + ((size_t)r * LG + lg) * (d + 2);
                if (Pp[0] == -INFINITY) continue;
                const float w = expf(Pp[0] - M);
                S += w * Pp[1];
                A += w * Pp[2 + k];
            }
        out[(size_t)lg * d + k] = A / S;
    }
}

extern "C" int mpa_merge_rank_partials(const float* parts, int n_ranks, int n_ledgers, int group, int head_dim,
                                       float* out, void* stream) {
    MPA_REQUIRE(parts && out, MPA_ERR_ARG, "mpa_merge_rank_partials: null argument");
    MPA_REQUIRE(n_ranks >= 1 && group >= 1 && head_dim >= 1, MPA_ERR_ARG, "mpa_merge_rank_partials: sizes");
    if (n_ledgers <= 0) return 0;
    merge_rank_partials_kernel<<<n_ledgers * group, 128, 0, (cudaStream_t)stream>>>(parts, n_ranks, n_ledgers * group,
                                                                                   head_dim, out);
    return check_launch("mpa_merge_rank_partials");
}
