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
// value centroid). Items are split over n_split CTAs per ledger balanced by bytes (a token
// costs two rows, a centroid one); the last CTA of a ledger (atomic ticket) LSE-merges the
// split partials and writes the output, so the step needs no separate merge launch.
//
// Two implementations share that structure:
//   * decode_mma_kernel (bf16, d in {64,128}, G <= 8): per-warp 16-item tiles staged in
//     swizzled smem by cp.async (3-4 stages in flight), S = K q^T and O^T += V^T P^T on the
//     tensor cores with mma.sync m16n8k16 (tokens on M, q-heads on N=8).  q and P are split
//     into bf16 hi + lo parts packed into the 8 MMA columns (G <= 4) so the only bf16
//     rounding left is the KV cache itself.  Base-2 online softmax.
//   * decode_ffma_kernel (any dtype, any even d): warp per item, FFMA, natural-log softmax,
//     fp32 accurate expf -- the fp32 parity mode (1e-5).
#include <climits>
#include <cstdlib>

#include "mpa_common.cuh"

namespace mpa {

constexpr float kLog2e = 1.4426950408889634f;

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

// Last-CTA merge of the n_split partials of ledger l (m in the kernel's log base).
template <bool BASE2>
__device__ void merge_splits(int l, int S, int G, int d, const float* part_ml, const float* part_acc, float* out) {
    for (int idx = threadIdx.x; idx < G * d; idx += blockDim.x) {
        const int g = idx / d, k = idx - g * d;
        float M = -INFINITY;
        for (int s = 0; s < S; ++s) M = fmaxf(M, __ldcg(part_ml + (((size_t)l * S + s) * G + g) * 2));
        float sum = 0.f, acc = 0.f;
        if (M != -INFINITY) {
            for (int s = 0; s < S; ++s) {
                const float m = __ldcg(part_ml + (((size_t)l * S + s) * G + g) * 2);
                if (m == -INFINITY) continue;
                const float w = BASE2 ? exp2f(m - M) : expf(m - M);
                sum += w * __ldcg(part_ml + (((size_t)l * S + s) * G + g) * 2 + 1);
                acc += w * __ldcg(part_acc + (((size_t)l * S + s) * G + g) * d + k);
            }
        }
        out[((size_t)l * G + g) * d + k] = acc / sum;
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

// ============================================================================
// FFMA path

constexpr int kFfmaWarps = 4;

template <typename T, int G, int NDL>
__global__ void __launch_bounds__(kFfmaWarps * 32)
decode_ffma_kernel(const T* __restrict__ k_rot, const T* __restrict__ vcache, int tcap, int d,
                   const float* __restrict__ q_rot, const int32_t* __restrict__ tok, const int32_t* __restrict__ n_tok,
                   int tok_cap, const int32_t* __restrict__ rej, const float* __restrict__ rej_w,
                   const int32_t* __restrict__ n_rej, int rej_cap, const T* __restrict__ fvc, int fcap,
                   const T* __restrict__ cvc, int ccap, int S, float* __restrict__ part_ml,
                   float* __restrict__ part_acc, int32_t* __restrict__ ticket, float* __restrict__ out) {
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
        const T* kp = k_rot + ((size_t)l * tcap + row) * d;
        const T* vp = vcache + ((size_t)l * tcap + row) * d;
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
        for (int g = 0; g < G; ++g) x[g] = rej_w[((size_t)l * rej_cap + r) * G + g];
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
    if (take_ticket(ticket, l, S)) merge_splits<false>(l, S, G, d, part_ml, part_acc, out);
}

// ============================================================================
// Tensor-core path (bf16, mma.sync m16n8k16)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(unsigned dst, const void* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async4(unsigned dst, const void* src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

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

template <int D> struct TileGeom {
    static constexpr int kChunks = D / 8;           // 16-byte chunks per row
    static constexpr int kRowBytes = D * 2;
    static constexpr int kMatBytes = 16 * kRowBytes;  // one 16-row K or V tile
    __device__ static __forceinline__ unsigned off(int row, int chunk) {
        return row * kRowBytes + ((chunk ^ (row & 7)) << 4);
    }
};

constexpr int kMmaWarps = 4;
constexpr int kSegTiles = 64;  // tiles whose row ids are staged in smem at a time

// PACKED: G <= 4, columns 0..3 carry the hi parts of q / P, columns 4..7 the lo parts.
// Otherwise (G <= 8) hi and lo run as two separate MMAs.
template <int G, int D, int NST>
__global__ void __launch_bounds__(kMmaWarps * 32)
decode_mma_kernel(const __nv_bfloat16* __restrict__ k_rot, const __nv_bfloat16* __restrict__ vcache, int tcap,
                  const float* __restrict__ q_rot, const int32_t* __restrict__ tok, const int32_t* __restrict__ n_tok,
                  int tok_cap, const int32_t* __restrict__ rej, const float* __restrict__ rej_w,
                  const int32_t* __restrict__ n_rej, int rej_cap, const __nv_bfloat16* __restrict__ fvc, int fcap,
                  const __nv_bfloat16* __restrict__ cvc, int ccap, int S, float* __restrict__ part_ml,
                  float* __restrict__ part_acc, int32_t* __restrict__ ticket, float* __restrict__ out) {
    constexpr bool PACKED = G <= 4;
    constexpr int KS = D / 16;  // k-steps for QK, m-tiles for PV
    using Geo = TileGeom<D>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int l = blockIdx.y, s = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gr = lane >> 2, tq = lane & 3;
    const int nt = n_tok[l], nr = rej ? n_rej[l] : 0;
    const SplitRange R = split_range(nt, nr, s, S);
    const int ntt = (R.t1 - R.t0 + 15) >> 4, nrt = (R.r1 - R.r0 + 15) >> 4, NT = ntt + nrt;

    unsigned char* wbase = smem + (size_t)w * NST * 2 * Geo::kMatBytes;
    const unsigned wbase_s = smem_u32(wbase);

    // ---- q fragments (B operand, col-major 16x8 per k-step), pre-scaled by log2(e)
    unsigned qhi[KS][2], qlo[KS][2];
    {
        auto qv = [&](int head, int k) -> float {
            return head < G ? q_rot[((size_t)l * G + head) * D + k] * kLog2e : 0.f;
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
                    qlo[ks][half] = pack_bf16(a - ah, b - bh);
                }
            }
        }
    }

    // heads owned by this lane's two accumulator columns
    const int hA = PACKED ? 2 * (tq & 1) : 2 * tq, hB = hA + 1;
    float mA = -INFINITY, mB = -INFINITY, sA = 0.f, sB = 0.f;
    float o[KS][4];
    float o2[PACKED ? 1 : KS][4];
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

    const size_t cache_base = (size_t)l * tcap;
    // Row ids (token id, or centroid code) of a segment of kSegTiles virtual tiles are staged in
    // smem by the whole CTA before the per-warp pipelines run over that segment, so no
    // dependent index load ever sits between a tile and its cp.async issue.
    constexpr int kNoRow = INT_MIN;
    int* ids_s = reinterpret_cast<int*>(smem + (size_t)kMmaWarps * NST * 2 * Geo::kMatBytes);
    int seg = 0;
    auto fetch = [&](int vt) -> int { return ids_s[(vt - seg) * 16 + (lane >> 1)]; };
    auto issue = [&](int vt, int st, int id) {
        const unsigned kst = wbase_s + st * 2 * Geo::kMatBytes, vst = kst + Geo::kMatBytes;
        const int row = lane >> 1;  // 2 lanes per row
        const bool ok = id != kNoRow;
        if (vt < ntt) {
            const int tokid = ok ? id : 0;
            const __nv_bfloat16* kp = k_rot + (cache_base + tokid) * D;
            const __nv_bfloat16* vp = vcache + (cache_base + tokid) * D;
#pragma unroll
            for (int j = 0; j < Geo::kChunks / 2; ++j) {
                const int ch = (lane & 1) * (Geo::kChunks / 2) + j;
                cp_async16(kst + Geo::off(row, ch), kp + ch * 8, ok ? 16 : 0);
                cp_async16(vst + Geo::off(row, ch), vp + ch * 8, ok ? 16 : 0);
            }
        } else {
            const int code = ok ? id : 0;
            const __nv_bfloat16* vp =
                code >= 0 ? fvc + ((size_t)l * fcap + code) * D : cvc + ((size_t)l * ccap + (-1 - code)) * D;
#pragma unroll
            for (int j = 0; j < Geo::kChunks / 2; ++j) {
                const int ch = (lane & 1) * (Geo::kChunks / 2) + j;
                cp_async16(vst + Geo::off(row, ch), vp + ch * 8, ok ? 16 : 0);
            }
            // the tile's reused lookup logits (16 x G fp32) ride along in the unused K slot
            const int r0 = R.r0 + (vt - ntt) * 16;
            for (int e = lane; e < 16 * G; e += 32) {
                const int rr = e / G;
                const bool okr = r0 + rr < R.r1;
                cp_async4(kst + e * 4, rej_w + ((size_t)l * rej_cap + (okr ? r0 + rr : 0)) * G + (e - rr * G),
                          okr ? 4 : 0);
            }
        }
    };

    for (seg = 0; seg < NT; seg += kSegTiles) {
        const int seg_n = min(kSegTiles, NT - seg);
        for (int k = threadIdx.x; k < seg_n * 16; k += blockDim.x) {
            const int vt = seg + (k >> 4), row = k & 15;
            int id;
            if (vt < ntt) {
                const int t = R.t0 + vt * 16 + row;
                id = t < R.t1 ? (tok ? __ldg(tok + (size_t)l * tok_cap + t) : t) : kNoRow;
            } else {
                const int r = R.r0 + (vt - ntt) * 16 + row;
                id = r < R.r1 ? __ldg(rej + (size_t)l * rej_cap + r) : kNoRow;
            }
            ids_s[k] = id;
        }
        __syncthreads();
        // this warp's tiles in the segment: vt = seg + w, seg + w + W, ...
        const int my_n = seg_n > w ? (seg_n - w + kMmaWarps - 1) / kMmaWarps : 0;
#pragma unroll
        for (int i = 0; i < NST - 1; ++i) {
            if (i < my_n) issue(seg + w + i * kMmaWarps, i, fetch(seg + w + i * kMmaWarps));
            cp_commit();
        }
        for (int i = 0; i < my_n; ++i) {
            {
                const int nxt = i + NST - 1;
                if (nxt < my_n) issue(seg + w + nxt * kMmaWarps, nxt % NST, fetch(seg + w + nxt * kMmaWarps));
                cp_commit();
            }
            cp_wait<NST - 1>();
            __syncwarp();
            const int vt = seg + w + i * kMmaWarps, st = i % NST;
            const unsigned kst = wbase_s + st * 2 * Geo::kMatBytes, vst = kst + Geo::kMatBytes;

            // logits x[row r / r+8][head hA / hB] in log2 units
            float x[4];
            if (vt < ntt) {
                float c[4] = {0.f, 0.f, 0.f, 0.f};
                float c2[4] = {0.f, 0.f, 0.f, 0.f};
    #pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    unsigned a[4];
                    const int row = (lane & 7) + ((lane >> 3) & 1) * 8, ch = ks * 2 + (lane >> 4);
                    ldsm_x4(kst + Geo::off(row, ch), a);
                    mma_bf16(c, a, qhi[ks][0], qhi[ks][1]);
                    if (!PACKED) mma_bf16(c2, a, qlo[ks][0], qlo[ks][1]);
                }
                if (PACKED) {
    #pragma unroll
                    for (int j = 0; j < 4; ++j) x[j] = c[j] + __shfl_xor_sync(0xffffffffu, c[j], 2);
                } else {
    #pragma unroll
                    for (int j = 0; j < 4; ++j) x[j] = c[j] + c2[j];
                }
                const int base = R.t0 + (vt << 4);
                if (base + gr >= R.t1) x[0] = x[1] = -INFINITY;
                if (base + gr + 8 >= R.t1) x[2] = x[3] = -INFINITY;
            } else {
                const int base = R.r0 + ((vt - ntt) << 4);
                const float* lg = reinterpret_cast<const float*>(wbase + (size_t)st * 2 * Geo::kMatBytes);
    #pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int rr = gr + (j >> 1) * 8;
                    const int h = (j & 1) ? hB : hA;
                    x[j] = base + rr < R.r1 ? (h < G ? lg[rr * G + h] * kLog2e : 0.f) : -INFINITY;
                }
            }
            // padded heads (>= G) must stay finite
            if (hA >= G) { x[0] = x[0] == -INFINITY ? -INFINITY : 0.f; x[2] = x[2] == -INFINITY ? -INFINITY : 0.f; }
            if (hB >= G) { x[1] = x[1] == -INFINITY ? -INFINITY : 0.f; x[3] = x[3] == -INFINITY ? -INFINITY : 0.f; }

            // online softmax (column = head) over the 16 rows of this tile
            float tA = fmaxf(x[0], x[2]), tB = fmaxf(x[1], x[3]);
    #pragma unroll
            for (int off = 4; off < 32; off <<= 1) {
                tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, off));
                tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, off));
            }
            const float nA = fmaxf(mA, tA), nB = fmaxf(mB, tB);
            const float cA = exp2f(mA - nA), cB = exp2f(mB - nB);  // mA=-inf -> 0
            mA = nA;
            mB = nB;
            const float p0 = exp2f(x[0] - nA), p1 = exp2f(x[1] - nB), p2 = exp2f(x[2] - nA), p3 = exp2f(x[3] - nB);
            sA = sA * cA + p0 + p2;
            sB = sB * cB + p1 + p3;
    #pragma unroll
            for (int mt = 0; mt < KS; ++mt) {
                o[mt][0] *= cA; o[mt][1] *= cB; o[mt][2] *= cA; o[mt][3] *= cB;
                if (!PACKED) { o2[mt][0] *= cA; o2[mt][1] *= cB; o2[mt][2] *= cA; o2[mt][3] *= cB; }
            }
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
                ldsm_x4_t(vst + Geo::off(row, ch), a);
                mma_bf16(o[mt], a, b0, b1);
                if (!PACKED) mma_bf16(o2[mt], a, b2, b3);
            }
            __syncwarp();
        }
        cp_wait<0>();
        __syncthreads();  // before the next segment's ids overwrite ids_s
    }
    cp_wait<0>();

    // ---- warp -> CTA partial
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
        sA += __shfl_xor_sync(0xffffffffu, sA, off);
        sB += __shfl_xor_sync(0xffffffffu, sB, off);
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
            for (int j = 0; j < 4; ++j) o[mt][j] += o2[mt][j];
    }
    __syncthreads();  // all warps done with their stage buffers: reuse smem for the reduction
    float* red = reinterpret_cast<float*>(smem);  // [warps][8 heads][2 + D]
    const bool owner = PACKED ? tq < 2 : true;
    if (owner) {
        float* rA = red + ((size_t)w * 8 + hA) * (2 + D);
        float* rB = red + ((size_t)w * 8 + hB) * (2 + D);
        if (gr == 0) {
            rA[0] = mA; rA[1] = sA;
            rB[0] = mB; rB[1] = sB;
        }
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
            rA[2 + mt * 16 + gr] = o[mt][0];
            rB[2 + mt * 16 + gr] = o[mt][1];
            rA[2 + mt * 16 + gr + 8] = o[mt][2];
            rB[2 + mt * 16 + gr + 8] = o[mt][3];
        }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
        const int g = idx / D, k = idx - g * D;
        float M = -INFINITY;
        for (int ww = 0; ww < kMmaWarps; ++ww) M = fmaxf(M, red[((size_t)ww * 8 + g) * (2 + D)]);
        float sum = 0.f, a = 0.f;
        if (M != -INFINITY)
            for (int ww = 0; ww < kMmaWarps; ++ww) {
                const float* p = red + ((size_t)ww * 8 + g) * (2 + D);
                if (p[0] == -INFINITY) continue;
                const float c = exp2f(p[0] - M);
                sum += c * p[1];
                a += c * p[2 + k];
            }
        part_acc[(((size_t)l * S + s) * G + g) * D + k] = a;
        if (k == 0) {
            part_ml[(((size_t)l * S + s) * G + g) * 2] = M;
            part_ml[(((size_t)l * S + s) * G + g) * 2 + 1] = sum;
        }
    }
    if (take_ticket(ticket, l, S)) merge_splits<true>(l, S, G, D, part_ml, part_acc, out);
}

}  // namespace mpa

using namespace mpa;

namespace {

template <int G>
int launch_ffma(const mpa_cache* c, const float* q_rot, const int32_t* tok, const int32_t* n_tok, int tok_cap,
                const int32_t* rej, const float* rej_w, const int32_t* n_rej, int rej_cap, const void* fvc, int fcap,
                const void* cvc, int ccap, int S, float* pml, float* pacc, int32_t* ticket, float* out,
                cudaStream_t st) {
    const int d = c->head_dim;
    const int ndl = ceil_div(d, 32);
    dim3 grid(S, c->n_ledgers);
    const size_t smem = sizeof(float) * kFfmaWarps * G * (2 + d);
#define MPA_FFMA_CASE(T, NDL)                                                                                   \
    {                                                                                                           \
        auto kern = decode_ffma_kernel<T, G, NDL>;                                                              \
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        kern<<<grid, kFfmaWarps * 32, smem, st>>>((const T*)c->k_rot, (const T*)c->v, c->tcap, d, q_rot, tok,   \
                                                  n_tok, tok_cap, rej, rej_w, n_rej, rej_cap, (const T*)fvc,    \
                                                  fcap, (const T*)cvc, ccap, S, pml, pacc, ticket, out);        \
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

template <int G, int D>
int launch_mma(const mpa_cache* c, const float* q_rot, const int32_t* tok, const int32_t* n_tok, int tok_cap,
               const int32_t* rej, const float* rej_w, const int32_t* n_rej, int rej_cap, const void* fvc, int fcap,
               const void* cvc, int ccap, int S, float* pml, float* pacc, int32_t* ticket, float* out,
               cudaStream_t st) {
    constexpr int NST = 3;
    dim3 grid(S, c->n_ledgers);
    const size_t stage_bytes = (size_t)kMmaWarps * NST * 2 * TileGeom<D>::kMatBytes + kSegTiles * 16 * sizeof(int);
    const size_t red_bytes = sizeof(float) * kMmaWarps * 8 * (2 + D);
    const size_t smem = stage_bytes > red_bytes ? stage_bytes : red_bytes;
    auto kern = decode_mma_kernel<G, D, NST>;
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set = true;
    }
    kern<<<grid, kMmaWarps * 32, smem, st>>>((const __nv_bfloat16*)c->k_rot, (const __nv_bfloat16*)c->v, c->tcap,
                                             q_rot, tok, n_tok, tok_cap, rej, rej_w, n_rej, rej_cap,
                                             (const __nv_bfloat16*)fvc, fcap, (const __nv_bfloat16*)cvc, ccap, S, pml,
                                             pacc, ticket, out);
    return check_launch("mpa_sparse_decode(mma)");
}

int g_force_ffma = -1;

bool force_ffma() {
    if (g_force_ffma < 0) {
        const char* e = getenv("MPA_FORCE_FFMA");
        g_force_ffma = (e && e[0] == '1') ? 1 : 0;
    }
    return g_force_ffma == 1;
}

}  // namespace

extern "C" int mpa_sparse_decode(const mpa_cache* c, const float* q_rot, int n_kv_heads, int group,
                                 const int32_t* tok, const int32_t* n_tok, int tok_cap, const int32_t* rej,
                                 const float* rej_w, const int32_t* n_rej, int rej_cap, const void* fine_vc,
                                 int fine_cap, const void* coarse_vc, int coarse_cap, int n_split, float* part_ml,
                                 float* part_acc, int32_t* ticket, float* out, void* stream) {
    MPA_REQUIRE(c && q_rot && n_tok && part_ml && part_acc && ticket && out, MPA_ERR_ARG,
                "mpa_sparse_decode: null argument");
    MPA_REQUIRE(!rej || (rej_w && n_rej), MPA_ERR_ARG, "mpa_sparse_decode: rej without weights/counts");
    MPA_REQUIRE(n_split >= 1, MPA_ERR_ARG, "mpa_sparse_decode: n_split %d", n_split);
    MPA_REQUIRE(c->head_dim >= 2 && c->head_dim % 2 == 0 && c->head_dim <= 256, MPA_ERR_UNSUPPORTED,
                "mpa_sparse_decode: head_dim %d", c->head_dim);
    (void)n_kv_heads;
    if (c->n_ledgers <= 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const bool mma_ok = c->dtype == MPA_BF16 && (c->head_dim == 64 || c->head_dim == 128) && group <= 8 &&
                        !force_ffma();
    if (mma_ok) {
        MPA_DISPATCH_G(group, {
            if (c->head_dim == 128)
                return launch_mma<kG, 128>(c, q_rot, tok, n_tok, tok_cap, rej, rej_w, n_rej, rej_cap, fine_vc,
                                           fine_cap, coarse_vc, coarse_cap, n_split, part_ml, part_acc, ticket, out,
                                           st);
            return launch_mma<kG, 64>(c, q_rot, tok, n_tok, tok_cap, rej, rej_w, n_rej, rej_cap, fine_vc, fine_cap,
                                      coarse_vc, coarse_cap, n_split, part_ml, part_acc, ticket, out, st);
        });
    }
    MPA_DISPATCH_G(group, {
        return launch_ffma<kG>(c, q_rot, tok, n_tok, tok_cap, rej, rej_w, n_rej, rej_cap, fine_vc, fine_cap,
                               coarse_vc, coarse_cap, n_split, part_ml, part_acc, ticket, out, st);
    });
    return 0;
}
