// K9 centroid lookup logits, K10 budgeted selection, and the work-list builder that feeds
// the fused decode kernel.
//
// Reference (pkg/src/multipole_attn/attention.py):
//   :267-290 `_scores_per_group`  logits = Q_lk Kc^T / sqrt(d); e = exp(l - max_g);
//                                  score = mean_g e / (e . N)
//   :192-207 `select_clusters`    visit by (score desc, ref asc); take while cum < B
//   :293-351 `hierarchical_lookup` promote coarse to ceil(p*total), fine children scored with
//                                  the union denominator {promoted fine} U {rejected coarse}
//   :354-375 `flat_lookup`, :469-496 work of one kv-head (sinks, buffer, selected, rejected)
//
// Numerics: logits, exps, normalisers and scores are fp64 like the reference, so the
// selected set matches the oracle except at true ties (|score gap| ~ 1e-16 relative).
// Selection is a size-weighted radix select on the 96-bit key (~score_bits, cluster id):
// it finds the crossing cluster without sorting, O(passes * n / threads).
#include <cstdlib>

#include "mpa_common.cuh"

namespace mpa {

constexpr int kLogitsThreads = 128;

// One thread per candidate centroid; q_lookup rows of the GQA group staged in smem.
template <typename T, int G>
__global__ void __launch_bounds__(kLogitsThreads)
centroid_logits_kernel(const double* __restrict__ q_lk, int n_kv_heads, int d, const T* __restrict__ kc, int kcap,
                       const int32_t* __restrict__ count, const int32_t* __restrict__ cand,
                       const int32_t* __restrict__ n_cand, int cand_cap, double* __restrict__ logits) {
    extern __shared__ double qs[];  // [G][d]
    const int l = blockIdx.y;
    const int n = cand ? n_cand[l] : count[l];
    const int i0 = blockIdx.x * kLogitsThreads;
    if (i0 >= n) return;
    const double* qsrc = q_lk + (size_t)l * G * d;  // q-heads of this ledger are contiguous
    for (int j = threadIdx.x; j < G * d; j += blockDim.x) qs[j] = qsrc[j];
    __syncthreads();
    const int i = i0 + threadIdx.x;
    if (i >= n) return;
    const int row = cand ? cand[(size_t)l * cand_cap + i] : i;
    const T* kr = kc + ((size_t)l * kcap + row) * d;
    double acc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g] = 0.0;
    for (int k = 0; k < d; ++k) {
        const double x = elem<T>::to_d(kr[k]);
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = fma(qs[g * d + k], x, acc[g]);
    }
    const double sq = sqrt((double)d);
    double* out = logits + (size_t)l * G * cand_cap + i;
#pragma unroll
    for (int g = 0; g < G; ++g) out[(size_t)g * cand_cap] = acc[g] / sq;
}

// Tiled variant for d in {64, 128}: a CTA stages kChunk centroid rows of one ledger with
// coalesced 16-byte loads into padded smem (all loads in flight at once), then each thread
// computes one centroid's G dot products in fp64 reading q_lookup interleaved [d][G] from smem
// (warp-broadcast 16-byte loads).  ~40 registers and ~40 KB smem per CTA keep several CTAs
// resident per SM so the tile loads of one CTA overlap the fp64 math of the others.  The CTA
// also emits the chunk's per-head (max, sum N e^(l - max)) partials of the Eq. 1 normaliser.
constexpr int kChunk = 128;
constexpr int kTiledThreads = 128;

template <typename T, int G, int D>
__global__ void __launch_bounds__(kTiledThreads)
centroid_logits_tiled(const double* __restrict__ q_lk, const T* __restrict__ kc, int kcap,
                      const int32_t* __restrict__ count, const int32_t* __restrict__ lv_size,
                      const int32_t* __restrict__ cand, const int32_t* __restrict__ n_cand, int cand_cap,
                      double* __restrict__ logits, double* __restrict__ cstats, int n_chunks) {
    constexpr int EPC = 16 / (int)sizeof(T);              // elements per 16-byte chunk
    constexpr int CPR = D / EPC;                          // chunks per row
    constexpr int ROWB = D * (int)sizeof(T) + 16;         // padded row bytes (conflict-free LDS.128)
    constexpr int GP = (G + 1) & ~1;                      // q row padded to an even count of doubles
    extern __shared__ __align__(16) unsigned char sm[];
    double* qs = reinterpret_cast<double*>(sm);                        // [D][GP]
    double* red = qs + D * GP;                                         // [4 warps][G][2]
    unsigned char* tile = reinterpret_cast<unsigned char*>(red + 4 * G * 2);
    const int l = blockIdx.y, chunk = blockIdx.x;
    const int n = cand ? n_cand[l] : count[l];
    const int i0 = chunk * kChunk;
    if (i0 >= n) {
        if (cstats && threadIdx.x < G) {
            cstats[(((size_t)l * n_chunks + chunk) * G + threadIdx.x) * 2] = -INFINITY;
            cstats[(((size_t)l * n_chunks + chunk) * G + threadIdx.x) * 2 + 1] = 0.0;
        }
        return;
    }
    const int nv = min(kChunk, n - i0);
    for (int j = threadIdx.x; j < G * D; j += blockDim.x) {
        const int g = j / D, k = j - g * D;
        qs[k * GP + g] = q_lk[(size_t)l * G * D + j];
    }
    {
        constexpr int PER = 16;  // 16-byte loads in flight per thread
        constexpr int TOTAL = kChunk * CPR;
        for (int base = 0; base < TOTAL; base += PER * kTiledThreads) {
            uint4 v[PER];
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int j = base + threadIdx.x + e * kTiledThreads;
                const int r = j / CPR, c = j - r * CPR;
                v[e] = make_uint4(0u, 0u, 0u, 0u);
                if (j < TOTAL && r < nv) {
                    const int row = cand ? __ldg(cand + (size_t)l * cand_cap + i0 + r) : i0 + r;
                    v[e] = __ldg(reinterpret_cast<const uint4*>(kc + ((size_t)l * kcap + row) * D) + c);
                }
            }
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int j = base + threadIdx.x + e * kTiledThreads;
                const int r = j / CPR, c = j - r * CPR;
                if (j < TOTAL) *reinterpret_cast<uint4*>(tile + r * ROWB + c * 16) = v[e];
            }
        }
    }
    __syncthreads();
    const int r = threadIdx.x;
    double acc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g] = 0.0;
#pragma unroll 2
    for (int c = 0; c < CPR; ++c) {
        const uint4 raw = *reinterpret_cast<const uint4*>(tile + r * ROWB + c * 16);
        double xv[EPC];
        unpack16<T>::run(raw, xv);
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
            const double* qk = qs + (c * EPC + e) * GP;
            double qv[GP];
#pragma unroll
            for (int g = 0; g < GP; g += 2) {
                const double2 t = *reinterpret_cast<const double2*>(qk + g);
                qv[g] = t.x;
                qv[g + 1] = t.y;
            }
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = fma(qv[g], xv[e], acc[g]);
        }
    }
    const double sq = sqrt((double)D);
    const bool valid = r < nv;
    double lg[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        lg[g] = acc[g] / sq;
        if (valid) logits[((size_t)l * G + g) * cand_cap + i0 + r] = lg[g];
    }
    if (!cstats) return;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int id = valid ? (cand ? cand[(size_t)l * cand_cap + i0 + r] : i0 + r) : 0;
    const double nsz = valid ? (double)lv_size[(size_t)l * kcap + id] : 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const double m = warp_max(valid ? lg[g] : -INFINITY);
        const double z = warp_sum(valid ? nsz * exp(lg[g] - m) : 0.0);
        if (lane == 0) {
            red[(w * G + g) * 2] = m;
            red[(w * G + g) * 2 + 1] = z;
        }
    }
    __syncthreads();
    if (threadIdx.x < G) {
        const int g = threadIdx.x;
        double M = -INFINITY;
        for (int ww = 0; ww < kTiledThreads / 32; ++ww) M = fmax(M, red[(ww * G + g) * 2]);
        double Z = 0.0;
        for (int ww = 0; ww < kTiledThreads / 32; ++ww) {
            const double m = red[(ww * G + g) * 2];
            if (m != -INFINITY) Z += red[(ww * G + g) * 2 + 1] * exp(m - M);
        }
        cstats[(((size_t)l * n_chunks + chunk) * G + g) * 2] = M;
        cstats[(((size_t)l * n_chunks + chunk) * G + g) * 2 + 1] = Z;
    }
}

// ---------------------------------------------------------------------------
// K10 selection. One CTA per ledger.

constexpr int kSelThreads = 1024;
constexpr int kBitonicMax = 8192;

__host__ __device__ __forceinline__ int sort_width(int cap) {
    int p = 1;
    while (p < cap) p <<= 1;
    if (p > kBitonicMax) p = cap;  // radix path only needs cap entries
    return p > cap ? p : cap;
}

__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double dsum(double a, double b) { return a + b; }

template <int G>
__device__ void select_core(const int l, const double* __restrict__ logits, const int32_t* __restrict__ cand,
                            const int32_t* __restrict__ n_cand, int cand_cap, const int32_t* __restrict__ lv_size,
                            int lv_cap, const double* __restrict__ elogits, const int32_t* __restrict__ esize,
                            const uint8_t* __restrict__ eflag, const int32_t* __restrict__ n_extra, int ecap,
                            const int64_t* __restrict__ budget, uint8_t* __restrict__ flag,
                            int32_t* __restrict__ sel_tokens, const double* __restrict__ cstats, int n_chunks,
                            unsigned char* smem_raw, int smem_n) {
    const int n = n_cand[l];
    // smem: keys / ids / pos sized P = max(cand_cap, bitonic width), sizes [cand_cap]
    const int P = sort_width(smem_n);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem_raw);  // [P]
    int* ids = reinterpret_cast<int*>(keys + P);                                  // [P]
    int* pos = ids + P;                                                           // [P]
    int* sizes = pos + P;                                                         // [smem_n]
    __shared__ double red[32];
    __shared__ unsigned int hist_w[256];
    __shared__ unsigned int hist_c[256];
    __shared__ unsigned long long s_prefix;
    __shared__ long long s_below;
    __shared__ int s_done;

    const double* lg = logits + (size_t)l * G * cand_cap;
    const int ne = elogits ? n_extra[l] : 0;
    const double* elg = elogits ? elogits + (size_t)l * G * ecap : nullptr;

    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int id = cand ? cand[(size_t)l * cand_cap + i] : i;
        ids[i] = id;
        sizes[i] = lv_size[(size_t)l * lv_cap + id];
    }
    __syncthreads();

    // per-head max and size-weighted normaliser over candidates + live extras
    double mx[G], z[G];
    const double* cs = cstats ? cstats + (size_t)l * n_chunks * G * 2 : nullptr;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        double m = -INFINITY;
        if (cs)
            for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) m = dmax(m, cs[(c * G + g) * 2]);
        else
            for (int i = threadIdx.x; i < n; i += blockDim.x) m = dmax(m, lg[(size_t)g * cand_cap + i]);
        for (int j = threadIdx.x; j < ne; j += blockDim.x)
            if (!eflag[(size_t)l * ecap + j]) m = dmax(m, elg[(size_t)g * ecap + j]);
        mx[g] = block_reduce(m, red, dmax);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
        double s = 0.0;
        if (cs) {
            for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) {
                const double cm = cs[(c * G + g) * 2];
                if (cm != -INFINITY) s += cs[(c * G + g) * 2 + 1] * exp(cm - mx[g]);
            }
        } else {
            for (int i = threadIdx.x; i < n; i += blockDim.x)
                s += (double)sizes[i] * exp(lg[(size_t)g * cand_cap + i] - mx[g]);
        }
        for (int j = threadIdx.x; j < ne; j += blockDim.x)
            if (!eflag[(size_t)l * ecap + j])
                s += (double)esize[(size_t)l * ecap + j] * exp(elg[(size_t)g * ecap + j] - mx[g]);
        z[g] = block_reduce(s, red, dsum);
    }
    // score_i = (sum_g e_gi / Z_g) / G, accumulated in head order like np.mean(axis=0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double sc = exp(lg[i] - mx[0]) / z[0];
#pragma unroll
        for (int g = 1; g < G; ++g) sc = sc + exp(lg[(size_t)g * cand_cap + i] - mx[g]) / z[g];
        sc = sc / (double)G;
        keys[i] = ~(unsigned long long)__double_as_longlong(sc);  // ascending key == descending score
    }
    if (threadIdx.x == 0) {
        s_prefix = 0ull;
        s_below = 0;
        s_done = 0;
    }
    __syncthreads();

    const long long B = budget[l];
    long long total = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) total += sizes[i];
    total = block_reduce(total, reinterpret_cast<long long*>(red), [](long long a, long long b) { return a + b; });

    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    if (np2 <= kBitonicMax) {
        // ---- bitonic sort of (key asc, id asc) in smem, then a size prefix sum in sorted order:
        // candidate at sorted rank k is selected iff sum of sizes of ranks < k is < B.
        for (int i = threadIdx.x; i < np2; i += blockDim.x) {
            pos[i] = i;
            if (i >= n) {
                keys[i] = ~0ull;
                ids[i] = 0x7fffffff;
            }
        }
        __syncthreads();
        for (int k = 2; k <= np2; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < np2; i += blockDim.x) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const unsigned long long ka = keys[i], kb = keys[ixj];
                        const int ia = ids[i], ib = ids[ixj];
                        const bool gt = ka > kb || (ka == kb && ia > ib);
                        if (gt == ((i & k) == 0)) {
                            keys[i] = kb;
                            keys[ixj] = ka;
                            ids[i] = ib;
                            ids[ixj] = ia;
                            const int t = pos[i];
                            pos[i] = pos[ixj];
                            pos[ixj] = t;
                        }
                    }
                }
                __syncthreads();
            }
        }
        __shared__ int scan_s[33];
        long long base = 0, tok = 0;
        for (int i0 = 0; i0 < n; i0 += blockDim.x) {
            const int i = i0 + threadIdx.x;
            const int sz = i < n ? sizes[pos[i]] : 0;
            int tot;
            const long long before = base + block_exclusive_scan(sz, scan_s, &tot);
            if (i < n) {
                const bool sel = before < B;
                flag[(size_t)l * cand_cap + pos[i]] = sel ? 1 : 0;
                if (sel) tok += sz;
            }
            base += tot;
        }
        tok = block_reduce(tok, reinterpret_cast<long long*>(red), [](long long a, long long b) { return a + b; });
        if (threadIdx.x == 0 && sel_tokens) sel_tokens[l] = (int32_t)tok;
        return;
    }

    // crossing key (key*, id*): smallest composite key with W(<=) >= B. None -> select all.
    unsigned long long kstar = ~0ull;
    int idstar = 0x7fffffff;
    bool select_all = total < B;
    bool select_none = B <= 0;
    if (!select_all && !select_none) {
        // 8 digit passes over the 64-bit score key, then 4 over the 32-bit id.
        unsigned long long kmask = 0ull;
        unsigned int imask = 0u, iprefix = 0u;
        for (int pass = 0; pass < 12; ++pass) {
            for (int j = threadIdx.x; j < 256; j += blockDim.x) hist_w[j] = hist_c[j] = 0u;
            __syncthreads();
            const unsigned long long kp = s_prefix;
            const int sh = pass < 8 ? 56 - 8 * pass : 24 - 8 * (pass - 8);
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                if ((keys[i] & kmask) != kp) continue;
                if (((unsigned)ids[i] & imask) != iprefix) continue;
                const unsigned dg = pass < 8 ? (unsigned)(keys[i] >> sh) & 255u : ((unsigned)ids[i] >> sh) & 255u;
                atomicAdd(&hist_w[dg], (unsigned)sizes[i]);
                atomicAdd(&hist_c[dg], 1u);
            }
            __syncthreads();
            if (threadIdx.x < 32) {
                // warp 0 scans 256 bins: lane owns bins [8*lane, 8*lane+8)
                const int lane = threadIdx.x;
                unsigned long long w8 = 0;
                for (int j = 0; j < 8; ++j) w8 += hist_w[lane * 8 + j];
                unsigned long long incl = w8;
                for (int o = 1; o < 32; o <<= 1) {
                    unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const long long below = s_below;
                const long long need = B - below;  // > 0
                const unsigned ballot = __ballot_sync(0xffffffffu, (long long)incl >= need);
                const int owner = __ffs(ballot) - 1;  // first lane whose inclusive sum reaches need
                if (lane == owner) {
                    long long run = (long long)(incl - w8);
                    int dg = lane * 8;
                    for (int j = 0; j < 8; ++j) {
                        if (run + (long long)hist_w[lane * 8 + j] >= need) { dg = lane * 8 + j; break; }
                        run += hist_w[lane * 8 + j];
                    }
                    s_below = below + run;
                    if (pass < 8) s_prefix = kp | ((unsigned long long)dg << sh);
                    else s_prefix = kp;
                    // digit for id passes is returned through s_done's upper bits
                    s_done = (hist_c[dg] == 1u ? 1 : 0) | (dg << 8);
                }
            }
            __syncthreads();
            const int dg = s_done >> 8;
            if (pass < 8) kmask |= 255ull << sh;
            else {
                imask |= 255u << sh;
                iprefix |= (unsigned)dg << sh;
            }
            const bool unique = s_done & 1;
            __syncthreads();
            if (unique || pass == 11) {
                // the unique (or fully-resolved) element matching the prefix is the crosser
                for (int i = threadIdx.x; i < n; i += blockDim.x)
                    if ((keys[i] & kmask) == s_prefix && ((unsigned)ids[i] & imask) == iprefix) {
                        kstar = keys[i];
                        idstar = ids[i];
                    }
                break;
            }
        }
        // broadcast crosser
        __shared__ unsigned long long s_k;
        __shared__ int s_id;
        if (threadIdx.x == 0) s_id = -1;
        __syncthreads();
        if (idstar != 0x7fffffff) {
            s_k = kstar;
            s_id = idstar;
        }
        __syncthreads();
        kstar = s_k;
        idstar = s_id;
    }
    long long tok = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        bool sel;
        if (select_none) sel = false;
        else if (select_all) sel = true;
        else sel = keys[i] < kstar || (keys[i] == kstar && ids[i] <= idstar);
        flag[(size_t)l * cand_cap + i] = sel ? 1 : 0;
        if (sel) tok += sizes[i];
    }
    tok = block_reduce(tok, reinterpret_cast<long long*>(red), [](long long a, long long b) { return a + b; });
    if (threadIdx.x == 0 && sel_tokens) sel_tokens[l] = (int32_t)tok;
}

template <int G>
__global__ void __launch_bounds__(kSelThreads)
select_kernel(const double* __restrict__ logits, const int32_t* __restrict__ cand, const int32_t* __restrict__ n_cand,
              int cand_cap, const int32_t* __restrict__ lv_size, int lv_cap, const double* __restrict__ elogits,
              const int32_t* __restrict__ esize, const uint8_t* __restrict__ eflag, const int32_t* __restrict__ n_extra,
              int ecap, const int64_t* __restrict__ budget, uint8_t* __restrict__ flag,
              int32_t* __restrict__ sel_tokens, const double* __restrict__ cstats, int n_chunks, int smem_n) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    select_core<G>(blockIdx.x, logits, cand, n_cand, cand_cap, lv_size, lv_cap, elogits, esize, eflag, n_extra, ecap,
                   budget, flag, sel_tokens, cstats, n_chunks, smem_raw, smem_n);
}

// ---------------------------------------------------------------------------

constexpr int kListThreads = 1024;

__global__ void __launch_bounds__(kListThreads)
hier_candidates_kernel(const int32_t* __restrict__ ccount, const int32_t* __restrict__ child_off,
                       const int32_t* __restrict__ child, int ccap, int child_cap, const uint8_t* __restrict__ cflag,
                       int32_t* __restrict__ cand, int32_t* __restrict__ n_cand, int cand_cap) {
    __shared__ int scan[33];
    pdl_wait();  // cflag comes from the coarse selection (PDL predecessor)
    pdl_trigger();
    const int l = blockIdx.x;
    const int nc = ccount[l];
    const int32_t* off = child_off + (size_t)l * (ccap + 1);
    int base = 0;
    for (int c0 = 0; c0 < nc; c0 += blockDim.x) {
        const int c = c0 + threadIdx.x;
        const int cnt = (c < nc && cflag[(size_t)l * ccap + c]) ? off[c + 1] - off[c] : 0;
        int tot;
        const int pos = base + block_exclusive_scan(cnt, scan, &tot);
        // children copied 8 at a time: the loads of a batch are in flight together
        const int32_t* src = child + (size_t)l * child_cap + (cnt ? off[c] : 0);
        int32_t* dst = cand + (size_t)l * cand_cap + pos;
        for (int j0 = 0; j0 < cnt; j0 += 8) {
            int v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = j0 + u < cnt ? __ldg(src + j0 + u) : 0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (j0 + u < cnt && pos + j0 + u < cand_cap) dst[j0 + u] = v[u];
        }
        base += tot;
    }
    if (threadIdx.x == 0) n_cand[l] = base < cand_cap ? base : cand_cap;
}

template <int G>
__device__ void worklist_body(const int l, const int L, const int32_t* __restrict__ fsize, const int32_t* __restrict__ fmem_off,
                      const int32_t* __restrict__ fmem, int fcap, int fmem_cap, const int32_t* __restrict__ csize,
                      const int32_t* __restrict__ ccount, int ccap, const int32_t* __restrict__ cand,
                      const int32_t* __restrict__ n_cand, const int32_t* __restrict__ fcount, int cand_cap,
                      const uint8_t* __restrict__ flag, const double* __restrict__ logits,
                      const uint8_t* __restrict__ cflag, const double* __restrict__ clogits,
                      const int32_t* __restrict__ sink_end, const int32_t* __restrict__ buffer_start,
                      const int32_t* __restrict__ cache_len, int n_kv_heads, int replacement,
                      int32_t* __restrict__ tok, int tok_cap, int32_t* __restrict__ rej, float* __restrict__ rej_w,
                      int rej_cap, int32_t* __restrict__ stats) {
    __shared__ int scan[33];
    const int seq = l / n_kv_heads;
    const int clen = cache_len[seq];
    const int ns = min(sink_end[seq], clen);
    const int bs = buffer_start[seq];
    const int nb = max(0, clen - bs);
    int32_t* T = tok + (size_t)l * tok_cap;
    for (int j = threadIdx.x; j < ns; j += blockDim.x) T[j] = j;
    for (int j = threadIdx.x; j < nb; j += blockDim.x) T[ns + j] = bs + j;
    const int n = cand ? n_cand[l] : fcount[l];
    int tbase = ns + nb, rbase = 0, nsel = 0;
    const int32_t* moff = fmem_off + (size_t)l * (fcap + 1);
    for (int i0 = 0; i0 < n; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        int id = 0, sz = 0, sel = 0;
        if (i < n) {
            id = cand ? cand[(size_t)l * cand_cap + i] : i;
            sz = fsize[(size_t)l * fcap + id];
            sel = flag[(size_t)l * cand_cap + i];
        }
        int ttot, rtot, stot;
        const int tpos = tbase + block_exclusive_scan(sel ? sz : 0, scan, &ttot);
        const int rpos = rbase + block_exclusive_scan((i < n && !sel && replacement) ? 1 : 0, scan, &rtot);
        block_exclusive_scan(sel, scan, &stot);
        if (i < n && sel) {
            const int32_t* m = fmem + (size_t)l * fmem_cap + moff[id];
            for (int j = 0; j < sz && tpos + j < tok_cap; ++j) T[tpos + j] = m[j];
        }
        if (i < n && !sel && replacement && rpos < rej_cap) {
            rej[(size_t)l * rej_cap + rpos] = id;
            const double lnN = log((double)sz);
#pragma unroll
            for (int g = 0; g < G; ++g)
                rej_w[((size_t)l * rej_cap + rpos) * (G <= 4 ? 4 : 8) + g] =
                    (float)(logits[((size_t)l * G + g) * cand_cap + i] + lnN);
        }
        tbase += ttot;
        rbase += rtot;
        nsel += stot;
    }
    if (cflag && replacement) {
        const int nc = ccount[l];
        for (int c0 = 0; c0 < nc; c0 += blockDim.x) {
            const int c = c0 + threadIdx.x;
            const int r = (c < nc && !cflag[(size_t)l * ccap + c]) ? 1 : 0;
            int rtot;
            const int rpos = rbase + block_exclusive_scan(r, scan, &rtot);
            if (r && rpos < rej_cap) {
                rej[(size_t)l * rej_cap + rpos] = -1 - c;
                const double lnN = log((double)csize[(size_t)l * ccap + c]);
#pragma unroll
                for (int g = 0; g < G; ++g)
                    rej_w[((size_t)l * rej_cap + rpos) * (G <= 4 ? 4 : 8) + g] =
                        (float)(clogits[((size_t)l * G + g) * ccap + c] + lnN);
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

#define MPA_WORKLIST_PARAMS                                                                                      \
    const int32_t *__restrict__ fsize, const int32_t *__restrict__ fmem_off, const int32_t *__restrict__ fmem,   \
        int fcap, int fmem_cap, const int32_t *__restrict__ csize, const int32_t *__restrict__ ccount, int ccap, \
        const int32_t *__restrict__ fcount, const uint8_t *__restrict__ cflag, const double *__restrict__ clogits, \
        const int32_t *__restrict__ sink_end, const int32_t *__restrict__ buffer_start,                           \
        const int32_t *__restrict__ cache_len, int n_kv_heads, int replacement, int32_t *__restrict__ tok,         \
        int tok_cap, int32_t *__restrict__ rej, float *__restrict__ rej_w, int rej_cap, int32_t *__restrict__ stats
#define MPA_WORKLIST_ARGS(cand, n_cand, cand_cap, flag, logits)                                                   \
    fsize, fmem_off, fmem, fcap, fmem_cap, csize, ccount, ccap, cand, n_cand, fcount, cand_cap, flag, logits,     \
        cflag, clogits, sink_end, buffer_start, cache_len, n_kv_heads, replacement, tok, tok_cap, rej, rej_w,     \
        rej_cap, stats

// K10 + work list in one launch per ledger (the flat path and the hierarchy's fine stage).
template <int G>
__global__ void __launch_bounds__(kSelThreads)
select_worklist_kernel(const double* __restrict__ logits, const int32_t* __restrict__ cand,
                       const int32_t* __restrict__ n_cand, int cand_cap, const int64_t* __restrict__ budget,
                       uint8_t* __restrict__ flag, int32_t* __restrict__ sel_tokens,
                       const double* __restrict__ cstats, int n_chunks, int smem_n, MPA_WORKLIST_PARAMS) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int l = blockIdx.x;
    select_core<G>(l, logits, cand, n_cand ? n_cand : fcount, cand_cap, fsize, fcap, clogits, csize, cflag, ccount,
                   ccap, budget, flag, sel_tokens, cstats, n_chunks, smem_raw, smem_n);
    __syncthreads();
    worklist_body<G>(l, gridDim.x, MPA_WORKLIST_ARGS(cand, n_cand, cand_cap, flag, logits));
}

}  // namespace mpa

using namespace mpa;

// serving kernels (mpa_select.cu)
int mpa_launch_logits_v2(const double* q_lk, int group, int d, const mpa_level* lv, const int32_t* cand,
                         const int32_t* n_cand, int cand_cap, double* logits, double* chunk_stats, double* e_local,
                         int n_chunks, int n_max, float* rej_w, int rej_cap, const float* q_raw,
                         const double* cs_lk, cudaStream_t st);
size_t mpa_select_v2_smem(int n_max);
int mpa_launch_select_v2(const double* logits, const double* e_local, int group, const int32_t* cand,
                         const int32_t* n_cand, int cand_cap, const int32_t* lv_size, int lv_cap,
                         const double* elogits, const int32_t* esize, const uint8_t* eflag, const int32_t* n_extra,
                         int ecap, const int64_t* budget, int n_ledgers, uint8_t* flag, int32_t* sel_tokens,
                         const double* chunk_stats, int n_chunks, int n_max, cudaStream_t st);
int mpa_launch_select_worklist_v2(const mpa_level* fine, const mpa_level* coarse, int group, const double* logits,
                                  const double* e_local, const int32_t* cand, const int32_t* n_cand, int cand_cap,
                                  const double* chunk_stats, int n_chunks, const uint8_t* cflag,
                                  const double* clogits, const int64_t* budget, const int32_t* sink_end,
                                  const int32_t* buffer_start, const int32_t* cache_len, int n_kv_heads,
                                  int n_ledgers, int replacement, uint8_t* flag, int32_t* sel_tokens, int32_t* tok,
                                  int tok_cap, int32_t* rej, float* rej_w, int rej_cap, int32_t* stats, int n_max,
                                  cudaStream_t st);

extern "C" int mpa_centroid_logits(const double* q_lk, int n_kv_heads, int group, int d, const mpa_level* lv,
                                   const int32_t* cand, const int32_t* n_cand, int cand_cap, double* logits,
                                   double* chunk_stats, double* e_local, int n_max, float* rej_w, int rej_cap,
                                   const float* q_raw, const double* cs_lk, void* stream) {
    MPA_REQUIRE((q_lk || (q_raw && cs_lk)) && lv && lv->kc && lv->count, MPA_ERR_ARG,
                "mpa_centroid_logits: null argument");
    MPA_REQUIRE(logits || rej_w, MPA_ERR_ARG, "mpa_centroid_logits: logits may be NULL only with rej_w");
    MPA_REQUIRE(!cand || n_cand, MPA_ERR_ARG, "mpa_centroid_logits: cand without n_cand");
    MPA_REQUIRE(cand ? cand_cap >= 1 : cand_cap >= lv->cap, MPA_ERR_ARG, "mpa_centroid_logits: cand_cap %d too small",
                cand_cap);
    MPA_REQUIRE(!chunk_stats || lv->size, MPA_ERR_ARG, "mpa_centroid_logits: chunk stats need sizes");
    (void)n_kv_heads;
    const int L = lv->n_ledgers;
    if (L <= 0) return 0;
    const int cap = cand ? cand_cap : lv->cap;
    cudaStream_t st = (cudaStream_t)stream;
    // bf16 centroids (the serving dtype): TMA / smem-blocked kernels of mpa_select.cu; fp32 / fp64
    // centroids (parity modes): smem-tiled kernel at d in {64, 128}, the generic kernel otherwise
    if ((d == 64 || d == 128) && lv->dtype == MPA_BF16)
        return mpa_launch_logits_v2(q_lk, group, d, lv, cand, n_cand, cand_cap, logits, chunk_stats, e_local,
                                    ceil_div(cap, kChunk), n_max > 0 && n_max < cap ? n_max : cap, rej_w, rej_cap,
                                    q_lk ? nullptr : q_raw, q_lk ? nullptr : cs_lk, st);
    MPA_REQUIRE(!rej_w, MPA_ERR_UNSUPPORTED, "mpa_centroid_logits: rej_w needs the bf16 TMA path");
    MPA_REQUIRE(q_lk, MPA_ERR_UNSUPPORTED, "mpa_centroid_logits: the fused lookup rotation needs the bf16 TMA path");
    if (d == 64 || d == 128) {
        const int nch = ceil_div(cap, kChunk);
        dim3 grid(nch, L);
#define MPA_TILED(T, D)                                                                                              \
    {                                                                                                                \
        auto kern = centroid_logits_tiled<T, kG, D>;                                                                 \
        const size_t smem = sizeof(double) * (D * ((kG + 1) & ~1) + 8 * kG) + (size_t)kChunk * (D * sizeof(T) + 16); \
        if (int rc = set_max_smem((const void*)kern, (int)smem)) return rc;                                           \
        kern<<<grid, kTiledThreads, smem, st>>>(q_lk, (const T*)lv->kc, lv->cap, lv->count, lv->size, cand, n_cand,  \
                                                cand_cap, logits, chunk_stats, nch);                                 \
    }
        MPA_DISPATCH_G(group, {
            if (lv->dtype == MPA_BF16) {
                if (d == 128) MPA_TILED(__nv_bfloat16, 128) else MPA_TILED(__nv_bfloat16, 64)
            } else if (lv->dtype == MPA_F32) {
                if (d == 128) MPA_TILED(float, 128) else MPA_TILED(float, 64)
            } else {
                if (d == 128) MPA_TILED(double, 128) else MPA_TILED(double, 64)
            }
        });
#undef MPA_TILED
        return check_launch("mpa_centroid_logits(tiled)");
    }
    MPA_REQUIRE(!chunk_stats, MPA_ERR_UNSUPPORTED, "mpa_centroid_logits: chunk stats need d in {64,128}");
    dim3 grid(ceil_div(cap, kLogitsThreads), L);
    MPA_DISPATCH_G(group, {
        const size_t smem = sizeof(double) * kG * d;
        if (lv->dtype == MPA_F32)
            centroid_logits_kernel<float, kG><<<grid, kLogitsThreads, smem, st>>>(
                q_lk, n_kv_heads, d, (const float*)lv->kc, lv->cap, lv->count, cand, n_cand, cand_cap, logits);
        else if (lv->dtype == MPA_F64)
            centroid_logits_kernel<double, kG><<<grid, kLogitsThreads, smem, st>>>(
                q_lk, n_kv_heads, d, (const double*)lv->kc, lv->cap, lv->count, cand, n_cand, cand_cap, logits);
        else
            centroid_logits_kernel<__nv_bfloat16, kG><<<grid, kLogitsThreads, smem, st>>>(
                q_lk, n_kv_heads, d, (const __nv_bfloat16*)lv->kc, lv->cap, lv->count, cand, n_cand, cand_cap, logits);
    });
    return check_launch("mpa_centroid_logits");
}

static const int kSelectMaxCap = 11264;  // radix path: 20 B of smem per candidate

extern "C" int mpa_select(const double* logits, int group, const int32_t* cand, const int32_t* n_cand, int cand_cap,
                          const int32_t* lv_size, int lv_cap, const double* elogits, const int32_t* esize,
                          const uint8_t* eflag, const int32_t* n_extra, int ecap, const int64_t* budget,
                          int n_ledgers, uint8_t* flag, int32_t* sel_tokens, const double* chunk_stats,
                          const double* e_local, int n_max, void* stream) {
    MPA_REQUIRE(logits && n_cand && lv_size && budget && flag, MPA_ERR_ARG, "mpa_select: null argument");
    MPA_REQUIRE(!elogits || (esize && eflag && n_extra), MPA_ERR_ARG, "mpa_select: incomplete extras");
    if (n_max <= 0 || n_max > cand_cap) n_max = cand_cap;
    MPA_REQUIRE(n_max <= kSelectMaxCap, MPA_ERR_UNSUPPORTED, "mpa_select: %d candidates > %d", n_max,
                kSelectMaxCap);
    if (n_ledgers <= 0) return 0;
    const size_t smem = (size_t)sort_width(n_max) * 16 + (size_t)n_max * 4;
    const int nch = ceil_div(cand_cap, kChunk);
    cudaStream_t st = (cudaStream_t)stream;
    // radix select (one CTA per ledger); the bitonic kernel when its per-candidate smem does not fit
    if (mpa_select_v2_smem(n_max) <= 200 * 1024)
        return mpa_launch_select_v2(logits, e_local, group, cand, n_cand, cand_cap, lv_size, lv_cap, elogits, esize,
                                    eflag, n_extra, ecap, budget, n_ledgers, flag, sel_tokens, chunk_stats, nch, n_max,
                                    st);
    MPA_DISPATCH_G(group, {
        auto kern = select_kernel<kG>;
        if (int rc = set_max_smem((const void*)kern, (int)smem)) return rc;
        kern<<<n_ledgers, kSelThreads, smem, st>>>(logits, cand, n_cand, cand_cap, lv_size, lv_cap, elogits, esize,
                                                   eflag, n_extra, ecap, budget, flag, sel_tokens, chunk_stats, nch,
                                                   n_max);
    });
    return check_launch("mpa_select");
}

extern "C" int mpa_select_worklist(const mpa_level* fine, const mpa_level* coarse, int group, const double* logits,
                                   const double* e_local, const int32_t* cand, const int32_t* n_cand, int cand_cap,
                                   const double* chunk_stats,
                                   const uint8_t* cflag, const double* clogits, const int64_t* budget,
                                   const int32_t* sink_end, const int32_t* buffer_start, const int32_t* cache_len,
                                   int n_kv_heads, int n_ledgers, int replacement, uint8_t* flag,
                                   int32_t* sel_tokens, int32_t* tok, int tok_cap, int32_t* rej, float* rej_w,
                                   int rej_cap, int32_t* stats, int n_max, void* stream) {
    MPA_REQUIRE(logits || (!rej && e_local && chunk_stats), MPA_ERR_ARG,
                "mpa_select_worklist: logits may be NULL only for the contiguous-centroid list");
    MPA_REQUIRE(fine && budget && flag && sink_end && buffer_start && cache_len && tok && rej_w && stats,
                MPA_ERR_ARG, "mpa_select_worklist: null argument");
    MPA_REQUIRE(rej || (!cand && !cflag), MPA_ERR_UNSUPPORTED,
                "mpa_select_worklist: the contiguous-centroid list (rej == NULL) needs the flat level");
    MPA_REQUIRE(!cflag || (coarse && clogits), MPA_ERR_ARG, "mpa_select_worklist: coarse flags without level");
    MPA_REQUIRE(cand ? n_cand != nullptr : cand_cap >= fine->cap, MPA_ERR_ARG,
                "mpa_select_worklist: candidate capacity");
    if (n_max <= 0 || n_max > cand_cap) n_max = cand_cap;
    MPA_REQUIRE(n_max <= kSelectMaxCap, MPA_ERR_UNSUPPORTED, "mpa_select_worklist: %d candidates > %d", n_max,
                kSelectMaxCap);
    if (n_ledgers <= 0) return 0;
    const size_t smem = (size_t)sort_width(n_max) * 16 + (size_t)n_max * 4;
    const int nch = ceil_div(cand_cap, kChunk);
    cudaStream_t st = (cudaStream_t)stream;
    MPA_REQUIRE(rej || mpa_select_v2_smem(n_max) <= 200 * 1024, MPA_ERR_UNSUPPORTED,
                "mpa_select_worklist: contiguous-centroid list needs the radix kernel");
    if (mpa_select_v2_smem(n_max) <= 200 * 1024)
        return mpa_launch_select_worklist_v2(fine, coarse, group, logits, e_local, cand, n_cand, cand_cap,
                                             chunk_stats, nch, cflag, clogits, budget, sink_end, buffer_start,
                                             cache_len, n_kv_heads, n_ledgers, replacement, flag, sel_tokens, tok,
                                             tok_cap, rej, rej_w, rej_cap, stats, n_max, st);
    MPA_DISPATCH_G(group, {
        auto kern = select_worklist_kernel<kG>;
        if (int rc = set_max_smem((const void*)kern, (int)smem)) return rc;
        kern<<<n_ledgers, kSelThreads, smem, st>>>(
            logits, cand, n_cand, cand_cap, budget, flag, sel_tokens, chunk_stats, nch, n_max, fine->size, fine->off,
            fine->idx, fine->cap, fine->idx_cap, coarse ? coarse->size : nullptr, coarse ? coarse->count : nullptr,
            coarse ? coarse->cap : 0, fine->count, cflag, clogits, sink_end, buffer_start, cache_len, n_kv_heads,
            replacement, tok, tok_cap, rej, rej_w, rej_cap, stats);
    });
    return check_launch("mpa_select_worklist");
}

extern "C" int mpa_hier_candidates(const mpa_level* coarse, const uint8_t* cflag, int n_ledgers, int32_t* cand,
                                   int32_t* n_cand, int cand_cap, void* stream) {
    MPA_REQUIRE(coarse && cflag && cand && n_cand && coarse->off && coarse->idx, MPA_ERR_ARG,
                "mpa_hier_candidates: null argument");
    if (n_ledgers <= 0) return 0;
    launch_pdl(hier_candidates_kernel, dim3(n_ledgers), dim3(kListThreads), 0, (cudaStream_t)stream, coarse->count,
               coarse->off, coarse->idx, coarse->cap, coarse->idx_cap, cflag, cand, n_cand, cand_cap);
    return check_launch("mpa_hier_candidates");
}


