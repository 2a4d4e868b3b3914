// K1 / K14: rotary views and KV-cache writes.
//
// Reference: rope.py:37-53 (`rotate`: interleaved pairs (2i, 2i+1) rotated by
// pos * theta^(-2i/d), computed in fp64), rope.py:66-68 (lookup query at the fixed
// offset Delta), attention.py:84-85 (exact view: both q and keys at true positions),
// pipeline.py:38-44 + 156-159 (append the step's key/value after attending).
//
// The rotated key is materialised ONCE per token at write time (K_rot cache), so the
// fused decode kernel reads exactly 2*d*sizeof(T) bytes per exact token. Angles are
// fp64 (pos * inv_freq with inv_freq computed by numpy on the host, identical bits to
// the reference), sincos in fp64, result rounded once to the cache dtype.
#include <algorithm>
#include <map>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>

#include "mpa_common.cuh"

namespace mpa {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return (int)e;
    }
    return 0;
}

int check_cache(const mpa_cache* c, const char* what) {
    MPA_REQUIRE(c, MPA_ERR_ARG, "%s: null cache", what);
    if (!c->block_table) return 0;
    MPA_REQUIRE(c->page_size >= 1 && (c->page_size & (c->page_size - 1)) == 0, MPA_ERR_ARG,
                "%s: page_size %d is not a power of two", what, c->page_size);
    MPA_REQUIRE(c->n_kv_heads >= 1 && c->n_ledgers % c->n_kv_heads == 0 && c->pages_per_seq >= 1 && c->n_pages >= 1,
                MPA_ERR_ARG, "%s: paged cache geometry", what);
    MPA_REQUIRE((long long)c->pages_per_seq * c->page_size >= c->tcap, MPA_ERR_ARG,
                "%s: %d pages of %d tokens < tcap %d", what, c->pages_per_seq, c->page_size, c->tcap);
    MPA_REQUIRE(kv_pool_rows(c) < (1ll << 31), MPA_ERR_UNSUPPORTED, "%s: page pool of %lld rows", what,
                kv_pool_rows(c));
    return 0;
}

// per-device launch facts: a process may drive several GPUs, so nothing is cached per process
namespace {
constexpr int kMaxDevices = 64;
std::mutex g_dev_mu;
int g_sms[kMaxDevices];
std::map<std::pair<int, const void*>, int> g_smem_set;
int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}
}  // namespace

int device_sms() {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (dev < 0 || dev >= kMaxDevices) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 1;
    }
    if (!g_sms[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        g_sms[dev] = n > 0 ? n : 1;
    }
    return g_sms[dev];
}

int set_max_smem(const void* fn, int bytes) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_dev_mu);
    int& have = g_smem_set[{dev, fn}];
    if (bytes > have) {
        const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        MPA_REQUIRE(e == cudaSuccess, (int)e, "cudaFuncSetAttribute(smem %d): %s", bytes, cudaGetErrorString(e));
        have = bytes;
    }
    return 0;
}

template <typename T>
__global__ void kv_write_kernel(T* __restrict__ k_rot, T* __restrict__ k_raw, T* __restrict__ v,
                                const float* __restrict__ k_src, const float* __restrict__ v_src,
                                const int32_t* __restrict__ pos0, int n_tok, int tcap, int d,
                                const double* __restrict__ inv_freq, KvRows kv) {
    const int l = blockIdx.y;
    const int t = blockIdx.x;                      // token within this write
    const int pos = pos0[l] + t;
    const size_t src = ((size_t)l * n_tok + t) * d;
    const size_t raw = ((size_t)l * tcap + pos) * d;
    const size_t dst = (size_t)kv.row(l, pos) * d;
    for (int i = threadIdx.x; i < d / 2; i += blockDim.x) {
        const double x = (double)k_src[src + 2 * i];
        const double y = (double)k_src[src + 2 * i + 1];
        double sn, cs;
        sincos((double)pos * inv_freq[i], &sn, &cs);
        // no FMA contraction: same rounding sequence as numpy's ev*cos - od*sin
        k_rot[dst + 2 * i] = elem<T>::from_d(__dsub_rn(__dmul_rn(x, cs), __dmul_rn(y, sn)));
        k_rot[dst + 2 * i + 1] = elem<T>::from_d(__dadd_rn(__dmul_rn(x, sn), __dmul_rn(y, cs)));
        k_raw[raw + 2 * i] = elem<T>::from_d(x);
        k_raw[raw + 2 * i + 1] = elem<T>::from_d(y);
        v[dst + 2 * i] = elem<T>::from_d((double)v_src[src + 2 * i]);
        v[dst + 2 * i + 1] = elem<T>::from_d((double)v_src[src + 2 * i + 1]);
    }
}

// Append at the current end of each sequence: token t of ledger l goes to position
// cache_len[l / n_kv_heads] + t; the last block to finish (atomic ticket) advances cache_len (and
// the dense-comparator lengths) by n_tok, so a decode step needs no host round trip or extra launch.
template <typename T>
__global__ void kv_append_kernel(T* __restrict__ k_rot, T* __restrict__ k_raw, T* __restrict__ v,
                                 const float* __restrict__ k_src, const float* __restrict__ v_src, int n_kv_heads,
                                 int n_seq, int32_t* __restrict__ cache_len, int32_t* __restrict__ ntok_dense,
                                 int n_tok, int tcap, int d, const double* __restrict__ inv_freq,
                                 int32_t* __restrict__ ticket, KvRows kv) {
    const int l = blockIdx.y, t = blockIdx.x;
    const int pos = cache_len[l / n_kv_heads] + t;
    const size_t src = ((size_t)l * n_tok + t) * d;
    const size_t raw = ((size_t)l * tcap + pos) * d;
    const size_t dst = (size_t)kv.row(l, pos) * d;
    for (int i = threadIdx.x; i < d / 2; i += blockDim.x) {
        const double x = (double)k_src[src + 2 * i];
        const double y = (double)k_src[src + 2 * i + 1];
        double sn, cs;
        sincos((double)pos * inv_freq[i], &sn, &cs);
        k_rot[dst + 2 * i] = elem<T>::from_d(__dsub_rn(__dmul_rn(x, cs), __dmul_rn(y, sn)));
        k_rot[dst + 2 * i + 1] = elem<T>::from_d(__dadd_rn(__dmul_rn(x, sn), __dmul_rn(y, cs)));
        k_raw[raw + 2 * i] = elem<T>::from_d(x);
        k_raw[raw + 2 * i + 1] = elem<T>::from_d(y);
        v[dst + 2 * i] = elem<T>::from_d((double)v_src[src + 2 * i]);
        v[dst + 2 * i + 1] = elem<T>::from_d((double)v_src[src + 2 * i + 1]);
    }
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int prev = atomicAdd(ticket, 1);
        s_last = prev == (int)(gridDim.x * gridDim.y) - 1;
    }
    __syncthreads();
    if (!s_last) return;
    for (int s = threadIdx.x; s < n_seq; s += blockDim.x) cache_len[s] += n_tok;
    if (ntok_dense)
        for (int j = threadIdx.x; j < n_seq * n_kv_heads; j += blockDim.x) ntok_dense[j] += n_tok;
    if (threadIdx.x == 0) *ticket = 0;
}

__global__ void rotate_queries_kernel(const float* __restrict__ q, int n_qh, int d,
                                      const int32_t* __restrict__ qpos, int delta,
                                      const double* __restrict__ inv_freq, float scale,
                                      float* __restrict__ q_rot, double* __restrict__ q_lk) {
    pdl_wait();     // (PDL kernels trigger only after their own wait: a dependent's early phase may
    pdl_trigger();  // then read anything older than this kernel -- the lookup starts its centroid loads)
    const int s = blockIdx.y, h = blockIdx.x;
    const size_t base = ((size_t)s * n_qh + h) * d;
    const double p = (double)qpos[s];
    for (int i = threadIdx.x; i < d / 2; i += blockDim.x) {
        const double x = (double)q[base + 2 * i], y = (double)q[base + 2 * i + 1];
        double sn, cs;
        if (q_rot) {  // either view may be skipped (the step graph computes them on two branches)
            sincos(p * inv_freq[i], &sn, &cs);
            q_rot[base + 2 * i] = (float)(__dsub_rn(__dmul_rn(x, cs), __dmul_rn(y, sn)) * (double)scale);
            q_rot[base + 2 * i + 1] = (float)(__dadd_rn(__dmul_rn(x, sn), __dmul_rn(y, cs)) * (double)scale);
        }
        if (q_lk) {
            sincos((double)delta * inv_freq[i], &sn, &cs);
            q_lk[base + 2 * i] = __dsub_rn(__dmul_rn(x, cs), __dmul_rn(y, sn));
            q_lk[base + 2 * i + 1] = __dadd_rn(__dmul_rn(x, sn), __dmul_rn(y, cs));
        }
    }
}

__global__ void stage3_kernel(float4* __restrict__ d0, const float4* __restrict__ s0, long long n0,
                              float4* __restrict__ d1, const float4* __restrict__ s1, long long n1,
                              float4* __restrict__ d2, const float4* __restrict__ s2, long long n2) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n0 + n1 + n2; i += stride) {
        if (i < n0) d0[i] = s0[i];
        else if (i < n0 + n1) d1[i - n0] = s1[i - n0];
        else d2[i - n0 - n1] = s2[i - n0 - n1];
    }
}

}  // namespace mpa

using namespace mpa;

extern "C" int mpa_stage3(float* dst0, const float* src0, long long n0, float* dst1, const float* src1, long long n1,
                          float* dst2, const float* src2, long long n2, void* stream) {
    const float* srcs[3] = {src0, src1, src2};
    float* dsts[3] = {dst0, dst1, dst2};
    const long long ns[3] = {n0, n1, n2};
    for (int i = 0; i < 3; ++i) {
        MPA_REQUIRE(ns[i] >= 0 && ns[i] % 4 == 0, MPA_ERR_ARG, "mpa_stage3: size %lld not a multiple of 4", ns[i]);
        MPA_REQUIRE(!ns[i] || (srcs[i] && dsts[i] && ((uintptr_t)srcs[i] & 15) == 0 && ((uintptr_t)dsts[i] & 15) == 0),
                    MPA_ERR_ARG, "mpa_stage3: buffer %d null or not 16-byte aligned", i);
    }
    const long long v = (n0 + n1 + n2) / 4;
    if (!v) return 0;
    const int blocks = (int)std::min<long long>(1184, (v + 255) / 256);
    stage3_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((float4*)dst0, (const float4*)src0, n0 / 4, (float4*)dst1,
                                                            (const float4*)src1, n1 / 4, (float4*)dst2,
                                                            (const float4*)src2, n2 / 4);
    return check_launch("mpa_stage3");
}

extern "C" int mpa_step_host(void* graph_exec, void* d_in, const void* h_q, long long q_bytes, const void* h_k,
                             long long k_bytes, const void* h_v, long long v_bytes, void* h_out, const void* d_out,
                             long long out_bytes, void* stream) {
    MPA_REQUIRE(graph_exec && d_in && h_q && h_k && h_v && h_out && d_out, MPA_ERR_ARG, "mpa_step_host: null argument");
    MPA_REQUIRE(q_bytes >= 0 && k_bytes >= 0 && v_bytes >= 0 && out_bytes >= 0, MPA_ERR_ARG, "mpa_step_host: sizes");
    cudaStream_t st = (cudaStream_t)stream;
    char* d = (char*)d_in;
    cudaError_t e = cudaMemcpyAsync(d, h_q, (size_t)q_bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d + q_bytes, h_k, (size_t)k_bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d + q_bytes + k_bytes, h_v, (size_t)v_bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaGraphLaunch((cudaGraphExec_t)graph_exec, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_out, d_out, (size_t)out_bytes, cudaMemcpyDeviceToHost, st);
    MPA_REQUIRE(e == cudaSuccess, (int)e, "mpa_step_host: %s", cudaGetErrorString(e));
    return 0;
}

extern "C" const char* mpa_last_error(void) { return g_err; }

extern "C" const char* mpa_version(void) { return "libmpattn 0.1 (sm_100a)"; }

extern "C" int mpa_kv_write(const mpa_cache* c, const float* k_src, const float* v_src,
                            const int32_t* pos0, int n_tok, const double* inv_freq, void* stream) {
    MPA_REQUIRE(c && k_src && v_src && pos0 && inv_freq, MPA_ERR_ARG, "mpa_kv_write: null argument");
    MPA_REQUIRE(c->head_dim >= 2 && c->head_dim % 2 == 0, MPA_ERR_ARG, "mpa_kv_write: bad head_dim %d", c->head_dim);
    if (int rc = check_cache(c, "mpa_kv_write")) return rc;
    if (n_tok <= 0 || c->n_ledgers <= 0) return 0;
    dim3 grid(n_tok, c->n_ledgers);
    const int threads = c->head_dim / 2 < 64 ? 32 : 64;
    cudaStream_t st = (cudaStream_t)stream;
    const KvRows kv = kv_rows(c);
    if (c->dtype == MPA_F32)
        kv_write_kernel<float><<<grid, threads, 0, st>>>((float*)c->k_rot, (float*)c->k_raw, (float*)c->v, k_src,
                                                         v_src, pos0, n_tok, c->tcap, c->head_dim, inv_freq, kv);
    else if (c->dtype == MPA_BF16)
        kv_write_kernel<__nv_bfloat16><<<grid, threads, 0, st>>>(
            (__nv_bfloat16*)c->k_rot, (__nv_bfloat16*)c->k_raw, (__nv_bfloat16*)c->v, k_src, v_src, pos0, n_tok,
            c->tcap, c->head_dim, inv_freq, kv);
    else
        MPA_REQUIRE(false, MPA_ERR_ARG, "mpa_kv_write: bad dtype %d", c->dtype);
    return check_launch("mpa_kv_write");
}

extern "C" int mpa_kv_append(const mpa_cache* c, const float* k_src, const float* v_src, int n_kv_heads, int n_tok,
                             int32_t* cache_len, int32_t* ntok_dense, const double* inv_freq, int32_t* ticket,
                             void* stream) {
    MPA_REQUIRE(c && k_src && v_src && cache_len && inv_freq && ticket, MPA_ERR_ARG, "mpa_kv_append: null argument");
    MPA_REQUIRE(c->head_dim >= 2 && c->head_dim % 2 == 0, MPA_ERR_ARG, "mpa_kv_append: bad head_dim %d",
                c->head_dim);
    MPA_REQUIRE(n_kv_heads >= 1 && c->n_ledgers % n_kv_heads == 0, MPA_ERR_ARG, "mpa_kv_append: n_kv_heads %d",
                n_kv_heads);
    if (int rc = check_cache(c, "mpa_kv_append")) return rc;
    if (n_tok <= 0 || c->n_ledgers <= 0) return 0;
    dim3 grid(n_tok, c->n_ledgers);
    const int threads = c->head_dim / 2 < 64 ? 32 : 64;
    const int n_seq = c->n_ledgers / n_kv_heads;
    const KvRows kv = kv_rows(c);
    cudaStream_t st = (cudaStream_t)stream;
    if (c->dtype == MPA_F32)
        kv_append_kernel<float><<<grid, threads, 0, st>>>((float*)c->k_rot, (float*)c->k_raw, (float*)c->v, k_src,
                                                          v_src, n_kv_heads, n_seq, cache_len, ntok_dense, n_tok,
                                                          c->tcap, c->head_dim, inv_freq, ticket, kv);
    else if (c->dtype == MPA_BF16)
        kv_append_kernel<__nv_bfloat16><<<grid, threads, 0, st>>>(
            (__nv_bfloat16*)c->k_rot, (__nv_bfloat16*)c->k_raw, (__nv_bfloat16*)c->v, k_src, v_src, n_kv_heads, n_seq,
            cache_len, ntok_dense, n_tok, c->tcap, c->head_dim, inv_freq, ticket, kv);
    else
        MPA_REQUIRE(false, MPA_ERR_ARG, "mpa_kv_append: bad dtype %d", c->dtype);
    return check_launch("mpa_kv_append");
}

extern "C" int mpa_rotate_queries(const float* q, int n_seq, int n_qh, int d, const int32_t* qpos, int delta,
                                  const double* inv_freq, float scale, float* q_rot, double* q_lk, void* stream) {
    MPA_REQUIRE(q && qpos && inv_freq && (q_rot || q_lk), MPA_ERR_ARG, "mpa_rotate_queries: null argument");
    MPA_REQUIRE(d >= 2 && d % 2 == 0, MPA_ERR_ARG, "mpa_rotate_queries: bad head_dim %d", d);
    if (n_seq <= 0 || n_qh <= 0) return 0;
    launch_pdl(rotate_queries_kernel, dim3(n_qh, n_seq), dim3(64), 0, (cudaStream_t)stream, q, n_qh, d, qpos, delta,
               inv_freq, scale, q_rot, q_lk);
    return check_launch("mpa_rotate_queries");
}
