// Shared helpers for the libmpattn sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdlib>
#include <utility>

#include "mpattn.h"

namespace mpa {

// ---- error plumbing: every C-ABI entry point returns 0 or an error code and
// stores a message readable through mpa_last_error().
void set_error(const char* fmt, ...);
int check_launch(const char* what);

// ---- per-device launch facts (mpa_rope.cu): SM count, and the max-dynamic-smem attribute of a
// kernel raised once per (device, kernel)
int device_sms();
int set_max_smem(const void* fn, int bytes);

#define MPA_REQUIRE(cond, code, ...)        \
    do {                                    \
        if (!(cond)) {                      \
            ::mpa::set_error(__VA_ARGS__);  \
            return (code);                  \
        }                                   \
    } while (0)

// ---- element types ---------------------------------------------------------
template <typename T> struct elem;
template <> struct elem<float> {
    static __device__ __forceinline__ float to_f(float x) { return x; }
    static __device__ __forceinline__ double to_d(float x) { return (double)x; }
    static __device__ __forceinline__ float from_d(double x) { return (float)x; }
};
template <> struct elem<double> {
    static __device__ __forceinline__ float to_f(double x) { return (float)x; }
    static __device__ __forceinline__ double to_d(double x) { return x; }
    static __device__ __forceinline__ double from_d(double x) { return x; }
};
template <> struct elem<__nv_bfloat16> {
    static __device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
    static __device__ __forceinline__ double to_d(__nv_bfloat16 x) { return (double)__bfloat162float(x); }
    static __device__ __forceinline__ __nv_bfloat16 from_d(double x) { return __double2bfloat16(x); }
};

// ---- 16-byte chunk unpacking to fp64 (register-only; no address-taken locals)
template <typename T> struct unpack16;
template <> struct unpack16<__nv_bfloat16> {
    static constexpr int N = 8;
    static __device__ __forceinline__ void run(const uint4& r, double (&o)[8]) {
        const unsigned w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            o[2 * i] = (double)__uint_as_float(w[i] << 16);
            o[2 * i + 1] = (double)__uint_as_float(w[i] & 0xffff0000u);
        }
    }
};
template <> struct unpack16<float> {
    static constexpr int N = 4;
    static __device__ __forceinline__ void run(const uint4& r, double (&o)[4]) {
        o[0] = (double)__uint_as_float(r.x);
        o[1] = (double)__uint_as_float(r.y);
        o[2] = (double)__uint_as_float(r.z);
        o[3] = (double)__uint_as_float(r.w);
    }
};
template <> struct unpack16<double> {
    static constexpr int N = 2;
    static __device__ __forceinline__ void run(const uint4& r, double (&o)[2]) {
        o[0] = __hiloint2double((int)r.y, (int)r.x);
        o[1] = __hiloint2double((int)r.w, (int)r.z);
    }
};

// ---- warp / block reductions -----------------------------------------------
// drop dead scratch from L2 without writing it back (discard.global.L2): every 128-byte line
// lying wholly inside [p, p + bytes) -- lines shared with live neighbours are left alone.
// Block-cooperative over threads [t0, t0 + nt).
__device__ __forceinline__ void discard_l2_range(const void* p, size_t bytes, int t, int nt) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uintptr_t lo = (a + 127) & ~(uintptr_t)127, hi = (a + bytes) & ~(uintptr_t)127;
    for (uintptr_t x = lo + (uintptr_t)t * 128; x < hi; x += (uintptr_t)nt * 128)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(x) : "memory");
}

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T> __device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide reduction of one value per thread; result broadcast to all threads.
// `scratch` needs blockDim.x/32 entries. Callers must __syncthreads() before reusing scratch.
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, T* scratch, Op op) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    T r = scratch[0];
    for (int i = 1; i < nw; ++i) r = op(r, scratch[i]);
    __syncthreads();
    return r;
}

// Exclusive block-wide prefix sum of one int per thread (blockDim.x <= 1024).
// Returns the exclusive prefix; *total receives the block total. scratch: 33 ints.
__device__ __forceinline__ int block_exclusive_scan(int v, int* scratch, int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) scratch[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int s = lane < nw ? scratch[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) scratch[lane] = s;  // inclusive warp totals
        if (lane == 31) scratch[32] = s;
    }
    __syncthreads();
    const int base = wid ? scratch[wid - 1] : 0;
    *total = scratch[32];
    __syncthreads();
    return base + incl - v;
}

__host__ __device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Row of token t of ledger l in k_rot / v: flat [L, tcap] or through the block table of a paged
// pool (mpa_cache).  Rows fit in int32 (tensor maps are limited to 2^31 rows).
struct KvRows {
    const int32_t* bt;
    int tcap, ps_shift, ppl, hkv;
    __device__ __forceinline__ int row(int l, int t) const {
        if (!bt) return l * tcap + t;
        const int s = l / hkv, h = l - s * hkv;
        const int page = __ldg(bt + (size_t)s * ppl + (t >> ps_shift));
        return ((page * hkv + h) << ps_shift) + (t & ((1 << ps_shift) - 1));
    }
};
inline KvRows kv_rows(const mpa_cache* c) {
    KvRows r{c->block_table, c->tcap, 0, c->pages_per_seq, c->n_kv_heads > 0 ? c->n_kv_heads : 1};
    if (c->block_table)
        while ((1 << r.ps_shift) < c->page_size) ++r.ps_shift;
    return r;
}
inline long long kv_pool_rows(const mpa_cache* c) {
    return c->block_table ? (long long)c->n_pages * c->page_size * c->n_kv_heads : (long long)c->n_ledgers * c->tcap;
}
// paged caches: page_size a power of two, the pool addressable with int32 rows
int check_cache(const mpa_cache* c, const char* what);

}  // namespace mpa

// Runtime GQA group size -> compile-time kG (1..8).
// ---- programmatic dependent launch (PDL): a kernel launched with launch_pdl may start while
// its stream predecessor finishes; it must pdl_wait() before touching that predecessor's outputs
// (and every PDL kernel waits at some point, so completion stays transitive along the chain)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define MPA_DISPATCH_G(G, ...)                                                                      \
    switch (G) {                                                                                    \
        case 1: { constexpr int kG = 1; __VA_ARGS__; } break;                                      \
        case 2: { constexpr int kG = 2; __VA_ARGS__; } break;                                      \
        case 3: { constexpr int kG = 3; __VA_ARGS__; } break;                                      \
        case 4: { constexpr int kG = 4; __VA_ARGS__; } break;                                      \
        case 5: { constexpr int kG = 5; __VA_ARGS__; } break;                                      \
        case 6: { constexpr int kG = 6; __VA_ARGS__; } break;                                      \
        case 7: { constexpr int kG = 7; __VA_ARGS__; } break;                                      \
        case 8: { constexpr int kG = 8; __VA_ARGS__; } break;                                      \
        default: ::mpa::set_error("group size %d not supported (1..8)", (int)(G));                \
                 return MPA_ERR_UNSUPPORTED;                                                        \
    }
