// Standalone check of the tcgen05 building blocks used by the k-means assignment kernel:
// TMA 2D tile loads (128B swizzle) -> UMMA smem descriptors (K-major, SW128) ->
// tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32 in TMEM) -> tcgen05.ld epilogue.
// D[128 x 256] = A[128 x 128] . B[256 x 128]^T, compared with a host fp64 reference.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2506_13059_b200/csrc/mpa_tc.cuh"

using namespace mpa;

constexpr int M = 128, N = 256, K = 128;

__global__ void __launch_bounds__(128) gemm_kernel(const __grid_constant__ CUtensorMap ta,
                                                   const __grid_constant__ CUtensorMap tb, float* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    unsigned char* sa = smem;                 // [2 chunks][128 rows][128 B]
    unsigned char* sb = smem + 2 * M * 128;   // [2 chunks][256 rows][128 B]
    __shared__ __align__(8) uint64_t bar_tma, bar_mma;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc(&tmem_base, 256);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar_tma), 1);
        mbar_init(smem_u32(&bar_mma), 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    if (threadIdx.x == 0) {
        mbar_expect_tx(smem_u32(&bar_tma), 2 * M * 128 + 2 * N * 128);
        for (int c = 0; c < 2; ++c) {
            tma_load_2d(smem_u32(sa + c * M * 128), &ta, c * 64, 0, smem_u32(&bar_tma));
            tma_load_2d(smem_u32(sb + c * N * 128), &tb, c * 64, 0, smem_u32(&bar_tma));
        }
        mbar_wait(smem_u32(&bar_tma), 0);
        tc_fence_after();
        const uint32_t idesc = umma_idesc_bf16_f32(M, N);
        for (int c = 0; c < 2; ++c)
            for (int k = 0; k < 4; ++k) {
                const uint64_t da = umma_desc_sw128(smem_u32(sa + c * M * 128) + k * 32);
                const uint64_t db = umma_desc_sw128(smem_u32(sb + c * N * 128) + k * 32);
                umma_bf16(tmem, da, db, idesc, (c | k) ? 1u : 0u);
            }
        umma_commit(smem_u32(&bar_mma));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar_mma), 0);
    tc_fence_after();
    // each warp reads its 32 TMEM lanes (rows), 32 columns at a time
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) out[row * N + c0 + j] = __uint_as_float(v[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

static int make_map(CUtensorMap* m, void* base, int rows, int box_rows) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return (int)((EncodeFn)fn)(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

int main() {
    std::vector<__nv_bfloat16> ha(M * K), hb(N * K);
    std::vector<float> fa(M * K), fb(N * K);
    srand(1);
    for (int i = 0; i < M * K; ++i) {
        ha[i] = __float2bfloat16((rand() % 2001 - 1000) / 250.0f);
        fa[i] = __bfloat162float(ha[i]);
    }
    for (int i = 0; i < N * K; ++i) {
        hb[i] = __float2bfloat16((rand() % 2001 - 1000) / 250.0f);
        fb[i] = __bfloat162float(hb[i]);
    }
    __nv_bfloat16 *da, *db;
    float* dout;
    cudaMalloc(&da, M * K * 2);
    cudaMalloc(&db, N * K * 2);
    cudaMalloc(&dout, M * N * 4);
    cudaMemcpy(da, ha.data(), M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), N * K * 2, cudaMemcpyHostToDevice);
    CUtensorMap ta, tb;
    if (make_map(&ta, da, M, M) || make_map(&tb, db, N, N)) {
        printf("tensor map failed\n");
        return 1;
    }
    const int smem = 1024 + 2 * M * 128 + 2 * N * 128;
    cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    gemm_kernel<<<1, 128, smem>>>(ta, tb, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("kernel error %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> out(M * N);
    cudaMemcpy(out.data(), dout, M * N * 4, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += (double)fa[i * K + k] * fb[j * K + k];
            worst = fmax(worst, fabs(ref - out[i * N + j]) / (1.0 + fabs(ref)));
        }
    printf("tcgen05 gemm max rel err %.3e  (%s)\n", worst, worst < 1e-5 ? "OK" : "FAIL");
    return worst < 1e-5 ? 0 : 1;
}
