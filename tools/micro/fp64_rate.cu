// Microbenchmark: sustained DFMA and F2F.F64.F32 throughput per SM on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int k = 0; k < iters; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.0) out[0] = s;
}
__global__ void f2f_kernel(double* out, int iters) {
    float f[8];
    double s[8];
    for (int i = 0; i < 8; ++i) { f[i] = threadIdx.x + i; s[i] = 0; }
    for (int k = 0; k < iters; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) { s[i] = s[i] + (double)f[i]; f[i] += 1.0f; }
    double t = 0;
    for (int i = 0; i < 8; ++i) t += s[i];
    if (t == 12345.0) out[0] = t;
}
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int k = 0; k < iters; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.0f) out[0] = s;
}
int main() {
    double* d;
    cudaMalloc(&d, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, blocks = sms * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double n = (double)blocks * threads * iters * 8;
        printf("DFMA: %.2f TFMA/s = %.1f TFLOPS, %.1f FMA/clk/SM at %d MHz max\n", n / ms / 1e9, 2 * n / ms / 1e9,
               n / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        cudaEventRecord(e0);
        f2f_kernel<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("F2F.F64+DADD: %.2f T/s\n", n / ms / 1e9);
        cudaEventRecord(e0);
        ffma_kernel<<<blocks, threads>>>((float*)d, iters, 1.0000001f, 1e-9f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA: %.2f TFMA/s\n", n / ms / 1e9);
    }
    return 0;
}
