// FP64 throughput probe on B200: DFMA (CUDA cores) vs DMMA m8n8k4 (mma.sync f64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters) {
    double a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 1.0000001, c = 1e-9;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    double s = 0;
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
}
__global__ void dmma_kernel(double* out, int iters) {
    double acc[8][2];
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.0) out[0] = s;
}
int main() {
    double* d; cudaMalloc(&d, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int blocks_per_sm : {4, 8}) {
        const int iters = 4096, threads = 256, grid = sms * blocks_per_sm;
        dfma_kernel<<<grid, threads>>>(d, 16);
        cudaEventRecord(e0); dfma_kernel<<<grid, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 16 * iters * double(grid) * threads;
        printf("DFMA  %d CTA/SM: %.1f TFLOP/s\n", blocks_per_sm, flops / ms / 1e9);
        dmma_kernel<<<grid, threads>>>(d, 16);
        cudaEventRecord(e0); dmma_kernel<<<grid, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 8 * 8 * 4 * 8 * double(iters) * grid * (threads / 32);
        printf("DMMA  %d CTA/SM: %.1f TFLOP/s\n", blocks_per_sm, flops / ms / 1e9);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
