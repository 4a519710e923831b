// Gather-throughput microbenchmark (B200, sm_100a): how many bytes per SM-cycle can
// the L1TEX data pipe deliver for RHS-row gathers of the SpMMV shapes, per lane
// mapping?  A warp gathers WR = 32/TPR rows of RB bytes per instruction, each lane
// VB bytes (TPR * VB = RB); U independent gathers per batch.  Table resident in L2
// (48 MB) or in HBM (4 GB).  Prints GB/s and B/clk/SM (clock from the driver).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/gather_bw tools/micro/gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int VB>
__device__ __forceinline__ unsigned long long ldv(const char* p) {
    if constexpr (VB == 32) {
        unsigned long long a, b, c, d;
        asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        return a ^ b ^ c ^ d;
    } else if constexpr (VB == 16) {
        unsigned long long a, b;
        asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
        return a ^ b;
    } else {
        unsigned long long a;
        asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(a) : "l"(p));
        return a;
    }
}

template <int RB, int VB, int U>
__global__ void gather(const char* __restrict__ t, unsigned rows, int iters, unsigned long long* sink) {
    constexpr int TPR = RB / VB;
    const int lane = threadIdx.x & 31;
    const int sub = lane % TPR, rl = lane / TPR;
    unsigned s = (blockIdx.x * blockDim.x + threadIdx.x) / TPR * 2654435761u + 12345u;
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned long long v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            s = s * 1664525u + 1013904223u;
            const unsigned r = (s >> 5) % rows;
            v[u] = ldv<VB>(t + (unsigned long long)r * RB + sub * VB);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 0x1234567) sink[0] = acc + rl;
}

template <int RB, int VB, int U>
void run(const char* t, unsigned rows, const char* tag, int sms, int clk_khz) {
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int threads = 256, per_sm = 8, iters = 2000;
    const int grid = sms * per_sm;
    gather<RB, VB, U><<<grid, threads>>>(t, rows, 10, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    gather<RB, VB, U><<<grid, threads>>>(t, rows, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = double(grid) * threads * VB * double(iters) * U;
    const double gbs = bytes / (ms * 1e-3) / 1e9;
    const double bpc = bytes / (ms * 1e-3) / (double(clk_khz) * 1e3) / sms;
    std::printf("{\"table\":\"%s\",\"row_bytes\":%d,\"lane_bytes\":%d,\"lanes_per_row\":%d,\"U\":%d,\"GBs\":%.1f,"
                "\"B_per_clk_per_SM\":%.1f}\n", tag, RB, VB, RB / VB, U, gbs, bpc);
    cudaFree(sink);
}

template <int RB>
void sweep(const char* t, unsigned rows, const char* tag, int sms, int clk) {
    run<RB, 32, 4>(t, rows, tag, sms, clk);
    run<RB, 16, 4>(t, rows, tag, sms, clk);
    run<RB, 8, 4>(t, rows, tag, sms, clk);
    run<RB, 32, 8>(t, rows, tag, sms, clk);
    run<RB, 16, 8>(t, rows, tag, sms, clk);
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    char* t;
    const size_t big = size_t(4) << 30, small = size_t(48) << 20;
    cudaMalloc(&t, big);
    cudaMemset(t, 1, big);
    cudaDeviceSynchronize();
    sweep<256>(t, unsigned((64u << 10) / 256), "L1 64KB", sms, clk);
    sweep<128>(t, unsigned((64u << 10) / 128), "L1 64KB", sms, clk);
    sweep<64>(t, unsigned((64u << 10) / 64), "L1 64KB", sms, clk);
    sweep<256>(t, unsigned(small / 256), "L2 48MB", sms, clk);
    sweep<128>(t, unsigned(small / 128), "L2 48MB", sms, clk);
    sweep<64>(t, unsigned(small / 64), "L2 48MB", sms, clk);
    sweep<256>(t, unsigned(big / 256), "HBM 4GB", sms, clk);
    sweep<64>(t, unsigned(big / 64), "HBM 4GB", sms, clk);
    cudaFree(t);
    return 0;
}
