// L1TEX cost of contiguous row streams (B200, sm_100a): a warp loads or stores WR = 32/TPR
// consecutive rows of RB bytes per instruction (lane: VB = 32 B), U instructions in flight,
// over an L2-resident 48 MB buffer -- the y-row traffic of the SpMMV epilogue.  Compare
// with random gathers (gather_bw.cu).  Prints B/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/stream_bw tools/micro/stream_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool STORE, int U>
__global__ void stream(char* __restrict__ t, unsigned long long span, int iters, unsigned long long* sink) {
    // each warp owns a 1 KB line-aligned region per instruction; the grid walks the buffer
    const int lane = threadIdx.x & 31;
    const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    unsigned long long acc = 0;
    unsigned long long pos = warp * 1024ull * U;
    for (int it = 0; it < iters; ++it) {
        if (pos + 1024ull * U > span) pos = (pos + 1024ull * U) % (span - 1024ull * U);
        unsigned long long v[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            char* p = t + pos + u * 1024ull + lane * 32;
            if constexpr (STORE) {
                asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(acc), "l"(acc + 1), "l"(acc + 2),
                             "l"(acc + 3)
                             : "memory");
            } else {
                asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                             : "=l"(v[u][0]), "=l"(v[u][1]), "=l"(v[u][2]), "=l"(v[u][3])
                             : "l"(p));
            }
        }
        if constexpr (!STORE) {
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u][0] ^ v[u][3];
        } else {
            acc += 1;
        }
        pos += nwarps * 1024ull * U;
    }
    if (acc == 0x1234567) sink[0] = acc;
}

template <bool STORE, int U>
void run(char* t, unsigned long long span, int sms, int clk) {
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int threads = 256, grid = sms * 8, iters = 4000;
    stream<STORE, U><<<grid, threads>>>(t, span, 10, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    stream<STORE, U><<<grid, threads>>>(t, span, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = double(grid) * threads * 32.0 * iters * U;
    std::printf("{\"op\":\"%s\",\"U\":%d,\"GBs\":%.1f,\"B_per_clk_per_SM\":%.1f,\"err\":\"%s\"}\n",
                STORE ? "STG.256 contiguous" : "LDG.256 contiguous", U, bytes / (ms * 1e-3) / 1e9,
                bytes / (ms * 1e-3) / (double(clk) * 1e3) / sms, cudaGetErrorString(cudaGetLastError()));
    cudaFree(sink);
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    char* t;
    const unsigned long long span = 48ull << 20;
    cudaMalloc(&t, span);
    cudaMemset(t, 1, span);
    run<false, 4>(t, span, sms, clk);
    run<false, 8>(t, span, sms, clk);
    run<true, 4>(t, span, sms, clk);
    run<true, 8>(t, span, sms, clk);
    return 0;
}
