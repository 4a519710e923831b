// Staged-gather microbenchmark (B200, sm_100a): rows of a table are copied into a
// shared-memory ring by one producer warp with per-row cp.async.bulk (TMA unit, not
// the LSU pipe), and 8 consumer warps read them back with LDS.128 (READS reads of
// each staged row).  Measures the fill rate and the read rate in B/clk/SM, to compare
// with LDG gathers (tools/micro/gather_bw.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1507_08101_b200/csrc -o tools/micro/stage_bw tools/micro/stage_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "tma.cuh"

using namespace skb;

constexpr int kRB = 256;       // row bytes
constexpr int kNR = 48;        // rows per stage
constexpr int kStages = 3;
constexpr int kThreads = 288;  // 8 consumer warps + 1 producer

template <int READS>
__global__ void __launch_bounds__(kThreads, 3) staged(const char* __restrict__ t, unsigned rows, int tiles,
                                                       unsigned long long* sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * kNR * kRB);
    std::uint64_t* empty = full + kStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 8);
        }
        mbar_fence_init();
    }
    __syncthreads();
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    if (warp == 8) {
        unsigned s32 = blockIdx.x * 7919u + lane * 104729u + 1u;
        for (int it = 0; it < tiles; ++it) {
            const int s = it % kStages;
            mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
            if (lane == 0) mbar_arrive_expect_tx(&full[s], kNR * kRB);
            __syncwarp();
            for (int q = lane; q < kNR; q += 32) {
                s32 = s32 * 1664525u + 1013904223u;
                const unsigned r = (s32 >> 5) % rows;
                bulk_g2s(smem + s * kNR * kRB + q * kRB, t + (unsigned long long)r * kRB, kRB, &full[s], pol);
            }
        }
    } else {
        unsigned long long acc = 0;
        unsigned s32 = threadIdx.x * 31u + blockIdx.x;
        for (int it = 0; it < tiles; ++it) {
            const int s = it % kStages;
            mbar_wait(&full[s], (it / kStages) & 1);
            if constexpr (READS > 0) {
                // each warp instruction: two staged rows (16 lanes x 16 B each); READS reads of
                // every row spread over the 8 warps
                const unsigned char* st = smem + s * kNR * kRB;
                constexpr int kInstr = kNR * READS / 2 / 8;  // per warp
#pragma unroll 4
                for (int i = 0; i < kInstr; ++i) {
                    s32 = s32 * 1664525u + 1013904223u;
                    const int row = ((s32 >> 8) + (lane >> 4)) % kNR;
                    const int4 v = *reinterpret_cast<const int4*>(st + row * kRB + (lane & 15) * 16);
                    acc += unsigned(v.x ^ v.y ^ v.z ^ v.w);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (acc == 0x12345) sink[0] = acc;
    }
}

template <int READS>
void run(const char* t, unsigned rows, const char* tag, int sms, int clk_khz) {
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int smem = kStages * kNR * kRB + 2 * kStages * 8;
    cudaFuncSetAttribute(staged<READS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, staged<READS>, kThreads, smem);
    const int grid = sms * per_sm, tiles = 4000;
    staged<READS><<<grid, kThreads, smem>>>(t, rows, 20, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    staged<READS><<<grid, kThreads, smem>>>(t, rows, tiles, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double fill = double(grid) * tiles * kNR * kRB;
    const double reads = fill * READS;
    const double cyc = (ms * 1e-3) * double(clk_khz) * 1e3;
    std::printf("{\"table\":\"%s\",\"ctas_per_sm\":%d,\"reads_per_row\":%d,\"fill_GBs\":%.1f,\"fill_B_per_clk_SM\":%.1f,"
                "\"read_B_per_clk_SM\":%.1f,\"err\":\"%s\"}\n",
                tag, per_sm, READS, fill / (ms * 1e-3) / 1e9, fill / cyc / sms, reads / cyc / sms,
                cudaGetErrorString(cudaGetLastError()));
    cudaFree(sink);
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
    for (int tab = 0; tab < 2; ++tab) {
        const unsigned rows = unsigned((tab ? big : small) / kRB);
        const char* tag = tab ? "HBM 4GB" : "L2 48MB";
        run<0>(t, rows, tag, sms, clk);
        run<2>(t, rows, tag, sms, clk);
        run<3>(t, rows, tag, sms, clk);
        run<6>(t, rows, tag, sms, clk);
    }
    cudaFree(t);
    return 0;
}
