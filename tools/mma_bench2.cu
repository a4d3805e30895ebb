// mma_bench2.cu — handoff-amortization experiments for the W4A8 mainloop on sm_100a.
// A "tile" = 4 x tcgen05.mma.kind::i8 (M=128, N, K=32) = one 128x128 expanded weight tile.
// Each experiment: D dequant-like warps (per issuer: 4 warps, one per TMEM lane quarter) wait for a
// buffer to be free (MMA commit), tcgen05.st 32*TPH columns, arrive; the issuer waits, issues 4*TPH
// MMAs, commits. Variants: tiles per handoff (TPH = 1, 2, 4) and number of issuing warps (1 or 2,
// each with its own accumulator and buffers).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_bench2 tools/mma_bench2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2405_04532_b200/csrc/sm100_ptx.cuh"

using namespace qoq;

template <int N, int TPH, int ISSUERS, int NBUF>
__global__ void __launch_bounds__(32 * ISSUERS * 5, 1) bench(int tiles, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t freeb[ISSUERS][NBUF], readyb[ISSUERS][NBUF];
    uint8_t* sb = smem;   // B: N x 128 B
    for (int i = threadIdx.x; i < N * 32; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 7);
    if (threadIdx.x == 0) {
        for (int j = 0; j < ISSUERS; ++j)
            for (int i = 0; i < NBUF; ++i) { mbar_init(&freeb[j][i], 1); mbar_init(&readyb[j][i], 4); }
        fence_mbar_init();
    }
    if (threadIdx.x < 32) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int iters = tiles / TPH / ISSUERS;
    constexpr int kBufCols = 32 * TPH;
    // TMEM map: issuer j: buffers at j*NBUF*kBufCols ..., accumulators at 512 - (j+1)*N
    unsigned long long t0 = 0, t1 = 0;
    if (warp < ISSUERS) {
        const int j = warp;
        if (lane == 0) {
            const uint32_t idesc = idesc_i8(128, N, true);
            const uint32_t d = tmem + 512 - (j + 1) * N;
            const uint32_t sbu = smem_u32(sb);
            t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const int b = i % NBUF;
                mbar_wait(&readyb[j][b], (i / NBUF) & 1);
                tc_fence_after();
                const uint32_t a = tmem + (j * NBUF + b) * kBufCols;
#pragma unroll
                for (int kk = 0; kk < 4 * TPH; ++kk)
                    mma_i8_ts(d, a + kk * 8, smem_desc_sw128(sbu + (kk & 3) * 32), idesc, (i | kk) ? 1u : 0u);
                tc_commit(&freeb[j][b]);
            }
            // drain
            const int last = (iters - 1) % NBUF;
            mbar_wait(&freeb[j][last], ((iters - 1) / NBUF) & 1);
            t1 = clock64();
            if (blockIdx.x == 0 && j == 0) out[0] = t1 - t0;
        }
    } else {
        const int dw = warp - ISSUERS;            // 0 .. 4*ISSUERS-1
        const int j = dw >> 2;
        const int qd = warp & 3;                  // TMEM lane quarter (warp id mod 4)
        const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
        uint32_t v[32];
        for (int i = 0; i < 32; ++i) v[i] = 0x01010101u * (i + lane);
        for (int i = 0; i < iters; ++i) {
            const int b = i % NBUF;
            mbar_wait(&freeb[j][b], ((i / NBUF) & 1) ^ 1);
            tc_fence_after();
#pragma unroll
            for (int t = 0; t < TPH; ++t) tmem_st_32x32b_x32(tmem + lane_off + (j * NBUF + b) * kBufCols + 32 * t, v);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&readyb[j][b]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, int TPH, int ISSUERS, int NBUF>
void run(unsigned long long* d_out) {
    const int tiles = 4096;
    auto k = bench<N, TPH, ISSUERS, NBUF>;
    int smem = N * 128 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 32 * ISSUERS * 5, smem>>>(tiles, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
    // issuer 0 handled tiles/ISSUERS tiles in cyc cycles; the SM handled `tiles` tiles in ~cyc
    double per_tile = (double)cyc / tiles;
    printf("N=%3d tiles/handoff=%d issuers=%d buffers=%d: %7.1f cycles per 128x128 tile (SM)  %s\n", N, TPH,
           ISSUERS, NBUF, per_tile, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    run<64, 1, 1, 4>(d);
    run<64, 1, 1, 8>(d);
    run<64, 2, 1, 4>(d);
    run<64, 4, 1, 2>(d);
    run<64, 1, 2, 4>(d);
    run<64, 2, 2, 2>(d);
    run<64, 2, 2, 3>(d);
    run<16, 2, 1, 4>(d);
    run<16, 2, 2, 3>(d);
    run<128, 2, 1, 4>(d);
    run<128, 1, 2, 4>(d);
    return 0;
}
