// mma_bench.cu — microbenchmark of tcgen05.mma.kind::i8 issue/execute rate on sm_100a.
// Variants: A from TMEM ("TS") vs A from SMEM ("SS"); N in {16, 64, 128, 256}; commit cadence.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench tools/mma_bench.cu
// Prints cycles per MMA (one CTA per SM, all SMs busy) and the implied INT8 MAC/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2405_04532_b200/csrc/sm100_ptx.cuh"

using namespace qoq;

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) { return smem_desc_sw128(saddr); }

__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

// MODE 0: MMAs only (+ optional commit/wait cadence)
// MODE 1: per 4 MMAs: 2 commits to two barriers (no waits) — the GEMM's MMA-thread pattern
// MODE 2: MODE 1 + 2 mbarrier waits per iteration on barriers completed by other warps
//         (4 "dequant" warps arrive each iteration after writing 32 TMEM columns with tcgen05.st)
template <int N, bool TS, int COMMIT_EVERY, int MODE = 0>
__global__ void __launch_bounds__(160, 1) bench(int iters, unsigned long long* out) {
    __shared__ unsigned long long stamp[8][8];
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t cbar[2][4];   // [0]: commit targets, [1]: dequant->MMA ready
    uint8_t* sa = smem;                 // A: 128 x 128 B (16 KB)
    uint8_t* sb = smem + 16384;         // B: N x 128 B
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 7);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        for (int i = 0; i < 4; ++i) { mbar_init(&cbar[0][i], 1); mbar_init(&cbar[1][i], 4); }
        fence_mbar_init();
    }
    if (threadIdx.x < 32) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    unsigned long long t0 = 0, t1 = 0;
    if (MODE >= 2 && threadIdx.x >= 32) {
        // 4 dequant-like warps: wait buffer free (cbar[0][a]), tcgen05.st 32 cols, signal ready
        const int w = (threadIdx.x >> 5) - 1, lane = threadIdx.x & 31;
        const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
        uint32_t v[32];
        for (int i = 0; i < 32; ++i) v[i] = 0x01010101u * (i + lane);
        for (int i = 0; i < iters; ++i) {
            const int a = i & 3;
            const uint32_t ph = (i >> 2) & 1;
            const bool rec = (w == 0 && lane == 0 && i >= 1000 && i < 1008);
            if (rec) stamp[i - 1000][3] = clock64();
            if (MODE == 5 || MODE == 6) {
                const uint32_t ba = smem_u32(&cbar[0][a]);
                while (!mbar_try_wait(ba, ph ^ 1)) __nanosleep(MODE == 5 ? 64 : 256);
            } else {
                mbar_wait(&cbar[0][a], ph ^ 1);
            }
            if (rec) stamp[i - 1000][4] = clock64();
            tc_fence_after();
            if (MODE != 4 && MODE != 5 && MODE != 6) tmem_st_32x32b_x32(tmem + lane_off + 128 + a * 32, v);
            if (rec) stamp[i - 1000][5] = clock64();
            tmem_wait_st();
            if (rec) stamp[i - 1000][6] = clock64();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&cbar[1][a]);
        }
    }
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_i8(128, N, true);
        const uint32_t d = tmem + 256;           // accumulator at column 256
        const uint32_t a_t = tmem;               // A (TS) at columns 0..31
        const uint32_t sa_u = smem_u32(sa), sb_u = smem_u32(sb);
        uint32_t ph = 0;
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t a_i = (MODE == 2 || MODE == 4) ? tmem + 128 + (i & 3) * 32 : a_t;
            const bool rec = (i >= 1000 && i < 1008);
            if (rec) stamp[i - 1000][0] = clock64();
            if (MODE >= 2) { mbar_wait(&cbar[1][i & 3], (i >> 2) & 1); tc_fence_after(); }
            if (rec) stamp[i - 1000][1] = clock64();
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (TS) mma_i8_ts(d, a_i + kk * 8, make_desc(sb_u + kk * 32), idesc, (i | kk) ? 1u : 0u);
                else mma_i8_ss(d, make_desc(sa_u + kk * 32), make_desc(sb_u + kk * 32), idesc, (i | kk) ? 1u : 0u);
            }
            if (MODE >= 1) { tc_commit(&cbar[0][i & 3]); tc_commit(&bar); }
            if (rec) stamp[i - 1000][2] = clock64();
            if (COMMIT_EVERY > 0 && (i % COMMIT_EVERY) == COMMIT_EVERY - 1) {
                tc_commit(&bar);
                mbar_wait(&bar, ph);
                ph ^= 1;
            }
        }
        if (MODE == 0) { tc_commit(&bar); mbar_wait(&bar, ph); }
        else { tc_commit(&cbar[0][0]); }
        t1 = clock64();
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        out[0] = t1 - t0;
        for (int i = 0; i < 8; ++i)
            for (int e = 0; e < 7; ++e) out[1 + i * 8 + e] = stamp[i][e] - stamp[0][0];
    }
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool TS, int CE, int MODE = 0>
void run(const char* name, unsigned long long* d_out) {
    const int iters = 2000;
    auto k = bench<N, TS, CE, MODE>;
    int smem = 16384 + N * 128 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 160, smem>>>(iters, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long cyc = 0, st[65];
    cudaMemcpy(st, d_out, 65 * 8, cudaMemcpyDeviceToHost);
    cyc = st[0];
    if (MODE >= 2) {
        printf("   iter: mma_wait0 mma_go mma_issued | deq_wait0 deq_go deq_st_issued deq_st_done\n");
        for (int i = 0; i < 8; ++i) {
            unsigned long long* r = st + 1 + i * 8;
            printf("   %4d: %6lld %6lld %6lld | %6lld %6lld %6lld %6lld\n", 1000 + i, (long long)r[0], (long long)r[1],
                   (long long)r[2], (long long)r[3], (long long)r[4], (long long)r[5], (long long)r[6]);
        }
    }
    double per = (double)cyc / (iters * 4.0);
    printf("%-34s N=%3d: %7.1f cycles/MMA  %7.0f MAC/clk/SM  %s\n", name, N, per, 128.0 * N * 32 / per,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 65 * 8);
    run<16, true, 0>("TS, no intermediate commit", d);
    run<64, true, 0>("TS, no intermediate commit", d);
    run<128, true, 0>("TS, no intermediate commit", d);
    run<256, true, 0>("TS, no intermediate commit", d);
    run<16, false, 0>("SS, no intermediate commit", d);
    run<64, false, 0>("SS, no intermediate commit", d);
    run<128, false, 0>("SS, no intermediate commit", d);
    run<256, false, 0>("SS, no intermediate commit", d);
    run<64, true, 1>("TS, commit+wait every 4 MMAs", d);
    run<256, true, 1>("TS, commit+wait every 4 MMAs", d);
    run<64, false, 1>("SS, commit+wait every 4 MMAs", d);
    run<256, false, 1>("SS, commit+wait every 4 MMAs", d);
    run<64, true, 0, 1>("TS, 2 commits per 4 MMAs", d);
    run<16, true, 0, 2>("TS, commits + dequant-style handoff", d);
    run<64, true, 0, 2>("TS, commits + dequant-style handoff", d);
    run<256, true, 0, 2>("TS, commits + dequant-style handoff", d);
    run<64, true, 0, 3>("TS, handoff, MMA reads a fixed A buffer", d);
    run<64, true, 0, 4>("TS, handoff without tcgen05.st", d);
    run<64, false, 0, 3>("SS, handoff (st to TMEM unused)", d);
    run<64, true, 0, 5>("TS, handoff no st, waiters nanosleep 64", d);
    run<64, true, 0, 6>("TS, handoff no st, waiters nanosleep 256", d);
    return 0;
}
