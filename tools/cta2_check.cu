// cta2_check.cu — semantics + cost of tcgen05.mma.cta_group::2.kind::i8 with A from TMEM on sm_100a.
// A CTA pair (cluster of 2): CTA r holds A rows [128r, 128r+128) (K=32) in its TMEM via tcgen05.st and
// B rows [r*N/2, (r+1)*N/2) (K-major, SWIZZLE_128B) in its SMEM; the leader issues one M=256 MMA;
// each CTA reads its D rows and writes them out. The host checks D = A · B^T exactly, then times a
// loop of dependent MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/cta2_check tools/cta2_check.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2405_04532_b200/csrc/sm100_ptx.cuh"

using namespace qoq;

constexpr int N = 64;
constexpr int K = 32;

__device__ __forceinline__ void mma_i8_ts_2cta(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                               uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit_2cta_mc(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
        ::"r"(smem_u32(bar)), "h"((uint16_t)0x3)
        : "memory");
}

// A[256][32] int8 (u8 format), B[N][32] int8 (s8). D = A B^T int32 [256][N].
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    kern(const uint8_t* A, const int8_t* B, int32_t* D, int iters, unsigned long long* cyc) {
    __shared__ __align__(1024) uint8_t sb[8 * 1024];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t rank = cluster_ctarank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // B half: rows [rank*N/2, ...) K-major 32 B per row, placed as SW128 rows of 128 B (k 0..31 valid)
    for (int i = threadIdx.x; i < 8 * 1024; i += blockDim.x) sb[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < (N / 2) * 32; i += blockDim.x) {
        const int row = i / 32, kb = i % 32;
        // SWIZZLE_128B: 16-B chunk index XOR (row % 8)
        const int chunk = kb / 16, within = kb % 16;
        const int phys = row * 128 + ((chunk ^ (row % 8)) * 16) + within;
        sb[phys] = (uint8_t)B[(rank * (N / 2) + row) * 32 + kb];
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tslot;
    // A rows of this CTA into TMEM columns 0..7 (lane = row, 4 k per column)
    {
        const int row = warp * 32 + lane;   // 0..127
        uint32_t v[8];
        for (int c = 0; c < 8; ++c) {
            uint32_t w = 0;
            for (int b = 0; b < 4; ++b) w |= (uint32_t)A[(rank * 128 + row) * 32 + c * 4 + b] << (8 * b);
            v[c] = w;
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     ::"r"(tmem + ((uint32_t)(warp * 32) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]),
                     "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    unsigned long long t0 = 0, t1 = 0;
    if (rank == 0 && warp == 0) {
        const uint32_t idesc = idesc_i8(256, N, /*a_signed=*/false);
        if (elect_one()) {
            t0 = clock64();
            for (int i = 0; i < iters; ++i)
                mma_i8_ts_2cta(tmem + 256, tmem, smem_desc_sw128(smem_u32(sb)), idesc, i > 0 ? 1u : 0u);
            commit_2cta_mc(&bar);
        }
        __syncwarp();
    }
    mbar_wait(&bar, 0);
    if (rank == 0 && threadIdx.x == 0) { t1 = clock64(); cyc[0] = t1 - t0; }
    tc_fence_after();
    // read D rows of this CTA: lane = row, N columns at 256..
    {
        const int row = warp * 32 + lane;
        for (int c0 = 0; c0 < N; c0 += 16) {
            uint32_t r[16];
            tmem_ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c0, r);
            tmem_wait_ld();
            for (int i = 0; i < 16; ++i) D[(rank * 128 + row) * N + c0 + i] = (int32_t)r[i];
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
    std::vector<uint8_t> A(256 * 32);
    std::vector<int8_t> B(N * 32);
    for (int i = 0; i < 256 * 32; ++i) A[i] = (uint8_t)((i * 37 + 11) % 251);
    for (int i = 0; i < N * 32; ++i) B[i] = (int8_t)(((i * 53 + 7) % 255) - 127);
    uint8_t* dA; int8_t* dB; int32_t* dD; unsigned long long* dc;
    cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dD, 256 * N * 4); cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    for (int iters : {1, 4000}) {
        cudaMemset(dD, 0, 256 * N * 4);
        kern<<<2, 128>>>(dA, dB, dD, iters, dc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<int32_t> D(256 * N);
        unsigned long long c;
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        long bad = 0;
        for (int m = 0; m < 256; ++m)
            for (int n = 0; n < N; ++n) {
                long long s = 0;
                for (int k = 0; k < K; ++k) s += (long long)A[m * 32 + k] * (long long)B[n * 32 + k];
                if ((long long)D[m * N + n] != s * iters) ++bad;
            }
        printf("iters=%d: %ld / %d mismatches; %.1f cycles per cta_group::2 MMA (M=256 N=%d K=32)\n", iters, bad,
               256 * N, (double)c / iters, N);
    }
    return 0;
}
