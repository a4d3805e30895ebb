// ingress_bench.cu — per-SM read bandwidth into shared memory from HBM with G CTAs (one per SM): TMA bulk
// copies (a 6-deep ring of 16,896-byte copies, as the GEMM's weight producer), cp.async 16-byte copies
// by 4 warps (LDGSTS), or both at once. Prints bytes/cycle per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ingress_bench.cu -o tools/ingress_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kStep = 16896, kRingMax = 12, kIters = 400;

__global__ void __launch_bounds__(160, 1) ingress(const uint8_t* w, size_t per, int use_tma, int use_lsu, int kRing,
                                                  long long* cyc, long long* bytes) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[kRingMax];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint8_t* base = w + per * blockIdx.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kRing; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const long long t0 = clock64();
    long long moved = 0;
    if (warp == 0 && lane == 0 && use_tma) {
        uint32_t ph[kRingMax] = {0};
        size_t off = 0;
        for (int it = 0; it < kIters; ++it) {
            const int i = it % kRing;
            if (it >= kRing) {
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(ok) : "r"(smem_u32(&bar[i])), "r"(ph[i]) : "memory");
                ph[i] ^= 1;
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(kStep));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(sm + i * 17408)), "l"(base + off), "r"(kStep), "r"(smem_u32(&bar[i])) : "memory");
            off += kStep;
            moved += kStep;
        }
        for (int k = 0; k < kRing; ++k) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(smem_u32(&bar[k])), "r"(ph[k]) : "memory");
        }
    }
    if (warp >= 1 && use_lsu) {   // 4 warps of cp.async 16-byte copies into a separate region, 4 groups in flight
        const int t = threadIdx.x - 32;   // 0..127
        uint8_t* dst = sm + 6 * 17408;
        const uint8_t* src = base + per / 2;
        for (int it = 0; it < kIters; ++it) {
            for (int c = 0; c < kStep / (128 * 16); ++c) {   // 8 x 2 KB = 16 KB per iteration
                const int o = (c * 128 + t) * 16;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + (it % 4) * 16384 + o)),
                             "l"(src + (size_t)it * 16384 + o) : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 3;" ::: "memory");
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        if (t == 0) moved += (long long)kIters * 16384;
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (warp == 0 && lane == 0) atomicAdd((unsigned long long*)bytes + blockIdx.x, (unsigned long long)moved);
    if (threadIdx.x == 32) atomicAdd((unsigned long long*)bytes + blockIdx.x, (unsigned long long)moved);
}

int main() {
    const size_t per = (size_t)16 << 20;
    uint8_t* w;
    long long *cyc, *bytes;
    cudaMalloc(&w, per * 148);
    cudaMemset(w, 1, per * 148);
    cudaMalloc(&cyc, 8 * 148);
    cudaMalloc(&bytes, 8 * 148);
    const int smem = kRingMax * 17408 + 8192;
    cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[3] = {"TMA bulk", "cp.async", "both"};
    for (int G : {32, 148}) for (int ring : {2, 4, 6, 9, 12}) {
        for (int mode = 0; mode < 1; ++mode) {
            long long hc[148], hb[148];
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(bytes, 0, 8 * 148);
                ingress<<<G, 160, smem>>>(w, per, mode != 1, mode != 0, ring, cyc, bytes);
                cudaDeviceSynchronize();
            }
            cudaMemcpy(hc, cyc, 8 * G, cudaMemcpyDeviceToHost);
            cudaMemcpy(hb, bytes, 8 * G, cudaMemcpyDeviceToHost);
            double s = 0;
            for (int b = 0; b < G; ++b) s += (double)hb[b] / hc[b];
            printf("ring=%2d G=%3d %-9s: %6.1f B/cycle per SM (%.2f TB/s at 1.965 GHz)\n", ring, G, names[mode], s / G, s * 1.965e9 / 1e12);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
