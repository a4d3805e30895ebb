// ingress_bench2.cu — main-loop ingress ceiling of the decode GEMM (M = 64): per step each CTA needs a
// unique 16,896-byte packed-weight step (HBM, TMA bulk, 6-deep ring) and a 16,384-byte activation step
// (two 64-row k-tiles, L2-resident, re-read by every CTA). Variants for the activation delivery:
//   0  TMA bulk by the CTA itself                              (what the GEMM does today)
//   1  TMA bulk multicast, cluster of 2: rank r issues half r   (each CTA's TMA issues 8 KB of activations)
//   2  TMA bulk multicast, cluster of 4
//   3  LSU: 4 warps ld.global.v4 + st.shared (no TMA for activations)
//   4  no activations (weights only)
//   5  TMA 2-D tensor loads (box 128 B x 64 rows, SWIZZLE_128B, two per step) from a row-major [64][4096] q_x,
//      as the GEMM's activation producer does
//   6  as 5, issued by the weight producer thread itself (one TMA issuer)
//   7  as 5, the weight copies with the GEMM's L2::cache_hint evict_first policy
//   8  as 5, plus 4 warps reading every weight step from shared memory (LDS.128, as the dequant warps)
//   9  as 8, plus the same 4 warps reading every activation step (as the MMA's B operand reads)
//  10  weights NOT staged in shared memory: the producer prefetches them into L2 (cp.async.bulk.prefetch.L2,
//      kPf steps ahead) and the 4 warps load them straight into registers (LDG.128, two steps in flight),
//      activations by TMA as in 9 and read from shared memory
//  11  as 10 with 3 steps of weights in flight per thread
// Prints weight bytes per cycle per SM and the aggregate weight TB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ingress_bench2.cu -o tools/ingress_bench2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda.h>
#include <cudaTypedefs.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint64_t* b, uint32_t cta) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(b)), "r"(cta));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_mc(void* dst, const void* src, uint32_t bytes, uint64_t* b, uint16_t mask) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)), "h"(mask) : "memory");
}

constexpr int kW = 16896, kWS = 17408, kWR = 6, kX = 16384, kXR = 5, kIters = 300;

__global__ void __launch_bounds__(224, 1) pipe(const __grid_constant__ CUtensorMap tmx, const uint8_t* w, size_t per,
                                               const uint8_t* act, int variant, int C, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t wfull[kWR], wfree[kWR], xfull[kXR], xfree[kXR];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t cr = C > 1 ? cluster_rank() : 0;
    uint8_t* xs = sm + kWR * kWS;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kWR; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&wfull[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&wfree[i])), "r"((variant == 8 || variant == 9) ? 4 : 1));
        }
        for (int i = 0; i < kXR; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&xfull[i])), "r"(variant == 3 ? 4 : 1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&xfree[i])), "r"(variant >= 9 ? 4 : C));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (C > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    const long long t0 = clock64();
    const bool acts = variant != 4;
    if (warp == 0 && lane == 0 && variant != 10 && variant != 11) {            // weight producer
        const uint8_t* base = w + per * blockIdx.x;
        for (int it = 0; it < kIters; ++it) {
            const int i = it % kWR;
            if (it >= kWR) wait(&wfree[i], ((it / kWR) - 1) & 1);
            expect(&wfull[i], kW);
            if (variant == 7) {
                uint64_t pol;
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                             ::"r"(smem_u32(sm + i * kWS)), "l"(base + (size_t)it * kW), "r"(kW), "r"(smem_u32(&wfull[i])),
                             "l"(pol) : "memory");
            } else {
                bulk(sm + i * kWS, base + (size_t)it * kW, kW, &wfull[i]);
            }
            if (variant == 6) {
                const int j = it % kXR;
                if (it >= kXR) wait(&xfree[j], ((it / kXR) - 1) & 1);
                expect(&xfull[j], kX);
                for (int t = 0; t < 2; ++t)
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                                 ::"r"(smem_u32(xs + j * kX + t * 8192)), "l"(&tmx), "r"(((2 * it + t) % 32) * 128), "r"(0),
                                 "r"(smem_u32(&xfull[j])) : "memory");
            }
        }
    } else if (warp == 1 && lane == 0 && (variant == 5 || variant >= 7)) {   // activation producer: 2-D tensor loads
        for (int it = 0; it < kIters; ++it) {
            const int i = it % kXR;
            if (it >= kXR) wait(&xfree[i], ((it / kXR) - 1) & 1);
            expect(&xfull[i], kX);
            for (int t = 0; t < 2; ++t)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                             ::"r"(smem_u32(xs + i * kX + t * 8192)), "l"(&tmx), "r"(((2 * it + t) % 32) * 128), "r"(0),
                             "r"(smem_u32(&xfull[i])) : "memory");
        }
    } else if (warp == 1 && lane == 0 && acts && variant != 3 && variant >= 0 && variant < 5) {   // activation producer (TMA)
        for (int it = 0; it < kIters; ++it) {
            const int i = it % kXR;
            if (it >= kXR) wait(&xfree[i], ((it / kXR) - 1) & 1);
            const uint8_t* src = act + (size_t)(it % 16) * kX;
            expect(&xfull[i], kX);   // every CTA receives the whole step
            if (variant == 0) {
                bulk(xs + i * kX, src, kX, &xfull[i]);
            } else {
                const uint32_t part = kX / C;
                bulk_mc(xs + i * kX + cr * part, src + cr * part, part, &xfull[i], (uint16_t)((1u << C) - 1));
            }
        }
    } else if (warp >= 3 && warp < 7 && variant == 3) {   // LSU activation loader
        const int t = threadIdx.x - 96;
        for (int it = 0; it < kIters; ++it) {
            const int i = it % kXR;
            if (it >= kXR) wait(&xfree[i], ((it / kXR) - 1) & 1);
            const uint4* src = reinterpret_cast<const uint4*>(act + (size_t)(it % 16) * kX);
            uint4* dst = reinterpret_cast<uint4*>(xs + i * kX);
            uint4 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = __ldcg(src + t + 128 * j);
#pragma unroll
            for (int j = 0; j < 8; ++j) dst[t + 128 * j] = v[j];
            __syncwarp();
            if (lane == 0) arrive(&xfull[i]);
        }
    } else if (warp == 0 && lane == 0 && (variant == 10 || variant == 11)) {   // L2 prefetch of the weights
        const uint8_t* base = w + per * blockIdx.x;
        for (int it = 0; it < kIters; it += 4)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + (size_t)it * kW), "r"(4 * kW) : "memory");
    } else if (warp >= 3 && warp < 7 && (variant == 10 || variant == 11)) {   // weights by LDG, acts from smem
        const int t = threadIdx.x - 96;
        const uint4* wg = reinterpret_cast<const uint4*>(w + per * blockIdx.x);
        uint32_t acc = 0;
        constexpr int kD = 3;
        uint4 buf[kD][8];
        const int D = variant == 10 ? 2 : 3;
        for (int d = 0; d < D; ++d)
#pragma unroll
            for (int k = 0; k < 8; ++k) buf[d][k] = __ldcg(wg + (size_t)d * (kW / 16) + t + 128 * k);
        for (int it = 0; it < kIters; ++it) {
            const int j = it % kXR, b = it % D;
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += buf[b][k].x ^ buf[b][k].w;
            if (it + D < kIters)
#pragma unroll
                for (int k = 0; k < 8; ++k) buf[b][k] = __ldcg(wg + (size_t)(it + D) * (kW / 16) + t + 128 * k);
            wait(&xfull[j], (it / kXR) & 1);
            const uint4* xv = reinterpret_cast<const uint4*>(xs + j * kX);
#pragma unroll
            for (int k = 0; k < 8; ++k) { const uint4 v = xv[t + 128 * k]; acc += v.y ^ v.z; }
            __syncwarp();
            if (lane == 0) arrive(&xfree[j]);
        }
        if (acc == 0x12345678u) cyc[0] = -1;
    } else if (warp >= 3 && warp < 7 && (variant == 8 || variant == 9)) {   // shared-memory readers
        const int t = threadIdx.x - 96;
        uint32_t acc = 0;
        for (int it = 0; it < kIters; ++it) {
            const int i = it % kWR, j = it % kXR;
            wait(&wfull[i], (it / kWR) & 1);
            const uint4* ws = reinterpret_cast<const uint4*>(sm + i * kWS);
#pragma unroll
            for (int k = 0; k < 8; ++k) { const uint4 v = ws[t + 128 * k]; acc += v.x ^ v.w; }
            if (variant == 9) {
                wait(&xfull[j], (it / kXR) & 1);
                const uint4* xv = reinterpret_cast<const uint4*>(xs + j * kX);
#pragma unroll
                for (int k = 0; k < 8; ++k) { const uint4 v = xv[t + 128 * k]; acc += v.y ^ v.z; }
            }
            if (variant == 8 && warp == 3 && lane == 0) {   // activations consumed unread (one arrival)
                wait(&xfull[j], (it / kXR) & 1);
                arrive(&xfree[j]);
            }
            __syncwarp();
            if (lane == 0) arrive(&wfree[i]);
            if (variant == 9 && lane == 0) arrive(&xfree[j]);
        }
        if (acc == 0x12345678u) cyc[0] = -1;   // keep the loads
    } else if (warp == 2 && lane == 0 && variant < 8) {     // consumer
        for (int it = 0; it < kIters; ++it) {
            const int i = it % kWR, j = it % kXR;
            wait(&wfull[i], (it / kWR) & 1);
            if (acts) wait(&xfull[j], (it / kXR) & 1);
            arrive(&wfree[i]);
            if (acts) {
                if (C > 1 && variant != 3) for (int c = 0; c < C; ++c) arrive_remote(&xfree[j], c);
                else for (int c = 0; c < C; ++c) arrive(&xfree[j]);
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (C > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
}

int main() {
    const size_t per = (size_t)8 << 20;
    uint8_t *w, *act;
    long long* cyc;
    cudaMalloc(&w, per * 148);
    cudaMemset(w, 1, per * 148);
    cudaMalloc(&act, 16 * kX);
    cudaMemset(act, 2, 16 * kX);
    cudaMalloc(&cyc, 8 * 148);
    const int smem = kWR * kWS + kXR * kX + 2048;
    cudaFuncSetAttribute(pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(pipe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const char* names[12] = {"TMA own", "TMA mcast2", "TMA mcast4", "LSU acts", "no acts", "TMA 2-D", "2-D 1 issuer", "2-D evict1st", "+LDS W", "+LDS W+X", "W by LDG x2", "W by LDG x3"};
    // q_x [64][4096] int8 row-major, box {128, 64}, SWIZZLE_128B (the GEMM's activation map at M = 64)
    uint8_t* qx;
    cudaMalloc(&qx, 64 * 4096);
    cudaMemset(qx, 3, 64 * 4096);
    CUtensorMap tm;
    {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
        auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        cuuint64_t dims[2] = {4096, 64};
        cuuint64_t strides[1] = {4096};
        cuuint32_t box[2] = {128, 64};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, qx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    for (int G : {32, 64, 128, 148}) {
        for (int variant : {9, 10, 11}) {
            const int C = variant == 1 ? 2 : variant == 2 ? 4 : 1;
            if (G % C) continue;
            long long hc[148];
            cudaError_t e = cudaSuccess;
            for (int rep = 0; rep < 3; ++rep) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(G);
                cfg.blockDim = dim3(224);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = C;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                e = cudaLaunchKernelEx(&cfg, pipe, tm, (const uint8_t*)w, per, (const uint8_t*)act, variant, C, cyc);
                if (e == cudaSuccess) e = cudaDeviceSynchronize();
            }
            if (e != cudaSuccess) {
                printf("G=%3d %-10s: %s\n", G, names[variant], cudaGetErrorString(e));
                cudaGetLastError();
                continue;
            }
            cudaMemcpy(hc, cyc, 8 * G, cudaMemcpyDeviceToHost);
            double s = 0, mx = 0;
            for (int b = 0; b < G; ++b) {
                s += (double)kW * kIters / hc[b];
                mx = hc[b] > mx ? hc[b] : mx;
            }
            printf("G=%3d %-10s: weights %6.1f B/cycle/SM  (%.2f TB/s aggregate at 1.965 GHz; slowest CTA %.0f cycles/step)\n",
                   G, names[variant], s / G, s * 1.965e9 / 1e12, mx / kIters);
            fflush(stdout);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
