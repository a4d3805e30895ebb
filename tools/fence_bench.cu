// fence_bench.cu — cost (SM cycles) of the synchronization primitives on the decode chain's critical path,
// with and without a background weight stream (a TMA bulk-copy ring from HBM, as the chain's weight
// producer runs). One CTA per SM; warp 1 lane 0 times each primitive; warp 0 lane 0 streams.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/fence_bench.cu -o /tmp/fence_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) bench(const uint8_t* w, size_t wbytes, int stream_on, int* flag, int* data,
                                                long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[8];
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        stop = 0;
    }
    __syncthreads();
    if (warp == 0 && lane == 0 && stream_on) {
        // 6-stage ring of 16896-byte bulk loads over this SM's slice of the buffer
        const size_t per = (wbytes / gridDim.x) & ~(size_t)1023;
        const uint8_t* base = w + per * blockIdx.x;
        uint32_t ph[6] = {0, 0, 0, 0, 0, 0};
        size_t off = 0;
        for (int i = 0; i < 6; ++i) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(16896));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(sm + i * 17408)), "l"(base + off), "r"(16896), "r"(smem_u32(&bar[i])) : "memory");
            off = (off + 16896) % ((per - 16896) & ~(size_t)15);
        }
        int i = 0;
        while (!stop) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(smem_u32(&bar[i])), "r"(ph[i]) : "memory");
            ph[i] ^= 1;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(16896));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(sm + i * 17408)), "l"(base + off), "r"(16896), "r"(smem_u32(&bar[i])) : "memory");
            off = (off + 16896) % ((per - 16896) & ~(size_t)15);
            i = (i + 1) % 6;
        }
        for (int k = 0; k < 6; ++k) {   // drain
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(smem_u32(&bar[k])), "r"(ph[k]) : "memory");
        }
    }
    if (warp == 1 && lane == 0) {
        for (int spin = 0; spin < 20000; ++spin) __nanosleep(100);   // let the stream reach steady state
        long long t[16];
        int* myd = data + blockIdx.x * 64;
        const int R = 32;
        long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int r = 0; r < R; ++r) {
            t[0] = clock64();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            t[1] = clock64();
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            t[2] = clock64();
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(flag + blockIdx.x) : "memory");
            t[3] = clock64();
            int v;
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag + blockIdx.x) : "memory");
            t[4] = clock64() + (v & 0);
            myd[r & 31] = v;   // a plain store, then a release (store-ack round trip)
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(flag + blockIdx.x) : "memory");
            t[5] = clock64();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            t[6] = clock64();
            int w2;
            asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(w2) : "l"(flag + (blockIdx.x + 1) % gridDim.x) : "memory");
            t[7] = clock64() + (w2 & 0);
            for (int k = 0; k < 7; ++k) acc[k] += t[k + 1] - t[k];
        }
        for (int k = 0; k < 7; ++k) out[blockIdx.x * 8 + k] = acc[k] / R;
        stop = 1;
    }
    __syncthreads();
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t wbytes = (size_t)2 << 30;
    uint8_t* w;
    int *flag, *data;
    long long* out;
    cudaMalloc(&w, wbytes);
    cudaMemset(w, 1, wbytes);
    cudaMalloc(&flag, 4 * sms);
    cudaMalloc(&data, 4 * 64 * sms);
    cudaMalloc(&out, 8 * 8 * sms);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 17408);
    const char* names[7] = {"fence.proxy.async.global", "fence.acq_rel.gpu", "red.release.gpu",
                            "ld.acquire.gpu", "st + red.release.gpu", "fence.proxy.async.shared::cta",
                            "ld.relaxed.gpu (remote line)"};
    for (int on = 0; on < 2; ++on) {
        for (int rep = 0; rep < 2; ++rep) bench<<<sms, 128, 6 * 17408>>>(w, wbytes, on, flag, data, out);
        cudaDeviceSynchronize();
        long long h[8 * 256];
        cudaMemcpy(h, out, 8 * 8 * sms, cudaMemcpyDeviceToHost);
        printf("background weight stream %s (%d SMs):\n", on ? "ON " : "OFF", sms);
        for (int k = 0; k < 7; ++k) {
            long long s = 0, mx = 0;
            for (int b = 0; b < sms; ++b) { s += h[b * 8 + k]; mx = h[b * 8 + k] > mx ? h[b * 8 + k] : mx; }
            printf("  %-32s mean %6lld  max %6lld cycles\n", names[k], s / sms, mx);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
