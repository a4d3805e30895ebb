// sync_bench.cu — cost of the synchronization primitives the W4A8 pipeline uses, on sm_100a.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/sync_bench tools/sync_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2405_04532_b200/csrc/sm100_ptx.cuh"

using namespace qoq;

__device__ __forceinline__ bool test_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}

template <int MODE>
__global__ void bench(int n, unsigned long long* out) {
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) { tmem_alloc(&tslot, 32); tmem_relinquish(); }
    __syncthreads();
    if (threadIdx.x == 0) mbar_arrive(&bar);   // phase 0 completes
    __syncthreads();
    const uint32_t a = smem_u32(&bar);
    unsigned long long t0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < n; ++i) {
        if (MODE == 0) acc += mbar_try_wait(a, 0);                       // try_wait, completed phase
        if (MODE == 1) { acc += mbar_try_wait(a, 0); tc_fence_after(); } // + tcgen05 fence
        if (MODE == 2) acc += test_wait(a, 0);                           // test_wait
        if (MODE == 3) { mbar_wait(&bar, 0); }                           // our wrapper (loop + watchdog)
        if (MODE == 4) { tc_fence_before(); __syncwarp(); }              // fence before + syncwarp
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = acc; }
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tslot, 32);
}

template <int MODE>
void run(const char* name, unsigned long long* d) {
    const int n = 4096;
    bench<MODE><<<148, 32>>>(n, d);
    cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-40s %6.1f cycles/op\n", name, (double)h[0] / n);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    run<0>("mbarrier.try_wait (completed phase)", d);
    run<1>("try_wait + tcgen05.fence::after", d);
    run<2>("mbarrier.test_wait (completed phase)", d);
    run<3>("mbar_wait wrapper (completed phase)", d);
    run<4>("tcgen05.fence::before + __syncwarp", d);
    return 0;
}
