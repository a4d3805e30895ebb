// quantize.cu — the two quantizers of the QoQ W4A8 hot path (sm_100a).
//
//  * Offline weight quantization + packing (§4.1 progressive group quantization;
//    layout P:434/P:447, frozen in include/qoq_b200.h):
//      level1_scale_kernel : s0[n] = fp16(max_k |W[n,k]| / 119)
//      level2_pack_kernel  : q8 = clamp(⌈W/s0⌋, ±119) -> per-group u8 scale, u4 zero, u4 codes
//                            -> packed 128x128 tile stream
//  * Per-token symmetric INT8 activation quantization, bandwidth-bound:
//      quantize_act_kernel : s_x[m] = fp16(max_k|X[m,k]| / 127), q = clamp(⌈X/s_x⌋, ±127),
//                            t_x[m] = Σ_k q (feeds the biased-u8 GEMM epilogue)
//
// Floating-point decisions use IEEE fp32 division (no fast-math), round-half-away (roundf) and
// __float2half_rn, so the codes are deterministic functions of the fp16 inputs.
#include <cuda_fp16.h>
#include <cstdint>

#include "qoq_internal.h"
#include "qoq_quant.cuh"
#include "sm100_ptx.cuh"

namespace qoq {

// block max of arbitrary-sign values (identity -inf; block_reduce_max above assumes v >= 0)
__device__ __forceinline__ float block_reduce_max_signed(float v, float* red) {
    const float ninf = -__int_as_float(0x7f800000);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    v = (l < nw) ? red[l] : ninf;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;  // valid in every thread
}

// ------------------------------------------------------------------ weights, level 1

__global__ void __launch_bounds__(256) level1_scale_kernel(const __half* __restrict__ W, int K,
                                                           __half* __restrict__ s0) {
    __shared__ float red[32];
    pdl_wait();
    const uint4* row = reinterpret_cast<const uint4*>(W + (size_t)blockIdx.x * K);
    float a = 0.0f;
    for (int i = threadIdx.x; i < K / 8; i += blockDim.x) a = amax8(__ldg(row + i), a);
    a = block_reduce_max(a, red);
    if (threadIdx.x == 0) s0[blockIdx.x] = sym_scale(a, 119.0f);
}

// round half away from zero of a/b for integers, b > 0 (the paper's ⌈·⌋ on integers)
__device__ __forceinline__ int rhai(int a, int b) {
    const int m = a < 0 ? -a : a;
    const int q = (2 * m + b) / (2 * b);
    return a < 0 ? -q : q;
}

__device__ __forceinline__ int q8_of(__half w, float s) {
    const int q = (int)roundf(__fdiv_rn(__half2float(w), s));
    return min(119, max(-119, q));
}

// grid (K/128, N/128), 128 threads: thread r owns output channel n = 128*blockIdx.y + r of
// group j = blockIdx.x and writes its 4 x 16 B of codes in the consumption order of the GEMM.
__global__ void __launch_bounds__(128) level2_pack_kernel(const __half* __restrict__ W, int K,
                                                          const __half* __restrict__ s0,
                                                          uint8_t* __restrict__ packed) {
    pdl_wait();
    const int j = blockIdx.x, nt = blockIdx.y, r = threadIdx.x;
    const int n = nt * 128 + r, KT = K / 128;
    const float s = __half2float(s0[n]);
    const uint4* src = reinterpret_cast<const uint4*>(W + (size_t)n * K + (size_t)j * 128);
    // pass 1: the group's level-1 code range
    int lo = 127, hi = -127;
#pragma unroll 4
    for (int v = 0; v < 16; ++v) {
        uint4 u = __ldg(src + v);
        const __half* h = reinterpret_cast<const __half*>(&u);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int q = q8_of(h[e], s);
            lo = min(lo, q);
            hi = max(hi, q);
        }
    }
    const int su = max(1, rhai(hi - lo, 15));
    const int z = min(15, max(0, rhai(-lo, su)));
    uint8_t* tile = packed + ((size_t)nt * KT + j) * 8448;
    // pass 2: codes, packed as byte b = w_b | w_{b+16} << 4 within each 32-wide chunk
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
        int code[32];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            uint4 u = __ldg(src + c * 4 + v);
            const __half* h = reinterpret_cast<const __half*>(&u);
#pragma unroll
            for (int e = 0; e < 8; ++e) code[v * 8 + e] = min(15, max(0, rhai(q8_of(h[e], s) + z * su, su)));
        }
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            w[i] = 0;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const int b = 4 * i + bb;
                w[i] |= (uint32_t)(code[b] | (code[b + 16] << 4)) << (8 * bb);
            }
        }
        *reinterpret_cast<uint4*>(tile + c * 2048 + r * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    tile[8192 + r] = (uint8_t)su;
    tile[8320 + r] = (uint8_t)(z * su);
}

// ------------------------------------------------------------------ weights, per-channel W4A8 (NEXT-1)
// Per-output-channel asymmetric UINT4 (Eq. 2, q_min = 0, q_max = 15; FP16 scale P:447;
// readings Q20-Q22 in DESIGN.md §3): s_w = fp16(fp32(max - min) / 15), z = clamp(⌈-min / s_w⌋, 0, 15),
// q = clamp(⌈fp32(W / s_w) + z⌋, 0, 15) with t + z summed exactly (double; offline, cost irrelevant).

__global__ void __launch_bounds__(256) pc_scale_kernel(const __half* __restrict__ W, int K,
                                                       __half* __restrict__ s_w, uint8_t* __restrict__ z_w) {
    __shared__ float red[32];
    pdl_wait();
    const __half* row = W + (size_t)blockIdx.x * K;
    float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);   // +-inf
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
        const float v = __half2float(row[i]);
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
    hi = block_reduce_max_signed(hi, red);
    lo = -block_reduce_max_signed(-lo, red);
    if (threadIdx.x == 0) {
        const float range = hi - lo;
        __half sh;
        if (range == 0.0f) {
            sh = __float2half_rn(1.0f);
        } else {
            sh = __float2half_rn(__fdiv_rn(range, 15.0f));
            if (__half_as_ushort(sh) == 0) sh = __ushort_as_half((unsigned short)1);   // 2^-24
        }
        const float s = __half2float(sh);
        const int z = min(15, max(0, (int)round(-(double)__fdiv_rn(lo, s))));
        s_w[blockIdx.x] = sh;
        z_w[blockIdx.x] = (uint8_t)z;
    }
}

// grid (K/128, N/128), 128 threads: thread r owns output channel n = 128*blockIdx.y + r and writes
// the 4 x 16 B of codes of k-tile blockIdx.x (the g128 tile's nibble layout, 8192-byte tiles).
__global__ void __launch_bounds__(128) pc_pack_kernel(const __half* __restrict__ W, int K,
                                                      const __half* __restrict__ s_w,
                                                      const uint8_t* __restrict__ z_w,
                                                      uint8_t* __restrict__ packed) {
    pdl_wait();
    const int j = blockIdx.x, nt = blockIdx.y, r = threadIdx.x;
    const int n = nt * 128 + r, KT = K / 128;
    const float s = __half2float(s_w[n]);
    const double z = (double)z_w[n];
    const uint4* src = reinterpret_cast<const uint4*>(W + (size_t)n * K + (size_t)j * 128);
    uint8_t* tile = packed + ((size_t)nt * KT + j) * 8192;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
        int code[32];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            uint4 u = __ldg(src + c * 4 + v);
            const __half* h = reinterpret_cast<const __half*>(&u);
#pragma unroll
            for (int e = 0; e < 8; ++e)
                code[v * 8 + e] = min(15, max(0, (int)round((double)__fdiv_rn(__half2float(h[e]), s) + z)));
        }
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            w[i] = 0;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const int b = 4 * i + bb;
                w[i] |= (uint32_t)(code[b] | (code[b + 16] << 4)) << (8 * bb);
            }
        }
        *reinterpret_cast<uint4*>(tile + c * 2048 + r * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// ------------------------------------------------------------------ activations

// One CTA per token row: the row (K <= 8 * kQThreads * kQVec) is read ONCE into registers with all
// loads in flight, reduced (amax, half2), quantized from registers (division-free, qoq_quant.cuh) and
// summed; longer rows stream with a second (L1/L2) read. 64 rows at decode leave most SMs free for
// the dependent GEMM, which PDL releases at entry: its CTAs stream their static weights while this
// kernel runs and read q_x only after griddepcontrol.wait. (Measured on the decode step: splitting
// rows over clusters to use more SMs, or capping registers to co-reside with GEMM CTAs, was slower.)
// 512 threads x 4 vectors (K <= 16384 from registers). Measured on the decode step (M = 64, Llama-3-8B,
// profiles/r2b_quantizer_threads.txt): 1.737 ms against 1.814 ms with 256 x 8 — 2.70 / 4.94 us per launch at
// K = 4096 / 14336 instead of 3.02 / 5.57 (384, 640, 768 and 1024 threads were within 1-3% or slower).
#ifndef QOQ_QTHREADS
#define QOQ_QTHREADS 512
#endif
#ifndef QOQ_QVEC
#define QOQ_QVEC 4
#endif
constexpr int kQThreads = QOQ_QTHREADS;   // (build knobs for A/B: threads per row, 16-byte vectors per thread)
constexpr int kQVec = QOQ_QVEC;

__global__ void __launch_bounds__(kQThreads) quantize_act_kernel(const __half* __restrict__ X, int K, int ldx,
                                                                 int8_t* __restrict__ qx, __half* __restrict__ sx,
                                                                 int32_t* __restrict__ tx) {
    __shared__ float redf[32];
    __shared__ int redi[32];
    pdl_launch_dependents();
    pdl_wait();
    const int m = blockIdx.x;
    const uint4* row = reinterpret_cast<const uint4*>(X + (size_t)m * ldx);
    uint2* out = reinterpret_cast<uint2*>(qx + (size_t)m * K);
    const int nv = K / 8;
    int t = 0;
    __half sh;
    if (nv <= kQThreads * kQVec) {
        uint4 r[kQVec];
#pragma unroll
        for (int j = 0; j < kQVec; ++j) {
            const int i = threadIdx.x + j * kQThreads;
            r[j] = (i < nv) ? __ldg(row + i) : make_uint4(0, 0, 0, 0);
        }
        __half2 a2 = __float2half2_rn(0.0f);
#pragma unroll
        for (int j = 0; j < kQVec; ++j) a2 = amax8h(r[j], a2);
        sh = sym_scale(block_reduce_max(amax_of(a2), redf), 127.0f);
        const float s = __half2float(sh), inv = __frcp_rn(s);
#pragma unroll
        for (int j = 0; j < kQVec; ++j) {
            const int i = threadIdx.x + j * kQThreads;
            if (i < nv) out[i] = quant8(r[j], s, inv, t);
        }
    } else {
        __half2 a2 = __float2half2_rn(0.0f);
        for (int i = threadIdx.x; i < nv; i += kQThreads) a2 = amax8h(__ldg(row + i), a2);
        sh = sym_scale(block_reduce_max(amax_of(a2), redf), 127.0f);
        const float s = __half2float(sh), inv = __frcp_rn(s);
        for (int i = threadIdx.x; i < nv; i += kQThreads) out[i] = quant8(__ldg(row + i), s, inv, t);
    }
    if (tx) t = block_reduce_sum(t, redi);
    if (threadIdx.x == 0) {
        sx[m] = sh;
        if (tx) tx[m] = t;
    }
}

// ------------------------------------------------------------------ launchers

cudaError_t launch_quantize_weights(const void* W, int N, int K, void* packed, void* s0, cudaStream_t st) {
    level1_scale_kernel<<<N, 256, 0, st>>>(static_cast<const __half*>(W), K, static_cast<__half*>(s0));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    level2_pack_kernel<<<dim3(K / 128, N / 128), 128, 0, st>>>(static_cast<const __half*>(W), K,
                                                                static_cast<const __half*>(s0),
                                                                static_cast<uint8_t*>(packed));
    return cudaGetLastError();
}

cudaError_t launch_pc_quantize_weights(const void* W, int N, int K, void* packed, void* s_w, uint8_t* z_w,
                                       cudaStream_t st) {
    pc_scale_kernel<<<N, 256, 0, st>>>(static_cast<const __half*>(W), K, static_cast<__half*>(s_w), z_w);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    pc_pack_kernel<<<dim3(K / 128, N / 128), 128, 0, st>>>(static_cast<const __half*>(W), K,
                                                            static_cast<const __half*>(s_w), z_w,
                                                            static_cast<uint8_t*>(packed));
    return cudaGetLastError();
}

cudaError_t launch_quantize_activations(const void* X, int M, int K, int ldx, int8_t* qx, void* sx,
                                        int32_t* tx, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(M);
    cfg.blockDim = dim3(kQThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, quantize_act_kernel, static_cast<const __half*>(X), K, ldx, qx,
                              static_cast<__half*>(sx), tx);
}

}  // namespace qoq
