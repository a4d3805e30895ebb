// fused_quant.cu — per-token INT8 activation quantization fused into the layer that produces the
// activation (NEXT-2; "we fuse activation quantization into the preceding layernorm for the
// QKV projection and the first FFN layer, or into the preceding activation kernel for the second FFN
// layer"; Fig. 7). Readings Q23-Q26:
//   rmsnorm_quant_kernel  : y = fp16((x · r) · γ), r = 1 / sqrt(S/K + eps), S = Σ x² EXACT (128-bit
//                           integer in units of 2^-48), rounded once to fp64 — so r does not depend on
//                           the reduction order; then the per-token quantizer of quantize.cu on y.
//   silu_mul_quant_kernel : h = fp16((g / (1 + exp(-g))) · u) in fp64; then the quantizer on h.
// Both write q_x / s_x / t_x exactly as qoq_quantize_activations_per_token would on the fp16 layer
// output (the composition is the definition, Q23), without that output ever touching HBM.
//
// One 256-thread CTA per token row (the quantizer's shape: memory-bound, the row is read once into
// registers when K <= 16384, else streamed from L2 per pass); PDL-released like the quantizer so the
// dependent GEMM's CTAs stream their weights while the row kernel runs.
#include <cuda_fp16.h>
#include <cstdint>

#include "qoq_internal.h"
#include "qoq_quant.cuh"
#include "sm100_ptx.cuh"

namespace qoq {

constexpr int kFThreads = 256;
constexpr int kFVec = 8;   // uint4 (8 fp16) per thread held in registers: K <= 16384 read once

struct U128 {
    unsigned long long lo, hi;
};

__device__ __forceinline__ void add128(U128& a, unsigned long long lo, unsigned long long hi) {
    a.lo += lo;
    a.hi += hi + (a.lo < lo ? 1ull : 0ull);
}

// a += x² · 2^48 for the fp16 bit pattern h: x = m · 2^(max(e,1) - 25) with m the integer
// significand, so x² · 2^48 = m² << (2 max(e,1) - 2), a shift in [0, 58] of m² < 2^22 (exact).
__device__ __forceinline__ void sq_acc(U128& a, unsigned h) {
    const unsigned e = (h >> 10) & 31u, man = h & 0x3ffu;
    const unsigned long long m = e ? (man | 0x400u) : man;
    const unsigned long long sq = m * m;
    const int sh = 2 * (e ? (int)e : 1) - 2;
    add128(a, sq << sh, sh > 42 ? (sq >> (64 - sh)) : 0ull);
}

__device__ __forceinline__ void sq_acc8(U128& a, uint4 v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        sq_acc(a, w[i] & 0xffffu);
        sq_acc(a, w[i] >> 16);
    }
}

__device__ __forceinline__ U128 block_reduce_u128(U128 v, U128* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long lo = __shfl_xor_sync(0xffffffffu, v.lo, o);
        const unsigned long long hi = __shfl_xor_sync(0xffffffffu, v.hi, o);
        add128(v, lo, hi);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    v = (l < nw) ? red[l] : U128{0ull, 0ull};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long lo = __shfl_xor_sync(0xffffffffu, v.lo, o);
        const unsigned long long hi = __shfl_xor_sync(0xffffffffu, v.hi, o);
        add128(v, lo, hi);
    }
    return v;   // valid in every thread
}

// Correctly rounded (RNE) conversion of a 128-bit unsigned integer to fp64: the top 64 bits with the
// bits below OR-ed into bit 0 as a sticky bit (bit 0 lies below the round bit of a 53-bit result),
// one __ull2double_rn, then an exact power-of-two scaling.
__device__ __forceinline__ double u128_to_double_rn(U128 a) {
    if (a.hi == 0) return __ull2double_rn(a.lo);
    const int lz = __clzll((long long)a.hi);
    const unsigned long long top = lz ? ((a.hi << lz) | (a.lo >> (64 - lz))) : a.hi;
    const unsigned long long rest = lz ? (a.lo << lz) : a.lo;
    return ldexp(__ull2double_rn(top | (rest != 0ull ? 1ull : 0ull)), 64 - lz);
}

// Q25: r = 1 / sqrt(S/K + eps) in IEEE fp64 (S = Σ x² · 2^48 exactly); 0 for S/K + eps == 0.
__device__ __forceinline__ double rms_rinv(U128 S, int K, double eps) {
    const double ms = ldexp(u128_to_double_rn(S), -48) / (double)K + eps;
    return ms == 0.0 ? 0.0 : 1.0 / sqrt(ms);
}

// 8 fp16 y = fp16_rn((x · r) · γ) (Q24: fp64 products left to right, one rounding)
__device__ __forceinline__ uint4 rms_apply8(uint4 xv, uint4 gv, double r) {
    const __half* x = reinterpret_cast<const __half*>(&xv);
    const __half* g = reinterpret_cast<const __half*>(&gv);
    uint4 out;
    __half* y = reinterpret_cast<__half*>(&out);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const double p = __dmul_rn((double)__half2float(x[e]), r);
        y[e] = __double2half(__dmul_rn(p, (double)__half2float(g[e])));
    }
    return out;
}

// 8 fp16 h = fp16_rn(silu(g) · u), silu(g) = g / (1 + exp(-g)) in fp64 (Q24, Q26)
__device__ __forceinline__ uint4 silu_mul8(uint4 gv, uint4 uv) {
    const __half* g = reinterpret_cast<const __half*>(&gv);
    const __half* u = reinterpret_cast<const __half*>(&uv);
    uint4 out;
    __half* h = reinterpret_cast<__half*>(&out);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const double gd = (double)__half2float(g[e]);
        const double s = __ddiv_rn(gd, __dadd_rn(1.0, exp(-gd)));
        h[e] = __double2half(__dmul_rn(s, (double)__half2float(u[e])));
    }
    return out;
}

// Quantize a row held as y[kFVec] (element i = threadIdx.x + j * kFThreads; out-of-row entries are 0)
__device__ __forceinline__ void quantize_regs(const uint4 (&y)[kFVec], int nv, int8_t* qrow, __half* sx,
                                              int32_t* tx, int m, float* redf, int* redi) {
    __half2 a2 = __float2half2_rn(0.0f);
#pragma unroll
    for (int j = 0; j < kFVec; ++j) a2 = amax8h(y[j], a2);
    const __half sh = sym_scale(block_reduce_max(amax_of(a2), redf), 127.0f);
    const float s = __half2float(sh), inv = __frcp_rn(s);
    uint2* out = reinterpret_cast<uint2*>(qrow);
    int t = 0;
#pragma unroll
    for (int j = 0; j < kFVec; ++j) {
        const int i = threadIdx.x + j * kFThreads;
        if (i < nv) out[i] = quant8(y[j], s, inv, t);
    }
    if (tx) t = block_reduce_sum(t, redi);
    if (threadIdx.x == 0) {
        sx[m] = sh;
        if (tx) tx[m] = t;
    }
}

__global__ void __launch_bounds__(kFThreads) rmsnorm_quant_kernel(const __half* __restrict__ X, int ldx,
                                                                  const __half* __restrict__ gamma, double eps,
                                                                  int K, int8_t* __restrict__ qx,
                                                                  __half* __restrict__ sx,
                                                                  int32_t* __restrict__ tx) {
    __shared__ U128 red128[32];
    __shared__ float redf[32];
    __shared__ int redi[32];
    pdl_launch_dependents();
    pdl_wait();
    const int m = blockIdx.x;
    const uint4* row = reinterpret_cast<const uint4*>(X + (size_t)m * ldx);
    const uint4* g4 = reinterpret_cast<const uint4*>(gamma);
    const int nv = K / 8;
    U128 S{0ull, 0ull};
    if (nv <= kFThreads * kFVec) {
        uint4 y[kFVec];
#pragma unroll
        for (int j = 0; j < kFVec; ++j) {
            const int i = threadIdx.x + j * kFThreads;
            y[j] = (i < nv) ? __ldg(row + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < kFVec; ++j) sq_acc8(S, y[j]);
        const double r = rms_rinv(block_reduce_u128(S, red128), K, eps);
#pragma unroll
        for (int j = 0; j < kFVec; ++j) {
            const int i = threadIdx.x + j * kFThreads;
            if (i < nv) y[j] = rms_apply8(y[j], __ldg(g4 + i), r);
        }
        quantize_regs(y, nv, qx + (size_t)m * K, sx, tx, m, redf, redi);
        return;
    }
    // long rows: three passes (Σx², amax of y, quantize y), y recomputed bit-identically each pass
    for (int i = threadIdx.x; i < nv; i += kFThreads) sq_acc8(S, __ldg(row + i));
    const double r = rms_rinv(block_reduce_u128(S, red128), K, eps);
    __half2 a2 = __float2half2_rn(0.0f);
    for (int i = threadIdx.x; i < nv; i += kFThreads) a2 = amax8h(rms_apply8(__ldg(row + i), __ldg(g4 + i), r), a2);
    const __half sh = sym_scale(block_reduce_max(amax_of(a2), redf), 127.0f);
    const float s = __half2float(sh), inv = __frcp_rn(s);
    uint2* out = reinterpret_cast<uint2*>(qx + (size_t)m * K);
    int t = 0;
    for (int i = threadIdx.x; i < nv; i += kFThreads)
        out[i] = quant8(rms_apply8(__ldg(row + i), __ldg(g4 + i), r), s, inv, t);
    if (tx) t = block_reduce_sum(t, redi);
    if (threadIdx.x == 0) {
        sx[m] = sh;
        if (tx) tx[m] = t;
    }
}

__global__ void __launch_bounds__(kFThreads) silu_mul_quant_kernel(const __half* __restrict__ G,
                                                                   const __half* __restrict__ U, int ldg, int K,
                                                                   int8_t* __restrict__ qx,
                                                                   __half* __restrict__ sx,
                                                                   int32_t* __restrict__ tx) {
    __shared__ float redf[32];
    __shared__ int redi[32];
    pdl_launch_dependents();
    pdl_wait();
    const int m = blockIdx.x;
    const uint4* g4 = reinterpret_cast<const uint4*>(G + (size_t)m * ldg);
    const uint4* u4 = reinterpret_cast<const uint4*>(U + (size_t)m * ldg);
    const int nv = K / 8;
    if (nv <= kFThreads * kFVec) {
        uint4 y[kFVec], u[kFVec];
#pragma unroll
        for (int j = 0; j < kFVec; ++j) {
            const int i = threadIdx.x + j * kFThreads;
            const bool in = i < nv;
            y[j] = in ? __ldg(g4 + i) : make_uint4(0, 0, 0, 0);
            u[j] = in ? __ldg(u4 + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < kFVec; ++j)
            if (threadIdx.x + j * kFThreads < nv) y[j] = silu_mul8(y[j], u[j]);
        quantize_regs(y, nv, qx + (size_t)m * K, sx, tx, m, redf, redi);
        return;
    }
    __half2 a2 = __float2half2_rn(0.0f);
    for (int i = threadIdx.x; i < nv; i += kFThreads) a2 = amax8h(silu_mul8(__ldg(g4 + i), __ldg(u4 + i)), a2);
    const __half sh = sym_scale(block_reduce_max(amax_of(a2), redf), 127.0f);
    const float s = __half2float(sh), inv = __frcp_rn(s);
    uint2* out = reinterpret_cast<uint2*>(qx + (size_t)m * K);
    int t = 0;
    for (int i = threadIdx.x; i < nv; i += kFThreads) out[i] = quant8(silu_mul8(__ldg(g4 + i), __ldg(u4 + i)), s, inv, t);
    if (tx) t = block_reduce_sum(t, redi);
    if (threadIdx.x == 0) {
        sx[m] = sh;
        if (tx) tx[m] = t;
    }
}

namespace {
cudaLaunchConfig_t row_cfg(int M, cudaStream_t st, cudaLaunchAttribute* attr, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(M);
    cfg.blockDim = dim3(kFThreads);
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cfg;
}
}  // namespace

cudaError_t launch_rmsnorm_quantize(const void* X, int ldx, const void* gamma, double eps, int M, int K,
                                    int8_t* qx, void* sx, int32_t* tx, cudaStream_t st, bool pdl) {
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = row_cfg(M, st, attr, pdl);
    return cudaLaunchKernelEx(&cfg, rmsnorm_quant_kernel, static_cast<const __half*>(X), ldx,
                              static_cast<const __half*>(gamma), eps, K, qx, static_cast<__half*>(sx), tx);
}

cudaError_t launch_silu_mul_quantize(const void* G, const void* U, int ldg, int M, int K, int8_t* qx, void* sx,
                                     int32_t* tx, cudaStream_t st, bool pdl) {
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = row_cfg(M, st, attr, pdl);
    return cudaLaunchKernelEx(&cfg, silu_mul_quant_kernel, static_cast<const __half*>(G),
                              static_cast<const __half*>(U), ldg, K, qx, static_cast<__half*>(sx), tx);
}

}  // namespace qoq
