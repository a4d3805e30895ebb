// qoq_quant.cuh — device helpers of the per-token symmetric INT8 activation quantization
// (P:813), shared by the standalone quantizer (quantize.cu) and the fused prologue of the
// W4A8 GEMM (w4a8_gemm.cu), so both produce bit-identical q_x / s_x / t_x.
// Floating-point decisions: IEEE fp32 division (__fdiv_rn, no fast-math), round-half-away (roundf),
// __float2half_rn (DESIGN.md §3 readings).
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

namespace qoq {

// Block-wide max of non-negative values / int sum over a 1-D CTA (valid in every thread).
// Block reductions with one REDUX per warp (redux.sync) and ONE barrier. Contract: each `red` array (>= 32
// slots) is used by at most one reduction per CTA (no barrier protects its reuse). block_reduce_max takes
// non-negative floats, whose bit patterns order like unsigned integers.
__device__ __forceinline__ float block_reduce_max(float v, float* red) {
    const unsigned u = __reduce_max_sync(0xffffffffu, __float_as_uint(v));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (l == 0) red[w] = __uint_as_float(u);
    __syncthreads();
    const unsigned x = (l < nw) ? __float_as_uint(red[l]) : 0u;
    return __uint_as_float(__reduce_max_sync(0xffffffffu, x));  // valid in every thread
}

__device__ __forceinline__ int block_reduce_sum(int v, int* red) {
    v = __reduce_add_sync(0xffffffffu, v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (l == 0) red[w] = v;
    __syncthreads();
    return __reduce_add_sync(0xffffffffu, (l < nw) ? red[l] : 0);
}

// Symmetric fp16 scale: fp16_rn(amax / qmax); 1.0 for amax == 0; 2^-24 if it underflows to 0.
__device__ __forceinline__ __half sym_scale(float amax, float qmax) {
    if (amax == 0.0f) return __float2half_rn(1.0f);
    __half s = __float2half_rn(__fdiv_rn(amax, qmax));
    if ((__half_as_ushort(s) & 0x7fff) == 0) s = __ushort_as_half(1);
    return s;
}

__device__ __forceinline__ float amax8(uint4 v, float a) {
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 f = __half22float2(h[i]);
        a = fmaxf(a, fmaxf(fabsf(f.x), fabsf(f.y)));
    }
    return a;
}

// max |x| over 8 fp16 in half2 arithmetic (exact: |x| and max are exact in fp16; finite inputs)
__device__ __forceinline__ __half2 amax8h(uint4 v, __half2 a) {
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) a = __hmax2(a, __habs2(h[i]));
    return a;
}
__device__ __forceinline__ float amax_of(__half2 a) {
    return fmaxf(__low2float(a), __high2float(a));
}



// q = clamp(round_half_away(fl32(x / s)), ±127), the oracle's definition, by the division (exact
// path, taken rarely — see quant8).
__device__ __forceinline__ int quant_code_exact(float x, float s) {
    return min(127, max(-127, (int)roundf(__fdiv_rn(x, s))));
}

static __device__ __noinline__ uint2 quant8_exact(uint4 u, float s, int& t) {
    const __half* h = reinterpret_cast<const __half*>(&u);
    uint32_t w[2] = {0, 0};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int q = quant_code_exact(__half2float(h[e]), s);
        t += q;
        w[e >> 2] |= (uint32_t)(q & 0xff) << (8 * (e & 3));
    }
    return make_uint2(w[0], w[1]);
}

// 8 fp16 -> 8 int8 codes clamp(⌈x / s⌋, ±127), bit-identical to quant_code_exact, accumulating their
// sum into t (inv = __frcp_rn(s)). Without a division: r = fl(x * inv) is within
// (2^-24 + 2^-24 + 2^-48)|x/s| of x/s and fl(x/s) within 2^-24 |x/s|, so for |x/s| < 128 the two
// differ by < 2^-15. Unless r lies within 2^-14 of a half-integer, both therefore round to the same
// integer, and away from ties round-half-away equals round-to-nearest (rintf). Clamping r to ±127
// first is exact too (r >= 127 implies fl(x/s) > 126.99, which rounds and clamps to 127). Only if
// one of the 8 is near a tie (probability ~6e-5 each) the exact path recomputes all 8.
__device__ __forceinline__ uint2 quant8(uint4 u, float s, float inv, int& t) {
    const __half2* h = reinterpret_cast<const __half2*>(&u);
    float r[8];
    bool near_tie = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(h[e]);
        r[2 * e] = __fmul_rn(f.x, inv);
        r[2 * e + 1] = __fmul_rn(f.y, inv);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float rc = fminf(fmaxf(r[i], -127.0f), 127.0f);
        const float ri = rintf(rc);
        near_tie |= fabsf(rc - ri) >= 0.5f - 0x1p-14f;
        r[i] = ri;
    }
    if (near_tie) return quant8_exact(u, s, t);
    uint32_t w[2] = {0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int q = __float2int_rz(r[i]);   // r[i] is integer-valued
        t += q;
        w[i >> 2] |= (uint32_t)(q & 0xff) << (8 * (i & 3));
    }
    return make_uint2(w[0], w[1]);
}

// quant8 with the exact division only for the element(s) near a tie (the persistent chain's quantizer,
// where one slow row delays the whole grid): bit-identical to quant8.
__device__ __forceinline__ uint2 quant8_pe(uint4 u, float s, float inv, int& t) {
    const __half2* h = reinterpret_cast<const __half2*>(&u);
    float x[8], r[8];
    bool near_tie = false;
    uint32_t near = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(h[e]);
        x[2 * e] = f.x;
        x[2 * e + 1] = f.y;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float rc = fminf(fmaxf(__fmul_rn(x[i], inv), -127.0f), 127.0f);
        const float ri = rintf(rc);
        const bool nt = fabsf(rc - ri) >= 0.5f - 0x1p-14f;
        near |= (uint32_t)nt << i;
        near_tie |= nt;
        r[i] = ri;
    }
    if (near_tie) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (near & (1u << i)) r[i] = (float)quant_code_exact(x[i], s);
    }
    uint32_t w[2] = {0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int q = __float2int_rz(r[i]);   // r[i] is integer-valued
        t += q;
        w[i >> 2] |= (uint32_t)(q & 0xff) << (8 * (i & 3));
    }
    return make_uint2(w[0], w[1]);
}

}  // namespace qoq
