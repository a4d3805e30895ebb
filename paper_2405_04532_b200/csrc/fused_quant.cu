// fused_quant.cu — per-token INT8 activation quantization fused into the layer that produces the
// activation (NEXT-2; "we fuse activation quantization into the preceding layernorm for the
// QKV projection and the first FFN layer, or into the preceding activation kernel for the second FFN
// layer"; Fig. 7). Readings Q23-Q26:
//   rmsnorm_quant_kernel  : y = fp16((x · r) · γ), r = 1 / sqrt(S/K + eps), S = Σ x² EXACT (128-bit
//                           integer in units of 2^-50), rounded once to fp64 — so r does not depend on
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
#include <cstdlib>

#include "qoq_internal.h"
#include "qoq_quant.cuh"
#include "sm100_ptx.cuh"

namespace qoq {


struct U128 {
    unsigned long long lo, hi;
};

__device__ __forceinline__ void add128(U128& a, unsigned long long lo, unsigned long long hi) {
    a.lo += lo;
    a.hi += hi + (a.lo < lo ? 1ull : 0ull);
}

// Exact Σx² in two 64-bit integer classes (units 2^-50). An fp16 x with exponent field e and
// significand field f is x = m · 2^(e - 25) with m = f | 0x400 (e > 0) or m = 2f (e == 0, subnormal),
// so x² · 2^50 = m² · 2^(2e), m² < 2^22. Class A (e < 16) adds m² · 2^(2e) (< 2^52), class B (e >= 16)
// adds m² · 2^(2e - 32) (< 2^50) in units of 2^-18; each is one IMAD.WIDE.U32 (FMA pipe), and 2^12
// terms per thread stay below 2^64 (K <= 65536 is enforced). Combined exactly: S = A + B · 2^32.
struct SqAcc {
    unsigned long long a, b;
};

__device__ __forceinline__ void sq_acc(SqAcc& acc, unsigned h) {
    const unsigned e = (h >> 10) & 31u, f = h & 0x3ffu;
    const unsigned m = e ? (f | 0x400u) : (f << 1);
    const unsigned sq = m * m;
    const unsigned p = 1u << ((2u * e) & 31u);
    acc.a += (unsigned long long)sq * (e < 16u ? p : 0u);   // IMAD.WIDE.U32
    acc.b += (unsigned long long)sq * (e < 16u ? 0u : p);
}

__device__ __forceinline__ void sq_acc8(SqAcc& acc, uint4 v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        sq_acc(acc, w[i] & 0xffffu);
        sq_acc(acc, w[i] >> 16);
    }
}

// per-thread classes -> one 128-bit integer (units 2^-50): A + B * 2^32
__device__ __forceinline__ U128 sq_total(SqAcc acc) {
    U128 r{acc.a, 0ull};
    add128(r, acc.b << 32, acc.b >> 32);
    return r;
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

// Q25: r = 1 / sqrt(S/K + eps) in IEEE fp64 (S = Σ x² · 2^50 exactly); 0 for S/K + eps == 0.
__device__ __forceinline__ double rms_rinv(U128 S, int K, double eps) {
    const double ms = ldexp(u128_to_double_rn(S), -50) / (double)K + eps;
    return ms == 0.0 ? 0.0 : 1.0 / sqrt(ms);
}

// fp16 rounding of a value v known only as an fp32 approximation y with |y - v| <= tol_ulps fp32 ulps:
// safe (fp16_rn(y) == fp16_rn(v)) when y is in the fp16 normal range and its 13 bits below the fp16
// significand are more than tol_ulps away from the midpoint pattern 0x1000 (no fp16 rounding boundary
// between y and v). Otherwise the caller recomputes v exactly in fp64.
__device__ __forceinline__ bool fp16_round_safe(float y, int tol_ulps) {
    const unsigned u = __float_as_uint(y) & 0x7fffffffu;
    // |y| in [2^-14, 2^15) (fp16 normal, no overflow): biased fp32 exponent in [113, 141]
    const bool in_range = u - (113u << 23) < ((142u - 113u) << 23);
    // low 13 bits outside [0x1000 - tol, 0x1000 + tol]
    const bool far = ((u - (0x1000u - (unsigned)tol_ulps)) & 0x1fffu) > 2u * (unsigned)tol_ulps;
    return in_range && far;
}

// exact element (Q24): fp16_rn((x · r) · γ) in fp64
static __device__ __noinline__ __half rms_exact(__half x, __half g, double r) {
    return __double2half(__dmul_rn(__dmul_rn((double)__half2float(x), r), (double)__half2float(g)));
}

// 8 fp16 y = fp16_rn((x · r) · γ) (Q24). Fast path in fp32 with r32 = fl32(r): |y32 - y| <= 3 ulp32
// (three roundings of 2^-24 relative, each <= 1 ulp of y's binade, plus <= 2^-50 for y in fp64); an
// element whose y32 lies within 16 ulp32 of an fp16 rounding boundary takes the fp64 path.
__device__ __forceinline__ uint4 rms_apply8(uint4 xv, uint4 gv, float r32, double r) {
    const __half2* x = reinterpret_cast<const __half2*>(&xv);
    const __half2* g = reinterpret_cast<const __half2*>(&gv);
    uint4 out;
    __half2* y = reinterpret_cast<__half2*>(&out);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 xf = __half22float2(x[e]), gf = __half22float2(g[e]);
        const float y0 = __fmul_rn(__fmul_rn(xf.x, r32), gf.x);
        const float y1 = __fmul_rn(__fmul_rn(xf.y, r32), gf.y);
        __half2 h = __floats2half2_rn(y0, y1);
        if (!fp16_round_safe(y0, 16)) h.x = rms_exact(__low2half(x[e]), __low2half(g[e]), r);
        if (!fp16_round_safe(y1, 16)) h.y = rms_exact(__high2half(x[e]), __high2half(g[e]), r);
        y[e] = h;
    }
    return out;
}

// exact element (Q24, Q26): fp16_rn(silu(g) · u), silu(g) = g / (1 + exp(-g)) in fp64
static __device__ __noinline__ __half silu_exact(__half g, __half u) {
    const double gd = (double)__half2float(g);
    const double s = __ddiv_rn(gd, __dadd_rn(1.0, exp(-gd)));
    return __double2half(__dmul_rn(s, (double)__half2float(u)));
}

// fp32 silu(g)·u: expf (<= 2 ulp), IEEE add, __fdividef (<= 2 ulp for a divisor in [1, 2^126]) and
// product: relative error < 2^-21 + 2^-22 + 2^-23 (expf's error carried through 1 + e, the division,
// the roundings) < 16 ulp32 of the result's binade; boundary band 48 ulp32, else the fp64 path (which
// also takes every |h| < 2^-14, so a divisor overflowing to inf for g < -88 never decides a result).
__device__ __forceinline__ float silu_mul_f32(float g, float u) {
    return __fmul_rn(__fdividef(g, __fadd_rn(1.0f, expf(-g))), u);
}

// 8 fp16 h = fp16_rn(silu(g) · u) (Q24, Q26)
__device__ __forceinline__ uint4 silu_mul8(uint4 gv, uint4 uv) {
    const __half2* g = reinterpret_cast<const __half2*>(&gv);
    const __half2* u = reinterpret_cast<const __half2*>(&uv);
    uint4 out;
    __half2* h = reinterpret_cast<__half2*>(&out);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 gf = __half22float2(g[e]), uf = __half22float2(u[e]);
        const float h0 = silu_mul_f32(gf.x, uf.x), h1 = silu_mul_f32(gf.y, uf.y);
        __half2 r = __floats2half2_rn(h0, h1);
        if (!fp16_round_safe(h0, 48)) r.x = silu_exact(__low2half(g[e]), __low2half(u[e]));
        if (!fp16_round_safe(h1, 48)) r.y = silu_exact(__high2half(g[e]), __high2half(u[e]));
        h[e] = r;
    }
    return out;
}

// Second half of both kernels: the fp16 layer output of this row is staged in shared memory
// (buf[0, nv)); amax (already reduced into the scale sh) -> codes, written coalesced, plus t_x.
__device__ __forceinline__ void quantize_staged(const uint4* buf, int nv, __half sh, uint2* out, __half* sx,
                                                int32_t* tx, int m, int* redi) {
    const float s = __half2float(sh), inv = __frcp_rn(s);
    int t = 0;
#pragma unroll 4
    for (int i = threadIdx.x; i < nv; i += blockDim.x) out[i] = quant8(buf[i], s, inv, t);
    if (tx) t = block_reduce_sum(t, redi);
    if (threadIdx.x == 0) {
        sx[m] = sh;
        if (tx) tx[m] = t;
    }
}

// One CTA per token row. Rows with K <= kStageMaxK are staged in dynamic shared memory (the row is read
// from HBM once; the passes over it run from shared memory, with rolled loops that keep the code small
// and the occupancy high); longer rows recompute y from L2 in each pass (bit-identical).
constexpr int kStageMaxK = 32768;

__global__ void __launch_bounds__(1024) rmsnorm_quant_kernel(const __half* __restrict__ X, int ldx,
                                                             const __half* __restrict__ gamma, double eps,
                                                             int K, int8_t* __restrict__ qx,
                                                             __half* __restrict__ sx,
                                                             int32_t* __restrict__ tx) {
    extern __shared__ uint4 buf[];
    __shared__ U128 red128[32];
    __shared__ float redf[32];
    __shared__ int redi[32];
    pdl_launch_dependents();
    pdl_wait();
    const int m = blockIdx.x, T = blockDim.x;
    const uint4* row = reinterpret_cast<const uint4*>(X + (size_t)m * ldx);
    const uint4* g4 = reinterpret_cast<const uint4*>(gamma);
    uint2* out = reinterpret_cast<uint2*>(qx + (size_t)m * K);
    const int nv = K / 8;
    const bool staged = K <= kStageMaxK;
    SqAcc S{0ull, 0ull};
    if (staged) {
#pragma unroll 4
        for (int i = threadIdx.x; i < nv; i += T) {
            const uint4 v = __ldg(row + i);
            sq_acc8(S, v);
            buf[i] = v;
        }
    } else {
        for (int i = threadIdx.x; i < nv; i += T) sq_acc8(S, __ldg(row + i));
    }
    const double r = rms_rinv(block_reduce_u128(sq_total(S), red128), K, eps);
    const float r32 = __double2float_rn(r);
    __half2 a2 = __float2half2_rn(0.0f);
    if (staged) {
#pragma unroll 2
        for (int i = threadIdx.x; i < nv; i += T) {
            const uint4 y = rms_apply8(buf[i], __ldg(g4 + i), r32, r);
            a2 = amax8h(y, a2);
            buf[i] = y;
        }
        const __half sh = sym_scale(block_reduce_max(amax_of(a2), redf), 127.0f);
        quantize_staged(buf, nv, sh, out, sx, tx, m, redi);
        return;
    }
    for (int i = threadIdx.x; i < nv; i += T) a2 = amax8h(rms_apply8(__ldg(row + i), __ldg(g4 + i), r32, r), a2);
    const __half sh = sym_scale(block_reduce_max(amax_of(a2), redf), 127.0f);
    const float s = __half2float(sh), inv = __frcp_rn(s);
    int t = 0;
    for (int i = threadIdx.x; i < nv; i += T) out[i] = quant8(rms_apply8(__ldg(row + i), __ldg(g4 + i), r32, r), s, inv, t);
    if (tx) t = block_reduce_sum(t, redi);
    if (threadIdx.x == 0) {
        sx[m] = sh;
        if (tx) tx[m] = t;
    }
}

__global__ void __launch_bounds__(1024) silu_mul_quant_kernel(const __half* __restrict__ G,
                                                              const __half* __restrict__ U, int ldg, int K,
                                                              int8_t* __restrict__ qx,
                                                              __half* __restrict__ sx,
                                                              int32_t* __restrict__ tx) {
    extern __shared__ uint4 buf[];
    __shared__ float redf[32];
    __shared__ int redi[32];
    pdl_launch_dependents();
    pdl_wait();
    const int m = blockIdx.x, T = blockDim.x;
    const uint4* g4 = reinterpret_cast<const uint4*>(G + (size_t)m * ldg);
    const uint4* u4 = reinterpret_cast<const uint4*>(U + (size_t)m * ldg);
    uint2* out = reinterpret_cast<uint2*>(qx + (size_t)m * K);
    const int nv = K / 8;
    __half2 a2 = __float2half2_rn(0.0f);
    if (K <= kStageMaxK) {
#pragma unroll 2
        for (int i = threadIdx.x; i < nv; i += T) {
            const uint4 h = silu_mul8(__ldg(g4 + i), __ldg(u4 + i));
            a2 = amax8h(h, a2);
            buf[i] = h;
        }
        const __half sh = sym_scale(block_reduce_max(amax_of(a2), redf), 127.0f);
        quantize_staged(buf, nv, sh, out, sx, tx, m, redi);
        return;
    }
    for (int i = threadIdx.x; i < nv; i += T) a2 = amax8h(silu_mul8(__ldg(g4 + i), __ldg(u4 + i)), a2);
    const __half sh = sym_scale(block_reduce_max(amax_of(a2), redf), 127.0f);
    const float s = __half2float(sh), inv = __frcp_rn(s);
    int t = 0;
    for (int i = threadIdx.x; i < nv; i += T) out[i] = quant8(silu_mul8(__ldg(g4 + i), __ldg(u4 + i)), s, inv, t);
    if (tx) t = block_reduce_sum(t, redi);
    if (threadIdx.x == 0) {
        sx[m] = sh;
        if (tx) tx[m] = t;
    }
}

namespace {
// Few rows (decode): 1024 threads per row (measured best at M = 64) so each thread's chain of loads is short; many rows
// (prefill): K/32 threads (128..256) per row, many CTAs per SM overlapping their reduction latencies.
int row_threads(int M, int K) {
    if (const int t = knobs().fq_threads) {            // tuning override (tools only): 128..1024
        if (t >= 128 && t <= 1024 && t % 32 == 0) return t;
    }
    if (M >= 2 * 148) return K >= 8192 ? 256 : 128;
    return 1024;
}

cudaLaunchConfig_t row_cfg(int M, int K, cudaStream_t st, cudaLaunchAttribute* attr, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(M);
    cfg.blockDim = dim3(row_threads(M, K));
    cfg.dynamicSmemBytes = K <= kStageMaxK ? (size_t)K * 2 : 0;
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
    cudaLaunchConfig_t cfg = row_cfg(M, K, st, attr, pdl);
    if (cfg.dynamicSmemBytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(rmsnorm_quant_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)cfg.dynamicSmemBytes);
        if (e != cudaSuccess) return e;
    }
    return cudaLaunchKernelEx(&cfg, rmsnorm_quant_kernel, static_cast<const __half*>(X), ldx,
                              static_cast<const __half*>(gamma), eps, K, qx, static_cast<__half*>(sx), tx);
}

cudaError_t launch_silu_mul_quantize(const void* G, const void* U, int ldg, int M, int K, int8_t* qx, void* sx,
                                     int32_t* tx, cudaStream_t st, bool pdl) {
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = row_cfg(M, K, st, attr, pdl);
    if (cfg.dynamicSmemBytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(silu_mul_quant_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)cfg.dynamicSmemBytes);
        if (e != cudaSuccess) return e;
    }
    return cudaLaunchKernelEx(&cfg, silu_mul_quant_kernel, static_cast<const __half*>(G),
                              static_cast<const __half*>(U), ldg, K, qx, static_cast<__half*>(sx), tx);
}

}  // namespace qoq
