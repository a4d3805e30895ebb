// kv4_attention.cu — the KV4 cache and decode attention (NEXT-4; §5.3).
// Readings Q27-Q29:
//   kv4_append_kernel      : per (sequence, kv head) the new token's K and V rows of D = 128 fp16 are
//                            quantized to asymmetric UINT4 with an fp16 scale and an fp16 (integer) zero
//                            point — the per-channel rule of Q20-Q22 — and written into the sequence's
//                            page slot ("dynamic", "updated on-the-fly").
//   kv4_decode_attn_kernel : o_h = softmax(q_h K̂ᵀ/√D) V̂ for every query head h sharing kv head g (GQA),
//                            one CTA per (sequence, kv head), 8 warps striding over the tokens with an
//                            online softmax in fp32, merged across warps in shared memory.
// Dequantization (q − z)·s is exact in fp32 (an 11-bit scale times an integer in [−15, 15]); the paper's
// FP16 arithmetic was an A100 CUDA-core roofline measure that B200 does not need.
#include <cuda_fp16.h>
#include <cstdint>

#include "qoq_internal.h"
#include "sm100_ptx.cuh"

namespace qoq {

constexpr int kKvD = 128;       // head dim (Llama / Qwen families)
constexpr int kAttnWarps = 8;

__device__ __forceinline__ size_t kv_head_bytes(int P) { return (size_t)P * (kKvD + 8); }

// grid (B, H_kv), 64 threads: warp 0 quantizes the K row, warp 1 the V row; lane l owns elements 4l..4l+3.
__global__ void __launch_bounds__(64) kv4_append_kernel(const __half* __restrict__ K, const __half* __restrict__ V,
                                                        const int32_t* __restrict__ slots, int H_kv, int P,
                                                        uint8_t* __restrict__ pages) {
    pdl_wait();
    const int b = blockIdx.x, g = blockIdx.y, w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const __half* src = (w == 0 ? K : V) + ((size_t)b * H_kv + g) * kKvD;
    const uint2 raw = reinterpret_cast<const uint2*>(src)[l];
    const __half* hx = reinterpret_cast<const __half*>(&raw);
    float x[4], lo, hi;
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = __half2float(hx[i]);
    lo = fminf(fminf(x[0], x[1]), fminf(x[2], x[3]));
    hi = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    // Eq. 2 with q_min = 0, q_max = 15 (Q20-Q22): s = fp16(fp32(hi - lo) / 15), z = ⌈-lo / s⌋, q = ⌈x / s + z⌋
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
    int q[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = min(15, max(0, (int)round((double)__fdiv_rn(x[i], s) + (double)z)));
    const int slot = slots[b];
    uint8_t* base = pages + (size_t)(slot / P) * H_kv * kv_head_bytes(P) + (size_t)g * kv_head_bytes(P);
    const int o = slot % P;
    uint8_t* codes = base + (size_t)w * P * (kKvD / 2) + (size_t)o * (kKvD / 2);
    reinterpret_cast<uint16_t*>(codes)[l] =
        (uint16_t)((q[0] | (q[1] << 4)) | ((q[2] | (q[3] << 4)) << 8));
    if (l == 0) {
        __half* par = reinterpret_cast<__half*>(base + (size_t)P * kKvD) + (size_t)w * 2 * P + 2 * o;
        par[0] = sh;
        par[1] = __float2half_rn((float)z);
    }
}

// 4 codes of one 16-bit word -> (q - z) * s, exact in fp32
__device__ __forceinline__ void dequant4(uint32_t c, float s, float zs, float (&v)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __fmaf_rn((float)((c >> (4 * i)) & 15u), s, zs);   // q s - z s: exact
}

template <int R>
__global__ void __launch_bounds__(kAttnWarps * 32) kv4_decode_attn_kernel(
    const __half* __restrict__ Q, const uint8_t* __restrict__ pages, const int32_t* __restrict__ block_table,
    const int32_t* __restrict__ seq_lens, int H_kv, int P, int max_pages, __half* __restrict__ O) {
    __shared__ float sm_m[kAttnWarps][R], sm_l[kAttnWarps][R];
    __shared__ float sm_acc[kAttnWarps][R][kKvD];
    pdl_wait();
    const int b = blockIdx.x, g = blockIdx.y, w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int H = H_kv * R;
    const int T = seq_lens[b];
    const float qscale = 1.4426950408889634f / sqrtf((float)kKvD);   // log2(e) / sqrt(D): scores in base 2
    float qf[R][4];
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const uint2 raw = reinterpret_cast<const uint2*>(Q + ((size_t)b * H + (size_t)g * R + j) * kKvD)[l];
        const __half* h = reinterpret_cast<const __half*>(&raw);
#pragma unroll
        for (int i = 0; i < 4; ++i) qf[j][i] = __half2float(h[i]) * qscale;
    }
    float m[R], lsum[R], acc[R][4];
#pragma unroll
    for (int j = 0; j < R; ++j) {
        m[j] = -INFINITY;
        lsum[j] = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[j][i] = 0.0f;
    }
    const size_t hb = kv_head_bytes(P), pb = (size_t)H_kv * hb;
    const int32_t* bt = block_table + (size_t)b * max_pages;
    for (int t = w; t < T; t += kAttnWarps) {
        const uint8_t* base = pages + (size_t)__ldg(bt + t / P) * pb + (size_t)g * hb;
        const int o = t % P;
        const uint32_t kc = __ldg(reinterpret_cast<const uint16_t*>(base + (size_t)o * (kKvD / 2)) + l);
        const uint32_t vc = __ldg(reinterpret_cast<const uint16_t*>(base + (size_t)(P + o) * (kKvD / 2)) + l);
        const __half2* par = reinterpret_cast<const __half2*>(base + (size_t)P * kKvD);
        const float2 kp = __half22float2(par[o]), vp = __half22float2(par[P + o]);
        float kh[4], vh[4];
        dequant4(kc, kp.x, -kp.y * kp.x, kh);   // z s exact in fp32 (integer z <= 15 times an fp16 scale)
        dequant4(vc, vp.x, -vp.y * vp.x, vh);
#pragma unroll
        for (int j = 0; j < R; ++j) {
            float sc = qf[j][0] * kh[0] + qf[j][1] * kh[1] + qf[j][2] * kh[2] + qf[j][3] * kh[3];
#pragma unroll
            for (int x = 16; x > 0; x >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, x);
            const float mn = fmaxf(m[j], sc);
            const float corr = exp2f(m[j] - mn), p = exp2f(sc - mn);
            m[j] = mn;
            lsum[j] = lsum[j] * corr + p;
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[j][i] = acc[j][i] * corr + p * vh[i];
        }
    }
    // merge the 8 warps' partial softmax states
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (l == 0) {
            sm_m[w][j] = m[j];
            sm_l[w][j] = lsum[j];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) sm_acc[w][j][4 * l + i] = acc[j][i];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * kKvD; e += blockDim.x) {
        const int j = e / kKvD, d = e % kKvD;
        float M = -INFINITY;
#pragma unroll
        for (int x = 0; x < kAttnWarps; ++x) M = fmaxf(M, sm_m[x][j]);
        float L = 0.0f, A = 0.0f;
        if (M != -INFINITY) {
#pragma unroll
            for (int x = 0; x < kAttnWarps; ++x) {
                const float f = exp2f(sm_m[x][j] - M);   // 0 for an idle warp (m = -inf)
                L += sm_l[x][j] * f;
                A += sm_acc[x][j][d] * f;
            }
        }
        O[((size_t)b * H + (size_t)g * R + j) * kKvD + d] = __float2half_rn(L > 0.0f ? A / L : 0.0f);
    }
}

cudaError_t launch_kv4_append(const void* K, const void* V, const int32_t* slots, int B, int H_kv, int P,
                              uint8_t* pages, cudaStream_t st) {
    kv4_append_kernel<<<dim3(B, H_kv), 64, 0, st>>>(static_cast<const __half*>(K), static_cast<const __half*>(V),
                                                    slots, H_kv, P, pages);
    return cudaGetLastError();
}

cudaError_t launch_kv4_decode_attention(const void* Q, const uint8_t* pages, const int32_t* block_table,
                                        const int32_t* seq_lens, int B, int H, int H_kv, int P, int max_pages,
                                        void* O, cudaStream_t st) {
    const dim3 grid(B, H_kv), block(kAttnWarps * 32);
    const __half* q = static_cast<const __half*>(Q);
    __half* o = static_cast<__half*>(O);
    switch (H / H_kv) {
        case 1: kv4_decode_attn_kernel<1><<<grid, block, 0, st>>>(q, pages, block_table, seq_lens, H_kv, P, max_pages, o); break;
        case 2: kv4_decode_attn_kernel<2><<<grid, block, 0, st>>>(q, pages, block_table, seq_lens, H_kv, P, max_pages, o); break;
        case 4: kv4_decode_attn_kernel<4><<<grid, block, 0, st>>>(q, pages, block_table, seq_lens, H_kv, P, max_pages, o); break;
        case 8: kv4_decode_attn_kernel<8><<<grid, block, 0, st>>>(q, pages, block_table, seq_lens, H_kv, P, max_pages, o); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace qoq
