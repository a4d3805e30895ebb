// kv4_attention.cu — the KV4 cache and decode attention (NEXT-4; §5.3).
// Readings Q27-Q29:
//   kv4_append_kernel      : per (sequence, kv head) the new token's K and V rows of D = 128 fp16 are
//                            quantized to asymmetric UINT4 with an fp16 scale and an fp16 (integer) zero
//                            point — the per-channel rule of Q20-Q22 — and written into the sequence's
//                            page slot ("dynamic", "updated on-the-fly").
//   kv4_decode_attn_kernel : o_h = softmax(q_h K̂ᵀ/√D) V̂ for every query head h sharing kv head g (GQA),
//                            a cluster of QOQ_KV4_SPLIT CTAs per (sequence, kv head) splitting its pages,
//                            4 warps each taking 16-token chunks on tensor cores (mma.sync m16n8k16,
//                            fp32 accumulation, online softmax in base 2), the warp states merged by CTA 0
//                            through distributed shared memory.
// The dequantization (q − z)·s is folded out of both contractions: the tensor cores multiply exact fp16
// integers (q − z) and the scales are applied to the fp32 results (QK) or to the probabilities (PV).
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "qoq_internal.h"
#include "sm100_ptx.cuh"

namespace qoq {

constexpr int kKvD = 128;       // head dim (Llama / Qwen families)
constexpr int kAttnWarps = 4;   // a warp takes 16-token chunks of the staged pages
#ifndef QOQ_KV4_SPLIT
#define QOQ_KV4_SPLIT 2
#endif
constexpr int kAttnSplit = QOQ_KV4_SPLIT;
#ifndef QOQ_KV4_MINB
#define QOQ_KV4_MINB 4   // CTAs per SM the register budget is sized for (4: 128 registers, measured best)
#endif
#ifndef QOQ_KV4_STAGES
#define QOQ_KV4_STAGES 3
#endif
constexpr int kKvStages = QOQ_KV4_STAGES;    // pages in flight per CTA (TMA bulk copies into shared memory)

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

// ------------------------------------------------------------------ decode attention on tensor cores
//
// Per warp, a chunk of 16 tokens of one staged page; the GQA group's R query heads are the MMA rows
// (padded to 16), so both contractions run as mma.sync.m16n8k16 (fp16 inputs, fp32 accumulation):
//   S[h][t] = Σ_d q[h][d] · (c_K[t][d] − z_K[t])           (QK: A = q, B = integer codes − zero point)
//   score    = S · s_K[t] · log2(e)/√D                       (the scale folded out of the dot product)
//   O[h][d] += Σ_t (p[h][t] · s_V[t]) · (c_V[t][d] − z_V[t]) (PV in bf16: A = p·s_V split into three bf16
//                                                             terms, B = integer codes − zero point)
// Every MMA input is exact: q as given (fp16), c − z ∈ [−15, 15], and p·s_V carried as three bf16 terms
// (≈ 24 significant bits over fp32's exponent range), so the only roundings are the fp32 accumulations —
// the error model of tests/kv4_tol.py. The QK accumulator fragment of two 8-token blocks IS the PV A fragment (heads ×
// tokens), so scores never leave registers. Online softmax in base 2 per head (a quad of lanes).

// mma.sync m16n8k16, row.col, f16 x f16 -> f32, accumulating rows gq (d0, d1) in place. A's rows gq + 8
// are always zero here (padding heads), so their accumulators (p2, p3) stay 0 — one scratch pair shared by
// every call (the B operands are finite integers, so 0·B adds exact zeros).
__device__ __forceinline__ void mma16816(float& d0, float& d1, float& p2, float& p3, uint32_t a0, uint32_t a2,
                                         uint32_t b0, uint32_t b1) {
    asm(   // not volatile: a pure function of its operands, so the scheduler may interleave independent chains
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d0), "+f"(d1), "+f"(p2), "+f"(p3)
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

// The same MMA with bf16 operands (PV: the probabilities need fp32's exponent range, see below).
__device__ __forceinline__ void mma16816_bf16(float& d0, float& d1, float& p2, float& p3, uint32_t a0, uint32_t a2,
                                              uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d0), "+f"(d1), "+f"(p2), "+f"(p3)
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t bf2bits(__nv_bfloat162 h) { return *reinterpret_cast<uint32_t*>(&h); }

// Codes to exact fp16 (c − z) with 3 instructions per half2: PRMT places the code bytes under 0x64 high
// bytes, LOP3 keeps one nibble per half (0x6400 | c = 1024 + c, or 0x6400 | 16c = 1024 + 16c), and one
// HFMA2 scales by (1 or 1/16) and subtracts (1024 + z or 64 + z): every step is exact in fp16.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ uint32_t hfma2_bits(uint32_t x, uint32_t m, uint32_t c) {
    const __half2 r = __hfma2(*reinterpret_cast<const __half2*>(&x), *reinterpret_cast<const __half2*>(&m),
                              *reinterpret_cast<const __half2*>(&c));
    return *reinterpret_cast<const uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t h2bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

template <int R>
__global__ void __launch_bounds__(kAttnWarps * 32, QOQ_KV4_MINB) kv4_decode_attn_kernel(
    const __half* __restrict__ Q, const uint8_t* __restrict__ pages, const int32_t* __restrict__ block_table,
    const int32_t* __restrict__ seq_lens, int H_kv, int P, int max_pages, __half* __restrict__ O) {
    static_assert(R >= 1 && R <= 8, "GQA group of <= 8 query heads (MMA rows 0..7)");
    __shared__ float sm_m[kAttnWarps][R], sm_l[kAttnWarps][R];
    __shared__ float sm_acc[kAttnWarps][R][kKvD];
    pdl_wait();
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int b = blockIdx.x, g = blockIdx.y, lane = threadIdx.x & 31;
    const int w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int rank = (int)cluster.block_rank();
    const int H = H_kv * R;
    const int T = seq_lens[b];
    const int gq = lane >> 2, tq = lane & 3;              // fragment row group / thread in quad
    const float qscale = 1.4426950408889634f / sqrtf((float)kKvD);
    // A fragments of q (rows = heads gq; rows gq + 8 are padding): a0a1 (d = 16kb + 2tq), a4a5 (+8)
    uint32_t qa[8][2];
    {
        const bool real = gq < R;
        const __half* qrow = Q + ((size_t)b * H + (size_t)g * R + (real ? gq : 0)) * kKvD;
#pragma unroll
        for (int kb = 0; kb < 8; ++kb) {
            qa[kb][0] = real ? *reinterpret_cast<const uint32_t*>(qrow + 16 * kb + 2 * tq) : 0u;
            qa[kb][1] = real ? *reinterpret_cast<const uint32_t*>(qrow + 16 * kb + 2 * tq + 8) : 0u;
        }
    }
    float o[16][2];                                        // O fragments: (head gq, d = 8nb + 2tq, +1)
#pragma unroll
    for (int nb = 0; nb < 16; ++nb) o[nb][0] = o[nb][1] = 0.0f;
    float pad2 = 0.0f, pad3 = 0.0f;                        // the padding rows' accumulators (stay 0)
    float m = -INFINITY, lsum = 0.0f;                      // online softmax state of head gq (base 2)
    const size_t hb = kv_head_bytes(P), pb = (size_t)H_kv * hb;
    const int32_t* bt = block_table + (size_t)b * max_pages;
    extern __shared__ __align__(16) uint8_t stage_buf[];
    __shared__ __align__(8) uint64_t full_bar[kKvStages];
    const int NP = (T + P - 1) / P;
    const int my_pages = NP > rank ? (NP - rank + kAttnSplit - 1) / kAttnSplit : 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kKvStages; ++i) mbar_init(&full_bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t policy = policy_evict_first();
    if (threadIdx.x == 0) {
        for (int n = 0; n < kKvStages && n < my_pages; ++n) {
            mbar_arrive_expect_tx(&full_bar[n], (uint32_t)hb);
            bulk_g2s(stage_buf + (size_t)n * hb, pages + (size_t)__ldg(bt + rank + kAttnSplit * n) * pb + (size_t)g * hb,
                     (uint32_t)hb, &full_bar[n], policy);
        }
    }
    const uint32_t ksel = 0x4040u | (0x0101u * (uint32_t)tq);   // PRMT: bytes (w.tq, 0x64, w.tq, 0x64)
    const uint32_t kscale = 0x2C003C00u;                   // half2 (1, 1/16)
    // V (bf16): nibble (gq & 1) of byte (gq >> 1) of word nb, for two tokens: PRMT (w0.byte, -, w1.byte, -),
    // shift the nibble down, OR in the bf16 128.0 exponent (0x4300 | c = 128 + c), subtract 128 + z
    const uint32_t vsel = (uint32_t)(gq >> 1) | ((4u + (gq >> 1)) << 8);
    const uint32_t vshift = 4u * (uint32_t)(gq & 1);
    for (int n = 0; n < my_pages; ++n) {
        const int stg = n % kKvStages;
        mbar_wait(&full_bar[stg], (uint32_t)((n / kKvStages) & 1));
        const uint8_t* base = stage_buf + (size_t)stg * hb;
        const uint32_t* par = reinterpret_cast<const uint32_t*>(base + (size_t)P * kKvD);   // (s, z) fp16 pairs
        const int tp = (rank + kAttnSplit * n) * P;        // first token of this page
        for (int o0 = 16 * w; o0 < P; o0 += 16 * kAttnWarps) {
            if (tp + o0 >= T) break;
            const int valid = T - (tp + o0);               // tokens of this chunk that exist (>= 1)
            // ---- S = q (c_K − z_K)ᵀ for the two 8-token blocks (two independent MMA chains, interleaved);
            // C fragment: (head gq, tokens 8nbt + 2tq, +1)
            float sc[2][4];
            {
                const uint4* row0 = reinterpret_cast<const uint4*>(base + (size_t)(o0 + gq) * (kKvD / 2));
                const uint4* row1 = reinterpret_cast<const uint4*>(base + (size_t)(o0 + 8 + gq) * (kKvD / 2));
                // c = (lo, hi) of byte tq of a word: (1024 + lo, 1024 + 16 hi) -> (lo − z, hi − z)
                const __half z0 = __ushort_as_half((unsigned short)(par[o0 + gq] >> 16));       // fp16 z (integer)
                const __half z1 = __ushort_as_half((unsigned short)(par[o0 + 8 + gq] >> 16));
                const uint32_t zb0 = h2bits(__halves2half2(__hneg(__hadd(__float2half(1024.0f), z0)),
                                                           __hneg(__hadd(__float2half(64.0f), z0))));
                const uint32_t zb1 = h2bits(__halves2half2(__hneg(__hadd(__float2half(1024.0f), z1)),
                                                           __hneg(__hadd(__float2half(64.0f), z1))));
                float acc0[2] = {0.0f, 0.0f}, acc1[2] = {0.0f, 0.0f};
#pragma unroll
                for (int qd = 0; qd < 4; ++qd) {           // 16 words of each code row, 4 at a time
                    const uint4 w0 = row0[qd], w1 = row1[qd];
                    const uint32_t x0[4] = {w0.x, w0.y, w0.z, w0.w}, x1[4] = {w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {       // kb = 2 qd + h2: words 2kb (d 16kb+2tq..) and 2kb+1 (+8)
                        const int kb = 2 * qd + h2;
                        const uint32_t b00 = hfma2_bits(prmt(x0[2 * h2], 0x64646464u, ksel) & 0xFFF0FF0Fu, kscale, zb0);
                        const uint32_t b01 = hfma2_bits(prmt(x0[2 * h2 + 1], 0x64646464u, ksel) & 0xFFF0FF0Fu, kscale, zb0);
                        const uint32_t b10 = hfma2_bits(prmt(x1[2 * h2], 0x64646464u, ksel) & 0xFFF0FF0Fu, kscale, zb1);
                        const uint32_t b11 = hfma2_bits(prmt(x1[2 * h2 + 1], 0x64646464u, ksel) & 0xFFF0FF0Fu, kscale, zb1);
                        mma16816(acc0[0], acc0[1], pad2, pad3, qa[kb][0], qa[kb][1], b00, b01);
                        mma16816(acc1[0], acc1[1], pad2, pad3, qa[kb][0], qa[kb][1], b10, b11);
                    }
                }
                // scores of tokens 8nbt + 2tq, +1 for head gq
#pragma unroll
                for (int nbt = 0; nbt < 2; ++nbt)
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int tt = 8 * nbt + 2 * tq + u;
                        const float sk = __half2float(__ushort_as_half((unsigned short)(par[o0 + tt] & 0xFFFFu)));
                        sc[nbt][u] = tt < valid ? (nbt ? acc1[u] : acc0[u]) * sk * qscale : -INFINITY;
                    }
            }
            // ---- online softmax for head gq over this chunk's 16 tokens (4 per lane of the quad)
            float cm = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
            cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 1));
            cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 2));
            const float mnew = fmaxf(m, cm);
            const float corr = (m == -INFINITY) ? 0.0f : exp2f(m - mnew);
            float pv[2][2], ps = 0.0f;
#pragma unroll
            for (int nbt = 0; nbt < 2; ++nbt)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    pv[nbt][u] = sc[nbt][u] == -INFINITY ? 0.0f : exp2f(sc[nbt][u] - mnew);
                    ps += pv[nbt][u];
                }
            ps += __shfl_xor_sync(0xffffffffu, ps, 1);
            ps += __shfl_xor_sync(0xffffffffu, ps, 2);
            lsum = lsum * corr + ps;
            m = mnew;
            if (__any_sync(0xffffffffu, corr != 1.0f)) {   // the running max moved for some head
#pragma unroll
                for (int nb = 0; nb < 16; ++nb) {
                    o[nb][0] *= corr;
                    o[nb][1] *= corr;
                }
            }
            // ---- PV: A = p · s_V for tokens (2tq, 2tq+1) and (8 + 2tq, 9 + 2tq) as THREE bf16 terms (≈ 24
            // significant bits with fp32's exponent range: a tiny p · s_V would lose its precision in fp16's
            // subnormals), B = V codes − z (exact small integers in bf16)
            uint32_t ap[3][2];
#pragma unroll
            for (int nbt = 0; nbt < 2; ++nbt) {
                float f[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int tt = 8 * nbt + 2 * tq + u;
                    const float sv = __half2float(__ushort_as_half((unsigned short)(par[P + o0 + tt] & 0xFFFFu)));
                    f[u] = pv[nbt][u] * sv;
                }
                const __nv_bfloat162 h1 = __floats2bfloat162_rn(f[0], f[1]);
                const float2 g1 = __bfloat1622float2(h1);
                const float r0 = f[0] - g1.x, r1 = f[1] - g1.y;
                const __nv_bfloat162 h2 = __floats2bfloat162_rn(r0, r1);
                const float2 g2 = __bfloat1622float2(h2);
                ap[0][nbt] = bf2bits(h1);
                ap[1][nbt] = bf2bits(h2);
                ap[2][nbt] = bf2bits(__floats2bfloat162_rn(r0 - g2.x, r1 - g2.y));
            }
            // B fragments: V codes of tokens 2tq, 2tq+1 (b0) and 8+2tq, 9+2tq (b1) at d = 8nb + gq
            const uint4* vr[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int tt = (i < 2 ? 0 : 8) + 2 * tq + (i & 1);
                vr[i] = reinterpret_cast<const uint4*>(base + (size_t)(P + o0 + tt) * (kKvD / 2));
            }
            __nv_bfloat162 vb[2];                          // 128 + z of the two tokens of each pair
#pragma unroll
            for (int pr = 0; pr < 2; ++pr) {
                const int t0 = 8 * pr + 2 * tq;
                const float z0 = __half2float(__ushort_as_half((unsigned short)(par[P + o0 + t0] >> 16)));
                const float z1 = __half2float(__ushort_as_half((unsigned short)(par[P + o0 + t0 + 1] >> 16)));
                vb[pr] = __floats2bfloat162_rn(128.0f + z0, 128.0f + z1);
            }
            // masked tokens (past the sequence end, only in its last chunk) take p = 0 and code = z (no
            // NaN / Inf from never-written page bytes)
            const bool full = valid >= 16;
            const uint32_t keep0 = full ? 0xFFFFFFFFu : ((2 * tq < valid ? 0xFFFFu : 0u) | (2 * tq + 1 < valid ? 0xFFFF0000u : 0u));
            const uint32_t keep1 = full ? 0xFFFFFFFFu : ((8 + 2 * tq < valid ? 0xFFFFu : 0u) | (9 + 2 * tq < valid ? 0xFFFF0000u : 0u));
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {               // words 4 q4 .. 4 q4 + 3 of the four code rows
                const uint4 r0 = vr[0][q4], r1 = vr[1][q4], r2 = vr[2][q4], r3 = vr[3][q4];
                const uint32_t a0[4] = {r0.x, r0.y, r0.z, r0.w}, a1[4] = {r1.x, r1.y, r1.z, r1.w};
                const uint32_t a2[4] = {r2.x, r2.y, r2.z, r2.w}, a3[4] = {r3.x, r3.y, r3.z, r3.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int nb = 4 * q4 + k;
                    uint32_t x0 = ((prmt(a0[k], a1[k], vsel) >> vshift) & 0x000F000Fu) | 0x43004300u;
                    uint32_t x1 = ((prmt(a2[k], a3[k], vsel) >> vshift) & 0x000F000Fu) | 0x43004300u;
                    const uint32_t b0 = bf2bits(__hsub2(*reinterpret_cast<const __nv_bfloat162*>(&x0), vb[0])) & keep0;
                    const uint32_t b1 = bf2bits(__hsub2(*reinterpret_cast<const __nv_bfloat162*>(&x1), vb[1])) & keep1;
#pragma unroll
                    for (int e = 0; e < 3; ++e) mma16816_bf16(o[nb][0], o[nb][1], pad2, pad3, ap[e][0], ap[e][1], b0, b1);
                }
            }
        }
        __syncthreads();                                   // every warp is done with stage stg
        if (threadIdx.x == 0 && n + kKvStages < my_pages) {
            mbar_arrive_expect_tx(&full_bar[stg], (uint32_t)hb);
            bulk_g2s(stage_buf + (size_t)stg * hb,
                     pages + (size_t)__ldg(bt + rank + kAttnSplit * (n + kKvStages)) * pb + (size_t)g * hb,
                     (uint32_t)hb, &full_bar[stg], policy);
        }
    }
    // merge the warps' partial softmax states (head gq of lanes 4gq..4gq+3)
    if (gq < R) {
        if (tq == 0) {
            sm_m[w][gq] = m;
            sm_l[w][gq] = lsum;
        }
#pragma unroll
        for (int nb = 0; nb < 16; ++nb) {
            sm_acc[w][gq][8 * nb + 2 * tq] = o[nb][0];
            sm_acc[w][gq][8 * nb + 2 * tq + 1] = o[nb][1];
        }
    }
    cluster.sync();                                       // every CTA's warp states are in its smem
    if (rank == 0) {
        const float* rm[kAttnSplit];
        const float* rl[kAttnSplit];
        const float* ra[kAttnSplit];
#pragma unroll
        for (int r = 0; r < kAttnSplit; ++r) {
            rm[r] = cluster.map_shared_rank(&sm_m[0][0], r);
            rl[r] = cluster.map_shared_rank(&sm_l[0][0], r);
            ra[r] = cluster.map_shared_rank(&sm_acc[0][0][0], r);
        }
        for (int e = threadIdx.x; e < R * kKvD; e += blockDim.x) {
            const int j = e / kKvD, d = e % kKvD;
            float M = -INFINITY;
#pragma unroll
            for (int r = 0; r < kAttnSplit; ++r)
#pragma unroll
                for (int x = 0; x < kAttnWarps; ++x) M = fmaxf(M, rm[r][x * R + j]);
            float L = 0.0f, A = 0.0f;
            if (M != -INFINITY) {
#pragma unroll
                for (int r = 0; r < kAttnSplit; ++r)
#pragma unroll
                    for (int x = 0; x < kAttnWarps; ++x) {
                        const float mx = rm[r][x * R + j];
                        if (mx == -INFINITY) continue;            // idle warp
                        const float f = exp2f(mx - M);
                        L += rl[r][x * R + j] * f;
                        A += ra[r][(x * R + j) * kKvD + d] * f;
                    }
            }
            O[((size_t)b * H + (size_t)g * R + j) * kKvD + d] = __float2half_rn(L > 0.0f ? A / L : 0.0f);
        }
    }
    cluster.sync();                                       // keep every CTA's smem alive until rank 0 is done
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
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(B, H_kv, kAttnSplit);
    cfg.blockDim = dim3(kAttnWarps * 32);
    cfg.dynamicSmemBytes = (size_t)kKvStages * P * (kKvD + 8);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = kAttnSplit;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const __half* q = static_cast<const __half*>(Q);
    __half* o = static_cast<__half*>(O);
    {   // static (merge buffers) + dynamic (page stages) may exceed the default 48 KB: opt in
        cudaError_t e = cudaSuccess;
        switch (H / H_kv) {
            case 1: e = cudaFuncSetAttribute(kv4_decode_attn_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes); break;
            case 2: e = cudaFuncSetAttribute(kv4_decode_attn_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes); break;
            case 4: e = cudaFuncSetAttribute(kv4_decode_attn_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes); break;
            case 8: e = cudaFuncSetAttribute(kv4_decode_attn_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes); break;
            default: return cudaErrorInvalidValue;
        }
        if (e != cudaSuccess) return e;
    }
    switch (H / H_kv) {
        case 1: return cudaLaunchKernelEx(&cfg, kv4_decode_attn_kernel<1>, q, pages, block_table, seq_lens, H_kv, P, max_pages, o);
        case 2: return cudaLaunchKernelEx(&cfg, kv4_decode_attn_kernel<2>, q, pages, block_table, seq_lens, H_kv, P, max_pages, o);
        case 4: return cudaLaunchKernelEx(&cfg, kv4_decode_attn_kernel<4>, q, pages, block_table, seq_lens, H_kv, P, max_pages, o);
        case 8: return cudaLaunchKernelEx(&cfg, kv4_decode_attn_kernel<8>, q, pages, block_table, seq_lens, H_kv, P, max_pages, o);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qoq
