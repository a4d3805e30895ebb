// kv4_attention.cu — the KV4 cache and decode attention (NEXT-4; §5.3).
// Readings Q27-Q29:
//   kv4_append_kernel      : per (sequence, kv head) the new token's K and V rows of D = 128 fp16 are
//                            quantized to asymmetric UINT4 with an fp16 scale and an fp16 (integer) zero
//                            point — the per-channel rule of Q20-Q22 — and written into the sequence's
//                            page slot ("dynamic", "updated on-the-fly").
//   kv4_decode_attn_kernel : o_h = softmax(q_h K̂ᵀ/√D) V̂ for every query head h sharing kv head g (GQA),
//                            a cluster of 4 CTAs per (sequence, kv head), 8 warps each striding over chunks
//                            of 32/R tokens (butterfly-reduced scores, online softmax in fp32), the 32 warp
//                            states merged by CTA 0 through distributed shared memory.
// Dequantization (q − z)·s is exact in fp32 (an 11-bit scale times an integer in [−15, 15]); the paper's
// FP16 arithmetic was an A100 CUDA-core roofline measure that B200 does not need.
#include <cooperative_groups.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "qoq_internal.h"
#include "sm100_ptx.cuh"

namespace qoq {

constexpr int kKvD = 128;       // head dim (Llama / Qwen families)
constexpr int kAttnWarps = 8;
#ifndef QOQ_KV4_SPLIT
#define QOQ_KV4_SPLIT 2
#endif
constexpr int kAttnSplit = QOQ_KV4_SPLIT;
#ifndef QOQ_KV4_MINB
#define QOQ_KV4_MINB 2   // CTAs per SM the register budget is sized for
#endif
#ifndef QOQ_KV4_STAGES
#define QOQ_KV4_STAGES 3
#endif
constexpr int kKvStages = QOQ_KV4_STAGES;    // pages in flight per CTA (TMA bulk copies into shared memory)   // CTAs (one thread-block cluster) per (sequence, kv head), merged over DSMEM

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

// Each warp walks its sequence in chunks of C = 32 / R tokens. For one chunk a lane (owning dims
// 4l..4l+3) forms the 32 partial dot products (token c, head j) from its 4 dequantized K values; one
// butterfly reduce-scatter (31 shuffles) leaves lane L with the full score of (c, j) = (L / R, L % R).
// The chunk's softmax update runs on those lanes (max over the lanes of one head, one exp2 each), the
// 32 probabilities are broadcast back by shuffles and the lane accumulates p · v̂ for its 4 dims.
template <int R>
__global__ void __launch_bounds__(kAttnWarps * 32, QOQ_KV4_MINB) kv4_decode_attn_kernel(
    const __half* __restrict__ Q, const uint8_t* __restrict__ pages, const int32_t* __restrict__ block_table,
    const int32_t* __restrict__ seq_lens, int H_kv, int P, int max_pages, __half* __restrict__ O) {
    constexpr int C = 32 / R;
    __shared__ float sm_m[kAttnWarps][R], sm_l[kAttnWarps][R];
    __shared__ float sm_acc[kAttnWarps][R][kKvD];
    pdl_wait();
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int b = blockIdx.x, g = blockIdx.y, l = threadIdx.x & 31;
    // warp index via a lane-0 broadcast: provably warp-uniform, so the token loop (and the shuffles in
    // it) need no per-shuffle reconvergence code
    const int w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int rank = (int)cluster.block_rank();           // = blockIdx.z: this CTA's share of the tokens
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
    const int myc = l / R, myj = l % R;
    // TMA pipeline: the (page, kv head) slice — K codes, V codes, (s, z) pairs: P·(D+8) contiguous bytes —
    // arrives in shared memory by one cp.async.bulk per page, kKvStages pages ahead of the warps.
    extern __shared__ __align__(16) uint8_t stage_buf[];
    __shared__ __align__(8) uint64_t full_bar[kKvStages];
    const int NP = (T + P - 1) / P;                        // pages of this sequence
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
    for (int n = 0; n < my_pages; ++n) {
        const int stg = n % kKvStages;
        mbar_wait(&full_bar[stg], (uint32_t)((n / kKvStages) & 1));
        const uint8_t* base = stage_buf + (size_t)stg * hb;
        const int tp = (rank + kAttnSplit * n) * P;        // first token of this page
        for (int o0 = w * C; o0 < P; o0 += kAttnWarps * C) {
            const int t0 = tp + o0;
            if (t0 >= T) break;
            uint32_t kc[C], vc[C], kp[C], vp[C];           // codes (16 bits), (s, z) fp16 pairs
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const bool in = t0 + c < T;
                kc[c] = in ? reinterpret_cast<const uint16_t*>(base + (size_t)(o0 + c) * (kKvD / 2))[l] : 0u;
                vc[c] = in ? reinterpret_cast<const uint16_t*>(base + (size_t)(P + o0 + c) * (kKvD / 2))[l] : 0u;
                kp[c] = in ? reinterpret_cast<const uint32_t*>(base + (size_t)P * kKvD)[o0 + c] : 0u;
                vp[c] = in ? reinterpret_cast<const uint32_t*>(base + (size_t)P * kKvD)[P + o0 + c] : 0u;
            }
            float v[32];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                float kh[4];
                const float2 k2 = __half22float2(*reinterpret_cast<const __half2*>(&kp[c]));
                dequant4(kc[c], k2.x, -k2.y * k2.x, kh);
#pragma unroll
                for (int j = 0; j < R; ++j)
                    v[c * R + j] = qf[j][0] * kh[0] + qf[j][1] * kh[1] + qf[j][2] * kh[2] + qf[j][3] * kh[3];
            }
            // butterfly reduce-scatter: lane L ends with the warp sum of v[L]
#pragma unroll
            for (int st = 16; st >= 1; st >>= 1) {
                const bool up = (l & st) != 0;
#pragma unroll
                for (int i = 0; i < st; ++i) {
                    const float send = up ? v[i] : v[i + st];
                    const float keep = up ? v[i + st] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
                }
            }
            const float sc = (t0 + myc < T) ? v[0] : -INFINITY;
            float cm = sc;                                          // chunk max over the lanes of head myj
#pragma unroll
            for (int x = R; x < 32; x <<= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, x));
            float mj = m[0];
#pragma unroll
            for (int j = 1; j < R; ++j) mj = (myj == j) ? m[j] : mj;
            const float mnew = fmaxf(mj, cm);
            const float p = (sc == -INFINITY) ? 0.0f : exp2f(sc - mnew);
            const float corr = (mj == -INFINITY) ? 0.0f : exp2f(mj - mnew);
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const float cj = __shfl_sync(0xffffffffu, corr, j);
                m[j] = __shfl_sync(0xffffffffu, mnew, j);
                lsum[j] *= cj;
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[j][i] *= cj;
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                float vh[4];
                const float2 v2 = __half22float2(*reinterpret_cast<const __half2*>(&vp[c]));
                dequant4(vc[c], v2.x, -v2.y * v2.x, vh);
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const float pc = __shfl_sync(0xffffffffu, p, c * R + j);
                    lsum[j] += pc;
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[j][i] = __fmaf_rn(pc, vh[i], acc[j][i]);
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
