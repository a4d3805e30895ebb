// qoq_internal.h — host-side declarations shared by the C-ABI shim (qoq_api.cu) and the kernel
// translation units. Not part of the public ABI (that is include/qoq_b200.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace qoq {

constexpr int kTileN = 128;          // output channels per packed tile (MMA M)
constexpr int kTileK = 128;          // input channels per packed tile (= group size g)
constexpr int kTileBytes = 8448;     // 8192 B of u4 codes + 128 B s_u8 + 128 B z*s_u8
constexpr int kPcTileBytes = 8192;   // per-channel W4A8 (NEXT-1): the u4 codes only

// Work decomposition of one GEMM launch (host planner <-> kernel scheduler).
struct GemmPlan {
    int BN;          // token tile = MMA N (16, 32, 64, 128 or 256)
    int MT, NT, KT;  // token tiles, 128-row weight tiles, 128-deep K tiles
    int MB;          // token tiles per band of the work order (tile_coords in w4a8_gemm.cu)
    int KS;          // pipeline steps per output tile (2 k-tiles each, last may hold 1)
    int T;           // output tiles = MT * NT
    long long I;     // steps = T * KS
    int G;           // CTAs (persistent, <= #SMs)
    int mode;        // 0: whole tiles round-robin; 1: stream-K (global workspace); 2: S-CTA cluster split-K
    int S;           // mode 2: CTAs (cluster size) per output tile
    int CG;          // 1, or 2: CTA pairs (cta_group::2); then T counts tile pairs and G pairs
    size_t ws_bytes; // INT32 partials + per-tile counters (mode 1), else 0
};

GemmPlan plan_gemm(int M, int N, int K, int num_sms);

struct GemmArgs {
    const int8_t* qx;
    const void* sx;
    const int32_t* tx;
    const void* packed;
    const void* s0;
    void* out;       // fp16 Y or int32 acc
    int ldo;
    bool out_i32;
    int M, N, K;
    void* ws;
    void* trace = nullptr;   // debug timeline buffer (16 u64 per CTA) or nullptr
    // fused per-token quantization (M <= kFuseMaxM): X [M][ldx] fp16 is quantized inside the GEMM
    // into qx / sx / tx (then outputs, not inputs); qsync: 2 zero-initialized ints
    const void* X = nullptr;
    int ldx = 0;
    int* qsync = nullptr;
    // per-channel W4A8 (NEXT-1): packed holds 8192-byte code tiles, s0 is s_w, zw the u8 zero points;
    // Y = s_x s_w (acc - z_w t_x) (tx required)
    const uint8_t* zw = nullptr;
};

constexpr int kFuseMaxM = 64;   // above: quantizer kernel + GEMM (the prologue would serialize M rows)

cudaError_t launch_w4a8_gemm(const GemmArgs& a, const GemmPlan& p, cudaStream_t st, bool pdl);
cudaError_t launch_quantize_weights(const void* W, int N, int K, void* packed, void* s0, cudaStream_t st);
cudaError_t launch_pc_quantize_weights(const void* W, int N, int K, void* packed, void* s_w, uint8_t* z_w,
                                       cudaStream_t st);
cudaError_t launch_quantize_activations(const void* X, int M, int K, int ldx, int8_t* qx, void* sx,
                                        int32_t* tx, cudaStream_t st, bool pdl);

// NEXT-2: per-token quantization fused into RMSNorm / SiLU·mul (fused_quant.cu)
cudaError_t launch_rmsnorm_quantize(const void* X, int ldx, const void* gamma, double eps, int M, int K,
                                    int8_t* qx, void* sx, int32_t* tx, cudaStream_t st, bool pdl);
cudaError_t launch_silu_mul_quantize(const void* G, const void* U, int ldg, int M, int K, int8_t* qx, void* sx,
                                     int32_t* tx, cudaStream_t st, bool pdl);

// NEXT-4: KV4 cache + decode attention (kv4_attention.cu), D = 128
cudaError_t launch_kv4_append(const void* K, const void* V, const int32_t* slots, int B, int H_kv, int P,
                              uint8_t* pages, cudaStream_t st);
cudaError_t launch_kv4_decode_attention(const void* Q, const uint8_t* pages, const int32_t* block_table,
                                        const int32_t* seq_lens, int B, int H, int H_kv, int P, int max_pages,
                                        void* O, cudaStream_t st);

}  // namespace qoq
