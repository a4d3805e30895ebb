// w4a8_common.cuh — device pieces shared by the per-GEMM W4A8 kernel (w4a8_gemm.cu) and the persistent
// decode-chain kernel (w4a8_chain.cu): warp roles, the in-register u4 -> INT8 expansion (P:447,
// P:483-495) and the TMEM accumulator helpers.
#pragma once
#include <cstdint>

#include "sm100_ptx.cuh"

// Timing ablations (never in production builds; results are garbage when set):
//   2: no activation TMA (xfull arrives without data)   4: no weight bulk copies (wfull arrives)
//   8: dequant skips the ALU expansion   16: dequant skips the TMEM stores
#ifndef QOQ_ABLATE
#define QOQ_ABLATE 0
#endif

namespace qoq {

// Warp roles: 0 weight producer, 1 MMA issuer 0 + TMEM owner, 2 .. 2+4G-1 dequant (G groups of 4
// warps taking steps round-robin), then 4 epilogue warps, MMA issuer 1, activation producer.
template <int G>
struct Roles {
    static constexpr int kDeqGroups = G;
    static constexpr int kDeqWarp1 = 2 + 4 * G;          // first warp after the dequant warps
    static constexpr int kEpiWarp0 = kDeqWarp1;          // epilogue: 4 warps
    static constexpr int kMma1Warp = kEpiWarp0 + 4;      // MMA issuer 1
    static constexpr int kXProdWarp = kMma1Warp + 1;     // activation producer
    static constexpr int kBlockThreads = 32 * (kXProdWarp + 1);
    static constexpr int kEpiThread0 = 32 * kEpiWarp0;   // first epilogue thread
};

// Expand one 128-weight row of a packed tile (4 x 16 B = 128 u4 codes) into 32 TMEM words of
// four 8-bit lanes each: lane = q_u4 * s_u8 + (128 - z*s_u8) = q̂ + 128 ∈ [7, 254] (no cross-lane
// carry: the protective range bounds q̂ to [-121, 126]). SIGNED additionally flips the
// lane MSBs (XOR 0x80) to give q̂ as s8. Per 8 weights: 2 LOP3 (ALU pipe) + IMAD.HI (the >> 4, on
// the FMA pipe) + 2 IMAD (FMA pipe) [+ 2 LOP3], balancing the two integer pipes.
template <bool SIGNED>
__device__ __forceinline__ void expand_row(const uint4 (&v)[4], uint32_t s, uint32_t bias, uint32_t (&out)[32]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint32_t wd[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t lo = wd[i] & 0x0F0F0F0Fu;                      // k = 32c + 4i .. +3
            const uint32_t hi = __umulhi(wd[i], 0x10000000u) & 0x0F0F0F0Fu;   // (w >> 4): k = 32c + 16 + 4i ..
            uint32_t a = lo * s + bias, b = hi * s + bias;
            if (SIGNED) { a ^= 0x80808080u; b ^= 0x80808080u; }
            out[c * 8 + i] = (QOQ_ABLATE & 8) ? wd[i] : a;
            out[c * 8 + 4 + i] = (QOQ_ABLATE & 8) ? wd[i] : b;
        }
    }
}

// kChunk TMEM columns of this warp's 32 lanes (32 or 16).
template <int kChunk>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&v)[kChunk]) {
    if constexpr (kChunk == 32) tmem_ld_32x32b_x32(taddr, v);
    else tmem_ld_32x32b_x16(taddr, v);
}

// Zero this warp's 32 TMEM lanes of a BN-column accumulator (tcgen05.st, then wait::st).
template <int BN>
__device__ __forceinline__ void zero_acc(uint32_t taddr) {
    if constexpr (BN >= 32) {
        const uint32_t z[32] = {0};
#pragma unroll
        for (int c = 0; c < BN; c += 32) tmem_st_32x32b_x32(taddr + c, z);
    } else {
        const uint32_t z[16] = {0};
        tmem_st_32x32b_x16(taddr, z);
    }
    tmem_wait_st();
}

}  // namespace qoq
