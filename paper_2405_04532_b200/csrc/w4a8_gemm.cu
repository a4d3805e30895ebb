// w4a8_gemm.cu — QoQ W4A8 per-group GEMM with progressive dequantization on sm_100a.
//
// Computes (swap-AB orientation: weights are the MMA "M" operand, tokens the "N" operand)
//     acc[n][m] = Σ_k q̂[n][k] · q_x[m][k],   q̂ = (q_u4 − z)·s_u8 ∈ INT8
//     Y[m][n]   = fp16( acc · s_x[m] · s0[n] )
//
// Paper design (A100/L40S, §5.2) -> B200 design:
//  * "multi-stage software pipelining and asynchronous memory copy" -> a persistent,
//    warp-specialized kernel: one producer warp streams each contiguous 8448-byte packed weight
//    tile with cp.async.bulk and the matching 128-wide INT8 activation tile with a TMA tensor map
//    (SWIZZLE_128B) into an mbarrier ring.
//  * "UINT4 to UINT8 ... with only three logical operations" + "subtraction after multiplication"
//    with register-level parallelism -> one 4-warp dequant group; per 4 weights:
//    AND (+SHR), then ONE 32-bit IMAD  w·s_u8 + (128 − z·s_u8)·0x01010101, which yields the four
//    lanes q̂+128 ∈ [7, 254] with no cross-lane carry — valid ONLY because the protective range
//    keeps q̂ ∈ [−121, 126]. With t_x available the MMA consumes these as UNSIGNED
//    8-bit weights and the epilogue subtracts 128·t_x[m]; otherwise an XOR 0x80808080 maps them to
//    signed INT8. The expanded tile goes straight to tensor memory (tcgen05.st), never to SMEM.
//  * INT8 tensor-core MMA "as if it was W8A8" -> tcgen05.mma.kind::i8, A from TMEM,
//    B (activations) from SMEM, D = 128 x BN INT32 accumulators in TMEM, issued by one thread.
//  * Split-K "when the number of input tokens (m) is small" -> stream-K style contiguous
//    k-ranges per CTA; partial INT32 tiles are reduced exactly in a global workspace, and the last
//    CTA to arrive on a tile applies the epilogue.
//  * Epilogue: tcgen05.ld -> (− 128·t_x) -> × s_x[m]·s0[n] -> fp16 stores.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "qoq_internal.h"
#include "sm100_ptx.cuh"

namespace qoq {

constexpr int kThreads = 384;       // warps: 0 producer, 1 MMA + TMEM owner, 2-3 idle, 4-7 dequant, 8-11 epilogue
constexpr int kAStages = 4;         // TMEM buffers for expanded weight tiles (32 columns each)

template <int BN>
struct Cfg {
    static constexpr int kActBytes = BN * 128;
    static constexpr int kStageBytes = ((kActBytes + kTileBytes + 1023) / 1024) * 1024;
    static constexpr int kStagesRaw = (200 * 1024) / kStageBytes;
    static constexpr int kStages = kStagesRaw > 16 ? 16 : kStagesRaw;
    static constexpr int kAccStages = BN <= 128 ? 2 : 1;
    static constexpr int kColsUsed = kAStages * 32 + kAccStages * BN;
    static constexpr int kTmemCols = kColsUsed <= 32 ? 32 : kColsUsed <= 64 ? 64 : kColsUsed <= 128 ? 128
                                   : kColsUsed <= 256 ? 256 : 512;
    static constexpr int kBarBytes = 8 * (2 * kStages + 2 * kAStages + 2 * kAccStages) + 16;
    static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kBarBytes;
    static constexpr int kChunk = BN < 32 ? BN : 32;   // TMEM columns per epilogue tcgen05.ld
    static_assert(kColsUsed <= 512, "TMEM overflow");
    static_assert(kSmemBytes <= 227 * 1024, "SMEM overflow");
};

struct KParams {
    const uint8_t* packed;
    const __half* s0;
    const __half* sx;
    const int32_t* tx;
    void* out;
    int ldo;
    int32_t* ws;
    int* counters;
    int M, MT, KT, T, G, mode;
    long long I;
};

// Iterates the (tile, k0, k1) segments one CTA owns. Every role runs an identical copy.
struct SegIter {
    long long cur, end;
    int b, G, KT, T, mode;
    __device__ SegIter(const KParams& p) : b(blockIdx.x), G(p.G), KT(p.KT), T(p.T), mode(p.mode) {
        if (mode == 0) {
            cur = 0;
            end = 0;
        } else {
            cur = (long long)b * p.I / p.G;
            end = (long long)(b + 1) * p.I / p.G;
        }
    }
    __device__ bool next(int& tile, int& k0, int& k1) {
        if (mode == 0) {
            const long long t = b + cur * G;
            if (t >= T) return false;
            tile = (int)t;
            k0 = 0;
            k1 = KT;
            ++cur;
            return true;
        }
        if (cur >= end) return false;
        tile = (int)(cur / KT);
        k0 = (int)(cur % KT);
        const long long rem = end - cur;
        k1 = (int)((long long)k0 + rem < KT ? k0 + rem : KT);
        cur += k1 - k0;
        return true;
    }
};

template <int BN, bool OUT_I32>
__device__ __forceinline__ void store_out(const KParams& p, int m, int n, int32_t a, float s0f) {
    if constexpr (OUT_I32) {
        static_cast<int32_t*>(p.out)[(size_t)m * p.ldo + n] = a;
    } else {
        const float sxf = __half2float(__ldg(p.sx + m));
        static_cast<__half*>(p.out)[(size_t)m * p.ldo + n] = __float2half_rn((float)a * (sxf * s0f));
    }
}

template <int BN, bool OUT_I32>
__global__ void __launch_bounds__(kThreads, 1)
    w4a8_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const KParams p) {
    using C = Cfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* afull = empty + C::kStages;
    uint64_t* aempty = afull + kAStages;
    uint64_t* accfull = aempty + kAStages;
    uint64_t* accempty = accfull + C::kAccStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + C::kAccStages);
    volatile int* fin_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < C::kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 4 + 1);   // 4 dequant warps + 1 MMA commit
        }
        for (int i = 0; i < kAStages; ++i) {
            mbar_init(&afull[i], 4);
            mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < C::kAccStages; ++i) {
            mbar_init(&accfull[i], 1);
            mbar_init(&accempty[i], 4);
        }
        fence_mbar_init();
        prefetch_tmap(&tmap_x);
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    pdl_wait();   // inputs produced by the previous kernel in the stream are visible from here on

    if (warp == 0) {
        // ===================== producer: TMA activations + bulk-copy packed weights
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();   // each weight byte is read once
            SegIter si(p);
            int tile, k0, k1, stage = 0;
            uint32_t phase = 0;
            while (si.next(tile, k0, k1)) {
                const int nt = tile / p.MT, mt = tile % p.MT;
                for (int kt = k0; kt < k1; ++kt) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* st = smem + stage * C::kStageBytes;
                    mbar_arrive_expect_tx(&full[stage], C::kActBytes + kTileBytes);
                    tma_load_2d(st, &tmap_x, kt * 128, mt * BN, &full[stage]);
                    bulk_g2s(st + C::kActBytes, p.packed + ((size_t)nt * p.KT + kt) * kTileBytes, kTileBytes,
                             &full[stage], pol);
                    if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (single thread)
        if (lane == 0) {
            const uint32_t idesc = idesc_i8(128, BN, /*a_signed=*/p.tx == nullptr);
            SegIter si(p);
            int tile, k0, k1, stage = 0, ast = 0, cst = 0;
            uint32_t phase = 0, aph = 0, cph = 0;
            while (si.next(tile, k0, k1)) {
                mbar_wait(&accempty[cst], cph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + kAStages * 32 + cst * BN;
                for (int kt = k0; kt < k1; ++kt) {
                    mbar_wait(&full[stage], phase);
                    mbar_wait(&afull[ast], aph);
                    tc_fence_after();
                    const uint32_t a = tmem + ast * 32;
                    const uint32_t sb = smem_u32(smem + stage * C::kStageBytes);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_i8_ts(d, a + kk * 8, smem_desc_sw128(sb + kk * 32), idesc, (kt > k0 || kk > 0) ? 1u : 0u);
                    tc_commit(&empty[stage]);    // activation tile consumed
                    tc_commit(&aempty[ast]);     // expanded weight buffer consumed
                    if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                    if (++ast == kAStages) { ast = 0; aph ^= 1; }
                }
                tc_commit(&accfull[cst]);        // accumulator tile complete
                if (++cst == C::kAccStages) { cst = 0; cph ^= 1; }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ===================== dequant: u4 -> (q̂ + 128) lanes -> TMEM A buffer
        const int q = warp - 4;                       // TMEM lane quarter this warp may access
        const int r = q * 32 + lane;                  // weight row within the tile
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t flip = (p.tx == nullptr) ? 0x80808080u : 0u;
        SegIter si(p);
        int tile, k0, k1, stage = 0, ast = 0;
        uint32_t phase = 0, aph = 0;
        while (si.next(tile, k0, k1)) {
            for (int kt = k0; kt < k1; ++kt) {
                mbar_wait(&full[stage], phase);
                const uint8_t* w = smem + stage * C::kStageBytes + C::kActBytes;
                const uint32_t s = w[8192 + r];
                const uint32_t bias = (128u - (uint32_t)w[8320 + r]) * 0x01010101u;
                uint4 v[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) v[c] = *reinterpret_cast<const uint4*>(w + c * 2048 + r * 16);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);   // packed bytes now live in registers
                uint32_t out[32];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t wd[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t lo = wd[i] & 0x0F0F0F0Fu;          // k = 32c + 4i .. +3
                        const uint32_t hi = (wd[i] >> 4) & 0x0F0F0F0Fu;   // k = 32c + 16 + 4i .. +3
                        out[c * 8 + i] = (lo * s + bias) ^ flip;
                        out[c * 8 + 4 + i] = (hi * s + bias) ^ flip;
                    }
                }
                mbar_wait(&aempty[ast], aph ^ 1);
                tc_fence_after();
                tmem_st_32x32b_x32(tmem + lane_off + ast * 32, out);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&afull[ast]);
                if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                if (++ast == kAStages) { ast = 0; aph ^= 1; }
            }
        }
    } else if (warp >= 8) {
        // ===================== epilogue
        const int q = warp - 8;
        const int r = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        SegIter si(p);
        int tile, k0, k1, cst = 0;
        uint32_t cph = 0;
        while (si.next(tile, k0, k1)) {
            const int nt = tile / p.MT, mt = tile % p.MT;
            const int n = nt * 128 + r;
            const int m0 = mt * BN;
            const bool whole = (k0 == 0 && k1 == p.KT);
            const float s0f = OUT_I32 ? 0.0f : __half2float(__ldg(p.s0 + n));
            int32_t* wst = p.ws + (size_t)tile * 128 * BN;
            mbar_wait(&accfull[cst], cph);
            tc_fence_after();
            const uint32_t d = tmem + lane_off + kAStages * 32 + cst * BN;
#pragma unroll 1
            for (int j0 = 0; j0 < BN; j0 += C::kChunk) {
                uint32_t v[C::kChunk];
                if constexpr (C::kChunk == 32) tmem_ld_32x32b_x32(d + j0, v);
                else tmem_ld_32x32b_x16(d + j0, v);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < C::kChunk; ++i) {
                    const int m = m0 + j0 + i;
                    if (m < p.M) {
                        int32_t a = (int32_t)v[i];
                        if (whole) {
                            if (p.tx) a -= 128 * __ldg(p.tx + m);
                            store_out<BN, OUT_I32>(p, m, n, a, s0f);
                        } else {
                            atomicAdd(wst + (size_t)(j0 + i) * 128 + r, a);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[cst]);
            if (++cst == C::kAccStages) { cst = 0; cph ^= 1; }
            if (!whole) {
                __threadfence();
                named_bar_sync(1, 128);
                if (r == 0) {
                    const int prev = atomicAdd(p.counters + tile, k1 - k0);
                    *fin_flag = (prev + (k1 - k0) == p.KT) ? 1 : 0;
                }
                named_bar_sync(1, 128);
                if (*fin_flag) {   // last contributor: finish the tile and restore the zero workspace
                    __threadfence();
                    for (int j = 0; j < BN; ++j) {
                        const int m = m0 + j;
                        if (m < p.M) {
                            int32_t a = __ldcg(wst + (size_t)j * 128 + r);
                            wst[(size_t)j * 128 + r] = 0;
                            if (p.tx) a -= 128 * __ldg(p.tx + m);
                            store_out<BN, OUT_I32>(p, m, n, a, s0f);
                        }
                    }
                    if (r == 0) p.counters[tile] = 0;
                }
                named_bar_sync(1, 128);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    pdl_launch_dependents();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, C::kTmemCols);
    }
}

// ------------------------------------------------------------------ host side

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;   // resolved once; immutable after
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

GemmPlan plan_gemm(int M, int N, int K, int num_sms) {
    GemmPlan p{};
    p.BN = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256;
    p.MT = (M + p.BN - 1) / p.BN;
    p.NT = N / kTileN;
    p.KT = K / kTileK;
    p.T = p.MT * p.NT;
    p.I = (long long)p.T * p.KT;
    if (p.T >= num_sms) {
        p.mode = 0;
        p.G = num_sms;
        p.ws_bytes = 0;
    } else {
        p.mode = 1;
        p.G = (int)(p.I < num_sms ? p.I : num_sms);
        p.ws_bytes = (size_t)p.T * 128 * p.BN * 4 + (size_t)p.T * 4;
    }
    return p;
}

template <int BN, bool OUT_I32>
static cudaError_t launch_bn(const GemmArgs& a, const GemmPlan& pl, cudaStream_t st, bool pdl) {
    using C = Cfg<BN>;
    auto kern = w4a8_gemm_kernel<BN, OUT_I32>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    auto enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.M};
    cuuint64_t strides[1] = {(cuuint64_t)a.K};
    cuuint32_t box[2] = {128u, (cuuint32_t)BN};
    cuuint32_t estr[2] = {1u, 1u};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(a.qx), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    KParams kp{};
    kp.packed = static_cast<const uint8_t*>(a.packed);
    kp.s0 = static_cast<const __half*>(a.s0);
    kp.sx = static_cast<const __half*>(a.sx);
    kp.tx = a.tx;
    kp.out = a.out;
    kp.ldo = a.ldo;
    kp.ws = static_cast<int32_t*>(a.ws);
    kp.counters = a.ws ? reinterpret_cast<int*>(static_cast<uint8_t*>(a.ws) + (size_t)pl.T * 128 * BN * 4) : nullptr;
    kp.M = a.M;
    kp.MT = pl.MT;
    kp.KT = pl.KT;
    kp.T = pl.T;
    kp.G = pl.G;
    kp.mode = pl.mode;
    kp.I = pl.I;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, tm, kp);
}

cudaError_t launch_w4a8_gemm(const GemmArgs& a, const GemmPlan& p, cudaStream_t st, bool pdl) {
    switch (p.BN) {
        case 16: return a.out_i32 ? launch_bn<16, true>(a, p, st, pdl) : launch_bn<16, false>(a, p, st, pdl);
        case 32: return a.out_i32 ? launch_bn<32, true>(a, p, st, pdl) : launch_bn<32, false>(a, p, st, pdl);
        case 64: return a.out_i32 ? launch_bn<64, true>(a, p, st, pdl) : launch_bn<64, false>(a, p, st, pdl);
        case 128: return a.out_i32 ? launch_bn<128, true>(a, p, st, pdl) : launch_bn<128, false>(a, p, st, pdl);
        case 256: return a.out_i32 ? launch_bn<256, true>(a, p, st, pdl) : launch_bn<256, false>(a, p, st, pdl);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qoq
