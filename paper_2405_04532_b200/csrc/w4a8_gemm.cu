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
#include <cstdlib>

#include "qoq_internal.h"
#include "sm100_ptx.cuh"
#include "qoq_quant.cuh"
#include "w4a8_common.cuh"

namespace qoq {

#ifndef QOQ_DEQ_GROUPS
#define QOQ_DEQ_GROUPS 3
#endif

// One pipeline STEP = up to two consecutive 128-deep k-tiles of one output tile: the handoff
// (dequant -> MMA, MMA -> producer) is amortized over 8 MMAs, and two MMA-issuing warps take
// alternate steps of a segment into separate accumulators (summed in the epilogue). Measured on
// B200 (tools/mma_bench2.cu): one issuer, one tile per handoff ~520 cycles per 128x128 tile; two
// issuers, two tiles per handoff ~193 cycles (MMA floor at N <= 64: 4 x 45 cycles).
// CG = 1: one CTA owns a 128-row weight tile (tcgen05 cta_group::1, MMA M = 128).
// CG = 2: a CTA pair (cluster of 2) owns two 128-row tiles; each CTA expands its own tile into its
// own TMEM and holds half of the activation rows; the leader issues cta_group::2 MMAs (M = 256) —
// half the MMA instructions, handoffs and activation SMEM traffic per SM (tools/cta2_check.cu:
// 32 cycles per 256x64x32 MMA vs 45.5 per 128x64x32 on one SM).
// PC = true: per-channel W4A8 (NEXT-1, §5.2.2): 8192-byte code tiles, no level-2 parameters; the
// dequant only unpacks (lanes = q_u4, fed as UNSIGNED 8-bit A) and the epilogue applies the zero
// point after the multiplication: Y = s_x s_w (acc - z_w t_x).
template <int BN, int CG = 1, bool PC = false, bool TP = false>
struct Cfg {
    static constexpr int kTB = PC ? kPcTileBytes : kTileBytes;        // bytes of one packed 128x128 tile
    // dequant groups: QOQ_DEQ_GROUPS (default 3; measured +1..9% over 2 at decode) where the TMEM budget allows a rotation-compatible
    // A ring, else 2. TP (fused reduction, short K shards): 2, so the 448-thread CTA has 144 registers for the
    // reduction's loads in flight (3 groups = 640 threads at the 96-register cap)
    static constexpr int kDeqGroups = (BN <= 64 && !TP) ? QOQ_DEQ_GROUPS : 2;
    using R = Roles<kDeqGroups>;
    static constexpr int kBlockThreads = R::kBlockThreads;
#ifndef QOQ_ISSUERS_BIG
#define QOQ_ISSUERS_BIG 2
#endif
    static constexpr int kIssuers = BN <= 128 ? 2 : QOQ_ISSUERS_BIG;
    static constexpr int kActRows = BN / CG;                          // activation rows held by this CTA
    static constexpr int kActBytes = kActRows * 128;                  // one k-tile of this CTA's activations
    static constexpr int kXStageBytes = 2 * kActBytes;                // activations of one step (1024-aligned)
#ifndef QOQ_CHUNK
#define QOQ_CHUNK 32
#endif
    static constexpr int kChunk = BN < QOQ_CHUNK ? BN : QOQ_CHUNK;    // TMEM columns per epilogue tcgen05.ld
    static constexpr int kStgBytes = kChunk * 128 * 4;                // one INT32 staging buffer [kChunk][128]
    static constexpr int kEpiBytes = 2 * kStgBytes + BN * 8;          // 2 staging buffers + per-token s_x, 128 t_x
    // QOQ_DEQ_SPLIT=1 (BN >= 128): the dequant groups split each step (group g expands k-tile g of
    // every step) instead of taking alternate steps. Measured on B200 prefill: 1-3% slower (the
    // step is bound by shared-memory bandwidth, not dequant latency), so off by default.
#ifndef QOQ_DEQ_SPLIT
#define QOQ_DEQ_SPLIT 0
#endif
    static constexpr bool kDeqSplit = QOQ_DEQ_SPLIT && BN >= 128 && kDeqGroups == 2;
    static constexpr int kDeqRot = kDeqSplit ? 1 : kDeqGroups;                // dequant roles per ring slot
    static constexpr int kARot = kDeqRot % 2 == 0 ? kDeqRot : 2 * kDeqRot;   // lcm(2 issuers, dequant roles)
    // two accumulator stages if they leave room for at least one A-ring rotation (2 x 64 columns
    // per rotation unit), else one
    // Both MMA issuers accumulate into ONE accumulator per stage (the tensor pipe applies their
    // MMAs in order; integer sums are order-free), pre-zeroed by the epilogue warps, so the
    // epilogue reads BN columns, not 2 BN (tcgen05.ld is ~64 B/cycle/SM: the epilogue's bound).
    // (BN = 192: 2 x 192 accumulator columns + a 2-step A ring fill TMEM exactly, so the epilogue of
    // one prefill tile overlaps the next tile's mainloop)
    static constexpr int kAccStages =
        ((512 - 2 * BN) / 64 >= (BN > 128 ? kARot : kARot > 4 ? kARot : 4)) ? 2 : 1;
    static constexpr int kAccCols = kAccStages * BN;
    // Three independent rings: W (packed weights, HBM-latency bound, SMEM), X (activation k-tiles,
    // L2-latency bound, SMEM) and A (expanded weights, 64 TMEM columns per step). (Loading weights
    // straight from L2 into registers after a bulk L2 prefetch was measured slower on B200: the
    // register loads stall at HBM latency with too few bytes in flight per SM.)
    // Ring depths are multiples of the number of roles that take turns on them (dequant groups on
    // W and A, the two MMA issuers on A and X), so every slot is always consumed by the same role
    // and no waiter can run two mbarrier phases ahead (parity waits would alias).
    static constexpr int kARaw0 = (512 - kAccCols) / 64;
    static constexpr int kARaw = kARaw0 > 6 ? 6 : kARaw0;
    static constexpr int kAStages = (kARaw / kARot) * kARot;
#ifndef QOQ_XSTAGES64
#define QOQ_XSTAGES64 6
#endif
#ifndef QOQ_SMEM_KB
#define QOQ_SMEM_KB 212
#endif
    static constexpr int kXStagesDef = BN <= 32 ? (kDeqGroups == 3 ? 6 : 8) : BN == 64 ? QOQ_XSTAGES64 : 2;
#ifndef QOQ_XSTAGES
    static constexpr int kXStages = kXStagesDef;
#else
    static constexpr int kXStages = (BN <= 64 && CG == 1) ? QOQ_XSTAGES : kXStagesDef;
#endif
    static constexpr int kWStageBytes = ((2 * kTB + 1023) / 1024) * 1024;   // packed weights of one step
    static constexpr int kWRaw = (QOQ_SMEM_KB * 1024 - kEpiBytes - kXStages * kXStageBytes) / kWStageBytes;
    static constexpr int kWCap = kWRaw > 12 ? 12 : kWRaw;
    static constexpr int kWStages = (kWCap / kDeqRot) * kDeqRot;
    static constexpr int kColsUsed = kAStages * 64 + kAccCols;
    static constexpr int kTmemCols = kColsUsed <= 32 ? 32 : kColsUsed <= 64 ? 64 : kColsUsed <= 128 ? 128
                                   : kColsUsed <= 256 ? 256 : 512;
    static constexpr int kXOff = 0;
    static constexpr int kWOff = kXStages * kXStageBytes;
    static constexpr int kEpiOff = kWOff + kWStages * kWStageBytes;
    static constexpr int kBarOff = kEpiOff + kEpiBytes;
    static constexpr int kBarBytes = 8 * (2 * kWStages + 2 * kXStages + 2 * kAStages + 2 * kAccStages + 1) + 16;
    static constexpr int kSmemBytes = 1024 + kBarOff + kBarBytes;
    static constexpr int kFinU = BN / 4 < 8 ? BN / 4 : 8;             // independent 16-B loads per finalize batch
    static_assert(kXStages >= 2 && kWStages >= 2 && kAStages >= 2, "pipeline too shallow");
    static_assert(kXStages % kIssuers == 0 && kWStages % kDeqRot == 0 && kAStages % kARot == 0, "ring rotation");
    static_assert(CG == 1 || kXStages % kDeqRot == 0, "ring rotation (pairs: dequant groups wait on X)");
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
    int M, MT, KT, KS, T, G, mode, S;   // mode 2: S-CTA clusters split one tile's K range
    int MB;                      // token tiles per band of the work order (tile_coords)
    long long I;                 // total steps = T * KS
    unsigned long long* trace;   // debug: per-CTA %globaltimer stamps (nullptr in production)
    // fused per-token activation quantization (qoq_w4a8_linear, M <= 64): X != nullptr. The
    // epilogue warps quantize rows m = blockIdx.x (mod gridDim.x) of X into q_x / s_x / t_x (the
    // buffers qx/sx/tx above point to), then a grid handshake on qsync releases the q_x TMA loads.
    const __half* X;
    int8_t* qx_rows;             // q_x [M][K] (the tensor map's global buffer)
    int ldx, K;
    int* qsync;                  // [2] arrivals / departures; the last departure re-zeroes both
    const uint8_t* zw;           // per-channel W4A8: z_w [N] (else nullptr)
    TpComm tp;                   // fused TP reduction (NEXT-3, the TP instantiation): whole tiles, CG = 1, fp16 out
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#ifndef QOQ_PDL_EARLY
#define QOQ_PDL_EARLY 0
#endif
#ifndef QOQ_W_L2_PREFETCH
#define QOQ_W_L2_PREFETCH 0   // bulk L2 prefetch of each decode segment's weights (A/B knob)
#endif
#ifndef QOQ_EXPAND_EARLY
#define QOQ_EXPAND_EARLY 1   // token tiles > 64: expand a step before waiting for its TMEM buffer (+1-1.5% prefill)
#endif
#ifndef QOQ_W_PREFILL
#define QOQ_W_PREFILL 1   // W-ring stages issued before the setup barrier (each issue costs ~250 cycles)
#endif
// trace buffer layout (u64): [148 CTAs][kTrEv] globaltimer | [64 it][8] CTA-0 step stamps |
// [16][8] CTA-0 per-MMA | [16][8] CTA-0 per-dequant-warp | [148][kTrEv] clock64
constexpr int kTrEv = 32;
constexpr int kTrIt = 148 * kTrEv;
constexpr int kTrMma = kTrIt + 64 * 8;
constexpr int kTrDq = kTrMma + 16 * 8;
constexpr int kTraceCyc = kTrDq + 16 * 8;
#ifndef QOQ_TRACING
#define QOQ_TRACING 0   // the `trace` library variant (tools/trace_gemm.py) compiles the stamps in
#endif
#if QOQ_TRACING
// per-CTA events: globaltimer (comparable across SMs) + clock64 (cycle-accurate within the CTA)
#define QOQ_TRACE(p, ev) \
    do { if ((p).trace) { (p).trace[blockIdx.x * kTrEv + (ev)] = gtimer(); \
                          (p).trace[kTraceCyc + blockIdx.x * kTrEv + (ev)] = clock64(); } } while (0)

// per-iteration stamps of CTA 0 use the SM cycle counter (clock64), cycle-accurate within the SM
#define QOQ_TRACE_IT(p, it, ev) \
    do { if ((p).trace && blockIdx.x == 0 && (it) < 64) (p).trace[kTrIt + (it) * 8 + (ev)] = clock64(); } while (0)
#else
#define QOQ_TRACE(p, ev) do { } while (0)
#define QOQ_TRACE_IT(p, it, ev) do { } while (0)
#endif

// Work unit t -> (n unit, token tile). Band-major: bands of MB token tiles; inside a band the n unit
// is major and the token tile minor, so the CTAs of one wave share each weight tile (L2) and keep
// re-reading one band of activations (MB x BN x K bytes, sized to stay in L2) instead of all of
// them — long-K prefill (down_proj) would otherwise re-stream q_x from HBM every wave. MB = MT is
// the plain token-tile-minor order (decode: MT = 1).
__device__ __forceinline__ void tile_coords(const KParams& p, int t, int& nu, int& mt) {
    const int nun = p.T / p.MT;                  // n units (128-row tiles, or tile pairs for CG = 2)
    const int band = t / (p.MB * nun), r = t - band * (p.MB * nun);
    const int mb = min(p.MB, p.MT - band * p.MB);
    nu = r / mb;
    mt = band * p.MB + (r - nu * mb);
}

// Iterates the (tile, s0, s1) segments (ranges of steps of one output tile) a CTA owns.
// Every role runs an identical copy.
struct SegIter {
    long long cur, end;
    int b, G, KS, T, mode;
    __device__ SegIter(const KParams& p, int cg = 1) : b(blockIdx.x / cg), G(p.G), KS(p.KS), T(p.T), mode(p.mode) {
        if (mode == 0) {
            cur = 0;
            end = 0;
        } else if (mode == 2) {   // one segment: tile b / S, steps [c KS / S, (c+1) KS / S), c = rank in cluster
            const int c = b % p.S, tile = b / p.S;
            cur = (long long)tile * KS + (long long)c * KS / p.S;
            end = (long long)tile * KS + (long long)(c + 1) * KS / p.S;
        } else {
            cur = (long long)b * p.I / p.G;
            end = (long long)(b + 1) * p.I / p.G;
        }
    }
    __device__ bool more() const { return mode == 0 ? (b + cur * G) < T : cur < end; }
    __device__ bool next(int& tile, int& s0, int& s1) {
        if (mode == 0) {
            const long long t = b + cur * G;
            if (t >= T) return false;
            tile = (int)t;
            s0 = 0;
            s1 = KS;
            ++cur;
            return true;
        }
        if (cur >= end) return false;
        tile = (int)(cur / KS);
        s0 = (int)(cur % KS);
        const long long rem = end - cur;
        s1 = (int)((long long)s0 + rem < KS ? s0 + rem : KS);
        cur += s1 - s0;
        return true;
    }
};

// Weight producer state (warp 0, lane 0): walks the CTA's segments step by step; issue() waits for the
// ring slot, then bulk-copies the step's 1-2 packed tiles (contiguous in the tile stream). Resumable,
// so the first ring's worth can be issued before the setup barrier.
template <class C>
struct WProducer {
    SegIter si;
    int nt = 0, sg = 0, s1 = 0, ws = 0, rank, cg;
    uint32_t wph = 0;
    bool live;
    uint64_t pol;
    __device__ WProducer(const KParams& p, int cg_, int rank_) : si(p, cg_), rank(rank_), cg(cg_) {
        int tile, s0;
        live = si.next(tile, s0, s1);
        sg = s0;
        int nu = 0, mt;
        if (live) tile_coords(p, tile, nu, mt);
        nt = nu * cg + rank;
        pol = policy_evict_first();   // each weight byte is read once
        if (live && threadIdx.x == 0) prefetch_segment(p, s0);   // the weight producer thread
    }
    // Decode (one token tile): ask L2 for the whole segment's packed weights up front, so the HBM reads run
    // at full parallelism and the SMEM ring's bulk copies hit L2 (one SM pulls only ~27 B/cycle from HBM
    // through its own copies; a 32-tile o_proj would otherwise stream at 32 SMs' ingress).
    __device__ void prefetch_segment(const KParams& p, int s0) {
#if QOQ_W_L2_PREFETCH
        if (p.MT != 1) return;
        const uint8_t* a = p.packed + ((size_t)nt * p.KT + 2 * s0) * C::kTB;
        const uint8_t* e = p.packed + ((size_t)nt * p.KT + (2 * s1 < p.KT ? 2 * s1 : p.KT)) * C::kTB;
        for (; a < e; a += 65536) prefetch_l2_bulk(a, (uint32_t)((e - a) < 65536 ? (e - a) : 65536));
#endif
    }
    __device__ bool issue(const KParams& p, uint8_t* smem, uint64_t* wfull, uint64_t* wfree) {
        if (!live) return false;
        const int kt0 = 2 * sg, nk = (kt0 + 1 < p.KT) ? 2 : 1;
        mbar_wait(&wfree[ws], wph ^ 1);
        uint8_t* dst = smem + C::kWOff + ws * C::kWStageBytes;
        if (QOQ_ABLATE & 4) {
            mbar_arrive(&wfull[ws]);
        } else {
            mbar_arrive_expect_tx(&wfull[ws], nk * C::kTB);
            bulk_g2s(dst, p.packed + ((size_t)nt * p.KT + kt0) * C::kTB, nk * C::kTB, &wfull[ws], pol);
        }
        if (++ws == C::kWStages) { ws = 0; wph ^= 1; }
        if (++sg == s1) {
            int tile, s0;
            live = si.next(tile, s0, s1);
            sg = s0;
            if (live) {
                int nu, mt;
                tile_coords(p, tile, nu, mt);
                nt = nu * cg + rank;
                prefetch_segment(p, s0);
            }
        }
        return true;
    }
};

// The zero-point multipliers of four consecutive output rows: z_w[n..n+3] (per-channel), else 1
// (the g128 path's bias 128·t_x applies to every row alike).
template <bool PC>
__device__ __forceinline__ void load_z4(const KParams& p, int n, int (&zv)[4]) {
    if constexpr (PC) {
        const uint32_t u = __ldg(reinterpret_cast<const uint32_t*>(p.zw + n));
        zv[0] = u & 255; zv[1] = (u >> 8) & 255; zv[2] = (u >> 16) & 255; zv[3] = u >> 24;
    } else {
        zv[0] = zv[1] = zv[2] = zv[3] = 1;
    }
}

// Four consecutive outputs Y[m][n..n+3] (or acc) from four INT32 accumulators: acc - bias·zv, then
// the s_x s0 outer-product scaling (per-channel: bias = t_x, zv = z_w).
template <bool OUT_I32>
__device__ __forceinline__ void write_out4(const KParams& p, int m, int n, int4 a, int bias, float sxf,
                                           const float (&s0v)[4], const int (&zv)[4]) {
    a.x -= bias * zv[0]; a.y -= bias * zv[1]; a.z -= bias * zv[2]; a.w -= bias * zv[3];
    if constexpr (OUT_I32) {
        *reinterpret_cast<int4*>(static_cast<int32_t*>(p.out) + (size_t)m * p.ldo + n) = a;
    } else {
        __half2 lo = __halves2half2(__float2half_rn((float)a.x * (sxf * s0v[0])),
                                    __float2half_rn((float)a.y * (sxf * s0v[1])));
        __half2 hi = __halves2half2(__float2half_rn((float)a.z * (sxf * s0v[2])),
                                    __float2half_rn((float)a.w * (sxf * s0v[3])));
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(static_cast<__half*>(p.out) + (size_t)m * p.ldo + n) = u;
    }
}

// Fused per-token quantization by the 128 epilogue threads (et) of this CTA: rows m ≡ blockIdx.x
// (mod gridDim.x), same arithmetic as quantize_act_kernel (qoq_quant.cuh): amax with kQVec loads
// per thread in flight, then a compact quantize loop over the (L1-resident) row. red/redi: >= 4
// floats / ints of shared scratch. Ends with this CTA's arrival on qsync[0] (release).
constexpr int kQVec = 8;

__device__ __forceinline__ void quant_row_finish(const KParams& p, int m, int et, float* red, int* redi, float a,
                                                 float& sc, __half& sh) {
    const int g = et >> 5, l = et & 31;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (l == 0) red[g] = a;
    named_bar_sync(1, 128);
    a = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    sh = sym_scale(a, 127.0f);
    sc = __half2float(sh);
}

__device__ __forceinline__ void quant_row_sum(const KParams& p, int m, int et, int* redi, int t, __half sh) {
    const int g = et >> 5, l = et & 31;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) redi[g] = t;
    named_bar_sync(1, 128);
    if (et == 0) {
        const_cast<__half*>(p.sx)[m] = sh;
        const_cast<int32_t*>(p.tx)[m] = redi[0] + redi[1] + redi[2] + redi[3];
    }
}

__device__ __forceinline__ void fused_quantize_rows(const KParams& p, int et, float* red, int* redi) {
    const int nv = p.K / 8;
    for (int m = blockIdx.x; m < p.M; m += gridDim.x) {
        const uint4* row = reinterpret_cast<const uint4*>(p.X + (size_t)m * p.ldx);
        uint2* out = reinterpret_cast<uint2*>(p.qx_rows + (size_t)m * p.K);
        __half2 a2 = __float2half2_rn(0.0f);
        for (int i0 = 0; i0 < nv; i0 += 128 * kQVec) {   // kQVec loads per thread in flight
            uint4 v[kQVec];
#pragma unroll
            for (int j = 0; j < kQVec; ++j) {
                const int i = i0 + et + 128 * j;
                v[j] = (i < nv) ? __ldg(row + i) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int j = 0; j < kQVec; ++j) a2 = amax8h(v[j], a2);
        }
        if (et == 0 && m == (int)blockIdx.x) QOQ_TRACE(p, 16);
        float sc;
        __half sh;
        quant_row_finish(p, m, et, red, redi, amax_of(a2), sc, sh);
        if (et == 0 && m == (int)blockIdx.x) QOQ_TRACE(p, 17);
        const float inv = __frcp_rn(sc);
        int t = 0;
#pragma unroll 2
        for (int i = et; i < nv; i += 128) out[i] = quant8(__ldg(row + i), sc, inv, t);   // L1 re-read
        if (et == 0 && m == (int)blockIdx.x) QOQ_TRACE(p, 18);
        quant_row_sum(p, m, et, redi, t, sh);
        if (et == 0 && m == (int)blockIdx.x) QOQ_TRACE(p, 19);
    }
    named_bar_sync(1, 128);   // all rows of this CTA written (CTA-scope), then one cumulative release
    if (et == 0) {
        QOQ_TRACE(p, 20);
        red_release_add_gpu(p.qsync, 1);   // cumulative through the CTA barrier above
        QOQ_TRACE(p, 21);
    }
}

// A consumer of the fused q_x is past the grid handshake: count it; the last of the 2 per CTA
// (activation producer + epilogue) re-zeroes the counters for the next launch.
__device__ __forceinline__ void fused_depart(const KParams& p) {
    if (atomicAdd(p.qsync + 1, 1) == 2 * (int)gridDim.x - 1) {
        atomicExch(p.qsync, 0);
        atomicExch(p.qsync + 1, 0);
    }
}

// ---------------------------------------------------------------- fused TP reduction (NEXT-3)
// Row-parallel layers (o, down) end in Y = Σ_r Y_r over the TP ranks (north_star). Instead of a separate
// all-reduce, each rank's epilogue PUSHES its fp16 partial of every whole tile into slot `rank` of every
// rank's receive buffer (peer stores over NVLink; the buffers are symmetric allocations) and then reduces
// its own slots 0 .. world-1 in rank order in fp32, rounding once to fp16 (reading Q32: deterministic,
// identical bits on every rank). The slots are in a flag-in-data format: every 8-byte word carries two
// fp16 values and the call's flag (gen + 1), written by ONE 16-byte relaxed system-scope store per four
// outputs, so a reader knows a word has landed by its flag alone — no fence, no counter, no barrier (a
// release fence costs microseconds on an SM with memory in flight). The buffers alternate by call parity:
// a rank can be at most one call ahead of a peer (it needs the peer's partials to finish a call), so the
// buffer it writes is never the one the peer still reads.
__device__ __forceinline__ size_t tp_word(const TpComm& c, int par, int slot, int m, int n) {
    // 8-byte words [2 parities][world slots][m_cap][n_cap / 2]; (m, n) with n % 4 == 0 -> words n/2, n/2 + 1
    return (((size_t)par * c.world + slot) * c.m_cap + m) * (c.n_cap / 2) + n / 2;
}
__device__ __forceinline__ void st_relaxed_sys_v4(void* p, uint4 v) {
    asm volatile("st.relaxed.sys.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 ld_relaxed_sys_v4(const void* p) {
    uint4 v;
    asm volatile("ld.relaxed.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p) : "memory");
    return v;
}
// Re-poll one 16-byte pair of words until both carry `flag`. Peers are other GPUs: a wait beyond 2 s (a peer
// not running the same call sequence) sets the status word and gives up instead of hanging the device.
__device__ __forceinline__ uint4 tp_poll(const TpComm& c, const void* w, uint32_t flag) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (uint32_t n = 1;; ++n) {
        const uint4 v = ld_relaxed_sys_v4(w);
        if (v.y == flag && v.w == flag) return v;
        if ((n & 255u) == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 2000000000ull) {
                atomicExch(c.status, 1);
                return make_uint4(0u, flag, 0u, flag);
            }
        }
        __nanosleep(20);
    }
}
__device__ __forceinline__ uint2 y4_bits(int4 a, int bias, float sxf, const float (&s0v)[4], const int (&zv)[4]) {
    a.x -= bias * zv[0]; a.y -= bias * zv[1]; a.z -= bias * zv[2]; a.w -= bias * zv[3];
    __half2 lo = __halves2half2(__float2half_rn((float)a.x * (sxf * s0v[0])), __float2half_rn((float)a.y * (sxf * s0v[1])));
    __half2 hi = __halves2half2(__float2half_rn((float)a.z * (sxf * s0v[2])), __float2half_rn((float)a.w * (sxf * s0v[3])));
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    return u;
}

template <int BN>
__device__ __forceinline__ void tmem_ld_chunk(uint32_t taddr, uint32_t (&v)[Cfg<BN, 1>::kChunk]) {
    tmem_ld_cols<Cfg<BN, 1>::kChunk>(taddr, v);
}

// TP = true: the fused TP reduction (NEXT-3) — its own instantiation, so the other kernels carry none of its
// registers (the BN <= 64 kernels run 640 threads at the 96-register cap)
// FQ = true: qoq_w4a8_linear's one-kernel path (per-token quantization in the prologue, QOQ_LINEAR_FUSED=1) —
// its own instantiation, so the production kernels carry none of its code
template <int BN, bool OUT_I32, int CG, bool PC = false, bool TP = false, bool FQ = false>
__global__ void __launch_bounds__(Cfg<BN, CG, PC, TP>::kBlockThreads, 1)
    w4a8_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const KParams p) {
    using C = Cfg<BN, CG, PC, TP>;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned base derived by pointer arithmetic on the __shared__ array, so the compiler keeps
    // the shared address space (LDS/STS, not generic LD/ST) for everything carved from it
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    int32_t* stg = reinterpret_cast<int32_t*>(smem + C::kEpiOff);   // [2][kChunk][128]
    float* sxs = reinterpret_cast<float*>(smem + C::kEpiOff + 2 * C::kStgBytes);
    int* txs = reinterpret_cast<int*>(sxs + BN);
    uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + C::kBarOff);   // weights of W stage landed
    uint64_t* wfree = wfull + C::kWStages;    // weights of W stage copied to registers (4 warps)
    uint64_t* xfull = wfree + C::kWStages;    // activations of X slot landed (TMA)
    uint64_t* xempty = xfull + C::kXStages;   // MMAs reading X slot complete (commit)
    uint64_t* afull = xempty + C::kXStages;   // expanded step in TMEM buffer a (4 dequant warps)
    uint64_t* aempty = afull + C::kAStages;   // MMAs reading TMEM buffer a complete (commit)
    uint64_t* accfull = aempty + C::kAStages; // both issuers committed the accumulator stage
    uint64_t* accempty = accfull + C::kAccStages;
    uint64_t* red_full = accempty + C::kAccStages;   // mode 2: all S partial slices reduced into stg
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_full + 1);
    volatile int* fin_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) QOQ_TRACE(p, 0);
    const bool clustered = (p.mode == 2);
    // mode 2 (reduce-scatter): cluster rank c owns rows [c*R, (c+1)*R) of the tile, R = 128 / S
    const int crank = clustered ? (int)cluster_ctarank() : 0;
    constexpr int kRP = BN + 4;                       // padded row pitch (ints) of a staged partial
    const int rank = (CG == 2) ? (int)cluster_ctarank() : 0;   // CTA-pair: which 128-row tile of the pair
    const bool epi_thread = threadIdx.x >= C::R::kEpiThread0 && threadIdx.x < C::R::kEpiThread0 + 128;
    if (clustered && epi_thread) {
        // mode 2: the (otherwise idle) epilogue warps zero this CTA's receive slice in the staging
        // area and arm red_full (one bulk reduce from every CTA of the cluster lands there), then
        // release them cluster-wide; only these threads pay for the cluster-scope fence.
        const int et = threadIdx.x - C::R::kEpiThread0;
        for (int i = et * 4; i < (128 / p.S) * kRP; i += 128 * 4)
            *reinterpret_cast<int4*>(stg + i) = make_int4(0, 0, 0, 0);
        if (et == 0) {
            mbar_init(red_full, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(red_full, (uint32_t)(128 * kRP * 4));
        }
        fence_proxy_async_smem();
        fence_acq_rel_cluster();
    }

    WProducer<C> wprod(p, CG, rank);
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < C::kWStages; ++i) {
            mbar_init(&wfull[i], 1);
            mbar_init(&wfree[i], 4 * (C::kDeqSplit ? C::kDeqGroups : 1));
        }
        for (int i = 0; i < C::kXStages; ++i) {
            mbar_init(&xfull[i], 1);
            mbar_init(&xempty[i], 1);
        }
        for (int i = 0; i < C::kAStages; ++i) {
            mbar_init(&afull[i], 4 * CG * (C::kDeqSplit ? C::kDeqGroups : 1));     // CG = 2: the peer's dequant warps arrive remotely on the leader's
            mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < C::kAccStages; ++i) {
            mbar_init(&accfull[i], C::kIssuers);
            mbar_init(&accempty[i], 4 * CG);  // CG = 2: both CTAs' epilogues free the pair's accumulators
        }
        fence_mbar_init();
        prefetch_tmap(&tmap_x);
#if QOQ_W_PREFILL
        // The weight producer (this thread) fills the W ring right away: the first bytes' HBM latency
        // overlaps TMEM allocation and the setup barriers. The proxy fence makes the barrier inits
        // visible to the async proxy that signals complete_tx on them.
        fence_proxy_async_smem();
        for (int i = 0; i < QOQ_W_PREFILL && i < C::kWStages && wprod.issue(p, smem, wfull, wfree); ++i) {
        }
#endif
    }
    if (threadIdx.x == 0) QOQ_TRACE(p, 11);
    if (warp == 1) {
        if constexpr (CG == 2) {
            tmem_alloc2(tmem_slot, C::kTmemCols);
            tmem_relinquish2();
        } else {
            tmem_alloc(tmem_slot, C::kTmemCols);
            tmem_relinquish();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) QOQ_TRACE(p, 13);
    // mode 2: leader's zeroed target + armed red_full visible cluster-wide; CG = 2: the pair's
    // barriers initialized before any remote arrive
    // CG = 2: the pair's barriers initialized before any remote arrive (full barrier). Mode 2: only
    // arrive here; the first remote operation (the epilogue's reduce-scatter) waits for this phase,
    // which has long completed by then.
    if (CG == 2) cluster_sync_all();
    else if (clustered) cluster_arrive_relaxed();   // the writers released above
    bool cl_done = false;   // mode 2: this thread has waited phase 0 and arrived on phase 1
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) QOQ_TRACE(p, 1);
#if QOQ_PDL_EARLY
    // PDL: release the dependent grid now. Its CTAs can only become resident on SMs this grid leaves
    // free (one GEMM CTA fills an SM's shared memory), where they set up and stream their own static
    // weights; everything they read from this grid sits behind their griddepcontrol.wait, which
    // still waits for this grid's completion and memory flush.
    pdl_launch_dependents();
#endif

    // PDL: weights and scales are static, so the weight producer streams them without waiting for the
    // previous kernel; everything that reads what the previous kernel wrote (q_x via TMA, s_x, t_x,
    // the split-K workspace) sits behind griddepcontrol.wait.
    if (warp == 0) {
        // ===================== weight producer: the rest of the stream (the first ring's worth was
        // issued before the CTA-wide setup barrier, above). Weights are static, so it runs ahead of
        // griddepcontrol.wait (overlaps the previous kernel).
        if (lane == 0)
            while (wprod.issue(p, smem, wfull, wfree)) {
            }
    } else if (warp == C::R::kXProdWarp) {
        // ===================== activation producer: TMA 2-D (SWIZZLE_128B) k-tiles of q_x
        if (lane == 0) {
            pdl_wait();
            if constexpr (FQ) {   // fused quantization: every CTA's q_x rows written (acquire), then visible
                spin_until_ge(p.qsync, (int)gridDim.x);   // to this thread's async-proxy (TMA) reads
                fence_proxy_async_global();
                fused_depart(p);
            }
            QOQ_TRACE(p, 2);
            SegIter si(p, CG);
            int tile, s0, s1, xs = 0, it = 0;
            uint32_t xph = 0;
            while (si.next(tile, s0, s1)) {
                int nu, mt;
                tile_coords(p, tile, nu, mt);
                const int row0 = mt * BN + rank * C::kActRows;   // CG = 2: this CTA's half of the tokens
                for (int sg = s0; sg < s1; ++sg, ++it) {
                    const int kt0 = 2 * sg, nk = (kt0 + 1 < p.KT) ? 2 : 1;
                    mbar_wait(&xempty[xs], xph ^ 1);         // previous step of this slot consumed by the MMAs
                    QOQ_TRACE_IT(p, it, 7);
                    uint8_t* dst = smem + C::kXOff + xs * C::kXStageBytes;
                    if ((QOQ_ABLATE & 2) && it >= C::kXStages) {
                        mbar_arrive(&xfull[xs]);
                    } else {
                        mbar_arrive_expect_tx(&xfull[xs], nk * C::kActBytes);
                        for (int t = 0; t < nk; ++t)
                            tma_load_2d(dst + t * C::kActBytes, &tmap_x, (kt0 + t) * 128, row0, &xfull[xs]);
                    }
                    if (++xs == C::kXStages) { xs = 0; xph ^= 1; }
                }
            }
        }
    } else if (warp == 1 || warp == C::R::kMma1Warp) {
        // ===================== MMA issuers (one thread each). Issuer j takes the steps of a segment
        // with global index % kIssuers == j; both accumulate (accumulate = 1 always) into the stage's
        // shared accumulator, which the epilogue zeroed before freeing it. It waits only on afull[x]:
        // the dequant warps arrive there after acquiring xfull[x], so the TMA-written activation tile
        // of slot x is visible through that release/acquire chain.
        const int j = (warp == 1) ? 0 : 1;
        if (j < C::kIssuers && rank == 0) {   // whole warp runs the loop (warp-uniform descriptors); one lane issues
            const uint32_t idesc = idesc_i8(128 * CG, BN, /*a_signed=*/!PC && p.tx == nullptr);
            SegIter si(p, CG);
            int tile, s0, s1, cst = 0, it0 = 0;
            uint32_t cph = 0;
            while (si.next(tile, s0, s1)) {
                mbar_wait(&accempty[cst], cph);   // phase k: zeroed for its k-th use (epilogue)
                tc_fence_after();
                const uint32_t d = tmem + C::kAStages * 64 + cst * BN;
                // issuer j takes the steps with GLOBAL index it % kIssuers == j (so each X slot / A
                // buffer is always consumed by the same issuer)
                const int first = (j - it0 % C::kIssuers + C::kIssuers) % C::kIssuers;
                for (int local = first; local < s1 - s0; local += C::kIssuers) {
                    const int it = it0 + local, sg = s0 + local;
                    const int xs = it % C::kXStages, as = it % C::kAStages;
                    const uint32_t xph = (uint32_t)(it / C::kXStages) & 1u, aph = (uint32_t)(it / C::kAStages) & 1u;
                    const int nk = (2 * sg + 1 < p.KT) ? 2 : 1;
                    if (lane == 0) QOQ_TRACE_IT(p, it, 4);
                    mbar_wait(&afull[as], aph);
                    if constexpr (CG == 1) mbar_wait(&xfull[xs], xph);   // CG = 2: the dequant warps of
                    // BOTH CTAs wait on their own xfull before arriving on the leader's afull
                    if (lane == 0) QOQ_TRACE_IT(p, it, 5);
                    tc_fence_after();
                    const uint32_t a = tmem + as * 64;
                    const uint32_t sb = smem_u32(smem + C::kXOff + xs * C::kXStageBytes);
                    if (elect_one()) {
                        for (int t = 0; t < nk; ++t) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const uint64_t bdesc = smem_desc_sw128(sb + t * C::kActBytes + kk * 32);
                                if constexpr (CG == 2) mma_i8_ts2(d, a + t * 32 + kk * 8, bdesc, idesc, 1u);
                                else mma_i8_ts(d, a + t * 32 + kk * 8, bdesc, idesc, 1u);
                                if (QOQ_TRACING && p.trace && blockIdx.x == 0 && it < 16)
                                    p.trace[kTrMma + it * 8 + t * 4 + kk] = clock64();
                            }
                        }
                        if constexpr (CG == 2) {     // free the buffers in both CTAs of the pair
                            tc_commit2_mc(&aempty[as]);
                            tc_commit2_mc(&xempty[xs]);
                        } else {
                            tc_commit(&aempty[as]);      // expanded weight buffer consumed
                            tc_commit(&xempty[xs]);      // activation slot consumed
                        }
                    }
                    __syncwarp();
                    if (lane == 0) QOQ_TRACE_IT(p, it, 6);
                }
                if (elect_one()) {                              // this issuer's accumulator is final
                    if constexpr (CG == 2) tc_commit2_mc(&accfull[cst]);
                    else tc_commit(&accfull[cst]);
                }
                __syncwarp();
                if (!si.more()) pdl_launch_dependents();      // mainloop issued: let the next kernel launch
                if (j == 0 && lane == 0) QOQ_TRACE(p, 5);
                it0 += s1 - s0;
                if (++cst == C::kAccStages) { cst = 0; cph ^= 1; }
            }
        }
    } else if (warp >= 2 && warp < C::R::kDeqWarp1) {
        // ===================== dequant: u4 -> (q̂ + 128) lanes -> TMEM buffer of the step's X slot
        // The 4-warp groups take alternate steps (kDeqSplit: group g expands k-tile g of every step);
        // in a group, warp (w & 3) owns TMEM lanes 32(w&3)..+31 and thread r expands weight row r of
        // each k-tile (32 TMEM columns per tile).
        const int q = warp & 3;                       // TMEM lane quarter this warp may access
        const int grp = (warp - 2) >> 2;              // steps it with it % kDeqGroups == grp
        const int r = q * 32 + lane;                  // weight row within the tile
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const bool signed_a = !PC && (p.tx == nullptr);   // no t_x: feed s8 lanes (XOR), else biased u8
        const bool tw = (warp == 2 && lane == 0);
        SegIter si(p, CG);
        int tile, s0, s1, ws = 0, it = 0;
        uint32_t wph = 0;
        while (si.next(tile, s0, s1)) {
            for (int sg = s0; sg < s1; ++sg, ++it) {
                if (C::kDeqSplit || it % C::kDeqGroups == grp) {
                    const int nk = (2 * sg + 1 < p.KT) ? 2 : 1;
                    mbar_wait(&wfull[ws], wph);
                    if (tw) QOQ_TRACE_IT(p, it, 0);
                    const uint8_t* wb = smem + C::kWOff + ws * C::kWStageBytes;
                    uint4 v[2][4];
                    uint32_t sc[2], bias[2];
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (t < nk && (!C::kDeqSplit || t == grp)) {
                            const uint8_t* w = wb + t * C::kTB;
                            if constexpr (PC) {          // lanes = q_u4: unpack only
                                sc[t] = 1u;
                                bias[t] = 0u;
                            } else {
                                sc[t] = w[8192 + r];
                                bias[t] = (128u - (uint32_t)w[8320 + r]) * 0x01010101u;
                            }
#pragma unroll
                            for (int c = 0; c < 4; ++c) v[t][c] = *reinterpret_cast<const uint4*>(w + c * 2048 + r * 16);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&wfree[ws]);      // packed bytes now live in registers
                    if (tw) QOQ_TRACE_IT(p, it, 1);
                    const int as = it % C::kAStages;
                    const uint32_t aph = (uint32_t)(it / C::kAStages) & 1u;
                    // (kXE: expand both k-tiles BEFORE waiting for the TMEM buffer: the ALU work overlaps the MMAs
                    // still reading it, and only the stores wait; 512-thread tiles only, for the registers)
                    constexpr bool kXE = QOQ_EXPAND_EARLY && BN > 64;
                    uint32_t out2[kXE ? 2 : 1][32];
                    if constexpr (kXE) {
#pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            if (t < nk && (!C::kDeqSplit || t == grp)) {
                                if (signed_a) expand_row<true>(v[t], sc[t], bias[t], out2[t]);
                                else expand_row<false>(v[t], sc[t], bias[t], out2[t]);
                            }
                        }
                    }
                    mbar_wait(&aempty[as], aph ^ 1);             // TMEM buffer free again
                    if constexpr (CG == 2) {                     // this CTA's activation half landed
                        const int xs = it % C::kXStages;
                        mbar_wait(&xfull[xs], (uint32_t)(it / C::kXStages) & 1u);
                    }
                    if (tw) QOQ_TRACE_IT(p, it, 2);
                    tc_fence_after();
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (t < nk && (!C::kDeqSplit || t == grp)) {
                            if constexpr (kXE) {
                                tmem_st_32x32b_x32(tmem + lane_off + as * 64 + t * 32, out2[t]);
                            } else {
                                uint32_t out[32];
                                if (signed_a) expand_row<true>(v[t], sc[t], bias[t], out);
                                else expand_row<false>(v[t], sc[t], bias[t], out);
                                if (!(QOQ_ABLATE & 16)) tmem_st_32x32b_x32(tmem + lane_off + as * 64 + t * 32, out);
                                else if (out[0] == 0x12345678u && out[31] == 0x9abcdef0u) asm volatile("trap;");
                            }
                        }
                    }
                    tmem_wait_st();
                    if (tw) QOQ_TRACE_IT(p, it, 3);
                    if (QOQ_TRACING && lane == 0 && p.trace && blockIdx.x == 0 && it < 16)   // per-warp completion
                        p.trace[kTrDq + it * 8 + (warp - 2)] = clock64();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&afull[as]), 0));
                        else mbar_arrive(&afull[as]);
                    }
                }
                if (++ws == C::kWStages) { ws = 0; wph ^= 1; }
            }
        }
    } else if (warp >= C::R::kEpiWarp0 && warp < C::R::kEpiWarp0 + 4) {
        // ===================== epilogue (warps 10-13)
        const int q = warp & 3;
        const int r = q * 32 + lane;                  // TMEM lane = weight row within the tile
        const int et = threadIdx.x - C::R::kEpiThread0;   // 0..127 for cooperative phases
        const int g = et >> 5, l = et & 31;           // vector mapping: rows 4l..4l+3, tokens g, g+4, ...
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        // every accumulator stage starts zeroed: completes phase 0 of accempty (the issuers' first wait)
        for (int st = 0; st < C::kAccStages; ++st) {
            zero_acc<BN>(tmem + lane_off + C::kAStages * 64 + st * BN);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&accempty[st]), 0));
                else mbar_arrive(&accempty[st]);
            }
        }
        pdl_wait();
        if (et == 0) QOQ_TRACE(p, 12);
        // fused TP reduction: this call's parity and expected flag count (gen was advanced by the previous
        // fused call's last CTA, complete before griddepcontrol.wait returns)
        uint32_t tp_par = 0, tp_flag = 0;
        if constexpr (TP) {
            const uint32_t gen = __ldcg(p.tp.gen);
            tp_par = gen & 1u;
            tp_flag = gen + 1u;
        }
        if constexpr (FQ) {   // fused per-token quantization of X, then the grid handshake (s_x / t_x below)
            fused_quantize_rows(p, et, sxs, txs);
            if (et == 0) {
                QOQ_TRACE(p, 3);
                spin_until_ge(p.qsync, (int)gridDim.x);
                QOQ_TRACE(p, 4);
                fused_depart(p);
            }
            named_bar_sync(1, 128);
        }
        SegIter si(p, CG);
        int tile, s0, s1, cst = 0;
        uint32_t cph = 0;
        while (si.next(tile, s0, s1)) {
            int nu, mt;
            tile_coords(p, tile, nu, mt);
            const int nt = nu * CG + rank;
            tile = nt * p.MT + mt;   // the real 128-row tile of this CTA (workspace / counters index)
            const int n0 = nt * 128, m0 = mt * BN;
            const bool whole = (s0 == 0 && s1 == p.KS);
            int32_t* wst = p.ws + (size_t)tile * 128 * BN;
            for (int jj = et; jj < BN; jj += 128) {
                const int m = m0 + jj;
                // coherent (L2) loads: with the fused quantization they were written by this grid
                sxs[jj] = (!OUT_I32 && m < p.M) ? __half2float(__ldcg(p.sx + m)) : 0.0f;
                txs[jj] = (p.tx && m < p.M) ? (PC ? 1 : 128) * __ldcg(p.tx + m) : 0;
            }
            float s0v[4] = {0.f, 0.f, 0.f, 0.f};
            int z0v[4];
            load_z4<PC>(p, n0 + 4 * l, z0v);
            if constexpr (!OUT_I32) {
                const uint2 u = __ldg(reinterpret_cast<const uint2*>(p.s0 + n0 + 4 * l));
                const __half2* h2 = reinterpret_cast<const __half2*>(&u);
                const float2 a = __half22float2(h2[0]), b = __half22float2(h2[1]);
                s0v[0] = a.x; s0v[1] = a.y; s0v[2] = b.x; s0v[3] = b.y;
            }
            named_bar_sync(1, 128);
            mbar_wait(&accfull[cst], cph);
            if (et == 0) QOQ_TRACE(p, 6);
            tc_fence_after();
            const uint32_t d = tmem + lane_off + C::kAStages * 64 + cst * BN;
            if (clustered) {
                // ---- cluster split-K, reduce-scatter through DSMEM: stage this CTA's partial (sum of
                // both issuers' accumulators) row-major [128][BN+4] in its now-idle X ring; the rows
                // of CTA c's slice are one contiguous block, bulk-reduce-added into CTA c's staging.
                int32_t* part = reinterpret_cast<int32_t*>(smem + C::kXOff);
#pragma unroll 1
                for (int ci = 0; ci < BN / C::kChunk; ++ci) {
                    const int j0 = ci * C::kChunk;
                    uint32_t v[C::kChunk];
                    tmem_ld_chunk<BN>(d + j0, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < C::kChunk; i += 4)
                        *reinterpret_cast<int4*>(part + r * kRP + j0 + i) =
                            make_int4((int)v[i], (int)v[i + 1], (int)v[i + 2], (int)v[i + 3]);
                }
                if (si.more()) {   // (the CTA's last segment: no issuer waits for this accumulator again)
                    zero_acc<BN>(d);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&accempty[cst]);
                }
                fence_proxy_async_smem();
                if (et == 0) QOQ_TRACE(p, 23);
                named_bar_sync(1, 128);
                if (et == 0) QOQ_TRACE(p, 24);
                cluster_wait_acquire();   // every CTA's zeroed slice + armed red_full (setup arrive)
                if (et == 0) QOQ_TRACE(p, 25);
                const int R = 128 / p.S;
                // this thread's output rows are the same 4 in every write-out iteration below
                // (w % nq is invariant): fetch their s0 now, off the critical path
                const int nq = R / 4;
                float s4[4] = {0.f, 0.f, 0.f, 0.f};
                int z4[4];
                load_z4<PC>(p, n0 + crank * R + (et % nq) * 4, z4);
                if constexpr (!OUT_I32) {
                    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p.s0 + n0 + crank * R + (et % nq) * 4));
                    const __half2* h2 = reinterpret_cast<const __half2*>(&u);
                    const float2 fa = __half22float2(h2[0]), fb = __half22float2(h2[1]);
                    s4[0] = fa.x; s4[1] = fa.y; s4[2] = fb.x; s4[3] = fb.y;
                }
                if (et < p.S) {   // thread c sends slice c to cluster rank c
                    const uint32_t bytes = (uint32_t)(R * kRP * 4);
                    bulk_reduce_add_s32_cluster(mapa_shared(smem_u32(stg), et), part + et * R * kRP, bytes,
                                                mapa_shared(smem_u32(red_full), et));
                }
                if (et == 0) QOQ_TRACE(p, 7);
                mbar_wait(red_full, 0);
                if (et == 0) QOQ_TRACE(p, 22);
                // every slice this CTA receives has landed, so every read of the peers' partials that
                // targets it is done: arrive on the exit barrier now and overlap its latency with
                // the write-out below (relaxed: the barrier orders lifetimes, it publishes no data)
                cluster_arrive_relaxed();
                cl_done = true;
                // this CTA's R rows, all BN tokens: thread -> (token jj, 4 consecutive rows); w % nq
                // is fixed per thread, so thread et covers tokens et / nq + (128 / nq) u. All
                // shared-memory reads first, then the guarded stores (see the mode-0 write-out).
                if constexpr (BN <= 64) {                       // mode 2 only runs BN <= 64 (plan_gemm)
                    constexpr int kU = BN / 8;                   // iterations at the smallest slice (S = 2)
                    constexpr int kB = kU < 4 ? kU : 4;          // batch (register budget)
                    const int rr = (et % nq) * 4, n = n0 + crank * R + rr, step = 128 / nq;
                    const int items = nq * BN;                   // item w = et + 128 u
#pragma unroll 1
                    for (int u0 = 0; u0 < kU && et + 128 * u0 < items; u0 += kB) {
                        int4 av[kB];
                        float sv[kB];
                        int tv[kB];
#pragma unroll
                        for (int b = 0; b < kB; ++b) {
                            const int u = u0 + b, jj = et / nq + step * u;
                            if (et + 128 * u < items) {
                                av[b] = make_int4(stg[(rr + 0) * kRP + jj], stg[(rr + 1) * kRP + jj],
                                                  stg[(rr + 2) * kRP + jj], stg[(rr + 3) * kRP + jj]);
                                sv[b] = sxs[jj];
                                tv[b] = txs[jj];
                            }
                        }
#pragma unroll
                        for (int b = 0; b < kB; ++b) {
                            const int u = u0 + b, m = m0 + et / nq + step * u;
                            if (et + 128 * u < items && m < p.M) write_out4<OUT_I32>(p, m, n, av[b], tv[b], sv[b], s4, z4);
                        }
                    }
                }
                if (et == 0) QOQ_TRACE(p, 9);
                if (++cst == C::kAccStages) { cst = 0; cph ^= 1; }
                named_bar_sync(1, 128);
                continue;
            }
#pragma unroll 1
            for (int ci = 0; ci < BN / C::kChunk; ++ci) {
                const int j0 = ci * C::kChunk;
                int32_t* sb = stg + (ci & 1) * (C::kChunk * 128);
                uint32_t v[C::kChunk];
                tmem_ld_chunk<BN>(d + j0, v);
                tmem_wait_ld();
                if (et == 0 && ci == 0) QOQ_TRACE(p, 27);
                // accumulator fully read: zero it and hand it back, unless this is the CTA's last segment (no
                // issuer waits for it again)
                if (ci == BN / C::kChunk - 1 && si.more()) {
                    zero_acc<BN>(d);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&accempty[cst]), 0));
                        else mbar_arrive(&accempty[cst]);
                    }
                }
                if (et == 0 && ci == 1) QOQ_TRACE(p, 30);
                if (et == 0) bulk_wait_read<1>();        // staging buffer (ci & 1) no longer read by TMA
                named_bar_sync(1, 128);
                if (et == 0 && ci == 0) QOQ_TRACE(p, 28);
#pragma unroll
                for (int i = 0; i < C::kChunk; ++i) sb[i * 128 + r] = (int32_t)v[i];
                if (et == 0 && ci == 0) QOQ_TRACE(p, 31);
                if (!whole) {
                    fence_proxy_async_smem();
                    named_bar_sync(1, 128);
                    if (et == 0) {
                        bulk_reduce_add_s32(wst + (size_t)j0 * 128, sb, C::kStgBytes);
                        bulk_commit();
                    }
                } else if constexpr (TP) {
                    // NEXT-3: this rank's partial -> slot `rank` of every rank, one 16-byte flag-in-data store per
                    // 4 outputs and rank; all shared-memory reads first, as in the plain write-out
                    named_bar_sync(1, 128);
                    constexpr int kU = C::kChunk / 4;
                    int4 av[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u) av[u] = *reinterpret_cast<const int4*>(sb + (g + 4 * u) * 128 + 4 * l);
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const int jj = g + 4 * u, m = m0 + j0 + jj;
                        if (m >= p.M) break;
                        const uint2 y = y4_bits(av[u], txs[j0 + jj], sxs[j0 + jj], s0v, z0v);
                        const uint4 w = make_uint4(y.x, tp_flag, y.y, tp_flag);
                        const size_t off = tp_word(p.tp, tp_par, p.tp.rank, m, n0 + 4 * l);
#pragma unroll 1
                        for (int q = 0; q < p.tp.world; ++q) st_relaxed_sys_v4(static_cast<uint2*>(p.tp.recv[q]) + off, w);
                    }
                } else {
                    named_bar_sync(1, 128);
                    // all shared-memory reads first, then the stores: the (m < M) guards would
                    // otherwise serialize one LDS -> convert -> STG latency chain per token
                    constexpr int kU = C::kChunk / 4;
                    int4 av[kU];
                    float sv[kU];
                    int tv[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const int jj = g + 4 * u;
                        av[u] = *reinterpret_cast<const int4*>(sb + jj * 128 + 4 * l);
                        sv[u] = sxs[j0 + jj];
                        tv[u] = txs[j0 + jj];
                    }
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const int m = m0 + j0 + g + 4 * u;
                        if (m < p.M && !(QOQ_ABLATE & 32)) write_out4<OUT_I32>(p, m, n0 + 4 * l, av[u], tv[u], sv[u], s0v, z0v);
                        else if ((QOQ_ABLATE & 32) && av[u].x == 0x7fffffff && sv[u] == 1.2345f) asm volatile("trap;");
                    }
                    if (et == 0 && ci == 0) QOQ_TRACE(p, 29);
                }
            }
            if (et == 0) QOQ_TRACE(p, 26);
            if constexpr (TP) {
                // reduce in rank order (fp32, one rounding to fp16): thread (g, l) owns Y[m][n0 + 4l .. +3] for
                // the tile's tokens m = m0 + g + 4j (the write-out mapping, so its own slot's words are its own
                // earlier stores); each word is valid once it carries this call's flag. kB tokens per batch:
                // all of a batch's loads of one slot in flight, then only the missing words re-polled
                const uint2* rb = static_cast<const uint2*>(p.tp.recv[p.tp.rank]);
                constexpr int kB = BN / 4 < 4 ? BN / 4 : 4;
#pragma unroll 1
                for (int j0 = g; j0 < BN && m0 + j0 < p.M; j0 += 4 * kB) {
                    const int n = n0 + 4 * l;
                    float a[kB][4];
#pragma unroll 1
                    for (int q = 0; q < p.tp.world; ++q) {
                        uint4 v[kB];
#pragma unroll
                        for (int b = 0; b < kB; ++b) {
                            const int m = m0 + j0 + 4 * b;
                            v[b] = (j0 + 4 * b < BN && m < p.M) ? ld_relaxed_sys_v4(rb + tp_word(p.tp, tp_par, q, m, n))
                                                                : make_uint4(0u, tp_flag, 0u, tp_flag);
                        }
#pragma unroll
                        for (int b = 0; b < kB; ++b) {
                            if (v[b].y != tp_flag || v[b].w != tp_flag)
                                v[b] = tp_poll(p.tp, rb + tp_word(p.tp, tp_par, q, m0 + j0 + 4 * b, n), tp_flag);
                            const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&v[b].x));
                            const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&v[b].z));
                            if (q == 0) { a[b][0] = f0.x; a[b][1] = f0.y; a[b][2] = f1.x; a[b][3] = f1.y; }
                            else { a[b][0] += f0.x; a[b][1] += f0.y; a[b][2] += f1.x; a[b][3] += f1.y; }
                        }
                    }
#pragma unroll
                    for (int b = 0; b < kB; ++b) {
                        const int m = m0 + j0 + 4 * b;
                        if (j0 + 4 * b >= BN || m >= p.M) continue;
                        __half2 lo = __halves2half2(__float2half_rn(a[b][0]), __float2half_rn(a[b][1]));
                        __half2 hi = __halves2half2(__float2half_rn(a[b][2]), __float2half_rn(a[b][3]));
                        uint2 u;
                        u.x = *reinterpret_cast<uint32_t*>(&lo);
                        u.y = *reinterpret_cast<uint32_t*>(&hi);
                        *reinterpret_cast<uint2*>(static_cast<__half*>(p.out) + (size_t)m * p.ldo + n) = u;
                    }
                }
            }
            if (++cst == C::kAccStages) { cst = 0; cph ^= 1; }
            if (!whole) {
                if (et == 0) {
                    bulk_wait<0>();                      // this CTA's partial tile is in L2
                    fence_proxy_async_global();
                    __threadfence();
                    QOQ_TRACE(p, 7);
                    const int prev = atomicAdd(p.counters + tile, s1 - s0);
                    *fin_flag = (prev + (s1 - s0) == p.KS) ? 1 : 0;
                }
                named_bar_sync(1, 128);
                if (*fin_flag) {   // last contributor: finish the tile and restore the zero workspace
                    __threadfence();
#pragma unroll 1
                    for (int jb = 0; jb < BN; jb += 4 * C::kFinU) {
                        int4 acc[C::kFinU];
#pragma unroll
                        for (int u = 0; u < C::kFinU; ++u)
                            acc[u] = ld_cg_v4(wst + (size_t)(jb + g + 4 * u) * 128 + 4 * l);
#pragma unroll
                        for (int u = 0; u < C::kFinU; ++u) {
                            const int jj = jb + g + 4 * u;
                            *reinterpret_cast<int4*>(wst + (size_t)jj * 128 + 4 * l) = make_int4(0, 0, 0, 0);
                            if (m0 + jj < p.M) write_out4<OUT_I32>(p, m0 + jj, n0 + 4 * l, acc[u], txs[jj], sxs[jj], s0v, z0v);
                        }
                    }
                    if (et == 0) {
                        p.counters[tile] = 0;
                        QOQ_TRACE(p, 9);
                    }
                }
            }
            named_bar_sync(1, 128);   // sxs / txs / staging / fin_flag reuse by the next segment
            if (et == 0) QOQ_TRACE(p, 8);
        }
        if (et == 0) bulk_wait<0>();
        // fused TP reduction: the last CTA out advances this rank's call counter (read by the next fused call
        // after its griddepcontrol.wait)
        if (TP && et == 0) {   // (no fence: the next call reads gen after grid completion)
            if (atomicAdd(p.tp.done, 1u) == gridDim.x - 1) {
                *p.tp.done = 0u;
                atomicAdd(p.tp.gen, 1u);
            }
        }
    }

    tc_fence_before();
    if (threadIdx.x == C::R::kEpiThread0) QOQ_TRACE(p, 14);
    // mode 2: the exit barrier (phase 1) must only wait for every CTA's slices to land (the epilogue
    // threads arrive right after red_full); threads that never touch peer memory arrive as soon as
    // their role is done, not after this CTA's write-out.
    if (clustered && !cl_done) {
        cluster_wait_acquire();
        cluster_arrive_relaxed();
        cl_done = true;
    }
    __syncthreads();
    if (threadIdx.x == 0) QOQ_TRACE(p, 15);
    // mode 2: no CTA may exit while a peer's bulk reduce still reads its partial or writes its slice:
    // the exit barrier completes once every CTA has seen its own slice complete (arrived above).
    // CG = 2: the leader's MMAs read the peer's TMEM; both CTAs are past their epilogues here
    if (CG == 2) {
        cluster_sync_all();
    } else if (clustered) {
        cluster_wait_acquire();
    }
    if (threadIdx.x == 0) QOQ_TRACE(p, 10);
    pdl_launch_dependents();
    if (warp == 1) {
        tc_fence_after();
        if constexpr (CG == 2) tmem_dealloc2(tmem, C::kTmemCols);
        else tmem_dealloc(tmem, C::kTmemCols);
    }
}

// ------------------------------------------------------------------ host side

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

// Largest number of co-resident S-CTA clusters of the BN kernel (cached per (BN, S); immutable after).
template <int BN>
static int max_clusters(int S) {
    static int cache[9] = {0};
    if (S < 1 || S > 8) return 0;
    if (cache[S] == 0) {
        auto kern = w4a8_gemm_kernel<BN, false, 1>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN, 1>::kSmemBytes);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(S * 64);
        cfg.blockDim = dim3(Cfg<BN, 1>::kBlockThreads);
        cfg.dynamicSmemBytes = Cfg<BN, 1>::kSmemBytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = S;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            n = -1;
        }
        cache[S] = n;
    }
    return cache[S];
}

static int max_clusters_bn(int BN, int S) {
    switch (BN) {
        case 16: return max_clusters<16>(S);
        case 32: return max_clusters<32>(S);
        case 64: return max_clusters<64>(S);
        default: return 0;
    }
}

GemmPlan plan_gemm(int M, int N, int K, int num_sms) {
    GemmPlan p{};
    // token tile: the smallest of 16/32/64/128 that holds M; above M = 128 the cost model below picks
    // 128, 192 (double-buffered TMEM accumulators: the epilogue overlaps the next tile) or 256 (single
    // accumulator) by whole waves x per-tile cost, among tiles that fill the GPU.
    p.BN = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : 128;
    if (M > 128) {
        // prefill: pick the token tile by whole waves x per-tile cost, among tiles that fill the GPU
        // (T >= #SMs: mode 0; below that the stream-K partials of wide tiles cost more than they
        // save). Relative per-token costs measured on B200 (tools/prefill_ab.sh): BN = 128 expands
        // each weight tile for half as many tokens (~1.2x); BN = 256 runs its epilogue without
        // overlap (~1.2x at K = 4096, shrinking with K). QOQ_BN_BIG=128/192/256 forces.
        const int force = knobs().bn_big;
        const int cand[3] = {128, 192, 256};
        const double eff[3] = {1.2, 1.0, 1.0 + 0.2 * 4096.0 / K};
        double best = 1e300;
        p.BN = 128;
        for (int i = 0; i < 3; ++i) {
            const long long mt = (M + cand[i] - 1) / cand[i], t = mt * (N / kTileN);
            const double cost = (double)((t + num_sms - 1) / num_sms) * cand[i] * eff[i];
            if (force ? force == cand[i] : (t >= num_sms && cost < best)) {
                best = cost;
                p.BN = cand[i];
            }
        }
    }
    p.MT = (M + p.BN - 1) / p.BN;
    {   // activation band of the work order: <= 32 MB of q_x (tile_coords)
        const long long per = (long long)p.BN * K;
        const long long mb = (32ll << 20) / (per > 0 ? per : 1);
        p.MB = (int)(mb < 1 ? 1 : mb > p.MT ? p.MT : mb);
    }
    p.NT = N / kTileN;
    p.KT = K / kTileK;
    p.T = p.MT * p.NT;
    p.KS = (p.KT + 1) / 2;
    p.I = (long long)p.T * p.KS;
    p.S = 1;
    // Decomposition policy (measured on B200, tools/mode_sweep.sh, Llama-3-8B decode shapes):
    //  * T >= #SMs: whole tiles (mode 0).
    //  * BN <= 32: S-CTA cluster split-K through DSMEM (mode 2) — the partial is only 8-16 KB/CTA.
    //  * BN = 64: no split while K <= 3072 steps-worth (KS <= 24; the pipeline fill/drain per CTA
    //    costs more than the idle SMs); for long K the cluster reduce-scatter (mode 2, 14.3 us for
    //    down_proj M=64) edges out stream-K through the L2 workspace (mode 1, 14.6 us).
    //  * BN >= 128 with T < #SMs: stream-K (mode 1).
    // QOQ_FORCE_MODE=0/1/2 overrides (debug / tests).
    const int force = knobs().force_mode;
    int want;
    if (force >= 0 && force <= 2) want = force;
    else if (p.T >= num_sms) want = 0;
    else if (p.BN <= 32) want = 2;
    else if (p.BN == 64) want = p.KS <= 24 ? 0 : 2;
    else want = 1;
    if (want == 2 && p.BN > 64) want = 1;   // the DSMEM reduction target holds at most 128 x 64 INT32
    int S = 1;
    if (want == 2) {
        // reduce-scatter slices of 128/S rows: S a power of two <= 8, <= #steps, all clusters resident
        S = 1;
        while (S * 2 <= 8 && (long long)p.T * S * 2 <= num_sms && S * 2 <= p.KS) S *= 2;
        while (S >= 2) {
            const int mc = max_clusters_bn(p.BN, S);
            if (mc < 0 || (long long)mc >= p.T) break;   // all T clusters co-resident (or query unavailable)
            S /= 2;
        }
        if (S < 2) want = (p.KS <= 24) ? 0 : 1;
    }
    if (want == 2) {
        p.mode = 2;
        p.S = S;
        p.G = p.T * S;
        p.ws_bytes = 0;
    } else if (want == 1) {
        p.mode = 1;
        p.G = (int)(p.I < num_sms ? p.I : num_sms);
        p.ws_bytes = (size_t)p.MT * p.NT * 128 * p.BN * 4 + (size_t)p.MT * p.NT * 4;
    } else {
        p.mode = 0;
        p.G = p.T < num_sms ? p.T : num_sms;
        p.ws_bytes = 0;
    }
    // CTA pairs (cta_group::2) for modes 0 / 1 when the 128-row tiles pair up. Work units become
    // tile pairs: T = units, G = pairs (the grid is 2G CTAs in clusters of 2).
    const int force_cg = knobs().force_cg;
    const bool pair_ok = p.mode != 2 && p.NT % 2 == 0 && p.BN >= 32;
    // Opt-in for now (QOQ_FORCE_CG=2): bit-exact, but on B200 two of the four dequant warps' tcgen05.st
    // stall for thousands of cycles while the pair's cta_group::2 MMAs run (tools/trace_gemm.py), so
    // the pair pipeline is slower than single CTAs at decode sizes. See DESIGN.md §6.
    p.CG = (pair_ok && force_cg == 2) ? 2 : 1;
    if (p.CG == 2) {
        p.T = p.MT * (p.NT / 2);
        p.I = (long long)p.T * p.KS;
        const int pairs = num_sms / 2;
        if (p.mode == 0) p.G = p.T < pairs ? p.T : pairs;
        else p.G = (int)(p.I < pairs ? p.I : pairs);
    }
    return p;
}

template <int BN, bool OUT_I32, int CG, bool PC = false, bool TP = false, bool FQ = false>
static cudaError_t launch_bn(const GemmArgs& a, const GemmPlan& pl, cudaStream_t st, bool pdl) {
    using C = Cfg<BN, CG, PC, TP>;
    auto kern = w4a8_gemm_kernel<BN, OUT_I32, CG, PC, TP, FQ>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    auto enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.M};
    cuuint64_t strides[1] = {(cuuint64_t)a.K};
    cuuint32_t box[2] = {128u, (cuuint32_t)(BN / CG)};
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
    kp.counters = a.ws ? reinterpret_cast<int*>(static_cast<uint8_t*>(a.ws) + (size_t)pl.MT * pl.NT * 128 * BN * 4)
                       : nullptr;
    kp.M = a.M;
    kp.MT = pl.MT;
    kp.MB = pl.MB;
    kp.KT = pl.KT;
    kp.KS = pl.KS;
    kp.T = pl.T;
    kp.G = pl.G;
    kp.mode = pl.mode;
    kp.S = pl.S;
    kp.I = pl.I;
    kp.trace = static_cast<unsigned long long*>(a.trace);
    kp.X = static_cast<const __half*>(a.X);
    kp.qx_rows = const_cast<int8_t*>(a.qx);
    kp.ldx = a.ldx;
    kp.K = a.K;
    kp.qsync = a.qsync;
    kp.zw = a.zw;
    if (TP) kp.tp = *a.tp;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.G * CG);
    cfg.blockDim = dim3(C::kBlockThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (pl.mode == 2 || CG == 2) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = CG == 2 ? 2 : pl.S;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, tm, kp);
}

template <int BN>
static cudaError_t launch_bn_cg(const GemmArgs& a, const GemmPlan& p, cudaStream_t st, bool pdl) {
    if (a.X) {    // qoq_w4a8_linear's one-kernel path: fp16 out, M <= kFuseMaxM (token tiles 16 / 32 / 64)
        if (a.out_i32 || a.zw || a.tp) return cudaErrorInvalidValue;
        if constexpr (BN <= 64) {
            if (p.CG == 2) {
                if constexpr (BN >= 32) return launch_bn<BN, false, 2, false, false, true>(a, p, st, pdl);
                return cudaErrorInvalidValue;
            }
            return launch_bn<BN, false, 1, false, false, true>(a, p, st, pdl);
        }
        return cudaErrorInvalidValue;
    }
    if (a.tp) {   // fused TP reduction: whole tiles, single CTAs, fp16 out (tp_plan)
        if (p.CG != 1 || p.mode != 0 || a.out_i32 || a.zw) return cudaErrorInvalidValue;
        if constexpr (BN <= 128) return launch_bn<BN, false, 1, false, true>(a, p, st, pdl);
        return cudaErrorInvalidValue;
    }
    if (a.zw) {   // per-channel W4A8: single-CTA tiles only
        if (p.CG != 1) return cudaErrorInvalidValue;
        return a.out_i32 ? launch_bn<BN, true, 1, true>(a, p, st, pdl) : launch_bn<BN, false, 1, true>(a, p, st, pdl);
    }
    if (p.CG == 2) {
        if constexpr (BN >= 32)
            return a.out_i32 ? launch_bn<BN, true, 2>(a, p, st, pdl) : launch_bn<BN, false, 2>(a, p, st, pdl);
        return cudaErrorInvalidValue;
    }
    return a.out_i32 ? launch_bn<BN, true, 1>(a, p, st, pdl) : launch_bn<BN, false, 1>(a, p, st, pdl);
}

cudaError_t launch_w4a8_gemm(const GemmArgs& a, const GemmPlan& p, cudaStream_t st, bool pdl) {
    switch (p.BN) {
        case 16: return launch_bn_cg<16>(a, p, st, pdl);
        case 32: return launch_bn_cg<32>(a, p, st, pdl);
        case 64: return launch_bn_cg<64>(a, p, st, pdl);
        case 128: return launch_bn_cg<128>(a, p, st, pdl);
        case 192: return launch_bn_cg<192>(a, p, st, pdl);
        case 256: return launch_bn_cg<256>(a, p, st, pdl);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qoq
