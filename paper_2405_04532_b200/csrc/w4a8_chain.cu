// w4a8_chain.cu — a chain of W4A8 linear layers in ONE persistent kernel (the decode regime, M <= 128).
//
// Computes, for j = 0 .. n-1 in order (each step the same arithmetic as qoq_w4a8_linear):
//     q_x, s_x, t_x = per-token INT8 quantization of X_j
//     Y_j[m][n]     = fp16( (Σ_k q̂_j[n][k] q_x[m][k]) · s_x[m] · s0_j[n] )
// with X_j read only after Y_0 .. Y_{j-1} are complete, so X_j may be (a view of) an earlier Y_i.
//
// Why one kernel: at decode sizes a W4A8 GEMM is a stream of static packed weights (HBM-bound)
// whose launches each pay a setup, a pipeline fill and an epilogue drain, and whose activation
// quantizer is another launch in between. Here every SM runs one CTA for the whole chain:
//  * the weight producer streams EVERY linear's packed tiles back to back, never waiting for
//    activations (weights are static), so HBM keeps streaming across layer boundaries while a
//    boundary's dependency (finish Y_{j-1} -> quantize X_j) resolves; the dequant warps expand the
//    next linear's weights into TMEM meanwhile;
//  * a decode-sized linear (fewer 128-row tiles than SMs) splits each tile's K range over S CTAs, a
//    large one runs stream-K over all CTAs ("partition the reduction dimension k into multiple
//    slices"); partial tiles are exact INT32 sums, finished by row slices in every contributor;
//  * the per-token quantization (fused into the producing kernel) runs inside the kernel:
//    CTA b's epilogue warps quantize rows m ≡ b (mod grid) once the previous linear is complete.
// Cross-CTA handoffs (partial tiles, Y, q_x) are written with TMA bulk stores, completed
// (cp.async.bulk.wait_group 0) and then published with a RELAXED counter increment; consumers acquire
// the counter and read with TMA. A gpu-scope release fence on an SM that streams weights waits for
// that SM's in-flight weight loads (~4,400 cycles measured, tools/fence_bench.cu, vs ~330 idle), so
// the critical path carries no release fence ("decode chain").
// The main loop (dequant -> TMEM -> tcgen05.mma kind::i8 -> TMEM accumulators) is the one of
// w4a8_gemm.cu (biased-u8 weights, the epilogue subtracts 128 t_x).
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

// ------------------------------------------------------------------ configuration

#ifndef QOQ_CHAIN_XSTAGES
#define QOQ_CHAIN_XSTAGES 4      // activation ring depth (BN <= 64)
#endif
#ifndef QOQ_CHAIN_DEQ_GROUPS
#define QOQ_CHAIN_DEQ_GROUPS 3   // dequant warpgroups (BN <= 64)
#endif

template <int BN>
struct ChainCfg {
    static constexpr int kDeqGroups = BN <= 64 ? QOQ_CHAIN_DEQ_GROUPS : 2;
    using R = Roles<kDeqGroups>;
    static constexpr int kBlockThreads = R::kBlockThreads;
    static constexpr int kIssuers = 2;
    static constexpr int kActBytes = BN * 128;                    // one k-tile of activations (BN rows)
    static constexpr int kXStageBytes = 2 * kActBytes;            // one step (2 k-tiles)
    static constexpr int kChunk = BN < 32 ? BN : 32;              // TMEM columns per tcgen05.ld
    static constexpr int kPartTok = BN < 64 ? BN : 64;            // tokens per staged partial (one bulk store)
    static constexpr int kG4 = kPartTok / 4;                      // 16-byte granules (4 tokens) per staged row
    // staging: a [128][kPartTok] INT32 partial tile, the <= 4 contributors' slices of a tile, or an X row
    static constexpr int kStgBytes = 36864;
    // fp16 output staging: [kPartTok][128] (a whole tile's Y, per token half) or an X row's codes
    static constexpr int kYStgBytes = 16384;
    static constexpr int kEpiBytes = kStgBytes + kYStgBytes + BN * 8 + 64;
    static constexpr int kARot = kDeqGroups % 2 == 0 ? kDeqGroups : 2 * kDeqGroups;   // lcm(2 issuers, G)
    static constexpr int kAccStages = 2;
    static constexpr int kAccCols = kAccStages * BN;
    static constexpr int kARaw0 = (512 - kAccCols) / 64;
    static constexpr int kARaw = kARaw0 > 6 ? 6 : kARaw0;
    static constexpr int kAStages = (kARaw / kARot) * kARot;
    static constexpr int kXStages = BN == 128 ? 2 : QOQ_CHAIN_XSTAGES;
    static constexpr int kWStageBytes = ((2 * kTileBytes + 1023) / 1024) * 1024;
    static constexpr int kBudget = 225 * 1024;
    static constexpr int kWRaw = (kBudget - kEpiBytes - kXStages * kXStageBytes) / kWStageBytes;
    static constexpr int kWCap = kWRaw > 12 ? 12 : kWRaw;
    static constexpr int kWStages = (kWCap / kDeqGroups) * kDeqGroups;
    static constexpr int kTmemCols = 512;
    static constexpr int kXOff = 0;
    static constexpr int kWOff = kXStages * kXStageBytes;
    static constexpr int kEpiOff = kWOff + kWStages * kWStageBytes;
    static constexpr int kBarOff = kEpiOff + kEpiBytes;
    static constexpr int kBarBytes = 8 * (2 * kWStages + 2 * kXStages + 2 * kAStages + 2 * kAccStages + 2) + 16;
    static constexpr int kSmemBytes = 1024 + kBarOff + kBarBytes;
    static_assert(kXStages >= 2 && kXStages % kIssuers == 0, "X ring");
    static_assert(kWStages >= 3 && kWStages % kDeqGroups == 0, "W ring");
    static_assert(kAStages >= 2 && kAStages % kARot == 0, "A ring");
    static_assert(kAStages * 64 + kAccCols <= 512, "TMEM overflow");
    static_assert(kSmemBytes <= 227 * 1024, "SMEM overflow");
    static_assert(kPartTok * 128 * 4 <= kStgBytes && kPartTok * 256 <= kYStgBytes, "staging");
};

// kChainQMaxK (qoq_internal.h): the in-kernel quantizer stages the fp16 row in the staging area and the
// codes (+ 16 B of meta) in the output staging area
static_assert(2 * kChainQMaxK <= 36864 && kChainQMaxK + 16 <= 16384, "quantizer staging");

// ------------------------------------------------------------------ debug timeline (QOQ_TRACING)

#ifndef QOQ_TRACING
#define QOQ_TRACING 0
#endif
// per (linear, CTA) %globaltimer stamps (tools/trace_chain.py): 0 quantization start (Y_{j-1} complete),
// 1 quantization released, 2 activation producer acquired q_x, 3 first MMA issued, 4 last MMA committed,
// 5 epilogue done (before the tile-count release), 6 first weights of the linear in SMEM (dequant),
// 7 first weight copy issued, 8 X row staged, 9 row scale known, 10 row codes stored, 11 before the
// q release, 12 first accumulator ready (epilogue), 13 partials announced, 14 first tile's contributors
// all landed, 15 finalize done
#if QOQ_TRACING
__device__ __forceinline__ unsigned long long chain_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// [n][G][32] %globaltimer (comparable across SMs), then [n][G][16] clock64 (cycle-exact within a CTA)
#define QOQ_CTRACE(p, j, ev) \
    do { if ((p).trace) { const size_t o_ = ((size_t)(j) * (p).G + blockIdx.x) * 32 + (ev); \
                          (p).trace[o_] = chain_gtimer(); \
                          (p).trace[(size_t)(p).njobs * (p).G * 32 + o_] = clock64(); } } while (0)
#else
#define QOQ_CTRACE(p, j, ev) do { } while (0)
#endif

// ------------------------------------------------------------------ scheduling

// Work of linear j for CTA b (host-planned, ChainJob::S):
//  * S >= 1 (NT < G, decode-sized linears): tile b / S, the (b % S)-th of S equal k-ranges, for b < NT S —
//    one segment per CTA, so a 32-tile o_proj runs on 128 SMs;
//  * S == 0 (NT >= G): stream-K, steps [b I / G, (b+1) I / G) of the I = NT KS tile-major steps (whole
//    tiles in the middle, a partial tile at either end; no wave quantization).
// Every role walks the same sequence.
// The CTA that owns step s of a stream-K linear: the largest b with floor(b I / G) <= s.
__device__ __forceinline__ int streamk_owner(long long s, long long I, int G) {
    return (int)(((s + 1) * G + I - 1) / I) - 1;
}

// Segment order inside a CTA's stream-K range [c0, c1): the (possibly partial) segments of its first and
// last tile come FIRST, the whole tiles in between last, so the partial tiles' reductions and their
// finishing overlap the whole tiles' main loop instead of trailing it.
struct ChainIter {
    int j, b, G, n;
    long long c0, c1;   // this CTA's steps of linear j
    int KS, t0, t1, idx, cnt;
    __device__ explicit ChainIter(const ChainParams& p) : j(-1), b(blockIdx.x), G(p.G), n(p.njobs), idx(0), cnt(0) {}
    __device__ void enter(const ChainParams& p, int jj) {
        j = jj;
        const ChainJob& J = p.job[jj];
        KS = J.KS;
        if (J.S > 0) {
            if (b < J.NT * J.S) {
                const long long t = b / J.S, c = b % J.S;
                c0 = t * J.KS + c * J.KS / J.S;
                c1 = t * J.KS + (c + 1) * J.KS / J.S;
            } else {
                c0 = c1 = 0;
            }
        } else {
            c0 = (long long)b * J.I / G;
            c1 = (long long)(b + 1) * J.I / G;
        }
        idx = 0;
        if (c1 > c0) {
            t0 = (int)(c0 / KS);
            t1 = (int)((c1 - 1) / KS);
            cnt = t1 - t0 + 1;
        } else {
            cnt = 0;
        }
    }
    __device__ void seg(int& tile, int& s0, int& s1) {
        // the end segments in order A (tile t0), B (tile t1), unless A is whole and B partial
        const bool swap = t1 > t0 && c0 == (long long)t0 * KS && c1 != (long long)(t1 + 1) * KS;
        const int e = idx < 2 ? (idx ^ (swap ? 1 : 0)) : idx;
        if (e == 0) {
            tile = t0;
            s0 = (int)(c0 - (long long)t0 * KS);
            s1 = t1 == t0 ? (int)(c1 - (long long)t0 * KS) : KS;
        } else if (e == 1) {
            tile = t1;
            s0 = 0;
            s1 = (int)(c1 - (long long)t1 * KS);
        } else {
            tile = t0 + idx - 1;
            s0 = 0;
            s1 = KS;
        }
        ++idx;
    }
    __device__ bool first_of_job() const { return idx == 1; }   // after seg(): the segment just taken was the first
    // slot of this CTA's partial of `tile` (2 per CTA and linear): 0 for its first tile, 1 for its last
    __device__ int slot_of(int tile) const { return tile == t0 ? 0 : 1; }
    // next segment of the chain (crossing linears)
    __device__ bool next(const ChainParams& p, int& job, int& tile, int& s0, int& s1) {
        while (idx >= cnt) {
            if (j + 1 >= n) return false;
            enter(p, j + 1);
        }
        seg(tile, s0, s1);
        job = j;
        return true;
    }
    // next segment of linear jj only (entering it if needed)
    __device__ bool next_in(const ChainParams& p, int jj, int& tile, int& s0, int& s1) {
        if (j != jj) enter(p, jj);
        if (idx >= cnt) return false;
        seg(tile, s0, s1);
        return true;
    }
};

// ------------------------------------------------------------------ in-kernel per-token quantization

__device__ __forceinline__ void red_relaxed_add_gpu(int* p, int v) {
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kQBatch = 4;   // 16-byte row loads per thread in flight

__device__ __forceinline__ uint4 ld_cg_u4(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// The 128 epilogue threads (et) quantize token row m of X (K fp16, row stride ldx) into q_x (row-major,
// row stride ldq) and meta[m] = {s_x fp16 bits, t_x}; bit-identical to quantize_act_kernel (qoq_quant.cuh).
// The codes are built in shared memory and leave by ONE bulk store (+ 16 B of meta); et == 0 owns the
// bulk group and completes it before the caller publishes. K <= kChainQMaxK (host-checked).
__device__ __forceinline__ void quantize_row(const __half* X, int ldx, int K, int m, int8_t* qx, int ldq,
                                             int4* meta, int et, float* redf, int* redi, uint8_t* stg, uint8_t* ystg,
                                             uint64_t* qbar, uint32_t& qph, unsigned long long* tr, size_t trc) {
    const int nv = K / 8;
    // the row through the LSU (all of a thread's loads in flight per batch, L2-coherent: X may be an
    // earlier Y), not the TMA unit, whose queue holds this SM's in-flight weight loads; each thread keeps
    // its own vectors in shared memory for the quantize pass
    uint4* src = reinterpret_cast<uint4*>(stg);
    const uint4* grow = reinterpret_cast<const uint4*>(X + (size_t)m * ldx);
    __half2 a2 = __float2half2_rn(0.0f);
    for (int i0 = et; i0 < nv; i0 += 128 * kQBatch) {
        uint4 v[kQBatch];
#pragma unroll
        for (int u = 0; u < kQBatch; ++u) {
            const int i = i0 + 128 * u;
            if (i < nv) v[u] = ld_cg_u4(grow + i);
        }
#pragma unroll
        for (int u = 0; u < kQBatch; ++u) {
            const int i = i0 + 128 * u;
            if (i < nv) {
                a2 = amax8h(v[u], a2);
                src[i] = v[u];
            }
        }
    }
#if QOQ_TRACING
    if (tr && et == 0) { tr[8] = chain_gtimer(); tr[trc + 8] = clock64(); }
#endif
    float a = amax_of(a2);
    const int g = et >> 5, l = et & 31;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (l == 0) redf[g] = a;
    named_bar_sync(1, 128);
    a = fmaxf(fmaxf(redf[0], redf[1]), fmaxf(redf[2], redf[3]));
    const __half sh = sym_scale(a, 127.0f);
    const float s = __half2float(sh), inv = __frcp_rn(s);
#if QOQ_TRACING
    if (tr && et == 0) { tr[9] = chain_gtimer(); tr[trc + 9] = clock64(); }
#endif
    int t = 0;
    uint2* codes = reinterpret_cast<uint2*>(ystg);
    for (int i = et; i < nv; i += 128) codes[i] = quant8_pe(src[i], s, inv, t);
#if QOQ_TRACING
    if (tr && et == 0) { tr[10] = chain_gtimer(); tr[trc + 10] = clock64(); }
#endif
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) redi[g] = t;
    fence_proxy_async_smem();                 // this thread's codes -> the bulk store
    named_bar_sync(1, 128);
    if (et == 0) {
        int4* ms = reinterpret_cast<int4*>(ystg + K);   // 16-byte meta record after the codes
        *ms = make_int4((int)__half_as_ushort(sh), redi[0] + redi[1] + redi[2] + redi[3], 0, 0);
        fence_proxy_async_smem();
        bulk_s2g(qx + (size_t)m * ldq, ystg, (uint32_t)K);
        bulk_s2g(meta + m, ms, 16u);
        bulk_commit();
    }
}

// Four consecutive outputs Y[m][n..n+3] from INT32 accumulators (biased-u8 MMA: acc − 128 t_x), then
// the s_x s0 outer-product scaling, as two half2.
__device__ __forceinline__ uint2 chain_y4(int4 a, int bias128, float sxf, const float (&s0v)[4]) {
    a.x -= bias128; a.y -= bias128; a.z -= bias128; a.w -= bias128;
    __half2 lo = __halves2half2(__float2half_rn((float)a.x * (sxf * s0v[0])), __float2half_rn((float)a.y * (sxf * s0v[1])));
    __half2 hi = __halves2half2(__float2half_rn((float)a.z * (sxf * s0v[2])), __float2half_rn((float)a.w * (sxf * s0v[3])));
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    return u;
}

// ------------------------------------------------------------------ the kernel

template <int BN>
__global__ void __launch_bounds__(ChainCfg<BN>::kBlockThreads, 1) w4a8_chain_kernel(const __grid_constant__ ChainParams p) {
    using C = ChainCfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* stgb = smem + C::kEpiOff;                                // staging (kStgBytes)
    int32_t* stg = reinterpret_cast<int32_t*>(stgb);
    uint8_t* ystg = stgb + C::kStgBytes;                              // output staging (kYStgBytes)
    float* sxs = reinterpret_cast<float*>(ystg + C::kYStgBytes);
    int* txs = reinterpret_cast<int*>(sxs + BN);
    float* redf = reinterpret_cast<float*>(txs + BN);                // 4 floats
    int* redi = reinterpret_cast<int*>(redf + 4);                    // 4 ints
    uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
    uint64_t* wfree = wfull + C::kWStages;
    uint64_t* xfull = wfree + C::kWStages;
    uint64_t* xempty = xfull + C::kXStages;
    uint64_t* afull = xempty + C::kXStages;
    uint64_t* aempty = afull + C::kAStages;
    uint64_t* accfull = aempty + C::kAStages;
    uint64_t* accempty = accfull + C::kAccStages;
    uint64_t* qbar = accempty + C::kAccStages;                        // staged rows / slices landed (epilogue)
    uint64_t* qready = qbar + 1;                                       // q_x / meta of the next linear acquired
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qready + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int M = p.M;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < C::kWStages; ++i) {
            mbar_init(&wfull[i], 1);
            mbar_init(&wfree[i], 4);
        }
        for (int i = 0; i < C::kXStages; ++i) {
            mbar_init(&xfull[i], 1);
            mbar_init(&xempty[i], 1);
        }
        for (int i = 0; i < C::kAStages; ++i) {
            mbar_init(&afull[i], 4);
            mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < C::kAccStages; ++i) {
            mbar_init(&accfull[i], C::kIssuers);
            mbar_init(&accempty[i], 4);
        }
        mbar_init(qbar, 1);
        mbar_init(qready, 1);
        fence_mbar_init();
        fence_proxy_async_smem();
        for (int i = 0; i < p.nmaps; ++i) prefetch_tmap(&p.tmap[i]);
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ===================== weight producer: every linear's packed steps back to back. Weights are
        // static, so it never waits for activations nor for the previous kernel (PDL).
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();   // each weight byte is read once
            ChainIter ci(p);
            int job, tile, s0, s1, ws = 0, last = -1;
            uint32_t wph = 0;
            while (ci.next(p, job, tile, s0, s1)) {
                const ChainJob& J = p.job[job];
                if (job != last) { QOQ_CTRACE(p, job, 7); last = job; }
                for (int sg = s0; sg < s1; ++sg) {
                    const int kt0 = 2 * sg, nk = (kt0 + 1 < J.KT) ? 2 : 1;
                    mbar_wait(&wfree[ws], wph ^ 1);
                    uint8_t* dst = smem + C::kWOff + ws * C::kWStageBytes;
                    mbar_arrive_expect_tx(&wfull[ws], nk * kTileBytes);
                    bulk_g2s(dst, J.packed + ((size_t)tile * J.KT + kt0) * kTileBytes, nk * kTileBytes, &wfull[ws], pol);
                    if (++ws == C::kWStages) { ws = 0; wph ^= 1; }
                }
            }
        }
    } else if (warp == C::R::kXProdWarp) {
        // ===================== activation producer: TMA 2-D (SWIZZLE_128B) k-tiles of the linear's q_x
        // (rows >= M zero-filled), after its quantization is complete grid-wide (acquire).
        if (lane == 0) {
            pdl_wait();
            ChainIter ci(p);
            int job, tile, s0, s1, xs = 0, cur_job = -1;
            bool xfirst = false;
            uint32_t xph = 0;
            while (ci.next(p, job, tile, s0, s1)) {
                if (job != cur_job) {
                    spin_until_ge_backoff(p.qdone + job, M);
                    fence_proxy_async_global();
                    mbar_arrive(qready);             // the epilogue's s_x / t_x loads (one poller per CTA)
                    cur_job = job;
                    QOQ_CTRACE(p, job, 2);
                    xfirst = true;
                }
                const ChainJob& J = p.job[job];
                const CUtensorMap* tm = &p.tmap[J.tm];
                for (int sg = s0; sg < s1; ++sg) {
                    const int kt0 = 2 * sg, nk = (kt0 + 1 < J.KT) ? 2 : 1;
                    mbar_wait(&xempty[xs], xph ^ 1);
                    mbar_arrive_expect_tx(&xfull[xs], nk * C::kActBytes);
                    uint8_t* dst = smem + C::kXOff + xs * C::kXStageBytes;
                    for (int t = 0; t < nk; ++t) tma_load_2d(dst + t * C::kActBytes, tm, (kt0 + t) * 128, 0, &xfull[xs]);
                    if (xfirst) { QOQ_CTRACE(p, job, 21); xfirst = false; }
                    if (++xs == C::kXStages) { xs = 0; xph ^= 1; }
                }
            }
        }
    } else if (warp == 1 || warp == C::R::kMma1Warp) {
        // ===================== MMA issuers: issuer j takes the chain's steps with global index % 2 == j,
        // both accumulate into the segment's (pre-zeroed) accumulator stage.
        const int j = (warp == 1) ? 0 : 1;
        const uint32_t idesc = idesc_i8(128, BN, /*a_signed=*/false);   // biased-u8 weights (t_x known)
        ChainIter ci(p);
        int job, tile, s0, s1, cst = 0, it0 = 0, last = -1;
        uint32_t cph = 0;
        while (ci.next(p, job, tile, s0, s1)) {
            const int KT = p.job[job].KT;
            mbar_wait(&accempty[cst], cph);
            if (j == 0 && lane == 0 && job != last) { QOQ_CTRACE(p, job, 3); last = job; }
            tc_fence_after();
            const uint32_t d = tmem + C::kAStages * 64 + cst * BN;
            const int first = (j - it0 % C::kIssuers + C::kIssuers) % C::kIssuers;
            for (int local = first; local < s1 - s0; local += C::kIssuers) {
                const int it = it0 + local, sg = s0 + local;
                const int xs = it % C::kXStages, as = it % C::kAStages;
                const uint32_t xph = (uint32_t)(it / C::kXStages) & 1u, aph = (uint32_t)(it / C::kAStages) & 1u;
                const int nk = (2 * sg + 1 < KT) ? 2 : 1;
                const bool first_step = QOQ_TRACING && lane == 0 && local == first && ci.first_of_job();
                mbar_wait(&afull[as], aph);
                if (first_step) QOQ_CTRACE(p, job, 22);
                mbar_wait(&xfull[xs], xph);
                if (first_step) QOQ_CTRACE(p, job, 23);
                tc_fence_after();
                const uint32_t a = tmem + as * 64;
                const uint32_t sb = smem_u32(smem + C::kXOff + xs * C::kXStageBytes);
                if (elect_one()) {
                    for (int t = 0; t < nk; ++t) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_i8_ts(d, a + t * 32 + kk * 8, smem_desc_sw128(sb + t * C::kActBytes + kk * 32), idesc, 1u);
                    }
                    tc_commit(&aempty[as]);
                    tc_commit(&xempty[xs]);
                }
                __syncwarp();
                if (first_step) QOQ_CTRACE(p, job, 24);
            }
            if (elect_one()) tc_commit(&accfull[cst]);
            __syncwarp();
            if (lane == 0) QOQ_CTRACE(p, job, 4);
            it0 += s1 - s0;
            if (++cst == C::kAccStages) { cst = 0; cph ^= 1; }
        }
    } else if (warp >= 2 && warp < C::R::kDeqWarp1) {
        // ===================== dequant: u4 -> (q̂ + 128) lanes -> TMEM (see w4a8_gemm.cu)
        const int q = warp & 3;
        const int grp = (warp - 2) >> 2;
        const int r = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        ChainIter ci(p);
        int job, tile, s0, s1, ws = 0, it = 0, last = -1;
        uint32_t wph = 0;
        while (ci.next(p, job, tile, s0, s1)) {
            const int KT = p.job[job].KT;
            for (int sg = s0; sg < s1; ++sg, ++it) {
                if (it % C::kDeqGroups == grp) {
                    const int nk = (2 * sg + 1 < KT) ? 2 : 1;
                    mbar_wait(&wfull[ws], wph);
                    if (warp == 2 && lane == 0 && job != last) { QOQ_CTRACE(p, job, 6); last = job; }
                    const uint8_t* wb = smem + C::kWOff + ws * C::kWStageBytes;
                    uint4 v[2][4];
                    uint32_t sc[2], bias[2];
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (t < nk) {
                            const uint8_t* w = wb + t * kTileBytes;
                            sc[t] = w[8192 + r];
                            bias[t] = (128u - (uint32_t)w[8320 + r]) * 0x01010101u;
#pragma unroll
                            for (int c = 0; c < 4; ++c) v[t][c] = *reinterpret_cast<const uint4*>(w + c * 2048 + r * 16);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&wfree[ws]);
                    const int as = it % C::kAStages;
                    const uint32_t aph = (uint32_t)(it / C::kAStages) & 1u;
                    mbar_wait(&aempty[as], aph ^ 1);
                    tc_fence_after();
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (t < nk) {
                            uint32_t out[32];
                            expand_row<false>(v[t], sc[t], bias[t], out);
                            tmem_st_32x32b_x32(tmem + lane_off + as * 64 + t * 32, out);
                        }
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&afull[as]);
                }
                if (++ws == C::kWStages) { ws = 0; wph ^= 1; }
            }
        }
    } else if (warp >= C::R::kEpiWarp0 && warp < C::R::kEpiWarp0 + 4) {
        // ===================== epilogue warps: per linear j, (1) quantize this CTA's rows of X_j once
        // Y_{j-1} is complete, (2) write out whole tiles / store partial tiles of this CTA's segments,
        // (3) once all of them are stored, finish this CTA's row slice of each partial tile, (4) publish
        // the finished units. Every cross-CTA write goes out by TMA bulk store; et == 0 owns the bulk
        // groups and completes them before each relaxed publication.
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const int et = threadIdx.x - C::R::kEpiThread0;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        for (int st = 0; st < C::kAccStages; ++st) {
            zero_acc<BN>(tmem + lane_off + C::kAStages * 64 + st * BN);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[st]);
        }
        pdl_wait();
        ChainIter ci(p);
        int cst = 0;
        uint32_t cph = 0, qph = 0, qrph = 0;
        const int myrows = (M > (int)blockIdx.x) ? (M - 1 - (int)blockIdx.x) / p.G + 1 : 0;
        for (int jb = 0; jb < p.njobs; ++jb) {
            const ChainJob& J = p.job[jb];
            const int par = jb & 1;
            // ---- (1) per-token quantization of X_jb, rows m ≡ blockIdx.x (mod G)
            if (myrows > 0) {
                if (et == 0) QOQ_CTRACE(p, jb, 25);
                if (jb > 0) {
                    if (et == 0) spin_until_ge_backoff(p.done + jb - 1, p.job[jb - 1].units);   // Y_{jb-1} complete
                    named_bar_sync(1, 128);
                }
                if (et == 0) QOQ_CTRACE(p, jb, 0);
                for (int m = blockIdx.x; m < M; m += p.G) {
                    if (m != (int)blockIdx.x) {   // the staging areas are reused by the next row
                        if (et == 0) bulk_wait_read<0>();
                        named_bar_sync(1, 128);
                    }
                    quantize_row(J.X, J.ldx, J.K, m, p.qx[par], p.ldq, p.meta[par], et, redf, redi, stgb, ystg, qbar, qph,
                                 QOQ_TRACING && p.trace ? p.trace + ((size_t)jb * p.G + blockIdx.x) * 32 : nullptr,
                                 (size_t)p.njobs * p.G * 32);
                }
                if (et == 0) {
                    QOQ_CTRACE(p, jb, 11);
                    bulk_wait<0>();                    // codes and meta are in global memory
                    red_relaxed_add_gpu(p.qdone + jb, myrows);
                    QOQ_CTRACE(p, jb, 1);
                }
            }
            // ---- (2) this CTA's segments of linear jb
            int tile, s0, s1;
            if (!ci.next_in(p, jb, tile, s0, s1)) continue;
            mbar_wait(qready, qrph);                       // the activation producer acquired qdone[jb] >= M
            qrph ^= 1u;
            for (int jj = et; jj < BN; jj += 128) {
                if (jj < M) {
                    const int4 mt = __ldcg(p.meta[par] + jj);
                    sxs[jj] = __half2float(__ushort_as_half((unsigned short)mt.x));
                    txs[jj] = 128 * mt.y;
                } else {
                    sxs[jj] = 0.0f;
                    txs[jj] = 0;
                }
            }
            int units = 0, npart = 0, seg_no = 0;
            int ptile[2] = {0, 0}, plo[2] = {0, 0}, pcnt[2] = {1, 1};
            int32_t* slots = p.slots[par];
            int* tcnt = p.tilecnt[par];                   // [NT][2]: partials landed, slices finalized
            // ---- (3) once this CTA's partials are in their slots: publish them, then finish this CTA's row
            // slice of each of its partial tiles when all of the tile's contributors have landed theirs.
            // Partial segments are taken first (ChainIter), so this runs before the whole tiles' epilogues,
            // overlapping their main loop.
            bool finished = false;
            auto finish_partials = [&]() {
            if (npart > 0) {
                    if (et == 0) {
                        bulk_wait<0>();                      // this CTA's slot stores (and earlier Y stores) are complete
                        QOQ_CTRACE(p, jb, 18);
                        for (int i = 0; i < npart; ++i) red_relaxed_add_gpu(tcnt + 2 * ptile[i], 1);
                        QOQ_CTRACE(p, jb, 13);
                    }
                    for (int i = 0; i < npart; ++i) {
                        const int t = ptile[i], n0 = t * 128, lo = plo[i], cnt = pcnt[i], idx = (int)blockIdx.x - lo;
                        // this CTA's rows [r0, r1) of the tile, in 32-row blocks (the Y map's box width)
                        const int r0 = 32 * ((4 * idx) / cnt), r1 = 32 * ((4 * (idx + 1)) / cnt);
                        if (et == 0) spin_until_ge_backoff(tcnt + 2 * t, cnt);
                        if (et == 0 && i == 0) QOQ_CTRACE(p, jb, 14);
                        // one round per (token half, 32-row block): the cnt contributors' [32][kPartTok] INT32
                        // blocks -> sum -> fp16 [kPartTok][32] -> one TMA tensor store
#pragma unroll 1
                        for (int rd = 0; rd < (BN / C::kPartTok) * ((r1 - r0) / 32); ++rd) {
                            const int h = (rd / ((r1 - r0) / 32)) * C::kPartTok, rb = r0 + 32 * (rd % ((r1 - r0) / 32));
                            if (et == 0) bulk_wait_read<0>();        // output staging no longer read by a store
                        named_bar_sync(1, 128);                  // staging free (earlier generic reads done)
                        if (et == 0) {
                            fence_proxy_async_smem();
                            fence_proxy_async_global();
                            mbar_arrive_expect_tx(qbar, (uint32_t)(cnt * 32 * C::kPartTok * 4));
                            for (int c = 0; c < cnt; ++c) {
                                const int b = lo + c;
                                // slot of contributor b for tile t: its first tile's, or its last tile's
                                int kk = 0;
                                if (J.S == 0) kk = (t == (int)(((long long)b * J.I / p.G) / J.KS)) ? 0 : 1;
                                const int32_t* sl = slots + (size_t)(2 * b + kk) * 128 * BN + (size_t)h * 128 + (size_t)rb * C::kPartTok;
                                bulk_g2s(stg + c * 32 * C::kPartTok, sl, (uint32_t)(32 * C::kPartTok * 4), qbar, policy_evict_first());
                            }
                        }
                        mbar_wait(qbar, qph);
                        qph ^= 1u;
                        if (et == 0 && i == 0 && rd == 0) QOQ_CTRACE(p, jb, 19);
                        __half* ys = reinterpret_cast<__half*>(ystg);   // [kPartTok tokens][32 rows] fp16
                        for (int w = et; w < 16 * C::kG4; w += 128) {
                            const int rp = w & 15, k = w >> 4;       // row pair, token granule
                            const int row0 = 2 * rp;                 // within the 32-row block
                            int4 a0 = make_int4(0, 0, 0, 0), a1 = make_int4(0, 0, 0, 0);
#pragma unroll 1
                            for (int c = 0; c < cnt; ++c) {
                                const int32_t* sc = stg + c * 32 * C::kPartTok;
                                const int4 x0 = *reinterpret_cast<const int4*>(
                                    sc + row0 * C::kPartTok + 4 * (k ^ ((rb + row0) & (C::kG4 - 1))));
                                const int4 x1 = *reinterpret_cast<const int4*>(
                                    sc + (row0 + 1) * C::kPartTok + 4 * (k ^ ((rb + row0 + 1) & (C::kG4 - 1))));
                                a0.x += x0.x; a0.y += x0.y; a0.z += x0.z; a0.w += x0.w;
                                a1.x += x1.x; a1.y += x1.y; a1.z += x1.z; a1.w += x1.w;
                            }
                            const float2 sf = __half22float2(*reinterpret_cast<const __half2*>(J.s0 + n0 + rb + row0));
                            const int m0 = h + 4 * k;
                            const int e0[4] = {a0.x, a0.y, a0.z, a0.w}, e1[4] = {a1.x, a1.y, a1.z, a1.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const float sx = sxs[m0 + u];
                                const int bias = txs[m0 + u];
                                *reinterpret_cast<__half2*>(ys + (4 * k + u) * 32 + 2 * rp) =
                                    __halves2half2(__float2half_rn((float)(e0[u] - bias) * (sx * sf.x)),
                                                   __float2half_rn((float)(e1[u] - bias) * (sx * sf.y)));
                            }
                        }
                            fence_proxy_async_smem();
                            named_bar_sync(1, 128);
                            if (et == 0) {
                                tma_store_2d(&p.ymap[jb], ys, n0 + rb, h);
                                bulk_commit();
                            }
                        }
                        if (et == 0 && i == 0) QOQ_CTRACE(p, jb, 20);
                        ++units;
                    }
                    if (et == 0) QOQ_CTRACE(p, jb, 15);
                }
                finished = true;
            };
            do {
                const int n0 = tile * 128;
                const bool whole = (s0 == 0 && s1 == J.KS);
                if (whole && npart > 0 && !finished) finish_partials();
                if (et == 0) bulk_wait_read<0>();        // staging areas no longer read by earlier bulk stores
                named_bar_sync(1, 128);
                mbar_wait(&accfull[cst], cph);
                if (et == 0 && seg_no == 0) QOQ_CTRACE(p, jb, 12);
                tc_fence_after();
                const uint32_t d = tmem + lane_off + C::kAStages * 64 + cst * BN;
                if (whole) {
                    // Y[m][n0 + r] for this thread's row r, staged as 4 column blocks [kPartTok tokens][32]
                    // fp16 per token half, then 4 TMA tensor stores (the Y map's box is {32, kPartTok})
                    const float s0r = __half2float(J.s0[n0 + r]);
#pragma unroll 1
                    for (int h = 0; h < BN; h += C::kPartTok) {
                        if (h > 0) {
                            if (et == 0) bulk_wait_read<0>();
                            named_bar_sync(1, 128);
                        }
                        __half* ys = reinterpret_cast<__half*>(ystg);
#pragma unroll 1
                        for (int ch = 0; ch < C::kPartTok / C::kChunk; ++ch) {
                            const int j0 = h + ch * C::kChunk;
                            uint32_t v[C::kChunk];
                            tmem_ld_cols<C::kChunk>(d + j0, v);
                            tmem_wait_ld();
#pragma unroll
                            for (int i = 0; i < C::kChunk; ++i)
                                ys[((r >> 5) * C::kPartTok + (j0 - h + i)) * 32 + (r & 31)] =
                                    __float2half_rn((float)((int)v[i] - txs[j0 + i]) * (sxs[j0 + i] * s0r));
                        }
                        if (h + C::kPartTok >= BN) {              // accumulator fully read: zero it, hand it back
                            zero_acc<BN>(d);
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&accempty[cst]);
                        }
                        fence_proxy_async_smem();
                        named_bar_sync(1, 128);
                        if (et == 0) {
                            for (int cb = 0; cb < 4; ++cb) tma_store_2d(&p.ymap[jb], ys + cb * C::kPartTok * 32, n0 + 32 * cb, h);
                            bulk_commit();
                        }
                    }
                    ++units;
                } else {
                    // stage the partial tile [row][token] (kPartTok tokens at a time) and store it to this
                    // CTA's slot (first or later segment of the linear) with ONE bulk copy per staging; the
                    // slot needs no zeroing (the finalizers sum the tile's slots)
                    int32_t* wst = slots + (size_t)(2 * blockIdx.x + ci.slot_of(tile)) * 128 * BN;
#pragma unroll 1
                    for (int h = 0; h < BN; h += C::kPartTok) {
                        if (h > 0) {
                            if (et == 0) bulk_wait_read<0>();
                            named_bar_sync(1, 128);
                        }
#pragma unroll 1
                        for (int ch = 0; ch < C::kPartTok / C::kChunk; ++ch) {
                            const int j0 = h + ch * C::kChunk;
                            uint32_t v[C::kChunk];
                            tmem_ld_cols<C::kChunk>(d + j0, v);
                            tmem_wait_ld();
                            // row r of the slot: kG4 granules of 4 tokens, granule k at k ^ (r mod kG4)
                            // (conflict-free shared stores; the finalizers undo it)
#pragma unroll
                            for (int k4 = 0; k4 < C::kChunk / 4; ++k4) {
                                const int k = (j0 - h) / 4 + k4;
                                *reinterpret_cast<int4*>(stg + r * C::kPartTok + 4 * (k ^ (r & (C::kG4 - 1)))) =
                                    make_int4((int)v[4 * k4], (int)v[4 * k4 + 1], (int)v[4 * k4 + 2], (int)v[4 * k4 + 3]);
                            }
                        }
                        if (h + C::kPartTok >= BN) {              // accumulator fully read
                            zero_acc<BN>(d);
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&accempty[cst]);
                        }
                        fence_proxy_async_smem();
                        if (et == 0) QOQ_CTRACE(p, jb, 16);
                        named_bar_sync(1, 128);
                        if (et == 0) {
                            bulk_s2g(wst + (size_t)h * 128, stg, C::kPartTok * 128 * 4);   // [h / 64][row][64 tokens]
                            bulk_commit();
                            QOQ_CTRACE(p, jb, 17);
                        }
                    }
                    // the tile's contributors: CTAs lo .. lo + cnt - 1
                    int cnt, lo;
                    if (J.S > 0) {
                        cnt = J.S;
                        lo = tile * J.S;
                    } else {
                        lo = streamk_owner((long long)tile * J.KS, J.I, p.G);
                        cnt = streamk_owner((long long)(tile + 1) * J.KS - 1, J.I, p.G) - lo + 1;
                    }
                    ptile[npart] = tile;
                    plo[npart] = lo;
                    pcnt[npart] = cnt;
                    ++npart;
                }
                ++seg_no;
                if (++cst == C::kAccStages) { cst = 0; cph ^= 1; }
            } while (ci.next_in(p, jb, tile, s0, s1));
            if (!finished) finish_partials();
            // ---- (4) publish this CTA's finished units of linear jb once its Y stores are complete
            if (et == 0) {
                bulk_wait<0>();
                QOQ_CTRACE(p, jb, 5);
                if (units > 0) red_relaxed_add_gpu(p.done + jb, units);
                // off the critical path: the last finalizer of each partial tile resets its counters (reused
                // by linear jb + 2, which starts long after every contributor of jb has passed its wait)
                for (int i = 0; i < npart; ++i)
                    if (atomicAdd(tcnt + 2 * ptile[i] + 1, 1) == pcnt[i] - 1) {
                        tcnt[2 * ptile[i]] = 0;
                        tcnt[2 * ptile[i] + 1] = 0;
                    }
            }
        }
        if (et == 0) bulk_wait<0>();
    }

    tc_fence_before();
    __syncthreads();
    pdl_launch_dependents();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, C::kTmemCols);
    }
    // the last CTA out re-zeroes the grid counters for the next launch (graph replay): every CTA
    // arrives only after all of its own waits on them are over
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p.exitcnt, 1) == p.G - 1) {
            for (int i = 0; i < p.njobs; ++i) {
                p.qdone[i] = 0;
                p.done[i] = 0;
            }
            __threadfence();
            *p.exitcnt = 0;
        }
    }
}

// ------------------------------------------------------------------ host side

int chain_bn(int M) { return M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : 128; }

template <int BN>
static cudaError_t launch_chain_bn(const ChainParams& p, cudaStream_t st) {
    using C = ChainCfg<BN>;
    auto kern = w4a8_chain_kernel<BN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.G);
    cfg.blockDim = dim3(C::kBlockThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t launch_w4a8_chain(const ChainParams& p, cudaStream_t st) {
    switch (chain_bn(p.M)) {
        case 16: return launch_chain_bn<16>(p, st);
        case 32: return launch_chain_bn<32>(p, st);
        case 64: return launch_chain_bn<64>(p, st);
        case 128: return launch_chain_bn<128>(p, st);
        default: return cudaErrorInvalidValue;
    }
}

int chain_block_threads(int M) {
    switch (chain_bn(M)) {
        case 16: return ChainCfg<16>::kBlockThreads;
        case 32: return ChainCfg<32>::kBlockThreads;
        case 64: return ChainCfg<64>::kBlockThreads;
        default: return ChainCfg<128>::kBlockThreads;
    }
}

}  // namespace qoq
