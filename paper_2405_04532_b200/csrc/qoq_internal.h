// qoq_internal.h — host-side declarations shared by the C-ABI shim (qoq_api.cu) and the kernel
// translation units. Not part of the public ABI (that is include/qoq_b200.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
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

// Debug / test overrides of the planner and of the linear path, read from the environment ONCE (first use)
// and re-read only by qoq_debug_reload_knobs() (the Python binding calls it when a QOQ_* variable it
// forwards changes, so pytest's monkeypatch works). Production launches never call getenv.
struct Knobs {
    int force_mode = -1;     // QOQ_FORCE_MODE: 0 / 1 / 2
    int bn_big = 0;          // QOQ_BN_BIG: 128 / 192 / 256 (prefill token tile)
    int force_cg = -1;       // QOQ_FORCE_CG: 2 = CTA pairs (slower, opt-in)
    int linear_fused = 0;    // QOQ_LINEAR_FUSED: 1 = the one-kernel linear for M <= 64 (slower, opt-in)
    int chain_smax = 0;      // QOQ_CHAIN_SMAX: cap on the decode chain's k-splits per tile (tuning)
    int fq_threads = 0;      // QOQ_FQ_THREADS: fused quantizer threads per row (tuning)
};
const Knobs& knobs();
void reload_knobs();

// Device-side view of qoq_tp_comm (include/qoq_b200.h): every rank pushes its fp16 partial of each whole
// output tile into slot `rank` of every rank's receive buffer (flag-in-data words), then reduces its own
// slots 0 .. world-1 in rank order (fp32) as their words arrive.
constexpr int kTpMaxWorld = 8;
struct TpComm {
    void* recv[kTpMaxWorld]; // rank q's receive buffer [2][world][m_cap][n_cap/2] 8-B words (kernel parameter)
    uint32_t* gen;           // this rank's count of completed fused calls (parity; flag = gen + 1)
    uint32_t* done;          // CTA exit counter of the running call
    int32_t* status;         // 1 after a peer wait timed out
    int rank, world, m_cap, n_cap;
};

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
    // fused TP reduction of row-parallel partials (NEXT-3; qoq_w4a8_gemm_allreduce): nullptr = off
    const TpComm* tp = nullptr;
};


constexpr int kFuseMaxM = 64;   // above: quantizer kernel + GEMM (the prologue would serialize M rows)

cudaError_t launch_w4a8_gemm(const GemmArgs& a, const GemmPlan& p, cudaStream_t st, bool pdl);
// cuTensorMapEncodeTiled through the runtime's driver entry point (nullptr if unavailable)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
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

// Persistent decode chain (w4a8_chain.cu): n W4A8 linear layers in one launch, M <= 128.
constexpr int kChainMaxJobs = 128;    // (one 128-byte Y tensor map per linear in the ~28 KB of parameters)
constexpr int kChainMaxM = 128;
constexpr int kChainMaxNT = 512;        // N <= 65536 per linear
constexpr int kChainQMaxK = 14336;      // K per linear (the in-kernel quantizer stages one row in SMEM)
constexpr int kChainCounterBytes = 12288;   // fixed-size zero-required head of the chain workspace
constexpr int kChainMaxMaps = 16;      // distinct (parity, K) activation tensor maps per chain
struct ChainJob {            // one linear layer (host-planned)
    const uint8_t* packed;   // tile stream [NT][KT][8448]
    const __half* s0;        // [N]
    const __half* X;         // input [M][ldx] fp16 (may be an earlier job's Y)
    __half* Y;               // output [M][ldy] fp16 (ldy % 8 == 0: 16-byte TMA store runs)
    int ldx, ldy, K, KT, KS, NT;
    int S;                   // k-splits per tile (NT < G: CTA b -> tile b / S), 0 = stream-K over all CTAs
    int units;               // (CTA, segment) pairs: the job is complete when done[j] reaches it
    int tm;                  // index of the TMA map of its q_x (parity j & 1, this K)
    long long I;             // NT * KS pipeline steps
};
struct ChainParams {
    CUtensorMap ymap[kChainMaxJobs];   // Y_j maps: dims {N, M} fp16, row stride ldy, box {32, min(BN, 64)}
    CUtensorMap tmap[kChainMaxMaps];   // q_x maps: dims {K, M}, row stride ldq, box {128, BN}, SWIZZLE_128B
    int M, njobs, G, nmaps;  // tokens, linears, CTAs (one per SM), maps
    int ldq;                 // q_x row stride (bytes)
    int8_t* qx[2];           // q_x [M][ldq] int8 (job parity)
    int4* meta[2];           // [M] {s_x fp16 bits, t_x, 0, 0}
    int32_t* slots[2];       // split-K partial tiles, one slot per (CTA, first/last segment): [2G][BN][128] int32
    int* tilecnt[2];         // per tile: partials landed, slices finalized [kChainMaxNT][2] (zero between uses)
    int* qdone;              // [njobs] rows quantized (zero at launch, re-zeroed at exit)
    int* done;               // [njobs] units complete
    int* exitcnt;            // CTAs finished
    unsigned long long* trace;   // debug (QOQ_TRACING builds): [njobs][G][32] stamps x2, else null
    ChainJob job[kChainMaxJobs];
};
int chain_bn(int M);
int chain_block_threads(int M);
cudaError_t launch_w4a8_chain(const ChainParams& p, cudaStream_t st);

}  // namespace qoq
