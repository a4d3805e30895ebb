// qoq_api.cu — the C-ABI shim (include/qoq_b200.h): host-side validation, planning and launch.
// No allocation, no device synchronization, no mutable global state (a resolved driver entry
// point is cached in w4a8_gemm.cu).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <memory>

#include "../../include/qoq_b200.h"
#include "qoq_internal.h"

namespace qoq {

static Knobs read_knobs() {
    Knobs k;
    auto get = [](const char* n, int def) { const char* e = getenv(n); return e ? atoi(e) : def; };
    k.force_mode = get("QOQ_FORCE_MODE", -1);
    k.bn_big = get("QOQ_BN_BIG", 0);
    k.force_cg = get("QOQ_FORCE_CG", -1);
    k.linear_fused = get("QOQ_LINEAR_FUSED", 0);
    k.chain_smax = get("QOQ_CHAIN_SMAX", 0);
    k.fq_threads = get("QOQ_FQ_THREADS", 0);
    return k;
}
static Knobs g_knobs = read_knobs();   // process start (the library's load)
const Knobs& knobs() { return g_knobs; }
void reload_knobs() { g_knobs = read_knobs(); }

}  // namespace qoq

namespace {

using namespace qoq;

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int check_arch(int* num_sms) {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return QOQ_ERR_CUDA;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
        return QOQ_ERR_CUDA;
    if (major != 10 || minor != 0) return QOQ_ERR_ARCH;
    if (num_sms && cudaDeviceGetAttribute(num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return QOQ_ERR_CUDA;
    return QOQ_OK;
}

int gemm_shape_status(int M, int N, int K, int group) {
    if (M < 0 || N <= 0 || K <= 0) return QOQ_ERR_INVALID_ARG;
    if (group != 128) return QOQ_ERR_UNSUPPORTED;
    if (N % kTileN != 0 || K % kTileK != 0) return QOQ_ERR_SHAPE;
    if (K > 65536) return QOQ_ERR_SHAPE;   // INT32 headroom of the biased-u8 accumulation
    return QOQ_OK;
}

int num_sms_or_default() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

int run_gemm(const int8_t* qx, const void* sx, const int32_t* tx, const void* packed, const void* s0,
             int M, int N, int K, int group, void* out, int ldo, bool out_i32,
             void* ws, size_t ws_bytes, cudaStream_t st, void* trace = nullptr, const uint8_t* zw = nullptr,
             bool pc = false) {
    int rc = gemm_shape_status(M, N, K, group);
    if (rc) return rc;
    if (M == 0) return QOQ_OK;
    if (!qx || !packed || !out || (!out_i32 && (!sx || !s0))) return QOQ_ERR_INVALID_ARG;
    // per-channel W4A8: t_x (the zero-point term) and the 4-byte-aligned zero points are required
    if (pc && (!tx || !zw || (reinterpret_cast<uintptr_t>(zw) & 3u))) return QOQ_ERR_INVALID_ARG;
    if (!aligned16(qx) || !aligned16(packed) || ldo < N) return QOQ_ERR_INVALID_ARG;
    // vectorized epilogue: 4 consecutive outputs per store, 8-byte aligned s0 loads
    if (ldo % 4 != 0 || !aligned16(out) || (!out_i32 && !aligned16(s0))) return QOQ_ERR_INVALID_ARG;
    int sms = 0;
    if ((rc = check_arch(&sms))) return rc;
    GemmPlan p = plan_gemm(M, N, K, sms);
    if (p.ws_bytes > 0 && (!ws || ws_bytes < p.ws_bytes || !aligned16(ws))) return QOQ_ERR_WORKSPACE;
    if (pc && p.CG != 1) return QOQ_ERR_UNSUPPORTED;   // the CTA-pair variant is g128 only
    GemmArgs a{qx, sx, tx, packed, s0, out, ldo, out_i32, M, N, K, p.ws_bytes ? ws : nullptr, trace};
    a.zw = pc ? zw : nullptr;
    return launch_w4a8_gemm(a, p, st, /*pdl=*/true) == cudaSuccess ? QOQ_OK : QOQ_ERR_CUDA;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// qoq_w4a8_linear workspace: [qsync 2 x int32][GEMM workspace][q_x M*K][s_x 2M][t_x 4M], 256-B aligned.
// The parts that must be zero at entry (sync words, split-K partials) come first, at offsets that do not
// depend on K, so a workspace shared by several shapes keeps its sync words at offset 0.
struct LinearWs {
    int* qsync;
    int8_t* qx;
    void* sx;
    int32_t* tx;
    void* gemm_ws;
    size_t gemm_ws_bytes, total;
};

LinearWs linear_ws_layout(void* base, int M, int N, int K) {
    LinearWs w{};
    uint8_t* b = static_cast<uint8_t*>(base);
    size_t off = 0;
    w.qsync = reinterpret_cast<int*>(b + off);  off += 256;
    w.gemm_ws_bytes = plan_gemm(M, N, K, num_sms_or_default()).ws_bytes;
    w.gemm_ws = b + off;                         off += align_up(w.gemm_ws_bytes, 256);
    w.qx = reinterpret_cast<int8_t*>(b + off);  off += align_up((size_t)M * K, 256);
    w.sx = b + off;                              off += align_up((size_t)M * 2, 256);
    w.tx = reinterpret_cast<int32_t*>(b + off); off += align_up((size_t)M * 4, 256);
    w.total = off;
    return w;
}

int run_linear(const void* X, int ldx, int M, int N, int K, int group, const void* packed, const void* s0,
               void* Y, int ldy, void* ws, size_t ws_bytes, cudaStream_t st, void* trace = nullptr) {
    int rc = gemm_shape_status(M, N, K, group);
    if (rc) return rc;
    if (ldx < K || ldx % 8 || ldy < N) return QOQ_ERR_INVALID_ARG;
    if (M == 0) return QOQ_OK;
    if (!X || !aligned16(X) || !packed || !s0 || !Y || !ws) return QOQ_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return QOQ_ERR_INVALID_ARG;
    LinearWs w = linear_ws_layout(ws, M, N, K);
    if (ws_bytes < w.total) return QOQ_ERR_WORKSPACE;
    // Default: quantizer kernel + GEMM, PDL-chained (measured faster on B200 at every decode M: the
    // fused kernel's grid-wide handshake costs more than the kernel boundary it removes).
    // QOQ_LINEAR_FUSED=1 selects the one-kernel path for M <= kFuseMaxM.
    const bool fused = knobs().linear_fused == 1;
    // the split-K region must be zero on entry; in a workspace shared by several shapes it may overlap
    // another shape's q_x, so the call clears it itself (mode-1 plans only: none at decode sizes)
    if (w.gemm_ws_bytes > 0 && cudaMemsetAsync(w.gemm_ws, 0, w.gemm_ws_bytes, st) != cudaSuccess) return QOQ_ERR_CUDA;
    if (M > kFuseMaxM || !fused) {
        if ((rc = qoq_quantize_activations_per_token(X, M, K, ldx, w.qx, w.sx, w.tx, st))) return rc;
        return run_gemm(w.qx, w.sx, w.tx, packed, s0, M, N, K, group, Y, ldy, false, w.gemm_ws, w.gemm_ws_bytes,
                        st);
    }
    if (ldy % 4 != 0 || !aligned16(Y) || !aligned16(s0) || !aligned16(packed)) return QOQ_ERR_INVALID_ARG;
    int sms = 0;
    if ((rc = check_arch(&sms))) return rc;
    GemmPlan p = plan_gemm(M, N, K, sms);
    GemmArgs a{w.qx, w.sx, w.tx, packed, s0, Y, ldy, false, M, N, K, p.ws_bytes ? w.gemm_ws : nullptr, trace};
    a.X = X;
    a.ldx = ldx;
    a.qsync = w.qsync;
    return launch_w4a8_gemm(a, p, st, /*pdl=*/true) == cudaSuccess ? QOQ_OK : QOQ_ERR_CUDA;
}

}  // namespace

extern "C" {

const char* qoq_status_string(int s) {
    switch (s) {
        case QOQ_OK: return "ok";
        case QOQ_ERR_INVALID_ARG: return "invalid argument";
        case QOQ_ERR_SHAPE: return "unsupported shape (N, K must be multiples of 128; K <= 65536)";
        case QOQ_ERR_UNSUPPORTED: return "unsupported configuration (group must be 128)";
        case QOQ_ERR_ARCH: return "device is not sm_100 (B200)";
        case QOQ_ERR_WORKSPACE: return "workspace or output buffer too small";
        case QOQ_ERR_CUDA: return "CUDA error";
        default: return "unknown status";
    }
}

int qoq_abi_version(void) { return QOQ_ABI_VERSION; }

size_t qoq_packed_weight_bytes(int N, int K, int group) {
    if (group != 128 || N <= 0 || K <= 0 || N % kTileN || K % kTileK) return 0;
    return (size_t)(N / kTileN) * (size_t)(K / kTileK) * kTileBytes;
}

int qoq_quantize_weights(const void* W, int N, int K, int group, void* packed, size_t packed_bytes, void* s0,
                         void* stream) {
    if (group != 128) return QOQ_ERR_UNSUPPORTED;
    if (N <= 0 || K <= 0) return QOQ_ERR_INVALID_ARG;
    if (N % kTileN || K % kTileK) return QOQ_ERR_SHAPE;
    if (!W || !packed || !s0 || !aligned16(W) || !aligned16(packed)) return QOQ_ERR_INVALID_ARG;
    if (packed_bytes < qoq_packed_weight_bytes(N, K, group)) return QOQ_ERR_WORKSPACE;
    int rc = check_arch(nullptr);
    if (rc) return rc;
    return launch_quantize_weights(W, N, K, packed, s0, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? QOQ_OK : QOQ_ERR_CUDA;
}

int qoq_quantize_activations_per_token(const void* X, int M, int K, int ldx, int8_t* qx, void* sx, int32_t* tx,
                                       void* stream) {
    if (M < 0 || K <= 0 || ldx < K) return QOQ_ERR_INVALID_ARG;
    if (K % 8 || ldx % 8) return QOQ_ERR_SHAPE;
    if (M == 0) return QOQ_OK;
    if (!X || !qx || !sx || !aligned16(X) || (reinterpret_cast<uintptr_t>(qx) & 7u)) return QOQ_ERR_INVALID_ARG;
    int rc = check_arch(nullptr);
    if (rc) return rc;
    return launch_quantize_activations(X, M, K, ldx, qx, sx, tx, static_cast<cudaStream_t>(stream), true) ==
                   cudaSuccess ? QOQ_OK : QOQ_ERR_CUDA;
}

int qoq_rmsnorm_quantize(const void* X, int ldx, const void* gamma, double eps, int M, int K, int8_t* qx,
                         void* sx, int32_t* tx, void* stream) {
    if (M < 0 || K <= 0 || K > 65536 || ldx < K || !(eps >= 0.0) || eps > 1e300) return QOQ_ERR_INVALID_ARG;
    if (K % 8 || ldx % 8) return QOQ_ERR_SHAPE;
    if (M == 0) return QOQ_OK;
    if (!X || !gamma || !qx || !sx || !aligned16(X) || !aligned16(gamma) || (reinterpret_cast<uintptr_t>(qx) & 7u))
        return QOQ_ERR_INVALID_ARG;
    int rc = check_arch(nullptr);
    if (rc) return rc;
    return launch_rmsnorm_quantize(X, ldx, gamma, eps, M, K, qx, sx, tx, static_cast<cudaStream_t>(stream), true) ==
                   cudaSuccess ? QOQ_OK : QOQ_ERR_CUDA;
}

int qoq_silu_mul_quantize(const void* gate, const void* up, int ldg, int M, int K, int8_t* qx, void* sx,
                          int32_t* tx, void* stream) {
    if (M < 0 || K <= 0 || ldg < K) return QOQ_ERR_INVALID_ARG;
    if (K % 8 || ldg % 8) return QOQ_ERR_SHAPE;
    if (M == 0) return QOQ_OK;
    if (!gate || !up || !qx || !sx || !aligned16(gate) || !aligned16(up) || (reinterpret_cast<uintptr_t>(qx) & 7u))
        return QOQ_ERR_INVALID_ARG;
    int rc = check_arch(nullptr);
    if (rc) return rc;
    return launch_silu_mul_quantize(gate, up, ldg, M, K, qx, sx, tx, static_cast<cudaStream_t>(stream), true) ==
                   cudaSuccess ? QOQ_OK : QOQ_ERR_CUDA;
}

size_t qoq_kv4_page_bytes(int H_kv, int D, int page_size) {
    if (H_kv <= 0 || D != 128 || page_size <= 0) return 0;
    return (size_t)H_kv * page_size * (D + 8);
}

namespace {
int kv4_shape_status(int B, int H, int H_kv, int D, int P) {
    if (B < 0 || H <= 0 || H_kv <= 0 || P <= 0) return QOQ_ERR_INVALID_ARG;
    if (D != 128) return QOQ_ERR_UNSUPPORTED;
    if (H % H_kv) return QOQ_ERR_SHAPE;
    const int r = H / H_kv;
    if (r != 1 && r != 2 && r != 4 && r != 8) return QOQ_ERR_UNSUPPORTED;
    if (P % 32 || P > 256) return QOQ_ERR_UNSUPPORTED;   // 32/r-token chunks within a page; 3 page stages in smem
    return QOQ_OK;
}
}  // namespace

int qoq_kv4_append(const void* K, const void* V, const int32_t* slots, int B, int H_kv, int D, int page_size,
                   void* pages, void* stream) {
    int rc = kv4_shape_status(B, H_kv, H_kv, D, page_size);
    if (rc) return rc;
    if (B == 0) return QOQ_OK;
    if (!K || !V || !slots || !pages || !aligned16(K) || !aligned16(V) || !aligned16(pages)) return QOQ_ERR_INVALID_ARG;
    if ((rc = check_arch(nullptr))) return rc;
    return launch_kv4_append(K, V, slots, B, H_kv, page_size, static_cast<uint8_t*>(pages),
                             static_cast<cudaStream_t>(stream)) == cudaSuccess ? QOQ_OK : QOQ_ERR_CUDA;
}

int qoq_kv4_decode_attention(const void* Q, const void* pages, const int32_t* block_table, const int32_t* seq_lens,
                             int B, int H, int H_kv, int D, int page_size, int max_pages, void* O, void* stream) {
    int rc = kv4_shape_status(B, H, H_kv, D, page_size);
    if (rc) return rc;
    if (max_pages <= 0) return QOQ_ERR_INVALID_ARG;
    if (B == 0) return QOQ_OK;
    if (!Q || !pages || !block_table || !seq_lens || !O || !aligned16(Q) || !aligned16(O) || !aligned16(pages))
        return QOQ_ERR_INVALID_ARG;
    if ((rc = check_arch(nullptr))) return rc;
    return launch_kv4_decode_attention(Q, static_cast<const uint8_t*>(pages), block_table, seq_lens, B, H, H_kv,
                                       page_size, max_pages, O, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? QOQ_OK : QOQ_ERR_CUDA;
}

size_t qoq_gemm_workspace_bytes(int M, int N, int K) {
    if (gemm_shape_status(M, N, K, 128) != QOQ_OK || M == 0) return 0;
    return plan_gemm(M, N, K, num_sms_or_default()).ws_bytes;
}

int qoq_w4a8_gemm(const int8_t* qx, const void* sx, const int32_t* tx, const void* packed, const void* s0, int M,
                  int N, int K, int group, void* Y, int ldy, void* ws, size_t ws_bytes, void* stream) {
    if (ldy < N) return QOQ_ERR_INVALID_ARG;
    return run_gemm(qx, sx, tx, packed, s0, M, N, K, group, Y, ldy, false, ws, ws_bytes,
                    static_cast<cudaStream_t>(stream));
}

int qoq_w4a8_gemm_i32(const int8_t* qx, const int32_t* tx, const void* packed, int M, int N, int K, int group,
                      int32_t* acc, int ldacc, void* ws, size_t ws_bytes, void* stream) {
    if (ldacc < N) return QOQ_ERR_INVALID_ARG;
    return run_gemm(qx, nullptr, tx, packed, nullptr, M, N, K, group, acc, ldacc, true, ws, ws_bytes,
                    static_cast<cudaStream_t>(stream));
}

// ---- fused TP reduction of row-parallel partials (NEXT-3)

size_t qoq_tp_recv_bytes(int world, int m_cap, int n_cap) {
    if (world < 1 || world > QOQ_TP_MAX_WORLD || m_cap < 1 || n_cap < 128 || n_cap % 128) return 0;
    return 2 * (size_t)world * m_cap * n_cap * 4;   // 8-byte words of two fp16 + a 32-bit flag
}

// The fused-reduction plan: whole tiles (mode 0, single CTAs), token tile by M alone (16 / 32 / 64 / 128),
// so every rank of a TP group runs the same tiles with the same CTAs.
GemmPlan tp_plan(int M, int N, int K, int sms) {
    GemmPlan p = plan_gemm(M < 128 ? M : 128, N, K, sms);
    p.MT = (M + p.BN - 1) / p.BN;
    p.MB = p.MT;
    p.T = p.MT * p.NT;
    p.I = (long long)p.T * p.KS;
    p.mode = 0;
    p.S = 1;
    p.CG = 1;
    p.G = p.T < sms ? p.T : sms;
    p.ws_bytes = 0;
    return p;
}

static_assert(QOQ_TP_MAX_WORLD == kTpMaxWorld, "TP world");

int qoq_w4a8_gemm_allreduce(const int8_t* qx, const void* sx, const int32_t* tx, const void* packed, const void* s0,
                            int M, int N, int K, int group, void* Y, int ldy, const qoq_tp_comm* comm, void* stream) {
    int rc = gemm_shape_status(M, N, K, group);
    if (rc) return rc;
    if (!comm || comm->world < 1 || comm->world > QOQ_TP_MAX_WORLD || comm->rank < 0 || comm->rank >= comm->world)
        return QOQ_ERR_INVALID_ARG;
    if (!comm->gen || !comm->done || !comm->status) return QOQ_ERR_INVALID_ARG;
    for (int q = 0; q < comm->world; ++q)
        if (!comm->recv[q] || !aligned16(comm->recv[q])) return QOQ_ERR_INVALID_ARG;
    if (M > comm->m_cap || N > comm->n_cap || comm->n_cap % 128) return QOQ_ERR_INVALID_ARG;
    if (M == 0) return QOQ_OK;
    if (!qx || !sx || !packed || !s0 || !Y || ldy < N || ldy % 4 || !aligned16(Y) || !aligned16(qx) ||
        !aligned16(packed) || !aligned16(s0))
        return QOQ_ERR_INVALID_ARG;
    int sms = 0;
    if ((rc = check_arch(&sms))) return rc;
    // whole tiles only (mode 0, single CTAs): the reduction is per output tile, in the tile's epilogue
    const GemmPlan p = tp_plan(M, N, K, sms);
    TpComm c{};
    for (int q = 0; q < comm->world; ++q) c.recv[q] = comm->recv[q];
    c.gen = comm->gen;
    c.done = comm->done;
    c.status = comm->status;
    c.rank = comm->rank;
    c.world = comm->world;
    c.m_cap = comm->m_cap;
    c.n_cap = comm->n_cap;
    GemmArgs a{qx, sx, tx, packed, s0, Y, ldy, false, M, N, K, nullptr, nullptr};
    a.tp = &c;
    return launch_w4a8_gemm(a, p, static_cast<cudaStream_t>(stream), /*pdl=*/true) == cudaSuccess ? QOQ_OK
                                                                                                 : QOQ_ERR_CUDA;
}

size_t qoq_linear_workspace_bytes(int M, int N, int K) {
    if (gemm_shape_status(M, N, K, 128) != QOQ_OK) return 0;
    return linear_ws_layout(nullptr, M, N, K).total;
}

int qoq_w4a8_linear(const void* X, int ldx, int M, int N, int K, int group, const void* packed, const void* s0,
                    void* Y, int ldy, void* ws, size_t ws_bytes, void* stream) {
    return run_linear(X, ldx, M, N, K, group, packed, s0, Y, ldy, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

// ---- per-channel W4A8 (NEXT-1, §5.2.2)

size_t qoq_pc_packed_weight_bytes(int N, int K) {
    if (N <= 0 || K <= 0 || N % kTileN || K % kTileK) return 0;
    return (size_t)(N / kTileN) * (size_t)(K / kTileK) * kPcTileBytes;
}

int qoq_pc_quantize_weights(const void* W, int N, int K, void* packed, size_t packed_bytes, void* s_w,
                            uint8_t* z_w, void* stream) {
    if (N <= 0 || K <= 0) return QOQ_ERR_INVALID_ARG;
    if (N % kTileN || K % kTileK) return QOQ_ERR_SHAPE;
    if (!W || !packed || !s_w || !z_w || !aligned16(W) || !aligned16(packed)) return QOQ_ERR_INVALID_ARG;
    if (packed_bytes < qoq_pc_packed_weight_bytes(N, K)) return QOQ_ERR_WORKSPACE;
    int rc = check_arch(nullptr);
    if (rc) return rc;
    return launch_pc_quantize_weights(W, N, K, packed, s_w, z_w, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? QOQ_OK : QOQ_ERR_CUDA;
}

int qoq_pc_w4a8_gemm(const int8_t* qx, const void* sx, const int32_t* tx, const void* packed, const void* s_w,
                     const uint8_t* z_w, int M, int N, int K, void* Y, int ldy, void* ws, size_t ws_bytes,
                     void* stream) {
    if (ldy < N) return QOQ_ERR_INVALID_ARG;
    return run_gemm(qx, sx, tx, packed, s_w, M, N, K, 128, Y, ldy, false, ws, ws_bytes,
                    static_cast<cudaStream_t>(stream), nullptr, z_w, true);
}

int qoq_pc_w4a8_gemm_i32(const int8_t* qx, const int32_t* tx, const void* packed, const uint8_t* z_w, int M,
                         int N, int K, int32_t* acc, int ldacc, void* ws, size_t ws_bytes, void* stream) {
    if (ldacc < N) return QOQ_ERR_INVALID_ARG;
    return run_gemm(qx, nullptr, tx, packed, nullptr, M, N, K, 128, acc, ldacc, true, ws, ws_bytes,
                    static_cast<cudaStream_t>(stream), nullptr, z_w, true);
}

// Debug (not in the public header): re-read the QOQ_* test / tuning overrides from the environment.
void qoq_debug_reload_knobs(void) { reload_knobs(); }

// Debug (not in the public header): the fp16 GEMM with a per-CTA %globaltimer trace
// (16 x u64 per CTA, grid <= #SMs) for pipeline timeline analysis (tools/trace_gemm.py).
int qoq_debug_w4a8_gemm_trace(const int8_t* qx, const void* sx, const int32_t* tx, const void* packed,
                              const void* s0, int M, int N, int K, void* Y, void* ws, size_t ws_bytes,
                              void* trace, void* stream) {
    return run_gemm(qx, sx, tx, packed, s0, M, N, K, 128, Y, N, false, ws, ws_bytes,
                    static_cast<cudaStream_t>(stream), trace);
}

// Debug (not in the public header): qoq_w4a8_linear with the same per-CTA trace.
int qoq_debug_w4a8_linear_trace(const void* X, int M, int N, int K, const void* packed, const void* s0, void* Y,
                                void* ws, size_t ws_bytes, void* trace, void* stream) {
    return run_linear(X, K, M, N, K, 128, packed, s0, Y, N, ws, ws_bytes, static_cast<cudaStream_t>(stream), trace);
}

// scratch layout: [linear workspace][X fp16 M*K][Y fp16 M*N], each 256-B aligned (the zero-required
// sync words sit at offset 0 whatever the shape)
size_t qoq_linear_host_scratch_bytes(int M, int N, int K) {
    if (gemm_shape_status(M, N, K, 128) != QOQ_OK) return 0;
    return align_up(qoq_linear_workspace_bytes(M, N, K), 256) + align_up((size_t)M * K * 2, 256) + (size_t)M * N * 2;
}

int qoq_linear_host(const void* X_host, int M, int K, const void* packed, const void* s0, int N, void* Y_host,
                    void* scratch, size_t scratch_bytes, void* stream) {
    int rc = gemm_shape_status(M, N, K, 128);
    if (rc) return rc;
    if (M == 0) return QOQ_OK;
    if (!X_host || !Y_host || !packed || !s0 || !scratch || (reinterpret_cast<uintptr_t>(scratch) & 255u))
        return QOQ_ERR_INVALID_ARG;
    if (scratch_bytes < qoq_linear_host_scratch_bytes(M, N, K)) return QOQ_ERR_WORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* b = static_cast<uint8_t*>(scratch);
    void* ws = b;                b += align_up(qoq_linear_workspace_bytes(M, N, K), 256);
    void* Xd = b;                b += align_up((size_t)M * K * 2, 256);
    void* Yd = b;
    if (cudaMemcpyAsync(Xd, X_host, (size_t)M * K * 2, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return QOQ_ERR_CUDA;
    if ((rc = run_linear(Xd, K, M, N, K, 128, packed, s0, Yd, N, ws, qoq_linear_workspace_bytes(M, N, K), st)))
        return rc;
    if (cudaMemcpyAsync(Y_host, Yd, (size_t)M * N * 2, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return QOQ_ERR_CUDA;
    return QOQ_OK;
}

}  // extern "C"

// ---- decode chain (w4a8_chain.cu)

namespace {

struct ChainWs {
    int* exitcnt;
    int* qdone;
    int* done;
    int* tilecnt[2];
    int32_t* slots[2];
    int8_t* qx[2];
    int4* meta[2];
    int ldq;
    size_t total;
};

// [exitcnt 256 B][qdone 256 x 4][done 256 x 4][tilecnt x2 [512][2]] (a FIXED head of kChainCounterBytes:
// the only part that must be zero, left zero by every call, so one workspace serves any chain) |
// partial slots x2 [2 G][BN][128] i32 | q_x x2 [M][ldq] | meta x2 [M][16 B], 256-B aligned parts.
ChainWs chain_ws_layout(void* base, int M, int n, const qoq_linear_desc* d, int sms) {
    ChainWs w{};
    int kmax = 128;
    for (int j = 0; j < n; ++j) kmax = d[j].K > kmax ? d[j].K : kmax;
    const int BN = chain_bn(M);
    w.ldq = kmax;
    uint8_t* b = static_cast<uint8_t*>(base);
    w.exitcnt = reinterpret_cast<int*>(b);
    w.qdone = reinterpret_cast<int*>(b + 256);
    w.done = reinterpret_cast<int*>(b + 256 + 4 * kChainMaxJobs);
    for (int i = 0; i < 2; ++i)
        w.tilecnt[i] = reinterpret_cast<int*>(b + 256 + 8 * kChainMaxJobs + (size_t)i * kChainMaxNT * 8);
    size_t off = kChainCounterBytes;
    for (int i = 0; i < 2; ++i) { w.slots[i] = reinterpret_cast<int32_t*>(b + off); off += (size_t)2 * sms * BN * 128 * 4; }
    for (int i = 0; i < 2; ++i) { w.qx[i] = reinterpret_cast<int8_t*>(b + off); off += align_up((size_t)M * kmax, 256); }
    for (int i = 0; i < 2; ++i) { w.meta[i] = reinterpret_cast<int4*>(b + off); off += align_up((size_t)M * 16, 256); }
    w.total = off;
    return w;
}

int chain_desc_status(int M, int n, const qoq_linear_desc* d) {
    if (M < 1 || M > kChainMaxM || n < 1 || n > kChainMaxJobs || !d) return QOQ_ERR_INVALID_ARG;
    for (int j = 0; j < n; ++j) {
        int rc = gemm_shape_status(M, d[j].N, d[j].K, 128);
        if (rc) return rc;
        if (d[j].N > kChainMaxNT * kTileN || d[j].K > kChainQMaxK) return QOQ_ERR_SHAPE;
        if (d[j].ldx < d[j].K || d[j].ldx % 8 || d[j].ldy < d[j].N || d[j].ldy % 8) return QOQ_ERR_INVALID_ARG;
        if (!d[j].X_fp16 || !d[j].packed || !d[j].s0_fp16 || !d[j].Y_fp16) return QOQ_ERR_INVALID_ARG;
        if (!aligned16(d[j].X_fp16) || !aligned16(d[j].packed) || !aligned16(d[j].s0_fp16) || !aligned16(d[j].Y_fp16))
            return QOQ_ERR_INVALID_ARG;
    }
    return QOQ_OK;
}

}  // namespace

extern "C" {

size_t qoq_linear_chain_workspace_bytes(int M, int n, const qoq_linear_desc* desc) {
    if (chain_desc_status(M, n, desc) != QOQ_OK) return 0;
    return chain_ws_layout(nullptr, M, n, desc, num_sms_or_default()).total;
}

static int run_chain(int M, int n, const qoq_linear_desc* desc, void* workspace, size_t workspace_bytes,
                     void* stream, void* trace) {
    int rc = chain_desc_status(M, n, desc);
    if (rc) return rc;
    if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255u)) return QOQ_ERR_INVALID_ARG;
    ChainWs w = chain_ws_layout(workspace, M, n, desc, num_sms_or_default());
    if (workspace_bytes < w.total) return QOQ_ERR_WORKSPACE;
    int sms = 0;
    if ((rc = check_arch(&sms))) return rc;
    if (sms != num_sms_or_default()) return QOQ_ERR_CUDA;
    std::unique_ptr<ChainParams> pp(new ChainParams());   // ~16 KB of launch parameters (host heap)
    const int chain_s_cap = knobs().chain_smax;             // tuning: cap on the k-splits per tile
    ChainParams& p = *pp;
    p.M = M;
    p.njobs = n;
    p.G = sms;
    for (int i = 0; i < 2; ++i) {
        p.qx[i] = w.qx[i];
        p.meta[i] = w.meta[i];
        p.slots[i] = w.slots[i];
        p.tilecnt[i] = w.tilecnt[i];
    }
    p.ldq = w.ldq;
    auto enc = tensor_map_encoder();
    if (!enc) return QOQ_ERR_CUDA;
    int map_par[kChainMaxMaps], map_k[kChainMaxMaps];
    p.nmaps = 0;
    p.qdone = w.qdone;
    p.done = w.done;
    p.exitcnt = w.exitcnt;
    p.trace = static_cast<unsigned long long*>(trace);
    for (int j = 0; j < n; ++j) {
        ChainJob& J = p.job[j];
        J.packed = static_cast<const uint8_t*>(desc[j].packed);
        J.s0 = static_cast<const __half*>(desc[j].s0_fp16);
        J.X = static_cast<const __half*>(desc[j].X_fp16);
        J.Y = static_cast<__half*>(desc[j].Y_fp16);
        J.ldx = desc[j].ldx;
        J.ldy = desc[j].ldy;
        J.K = desc[j].K;
        J.KT = desc[j].K / kTileK;
        J.KS = (J.KT + 1) / 2;
        J.NT = desc[j].N / kTileN;
        J.I = (long long)J.NT * J.KS;
        // the TMA map of this linear's q_x: (parity, K) -> dims {K, M}, box {128, BN}, SWIZZLE_128B
        J.tm = -1;
        for (int i = 0; i < p.nmaps; ++i)
            if (map_par[i] == (j & 1) && map_k[i] == J.K) J.tm = i;
        if (J.tm < 0) {
            if (p.nmaps == kChainMaxMaps) return QOQ_ERR_UNSUPPORTED;
            const int i = p.nmaps++;
            map_par[i] = j & 1;
            map_k[i] = J.K;
            cuuint64_t dims[2] = {(cuuint64_t)J.K, (cuuint64_t)M};
            cuuint64_t strides[1] = {(cuuint64_t)w.ldq};
            cuuint32_t box[2] = {128u, (cuuint32_t)chain_bn(M)};
            cuuint32_t estr[2] = {1u, 1u};
            if (enc(&p.tmap[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, w.qx[j & 1], dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return QOQ_ERR_CUDA;
            J.tm = i;
        }
        // decode-sized linears (fewer tiles than SMs): S equal k-splits per tile, one segment per CTA;
        // otherwise stream-K over all CTAs (no wave quantization)
        // (at most 4 splits: a finalizer stages every contributor's 32-row block of its slice in 32 KB)
        J.S = J.NT < sms ? std::min(std::min(sms / J.NT, J.KS), 4) : 0;
        if (J.S > 0 && chain_s_cap > 0) J.S = std::min(J.S, chain_s_cap);
        {   // the TMA map of Y_j: dims {N, M} fp16, row stride ldy, box {32, min(BN, 64)}
            cuuint64_t dims[2] = {(cuuint64_t)desc[j].N, (cuuint64_t)M};
            cuuint64_t strides[1] = {(cuuint64_t)desc[j].ldy * 2};
            cuuint32_t box[2] = {32u, (cuuint32_t)std::min(chain_bn(M), 64)};
            cuuint32_t estr[2] = {1u, 1u};
            if (enc(&p.ymap[j], CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, desc[j].Y_fp16, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return QOQ_ERR_CUDA;
        }
        if (J.S > 0) {
            J.units = J.NT * J.S;
        } else {   // (CTA, segment) pairs of the stream-K split
            long long units = 0;
            for (int b = 0; b < sms; ++b) {
                const long long c0 = (long long)b * J.I / sms, c1 = (long long)(b + 1) * J.I / sms;
                if (c1 > c0) units += (c1 - 1) / J.KS - c0 / J.KS + 1;
            }
            J.units = (int)units;
        }
    }
    return launch_w4a8_chain(p, static_cast<cudaStream_t>(stream)) == cudaSuccess ? QOQ_OK : QOQ_ERR_CUDA;
}

int qoq_w4a8_linear_chain(int M, int n, const qoq_linear_desc* desc, void* workspace, size_t workspace_bytes,
                          void* stream) {
    return run_chain(M, n, desc, workspace, workspace_bytes, stream, nullptr);
}

// Debug (not in the public header): the chain with a [n][G][8] u64 %globaltimer trace (trace builds).
int qoq_debug_w4a8_linear_chain_trace(int M, int n, const qoq_linear_desc* desc, void* workspace,
                                      size_t workspace_bytes, void* trace, void* stream) {
    return run_chain(M, n, desc, workspace, workspace_bytes, stream, trace);
}

}  // extern "C"
