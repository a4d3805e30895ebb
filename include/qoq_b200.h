/* qoq_b200.h — C ABI of the B200-native (sm_100a) QoQ W4A8 hot path of QServe (arXiv 2405.04532).
 *
 * The problem statement this library implements, PAPER.md P:407 (§5.1): "All GEMM layers in
 * QServe operate on W4A8 inputs, perform computation on INT8 tensor cores, and generate FP16
 * outputs." Weights are progressively group-quantized (§4.1; g = 128 per P:814);
 * activations are quantized per token, symmetric INT8 (§6.1).
 *
 * Conventions (every entry point):
 *   - Pointers are DEVICE pointers unless the name ends in _host. All buffers are caller-owned;
 *     the library never allocates, never synchronizes the device, and keeps no mutable global
 *     state. Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).
 *   - fp16 buffers are IEEE binary16 (void* to stay free of CUDA headers).
 *   - Arguments are validated on the host, synchronously; on failure nothing is launched and a
 *     qoq_status != QOQ_OK is returned. A launch failure returns QOQ_ERR_CUDA. Faults inside a
 *     kernel surface as CUDA errors at the caller's next synchronization. Nothing throws.
 *   - Device buffers must be 16-byte aligned. Requires an sm_100 device (else QOQ_ERR_ARCH).
 *   - Inputs containing NaN/Inf are a precondition violation (results unspecified).
 */
#ifndef QOQ_B200_H
#define QOQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    QOQ_OK = 0,
    QOQ_ERR_INVALID_ARG = 1,  /* null pointer, misalignment, negative size, ldx < K, ...      */
    QOQ_ERR_SHAPE = 2,        /* N or K not a multiple of 128, K too large for INT32 headroom */
    QOQ_ERR_UNSUPPORTED = 3,  /* group != 128                                                 */
    QOQ_ERR_ARCH = 4,         /* current device is not sm_100                                 */
    QOQ_ERR_WORKSPACE = 5,    /* workspace / packed buffer smaller than required             */
    QOQ_ERR_CUDA = 6          /* a CUDA runtime call or kernel launch failed                 */
} qoq_status;

/* Static description of a status code; never NULL. */
const char* qoq_status_string(int status);
/* ABI version of this header (incremented on any signature or layout change). */
int qoq_abi_version(void);
#define QOQ_ABI_VERSION 7

/* ----------------------------------------------------------------------------------------------
 * Packed weight layout (frozen). The B200 form of "store the weights in the order
 * they are used during computation" (§5.2.1) with the register-level-parallel nibble
 * interleave w0,w16,w1,w17,... (§5.2.2, Fig. 9):
 *   tiles of 128 output channels x 128 input channels (= one group), n-tile-major:
 *   tile(nt, j) starts at byte (nt*(K/128) + j) * 8448;
 *   bytes [0, 8192): q_u4; chunk c = 0..3 covers k = 128j+32c .. +31; row r (0..127) of chunk c
 *                    is at c*2048 + r*16; byte b (0..15) = q[r][32c+b] | q[r][32c+16+b] << 4;
 *   bytes [8192, 8320): s_u8[r]       (level-2 group scale)
 *   bytes [8320, 8448): zs_u8[r] = z_u4 * s_u8  (precomputed zero term; <= 126 by the
 *                                   protective range)
 * -------------------------------------------------------------------------------------------- */

/* Bytes of the packed weight stream for an [N][K] weight; 0 if the shape is unsupported
 * (group != 128, N or K not a positive multiple of 128). */
size_t qoq_packed_weight_bytes(int N, int K, int group);

/* Offline weight quantization + packing (P:238-275 levels 1 and 2; P:434/P:447 layout).
 *   W        [N][K] fp16 row-major (nn.Linear layout: Y = X W^T).
 *   packed   out, qoq_packed_weight_bytes(N,K,group) bytes (packed_bytes must be >= that).
 *   s0_fp16  out, [N] level-1 per-channel scales s0 = fp16(max_k|W[n,k]| / 119).
 * Level 1: q8 = clamp(round_half_away(W / s0), -119, 119) (protective range).
 * Level 2 (per 128-group): s_u8 = max(1, ⌈(hi-lo)/15⌋), z = clamp(⌈-lo/s_u8⌋, 0, 15),
 *          q_u4 = clamp(⌈(q8 + z s_u8)/s_u8⌋, 0, 15) (Eq. 2 P:111-116 with q_min=0, q_max=15). */
int qoq_quantize_weights(const void* W_fp16, int N, int K, int group,
                         void* packed, size_t packed_bytes, void* s0_fp16, void* stream);

/* Per-token symmetric INT8 activation quantization (symmetric form P:132).
 *   X_fp16  [M][ldx] fp16 (ldx >= K, ldx % 8 == 0; lets a TP rank quantize a K-shard view).
 *   qx      out [M][K] int8 (contiguous), q = clamp(round_half_away(x / s_x), -127, 127).
 *   sx_fp16 out [M], s_x = fp16(max_k|X[m,k]| / 127); 1.0 for an all-zero row.
 *   tx      out [M] int32 row sums Σ_k qx (nullable). Lets the GEMM feed biased-u8 weights.
 * Requires K % 8 == 0. M == 0 is a no-op. */
int qoq_quantize_activations_per_token(const void* X_fp16, int M, int K, int ldx,
                                       int8_t* qx, void* sx_fp16, int32_t* tx, void* stream);

/* Scratch needed by qoq_w4a8_gemm / qoq_w4a8_gemm_i32 for this shape (split-K INT32 partials and
 * per-tile arrival counters). The workspace must be ZERO-FILLED before its first use; every
 * successful call leaves it zero-filled again. One workspace per concurrently running stream. */
size_t qoq_gemm_workspace_bytes(int M, int N, int K);

/* The W4A8 per-group GEMM with progressive dequantization (§5.2):
 *   Y[m][n] = fp16( s_x[m] * s0[n] * Σ_k qx[m][k] * q̂[n][k] ),  q̂ = (q_u4 - z) * s_u8 ∈ INT8,
 * with q_u4 expanded to INT8 in registers, contracted on tcgen05 INT8 tensor
 * cores with INT32 accumulation in tensor memory, scaled in the epilogue.
 *   qx [M][K] int8, sx_fp16 [M], tx [M] int32 or NULL (if given, must equal Σ_k qx[m][k]).
 *   packed / s0_fp16 from qoq_quantize_weights.  Y_fp16 [M][ldy], ldy >= N, ldy % 4 == 0.
 * Requires group == 128, N % 128 == 0, K % 128 == 0, K <= 65536. M == 0 is a no-op. */
int qoq_w4a8_gemm(const int8_t* qx, const void* sx_fp16, const int32_t* tx,
                  const void* packed, const void* s0_fp16,
                  int M, int N, int K, int group,
                  void* Y_fp16, int ldy,
                  void* workspace, size_t workspace_bytes, void* stream);

/* Parity/debug entry: the same main loop; the epilogue writes the exact INT32 accumulators
 * acc[m][n] = Σ_k qx[m][k] * q̂[n][k] (bias-corrected) into acc [M][ldacc] (ldacc % 4 == 0). */
int qoq_w4a8_gemm_i32(const int8_t* qx, const int32_t* tx, const void* packed,
                      int M, int N, int K, int group,
                      int32_t* acc, int ldacc,
                      void* workspace, size_t workspace_bytes, void* stream);

/* The W4A8 linear layer on fp16 activations: per-token INT8 quantization of X (exactly
 * qoq_quantize_activations_per_token) followed by the W4A8 GEMM (exactly qoq_w4a8_gemm), so
 *   Y = qoq_w4a8_gemm(quantize(X))  bit for bit.
 * By default it launches the quantizer kernel and then the GEMM (PDL-chained). With the
 * environment variable QOQ_LINEAR_FUSED=1 and M <= 64 both run in ONE kernel instead: the GEMM's
 * epilogue warps quantize rows m ≡ cta (mod grid) into the workspace while the weight stream is
 * already in flight, and a grid handshake in the workspace releases the activation loads
 * (measured slower on B200 than the two-kernel chain, hence opt-in).
 *   X_fp16 [M][ldx] (ldx >= K, ldx % 8 == 0, 16-byte aligned).  packed / s0_fp16 from
 *   qoq_quantize_weights.  Y_fp16 [M][ldy], ldy >= N, ldy % 4 == 0.
 * workspace: qoq_linear_workspace_bytes(M,N,K) bytes, 256-byte aligned, ZERO-FILLED before first
 * use; each call leaves its synchronization words and split-K partials zeroed again. Layout, each
 * part 256-byte aligned: [256 B sync][GEMM workspace, qoq_gemm_workspace_bytes(M,N,K)]
 * [q_x int8 M*K][s_x fp16 M][t_x int32 M]; after the call q_x / s_x / t_x hold this call's
 * quantized activations. One workspace per stream; it may be reused for any shape: when the GEMM
 * needs split-K partials (qoq_gemm_workspace_bytes > 0) the call first clears that region with an
 * async memset on `stream` (it may overlap another shape's q_x), so only the 256 sync bytes must be
 * zero on entry.
 * Same shape requirements as qoq_w4a8_gemm. */
size_t qoq_linear_workspace_bytes(int M, int N, int K);
int qoq_w4a8_linear(const void* X_fp16, int ldx, int M, int N, int K, int group,
                    const void* packed, const void* s0_fp16,
                    void* Y_fp16, int ldy,
                    void* workspace, size_t workspace_bytes, void* stream);

/* End-to-end linear layer with HOST activations (the e2e measurement path): copies X_host
 * (pinned host memory, [M][K] fp16) to the device, runs qoq_w4a8_linear against device-resident
 * packed weights and copies Y back to Y_host ([M][N] fp16, pinned).
 * dev_scratch: qoq_linear_host_scratch_bytes(M,N,K) bytes of device memory (256-byte aligned),
 * zero-filled before first use. Layout: [linear workspace][X M*K fp16][Y M*N fp16], so the
 * workspace rules of qoq_w4a8_linear (including reuse across shapes) apply to it. Asynchronous
 * on `stream`. */
size_t qoq_linear_host_scratch_bytes(int M, int N, int K);
int qoq_linear_host(const void* X_host_fp16, int M, int K,
                    const void* packed, const void* s0_fp16, int N,
                    void* Y_host_fp16, void* dev_scratch, size_t scratch_bytes, void* stream);

/* ---- Decode chain: n linear layers in ONE persistent launch (ABI v6) ----
 * The decode-regime form of the whole hot path (SURVEY §8(a) rows a2-a7 for a sequence of linears):
 * for j = 0 .. n-1, in order, exactly what qoq_w4a8_linear computes,
 *   Y_j = fp16( (Σ_k q̂_j[n][k] q_x[m][k]) · s_x[m] · s0_j[n] ),  q_x, s_x = per-token INT8 of X_j,
 * bit-identical to n successive qoq_w4a8_linear calls. Linear j reads X_j only after Y_0..Y_{j-1} are
 * complete, so X_j may be (a view of) an earlier linear's Y, as in a model. One CTA per SM streams
 * every linear's packed weights back to back; each linear's K-steps are split over all SMs (stream-K,
 * P:501) with exact INT32 partial sums reduced in L2; the per-token quantization runs inside the
 * kernel between linears. DESIGN.md §5.
 *   desc[j]: X_fp16 [M][ldx] (ldx >= K, ldx % 8 == 0), packed / s0_fp16 as qoq_w4a8_gemm for an [N][K]
 *            weight, Y_fp16 [M][ldy] (ldy >= N, ldy % 8 == 0). The descriptor array is read on the host
 *            during the call (the launch captures it by value; it may be freed on return).
 *   M:       1 .. 128 tokens (the decode regime; above, use the per-GEMM path).
 *   n:       1 .. 128 linears (one launch; split longer stacks into several chains).
 *   workspace: qoq_linear_chain_workspace_bytes(M, n, desc) bytes, 256-byte aligned. Only its first
 *            12288 bytes (grid counters) must be ZERO before the first use; every call leaves them zero
 *            again, so a workspace can be reused (and graph-replayed) by later calls with any
 *            descriptors (if large enough), one call at a time. The rest (split-K partial slots, the
 *            q_x, s_x, t_x) needs no initialization. N <= 65536 and K <= 14336 per linear (else
 *            QOQ_ERR_SHAPE); at most 16 distinct (K, j % 2) pairs per chain (else QOQ_ERR_UNSUPPORTED).
 * Requires the whole GPU: the grid is one CTA per SM and all CTAs must be co-resident (grid-wide
 * release/acquire counters order the linears). Errors: as qoq_w4a8_gemm per descriptor; M or n out of
 * range -> QOQ_ERR_INVALID_ARG; workspace too small -> QOQ_ERR_WORKSPACE. Launches 1 kernel. */
typedef struct {
    const void* X_fp16;
    int ldx;
    int N, K;
    const void* packed;
    const void* s0_fp16;
    void* Y_fp16;
    int ldy;
} qoq_linear_desc;

size_t qoq_linear_chain_workspace_bytes(int M, int n, const qoq_linear_desc* desc);
int qoq_w4a8_linear_chain(int M, int n, const qoq_linear_desc* desc, void* workspace, size_t workspace_bytes,
                          void* stream);

/* ---- Per-channel W4A8 (the paper's other precision mode, §5.2.2; NEXT-1) ----
 * Weights: per-output-channel asymmetric UINT4 (Eq. 2, q_min = 0, q_max = 15) with an
 * FP16 scale s_w[n] and a u8 zero point z_w[n] in [0,15]; no level-2 parameters. The GEMM unpacks
 * the codes in the main loop (lanes = q_u4, unsigned 8-bit MMA operand) and applies the zero point
 * AFTER the multiplication, in the epilogue (exact t_x = Σ_k q_x, Q19):
 *   Y[m][n] = fp16( s_x[m] · s_w[n] · (Σ_k q_x[m][k] q_u4[n][k] − z_w[n] · t_x[m]) ).
 * Packed layout: the tile stream above without the 256 level-2 bytes (8192-byte tiles).
 * Shapes and errors as qoq_quantize_weights / qoq_w4a8_gemm; t_x is REQUIRED (the quantizer's row
 * sums) and z_w must be 4-byte aligned, else QOQ_ERR_INVALID_ARG. Workspace: qoq_gemm_workspace_bytes.
 * W [N][K] fp16; s_w_fp16 [N] and z_w [N] are outputs of the packer, inputs of the GEMM. */
size_t qoq_pc_packed_weight_bytes(int N, int K);
int qoq_pc_quantize_weights(const void* W_fp16, int N, int K, void* packed, size_t packed_bytes,
                            void* s_w_fp16, uint8_t* z_w, void* stream);
int qoq_pc_w4a8_gemm(const int8_t* qx, const void* sx_fp16, const int32_t* tx, const void* packed,
                     const void* s_w_fp16, const uint8_t* z_w, int M, int N, int K,
                     void* Y_fp16, int ldy, void* workspace, size_t workspace_bytes, void* stream);
/* parity entry: the exact INT32 Σ_k q_x (q_u4 − z_w) into acc [M][ldacc] (ldacc % 4 == 0) */
int qoq_pc_w4a8_gemm_i32(const int8_t* qx, const int32_t* tx, const void* packed, const uint8_t* z_w,
                         int M, int N, int K, int32_t* acc, int ldacc,
                         void* workspace, size_t workspace_bytes, void* stream);

/* ---- Activation quantization fused into the producing layer (NEXT-2) ----
 * P:410 (§5.1, Fig. 7): "we fuse activation quantization into the preceding layernorm for
 * the QKV projection and the first FFN layer, or into the preceding activation kernel for the second
 * FFN layer". Each call writes exactly what qoq_quantize_activations_per_token would write for the
 * layer's fp16 output (Q23), without that output being stored:
 *
 * qoq_rmsnorm_quantize — Llama RMSNorm before qkv / gate_up (Q23-Q25):
 *   y[m][k] = fp16_rn((x[m][k] · r_m) · gamma[k]) in fp64, r_m = 1 / sqrt(S_m / K + eps) in fp64,
 *   S_m = Σ_k x[m][k]² summed EXACTLY and rounded once (r is independent of reduction order);
 *   S_m / K + eps == 0 gives r_m = 0. Then q_x, s_x, t_x of y as in the per-token quantizer.
 *   X_fp16 [M][ldx] (ldx >= K, ldx % 8 == 0), gamma_fp16 [K], eps >= 0 finite (Llama: 1e-5); K <= 65536.
 * qoq_silu_mul_quantize — the FFN activation before down (Q24, Q26):
 *   h[m][k] = fp16_rn(silu(g) · u), silu(g) = g / (1 + exp(-g)) in fp64, g = gate[m][k], u = up[m][k];
 *   gate_fp16 / up_fp16 [M][ldg] (e.g. the fused gate_up GEMM output: up = gate + K, ldg = 2K).
 * Outputs (both): qx [M][K] int8 (8-byte aligned), sx_fp16 [M], tx [M] int32 row sums (nullable).
 * Requires K % 8 == 0, 16-byte aligned fp16 inputs. M == 0 is a no-op. Errors as
 * qoq_quantize_activations_per_token (QOQ_ERR_INVALID_ARG also for a negative / non-finite eps). */
int qoq_rmsnorm_quantize(const void* X_fp16, int ldx, const void* gamma_fp16, double eps, int M, int K,
                         int8_t* qx, void* sx_fp16, int32_t* tx, void* stream);
int qoq_silu_mul_quantize(const void* gate_fp16, const void* up_fp16, int ldg, int M, int K,
                          int8_t* qx, void* sx_fp16, int32_t* tx, void* stream);

/* ---- KV4 cache and decode attention (NEXT-4; §5.3; Q27-Q29) ----
 * "per-head asymmetric INT4 quantization on KV cache", "FP16 scaling factors and zero points for
 * each head immediately following the quantized KV features in each KV cache page".
 * Page (one layer, page_size P tokens, all H_kv heads; D must be 128): per kv head g, at byte g*P*(D+8):
 *   K codes [P][D/2] (byte j = q[2j] | q[2j+1] << 4), V codes [P][D/2], K (s, z) fp16 pairs [P],
 *   V (s, z) fp16 pairs [P]. Token t of a sequence lives in page block_table[t / P], slot t % P.
 * Quantization of each (token, head) row: the per-channel rule of qoq_pc_quantize_weights
 *   (s = fp16(fp32(max - min) / 15), z = clamp(⌈-min/s⌋, 0, 15) stored as fp16, q = clamp(⌈x/s + z⌋, 0, 15)).
 * qoq_kv4_page_bytes: H_kv * P * (D + 8); 0 if unsupported. page_size must be a multiple of 32, at most 256 (64 typical).
 * qoq_kv4_append: K_fp16, V_fp16 [B][H_kv][D] (one new token per sequence); slots [B] int32 (device) =
 *   page * P + offset of each sequence's new token; pages: the page pool (device, 16-byte aligned).
 * qoq_kv4_decode_attention: O[b][h] = softmax(Q[b][h] · K̂ᵀ / sqrt(D)) · V̂ over the first seq_lens[b] tokens
 *   of sequence b, kv head h / (H / H_kv) (H / H_kv in {1, 2, 4, 8}); fp32 arithmetic, fp16 output.
 *   Q_fp16, O_fp16 [B][H][D]; block_table [B][max_pages] int32; seq_lens [B] int32 (device; a length
 *   <= 0 gives zeros; lengths must not exceed max_pages * P).
 * Errors: D != 128, page_size % 32 != 0 or > 256, or an unsupported H / H_kv -> QOQ_ERR_UNSUPPORTED; H % H_kv -> QOQ_ERR_SHAPE;
 * null / misaligned pointers, non-positive sizes -> QOQ_ERR_INVALID_ARG. B == 0 is a no-op. */
size_t qoq_kv4_page_bytes(int H_kv, int D, int page_size);
int qoq_kv4_append(const void* K_fp16, const void* V_fp16, const int32_t* slots, int B, int H_kv, int D,
                   int page_size, void* pages, void* stream);
int qoq_kv4_decode_attention(const void* Q_fp16, const void* pages, const int32_t* block_table,
                             const int32_t* seq_lens, int B, int H, int H_kv, int D, int page_size, int max_pages,
                             void* O_fp16, void* stream);

/* ----------------------------------------------------------------------------------------------
 * Fused tensor-parallel reduction of a row-parallel linear (NEXT-3; ABI v7). The north_star's
 * Megatron split: o_proj / down are row-sharded over K, and Y = Σ_r Y_r over the TP ranks, where rank r's
 * partial is Y_r = fp16(acc_r · s_x^r · s0) of its K shard (reading Q17; the paper itself is single-GPU,
 * P:754). qoq_w4a8_gemm_allreduce computes Y_r tile by tile (whole 128-row tiles) and, in the same
 * kernel's epilogue, PUSHES each fp16 partial tile into slot `rank` of every rank's receive buffer (peer
 * stores over NVLink), then writes
 *     Y[m][n] = fp16( Σ_{q = 0 .. world-1} fp32(Y_q[m][n]) )      summed in rank order (reading Q32)
 * from its own buffer as the peers' words arrive, so every rank ends with identical bits and the transfer
 * of one tile overlaps the math of the others. Slots hold 8-byte words {two fp16, uint32 flag}; a word is
 * valid when its flag equals this call's number (no fences, no counters).
 *
 * qoq_tp_comm (host struct, read during the call; every pointer is a DEVICE pointer):
 *   recv[q] (q < world) rank q's receive buffer, a device pointer valid on this GPU (peer-mapped, e.g.
 *          symmetric memory): qoq_tp_recv_bytes(world, m_cap, n_cap) bytes ([2 parities][world slots][m_cap]
 *          [n_cap / 2] words), 16-byte aligned, zero-initialized once; entries >= world are ignored;
 *   gen, done  one uint32 each (this rank's call counter and CTA exit counter), zero-initialized once;
 *   status one int32, zero-initialized; set to 1 if a wait for a peer exceeded 2 s (the call then gives up
 *          and Y is unspecified) — check it after synchronizing;
 *   rank, world (1 .. QOQ_TP_MAX_WORLD), m_cap >= M, n_cap >= N (n_cap % 128 == 0).
 * Every rank must issue the same sequence of qoq_w4a8_gemm_allreduce calls (same M, N) on its own GPU with
 * the same comm layout; the buffers alternate by call parity, so no barrier is needed between calls.
 * world == 1 is valid (the push and the wait are local; Y equals qoq_w4a8_gemm bit for bit).
 * Other arguments and errors as qoq_w4a8_gemm (tx nullable); comm / capacity violations ->
 * QOQ_ERR_INVALID_ARG. Launches 1 kernel. Ownership: the caller allocates and shares the buffers; the
 * library only reads and writes them inside the kernel. */
#define QOQ_TP_MAX_WORLD 8
typedef struct {
    void* recv[QOQ_TP_MAX_WORLD];
    uint32_t* gen;
    uint32_t* done;
    int32_t* status;
    int rank, world;
    int m_cap, n_cap;
} qoq_tp_comm;
size_t qoq_tp_recv_bytes(int world, int m_cap, int n_cap);
int qoq_w4a8_gemm_allreduce(const int8_t* qx, const void* sx_fp16, const int32_t* tx, const void* packed,
                            const void* s0_fp16, int M, int N, int K, int group, void* Y_fp16, int ldy,
                            const qoq_tp_comm* comm, void* stream);

/* Kernels launched per successful call (launch accounting for benchmarks):
 * quantize_weights 2, quantize_activations_per_token 1, rmsnorm_quantize 1, silu_mul_quantize 1,
 * kv4_append 1, kv4_decode_attention 1, w4a8_gemm 1, w4a8_gemm_i32 1,
 * pc_quantize_weights 2, pc_w4a8_gemm 1, pc_w4a8_gemm_i32 1,
 * w4a8_linear 2 (1 when fused: QOQ_LINEAR_FUSED=1 and M <= 64), linear_host as w4a8_linear,
 * w4a8_linear_chain 1 (for the whole chain), w4a8_gemm_allreduce 1
 * (plus 2 async copies). */

#ifdef __cplusplus
}
#endif
#endif /* QOQ_B200_H */
