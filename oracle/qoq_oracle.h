/* qoq_oracle.h — CPU oracle for the QoQ W4A8 hot path of QServe (arXiv 2405.04532).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path (include/qoq_b200.h,
 * paper_2405_04532_b200/) never includes, links or calls anything here, and this oracle
 * shares no code, header, table or constant generator with it.
 *
 * Citations: "P:n" = line n of the paper's LaTeX source, with its section/equation.
 * Readings of silent/ambiguous passages are numbered Q1..Q26 as in DESIGN.md §3.
 *
 * fp16 values are carried as raw IEEE binary16 bit patterns (uint16_t).
 * All functions return 0 on success, a negative value on a precondition failure.
 */
#ifndef QOQ_ORACLE_H
#define QOQ_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* IEEE binary16 <-> binary32. f2h rounds to nearest, ties to even (Q8, Q10). */
float    oracle_h2f(uint16_t h);
uint16_t oracle_f2h_rn(float f);
uint16_t oracle_d2h_rn(double f);   /* binary64 -> binary16, one RNE rounding (Q24) */

/* Round half away from zero of the integer quotient a/b, b > 0 (Q1: the paper's ⌈·⌋). */
int      oracle_rhai(int a, int b);

/* O1 — level-1 progressive quantization, per output channel, symmetric INT8 into the
 * protective range [-119, 119]. Eq. (progressive_quant:int8); range P:257-275.
 * W: [N][K] fp16 (nn.Linear layout, Q9). q8: [N][K] int8 out. s0: [N] fp16 out. */
int oracle_level1(const uint16_t* W, int N, int K, int8_t* q8, uint16_t* s0);

/* O2 — level-2 progressive quantization of ONE group of g level-1 codes: per-group
 * asymmetric UINT4 with an unsigned 8-bit integer scale. Eq. (progressive_quant:int4)
 * P:247-253 with Eq. 2 at q_min = 0, q_max = 15; worked example P:257.
 * Writes qu4[g] in [0,15], *s_u8 >= 1, *z in [0,15]. */
int oracle_level2_group(const int8_t* q8, int g, uint8_t* qu4, uint8_t* s_u8, uint8_t* z);

/* O2 over a whole [N][K] level-1 tensor, group size g along K.
 * qu4: [N][K]; s_u8, z: [N][K/g]. */
int oracle_level2(const int8_t* q8, int N, int K, int g, uint8_t* qu4, uint8_t* s_u8, uint8_t* z);

/* Level-2 dequantization, Eq. (progressive_quant:int4) read right to left:
 * qhat[n][k] = (qu4 - z) * s_u8 (exact integer, may exceed INT8 only if the protective
 * range is violated). qhat is int16 so an overflow is observable. */
int oracle_dequant_level2(const uint8_t* qu4, const uint8_t* s_u8, const uint8_t* z,
                          int N, int K, int g, int16_t* qhat);

/* O3 — pack into the frozen tile stream (DESIGN.md §4 "Packed weight layout"; the B200 form
 * of "store the weights in the order they are used", with the RLP nibble interleave
 * w0,w16,w1,w17,... of P:447, reading Q15). 128x128 tiles of 8448 bytes, n-tile-major.
 * packed must hold (N/128)*(K/128)*8448 bytes. Requires g == 128, N%128 == K%128 == 0. */
int oracle_pack(const uint8_t* qu4, const uint8_t* s_u8, const uint8_t* z, int N, int K, int g,
                uint8_t* packed);
/* Inverse of oracle_pack. */
int oracle_unpack(const uint8_t* packed, int N, int K, int g,
                  uint8_t* qu4, uint8_t* s_u8, uint8_t* z);

/* O4 — per-token symmetric INT8 activation quantization (§6.1; symmetric form P:132).
 * X: [M][ldx] fp16. qx: [M][K] int8; sx: [M] fp16; tx: [M] int32 row sums of qx (nullable). */
int oracle_quantize_activations(const uint16_t* X, int M, int K, int ldx,
                                int8_t* qx, uint16_t* sx, int32_t* tx);

/* O5 — integer GEMM: acc[m][n] = sum_k qx[m][k] * qhat[n][k], accumulated in int64 and
 * checked to fit INT32 ("INT32 partial sums", "INT8 matrix multiplication as if it
 * was W8A8"). Returns -2 if any result leaves the int32 range. Rows [m0, m1) only. */
int oracle_gemm_i32(const int8_t* qx, const int16_t* qhat, int M, int N, int K,
                    int m0, int m1, int32_t* acc);

/* O6 — epilogue reference y = acc * s_x[m] * s0[n] in fp64 (the s_W x s_X outer
 * product scaling in the epilogue). Exact in fp64 (<= 51 significant bits). */
int oracle_epilogue_f64(const int32_t* acc, const uint16_t* sx, const uint16_t* s0,
                        int M, int N, double* y);

/* The whole linear layer from packed weights, rows [m0, m1) of X only (used for sampled
 * parity at full size and for the timed CPU baseline): O4 on those rows -> unpack (O3^-1) ->
 * dequant level 2 -> O5 -> O6. y: [(m1-m0)][N]. qhat_scratch: N*K int16 or NULL (allocated). */
int oracle_linear_rows(const uint16_t* X, int K, int ldx, int m0, int m1,
                       const uint8_t* packed, const uint16_t* s0, int N, double* y);

/* ---------------- NEXT-1: per-channel W4A8 (§5.2.2) ---------------- */

/* PC1 — per-output-channel asymmetric UINT4 weight quantization: Eq. 2 with
 * q_min = 0, q_max = 15, s and z shared within each row (per-channel), FP16 scale
 * ("first-level FP16 scaling"). Readings (Q20-Q22):
 *   range = fp32(max_k W) - fp32(min_k W) (IEEE fp32 subtraction);
 *   s = fp16_rn(range / 15.0f) (fp32 division); range == 0 -> 1.0; fp16 underflow -> 2^-24;
 *   z = clamp(⌈0 - t_min⌋, 0, 15), t_min = fp32(min / s) with the fp16-rounded s (Q1: ⌈·⌋ rounds
 *       half away from zero);
 *   q = clamp(⌈t + z⌋, 0, 15), t = fp32(W / s), t + z summed exactly (in double).
 * W: [N][K] fp16. qu4: [N][K] in [0,15]; s_w: [N] fp16; z_w: [N] in [0,15]. */
int oracle_pc_quantize(const uint16_t* W, int N, int K, uint8_t* qu4, uint16_t* s_w, uint8_t* z_w);

/* PC pack: the O3 nibble stream without level-2 bytes — 128x128 tiles of 8192 bytes, n-tile-major,
 * chunk c / row r at c*2048 + r*16, byte b = q[32c+b] | q[32c+16+b] << 4 (Q15). */
int oracle_pc_pack(const uint8_t* qu4, int N, int K, uint8_t* packed);
int oracle_pc_unpack(const uint8_t* packed, int N, int K, uint8_t* qu4);

/* PC GEMM, the definition Eq. (per_channel_qmm) P:454 in integers: acc[m][n] =
 * sum_k qx[m][k] * (qu4[n][k] - z_w[n]), accumulated in int64 and checked into int32 (-2 if not).
 * The epilogue reference is oracle_epilogue_f64(acc, s_x, s_w): y = acc * s_x[m] * s_w[n]. */
int oracle_pc_gemm_i32(const int8_t* qx, const uint8_t* qu4, const uint8_t* z_w, int M, int N, int K,
                       int32_t* acc);

/* ---------------- NEXT-2: fused activation quantization (Fig. 7) ----------------
 * "we fuse activation quantization into the preceding layernorm for the QKV projection and the first
 * FFN layer, or into the preceding activation kernel for the second FFN layer". The paper
 * does not define the layers; readings Q23-Q26: Llama RMSNorm and SiLU·mul, the fp16
 * layer output rounded once from fp64, then O4 on it (fused == unfused composition, bit for bit). */

/* r = 1 / sqrt(S/K + eps), S = Σ x^2 summed exactly and rounded once to fp64 (Q25); 0 if S/K+eps==0. */
double oracle_rmsnorm_rinv(const uint16_t* x, int K, double eps);
/* Y[m][k] = fp16_rn((x[m][k] * r_m) * gamma[k]) in fp64. X [M][ldx], gamma [K], Y [M][K]. */
int oracle_rmsnorm_fp16(const uint16_t* X, int M, int K, int ldx, const uint16_t* gamma, double eps,
                        uint16_t* Y);
/* O4 of oracle_rmsnorm_fp16's output: qx [M][K], sx [M], tx [M] (nullable). */
int oracle_rmsnorm_quantize(const uint16_t* X, int M, int K, int ldx, const uint16_t* gamma, double eps,
                            int8_t* qx, uint16_t* sx, int32_t* tx);
/* silu(g) = g / (1 + exp(-g)) in fp64 (Q26). */
double oracle_silu_f64(double g);
/* H[m][k] = fp16_rn(silu(G[m][k]) * U[m][k]) in fp64. G, U [M][ldg] (e.g. the two halves of the
 * fused gate_up output, ldg = 2K), H [M][K]. */
int oracle_silu_mul_fp16(const uint16_t* G, const uint16_t* U, int M, int K, int ldg, uint16_t* H);
/* O4 of oracle_silu_mul_fp16's output. */
int oracle_silu_mul_quantize(const uint16_t* G, const uint16_t* U, int M, int K, int ldg,
                             int8_t* qx, uint16_t* sx, int32_t* tx);

/* ---------------- NEXT-4: KV4 cache + decode attention (§5.3) ----------------
 * Readings Q27-Q29. */
/* per-(token, kv head) asymmetric UINT4 of rows of D values: the Q20-Q22 rule (oracle_pc_quantize),
 * zero point returned as fp16 bits. q [rows][D]; s, z [rows]. */
int oracle_kv4_quantize(const uint16_t* X, int rows, int D, uint8_t* q, uint16_t* s, uint16_t* z);
/* bytes of one page (P tokens, all kv heads, K and V): H_kv * P * (D + 8) */
size_t oracle_kv4_page_bytes(int H_kv, int D, int P);
/* write T tokens of one sequence into pages (layout in qoq_oracle.c / DESIGN.md §4) */
int oracle_kv4_store(const uint8_t* qk, const uint16_t* sk, const uint16_t* zk, const uint8_t* qv,
                     const uint16_t* sv, const uint16_t* zv, int T, int H_kv, int D, int P,
                     const int32_t* block_table, uint8_t* pages);
/* xhat = (q - z) s in fp64 */
int oracle_kv4_dequant(const uint8_t* q, const uint16_t* s, const uint16_t* z, int rows, int D, double* xhat);
/* o_h = softmax(q_h K^T / sqrt(D)) V over T tokens, kv head h / (H / H_kv); fp64 */
int oracle_attention_f64(const uint16_t* Q, const double* Khat, const double* Vhat, int T, int H, int H_kv, int D,
                         double* O);

/* Number of OpenMP threads the oracle's parallel loops use (1 without OpenMP). */
int oracle_num_threads(void);
void oracle_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
