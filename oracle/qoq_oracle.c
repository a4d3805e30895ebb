/* qoq_oracle.c — plain, slow, obviously-correct CPU oracle for the QoQ W4A8 hot path
 * (QServe, arXiv 2405.04532). See qoq_oracle.h for the contract of every function.
 *
 * TEST INFRASTRUCTURE ONLY (see header). Scalar loops, no intrinsics, no fast-math; the only
 * parallelism is an OpenMP parallel-for over independent output elements of the GEMM.
 * Compiled with: gcc -O2 -std=c11 -fno-fast-math -fopenmp -shared -fPIC.
 *
 * Parity status: every function below is pinned by tests/test_oracle_pins.py.
 */
#include "qoq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TILE_N 128
#define TILE_K 128
#define TILE_BYTES 8448 /* 8192 packed nibbles + 128 s_u8 + 128 z*s_u8 */

/* Thread count of the OpenMP GEMM loops (bench.py times the oracle single-threaded and on all cores). */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------- IEEE binary16 ---------------- */

float oracle_h2f(uint16_t h) {
    int sign = (h >> 15) & 1, e = (h >> 10) & 0x1f, man = h & 0x3ff;
    float v;
    if (e == 0)
        v = ldexpf((float)man, -24);                 /* subnormal: man * 2^-24 */
    else if (e == 31)
        v = man ? NAN : INFINITY;
    else
        v = ldexpf((float)(man | 0x400), e - 25);    /* 1.man * 2^(e-15) */
    return sign ? -v : v;
}

/* binary64 -> binary16, round to nearest, ties to even (one rounding; Q8, Q10, Q24). */
uint16_t oracle_d2h_rn(double f) {
    uint16_t sign = signbit(f) ? 0x8000 : 0;
    if (isnan(f)) return 0x7e00;
    double a = fabs(f);
    if (a == 0.0) return sign;
    if (isinf(a)) return sign | 0x7c00;
    int E;
    frexp(a, &E);                                    /* a = m * 2^E, m in [0.5, 1) */
    int e = E - 1;                                   /* a in [2^e, 2^(e+1)) */
    int qexp = (e < -14) ? -24 : e - 10;             /* quantum: subnormal spacing or 2^(e-10) */
    double r = rint(ldexp(a, -qexp));                /* exact scaling; rint = ties-to-even */
    double v = ldexp(r, qexp);                       /* rounded magnitude, exact */
    if (v > 65504.0) return sign | 0x7c00;           /* overflow to infinity */
    if (v < ldexp(1.0, -14))                         /* subnormal (or zero) */
        return sign | (uint16_t)(int)ldexp(v, 24);
    frexp(v, &E);
    e = E - 1;
    int man = (int)(ldexp(v, -e) * 1024.0) - 1024;
    return sign | (uint16_t)((e + 15) << 10) | (uint16_t)man;
}

/* binary32 -> binary16: every float is exactly a double, so one rounding of that double. */
uint16_t oracle_f2h_rn(float f) { return oracle_d2h_rn((double)f); }

/* Q1: ⌈·⌋ = round half away from zero; exact integer form for a/b, b > 0. */
int oracle_rhai(int a, int b) {
    int m = a < 0 ? -a : a;
    int q = (2 * m + b) / (2 * b);
    return a < 0 ? -q : q;
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Symmetric scale rule shared in form (not code) by level 1 and the activations, Q8/Q10:
 * s = fp16_rn(amax / qmax) in fp32; amax == 0 -> 1.0; fp16 underflow to 0 -> 2^-24. */
static uint16_t sym_scale_fp16(float amax, float qmax) {
    if (amax == 0.0f) return 0x3c00;                 /* 1.0 */
    uint16_t s = oracle_f2h_rn(amax / qmax);         /* IEEE fp32 division */
    if ((s & 0x7fff) == 0) s = 0x0001;               /* 2^-24 */
    return s;
}

/* ---------------- O1: level 1 (protective range P:257-275) ---------------- */

int oracle_level1(const uint16_t* W, int N, int K, int8_t* q8, uint16_t* s0) {
    if (N < 0 || K <= 0) return -1;
    for (int n = 0; n < N; ++n) {
        const uint16_t* w = W + (size_t)n * K;
        float amax = 0.0f;
        for (int k = 0; k < K; ++k) {
            float a = fabsf(oracle_h2f(w[k]));
            if (a > amax) amax = a;
        }
        s0[n] = sym_scale_fp16(amax, 119.0f);
        float s = oracle_h2f(s0[n]);                 /* quantize with the fp16-rounded scale (Q8) */
        for (int k = 0; k < K; ++k) {
            float t = oracle_h2f(w[k]) / s;
            q8[(size_t)n * K + k] = (int8_t)clampi((int)roundf(t), -119, 119);
        }
    }
    return 0;
}

/* ---------------- O2: level 2 (Eq. 2; example P:257) ---------------- */

int oracle_level2_group(const int8_t* q8, int g, uint8_t* qu4, uint8_t* s_u8, uint8_t* z) {
    if (g <= 0) return -1;
    int lo = q8[0], hi = q8[0];
    for (int i = 1; i < g; ++i) {
        if (q8[i] < lo) lo = q8[i];
        if (q8[i] > hi) hi = q8[i];
    }
    /* s = (X_max - X_min) / (q_max - q_min), an unsigned 8-bit integer (⌈233/15⌋=16);
     * a degenerate range gives s = 1 (Q3). */
    int s = oracle_rhai(hi - lo, 15);
    if (s < 1) s = 1;
    /* z = ⌈q_min - X_min / s⌋ with q_min = 0, clamped to the u4 range (Q4). */
    int zz = clampi(oracle_rhai(-lo, s), 0, 15);
    /* Q = ⌈X / s + z⌋ = ⌈(X + z*s) / s⌋ (z integer), clamped to [0, 15] (Q2). */
    for (int i = 0; i < g; ++i)
        qu4[i] = (uint8_t)clampi(oracle_rhai((int)q8[i] + zz * s, s), 0, 15);
    *s_u8 = (uint8_t)s;
    *z = (uint8_t)zz;
    return 0;
}

int oracle_level2(const int8_t* q8, int N, int K, int g, uint8_t* qu4, uint8_t* s_u8, uint8_t* z) {
    if (g <= 0 || K % g != 0) return -1;
    int G = K / g;
    for (int n = 0; n < N; ++n)
        for (int j = 0; j < G; ++j) {
            size_t off = (size_t)n * K + (size_t)j * g;
            int rc = oracle_level2_group(q8 + off, g, qu4 + off, s_u8 + (size_t)n * G + j,
                                         z + (size_t)n * G + j);
            if (rc) return rc;
        }
    return 0;
}

int oracle_dequant_level2(const uint8_t* qu4, const uint8_t* s_u8, const uint8_t* z,
                          int N, int K, int g, int16_t* qhat) {
    if (g <= 0 || K % g != 0) return -1;
    int G = K / g;
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) {
            int j = k / g;
            qhat[(size_t)n * K + k] = (int16_t)(((int)qu4[(size_t)n * K + k] - (int)z[(size_t)n * G + j])
                                                * (int)s_u8[(size_t)n * G + j]);
        }
    return 0;
}

/* ---------------- O3: packed tile stream (layout frozen in DESIGN.md §4) ---------------- */

static int pack_shape_ok(int N, int K, int g) {
    return g == 128 && N > 0 && K > 0 && N % TILE_N == 0 && K % TILE_K == 0;
}

int oracle_pack(const uint8_t* qu4, const uint8_t* s_u8, const uint8_t* z, int N, int K, int g,
                uint8_t* packed) {
    if (!pack_shape_ok(N, K, g)) return -1;
    int KT = K / TILE_K, G = K / g;
    for (int nt = 0; nt < N / TILE_N; ++nt)
        for (int j = 0; j < KT; ++j) {
            uint8_t* tile = packed + ((size_t)nt * KT + j) * TILE_BYTES;
            for (int r = 0; r < TILE_N; ++r) {
                int n = nt * TILE_N + r;
                const uint8_t* q = qu4 + (size_t)n * K + (size_t)j * TILE_K;
                for (int c = 0; c < 4; ++c)            /* chunk c: k = 32c .. 32c+31 of this group */
                    for (int b = 0; b < 16; ++b)       /* byte b = w_b | w_{b+16} << 4 */
                        tile[c * 2048 + r * 16 + b] =
                            (uint8_t)((q[32 * c + b] & 15) | ((q[32 * c + 16 + b] & 15) << 4));
                uint8_t s = s_u8[(size_t)n * G + j];
                tile[8192 + r] = s;
                tile[8320 + r] = (uint8_t)(z[(size_t)n * G + j] * s);   /* z * s_u8 (north_star) */
            }
        }
    return 0;
}

int oracle_unpack(const uint8_t* packed, int N, int K, int g,
                  uint8_t* qu4, uint8_t* s_u8, uint8_t* z) {
    if (!pack_shape_ok(N, K, g)) return -1;
    int KT = K / TILE_K, G = K / g;
    for (int nt = 0; nt < N / TILE_N; ++nt)
        for (int j = 0; j < KT; ++j) {
            const uint8_t* tile = packed + ((size_t)nt * KT + j) * TILE_BYTES;
            for (int r = 0; r < TILE_N; ++r) {
                int n = nt * TILE_N + r;
                uint8_t* q = qu4 + (size_t)n * K + (size_t)j * TILE_K;
                for (int c = 0; c < 4; ++c)
                    for (int b = 0; b < 16; ++b) {
                        uint8_t byte = tile[c * 2048 + r * 16 + b];
                        q[32 * c + b] = byte & 15;
                        q[32 * c + 16 + b] = byte >> 4;
                    }
                uint8_t s = tile[8192 + r], zs = tile[8320 + r];
                if (s == 0 || zs % s != 0) return -3;  /* not a valid packed tile */
                s_u8[(size_t)n * G + j] = s;
                z[(size_t)n * G + j] = (uint8_t)(zs / s);
            }
        }
    return 0;
}

/* ---------------- O4: per-token symmetric INT8 activations ---------------- */

int oracle_quantize_activations(const uint16_t* X, int M, int K, int ldx,
                                int8_t* qx, uint16_t* sx, int32_t* tx) {
    if (M < 0 || K <= 0 || ldx < K) return -1;
    for (int m = 0; m < M; ++m) {
        const uint16_t* x = X + (size_t)m * ldx;
        float amax = 0.0f;
        for (int k = 0; k < K; ++k) {
            float a = fabsf(oracle_h2f(x[k]));
            if (a > amax) amax = a;
        }
        sx[m] = sym_scale_fp16(amax, 127.0f);
        float s = oracle_h2f(sx[m]);
        int32_t t = 0;
        for (int k = 0; k < K; ++k) {
            int q = clampi((int)roundf(oracle_h2f(x[k]) / s), -127, 127);
            qx[(size_t)m * K + k] = (int8_t)q;
            t += q;
        }
        if (tx) tx[m] = t;
    }
    return 0;
}

/* ---------------- O5: integer GEMM ---------------- */

int oracle_gemm_i32(const int8_t* qx, const int16_t* qhat, int M, int N, int K,
                    int m0, int m1, int32_t* acc) {
    if (m0 < 0 || m1 > M || m0 > m1) return -1;
    int overflow = 0;
#pragma omp parallel for collapse(2) schedule(static) reduction(|:overflow)
    for (int m = m0; m < m1; ++m)
        for (int n = 0; n < N; ++n) {
            int64_t s = 0;
            for (int k = 0; k < K; ++k)
                s += (int64_t)qx[(size_t)m * K + k] * (int64_t)qhat[(size_t)n * K + k];
            if (s > INT32_MAX || s < INT32_MIN) overflow = 1;
            acc[(size_t)(m - m0) * N + n] = (int32_t)s;
        }
    return overflow ? -2 : 0;
}

/* ---------------- O6: epilogue reference ---------------- */

int oracle_epilogue_f64(const int32_t* acc, const uint16_t* sx, const uint16_t* s0,
                        int M, int N, double* y) {
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n)
            y[(size_t)m * N + n] = (double)acc[(size_t)m * N + n] * (double)oracle_h2f(sx[m])
                                   * (double)oracle_h2f(s0[n]);
    return 0;
}

/* ---------------- whole linear layer from packed weights ---------------- */

int oracle_linear_rows(const uint16_t* X, int K, int ldx, int m0, int m1,
                       const uint8_t* packed, const uint16_t* s0, int N, double* y) {
    int g = 128, rows = m1 - m0, rc = 0;
    if (rows < 0 || !pack_shape_ok(N, K, g)) return -1;
    size_t NK = (size_t)N * K;
    uint8_t* qu4 = malloc(NK);
    uint8_t* su8 = malloc((size_t)N * (K / g));
    uint8_t* z = malloc((size_t)N * (K / g));
    int16_t* qhat = malloc(NK * sizeof(int16_t));
    int8_t* qx = malloc((size_t)(rows ? rows : 1) * K);
    uint16_t* sx = malloc((size_t)(rows ? rows : 1) * sizeof(uint16_t));
    int32_t* acc = malloc((size_t)(rows ? rows : 1) * N * sizeof(int32_t));
    if (!qu4 || !su8 || !z || !qhat || !qx || !sx || !acc) { rc = -4; goto done; }
    if ((rc = oracle_quantize_activations(X + (size_t)m0 * ldx, rows, K, ldx, qx, sx, NULL))) goto done;
    if ((rc = oracle_unpack(packed, N, K, g, qu4, su8, z))) goto done;
    if ((rc = oracle_dequant_level2(qu4, su8, z, N, K, g, qhat))) goto done;
    if ((rc = oracle_gemm_i32(qx, qhat, rows, N, K, 0, rows, acc))) goto done;
    rc = oracle_epilogue_f64(acc, sx, s0, rows, N, y);
done:
    free(qu4); free(su8); free(z); free(qhat); free(qx); free(sx); free(acc);
    return rc;
}

/* ---------------- NEXT-1: per-channel W4A8 (§5.2.2) ---------------- */

/* Round half away from zero of a double (Q1), as an int. */
static int rha_d(double v) { return (int)round(v); }

int oracle_pc_quantize(const uint16_t* W, int N, int K, uint8_t* qu4, uint16_t* s_w, uint8_t* z_w) {
    if (N < 0 || K <= 0) return -1;
    for (int n = 0; n < N; ++n) {
        const uint16_t* w = W + (size_t)n * K;
        float lo = oracle_h2f(w[0]), hi = lo;
        for (int k = 1; k < K; ++k) {
            float v = oracle_h2f(w[k]);
            if (v < lo) lo = v;
            if (v > hi) hi = v;
        }
        /* Eq. 2: s = (X_max - X_min) / (q_max - q_min), stored as fp16 (Q20) */
        float range = hi - lo;
        uint16_t sh;
        if (range == 0.0f) {
            sh = 0x3c00;                                  /* 1.0 */
        } else {
            sh = oracle_f2h_rn(range / 15.0f);
            if ((sh & 0x7fff) == 0) sh = 0x0001;          /* 2^-24 */
        }
        float s = oracle_h2f(sh);
        /* z = ⌈q_min - X_min / s⌋, q_min = 0, clamped to the u4 range (Q21) */
        int z = clampi(rha_d(-(double)(lo / s)), 0, 15);
        /* Q = ⌈X / s + z⌋ clamped to [0, 15] (Q22: t = fp32(X / s), t + z exact) */
        for (int k = 0; k < K; ++k) {
            float t = oracle_h2f(w[k]) / s;
            qu4[(size_t)n * K + k] = (uint8_t)clampi(rha_d((double)t + (double)z), 0, 15);
        }
        s_w[n] = sh;
        z_w[n] = (uint8_t)z;
    }
    return 0;
}

#define PC_TILE_BYTES 8192

int oracle_pc_pack(const uint8_t* qu4, int N, int K, uint8_t* packed) {
    if (!pack_shape_ok(N, K, 128)) return -1;
    int KT = K / TILE_K;
    for (int nt = 0; nt < N / TILE_N; ++nt)
        for (int j = 0; j < KT; ++j) {
            uint8_t* tile = packed + ((size_t)nt * KT + j) * PC_TILE_BYTES;
            for (int r = 0; r < TILE_N; ++r) {
                const uint8_t* q = qu4 + (size_t)(nt * TILE_N + r) * K + (size_t)j * TILE_K;
                for (int c = 0; c < 4; ++c)
                    for (int b = 0; b < 16; ++b)
                        tile[c * 2048 + r * 16 + b] =
                            (uint8_t)((q[32 * c + b] & 15) | ((q[32 * c + 16 + b] & 15) << 4));
            }
        }
    return 0;
}

int oracle_pc_unpack(const uint8_t* packed, int N, int K, uint8_t* qu4) {
    if (!pack_shape_ok(N, K, 128)) return -1;
    int KT = K / TILE_K;
    for (int nt = 0; nt < N / TILE_N; ++nt)
        for (int j = 0; j < KT; ++j) {
            const uint8_t* tile = packed + ((size_t)nt * KT + j) * PC_TILE_BYTES;
            for (int r = 0; r < TILE_N; ++r) {
                uint8_t* q = qu4 + (size_t)(nt * TILE_N + r) * K + (size_t)j * TILE_K;
                for (int c = 0; c < 4; ++c)
                    for (int b = 0; b < 16; ++b) {
                        uint8_t byte = tile[c * 2048 + r * 16 + b];
                        q[32 * c + b] = byte & 15;
                        q[32 * c + 16 + b] = byte >> 4;
                    }
            }
        }
    return 0;
}

int oracle_pc_gemm_i32(const int8_t* qx, const uint8_t* qu4, const uint8_t* z_w, int M, int N, int K,
                       int32_t* acc) {
    if (M < 0 || N < 0 || K <= 0) return -1;
    int overflow = 0;
#pragma omp parallel for collapse(2) schedule(static) reduction(|:overflow)
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            int64_t s = 0;
            for (int k = 0; k < K; ++k)
                s += (int64_t)qx[(size_t)m * K + k] * ((int64_t)qu4[(size_t)n * K + k] - (int64_t)z_w[n]);
            if (s > INT32_MAX || s < INT32_MIN) overflow = 1;
            acc[(size_t)m * N + n] = (int32_t)s;
        }
    return overflow ? -2 : 0;
}

/* ---------------- NEXT-2: activation quantization fused into RMSNorm / SiLU·mul (Fig. 7) ----
 * The fused kernels are defined as the composition "fp16 output of the layer, then O4", so these
 * oracles compute the fp16 layer output and call oracle_quantize_activations on it (Q23). */

/* Q25: S = Σ_k x_k^2 exactly (each x^2 of an fp16 x is an integer multiple of 2^-48 below 2^32, so
 * Σ x^2 * 2^48 is an integer < 2^95 for K < 2^31: a 128-bit integer sum), rounded ONCE to fp64;
 * then r = 1 / sqrt(S / K + eps) in IEEE fp64 (each operation correctly rounded). S / K + eps == 0
 * (all-zero row, eps == 0) gives r = 0. */
double oracle_rmsnorm_rinv(const uint16_t* x, int K, double eps) {
    unsigned __int128 S = 0;
    for (int k = 0; k < K; ++k) {
        double v = (double)oracle_h2f(x[k]);
        S += (unsigned __int128)ldexp(v * v, 48);   /* v*v exact (22 bits); integer-valued */
    }
    double ms = ldexp((double)S, -48) / (double)K + eps;
    return ms == 0.0 ? 0.0 : 1.0 / sqrt(ms);
}

/* RMSNorm (Llama form, Q23): y[m][k] = fp16_rn( (x[m][k] * r_m) * gamma[k] ), products in fp64,
 * left to right, one rounding to fp16 (Q24). X [M][ldx], gamma [K], Y [M][K] (fp16 bits). */
int oracle_rmsnorm_fp16(const uint16_t* X, int M, int K, int ldx, const uint16_t* gamma, double eps,
                        uint16_t* Y) {
    if (M < 0 || K <= 0 || ldx < K || eps < 0.0) return -1;
    for (int m = 0; m < M; ++m) {
        const uint16_t* x = X + (size_t)m * ldx;
        double r = oracle_rmsnorm_rinv(x, K, eps);
        for (int k = 0; k < K; ++k)
            Y[(size_t)m * K + k] = oracle_d2h_rn((double)oracle_h2f(x[k]) * r * (double)oracle_h2f(gamma[k]));
    }
    return 0;
}

int oracle_rmsnorm_quantize(const uint16_t* X, int M, int K, int ldx, const uint16_t* gamma, double eps,
                            int8_t* qx, uint16_t* sx, int32_t* tx) {
    if (M < 0 || K <= 0 || ldx < K || eps < 0.0) return -1;
    uint16_t* Y = (uint16_t*)malloc((size_t)(M > 0 ? M : 1) * K * sizeof(uint16_t));
    if (!Y) return -3;
    int rc = oracle_rmsnorm_fp16(X, M, K, ldx, gamma, eps, Y);
    if (!rc) rc = oracle_quantize_activations(Y, M, K, K, qx, sx, tx);
    free(Y);
    return rc;
}

/* SiLU (Llama FFN activation, Q26): silu(g) = g / (1 + exp(-g)) in fp64. */
double oracle_silu_f64(double g) { return g / (1.0 + exp(-g)); }

/* h[m][k] = fp16_rn( silu(g[m][k]) * u[m][k] ) in fp64 (Q24, Q26). G, U: [M][ldg]. H: [M][K]. */
int oracle_silu_mul_fp16(const uint16_t* G, const uint16_t* U, int M, int K, int ldg, uint16_t* H) {
    if (M < 0 || K <= 0 || ldg < K) return -1;
    for (int m = 0; m < M; ++m)
        for (int k = 0; k < K; ++k) {
            double g = (double)oracle_h2f(G[(size_t)m * ldg + k]);
            double u = (double)oracle_h2f(U[(size_t)m * ldg + k]);
            H[(size_t)m * K + k] = oracle_d2h_rn(oracle_silu_f64(g) * u);
        }
    return 0;
}

int oracle_silu_mul_quantize(const uint16_t* G, const uint16_t* U, int M, int K, int ldg,
                             int8_t* qx, uint16_t* sx, int32_t* tx) {
    if (M < 0 || K <= 0 || ldg < K) return -1;
    uint16_t* H = (uint16_t*)malloc((size_t)(M > 0 ? M : 1) * K * sizeof(uint16_t));
    if (!H) return -3;
    int rc = oracle_silu_mul_fp16(G, U, M, K, ldg, H);
    if (!rc) rc = oracle_quantize_activations(H, M, K, K, qx, sx, tx);
    free(H);
    return rc;
}

/* ---------------- NEXT-4: KV4 cache and decode attention (§5.3) ----------------
 * Q27: each (token, kv head) vector of D values is quantized with the per-channel rule of Q20-Q22 (Eq. 2,
 * asymmetric UINT4, FP16 scale; the integer zero point stored as FP16, "FP16 scaling factors and
 * zero points for each head"). Q28: page layout. Q29: attention o_h = softmax(q_h K^T/√D) V
 * on the dequantized cache, kv head = h / (H / H_kv) (GQA). */

int oracle_kv4_quantize(const uint16_t* X, int rows, int D, uint8_t* q, uint16_t* s, uint16_t* z) {
    uint8_t* zz = (uint8_t*)malloc((size_t)(rows > 0 ? rows : 1));
    if (!zz) return -3;
    int rc = oracle_pc_quantize(X, rows, D, q, s, zz);
    for (int i = 0; rc == 0 && i < rows; ++i) z[i] = oracle_f2h_rn((float)zz[i]);
    free(zz);
    return rc;
}

size_t oracle_kv4_page_bytes(int H_kv, int D, int P) { return (size_t)H_kv * P * (D + 8); }

/* Store T tokens of one sequence (codes q*[T][H_kv][D], params s*, z* [T][H_kv]) into pages following
 * block_table (token t -> page block_table[t / P], slot t % P). Page layout per kv head h, at
 * page + h * P * (D + 8): K codes [P][D/2] (byte j = q[2j] | q[2j+1] << 4), V codes [P][D/2],
 * K params [P][s, z] fp16, V params [P][s, z] fp16. */
int oracle_kv4_store(const uint8_t* qk, const uint16_t* sk, const uint16_t* zk, const uint8_t* qv,
                     const uint16_t* sv, const uint16_t* zv, int T, int H_kv, int D, int P,
                     const int32_t* block_table, uint8_t* pages) {
    if (D % 2 || P <= 0 || T < 0) return -1;
    size_t pb = oracle_kv4_page_bytes(H_kv, D, P), hb = (size_t)P * (D + 8);
    for (int t = 0; t < T; ++t)
        for (int h = 0; h < H_kv; ++h) {
            uint8_t* base = pages + (size_t)block_table[t / P] * pb + (size_t)h * hb;
            int o = t % P;
            size_t row = ((size_t)t * H_kv + h) * D;
            for (int j = 0; j < D / 2; ++j) {
                base[(size_t)o * (D / 2) + j] = (uint8_t)(qk[row + 2 * j] | (qk[row + 2 * j + 1] << 4));
                base[(size_t)P * (D / 2) + (size_t)o * (D / 2) + j] = (uint8_t)(qv[row + 2 * j] | (qv[row + 2 * j + 1] << 4));
            }
            uint16_t* par = (uint16_t*)(base + (size_t)P * D);
            par[2 * o] = sk[(size_t)t * H_kv + h];
            par[2 * o + 1] = zk[(size_t)t * H_kv + h];
            par[2 * P + 2 * o] = sv[(size_t)t * H_kv + h];
            par[2 * P + 2 * o + 1] = zv[(size_t)t * H_kv + h];
        }
    return 0;
}

/* Dequantize: xhat = (q - z) * s in fp64 (exact: an 11-bit scale times an integer in [-15, 15]). */
int oracle_kv4_dequant(const uint8_t* q, const uint16_t* s, const uint16_t* z, int rows, int D, double* xhat) {
    for (int i = 0; i < rows; ++i)
        for (int d = 0; d < D; ++d)
            xhat[(size_t)i * D + d] = ((double)q[(size_t)i * D + d] - (double)oracle_h2f(z[i])) * (double)oracle_h2f(s[i]);
    return 0;
}

/* Decode attention for one sequence, the definition (§2.1; P:412 GQA via kv head h / (H / H_kv)):
 * o[h] = Σ_t p_t v_t, p = softmax_t(q_h · k_t / sqrt(D)), all in fp64 (max-subtracted exp).
 * Q [H][D] fp16; Khat, Vhat [T][H_kv][D] fp64; O [H][D] fp64. */
int oracle_attention_f64(const uint16_t* Q, const double* Khat, const double* Vhat, int T, int H, int H_kv, int D,
                         double* O) {
    if (T <= 0 || H_kv <= 0 || H % H_kv) return -1;
    double* sc = (double*)malloc((size_t)T * sizeof(double));
    if (!sc) return -3;
    int r = H / H_kv;
    for (int h = 0; h < H; ++h) {
        int g = h / r;
        double mx = -INFINITY;
        for (int t = 0; t < T; ++t) {
            double a = 0.0;
            for (int d = 0; d < D; ++d)
                a += (double)oracle_h2f(Q[(size_t)h * D + d]) * Khat[((size_t)t * H_kv + g) * D + d];
            sc[t] = a / sqrt((double)D);
            if (sc[t] > mx) mx = sc[t];
        }
        double L = 0.0;
        for (int t = 0; t < T; ++t) {
            sc[t] = exp(sc[t] - mx);
            L += sc[t];
        }
        for (int d = 0; d < D; ++d) {
            double acc = 0.0;
            for (int t = 0; t < T; ++t) acc += sc[t] * Vhat[((size_t)t * H_kv + g) * D + d];
            O[(size_t)h * D + d] = acc / L;
        }
    }
    free(sc);
    return 0;
}
