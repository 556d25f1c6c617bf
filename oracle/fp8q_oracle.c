/*
 * fp8q_oracle.c -- CPU ORACLE for the FP8 W8A8 rollout hot path of
 * "FP8-RL: A Practical and Stable Low-Precision Stack for LLM RL" (arXiv 2601.18150).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2601_18150_b200/) never includes, links or calls anything in oracle/, and
 * this file includes no header of the product path: the two share no code.
 *
 * What it computes: the plain DEFINITIONS, written out element by element, in the
 * paper's order (§2.1.1, Eq. (1), lines 52-58) with the readings fixed in
 * DESIGN.md §3:
 *
 *   O1  e4m3 decode      value(c) = (-1)^s 2^(e-7) (1 + m/8), e>0;  (-1)^s 2^-6 (m/8), e=0;
 *                        S.1111.111 = NaN
 *   O2  e4m3 encode      nearest finite E4M3 value, ties to the even code (LSB 0),
 *                        |q| >= 448 -> +-448 (saturating), sign kept (-0 -> 0x80),
 *                        NaN -> 0x7F/0xFF                  (reading Q1,Q6,Q7)
 *   O3  block amax       max |x| over the in-bounds elements (BF16 widened exactly)
 *                                                          ("maximum absolute value")
 *   O4  scale            s = RN32(amax / 448), amax == 0 -> s = 1   (reading Q2,Q4,Q5)
 *   O5  element          code = O2(RN32(x / s))            (Eq. (1); reading Q3)
 *   O6  layouts          weight blocks 128x128 over nn.Linear [N=out, K=in]; activation
 *                        groups 1x128 per token (reading Q10-Q12)
 *   O7  GEMM             Y[m,n] = sum_k (dec(a[m,k]) sa[m,k/128]) (dec(b[n,k]) sb[n/128,k/128])
 *                        accumulated in binary64           (north_star)
 *
 * Precision: binary32 where the paper's reading fixes binary32 (the scale and the
 * quotient, Q3/Q4), binary64 for the GEMM reference.  Build with
 *   gcc -O2 -ffp-contract=off -fno-fast-math   (no FMA contraction, IEEE division,
 *   default MXCSR: subnormals honoured; 1,247 BF16 amax values give subnormal scales).
 *
 * Threads: the quantizers and the GEMM are element-wise / row-wise independent maps; the
 * optional nthreads argument splits the OUTPUT index space across std pthreads without
 * changing any arithmetic (every result is computed exactly as in the 1-thread case).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if defined(__FAST_MATH__)
#error "the oracle must not be built with fast-math"
#endif

#define ORACLE_OK 0
#define ORACLE_ENONFINITE 1 /* non-finite input is rejected */
#define ORACLE_EINVAL 2

/* ------------------------------------------------------------------ O1: decode */
/* normals (-1)^s 2^(e-7) (1+m/8); subnormals (e=0) (-1)^s 2^-6 (m/8); NaN at
 * exponent and mantissa all ones (E4M3FN variant, reading Q9). */
double oracle_e4m3_decode(uint8_t c) {
    int s = (c >> 7) & 1;
    int e = (c >> 3) & 0xF;
    int m = c & 0x7;
    double v;
    if (e == 0xF && m == 0x7) return NAN;
    if (e == 0)
        v = ldexp((double)m / 8.0, -6);
    else
        v = ldexp(1.0 + (double)m / 8.0, e - 7);
    return s ? -v : v;
}

/* ------------------------------------------------------------------ O2: encode */
/* The 127 non-negative finite values, ascending: code i (0x00..0x7E) decodes to g_tab[i]
 * (decode is monotone in the code for non-negative codes). */
static double g_tab[127];
static pthread_once_t g_tab_once = PTHREAD_ONCE_INIT;
static void build_table(void) {
    for (int i = 0; i < 127; ++i) g_tab[i] = oracle_e4m3_decode((uint8_t)i);
}

/* Nearest E4M3 value to q with ties to the even code; saturating at 448; sign kept. */
uint8_t oracle_e4m3_encode(float q) {
    pthread_once(&g_tab_once, build_table);
    if (isnan(q)) return signbit(q) ? 0xFF : 0x7F;
    uint8_t sign = signbit(q) ? 0x80 : 0x00;
    double a = fabs((double)q); /* exact widening */
    if (a >= 448.0) return sign | 0x7E; /* satfinite (reading Q7) */
    /* find i with g_tab[i] <= a < g_tab[i+1] (binary search over the ascending table) */
    int lo = 0, hi = 126; /* invariant: g_tab[lo] <= a < g_tab[hi] */
    while (hi - lo > 1) {
        int mid = (lo + hi) / 2;
        if (g_tab[mid] <= a)
            lo = mid;
        else
            hi = mid;
    }
    /* the midpoint of two adjacent E4M3 values has <= 5 significant bits: exact in double */
    double midpoint = 0.5 * (g_tab[lo] + g_tab[hi]);
    int code;
    if (a < midpoint)
        code = lo;
    else if (a > midpoint)
        code = hi;
    else
        code = (lo % 2 == 0) ? lo : hi; /* tie: even code (mantissa LSB 0) */
    return sign | (uint8_t)code;
}

/* O2 over an array (for the all-2^32 hardware comparison; same function per element). */
typedef struct {
    const float* q;
    uint8_t* out;
} enc_ctx;
static void enc_range(void* p, int64_t begin, int64_t end);

/* BF16 is the upper half of a binary32: widening is exact. */
float oracle_bf16_to_float(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* ------------------------------------------------------------------ O4: scale */
/* s = RN32(amax / 448) (one IEEE binary32 division), amax == 0 -> 1. */
float oracle_block_scale(float amax) {
    if (amax == 0.0f) return 1.0f;
    volatile float num = amax; /* keep it one binary32 division */
    return num / 448.0f;
}

/* ------------------------------------------------------------------ O5: element */
/* code = O2(RN32(x / s)), Eq. (1) with reading Q3. */
uint8_t oracle_quantize_element(float x, float s) {
    volatile float q = x / s;
    return oracle_e4m3_encode(q);
}

/* ------------------------------------------------------------------ threading helper */
typedef void (*range_fn)(void* ctx, int64_t begin, int64_t end);
typedef struct {
    range_fn fn;
    void* ctx;
    int64_t begin, end;
} range_job;
static void* range_trampoline(void* p) {
    range_job* j = (range_job*)p;
    j->fn(j->ctx, j->begin, j->end);
    return NULL;
}
/* Run fn over [0, total) split into nthreads contiguous ranges.  No arithmetic changes. */
static void parallel_for(range_fn fn, void* ctx, int64_t total, int nthreads) {
    if (nthreads <= 1 || total <= 1) {
        fn(ctx, 0, total);
        return;
    }
    if (nthreads > 256) nthreads = 256;
    if (nthreads > total) nthreads = (int)total;
    pthread_t th[256];
    range_job jobs[256];
    int64_t chunk = (total + nthreads - 1) / nthreads;
    int launched = 0;
    for (int t = 0; t < nthreads; ++t) {
        int64_t b = t * chunk, e = b + chunk;
        if (b >= total) break;
        if (e > total) e = total;
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].begin = b;
        jobs[t].end = e;
        if (pthread_create(&th[t], NULL, range_trampoline, &jobs[t]) != 0) {
            fn(ctx, b, e); /* fall back to running the range inline */
            jobs[t].fn = NULL;
        }
        launched = t + 1;
    }
    for (int t = 0; t < launched; ++t)
        if (jobs[t].fn) pthread_join(th[t], NULL);
}

static void enc_range(void* p, int64_t begin, int64_t end) {
    enc_ctx* c = (enc_ctx*)p;
    for (int64_t i = begin; i < end; ++i) c->out[i] = oracle_e4m3_encode(c->q[i]);
}

void oracle_e4m3_encode_array(const float* q, int64_t n, uint8_t* out, int nthreads) {
    enc_ctx c = {q, out};
    parallel_for(enc_range, &c, n, nthreads);
}

/* ------------------------------------------------------------------ weights (O3-O6) */
/* codes[i][j] = O5(w[i][j], s(block(i/128, j/128))); scales[bi][bj] = O4(amax(block)).
 * Block (bi, bj) covers rows [128 bi, min(128 bi + 128, n)) and columns
 * [128 bj, min(128 bj + 128, k)) (ragged edges clipped; reading Q12). */
typedef struct {
    const uint16_t* w;
    int64_t n, k, ld_w;
    uint8_t* codes;
    int64_t ld_q;
    float* scales;
    int64_t ld_s;
    int64_t nbk;
    volatile int nonfinite;
} wq_ctx;

static void wq_range(void* p, int64_t begin, int64_t end) {
    wq_ctx* c = (wq_ctx*)p;
    for (int64_t blk = begin; blk < end; ++blk) {
        int64_t bi = blk / c->nbk, bj = blk % c->nbk;
        int64_t r0 = bi * 128, r1 = r0 + 128 < c->n ? r0 + 128 : c->n;
        int64_t c0 = bj * 128, c1 = c0 + 128 < c->k ? c0 + 128 : c->k;
        /* O3: block amax over the in-bounds elements */
        float amax = 0.0f;
        for (int64_t i = r0; i < r1; ++i)
            for (int64_t j = c0; j < c1; ++j) {
                float x = oracle_bf16_to_float(c->w[i * c->ld_w + j]);
                if (!isfinite(x)) c->nonfinite = 1;
                float ax = fabsf(x);
                if (ax > amax) amax = ax;
            }
        /* O4 */
        float s = oracle_block_scale(amax);
        c->scales[bi * c->ld_s + bj] = s;
        /* O5 */
        for (int64_t i = r0; i < r1; ++i)
            for (int64_t j = c0; j < c1; ++j)
                c->codes[i * c->ld_q + j] =
                    oracle_quantize_element(oracle_bf16_to_float(c->w[i * c->ld_w + j]), s);
    }
}

int oracle_quantize_weight_blockwise(const uint16_t* w, int64_t n, int64_t k, int64_t ld_w,
                                     uint8_t* codes, int64_t ld_q, float* scales, int64_t ld_s,
                                     int nthreads) {
    if (n < 0 || k < 0 || ld_w < k || ld_q < k) return ORACLE_EINVAL;
    int64_t nbn = (n + 127) / 128, nbk = (k + 127) / 128;
    if (ld_s < nbk) return ORACLE_EINVAL;
    wq_ctx c = {w, n, k, ld_w, codes, ld_q, scales, ld_s, nbk, 0};
    parallel_for(wq_range, &c, nbn * nbk, nthreads);
    return c.nonfinite ? ORACLE_ENONFINITE : ORACLE_OK;
}

/* ------------------------------------------------------------------ activations (O3-O6) */
/* Per token m and 128-channel group g (PAPER.md:65 dynamic; PAPER.md:233 1x128 tiles):
 * scales[m][g] = O4(max_{j in g} |x[m][j]|), codes[m][j] = O5(x[m][j], scales[m][g]).
 * The scale array here is the LOGICAL [m][k/128] row-major layout (reading Q21). */
typedef struct {
    const uint16_t* x;
    int64_t m, k, ld_x;
    uint8_t* codes;
    int64_t ld_q;
    float* scales;
    int64_t ng;
    volatile int nonfinite;
} aq_ctx;

static void aq_range(void* p, int64_t begin, int64_t end) {
    aq_ctx* c = (aq_ctx*)p;
    for (int64_t item = begin; item < end; ++item) {
        int64_t row = item / c->ng, g = item % c->ng;
        const uint16_t* xr = c->x + row * c->ld_x + g * 128;
        float amax = 0.0f;
        for (int j = 0; j < 128; ++j) {
            float v = oracle_bf16_to_float(xr[j]);
            if (!isfinite(v)) c->nonfinite = 1;
            float av = fabsf(v);
            if (av > amax) amax = av;
        }
        float s = oracle_block_scale(amax);
        c->scales[row * c->ng + g] = s;
        for (int j = 0; j < 128; ++j)
            c->codes[row * c->ld_q + g * 128 + j] =
                oracle_quantize_element(oracle_bf16_to_float(xr[j]), s);
    }
}

int oracle_quantize_act_per_token_group(const uint16_t* x, int64_t m, int64_t k, int64_t ld_x,
                                        uint8_t* codes, int64_t ld_q, float* scales,
                                        int nthreads) {
    if (m < 0 || k < 0 || k % 128 != 0 || ld_x < k || ld_q < k) return ORACLE_EINVAL;
    aq_ctx c = {x, m, k, ld_x, codes, ld_q, scales, k / 128, 0};
    parallel_for(aq_range, &c, m * (k / 128), nthreads);
    return c.nonfinite ? ORACLE_ENONFINITE : ORACLE_OK;
}

/* ------------------------------------------------------------------ O7: GEMM reference */
/* out[r][n] = sum_k (dec(a[rows[r]][k]) * sa[rows[r]][k/128]) * (dec(b[n][k]) * sb[n/128][k/128])
 * in binary64, k ascending.  sa is the LOGICAL [m][k/128] activation-scale array (ld_sa
 * elements per row); sb is [ceil(n/128)][k/128] with ld_sb elements per row.  Each
 * dequantized operand is exact in binary64 (4-bit code significand x 24-bit scale). */
typedef struct {
    const uint8_t* a;
    int64_t ld_a;
    const float* sa;
    int64_t ld_sa;
    const uint8_t* b;
    int64_t ld_b;
    const float* sb;
    int64_t ld_sb;
    int64_t n, k;
    const int64_t* rows;
    double* out;
} gemm_ctx;

/* Work items are (row, 64-column block) pairs so that a small row sample still spreads over
 * every host thread; each output element is computed exactly as written above (same
 * operands, same k order) whichever thread owns it. */
#define GEMM_COLS_PER_ITEM 64
static void gemm_range(void* p, int64_t begin, int64_t end) {
    gemm_ctx* c = (gemm_ctx*)p;
    pthread_once(&g_tab_once, build_table);
    int64_t ncb = (c->n + GEMM_COLS_PER_ITEM - 1) / GEMM_COLS_PER_ITEM;
    for (int64_t item = begin; item < end; ++item) {
        int64_t r = item / ncb, cb = item % ncb;
        int64_t row = c->rows[r];
        const uint8_t* ar = c->a + row * c->ld_a;
        int64_t col1 = (cb + 1) * GEMM_COLS_PER_ITEM < c->n ? (cb + 1) * GEMM_COLS_PER_ITEM : c->n;
        for (int64_t col = cb * GEMM_COLS_PER_ITEM; col < col1; ++col) {
            const uint8_t* br = c->b + col * c->ld_b;
            double acc = 0.0;
            for (int64_t kk = 0; kk < c->k; ++kk) {
                double av = oracle_e4m3_decode(ar[kk]) * (double)c->sa[row * c->ld_sa + kk / 128];
                double bv = oracle_e4m3_decode(br[kk]) *
                            (double)c->sb[(col / 128) * c->ld_sb + kk / 128];
                acc += av * bv;
            }
            c->out[r * c->n + col] = acc;
        }
    }
}

int oracle_gemm_rows(const uint8_t* a, int64_t ld_a, const float* sa, int64_t ld_sa,
                     const uint8_t* b, int64_t ld_b, const float* sb, int64_t ld_sb, int64_t n,
                     int64_t k, const int64_t* rows, int64_t nrows, double* out, int nthreads) {
    if (n < 0 || k < 0 || k % 128 != 0 || nrows < 0) return ORACLE_EINVAL;
    gemm_ctx c = {a, ld_a, sa, ld_sa, b, ld_b, sb, ld_sb, n, k, rows, out};
    parallel_for(gemm_range, &c, nrows * ((n + GEMM_COLS_PER_ITEM - 1) / GEMM_COLS_PER_ITEM), nthreads);
    return ORACLE_OK;
}

/* ================================================================== NEXT-2: producers
 * the activation quantizer's producers on the Qwen3 rollout forward,
 * RMSNorm (input of qkv and gate_up) and SiLU(gate) * up (input of down_proj).  The
 * unfused pipeline materialises the producer's output in BF16 and then quantizes it
 * (PAPER.md:65,73).  The producers themselves (readings N1, N2) live in oracle/producers.py
 * (exact integer / rational / decimal arithmetic); this file keeps the binary64 -> BF16
 * rounding helper.
 */

/* binary64 -> BF16 bits, round to nearest even (direct: no double rounding through fp32). */
uint16_t oracle_f64_to_bf16(double d) {
    if (isnan(d)) return 0x7FC0;
    uint16_t sign = signbit(d) ? 0x8000 : 0;
    double a = fabs(d);
    if (a == 0.0) return sign;
    if (isinf(a)) return sign | 0x7F80;
    int e;
    frexp(a, &e); /* a = f * 2^e, f in [0.5, 1) */
    /* quantum of the result: 2^(e-8) for normals (8 significant bits), 2^-133 below 2^-126 */
    int qexp = e - 8;
    if (qexp < -133) qexp = -133;
    double r = nearbyint(ldexp(a, -qexp)); /* RNE, exact */
    double v = ldexp(r, qexp);
    if (v > 3.3895313892515355e38) return sign | 0x7F80; /* overflow to inf */
    float f = (float)v; /* exact: <= 8 significant bits */
    uint32_t u;
    memcpy(&u, &f, 4);
    return sign | (uint16_t)((u >> 16) & 0x7FFF);
}

/* ================================================================== NEXT-3: FP8 KV cache
 * PAPER.md §2.3.1 (lines 159-166) "dynamic QKV scale recalibration": per layer, the K (and V,
 * Q) scale is recomputed from the first forward after every weight sync (inference side) or
 * from a calibration subset (trainer side), then K/V are stored as FP8 E4M3.  Readings
 * (K1-K4):
 *   K1  calibration scale = O4 applied to the per-tensor amax over every calibration
 *       element:  s = RN32(amax / 448), amax == 0 -> 1   (one scalar per layer and tensor);
 *       several calibration batches: amax is the max over all of them (set-monotone).
 *   K2  stored code = O5:  O2(RN32(x / s))   (the same element map as the weights).
 *   K3  values beyond the calibrated range saturate (O2's +-448), and are COUNTED: an
 *       element is saturated iff |RN32(x / s)| >= 464, i.e. iff the satfinite clamp
 *       decides its code (464 is the midpoint between 448 and the next E4M3 binade's 480).
 *   K4  append: token row r of the new K (or V) is written to cache row slot[r]
 *       (slot = identity when no mapping is given).
 */

/* K1: amax over a BF16 [rows, cols] matrix (row stride ld), exact; returns 1 if any element
 * is NaN/Inf (and leaves *amax undefined), else 0. */
int oracle_kv_amax(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld, float* amax) {
    float a = 0.0f;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            float v = fabsf(oracle_bf16_to_float(x[r * ld + c]));
            if (!isfinite(v)) return ORACLE_ENONFINITE;
            if (v > a) a = v;
        }
    *amax = a;
    return ORACLE_OK;
}

/* K2-K4: quantize rows of x with the scalar scale s into cache rows slot[r] (slot may be
 * NULL = identity); returns the number of saturated elements (K3). */
int64_t oracle_kv_quantize_append(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld, float s,
                                  const int32_t* slot, uint8_t* cache, int64_t ld_cache) {
    int64_t saturated = 0;
    for (int64_t r = 0; r < rows; ++r) {
        int64_t dst = slot ? (int64_t)slot[r] : r;
        for (int64_t c = 0; c < cols; ++c) {
            float v = oracle_bf16_to_float(x[r * ld + c]);
            volatile float q = v / s;
            if (fabsf(q) >= 464.0f) ++saturated;
            cache[dst * ld_cache + c] = oracle_e4m3_encode(q);
        }
    }
    return saturated;
}

/* ================================================================== NEXT-4: MXFP8 variant
 * SURVEY §8(f) NEXT-4 ("Blackwell ... FP8"): power-of-two (UE8M0) scales on
 * 1x32 blocks along K for both operands, so the tensor core applies them inside the MMA
 * (tcgen05 kind::mxf8f6f4.block_scale) and no per-k-block promotion is needed.  A DIFFERENT
 * quantizer from the paper's amax/448 (readings X1-X3):
 *   X1  block: 32 consecutive elements of a row along K (tokens for activations, output rows
 *       for weights); ragged tail blocks use the in-bounds elements.
 *   X2  scale: the smallest power of two s = 2^e with 448 s >= amax (no element saturates),
 *       e clamped to >= -127 (the E8M0 range; codes of such tiny blocks are 0 anyway);
 *       amax == 0 -> e = 0.  Stored as the E8M0 byte e + 127.
 *   X3  code: O2(x / s) -- the division by a power of two is exact (a quotient that would be
 *       an fp32 subnormal is < 2^-126, far below the E4M3 rounding point 2^-10).
 */
int oracle_mx_exponent(float amax) {
    if (amax == 0.0f) return 0;
    int e = -127;
    while (448.0 * ldexp(1.0, e) < (double)amax) ++e; /* smallest e with 448 2^e >= amax */
    return e;
}

/* rows x cols BF16 (row stride ld) -> codes [rows][cols], scale bytes [rows][ceil(cols/32)] */
int oracle_mx_quantize(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld, uint8_t* codes,
                       uint8_t* sf) {
    int64_t nb = (cols + 31) / 32;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t b = 0; b < nb; ++b) {
            int64_t c0 = b * 32, c1 = c0 + 32 < cols ? c0 + 32 : cols;
            float amax = 0.0f;
            for (int64_t c = c0; c < c1; ++c) {
                float v = fabsf(oracle_bf16_to_float(x[r * ld + c]));
                if (!isfinite(v)) return ORACLE_ENONFINITE;
                if (v > amax) amax = v;
            }
            int e = oracle_mx_exponent(amax);
            sf[r * nb + b] = (uint8_t)(e + 127);
            for (int64_t c = c0; c < c1; ++c) {
                double q = (double)oracle_bf16_to_float(x[r * ld + c]) / ldexp(1.0, e); /* exact */
                codes[r * cols + c] = oracle_e4m3_encode((float)q);
            }
        }
    return ORACLE_OK;
}

/* fp64 reference of the MXFP8 GEMM for the listed rows:
 *   Y[m,n] = sum_k dec(a[m,k]) 2^(sfa[m,k/32]-127) dec(b[n,k]) 2^(sfb[n,k/32]-127)          */
int oracle_mx_gemm_rows(const uint8_t* a, const uint8_t* sfa, const uint8_t* b, const uint8_t* sfb,
                        int64_t n, int64_t k, const int64_t* rows, int64_t nrows, double* out) {
    int64_t nb = (k + 31) / 32;
    for (int64_t i = 0; i < nrows; ++i) {
        int64_t m = rows[i];
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int64_t kk = 0; kk < k; ++kk) {
                double av = oracle_e4m3_decode(a[m * k + kk]) * ldexp(1.0, (int)sfa[m * nb + kk / 32] - 127);
                double bv = oracle_e4m3_decode(b[j * k + kk]) * ldexp(1.0, (int)sfb[j * nb + kk / 32] - 127);
                acc += av * bv;
            }
            out[i * n + j] = acc;
        }
    }
    return ORACLE_OK;
}
