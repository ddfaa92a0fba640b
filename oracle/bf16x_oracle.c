/*
 * oracle/bf16x_oracle.c -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct C99 implementation of what the paper
 * (Henry, Tang, Heinecke, arXiv 1904.06376; /root/reference/PAPER.md, cited as
 * P:<line>) computes on the hot path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header or constant with paper_1904_06376_b200/ (the product),
 * and the product never loads it.
 *
 * Build flags (Makefile): -O2 -fno-fast-math -ffp-contract=off, no FTZ/DAZ, so
 * every FP32 operation below is one IEEE-754 round-to-nearest-even operation
 * and subnormals are kept (reading R6).
 *
 * Storage is column-major (BLAS): element (i,j) of X is X[i + j*ldx].
 *
 * Functions and the passage each follows:
 *   orc_bf16_round        (B16) operator, §II-A; readings R1, R3, R4
 *   orc_bf16_widen        (F32) operator, §II-A (exact widening)
 *   orc_split             3-way split, §II-A; readings R4, R5
 *   orc_partial           Z^(i,j) partial inner products, §II-D
 *   orc_gemm_split_cols   bins Z^(0..4) P:257-265, Z_2 (x6) P:269-272,
 *                         x3 P:378-380, x9 reading R9 ("smallest to
 *                         largest"), x8 = Z_3 P:274-277; alpha/beta R19
 *   orc_split_scaled      N2 power-of-two scaled pieces (SURVEY 8(f) N2 on
 *                         P:344-351; reading R29): b1, b2 stored times 2^8, 2^16
 *   orc_gemm_split_ex_cols  the split GEMM with options: scaled pieces (R29)
 *                         and/or the final combine in FP64 ("d", P:420,
 *                         P:425 caption "collect the final answer with d";
 *                         reading R30)
 *   orc_sgemm_fma_cols    FP32 FMA reference dot product, §II-C
 *   orc_dgemm_cols        FP64 reference ("DGEMM")
 *   orc_getrf_split       blocked right-looking LU with partial pivoting
 *                         whose trailing update is the split GEMM
 *                         (§III; §IV-A)
 *   orc_lu_solve_f64      FP64 triangular solves with the low-precision
 *                         factors ("do the solve in a higher precision")
 *
 * Pins: tests/test_oracle_*.py (values the paper prints, closed forms,
 * brute force, library special cases).  Parity status per function is listed
 * in DESIGN.md section "Oracle pins".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* bit views                                                                */
/* ------------------------------------------------------------------------ */
static uint32_t bits_of(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float float_of(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* ------------------------------------------------------------------------ */
/* O-1  (B16) conversion operator.  P:177-179 (§II-A): "(F32) and (B16) shall
 * denote the conversion operator to the respective type".  The paper does not
 * state the rounding; R1 reads round-to-nearest-even (the only
 * reading consistent with the 1/768 statistic of P:372).  R3: a finite value
 * whose RNE result would be +-Inf saturates to the largest finite BF16
 * (+-0x7F7F).  R4: NaN -> 0x7FC0.  Subnormals are rounded like any other
 * pattern (no flush).
 *
 * BF16 is the top half of an FP32 pattern ("BF16 cuts 16 bits from
 * the 24-bit FP32 mantissa").  Sign-magnitude encoding means incrementing the
 * truncated 16-bit pattern moves one BF16 ulp away from zero, so rounding to
 * nearest is: keep the top 16 bits, and add one when the discarded 16 bits are
 * more than half an ulp (> 0x8000), or exactly half and the kept pattern is odd.
 * ------------------------------------------------------------------------ */
uint16_t orc_bf16_round(float x)
{
    uint32_t u = bits_of(x);
    uint32_t exponent = (u >> 23) & 0xFFu;
    uint32_t mantissa = u & 0x7FFFFFu;
    if (exponent == 0xFFu) {
        if (mantissa != 0) return 0x7FC0u;          /* NaN (R4) */
        return (uint16_t)(u >> 16);                 /* +-Inf stays +-Inf */
    }
    uint32_t kept = u >> 16;
    uint32_t discarded = u & 0xFFFFu;
    if (discarded > 0x8000u || (discarded == 0x8000u && (kept & 1u)))
        kept += 1u;                                 /* round magnitude up */
    if ((kept & 0x7FFFu) == 0x7F80u)                /* rounded to Inf (R3) */
        kept -= 1u;                                 /* -> +-0x7F7F */
    return (uint16_t)kept;
}

/* (F32) widening of a BF16 pattern: exact. */
float orc_bf16_widen(uint16_t b) { return float_of((uint32_t)b << 16); }

/* ------------------------------------------------------------------------ */
/* O-2  split.  P:180-184 (§II-A):
 *    b0 = (B16) a
 *    b1 = (B16)((F32)(a - (F32)b0))
 *    b2 = (B16)((F32)(a - (F32)b0 - (F32)b1))
 * The subtraction in b2 is evaluated left to right, (a - b0) - b1 (R5); each
 * subtraction is one FP32 operation.  Non-finite a: (bf16(a), +0, +0) (R4).
 * ------------------------------------------------------------------------ */
static void split_scalar(float a, uint16_t *b0, uint16_t *b1, uint16_t *b2)
{
    uint16_t p0 = orc_bf16_round(a);
    if (!isfinite(a)) { *b0 = p0; *b1 = 0; *b2 = 0; return; }
    float r1 = a - orc_bf16_widen(p0);
    uint16_t p1 = orc_bf16_round(r1);
    float r2 = r1 - orc_bf16_widen(p1);
    uint16_t p2 = orc_bf16_round(r2);
    *b0 = p0; *b1 = p1; *b2 = p2;
}

/* Split n consecutive FP32 values (any may be NaN/Inf).  b1/b2 may be NULL. */
void orc_split(int64_t n, const float *x, uint16_t *b0, uint16_t *b1, uint16_t *b2)
{
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < n; ++i) {
        uint16_t p0, p1, p2;
        split_scalar(x[i], &p0, &p1, &p2);
        b0[i] = p0;
        if (b1) b1[i] = p1;
        if (b2) b2[i] = p2;
    }
}

/* Split all 2^32 bit patterns in [first, first+count) (for the exhaustive
 * parity sweep: the oracle generates the patterns itself). */
void orc_split_patterns(uint64_t first, int64_t count, uint16_t *b0, uint16_t *b1, uint16_t *b2)
{
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < count; ++i) {
        uint16_t p0, p1, p2;
        split_scalar(float_of((uint32_t)(first + (uint64_t)i)), &p0, &p1, &p2);
        b0[i] = p0; b1[i] = p1; b2[i] = p2;
    }
}

/* ------------------------------------------------------------------------ */
/* N2 scaled pieces (reading R29).  P:344-351 (§II-F) explains that the split
 * loses bits when the pieces b1, b2 fall below the BF16 normal range (exponent
 * "no smaller than -110").  The scaled split keeps each residual at the
 * magnitude of x by multiplying it by 2^8 before it is rounded:
 *    b0  = (B16) a
 *    s1  = (F32)(a - (F32)b0) * 2^8        (one subtraction, one multiply)
 *    b1' = (B16) s1
 *    s2  = (F32)(s1 - (F32)b1') * 2^8
 *    b2' = (B16) s2
 * so that a = b0 + 2^-8 b1' + 2^-16 b2' (exactly, for every finite a; pinned
 * in tests/test_oracle_scaled.py).  Multiplying by 2^8 is exact in FP32 here
 * (no overflow: |a - b0| <= 2^119).  Non-finite a: (bf16(a), +0, +0) (R4).
 * ------------------------------------------------------------------------ */
static void split_scalar_scaled(float a, uint16_t *b0, uint16_t *b1, uint16_t *b2)
{
    uint16_t p0 = orc_bf16_round(a);
    if (!isfinite(a)) { *b0 = p0; *b1 = 0; *b2 = 0; return; }
    float s1 = (a - orc_bf16_widen(p0)) * 256.0f;
    uint16_t p1 = orc_bf16_round(s1);
    float s2 = (s1 - orc_bf16_widen(p1)) * 256.0f;
    uint16_t p2 = orc_bf16_round(s2);
    *b0 = p0; *b1 = p1; *b2 = p2;
}

void orc_split_scaled(int64_t n, const float *x, uint16_t *b0, uint16_t *b1, uint16_t *b2)
{
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < n; ++i) {
        uint16_t p0, p1, p2;
        split_scalar_scaled(x[i], &p0, &p1, &p2);
        b0[i] = p0;
        if (b1) b1[i] = p1;
        if (b2) b2[i] = p2;
    }
}

void orc_split_scaled_patterns(uint64_t first, int64_t count, uint16_t *b0, uint16_t *b1, uint16_t *b2)
{
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < count; ++i) {
        uint16_t p0, p1, p2;
        split_scalar_scaled(float_of((uint32_t)(first + (uint64_t)i)), &p0, &p1, &p2);
        b0[i] = p0; b1[i] = p1; b2[i] = p2;
    }
}

/* ------------------------------------------------------------------------ */
/* Split an FP32 column-major matrix into 3 FP32 planes holding the (exactly
 * widened) BF16 pieces, packed with leading dimension `rows`. */
static void split_matrix_widened_opt(int rows, int cols, const float *X, int ldx, float *P[3], int scaled)
{
    int64_t j;
#pragma omp parallel for schedule(static)
    for (j = 0; j < cols; ++j) {
        for (int i = 0; i < rows; ++i) {
            uint16_t p0, p1, p2;
            if (scaled) split_scalar_scaled(X[i + j * (int64_t)ldx], &p0, &p1, &p2);
            else split_scalar(X[i + j * (int64_t)ldx], &p0, &p1, &p2);
            int64_t o = i + j * (int64_t)rows;
            P[0][o] = orc_bf16_widen(p0);
            P[1][o] = orc_bf16_widen(p1);
            P[2][o] = orc_bf16_widen(p2);
        }
    }
}

static void split_matrix_widened(int rows, int cols, const float *X, int ldx, float *P[3])
{
    split_matrix_widened_opt(rows, cols, X, ldx, P, 0);
}

/* ------------------------------------------------------------------------ */
/* O-3  one partial inner-product column.  P:247-255 (§II-D), P:253 literally:
 *    Z^(i,j) <- 0;  for l = 1..n:  Z^(i,j) <- FMA(x_l^(i), y_l^(j), Z^(i,j))
 * one fused multiply-add (one rounding) per term (R10).  A BF16 x BF16 product
 * has <= 16 significant bits, so the FMA equals a multiply followed by an add
 * wherever the product is a normal FP32 number; where it is subnormal in FP32
 * (|product| < 2^-126) the separate multiply would round it first, so the FMA
 * is spelled out.  For every output row r the sum runs over l strictly in
 * increasing order; the loop over r is only a vectorisable sweep across
 * independent outputs.
 *   Ai: m x k piece plane (ld m), bj: column c of a k x n piece plane.
 * ------------------------------------------------------------------------ */
static void partial_column(int m, int k, const float *Ai, const float *bj, float *Z)
{
    for (int r = 0; r < m; ++r) Z[r] = 0.0f;
    for (int l = 0; l < k; ++l) {
        const float y = bj[l];
        const float *a = Ai + (int64_t)l * m;
        for (int r = 0; r < m; ++r) Z[r] = fmaf(a[r], y, Z[r]);   /* one rounding */
    }
}

/* Public: the 9 (or fewer) Z^(i,j) planes of an m x n x k problem, for bound
 * audits.  Z must hold 9*m*ncols floats, plane (i,j) at offset (3*i+j)*m*ncols;
 * cols lists the output columns to compute (NULL = 0..n-1, ncols = n). */
int orc_partials(int m, int n, int k, const float *A, int lda, const float *B, int ldb,
                 const int *cols, int ncols, float *Z)
{
    if (m <= 0 || ncols <= 0) return 0;
    float *Ap[3], *Bp[3];
    for (int p = 0; p < 3; ++p) {
        Ap[p] = (float *)malloc(sizeof(float) * (size_t)m * (size_t)(k > 0 ? k : 1));
        Bp[p] = (float *)malloc(sizeof(float) * (size_t)(k > 0 ? k : 1) * (size_t)n);
    }
    split_matrix_widened(m, k, A, lda, Ap);
    split_matrix_widened(k, n, B, ldb, Bp);
    int64_t t;
#pragma omp parallel for schedule(dynamic)
    for (t = 0; t < ncols; ++t) {
        int c = cols ? cols[t] : (int)t;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                partial_column(m, k, Ap[i], Bp[j] + (int64_t)c * k,
                               Z + ((size_t)(3 * i + j) * ncols + (size_t)t) * m);
    }
    for (int p = 0; p < 3; ++p) { free(Ap[p]); free(Bp[p]); }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O-4  bins and their combination, P:257-277 (§II-D), P:376-380 (§II-G):
 *    Z0 = Z00;  Z1 = Z01 + Z10;  Z2 = Z02 + (Z11 + Z20);  Z3 = Z12 + Z21;  Z4 = Z22
 *    x3 (pair of BF16, 3 products):  Z0 + Z1
 *    x6 (Z_2):                            Z0 + (Z1 + Z2)
 *    x8 (Z_3):                            Z0 + (Z1 + (Z2 + Z3))
 *    x9 (all nine, R9, "bins ... added from smallest to largest"):
 *                                                Z0 + (Z1 + (Z2 + (Z3 + Z4)))
 *    x7 ("computing at least 7 products instead of just 6": x6 plus the
 *        2^-24-bin term a1*b2 of the worked example, R27):
 *                                                Z0 + (Z1 + (Z2 + Z^(1,2)))
 *    x5 (A split in two, B in three: "taking only the a1 b1 and a0 b2 terms
 *        from the 2^-16 bin", R27):               Z0 + (Z1 + (Z^(0,2) + Z^(1,1)))
 *    1  (single BF16, debug):             Z0
 * all in FP32 round-to-nearest.
 * O-5  C = alpha*Z + beta*C (BLAS, R19): beta == 0 never reads C, the product
 * is formed as fmaf(alpha, Z, beta*C).
 * ------------------------------------------------------------------------ */
static int variant_pieces(int variant)
{
    switch (variant) { case 1: return 1; case 3: return 2; case 5: case 6: case 7: case 8: case 9: return 3; }
    return 0;
}

static float combine_bins(int variant, const float Z[3][3])
{
    float Z0 = Z[0][0];
    float Z1 = Z[0][1] + Z[1][0];
    float Z2 = Z[0][2] + (Z[1][1] + Z[2][0]);
    float Z3 = Z[1][2] + Z[2][1];
    float Z4 = Z[2][2];
    switch (variant) {
    case 1: return Z0;
    case 3: return Z0 + Z1;
    case 5: return Z0 + (Z1 + (Z[0][2] + Z[1][1]));
    case 6: return Z0 + (Z1 + Z2);
    case 7: return Z0 + (Z1 + (Z2 + Z[1][2]));
    case 8: return Z0 + (Z1 + (Z2 + Z3));
    case 9: return Z0 + (Z1 + (Z2 + (Z3 + Z4)));
    }
    return NAN;
}

/* N2 scaled pieces (R29): Z'^(i,j) are the partial sums of the scaled pieces,
 * so bin s is held at 2^(8s) times its unscaled value.  Bins are still added
 * smallest first, each partial result brought down one bin with
 * an FP32 multiply by q = 2^-8 (Horner form; exact unless it underflows):
 *    x6: Z'0 + (Z'1 + Z'2*q)*q,  x9: Z'0 + (Z'1 + (Z'2 + (Z'3 + Z'4*q)*q)*q)*q
 * When no scaling underflows this equals combine_bins on the unscaled pieces
 * bit for bit (power-of-two scaling commutes with round-to-nearest). */
static float combine_bins_scaled(int variant, const float Z[3][3])
{
    const float q = 0x1p-8f;
    float Z0 = Z[0][0];
    float Z1 = Z[0][1] + Z[1][0];
    float Z2 = Z[0][2] + (Z[1][1] + Z[2][0]);
    float Z3 = Z[1][2] + Z[2][1];
    float Z4 = Z[2][2];
    switch (variant) {
    case 1: return Z0;
    case 3: return Z0 + Z1 * q;
    case 5: return Z0 + (Z1 + (Z[0][2] + Z[1][1]) * q) * q;
    case 6: return Z0 + (Z1 + Z2 * q) * q;
    case 7: return Z0 + (Z1 + (Z2 + Z[1][2] * q) * q) * q;
    case 8: return Z0 + (Z1 + (Z2 + Z3 * q) * q) * q;
    case 9: return Z0 + (Z1 + (Z2 + (Z3 + Z4 * q) * q) * q) * q;
    }
    return NAN;
}

/* "d" variants (R30): "the same as the last but adding the final
 * results together in FP64"; P:425 caption "Optionally, collect the final
 * answer with d (double precision)".  The FP32 partial sums Z^(i,j) of O-3
 * are widened (exactly) and every addition of the combine -- inside the bins
 * and between them, in the order of combine_bins -- is one FP64 operation;
 * the result is rounded once to FP32.  scaled: the Z' of R29, brought down by
 * exact FP64 multiplies by 2^-8. */
static float combine_bins_f64(int variant, const float Zf[3][3], int scaled)
{
    const double q = scaled ? 0x1p-8 : 1.0;
    double Z[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Z[i][j] = (double)Zf[i][j];
    double Z0 = Z[0][0];
    double Z1 = Z[0][1] + Z[1][0];
    double Z2 = Z[0][2] + (Z[1][1] + Z[2][0]);
    double Z3 = Z[1][2] + Z[2][1];
    double Z4 = Z[2][2];
    double r;
    switch (variant) {
    case 1: r = Z0; break;
    case 3: r = Z0 + Z1 * q; break;
    case 5: r = Z0 + (Z1 + (Z[0][2] + Z[1][1]) * q) * q; break;
    case 6: r = Z0 + (Z1 + Z2 * q) * q; break;
    case 7: r = Z0 + (Z1 + (Z2 + Z[1][2] * q) * q) * q; break;
    case 8: r = Z0 + (Z1 + (Z2 + Z3 * q) * q) * q; break;
    case 9: r = Z0 + (Z1 + (Z2 + (Z3 + Z4 * q) * q) * q) * q; break;
    default: return NAN;
    }
    return (float)r;
}

static int product_needed(int variant, int i, int j)
{
    switch (variant) {
    case 1: return i + j == 0;
    case 3: return i + j <= 1;
    case 5: return i <= 1 && i + j <= 2;   /* A has pieces 0, 1 only */
    case 6: return i + j <= 2;
    case 7: return i + j <= 2 || (i == 1 && j == 2);
    case 8: return i + j <= 3;
    case 9: return 1;
    }
    return 0;
}

static float scale_output(float alpha, float z, float beta, float c_old)
{
    float bc = (beta == 0.0f) ? 0.0f : beta * c_old;
    return fmaf(alpha, z, bc);
}

/* Split GEMM on a list of output columns.
 *   C_out (m x ncols, ld m) receives alpha*A*B[:,cols] + beta*C_in[:,cols];
 *   C_in (m x n, ldc) may be NULL when beta == 0.
 * Quick returns (R19): alpha == 0 or k == 0 -> beta*C. */
/* mode bits: 1 = scaled pieces (R29), 2 = FP64 final combine (R30). */
int orc_gemm_split_ex_cols(int m, int n, int k, float alpha, const float *A, int lda,
                           const float *B, int ldb, float beta, const float *C_in, int ldc,
                           int variant, int mode, const int *cols, int ncols, float *C_out)
{
    const int scaled = (mode & 1) != 0, f64 = (mode & 2) != 0;
    if (mode & ~3) return -13;
    if (variant_pieces(variant) == 0) return -12;
    if (m <= 0 || ncols <= 0) return 0;
    int64_t t;
    if (alpha == 0.0f || k == 0) {
        for (t = 0; t < ncols; ++t) {
            int c = cols ? cols[t] : (int)t;
            for (int r = 0; r < m; ++r) {
                float cold = (beta == 0.0f) ? 0.0f : C_in[r + (int64_t)c * ldc];
                C_out[r + t * (int64_t)m] = (beta == 0.0f) ? 0.0f : beta * cold;
            }
        }
        return 0;
    }
    /* A is split whole (every output column needs every row); of B only the requested
     * columns are gathered (k x ncols, ld k) and split, so a column-sampled call costs the
     * sample, not the whole of B */
    float *Ap[3], *Bp[3];
    float *Bsel = (float *)malloc(sizeof(float) * (size_t)k * (size_t)ncols);
    for (int p = 0; p < 3; ++p) {
        Ap[p] = (float *)malloc(sizeof(float) * (size_t)m * (size_t)k);
        Bp[p] = (float *)malloc(sizeof(float) * (size_t)k * (size_t)ncols);
    }
    for (t = 0; t < ncols; ++t) {
        const int c = cols ? cols[t] : (int)t;
        memcpy(Bsel + (size_t)t * k, B + (int64_t)c * ldb, sizeof(float) * (size_t)k);
    }
    split_matrix_widened_opt(m, k, A, lda, Ap, scaled);
    split_matrix_widened_opt(k, ncols, Bsel, k, Bp, scaled);
    free(Bsel);
#pragma omp parallel
    {
        float *Zcol[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                Zcol[i][j] = (float *)malloc(sizeof(float) * (size_t)m);
#pragma omp for schedule(dynamic)
        for (t = 0; t < ncols; ++t) {
            int c = cols ? cols[t] : (int)t;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    if (product_needed(variant, i, j))
                        partial_column(m, k, Ap[i], Bp[j] + (int64_t)t * k, Zcol[i][j]);
                    else
                        for (int r = 0; r < m; ++r) Zcol[i][j][r] = 0.0f;
                }
            for (int r = 0; r < m; ++r) {
                float Z[3][3];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) Z[i][j] = Zcol[i][j][r];
                float z = f64 ? combine_bins_f64(variant, Z, scaled)
                              : (scaled ? combine_bins_scaled(variant, Z) : combine_bins(variant, Z));
                float cold = (beta == 0.0f) ? 0.0f : C_in[r + (int64_t)c * ldc];
                C_out[r + t * (int64_t)m] = scale_output(alpha, z, beta, cold);
            }
        }
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) free(Zcol[i][j]);
    }
    for (int p = 0; p < 3; ++p) { free(Ap[p]); free(Bp[p]); }
    return 0;
}

int orc_gemm_split_cols(int m, int n, int k, float alpha, const float *A, int lda,
                        const float *B, int ldb, float beta, const float *C_in, int ldc,
                        int variant, const int *cols, int ncols, float *C_out)
{
    return orc_gemm_split_ex_cols(m, n, k, alpha, A, lda, B, ldb, beta, C_in, ldc, variant, 0,
                                  cols, ncols, C_out);
}

/* Full split GEMM in place, BLAS sgemm('N','N') semantics. */
int orc_gemm_split(int m, int n, int k, float alpha, const float *A, int lda,
                   const float *B, int ldb, float beta, float *C, int ldc, int variant)
{
    if (variant_pieces(variant) == 0) return -12;
    if (m <= 0 || n <= 0) return 0;
    float *out = (float *)malloc(sizeof(float) * (size_t)m * (size_t)n);
    int rc = orc_gemm_split_cols(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, variant,
                                 NULL, n, out);
    for (int64_t c = 0; c < n; ++c)
        memcpy(C + c * (int64_t)ldc, out + c * (int64_t)m, sizeof(float) * (size_t)m);
    free(out);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* O-6  FP32 reference, P:219-225 (§II-C): Z <- 0; for l: Z <- FMA(x_l, y_l, Z)
 * (one rounding per step), then the O-5 scaling.  C_out is m x ncols. */
int orc_sgemm_fma_cols(int m, int n, int k, float alpha, const float *A, int lda,
                       const float *B, int ldb, float beta, const float *C_in, int ldc,
                       const int *cols, int ncols, float *C_out)
{
    (void)n;
    int64_t t;
#pragma omp parallel
    {
        float *Z = (float *)malloc(sizeof(float) * (size_t)(m > 0 ? m : 1));
#pragma omp for schedule(dynamic)
        for (t = 0; t < ncols; ++t) {
            int c = cols ? cols[t] : (int)t;
            for (int r = 0; r < m; ++r) Z[r] = 0.0f;
            for (int l = 0; l < k; ++l) {
                const float y = B[l + (int64_t)c * ldb];
                const float *a = A + (int64_t)l * lda;
                for (int r = 0; r < m; ++r) Z[r] = fmaf(a[r], y, Z[r]);
            }
            for (int r = 0; r < m; ++r) {
                float cold = (beta == 0.0f) ? 0.0f : C_in[r + (int64_t)c * ldc];
                C_out[r + t * (int64_t)m] = (alpha == 0.0f || k == 0)
                    ? ((beta == 0.0f) ? 0.0f : beta * cold)
                    : scale_output(alpha, Z[r], beta, cold);
            }
        }
        free(Z);
    }
    return 0;
}

/* FP64 reference product of FP32 data ("DGEMM"): every product of two
 * FP32 values is exact in FP64; the k-sum runs sequentially in FP64.
 * C64 is m x ncols (ld m), the plain product A*B[:,cols] (no alpha/beta). */
int orc_dgemm_cols(int m, int n, int k, const float *A, int lda, const float *B, int ldb,
                   const int *cols, int ncols, double *C64)
{
    (void)n;
    int64_t t;
#pragma omp parallel for schedule(dynamic)
    for (t = 0; t < ncols; ++t) {
        int c = cols ? cols[t] : (int)t;
        double *z = C64 + t * (int64_t)m;
        for (int r = 0; r < m; ++r) z[r] = 0.0;
        for (int l = 0; l < k; ++l) {
            const double y = (double)B[l + (int64_t)c * ldb];
            const float *a = A + (int64_t)l * lda;
            for (int r = 0; r < m; ++r) z[r] = z[r] + (double)a[r] * y;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O-7  LU with partial pivoting whose cubic work (the trailing update) runs in
 * the split GEMM, P:404-406 (§III): "Only the cubic work of the initial LU
 * factorization should be done in the lower precision".  Right-looking,
 * blocked by nb columns:
 *   panel  (FP32): for each column j: pivot = first index of max |A[i,j]|
 *                  (LAPACK isamax), swap whole rows, L column = A[i,j]/A[j,j],
 *                  rank-1 update of the remaining panel columns;
 *   U12    (FP32): forward substitution with the unit-lower L11;
 *   A22         : A22 <- -1 * L21 * U12 + 1 * A22 with orc_gemm_split(variant);
 *                 variant 0 = plain FP32 FMA update (the SGETRF comparator).
 * ipiv[j] = 0-based row swapped with j.  Returns 0, or j+1 for the first exact
 * zero pivot (the factorisation is abandoned there).
 * ------------------------------------------------------------------------ */
int orc_getrf_split(int n, float *A, int lda, int *ipiv, int nb, int variant)
{
    if (nb <= 0) nb = 64;
    for (int j0 = 0; j0 < n; j0 += nb) {
        int jb = (n - j0 < nb) ? n - j0 : nb;
        for (int j = j0; j < j0 + jb; ++j) {
            int p = j;
            float best = fabsf(A[j + (int64_t)j * lda]);
            for (int i = j + 1; i < n; ++i) {
                float v = fabsf(A[i + (int64_t)j * lda]);
                if (v > best) { best = v; p = i; }
            }
            ipiv[j] = p;
            if (A[p + (int64_t)j * lda] == 0.0f) return j + 1;
            if (p != j)
                for (int c = 0; c < n; ++c) {
                    float tmp = A[j + (int64_t)c * lda];
                    A[j + (int64_t)c * lda] = A[p + (int64_t)c * lda];
                    A[p + (int64_t)c * lda] = tmp;
                }
            float piv = A[j + (int64_t)j * lda];
            for (int i = j + 1; i < n; ++i) A[i + (int64_t)j * lda] = A[i + (int64_t)j * lda] / piv;
            for (int c = j + 1; c < j0 + jb; ++c) {
                float u = A[j + (int64_t)c * lda];
                for (int i = j + 1; i < n; ++i)
                    A[i + (int64_t)c * lda] = A[i + (int64_t)c * lda] - A[i + (int64_t)j * lda] * u;
            }
        }
        int j1 = j0 + jb, rest = n - j1;
        if (rest <= 0) continue;
        for (int c = j1; c < n; ++c)
            for (int j = j0; j < j1; ++j) {
                float u = A[j + (int64_t)c * lda];
                for (int i = j + 1; i < j1; ++i)
                    A[i + (int64_t)c * lda] = A[i + (int64_t)c * lda] - A[i + (int64_t)j * lda] * u;
            }
        float *L21 = A + j1 + (int64_t)j0 * lda;
        float *U12 = A + j0 + (int64_t)j1 * lda;
        float *A22 = A + j1 + (int64_t)j1 * lda;
        if (variant == 0) {
            float *out = (float *)malloc(sizeof(float) * (size_t)rest * (size_t)rest);
            orc_sgemm_fma_cols(rest, rest, jb, -1.0f, L21, lda, U12, lda, 1.0f, A22, lda,
                               NULL, rest, out);
            for (int c = 0; c < rest; ++c)
                memcpy(A22 + (int64_t)c * lda, out + (int64_t)c * rest, sizeof(float) * (size_t)rest);
            free(out);
        } else {
            int rc = orc_gemm_split(rest, rest, jb, -1.0f, L21, lda, U12, lda, 1.0f, A22, lda, variant);
            if (rc) return rc;
        }
    }
    return 0;
}

/* FP64 solve with FP32 LU factors: "use the LU factorization, but do
 * the solve in a higher precision like FP64".  x <- U^-1 L^-1 P b, in place. */
void orc_lu_solve_f64(int n, const float *LU, int lda, const int *ipiv, double *x)
{
    for (int j = 0; j < n; ++j)
        if (ipiv[j] != j) { double t = x[j]; x[j] = x[ipiv[j]]; x[ipiv[j]] = t; }
    for (int j = 0; j < n; ++j) {             /* L y = P b, unit diagonal */
        double v = x[j];
        for (int i = j + 1; i < n; ++i) x[i] -= (double)LU[i + (int64_t)j * lda] * v;
    }
    for (int j = n - 1; j >= 0; --j) {        /* U x = y */
        x[j] /= (double)LU[j + (int64_t)j * lda];
        double v = x[j];
        for (int i = 0; i < j; ++i) x[i] -= (double)LU[i + (int64_t)j * lda] * v;
    }
}

/* FP64 residual r = b - A x with FP32 A ("compute the residual in
 * higher precision"). */
void orc_residual_f64(int n, const float *A, int lda, const double *b, const double *x, double *r)
{
    for (int i = 0; i < n; ++i) r[i] = b[i];
    for (int j = 0; j < n; ++j) {
        double v = x[j];
        for (int i = 0; i < n; ++i) r[i] -= (double)A[i + (int64_t)j * lda] * v;
    }
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* O-10  Fully 16-bit LU (N4; §IV-B: "For iterative refinement on
 * solutions to Ax = b with LU, using lower precision ... comparing FP32, with
 * FP16 and bfloat16").  Working formats (reading R28):
 *   fmt 0: FP32 (no extra rounding);
 *   fmt 1: BF16 = the (B16) operator above (RNE, saturating);
 *   fmt 2: IEEE binary16 ("reduce the exponent to 5 bits"): 1 sign,
 *          5 exponent (bias 15), 10 mantissa bits, round to nearest even,
 *          gradual underflow, overflow to +-Inf.
 * ------------------------------------------------------------------------ */
uint16_t orc_fp16_round(float x)
{
    uint32_t u = bits_of(x);
    uint32_t sign = (u >> 16) & 0x8000u;
    uint32_t exponent = (u >> 23) & 0xFFu;
    uint32_t mantissa = u & 0x7FFFFFu;
    if (exponent == 0xFFu) return (uint16_t)(sign | (mantissa ? 0x7E00u : 0x7C00u));
    /* value = 1.m * 2^(exponent-127); binary16 normal exponents are -14..15 */
    int e = (int)exponent - 127;
    uint32_t sig = (exponent ? (mantissa | 0x800000u) : mantissa);   /* 24-bit significand */
    if (exponent == 0) e = -126;                                      /* FP32 subnormal */
    /* number of low significand bits to drop so the result has the binary16 ulp:
       normal: ulp 2^(e-10) -> drop (e - 10) - (e - 23) = 13 bits; below 2^-14 the
       ulp is fixed at 2^-24 -> drop 13 + (-14 - e) bits */
    int drop = (e >= -14) ? 13 : 13 + (-14 - e);
    if (drop > 25) return (uint16_t)sign;                             /* < 2^-25: rounds to 0 */
    uint32_t kept = sig >> drop;
    uint32_t rem = sig & ((1u << drop) - 1u), half = 1u << (drop - 1);
    if (rem > half || (rem == half && (kept & 1u))) kept += 1u;
    /* kept is the significand in units of the result ulp; rebuild the pattern */
    uint32_t out;
    if (e >= -14) {
        int ee = e;
        if (kept >= 0x800u) { kept >>= 1; ee += 1; }                  /* carry into the exponent */
        if (ee > 15) return (uint16_t)(sign | 0x7C00u);               /* overflow */
        out = ((uint32_t)(ee + 15) << 10) | (kept & 0x3FFu);
    } else {
        out = kept;                                                   /* subnormal (or carry to 2^-14) */
    }
    return (uint16_t)(sign | out);
}

float orc_fp16_widen(uint16_t h)
{
    uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
    if (e == 0x1Fu) return float_of(sign | 0x7F800000u | (m << 13));
    if (e == 0) {                                                     /* subnormal: m * 2^-24 */
        float v = (float)m * 5.9604644775390625e-8f;
        return sign ? -v : v;
    }
    return float_of(sign | ((e - 15 + 127) << 23) | (m << 13));
}

/* round an FP32 value to the working format and back (exactly representable result) */
static float work_round(int fmt, float x)
{
    if (fmt == 1) return orc_bf16_widen(orc_bf16_round(x));
    if (fmt == 2) return orc_fp16_widen(orc_fp16_round(x));
    return x;
}

/* Unblocked right-looking Gaussian elimination in the working format: the input is
 * stored in the format, and every stored result -- each multiplier l = a/p and each
 * updated entry a - l*u (one FP32 product, one FP32 subtraction) -- is rounded to it.
 * pivot != 0: partial pivoting on the stored values (largest |a|, lowest row on ties);
 * pivot == 0: no interchanges (ipiv[j] = j).  Returns 0, or j+1 for the first exact
 * zero pivot. */
int orc_getrf16(int n, float *A, int lda, int *ipiv, int fmt, int pivot)
{
    for (int c = 0; c < n; ++c)
        for (int i = 0; i < n; ++i) A[i + (int64_t)c * lda] = work_round(fmt, A[i + (int64_t)c * lda]);
    for (int j = 0; j < n; ++j) {
        int p = j;
        if (pivot) {
            float best = fabsf(A[j + (int64_t)j * lda]);
            for (int i = j + 1; i < n; ++i) {
                float v = fabsf(A[i + (int64_t)j * lda]);
                if (v > best) { best = v; p = i; }
            }
        }
        ipiv[j] = p;
        if (A[p + (int64_t)j * lda] == 0.0f) return j + 1;
        if (p != j)
            for (int c = 0; c < n; ++c) {
                float t = A[j + (int64_t)c * lda];
                A[j + (int64_t)c * lda] = A[p + (int64_t)c * lda];
                A[p + (int64_t)c * lda] = t;
            }
        float piv = A[j + (int64_t)j * lda];
        for (int i = j + 1; i < n; ++i)
            A[i + (int64_t)j * lda] = work_round(fmt, A[i + (int64_t)j * lda] / piv);
        for (int c = j + 1; c < n; ++c) {
            float u = A[j + (int64_t)c * lda];
            for (int i = j + 1; i < n; ++i) {
                float prod = A[i + (int64_t)j * lda] * u;
                A[i + (int64_t)c * lda] = work_round(fmt, A[i + (int64_t)c * lda] - prod);
            }
        }
    }
    return 0;
}
