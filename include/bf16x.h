/*
 * bf16x.h -- C ABI of libbf16x.so: FP32 GEMM emulated with BF16 splits on B200 (sm_100a).
 *
 * Method: Henry, Tang, Heinecke, "Leveraging the bfloat16 Artificial Intelligence
 * Datatype For Higher-Precision Computations", arXiv 1904.06376 (cited P:<line> of
 * /root/reference/PAPER.md).  Readings of the paper are numbered R<n> in DESIGN.md.
 *
 * Conventions for every entry point
 *  - Storage is column-major (BLAS): element (i,j) of X is X[i + j*ldx].
 *  - Matrix/vector pointers are CUDA DEVICE pointers unless the name ends in _host.
 *  - Work is enqueued on `stream` (or the library stream set by bf16x_set_stream for
 *    entry points without a stream argument); the call returns before the work is
 *    done, cuBLAS-style.  Buffers must stay valid until the stream reaches the work.
 *    bf16x_gemm_host and bf16x_gesv_ir are synchronous.
 *  - The caller owns every buffer it passes.  The library owns a cached device
 *    workspace PER STREAM (pieces of A and B, stream-K fix-up buffers), released by
 *    bf16x_release(): calls on different streams never share library memory and may run
 *    concurrently; calls on one stream are ordered by the stream.  The synchronous LU
 *    entry points (bf16x_getrf, bf16x_gesv_ir, bf16x_gesv_gmres_ir) keep their device
 *    workspace between calls (one call at a time uses it; a concurrent call allocates its
 *    own), also released by bf16x_release().
 *  - Return value: BF16X_SUCCESS (0), a positive BF16X_* status, or -i when argument
 *    i (1-based) is invalid (LAPACK xerbla convention).  NaN/Inf inputs are never
 *    rejected; they propagate (reading R4).
 *  - There is no CPU fallback: on a device that is not sm_100 every compute entry
 *    point returns BF16X_ERR_ARCH.
 *  - C must not alias A or B.
 */
#ifndef BF16X_H
#define BF16X_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *bf16x_stream_t; /* == cudaStream_t; NULL = legacy default stream */

enum {
    BF16X_SUCCESS = 0,
    BF16X_ERR_CUDA = 1,      /* CUDA runtime / launch error (see bf16x_status_string) */
    BF16X_ERR_ALLOC = 2,     /* device or host allocation failed */
    BF16X_ERR_ARCH = 3,      /* current device is not sm_100 */
    BF16X_ERR_SINGULAR = 4,  /* exact zero pivot in bf16x_gesv_ir (report->info = column) */
    BF16X_NOT_CONVERGED = 5  /* iterative refinement stopped without meeting its test */
};

/* gemm_ex flags: FP32 promoted-accumulator carry between k-chunks (multi-GPU overlap). */
#define BF16X_ACC_IN  1u  /* the promoted accumulator starts from acc_carry instead of 0 */
#define BF16X_ACC_OUT 2u  /* store the raw accumulator to acc_carry; skip alpha/beta/C  */
/* N2 options, gemm_ex and split_ex flags:
 * BF16X_SCALED_PIECES: power-of-two scaled pieces (R29; the loss the paper notes
 *   below exponent -110, removed): b1' = (B16)(2^8 (x - b0)), b2' = (B16)(2^8 (2^8
 *   (x - b0) - b1')), so x = b0 + 2^-8 b1' + 2^-16 b2' for every finite x.  The GEMM scales its
 *   tensor-memory accumulator by 2^-8 (tcgen05.mma scale-input-d) on each move to the next
 *   larger bin, so bins are still added smallest first.  Pre-split pieces passed to
 *   bf16x_gemm_ex with this flag must come from bf16x_split_ex(.., BF16X_SCALED_PIECES, ..).
 * BF16X_FP64_COMBINE (gemm_ex only): the paper's "d" variants ("adding the final results
 *   together in FP64"; R30): bins >= 1 and bin 0 accumulate in separate FP32 tensor-memory
 *   accumulators per 64-k interval and are collected in an FP64 accumulator, rounded once to
 *   FP32 before alpha/beta.  Variants 3, 5, 6, 7, 8, 9; not with BF16X_ACC_IN / _OUT.
 * BF16X_SPLIT_TRANSPOSED (split_ex only): write the pieces transposed, as bf16x_split_t.
 * BF16X_NO_STREAM_K (gemm_ex only): every output tile's k-range runs in one CTA pair, so each
 *   element's value depends only on its row of A, its column of B, k and the variant -- not
 *   on m, n or the SM count.  Without it the last waves of tiles may be split in k between two
 *   CTA pairs (stream-K), whose two FP32 partial sums are then added with one extra
 *   round-to-nearest: still within the accuracy contract, but a sub-matrix computed alone
 *   (e.g. one rank's column block, distributed.py) can differ in the last bit from the same
 *   columns of a larger call. */
#define BF16X_SCALED_PIECES    4u
#define BF16X_FP64_COMBINE     8u
#define BF16X_SPLIT_TRANSPOSED 16u
#define BF16X_NO_STREAM_K      32u
/* BF16X_A_PIECES_MN (gemm_ex and split_operands_ex): A's pieces are in A's own column-major
 *   layout, as bf16x_split writes them -- element (i,l) of piece q at A_pieces[q*a_plane + i +
 *   l*ldap], ldap >= max(1, m), ldap % 8 == 0, a_plane >= ldap*k, a_plane % 8 == 0 -- and the
 *   tensor cores read them MN-major (tcgen05 a_major = MN, 128-byte swizzle).  The products are
 *   the same; only the layout differs (the split of A then needs no transpose; this is the
 *   layout bf16x_gemm uses internally). */
#define BF16X_A_PIECES_MN      64u

/* ------------------------------------------------------------------------------------
 * bf16x_split -- the 3-way decomposition of P:180-184 (section II-A):
 *     b0 = (B16) x,   b1 = (B16)((F32)(x - b0)),   b2 = (B16)((F32)(x - b0 - b1))
 * with (B16) = round-to-nearest-even, finite overflow saturating to +-0x7F7F, NaN ->
 * 0x7FC0 (R1, R3, R4); residuals are single FP32 subtractions left to right (R5);
 * subnormals are kept (R6).  Non-finite x gives (bf16(x), +0, +0).
 *   rows, cols : matrix shape (>= 0)
 *   X, ldx     : FP32 source, ldx >= max(1, rows)
 *   P0, P1, P2 : BF16 bit-pattern outputs (uint16), same shape as X with leading
 *                dimension ldp >= max(1, rows).  P1 and P2 may be NULL (fewer pieces:
 *                P0 only = 1 piece, P0+P1 = the pair used by bf16x3);
 *                P2 != NULL requires P1 != NULL.
 * Errors: -1 rows<0, -2 cols<0, -4 ldx, -5 P0 NULL, -7 P2 without P1, -8 ldp.
 * ---------------------------------------------------------------------------------- */
int bf16x_split(int64_t rows, int64_t cols, const float *X, int64_t ldx,
                uint16_t *P0, uint16_t *P1, uint16_t *P2, int64_t ldp, bf16x_stream_t stream);

/* Same decomposition, written transposed: piece element (i,j) lands at P[j + i*ldp]
 * (ldp >= max(1, cols)).  This is the K-major layout the GEMM consumes for A.
 * Errors as bf16x_split, with -8 for ldp < max(1, cols). */
int bf16x_split_t(int64_t rows, int64_t cols, const float *X, int64_t ldx,
                  uint16_t *P0, uint16_t *P1, uint16_t *P2, int64_t ldp, bf16x_stream_t stream);

/* Split with options (flags: BF16X_SCALED_PIECES, BF16X_SPLIT_TRANSPOSED; see above).  With
 * BF16X_SCALED_PIECES the pieces are (b0, b1', b2') of reading R29.  Arguments and errors as
 * bf16x_split (bf16x_split_t when transposed), plus -9 for unknown flags. */
int bf16x_split_ex(int64_t rows, int64_t cols, const float *X, int64_t ldx,
                   uint16_t *P0, uint16_t *P1, uint16_t *P2, int64_t ldp, unsigned flags, bf16x_stream_t stream);

/* Both GEMM operands in one launch (the pre-pass bf16x_gemm runs): A (m x k, lda) is split
 * transposed into K-major pieces (element (i,l) of piece q at Ap[q*a_plane + l + i*ldap]),
 * B (k x n, ldb) in place (element (l,j) of piece q at Bp[q*b_plane + l + j*ldbp]).
 *   pieces : 1, 2 or 3 (bf16x3 uses 2, bf16x6/x9 use 3)
 * Errors: -1 m, -2 n, -3 k, -5 lda, -7 ldb, -8 pieces, -9 Ap/ldap/a_plane, -12 Bp/ldbp/b_plane. */
int bf16x_split_operands(int m, int n, int k, const float *A, int64_t lda, const float *B, int64_t ldb,
                         int pieces, uint16_t *Ap, int64_t ldap, int64_t a_plane, uint16_t *Bp, int64_t ldbp,
                         int64_t b_plane, bf16x_stream_t stream);

/* bf16x_split_operands with flags: BF16X_A_PIECES_MN (A split in its own layout, element (i,l) of
 * piece q at Ap[q*a_plane + i + l*ldap], ldap >= max(1, m), a_plane >= ldap*k: both operands are
 * then same-layout splits; this is the pre-pass bf16x_gemm runs) and BF16X_SCALED_PIECES (R29).
 * Errors as bf16x_split_operands, plus -13 for unknown flags. */
int bf16x_split_operands_ex(int m, int n, int k, const float *A, int64_t lda, const float *B, int64_t ldb,
                            int pieces, uint16_t *Ap, int64_t ldap, int64_t a_plane, uint16_t *Bp, int64_t ldbp,
                            int64_t b_plane, unsigned flags, bf16x_stream_t stream);

/* ------------------------------------------------------------------------------------
 * bf16x_gemm -- C = alpha*A*B + beta*C (BLAS sgemm, transa = transb = 'N') with the
 * FP32 product emulated by BF16 x BF16 -> FP32 tensor-core products (section IV-A):
 *   variant 3: pieces 0-1, products {00,01,10}            ("pair of BF16s")
 *   variant 6: pieces 0-2, products {00,01,10,02,11,20}   (Z_2)
 *   variant 7: x6 + a1*b2 (the 2^-24-bin term of P:376's example: "at least 7 products"; R27)
 *   variant 8: eight products, bins 0..3 = the paper's Z_3
 *   variant 9: all nine products                          (R9)
 *   variant 5: A in two pieces, B in three, products {00,01,10,02,11} (R27)
 *   variant 1: b0 only, one product (debug / plain-BF16 peak)
 * Products are accumulated smallest bin first into an FP32 tensor-memory
 * partial that is added, with FP32 round-to-nearest, into a promoted accumulator every
 * 64 values of k ("promotion").  alpha/beta follow BLAS (R19):
 * beta == 0 never reads C; alpha == 0 or k == 0 returns beta*C.
 *   A: m x k, lda >= max(1,m);  B: k x n, ldb >= max(1,k);  C: m x n, ldc >= max(1,m).
 * Runs on the library stream (bf16x_set_stream).  Errors: -1 m, -2 n, -3 k, -6 lda,
 * -8 ldb, -11 ldc, -12 variant (not 1/3/5/6/7/8/9); BF16X_ERR_ALLOC if the workspace cannot grow.
 * ---------------------------------------------------------------------------------- */
int bf16x_gemm(int m, int n, int k, float alpha, const float *A, int lda,
               const float *B, int ldb, float beta, float *C, int ldc, int variant);

/* Bytes of caller workspace bf16x_gemm_ex needs: 2 * (pA * round_up(m, 8) + pB * n) * round_up(k, 8),
 * with (pA, pB) the variant's pieces per operand: x1 (1,1), x3 (2,2), x5 (2,3), others (3,3). */
size_t bf16x_gemm_workspace_size(int m, int n, int k, int variant);

/* Extended GEMM: explicit stream, caller workspace (NULL = library cache), optional
 * pre-split pieces, optional accumulator carry.
 *   A_pieces : NULL, or the base of pA K-major piece planes of A as written by
 *              bf16x_split_t: element (i,l) of piece q at A_pieces[q*a_plane + l + i*ldap],
 *              ldap >= k, ldap % 8 == 0, a_plane % 8 == 0, 16-byte aligned base;
 *              with BF16X_A_PIECES_MN, planes in A's own layout as written by bf16x_split
 *              (element (i,l) at A_pieces[q*a_plane + i + l*ldap], ldap >= m, ldap % 8 == 0,
 *              a_plane >= ldap*k, a_plane % 8 == 0); then A may be NULL.
 *   B_pieces : NULL, or the base of pB piece planes of B as written by bf16x_split:
 *              element (l,j) of piece q at B_pieces[q*b_plane + l + j*ldbp], ldbp >= k,
 *              ldbp % 8 == 0, b_plane % 8 == 0; then B may be NULL.
 *   acc_carry: m x n FP32 (ld = ldc) used by BF16X_ACC_IN / BF16X_ACC_OUT.
 *   flags    : BF16X_ACC_IN | BF16X_ACC_OUT | BF16X_SCALED_PIECES | BF16X_FP64_COMBINE |
 *              BF16X_NO_STREAM_K | BF16X_A_PIECES_MN (above).
 *   workspace: NULL (the library's cache for `stream`), or ws_bytes >= bf16x_gemm_workspace_size
 *              bytes of device memory owned by the caller, not used by other work meanwhile.
 * Errors: as bf16x_gemm, plus -13 flags (unknown bits, FP64_COMBINE with ACC_* or with
 * variant 1), -14 A_pieces layout, -16 B_pieces layout,
 * -19 acc_carry NULL with ACC flags, -21 ws_bytes too small. */
int bf16x_gemm_ex(int m, int n, int k, float alpha, const float *A, int lda,
                  const float *B, int ldb, float beta, float *C, int ldc, int variant,
                  unsigned flags, const uint16_t *A_pieces, int64_t ldap, int64_t a_plane,
                  const uint16_t *B_pieces, int64_t ldbp, int64_t b_plane, float *acc_carry,
                  void *workspace, size_t ws_bytes, bf16x_stream_t stream);

/* Host-buffer GEMM (synchronous): copies A, B (and C when beta != 0) from host memory
 * into cached device buffers, runs the split GEMM, copies C back.  Same arguments and
 * errors as bf16x_gemm with HOST pointers.  Large problems (m*k >= 2^20, n >= 1024) are
 * pipelined over column chunks of B/C (width n / min(8, n/512) rounded up to 256): A is
 * copied and split once, each chunk's B copy overlaps the previous chunk's GEMM and each
 * chunk's C copy-back overlaps the next; every chunk equals bf16x_gemm on that column block.
 * With beta == 0, m, n >= 4096 and a GEMM not much shorter than the copy-in
 * (m*n*variant/(m+n) >= 32400) the pipeline is two-dimensional instead: A in row blocks and
 * B in column blocks (each min(8, dim/1024) blocks, multiples of 256), copied in alternately,
 * each split once as it lands; block (i, j) of C is computed as soon as A_i and B_j are split
 * and copied back as soon as it is done.  Every element of C then equals
 * bf16x_gemm_ex(..., BF16X_NO_STREAM_K) (R32: shape-independent results).
 * Pinned host memory is needed for the copies to overlap (pageable memory still works). */
int bf16x_gemm_host(int m, int n, int k, float alpha, const float *A_host, int lda,
                    const float *B_host, int ldb, float beta, float *C_host, int ldc, int variant);

/* ------------------------------------------------------------------------------------
 * bf16x_gesv_ir -- solve A x = b by LU with partial pivoting whose cubic work (the
 * trailing updates A22 -= L21*U12) runs in bf16x_gemm(variant), followed by FP64
 * iterative refinement (section III: "compute the residual in higher precision,
 * r = A*x - b, and use the results from the lower precision solver to solve the updated
 * system Ay = r ... and then update x with x + y").  Panel factorisation and U12 solves
 * are FP32; residuals and triangular solves are FP64 (the factors widened exactly).
 * Stopping rule: with tol > 0, ||r||_inf <= tol * ||b||_inf -- the paper's "residual
 * tolerance of cond(A)*eps" is tol = cond(A) * 2^-53; with tol <= 0 the default
 * (R14) ||r||_inf <= sqrt(n)*||x||_inf*||A||_inf*2^-53 (LAPACK dsgesv).  Stagnation =
 * residual not halved over 3 iterations.  Synchronous.
 *   n         : order (>= 0);  A: n x n FP32 device, lda >= max(1,n), NOT modified
 *   b, x      : FP64 device vectors of length n (x is output)
 *   variant   : 3, 6 or 9;  nb: panel width (<= 0: 256)
 *   tol       : relative residual tolerance (above; NaN: error -8)
 *   max_iter  : refinement iterations (<= 0: 30)
 *   residual_history : HOST, nullable, max_iter+1 doubles (||r||_inf per iteration)
 *   report    : HOST, required; always filled.
 * Returns BF16X_SUCCESS, BF16X_ERR_SINGULAR (report->info = 1-based column),
 * BF16X_NOT_CONVERGED (x = last iterate), or an error: -1 n, -3 lda, -6 variant, -8 tol,
 * -11 report NULL. */
typedef struct {
    int converged;           /* 1 if the stopping test was met */
    int iterations;          /* refinement corrections applied */
    int info;                /* 0, or the 1-based column of an exact zero pivot */
    double final_residual;   /* ||b - A x||_inf at exit */
    double backward_error;   /* ||r||_inf / (||A||_inf ||x||_inf) at exit */
    double tol;              /* threshold the test compared ||r||_inf against */
    double factor_ms;        /* device time of the LU factorisation */
    double refine_ms;        /* device time of the refinement loop */
    int inner_iterations;    /* bf16x_gesv_gmres_ir: total Arnoldi steps (0 for bf16x_gesv_ir) */
} bf16x_ir_report;

int bf16x_gesv_ir(int n, const float *A, int lda, const double *b, double *x, int variant,
                  int nb, double tol, int max_iter, double *residual_history, bf16x_ir_report *report);

/* ------------------------------------------------------------------------------------
 * bf16x_gesv_gmres_ir -- GMRES-IR (section III: "combining Iterative Refinement with
 * an Iterative Solver like GMRES"; section IV-B: "apply GMRES instead of iterative
 * refinement, and use the LU decomposition in the lower precision ... as a pre-conditioner").
 * Same factorisation and outer loop as bf16x_gesv_ir (x0 = 0; r = b - A x in FP64; the same
 * stopping and stagnation rules, R14), but each correction A d = r is solved by one cycle
 * of FP64 GMRES on M^-1 A d = M^-1 r with M^-1 = U^-1 L^-1 P from the bf16x factors:
 * Arnoldi by classical Gram-Schmidt applied twice, Givens rotations, cycle ends after
 * `restart` steps, on breakdown, or when the rotated residual <= inner_tol * ||M^-1 r||_2
 * (reading R25).  Synchronous.
 *   n, A, lda, b, x, variant, nb, tol, max_iter, residual_history, report: as bf16x_gesv_ir
 *     (report->iterations = outer corrections, report->inner_iterations = Arnoldi steps)
 *   restart   : Arnoldi steps per correction (<= 0: 200; capped at n and at 8190)
 *   inner_tol : relative tolerance of each GMRES cycle (0: 1e-10; < 0 or NaN: error -9)
 * Device workspace: n*(restart+1) doubles for the Krylov basis on top of bf16x_gesv_ir's.
 * Returns as bf16x_gesv_ir; errors -1 n, -3 lda, -6 variant, -9 inner_tol, -10 tol,
 * -13 report NULL. */
int bf16x_gesv_gmres_ir(int n, const float *A, int lda, const double *b, double *x, int variant,
                        int nb, int restart, double inner_tol, double tol, int max_iter,
                        double *residual_history, bf16x_ir_report *report);

/* ------------------------------------------------------------------------------------
 * bf16x_gesv16_batched -- the paper's refinement experiment (section IV-B: "100
 * tests for unsymmetric dense matrices of order 50, setting the condition number and using
 * a residual tolerance of cond(A)*eps"; N4, reading R28) for a batch of small systems, one
 * thread block each.  Gaussian elimination in the working `format` with every stored result
 * rounded to it, then FP64 refinement: x0 = U^-1 L^-1 P b; loop { r = b - A x;
 * converged if ||r||_2 <= tol[s] * ||b||_2; stop after max_iter corrections or a non-finite
 * x; x += U^-1 L^-1 P r }.  Bit-identical to the oracle's gesv16_ir.  Asynchronous (stream).
 *   n        : order, 0..64;  batch : number of systems (>= 0)
 *   A        : DEVICE FP32, system s at A + s*strideA, column-major with lda >= max(1,n),
 *              strideA >= lda*n; not modified
 *   b, x     : DEVICE FP64, system s at b + s*strideb / x + s*stridex (strides >= n)
 *   format   : 0 FP32, 1 BF16 (the (B16) operator of P:177-179), 2 IEEE binary16
 *   pivot    : nonzero = partial pivoting on the stored values, 0 = none
 *   max_iter : corrections allowed (>= 0);  tol : DEVICE FP64[batch] (e.g. cond(A)*2^-53)
 *   converged, iterations, info : DEVICE int[batch] outputs (info = 1-based column of an
 *              exact zero pivot, then x = 0 and converged = 0)
 * Errors: -1 n, -2 batch, -3 NULL pointer, -4 lda, -5 strideA, -7 strideb, -9 stridex,
 * -10 format, -12 max_iter. */
int bf16x_gesv16_batched(int n, int batch, const float *A, int lda, int64_t strideA, const double *b,
                         int64_t strideb, double *x, int64_t stridex, int format, int pivot, int max_iter,
                         const double *tol, int *converged, int *iterations, int *info,
                         bf16x_stream_t stream);

/* ------------------------------------------------------------------------------------
 * bf16x_getrf -- the factorisation alone (LAPACK sgetrf semantics, "a SGETRF
 * based on triplets of BF16s and six products"): P A = L U in place, right-looking blocked,
 * FP32 panel + TRSM, trailing updates A22 -= L21 U12 in bf16x_gemm(variant).
 *   A    : n x n FP32 DEVICE, lda >= max(1,n); overwritten by L (unit, below the diagonal)
 *          and U (on and above)
 *   ipiv : DEVICE int32[n], 0-based: row j was interchanged with row ipiv[j] (in order)
 *   variant : 1, 3, 5, 6, 7, 8 or 9;  nb : panel width (<= 0: 256)
 *   info : HOST, nullable; 0 or the 1-based column of the first exact zero pivot
 * Synchronous.  Returns BF16X_SUCCESS, BF16X_ERR_SINGULAR (factorisation continued past
 * the zero pivot as LAPACK does only for the remaining columns' interchanges), or -1 n,
 * -2 A NULL, -3 lda, -4 ipiv NULL, -5 variant. */
int bf16x_getrf(int n, float *A, int lda, int *ipiv, int variant, int nb, int *info);

/* ------------------------------------------------------------------------------------
 * Library state.
 * ---------------------------------------------------------------------------------- */
int bf16x_set_stream(bf16x_stream_t stream);   /* stream used by bf16x_gemm / _host */
bf16x_stream_t bf16x_get_stream(void);
void bf16x_release(void);                      /* free cached device/host workspace (GEMM and LU) */
const char *bf16x_status_string(int status);   /* static string; includes the last CUDA error */
int bf16x_device_check(void);                  /* BF16X_SUCCESS iff the current device is sm_100 */
/* Number of library kernels launched by this process so far (all entry points). */
uint64_t bf16x_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* BF16X_H */
