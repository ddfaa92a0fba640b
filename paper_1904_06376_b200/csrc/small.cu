// small.cu -- N4: the paper's refinement experiment on the GPU (section IV-B:
// "We ran 100 tests for unsymmetric dense matrices of order 50, setting the condition number
// and using a residual tolerance of cond(A)*eps").  A batch of small systems, one CTA each:
//   (1) Gaussian elimination in a 16-bit working format (BF16 = the (B16) operator of P:177-179,
//       or IEEE binary16; or FP32): the input is stored in the format and every
//       stored result -- each multiplier l = a / p and each updated entry a - l*u (one FP32
//       product, one FP32 subtraction) -- is rounded to it (reading R28);
//   (2) FP64 refinement as P:406: x0 = U^-1 L^-1 P b, then { r = b - A x ; stop if
//       ||r||_2 <= tol ||b||_2 ; x += U^-1 L^-1 P r }, with the FP32 matrix and the widened
//       factors.
// Every operation is the oracle's, in the oracle's order, with explicit round-to-nearest
// intrinsics (no FMA contraction), so factors, iterates and iteration counts are bit-identical
// to oracle/gesv16_ir.  The matrix (n <= 64) and both copies live in shared memory.
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.cuh"

namespace bf16x {

constexpr int kSmallMax = 64;
constexpr int kSmallLd = kSmallMax + 1;      // column stride in shared memory (bank spread)
constexpr int kSmallThreads = 128;

template <int FMT>
__device__ __forceinline__ float work_round(float x) {
    if constexpr (FMT == 1) return bf16_bits_to_float(rne_sat_bf16(x));
    else if constexpr (FMT == 2) return __half2float(__float2half_rn(x));
    else return x;
}

// y <- U^-1 L^-1 P y in FP64 (the oracle's orc_lu_solve_f64 order: interchanges in sequence,
// column-oriented forward then backward substitution, separate multiply and subtract).
__device__ void small_solve(int n, const float *LU, const int *ipiv, double *y) {
    const int tid = threadIdx.x;
    if (tid == 0)
        for (int j = 0; j < n; ++j)
            if (ipiv[j] != j) { const double t = y[j]; y[j] = y[ipiv[j]]; y[ipiv[j]] = t; }
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        const double v = y[j];
        for (int i = j + 1 + tid; i < n; i += blockDim.x)
            y[i] = __dsub_rn(y[i], __dmul_rn((double)LU[j * kSmallLd + i], v));
        __syncthreads();
    }
    for (int j = n - 1; j >= 0; --j) {
        if (tid == 0) y[j] = __ddiv_rn(y[j], (double)LU[j * kSmallLd + j]);
        __syncthreads();
        const double v = y[j];
        for (int i = tid; i < j; i += blockDim.x) y[i] = __dsub_rn(y[i], __dmul_rn((double)LU[j * kSmallLd + i], v));
        __syncthreads();
    }
}

// sqrt(sum_i v_i^2) accumulated sequentially (the oracle's norm2_seq)
__device__ double seq_norm2(int n, const double *v) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, __dmul_rn(v[i], v[i]));
    return __dsqrt_rn(s);
}

template <int FMT>
__global__ void __launch_bounds__(kSmallThreads) gesv16_kernel(int n, const float *A, int lda, int64_t sA,
                                                               const double *B, int64_t sb, double *X, int64_t sx,
                                                               int pivot, int max_iter, const double *tol,
                                                               int *converged, int *iterations, int *info) {
    __shared__ float LU[kSmallMax * kSmallLd], A0[kSmallMax * kSmallLd];
    __shared__ double x[kSmallMax], r[kSmallMax], bsh[kSmallMax];
    __shared__ int ipiv[kSmallMax];
    __shared__ int s_p, s_info;
    __shared__ double s_res;
    const int sys = blockIdx.x, tid = threadIdx.x;
    const float *a = A + sys * sA;
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int i = e % n, c = e / n;
        const float v = a[(int64_t)c * lda + i];
        A0[c * kSmallLd + i] = v;
        LU[c * kSmallLd + i] = work_round<FMT>(v);
    }
    for (int i = tid; i < n; i += blockDim.x) bsh[i] = B[sys * sb + i];
    if (tid == 0) s_info = 0;
    __syncthreads();
    // ---- (1) elimination in the working format ----
    for (int j = 0; j < n; ++j) {
        if (tid == 0) {
            int p = j;
            if (pivot) {
                float best = fabsf(LU[j * kSmallLd + j]);
                for (int i = j + 1; i < n; ++i) {
                    const float v = fabsf(LU[j * kSmallLd + i]);
                    if (v > best) { best = v; p = i; }
                }
            }
            ipiv[j] = p;
            s_p = p;
            if (LU[j * kSmallLd + p] == 0.0f) s_info = j + 1;
        }
        __syncthreads();
        if (s_info) break;
        const int p = s_p;
        if (p != j)
            for (int c = tid; c < n; c += blockDim.x) {
                const float t = LU[c * kSmallLd + j];
                LU[c * kSmallLd + j] = LU[c * kSmallLd + p];
                LU[c * kSmallLd + p] = t;
            }
        __syncthreads();
        const float piv = LU[j * kSmallLd + j];
        for (int i = j + 1 + tid; i < n; i += blockDim.x)
            LU[j * kSmallLd + i] = work_round<FMT>(__fdiv_rn(LU[j * kSmallLd + i], piv));
        __syncthreads();
        const int m = n - j - 1;
        for (int e = tid; e < m * m; e += blockDim.x) {
            const int i = j + 1 + e % m, c = j + 1 + e / m;
            const float prod = __fmul_rn(LU[j * kSmallLd + i], LU[c * kSmallLd + j]);
            LU[c * kSmallLd + i] = work_round<FMT>(__fsub_rn(LU[c * kSmallLd + i], prod));
        }
        __syncthreads();
    }
    if (s_info) {
        if (tid == 0) { converged[sys] = 0; iterations[sys] = 0; info[sys] = s_info; }
        for (int i = tid; i < n; i += blockDim.x) X[sys * sx + i] = 0.0;
        return;
    }
    // ---- (2) FP64 refinement ----
    for (int i = tid; i < n; i += blockDim.x) x[i] = bsh[i];
    __syncthreads();
    small_solve(n, LU, ipiv, x);
    const double t = tol[sys];
    double nb = 0.0;
    if (tid == 0) nb = seq_norm2(n, bsh);
    int it = 0, conv = 0;
    for (;; ++it) {
        for (int i = tid; i < n; i += blockDim.x) {
            double s = bsh[i];
            for (int c = 0; c < n; ++c) s = __dsub_rn(s, __dmul_rn((double)A0[c * kSmallLd + i], x[c]));
            r[i] = s;
        }
        __syncthreads();
        if (tid == 0) {
            const double rn = seq_norm2(n, r);
            bool finite = true;
            for (int i = 0; i < n; ++i) finite = finite && isfinite(x[i]);
            s_res = (rn <= __dmul_rn(t, nb)) ? 1.0 : (finite ? 0.0 : -1.0);
        }
        __syncthreads();
        if (s_res > 0.0) { conv = 1; break; }
        if (it == max_iter || s_res < 0.0) break;
        small_solve(n, LU, ipiv, r);
        for (int i = tid; i < n; i += blockDim.x) x[i] = __dadd_rn(x[i], r[i]);
        __syncthreads();
    }
    for (int i = tid; i < n; i += blockDim.x) X[sys * sx + i] = x[i];
    if (tid == 0) { converged[sys] = conv; iterations[sys] = it; info[sys] = 0; }
}

}  // namespace bf16x

using namespace bf16x;

extern "C" int bf16x_gesv16_batched(int n, int batch, const float *A, int lda, int64_t strideA, const double *b,
                                    int64_t strideb, double *x, int64_t stridex, int format, int pivot, int max_iter,
                                    const double *tol, int *converged, int *iterations, int *info,
                                    bf16x_stream_t stream) {
    if (n < 0 || n > kSmallMax) return -1;
    if (batch < 0) return -2;
    if (lda < (n > 1 ? n : 1)) return -4;
    if (strideA < (int64_t)lda * n) return -5;
    if (strideb < n) return -7;
    if (stridex < n) return -9;
    if (format < 0 || format > 2) return -10;
    if (max_iter < 0) return -12;
    if (batch > 0 && n > 0 && (!A || !b || !x || !tol || !converged || !iterations || !info)) return -3;
    int rc = arch_ok();
    if (rc || batch == 0 || n == 0) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (format == 0)
        gesv16_kernel<0><<<batch, kSmallThreads, 0, st>>>(n, A, lda, strideA, b, strideb, x, stridex, pivot, max_iter,
                                                          tol, converged, iterations, info);
    else if (format == 1)
        gesv16_kernel<1><<<batch, kSmallThreads, 0, st>>>(n, A, lda, strideA, b, strideb, x, stridex, pivot, max_iter,
                                                          tol, converged, iterations, info);
    else
        gesv16_kernel<2><<<batch, kSmallThreads, 0, st>>>(n, A, lda, strideA, b, strideb, x, stridex, pivot, max_iter,
                                                          tol, converged, iterations, info);
    count_launch();
    return check_launch("gesv16");
}
