// lu.cu -- a6: LU with partial pivoting whose cubic work runs in the split GEMM, followed by
// FP64 iterative refinement (section III: "Only the cubic work of the initial LU
// factorization should be done in the lower precision: all the other steps ... in the higher
// precision").
//
//   factor (FP32, in a device copy of A), blocked right-looking, panel width nb:
//     K4 panel_kernel   cooperative grid, one grid barrier per column: pivot search (argmax |a|,
//                       ties -> lowest row), L multipliers and the rank-1 updates restricted to
//                       the panel, rows left in place (pivoted rows are marked instead of
//                       swapped) -- the LAPACK interchange sequence is derived afterwards
//     K5 laswp_kernel   applies the panel's interchanges to all n columns
//        trsm_kernel    U12 = L11^-1 A12 (FP32, unit lower)
//     K2 bf16x GEMM     A22 <- -1 * L21 U12 + 1 * A22 in bf16x<variant>   (the cubic work)
//   refine (FP64, factors widened exactly):
//     K6 residual       r = b - A x, deterministic two-phase row sums
//        trsv_kernel    cooperative blocked forward / backward substitution
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace bf16x {

int gemm_core(int m, int n, int k, float alpha, const float *A, int lda, const float *B, int ldb, float beta,
              float *C, int ldc, int variant, unsigned flags, const uint16_t *Ap, int64_t ldap, int64_t a_plane,
              const uint16_t *Bp, int64_t ldbp, int64_t b_plane, float *acc, void *ws, size_t ws_bytes,
              cudaStream_t st, int cta_group);

constexpr int kLuThreads = 256;

// ------------------------------------------------------------------------------------
// grid barrier for cooperative launches (all CTAs co-resident): sense reversal on a global
// counter / generation pair.
// ------------------------------------------------------------------------------------
struct GridBar {
    unsigned int count;
    unsigned int gen;
};

__device__ __forceinline__ void grid_sync(GridBar *gb, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int *vgen = &gb->gen;
        const unsigned int g = *vgen;
        __threadfence();
        if (atomicAdd(&gb->count, 1u) == nblocks - 1) {
            gb->count = 0;
            __threadfence();
            atomicAdd(&gb->gen, 1u);
        } else {
            while (*vgen == g) { __nanosleep(32); }
        }
        __threadfence();
    }
    __syncthreads();
}

struct PivotCand {
    float v;
    int i;
};

__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
    return v > bv || (v == bv && i < bi);  // larger |a|, ties -> lowest row index
}

// ------------------------------------------------------------------------------------
// K4: panel factorisation of columns [j0, j0+jb) over rows [j0, n).  Rows are distributed in
// contiguous chunks over the grid.  Step t (column c = j0+t):
//   (a) rows not yet pivoted apply the previous step: l = a[i,c-1] / a[p,c-1] stored in place,
//       a[i,c'] -= l * a[p,c'] for the panel columns c' >= c;
//   (b) local argmax |a[i,c]| over unpivoted rows -> cand[block];  grid barrier;
//   (c) every block reduces the candidates identically -> p_t; the owner marks row p_t.
// The interchange sequence is built afterwards from piv_rows (build_ipiv_kernel).
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kLuThreads) panel_kernel(float *LU, int ld, int n, int j0, int jb,
                                                           PivotCand *cand, int *piv_rows, int *mark,
                                                           int *info, GridBar *gb) {
    const int nb = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
    const int R = n - j0;
    const int r0 = j0 + (int)(((int64_t)R * b) / nb), r1 = j0 + (int)(((int64_t)R * (b + 1)) / nb);
    __shared__ float s_v[kLuThreads / 32];
    __shared__ int s_i[kLuThreads / 32];
    __shared__ int s_p;
    for (int i = r0 + tid; i < r1; i += blockDim.x) mark[i] = 0;
    __syncthreads();
    int p_prev = -1;
    for (int t = 0; t <= jb; ++t) {
        const int c = j0 + t;
        // (a) apply step t-1 to this block's unpivoted rows
        if (t > 0) {
            const int cp = c - 1;
            const float piv = LU[(int64_t)cp * ld + p_prev];
            const int ncols = j0 + jb - c;              // columns c .. j0+jb-1
            const int rows = r1 - r0;
            // element (row, col) pairs: first the multiplier column, then the updates
            for (int e = tid; e < rows; e += blockDim.x) {
                const int i = r0 + e;
                if (mark[i]) continue;
                float *a = LU + (int64_t)cp * ld + i;
                const float l = (piv != 0.f) ? (*a / piv) : 0.f;
                *a = l;
            }
            __syncthreads();
            if (ncols > 0) {
                // one warp per column, lanes over rows (coalesced in column-major storage)
                const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
                for (int cc = c + wid; cc < j0 + jb; cc += nw) {
                    const float u = LU[(int64_t)cc * ld + p_prev];
                    float *acol = LU + (int64_t)cc * ld;
                    const float *lcol = LU + (int64_t)cp * ld;
                    for (int i = r0 + lane; i < r1; i += 32) {
                        if (mark[i]) continue;
                        acol[i] = acol[i] - lcol[i] * u;
                    }
                }
            }
            __syncthreads();
        }
        if (t == jb) break;
        // (b) local argmax of |a[i,c]| over unpivoted rows
        float bv = -1.f;
        int bi = 0x7FFFFFFF;
        for (int i = r0 + tid; i < r1; i += blockDim.x) {
            if (mark[i]) continue;
            const float v = fabsf(LU[(int64_t)c * ld + i]);
            if (better(v, i, bv, bi)) { bv = v; bi = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
        }
        if ((tid & 31) == 0) { s_v[tid >> 5] = bv; s_i[tid >> 5] = bi; }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < kLuThreads / 32; ++w)
                if (better(s_v[w], s_i[w], bv, bi)) { bv = s_v[w]; bi = s_i[w]; }
            cand[(t & 1) * nb + b] = {bv, bi};
        }
        grid_sync(gb, nb);
        // (c) global pivot (identical reduction in every block)
        if (tid < 32) {
            float gv = -1.f;
            int gi = 0x7FFFFFFF;
            for (int k = tid; k < nb; k += 32) {
                const PivotCand pc = cand[(t & 1) * nb + k];
                if (better(pc.v, pc.i, gv, gi)) { gv = pc.v; gi = pc.i; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, gv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, gi, o);
                if (better(ov, oi, gv, gi)) { gv = ov; gi = oi; }
            }
            if (tid == 0) {
                s_p = gi;
                if (b == 0) {
                    piv_rows[t] = gi;
                    if (gv == 0.f && *info == 0) *info = c + 1;
                }
            }
        }
        __syncthreads();
        p_prev = s_p;
        if (p_prev >= r0 && p_prev < r1 && tid == 0) mark[p_prev] = 1;
        __syncthreads();
    }
}

// LAPACK interchange sequence from the chosen physical rows: step t swaps position j0+t with
// the current position of row piv_rows[t].  One thread; pos/row_at are n-length scratch.
__global__ void build_ipiv_kernel(int n, int j0, int jb, const int *piv_rows, int *ipiv, int *pos, int *row_at) {
    for (int i = j0 + threadIdx.x; i < n; i += blockDim.x) { pos[i] = i; row_at[i] = i; }
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int t = 0; t < jb; ++t) {
        const int r = piv_rows[t];
        const int q = pos[r];              // where the chosen row currently is
        const int here = j0 + t;
        const int other = row_at[here];    // row currently at the target position
        ipiv[here] = q;
        row_at[q] = other;
        pos[other] = q;
        row_at[here] = r;
        pos[r] = here;
    }
}

// K5a: apply ipiv[j0..j0+jb) (in order) to columns [c0, c1).  One thread per column.
__global__ void laswp_kernel(float *LU, int ld, int c0, int c1, int j0, int jb, const int *ipiv) {
    const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= c1) return;
    float *col = LU + (int64_t)c * ld;
    for (int t = 0; t < jb; ++t) {
        const int q = ipiv[j0 + t];
        if (q != j0 + t) {
            const float a = col[j0 + t];
            col[j0 + t] = col[q];
            col[q] = a;
        }
    }
}

// K5b: U12 = L11^-1 A12 with L11 = unit lower jb x jb at (j0, j0), A12 = rows j0..j0+jb of
// columns [c0, c0 + ncols).  One CTA per 32 columns; the 32 columns live in shared memory.
constexpr int kTrsmCols = 32;
__global__ void __launch_bounds__(256) trsm_kernel(float *LU, int ld, int j0, int jb, int c0, int ncols) {
    extern __shared__ float sB[];           // jb x kTrsmCols, row-major [row][col]
    const int cb = c0 + blockIdx.x * kTrsmCols;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 columns x 8 row groups
    const bool valid = (cb + tx) < c0 + ncols;
    for (int r = ty; r < jb; r += 8) sB[r * kTrsmCols + tx] = valid ? LU[(int64_t)(cb + tx) * ld + j0 + r] : 0.f;
    __syncthreads();
    for (int i = 0; i < jb - 1; ++i) {
        const float xi = sB[i * kTrsmCols + tx];
        const float *Lcol = LU + (int64_t)(j0 + i) * ld + j0;
        for (int r = i + 1 + ty; r < jb; r += 8) sB[r * kTrsmCols + tx] -= Lcol[r] * xi;
        __syncthreads();
    }
    if (valid)
        for (int r = ty; r < jb; r += 8) LU[(int64_t)(cb + tx) * ld + j0 + r] = sB[r * kTrsmCols + tx];
}

// ------------------------------------------------------------------------------------
// K6: FP64 residual r = b - A x (A FP32, exact widening), deterministic two-phase sums.
// ------------------------------------------------------------------------------------
constexpr int kResRows = 256, kResChunk = 256;
__global__ void residual_partial_kernel(const float *A, int ld, int n, const double *x, double *part, int absval) {
    const int i = blockIdx.x * kResRows + threadIdx.x;
    const int j0 = blockIdx.y * kResChunk, j1 = min(n, j0 + kResChunk);
    if (i >= n) return;
    double s = 0.0;
    for (int j = j0; j < j1; ++j) {
        const double a = (double)A[(int64_t)j * ld + i];
        s += absval ? fabs(a) * (x ? x[j] : 1.0) : a * x[j];
    }
    part[(int64_t)blockIdx.y * n + i] = s;
}
__global__ void residual_final_kernel(int n, int nchunk, const double *part, const double *b, double *r) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int c = 0; c < nchunk; ++c) s += part[(int64_t)c * n + i];
    r[i] = b ? b[i] - s : s;
}

// max |v| over a vector (single CTA, deterministic) -> out[0]
__global__ void absmax_kernel(int n, const double *v, double *out) {
    __shared__ double s[256];
    double m = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(v[i]));
    s[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] = fmax(s[threadIdx.x], s[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = s[0];
}

__global__ void axpy_kernel(int n, double *x, const double *d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] += d[i];
}

// y = P v from the interchanges (applied in order) -- one CTA, vector staged in shared memory.
__global__ void permute_kernel(int n, const int *ipiv, const double *v, double *y) {
    extern __shared__ double sv[];
    for (int i = threadIdx.x; i < n; i += blockDim.x) sv[i] = v[i];
    __syncthreads();
    if (threadIdx.x == 0)
        for (int j = 0; j < n; ++j) {
            const int q = ipiv[j];
            if (q != j) { const double t = sv[j]; sv[j] = sv[q]; sv[q] = t; }
        }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = sv[i];
}

// Blocked triangular solve in FP64 with the FP32 factors, cooperative grid.  lower != 0:
// L y = y (unit diagonal, forward); else U y = y (backward).  Block bs rows: block 0 of the
// grid solves the diagonal block, grid barrier, every block updates its share of the rows
// beyond it, grid barrier.
constexpr int kTrsvBlock = 64;
__global__ void __launch_bounds__(256) trsv_kernel(const float *LU, int ld, int n, double *y, int lower, GridBar *gb) {
    __shared__ double sx[kTrsvBlock];
    const int nblk = (n + kTrsvBlock - 1) / kTrsvBlock;
    for (int s = 0; s < nblk; ++s) {
        const int bidx = lower ? s : nblk - 1 - s;
        const int c0 = bidx * kTrsvBlock, c1 = min(n, c0 + kTrsvBlock);
        if (blockIdx.x == 0) {
            if (threadIdx.x < 32) {
                // sequential solve of the diagonal block by one warp: lane handles rows
                for (int jj = 0; jj < c1 - c0; ++jj) {
                    const int j = lower ? c0 + jj : c1 - 1 - jj;
                    double xj = 0.0;
                    if (threadIdx.x == 0) {
                        xj = y[j];
                        if (!lower) xj /= (double)LU[(int64_t)j * ld + j];
                        y[j] = xj;
                    }
                    xj = __shfl_sync(0xffffffffu, xj, 0);
                    __syncwarp();
                    for (int i = threadIdx.x; i < c1 - c0; i += 32) {
                        const int r = c0 + i;
                        if (lower ? (r > j) : (r < j)) y[r] -= (double)LU[(int64_t)j * ld + r] * xj;
                    }
                    __syncwarp();
                }
            }
        }
        grid_sync(gb, gridDim.x);
        for (int i = threadIdx.x; i < c1 - c0; i += blockDim.x) sx[i] = y[c0 + i];
        __syncthreads();
        // rows outside the block that still depend on it
        const int lo = lower ? c1 : 0, hi = lower ? n : c0;
        for (int r = lo + blockIdx.x * blockDim.x + threadIdx.x; r < hi; r += gridDim.x * blockDim.x) {
            double s = 0.0;
            for (int j = 0; j < c1 - c0; ++j) s += (double)LU[(int64_t)(c0 + j) * ld + r] * sx[j];
            y[r] -= s;
        }
        grid_sync(gb, gridDim.x);
    }
}

__global__ void copy_matrix_kernel(int n, const float *A, int lda, float *B, int ldb) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % n, j = t / n;
        B[j * ldb + i] = A[j * lda + i];
    }
}

// ------------------------------------------------------------------------------------
// host driver
// ------------------------------------------------------------------------------------
struct LuWork {
    float *LU = nullptr;
    int *ipiv = nullptr, *piv_rows = nullptr, *mark = nullptr, *pos = nullptr, *row_at = nullptr, *info = nullptr;
    PivotCand *cand = nullptr;
    GridBar *gb = nullptr;
    double *r = nullptr, *d = nullptr, *part = nullptr, *scal = nullptr, *x = nullptr;
};

static int coop_launch(const void *fn, int grid, int threads, void **args, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), args, smem, st);
    if (e != cudaSuccess) {
        set_cuda_error(e, "cooperative launch");
        return BF16X_ERR_CUDA;
    }
    count_launch();
    return BF16X_SUCCESS;
}

static int solve_with_factors(const LuWork &w, int n, const double *v, double *out, int coop_grid, cudaStream_t st) {
    // out = U^-1 L^-1 P v
    permute_kernel<<<1, 1024, (size_t)n * sizeof(double), st>>>(n, w.ipiv, v, out);
    count_launch();
    int ld = n, lower = 1;
    const float *LU = w.LU;
    double *y = out;
    GridBar *gb = w.gb;
    void *args[] = {(void *)&LU, (void *)&ld, (void *)&n, (void *)&y, (void *)&lower, (void *)&gb};
    int rc = coop_launch((const void *)trsv_kernel, coop_grid, 256, args, 0, st);
    if (rc) return rc;
    lower = 0;
    return coop_launch((const void *)trsv_kernel, coop_grid, 256, args, 0, st);
}

static void residual(const float *A, int lda, int n, const double *x, const double *b, double *r, double *part,
                     int absval, cudaStream_t st) {
    const int nchunk = (n + kResChunk - 1) / kResChunk;
    dim3 grid((n + kResRows - 1) / kResRows, nchunk);
    residual_partial_kernel<<<grid, kResRows, 0, st>>>(A, lda, n, x, part, absval);
    residual_final_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, nchunk, part, b, r);
    count_launch(2);
}

}  // namespace bf16x

using namespace bf16x;

extern "C" int bf16x_gesv_ir(int n, const float *A, int lda, const double *b, double *x, int variant, int nb,
                             int max_iter, double *residual_history, bf16x_ir_report *report) {
    if (n < 0) return -1;
    if (lda < (n > 1 ? n : 1)) return -3;
    if (variant != 3 && variant != 6 && variant != 9) return -6;
    if (!report) return -10;
    *report = bf16x_ir_report{0, 0, 0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int rc = arch_ok();
    if (rc) return rc;
    if (n == 0) {
        report->converged = 1;
        return BF16X_SUCCESS;
    }
    if (nb <= 0) nb = 256;
    if (max_iter <= 0) max_iter = 30;
    cudaStream_t st = current_stream();
    LuWork w;
    const int nchunk = (n + kResChunk - 1) / kResChunk;
    int coop_grid = 0;
    {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trsv_kernel, 256, 0);
        int per_sm2 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, panel_kernel, kLuThreads, 0);
        coop_grid = num_sms() * std::max(1, std::min(per_sm, per_sm2));
        coop_grid = std::min(coop_grid, num_sms());
    }
    auto alloc = [&](void **p, size_t bytes) {
        if (rc) return;
        if (cudaMalloc(p, bytes) != cudaSuccess) {
            cudaGetLastError();
            rc = BF16X_ERR_ALLOC;
        }
    };
    alloc((void **)&w.LU, sizeof(float) * (size_t)n * n);
    alloc((void **)&w.ipiv, sizeof(int) * n);
    alloc((void **)&w.piv_rows, sizeof(int) * (size_t)nb);
    alloc((void **)&w.mark, sizeof(int) * n);
    alloc((void **)&w.pos, sizeof(int) * n);
    alloc((void **)&w.row_at, sizeof(int) * n);
    alloc((void **)&w.info, sizeof(int));
    alloc((void **)&w.cand, sizeof(PivotCand) * 2 * (size_t)coop_grid);
    alloc((void **)&w.gb, sizeof(GridBar));
    alloc((void **)&w.r, sizeof(double) * n);
    alloc((void **)&w.d, sizeof(double) * n);
    alloc((void **)&w.part, sizeof(double) * (size_t)n * nchunk);
    alloc((void **)&w.scal, sizeof(double) * 4);
    auto cleanup = [&]() {
        cudaFree(w.LU); cudaFree(w.ipiv); cudaFree(w.piv_rows); cudaFree(w.mark); cudaFree(w.pos);
        cudaFree(w.row_at); cudaFree(w.info); cudaFree(w.cand); cudaFree(w.gb); cudaFree(w.r);
        cudaFree(w.d); cudaFree(w.part); cudaFree(w.scal);
    };
    if (rc) {
        cleanup();
        return rc;
    }
    {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(permute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            attr = true;
        }
    }
    if ((size_t)n * sizeof(double) > 227 * 1024) {
        cleanup();
        set_error_msg("gesv_ir: n too large for the shared-memory permutation (n <= 29056)");
        return -1;
    }
    cudaMemsetAsync(w.gb, 0, sizeof(GridBar), st);
    cudaMemsetAsync(w.info, 0, sizeof(int), st);
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
    cudaEventRecord(e0, st);

    // ---------------- factorisation ----------------
    copy_matrix_kernel<<<num_sms() * 8, 256, 0, st>>>(n, A, lda, w.LU, n);
    count_launch();
    const int ld = n;
    for (int j0 = 0; j0 < n && !rc; j0 += nb) {
        const int jb = std::min(nb, n - j0);
        {
            float *LU = w.LU;
            int ldv = ld, nv = n, j0v = j0, jbv = jb;
            PivotCand *cand = w.cand;
            int *piv = w.piv_rows, *mark = w.mark, *info = w.info;
            GridBar *gb = w.gb;
            void *args[] = {&LU, &ldv, &nv, &j0v, &jbv, &cand, &piv, &mark, &info, &gb};
            const int g = std::max(1, std::min(coop_grid, (n - j0 + 31) / 32));
            rc = coop_launch((const void *)panel_kernel, g, kLuThreads, args, 0, st);
            if (rc) break;
        }
        build_ipiv_kernel<<<1, 1024, 0, st>>>(n, j0, jb, w.piv_rows, w.ipiv, w.pos, w.row_at);
        laswp_kernel<<<(n + 127) / 128, 128, 0, st>>>(w.LU, ld, 0, n, j0, jb, w.ipiv);
        count_launch(2);
        const int j1 = j0 + jb, rest = n - j1;
        if (rest > 0) {
            trsm_kernel<<<(rest + kTrsmCols - 1) / kTrsmCols, 256, (size_t)jb * kTrsmCols * sizeof(float), st>>>(
                w.LU, ld, j0, jb, j1, rest);
            count_launch();
            rc = check_launch("trsm");
            if (rc) break;
            // A22 <- -L21 U12 + A22 : the cubic work, in the split GEMM
            rc = gemm_core(rest, rest, jb, -1.0f, w.LU + (int64_t)j0 * ld + j1, ld, w.LU + (int64_t)j1 * ld + j0, ld,
                           1.0f, w.LU + (int64_t)j1 * ld + j1, ld, variant, 0u, nullptr, 0, 0, nullptr, 0, 0, nullptr,
                           nullptr, 0, st, 0);
        }
    }
    if (rc == BF16X_SUCCESS) rc = check_launch("lu");
    cudaEventRecord(e1, st);
    int info = 0;
    if (rc == BF16X_SUCCESS) {
        cudaMemcpyAsync(&info, w.info, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) rc = check_launch("lu sync");
    }
    report->info = info;
    if (rc == BF16X_SUCCESS && info != 0) rc = BF16X_ERR_SINGULAR;

    // ---------------- refinement ----------------
    if (rc == BF16X_SUCCESS) {
        // ||A||_inf (row abs sums)
        residual(A, lda, n, nullptr, nullptr, w.r, w.part, 1, st);
        absmax_kernel<<<1, 256, 0, st>>>(n, w.r, w.scal + 2);
        count_launch();
        double anrm = 0.0;
        cudaMemcpyAsync(&anrm, w.scal + 2, sizeof(double), cudaMemcpyDeviceToHost, st);
        rc = solve_with_factors(w, n, b, x, coop_grid, st);
        const double eps = std::ldexp(1.0, -53);
        std::vector<double> hist;
        int it = 0;
        bool converged = false;
        double rn = 0.0, xn = 0.0;
        for (; rc == BF16X_SUCCESS; ++it) {
            residual(A, lda, n, x, b, w.r, w.part, 0, st);
            absmax_kernel<<<1, 256, 0, st>>>(n, w.r, w.scal);
            absmax_kernel<<<1, 256, 0, st>>>(n, x, w.scal + 1);
            count_launch(2);
            double h[2];
            cudaMemcpyAsync(h, w.scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, st);
            if (cudaStreamSynchronize(st) != cudaSuccess) {
                rc = check_launch("ir sync");
                break;
            }
            rn = h[0];
            xn = h[1];
            hist.push_back(rn);
            report->tol = std::sqrt((double)n) * xn * anrm * eps;
            if (rn <= report->tol) {
                converged = true;
                break;
            }
            if (it >= max_iter) break;
            if (hist.size() >= 4 && hist.back() > 0.5 * hist[hist.size() - 4]) break;  // stagnation
            rc = solve_with_factors(w, n, w.r, w.d, coop_grid, st);
            if (rc) break;
            axpy_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, x, w.d);
            count_launch();
        }
        report->converged = converged ? 1 : 0;
        report->iterations = it;
        report->final_residual = rn;
        report->backward_error = (anrm > 0 && xn > 0) ? rn / (anrm * xn) : 0.0;
        if (residual_history)
            for (size_t q = 0; q < hist.size() && q <= (size_t)max_iter; ++q) residual_history[q] = hist[q];
        if (rc == BF16X_SUCCESS && !converged) rc = BF16X_NOT_CONVERGED;
    }
    cudaEventRecord(e2, st);
    cudaEventSynchronize(e2);
    float f_ms = 0.f, r_ms = 0.f;
    cudaEventElapsedTime(&f_ms, e0, e1);
    cudaEventElapsedTime(&r_ms, e1, e2);
    report->factor_ms = f_ms;
    report->refine_ms = r_ms;
    cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2);
    cleanup();
    return rc;
}
