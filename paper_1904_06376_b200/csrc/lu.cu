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
// Grid barrier for cooperative launches (all CTAs co-resident).  Every CTA publishes its
// arrival epoch in its own flag word (no atomic serialisation); CTA 0 gathers the flags in
// parallel and publishes the release epoch.  Epochs increase monotonically across launches
// (the host passes each launch its first epoch), so no reset is needed.
// ------------------------------------------------------------------------------------
struct GridBar {
    unsigned int *arrive;   // [gridDim.x]
    unsigned int *release;  // [1]
};

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned int *p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void grid_sync(const GridBar &gb, unsigned int epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        st_release(gb.arrive + blockIdx.x, epoch);
    }
    if (blockIdx.x == 0) {
        for (unsigned int i = threadIdx.x; i < gridDim.x; i += blockDim.x)
            while (ld_acquire(gb.arrive + i) < epoch) {}
        __syncthreads();
        if (threadIdx.x == 0) st_release(gb.release, epoch);
    }
    if (threadIdx.x == 0) {
        while (ld_acquire(gb.release) < epoch) {}
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
// K4: panel factorisation of columns [j0, j0+jb) over rows [j0, n).  Rows are split into
// contiguous chunks, one per CTA, held in shared memory for the whole panel ([col][row]).
// Step t (column c = j0+t):
//   (a) unpivoted rows apply step t-1: l = a[i,c-1] / p[c-1] stored in place (the L
//       multiplier), a[i,c'] -= l * p[c'] for panel columns c' >= c, p = pivot row of step t-1;
//   (b) local argmax |a[i,c]| over unpivoted rows; the CTA publishes (|a|, row) and that row's
//       entries c..j0+jb-1; grid barrier;
//   (c) every CTA reduces the candidates identically (ties -> lowest row, LAPACK isamax on
//       the unswapped order) and copies the winner's row; the owner marks it pivoted.
// Rows are not moved: the LAPACK interchange sequence is derived afterwards (build_ipiv).
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kLuThreads) panel_kernel(float *LU, int ld, int n, int j0, int jb, int rl_max,
                                                           PivotCand *cand, float *cand_rows, int *piv_rows,
                                                           int *info, GridBar gb, unsigned int epoch) {
    extern __shared__ float sp[];            // [jb][rl_max] panel rows, then prow[jb], then marks
    float *prow = sp + (size_t)jb * rl_max;
    unsigned char *smark = reinterpret_cast<unsigned char *>(prow + jb);
    __shared__ float s_v[kLuThreads / 32];
    __shared__ int s_i[kLuThreads / 32];
    __shared__ int s_p, s_owner_e;
    const int nbk = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nw = blockDim.x >> 5;
    const int R = n - j0;
    const int r0 = j0 + (int)(((int64_t)R * b) / nbk), r1 = j0 + (int)(((int64_t)R * (b + 1)) / nbk);
    const int rl = r1 - r0;
    for (int cc = wid; cc < jb; cc += nw)
        for (int e = lane; e < rl; e += 32) sp[cc * rl_max + e] = LU[(int64_t)(j0 + cc) * ld + r0 + e];
    for (int e = tid; e < rl; e += blockDim.x) smark[e] = 0;
    __syncthreads();
    for (int t = 0; t <= jb; ++t) {
        if (t > 0) {
            const int tp = t - 1;
            const float piv = prow[tp];
            for (int e = tid; e < rl; e += blockDim.x)
                if (!smark[e]) sp[tp * rl_max + e] = (piv != 0.f) ? sp[tp * rl_max + e] / piv : 0.f;
            __syncthreads();
            for (int cc = t + wid; cc < jb; cc += nw) {
                const float u = prow[cc];
                for (int e = lane; e < rl; e += 32)
                    if (!smark[e]) sp[cc * rl_max + e] = sp[cc * rl_max + e] - sp[tp * rl_max + e] * u;
            }
            __syncthreads();
        }
        if (t == jb) break;
        float bv = -1.f;
        int bi = 0x7FFFFFFF;
        for (int e = tid; e < rl; e += blockDim.x) {
            if (smark[e]) continue;
            const float v = fabsf(sp[t * rl_max + e]);
            if (better(v, r0 + e, bv, bi)) { bv = v; bi = r0 + e; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
        }
        if (lane == 0) { s_v[wid] = bv; s_i[wid] = bi; }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < nw; ++w)
                if (better(s_v[w], s_i[w], bv, bi)) { bv = s_v[w]; bi = s_i[w]; }
            cand[(t & 1) * nbk + b] = {bv, bi};
            s_owner_e = (bi >= r0 && bi < r1) ? bi - r0 : -1;
        }
        __syncthreads();
        if (s_owner_e >= 0) {
            float *dst = cand_rows + ((size_t)(t & 1) * nbk + b) * jb;
            for (int cc = t + tid; cc < jb; cc += blockDim.x) dst[cc] = sp[cc * rl_max + s_owner_e];
        }
        grid_sync(gb, epoch + t);
        if (tid < 32) {
            float gv = -1.f;
            int gi = 0x7FFFFFFF, gb_ = 0;
            for (int k = tid; k < nbk; k += 32) {
                const float2 raw = __ldcg(reinterpret_cast<const float2 *>(cand + (t & 1) * nbk + k));
                const float v = raw.x;
                const int i = __float_as_int(raw.y);
                if (better(v, i, gv, gi)) { gv = v; gi = i; gb_ = k; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, gv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, gi, o);
                const int ob = __shfl_xor_sync(0xffffffffu, gb_, o);
                if (better(ov, oi, gv, gi)) { gv = ov; gi = oi; gb_ = ob; }
            }
            if (tid == 0) {
                s_p = gb_;
                if (gi >= r0 && gi < r1) smark[gi - r0] = 1;
                if (b == 0) {
                    piv_rows[t] = gi;
                    if (gv == 0.f && *info == 0) *info = j0 + t + 1;
                }
            }
        }
        __syncthreads();
        const float *src = cand_rows + ((size_t)(t & 1) * nbk + s_p) * jb;
        for (int cc = t + tid; cc < jb; cc += blockDim.x) prow[cc] = __ldcg(src + cc);
        __syncthreads();
    }
    for (int cc = wid; cc < jb; cc += nw)
        for (int e = lane; e < rl; e += 32) LU[(int64_t)(j0 + cc) * ld + r0 + e] = sp[cc * rl_max + e];
}

// LAPACK interchange sequence from the chosen physical rows: step t swaps position j0+t with
// the current position of row piv_rows[t] (ipiv, 0-based).  The net effect on the touched
// positions is emitted as gather pairs (dst <- src) for laswp.  One CTA: parallel init, the
// jb-step simulation on thread 0.
__global__ void build_ipiv_kernel(int n, int j0, int jb, const int *piv_rows, int *ipiv, int *pos, int *row_at,
                                  int2 *pairs, int *npairs) {
    for (int i = j0 + threadIdx.x; i < n; i += blockDim.x) { pos[i] = i; row_at[i] = i; }
    __syncthreads();
    if (threadIdx.x != 0) return;
    int np = 0;
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
    // touched positions: j0..j0+jb-1 and every q that received a displaced row
    for (int t = 0; t < jb; ++t) {
        const int here = j0 + t;
        if (row_at[here] != here) pairs[np++] = make_int2(here, row_at[here]);
    }
    for (int t = 0; t < jb; ++t) {
        const int q = ipiv[j0 + t];
        if (q >= j0 + jb && row_at[q] != q && pos[q] != -1) {
            pairs[np++] = make_int2(q, row_at[q]);
            pos[q] = -1;                   // pos is dead after the simulation: reuse as "emitted"
        }
    }
    *npairs = np;
}

// K5a: apply the panel's row interchanges to columns [c0, c1) as a gather through shared
// memory: one warp per column, lanes over the (dst <- src) pairs.
__global__ void __launch_bounds__(256) laswp_kernel(float *LU, int ld, int c0, int c1, const int2 *pairs,
                                                    const int *npairs) {
    extern __shared__ float sv[];          // [8 warps][np]
    const int np = *npairs;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = c0 + blockIdx.x * 8 + wid;
    if (np == 0 || c >= c1) return;
    float *col = LU + (int64_t)c * ld;
    float *buf = sv + wid * np;
    for (int e = lane; e < np; e += 32) buf[e] = col[pairs[e].y];
    __syncwarp();
    for (int e = lane; e < np; e += 32) col[pairs[e].x] = buf[e];
}

// K5b: U12 = L11^-1 A12 with L11 = unit lower jb x jb at (j0, j0), A12 = rows j0..j0+jb of
// columns [c0, c0 + ncols).  One CTA per 32 columns held in shared memory; L11 is staged in
// 32-column chunks: each chunk's 32x32 diagonal triangle is solved step by step, then the
// rows below it take the chunk's contribution as one small product (no barrier per row).
constexpr int kTrsmCols = 32;
__global__ void __launch_bounds__(256) trsm_kernel(float *LU, int ld, int j0, int jb, int c0, int ncols) {
    extern __shared__ float sm[];
    float *sB = sm;                                   // [jb][32]
    float *sL = sm + (size_t)jb * kTrsmCols;          // [jb][33]: rows i0.., chunk columns
    const int cb = c0 + blockIdx.x * kTrsmCols;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 columns x 8 row groups
    const bool valid = (cb + tx) < c0 + ncols;
    for (int r = ty; r < jb; r += 8) sB[r * kTrsmCols + tx] = valid ? LU[(int64_t)(cb + tx) * ld + j0 + r] : 0.f;
    for (int i0 = 0; i0 < jb; i0 += 32) {
        const int ib = min(32, jb - i0);
        __syncthreads();
        for (int e = threadIdx.x; e < (jb - i0) * ib; e += blockDim.x) {
            const int r = e % (jb - i0), c = e / (jb - i0);
            sL[r * 33 + c] = LU[(int64_t)(j0 + i0 + c) * ld + j0 + i0 + r];
        }
        __syncthreads();
        for (int i = 0; i < ib - 1; ++i) {
            const float xi = sB[(i0 + i) * kTrsmCols + tx];
            for (int r = i + 1 + ty; r < ib; r += 8) sB[(i0 + r) * kTrsmCols + tx] -= sL[r * 33 + i] * xi;
            __syncthreads();
        }
        for (int r = i0 + ib + ty; r < jb; r += 8) {
            float acc = 0.f;
            for (int i = 0; i < ib; ++i) acc = fmaf(sL[(r - i0) * 33 + i], sB[(i0 + i) * kTrsmCols + tx], acc);
            sB[r * kTrsmCols + tx] -= acc;
        }
    }
    __syncthreads();
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
        s += absval ? fabs(a) : a * x[j];
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

// perm[i] = source index of y[i] in y = P v (interchanges applied in order); one CTA.
__global__ void build_perm_kernel(int n, const int *ipiv, int *perm) {
    extern __shared__ int sp_i[];
    for (int i = threadIdx.x; i < n; i += blockDim.x) sp_i[i] = i;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int j = 0; j < n; ++j) {
            const int q = ipiv[j];
            if (q != j) { const int t = sp_i[j]; sp_i[j] = sp_i[q]; sp_i[q] = t; }
        }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = sp_i[i];
}
__global__ void gather_kernel(int n, const int *perm, const double *v, double *y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = v[perm[i]];
}

// Blocked triangular solve in FP64 with the FP32 factors, cooperative grid.  lower != 0:
// L y = y (unit diagonal, forward); else U y = y (backward).  Step s handles block b_s: CTA 0
// applies the previous block's solution to b_s's rows and solves b_s's diagonal triangle in
// shared memory, while CTAs 1.. apply the previous block to every other dependent row; one
// grid barrier per block.  y is accessed with L2-coherent loads/stores.
constexpr int kTrsvBlock = 64;
__global__ void __launch_bounds__(256) trsv_kernel(const float *LU, int ld, int n, double *y, int lower, GridBar gb,
                                                   unsigned int epoch) {
    __shared__ double sx[kTrsvBlock];      // solution of the previous block
    __shared__ double sy[kTrsvBlock];      // right-hand side of the current block (CTA 0)
    __shared__ float sL[kTrsvBlock][kTrsvBlock + 1];
    const int nblk = (n + kTrsvBlock - 1) / kTrsvBlock;
    const int G = gridDim.x;
    int pc0 = 0, pw = 0;                  // previous block [pc0, pc0+pw)
    for (int s = 0; s < nblk; ++s) {
        const int bidx = lower ? s : nblk - 1 - s;
        const int c0 = bidx * kTrsvBlock, c1 = min(n, c0 + kTrsvBlock), w = c1 - c0;
        if (s > 0) {
            for (int e = threadIdx.x; e < pw; e += blockDim.x) sx[e] = __ldcg(y + pc0 + e);
            __syncthreads();
        }
        if (blockIdx.x == 0) {
            for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
                const int r = e % w, c = e / w;
                sL[r][c] = LU[(int64_t)(c0 + c) * ld + c0 + r];
            }
            for (int e = threadIdx.x; e < w; e += blockDim.x) {
                double v = __ldcg(y + c0 + e);
                for (int j = 0; j < pw; ++j) v -= (double)LU[(int64_t)(pc0 + j) * ld + c0 + e] * sx[j];
                sy[e] = v;
            }
            __syncthreads();
            if (threadIdx.x < 32) {
                for (int jj = 0; jj < w; ++jj) {
                    const int j = lower ? jj : w - 1 - jj;
                    if (!lower && threadIdx.x == 0) sy[j] /= (double)sL[j][j];
                    __syncwarp();
                    const double xj = sy[j];
                    for (int r = threadIdx.x; r < w; r += 32)
                        if (lower ? (r > j) : (r < j)) sy[r] -= (double)sL[r][j] * xj;
                    __syncwarp();
                }
            }
            __syncthreads();
            for (int e = threadIdx.x; e < w; e += blockDim.x) __stcg(y + c0 + e, sy[e]);
        } else if (s > 0) {
            // rows still depending on the previous block, except the current block's rows
            const int lo = lower ? c1 : 0, hi = lower ? n : c0;
            for (int r = lo + (blockIdx.x - 1) * blockDim.x + threadIdx.x; r < hi; r += (G - 1) * blockDim.x) {
                double acc = 0.0;
                for (int j = 0; j < pw; ++j) acc += (double)LU[(int64_t)(pc0 + j) * ld + r] * sx[j];
                __stcg(y + r, __ldcg(y + r) - acc);
            }
        }
        grid_sync(gb, epoch + s);
        pc0 = c0;
        pw = w;
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
    float *LU = nullptr, *cand_rows = nullptr;
    int *ipiv = nullptr, *piv_rows = nullptr, *pos = nullptr, *row_at = nullptr, *info = nullptr;
    int *perm = nullptr, *npairs = nullptr;
    int2 *pairs = nullptr;
    PivotCand *cand = nullptr;
    unsigned int *bar = nullptr;  // [grid] arrive flags + [1] release
    GridBar gb;
    unsigned int epoch = 1;
    double *r = nullptr, *d = nullptr, *part = nullptr, *scal = nullptr;
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

static int solve_with_factors(LuWork &w, int n, const double *v, double *out, int coop_grid, cudaStream_t st) {
    // out = U^-1 L^-1 P v
    gather_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, w.perm, v, out);
    count_launch();
    int ld = n, lower = 1;
    const float *LU = w.LU;
    double *y = out;
    GridBar gb = w.gb;
    unsigned int ep = w.epoch;
    void *args[] = {(void *)&LU, (void *)&ld, (void *)&n, (void *)&y, (void *)&lower, (void *)&gb, (void *)&ep};
    const int nblk = (n + kTrsvBlock - 1) / kTrsvBlock;
    int rc = coop_launch((const void *)trsv_kernel, coop_grid, 256, args, 0, st);
    w.epoch += nblk;
    if (rc) return rc;
    lower = 0;
    ep = w.epoch;
    rc = coop_launch((const void *)trsv_kernel, coop_grid, 256, args, 0, st);
    w.epoch += nblk;
    return rc;
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
    nb = std::min(nb, n);
    if (max_iter <= 0) max_iter = 30;
    cudaStream_t st = current_stream();
    const int coop_grid = num_sms();
    // panel rows per CTA held in shared memory for the whole panel
    const int rl_max = (n + coop_grid - 1) / coop_grid + 1;
    const size_t panel_smem = (size_t)nb * rl_max * sizeof(float) + (size_t)nb * sizeof(float) + rl_max + 16;
    if (panel_smem > 200 * 1024 || (size_t)n * sizeof(int) > 200 * 1024) {
        set_error_msg("gesv_ir: n * nb too large for the shared-memory panel (n/148 * nb * 4 B <= 200 KB)");
        return -1;
    }
    {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
            cudaFuncSetAttribute(build_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
            cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
            attr = true;
        }
    }
    LuWork w;
    const int nchunk = (n + kResChunk - 1) / kResChunk;
    auto alloc = [&](void **p, size_t bytes) {
        if (rc) return;
        if (cudaMalloc(p, bytes) != cudaSuccess) {
            cudaGetLastError();
            rc = BF16X_ERR_ALLOC;
        }
    };
    alloc((void **)&w.LU, sizeof(float) * (size_t)n * n);
    alloc((void **)&w.ipiv, sizeof(int) * n);
    alloc((void **)&w.perm, sizeof(int) * n);
    alloc((void **)&w.piv_rows, sizeof(int) * (size_t)nb);
    alloc((void **)&w.pos, sizeof(int) * n);
    alloc((void **)&w.row_at, sizeof(int) * n);
    alloc((void **)&w.info, sizeof(int));
    alloc((void **)&w.npairs, sizeof(int));
    alloc((void **)&w.pairs, sizeof(int2) * 2 * (size_t)nb);
    alloc((void **)&w.cand, sizeof(PivotCand) * 2 * (size_t)coop_grid);
    alloc((void **)&w.cand_rows, sizeof(float) * 2 * (size_t)coop_grid * nb);
    alloc((void **)&w.bar, sizeof(unsigned int) * ((size_t)coop_grid + 1));
    alloc((void **)&w.r, sizeof(double) * n);
    alloc((void **)&w.d, sizeof(double) * n);
    alloc((void **)&w.part, sizeof(double) * (size_t)n * nchunk);
    alloc((void **)&w.scal, sizeof(double) * 4);
    auto cleanup = [&]() {
        cudaFree(w.LU); cudaFree(w.ipiv); cudaFree(w.perm); cudaFree(w.piv_rows); cudaFree(w.pos);
        cudaFree(w.row_at); cudaFree(w.info); cudaFree(w.npairs); cudaFree(w.pairs); cudaFree(w.cand);
        cudaFree(w.cand_rows); cudaFree(w.bar); cudaFree(w.r); cudaFree(w.d); cudaFree(w.part); cudaFree(w.scal);
    };
    if (rc) {
        cleanup();
        return rc;
    }
    w.gb.arrive = w.bar;
    w.gb.release = w.bar + coop_grid;
    cudaMemsetAsync(w.bar, 0, sizeof(unsigned int) * ((size_t)coop_grid + 1), st);
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
            float *LU = w.LU, *cand_rows = w.cand_rows;
            int ldv = ld, nv = n, j0v = j0, jbv = jb, rlv = rl_max;
            PivotCand *cand = w.cand;
            int *piv = w.piv_rows, *info = w.info;
            GridBar gb = w.gb;
            unsigned int ep = w.epoch;
            void *args[] = {&LU, &ldv, &nv, &j0v, &jbv, &rlv, &cand, &cand_rows, &piv, &info, &gb, &ep};
            const size_t smem = (size_t)jb * rl_max * sizeof(float) + (size_t)jb * sizeof(float) + rl_max + 16;
            rc = coop_launch((const void *)panel_kernel, coop_grid, kLuThreads, args, smem, st);
            w.epoch += jb;
            if (rc) break;
        }
        build_ipiv_kernel<<<1, 1024, 0, st>>>(n, j0, jb, w.piv_rows, w.ipiv, w.pos, w.row_at, w.pairs, w.npairs);
        laswp_kernel<<<(n + 7) / 8, 256, 8 * 2 * (size_t)jb * sizeof(float), st>>>(w.LU, ld, 0, n, w.pairs, w.npairs);
        count_launch(2);
        const int j1 = j0 + jb, rest = n - j1;
        if (rest > 0) {
            trsm_kernel<<<(rest + kTrsmCols - 1) / kTrsmCols, 256, (size_t)jb * (kTrsmCols + 33) * sizeof(float), st>>>(
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
    if (rc == BF16X_SUCCESS) {
        build_perm_kernel<<<1, 1024, (size_t)n * sizeof(int), st>>>(n, w.ipiv, w.perm);
        count_launch();
        rc = check_launch("lu");
    }
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
