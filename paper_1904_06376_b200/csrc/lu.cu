// lu.cu -- a6: LU with partial pivoting whose cubic work runs in the split GEMM, followed by
// FP64 iterative refinement (section III: "Only the cubic work of the initial LU
// factorization should be done in the lower precision: all the other steps ... in the higher
// precision").
//
//   factor (FP32, in a device copy of A), blocked right-looking, panel width nb:
//     K4 subpanel_kernel    32-column sub-panels on one thread-block cluster (8-16 CTAs, rows in
//                           shared memory, pivot exchange through DSMEM + cluster barrier);
//        panel_update_kernel   TRSM + rank-32 update of the rest of the 256-wide panel
//     K5 laswp_kernel   applies the panel's interchanges to all n columns
//        trsm_kernel    U12 = L11^-1 A12 (FP32, unit lower)
//     K2 bf16x GEMM     A22 <- -1 * L21 U12 + 1 * A22 in bf16x<variant>   (the cubic work)
//   refine (FP64, factors widened exactly):
//     K6 residual       r = b - A x, deterministic two-phase row sums
//        trsv_kernel    cooperative blocked forward / backward substitution
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include <cooperative_groups.h>

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

// 4-byte global -> shared copy that does not occupy a register until it lands (LDGSTS), so
// tile-staging loops keep many loads in flight; finish with async_wait_all().
__device__ __forceinline__ void async_copy_f32(float *dst, const float *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------------------------
// K4: panel factorisation by sub-panels of kSubW columns.  Each sub-panel [s0, s0+w) is
// factored over rows [s0, n) by one thread-block cluster: the rows are split in contiguous
// chunks over the cluster's CTAs and held in shared memory ([col][row]).  Step t (column
// c = s0+t):
//   (a) unpivoted rows apply step t-1: l = a[i,c-1] / p[c-1] stored in place (the L
//       multiplier), a[i,c'] -= l * p[c'] for c' >= c, p = pivot row of step t-1;
//   (b) local argmax |a[i,c]| over unpivoted rows (ties -> lowest row, LAPACK isamax on the
//       unswapped order); the CTA publishes (|a|, row) and that row's entries in its own
//       shared memory; cluster barrier;
//   (c) every CTA reads the candidates and the winner's row through distributed shared memory
//       (identical reduction everywhere); the owner marks its row pivoted.
// Rows are not moved inside the sub-panel: the LAPACK interchange sequence is derived
// afterwards (build_ipiv_kernel) and applied to the panel columns (laswp_kernel); the
// remaining panel columns then receive the sub-panel's TRSM + rank-w update
// (panel_update_kernel).  All panel arithmetic is FP32.
// ------------------------------------------------------------------------------------
constexpr int kSubW = 32;
constexpr int kSubThreads = 512;

__global__ void __launch_bounds__(kSubThreads) subpanel_kernel(float *LU, int ld, int n, int s0, int w, int rl_max,
                                                              int *piv_rows, int *info) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int ncta = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    extern __shared__ float sm[];
    float *sp = sm;                                  // [w][rl_max]
    float *prow = sp + (size_t)w * rl_max;           // [w]    pivot row of the current step
    float *crow = prow + w;                          // [2][w] this CTA's candidate row
    float *cval = crow + 2 * w;                      // [2]    candidate |a|
    int *cidx = reinterpret_cast<int *>(cval + 2);   // [2]    candidate row
    unsigned char *smark = reinterpret_cast<unsigned char *>(cidx + 2);
    __shared__ float s_v[kSubThreads / 32];
    __shared__ int s_i[kSubThreads / 32];
    __shared__ int s_wr, s_gi;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int R = n - s0;
    const int r0 = s0 + (int)(((int64_t)R * rank) / ncta), r1 = s0 + (int)(((int64_t)R * (rank + 1)) / ncta);
    const int rl = r1 - r0;
    for (int cc = wid; cc < w; cc += nw)
        for (int e = lane; e < rl; e += 32) async_copy_f32(sp + cc * rl_max + e, LU + (int64_t)(s0 + cc) * ld + r0 + e);
    for (int e = tid; e < rl; e += blockDim.x) smark[e] = 0;
    async_wait_all();
    __syncthreads();
    for (int t = 0; t <= w; ++t) {
        if (t > 0) {
            const int tp = t - 1;
            const float piv = prow[tp];
            for (int e = tid; e < rl; e += blockDim.x)
                if (!smark[e]) sp[tp * rl_max + e] = (piv != 0.f) ? sp[tp * rl_max + e] / piv : 0.f;
            __syncthreads();
            for (int cc = t + wid; cc < w; cc += nw) {
                const float u = prow[cc];
                for (int e = lane; e < rl; e += 32)
                    if (!smark[e]) sp[cc * rl_max + e] = sp[cc * rl_max + e] - sp[tp * rl_max + e] * u;
            }
            __syncthreads();
        }
        if (t == w) break;
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
            for (int q = 1; q < nw; ++q)
                if (better(s_v[q], s_i[q], bv, bi)) { bv = s_v[q]; bi = s_i[q]; }
            cval[t & 1] = bv;
            cidx[t & 1] = bi;
            s_gi = (bi >= r0 && bi < r1) ? bi - r0 : -1;
        }
        __syncthreads();
        if (s_gi >= 0)
            for (int cc = t + tid; cc < w; cc += blockDim.x) crow[(t & 1) * w + cc] = sp[cc * rl_max + s_gi];
        cl.sync();
        if (tid < 32) {
            float gv = -1.f;
            int gi = 0x7FFFFFFF, gr = 0;
            for (int q = tid; q < ncta; q += 32) {
                const float v = *cl.map_shared_rank(&cval[t & 1], q);
                const int i = *cl.map_shared_rank(&cidx[t & 1], q);
                if (better(v, i, gv, gi)) { gv = v; gi = i; gr = q; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, gv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, gi, o);
                const int orr = __shfl_xor_sync(0xffffffffu, gr, o);
                if (better(ov, oi, gv, gi)) { gv = ov; gi = oi; gr = orr; }
            }
            if (tid == 0) {
                s_wr = gr;
                if (gi >= r0 && gi < r1) smark[gi - r0] = 1;
                if (rank == 0) {
                    piv_rows[t] = gi;
                    if (gv == 0.f && *info == 0) *info = s0 + t + 1;
                }
            }
        }
        __syncthreads();
        const float *src = cl.map_shared_rank(crow, s_wr) + (t & 1) * w;
        for (int cc = t + tid; cc < w; cc += blockDim.x) prow[cc] = src[cc];
        __syncthreads();
    }
    for (int cc = wid; cc < w; cc += nw)
        for (int e = lane; e < rl; e += 32) LU[(int64_t)(s0 + cc) * ld + r0 + e] = sp[cc * rl_max + e];
    cl.sync();   // peers may still read this CTA's candidate row
}

// After sub-panel [s0, s0+w) (rows already interchanged): remaining panel columns [c1, c2)
// get U = L11^-1 A[s0:s0+w, c1:c2] (L11 unit lower w x w; every block recomputes it, block 0
// stores it) and rows [c1, n) get A -= L21 U.  64 rows per block.
constexpr int kUpdRows = 64;
__global__ void __launch_bounds__(256) panel_update_kernel(float *LU, int ld, int n, int s0, int w, int c1, int c2) {
    extern __shared__ float su[];
    const int nc = c2 - c1;
    float *sU = su;                           // [w][nc]
    float *sL11 = sU + (size_t)w * nc;        // [w][w]   (row r, col i) at r*w + i
    float *sL21 = sL11 + (size_t)w * w;       // [w][kUpdRows] (col t, row r)
    const int tid = threadIdx.x;
    for (int e = tid; e < w * nc; e += blockDim.x) {
        const int r = e % w, c = e / w;
        async_copy_f32(sU + r * nc + c, LU + (int64_t)(c1 + c) * ld + s0 + r);
    }
    for (int e = tid; e < w * w; e += blockDim.x) {
        const int r = e % w, i = e / w;
        async_copy_f32(sL11 + r * w + i, LU + (int64_t)(s0 + i) * ld + s0 + r);
    }
    const int rb = c1 + blockIdx.x * kUpdRows;
    const int nr = min(kUpdRows, n - rb);
    for (int e = tid; e < w * kUpdRows; e += blockDim.x) {
        const int r = e % kUpdRows, t = e / kUpdRows;
        if (r < nr) async_copy_f32(sL21 + t * kUpdRows + r, LU + (int64_t)(s0 + t) * ld + rb + r);
        else sL21[t * kUpdRows + r] = 0.f;
    }
    async_wait_all();
    __syncthreads();
    for (int c = tid; c < nc; c += blockDim.x)       // forward substitution per column
        for (int i = 0; i < w - 1; ++i) {
            const float xi = sU[i * nc + c];
            for (int r = i + 1; r < w; ++r) sU[r * nc + c] -= sL11[r * w + i] * xi;
        }
    __syncthreads();
    if (blockIdx.x == 0)
        for (int e = tid; e < w * nc; e += blockDim.x) {
            const int r = e % w, c = e / w;
            LU[(int64_t)(c1 + c) * ld + s0 + r] = sU[r * nc + c];
        }
    // 8 outputs per round: their old values are loaded together (independent loads in flight)
    const int nout = kUpdRows * nc;
    for (int e0 = tid; e0 < nout; e0 += 8 * blockDim.x) {
        float old[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = e0 + q * blockDim.x;
            const int r = e % kUpdRows, c = e / kUpdRows;
            old[q] = (e < nout && r < nr) ? LU[(int64_t)(c1 + c) * ld + rb + r] : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = e0 + q * blockDim.x;
            const int r = e % kUpdRows, c = e / kUpdRows;
            if (e >= nout || r >= nr) continue;
            float acc = 0.f;
            for (int t = 0; t < w; ++t) acc = fmaf(sL21[t * kUpdRows + r], sU[t * nc + c], acc);
            LU[(int64_t)(c1 + c) * ld + rb + r] = old[q] - acc;
        }
    }
}

// Gather pairs (dst <- src) for an interchange sequence ipiv[j0 .. j0+jb) applied in order.
__global__ void build_pairs_kernel(int n, int j0, int jb, const int *ipiv, int *pos, int *row_at, int2 *pairs,
                                   int *npairs) {
    for (int i = j0 + threadIdx.x; i < n; i += blockDim.x) { pos[i] = i; row_at[i] = i; }
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int t = 0; t < jb; ++t) {
        const int here = j0 + t, q = ipiv[here];
        if (q == here) continue;
        const int a = row_at[here], b = row_at[q];
        row_at[here] = b; pos[b] = here;
        row_at[q] = a; pos[a] = q;
    }
    int np = 0;
    for (int t = 0; t < jb; ++t) {
        const int here = j0 + t;
        if (row_at[here] != here) pairs[np++] = make_int2(here, row_at[here]);
    }
    for (int t = 0; t < jb; ++t) {
        const int q = ipiv[j0 + t];
        if (q >= j0 + jb && row_at[q] != q && pos[q] != -1) {
            pairs[np++] = make_int2(q, row_at[q]);
            pos[q] = -1;
        }
    }
    *npairs = np;
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
    for (int r = ty; r < jb; r += 8) {
        if (valid) async_copy_f32(sB + r * kTrsmCols + tx, LU + (int64_t)(cb + tx) * ld + j0 + r);
        else sB[r * kTrsmCols + tx] = 0.f;
    }
    for (int i0 = 0; i0 < jb; i0 += 32) {
        const int ib = min(32, jb - i0);
        __syncthreads();
        for (int e = threadIdx.x; e < (jb - i0) * ib; e += blockDim.x) {
            const int r = e % (jb - i0), c = e / (jb - i0);
            async_copy_f32(sL + r * 33 + c, LU + (int64_t)(j0 + i0 + c) * ld + j0 + i0 + r);
        }
        async_wait_all();
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
    for (int jb = j0; jb < j1; jb += 16) {
        float a[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) a[q] = (jb + q < j1) ? __ldg(A + (int64_t)(jb + q) * ld + i) : 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (jb + q < j1) s += absval ? fabs((double)a[q]) : (double)a[q] * x[jb + q];
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

constexpr int kTrsvBlock = 128;

constexpr int kTS = kTrsvBlock + 4;   // smem column stride (floats): 16-byte aligned columns
constexpr int kTrsvSmem = 2 * kTrsvBlock * kTS * sizeof(float) + 3 * kTrsvBlock * sizeof(double);

// acc = sum_{j < pw} LU[(pc0 + j) * ld + r] * sx[j], 16 independent loads in flight per batch
// acc = sum_{j < pw} LU[(pc0 + j) * ld + r] * sx[j] (pw <= kTrsvBlock): all loads are issued
// before the first FMA, so the row costs one memory round trip.
__device__ __forceinline__ double dot_col_block(const float *LU, int64_t ld, int pc0, int pw, int r, const double *sx) {
    float a[kTrsvBlock];
#pragma unroll
    for (int q = 0; q < kTrsvBlock; ++q) a[q] = (q < pw) ? __ldg(LU + (int64_t)(pc0 + q) * ld + r) : 0.f;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < kTrsvBlock; ++q) acc = fma((double)a[q], (q < pw) ? sx[q] : 0.0, acc);
    return acc;
}

// Asynchronously copy the rows x cols tile LU[r0.., c0..] into smem [col][kTS] (LDGSTS).
__device__ __forceinline__ void prefetch_tile(float *dst, const float *LU, int64_t ld, int r0, int rows, int c0,
                                              int cols) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c = wid; c < cols; c += nw) {
        const float *src = LU + (int64_t)(c0 + c) * ld + r0;
        for (int r = lane; r < rows; r += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst + c * kTS + r)), "l"(src + r)
                         : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// Blocked triangular solve in FP64 with the FP32 factors, cooperative grid.  lower != 0:
// L y = y (unit diagonal, forward); else U y = y (backward).  Step s handles block b_s (128
// rows): CTA 0 owns the critical path -- the block's diagonal tile and the tile coupling it to
// the previous block were prefetched into shared memory (cp.async) during the previous
// barrier, so it applies the previous block to b_s's rows, solves the diagonal triangle and
// publishes x_{b_s}; CTAs 1.. apply the previous block to every other dependent row.  One
// grid barrier per block.  y is accessed with L2-coherent loads/stores.
__global__ void __launch_bounds__(256) trsv_kernel(const float *LU, int ld, int n, double *y, int lower, GridBar gb,
                                                   unsigned int epoch) {
    extern __shared__ double sdyn[];
    double *sx = sdyn;                             // [kTrsvBlock] solution of the previous block
    double *sy = sx + kTrsvBlock;                  // [kTrsvBlock] current block (CTA 0)
    double *sp = sy + kTrsvBlock;                  // [kTrsvBlock] partial sums (CTA 0)
    float *sL = reinterpret_cast<float *>(sp + kTrsvBlock);   // [col][kTS] diagonal tile
    float *sB = sL + kTrsvBlock * kTS;                        // [col][kTS] coupling tile
    const int nblk = (n + kTrsvBlock - 1) / kTrsvBlock;
    const int G = gridDim.x, tid = threadIdx.x;
    auto blk = [&](int s, int &c0, int &w) {
        const int b = lower ? s : nblk - 1 - s;
        c0 = b * kTrsvBlock;
        w = min(n, c0 + kTrsvBlock) - c0;
    };
    if (blockIdx.x == 0) {
        int c0, w;
        blk(0, c0, w);
        prefetch_tile(sL, LU, ld, c0, w, c0, w);
    }
    int pc0 = 0, pw = 0;                  // previous block [pc0, pc0+pw)
    for (int s = 0; s < nblk; ++s) {
        int c0, w;
        blk(s, c0, w);
        const int c1 = c0 + w;
        if (s > 0) {
            for (int e = tid; e < pw; e += blockDim.x) sx[e] = __ldcg(y + pc0 + e);
            __syncthreads();
        }
        if (blockIdx.x == 0) {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            // y_b - (coupling tile) x_prev : 2 threads per row, half of the previous block each
            if (tid < 2 * w) {
                const int r = tid % w, hsel = tid / w, half = pw / 2;
                const int jb = hsel ? half : 0, je = hsel ? pw : half;
                double part = 0.0;
                for (int j = jb; j < je; ++j) part = fma((double)sB[j * kTS + r], sx[j], part);
                if (hsel) sp[r] = part; else sy[r] = part;
            }
            __syncthreads();
            for (int e = tid; e < w; e += blockDim.x) sy[e] = __ldcg(y + c0 + e) - (sy[e] + sp[e]);
            __syncthreads();
            // diagonal triangle: 32-row sub-blocks, each solved by warp 0 in registers with
            // shuffles, then applied to the rest of the block by all threads
            const int nsb = (w + 31) / 32;
            for (int q = 0; q < nsb; ++q) {
                const int sb = lower ? q * 32 : (nsb - 1 - q) * 32;
                const int sw = min(32, w - sb);
                if (tid < 32) {
                    double v = (tid < sw) ? sy[sb + tid] : 0.0;
                    if (lower) {
                        for (int j = 0; j < sw; ++j) {
                            const double xj = __shfl_sync(0xffffffffu, v, j);
                            if (tid > j && tid < sw) v -= (double)sL[(sb + j) * kTS + sb + tid] * xj;
                        }
                    } else {
                        for (int j = sw - 1; j >= 0; --j) {
                            if (tid == j) v /= (double)sL[(sb + j) * kTS + sb + j];
                            const double xj = __shfl_sync(0xffffffffu, v, j);
                            if (tid < j) v -= (double)sL[(sb + j) * kTS + sb + tid] * xj;
                        }
                    }
                    if (tid < sw) sy[sb + tid] = v;
                }
                __syncthreads();
                const int lo = lower ? sb + sw : 0, hi = lower ? w : sb;
                for (int r = lo + tid; r < hi; r += blockDim.x) {
                    double acc = 0.0;
                    for (int j = 0; j < sw; ++j) acc = fma((double)sL[(sb + j) * kTS + r], sy[sb + j], acc);
                    sy[r] -= acc;
                }
                __syncthreads();
            }
            for (int e = tid; e < w; e += blockDim.x) __stcg(y + c0 + e, sy[e]);
            __syncthreads();
            if (s + 1 < nblk) {          // next step's tiles, in flight during the barrier
                int n0, nw_;
                blk(s + 1, n0, nw_);
                prefetch_tile(sL, LU, ld, n0, nw_, n0, nw_);
                prefetch_tile(sB, LU, ld, n0, nw_, c0, w);
            }
        } else if (s > 0) {
            const int lo = lower ? c1 : 0, hi = lower ? n : c0;
            for (int r = lo + (blockIdx.x - 1) * blockDim.x + tid; r < hi; r += (G - 1) * blockDim.x) {
                const double acc = dot_col_block(LU, ld, pc0, pw, r, sx);
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
    float *LU = nullptr;
    int *ipiv = nullptr, *piv_rows = nullptr, *pos = nullptr, *row_at = nullptr, *info = nullptr;
    int *perm = nullptr, *npairs = nullptr;
    int2 *pairs = nullptr;
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
    int rc = coop_launch((const void *)trsv_kernel, coop_grid, 256, args, kTrsvSmem, st);
    w.epoch += nblk;
    if (rc) return rc;
    lower = 0;
    ep = w.epoch;
    rc = coop_launch((const void *)trsv_kernel, coop_grid, 256, args, kTrsvSmem, st);
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
    // sub-panel rows per cluster CTA in shared memory: cluster of 8 (portable) or 16
    int cl = 16;                           // non-portable cluster size (falls back to 8)
    int rl_max = (n + cl - 1) / cl + 1;
    auto sub_smem = [&](int rl) {
        return (size_t)kSubW * rl * sizeof(float) + (size_t)3 * kSubW * sizeof(float) + 16 + (size_t)rl + 16;
    };
    if (sub_smem(rl_max) > 200 * 1024) {
        cl = 16;
        rl_max = (n + cl - 1) / cl + 1;
    }
    if (sub_smem(rl_max) > 200 * 1024 || (size_t)n * sizeof(int) > 200 * 1024) {
        set_error_msg("gesv_ir: n too large for the shared-memory sub-panel (n <= ~51000)");
        return -1;
    }
    {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(subpanel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
            cudaFuncSetAttribute(subpanel_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaFuncSetAttribute(build_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
            cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
            cudaFuncSetAttribute(panel_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
            cudaFuncSetAttribute(trsv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsvSmem);
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
    alloc((void **)&w.piv_rows, sizeof(int) * (size_t)kSubW);
    alloc((void **)&w.pos, sizeof(int) * n);
    alloc((void **)&w.row_at, sizeof(int) * n);
    alloc((void **)&w.info, sizeof(int));
    alloc((void **)&w.npairs, sizeof(int));
    alloc((void **)&w.pairs, sizeof(int2) * 2 * (size_t)nb);
    alloc((void **)&w.bar, sizeof(unsigned int) * ((size_t)coop_grid + 1));
    alloc((void **)&w.r, sizeof(double) * n);
    alloc((void **)&w.d, sizeof(double) * n);
    alloc((void **)&w.part, sizeof(double) * (size_t)n * nchunk);
    alloc((void **)&w.scal, sizeof(double) * 4);
    auto cleanup = [&]() {
        cudaFree(w.LU); cudaFree(w.ipiv); cudaFree(w.perm); cudaFree(w.piv_rows); cudaFree(w.pos);
        cudaFree(w.row_at); cudaFree(w.info); cudaFree(w.npairs); cudaFree(w.pairs);
        cudaFree(w.bar); cudaFree(w.r); cudaFree(w.d); cudaFree(w.part); cudaFree(w.scal);
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
    auto laswp = [&](int c0, int c1, int pair_cap) {
        if (c1 <= c0) return;
        laswp_kernel<<<(c1 - c0 + 7) / 8, 256, 8 * (size_t)pair_cap * sizeof(float), st>>>(w.LU, ld, c0, c1, w.pairs,
                                                                                          w.npairs);
        count_launch();
    };
    for (int j0 = 0; j0 < n && !rc; j0 += nb) {
        const int jb = std::min(nb, n - j0);
        for (int s0 = j0; s0 < j0 + jb && !rc; s0 += kSubW) {
            const int sw = std::min(kSubW, j0 + jb - s0);
            // (1) sub-panel factorisation on one cluster
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cl);
            cfg.blockDim = dim3(kSubThreads);
            cfg.dynamicSmemBytes = sub_smem(rl_max);
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaError_t e = cudaLaunchKernelEx(&cfg, subpanel_kernel, w.LU, ld, n, s0, sw, rl_max, w.piv_rows, w.info);
            if (e != cudaSuccess && cl == 16) {    // 16-CTA clusters unavailable: use 8
                cudaGetLastError();
                cl = 8;
                rl_max = (n + cl - 1) / cl + 1;
                if (sub_smem(rl_max) <= 200 * 1024) {
                    cfg.gridDim = dim3(cl);
                    at[0].val.clusterDim.x = cl;
                    cfg.dynamicSmemBytes = sub_smem(rl_max);
                    e = cudaLaunchKernelEx(&cfg, subpanel_kernel, w.LU, ld, n, s0, sw, rl_max, w.piv_rows, w.info);
                }
            }
            if (e != cudaSuccess) {
                set_cuda_error(e, "subpanel launch");
                rc = BF16X_ERR_CUDA;
                break;
            }
            count_launch();
            // (2) its interchanges, applied to the panel columns
            build_ipiv_kernel<<<1, 1024, 0, st>>>(n, s0, sw, w.piv_rows, w.ipiv, w.pos, w.row_at, w.pairs, w.npairs);
            count_launch();
            laswp(j0, j0 + jb, 2 * sw);
            // (3) TRSM + rank-sw update of the rest of the panel
            const int c1 = s0 + sw, c2 = j0 + jb;
            if (c1 < c2) {
                const size_t smem = ((size_t)sw * (c2 - c1) + (size_t)sw * sw + (size_t)sw * kUpdRows) * sizeof(float);
                panel_update_kernel<<<(n - c1 + kUpdRows - 1) / kUpdRows, 256, smem, st>>>(w.LU, ld, n, s0, sw, c1,
                                                                                            c2);
                count_launch();
            }
            rc = check_launch("panel");
        }
        if (rc) break;
        // the panel's whole interchange sequence on the columns outside it
        build_pairs_kernel<<<1, 1024, 0, st>>>(n, j0, jb, w.ipiv, w.pos, w.row_at, w.pairs, w.npairs);
        count_launch();
        laswp(0, j0, 2 * jb);
        laswp(j0 + jb, n, 2 * jb);
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
