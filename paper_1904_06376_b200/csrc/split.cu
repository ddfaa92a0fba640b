// split.cu -- K1: the FP32 -> {b0, b1, b2} BF16 split of P:180-184 (section II-A) as an
// HBM-bound pre-pass.  Two layouts:
//   split_same  : pieces keep the source's column-major layout (bf16x_split; also the
//                 K-major B operand of the GEMM, since B is k x n column-major)
//   split_trans : pieces are written transposed (bf16x_split_t; the K-major A operand)
// Algorithmic traffic: 4 B read + 2p B written per element (p = pieces kept).
#include "common.cuh"
#include "kernels.cuh"

namespace bf16x {

// ---------------------------------------------------------------------------------
// same layout: each thread splits 8 consecutive rows of one column; 16-byte vector
// loads/stores when the whole matrix is 16-byte aligned (vec != 0).
// ---------------------------------------------------------------------------------
template <int NP>
__global__ void __launch_bounds__(256) split_same_kernel(int64_t rows, int64_t cols, const float *__restrict__ X,
                                                         int64_t ldx, uint16_t *__restrict__ P0,
                                                         uint16_t *__restrict__ P1, uint16_t *__restrict__ P2,
                                                         int64_t ldp, int vec) {
    const int64_t nchunk = (rows + 7) / 8;
    for (int64_t col = blockIdx.y; col < cols; col += gridDim.y) {
        const float *x = X + col * ldx;
        const int64_t o = col * ldp;
        for (int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ch < nchunk;
             ch += (int64_t)gridDim.x * blockDim.x) {
            const int64_t r0 = ch * 8;
            if (vec && r0 + 8 <= rows) {
                float4 u = __ldcs(reinterpret_cast<const float4 *>(x + r0));
                float4 w = __ldcs(reinterpret_cast<const float4 *>(x + r0 + 4));
                float v[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
                uint32_t q0[4], q1[4], q2[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    Split3 a = split3(v[2 * i]), b = split3(v[2 * i + 1]);
                    q0[i] = a.b0 | (b.b0 << 16);
                    q1[i] = a.b1 | (b.b1 << 16);
                    q2[i] = a.b2 | (b.b2 << 16);
                }
                __stcs(reinterpret_cast<uint4 *>(P0 + o + r0), make_uint4(q0[0], q0[1], q0[2], q0[3]));
                if (NP >= 2) __stcs(reinterpret_cast<uint4 *>(P1 + o + r0), make_uint4(q1[0], q1[1], q1[2], q1[3]));
                if (NP >= 3) __stcs(reinterpret_cast<uint4 *>(P2 + o + r0), make_uint4(q2[0], q2[1], q2[2], q2[3]));
            } else {
                for (int64_t r = r0; r < rows && r < r0 + 8; ++r) {
                    Split3 s = split3(x[r]);
                    P0[o + r] = (uint16_t)s.b0;
                    if (NP >= 2) P1[o + r] = (uint16_t)s.b1;
                    if (NP >= 3) P2[o + r] = (uint16_t)s.b2;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------
// transposed: 64 x 64 tiles through shared memory.  Reads are coalesced along the
// rows of the column-major source, writes along its columns (the output's
// contiguous dimension).
// ---------------------------------------------------------------------------------
constexpr int TT = 64;
template <int NP>
__global__ void __launch_bounds__(256) split_trans_kernel(int64_t rows, int64_t cols, const float *__restrict__ X,
                                                          int64_t ldx, uint16_t *__restrict__ P0,
                                                          uint16_t *__restrict__ P1, uint16_t *__restrict__ P2,
                                                          int64_t ldp) {
    __shared__ uint16_t s[NP][TT][TT + 2];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8 threads
    const int64_t tiles_r = (rows + TT - 1) / TT, tiles_c = (cols + TT - 1) / TT;
    uint16_t *P[3] = {P0, P1, P2};
    for (int64_t t = blockIdx.x; t < tiles_r * tiles_c; t += gridDim.x) {
        const int64_t r0 = (t % tiles_r) * TT, c0 = (t / tiles_r) * TT;
        // load + split: thread covers rows r0+2tx, r0+2tx+1 of columns c0+ty+8i
#pragma unroll
        for (int i = 0; i < TT / 8; ++i) {
            const int cl = ty + 8 * i;
            const int64_t c = c0 + cl;
            const int64_t r = r0 + 2 * tx;
            float v0 = 0.f, v1 = 0.f;
            if (c < cols) {
                const float *x = X + c * ldx + r;
                if (r < rows) v0 = x[0];
                if (r + 1 < rows) v1 = x[1];
            }
            Split3 a = split3(v0), b = split3(v1);
            s[0][2 * tx][cl] = (uint16_t)a.b0;
            s[0][2 * tx + 1][cl] = (uint16_t)b.b0;
            if constexpr (NP >= 2) { s[1][2 * tx][cl] = (uint16_t)a.b1; s[1][2 * tx + 1][cl] = (uint16_t)b.b1; }
            if constexpr (NP >= 3) { s[2][2 * tx][cl] = (uint16_t)a.b2; s[2][2 * tx + 1][cl] = (uint16_t)b.b2; }
        }
        __syncthreads();
        // store: output row (source row) r, contiguous source columns c0 + 2tx, +1
#pragma unroll
        for (int i = 0; i < TT / 8; ++i) {
            const int rl = ty + 8 * i;
            const int64_t r = r0 + rl;
            const int64_t c = c0 + 2 * tx;
            if (r >= rows) continue;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                uint16_t *dst = P[q] + r * ldp + c;
                const uint16_t lo = s[q][rl][2 * tx], hi = s[q][rl][2 * tx + 1];
                if (c + 1 < cols && ((reinterpret_cast<uintptr_t>(dst) & 3u) == 0)) {
                    *reinterpret_cast<uint32_t *>(dst) = (uint32_t)lo | ((uint32_t)hi << 16);
                } else {
                    if (c < cols) dst[0] = lo;
                    if (c + 1 < cols) dst[1] = hi;
                }
            }
        }
        __syncthreads();
    }
}

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

int launch_split(int64_t rows, int64_t cols, const float *X, int64_t ldx, uint16_t *P0, uint16_t *P1, uint16_t *P2,
                 int64_t ldp, bool transpose, cudaStream_t st) {
    if (rows == 0 || cols == 0) return BF16X_SUCCESS;
    const int np = P2 ? 3 : (P1 ? 2 : 1);
    if (!transpose) {
        const bool vec = ((reinterpret_cast<uintptr_t>(X) & 15u) == 0) && ldx % 4 == 0 &&
                         ((reinterpret_cast<uintptr_t>(P0) & 15u) == 0) &&
                         (!P1 || (reinterpret_cast<uintptr_t>(P1) & 15u) == 0) &&
                         (!P2 || (reinterpret_cast<uintptr_t>(P2) & 15u) == 0) && ldp % 8 == 0;
        const int64_t nchunk = (rows + 7) / 8;
        int64_t gx = (nchunk + 255) / 256;
        int64_t gy = cols;
        // keep roughly 16 waves of 256-thread blocks in flight
        const int64_t target = (int64_t)sm_count() * 8 * 16;
        if (gx > target) gx = target;
        if (gx * gy > target) gy = (target + gx - 1) / gx;
        if (gy > 65535) gy = 65535;
        if (gy < 1) gy = 1;
        dim3 grid((unsigned)gx, (unsigned)gy);
        if (np == 1) split_same_kernel<1><<<grid, 256, 0, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp, vec);
        else if (np == 2) split_same_kernel<2><<<grid, 256, 0, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp, vec);
        else split_same_kernel<3><<<grid, 256, 0, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp, vec);
    } else {
        const int64_t tiles = ((rows + TT - 1) / TT) * ((cols + TT - 1) / TT);
        int64_t g = tiles;
        const int64_t cap = (int64_t)sm_count() * 8;
        if (g > cap) g = cap;
        if (np == 1) split_trans_kernel<1><<<(unsigned)g, 256, 0, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp);
        else if (np == 2) split_trans_kernel<2><<<(unsigned)g, 256, 0, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp);
        else split_trans_kernel<3><<<(unsigned)g, 256, 0, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp);
    }
    count_launch();
    return check_launch("split");
}

}  // namespace bf16x

using namespace bf16x;

static int split_args(int64_t rows, int64_t cols, int64_t ldx, const uint16_t *P0, const uint16_t *P1,
                      const uint16_t *P2, int64_t ldp, int64_t ldp_min) {
    if (rows < 0) return -1;
    if (cols < 0) return -2;
    if (ldx < (rows > 1 ? rows : 1)) return -4;
    if (!P0) return -5;
    if (P2 && !P1) return -7;
    if (ldp < (ldp_min > 1 ? ldp_min : 1)) return -8;
    return 0;
}

extern "C" int bf16x_split(int64_t rows, int64_t cols, const float *X, int64_t ldx, uint16_t *P0, uint16_t *P1,
                           uint16_t *P2, int64_t ldp, bf16x_stream_t stream) {
    int a = split_args(rows, cols, ldx, P0, P1, P2, ldp, rows);
    if (a) return a;
    int ok = arch_ok();
    if (ok) return ok;
    return launch_split(rows, cols, X, ldx, P0, P1, P2, ldp, false, (cudaStream_t)stream);
}

extern "C" int bf16x_split_t(int64_t rows, int64_t cols, const float *X, int64_t ldx, uint16_t *P0, uint16_t *P1,
                             uint16_t *P2, int64_t ldp, bf16x_stream_t stream) {
    int a = split_args(rows, cols, ldx, P0, P1, P2, ldp, cols);
    if (a) return a;
    int ok = arch_ok();
    if (ok) return ok;
    return launch_split(rows, cols, X, ldx, P0, P1, P2, ldp, true, (cudaStream_t)stream);
}
