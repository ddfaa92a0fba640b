// split.cu -- K1: the FP32 -> {b0, b1, b2} BF16 split of P:180-184 (section II-A) as an
// HBM-bound pre-pass.  Two layouts:
//   split_same  : pieces keep the source's column-major layout (bf16x_split; also the
//                 K-major B operand of the GEMM, since B is k x n column-major)
//   split_trans : pieces are written transposed (bf16x_split_t; the K-major A operand)
// Algorithmic traffic: 4 B read + 2p B written per element (p = pieces kept).
//
// Arithmetic: pairs of values whose magnitude is below the b0-overflow band (|x| <
// 0x7F7F8000, so finite) take the hardware path -- cvt.rn.bf16x2.f32 is IEEE
// round-to-nearest-even on two values at once and cannot overflow there; the FP32
// residual subtractions are exact.  Anything else (NaN, Inf, the overflow band) takes the
// integer path of common.cuh::split3 (saturation R3, NaN -> 0x7FC0 R4).  Both paths are
// bit-exact against the oracle over all 2^32 patterns (tests/test_gpu_split.py).
#include "common.cuh"
#include "kernels.cuh"

namespace bf16x {

// ---------------------------------------------------------------------------------
// same layout: each thread splits 8 consecutive rows of one column per iteration;
// 16-byte vector loads/stores when the whole matrix is 16-byte aligned (vec != 0).
// ---------------------------------------------------------------------------------
// U chunks per thread per loop trip: all U chunks' loads are issued before the first split, so each
// thread keeps U x 32 bytes in flight.  U = 4 in the grid-stride launch of both operands in their
// own layout (8 blocks per SM: 4096^2 x 2 5422 -> 5818 GB/s, 8192^2 5502 -> 6042; r09
// tools/split_bw.py); U = 1 where the grid covers the matrix (the standalone split: U = 4 costs
// registers and residency there, 5779 -> 4516 GB/s at 4096^2) and beside the transposed A half.
template <int NP, bool SC, int U = 1>
__device__ __forceinline__ void split_same_body(int64_t rows, int64_t cols, const float *__restrict__ X, int64_t ldx,
                                                uint16_t *__restrict__ P0, uint16_t *__restrict__ P1,
                                                uint16_t *__restrict__ P2, int64_t ldp, int vec, int64_t vblock,
                                                int64_t vgrid) {
    const int64_t nchunk = (rows + 7) / 8;
    const int64_t total = nchunk * cols;
    const int64_t stride = vgrid * blockDim.x;
    for (int64_t t0 = vblock * blockDim.x + threadIdx.x; t0 < total; t0 += U * stride) {
        float4 u[U], w[U];
        bool full[U];
        int64_t xo[U], o[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int64_t t = t0 + q * stride;
            const int64_t col = t / nchunk, r0 = (t - col * nchunk) * 8;
            xo[q] = col * ldx + r0;
            o[q] = col * ldp + r0;
            full[q] = t < total && vec && r0 + 8 <= rows;
            if (full[q]) {
                u[q] = __ldcs(reinterpret_cast<const float4 *>(X + xo[q]));
                w[q] = __ldcs(reinterpret_cast<const float4 *>(X + xo[q] + 4));
            }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int64_t t = t0 + q * stride;
            if (t >= total) break;
            if (full[q]) {
                uint32_t v[4][3];
                split_pair<NP, SC>(u[q].x, u[q].y, v[0]);
                split_pair<NP, SC>(u[q].z, u[q].w, v[1]);
                split_pair<NP, SC>(w[q].x, w[q].y, v[2]);
                split_pair<NP, SC>(w[q].z, w[q].w, v[3]);
                __stcs(reinterpret_cast<uint4 *>(P0 + o[q]), make_uint4(v[0][0], v[1][0], v[2][0], v[3][0]));
                if constexpr (NP >= 2)
                    __stcs(reinterpret_cast<uint4 *>(P1 + o[q]), make_uint4(v[0][1], v[1][1], v[2][1], v[3][1]));
                if constexpr (NP >= 3)
                    __stcs(reinterpret_cast<uint4 *>(P2 + o[q]), make_uint4(v[0][2], v[1][2], v[2][2], v[3][2]));
            } else {
                const int64_t col = t / nchunk, r0 = (t - col * nchunk) * 8;
                const float *x = X + col * ldx;
                for (int64_t r = r0; r < rows && r < r0 + 8; ++r) {
                    Split3 sp = split3_t<SC>(x[r]);
                    P0[o[q] - r0 + r] = (uint16_t)sp.b0;
                    if constexpr (NP >= 2) P1[o[q] - r0 + r] = (uint16_t)sp.b1;
                    if constexpr (NP >= 3) P2[o[q] - r0 + r] = (uint16_t)sp.b2;
                }
            }
        }
    }
}

template <int NP, bool SC>
__global__ void __launch_bounds__(256) split_same_kernel(int64_t rows, int64_t cols, const float *__restrict__ X,
                                                         int64_t ldx, uint16_t *__restrict__ P0,
                                                         uint16_t *__restrict__ P1, uint16_t *__restrict__ P2,
                                                         int64_t ldp, int vec) {
    asm volatile("griddepcontrol.launch_dependents;");
    split_same_body<NP, SC>(rows, cols, X, ldx, P0, P1, P2, ldp, vec, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------------
// transposed: 64 (source rows) x TC (source columns) tiles.  Warp w loads source columns
// [w TC/8, (w+1) TC/8) of the tile: lane = (row quad mq: 0..15) + 16 * (column pair half);
// every lane splits pairs of adjacent columns (= adjacent output elements) and stores packed
// words to shared memory [piece][row][column pair] (row stride TC/2 + 1 words), then each
// warp writes whole output rows: TC/2 words = TC bf16 per row and piece, i.e. contiguous runs
// of 2 TC bytes in the K-major output (TC = 128: 256-byte runs, like the 256-byte column
// runs read from the source).  Shared memory is dynamic: NP * 64 * (TC/2 + 1) words.
// ---------------------------------------------------------------------------------
constexpr int TT = 64;
constexpr int kTransTC = 128;   // standalone transposed split (measured r08: 4066 -> 4278 GB/s at 4096^2)
constexpr int kTransTCab = 64;  // in split_ab, whose B blocks share the launch's smem (occupancy)
template <int TC>
constexpr int trans_smem_words(int np) { return np * TT * (TC / 2 + 1); }
template <int NP, bool SC, int TC = kTransTC>
__device__ __forceinline__ void split_trans_body(int64_t rows, int64_t cols, const float *__restrict__ X, int64_t ldx,
                                                 uint16_t *__restrict__ P0, uint16_t *__restrict__ P1,
                                                 uint16_t *__restrict__ P2, int64_t ldp, int vec, int64_t vblock,
                                                 int64_t vgrid, uint32_t *__restrict__ sm) {
    constexpr int TW = TC / 2 + 1;   // words per smem row (+1 pad)
    constexpr int J = TC / 32;       // column pairs per lane
    auto s = [&](int p, int r, int w) -> uint32_t & { return sm[(p * TT + r) * TW + w]; };
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int mq = lane & 15, half = lane >> 4;
    const int64_t tiles_r = (rows + TT - 1) / TT, tiles_c = (cols + TC - 1) / TC;
    uint16_t *P[3] = {P0, P1, P2};
    const bool out_words = (ldp % 2 == 0) && ((reinterpret_cast<uintptr_t>(P0) & 3u) == 0) &&
                           (!P1 || (reinterpret_cast<uintptr_t>(P1) & 3u) == 0) &&
                           (!P2 || (reinterpret_cast<uintptr_t>(P2) & 3u) == 0);
    for (int64_t t = vblock; t < tiles_r * tiles_c; t += vgrid) {
        const int64_t r0 = (t % tiles_r) * TT, c0 = (t / tiles_r) * TC;
        const bool full = (r0 + TT <= rows) && (c0 + TC <= cols) && vec;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int cp = wid * (2 * J) + half * J + j;  // column pair within the tile (0..TC/2-1)
            const int64_t c = c0 + 2 * cp;
            const int64_t r = r0 + 4 * mq;
            float a[4], b[4];
            if (full) {
                const float4 fa = __ldcs(reinterpret_cast<const float4 *>(X + c * ldx + r));
                const float4 fb = __ldcs(reinterpret_cast<const float4 *>(X + (c + 1) * ldx + r));
                a[0] = fa.x; a[1] = fa.y; a[2] = fa.z; a[3] = fa.w;
                b[0] = fb.x; b[1] = fb.y; b[2] = fb.z; b[3] = fb.w;
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    a[i] = (c < cols && r + i < rows) ? X[c * ldx + r + i] : 0.f;
                    b[i] = (c + 1 < cols && r + i < rows) ? X[(c + 1) * ldx + r + i] : 0.f;
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                uint32_t q[3];
                split_pair<NP, SC>(a[i], b[i], q);     // lo = column c, hi = column c+1
#pragma unroll
                for (int p = 0; p < NP; ++p) s(p, 4 * mq + i, cp) = q[p];
            }
        }
        __syncthreads();
        // output: row rl of the tile, word w = lane + 32 u = source columns c0 + 2 w, +1
#pragma unroll
        for (int i = 0; i < TT / 8; ++i) {
            const int rl = wid + 8 * i;
            const int64_t r = r0 + rl;
            if (r >= rows) continue;
#pragma unroll
            for (int u = 0; u < TC / 64; ++u)
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const int wi = lane + 32 * u;
                const int64_t c = c0 + 2 * wi;
                const uint32_t wv = s(p, rl, wi);
                uint16_t *dst = P[p] + r * ldp + c;
                if (out_words && c + 1 < cols) {
                    __stcs(reinterpret_cast<unsigned int *>(dst), wv);
                } else {
                    if (c < cols) dst[0] = (uint16_t)(wv & 0xFFFFu);
                    if (c + 1 < cols) dst[1] = (uint16_t)(wv >> 16);
                }
            }
        }
        __syncthreads();
    }
}

template <int NP, bool SC>
__global__ void __launch_bounds__(256) split_trans_kernel(int64_t rows, int64_t cols, const float *__restrict__ X,
                                                          int64_t ldx, uint16_t *__restrict__ P0,
                                                          uint16_t *__restrict__ P1, uint16_t *__restrict__ P2,
                                                          int64_t ldp, int vec) {
    extern __shared__ uint32_t s_trans[];
    asm volatile("griddepcontrol.launch_dependents;");
    split_trans_body<NP, SC>(rows, cols, X, ldx, P0, P1, P2, ldp, vec, blockIdx.x, gridDim.x, s_trans);
}

// Both GEMM operands in one launch: blocks [0, gA) split A transposed (K-major pieces),
// blocks [gA, grid) split B in place.  One ramp-up/tail instead of two.
struct SplitArgs {
    int64_t rows, cols, ldx, ldp;
    const float *X;
    uint16_t *P0, *P1, *P2;
    int vec;
};
// TA = false: A is split in its own (column-major = MN-major) layout too, like B.
template <int NPA, int NPB, bool SC, bool TA = true>
__global__ void __launch_bounds__(256) split_ab_kernel(SplitArgs a, SplitArgs b, int gA) {
    extern __shared__ uint32_t s_trans[];
    asm volatile("griddepcontrol.launch_dependents;");   // let the GEMM's prologue start early
    if ((int)blockIdx.x < gA) {
        if constexpr (TA)
            split_trans_body<NPA, SC, kTransTCab>(a.rows, a.cols, a.X, a.ldx, a.P0, a.P1, a.P2, a.ldp, a.vec, blockIdx.x,
                                                  gA, s_trans);
        else
            split_same_body<NPA, SC, 4>(a.rows, a.cols, a.X, a.ldx, a.P0, a.P1, a.P2, a.ldp, a.vec, blockIdx.x, gA);
    } else
        split_same_body<NPB, SC, TA ? 1 : 4>(b.rows, b.cols, b.X, b.ldx, b.P0, b.P1, b.P2, b.ldp, b.vec, blockIdx.x - gA,
                             gridDim.x - gA);
}

// dynamic shared memory of the transposed tiles (> 48 KB for 3 pieces: opt-in once per kernel)
template <int TC, typename K>
static size_t trans_smem(K kern, int np) {
    const size_t bytes = (size_t)trans_smem_words<TC>(np) * 4;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    return bytes;
}

template <bool SC>
static void split_ab_launch(const SplitArgs &a, const SplitArgs &b, int gA, unsigned grid, int npa, int npb,
                            cudaStream_t st, bool ta) {
    if (!ta) {   // both operands in their own layout: no shared memory
        if (npa == 1 && npb == 1) split_ab_kernel<1, 1, SC, false><<<grid, 256, 0, st>>>(a, b, gA);
        else if (npa == 2 && npb == 2) split_ab_kernel<2, 2, SC, false><<<grid, 256, 0, st>>>(a, b, gA);
        else if (npa == 2 && npb == 3) split_ab_kernel<2, 3, SC, false><<<grid, 256, 0, st>>>(a, b, gA);
        else split_ab_kernel<3, 3, SC, false><<<grid, 256, 0, st>>>(a, b, gA);
        return;
    }
    if (npa == 1 && npb == 1) {
        static size_t sm = trans_smem<kTransTCab>(split_ab_kernel<1, 1, SC>, 1);
        split_ab_kernel<1, 1, SC><<<grid, 256, sm, st>>>(a, b, gA);
    } else if (npa == 2 && npb == 2) {
        static size_t sm = trans_smem<kTransTCab>(split_ab_kernel<2, 2, SC>, 2);
        split_ab_kernel<2, 2, SC><<<grid, 256, sm, st>>>(a, b, gA);
    } else if (npa == 2 && npb == 3) {
        static size_t sm = trans_smem<kTransTCab>(split_ab_kernel<2, 3, SC>, 2);
        split_ab_kernel<2, 3, SC><<<grid, 256, sm, st>>>(a, b, gA);
    } else {
        static size_t sm = trans_smem<kTransTCab>(split_ab_kernel<3, 3, SC>, 3);
        split_ab_kernel<3, 3, SC><<<grid, 256, sm, st>>>(a, b, gA);
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

template <bool SC>
static void split_launch(int64_t rows, int64_t cols, const float *X, int64_t ldx, uint16_t *P0, uint16_t *P1,
                         uint16_t *P2, int64_t ldp, bool transpose, cudaStream_t st) {
    const int np = P2 ? 3 : (P1 ? 2 : 1);
    if (!transpose) {
        const bool vec = ((reinterpret_cast<uintptr_t>(X) & 15u) == 0) && ldx % 4 == 0 &&
                         ((reinterpret_cast<uintptr_t>(P0) & 15u) == 0) &&
                         (!P1 || (reinterpret_cast<uintptr_t>(P1) & 15u) == 0) &&
                         (!P2 || (reinterpret_cast<uintptr_t>(P2) & 15u) == 0) && ldp % 8 == 0;
        const int64_t total = ((rows + 7) / 8) * cols;
        int64_t g = (total + 255) / 256;
        const int64_t cap = (int64_t)sm_count() * 8 * 8;
        if (g > cap) g = cap;
        if (np == 1) split_same_kernel<1, SC><<<(unsigned)g, 256, 0, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp, vec);
        else if (np == 2) split_same_kernel<2, SC><<<(unsigned)g, 256, 0, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp, vec);
        else split_same_kernel<3, SC><<<(unsigned)g, 256, 0, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp, vec);
    } else {
        const bool vec = ((reinterpret_cast<uintptr_t>(X) & 15u) == 0) && ldx % 4 == 0;
        const int64_t tiles = ((rows + TT - 1) / TT) * ((cols + kTransTC - 1) / kTransTC);
        int64_t g = tiles;
        const int64_t cap = (int64_t)sm_count() * 8;
        if (g > cap) g = cap;
        if (np == 1) {
            static size_t sm = trans_smem<kTransTC>(split_trans_kernel<1, SC>, 1);
            split_trans_kernel<1, SC><<<(unsigned)g, 256, sm, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp, vec);
        } else if (np == 2) {
            static size_t sm = trans_smem<kTransTC>(split_trans_kernel<2, SC>, 2);
            split_trans_kernel<2, SC><<<(unsigned)g, 256, sm, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp, vec);
        } else {
            static size_t sm = trans_smem<kTransTC>(split_trans_kernel<3, SC>, 3);
            split_trans_kernel<3, SC><<<(unsigned)g, 256, sm, st>>>(rows, cols, X, ldx, P0, P1, P2, ldp, vec);
        }
    }
}

int launch_split(int64_t rows, int64_t cols, const float *X, int64_t ldx, uint16_t *P0, uint16_t *P1, uint16_t *P2,
                 int64_t ldp, bool transpose, cudaStream_t st, bool scaled) {
    if (rows == 0 || cols == 0) return BF16X_SUCCESS;
    if (scaled) split_launch<true>(rows, cols, X, ldx, P0, P1, P2, ldp, transpose, st);
    else split_launch<false>(rows, cols, X, ldx, P0, P1, P2, ldp, transpose, st);
    count_launch();
    return check_launch("split");
}

int launch_split_ab(int m, int n, int k, const float *A, int64_t lda, uint16_t *Ap, int64_t ldap, int64_t a_plane,
                    const float *B, int64_t ldb, uint16_t *Bp, int64_t ldbp, int64_t b_plane, int npa, int npb,
                    cudaStream_t st, bool scaled, bool a_trans) {
    if (m == 0 || n == 0 || k == 0) return BF16X_SUCCESS;
    SplitArgs a{m, k, lda, ldap, A, Ap, npa > 1 ? Ap + a_plane : nullptr, npa > 2 ? Ap + 2 * a_plane : nullptr, 0};
    SplitArgs b{k, n, ldb, ldbp, B, Bp, npb > 1 ? Bp + b_plane : nullptr, npb > 2 ? Bp + 2 * b_plane : nullptr, 0};
    a.vec = ((reinterpret_cast<uintptr_t>(A) & 15u) == 0) && lda % 4 == 0;
    if (!a_trans)   // same-layout vector stores need the pieces 16-byte aligned too
        a.vec = a.vec && ((reinterpret_cast<uintptr_t>(Ap) & 15u) == 0) && ldap % 8 == 0 && a_plane % 8 == 0;
    b.vec = ((reinterpret_cast<uintptr_t>(B) & 15u) == 0) && ldb % 4 == 0 &&
            ((reinterpret_cast<uintptr_t>(Bp) & 15u) == 0) && ldbp % 8 == 0 && b_plane % 8 == 0;
    const int64_t grid = (int64_t)sm_count() * 8;
    const double wa = (double)m * k, wb = (double)k * n;
    int gA = (int)(grid * wa / (wa + wb));
    gA = gA < 1 ? 1 : (gA > grid - 1 ? (int)grid - 1 : gA);
    if (scaled) split_ab_launch<true>(a, b, gA, (unsigned)grid, npa, npb, st, a_trans);
    else split_ab_launch<false>(a, b, gA, (unsigned)grid, npa, npb, st, a_trans);
    count_launch();
    return check_launch("split_ab");
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
    return launch_split(rows, cols, X, ldx, P0, P1, P2, ldp, false, (cudaStream_t)stream, false);
}

extern "C" int bf16x_split_operands(int m, int n, int k, const float *A, int64_t lda, const float *B, int64_t ldb,
                                    int pieces, uint16_t *Ap, int64_t ldap, int64_t a_plane, uint16_t *Bp,
                                    int64_t ldbp, int64_t b_plane, bf16x_stream_t stream) {
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (k < 0) return -3;
    if (lda < (m > 1 ? m : 1)) return -5;
    if (ldb < (k > 1 ? k : 1)) return -7;
    if (pieces < 1 || pieces > 3) return -8;
    if (!Ap || ldap < (k > 1 ? k : 1) || a_plane < ldap * (int64_t)m) return -9;
    if (!Bp || ldbp < (k > 1 ? k : 1) || b_plane < ldbp * (int64_t)n) return -12;
    int ok = arch_ok();
    if (ok) return ok;
    return launch_split_ab(m, n, k, A, lda, Ap, ldap, a_plane, B, ldb, Bp, ldbp, b_plane, pieces, pieces,
                           (cudaStream_t)stream, false, true);
}

// Both operands, options: BF16X_A_PIECES_MN (A's pieces in A's own layout: element (i,l) of piece q at
// Ap[q*a_plane + i + l*ldap], ldap >= m -- what bf16x_gemm_ex takes with the same flag),
// BF16X_SCALED_PIECES (R29).
extern "C" int bf16x_split_operands_ex(int m, int n, int k, const float *A, int64_t lda, const float *B, int64_t ldb,
                                       int pieces, uint16_t *Ap, int64_t ldap, int64_t a_plane, uint16_t *Bp,
                                       int64_t ldbp, int64_t b_plane, unsigned flags, bf16x_stream_t stream) {
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (k < 0) return -3;
    if (lda < (m > 1 ? m : 1)) return -5;
    if (ldb < (k > 1 ? k : 1)) return -7;
    if (pieces < 1 || pieces > 3) return -8;
    if (flags & ~(BF16X_A_PIECES_MN | BF16X_SCALED_PIECES)) return -13;
    const bool mn = (flags & BF16X_A_PIECES_MN) != 0;
    if (!Ap || (mn ? (ldap < (m > 1 ? m : 1) || a_plane < ldap * (int64_t)k)
                   : (ldap < (k > 1 ? k : 1) || a_plane < ldap * (int64_t)m)))
        return -9;
    if (!Bp || ldbp < (k > 1 ? k : 1) || b_plane < ldbp * (int64_t)n) return -12;
    int ok = arch_ok();
    if (ok) return ok;
    return launch_split_ab(m, n, k, A, lda, Ap, ldap, a_plane, B, ldb, Bp, ldbp, b_plane, pieces, pieces,
                           (cudaStream_t)stream, (flags & BF16X_SCALED_PIECES) != 0, !mn);
}

extern "C" int bf16x_split_t(int64_t rows, int64_t cols, const float *X, int64_t ldx, uint16_t *P0, uint16_t *P1,
                             uint16_t *P2, int64_t ldp, bf16x_stream_t stream) {
    int a = split_args(rows, cols, ldx, P0, P1, P2, ldp, cols);
    if (a) return a;
    int ok = arch_ok();
    if (ok) return ok;
    return launch_split(rows, cols, X, ldx, P0, P1, P2, ldp, true, (cudaStream_t)stream, false);
}

// N2 scaled pieces (R29), either layout: flags BF16X_SCALED_PIECES (required, documents the
// piece format) | BF16X_SPLIT_TRANSPOSED (K-major output as bf16x_split_t).
extern "C" int bf16x_split_ex(int64_t rows, int64_t cols, const float *X, int64_t ldx, uint16_t *P0, uint16_t *P1,
                              uint16_t *P2, int64_t ldp, unsigned flags, bf16x_stream_t stream) {
    const bool tr = (flags & BF16X_SPLIT_TRANSPOSED) != 0;
    int a = split_args(rows, cols, ldx, P0, P1, P2, ldp, tr ? cols : rows);
    if (a) return a;
    if (flags & ~(BF16X_SCALED_PIECES | BF16X_SPLIT_TRANSPOSED)) return -9;
    int ok = arch_ok();
    if (ok) return ok;
    return launch_split(rows, cols, X, ldx, P0, P1, P2, ldp, tr, (cudaStream_t)stream,
                        (flags & BF16X_SCALED_PIECES) != 0);
}
