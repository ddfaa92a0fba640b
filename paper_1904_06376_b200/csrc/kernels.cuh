// kernels.cuh -- internal (non-ABI) launch entry points shared by the .cu files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bf16x {

// internal gemm_core flag (not in the public header): red.global.add epilogue for C += +-Z
// (alpha = +-1, beta = 1), see gemm_impl.cuh
constexpr unsigned kFlagRedAdd = 1u << 30;

int launch_split(int64_t rows, int64_t cols, const float *X, int64_t ldx, uint16_t *P0, uint16_t *P1,
                 uint16_t *P2, int64_t ldp, bool transpose, cudaStream_t st, bool scaled = false);

int launch_split_ab(int m, int n, int k, const float *A, int64_t lda, uint16_t *Ap, int64_t ldap, int64_t a_plane,
                    const float *B, int64_t ldb, uint16_t *Bp, int64_t ldbp, int64_t b_plane, int npa, int npb,
                    cudaStream_t st, bool scaled = false, bool a_trans = true);

struct GemmPlan {
    int m, n, k;
    float alpha, beta;
    float *C;
    int ldc;
    int variant;
    unsigned flags;
    const uint16_t *Ap;  // A pieces: plane q at Ap + q*a_plane, element (i,l) at i*ldap + l (K-major)
                         // or, with a_mn, at i + l*ldap (MN-major: A's own layout)
    int a_mn;
    int64_t ldap, a_plane;
    const uint16_t *Bp;  // K-major B pieces: plane q at Bp + q*b_plane, element (j,l) at j*ldbp + l
    int64_t ldbp, b_plane;
    float *acc;          // carry (ld = ldc) or nullptr
    int cta_group;       // 1 or 2 (0 = choose)
    int max_ctas;        // 0 = all SMs
    int tile_n;          // reserved (256)
    int stages_per_interval;  // 0 = choose; 1 or 2 stages of 32 k per promotion interval
    int stream_k;        // 0 = data-parallel only, else hybrid stream-K for the last waves
    int multicast;       // 2 = two CTA pairs per cluster share B tiles (TMA multicast), else 1
    int split_acc;       // 1 = separate TMEM accumulators for bin 0 and bins >= 1 (tile N 128)
    int scaled;          // 1 = N2 scaled pieces (R29): band transitions scale the accumulator by 2^-8
    int fp64;            // 1 = FP64 collection of the bins ("d" variants, R30; implies split_acc)
    int group_m;         // tile raster group height in m-tiles (0 = default 8)
    int fused_a;         // 1 = A converted inside the GEMM from FP32 tiles (Af), B pre-split (Bp)
    // fused A: the FP32 A operand, converted to pieces inside the GEMM (B is pre-split)
    const float *Af, *Bf;   // A (m x k, lda), B (k x n, ldb), column-major, 16-byte aligned
    int64_t lda, ldb;
};

int launch_gemm_pieces(const GemmPlan &p, cudaStream_t st);
// Whether the fused-A kernel can run this plan (2-CTA pairs, tile N 256, no multicast / split
// accumulators / FP64 collection / scaled pieces, A 16-byte aligned with lda % 4 == 0).
bool fused_a_ok(const GemmPlan &p);
// Whether the library schedule promotes every MMA on its own (short k; gemm_impl.cuh PM).
bool use_pm(const GemmPlan &p);
int launch_scale(int m, int n, float beta, float *C, int ldc, cudaStream_t st);
int pieces_a(int variant);   // BF16 pieces of A / B for a variant (x5: 2 / 3)
int pieces_b(int variant);
int num_sms();
void lu_release_cache();   // lu.cu: the LU / solve workspace kept between calls
int default_cta_group();

}  // namespace bf16x
