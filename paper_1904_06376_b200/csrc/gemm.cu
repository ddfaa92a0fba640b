// gemm.cu -- K2: the multi-product BF16-split GEMM on tcgen05 tensor cores (sm_100a).
//
// Method: the FP32 product A*B is the sum of BF16 x BF16 partial products
// Z^(i,j) = A_i * B_j accumulated in FP32 (section II-D), grouped into bins of
// equal i+j and added smallest bin first ("the terms should be added in
// the reverse order, so that the smallest terms come first").  Variants: 3 products
// {00,01,10}, 6 products = Z_2, 9 products (R9).
//
// B200 mapping:
//   * persistent grid, one CTA per SM (cta_group::1, 128 x 256 tile) or one CTA pair per
//     two SMs (cta_group::2, 256 x 256 tile, B halves split across the pair);
//   * warp 0: TMA producer.  Per stage (BK = 32 values of k, all p pieces): B by one 3D TMA box,
//     smem [piece][rows][32 bf16] with the 64-byte swizzle (K-major); A either the same way
//     (K-major pieces from bf16x_split_t) or, as bf16x_gemm splits it since r09, in A's own
//     column-major layout by two boxes [piece][k 32][m 64] with the 128-byte swizzle, which the
//     MMA reads MN-major (instruction descriptor a_major = MN);
//   * warp 1: MMA issuer (one thread).  Per stage (= one promotion interval of 32 k) it
//     issues the variant's products band by band, smallest bin first, both K=16 halves
//     of a band before the next band, into one TMEM accumulator whose first MMA
//     overwrites it (enable-input-d = 0);
//   * warps 4..11: promotion + epilogue.  After each interval they read the 128 x 256 FP32
//     partial from TMEM (tcgen05.ld) and add it with FP32 round-to-nearest into a
//     register accumulator G (the B200 form of the paper's FP32-accumulated bins); TMEM
//     is double buffered so the tensor core fills one buffer while the other drains.
//     After the last interval: C = fmaf(alpha, G, beta*C) (beta == 0: C is not read).
#include "gemm_impl.cuh"

namespace bf16x {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(f);
    });
    return fn;
}

// 3D map over p K-major piece planes: dims (k, rows, p), box (BK, box_rows, p).
int make_piece_map(CUtensorMap *map, const uint16_t *base, int k, int rows, int64_t ld, int64_t plane,
                          int p, int box_rows, int box_p) {
    if (box_p <= 0) box_p = p;
    EncodeTiledFn enc = encode_fn();
    if (!enc) return BF16X_ERR_CUDA;
    cuuint64_t dims[3] = {(cuuint64_t)k, (cuuint64_t)rows, (cuuint64_t)p};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)plane * 2};
    cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, (cuuint32_t)box_p};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? BF16X_SUCCESS : BF16X_ERR_CUDA;
}

int make_piece_map_mn(CUtensorMap *map, const uint16_t *base, int m, int k, int64_t ld, int64_t plane, int p) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return BF16X_ERR_CUDA;
    cuuint64_t dims[3] = {(cuuint64_t)m, (cuuint64_t)k, (cuuint64_t)p};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)plane * 2};
    cuuint32_t box[3] = {64u, (cuuint32_t)kBK, (cuuint32_t)p};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? BF16X_SUCCESS : BF16X_ERR_CUDA;
}

// 2D map over a column-major FP32 matrix: dims (rows [inner], cols), box (box_rows, box_cols);
// out-of-range elements read as zero (they become zero pieces).
int make_f32_map(CUtensorMap *map, const float *base, int rows, int cols, int64_t ld, int box_rows,
                        int box_cols, CUtensorMapSwizzle swz) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return BF16X_ERR_CUDA;
    cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? BF16X_SUCCESS : BF16X_ERR_CUDA;
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

int pieces_a(int variant) { return variant_pieces_a(variant); }
int pieces_b(int variant) { return variant_pieces_b(variant); }
int default_cta_group() { return kDefaultCtaGroup; }


// Promote-every-MMA schedule for short k on small outputs: the library's automatic schedule only
// (no forced promotion interval), no accumulator carry, plain pieces (scaled pieces keep the
// band-scaled accumulator), no split accumulators / FP64 collection.  Largest k: bf16x_pm_max_k
// (default 128); outputs of at most 2^20 elements, where the extra promotions cost a few us
// (measured r08, tools/pm_probe.py: 512^2 x 64 x6 10.6 -> 17.0 us) -- on 4096^2 outputs they
// would cost 2-3.5x (x6, k = 128: 33 -> 97 us), so large outputs keep the 32-k intervals.
static int g_pm_max_k = 128;
bool use_pm(const GemmPlan &pl) {
    return pl.k <= g_pm_max_k && (int64_t)pl.m * pl.n <= (1LL << 20) && pl.stages_per_interval == 0 &&
           !(pl.flags & (BF16X_ACC_IN | BF16X_ACC_OUT)) && !pl.scaled && !pl.fp64 && !pl.split_acc && !pl.fused_a &&
           pl.tile_n != 192;
}

bool fused_a_ok(const GemmPlan &pl) {
    const int cg = pl.cta_group ? pl.cta_group : kDefaultCtaGroup;
    if (cg != 2 || pl.fp64 || pl.split_acc || pl.scaled || pl.k <= 0 || pl.tile_n == 192 || !pl.Af) return false;
    if (use_pm(pl)) return false;    // short k: the promote-every-MMA schedule instead
    if ((reinterpret_cast<uintptr_t>(pl.Af) & 15u) || pl.lda % 4) return false;
    const bool mc2 = pl.multicast >= 2 || (pl.multicast == 0 && (int64_t)pl.m * pl.n >= 12288LL * 12288LL);
    return !mc2;
}

static int dispatch(const GemmPlan &pl, cudaStream_t st, int kind) {
    switch (pl.variant) {
    case 1: return launch_variant_1(pl, st, kind);
    case 3: return launch_variant_3(pl, st, kind);
    case 5: return launch_variant_5(pl, st, kind);
    case 6: return launch_variant_6(pl, st, kind);
    case 7: return launch_variant_7(pl, st, kind);
    case 8: return launch_variant_8(pl, st, kind);
    case 9: return launch_variant_9(pl, st, kind);
    }
    return -12;
}

int launch_gemm_pieces(const GemmPlan &pl, cudaStream_t st) {
    int cg = pl.cta_group;
    if (cg == 0) cg = kDefaultCtaGroup;
    return dispatch(pl, st, cg == 1 ? 1 : 2);
}

// C <- beta*C (quick return of BLAS sgemm when alpha == 0 or k == 0; beta == 0 -> 0).
__global__ void scale_kernel(int m, int n, float beta, float *C, int ldc) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)m * n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % m, j = t / m;
        float *c = C + j * ldc + i;
        *c = (beta == 0.f) ? 0.f : beta * *c;
    }
}

int launch_scale(int m, int n, float beta, float *C, int ldc, cudaStream_t st) {
    if (m == 0 || n == 0) return BF16X_SUCCESS;
    const int64_t total = (int64_t)m * n;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
    scale_kernel<<<blocks, 256, 0, st>>>(m, n, beta, C, ldc);
    count_launch();
    return check_launch("scale");
}

}  // namespace bf16x

// testing hook (not in the public header): lazy stage waits in the MMA issuer (1, default) or
// all of an interval's stages waited for before its first MMA (0)
extern "C" void bf16x_lazy_full(int on) { bf16x::g_lazy_full = on ? 1 : 0; }
// testing hook (not in the public header): red.global.add epilogue for C += +-Z (alpha = +-1,
// beta = 1): -1 where the caller asks for it (the LU's trailing update), 0 never, 1 always
extern "C" void bf16x_red_add(int mode) { bf16x::g_red_add = mode; }
// testing hook (not in the public header): KParams::dbg bits (bit 0: skip beta = 0 C stores)
extern "C" void bf16x_gemm_debug(int bits) { bf16x::g_gemm_debug = bits; }
// testing hook: device buffer of >= 32 * grid uint64 for the dbg bit 1 timeline (tools/gemm_trace.py)
extern "C" void bf16x_gemm_trace(unsigned long long *buf) { bf16x::g_gemm_trace = buf; }
// testing / tuning hook: largest k for the promote-every-MMA schedule (0: never)
extern "C" void bf16x_pm_max_k(int k) { bf16x::g_pm_max_k = k; }
