// gemm_impl.cuh -- K2 kernel template and its launch templates (included by gemm.cu and by the
// per-variant instantiation units gemm_v<V>.cu, which compile in parallel).  See gemm.cu for the
// method and the B200 mapping.
#pragma once
#include <algorithm>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace bf16x {

constexpr int kBM = 128;              // accumulator lanes (rows) per CTA
constexpr int kBK = 32;               // k per stage = promotion interval
constexpr int kUK = 16;               // k per tcgen05.mma kind::f16
constexpr int kRowBytes = kBK * 2;    // 64 B rows -> SWIZZLE_64B
constexpr int kSwizzleAtom = 8 * kRowBytes;  // 8 rows x 64 B: stride between row groups (SBO)
constexpr int kNumEpiWarps = 8;       // 2 per TMEM lane quadrant, BN/2 columns each
constexpr int kThreads = (4 + kNumEpiWarps) * 32;
constexpr int kNumXfWarps = 8;        // fused A: warps 12..19 convert FP32 A tiles to pieces
constexpr int kThreadsFused = kThreads + kNumXfWarps * 32;
constexpr int kF32Tile = kBM * kBK * 4;   // one FP32 operand tile per CTA per stage (16 KB)
// MN-major A (KParams::a_mn): per stage and CTA two TMA boxes (m 64 x k 32 x pieces), smem
// [m half][piece][k 32][m 64] with the 128-byte swizzle: 8-row k groups 1024 B apart (SBO), the two
// 64-row m atoms PA * 4 KB apart (LBO); a K = 16 step starts 2 groups (2 KB) further
constexpr int kMnBox = 64 * kBK * 2;      // one piece of one 64-row half: 4 KB
constexpr int kTmemCols = 512;        // two accumulator buffers at column 0 and 256
constexpr int kTmemBufStride = 256;
constexpr int kGroupM = 8;            // tile raster: 8 m-tiles per group for L2 reuse (default)
constexpr int kDefaultCtaGroup = 2;   // 2-CTA pairs, 64-k promotion interval
constexpr int kSmemBudget = 232448 - 1024;   // 227 KB opt-in maximum
// C epilogue staging (TMA store): per column half (the 4 epilogue warps of TMEM lane quadrants
// 0..3) two buffers of one 128-row x 16-column FP32 box (r09: 128-row boxes instead of one 32-row
// box per warp, x6 short k -4 %; 1-4 buffers measured alike, profiles/r09/shortk_epi_*.txt)
constexpr int kEpiRows = 128, kEpiCols = 16, kEpiNBuf = 2;
constexpr int kEpiBytes = 2 * kEpiNBuf * kEpiRows * kEpiCols * 4;   // 32 KB
inline int g_lazy_full = 1;           // lazy stage waits in the MMA issuer (bf16x_lazy_full hook)
inline int g_gemm_debug = 0;          // KParams::dbg (bf16x_gemm_debug hook; tests / probes only)
inline unsigned long long *g_gemm_trace = nullptr;   // KParams::trace (bf16x_gemm_trace hook)
// Internal flag (not in the public header): C += alpha * Z with alpha = +-1, beta = 1 written as
// red.global.add.f32 -- RN(C + (+-Z)) is exactly fmaf(+-1, Z, C) -- so the epilogue never waits
// for the old C (the LU's trailing update, csrc/lu.cu).  g_red_add: -1 as requested (default),
// 0 never, 1 for every eligible call (bf16x_red_add hook, tests).
inline int g_red_add = -1;            // kFlagRedAdd (kernels.cuh) override: bf16x_red_add hook

// pieces per operand: x1 1; x3 2; x5 A 2, B 3; x6 / x7 / x8 / x9 3
__host__ __device__ constexpr int variant_pieces_a(int v) { return v == 1 ? 1 : ((v == 3 || v == 5) ? 2 : 3); }
__host__ __device__ constexpr int variant_pieces_b(int v) { return v == 1 ? 1 : (v == 3 ? 2 : 3); }

template <int CG, int V, int BN>
struct Cfg {
    static constexpr int PA = variant_pieces_a(V), PB = variant_pieces_b(V);
    static constexpr int TILE_M = kBM * CG;
    static constexpr int BN_LOCAL = BN / CG;          // B rows (output columns) loaded per CTA
    static constexpr int EPI_COLS = BN / 2;           // accumulator columns per epilogue warp
    static constexpr int A_PIECE = kBM * kRowBytes;
    static constexpr int B_PIECE = BN_LOCAL * kRowBytes;
    static constexpr int A_STAGE = PA * A_PIECE;
    static constexpr int B_STAGE = PB * B_PIECE;
    static constexpr int STAGE = A_STAGE + B_STAGE;
    static constexpr int BAR_BYTES = 256;
    // C staging for the TMA epilogue only where the ring keeps >= 4 stages with it (1-CTA x5-x9
    // tiles would drop to 2-3 stages: they keep per-thread C stores)
    static constexpr int STAGES_EPI = (kSmemBudget - BAR_BYTES - 1024 - kEpiBytes) / STAGE;
    static constexpr bool EPI = STAGES_EPI >= 4;
    static constexpr int EPI_BYTES = EPI ? kEpiBytes : 0;
    static constexpr int STAGES_RAW = (kSmemBudget - BAR_BYTES - 1024 - EPI_BYTES) / STAGE;
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
    static constexpr int SMEM = STAGES * STAGE + EPI_BYTES + BAR_BYTES + 1024;
    static_assert(STAGES >= 2, "need at least two pipeline stages");
    static_assert(BN % (16 * CG) == 0 && BN <= 256 && EPI_COLS % 32 == 0, "invalid tile N");
};

// Fused-A configuration (FA: A converted inside the GEMM from FP32 tiles, B pre-split): a ring of
// FSTAGES FP32 A tiles (128 rows x 32 k per CTA, 16 KB) beside the piece ring, 227 KB in all.
#ifndef FA_FST
#define FA_FST 2
#endif
template <int V>
struct CfgFA {
    using Cf = Cfg<2, V, 256>;
    static constexpr int FSTAGES = FA_FST;
    // (no C staging: the fused-A kernel keeps per-thread C stores and its fourth piece stage --
    // with the 32 KB staging it had 3, and bf16x9 lost 28 % at 4096^3 / 8192^3, r08 sweep)
    static constexpr int STAGES_RAW = (232448 - 1280 - FSTAGES * kF32Tile) / Cf::STAGE;
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
    static constexpr int SMEM = STAGES * Cf::STAGE + FSTAGES * kF32Tile + 256 + 1024;
    static_assert(STAGES >= 3, "fused A needs three piece stages");
};

struct KParams {
    int m, n, k;
    float alpha, beta;
    float *C;
    int ldc;
    unsigned flags;
    float *acc;
    int tiles_m, tiles_n, nkb;
    // schedule: tiles [0, dp_tiles) data-parallel (one cluster per tile); tiles
    // [dp_tiles, dp_tiles + sk_tiles) stream-K: their sk_tiles * n_int promotion intervals are
    // split evenly over the clusters; a tile cut in two is finished by the cluster holding its
    // first intervals ("owner"), which adds the other part's raw FP32 accumulator (sk_ws,
    // published with sk_flags = epoch) before the epilogue.
    int dp_tiles, sk_tiles, n_int;
    float *sk_ws;
    unsigned int *sk_flags;
    unsigned int epoch;
    int scaled;            // N2 scaled pieces (R29): scale the accumulator by 2^-8 per bin step
    int group_m;           // tile raster: m-tiles per group
    int lazy_full;         // issuer waits for each stage just before its first MMA (issue_interval)
    int dbg;               // testing hook (bf16x_gemm_debug): bit 0 = skip the C stores of beta = 0 tiles
    int tma_c;             // C stored (beta = 0) / added (red-add) by TMA from the staging buffers
    unsigned long long *trace;   // dbg bit 1: %globaltimer per CTA (tools/gemm_trace.py), 32 slots each
    // (measured, nvcc 12.9: with the parameter block ending at lazy_full ptxas spills 96 bytes
    // in the 2-CTA kernels; with >= 32 more bytes it allocates 168 registers without spills)
    int a_mn;              // A pieces MN-major (A's own column-major layout; 128-byte swizzle)
    int reserved_i;
    int64_t reserved[3];
};

struct Work {
    int tile, i0, i1;      // promotion intervals [i0, i1) of `tile`
    int role;              // 0 complete tile, 1 owner of a split tile, 2 contributor
    int sk_slot;           // stream-K tile index (sk workspace slot)
};

// Identical on every role of a cluster: data-parallel tiles first, then this cluster's
// contiguous range of stream-K intervals.
struct WorkIter {
    int cid, ncl, dp_next, u, u_end;
    __device__ __forceinline__ WorkIter(const KParams &p, int cid_, int ncl_) : cid(cid_), ncl(ncl_), dp_next(cid_) {
        const int64_t U = (int64_t)p.sk_tiles * p.n_int;
        u = (int)(U * cid / ncl);
        u_end = (int)(U * (cid + 1) / ncl);
    }
    __device__ __forceinline__ bool next(const KParams &p, Work &w) {
        if (dp_next < p.dp_tiles) {
            w.tile = dp_next;
            w.i0 = 0;
            w.i1 = p.n_int;
            w.role = 0;
            w.sk_slot = -1;
            dp_next += ncl;
            return true;
        }
        if (u >= u_end) return false;
        const int t = u / p.n_int, j0 = u - t * p.n_int;
        const int j1 = min(p.n_int, j0 + (u_end - u));
        w.tile = p.dp_tiles + t;
        w.i0 = j0;
        w.i1 = j1;
        w.role = (j0 == 0) ? ((j1 == p.n_int) ? 0 : 1) : 2;
        w.sk_slot = t;
        u += j1 - j0;
        return true;
    }
};

__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int group_m, int &tm, int &tn) {
    const int per_group = group_m * tiles_n;
    const int group = tile / per_group;
    const int first_m = group * group_m;
    const int gm = min(group_m, tiles_m - first_m);
    const int r = tile - group * per_group;
    tm = first_m + r % gm;
    tn = r / gm;
}

// Issue one promotion interval's MMAs, smallest bin first: every band is
// issued over all K=16 halves of the interval's ns stages (ns <= S) before the next,
// larger band.  SA = false: one TMEM accumulator for all bands.  SA = true ("split
// accumulators"): bins >= 1 go to d_small and bin 0 to d_big, so the tensor core's
// alignment truncation of each MMA step (K3 probe) never cuts the small bins against the
// bin-0 products; the epilogue combines them as (small + big) in FP32 round-to-nearest.
// Each accumulator's first MMA of the interval overwrites it.
// scaled (R29): the pieces of bin s are scaled by 2^(8s), so the first MMA of each band that
// adds into an already-started accumulator scales it by 2^-8 (scale-input-d): the accumulator
// always holds the current band's scale and ends at bin 0's (bin 1's for SA's small one).
// Lazy stage waits (LZ and fullw != nullptr): the interval's stage q is waited for just before
// its first MMA (in the first band), so the first band starts as soon as stage 0 has landed
// instead of after all S stages; the MMAs and their order are unchanged.  Compiled in only
// where it measured faster (x3, 128-k intervals): the runtime check in every other kernel's
// issuer cost x6 10 % at 4096^3 (r07, profiles/r07/old_vs_head.txt).
template <int CG, int V, int BN, int S, bool SA, bool LZ>
__device__ __forceinline__ void issue_interval(uint32_t d_big, uint32_t d_small, const uint64_t (&a_desc)[S],
                                               const uint64_t (&b_desc)[S], int ns, uint32_t idesc, bool scaled,
                                               uint64_t *fullw, const int (&stg)[S], const uint32_t (&phs)[S],
                                               uint32_t a_ps, uint32_t a_ks) {
    using Cf = Cfg<CG, V, BN>;
    constexpr int H = S * (kBK / kUK);     // K=16 halves per interval (max)
    const int nh = ns * (kBK / kUK);
    bool first_small = true, first_big = true;
    bool band_start = false;   // next MMA is the first of a band
    uint32_t waited = 0u;
    // descriptor start-address field is in 16-byte units: piece / K-half offsets add directly
    auto mma = [&](int i, int j, int h) {
        const int st = h / (kBK / kUK), kk = h % (kBK / kUK);
        if (LZ && fullw && !((waited >> st) & 1u)) {
            mbar_wait(&fullw[stg[st]], phs[st]);
            tc_fence_after();
            waited |= 1u << st;
        }
        const uint64_t ad = a_desc[st] + (uint64_t)(i * a_ps + kk * a_ks);   // 16-byte units
        const uint64_t bd = b_desc[st] + (uint64_t)((j * Cf::B_PIECE + kk * (kUK * 2)) >> 4);
        const bool big = SA && (i + j == 0);
        bool &first = (SA && !big) ? first_small : first_big;
        const uint32_t d = (big || !SA) ? d_big : d_small;
        if (scaled && band_start && !first) umma_bf16_elect_sc8<CG>(d, ad, bd, idesc);
        else umma_bf16_elect<CG>(d, ad, bd, idesc, first ? 0u : 1u);
        band_start = false;
        first = false;
        if constexpr (!SA) first_small = false;
    };
    if constexpr (V == 9) {
        band_start = true;
#pragma unroll
        for (int h = 0; h < H; ++h) if (h < nh) mma(2, 2, h);                              // bin 4: 2^-32
    }
    if constexpr (V >= 8) {   // x8 = the paper's Z_3: bins 0..3
        band_start = true;
#pragma unroll
        for (int h = 0; h < H; ++h) if (h < nh) { mma(1, 2, h); mma(2, 1, h); }           // bin 3: 2^-24
    }
    if constexpr (V == 7) {   // x7: x6 + the a1*b2 term ("at least 7 products"; R27)
        band_start = true;
#pragma unroll
        for (int h = 0; h < H; ++h) if (h < nh) mma(1, 2, h);
    }
    if constexpr (V >= 6) {
        band_start = true;
#pragma unroll
        for (int h = 0; h < H; ++h) if (h < nh) { mma(0, 2, h); mma(1, 1, h); mma(2, 0, h); }  // bin 2: 2^-16
    }
    if constexpr (V == 5) {   // x5: A in two pieces, bin 2 = {02, 11} (R27)
        band_start = true;
#pragma unroll
        for (int h = 0; h < H; ++h) if (h < nh) { mma(0, 2, h); mma(1, 1, h); }
    }
    if constexpr (V >= 3) {
        band_start = true;
#pragma unroll
        for (int h = 0; h < H; ++h) if (h < nh) { mma(0, 1, h); mma(1, 0, h); }           // bin 1: 2^-8
    }
    band_start = true;
#pragma unroll
    for (int h = 0; h < H; ++h) if (h < nh) mma(0, 0, h);                                  // bin 0
}

// The variant's products over nh K=16 halves in the issue order of issue_interval (bands
// smallest bin first; every band over all nh halves; the band's pairs in order).
template <int V, typename F>
__device__ __forceinline__ void for_each_product(int nh, F &&f) {
    if constexpr (V == 9)
        for (int h = 0; h < nh; ++h) f(2, 2, h);
    if constexpr (V >= 8)
        for (int h = 0; h < nh; ++h) { f(1, 2, h); f(2, 1, h); }
    if constexpr (V == 7)
        for (int h = 0; h < nh; ++h) f(1, 2, h);
    if constexpr (V >= 6)
        for (int h = 0; h < nh; ++h) { f(0, 2, h); f(1, 1, h); f(2, 0, h); }
    if constexpr (V == 5)
        for (int h = 0; h < nh; ++h) { f(0, 2, h); f(1, 1, h); }
    if constexpr (V >= 3)
        for (int h = 0; h < nh; ++h) { f(0, 1, h); f(1, 0, h); }
    for (int h = 0; h < nh; ++h) f(0, 0, h);
}

// MC = number of CTA pairs per cluster (1; 2: two vertically adjacent 256 x BN tiles sharing
// the B tile -- each pair loads half of every B slice and multicasts it to both pairs; 4: a 2 x 2
// block of tiles, pairs (pm, pn) = (pair % 2, pair / 2): B shared down each column of the block as
// for 2, and A (MN-major pieces only) shared along each row -- pair pn loads the 64-row box pn of
// its CTA's A rows and multicasts it to the pair beside it, so every A and B byte a cluster
// reads leaves L2 once for two pairs).
// GD ("d" variants, R30; requires SA): the bins >= 1 and bin 0 are promoted into two separate
// FP32 register accumulators (G[0, EC) = bin 0, G[EC, 2 EC) = bins >= 1: the paper's FP32
// partial sums Z^(i,j), pooled per accumulator) and only their final collection is
// FP64, rounded once to FP32 ("adding the final results together in FP64").
// FA (fused A): A is read as FP32 tiles by TMA and converted by 4 extra warps (warps 12..15,
// thread t = row t of the CTA's 128 A rows) into the A half of the piece ring; B's pieces come
// from the pre-pass by TMA as usual.  The piece-ring "full" barrier counts the leader's
// expect-tx arrival (B bytes) plus the converters' arrivals of both CTAs.
// PM (promote every MMA, short k): every K=16 MMA of every product is its own promotion unit --
// the MMA overwrites a TMEM buffer and the epilogue adds it into G with FP32 round-to-nearest --
// so no tensor-core accumulation ever spans more than 16 products, and the units of a tile (all
// its k, at most S stages) go bin by bin, smallest first: G collects the small bins before bin 0,
// the paper's "bins added from smallest to largest" at the promotion level
// (R24).
template <int CG, int V, int BN, int S, int MC, bool SA, bool GD = false, bool FA = false, bool PM = false>
__global__ void __launch_bounds__(FA ? kThreadsFused : kThreads, 1)
    gemm_split_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC, const KParams p) {
    using Cf = Cfg<CG, V, BN>;
    static_assert(!PM || (MC == 1 && !SA && !GD && !FA && BN == 256), "PM: plain kernel");
    constexpr int NST = FA ? CfgFA<V>::STAGES : Cf::STAGES;   // piece ring stages
    constexpr int NF = FA ? CfgFA<V>::FSTAGES : 0;            // FP32 ring stages (fused A)
    constexpr int F32_STAGE = kF32Tile;                       // FP32 ring stage bytes
    static_assert(!FA || (CG == 2 && BN == 256 && MC == 1 && !SA && !GD), "fused A: 2-CTA, N 256");
    constexpr int CL = CG * MC;   // cluster size
    static_assert(MC == 1 || CG == 2, "multicast needs 2-CTA pairs");
    static_assert(MC == 1 || MC == 2 || (MC == 4 && !SA && !GD && !FA && !PM), "multicast: 1, 2 or 2 x 2 pairs");
    constexpr int MCB = MC == 4 ? 2 : MC;   // pairs sharing B (tile rows of the cluster block)
    constexpr int MCA = MC == 4 ? 2 : 1;    // pairs sharing A (tile columns of the cluster block)
    static_assert(!SA || 2 * BN <= kTmemBufStride, "split accumulators need 4 x BN TMEM columns");
    constexpr int NB = 2, ACC_STRIDE = kTmemBufStride;   // TMEM accumulator buffers, columns apart
    static_assert(!GD || SA, "FP64 collection needs split accumulators");
    constexpr int NG = GD ? 2 : 1;     // promoted accumulators per output element
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;
    uint8_t *sB = smem + NST * Cf::A_STAGE;
    uint8_t *f32 = smem + NST * Cf::STAGE;                      // FA: [NF][A tile]
    constexpr int EPI_BYTES = FA ? 0 : Cf::EPI_BYTES;
    constexpr bool TMA_EPI = !FA && Cf::EPI;
    uint8_t *epi = f32 + NF * F32_STAGE;                        // [epilogue warp][2][32 x 16 FP32]
    uint64_t *full = reinterpret_cast<uint64_t *>(epi + EPI_BYTES);
    uint64_t *empty = full + NST;
    uint64_t *acc_full = empty + NST;
    uint64_t *acc_empty = acc_full + NB;
    uint64_t *f32_full = acc_empty + NB;
    uint64_t *f32_empty = f32_full + (NF > 2 ? NF : 2);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(f32_empty + (NF > 2 ? NF : 2));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = (CL > 1) ? cluster_ctarank() : 0u;   // rank in the cluster
    const uint32_t rank = crank % CG;                            // rank in the CTA pair
    const uint32_t pair = crank / CG;                            // which pair of the cluster
    const uint32_t pm = pair % MCB, pn = pair / MCB;             // its place in the cluster block

    // dbg bit 1: trace slot 0 = kernel start, 1 = prologue done, 2 + 3 t .. = tile t (first
    // interval promoted, last interval promoted, C issued), 31 = all stores complete
    // (compiled in only with -DBF16X_TRACE: `make trace` builds build/trace/libbf16x.so)
    auto trace = [&](int slot) {
#ifdef BF16X_TRACE
        if ((p.dbg & 2) && slot < 32) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            p.trace[blockIdx.x * 32 + slot] = t;
        }
#else
        (void)slot;
#endif
    };
    if (threadIdx.x == 4 * 32) trace(0);
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], FA ? 1 + kNumXfWarps * CG : 1);
            mbar_init(&empty[s], MC);     // one commit per pair reading the (shared) stage
        }
        for (int b = 0; b < NB; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], kNumEpiWarps * CG);
        }
        if constexpr (FA)
            for (int b = 0; b < NF; ++b) {
                mbar_init(&f32_full[b], 1);
                mbar_init(&f32_empty[b], kNumXfWarps);
            }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<CG>(tmem_slot, kTmemCols);
    tc_fence_before();
    if constexpr (CL > 1) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // Programmatic dependent launch: everything above overlapped the previous kernel's tail;
    // from here on we read its outputs (the pieces) and may overwrite what it read.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 4 * 32) trace(1);
    // FA register split (per warpgroup, at the top of each role): the epilogue warpgroups hold
    // G (160 registers), producer / MMA and the two converter warpgroups need few (48); the sum
    // must not exceed the launch allocation (96 x 640 = 61440: 128 x 48 + 256 x 48 + 256 x 160 =
    // 59392), or the increase waits forever (176 hung the kernel, r08)

    const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;

    if (warp < 4) {
        if constexpr (FA) asm volatile("setmaxnreg.dec.sync.aligned.u32 48;" ::: "memory");
        if (warp == 0) {
            // ------------------------------ TMA producer ------------------------------
            if (lane == 0) {
                int stage = 0;
                uint32_t phase = 0;
                int fstage = 0;        // FA: FP32 ring
                uint32_t fphase = 0;
                WorkIter it(p, cid, ncl);
                Work w;
                int ptc = -1;          // trace: tile count
                while (it.next(p, w)) {
                    ++ptc;
                    int tm, tn;
                    tile_coords(w.tile, p.tiles_m, p.tiles_n, p.group_m, tm, tn);
                    tm = tm * MCB + (int)pm;
                    tn = tn * MCA + (int)pn;
                    const int a_row = tm * Cf::TILE_M + (int)rank * kBM;
                    const int b_row = tn * BN + (int)rank * Cf::BN_LOCAL;
                    const int kb_end = min(p.nkb, w.i1 * S);
                    if constexpr (FA) {
                        // FP32 tile of this CTA's 128 A rows (local completion, converted by
                        // warps 12..15) and the B pieces of the pair (TMA to the leader's barrier)
                        for (int kb = w.i0 * S; kb < kb_end; ++kb) {
                            mbar_wait(&f32_empty[fstage], fphase ^ 1u);
                            mbar_arrive_expect_tx(&f32_full[fstage], kF32Tile);
                            tma_load_2d(f32 + fstage * kF32Tile, &tmA, &f32_full[fstage], a_row, kb * kBK);
                            if (++fstage == NF) { fstage = 0; fphase ^= 1u; }
                            mbar_wait(&empty[stage], phase ^ 1u);
                            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * Cf::B_STAGE);
                            tma_load_3d_2sm(sB + stage * Cf::B_STAGE, &tmB, &full[stage], kb * kBK, b_row, 0);
                            if (++stage == NST) { stage = 0; phase ^= 1u; }
                        }
                        continue;
                    }
                    for (int kb = w.i0 * S; kb < kb_end; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1u);
                        if (kb == w.i0 * S && ptc < 5) trace(17 + ptc);   // first load of the tile issued
                        uint8_t *a_dst = sA + stage * Cf::A_STAGE;
                        uint8_t *b_dst = sB + stage * Cf::B_STAGE;
                        if constexpr (CG == 1) {
                            mbar_arrive_expect_tx(&full[stage], Cf::STAGE);
                            if (p.a_mn) {
                                tma_load_3d(a_dst, &tmA, &full[stage], a_row, kb * kBK, 0);
                                tma_load_3d(a_dst + Cf::PA * kMnBox, &tmA, &full[stage], a_row + 64, kb * kBK, 0);
                            } else {
                                tma_load_3d(a_dst, &tmA, &full[stage], kb * kBK, a_row, 0);
                            }
                            tma_load_3d(b_dst, &tmB, &full[stage], kb * kBK, b_row, 0);
                        } else {
                            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * Cf::STAGE);
                            if constexpr (MCA == 2) {
                                // this pair's 64-row box of the CTA's A rows, to both pairs of the row
                                const uint16_t amask = (uint16_t)((1u << ((pm * CG) + rank)) | (1u << (((MCB + pm) * CG) + rank)));
                                tma_load_3d_2sm_mc(a_dst + (int)pn * Cf::PA * kMnBox, &tmA, &full[stage], a_row + 64 * (int)pn,
                                                   kb * kBK, 0, amask);
                            } else if (p.a_mn) {
                                tma_load_3d_2sm(a_dst, &tmA, &full[stage], a_row, kb * kBK, 0);
                                tma_load_3d_2sm(a_dst + Cf::PA * kMnBox, &tmA, &full[stage], a_row + 64, kb * kBK, 0);
                            } else {
                                tma_load_3d_2sm(a_dst, &tmA, &full[stage], kb * kBK, a_row, 0);
                            }
                            if constexpr (MC == 1) {
                                tma_load_3d_2sm(b_dst, &tmB, &full[stage], kb * kBK, b_row, 0);
                            } else {
                                // this pair's half of the B slice, piece by piece, to both pairs
                                constexpr int HB = Cf::BN_LOCAL / MCB;
                                const uint16_t mask = (uint16_t)((1u << ((pn * MCB) * CG + rank)) | (1u << ((pn * MCB + 1) * CG + rank)));
#pragma unroll
                                for (int q = 0; q < Cf::PB; ++q)
                                    tma_load_3d_2sm_mc(b_dst + q * Cf::B_PIECE + (int)pm * HB * kRowBytes, &tmB,
                                                       &full[stage], kb * kBK, b_row + (int)pm * HB, q, mask);
                            }
                        }
                        if (++stage == NST) { stage = 0; phase ^= 1u; }
                    }
                }
            }
        } else if (warp == 1) {
            // ------------------------------ MMA issuer --------------------------------
            if (rank == 0) {   // warp-uniform loop; one elected lane issues (umma_*_elect)
                const uint32_t idesc = idesc_bf16_f32(kBM * CG, BN) | (p.a_mn ? (1u << 15) : 0u);   // a_major
                // A descriptor of a stage, piece and K = 16 step strides (16-byte units)
                const bool amn = p.a_mn != 0;
                const uint32_t a_ps = amn ? (uint32_t)(kMnBox >> 4) : (uint32_t)(Cf::A_PIECE >> 4);
                const uint32_t a_ks = amn ? (uint32_t)((2 * 8 * 128) >> 4) : (uint32_t)((kUK * 2) >> 4);
                auto adesc = [&](int stg_) -> uint64_t {
                    const uint32_t sa = smem_u32(sA + stg_ * Cf::A_STAGE);
                    return amn ? smem_desc_mn128(sa, Cf::PA * kMnBox, 1024) : smem_desc_kmajor(sa, kSwizzleAtom, 4);
                };
                int stage = 0;
                uint32_t phase = 0, acc_it = 0;
                WorkIter it(p, cid, ncl);
                Work w;
                int mtc = -1;          // trace: tile count
#ifdef BF16X_TRACE
                long long wait_acc = 0, wait_full = 0, t_issue0 = clock64();   // issuer wait cycles
#endif
                while (it.next(p, w)) {
                    ++mtc;
                    const int kb_end = min(p.nkb, w.i1 * S);
                    if constexpr (PM) {
                        // the whole tile (k <= 32 S) at once: wait for its stages, issue every
                        // product of every K=16 half as its own unit, bins smallest first
                        const int ns = kb_end - w.i0 * S;
                        uint64_t ad[S], bd[S];
                        int stg[S];
#pragma unroll
                        for (int q = 0; q < S; ++q) {
                            stg[q] = stage;
                            if (q < ns) {
                                mbar_wait(&full[stage], phase);
                                ad[q] = adesc(stage);
                                bd[q] = smem_desc_kmajor(smem_u32(sB + stage * Cf::B_STAGE), kSwizzleAtom, 4);
                                if (++stage == NST) { stage = 0; phase ^= 1u; }
                            } else {
                                ad[q] = ad[0];
                                bd[q] = bd[0];
                            }
                        }
                        tc_fence_after();
                        const int nh = (p.k - w.i0 * S * kBK + kUK - 1) / kUK;   // K=16 halves inside k
                        for_each_product<V>(nh, [&](int i, int j, int h) {
                            const uint32_t buf = acc_it & 1u, apar = (acc_it >> 1) & 1u;
                            mbar_wait(&acc_empty[buf], apar ^ 1u);
                            tc_fence_after();
                            const int q = h >> 1, kk = h & 1;
                            uint64_t a0 = ad[0], b0 = bd[0];
#pragma unroll
                            for (int r = 1; r < S; ++r)
                                if (q == r) { a0 = ad[r]; b0 = bd[r]; }
                            umma_bf16_elect<CG>(tmem_base + buf * ACC_STRIDE,
                                                a0 + (uint64_t)(i * a_ps + kk * a_ks),
                                                b0 + (uint64_t)((j * Cf::B_PIECE + kk * (kUK * 2)) >> 4), idesc, 0u);
                            umma_commit_elect<CG>(&acc_full[buf]);
                            ++acc_it;
                        });
#pragma unroll
                        for (int q = 0; q < S; ++q)
                            if (q < ns) umma_commit_elect<CG>(&empty[stg[q]]);
                        continue;
                    }
                    for (int kb = w.i0 * S; kb < kb_end; kb += S, ++acc_it) {
                        const int ns = min(S, kb_end - kb);
                        const uint32_t buf = acc_it % NB, apar = (acc_it / NB) & 1u;
#ifdef BF16X_TRACE
                        const long long tw0 = clock64();
#endif
                        mbar_wait(&acc_empty[buf], apar ^ 1u);
#ifdef BF16X_TRACE
                        const long long tw1 = clock64();
                        wait_acc += tw1 - tw0;
#endif
                        uint64_t a_desc[S], b_desc[S];
                        int stages[S];
                        uint32_t phs[S];
                        constexpr bool kLazy = (V == 3 && S == 4 && !SA);
                        const bool lz = kLazy && p.lazy_full;
#pragma unroll
                        for (int q = 0; q < S; ++q) {
                            stages[q] = stage;
                            phs[q] = phase;
                            if (q < ns) {
                                if (!lz) mbar_wait(&full[stage], phase);
                                a_desc[q] = adesc(stage);
                                b_desc[q] = smem_desc_kmajor(smem_u32(sB + stage * Cf::B_STAGE), kSwizzleAtom, 4);
                                if (++stage == NST) { stage = 0; phase ^= 1u; }
                            } else {
                                a_desc[q] = a_desc[0];
                                b_desc[q] = b_desc[0];
                            }
                        }
                        tc_fence_after();
#ifdef BF16X_TRACE
                        const long long tw2 = clock64();
                        wait_full += tw2 - tw1;
#endif
                        if (kb == w.i0 * S && mtc < 5 && lane == 0) trace(22 + mtc);   // first MMAs of the tile
                        // buffer layout: SA -> small at buf*BN, big at 256 + buf*BN; else one at buf*256
                        const uint32_t d_big = SA ? tmem_base + kTmemBufStride + buf * BN : tmem_base + buf * ACC_STRIDE;
                        const uint32_t d_small = SA ? tmem_base + buf * BN : d_big;
                        issue_interval<CG, V, BN, S, SA, kLazy>(d_big, d_small, a_desc, b_desc, ns, idesc, p.scaled != 0,
                                                                lz ? full : nullptr, stages, phs, a_ps, a_ks);
#pragma unroll
                        for (int q = 0; q < S; ++q)
                            if (q < ns) {
                                if constexpr (MC == 1) umma_commit_elect<CG>(&empty[stages[q]]);
                                else umma_commit2_mask_elect(&empty[stages[q]], (uint16_t)((1u << CL) - 1));
                            }
                        if constexpr (MC == 1) umma_commit_elect<CG>(&acc_full[buf]);
                        else umma_commit2_mask_elect(&acc_full[buf], (uint16_t)(3u << (CG * pair)));
                    }
                }
#ifdef BF16X_TRACE
                if ((p.dbg & 2) && lane == 0) {   // slots 27 / 28 / 29: cycles waiting acc_empty / full, total
                    p.trace[blockIdx.x * 32 + 27] = (unsigned long long)wait_acc;
                    p.trace[blockIdx.x * 32 + 28] = (unsigned long long)wait_full;
                    p.trace[blockIdx.x * 32 + 29] = (unsigned long long)(clock64() - t_issue0);
                }
#endif
            }
        }
    } else if (warp < 4 + kNumEpiWarps) {
        if constexpr (FA) asm volatile("setmaxnreg.inc.sync.aligned.u32 160;" ::: "memory");
        // ------------------------- promotion + epilogue ---------------------------
        constexpr int EC = Cf::EPI_COLS;
        const int ew = warp - 4;
        const int quad = warp & 3;                // TMEM lane quadrant this warp may access
        const int half = ew >> 2;                 // which half of the accumulator columns
        const uint32_t tm_lane = tmem_base + ((uint32_t)(quad * 32) << 16) + half * EC;
        uint32_t acc_it = 0;
        WorkIter it(p, cid, ncl);
        Work w;
        int tcount = 0;
        const bool tr = ew == 0 && lane == 0;
        while (it.next(p, w)) {
            int tm, tn;
            tile_coords(w.tile, p.tiles_m, p.tiles_n, p.group_m, tm, tn);
            tm = tm * MCB + (int)pm;
            tn = tn * MCA + (int)pn;
            const int row = tm * Cf::TILE_M + (int)rank * kBM + quad * 32 + lane;
            const int col0 = tn * BN + half * EC;
            // beta != 0: the old C values this thread will read (its row, its EC columns; one
            // 128-byte line per warp and column) are prefetched into L2 when the tile starts,
            // so all of them are in flight at once instead of one batch of 8 loads at a time
            // (r07 tools/shortk_probe.py: the LU's k = 256 trailing updates ran at 1.2-1.6 TB/s
            // of C traffic with beta = 1, 2.3x the beta = 0 time)
            // (compiled into the default 2-CTA, N = 256 kernels only: the others, tuner options,
            // keep the fmaf epilogue, which gives the same bits, and their register allocation)
            const bool red_add = (CG == 2 && BN == 256 && !GD) && (p.flags & kFlagRedAdd) && p.beta == 1.f &&
                                 (p.alpha == 1.f || p.alpha == -1.f);
            if (p.beta != 0.f && !red_add && !(p.flags & BF16X_ACC_OUT) && w.role != 2 && row < p.m) {
                const float *pc = p.C + row;
#pragma unroll 8
                for (int j = 0; j < EC; ++j)
                    if (col0 + j < p.n) asm volatile("prefetch.global.L2 [%0];" ::"l"(pc + (int64_t)(col0 + j) * p.ldc));
            }
            float G[NG * EC];
            if (!GD && (p.flags & BF16X_ACC_IN) && w.i0 == 0) {   // (never with GD)
#pragma unroll
                for (int j = 0; j < EC; ++j)
                    G[j] = (row < p.m && col0 + j < p.n) ? p.acc[(int64_t)(col0 + j) * p.ldc + row] : 0.f;
            } else {
#pragma unroll
                for (int j = 0; j < NG * EC; ++j) G[j] = 0.f;
            }
            const int kb_end = min(p.nkb, w.i1 * S);
            if constexpr (PM) {
                {
                    const int units = V * ((p.k - w.i0 * S * kBK + kUK - 1) / kUK);   // products x halves
                    for (int u = 0; u < units; ++u, ++acc_it) {
                        const uint32_t buf = acc_it & 1u, apar = (acc_it >> 1) & 1u;
                        mbar_wait(&acc_full[buf], apar);
                        tc_fence_after();
                        const uint32_t taddr = tm_lane + buf * kTmemBufStride;
#pragma unroll
                        for (int c = 0; c < EC / 16; ++c) {
                            float v[16];
                            tmem_ld16(taddr + c * 16, v);
                            tmem_ld_wait();
#pragma unroll
                            for (int j = 0; j < 16; ++j) G[c * 16 + j] = __fadd_rn(G[c * 16 + j], v[j]);
                        }
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            if (CG == 1 || rank == 0) mbar_arrive(&acc_empty[buf]);
                            else mbar_arrive_cluster(&acc_empty[buf], pair * CG);
                        }
                    }
                }
            } else
            for (int kb = w.i0 * S; kb < kb_end; kb += S, ++acc_it) {
                const uint32_t buf = acc_it % NB, apar = (acc_it / NB) & 1u;
                mbar_wait(&acc_full[buf], apar);
                tc_fence_after();
                if constexpr (!SA) {
                    const uint32_t taddr = tm_lane + buf * ACC_STRIDE;
#pragma unroll
                    for (int c = 0; c < EC / 16; ++c) {
                        float v[16];
                        tmem_ld16(taddr + c * 16, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 16; ++j) G[c * 16 + j] = __fadd_rn(G[c * 16 + j], v[j]);
                    }
                } else {
                    // interval total = small bins + bin 0 (RN), then into G (RN); GD: each into
                    // its own accumulator.  Scaled pieces: the small one is at bin 1's scale, 2^8.
                    const uint32_t ts = tm_lane + buf * BN, tb = tm_lane + kTmemBufStride + buf * BN;
                    const float qs = p.scaled ? 0x1p-8f : 1.f;
                    if constexpr (GD) {   // one accumulator at a time: 16 live temporaries
#pragma unroll
                        for (int c = 0; c < 2 * EC / 16; ++c) {
                            float v[16];
                            tmem_ld16((c < EC / 16 ? tb : ts) + (c % (EC / 16)) * 16, v);
                            tmem_ld_wait();
#pragma unroll
                            for (int j = 0; j < 16; ++j) G[c * 16 + j] = __fadd_rn(G[c * 16 + j], v[j]);
                        }
                    } else
#pragma unroll
                    for (int c = 0; c < EC / 16; ++c) {
                        float vs[16], vb[16];
                        tmem_ld16(ts + c * 16, vs);
                        tmem_ld16(tb + c * 16, vb);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            G[c * 16 + j] = __fadd_rn(G[c * 16 + j], __fadd_rn(__fmul_rn(vs[j], qs), vb[j]));
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 1 || rank == 0) mbar_arrive(&acc_empty[buf]);
                    else mbar_arrive_cluster(&acc_empty[buf], pair * CG);
                }
                if (tr && kb == w.i0 * S) trace(2 + 3 * tcount);
            }
            if (tr) trace(3 + 3 * tcount);
            if (w.role != 0) {
                // stream-K fix-up: slot layout [sk tile][cta rank][column 0..BN)[row 0..127]
                float *slot = p.sk_ws + ((size_t)w.sk_slot * CL + crank) * (size_t)NG * BN * kBM;
                const int lrow = quad * 32 + lane;
                unsigned int *flag = p.sk_flags + (size_t)w.sk_slot * CL + crank;
                if (w.role == 2) {
#pragma unroll
                    for (int j = 0; j < NG * EC; ++j) __stcg(slot + (size_t)(half * NG * EC + j) * kBM + lrow, G[j]);
                    __threadfence();
                    asm volatile("bar.sync 1, %0;" ::"n"(kNumEpiWarps * 32));
                    if (ew == 0 && lane == 0) st_release_u32(flag, p.epoch);
                    if (tr) trace(4 + 3 * tcount);
                    ++tcount;
                    continue;
                }
                if (lane == 0)
                    while (ld_acquire_u32(flag) != p.epoch) __nanosleep(64);
                __syncwarp();
#pragma unroll
                for (int j = 0; j < NG * EC; ++j) G[j] = __fadd_rn(G[j], __ldcg(slot + (size_t)(half * NG * EC + j) * kBM + lrow));
            }
            // GD: final collection in FP64, rounded once (R30), in place into G[0, EC)
            if constexpr (GD) {
                const double qd = p.scaled ? 0x1p-8 : 1.0;
#pragma unroll
                for (int j = 0; j < EC; ++j) G[j] = __double2float_rn(__dadd_rn((double)G[EC + j] * qd, (double)G[j]));
            }
            auto zval = [&](int j) -> float { return G[j]; };
            // beta = 0 stores and the red-add update go through shared memory and TMA: the four warps
            // of a column half stage a 128-row x 16-column box (8 KB, double-buffered) and warp quad 0's
            // lane 0 issues a 2D tensor store (or element-wise add in L2) of it; the warps continue with
            // the next tile while the TMA engine drains (rows / columns outside C are clipped by the TMA)
            const bool radd = CG == 2 && BN == 256 && !GD && red_add;
            if (TMA_EPI && p.tma_c && !(p.flags & BF16X_ACC_OUT) && (p.beta == 0.f || radd)) {
                if (!(p.dbg & 1)) {
                    float *gbuf = reinterpret_cast<float *>(epi) + half * (kEpiNBuf * kEpiRows * kEpiCols);
                    const int grow = tm * Cf::TILE_M + (int)rank * kBM;
                    const bool issuer = quad == 0 && lane == 0;
#pragma unroll
                    for (int q = 0; q < EC / kEpiCols; ++q) {
                        float *dst = gbuf + (q % kEpiNBuf) * (kEpiRows * kEpiCols);
                        if (issuer) bulk_wait_read<kEpiNBuf - 1>();   // this buffer's last store has read it
                        asm volatile("bar.sync %0, 128;" ::"r"(2 + half) : "memory");
#pragma unroll
                        for (int j = 0; j < kEpiCols; ++j)
                            dst[j * kEpiRows + quad * 32 + lane] = radd ? p.alpha * zval(q * kEpiCols + j)
                                                                        : fmaf(p.alpha, zval(q * kEpiCols + j), 0.f);
                        fence_proxy_async_smem();
                        asm volatile("bar.sync %0, 128;" ::"r"(2 + half) : "memory");
                        if (issuer) {
                            if (radd) tma_reduce_add_2d(&tmC, dst, grow, col0 + q * kEpiCols);
                            else tma_store_2d(&tmC, dst, grow, col0 + q * kEpiCols);
                            bulk_commit();
                        }
                    }
                }
            } else if (row < p.m) {
                float *crow = p.C + row;
                if (!GD && (p.flags & BF16X_ACC_OUT)) {   // (never with GD)
#pragma unroll
                    for (int j = 0; j < EC; ++j)
                        if (col0 + j < p.n) p.acc[(int64_t)(col0 + j) * p.ldc + row] = G[j];
                } else if (p.beta == 0.f) {
                    if (!(p.dbg & 1))
#pragma unroll
                    for (int j = 0; j < EC; ++j)
                        if (col0 + j < p.n) __stcs(crow + (int64_t)(col0 + j) * p.ldc, fmaf(p.alpha, zval(j), 0.f));
                } else if (radd) {
                    // alpha * Z is exact (alpha = +-1): the L2 adds it to C with one RN rounding
#pragma unroll
                    for (int j = 0; j < EC; ++j)
                        if (col0 + j < p.n)
                            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(crow + (int64_t)(col0 + j) * p.ldc),
                                         "f"(p.alpha * zval(j)) : "memory");
                } else {
                    // beta != 0: batch 8 independent loads of C before the FMAs and stores, so
                    // the old values stream in parallel instead of one round trip per column
#pragma unroll
                    for (int j0 = 0; j0 < EC; j0 += 8) {
                        float cold[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            cold[j] = (col0 + j0 + j < p.n) ? __ldcs(crow + (int64_t)(col0 + j0 + j) * p.ldc) : 0.f;
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            if (col0 + j0 + j < p.n)
                                __stcs(crow + (int64_t)(col0 + j0 + j) * p.ldc, fmaf(p.alpha, zval(j0 + j), p.beta * cold[j]));
                    }
                }
            }
            if (tr) trace(4 + 3 * tcount);
            ++tcount;
        }
        if (lane == 0) bulk_wait<0>();          // every TMA store of this warp is complete
        if (tr) trace(31);
    } else if constexpr (FA) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 48;" ::: "memory");
        // ------------------- fused A: FP32 A tiles -> A pieces -------------------
        // 8 warps: thread tx converts half (16 values of k) of row t = tx % 128 of the A tile,
        // which is [k][128 rows] FP32 (no swizzle): element (t, k) at k*512 + 4t, so the 32
        // lanes of a warp read 32 consecutive words per k.  The 16 values are loaded first,
        // then split in pairs (same arithmetic as the pre-pass) and stored as two 16-byte chunks
        // of the row's 64-byte K-major piece rows, with the 64-byte swizzle of the descriptors.
        const int tx = threadIdx.x - kThreads;
        const int t = tx & (kBM - 1), hk = tx >> 7;
        const uint32_t swz = (uint32_t)((t >> 1) & 3);
        const uint32_t f32_s = smem_u32(f32), sA_s = smem_u32(sA);
        int fs = 0, ps = 0;
        uint32_t fph = 0, pph = 0;
        WorkIter it(p, cid, ncl);
        Work w;
        while (it.next(p, w)) {
            const int kb_end = min(p.nkb, w.i1 * S);
            for (int kb = w.i0 * S; kb < kb_end; ++kb) {
                mbar_wait(&f32_full[fs], fph);
                const uint32_t fa = f32_s + (uint32_t)(fs * kF32Tile) + (uint32_t)t * 4u;
                float x[kBK / 2];
#pragma unroll
                for (int j = 0; j < kBK / 2; ++j) x[j] = lds_f32(fa + (uint32_t)((hk * 16 + j) * kBM * 4));
                __syncwarp();
                if (lane == 0) mbar_arrive(&f32_empty[fs]);      // the FP32 tile is in registers
                if (++fs == NF) { fs = 0; fph ^= 1u; }
                mbar_wait(&empty[ps], pph ^ 1u);
                const uint32_t pa = sA_s + (uint32_t)(ps * Cf::A_STAGE) + (uint32_t)t * kRowBytes;
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    const uint32_t hh = (uint32_t)(2 * hk + h2);     // 16-byte chunk of the row
                    uint32_t q[4][3];
                    bool ok = true;
#pragma unroll
                    for (int j = 0; j < 8; ++j) ok = ok && regular(x[h2 * 8 + j]);
                    if (ok) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) split_pair_fast<Cf::PA>(x[h2 * 8 + 2 * j], x[h2 * 8 + 2 * j + 1], q[j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) split_pair<Cf::PA>(x[h2 * 8 + 2 * j], x[h2 * 8 + 2 * j + 1], q[j]);
                    }
#pragma unroll
                    for (int pc = 0; pc < Cf::PA; ++pc)
                        sts_u32x4(pa + (uint32_t)(pc * Cf::A_PIECE) + ((hh ^ swz) << 4), q[0][pc], q[1][pc], q[2][pc],
                                  q[3][pc]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // visible to the tensor core
                __syncwarp();
                if (lane == 0) {
                    if (rank == 0) mbar_arrive(&full[ps]);
                    else mbar_arrive_release_cluster(&full[ps], pair * CG);
                }
                if (++ps == NST) { ps = 0; pph ^= 1u; }
            }
        }
    }

    tc_fence_before();
    if constexpr (CL > 1) cluster_sync(); else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<CG>(tmem_base, kTmemCols);
    }
}

// ------------------------------------------------------------------------------------
// host side (helpers defined in gemm.cu)
// ------------------------------------------------------------------------------------
int make_piece_map(CUtensorMap *map, const uint16_t *base, int k, int rows, int64_t ld, int64_t plane, int p,
                   int box_rows, int box_p = 0);
int make_f32_map(CUtensorMap *map, const float *base, int rows, int cols, int64_t ld, int box_rows, int box_cols,
                 CUtensorMapSwizzle swz);
// 3D map over p MN-major piece planes (element (i, l) at i + l * ld): dims (m, k, p), box (64, BK, p),
// 128-byte swizzle
int make_piece_map_mn(CUtensorMap *map, const uint16_t *base, int m, int k, int64_t ld, int64_t plane, int p);
// stream-K fix-up buffers of stream st (per-stream resources, capi.cu): ws_floats partial
// accumulators and nflags ready flags compared against the returned per-launch epoch
int sk_workspace(cudaStream_t st, size_t ws_floats, size_t nflags, float **ws, unsigned int **flags,
                 unsigned int *epoch);

template <int CG, int V, int BN, int S, int MC, bool SA = false, bool GD = false, bool FA = false, bool PM = false>
int launch_t(const GemmPlan &pl, cudaStream_t st) {
    using Cf = Cfg<CG, V, BN>;
    constexpr int CL = CG * MC;
    constexpr int THREADS = FA ? kThreadsFused : kThreads;
    constexpr int SMEM = FA ? CfgFA<V>::SMEM : Cf::SMEM;
    auto kern = gemm_split_kernel<CG, V, BN, S, MC, SA, GD, FA, PM>;
    CUtensorMap tmA, tmB, tmC;
    int rc;
    if constexpr (FA) {
        rc = make_f32_map(&tmA, pl.Af, pl.m, pl.k, pl.lda, kBM, kBK, CU_TENSOR_MAP_SWIZZLE_NONE);
        if (rc) return rc;
        rc = make_piece_map(&tmB, pl.Bp, pl.k, pl.n, pl.ldbp, pl.b_plane, Cf::PB, Cf::BN_LOCAL);
    } else {
        rc = pl.a_mn ? make_piece_map_mn(&tmA, pl.Ap, pl.m, pl.k, pl.ldap, pl.a_plane, Cf::PA)
                     : make_piece_map(&tmA, pl.Ap, pl.k, pl.m, pl.ldap, pl.a_plane, Cf::PA, kBM);
        if (rc) return rc;
        if (MC == 1) rc = make_piece_map(&tmB, pl.Bp, pl.k, pl.n, pl.ldbp, pl.b_plane, Cf::PB, Cf::BN_LOCAL);
        else rc = make_piece_map(&tmB, pl.Bp, pl.k, pl.n, pl.ldbp, pl.b_plane, Cf::PB, Cf::BN_LOCAL / (MC == 4 ? 2 : MC), 1);
    }
    if (rc) return rc;
    KParams kp;
    kp.m = pl.m; kp.n = pl.n; kp.k = pl.k;
    kp.alpha = pl.alpha; kp.beta = pl.beta;
    kp.C = pl.C; kp.ldc = pl.ldc; kp.acc = pl.acc;
    kp.flags = g_red_add == 0 ? (pl.flags & ~kFlagRedAdd) : (g_red_add == 1 ? (pl.flags | kFlagRedAdd) : pl.flags);
    constexpr int MCB = MC == 4 ? 2 : MC, MCA = MC == 4 ? 2 : 1;
    if (MCA > 1 && (!pl.a_mn || FA)) {
        set_error_msg("2 x 2 multicast needs MN-major A pieces");
        return BF16X_ERR_CUDA;
    }
    kp.tiles_m = ((pl.m + Cf::TILE_M - 1) / Cf::TILE_M + MCB - 1) / MCB;   // rows of (MCB-tall) super-tiles
    kp.tiles_n = ((pl.n + BN - 1) / BN + MCA - 1) / MCA;                   // columns of MCA-wide super-tiles
    kp.nkb = (pl.k + kBK - 1) / kBK;
    const int tiles = kp.tiles_m * kp.tiles_n;
    int units = num_sms() / CL;
    if (pl.max_ctas > 0) units = std::max(1, pl.max_ctas / CL);
    if constexpr (CL > 2) {
        // clusters of 4 do not tile every GPC: only co-resident clusters may be launched
        static int max_clusters = -1;
        if (max_clusters < 0) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
            cudaLaunchConfig_t qc = {};
            qc.gridDim = dim3(units * CL);
            qc.blockDim = dim3(THREADS);
            qc.dynamicSmemBytes = SMEM;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = CL;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            qc.attrs = qa;
            qc.numAttrs = 1;
            int nclu = 0;
            if (cudaOccupancyMaxActiveClusters(&nclu, kern, &qc) != cudaSuccess) {
                cudaGetLastError();
                nclu = 0;
            }
            max_clusters = nclu;
        }
        if (max_clusters > 0) units = std::min(units, max_clusters);
    }
    const int grid = std::min(tiles, units) * CL;
    // Hybrid schedule: all full waves but the last run data-parallel; the last full wave plus
    // the partial one are spread over every cluster by promotion interval (stream-K), so the
    // partial wave no longer idles most of the GPU.  Disabled for accumulator-carry launches.
    kp.n_int = (kp.nkb + S - 1) / S;
    kp.dp_tiles = tiles;
    kp.sk_tiles = 0;
    kp.sk_ws = nullptr;
    kp.sk_flags = nullptr;
    kp.epoch = 0;
    kp.scaled = pl.scaled;
    // raster group height: row-major raster (1) while a wave spans whole rows of at most 16
    // tiles (measured r06, tools/raster_probe.py: 4096^3 x6 +1.5 %, GEMM DRAM reads 830 -> 630
    // MB), 8-tall groups for wider outputs (8192^3: 8 beats 1 and 2 by 3-5 %), and groups of 2
    // super-rows on the multicast schedule of the largest outputs (16384^3 x6: 228 vs 215
    // TFLOPS, DRAM reads ~50 vs ~85 GB per launch -- power-limited, so traffic costs clock);
    // from 48 tile columns the row-major raster beats those groups again (r08,
    // tools/raster_probe.py, alternating repetitions: 16384^3 x6 212.1 vs 209.7, 32768^3 212.1 vs
    // 207.7 TFLOPS; DRAM reads 65.6 vs 65.9 GB at 16384^3 under ncu, so not a traffic effect),
    // and below it 8-tall groups (8192^3 x6: 214.5 vs 207 TFLOPS for 2 or 1)
    kp.lazy_full = g_lazy_full;
    kp.a_mn = (!FA && pl.a_mn) ? 1 : 0;
    kp.reserved_i = 0;
    kp.dbg = g_gemm_debug;
    kp.trace = g_gemm_trace;
    // C through TMA when its base and columns are 16-byte aligned (else per-thread stores)
    kp.tma_c = 0;
    std::memset(&tmC, 0, sizeof(tmC));
    if (!FA && Cf::EPI && !(pl.flags & BF16X_ACC_OUT) && (reinterpret_cast<uintptr_t>(pl.C) & 15u) == 0 && pl.ldc % 4 == 0 &&
        make_f32_map(&tmC, pl.C, pl.m, pl.n, pl.ldc, kEpiRows, kEpiCols, CU_TENSOR_MAP_SWIZZLE_NONE) == BF16X_SUCCESS)
        kp.tma_c = 1;
    kp.group_m = pl.group_m > 0 ? pl.group_m : (MC >= 2 ? (kp.tiles_n >= 48 ? 1 : kGroupM) : (kp.tiles_n <= 16 ? 1 : kGroupM));
    const int ncl = grid / CL;
    // (not for short k: a split tile's fix-up -- the contributor's FP32 partial written and read
    // back -- costs more than the balanced tail wins below 12 promotion intervals; measured r08,
    // tools/shortk_sched_probe.py: 4096^2 x k = 256 x3 37.9 -> 34.0 us, k = 1024 x6 133.4 vs 136.0)
    if (pl.stream_k != 0 && !(pl.flags & (BF16X_ACC_IN | BF16X_ACC_OUT)) && tiles > ncl && tiles % ncl != 0 &&
        kp.n_int >= 12) {
        const int full = tiles / ncl;
        kp.dp_tiles = (full - 1) * ncl;
        kp.sk_tiles = tiles - kp.dp_tiles;
        int rc2 = sk_workspace(st, (size_t)kp.sk_tiles * CL * BN * kBM * (GD ? 2 : 1), (size_t)kp.sk_tiles * CL, &kp.sk_ws, &kp.sk_flags,
                               &kp.epoch);
        if (rc2) return rc2;
    }

    static bool attr_set = false;  // per template instance
    if (!attr_set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
            return check_launch("gemm attr");
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmC, kp);
    if (e != cudaSuccess) {
        set_cuda_error(e, "gemm launch");
        return BF16X_ERR_CUDA;
    }
    count_launch();
    return check_launch("gemm");
}

// Stages per promotion interval: 2 (64 values of k) for the 2-CTA kernel, whose promotion
// round trip (TMEM drain in both CTAs + remote mbarrier arrivals) needs the longer
// interval to stay hidden behind the MMAs; 1 (32 values of k) otherwise.
//
// Tile N (2-CTA kernel only): 256, or 192 / 128 when that needs fewer waves-of-work on the
// persistent grid (wave quantisation: cost ~ ceil(tiles / clusters) * N).
// Measured (r02, x3/x6/x9 at 4096-16384): N = 192 and 128 lose more per-MMA efficiency than
// they win on wave quantisation, so 256 is the default; 192 stays available to the tuner.
inline int choose_tile_n(int m, int n, int cg, int units, int forced) {
    (void)m; (void)n; (void)units;
    if (cg == 1) return 256;
    if (forced == 192) return 192;
    return 256;
}

template <int CG, int V>
int launch_s(const GemmPlan &pl, cudaStream_t st) {
    int s = pl.stages_per_interval;
    // A carried accumulator (k-chunked calls) keeps the interval of the unchunked problem, so
    // chunks whose widths are multiples of 128 reproduce it bit for bit (distributed.py).
    const bool carry = (pl.flags & (BF16X_ACC_IN | BF16X_ACC_OUT)) != 0;
    // 128-k promotion intervals (4 stages) as a tuning hook: x1 (r06 tools/spi_probe.py +13 %)
    // and x3 (issuer with lazy stage waits, 7-stage ring).  x3 keeps 64-k intervals by default:
    // r07 tools/lazy_probe.py, burst clocks, 64-k vs 128-k step time 353.6 vs 386.6 us at
    // 4096^3 and 2.60 vs 2.82 ms at 8192^3 (profiles/r07/old_vs_fix.txt).  The opt-in fused-A
    // and split-ahead x3 kernels follow the hook, so they stay bit-identical to the pre-pass path.
    // Short k, bf16x3 (library schedule, 64 < k <= 256): 128-k intervals, so a 256-k tile is
    // two promotions and the tensor core runs further ahead of the epilogue's C stores
    // (r10 tools/shortk_spi_probe.py, 4096^2 K2 alone: k = 128 24.2 -> 23.5 us, 192 29.1 -> 27.6,
    // 256 33.4 -> 31.3; k = 64 and 320 unchanged; profiles/r10/shortk_spi_probe*.txt).  x3's error
    // is that of its dropped products (2^-16 relative), far above the tensor core's
    // accumulation truncation, so the longer interval costs it no accuracy.
    if constexpr (CG == 2 && V == 3)
        if (s == 0 && !carry && pl.k > 64 && pl.k <= 256 && !use_pm(pl) && !pl.fp64 && !pl.split_acc && !pl.fused_a)
            s = 4;
    if constexpr (CG == 2 && V == 3)
        if (s == 4 && !pl.fp64 && !pl.split_acc) {
            if (pl.multicast == 2 || (pl.multicast == 0 && (int64_t)pl.m * pl.n >= 12288LL * 12288LL))
                return launch_t<2, V, 256, 4, 2>(pl, st);
            return launch_t<2, V, 256, 4, 1>(pl, st);
        }
    if constexpr (CG == 2 && V == 1)
        if (s == 4 && !pl.fp64 && !pl.split_acc && !pl.fused_a) return launch_t<2, V, 256, 4, 1>(pl, st);
    // Short k (<= 128): the whole product is one or two intervals, so the tensor core's
    // truncating accumulation dominates the error; 32-k intervals halve it (measured wide
    // exponents, k = 64: max ratio to the oracle 2.07 -> 1.66) at no cost that matters.
    // Short k (<= pm_max_k, library schedule): every MMA promoted on its own (PM above) -- the
    // accuracy of configs[0]-sized products then no longer depends on the tensor core's
    // truncating accumulation across products
    if (s == 0 && use_pm(pl) && (pl.k + kBK - 1) / kBK <= std::min(4, Cfg<CG, V, 256>::STAGES))
        return launch_t<CG, V, 256, 4, 1, false, false, false, true>(pl, st);
    if (s != 1 && s != 2) s = (CG == 2 && (pl.k > 128 || carry)) ? 2 : 1;
    if (s == 2 && Cfg<CG, V, 256>::STAGES < 4) s = 1;
    // "d" variants (R30): 2-CTA pairs, tile N 128, split accumulators, FP64 collection, 64-k
    // intervals (one instance per variant)
    if constexpr (V >= 3)
        if (pl.fp64) {
            // x3d: 128-k intervals (fewer promotions of the two accumulators; +12 % at 4096^3,
            // r06 tools/gd_probe.py); the longer-product variants keep 64-k intervals (x6d -4 %,
            // x9d -15 % with 128-k ones: their 6-stage ring then stalls between intervals)
            if (pl.stages_per_interval == 4 || (V <= 3 && pl.stages_per_interval == 0))
                return launch_t<2, V, 128, 4, 1, true, true>(pl, st);
            return launch_t<2, V, 128, 2, 1, true, true>(pl, st);
        }
    // fused A (bf16x9 only, where it measured faster): the caller (gemm_core) chose it with
    // fused_a_ok() and split only B
    if (pl.fused_a) {
        if constexpr (CG == 2 && V == 9)
            return s == 2 ? launch_t<2, V, 256, 2, 1, false, false, true>(pl, st)
                          : launch_t<2, V, 256, 1, 1, false, false, true>(pl, st);
        set_error_msg("fused-A plan not launchable");
        return BF16X_ERR_CUDA;
    }
    if constexpr (CG == 2) {
        if (s == 2) {
            const int units = (pl.max_ctas > 0 ? pl.max_ctas : num_sms()) / CG;
            const int bn = choose_tile_n(pl.m, pl.n, CG, units, pl.tile_n);
            if (bn == 192) return launch_t<CG, V, 192, 2, 1>(pl, st);
            if (pl.split_acc && V >= 3) return launch_t<CG, V, 128, 2, 1, true>(pl, st);
            // Two pairs per cluster sharing B (TMA multicast) cut L2->SM and DRAM traffic by a
            // quarter but clusters of 4 leave 16 SMs idle; measured (r05) a win only for large
            // outputs, where the kernel runs long enough to be power-limited (16384^3: x3 +17 %,
            // x6 +7 %), and a loss at 8192^3.  Auto: multicast for m*n >= 12288^2.
            const bool mc2 = pl.multicast >= 2 || (pl.multicast == 0 && (int64_t)pl.m * pl.n >= 12288LL * 12288LL);
            if (pl.multicast == 4 && pl.a_mn && !pl.fused_a) return launch_t<CG, V, 256, 2, 4>(pl, st);
            if (mc2) return launch_t<CG, V, 256, 2, 2>(pl, st);
        }
    }
    return s == 2 ? launch_t<CG, V, 256, 2, 1>(pl, st) : launch_t<CG, V, 256, 1, 1>(pl, st);
}

// Per-variant entry points, one translation unit each (gemm_v<V>.cu):
//   kind 1 / 2: pre-split pieces (or fused A), CTA group 1 / 2
#define BF16X_DEFINE_VARIANT(V)                                                        \
    int launch_variant_##V(const GemmPlan &pl, cudaStream_t st, int kind) {            \
        switch (kind) {                                                                \
        case 1: return launch_s<1, V>(pl, st);                                         \
        case 2: return launch_s<2, V>(pl, st);                                         \
        }                                                                              \
        return -12;                                                                    \
    }

int launch_variant_1(const GemmPlan &pl, cudaStream_t st, int kind);
int launch_variant_3(const GemmPlan &pl, cudaStream_t st, int kind);
int launch_variant_5(const GemmPlan &pl, cudaStream_t st, int kind);
int launch_variant_6(const GemmPlan &pl, cudaStream_t st, int kind);
int launch_variant_7(const GemmPlan &pl, cudaStream_t st, int kind);
int launch_variant_8(const GemmPlan &pl, cudaStream_t st, int kind);
int launch_variant_9(const GemmPlan &pl, cudaStream_t st, int kind);

}  // namespace bf16x
