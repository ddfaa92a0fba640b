// capi.cu -- the C ABI of libbf16x.so (include/bf16x.h): argument checks, library stream,
// cached workspace, quick returns, and the split -> GEMM sequence of bf16x_gemm.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "kernels.cuh"

namespace bf16x {

static thread_local char g_err[256] = "";
static cudaStream_t g_stream = nullptr;
static std::atomic<uint64_t> g_launches{0};
static int g_max_ctas = 0;  // cap on the GEMM's persistent grid (bf16x_max_ctas hook; 0 = all SMs)
static int g_group_m = 0;   // tile raster group (bf16x_group_m hook; 0 = default)
// bf16x9 converts A inside the GEMM and splits only B (bf16x_fused_a hook: 0 off, else on; the
// variant where it measured faster: +1..6 % for 2048^3..8192^3, r06 tools/fa9_probe.py; slower
// for x3 / x6, so not compiled for them)
static int g_fused_a = -1;
static int g_force_cg = 0, g_force_bn = 0, g_force_spi = 0, g_stream_k = 1, g_multicast = 0, g_split_acc = 0;  // tuning overrides (bf16x_tune; not in the public ABI)

void set_cuda_error(cudaError_t e, const char *where) {
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
}
void set_error_msg(const char *msg) { snprintf(g_err, sizeof(g_err), "%s", msg); }
int check_launch(const char *where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_cuda_error(e, where);
        return BF16X_ERR_CUDA;
    }
    return BF16X_SUCCESS;
}
void count_launch(uint64_t n) { g_launches += n; }
cudaStream_t current_stream() { return g_stream; }

int arch_ok() {
    static int cached = -1;
    if (cached < 0) {
        int dev = 0, major = 0, minor = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
            cudaGetLastError();
            snprintf(g_err, sizeof(g_err), "no CUDA device");
            return BF16X_ERR_ARCH;  // not cached: a device may appear later
        }
        cached = (major == 10 && minor == 0) ? BF16X_SUCCESS : BF16X_ERR_ARCH;
        if (cached) snprintf(g_err, sizeof(g_err), "device is sm_%d%d, library is built for sm_100a", major, minor);
    }
    return cached;
}

static int64_t round_up8(int64_t v) { return (v + 7) / 8 * 8; }

// Per-stream library resources (bf16x.h: "the library owns a cached workspace per stream"):
// the piece workspace of calls without a caller workspace, and the stream-K fix-up buffers
// (partial accumulators + ready flags compared against a per-stream launch epoch).  Keyed by
// cudaStreamGetId, which is unique for the lifetime of the process (a destroyed stream's
// handle reused by a new stream gets a new id), so calls on different streams never share a
// buffer and may run concurrently.  A buffer grows after a synchronisation of its own stream
// (its earlier work may still read it); bf16x_release frees everything.
struct StreamRes {
    void *ws = nullptr;
    size_t ws_bytes = 0;
    float *sk = nullptr;
    size_t sk_n = 0;
    unsigned int *flags = nullptr;
    size_t flags_n = 0;
    unsigned int epoch = 0;
};
static std::mutex g_res_mu;
static std::unordered_map<unsigned long long, StreamRes> g_res;

static unsigned long long stream_key(cudaStream_t st) {
    unsigned long long id = 0;
    if (cudaStreamGetId(st, &id) != cudaSuccess) {
        cudaGetLastError();
        id = (unsigned long long)(uintptr_t)st;
    }
    return id;
}

static int grow(cudaStream_t st, void **buf, size_t *have, size_t bytes, bool zero, const char *what) {
    if (bytes <= *have) return BF16X_SUCCESS;
    if (*buf) {
        cudaStreamSynchronize(st);
        cudaFree(*buf);
    }
    *buf = nullptr;
    *have = 0;
    if (cudaMalloc(buf, bytes) != cudaSuccess || (zero && cudaMemset(*buf, 0, bytes) != cudaSuccess)) {
        cudaGetLastError();
        if (*buf) cudaFree(*buf);
        *buf = nullptr;
        snprintf(g_err, sizeof(g_err), "%s: cannot allocate %zu bytes", what, bytes);
        return BF16X_ERR_ALLOC;
    }
    *have = bytes;
    return BF16X_SUCCESS;
}

static void *workspace(cudaStream_t st, size_t bytes, int *rc) {
    std::lock_guard<std::mutex> g(g_res_mu);
    StreamRes &r = g_res[stream_key(st)];
    *rc = grow(st, &r.ws, &r.ws_bytes, bytes, false, "workspace");
    return *rc ? nullptr : r.ws;
}

int sk_workspace(cudaStream_t st, size_t ws_floats, size_t nflags, float **ws, unsigned int **flags,
                 unsigned int *epoch) {
    std::lock_guard<std::mutex> g(g_res_mu);
    StreamRes &r = g_res[stream_key(st)];
    size_t skb = r.sk_n * sizeof(float), flb = r.flags_n * sizeof(unsigned int);
    int rc = grow(st, reinterpret_cast<void **>(&r.sk), &skb, ws_floats * sizeof(float), false, "stream-K workspace");
    r.sk_n = skb / sizeof(float);
    if (rc) return rc;
    const bool fresh = nflags > r.flags_n;
    rc = grow(st, reinterpret_cast<void **>(&r.flags), &flb, nflags * sizeof(unsigned int), true, "stream-K flags");
    r.flags_n = flb / sizeof(unsigned int);
    if (rc) return rc;
    if (fresh) r.epoch = 0;                  // new flags are zero: any epoch > 0 is unseen
    if (++r.epoch == 0) ++r.epoch;           // never 0 (the reset value)
    *ws = r.sk;
    *flags = r.flags;
    *epoch = r.epoch;
    return BF16X_SUCCESS;
}

static void release_all_streams() {
    std::lock_guard<std::mutex> g(g_res_mu);
    cudaDeviceSynchronize();
    for (auto &kv : g_res) {
        if (kv.second.ws) cudaFree(kv.second.ws);
        if (kv.second.sk) cudaFree(kv.second.sk);
        if (kv.second.flags) cudaFree(kv.second.flags);
    }
    g_res.clear();
}

static bool variant_ok(int v) { return v == 1 || v == 3 || v == 5 || v == 6 || v == 7 || v == 8 || v == 9; }

static int gemm_args(int m, int n, int k, int lda, int ldb, int ldc, int variant) {
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (k < 0) return -3;
    if (lda < (m > 1 ? m : 1)) return -6;
    if (ldb < (k > 1 ? k : 1)) return -8;
    if (ldc < (m > 1 ? m : 1)) return -11;
    if (!variant_ok(variant)) return -12;
    return 0;
}

int gemm_core(int m, int n, int k, float alpha, const float *A, int lda, const float *B, int ldb, float beta,
              float *C, int ldc, int variant, unsigned flags, const uint16_t *Ap, int64_t ldap, int64_t a_plane,
              const uint16_t *Bp, int64_t ldbp, int64_t b_plane, float *acc, void *ws, size_t ws_bytes,
              cudaStream_t st, int cta_group, bool allow_stream_k, int max_ctas) {
    int rc = arch_ok();
    if (rc) return rc;
    if (m == 0 || n == 0) return BF16X_SUCCESS;
    if ((alpha == 0.f || k == 0) && !(flags & (BF16X_ACC_IN | BF16X_ACC_OUT)))
        return launch_scale(m, n, beta, C, ldc, st);
    const int pa = pieces_a(variant), pb = pieces_b(variant);
    const int64_t kp = round_up8(k), mp = round_up8(m);
    const size_t need = 2ull * ((Ap ? 0 : (size_t)pa * mp) + (Bp ? 0 : (size_t)pb * n)) * (size_t)kp;
    uint8_t *w = nullptr;
    if (need) {
        if (ws) {
            if (ws_bytes < need) return -21;
            w = (uint8_t *)ws;
        } else {
            w = (uint8_t *)workspace(st, need, &rc);
            if (rc) return rc;
        }
    }
    GemmPlan pl;
    pl.m = m; pl.n = n; pl.k = k;
    pl.alpha = alpha; pl.beta = beta;
    pl.C = C; pl.ldc = ldc;
    pl.variant = variant; pl.flags = flags;
    pl.acc = acc;
    pl.cta_group = cta_group ? cta_group : g_force_cg;
    pl.max_ctas = max_ctas > 0 ? max_ctas : g_max_ctas;
    pl.tile_n = g_force_bn;
    pl.stages_per_interval = g_force_spi;
    pl.stream_k = (allow_stream_k && !(flags & BF16X_NO_STREAM_K)) ? g_stream_k : 0;
    pl.multicast = g_multicast;
    pl.split_acc = g_split_acc;
    pl.scaled = (flags & BF16X_SCALED_PIECES) ? 1 : 0;
    pl.fp64 = (flags & BF16X_FP64_COMBINE) ? 1 : 0;
    pl.group_m = g_group_m;
    pl.fused_a = 0;
    pl.a_mn = (flags & BF16X_A_PIECES_MN) ? 1 : 0;
    const bool sc = pl.scaled != 0;
    pl.Af = A; pl.Bf = B; pl.lda = lda; pl.ldb = ldb;
    if (!Ap && !Bp && g_fused_a != 0 && variant == 9 && fused_a_ok(pl)) {
        // only B is split in the pre-pass; the GEMM converts A from FP32 tiles
        uint16_t *b = (uint16_t *)w;
        b_plane = (int64_t)n * kp;
        ldbp = kp;
        rc = launch_split(k, n, B, ldb, b, pb > 1 ? b + b_plane : nullptr, pb > 2 ? b + 2 * b_plane : nullptr, ldbp,
                          false, st, false);
        if (rc) return rc;
        pl.Ap = nullptr;
        pl.Bp = b; pl.ldbp = ldbp; pl.b_plane = b_plane;
        pl.fused_a = 1;
        return launch_gemm_pieces(pl, st);
    }
    // A is split in its own layout (MN-major pieces, ld round_up(m, 8)): no transpose in the pre-pass
    if (!Ap && !Bp) {   // both operands: one pre-pass launch
        uint16_t *a = (uint16_t *)w;
        ldap = mp;
        a_plane = mp * (int64_t)k;
        uint16_t *b = a + pa * a_plane;
        b_plane = (int64_t)n * kp;
        ldbp = kp;
        rc = launch_split_ab(m, n, k, A, lda, a, ldap, a_plane, B, ldb, b, ldbp, b_plane, pa, pb, st, sc, false);
        if (rc) return rc;
        Ap = a;
        Bp = b;
        pl.a_mn = 1;
    }
    if (!Ap) {
        uint16_t *a = (uint16_t *)w;
        ldap = mp;
        a_plane = mp * (int64_t)k;
        rc = launch_split(m, k, A, lda, a, pa > 1 ? a + a_plane : nullptr, pa > 2 ? a + 2 * a_plane : nullptr, ldap,
                          false, st, sc);
        if (rc) return rc;
        Ap = a;
        pl.a_mn = 1;
        w += 2ull * pa * (size_t)a_plane;
    }
    if (!Bp) {
        uint16_t *b = (uint16_t *)w;
        b_plane = (int64_t)n * kp;
        ldbp = kp;
        rc = launch_split(k, n, B, ldb, b, pb > 1 ? b + b_plane : nullptr, pb > 2 ? b + 2 * b_plane : nullptr, ldbp,
                          false, st, sc);
        if (rc) return rc;
        Bp = b;
    }
    pl.Ap = Ap; pl.ldap = ldap; pl.a_plane = a_plane;
    pl.Bp = Bp; pl.ldbp = ldbp; pl.b_plane = b_plane;
    return launch_gemm_pieces(pl, st);
}

}  // namespace bf16x

using namespace bf16x;

extern "C" {

int bf16x_gemm(int m, int n, int k, float alpha, const float *A, int lda, const float *B, int ldb, float beta,
               float *C, int ldc, int variant) {
    int a = gemm_args(m, n, k, lda, ldb, ldc, variant);
    if (a) return a;
    return gemm_core(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, variant, 0u, nullptr, 0, 0, nullptr, 0, 0,
                     nullptr, nullptr, 0, g_stream, 0, true, 0);
}

size_t bf16x_gemm_workspace_size(int m, int n, int k, int variant) {
    if (m < 0 || n < 0 || k < 0) return 0;
    const int v = variant_ok(variant) ? variant : 9;
    return 2ull * ((size_t)pieces_a(v) * round_up8(m) + (size_t)pieces_b(v) * n) * (size_t)round_up8(k);
}

int bf16x_gemm_ex(int m, int n, int k, float alpha, const float *A, int lda, const float *B, int ldb, float beta,
                  float *C, int ldc, int variant, unsigned flags, const uint16_t *A_pieces, int64_t ldap,
                  int64_t a_plane, const uint16_t *B_pieces, int64_t ldbp, int64_t b_plane, float *acc_carry,
                  void *workspace_ptr, size_t ws_bytes, bf16x_stream_t stream) {
    int a = gemm_args(m, n, k, A_pieces ? (m > 1 ? m : 1) : lda, B_pieces ? (k > 1 ? k : 1) : ldb, ldc, variant);
    if (a) return a;
    if (flags & ~(BF16X_ACC_IN | BF16X_ACC_OUT | BF16X_SCALED_PIECES | BF16X_FP64_COMBINE | BF16X_NO_STREAM_K |
                  BF16X_A_PIECES_MN))
        return -13;
    if ((flags & BF16X_FP64_COMBINE) && ((flags & (BF16X_ACC_IN | BF16X_ACC_OUT)) || variant == 1)) return -13;
    const bool amn = (flags & BF16X_A_PIECES_MN) != 0;
    if (A_pieces && ((amn ? (ldap < (m > 1 ? m : 1) || a_plane < ldap * (int64_t)k)
                          : (ldap < k || a_plane < ldap * (int64_t)m)) ||
                     ldap % 8 || a_plane % 8 || (reinterpret_cast<uintptr_t>(A_pieces) & 15u)))
        return -14;
    if (B_pieces && (ldbp < k || ldbp % 8 || b_plane % 8 || b_plane < ldbp * (int64_t)n ||
                     (reinterpret_cast<uintptr_t>(B_pieces) & 15u)))
        return -16;
    if ((flags & (BF16X_ACC_IN | BF16X_ACC_OUT)) && !acc_carry) return -19;
    return gemm_core(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, variant, flags, A_pieces, ldap, a_plane,
                     B_pieces, ldbp, b_plane, acc_carry, workspace_ptr, ws_bytes, (cudaStream_t)stream, 0, true, 0);
}

// testing hook (not in the public header): force cta_group 1 or 2
int bf16x_gemm_cg(int m, int n, int k, float alpha, const float *A, int lda, const float *B, int ldb, float beta,
                  float *C, int ldc, int variant, int cta_group, bf16x_stream_t stream) {
    int a = gemm_args(m, n, k, lda, ldb, ldc, variant);
    if (a) return a;
    return gemm_core(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, variant, 0u, nullptr, 0, 0, nullptr, 0, 0,
                     nullptr, nullptr, 0, (cudaStream_t)stream, cta_group, true, 0);
}

static std::mutex g_host_mu;
static float *g_hA = nullptr, *g_hB = nullptr, *g_hC = nullptr, *g_hAp = nullptr;   // g_hAp: A's pieces
static size_t g_hA_n = 0, g_hB_n = 0, g_hC_n = 0, g_hAp_n = 0;
// host-path pipeline: copy-in / copy-out streams and per-chunk events (created once)
constexpr int kHostChunks = 16;     // event slots; the chunk count is min(g_host_chunks, n / 256)
constexpr int kHostStreams = 4;     // compute streams: consecutive chunk GEMMs run concurrently
static int g_host_chunks = 12;
static cudaStream_t g_s_in = nullptr, g_s_out = nullptr, g_s_comp[kHostStreams] = {};
static float *g_hBp = nullptr;      // per-compute-stream B piece slices
static size_t g_hBp_n = 0;
static cudaEvent_t g_ev_asplit = nullptr, g_ev_end[kHostStreams] = {};
// optional timeline of the last pipelined call (bf16x_host_timeline): events with timing
static bool g_tl_on = false;
static cudaEvent_t g_tl_ev[4 + 3 * kHostChunks] = {};
static int g_tl_n = 0;
static int tl_record(int slot, cudaStream_t s) {
    if (!g_tl_on) return 0;
    if (!g_tl_ev[slot] && cudaEventCreate(&g_tl_ev[slot]) != cudaSuccess) return 1;
    if (slot + 1 > g_tl_n) g_tl_n = slot + 1;
    return cudaEventRecord(g_tl_ev[slot], s) != cudaSuccess;
}
static cudaEvent_t g_ev_a = nullptr, g_ev_b[kHostChunks], g_ev_c[kHostChunks], g_ev_done = nullptr;
// 2D block pipeline (beta == 0, large m and n): row blocks of A x column blocks of B
constexpr int kH2dMax = 8;
static int g_host_2d = 1;                               // bf16x_host_2d hook: 0 = column chunks only
static cudaStream_t g_s_split = nullptr;
static cudaEvent_t g_ev_ar[kH2dMax], g_ev_bc[kH2dMax], g_ev_as[kH2dMax], g_ev_bs[kH2dMax];
static cudaEvent_t g_ev_blk[kH2dMax * kH2dMax];
static bool g_h2d_init = false;

static int ensure(float **p, size_t *cap, size_t n) {
    if (n <= *cap) return BF16X_SUCCESS;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    if (cudaMalloc((void **)p, n * sizeof(float)) != cudaSuccess) {
        cudaGetLastError();
        return BF16X_ERR_ALLOC;
    }
    *cap = n;
    return BF16X_SUCCESS;
}

static int host_pipeline_init() {
    if (g_s_in) return BF16X_SUCCESS;
    cudaError_t e = cudaStreamCreateWithFlags(&g_s_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g_s_out, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_ev_a, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_ev_done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_ev_asplit, cudaEventDisableTiming);
    for (int q = 0; q < kHostStreams && e == cudaSuccess; ++q) {
        e = cudaStreamCreateWithFlags(&g_s_comp[q], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_ev_end[q], cudaEventDisableTiming);
    }
    for (int j = 0; j < kHostChunks && e == cudaSuccess; ++j) {
        e = cudaEventCreateWithFlags(&g_ev_b[j], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_ev_c[j], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        set_cuda_error(e, "gemm_host streams");
        return BF16X_ERR_CUDA;
    }
    return BF16X_SUCCESS;
}

// Host-buffer GEMM.  Small problems: copy in, GEMM, copy out on the library stream.  Large ones
// are pipelined over column chunks of B and C so the PCIe transfers overlap the device work:
//   copy-in stream : A, then B chunk 0, 1, ... (and C chunks when beta != 0)
//   library stream : split A once (K-major pieces)
//   compute streams: chunk j on stream j % 4, once its B has landed: split the chunk (own piece
//                    slice) and run the GEMM on the pre-split A.  A narrow chunk fills only part
//                    of the GPU, so consecutive chunks' GEMMs run side by side and keep up with
//                    the PCIe stream; the tail after the last byte lands is one chunk's GEMM
//   copy-out stream: C chunk j as soon as its GEMM is done (overlaps the next chunks' copy-in)
// Each chunk is an independent GEMM: its columns equal bf16x_gemm on that column block without
// the stream-K schedule (chunk width: n / min(12, n / 256) rounded up to 256 columns when
// m*k >= 2^20 and n >= 1024).
// 2D block pipeline for beta == 0: A is cut into R row blocks and B into Cb column blocks
// (<= 8 each, multiples of 256); the copy-in stream sends A_0, B_0, A_1, B_1, ... so block
// (i, j) of C can start as soon as A_i and B_j have landed -- after 1/R + 1/Cb of the inputs
// instead of all of A -- each block of A / B is split once (K-major pieces at its offset, on a
// split stream), the block GEMMs run on 4 compute streams in order of readiness, and each C block
// goes back as soon as its GEMM is done.  PCIe carries A and B once each; every block of C
// equals bf16x_gemm_ex(..., BF16X_NO_STREAM_K) on the same rows and columns.
static int host_gemm_2d(int m, int n, int k, float alpha, const float *A_host, int lda, const float *B_host, int ldb,
                        float *C_host, int ldc, int variant, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    if (!g_h2d_init) {
        e = cudaStreamCreateWithFlags(&g_s_split, cudaStreamNonBlocking);
        for (int i = 0; i < kH2dMax && e == cudaSuccess; ++i) {
            e = cudaEventCreateWithFlags(&g_ev_ar[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_ev_bc[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_ev_as[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_ev_bs[i], cudaEventDisableTiming);
        }
        for (int i = 0; i < kH2dMax * kH2dMax && e == cudaSuccess; ++i)
            e = cudaEventCreateWithFlags(&g_ev_blk[i], cudaEventDisableTiming);
        if (e != cudaSuccess) {
            set_cuda_error(e, "gemm_host 2d init");
            return BF16X_ERR_CUDA;
        }
        g_h2d_init = true;
    }
    const int pa = pieces_a(variant), pb = pieces_b(variant);
    const int64_t kp = round_up8(k);
    int R = std::max(1, std::min(kH2dMax, m / 1024)), Cb = std::max(1, std::min(kH2dMax, n / 1024));
    if (g_host_2d > 1) {                                     // tuning hook: explicit (R << 4) | Cb
        R = std::max(1, std::min(kH2dMax, g_host_2d >> 4));
        Cb = std::max(1, std::min(kH2dMax, g_host_2d & 15));
    }
    const int mb = ((m + R - 1) / R + 255) / 256 * 256, nbk = ((n + Cb - 1) / Cb + 255) / 256 * 256;
    R = (m + mb - 1) / mb;
    Cb = (n + nbk - 1) / nbk;
    const int64_t mp = round_up8(m);      // A's pieces in A's own layout (MN-major), ld mp
    int rc = ensure(&g_hAp, &g_hAp_n, ((size_t)pa * mp * kp + 1) / 2);
    if (!rc) rc = ensure(&g_hBp, &g_hBp_n, ((size_t)pb * n * kp + 1) / 2);
    if (rc) return rc;
    uint16_t *ap = reinterpret_cast<uint16_t *>(g_hAp), *bp = reinterpret_cast<uint16_t *>(g_hBp);
    const int64_t a_plane = mp * (int64_t)k, b_plane = (int64_t)n * kp;
    e = cudaEventRecord(g_ev_done, st);                      // the caller's earlier work first
    if (e == cudaSuccess) e = cudaStreamWaitEvent(g_s_in, g_ev_done, 0);
    for (int t = 0; t < std::max(R, Cb) && e == cudaSuccess; ++t) {
        if (t < R) {
            const int r0 = t * mb, mi = std::min(mb, m - r0);
            e = cudaMemcpy2DAsync(g_hA + r0, (size_t)m * 4, A_host + r0, (size_t)lda * 4, (size_t)mi * 4, k,
                                  cudaMemcpyHostToDevice, g_s_in);
            if (e == cudaSuccess) e = cudaEventRecord(g_ev_ar[t], g_s_in);
        }
        if (t < Cb && e == cudaSuccess) {
            const int c0 = t * nbk, nj = std::min(nbk, n - c0);
            e = cudaMemcpy2DAsync(g_hB + (size_t)c0 * k, (size_t)k * 4, B_host + (size_t)c0 * ldb, (size_t)ldb * 4,
                                  (size_t)k * 4, nj, cudaMemcpyHostToDevice, g_s_in);
            if (e == cudaSuccess) e = cudaEventRecord(g_ev_bc[t], g_s_in);
        }
    }
    // splits, in arrival order
    for (int t = 0; t < std::max(R, Cb) && e == cudaSuccess && !rc; ++t) {
        if (t < R) {
            const int r0 = t * mb, mi = std::min(mb, m - r0);
            e = cudaStreamWaitEvent(g_s_split, g_ev_ar[t], 0);
            uint16_t *a0 = ap + r0;
            if (e == cudaSuccess)
                rc = launch_split(mi, k, g_hA + r0, m, a0, pa > 1 ? a0 + a_plane : nullptr, pa > 2 ? a0 + 2 * a_plane : nullptr,
                                  mp, false, g_s_split);
            if (!rc && e == cudaSuccess) e = cudaEventRecord(g_ev_as[t], g_s_split);
        }
        if (t < Cb && e == cudaSuccess && !rc) {
            const int c0 = t * nbk, nj = std::min(nbk, n - c0);
            e = cudaStreamWaitEvent(g_s_split, g_ev_bc[t], 0);
            uint16_t *b0 = bp + (int64_t)c0 * kp;
            if (e == cudaSuccess)
                rc = launch_split(k, nj, g_hB + (size_t)c0 * k, k, b0, pb > 1 ? b0 + b_plane : nullptr,
                                  pb > 2 ? b0 + 2 * b_plane : nullptr, kp, false, g_s_split);
            if (!rc && e == cudaSuccess) e = cudaEventRecord(g_ev_bs[t], g_s_split);
        }
    }
    // block GEMMs in order of readiness (shell t: blocks (t, 0..t) then (0..t-1, t)), C blocks back
    int blk = 0;
    for (int t = 0; t < std::max(R, Cb) && e == cudaSuccess && !rc; ++t) {
        for (int u = 0; u <= 2 * t && e == cudaSuccess && !rc; ++u) {
            const int i = u <= t ? t : u - t - 1, j = u <= t ? u : t;
            if (i >= R || j >= Cb) continue;
            const int r0 = i * mb, mi = std::min(mb, m - r0), c0 = j * nbk, nj = std::min(nbk, n - c0);
            cudaStream_t cs = g_s_comp[blk % kHostStreams];
            e = cudaStreamWaitEvent(cs, g_ev_as[i], 0);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, g_ev_bs[j], 0);
            if (e != cudaSuccess) break;
            rc = gemm_core(mi, nj, k, alpha, nullptr, m, nullptr, k, 0.f, g_hC + r0 + (size_t)c0 * m, m, variant,
                           BF16X_A_PIECES_MN, ap + r0, mp, a_plane, bp + (int64_t)c0 * kp, kp, b_plane, nullptr, nullptr, 0,
                           cs, 0, false, 0);
            if (rc) break;
            cudaEvent_t ev = g_ev_blk[i * kH2dMax + j];
            e = cudaEventRecord(ev, cs);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(g_s_out, ev, 0);
            if (e == cudaSuccess)
                e = cudaMemcpy2DAsync(C_host + r0 + (size_t)c0 * ldc, (size_t)ldc * 4, g_hC + r0 + (size_t)c0 * m,
                                      (size_t)m * 4, (size_t)mi * 4, nj, cudaMemcpyDeviceToHost, g_s_out);
            ++blk;
        }
    }
    for (int q = 0; q < kHostStreams && e == cudaSuccess; ++q) {   // the library stream joins
        e = cudaEventRecord(g_ev_end[q], g_s_comp[q]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, g_ev_end[q], 0);
    }
    if (rc) return rc;
    if (e == cudaSuccess) e = cudaStreamSynchronize(g_s_out);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        set_cuda_error(e, "gemm_host 2d pipeline");
        return BF16X_ERR_CUDA;
    }
    return BF16X_SUCCESS;
}

int bf16x_gemm_host(int m, int n, int k, float alpha, const float *A_host, int lda, const float *B_host, int ldb,
                    float beta, float *C_host, int ldc, int variant) {
    int a = gemm_args(m, n, k, lda, ldb, ldc, variant);
    if (a) return a;
    int rc = arch_ok();
    if (rc) return rc;
    if (m == 0 || n == 0) return BF16X_SUCCESS;
    std::lock_guard<std::mutex> g(g_host_mu);
    cudaStream_t st = g_stream;
    if ((rc = ensure(&g_hA, &g_hA_n, (size_t)m * (k > 0 ? k : 1))) ||
        (rc = ensure(&g_hB, &g_hB_n, (size_t)(k > 0 ? k : 1) * n)) || (rc = ensure(&g_hC, &g_hC_n, (size_t)m * n)))
        return rc;
    const int p = pieces_a(variant);
    const int64_t kp = round_up8(k);
    // chunk width: a multiple of 256 columns, at most g_host_chunks chunks
    int nchunk = 1;
    if (k > 0 && alpha != 0.f && (int64_t)m * k >= (1 << 20) && n >= 1024)
        nchunk = std::max(1, std::min(std::min(g_host_chunks, kHostChunks), n / 256));
    if (nchunk > 1) {
        if ((rc = host_pipeline_init())) return rc;
        // 2D blocks pay off once the GEMM is not much shorter than the copy-in (tools/e2e_2d_sweep.py:
        // 16384^3 x6 49 vs 56 ms, x9 60 vs 68; 8192^3 x6 / 16384^3 x3 the column chunks by 1-4 %):
        // t_gemm / t_in ~ (2mnk v / 1.35 PFLOP/s) / (4 (mk + kn) / 50 GB/s) >= 0.6, i.e.
        // m n v / (m + n) >= 32400, v = the variant's number of products
        const bool two_d = g_host_2d > 1 ||
                           (g_host_2d == 1 && beta == 0.f && m >= 4096 && n >= 4096 &&
                            (double)m * n * variant / ((double)m + n) >= 32400.0);
        if (two_d && beta == 0.f)
            return host_gemm_2d(m, n, k, alpha, A_host, lda, B_host, ldb, C_host, ldc, variant, st);
        if ((rc = ensure(&g_hAp, &g_hAp_n, ((size_t)p * round_up8(m) * kp + 1) / 2))) return rc;
    }
    cudaError_t e = cudaSuccess;
    if (nchunk == 1) {
        if (k > 0) {
            e = cudaMemcpy2DAsync(g_hA, (size_t)m * 4, A_host, (size_t)lda * 4, (size_t)m * 4, k,
                                  cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess)
                e = cudaMemcpy2DAsync(g_hB, (size_t)k * 4, B_host, (size_t)ldb * 4, (size_t)k * 4, n,
                                      cudaMemcpyHostToDevice, st);
        }
        if (e == cudaSuccess && beta != 0.f)
            e = cudaMemcpy2DAsync(g_hC, (size_t)m * 4, C_host, (size_t)ldc * 4, (size_t)m * 4, n,
                                  cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) {
            set_cuda_error(e, "gemm_host h2d");
            return BF16X_ERR_CUDA;
        }
        rc = gemm_core(m, n, k, alpha, g_hA, m, g_hB, k > 0 ? k : 1, beta, g_hC, m, variant, 0u, nullptr, 0, 0,
                       nullptr, 0, 0, nullptr, nullptr, 0, st, 0, true, 0);
        if (rc) return rc;
        e = cudaMemcpy2DAsync(C_host, (size_t)ldc * 4, g_hC, (size_t)m * 4, (size_t)m * 4, n, cudaMemcpyDeviceToHost,
                              st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            set_cuda_error(e, "gemm_host d2h");
            return BF16X_ERR_CUDA;
        }
        return BF16X_SUCCESS;
    }
    const int cw = ((n + nchunk - 1) / nchunk + 255) / 256 * 256;
    nchunk = (n + cw - 1) / cw;
    uint16_t *ap = reinterpret_cast<uint16_t *>(g_hAp);
    const int64_t mp = round_up8(m);     // A's pieces in A's own layout (MN-major), ld mp
    const int64_t a_plane = mp * (int64_t)k;
    // the caller's stream may still be using the device buffers / host arrays
    e = cudaEventRecord(g_ev_done, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(g_s_in, g_ev_done, 0);
    g_tl_n = 0;
    tl_record(0, g_s_in);                                     // timeline: start
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(g_hA, (size_t)m * 4, A_host, (size_t)lda * 4, (size_t)m * 4, k, cudaMemcpyHostToDevice,
                              g_s_in);
    if (e == cudaSuccess) e = cudaEventRecord(g_ev_a, g_s_in);
    tl_record(1, g_s_in);                                     // A landed
    for (int j = 0; j < nchunk && e == cudaSuccess; ++j) {
        const int c0 = j * cw, nj = std::min(cw, n - c0);
        e = cudaMemcpy2DAsync(g_hB + (size_t)c0 * k, (size_t)k * 4, B_host + (size_t)c0 * ldb, (size_t)ldb * 4,
                              (size_t)k * 4, nj, cudaMemcpyHostToDevice, g_s_in);
        if (e == cudaSuccess && beta != 0.f)
            e = cudaMemcpy2DAsync(g_hC + (size_t)c0 * m, (size_t)m * 4, C_host + (size_t)c0 * ldc, (size_t)ldc * 4,
                                  (size_t)m * 4, nj, cudaMemcpyHostToDevice, g_s_in);
        if (e == cudaSuccess) e = cudaEventRecord(g_ev_b[j], g_s_in);
        tl_record(4 + 3 * j, g_s_in);                         // B chunk j landed
    }
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, g_ev_a, 0);
    if (e != cudaSuccess) {
        set_cuda_error(e, "gemm_host h2d");
        return BF16X_ERR_CUDA;
    }
    rc = launch_split(m, k, g_hA, m, ap, p > 1 ? ap + a_plane : nullptr, p > 2 ? ap + 2 * a_plane : nullptr, mp, false,
                      st);
    if (rc == BF16X_SUCCESS) e = cudaEventRecord(g_ev_asplit, st);
    tl_record(2, st);                                         // A split
    const int pb = pieces_b(variant);
    const size_t slice = 2ull * pb * (size_t)cw * (size_t)kp;   // bytes of one chunk's B pieces
    if (rc == BF16X_SUCCESS && e == cudaSuccess)
        rc = ensure(&g_hBp, &g_hBp_n, (kHostStreams * slice + 3) / 4);
    for (int q = 0; q < kHostStreams && rc == BF16X_SUCCESS && e == cudaSuccess; ++q)
        e = cudaStreamWaitEvent(g_s_comp[q], g_ev_asplit, 0);
    for (int j = 0; j < nchunk && rc == BF16X_SUCCESS && e == cudaSuccess; ++j) {
        const int c0 = j * cw, nj = std::min(cw, n - c0);
        cudaStream_t cs = g_s_comp[j % kHostStreams];
        e = cudaStreamWaitEvent(cs, g_ev_b[j], 0);
        if (e != cudaSuccess) break;
        rc = gemm_core(m, nj, k, alpha, nullptr, m, g_hB + (size_t)c0 * k, k, beta, g_hC + (size_t)c0 * m, m, variant,
                       BF16X_A_PIECES_MN, ap, mp, a_plane, nullptr, 0, 0, nullptr,
                       reinterpret_cast<uint8_t *>(g_hBp) + (j % kHostStreams) * slice, slice, cs, 0, false, 0);
        if (rc) break;
        e = cudaEventRecord(g_ev_c[j], cs);
        tl_record(5 + 3 * j, cs);                             // GEMM j done
        if (e == cudaSuccess) e = cudaStreamWaitEvent(g_s_out, g_ev_c[j], 0);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(C_host + (size_t)c0 * ldc, (size_t)ldc * 4, g_hC + (size_t)c0 * m, (size_t)m * 4,
                                  (size_t)m * 4, nj, cudaMemcpyDeviceToHost, g_s_out);
        tl_record(6 + 3 * j, g_s_out);                        // C chunk j back on the host
        if (e != cudaSuccess) break;
    }
    for (int q = 0; q < kHostStreams && e == cudaSuccess; ++q) {   // the library stream joins the
        e = cudaEventRecord(g_ev_end[q], g_s_comp[q]);               // compute streams (error paths too)
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, g_ev_end[q], 0);
    }
    if (rc) return rc;
    if (e == cudaSuccess) e = cudaStreamSynchronize(g_s_out);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        set_cuda_error(e, "gemm_host pipeline");
        return BF16X_ERR_CUDA;
    }
    return BF16X_SUCCESS;
}

int bf16x_set_stream(bf16x_stream_t stream) {
    g_stream = (cudaStream_t)stream;
    return BF16X_SUCCESS;
}
bf16x_stream_t bf16x_get_stream(void) { return (bf16x_stream_t)g_stream; }

void bf16x_release(void) {
    release_all_streams();
    lu_release_cache();
    std::lock_guard<std::mutex> h(g_host_mu);
    if (g_hA) cudaFree(g_hA);
    if (g_hB) cudaFree(g_hB);
    if (g_hC) cudaFree(g_hC);
    if (g_hAp) cudaFree(g_hAp);
    if (g_hBp) cudaFree(g_hBp);
    g_hA = g_hB = g_hC = g_hAp = g_hBp = nullptr;
    g_hA_n = g_hB_n = g_hC_n = g_hAp_n = g_hBp_n = 0;
}

const char *bf16x_status_string(int status) {
    static thread_local char buf[320];
    const char *s = "unknown status";
    switch (status) {
    case BF16X_SUCCESS: s = "success"; break;
    case BF16X_ERR_CUDA: s = "CUDA error"; break;
    case BF16X_ERR_ALLOC: s = "allocation failed"; break;
    case BF16X_ERR_ARCH: s = "device is not sm_100 (no CPU fallback)"; break;
    case BF16X_ERR_SINGULAR: s = "exactly singular matrix"; break;
    case BF16X_NOT_CONVERGED: s = "iterative refinement did not converge"; break;
    default:
        if (status < 0) s = "invalid argument";
    }
    if (status < 0)
        snprintf(buf, sizeof(buf), "%s %d", s, -status);
    else
        snprintf(buf, sizeof(buf), "%s%s%s", s, g_err[0] ? ": " : "", g_err);
    return buf;
}

int bf16x_device_check(void) { return arch_ok(); }

uint64_t bf16x_launch_count(void) { return g_launches.load(); }

// testing/bench hooks (not in the public header)
int bf16x_default_cta_group(void) { return default_cta_group(); }
void bf16x_stream_k(int on) { g_stream_k = on; }
void bf16x_split_acc(int on) { g_split_acc = on; }
void bf16x_group_m(int g) { g_group_m = g; }
void bf16x_max_ctas(int c) { g_max_ctas = c; }   // tile raster group height (0 = default)
void bf16x_fused_a(int on) { g_fused_a = on; }   // 1 on, 0 off, -1 auto (fused-A warps)
// Timeline of the last pipelined bf16x_gemm_host call, ms since its start: [0] start, [1] A
// landed, [2] A split, [3] unused, then per chunk j: [4+3j] B_j landed, [5+3j] GEMM_j done,
// [6+3j] C_j copied back (-1 = not recorded).  on: enable recording for later calls.
int bf16x_host_timeline(int on, float *ms, int cap) {
    g_tl_on = on != 0;
    int n = 0;
    for (int i = 0; i < g_tl_n && i < cap; ++i, ++n) {
        float t = -1.f;
        if (g_tl_ev[i] && g_tl_ev[0] && cudaEventElapsedTime(&t, g_tl_ev[0], g_tl_ev[i]) != cudaSuccess) {
            cudaGetLastError();
            t = -1.f;
        }
        ms[i] = t;
    }
    return n;
}
void bf16x_host_chunks(int n) { g_host_chunks = n > 0 ? n : 12; }   // bf16x_gemm_host pipeline depth
void bf16x_host_2d(int on) { g_host_2d = on; }   // 0 off, 1 auto (default), >1 forced for beta = 0 with (R<<4)|Cb blocks
void bf16x_multicast(int pairs) { g_multicast = pairs; }   // 0 = auto, 1 = off, 2 = B across 2 pairs, 4 = 2 x 2 pairs (A and B)
void bf16x_tune(int cta_group, int tile_n, int stages_per_interval) {
    g_force_cg = cta_group;
    g_force_bn = tile_n;
    g_force_spi = stages_per_interval;
}

}  // extern "C"
