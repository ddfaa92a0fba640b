// lu.cu -- a6: LU with partial pivoting whose cubic work runs in the split GEMM, followed by
// FP64 iterative refinement (section III: "Only the cubic work of the initial LU
// factorization should be done in the lower precision: all the other steps ... in the higher
// precision").
//
//   factor (FP32, in a device copy of A), blocked right-looking, panel width nb:
//     K4 subpanel_kernel    32-column sub-panels on one thread-block cluster (8-16 CTAs, rows in
//                           shared memory, pivot exchange through DSMEM + cluster barrier);
//        panel_update_kernel   TRSM + rank-32 update of the rest of the 256-wide panel
//        (tail of K4)   the sub-panel's interchanges on the panel's columns and the permutation
//     K5 laswp_multi_kernel  the panel's interchanges on the columns outside it
//        trsm_kernel    U12 = L11^-1 A12 (FP32, unit lower)
//     K2 bf16x GEMM     A22 <- -1 * L21 U12 + 1 * A22 in bf16x<variant>   (the cubic work)
//   refine (FP64, factors widened exactly):
//     K6 residual       r = b - A x, deterministic two-phase row sums
//        trsv_kernel    cooperative blocked forward / backward substitution
#include <chrono>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace bf16x {

int gemm_core(int m, int n, int k, float alpha, const float *A, int lda, const float *B, int ldb, float beta,
              float *C, int ldc, int variant, unsigned flags, const uint16_t *Ap, int64_t ldap, int64_t a_plane,
              const uint16_t *Bp, int64_t ldbp, int64_t b_plane, float *acc, void *ws, size_t ws_bytes,
              cudaStream_t st, int cta_group, bool allow_stream_k = true, int max_ctas = 0);

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
// chunks over the cluster's CTAs and held in shared memory ([col][row]); thread e owns rows
// e, e + 512, ... of its CTA, so the per-column work needs no CTA barrier.  Step t (column
// c = s0+t), per owned unpivoted row:
//   (a) apply step t-1: l = a[i,c-1] / p[c-1] stored in place (the L multiplier),
//       a[i,c'] -= l * p[c'] for c' >= c (p = pivot row of step t-1);
//   (b) candidate |a[i,c]| (ties -> lowest row, LAPACK isamax on the unswapped order): each
//       warp's best key into its shared slot (its best row into its record); warp 0 reduces
//       the 16 warp keys and PUSHES the CTA's key (|a|, row) into every peer's receive slot
//       with st.async, completing bytes on the peer's mbarrier;
//   (c) warp 0 waits on its own mbarrier for all peers' keys (no cluster barrier, no
//       GPU-scope fence per column), picks the same winner everywhere and reads the winning
//       row from the winner CTA's record (DSMEM load) as p.
// Rows are not moved inside the sub-panel: at the end CTA 0 turns the chosen rows into the
// LAPACK interchange sequence (ipiv) and the equivalent gather pairs, which the cluster applies
// to the panel's columns after its last barrier (r10; laswp_multi_kernel later to the others).  All panel arithmetic is FP32.
// ------------------------------------------------------------------------------------
constexpr int kSubW = 32;
constexpr int kSubThreads = 512;
constexpr int kSubWarps = kSubThreads / 32;
constexpr int kSubRec = 36;              // receive record: |a|, row index, 2 pad, 32 row entries
constexpr int kSubMaxCl = 16;

__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                            uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     raddr),
                 "r"(a), "r"(b), "r"(c), "r"(d), "r"(rbar)
                 : "memory");
}

// One bulk DSMEM copy (async proxy) of `bytes` (multiple of 16) from this CTA's shared memory
// into a peer's, completing the bytes on the peer's mbarrier: one transaction-count update per
// record at the receiver instead of one per 16-byte st.async.
__device__ __forceinline__ void bulk_to_peer(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes,
                                             uint32_t mbar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst_cluster),
                 "r"(src_cta), "r"(bytes), "r"(mbar_cluster)
                 : "memory");
}

__device__ __forceinline__ void st_async_v2(uint32_t raddr, uint32_t a, uint32_t b, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "r"(a), "r"(b), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t caddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(caddr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_volatile_v4(uint32_t saddr) {
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(saddr)
                 : "memory");
    return v;
}
__device__ __forceinline__ float ld_cluster_f32(uint32_t caddr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(caddr) : "memory");
    return v;
}

// Candidate key: |a| (non-negative float bits, monotone as unsigned) in the high word, the
// complemented row index in the low word, so the largest key is the largest |a| with ties
// going to the lowest row (LAPACK isamax on the unswapped order).  0 = no candidate.
__device__ __forceinline__ uint64_t cand_key(uint32_t vbits, uint32_t row) {
    return ((uint64_t)vbits << 32) | (uint64_t)(0xFFFFFFFFu - row);
}
// warp-wide maximum of (hi, lo) pairs with two redux operations
__device__ __forceinline__ uint64_t warp_max_key(uint32_t hi, uint32_t lo) {
    const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return ((uint64_t)mh << 32) | ml;
}

__device__ unsigned long long g_sp_trace[kSubMaxCl * 32];   // [cta][0..7 phases, 8..23 warp work, 24..31 max-warp hist]
extern "C" int bf16x_lu_subpanel_trace(unsigned long long *host, int clear) {   // diagnostic hook
    if (clear) {
        static const unsigned long long z[kSubMaxCl * 32] = {};
        return cudaMemcpyToSymbol(g_sp_trace, z, sizeof(z)) == cudaSuccess ? 0 : 1;
    }
    return cudaMemcpyFromSymbol(host, g_sp_trace, sizeof(unsigned long long) * kSubMaxCl * 32) == cudaSuccess ? 0 : 1;
}

template <int RPT, bool TRACE>
__global__ void __launch_bounds__(kSubThreads, 1) subpanel_kernel(float *LU, int ld, int n, int s0, int w, int *ipiv,
                                                              int2 *pairs, int *npairs, int *info, int bulk, int pc0,
                                                              int pc1, int *perm) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int ncta = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    __shared__ __align__(16) uint64_t rbar[2];                   // receive barriers
    __shared__ __align__(16) float rbuf[2 * kSubMaxCl * kSubRec];  // [2][cluster][record]
    // each warp's candidate record (header: key lo, key hi, 2 pad; then the row), double-buffered
    // by step parity: a bulk copy of step t may still read its source while step t+1 runs, never
    // at step t+2 (every peer's step-(t+1) record, which needs ours of step t, has arrived)
    __shared__ __align__(16) float wrec[2 * kSubWarps * kSubRec];
    __shared__ __align__(16) float prow[kSubW];                   // pivot row, columns t.. (shifted)
    __shared__ unsigned long long s_wkey[kSubWarps];              // each warp's candidate key
    __shared__ __align__(16) uint4 rk[2 * kSubMaxCl];             // mode 3: [parity][cta] (key lo, hi, seq)
    __shared__ int s_rows[kSubW];                                 // chosen rows, step order
    __shared__ int s_r0[kSubMaxCl];                               // first row of every CTA
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long tc_start = clock64();
    const int R = n - s0;
    const int r0 = s0 + (int)(((int64_t)R * rank) / ncta), r1 = s0 + (int)(((int64_t)R * (rank + 1)) / ncta);
    const int rl = r1 - r0;
    // The thread's rows (e = tid + k * 512) live in registers for the whole sub-panel, SHIFTED:
    // at step t, a[k][j] holds column s0 + t + j, so every index is a compile-time constant.
    // Multipliers go to global memory as they are produced; a row's U part when it is chosen.
    float a[RPT][kSubW];
    bool live[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int e = tid + k * kSubThreads;
        live[k] = e < rl;
#pragma unroll
        for (int cc = 0; cc < kSubW; ++cc)
            a[k][cc] = (live[k] && cc < w) ? LU[(int64_t)(s0 + cc) * ld + r0 + e] : 0.f;
    }
    if (tid == 0) {
        mbar_init(&rbar[0], 1);
        mbar_init(&rbar[1], 1);
        fence_barrier_init();
    }
    if (tid < 2 * kSubMaxCl) rk[tid] = make_uint4(0u, 0u, 0u, 0u);   // mode 3 sequence numbers start at 1
    if (tid < ncta) s_r0[tid] = s0 + (int)(((int64_t)R * tid) / ncta);
    cl.sync();                                       // barriers initialised cluster-wide
    const uint32_t rbar_s = smem_u32(rbar), rbuf_s = smem_u32(rbuf);
    // interchange bookkeeping (CTA 0, warp 1, overlapped with the exchange): rows are at their
    // own positions when the sub-panel starts; step t swaps position s0+t with the current
    // position of row s_rows[t].  Only <= 2w positions are touched: a (position -> row) map of
    // <= 64 entries held two per lane (identity elsewhere), searched with ballots.
    const bool book = (rank == 0 && wid == 1);
    int mp[2] = {-1, -1}, mr[2] = {-1, -1}, nm = 0;
    auto book_step = [&](int t) {
        const unsigned FULL = 0xffffffffu;
        auto find = [&](const int *key, int v) -> int {
            const unsigned b0 = __ballot_sync(FULL, key[0] == v), b1 = __ballot_sync(FULL, key[1] == v);
            return b0 ? __ffs(b0) - 1 : (b1 ? 32 + __ffs(b1) - 1 : -1);
        };
        auto get = [&](const int *arr, int k) -> int {
            const int v0 = __shfl_sync(FULL, arr[0], k & 31), v1 = __shfl_sync(FULL, arr[1], k & 31);
            return k < 32 ? v0 : v1;
        };
        auto set = [&](int p, int r) {
            int k = find(mp, p);
            if (k < 0) k = nm++;
            if (lane == (k & 31)) {
                if (k < 32) { mp[0] = p; mr[0] = r; } else { mp[1] = p; mr[1] = r; }
            }
            __syncwarp();
        };
        const int r = s_rows[t], here = s0 + t;
        const int kr = find(mr, r);
        const int q = kr >= 0 ? get(mp, kr) : r;          // current position of row r
        const int kh = find(mp, here);
        const int other = kh >= 0 ? get(mr, kh) : here;   // row currently at s0+t
        if (lane == 0) ipiv[here] = q;
        set(q, other);
        set(here, r);
    };
    // diagnostic trace (mode bit 4): thread 0's cycles per phase, summed over the steps, and
    // CTA 0 warp 1's bookkeeping cycles; slots [rank][0..7] of g_sp_trace
    constexpr bool trace = TRACE;
    bulk &= 3;
    long long tc0 = clock64(), tc1 = 0, tc2 = 0, tc3 = 0, tc4 = 0;
    long long acc[6] = {0, 0, 0, 0, 0, 0};
    long long wstart = clock64(), wwork = 0;   // this warp's cycles from sync2 to its arrival at sync1
    for (int t = 0; t <= w; ++t) {
        if (trace && tid == 0) { tc0 = clock64(); if (t > 0) acc[4] += tc0 - tc4; }
        if (t > 0) {
            // apply step t-1: l = a[i,c-1] / p[c-1] (stored), a[i,c'] -= l * p[c'], shift by one
            const float piv = prow[0];
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                if (!live[k]) continue;
                const float l = (piv != 0.f) ? a[k][0] / piv : 0.f;
                LU[(int64_t)(s0 + t - 1) * ld + r0 + tid + k * kSubThreads] = l;
#pragma unroll
                for (int c4 = 0; c4 < kSubW / 4; ++c4) {
                    const float4 q = reinterpret_cast<const float4 *>(prow)[c4];
                    const float pq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int j = 4 * c4 + u;
                        if (j >= 1) a[k][j - 1] = a[k][j] - l * pq[u];
                    }
                }
                a[k][kSubW - 1] = 0.f;
            }
        }
        if (t == w) break;
        if (trace && tid == 0) { tc1 = clock64(); acc[0] += tc1 - tc0; }
        // this thread's best live row, then the warp's (two redux), then the CTA's (smem atomic)
        uint32_t bh = 0u, bl = 0u;
        int bk = -1;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            if (!live[k]) continue;
            float v = fabsf(a[k][0]);
            if (!(v >= 0.f)) v = INFINITY;           // NaN: chosen (and propagated), never skipped
            const uint32_t vh = __float_as_uint(v), vl = 0xFFFFFFFFu - (uint32_t)(r0 + tid + k * kSubThreads);
            if (vh > bh || (vh == bh && vl > bl) || bk < 0) { bh = vh; bl = vl; bk = k; }
        }
        const uint64_t wk = warp_max_key(bh, bk >= 0 ? bl : 0u);
        if (bk >= 0 && wk == (((uint64_t)bh << 32) | bl)) {   // this lane holds the warp's best row
            float *wrow = wrec + ((t & 1) * kSubWarps + wid) * kSubRec + 4;
#pragma unroll
            for (int k = 0; k < RPT; ++k)
                if (k == bk) {
#pragma unroll
                    for (int c4 = 0; c4 < kSubW / 4; ++c4)
                        reinterpret_cast<float4 *>(wrow)[c4] =
                            make_float4(a[k][4 * c4], a[k][4 * c4 + 1], a[k][4 * c4 + 2], a[k][4 * c4 + 3]);
                }
            if (bulk == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // read by the bulk copy
        }
        if (lane == 0) s_wkey[wid] = wk;                   // 0: no live row in this warp
        if (trace) wwork += clock64() - wstart;
        __syncthreads();
        if (trace && tid == 0) { tc2 = clock64(); acc[1] += tc2 - tc1; }
        if (wid == 0) {
            const int buf = t & 1;
            // the CTA's candidate: maximum of the warps' keys (no shared atomics)
            const uint64_t kq = (lane < kSubWarps) ? s_wkey[lane] : 0ull;
            const uint64_t ck = warp_max_key((uint32_t)(kq >> 32), (uint32_t)kq);
            const unsigned wh = __ballot_sync(0xffffffffu, lane < kSubWarps && kq == ck && ck != 0ull);
            const int cw = wh ? __ffs(wh) - 1 : 0;                   // winner warp
            float *crec = wrec + (buf * kSubWarps + cw) * kSubRec;   // the CTA's record
            // exchange modes: 3 keys by plain remote stores + local polling, 2 keys by st.async,
            // 1 whole records by bulk copy, 0 whole records by 9 st.async; 2 and 3 read the
            // winning row from its CTA afterwards (pull)
            const bool pull = bulk >= 2;
            uint32_t ql = 0u, qh = 0u;
            const float *rec = rbuf + buf * kSubMaxCl * (pull ? 2 : kSubRec);
            const int rs = pull ? 2 : kSubRec;
            if (bulk == 3) {
                const uint32_t seq = (uint32_t)t + 1u;
                if (lane < ncta)
                    st_cluster_v4(mapa_u32(smem_u32(&rk[buf * kSubMaxCl + rank]), (uint32_t)lane), (uint32_t)ck,
                                  (uint32_t)(ck >> 32), seq, 0u);
                if (lane < ncta) {
                    uint4 v;
                    do { v = ld_volatile_v4(smem_u32(&rk[buf * kSubMaxCl + lane])); } while (v.z != seq);
                    ql = v.x;
                    qh = v.y;
                }
                __syncwarp();
                if (trace && tid == 0) { tc3 = clock64(); acc[2] += tc3 - tc2; }
            } else {
                if (bulk == 1 && lane == 0) {
                    reinterpret_cast<uint4 *>(crec)[0] = make_uint4((uint32_t)ck, (uint32_t)(ck >> 32), 0u, 0u);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                if (lane == 0) mbar_arrive_expect_tx(&rbar[buf], (uint32_t)(ncta * (pull ? 8 : kSubRec * 4)));
                if (bulk == 1) __syncwarp();
                // lane q pushes into slot `rank` of CTA q's receive buffer
                if (pull) {
                    if (lane < ncta)
                        st_async_v2(mapa_u32(rbuf_s + (uint32_t)((buf * kSubMaxCl + rank) * 2) * 4u, lane),
                                    (uint32_t)ck, (uint32_t)(ck >> 32), mapa_u32(rbar_s + (uint32_t)buf * 8u, lane));
                } else if (bulk == 1 && lane < ncta) {
                    const uint32_t slot = rbuf_s + (uint32_t)((buf * kSubMaxCl + rank) * kSubRec) * 4u;
                    bulk_to_peer(mapa_u32(slot, lane), smem_u32(crec), (uint32_t)(kSubRec * 4),
                                 mapa_u32(rbar_s + (uint32_t)buf * 8u, lane));
                } else if (lane < ncta) {
                    const uint32_t slot = rbuf_s + (uint32_t)((buf * kSubMaxCl + rank) * kSubRec) * 4u;
                    const uint32_t rsl = mapa_u32(slot, lane), rb = mapa_u32(rbar_s + (uint32_t)buf * 8u, lane);
                    st_async_v4(rsl, (uint32_t)ck, (uint32_t)(ck >> 32), 0u, 0u, rb);
                    const float4 *src = reinterpret_cast<const float4 *>(crec + 4);
#pragma unroll
                    for (int c4 = 0; c4 < kSubW / 4; ++c4) {
                        const float4 r4 = src[c4];
                        st_async_v4(rsl + 16u + 16u * c4, __float_as_uint(r4.x), __float_as_uint(r4.y),
                                    __float_as_uint(r4.z), __float_as_uint(r4.w), rb);
                    }
                }
                {   // spin (no suspend): this wait is on the factorisation's critical path
                    const uint32_t par = (uint32_t)((t >> 1) & 1);
                    uint32_t done = 0;
                    while (!done)
                        asm volatile(
                            "{\n\t.reg .pred p;\n\t"
                            "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                            "selp.u32 %0, 1, 0, p;\n\t}"
                            : "=r"(done)
                            : "r"(rbar_s + (uint32_t)buf * 8u), "r"(par)
                            : "memory");
                }
                if (trace && tid == 0) { tc3 = clock64(); acc[2] += tc3 - tc2; }
                ql = (lane < ncta) ? __float_as_uint(rec[lane * rs]) : 0u;
                qh = (lane < ncta) ? __float_as_uint(rec[lane * rs + 1]) : 0u;
            }
            // the cluster's winner, identical in every CTA: lane q holds CTA q's key
            const uint64_t gk = warp_max_key(qh, ql);
            const unsigned hit = __ballot_sync(0xffffffffu, lane < ncta && qh == (uint32_t)(gk >> 32) &&
                                                                ql == (uint32_t)gk);
            const int gq = __ffs(hit) - 1;
            if (pull) {
                // the winning row sits in CTA gq's record of its winning warp (same step parity)
                const int grow = (int)(0xFFFFFFFFu - (uint32_t)gk);
                const int r0q = s_r0[gq];
                const int cwq = ((uint32_t)gk != 0u) ? ((grow - r0q) % kSubThreads) / 32 : 0;
                const uint32_t src = smem_u32(wrec + (buf * kSubWarps + cwq) * kSubRec + 4 + lane);
                prow[lane] = ld_cluster_f32(mapa_u32(src, (uint32_t)gq));
            } else {
                prow[lane] = rec[gq * kSubRec + 4 + lane];
            }
            if (lane == 0) {
                s_rows[t] = (int)(0xFFFFFFFFu - (uint32_t)gk);
                if (rank == 0 && (uint32_t)(gk >> 32) == 0u && *info == 0) *info = s0 + t + 1;
            }
        } else if (book && t > 0) {
            const long long b0 = clock64();
            book_step(t - 1);
            if (trace && lane == 0) acc[5] += clock64() - b0;
        }
        __syncthreads();
        if (trace && tid == 0) { tc4 = clock64(); acc[3] += tc4 - tc3; }
        if (trace) wstart = clock64();
        const int gi = s_rows[t];                    // the owner retires its pivot row: U part
#pragma unroll
        for (int k = 0; k < RPT; ++k)
            if (live[k] && r0 + tid + k * kSubThreads == gi) {
                live[k] = false;
#pragma unroll
                for (int j = 0; j < kSubW; ++j)
                    if (j < w - t) LU[(int64_t)(s0 + t + j) * ld + gi] = a[k][j];
            }
    }
    if (book) {
        if (w > 0) book_step(w - 1);
        int np = 0;
        for (int h = 0; h < 2; ++h) {
            const bool emit = mp[h] >= 0 && mr[h] != mp[h];
            const unsigned bal = __ballot_sync(0xffffffffu, emit);
            if (emit) pairs[np + __popc(bal & ((1u << lane) - 1))] = make_int2(mp[h], mr[h]);
            np += __popc(bal);
        }
        if (lane == 0) *npairs = np;
    }
    cl.sync();   // no CTA exits while a peer may still push into it; pairs / *npairs are published
    // The sub-panel's interchanges on the panel's columns [pc0, pc1) and on the row permutation, as
    // a gather (every source read before any destination is written; <= 2w pairs, two per lane),
    // one warp per column over all warps of the cluster -- fused here in r10 instead of a separate
    // laswp launch.  The pairs and the columns' rows were written by other CTAs of the cluster
    // before the barrier: read through L2.
    {
        const int np = __ldcg(npairs);
        const int gw = rank * kSubWarps + wid, nw = ncta * kSubWarps;
        int2 q[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) q[h] = (h * 32 + lane < np) ? __ldcg(pairs + h * 32 + lane) : make_int2(0, 0);
        for (int c = pc0 + gw; c < pc1 && np > 0; c += nw) {
            float *col = LU + (int64_t)c * ld;
            float v[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) v[h] = (h * 32 + lane < np) ? __ldcg(col + q[h].y) : 0.f;
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (h * 32 + lane < np) col[q[h].x] = v[h];
        }
        if (perm && np > 0 && gw == nw - 1) {       // the last warp (CTA 0 warp 1 builds the pairs)
            int pv[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) pv[h] = (h * 32 + lane < np) ? __ldcg(perm + q[h].y) : 0;
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (h * 32 + lane < np) perm[q[h].x] = pv[h];
        }
    }
    if (trace && lane == 0) atomicAdd(g_sp_trace + rank * 32 + 8 + wid, (unsigned long long)wwork);
    if (trace && (tid == 0 || (book && lane == 0))) {
        unsigned long long *tr = g_sp_trace + rank * 32;
        if (tid == 0) {
            for (int q = 0; q < 5; ++q) atomicAdd(tr + q, (unsigned long long)acc[q]);
            atomicAdd(tr + 6, (unsigned long long)(clock64() - tc_start));
            atomicAdd(tr + 7, 1ull);
        } else {
            atomicAdd(tr + 5, (unsigned long long)acc[5]);
        }
    }
}

// After sub-panel [s0, s0+w) (rows already interchanged): remaining panel columns [c1, c2)
// get U = L11^-1 A[s0:s0+w, c1:c2] (L11 unit lower w x w; every block recomputes it with one
// column per thread held in registers) and rows [c1, n) get A -= L21 U, 64 rows per block,
// 4 x 4 outputs per thread from shared-memory tiles.  U overwrites its source rows, which every
// block reads first: the store is made by the LAST block to finish its reads (arrival counter
// `ctr`, reset by that block for the next launch), so no block can read U instead of A whatever
// the order or residency of the blocks.
constexpr int kUpdRows = 64;
// sU row stride: a multiple of 4 (16-byte rows for the float4 reads) with an odd number of 16-byte
// chunks, so the column copies (lanes along a column's 32 rows) are 4-way instead of 32-way bank
// conflicted (r10)
__host__ __device__ inline int upd_ncp(int nc) {
    const int ncp = (nc + 3) & ~3;
    return ((ncp >> 2) & 1) ? ncp : ncp + 4;
}
static size_t panel_update_smem(int nc) {
    const int ncp = upd_ncp(nc);
    return ((size_t)kSubW * ncp + (size_t)kSubW * (kSubW + 1) + (size_t)kSubW * kUpdRows) * sizeof(float);
}
__global__ void __launch_bounds__(256, 1) panel_update_kernel(float *LU, int ld, int n, int s0, int w, int c1, int c2,
                                                           unsigned int *ctr) {
    extern __shared__ __align__(16) float su[];
    __shared__ int store_u;
    const int nc = c2 - c1, ncp = upd_ncp(nc);
    float *sU = su;                                   // [kSubW][ncp]      row r of the w x nc block
    float *sL11 = sU + (size_t)kSubW * ncp;           // [kSubW][kSubW+1]  L11[r][i]
    float *sL21 = sL11 + kSubW * (kSubW + 1);         // [kSubW][kUpdRows] (col t, row r)
    const int tid = threadIdx.x;
    for (int e = tid; e < kSubW * ncp; e += blockDim.x) {
        const int r = e % kSubW, c = e / kSubW;
        if (r < w && c < nc) async_copy_f32(sU + r * ncp + c, LU + (int64_t)(c1 + c) * ld + s0 + r);
        else sU[r * ncp + c] = 0.f;
    }
    for (int e = tid; e < kSubW * kSubW; e += blockDim.x) {
        const int r = e % kSubW, i = e / kSubW;
        if (r < w && i < w && r > i) async_copy_f32(sL11 + r * (kSubW + 1) + i, LU + (int64_t)(s0 + i) * ld + s0 + r);
        else sL11[r * (kSubW + 1) + i] = 0.f;
    }
    const int rb = c1 + blockIdx.x * kUpdRows;
    const int nr = min(kUpdRows, n - rb);
    for (int e = tid; e < kSubW * kUpdRows; e += blockDim.x) {
        const int r = e % kUpdRows, t = e / kUpdRows;
        if (r < nr && t < w) async_copy_f32(sL21 + t * kUpdRows + r, LU + (int64_t)(s0 + t) * ld + rb + r);
        else sL21[t * kUpdRows + r] = 0.f;
    }
    // this thread's first 4 x 4 block of the update target, loaded now so its latency overlaps
    // the staging copies and the forward substitution (rows rb.. are disjoint from the U rows
    // s0..s0+w that block 0 writes below)
    // rows 4ty.. (ty = tid % 16), columns 4tx.. (tx = tid / 16): a warp covers 2 columns x 64
    // consecutive rows, so each load / store instruction touches 4 cache lines (r10: was 16 columns
    // x 8 rows = 16 lines)
    const int ty = tid & 15, tx = tid >> 4;
    // 16-byte accesses of a thread's 4 rows when they are aligned and inside the matrix
    const bool vec = ((reinterpret_cast<uintptr_t>(LU) & 15u) == 0) && (ld % 4 == 0) && (rb % 4 == 0) && (4 * ty + 4 <= nr);
    float old[4][4];
    auto load_old = [&](int cq) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (vec && cq + j < nc) {
                const float4 v = *reinterpret_cast<const float4 *>(LU + (int64_t)(c1 + cq + j) * ld + rb + 4 * ty);
                old[j][0] = v.x; old[j][1] = v.y; old[j][2] = v.z; old[j][3] = v.w;
                continue;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = 4 * ty + i;
                old[j][i] = (cq + j < nc && r < nr) ? LU[(int64_t)(c1 + cq + j) * ld + rb + r] : 0.f;
            }
        }
    };
    load_old(4 * tx);
    async_wait_all();
    __syncthreads();                                   // this block's reads of the U rows are done
    if (tid == 0) {
        const bool last = atomicAdd(ctr, 1u) == gridDim.x - 1;
        if (last) *ctr = 0u;                           // every block has arrived: ready for the next launch
        store_u = last;
    }
    __syncthreads();
    for (int c = tid; c < nc; c += blockDim.x) {      // forward substitution, column in registers
        float x[kSubW];
#pragma unroll
        for (int r = 0; r < kSubW; ++r) x[r] = sU[r * ncp + c];
#pragma unroll
        for (int i = 0; i < kSubW - 1; ++i)
#pragma unroll
            for (int r = i + 1; r < kSubW; ++r) x[r] = x[r] - sL11[r * (kSubW + 1) + i] * x[i];
#pragma unroll
        for (int r = 0; r < kSubW; ++r) sU[r * ncp + c] = x[r];
        if (store_u)
#pragma unroll
            for (int r = 0; r < kSubW; ++r)
                if (r < w) LU[(int64_t)(c1 + c) * ld + s0 + r] = x[r];
    }
    __syncthreads();
    // A[rb + 4ty + i, c1 + cq + j] -= sum_t L21[., t] U[t, .]
    for (int cq = 4 * tx; cq < nc; cq += 64) {
        if (cq != 4 * tx) load_old(cq);
        float acc[4][4] = {};
#pragma unroll 8
        for (int t = 0; t < kSubW; ++t) {
            const float4 l = *reinterpret_cast<const float4 *>(sL21 + t * kUpdRows + 4 * ty);
            const float4 u = *reinterpret_cast<const float4 *>(sU + t * ncp + cq);
            const float lv[4] = {l.x, l.y, l.z, l.w}, uv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[j][i] = fmaf(lv[i], uv[j], acc[j][i]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (vec && cq + j < nc) {
                *reinterpret_cast<float4 *>(LU + (int64_t)(c1 + cq + j) * ld + rb + 4 * ty) =
                    make_float4(old[j][0] - acc[j][0], old[j][1] - acc[j][1], old[j][2] - acc[j][2], old[j][3] - acc[j][3]);
                continue;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = 4 * ty + i;
                if (cq + j < nc && r < nr) LU[(int64_t)(c1 + cq + j) * ld + rb + r] = old[j][i] - acc[j][i];
            }
        }
    }
}

// K5a': a whole panel's interchanges (nmaps sub-panel gather maps of <= 64 pairs each, applied
// in order) on the columns outside the panel, deferred from the sub-panels (lookahead schedule).
__global__ void __launch_bounds__(256) laswp_multi_kernel(float *LU, int ld, int c0, int c1, const int2 *pairs,
                                                          const int *npairs, int nmaps) {
    __shared__ float sv[8][2 * 32];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = c0 + blockIdx.x * 8 + wid;
    if (c >= c1) return;
    float *col = LU + (int64_t)c * ld;
    for (int s = 0; s < nmaps; ++s) {
        const int np = npairs[s];
        const int2 *pr = pairs + 64 * s;
        for (int e = lane; e < np; e += 32) sv[wid][e] = col[pr[e].y];
        __syncwarp();
        for (int e = lane; e < np; e += 32) col[pr[e].x] = sv[wid][e];
        __syncwarp();
    }
}

// K5b: U12 = L11^-1 A12 with L11 = unit lower jb x jb at (j0, j0), A12 = rows j0..j0+jb of
// columns [c0, c0 + ncols).  One CTA per 32 columns held in shared memory; L11 is staged in
// 32-column chunks.  Per chunk: the 32 x 32 diagonal triangle is solved by warp shuffles
// (warp w owns 4 columns, lanes are rows: no CTA barrier per row), then the rows below take
// the chunk's contribution as a small product, 4 rows per thread from a transposed L tile.
constexpr int kTrsmCols = 32;
constexpr int kTrsmLd = kTrsmCols + 1;    // sB row stride: column reads of a row block are conflict-free
static size_t trsm_smem(int jb) {
    const int jbp = (jb + 3) & ~3;
    return ((size_t)jbp * kTrsmLd + 32 * 33 + (size_t)32 * jbp) * sizeof(float);
}
__global__ void __launch_bounds__(256) trsm_kernel(float *LU, int ld, int j0, int jb, int c0, int ncols) {
    extern __shared__ __align__(16) float sm[];
    const int jbp = (jb + 3) & ~3;
    float *sB = sm;                                   // [jb][33]   (row r, column c)
    float *sLd = sB + (size_t)jbp * kTrsmLd;          // [32][33]   L[i0+r][i0+i]
    float *sLt = sLd + 32 * 33;                       // [32][jbp]  L[i0+ib+r][i0+i] at i*jbp + r
    const int cb = c0 + blockIdx.x * kTrsmCols;
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5, lane = tx;
    // the 32 columns' rows j0.. with lanes along a column (coalesced; r10, was one column per lane)
    for (int e = tid; e < jb * kTrsmCols; e += blockDim.x) {
        const int r = e % jb, cc = e / jb;
        if (cb + cc < c0 + ncols) async_copy_f32(sB + r * kTrsmLd + cc, LU + (int64_t)(cb + cc) * ld + j0 + r);
        else sB[r * kTrsmLd + cc] = 0.f;
    }
    for (int i0 = 0; i0 < jb; i0 += 32) {
        const int ib = min(32, jb - i0), below = jb - i0 - ib;
        __syncthreads();
        for (int e = tid; e < 32 * 32; e += blockDim.x) {
            const int r = e & 31, i = e >> 5;
            if (r < ib && i < ib && r > i) async_copy_f32(sLd + r * 33 + i, LU + (int64_t)(j0 + i0 + i) * ld + j0 + i0 + r);
            else sLd[r * 33 + i] = 0.f;
        }
        for (int i = ty; i < ib; i += 8)
            for (int r = lane; r < below; r += 32)
                async_copy_f32(sLt + i * jbp + r, LU + (int64_t)(j0 + i0 + i) * ld + j0 + i0 + ib + r);
        async_wait_all();
        __syncthreads();
        {   // diagonal triangle: warp ty owns columns 4ty .. 4ty+3, lane = row
            float v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = (lane < ib) ? sB[(i0 + lane) * kTrsmLd + 4 * ty + q] : 0.f;
            for (int i = 0; i < ib - 1; ++i) {
                const float l = sLd[lane * 33 + i];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float xi = __shfl_sync(0xffffffffu, v[q], i);
                    if (lane > i) v[q] -= l * xi;
                }
            }
            if (lane < ib)
#pragma unroll
                for (int q = 0; q < 4; ++q) sB[(i0 + lane) * kTrsmLd + 4 * ty + q] = v[q];
        }
        __syncthreads();
        if (below > 0) {  // rows below the chunk: column tx, 4 rows per step
            float x[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = (i < ib) ? sB[(i0 + i) * kTrsmLd + tx] : 0.f;
            for (int rq = 4 * ty; rq < below; rq += 32) {
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (i >= ib) break;
                    const float4 l4 = *reinterpret_cast<const float4 *>(sLt + i * jbp + rq);
                    acc[0] = fmaf(l4.x, x[i], acc[0]);
                    acc[1] = fmaf(l4.y, x[i], acc[1]);
                    acc[2] = fmaf(l4.z, x[i], acc[2]);
                    acc[3] = fmaf(l4.w, x[i], acc[3]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (rq + u < below) sB[(i0 + ib + rq + u) * kTrsmLd + tx] -= acc[u];
            }
        }
    }
    __syncthreads();
    for (int e = tid; e < jb * kTrsmCols; e += blockDim.x) {
        const int r = e % jb, cc = e / jb;
        if (cb + cc < c0 + ncols) LU[(int64_t)(cb + cc) * ld + j0 + r] = sB[r * kTrsmLd + cc];
    }
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

// perm[i] = original row now at position i (the interchanges composed by the sub-panel tails)
__global__ void iota_kernel(int n, int *perm) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) perm[i] = i;
}
__global__ void gather_kernel(int n, const int *perm, const double *v, double *y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = v[perm[i]];
}

// ------------------------------------------------------------------------------------
// K6b: triangular solves in FP64 with the FP32 factors widened exactly ("do the solve
// in a higher precision like FP64").  Two kernels:
//   diag_inverse_kernel  once per factorisation: the FP64 inverse of every 128 x 128
//                        diagonal block of L (unit lower) and U (upper), by row-oriented
//                        substitution (all columns of a row in parallel).
//   trsv_kernel          per solve: block b's CTA accumulates sum_{b' before b} T_{b,b'} x_{b'}
//                        as each x_{b'} is published (per-block ready flags, no grid barrier;
//                        the tiles are streamed into shared memory with cp.async before their
//                        x arrives), then x_b = inv(T_bb) (y_b - sum) -- one 128 x 128 FP64
//                        product on the critical path instead of a 128-step substitution.
// Blocks are numbered in processing order p (lower: b = p; upper: b = nblk-1-p), so both
// solves have the same dependency pattern: p depends on every p' < p.
// ------------------------------------------------------------------------------------
constexpr int kTB = 128;                 // rows / columns per block
constexpr int kTChunk = 64;              // tile columns per streamed chunk
constexpr int kTrsvThreads = 256;
constexpr size_t kTinvBlock = (size_t)kTB * kTB;                         // doubles per inverse
constexpr int kTrsvSmem = (int)(kTinvBlock * sizeof(double) + 2 * (size_t)kTChunk * kTB * sizeof(float) +
                                4 * kTB * sizeof(double));

// Tinv layout: [tri][block][col][row] FP64 (tri 0 = inv(L_bb), 1 = inv(U_bb)); entries outside
// a ragged block's w x w are 0.
__global__ void __launch_bounds__(kTB) diag_inverse_kernel(const float *LU, int ld, int n, double *Tinv) {
    extern __shared__ double sx_inv[];   // X [row][col] (kTB x kTB) then T [row][col] as FP32
    float *sT = reinterpret_cast<float *>(sx_inv + kTinvBlock);
    const int b = blockIdx.x, upper = blockIdx.y, j = threadIdx.x;
    const int c0 = b * kTB, w = min(n, c0 + kTB) - c0;
    for (int r = 0; r < kTB; ++r) {
        sT[r * kTB + j] = (r < w && j < w) ? LU[(int64_t)(c0 + j) * ld + c0 + r] : 0.f;
        sx_inv[r * kTB + j] = 0.0;
    }
    __syncthreads();
    if (!upper) {
        // X = L^-1 (unit lower): X[i][i] = 1, X[i][j] = -sum_{k=j}^{i-1} L[i][k] X[k][j] (j < i)
        for (int i = 0; i < w; ++i) {
            if (j < i) {
                double acc = 0.0;
                for (int k = j; k < i; ++k) acc = fma((double)sT[i * kTB + k], sx_inv[k * kTB + j], acc);
                sx_inv[i * kTB + j] = -acc;
            } else if (j == i) {
                sx_inv[i * kTB + j] = 1.0;
            }
            __syncthreads();
        }
    } else {
        // X = U^-1: X[i][i] = 1/U[i][i], X[i][j] = -(sum_{k=i+1}^{j} U[i][k] X[k][j]) / U[i][i] (j > i)
        for (int i = w - 1; i >= 0; --i) {
            const double d = (double)sT[i * kTB + i];
            if (j > i && j < w) {
                double acc = 0.0;
                for (int k = i + 1; k <= j; ++k) acc = fma((double)sT[i * kTB + k], sx_inv[k * kTB + j], acc);
                sx_inv[i * kTB + j] = -acc / d;
            } else if (j == i) {
                sx_inv[i * kTB + j] = 1.0 / d;
            }
            __syncthreads();
        }
    }
    const int nblk = (n + kTB - 1) / kTB;
    double *out = Tinv + ((size_t)upper * nblk + b) * kTinvBlock;
    for (int c = 0; c < kTB; ++c) out[(size_t)c * kTB + j] = sx_inv[j * kTB + c];   // [col][row]
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// y <- T^-1 y in place (T = L unit lower if lower, else U), y FP64 of length n.  LU: ld % 4
// == 0, 16-byte aligned.  flags[p] = epoch once block p's solution is in y.  Cooperative launch
// (all CTAs co-resident: CTA g owns blocks p = g, g + G, ...).
__global__ void __launch_bounds__(kTrsvThreads, 1) trsv_kernel(const float *LU, int ld, int n, double *y, int lower,
                                                            const double *Tinv, unsigned int *flags,
                                                            unsigned int epoch) {
    extern __shared__ double sm_tr[];
    double *sTi = sm_tr;                                           // [col][row] inverse of T_bb
    float *sC = reinterpret_cast<float *>(sTi + kTinvBlock);        // [2][kTChunk][kTB] tile chunks
    double *sx = reinterpret_cast<double *>(sC + 2 * kTChunk * kTB);   // [kTB] x of the current dependency
    double *sacc = sx + kTB;                                       // [2][kTB] half sums
    double *sy = sacc + 2 * kTB;                                   // [kTB] y_b - sum
    const int nblk = (n + kTB - 1) / kTB;
    const int tid = threadIdx.x, r = tid & (kTB - 1), h = tid >> 7;
    const int nchk = kTB / kTChunk;
    for (int p = blockIdx.x; p < nblk; p += gridDim.x) {
        const int b = lower ? p : nblk - 1 - p;
        const int r0 = b * kTB, w = min(n, r0 + kTB) - r0;
        const int wg = (w + 3) >> 2;                               // 16-byte row groups to copy
        // this block's inverse (consumed last; lands while the dependencies stream)
        const double *ti = Tinv + ((size_t)(lower ? 0 : 1) * nblk + b) * kTinvBlock;
        for (int e = tid; e < (int)(kTinvBlock / 2); e += kTrsvThreads) cp_async16(sTi + 2 * e, ti + 2 * e);
        cp_async_commit();
        auto issue = [&](int s) {        // chunk s of the dependency stream into buffer s & 1
            const int pd = s / nchk, q = s % nchk;
            const int bd = lower ? pd : nblk - 1 - pd;
            const int cc0 = bd * kTB + q * kTChunk;
            const int ncol = max(0, min(kTChunk, min(n, bd * kTB + kTB) - cc0));
            float *dst = sC + (s & 1) * kTChunk * kTB;
            for (int e = tid; e < ncol * wg; e += kTrsvThreads) {
                const int c = e / wg, g = e % wg;
                cp_async16(dst + c * kTB + 4 * g, LU + (int64_t)(cc0 + c) * ld + r0 + 4 * g);
            }
            cp_async_commit();
        };
        double acc = 0.0;
        const int nsteps = p * nchk;
        if (nsteps > 0) issue(0);
        for (int s = 0; s < nsteps; ++s) {
            const int pd = s / nchk, q = s % nchk;
            if (s + 1 < nsteps) {
                issue(s + 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            if (q == 0) {                 // dependency pd's solution: wait for its flag
                if (tid == 0) {
                    while (ld_acquire(flags + pd) < epoch) {}
                    __threadfence();
                }
                __syncthreads();
                const int bd = lower ? pd : nblk - 1 - pd;
                const int wd = min(n, bd * kTB + kTB) - bd * kTB;
                if (tid < kTB) sx[tid] = (tid < wd) ? __ldcg(y + bd * kTB + tid) : 0.0;
            }
            __syncthreads();
            const int bd = lower ? pd : nblk - 1 - pd;
            const int ncol = max(0, min(kTChunk, min(n, bd * kTB + kTB) - (bd * kTB + q * kTChunk)));
            const float *cb = sC + (s & 1) * kTChunk * kTB;
            const int ca = h * (kTChunk / 2), ce = min(ncol, ca + kTChunk / 2);
#pragma unroll 8
            for (int c = ca; c < ce; ++c) acc = fma((double)cb[c * kTB + r], sx[q * kTChunk + c], acc);
            __syncthreads();              // buffer s & 1 is refilled by issue(s + 2)
        }
        if (nsteps == 0) cp_async_wait<0>();
        sacc[h * kTB + r] = acc;
        __syncthreads();
        if (tid < kTB) sy[tid] = (tid < w) ? y[r0 + tid] - (sacc[tid] + sacc[kTB + tid]) : 0.0;
        __syncthreads();
        // x_b = inv(T_bb) y_b : two threads per row, half of the columns each
        double xv = 0.0;
        const int ka = h * (kTB / 2);
#pragma unroll 8
        for (int k = ka; k < ka + kTB / 2; ++k) xv = fma(sTi[(size_t)k * kTB + r], sy[k], xv);
        sacc[h * kTB + r] = xv;
        __syncthreads();
        if (tid < w) __stcg(y + r0 + tid, sacc[tid] + sacc[kTB + tid]);
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release(flags + p, epoch);
        }
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
// N1: GMRES-IR kernels.  The Krylov basis V (n x (m+1) FP64, ld n) is
// small (m <= a few hundred) and L2-resident; the dominant costs per Arnoldi step are the
// FP32-A matvec (HBM) and the two triangular solves.
// ------------------------------------------------------------------------------------
constexpr int kArnThreads = 256;

// One Arnoldi step, classical Gram-Schmidt applied twice (CGS2), on a cooperative grid.
// Column j+1 of V holds w = M^-1 A v_j on entry; on exit it holds v_{j+1} = w' / ||w'||
// (w' = w orthogonalised against v_0..v_j) and hcol[0..j+1] holds Hessenberg column j
// (h_ij = sum of both passes' projections, h_{j+1,j} = ||w'||_2).  j = -1 normalises column 0
// (hcol[0] = its norm).  Rows are split in contiguous chunks over the CTAs; each reduction
// goes through per-CTA partials that every CTA sums in the same order (deterministic).
//   part : [3][gridDim.x][pstride] FP64 scratch, pstride >= j + 2
__global__ void __launch_bounds__(kArnThreads) arnoldi_kernel(double *V, int n, int j, double *part, int pstride,
                                                              double *hcol, GridBar gb, unsigned int epoch) {
    extern __shared__ double sh[];                 // [pstride] projections of the current pass
    __shared__ double sred[kArnThreads / 32];
    const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = kArnThreads / 32;
    const int chunk = (n + G - 1) / G;
    const int r0 = min(n, blockIdx.x * chunk), r1 = min(n, r0 + chunk);
    double *w = V + (int64_t)(j + 1) * n;
    for (int pass = 0; pass < 2 && j >= 0; ++pass) {
        double *pp = part + (size_t)pass * G * pstride;
        for (int c = wid; c <= j; c += nw) {       // partial dots over this CTA's rows
            const double *vc = V + (int64_t)c * n;
            double acc = 0.0;
            for (int r = r0 + lane; r < r1; r += 32) acc = fma(vc[r], w[r], acc);
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) pp[(size_t)blockIdx.x * pstride + c] = acc;
        }
        grid_sync(gb, epoch++);
        for (int c = tid; c <= j; c += kArnThreads) {
            double h = 0.0;
            for (int g = 0; g < G; ++g) h += __ldcg(pp + (size_t)g * pstride + c);
            sh[c] = h;
            if (blockIdx.x == 0) hcol[c] = pass ? hcol[c] + h : h;
        }
        __syncthreads();
        for (int r = r0 + tid; r < r1; r += kArnThreads) {   // w -= V h on this CTA's rows
            double acc = 0.0;
#pragma unroll 8
            for (int c = 0; c <= j; ++c) acc = fma(V[(int64_t)c * n + r], sh[c], acc);
            w[r] -= acc;
        }
        __syncthreads();
    }
    double *pn = part + (size_t)2 * G * pstride;
    double ss = 0.0;
    for (int r = r0 + tid; r < r1; r += kArnThreads) ss = fma(w[r], w[r], ss);
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) sred[wid] = ss;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int q = 0; q < nw; ++q) t += sred[q];
        pn[blockIdx.x] = t;
    }
    grid_sync(gb, epoch++);
    if (tid == 0) {
        double t = 0.0;
        for (int g = 0; g < G; ++g) t += __ldcg(pn + g);
        sred[0] = sqrt(t);
        if (blockIdx.x == 0) hcol[j + 1] = sred[0];
    }
    __syncthreads();
    const double nrm = sred[0];
    if (nrm > 0.0)
        for (int r = r0 + tid; r < r1; r += kArnThreads) w[r] = w[r] / nrm;
}

// x += V[:, 0:jm] y  (y: jm FP64 on the device)
__global__ void krylov_update_kernel(int n, int jm, const double *V, const double *y, double *x) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int c = 0; c < jm; ++c) acc = fma(V[(int64_t)c * n + i], y[c], acc);
    x[i] += acc;
}

// ------------------------------------------------------------------------------------
// host driver
// ------------------------------------------------------------------------------------
struct LuWork {
    float *LU = nullptr;
    int ld = 0;
    bool own_LU = true, own_ipiv = true;
    int *ipiv = nullptr, *info = nullptr;
    int *perm = nullptr, *npairs = nullptr;
    int2 *pairs = nullptr;
    unsigned int *bar = nullptr;  // [grid] arrive flags + [1] release
    unsigned int *pu_ctr = nullptr;   // panel_update_kernel arrival counter (zero between launches)
    GridBar gb;
    unsigned int epoch = 1;
    double *r = nullptr, *d = nullptr, *part = nullptr, *scal = nullptr;
    double *tinv = nullptr;       // FP64 inverses of the diagonal blocks (solves only)
    unsigned int *tflags = nullptr, tepoch = 0;
    int n = 0, nb = 0, cl = 16, coop_grid = 0;
    bool cached = false;          // buffers from the LU cache (lu_free keeps them)
    std::vector<void *> extra;    // further device buffers owned by the solve
};

// rows per thread of the register-resident sub-panel for a cluster of cl CTAs (0: too large)
static int sub_rpt(int n, int cl) {
    const int rl = (n + cl - 1) / cl;            // max rows of one CTA (contiguous split)
    for (int r : {1, 2, 4})
        if (rl <= r * kSubThreads) return r;
    return 0;
}

// sub-panel exchange mode (diagnostic hook bf16x_lu_subpanel_bulk; bit 4 = clock64 trace):
// 2 = keys by st.async + winning row read from its CTA (default), 0 = whole records by 9 st.async
// per peer, 1 = whole records by one bulk copy per peer, 3 = keys by plain remote stores polled
// locally.  All four are bit-identical; measured (r06, tools/lu_bulk_probe.py / lu_time.py) the
// factorisation device time is the same within 1 % (26.4 ms at n = 8192): how the keys travel does
// not change the ~1.9 us per column, whose critical path is warp 0's exchange chain itself (r09 ncu:
// the row warps wait at its closing barrier for ~half of all stall samples).
static int g_sub_bulk = 2;
extern "C" void bf16x_lu_subpanel_bulk(int mode) { g_sub_bulk = mode & 7; }   // bit 4: trace

static cudaError_t launch_subpanel(const LuWork &w, int s0, int sw, cudaStream_t st, int2 *pairs, int *npairs, int pc0,
                                   int pc1) {
    const int rpt = sub_rpt(w.n, w.cl);
    if (rpt == 0) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(w.cl);
    cfg.blockDim = dim3(kSubThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = w.cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int bulk = g_sub_bulk;
#define SUBPANEL_LAUNCH(R_, T_) \
    cudaLaunchKernelEx(&cfg, subpanel_kernel<R_, T_>, w.LU, w.ld, w.n, s0, sw, w.ipiv, pairs, npairs, w.info, bulk, pc0, \
                       pc1, w.perm)
    if (bulk & 4) {
        if (rpt == 1) return SUBPANEL_LAUNCH(1, true);
        if (rpt == 2) return SUBPANEL_LAUNCH(2, true);
        return SUBPANEL_LAUNCH(4, true);
    }
    if (rpt == 1) return SUBPANEL_LAUNCH(1, false);
    if (rpt == 2) return SUBPANEL_LAUNCH(2, false);
    return SUBPANEL_LAUNCH(4, false);
#undef SUBPANEL_LAUNCH
}

static int coop_launch(const void *fn, int grid, int threads, void **args, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), args, smem, st);
    if (e != cudaSuccess) {
        set_cuda_error(e, "cooperative launch");
        return BF16X_ERR_CUDA;
    }
    count_launch();
    return BF16X_SUCCESS;
}

// Device buffers of the factorisation state, kept between calls (r10): a getrf / gesv call
// otherwise spent its first milliseconds in cudaMalloc (the n x n copy of A for the solves
// alone is 256 MB at n = 8192) while the GPU idled.  One call at a time owns the cache (try_lock;
// a concurrent call allocates its own buffers as before); every user synchronises before it
// returns, so the buffers are idle between calls.  bf16x_release frees them.
constexpr int kLuSlots = 14;
static std::mutex g_lu_cache_mu;
static void *g_lu_cache[kLuSlots] = {};
static size_t g_lu_cache_cap[kLuSlots] = {};
void lu_release_cache() {
    std::lock_guard<std::mutex> g(g_lu_cache_mu);
    for (int i = 0; i < kLuSlots; ++i) {
        if (g_lu_cache[i]) cudaFree(g_lu_cache[i]);
        g_lu_cache[i] = nullptr;
        g_lu_cache_cap[i] = 0;
    }
}

static void lu_free(LuWork &w) {
    if (!w.cached) {
        if (w.own_LU) cudaFree(w.LU);
        if (w.own_ipiv) cudaFree(w.ipiv);
        cudaFree(w.perm); cudaFree(w.info); cudaFree(w.npairs); cudaFree(w.pairs);
        cudaFree(w.bar); cudaFree(w.pu_ctr); cudaFree(w.r); cudaFree(w.d); cudaFree(w.part); cudaFree(w.scal);
        cudaFree(w.tinv); cudaFree(w.tflags);
    }
    for (void *p : w.extra) cudaFree(p);
    if (w.cached) g_lu_cache_mu.unlock();
    w = LuWork{};
}

static int dev_alloc(void **p, size_t bytes) {
    if (cudaMalloc(p, bytes) != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return BF16X_ERR_ALLOC;
    }
    return BF16X_SUCCESS;
}

// Configure and allocate the factorisation state for order n.  LU/ipiv: caller buffers
// (factor in place) or nullptr (allocated here, ld = n rounded up to 4 floats for the
// 16-byte tile copies of the solves).  solves: also allocate the triangular-solve state.
static int lu_prepare(LuWork &w, int n, int nb, float *LU, int ld, int *ipiv, bool solves, cudaStream_t st) {
    w.n = n;
    w.nb = std::min(nb <= 0 ? 256 : nb, n);
    w.coop_grid = num_sms();
    w.cl = 16;                                   // non-portable cluster size (falls back to 8)
    if (sub_rpt(n, 8) == 0) {
        set_error_msg("LU: n too large for the register-resident sub-panel (n <= 16384)");
        return -1;
    }
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(subpanel_kernel<1, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(subpanel_kernel<2, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(subpanel_kernel<4, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(subpanel_kernel<1, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(subpanel_kernel<2, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(subpanel_kernel<4, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
        cudaFuncSetAttribute(panel_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
        cudaFuncSetAttribute(trsv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsvSmem);
        cudaFuncSetAttribute(diag_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kTinvBlock * sizeof(double) + kTinvBlock * sizeof(float)));
        attr = true;
    }
    int rc = BF16X_SUCCESS;
    w.cached = g_lu_cache_mu.try_lock();            // released by lu_free
    int slot = 0;
    auto alloc = [&](void **p, size_t bytes) {
        const int i = slot++;
        if (rc) return;
        if (!w.cached) {
            rc = dev_alloc(p, bytes);
            return;
        }
        if (g_lu_cache_cap[i] < bytes) {           // grow this slot
            if (g_lu_cache[i]) cudaFree(g_lu_cache[i]);
            g_lu_cache[i] = nullptr;
            g_lu_cache_cap[i] = 0;
            rc = dev_alloc(&g_lu_cache[i], bytes);
            if (rc) return;
            g_lu_cache_cap[i] = bytes;
        }
        *p = g_lu_cache[i];
    };
    w.own_LU = (LU == nullptr);
    w.own_ipiv = (ipiv == nullptr);
    if (LU) {
        w.LU = LU;
        w.ld = ld;
        ++slot;
    } else {
        w.ld = (n + 3) & ~3;
        alloc((void **)&w.LU, sizeof(float) * (size_t)w.ld * n);
    }
    if (ipiv) {
        w.ipiv = ipiv;
        ++slot;
    } else {
        alloc((void **)&w.ipiv, sizeof(int) * n);
    }
    const int nchunk = (n + kResChunk - 1) / kResChunk;
    alloc((void **)&w.perm, sizeof(int) * n);
    alloc((void **)&w.info, sizeof(int));
    const int nmap = (w.nb + kSubW - 1) / kSubW;
    alloc((void **)&w.npairs, sizeof(int) * (size_t)nmap);            // one gather map per sub-panel
    alloc((void **)&w.pairs, sizeof(int2) * (size_t)nmap * 64);
    alloc((void **)&w.bar, sizeof(unsigned int) * ((size_t)w.coop_grid + 1));
    alloc((void **)&w.pu_ctr, sizeof(unsigned int));
    alloc((void **)&w.r, sizeof(double) * n);
    alloc((void **)&w.d, sizeof(double) * n);
    alloc((void **)&w.part, sizeof(double) * (size_t)n * nchunk);
    alloc((void **)&w.scal, sizeof(double) * 4);
    const int nblk = (n + kTB - 1) / kTB;
    if (solves) {
        alloc((void **)&w.tinv, sizeof(double) * 2 * kTinvBlock * nblk);
        alloc((void **)&w.tflags, sizeof(unsigned int) * nblk);
    }
    static_assert(kLuSlots >= 14, "one cache slot per buffer above");
    if (rc) return rc;
    if (solves) cudaMemsetAsync(w.tflags, 0, sizeof(unsigned int) * nblk, st);
    w.gb.arrive = w.bar;
    w.gb.release = w.bar + w.coop_grid;
    cudaMemsetAsync(w.bar, 0, sizeof(unsigned int) * ((size_t)w.coop_grid + 1), st);
    cudaMemsetAsync(w.info, 0, sizeof(int), st);
    cudaMemsetAsync(w.pu_ctr, 0, sizeof(unsigned int), st);
    return BF16X_SUCCESS;
}

// Factor w.LU (order w.n, ld w.ld) in place: P A = L U, ipiv 0-based, perm for the solves.
// Enqueued on st; the zero-pivot column lands in w.info (device).
static double g_lu_host_ms = 0.0;   // host time to enqueue the last factorisation (diagnostic)
static int lu_factor(LuWork &w, int variant, cudaStream_t st) {
    const auto t_host0 = std::chrono::steady_clock::now();
    // Right-looking blocked LU.  Each sub-panel's interchanges are applied at once only inside
    // the panel (the sub-panels and the in-panel updates need them); the whole panel's gather
    // maps are then applied to the columns outside it in one pass (laswp_multi), before the
    // TRSM of U12 and the trailing GEMM.  (A lookahead schedule -- panel p+1 factored while
    // panel p's wide update runs on a second stream -- was measured at equal time: the
    // sub-panel's 16-CTA cluster cannot be placed beside the persistent GEMM, r06.)
    const int n = w.n, nb = w.nb, ld = w.ld;
    int rc = BF16X_SUCCESS;
    auto laswp_multi = [&](int nm, int c0, int c1) {
        if (c1 <= c0) return;
        laswp_multi_kernel<<<(c1 - c0 + 7) / 8, 256, 0, st>>>(w.LU, ld, c0, c1, w.pairs, w.npairs, nm);
        count_launch();
    };
    iota_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, w.perm);
    count_launch();
    for (int j0 = 0; j0 < n && !rc; j0 += nb) {
        const int jb = std::min(nb, n - j0), j1 = j0 + jb;
        int nm = 0;
        for (int s0 = j0; s0 < j1 && !rc; s0 += kSubW, ++nm) {
            const int sw = std::min(kSubW, j1 - s0);
            int2 *pr = w.pairs + 64 * nm;
            int *np = w.npairs + nm;
            // (1) sub-panel factorisation on one cluster (rows in registers, RPT per thread), then
            //     (2) its interchanges inside the panel and on the row permutation (fused, r10)
            cudaError_t e = launch_subpanel(w, s0, sw, st, pr, np, j0, j1);
            if (e != cudaSuccess && w.cl == 16) {    // 16-CTA clusters unavailable: use 8
                cudaGetLastError();
                w.cl = 8;
                e = launch_subpanel(w, s0, sw, st, pr, np, j0, j1);
            }
            if (e != cudaSuccess) {
                set_cuda_error(e, "subpanel launch");
                rc = BF16X_ERR_CUDA;
                break;
            }
            count_launch();
            // (3) TRSM + rank-sw update of the rest of the panel
            const int c1 = s0 + sw;
            if (c1 < j1) {
                const size_t smem = panel_update_smem(j1 - c1);
                panel_update_kernel<<<(n - c1 + kUpdRows - 1) / kUpdRows, 256, smem, st>>>(w.LU, ld, n, s0, sw, c1, j1,
                                                                                          w.pu_ctr);
                count_launch();
            }
            rc = check_launch("panel");
        }
        if (rc) break;
        // the panel's interchanges on the columns outside it
        laswp_multi(nm, 0, j0);
        laswp_multi(nm, j1, n);
        const int rest = n - j1;
        if (rest > 0) {
            trsm_kernel<<<(rest + kTrsmCols - 1) / kTrsmCols, 256, trsm_smem(jb), st>>>(w.LU, ld, j0, jb, j1, rest);
            count_launch();
            rc = check_launch("trsm");
            if (rc) break;
            // A22 <- -L21 U12 + A22 : the cubic work, in the split GEMM
            rc = gemm_core(rest, rest, jb, -1.0f, w.LU + (int64_t)j0 * ld + j1, ld, w.LU + (int64_t)j1 * ld + j0, ld,
                           1.0f, w.LU + (int64_t)j1 * ld + j1, ld, variant, kFlagRedAdd, nullptr, 0, 0, nullptr, 0, 0, nullptr,
                           nullptr, 0, st, 0);
        }
    }
    if (rc == BF16X_SUCCESS) {
        if (w.tinv) {
            diag_inverse_kernel<<<dim3((n + kTB - 1) / kTB, 2), kTB, kTinvBlock * (sizeof(double) + sizeof(float)),
                                  st>>>(w.LU, ld, n, w.tinv);
            count_launch();
        }
        rc = check_launch("lu");
    }
    g_lu_host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
    return rc;
}

// Wait for the factorisation; *info = first zero-pivot column (1-based) or 0.
static int lu_sync_info(LuWork &w, cudaStream_t st, int *info) {
    *info = 0;
    cudaMemcpyAsync(info, w.info, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("lu sync");
    return *info ? BF16X_ERR_SINGULAR : BF16X_SUCCESS;
}

static int solve_with_factors(LuWork &w, int n, const double *v, double *out, int coop_grid, cudaStream_t st) {
    // out = U^-1 L^-1 P v
    gather_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, w.perm, v, out);
    count_launch();
    int ld = w.ld, lower = 1;
    const float *LU = w.LU;
    const double *ti = w.tinv;
    unsigned int *fl = w.tflags;
    double *y = out;
    unsigned int ep = ++w.tepoch;
    void *args[] = {(void *)&LU, (void *)&ld, (void *)&n, (void *)&y, (void *)&lower, (void *)&ti, (void *)&fl,
                    (void *)&ep};
    const int grid = std::min((n + kTB - 1) / kTB, coop_grid);
    int rc = coop_launch((const void *)trsv_kernel, grid, kTrsvThreads, args, kTrsvSmem, st);
    if (rc) return rc;
    lower = 0;
    ep = ++w.tepoch;
    return coop_launch((const void *)trsv_kernel, grid, kTrsvThreads, args, kTrsvSmem, st);
}

// r = b - A x (b != nullptr), r = A x (b == nullptr), or row abs sums (absval).
static void residual(const float *A, int lda, int n, const double *x, const double *b, double *r, double *part,
                     int absval, cudaStream_t st) {
    const int nchunk = (n + kResChunk - 1) / kResChunk;
    dim3 grid((n + kResRows - 1) / kResRows, nchunk);
    residual_partial_kernel<<<grid, kResRows, 0, st>>>(A, lda, n, x, part, absval);
    residual_final_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, nchunk, part, b, r);
    count_launch(2);
}

static double inf_norm_A(LuWork &w, const float *A, int lda, int n, cudaStream_t st) {
    residual(A, lda, n, nullptr, nullptr, w.r, w.part, 1, st);
    absmax_kernel<<<1, 256, 0, st>>>(n, w.r, w.scal + 2);
    count_launch();
    double anrm = 0.0;
    cudaMemcpyAsync(&anrm, w.scal + 2, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return anrm;
}

// ||b - A x||_inf and ||x||_inf (synchronises).
static int residual_norms(LuWork &w, const float *A, int lda, int n, const double *x, const double *b,
                          cudaStream_t st, double *rn, double *xn) {
    residual(A, lda, n, x, b, w.r, w.part, 0, st);
    absmax_kernel<<<1, 256, 0, st>>>(n, w.r, w.scal);
    absmax_kernel<<<1, 256, 0, st>>>(n, x, w.scal + 1);
    count_launch(2);
    double h[2];
    cudaMemcpyAsync(h, w.scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("ir sync");
    *rn = h[0];
    *xn = h[1];
    return BF16X_SUCCESS;
}

static int check_common(int n, int lda, int variant) {
    if (n < 0) return -1;
    if (lda < (n > 1 ? n : 1)) return -3;
    if (variant != 3 && variant != 6 && variant != 9) return -6;
    return BF16X_SUCCESS;
}

}  // namespace bf16x

using namespace bf16x;

extern "C" int bf16x_getrf(int n, float *A, int lda, int *ipiv, int variant, int nb, int *info) {
    if (n < 0) return -1;
    if (n > 0 && !A) return -2;
    if (lda < (n > 1 ? n : 1)) return -3;
    if (n > 0 && !ipiv) return -4;
    if (variant != 1 && variant != 3 && variant != 5 && variant != 6 && variant != 7 && variant != 8 && variant != 9)
        return -5;
    if (info) *info = 0;
    int rc = arch_ok();
    if (rc || n == 0) return rc;
    cudaStream_t st = current_stream();
    LuWork w;
    rc = lu_prepare(w, n, nb, A, lda, ipiv, false, st);
    if (!rc) rc = lu_factor(w, variant, st);
    int inf = 0;
    if (!rc) rc = lu_sync_info(w, st, &inf);
    if (info) *info = inf;
    lu_free(w);
    return rc;
}

// ||b||_inf of a device vector (the relative-residual test of a caller tolerance, R14)
static double host_inf_norm(const double *b, int n, cudaStream_t st) {
    std::vector<double> h((size_t)n);
    if (cudaMemcpyAsync(h.data(), b, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
        cudaGetLastError();
        return -1.0;
    }
    double m = 0.0;
    for (double v : h) m = std::max(m, std::fabs(v));
    return m;
}

// the stopping threshold on ||r||_inf: the caller's relative tolerance tol * ||b||_inf (tol > 0:
// the paper's "residual tolerance of cond(A)*eps", with tol = cond(A) * 2^-53), else
// LAPACK dsgesv's sqrt(n) ||x||_inf ||A||_inf 2^-53 (R14)
static double ir_threshold(double tol, double bnrm, int n, double xn, double anrm) {
    return tol > 0.0 ? tol * bnrm : std::sqrt((double)n) * xn * anrm * std::ldexp(1.0, -53);
}

extern "C" int bf16x_gesv_ir(int n, const float *A, int lda, const double *b, double *x, int variant, int nb,
                             double tol, int max_iter, double *residual_history, bf16x_ir_report *report) {
    if (!report) return -11;
    if (tol != tol) return -8;
    *report = bf16x_ir_report{};
    int rc = check_common(n, lda, variant);
    if (rc) return rc;
    rc = arch_ok();
    if (rc) return rc;
    if (n == 0) {
        report->converged = 1;
        return BF16X_SUCCESS;
    }
    if (max_iter <= 0) max_iter = 30;
    cudaStream_t st = current_stream();
    LuWork w;
    rc = lu_prepare(w, n, nb, nullptr, 0, nullptr, true, st);
    if (rc) {
        lu_free(w);
        return rc;
    }
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
    cudaEventRecord(e0, st);
    copy_matrix_kernel<<<num_sms() * 8, 256, 0, st>>>(n, A, lda, w.LU, w.ld);
    count_launch();
    rc = lu_factor(w, variant, st);
    cudaEventRecord(e1, st);
    int info = 0;
    if (rc == BF16X_SUCCESS) rc = lu_sync_info(w, st, &info);
    report->info = info;

    // ---------------- refinement ----------------
    if (rc == BF16X_SUCCESS) {
        const double anrm = inf_norm_A(w, A, lda, n, st);
        const double bnrm = tol > 0.0 ? host_inf_norm(b, n, st) : 0.0;
        rc = solve_with_factors(w, n, b, x, w.coop_grid, st);
        std::vector<double> hist;
        int it = 0;
        bool converged = false;
        double rn = 0.0, xn = 0.0;
        for (; rc == BF16X_SUCCESS; ++it) {
            rc = residual_norms(w, A, lda, n, x, b, st, &rn, &xn);
            if (rc) break;
            hist.push_back(rn);
            report->tol = ir_threshold(tol, bnrm, n, xn, anrm);
            if (rn <= report->tol) {
                converged = true;
                break;
            }
            if (it >= max_iter) break;
            if (hist.size() >= 4 && hist.back() > 0.5 * hist[hist.size() - 4]) break;  // stagnation
            rc = solve_with_factors(w, n, w.r, w.d, w.coop_grid, st);
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
    lu_free(w);
    return rc;
}

extern "C" int bf16x_gesv_gmres_ir(int n, const float *A, int lda, const double *b, double *x, int variant, int nb,
                                   int restart, double inner_tol, double tol, int max_iter, double *residual_history,
                                   bf16x_ir_report *report) {
    if (!report) return -13;
    *report = bf16x_ir_report{};
    int rc = check_common(n, lda, variant);
    if (rc) return rc;
    if (inner_tol < 0.0 || inner_tol != inner_tol) return -9;
    if (tol != tol) return -10;
    rc = arch_ok();
    if (rc) return rc;
    if (n == 0) {
        report->converged = 1;
        return BF16X_SUCCESS;
    }
    if (max_iter <= 0) max_iter = 30;
    if (inner_tol == 0.0) inner_tol = 1e-10;
    const int m = std::min(std::min(restart <= 0 ? 200 : restart, n), 8190);   // shared-memory projections
    cudaStream_t st = current_stream();
    LuWork w;
    rc = lu_prepare(w, n, nb, nullptr, 0, nullptr, true, st);
    double *V = nullptr, *part = nullptr, *hcol = nullptr, *ydev = nullptr, *t = nullptr;
    const int pstride = m + 2;
    if (!rc) rc = dev_alloc((void **)&V, sizeof(double) * (size_t)n * (m + 1));
    if (!rc) rc = dev_alloc((void **)&part, sizeof(double) * 3 * (size_t)w.coop_grid * pstride);
    if (!rc) rc = dev_alloc((void **)&hcol, sizeof(double) * pstride);
    if (!rc) rc = dev_alloc((void **)&ydev, sizeof(double) * (m + 1));
    if (!rc) rc = dev_alloc((void **)&t, sizeof(double) * n);
    for (void *p : {(void *)V, (void *)part, (void *)hcol, (void *)ydev, (void *)t}) w.extra.push_back(p);
    if (rc) {
        lu_free(w);
        return rc;
    }
    {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(arnoldi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
            attr = true;
        }
    }
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
    cudaEventRecord(e0, st);
    copy_matrix_kernel<<<num_sms() * 8, 256, 0, st>>>(n, A, lda, w.LU, w.ld);
    count_launch();
    rc = lu_factor(w, variant, st);
    cudaEventRecord(e1, st);
    int info = 0;
    if (rc == BF16X_SUCCESS) rc = lu_sync_info(w, st, &info);
    report->info = info;

    auto arnoldi = [&](int j) -> int {
        double *Vp = V, *pp = part, *hp = hcol;
        int nn = n, jj = j, ps = pstride;
        GridBar gb = w.gb;
        unsigned int ep = w.epoch;
        void *args[] = {(void *)&Vp, (void *)&nn, (void *)&jj, (void *)&pp, (void *)&ps, (void *)&hp, (void *)&gb,
                        (void *)&ep};
        const int rc2 = coop_launch((const void *)arnoldi_kernel, w.coop_grid, kArnThreads, args,
                                    (size_t)pstride * sizeof(double), st);
        w.epoch += (j >= 0) ? 3 : 1;
        return rc2;
    };

    // ---------------- GMRES-IR (reading R25) ----------------
    if (rc == BF16X_SUCCESS) {
        const double anrm = inf_norm_A(w, A, lda, n, st);
        const double bnrm = tol > 0.0 ? host_inf_norm(b, n, st) : 0.0;
        cudaMemsetAsync(x, 0, sizeof(double) * n, st);
        std::vector<double> hist, H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m), hc(m + 2);
        int it = 0, inner = 0;
        bool converged = false;
        double rn = 0.0, xn = 0.0;
        for (; rc == BF16X_SUCCESS; ++it) {
            rc = residual_norms(w, A, lda, n, x, b, st, &rn, &xn);
            if (rc) break;
            hist.push_back(rn);
            report->tol = ir_threshold(tol, bnrm, n, xn, anrm);
            if (rn <= report->tol) {
                converged = true;
                break;
            }
            if (it >= max_iter) break;
            if (hist.size() >= 4 && hist.back() > 0.5 * hist[hist.size() - 4]) break;  // stagnation
            // one GMRES cycle on M^-1 A d = M^-1 r, d0 = 0
            rc = solve_with_factors(w, n, w.r, V, w.coop_grid, st);
            if (!rc) rc = arnoldi(-1);
            double beta = 0.0;
            if (!rc) {
                cudaMemcpyAsync(&beta, hcol, sizeof(double), cudaMemcpyDeviceToHost, st);
                if (cudaStreamSynchronize(st) != cudaSuccess) rc = check_launch("gmres sync");
            }
            if (rc || beta == 0.0) break;
            std::fill(g.begin(), g.end(), 0.0);
            g[0] = beta;
            int jm = 0;
            for (int j = 0; j < m && !rc; ++j) {
                // w = M^-1 A v_j into column j+1, then CGS2 + normalisation
                residual(A, lda, n, V + (int64_t)j * n, nullptr, t, w.part, 0, st);
                rc = solve_with_factors(w, n, t, V + (int64_t)(j + 1) * n, w.coop_grid, st);
                if (!rc) rc = arnoldi(j);
                if (!rc) {
                    cudaMemcpyAsync(hc.data(), hcol, sizeof(double) * (j + 2), cudaMemcpyDeviceToHost, st);
                    if (cudaStreamSynchronize(st) != cudaSuccess) rc = check_launch("gmres sync");
                }
                if (rc) break;
                // Givens rotations on Hessenberg column j (host, FP64), as the oracle's template
                double *Hc = H.data() + (size_t)j * (m + 1);      // column j, rows 0..j+1
                for (int i = 0; i <= j + 1; ++i) Hc[i] = hc[i];
                const double hnext = hc[j + 1];
                for (int i = 0; i < j; ++i) {
                    const double a = cs[i] * Hc[i] + sn[i] * Hc[i + 1];
                    Hc[i + 1] = -sn[i] * Hc[i] + cs[i] * Hc[i + 1];
                    Hc[i] = a;
                }
                const double dd = std::hypot(Hc[j], Hc[j + 1]);
                cs[j] = Hc[j] / dd;
                sn[j] = Hc[j + 1] / dd;
                Hc[j] = dd;
                Hc[j + 1] = 0.0;
                g[j + 1] = -sn[j] * g[j];
                g[j] = cs[j] * g[j];
                ++inner;
                jm = j + 1;
                if (std::fabs(g[j + 1]) <= inner_tol * beta || hnext == 0.0) break;
            }
            if (rc) break;
            // least squares: H(0:jm, 0:jm) y = g, then x += V y
            for (int i = jm - 1; i >= 0; --i) {
                double s = g[i];
                for (int c = i + 1; c < jm; ++c) s -= H[(size_t)c * (m + 1) + i] * y[c];
                y[i] = s / H[(size_t)i * (m + 1) + i];
            }
            cudaMemcpyAsync(ydev, y.data(), sizeof(double) * jm, cudaMemcpyHostToDevice, st);
            krylov_update_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, jm, V, ydev, x);
            count_launch();
            rc = check_launch("gmres update");
        }
        report->converged = converged ? 1 : 0;
        report->iterations = it;
        report->inner_iterations = inner;
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
    lu_free(w);
    return rc;
}

extern "C" double bf16x_lu_host_ms(void) { return g_lu_host_ms; }   // diagnostic hook
