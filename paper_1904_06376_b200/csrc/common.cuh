// common.cuh -- device helpers shared by the sm_100a kernels of libbf16x.so:
// the BF16 split arithmetic, mbarrier / TMA / tcgen05 PTX wrappers, and
// host-side status plumbing.  Product code only; the oracle shares nothing with it.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "bf16x.h"

namespace bf16x {

// ----------------------------------------------------------------------------------
// host status plumbing
// ----------------------------------------------------------------------------------
void set_cuda_error(cudaError_t e, const char *where);
void set_error_msg(const char *msg);
int check_launch(const char *where);     // BF16X_ERR_CUDA on a pending launch error
void count_launch(uint64_t n = 1);
cudaStream_t current_stream();
int arch_ok();                           // BF16X_SUCCESS iff device is sm_100

// ----------------------------------------------------------------------------------
// (B16) conversion, P:177-179 (section II-A), readings R1/R3/R4:
// round to nearest even on the FP32 bit pattern, finite overflow saturates to the
// largest finite BF16, NaN -> 0x7FC0.  Implemented with the rounding-bias identity
//     rne16(u) = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
// which, for the sign-magnitude encoding, rounds the magnitude to the nearest
// 16-bit pattern with ties going to the even pattern.
// ----------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t rne_sat_bf16(float x) {
    uint32_t u = __float_as_uint(x);
    if ((u & 0x7F800000u) == 0x7F800000u)               // Inf / NaN
        return (u & 0x007FFFFFu) ? 0x7FC0u : (u >> 16);
    uint32_t r = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
    return ((r & 0x7FFFu) == 0x7F80u) ? r - 1u : r;     // saturate +-Inf -> +-0x7F7F
}

__device__ __forceinline__ float bf16_bits_to_float(uint32_t b) { return __uint_as_float(b << 16); }

// The 3-way split of P:180-184: b0 = (B16)x, r1 = x - b0 (FP32), b1 = (B16)r1,
// r2 = r1 - b1 (FP32, left to right, R5), b2 = (B16)r2.  Non-finite x -> (b0, +0, +0).
// Both subtractions are exact in FP32 for finite x (no FTZ: nvcc default -ftz=false).
struct Split3 { uint32_t b0, b1, b2; };
__device__ __forceinline__ Split3 split3(float x) {
    Split3 s;
    s.b0 = rne_sat_bf16(x);
    if (!isfinite(x)) { s.b1 = 0u; s.b2 = 0u; return s; }
    float r1 = __fsub_rn(x, bf16_bits_to_float(s.b0));
    s.b1 = rne_sat_bf16(r1);
    float r2 = __fsub_rn(r1, bf16_bits_to_float(s.b1));
    s.b2 = rne_sat_bf16(r2);
    return s;
}

// N2 scaled pieces (R29): the residuals are multiplied by 2^8 (exact) before each
// rounding, b1' = (B16)(2^8 (x - b0)), b2' = (B16)(2^8 (2^8 (x - b0) - b1')), so every piece
// stays at the magnitude of x and x = b0 + 2^-8 b1' + 2^-16 b2' for every finite x.
__device__ __forceinline__ Split3 split3_scaled(float x) {
    Split3 s;
    s.b0 = rne_sat_bf16(x);
    if (!isfinite(x)) { s.b1 = 0u; s.b2 = 0u; return s; }
    float s1 = __fmul_rn(__fsub_rn(x, bf16_bits_to_float(s.b0)), 256.f);
    s.b1 = rne_sat_bf16(s1);
    float s2 = __fmul_rn(__fsub_rn(s1, bf16_bits_to_float(s.b1)), 256.f);
    s.b2 = rne_sat_bf16(s2);
    return s;
}
template <bool SC>
__device__ __forceinline__ Split3 split3_t(float x) {
    if constexpr (SC) return split3_scaled(x);
    else return split3(x);
}
// residual scaling of the fast path: 2^8 for scaled pieces (exact: |residual| <= 2^119 below
// the b0-overflow band), identity otherwise
template <bool SC>
__device__ __forceinline__ float res_scale(float r) {
    if constexpr (SC) return __fmul_rn(r, 256.f);
    else return r;
}

// Hardware fast path of the split for two values below the b0-overflow band (shared by the
// split pre-pass and the GEMM's in-kernel transform): cvt.rn.bf16x2.f32 is IEEE RNE on two
// values, the FP32 residual subtractions are exact; anything else takes split3.
__device__ __forceinline__ uint32_t cvt_bf16x2(float hi, float lo) {
    uint32_t d;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    return d;
}

__device__ __forceinline__ bool regular(float x) { return (__float_as_uint(x) & 0x7FFFFFFFu) < 0x7F7F8000u; }

// Fast path only (both values known to be below the b0-overflow band): branch-free, so many
// pairs' dependency chains interleave.
template <int NP, bool SC = false>
__device__ __forceinline__ void split_pair_fast(float lo, float hi, uint32_t (&p)[3]) {
    const uint32_t a = cvt_bf16x2(hi, lo);
    p[0] = a;
    if constexpr (NP >= 2) {
        const float r1lo = res_scale<SC>(__fsub_rn(lo, __uint_as_float(a << 16)));
        const float r1hi = res_scale<SC>(__fsub_rn(hi, __uint_as_float(a & 0xFFFF0000u)));
        const uint32_t b = cvt_bf16x2(r1hi, r1lo);
        p[1] = b;
        if constexpr (NP >= 3) {
            const float r2lo = res_scale<SC>(__fsub_rn(r1lo, __uint_as_float(b << 16)));
            const float r2hi = res_scale<SC>(__fsub_rn(r1hi, __uint_as_float(b & 0xFFFF0000u)));
            p[2] = cvt_bf16x2(r2hi, r2lo);
        }
    }
}

// Split two values; packs piece q of (lo, hi) as (hi << 16) | lo in p[q].
template <int NP, bool SC = false>
__device__ __forceinline__ void split_pair(float lo, float hi, uint32_t (&p)[3]) {
    if (regular(lo) && regular(hi)) {
        split_pair_fast<NP, SC>(lo, hi, p);
    } else {
        const Split3 a = split3_t<SC>(lo), b = split3_t<SC>(hi);
        p[0] = a.b0 | (b.b0 << 16);
        p[1] = a.b1 | (b.b1 << 16);
        p[2] = a.b2 | (b.b2 << 16);
    }
}


// ----------------------------------------------------------------------------------
// PTX wrappers: shared-memory addresses, mbarrier, TMA, tcgen05
// ----------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
// arrive on the barrier at the same smem offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(cta)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int *p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// explicit shared-space accesses (32-bit shared addresses): keep the transform's loads and
// stores on the LDS/STS path instead of generic addressing
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds_f32x4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u32x4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w));
}

// 2D TMA tile load into this CTA's shared memory, completion counted on `bar` (local).
__device__ __forceinline__ void tma_load_2d(void *smem_dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// arrive with release semantics at cluster scope on the barrier at the same smem offset in
// CTA `cta` (publishes this thread's prior shared-memory writes to that CTA's waiters)
__device__ __forceinline__ void mbar_arrive_release_cluster(uint64_t *bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(cta)
        : "memory");
}

// 3D TMA tile load into this CTA's shared memory, completion counted on `bar`.
__device__ __forceinline__ void tma_load_3d(void *smem_dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                            int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// 2-CTA form: data lands in this CTA's smem, the byte count is signalled on the
// barrier at the same offset in the leader (even) CTA of the pair.
__device__ __forceinline__ void tma_load_3d_2sm(void *smem_dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                                int c1, int c2) {
    uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(b), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// 2-CTA multicast form: the box lands at the same smem offset in every CTA of `mask`; each
// destination signals the barrier at this offset in its pair's leader (even) CTA.
__device__ __forceinline__ void tma_load_3d_2sm_mc(void *smem_dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                                   int c1, int c2, uint16_t mask) {
    uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(b), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
        : "memory");
}

// 2D TMA tensor store / element-wise add (the add in L2) of a shared-memory box into global
// memory, tracked by this thread's bulk async-groups (bulk_commit / bulk_wait_read / bulk_wait).
// Elements of the box outside the tensor are not written.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, const void *smem_src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap *map, const void *smem_src, int c0, int c1) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N of this thread's committed bulk groups still read shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
// wait until at most N of this thread's committed bulk groups are incomplete
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (TMA reads them)
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- tcgen05 ----
template <int CG>
__device__ __forceinline__ void tmem_alloc(uint32_t *smem_result, uint32_t ncols) {
    if constexpr (CG == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    if constexpr (CG == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
    else
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, BF16 inputs, FP32 accumulate (kind::f16).
template <int CG>
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    if constexpr (CG == 1)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Warp-uniform variants: every lane of the warp executes the call, one elected lane issues.
// (elect.sync with a full mask always elects the same lane, so the commits below track the
// MMAs issued by that lane.)
template <int CG>
__device__ __forceinline__ void umma_bf16_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
    if constexpr (CG == 1)
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
    else
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Accumulating MMA that first scales the accumulator by 2^-8 (tcgen05.mma scale-input-d = 8:
// D = A*B + D * 2^-8), used on the move to the next larger bin with scaled pieces (R29).
template <int CG>
__device__ __forceinline__ void umma_bf16_elect_sc8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
    if constexpr (CG == 1)
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, 1, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p, 8;\n\t}" ::"r"(d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc));
    else
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, 1, 1;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p, 8;\n\t}" ::"r"(d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc));
}
template <int CG>
__device__ __forceinline__ void umma_commit_elect(uint64_t *bar) {
    if constexpr (CG == 1)
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                smem_u32(bar)),
            "h"((uint16_t)3)
            : "memory");
}

// 2-CTA commit arriving on the barrier at this offset in every CTA of `mask`.
__device__ __forceinline__ void umma_commit2_mask_elect(uint64_t *bar, uint16_t mask) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// Make `bar` track completion of all prior tcgen05 async ops of this thread.
template <int CG>
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    if constexpr (CG == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(bar))
                     : "memory");
    else  // signal the barrier at this offset in both CTAs of the pair
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(bar)),
            "h"((uint16_t)3)
            : "memory");
}

// 32 lanes x 32 consecutive 32-bit TMEM columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t *r = reinterpret_cast<uint32_t *>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
// 32 lanes x 16 consecutive 32-bit TMEM columns -> 16 registers per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t *r = reinterpret_cast<uint32_t *>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor (tcgen05 "smem descriptor"), K-major operand tile
// with the given swizzle: start address and stride byte offset in 16-byte units,
// leading byte offset 1 (unused for swizzled K-major), version 1 (sm_100).
// layout: 2 = SWIZZLE_128B, 4 = SWIZZLE_64B, 6 = SWIZZLE_32B.
__device__ __forceinline__ uint64_t smem_desc_kmajor(uint32_t saddr, uint32_t sbo_bytes, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;                              // LBO (ignored for swizzled K-major)
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;    // SBO
    d |= (uint64_t)1u << 46;                              // version = 1
    d |= (uint64_t)(layout & 7u) << 61;
    return d;
}

// MN-major operand, 128-byte swizzle (canonical ((64 elements, n), (8 rows, k)) atoms of 1 KB):
// lbo_bytes = stride between 64-element MN atoms, sbo_bytes = stride between 8-row K groups
__device__ __forceinline__ uint64_t smem_desc_mn128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;    // LBO
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;    // SBO
    d |= (uint64_t)1u << 46;                              // version = 1
    d |= (uint64_t)2u << 61;                              // SWIZZLE_128B
    return d;
}

// Instruction descriptor for kind::f16: BF16 x BF16 -> FP32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
    return (1u << 4)                          // c_format = F32
         | (1u << 7)                          // a_format = BF16
         | (1u << 10)                         // b_format = BF16
         | ((uint32_t)(N >> 3) << 17)         // N / 8
         | ((uint32_t)(M >> 4) << 24);        // M / 16
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <uint32_t R>
__device__ __forceinline__ void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R)); }
template <uint32_t R>
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R)); }

}  // namespace bf16x
