// l2f_tcgen05.cuh -- minimal inline-PTX wrappers for sm_100a 5th-gen tensor cores:
// UMMA shared-memory descriptors, tcgen05.mma (kind::f16, cta_group::1), tcgen05.commit ->
// mbarrier, TMEM alloc / ld, and the proxy / thread-sync fences that order them.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

namespace l2f {
namespace tc {

// Debug build: a TMEM access of `ncols` columns at taddr stays inside the 512 allocated columns
// and addresses the 32-lane quadrant of the calling warp (tcgen05.ld/st 32x32b access rule).
#ifdef L2F_DEBUG_CHECKS
#define L2F_TMEM_CHECK(taddr, ncols)                                                             \
    L2F_CHECK(((taddr) & 0xFFFFu) + (ncols) <= 512u && ((taddr) >> 16) == 32u * ((threadIdx.x >> 5) & 3u), \
              "tmem address")
#else
#define L2F_TMEM_CHECK(taddr, ncols) \
    do {                             \
    } while (0)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory matrix descriptor, SWIZZLE_NONE ("interleaved" canonical layout):
//  bits [0,14) start address >> 4, [16,30) leading-dimension byte offset >> 4,
//  [32,46) stride-dimension byte offset >> 4, [46,48) version = 1 (sm_100),
//  [49,52) base offset = 0, [52] LBO mode = 0, [61,64) layout = 0 (no swizzle).
// K-major operand: 8x16-byte core matrices (8 rows x 8 fp16 of K); LBO = byte stride
// between the two K halves of a K16 slice, SBO = byte stride between 8-row groups.
// MN-major operand: core matrix = 8 K-rows x 8 fp16 of M/N; LBO = stride between 8-K-row
// groups, SBO = stride between 8-wide M/N groups.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// Instruction descriptor for kind::f16: A/B fp16, D fp32, dense.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn_major, int b_mn_major)
{
    return (1u << 4)                        // D format F32
           | (0u << 7) | (0u << 10)         // A, B format F16
           | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16)
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// A operand from tensor memory (row m = TMEM lane m, K packed two fp16 per 32-bit column).
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Warp-converged issue: all 32 lanes execute the asm, elect.sync picks the one lane that
// issues (no divergent single-thread region around the MMA sequence).
__device__ __forceinline__ void mma_f16_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_f16_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// Layer-1 MMAs of one 128-row tile in one elected issue: the observation part (K = 32: two
// K16 steps, A at +0 / +256 descriptor units, B at +0 / +128) then kHist history K16 steps
// (A at +512 + 256 j, B at + 16 j, MN-major B), accumulating into d.  One elect.sync for the
// whole sequence; every descriptor is its base plus an immediate.
template <int kHist>
__device__ __forceinline__ void issue_l1_elect(uint32_t d, uint64_t a, uint64_t bo, uint64_t bh, uint32_t idesc,
                                               uint32_t idesc_bmn)
{
    static_assert(kHist == 8, "specialised for N_H = 32");
    asm volatile(
        "{\n\t.reg .pred e, p0, p1;\n\t.reg .b64 ra, rb;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p0, %5, %5;\n\t"
        "setp.eq.b32 p1, %5, %5;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p0;\n\t"
        "add.s64 ra, %1, 256;\n\tadd.s64 rb, %2, 128;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %4, p1;\n\t"
        "add.s64 ra, %1, 512;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, %3, %5, p1;\n\t"
        "add.s64 ra, %1, 768;\n\tadd.s64 rb, %3, 16;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %5, p1;\n\t"
        "add.s64 ra, %1, 1024;\n\tadd.s64 rb, %3, 32;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %5, p1;\n\t"
        "add.s64 ra, %1, 1280;\n\tadd.s64 rb, %3, 48;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %5, p1;\n\t"
        "add.s64 ra, %1, 1536;\n\tadd.s64 rb, %3, 64;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %5, p1;\n\t"
        "add.s64 ra, %1, 1792;\n\tadd.s64 rb, %3, 80;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %5, p1;\n\t"
        "add.s64 ra, %1, 2048;\n\tadd.s64 rb, %3, 96;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %5, p1;\n\t"
        "add.s64 ra, %1, 2304;\n\tadd.s64 rb, %3, 112;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %5, p1;\n\t}\n" ::"r"(d),
        "l"(a), "l"(bo), "l"(bh), "r"(idesc), "r"(idesc_bmn));
}

// Layers 2 / 3 of one tile in one elected issue: 5 K16 steps with A from TMEM columns
// a_tmem + 8 j and B at + b_step j descriptor units (K = 80: 64 hidden + the ones column).
template <int kBStep>
__device__ __forceinline__ void issue_ts5_elect(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc)
{
    asm volatile(
        "{\n\t.reg .pred e, p0, p1;\n\t.reg .b64 rb;\n\t.reg .b32 ra;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p0, %3, %3;\n\t"
        "setp.eq.b32 p1, %3, %3;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n\t"
        "add.s32 ra, %1, 8;\n\tadd.s64 rb, %2, %4;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, p1;\n\t"
        "add.s32 ra, %1, 16;\n\tadd.s64 rb, %2, %5;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, p1;\n\t"
        "add.s32 ra, %1, 24;\n\tadd.s64 rb, %2, %6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, p1;\n\t"
        "add.s32 ra, %1, 32;\n\tadd.s64 rb, %2, %7;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, p1;\n\t}\n" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "n"(kBStep), "n"(2 * kBStep), "n"(3 * kBStep), "n"(4 * kBStep));
}

__device__ __forceinline__ void commit_elect(uint32_t mbar_saddr)
{
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(mbar_saddr)
        : "memory");
}

// All prior tcgen05.mma of this thread arrive (once) on the mbarrier when complete.
__device__ __forceinline__ void commit(uint32_t mbar_saddr)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_saddr)
                 : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy smem writes -> visible to the async proxy (tensor core operand reads)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint32_t mbar_saddr, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar_saddr), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t mbar_saddr)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(mbar_saddr) : "memory");
}

#ifndef L2F_MBAR_SUSPEND_NS
#define L2F_MBAR_SUSPEND_NS 100000  // try_wait suspend-time hint (ns): sleep until the phase flips instead of polling
#endif
__device__ __forceinline__ void mbar_wait(uint32_t mbar_saddr, uint32_t parity)
{
#ifdef L2F_DEBUG_CHECKS
    // bounded wait: a phase that never completes (lost commit, wrong parity) traps instead of hanging
    uint32_t done = 0;
    for (uint32_t it = 0; it < (1u << 24) && !done; ++it)
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(mbar_saddr), "r"(parity)
            : "memory");
    L2F_CHECK(done, "mbarrier wait timed out");
    return;
#endif
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(mbar_saddr),
        "r"(parity), "n"(L2F_MBAR_SUSPEND_NS)
        : "memory");
}

// Named barrier over `count` threads (ids 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t count)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void named_arrive(uint32_t id, uint32_t count)
{
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// TMEM allocation by one full warp; the base address is written to smem.
__device__ __forceinline__ void tmem_alloc(uint32_t dst_saddr, uint32_t ncols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_saddr), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 lanes x 32-bit, 16 consecutive columns: thread t of the warp gets row (lane base + t).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16])
{
    L2F_TMEM_CHECK(taddr, 16u);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4])
{
    L2F_TMEM_CHECK(taddr, 4u);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 32-bit stores of consecutive columns (thread t -> its own lane).
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v, int off)
{
    L2F_TMEM_CHECK(taddr, 8u);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "f"(v[off + 0]), "f"(v[off + 1]), "f"(v[off + 2]), "f"(v[off + 3]), "f"(v[off + 4]),
                 "f"(v[off + 5]), "f"(v[off + 6]), "f"(v[off + 7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16])
{
    L2F_TMEM_CHECK(taddr, 16u);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st8u(uint32_t taddr, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t a4, uint32_t a5, uint32_t a6, uint32_t a7)
{
    L2F_TMEM_CHECK(taddr, 8u);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(a0),
                 "r"(a1), "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7)
                 : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const float (&v)[4])
{
    L2F_TMEM_CHECK(taddr, 4u);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3])
                 : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, float a, float b)
{
    L2F_TMEM_CHECK(taddr, 2u);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "f"(a), "f"(b) : "memory");
}

__device__ __forceinline__ void sts128(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
// The same 16 bytes at saddr + k * stride for k = 0..15, as 32 volatile 8-byte stores of one
// register pair (ptxas otherwise fuses them into 16-byte stores and copies the quad for each).
template <uint32_t kStride>
__device__ __forceinline__ void sts128_x16(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
#define L2F_ST16(k) "st.volatile.shared.v2.b32 [%0+" #k "*%5], {%1,%2};\n\tst.volatile.shared.v2.b32 [%0+" #k "*%5+8], {%3,%4};\n\t"
    asm volatile(L2F_ST16(0) L2F_ST16(1) L2F_ST16(2) L2F_ST16(3) L2F_ST16(4) L2F_ST16(5) L2F_ST16(6) L2F_ST16(7)
                     L2F_ST16(8) L2F_ST16(9) L2F_ST16(10) L2F_ST16(11) L2F_ST16(12) L2F_ST16(13) L2F_ST16(14)
                         L2F_ST16(15)::"r"(saddr),
                 "r"(a), "r"(b), "r"(c), "r"(d), "n"(kStride)
                 : "memory");
#undef L2F_ST16
}

__device__ __forceinline__ void sts64(uint32_t saddr, uint32_t a, uint32_t b)
{
    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(saddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void lds64(uint32_t saddr, uint32_t& a, uint32_t& b)
{
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(saddr) : "memory");
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi)
{
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}
// relu on two fp32 accumulators -> packed fp16 in one cvt (relu commutes with RNE rounding);
// a goes to the low half (lower K index).
__device__ __forceinline__ uint32_t relu_pack(uint32_t a, uint32_t b)
{
    uint32_t d;
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(d) : "r"(b), "r"(a));
    return d;
}

}  // namespace tc
}  // namespace l2f
