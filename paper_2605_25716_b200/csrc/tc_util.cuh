// tc_util.cuh -- thin inline-PTX layer for the sm_100a tensor-core kernels: mbarriers, bulk
// copies (1D and tensor TMA), tcgen05 TMEM allocation / MMA / loads, and UMMA descriptors.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sda {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Spinning variant (test_wait: never suspends): lower wake-up latency for a lone issuer warp whose
// waits sit on the critical path, at the price of issue slots on its SMSP.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Polling with a nanosleep between test_waits: the spinning warp leaves its SMSP's issue slots to
// the warps it shares them with (the prefill K2's MMA warp sits on a softmax warp pair's SMSP).
template <int NS>
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "nanosleep.u32 %2;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(NS)
        : "memory");
}
// try_wait with a suspend-time hint (ns): the warp sleeps until the phase completes or the hint
// elapses, then polls again.
template <int NS>
__device__ __forceinline__ void mbar_wait_hint(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(NS)
        : "memory");
}
// 16-byte async copy global -> shared (LDGSTS), L2-only caching.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// Arrive on `bar` when all of this thread's prior cp.async have landed (counts as one of the
// barrier's expected arrivals).
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------------------- proxies / fences
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ---------------------------------------------------------------------------- bulk copies
// 1D bulk copy global -> shared, completes `bytes` on `bar` (size multiple of 16, 16B aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 2D tensor TMA load (tile mode) into shared, completing on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// 2D tensor TMA store (tile mode) shared -> global; bulk-group completion.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Bulk prefetch of `bytes` (multiple of 16) into L2.
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// ---------------------------------------------------------------------------- TMEM
// Allocate `ncols` (power of 2, >= 32) TMEM columns; the base address lands in *dst (smem).
// Must be executed by one full warp.
template <uint32_t ncols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
                 "n"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <uint32_t ncols>
__device__ __forceinline__ void tmem_dealloc(uint32_t addr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "n"(ncols));
}

// D[tmem] (+)= A[smem] . B[smem]^T, bf16 x bf16 -> f32, issued by one thread.
__device__ __forceinline__ void mma_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// D[tmem] (+)= A[tmem] . B[smem]^T (A operand from tensor memory).
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// One lane of a fully active warp (the lowest): the MMA issuer runs its loop with the whole warp
// so the operand descriptors stay warp-uniform (uniform registers, no R2UR per instruction) and
// only the tcgen05.mma / commit instructions are predicated on the elected lane.
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(pred));
    return pred != 0;
}
// Arrive on `bar` once every previously issued tcgen05.mma of this thread has completed.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// ---------------------------------------------------------------------------- CTA pair (cta_group::2)
// Two CTAs of a cluster (ranks 0, 1) share each MMA: M = 256 rows (128 in each CTA's TMEM, A
// from each CTA's shared memory), B split along N between the two CTAs' shared memory. Rank 0
// issues the MMAs; its barriers collect the pair's TMA bytes and the softmax arrivals.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of the same object in CTA 0 of the cluster
__device__ __forceinline__ uint32_t at_rank0(const void* p) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// relaxed: no MEMBAR.GPU (the release form costs ~0.7 us per arrive). For hand-offs whose data
// the arriving thread has already ordered locally (an acquire of this CTA's own barrier, whose
// writers fenced their shared-memory stores for the async proxy).
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Spins (test_wait): a try_wait suspended on a barrier that a peer CTA completes is not woken by
// that remote arrive and sleeps out its time slice (~0.9 us per hand-off, tools/k2_trace.py PAIR=1).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 2D tensor TMA into this CTA's shared memory, completing the bytes on a barrier of either CTA of
// the pair (cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(bar_cluster)
        : "memory");
}
template <uint32_t ncols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "n"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t ncols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t addr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(addr), "n"(ncols));
}
__device__ __forceinline__ void mma_bf16_ss_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// arrive on `bar` (same offset) in both CTAs of the pair once this thread's MMAs have completed
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "h"((uint16_t)3)
                 : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread (thread i <- TMEM lane (warp%4)*32 + i).
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 32 lanes x 32 bit, 8 consecutive columns per thread.
__device__ __forceinline__ void tmem_st8(uint32_t addr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------------------- descriptors
// Shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), sm_100 version bit.
//   K-major   : rows of 128 B (64 bf16 along K), 8-row swizzle atoms, SBO = 1024 B between
//               8-row groups, LBO unused. Advance along K inside the atom by adding bytes.
//   MN-major  : 128 B along MN (64 bf16), 8 K-rows per atom; SBO = 1024 B between 8-row K
//               groups, LBO = bytes between 64-wide MN blocks.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // version (sm_100)
    d |= (uint64_t)2 << 61;   // SWIZZLE_128B
    return d;
}

// Instruction descriptor for kind::f16: bf16 x bf16 -> f32, dense.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N, bool a_mn_major, bool b_mn_major) {
    return (1u << 4)                              // c_format = F32
           | (1u << 7)                            // a_format = BF16
           | (1u << 10)                           // b_format = BF16
           | ((a_mn_major ? 1u : 0u) << 15)       // a_major
           | ((b_mn_major ? 1u : 0u) << 16)       // b_major
           | ((uint32_t)(N >> 3) << 17)           // n_dim
           | ((uint32_t)(M >> 4) << 24);          // m_dim
}

// Byte offset of 16-byte chunk `c16` (0..7) of row `r` inside a SWIZZLE_128B region whose rows
// are 128 B apart (1024-byte aligned base).
__device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t c16) {
    return r * 128u + ((c16 ^ (r & 7u)) << 4);
}

// Packed f32x2 arithmetic (sm_100 FFMA2 / FADD2) and the 3-input max (FMNMX3).
__device__ __forceinline__ uint64_t f2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2_split(uint64_t r, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// 2^x for two values x <= 0 on the FMA pipe instead of the MUFU (XU) pipe, which on B200 is the
// softmax's bottleneck (16 MUFU ops per clock per SM vs 128 FMA lanes). x = n + f with
// n = round(x) (magic-number add), 2^f by a degree-3 minimax polynomial on [-1/2, 1/2]
// (max relative error 7.5e-5, far below the bf16 rounding P gets next), 2^n by adding n to the
// exponent field. x is clamped at -125 so the exponent never underflows (2^-125 ~ 2e-38 where
// the MUFU would return 0 or a denormal: negligible in any row sum).
__device__ __forceinline__ float exp2_fma(float x) {
    // scalar FADD / FFMA with immediate operands: no registers tied up in constants
    constexpr float kMagic = 12582912.f;   // 1.5 * 2^23
    x = fmaxf(x, -125.f);
    const float t = __fadd_rn(x, kMagic);                 // round(x) in the low mantissa bits
    const float n = __fadd_rn(t, -kMagic);                // round(x) as a float
    const float f = __fadd_rn(x, -n);                     // x - round(x) in [-1/2, 1/2]
    float p = __fmaf_rn(0.05517143f, f, 0.24261081f);
    p = __fmaf_rn(p, f, 0.69326097f);
    p = __fmaf_rn(p, f, 0.9999281f);
    uint32_t r;   // bits(2^f) + (n << 23): the low bits of t hold n (two's complement)
    asm("mad.lo.u32 %0, %1, 8388608, %2;" : "=r"(r) : "r"(__float_as_uint(t)), "r"(__float_as_uint(p)));
    return __uint_as_float(r);
}
__device__ __forceinline__ void exp2_fma2(float x0, float x1, float& p0, float& p1) {
    p0 = exp2_fma(x0);
    p1 = exp2_fma(x1);
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// The same 2^x on a packed pair: the rounding, the reduction and the polynomial as FADD2 / FFMA2
// (half the issue slots of the scalar form; the FMA-pipe time per value is the same), the clamp
// as two FMNMX and the exponent insertion as integer ops on the ALU pipe.
__device__ __forceinline__ void exp2_fma2_packed(float x0, float x1, float& p0, float& p1) {
    constexpr float kMagic = 12582912.f;
    const uint64_t x = f2(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
    const uint64_t t = fadd2(x, f2(kMagic, kMagic));
    const uint64_t f = fsub2(x, fsub2(t, f2(kMagic, kMagic)));
    uint64_t p = ffma2(f2(0.05517143f, 0.05517143f), f, f2(0.24261081f, 0.24261081f));
    p = ffma2(p, f, f2(0.69326097f, 0.69326097f));
    p = ffma2(p, f, f2(0.9999281f, 0.9999281f));
    float t0, t1, q0, q1;
    f2_split(t, t0, t1);
    f2_split(p, q0, q1);
    p0 = __uint_as_float((__float_as_uint(t0) << 23) + __float_as_uint(q0));
    p1 = __uint_as_float((__float_as_uint(t1) << 23) + __float_as_uint(q1));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
    return r;
}

}  // namespace tc
}  // namespace sda
