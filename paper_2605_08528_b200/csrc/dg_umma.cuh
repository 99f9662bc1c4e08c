// dg_umma.cuh -- minimal tcgen05 (5th-gen tensor core) toolkit for sm_100a.
//
// Operands live in shared memory in the canonical K-major, no-swizzle UMMA
// layout: an R x K bf16 tile is a grid of 8x8 "core matrices" (8 rows x 16 B,
// 128 B contiguous); element (r, k) sits at byte
//     ((r / 8) * (K / 8) + k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2,
// so the K-direction core-matrix stride (LBO) is 128 B and the 8-row-group
// stride (SBO) is K / 8 * 128 B.  D = A . B^T with A = M x K (activations,
// one row per sample) and B = N x K (a torch Linear weight [out][in] as is);
// the fp32 accumulator lives in tensor memory (row m -> TMEM lane m, column n
// -> column base + n).  Descriptor bit layouts: CUTLASS cute/arch/
// mma_sm100_desc.hpp (SmemDescriptor, InstrDescriptor).
#pragma once
#include <cstdint>

namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of element (r, k) inside a canonical K-major tile with K columns
__host__ __device__ __forceinline__ uint32_t kmajor_offset(int r, int k, int K) {
    return uint32_t(((r >> 3) * (K >> 3) + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

// shared-memory matrix descriptor: start, LBO, SBO (bytes), SWIZZLE_NONE, version 1
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;             // version (Blackwell)
    return d;                           // base_offset 0, lbo_mode 0, layout_type 0 (no swizzle)
}

// instruction descriptor, kind::f16: bf16 x bf16 -> f32, both K-major
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4)                    // D format f32
         | (1u << 7)                    // A bf16
         | (1u << 10)                   // B bf16
         | (uint32_t(N >> 3) << 17)
         | (uint32_t(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] . B[smem]^T, one K=16 step; issued by ONE thread
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}

// Full GEMM D[M=128 x N] = A[128 x K] . B[N x K]^T over K in steps of 16,
// both operands canonical K-major tiles (K columns, multiple of 16).
__device__ __forceinline__ void gemm_128xN(uint32_t tmem_d, const void* a, const void* b, int N, int K) {
    const uint32_t sa = smem_u32(a), sb = smem_u32(b);
    const uint32_t sbo = uint32_t(K >> 3) * 128u;
    const uint32_t id = idesc_bf16(128, N);
    for (int k = 0; k < K; k += 16) {
        const uint32_t off = uint32_t(k >> 3) * 128u;   // two K core matrices per step
        mma_bf16(tmem_d, sdesc(sa + off, 128u, sbo), sdesc(sb + off, 128u, sbo), id, k > 0 ? 1u : 0u);
    }
}

// MMA completion -> mbarrier arrive (implies tcgen05.fence::before_thread_sync)
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy smem stores -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "UMMA_WAIT_%=:\n\t"
#ifdef DG_EXP_SUSPEND
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
#else
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
#endif
        "@!p bra UMMA_WAIT_%=;\n}"
        ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// TMEM allocation: one full warp; the base address lands in *dst (shared)
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(dst)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 16 consecutive fp32 columns of this thread's TMEM lane (warp w reads lanes
// 32*(w%4) .. +31; taddr must carry that lane base in bits 16..31).
// Split load: issue several, then wait.  The wait takes the destination
// registers as in/out operands, so no use of them can be scheduled before it
// (a second wait on already-landed loads returns at once).
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait16(uint32_t* r) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15])
                 :: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    tmem_ld16_issue(taddr, r);
    tmem_wait16(r);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

}  // namespace umma
