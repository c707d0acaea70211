// tc.cuh -- sm_100a primitives: mbarriers, TMA (cp.async.bulk.tensor), and
// tcgen05 (UMMA descriptors, MMA issue/commit, TMEM alloc/ld/st), written as
// inline PTX.  Encodings follow the sm_100 descriptor formats (see the CuTe
// headers cute/arch/mma_sm100_desc.hpp for the bit layout).
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "common.cuh"

namespace wgkv {
namespace tc {

// ---------------------------------------------------------------- mbarrier --
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// try_wait with a suspend-time hint: a waiting warp yields its issue slots
// (for warps that share SM sub-partitions with compute warps)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
// non-suspending poll (test_wait): lower wake-up latency for a thread on the
// critical path (the MMA issuer), at the cost of issue slots while spinning
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---------------------------------------------------------------------- TMA --
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
        "%6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
// the same with an L2 cache policy (createpolicy), e.g. evict_first for data
// streamed once
__device__ __forceinline__ void tma_load_4d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 int c2, int c3, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
        "{%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// TMA store (bulk group): smem tile -> global through a 4-D map; rows outside
// the map's extent are not written
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                             int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until every committed bulk group has finished READING its shared memory source
__device__ __forceinline__ void bulk_wait_group_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// plain bulk copy global -> shared (bytes a multiple of 16, both 16-byte aligned)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// generic-proxy global writes (made visible by an acquire) -> a following async-proxy read
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------------ tcgen05 --
// Shared-memory matrix descriptor (sm_100): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version=1 [46,48), base_offset=0, layout [61,64):
// SWIZZLE_128B = 2.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor, kind::f16: D=F32 [4,6)=1, A=BF16 [7,10)=1,
// B=BF16 [10,13)=1, a_major [15], b_major [16], N>>3 [17,23), M>>4 [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accum) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum));
}
// A operand from tensor memory (M lanes x K/2 32-bit columns of packed bf16x2)
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accum) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum));
}
// warp-wide issue: every lane runs the issue loop with warp-uniform operands
// (kept in uniform registers) and elect.sync picks the one issuing thread
__device__ __forceinline__ void mma_ss_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accum) {
    asm volatile(
        "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accum) {
    asm volatile(
        "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
        : "memory");
}
// arrive on `bar` once all previously issued tcgen05 ops of this thread complete
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// TMEM allocation by one full warp; writes the base address to *dst_smem
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread i of the warp gets row
// (lane_base + i), columns [col, col+32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// byte offset of 16-byte chunk `chunk` (0..7) of row `row` inside a
// [rows][64 bf16] SWIZZLE_128B tile (1024-byte aligned base)
__device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t chunk) {
    return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

}  // namespace tc
}  // namespace wgkv

// host: tensor-map encoder via the driver entry point (no -lcuda)
namespace wgkv {
// 4-D bf16 map, SWIZZLE_128B (box0 * 2 bytes must be 128)
int make_tmap_4d_bf16(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint64_t strides_bytes[3],
                      const uint32_t box[4]);
int make_tmap_3d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                      uint64_t stride2_bytes, uint32_t box0, uint32_t box1, uint32_t box2);
// 2-D bf16 map [d1 rows][d0 elements], row stride in bytes, SWIZZLE_128B (box0 * 2 bytes must be 128)
int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t stride1_bytes,
                      uint32_t box0, uint32_t box1);
}

namespace wgkv {
namespace tc {
// One K = 128 group of 8 warp-issued MMAs (K step 16 each) in a single asm
// block: one elect.sync, descriptors advanced by immediates inside the block
// (start-address field, units of 16 bytes), so the issue costs ~2 instructions
// per MMA instead of recomputing and re-broadcasting every operand.
//   SS: a_desc(kk) = a0 + a_step(kk), b_desc(kk) = b0 + b_step(kk); accumulate from kk > 0 or acc
//   TS: A from TMEM at a_tmem + 8 kk
// K-major SW128 [128][64] sub-tile pairs step {0,2,4,6,1024,1026,1028,1030}
// (32 bytes per k16 inside a 128-byte row, next sub-tile at +16 KB);
// MN-major V sub-tiles of 16 rows step 128 (2 KB) per k16.
__device__ __forceinline__ void mma8_ss_kmajor_w(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc,
                                                 uint32_t acc) {
    asm volatile(
        "{\n.reg .pred e, p;\n.reg .b64 a, b;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "add.s64 a, %1, 2;\n add.s64 b, %2, 2;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, 4;\n add.s64 b, %2, 4;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, 6;\n add.s64 b, %2, 6;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, 1024;\n add.s64 b, %2, 1024;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, 1026;\n add.s64 b, %2, 1026;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, 1028;\n add.s64 b, %2, 1028;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, 1030;\n add.s64 b, %2, 1030;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a0), "l"(b0), "r"(idesc), "r"(acc));
}
// TS with B K-major (S = Q K^T, Q in TMEM)
__device__ __forceinline__ void mma8_ts_kmajor_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b0, uint32_t idesc,
                                                 uint32_t acc) {
    asm volatile(
        "{\n.reg .pred e, p;\n.reg .b64 b;\n.reg .b32 a;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "add.s32 a, %1, 8;\n add.s64 b, %2, 2;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 16;\n add.s64 b, %2, 4;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 24;\n add.s64 b, %2, 6;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 32;\n add.s64 b, %2, 1024;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 40;\n add.s64 b, %2, 1026;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 48;\n add.s64 b, %2, 1028;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 56;\n add.s64 b, %2, 1030;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b0), "r"(idesc), "r"(acc));
}
// TS with B MN-major V sub-tiles (O += P V): b_desc(kk) = b0 + 128 kk
__device__ __forceinline__ void mma8_ts_vmn_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b0, uint32_t idesc,
                                              uint32_t acc) {
    asm volatile(
        "{\n.reg .pred e, p;\n.reg .b64 b;\n.reg .b32 a;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "add.s32 a, %1, 8;\n add.s64 b, %2, 128;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 16;\n add.s64 b, %2, 256;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 24;\n add.s64 b, %2, 384;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 32;\n add.s64 b, %2, 512;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 40;\n add.s64 b, %2, 640;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 48;\n add.s64 b, %2, 768;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 56;\n add.s64 b, %2, 896;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b0), "r"(idesc), "r"(acc));
}
}  // namespace tc
}  // namespace wgkv

namespace wgkv {
namespace tc {
// 8 K16 steps of an SS MMA over a K = 128 operand pair whose SW128 K-major
// sub-tiles (64 of K) are `a_sub16` / `b_sub16` descriptor units (16 bytes)
// apart: one elect.sync, descriptors advanced by immediates; accumulate from
// the second step (the first step overwrites D)
template <int A_SUB16, int B_SUB16>
__device__ __forceinline__ void mma8_ss_k128_w(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc) {
    asm volatile(
        "{\n.reg .pred e;\n.reg .b64 a, b;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;\n"
        "add.s64 a, %1, 2;\n add.s64 b, %2, 2;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, 4;\n add.s64 b, %2, 4;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, 6;\n add.s64 b, %2, 6;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, %4;\n add.s64 b, %2, %5;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, %4 + 2;\n add.s64 b, %2, %5 + 2;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, %4 + 4;\n add.s64 b, %2, %5 + 4;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "add.s64 a, %1, %4 + 6;\n add.s64 b, %2, %5 + 6;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a0), "l"(b0), "r"(idesc), "n"(A_SUB16), "n"(B_SUB16));
}
// 4 K16 steps of a TS MMA: A from TMEM at a_tmem + 8 kk, B MN-major advancing 128 units (2 KB) per step
__device__ __forceinline__ void mma4_ts_vmn_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b0, uint32_t idesc,
                                              uint32_t acc) {
    asm volatile(
        "{\n.reg .pred e, p;\n.reg .b64 b;\n.reg .b32 a;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "add.s32 a, %1, 8;\n add.s64 b, %2, 128;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 16;\n add.s64 b, %2, 256;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "add.s32 a, %1, 24;\n add.s64 b, %2, 384;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b0), "r"(idesc), "r"(acc));
}
}  // namespace tc
}  // namespace wgkv
