// attn_tc.cu -- K3: vertical-slash prefill attention on the 5th-gen tensor
// cores (tcgen05 + TMEM + TMA), bf16 inputs, fp32 accumulation, d = 128.
//
// Replaces build_vs_mask + attn_vertical_slash (attention.cpp:116-153) for
// the Session::prefill call site (engine.cpp:222-240).  One CTA owns a
// 128-row query tile of NT = 2 query heads of the same GQA group (they share
// every K/V tile and every mask), and visits exactly the key set
//   vertical : the admitted Global prefix j < i0-W+1 (all rows see it; read in
//              place from the pages K2 filled, one TMA per page half)
//   band     : keys [i0-W+1, i0+127] of k_post / v (TMA tiles), with per
//              element masks only on the <= 2 edge tiles
// (SURVEY.md App. A.9).  Warp roles, 19 warps (608 threads), 1 CTA / SM:
//   warps 0-15 : softmax; warp = (tile t, column half c, lane quarter wq)
//                owns rows 32wq..32wq+31 (its TMEM lane quarter) and S/P/O
//                columns [64c, 64c+64) of tile t: RoPE(q) in smem, then per key
//                block tcgen05.ld S, mask, row max exchanged with the other
//                half through smem (named barrier), online softmax (lazy
//                rescale, threshold 2^8; 1/4 of the exp2 on the FMA pipe,
//                F2FP bf16 packing), P as bf16x2
//                written back into TMEM over S, O rescale in TMEM
//   warp 16/17 : TMA producers for K / V (Q once), 2-stage ring each with its
//                own full/empty barriers
//   warp 18    : TMEM allocator + single-thread MMA issuer, tiles in turn:
//                S_t = Q_t K^T (SS, K-major x K-major, M=N=128, K=128)
//                O_t += P_t V  (TS: P from TMEM, V MN-major from smem)
// TMEM: tile t owns O_t = cols [256t, 256t+128) and S_t/P_t = [256t+128, 256t+256).
// Measured alternatives (profiles/r1_k3_notes.md): one head per CTA with a
// double-buffered S (smem/TMA-bound, -20 %), one MMA issuer per tile (the
// two softmax groups fall into phase and contend for the MUFU, -16 %).
#include <cuda.h>

#include <cstdio>

#include "attn_tc.cuh"
#include "tc.cuh"

#ifndef WGKV_K3_WARP_ISSUE
#define WGKV_K3_WARP_ISSUE 1
#endif
// each 8-MMA group as one asm block (one elect, descriptors advanced by
// immediates): halves the issue instructions, measured neutral (r2_k3_notes.md)
#ifndef WGKV_K3_MMA8
#define WGKV_K3_MMA8 0
#endif
// waits with a suspend-time hint (spinning warps give their issue slots to the
// softmax warps of the same SM sub-partition): bit 0 producers, 1 MMA issuer, 2 softmax
#ifndef WGKV_K3_SLEEP
#define WGKV_K3_SLEEP 2
#endif
#define K3_WAIT(role, bar_, par_) \
    ((WGKV_K3_SLEEP >> (role)) & 1 ? tc::mbar_wait_sleep((bar_), (par_)) : tc::mbar_wait((bar_), (par_)))

namespace wgkv {

namespace {

constexpr int NT = 2;       // query heads (128-row tiles) per CTA
constexpr int NSTAGE = 2;   // K/V ring depth
constexpr uint32_t TILE_BYTES = 128 * 128 * 2;        // one [128][128] bf16 tile
constexpr uint32_t SUB_BYTES = TILE_BYTES / 2;        // [128][64] SW128 sub-tile
constexpr uint32_t OFF_Q = 0;
constexpr uint32_t OFF_KV = NT * TILE_BYTES;
constexpr uint32_t STAGE_BYTES = 2 * TILE_BYTES;      // K then V
constexpr uint32_t OFF_BAR = OFF_KV + NSTAGE * STAGE_BYTES;
constexpr int NSPLIT = 2;                   // softmax warpgroups per tile (column halves)
constexpr int HC = 128 / NSPLIT;            // S columns per softmax thread
constexpr int NSOFT = NT * NSPLIT * 4;      // softmax warps
constexpr int WARP_TMA = NSOFT, WARP_MMA = NSOFT + 2;  // K producer, V producer, MMA issuer
constexpr uint32_t OFF_X = OFF_BAR + 512;   // [NT][NSPLIT][128] f32 row-max / row-sum exchange
constexpr uint32_t SMEM_BYTES = OFF_X + NT * NSPLIT * 128 * 4 + 1024;  // + alignment slack
constexpr int NTHREADS = (NSOFT + 3) * 32;
constexpr float LOG2E = 1.4426950408889634f;

struct Bars {
    uint64_t q_full, q_ready;
    uint64_t k_full[NSTAGE], k_empty[NSTAGE], v_full[NSTAGE], v_empty[NSTAGE];
    uint64_t s_full[NT], p_full[NT], o_final[NT];
    uint32_t tmem;
    int C;
};

#ifndef WGKV_K3_MAX3
#define WGKV_K3_MAX3 0
#endif
__device__ __forceinline__ float max3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

#ifndef WGKV_PACK_ALU
#define WGKV_PACK_ALU 0  // bit e: pair e packed on the ALU (2 IADD + PRMT) instead of F2FP.  F2FP shares the MUFU
                         // pipe on B200 (tools/ubench_mufu.cu): ALU packing won 3.5 % with a lane-0 MMA issuer;
                         // with the warp-uniform issuer all-F2FP is 0.6-1 % faster and mixed masks are slower
                         // (profiles/r1_k3_notes.md)
#endif
// fp32 pair -> bf16x2 on the ALU pipe (two IADD + one PRMT) instead of F2FP,
// which competes with MUFU.EX2 for the same pipe on B200.
// Round-half-up on the (finite, non-negative) P values.
__device__ __forceinline__ uint32_t pack_bf16x2_alu(float lo, float hi) {
    return __byte_perm(__float_as_uint(lo) + 0x8000u, __float_as_uint(hi) + 0x8000u, 0x7632);
}
#ifndef WGKV_EMU_MASK
#define WGKV_EMU_MASK 0x8888  // bit e set: exp2 pair e of each 32-column chunk runs on the FMA pipe
                              // (measured with packing on the ALU: 1/4 -> -0.7 %, 5/16 +1 %, 1/2 +7 %)
#endif
// 2^x for a pair on the FMA/ALU pipes (offloads the MUFU, which otherwise
// paces the softmax), packed f32x2 arithmetic: Cody-Waite split x = n + f with
// f in [-1/2, 1/2] via the 1.5*2^23 rounding trick, cubic near-minimax for
// 2^f (max rel. error 7.5e-5, far below the bf16 rounding of P), exponent
// add for 2^n.  x is clamped at -127.5, where the exponent field goes negative
// and the integer max returns exactly +0 (so masked -inf keys give P = 0).
__device__ __forceinline__ float2 ex2_emu2(float x0, float x1) {
    const float2 xc = make_float2(fmaxf(x0, -127.5f), fmaxf(x1, -127.5f));
    const float2 big = make_float2(12582912.f, 12582912.f);
    const float2 t = __fadd2_rn(xc, big);
    const float2 tb = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = __ffma2_rn(tb, make_float2(-1.f, -1.f), xc);
    float2 p = __ffma2_rn(f, make_float2(0.05517161f, 0.05517161f), make_float2(0.24261111f, 0.24261111f));
    p = __ffma2_rn(p, f, make_float2(0.69326097f, 0.69326097f));
    p = __ffma2_rn(p, f, make_float2(0.99992806f, 0.99992806f));
    const int r0 = max(__float_as_int(p.x) + (__float_as_int(t.x) << 23), 0);
    const int r1 = max(__float_as_int(p.y) + (__float_as_int(t.y) << 23), 0);
    return make_float2(__int_as_float(r0), __int_as_float(r1));
}

#ifndef WGKV_EMU_PACK_INT
#define WGKV_EMU_PACK_INT 0
#endif
// emulated pair straight to bf16x2 (no F2FP on the MUFU pipe): the same cubic,
// the exponent add and a round-half-up bias folded into one IADD3 per value,
// the two high halves joined by one PRMT.  x is clamped at -126 so the biased
// exponent never goes negative (masked -inf keys give a ~1e-38 weight, zero at
// bf16 resolution of any row sum they join).  *s0 / *s1 receive the fp32 values
// (bias excluded) for the row sum.
__device__ __forceinline__ uint32_t ex2_emu2_bf16(float x0, float x1, float& s0, float& s1) {
    const float2 xc = make_float2(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
    const float2 big = make_float2(12582912.f, 12582912.f);
    const float2 t = __fadd2_rn(xc, big);
    const float2 tb = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = __ffma2_rn(tb, make_float2(-1.f, -1.f), xc);
    float2 p = __ffma2_rn(f, make_float2(0.05517161f, 0.05517161f), make_float2(0.24261111f, 0.24261111f));
    p = __ffma2_rn(p, f, make_float2(0.69326097f, 0.69326097f));
    p = __ffma2_rn(p, f, make_float2(0.99992806f, 0.99992806f));
    const uint32_t e0 = (uint32_t)__float_as_int(t.x) << 23, e1 = (uint32_t)__float_as_int(t.y) << 23;
    const uint32_t r0 = (uint32_t)__float_as_int(p.x) + e0, r1 = (uint32_t)__float_as_int(p.y) + e1;
    s0 = __uint_as_float(r0);
    s1 = __uint_as_float(r1);
    return __byte_perm(r0 + 0x8000u, r1 + 0x8000u, 0x7632);
}

__device__ __forceinline__ uint64_t kmajor_desc(uint32_t tile_saddr, int kk) {
    // K-major SW128 operand, K step kk (16 bf16 = 32 bytes); sub-tile per 64 K
    return tc::smem_desc_sw128(tile_saddr + (uint32_t)(kk >> 2) * SUB_BYTES + (uint32_t)(kk & 3) * 32u, 16, 1024);
}

}  // namespace

#ifdef WGKV_TRACE  // diagnostic build only: per-block event clocks of CTA (0,0,0)
__device__ unsigned long long g_k3_trace[4][4096][8];
#define K3_TR(who, j, ev)                                                                          \
    do {                                                                                           \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 4096) g_k3_trace[who][j][ev] = clock64(); \
    } while (0)
#else
#define K3_TR(who, j, ev) \
    do {                  \
    } while (0)
#endif
__global__ void __launch_bounds__(NTHREADS, 1)
    vs_prefill_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                         const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tpool,
                         const __grid_constant__ CUtensorMap tkrun, const __grid_constant__ CUtensorMap tvrun,
                         VsArgs a, __nv_bfloat16* __restrict__ out) {
    extern __shared__ uint8_t smem_raw[];
    // 1 KB-aligned through an integer round trip: the few accesses through sm
    // (not TMA / tcgen05 / ldmatrix, which take 32-bit smem addresses) are then
    // generic.  Kept here on purpose: the shared-space variant measured 3 %
    // slower K3 (141.9 vs 137.7 ms, interleaved A/B, different scheduling);
    // the other kernels use pointer arithmetic on the __shared__ array
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bar = reinterpret_cast<Bars*>(sm + OFF_BAR);
    const uint32_t sbase = smem_u32(sm);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long i0 = (long)(gridDim.x - 1 - blockIdx.x) * 128;  // longest tiles first
    const int p0 = blockIdx.y * NT;
    const int s = blockIdx.z;
    const int Hq = a.q_heads, Hkv = a.pv.kv_heads;
    const int h = p0 / (Hq / Hkv);
    const long T = a.T, W = a.W;
    const long hidx = a.pv.head_index(a.layer, a.seq0 + s, h);
    const uint8_t* bits = a.bits + ((size_t)s * Hkv + h) * T;
    const long nchunk = (T + 127) / 128;
    const int32_t* co = a.chunk_off + ((size_t)s * Hkv + h) * (nchunk + 1);

    // ---- key-set geometry (identical in every role) ----------------------
    const long s_lo = i0 - W + 1 > 0 ? i0 - W + 1 : 0;
    int cnt = 0;
    {
        const long c = s_lo / 128, rem = s_lo - c * 128;
        cnt = __syncthreads_count(threadIdx.x < rem && bits[c * 128 + threadIdx.x] != 0);
    }
    if (threadIdx.x == 0) {
        int C = s_lo > 0 ? co[s_lo / 128] + cnt : 0;
        C = min(C, a.pv.state[hidx].global_len);  // 0 after a failed page claim
        bar->C = C;
        tc::mbar_init(&bar->q_full, 1);
        tc::mbar_init(&bar->q_ready, NSOFT * 32);
        for (int i = 0; i < NSTAGE; ++i) {
            tc::mbar_init(&bar->k_full[i], 1);
            tc::mbar_init(&bar->k_empty[i], 1);
            tc::mbar_init(&bar->v_full[i], 1);
            tc::mbar_init(&bar->v_empty[i], 1);
        }
        for (int t = 0; t < NT; ++t) {
            tc::mbar_init(&bar->s_full[t], 1);
            tc::mbar_init(&bar->p_full[t], NSPLIT * 128);
            tc::mbar_init(&bar->o_final[t], 1);
        }
        tc::fence_barrier_init();
    }
    if (warp == WARP_MMA) tc::tmem_alloc(&bar->tmem, 512);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const int C = bar->C;
    const uint32_t tmem = bar->tmem;
    const long band_hi = min(i0 + 127, T - 1);
    const int nv = (C + 127) / 128;
    const int nb = (int)((band_hi - s_lo + 1 + 127) / 128);
    const int nblk = nv + nb;
    const int ps = a.pv.page_size;

    if (warp == WARP_TMA || warp == WARP_TMA + 1) {
        // ============================ TMA producers ===========================
        // one warp for K, one for V: each runs ahead by the ring depth on its
        // own (one in-order producer holds K(j+1) behind the release of
        // V(j+1-NSTAGE), which comes a whole PV later)
        const int kv = warp - WARP_TMA;
        if (lane == 0 && kv == 0) {
            tc::tma_prefetch(&tq);
            tc::tma_prefetch(&tk);
            tc::tma_prefetch(&tv);
            tc::tma_prefetch(&tpool);
            tc::tma_prefetch(&tkrun);
            tc::tma_prefetch(&tvrun);
            tc::mbar_arrive_expect_tx(&bar->q_full, NT * TILE_BYTES);
            for (int t = 0; t < NT; ++t)
                for (int hh = 0; hh < 2; ++hh)
                    tc::tma_load_3d(sm + OFF_Q + t * TILE_BYTES + hh * SUB_BYTES, &tq, &bar->q_full, hh * 64, p0 + t,
                                    (int)(s * T + i0));
        }
        // Global page ids of vertical blocks: lane i holds page i of a block; the
        // next block's ids are loaded (in flight) before waiting on this one's
        // slot, so the page-table reads never serialise the TMA issue.
        const int ppb = 128 / ps;  // pages per 128-key block (<= 16)
        const int last_page = C > 0 ? (C - 1) / ps : 0;
        const int32_t* gpt = a.pv.gpt + hidx * a.pv.n_gp;
        auto page_ids = [&](int jb) -> int {
            return (jb < nv && lane < ppb) ? gpt[min(jb * ppb + lane, last_page)] : 0;
        };
        int next_ids = page_ids(0);
        // K and V of a block have separate full/empty barriers: K(j) is free
        // once both tiles' S(j) are done, long before PV(j) releases V(j), so
        // the K refill gets a whole extra MMA round of slack.
        for (int j = 0; j < nblk; ++j) {
            const int st = j & 1;
            const int cur_ids = next_ids;
            if (j + 1 < nblk) next_ids = page_ids(j + 1);
            const bool band = j >= nv;
            const long kb0 = band ? s_lo + 128L * (j - nv) : 0;
            // vertical copy `lane` = (page lane/2, dim half lane%2), 2*ppb <= 32
            const int pg = __shfl_sync(0xffffffffu, cur_ids, lane >> 1);
            {
                uint64_t* full = kv ? &bar->v_full[st] : &bar->k_full[st];
                if (j >= NSTAGE) K3_WAIT(0, kv ? &bar->v_empty[st] : &bar->k_empty[st], ((j - NSTAGE) >> 1) & 1);
                if (lane == 0) K3_TR(3, j, kv);
                uint8_t* dst = sm + OFF_KV + st * STAGE_BYTES + kv * TILE_BYTES;
                if (lane == 0) tc::mbar_arrive_expect_tx(full, TILE_BYTES);
                __syncwarp();
                if (!band) {
                    // physically consecutive pages (the usual case after a prefill's
                    // single claim): one box of ppb pages per dim half
                    const int pg0 = __shfl_sync(0xffffffffu, cur_ids, 0);
                    if (__all_sync(0xffffffffu, lane >= ppb || cur_ids == pg0 + lane)) {
                        if (lane < 2)
                            tc::tma_load_3d(dst + lane * SUB_BYTES, kv ? &tvrun : &tkrun, full, lane * 64, 0, pg0);
                    } else if (lane < 2 * ppb) {
                        tc::tma_load_3d(dst + (lane & 1) * SUB_BYTES + (lane >> 1) * ps * 128, &tpool, full,
                                        (lane & 1) * 64, 0, 2 * pg + kv);
                    }
                } else if (lane < 2) {
                    tc::tma_load_3d(dst + lane * SUB_BYTES, kv ? &tv : &tk, full, lane * 64, h, (int)(s * T + kb0));
                }
            }
        }
    } else if (warp == WARP_MMA) {
        // ================================ MMA issuer =============================
#if WGKV_K3_WARP_ISSUE
        // the whole warp runs the loop (warp-uniform operands stay in uniform
        // registers); elect.sync issues each tcgen05 op from one lane
#define K3_MMA_SS tc::mma_ss_w
#define K3_MMA_TS tc::mma_ts_w
#define K3_COMMIT tc::mma_commit_w
        {
#else
#define K3_MMA_SS tc::mma_ss
#define K3_MMA_TS tc::mma_ts
#define K3_COMMIT tc::mma_commit
        if (lane == 0) {
#endif
            constexpr uint32_t idS = tc::idesc_bf16(128, 128, false, false);
            constexpr uint32_t idPV = tc::idesc_bf16(128, 128, false, true);
            auto issue_S = [&](int t, int st) {
                const uint32_t qa = sbase + OFF_Q + t * TILE_BYTES;
                const uint32_t ka = sbase + OFF_KV + st * STAGE_BYTES;
                const uint32_t d = tmem + 256 * t + 128;
#if WGKV_K3_MMA8
                tc::mma8_ss_kmajor_w(d, kmajor_desc(qa, 0), kmajor_desc(ka, 0), idS, 0);
#else
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) K3_MMA_SS(d, kmajor_desc(qa, kk), kmajor_desc(ka, kk), idS, kk > 0);
#endif
            };
            auto issue_PV = [&](int t, int st, bool acc) {
                const uint32_t va = sbase + OFF_KV + st * STAGE_BYTES + TILE_BYTES;
                const uint32_t d = tmem + 256 * t, pa = tmem + 256 * t + 128;
#if WGKV_K3_MMA8
                tc::mma8_ts_vmn_w(d, pa, tc::smem_desc_sw128(va, SUB_BYTES, 1024), idPV, acc ? 1u : 0u);
#else
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    K3_MMA_TS(d, pa + 8 * kk, tc::smem_desc_sw128(va + kk * 2048u, SUB_BYTES, 1024), idPV,
                               (acc || kk > 0) ? 1u : 0u);
#endif
            };
            tc::mbar_wait(&bar->q_ready, 0);
            tc::mbar_wait(&bar->k_full[0], 0);
            tc::fence_after_sync();
            for (int t = 0; t < NT; ++t) {
                issue_S(t, 0);
                K3_COMMIT(&bar->s_full[t]);
            }
            K3_COMMIT(&bar->k_empty[0]);
            for (int j = 0; j < nblk; ++j) {
                const int st = j & 1;
                for (int t = 0; t < NT; ++t) {
                    K3_WAIT(1, &bar->p_full[t], j & 1);
                    K3_TR(2, j, 3 * t);
                    if (t == 0) K3_WAIT(1, &bar->v_full[st], (j >> 1) & 1);
                    K3_TR(2, j, 3 * t + 1);
                    tc::fence_after_sync();
                    issue_PV(t, st, j > 0);
                    if (j == nblk - 1) K3_COMMIT(&bar->o_final[t]);
                    if (t == NT - 1) K3_COMMIT(&bar->v_empty[st]);
                    if (j + 1 < nblk) {
                        const int sn = (j + 1) & 1;
                        if (t == 0) {
                            K3_WAIT(1, &bar->k_full[sn], ((j + 1) >> 1) & 1);
                            tc::fence_after_sync();
                        }
                        issue_S(t, sn);
                        K3_COMMIT(&bar->s_full[t]);
                        K3_TR(2, j, 3 * t + 2);
                        if (t == NT - 1) K3_COMMIT(&bar->k_empty[sn]);
                    }
                }
            }
        }
        __syncwarp();
#undef K3_MMA_SS
#undef K3_MMA_TS
#undef K3_COMMIT
    } else {
        // ================================ softmax ================================
        // warp = (tile t, column half c, lane quarter wq): rows r of tile t,
        // S/P/O columns [HC*c, HC*c + HC).  The two halves of a row exchange
        // their row max through smem (named barrier per row quarter).
        const int t = warp >> 3, c = (warp >> 2) & 1, wq = warp & 3;
        const int r = wq * 32 + lane;  // row inside the tile == TMEM lane
        const long i = i0 + r;
        const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
        const uint32_t colO = 256 * t + HC * c, colS = 256 * t + 128;
        const uint32_t barid = 1 + t * 4 + wq;
        float* xm = reinterpret_cast<float*>(sm + OFF_X) + t * NSPLIT * 128;
        auto pair_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(barid), "r"(NSPLIT * 32) : "memory"); };
        // RoPE(q) in place (engine.cpp:229), pre-scaled by log2(e)/sqrt(d); half c
        // rotates the d-columns of SW128 sub-tile c
        tc::mbar_wait(&bar->q_full, 0);
        {
            const float qs = rsqrtf(128.f) * LOG2E;
            uint8_t* qt = sm + OFF_Q + t * TILE_BYTES;
            const int hh = c;
            for (int cc = 0; cc < 8; ++cc) {
                uint4* p = reinterpret_cast<uint4*>(qt + hh * SUB_BYTES + tc::sw128_off(r, cc));
                uint4 v = *p;
                uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float x0 = __uint_as_float(w[u] << 16), x1 = __uint_as_float(w[u] & 0xffff0000u);
                    float cs, sn;
                    rope_cs_fast(a.freq, hh * 32 + cc * 4 + u, i, cs, sn);
                    w[u] = tc::pack_bf16x2((x0 * cs - x1 * sn) * qs, (x0 * sn + x1 * cs) * qs);
                }
                *p = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&bar->q_ready);

        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nblk; ++j) {
            K3_WAIT(2, &bar->s_full[t], j & 1);
            tc::fence_after_sync();
            if (lane == 0 && c == 0 && wq == 0) K3_TR(t, j, 0);
#ifdef WGKV_DBG_NO_SOFTMAX  // diagnostic: MMA/TMA pipeline speed with the softmax removed
            tc::fence_before_sync();
            tc::mbar_arrive(&bar->p_full[t]);
            continue;
#endif
            uint32_t s0[32], s1[32];
            tc::tmem_ld32(trow + colS + HC * c, s0);
            tc::tmem_ld32(trow + colS + HC * c + 32, s1);
            tc::tmem_ld_wait();
            const uint32_t NEG_INF = 0xff800000u;
            // ---- masks -------------------------------------------------------
            if (j < nv) {
                const int vc = min(128, C - 128 * j);
                if (vc < 128) {
                    auto cut = [&](uint32_t(&x)[32], int base) {
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (base + e >= vc) x[e] = NEG_INF;
                    };
                    cut(s0, HC * c);
                    cut(s1, HC * c + 32);
                }
            } else {
                const long kb0 = s_lo + 128L * (j - nv);
                if (!(kb0 + 127 <= i0 && i0 + 127 - kb0 < W)) {
                    // admitted-key masks of this tile's 64 columns (edge tiles only)
                    const long kc = kb0 + 64 * c + lane;
                    const uint32_t mk0 = __ballot_sync(0xffffffffu, kc < T && bits[kc] != 0);
                    const uint32_t mk1 = __ballot_sync(0xffffffffu, kc + 32 < T && bits[kc + 32] != 0);
                    const long dd = i - kb0;  // key col is causal iff col <= dd; in-window iff dd - col < W
                    auto cut = [&](uint32_t(&x)[32], int w) {
                        const uint32_t mw = (w & 1) ? mk1 : mk0;
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const long col = 32 * w + e;
                            const bool ok = col <= dd && ((dd - col) < W || ((mw >> e) & 1u));
                            if (!ok) x[e] = NEG_INF;
                        }
                    };
                    cut(s0, 2 * c);
                    cut(s1, 2 * c + 1);
                }
            }
#if WGKV_K3_MAX3
            // three-input FMNMX3: 32 instead of 64 max instructions per row half
            float pm[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) pm[e] = max3f(__uint_as_float(s0[e]), __uint_as_float(s0[e + 8]), __uint_as_float(s0[e + 16]));
#pragma unroll
            for (int e = 0; e < 8; ++e) pm[e] = max3f(pm[e], __uint_as_float(s0[e + 24]), __uint_as_float(s1[e]));
#pragma unroll
            for (int e = 0; e < 8; ++e) pm[e] = max3f(pm[e], __uint_as_float(s1[e + 8]), __uint_as_float(s1[e + 16]));
#pragma unroll
            for (int e = 0; e < 8; ++e) pm[e] = fmaxf(pm[e], __uint_as_float(s1[e + 24]));
            float mx = max3f(max3f(pm[0], pm[1], pm[2]), max3f(pm[3], pm[4], pm[5]), fmaxf(pm[6], pm[7]));
#else
            float pm[8] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY};
            auto rmax = [&](const uint32_t(&x)[32]) {
#pragma unroll
                for (int e = 0; e < 32; ++e) pm[e & 7] = fmaxf(pm[e & 7], __uint_as_float(x[e]));
            };
            rmax(s0);
            rmax(s1);
            float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                             fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
#endif
            // both halves hold their S in registers past this barrier, so the
            // P stores below may overwrite any S column
            if (lane == 0 && c == 0 && wq == 0) K3_TR(t, j, 1);
            xm[c * 128 + r] = mx;
            pair_sync();
            mx = fmaxf(mx, xm[(c ^ 1) * 128 + r]);
            if (lane == 0 && c == 0 && wq == 0) K3_TR(t, j, 2);
            // ---- lazy rescale: only when the max grows by more than 2^8 -----
            // (both halves see the same m and mx, so they take the same branch)
            const bool rescale = __any_sync(0xffffffffu, mx > m + 8.f);
            float alpha = 1.f;
            if (rescale) {
                const float mn = fmaxf(m, mx);
                alpha = (m == -INFINITY) ? 0.f : ex2(m - mn);
                l *= alpha;
                m = mn;
            }
            const float mu = (m == -INFINITY) ? 0.f : m;
            // packed f32x2 arithmetic (FADD2) halves the subtract and row-sum
            // instruction count; 4 independent float2 partial sums
            float2 lsv[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
            const float2 nmu = make_float2(-mu, -mu);
            uint32_t pa[32];
            auto expo = [&](const uint32_t(&x)[32], int off) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const float2 xd = __fadd2_rn(make_float2(__uint_as_float(x[2 * e]), __uint_as_float(x[2 * e + 1])), nmu);
                    // selected pairs on the FMA pipe, the rest on the MUFU
                    float e0, e1;
                    if (WGKV_EMU_PACK_INT && ((WGKV_EMU_MASK >> e) & 1)) {
                        pa[off + e] = ex2_emu2_bf16(xd.x, xd.y, e0, e1);
                        lsv[e & 3] = __fadd2_rn(lsv[e & 3], make_float2(e0, e1));
                        continue;
                    }
                    if ((WGKV_EMU_MASK >> e) & 1) {
                        const float2 ee = ex2_emu2(xd.x, xd.y);
                        e0 = ee.x;
                        e1 = ee.y;
                    } else {
                        e0 = ex2(xd.x);
                        e1 = ex2(xd.y);
                    }
                    lsv[e & 3] = __fadd2_rn(lsv[e & 3], make_float2(e0, e1));
                    pa[off + e] = ((WGKV_PACK_ALU >> e) & 1) ? pack_bf16x2_alu(e0, e1) : tc::pack_bf16x2(e0, e1);
                }
            };
            expo(s0, 0);
            expo(s1, 16);
            {
                const float2 a01 = __fadd2_rn(lsv[0], lsv[1]), a23 = __fadd2_rn(lsv[2], lsv[3]);
                const float2 tt = __fadd2_rn(a01, a23);
                l += tt.x + tt.y;
            }
            if (lane == 0 && c == 0 && wq == 0) K3_TR(t, j, 3);
            // P (bf16x2) of keys [HC*c, HC*c + HC) -> packed columns [HC/2*c, ...)
            tc::tmem_st32(trow + colS + (HC / 2) * c, pa);
            // O_t is complete up to PV(j-1) (s_full(j) was committed after it);
            // PV(j) waits for p_full below, so the rescale lands in between
            if (rescale && j > 0) {
#pragma unroll 1
                for (int k = 0; k < HC / 32; ++k) {
                    uint32_t o[32];
                    tc::tmem_ld32(trow + colO + 32 * k, o);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const float2 v = __fmul2_rn(make_float2(__uint_as_float(o[e]), __uint_as_float(o[e + 1])),
                                                    make_float2(alpha, alpha));
                        o[e] = __float_as_uint(v.x);
                        o[e + 1] = __float_as_uint(v.y);
                    }
                    tc::tmem_st32(trow + colO + 32 * k, o);
                }
            }
            tc::tmem_st_wait();
            tc::fence_before_sync();
            tc::mbar_arrive(&bar->p_full[t]);
            if (lane == 0 && c == 0 && wq == 0) K3_TR(t, j, 4);
        }
        // ---- epilogue: O / l -> bf16 (row sum = both halves) -------------------
        tc::mbar_wait(&bar->o_final[t], 0);
        tc::fence_after_sync();
        xm[c * 128 + r] = l;
        pair_sync();
        const float lt = l + xm[(c ^ 1) * 128 + r];
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        __nv_bfloat16* orow = out + (((size_t)s * T + i) * Hq + p0 + t) * 128 + HC * c;
#pragma unroll 1
        for (int k = 0; k < HC / 32; ++k) {
            uint32_t o[32];
            tc::tmem_ld32(trow + colO + 32 * k, o);
            tc::tmem_ld_wait();
            if (i < T) {
                uint4* dst = reinterpret_cast<uint4*>(orow + 32 * k);
                uint4 ov[4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    ov[q4] = make_uint4(tc::pack_bf16x2(__uint_as_float(o[8 * q4]) * inv, __uint_as_float(o[8 * q4 + 1]) * inv),
                                        tc::pack_bf16x2(__uint_as_float(o[8 * q4 + 2]) * inv, __uint_as_float(o[8 * q4 + 3]) * inv),
                                        tc::pack_bf16x2(__uint_as_float(o[8 * q4 + 4]) * inv, __uint_as_float(o[8 * q4 + 5]) * inv),
                                        tc::pack_bf16x2(__uint_as_float(o[8 * q4 + 6]) * inv, __uint_as_float(o[8 * q4 + 7]) * inv));
                    dst[q4] = ov[q4];
                }
                if (a.pb.world) {  // C1: the same 64 bytes into every rank's bulk slot (NVLink stores)
                    const size_t off = a.pb.slot_off +
                                       ((((size_t)s * T + i) * a.pb.world + a.pb.rank) * Hq + p0 + t) * 256 +
                                       (size_t)(HC * c + 32 * k) * 2;
#pragma unroll 1
                    for (int pp = 0; pp < a.pb.world; ++pp) {
                        uint4* pd = reinterpret_cast<uint4*>(a.pb.peers.base[pp] + off);
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) pd[q4] = ov[q4];
                    }
                }
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == WARP_MMA) {
        tc::fence_after_sync();
        tc::tmem_dealloc(tmem, 512);
    }
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_tmap_3d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1, uint32_t box2) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return WGKV_ECUDA;
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
    const cuuint32_t box[3] = {box0, box1, box2};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? WGKV_OK : WGKV_ECUDA;
}

int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t stride1_bytes,
                      uint32_t box0, uint32_t box1) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return WGKV_ECUDA;
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    const cuuint64_t dims[2] = {d0, d1};
    const cuuint64_t strides[1] = {stride1_bytes};
    const cuuint32_t box[2] = {box0, box1};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? WGKV_OK : WGKV_ECUDA;
}

int make_tmap_4d_bf16(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint64_t strides_bytes[3],
                      const uint32_t box[4]) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return WGKV_ECUDA;
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    const cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
    const cuuint64_t st[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
    const cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), d, st, bx, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? WGKV_OK : WGKV_ECUDA;
}

#ifdef WGKV_TRACE
extern "C" int wgkv_dbg_k3_trace(void* host, size_t bytes) {
    return cudaMemcpyFromSymbol(host, g_k3_trace, bytes) == cudaSuccess ? 0 : -1;
}
#endif

int launch_vs_prefill_tc(const VsArgs& a, int nseq, const __nv_bfloat16* q, const __nv_bfloat16* k_post,
                         const __nv_bfloat16* v, __nv_bfloat16* out, cudaStream_t st) {
    const int d = a.pv.head_dim, ps = a.pv.page_size;
    const int Hq = a.q_heads, Hkv = a.pv.kv_heads;
    if (d != 128 || 128 % ps != 0 || ps < 8 || (Hq / Hkv) % NT != 0) return WGKV_ENOTSUP;
    CUtensorMap tq, tk, tv, tp;
    const uint64_t rows = (uint64_t)nseq * a.T;
    int r = make_tmap_3d_bf16(&tq, q, 128, Hq, rows, 256, (uint64_t)Hq * 256, 64, 1, 128);
    r |= make_tmap_3d_bf16(&tk, k_post, 128, Hkv, rows, 256, (uint64_t)Hkv * 256, 64, 1, 128);
    r |= make_tmap_3d_bf16(&tv, v, 128, Hkv, rows, 256, (uint64_t)Hkv * 256, 64, 1, 128);
    r |= make_tmap_3d_bf16(&tp, a.pv.data, 128, ps, 2 * (uint64_t)a.pv.capacity, 256, (uint64_t)ps * 256, 64, ps, 1);
    // K (V) planes of consecutive pages: [page][ps slots][128 dims], page stride = 2 planes
    CUtensorMap tkr, tvr;
    const uint64_t plane = (uint64_t)ps * 256;
    r |= make_tmap_3d_bf16(&tkr, a.pv.data, 128, ps, (uint64_t)a.pv.capacity, 256, 2 * plane, 64, ps, 128 / ps);
    r |= make_tmap_3d_bf16(&tvr, static_cast<const uint8_t*>(a.pv.data) + plane, 128, ps, (uint64_t)a.pv.capacity,
                           256, 2 * plane, 64, ps, 128 / ps);
    if (r) return WGKV_ECUDA;
    if (ensure_smem(vs_prefill_tc_kernel, SMEM_BYTES) != cudaSuccess) return WGKV_ECUDA;
    dim3 grid((unsigned)((a.T + 127) / 128), Hq / NT, nseq);
    vs_prefill_tc_kernel<<<grid, NTHREADS, SMEM_BYTES, st>>>(tq, tk, tv, tp, tkr, tvr, a, out);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

}  // namespace wgkv
