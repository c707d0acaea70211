// gate_proj.cu -- f1: the key projection fused into K1.
//
// Session::prefill forms, per kv head h and token t (engine.cpp:190-205),
//   k_pre[t]  = Wk[h*d .. h*d+d-1] . a[t]         (the projection)
//   k_post[t] = RoPE(k_pre[t], t)                 (apply_rope_inplace)
//   g[t]      = gate_forward([k_pre; k_post])     (gate_forward_batch)
// and the bits are binarize(g).  gate_tc.cu (K1) starts from a k_pre tensor in
// HBM; this kernel starts from the layer input a [nseq][T][dm] and the head's
// Wk rows, so k_pre never makes a round trip before the gate: per 128-token
// tile of one (seq, kv head), a tcgen05 GEMM accumulates the projection tile
// in TMEM (M = 128 tokens, N = 128 dims, K = dm, a / Wk streamed by TMA
// through a 3-stage ring), the producer warps read it from TMEM, round it to
// bf16 (the k_pre the gate and the recheck see, also written out for the fp64
// recheck and for callers), rotate it, and build the gate GEMM's A tiles in
// the same shared memory the ring used; then K1's split-bf16 gate GEMM (5
// segments, W1 hi/lo tiles resident per head) and K1's epilogue (fast-erf
// GELU, w2 dot, sigmoid, threshold, recheck band) run unchanged.
//
// Layout: Wk rows of this context's kv heads, [kv_heads][d][dm] bf16 row-major
// (LayerWeights::wk, model.hpp:24-31, rows h*d + r); a [nseq][T][dm] bf16.
//
// Persistent, one CTA per SM over contiguous (seq, kv head, tile) ranges in
// head order (W1 tiles reload only when the head changes).  Roles (544 threads):
//   warps 0-7   producers: warp w reads TMEM lane quarter w%4, dims 64*(w/4)..
//   warp 8      TMEM owner, TMA (a / Wk ring, W1 tiles) and MMA issuer
//   warps 9-16  epilogue, two groups taking alternate tiles / TMEM buffers
// TMEM: Z0 [0,128) | Z1 [128,256) | P [256,384) (projection accumulator).
#include <cuda.h>

#include <algorithm>

#include "gate.cuh"
#include "tc.cuh"

namespace wgkv {

namespace {
constexpr uint32_t GP_TILE = 128 * 128 * 2;       // [128][128] bf16 operand tile (2 SW128 sub-tiles)
constexpr uint32_t GP_SUB = GP_TILE / 2;          // [128][64] SW128 sub-tile
constexpr uint32_t GP_OFF_B = 0;                  // 4 B tiles: Wpre_hi, Wpost_hi, Wpre_lo, Wpost_lo
constexpr uint32_t GP_OFF_A = 4 * GP_TILE;        // 3 A tiles (k_pre, k_post hi, lo) == the projection ring
constexpr int GP_RING = 3;                        // ring stages: [a 128x64 | Wk 128x64] = 32 KB each
constexpr uint32_t GP_STAGE = 2 * GP_SUB;
constexpr uint32_t GP_OFF_BAR = GP_OFF_A + 3 * GP_TILE;
// |x|^2 partials per (token row, dim half), bf16 rounded up, slot it % 3.  The
// epilogue of tile i reads its slot before arriving on t_empty; the gate MMAs
// of tile i+2 wait for that arrival, the projection of tile i+3 for those MMAs
// (hl_empty) and its producer for the projection (p_full): slot i is free.
constexpr int GP_XX_SLOTS = 3;
constexpr uint32_t GP_OFF_XX = GP_OFF_BAR + 256;  // [slot][half][128] bf16
constexpr uint32_t GP_SMEM = GP_OFF_XX + GP_XX_SLOTS * 2 * 128 * 2 + 1024;
static_assert(GP_SMEM <= 227 * 1024, "gate_proj shared memory");
static_assert(GP_RING * GP_STAGE <= 3 * GP_TILE, "ring inside the A region");
constexpr int GP_PROD = 256, GP_EPI = 256;
constexpr int GP_THREADS = GP_PROD + 32 + GP_EPI;  // 544
constexpr uint32_t COL_P = 256;

__device__ __forceinline__ uint64_t kdesc(uint32_t tile, int kk) {
    return tc::smem_desc_sw128(tile + (uint32_t)(kk >> 2) * GP_SUB + (uint32_t)(kk & 3) * 32u, 16, 1024);
}
// one [128][64] SW128 sub-tile, K step kk of 4
__device__ __forceinline__ uint64_t sdesc(uint32_t sub, int kk) {
    return tc::smem_desc_sw128(sub + (uint32_t)kk * 32u, 16, 1024);
}
constexpr float ERF_EPS = 1.0e-6f;
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// the same fast GELU as gate_tc.cu (Eigen's rational erf; error bound ERF_EPS)
__device__ __forceinline__ float2 gelu_fast2(float2 z1) {
    float2 x = __fmul2_rn(z1, f2(0.70710678118654752f));
    x.x = fminf(fmaxf(x.x, -4.f), 4.f);
    x.y = fminf(fmaxf(x.y, -4.f), 4.f);
    const float2 x2 = __fmul2_rn(x, x);
    float2 p = __ffma2_rn(x2, f2(-2.72614225801306e-10f), f2(2.77068142495902e-08f));
    p = __ffma2_rn(x2, p, f2(-2.10102402082508e-06f));
    p = __ffma2_rn(x2, p, f2(-5.69250639462346e-05f));
    p = __ffma2_rn(x2, p, f2(-7.34990630326855e-04f));
    p = __ffma2_rn(x2, p, f2(-2.95459980854025e-03f));
    p = __ffma2_rn(x2, p, f2(-1.60960333262415e-02f));
    p = __fmul2_rn(p, x);
    float2 q = __ffma2_rn(x2, f2(-1.45660718464996e-05f), f2(-2.13374055278905e-04f));
    q = __ffma2_rn(x2, q, f2(-1.68282697438203e-03f));
    q = __ffma2_rn(x2, q, f2(-7.37332916720468e-03f));
    q = __ffma2_rn(x2, q, f2(-1.42647390514189e-02f));
    const float2 e = __fmul2_rn(p, make_float2(rcp_approx(q.x), rcp_approx(q.y)));
    const float2 hz = __fmul2_rn(z1, f2(0.5f));
    return __ffma2_rn(hz, e, hz);
}
__device__ __forceinline__ uint16_t bf16_bits(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }
}  // namespace

struct GateProjArgs {
    GateArgs g;
    int nseq, dm;
    long tiles_per_pair, total_tiles;
    // head-interleaved schedule (head_sched = 1): CTA k takes kv head k % H and the
    // (k / H)-th of gridDim / H contiguous ranges of token tiles, so the H CTAs of
    // a range stream the same layer-input tiles at the same time (one HBM read,
    // the other heads hit L2) while each CTA keeps one head's W1 resident
    int head_sched;
    const float2* rope;  // [T][d/2] (cos, sin) of position pos0 + t
};

__global__ void __launch_bounds__(GP_THREADS, 1)
    gate_proj_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap ta,
                     const __grid_constant__ CUtensorMap twk, GateProjArgs A, __nv_bfloat16* __restrict__ k_pre,
                     __nv_bfloat16* __restrict__ k_post, float* __restrict__ g_out, uint8_t* __restrict__ bits_out,
                     int32_t* __restrict__ cand, int* __restrict__ pcnt) {
    extern __shared__ uint8_t gsm_raw[];
    // 1 KB-aligned, by pointer arithmetic on the __shared__ array (an integer round
    // trip would lose the address space: every access through sm would be generic)
    uint8_t* sm = gsm_raw + ((1024u - (smem_u32(gsm_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(sm);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + GP_OFF_BAR);
    uint64_t* b_full = bars + 0;
    uint64_t* r_full = bars + 1;    // [GP_RING]
    uint64_t* r_empty = bars + 4;   // [GP_RING]
    uint64_t* p_full = bars + 7;    // projection tile complete in TMEM
    uint64_t* p_read = bars + 8;    // producers hold it in registers
    uint64_t* hl_full = bars + 9;   // A tiles written
    uint64_t* hl_empty = bars + 10; // gate MMAs done with the A tiles (the ring may refill)
    uint64_t* t_full = bars + 11;   // [2]
    uint64_t* t_empty = bars + 13;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
    __nv_bfloat16* xxs = reinterpret_cast<__nv_bfloat16*>(sm + GP_OFF_XX);
    const GateArgs& a = A.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long t_begin, t_end;
    int hsched = 0;  // this CTA's kv head (head-interleaved schedule)
    if (A.head_sched) {
        const int R = (int)gridDim.x / a.kv_heads, r = (int)blockIdx.x / a.kv_heads;
        hsched = (int)blockIdx.x % a.kv_heads;
        const long ntt = (long)A.nseq * A.tiles_per_pair;  // token tiles over all sequences
        t_begin = ntt * r / R;
        t_end = ntt * (r + 1) / R;
    } else {
        t_begin = A.total_tiles * blockIdx.x / gridDim.x;
        t_end = A.total_tiles * (blockIdx.x + 1) / gridDim.x;
    }
    // tile -> (seq * kv_heads + head, first token)
    auto pair_of = [&](long tile) -> int {
        return A.head_sched ? (int)(tile / A.tiles_per_pair) * a.kv_heads + hsched : (int)(tile / A.tiles_per_pair);
    };
    const int nk = A.dm / 64;  // projection K steps of 64
    if (threadIdx.x == 0) {
        tc::mbar_init(b_full, 1);
        for (int i = 0; i < GP_RING; ++i) {
            tc::mbar_init(&r_full[i], 1);
            tc::mbar_init(&r_empty[i], 1);
        }
        tc::mbar_init(p_full, 1);
        tc::mbar_init(p_read, GP_PROD);
        tc::mbar_init(hl_full, GP_PROD);
        tc::mbar_init(hl_empty, 1);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&t_full[b], 1);
            tc::mbar_init(&t_empty[b], GP_EPI / 2);
        }
        tc::fence_barrier_init();
    }
    if (warp == 8) tc::tmem_alloc(tmem_slot, 512);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp < 8) {
        // ============ producers: P (TMEM) -> k_pre (bf16) -> RoPE -> A tiles ============
        const int quarter = warp & 3, half = warp >> 2;
        const int r = quarter * 32 + lane;  // token row == TMEM lane
        const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16) + COL_P + 64u * half;
        for (long tile = t_begin; tile < t_end; ++tile) {
            const int it = (int)(tile - t_begin);
            const int pair = pair_of(tile);
            const long t0 = (tile % A.tiles_per_pair) * 128;
            const int s = pair / a.kv_heads, h = pair % a.kv_heads;
            const long t = t0 + r;
            const bool valid = t < a.T;
            const size_t off = (((size_t)s * a.T + min(t, a.T - 1)) * a.kv_heads + h) * 128 + 64 * half;
            const float4* rt = reinterpret_cast<const float4*>(A.rope + (size_t)min(t, a.T - 1) * 64) + 16 * half;
            tc::mbar_wait_sleep(p_full, it & 1);
            tc::fence_after_sync();
            float xx = 0.f;
            uint4* dpre = reinterpret_cast<uint4*>(k_pre + off);
            uint4* dpost = reinterpret_cast<uint4*>(k_post + off);
#pragma unroll 1
            for (int q = 0; q < 2; ++q) {  // 32 projected dims at a time (register budget)
                uint32_t pv[32];
                tc::tmem_ld32(trow + 32 * q, pv);
                tc::tmem_ld_wait();
                if (q == 1) {  // the whole tile is in registers or written: P may be overwritten
                    tc::fence_before_sync();
                    tc::mbar_arrive(p_read);
                }
                // (the ring's last MMAs completed before p_full: the A region is free)
#pragma unroll
                for (int uu = 0; uu < 4; ++uu) {  // 16-byte chunk u = dims 64*half + 8u .. +7
                    const int u = 4 * q + uu;
                    const float4 cs0 = __ldg(rt + 2 * u), cs1 = __ldg(rt + 2 * u + 1);
                    const float cc[4] = {cs0.x, cs0.z, cs1.x, cs1.z};
                    const float ss[4] = {cs0.y, cs0.w, cs1.y, cs1.w};
                    uint32_t pre[4], hi[4], lo[4];
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        const uint16_t b0 = bf16_bits(__uint_as_float(pv[8 * uu + 2 * p]));
                        const uint16_t b1 = bf16_bits(__uint_as_float(pv[8 * uu + 2 * p + 1]));
                        pre[p] = (uint32_t)b0 | ((uint32_t)b1 << 16);
                        const float x0 = __uint_as_float((uint32_t)b0 << 16), x1 = __uint_as_float((uint32_t)b1 << 16);
                        const float y0 = x0 * cc[p] - x1 * ss[p], y1 = x0 * ss[p] + x1 * cc[p];
                        xx = fmaf(x0, x0, fmaf(x1, x1, fmaf(y0, y0, fmaf(y1, y1, xx))));
                        const uint16_t h0 = bf16_bits(y0), h1 = bf16_bits(y1);
                        const float r0 = y0 - __uint_as_float((uint32_t)h0 << 16);
                        const float r1 = y1 - __uint_as_float((uint32_t)h1 << 16);
                        hi[p] = (uint32_t)h0 | ((uint32_t)h1 << 16);
                        lo[p] = (uint32_t)bf16_bits(r0) | ((uint32_t)bf16_bits(r1) << 16);
                    }
                    const uint32_t so = (uint32_t)half * GP_SUB + tc::sw128_off(r, u);
                    const uint4 pw = make_uint4(pre[0], pre[1], pre[2], pre[3]);
                    const uint4 hv = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<uint4*>(sm + GP_OFF_A + so) = pw;
                    *reinterpret_cast<uint4*>(sm + GP_OFF_A + GP_TILE + so) = hv;
                    *reinterpret_cast<uint4*>(sm + GP_OFF_A + 2 * GP_TILE + so) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                    if (valid) {
                        dpre[u] = pw;
                        dpost[u] = hv;
                    }
                }
            }
            xxs[((it % GP_XX_SLOTS) * 2 + half) * 128 + r] = __float2bfloat16_ru(xx);  // upper bound for the band
            tc::fence_proxy_async_smem();
            tc::mbar_arrive(hl_full);
        }
    } else if (warp == 8) {
        // ============ TMA + MMA issuer ============
        constexpr uint32_t idG = tc::idesc_bf16(128, 128, false, false);
        const uint32_t Apre = sbase + GP_OFF_A, Ahi = Apre + GP_TILE, Alo = Apre + 2 * GP_TILE;
        const uint32_t Bph = sbase + GP_OFF_B, Bqh = Bph + GP_TILE, Bpl = Bph + 2 * GP_TILE, Bql = Bph + 3 * GP_TILE;
        int cur_blk = -1, b_loads = 0;
        long rl = 0;  // ring loads issued so far (stage = rl % GP_RING, phase = (rl / GP_RING) & 1)
        long rc = 0;  // ring stages consumed so far
        auto ring_load = [&](int s, int h, long t0, int kb) {
            const int st = (int)(rl % GP_RING);
            if (rl >= GP_RING) tc::mbar_wait(&r_empty[st], (int)(((rl / GP_RING) - 1) & 1));
            if (lane == 0) {
                uint8_t* dst = sm + GP_OFF_A + st * GP_STAGE;
                tc::mbar_arrive_expect_tx(&r_full[st], GP_STAGE);
                tc::tma_load_2d(dst, &ta, &r_full[st], kb * 64, s * (int)a.T + (int)t0);
                tc::tma_load_2d(dst + GP_SUB, &twk, &r_full[st], kb * 64, h * 128);
            }
            __syncwarp();
            ++rl;
        };
        for (long tile = t_begin; tile < t_end; ++tile) {
            const int it = (int)(tile - t_begin);
            const int pair = pair_of(tile);
            const long t0 = (tile % A.tiles_per_pair) * 128;
            const int s = pair / a.kv_heads, h = pair % a.kv_heads;
            const int blk = a.layer * a.kv_heads + h;
            // the A region (ring) and P are free once the previous tile's gate
            // MMAs are done and the producers have read its projection
            if (it > 0) {
                tc::mbar_wait(hl_empty, (it - 1) & 1);
                tc::mbar_wait(p_read, (it - 1) & 1);
            }
            if (blk != cur_blk) {
                if (lane == 0) {
                    tc::mbar_arrive_expect_tx(b_full, 4 * GP_TILE);
                    for (int q = 0; q < 4; ++q)
                        for (int hh = 0; hh < 2; ++hh)
                            tc::tma_load_3d(sm + GP_OFF_B + q * GP_TILE + hh * GP_SUB, &tw, b_full, hh * 64, 0,
                                            blk * 4 + q);
                }
                __syncwarp();
            }
            // ---- projection: P = a_tile . Wk_h^T over dm ----
            const int pre = min(GP_RING, nk);
            for (int kb = 0; kb < pre; ++kb) ring_load(s, h, t0, kb);
            for (int kb = 0; kb < nk; ++kb) {
                const int st = (int)(rc % GP_RING);
                tc::mbar_wait(&r_full[st], (int)((rc / GP_RING) & 1));
                tc::fence_after_sync();
                const uint32_t sa = sbase + GP_OFF_A + st * GP_STAGE;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    tc::mma_ss_w(tmem + COL_P, sdesc(sa, kk), sdesc(sa + GP_SUB, kk), idG, (kb | kk) ? 1u : 0u);
                tc::mma_commit_w(&r_empty[st]);
                ++rc;
                if (kb + GP_RING < nk) ring_load(s, h, t0, kb + GP_RING);
            }
            tc::mma_commit_w(p_full);
            if (blk != cur_blk) {
                tc::mbar_wait(b_full, b_loads & 1);
                ++b_loads;
                cur_blk = blk;
            }
            // ---- gate: z1 = W1 . [k_pre ; k_post] in 5 split segments (gate_tc.cu) ----
            const int buf = it & 1;
            const uint32_t dt = tmem + (uint32_t)buf * 128u;
            tc::mbar_wait(hl_full, it & 1);
            if (it >= 2) tc::mbar_wait(&t_empty[buf], ((it - 2) >> 1) & 1);
            tc::fence_after_sync();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) tc::mma_ss_w(dt, kdesc(Apre, kk), kdesc(Bph, kk), idG, kk ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) tc::mma_ss_w(dt, kdesc(Apre, kk), kdesc(Bpl, kk), idG, 1u);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) tc::mma_ss_w(dt, kdesc(Ahi, kk), kdesc(Bqh, kk), idG, 1u);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) tc::mma_ss_w(dt, kdesc(Ahi, kk), kdesc(Bql, kk), idG, 1u);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) tc::mma_ss_w(dt, kdesc(Alo, kk), kdesc(Bqh, kk), idG, 1u);
            tc::mma_commit_w(hl_empty);
            tc::mma_commit_w(&t_full[buf]);
        }
        __syncwarp();
    } else {
        // ============ epilogue (gate_tc.cu) ============
        const int grp = (warp - 9) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const float u_eff = 3.0e-5f;
        for (long tile = t_begin + grp; tile < t_end; tile += 2) {
            const int it = (int)(tile - t_begin);
            const int pair = pair_of(tile);
            const long t0 = (tile % A.tiles_per_pair) * 128;
            const int s = pair / a.kv_heads, h = pair % a.kv_heads;
            const int blk = a.layer * a.kv_heads + h;
            const float4* bw = a.bw + (size_t)blk * 64;
            tc::mbar_wait_sleep(&t_full[grp], (it >> 1) & 1);
            tc::fence_after_sync();
            const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)grp * 128u;
            float2 part = make_float2(0.f, 0.f), az = make_float2(0.f, 0.f);
#pragma unroll 1
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t z[32];
                tc::tmem_ld32(trow + 32 * cc, z);
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float4 c = __ldg(bw + 16 * cc + j);
                    const float2 z1 = __fadd2_rn(make_float2(__uint_as_float(z[2 * j]), __uint_as_float(z[2 * j + 1])),
                                                 make_float2(c.x, c.y));
                    const float2 ge = gelu_fast2(z1);
                    part = __ffma2_rn(make_float2(c.z, c.w), ge, part);
                    az = __ffma2_rn(make_float2(fabsf(c.z), fabsf(c.w)), make_float2(fabsf(z1.x), fabsf(z1.y)), az);
                }
            }
            const __nv_bfloat16* xs = xxs + (it % GP_XX_SLOTS) * 256;
            const float xx = __bfloat162float(xs[row]) + __bfloat162float(xs[128 + row]);
            tc::fence_before_sync();
            tc::mbar_arrive(&t_empty[grp]);
            const long t = t0 + row;
            if (t < a.T) {
                const float z2 = (float)a.b2f[blk] + (part.x + part.y);
                const float azs = az.x + az.y;
                const size_t gi = ((size_t)s * a.kv_heads + h) * a.T + t;
                g_out[gi] = 1.f / (1.f + __expf(-z2));
                bits_out[gi] = z2 >= a.ztau ? 1 : 0;
                const float band =
                    4.f * (1.13f * u_eff * sqrtf(xx) * a.bandc[blk] + 0.5f * ERF_EPS * azs +
                           134.f * 5.9604645e-8f * (azs + fabsf((float)a.b2f[blk]) + fabsf(a.ztau)));
                if (fabsf(z2 - a.ztau) <= band) cand[(size_t)pair * a.T + atomicAdd(&pcnt[pair], 1)] = (int32_t)t;
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 8) {
        tc::fence_after_sync();
        tc::tmem_dealloc(tmem, 512);
    }
}


int launch_gate_proj_tc(const GateArgs& a, int nseq, const __nv_bfloat16* x, const __nv_bfloat16* wk, int dm,
                        __nv_bfloat16* k_pre, __nv_bfloat16* k_post, float* g, uint8_t* bits, int32_t* cand, int* pcnt,
                        const __nv_bfloat16* w1split, long n_wtiles, float2* rope_ws, cudaStream_t st) {
    if (a.d != 128 || a.hidden != 128 || dm < 64 || dm % 64 != 0) return WGKV_ENOTSUP;
    CUtensorMap tw, ta, twk;
    if (make_tmap_3d_bf16(&tw, w1split, 128, 128, (uint64_t)n_wtiles, 256, 128 * 256, 64, 128, 1)) return WGKV_ECUDA;
    // a as [nseq*T rows][dm], Wk as [kv_heads*128 rows][dm]: boxes {64 k, 128 rows}
    if (make_tmap_2d_bf16(&ta, x, (uint64_t)dm, (uint64_t)nseq * a.T, (uint64_t)dm * 2, 64, 128)) return WGKV_ECUDA;
    if (make_tmap_2d_bf16(&twk, wk, (uint64_t)dm, (uint64_t)a.kv_heads * 128, (uint64_t)dm * 2, 64, 128))
        return WGKV_ECUDA;
    if (ensure_smem(gate_proj_kernel, GP_SMEM) != cudaSuccess) return WGKV_ECUDA;
    launch_rope_table(a.freq, a.pos0, a.T, a.d / 2, rope_ws, st);
    GateProjArgs A;
    A.g = a;
    A.nseq = nseq;
    A.dm = dm;
    A.tiles_per_pair = (a.T + 127) / 128;
    A.total_tiles = A.tiles_per_pair * nseq * a.kv_heads;
    A.rope = rope_ws;
    const int R = num_sms() / a.kv_heads;  // token-tile ranges per head
    A.head_sched = R >= 1 && (long)nseq * A.tiles_per_pair >= R;
    const int grid = A.head_sched ? R * a.kv_heads : (int)std::min<long>(num_sms(), A.total_tiles);
    gate_proj_kernel<<<grid, GP_THREADS, GP_SMEM, st>>>(tw, ta, twk, A, k_pre, k_post, g, bits, cand, pcnt);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

}  // namespace wgkv
