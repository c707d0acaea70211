// gate_tc.cu -- K1 on the 5th-gen tensor cores: z1 = W1 . [k_pre ; k_post]
// as a tcgen05 GEMM (M = 128 tokens, N = 128 hidden, K = 2d = 256) with a
// split-bf16 scheme that keeps ~fp32 accuracy:
//     k_pre        is exact in bf16 (it is the bf16 input);
//     k_post = hi + lo,  W1 = W_hi + W_lo   (bf16 pairs, |rest| <= 2^-17 rel.)
//     z1 = Apre.(Wpre_hi + Wpre_lo) + Ahi.(Wpost_hi + Wpost_lo) + Alo.Wpost_hi
// i.e. 5 K=128 segments accumulated in one fp32 TMEM tile.  The epilogue adds
// b1, applies the exact-erf GELU, the w2 dot, sigmoid and threshold, and lists
// tokens inside a worst-case error band for the fp64 recheck (gate.cu), so the
// final bits are the reference's (gating.cpp:158-190) except reported
// |g - tau| < 1e-6 tokens.
//
// Persistent, one CTA per SM walking a contiguous range of (seq, kv head,
// 128-token tile) ordered by head (W1's split tiles are reloaded by TMA only
// when the head changes).  Three warp roles run as a pipeline:
//   warps 0-7   producers: read the k_pre tile (TMA'd into the SW128 A layout),
//               rotate with the per-call cos/sin table (rope_table_kernel: the
//               same rope_cs values, computed once per position instead of once
//               per (position, head)), split into hi/lo, write the hi/lo A
//               tiles and k_post; two threads per token row (64 dims each);
//   warp 8      TMEM owner, TMA (W1 splits, k_pre) and MMA issuer: 40 MMAs
//               per tile into one of two TMEM accumulators, the k_pre segments
//               first so they overlap the producers' hi/lo work;
//   warps 9-16  epilogue from TMEM: two groups of 4 warps (one per 32-row
//               lane quarter) that take alternate tiles / TMEM buffers.
// A is single-buffered (B + A fill 224 KB of smem) but released per operand:
// the k_pre tile of i+1 loads while the MMAs of i still read hi/lo, and the
// epilogue drains tile i from the other TMEM buffer.
#include <cuda.h>

#include <algorithm>

#include "gate.cuh"
#include "tc.cuh"

namespace wgkv {

namespace {
constexpr uint32_t GT_TILE = 128 * 128 * 2;  // one [128][128] bf16 operand tile (2 SW128 sub-tiles)
constexpr uint32_t GT_SUB = GT_TILE / 2;
constexpr uint32_t G_OFF_B = 0;               // 4 B tiles: Wpre_hi, Wpost_hi, Wpre_lo, Wpost_lo
constexpr uint32_t G_OFF_A = 4 * GT_TILE;     // 3 A tiles: k_pre, k_post hi, k_post lo
constexpr uint32_t G_OFF_BAR = G_OFF_A + 3 * GT_TILE;
// |x|^2 per token row, bf16 rounded up, slot it % 6.  The producer of tile
// i+5 runs after the MMAs of tile i+4 were issued, which waited for the
// epilogue of tile i+2 to arrive -- after that epilogue group read slot i.
constexpr int XX_SLOTS = 6;
constexpr uint32_t G_OFF_XX = G_OFF_BAR + 128;
constexpr uint32_t G_SMEM = G_OFF_XX + XX_SLOTS * 128 * 2 + 1024;
static_assert(G_SMEM <= 227 * 1024, "K1 shared memory");
constexpr int G_PROD = 256, G_EPI = 256;
constexpr int G_THREADS = G_PROD + 32 + G_EPI;  // 544

__device__ __forceinline__ uint64_t kdesc(uint32_t tile, int kk) {
    return tc::smem_desc_sw128(tile + (uint32_t)(kk >> 2) * GT_SUB + (uint32_t)(kk & 3) * 32u, 16, 1024);
}
// erf on [-4, 4] (clamped outside) as the odd/even rational p(x)/q(x) of
// Eigen's generic_fast_erf_float, in packed f32x2 arithmetic with the MUFU
// reciprocal.  Max |error| over EVERY fp32 input, measured exhaustively with
// this operation order (FMA, exact reciprocal): 4.4e-7; rcp.approx adds
// <= 2^-22 relative.  ERF_EPS = 1e-6 is the bound the recheck band uses.
constexpr float ERF_EPS = 1.0e-6f;
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 gelu_fast2(float2 z1) {  // z1 * Phi(z1) = z1/2 (1 + erf(z1/sqrt2))
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
__device__ __forceinline__ uint16_t bf16_bits(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}
}  // namespace

struct GateTcArgs {
    GateArgs g;
    int nseq;
    int head_sched;
    long tiles_per_pair;
    long total_tiles;
    const float2* rope;  // [T][d/2] (cos, sin) of position pos0 + t
};

__global__ void __launch_bounds__(G_THREADS, 1)
    gate_tc_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tk,
                   const __grid_constant__ CUtensorMap tpost, GateTcArgs A, const __nv_bfloat16* __restrict__ k_pre,
                   __nv_bfloat16* __restrict__ k_post, float* __restrict__ g_out, uint8_t* __restrict__ bits_out,
                   int32_t* __restrict__ cand, int* __restrict__ pcnt) {
    extern __shared__ uint8_t gsm_raw[];
    // 1 KB-aligned, by pointer arithmetic on the __shared__ array (an integer round
    // trip would lose the address space: every access through sm would be generic)
    uint8_t* sm = gsm_raw + ((1024u - (smem_u32(gsm_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(sm);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + G_OFF_BAR);
    uint64_t* b_full = bars + 0;
    uint64_t* t_full = bars + 3;    // [2]
    uint64_t* t_empty = bars + 5;   // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);  // (bars + 13: st_read)
    __nv_bfloat16* xxs = reinterpret_cast<__nv_bfloat16*>(sm + G_OFF_XX);
    const GateArgs& a = A.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // head-interleaved schedule (head_sched): CTA k takes kv head k % H and the
    // (k / H)-th of gridDim / H ranges of token tiles, so the H CTAs of a range
    // walk the same positions together (the cos/sin table rows are shared in L2)
    // and each keeps its head's W1 resident
    long t_begin, t_end;
    int hsched = 0;
    if (A.head_sched) {
        const int R = (int)gridDim.x / a.kv_heads, r = (int)blockIdx.x / a.kv_heads;
        hsched = (int)blockIdx.x % a.kv_heads;
        const long ntt = (long)A.nseq * A.tiles_per_pair;
        t_begin = ntt * r / R;
        t_end = ntt * (r + 1) / R;
    } else {
        t_begin = A.total_tiles * blockIdx.x / gridDim.x;
        t_end = A.total_tiles * (blockIdx.x + 1) / gridDim.x;
    }
    auto pair_of = [&](long tile) -> int {
        return A.head_sched ? (int)(tile / A.tiles_per_pair) * a.kv_heads + hsched : (int)(tile / A.tiles_per_pair);
    };
    uint64_t* pre_full = bars + 7;  // k_pre tile landed (TMA)
    uint64_t* pre_empty = bars + 8; // MMAs of segments 1-2 (the k_pre operand) done
    uint64_t* hl_full = bars + 9;   // producers wrote the hi / lo tiles
    uint64_t* hl_empty = bars + 10; // MMAs of segments 3-5 (hi / lo operands) done
    uint64_t* pre_read = bars + 11; // producers hold the k_pre tile in registers
    uint64_t* st_read = bars + 13;  // the k_post (= hi) tile's TMA store has read shared memory
    if (threadIdx.x == 0) {
        tc::mbar_init(b_full, 1);
        tc::mbar_init(pre_full, 1);
        tc::mbar_init(pre_empty, 1);
        tc::mbar_init(hl_full, G_PROD);
        tc::mbar_init(hl_empty, 1);
        tc::mbar_init(pre_read, G_PROD);
        tc::mbar_init(st_read, 1);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&t_full[b], 1);
            tc::mbar_init(&t_empty[b], G_EPI / 2);
        }
        tc::fence_barrier_init();
    }
    if (warp == 8) tc::tmem_alloc(tmem_slot, 256);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp < 8) {
        // ======================= producers: hi / lo tiles ====================
        // k_pre arrives by TMA in the SW128 A layout; each thread takes its half
        // row (64 dims) into registers (releasing the tile for the next load),
        // then, once the previous tile's MMAs have released hi / lo, rotates
        // it, writes k_post and the hi / lo operand rows.
        const int r = threadIdx.x >> 1, half = threadIdx.x & 1;  // adjacent lanes share a row
        for (long tile = t_begin; tile < t_end; ++tile) {
            const int it = (int)(tile - t_begin);
            const int pair = pair_of(tile);
            const long t0 = (tile % A.tiles_per_pair) * 128;
            const int s = pair / a.kv_heads, h = pair % a.kv_heads;
            const long t = t0 + r;
            const bool valid = t < a.T;
            const size_t off = (((size_t)s * a.T + min(t, a.T - 1)) * a.kv_heads + h) * 128;
            const float4* rt = reinterpret_cast<const float4*>(A.rope + (size_t)min(t, a.T - 1) * 64) + 16 * half;
            uint4* dpost = reinterpret_cast<uint4*>(k_post + off) + 8 * half;
            float4 cs[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) cs[q] = __ldg(rt + q);  // cos/sin of the first 8 pairs
            // take the k_pre half-row into registers and release the k_pre tile
            // so the next one can be loaded while this tile is finished
            tc::mbar_wait_sleep(pre_full, it & 1);
            uint4 raw8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                raw8[u] = *reinterpret_cast<const uint4*>(sm + G_OFF_A + (uint32_t)half * GT_SUB + tc::sw128_off(r, u));
            tc::mbar_arrive(pre_read);
            if (it > 0) {
                tc::mbar_wait_sleep(hl_empty, (it - 1) & 1);  // previous tile's hi / lo consumed by the MMAs
                tc::mbar_wait_sleep(st_read, (it - 1) & 1);   // and the hi tile read by its k_post store
            }
            float xx = 0.f;
#pragma unroll
            for (int u4 = 0; u4 < 8; u4 += 2) {
                if (u4) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) cs[q] = __ldg(rt + 2 * u4 + q);  // cos/sin of 8 pairs
                }
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int u = u4 + v;
                    const uint32_t so = (uint32_t)half * GT_SUB + tc::sw128_off(r, u);
                    const uint4 raw = raw8[u];
                    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
                    const float cc[4] = {cs[2 * v].x, cs[2 * v].z, cs[2 * v + 1].x, cs[2 * v + 1].z};
                    const float ss[4] = {cs[2 * v].y, cs[2 * v].w, cs[2 * v + 1].y, cs[2 * v + 1].w};
                    uint32_t hi[4], lo[4];
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        const float x0 = __uint_as_float(w[p] << 16), x1 = __uint_as_float(w[p] & 0xffff0000u);
                        const float y0 = x0 * cc[p] - x1 * ss[p], y1 = x0 * ss[p] + x1 * cc[p];
                        xx = fmaf(x0, x0, fmaf(x1, x1, fmaf(y0, y0, fmaf(y1, y1, xx))));
                        const uint16_t h0 = bf16_bits(y0), h1 = bf16_bits(y1);
                        const float r0 = y0 - __uint_as_float((uint32_t)h0 << 16);
                        const float r1 = y1 - __uint_as_float((uint32_t)h1 << 16);
                        hi[p] = (uint32_t)h0 | ((uint32_t)h1 << 16);
                        lo[p] = (uint32_t)bf16_bits(r0) | ((uint32_t)bf16_bits(r1) << 16);
                    }
                    const uint4 hv = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<uint4*>(sm + G_OFF_A + GT_TILE + so) = hv;
                    *reinterpret_cast<uint4*>(sm + G_OFF_A + 2 * GT_TILE + so) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                    (void)dpost;
                }
            }
            xx += __shfl_xor_sync(0xffffffffu, xx, 1);
            if (half == 0) xxs[(it % XX_SLOTS) * 128 + r] = __float2bfloat16_ru(xx);  // upper bound for the band
            tc::fence_proxy_async_smem();
            tc::mbar_arrive(hl_full);
        }
    } else if (warp == 8) {
        // ======================= TMA + MMA issuer ============================
        // per tile: S1 = Apre.Bpre_hi, S2 = Apre.Bpre_lo (need only the TMA'd
        // k_pre) -> commit pre_empty; then, once the producers are done,
        // S3 = Ahi.Bpost_hi, S4 = Ahi.Bpost_lo, S5 = Alo.Bpost_hi -> commit
        // hl_empty + t_full; the next k_pre tile is loaded as soon as S1-S2
        // completed (and the producers have read the current one).
        // the whole warp runs the loop (warp-uniform operands stay in uniform
        // registers); elect.sync / lane 0 issue the tcgen05 and TMA operations
        {
            int cur_blk = -1, b_loads = 0;
            constexpr uint32_t idG = tc::idesc_bf16(128, 128, false, false);
            const uint32_t Apre = sbase + G_OFF_A, Ahi = Apre + GT_TILE, Alo = Apre + 2 * GT_TILE;
            const uint32_t Bph = sbase + G_OFF_B, Bqh = Bph + GT_TILE, Bpl = Bph + 2 * GT_TILE,
                           Bql = Bph + 3 * GT_TILE;
            auto load_pre = [&](long tile) {
                const int pair = pair_of(tile);
                const int t0 = (int)((tile % A.tiles_per_pair) * 128);
                const int s = pair / a.kv_heads, h = pair % a.kv_heads;
                if (lane == 0) {
                    tc::mbar_arrive_expect_tx(pre_full, GT_TILE);
                    for (int hh = 0; hh < 2; ++hh)
                        tc::tma_load_3d(sm + G_OFF_A + hh * GT_SUB, &tk, pre_full, hh * 64, h, s * (int)a.T + t0);
                }
                __syncwarp();
            };
            if (t_begin < t_end) load_pre(t_begin);
            for (long tile = t_begin; tile < t_end; ++tile) {
                const int it = (int)(tile - t_begin);
                const int pair = pair_of(tile);
                const int blk = a.layer * a.kv_heads + pair % a.kv_heads;
                if (blk != cur_blk) {  // (re)load W1's split tiles once the previous MMAs are done with B
                    if (it > 0) tc::mbar_wait(hl_empty, (it - 1) & 1);
                    if (lane == 0) {
                        tc::mbar_arrive_expect_tx(b_full, 4 * GT_TILE);
                        for (int q = 0; q < 4; ++q)
                            for (int hh = 0; hh < 2; ++hh)
                                tc::tma_load_3d(sm + G_OFF_B + q * GT_TILE + hh * GT_SUB, &tw, b_full, hh * 64, 0,
                                                blk * 4 + q);
                    }
                    __syncwarp();
                    tc::mbar_wait(b_full, b_loads & 1);
                    ++b_loads;
                    cur_blk = blk;
                }
                const int buf = it & 1;
                const uint32_t dt = tmem + (uint32_t)buf * 128u;
                tc::mbar_wait(pre_full, it & 1);
                if (it >= 2) tc::mbar_wait(&t_empty[buf], ((it - 2) >> 1) & 1);
                tc::fence_after_sync();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) tc::mma_ss_w(dt, kdesc(Apre, kk), kdesc(Bph, kk), idG, kk ? 1u : 0u);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) tc::mma_ss_w(dt, kdesc(Apre, kk), kdesc(Bpl, kk), idG, 1u);
                tc::mma_commit_w(pre_empty);
                if (tile + 1 < t_end) {  // next k_pre tile once S1-S2 and the producers are done with this one
                    tc::mbar_wait(pre_read, it & 1);
                    tc::mbar_wait(pre_empty, it & 1);
                    load_pre(tile + 1);
                }
                tc::mbar_wait(hl_full, it & 1);
                tc::fence_after_sync();
                // k_post = the hi tile: one TMA store per 64-dim half (full lines, rows
                // past the sequence's T clipped by the 4-D map) instead of every
                // producer's strided 16-byte stores
                if (lane == 0) {
                    const int s = pair / a.kv_heads, h = pair % a.kv_heads;
                    const int t0 = (int)((tile % A.tiles_per_pair) * 128);
                    for (int hh = 0; hh < 2; ++hh)
                        tc::tma_store_4d(&tpost, sm + G_OFF_A + GT_TILE + hh * GT_SUB, hh * 64, h, t0, s);
                    tc::bulk_commit_group();
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) tc::mma_ss_w(dt, kdesc(Ahi, kk), kdesc(Bqh, kk), idG, 1u);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) tc::mma_ss_w(dt, kdesc(Ahi, kk), kdesc(Bql, kk), idG, 1u);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) tc::mma_ss_w(dt, kdesc(Alo, kk), kdesc(Bqh, kk), idG, 1u);
                tc::mma_commit_w(hl_empty);
                tc::mma_commit_w(&t_full[buf]);
                if (lane == 0) {  // the hi tile may be rewritten once the store has read it
                    tc::bulk_wait_group_read0();
                    tc::mbar_arrive(st_read);
                }
                __syncwarp();
            }
            if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // k_post written
        }
        __syncwarp();
    } else {
        // ======================= epilogue ====================================
        // two groups of 4 warps: group g drains the tiles with it % 2 == g (TMEM
        // buffer g), each warp over all 128 hidden units of its 32 rows
        const int grp = (warp - 9) >> 2;
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int row = quarter * 32 + lane;
        // Worst-case relative error of each z1_h w.r.t. sum_k |W1_hk x_k|: split
        // residuals 2 * 2^-17 + dropped lo.lo 2^-18 + 40 fp32 accumulator adds
        // (<= 40 * 2^-23) ~= 2.4e-5; 3e-5 used.
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
            // z2 - b2 = sum_h w2_h gelu(z1_h) with the fast erf (packed f32x2);
            // az = sum_h |w2_h z1_h| bounds both the erf error and the roundings
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
                    const float2 w2 = make_float2(c.z, c.w);
                    part = __ffma2_rn(w2, ge, part);
                    az = __ffma2_rn(make_float2(fabsf(c.z), fabsf(c.w)), make_float2(fabsf(z1.x), fabsf(z1.y)), az);
                }
            }
            tc::fence_before_sync();
            tc::mbar_arrive(&t_empty[grp]);
            const long t = t0 + row;
            const float xx = __bfloat162float(xxs[(it % XX_SLOTS) * 128 + row]);
            if (t < a.T) {
                const float z2 = (float)a.b2f[blk] + (part.x + part.y);
                const float azs = az.x + az.y;
                const size_t gi = ((size_t)s * a.kv_heads + h) * a.T + t;
                g_out[gi] = 1.f / (1.f + __expf(-z2));
                bits_out[gi] = z2 >= a.ztau ? 1 : 0;
                // |gelu_fast - gelu| <= |z| ERF_EPS / 2 per unit; fp32 roundings of
                // the epilogue <= (hidden + 6) u (sum |w2 gelu| + |b2| + |ztau|) with
                // sum |w2 gelu| <= az; x4 margin on all terms.
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
        tc::tmem_dealloc(tmem, 256);
    }
}

// cos/sin of every (position, pair) of one call: the values rope_cs gives
__global__ void rope_table_kernel(const double* __restrict__ freq, long pos0, long T, int hp,
                                  float2* __restrict__ out) {
    const size_t n = (size_t)T * hp;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        float c, s;
        rope_cs(freq, (int)(e % hp), pos0 + (long)(e / hp), c, s);
        out[e] = make_float2(c, s);
    }
}

void launch_rope_table(const double* freq, long pos0, long T, int hp, float2* out, cudaStream_t st) {
    rope_table_kernel<<<num_sms() * 8, 256, 0, st>>>(freq, pos0, T, hp, out);
}

int launch_gate_tc(const GateArgs& a, int nseq, const __nv_bfloat16* k_pre, __nv_bfloat16* k_post, float* g,
                   uint8_t* bits, int32_t* cand, int* pcnt, const __nv_bfloat16* w1split, long n_wtiles,
                   float2* rope_ws, cudaStream_t st) {
    if (a.d != 128 || a.hidden != 128) return WGKV_ENOTSUP;
    CUtensorMap tw, tk;  // [L*H*4][128 hidden][128 k] split W1 tiles; k_pre [nseq*T][kv_heads][128]
    if (make_tmap_3d_bf16(&tw, w1split, 128, 128, (uint64_t)n_wtiles, 256, 128 * 256, 64, 128, 1)) return WGKV_ECUDA;
    if (make_tmap_3d_bf16(&tk, k_pre, 128, (uint64_t)a.kv_heads, (uint64_t)nseq * a.T, 256, (uint64_t)a.kv_heads * 256,
                          64, 1, 128))
        return WGKV_ECUDA;
    CUtensorMap tpost;  // k_post [nseq][T][kv_heads][128] as {128, kv_heads, T, nseq}
    {
        const uint64_t dims[4] = {128, (uint64_t)a.kv_heads, (uint64_t)a.T, (uint64_t)nseq};
        const uint64_t strides[3] = {256, (uint64_t)a.kv_heads * 256, (uint64_t)a.T * a.kv_heads * 256};
        const uint32_t box[4] = {64, 1, 128, 1};
        if (make_tmap_4d_bf16(&tpost, k_post, dims, strides, box)) return WGKV_ECUDA;
    }
    if (ensure_smem(gate_tc_kernel, G_SMEM) != cudaSuccess) return WGKV_ECUDA;
    rope_table_kernel<<<num_sms() * 8, 256, 0, st>>>(a.freq, a.pos0, a.T, a.d / 2, rope_ws);
    GateTcArgs A;
    A.g = a;
    A.nseq = nseq;
    A.tiles_per_pair = (a.T + 127) / 128;
    A.total_tiles = A.tiles_per_pair * nseq * a.kv_heads;
    A.rope = rope_ws;
    const int R = num_sms() / a.kv_heads;  // token-tile ranges per head
    A.head_sched = R >= 1 && (long)nseq * A.tiles_per_pair >= R;
    const int grid = A.head_sched ? R * a.kv_heads : (int)std::min<long>(num_sms(), A.total_tiles);
    gate_tc_kernel<<<grid, G_THREADS, G_SMEM, st>>>(tw, tk, tpost, A, k_pre, k_post, g, bits, cand, pcnt);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

}  // namespace wgkv
