// EXPERIMENT (not built into the product; parity-green but slower, profiles/r2_k3_notes.md).
// Build as an A/B variant: copy into paper_2512_17452_b200/csrc/ and route wgkv_vs_prefill to
// launch_vs_prefill_tc4.
// attn_tc4.cu -- K3 v4: vertical-slash prefill attention over 64-key blocks
// with the S tile of each query head double-buffered in TMEM.
//
// Same contract and key set as attn_tc.cu (build_vs_mask + attn_vertical_slash,
// attention.cpp:116-153).  attn_tc.cu's 128-key blocks
// fill TMEM with O_t and ONE S_t per head (P aliases S), so each head's chain
// softmax(j) -> PV(j) -> S(j+1) -> softmax(j+1) is serial.  Halving the key
// block to 64 halves S, and TMEM holds
//   O_0 [0,128) | O_1 [128,256) | S_0,0 S_0,1 S_1,0 S_1,1 (64 columns each) [256,512)
// so S(t, j+1) is computed while head t's softmax works on S(t, j); P(t, j)
// aliases S(t, j%2) and S(t, j+2) is issued after PV(t, j) (in-order pipe).
// Two query heads of a GQA group per CTA still share every K/V tile.  Cost:
// the S MMAs have N = 64 (Q re-read per 64 keys), the softmax's per-block
// fixed work (TMEM load, max exchange, barriers) comes twice per 128 keys.
// Warp roles as attn_tc.cu (19 warps): 16 softmax (head t, column half c of
// the 64 keys, lane quarter wq), K and V TMA producers (4-deep rings of 16 KB
// tiles), MMA issuer.
#include <cuda.h>

#include <cstdio>

#include "attn_tc.cuh"
#include "tc.cuh"

namespace wgkv {

namespace {

constexpr int NT = 2;
constexpr int BN = 64;     // keys per block
constexpr int NSK = 4;     // K / V ring depth
constexpr uint32_t QTILE = 128 * 128 * 2;  // [128 rows][128 d]
constexpr uint32_t QSUB = QTILE / 2;       // [128][64] SW128 sub-tile
constexpr uint32_t KVTILE = BN * 128 * 2;  // [64 keys][128 d]
constexpr uint32_t KVSUB = KVTILE / 2;     // [64][64] SW128 sub-tile
constexpr uint32_t OFF_Q = 0;
constexpr uint32_t OFF_K = NT * QTILE;
constexpr uint32_t OFF_V = OFF_K + NSK * KVTILE;
constexpr uint32_t OFF_BAR = OFF_V + NSK * KVTILE;
constexpr uint32_t OFF_X = OFF_BAR + 512;  // [2 parities][NT][2 halves][128] f32 row-max exchange
constexpr uint32_t SMEM_BYTES = OFF_X + 2 * NT * 2 * 128 * 4 + 1024;
constexpr int NSPLIT = 2, HC = BN / NSPLIT;  // 32 columns of S per softmax thread
constexpr int NSOFT = NT * NSPLIT * 4;
constexpr int WARP_TMA = NSOFT, WARP_MMA = NSOFT + 2;
constexpr int NTHREADS = (NSOFT + 3) * 32;
constexpr float LOG2E = 1.4426950408889634f;
constexpr uint32_t COL_S = 256;

struct Bars {
    uint64_t q_full, q_ready;
    uint64_t k_full[NSK], k_empty[NSK], v_full[NSK], v_empty[NSK];
    uint64_t s_full[NT][2], p_full[NT][2], pv_done[NT], o_final[NT];
    uint32_t tmem;
    int C;
};

#ifndef WGKV_K3D_EMU_MASK
#define WGKV_K3D_EMU_MASK 0x8888  // exp2 pairs on the FMA pipe (pair e of the thread's 16)
#endif
#ifndef WGKV_K3D_SLEEP
#define WGKV_K3D_SLEEP 2  // suspend-hint waits: bit 0 producers, 1 MMA issuer, 2 softmax
#endif
#define K3D_WAIT(role, bar_, par_) \
    ((WGKV_K3D_SLEEP >> (role)) & 1 ? tc::mbar_wait_sleep((bar_), (par_)) : tc::mbar_wait((bar_), (par_)))

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x for a pair on the FMA/ALU pipes (attn_tc.cu ex2_emu2)
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
// K-major SW128 operand, K step kk (16 bf16 = 32 bytes); sub-tile (64 of K) of `sub` bytes
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t tile_saddr, int kk, uint32_t sub) {
    return tc::smem_desc_sw128(tile_saddr + (uint32_t)(kk >> 2) * sub + (uint32_t)(kk & 3) * 32u, 16, 1024);
}

}  // namespace

#ifdef WGKV_TRACE  // diagnostic build only: per-block event clocks of CTA (0,0,0)
__device__ unsigned long long g_k3_trace4[4][4096][8];
#define K3_TR(who, j, ev)                                                                                      \
    do {                                                                                                       \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 4096) g_k3_trace4[who][j][ev] = clock64(); \
    } while (0)
extern "C" int wgkv_dbg_k3_trace4(void* host, size_t bytes) {
    return cudaMemcpyFromSymbol(host, g_k3_trace4, bytes) == cudaSuccess ? 0 : -1;
}
#else
#define K3_TR(who, j, ev) \
    do {                  \
    } while (0)
#endif

__global__ void __launch_bounds__(NTHREADS, 1)
    vs_prefill_tc4_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                          const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tpool,
                          const __grid_constant__ CUtensorMap tkrun, const __grid_constant__ CUtensorMap tvrun,
                          VsArgs a, __nv_bfloat16* __restrict__ out) {
    extern __shared__ uint8_t smem_raw[];
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

    const long s_lo = i0 - W + 1 > 0 ? i0 - W + 1 : 0;
    int cnt = 0;
    {
        const long c = s_lo / 128, rem = s_lo - c * 128;
        cnt = __syncthreads_count(threadIdx.x < rem && bits[c * 128 + threadIdx.x] != 0);
    }
    if (threadIdx.x == 0) {
        int C = s_lo > 0 ? co[s_lo / 128] + cnt : 0;
        C = min(C, a.pv.state[hidx].global_len);
        bar->C = C;
        tc::mbar_init(&bar->q_full, 1);
        tc::mbar_init(&bar->q_ready, NSOFT * 32);
        for (int i = 0; i < NSK; ++i) {
            tc::mbar_init(&bar->k_full[i], 1);
            tc::mbar_init(&bar->k_empty[i], 1);
            tc::mbar_init(&bar->v_full[i], 1);
            tc::mbar_init(&bar->v_empty[i], 1);
        }
        for (int t = 0; t < NT; ++t) {
            for (int b = 0; b < 2; ++b) {
                tc::mbar_init(&bar->s_full[t][b], 1);
                tc::mbar_init(&bar->p_full[t][b], NSPLIT * 128);
            }
            tc::mbar_init(&bar->pv_done[t], 1);
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
    const int nv = (C + BN - 1) / BN;
    const int nb = (int)((band_hi - s_lo + 1 + BN - 1) / BN);
    const int nblk = nv + nb;
    const int ps = a.pv.page_size;

    if (warp == WARP_TMA || warp == WARP_TMA + 1) {
        // ============================ TMA producers ===========================
        const int kv = warp - WARP_TMA;
        if (lane == 0 && kv == 0) {
            tc::tma_prefetch(&tq);
            tc::tma_prefetch(&tk);
            tc::tma_prefetch(&tv);
            tc::tma_prefetch(&tpool);
            tc::tma_prefetch(&tkrun);
            tc::tma_prefetch(&tvrun);
            tc::mbar_arrive_expect_tx(&bar->q_full, NT * QTILE);
            for (int t = 0; t < NT; ++t)
                for (int hh = 0; hh < 2; ++hh)
                    tc::tma_load_3d(sm + OFF_Q + t * QTILE + hh * QSUB, &tq, &bar->q_full, hh * 64, p0 + t,
                                    (int)(s * T + i0));
        }
        const int ppb = BN / ps;  // pages per 64-key block (<= 8)
        const int last_page = C > 0 ? (C - 1) / ps : 0;
        const int32_t* gpt = a.pv.gpt + hidx * a.pv.n_gp;
        auto page_ids = [&](int jb) -> int {
            return (jb < nv && lane < ppb) ? gpt[min(jb * ppb + lane, last_page)] : 0;
        };
        int next_ids = page_ids(0);
        for (int j = 0; j < nblk; ++j) {
            const int st = j % NSK;
            const int cur_ids = next_ids;
            if (j + 1 < nblk) next_ids = page_ids(j + 1);
            const bool band = j >= nv;
            const long kb0 = band ? s_lo + (long)BN * (j - nv) : 0;
            const int pg = __shfl_sync(0xffffffffu, cur_ids, lane >> 1);
            uint64_t* full = kv ? &bar->v_full[st] : &bar->k_full[st];
            if (j >= NSK) K3D_WAIT(0, kv ? &bar->v_empty[st] : &bar->k_empty[st], ((j - NSK) / NSK) & 1);
            uint8_t* dst = sm + (kv ? OFF_V : OFF_K) + st * KVTILE;
            if (lane == 0) tc::mbar_arrive_expect_tx(full, KVTILE);
            __syncwarp();
            if (!band) {
                const int pg0 = __shfl_sync(0xffffffffu, cur_ids, 0);
                if (__all_sync(0xffffffffu, lane >= ppb || cur_ids == pg0 + lane)) {
                    if (lane < 2) tc::tma_load_3d(dst + lane * KVSUB, kv ? &tvrun : &tkrun, full, lane * 64, 0, pg0);
                } else if (lane < 2 * ppb) {
                    tc::tma_load_3d(dst + (lane & 1) * KVSUB + (lane >> 1) * ps * 128, &tpool, full, (lane & 1) * 64, 0,
                                    2 * pg + kv);
                }
            } else if (lane < 2) {
                tc::tma_load_3d(dst + lane * KVSUB, kv ? &tv : &tk, full, lane * 64, h, (int)(s * T + kb0));
            }
        }
    } else if (warp == WARP_MMA) {
        // ================================ MMA issuer =============================
        constexpr uint32_t idS = tc::idesc_bf16(128, BN, false, false);
        constexpr uint32_t idPV = tc::idesc_bf16(128, 128, false, true);
        auto issue_S = [&](int t, int j) {  // S(t, j) = Q_t K(j)^T into buffer j % 2
            const uint32_t qa = sbase + OFF_Q + t * QTILE;
            const uint32_t ka = sbase + OFF_K + (j % NSK) * KVTILE;
            const uint32_t d = tmem + COL_S + 64 * (2 * t + (j & 1));
            tc::mma8_ss_k128_w<QSUB / 16, KVSUB / 16>(d, kmajor_desc(qa, 0, QSUB), kmajor_desc(ka, 0, KVSUB), idS);
            tc::mma_commit_w(&bar->s_full[t][j & 1]);
        };
        auto issue_PV = [&](int t, int j) {  // O_t += P(t, j) V(j): P in TMEM over S(t, j % 2)
            const uint32_t va = sbase + OFF_V + (j % NSK) * KVTILE;
            const uint32_t pa = tmem + COL_S + 64 * (2 * t + (j & 1));
            tc::mma4_ts_vmn_w(tmem + 128 * t, pa, tc::smem_desc_sw128(va, KVSUB, 1024), idPV, j > 0 ? 1u : 0u);
            tc::mma_commit_w(&bar->pv_done[t]);
            if (j == nblk - 1) tc::mma_commit_w(&bar->o_final[t]);
        };
        K3D_WAIT(1, &bar->q_ready, 0);
        tc::fence_after_sync();
        for (int jj = 0; jj < 2 && jj < nblk; ++jj) {
            K3D_WAIT(1, &bar->k_full[jj % NSK], (jj / NSK) & 1);
            tc::fence_after_sync();
            for (int t = 0; t < NT; ++t) issue_S(t, jj);
            tc::mma_commit_w(&bar->k_empty[jj % NSK]);
        }
        for (int j = 0; j < nblk; ++j) {
            for (int t = 0; t < NT; ++t) {
                K3D_WAIT(1, &bar->p_full[t][j & 1], (j >> 1) & 1);
                if (lane == 0) K3_TR(2, j, t);
                if (t == 0) K3D_WAIT(1, &bar->v_full[j % NSK], (j / NSK) & 1);
                tc::fence_after_sync();
                issue_PV(t, j);
                if (t == NT - 1) tc::mma_commit_w(&bar->v_empty[j % NSK]);
                if (j + 2 < nblk) {
                    if (t == 0) {
                        K3D_WAIT(1, &bar->k_full[(j + 2) % NSK], ((j + 2) / NSK) & 1);
                        tc::fence_after_sync();
                    }
                    issue_S(t, j + 2);  // into S(t, j % 2), after PV(t, j) read P(t, j)
                    if (t == NT - 1) tc::mma_commit_w(&bar->k_empty[(j + 2) % NSK]);
                }
            }
        }
        __syncwarp();
    } else {
        // ================================ softmax ================================
        const int t = warp >> 3, c = (warp >> 2) & 1, wq = warp & 3;
        const int r = wq * 32 + lane;
        const long i = i0 + r;
        const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
        const uint32_t colO = 128 * t + 64 * c;
        const uint32_t barid = 1 + t * 4 + wq;
        float* xm = reinterpret_cast<float*>(sm + OFF_X);  // [parity][t][half][128]
        auto pair_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(barid), "r"(NSPLIT * 32) : "memory"); };
        // RoPE(q) in place (engine.cpp:229), pre-scaled by log2(e)/sqrt(d); half c rotates sub-tile c
        tc::mbar_wait(&bar->q_full, 0);
        {
            const float qs = rsqrtf(128.f) * LOG2E;
            uint8_t* qt = sm + OFF_Q + t * QTILE + c * QSUB;
            for (int cc = 0; cc < 8; ++cc) {
                uint4* p = reinterpret_cast<uint4*>(qt + tc::sw128_off(r, cc));
                uint4 v = *p;
                uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float x0 = __uint_as_float(w[u] << 16), x1 = __uint_as_float(w[u] & 0xffff0000u);
                    float cs, sn;
                    rope_cs_fast(a.freq, c * 32 + cc * 4 + u, i, cs, sn);
                    w[u] = tc::pack_bf16x2((x0 * cs - x1 * sn) * qs, (x0 * sn + x1 * cs) * qs);
                }
                *p = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&bar->q_ready);

        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nblk; ++j) {
            const int b = j & 1;
            const uint32_t colS = COL_S + 64 * (2 * t + b);
            K3D_WAIT(2, &bar->s_full[t][b], (j >> 1) & 1);
            tc::fence_after_sync();
            if (lane == 0 && c == 0 && wq == 0) K3_TR(t, j, 0);
            uint32_t s0[32];
            tc::tmem_ld32(trow + colS + HC * c, s0);
            tc::tmem_ld_wait();
            const uint32_t NEG_INF = 0xff800000u;
            if (j < nv) {
                const int vc = min(BN, C - BN * j);
                if (vc < BN) {
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (HC * c + e >= vc) s0[e] = NEG_INF;
                }
            } else {
                const long kb0 = s_lo + (long)BN * (j - nv);
                if (!(kb0 + BN - 1 <= i0 && i0 + 127 - kb0 < W)) {
                    const long kc = kb0 + HC * c + lane;
                    const uint32_t mk = __ballot_sync(0xffffffffu, kc < T && bits[kc] != 0);
                    const long dd = i - kb0;
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const long col = HC * c + e;
                        const bool ok = col <= dd && ((dd - col) < W || ((mk >> e) & 1u));
                        if (!ok) s0[e] = NEG_INF;
                    }
                }
            }
            float pm[8] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int e = 0; e < 32; ++e) pm[e & 7] = fmaxf(pm[e & 7], __uint_as_float(s0[e]));
            float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                             fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
            float* xb = xm + (b * NT + t) * 256;  // parity buffers: the other half may still read block j-1's
            xb[c * 128 + r] = mx;
            pair_sync();
            mx = fmaxf(mx, xb[(c ^ 1) * 128 + r]);
            if (lane == 0 && c == 0 && wq == 0) K3_TR(t, j, 1);
            const bool rescale = __any_sync(0xffffffffu, mx > m + 8.f);
            float alpha = 1.f;
            if (rescale) {
                const float mn = fmaxf(m, mx);
                alpha = (m == -INFINITY) ? 0.f : ex2(m - mn);
                l *= alpha;
                m = mn;
            }
            const float mu = (m == -INFINITY) ? 0.f : m;
            float2 lsv[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
            const float2 nmu = make_float2(-mu, -mu);
            uint32_t pa[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const float2 xd = __fadd2_rn(make_float2(__uint_as_float(s0[2 * e]), __uint_as_float(s0[2 * e + 1])), nmu);
                float e0, e1;
                if ((WGKV_K3D_EMU_MASK >> e) & 1) {
                    const float2 ee = ex2_emu2(xd.x, xd.y);
                    e0 = ee.x;
                    e1 = ee.y;
                } else {
                    e0 = ex2(xd.x);
                    e1 = ex2(xd.y);
                }
                lsv[e & 3] = __fadd2_rn(lsv[e & 3], make_float2(e0, e1));
                pa[e] = tc::pack_bf16x2(e0, e1);
            }
            {
                const float2 a01 = __fadd2_rn(lsv[0], lsv[1]), a23 = __fadd2_rn(lsv[2], lsv[3]);
                const float2 tt = __fadd2_rn(a01, a23);
                l += tt.x + tt.y;
            }
            if (lane == 0 && c == 0 && wq == 0) K3_TR(t, j, 2);
            // P (bf16x2) of keys [32c, 32c+32) -> packed columns [16c, 16c+16) of S(t, b)
            tc::tmem_st16(trow + colS + (HC / 2) * c, pa);
            // O_t holds PV(0..j-1) only once PV(t, j-1) completed: S(t, j) was issued
            // after PV(t, j-2), so s_full does not imply it -- wait before rescaling
            if (rescale && j > 0) {
                K3D_WAIT(2, &bar->pv_done[t], (j - 1) & 1);
                tc::fence_after_sync();
#pragma unroll 1
                for (int k = 0; k < 2; ++k) {
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
            tc::mbar_arrive(&bar->p_full[t][b]);
            if (lane == 0 && c == 0 && wq == 0) K3_TR(t, j, 3);
        }
        // ---- epilogue: O / l -> bf16 (row sum = both halves) -------------------
        tc::mbar_wait(&bar->o_final[t], 0);
        tc::fence_after_sync();
        float* xl = xm + ((nblk & 1) * NT + t) * 256;  // the parity buffer the last block did not use
        xl[c * 128 + r] = l;
        pair_sync();
        const float lt = l + xl[(c ^ 1) * 128 + r];
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        __nv_bfloat16* orow = out + (((size_t)s * T + i) * Hq + p0 + t) * 128 + 64 * c;
#pragma unroll 1
        for (int k = 0; k < 2; ++k) {
            uint32_t o[32];
            tc::tmem_ld32(trow + colO + 32 * k, o);
            tc::tmem_ld_wait();
            if (i < T) {
                uint4* dst = reinterpret_cast<uint4*>(orow + 32 * k);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                    dst[q4] = make_uint4(
                        tc::pack_bf16x2(__uint_as_float(o[8 * q4]) * inv, __uint_as_float(o[8 * q4 + 1]) * inv),
                        tc::pack_bf16x2(__uint_as_float(o[8 * q4 + 2]) * inv, __uint_as_float(o[8 * q4 + 3]) * inv),
                        tc::pack_bf16x2(__uint_as_float(o[8 * q4 + 4]) * inv, __uint_as_float(o[8 * q4 + 5]) * inv),
                        tc::pack_bf16x2(__uint_as_float(o[8 * q4 + 6]) * inv, __uint_as_float(o[8 * q4 + 7]) * inv));
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

int launch_vs_prefill_tc4(const VsArgs& a, int nseq, const __nv_bfloat16* q, const __nv_bfloat16* k_post,
                          const __nv_bfloat16* v, __nv_bfloat16* out, cudaStream_t st) {
    const int d = a.pv.head_dim, ps = a.pv.page_size;
    const int Hq = a.q_heads, Hkv = a.pv.kv_heads;
    if (d != 128 || BN % ps != 0 || ps < 8 || (Hq / Hkv) % NT != 0) return WGKV_ENOTSUP;
    CUtensorMap tq, tk, tv, tp;
    const uint64_t rows = (uint64_t)nseq * a.T;
    int r = make_tmap_3d_bf16(&tq, q, 128, Hq, rows, 256, (uint64_t)Hq * 256, 64, 1, 128);
    r |= make_tmap_3d_bf16(&tk, k_post, 128, Hkv, rows, 256, (uint64_t)Hkv * 256, 64, 1, BN);
    r |= make_tmap_3d_bf16(&tv, v, 128, Hkv, rows, 256, (uint64_t)Hkv * 256, 64, 1, BN);
    r |= make_tmap_3d_bf16(&tp, a.pv.data, 128, ps, 2 * (uint64_t)a.pv.capacity, 256, (uint64_t)ps * 256, 64, ps, 1);
    CUtensorMap tkr, tvr;
    const uint64_t plane = (uint64_t)ps * 256;
    r |= make_tmap_3d_bf16(&tkr, a.pv.data, 128, ps, (uint64_t)a.pv.capacity, 256, 2 * plane, 64, ps, BN / ps);
    r |= make_tmap_3d_bf16(&tvr, static_cast<const uint8_t*>(a.pv.data) + plane, 128, ps, (uint64_t)a.pv.capacity,
                           256, 2 * plane, 64, ps, BN / ps);
    if (r) return WGKV_ECUDA;
    if (ensure_smem(vs_prefill_tc4_kernel, SMEM_BYTES) != cudaSuccess) return WGKV_ECUDA;
    dim3 grid((unsigned)((a.T + 127) / 128), Hq / NT, nseq);
    vs_prefill_tc4_kernel<<<grid, NTHREADS, SMEM_BYTES, st>>>(tq, tk, tv, tp, tkr, tvr, a, out);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

}  // namespace wgkv
