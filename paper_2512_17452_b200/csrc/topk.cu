// topk.cu -- K6: select_topk_pages (engine.cpp:36-84) + attention over the
// selected Global pages and the Local ring, per q head (wgkv_plus_topk,
// engine.cpp:320-324; BASELINE configs[4]).
//
//   quest_meta/score       WGKV_TOPK_QUEST: Quest's upper bound from per-page
//                          key min / max (approximate; not the reference's)
//   topk_score_mma_kernel  page score = max over the page's slots of the
//                          UNSCALED q.k (q RoPE'd at the decode position) for
//                          every q head of the GQA group, on the tensor pipe
//                          (bf16; each K byte read once per group).
//                          topk_score_kernel is the SIMT form (fp32 parity mode).
//   topk_thresh_kernel     exact top-min(budget, pages) per q head: radix select
//                          on 64-bit keys (orderable(score) << 32 | ~page), i.e.
//                          higher score first and ties to the OLDER page, exactly
//                          std::stable_sort + the reference comparator.
//   topk_mask/compact      bf16: the group's selections merged in ascending
//                          logical order with a per-page q-head mask; K5
//                          (decode_attn_mma_kernel<true>) streams them once per
//                          group plus the Local ring, masking unselected rows.
//   topk_emit_kernel +     fp32 parity mode: per-q-head ascending selection
//   topk_attn_kernel       and SIMT split-KV attention over it.
#include <algorithm>
#include <cstdlib>

#include "attn.cuh"

namespace wgkv {

namespace {
constexpr int TK_PPB = 32;  // pages per score CTA (4 warps x 8)
__device__ __forceinline__ uint32_t orderable(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {  // lo -> bits 0-15
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
}  // namespace

template <typename E>
__global__ void __launch_bounds__(128) topk_score_kernel(DecArgs a, const E* __restrict__ q,
                                                          float* __restrict__ scores) {
    extern __shared__ float tsm[];
    const int d = a.pv.head_dim, ps = a.pv.page_size;
    const int gs = a.q_heads / a.pv.kv_heads;
    const int bh = blockIdx.y, s = bh / a.pv.kv_heads, h = bh % a.pv.kv_heads;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long hidx = a.pv.head_index(a.layer, a.seq0 + s, h);
    const HeadState st = a.pv.state[hidx];
    const int ng = (st.global_len + ps - 1) / ps;
    const int p0 = blockIdx.x * TK_PPB;
    if (p0 >= ng) return;
    const long pos = st.tokens_seen - 1;
    float* Qs = tsm;  // [gs][d], RoPE'd, unscaled (select_topk_pages uses dot(q, k))
    for (int e = threadIdx.x; e < gs * (d / 2); e += blockDim.x) {
        const int g = e / (d / 2), i = e % (d / 2);
        const size_t off = ((size_t)s * a.q_heads + h * gs + g) * d + 2 * i;
        const float x0 = to_f(q[off]), x1 = to_f(q[off + 1]);
        float c, sn;
        rope_cs(a.freq, i, pos, c, sn);
        Qs[g * d + 2 * i] = x0 * c - x1 * sn;
        Qs[g * d + 2 * i + 1] = x0 * sn + x1 * c;
    }
    __syncthreads();
    const E* pool = reinterpret_cast<const E*>(a.pv.data);
    const int half = lane >> 4, slot = lane & 15;  // lanes 0-15 / 16-31 share the slots, split the heads
    for (int lp = p0 + warp; lp < min(ng, p0 + TK_PPB); lp += 4) {
        const int page = a.pv.gpt[hidx * a.pv.n_gp + lp];
        const int valid = min(ps, st.global_len - lp * ps);
        for (int g0 = 0; g0 < gs; g0 += 2) {
            const int g = g0 + half;
            float sc = -INFINITY;
            if (g < gs && slot < valid && page >= 0) {
                const E* kr = pool + (size_t)page * a.pv.page_elems() + (size_t)slot * d;
                float acc = 0.f;
                for (int c = 0; c < d; ++c) acc = fmaf(Qs[g * d + c], to_f(kr[c]), acc);
                sc = acc;
            }
            for (int o = 8; o >= 1; o >>= 1) sc = fmaxf(sc, __shfl_xor_sync(0xffffffffu, sc, o));
            if (slot == 0 && g < gs) scores[((size_t)s * a.q_heads + h * gs + g) * a.pv.n_gp + lp] = sc;
        }
    }
}

// ---------------------------------------------------------------------------
// bf16 scoring on the tensor pipe.  One warp scores one 16-slot page for the
// whole GQA group with 8 mma.sync m16n8k16: A = the page's K rows (slots are
// the M rows), B = the group's RoPE'd q split into bf16 hi + lo halves (columns
// 0-3 hi, 4-7 lo of up to 4 heads), so score = C[hi] + C[lo] carries ~17
// mantissa bits of q (K is exact in bf16) with fp32 accumulation.  K rows are
// loaded straight from HBM as 16-byte vectors into the A-fragment registers:
// the dot product is invariant under a permutation of d applied to both
// operands, so lane (row r, quad t) takes dims [32b + 8t, 32b + 8t + 8) of
// rows r and r + 8 and the B fragment uses the same dim order.  Each warp
// keeps 2 pages (16 x 16-byte loads per lane) in flight.
// ---------------------------------------------------------------------------
constexpr int SC_WARPS = 8;
#ifndef WGKV_SC_PAGES
#define WGKV_SC_PAGES 64
#endif
constexpr int SC_PAGES = WGKV_SC_PAGES;  // pages per CTA (8 per warp)

__global__ void __launch_bounds__(SC_WARPS * 32) topk_score_mma_kernel(DecArgs a, const __nv_bfloat16* __restrict__ q,
                                                                        float* __restrict__ scores) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the previous kernel
    constexpr int d = 128, ps = 16;
    const int gs = a.q_heads / a.pv.kv_heads;
    const int bh = blockIdx.y, s = bh / a.pv.kv_heads, h = bh % a.pv.kv_heads;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long hidx = a.pv.head_index(a.layer, a.seq0 + s, h);
    const HeadState st = a.pv.state[hidx];
    const int ng = (st.global_len + ps - 1) / ps;
    const int p0 = blockIdx.x * SC_PAGES;
    if (p0 >= ng) return;
    __shared__ float Qs[4][d];
    __shared__ int pid[SC_PAGES];
    const long pos = st.tokens_seen - 1;
    for (int e = tid; e < 4 * (d / 2); e += blockDim.x) {
        const int g = e / (d / 2), i = e % (d / 2);
        float y0 = 0.f, y1 = 0.f;
        if (g < gs) {
            const size_t off = ((size_t)s * a.q_heads + h * gs + g) * d + 2 * i;
            const float x0 = __bfloat162float(q[off]), x1 = __bfloat162float(q[off + 1]);
            float c, sn;
            rope_cs(a.freq, i, pos, c, sn);
            y0 = x0 * c - x1 * sn;
            y1 = x0 * sn + x1 * c;
        }
        Qs[g][2 * i] = y0;
        Qs[g][2 * i + 1] = y1;
    }
    if (tid < SC_PAGES) {
        const int lp = p0 + tid;
        pid[tid] = lp < ng ? a.pv.gpt[hidx * a.pv.n_gp + lp] : -1;
    }
    __syncthreads();
    const int q4 = lane & 3, gr = lane >> 2;
    uint32_t bq[4][2][2];
    {
        const int head = gr & 3;
        const bool lo = gr >= 4;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int k2 = 0; k2 < 2; ++k2) {
                float x[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float v = Qs[head][32 * b + 8 * q4 + 4 * k2 + j];
                    const float hi = __bfloat162float(__float2bfloat16_rn(v));
                    x[j] = lo ? v - hi : hi;
                }
                bq[b][k2][0] = pack2(x[0], x[1]);
                bq[b][k2][1] = pack2(x[2], x[3]);
            }
    }
    const __nv_bfloat16* pool = reinterpret_cast<const __nv_bfloat16*>(a.pv.data);
    constexpr int PPW = SC_PAGES / SC_WARPS;
#pragma unroll 1
    for (int i = 0; i < PPW; i += 2) {
        uint4 ra[2][4], rb[2][4];
        int valid[2], lpu[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int li = warp * PPW + i + u, lp = p0 + li, page = pid[li];
            lpu[u] = lp;
            valid[u] = (lp < ng && page >= 0) ? min(ps, st.global_len - lp * ps) : 0;
            const uint4* kr = reinterpret_cast<const uint4*>(pool + (size_t)max(page, 0) * a.pv.page_elems());
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                if (valid[u] > 0) {
                    ra[u][b] = __ldg(kr + gr * 16 + b * 4 + q4);
                    rb[u][b] = __ldg(kr + (gr + 8) * 16 + b * 4 + q4);
                } else {
                    ra[u][b] = rb[u][b] = make_uint4(0u, 0u, 0u, 0u);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (valid[u] == 0) continue;  // warp-uniform
            float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                mma16816(c, ra[u][b].x, rb[u][b].x, ra[u][b].y, rb[u][b].y, bq[b][0][0], bq[b][0][1]);
                mma16816(c, ra[u][b].z, rb[u][b].z, ra[u][b].w, rb[u][b].w, bq[b][1][0], bq[b][1][1]);
            }
            // columns 2t, 2t+1: t = 0/1 hold hi of heads (0,1)/(2,3), t = 2/3 the lo halves
#pragma unroll
            for (int e = 0; e < 4; ++e) c[e] += __shfl_xor_sync(0xffffffffu, c[e], 2);
            if (gr >= valid[u]) c[0] = c[1] = -INFINITY;
            if (gr + 8 >= valid[u]) c[2] = c[3] = -INFINITY;
            float m0 = fmaxf(c[0], c[2]), m1 = fmaxf(c[1], c[3]);
#pragma unroll
            for (int o = 4; o <= 16; o <<= 1) {
                m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
                m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
            }
            if (lane < 2) {
                const int g0 = 2 * lane;
                float* dst = scores + ((size_t)s * a.q_heads + h * gs + g0) * a.pv.n_gp + lpu[u];
                if (g0 < gs) dst[0] = m0;
                if (g0 + 1 < gs) dst[a.pv.n_gp] = m1;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Quest bound (wgkv_config.topk_mode = WGKV_TOPK_QUEST; not the reference's
// selection): score(page) = sum_d max(q_d min_d, q_d max_d) >= max_slot q.k,
// from per-page elementwise key min / max (bf16: exact for the bf16 keys),
// 512 B per page instead of the page's 4 KB of K.  The metadata is kept
// current incrementally: quest_meta_kernel recomputes Global pages
// [meta_full, ng) of each head (after a prefill all of them, then the tail page
// and pages filled since), quest_score_kernel advances meta_full to the count
// of full pages (a later launch, so the meta kernel's blocks all read the old
// value).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) quest_meta_kernel(DecArgs a, const int* __restrict__ meta_full,
                                                         __nv_bfloat16* __restrict__ meta) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the previous kernel
    constexpr int d = 128;
    const int bh = blockIdx.y, s = bh / a.pv.kv_heads, h = bh % a.pv.kv_heads;
    const long hidx = a.pv.head_index(a.layer, a.seq0 + s, h);
    const HeadState st = a.pv.state[hidx];
    const int ps = a.pv.page_size;
    const int ng = (st.global_len + ps - 1) / ps;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const __nv_bfloat16* pool = reinterpret_cast<const __nv_bfloat16*>(a.pv.data);
    for (int lp = meta_full[hidx] + blockIdx.x * 8 + warp; lp < ng; lp += gridDim.x * 8) {
        const int page = a.pv.gpt[hidx * a.pv.n_gp + lp];
        if (page < 0) continue;
        const int valid = min(ps, st.global_len - lp * ps);
        const __nv_bfloat16* kr = pool + (size_t)page * a.pv.page_elems() + 4 * lane;
        float mn[4] = {INFINITY, INFINITY, INFINITY, INFINITY}, mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        for (int r = 0; r < valid; ++r) {
            const uint2 raw = __ldg(reinterpret_cast<const uint2*>(kr + (size_t)r * d));
            const float x[4] = {__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xffff0000u),
                                __uint_as_float(raw.y << 16), __uint_as_float(raw.y & 0xffff0000u)};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                mn[e] = fminf(mn[e], x[e]);
                mx[e] = fmaxf(mx[e], x[e]);
            }
        }
        __nv_bfloat16* mo = meta + (size_t)page * 2 * d + 4 * lane;  // [min 128 | max 128], exact in bf16
        *reinterpret_cast<uint2*>(mo) = make_uint2(pack2(mn[0], mn[1]), pack2(mn[2], mn[3]));
        *reinterpret_cast<uint2*>(mo + d) = make_uint2(pack2(mx[0], mx[1]), pack2(mx[2], mx[3]));
    }
}

template <int QG>  // GQA group size
__global__ void __launch_bounds__(256) quest_score_kernel(DecArgs a, const __nv_bfloat16* __restrict__ q,
                                                          const __nv_bfloat16* __restrict__ meta,
                                                          int* __restrict__ meta_full, float* __restrict__ scores) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the previous kernel
    constexpr int d = 128, PPW = 2;  // pages per warp (all loads issued up front)
    const int bh = blockIdx.y, s = bh / a.pv.kv_heads, h = bh % a.pv.kv_heads;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long hidx = a.pv.head_index(a.layer, a.seq0 + s, h);
    const HeadState st = a.pv.state[hidx];
    const int ps = a.pv.page_size;
    const int ng = (st.global_len + ps - 1) / ps;
    if (blockIdx.x == 0 && tid == 0) meta_full[hidx] = st.global_len / ps;
    const int p0 = blockIdx.x * 8 * PPW;
    if (p0 >= ng) return;
    __shared__ float Qs[QG][d];
    __shared__ int pid[8 * PPW];
    if (tid < 8 * PPW) pid[tid] = p0 + tid < ng ? a.pv.gpt[hidx * a.pv.n_gp + p0 + tid] : -1;
    const long pos = st.tokens_seen - 1;
    for (int e = tid; e < QG * (d / 2); e += blockDim.x) {
        const int g = e / (d / 2), i = e % (d / 2);
        const size_t off = ((size_t)s * a.q_heads + h * QG + g) * d + 2 * i;
        const float x0 = __bfloat162float(q[off]), x1 = __bfloat162float(q[off + 1]);
        float c, sn;
        rope_cs(a.freq, i, pos, c, sn);
        Qs[g][2 * i] = x0 * c - x1 * sn;
        Qs[g][2 * i + 1] = x0 * sn + x1 * c;
    }
    __syncthreads();
    uint2 mn_raw[PPW], mx_raw[PPW];
#pragma unroll
    for (int u = 0; u < PPW; ++u) {
        const int page = pid[warp * PPW + u];
        const __nv_bfloat16* mp = meta + (size_t)max(page, 0) * 2 * d + 4 * lane;
        mn_raw[u] = __ldg(reinterpret_cast<const uint2*>(mp));
        mx_raw[u] = __ldg(reinterpret_cast<const uint2*>(mp + d));
    }
#pragma unroll
    for (int u = 0; u < PPW; ++u) {
        const int lp = p0 + warp * PPW + u;
        if (lp >= ng) break;  // warp-uniform
        const float mn[4] = {__uint_as_float(mn_raw[u].x << 16), __uint_as_float(mn_raw[u].x & 0xffff0000u),
                             __uint_as_float(mn_raw[u].y << 16), __uint_as_float(mn_raw[u].y & 0xffff0000u)};
        const float mx[4] = {__uint_as_float(mx_raw[u].x << 16), __uint_as_float(mx_raw[u].x & 0xffff0000u),
                             __uint_as_float(mx_raw[u].y << 16), __uint_as_float(mx_raw[u].y & 0xffff0000u)};
        float sc[QG];
#pragma unroll
        for (int g = 0; g < QG; ++g) {
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float qq = Qs[g][4 * lane + e];
                acc += fmaxf(qq * mn[e], qq * mx[e]);
            }
            sc[g] = acc;
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
            for (int g = 0; g < QG; ++g) sc[g] += __shfl_xor_sync(0xffffffffu, sc[g], o);
        if (lane < QG) {
            float v = sc[0];
#pragma unroll
            for (int g = 1; g < QG; ++g) v = lane == g ? sc[g] : v;
            scores[((size_t)s * a.q_heads + h * QG + lane) * a.pv.n_gp + lp] =
                pid[warp * PPW + u] >= 0 ? v : -INFINITY;
        }
    }
}

// ---------------------------------------------------------------------------
// exact top-k threshold per (seq, q head) over the 64-bit keys
// (orderable(score) << 32 | ~page): a page is selected iff key >= thr[sp]
// (higher score first, ties to the OLDER page); thr = 0 selects every page.
//   pass A   one sweep over the scores (staged into smem on the way) builds a
//            4096-bin histogram of the key's top 12 bits (sign, exponent, 3
//            mantissa bits) and a block scan
//            finds the bin holding the k-th largest key;
//   compact  the keys of that bin (a few % of the pages) are gathered into a
//            smem candidate list;
//   refine   8-bit radix passes over the candidates for the remaining 52 bits,
//            stopping as soon as the chosen bin holds exactly the keys still
//            needed.  (A bin too large for the list -- massive score ties --
//            refines over all pages instead.)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long page_key(float score, int lp) {
    return ((unsigned long long)orderable(score) << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)lp);
}

constexpr int TH_BINS = 4096;
constexpr int TH_CAND = 4096;
constexpr int TH_STAGE_CAP = 44 * 1024;  // staged scores (dynamic smem floats)

__global__ void __launch_bounds__(1024) topk_thresh_kernel(DecArgs a, long budget, int smem_cap,
                                                           const float* __restrict__ scores,
                                                           unsigned long long* __restrict__ thr) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the previous kernel
    extern __shared__ unsigned long long cand[];   // [TH_CAND] candidate keys, then the staged scores
    float* ssc = reinterpret_cast<float*>(cand + TH_CAND);
    __shared__ unsigned hist[TH_BINS];
    __shared__ unsigned wtot[32];
    __shared__ unsigned long long prefix_s;
    __shared__ int remain_s, cnt_s, done_s, ncand_s;
    const int sp = blockIdx.x, s = sp / a.q_heads, p = sp % a.q_heads;
    const int h = p / (a.q_heads / a.pv.kv_heads), ps = a.pv.page_size;
    const HeadState st = a.pv.state[a.pv.head_index(a.layer, a.seq0 + s, h)];
    const int n = (st.global_len + ps - 1) / ps;
    const int k = (int)min((long)n, budget);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (k >= n) {
        if (tid == 0) thr[sp] = 0ull;
        return;
    }
    const float* sc = scores + (size_t)sp * a.pv.n_gp;
    const bool staged = n <= smem_cap;
    static_assert(TH_BINS == 4 * 1024, "pass A scan assumes 4 bins per thread");
    // ---- pass A: top-12-bit histogram (+ staging) ----------------------------
    for (int i = tid; i < TH_BINS; i += blockDim.x) hist[i] = 0;
    if (tid == 0) ncand_s = 0;
    if (staged) {  // independent loads, 8 in flight per thread
        for (int base = 0; base < n; base += 8 * 1024) {
            float x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int lp = base + j * 1024 + tid;
                x[j] = lp < n ? sc[lp] : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int lp = base + j * 1024 + tid;
                if (lp < n) ssc[lp] = x[j];
            }
        }
    }
    __syncthreads();
    // plain shared atomics: the 4096 bins spread a warp's keys (match.any
    // costs more than the occasional same-address conflict)
    if (staged) {
        for (int lp = tid; lp < n; lp += blockDim.x) atomicAdd(&hist[orderable(ssc[lp]) >> 20], 1u);
    } else {
        for (int lp = tid; lp < n; lp += blockDim.x) atomicAdd(&hist[orderable(__ldg(sc + lp)) >> 20], 1u);
    }
    __syncthreads();
    {  // block suffix scan: thread t owns bins 4095-4t .. 4092-4t (thread 0 the top)
        unsigned c4[4], tot = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            c4[j] = hist[TH_BINS - 1 - 4 * tid - j];
            tot += c4[j];
        }
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wtot[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            unsigned w = wtot[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            wtot[lane] = w - wtot[lane];  // exclusive warp offsets
        }
        __syncthreads();
        incl += wtot[warp];
        const unsigned excl = incl - tot;
        if (excl < (unsigned)k && (unsigned)k <= incl) {
            unsigned acc = excl;
            int j = 0;
            for (; j < 3; ++j) {
                if (acc + c4[j] >= (unsigned)k) break;
                acc += c4[j];
            }
            const unsigned b = TH_BINS - 1 - 4 * tid - j;
            prefix_s = (unsigned long long)b << 52;
            remain_s = k - (int)acc;
            cnt_s = (int)c4[j];
        }
    }
    __syncthreads();
    unsigned long long prefix = prefix_s, mask = 0xFFFull << 52;
    int remain = remain_s;
    if (cnt_s == remain) {  // the whole bin is taken
        if (tid == 0) thr[sp] = prefix;
        return;
    }
    // ---- compact the chosen bin's keys --------------------------------------
    const bool use_cand = cnt_s <= TH_CAND;
    if (use_cand) {
        for (int base = 0; base < n; base += blockDim.x) {
            const int lp = base + tid;
            unsigned long long key = 0;
            bool hit = false;
            if (lp < n) {
                key = page_key(staged ? ssc[lp] : __ldg(sc + lp), lp);
                hit = (key & mask) == prefix;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            int wbase = 0;
            if (lane == 0 && bal) wbase = atomicAdd(&ncand_s, __popc(bal));
            wbase = __shfl_sync(0xffffffffu, wbase, 0);
            if (hit) cand[wbase + __popc(bal & ((1u << lane) - 1u))] = key;
        }
        __syncthreads();
    }
    const int nitems = use_cand ? cnt_s : n;
    // ---- refine: 8-bit digits below the 12 leading bits ---------------------
    for (int shift = 44; shift >= -4; shift -= 8) {
        const int sh = max(shift, 0), width = shift >= 0 ? 8 : 4;
        const unsigned dmask = (1u << width) - 1u;
        if (tid < 256) hist[tid] = 0;
        __syncthreads();
        for (int i = tid; i < nitems; i += blockDim.x) {
            const unsigned long long key =
                use_cand ? cand[i] : page_key(staged ? ssc[i] : __ldg(sc + i), i);
            if ((key & mask) == prefix) atomicAdd(&hist[(unsigned)(key >> sh) & dmask], 1u);
        }
        __syncthreads();
        if (warp == 0) {  // suffix scan of 256 bins: lane l owns bins 255-8l .. 248-8l
            unsigned cnt[8], tot = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                cnt[j] = hist[255 - 8 * lane - j];
                tot += cnt[j];
            }
            unsigned incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const unsigned excl = incl - tot;
            if (excl < (unsigned)remain && (unsigned)remain <= incl) {
                unsigned acc = excl, cj = cnt[0];
                int j = 0;
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {  // static indexing keeps cnt[] in registers
                    if (jj == j) {
                        if (acc + cnt[jj] >= (unsigned)remain || jj == 7) {
                            cj = cnt[jj];
                        } else {
                            acc += cnt[jj];
                            ++j;
                        }
                    }
                }
                const int b = 255 - 8 * lane - j;
                prefix_s = prefix | ((unsigned long long)b << sh);
                remain_s = remain - (int)acc;
                done_s = cj == (unsigned)(remain - (int)acc);
            }
        }
        __syncthreads();
        prefix = prefix_s;
        remain = remain_s;
        mask |= (unsigned long long)dmask << sh;
        if (done_s || shift <= 0) break;  // uniform
    }
    if (tid == 0) thr[sp] = prefix;
}

// fp32 parity path: emit one q head's selection in ascending logical order
__global__ void __launch_bounds__(1024) topk_emit_kernel(DecArgs a, const float* __restrict__ scores,
                                                         const unsigned long long* __restrict__ thr,
                                                         int32_t* __restrict__ sel, int32_t* __restrict__ nsel) {
    const int sp = blockIdx.x, s = sp / a.q_heads, p = sp % a.q_heads;
    const int h = p / (a.q_heads / a.pv.kv_heads), ps = a.pv.page_size;
    const HeadState st = a.pv.state[a.pv.head_index(a.layer, a.seq0 + s, h)];
    const int n = (st.global_len + ps - 1) / ps;
    const float* sc = scores + (size_t)sp * a.pv.n_gp;
    const unsigned long long t = thr[sp];
    int32_t* out = sel + (size_t)sp * a.pv.n_gp;
    __shared__ int wsum[32];
    __shared__ int carry;
    const int tid = threadIdx.x;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += blockDim.x) {
        const int lp = base + tid;
        const bool take = lp < n && page_key(sc[lp], lp) >= t;
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if ((tid & 31) == 0) wsum[tid >> 5] = __popc(bal);
        __syncthreads();
        int before = carry;
        for (int w = 0; w < (tid >> 5); ++w) before += wsum[w];
        if (take) out[before + __popc(bal & ((1u << (tid & 31)) - 1u))] = lp;
        __syncthreads();
        if (tid == 0) {
            int tt = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tt += wsum[w];
            carry += tt;
        }
        __syncthreads();
    }
    if (tid == 0) nsel[sp] = carry;
}

// bf16 path: union of the GQA group's selections per (seq, kv head), ascending,
// each entry = logical page | (bitmask of the group's q heads that chose it) << 24
// -- K5 streams every union page once and masks the rows that did not choose it.
// Two fully parallel passes over blocks of UB pages: masks + per-block counts,
// then each block compacts its pages after the counts of the blocks before it.
constexpr int UB = 1024;  // pages per block (256 threads x 4)

__global__ void __launch_bounds__(256) topk_mask_kernel(DecArgs a, const float* __restrict__ scores,
                                                        const unsigned long long* __restrict__ thr,
                                                        uint8_t* __restrict__ umask, int* __restrict__ ucnt,
                                                        int nblk) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the previous kernel
    const int bh = blockIdx.y, s = bh / a.pv.kv_heads, h = bh % a.pv.kv_heads, blk = blockIdx.x;
    const int gs = a.q_heads / a.pv.kv_heads, ps = a.pv.page_size;
    const HeadState st = a.pv.state[a.pv.head_index(a.layer, a.seq0 + s, h)];
    const int n = (st.global_len + ps - 1) / ps;
    const int tid = threadIdx.x;
    __shared__ int wc[8];
    if (blk * UB >= n) {
        if (tid == 0) ucnt[(size_t)bh * nblk + blk] = 0;
        return;
    }
    const float* sc = scores + ((size_t)s * a.q_heads + h * gs) * a.pv.n_gp;
    const int lp0 = blk * UB + tid * 4;
    uint32_t m[4] = {0u, 0u, 0u, 0u};
    for (int g = 0; g < gs; ++g) {
        const unsigned long long t = thr[(size_t)s * a.q_heads + h * gs + g];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (lp0 + j < n && page_key(sc[(size_t)g * a.pv.n_gp + lp0 + j], lp0 + j) >= t) m[j] |= 1u << g;
    }
    int c = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (lp0 + j < n) {
            umask[(size_t)bh * a.pv.n_gp + lp0 + j] = (uint8_t)m[j];
            c += m[j] != 0u;
        }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((tid & 31) == 0) wc[tid >> 5] = c;
    __syncthreads();
    if (tid == 0) {
        int t = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += wc[w];
        ucnt[(size_t)bh * nblk + blk] = t;
    }
}

__global__ void __launch_bounds__(256) topk_compact_kernel(DecArgs a, const uint8_t* __restrict__ umask,
                                                           const int* __restrict__ ucnt, int nblk,
                                                           int32_t* __restrict__ uni, int32_t* __restrict__ nuni,
                                                           int* __restrict__ k5_counter) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the previous kernel
    // K5 (next, a programmatic dependent) steals work from this counter
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && k5_counter) *k5_counter = 0;
    const int bh = blockIdx.y, s = bh / a.pv.kv_heads, h = bh % a.pv.kv_heads, blk = blockIdx.x;
    const int ps = a.pv.page_size;
    const HeadState st = a.pv.state[a.pv.head_index(a.layer, a.seq0 + s, h)];
    const int n = (st.global_len + ps - 1) / ps;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (n == 0) {
        if (blk == 0 && tid == 0) nuni[bh] = 0;
        return;
    }
    if (blk * UB >= n) return;
    __shared__ int wsum[8], wpre[8], s_base;
    // entries of the blocks before this one
    int pre = 0;
    for (int b = tid; b < blk; b += blockDim.x) pre += ucnt[(size_t)bh * nblk + b];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    if (lane == 0) wpre[warp] = pre;
    const int lp0 = blk * UB + tid * 4;
    uint32_t m[4];
    int c = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        m[j] = lp0 + j < n ? umask[(size_t)bh * a.pv.n_gp + lp0 + j] : 0u;
        c += m[j] != 0u;
    }
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (tid == 0) {
        int b = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) b += wpre[w];
        s_base = b;
    }
    __syncthreads();
    int pos = s_base + incl - c;
    for (int w = 0; w < warp; ++w) pos += wsum[w];
    int32_t* out = uni + (size_t)bh * a.pv.n_gp;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (m[j]) out[pos++] = (int32_t)((uint32_t)(lp0 + j) | (m[j] << 24));
    if (blk == (n - 1) / UB && tid == blockDim.x - 1) {
        int t = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += wsum[w];
        nuni[bh] = s_base + t;
    }
}

// split-KV attention of one q head over selected Global pages + Local pages
template <typename E>
__global__ void __launch_bounds__(128) topk_attn_kernel(DecArgs a, const E* __restrict__ q,
                                                         const int32_t* __restrict__ sel,
                                                         const int32_t* __restrict__ nsel, float* __restrict__ part) {
    extern __shared__ float asmem[];
    const int d = a.pv.head_dim, ps = a.pv.page_size;
    const int sp = blockIdx.y, s = sp / a.q_heads, p = sp % a.q_heads;
    const int h = p / (a.q_heads / a.pv.kv_heads);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long hidx = a.pv.head_index(a.layer, a.seq0 + s, h);
    const HeadState st = a.pv.state[hidx];
    const int nsg = nsel[sp];
    const int nl = (st.local_len + ps - 1) / ps;
    const int NP = nsg + nl;
    const int vp0 = blockIdx.x * a.chunk_pages, vp1 = min(NP, vp0 + a.chunk_pages);
    float* pout = part + ((size_t)sp * a.max_chunks + blockIdx.x) * (d + 2);
    if (vp0 >= vp1) {
        if (tid == 0) {
            pout[d] = -INFINITY;
            pout[d + 1] = 0.f;
        }
        return;
    }
    float* Qs = asmem;          // [d] RoPE'd
    float* red = Qs + d;        // [4][d + 2]
    const long pos = st.tokens_seen - 1;
    const float scale = rsqrtf((float)d);
    for (int i = tid; i < d / 2; i += blockDim.x) {
        const size_t off = ((size_t)s * a.q_heads + p) * d + 2 * i;
        const float x0 = to_f(q[off]), x1 = to_f(q[off + 1]);
        float c, sn;
        rope_cs(a.freq, i, pos, c, sn);
        Qs[2 * i] = x0 * c - x1 * sn;
        Qs[2 * i + 1] = x0 * sn + x1 * c;
    }
    __syncthreads();
    const E* pool = reinterpret_cast<const E*>(a.pv.data);
    const int nc = (d + 31) / 32;  // column blocks of 32 (the last one partial when d % 32 != 0)
    float m = -INFINITY, l = 0.f, o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int vp = vp0 + warp; vp < vp1; vp += 4) {
        int page, valid;
        if (vp < nsg) {
            const int lp = sel[(size_t)sp * a.pv.n_gp + vp];
            page = a.pv.gpt[hidx * a.pv.n_gp + lp];
            valid = min(ps, st.global_len - lp * ps);
        } else {
            page = a.pv.lpt[hidx * a.pv.n_lp + (vp - nsg)];
            valid = min(ps, st.local_len - (vp - nsg) * ps);
        }
        if (page < 0) continue;
        const E* kb = pool + (size_t)page * a.pv.page_elems();
        const E* vb = kb + (size_t)ps * d;
        for (int j0 = 0; j0 < valid; j0 += 32) {
            const int j = j0 + lane;
            float sc = -INFINITY;
            if (j < valid) {
                float acc = 0.f;
                for (int c = 0; c < d; ++c) acc = fmaf(Qs[c], to_f(kb[(size_t)j * d + c]), acc);
                sc = acc * scale;
            }
            float mx = sc;
            for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            const float mn = fmaxf(m, mx);
            const float alpha = (m == -INFINITY) ? 0.f : __expf(m - mn);
            const float pj = j < valid ? __expf(sc - mn) : 0.f;
            float sum = pj;
            for (int off = 16; off >= 1; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
            l = l * alpha + sum;
            m = mn;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c < nc) o[c] *= alpha;
            const int jn = min(32, valid - j0);
            for (int jj = 0; jj < jn; ++jj) {
                const float pjj = __shfl_sync(0xffffffffu, pj, jj);
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c < nc && lane + 32 * c < d) o[c] = fmaf(pjj, to_f(vb[(size_t)(j0 + jj) * d + lane + 32 * c]), o[c]);
            }
        }
    }
    float* rw = red + (size_t)warp * (d + 2);
#pragma unroll
    for (int c = 0; c < 8; ++c)
        if (c < nc && lane + 32 * c < d) rw[lane + 32 * c] = o[c];
    if (lane == 0) {
        rw[d] = m;
        rw[d + 1] = l;
    }
    __syncthreads();
    for (int c = tid; c < d; c += blockDim.x) {
        float M = -INFINITY;
        for (int w = 0; w < 4; ++w) M = fmaxf(M, red[(size_t)w * (d + 2) + d]);
        float acc = 0.f, L = 0.f;
        for (int w = 0; w < 4; ++w) {
            const float* r = red + (size_t)w * (d + 2);
            const float f = r[d] == -INFINITY ? 0.f : __expf(r[d] - M);
            acc += f * r[c];
            L += f * r[d + 1];
        }
        pout[c] = acc;
        if (c == 0) {
            pout[d] = M;
            pout[d + 1] = L;
        }
    }
}

template <typename E>
__global__ void topk_combine_kernel(DecArgs a, const float* __restrict__ part, E* __restrict__ out) {
    // per (seq, q head): merge chunk partials (decode_combine with group size 1)
    const int d = a.pv.head_dim, sp = blockIdx.x;
    const float* base = part + (size_t)sp * a.max_chunks * (d + 2);
    __shared__ float M, invL;
    if (threadIdx.x == 0) {
        float mx = -INFINITY;
        for (int c = 0; c < a.n_chunks; ++c) mx = fmaxf(mx, base[(size_t)c * (d + 2) + d]);
        float L = 0.f;
        for (int c = 0; c < a.n_chunks; ++c) {
            const float mc = base[(size_t)c * (d + 2) + d];
            if (mc != -INFINITY) L += __expf(mc - mx) * base[(size_t)c * (d + 2) + d + 1];
        }
        M = mx;
        invL = 1.f / L;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < d; e += blockDim.x) {
        float acc = 0.f;
        for (int c = 0; c < a.n_chunks; ++c) {
            const float mc = base[(size_t)c * (d + 2) + d];
            if (mc != -INFINITY) acc += __expf(mc - M) * base[(size_t)c * (d + 2) + e];
        }
        out[(size_t)sp * d + e] = from_f<E>(acc * invL);
    }
}

// launch as a programmatic dependent of the previous kernel in the stream (its
// launch overlaps the predecessor's tail; the kernel's griddepcontrol.wait
// orders every read after the predecessor completes)
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    static const bool off = getenv("WGKV_TOPK_NOPDL") != nullptr;  // A/B switch
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = off ? 0 : 1;
    cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...);
}

template <typename E>
int launch_topk_decode(const DecArgs& a0, int nseq, long budget, const E* q, float* scores, int32_t* sel,
                       int32_t* nsel, unsigned long long* thr, uint8_t* umask, int* ucnt, float* part, int* nchunks,
                       E* out, int mode, __nv_bfloat16* meta, int* meta_full, cudaStream_t st) {
    DecArgs a = a0;
    const int d = a.pv.head_dim, gs = a.q_heads / a.pv.kv_heads;
    if (d % 2 != 0 || d > 256) return WGKV_ENOTSUP;
    const int max_pages = a.pv.n_gp;
    // bf16 production path: tensor-pipe scoring + union selection streamed by K5
    constexpr bool kBf16 = sizeof(E) == 2;
    const bool fast = kBf16 && d == 128 && a.pv.page_size == 16 && gs <= 8 && a.pv.capacity < (1L << 24);
    if (mode == WGKV_TOPK_QUEST) {
        if (!fast || !meta || !meta_full) return WGKV_ENOTSUP;
        launch_pdl(quest_meta_kernel, dim3(16, nseq * a.pv.kv_heads), 256, 0, st, a, meta_full, meta);
        const dim3 qgrid((max_pages + 15) / 16, nseq * a.pv.kv_heads);
        const __nv_bfloat16* qb = reinterpret_cast<const __nv_bfloat16*>(q);
        switch (gs) {
            case 1: launch_pdl(quest_score_kernel<1>, qgrid, 256, 0, st, a, qb, meta, meta_full, scores); break;
            case 2: launch_pdl(quest_score_kernel<2>, qgrid, 256, 0, st, a, qb, meta, meta_full, scores); break;
            case 4: launch_pdl(quest_score_kernel<4>, qgrid, 256, 0, st, a, qb, meta, meta_full, scores); break;
            case 8: launch_pdl(quest_score_kernel<8>, qgrid, 256, 0, st, a, qb, meta, meta_full, scores); break;
            default: return WGKV_ENOTSUP;
        }
    } else if (fast && gs <= 4)
        launch_pdl(topk_score_mma_kernel, dim3((max_pages + SC_PAGES - 1) / SC_PAGES, nseq * a.pv.kv_heads),
                   SC_WARPS * 32, 0, st, a, reinterpret_cast<const __nv_bfloat16*>(q), scores);
    else
        topk_score_kernel<E><<<dim3((max_pages + TK_PPB - 1) / TK_PPB, nseq * a.pv.kv_heads), 128,
                              sizeof(float) * gs * d, st>>>(a, q, scores);
    const int cap = std::min(max_pages, TH_STAGE_CAP);
    const size_t th_smem = (size_t)TH_CAND * 8 + (size_t)cap * 4;
    if (ensure_smem(topk_thresh_kernel, th_smem) != cudaSuccess) return WGKV_ECUDA;
    launch_pdl(topk_thresh_kernel, nseq * a.q_heads, 1024, th_smem, st, a, budget, cap, (const float*)scores, thr);
    if (fast) {
        const int nblk = (max_pages + UB - 1) / UB;
        static const bool nopdl = getenv("WGKV_TOPK_NOPDL") != nullptr;  // A/B switch
        int* k5_counter = nchunks + (size_t)a.pv.max_seqs * a.pv.kv_heads;  // K5's work-stealing counter
        launch_pdl(topk_mask_kernel, dim3(nblk, nseq * a.pv.kv_heads), 256, 0, st, a, (const float*)scores,
                   (const unsigned long long*)thr, umask, ucnt, nblk);
        launch_pdl(topk_compact_kernel, dim3(nblk, nseq * a.pv.kv_heads), 256, 0, st, a, (const uint8_t*)umask,
                   (const int*)ucnt, nblk, sel, nsel, nopdl ? nullptr : k5_counter);
        a.sel = sel;
        a.nsel = nsel;
        if constexpr (kBf16)
            return launch_decode_attn_mma(a, nseq, q, part, nchunks, out, st, !nopdl);
        return WGKV_ENOTSUP;
    }
    topk_emit_kernel<<<nseq * a.q_heads, 1024, 0, st>>>(a, scores, thr, sel, nsel);
    // at most budget Global pages + the Local ring per q head
    const long np = budget + a.pv.n_lp;
    long cp = std::max(4L, (np + a.max_chunks - 1) / a.max_chunks);
    a.chunk_pages = (int)cp;
    a.n_chunks = (int)((np + cp - 1) / cp);
    topk_attn_kernel<E><<<dim3(a.n_chunks, nseq * a.q_heads), 128, sizeof(float) * (d + 4 * (d + 2)), st>>>(
        a, q, sel, nsel, part);
    topk_combine_kernel<E><<<nseq * a.q_heads, 128, 0, st>>>(a, part, out);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

template int launch_topk_decode<float>(const DecArgs&, int, long, const float*, float*, int32_t*, int32_t*,
                                       unsigned long long*, uint8_t*, int*, float*, int*, float*, int,
                                       __nv_bfloat16*, int*, cudaStream_t);
template int launch_topk_decode<__nv_bfloat16>(const DecArgs&, int, long, const __nv_bfloat16*, float*, int32_t*,
                                               int32_t*, unsigned long long*, uint8_t*, int*, float*, int*,
                                               __nv_bfloat16*, int, __nv_bfloat16*, int*, cudaStream_t);

}  // namespace wgkv
