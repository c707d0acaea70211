// decode_mma.cu -- K5: memory-bound split-KV decode attention over the paged
// Global + Local cache, read in place (no gather copy).
//
// Replaces HeadCache::gather + attn_ragged (kvstore.cpp:205-241,
// attention.cpp:155-180) for Session::decode_step (engine.cpp:309-326).
// Grid = (page chunks, seq x kv head).  Each CTA serves the whole GQA group
// (every K/V byte is read from HBM once per group), 6 warps stream pages
// independently through a 2-deep per-warp TMA ring (one 16-token page = K 4 KB
// + V 4 KB, ONE 4-D TMA box per page through a transposed view of the pool,
// SWIZZLE_128B so ldmatrix is conflict-free), and compute with
// mma.sync m16n8k16 (bf16 -> fp32): S = Q K^T with the group's q heads as
// rows, P V with P re-used from the S accumulators in registers.  The CTA
// merges its warps; decode_combine_kernel (attn_simt.cu) merges chunks.
#include <cuda.h>

#include <cstring>

#include "attn.cuh"
#include "tc.cuh"
#include "timeline.cuh"
#include "fused.cuh"

namespace wgkv {

namespace {

// 6 warps x 2-deep rings (12 pages in flight per CTA, as 4 x 3) measured +1.1 % decode tok/s at 128K x 4 and
// +2.3 % on the serving mix over 4 x 3 (graph-captured bench, same box)
#ifndef WGKV_K5_DW
#define WGKV_K5_DW 6
#endif
#ifndef WGKV_K5_DNS
#define WGKV_K5_DNS 2
#endif
#ifndef WGKV_K5_CPS
#define WGKV_K5_CPS 2
#endif
constexpr int DW = WGKV_K5_DW;    // warps per CTA
constexpr int DNS = WGKV_K5_DNS;  // ring stages per warp
constexpr int CPS = WGKV_K5_CPS;  // CTAs per SM
constexpr int PAGE_B = 8192; // bf16 page of 16 tokens: K 4 KB | V 4 KB
constexpr int QROW = 136;    // padded Q row (bf16 elements)
constexpr int PID_CAP = kDecPidCap;  // pages per work item (staged page ids)
#ifndef WGKV_GATE_K5_MAX
#define WGKV_GATE_K5_MAX 64
#endif
constexpr int kGateInK5MaxCtas = WGKV_GATE_K5_MAX;  // gate CTAs carried by the K5 launch at most
#ifndef WGKV_K5_PARAM_WARM
#define WGKV_K5_PARAM_WARM 0
#endif
#ifndef WGKV_K5_EVICT_FIRST
#define WGKV_K5_EVICT_FIRST 0
#endif
#ifndef WGKV_FUSED_MAX_FRONT
#define WGKV_FUSED_MAX_FRONT 148
#endif
constexpr int kFusedMaxFront = WGKV_FUSED_MAX_FRONT;  // fused layer: route + gate CTAs at most
#ifndef WGKV_FUSED_MAX_PAIRS
#define WGKV_FUSED_MAX_PAIRS 8
#endif
constexpr int kFusedMaxPairs = WGKV_FUSED_MAX_PAIRS;  // fused layer: (seq, kv head) pairs at most
#ifndef WGKV_K5_IPC
#define WGKV_K5_IPC 0  // work items per CTA, 0 = by pair count: work stealing balance vs per-item fixed
                       // costs.  With the first item before the PDL wait, 2 beats 3 by 2.4 % at 128K x 4
                       // (32 pairs) and 1.8 % at 64K x 8 (64 pairs); 3 beats 2 by 1.5-3 % on the serving
                       // mix (512 pairs) (profiles/r2_decode_peer_ab.txt)
#endif
#ifndef WGKV_GATE_EARLY
#define WGKV_GATE_EARLY 1  // fused layer: the gate CTAs compute before the PDL wait (parity-split scratch)
#endif
#ifndef WGKV_K5_RULE
#define WGKV_K5_RULE 1
#endif
#ifndef WGKV_K5_CAPCH
#define WGKV_K5_CAPCH 24  // chunks per (seq, kv head) pair the few-long-pairs rule aims at
#endif
#ifndef WGKV_K5_ITEMS_DIV
#define WGKV_K5_ITEMS_DIV 2  // the few-long-pairs cap keeps >= grid / ITEMS_DIV items
#endif
#ifndef WGKV_K5_MIN_PAGES
#define WGKV_K5_MIN_PAGES 8
#endif

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    return x;
}
__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, off));
    return x;
}
// address of the 16-byte chunk (row, chunk 0..7) of a [rows][64] SW128 tile
__device__ __forceinline__ uint32_t swz(uint32_t base, uint32_t row, uint32_t chunk) {
    return base + row * 128u + ((chunk ^ (row & 7u)) << 4);
}

}  // namespace

// fused layer (fused.cuh): the last item of pair bh merges the pair's nc chunk
// partials (m in natural-log units, l, unnormalised O) with the new token --
// logit RoPE(q) . bf16(RoPE(k_new)) / sqrt(d) with q from Qs (hi rows 0..7 +
// lo rows 8..15, pre-scaled by log2(e)/sqrt(d)), weight on v_new -- into the
// output rows of the pair's gs q heads.  The pair's partials (contiguous) come
// in by one bulk copy into the idle ring.  The last warp forms the new key and
// value, then -- off the merge's path, since the commit needs only that every
// item of the pair is done -- arrives for the merge party and, when last,
// commits the append; warps 0..DW-2 merge.  This code runs once per pair and
// launch, i.e. with a cold instruction cache (ncu: stall_no_instruction leads
// the small-batch K5): it is kept short -- rolled loops, one instantiation.
__device__ __forceinline__ void fused_tail(const DecArgs& a, const FinishArgs& fin, int bh, int nc, long pos,
                                           const __nv_bfloat16* Qs, uint8_t* scratch, const float* __restrict__ part,
                                           uint64_t* tbar, uint32_t& tpar TL_PARAM) {
    constexpr int d = 128, NM = (DW - 1) * 32;  // merging threads
    constexpr int RING = DW * DNS * PAGE_B;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gs = a.q_heads / a.pv.kv_heads;
    const int s = bh / a.pv.kv_heads, h = bh % a.pv.kv_heads;
    const int pairg = a.seq0 * a.pv.kv_heads + bh;
    const size_t o = (size_t)bh;  // = s * kv_heads + h
    const int pstride = gs * (d + 2);
    const float* pb = part + (size_t)bh * a.max_chunks * pstride;
    float* kn = reinterpret_cast<float*>(scratch);  // [d] the new key as cached
    float* vn = kn + d;                              // [d] the new value
    float* acc = vn + d;                             // [gs][d] (several batches)
    float* wgt = acc + gs * d;                       // [nc][gs] chunk weights
    const int rows_off = ((2 * d + gs * d + nc * gs) * 4 + 127) & ~127;
    float* rows = reinterpret_cast<float*>(scratch + rows_off);  // [cb][pstride] a batch of partials
    const int cap = (RING - rows_off) / (pstride * 4);             // chunks per batch
    __shared__ float s_L[8], s_wn[8];
    // a batch of chunks -> rows: one bulk copy (the partial buffer has 16 B of
    // slack past its end for the rounding) by thread 0, which holds the item
    // counter's acquire
    auto load_batch = [&](int c0, int cb) {
        if (tid == 0) {
            const uint32_t bytes = ((uint32_t)(cb * pstride) * 4u + 15u) & ~15u;
            tc::fence_proxy_async_global();
            tc::fence_proxy_async_smem();  // the CTA's generic use of the ring (after a barrier) first
            tc::mbar_arrive_expect_tx(tbar, bytes);
            tc::bulk_load(rows, pb + (size_t)c0 * pstride, bytes, tbar);
        }
    };
    load_batch(0, min(nc, cap));
    if (warp == DW - 1) {
        const size_t io = o * d;
        const float v0 = __bfloat162float(fin.v_new[io + lane]), v1 = __bfloat162float(fin.v_new[io + lane + 32]),
                    v2 = __bfloat162float(fin.v_new[io + lane + 64]), v3 = __bfloat162float(fin.v_new[io + lane + 96]);
        const __nv_bfloat162 k0 = reinterpret_cast<const __nv_bfloat162*>(fin.k_new + io)[lane];
        const __nv_bfloat162 k1 = reinterpret_cast<const __nv_bfloat162*>(fin.k_new + io)[lane + 32];
        vn[lane] = v0;
        vn[lane + 32] = v1;
        vn[lane + 64] = v2;
        vn[lane + 96] = v3;
#pragma unroll 1
        for (int j = 0; j < 2; ++j) {  // the key as it is cached: fp64 angle, fp32 rotation, bf16
            const int i = lane + 32 * j;
            const float2 kx = __bfloat1622float2(j ? k1 : k0);
            float c, sn, y0, y1;
            rope_cs(a.freq, i, pos, c, sn);
            rope_pair_f32(kx.x, kx.y, c, sn, y0, y1);
            kn[2 * i] = __bfloat162float(__float2bfloat16_rn(y0));
            kn[2 * i + 1] = __bfloat162float(__float2bfloat16_rn(y1));
        }
    } else {
        tc::mbar_wait(tbar, tpar);
    }
    tpar ^= 1u;
    __syncthreads();
    TL_MARK(3);
    if (warp == DW - 1) {
        // ---- the merge's arrival for the K/V commit (every item is done) and, when last, the commit
        const bool last = __shfl_sync(0xffffffffu, lane == 0 ? (int)pair_arrive(&fin.fw.cnt_kv[pairg]) : 0, 0);
        if (last)
            fused_commit_kv<__nv_bfloat16>(a.pv, fin.ga, a.layer, a.seq0, s, h, fin.k_new, fin.v_new, fin.forced_g,
                                           fin.tr, fin.wk, fin.fw, kn, vn);
        return;
    }
    const bool single = nc <= cap;
    // per head (a warp each): the new token's logit, the max, chunk weights, the denominator
#pragma unroll 1
    for (int g = warp; g < gs; g += DW - 1) {
        float dot = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = 4 * lane + j;
            dot = fmaf(__bfloat162float(Qs[g * QROW + i]) + __bfloat162float(Qs[(g + 8) * QROW + i]), kn[i], dot);
        }
        const float mn = warp_sum(dot) * 0.6931471805599453f;  // log2 units -> natural
        float M = mn;
#pragma unroll 1
        for (int c = lane; c < nc; c += 32) {
            const float* r = (single ? rows : pb) + (size_t)c * pstride + (size_t)g * (d + 2) + d;
            const float m = single ? r[0] : __ldcg(r);
            wgt[c * gs + g] = m;
            M = fmaxf(M, m);
        }
        M = warp_max(M);
        float L = 0.f;
#pragma unroll 1
        for (int c = lane; c < nc; c += 32) {
            const float* r = (single ? rows : pb) + (size_t)c * pstride + (size_t)g * (d + 2) + d + 1;
            const float m = wgt[c * gs + g], w = m == -INFINITY ? 0.f : __expf(m - M);
            wgt[c * gs + g] = w;
            L = fmaf(w, single ? r[0] : __ldcg(r), L);
        }
        L = warp_sum(L);
        if (lane == 0) {
            s_wn[g] = __expf(mn - M);
            s_L[g] = L + s_wn[g];
        }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NM) : "memory");  // merging warps only
    TL_MARK(4);
#pragma unroll 1
    for (int c0 = 0; c0 < nc; c0 += cap) {
        const int cb = min(cap, nc - c0);
        if (c0 > 0) {  // the next batch (many chunks of a wide group)
            asm volatile("bar.sync 1, %0;" ::"n"(NM) : "memory");
            load_batch(c0, cb);
            tc::mbar_wait(tbar, tpar);
            tpar ^= 1u;
        }
#pragma unroll 1
        for (int e = tid; e < gs * (d / 2); e += NM) {  // (head, column pair)
            const int g = e / (d / 2), col = 2 * (e - g * (d / 2));
            const float2* r = reinterpret_cast<const float2*>(rows + (size_t)g * (d + 2) + col);
            const float* w = wgt + (size_t)c0 * gs + g;
            float2 t = c0 == 0 ? make_float2(s_wn[g] * vn[col], s_wn[g] * vn[col + 1])
                               : reinterpret_cast<const float2*>(acc)[e];
#pragma unroll 4
            for (int c = 0; c < cb; ++c) {
                const float wc = w[c * gs];
                const float2 x = r[(size_t)c * (pstride / 2)];
                t.x = fmaf(wc, x.x, t.x);
                t.y = fmaf(wc, x.y, t.y);
            }
            if (c0 + cb < nc) {
                reinterpret_cast<float2*>(acc)[e] = t;
            } else {
                const float il = 1.f / s_L[g];
                const __nv_bfloat162 ov = __floats2bfloat162_rn(t.x * il, t.y * il);
                *reinterpret_cast<__nv_bfloat162*>(fin.out + ((size_t)s * a.q_heads + h * gs + g) * d + col) = ov;
                if (fin.px.do_push)  // C1: the same 4 bytes into every rank's exchange slot (LL words)
                    peer_push_word(fin.px, peer_push_flag(fin.px), s, ((h * gs + g) * d + col) / 2,
                                   *reinterpret_cast<const uint32_t*>(&ov));
            }
        }
    }
    TL_MARK(5);
}

// TOPK: the Global part of each (seq, kv head) is K6's union selection
// (a.sel / a.nsel: logical page | q-head mask << 24) instead of every page;
// rows (q heads) that did not select a page get -inf logits for it.
template <bool TOPK>
__global__ void __launch_bounds__(DW * 32, CPS) decode_attn_mma_kernel(const __grid_constant__ CUtensorMap tpool,
                                                                      const __grid_constant__ DecArgs a,
                                                                      const __nv_bfloat16* __restrict__ q,
                                                                      float* __restrict__ part,
                                                                      int* __restrict__ nchunks,
                                                                      int* __restrict__ work_counter,
                                                                      const __grid_constant__ FinishArgs fin) {
    extern __shared__ uint8_t dsm_raw[];
    // 1 KB-aligned, by pointer arithmetic on the __shared__ array (an integer round
    // trip would lose the address space: every access through sm would be generic)
    uint8_t* sm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
    constexpr int d = 128;
    const int ps = 16;
    const int gs = a.q_heads / a.pv.kv_heads;
    const int npairs = a.n_pairs;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    TL_DECL
    TL_MARK(0);
#if WGKV_K5_PARAM_WARM
    {  // this launch's parameters into the SM's constant cache (a new block every
       // launch): the roles' first touches of them would otherwise be serial L2
       // round trips on the layer's critical path
        const uint32_t* pa = reinterpret_cast<const uint32_t*>(&a);
        const uint32_t* pf = reinterpret_cast<const uint32_t*>(&fin);
        uint32_t x = 0;
        for (int i = tid * 16; i < (int)(sizeof(DecArgs) / 4); i += blockDim.x * 16) x ^= pa[i];
        for (int i = tid * 16; i < (int)(sizeof(FinishArgs) / 4); i += blockDim.x * 16) x ^= pf[i];
        asm volatile("" ::"r"(x));
    }
#endif
#if WGKV_K5_EVICT_FIRST
    const uint64_t l2pol = tc::policy_evict_first();  // the cache is streamed once per token step
#endif
    __shared__ int s_rlast;
    if (!TOPK && (int)blockIdx.x < a.n_route_ctas) {
        // fused layer: the append's route CTA (fused.cuh), before the PDL wait
        // when the predecessor is another layer's launch
        const int pr = blockIdx.x, s = pr / a.pv.kv_heads, h = pr % a.pv.kv_heads;
        fused_route<__nv_bfloat16>(a.pv, a.layer, a.seq0, s, h, a.window, fin.wk, fin.fw, !a.prewait);
        __syncthreads();  // the route's writes, then its arrivals (thread 0)
        if (tid == 0) {
            const int pairg = a.seq0 * a.pv.kv_heads + pr;
            // last on either only after a party that passed the PDL wait: the
            // commits' caller outputs then follow it too
            s_rlast = (pair_arrive(&fin.fw.cnt_kv[pairg]) ? 1 : 0) |
                      (!fin.forced_g && pair_arrive(&fin.fw.cnt_gw[pairg]) ? 2 : 0);
            if (s_rlast) asm volatile("griddepcontrol.wait;" ::: "memory");
            if (s_rlast & 2) fused_commit_gate(a.pv, fin.ga, a.seq0, s, h, fin.tr, fin.wk, fin.fw);
        }
        __syncthreads();
        if ((s_rlast & 1) && warp == 0)
            fused_commit_kv<__nv_bfloat16>(a.pv, fin.ga, a.layer, a.seq0, s, h, fin.k_new, fin.v_new, fin.forced_g,
                                           fin.tr, fin.wk, fin.fw, nullptr, nullptr);
        // C1 (fused layer): route CTA 0 also unpacks the previous layer's peer
        // exchange (it has finished its own role; nothing waits for it here)
        if (pr == 0 && fin.px.do_unpack) peer_unpack_cta(fin.px);
        TL_COMMIT(5, a.layer, 0);
        return;
    }
    if (!TOPK && (int)blockIdx.x < a.n_route_ctas + a.n_gate_ctas) {
        // deferred append's gate CTAs (append.cuh): the new token's exact fp64
        // gate (engine.cpp:300-303) is only consumed W steps later (when the
        // token leaves the ring), so it runs beside the attention instead of
        // behind it; W1 is staged before the PDL wait
        const int gpp = gate_ctas_per_pair(fin.ga.hidden);
        const int gb = blockIdx.x - a.n_route_ctas;
        const int pr = gb / gpp, j = gb % gpp;
        const int s = pr / a.pv.kv_heads, h = pr % a.pv.kv_heads;
        // fused layer behind another layer's launch: the gate scratch (terms,
        // counters, g) is split by layer parity, so only the commit (caller
        // trace outputs) waits for the predecessor; the other gate CTAs exit early
        const bool gate_early = WGKV_GATE_EARLY && a.fused && a.prewait;
        append_gate_part<__nv_bfloat16>(a.pv, fin.ga, a.layer, a.seq0, s, h, j, fin.k_new, fin.wk, sm, !gate_early,
                                        a.prewait != 0);
        if (a.fused) {
            // the last gate CTA of the pair sums z2, then arrives for the gate group (fused.cuh)
            const int pairg = a.seq0 * a.pv.kv_heads + pr;
            if (fused_gate_arrive(a.pv, fin.ga, a.layer, pairg, h, fin.wk, fin.fw, sm)) {
                __syncthreads();  // fw.g written (thread 0)
                if (tid == 0) {
                    if (gate_early) asm volatile("griddepcontrol.wait;" ::: "memory");
                    if (pair_arrive(&fin.fw.cnt_gw[pairg]))
                        fused_commit_gate(a.pv, fin.ga, a.seq0, s, h, fin.tr, fin.wk, fin.fw);
                }
            }
        } else {
            append_arrive(a.pv, fin.ga, a.layer, a.seq0, s, h, fin.forced_g, fin.tr, fin.wk, gpp + 1, sm);
        }
        TL_COMMIT(2, a.layer, 0);
        return;
    }
    const int nfront = a.n_route_ctas + a.n_gate_ctas;
    const int kcta = (int)blockIdx.x - nfront, kgrid = (int)gridDim.x - nfront;
    // Launched as a programmatic dependent of the previous kernel (K4, the
    // previous layer's finish kernel, or K6's compaction).  Deferred path: the
    // predecessor (finish of another layer) owns only the shared workspace
    // (partials, chunk counts, work counter) and its own layer's pages, so the
    // planning pass, the first item's page ids and its first TMA loads -- this
    // layer's state and pages -- run before griddepcontrol.wait; q (a caller
    // input) and every workspace write come after it.  Only when the host saw
    // that the kernel in front is ANOTHER layer's finish kernel (a.prewait):
    // the same layer's finish publishes the state and writes the ring.  Top-k:
    // the selection is the predecessor's output, so everything waits.
    bool waited = false;
    auto pdl_wait = [&]() {
        if (waited) return;
        asm volatile("griddepcontrol.wait;" ::: "memory");
        TL_MARK(2);
        // let the kernel that merges our partials launch now (it waits for our completion)
        if (a.early_trigger) asm volatile("griddepcontrol.launch_dependents;");
        waited = true;
    };
    if (TOPK || !a.defer || !a.prewait) pdl_wait();
    uint8_t* ring = sm;                                                                    // [DW][DNS][8 KB]
    __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(sm + DW * DNS * PAGE_B);          // [16][QROW]
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + DW * DNS * PAGE_B + 16 * QROW * 2);  // [DW][DNS]
    float* red = reinterpret_cast<float*>(ring);  // [DW][16][d + 2], aliases the idle ring at merge time
    int* item_base = reinterpret_cast<int*>(full + DW * DNS);                              // [npairs + 1]
    int* pids = item_base + npairs + 1;                                                    // [PID_CAP]
    // per-pair head state, loaded once by the planning pass (an item then needs
    // no dependent global round trip before its page ids)
    HeadState* sst = reinterpret_cast<HeadState*>(pids + PID_CAP);                         // [npairs]
    __shared__ int s_cp, s_items;

    // ---- device-side split: uniform chunk size from the actual page counts --
    // (all threads: the per-pair state loads are independent, so they are
    // spread over the block instead of a serial loop of dependent round trips)
    __shared__ long s_wtot[DW];
    __shared__ int s_wmax[DW], s_wscan[DW];
    {
        // pass 1: each thread owns a contiguous run of pairs; page counts staged in item_base
        const int run = (npairs + blockDim.x - 1) / blockDim.x;
        const int p0 = tid * run, p1 = min(npairs, p0 + run);
        long tot = 0;
        int npmax = 0;
        for (int p = p0; p < p1; ++p) {
            const HeadState st = a.pv.state[a.pv.head_index(a.layer, a.seq0 + p / a.pv.kv_heads, p % a.pv.kv_heads)];
            if (a.state_in_smem) sst[p] = st;
            const int ngv = TOPK ? a.nsel[p] : (st.global_len + ps - 1) / ps;
            const int np = ngv + (st.local_len + ps - 1) / ps;
            item_base[p] = np;
            tot += np;
            npmax = max(npmax, np);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            tot += __shfl_xor_sync(0xffffffffu, tot, o);
            npmax = max(npmax, __shfl_xor_sync(0xffffffffu, npmax, o));
        }
        if (lane == 0) {
            s_wtot[warp] = tot;
            s_wmax[warp] = npmax;
        }
        __syncthreads();
        tot = 0;
        npmax = 0;
#pragma unroll
        for (int w = 0; w < DW; ++w) {
            tot += s_wtot[w];
            npmax = max(npmax, s_wmax[w]);
        }
        const long total = tot;
        // ~2 items per CTA, taken dynamically (work stealing) for balance
        const int ipc = WGKV_K5_IPC ? WGKV_K5_IPC : (npairs <= 64 ? 2 : 3);
        int cp = (int)((total + ipc * kgrid - 1) / (ipc * (long)kgrid));
        cp = max(cp, WGKV_K5_MIN_PAGES);  // per-item fixed costs (page ids, ring fill, merge) amortised
#if WGKV_K5_RULE == 1
        // few, long pairs (small batches): cap the chunks per pair near 24 (the
        // combine merges every chunk) while keeping >= grid/2 items in flight
        cp = max(cp, (int)min((long)(npmax + WGKV_K5_CAPCH - 1) / WGKV_K5_CAPCH,
                              (WGKV_K5_ITEMS_DIV * total + kgrid - 1) / kgrid));
#endif
        if (a.pin_cp > 0) cp = a.pin_cp;  // pinned split: per-head arithmetic independent of the launch
        cp = max(cp, (npmax + a.max_chunks - 1) / a.max_chunks);
        cp = min(cp, PID_CAP);  // host guarantees npmax <= max_chunks * PID_CAP
        // pass 2: chunks per pair, exclusive scan into item_base
        int nc_run = 0;
        for (int p = p0; p < p1; ++p) nc_run += max(1, (item_base[p] + cp - 1) / cp);
        int incl = nc_run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_wscan[warp] = incl;
        __syncthreads();  // also: every pass-1 read of s_wtot / s_wmax is done
        int acc = incl - nc_run;
        for (int w = 0; w < warp; ++w) acc += s_wscan[w];
        for (int p = p0; p < p1; ++p) {
            const int nc = max(1, (item_base[p] + cp - 1) / cp);
            item_base[p] = acc;
            acc += nc;
        }
        if (p1 == npairs && p0 < p1) {
            item_base[npairs] = acc;
            s_items = acc;
        }
        if (tid == 0) s_cp = cp;
    }
    __shared__ __align__(8) uint64_t s_tbar;  // fused layer: the tail's bulk copies
    uint32_t tpar = 0;
    if (tid < DW * DNS) tc::mbar_init(&full[tid], 1);
    if (tid == DW * DNS) tc::mbar_init(&s_tbar, 1);
    tc::fence_barrier_init();
    __syncthreads();
    const int cp = s_cp, nitems = s_items;
    TL_MARK(1);
    // fused layer: this CTA has planned from the old head states (the result
    // is only looked at when the CTA ends: the last planner publishes)
    int planned_rank = 0;
    if (!TOPK && a.fused && tid == 0) planned_rank = atomicAdd(fin.fw.started, 1);
    int tl_items = 0;
    const float qs = rsqrtf((float)d) * 1.4426950408889634f;
    const float LN2 = 0.6931471805599453f;
    const uint32_t wring = smem_u32(ring) + warp * DNS * PAGE_B;
    uint32_t kq = 0;  // pages this warp has issued / consumed so far (ring position + parity)

    // after the PDL wait: the plan's chunk counts and (deferred) the new tokens'
    // positions for the merging kernel -- the workspace the predecessor read
    bool published = false;
    auto publish_plan = [&]() {
        pdl_wait();
        if (published) return;
        published = true;
        if (kcta != 0 || a.fused) return;
        for (int p = tid; p < npairs; p += blockDim.x) {
            nchunks[p] = item_base[p + 1] - item_base[p];
            if (!TOPK && a.defer)
                a.tokpos[p] = a.state_in_smem
                                  ? sst[p].tokens_seen
                                  : a.pv.state[a.pv.head_index(a.layer, a.seq0 + p / a.pv.kv_heads, p % a.pv.kv_heads)]
                                        .tokens_seen;
        }
    };
    __shared__ int s_item;
#ifndef WGKV_K5_EARLY_ITEM
#define WGKV_K5_EARLY_ITEM 1
#endif
#ifndef WGKV_K5_WAIT_WARP_PAIRS
#define WGKV_K5_WAIT_WARP_PAIRS 16  // early first item: one warp waits (and triggers) up to this many pairs
#endif
#ifndef WGKV_K5_EARLY_FUSED
#define WGKV_K5_EARLY_FUSED 1
#endif
    const bool early_item = WGKV_K5_EARLY_ITEM && !TOPK && a.defer && a.prewait && (!a.fused || WGKV_K5_EARLY_FUSED);
    int next_draw = 0;  // fused layer: the next item's draw, claimed at the end of the previous item
    // first item static (kcta): no atomic round trip in front of it; later items
    // are stolen from kgrid on (the merging kernel resets the counter to 0 --
    // only read after the PDL wait, which the first item passes)
    for (int first = 1;; first = 0) {
        if (tid == 0) {
            if (first) {
                s_item = kcta;
            } else {
                const int v = a.fused ? next_draw : atomicAdd(work_counter, 1);
                s_item = kgrid + v;
                // fused layer: no merging kernel follows; the last of the
                // min(kgrid, nitems) + max(0, nitems - kgrid) draws resets it
                if (a.fused && v == min(kgrid, nitems) + max(0, nitems - kgrid) - 1) *work_counter = 0;
            }
        }
        __syncthreads();
        const int item = s_item;
        if (item >= nitems) {
            publish_plan();
            break;
        }
        ++tl_items;
        // pair of this item: the last bh with item_base[bh] <= item (binary search)
        int bh = 0;
        for (int lo = 0, hi = npairs - 1; lo <= hi;) {
            const int mid = (lo + hi) >> 1;
            if (item_base[mid] <= item) {
                bh = mid;
                lo = mid + 1;
            } else {
                hi = mid - 1;
            }
        }
        const int chunk = item - item_base[bh];
        const int s = bh / a.pv.kv_heads, h = bh % a.pv.kv_heads;
        const long hidx = a.pv.head_index(a.layer, a.seq0 + s, h);
        const HeadState st = a.state_in_smem ? sst[bh] : a.pv.state[hidx];
        // the query's position: after the append (K4 ran first) or, deferred, the
        // token about to be appended
        const long pos = (!TOPK && a.defer) ? st.tokens_seen : st.tokens_seen - 1;
        const int ngp = (st.global_len + ps - 1) / ps;
        const int ng = TOPK ? a.nsel[bh] : ngp;  // virtual Global pages
        const int NP = ng + (st.local_len + ps - 1) / ps;
        // TOPK: the partial last Global page can only be the last union entry
        const int32_t* usel = TOPK ? a.sel + (size_t)bh * a.pv.n_gp : nullptr;
        const bool last_sel = TOPK && ng > 0 && (usel[ng - 1] & 0xFFFFFF) == ngp - 1;
        const int vp0 = chunk * cp, vp1 = min(NP, vp0 + cp);
        // deferred append: a full ring's victim (slot local_ptr, position pos - W)
        // stays attended only when admitted (it is being promoted); a dropped
        // victim is masked -- the attended set equals the reference's after
        // local_write (kvstore.cpp:135-158, engine.cpp:308-326)
        int vm_vp = -1, vm_slot = 0;
        if (!TOPK && a.defer && st.local_len >= a.window) {
            const int vvp = ng + st.local_ptr / ps;
            if (vvp >= vp0 && vvp < vp1) {
                const int lpg = a.pv.lpt[hidx * a.pv.n_lp + st.local_ptr / ps];
                if (lpg >= 0 && !a.pv.adm[(size_t)lpg * ps + st.local_ptr % ps]) {
                    vm_vp = vvp;
                    vm_slot = st.local_ptr % ps;
                }
            }
        }
        const size_t pstride = (size_t)gs * (d + 2);
        float* pout = part + ((size_t)bh * a.max_chunks + chunk) * pstride;

        // stage this item's physical page ids (coalesced) so the TMA issue
        // never waits on a dependent global load
        for (int v = vp0 + tid; v < vp1; v += blockDim.x) {
            if (TOPK) {  // page id | q-head mask << 24 (local pages: every head)
                int pg;
                uint32_t mk;
                if (v < ng) {
                    const uint32_t e = (uint32_t)usel[v];
                    pg = a.pv.gpt[hidx * a.pv.n_gp + (e & 0xFFFFFFu)];
                    mk = e >> 24;
                } else {
                    pg = a.pv.lpt[hidx * a.pv.n_lp + (v - ng)];
                    mk = 0xFFu;
                }
                if (pg < 0) pg = mk = 0;  // failed allocation (latched ENOPAGES): masked
                pids[v - vp0] = (int)((uint32_t)pg | (mk << 24));
            } else {
                pids[v - vp0] = v < ng ? a.pv.gpt[hidx * a.pv.n_gp + v] : a.pv.lpt[hidx * a.pv.n_lp + (v - ng)];
            }
        }
        __syncthreads();

        const int nmine = vp1 > vp0 ? (vp1 - vp0 - warp + DW - 1) / DW : 0;  // pages vp0+warp, +DW, ...
        auto page_of = [&](int vp, int& valid) -> int {
            if (TOPK)
                valid = vp < ng ? ((vp == ng - 1 && last_sel) ? st.global_len - (ngp - 1) * ps : ps)
                                : min(ps, st.local_len - (vp - ng) * ps);
            else
                valid = vp < ng ? min(ps, st.global_len - vp * ps) : min(ps, st.local_len - (vp - ng) * ps);
            const int pid = pids[vp - vp0];
            if (!TOPK && pid < 0) valid = 0;  // failed allocation (latched ENOPAGES): fully masked
            return pid;
        };
        auto issue = [&](int k) {  // k-th page of this warp (ring slot (kq + k) % DNS)
            int valid;
            int page = page_of(vp0 + warp + k * DW, valid);
            if (TOPK) page &= 0xFFFFFF;
            if (page < 0) page = 0;  // failed allocation (latched ENOPAGES): stream a harmless page
            const uint32_t slot = (kq + k) % DNS;
            uint8_t* dst = ring + (warp * DNS + slot) * PAGE_B;
            uint64_t* bar = &full[warp * DNS + slot];
            tc::mbar_arrive_expect_tx(bar, PAGE_B);
            // one box per page: {64 dims, 16 slots, 2 dim halves, K and V} lands as
            // K lo | K hi | V lo | V hi, each a [16][64] SW128 sub-tile
#if WGKV_K5_EVICT_FIRST
            tc::tma_load_4d_hint(dst, &tpool, bar, 0, 0, 0, 2 * page, l2pol);
#else
            tc::tma_load_4d(dst, &tpool, bar, 0, 0, 0, 2 * page);
#endif
        };
        if (lane == 0) {
            tc::fence_proxy_async_smem();
            for (int k = 0; k < min(DNS, nmine); ++k) issue(k);
        }
        // deferred layer behind another layer's launch (a.prewait): the first
        // item runs whole before the PDL wait -- its pages, state and q are
        // not the predecessor's; only its partial goes to the workspace the
        // predecessor reads, and is written after the wait below
        // (128K x 4: 88.2 -> 83.6 us per layer; 8-way shard 19.3 -> 18.2)
        if (!(early_item && first)) publish_plan();
        // RoPE(q) at pos, pre-scaled by log2(e)/sqrt(d), split q = hi + lo into two
        // bf16 halves (to ~2^-17 relative): row r < 8 holds hi, row r + 8 its lo, so
        // the one m16 S MMA yields both halves' dots (gs <= 8) and the only score
        // rounding left is the cache's own bf16 k; rows >= gs are zero
        // (computed while the first pages of the item are in flight)
        for (int e = tid; e < 8 * (d / 2); e += blockDim.x) {
            const int r = e / (d / 2), i = e % (d / 2);
            float y0 = 0.f, y1 = 0.f;
            if (r < gs) {
                const size_t off = ((size_t)s * a.q_heads + h * gs + r) * d + 2 * i;
                const float x0 = __bfloat162float(q[off]), x1 = __bfloat162float(q[off + 1]);
                float c, sn;
                rope_cs(a.freq, i, pos, c, sn);
                y0 = (x0 * c - x1 * sn) * qs;
                y1 = (x0 * sn + x1 * c) * qs;
            }
            const __nv_bfloat16 h0 = __float2bfloat16_rn(y0), h1 = __float2bfloat16_rn(y1);
            Qs[r * QROW + 2 * i] = h0;
            Qs[r * QROW + 2 * i + 1] = h1;
            Qs[(r + 8) * QROW + 2 * i] = __float2bfloat16_rn(y0 - __bfloat162float(h0));
            Qs[(r + 8) * QROW + 2 * i + 1] = __float2bfloat16_rn(y1 - __bfloat162float(h1));
        }
        __syncthreads();
        // Q A-fragments: 8 k-steps of 16 dims (rows 0..7 hi, 8..15 lo, only heads < gs nonzero)
        uint32_t qa[8][4];
        {
            const uint32_t qb = smem_u32(Qs);
            const int r = lane & 15, cb = (lane >> 4) * 8;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                ldsm_x4(qb + (uint32_t)(r * QROW + kk * 16 + cb) * 2u, qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
        }
        // early first item, few pairs: one warp passes the PDL wait now --
        // releasing our programmatic dependent as soon as the predecessor has
        // drained -- while the other warps stream their pages (no CTA barrier
        // until the merge).  2-way shard 47.1 -> 43.1 us per layer, 4-way 28.2 ->
        // 26.3; with 32 pairs (128K x 4) the earlier dependent costs 3 %
        if (early_item && first && warp == DW - 1 && npairs <= WGKV_K5_WAIT_WARP_PAIRS) pdl_wait();
        float o[16][4];
#pragma unroll
        for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
        float m = -INFINITY, l = 0.f;  // row (head) lane/4, log2 domain
        const int t0 = (lane & 3) * 2;
        for (int k = 0; k < nmine; ++k) {
            int valid;
            const int pidv = page_of(vp0 + warp + k * DW, valid);
            const uint32_t slot = (kq + k) % DNS;
            tc::mbar_wait(&full[warp * DNS + slot], ((kq + k) / DNS) & 1);
            const uint32_t kb = wring + slot * PAGE_B, vb = kb + 4096;
            // ---- S = Q K^T : two n8 tiles (tokens 0-7, 8-15) ------------------
            float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                // matrices: (tok 0-7, dims lo), (tok 0-7, hi), (tok 8-15, lo), (tok 8-15, hi)
                const int mi = lane >> 3, rr = lane & 7;
                const uint32_t tok = (mi >> 1) * 8 + rr;
                const uint32_t dch = (kk & 3) * 2 + (mi & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(swz(kb + (kk >> 2) * 2048u, tok, dch), b0, b1, b2, b3);
                mma16816(sc[0], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
                mma16816(sc[1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b2, b3);
            }
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {  // head lane/4: hi.k (row lane/4) + lo.k (row lane/4 + 8)
                sc[nt][0] += sc[nt][2];
                sc[nt][1] += sc[nt][3];
            }
            if (valid < 16) {  // partial page: token = nt*8 + t0 + e
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (nt * 8 + t0 + e >= valid) sc[nt][e] = -INFINITY;
            }
            if (!TOPK && vp0 + warp + k * DW == vm_vp) {  // the dropped victim (deferred append)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (nt * 8 + t0 + e == vm_slot) sc[nt][e] = -INFINITY;
            }
            if (TOPK && !(((uint32_t)pidv >> (24 + (lane >> 2))) & 1u))  // row lane/4 did not select this page
                sc[0][0] = sc[0][1] = sc[1][0] = sc[1][1] = -INFINITY;
            float mx = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float mn = fmaxf(m, mx);
            const float alpha = (m == -INFINITY) ? 0.f : ex2f(m - mn);
            const float mb = mn == -INFINITY ? 0.f : mn;  // row with nothing attended yet (masked pages)
            const float p00 = ex2f(sc[0][0] - mb), p01 = ex2f(sc[0][1] - mb);
            const float p10 = ex2f(sc[1][0] - mb), p11 = ex2f(sc[1][1] - mb);
            float ls = p00 + p01 + p10 + p11;
            ls += __shfl_xor_sync(0xffffffffu, ls, 1);
            ls += __shfl_xor_sync(0xffffffffu, ls, 2);
            l = l * alpha + ls;
            m = mn;
            const uint32_t pa0 = tc::pack_bf16x2(p00, p01), pa2 = tc::pack_bf16x2(p10, p11);
            // ---- O += P V : 16 n8 tiles over d, one k16 step over the tokens -----
#pragma unroll
            for (int n2 = 0; n2 < 8; ++n2) {
                // x4.trans: (tok 0-7, dims 16n2..+7), (tok 8-15, same), (tok 0-7, +8..15), (tok 8-15, +8..15)
                const int mi = lane >> 3, rr = lane & 7;
                const uint32_t tok = (mi & 1) * 8 + rr;
                const uint32_t dim0 = n2 * 16 + (mi >> 1) * 8;
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(swz(vb + (dim0 >> 6) * 2048u, tok, (dim0 & 63) >> 3), b0, b1, b2, b3);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    o[2 * n2][e] *= alpha;
                    o[2 * n2 + 1][e] *= alpha;
                }
                mma16816(o[2 * n2], pa0, 0u, pa2, 0u, b0, b1);
                mma16816(o[2 * n2 + 1], pa0, 0u, pa2, 0u, b2, b3);
            }
            __syncwarp();
            if (lane == 0 && k + DNS < nmine) {
                tc::fence_proxy_async_smem();
                issue(k + DNS);
            }
        }
        kq += nmine;
        // ---- merge warps: rows h = lane/4 < gs hold (m, l, O[h][:]) -------------
        __syncthreads();  // every warp is done with its ring slots (red aliases them)
        const int hrow = lane >> 2;
        float* rw = red + (size_t)warp * 16 * (d + 2);
        if (hrow < gs) {
#pragma unroll
            for (int n = 0; n < 16; ++n) {
                rw[hrow * (d + 2) + n * 8 + t0] = o[n][0];
                rw[hrow * (d + 2) + n * 8 + t0 + 1] = o[n][1];
            }
            if ((lane & 3) == 0) {
                rw[hrow * (d + 2) + d] = nmine > 0 ? m : -INFINITY;
                rw[hrow * (d + 2) + d + 1] = nmine > 0 ? l : 0.f;
            }
        }
        __syncthreads();
        publish_plan();  // the partial buffer is the predecessor's workspace (no-op after the first item)
        for (int e = tid; e < gs * d; e += blockDim.x) {
            const int g = e / d, c = e % d;
            float M = -INFINITY;
            for (int w = 0; w < DW; ++w) M = fmaxf(M, red[(size_t)w * 16 * (d + 2) + g * (d + 2) + d]);
            float acc = 0.f, L = 0.f;
            for (int w = 0; w < DW; ++w) {
                const float* r = red + (size_t)w * 16 * (d + 2) + g * (d + 2);
                const float sc = r[d] == -INFINITY ? 0.f : ex2f(r[d] - M);
                acc += sc * r[c];
                L += sc * r[d + 1];
            }
            pout[g * (d + 2) + c] = acc;
            if (c == 0) {  // partials carry m in natural-log units for decode_combine_kernel
                pout[g * (d + 2) + d] = M == -INFINITY ? -INFINITY : M * LN2;
                pout[g * (d + 2) + d + 1] = L;
            }
        }
        if (!TOPK && a.fused) {
            // the next item is claimed now: the atomic's round trip overlaps
            // the merge below instead of following it
            if (tid == 0) next_draw = atomicAdd(work_counter, 1);
            // the pair's last item merges its chunks and the new token; the
            // last party of the pair commits the append (fused.cuh)
            const int pairg = a.seq0 * a.pv.kv_heads + bh;
            if (cta_arrive(&fin.fw.cnt_items[pairg], item_base[bh + 1] - item_base[bh])) {
                TL_MARK(1);
                tl_items += 1000;
                fused_tail(a, fin, bh, item_base[bh + 1] - item_base[bh], pos, Qs, ring, part, &s_tbar, tpar TL_ARG);
            }
        }
        __syncthreads();
    }
    if (!TOPK && a.fused) {
        // the last CTA to plan: every CTA has read the old head states, so a
        // committed pair's new state may be published (handshake, fused.cuh)
        __shared__ int s_lastplan;
        if (tid == 0) {
            s_lastplan = planned_rank == kgrid - 1;
            if (s_lastplan) *fin.fw.started = 0;
        }
        __syncthreads();
        if (s_lastplan)
            for (int p = tid; p < npairs; p += blockDim.x)
                fused_pub(a.pv, fin.wk, fin.fw, a.layer, a.seq0 * a.pv.kv_heads + p);
    }
    TL_COMMIT(0, a.layer, tl_items);
    (void)tl_items;
}

int launch_decode_attn_mma(const DecArgs& a0, int nseq, const __nv_bfloat16* q, float* part, int* nchunks,
                           __nv_bfloat16* out, cudaStream_t st, bool counter_reset_by_append, const FinishArgs* fin) {
    DecArgs a = a0;
    const int gs = a.q_heads / a.pv.kv_heads;
    if (a.pv.head_dim != 128 || a.pv.page_size != 16 || gs > 16) return WGKV_ENOTSUP;
    // cached per pool (a new context may reuse a freed pool's address with
    // another capacity, so the key includes it); per host thread, since each
    // context is driven by one host thread
    static thread_local CUtensorMap tp;
    static thread_local const void* tp_base = nullptr;
    static thread_local long tp_cap = -1;
    if (tp_base != a.pv.data || tp_cap != a.pv.capacity) {
        // pool as [2*cap planes][2 dim halves][16 slots][64 dims] (the half stride is
        // smaller than the slot stride: a transposed view of [plane][slot][128])
        const uint64_t dims[4] = {64, 16, 2, 2 * (uint64_t)a.pv.capacity};
        const uint64_t strides[3] = {256, 128, 16 * 256};
        const uint32_t box[4] = {64, 16, 2, 2};
        if (make_tmap_4d_bf16(&tp, a.pv.data, dims, strides, box))
            return WGKV_ECUDA;
        tp_base = a.pv.data;
        tp_cap = a.pv.capacity;
    }
    a.n_pairs = nseq * a.pv.kv_heads;
    // CPS CTAs per SM: 228 KB per SM, 1 KB reserved per CTA, the kernels' static smem
    static size_t static_smem = 0;
    if (!static_smem) {
        cudaFuncAttributes fa0{}, fa1{};
        cudaFuncGetAttributes(&fa0, decode_attn_mma_kernel<false>);
        cudaFuncGetAttributes(&fa1, decode_attn_mma_kernel<true>);
        static_smem = std::max(fa0.sharedSizeBytes, fa1.sharedSizeBytes) + 1;
    }
    const size_t smem_cap = (size_t)(228 / CPS - 1) * 1024 - ((static_smem + 127) & ~size_t(127));
    size_t smem = 1024 + DW * DNS * PAGE_B + 16 * QROW * 2 + DW * DNS * 8 + 4 * ((size_t)a.n_pairs + 1) + 4 * PID_CAP;
    if (smem > smem_cap) return WGKV_ENOTSUP;
    // per-pair state cached in smem when it still fits CPS CTAs per SM
    a.state_in_smem = a.n_pairs <= kDecSmemStatePairs && smem + sizeof(HeadState) * (size_t)a.n_pairs <= smem_cap;
    if (a.state_in_smem) smem += sizeof(HeadState) * (size_t)a.n_pairs;
    const bool topk = a.sel != nullptr;
    auto kern = topk ? decode_attn_mma_kernel<true> : decode_attn_mma_kernel<false>;
    if (ensure_smem(kern, smem) != cudaSuccess) return WGKV_ECUDA;
    // work-stealing counter: one int past the per-(seq, kv head) chunk counts;
    // left at 0 by every kernel that merges K5's partials (combine / finish),
    // zeroed again by the kernel before us (PDL) or by a memset here
    int* counter = nchunks + (size_t)a.pv.max_seqs * a.pv.kv_heads;
    a.counter = counter;
    if (!counter_reset_by_append) cudaMemsetAsync(counter, 0, sizeof(int), st);
    // the deferred append's gate CTAs ride in this launch (see the kernel); the
    // finish kernel then runs only the route CTAs
    // Few gate CTAs (small batches): in this launch, where they cost K5 a few
    // slots for ~2 us.  Many (large batches, where they would displace most of
    // K5's first wave): first in the finish kernel's grid, which K5 releases
    // early, so they fill the slots K5's tail frees and overlap it.
    static const char* gp_env = getenv("WGKV_GATE_PLACE");  // A/B switch: "k5" | "finish"
    static const int gate_k5_max = gp_env ? (strcmp(gp_env, "k5") == 0 ? 1 << 30 : 0) : kGateInK5MaxCtas;
    static const bool no_trigger = getenv("WGKV_K5_NO_TRIGGER") != nullptr;  // A/B switch
    FinishArgs fa{};
    a.n_gate_ctas = 0;
    a.n_route_ctas = 0;
    a.fused = 0;
    const int ngate = fin && !fin->forced_g ? a.n_pairs * gate_ctas_per_pair(fin->ga.hidden) : 0;
    // fused layer (fused.cuh): while the route and gate CTAs fit in half a wave
    static const char* fu_env = getenv("WGKV_DECODE_FUSED");  // A/B switch: "0" off
    static const int fused_max = fu_env ? atoi(fu_env) : kFusedMaxFront;
    int kgrid = CPS * num_sms();
    // few pairs and narrow groups only: with more pairs (several items per CTA)
    // the per-item arrivals and the one-CTA merges cost more than a second
    // kernel's drain (profiles/r2_decode_fused_ab.txt)
    if (fin && fin->fw.cnt_items && !fin->gate_side && a.pin_cp == 0 && a.n_pairs + ngate <= fused_max &&
        a.n_pairs <= kFusedMaxPairs && gs <= 4) {
        a.fused = 1;
        a.n_route_ctas = a.n_pairs;
        a.n_gate_ctas = ngate;
        // every K5 CTA resident beside the route and gate CTAs (no late static items)
        kgrid -= a.n_pairs + ngate;
        fa = *fin;
        fa.out = out;
    } else if (fin && !fin->forced_g && !fin->gate_side && ngate <= gate_k5_max) {
        a.n_gate_ctas = ngate;
        fa = *fin;
    }
    // C1 over peer memory: the fused layer's merges push and its route CTA 0
    // unpacks; otherwise the finish kernel does both (fin->px)
    if (!a.fused) fa.px = PeerXchg{};
    a.early_trigger = fin && !no_trigger;
    a.prewait = fin && fin->prewait;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.n_route_ctas + a.n_gate_ctas + kgrid);
    cfg.blockDim = dim3(DW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = counter_reset_by_append ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, tp, a, q, part, nchunks, counter, fa);
    a.nchunks = nchunks;
    if (a.fused) return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
    if (fin) return launch_decode_finish(a, nseq, q, part, out, *fin, st);
    extern int launch_decode_combine_bf16(const DecArgs&, int, const float*, __nv_bfloat16*, cudaStream_t);
    return launch_decode_combine_bf16(a, nseq, part, out, st);
}

}  // namespace wgkv

TL_EXPORT(wgkv_tl_k5)
