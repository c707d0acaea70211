// append.cuh -- K4: one decode token of each (seq, kv head) into the dual cache.
//
// HeadCache::local_write + promote (kvstore.cpp:102-158) fused with the
// decode-time gate (gate_forward, gating.cpp:158-171) and RoPE
// (numerics.cpp:50-77).  One token per (seq, kv head) is a chain of dependent
// memory round trips (state -> ring page -> victim bit -> page pop -> copies)
// plus an fp64 gate whose weights (hidden x 2d doubles, 256 KB per head at
// d = hidden = 128) one SM would need several microseconds to stream.  So a
// pair's work is split over CTAs of one launch that run concurrently:
//   * the route CTA: RoPE of the new key, the routing decision (lazy promotion
//     of the ring victim on its stored bit, device page allocation), the
//     victim's copy into Global and the new token's K/V into the ring slot;
//   * ceil(hidden / 16) gate CTAs: 16 hidden units each, W1 rows staged
//     through shared memory, every z1 a sequential fp64 dot in the reference's
//     order (dot, numerics.cpp:94-99, no FMA) -> w2 * gelu(z1 + b1);
//   * whichever CTA of the pair arrives last (an arrival counter) sums
//     z2 = b2 + terms in order, applies sigmoid and the clamp, writes the
//     token's gate and bit into its slot, publishes the new HeadState (only
//     now, so every CTA of the pair saw the old one) and the GateTrace.
// Used by the standalone append kernel (admit.cu) and by the decode finish
// kernel (decode_finish.cu), which runs these CTAs beside the chunk merge.
#pragma once
#include "common.cuh"
#include "gate.cuh"

namespace wgkv {

// GateTrace outputs of one decode step (records.hpp:11-29, engine.cpp:300-305),
// [nseq][kv_heads] each, any may be null
struct DecodeTrace {
    float* g;          // gate score of the new token (fp32 copy of the fp64 value)
    uint8_t* bits;     // g >= tau
    uint8_t* near_tau; // |g - tau| < 1e-6 (the band north_star asks to report)
    int32_t* events;   // PromotionEvent of the ring victim: 0 none, 1 promoted, 2 dropped, -1 failed
};

// per-(seq, kv head) scratch of the split append, [max_seqs * kv_heads] (+ terms)
struct AppendWork {
    double* terms;       // [pair][hidden] w2 * gelu(z1 + b1) from the gate CTAs
    int* count;          // arrivals of the pair's CTAs; the last one resets it to 0
    int* slot;           // new token's pool slot (page * ps + slot) or -1
    int* event;          // promotion event (0 none, 1 promoted, 2 dropped, -1 failed)
    HeadState* next;     // the state after the append, published by the last arrival
    int* pos;            // the new token's position (split launch: route kernel -> gate kernel)
    // split launch (route CTAs, then the gate CTAs in a kernel on a side stream
    // that overlaps the attention): the route CTA publishes the head state
    // itself -- the attention reads it -- and leaves the position in `pos`
    int early_state;
};

constexpr int kAppendThreads = 256;
#ifndef WGKV_GATE_UNITS
#define WGKV_GATE_UNITS 16
#endif
constexpr int kGateUnits = WGKV_GATE_UNITS;  // hidden units per gate CTA
__host__ __device__ inline int gate_ctas_per_pair(int hidden) { return (hidden + kGateUnits - 1) / kGateUnits; }
// dynamic smem of the roles: gate = feature [2d] + W1 rows [16][2d + 1] doubles
__host__ __device__ inline size_t append_smem_bytes(int d, int hidden) {
    return sizeof(double) * (2 * (size_t)d + (size_t)kGateUnits * (2 * d + 1)) + 16;
}

// ---------------------------------------------------------------------------
// the last arrival of a pair finishes the token (thread 0 only)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void append_finalize(const PoolView& pv, const GateArgs& ga, int layer, int seq0, int s,
                                                int h, const float* __restrict__ forced_g, const DecodeTrace& tr,
                                                const AppendWork& wk, const double* terms) {
    const int pair = (seq0 + s) * pv.kv_heads + h;
    const int blk = layer * pv.kv_heads + h;
    const int sl = __ldcg(&wk.slot[pair]);
    const int ev = __ldcg(&wk.event[pair]);
    double g;
    if (forced_g) {
        g = (double)forced_g[(size_t)s * pv.kv_heads + h];
    } else {  // z2 = b2 + sum_h terms, sequential (gating.cpp:162-166)
        double z2 = ga.b2d[blk];
        for (int u = 0; u < ga.hidden; ++u) z2 = __dadd_rn(z2, terms[u]);
        g = gate_from_z2(z2);
    }
    const uint8_t bit = g >= ga.tau ? 1 : 0;
    if (sl >= 0) {
        pv.gate[sl] = (float)g;
        pv.adm[sl] = bit;
    }
    if (ev >= 0 && !wk.early_state) {
        const int4 ns = __ldcg(reinterpret_cast<const int4*>(wk.next + pair));
        pv.state[pv.head_index(layer, seq0 + s, h)] = HeadState{ns.x, ns.y, ns.z, ns.w};
    }
    const size_t o = (size_t)s * pv.kv_heads + h;
    if (tr.g) tr.g[o] = (float)g;
    if (tr.bits) tr.bits[o] = bit;
    if (tr.near_tau) tr.near_tau[o] = fabs(g - ga.tau) < 1e-6 ? 1 : 0;
    if (tr.events) tr.events[o] = ev;
    wk.count[pair] = 0;  // ready for the next step
}

// every CTA of a pair calls this once its writes are issued (whole CTA); the
// last one finalises.  smem: >= hidden doubles (free by now): the gate CTAs'
// terms come in one parallel round of loads for the sequential z2 sum
__device__ __forceinline__ void append_arrive(const PoolView& pv, const GateArgs& ga, int layer, int seq0, int s, int h,
                                              const float* __restrict__ forced_g, const DecodeTrace& tr,
                                              const AppendWork& wk, int arrivals, uint8_t* smem) {
    __shared__ int last;
    const int pair = (seq0 + s) * pv.kv_heads + h;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();  // release this CTA's writes
        last = atomicAdd(&wk.count[pair], 1) == arrivals - 1;
        if (last) __threadfence();  // acquire: the other CTAs' terms / slot / state
    }
    __syncthreads();
    if (!last) return;
    double* terms = reinterpret_cast<double*>(smem);
    if (!forced_g)
        for (int u = threadIdx.x; u < ga.hidden; u += blockDim.x) terms[u] = __ldcg(wk.terms + (size_t)pair * ga.hidden + u);
    __syncthreads();
    if (threadIdx.x == 0) append_finalize(pv, ga, layer, seq0, s, h, forced_g, tr, wk, terms);
}

// ---------------------------------------------------------------------------
// the routing decision of one new token (thread 0): lazy promotion of the ring
// victim on its stored bit, device page allocation, the victim's metadata copy
// into Global and the new token's position in its slot (kvstore.cpp:102-158)
// ---------------------------------------------------------------------------
struct RouteDecision {
    int ev;     // promotion event (0 none, 1 promoted, 2 dropped, -1 failed)
    int gpage;  // promoted victim's Global page / slot
    int gslot;
    int npage;  // the new token's ring page / slot (npage < 0: failed)
    int nslot;
    HeadState ns;  // the head state after the append
};
__device__ __forceinline__ RouteDecision route_decide(const PoolView& pv, long hidx, const HeadState& st, long W,
                                                      int lp0) {
    const int ps = pv.page_size;
    const long pos = st.tokens_seen;
    const int slot = st.local_ptr;
    const bool ring_full = st.local_len >= W;
    int lp = lp0;
    int ev = 0, vp = -1, gp = -1, gs_ = 0;
    HeadState ns = st;
    // the Global tail page (needed if the victim is promoted into a partly
    // filled page), loaded alongside
    const int gi = st.global_len;
    const int gp_tail = (gi % ps != 0) ? pv.gpt[hidx * pv.n_gp + gi / ps] : -1;
    // an allocation failure behaves like the reference's throw from
    // alloc_page inside local_write (kvstore.cpp:23-31, 102-158): nothing of
    // this head changes, the error is latched, the event reads -1
    bool fail = false;
    if (!ring_full) {
        // not full: slot == local_len; a slot at a page boundary is the first
        // touch of that ring page (kvstore.cpp:102-107)
        if (slot % ps == 0) {
            lp = pool_pop(pv);
            if (lp >= 0) pv.lpt[hidx * pv.n_lp + slot / ps] = lp;
        }
        fail = lp < 0;
        if (!fail) ns.local_len += 1;
    } else if (lp < 0) {
        fail = true;  // the head lost its pages to an earlier ENOPAGES
    } else if (pv.adm[(size_t)lp * ps + slot % ps]) {
        // the victim under local_ptr is admitted: promote (kvstore.cpp:122-147)
        gp = gp_tail;
        if (gi % ps == 0) {
            gp = pool_pop(pv);
            if (gp >= 0) pv.gpt[hidx * pv.n_gp + gi / ps] = gp;
        }
        if (gp < 0) {
            fail = true;
        } else {
            ev = 1;
            vp = lp;
            gs_ = gi % ps;
            ns.global_len += 1;
        }
    } else {
        ev = 2;  // dropped
    }
    if (fail) {
        ev = -1;
        lp = -1;
    } else {
        ns.local_ptr = (int)((st.local_ptr + 1) % W);
        ns.tokens_seen += 1;
    }
    if (ev == 1) {  // the victim's metadata, read before the new token overwrites the slot
        const size_t a = (size_t)vp * ps + slot % ps, b = (size_t)gp * ps + gs_;
        pv.gate[b] = pv.gate[a];
        pv.pos[b] = pv.pos[a];
        pv.adm[b] = pv.adm[a];
    }
    if (lp >= 0) pv.pos[(size_t)lp * ps + slot % ps] = (int32_t)pos;
    return RouteDecision{ev, gp, gs_, lp, slot % ps, ns};
}

// ---------------------------------------------------------------------------
// route CTA: RoPE, lazy promotion, ring write (no gate)
// ---------------------------------------------------------------------------
template <typename E>
// pdl_wait (the decode finish kernel, a programmatic dependent of K5): every
// read, the routing decision, page pops, page-table and metadata writes happen
// before griddepcontrol.wait -- K5 reads none of them (new pages lie past the
// attended ones; a promoted victim lands past the tail page's valid rows) --
// and only the K/V stores into the victim's ring slot, which K5 is streaming,
// wait for K5 to complete.
__device__ __forceinline__ void append_route(const PoolView& pv, const GateArgs& ga, int layer, int seq0, int s, int h,
                                             long W, const E* __restrict__ k_pre, const E* __restrict__ v,
                                             const AppendWork& wk, bool pdl_wait = false) {
    const int tid = threadIdx.x, d = pv.head_dim, ps = pv.page_size;
    const long hidx = pv.head_index(layer, seq0 + s, h);
    const int pair = (seq0 + s) * pv.kv_heads + h;
    __shared__ int gpage, gslot, npage, nslot, event;
    const size_t in = ((size_t)s * pv.kv_heads + h) * d;
    E* pool = reinterpret_cast<E*>(pv.data);
    // the new token's inputs do not depend on the cache state: loads first;
    // every thread reads the state and the ring page under local_ptr itself, so
    // the victim's K/V is fetched in the same round as its admission bit
    const bool kt = tid < d / 2, et = tid < d;
    const float x0 = kt ? to_f(k_pre[in + 2 * tid]) : 0.f, x1 = kt ? to_f(k_pre[in + 2 * tid + 1]) : 0.f;
    const E vnew = et ? v[in + tid] : E();
    const HeadState st = pv.state[hidx];
    const long pos = st.tokens_seen;
    const int slot = st.local_ptr;
    const int lp0 = pv.lpt[hidx * pv.n_lp + slot / ps];
    const bool ring_full = st.local_len >= W;
    E vk = E(), vv = E();
    if (ring_full && lp0 >= 0 && et) {
        const E* ks = pool + (size_t)lp0 * pv.page_elems() + (size_t)(slot % ps) * d;
        vk = ks[tid];
        vv = ks[tid + (size_t)ps * d];
    }
    float y0 = 0.f, y1 = 0.f;  // the cached key: fp64 angle, fp32 rotation
    if (kt) {
        float c, sn;
        rope_cs(ga.freq, tid, pos, c, sn);
        rope_pair_f32(x0, x1, c, sn, y0, y1);
    }
    if (tid == 0) {
        const RouteDecision r = route_decide(pv, hidx, st, W, lp0);
        event = r.ev;
        gpage = r.gpage;
        gslot = r.gslot;
        npage = r.npage;
        nslot = r.nslot;
        wk.next[pair] = r.ns;
        wk.event[pair] = r.ev;
        if (wk.early_state) {
            wk.pos[pair] = (int)pos;
            if (r.ev >= 0) pv.state[hidx] = r.ns;
        }
        wk.slot[pair] = r.npage >= 0 ? r.npage * ps + r.nslot : -1;
    }
    __syncthreads();
    if (pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    // promote the victim (K/V fetched above), then the new token into the ring
    if (event == 1 && et) {
        E* kd = pool + (size_t)gpage * pv.page_elems() + (size_t)gslot * d;
        kd[tid] = vk;
        kd[tid + (size_t)ps * d] = vv;
    }
    if (npage >= 0) {
        E* kd = pool + (size_t)npage * pv.page_elems() + (size_t)nslot * d;
        if (kt) {
            kd[2 * tid] = from_f<E>(y0);
            kd[2 * tid + 1] = from_f<E>(y1);
        }
        if (et) kd[tid + (size_t)ps * d] = vnew;
    }
}

// ---------------------------------------------------------------------------
// gate CTA j of a pair: terms of hidden units [16 j, 16 j + 16)
// ---------------------------------------------------------------------------
// pdl_wait: the CTA runs in the K5 launch, a programmatic dependent whose
// predecessor may still own the pair's scratch and the head state: only the
// W1 rows (gate parameters, unchanged while decoding) are staged before
// griddepcontrol.wait.  In the finish kernel the gate CTAs need no wait: K5
// (their primary) passed its own wait before releasing them, so every earlier
// kernel -- the previous layer's finalize included -- has completed.
template <typename E>
__device__ __forceinline__ void append_gate_part(const PoolView& pv, const GateArgs& ga, int layer, int seq0, int s,
                                                 int h, int j, const E* __restrict__ k_pre, const AppendWork& wk,
                                                 uint8_t* smem, bool pdl_wait = false, bool early_pos = false) {
    const int tid = threadIdx.x, d = pv.head_dim, fd = 2 * d, hid = ga.hidden;
    const int pair = (seq0 + s) * pv.kv_heads + h;
    const int blk = layer * pv.kv_heads + h;
    const int u0 = j * kGateUnits, nu = min(kGateUnits, hid - u0);
    double* xs = reinterpret_cast<double*>(smem);  // [2d] feature [k_pre ; RoPE(k_pre)] (fp64)
    double* ws = xs + fd;                          // [16][2d + 1] W1 rows (padded: conflict-free columns)
    const double* w1 = ga.w1d + ((size_t)blk * hid + u0) * fd;
    // W1 rows, coalesced (16-byte vectors when 2d is even: it is)
    for (int e = tid; e < nu * fd / 2; e += blockDim.x) {
        const int r = e / (fd / 2), c2 = e % (fd / 2);
        const double2 w = reinterpret_cast<const double2*>(w1 + (size_t)r * fd)[c2];
        ws[r * (fd + 1) + 2 * c2] = w.x;
        ws[r * (fd + 1) + 2 * c2 + 1] = w.y;
    }
    // the state is published only by the pair's last arrival: tokens_seen is the new token's position
    // (split launch: the route CTA published it already and left the position in wk.pos)
    auto position = [&]() -> long {
        return wk.early_state ? (long)wk.pos[pair] : pv.state[pv.head_index(layer, seq0 + s, h)].tokens_seen;
    };
    // early_pos (K5 launch whose predecessor is another layer's: this layer's
    // state is final): the fp64 angles' cos / sin before the wait, off the path
    double* cs = ws + kGateUnits * (fd + 1);  // [d/2][2] (early_pos)
    if (early_pos) {
        const long pos = position();
        for (int i = tid; i < d / 2; i += blockDim.x) {
            const double angle = __dmul_rn((double)pos, ga.freq[i]);
            cs[2 * i] = cos(angle);
            cs[2 * i + 1] = sin(angle);
        }
    }
    if (pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    const long pos = early_pos ? 0 : position();
    const size_t in = ((size_t)s * pv.kv_heads + h) * d;
    // the feature in the reference's arithmetic (numerics.cpp:53-62)
    for (int i = tid; i < d / 2; i += blockDim.x) {
        const double a = to_f(k_pre[in + 2 * i]), b = to_f(k_pre[in + 2 * i + 1]);
        double cd, sd;
        if (early_pos) {
            cd = cs[2 * i];
            sd = cs[2 * i + 1];
        } else {
            const double angle = __dmul_rn((double)pos, ga.freq[i]);
            cd = cos(angle);
            sd = sin(angle);
        }
        xs[2 * i] = a;
        xs[2 * i + 1] = b;
        xs[d + 2 * i] = __dsub_rn(__dmul_rn(a, cd), __dmul_rn(b, sd));
        xs[d + 2 * i + 1] = __dadd_rn(__dmul_rn(a, sd), __dmul_rn(b, cd));
    }
    __syncthreads();
    if (tid < nu) {
        const double* wr = ws + tid * (fd + 1);
        double z1 = 0.0;  // dot (numerics.cpp:94-99)
        for (int k = 0; k < fd; ++k) z1 = __dadd_rn(z1, __dmul_rn(wr[k], xs[k]));
        const int u = u0 + tid;
        wk.terms[(size_t)pair * hid + u] = __dmul_rn(ga.w2d[(size_t)blk * hid + u], gelu_ref(__dadd_rn(z1, ga.b1d[(size_t)blk * hid + u])));
    }
}

// CTA role dispatch of the split append: r in [0, npairs) route CTAs, then
// npairs * gpp gate CTAs of this launch (0 with forced gates, or when the K5
// launch ran the pair's gate CTA); `arrivals` = CTAs per pair over both launches
template <typename E>
__device__ __forceinline__ void append_role(const PoolView& pv, const GateArgs& ga, int layer, int seq0, long W,
                                            int npairs, int r, int gpp, int arrivals, const E* __restrict__ k_pre,
                                            const E* __restrict__ v, const float* __restrict__ forced_g,
                                            const DecodeTrace& tr, const AppendWork& wk, uint8_t* smem,
                                            bool pdl_wait = false) {
    int pr, j = -1;
    if (r < npairs) {
        pr = r;
    } else {
        pr = (r - npairs) / gpp;
        j = (r - npairs) % gpp;
    }
    const int s = pr / pv.kv_heads, h = pr % pv.kv_heads;
    if (j < 0)
        append_route<E>(pv, ga, layer, seq0, s, h, W, k_pre, v, wk, pdl_wait);
    else
        append_gate_part<E>(pv, ga, layer, seq0, s, h, j, k_pre, wk, smem);
    append_arrive(pv, ga, layer, seq0, s, h, forced_g, tr, wk, arrivals, smem);
}

}  // namespace wgkv
