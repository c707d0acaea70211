// append.cuh -- K4: one decode token of one (seq, kv head) into the dual cache.
//
// HeadCache::local_write + promote (kvstore.cpp:102-158) fused with the
// decode-time gate (gate_forward, gating.cpp:158-171, in the reference's exact
// fp64 operation order) and RoPE (numerics.cpp:50-77), run by one 256-thread
// CTA.  Used by the standalone append kernel (admit.cu) and by the decode
// finish kernel (decode_finish.cu), which runs it beside the chunk merge of
// the same layer.
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

constexpr int kAppendThreads = 256;
// dynamic smem of append_token: xs [2d] + terms [hidden] doubles, kpost [d] floats
__host__ __device__ inline size_t append_smem_bytes(int d, int hidden) {
    return sizeof(double) * (2 * (size_t)d + (size_t)hidden) + sizeof(float) * (size_t)d;
}

// s: call-relative sequence index (inputs are [nseq][kv_heads][d]); the cache
// slot is seq0 + s.  Whole CTA (kAppendThreads threads), smem from the caller.
template <typename E>
__device__ __forceinline__ void append_token(const PoolView& pv, const GateArgs& ga, int layer, int seq0, int s, int h,
                                             long W, const E* __restrict__ k_pre, const E* __restrict__ v,
                                             const float* __restrict__ forced_g, const DecodeTrace& tr,
                                             uint8_t* smem) {
    const int tid = threadIdx.x, d = pv.head_dim, ps = pv.page_size;
    const long hidx = pv.head_index(layer, seq0 + s, h);
    double* xs = reinterpret_cast<double*>(smem);  // [2d] gate feature [k_pre ; RoPE(k_pre)] (fp64)
    double* terms = xs + 2 * d;                    // [hidden]
    float* kpost = reinterpret_cast<float*>(terms + ga.hidden);  // [d] RoPE'd key (fp32) for the cache
    __shared__ int vpage, vslot, gpage, gslot, npage, nslot, event;
    __shared__ HeadState nst;
    const size_t in = ((size_t)s * pv.kv_heads + h) * d;
    const int blk = layer * pv.kv_heads + h;
    E* pool = reinterpret_cast<E*>(pv.data);

    // ---- phase A: inputs, state, speculative victim fetch, RoPE, feature ----
    // (the new token's inputs do not depend on the cache state: loads first;
    // every thread reads the state and the ring page under local_ptr itself, so
    // the victim's K/V is fetched in the same round as its admission bit)
    const bool kt = tid < d / 2, et = tid < d;
    const float x0 = kt ? to_f(k_pre[in + 2 * tid]) : 0.f, x1 = kt ? to_f(k_pre[in + 2 * tid + 1]) : 0.f;
    const E vnew = et ? v[in + tid] : E();
    HeadState st = pv.state[hidx];
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
    if (kt) {
        float c, sn;
        rope_cs(ga.freq, tid, pos, c, sn);  // the cached key: fp64 angle, fp32 rotation
        rope_pair_f32(x0, x1, c, sn, kpost[2 * tid], kpost[2 * tid + 1]);
        if (!forced_g) {  // the gate feature in the reference's arithmetic (numerics.cpp:53-62)
            const double a = x0, b = x1;
            const double angle = __dmul_rn((double)pos, ga.freq[tid]);
            const double cd = cos(angle), sd = sin(angle);
            xs[2 * tid] = a;
            xs[2 * tid + 1] = b;
            xs[d + 2 * tid] = __dsub_rn(__dmul_rn(a, cd), __dmul_rn(b, sd));
            xs[d + 2 * tid + 1] = __dadd_rn(__dmul_rn(a, sd), __dmul_rn(b, cd));
        }
    }
    __syncthreads();

    // ---- phase B: the gate's hidden units (threads 0-127) beside the routing
    // decision (thread 128): lazy promotion inspects the VICTIM's stored bit
    // (written W steps ago), never the new token's gate ----------------------
    if (!forced_g) gate_terms_ref(ga.gd(), blk, xs, d, terms, 0, 128);
    if (tid == 128) {
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
        event = ev;
        vpage = vp;
        vslot = slot % ps;
        gpage = gp;
        gslot = gs_;
        npage = lp;
        nslot = slot % ps;
        nst = ns;
    }
    __syncthreads();

    // ---- phase C: promote the victim (K/V fetched in phase A; gate, pos, bit),
    // write the new token into the ring slot, its gate, the state ------------
    if (event == 1 && et) {
        E* kd = pool + (size_t)gpage * pv.page_elems() + (size_t)gslot * d;
        kd[tid] = vk;
        kd[tid + (size_t)ps * d] = vv;
    }
    if (npage >= 0 && et) {
        E* kd = pool + (size_t)npage * pv.page_elems() + (size_t)nslot * d;
        kd[tid] = from_f<E>(kpost[tid]);
        kd[tid + (size_t)ps * d] = vnew;
    }
    if (tid == 0) {
        if (event == 1) {  // the victim's metadata, read before the new token overwrites the slot
            const size_t a = (size_t)vpage * ps + vslot, b = (size_t)gpage * ps + gslot;
            pv.gate[b] = pv.gate[a];
            pv.pos[b] = pv.pos[a];
            pv.adm[b] = pv.adm[a];
        }
        const double g = forced_g ? (double)forced_g[(size_t)s * pv.kv_heads + h] : gate_from_z2(gate_z2_ref(ga.gd(), blk, terms));
        const uint8_t bit = g >= ga.tau ? 1 : 0;
        if (npage >= 0) {
            const size_t b = (size_t)npage * ps + nslot;
            pv.gate[b] = (float)g;
            pv.adm[b] = bit;
            pv.pos[b] = (int32_t)pos;
        }
        if (event >= 0) pv.state[hidx] = nst;
        const size_t o = (size_t)s * pv.kv_heads + h;
        if (tr.g) tr.g[o] = (float)g;
        if (tr.bits) tr.bits[o] = bit;
        if (tr.near_tau) tr.near_tau[o] = fabs(g - ga.tau) < 1e-6 ? 1 : 0;
        if (tr.events) tr.events[o] = event;
    }
}

}  // namespace wgkv
