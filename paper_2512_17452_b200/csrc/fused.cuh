// fused.cuh -- one deferred decode layer in ONE launch (small batches).
//
// Session::decode_step (engine.cpp:291-327) for few (seq, kv head) pairs is
// latency-bound: with K5 (attention over the pre-append cache) followed by a
// finish kernel (chunk merge + the new token + the append), every layer pays
// two kernel drains and the append's chain of dependent round trips after the
// attention.  Here the K5 launch carries every role of the layer:
//   * route CTAs (one per pair): the routing decision, page pops, page-table
//     and metadata writes and the promoted victim's copy into Global -- all of
//     it before the PDL wait when the predecessor is another layer's decode
//     (nothing of this layer is in flight), since the attention of this layer
//     reads none of it (new pages lie past the attended ones, a promoted victim
//     lands past the tail page's valid rows);
//   * gate CTAs (ceil(hidden/16) per pair, append.cuh): the exact fp64 gate;
//     the last one of a pair sums z2 in the reference's order;
//   * K5 CTAs: the attention items; the last item of a pair merges the pair's
//     chunk partials with the new token (logit RoPE(q) . bf16(RoPE(k_new)),
//     weight on v_new) and writes the output.
// Two commits per pair, each by the last of its two parties: the new token's
// K/V into its ring slot (route + merge: every item of the pair, hence every
// read of the victim's slot, is done; with forced gates also its gate), and
// its gate and bit with the GateTrace's g (route + gate group), so neither the
// attention nor the gate waits for the other.  The new
// head state is published only once every K5 CTA has planned from the old one
// (a two-party handshake per pair: the commit and the last CTA to plan).
// Scratch lives in FusedWork and in AppendWork's next / event / slot (route
// outputs), parity-split where a CTA may touch it before the PDL wait.
#pragma once
#include "append.cuh"

namespace wgkv {

// Per (seq, kv head) pair [S*H].  Whatever a CTA may touch before the PDL wait
// (route outputs, the party counter, the publication handshake, the planner
// count) is passed as this layer's half of a [2][...] buffer chosen by layer
// parity (the previous layer's launch may still be using the other half);
// the rest is only touched after the wait.
struct FusedWork {
    int* cnt_items;  // K5 items of the pair done; the last one merges
    int* cnt_kv;     // [parity] route + merge arrivals; the last one stores the new K / V
    int* cnt_gw;     // [parity] route + gate group arrivals; the last one writes the gate
    int* cnt_gate;   // gate CTAs done; the last one sums z2
    int* pub;        // [parity] publication handshake (K/V commit, every K5 CTA planned)
    int* started;    // [parity] K5 CTAs that have planned (one int)
    double* g;       // the new token's gate (fp64), from the gate group
};

// arrive as one of two parties on cnt (thread-level, lane 0 of the arriving
// warp; the caller has ordered its writes before with a barrier): an acquire
// read first -- the other party is usually done, and then no atomic round trip
// is needed -- else the atomic.  True in the last one, which resets cnt.
__device__ __forceinline__ bool pair_arrive(int* cnt);

// whole CTA: arrive on a counter; true in every thread of the CTA that arrived
// last (which resets the counter).  Release / acquire: threadfence around the
// atomic, bar.sync to the rest of the CTA.
__device__ __forceinline__ bool cta_arrive(int* cnt, int target) {
    __shared__ int s_last;
    __syncthreads();  // the CTA's writes are ordered before thread 0's release fence
    if (threadIdx.x == 0) {
        __threadfence();
        const int last = atomicAdd(cnt, 1) == target - 1;
        if (last) {
            *cnt = 0;
            __threadfence();
        }
        s_last = last;
    }
    __syncthreads();
    return s_last != 0;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ bool pair_arrive(int* cnt) {
    bool last = ld_acquire(cnt) == 1;
    if (!last) {
        __threadfence();
        last = atomicAdd(cnt, 1) == 1;
        if (last) __threadfence();
    }
    if (last) *cnt = 0;
    return last;
}

// the last planner's side of the publication handshake of pair pairg
// (thread-level); the second arrival writes the new head state
__device__ __forceinline__ void fused_pub(const PoolView& pv, const AppendWork& wk, const FusedWork& fw, int layer,
                                          int pairg) {
    if (atomicAdd(&fw.pub[pairg], 1) == 1) {
        __threadfence();
        fw.pub[pairg] = 0;
        const int ev = __ldcg(&wk.event[pairg]);
        if (ev >= 0) {
            const HeadState* nx = wk.next + pairg;
            HeadState ns;
            ns.local_len = __ldcg(&nx->local_len);
            ns.local_ptr = __ldcg(&nx->local_ptr);
            ns.global_len = __ldcg(&nx->global_len);
            ns.tokens_seen = __ldcg(&nx->tokens_seen);
            pv.state[pv.head_index(layer, pairg / pv.kv_heads, pairg % pv.kv_heads)] = ns;
        }
    }
}

// the committer's side, with the route outputs in hand; pub_seen = pub[pairg]
// as loaded after the party acquire: 1 = the last planner has arrived (it
// touches pub[pairg] once), so no atomic round trip is needed
__device__ __forceinline__ void fused_pub_commit(const PoolView& pv, const FusedWork& fw, int layer, int pairg,
                                                 int pub_seen, int ev, const HeadState& ns) {
    if (pub_seen == 1 || atomicAdd(&fw.pub[pairg], 1) == 1) {
        fw.pub[pairg] = 0;
        if (ev >= 0) pv.state[pv.head_index(layer, pairg / pv.kv_heads, pairg % pv.kv_heads)] = ns;
    }
}

// route CTA of pair (s, h); wait: pass griddepcontrol.wait first (the
// predecessor may own this layer's state)
template <typename E>
__device__ __forceinline__ void fused_route(const PoolView& pv, int layer, int seq0, int s, int h, long W,
                                            const AppendWork& wk, const FusedWork& fw, bool wait) {
    if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    const int tid = threadIdx.x, d = pv.head_dim, ps = pv.page_size;
    const long hidx = pv.head_index(layer, seq0 + s, h);
    const int pairg = (seq0 + s) * pv.kv_heads + h;
    __shared__ int s_ev, s_gpage, s_gslot;
    E* pool = reinterpret_cast<E*>(pv.data);
    const bool et = tid < d;
    const HeadState st = pv.state[hidx];
    const int slot = st.local_ptr;
    const int lp0 = pv.lpt[hidx * pv.n_lp + slot / ps];
    E vk = E(), vv = E();
    if (st.local_len >= W && lp0 >= 0 && et) {  // the victim's K/V, fetched with its bit
        const E* ks = pool + (size_t)lp0 * pv.page_elems() + (size_t)(slot % ps) * d;
        vk = ks[tid];
        vv = ks[tid + (size_t)ps * d];
    }
    if (tid == 0) {
        const RouteDecision r = route_decide(pv, hidx, st, W, lp0);
        s_ev = r.ev;
        s_gpage = r.gpage;
        s_gslot = r.gslot;
        wk.next[pairg] = r.ns;
        wk.event[pairg] = r.ev;
        wk.slot[pairg] = r.npage >= 0 ? r.npage * ps + r.nslot : -1;
    }
    __syncthreads();
    if (s_ev == 1 && et) {  // promote: the victim's K/V into its Global slot
        E* kd = pool + (size_t)s_gpage * pv.page_elems() + (size_t)s_gslot * d;
        kd[tid] = vk;
        kd[tid + (size_t)ps * d] = vv;
    }
}

// the last gate CTA of a pair: z2 = b2 + the terms in order (gating.cpp:
// 162-166) -> g into fw.g.  Whole CTA; true in the last one.  smem: >= hidden
// doubles (the gate part's staging, free by now).
__device__ __forceinline__ bool fused_gate_arrive(const PoolView& pv, const GateArgs& ga, int layer, int pairg,
                                                  int h, const AppendWork& wk, const FusedWork& fw, uint8_t* smem) {
    if (!cta_arrive(&fw.cnt_gate[pairg], gate_ctas_per_pair(ga.hidden))) return false;
    double* terms = reinterpret_cast<double*>(smem);
    for (int u = threadIdx.x; u < ga.hidden; u += blockDim.x) terms[u] = __ldcg(wk.terms + (size_t)pairg * ga.hidden + u);
    __syncthreads();
    if (threadIdx.x == 0) {
        double z2 = ga.b2d[layer * pv.kv_heads + h];
        for (int u = 0; u < ga.hidden; ++u) z2 = __dadd_rn(z2, terms[u]);
        fw.g[pairg] = gate_from_z2(z2);
    }
    return true;
}

// the K/V commit of pair (s, h), by ONE warp of the last of route + merge:
// the new token's K / V into its ring slot (kn / vn: the key as cached and the
// value, in shared memory, or null: formed here from k_new / v_new), the
// promotion event, with forced gates the gate, bit and GateTrace too, and this
// side of the publication handshake
template <typename E>
__device__ __forceinline__ void fused_commit_kv(const PoolView& pv, const GateArgs& ga, int layer, int seq0, int s,
                                                int h, const E* __restrict__ k_new, const E* __restrict__ v_new,
                                                const float* __restrict__ forced_g, const DecodeTrace& tr,
                                                const AppendWork& wk, const FusedWork& fw, const float* kn,
                                                const float* vn) {
    const int lane = threadIdx.x & 31, d = pv.head_dim, ps = pv.page_size;
    const int pairg = (seq0 + s) * pv.kv_heads + h;
    const size_t o = (size_t)s * pv.kv_heads + h;
    int sl = 0, ev = 0, pub = 0;  // one round of loads (after the arrival's acquire)
    HeadState ns{};
    if (lane == 0) {
        sl = __ldcg(&wk.slot[pairg]);
        ev = __ldcg(&wk.event[pairg]);
        ns.local_len = __ldcg(&wk.next[pairg].local_len);
        ns.local_ptr = __ldcg(&wk.next[pairg].local_ptr);
        ns.global_len = __ldcg(&wk.next[pairg].global_len);
        ns.tokens_seen = __ldcg(&wk.next[pairg].tokens_seen);
        pub = __ldcg(&fw.pub[pairg]);
    }
    sl = __shfl_sync(0xffffffffu, sl, 0);
    const int pos = __shfl_sync(0xffffffffu, ns.tokens_seen, 0) - 1;  // valid when sl >= 0
    if (sl >= 0) {
        E* kd = reinterpret_cast<E*>(pv.data) + (size_t)(sl / ps) * pv.page_elems() + (size_t)(sl % ps) * d;
#pragma unroll 1
        for (int i = lane; i < d / 2; i += 32) {
            float y0, y1;
            if (kn) {
                y0 = kn[2 * i];
                y1 = kn[2 * i + 1];
            } else {  // the cached key: fp64 angle, fp32 rotation (as K1 / K4)
                float c, sn;
                rope_cs(ga.freq, i, pos, c, sn);
                rope_pair_f32(to_f(k_new[o * d + 2 * i]), to_f(k_new[o * d + 2 * i + 1]), c, sn, y0, y1);
            }
            kd[2 * i] = from_f<E>(y0);
            kd[2 * i + 1] = from_f<E>(y1);
        }
#pragma unroll 1
        for (int i = lane; i < d; i += 32) kd[i + (size_t)ps * d] = vn ? from_f<E>(vn[i]) : v_new[o * d + i];
    }
    if (lane == 0) {
        if (tr.events) tr.events[o] = ev;
        if (forced_g) {
            const double g = (double)forced_g[o];
            const uint8_t bit = g >= ga.tau ? 1 : 0;
            if (sl >= 0) {
                pv.gate[sl] = (float)g;
                pv.adm[sl] = bit;
            }
            if (tr.g) tr.g[o] = (float)g;
            if (tr.bits) tr.bits[o] = bit;
            if (tr.near_tau) tr.near_tau[o] = fabs(g - ga.tau) < 1e-6 ? 1 : 0;
        }
        fused_pub_commit(pv, fw, layer, pairg, pub, ev, ns);
    }
}

// the gate commit of pair (s, h), thread-level, by the last of route + gate
// group: the new token's gate and bit into its slot, the GateTrace's g / bits /
// near-tau flag
__device__ __forceinline__ void fused_commit_gate(const PoolView& pv, const GateArgs& ga, int seq0, int s, int h,
                                                  const DecodeTrace& tr, const AppendWork& wk, const FusedWork& fw) {
    const int pairg = (seq0 + s) * pv.kv_heads + h;
    const size_t o = (size_t)s * pv.kv_heads + h;
    const int sl = __ldcg(&wk.slot[pairg]);
    const double g = __ldcg(&fw.g[pairg]);
    const uint8_t bit = g >= ga.tau ? 1 : 0;
    if (sl >= 0) {
        pv.gate[sl] = (float)g;
        pv.adm[sl] = bit;
    }
    if (tr.g) tr.g[o] = (float)g;
    if (tr.bits) tr.bits[o] = bit;
    if (tr.near_tau) tr.near_tau[o] = fabs(g - ga.tau) < 1e-6 ? 1 : 0;
}

}  // namespace wgkv
