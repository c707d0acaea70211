// admit.cu -- K2 (prefill admission/compaction) and K4 (decode append with
// lazy promotion) over the device-resident paged dual cache.
//
// K2 replaces HeadCache::prefill_populate (kvstore.cpp:160-203):
//   admit_plan_kernel    one CTA per (seq, kv head): counts admitted tokens
//                        j < T-W per 128-token chunk, block-scans the counts,
//                        claims ceil(G/ps) Global + ceil(min(T,W)/ps) Local
//                        pages from the device free stack in one atomic, and
//                        writes the page tables and ring state.
//   admit_scatter_kernel one warp per 32 tokens: ballot/popc rank inside the
//                        chunk + the scanned chunk base gives each admitted
//                        row its Global slot (ascending order, exactly the
//                        reference's append order); window rows go to ring
//                        slots 0..; each row's K and V move with 128-bit
//                        loads/stores, gate/position/bit ride along.
// K4 replaces HeadCache::local_write + promote (kvstore.cpp:122-158) fused
// with the decode-time gate (gate_forward, gating.cpp:158-171) and RoPE.
#include "admit.cuh"
#include "append.cuh"
#include "gate.cuh"

namespace wgkv {

constexpr int ADM_CHUNK = 128;

__global__ void __launch_bounds__(1024) admit_plan_kernel(PoolView pv, int layer, int seq0, long T, long W,
                                                          const uint8_t* __restrict__ bits, int32_t* __restrict__ chunk_off) {
    const int s = blockIdx.x, h = blockIdx.y;
    const int tid = threadIdx.x;
    const long ws = T > W ? T - W : 0;  // window_start (kvstore.cpp:169)
    const long nchunk = (T + ADM_CHUNK - 1) / ADM_CHUNK;
    const uint8_t* b = bits + ((size_t)s * pv.kv_heads + h) * T;
    int32_t* co = chunk_off + ((size_t)s * pv.kv_heads + h) * (nchunk + 1);
    __shared__ int warp_tot[32];
    __shared__ int carry;
    __shared__ int page_base;
    if (tid == 0) carry = 0;
    __syncthreads();
    // exclusive scan of per-chunk admitted counts, 1024 chunks per pass
    for (long c0 = 0; c0 < nchunk; c0 += 1024) {
        const long c = c0 + tid;
        int cnt = 0;
        if (c < nchunk) {
            const long lo = c * ADM_CHUNK, hi = min((long)(c + 1) * ADM_CHUNK, ws);
            for (long j = lo; j < hi; j += 4) {
                if (j + 4 <= hi && ((((uintptr_t)(b + j)) & 3) == 0)) {
                    const uint32_t w = *reinterpret_cast<const uint32_t*>(b + j);
                    cnt += __popc(w & 0x01010101u);
                } else {
                    for (long jj = j; jj < min(j + 4, hi); ++jj) cnt += b[jj] != 0;
                }
            }
        }
        int x = cnt;
        const int lane = tid & 31, wid = tid >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int t = warp_tot[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            warp_tot[lane] = t;
        }
        __syncthreads();
        const int excl = carry + (wid ? warp_tot[wid - 1] : 0) + x - cnt;
        if (c < nchunk) co[c] = excl;
        __syncthreads();
        if (tid == 1023) carry = excl + cnt;
        __syncthreads();
    }
    const int G = carry;
    const long Lc = T - ws;  // min(T, W) ring entries
    const int ng = (G + pv.page_size - 1) / pv.page_size;
    const int nl = (int)((Lc + pv.page_size - 1) / pv.page_size);
    const long hidx = pv.head_index(layer, seq0 + s, h);
    if (tid == 0) {
        co[nchunk] = G;
        page_base = pool_claim(pv, ng + nl);
        // on a failed claim the head keeps no pages (the error is latched and
        // surfaces at the next wgkv_sync, like the reference's throw)
        HeadState st;
        st.local_len = page_base < 0 ? 0 : (int)Lc;
        st.local_ptr = page_base < 0 ? 0 : (int)(Lc % W);
        st.global_len = page_base < 0 ? 0 : G;
        st.tokens_seen = (int)T;
        pv.state[hidx] = st;
    }
    __syncthreads();
    if (page_base < 0) return;
    // LIFO pops in order: page i = stack[top - 1 - i] (KvPool::alloc_page)
    for (int i = tid; i < ng + nl; i += blockDim.x) {
        const int page = pv.free_stack[page_base - 1 - i];
        if (i < ng)
            pv.gpt[hidx * pv.n_gp + i] = page;
        else
            pv.lpt[hidx * pv.n_lp + (i - ng)] = page;
    }
}

template <typename E>
__device__ __forceinline__ void copy_row_warp(E* __restrict__ dst, const E* __restrict__ src, int d, int lane) {
    // 16-byte vectors; d*sizeof(E) is a multiple of 16 for d % 8 == 0
    const int nvec = d * (int)sizeof(E) / 16;
    if ((d * sizeof(E)) % 16 == 0) {
        const int4* s4 = reinterpret_cast<const int4*>(src);
        int4* d4 = reinterpret_cast<int4*>(dst);
        for (int e = lane; e < nvec; e += 32) d4[e] = s4[e];
    } else {
        for (int e = lane; e < d; e += 32) dst[e] = src[e];
    }
}

template <typename E>
__global__ void __launch_bounds__(128) admit_scatter_kernel(PoolView pv, int layer, int seq0, long T, long W,
                                                             const E* __restrict__ k_post, const E* __restrict__ v,
                                                             const float* __restrict__ g,
                                                             const uint8_t* __restrict__ bits,
                                                             const int32_t* __restrict__ chunk_off) {
    const int c = blockIdx.x, h = blockIdx.y, s = blockIdx.z;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long ws = T > W ? T - W : 0;
    const long nchunk = (T + ADM_CHUNK - 1) / ADM_CHUNK;
    const size_t bh = (size_t)s * pv.kv_heads + h;
    const long hidx = pv.head_index(layer, seq0 + s, h);
    const int d = pv.head_dim, ps = pv.page_size;
    const int G = chunk_off[bh * (nchunk + 1) + nchunk];
    // a failed page claim leaves global_len = 0 (admit_plan_kernel)
    if (G > 0 && pv.state[hidx].global_len != G) return;
    if (pv.state[hidx].tokens_seen != (int)T || (T > 0 && pv.state[hidx].local_len == 0)) return;

    __shared__ int wcnt[4];
    const long t = (long)c * ADM_CHUNK + wid * 32 + lane;
    const bool valid = t < T;
    const bool glob = valid && t < ws && bits[bh * T + t] != 0;
    const unsigned gm = __ballot_sync(0xffffffffu, glob);
    if (lane == 0) wcnt[wid] = __popc(gm);
    __syncthreads();
    int base = chunk_off[bh * (nchunk + 1) + c];
    for (int w = 0; w < wid; ++w) base += wcnt[w];
    const int rank = base + __popc(gm & ((1u << lane) - 1u));

    // per-lane destination (page, slot) or -1
    int dpage = -1, dslot = 0;
    if (glob) {
        dpage = pv.gpt[hidx * pv.n_gp + rank / ps];
        dslot = rank % ps;
    } else if (valid && t >= ws) {
        const long r = t - ws;  // ring slot (local_ptr starts at 0)
        dpage = pv.lpt[hidx * pv.n_lp + r / ps];
        dslot = (int)(r % ps);
    }
    if (dpage >= 0) {
        const size_t mi = (size_t)dpage * ps + dslot;
        pv.gate[mi] = g[bh * T + t];
        pv.pos[mi] = (int32_t)t;
        pv.adm[mi] = bits[bh * T + t];
    }
    unsigned mv = __ballot_sync(0xffffffffu, dpage >= 0);
    E* pool = reinterpret_cast<E*>(pv.data);
    if (d * sizeof(E) == 256) {
        // 256-byte rows (bf16, d = 128): a half warp moves one row with 16-byte
        // vectors, so a warp moves 2 rows per instruction; up to 8 rows' K and V
        // loads are issued before their stores (bytes in flight, not latency)
        const int hw = lane >> 4, hl = lane & 15;
        while (mv) {
            int4 kr[4], vr[4];
            int4* kd[4];
            bool on[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                // rows 2u and 2u+1 of this batch: the (2u + hw)-th remaining lane of mv
                unsigned m2 = mv;
                for (int k = 0; k < 2 * u + hw && m2; ++k) m2 &= m2 - 1;
                on[u] = m2 != 0;
                const int src = on[u] ? __ffs(m2) - 1 : 0;
                const int p = __shfl_sync(0xffffffffu, dpage, src);
                const int sl = __shfl_sync(0xffffffffu, dslot, src);
                const long ts = (long)c * ADM_CHUNK + wid * 32 + src;
                const size_t row = (((size_t)s * T + ts) * pv.kv_heads + h) * d;
                kd[u] = reinterpret_cast<int4*>(pool + (size_t)max(p, 0) * pv.page_elems() + (size_t)sl * d) + hl;
                if (on[u]) {
                    kr[u] = __ldg(reinterpret_cast<const int4*>(k_post + row) + hl);
                    vr[u] = __ldg(reinterpret_cast<const int4*>(v + row) + hl);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (on[u]) {
                    kd[u][0] = kr[u];
                    kd[u][(size_t)ps * d * sizeof(E) / 16] = vr[u];
                }
            for (int k = 0; k < 8 && mv; ++k) mv &= mv - 1;
        }
        return;
    }
    while (mv) {
        const int src = __ffs(mv) - 1;
        mv &= mv - 1;
        const int p = __shfl_sync(0xffffffffu, dpage, src);
        const int sl = __shfl_sync(0xffffffffu, dslot, src);
        const long ts = (long)c * ADM_CHUNK + wid * 32 + src;
        const size_t row = (((size_t)s * T + ts) * pv.kv_heads + h) * d;
        E* kdst = pool + (size_t)p * pv.page_elems() + (size_t)sl * d;
        copy_row_warp(kdst, k_post + row, d, lane);
        copy_row_warp(kdst + (size_t)ps * d, v + row, d, lane);
    }
}

template <typename E>
int launch_admit_prefill(const PoolView& pv, int layer, int seq0, int nseq, long T, long W, const E* k_post,
                         const E* v, const float* g, const uint8_t* bits, int32_t* chunk_off, cudaStream_t st) {
    admit_plan_kernel<<<dim3(nseq, pv.kv_heads), 1024, 0, st>>>(pv, layer, seq0, T, W, bits, chunk_off);
    const long nchunk = (T + ADM_CHUNK - 1) / ADM_CHUNK;
    admit_scatter_kernel<E><<<dim3((unsigned)nchunk, pv.kv_heads, nseq), 128, 0, st>>>(pv, layer, seq0, T, W, k_post,
                                                                                      v, g, bits, chunk_off);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

// ---------------------------------------------------------------------------
// K4 standalone: the split append's route + gate CTAs (append.cuh)
// ---------------------------------------------------------------------------
// mode 0: route + gate CTAs in one launch; 1: route CTAs only (the gate CTAs
// follow in a mode-2 launch on a side stream, overlapping the attention);
// 3: gate CTAs only, beside a deferred decode whose finish kernel routes
template <typename E>
__global__ void __launch_bounds__(kAppendThreads) decode_append_kernel(PoolView pv, GateArgs ga, int layer, int seq0,
                                                                        long W, int npairs,
                                                                        const E* __restrict__ k_pre,
                                                                        const E* __restrict__ v,
                                                                        const float* __restrict__ forced_g,
                                                                        DecodeTrace tr, AppendWork wk, int mode) {
    extern __shared__ __align__(16) uint8_t append_smem[];
    const int gpp = forced_g ? 0 : gate_ctas_per_pair(ga.hidden);
    const int r = mode >= 2 ? npairs + (int)blockIdx.x : (int)blockIdx.x;
    append_role<E>(pv, ga, layer, seq0, W, npairs, r, gpp, gpp + 1, k_pre, v, forced_g, tr, wk, append_smem);
}

template <typename E>
int launch_decode_append(const PoolView& pv, const GateArgs& ga, int layer, int seq0, int nseq, long W,
                         const E* k_pre, const E* v, const float* forced_g, const DecodeTrace& tr,
                         const AppendWork& wk0, cudaStream_t st, int mode) {
    const size_t smem = append_smem_bytes(pv.head_dim, ga.hidden);
    if (ensure_smem(decode_append_kernel<E>, smem) != cudaSuccess) return WGKV_ECUDA;
    const int npairs = nseq * pv.kv_heads;
    const int gpp = forced_g ? 0 : gate_ctas_per_pair(ga.hidden);
    AppendWork wk = wk0;
    wk.early_state = mode == 1 || mode == 2;
    const int grid = mode == 0 ? npairs * (1 + gpp) : (mode == 1 ? npairs : npairs * gpp);
    if (grid > 0)
        decode_append_kernel<E><<<grid, kAppendThreads, smem, st>>>(pv, ga, layer, seq0, W, npairs, k_pre, v, forced_g,
                                                                     tr, wk, mode);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

#define INST(E)                                                                                                   \
    template int launch_admit_prefill<E>(const PoolView&, int, int, int, long, long, const E*, const E*,          \
                                         const float*, const uint8_t*, int32_t*, cudaStream_t);                   \
    template int launch_decode_append<E>(const PoolView&, const GateArgs&, int, int, int, long, const E*, const E*, \
                                         const float*, const DecodeTrace&, const AppendWork&, cudaStream_t, int);
INST(float)
INST(__nv_bfloat16)
#undef INST

}  // namespace wgkv
