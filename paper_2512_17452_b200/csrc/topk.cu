// topk.cu -- K6: select_topk_pages (engine.cpp:36-84) + attention over the
// selected Global pages and the Local ring, per q head (wgkv_plus_topk,
// engine.cpp:320-324; BASELINE configs[4]).
//
//   topk_score_kernel   page score = max over the page's slots of the UNSCALED
//                       q.k (q RoPE'd at the decode position), per q head; one
//                       warp per page serves the whole GQA group (each K byte
//                       read once per group).
//   topk_select_kernel  exact top-min(budget, pages) per q head: 8-pass radix
//                       select on 64-bit keys (orderable(score) << 32 | ~page),
//                       i.e. higher score first and ties to the OLDER page,
//                       exactly std::stable_sort + the reference comparator;
//                       the selection is emitted in ascending logical order.
//   topk_attn_kernel    split-KV online-softmax attention of one q head over
//                       its selected pages then the Local pages; chunk partials
//                       are merged by decode_combine_kernel.
#include <algorithm>

#include "attn.cuh"

namespace wgkv {

namespace {
constexpr int TK_PPB = 32;  // pages per score CTA (4 warps x 8)
__device__ __forceinline__ uint32_t orderable(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
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

// one 1024-thread CTA per (seq, q head)
__global__ void __launch_bounds__(1024) topk_select_kernel(DecArgs a, long budget, const float* __restrict__ scores,
                                                           int32_t* __restrict__ sel, int32_t* __restrict__ nsel) {
    const int sp = blockIdx.x, s = sp / a.q_heads, p = sp % a.q_heads;
    const int h = p / (a.q_heads / a.pv.kv_heads), ps = a.pv.page_size;
    const HeadState st = a.pv.state[a.pv.head_index(a.layer, a.seq0 + s, h)];
    const int n = (st.global_len + ps - 1) / ps;
    const float* sc = scores + (size_t)sp * a.pv.n_gp;
    int32_t* out = sel + (size_t)sp * a.pv.n_gp;
    const int k = (int)min((long)n, budget);
    const int tid = threadIdx.x;
    __shared__ unsigned hist[256];
    __shared__ unsigned long long prefix_s;
    __shared__ int remain_s;
    __shared__ int wsum[32];
    __shared__ int carry;
    unsigned long long thr = 0;  // keys >= thr are selected
    if (k < n) {
        unsigned long long prefix = 0, mask = 0;
        int remain = k;
        for (int byte = 7; byte >= 0; --byte) {
            for (int b = tid; b < 256; b += blockDim.x) hist[b] = 0;
            __syncthreads();
            for (int lp = tid; lp < n; lp += blockDim.x) {
                const unsigned long long key =
                    ((unsigned long long)orderable(sc[lp]) << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)lp);
                if ((key & mask) == prefix) atomicAdd(&hist[(key >> (8 * byte)) & 255], 1u);
            }
            __syncthreads();
            if (tid == 0) {
                int acc = 0, b = 255;
                for (; b >= 0; --b) {
                    if (acc + (int)hist[b] >= remain) break;
                    acc += hist[b];
                }
                prefix_s = prefix | ((unsigned long long)b << (8 * byte));
                remain_s = remain - acc;
            }
            __syncthreads();
            prefix = prefix_s;
            remain = remain_s;
            mask |= 255ull << (8 * byte);
        }
        thr = prefix;  // the k-th largest key (keys are unique)
    }
    // emit selected logical pages in ascending order (block scan over lp)
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += blockDim.x) {
        const int lp = base + tid;
        bool take = false;
        if (lp < n) {
            if (k == n) {
                take = true;
            } else {
                const unsigned long long key =
                    ((unsigned long long)orderable(sc[lp]) << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)lp);
                take = key >= thr;
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if ((tid & 31) == 0) wsum[tid >> 5] = __popc(bal);
        __syncthreads();
        int before = carry;
        for (int w = 0; w < (tid >> 5); ++w) before += wsum[w];
        if (take) out[before + __popc(bal & ((1u << (tid & 31)) - 1u))] = lp;
        __syncthreads();
        if (tid == 0) {
            int t = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wsum[w];
            carry += t;
        }
        __syncthreads();
    }
    if (tid == 0) nsel[sp] = carry;
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
    const int nc = d / 32;
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
                    if (c < nc) o[c] = fmaf(pjj, to_f(vb[(size_t)(j0 + jj) * d + lane + 32 * c]), o[c]);
            }
        }
    }
    float* rw = red + (size_t)warp * (d + 2);
#pragma unroll
    for (int c = 0; c < 8; ++c)
        if (c < nc) rw[lane + 32 * c] = o[c];
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

template <typename E>
int launch_topk_decode(const DecArgs& a0, int nseq, long budget, const E* q, float* scores, int32_t* sel,
                       int32_t* nsel, float* part, E* out, cudaStream_t st) {
    DecArgs a = a0;
    const int d = a.pv.head_dim, gs = a.q_heads / a.pv.kv_heads;
    if (d % 32 != 0 || d > 256) return WGKV_ENOTSUP;
    const int max_pages = a.pv.n_gp;
    topk_score_kernel<E><<<dim3((max_pages + TK_PPB - 1) / TK_PPB, nseq * a.pv.kv_heads), 128,
                          sizeof(float) * gs * d, st>>>(a, q, scores);
    topk_select_kernel<<<nseq * a.q_heads, 1024, 0, st>>>(a, budget, scores, sel, nsel);
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

template int launch_topk_decode<float>(const DecArgs&, int, long, const float*, float*, int32_t*, int32_t*, float*,
                                       float*, cudaStream_t);
template int launch_topk_decode<__nv_bfloat16>(const DecArgs&, int, long, const __nv_bfloat16*, float*, int32_t*,
                                               int32_t*, float*, __nv_bfloat16*, cudaStream_t);

}  // namespace wgkv
