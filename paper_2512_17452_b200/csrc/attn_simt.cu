// attn_simt.cu -- fp32 SIMT attention kernels: the parity-mode (fp32 storage)
// path and the always-available cross-check for the tensor-core kernels.
//
//   vs_prefill_simt_kernel  K3 (attn_vertical_slash, attention.cpp:123-153):
//       per 32-row query tile, the admitted Global prefix (j < i0-W+1, read in
//       place from the pages K2 filled) then the band [i0-W+1, i0+31] of
//       k_post/v with allowed(i,j) = j<=i && (i-j<W || bit_j), online softmax.
//   decode_attn_simt_kernel K5 (gather + attn_ragged, kvstore.cpp:205-241,
//       attention.cpp:155-180): split-KV over the Global and Local pages in
//       place, one CTA per (seq, kv head, page chunk) serving the whole GQA
//       group, then decode_combine_kernel merges the chunk partials.
// Softmax is order-invariant (test_attention.cpp:375-396), so pages are
// visited in physical order.
#include "attn.cuh"

namespace wgkv {

constexpr int VS_QT = 32;  // query rows per CTA
constexpr int VS_KT = 32;  // keys per smem tile

// number of admitted tokens j < x (x <= T - W), from K2's chunk prefix counts
__device__ __forceinline__ int admitted_before(const int32_t* co, const uint8_t* b, long x) {
    if (x <= 0) return 0;
    const long c = x / 128;
    int n = co[c];
    for (long j = c * 128; j < x; ++j) n += b[j] != 0;
    return n;
}

template <typename E>
__global__ void __launch_bounds__(128) vs_prefill_simt_kernel(VsArgs a, const E* __restrict__ q,
                                                               const E* __restrict__ k_post, const E* __restrict__ v,
                                                               E* __restrict__ out) {
    extern __shared__ float sm[];
    const int d = a.pv.head_dim, dp = d + 1, ps = a.pv.page_size;
    float* Qs = sm;                 // [VS_QT][d]
    float* Ks = Qs + VS_QT * d;     // [VS_KT][d+1]
    float* Vs = Ks + VS_KT * dp;    // [VS_KT][d]
    float* Ps = Vs + VS_KT * d;     // [4 warps][32]
    __shared__ int kidx[VS_KT];     // key position (band) or -1

    const int p = blockIdx.y, s = blockIdx.z, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int h = p / (a.q_heads / a.pv.kv_heads);
    const long i0 = (long)blockIdx.x * VS_QT;
    const long T = a.T, W = a.W;
    const float scale = rsqrtf((float)d);
    const size_t bh = (size_t)s * a.pv.kv_heads + h;
    const long hidx = a.pv.head_index(a.layer, a.seq0 + s, h);
    const uint8_t* bits = a.bits + bh * T;
    const long nchunk = (T + 127) / 128;
    const int32_t* co = a.chunk_off + bh * (nchunk + 1);
    const E* pool = reinterpret_cast<const E*>(a.pv.data);

    // RoPE(q) rows i0..i0+31 at positions i (engine.cpp:229)
    for (int e = tid; e < VS_QT * (d / 2); e += blockDim.x) {
        const int r = e / (d / 2), i = e % (d / 2);
        const long t = i0 + r;
        float y0 = 0.f, y1 = 0.f;
        if (t < T) {
            const size_t off = (((size_t)s * T + t) * a.q_heads + p) * d + 2 * i;
            const float x0 = to_f(q[off]), x1 = to_f(q[off + 1]);
            float c, sn;
            rope_cs(a.freq, i, t, c, sn);
            y0 = x0 * c - x1 * sn;
            y1 = x0 * sn + x1 * c;
        }
        Qs[r * d + 2 * i] = y0;
        Qs[r * d + 2 * i + 1] = y1;
    }

    constexpr int RPW = VS_QT / 4;  // rows per warp
    constexpr int MAXC = 8;         // d <= 256
    float m[RPW], l[RPW], o[RPW][MAXC];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        m[r] = -INFINITY;
        l[r] = 0.f;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) o[r][c] = 0.f;
    }
    const int nc = (d + 31) / 32;  // column blocks of 32 (the last one partial when d % 32 != 0)

    const long s_lo = i0 - W + 1 > 0 ? i0 - W + 1 : 0;
    // vertical prefix length (clamped to what K2 stored: 0 after a failed page claim)
    const int C = min(admitted_before(co, bits, s_lo), a.pv.state[hidx].global_len);
    const long band_hi = min(i0 + VS_QT - 1, T - 1);
    const long n_band = band_hi - s_lo + 1;
    const long n_keys = C + n_band;
    __syncthreads();

    for (long k0 = 0; k0 < n_keys; k0 += VS_KT) {
        // ---- load a key tile: entries k0.. (vertical first, then band) ------
        if (tid < VS_KT) {
            const long kk = k0 + tid;
            kidx[tid] = kk < C ? -2 : (kk < n_keys ? (int)(s_lo + (kk - C)) : -1);
        }
        for (int e = tid; e < VS_KT * d; e += blockDim.x) {
            const int r = e / d, c = e % d;
            const long kk = k0 + r;
            float kv = 0.f, vv = 0.f;
            if (kk < C) {
                const int pg = a.pv.gpt[hidx * a.pv.n_gp + kk / ps];
                const E* base = pool + (size_t)pg * a.pv.page_elems() + (size_t)(kk % ps) * d;
                kv = to_f(base[c]);
                vv = to_f(base[(size_t)ps * d + c]);
            } else if (kk < n_keys) {
                const long j = s_lo + (kk - C);
                const size_t off = (((size_t)s * T + j) * a.pv.kv_heads + h) * d + c;
                kv = to_f(k_post[off]);
                vv = to_f(v[off]);
            }
            Ks[r * dp + c] = kv;
            Vs[r * d + c] = vv;
        }
        __syncthreads();
        const int key = kidx[lane];
        const bool key_bit = key >= 0 ? bits[key] != 0 : false;
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const int row = wid * RPW + r;
            const long i = i0 + row;
            if (i >= T) continue;  // warp-uniform
            bool ok;
            if (key == -2)
                ok = true;  // vertical: admitted and out of every row's window
            else if (key == -1)
                ok = false;
            else
                ok = key <= i && ((i - key) < W || key_bit);
            float sc = -INFINITY;
            if (ok) {
                float acc = 0.f;
                for (int c = 0; c < d; ++c) acc = fmaf(Qs[row * d + c], Ks[lane * dp + c], acc);
                sc = acc * scale;
            }
            float mx = sc;
            for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            const float mnew = fmaxf(m[r], mx);
            if (mnew == -INFINITY) continue;  // nothing permitted yet (warp-uniform)
            const float alpha = __expf(m[r] - mnew);
            const float pj = ok ? __expf(sc - mnew) : 0.f;
            float ps_ = pj;
            for (int off = 16; off >= 1; off >>= 1) ps_ += __shfl_xor_sync(0xffffffffu, ps_, off);
            l[r] = l[r] * alpha + ps_;
            m[r] = mnew;
            Ps[wid * 32 + lane] = pj;
            __syncwarp();
#pragma unroll
            for (int c = 0; c < MAXC; ++c)
                if (c < nc) o[r][c] *= alpha;
            for (int j = 0; j < VS_KT; ++j) {
                const float pjj = Ps[wid * 32 + j];
                if (pjj != 0.f) {
#pragma unroll
                    for (int c = 0; c < MAXC; ++c)
                        if (c < nc && lane + 32 * c < d) o[r][c] = fmaf(pjj, Vs[j * d + lane + 32 * c], o[r][c]);
                }
            }
            __syncwarp();
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        const long i = i0 + wid * RPW + r;
        if (i >= T) continue;
        const float inv = 1.f / l[r];
        const size_t off = (((size_t)s * T + i) * a.q_heads + p) * d;
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
            if (c < nc && lane + 32 * c < d) out[off + lane + 32 * c] = from_f<E>(o[r][c] * inv);
    }
}

template <typename E>
int launch_vs_prefill_simt(const VsArgs& a, int nseq, const E* q, const E* k_post, const E* v, E* out,
                           cudaStream_t st) {
    const int d = a.pv.head_dim;
    if (d % 2 != 0 || d > 256) return WGKV_ENOTSUP;
    const size_t smem = sizeof(float) * ((size_t)VS_QT * d + (size_t)VS_KT * (d + 1) + (size_t)VS_KT * d + 128);
    if (ensure_smem(vs_prefill_simt_kernel<E>, smem) != cudaSuccess) return WGKV_ECUDA;
    dim3 grid((unsigned)((a.T + VS_QT - 1) / VS_QT), a.q_heads, nseq);
    vs_prefill_simt_kernel<E><<<grid, 128, smem, st>>>(a, q, k_post, v, out);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

// ---------------------------------------------------------------------------
// K5 SIMT decode
// ---------------------------------------------------------------------------
constexpr int DC_MAXG = 8;  // GQA group size supported by the SIMT decode

template <typename E>
__global__ void __launch_bounds__(128) decode_attn_simt_kernel(DecArgs a, const E* __restrict__ q,
                                                                float* __restrict__ part) {
    extern __shared__ float dsm[];
    const int d = a.pv.head_dim, ps = a.pv.page_size;
    const int gs = a.q_heads / a.pv.kv_heads;
    const int bh = blockIdx.y, s = bh / a.pv.kv_heads, h = bh % a.pv.kv_heads;
    const int chunk = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long hidx = a.pv.head_index(a.layer, a.seq0 + s, h);
    const HeadState st = a.pv.state[hidx];
    const long pos = st.tokens_seen - 1;
    const int ng = (st.global_len + ps - 1) / ps;
    const int nl = (st.local_len + ps - 1) / ps;
    const int NP = ng + nl;
    const int vp0 = chunk * a.chunk_pages, vp1 = min(NP, vp0 + a.chunk_pages);
    float* Qs = dsm;                 // [gs][d]
    float* red = Qs + gs * d;        // [4][gs][d + 2]
    const float scale = rsqrtf((float)d);
    const size_t pstride = (size_t)gs * (d + 2);
    float* pout = part + ((size_t)bh * a.max_chunks + chunk) * pstride;
    if (vp0 >= vp1) {  // empty chunk
        for (int e = tid; e < gs; e += blockDim.x) {
            pout[e * (d + 2) + d] = -INFINITY;
            pout[e * (d + 2) + d + 1] = 0.f;
        }
        return;
    }
    for (int e = tid; e < gs * (d / 2); e += blockDim.x) {
        const int hh = e / (d / 2), i = e % (d / 2);
        const size_t off = ((size_t)s * a.q_heads + h * gs + hh) * d + 2 * i;
        const float x0 = to_f(q[off]), x1 = to_f(q[off + 1]);
        float c, sn;
        rope_cs(a.freq, i, pos, c, sn);
        Qs[hh * d + 2 * i] = x0 * c - x1 * sn;
        Qs[hh * d + 2 * i + 1] = x0 * sn + x1 * c;
    }
    __syncthreads();
    const E* pool = reinterpret_cast<const E*>(a.pv.data);
    const int nc = (d + 31) / 32;  // column blocks of 32 (the last one partial when d % 32 != 0)
    float m[DC_MAXG], l[DC_MAXG], o[DC_MAXG][8];
#pragma unroll
    for (int g = 0; g < DC_MAXG; ++g) {
        m[g] = -INFINITY;
        l[g] = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) o[g][c] = 0.f;
    }
    for (int vp = vp0 + wid; vp < vp1; vp += 4) {
        int page, valid;
        if (vp < ng) {
            page = a.pv.gpt[hidx * a.pv.n_gp + vp];
            valid = min(ps, st.global_len - vp * ps);
        } else {
            page = a.pv.lpt[hidx * a.pv.n_lp + (vp - ng)];
            valid = min(ps, st.local_len - (vp - ng) * ps);
        }
        if (page < 0) continue;  // failed allocation (latched ENOPAGES)
        const E* kb = pool + (size_t)page * a.pv.page_elems();
        const E* vb = kb + (size_t)ps * d;
        for (int j0 = 0; j0 < valid; j0 += 32) {
            const int j = j0 + lane;
            const bool ok = j < valid;
#pragma unroll
            for (int g = 0; g < DC_MAXG; ++g) {
                if (g >= gs) break;
                float sc = -INFINITY;
                if (ok) {
                    float acc = 0.f;
                    for (int c = 0; c < d; ++c) acc = fmaf(Qs[g * d + c], to_f(kb[(size_t)j * d + c]), acc);
                    sc = acc * scale;
                }
                float mx = sc;
                for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
                const float mnew = fmaxf(m[g], mx);
                const float alpha = __expf(m[g] - mnew);
                const float pj = ok ? __expf(sc - mnew) : 0.f;
                float sum = pj;
                for (int off = 16; off >= 1; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
                l[g] = l[g] * alpha + sum;
                m[g] = mnew;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c < nc) o[g][c] *= alpha;
                const int jn = min(32, valid - j0);
                for (int jj = 0; jj < jn; ++jj) {
                    const float pjj = __shfl_sync(0xffffffffu, pj, jj);
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        if (c < nc && lane + 32 * c < d) o[g][c] = fmaf(pjj, to_f(vb[(size_t)(j0 + jj) * d + lane + 32 * c]), o[g][c]);
                }
            }
        }
    }
    // merge the 4 warps
    float* rw = red + (size_t)wid * gs * (d + 2);
    for (int g = 0; g < gs && g < DC_MAXG; ++g) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (c < nc && lane + 32 * c < d) rw[g * (d + 2) + lane + 32 * c] = o[g][c];
        if (lane == 0) {
            rw[g * (d + 2) + d] = m[g];
            rw[g * (d + 2) + d + 1] = l[g];
        }
    }
    __syncthreads();
    for (int e = tid; e < gs * d; e += blockDim.x) {
        const int g = e / d, c = e % d;
        float M = -INFINITY;
        for (int w = 0; w < 4; ++w) M = fmaxf(M, red[(size_t)w * gs * (d + 2) + g * (d + 2) + d]);
        float acc = 0.f, L = 0.f;
        for (int w = 0; w < 4; ++w) {
            const float* r = red + (size_t)w * gs * (d + 2) + g * (d + 2);
            const float sc = r[d] == -INFINITY ? 0.f : __expf(r[d] - M);
            acc += sc * r[c];
            L += sc * r[d + 1];
        }
        pout[g * (d + 2) + c] = acc;
        if (c == 0) {
            pout[g * (d + 2) + d] = M;
            pout[g * (d + 2) + d + 1] = L;
        }
    }
}

// merge chunk partials of one (seq, q head): out = sum e^(m_c-M) o_c / sum e^(m_c-M) l_c.
// Latency-bound: each of the 8 warps merges every 8th chunk online (m, l and
// the row of a chunk are loaded together, the loads of successive chunks are
// independent), so the partials are read in one round of L2 accesses; the
// 8 warp results are merged through smem.
// NW warps per (seq, q head), each merging every NW-th chunk online; SPEC > 0:
// the rows of each warp's first SPEC chunks are loaded in the same round as
// the chunk count (speculatively: the partial buffer holds max_chunks of them)
template <typename E, int NW, int SPEC, int NJ>  // NJ: float2 columns per lane (d <= 64 * NJ)
__global__ void __launch_bounds__(NW * 32) decode_combine_kernel(DecArgs a, const float* __restrict__ part,
                                                                 E* __restrict__ out) {
    const int d = a.pv.head_dim, gs = a.q_heads / a.pv.kv_heads;
    const int sp = blockIdx.x, s = sp / a.q_heads, p = sp % a.q_heads, h = p / gs, g = p % gs;
    const int bh = s * a.pv.kv_heads + h;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t pstride = (size_t)gs * (d + 2);
    const float* base = part + (size_t)bh * a.max_chunks * pstride + (size_t)g * (d + 2);
    __shared__ float wm[NW], wl[NW];
    __shared__ float wacc[NW][64 * NJ];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // partials of the attention kernel (PDL)
    if (blockIdx.x == 0 && tid == 0 && a.counter) *a.counter = 0;  // K5's work counter, for the next launch
    float m = -INFINITY, l = 0.f;
    float2 acc[NJ];  // columns 2*lane + 64*j
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[j] = make_float2(0.f, 0.f);
    auto load = [&](int c, float& mc, float& lc, float2 (&x)[NJ]) {
        const float* r = base + (size_t)c * pstride;
        mc = r[d];
        lc = r[d + 1];
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            x[j] = 2 * lane + 64 * j < d ? *reinterpret_cast<const float2*>(r + 2 * lane + 64 * j) : make_float2(0.f, 0.f);
    };
    auto merge = [&](float mc, float lc, const float2 (&x)[NJ]) {
        if (mc == -INFINITY) return;  // empty chunk (uniform across the warp)
        const float mn = fmaxf(m, mc);
        const float sa = m == -INFINITY ? 0.f : __expf(m - mn), sb = __expf(mc - mn);
        l = l * sa + lc * sb;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            acc[j].x = acc[j].x * sa + x[j].x * sb;
            acc[j].y = acc[j].y * sa + x[j].y * sb;
        }
        m = mn;
    };
    float smc[SPEC > 0 ? SPEC : 1], slc[SPEC > 0 ? SPEC : 1];
    float2 sx[SPEC > 0 ? SPEC : 1][NJ];
#pragma unroll
    for (int j = 0; j < SPEC; ++j) load(min(warp + j * NW, a.max_chunks - 1), smc[j], slc[j], sx[j]);
    const int nch = min(a.nchunks ? a.nchunks[bh] : a.n_chunks, kMaxChunks);
#pragma unroll
    for (int j = 0; j < SPEC; ++j)
        if (warp + j * NW < nch) merge(smc[j], slc[j], sx[j]);
#pragma unroll 4
    for (int c = warp + SPEC * NW; c < nch; c += NW) {
        float mc, lc;
        float2 x[NJ];
        load(c, mc, lc, x);
        merge(mc, lc, x);
    }
    if (lane == 0) {
        wm[warp] = m;
        wl[warp] = l;
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j)
        if (2 * lane + 64 * j < d) {
            wacc[warp][2 * lane + 64 * j] = acc[j].x;
            wacc[warp][2 * lane + 64 * j + 1] = acc[j].y;
        }
    __syncthreads();
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, wm[w]);
    for (int e = tid; e < d; e += blockDim.x) {
        float t = 0.f, L = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float f = wm[w] == -INFINITY ? 0.f : __expf(wm[w] - M);
            t += f * wacc[w][e];
            L += f * wl[w];
        }
        out[((size_t)s * a.q_heads + p) * d + e] = from_f<E>(t / L);
    }
}

template <typename E>
int launch_decode_attn_simt(const DecArgs& a, int nseq, const E* q, float* part, E* out, cudaStream_t st) {
    const int d = a.pv.head_dim, gs = a.q_heads / a.pv.kv_heads;
    if (d % 2 != 0 || d > 256 || gs > DC_MAXG) return WGKV_ENOTSUP;
    const size_t smem = sizeof(float) * ((size_t)gs * d + (size_t)4 * gs * (d + 2));
    if (ensure_smem(decode_attn_simt_kernel<E>, smem) != cudaSuccess) return WGKV_ECUDA;
    decode_attn_simt_kernel<E><<<dim3(a.n_chunks, nseq * a.pv.kv_heads), 128, smem, st>>>(a, q, part);
    decode_combine_kernel<E, 8, 0, 4><<<nseq * a.q_heads, 256, 0, st>>>(a, part, out);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

int launch_decode_combine_bf16(const DecArgs& a, int nseq, const float* part, __nv_bfloat16* out, cudaStream_t st) {
    // programmatic dependent of the attention kernel: launch latency overlaps its tail
    cudaLaunchConfig_t cfg = {};
    // 16 warps, 10 chunks each in the first round of loads: one round of L2 reads
    // for up to 160 chunks (one kv head spread over every SM: ~150)
    constexpr int NW = 16;
    cfg.gridDim = dim3(nseq * a.q_heads);
    cfg.blockDim = dim3(NW * 32);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, decode_combine_kernel<__nv_bfloat16, NW, 10, 2>, a, part, out);  // d = 128
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

#define INST(E)                                                                                              \
    template int launch_vs_prefill_simt<E>(const VsArgs&, int, const E*, const E*, const E*, E*, cudaStream_t); \
    template int launch_decode_attn_simt<E>(const DecArgs&, int, const E*, float*, E*, cudaStream_t);
INST(float)
INST(__nv_bfloat16)
#undef INST

}  // namespace wgkv
