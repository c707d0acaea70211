// decode_finish.cu -- the second kernel of a decode layer with the deferred
// append (bf16 fast path, DecArgs::defer).
//
// Session::decode_step (engine.cpp:291-327) appends the new token
// (HeadCache::local_write, kvstore.cpp:135-158) and then attends Global ||
// Local (attn_ragged, attention.cpp:155-180).  On B200 the attention kernel
// (K5, decode_mma.cu) instead streams the cache as it was BEFORE the append --
// every Global page, the ring minus a dropped victim -- so nothing sits in
// front of it; this kernel then, in one launch:
//   * combine CTAs, one per (seq, q head): merge K5's chunk partials and the
//     new token itself (its logit from the RoPE'd q and k, value v), which is
//     exactly the reference's attended set after local_write;
//   * append CTAs: K4 (append.cuh) -- per (seq, kv head) a route CTA (lazy
//     promotion of the ring victim, the new token into the ring) and gate CTAs
//     (its exact fp64 gate) -- which may only start once K5 has read the
//     victim slot, i.e. now.
// Both roles run concurrently, so K4 costs no extra step on the layer's path.
#include "attn.cuh"
#include "timeline.cuh"

namespace wgkv {


__global__ void __launch_bounds__(kAppendThreads) decode_finish_kernel(DecArgs a, const __nv_bfloat16* __restrict__ q,
                                                                       const float* __restrict__ part,
                                                                       __nv_bfloat16* __restrict__ out, FinishArgs fin,
                                                                       int ncomb) {
    extern __shared__ __align__(16) uint8_t fsm[];
    TL_DECL
    TL_MARK(0);
    // the next kernel on the stream may launch now; it waits for our completion
    asm volatile("griddepcontrol.launch_dependents;");
    const int tid = threadIdx.x;
    // grid: [gate CTAs of the append, when not in the K5 launch][combine CTAs][route CTAs]
    const int gpp = (fin.forced_g || a.n_gate_ctas > 0 || fin.gate_side) ? 0 : gate_ctas_per_pair(fin.ga.hidden);
    const int ngate = a.n_pairs * gpp;
    const int arrivals = fin.forced_g ? 1 : gate_ctas_per_pair(fin.ga.hidden) + 1;
    if ((int)blockIdx.x < ngate) {
        // gate CTAs first: they need nothing K5 produces (see append_gate_part),
        // so they run in the slots K5's tail frees, without the PDL wait
        const int pr = blockIdx.x / gpp, j = blockIdx.x % gpp;
        const int s = pr / a.pv.kv_heads, h = pr % a.pv.kv_heads;
        append_gate_part<__nv_bfloat16>(a.pv, fin.ga, a.layer, a.seq0, s, h, j, fin.k_new, fin.wk, fsm);
        append_arrive(a.pv, fin.ga, a.layer, a.seq0, s, h, fin.forced_g, fin.tr, fin.wk, arrivals, fsm);
        TL_COMMIT(3, a.layer, 0);
        return;
    }
    if (fin.px.do_unpack && blockIdx.x == gridDim.x - 1) {  // ---- C1: the previous layer's peer exchange
        peer_unpack_cta(fin.px);
        return;
    }
    if ((int)blockIdx.x >= ngate + ncomb) {  // ---- route CTAs of the append (K4, append.cuh)
        // reads and routing run while K5 streams; the ring-slot stores wait for it
        append_role<__nv_bfloat16>(a.pv, fin.ga, a.layer, a.seq0, a.window, a.n_pairs, blockIdx.x - ngate - ncomb,
                                   0, arrivals, fin.k_new, fin.v_new, fin.forced_g, fin.tr, fin.wk, fsm, true);
        TL_COMMIT(4, a.layer, 0);
        return;
    }
    // ---- combine role: one (seq, q head) --------------------------------------
    constexpr int NW = kAppendThreads / 32;
    constexpr int d = 128;
    const int gs = a.q_heads / a.pv.kv_heads;
    const int sp = blockIdx.x - ngate, s = sp / a.q_heads, p = sp % a.q_heads, h = p / gs, g = p % gs;
    const int bh = s * a.pv.kv_heads + h;
    const int lane = tid & 31, warp = tid >> 5;
    const size_t pstride = (size_t)gs * (d + 2);
    const float* base = part + (size_t)bh * a.max_chunks * pstride + (size_t)g * (d + 2);
    float* wm = reinterpret_cast<float*>(fsm);  // [NW]
    float* wl = wm + NW;                         // [NW]
    float* wacc = wl + NW;                       // [NW][d]
    // K5 has finished: partials written
    asm volatile("griddepcontrol.wait;" ::: "memory");
    TL_MARK(2);
    if (sp == 0 && tid == 0) *a.counter = 0;  // K5's work counter, for the next launch
    // one round of loads: the chunk count, the rows of this warp's first three
    // chunks (speculatively: the partial buffer holds max_chunks of them), and
    // in the last warp the new token's q / k / v and position
    constexpr int SPEC = 3;
    float mcs[SPEC], lcs[SPEC];
    float2 xs[SPEC][2];
#pragma unroll
    for (int j = 0; j < SPEC; ++j) {
        const int c = min(warp + j * NW, a.max_chunks - 1);
        const float* rr = base + (size_t)c * pstride;
        mcs[j] = rr[d];
        lcs[j] = rr[d + 1];
#pragma unroll
        for (int i = 0; i < 2; ++i) xs[j][i] = *reinterpret_cast<const float2*>(rr + 2 * lane + 64 * i);
    }
    const size_t qo = ((size_t)s * a.q_heads + p) * d, ko = ((size_t)s * a.pv.kv_heads + h) * d;
    __nv_bfloat162 qv[2], kv[2], vv[2];
    long pos = 0;
    if (warp == NW - 1) {
        pos = a.tokpos[bh];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int i = lane + 32 * j;  // pair index (d / 2 = 64 pairs)
            qv[j] = reinterpret_cast<const __nv_bfloat162*>(q + qo)[i];
            kv[j] = reinterpret_cast<const __nv_bfloat162*>(fin.k_new + ko)[i];
            vv[j] = *reinterpret_cast<const __nv_bfloat162*>(fin.v_new + ko + 2 * lane + 64 * j);
        }
    }
    const int nch = min(a.nchunks[bh], kMaxChunks);
    float m = -INFINITY, l = 0.f;
    float2 acc[2];  // columns 2*lane + 64*j
    acc[0] = acc[1] = make_float2(0.f, 0.f);
    auto merge = [&](float mc, float lc, const float2 (&x)[2]) {
        const float mn = fmaxf(m, mc);
        const float sa = m == -INFINITY ? 0.f : __expf(m - mn), sb = __expf(mc - mn);
        l = l * sa + lc * sb;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            acc[j].x = acc[j].x * sa + x[j].x * sb;
            acc[j].y = acc[j].y * sa + x[j].y * sb;
        }
        m = mn;
    };
    // each warp merges every NW-th chunk online (m = -inf: an empty chunk)
#pragma unroll
    for (int j = 0; j < SPEC; ++j)
        if (warp + j * NW < nch && mcs[j] != -INFINITY) merge(mcs[j], lcs[j], xs[j]);
#pragma unroll 1
    for (int c = warp + SPEC * NW; c < nch; c += NW) {
        const float* rr = base + (size_t)c * pstride;
        const float mc = rr[d], lc = rr[d + 1];
        float2 x[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) x[j] = *reinterpret_cast<const float2*>(rr + 2 * lane + 64 * j);
        if (mc == -INFINITY) continue;  // empty chunk (uniform across the warp)
        merge(mc, lc, x);
    }
    if (warp == NW - 1) {
        // the new token at its position: logit = RoPE(q) . bf16(RoPE(k)) / sqrt(d)
        // (the key as it will be cached), weight on v.  (tokpos comes from K5:
        // the head state may already hold the next position once this kernel's
        // append has finalised.)
        float dotp = 0.f;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int i = lane + 32 * j;
            float c, sn;
            rope_cs(a.freq, i, pos, c, sn);
            float q0, q1, k0, k1;
            const float2 qf = __bfloat1622float2(qv[j]), kf = __bfloat1622float2(kv[j]);
            rope_pair_f32(qf.x, qf.y, c, sn, q0, q1);
            rope_pair_f32(kf.x, kf.y, c, sn, k0, k1);
            k0 = __bfloat162float(__float2bfloat16_rn(k0));
            k1 = __bfloat162float(__float2bfloat16_rn(k1));
            dotp = fmaf(q0, k0, fmaf(q1, k1, dotp));
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) dotp += __shfl_xor_sync(0xffffffffu, dotp, o);
        float2 x[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) x[j] = __bfloat1622float2(vv[j]);
        merge(dotp * rsqrtf((float)d), 1.f, x);
    }
    if (lane == 0) {
        wm[warp] = m;
        wl[warp] = l;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        wacc[warp * d + 2 * lane + 64 * j] = acc[j].x;
        wacc[warp * d + 2 * lane + 64 * j + 1] = acc[j].y;
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
            t += f * wacc[w * d + e];
            L += f * wl[w];
        }
        out[((size_t)s * a.q_heads + p) * d + e] = __float2bfloat16_rn(t / L);
    }
    if (fin.px.do_push) {  // C1: this row into every rank's exchange slot (LL words)
        __syncthreads();   // the row's stores above, by the other threads
        const uint32_t flag = peer_push_flag(fin.px);
        const uint32_t* row = reinterpret_cast<const uint32_t*>(out + ((size_t)s * a.q_heads + p) * d);
        for (int j = tid; j < d / 2; j += blockDim.x) peer_push_word(fin.px, flag, s, (p * d) / 2 + j, row[j]);
    }
    TL_COMMIT(1, a.layer, nch);
}

int launch_decode_finish(const DecArgs& a, int nseq, const __nv_bfloat16* q, const float* part, __nv_bfloat16* out,
                         const FinishArgs& fin, cudaStream_t st) {
    if (a.pv.head_dim != 128 || !a.tokpos || !a.counter || !a.nchunks) return WGKV_ENOTSUP;
    const int ncomb = nseq * a.q_heads;
    // route CTAs, plus the gate CTAs unless K5 ran them (a.n_gate_ctas > 0)
    const int napp = nseq * a.pv.kv_heads *
                     (1 + ((fin.forced_g || a.n_gate_ctas > 0 || fin.gate_side) ? 0 : gate_ctas_per_pair(fin.ga.hidden)));
    const size_t smem = std::max(append_smem_bytes(a.pv.head_dim, fin.ga.hidden),
                                 sizeof(float) * (2 * (kAppendThreads / 32) + (kAppendThreads / 32) * 128));
    if (ensure_smem(decode_finish_kernel, smem) != cudaSuccess) return WGKV_ECUDA;
    // programmatic dependent of K5: the launch overlaps K5's tail
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncomb + napp + (fin.px.do_unpack ? 1 : 0));
    cfg.blockDim = dim3(kAppendThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, decode_finish_kernel, a, q, part, out, fin, ncomb);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

}  // namespace wgkv

TL_EXPORT(wgkv_tl_fin)
