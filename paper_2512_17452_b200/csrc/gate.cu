// gate.cu -- K1: fused RoPE -> write-gate MLP -> sigmoid -> threshold.
//
// Replaces gate_forward_batch + build_gate_feature + binarize + apply_rope
// (gating.cpp:149-190, numerics.cpp:50-77).  Two stages:
//   gate_prefill_kernel : fp32 SIMT register-tiled GEMM [64 tok x 2d] . [2d x
//       128 hidden] per CTA with the GELU . w2 reduction, sigmoid and
//       threshold fused in the epilogue; writes k_post (RoPE'd keys, stored
//       once for the cache and the band of K3), g and bits, and lists every
//       token whose z2 lies within a conservative fp32 error band of
//       logit(tau).
//   gate_recheck_kernel : one warp per listed token recomputes the gate in
//       fp64 in the reference's exact operation order (no FMA contraction)
//       and overwrites g/bit, so bits equal the reference's except where the
//       fp64 score itself is within 1e-6 of tau (reported).
// The fp64 routine is shared with decode (K4), where it is the only path.
#include <algorithm>

#include "gate.cuh"

namespace wgkv {

// ---------------------------------------------------------------------------
// K1 fp32 main path
// ---------------------------------------------------------------------------
constexpr int GT_TOK = 64;   // tokens per CTA
constexpr int GT_HID = 128;  // hidden units per pass
constexpr int GT_KC = 32;    // k chunk
constexpr int GT_XS = GT_TOK + 4;

template <typename T>
__global__ void __launch_bounds__(256, 2)
    gate_prefill_kernel(GateArgs a, const T* __restrict__ k_pre, T* __restrict__ k_post, float* __restrict__ g_out,
                        uint8_t* __restrict__ bits_out, int32_t* __restrict__ cand, int* __restrict__ pcnt) {
    extern __shared__ float4 smem_f4[];
    float* Xs = reinterpret_cast<float*>(smem_f4);     // [2d][GT_XS]   transposed feature
    float* Ws = Xs + 2 * a.d * GT_XS;                  // [2][GT_KC][GT_HID]
    float* zacc = Ws + 2 * GT_KC * GT_HID;             // [GT_TOK]
    float* sacc = zacc + GT_TOK;                        // [GT_TOK]

    const int tid = threadIdx.x;
    const int h = blockIdx.y, s = blockIdx.z;
    const long t0 = (long)blockIdx.x * GT_TOK;
    const int d = a.d, fd = 2 * d;
    const int blk = a.layer * a.bank_heads + a.head_offset + h;

    // ---- stage 1: load k_pre, RoPE, write k_post, build Xs ----------------
    for (int e = tid; e < GT_TOK * (d / 2); e += blockDim.x) {
        const int tok = e / (d / 2), i = e % (d / 2);
        const long t = t0 + tok;
        float x0 = 0.f, x1 = 0.f, y0 = 0.f, y1 = 0.f;
        if (t < a.T) {
            const size_t off = (((size_t)s * a.T + t) * a.kv_heads + h) * d + 2 * i;
            x0 = to_f(k_pre[off]);
            x1 = to_f(k_pre[off + 1]);
            float c, sn;
            rope_cs(a.freq, i, a.pos0 + t, c, sn);
            y0 = x0 * c - x1 * sn;
            y1 = x0 * sn + x1 * c;
            k_post[off] = from_f<T>(y0);
            k_post[off + 1] = from_f<T>(y1);
        }
        Xs[(2 * i) * GT_XS + tok] = x0;
        Xs[(2 * i + 1) * GT_XS + tok] = x1;
        Xs[(d + 2 * i) * GT_XS + tok] = y0;
        Xs[(d + 2 * i + 1) * GT_XS + tok] = y1;
    }
    if (tid < GT_TOK) {
        zacc[tid] = 0.f;
        sacc[tid] = 0.f;
    }

    // thread micro-tile: tokens 4*ty .. +3, hidden 8*tx .. +7
    const int tx = tid & 15, ty = tid >> 4;
    const float* w1t = a.w1t + (size_t)blk * fd * a.hidden;  // [2d][hidden]
    const int nkc = (fd + GT_KC - 1) / GT_KC;

    for (int hb = 0; hb < a.hidden; hb += GT_HID) {
        float acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

        auto load_w = [&](int kc, int buf) {
            float* dst = Ws + buf * GT_KC * GT_HID;
            for (int e = tid; e < GT_KC * GT_HID; e += blockDim.x) {
                const int kk = kc * GT_KC + e / GT_HID, hh = hb + e % GT_HID;
                dst[e] = (kk < fd && hh < a.hidden) ? w1t[(size_t)kk * a.hidden + hh] : 0.f;
            }
        };
        load_w(0, 0);
        __syncthreads();
        for (int kc = 0; kc < nkc; ++kc) {
            if (kc + 1 < nkc) load_w(kc + 1, (kc + 1) & 1);
            const float* W = Ws + (kc & 1) * GT_KC * GT_HID;
            const int kmax = min(GT_KC, fd - kc * GT_KC);
            for (int k = 0; k < kmax; ++k) {
                const float4 xv = *reinterpret_cast<const float4*>(&Xs[(kc * GT_KC + k) * GT_XS + 4 * ty]);
                const float4 w0 = *reinterpret_cast<const float4*>(&W[k * GT_HID + 8 * tx]);
                const float4 w1 = *reinterpret_cast<const float4*>(&W[k * GT_HID + 8 * tx + 4]);
                const float xr[4] = {xv.x, xv.y, xv.z, xv.w};
                const float wr[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(xr[i], wr[j], acc[i][j]);
            }
            __syncthreads();
        }
        // epilogue of this hidden block: sum_j w2 * gelu(z1 + b1)
        float part[4] = {0.f, 0.f, 0.f, 0.f}, apart[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int hh = hb + 8 * tx + j;
            if (hh < a.hidden) {
                const float b1 = a.b1f[(size_t)blk * a.hidden + hh];
                const float w2 = a.w2f[(size_t)blk * a.hidden + hh];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float z1 = acc[i][j] + b1;
                    const float ge = 0.5f * z1 * (1.f + erff(z1 * 0.70710678118654752f));
                    part[i] = fmaf(w2, ge, part[i]);
                    apart[i] += fabsf(w2 * ge);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#pragma unroll
            for (int o = 8; o >= 1; o >>= 1) {
                part[i] += __shfl_xor_sync(0xffffffffu, part[i], o);
                apart[i] += __shfl_xor_sync(0xffffffffu, apart[i], o);
            }
        }
        if (tx == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                zacc[4 * ty + i] += part[i];
                sacc[4 * ty + i] += apart[i];
            }
        }
        __syncthreads();
    }

    // ---- final: sigmoid, threshold, candidate list -------------------------
    if (tid < GT_TOK) {
        const long t = t0 + tid;
        if (t < a.T) {
            const float z2 = (float)a.b2f[blk] + zacc[tid];
            const float g = 1.f / (1.f + __expf(-z2));
            const size_t gi = ((size_t)s * a.kv_heads + h) * a.T + t;
            g_out[gi] = g;
            bits_out[gi] = z2 >= a.ztau ? 1 : 0;
            // Worst-case fp32 error of z2 (u = 2^-24, n = 2d products/unit):
            //   sum_h |w2_h| |gelu'| n u sum_k |W1_hk x_k|
            //     <= 1.13 (n+1) u ||x||_2 * C,  C = sum_h |w2_h| ||W1_h||_2 (host),
            // plus the GELU/sum/threshold roundings ~ (hidden + 6) u (S + |b2| + |ztau|);
            // x4 margin.  Tokens inside the band are recomputed in fp64.
            float xx = 0.f;
            for (int k = 0; k < fd; ++k) xx = fmaf(Xs[k * GT_XS + tid], Xs[k * GT_XS + tid], xx);
            const float u = 5.9604645e-8f;
            const float band = 4.f * (1.13f * (fd + 1) * u * sqrtf(xx) * a.bandc[blk] +
                                      (a.hidden + 6) * u * (sacc[tid] + fabsf((float)a.b2f[blk]) + fabsf(a.ztau)));
            if (fabsf(z2 - a.ztau) <= band) {  // per-(seq, kv head) candidate list
                const int pair = s * a.kv_heads + h;
                cand[(size_t)pair * a.T + atomicAdd(&pcnt[pair], 1)] = (int32_t)t;
            }
        }
    }
}

// One warp per candidate: exact fp64 gate, overwrite g/bit, report |g-tau|<1e-6.
// Candidates are listed per (seq, kv head) pair (blockIdx.y): cand[pair*T + i] = t.
template <typename T>
__global__ void gate_recheck_kernel(GateArgs a, const T* __restrict__ k_pre, float* __restrict__ g_out,
                                    uint8_t* __restrict__ bits_out, const int32_t* __restrict__ cand,
                                    const int* __restrict__ pcnt, int64_t* __restrict__ near_idx, int near_cap,
                                    int* __restrict__ near_cnt) {
    extern __shared__ double dsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int d = a.d;
    double* xs = dsm + (size_t)warp * (2 * d + a.hidden);
    double* terms = xs + 2 * d;
    float* kf = reinterpret_cast<float*>(dsm + (size_t)nw * (2 * d + a.hidden)) + warp * d;
    const int pair = blockIdx.y, s = pair / a.kv_heads, h = pair % a.kv_heads;
    const int n = pcnt[pair];
    for (int c = blockIdx.x * nw + warp; c < n; c += gridDim.x * nw) {
        const long t = cand[(size_t)pair * a.T + c];
        const int64_t gi = ((int64_t)s * a.kv_heads + h) * a.T + t;
        const size_t off = (((size_t)s * a.T + t) * a.kv_heads + h) * d;
        for (int k = lane; k < d; k += 32) kf[k] = to_f(k_pre[off + k]);
        __syncwarp();
        feature_fp64_warp(kf, d, a.pos0 + t, a.freq, xs);
        const int blk = a.layer * a.bank_heads + a.head_offset + h;
        const double g = gate_fp64_warp(a.gd(), blk, xs, d, terms);
        if (lane == 0) {
            g_out[gi] = (float)g;
            bits_out[gi] = g >= a.tau ? 1 : 0;
            if (fabs(g - a.tau) < 1e-6) {
                const int slot = atomicAdd(near_cnt, 1);
                if (slot < near_cap) near_idx[slot] = gi;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// fp64 recheck as a blocked GEMM (d = hidden = 128): one work item = up to 64
// listed tokens of one (seq, kv head), so every W1 element fetched serves 64
// tokens (the per-token warp form re-reads the head's 256 KB fp64 W1 from L2
// for every token).  X = [k_pre ; RoPE_fp64(k_pre)] for the 64 tokens is built
// in smem exactly as feature_fp64_warp does; z1 = W1 . x in fp64 with k in
// ascending order and the product and sum rounded separately (dot,
// numerics.cpp:94-99, built without FMA contraction); then, per token, the
// reference's order for the rest: terms w2_h * gelu(z1_h + b1_h),
// z2 = b2 + sum_h terms (sequential), sigmoid, clamp (gating.cpp:158-171).
// The fp64 score equals the reference's up to libm ulps (cos/sin/erf/exp).
// ---------------------------------------------------------------------------
constexpr int RC_C = 64;   // tokens per work item
constexpr int RC_KC = 32;  // k chunk of W1 staged per step
constexpr int RC_TP = 129; // padded terms row (doubles)
constexpr size_t RC_SMEM = sizeof(double) * (256 * RC_C + (size_t)RC_C * RC_TP) + 4 * RC_C + 16;

template <typename T>
__global__ void __launch_bounds__(256, 1)
    gate_recheck_gemm_kernel(GateArgs a, int npairs, const T* __restrict__ k_pre, float* __restrict__ g_out,
                             uint8_t* __restrict__ bits_out, const int32_t* __restrict__ cand,
                             const int* __restrict__ pcnt, int64_t* __restrict__ near_idx, int near_cap,
                             int* __restrict__ near_cnt) {
    extern __shared__ double rsm[];
    double* X = rsm;                         // [256 k][RC_C]
    double* Wt = X + 256 * RC_C;             // [RC_KC][128] W1 chunk (k-major); then terms [RC_C][RC_TP]
    int* ts = reinterpret_cast<int*>(Wt + RC_C * RC_TP);  // [RC_C] token index t
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    constexpr int d = 128, fd = 256, hid = 128;
    // items: pair-major chunks of RC_C listed tokens
    int item = blockIdx.x;
    int pair = 0, before = 0;
    for (;; item += gridDim.x) {
        // locate (pair, chunk) of this item (pairs are few; a linear walk)
        int acc = 0, p = 0, nc = 0;
        for (; p < npairs; ++p) {
            nc = (pcnt[p] + RC_C - 1) / RC_C;
            if (item < acc + nc) break;
            acc += nc;
        }
        if (p >= npairs) break;
        pair = p;
        before = (item - acc) * RC_C;
        const int n = min(RC_C, pcnt[pair] - before);
        const int s = pair / a.kv_heads, h = pair % a.kv_heads;
        const int blk = a.layer * a.bank_heads + a.head_offset + h;
        __syncthreads();  // previous item done with X / Wt / ts
        if (tid < RC_C) ts[tid] = tid < n ? cand[(size_t)pair * a.T + before + tid] : 0;
        __syncthreads();
        // ---- features (feature_fp64_warp's arithmetic) ---------------------
        for (int e = tid; e < RC_C * (d / 2); e += blockDim.x) {
            const int c = e % RC_C, i = e / RC_C;
            double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
            if (c < n) {
                const long t = ts[c];
                const size_t off = (((size_t)s * a.T + t) * a.kv_heads + h) * d + 2 * i;
                x0 = (double)to_f(k_pre[off]);
                x1 = (double)to_f(k_pre[off + 1]);
                const double angle = __dmul_rn((double)(a.pos0 + t), a.freq[i]);
                const double cs = cos(angle), sn = sin(angle);
                y0 = __dsub_rn(__dmul_rn(x0, cs), __dmul_rn(x1, sn));
                y1 = __dadd_rn(__dmul_rn(x0, sn), __dmul_rn(x1, cs));
            }
            X[(2 * i) * RC_C + c] = x0;
            X[(2 * i + 1) * RC_C + c] = x1;
            X[(d + 2 * i) * RC_C + c] = y0;
            X[(d + 2 * i + 1) * RC_C + c] = y1;
        }
        // ---- z1 = W1 . x: thread owns tokens 8ty..8ty+7, hidden tx + 32j ---
        double acc8[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc8[i][j] = 0.0;
        const double* w1 = a.w1d + (size_t)blk * hid * fd;
        // register prefetch of the next W1 chunk: 8 double2 per thread
        double2 pre[8];
        auto fetch = [&](int kc) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int e = tid + 256 * q;  // 2048 double2 = [128 h][16 k-pairs]
                const int hh = e & 127, kp = e >> 7;
                pre[q] = *reinterpret_cast<const double2*>(w1 + (size_t)hh * fd + kc * RC_KC + 2 * kp);
            }
        };
        fetch(0);
        for (int kc = 0; kc < fd / RC_KC; ++kc) {
            __syncthreads();  // previous chunk consumed (and, first time, X written)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int e = tid + 256 * q;
                const int hh = e & 127, kp = e >> 7;
                Wt[(2 * kp) * 128 + hh] = pre[q].x;
                Wt[(2 * kp + 1) * 128 + hh] = pre[q].y;
            }
            __syncthreads();
            if (kc + 1 < fd / RC_KC) fetch(kc + 1);
#pragma unroll 4
            for (int kk = 0; kk < RC_KC; ++kk) {
                const double* xr = X + (size_t)(kc * RC_KC + kk) * RC_C + 8 * ty;
                const double2 x01 = *reinterpret_cast<const double2*>(xr);
                const double2 x23 = *reinterpret_cast<const double2*>(xr + 2);
                const double2 x45 = *reinterpret_cast<const double2*>(xr + 4);
                const double2 x67 = *reinterpret_cast<const double2*>(xr + 6);
                const double xv[8] = {x01.x, x01.y, x23.x, x23.y, x45.x, x45.y, x67.x, x67.y};
                double wv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) wv[j] = Wt[kk * 128 + tx + 32 * j];
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc8[i][j] = __dadd_rn(acc8[i][j], __dmul_rn(wv[j], xv[i]));
            }
        }
        __syncthreads();  // Wt becomes the terms buffer
        double* terms = Wt;
        const double* b1 = a.b1d + (size_t)blk * hid;
        const double* w2 = a.w2d + (size_t)blk * hid;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int hh = tx + 32 * j;
            const double bb = b1[hh], ww = w2[hh];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                terms[(8 * ty + i) * RC_TP + hh] = __dmul_rn(ww, gelu_ref(__dadd_rn(acc8[i][j], bb)));
        }
        __syncthreads();
        if (tid < n) {
            double z2 = a.b2d[blk];
            for (int hh = 0; hh < hid; ++hh) z2 = __dadd_rn(z2, terms[tid * RC_TP + hh]);
            double g = sigmoid_ref(z2);
            const double lo = 4.9406564584124654e-324, hi = 0.99999999999999988898;
            g = g < lo ? lo : (g > hi ? hi : g);
            const int64_t gi = ((int64_t)s * a.kv_heads + h) * a.T + ts[tid];
            g_out[gi] = (float)g;
            bits_out[gi] = g >= a.tau ? 1 : 0;
            if (fabs(g - a.tau) < 1e-6) {
                const int slot = atomicAdd(near_cnt, 1);
                if (slot < near_cap) near_idx[slot] = gi;
            }
        }
    }
}

template <typename T>
int launch_gate_prefill(const GateArgs& a, int nseq, const T* k_pre, T* k_post, float* g, uint8_t* bits,
                        int32_t* cand, int* pcnt, int64_t* near_idx, int near_cap, int* near_cnt,
                        const __nv_bfloat16* w1split, long n_wtiles, float2* rope_ws, cudaStream_t st) {
    const int npairs = nseq * a.kv_heads;
    cudaMemsetAsync(pcnt, 0, sizeof(int) * npairs, st);
    bool done = false;
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        // tensor-core path (d = hidden = 128, split-bf16 W1 prepared by wgkv_gate_set)
        if (w1split && a.d == 128 && a.hidden == 128) {
            const int r = launch_gate_tc(a, nseq, k_pre, k_post, g, bits, cand, pcnt, w1split, n_wtiles, rope_ws, st);
            if (r != WGKV_OK) return r;
            done = true;
        }
    }
    if (!done) {
        const size_t smem = sizeof(float) * ((size_t)2 * a.d * GT_XS + 2 * GT_KC * GT_HID + 2 * GT_TOK);
        if (ensure_smem(gate_prefill_kernel<T>, smem) != cudaSuccess) return WGKV_ECUDA;
        dim3 grid((unsigned)((a.T + GT_TOK - 1) / GT_TOK), a.kv_heads, nseq);
        gate_prefill_kernel<T><<<grid, 256, smem, st>>>(a, k_pre, k_post, g, bits, cand, pcnt);
    }
    return launch_gate_recheck<T>(a, nseq, k_pre, g, bits, cand, pcnt, near_idx, near_cap, near_cnt, st);
}

// the fp64 recheck of the listed tokens (reference operation order), bits overwritten
template <typename T>
int launch_gate_recheck(const GateArgs& a, int nseq, const T* k_pre, float* g, uint8_t* bits, int32_t* cand,
                        int* pcnt, int64_t* near_idx, int near_cap, int* near_cnt, cudaStream_t st) {
    const int npairs = nseq * a.kv_heads;
    if (a.d == 128 && a.hidden == 128) {
        if (ensure_smem(gate_recheck_gemm_kernel<T>, RC_SMEM) != cudaSuccess) return WGKV_ECUDA;
        gate_recheck_gemm_kernel<T><<<num_sms(), 256, RC_SMEM, st>>>(a, npairs, k_pre, g, bits, cand, pcnt, near_idx,
                                                                   near_cap, near_cnt);
        return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
    }
    const int nw = 8;
    const size_t rsm = sizeof(double) * nw * (2 * a.d + a.hidden) + sizeof(float) * nw * a.d;
    gate_recheck_kernel<T><<<dim3(std::max(1, num_sms() * 4 / npairs), npairs), 32 * nw, rsm, st>>>(
        a, k_pre, g, bits, cand, pcnt, near_idx, near_cap, near_cnt);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

template <typename T>
__global__ void forced_gate_kernel(GateArgs a, int nseq, const T* __restrict__ k_pre, T* __restrict__ k_post,
                                   const float* __restrict__ forced, float* __restrict__ g_out,
                                   uint8_t* __restrict__ bits_out) {
    const int d = a.d, hp = d / 2;
    const size_t n = (size_t)nseq * a.T * a.kv_heads * hp;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(e % hp);
        const size_t row = e / hp;  // (s*T + t)*H + h
        const int h = (int)(row % a.kv_heads);
        const long t = (long)((row / a.kv_heads) % a.T);
        const int s = (int)(row / ((size_t)a.kv_heads * a.T));
        const size_t off = row * d + 2 * i;
        const float x0 = to_f(k_pre[off]), x1 = to_f(k_pre[off + 1]);
        float c, sn;
        rope_cs(a.freq, i, a.pos0 + t, c, sn);
        k_post[off] = from_f<T>(x0 * c - x1 * sn);
        k_post[off + 1] = from_f<T>(x0 * sn + x1 * c);
        if (i == 0) {
            const size_t gi = ((size_t)s * a.kv_heads + h) * a.T + t;
            const float g = forced[gi];
            g_out[gi] = g;
            bits_out[gi] = (double)g >= a.tau ? 1 : 0;
        }
    }
}

int launch_forced_gate(const GateArgs& a, int nseq, const void* k_pre, void* k_post, const float* forced, float* g,
                       uint8_t* bits, size_t esz, cudaStream_t st) {
    if (esz == 2)
        forced_gate_kernel<__nv_bfloat16><<<num_sms() * 8, 256, 0, st>>>(
            a, nseq, (const __nv_bfloat16*)k_pre, (__nv_bfloat16*)k_post, forced, g, bits);
    else
        forced_gate_kernel<float><<<num_sms() * 8, 256, 0, st>>>(a, nseq, (const float*)k_pre, (float*)k_post, forced,
                                                               g, bits);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

template int launch_gate_recheck<__nv_bfloat16>(const GateArgs&, int, const __nv_bfloat16*, float*, uint8_t*,
                                                int32_t*, int*, int64_t*, int, int*, cudaStream_t);
template int launch_gate_prefill<float>(const GateArgs&, int, const float*, float*, float*, uint8_t*, int32_t*, int*,
                                        int64_t*, int, int*, const __nv_bfloat16*, long, float2*, cudaStream_t);
template int launch_gate_prefill<__nv_bfloat16>(const GateArgs&, int, const __nv_bfloat16*, __nv_bfloat16*, float*,
                                                uint8_t*, int32_t*, int*, int64_t*, int, int*, const __nv_bfloat16*,
                                                long, float2*, cudaStream_t);

}  // namespace wgkv
