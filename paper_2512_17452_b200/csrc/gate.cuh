// gate.cuh -- K1 (write-gate) declarations shared by prefill and decode.
#pragma once
#include "common.cuh"

namespace wgkv {

// fp64 copy of the gate bank for the exact path (local kv heads only,
// block index = layer * kv_heads + h).
struct GateDev {
    const double* w1d;  // [blk][hidden][2d]
    const double* b1d;  // [blk][hidden]
    const double* w2d;  // [blk][hidden]
    const double* b2d;  // [blk]
    int hidden;
};

struct GateArgs {
    int layer, kv_heads, bank_heads, head_offset, d, hidden;
    long T, pos0;
    double tau;
    float ztau;          // logit(tau) in fp32 (threshold on z2 for the fp32 path)
    const double* freq;  // [d/2] base^(-2i/d), host-computed (numerics.cpp:54)
    const float* w1t;    // [blk][2d][hidden]  (transposed fp32 W1)
    const float* b1f;    // [blk][hidden]
    const float* w2f;    // [blk][hidden]
    const double* b2f;   // [blk]
    const float* bandc;  // [blk] sum_h |w2_h| * ||W1_h||_2 (fp32 error bound constant)
    const float4* bw;    // [blk][hidden/2] interleaved b1 / w2 pairs (tensor-core epilogue)
    const double* w1d;
    const double* b1d;
    const double* w2d;
    const double* b2d;
    __device__ GateDev gd() const { return GateDev{w1d, b1d, w2d, b2d, hidden}; }
};

// ---------------------------------------------------------------------------
// exact fp64 gate for ONE token, reference operation order
// ---------------------------------------------------------------------------
__device__ __forceinline__ double gelu_ref(double x) {
    // x * 0.5 * (1.0 + erf(x * sqrt2 * 0.5))   numerics.cpp:33-36
    const double a = __dmul_rn(x, 0.5);
    const double e = erf(__dmul_rn(__dmul_rn(x, 1.41421356237309504880), 0.5));
    return __dmul_rn(a, __dadd_rn(1.0, e));
}

__device__ __forceinline__ double sigmoid_ref(double x) {  // numerics.cpp:44-48
    if (x >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));
    const double e = exp(x);
    return __ddiv_rn(e, __dadd_rn(1.0, e));
}

// Builds x = [k_pre ; RoPE(k_pre)] in fp64 (gating.cpp:149-156,
// numerics.cpp:53-62) into xs[0..2d) using the calling warp.
__device__ __forceinline__ void feature_fp64_warp(const float* kpre, int d, long pos, const double* freq, double* xs) {
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < d / 2; i += 32) {
        const double angle = __dmul_rn((double)pos, freq[i]);
        const double c = cos(angle), s = sin(angle);
        const double a = kpre[2 * i], b = kpre[2 * i + 1];
        xs[2 * i] = a;
        xs[2 * i + 1] = b;
        xs[d + 2 * i] = __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, s));
        xs[d + 2 * i + 1] = __dadd_rn(__dmul_rn(a, s), __dmul_rn(b, c));
    }
    __syncwarp();
}

// dot (numerics.cpp:94-99) in the reference's operation order: s = 0, then
// s += w[k] * x[k] for ascending k with the product and the sum rounded
// separately (the reference is built without FMA contraction).
__device__ __forceinline__ double dot_ref(const double* __restrict__ w, const double* __restrict__ x, int n) {
    double s = 0.0;
    int k = 0;
    for (; k + 4 <= n; k += 4) {  // loads of a group issued together; the sum stays sequential
        const double2 w01 = *reinterpret_cast<const double2*>(w + k);
        const double2 w23 = *reinterpret_cast<const double2*>(w + k + 2);
        s = __dadd_rn(s, __dmul_rn(w01.x, x[k]));
        s = __dadd_rn(s, __dmul_rn(w01.y, x[k + 1]));
        s = __dadd_rn(s, __dmul_rn(w23.x, x[k + 2]));
        s = __dadd_rn(s, __dmul_rn(w23.y, x[k + 3]));
    }
    for (; k < n; ++k) s = __dadd_rn(s, __dmul_rn(w[k], x[k]));
    return s;
}

// sigmoid + the reference clamp to [5e-324, nextafter(1, 0)] (gating.cpp:168-170)
__device__ __forceinline__ double gate_from_z2(double z2) {
    const double g = sigmoid_ref(z2);
    const double lo = 4.9406564584124654e-324, hi = 0.99999999999999988898;
    return g < lo ? lo : (g > hi ? hi : g);
}

// gate_forward (gating.cpp:158-171) by one warp, reference operation order
// throughout: lanes own hidden units h = lane, lane + 32, ...; each z1 is a
// sequential dot_ref over the feature; terms w2[h] * gelu(z1 + b1[h]) go to
// smem and lane 0 sums z2 = b2 + terms[0] + terms[1] + ... in order.  So the
// fp64 result equals the reference's up to the libm ulps of cos/sin (RoPE),
// erf and exp.  terms: smem scratch [hidden].  W1 rows are 16-byte aligned
// (2d even).
__device__ __forceinline__ double gate_fp64_warp(const GateDev& gd, int blk, const double* xs, int d, double* terms) {
    const int lane = threadIdx.x & 31;
    const int fd = 2 * d, hid = gd.hidden;
    const double* w1 = gd.w1d + (size_t)blk * hid * fd;
    const double* b1 = gd.b1d + (size_t)blk * hid;
    const double* w2 = gd.w2d + (size_t)blk * hid;
    for (int h = lane; h < hid; h += 32)
        terms[h] = __dmul_rn(w2[h], gelu_ref(__dadd_rn(dot_ref(w1 + (size_t)h * fd, xs, fd), b1[h])));
    __syncwarp();
    double z2 = 0.0;
    if (lane == 0) {
        z2 = gd.b2d[blk];
        for (int h = 0; h < hid; ++h) z2 = __dadd_rn(z2, terms[h]);
    }
    z2 = __shfl_sync(0xffffffffu, z2, 0);
    return gate_from_z2(z2);
}

// The hidden-unit terms of gate_forward for one token by `nthr` threads
// starting at thread `t0` of the block (thread t0 + u owns units u, u + nthr,
// ...): terms[h] = w2[h] * gelu(dot_ref(W1[h], x) + b1[h]).  The caller sums
// them in order with gate_z2_ref after a barrier.
__device__ __forceinline__ void gate_terms_ref(const GateDev& gd, int blk, const double* xs, int d, double* terms,
                                               int t0, int nthr) {
    const int u0 = (int)threadIdx.x - t0;
    if (u0 < 0 || u0 >= nthr) return;
    const int fd = 2 * d, hid = gd.hidden;
    const double* w1 = gd.w1d + (size_t)blk * hid * fd;
    const double* b1 = gd.b1d + (size_t)blk * hid;
    const double* w2 = gd.w2d + (size_t)blk * hid;
    for (int h = u0; h < hid; h += nthr)
        terms[h] = __dmul_rn(w2[h], gelu_ref(__dadd_rn(dot_ref(w1 + (size_t)h * fd, xs, fd), b1[h])));
}
__device__ __forceinline__ double gate_z2_ref(const GateDev& gd, int blk, const double* terms) {
    double z2 = gd.b2d[blk];
    for (int h = 0; h < gd.hidden; ++h) z2 = __dadd_rn(z2, terms[h]);
    return z2;
}

// effective_gate override (engine.cpp:126-151): RoPE only; g = forced, bit = g >= tau
int launch_forced_gate(const GateArgs& a, int nseq, const void* k_pre, void* k_post, const float* forced, float* g,
                       uint8_t* bits, size_t esz, cudaStream_t st);

// cand: [nseq*kv_heads][T] token indices listed for the fp64 recheck, pcnt:
// [nseq*kv_heads] list lengths; rope_ws: [T][d/2] cos/sin workspace (bf16 tc path)
template <typename T>
int launch_gate_prefill(const GateArgs& a, int nseq, const T* k_pre, T* k_post, float* g, uint8_t* bits,
                        int32_t* cand, int* pcnt, int64_t* near_idx, int near_cap, int* near_cnt,
                        const __nv_bfloat16* w1split, long n_wtiles, float2* rope_ws, cudaStream_t st);

// tensor-core K1 (gate_tc.cu): w1split = [L*H][4][128][128] bf16 split W1 tiles
int launch_gate_tc(const GateArgs& a, int nseq, const __nv_bfloat16* k_pre, __nv_bfloat16* k_post, float* g,
                   uint8_t* bits, int32_t* cand, int* pcnt, const __nv_bfloat16* w1split, long n_wtiles,
                   float2* rope_ws, cudaStream_t st);

// cos/sin table of one call's positions (gate_tc.cu), [T][d/2] float2
void launch_rope_table(const double* freq, long pos0, long T, int hp, float2* out, cudaStream_t st);
// f1 (gate_proj.cu): the key projection fused into K1 -- x [nseq][T][dm], wk [kv_heads][128][dm]
// bf16; writes k_pre (bf16 of the fp32 projection), k_post, g, bits and the recheck list
int launch_gate_proj_tc(const GateArgs& a, int nseq, const __nv_bfloat16* x, const __nv_bfloat16* wk, int dm,
                        __nv_bfloat16* k_pre, __nv_bfloat16* k_post, float* g, uint8_t* bits, int32_t* cand, int* pcnt,
                        const __nv_bfloat16* w1split, long n_wtiles, float2* rope_ws, cudaStream_t st);
template <typename T>
int launch_gate_recheck(const GateArgs& a, int nseq, const T* k_pre, float* g, uint8_t* bits, int32_t* cand,
                        int* pcnt, int64_t* near_idx, int near_cap, int* near_cnt, cudaStream_t st);

}  // namespace wgkv
