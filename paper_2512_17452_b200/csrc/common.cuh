// common.cuh -- shared device/host definitions for the WG-KV B200 kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/wgkv_b200.h"

namespace wgkv {

// SM count of the current device (148 on B200), cached per device; grids are
// sized from it, never from a constant
int num_sms();
// cudaFuncAttributeMaxDynamicSharedMemorySize is per device context: set it
// once per (kernel, device) for the largest size requested so far (host-only,
// thread-safe; never a stream operation, so graph capture is unaffected)
cudaError_t ensure_smem_attr(const void* func, size_t smem);
template <typename F>
inline cudaError_t ensure_smem(F* func, size_t smem) {
    return ensure_smem_attr(reinterpret_cast<const void*>(func), smem);
}

// ---------------------------------------------------------------------------
// element conversion
// ---------------------------------------------------------------------------
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// ---------------------------------------------------------------------------
// per-(layer, seq, kv head) dual-cache state (HeadCache members, kvstore.hpp:135-143)
// ---------------------------------------------------------------------------
struct HeadState {
    int local_len;
    int local_ptr;
    int global_len;
    int tokens_seen;
};

// Device view of the paged pool + tables, passed by value to kernels.
// Page p holds K rows [ps][d] then V rows [ps][d] (elements of type T).
struct PoolView {
    void* data;          // [cap][2][ps][d]
    float* gate;         // [cap][ps]
    int32_t* pos;        // [cap][ps]
    uint8_t* adm;        // [cap][ps]
    int32_t* free_stack; // [cap] (LIFO, KvPool::free_ kvstore.cpp:9-21)
    int32_t* free_top;   // number of free pages
    int32_t* err;        // latched device error (WGKV_ENOPAGES)
    int32_t* lpt;        // [L][S][H][n_lp] local page table
    int32_t* gpt;        // [L][S][H][n_gp] global page table
    HeadState* state;    // [L][S][H]
    int page_size, head_dim, n_lp, n_gp, max_seqs, kv_heads;
    long capacity;

    __host__ __device__ long head_index(int layer, int seq, int h) const {
        return ((long)layer * max_seqs + seq) * kv_heads + h;
    }
    __host__ __device__ size_t page_elems() const { return (size_t)2 * page_size * head_dim; }
};

// Pops one page from the device free stack; -1 (and the error latch) when
// exhausted (KvPool::alloc_page "out of pages", kvstore.cpp:23-31).
__device__ __forceinline__ int pool_pop(const PoolView& pv) {
    // CAS loop: the counter only ever moves down by a claim that succeeds, so a
    // failing pop never makes a concurrent claim fail spuriously
    int top = *reinterpret_cast<volatile int32_t*>(pv.free_top);
    for (;;) {
        if (top <= 0) {
            atomicExch(pv.err, WGKV_ENOPAGES);
            return -1;
        }
        const int seen = atomicCAS(pv.free_top, top, top - 1);
        if (seen == top) break;
        top = seen;
    }
    const int page = pv.free_stack[top - 1];
    if (page < 0) {  // a corrupted stack entry is an allocation failure, never a page
        atomicExch(pv.err, WGKV_ENOPAGES);
        return -1;
    }
    return page;
}
// claims n pages at once (LIFO order: page i = free_stack[base - 1 - i]);
// returns base (the old top) or -1 with the error latched
__device__ __forceinline__ int pool_claim(const PoolView& pv, int n) {
    int top = *reinterpret_cast<volatile int32_t*>(pv.free_top);
    for (;;) {
        if (top < n) {
            atomicExch(pv.err, WGKV_ENOPAGES);
            return -1;
        }
        const int seen = atomicCAS(pv.free_top, top, top - n);
        if (seen == top) return top;
        top = seen;
    }
}

// ---------------------------------------------------------------------------
// RoPE: interleaved pairs (2i, 2i+1) rotated by pos * base^(-2i/d)
// (numerics.cpp:50-63).  freq[i] is computed on the host with the reference
// expression; the angle is formed and range-reduced in fp64 (exact to ~1e-15
// rad at 1M positions) and the rotation runs in fp32.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void rope_cs(const double* __restrict__ freq, int i, long pos, float& c, float& s) {
    const double angle = (double)pos * freq[i];
    const double k = rint(angle * 0.15915494309189533576888376337251436);
    double r = fma(-k, 6.28318530717958623199592693708837032, angle);
    r = fma(-k, 2.44929359829470635445213186455000e-16, r);
    sincosf((float)r, &s, &c);
}
// same angle, MUFU sin/cos (|error| < 1e-6 on the reduced range): used where
// the rotated value is stored as bf16 anyway (K3's in-smem RoPE of q)
__device__ __forceinline__ void rope_cs_fast(const double* __restrict__ freq, int i, long pos, float& c, float& s) {
    const double angle = (double)pos * freq[i];
    const double k = rint(angle * 0.15915494309189533576888376337251436);
    double r = fma(-k, 6.28318530717958623199592693708837032, angle);
    r = fma(-k, 2.44929359829470635445213186455000e-16, r);
    __sincosf((float)r, &s, &c);
}

// one interleaved pair rotated in fp32 with pinned roundings (no contraction),
// so every site that forms a cached key from k_pre produces the same bits
__device__ __forceinline__ void rope_pair_f32(float x0, float x1, float c, float s, float& y0, float& y1) {
    y0 = __fsub_rn(__fmul_rn(x0, c), __fmul_rn(x1, s));
    y1 = __fadd_rn(__fmul_rn(x0, s), __fmul_rn(x1, c));
}

// ---------------------------------------------------------------------------
// misc
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

}  // namespace wgkv

// host-side error plumbing (api.cu)
void wgkv_set_error(const std::string& msg);
#define WGKV_CUDA_TRY(expr)                                                                   \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess) {                                                              \
            wgkv_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));               \
            return WGKV_ECUDA;                                                                \
        }                                                                                     \
    } while (0)
