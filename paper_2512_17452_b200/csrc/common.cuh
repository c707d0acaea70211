// common.cuh -- shared device/host definitions for the WG-KV B200 kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/wgkv_b200.h"

namespace wgkv {

constexpr int kNumSMs = 148;

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
    int top = atomicSub(pv.free_top, 1);
    if (top <= 0) {
        atomicAdd(pv.free_top, 1);
        atomicExch(pv.err, WGKV_ENOPAGES);
        return -1;
    }
    return pv.free_stack[top - 1];
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
