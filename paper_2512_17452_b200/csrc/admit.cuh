// admit.cuh -- K2 / K4 launchers.
#pragma once
#include "common.cuh"
#include "append.cuh"
#include "gate.cuh"

namespace wgkv {

template <typename E>
int launch_admit_prefill(const PoolView& pv, int layer, int seq0, int nseq, long T, long W, const E* k_post,
                         const E* v, const float* g, const uint8_t* bits, int32_t* chunk_off, cudaStream_t st);

// K4 as its own launch (one CTA per (seq, kv head)), append.cuh
template <typename E>
int launch_decode_append(const PoolView& pv, const GateArgs& ga, int layer, int seq0, int nseq, long W,
                         const E* k_pre, const E* v, const float* forced_g, const DecodeTrace& tr,
                         const AppendWork& wk, cudaStream_t st);

}  // namespace wgkv
