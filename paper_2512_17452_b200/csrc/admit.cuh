// admit.cuh -- K2 / K4 launchers.
#pragma once
#include "common.cuh"
#include "append.cuh"
#include "gate.cuh"

namespace wgkv {

template <typename E>
int launch_admit_prefill(const PoolView& pv, int layer, int seq0, int nseq, long T, long W, const E* k_post,
                         const E* v, const float* g, const uint8_t* bits, int32_t* chunk_off, cudaStream_t st);

// K4 as its own launch (append.cuh): mode 0 route + gate CTAs; mode 1 the route
// CTAs only (they publish the head state); mode 2 the gate CTAs of a mode-1 append;
// mode 3 the gate CTAs of a deferred decode (the finish kernel's route CTAs arrive too)
template <typename E>
int launch_decode_append(const PoolView& pv, const GateArgs& ga, int layer, int seq0, int nseq, long W,
                         const E* k_pre, const E* v, const float* forced_g, const DecodeTrace& tr,
                         const AppendWork& wk, cudaStream_t st, int mode = 0);

}  // namespace wgkv
