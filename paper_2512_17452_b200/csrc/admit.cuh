// admit.cuh -- K2 / K4 launchers.
#pragma once
#include "common.cuh"
#include "gate.cuh"

namespace wgkv {

template <typename E>
int launch_admit_prefill(const PoolView& pv, int layer, int seq0, int nseq, long T, long W, const E* k_post,
                         const E* v, const float* g, const uint8_t* bits, int32_t* chunk_off, cudaStream_t st);

template <typename E>
int launch_decode_append(const PoolView& pv, const GateArgs& ga, int layer, int seq0, int nseq, long W,
                         const E* k_pre, const E* v, const float* forced_g, float* g_out, int32_t* events,
                         int* work_counter, int* slot_rec, cudaStream_t st, cudaStream_t side,
                         cudaEvent_t ev_fork, cudaEvent_t ev_join);

}  // namespace wgkv
