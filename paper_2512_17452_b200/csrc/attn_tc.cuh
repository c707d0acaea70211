// attn_tc.cuh -- K3 tcgen05/TMEM/TMA vertical-slash prefill (bf16, d = 128).
#pragma once
#include <cuda.h>

#include "attn.cuh"

namespace wgkv {
int launch_vs_prefill_tc(const VsArgs& a, int nseq, const __nv_bfloat16* q, const __nv_bfloat16* k_post,
                         const __nv_bfloat16* v, __nv_bfloat16* out, cudaStream_t st);
int make_tmap_3d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1, uint32_t box2);
}
