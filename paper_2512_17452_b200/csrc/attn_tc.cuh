// attn_tc.cuh -- K3 tcgen05/TMEM/TMA vertical-slash prefill (bf16, d = 128).
#pragma once
#include "attn.cuh"

namespace wgkv {
int launch_vs_prefill_tc(const VsArgs& a, int nseq, const __nv_bfloat16* q, const __nv_bfloat16* k_post,
                         const __nv_bfloat16* v, __nv_bfloat16* out, cudaStream_t st);
}
