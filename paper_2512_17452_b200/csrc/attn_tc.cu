// attn_tc.cu -- K3 tcgen05 path (work in progress; selected only with
// attn_impl = WGKV_ATTN_TCGEN05 until it is parity-green).
#include "attn_tc.cuh"

namespace wgkv {
int launch_vs_prefill_tc(const VsArgs&, int, const __nv_bfloat16*, const __nv_bfloat16*, const __nv_bfloat16*,
                         __nv_bfloat16*, cudaStream_t) {
    return WGKV_ENOTSUP;
}
}  // namespace wgkv
