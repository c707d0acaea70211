// attn.cuh -- K3 / K5 argument blocks and launchers.
#pragma once
#include "append.cuh"
#include "fused.cuh"
#include "comm.cuh"
#include "common.cuh"
#include "gate.cuh"

namespace wgkv {

struct VsArgs {
    PoolView pv;
    int layer, seq0, q_heads;
    long T, W;
    const double* freq;        // [d/2]
    const uint8_t* bits;       // [nseq][kv_heads][T]
    const int32_t* chunk_off;  // [nseq][kv_heads][nchunk+1] admitted-before-chunk (K2)
    PeerBulk pb;               // C1 fused into K3 (tcgen05 path): output rows into every rank's bulk slot
};

// partial-buffer chunks per (seq, kv head): enough for a single kv head to
// spread over every SM (1M-token contexts with 8-way head sharding)
constexpr int kMaxChunks = 512;
// K5 pages per work item (staged page ids); max_tokens per head is bounded by
// kMaxChunks * kDecPidCap pages (checked at context creation)
constexpr int kDecPidCap = 2048;
constexpr int kDecSmemStatePairs = 512;  // K5 caches per-pair head state in smem up to this many pairs

struct DecArgs {
    PoolView pv;
    int layer, seq0, q_heads;
    int chunk_pages;  // virtual pages per CTA
    int n_chunks;     // chunks launched per (seq, kv head)
    int max_chunks;   // partial-buffer stride
    const double* freq;
    int n_pairs;          // nseq * kv_heads (persistent kernel)
    const int* nchunks;   // per (seq, kv head) chunk count written on device, or null (use n_chunks)
    // K6 union selection (bf16 top-k): per (seq, kv head) [n_gp] entries
    // logical page | q-head mask << 24, and their count; null = all pages
    const int32_t* sel;
    const int32_t* nsel;
    // deferred append (bf16 fast path): K5 attends the cache as it was BEFORE
    // this step's append -- Global, the ring minus a dropped victim -- and the
    // finish kernel adds the new token and runs the append (K4) beside the
    // chunk merge.  tokpos [nseq*kv_heads] receives the new token's position.
    int defer;
    long window;
    int* tokpos;
    int* counter;  // K5 work-stealing counter, reset to 0 by the kernel that merges its partials
    int pin_cp;    // > 0: pages per chunk fixed (wgkv_config.decode_chunk_pages)
    // deferred append with the MLP gate: the first n_gate_ctas CTAs of the K5
    // launch are the append's gate CTAs (append.cuh), off the layer's critical
    // path; the K5 work CTAs follow them
    int n_gate_ctas;
    int early_trigger;  // K5 releases its programmatic dependent right after its PDL wait
    int state_in_smem;  // K5 keeps every pair's HeadState in shared memory (fits for <= kDecSmemStatePairs)
    int prewait;        // K5's predecessor is another layer's finish kernel: plan before the PDL wait
    // fused layer (fused.cuh, small batches): the launch also carries the
    // append's route CTAs (first n_route_ctas) and merges + commits in place of
    // the finish kernel
    int fused;
    int n_route_ctas;
};

// K6: select_topk_pages + per-q-head attention over the selection (topk.cu).
// scores/sel: [nseq][q_heads][n_gp]; nsel, thr: [nseq][q_heads];
// umask [nseq][kv_heads][n_gp], ucnt [nseq][kv_heads][ceil(n_gp/1024)]
template <typename E>
int launch_topk_decode(const DecArgs& a, int nseq, long budget, const E* q, float* scores, int32_t* sel,
                       int32_t* nsel, unsigned long long* thr, uint8_t* umask, int* ucnt, float* part, int* nchunks,
                       E* out, int mode, __nv_bfloat16* meta, int* meta_full, cudaStream_t st);

// the deferred append (a.defer): inputs of the new token and the gate / trace
// outputs, consumed by the finish kernel (decode_finish.cu)
struct FinishArgs {
    GateArgs ga;
    const __nv_bfloat16* k_new;  // [nseq][kv_heads][d] pre-RoPE
    const __nv_bfloat16* v_new;  // [nseq][kv_heads][d]
    const float* forced_g;       // [nseq][kv_heads] or null
    DecodeTrace tr;
    AppendWork wk;
    bool prewait;  // K5 may plan and start its first loads before the PDL wait (see api.cu)
    bool gate_side;  // the append's gate CTAs run in their own launch on a side stream
    FusedWork fw;    // fused layer scratch (this layer's parity halves); cnt_items null = not available
    __nv_bfloat16* out;  // fused layer: the attention output [nseq][q_heads][d] (set by the launcher)
    // C1 over peer memory (comm.cuh): the merges also push the output rows into
    // every rank's exchange slot; one extra K5 CTA unpacks the previous exchange
    PeerXchg px;
};

// counter_reset_by_append: the kernel just before on the stream zeroed the work
// counter; K5 is then launched as its programmatic dependent (PDL).  fin != null
// (deferred append, a.defer = 1): K5 then the finish kernel (merge + new token
// + K4) instead of the combine kernel.
int launch_decode_attn_mma(const DecArgs& a, int nseq, const __nv_bfloat16* q, float* part, int* nchunks,
                           __nv_bfloat16* out, cudaStream_t st, bool counter_reset_by_append,
                           const FinishArgs* fin = nullptr);
int launch_decode_finish(const DecArgs& a, int nseq, const __nv_bfloat16* q, const float* part,
                         __nv_bfloat16* out, const FinishArgs& fin, cudaStream_t st);

template <typename T>
int launch_vs_prefill_simt(const VsArgs& a, int nseq, const T* q, const T* k_post, const T* v, T* out,
                           cudaStream_t st);
template <typename T>
int launch_decode_attn_simt(const DecArgs& a, int nseq, const T* q, float* part, T* out, cudaStream_t st);

}  // namespace wgkv
