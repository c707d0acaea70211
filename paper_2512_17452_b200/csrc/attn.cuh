// attn.cuh -- K3 / K5 argument blocks and launchers.
#pragma once
#include "common.cuh"

namespace wgkv {

struct VsArgs {
    PoolView pv;
    int layer, seq0, q_heads;
    long T, W;
    const double* freq;        // [d/2]
    const uint8_t* bits;       // [nseq][kv_heads][T]
    const int32_t* chunk_off;  // [nseq][kv_heads][nchunk+1] admitted-before-chunk (K2)
};

// partial-buffer chunks per (seq, kv head): enough for a single kv head to
// spread over every SM (1M-token contexts with 8-way head sharding)
constexpr int kMaxChunks = 512;
// K5 pages per work item (staged page ids); max_tokens per head is bounded by
// kMaxChunks * kDecPidCap pages (checked at context creation)
constexpr int kDecPidCap = 2048;

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
};

// K6: select_topk_pages + per-q-head attention over the selection (topk.cu).
// scores/sel: [nseq][q_heads][n_gp]; nsel, thr: [nseq][q_heads];
// umask [nseq][kv_heads][n_gp], ucnt [nseq][kv_heads][ceil(n_gp/1024)]
template <typename E>
int launch_topk_decode(const DecArgs& a, int nseq, long budget, const E* q, float* scores, int32_t* sel,
                       int32_t* nsel, unsigned long long* thr, uint8_t* umask, int* ucnt, float* part, int* nchunks,
                       E* out, int mode, __nv_bfloat16* meta, int* meta_full, cudaStream_t st);

// counter_reset_by_append: K4 ran just before on the stream and zeroed the
// work counter; K5 is then launched as its programmatic dependent (PDL)
int launch_decode_attn_mma(const DecArgs& a, int nseq, const __nv_bfloat16* q, float* part, int* nchunks,
                           __nv_bfloat16* out, cudaStream_t st, bool counter_reset_by_append);

template <typename T>
int launch_vs_prefill_simt(const VsArgs& a, int nseq, const T* q, const T* k_post, const T* v, T* out,
                           cudaStream_t st);
template <typename T>
int launch_decode_attn_simt(const DecArgs& a, int nseq, const T* q, float* part, T* out, cudaStream_t st);

}  // namespace wgkv
