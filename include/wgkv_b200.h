/*
 * wgkv_b200.h -- C-ABI of the B200-native Write-Gated KV hot path.
 *
 * The reference (/root/reference/proj) exposes this path only as in-process
 * C++20 calls in namespace wgkv; there is no FFI.  This header
 * is the drop-in boundary a host binds: plain pointers and sizes, no torch or
 * C++ types, int status codes instead of exceptions (include/wgkv_b200.hpp
 * rethrows the reference's exception types).  Each entry point names the
 * reference interface it replaces.
 *
 * Conventions
 *   - A context (wgkv_ctx) owns one device's state for the KV heads it is
 *     given: gate parameters, the paged KV pool, per-(layer, sequence,
 *     kv-head) page tables and ring state, and workspaces.  One host thread per
 *     context; every call is stream-ordered on the context stream
 *     (wgkv_set_stream) and returns without synchronising unless stated.
 *   - Tensor arguments are DEVICE pointers, caller-owned, row-major:
 *       q     [nseq][T][q_heads][d]     (pre-RoPE, as engine.cpp:226-228)
 *       k_pre [nseq][T][kv_heads][d]    (pre-RoPE, as engine.cpp:191-198)
 *       v     [nseq][T][kv_heads][d]
 *       out   [nseq][T][q_heads][d]     (q head p at cols p*d: engine.cpp:234-238)
 *     element type = cfg.dtype (bf16 storage + fp32 math, or fp32 parity mode).
 *   - Sequences live in slots [0, max_seqs); a call covers slots
 *     [seq0, seq0 + nseq).  Positions are 0-based (engine.cpp:256, 296).
 *   - Device-side failures that the reference reports by exception inside a
 *     loop ("out of pages", kvstore.cpp:23-31) are latched in a device flag and
 *     returned by the next wgkv_sync() (or any call documented as syncing).
 */
#ifndef WGKV_B200_H
#define WGKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: 1:1 with the reference's exception classes */
enum {
    WGKV_OK = 0,
    WGKV_EINVAL = 1,   /* std::invalid_argument: shapes, tau not in (0,1), window < 1 */
    WGKV_ENOPAGES = 2, /* std::runtime_error("out of pages ...") kvstore.cpp:23-31 */
    WGKV_ESTATE = 3,   /* std::logic_error: prefill twice, decode before prefill */
    WGKV_ERUNTIME = 4, /* std::runtime_error: empty KV, fully masked row */
    WGKV_ECUDA = 5,    /* CUDA error (no reference equivalent) */
    WGKV_ENOTSUP = 6   /* configuration this build does not implement */
};

enum { WGKV_BF16 = 0, WGKV_F32 = 1 };

/* prefill attention implementation (wgkv_config.attn_impl) */
enum { WGKV_ATTN_AUTO = 0, WGKV_ATTN_SIMT = 1, WGKV_ATTN_TCGEN05 = 2 };

typedef struct wgkv_config {
    int layers;          /* L (engine.hpp:106-107 one HeadCache per (layer, kv head)) */
    int q_heads;         /* q heads on this device (GQA group = q_heads / kv_heads, engine.cpp:224) */
    int kv_heads;        /* kv heads on this device */
    int kv_head_offset;  /* global index of local kv head 0 (gate bank row, KV-head sharding) */
    int head_dim;        /* d, even (numerics.cpp:51) */
    int hidden;          /* gate MLP hidden width (gating.hpp:18-26) */
    long window;         /* W >= 1 (kvstore.cpp:99) */
    double tau;          /* admission threshold in (0,1) (gating.cpp:185) */
    double rope_base;    /* RopeConfig::base (numerics.hpp:30-33) */
    int page_size;       /* KvPool page size (engine.cpp:102 uses 16) */
    int max_seqs;        /* sequence slots */
    long max_tokens;     /* per sequence, prompt + decode */
    long max_prefill_tokens; /* largest T of one prefill call (workspace sizing) */
    long capacity_pages; /* 0 -> default_capacity (engine.cpp:88-93) over all slots */
    int dtype;           /* WGKV_BF16 | WGKV_F32 */
    long topk_budget;    /* 0: attend all Global pages; >0: select_topk_pages (engine.cpp:36-84) */
    int attn_impl;       /* WGKV_ATTN_* */
    int device;          /* CUDA device ordinal */
    int topk_mode;       /* WGKV_TOPK_*: how select_topk_pages scores a page (topk_budget > 0) */
    long decode_chunk_pages; /* 0: K5 sizes its split-KV chunks from the step's work (fastest);
                              * > 0: pages per chunk pinned, so a (seq, kv head)'s decode arithmetic
                              * -- and its output bits -- do not depend on which other heads share
                              * the launch (KV-head sharding reproduces the unsharded result) */
} wgkv_config;

/* page score used by the top-k selection (wgkv_config.topk_mode)
 *   EXACT  max over the page's slots of q.k -- the reference's select_topk_pages
 *          (engine.cpp:36-84); parity mode
 *   QUEST  Quest's upper bound sum_d max(q_d min_d, q_d max_d) over per-page
 *          elementwise key min / max kept on device; reads 1/8 of the Global K
 *          bytes per step, NOT the reference's selection (approximate) */
enum { WGKV_TOPK_EXACT = 0, WGKV_TOPK_QUEST = 1 };

typedef struct wgkv_ctx wgkv_ctx;

/* last error message of the calling thread (never NULL) */
const char* wgkv_last_error(void);
/* build/arch string, e.g. "wgkv_b200 sm_100a" */
const char* wgkv_version(void);

/* Session::Session (engine.cpp:97-120): validates cfg, allocates the pool
 * and all tables; no allocation happens on later hot calls. */
int wgkv_ctx_create(const wgkv_config* cfg, wgkv_ctx** out);
int wgkv_ctx_destroy(wgkv_ctx* ctx);
/* cudaStream_t as void*; NULL = legacy default stream */
int wgkv_set_stream(wgkv_ctx* ctx, void* stream);
/* waits for the stream; returns latched device errors (e.g. WGKV_ENOPAGES) */
int wgkv_sync(wgkv_ctx* ctx);

/* ---- gate parameters (GateBank, gating.hpp:41-68) ------------------------
 * bank: host fp64, layer-major blocks of hidden*2d + 2*hidden + 1 doubles
 * (W1[hidden][2d] | b1 | w2 | b2) for `bank_heads` kv heads; the context
 * takes rows [kv_head_offset, kv_head_offset + kv_heads). */
int wgkv_gate_set(wgkv_ctx* ctx, const double* bank, int bank_layers, int bank_heads);
/* GateBank::load (gating.cpp:107-147), ".wgkv" v1 file */
int wgkv_gate_load(wgkv_ctx* ctx, const char* path);

/* ---- K1: gate_forward_batch + binarize (gating.cpp:149-190) --------------
 * Fused RoPE(k_pre) -> MLP -> sigmoid -> threshold for tokens at positions
 * pos0 .. pos0+T-1 of layer `layer`.  fp32 main path; every token whose score
 * lies near tau is recomputed in fp64 in the reference's operation order, so
 * bits equal the reference's except where |g - tau| < 1e-6; those tokens are
 * reported in near_idx (flat index s*kv_heads*T + h*T + t) up to near_cap.
 *   k_post_out [nseq][T][kv_heads][d]  (dtype)      RoPE'd keys
 *   g_out      [nseq][kv_heads][T]     float        gate scores
 *   bits_out   [nseq][kv_heads][T]     uint8        admission bits
 * forced_g (optional, device float [nseq][kv_heads][T]) replaces the MLP
 * (effective_gate policies, engine.cpp:126-151).  Syncs when near_count != NULL. */
int wgkv_gate_score(wgkv_ctx* ctx, int layer, int nseq, long T, long pos0, const void* k_pre, const float* forced_g,
                    void* k_post_out, float* g_out, uint8_t* bits_out, int64_t* near_idx, int near_cap,
                    int* near_count);

/* f1: wgkv_gate_score with the key projection fused in (engine.cpp:190-205:
 * k_pre = Wk_h . a, k_post = RoPE(k_pre), gate, binarize): one tcgen05 kernel
 * projects each 128-token tile into TMEM, rounds it to bf16 and feeds it
 * straight to the gate GEMM, so k_pre is not re-read from HBM.
 *   x  [nseq][T][dm]     bf16 layer input (after the RMSNorm, engine.cpp:178-182)
 *   wk [kv_heads][d][dm] bf16 this context's rows of LayerWeights::wk
 *   k_pre_out [nseq][T][kv_heads][d] bf16(x . wk^T) (fp32 accumulation) -- the
 *   k_pre the gate was evaluated on; the rest as wgkv_gate_score.  bf16
 *   contexts with d = hidden = 128 and dm a multiple of 64 (WGKV_ENOTSUP). */
int wgkv_gate_score_proj(wgkv_ctx* ctx, int layer, int nseq, long T, long pos0, const void* x, const void* wk, int dm,
                         void* k_pre_out, void* k_post_out, float* g_out, uint8_t* bits_out, int64_t* near_idx,
                         int near_cap, int* near_count);

/* ---- K2: HeadCache::prefill_populate (kvstore.cpp:160-203) ---------------
 * Warp-scan compaction: admitted rows j < T-W appended to the paged Global
 * cache in ascending order, rows [T-W, T) into the Local ring slots 0.. .
 * Requires empty caches for the slots (WGKV_ESTATE otherwise). */
int wgkv_admit_prefill(wgkv_ctx* ctx, int layer, int seq0, int nseq, long T, const void* k_post, const void* v,
                       const float* g, const uint8_t* bits);

/* ---- K3: build_vs_mask + attn_vertical_slash (attention.cpp:116-153) -----
 * RoPE(q) then, per query tile, the admitted Global prefix (read in place
 * from the pages K2 filled) plus the band [i0-W+1, i0+tile-1] of k_post/v
 * with per-element masks allowed(i,j) = j<=i && (i-j<W || bits[j]).  Must
 * follow wgkv_admit_prefill for the same slots and bits (it reuses K2's
 * prefix counts). */
int wgkv_vs_prefill(wgkv_ctx* ctx, int layer, int seq0, int nseq, long T, const void* q, const void* k_post,
                    const void* v, const uint8_t* bits, void* out);

/* Session::prefill layer body (engine.cpp:188-257 minus projections/MLP):
 * K1 + K2 + K3 in one stream-ordered call. g_out/bits_out optional. */
int wgkv_prefill_layer(wgkv_ctx* ctx, int layer, int seq0, int nseq, long T, const void* q, const void* k_pre,
                       const void* v, const float* forced_g, void* out, float* g_out, uint8_t* bits_out);

/* ---- decode (Session::decode_step, engine.cpp:291-327) -------------------
 * K1(T=1, exact fp64) + K4: RoPE + gate + HeadCache::local_write with lazy
 * promotion (kvstore.cpp:122-158) for the token at position tokens_seen.
 *   k_pre, v [nseq][kv_heads][d]; events_out (optional, device int32
 *   [nseq][kv_heads]): 0 none, 1 promoted, 2 dropped, -1 failed (out of
 *   pages, latched; the head is left unchanged); g_out optional float. */
int wgkv_decode_step_kv(wgkv_ctx* ctx, int layer, int seq0, int nseq, const void* k_pre, const void* v,
                        const float* forced_g, float* g_out, int32_t* events_out);
/* K5 (+K6 when topk_budget > 0): gather-free split-KV attention over the
 * Global and Local pages in place (HeadCache::gather + attn_ragged,
 * kvstore.cpp:205-241, attention.cpp:155-180; select_topk_pages,
 * engine.cpp:36-84).  q [nseq][q_heads][d] pre-RoPE; out [nseq][q_heads][d]. */
int wgkv_decode_attn(wgkv_ctx* ctx, int layer, int seq0, int nseq, const void* q, void* out);
int wgkv_decode_layer(wgkv_ctx* ctx, int layer, int seq0, int nseq, const void* q, const void* k_pre, const void* v,
                      const float* forced_g, void* out, float* g_out, int32_t* events_out);

/* GateTrace of one decode step (records.hpp:11-29; engine.cpp:300-305 records
 * g and g >= tau for every decoded token).  Device pointers, [nseq][kv_heads],
 * any may be NULL.  The decode gate is evaluated in fp64 in the reference's
 * exact operation order (sequential dots, sequential z2 sum), so bits equal
 * the reference's except possibly where near_tau is set. */
typedef struct wgkv_decode_trace {
    float* g;          /* the new token's gate score (fp32 copy of the fp64 value) */
    uint8_t* bits;     /* g >= tau (admission bit the ring will promote on) */
    uint8_t* near_tau; /* 1 where |g - tau| < 1e-6: reported per north_star */
    int32_t* events;   /* ring victim: 0 none, 1 promoted, 2 dropped, -1 failed (ENOPAGES latched) */
} wgkv_decode_trace;
/* wgkv_decode_layer with the full trace (trace may be NULL) */
int wgkv_decode_layer_traced(wgkv_ctx* ctx, int layer, int seq0, int nseq, const void* q, const void* k_pre,
                             const void* v, const float* forced_g, void* out, const wgkv_decode_trace* trace);

/* ---- state, export, lifecycle (host, synchronising) ----------------------
 * lens[0..5] = local_len, local_ptr, global_len, tokens_seen, n_local_pages,
 * n_global_pages  (HeadCache accessors, kvstore.hpp:120-127) */
int wgkv_cache_state(wgkv_ctx* ctx, int layer, int seq, int kv_head, int64_t* lens);
/* HeadCache::gather to HOST buffers (any may be NULL): Global then Local in
 * position order; k/v as fp32 [rows][d]; sized from wgkv_cache_state. */
int wgkv_cache_export(wgkv_ctx* ctx, int layer, int seq, int kv_head, float* gk, float* gv, int64_t* gpos,
                      float* ggate, float* lk, float* lv, int64_t* lpos, float* lgate);
/* cache_stats (kvstore.cpp:253-267) over all heads of the slots: out[0] =
 * resident entries, out[1] = global entries, out[2] = tokens seen,
 * out[3] = pages allocated */
int wgkv_cache_stats(wgkv_ctx* ctx, int seq0, int nseq, int64_t* out);
/* cache_snapshot (kvstore.cpp:269-286) of sequence slot `seq`: lines
 * "layer head global|local pos gate" (gate %.17g of the stored fp32 value),
 * caches layer-major then kv head, Global then Local in position order.
 * *len = text length; buf (may be NULL) receives it NUL-terminated when
 * cap > *len, else WGKV_EINVAL. */
int wgkv_cache_snapshot(wgkv_ctx* ctx, int seq, char* buf, size_t cap, size_t* len);
/* HeadCache::release for every (layer, kv head) of the slots */
int wgkv_release(wgkv_ctx* ctx, int seq0, int nseq);
/* pool occupancy: out[0] = capacity, out[1] = free pages */
int wgkv_pool_info(wgkv_ctx* ctx, int64_t* out);

/* ---- C1: head-output all-gather of KV-head sharding (no reference
 * equivalent) -------------------------------------------
 * N contexts (one per GPU, one process per GPU or one process driving all),
 * rank r created with kv_head_offset = r * kv_heads, own the q heads
 * [r * q_heads, (r + 1) * q_heads).  wgkv_allgather_heads rebuilds Session's
 * concat layout on every rank: full_out[s][t][p][:] = q head p's output
 * (engine.cpp:234-238), full_out [nseq][T][N * q_heads][d] (cfg.dtype), from
 * each rank's local_out [nseq][T][q_heads][d] (wgkv_vs_prefill /
 * wgkv_decode_layer output; decode: T = 1).  NCCL over NVLink into a staging
 * buffer, then an assemble kernel.  async = 0: on the context stream;
 * async = 1: on the context's comm stream after the work enqueued so far, so
 * the caller's next layer overlaps it -- wgkv_comm_join orders the context
 * stream after it (before full_out is read or local_out reused).  Without a
 * communicator (single device) it is a copy.  NCCL is loaded at run time. */
int wgkv_comm_unique_id(uint8_t* id128);                         /* ncclGetUniqueId, on one rank */
int wgkv_comm_init(wgkv_ctx* ctx, const uint8_t* id128, int world, int rank); /* ncclCommInitRank */
int wgkv_comm_attach(wgkv_ctx* ctx, void* nccl_comm, int world, int rank);   /* caller-owned ncclComm_t */
int wgkv_allgather_heads(wgkv_ctx* ctx, int nseq, long T, const void* local_out, void* full_out, int async);
int wgkv_comm_join(wgkv_ctx* ctx);
/* ---- C1 over NVLink peer memory (no reference equivalent: the reference runs
 * every head in one process; this replaces its concat, engine.cpp:234-238,
 * across KV-head shards -- SURVEY.md §8e) ------------------------------------
 * A decode layer's head outputs are a few KB per rank: NCCL's all-gather is
 * latency-bound there.  Instead every rank owns an exchange region
 * (wgkv_peer_region_bytes) mapped into every other rank: wgkv_peer_alloc
 * allocates it and exports a cudaIpcMemHandle_t (64 bytes), the caller
 * exchanges the handles over its own plumbing, wgkv_peer_open maps them;
 * wgkv_peer_attach takes already-mapped pointers instead (one process driving
 * all GPUs with peer access, or regions on one GPU).  Protocol (LL, as NCCL's
 * low-latency one): a rank stores its rows local_out [rows][q_heads][d] as
 * 8-byte words {4 data bytes, flag} straight into every rank's region (NVLink
 * stores, no fence, no counter); a reader polls the words themselves and
 * writes the reference's concat layout [rows][world * q_heads][d]
 * (engine.cpp:234-238) into its result slot.  Exchanges rotate over 4 slots.
 * wgkv_peer_allgather_heads: a push kernel; wait = 1 also unpacks it now,
 * else it stays pending.  wgkv_peer_decode(ctx, 1): every wgkv_decode_layer
 * pushes its output rows from inside its merge (no extra kernel) and unpacks
 * the pending exchange in one of its CTAs, so exchange k is complete once
 * decode layer k + 1 (or wgkv_peer_wait) has run.  wgkv_peer_wait unpacks the
 * pending exchange.  wgkv_peer_result(back): this rank's result slot of the
 * exchange `back` exchanges ago (0 = the last), [rows][world * q_heads][d].
 * Contract (as NCCL's): every rank makes the same sequence of exchanges with
 * the same rows; a captured CUDA graph that replays exchanges holds a
 * multiple of 4 of them and leaves none pending; bf16 contexts.  wait_ranks
 * = world normally (fewer only to emulate a shard on one GPU: only ranks
 * [0, wait_ranks) are awaited and unpacked). */
int wgkv_peer_region_bytes(int world, long max_rows, long max_bulk_rows, int q_heads, int head_dim, int dtype,
                           size_t* bytes);
int wgkv_peer_alloc(wgkv_ctx* ctx, int world, long max_rows, long max_bulk_rows, uint8_t* ipc_handle64,
                    void** base);
int wgkv_peer_open(wgkv_ctx* ctx, int world, int rank, const uint8_t* handles /* world x 64 */, int wait_ranks);
int wgkv_peer_attach(wgkv_ctx* ctx, int world, int rank, long max_rows, long max_bulk_rows, void* const* bases,
                     int wait_ranks);
int wgkv_peer_allgather_heads(wgkv_ctx* ctx, long rows, const void* local_out, int wait);
int wgkv_peer_wait(wgkv_ctx* ctx);
int wgkv_peer_decode(wgkv_ctx* ctx, int on);
int wgkv_peer_result(wgkv_ctx* ctx, int back, void** ptr);
/* prefill: with a bulk part (max_bulk_rows > 0: two slots of [max_bulk_rows]
 * [world * q_heads][d]) and wgkv_peer_prefill(ctx, 1), wgkv_vs_prefill's
 * tcgen05 epilogue stores each output row into every rank's bulk slot as well
 * as into `out` (the all-gather fused into the attention: NVLink stores
 * overlap the tensor-core work), then a signal kernel (system fence, this
 * rank's flag into every region) and a wait kernel (every rank's flag here).
 * Rows are (seq - seq0) * T + t of the call.  wgkv_peer_bulk_result(back):
 * the bulk slot of the last (0) or previous (1) prefill exchange. */
int wgkv_peer_prefill(wgkv_ctx* ctx, int on);
int wgkv_peer_bulk_result(wgkv_ctx* ctx, int back, void** ptr);
/* ---- f3: output projection overlapped with the head all-gather -----------
 * Session's x[t] += Wo . concat[t] (engine.cpp:243-245 prefill, :331 decode)
 * on top of wgkv_allgather_heads: local_out [nseq][T][q_heads][d] (bf16, this
 * rank's heads), wo [dim][world * q_heads * d] bf16 row-major
 * (LayerWeights::wo, model.hpp), x [nseq][T][dim] fp32 residual stream,
 * updated in place.  With a communicator the rows go in chunks: the NCCL
 * all-gather + assembly of chunk c+1 (comm stream) overlaps the Wo GEMM of
 * chunk c (cuBLAS, bf16 tensor cores, fp32 accumulation; context stream).
 * Without one the local heads are the concat and only the GEMM runs.
 * bf16 contexts only (WGKV_ENOTSUP otherwise). */
int wgkv_output_proj(wgkv_ctx* ctx, int nseq, long T, const void* local_out, const void* wo, int dim, float* x);
/* the assembly step alone: rank-major [world][rows][blk_bytes] -> [rows][world * blk_bytes]
 * on `stream` (cudaStream_t); blk_bytes a multiple of 16 */
int wgkv_assemble_heads(int world, long rows, size_t blk_bytes, const void* rank_major, void* full_out,
                        void* stream);

/* vs_mask_pair_count (attention.cpp:182-191) of one head's bits, computed in
 * closed form on the host: sum_i min(i+1, W) + C(i-W+1). */
uint64_t wgkv_vs_pair_count(const uint8_t* bits, long T, long window);

#ifdef __cplusplus
}
#endif
#endif
