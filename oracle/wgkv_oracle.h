/*
 * wgkv_oracle.h -- CPU parity oracle for the WG-KV hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may include, link or
 * call this library: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, and only as the checker.
 *
 * This is a plain-C, fp64 restatement of the reference algorithm
 * (/root/reference/proj, C++20).  Every function cites the reference
 * file:line it follows.  Parity is pinned two ways (see tests/):
 *   1. the reference's own known-answer tests, restated in
 *      tests/test_oracle_golden.py, and
 *   2. golden vectors produced by the reference itself (oracle/_ref, compiled
 *      from /root/reference sources by oracle/Makefile) committed under
 *      tests/golden/ by tests/golden/make_golden.py.
 *
 * Status codes match include/wgkv_b200.h (WGKV_OK, WGKV_EINVAL, ...).
 */
#ifndef WGKV_ORACLE_H
#define WGKV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    WO_OK = 0,
    WO_EINVAL = 1,   /* std::invalid_argument in the reference */
    WO_ENOPAGES = 2, /* std::runtime_error("out of pages ...") */
    WO_ESTATE = 3,   /* std::logic_error (lifecycle, double free, non-empty populate) */
    WO_ERUNTIME = 4  /* std::runtime_error (fully masked row, empty KV) */
};

/* ---- numerics (numerics.hpp:53-79, numerics.cpp:13-99) ---------------- */
typedef struct {
    uint64_t mt[312];
    int mti;
    int has_spare;
    double spare;
} wo_rng;

void wo_rng_init(wo_rng* r, uint64_t seed);
uint64_t wo_rng_next(wo_rng* r);
double wo_rng_uniform(wo_rng* r);
long wo_rng_uniform_int(wo_rng* r, long lo, long hi);
double wo_rng_gaussian(wo_rng* r);
/* n draws of scale * gaussian() from a fresh Rng(seed) */
void wo_gaussian_fill(uint64_t seed, double scale, double* out, long n);
void wo_uniform_fill(uint64_t seed, double* out, long n);
void wo_uniform_int_fill(uint64_t seed, long lo, long hi, long* out, long n);

double wo_gelu(double x);
double wo_sigmoid(double x);
double wo_dot(const double* a, const double* b, long n);
int wo_rope(double* k, int head_dim, long position, double base, double sign);
int wo_softmax(const double* logits, long n, double* out);
/* wo_rope over rows [rows][head_dim], row r at position pos0 + r (sign +1) */
int wo_rope_rows(double* k, long rows, int head_dim, long pos0, double base);

/* ---- gating (gating.cpp:49-59, 149-190) --------------------------------
 * One parameter block per (layer, kv-head) in layer-major order, each of
 * wo_gate_block_len(d, hidden) doubles laid out as
 *   W1[hidden][2d] | b1[hidden] | w2[hidden] | b2
 * which is exactly the per-block order of the ".wgkv" v1 file.
 */
long wo_gate_block_len(int head_dim, int hidden);
int wo_gate_random_init(int layers, int heads, int head_dim, int hidden, uint64_t seed, double w_std,
                        double b2_init, double* bank_out);
double wo_gate_forward(const double* block, int head_dim, int hidden, const double* feature);
int wo_gate_forward_batch(const double* block, int head_dim, int hidden, const double* k_pre,
                          const double* k_post, long t, double* g_out);
int wo_binarize(const double* g, long n, double tau, uint8_t* bits_out);
/* gate bank file I/O, ".wgkv" v1 (gating.cpp:107-147) */
int wo_gate_save(const char* path, int layers, int heads, int head_dim, int hidden, const double* bank);
int wo_gate_load_header(const char* path, int* layers, int* heads, int* head_dim, int* hidden);
int wo_gate_load(const char* path, double* bank_out, long bank_len);

/* ---- attention (attention.cpp:19-36, 116-191) -------------------------- */
int wo_attn_dense(const double* q, long tq, const double* k, const double* v, long tk, int d, double scale,
                  long causal_offset, double* out, uint64_t* score_evals);
int wo_attn_vertical_slash(const double* q, long tq, const double* k, const double* v, long tk, int d,
                           double scale, long causal_offset, long window, const uint8_t* admitted, double* out,
                           uint64_t* score_evals);
uint64_t wo_vs_pair_count(long window, const uint8_t* admitted, long query_count, long key_count,
                          long causal_offset);
int wo_attn_ragged(const double* q, const double* gk, const double* gv, long g_rows, const double* lk,
                   const double* lv, long l_rows, int d, double scale, double* out, uint64_t* score_evals);

/* ---- paged dual cache (kvstore.cpp:9-286) ------------------------------- */
typedef struct wo_pool wo_pool;
typedef struct wo_head wo_head;

wo_pool* wo_pool_create(int page_size, int head_dim, long capacity_pages);
void wo_pool_destroy(wo_pool* p);
long wo_pool_free_pages(const wo_pool* p);
long wo_pool_capacity(const wo_pool* p);
/* region 0 = local, 1 = global; returns page id or -WO_ENOPAGES */
int wo_pool_alloc(wo_pool* p, int layer, int head, int region);
int wo_pool_free(wo_pool* p, int page);
int wo_pool_owner(const wo_pool* p, int page, int* layer, int* head, int* region, int* in_use);
/* direct slot access, used by tests that plant keys (test_engine.cpp:306-317) */
double* wo_pool_k_slot(wo_pool* p, int page, int slot);

wo_head* wo_head_create(int layer, int head, long window);
void wo_head_destroy(wo_head* h);
/* returns 0 none, 1 promoted, 2 dropped, or -status */
int wo_local_write(wo_head* h, wo_pool* p, const double* k, const double* v, double gate, double tau, long position);
int wo_prefill_populate(wo_head* h, wo_pool* p, const double* keys, const double* values, const double* gates,
                        long t_total, double tau, long first_position);
/* lens[0..5] = local_len, local_ptr, global_len, tokens_seen, n_local_pages, n_global_pages */
void wo_head_state(const wo_head* h, long* lens);
int wo_head_pages(const wo_head* h, int* local_pages, int* global_pages);
/* position-ordered materialisation; any output pointer may be NULL */
int wo_gather(const wo_head* h, const wo_pool* p, double* gk, double* gv, long* gpos, double* ggate, double* lk,
              double* lv, long* lpos, double* lgate);
int wo_release(wo_head* h, wo_pool* p);

/* select_topk_pages (engine.cpp:36-84): logical_pages_out gets min(budget, pages)
 * logical ids ascending; k/v gets the selected rows; *entries the row count.
 * Any of logical_pages_out/k_out/v_out may be NULL. */
int wo_select_topk_pages(const double* q, const wo_head* h, const wo_pool* p, long budget, long* logical_pages_out,
                         long* n_selected, double* k_out, double* v_out, long* entries);

/* ---- path-level session (engine.cpp:153-341 minus the model) ------------
 * Mirrors Session::prefill / decode_step for ONE sequence with the toy model's
 * projections removed: callers pass pre-RoPE q/k and v per layer, exactly the
 * tensors engine.cpp:191-198/226-228 produce.  Policy: MLP gates unless
 * forced_gates != NULL (effective_gate override, engine.cpp:126-151).
 * topk_budget > 0 selects the wgkv_plus_topk decode path (engine.cpp:320-324).
 */
typedef struct wo_session wo_session;
wo_session* wo_session_create(int layers, int q_heads, int kv_heads, int head_dim, int hidden, long window,
                              double tau, double rope_base, int page_size, long capacity_pages, long topk_budget,
                              const double* gate_bank);
void wo_session_destroy(wo_session* s);
/* q_pre [t][q_heads][d], k_pre/v [t][kv_heads][d] -> out [t][q_heads][d];
 * g_out/bits_out [kv_heads][t] (may be NULL) */
int wo_session_prefill_layer(wo_session* s, int layer, const double* q_pre, const double* k_pre, const double* v,
                             long t, const double* forced_gates, double* out, double* g_out, uint8_t* bits_out,
                             uint64_t* score_evals);
/* one token at position = tokens seen by this layer; events_out [kv_heads] */
int wo_session_decode_layer(wo_session* s, int layer, const double* q_pre, const double* k_pre, const double* v,
                            const double* forced_gates, double* out, double* g_out, int* events_out,
                            uint64_t* score_evals);
wo_head* wo_session_head(wo_session* s, int layer, int kv_head);
wo_pool* wo_session_pool(wo_session* s);

#ifdef __cplusplus
}
#endif
#endif
