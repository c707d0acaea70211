/*
 * wgkv_oracle.c -- plain-C fp64 restatement of the WG-KV reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see wgkv_oracle.h).  Citations are
 * /root/reference/proj/<file>:<line>.  Floating-point expressions keep the
 * reference's evaluation order so that results are bitwise identical with the
 * reference compiled by the same gcc/libm (tests/test_oracle_vs_ref.py checks
 * exactly that against oracle/_ref).
 */
#include "wgkv_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================= */
/* numerics                                                                 */
/* ======================================================================= */

/* std::mt19937_64 (numerics.hpp:55-57 uses the standard engine). */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x7FFFFFFFULL

void wo_rng_init(wo_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
    r->has_spare = 0;
    r->spare = 0.0;
}

static void mt_twist(wo_rng* r) {
    for (int i = 0; i < MT_N; ++i) {
        uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
}

uint64_t wo_rng_next(wo_rng* r) {
    if (r->mti >= MT_N) mt_twist(r);
    uint64_t y = r->mt[r->mti++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* Rng::uniform (numerics.hpp:63) */
double wo_rng_uniform(wo_rng* r) { return (double)(wo_rng_next(r) >> 11) * 0x1.0p-53; }

/* Rng::uniform_int (numerics.hpp:68-70) */
long wo_rng_uniform_int(wo_rng* r, long lo, long hi) {
    return lo + (long)(wo_rng_next(r) % (uint64_t)(hi - lo));
}

/* Rng::gaussian, Box-Muller with a cached spare (numerics.cpp:79-92) */
double wo_rng_gaussian(wo_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    const double u1 = ((double)(wo_rng_next(r) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = wo_rng_uniform(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
    r->spare = rad * sin(theta);
    r->has_spare = 1;
    return rad * cos(theta);
}

void wo_gaussian_fill(uint64_t seed, double scale, double* out, long n) {
    wo_rng r;
    wo_rng_init(&r, seed);
    for (long i = 0; i < n; ++i) out[i] = scale * wo_rng_gaussian(&r);
}

void wo_uniform_int_fill(uint64_t seed, long lo, long hi, long* out, long n) {
    wo_rng r;
    wo_rng_init(&r, seed);
    for (long i = 0; i < n; ++i) out[i] = wo_rng_uniform_int(&r, lo, hi);
}

void wo_uniform_fill(uint64_t seed, double* out, long n) {
    wo_rng r;
    wo_rng_init(&r, seed);
    for (long i = 0; i < n; ++i) out[i] = wo_rng_uniform(&r);
}

/* gelu: x * Phi(x) with Phi via erf (numerics.cpp:33-36) */
double wo_gelu(double x) { return x * 0.5 * (1.0 + erf(x * 1.41421356237309504880168872420969808 * 0.5)); }

/* branchy overflow-safe logistic (numerics.cpp:44-48) */
double wo_sigmoid(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    const double e = exp(x);
    return e / (1.0 + e);
}

/* sequential inner product (numerics.cpp:94-99) */
double wo_dot(const double* a, const double* b, long n) {
    double s = 0.0;
    for (long i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* interleaved-pair rotary embedding (numerics.cpp:50-63) */
int wo_rope(double* k, int head_dim, long position, double base, double sign) {
    if (head_dim % 2 != 0 || head_dim <= 0) return WO_EINVAL;
    for (int i = 0; i * 2 < head_dim; ++i) {
        const double freq = pow(base, -2.0 * i / head_dim);
        const double angle = sign * (double)position * freq;
        const double c = cos(angle);
        const double s = sin(angle);
        const double a = k[2 * i];
        const double b = k[2 * i + 1];
        k[2 * i] = a * c - b * s;
        k[2 * i + 1] = a * s + b * c;
    }
    return WO_OK;
}

/* apply_rope_inplace over consecutive rows (numerics.cpp:71-77): row r of
 * [rows][head_dim] at position pos0 + r */
int wo_rope_rows(double* k, long rows, int head_dim, long pos0, double base) {
    for (long r = 0; r < rows; ++r) {
        const int st = wo_rope(k + r * head_dim, head_dim, pos0 + r, base, 1.0);
        if (st != WO_OK) return st;
    }
    return WO_OK;
}

/* max-subtracted softmax; -inf -> exact 0; all -inf is an error (numerics.cpp:13-31) */
int wo_softmax(const double* logits, long n, double* out) {
    if (n <= 0) return WO_EINVAL;
    double mx = -INFINITY;
    for (long i = 0; i < n; ++i) {
        if (isnan(logits[i])) return WO_EINVAL;
        if (logits[i] > mx) mx = logits[i];
    }
    if (isinf(mx) && mx < 0) return WO_ERUNTIME;
    double sum = 0.0;
    for (long i = 0; i < n; ++i) {
        out[i] = exp(logits[i] - mx);
        sum += out[i];
    }
    for (long i = 0; i < n; ++i) out[i] /= sum;
    return WO_OK;
}

/* ======================================================================= */
/* gating                                                                   */
/* ======================================================================= */

long wo_gate_block_len(int head_dim, int hidden) { return (long)hidden * 2 * head_dim + 2L * hidden + 1; }

/* GateBank::random_init: one Rng(seed) stream, per block W1 then w2, b1 = 0,
 * b2 = b2_init (gating.cpp:49-59) */
int wo_gate_random_init(int layers, int heads, int head_dim, int hidden, uint64_t seed, double w_std,
                        double b2_init, double* bank) {
    if (layers < 1 || heads < 1 || head_dim < 1 || hidden < 1) return WO_EINVAL;
    const long blen = wo_gate_block_len(head_dim, hidden);
    const long w1n = (long)hidden * 2 * head_dim;
    wo_rng r;
    wo_rng_init(&r, seed);
    for (long b = 0; b < (long)layers * heads; ++b) {
        double* blk = bank + b * blen;
        for (long i = 0; i < w1n; ++i) blk[i] = w_std * wo_rng_gaussian(&r);
        for (int i = 0; i < hidden; ++i) blk[w1n + i] = 0.0;
        for (int i = 0; i < hidden; ++i) blk[w1n + hidden + i] = w_std * wo_rng_gaussian(&r);
        blk[w1n + 2 * hidden] = b2_init;
    }
    return WO_OK;
}

/* gate_forward: z2 = b2 + sum_h w2[h]*gelu(W1[h].x + b1[h]); sigmoid; clamp
 * into (0,1) (gating.cpp:158-171) */
double wo_gate_forward(const double* blk, int head_dim, int hidden, const double* feature) {
    const long fdim = 2L * head_dim;
    const double* w1 = blk;
    const double* b1 = blk + (long)hidden * fdim;
    const double* w2 = b1 + hidden;
    double z2 = w2[hidden];
    for (int h = 0; h < hidden; ++h) {
        const double z1 = wo_dot(w1 + (long)h * fdim, feature, fdim) + b1[h];
        z2 += w2[h] * wo_gelu(z1);
    }
    double g = wo_sigmoid(z2);
    const double lo = 5e-324, hi = nextafter(1.0, 0.0);
    if (g < lo) g = lo;
    if (g > hi) g = hi;
    return g;
}

/* gate_forward_batch over rows of [k_pre ; k_post] (gating.cpp:149-156, 173-182) */
int wo_gate_forward_batch(const double* blk, int head_dim, int hidden, const double* k_pre, const double* k_post,
                          long t, double* g_out) {
    double* feature = (double*)malloc(sizeof(double) * 2 * (size_t)head_dim);
    if (!feature) return WO_ERUNTIME;
    for (long i = 0; i < t; ++i) {
        memcpy(feature, k_pre + i * head_dim, sizeof(double) * (size_t)head_dim);
        memcpy(feature + head_dim, k_post + i * head_dim, sizeof(double) * (size_t)head_dim);
        g_out[i] = wo_gate_forward(blk, head_dim, hidden, feature);
    }
    free(feature);
    return WO_OK;
}

/* bit = g >= tau, tau must lie in (0,1) (gating.cpp:184-190) */
int wo_binarize(const double* g, long n, double tau, uint8_t* bits) {
    if (!(tau > 0.0 && tau < 1.0)) return WO_EINVAL;
    for (long i = 0; i < n; ++i) bits[i] = g[i] >= tau ? 1 : 0;
    return WO_OK;
}

/* ".wgkv" v1: magic, u32 version/L/H/head_dim/hidden, f64 blocks, little
 * endian (gating.cpp:107-147).  x86-64 is little endian, so fwrite works. */
int wo_gate_save(const char* path, int layers, int heads, int head_dim, int hidden, const double* bank) {
    FILE* f = fopen(path, "wb");
    if (!f) return WO_ERUNTIME;
    const uint32_t hdr[5] = {1u, (uint32_t)layers, (uint32_t)heads, (uint32_t)head_dim, (uint32_t)hidden};
    fwrite("WGKV", 1, 4, f);
    fwrite(hdr, 4, 5, f);
    const size_t n = (size_t)layers * heads * (size_t)wo_gate_block_len(head_dim, hidden);
    const size_t w = fwrite(bank, sizeof(double), n, f);
    fclose(f);
    return w == n ? WO_OK : WO_ERUNTIME;
}

int wo_gate_load_header(const char* path, int* layers, int* heads, int* head_dim, int* hidden) {
    FILE* f = fopen(path, "rb");
    if (!f) return WO_ERUNTIME;
    char magic[4];
    uint32_t hdr[5];
    int ok = fread(magic, 1, 4, f) == 4 && memcmp(magic, "WGKV", 4) == 0;
    ok = ok && fread(hdr, 4, 5, f) == 5 && hdr[0] == 1u;
    fclose(f);
    if (!ok) return WO_ERUNTIME;
    *layers = (int)hdr[1];
    *heads = (int)hdr[2];
    *head_dim = (int)hdr[3];
    *hidden = (int)hdr[4];
    return WO_OK;
}

int wo_gate_load(const char* path, double* bank, long bank_len) {
    int L, H, d, hid;
    int st = wo_gate_load_header(path, &L, &H, &d, &hid);
    if (st) return st;
    const long n = (long)L * H * wo_gate_block_len(d, hid);
    if (n != bank_len) return WO_EINVAL;
    FILE* f = fopen(path, "rb");
    if (!f) return WO_ERUNTIME;
    fseek(f, 24, SEEK_SET);
    const size_t r = fread(bank, sizeof(double), (size_t)n, f);
    fclose(f);
    return r == (size_t)n ? WO_OK : WO_ERUNTIME;
}

/* ======================================================================= */
/* attention                                                                */
/* ======================================================================= */

/* dense causal attention (attention.cpp:19-36) */
int wo_attn_dense(const double* q, long tq, const double* k, const double* v, long tk, int d, double scale,
                  long causal_offset, double* out, uint64_t* score_evals) {
    double* logits = (double*)malloc(sizeof(double) * (size_t)(tk > 0 ? tk : 1));
    double* w = (double*)malloc(sizeof(double) * (size_t)(tk > 0 ? tk : 1));
    int st = WO_OK;
    memset(out, 0, sizeof(double) * (size_t)tq * d);
    for (long i = 0; i < tq && st == WO_OK; ++i) {
        long limit = causal_offset + i;
        if (tk - 1 < limit) limit = tk - 1;
        if (limit < 0) {
            st = WO_ERUNTIME;
            break;
        }
        for (long j = 0; j <= limit; ++j) logits[j] = scale * wo_dot(q + i * d, k + j * d, d);
        if (score_evals) *score_evals += (uint64_t)(limit + 1);
        st = wo_softmax(logits, limit + 1, w);
        for (long j = 0; j <= limit && st == WO_OK; ++j)
            for (int c = 0; c < d; ++c) out[i * d + c] += w[j] * v[j * d + c];
    }
    free(logits);
    free(w);
    return st;
}

/* allowed(i,j) = (i - j) < window || admitted[j]  (attention.hpp:31-36) */
static int vs_allowed(long window, const uint8_t* admitted, long i, long j) {
    return (i - j) < window || admitted[j] != 0;
}

/* attn_vertical_slash: softmax over the permitted j <= min(i, tk-1) only
 * (attention.cpp:123-153) */
int wo_attn_vertical_slash(const double* q, long tq, const double* k, const double* v, long tk, int d,
                           double scale, long causal_offset, long window, const uint8_t* admitted, double* out,
                           uint64_t* score_evals) {
    if (window < 1) return WO_EINVAL;
    long* permitted = (long*)malloc(sizeof(long) * (size_t)(tk > 0 ? tk : 1));
    double* logits = (double*)malloc(sizeof(double) * (size_t)(tk > 0 ? tk : 1));
    double* w = (double*)malloc(sizeof(double) * (size_t)(tk > 0 ? tk : 1));
    int st = WO_OK;
    memset(out, 0, sizeof(double) * (size_t)tq * d);
    for (long r = 0; r < tq && st == WO_OK; ++r) {
        const long i = causal_offset + r;
        long limit = i < tk - 1 ? i : tk - 1;
        long n = 0;
        for (long j = 0; j <= limit; ++j) {
            if (!vs_allowed(window, admitted, i, j)) continue;
            permitted[n] = j;
            logits[n] = scale * wo_dot(q + r * d, k + j * d, d);
            ++n;
        }
        if (n == 0) {
            st = WO_ERUNTIME;
            break;
        }
        if (score_evals) *score_evals += (uint64_t)n;
        st = wo_softmax(logits, n, w);
        for (long m = 0; m < n && st == WO_OK; ++m) {
            const double* vr = v + permitted[m] * d;
            for (int c = 0; c < d; ++c) out[r * d + c] += w[m] * vr[c];
        }
    }
    free(permitted);
    free(logits);
    free(w);
    return st;
}

/* exact permitted-pair count (attention.cpp:182-191) */
uint64_t wo_vs_pair_count(long window, const uint8_t* admitted, long query_count, long key_count,
                          long causal_offset) {
    uint64_t count = 0;
    for (long r = 0; r < query_count; ++r) {
        const long i = causal_offset + r;
        const long limit = key_count - 1 < i ? key_count - 1 : i;
        for (long j = 0; j <= limit; ++j)
            if (vs_allowed(window, admitted, i, j)) ++count;
    }
    return count;
}

/* one query over global || local (attention.cpp:155-180) */
int wo_attn_ragged(const double* q, const double* gk, const double* gv, long g_rows, const double* lk,
                   const double* lv, long l_rows, int d, double scale, double* out, uint64_t* score_evals) {
    const long total = g_rows + l_rows;
    if (total == 0) return WO_ERUNTIME;
    if (l_rows == 0) return WO_EINVAL;
    double* logits = (double*)malloc(sizeof(double) * (size_t)total);
    double* w = (double*)malloc(sizeof(double) * (size_t)total);
    for (long j = 0; j < g_rows; ++j) logits[j] = scale * wo_dot(q, gk + j * d, d);
    for (long j = 0; j < l_rows; ++j) logits[g_rows + j] = scale * wo_dot(q, lk + j * d, d);
    if (score_evals) *score_evals += (uint64_t)total;
    int st = wo_softmax(logits, total, w);
    for (int c = 0; c < d; ++c) out[c] = 0.0;
    if (st == WO_OK) {
        for (long j = 0; j < g_rows; ++j)
            for (int c = 0; c < d; ++c) out[c] += w[j] * gv[j * d + c];
        for (long j = 0; j < l_rows; ++j)
            for (int c = 0; c < d; ++c) out[c] += w[g_rows + j] * lv[j * d + c];
    }
    free(logits);
    free(w);
    return st;
}

/* ======================================================================= */
/* paged dual cache                                                         */
/* ======================================================================= */

struct wo_pool {
    int page_size, head_dim;
    long capacity;
    double *k, *v, *gates; /* [capacity][page_size][(head_dim)] */
    long* positions;       /* [capacity][page_size] */
    int *owner_layer, *owner_head, *owner_region, *in_use;
    int* free_stack; /* LIFO; first alloc returns page 0 (kvstore.cpp:9-21) */
    long n_free;
};

wo_pool* wo_pool_create(int page_size, int head_dim, long capacity) {
    if (page_size < 1 || head_dim < 1 || capacity < 0) return NULL;
    wo_pool* p = (wo_pool*)calloc(1, sizeof(wo_pool));
    const size_t slots = (size_t)capacity * page_size;
    p->page_size = page_size;
    p->head_dim = head_dim;
    p->capacity = capacity;
    p->k = (double*)calloc(slots * head_dim + 1, sizeof(double));
    p->v = (double*)calloc(slots * head_dim + 1, sizeof(double));
    p->gates = (double*)calloc(slots + 1, sizeof(double));
    p->positions = (long*)malloc(sizeof(long) * (slots + 1));
    for (size_t i = 0; i < slots; ++i) p->positions[i] = -1;
    p->owner_layer = (int*)calloc((size_t)capacity + 1, sizeof(int));
    p->owner_head = (int*)calloc((size_t)capacity + 1, sizeof(int));
    p->owner_region = (int*)calloc((size_t)capacity + 1, sizeof(int));
    p->in_use = (int*)calloc((size_t)capacity + 1, sizeof(int));
    p->free_stack = (int*)malloc(sizeof(int) * ((size_t)capacity + 1));
    for (long i = 0; i < capacity; ++i) {
        p->free_stack[i] = (int)(capacity - 1 - i);
        p->owner_layer[i] = p->owner_head[i] = -1;
    }
    p->n_free = capacity;
    return p;
}

void wo_pool_destroy(wo_pool* p) {
    if (!p) return;
    free(p->k);
    free(p->v);
    free(p->gates);
    free(p->positions);
    free(p->owner_layer);
    free(p->owner_head);
    free(p->owner_region);
    free(p->in_use);
    free(p->free_stack);
    free(p);
}

long wo_pool_free_pages(const wo_pool* p) { return p->n_free; }
long wo_pool_capacity(const wo_pool* p) { return p->capacity; }

/* KvPool::alloc_page (kvstore.cpp:23-34) */
int wo_pool_alloc(wo_pool* p, int layer, int head, int region) {
    if (p->n_free == 0) return -WO_ENOPAGES;
    const int page = p->free_stack[--p->n_free];
    p->owner_layer[page] = layer;
    p->owner_head[page] = head;
    p->owner_region[page] = region;
    p->in_use[page] = 1;
    return page;
}

/* KvPool::free_page (kvstore.cpp:39-46) */
int wo_pool_free(wo_pool* p, int page) {
    if (page < 0 || page >= p->capacity) return WO_EINVAL;
    if (!p->in_use[page]) return WO_ESTATE;
    p->in_use[page] = 0;
    p->owner_layer[page] = p->owner_head[page] = -1;
    p->owner_region[page] = 0;
    for (int s = 0; s < p->page_size; ++s) p->positions[(size_t)page * p->page_size + s] = -1;
    p->free_stack[p->n_free++] = page;
    return WO_OK;
}

int wo_pool_owner(const wo_pool* p, int page, int* layer, int* head, int* region, int* in_use) {
    if (page < 0 || page >= p->capacity) return WO_EINVAL;
    *layer = p->owner_layer[page];
    *head = p->owner_head[page];
    *region = p->owner_region[page];
    *in_use = p->in_use[page];
    return WO_OK;
}

static size_t slot_index(const wo_pool* p, int page, int slot) { return (size_t)page * p->page_size + slot; }

double* wo_pool_k_slot(wo_pool* p, int page, int slot) {
    if (page < 0 || page >= p->capacity || slot < 0 || slot >= p->page_size || !p->in_use[page]) return NULL;
    return p->k + slot_index(p, page, slot) * p->head_dim;
}

struct wo_head {
    int layer, head;
    long window, local_len, local_ptr, global_len, tokens_seen;
    int* local_pages;
    long n_local, cap_local;
    int* global_pages;
    long n_global, cap_global;
};

wo_head* wo_head_create(int layer, int head, long window) {
    if (window < 1) return NULL; /* kvstore.cpp:98-100 */
    wo_head* h = (wo_head*)calloc(1, sizeof(wo_head));
    h->layer = layer;
    h->head = head;
    h->window = window;
    return h;
}

void wo_head_destroy(wo_head* h) {
    if (!h) return;
    free(h->local_pages);
    free(h->global_pages);
    free(h);
}

static void push_page(int** arr, long* n, long* cap, int page) {
    if (*n == *cap) {
        *cap = *cap ? *cap * 2 : 8;
        *arr = (int*)realloc(*arr, sizeof(int) * (size_t)*cap);
    }
    (*arr)[(*n)++] = page;
}

/* ring slot; allocates backing pages on first touch (kvstore.cpp:102-107) */
static int local_slot(wo_head* h, wo_pool* p, long ring, int* page, int* slot) {
    const long pidx = ring / p->page_size;
    while (h->n_local <= pidx) {
        const int pg = wo_pool_alloc(p, h->layer, h->head, 0);
        if (pg < 0) return -pg;
        push_page(&h->local_pages, &h->n_local, &h->cap_local, pg);
    }
    *page = h->local_pages[pidx];
    *slot = (int)(ring % p->page_size);
    return WO_OK;
}

/* next Global slot; new page when the last is full (kvstore.cpp:115-120) */
static int global_append_slot(wo_head* h, wo_pool* p, int* page, int* slot) {
    const long pidx = h->global_len / p->page_size;
    if (h->n_global <= pidx) {
        const int pg = wo_pool_alloc(p, h->layer, h->head, 1);
        if (pg < 0) return -pg;
        push_page(&h->global_pages, &h->n_global, &h->cap_global, pg);
    }
    *page = h->global_pages[pidx];
    *slot = (int)(h->global_len % p->page_size);
    return WO_OK;
}

static void copy_slot(wo_pool* p, int dp, int ds, const double* k, const double* v, double gate, long pos) {
    const size_t si = slot_index(p, dp, ds);
    memcpy(p->k + si * p->head_dim, k, sizeof(double) * (size_t)p->head_dim);
    memcpy(p->v + si * p->head_dim, v, sizeof(double) * (size_t)p->head_dim);
    p->gates[si] = gate;
    p->positions[si] = pos;
}

/* HeadCache::local_write with lazy promotion of the victim (kvstore.cpp:122-158) */
int wo_local_write(wo_head* h, wo_pool* p, const double* k, const double* v, double gate, double tau, long position) {
    int event = 0, page, slot, st;
    st = local_slot(h, p, h->local_ptr, &page, &slot);
    if (st) return -st;
    if (h->local_len < h->window) {
        ++h->local_len;
    } else {
        const size_t vi = slot_index(p, page, slot);
        event = p->gates[vi] >= tau ? 1 : 2;
        if (event == 1) { /* promote (kvstore.cpp:122-133) */
            int gp, gs;
            st = global_append_slot(h, p, &gp, &gs);
            if (st) return -st;
            copy_slot(p, gp, gs, p->k + vi * p->head_dim, p->v + vi * p->head_dim, p->gates[vi], p->positions[vi]);
            ++h->global_len;
        }
    }
    copy_slot(p, page, slot, k, v, gate, position);
    h->local_ptr = (h->local_ptr + 1) % h->window;
    ++h->tokens_seen;
    return event;
}

/* HeadCache::prefill_populate (kvstore.cpp:160-203) */
int wo_prefill_populate(wo_head* h, wo_pool* p, const double* keys, const double* values, const double* gates,
                        long t_total, double tau, long first_position) {
    if (h->local_len != 0 || h->global_len != 0 || h->tokens_seen != 0) return WO_ESTATE;
    const int d = p->head_dim;
    const long window_start = t_total - h->window > 0 ? t_total - h->window : 0;
    int page, slot, st;
    for (long j = 0; j < window_start; ++j) {
        if (gates[j] < tau) continue;
        st = global_append_slot(h, p, &page, &slot);
        if (st) return st;
        copy_slot(p, page, slot, keys + j * d, values + j * d, gates[j], first_position + j);
        ++h->global_len;
    }
    for (long j = window_start; j < t_total; ++j) {
        st = local_slot(h, p, h->local_ptr, &page, &slot);
        if (st) return st;
        copy_slot(p, page, slot, keys + j * d, values + j * d, gates[j], first_position + j);
        ++h->local_len;
        h->local_ptr = (h->local_ptr + 1) % h->window;
    }
    h->tokens_seen = t_total;
    return WO_OK;
}

void wo_head_state(const wo_head* h, long* lens) {
    lens[0] = h->local_len;
    lens[1] = h->local_ptr;
    lens[2] = h->global_len;
    lens[3] = h->tokens_seen;
    lens[4] = h->n_local;
    lens[5] = h->n_global;
}

int wo_head_pages(const wo_head* h, int* local_pages, int* global_pages) {
    if (local_pages) memcpy(local_pages, h->local_pages, sizeof(int) * (size_t)h->n_local);
    if (global_pages) memcpy(global_pages, h->global_pages, sizeof(int) * (size_t)h->n_global);
    return WO_OK;
}

/* HeadCache::gather: Global by logical index, Local unrolled oldest-first
 * from local_ptr once the ring is full (kvstore.cpp:205-241) */
int wo_gather(const wo_head* h, const wo_pool* p, double* gk, double* gv, long* gpos, double* ggate, double* lk,
              double* lv, long* lpos, double* lgate) {
    const int d = p->head_dim, ps = p->page_size;
    for (long g = 0; g < h->global_len; ++g) {
        const size_t si = slot_index(p, h->global_pages[g / ps], (int)(g % ps));
        if (gk) memcpy(gk + g * d, p->k + si * d, sizeof(double) * (size_t)d);
        if (gv) memcpy(gv + g * d, p->v + si * d, sizeof(double) * (size_t)d);
        if (gpos) gpos[g] = p->positions[si];
        if (ggate) ggate[g] = p->gates[si];
    }
    const long start = h->local_len < h->window ? 0 : h->local_ptr;
    for (long n = 0; n < h->local_len; ++n) {
        const long ring = (start + n) % h->window;
        const size_t si = slot_index(p, h->local_pages[ring / ps], (int)(ring % ps));
        if (lk) memcpy(lk + n * d, p->k + si * d, sizeof(double) * (size_t)d);
        if (lv) memcpy(lv + n * d, p->v + si * d, sizeof(double) * (size_t)d);
        if (lpos) lpos[n] = p->positions[si];
        if (lgate) lgate[n] = p->gates[si];
    }
    return WO_OK;
}

/* HeadCache::release (kvstore.cpp:243-251) */
int wo_release(wo_head* h, wo_pool* p) {
    for (long i = 0; i < h->n_local; ++i) wo_pool_free(p, h->local_pages[i]);
    for (long i = 0; i < h->n_global; ++i) wo_pool_free(p, h->global_pages[i]);
    h->n_local = h->n_global = 0;
    h->local_len = h->local_ptr = h->global_len = h->tokens_seen = 0;
    return WO_OK;
}

/* select_topk_pages: score = max slot q.k (unscaled); higher first, ties to
 * the older page; keep min(budget, pages); re-sort ascending (engine.cpp:36-84) */
typedef struct {
    double score;
    long page;
} scored_page;

static int scored_cmp(const void* a, const void* b) {
    const scored_page* x = (const scored_page*)a;
    const scored_page* y = (const scored_page*)b;
    if (x->score != y->score) return x->score > y->score ? -1 : 1;
    return x->page < y->page ? -1 : (x->page > y->page ? 1 : 0);
}

static int long_cmp(const void* a, const void* b) {
    const long x = *(const long*)a, y = *(const long*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

int wo_select_topk_pages(const double* q, const wo_head* h, const wo_pool* p, long budget, long* logical_out,
                         long* n_selected, double* k_out, double* v_out, long* entries) {
    if (budget < 1) return WO_EINVAL;
    const int d = p->head_dim, ps = p->page_size;
    const long n_pages = h->n_global;
    scored_page* sc = (scored_page*)malloc(sizeof(scored_page) * (size_t)(n_pages + 1));
    for (long lp = 0; lp < n_pages; ++lp) {
        const long first = lp * ps;
        const long last = h->global_len < first + ps ? h->global_len : first + ps;
        double best = -INFINITY;
        for (long g = first; g < last; ++g) {
            const double s = wo_dot(q, p->k + slot_index(p, h->global_pages[lp], (int)(g - first)) * d, d);
            if (s > best) best = s;
        }
        sc[lp].score = best;
        sc[lp].page = lp;
    }
    /* the comparator is a total order (ties broken by page id), so qsort
     * reproduces std::stable_sort's result */
    qsort(sc, (size_t)n_pages, sizeof(scored_page), scored_cmp);
    const long keep = budget < n_pages ? budget : n_pages;
    long* sel = (long*)malloc(sizeof(long) * (size_t)(keep + 1));
    for (long i = 0; i < keep; ++i) sel[i] = sc[i].page;
    qsort(sel, (size_t)keep, sizeof(long), long_cmp);
    long row = 0;
    for (long i = 0; i < keep; ++i) {
        const long lp = sel[i];
        const long first = lp * ps;
        const long last = h->global_len < first + ps ? h->global_len : first + ps;
        for (long g = first; g < last; ++g) {
            const size_t si = slot_index(p, h->global_pages[lp], (int)(g - first));
            if (k_out) memcpy(k_out + row * d, p->k + si * d, sizeof(double) * (size_t)d);
            if (v_out) memcpy(v_out + row * d, p->v + si * d, sizeof(double) * (size_t)d);
            ++row;
        }
        if (logical_out) logical_out[i] = lp;
    }
    if (n_selected) *n_selected = keep;
    if (entries) *entries = row;
    free(sc);
    free(sel);
    return WO_OK;
}

/* ======================================================================= */
/* path-level session                                                       */
/* ======================================================================= */

struct wo_session {
    int layers, q_heads, kv_heads, head_dim, hidden;
    long window, topk_budget;
    double tau, rope_base;
    double* bank; /* [layers*kv_heads][block] */
    wo_pool* pool;
    wo_head** heads; /* [layers*kv_heads] */
    int* prefilled;  /* per layer */
};

wo_session* wo_session_create(int layers, int q_heads, int kv_heads, int head_dim, int hidden, long window,
                              double tau, double rope_base, int page_size, long capacity_pages, long topk_budget,
                              const double* gate_bank) {
    if (layers < 1 || q_heads < 1 || kv_heads < 1 || q_heads % kv_heads != 0 || window < 1) return NULL;
    wo_session* s = (wo_session*)calloc(1, sizeof(wo_session));
    s->layers = layers;
    s->q_heads = q_heads;
    s->kv_heads = kv_heads;
    s->head_dim = head_dim;
    s->hidden = hidden;
    s->window = window;
    s->tau = tau;
    s->rope_base = rope_base;
    s->topk_budget = topk_budget;
    const long blen = wo_gate_block_len(head_dim, hidden);
    if (gate_bank) {
        s->bank = (double*)malloc(sizeof(double) * (size_t)(blen * layers * kv_heads));
        memcpy(s->bank, gate_bank, sizeof(double) * (size_t)(blen * layers * kv_heads));
    }
    s->pool = wo_pool_create(page_size, head_dim, capacity_pages);
    s->heads = (wo_head**)calloc((size_t)layers * kv_heads, sizeof(wo_head*));
    for (int l = 0; l < layers; ++l)
        for (int h = 0; h < kv_heads; ++h) s->heads[l * kv_heads + h] = wo_head_create(l, h, window);
    s->prefilled = (int*)calloc((size_t)layers, sizeof(int));
    return s;
}

void wo_session_destroy(wo_session* s) {
    if (!s) return;
    for (int i = 0; i < s->layers * s->kv_heads; ++i) wo_head_destroy(s->heads[i]);
    free(s->heads);
    wo_pool_destroy(s->pool);
    free(s->bank);
    free(s->prefilled);
    free(s);
}

wo_head* wo_session_head(wo_session* s, int layer, int kv_head) { return s->heads[layer * s->kv_heads + kv_head]; }
wo_pool* wo_session_pool(wo_session* s) { return s->pool; }

/* Session::prefill, one layer, projections removed (engine.cpp:188-257):
 * per kv head K_post = RoPE(K_pre), g = gate MLP (or forced), mask; per q
 * head (kv head = p / group, engine.cpp:224) Q = RoPE(Q_pre), VS attention
 * into out[:, p, :]; then prefill_populate per kv head. */
int wo_session_prefill_layer(wo_session* s, int layer, const double* q_pre, const double* k_pre, const double* v,
                             long t, const double* forced_gates, double* out, double* g_out, uint8_t* bits_out,
                             uint64_t* score_evals) {
    if (layer < 0 || layer >= s->layers) return WO_EINVAL;
    if (s->prefilled[layer]) return WO_ESTATE;
    if (t <= 0) return WO_EINVAL;
    const int d = s->head_dim, hkv = s->kv_heads, hq = s->q_heads, gsz = hq / hkv;
    const double scale = 1.0 / sqrt((double)d);
    const long blen = wo_gate_block_len(d, s->hidden);
    double* kp = (double*)malloc(sizeof(double) * (size_t)t * d);
    double* kr = (double*)malloc(sizeof(double) * (size_t)t * d * hkv);
    double* vv = (double*)malloc(sizeof(double) * (size_t)t * d * hkv);
    double* g = (double*)malloc(sizeof(double) * (size_t)t * hkv);
    uint8_t* bits = (uint8_t*)malloc((size_t)t * hkv);
    double* q = (double*)malloc(sizeof(double) * (size_t)t * d);
    double* o = (double*)malloc(sizeof(double) * (size_t)t * d);
    int st = WO_OK;
    for (int h = 0; h < hkv && st == WO_OK; ++h) {
        double* krh = kr + (size_t)h * t * d;
        for (long i = 0; i < t; ++i) {
            memcpy(kp + i * d, k_pre + ((size_t)i * hkv + h) * d, sizeof(double) * (size_t)d);
            memcpy(krh + i * d, kp + i * d, sizeof(double) * (size_t)d);
            wo_rope(krh + i * d, d, i, s->rope_base, 1.0);
            memcpy(vv + ((size_t)h * t + i) * d, v + ((size_t)i * hkv + h) * d, sizeof(double) * (size_t)d);
        }
        if (forced_gates)
            memcpy(g + (size_t)h * t, forced_gates + (size_t)h * t, sizeof(double) * (size_t)t);
        else
            wo_gate_forward_batch(s->bank + (size_t)(layer * hkv + h) * blen, d, s->hidden, kp, krh, t,
                                  g + (size_t)h * t);
        st = wo_binarize(g + (size_t)h * t, t, s->tau, bits + (size_t)h * t);
    }
    for (int p = 0; p < hq && st == WO_OK; ++p) {
        const int h = p / gsz;
        for (long i = 0; i < t; ++i) {
            memcpy(q + i * d, q_pre + ((size_t)i * hq + p) * d, sizeof(double) * (size_t)d);
            wo_rope(q + i * d, d, i, s->rope_base, 1.0);
        }
        st = wo_attn_vertical_slash(q, t, kr + (size_t)h * t * d, vv + (size_t)h * t * d, t, d, scale, 0, s->window,
                                    bits + (size_t)h * t, o, score_evals);
        for (long i = 0; i < t && st == WO_OK; ++i)
            memcpy(out + ((size_t)i * hq + p) * d, o + i * d, sizeof(double) * (size_t)d);
    }
    for (int h = 0; h < hkv && st == WO_OK; ++h)
        st = wo_prefill_populate(s->heads[layer * hkv + h], s->pool, kr + (size_t)h * t * d, vv + (size_t)h * t * d,
                                 g + (size_t)h * t, t, s->tau, 0);
    if (st == WO_OK) {
        if (g_out) memcpy(g_out, g, sizeof(double) * (size_t)t * hkv);
        if (bits_out) memcpy(bits_out, bits, (size_t)t * hkv);
        s->prefilled[layer] = 1;
    }
    free(kp);
    free(kr);
    free(vv);
    free(g);
    free(bits);
    free(q);
    free(o);
    return st;
}

/* Session::decode_step, one layer, projections removed (engine.cpp:291-327) */
int wo_session_decode_layer(wo_session* s, int layer, const double* q_pre, const double* k_pre, const double* v,
                            const double* forced_gates, double* out, double* g_out, int* events_out,
                            uint64_t* score_evals) {
    if (layer < 0 || layer >= s->layers) return WO_EINVAL;
    if (!s->prefilled[layer]) return WO_ESTATE;
    const int d = s->head_dim, hkv = s->kv_heads, hq = s->q_heads, gsz = hq / hkv;
    const double scale = 1.0 / sqrt((double)d);
    const long blen = wo_gate_block_len(d, s->hidden);
    const long pos = s->heads[layer * hkv]->tokens_seen;
    double* feat = (double*)malloc(sizeof(double) * 2 * (size_t)d);
    double* q = (double*)malloc(sizeof(double) * (size_t)d);
    int st = WO_OK;
    for (int h = 0; h < hkv && st == WO_OK; ++h) {
        memcpy(feat, k_pre + (size_t)h * d, sizeof(double) * (size_t)d);
        memcpy(feat + d, feat, sizeof(double) * (size_t)d);
        wo_rope(feat + d, d, pos, s->rope_base, 1.0);
        const double gv = forced_gates ? forced_gates[h]
                                       : wo_gate_forward(s->bank + (size_t)(layer * hkv + h) * blen, d, s->hidden, feat);
        if (g_out) g_out[h] = gv;
        const int ev = wo_local_write(s->heads[layer * hkv + h], s->pool, feat + d, v + (size_t)h * d, gv, s->tau, pos);
        if (ev < 0) st = -ev;
        if (events_out) events_out[h] = ev;
    }
    for (int p = 0; p < hq && st == WO_OK; ++p) {
        const wo_head* hc = s->heads[layer * hkv + p / gsz];
        memcpy(q, q_pre + (size_t)p * d, sizeof(double) * (size_t)d);
        wo_rope(q, d, pos, s->rope_base, 1.0);
        double* lk = (double*)malloc(sizeof(double) * (size_t)(hc->local_len * d + 1));
        double* lv = (double*)malloc(sizeof(double) * (size_t)(hc->local_len * d + 1));
        long gl = hc->global_len;
        double* gk = (double*)malloc(sizeof(double) * (size_t)(gl * d + 1));
        double* gvv = (double*)malloc(sizeof(double) * (size_t)(gl * d + 1));
        wo_gather(hc, s->pool, gk, gvv, NULL, NULL, lk, lv, NULL, NULL);
        if (s->topk_budget > 0) {
            long entries = 0;
            st = wo_select_topk_pages(q, hc, s->pool, s->topk_budget, NULL, NULL, gk, gvv, &entries);
            gl = entries;
        }
        if (st == WO_OK)
            st = wo_attn_ragged(q, gk, gvv, gl, lk, lv, hc->local_len, d, scale, out + (size_t)p * d, score_evals);
        free(lk);
        free(lv);
        free(gk);
        free(gvv);
    }
    free(feat);
    free(q);
    return st;
}
