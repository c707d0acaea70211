// api.cu -- the C-ABI (include/wgkv_b200.h): context, device state, and the
// host orchestration of K1..K5 mirroring Session::prefill / decode_step
// (engine.cpp:153-341).  No allocation on hot calls; everything is
// stream-ordered on the context stream.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <fstream>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "admit.cuh"
#include "attn.cuh"
#include "attn_tc.cuh"
#include "comm.cuh"
#include "outproj.cuh"
#include "gate.cuh"

using namespace wgkv;

static thread_local std::string g_last_error;
void wgkv_set_error(const std::string& msg) { g_last_error = msg; }

namespace wgkv {

int num_sms() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
    return n;
}

cudaError_t ensure_smem_attr(const void* func, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{func, dev}];
    if (smem <= have) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) have = smem;
    return e;
}

}  // namespace wgkv

namespace {

// every entry point runs on its context's device (one host thread may drive
// contexts on several GPUs) and restores the caller's device on return
struct DevGuard {
    int prev = -1, dev;
    explicit DevGuard(int d) : dev(d) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
};

int fail(int code, const std::string& msg) {
    wgkv_set_error(msg);
    return code;
}

template <typename T>
T* dalloc(size_t n, std::vector<void*>& owned) {
    void* p = nullptr;
    if (n == 0) n = 1;
    if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return nullptr;
    owned.push_back(p);
    return static_cast<T*>(p);
}

__global__ void init_stack_kernel(int32_t* stack, long cap) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < cap; i += (long)gridDim.x * blockDim.x)
        stack[i] = (int32_t)(cap - 1 - i);
}

// HeadCache::release (kvstore.cpp:243-251) for every (layer, slot, head)
__global__ void release_kernel(PoolView pv, int layers, int seq0, int nseq) {
    const int idx = blockIdx.x;
    const int l = idx / (nseq * pv.kv_heads), r = idx % (nseq * pv.kv_heads);
    const int s = seq0 + r / pv.kv_heads, h = r % pv.kv_heads;
    const long hidx = pv.head_index(l, s, h);
    const HeadState st = pv.state[hidx];
    const int ng = (st.global_len + pv.page_size - 1) / pv.page_size;
    const int nl = (min(st.local_len, 0x7fffffff) + pv.page_size - 1) / pv.page_size;
    const int n = nl + ng;
    auto page_at = [&](int i) -> int {  // i-th page in reverse allocation order
        const int k = n - 1 - i;
        return k < ng ? pv.gpt[hidx * pv.n_gp + k] : pv.lpt[hidx * pv.n_lp + (k - ng)];
    };
    // pass 1: count the pages the head really owns (a failed allocation left
    // -1 in its table; those are never pushed)
    __shared__ int wsum[32];
    __shared__ int base;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int cnt = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) cnt += page_at(i) >= 0;
    for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) wsum[wid] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < nw; ++w) tot += wsum[w];
        base = atomicAdd(pv.free_top, tot);
    }
    __syncthreads();
    // pass 2: order-preserving compaction.  Pushed in reverse allocation order
    // (Global pages then Local, admit_plan's pop order), so re-allocating pops
    // the same ascending physical runs: a head's Global pages stay physically
    // contiguous, which lets K3 load a 128-key vertical block with one TMA box
    // per dim half
    __shared__ int wpre[32];
    int run = base;
    for (int i0 = 0; i0 < n; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const int page = i < n ? page_at(i) : -1;
        const unsigned m = __ballot_sync(0xffffffffu, page >= 0);
        __syncthreads();
        if (lane == 0) wpre[wid] = __popc(m);
        __syncthreads();
        int off = run;
        for (int w = 0; w < wid; ++w) off += wpre[w];
        if (page >= 0) pv.free_stack[off + __popc(m & ((1u << lane) - 1u))] = page;
        for (int w = 0; w < nw; ++w) run += wpre[w];
    }
    __syncthreads();
    if (threadIdx.x == 0) pv.state[hidx] = HeadState{0, 0, 0, 0};
}

// HeadCache::gather (kvstore.cpp:205-241) of one head into position order:
// rows [0, G) Global by logical index, rows [G, G+Lc) the ring unrolled from
// `start`; one warp per row, K/V widened to fp32 (k/v may be null)
__global__ void export_rows_kernel(PoolView pv, long hidx, long W, int G, int Lc, int start, int esz,
                                   float* __restrict__ k, float* __restrict__ v, float* __restrict__ gate,
                                   int32_t* __restrict__ pos) {
    const int lane = threadIdx.x & 31;
    const long r = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= (long)G + Lc) return;
    const int ps = pv.page_size, d = pv.head_dim;
    int page, slot;
    if (r < G) {
        page = pv.gpt[hidx * pv.n_gp + r / ps];
        slot = (int)(r % ps);
    } else {
        const long ring = (start + (r - G)) % W;
        page = pv.lpt[hidx * pv.n_lp + ring / ps];
        slot = (int)(ring % ps);
    }
    if (page < 0) {  // failed allocation (latched ENOPAGES): report an empty entry
        if (lane == 0) {
            gate[r] = 0.f;
            pos[r] = -1;
        }
        return;
    }
    const size_t mi = (size_t)page * ps + slot;
    if (lane == 0) {
        gate[r] = pv.gate[mi];
        pos[r] = pv.pos[mi];
    }
    if (!k) return;
    const size_t e0 = (size_t)page * pv.page_elems() + (size_t)slot * d, e1 = e0 + (size_t)ps * d;
    for (int e = lane; e < d; e += 32) {
        if (esz == 2) {
            const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(pv.data);
            k[r * d + e] = __bfloat162float(p[e0 + e]);
            v[r * d + e] = __bfloat162float(p[e1 + e]);
        } else {
            const float* p = reinterpret_cast<const float*>(pv.data);
            k[r * d + e] = p[e0 + e];
            v[r * d + e] = p[e1 + e];
        }
    }
}

}  // namespace

struct wgkv_ctx {
    wgkv_config cfg{};
    cudaStream_t stream = nullptr;
    size_t esz = 2;
    std::vector<void*> owned;
    PoolView pv{};
    // gate parameters
    float *w1t = nullptr, *b1f = nullptr, *w2f = nullptr;
    double *b2f = nullptr, *w1d = nullptr, *b1d = nullptr, *w2d = nullptr, *freq = nullptr;
    float* bandc = nullptr;  // per (layer, kv head) fp32 error-bound constant for K1's recheck band
    float4* bw = nullptr;    // [blk][hidden/2] {b1[2j], b1[2j+1], w2[2j], w2[2j+1]} (K1 tc epilogue)
    __nv_bfloat16* w1split = nullptr;  // [L*H][Wpre_hi, Wpost_hi, Wpre_lo, Wpost_lo][128][128] (K1 tcgen05)
    bool gates_set = false;
    // workspaces
    void* ws_kpost = nullptr;
    float* ws_g = nullptr;
    uint8_t* ws_bits = nullptr;
    int32_t* ws_chunk = nullptr;
    int64_t* ws_cand = nullptr;
    int* ws_cnt = nullptr;  // [1] near count
    int* ws_pcnt = nullptr;      // [S][H] recheck-list lengths (K1)
    float2* ws_rope = nullptr;   // [max_prefill_tokens][d/2] cos/sin table (K1)
    int64_t* ws_near = nullptr;
    float* ws_part = nullptr;
    int* ws_nchunks = nullptr;
    int* ws_tokpos = nullptr;  // [S*H] the new token's position per (seq, kv head) (deferred append)
    AppendWork wk{};           // split-append scratch (append.cuh); next / event / slot are [2][S*H]
    FusedWork fw{};            // fused decode layer scratch (fused.cuh), parity-split halves as [2][...]
    // non-deferred decode: the append's gate CTAs run on gate_stream, forked after
    // the route kernel and joined after the attention of the same layer call
    cudaStream_t gate_stream = nullptr;
    cudaEvent_t ev_route = nullptr, ev_gate = nullptr;
    bool gate_join = false;
    // K5's work before its PDL wait is only safe when the kernel in front of it
    // is the finish kernel of ANOTHER layer: every API call bumps api_gen, and
    // a deferred decode_layer records its own generation and layer when done
    uint64_t api_gen = 0, finish_gen = 0;
    int finish_layer = -1;
    float* ws_score = nullptr;  // K6: [S][Hq][n_gp] page scores
    int32_t* ws_sel = nullptr;  // K6: [S][Hq][n_gp] selected logical pages
    int32_t* ws_nsel = nullptr; // K6: [S][Hq]
    unsigned long long* ws_thr = nullptr;  // K6: [S][Hq] selection thresholds
    uint8_t* ws_umask = nullptr;           // K6: [S][H][n_gp] union q-head masks
    int* ws_ucnt = nullptr;                // K6: [S][H][ceil(n_gp/1024)] union block counts
    __nv_bfloat16* quest_meta = nullptr;   // K6 Quest mode: [capacity][min 128 | max 128]
    int* quest_full = nullptr;             // K6 Quest mode: [L][S][H] pages whose metadata is final
    int max_chunks = kMaxChunks;
    long near_cap = 0;
    // C1 (comm.cu): head-output all-gather over a world of KV-head shards
    void* comm = nullptr;
    bool own_comm = false;
    int world = 1, rank = 0;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_comm_in = nullptr, ev_comm_done = nullptr;
    uint8_t* stage = nullptr;  // [world][stage_rows][q_heads * d] elements
    // C1 over peer memory (comm.cuh): every rank's exchange region as mapped here
    PeerXchg px{};        // world = 0: not attached
    int peer_wait_ranks = 0;
    bool peer_decode = false;     // decode layers push their output rows themselves
    bool peer_prefill = false;    // K3 stores its output rows into every rank's bulk slot
    uint64_t peer_bulk_seq = 0;   // bulk exchanges so far (slot = seq % 2)
    uint64_t peer_seq = 0;        // exchanges so far (slot = seq % kPeerSlots)
    int pend_slot = -1;           // the last exchange, not unpacked yet
    long pend_rows = 0;
    uint8_t* peer_own = nullptr;  // wgkv_peer_alloc's region
    int peer_own_world = 0;
    long peer_own_rows = 0, peer_own_bulk = 0;
    std::vector<void*> peer_ipc;  // regions opened with cudaIpcOpenMemHandle
    long stage_rows = 0;
    // f3 (outproj.cu): cuBLAS handle and the two-slot concat ring of the chunked Wo
    void* blas = nullptr;
    uint8_t* cring = nullptr;  // [2][cring_rows][world * q_heads * d] elements
    long cring_rows = 0;
    cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_gemm[2] = {nullptr, nullptr};
    // host mirrors for lifecycle checks and grid sizing
    std::vector<uint8_t> prefilled;  // [L][S]
    std::vector<long> tokens;        // [L][S] tokens seen

    GateArgs gate_args(int layer, long T, long pos0) const {
        GateArgs a{};
        a.layer = layer;
        a.kv_heads = cfg.kv_heads;
        a.bank_heads = cfg.kv_heads;
        a.head_offset = 0;
        a.d = cfg.head_dim;
        a.hidden = cfg.hidden;
        a.T = T;
        a.pos0 = pos0;
        a.tau = cfg.tau;
        a.ztau = (float)std::log(cfg.tau / (1.0 - cfg.tau));
        a.freq = freq;
        a.w1t = w1t;
        a.b1f = b1f;
        a.w2f = w2f;
        a.b2f = b2f;
        a.w1d = w1d;
        a.b1d = b1d;
        a.w2d = w2d;
        a.b2d = b2f;
        a.bandc = bandc;
        a.bw = bw;
        return a;
    }
    bool use_tc() const {
        // tcgen05 path: bf16, d = 128, pages tiling a 128-key block, GQA groups
        // of an even size (two heads per CTA); everything else runs SIMT
        if (cfg.attn_impl == WGKV_ATTN_SIMT) return false;
        return cfg.dtype == WGKV_BF16 && cfg.head_dim == 128 && cfg.page_size >= 8 && 128 % cfg.page_size == 0 &&
               (cfg.q_heads / cfg.kv_heads) % 2 == 0;
    }
};

extern "C" {

const char* wgkv_last_error(void) { return g_last_error.c_str(); }
const char* wgkv_version(void) { return "wgkv_b200 0.1 sm_100a"; }

int wgkv_ctx_create(const wgkv_config* cfg_in, wgkv_ctx** out) {
    if (!cfg_in || !out) return fail(WGKV_EINVAL, "wgkv_ctx_create: null argument");
    const wgkv_config c = *cfg_in;
    if (c.layers < 1 || c.q_heads < 1 || c.kv_heads < 1 || c.q_heads % c.kv_heads != 0)
        return fail(WGKV_EINVAL, "wgkv_ctx_create: bad head/layer geometry");
    if (c.head_dim <= 0 || c.head_dim % 2 != 0) return fail(WGKV_EINVAL, "rope: head_dim must be even");
    // any even d <= 256 (the reference's ModelConfig default is 16, model.hpp:15); the
    // tensor-core kernels take d = 128, everything else runs the SIMT kernels
    if (c.head_dim > 256) return fail(WGKV_ENOTSUP, "head_dim must be <= 256");
    if (c.window < 1) return fail(WGKV_EINVAL, "HeadCache: window must be >= 1");
    if (!(c.tau > 0.0 && c.tau < 1.0)) return fail(WGKV_EINVAL, "binarize: tau must lie in (0,1)");
    if (c.page_size < 1 || c.page_size > 32) return fail(WGKV_ENOTSUP, "page_size must be in [1, 32]");
    if (c.hidden < 1 || c.max_seqs < 1 || c.max_tokens < 1) return fail(WGKV_EINVAL, "bad sizes");
    if (c.dtype != WGKV_BF16 && c.dtype != WGKV_F32) return fail(WGKV_EINVAL, "bad dtype");
    if (c.topk_mode != WGKV_TOPK_EXACT && c.topk_mode != WGKV_TOPK_QUEST) return fail(WGKV_EINVAL, "bad topk_mode");
    if (c.decode_chunk_pages < 0) return fail(WGKV_EINVAL, "decode_chunk_pages must be >= 0");
    if (c.topk_mode == WGKV_TOPK_QUEST &&
        (c.dtype != WGKV_BF16 || c.head_dim != 128 || c.page_size != 16 || c.q_heads / c.kv_heads > 8))
        return fail(WGKV_ENOTSUP, "Quest page selection needs bf16, head_dim 128, page 16, GQA group <= 8");
    if ((c.max_tokens + c.page_size - 1) / c.page_size + 1 + (c.window + c.page_size - 1) / c.page_size >
        (long)kMaxChunks * kDecPidCap)
        return fail(WGKV_ENOTSUP, "max_tokens exceeds the decode work split (kMaxChunks * kDecPidCap pages per head)");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || c.device < 0 || c.device >= ndev)
        return fail(WGKV_EINVAL, "wgkv_ctx_create: no such CUDA device");
    DevGuard dg_(c.device);

    auto* ctx = new wgkv_ctx();
    ctx->cfg = c;
    if (ctx->cfg.max_prefill_tokens <= 0) ctx->cfg.max_prefill_tokens = c.max_tokens;
    ctx->esz = c.dtype == WGKV_BF16 ? 2 : 4;
    const int ps = c.page_size, d = c.head_dim, H = c.kv_heads, S = c.max_seqs, L = c.layers;
    const int n_lp = (int)((c.window + ps - 1) / ps);
    const int n_gp = (int)((c.max_tokens + ps - 1) / ps + 1);
    long cap = c.capacity_pages;
    if (cap <= 0) cap = (long)L * H * S * (n_lp + n_gp);  // default_capacity (engine.cpp:88-93)
    ctx->cfg.capacity_pages = cap;
    auto& o = ctx->owned;
    PoolView& pv = ctx->pv;
    pv.page_size = ps;
    pv.head_dim = d;
    pv.n_lp = n_lp;
    pv.n_gp = n_gp;
    pv.max_seqs = S;
    pv.kv_heads = H;
    pv.capacity = cap;
    pv.data = dalloc<uint8_t>((size_t)cap * 2 * ps * d * ctx->esz, o);
    pv.gate = dalloc<float>((size_t)cap * ps, o);
    pv.pos = dalloc<int32_t>((size_t)cap * ps, o);
    pv.adm = dalloc<uint8_t>((size_t)cap * ps, o);
    pv.free_stack = dalloc<int32_t>((size_t)cap, o);
    pv.free_top = dalloc<int32_t>(1, o);
    pv.err = dalloc<int32_t>(1, o);
    pv.lpt = dalloc<int32_t>((size_t)L * S * H * n_lp, o);
    pv.gpt = dalloc<int32_t>((size_t)L * S * H * n_gp, o);
    pv.state = dalloc<HeadState>((size_t)L * S * H, o);
    const size_t blocks = (size_t)L * H, fd = 2 * (size_t)d;
    ctx->w1t = dalloc<float>(blocks * fd * c.hidden, o);
    ctx->b1f = dalloc<float>(blocks * c.hidden, o);
    ctx->w2f = dalloc<float>(blocks * c.hidden, o);
    ctx->b2f = dalloc<double>(blocks, o);
    ctx->bandc = dalloc<float>(blocks, o);
    ctx->bw = dalloc<float4>(blocks * ((c.hidden + 1) / 2), o);
    ctx->w1d = dalloc<double>(blocks * fd * c.hidden, o);
    if (c.dtype == WGKV_BF16 && d == 128 && c.hidden == 128)  // K1 tensor-core operand: split-bf16 W1 tiles
        ctx->w1split = dalloc<__nv_bfloat16>(blocks * 4 * 128 * 128, o);
    ctx->b1d = dalloc<double>(blocks * c.hidden, o);
    ctx->w2d = dalloc<double>(blocks * c.hidden, o);
    ctx->freq = dalloc<double>((size_t)d / 2, o);
    const long Tm = ctx->cfg.max_prefill_tokens;
    const size_t toks = (size_t)S * Tm * H;
    ctx->ws_kpost = dalloc<uint8_t>(toks * d * ctx->esz, o);
    ctx->ws_g = dalloc<float>(toks, o);
    ctx->ws_bits = dalloc<uint8_t>(toks, o);
    ctx->ws_chunk = dalloc<int32_t>((size_t)S * H * ((Tm + 127) / 128 + 1), o);
    ctx->ws_cand = dalloc<int64_t>(toks, o);
    ctx->ws_cnt = dalloc<int>(4, o);
    ctx->ws_pcnt = dalloc<int>((size_t)S * H, o);
    ctx->ws_rope = dalloc<float2>((size_t)Tm * (d / 2), o);
    ctx->near_cap = 1 << 20;
    ctx->ws_near = dalloc<int64_t>((size_t)ctx->near_cap, o);
    const int gs = c.q_heads / c.kv_heads;
    // (+4: the fused layer's bulk copies round a pair's partials up to 16 bytes)
    ctx->ws_part = dalloc<float>((size_t)S * H * ctx->max_chunks * gs * (d + 2) + 4, o);
    // per-pair chunk counts | work-stealing counter | per-pair merge counters
    ctx->ws_nchunks = dalloc<int>(2 * (size_t)S * H + 1, o);
    ctx->ws_tokpos = dalloc<int>((size_t)S * H, o);
    ctx->wk.terms = dalloc<double>(2 * (size_t)S * H * c.hidden, o);  // [parity] (deferred decode)
    ctx->wk.count = dalloc<int>((size_t)S * H, o);
    // route outputs: two halves by layer parity (fused layer, fused.cuh)
    ctx->wk.slot = dalloc<int>(2 * (size_t)S * H, o);
    ctx->wk.event = dalloc<int>(2 * (size_t)S * H, o);
    ctx->wk.next = dalloc<HeadState>(2 * (size_t)S * H, o);
    ctx->wk.pos = dalloc<int>((size_t)S * H, o);
    ctx->fw.cnt_items = dalloc<int>((size_t)S * H, o);
    ctx->fw.cnt_kv = dalloc<int>(2 * (size_t)S * H, o);
    ctx->fw.cnt_gw = dalloc<int>(2 * (size_t)S * H, o);
    ctx->fw.cnt_gate = dalloc<int>(2 * (size_t)S * H, o);
    ctx->fw.g = dalloc<double>(2 * (size_t)S * H, o);
    ctx->fw.pub = dalloc<int>(2 * (size_t)S * H, o);
    ctx->fw.started = dalloc<int>(2, o);

    if (c.topk_budget > 0) {
        ctx->ws_score = dalloc<float>((size_t)S * c.q_heads * n_gp, o);
        ctx->ws_sel = dalloc<int32_t>((size_t)S * c.q_heads * n_gp, o);
        ctx->ws_nsel = dalloc<int32_t>((size_t)S * c.q_heads, o);
        ctx->ws_thr = dalloc<unsigned long long>((size_t)S * c.q_heads, o);
        ctx->ws_umask = dalloc<uint8_t>((size_t)S * H * n_gp, o);
        ctx->ws_ucnt = dalloc<int>((size_t)S * H * ((n_gp + 1023) / 1024), o);
        if (c.topk_mode == WGKV_TOPK_QUEST) {
            ctx->quest_meta = dalloc<__nv_bfloat16>((size_t)cap * 2 * d, o);
            ctx->quest_full = dalloc<int>((size_t)L * S * H, o);
        }
    }
    for (void* p : o)
        if (!p) {
            for (void* q : o) cudaFree(q);
            delete ctx;
            return fail(WGKV_ECUDA, "wgkv_ctx_create: cudaMalloc failed (pool of " + std::to_string(cap) + " pages)");
        }
    // RoPE frequencies with the reference expression (numerics.cpp:54)
    std::vector<double> fr(d / 2);
    for (int i = 0; i < d / 2; ++i) fr[i] = std::pow(c.rope_base, -2.0 * i / d);
    cudaMemcpy(ctx->freq, fr.data(), sizeof(double) * fr.size(), cudaMemcpyHostToDevice);
    init_stack_kernel<<<256, 256>>>(pv.free_stack, cap);
    const int32_t top = (int32_t)cap, zero = 0;
    cudaMemcpy(pv.free_top, &top, sizeof(top), cudaMemcpyHostToDevice);
    cudaMemcpy(pv.err, &zero, sizeof(zero), cudaMemcpyHostToDevice);
    cudaMemset(pv.state, 0, sizeof(HeadState) * (size_t)L * S * H);
    cudaMemset(ctx->ws_nchunks, 0, sizeof(int) * (2 * (size_t)S * H + 1));  // K5 work counter starts at 0
    cudaMemset(ctx->wk.count, 0, sizeof(int) * (size_t)S * H);              // split-append arrivals
    if (ctx->fw.cnt_items) {  // fused-layer counters start at 0 (each is reset by its last user)
        cudaMemset(ctx->fw.cnt_items, 0, sizeof(int) * (size_t)S * H);
        cudaMemset(ctx->fw.cnt_kv, 0, sizeof(int) * 2 * (size_t)S * H);
        cudaMemset(ctx->fw.cnt_gw, 0, sizeof(int) * 2 * (size_t)S * H);
        cudaMemset(ctx->fw.cnt_gate, 0, sizeof(int) * 2 * (size_t)S * H);
        cudaMemset(ctx->fw.pub, 0, sizeof(int) * 2 * (size_t)S * H);
        cudaMemset(ctx->fw.started, 0, sizeof(int) * 2);
    }
    // zeroed pages: K3/K5 may stream stale slots of a partially filled page
    // (masked out), which must at least be finite
    cudaMemset(pv.data, 0, (size_t)cap * 2 * ps * d * ctx->esz);
    cudaMemset(pv.lpt, 0xff, sizeof(int32_t) * (size_t)L * S * H * n_lp);
    cudaMemset(pv.gpt, 0xff, sizeof(int32_t) * (size_t)L * S * H * n_gp);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        for (void* q : o) cudaFree(q);
        delete ctx;
        return fail(WGKV_ECUDA, "wgkv_ctx_create: init failed");
    }
    ctx->prefilled.assign((size_t)L * S, 0);
    ctx->tokens.assign((size_t)L * S, 0);
    *out = ctx;
    return WGKV_OK;
}

int wgkv_ctx_destroy(wgkv_ctx* ctx) {
    if (!ctx) return WGKV_OK;
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    cudaDeviceSynchronize();
    if (ctx->own_comm) comm_destroy(ctx->comm);
    if (ctx->stage) cudaFree(ctx->stage);
    if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
    if (ctx->gate_stream) cudaStreamDestroy(ctx->gate_stream);
    if (ctx->ev_route) cudaEventDestroy(ctx->ev_route);
    if (ctx->ev_gate) cudaEventDestroy(ctx->ev_gate);
    blas_destroy(ctx->blas);
    if (ctx->cring) cudaFree(ctx->cring);
    for (int b = 0; b < 2; ++b) {
        if (ctx->ev_ready[b]) cudaEventDestroy(ctx->ev_ready[b]);
        if (ctx->ev_gemm[b]) cudaEventDestroy(ctx->ev_gemm[b]);
    }
    if (ctx->ev_comm_in) cudaEventDestroy(ctx->ev_comm_in);
    if (ctx->ev_comm_done) cudaEventDestroy(ctx->ev_comm_done);
    for (void* p : ctx->peer_ipc) cudaIpcCloseMemHandle(p);
    if (ctx->peer_own) cudaFree(ctx->peer_own);
    for (void* p : ctx->owned) cudaFree(p);
    delete ctx;
    return WGKV_OK;
}

int wgkv_set_stream(wgkv_ctx* ctx, void* stream) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    ctx->stream = static_cast<cudaStream_t>(stream);
    return WGKV_OK;
}

int wgkv_sync(wgkv_ctx* ctx) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    WGKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    int32_t err = 0;
    WGKV_CUDA_TRY(cudaMemcpy(&err, ctx->pv.err, sizeof(err), cudaMemcpyDeviceToHost));
    if (err == WGKV_ENOPAGES) {
        const int32_t zero = 0;
        cudaMemcpy(ctx->pv.err, &zero, sizeof(zero), cudaMemcpyHostToDevice);
        char msg[160];
        std::snprintf(msg, sizeof(msg), "out of pages: capacity=%ld", ctx->pv.capacity);
        return fail(WGKV_ENOPAGES, msg);
    }
    return err;
}

int wgkv_gate_set(wgkv_ctx* ctx, const double* bank, int bank_layers, int bank_heads) {
    if (!ctx || !bank) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    const auto& c = ctx->cfg;
    if (bank_layers != c.layers || bank_heads < c.kv_head_offset + c.kv_heads)
        return fail(WGKV_EINVAL, "Session: gate bank shape does not match model");
    const int d = c.head_dim, hid = c.hidden, fd = 2 * d;
    const size_t blen = (size_t)hid * fd + 2 * (size_t)hid + 1;
    const size_t nb = (size_t)c.layers * c.kv_heads;
    std::vector<float> w1t(nb * fd * hid), b1f(nb * hid), w2f(nb * hid);
    std::vector<double> w1d(nb * fd * hid), b1d(nb * hid), w2d(nb * hid), b2(nb);
    std::vector<float> bandc(nb);
    for (int l = 0; l < c.layers; ++l)
        for (int h = 0; h < c.kv_heads; ++h) {
            const double* blk = bank + ((size_t)l * bank_heads + c.kv_head_offset + h) * blen;
            const size_t b = (size_t)l * c.kv_heads + h;
            for (int u = 0; u < hid; ++u)
                for (int k = 0; k < fd; ++k) {
                    w1d[(b * hid + u) * fd + k] = blk[(size_t)u * fd + k];
                    w1t[(b * fd + k) * hid + u] = (float)blk[(size_t)u * fd + k];
                }
            for (int u = 0; u < hid; ++u) {
                b1d[b * hid + u] = blk[(size_t)hid * fd + u];
                w2d[b * hid + u] = blk[(size_t)hid * fd + hid + u];
                b1f[b * hid + u] = (float)b1d[b * hid + u];
                w2f[b * hid + u] = (float)w2d[b * hid + u];
            }
            b2[b] = blk[(size_t)hid * fd + 2 * hid];
            double cb = 0.0;  // sum_h |w2_h| ||W1_h||_2
            for (int u = 0; u < hid; ++u) {
                double n2 = 0.0;
                for (int k = 0; k < fd; ++k) n2 += blk[(size_t)u * fd + k] * blk[(size_t)u * fd + k];
                cb += std::fabs(w2d[b * hid + u]) * std::sqrt(n2);
            }
            bandc[b] = (float)cb;
        }
    WGKV_CUDA_TRY(cudaMemcpy(ctx->w1t, w1t.data(), w1t.size() * 4, cudaMemcpyHostToDevice));
    WGKV_CUDA_TRY(cudaMemcpy(ctx->b1f, b1f.data(), b1f.size() * 4, cudaMemcpyHostToDevice));
    WGKV_CUDA_TRY(cudaMemcpy(ctx->w2f, w2f.data(), w2f.size() * 4, cudaMemcpyHostToDevice));
    WGKV_CUDA_TRY(cudaMemcpy(ctx->w1d, w1d.data(), w1d.size() * 8, cudaMemcpyHostToDevice));
    WGKV_CUDA_TRY(cudaMemcpy(ctx->b1d, b1d.data(), b1d.size() * 8, cudaMemcpyHostToDevice));
    WGKV_CUDA_TRY(cudaMemcpy(ctx->w2d, w2d.data(), w2d.size() * 8, cudaMemcpyHostToDevice));
    WGKV_CUDA_TRY(cudaMemcpy(ctx->b2f, b2.data(), b2.size() * 8, cudaMemcpyHostToDevice));
    WGKV_CUDA_TRY(cudaMemcpy(ctx->bandc, bandc.data(), bandc.size() * 4, cudaMemcpyHostToDevice));
    {
        const int hp = (hid + 1) / 2;
        std::vector<float4> bw(nb * hp);
        for (size_t b = 0; b < nb; ++b)
            for (int j = 0; j < hp; ++j) {
                const int u0 = 2 * j, u1 = std::min(2 * j + 1, hid - 1);
                const float z = (2 * j + 1 < hid) ? 1.f : 0.f;
                bw[b * hp + j] = make_float4(b1f[b * hid + u0], b1f[b * hid + u1] * z, w2f[b * hid + u0],
                                             w2f[b * hid + u1] * z);
            }
        WGKV_CUDA_TRY(cudaMemcpy(ctx->bw, bw.data(), bw.size() * sizeof(float4), cudaMemcpyHostToDevice));
    }
    if (ctx->w1split) {  // W1 = hi + lo in bf16, as four K-major [128 hidden][128 k] tiles per head
        std::vector<__nv_bfloat16> ws(nb * 4 * 128 * 128);
        for (size_t b = 0; b < nb; ++b)
            for (int u = 0; u < 128; ++u)
                for (int k = 0; k < 256; ++k) {
                    const double w = w1d[(b * 128 + u) * 256 + k];
                    const __nv_bfloat16 hi = __float2bfloat16_rn((float)w);
                    const __nv_bfloat16 lo = __float2bfloat16_rn((float)(w - (double)__bfloat162float(hi)));
                    const size_t seg = k < 128 ? 0 : 1;  // 0: k_pre columns, 1: k_post columns
                    ws[((b * 4 + seg) * 128 + u) * 128 + (k & 127)] = hi;
                    ws[((b * 4 + 2 + seg) * 128 + u) * 128 + (k & 127)] = lo;
                }
        WGKV_CUDA_TRY(cudaMemcpy(ctx->w1split, ws.data(), ws.size() * 2, cudaMemcpyHostToDevice));
    }
    ctx->gates_set = true;
    return WGKV_OK;
}

// GateBank::load (gating.cpp:107-147): "WGKV", u32 version/L/H/head_dim/hidden, f64 blocks
int wgkv_gate_load(wgkv_ctx* ctx, const char* path) {
    if (!ctx || !path) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    std::ifstream is(path, std::ios::binary);
    if (!is) return fail(WGKV_ERUNTIME, std::string("GateBank::load: cannot open ") + path);
    char magic[4];
    uint32_t hdr[5];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "WGKV", 4) != 0)
        return fail(WGKV_ERUNTIME, std::string("GateBank::load: bad magic in ") + path);
    is.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
    if (!is || hdr[0] != 1u) return fail(WGKV_ERUNTIME, "GateBank::load: unsupported version");
    const int L = (int)hdr[1], H = (int)hdr[2], d = (int)hdr[3], hid = (int)hdr[4];
    if (d != ctx->cfg.head_dim || hid != ctx->cfg.hidden)
        return fail(WGKV_EINVAL, "Session: gate bank shape does not match model");
    const size_t n = (size_t)L * H * ((size_t)hid * 2 * d + 2 * hid + 1);
    std::vector<double> bank(n);
    is.read(reinterpret_cast<char*>(bank.data()), (std::streamsize)(n * 8));
    if (!is) return fail(WGKV_ERUNTIME, std::string("GateBank::load: truncated file ") + path);
    return wgkv_gate_set(ctx, bank.data(), L, H);
}

static int check_slots(wgkv_ctx* ctx, int layer, int seq0, int nseq, long T) {
    const auto& c = ctx->cfg;
    if (layer < 0 || layer >= c.layers) return fail(WGKV_EINVAL, "layer out of range");
    if (seq0 < 0 || nseq < 1 || seq0 + nseq > c.max_seqs) return fail(WGKV_EINVAL, "sequence slots out of range");
    if (T < 0 || T > c.max_prefill_tokens) return fail(WGKV_EINVAL, "T exceeds max_prefill_tokens");
    return WGKV_OK;
}

int wgkv_gate_score(wgkv_ctx* ctx, int layer, int nseq, long T, long pos0, const void* k_pre, const float* forced_g,
                    void* k_post_out, float* g_out, uint8_t* bits_out, int64_t* near_idx, int near_cap,
                    int* near_count) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    int st = check_slots(ctx, layer, 0, nseq, T);
    if (st) return st;
    if (!forced_g && !ctx->gates_set) return fail(WGKV_ESTATE, "gate parameters not set");
    if (T == 0) return WGKV_OK;
    GateArgs a = ctx->gate_args(layer, T, pos0);
    int64_t* nidx = near_idx ? near_idx : ctx->ws_near;
    const int ncap = near_idx ? near_cap : (int)ctx->near_cap;
    WGKV_CUDA_TRY(cudaMemsetAsync(ctx->ws_cnt + 1, 0, sizeof(int), ctx->stream));
    if (forced_g) {
        // effective_gate override (engine.cpp:126-151): RoPE only, g = forced, bit = g >= tau
        st = launch_forced_gate(a, nseq, k_pre, k_post_out, forced_g, g_out, bits_out, ctx->esz, ctx->stream);
    } else if (ctx->cfg.dtype == WGKV_BF16) {
        const bool tc = ctx->cfg.attn_impl != WGKV_ATTN_SIMT && ctx->w1split;
        st = launch_gate_prefill<__nv_bfloat16>(a, nseq, (const __nv_bfloat16*)k_pre, (__nv_bfloat16*)k_post_out,
                                                g_out, bits_out, (int32_t*)ctx->ws_cand, ctx->ws_pcnt, nidx, ncap,
                                                ctx->ws_cnt + 1, tc ? ctx->w1split : nullptr,
                                                (long)ctx->cfg.layers * ctx->cfg.kv_heads * 4, ctx->ws_rope,
                                                ctx->stream);
    } else {
        st = launch_gate_prefill<float>(a, nseq, (const float*)k_pre, (float*)k_post_out, g_out, bits_out,
                                        (int32_t*)ctx->ws_cand, ctx->ws_pcnt, nidx, ncap, ctx->ws_cnt + 1, nullptr, 0,
                                        ctx->ws_rope, ctx->stream);
    }
    if (st) return fail(st, std::string("gate kernels: ") + cudaGetErrorString(cudaGetLastError()));
    if (near_count) {
        WGKV_CUDA_TRY(cudaMemcpyAsync(near_count, ctx->ws_cnt + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        WGKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    }
    return WGKV_OK;
}

int wgkv_gate_score_proj(wgkv_ctx* ctx, int layer, int nseq, long T, long pos0, const void* x, const void* wk, int dm,
                         void* k_pre_out, void* k_post_out, float* g_out, uint8_t* bits_out, int64_t* near_idx,
                         int near_cap, int* near_count) {
    if (!ctx || !x || !wk || !k_pre_out || !k_post_out || !g_out || !bits_out) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    int st = check_slots(ctx, layer, 0, nseq, T);
    if (st) return st;
    if (!ctx->gates_set) return fail(WGKV_ESTATE, "gate parameters not set");
    if (ctx->cfg.dtype != WGKV_BF16 || !ctx->w1split)
        return fail(WGKV_ENOTSUP, "gate_score_proj: bf16 contexts with d = hidden = 128 only");
    if (dm < 64 || dm % 64 != 0) return fail(WGKV_ENOTSUP, "gate_score_proj: model dim must be a multiple of 64");
    if (T == 0) return WGKV_OK;
    GateArgs a = ctx->gate_args(layer, T, pos0);
    int64_t* nidx = near_idx ? near_idx : ctx->ws_near;
    const int ncap = near_idx ? near_cap : (int)ctx->near_cap;
    WGKV_CUDA_TRY(cudaMemsetAsync(ctx->ws_cnt + 1, 0, sizeof(int), ctx->stream));
    WGKV_CUDA_TRY(cudaMemsetAsync(ctx->ws_pcnt, 0, sizeof(int) * nseq * ctx->cfg.kv_heads, ctx->stream));
    st = launch_gate_proj_tc(a, nseq, (const __nv_bfloat16*)x, (const __nv_bfloat16*)wk, dm, (__nv_bfloat16*)k_pre_out,
                             (__nv_bfloat16*)k_post_out, g_out, bits_out, (int32_t*)ctx->ws_cand, ctx->ws_pcnt,
                             ctx->w1split, (long)ctx->cfg.layers * ctx->cfg.kv_heads * 4, ctx->ws_rope, ctx->stream);
    if (!st)
        st = launch_gate_recheck<__nv_bfloat16>(a, nseq, (const __nv_bfloat16*)k_pre_out, g_out, bits_out,
                                                (int32_t*)ctx->ws_cand, ctx->ws_pcnt, nidx, ncap, ctx->ws_cnt + 1,
                                                ctx->stream);
    if (st) return fail(st, std::string("gate_proj kernels: ") + cudaGetErrorString(cudaGetLastError()));
    if (near_count) {
        WGKV_CUDA_TRY(cudaMemcpyAsync(near_count, ctx->ws_cnt + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        WGKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    }
    return WGKV_OK;
}

int wgkv_admit_prefill(wgkv_ctx* ctx, int layer, int seq0, int nseq, long T, const void* k_post, const void* v,
                       const float* g, const uint8_t* bits) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    int st = check_slots(ctx, layer, seq0, nseq, T);
    if (st) return st;
    if (T < 1) return fail(WGKV_EINVAL, "Session::prefill: empty prompt");
    if (T > ctx->cfg.max_tokens) return fail(WGKV_EINVAL, "T exceeds max_tokens");
    for (int s = seq0; s < seq0 + nseq; ++s)
        if (ctx->prefilled[(size_t)layer * ctx->cfg.max_seqs + s])
            return fail(WGKV_ESTATE, "prefill_populate: cache not empty");
    if (ctx->cfg.dtype == WGKV_BF16)
        st = launch_admit_prefill<__nv_bfloat16>(ctx->pv, layer, seq0, nseq, T, ctx->cfg.window,
                                                 (const __nv_bfloat16*)k_post, (const __nv_bfloat16*)v, g, bits,
                                                 ctx->ws_chunk, ctx->stream);
    else
        st = launch_admit_prefill<float>(ctx->pv, layer, seq0, nseq, T, ctx->cfg.window, (const float*)k_post,
                                         (const float*)v, g, bits, ctx->ws_chunk, ctx->stream);
    if (st) return fail(st, "admit kernels failed");
    for (int s = seq0; s < seq0 + nseq; ++s) {
        ctx->prefilled[(size_t)layer * ctx->cfg.max_seqs + s] = 1;
        ctx->tokens[(size_t)layer * ctx->cfg.max_seqs + s] = T;
    }
    if (ctx->quest_full)  // fresh Global pages: their Quest metadata is rebuilt at the next decode
        WGKV_CUDA_TRY(cudaMemsetAsync(ctx->quest_full + ctx->pv.head_index(layer, seq0, 0), 0,
                                      sizeof(int) * (size_t)nseq * ctx->cfg.kv_heads, ctx->stream));
    return WGKV_OK;
}

int wgkv_vs_prefill(wgkv_ctx* ctx, int layer, int seq0, int nseq, long T, const void* q, const void* k_post,
                    const void* v, const uint8_t* bits, void* out) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    int st = check_slots(ctx, layer, seq0, nseq, T);
    if (st) return st;
    VsArgs a{};
    a.pv = ctx->pv;
    a.layer = layer;
    a.seq0 = seq0;
    a.q_heads = ctx->cfg.q_heads;
    a.T = T;
    a.W = ctx->cfg.window;
    a.freq = ctx->freq;
    a.bits = bits;
    a.chunk_off = ctx->ws_chunk;
    if (ctx->peer_prefill) {  // C1 fused into K3: its epilogue also stores into every rank's bulk slot
        if ((long)nseq * T > ctx->px.max_bulk_rows)
            return fail(WGKV_EINVAL, "vs_prefill: nseq * T exceeds the peer exchange's max_bulk_rows");
        a.pb.peers = ctx->px.peers;
        a.pb.world = ctx->px.world;
        a.pb.rank = ctx->px.rank;
        a.pb.slot_off = peer_bulk_off(ctx->px, (int)(ctx->peer_bulk_seq % 2));
    }
    if (ctx->use_tc())
        st = launch_vs_prefill_tc(a, nseq, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k_post,
                                  (const __nv_bfloat16*)v, (__nv_bfloat16*)out, ctx->stream);
    else if (ctx->cfg.dtype == WGKV_BF16)
        st = launch_vs_prefill_simt<__nv_bfloat16>(a, nseq, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k_post,
                                                   (const __nv_bfloat16*)v, (__nv_bfloat16*)out, ctx->stream);
    else
        st = launch_vs_prefill_simt<float>(a, nseq, (const float*)q, (const float*)k_post, (const float*)v,
                                           (float*)out, ctx->stream);
    if (st) {
        const std::string detail = wgkv_last_error();  // the launcher's own message, if it set one
        return fail(st, std::string("vs prefill kernel: ") + cudaGetErrorString(cudaGetLastError()) +
                            (detail.empty() ? "" : " [" + detail + "]"));
    }
    if (ctx->peer_prefill) {  // completion: this rank's flag in every region, then every rank's here
        st = launch_peer_bulk_signal_wait(ctx->px, ctx->peer_wait_ranks, ctx->stream);
        if (st) return fail(st, "peer bulk signal / wait kernels failed");
        ++ctx->peer_bulk_seq;
    }
    return WGKV_OK;
}

int wgkv_prefill_layer(wgkv_ctx* ctx, int layer, int seq0, int nseq, long T, const void* q, const void* k_pre,
                       const void* v, const float* forced_g, void* out, float* g_out, uint8_t* bits_out) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    int st = check_slots(ctx, layer, seq0, nseq, T);
    if (st) return st;
    if (T < 1) return fail(WGKV_EINVAL, "Session::prefill: empty prompt");
    for (int s = seq0; s < seq0 + nseq; ++s)
        if (ctx->prefilled[(size_t)layer * ctx->cfg.max_seqs + s])
            return fail(WGKV_ESTATE, "Session::prefill: already prefilled");
    float* g = g_out ? g_out : ctx->ws_g;
    uint8_t* bits = bits_out ? bits_out : ctx->ws_bits;
    st = wgkv_gate_score(ctx, layer, nseq, T, 0, k_pre, forced_g, ctx->ws_kpost, g, bits, nullptr, 0, nullptr);
    if (st) return st;
    st = wgkv_admit_prefill(ctx, layer, seq0, nseq, T, ctx->ws_kpost, v, g, bits);
    if (st) return st;
    return wgkv_vs_prefill(ctx, layer, seq0, nseq, T, q, ctx->ws_kpost, v, bits, out);
}

static int decode_check(wgkv_ctx* ctx, int layer, int seq0, int nseq) {
    int st = check_slots(ctx, layer, seq0, nseq, 0);
    if (st) return st;
    for (int s = seq0; s < seq0 + nseq; ++s) {
        const size_t i = (size_t)layer * ctx->cfg.max_seqs + s;
        if (!ctx->prefilled[i]) return fail(WGKV_ESTATE, "Session::decode_step: prefill required first");
    }
    return WGKV_OK;
}

// split = true (decode_layer, non-deferred path): the route CTAs on the context
// stream, the gate CTAs forked onto gate_stream -- their g / bit is consumed
// only when the token leaves the ring -- and joined after the layer's attention
static int decode_append_impl(wgkv_ctx* ctx, int layer, int seq0, int nseq, const void* k_pre, const void* v,
                              const float* forced_g, const DecodeTrace& tr, bool split = false) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    int st = decode_check(ctx, layer, seq0, nseq);
    if (st) return st;
    for (int s = seq0; s < seq0 + nseq; ++s)
        if (ctx->tokens[(size_t)layer * ctx->cfg.max_seqs + s] >= ctx->cfg.max_tokens)
            return fail(WGKV_EINVAL, "sequence exceeds max_tokens");
    if (!forced_g && !ctx->gates_set) return fail(WGKV_ESTATE, "gate parameters not set");
    static const bool no_split = getenv("WGKV_APPEND_NOSPLIT") != nullptr;  // A/B switch
    split = split && !forced_g && !no_split;
    if (split && !ctx->gate_stream) {
        WGKV_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->gate_stream, cudaStreamNonBlocking));
        WGKV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_route, cudaEventDisableTiming));
        WGKV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_gate, cudaEventDisableTiming));
    }
    GateArgs ga = ctx->gate_args(layer, 1, 0);
    auto launch = [&](cudaStream_t sm, int mode) {
        if (ctx->cfg.dtype == WGKV_BF16)
            return launch_decode_append<__nv_bfloat16>(ctx->pv, ga, layer, seq0, nseq, ctx->cfg.window,
                                                       (const __nv_bfloat16*)k_pre, (const __nv_bfloat16*)v,
                                                       forced_g, tr, ctx->wk, sm, mode);
        return launch_decode_append<float>(ctx->pv, ga, layer, seq0, nseq, ctx->cfg.window, (const float*)k_pre,
                                           (const float*)v, forced_g, tr, ctx->wk, sm, mode);
    };
    if (split) {
        st = launch(ctx->stream, 1);
        if (!st) {
            WGKV_CUDA_TRY(cudaEventRecord(ctx->ev_route, ctx->stream));
            WGKV_CUDA_TRY(cudaStreamWaitEvent(ctx->gate_stream, ctx->ev_route, 0));
            st = launch(ctx->gate_stream, 2);
            WGKV_CUDA_TRY(cudaEventRecord(ctx->ev_gate, ctx->gate_stream));
            ctx->gate_join = true;
        }
    } else {
        st = launch(ctx->stream, 0);
    }
    if (st) return fail(st, "decode append kernel failed");
    for (int s = seq0; s < seq0 + nseq; ++s) ctx->tokens[(size_t)layer * ctx->cfg.max_seqs + s] += 1;
    return WGKV_OK;
}

static bool fast_decode(const wgkv_config& c) {
    return c.dtype == WGKV_BF16 && c.head_dim == 128 && c.page_size == 16 && c.q_heads / c.kv_heads <= 16 &&
           c.attn_impl != WGKV_ATTN_SIMT;
}

// the deferred append (decode_finish.cu): bf16 fast path without top-k
static bool defer_append(const wgkv_config& c) {
    static const bool off = getenv("WGKV_DECODE_NODEFER") != nullptr;  // A/B switch
    return !off && fast_decode(c) && c.topk_budget == 0;
}

// fin != null: deferred append -- K5 over the pre-append cache, then the
// finish kernel (merge + the new token + K4); the K5 counter was left at 0 by
// the previous merge kernel
static int decode_attn_impl(wgkv_ctx* ctx, int layer, int seq0, int nseq, const void* q, void* out,
                            const FinishArgs* fin) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    int st = decode_check(ctx, layer, seq0, nseq);
    if (st) return st;
    const auto& c = ctx->cfg;
    long tmax = 0;
    for (int s = seq0; s < seq0 + nseq; ++s) tmax = std::max(tmax, ctx->tokens[(size_t)layer * c.max_seqs + s]);
    // upper bound of resident pages per head: Global <= tokens - W entries
    const long gmax = tmax > c.window ? tmax - c.window : 0;
    const long np = (gmax + c.page_size - 1) / c.page_size + (c.window + c.page_size - 1) / c.page_size;
    const long target = (long)num_sms() * 4;
    long cp = (np * nseq * c.kv_heads + target - 1) / target;
    cp = std::max(cp, 4L);
    if (c.decode_chunk_pages > 0) cp = c.decode_chunk_pages;  // pinned split (SIMT path; K5 pins on device)
    cp = std::max(cp, (np + ctx->max_chunks - 1) / ctx->max_chunks);
    DecArgs a{};
    a.pv = ctx->pv;
    a.layer = layer;
    a.seq0 = seq0;
    a.q_heads = c.q_heads;
    a.chunk_pages = (int)cp;
    a.n_chunks = (int)((np + cp - 1) / cp);
    a.max_chunks = ctx->max_chunks;
    a.freq = ctx->freq;
    a.n_pairs = nseq * c.kv_heads;
    a.nchunks = nullptr;
    a.window = c.window;
    a.pin_cp = (int)std::min<long>(c.decode_chunk_pages, kDecPidCap);
    if (c.topk_budget > 0) {  // wgkv_plus_topk (engine.cpp:320-324)
        if (c.dtype == WGKV_BF16)
            st = launch_topk_decode<__nv_bfloat16>(a, nseq, c.topk_budget, (const __nv_bfloat16*)q, ctx->ws_score,
                                                   ctx->ws_sel, ctx->ws_nsel, ctx->ws_thr, ctx->ws_umask,
                                                   ctx->ws_ucnt, ctx->ws_part, ctx->ws_nchunks, (__nv_bfloat16*)out,
                                                   c.topk_mode, ctx->quest_meta, ctx->quest_full, ctx->stream);
        else
            st = launch_topk_decode<float>(a, nseq, c.topk_budget, (const float*)q, ctx->ws_score, ctx->ws_sel,
                                           ctx->ws_nsel, ctx->ws_thr, ctx->ws_umask, ctx->ws_ucnt, ctx->ws_part,
                                           ctx->ws_nchunks, (float*)out, c.topk_mode, nullptr, nullptr,
                                           ctx->stream);
        if (st) return fail(st, std::string("topk decode: ") + cudaGetErrorString(cudaGetLastError()));
        return WGKV_OK;
    }
    if (fin) {
        a.defer = 1;
        a.tokpos = ctx->ws_tokpos;
        st = launch_decode_attn_mma(a, nseq, (const __nv_bfloat16*)q, ctx->ws_part, ctx->ws_nchunks,
                                    (__nv_bfloat16*)out, ctx->stream, true, fin);
    } else if (fast_decode(c)) {
        st = launch_decode_attn_mma(a, nseq, (const __nv_bfloat16*)q, ctx->ws_part, ctx->ws_nchunks,
                                    (__nv_bfloat16*)out, ctx->stream, false);
    } else if (c.dtype == WGKV_BF16) {
        st = launch_decode_attn_simt<__nv_bfloat16>(a, nseq, (const __nv_bfloat16*)q, ctx->ws_part,
                                                    (__nv_bfloat16*)out, ctx->stream);
    } else {
        st = launch_decode_attn_simt<float>(a, nseq, (const float*)q, ctx->ws_part, (float*)out, ctx->stream);
    }
    if (st) return fail(st, std::string("decode attention: ") + cudaGetErrorString(cudaGetLastError()));
    return WGKV_OK;
}

int wgkv_decode_step_kv(wgkv_ctx* ctx, int layer, int seq0, int nseq, const void* k_pre, const void* v,
                        const float* forced_g, float* g_out, int32_t* events_out) {
    return decode_append_impl(ctx, layer, seq0, nseq, k_pre, v, forced_g,
                              DecodeTrace{g_out, nullptr, nullptr, events_out});
}

int wgkv_decode_attn(wgkv_ctx* ctx, int layer, int seq0, int nseq, const void* q, void* out) {
    return decode_attn_impl(ctx, layer, seq0, nseq, q, out, nullptr);
}

static PeerXchg peer_next(wgkv_ctx* ctx, bool push, bool unpack);
static void peer_pushed(wgkv_ctx* ctx, long rows);
static int peer_unpack_pending(wgkv_ctx* ctx);

// One decode layer.  bf16 fast path: K5 streams the cache as it was before
// this step's append and needs nothing in front of it; the finish kernel
// merges K5's chunks with the new token and runs the append (K4, exact fp64
// gate) beside the merge.  Other configurations: K4, then K5 / SIMT.
int wgkv_decode_layer_traced(wgkv_ctx* ctx, int layer, int seq0, int nseq, const void* q, const void* k_pre,
                             const void* v, const float* forced_g, void* out, const wgkv_decode_trace* trace) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    DecodeTrace tr{};
    if (trace) tr = DecodeTrace{trace->g, trace->bits, trace->near_tau, trace->events};
    if (ctx->peer_decode && nseq > ctx->px.max_rows)
        return fail(WGKV_EINVAL, "decode_layer: nseq exceeds the peer exchange's max_rows");
    if (!defer_append(ctx->cfg)) {
        int st = decode_append_impl(ctx, layer, seq0, nseq, k_pre, v, forced_g, tr, true);
        if (st) return st;
        st = decode_attn_impl(ctx, layer, seq0, nseq, q, out, nullptr);
        if (ctx->gate_join) {  // the append's gate CTAs ran beside the attention
            WGKV_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_gate, 0));
            ctx->gate_join = false;
        }
        if (st || !ctx->peer_decode) return st;
        // C1 over peer memory: a push kernel behind the layer (fp32 / top-k paths)
        st = launch_peer_push(static_cast<const uint8_t*>(out), peer_next(ctx, true, false), nseq, ctx->stream);
        if (st) return fail(st, "peer push kernel failed");
        if ((st = peer_unpack_pending(ctx))) return st;
        peer_pushed(ctx, nseq);
        return WGKV_OK;
    }
    int st = decode_check(ctx, layer, seq0, nseq);
    if (st) return st;
    for (int s = seq0; s < seq0 + nseq; ++s)
        if (ctx->tokens[(size_t)layer * ctx->cfg.max_seqs + s] >= ctx->cfg.max_tokens)
            return fail(WGKV_EINVAL, "sequence exceeds max_tokens");
    if (!forced_g && !ctx->gates_set) return fail(WGKV_ESTATE, "gate parameters not set");
    const bool prewait = ctx->finish_layer >= 0 && ctx->finish_layer != layer && ctx->finish_gen + 1 == ctx->api_gen;
    FinishArgs fin{};
    fin.prewait = prewait;
    fin.ga = ctx->gate_args(layer, 1, 0);
    fin.k_new = (const __nv_bfloat16*)k_pre;
    fin.v_new = (const __nv_bfloat16*)v;
    fin.forced_g = forced_g;
    fin.tr = tr;
    fin.wk = ctx->wk;
    // C1 over peer memory: the layer's merges push its output rows into every
    // rank's slot; the previous exchange is unpacked by one of its CTAs
    if (ctx->peer_decode) fin.px = peer_next(ctx, true, true);
    {  // this layer's parity halves (a fused launch may start before the previous layer's drained)
        const size_t SH = (size_t)ctx->cfg.max_seqs * ctx->cfg.kv_heads, par = (size_t)(layer & 1) * SH;
        fin.wk.slot += par;
        fin.wk.event += par;
        fin.wk.next += par;
        fin.wk.terms += par * ctx->cfg.hidden;  // the gate scratch too: a fused layer's gate CTAs
        fin.fw = ctx->fw;                        // run before the previous launch has drained
        fin.fw.cnt_gate += par;
        fin.fw.g += par;
        fin.fw.cnt_kv += par;
        fin.fw.cnt_gw += par;
        fin.fw.pub += par;
        fin.fw.started += layer & 1;
    }
    // the append's gate CTAs on a side stream forked before K5 and joined after
    // the finish kernel (WGKV_GATE_PLACE=side): they need nothing K5 produces
    static const char* gp_env = getenv("WGKV_GATE_PLACE");
    fin.gate_side = !forced_g && gp_env && strcmp(gp_env, "side") == 0;
    if (fin.gate_side) {
        if (!ctx->gate_stream) {
            WGKV_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->gate_stream, cudaStreamNonBlocking));
            WGKV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_route, cudaEventDisableTiming));
            WGKV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_gate, cudaEventDisableTiming));
        }
        WGKV_CUDA_TRY(cudaEventRecord(ctx->ev_route, ctx->stream));
        WGKV_CUDA_TRY(cudaStreamWaitEvent(ctx->gate_stream, ctx->ev_route, 0));
        st = launch_decode_append<__nv_bfloat16>(ctx->pv, fin.ga, layer, seq0, nseq, ctx->cfg.window, fin.k_new,
                                                 fin.v_new, nullptr, tr, ctx->wk, ctx->gate_stream, 3);
        if (st) return fail(st, "decode gate kernel failed");
        WGKV_CUDA_TRY(cudaEventRecord(ctx->ev_gate, ctx->gate_stream));
    }
    st = decode_attn_impl(ctx, layer, seq0, nseq, q, out, &fin);
    if (fin.gate_side) WGKV_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_gate, 0));
    if (st) return st;
    for (int s = seq0; s < seq0 + nseq; ++s) ctx->tokens[(size_t)layer * ctx->cfg.max_seqs + s] += 1;
    if (ctx->peer_decode) peer_pushed(ctx, nseq);
    ctx->finish_gen = ctx->api_gen;
    ctx->finish_layer = layer;
    return WGKV_OK;
}

int wgkv_decode_layer(wgkv_ctx* ctx, int layer, int seq0, int nseq, const void* q, const void* k_pre, const void* v,
                      const float* forced_g, void* out, float* g_out, int32_t* events_out) {
    const wgkv_decode_trace tr{g_out, nullptr, nullptr, events_out};
    return wgkv_decode_layer_traced(ctx, layer, seq0, nseq, q, k_pre, v, forced_g, out, &tr);
}

int wgkv_cache_state(wgkv_ctx* ctx, int layer, int seq, int kv_head, int64_t* lens) {
    if (!ctx || !lens) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    const auto& c = ctx->cfg;
    if (layer < 0 || layer >= c.layers || seq < 0 || seq >= c.max_seqs || kv_head < 0 || kv_head >= c.kv_heads)
        return fail(WGKV_EINVAL, "index out of range");
    WGKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    HeadState st;
    WGKV_CUDA_TRY(cudaMemcpy(&st, ctx->pv.state + ctx->pv.head_index(layer, seq, kv_head), sizeof(st),
                             cudaMemcpyDeviceToHost));
    const int ps = c.page_size;
    lens[0] = st.local_len;
    lens[1] = st.local_ptr;
    lens[2] = st.global_len;
    lens[3] = st.tokens_seen;
    lens[4] = (st.local_len + ps - 1) / ps;
    lens[5] = (st.global_len + ps - 1) / ps;
    return WGKV_OK;
}

int wgkv_cache_export(wgkv_ctx* ctx, int layer, int seq, int kv_head, float* gk, float* gv, int64_t* gpos,
                      float* ggate, float* lk, float* lv, int64_t* lpos, float* lgate) {
    int64_t lens[6];
    int st = wgkv_cache_state(ctx, layer, seq, kv_head, lens);
    if (st) return st;
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    const auto& c = ctx->cfg;
    const int d = c.head_dim;
    const long G = lens[2], Lc = lens[0], rows = G + Lc;
    if (rows == 0) return WGKV_OK;
    // one device gather (position order, kvstore.cpp:205-241) into a scratch
    // buffer, then one copy per output: K/V only when asked for
    const bool kv = gk || gv || lk || lv;
    const size_t kvn = kv ? (size_t)rows * d : 0;
    void* scratch = nullptr;
    const size_t bytes = 2 * kvn * sizeof(float) + (size_t)rows * (sizeof(float) + sizeof(int32_t));
    WGKV_CUDA_TRY(cudaMalloc(&scratch, bytes));
    float* dk = kv ? static_cast<float*>(scratch) : nullptr;
    float* dv = kv ? dk + kvn : nullptr;
    float* dg = static_cast<float*>(scratch) + 2 * kvn;
    int32_t* dp = reinterpret_cast<int32_t*>(dg + rows);
    const long hidx = ctx->pv.head_index(layer, seq, kv_head);
    const long start = Lc < c.window ? 0 : lens[1];  // ring unrolled oldest-first from local_ptr when full
    export_rows_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, ctx->stream>>>(ctx->pv, hidx, c.window, (int)G,
                                                                             (int)Lc, (int)start, (int)ctx->esz, dk,
                                                                             dv, dg, dp);
    cudaError_t e = cudaGetLastError();
    std::vector<int32_t> pos(rows);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    auto cp = [&](void* dst, const void* src, size_t n) {
        if (dst && n && e == cudaSuccess) e = cudaMemcpy(dst, src, n, cudaMemcpyDeviceToHost);
    };
    cp(gk, dk, sizeof(float) * G * d);
    cp(gv, dv, sizeof(float) * G * d);
    cp(lk, dk ? dk + G * d : nullptr, sizeof(float) * Lc * d);
    cp(lv, dv ? dv + G * d : nullptr, sizeof(float) * Lc * d);
    cp(ggate, dg, sizeof(float) * G);
    cp(lgate, dg + G, sizeof(float) * Lc);
    cp(pos.data(), dp, sizeof(int32_t) * rows);
    cudaFree(scratch);
    WGKV_CUDA_TRY(e);
    for (long r = 0; r < G; ++r)
        if (gpos) gpos[r] = pos[r];
    for (long r = 0; r < Lc; ++r)
        if (lpos) lpos[r] = pos[G + r];
    return WGKV_OK;
}

// cache_snapshot (kvstore.cpp:269-286) of one sequence slot: the reference's
// text format, caches in Session order (layer-major, then kv head), Global
// then Local entries in position order, gate printed with %.17g (the device
// keeps gates in fp32, so the digits are those of the fp32 value).
int wgkv_cache_snapshot(wgkv_ctx* ctx, int seq, char* buf, size_t cap, size_t* len) {
    if (!ctx || !len) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    const auto& c = ctx->cfg;
    if (seq < 0 || seq >= c.max_seqs) return fail(WGKV_EINVAL, "seq out of range");
    std::string text;
    char line[128];
    for (int l = 0; l < c.layers; ++l)
        for (int h = 0; h < c.kv_heads; ++h) {
            int64_t lens[6];
            int st = wgkv_cache_state(ctx, l, seq, h, lens);
            if (st) return st;
            const size_t G = (size_t)lens[2], Lc = (size_t)lens[0];
            std::vector<int64_t> gpos(G), lpos(Lc);
            std::vector<float> gg(G), lg(Lc);
            st = wgkv_cache_export(ctx, l, seq, h, nullptr, nullptr, gpos.data(), gg.data(), nullptr, nullptr,
                                   lpos.data(), lg.data());
            if (st) return st;
            for (size_t i = 0; i < G; ++i) {
                std::snprintf(line, sizeof(line), "%d %d global %ld %.17g\n", l, c.kv_head_offset + h, (long)gpos[i], (double)gg[i]);
                text += line;
            }
            for (size_t i = 0; i < Lc; ++i) {
                std::snprintf(line, sizeof(line), "%d %d local %ld %.17g\n", l, c.kv_head_offset + h, (long)lpos[i], (double)lg[i]);
                text += line;
            }
        }
    *len = text.size();
    if (buf) {
        if (cap <= text.size()) return fail(WGKV_EINVAL, "snapshot buffer too small (see *len)");
        std::memcpy(buf, text.data(), text.size());
        buf[text.size()] = 0;
    }
    return WGKV_OK;
}

int wgkv_cache_stats(wgkv_ctx* ctx, int seq0, int nseq, int64_t* out) {
    if (!ctx || !out) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    const auto& c = ctx->cfg;
    if (seq0 < 0 || nseq < 1 || seq0 + nseq > c.max_seqs) return fail(WGKV_EINVAL, "sequence slots out of range");
    WGKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    std::vector<HeadState> st((size_t)c.layers * c.max_seqs * c.kv_heads);
    WGKV_CUDA_TRY(cudaMemcpy(st.data(), ctx->pv.state, sizeof(HeadState) * st.size(), cudaMemcpyDeviceToHost));
    int64_t res = 0, glob = 0, seen = 0, pages = 0;
    for (int l = 0; l < c.layers; ++l)
        for (int s = seq0; s < seq0 + nseq; ++s)
            for (int h = 0; h < c.kv_heads; ++h) {
                const HeadState& x = st[ctx->pv.head_index(l, s, h)];
                res += x.local_len + x.global_len;
                glob += x.global_len;
                seen += x.tokens_seen;
                pages += (x.local_len + c.page_size - 1) / c.page_size + (x.global_len + c.page_size - 1) / c.page_size;
            }
    out[0] = res;
    out[1] = glob;
    out[2] = seen;
    out[3] = pages;
    return WGKV_OK;
}

int wgkv_release(wgkv_ctx* ctx, int seq0, int nseq) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    const auto& c = ctx->cfg;
    if (seq0 < 0 || nseq < 1 || seq0 + nseq > c.max_seqs) return fail(WGKV_EINVAL, "sequence slots out of range");
    release_kernel<<<c.layers * nseq * c.kv_heads, 256, 0, ctx->stream>>>(ctx->pv, c.layers, seq0, nseq);
    WGKV_CUDA_TRY(cudaGetLastError());
    for (int l = 0; l < c.layers; ++l) {
        for (int s = seq0; s < seq0 + nseq; ++s) {
            ctx->prefilled[(size_t)l * c.max_seqs + s] = 0;
            ctx->tokens[(size_t)l * c.max_seqs + s] = 0;
        }
        if (ctx->quest_full)
            WGKV_CUDA_TRY(cudaMemsetAsync(ctx->quest_full + ctx->pv.head_index(l, seq0, 0), 0,
                                          sizeof(int) * (size_t)nseq * c.kv_heads, ctx->stream));
    }
    return WGKV_OK;
}

int wgkv_pool_info(wgkv_ctx* ctx, int64_t* out) {
    if (!ctx || !out) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    WGKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    int32_t top = 0;
    WGKV_CUDA_TRY(cudaMemcpy(&top, ctx->pv.free_top, sizeof(top), cudaMemcpyDeviceToHost));
    out[0] = ctx->pv.capacity;
    out[1] = top;
    return WGKV_OK;
}

// ---- C1: head-output all-gather (comm.cu) ------------------------------------
int wgkv_comm_unique_id(uint8_t* id128) {
    if (!id128) return fail(WGKV_EINVAL, "null argument");
    const int st = comm_unique_id(id128);
    if (st) {
        std::string why;
        nccl_available(&why);
        return fail(st, "ncclGetUniqueId: " + why);
    }
    return WGKV_OK;
}

static int comm_setup(wgkv_ctx* ctx, int world, int rank) {
    const auto& c = ctx->cfg;
    if (c.kv_head_offset != rank * c.kv_heads)
        return fail(WGKV_EINVAL, "comm: rank r must own kv heads [r*kv_heads, (r+1)*kv_heads) (kv_head_offset)");
    if ((size_t)c.q_heads * c.head_dim * ctx->esz % 16 != 0)
        return fail(WGKV_ENOTSUP, "comm: a rank's head block per token must be a multiple of 16 bytes");
    ctx->world = world;
    ctx->rank = rank;
    // staging for one chunk of tokens from every rank (bounded: 8192 rows)
    ctx->stage_rows = std::max<long>(1, std::min<long>(ctx->cfg.max_prefill_tokens, 8192));
    const size_t bytes = (size_t)world * ctx->stage_rows * c.q_heads * c.head_dim * ctx->esz;
    WGKV_CUDA_TRY(cudaMalloc(&ctx->stage, bytes));
    WGKV_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    WGKV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_comm_in, cudaEventDisableTiming));
    WGKV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_comm_done, cudaEventDisableTiming));
    // f3: the chunked Wo's concat ring (chunks of <= 1024 rows: a 1024 x 4096 x 4096
    // GEMM chunk is ~25 us, enough to hide the next chunk's 8 MB exchange)
    ctx->cring_rows = std::min<long>(ctx->stage_rows, kOutProjChunkRows);
    WGKV_CUDA_TRY(cudaMalloc(&ctx->cring, 2 * (size_t)ctx->cring_rows * world * c.q_heads * c.head_dim * ctx->esz));
    for (int b = 0; b < 2; ++b) {
        WGKV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_ready[b], cudaEventDisableTiming));
        WGKV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_gemm[b], cudaEventDisableTiming));
    }
    return WGKV_OK;
}

int wgkv_comm_init(wgkv_ctx* ctx, const uint8_t* id128, int world, int rank) {
    if (!ctx || !id128) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    if (ctx->comm) return fail(WGKV_ESTATE, "comm: already initialised");
    if (world < 1 || rank < 0 || rank >= world) return fail(WGKV_EINVAL, "comm: bad world / rank");
    int st = comm_setup(ctx, world, rank);
    if (st) return st;
    std::string err;
    st = comm_init(&ctx->comm, id128, world, rank, &err);
    if (st) return fail(st, err);
    ctx->own_comm = true;
    return WGKV_OK;
}

int wgkv_comm_attach(wgkv_ctx* ctx, void* nccl_comm, int world, int rank) {
    if (!ctx || !nccl_comm) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    if (ctx->comm) return fail(WGKV_ESTATE, "comm: already initialised");
    if (world < 1 || rank < 0 || rank >= world) return fail(WGKV_EINVAL, "comm: bad world / rank");
    std::string why;
    if (!nccl_available(&why)) return fail(WGKV_ENOTSUP, why);
    const int st = comm_setup(ctx, world, rank);
    if (st) return st;
    ctx->comm = nccl_comm;
    return WGKV_OK;
}

int wgkv_allgather_heads(wgkv_ctx* ctx, int nseq, long T, const void* local_out, void* full_out, int async) {
    if (!ctx || !local_out || !full_out) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    const auto& c = ctx->cfg;
    if (nseq < 1 || T < 1) return fail(WGKV_EINVAL, "allgather_heads: empty");
    const size_t blk = (size_t)c.q_heads * c.head_dim * ctx->esz;  // one rank's heads of one token
    if (!ctx->comm) {  // a single device owns every head: the layout is already the reference's
        if (local_out != full_out)
            WGKV_CUDA_TRY(cudaMemcpyAsync(full_out, local_out, (size_t)nseq * T * blk, cudaMemcpyDeviceToDevice,
                                          ctx->stream));
        return WGKV_OK;
    }
    cudaStream_t st = ctx->stream;
    if (async) {  // on the comm stream, after everything enqueued so far on the compute stream
        WGKV_CUDA_TRY(cudaEventRecord(ctx->ev_comm_in, ctx->stream));
        WGKV_CUDA_TRY(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_comm_in, 0));
        st = ctx->comm_stream;
    }
    const auto* src = static_cast<const uint8_t*>(local_out);
    auto* dst = static_cast<uint8_t*>(full_out);
    std::string err;
    for (int s = 0; s < nseq; ++s)
        for (long t0 = 0; t0 < T; t0 += ctx->stage_rows) {
            const long n = std::min(ctx->stage_rows, T - t0);
            const int r = comm_allgather_assemble(ctx->comm, src + ((size_t)s * T + t0) * blk, ctx->stage, n * blk,
                                                  dst + ((size_t)s * T + t0) * blk * ctx->world, n, ctx->world, blk,
                                                  blk * ctx->world, st, &err);
            if (r) return fail(r, err.empty() ? std::string("assemble kernel failed") : err);
        }
    if (async) WGKV_CUDA_TRY(cudaEventRecord(ctx->ev_comm_done, ctx->comm_stream));
    return WGKV_OK;
}

int wgkv_output_proj(wgkv_ctx* ctx, int nseq, long T, const void* local_out, const void* wo, int dim, float* x) {
    if (!ctx || !local_out || !wo || !x) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    const auto& c = ctx->cfg;
    if (nseq < 1 || T < 1 || dim < 1) return fail(WGKV_EINVAL, "output_proj: empty");
    if (c.dtype != WGKV_BF16) return fail(WGKV_ENOTSUP, "output_proj: bf16 contexts only");
    const size_t blk = (size_t)c.q_heads * c.head_dim * ctx->esz;  // one rank's heads of one token
    const int K = ctx->world * c.q_heads * c.head_dim;               // Session's concat width
    const long rows = (long)nseq * T;
    std::string err;
    int st = blas_handle(&ctx->blas, &err);
    if (st) return fail(st, "output_proj: " + err);
    if (!ctx->comm) {  // one device owns every head: local_out is the concat
        st = gemm_rows_wt(ctx->blas, ctx->stream, rows, dim, K, local_out, wo, x, &err);
        return st ? fail(st, "output_proj: " + err) : WGKV_OK;
    }
    // chunk c: gather + assemble on the comm stream into ring slot c % 2 (after
    // the GEMM of chunk c - 2 released it), then its GEMM on the compute stream
    WGKV_CUDA_TRY(cudaEventRecord(ctx->ev_comm_in, ctx->stream));
    WGKV_CUDA_TRY(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_comm_in, 0));
    const auto* src = static_cast<const uint8_t*>(local_out);
    const size_t slot = (size_t)ctx->cring_rows * blk * ctx->world;
    long ci = 0;
    for (long r0 = 0; r0 < rows; r0 += ctx->cring_rows, ++ci) {
        const int b = (int)(ci & 1);
        const long n = std::min(ctx->cring_rows, rows - r0);
        uint8_t* buf = ctx->cring + b * slot;
        if (ci >= 2) WGKV_CUDA_TRY(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_gemm[b], 0));
        st = comm_allgather_assemble(ctx->comm, src + r0 * blk, ctx->stage, n * blk, buf, n, ctx->world, blk,
                                     blk * ctx->world, ctx->comm_stream, &err);
        if (st) return fail(st, err.empty() ? std::string("output_proj: assemble kernel failed") : err);
        WGKV_CUDA_TRY(cudaEventRecord(ctx->ev_ready[b], ctx->comm_stream));
        WGKV_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_ready[b], 0));
        st = gemm_rows_wt(ctx->blas, ctx->stream, n, dim, K, buf, wo, x + r0 * dim, &err);
        if (st) return fail(st, "output_proj: " + err);
        WGKV_CUDA_TRY(cudaEventRecord(ctx->ev_gemm[b], ctx->stream));
    }
    return WGKV_OK;
}

int wgkv_comm_join(wgkv_ctx* ctx) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    if (ctx->comm_stream) WGKV_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_comm_done, 0));
    return WGKV_OK;
}

// ---- C1 over peer memory ----------------------------------------------------

int wgkv_peer_region_bytes(int world, long max_rows, long max_bulk_rows, int q_heads, int head_dim, int dtype,
                           size_t* bytes) {
    if (!bytes || world < 1 || world > kMaxPeers || max_rows < 1 || max_bulk_rows < 0 || q_heads < 1 ||
        head_dim < 1 || (dtype != WGKV_BF16 && dtype != WGKV_F32))
        return fail(WGKV_EINVAL, "peer_region_bytes: bad argument");
    *bytes = peer_region_size(world, max_rows, max_bulk_rows, q_heads * head_dim * (dtype == WGKV_BF16 ? 2 : 4));
    return WGKV_OK;
}

int wgkv_peer_alloc(wgkv_ctx* ctx, int world, long max_rows, long max_bulk_rows, uint8_t* ipc_handle64,
                    void** base) {
    if (!ctx || !ipc_handle64) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    if (ctx->peer_own) return fail(WGKV_ESTATE, "peer_alloc: region already allocated");
    size_t bytes = 0;
    int st = wgkv_peer_region_bytes(world, max_rows, max_bulk_rows, ctx->cfg.q_heads, ctx->cfg.head_dim,
                                    ctx->cfg.dtype, &bytes);
    if (st) return st;
    WGKV_CUDA_TRY(cudaMalloc(&ctx->peer_own, bytes));
    WGKV_CUDA_TRY(cudaMemset(ctx->peer_own, 0, bytes));
    cudaIpcMemHandle_t h;
    WGKV_CUDA_TRY(cudaIpcGetMemHandle(&h, ctx->peer_own));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(ipc_handle64, &h, 64);
    ctx->peer_own_world = world;
    ctx->peer_own_rows = max_rows;
    ctx->peer_own_bulk = max_bulk_rows;
    if (base) *base = ctx->peer_own;
    return WGKV_OK;
}

static int peer_check_args(wgkv_ctx* ctx, int world, int rank, long max_rows, int wait_ranks) {
    if (ctx->px.world) return fail(WGKV_ESTATE, "peer: already attached");
    if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world || max_rows < 1 || wait_ranks < 1 ||
        wait_ranks > world)
        return fail(WGKV_EINVAL, "peer: bad world / rank / max_rows / wait_ranks");
    if (ctx->cfg.dtype != WGKV_BF16) return fail(WGKV_ENOTSUP, "peer: bf16 contexts only");
    return WGKV_OK;
}

static int peer_bind(wgkv_ctx* ctx, int world, int rank, long max_rows, long max_bulk_rows, uint8_t* const* bases,
                     int wait_ranks) {
    PeerXchg x{};
    for (int p = 0; p < world; ++p) x.peers.base[p] = bases[p];
    x.world = world;
    x.rank = rank;
    x.blk = ctx->cfg.q_heads * ctx->cfg.head_dim * (int)ctx->esz;
    x.max_rows = max_rows;
    x.max_bulk_rows = max_bulk_rows;
    ctx->px = x;
    ctx->peer_wait_ranks = wait_ranks;
    ctx->peer_seq = 0;
    ctx->peer_bulk_seq = 0;
    ctx->pend_slot = -1;
    return WGKV_OK;
}

int wgkv_peer_open(wgkv_ctx* ctx, int world, int rank, const uint8_t* handles, int wait_ranks) {
    if (!ctx || !handles) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    if (!ctx->peer_own) return fail(WGKV_ESTATE, "peer_open: wgkv_peer_alloc first");
    int st = peer_check_args(ctx, world, rank, ctx->peer_own_rows, wait_ranks);
    if (st) return st;
    if (world != ctx->peer_own_world) return fail(WGKV_EINVAL, "peer_open: world differs from peer_alloc's");
    uint8_t* bases[kMaxPeers] = {};
    for (int p = 0; p < world; ++p) {
        if (p == rank) {
            bases[p] = ctx->peer_own;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + 64 * (size_t)p, 64);
        void* ptr = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            for (void* q : ctx->peer_ipc) cudaIpcCloseMemHandle(q);
            ctx->peer_ipc.clear();
            return fail(WGKV_ECUDA, std::string("peer_open: cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
        }
        ctx->peer_ipc.push_back(ptr);
        bases[p] = static_cast<uint8_t*>(ptr);
    }
    return peer_bind(ctx, world, rank, ctx->peer_own_rows, ctx->peer_own_bulk, bases, wait_ranks);
}

int wgkv_peer_attach(wgkv_ctx* ctx, int world, int rank, long max_rows, long max_bulk_rows, void* const* bases,
                     int wait_ranks) {
    if (!ctx || !bases) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    int st = peer_check_args(ctx, world, rank, max_rows, wait_ranks);
    if (st) return st;
    if (max_bulk_rows < 0) return fail(WGKV_EINVAL, "peer_attach: max_bulk_rows < 0");
    uint8_t* b[kMaxPeers] = {};
    for (int p = 0; p < world; ++p) {
        b[p] = static_cast<uint8_t*>(bases[p]);
        if (!b[p] || reinterpret_cast<uintptr_t>(b[p]) % 16 != 0)
            return fail(WGKV_EINVAL, "peer_attach: null or unaligned region");
    }
    return peer_bind(ctx, world, rank, max_rows, max_bulk_rows, b, wait_ranks);
}

// the exchange description for the next push (rows) and the pending unpack
static PeerXchg peer_next(wgkv_ctx* ctx, bool push, bool unpack) {
    PeerXchg x = ctx->px;
    x.do_push = push ? 1 : 0;
    x.push_slot = (int)(ctx->peer_seq % kPeerSlots);
    x.do_unpack = unpack && ctx->pend_slot >= 0 ? 1 : 0;
    x.unpack_slot = ctx->pend_slot;
    x.unpack_rows = (int)ctx->pend_rows;
    x.unpack_ranks = ctx->peer_wait_ranks;
    return x;
}

// the exchange just pushed becomes the pending one (the previous pending one
// was unpacked by the caller: peer_unpack_pending or the decode layer's CTA)
static void peer_pushed(wgkv_ctx* ctx, long rows) {
    ctx->pend_slot = (int)(ctx->peer_seq % kPeerSlots);
    ctx->pend_rows = rows;
    ++ctx->peer_seq;
}

// a peer kernel right behind a decode layer keeps that layer's launch chain:
// the next layer's K5 may still plan before its PDL wait (see wgkv_decode_layer)
static void peer_keep_chain(wgkv_ctx* ctx, uint64_t gen_before) {
    if (ctx->finish_gen == gen_before) ctx->finish_gen = ctx->api_gen;
}

static int peer_unpack_pending(wgkv_ctx* ctx) {
    if (ctx->pend_slot < 0) return WGKV_OK;
    const int st = launch_peer_unpack(peer_next(ctx, false, true), ctx->stream);
    if (st) return fail(st, "peer unpack kernel failed");
    ctx->pend_slot = -1;
    return WGKV_OK;
}

int wgkv_peer_allgather_heads(wgkv_ctx* ctx, long rows, const void* local_out, int wait) {
    if (!ctx || !local_out) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    const uint64_t g0 = ctx->api_gen++;
    if (!ctx->px.world) return fail(WGKV_ESTATE, "peer_allgather_heads: no peer regions attached");
    if (rows < 1 || rows > ctx->px.max_rows) return fail(WGKV_EINVAL, "peer_allgather_heads: rows outside [1, max_rows]");
    int st = launch_peer_push(static_cast<const uint8_t*>(local_out), peer_next(ctx, true, false), rows, ctx->stream);
    if (st) return fail(st, "peer push kernel failed");
    if ((st = peer_unpack_pending(ctx))) return st;  // exchanges are unpacked in order
    peer_pushed(ctx, rows);
    if (wait && (st = peer_unpack_pending(ctx))) return st;
    peer_keep_chain(ctx, g0);
    return WGKV_OK;
}

int wgkv_peer_wait(wgkv_ctx* ctx) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    DevGuard dg_(ctx->cfg.device);
    const uint64_t g0 = ctx->api_gen++;
    if (!ctx->px.world) return fail(WGKV_ESTATE, "peer_wait: no peer regions attached");
    const int st = peer_unpack_pending(ctx);
    if (st) return st;
    peer_keep_chain(ctx, g0);
    return WGKV_OK;
}

int wgkv_peer_decode(wgkv_ctx* ctx, int on) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    ++ctx->api_gen;
    if (on && !ctx->px.world) return fail(WGKV_ESTATE, "peer_decode: no peer regions attached");
    ctx->peer_decode = on != 0;
    return WGKV_OK;
}

int wgkv_peer_prefill(wgkv_ctx* ctx, int on) {
    if (!ctx) return fail(WGKV_EINVAL, "null ctx");
    ++ctx->api_gen;
    if (on && (!ctx->px.world || ctx->px.max_bulk_rows < 1))
        return fail(WGKV_ESTATE, "peer_prefill: no peer regions with a bulk part attached");
    if (on && !ctx->use_tc()) return fail(WGKV_ENOTSUP, "peer_prefill: the tcgen05 prefill path only");
    ctx->peer_prefill = on != 0;
    return WGKV_OK;
}

int wgkv_peer_bulk_result(wgkv_ctx* ctx, int back, void** ptr) {
    if (!ctx || !ptr) return fail(WGKV_EINVAL, "null argument");
    ++ctx->api_gen;
    if (!ctx->px.world || ctx->px.max_bulk_rows < 1) return fail(WGKV_ESTATE, "peer_bulk_result: no bulk part");
    if (back < 0 || back >= 2 || (uint64_t)back >= ctx->peer_bulk_seq)
        return fail(WGKV_EINVAL, "peer_bulk_result: no such exchange");
    *ptr = ctx->px.peers.base[ctx->px.rank] + peer_bulk_off(ctx->px, (int)((ctx->peer_bulk_seq - 1 - back) % 2));
    return WGKV_OK;
}

int wgkv_peer_result(wgkv_ctx* ctx, int back, void** ptr) {
    if (!ctx || !ptr) return fail(WGKV_EINVAL, "null argument");
    ++ctx->api_gen;
    if (!ctx->px.world) return fail(WGKV_ESTATE, "peer_result: no peer regions attached");
    if (back < 0 || back >= kPeerSlots || (uint64_t)back >= ctx->peer_seq)
        return fail(WGKV_EINVAL, "peer_result: no such exchange");
    const int slot = (int)((ctx->peer_seq - 1 - back) % kPeerSlots);
    *ptr = ctx->px.peers.base[ctx->px.rank] + peer_res_off(ctx->px, slot);
    return WGKV_OK;
}

int wgkv_assemble_heads(int world, long rows, size_t blk_bytes, const void* rank_major, void* full_out,
                        void* stream) {
    if (world < 1 || rows < 0 || !rank_major || !full_out) return fail(WGKV_EINVAL, "bad argument");
    const int st = launch_assemble(static_cast<const uint8_t*>(rank_major), static_cast<uint8_t*>(full_out), rows,
                                   world, blk_bytes, blk_bytes * world, static_cast<cudaStream_t>(stream));
    return st ? fail(st, "assemble_heads: blocks must be 16-byte multiples") : WGKV_OK;
}

// diagnostics (not part of the C-ABI contract): out[0] = tokens the last
// wgkv_gate_score listed for the fp64 recheck, out[1] = reported near-tau tokens
extern "C" int wgkv_dbg_gate_counts(wgkv_ctx* ctx, int* out) {
    if (!ctx || !out) return fail(WGKV_EINVAL, "null argument");
    DevGuard dg_(ctx->cfg.device);
    ++ctx->api_gen;
    WGKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    std::vector<int> pc((size_t)ctx->cfg.max_seqs * ctx->cfg.kv_heads);
    WGKV_CUDA_TRY(cudaMemcpy(pc.data(), ctx->ws_pcnt, sizeof(int) * pc.size(), cudaMemcpyDeviceToHost));
    out[0] = 0;
    for (int v : pc) out[0] += v;
    WGKV_CUDA_TRY(cudaMemcpy(out + 1, ctx->ws_cnt + 1, sizeof(int), cudaMemcpyDeviceToHost));
    return WGKV_OK;
}

// closed form of vs_mask_pair_count (attention.cpp:182-191) for T queries
// over T keys at offset 0: sum_i min(i+1, W) + C(i-W+1), C(x) = #admitted j < x
uint64_t wgkv_vs_pair_count(const uint8_t* bits, long T, long W) {
    uint64_t total = 0, c = 0;
    for (long i = 0; i < T; ++i) {
        const long x = i - W + 1;  // admitted j < x are outside the window
        if (x > 0) c += bits[x - 1] != 0;
        total += (uint64_t)std::min(i + 1, W) + (x > 0 ? c : 0);
    }
    return total;
}

}  // extern "C"
