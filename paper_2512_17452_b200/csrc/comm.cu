// comm.cu -- C1: the head-output all-gather of KV-head sharding.
//
// The path partitions by KV head (gate MLPs, caches and attention are per
// (layer, kv head)): rank r of N owns kv heads [r*H/N, (r+1)*H/N) and their GQA
// q heads, so its attention output holds q heads [r*Hq/N, (r+1)*Hq/N).  The
// only exchange is rebuilding Session's concat layout -- q head p at columns
// p*d of row t (engine.cpp:234-238) -- on every rank: NCCL all-gathers each
// rank's [T][Hq/N][d] block over NVLink into a rank-major staging buffer, and
// an assemble kernel scatters the blocks into [T][Hq][d].  Prefill moves the
// tokens in chunks through a staging buffer sized at wgkv_comm_init, on the
// context's comm stream when asked (async: the exchange of layer l overlaps
// the attention of layer l+1 the caller enqueues next on the compute stream);
// decode messages are KB-sized and go straight through on the compute stream
// (capturable in the per-token CUDA graph).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2", reusing the copy torch
// already loaded if any), so the library itself loads on hosts without it;
// only wgkv_comm_init / wgkv_comm_attach need it.
//
// The same exchange without NCCL (wgkv_peer_*, layout and device helpers in
// comm.cuh): the decode merge and K3's epilogue store their rows straight into
// every rank's mapped region; this file holds the standalone push / unpack /
// bulk signal / wait kernels around them.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "comm.cuh"

namespace wgkv {

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.error_string;
        if (!api.ok) api.why = "libnccl.so.2 lacks the expected symbols";
    });
    return api;
}

// rank-major staging [world][rows][blk] -> out rows [rows][world * blk]; 16-byte vectors
__global__ void assemble_heads_kernel(const uint8_t* __restrict__ stage, uint8_t* __restrict__ out, long rows,
                                      int world, size_t blk_bytes, size_t out_row_bytes) {
    const size_t vec_per_blk = blk_bytes / 16;
    const size_t total = (size_t)rows * world * vec_per_blk;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t v = i % vec_per_blk, rb = i / vec_per_blk;
        const int r = (int)(rb % world);
        const size_t row = rb / world;
        const int4 x = reinterpret_cast<const int4*>(stage + ((size_t)r * rows + row) * blk_bytes)[v];
        reinterpret_cast<int4*>(out + row * out_row_bytes + (size_t)r * blk_bytes)[v] = x;
    }
}

}  // namespace

bool nccl_available(std::string* why) {
    const NcclApi& a = nccl();
    if (!a.ok && why) *why = a.why;
    return a.ok;
}

int comm_unique_id(uint8_t* out) {
    const NcclApi& a = nccl();
    if (!a.ok) return WGKV_ENOTSUP;
    ncclUniqueId id;
    if (a.get_unique_id(&id) != ncclSuccess) return WGKV_ERUNTIME;
    std::memcpy(out, id.internal, sizeof(id.internal));
    return WGKV_OK;
}

int comm_init(void** comm, const uint8_t* id_bytes, int world, int rank, std::string* err) {
    const NcclApi& a = nccl();
    if (!a.ok) {
        *err = a.why;
        return WGKV_ENOTSUP;
    }
    ncclUniqueId id;
    std::memcpy(id.internal, id_bytes, sizeof(id.internal));
    ncclComm_t c = nullptr;
    const ncclResult_t r = a.comm_init_rank(&c, world, id, rank);
    if (r != ncclSuccess) {
        *err = std::string("ncclCommInitRank: ") + a.error_string(r);
        return WGKV_ERUNTIME;
    }
    *comm = c;
    return WGKV_OK;
}

void comm_destroy(void* comm) {
    if (comm && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

// one all-gather of `bytes` per rank into stage ([world][bytes]), then the
// assembly of `rows` rows of `blk` bytes per rank into out
int comm_allgather_assemble(void* comm, const void* send, uint8_t* stage, size_t bytes, uint8_t* out, long rows,
                            int world, size_t blk, size_t out_row_bytes, cudaStream_t st, std::string* err) {
    const NcclApi& a = nccl();
    const ncclResult_t r = a.all_gather(send, stage, bytes, ncclUint8, static_cast<ncclComm_t>(comm), st);
    if (r != ncclSuccess) {
        *err = std::string("ncclAllGather: ") + a.error_string(r);
        return WGKV_ERUNTIME;
    }
    return launch_assemble(stage, out, rows, world, blk, out_row_bytes, st);
}

int launch_assemble(const uint8_t* stage, uint8_t* out, long rows, int world, size_t blk, size_t out_row_bytes,
                    cudaStream_t st) {
    if (blk % 16 != 0 || out_row_bytes % 16 != 0) return WGKV_ENOTSUP;
    const size_t total = (size_t)rows * world * (blk / 16);
    const int grid = (int)std::min<size_t>((total + 255) / 256, (size_t)num_sms() * 8);
    if (grid > 0) assemble_heads_kernel<<<grid, 256, 0, st>>>(stage, out, rows, world, blk, out_row_bytes);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}


// ---- C1 over peer memory (decode-sized exchanges; layout in comm.cuh) ----------
namespace {

// this rank's rows [rows][blk] as LL words into every rank's push slot
__global__ void __launch_bounds__(256) peer_push_kernel(const uint8_t* __restrict__ src, PeerXchg x, long rows) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // src: the attention output in front of us
    const uint32_t flag = peer_push_flag(x);
    const int wpr = x.blk / 4;
    const long total = rows * wpr;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x)
        peer_push_word(x, flag, i / wpr, (int)(i % wpr), reinterpret_cast<const uint32_t*>(src)[i]);
}

__global__ void __launch_bounds__(256) peer_unpack_kernel(PeerXchg x) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    peer_unpack_cta(x);
}

// after K3 (stream order: its stores, local and remote, are performed): a
// system-scope fence, then this rank's flag (bulk epoch + 1) in every region
__global__ void peer_bulk_signal_kernel(PeerXchg x) {
    if (threadIdx.x != 0) return;
    __threadfence_system();
    const uint32_t e = *reinterpret_cast<volatile uint32_t*>(x.peers.base[x.rank] + 4 * kPeerBulkEpoch) + 1u;
    for (int p = 0; p < x.world; ++p)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(x.peers.base[p] + 4 * (kPeerBulkFlag + x.rank)),
                     "r"(e)
                     : "memory");
}

// every awaited rank's flag has reached this exchange (>=: a faster rank may
// already have signalled the next one), then the epoch advances
__global__ void peer_bulk_wait_kernel(PeerXchg x, int ranks) {
    if (threadIdx.x != 0) return;
    uint8_t* own = x.peers.base[x.rank];
    const uint32_t e = *reinterpret_cast<volatile uint32_t*>(own + 4 * kPeerBulkEpoch) + 1u;
    const unsigned long long t0 = peer_now();
    for (int r = 0; r < ranks; ++r) {
        uint32_t f;
        do {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(f) : "l"(own + 4 * (kPeerBulkFlag + r)) : "memory");
            if ((int)(f - e) < 0) {
                if (peer_now() - t0 > kPeerTimeoutNs) __trap();  // a rank never signalled (comm.cuh)
                __nanosleep(64);
            }
        } while ((int)(f - e) < 0);
    }
    *reinterpret_cast<volatile uint32_t*>(own + 4 * kPeerBulkEpoch) = e;
}

template <typename K, typename... Args>
int launch_pdl(K kern, int grid, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

}  // namespace

int launch_peer_push(const uint8_t* src, const PeerXchg& x, long rows, cudaStream_t st) {
    const long total = rows * (x.blk / 4);
    return launch_pdl(peer_push_kernel, (int)std::max<long>(1, std::min<long>((total + 255) / 256, 64)), st, src, x,
                      rows);
}

int launch_peer_unpack(const PeerXchg& x, cudaStream_t st) { return launch_pdl(peer_unpack_kernel, 1, st, x); }

int launch_peer_bulk_signal_wait(const PeerXchg& x, int ranks, cudaStream_t st) {
    peer_bulk_signal_kernel<<<1, 32, 0, st>>>(x);
    peer_bulk_wait_kernel<<<1, 32, 0, st>>>(x, ranks);
    return cudaGetLastError() == cudaSuccess ? WGKV_OK : WGKV_ECUDA;
}

}  // namespace wgkv
