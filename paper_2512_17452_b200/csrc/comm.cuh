// comm.cuh -- C1 head-output all-gather (comm.cu): NCCL resolved at run time.
#pragma once
#include <string>

#include "common.cuh"

namespace wgkv {

bool nccl_available(std::string* why);
int comm_unique_id(uint8_t* out128);
int comm_init(void** comm, const uint8_t* id128, int world, int rank, std::string* err);
void comm_destroy(void* comm);
// all-gather `bytes` per rank into stage [world][bytes], then assemble `rows`
// rows of `blk` bytes per rank into out rows of out_row_bytes
int comm_allgather_assemble(void* comm, const void* send, uint8_t* stage, size_t bytes, uint8_t* out, long rows,
                            int world, size_t blk, size_t out_row_bytes, cudaStream_t st, std::string* err);
// rank-major [world][rows][blk] -> rows [rows][world * blk] (16-byte multiples)
int launch_assemble(const uint8_t* stage, uint8_t* out, long rows, int world, size_t blk, size_t out_row_bytes,
                    cudaStream_t st);

// ---- C1 over peer memory (comm.cu) --------------------------------------------
// Every rank owns an exchange region, mapped into every rank:
//   [kPeerHeader: uint32 epoch per slot, bulk epoch, bulk flags][kPeerSlots LL slots]
//   [kPeerSlots result slots][2 bulk slots]
// LL slot: [max_rows][world][blk / 4] 8-byte words {4 data bytes, 4 flag bytes}
// (the flag is the slot's epoch + 1: a reader polls the data itself, so a push
// needs no fence and no counter); result slot: [max_rows][world * blk] bytes,
// the reference's concat layout.  Exchange k uses slot k % kPeerSlots.
// Bulk slot (prefill): [max_bulk_rows][world * blk], written by K3's epilogue
// straight into every rank's region (plain stores: the data is large, the
// completion is one flag per rank: fence + release store, acquire polls).
constexpr int kMaxPeers = 8;
constexpr int kPeerSlots = 4;        // see wgkv_b200.h: the slot reuse distance that no rank can outrun
constexpr size_t kPeerHeader = 256;  // uint32 epoch per slot, padded
constexpr int kPeerBulkEpoch = 16;   // header word: bulk exchanges completed here
constexpr int kPeerBulkFlag = 32;    // header words [32, 32 + kMaxPeers): rank r's last bulk signal

struct PeerBases {
    uint8_t* base[kMaxPeers];  // every rank's region, as mapped in this process
};

// one exchange as the kernels see it (push of this layer's rows, unpack of a
// pending exchange); slot < 0 = none
struct PeerXchg {
    PeerBases peers;
    int world, rank;
    int blk;        // bytes of one row of one rank (q_heads * d * esz)
    long max_rows;
    long max_bulk_rows;
    int do_push, push_slot;                               // push this layer's output rows
    int do_unpack, unpack_slot, unpack_rows, unpack_ranks;  // unpack a pending exchange (one CTA)
};

__host__ __device__ inline size_t peer_round(size_t x) { return (x + kPeerHeader - 1) / kPeerHeader * kPeerHeader; }
__host__ __device__ inline size_t peer_ll_bytes(int world, long max_rows, int blk) {
    return peer_round((size_t)max_rows * world * (blk / 4) * 8);
}
__host__ __device__ inline size_t peer_res_bytes(int world, long max_rows, int blk) {
    return peer_round((size_t)max_rows * world * blk);
}
__host__ __device__ inline size_t peer_bulk_bytes(int world, long max_bulk_rows, int blk) {
    return peer_round((size_t)max_bulk_rows * world * blk);
}
__host__ __device__ inline size_t peer_region_size(int world, long max_rows, long max_bulk_rows, int blk) {
    return kPeerHeader + kPeerSlots * (peer_ll_bytes(world, max_rows, blk) + peer_res_bytes(world, max_rows, blk)) +
           2 * peer_bulk_bytes(world, max_bulk_rows, blk);
}
__host__ __device__ inline size_t peer_ll_off(const PeerXchg& x, int slot) {
    return kPeerHeader + (size_t)slot * peer_ll_bytes(x.world, x.max_rows, x.blk);
}
__host__ __device__ inline size_t peer_res_off(const PeerXchg& x, int slot) {
    return kPeerHeader + kPeerSlots * peer_ll_bytes(x.world, x.max_rows, x.blk) +
           (size_t)slot * peer_res_bytes(x.world, x.max_rows, x.blk);
}

__host__ __device__ inline size_t peer_bulk_off(const PeerXchg& x, int slot) {
    return kPeerHeader + kPeerSlots * (peer_ll_bytes(x.world, x.max_rows, x.blk) + peer_res_bytes(x.world, x.max_rows, x.blk)) +
           (size_t)slot * peer_bulk_bytes(x.world, x.max_bulk_rows, x.blk);
}

// K3's view of a bulk exchange: its output rows also go to every rank's bulk slot
struct PeerBulk {
    PeerBases peers;
    int world, rank;   // world = 0: off
    size_t slot_off;   // byte offset of the bulk slot in every region
};

#ifdef __CUDACC__
// a peer that never arrives (a rank died or diverged from the exchange
// sequence) must not hang the GPU forever: after kPeerTimeoutNs of polling the
// kernel traps, and the host sees a launch failure instead of a hang
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long peer_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// the flag of this rank's push into x.push_slot: the slot's epoch (unpacks so
// far, identical on every rank) + 1
__device__ __forceinline__ uint32_t peer_push_flag(const PeerXchg& x) {
    uint32_t e;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];"
                 : "=r"(e)
                 : "l"(reinterpret_cast<const uint32_t*>(x.peers.base[x.rank]) + x.push_slot));
    return e + 1u;
}
// word j (4 bytes) of row `row` of this rank's block, into every rank's LL slot
__device__ __forceinline__ void peer_push_word(const PeerXchg& x, uint32_t flag, long row, int j, uint32_t data) {
    const size_t off = peer_ll_off(x, x.push_slot) + (((size_t)row * x.world + x.rank) * (x.blk / 4) + j) * 8;
#pragma unroll 1
    for (int p = 0; p < x.world; ++p)
        asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(x.peers.base[p] + off), "r"(data), "r"(flag)
                     : "memory");
}
// one CTA: wait for ranks [0, unpack_ranks)'s words of x.unpack_slot (flag =
// epoch + 1), write them into the result slot, then advance the slot's epoch
__device__ __forceinline__ void peer_unpack_cta(const PeerXchg& x) {
    uint8_t* own = x.peers.base[x.rank];
    uint32_t* ep = reinterpret_cast<uint32_t*>(own) + x.unpack_slot;
    const uint32_t flag = *reinterpret_cast<volatile uint32_t*>(ep) + 1u;
    const uint8_t* ll = own + peer_ll_off(x, x.unpack_slot);
    uint8_t* res = own + peer_res_off(x, x.unpack_slot);
    const int wpr = x.blk / 4;
    const long total = (long)x.unpack_rows * x.unpack_ranks * wpr;
    for (long i = threadIdx.x; i < total; i += blockDim.x) {
        const long row = i / ((long)x.unpack_ranks * wpr);
        const int r = (int)((i / wpr) % x.unpack_ranks), j = (int)(i % wpr);
        const uint8_t* src = ll + (((size_t)row * x.world + r) * wpr + j) * 8;
        uint32_t dv, fv;
        asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(dv), "=r"(fv) : "l"(src) : "memory");
        if (fv != flag) {
            const unsigned long long t0 = peer_now();
            do {
                if (peer_now() - t0 > kPeerTimeoutNs) __trap();
                asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(dv), "=r"(fv) : "l"(src) : "memory");
            } while (fv != flag);
        }
        *reinterpret_cast<uint32_t*>(res + (size_t)row * x.world * x.blk + (size_t)r * x.blk + (size_t)j * 4) = dv;
    }
    __syncthreads();
    if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t*>(ep) = flag;
}
#endif

// standalone kernels (wgkv_peer_allgather_heads, wgkv_peer_wait, non-deferred decode)
int launch_peer_push(const uint8_t* src, const PeerXchg& x, long rows, cudaStream_t st);
int launch_peer_unpack(const PeerXchg& x, cudaStream_t st);
// bulk completion: this rank's signal to every rank, then the wait for ranks [0, ranks)
int launch_peer_bulk_signal_wait(const PeerXchg& x, int ranks, cudaStream_t st);

}  // namespace wgkv
