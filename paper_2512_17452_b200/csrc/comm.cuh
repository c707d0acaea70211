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

}  // namespace wgkv
