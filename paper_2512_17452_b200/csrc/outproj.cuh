// outproj.cuh -- f3 output projection helpers (outproj.cu): cuBLAS at run time.
#pragma once
#include <string>

#include "common.cuh"

namespace wgkv {

constexpr long kOutProjChunkRows = 1024;  // rows per overlapped chunk of wgkv_output_proj

int blas_handle(void** handle, std::string* err);  // create on first use
void blas_destroy(void* handle);
// x[rows][dim] (fp32) += a[rows][k] (bf16) . w[dim][k]^T (bf16) on stream st
int gemm_rows_wt(void* handle, cudaStream_t st, long rows, int dim, int k, const void* a, const void* w, float* x,
                 std::string* err);

}  // namespace wgkv
