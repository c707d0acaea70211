// outproj.cu -- f3: the output projection Wo after the head all-gather
// (engine.cpp:243-245 prefill: x[t] += Wo . concat[t]; engine.cpp:331 decode).
//
// Wo is a plain dense GEMM (concat [rows][Hq*d] x Wo^T [Hq*d][dim]), so it runs
// on cuBLAS (bf16 operands, fp32 accumulation into the fp32 residual stream,
// tensor cores); what is ours is the schedule around it (api.cu,
// wgkv_output_proj): the rows are cut into chunks, the all-gather + assembly of
// chunk c+1 runs on the context's comm stream while chunk c's GEMM runs on the
// compute stream, through a two-slot concat ring ordered by events -- so the
// NVLink exchange hides under the projection instead of preceding it.
//
// cuBLAS is resolved at run time (dlopen "libcublas.so.12", reusing the copy
// torch already loaded if any) like NCCL in comm.cu.
#include <dlfcn.h>

#include <mutex>
#include <string>

#include "outproj.cuh"

namespace wgkv {

namespace {

// the few cuBLAS v2 entry points used (cublas_api.h signatures; enums as int)
struct CublasApi {
    int (*create)(void**) = nullptr;
    int (*destroy)(void*) = nullptr;
    int (*set_stream)(void*, cudaStream_t) = nullptr;
    int (*gemm_ex)(void*, int, int, int, int, int, const void*, const void*, int, int, const void*, int, int,
                   const void*, void*, int, int, int, int) = nullptr;
    bool ok = false;
    std::string why;
};

const CublasApi& cublas() {
    static CublasApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libcublas.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("dlopen libcublas.so.12 failed: ") + dlerror();
            return;
        }
        api.create = reinterpret_cast<decltype(api.create)>(dlsym(h, "cublasCreate_v2"));
        api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "cublasDestroy_v2"));
        api.set_stream = reinterpret_cast<decltype(api.set_stream)>(dlsym(h, "cublasSetStream_v2"));
        api.gemm_ex = reinterpret_cast<decltype(api.gemm_ex)>(dlsym(h, "cublasGemmEx"));
        api.ok = api.create && api.destroy && api.set_stream && api.gemm_ex;
        if (!api.ok) api.why = "libcublas.so.12 lacks the expected symbols";
    });
    return api;
}

// cublas_api.h / library_types.h values
constexpr int CUBLAS_OP_N = 0, CUBLAS_OP_T = 1;
constexpr int CUDA_R_32F = 0, CUDA_R_16BF = 14;
constexpr int CUBLAS_COMPUTE_32F = 68;
constexpr int CUBLAS_GEMM_DEFAULT = -1;

}  // namespace

int blas_handle(void** handle, std::string* err) {
    if (*handle) return WGKV_OK;
    const CublasApi& a = cublas();
    if (!a.ok) {
        *err = a.why;
        return WGKV_ENOTSUP;
    }
    if (a.create(handle) != 0) {
        *err = "cublasCreate failed";
        return WGKV_ERUNTIME;
    }
    return WGKV_OK;
}

void blas_destroy(void* handle) {
    if (handle && cublas().ok) cublas().destroy(handle);
}

// x[rows][dim] (fp32, row-major) += a[rows][k] (bf16) . w[dim][k]^T (bf16):
// column-major, X^T (dim x rows) += W^T-as-stored (k x dim)^T . A^T (k x rows)
int gemm_rows_wt(void* handle, cudaStream_t st, long rows, int dim, int k, const void* a, const void* w, float* x,
                 std::string* err) {
    const CublasApi& api = cublas();
    if (api.set_stream(handle, st) != 0) {
        *err = "cublasSetStream failed";
        return WGKV_ERUNTIME;
    }
    const float one = 1.f;
    const int r = api.gemm_ex(handle, CUBLAS_OP_T, CUBLAS_OP_N, dim, (int)rows, k, &one, w, CUDA_R_16BF, k, a,
                              CUDA_R_16BF, k, &one, x, CUDA_R_32F, dim, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (r != 0) {
        *err = "cublasGemmEx failed (status " + std::to_string(r) + ")";
        return WGKV_ERUNTIME;
    }
    return WGKV_OK;
}

}  // namespace wgkv
