// Per-CTA %globaltimer timeline of the decode kernels (diagnostics only:
// compiled in with -DWGKV_TIMELINE into an experiment build, see
// tools/timeline_build.sh and profiles/decode_timeline.py; the product
// library is built without it and these macros expand to nothing).
#pragma once
#ifdef WGKV_TIMELINE
#include <cuda_runtime.h>
namespace wgkv {
struct TlRec {
    unsigned long long t[8];  // entry, phases 1..6, exit (ns, 0 = not reached)
    int tag, layer, cta, sm, n, pad;
};
constexpr unsigned kTlCap = 1u << 17;
static __device__ TlRec g_tl[kTlCap];
static __device__ unsigned g_tl_n;
__device__ __forceinline__ unsigned long long tl_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void tl_commit(const unsigned long long (&t)[8], int tag, int layer, int n) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    const unsigned i = atomicAdd(&g_tl_n, 1u);
    if (i < kTlCap) {
        TlRec r;
        for (int k = 0; k < 8; ++k) r.t[k] = t[k];
        r.tag = tag;
        r.layer = layer;
        r.cta = (int)blockIdx.x;
        r.sm = (int)sm;
        r.n = n;
        r.pad = 0;
        g_tl[i] = r;
    }
}
}  // namespace wgkv
#define TL_DECL unsigned long long tl_t[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
#define TL_MARK(i)                                  \
    do {                                            \
        if (threadIdx.x == 0) tl_t[i] = wgkv::tl_now(); \
    } while (0)
#define TL_COMMIT(tag, layer, n)                              \
    do {                                                      \
        if (threadIdx.x == 0) {                               \
            tl_t[7] = wgkv::tl_now();                         \
            wgkv::tl_commit(tl_t, (tag), (layer), (n));       \
        }                                                     \
    } while (0)
// pass the record to a device function: f(... TL_ARG) / f(... TL_PARAM)
#define TL_PARAM , unsigned long long* tl_t
#define TL_ARG , tl_t
// host reader: copies up to max records into out, returns the count and resets
#define TL_EXPORT(fn)                                                                \
    extern "C" int fn(void* out, int max) {                                          \
        unsigned n = 0;                                                              \
        cudaMemcpyFromSymbol(&n, wgkv::g_tl_n, sizeof(n));                           \
        n = n < wgkv::kTlCap ? n : wgkv::kTlCap;                                     \
        const unsigned m = n < (unsigned)max ? n : (unsigned)max;                    \
        if (m) cudaMemcpyFromSymbol(out, wgkv::g_tl, m * sizeof(wgkv::TlRec));       \
        const unsigned z = 0;                                                        \
        cudaMemcpyToSymbol(wgkv::g_tl_n, &z, sizeof(z));                             \
        return (int)m;                                                               \
    }
#else
#define TL_DECL
#define TL_MARK(i) \
    do {           \
    } while (0)
#define TL_COMMIT(tag, layer, n) \
    do {                         \
    } while (0)
#define TL_EXPORT(fn)
#define TL_PARAM
#define TL_ARG
#endif
