// Micro-benchmark (diagnostic, not product): issue throughput of MUFU.EX2,
// F2FP bf16x2 packing and FADD2 on one SM, for 1..16 warps.  Prints clocks
// per warp-instruction per SM sub-partition.
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pk(float a, float b) {
    uint32_t r;
    asm volatile("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
    return r;
}

__device__ __forceinline__ uint32_t ex2b(uint32_t x) {
    uint32_t y;
    asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ uint32_t ex2h(uint32_t x) {
    uint32_t y;
    asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

template <int MODE>
__global__ void k(float* out, long long* clk, int iters) {
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = -0.001f * (threadIdx.x + i);
    uint32_t acc = 0;
    uint32_t u[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) u[i] = 0xbc00bc00u + threadIdx.x + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) v[i] = ex2(v[i]);                       // 16 MUFU
            if (MODE == 1 && (i & 1)) acc += pk(v[i], v[i - 1]);   // 8 F2FP (+IADD)
            if (MODE == 1 && !(i & 1)) v[i] = v[i] * 0.999f;
            if (MODE == 2) {                                       // 8 FADD2
                if (i & 1) {
                    float2 r = __fadd2_rn(make_float2(v[i], v[i - 1]), make_float2(1e-7f, 1e-7f));
                    v[i] = r.x; v[i - 1] = r.y;
                }
            }
            if (MODE == 4) u[i] = ex2b(u[i]);  // 16 bf16x2 ex2 (32 results)
            if (MODE == 5) u[i] = ex2h(u[i]);  // 16 f16x2 ex2 (32 results)
            if (MODE == 3) {  // 8 MUFU + 4 F2FP
                if (i & 1) { v[i] = ex2(v[i]); v[i - 1] = ex2(v[i - 1]); acc += pk(v[i], v[i - 1]); }
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 16; ++i) s += v[i] + (float)(u[i] & 1);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
    float* out;
    long long* clk;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&clk, 148 * 8);
    const int iters = 4096;
    const char* names[] = {"ex2 (MUFU)", "F2FP pack", "FADD2", "2 ex2 + 1 F2FP", "ex2 bf16x2", "ex2 f16x2"};
    const int per_iter[] = {16, 8, 8, 12, 16, 16};  // warp-instructions of interest per iteration
    for (int mode = 0; mode < 6; ++mode)
        for (int w = 1; w <= 16; w *= 2) {
            void (*fn)(float*, long long*, int) = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : mode == 4 ? k<4> : k<5>;
            fn<<<148, 32 * w>>>(out, clk, iters);
            fn<<<148, 32 * w>>>(out, clk, iters);
            long long h[148];
            cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
            const double instr_per_smsp = (double)per_iter[mode] * iters * w / (w < 4 ? w : 4);
            printf("%-16s warps/SM %2d: %.2f clk per warp-instr per SMSP (sub-partitions used %d)\n", names[mode], w,
                   h[0] / instr_per_smsp, w < 4 ? w : 4);
        }
    return 0;
}
