// FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ffma2_bench ffma2_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float *out, int iters, float s) {
    float a[8];
    unsigned long long p[4];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
    for (int i = 0; i < 4; i++) p[i] = ((unsigned long long)__float_as_uint(a[2 * i + 1]) << 32) | __float_as_uint(a[2 * i]);
    const unsigned long long ss = ((unsigned long long)__float_as_uint(s) << 32) | __float_as_uint(s);
    const unsigned long long tt = ((unsigned long long)__float_as_uint(0.5f) << 32) | __float_as_uint(0.5f);
    for (int it = 0; it < iters; it++) {
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 8; i++) a[i] = __fmaf_rn(a[i], s, 0.5f);
        } else if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 4; i++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(ss), "l"(tt));
        } else {
            // mixed: 4 FFMA + 2 FFMA2 (same 8 flops)
#pragma unroll
            for (int i = 0; i < 4; i++) a[i] = __fmaf_rn(a[i], s, 0.5f);
#pragma unroll
            for (int i = 0; i < 2; i++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(ss), "l"(tt));
        }
    }
    float r = 0.f;
#pragma unroll
    for (int i = 0; i < 8; i++) r += a[i];
#pragma unroll
    for (int i = 0; i < 4; i++) r += __uint_as_float((unsigned)p[i]) + __uint_as_float((unsigned)(p[i] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    float *o;
    cudaMalloc(&o, 148 * 8 * 256 * sizeof(float));
    const int iters = 1 << 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; mode++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<148 * 8, 256>>>(o, iters, 0.999f);
            else if (mode == 1) k<1><<<148 * 8, 256>>>(o, iters, 0.999f);
            else k<2><<<148 * 8, 256>>>(o, iters, 0.999f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * 8 * iters * 148.0 * 8 * 256;
            const double insts = (mode == 0 ? 8.0 : mode == 1 ? 4.0 : 6.0) * iters * 148.0 * 8 * 256 / 32;
            if (rep) printf("mode %d (%s): %.3f ms  %.1f TFLOP/s fp32  %.3f Twarp-inst/s\n", mode,
                            mode == 0 ? "FFMA" : mode == 1 ? "FFMA2" : "mixed", ms, flops / ms / 1e9, insts / ms / 1e9);
        }
    }
    return 0;
}
