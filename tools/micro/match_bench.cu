// Throughput of warp match/vote/shfl/atoms on this GPU: 148 x NB blocks x 256 threads, ITER rounds.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(unsigned *out, int iters) {
    unsigned v = threadIdx.x * 2654435761u + blockIdx.x, acc = 0;
    __shared__ unsigned sm[256 * 8];
    for (int i = 0; i < 256 * 8; i += blockDim.x) sm[i + threadIdx.x] = 0;
    __syncthreads();
    for (int i = 0; i < iters; i++) {
        v = v * 1664525u + 1013904223u;
        const unsigned d = (v >> 24) & 255;
        if (OP == 0) acc += __match_any_sync(0xffffffffu, d);
        if (OP == 1) acc += __ballot_sync(0xffffffffu, d & 1);
        if (OP == 2) acc += __shfl_sync(0xffffffffu, d, (threadIdx.x + i) & 31);
        if (OP == 3) acc += atomicAdd(&sm[(threadIdx.x >> 5) * 256 + d], 1u);
        if (OP == 4) {  // 8 ballots = one 8-bit multisplit
            unsigned p = 0xffffffffu;
#pragma unroll
            for (int b = 0; b < 8; b++) { unsigned bb = __ballot_sync(0xffffffffu, (d >> b) & 1); p &= ((d >> b) & 1) ? bb : ~bb; }
            acc += p;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    unsigned *o; cudaMalloc(&o, 148 * 8 * 256 * 4);
    const char *names[] = {"match_any", "ballot", "shfl", "atoms", "8xballot"};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int nb : {2, 8}) {
        for (int op = 0; op < 5; op++) {
            const int iters = 4096;
            for (int rep = 0; rep < 2; rep++) {
                cudaEventRecord(a);
                switch (op) {
                    case 0: k<0><<<148 * nb, 256>>>(o, iters); break;
                    case 1: k<1><<<148 * nb, 256>>>(o, iters); break;
                    case 2: k<2><<<148 * nb, 256>>>(o, iters); break;
                    case 3: k<3><<<148 * nb, 256>>>(o, iters); break;
                    case 4: k<4><<<148 * nb, 256>>>(o, iters); break;
                }
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep) {
                    double per = ms * 1e-3 * 1.965e9 / ((double)iters * nb * 8 / 4);  // cycles per op per SMSP (nb*8 warps / 4 SMSPs)
                    printf("%-10s blocks/SM=%d  %.3f ms  ~%.2f SMSP-cycles per warp-op\n", names[op], nb, ms, per);
                }
            }
        }
    }
    return 0;
}
