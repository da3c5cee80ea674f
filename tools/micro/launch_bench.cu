// Back-to-back launch cost of (nearly) empty kernels with various grid / smem sizes.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int *p) { if (p && threadIdx.x == 9999) p[0] = 1; }
__global__ void k_smem(int *p) {
    extern __shared__ int s[];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (p && s[(threadIdx.x + 1) % blockDim.x] == 9999) p[0] = 1;
}
int main() {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    struct Cfg { int grid, threads, smem; } cfgs[] = {{1, 32, 0}, {148, 256, 0}, {296, 256, 0}, {296, 256, 33000}, {592, 256, 1024}, {8160, 256, 12288}};
    for (auto c : cfgs) {
        for (int rep = 0; rep < 2; rep++) {
            const int N = 200;
            cudaEventRecord(a);
            for (int i = 0; i < N; i++) {
                if (c.smem) k_smem<<<c.grid, c.threads, c.smem>>>(nullptr);
                else k_empty<<<c.grid, c.threads>>>(nullptr);
            }
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("grid %5d x %3d smem %6d: %.2f us per launch\n", c.grid, c.threads, c.smem, ms * 1e3 / N);
        }
    }
    // graph of 20 dependent launches
    cudaStream_t s; cudaStreamCreate(&s);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 20; i++) k_smem<<<296, 256, 33000, s>>>(nullptr);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(a, s);
        for (int i = 0; i < 10; i++) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep == 2) printf("graph: %.2f us per kernel node\n", ms * 1e3 / 200);
    }
    return 0;
}
