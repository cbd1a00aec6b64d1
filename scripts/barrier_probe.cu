// time the counter/generation grid barrier of recon.cu on a cooperative grid
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void grid_barrier(unsigned *count, unsigned *gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *vg = gen;
        const unsigned g = *vg;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0u;
            __threadfence();
            atomicExch(gen, g + 1u);
        } else {
            while (*vg == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}
__global__ void k(unsigned *bar, int n, unsigned long long *t) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; i++) grid_barrier(bar, bar + 1, gridDim.x);
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *t = t1 - t0;
}
int main() {
    unsigned *bar; unsigned long long *t, h;
    cudaMalloc(&bar, 8); cudaMalloc(&t, 8);
    for (int grid : {16, 64, 148, 296}) {
        cudaMemset(bar, 0, 8);
        int n = 1000;
        void *args[] = {&bar, &n, &t};
        cudaLaunchCooperativeKernel((void *)k, grid, 256, args, 0, 0);
        cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
        printf("grid %d: %.2f us per barrier (%s)\n", grid, h * 1e-3 / n, cudaGetErrorString(cudaGetLastError()));
    }
}
