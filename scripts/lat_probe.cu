// lat_probe.cu -- dependent-chain latencies on B200 (cycles per op): DFMA, DADD, FFMA,
// double shuffle (two SHFL), LDS.64, and a named barrier of 256 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/lat_probe scripts/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double *out, long long *cyc, int n) {
    __shared__ double sm[64];
    const int tid = threadIdx.x;
    double a = 1.0 + tid * 1e-9, b = 0.999999, c = 1e-7;
    float fa = 1.0f + tid, fb = 0.9999f, fc = 1e-5f;
    sm[tid & 63] = a;
    __syncthreads();
    long long t[8];
    t[0] = clock64();
    for (int i = 0; i < n; i++) a = fma(a, b, c);
    t[1] = clock64();
    for (int i = 0; i < n; i++) a = a + c;
    t[2] = clock64();
    for (int i = 0; i < n; i++) fa = fmaf(fa, fb, fc);
    t[3] = clock64();
    for (int i = 0; i < n; i++) a = __shfl_xor_sync(0xffffffffu, a, 1) * b;
    t[4] = clock64();
    int idx = tid & 63;
    for (int i = 0; i < n; i++) {
        double x = sm[idx];
        idx = ((int)x) & 63;
    }
    t[5] = clock64();
    for (int i = 0; i < n; i++) asm volatile("bar.sync 1, 256;" ::: "memory");
    t[6] = clock64();
    if (tid == 0)
        for (int p = 0; p < 6; p++) cyc[p] = t[p + 1] - t[p];
    out[tid] = a + fa + idx;
}

int main() {
    double *o;
    long long *c, h[6];
    cudaMalloc(&o, 256 * 8);
    cudaMalloc(&c, 6 * 8);
    const int n = 4096;
    lat<<<1, 256>>>(o, c, n);
    lat<<<1, 256>>>(o, c, n);
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    const char *names[6] = {"DFMA", "DADD", "FFMA", "double shfl + DMUL", "LDS.64 (dependent)", "bar.sync 256"};
    for (int p = 0; p < 6; p++) printf("%-22s %6.1f cycles/op\n", names[p], (double)h[p] / n);
    return 0;
}
