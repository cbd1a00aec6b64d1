// Latency probe for the EIM forward-substitution chain (DESIGN.md f-2): clocks per step of
// one warp doing  c = cdiv(v, t) -> shfl -> v = v - c*t  with variants that drop parts.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false chain_probe.cu -o chain_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void chain(double *out, long long *cyc, int n, double seed) {
    const int lane = threadIdx.x;
    double vx = seed + lane, vy = 0.5 * seed - lane, tx = 1.25 + 0.01 * lane, ty = 0.75;
    const double dd = fma(tx, tx, ty * ty);
    long long t0 = clock64();
    for (int b = 0; b < n; b++) {
        double cx, cy;
        if (MODE == 3 || MODE == 4) {      // owner-only division (divergent branch)
            cx = 0.0;
            cy = 0.0;
            if (lane == (b & 31)) {
                cx = fma(vx, tx, vy * ty) / dd;
                cy = fma(vy, tx, -(vx * ty)) / dd;
                if (MODE == 4) out[32 + b] = cx + cy;
            }
        } else if (MODE == 0 || MODE == 2) {      // IEEE division (the oracle's cdiv)
            cx = fma(vx, tx, vy * ty) / dd;
            cy = fma(vy, tx, -(vx * ty)) / dd;
        } else {                           // multiply instead (timing only)
            cx = fma(vx, tx, vy * ty) * dd;
            cy = fma(vy, tx, -(vx * ty)) * dd;
        }
        if (MODE != 2) {
            cx = __shfl_sync(0xffffffffu, cx, b & 31);
            cy = __shfl_sync(0xffffffffu, cy, b & 31);
        }
        vx = fma(-cx, tx, vx);
        vx = fma(cy, ty, vx);
        vy = fma(-cx, ty, vy);
        vy = fma(-cy, tx, vy);
    }
    long long t1 = clock64();
    out[lane] = vx + vy;
    if (lane == 0) *cyc = t1 - t0;
}

int main() {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, (32 + 8192) * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    const int n = 4096;
    const char *names[5] = {"div+shfl", "mul+shfl", "div only", "owner div", "owner div+st"};
    for (int rep = 0; rep < 2; rep++) {
        chain<0><<<1, 32>>>(out, cyc, n, 1e-3);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("%-10s %.1f clk/step\n", names[0], (double)h / n);
        chain<1><<<1, 32>>>(out, cyc, n, 1e-3);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("%-10s %.1f clk/step\n", names[1], (double)h / n);
        chain<2><<<1, 32>>>(out, cyc, n, 1e-3);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("%-10s %.1f clk/step\n", names[2], (double)h / n);
        chain<3><<<1, 32>>>(out, cyc, n, 1e-3);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("%-10s %.1f clk/step\n", names[3], (double)h / n);
        chain<4><<<1, 32>>>(out, cyc, n, 1e-3);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("%-10s %.1f clk/step\n", names[4], (double)h / n);
    }
    return 0;
}
