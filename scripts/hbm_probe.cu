// hbm_probe.cu -- measured HBM ceilings on this B200 for the roofline of the fused sweep
// (R26): a read-only stream with the sweep's access pattern (one warp per
// 160 KB "column", 16-byte non-coherent loads) at several occupancies / unroll depths,
// a plain grid-stride read, and a copy (the MEASURED_PEAKS.json reference).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hbm_probe scripts/hbm_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ double2 ldnc(const double2 *p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

// warp per column, lanes strided, U loads in flight per lane (double buffered)
template <int T, int U>
__global__ void __launch_bounds__(T) col_stream(const double2 *S, long long nvec, long long M, double *out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = T / 32;
    double acc = 0.0;
    const long long c0 = (long long)blockIdx.x * M / gridDim.x, c1 = (long long)(blockIdx.x + 1) * M / gridDim.x;
    for (long long c = c0 + warp; c < c1; c += nw) {
        const double2 *col = S + c * nvec;
        double2 xa[U];
#pragma unroll
        for (int t = 0; t < U; t++) { long long u = t * 32 + lane; xa[t] = u < nvec ? ldnc(col + u) : make_double2(0, 0); }
        for (long long b = 0; b < nvec; b += 32 * U) {
            double2 xb[U];
#pragma unroll
            for (int t = 0; t < U; t++) { long long u = b + 32 * U + t * 32 + lane; xb[t] = u < nvec ? ldnc(col + u) : make_double2(0, 0); }
#pragma unroll
            for (int t = 0; t < U; t++) { acc = fma(xa[t].x, xa[t].y, acc); xa[t] = xb[t]; }
        }
    }
    if (acc == 12345.678) out[0] = acc;
}

__global__ void grid_read(const double2 *S, long long n, double *out) {
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double2 x = ldnc(S + i);
        acc = fma(x.x, x.y, acc);
    }
    if (acc == 12345.678) out[0] = acc;
}

__global__ void grid_copy(const double2 *S, double2 *D, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        D[i] = ldnc(S + i);
}

template <typename F>
float timeit(F f, int reps = 5) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; r++) {
        cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    return best;
}

int main() {
    const long long nvec = 10000, M = 102400;   // 16.4 GB of "columns"
    const long long n = nvec * M;
    double2 *S, *D; double *out;
    CK(cudaMalloc(&S, n * 16)); CK(cudaMalloc(&out, 8));
    CK(cudaMemset(S, 0, n * 16));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double bytes = (double)n * 16;
    auto rep = [&](const char *name, float ms) { printf("%-44s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / ms / 1e6); };
#define COL(T, U, OCC) rep("col_stream T=" #T " U=" #U " ctas/SM=" #OCC, timeit([&] { col_stream<T, U><<<sms * OCC, T>>>(S, nvec, M, out); }));
    COL(512, 4, 1) COL(512, 8, 1) COL(512, 12, 1) COL(1024, 4, 1) COL(1024, 8, 1) COL(512, 8, 2) COL(256, 8, 4) COL(256, 16, 4) COL(512, 16, 1)
    rep("grid_read 148x8x256", timeit([&] { grid_read<<<sms * 8, 256>>>(S, n, out); }));
    rep("grid_read 148x4x1024", timeit([&] { grid_read<<<sms * 2, 1024>>>(S, n, out); }));
    const long long nc = n / 2;
    CK(cudaMalloc(&D, nc * 16));
    float ms = timeit([&] { grid_copy<<<sms * 8, 256>>>(S, D, nc); });
    printf("%-44s %8.3f ms  %8.1f GB/s (read+write)\n", "grid_copy 8.2 GB", ms, 2.0 * nc * 16 / ms / 1e6);
    return 0;
}
