// reduce_probe.cu -- latency of the IMGS cluster reduction building blocks on B200
// (8-CTA cluster x 256 threads, as in csrc/imgs.cu).  Prints ns per reduction for:
//   A: warp butterfly only (5 levels, 2 doubles)
//   B: A + st.async all-to-all of 64 warp partials + mbarrier wait + 64-leaf tree
//   C: A + smem tree over 8 warps + DSMEM stores + barrier.cluster (the r01 design)
//   D: B + 5-vector dot/axpy fma chain (one full MGS step without loads)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1805_06124_b200/csrc -o /tmp/rp scripts/reduce_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace rbg;

template <int MODE>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(256, 1) probe(int iters, double *out, long long *cyc) {
    __shared__ double2 slots[2][64];
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ double2 s_warp[2][8], s_cta[2][8];
    const uint32_t rank = cluster_ctarank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_arrive_expect_tx(&bars[0], 1024);
        mbar_arrive_expect_tx(&bars[1], 1024);
    }
    cluster_sync_all();
    double re = tid * 1e-3, im = rank * 1e-2;
    double2 v[5];
    for (int m = 0; m < 5; m++) v[m] = make_double2(re + m, im - m);
    int par = 0;
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        double pr = re, pi = im;
        if (MODE == 3) {
            pr = 0; pi = 0;
#pragma unroll
            for (int m = 0; m < 5; m++) {
                pr = fma(v[m].x, v[m].x, pr); pr = fma(v[m].y, v[m].y, pr);
                pi = fma(v[m].x, v[m].y, pi); pi = fma(-v[m].y, v[m].x, pi);
            }
        }
        for (int h = 1; h < 32; h <<= 1) {
            pr = pr + __shfl_xor_sync(0xffffffffu, pr, h);
            pi = pi + __shfl_xor_sync(0xffffffffu, pi, h);
        }
        if (MODE == 1 || MODE == 3) {
            if (lane < 8) {
                uint32_t dst = map_dsmem(smem_u32(&slots[par][rank * 8 + warp]), lane);
                uint32_t bar = map_dsmem(smem_u32(&bars[par]), lane);
                st_async_v2(dst, pr, pi, bar);
            }
            mbar_wait(&bars[par], (phase >> par) & 1u);
            phase ^= 1u << par;
            if (tid == 0) mbar_arrive_expect_tx(&bars[par], 1024);
            double2 a = slots[par][2 * lane], b = slots[par][2 * lane + 1];
            pr = a.x + b.x; pi = a.y + b.y;
            for (int h = 1; h < 32; h <<= 1) {
                pr = pr + __shfl_xor_sync(0xffffffffu, pr, h);
                pi = pi + __shfl_xor_sync(0xffffffffu, pi, h);
            }
        } else if (MODE == 2) {
            if (lane == 0) s_warp[par][warp] = make_double2(pr, pi);
            __syncthreads();
            if (tid < 8) {
                double x = 0, y = 0;
                for (int w = 0; w < 8; w++) { x += s_warp[par][w].x; y += s_warp[par][w].y; }
                st_dsmem_v2(map_dsmem(smem_u32(&s_cta[par][rank]), tid), x, y);
            }
            cluster_sync_all();
            pr = 0; pi = 0;
            for (int c = 0; c < 8; c++) { pr += s_cta[par][c].x; pi += s_cta[par][c].y; }
        }
        if (MODE == 3) {
#pragma unroll
            for (int m = 0; m < 5; m++) {
                v[m].x = fma(-pr * 1e-9, v[m].x, v[m].x); v[m].x = fma(pi * 1e-9, v[m].y, v[m].x);
                v[m].y = fma(-pr * 1e-9, v[m].y, v[m].y); v[m].y = fma(-pi * 1e-9, v[m].x, v[m].y);
            }
        }
        re = pr * 1e-6; im = pi * 1e-6;
        par ^= 1;
    }
    long long t1 = clock64();
    if (tid == 0 && rank == 0) { out[0] = re + im + v[0].x; cyc[MODE] = t1 - t0; }
}

int main() {
    double *out; long long *cyc;
    cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * 8);
    const int iters = 20000;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](auto kern, const char *name, int mode) {
        kern<<<8, 256>>>(100, out, cyc);
        cudaEventRecord(a); kern<<<8, 256>>>(iters, out, cyc); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        long long c[8]; cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
        printf("%-58s %8.1f ns/iter  %7.0f cycles/iter  (%s)\n", name, ms * 1e6 / iters, (double)c[mode] / iters,
               cudaGetErrorString(cudaGetLastError()));
    };
    run(probe<0>, "A warp butterfly only", 0);
    run(probe<1>, "B butterfly + st.async all-to-all + mbarrier + 64-leaf tree", 1);
    run(probe<2>, "C butterfly + smem 8-warp tree + DSMEM + barrier.cluster", 2);
    run(probe<3>, "D = B + 5-vector dot and axpy fma chains", 3);
    return 0;
}
