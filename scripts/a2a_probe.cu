// a2a_probe.cu -- the IMGS cluster reduction (16 CTAs x 128 lanes, csrc/imgs.cu
// ClusterReducerPre) in isolation, with two ways to move the 16 CTA partials to every CTA:
//   A: st.async into every CTA's slots, completion counted on an mbarrier, mbarrier wait (imgs.cu);
//   B: plain remote stores (st.shared::cluster.v2.f64) into slots that hold a NaN sentinel, and
//      every warp polls its CTA's 16 slots (one per lane) until none is the sentinel; the slots
//      of a parity are reset to the sentinel after the next reduction's CTA barrier (all of the
//      CTA's warps have read them by then) and before the CTA's next send.
// Prints ns and cycles per reduction (butterfly + CTA tree + exchange + cross-CTA tree).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1805_06124_b200/csrc -o scripts/a2a_probe scripts/a2a_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace rbg;

constexpr int CTAS = 16, THREADS = 128, WPC = THREADS / 32;

__device__ __forceinline__ void st_cluster_v2(uint32_t addr, double a, double b) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ double2 ld_volatile_v2(const double2 *p) {
    double2 r;
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(smem_u32(p)));
    return r;
}

__device__ __forceinline__ unsigned long long bits(double x) { return (unsigned long long)__double_as_longlong(x); }
constexpr unsigned long long kSentinel = 0x7FF00000DEADBEEFull;  // a signalling NaN: never produced by arithmetic

template <int MODE>
__global__ void __cluster_dims__(CTAS, 1, 1) __launch_bounds__(THREADS, 1) probe(int iters, double *out, long long *cyc) {
    __shared__ double2 slots[2][CTAS];
    __shared__ double2 wp[2][WPC];
    __shared__ __align__(8) uint64_t bars[2];
    const uint32_t rank = cluster_ctarank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const double sent = __longlong_as_double((long long)kSentinel);
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_arrive_expect_tx(&bars[0], CTAS * 16);
        mbar_arrive_expect_tx(&bars[1], CTAS * 16);
    }
    if (tid < 2 * CTAS) slots[tid / CTAS][tid % CTAS] = make_double2(sent, sent);
    cluster_sync_all();
    double re = 1e-3 * (tid + 1) + rank, im = 1e-4 * tid - rank;
    int par = 0;
    uint32_t phase = 0;
    double acc = 0.0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        double pr = re * (1.0 + 1e-9 * it), pi = im;
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) {
            pr = pr + __shfl_xor_sync(0xffffffffu, pr, h);
            pi = pi + __shfl_xor_sync(0xffffffffu, pi, h);
        }
        if (lane == 0) wp[par][warp] = make_double2(pr, pi);
        asm volatile("bar.sync 1, %0;" ::"r"(THREADS) : "memory");
        double2 t[WPC];
#pragma unroll
        for (int w = 0; w < WPC; w++) t[w] = wp[par][w];
#pragma unroll
        for (int h = 1; h < WPC; h <<= 1)
#pragma unroll
            for (int w = 0; w < WPC; w += 2 * h) t[w] = make_double2(t[w].x + t[w + h].x, t[w].y + t[w + h].y);
        double2 c[CTAS];
        if (MODE == 0) {
            if (warp == 0 && lane < CTAS) {
                const uint32_t dst = map_dsmem(smem_u32(&slots[par][rank]), (uint32_t)lane);
                const uint32_t bar = map_dsmem(smem_u32(&bars[par]), (uint32_t)lane);
                st_async_v2(dst, t[0].x, t[0].y, bar);
            }
            mbar_wait(&bars[par], (phase >> par) & 1u);
            phase ^= 1u << par;
            if (warp == WPC - 1 && lane == 31) mbar_arrive_expect_tx(&bars[par], CTAS * 16);
#pragma unroll
            for (int l = 0; l < CTAS; l++) c[l] = slots[par][l];
        } else {
            // slots[par ^ 1] were read by every warp of this CTA in the previous reduction
            // (all of them passed this reduction's barrier): back to the sentinel before anyone
            // can write them again (a writer first needs this CTA's partial sent below)
            if (warp == 0 && lane < CTAS) {
                slots[par ^ 1][lane] = make_double2(sent, sent);
                const uint32_t dst = map_dsmem(smem_u32(&slots[par][rank]), (uint32_t)lane);
                st_cluster_v2(dst, t[0].x, t[0].y);
            }
            // poll: lane l < CTAS watches slot l until it no longer holds the sentinel
            double2 mine = make_double2(sent, sent);
            bool ready = lane >= CTAS;
            while (!__all_sync(0xffffffffu, ready)) {
                if (!ready) {
                    mine = ld_volatile_v2(&slots[par][lane]);
                    ready = bits(mine.x) != kSentinel && bits(mine.y) != kSentinel;
                }
            }
#pragma unroll
            for (int l = 0; l < CTAS; l++) {
                c[l].x = __shfl_sync(0xffffffffu, mine.x, l);
                c[l].y = __shfl_sync(0xffffffffu, mine.y, l);
            }
        }
#pragma unroll
        for (int h = 1; h < CTAS; h <<= 1)
#pragma unroll
            for (int l = 0; l < CTAS; l += 2 * h) c[l] = make_double2(c[l].x + c[l + h].x, c[l].y + c[l + h].y);
        acc += c[0].x;
        par ^= 1;
    }
    const long long t1 = clock64();
    cluster_sync_all();
    out[rank * THREADS + tid] = acc;
    if (rank == 0 && tid == 0) *cyc = t1 - t0;
}

int main() {
    double *o;
    long long *c;
    cudaMalloc(&o, CTAS * THREADS * 8);
    cudaMalloc(&c, 8);
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto kern, const char *name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        kern<<<CTAS, THREADS>>>(iters, o, c);
        cudaEventRecord(e0);
        kern<<<CTAS, THREADS>>>(iters, o, c);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        double r0[4];
        cudaMemcpy(r0, o, sizeof r0, cudaMemcpyDeviceToHost);
        printf("%-52s %7.1f ns/reduction %6.0f cycles (%s) acc %.6e\n", name, ms * 1e6 / iters, (double)h / iters,
               cudaGetErrorString(cudaGetLastError()), r0[0]);
    };
    run(probe<0>, "A st.async + mbarrier (imgs.cu)");
    run(probe<1>, "B remote stores + sentinel polling");
    return 0;
}
