// mgs_cta_probe.cu -- per-step latency of a single-CTA iterated-MGS step for small vectors
// (nvec <= 2048 16-byte vectors, nvec % 8 == 0), the candidate design for IMGS on configs
// 0/1/4: 256 threads, thread t owns the 8 consecutive CAC lanes 8t..8t+7 (L_I = 2048
// unchanged), so tree levels 1-3 are in registers, 4-8 a warp butterfly, 9-11 over the 8 warp
// partials from shared memory (one named barrier).  The basis vectors w o q_i and q_i come in
// through a 3D tensor-map TMA with the 128-byte swizzle (a row = the 8 vectors of one thread,
// 16-byte chunks XOR-permuted by the row index) so that the per-thread reads of 8 consecutive
// vectors are bank-conflict free; a producer warp keeps STG stages in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I paper_1805_06124_b200/csrc \
//        -o scripts/mgs_cta_probe scripts/mgs_cta_probe.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace rbg;

constexpr int T = 256;  // consumer threads
constexpr int STG = 3;  // stages of (w o q, q): 2 x 32 KB each

__device__ __forceinline__ void tma_3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// 16-byte chunk j of row r of a 128B-swizzled tile
__device__ __forceinline__ const double2 *swz(const unsigned char *tile, int r, int j) {
    return reinterpret_cast<const double2 *>(tile + r * 128 + ((j ^ (r & 7)) << 4));
}

// VAR bit 0: skip the stage waits (reuse stage 0); bit 1: no warp butterfly; bit 2: no named
// barrier / cross-warp tree; bit 3: butterfly on 32-bit halves packed (same shuffle count)
template <int VAR>
__global__ void __launch_bounds__(T + 32, 1)
    mgs_cta(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmQ, int nvec, int k, int steps,
            double2 *vout, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ double2 wp[2][8];
    __shared__ __align__(8) uint64_t full[STG], empty[STG];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int rows = nvec / 8;
    const uint32_t tile_bytes = (uint32_t)rows * 128;
    auto wtile = [&](int s) { return smem + (size_t)(s % STG) * 2 * 32768; };
    auto qtile = [&](int s) { return smem + (size_t)(s % STG) * 2 * 32768 + 32768; };
    if (tid == T) {
        for (int i = 0; i < STG; i++) {
            mbar_init_nofence(&full[i], 1);
            mbar_init_nofence(&empty[i], T / 32);
        }
        fence_mbarrier_init();
    }
    __syncthreads();
    if (tid >= T) {  // producer warp
        if (tid == T && (VAR & 1)) {
            mbar_arrive_expect_tx(&full[0], 2 * tile_bytes);
            tma_3d(wtile(0), &tmW, 0, 0, 0, &full[0]);
            tma_3d(qtile(0), &tmQ, 0, 0, 0, &full[0]);
        } else if (tid == T) {
            for (int s = 0; s < steps; s++) {
                if (s >= STG) mbar_wait(&empty[s % STG], (uint32_t)((s / STG - 1) & 1));
                mbar_arrive_expect_tx(&full[s % STG], 2 * tile_bytes);
                const int b = s % k;
                tma_3d(wtile(s), &tmW, 0, 0, b, &full[s % STG]);
                tma_3d(qtile(s), &tmQ, 0, 0, b, &full[s % STG]);
            }
        }
        return;
    }
    double2 v[8];
    for (int j = 0; j < 8; j++) {
        const int u = 8 * tid + j;
        v[j] = u < nvec ? make_double2(1.0 + u * 1e-3, 0.5 - u * 1e-3) : make_double2(0.0, 0.0);
    }
    const bool act = tid < rows;
    int par = 0;
    const long long t0 = clock64();
    if (VAR & 1) mbar_wait(&full[0], 0u);
    for (int s = 0; s < steps; s++) {
        if (!(VAR & 1)) mbar_wait(&full[s % STG], (uint32_t)((s / STG) & 1));
        const unsigned char *wt = wtile((VAR & 1) ? 0 : s), *qt = qtile((VAR & 1) ? 0 : s);
        double pr[8], pi[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const double2 e = act ? *swz(wt, tid, j) : make_double2(0.0, 0.0);
            pr[j] = fma(e.x, v[j].x, 0.0);
            pr[j] = fma(e.y, v[j].y, pr[j]);
            pi[j] = fma(e.x, v[j].y, 0.0);
            pi[j] = fma(-e.y, v[j].x, pi[j]);
        }
#pragma unroll
        for (int h = 1; h < 8; h <<= 1)
#pragma unroll
            for (int j = 0; j < 8; j += 2 * h) {
                pr[j] = pr[j] + pr[j + h];
                pi[j] = pi[j] + pi[j + h];
            }
        double re = pr[0], im = pi[0];
        double2 qr[8];
#pragma unroll
        for (int j = 0; j < 8; j++) qr[j] = act ? *swz(qt, tid, j) : make_double2(0.0, 0.0);
        if (!(VAR & 2)) {
#pragma unroll
            for (int h = 1; h < 32; h <<= 1) {
                re = re + __shfl_xor_sync(0xffffffffu, re, h);
                im = im + __shfl_xor_sync(0xffffffffu, im, h);
            }
        }
        double2 c8[8];
        if (!(VAR & 4)) {
            if (lane == 0) wp[par][warp] = make_double2(re, im);
            asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");
#pragma unroll
            for (int w = 0; w < 8; w++) c8[w] = wp[par][w];
        } else {
#pragma unroll
            for (int w = 0; w < 8; w++) c8[w] = make_double2(re, im);
        }
#pragma unroll
        for (int h = 1; h < 8; h <<= 1)
#pragma unroll
            for (int w = 0; w < 8; w += 2 * h) c8[w] = make_double2(c8[w].x + c8[w + h].x, c8[w].y + c8[w + h].y);
        const double2 c = make_double2(c8[0].x * 1e-6, c8[0].y * 1e-6);
        par ^= 1;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            double vr = v[j].x, vi = v[j].y;
            vr = fma(-c.x, qr[j].x, vr);
            vr = fma(c.y, qr[j].y, vr);
            vi = fma(-c.x, qr[j].y, vi);
            vi = fma(-c.y, qr[j].x, vi);
            v[j] = make_double2(vr, vi);
        }
        __syncwarp();
        if (!(VAR & 1) && lane == 31) mbar_arrive(&empty[s % STG]);
    }
    const long long t1 = clock64();
    for (int j = 0; j < 8; j++)
        if (8 * tid + j < nvec) vout[8 * tid + j] = v[j];
    if (tid == 0) *cyc = t1 - t0;
}

int main(int argc, char **argv) {
    const int nvec = argc > 1 ? atoi(argv[1]) : 2000;
    const int k = argc > 2 ? atoi(argv[2]) : 80;
    const int steps = 4800;
    std::vector<double2> h((size_t)k * nvec);
    for (size_t i = 0; i < h.size(); i++) h[i] = make_double2(1e-3 * (i % 97), -1e-3 * (i % 89));
    double2 *WQ, *Q, *vo;
    long long *cyc;
    cudaMalloc(&WQ, h.size() * 16);
    cudaMalloc(&Q, h.size() * 16);
    cudaMalloc(&vo, nvec * 16);
    cudaMalloc(&cyc, 8);
    cudaMemcpy(WQ, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(Q, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
    CUtensorMap tm[2];
    double2 *base[2] = {WQ, Q};
    for (int i = 0; i < 2; i++) {
        // (16 doubles = one thread's 8 vectors) x (nvec/8 rows) x (k basis vectors)
        const cuuint64_t dims[3] = {16, (cuuint64_t)(nvec / 8), (cuuint64_t)k};
        const cuuint64_t strides[2] = {128, (cuuint64_t)nvec * 16};
        const cuuint32_t box[3] = {16, (cuuint32_t)(nvec / 8), 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = cuTensorMapEncodeTiled(&tm[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base[i], dims, strides, box, estr,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", (int)r);
            return 1;
        }
    }
    const size_t smem = (size_t)STG * 2 * 32768;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto kern, const char *name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<1, T + 32, smem>>>(tm[0], tm[1], nvec, k, steps, vo, cyc);
        cudaEventRecord(e0);
        kern<<<1, T + 32, smem>>>(tm[0], tm[1], nvec, k, steps, vo, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-44s nvec %5d k %4d: %7.1f ns/step %6.0f cycles/step (%s)\n", name, nvec, k, ms * 1e6 / steps,
               (double)c / steps, cudaGetErrorString(cudaGetLastError()));
    };
    run(mgs_cta<0>, "full step (TMA stages)");
    run(mgs_cta<1>, "no stage waits");
    run(mgs_cta<3>, "no stage waits, no butterfly");
    run(mgs_cta<5>, "no stage waits, no CTA tree");
    run(mgs_cta<7>, "no stage waits/butterfly/CTA tree");
    return 0;
}
