// hbm_probe2.cu -- can another read path beat the sweep's LDG ring on this B200?
//  (a) the column stream of hbm_probe.cu with the .L2::256B prefetch qualifier;
//  (b) TMA bulk streaming (cp.async.bulk global->shared, mbarrier ring, producer thread,
//      4 consumer warps summing the staged bytes) at several chunk sizes / depths.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hbm_probe2 scripts/hbm_probe2.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ double2 ldnc(const double2 *p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ldnc256(const double2 *p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

template <int T, int U, bool P256>
__global__ void __launch_bounds__(T) col_stream(const double2 *S, long long nvec, long long M, double *out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = T / 32;
    double acc = 0.0;
    const long long c0 = (long long)blockIdx.x * M / gridDim.x, c1 = (long long)(blockIdx.x + 1) * M / gridDim.x;
    for (long long c = c0 + warp; c < c1; c += nw) {
        const double2 *col = S + c * nvec;
        double2 xa[U];
#pragma unroll
        for (int t = 0; t < U; t++) {
            long long u = t * 32 + lane;
            xa[t] = u < nvec ? (P256 ? ldnc256(col + u) : ldnc(col + u)) : make_double2(0, 0);
        }
        for (long long b = 0; b < nvec; b += 32 * U) {
            double2 xb[U];
#pragma unroll
            for (int t = 0; t < U; t++) {
                long long u = b + 32 * U + t * 32 + lane;
                xb[t] = u < nvec ? (P256 ? ldnc256(col + u) : ldnc(col + u)) : make_double2(0, 0);
            }
#pragma unroll
            for (int t = 0; t < U; t++) { acc = fma(xa[t].x, xa[t].y, acc); xa[t] = xb[t]; }
        }
    }
    if (acc == 12345.678) out[0] = acc;
}

// the same column stream with dynamic column assignment (grid-wide atomic counter, a column
// taken one ahead), as the sweep's k_sweep_dyn
template <int T, int U>
__global__ void __launch_bounds__(T) col_stream_dyn(const double2 *S, long long nvec, long long M, double *out,
                                                    unsigned long long *ctr) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long nwg = (long long)gridDim.x * (T / 32);
    double acc = 0.0;
    long long c = (long long)blockIdx.x * (T / 32) + warp;
    unsigned long long raw = 0;
    if (lane == 0) raw = atomicAdd(ctr, 1ull);
    while (c < M) {
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
        c = (long long)__shfl_sync(0xffffffffu, raw, 0) + nwg;
        if (lane == 0) raw = atomicAdd(ctr, 1ull);
    }
    if (acc == 12345.678) out[0] = acc;
}

// the same dynamic column stream with a bulk L2 prefetch PF batches (of 32*U vectors) ahead of
// the register ring, issued by lane 0: DRAM -> L2 traffic in flight not bounded by registers
template <int T, int U, int PF>
__global__ void __launch_bounds__(T) col_stream_dyn_pf(const double2 *S, long long nvec, long long M, double *out,
                                                       unsigned long long *ctr) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long nwg = (long long)gridDim.x * (T / 32);
    const long long batch = 32 * U;
    double acc = 0.0;
    long long c = (long long)blockIdx.x * (T / 32) + warp;
    unsigned long long raw = 0;
    if (lane == 0) raw = atomicAdd(ctr, 1ull);
    while (c < M) {
        const double2 *col = S + c * nvec;
        if (lane == 0)
            for (int p = 0; p < PF; p++) {
                const long long u0 = p * batch;
                if (u0 < nvec) {
                    const long long n = (nvec - u0 < batch ? nvec - u0 : batch) * 16;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(col + u0), "r"((unsigned)n) : "memory");
                }
            }
        double2 xa[U];
#pragma unroll
        for (int t = 0; t < U; t++) { long long u = t * 32 + lane; xa[t] = u < nvec ? ldnc(col + u) : make_double2(0, 0); }
        for (long long b = 0; b < nvec; b += batch) {
            if (lane == 0) {
                const long long u0 = b + (long long)PF * batch;
                if (u0 < nvec) {
                    const long long n = (nvec - u0 < batch ? nvec - u0 : batch) * 16;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(col + u0), "r"((unsigned)n) : "memory");
                }
            }
            double2 xb[U];
#pragma unroll
            for (int t = 0; t < U; t++) { long long u = b + batch + t * 32 + lane; xb[t] = u < nvec ? ldnc(col + u) : make_double2(0, 0); }
#pragma unroll
            for (int t = 0; t < U; t++) { acc = fma(xa[t].x, xa[t].y, acc); xa[t] = xb[t]; }
        }
        c = (long long)__shfl_sync(0xffffffffu, raw, 0) + nwg;
        if (lane == 0) raw = atomicAdd(ctr, 1ull);
    }
    if (acc == 12345.678) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t par) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(b)),
                 "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

template <int CHUNK, int STAGES>
__global__ void __launch_bounds__(160) tma_stream(const unsigned char *S, long long per_cta, double *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned char *base = S + blockIdx.x * per_cta;
    const long long nch = per_cta / CHUNK;
    if (tid == 0) {
        for (int i = 0; i < STAGES; i++) { mb_init(&full[i], 1); mb_init(&empty[i], 4); }
    }
    __syncthreads();
    double acc = 0.0;
    if (warp == 4) {
        if (lane == 0)
            for (long long c = 0; c < nch; c++) {
                const int s = (int)(c % STAGES);
                if (c >= STAGES) mb_wait(&empty[s], (uint32_t)(((c / STAGES) - 1) & 1));
                mb_expect(&full[s], CHUNK);
                bulk(sm + (size_t)s * CHUNK, base + c * CHUNK, CHUNK, &full[s]);
            }
    } else {
        for (long long c = 0; c < nch; c++) {
            const int s = (int)(c % STAGES);
            mb_wait(&full[s], (uint32_t)((c / STAGES) & 1));
            const double2 *p = reinterpret_cast<const double2 *>(sm + (size_t)s * CHUNK);
#pragma unroll 4
            for (int i = tid; i < CHUNK / 16; i += 128) { double2 x = p[i]; acc = fma(x.x, x.y, acc); }
            __syncwarp();
            if (lane == 0) mb_arrive(&empty[s]);
        }
    }
    if (acc == 12345.678) out[0] = acc;
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
    CK(cudaGetLastError());
    return best;
}

int main() {
    const long long nvec = 10000, M = 409600 / 4;   // 16.4 GB of "columns"
    const long long n = nvec * M;
    double2 *S; double *out;
    CK(cudaMalloc(&S, n * 16)); CK(cudaMalloc(&out, 8));
    CK(cudaMemset(S, 1, n * 16));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double bytes = (double)n * 16;
    auto rep = [&](const char *name, float ms, double b) { printf("%-46s %8.3f ms  %8.1f GB/s\n", name, ms, b / ms / 1e6); };
#define COL(T, U, OCC, P) rep("col_stream T=" #T " U=" #U " ctas/SM=" #OCC " L2::256B=" #P, \
        timeit([&] { col_stream<T, U, P><<<sms * OCC, T>>>(S, nvec, M, out); }), bytes);
    COL(512, 12, 1, false) COL(512, 12, 1, true) COL(512, 8, 1, true) COL(256, 16, 4, false) COL(256, 16, 4, true)
    unsigned long long *ctr;
    CK(cudaMalloc(&ctr, 8));
#define DYN(T, U, OCC) rep("col_stream_dyn T=" #T " U=" #U " ctas/SM=" #OCC, \
        timeit([&] { cudaMemsetAsync(ctr, 0, 8); col_stream_dyn<T, U><<<sms * OCC, T>>>(S, nvec, M, out, ctr); }), bytes);
    DYN(512, 12, 1) DYN(512, 16, 1) DYN(256, 16, 4) DYN(1024, 8, 1)
#define DYNPF(T, U, PF, OCC) rep("col_stream_dyn_pf T=" #T " U=" #U " PF=" #PF " ctas/SM=" #OCC, \
        timeit([&] { cudaMemsetAsync(ctr, 0, 8); col_stream_dyn_pf<T, U, PF><<<sms * OCC, T>>>(S, nvec, M, out, ctr); }), bytes);
    for (int rep2 = 0; rep2 < 2; rep2++) {
        DYNPF(512, 16, 2, 1) DYNPF(512, 16, 3, 1) DYNPF(512, 12, 3, 1) DYNPF(512, 12, 4, 1) DYNPF(512, 8, 4, 1)
        DYNPF(512, 8, 6, 1) DYNPF(256, 16, 3, 4)
        DYN(512, 16, 1) DYN(256, 16, 4)
    }
#define TMA(CH, ST, OCC) { \
        auto k = tma_stream<CH, ST>; const int smem = CH * ST; \
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
        const long long ctas = (long long)sms * OCC; const long long per = (long long)(bytes / ctas) / CH * CH; \
        rep("tma_stream chunk=" #CH " stages=" #ST " ctas/SM=" #OCC, \
            timeit([&] { k<<<ctas, 160, smem>>>((const unsigned char *)S, per, out); }), (double)per * ctas); }
    TMA(16384, 12, 1) TMA(32768, 6, 1) TMA(49152, 4, 1) TMA(65536, 3, 1) TMA(16384, 6, 2) TMA(32768, 3, 2)
    TMA(8192, 12, 2) TMA(24576, 4, 2)
    // what is left next to a 160 KB staged basis vector (1 CTA/SM): <= 64 KB of stages
    TMA(16384, 4, 1) TMA(8192, 8, 1) TMA(32768, 2, 1) TMA(12288, 5, 1)
    return 0;
}
