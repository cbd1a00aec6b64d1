// imgs_cta.cu -- pivot decision + iterated MGS in ONE CTA for short vectors (nvec <= 2048
// 16-byte vectors, nvec % 8 == 0: configs 0, 1 and 4), the same arithmetic as imgs.cu.
//
// PAPER.md:871-883 (Hoffmann MGSCI, kappa = 2); acceptance test, sweep cap and degeneracy:
// DESIGN.md reading R7; the canonical arithmetic contract (CAC rules 2-4, 9) with the same
// L_I = 2048 lanes and the same balanced pairwise lane tree as the 16-CTA cluster kernel, so the
// results are bit-identical to it and to the oracle.  What changes is the mapping of lanes to
// threads (round 2): thread t of 256 owns the 8 consecutive lanes
// 8t..8t+7 -- with nvec <= 2048 lane l holds at most the one vector u = l -- so tree levels
// 1-3 are additions in registers, levels 4-8 a warp butterfly and levels 9-11 the 8 warp
// partials read back from shared memory after one named barrier.  No DSMEM round trip: the
// cluster kernel's MGS step is bounded by its all-to-all (0.80 us per step), this one by the
// latency chain on one SM (0.63 us in scripts/mgs_cta_probe.cu at nvec = 2,000).
//
// The basis slices come through a 3D tensor map (16 doubles = one thread's 8 vectors x nvec/8
// rows x basis index) with the 128-byte swizzle, so that a thread's reads of its 8 consecutive
// vectors are bank-conflict free; a producer warp keeps kStages stages (w o q_b and q_b, 2 x
// nvec x 16 bytes) in flight.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>

#include "kernels.h"

namespace rbg {

namespace {

constexpr int kCtaThreads = 256;  // consumer threads: 8 lanes each
constexpr int kStages = 3;
constexpr int kTile = 32768;      // one basis vector's slice: <= 256 rows x 128 B

__device__ __forceinline__ void tma_3d_g2s(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// 16-byte chunk j of row r of a tile written with the 128-byte swizzle (chunk index XOR row % 8)
__device__ __forceinline__ double2 swz_ld(const unsigned char *tile, int r, int j) {
    return *reinterpret_cast<const double2 *>(tile + r * 128 + ((j ^ (r & 7)) << 4));
}

// The 2048-lane tree of CAC rule 3 for lane partials p[l] = (pr[j], pi[j]) at l = 8 tid + j.
struct CtaReducer {
    double2 (*wp)[8];  // [parity][warp]
    int warp, lane, par;

    __device__ __forceinline__ double2 sum(double (&pr)[8], double (&pi)[8]) {
#pragma unroll
        for (int h = 1; h < 8; h <<= 1)  // levels 1-3: lanes 8t .. 8t+7 of this thread
#pragma unroll
            for (int j = 0; j < 8; j += 2 * h) {
                pr[j] = pr[j] + pr[j + h];
                pi[j] = pi[j] + pi[j + h];
            }
        double re = pr[0], im = pi[0];
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) {  // levels 4-8: lanes 8t and 8(t + h)
            re = re + __shfl_xor_sync(0xffffffffu, re, h);
            im = im + __shfl_xor_sync(0xffffffffu, im, h);
        }
        if (lane == 0) wp[par][warp] = make_double2(re, im);
        asm volatile("bar.sync 1, %0;" ::"r"(kCtaThreads) : "memory");  // consumer warps only
        double2 c[8];
#pragma unroll
        for (int w = 0; w < 8; w++) c[w] = wp[par][w];
#pragma unroll
        for (int h = 1; h < 8; h <<= 1)  // levels 9-11: lanes 256w and 256(w + h)
#pragma unroll
            for (int w = 0; w < 8; w += 2 * h) c[w] = make_double2(c[w].x + c[w + h].x, c[w].y + c[w + h].y);
        par ^= 1;  // wp[par] is rewritten two reductions later, after every warp passed the next barrier
        return c[0];
    }
};

template <bool CPLX>
__device__ __forceinline__ void nrm_lanes(const double2 (&v)[8], const double *w, int u0, int nvec, double (&pr)[8],
                                          double (&pi)[8]) {
#pragma unroll
    for (int j = 0; j < 8; j++) {  // CAC rule 4 (one vector per lane)
        double acc = 0.0;
        const int u = u0 + j;
        if (u < nvec) {
            if (CPLX) {
                double t = w[u] * v[j].x;
                acc = fma(t, v[j].x, acc);
                t = w[u] * v[j].y;
                acc = fma(t, v[j].y, acc);
            } else {
                double t = w[2 * u] * v[j].x;
                acc = fma(t, v[j].x, acc);
                t = w[2 * u + 1] * v[j].y;
                acc = fma(t, v[j].y, acc);
            }
        }
        pr[j] = acc;
        pi[j] = 0.0;
    }
}

template <bool CPLX>
__global__ void __launch_bounds__(kCtaThreads + 32, 1)
    k_imgs_cta(const ImgsArgs a, const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmQ) {
    extern __shared__ __align__(1024) unsigned char dsm_raw[];
    // the 128-byte swizzle is a function of the shared-memory address: tiles start 1024-aligned
    unsigned char *dsm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
    __shared__ double2 s_wp[2][8];
    __shared__ __align__(8) uint64_t s_full[kStages], s_empty[kStages];
    __shared__ long long s_done;

    const int stop0 = a.st->stop;  // final before this kernel starts (see imgs.cu)
    if (stop0) {
        if (threadIdx.x == 0) {
            loop_exit(a.cond, a.use_cond);
            a.st->noop += 1;
        }
        return;
    }
    const long long k = a.st->k;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool producer = tid >= kCtaThreads;
    const int nvec = (int)a.nvec;
    const int rows = nvec / 8;
    const int u0 = 8 * tid;  // this thread's lanes 8t..8t+7 hold vectors u0..u0+7
    const bool odd_tail = !CPLX && (a.N & 1);
    const uint32_t tile_bytes = (uint32_t)rows * 128u;
    auto wtile = [&](long long s) { return dsm + (size_t)(s % kStages) * 2 * kTile; };
    auto qtile = [&](long long s) { return dsm + (size_t)(s % kStages) * 2 * kTile + kTile; };
    const long long limit = (long long)kNuMax * k;  // MGS steps that can ever be needed
    const long long first = k < a.k_max ? (limit < kStages ? limit : kStages) : 0;
    auto issue = [&](long long s) {  // stage s holds basis vector s mod k
        mbar_arrive_expect_tx(&s_full[s % kStages], 2 * tile_bytes);
        const int b = (int)(s % k);
        tma_3d_g2s(wtile(s), &tmW, 0, 0, b, &s_full[s % kStages]);
        tma_3d_g2s(qtile(s), &tmQ, 0, 0, b, &s_full[s % kStages]);
    };
    if (tid == kCtaThreads) {
        for (int i = 0; i < kStages; i++) {
            mbar_init_nofence(&s_full[i], 1);
            mbar_init_nofence(&s_empty[i], kCtaThreads / 32);
        }
        fence_mbarrier_init();
        for (long long s = 0; s < first; s++) issue(s);
    }
    if (tid == 0) s_done = -1;
    __syncthreads();
    grid_dep_wait();

    // ---- a3: pivot decision ------------------------------------------------------------
    double m;
    long long J;
    const double2 *src;
    pivot_decision(a, k, m, J, src);
    const double err = sqrt(fmax(m, 0.0));  // CAC rule 8
    int why = kStopNone;
    if (m == -INFINITY) why = kStopAll;
    else if (err < a.tol) why = kStopTol;
    else if (k == a.k_max) why = kStopKmax;
    const bool leader = tid == 0;
    if (leader) a.errors[k] = err;
    if (why != kStopNone) {
        if (leader) {
            a.st->stop = why;
            loop_exit(a.cond, a.use_cond);
        }
        if (tid == kCtaThreads)  // no copy may outlive the CTA
            for (long long s = 0; s < first; s++) mbar_wait(&s_full[s % kStages], 0u);
        return;
    }
    if (producer) {  // steps kStages.. until the consumers publish their step count
        if (tid == kCtaThreads) {
            long long issued = first;
            while (issued < limit) {
                const uint32_t par = (uint32_t)((issued / kStages - 1) & 1);
                bool ok = false;
                while (!(ok = mbar_try_wait(&s_empty[issued % kStages], par)))
                    if (*(volatile long long *)&s_done >= 0) break;
                if (!ok) break;
                issue(issued++);
            }
            long long consumed;
            while ((consumed = *(volatile long long *)&s_done) < 0) {
            }
            for (long long s = consumed; s < issued; s++) mbar_wait(&s_full[s % kStages], (uint32_t)((s / kStages) & 1));
        }
        return;
    }

    // ---- a5: Hoffmann IMGS (CAC rule 9) ---------------------------------------------------
    double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const int u = u0 + j;
        v[j] = (u < nvec) ? (a.peer_mine ? ld_cv(src + u) : src[u]) : make_double2(0.0, 0.0);
        if (odd_tail && u == nvec - 1) v[j].y = 0.0;
    }
    CtaReducer red{s_wp, warp, lane, 0};
    const bool act = tid < rows;  // rows = nvec / 8: every lane of an active thread holds a vector
    double pr[8], pi[8];
    nrm_lanes<CPLX>(v, a.w, u0, nvec, pr, pi);
    const double n0 = sqrt(red.sum(pr, pi).x);
    double n_prev = n0, nn = 0.0;
    int nu = 0;
    bool accepted = false;
    long long s = 0;
    while (nu < kNuMax) {
        nu++;
        for (long long i = 0; i < k; i++, s++) {
            mbar_wait(&s_full[s % kStages], (uint32_t)((s / kStages) & 1));
            const unsigned char *wt = wtile(s), *qt = qtile(s);
#pragma unroll
            for (int j = 0; j < 8; j++) {  // DOT(WQ_i, v), CAC rule 2 (one vector per lane)
                const double2 e = act ? swz_ld(wt, tid, j) : make_double2(0.0, 0.0);
                double r = 0.0, q = 0.0;
                if (CPLX) {
                    r = fma(e.x, v[j].x, r);
                    r = fma(e.y, v[j].y, r);
                    q = fma(e.x, v[j].y, q);
                    q = fma(-e.y, v[j].x, q);
                } else {
                    r = fma(e.x, v[j].x, r);
                    r = fma(e.y, v[j].y, r);
                }
                pr[j] = r;
                pi[j] = q;
            }
            double2 qr[8];
#pragma unroll
            for (int j = 0; j < 8; j++) qr[j] = act ? swz_ld(qt, tid, j) : make_double2(0.0, 0.0);
            const double2 c = red.sum(pr, pi);
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (!act) continue;  // v <- v - c q_i, CAC rule 9
                if (CPLX) {
                    double vr = v[j].x, vi = v[j].y;
                    vr = fma(-c.x, qr[j].x, vr);
                    vr = fma(c.y, qr[j].y, vr);
                    vi = fma(-c.x, qr[j].y, vi);
                    vi = fma(-c.y, qr[j].x, vi);
                    v[j] = make_double2(vr, vi);
                } else {
                    v[j].x = fma(-c.x, qr[j].x, v[j].x);
                    v[j].y = fma(-c.x, qr[j].y, v[j].y);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[s % kStages]);  // no remote stores here
        }
        nrm_lanes<CPLX>(v, a.w, u0, nvec, pr, pi);
        nn = sqrt(red.sum(pr, pi).x);
        if (nn > n_prev / 2.0) {  // Hoffmann's test with kappa = 2
            accepted = true;
            break;
        }
        n_prev = nn;
    }
    if (tid == 0) s_done = s;  // release the producer: it drains the copies it issued
    grid_dep_launch();
    const double delta = 1000.0 * 0x1p-52;
    if (!accepted || !(nn >= delta * n0) || nn == 0.0) {
        if (leader) {
            a.nu[k] = nu;
            a.st->stop = kStopRank;
            loop_exit(a.cond, a.use_cond);
        }
        return;
    }

    // ---- q_{k+1} = v / n, w o q_{k+1}; a6 bookkeeping -----------------------------------
    const uint64_t keep = policy_evict_last();
    double2 *qo = a.Q + k * a.ldq_v;
    double2 *wqo = a.WQ + k * a.ldq_v;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const int u = u0 + j;
        if (u < nvec) {
            const double2 qq = make_double2(v[j].x / nn, v[j].y / nn);
            st_keep(qo + u, qq, keep);
            if (CPLX) {
                const double wu = a.w[u];
                st_keep(wqo + u, make_double2(wu * qq.x, wu * qq.y), keep);
            } else {
                st_keep(wqo + u, make_double2(a.w[2 * u] * qq.x, a.w[2 * u + 1] * qq.y), keep);
            }
        }
    }
    if (leader) {
        a.piv[k] = J;
        a.nu[k] = nu;
        a.rdiag[k] = nn;
        const long long jl = local_col(a, J);
        if (jl >= 0) a.r2[jl] = -INFINITY;
        a.st->k = k + 1;
    }
}

}  // namespace

bool imgs_cta_fits(long long nvec) {
    static const bool off = getenv("RBG_IMGS_CLUSTER") != nullptr;
    return !off && nvec >= 8 && nvec <= 2048 && nvec % 8 == 0;
}

cudaError_t make_imgs_cta_maps(const double2 *WQ, const double2 *Q, long long nvec, long long ldq_v, long long k_max,
                               void *maps) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    CUtensorMap *tm = static_cast<CUtensorMap *>(maps);
    const void *base[2] = {WQ, Q};
    for (int i = 0; i < 2; i++) {
        // (16 doubles = one thread's 8 vectors) x (nvec / 8 rows) x (k_max basis vectors)
        const cuuint64_t dims[3] = {16, (cuuint64_t)(nvec / 8), (cuuint64_t)k_max};
        const cuuint64_t strides[2] = {128, (cuuint64_t)ldq_v * 16};
        const cuuint32_t box[3] = {16, (cuuint32_t)(nvec / 8), 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        const CUresult r = encode(&tm[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void *>(base[i]), dims, strides,
                                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    return cudaSuccess;
}

cudaError_t launch_imgs_cta(const ImgsArgs &a, bool cplx, const void *maps, cudaStream_t s) {
    const CUtensorMap *tm = static_cast<const CUtensorMap *>(maps);
    auto kern = cplx ? k_imgs_cta<true> : k_imgs_cta<false>;
    const size_t smem = (size_t)kStages * 2 * kTile + 1024;  // + alignment slack
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, 1, 1);
    cfg.blockDim = dim3(kCtaThreads + 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kern, a, tm[0], tm[1]);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace rbg
