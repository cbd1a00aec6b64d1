// coeff.cu -- the coefficient block C = (W Q_k)^H V of a block of columns V against the
// whole current basis, for out-of-sample validation and enrichment (
// "as a batch it becomes a dense Q^H W V contraction").
//
// The k coefficient passes of the recurrence (one streaming sweep per basis vector) read V
// k times; here every (basis vector, column) pair of a 16 x 16 tile is accumulated in one
// pass over the rows, so V crosses HBM about once and the work is FP64-FMA bound
// (8 flops per complex element and basis vector; the basis, k x N x 16 B = 48 MB at k = 300,
// stays in L2).  No tensor cores: the CAC fixes each dot's summation order, which an MMA
// does not expose, so the contraction runs on the FP64 pipes with explicit fma().
//
// Arithmetic (bit-identical to k_sweep's coefficient pass and to orc_validate):
//  * CAC rules 1-2: pair (q_i, v_j) has 32 lane partials; lane l accumulates the 16-byte
//    vectors u = l (mod 32) of the column in increasing u, starting from +0.0, with the
//    same fma sequence as k_sweep's accum();
//  * rule 3: the pairwise lane tree with ascending offsets over the 32 lanes of the warp
//    (evaluated as a reduce-scatter: same tree nodes, fewer shuffles);
//  * rules 5-6 in k_coeff_r2: r2_j <- r2_j - |C(i,j)|^2 for i = 0..k-1 in order.
//
// Layout: CTA = 8 compute warps + 1 producer warp.  A warp owns 4 columns x 8 basis
// vectors (32 pairs, 64 fp64 accumulators per lane); the CTA tile is 16 columns x 16 basis
// vectors.  The producer stages, per stage of 64 vectors (2 lane rounds), the 16 column
// slices and the 16 basis slices (1 KB each, cp.async.bulk) into a 5-deep shared-memory
// ring with full/empty mbarriers.  CTAs of one column tile are consecutive in the grid
// (basis tile fastest), so the ~19 CTAs that read the same V columns run at the same time
// and V is fetched from HBM once.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace rbg {

constexpr int kCbTJ = 4, kCbTK = 8;        // pairs per warp: 4 columns x 8 basis vectors
constexpr int kCbWJ = 4, kCbWK = 2;        // compute warps per CTA (column x basis)
constexpr int kCbWarps = kCbWJ * kCbWK;
constexpr int kCbThreads = kCbWarps * 32;   // no producer warp: 2 warps per SMSP, 255 regs
constexpr int kCbCols = kCbTJ * kCbWJ;     // 16 columns per CTA
constexpr int kCbQs = kCbTK * kCbWK;       // 16 basis vectors per CTA
// stage geometry: RND 32-vector lane rounds per stage (slices of RND KB), STG stages
template <int RND, int STG>
struct CbGeom {
    static constexpr int kUnits = 32 * RND;
    static constexpr size_t kSlice = (size_t)kUnits * 16;
    static constexpr size_t kStage = (size_t)(kCbCols + kCbQs) * kSlice;
    static constexpr size_t kSmem = kStage * STG + STG * (sizeof(uint64_t) + sizeof(int));
    static_assert(2 * kUnits <= 256, "TMA box inner dimension is at most 256 elements");
};

// 2D tensor-map TMA load of a box (16 columns x 2*kUnits doubles) into shared memory.
__device__ __forceinline__ void tma_box_g2s(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

struct CoeffArgs {
    const double2 *V;      // column j at V + j*ldv (vectors)
    long long ldv, M;
    const double2 *WQ;     // basis vector i at WQ + i*ldq_v
    long long ldq_v, k;
    long long nvec;
    bool odd_tail;         // real, N odd: the last vector's second element is padding
    double *C;             // C(i, j) at C[i*ldc + j] (complex: double2 elements)
    long long ldc;
    int nqt;               // basis tiles
};

template <bool CPLX>
__device__ __forceinline__ void cb_accum(double &re, double &im, const double2 x, const double2 e) {
    // k_sweep accum<CPLX, false>: conj(e) * x
    if (CPLX) {
        re = fma(e.x, x.x, re);
        re = fma(e.y, x.y, re);
        im = fma(e.x, x.y, im);
        im = fma(-e.y, x.x, im);
    } else {
        re = fma(e.x, x.x, re);
        re = fma(e.y, x.y, re);
    }
}

// One reduce-scatter level over N pair partials (see the epilogue of k_coeff_block).
template <int N, bool CPLX>
__device__ __forceinline__ void cb_scatter_step(double *vr, double *vi, int lane, int h) {
    const bool up = (lane & h) != 0;
#pragma unroll
    for (int i = 0; i < N / 2; i++) {
        const double kr = up ? vr[N / 2 + i] : vr[i], sr = up ? vr[i] : vr[N / 2 + i];
        vr[i] = kr + __shfl_xor_sync(0xffffffffu, sr, h);
        if (CPLX) {
            const double ki = up ? vi[N / 2 + i] : vi[i], si = up ? vi[i] : vi[N / 2 + i];
            vi[i] = ki + __shfl_xor_sync(0xffffffffu, si, h);
        }
    }
}

// One lane round: the lane's vector ul of 4 columns and 8 basis vectors, 32 pair updates.
template <bool CPLX, int UNITS>
__device__ __forceinline__ void cb_round(double (&re)[kCbTJ][kCbTK], double (&im)[kCbTJ][kCbTK], const double2 *sv,
                                         const double2 *se, int ul, bool pad_tail) {
    double2 x[kCbTJ], e[kCbTK];
#pragma unroll
    for (int j = 0; j < kCbTJ; j++) {
        x[j] = sv[j * UNITS + ul];
        if (pad_tail) x[j].y = 0.0;  // real, N odd: row N is padding
    }
#pragma unroll
    for (int q = 0; q < kCbTK; q++) e[q] = se[q * UNITS + ul];
#pragma unroll
    for (int q = 0; q < kCbTK; q++)
#pragma unroll
        for (int j = 0; j < kCbTJ; j++) cb_accum<CPLX>(re[j][q], im[j][q], x[j], e[q]);
}

template <bool CPLX, int RND, int STG>
__global__ void __launch_bounds__(kCbThreads, 1)
    k_coeff_block(const CoeffArgs a, const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmQ) {
    using G = CbGeom<RND, STG>;
    constexpr int kCbRounds = RND, kCbUnits = G::kUnits, kCbStages = STG;
    constexpr size_t kCbStageBytes = G::kStage;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kCbStageBytes * kCbStages);
    int *done = reinterpret_cast<int *>(full + kCbStages);   // warps finished with the slot
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int qt = (int)(blockIdx.x % (unsigned)a.nqt);
    const long long ct = blockIdx.x / (unsigned)a.nqt;
    const long long j0 = ct * kCbCols, q0 = (long long)qt * kCbQs;
    const long long nvec = a.nvec;
    const long long nst = (nvec + kCbUnits - 1) / kCbUnits;
    // a box is always counted in full: rows past nvec and columns past M / k are zero-filled
    // by the TMA unit (and never stored)
    constexpr uint32_t kBox = (uint32_t)G::kSlice * kCbCols;
    static_assert(kCbCols == kCbQs, "one box size for V and WQ");
    auto issue = [&](long long st_i) {
        const int slot = (int)(st_i % kCbStages);
        const int x = (int)(st_i * kCbUnits * 2);  // in doubles
        unsigned char *dst = smem + (size_t)slot * kCbStageBytes;
        mbar_arrive_expect_tx(&full[slot], 2 * kBox);
        tma_box_g2s(dst, &tmV, x, (int)j0, &full[slot]);
        tma_box_g2s(dst + kBox, &tmQ, x, (int)q0, &full[slot]);
    };
    if (tid == 0) {
        for (int s = 0; s < kCbStages; s++) {
            mbar_init(&full[s], 1);
            done[s] = 0;
        }
        for (long long s = 0; s < nst && s < kCbStages; s++) issue(s);
    }
    __syncthreads();

    // ---- compute warps
    const int wj = warp % kCbWJ, wk = warp / kCbWJ;
    double re[kCbTJ][kCbTK], im[kCbTJ][kCbTK];
#pragma unroll
    for (int j = 0; j < kCbTJ; j++)
#pragma unroll
        for (int q = 0; q < kCbTK; q++) {
            re[j][q] = 0.0;
            im[j][q] = 0.0;
        }
    for (long long s = 0; s < nst; s++) {
        const int slot = (int)(s % kCbStages);
        mbar_wait(&full[slot], (uint32_t)((s / kCbStages) & 1));
        const double2 *sv = reinterpret_cast<const double2 *>(smem + (size_t)slot * kCbStageBytes) +
                            (size_t)wj * kCbTJ * kCbUnits;
        const double2 *se = reinterpret_cast<const double2 *>(smem + (size_t)slot * kCbStageBytes) +
                            (size_t)(kCbCols + wk * kCbTK) * kCbUnits;
        if ((s + 1) * kCbUnits <= nvec) {
            // full stage: no guards, so the scheduler can hoist the next round's shared-memory
            // loads above this round's FMAs
#pragma unroll
            for (int r = 0; r < kCbRounds; r++)
                cb_round<CPLX, kCbUnits>(re, im, sv, se, r * 32 + lane, false);
        } else {
#pragma unroll
            for (int r = 0; r < kCbRounds; r++) {
                const long long u = s * kCbUnits + r * 32 + lane;
                if (u < nvec) cb_round<CPLX, kCbUnits>(re, im, sv, se, r * 32 + lane, !CPLX && a.odd_tail && u == nvec - 1);
            }
        }
        // the last warp done with the slot refills it with stage s + kCbStages (its loads are
        // consumed: every value read from the slot has fed an FMA above)
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&done[slot], 1) == kCbWarps - 1) {
                done[slot] = 0;
                if (s + kCbStages < nst) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(s + kCbStages);
                }
            }
        }
    }

    // lane tree, ascending offsets (CAC rule 3), as a reduce-scatter: at offset h a lane keeps
    // the half of its pairs selected by bit h of its lane id and adds the partner's partials
    // of that half -- the same tree node sums as the butterfly (p[l] + p[l ^ h], IEEE +
    // commutes), 31 shuffles per component instead of 160.  Lane l ends with pair brev5(l).
    __syncwarp();
    double vr[32], vi[32];
#pragma unroll
    for (int j = 0; j < kCbTJ; j++)
#pragma unroll
        for (int q = 0; q < kCbTK; q++) {
            vr[j * kCbTK + q] = re[j][q];
            vi[j * kCbTK + q] = im[j][q];
        }
    cb_scatter_step<32, CPLX>(vr, vi, lane, 1);
    cb_scatter_step<16, CPLX>(vr, vi, lane, 2);
    cb_scatter_step<8, CPLX>(vr, vi, lane, 4);
    cb_scatter_step<4, CPLX>(vr, vi, lane, 8);
    cb_scatter_step<2, CPLX>(vr, vi, lane, 16);
    const int p = (int)(__brev((unsigned)lane) >> 27);
    const long long jc = j0 + wj * kCbTJ + p / kCbTK;
    const long long qi = q0 + wk * kCbTK + p % kCbTK;
    if (jc < a.M && qi < a.k) {
        if (CPLX) reinterpret_cast<double2 *>(a.C)[qi * a.ldc + jc] = make_double2(vr[0], vi[0]);
        else a.C[qi * a.ldc + jc] = vr[0];
    }
}

// r2_j <- r2_j - |C(i, j)|^2, i = 0..k-1 in order (CAC rules 5-6, as k_sweep does per pass).
template <bool CPLX>
__global__ void k_coeff_r2(const double *C, long long ldc, long long k, long long M, double *r2) {
    const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (j >= M) return;
    double r = r2[j];
    for (long long i = 0; i < k; i++) {
        double cc;
        if (CPLX) {
            const double2 c = reinterpret_cast<const double2 *>(C)[i * ldc + j];
            cc = fma(c.x, c.x, c.y * c.y);
        } else {
            const double c = C[i * ldc + j];
            cc = c * c;
        }
        r = r - cc;
    }
    r2[j] = r;
}

bool coeff_block_enabled() {
    const char *v = getenv("RBG_COEFF");  // "passes": k streaming coefficient sweeps instead
    return !(v && strcmp(v, "passes") == 0);
}

cudaError_t launch_coeff_block(const double2 *V, long long ldv, long long M, const double2 *WQ, long long ldq_v,
                               long long k, long long nvec, long long N, bool cplx, double *C, long long ldc,
                               double *r2, cudaStream_t s) {
    if (k <= 0 || M <= 0) return cudaSuccess;
    CoeffArgs a{};
    a.V = V;
    a.ldv = ldv;
    a.M = M;
    a.WQ = WQ;
    a.ldq_v = ldq_v;
    a.k = k;
    a.nvec = nvec;
    a.odd_tail = !cplx && (N & 1);
    a.C = C;
    a.ldc = ldc;
    a.nqt = (int)((k + kCbQs - 1) / kCbQs);
    const long long nct = (M + kCbCols - 1) / kCbCols;
    const long long grid = nct * a.nqt;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
    // tensor maps: a 2D view (2*nvec doubles x columns) of V and of the first k basis vectors
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    // RBG_COEFF_CFG = "<rounds>x<stages>" (default 4x3; 2x6 selectable)
    const char *cfg = getenv("RBG_COEFF_CFG");
    const bool small = cfg && !strcmp(cfg, "2x6");
    const int units = small ? CbGeom<2, 6>::kUnits : CbGeom<4, 3>::kUnits;
    CUtensorMap tm[2];
    const void *base[2] = {V, WQ};
    const long long cols[2] = {M, k}, ld[2] = {ldv, ldq_v};
    for (int i = 0; i < 2; i++) {
        const cuuint64_t dims[2] = {(cuuint64_t)(2 * nvec), (cuuint64_t)cols[i]};
        const cuuint64_t strides[1] = {(cuuint64_t)ld[i] * 16};
        const cuuint32_t box[2] = {(cuuint32_t)(2 * units), (cuuint32_t)kCbCols};
        const cuuint32_t estr[2] = {1, 1};
        const CUresult r = encode(&tm[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(base[i]), dims, strides,
                                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    void (*kern)(CoeffArgs, CUtensorMap, CUtensorMap) = cplx ? k_coeff_block<true, 4, 3> : k_coeff_block<false, 4, 3>;
    size_t smem = CbGeom<4, 3>::kSmem;
    if (small) {
        kern = cplx ? k_coeff_block<true, 2, 6> : k_coeff_block<false, 2, 6>;
        smem = CbGeom<2, 6>::kSmem;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, kCbThreads, smem, s>>>(a, tm[0], tm[1]);
    e = cudaGetLastError();
    if (e != cudaSuccess || !r2) return e;
    const unsigned blocks = (unsigned)((M + 255) / 256);
    if (cplx) k_coeff_r2<true><<<blocks, 256, 0, s>>>(C, ldc, k, M, r2);
    else k_coeff_r2<false><<<blocks, 256, 0, s>>>(C, ldc, k, M, r2);
    return cudaGetLastError();
}

}  // namespace rbg
