// eim.cu -- empirical interpolation nodes from the greedy basis ("the code
// also selects a set of empirical interpolation (EI) nodes using a fast algorithm"; the cited
// Alg. 5 is not in the container, so this is the standard greedy EIM in residual form,
// DESIGN.md reading R31):
//     xi_1 = q_1,  p_1 = argmax_i |xi_1(i)|^2
//     for l = 2..k:  solve T c = q_l(P) by forward substitution, T_ab = xi_b(p_a) (a >= b)
//                    xi_l = q_l - sum_{b<l} c_b xi_b,   p_l = argmax_i |xi_l(i)|^2
// Ties go to the lowest row index.  Every sum runs sequentially in b with explicit fma, the
// complex division uses one fixed formula, so the GPU and the oracle (orc_eim) take the same
// argmax decisions bit for bit.  Per step: one CTA does the forward substitution column by
// column (a barrier per column, rows in parallel -- the same per-row DAG as the row-wise
// sequential sum), then a grid over the N rows forms xi_l, |xi_l|^2 and a deterministic
// maxloc (last-block-done), and gathers row l of T.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace rbg {

__device__ __forceinline__ double2 load_q(const double2 *Q, long long ldq_v, bool cplx, int col, long long row) {
    // complex: element row is vector row; real: element row is half of vector row/2
    const double2 *c = Q + (long long)col * ldq_v;
    if (cplx) return c[row];
    const double2 v = c[row >> 1];
    return make_double2((row & 1) ? v.y : v.x, 0.0);
}

// acc - c * x  (CAC rule 9 pattern)
__device__ __forceinline__ double2 cmsub(double2 acc, double2 c, double2 x) {
    acc.x = fma(-c.x, x.x, acc.x);
    acc.x = fma(c.y, x.y, acc.x);
    acc.y = fma(-c.x, x.y, acc.y);
    acc.y = fma(-c.y, x.x, acc.y);
    return acc;
}

// a / b with den = fma(b.x, b.x, b.y*b.y) (R31)
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
    const double den = fma(b.x, b.x, b.y * b.y);
    return make_double2(fma(a.x, b.x, a.y * b.y) / den, fma(a.y, b.x, -(a.x * b.y)) / den);
}

struct EimArgs {
    const double2 *Q;
    long long ldq_v;
    long long N;
    bool cplx;
    int k;
    double2 *Xi;     // k columns of N complex
    double2 *T;      // k x k row-major, T[a*k + b] = xi_b(p_a)
    double2 *Tt;     // the same, column-major: Tt[b*k + a] = xi_b(p_a)
    double2 *c;      // k coefficients
    long long *nodes;
    double *bm;      // per-block maxloc values
    long long *bj;   // per-block maxloc rows
    unsigned *ticket;
    int *status;     // 0 ok, 1 degenerate (zero residual)
};

// Forward substitution for step l (l >= 1): c_a for a < l.  One thread per row r; the row's
// entries T[r][b] are loaded 4 columns at a time, one batch ahead of use, so no step waits on
// memory; c_b is broadcast through a two-slot shared buffer (one barrier per column: slot
// b & 1 is rewritten at column b + 2, after every thread passed the barrier of b + 1).
constexpr int kEimBatch = 4;

__global__ void __launch_bounds__(1024) k_eim_solve(EimArgs a, int l) {
    __shared__ double2 cb[2];
    const int r = threadIdx.x;
    const bool mine = r < l;
    double2 v = make_double2(0.0, 0.0), tdiag = make_double2(1.0, 0.0);
    if (mine) {
        v = load_q(a.Q, a.ldq_v, a.cplx, l, a.nodes[r]);   // rhs q_l(p_r)
        tdiag = a.T[(long long)r * a.k + r];
    }
    const double2 *trow = a.T + (long long)r * a.k;
    double2 tn[kEimBatch];
#pragma unroll
    for (int j = 0; j < kEimBatch; j++) tn[j] = (mine && j < r) ? trow[j] : make_double2(0.0, 0.0);
    for (int b0 = 0; b0 < l; b0 += kEimBatch) {
        double2 t[kEimBatch];
#pragma unroll
        for (int j = 0; j < kEimBatch; j++) {
            t[j] = tn[j];
            const int bn = b0 + kEimBatch + j;
            tn[j] = (mine && bn < r) ? trow[bn] : make_double2(0.0, 0.0);   // next batch
        }
#pragma unroll 1
        for (int j = 0; j < kEimBatch && b0 + j < l; j++) {  // uniform over the block
            const int b = b0 + j;
            if (r == b) {
                const double2 cv = cdiv(v, tdiag);
                cb[b & 1] = cv;
                a.c[b] = cv;
            }
            __syncthreads();
            if (r > b && mine) v = cmsub(v, cb[b & 1], t[0]);
#pragma unroll
            for (int m = 0; m + 1 < kEimBatch; m++) t[m] = t[m + 1];  // t[0] = T[r][b + 1]
        }
    }
}

// xi_l over all rows + maxloc of |xi_l|^2; the last block sets p_l and row l of T.
constexpr int kEimThreads = 128;

__global__ void __launch_bounds__(kEimThreads) k_eim_residual(EimArgs a, int l) {
    __shared__ double s_m[kEimThreads / 32];
    __shared__ long long s_j[kEimThreads / 32];
    __shared__ int s_last;
    extern __shared__ double2 s_c[];  // c_0 .. c_{l-1}
    for (int b = threadIdx.x; b < l; b += blockDim.x) s_c[b] = a.c[b];
    __syncthreads();
    double bm = -1.0;
    long long bj = 0x7fffffffffffffffLL;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.N; i += (long long)gridDim.x * blockDim.x) {
        double2 x = load_q(a.Q, a.ldq_v, a.cplx, l, i);
        // x -= c_b xi_b in increasing b; the xi loads of a batch are issued together
        for (int b0 = 0; b0 < l; b0 += 16) {
            double2 xi[16];
#pragma unroll
            for (int j = 0; j < 16; j++)
                xi[j] = (b0 + j < l) ? a.Xi[(long long)(b0 + j) * a.N + i] : make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < 16; j++)
                if (b0 + j < l) x = cmsub(x, s_c[b0 + j], xi[j]);
        }
        a.Xi[(long long)l * a.N + i] = x;
        const double m = fma(x.x, x.x, x.y * x.y);
        if (m > bm) {  // rows visited in increasing order per thread
            bm = m;
            bj = i;
        }
    }
    for (int h = 16; h >= 1; h >>= 1) {
        const double om = __shfl_xor_sync(0xffffffffu, bm, h);
        const long long oj = __shfl_xor_sync(0xffffffffu, bj, h);
        if (rec_better(om, oj, bm, bj)) {
            bm = om;
            bj = oj;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        s_m[threadIdx.x >> 5] = bm;
        s_j[threadIdx.x >> 5] = bj;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kEimThreads / 32; w++)
            if (rec_better(s_m[w], s_j[w], bm, bj)) {
                bm = s_m[w];
                bj = s_j[w];
            }
        a.bm[blockIdx.x] = bm;
        a.bj[blockIdx.x] = bj;
        __threadfence();
        s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) {
        bm = -1.0;
        bj = 0x7fffffffffffffffLL;
        for (int b = 0; b < (int)gridDim.x; b++) {
            const double m = __ldcg(&a.bm[b]);
            const long long j = __ldcg(&a.bj[b]);
            if (rec_better(m, j, bm, bj)) {
                bm = m;
                bj = j;
            }
        }
        *a.ticket = 0u;
        if (!(bm > 0.0)) {
            *a.status = 1;
            bj = 0;
        }
        a.nodes[l] = bj;
        s_j[0] = bj;
    }
    __syncthreads();
    const long long p = s_j[0];
    for (int b = threadIdx.x; b <= l; b += blockDim.x) {
        const double2 t = __ldcg(&a.Xi[(long long)b * a.N + p]);
        a.T[(long long)l * a.k + b] = t;
        a.Tt[(long long)b * a.k + l] = t;
    }
}

// ---- warp-level forward substitution (default) -----------------------------------------
// One solver warp; row a lives in lane a % 32, register slot a / 32.  Blocked right-looking
// substitution, 32 columns b at a time (block sb = the columns whose rows are slot sb):
//  * phase A (the serial chain): for b in the block, c_b = v_b / T_bb from the owner lane's
//    numerators, the real and imaginary quotients divided by lanes 0 and 1 at once (a
//    division of an exact zero is skipped: it would take the ~1,000-clock slow path,
//    scripts/chain_probe.cu), two shuffles broadcast it and the lanes update slot sb's rows;
//  * phase B (no per-column dependency): the rows of each later slot receive the block's 32
//    updates in increasing b.
// Every row still receives its updates in increasing b -- the oracle's sequential sum -- so
// the bits are those of the unblocked substitution.  T arrives as 32 x 32 tiles of the
// column-major copy Tt (tile (sb, s) = columns of block sb, rows of slot s), one 2D TMA box
// each, in consumption order, through a shared-memory ring filled by a producer warp.
constexpr int kEimRing = 8;                  // 16 KB tiles
constexpr size_t kEimTile = 32 * 32 * 16;
constexpr size_t kEimSmem = kEimRing * kEimTile + 2 * kEimRing * sizeof(uint64_t) + 32 * sizeof(double2);

__device__ __forceinline__ void tma_tile_g2s(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

template <int SLOTS>
__global__ void __launch_bounds__(64) k_eim_solve_w(EimArgs a, int l, const __grid_constant__ CUtensorMap tmT) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const double2(*ring)[32][32] = reinterpret_cast<const double2(*)[32][32]>(sm);
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + kEimRing * kEimTile), *empty = full + kEimRing;
    double2 *s_c = reinterpret_cast<double2 *>(empty + kEimRing);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nblk = (l + 31) / 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kEimRing; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
    }
    __syncthreads();
    if (warp == 1) {  // producer: tiles (sb, s), s = sb..nblk-1, in the solver's order
        if (lane == 0) {
            int n = 0;
            for (int sb = 0; sb < nblk; sb++)
                for (int s = sb; s < nblk; s++, n++) {
                    const int slot = n % kEimRing;
                    if (n >= kEimRing) mbar_wait(&empty[slot], (uint32_t)((n / kEimRing - 1) & 1));
                    mbar_arrive_expect_tx(&full[slot], (uint32_t)kEimTile);
                    // x = row offset in doubles (2 per complex row), y = column b
                    tma_tile_g2s((void *)&ring[slot][0][0], &tmT, s * 64, sb * 32, &full[slot]);
                }
        }
        return;
    }
    double2 v[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; s++) {
        const int r = s * 32 + lane;
        v[s] = r < l ? load_q(a.Q, a.ldq_v, a.cplx, l, a.nodes[r]) : make_double2(0.0, 0.0);   // q_l(p_r)
    }
    int n = 0;   // tiles consumed
#pragma unroll
    for (int sb = 0; sb < SLOTS; sb++) {
        if (sb < nblk) {
            const int b0 = sb * 32, bl_end = l - b0 < 32 ? l - b0 : 32;
            const int r = b0 + lane;
            const double2 td = r < l ? a.Tt[(long long)r * a.k + r] : make_double2(1.0, 0.0);
            const double dd = fma(td.x, td.x, td.y * td.y);
            // phase A on tile (sb, sb)
            int slot = n % kEimRing;
            mbar_wait(&full[slot], (uint32_t)((n / kEimRing) & 1));
#pragma unroll 1
            for (int bl = 0; bl < bl_end; bl++) {
                // cdiv(v_b, T_bb): the owner's two numerators and den go to lanes 0 and 1, which
                // divide at the same time (one division latency on the chain, not two); an
                // exactly zero numerator is not divided (0 / den = +-0 exactly, den > 0), as it
                // would take the division's slow path (real data: every imaginary part)
                const double n1 = __shfl_sync(0xffffffffu, fma(v[sb].x, td.x, v[sb].y * td.y), bl);
                const double n2 = __shfl_sync(0xffffffffu, fma(v[sb].y, td.x, -(v[sb].x * td.y)), bl);
                const double den = __shfl_sync(0xffffffffu, dd, bl);
                double q = 0.0;
                if (lane < 2) {
                    const double num = lane ? n2 : n1;
                    q = num == 0.0 ? num : num / den;
                }
                const double2 cb = make_double2(__shfl_sync(0xffffffffu, q, 0), __shfl_sync(0xffffffffu, q, 1));
                if (lane == bl) {
                    a.c[b0 + bl] = cb;
                    s_c[bl] = cb;
                }
                if (lane > bl && lane < bl_end) v[sb] = cmsub(v[sb], cb, ring[slot][bl][lane]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            n++;
            // phase B on tiles (sb, s), s > sb
#pragma unroll
            for (int s = sb + 1; s < SLOTS; s++) {
                if (s < nblk) {
                    slot = n % kEimRing;
                    mbar_wait(&full[slot], (uint32_t)((n / kEimRing) & 1));
                    double2 x = v[s];
#pragma unroll 8
                    for (int bl = 0; bl < bl_end; bl++) x = cmsub(x, s_c[bl], ring[slot][bl][lane]);
                    v[s] = x;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[slot]);
                    n++;
                }
            }
        }
    }
}

// IEEE num / den (round to nearest) from y = RN(1 / den), precomputed off the chain: q0 = num y,
// then two FMA remainder corrections; with y correctly rounded and the second correction
// starting within one ulp, the result is the correctly rounded quotient (Markstein's theorem)
// whenever nothing over- or underflows -- guaranteed here by |num|, den in [2^-500, 2^500];
// outside that range (and for num = 0, NaN, inf) the division itself is used.  Checked against
// the division on 3.5e9 random and adversarial operand pairs (scripts/div_check.c,
// tests/test_div_check.py): no difference.  Three dependent FMAs instead of the division's ~400-clock sequence on the
// substitution's serial chain.
__device__ __forceinline__ double div_rn_pre(double num, double den, double y, bool den_ok) {
    const double an = fabs(num);
    const double q0 = num * y;
    const double q1 = fma(fma(-q0, den, num), y, q0);
    const double q2 = fma(fma(-q1, den, num), y, q1);
    if (den_ok && an >= 0x1p-500 && an <= 0x1p500) return q2;
    if (num == 0.0) return num;   // 0 / den = +-0 exactly (den > 0)
    return num / den;
}

// Both components of a complex quotient (n1 + i n2) / den with one range test: when both
// numerators are in range (and den is) each component is div_rn_pre's fast path, so the two
// three-FMA chains interleave instead of running one after the other behind their branches;
// otherwise each component goes through div_rn_pre itself.  Same bits either way.
__device__ __forceinline__ double2 div2_rn_pre(double n1, double n2, double den, double y, bool den_ok) {
    const double q01 = n1 * y, q02 = n2 * y;
    const double q11 = fma(fma(-q01, den, n1), y, q01), q12 = fma(fma(-q02, den, n2), y, q02);
    const double q21 = fma(fma(-q11, den, n1), y, q11), q22 = fma(fma(-q12, den, n2), y, q12);
    const double a1 = fabs(n1), a2 = fabs(n2);
    if (den_ok && a1 >= 0x1p-500 && a1 <= 0x1p500 && a2 >= 0x1p-500 && a2 <= 0x1p500) return make_double2(q21, q22);
    return make_double2(div_rn_pre(n1, den, y, den_ok), div_rn_pre(n2, den, y, den_ok));
}

// ---- multi-warp forward substitution (default, round 2) ----------------------------------
// The serial chain of k_eim_solve_w is A(0) -> B(0,1) -> A(1) -> B(1,2) -> ... (phase A of a
// block, then the next block's update by it); the other phase-B tiles (sb, s), s > sb + 1, only
// have to be done before block s's turn.  So one main warp runs the chain (its tiles (sb, sb) and
// (sb, sb+1) through the TMA ring), and helper warp s - 2 owns row block s >= 2: it applies the
// tiles (0, s) .. (s-2, s) in increasing sb as each block's coefficients are published (an
// mbarrier per block), reading T from L2 with 8 loads in flight, then hands its rows to the main
// warp (an mbarrier per block).  Every row still receives its updates in increasing b, one
// cmsub each, so the bits are those of the unblocked substitution.  Threads 32 (nblk + 1) for
// nblk = ceil(l / 32) <= 15 row blocks (512 threads, so 128 registers per thread and no spills
// on the chain; longer solves, l > 480, take the single-warp solver -- same bits).
constexpr int kEimMwMaxBlk = 15;
constexpr int kEimMwRing = 4;
constexpr size_t kEimMwSmem = kEimMwRing * kEimTile + 2 * kEimMwRing * sizeof(uint64_t) +
                              2 * 32 * sizeof(uint64_t) + 1024 * sizeof(double2) + 32 * 32 * sizeof(double2);

__global__ void __launch_bounds__(512) k_eim_solve_mw(EimArgs a, int l, const __grid_constant__ CUtensorMap tmT) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const double2(*ring)[32][32] = reinterpret_cast<const double2(*)[32][32]>(sm);
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + kEimMwRing * kEimTile), *empty = full + kEimMwRing;
    uint64_t *coefbar = empty + kEimMwRing;        // [32]: block sb's coefficients are in s_c
    uint64_t *vbar = coefbar + 32;                 // [32]: block s's rows are in s_v[s]
    double2 *s_c = reinterpret_cast<double2 *>(vbar + 32);   // c_0 .. c_{l-1}
    double2(*s_v)[32] = reinterpret_cast<double2(*)[32]>(s_c + 1024);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nblk = (l + 31) / 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kEimMwRing; i++) {
            mbar_init_nofence(&full[i], 1);
            mbar_init_nofence(&empty[i], 1);
        }
        for (int i = 0; i < 32; i++) {
            mbar_init_nofence(&coefbar[i], 1);
            mbar_init_nofence(&vbar[i], 1);
        }
        fence_mbarrier_init();
    }
    grid_dep_wait();     // programmatic dependent launch: T, the nodes and Q are the residual's
    grid_dep_launch();
    __syncthreads();
    if (warp == 1) {  // producer: the main warp's tiles (sb, sb), (sb, sb + 1) in its order
        if (lane == 0) {
            int n = 0;
            for (int sb = 0; sb < nblk; sb++)
                for (int s = sb; s < nblk && s <= sb + 1; s++, n++) {
                    const int slot = n % kEimMwRing;
                    if (n >= kEimMwRing) mbar_wait(&empty[slot], (uint32_t)((n / kEimMwRing - 1) & 1));
                    mbar_arrive_expect_tx(&full[slot], (uint32_t)kEimTile);
                    tma_tile_g2s((void *)&ring[slot][0][0], &tmT, s * 64, sb * 32, &full[slot]);
                }
        }
        return;
    }
    if (warp >= 2) {  // helper for row block s = warp: tiles (0, s) .. (s - 2, s)
        const int sblk = warp;
        const int r = sblk * 32 + lane;
        const bool mine = r < l;
        double2 x = mine ? load_q(a.Q, a.ldq_v, a.cplx, l, a.nodes[r]) : make_double2(0.0, 0.0);
        const int ncols = 32 * (sblk - 1);            // columns 0 .. 32 (s - 1) - 1, all full blocks
        const double2 *tcol = a.Tt + r;               // Tt[b * k + r]
        double2 tr[8];
#pragma unroll
        for (int j = 0; j < 8; j++) tr[j] = (mine && j < ncols) ? tcol[(long long)j * a.k] : make_double2(0.0, 0.0);
        for (int b = 0; b < ncols; b += 8) {
            if ((b & 31) == 0) mbar_wait(&coefbar[b >> 5], 0u);
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const double2 t = tr[j];
                const int bn = b + 8 + j;
                tr[j] = (mine && bn < ncols) ? tcol[(long long)bn * a.k] : make_double2(0.0, 0.0);
                if (mine) x = cmsub(x, s_c[b + j], t);
            }
        }
        s_v[sblk][lane] = x;
        __syncwarp();
        if (lane == 0) mbar_arrive(&vbar[sblk]);
        return;
    }
    // main warp (warp 0)
    __shared__ double s_den[32], s_y[32];
    __shared__ int s_ok[32];
    double2 v = lane < l ? load_q(a.Q, a.ldq_v, a.cplx, l, a.nodes[lane]) : make_double2(0.0, 0.0);
    double2 td = lane < l ? a.Tt[(long long)lane * a.k + lane] : make_double2(1.0, 0.0);   // T[r][r], r = lane
    int n = 0;
    for (int sb = 0; sb < nblk; sb++) {
        const int b0 = sb * 32, bl_end = l - b0 < 32 ? l - b0 : 32;
        const int r = b0 + lane;
        // the next block's diagonal, loaded a block ahead (its latency off the chain)
        const double2 td_next = r + 32 < l ? a.Tt[(long long)(r + 32) * a.k + r + 32] : make_double2(1.0, 0.0);
        const double dd = fma(td.x, td.x, td.y * td.y);
        const double yy = 1.0 / dd;   // RN(1 / den) of this lane's column, off the chain
        const int dok = dd >= 0x1p-500 && dd <= 0x1p500;
        // the block's per-column constants go to shared memory: broadcast reads off the chain
        // instead of three more shuffles per column in the MIO queue ahead of the numerators'
        s_den[lane] = dd;
        s_y[lane] = yy;
        s_ok[lane] = dok;
        __syncwarp();
        int slot = n % kEimMwRing;
        mbar_wait(&full[slot], (uint32_t)((n / kEimMwRing) & 1));
        // lane predicates as loop-carried bit masks shifted once per column (bit 0: this column),
        // so the compiler cannot re-derive them from the lane id on the chain
        unsigned updb = (lane < bl_end) ? ((1u << lane) - 1u) : 0u;   // bit bl set iff bl < lane
        unsigned meb = 1u << lane;                                      // bit bl set iff bl == lane
        double2 mycb = make_double2(0.0, 0.0);
#pragma unroll 1
        for (int bl = 0; bl < bl_end; bl++) {  // phase A: the same quotients as k_eim_solve_w
            // every lane forms c_b itself from the owner's numerators (no divergent branch and
            // no broadcast of the quotients); the tile entry is read before the chain needs it
            const double2 t = ring[slot][bl][lane];
            const double den = s_den[bl], y = s_y[bl];
            const bool den_ok = s_ok[bl] != 0;
            const double n1 = __shfl_sync(0xffffffffu, fma(v.x, td.x, v.y * td.y), bl);
            const double n2 = __shfl_sync(0xffffffffu, fma(v.y, td.x, -(v.x * td.y)), bl);
            const double2 cb = div2_rn_pre(n1, n2, den, y, den_ok);
            if (meb & 1u) mycb = cb;   // this lane's coefficient, stored after the loop
            if (updb & 1u) v = cmsub(v, cb, t);
            updb >>= 1;
            meb >>= 1;
        }
        if (lane < bl_end) {
            a.c[b0 + lane] = mycb;
            s_c[b0 + lane] = mycb;
        }
        __syncwarp();   // the coefficients are in place; s_den / s_y / s_ok are rewritten next block
        if (lane == 0) {
            mbar_arrive(&empty[slot]);
            mbar_arrive(&coefbar[sb]);  // release: block sb's coefficients for the helpers
        }
        n++;
        if (sb + 1 < nblk) {  // the next block's rows, then its update by block sb
            double2 x;
            if (sb + 1 >= 2) {
                mbar_wait(&vbar[sb + 1], 0u);
                x = s_v[sb + 1][lane];
            } else {
                x = 32 + lane < l ? load_q(a.Q, a.ldq_v, a.cplx, l, a.nodes[32 + lane]) : make_double2(0.0, 0.0);
            }
            slot = n % kEimMwRing;
            mbar_wait(&full[slot], (uint32_t)((n / kEimMwRing) & 1));
#pragma unroll 8
            for (int bl = 0; bl < 32; bl++) x = cmsub(x, s_c[b0 + bl], ring[slot][bl][lane]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            n++;
            v = x;
        }
        td = td_next;
    }
}

// The EIM steps' kernels go out as programmatic dependents of their predecessor (each calls
// grid_dep_wait before it reads anything): the launch latency between the ~600 short kernels
// of an EIM run overlaps the predecessor's tail.  RBG_NO_PDL turns it off (same bits).
static bool eim_pdl() {
    static const bool off = getenv("RBG_NO_PDL") != nullptr;
    return !off;
}

template <typename... Args>
static cudaError_t launch_dep(void (*kern)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = eim_pdl() ? 1 : 0;
    lc.attrs = attr;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, kern, args...);
}

static cudaError_t launch_solve_mw(const EimArgs &a, int l, const CUtensorMap &tm, cudaStream_t s) {
    const int nblk = (l + 31) / 32;
    cudaError_t e = cudaFuncSetAttribute(k_eim_solve_mw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEimMwSmem);
    if (e != cudaSuccess) return e;
    e = launch_dep(k_eim_solve_mw, dim3(1), dim3(32 * (nblk > 2 ? nblk : 2)), kEimMwSmem, s, a, l, tm);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// xi_l over all rows with a ring of kEimU loads in flight per thread (one row per thread, the
// xi_b of row i consumed in increasing b: the oracle's sequential sum), maxloc as k_eim_residual.
constexpr int kEimU = 32;
constexpr int kEimThreadsW = 64;

// The end of a residual step (every thread of the block): xi_l(i) stored, |xi_l(i)|^2 into the
// block's maxloc, the last block to finish reduces the per-block records (ties: lowest row),
// records the node p_l and gathers row l of T (T[l][b] = xi_b(p_l), b <= l).
template <int WARPS>
__device__ __forceinline__ void eim_residual_finish(const EimArgs &a, int l, double2 x, bool mine, long long i) {
    __shared__ double s_m[WARPS];
    __shared__ long long s_j[WARPS];
    __shared__ int s_last;
    double bm = -1.0;
    long long bj = 0x7fffffffffffffffLL;
    if (mine) {
        a.Xi[(long long)l * a.N + i] = x;
        bm = fma(x.x, x.x, x.y * x.y);
        bj = i;
    }
    for (int h = 16; h >= 1; h >>= 1) {
        const double om = __shfl_xor_sync(0xffffffffu, bm, h);
        const long long oj = __shfl_xor_sync(0xffffffffu, bj, h);
        if (rec_better(om, oj, bm, bj)) {
            bm = om;
            bj = oj;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        s_m[threadIdx.x >> 5] = bm;
        s_j[threadIdx.x >> 5] = bj;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++)  // WARPS >= the block's warps
            if (rec_better(s_m[w], s_j[w], bm, bj)) {
                bm = s_m[w];
                bj = s_j[w];
            }
        a.bm[blockIdx.x] = bm;
        a.bj[blockIdx.x] = bj;
        __threadfence();
        s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < 32) {  // one warp reduces the per-block records
        bm = -1.0;
        bj = 0x7fffffffffffffffLL;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
            const double m = __ldcg(&a.bm[b]);
            const long long j = __ldcg(&a.bj[b]);
            if (rec_better(m, j, bm, bj)) {
                bm = m;
                bj = j;
            }
        }
        for (int h = 16; h >= 1; h >>= 1) {
            const double om = __shfl_xor_sync(0xffffffffu, bm, h);
            const long long oj = __shfl_xor_sync(0xffffffffu, bj, h);
            if (rec_better(om, oj, bm, bj)) {
                bm = om;
                bj = oj;
            }
        }
        if (threadIdx.x == 0) {
            *a.ticket = 0u;
            if (!(bm > 0.0)) {
                *a.status = 1;
                bj = 0;
            }
            a.nodes[l] = bj;
            s_j[0] = bj;
        }
    }
    __syncthreads();
    const long long p = s_j[0];
    for (int b = threadIdx.x; b <= l; b += blockDim.x) {
        const double2 t = __ldcg(&a.Xi[(long long)b * a.N + p]);
        a.T[(long long)l * a.k + b] = t;
        a.Tt[(long long)b * a.k + l] = t;
    }
}

__global__ void __launch_bounds__(kEimThreadsW) k_eim_residual_w(EimArgs a, int l) {
    extern __shared__ double2 s_c[];  // c_0 .. c_{l-1}
    for (int b = threadIdx.x; b < l; b += blockDim.x) s_c[b] = a.c[b];
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const bool mine = i < a.N;
    double2 xr[kEimU];
#pragma unroll
    for (int t = 0; t < kEimU; t++) xr[t] = (mine && t < l) ? a.Xi[(long long)t * a.N + i] : make_double2(0.0, 0.0);
    double2 x = mine ? load_q(a.Q, a.ldq_v, a.cplx, l, i) : make_double2(0.0, 0.0);
    __syncthreads();
    for (int b0 = 0; b0 < l; b0 += kEimU) {
#pragma unroll
        for (int t = 0; t < kEimU; t++) {
            const int b = b0 + t, bn = b + kEimU;
            const double2 xi = xr[t];
            xr[t] = (mine && bn < l) ? a.Xi[(long long)bn * a.N + i] : make_double2(0.0, 0.0);
            if (b < l) x = cmsub(x, s_c[b], xi);
        }
    }
    eim_residual_finish<kEimThreadsW / 32>(a, l, x, mine, i);
}

// The same step with the xi_b staged through shared memory by a 2D tensor-map TMA (round 2):
// one CTA per SM owns `rows` consecutive rows (ceil(N / SMs), at most 128); a producer warp
// streams the (rows x kEimSb) tiles of Xi -- rows r0.., basis columns b0.. -- into `nst`
// shared-memory stages (full / empty mbarriers, as many stages as fit: 6 at N = 10,000), and
// each compute thread consumes its row's xi_b from shared memory in increasing b (the same
// cmsub chain as k_eim_residual_w, so the same bits).  k_eim_residual_w keeps 32 loads in
// flight per row thread (5 MB over the device), which holds a step at ~1.3 TB/s from L2.
constexpr int kEimSb = 32;        // basis columns per stage
constexpr int kEimMaxRows = 128;  // box inner dimension 2 * rows <= 256 doubles
constexpr int kEimMaxStages = 8;

struct EimTiles {
    int rows;     // rows per CTA (a multiple of 4)
    int nst;      // stages
    size_t smem;  // dynamic shared memory
};

static EimTiles eim_tiles(long long N, int k, int num_sms) {
    EimTiles t;
    long long r = (N + num_sms - 1) / num_sms;
    r = (r + 3) / 4 * 4;
    t.rows = (int)(r < 4 ? 4 : (r > kEimMaxRows ? kEimMaxRows : r));
    const size_t stage = (size_t)t.rows * kEimSb * 16;
    const size_t fixed = 2 * kEimMaxStages * sizeof(uint64_t) + sizeof(double2) * (size_t)k;
    const size_t budget = 220 * 1024;
    int n = (int)((budget - fixed) / stage);
    t.nst = n < 2 ? 2 : (n > kEimMaxStages ? kEimMaxStages : n);
    t.smem = (size_t)t.nst * stage + fixed;
    return t;
}

__global__ void __launch_bounds__(kEimMaxRows + 32, 1) k_eim_residual_t(EimArgs a, int l, int rows, int nst,
                                                                       const __grid_constant__ CUtensorMap tmXi) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const double2 *stage = reinterpret_cast<const double2 *>(sm);       // [nst][kEimSb][rows]
    const size_t stage_elems = (size_t)kEimSb * rows;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + nst * stage_elems * 16), *empty = full + kEimMaxStages;
    double2 *s_c = reinterpret_cast<double2 *>(empty + kEimMaxStages);   // c_0 .. c_{l-1}
    const int tid = threadIdx.x;
    const int cthreads = (rows + 31) / 32 * 32;   // compute warps; the producer warp follows
    const long long r0 = (long long)blockIdx.x * rows;
    const int nt = (l + kEimSb - 1) / kEimSb;
    if (tid == 0) {
        for (int i = 0; i < nst; i++) {
            mbar_init_nofence(&full[i], 1);
            mbar_init_nofence(&empty[i], cthreads / 32);
        }
        fence_mbarrier_init();
    }
    // programmatic dependent launch (run_eim): everything below reads the solve's and the
    // previous steps' outputs; the next solve may be launched now (it waits the same way)
    grid_dep_wait();
    grid_dep_launch();
    for (int b = tid; b < l; b += blockDim.x) s_c[b] = a.c[b];
    __syncthreads();
    double2 x = make_double2(0.0, 0.0);
    bool mine = false;
    long long i = 0;
    if (tid >= cthreads) {  // producer warp
        if (tid == cthreads) {
            for (int st = 0; st < nt; st++) {
                const int slot = st % nst;
                if (st >= nst) mbar_wait(&empty[slot], (uint32_t)((st / nst - 1) & 1));
                mbar_arrive_expect_tx(&full[slot], (uint32_t)(stage_elems * 16));
                tma_tile_g2s((void *)(stage + slot * stage_elems), &tmXi, (int)(2 * r0), st * kEimSb, &full[slot]);
            }
        }
    } else {
        i = r0 + tid;
        mine = tid < rows && i < a.N;
        x = mine ? load_q(a.Q, a.ldq_v, a.cplx, l, i) : make_double2(0.0, 0.0);
        const int col = tid < rows ? tid : 0;
        for (int st = 0; st < nt; st++) {
            const int slot = st % nst;
            mbar_wait(&full[slot], (uint32_t)((st / nst) & 1));
            const int b0 = st * kEimSb, bend = l - b0 < kEimSb ? l - b0 : kEimSb;
            const double2 *tile = stage + slot * stage_elems + col;
            if (bend == kEimSb) {
#pragma unroll 8
                for (int bb = 0; bb < kEimSb; bb++) x = cmsub(x, s_c[b0 + bb], tile[bb * rows]);
            } else {
                for (int bb = 0; bb < bend; bb++) x = cmsub(x, s_c[b0 + bb], tile[bb * rows]);
            }
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
        }
    }
    eim_residual_finish<kEimMaxRows / 32 + 1>(a, l, x, mine, i);
}

template <int SLOTS>
static cudaError_t launch_solve_w(const EimArgs &a, int l, const CUtensorMap &tm, cudaStream_t s) {
    // set on every call: the attribute is per device, and a process may drive several
    cudaError_t e = cudaFuncSetAttribute(k_eim_solve_w<SLOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEimSmem);
    if (e != cudaSuccess) return e;
    k_eim_solve_w<SLOTS><<<1, 64, kEimSmem, s>>>(a, l, tm);
    return cudaGetLastError();
}

static bool eim_single_warp() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("RBG_EIM");
        v = (e && !strcmp(e, "warp1")) ? 1 : 0;
    }
    return v != 0;
}

static cudaError_t launch_solve(const EimArgs &a, int l, const CUtensorMap &tm, cudaStream_t s) {
    const int slots = (l + 31) / 32;
    if (slots <= kEimMwMaxBlk && !eim_single_warp()) return launch_solve_mw(a, l, tm, s);
    if (slots <= 1) return launch_solve_w<1>(a, l, tm, s);
    if (slots <= 2) return launch_solve_w<2>(a, l, tm, s);
    if (slots <= 4) return launch_solve_w<4>(a, l, tm, s);
    if (slots <= 6) return launch_solve_w<6>(a, l, tm, s);
    if (slots <= 8) return launch_solve_w<8>(a, l, tm, s);
    if (slots <= 10) return launch_solve_w<10>(a, l, tm, s);
    if (slots <= 12) return launch_solve_w<12>(a, l, tm, s);
    if (slots <= 16) return launch_solve_w<16>(a, l, tm, s);
    if (slots <= 24) return launch_solve_w<24>(a, l, tm, s);
    return launch_solve_w<32>(a, l, tm, s);
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    return encode;
}

// 2D view of Xi for k_eim_residual_t: inner dimension 2N doubles (rows), outer k columns b;
// rows past N in the last CTA's box are zero-filled.
static cudaError_t make_xi_map(const EimArgs &a, int rows, CUtensorMap *tm) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (!encode) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {(cuuint64_t)(2 * a.N), (cuuint64_t)a.k};
    const cuuint64_t strides[1] = {(cuuint64_t)a.N * 16};
    const cuuint32_t box[2] = {(cuuint32_t)(2 * rows), kEimSb};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a.Xi, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 2D view of Tt for the solver's tiles: inner dimension 2k doubles (rows a), outer k columns b.
static cudaError_t make_tt_map(const EimArgs &a, CUtensorMap *tm) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (!encode) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {(cuuint64_t)(2 * a.k), (cuuint64_t)a.k};
    const cuuint64_t strides[1] = {(cuuint64_t)a.k * 16};
    const cuuint32_t box[2] = {64, 32};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a.Tt, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// B_ab = q_b(p_a), column-major k x k (the EIM node matrix).
__global__ void k_eim_nodes_matrix(EimArgs a, double2 *B) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)a.k * a.k;
         e += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(e % a.k), col = (int)(e / a.k);
        B[e] = load_q(a.Q, a.ldq_v, a.cplx, col, a.nodes[row]);
    }
}

cudaError_t run_eim(const double2 *Q, long long ldq_v, long long N, bool cplx, int k, long long *nodes_d, double2 *B_d,
                    int *status_d, cudaStream_t s, ScratchPool *pool) {
    if (k < 1 || k > 1024) return cudaErrorInvalidValue;
    const int blocks = (int)((N + kEimThreads - 1) / kEimThreads < 296 ? (N + kEimThreads - 1) / kEimThreads : 296);
    const long long nrec = std::max<long long>(blocks, (N + 3) / 4);   // per-block maxloc records (>= 4 rows per block)
    EimArgs a{};
    a.Q = Q;
    a.ldq_v = ldq_v;
    a.N = N;
    a.cplx = cplx;
    a.k = k;
    a.nodes = nodes_d;
    a.status = status_d;
    cudaError_t e = salloc(pool, kScEimXi, &a.Xi, sizeof(double2) * (size_t)k * N);
    if (e == cudaSuccess) e = salloc(pool, kScEimT, &a.T, sizeof(double2) * (size_t)k * k);
    if (e == cudaSuccess) e = salloc(pool, kScEimTt, &a.Tt, sizeof(double2) * (size_t)k * k);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.Tt, 0, sizeof(double2) * (size_t)k * k, s);
    CUtensorMap tmT, tmXi;
    if (e == cudaSuccess) e = make_tt_map(a, &tmT);
    if (e == cudaSuccess) e = salloc(pool, kScEimC, &a.c, sizeof(double2) * k);
    if (e == cudaSuccess) e = salloc(pool, kScEimBm, &a.bm, sizeof(double) * nrec);
    if (e == cudaSuccess) e = salloc(pool, kScEimBj, &a.bj, sizeof(long long) * nrec);
    if (e == cudaSuccess) e = salloc(pool, kScEimTicket, &a.ticket, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemsetAsync(a.ticket, 0, sizeof(unsigned), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(status_d, 0, sizeof(int), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.c, 0, sizeof(double2) * k, s);
    // RBG_EIM=block: the first version (one CTA of up to 1024 threads with a barrier per
    // column; 128-thread residual blocks with batches of 16 loads); same bits
    const char *ev = getenv("RBG_EIM");
    const bool v1 = ev && !strcmp(ev, "block");
    const int blocks_w = (int)((N + kEimThreadsW - 1) / kEimThreadsW);
    // RBG_EIM_RESID=w: the residual with per-thread load rings (round 1-2), same bits
    const char *rv = getenv("RBG_EIM_RESID");
    const bool resid_w = rv && !strcmp(rv, "w");
    int dev = 0, sms = 148;
    if (e == cudaSuccess) cudaGetDevice(&dev);
    if (e == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const EimTiles tl = eim_tiles(N, k, sms);
    const int blocks_t = (int)((N + tl.rows - 1) / tl.rows);
    const size_t t_smem = tl.smem;
    if (e == cudaSuccess && !v1 && !resid_w) e = make_xi_map(a, tl.rows, &tmXi);
    if (e == cudaSuccess && !v1 && !resid_w)
        e = cudaFuncSetAttribute(k_eim_residual_t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t_smem);
    for (int l = 0; l < k && e == cudaSuccess; l++) {
        if (l > 0) {
            if (v1) {
                k_eim_solve<<<1, (l + 31) / 32 * 32, 0, s>>>(a, l);
                e = cudaGetLastError();
            } else {
                e = launch_solve(a, l, tmT, s);
            }
        }
        if (e == cudaSuccess) {
            const size_t sh = sizeof(double2) * (size_t)(l > 0 ? l : 1);
            if (v1) k_eim_residual<<<blocks, kEimThreads, sh, s>>>(a, l);
            else if (resid_w) k_eim_residual_w<<<blocks_w, kEimThreadsW, sh, s>>>(a, l);
            else e = launch_dep(k_eim_residual_t, dim3(blocks_t), dim3((tl.rows + 31) / 32 * 32 + 32), t_smem, s, a, l,
                                tl.rows, tl.nst, tmXi);
            if (e == cudaSuccess) e = cudaGetLastError();
        }
    }
    if (e == cudaSuccess) {
        k_eim_nodes_matrix<<<64, 256, 0, s>>>(a, B_d);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    sfree(pool, a.Xi);
    sfree(pool, a.T);
    sfree(pool, a.Tt);
    sfree(pool, a.c);
    sfree(pool, a.bm);
    sfree(pool, a.bj);
    sfree(pool, a.ticket);
    return e;
}

}  // namespace rbg
