// recon.cu -- Algorithm 4 "Reconstruction" (Thm 5.8):
// after a j-term MGS with pivoting S = Q_j R(1:j, 1:M), take the SVD of the j x M block
// R(1:j, :) = V Sigma W^H and return X_k = Q_j V(:, 1:k) with sigma_{k+1} < tau2 < sigma_k,
// a POD-quality basis at O(M j^2 + N j^2) cost.
//
// The SVD is taken through the j x j Gram matrix G = R R^H = V Sigma^2 V^H (DESIGN.md
// reading R30), in three deterministic kernels:
//  * k_gram: G = R R^H over 64 x 64 tiles of (a, b) pairs (upper triangle of tiles), the
//    column range cut into chunks of kGramChunk columns; within a chunk every pair is one
//    sequential fma chain in increasing column index, chunk partials are summed in chunk
//    order by k_gram_reduce (the order the oracle's orc_gram writes out);
//  * k_jacobi: cyclic two-sided Jacobi on the Hermitian G with the round-robin (tournament)
//    ordering, one cooperative grid, three grid-wide barriers per round; converges when
//    max |g_pq| / sqrt(g_pp g_qq) < 1e-15 (or 40 sweeps);
//  * k_recon_x: X = Q V(:, 1:k), each element one sequential sum over the basis index.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace rbg {

constexpr int kGramTile = 64;   // pairs per tile side
constexpr int kGramSub = 16;    // columns staged per shared-memory step
constexpr int kGramReg = 4;     // pairs per thread per side (4 x 4 register tile)

int gram_tile() { return kGramTile; }

// R: k rows of ldr elements (row-major).  P: nchunks x k x k partial sums (complex).
// 256 threads own 4 x 4 pairs each, strided by 16 (thread (ta, tb) has pairs
// (a0 + ta + 16u, b0 + tb + 16v)); every pair is one sequential fma chain over the chunk's
// columns in increasing index (the order k_gram_reduce and the oracle's orc_gram assume).
// The pairs a CTA computes: register rows u < NU and columns v < NV hold rows / columns
// below k (the tile's last 16-row groups past k are skipped), and on a diagonal tile (DIAG)
// the groups v < u lie wholly below the diagonal (b - a <= 15 - 16 < 0) and are skipped:
// at k = 300 with 64 x 64 tiles this drops 21 % of the FMAs.
//
// Operand staging (round 2): the 64-row x 16-column slices of R for rows a0.. and b0.. come
// through a 2D tensor-map TMA with the 128-byte swizzle into kGStages shared-memory stages
// filled by a producer warp (full / empty mbarriers), so the FP64 pipes never wait for a
// global load or a CTA barrier (round 1 staged through registers between two __syncthreads:
// ncu long_scoreboard 26 % + barrier 6 % of the stall samples, FP64 pipe 55 % busy).  A row of
// a box is 128 bytes (8 complex or 16 real columns), 16-byte chunk c of row r at chunk
// c ^ (r & 7): a warp's reads of one column over 16 rows hit 8 distinct bank groups.  Rows past
// k and columns past M are zero-filled by the TMA; a diagonal tile loads its slice once.
constexpr int kGStages = 3;
constexpr int kGBox = 64 * 128;  // one box: 64 rows x 128 bytes

__device__ __forceinline__ void tma2d_g2s(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// element (row r of the tile, column cc of the stage) of a swizzled operand slice
template <bool CPLX>
__device__ __forceinline__ double2 gram_op(const unsigned char *t, int r, int cc) {
    if (CPLX)  // two boxes of 8 complex columns
        return *reinterpret_cast<const double2 *>(t + (cc >> 3) * kGBox + r * 128 + (((cc & 7) ^ (r & 7)) << 4));
    return make_double2(*reinterpret_cast<const double *>(t + r * 128 + ((((cc >> 1) ^ (r & 7))) << 4) + (cc & 1) * 8),
                        0.0);
}

template <bool CPLX, int NU, int NV, bool DIAG>
__device__ __forceinline__ void gram_tile_body(unsigned char *stg, uint64_t *full, uint64_t *empty, long long js0,
                                               long long j1, long long nst, double (&re)[kGramReg][kGramReg],
                                               double (&im)[kGramReg][kGramReg]) {
    constexpr int kOpBytes = (CPLX ? 2 : 1) * kGBox;
    const int tid = threadIdx.x, lane = tid & 31;
    const int ta = tid >> 4, tb = tid & 15;
    for (long long st = 0; st < nst; st++) {
        mbar_wait(&full[st % kGStages], (uint32_t)((st / kGStages) & 1));
        const unsigned char *A = stg + (size_t)(st % kGStages) * 2 * kOpBytes;
        const unsigned char *B = DIAG ? A : A + kOpBytes;
        const long long js = js0 + st * kGramSub;
        const int n = (int)((j1 - js) < kGramSub ? (j1 - js) : kGramSub);
        for (int cc = 0; cc < n; cc++) {
            double2 x[kGramReg], y[kGramReg];
#pragma unroll
            for (int u = 0; u < NU; u++) x[u] = gram_op<CPLX>(A, ta + 16 * u, cc);
#pragma unroll
            for (int v = 0; v < NV; v++) y[v] = gram_op<CPLX>(B, tb + 16 * v, cc);
#pragma unroll
            for (int u = 0; u < NU; u++)
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    if (DIAG && v < u) continue;
                    // G_ab += R_a conj(R_b) = DOT(R_b, R_a) term: (p,q) = R_b, (x,y) = R_a
                    re[u][v] = fma(y[v].x, x[u].x, re[u][v]);
                    re[u][v] = fma(y[v].y, x[u].y, re[u][v]);
                    im[u][v] = fma(y[v].x, x[u].y, im[u][v]);
                    im[u][v] = fma(-y[v].y, x[u].x, im[u][v]);
                }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st % kGStages]);
    }
}

template <bool CPLX, int NU>
__device__ __forceinline__ void gram_tile_nv(int nv, bool diag, unsigned char *stg, uint64_t *full, uint64_t *empty,
                                             long long js0, long long j1, long long nst,
                                             double (&re)[kGramReg][kGramReg], double (&im)[kGramReg][kGramReg]) {
#define RBG_GRAM_CASE(NV)                                                                                         \
    if (diag) gram_tile_body<CPLX, NU, NV, true>(stg, full, empty, js0, j1, nst, re, im);                         \
    else gram_tile_body<CPLX, NU, NV, false>(stg, full, empty, js0, j1, nst, re, im);
    switch (nv) {
        case 1: RBG_GRAM_CASE(1) break;
        case 2: RBG_GRAM_CASE(2) break;
        case 3: RBG_GRAM_CASE(3) break;
        default: RBG_GRAM_CASE(4) break;
    }
#undef RBG_GRAM_CASE
}

// One CTA per work item {tile a, tile b, chunk}: the host orders the items by decreasing
// work (full off-diagonal tiles, edge tiles, diagonal tiles) and, within a class, chunk-major
// (the tiles of one chunk run together and share R's slices in L2), so the block scheduler's
// last wave is made of the cheapest items (round 2: 1,500 items over 296 slots = 5.07 waves).
template <bool CPLX>
__global__ void __launch_bounds__(256 + 32, 2) k_gram(const __grid_constant__ CUtensorMap tmR, int k, long long M,
                                                      long long chunk, const int4 *items, double2 *P) {
    extern __shared__ __align__(1024) unsigned char gsm_raw[];
    unsigned char *stg = gsm_raw + ((1024u - (smem_u32(gsm_raw) & 1023u)) & 1023u);  // swizzle needs 1024-B tiles
    __shared__ __align__(8) uint64_t full[kGStages], empty[kGStages];
    constexpr int kOpBytes = (CPLX ? 2 : 1) * kGBox;
    const int4 t = items[blockIdx.x];
    const int a0 = t.x * kGramTile, b0 = t.y * kGramTile;
    const bool diag = t.x == t.y;
    const long long c = t.z;
    const long long j0 = c * chunk, j1 = (j0 + chunk < M) ? j0 + chunk : M;
    const long long nst = (j1 - j0 + kGramSub - 1) / kGramSub;
    const int tid = threadIdx.x;
    if (tid == 256) {
        for (int i = 0; i < kGStages; i++) {
            mbar_init_nofence(&full[i], 1);
            mbar_init_nofence(&empty[i], 8);
        }
        fence_mbarrier_init();
    }
    __syncthreads();
    if (tid >= 256) {  // producer warp: one thread issues the stages
        if (tid == 256) {
            const uint32_t bytes = (uint32_t)(diag ? 1 : 2) * kOpBytes;
            const int xs = CPLX ? 2 : 1;  // doubles per element
            for (long long st = 0; st < nst; st++) {
                if (st >= kGStages) mbar_wait(&empty[st % kGStages], (uint32_t)((st / kGStages - 1) & 1));
                uint64_t *bar = &full[st % kGStages];
                mbar_arrive_expect_tx(bar, bytes);
                unsigned char *A = stg + (size_t)(st % kGStages) * 2 * kOpBytes;
                const int x = (int)((j0 + st * kGramSub) * xs);
                tma2d_g2s(A, &tmR, x, a0, bar);
                if (CPLX) tma2d_g2s(A + kGBox, &tmR, x + 16, a0, bar);
                if (!diag) {
                    tma2d_g2s(A + kOpBytes, &tmR, x, b0, bar);
                    if (CPLX) tma2d_g2s(A + kOpBytes + kGBox, &tmR, x + 16, b0, bar);
                }
            }
        }
        return;
    }
    const int ta = tid >> 4, tb = tid & 15;
    double re[kGramReg][kGramReg], im[kGramReg][kGramReg];
#pragma unroll
    for (int u = 0; u < kGramReg; u++)
#pragma unroll
        for (int v = 0; v < kGramReg; v++) re[u][v] = im[u][v] = 0.0;
    // 16-row groups of the tile that hold rows / columns below k (uniform over the CTA)
    const int nu = (k - a0 + 15) / 16 < 4 ? (k - a0 + 15) / 16 : 4;
    const int nv = (k - b0 + 15) / 16 < 4 ? (k - b0 + 15) / 16 : 4;
    switch (nu) {
        case 1: gram_tile_nv<CPLX, 1>(nv, diag, stg, full, empty, j0, j1, nst, re, im); break;
        case 2: gram_tile_nv<CPLX, 2>(nv, diag, stg, full, empty, j0, j1, nst, re, im); break;
        case 3: gram_tile_nv<CPLX, 3>(nv, diag, stg, full, empty, j0, j1, nst, re, im); break;
        default: gram_tile_nv<CPLX, 4>(nv, diag, stg, full, empty, j0, j1, nst, re, im); break;
    }
#pragma unroll
    for (int u = 0; u < kGramReg; u++)
#pragma unroll
        for (int v = 0; v < kGramReg; v++) {
            const int a = a0 + ta + 16 * u, b = b0 + tb + 16 * v;
            if (a < k && b < k && b >= a) P[(c * k + a) * k + b] = make_double2(re[u][v], im[u][v]);
        }
}

// G (kp x kp column-major, ld kp, zero padded) from chunk partials, summed in chunk order,
// starting from G0 (the running sum of the previous ranks of a sharded context, same layout)
// or from zero; the lower triangle is the conjugate of the upper.  Real and imaginary parts
// are independent sums, so zeroing the diagonal's imaginary part between ranks does not
// change any other bit.
__global__ void k_gram_reduce(const double2 *P, long long nchunks, int k, int kp, const double2 *G0, double2 *G) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)kp * kp;
         e += (long long)gridDim.x * blockDim.x) {
        const int a = (int)(e % kp), b = (int)(e / kp);   // G(a, b) at a + b*kp
        double2 g = make_double2(0.0, 0.0);
        if (a < k && b < k) {
            const int lo = a < b ? a : b, hi = a < b ? b : a;
            if (G0) g = G0[lo + (long long)hi * kp];        // upper triangle of the running sum
            for (long long c = 0; c < nchunks; c++) {
                const double2 p = P[(c * k + lo) * k + hi];
                g.x = g.x + p.x;
                g.y = g.y + p.y;
            }
            if (a > b) g.y = -g.y;
            if (a == b) g.y = 0.0;  // a Hermitian matrix has a real diagonal
        }
        G[e] = g;
    }
}

// ------------------------------------------------------------------ Jacobi eigen-solver
struct Rot {
    double cs, sn, er, ei;  // rotation J = [[cs, sn], [-sn e^{-i phi}, cs e^{-i phi}]], e = e^{i phi}
    int p, q;
};

__device__ __forceinline__ void round_pair(int r, int i, int kp, int &p, int &q) {
    // round-robin tournament: player kp-1 fixed, the others rotate
    if (i == 0) {
        p = r;
        q = kp - 1;
    } else {
        p = (r + i) % (kp - 1);
        q = (r - i + kp - 1) % (kp - 1);
    }
    if (p > q) {
        const int t = p;
        p = q;
        q = t;
    }
}

__device__ __forceinline__ unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }

// Grid-wide barrier for the co-resident blocks of a cooperative launch: arrival counter +
// generation word (sense reversal), ~1-2 us instead of cooperative_groups' grid.sync.
__device__ __forceinline__ void grid_barrier(unsigned *count, unsigned *gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *vg = gen;
        const unsigned g = *vg;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0u;
            __threadfence();
            atomicExch(gen, g + 1u);
        } else {
            while (*vg == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ Rot make_rot(const double2 *G, int kp, int p, int q, unsigned long long *flag, bool note) {
    const double a = G[p + (long long)p * kp].x, b = G[q + (long long)q * kp].x;
    const double2 c = G[p + (long long)q * kp];  // g_pq
    const double ac = sqrt(c.x * c.x + c.y * c.y);
    Rot R;
    R.p = p;
    R.q = q;
    if (ac == 0.0) {
        R.cs = 1.0;
        R.sn = 0.0;
        R.er = 1.0;
        R.ei = 0.0;
    } else {
        const double den = sqrt(fabs(a * b));
        const double ratio = den > 0.0 ? ac / den : 1.0;
        if (note) atomicMax(flag, dbits(ratio));
        const double tau = (b - a) / (2.0 * ac);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        R.cs = 1.0 / sqrt(1.0 + t * t);
        R.sn = t * R.cs;
        R.er = c.x / ac;
        R.ei = c.y / ac;
    }
    return R;
}

// G: kp x kp Hermitian (column-major), V: kp x kp (column-major), identity on entry.
// flags[0..1]: per-sweep max off-diagonal ratio (double bits, atomicMax; non-negative);
// flags[2]: barrier counter / generation (two 32-bit words, zero on entry).
// Per round of the tournament: every block computes all kp/2 rotations of the round into
// its shared memory (deterministic, identical bits in every block; block 0 records the
// ratios), then G <- G J and V <- V J (columns p, q), barrier, G <- J^H G (rows p, q),
// barrier: two grid-wide barriers per round.  Phase A reads only g_pp, g_qq, g_pq of the
// round's pairs; so that no block's phase B can overwrite them while another block is still
// in phase A, phase B leaves each pair's own 2 x 2 block (rows p, q of columns p, q) in G
// untouched and writes it to the scratch B4 (4 entries per pair), which phase C reads.
__global__ void __launch_bounds__(256) k_jacobi(double2 *G, double2 *V, int kp, Rot *scratch,
                                                unsigned long long *flags, int *sweeps_out) {
    extern __shared__ __align__(16) unsigned char jsm[];
    Rot *rots = reinterpret_cast<Rot *>(jsm);
    double2 *B4 = reinterpret_cast<double2 *>(scratch);  // [pair][(row q?) + 2 (col q?)]
    unsigned *bar = reinterpret_cast<unsigned *>(flags + 2);
    const unsigned nblocks = gridDim.x;
    const int half = kp / 2;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    int sweep = 0;
    for (; sweep < 40; sweep++) {
        unsigned long long *flag = &flags[sweep & 1];
        for (int r = 0; r < kp - 1; r++) {
            // A: this round's rotations from the current 2x2 blocks (every block)
            for (int i = threadIdx.x; i < half; i += blockDim.x) {
                int p, q;
                round_pair(r, i, kp, p, q);
                rots[i] = make_rot(G, kp, p, q, flag, blockIdx.x == 0);
            }
            __syncthreads();
            // B: columns p, q of G and V: G <- G J, V <- V J
            for (long long e = gtid; e < (long long)half * kp * 2; e += nthreads) {
                const long long pair = e / (2LL * kp), rem = e % (2LL * kp);
                const int row = (int)(rem % kp);
                double2 *M = (rem < kp) ? G : V;
                const Rot R = rots[pair];
                const double2 gp = M[row + (long long)R.p * kp], gq = M[row + (long long)R.q * kp];
                // e^{-i phi} g_q
                const double2 eq = make_double2(R.er * gq.x + R.ei * gq.y, R.er * gq.y - R.ei * gq.x);
                const double2 np = make_double2(R.cs * gp.x - R.sn * eq.x, R.cs * gp.y - R.sn * eq.y);
                const double2 nq = make_double2(R.sn * gp.x + R.cs * eq.x, R.sn * gp.y + R.cs * eq.y);
                if (M == G && (row == R.p || row == R.q)) {
                    const int rq = row == R.q ? 1 : 0;
                    B4[pair * 4 + rq] = np;       // (row, p) after B
                    B4[pair * 4 + rq + 2] = nq;   // (row, q) after B
                } else {
                    M[row + (long long)R.p * kp] = np;
                    M[row + (long long)R.q * kp] = nq;
                }
            }
            grid_barrier(bar, bar + 1, nblocks);
            // C: rows p, q of G: G <- J^H G, and the annihilated pair set to zero
            for (long long e = gtid; e < (long long)half * kp; e += nthreads) {
                const long long pair = e / kp;
                const int col = (int)(e % kp);
                const Rot R = rots[pair];
                double2 rp, rq;
                if (col == R.p || col == R.q) {
                    const int cq = col == R.q ? 2 : 0;
                    rp = B4[pair * 4 + cq];
                    rq = B4[pair * 4 + 1 + cq];
                } else {
                    rp = G[R.p + (long long)col * kp];
                    rq = G[R.q + (long long)col * kp];
                }
                // e^{i phi} r_q
                const double2 eq = make_double2(R.er * rq.x - R.ei * rq.y, R.er * rq.y + R.ei * rq.x);
                double2 np = make_double2(R.cs * rp.x - R.sn * eq.x, R.cs * rp.y - R.sn * eq.y);
                double2 nq = make_double2(R.sn * rp.x + R.cs * eq.x, R.sn * rp.y + R.cs * eq.y);
                if (col == R.q) np = make_double2(0.0, 0.0);
                if (col == R.p) nq = make_double2(0.0, 0.0);
                if (col == R.p) np.y = 0.0;  // diagonal stays real
                if (col == R.q) nq.y = 0.0;
                G[R.p + (long long)col * kp] = np;
                G[R.q + (long long)col * kp] = nq;
            }
            grid_barrier(bar, bar + 1, nblocks);
        }
        const double off = __longlong_as_double((long long)*(volatile unsigned long long *)flag);
        grid_barrier(bar, bar + 1, nblocks);  // everybody has read this sweep's flag
        if (gtid == 0) flags[(sweep + 1) & 1] = 0ull;
        grid_barrier(bar, bar + 1, nblocks);
        if (off < 1e-15) {
            sweep++;
            break;
        }
    }
    if (gtid == 0) *sweeps_out = sweep;
}

// ------------------------------------------------------------------ block Jacobi
// Two-sided block Jacobi on the Hermitian G (kp x kp, kp a multiple of 2 kJB): the index set
// is cut into nb = kp / kJB blocks paired by the round-robin tournament (nb - 1 rounds per
// sweep, nb / 2 block pairs per round).  Per round, in one cooperative grid:
//   P1  one CTA per block pair (I, J): A = G[I u J, I u J] (32 x 32) into shared memory, one
//       cyclic 2 x 2 Jacobi sweep on A (the same rotation formulas as k_jacobi) accumulating
//       U = J_1 J_2 ...; U to a scratch; the max off-diagonal ratio of A before the sweep
//       feeds the convergence flag;
//   P2  G[:, I u J] <- G[:, I u J] U and V[:, I u J] <- V[:, I u J] U (one warp per row);
//   P3  G[I u J, :] <- U^H G[I u J, :] (one warp per column), diagonal made real;
// with a grid barrier after each phase: 3 (nb - 1) barriers per sweep instead of 2 (kp - 1).
constexpr int kJB = 16;        // block size
constexpr int kJL = 2 * kJB;   // local problem size (one warp wide)

__device__ __forceinline__ int blk_idx(int I, int J, int a) { return a < kJB ? I * kJB + a : J * kJB + (a - kJB); }

constexpr int kBjThreads = 1024;  // 32 warps per SM: P2/P3 are latency-bound row/column passes
constexpr int kJLoc = (kJL / 2) * (kJL / 2);   // threads of a local round: one per 2 x 2 block

// Rotation of the local problem's pair (p, q): a = A_pp, b = A_qq (real), c = A_pq.  The
// classical formulas (tau = (b - a) / 2|c|, t = sgn(tau) / (|tau| + sqrt(1 + tau^2)),
// cs = 1 / sqrt(1 + t^2), sn = t cs, e = c / |c|) evaluated with three reciprocal square roots
// instead of a chain of square roots and divisions: with r1 = 1 / sqrt(1 + tau^2),
// cos 2theta = |tau| r1 and sin 2theta = sgn(tau) r1, and the half-angle forms give
// cs = sqrt(h), sn = sin 2theta / (2 sqrt(h)), h = (1 + cos 2theta) / 2 in [1/2, 1] (no
// cancellation).  Each result is within a few ulps of the classical one, which is all the
// Jacobi iteration needs (a rotation orthogonal to working precision); the reconstruction is
// checked against the oracle to a tolerance, not bit for bit (R30).
__device__ __forceinline__ Rot rot_params(double a, double b, double2 c, int p, int q) {
    Rot R;
    R.p = p;
    R.q = q;
    const double ac2 = fma(c.x, c.x, c.y * c.y);
    if (ac2 == 0.0) {
        R.cs = 1.0;
        R.sn = 0.0;
        R.er = 1.0;
        R.ei = 0.0;
        return R;
    }
    const double ri = rsqrt(ac2);                 // 1 / |c|
    R.er = c.x * ri;
    R.ei = c.y * ri;
    const double tau = 0.5 * (b - a) * ri;
    if (fabs(tau) > 1e150) {                      // negligible rotation: theta = 1 / (2 tau)
        R.cs = 1.0;
        R.sn = 0.5 / tau;
        return R;
    }
    const double r1 = rsqrt(fma(tau, tau, 1.0));
    const double h = 0.5 * fma(fabs(tau), r1, 1.0);
    const double rh = rsqrt(h);
    R.cs = h * rh;
    R.sn = (tau >= 0.0 ? r1 : -r1) * 0.5 * rh;
    return R;
}

__global__ void __launch_bounds__(kBjThreads) k_bjacobi(double2 *G, double2 *V, int kp, double2 *Us,
                                                 unsigned long long *flags, int *sweeps_out,
                                                 unsigned long long *trace, int merged) {
    extern __shared__ double2 bj_dyn[];   // merged phase: V, U_p and T tiles (3 x 32 x 33)
    __shared__ double2 A[kJL][kJL + 1];   // A[row][col]
    __shared__ double2 U[kJL][kJL + 1];
    __shared__ Rot srot[kJL / 2];
    unsigned *bar = reinterpret_cast<unsigned *>(flags + 2);
    const unsigned nblocks = gridDim.x;
    const int nb = kp / kJB, npairs = nb / 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int sweep = 0;
    for (; sweep < 40; sweep++) {
        unsigned long long *flag = &flags[sweep & 1];
        for (int r = 0; r < nb - 1; r++) {
            const bool trc = trace && sweep == 0 && r < 8 && blockIdx.x == 0;  // CTA 0 (uniform)
            const bool tr = trc && tid == 0;
            if (tr) trace[r * 4 + 0] = globaltimer_ns();
            // ---- P1: local problems
            for (int pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
                int I, J;
                round_pair(r, pr, nb, I, J);
                for (int e = tid; e < kJL * kJL; e += blockDim.x) {
                    const int a = e % kJL, b = e / kJL;
                    A[a][b] = G[blk_idx(I, J, a) + (long long)blk_idx(I, J, b) * kp];
                    U[a][b] = make_double2(a == b ? 1.0 : 0.0, 0.0);
                }
                __syncthreads();
                {  // convergence measure: the CTA's largest ratio, one atomic per CTA
                    double mx = 0.0;   // ratios are >= 0: their bit patterns order as the values
                    for (int e = tid; e < kJL * kJL; e += blockDim.x) {
                        const int a = e % kJL, b = e / kJL;
                        if (a < b) {
                            const double2 c = A[a][b];
                            const double ac = sqrt(c.x * c.x + c.y * c.y);
                            if (ac > 0.0) {
                                const double den = sqrt(fabs(A[a][a].x * A[b][b].x));
                                mx = fmax(mx, den > 0.0 ? ac / den : 1.0);
                            }
                        }
                    }
#pragma unroll
                    for (int h = 16; h > 0; h >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, h));
                    if (lane == 0 && mx > 0.0) atomicMax(flag, dbits(mx));
                }
                // the local rounds run on the first 256 threads only (one per 2 x 2 block of the
                // update), synchronised by a named barrier: cheaper than a 1,024-thread barrier
                if (trc && pr == 0) {
                    __syncthreads();
                    if (tid == 0) trace[64 + r * 4] = globaltimer_ns();
                }
                if (tid < kJLoc)
                for (int lr = 0; lr < kJL - 1; lr++) {
                    if (tid < kJL / 2) {
                        int p, q;
                        round_pair(lr, tid, kJL, p, q);
                        srot[tid] = rot_params(A[p][p].x, A[q][q].x, A[p][q], p, q);
                    }
                    asm volatile("bar.sync 1, %0;" ::"r"(kJLoc) : "memory");
                    // A <- J^H A J and U <- U J, fused: the rotation pairs partition the indices,
                    // so thread (i, j) owns the 2 x 2 blocks (rows of pair i, columns of pair j)
                    // of A and U -- it reads all four entries before writing them and no other
                    // thread touches them (same per-element operations as column-then-row
                    // passes; one barrier per local round instead of two)
                    for (int e = tid; e < (kJL / 2) * (kJL / 2); e += blockDim.x) {
                        const Rot Ri = srot[e / (kJL / 2)], Rj = srot[e % (kJL / 2)];
                        const int rows[2] = {Ri.p, Ri.q}, cols[2] = {Rj.p, Rj.q};
                        double2 a[2][2];
#pragma unroll
                        for (int x = 0; x < 2; x++) {  // columns: [a_p, a_q] <- [a_p, a_q] J_j
                            const double2 gp = A[rows[x]][Rj.p], gq = A[rows[x]][Rj.q];
                            const double2 eq = make_double2(Rj.er * gq.x + Rj.ei * gq.y, Rj.er * gq.y - Rj.ei * gq.x);
                            a[x][0] = make_double2(Rj.cs * gp.x - Rj.sn * eq.x, Rj.cs * gp.y - Rj.sn * eq.y);
                            a[x][1] = make_double2(Rj.sn * gp.x + Rj.cs * eq.x, Rj.sn * gp.y + Rj.cs * eq.y);
                            const double2 up = U[rows[x]][Rj.p], uq = U[rows[x]][Rj.q];
                            const double2 fq = make_double2(Rj.er * uq.x + Rj.ei * uq.y, Rj.er * uq.y - Rj.ei * uq.x);
                            U[rows[x]][Rj.p] = make_double2(Rj.cs * up.x - Rj.sn * fq.x, Rj.cs * up.y - Rj.sn * fq.y);
                            U[rows[x]][Rj.q] = make_double2(Rj.sn * up.x + Rj.cs * fq.x, Rj.sn * up.y + Rj.cs * fq.y);
                        }
#pragma unroll
                        for (int y = 0; y < 2; y++) {  // rows: [a_p; a_q] <- J_i^H [a_p; a_q]
                            const int col = cols[y];
                            const double2 rp = a[0][y], rq = a[1][y];
                            const double2 eq = make_double2(Ri.er * rq.x - Ri.ei * rq.y, Ri.er * rq.y + Ri.ei * rq.x);
                            double2 np = make_double2(Ri.cs * rp.x - Ri.sn * eq.x, Ri.cs * rp.y - Ri.sn * eq.y);
                            double2 nq = make_double2(Ri.sn * rp.x + Ri.cs * eq.x, Ri.sn * rp.y + Ri.cs * eq.y);
                            if (col == Ri.q) np = make_double2(0.0, 0.0);
                            if (col == Ri.p) nq = make_double2(0.0, 0.0);
                            if (col == Ri.p) np.y = 0.0;
                            if (col == Ri.q) nq.y = 0.0;
                            A[Ri.p][col] = np;
                            A[Ri.q][col] = nq;
                        }
                    }
                    asm volatile("bar.sync 1, %0;" ::"r"(kJLoc) : "memory");
                }
                __syncthreads();
                if (tr && pr == 0) trace[64 + r * 4 + 1] = globaltimer_ns();
                double2 *Up = Us + (size_t)pr * kJL * kJL;   // column-major 32 x 32
                for (int e = tid; e < kJL * kJL; e += blockDim.x) Up[e] = U[e % kJL][e / kJL];
                __syncthreads();
                if (tr && pr == 0) trace[64 + r * 4 + 2] = globaltimer_ns();
            }
            grid_barrier(bar, bar + 1, nblocks);
            if (tr) trace[r * 4 + 1] = globaltimer_ns();
            if (merged) {
                // ---- P2+P3 merged: every 32 x 32 tile (rows of pair p, columns of pair q) of the
                // two-sided update depends only on its own old entries and two local rotations,
                // G_pq <- U_p^H (G_pq U_q) and V_pq <- V_pq U_q, so one grid phase and one barrier
                // replace the column pass, its barrier and the row pass (the products associate
                // differently: tolerance parity, as the rest of the eigen-step)
                double2(*Vt)[kJL + 1] = reinterpret_cast<double2(*)[kJL + 1]>(bj_dyn);
                double2(*Up)[kJL + 1] = Vt + kJL;
                double2(*Tt)[kJL + 1] = Up + kJL;
                const int ta = tid >> 5, tb = tid & 31;   // output element (ta, tb) of the tile
                const int ea = tid & 31, eb = tid >> 5;   // staging element (ea, eb): rows contiguous
                // work items: the nG tiles p <= q of the Hermitian G (two products each; the (q, p)
                // tile is written as the conjugate transpose, so G stays exactly Hermitian) and
                // the nV tiles of V (one product each).  With more CTAs than G tiles, CTA b < nG
                // takes G tile b and the others share the V tiles, so no CTA does more than two
                // products (three when every CTA did G_pq and V_pq of one tile)
                const int nG = npairs * (npairs + 1) / 2, nV = npairs * npairs;
                const int G_ctas = (int)gridDim.x > nG ? nG : 0;   // 0: one grid-stride list
                auto tile_pq = [&](int g, int &p, int &q) {          // g-th pair p <= q, row-major
                    p = 0;
                    while (g >= npairs - p) {
                        g -= npairs - p;
                        p++;
                    }
                    q = p + g;
                };
                const int first = G_ctas ? ((int)blockIdx.x < nG ? (int)blockIdx.x : nG + (int)blockIdx.x - nG)
                                         : (int)blockIdx.x;
                const int stride = G_ctas ? ((int)blockIdx.x < nG ? nG + nV : (int)gridDim.x - nG) : (int)gridDim.x;
                for (int t = first; t < nG + nV; t += stride) {
                    const bool gtile = t < nG;
                    int p, q;
                    if (gtile) tile_pq(t, p, q);
                    else {
                        p = (t - nG) / npairs;
                        q = (t - nG) % npairs;
                    }
                    int I, J, K, L;
                    round_pair(r, p, nb, I, J);
                    round_pair(r, q, nb, K, L);
                    // coalesced staging: consecutive threads take consecutive rows of a column
                    const long long sa = blk_idx(I, J, ea), sb = blk_idx(K, L, eb);
                    if (gtile) {
                        A[ea][eb] = G[sa + sb * kp];
                        Up[ea][eb] = Us[(size_t)p * kJL * kJL + tid];     // U_p[ea][eb] (column-major)
                    } else {
                        Vt[ea][eb] = V[sa + sb * kp];
                    }
                    U[ea][eb] = Us[(size_t)q * kJL * kJL + tid];          // U_q[ea][eb]
                    __syncthreads();
                    double2 acc = make_double2(0.0, 0.0);
                    if (gtile) {
#pragma unroll 8
                        for (int m = 0; m < kJL; m++) {   // (G U_q)[ta][tb]
                            const double2 uu = U[m][tb], g = A[ta][m];
                            acc.x = fma(g.x, uu.x, acc.x);
                            acc.x = fma(-g.y, uu.y, acc.x);
                            acc.y = fma(g.x, uu.y, acc.y);
                            acc.y = fma(g.y, uu.x, acc.y);
                        }
                        Tt[ta][tb] = acc;
                        __syncthreads();
                        acc = make_double2(0.0, 0.0);
#pragma unroll 8
                        for (int m = 0; m < kJL; m++) {   // (U_p^H T)[ta][tb] = sum_m conj(U_p[m][ta]) T[m][tb]
                            const double2 uu = Up[m][ta], y = Tt[m][tb];
                            acc.x = fma(uu.x, y.x, acc.x);
                            acc.x = fma(uu.y, y.y, acc.x);
                            acc.y = fma(uu.x, y.y, acc.y);
                            acc.y = fma(-uu.y, y.x, acc.y);
                        }
                        if (blk_idx(I, J, ta) == blk_idx(K, L, tb)) acc.y = 0.0;  // Hermitian: real diagonal
                        __syncthreads();   // A fully read before it is overwritten
                        A[ta][tb] = acc;
                        __syncthreads();
                        G[sa + sb * kp] = A[ea][eb];   // coalesced write-back
                        if (p != q) {                  // G_qp = G_pq^H
                            const double2 x = A[eb][ea];
                            G[blk_idx(K, L, ea) + blk_idx(I, J, eb) * kp] = make_double2(x.x, -x.y);
                        }
                    } else {
#pragma unroll 8
                        for (int m = 0; m < kJL; m++) {   // (V U_q)[ta][tb]
                            const double2 uu = U[m][tb], v = Vt[ta][m];
                            acc.x = fma(v.x, uu.x, acc.x);
                            acc.x = fma(-v.y, uu.y, acc.x);
                            acc.y = fma(v.x, uu.y, acc.y);
                            acc.y = fma(v.y, uu.x, acc.y);
                        }
                        __syncthreads();
                        Vt[ta][tb] = acc;
                        __syncthreads();
                        V[sa + sb * kp] = Vt[ea][eb];
                    }
                    __syncthreads();   // the tile arrays are refilled for the next item
                }
                grid_barrier(bar, bar + 1, nblocks);
                if (tr) trace[r * 4 + 2] = trace[r * 4 + 3] = globaltimer_ns();
                continue;
            }
            // ---- P2: columns: M[row, I u J] <- M[row, I u J] U.  The grid is cut into npairs
            // groups of CTAs, each group owns one block pair; a CTA stages that pair's U in
            // shared memory (conflict-free U[m][lane] reads) and its warps take rows.
            {
                const int S = (int)gridDim.x / npairs > 0 ? (int)gridDim.x / npairs : 1;
                const int wpc = blockDim.x >> 5;
                for (int u = blockIdx.x; u < npairs * S; u += gridDim.x) {
                    const int pr = u / S, slice = u % S;
                    int I, J;
                    round_pair(r, pr, nb, I, J);
                    const double2 *Up = Us + (size_t)pr * kJL * kJL;
                    for (int e = tid; e < kJL * kJL; e += blockDim.x) U[e % kJL][e / kJL] = Up[e];
                    __syncthreads();
                    const long long col = blk_idx(I, J, lane);
                    for (int rit = slice * wpc + warp; rit < 2 * kp; rit += S * wpc) {
                        double2 *M = rit < kp ? G : V;
                        const int row = rit % kp;
                        const double2 x = M[row + col * kp];
                        double2 acc = make_double2(0.0, 0.0);
#pragma unroll 8
                        for (int m = 0; m < kJL; m++) {
                            const double xr = __shfl_sync(0xffffffffu, x.x, m), xi = __shfl_sync(0xffffffffu, x.y, m);
                            const double2 uu = U[m][lane];
                            acc.x = fma(xr, uu.x, acc.x);
                            acc.x = fma(-xi, uu.y, acc.x);
                            acc.y = fma(xr, uu.y, acc.y);
                            acc.y = fma(xi, uu.x, acc.y);
                        }
                        M[row + col * kp] = acc;
                    }
                    __syncthreads();
                }
            }
            grid_barrier(bar, bar + 1, nblocks);
            if (tr) trace[r * 4 + 2] = globaltimer_ns();
            // ---- P3: rows: G[I u J, col] <- U^H G[I u J, col], same grouping, warps take columns
            {
                const int S = (int)gridDim.x / npairs > 0 ? (int)gridDim.x / npairs : 1;
                const int wpc = blockDim.x >> 5;
                for (int u = blockIdx.x; u < npairs * S; u += gridDim.x) {
                    const int pr = u / S, slice = u % S;
                    int I, J;
                    round_pair(r, pr, nb, I, J);
                    const double2 *Up = Us + (size_t)pr * kJL * kJL;
                    for (int e = tid; e < kJL * kJL; e += blockDim.x) U[e % kJL][e / kJL] = Up[e];
                    __syncthreads();
                    const long long row = blk_idx(I, J, lane);
                    for (int col = slice * wpc + warp; col < kp; col += S * wpc) {
                        const double2 y = G[row + (long long)col * kp];
                        double2 acc = make_double2(0.0, 0.0);
#pragma unroll 8
                        for (int m = 0; m < kJL; m++) {
                            const double yr = __shfl_sync(0xffffffffu, y.x, m), yi = __shfl_sync(0xffffffffu, y.y, m);
                            const double2 uu = U[m][lane];   // conj(U[m][lane]) y_m
                            acc.x = fma(uu.x, yr, acc.x);
                            acc.x = fma(uu.y, yi, acc.x);
                            acc.y = fma(uu.x, yi, acc.y);
                            acc.y = fma(-uu.y, yr, acc.y);
                        }
                        if (row == col) acc.y = 0.0;  // Hermitian: real diagonal
                        G[row + (long long)col * kp] = acc;
                    }
                    __syncthreads();
                }
            }
            grid_barrier(bar, bar + 1, nblocks);
            if (tr) trace[r * 4 + 3] = globaltimer_ns();
        }
        const double off = __longlong_as_double((long long)*(volatile unsigned long long *)flag);
        if (trace && blockIdx.x == 0 && tid == 0 && sweep < 32) trace[32 + sweep] = dbits(off);
        grid_barrier(bar, bar + 1, nblocks);
        if (blockIdx.x == 0 && tid == 0) flags[(sweep + 1) & 1] = 0ull;
        grid_barrier(bar, bar + 1, nblocks);
        if (off < 1e-15) {
            sweep++;
            break;
        }
    }
    if (blockIdx.x == 0 && tid == 0) *sweeps_out = sweep;
}

int jacobi_pad(int k) {  // kp for the block Jacobi: a multiple of 2 kJB
    return (k + kJL - 1) / kJL * kJL;
}

size_t bjacobi_scratch_bytes(int kp) { return sizeof(double2) * (size_t)(kp / kJL) * kJL * kJL; }

cudaError_t launch_bjacobi(double2 *G, double2 *V, int kp, double2 *Us, unsigned long long *flags, int *sweeps,
                           int num_sms, cudaStream_t s, unsigned long long *trace) {
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bjacobi, kBjThreads, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    int grid = num_sms;
    // RBG_JACOBI_SPLIT=1: the separate column and row passes (two barriers) instead of the
    // merged tile update (one)
    static const bool split = getenv("RBG_JACOBI_SPLIT") != nullptr;
    int merged = split ? 0 : 1;
    const size_t dyn = merged ? (size_t)3 * kJL * (kJL + 1) * sizeof(double2) : 0;
    if (dyn) {
        e = cudaFuncSetAttribute(k_bjacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bjacobi, kBjThreads, dyn);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    }
    void *args[] = {&G, &V, &kp, &Us, &flags, &sweeps, &trace, &merged};
    return cudaLaunchCooperativeKernel((void *)k_bjacobi, grid, kBjThreads, args, dyn, s);
}

// X(:, r) = Q V(:, order[r]) for r < kr: X is N_v x kr vectors (column stride ldx_v), Q is
// k columns of nvec vectors (stride ldq_v); each element a sequential sum over i.
template <bool CPLX>
__global__ void k_recon_x(const double2 *Q, long long ldq_v, long long nvec, int k, const double2 *V, int kp,
                          const int *order, int kr, double2 *X, long long ldx_v) {
    const long long total = nvec * kr;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long u = e % nvec;
        const int r = (int)(e / nvec);
        const double2 *v = V + (long long)order[r] * kp;
        double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
        for (int i = 0; i < k; i++) {
            const double2 q = Q[(long long)i * ldq_v + u];
            const double2 c = v[i];
            if (CPLX) {  // q * c
                acc.x = fma(q.x, c.x, acc.x);
                acc.x = fma(-q.y, c.y, acc.x);
                acc.y = fma(q.x, c.y, acc.y);
                acc.y = fma(q.y, c.x, acc.y);
            } else {     // two real rows per vector, real eigenvector entries
                acc.x = fma(q.x, c.x, acc.x);
                acc2.x = fma(q.y, c.x, acc2.x);
            }
        }
        X[(long long)r * ldx_v + u] = CPLX ? acc : make_double2(acc.x, acc2.x);
    }
}

// Eigenvalues (diag of the converged G) in descending order, ties by index; sigma =
// sqrt(max(lambda, 0)); kr = #{sigma > tau2} capped at kr_max (Algorithm 4 step 6).
// Eigenvalues (the converged diagonal of G) in descending order, ties by index, as a rank
// sort: element i goes to position #{j : l_j > l_i or (l_j == l_i and j < i)}; sigma = sqrt of
// the clamped values; kr = length of the prefix with sigma > tau2, capped at kr_max.
__global__ void __launch_bounds__(1024) k_eig_sort(const double2 *G, int k, int kp, double tau2, int kr_max,
                                                   int *order, double *sigma, int *kr) {
    __shared__ int s_first;  // first position with sigma <= tau2
    if (threadIdx.x == 0) s_first = k;
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        const double li = G[i + (long long)i * kp].x;
        int r = 0;
        for (int j = 0; j < k; j++) {
            const double lj = G[j + (long long)j * kp].x;
            r += (lj > li || (lj == li && j < i)) ? 1 : 0;
        }
        order[r] = i;
        const double sg = sqrt(fmax(li, 0.0));
        sigma[r] = sg;
        if (!(sg > tau2)) atomicMin(&s_first, r);
    }
    __syncthreads();
    if (threadIdx.x == 0) *kr = s_first < kr_max ? s_first : kr_max;
}

cudaError_t launch_eig_sort(const double2 *G, int k, int kp, double tau2, int kr_max, int *order, double *sigma,
                            int *kr, cudaStream_t s) {
    k_eig_sort<<<1, 1024, 0, s>>>(G, k, kp, tau2, kr_max, order, sigma, kr);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ host launchers
cudaError_t launch_gram(const double *R, long long ldr, int k, long long M, bool cplx, double2 *P, long long chunk,
                        const int4 *items_d, int nitems, cudaStream_t s) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    // R as a 2D array of doubles: M (x 2 complex) columns x k rows, row pitch ldr elements;
    // boxes of 16 doubles (128 bytes) x 64 rows, 128-byte swizzle, out-of-range rows / columns 0.
    // A tensor map needs a 16-byte row pitch: a real R with odd ldr is first copied to even.
    const int xs = cplx ? 2 : 1;
    double *Rp = nullptr;
    if ((ldr * xs * 8) % 16 != 0) {
        const long long ldp = ldr + 1;
        cudaError_t e = dmalloc(&Rp, (size_t)k * ldp * 8);
        if (e == cudaSuccess) e = cudaMemcpy2DAsync(Rp, (size_t)ldp * 8, R, (size_t)ldr * 8, (size_t)M * 8, k,
                                                    cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) {
            dfree(Rp);
            return e;
        }
        R = Rp;
        ldr = ldp;
    }
    CUtensorMap tm;
    const cuuint64_t dims[2] = {(cuuint64_t)(M * xs), (cuuint64_t)k};
    const cuuint64_t strides[1] = {(cuuint64_t)ldr * xs * 8};
    const cuuint32_t box[2] = {16, 64};
    const cuuint32_t estr[2] = {1, 1};
    cudaError_t e = cudaSuccess;
    if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(R), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        e = cudaErrorInvalidValue;
    auto kern = cplx ? k_gram<true> : k_gram<false>;
    const size_t smem = (size_t)kGStages * 2 * xs * kGBox + 1024;
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) {
        kern<<<nitems, 256 + 32, smem, s>>>(tm, k, M, chunk, items_d, P);
        e = cudaGetLastError();
    }
    if (Rp) {  // the caller synchronises before freeing its own buffers; so do we here
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        dfree(Rp);
    }
    return e;
}

cudaError_t launch_gram_reduce(const double2 *P, long long nchunks, int k, int kp, const double2 *G0, double2 *G,
                               cudaStream_t s) {
    const long long n = (long long)kp * kp;
    k_gram_reduce<<<(unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, s>>>(P, nchunks, k, kp, G0, G);
    return cudaGetLastError();
}

cudaError_t launch_jacobi(double2 *G, double2 *V, int kp, Rot *rots, unsigned long long *flags, int *sweeps,
                          int num_sms, cudaStream_t s) {
    const size_t smem = rot_bytes(kp);
    cudaError_t e = cudaSuccess;
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi, 256, smem);
    if (e != cudaSuccess) return e;
    // one block per SM at most: the per-round work is small and the barrier cost grows with
    // the number of arriving blocks
    const int want = (kp * kp + 255) / 256;
    int grid = (per_sm > 0 ? 1 : 0) * num_sms;
    if (grid > want) grid = want;
    if (grid < 1) grid = 1;
    void *args[] = {&G, &V, &kp, &rots, &flags, &sweeps};
    return cudaLaunchCooperativeKernel((void *)k_jacobi, grid, 256, args, smem, s);
}

cudaError_t launch_recon_x(const double2 *Q, long long ldq_v, long long nvec, int k, const double2 *V, int kp,
                           const int *order, int kr, double2 *X, long long ldx_v, bool cplx, cudaStream_t s) {
    const long long n = nvec * kr;
    const unsigned blocks = (unsigned)((n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192);
    if (cplx) k_recon_x<true><<<blocks ? blocks : 1, 256, 0, s>>>(Q, ldq_v, nvec, k, V, kp, order, kr, X, ldx_v);
    else k_recon_x<false><<<blocks ? blocks : 1, 256, 0, s>>>(Q, ldq_v, nvec, k, V, kp, order, kr, X, ldx_v);
    return cudaGetLastError();
}

size_t rot_bytes(int kp) { return sizeof(Rot) * (size_t)(kp / 2); }
size_t jacobi_scratch_bytes(int kp) { return 4 * sizeof(double2) * (size_t)(kp / 2); }

}  // namespace rbg
