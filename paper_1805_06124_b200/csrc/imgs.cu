// imgs.cu -- pivot decision + iterated modified Gram-Schmidt (the orthogonalisation half).
//
// PAPER.md:871-883 (Sec. 6.1.2): "the newly selected pivot column is orthogonalized with
// respect to the existing basis set ... We use the iterative modified Gram-Schmidt (IMGS)
// algorithm of Hoffman (MGSCI with kappa = 2)".  Cost O(nu_j j N) with nu_j < 3 typically.
// Acceptance test, sweep cap and degeneracy threshold: DESIGN.md reading R7.
//
// B200 design: the method is a chain of 2*nu*k dependent
// reductions of length N, so the kernel is latency-bound.  It runs as ONE thread-block
// cluster of 8 CTAs x 256 threads (L_I = 2048 lanes); the candidate vector v lives in
// registers (vector u on lane u mod 2048); each MGS step is a lane-local fma chain, a
// warp xor-butterfly, an all-to-all of the 64 warp partials through distributed shared
// memory (st.async + mbarrier transaction counts, no CTA or cluster barrier) and a
// 64-leaf tree evaluated by every warp, after which every CTA holds the bit-identical
// coefficient and updates its slice of v.  The next step's basis vectors are loaded
// (L2 evict-last) before the reduction so their latency overlaps it.  The kernel is
// replicated on every GPU of a sharded run (no broadcast of q needed).
#include <cmath>

#include "kernels.h"

namespace rbg {

// Sum over the 2048 lanes with the balanced pairwise tree of CAC rule 3.
//  1. xor-butterfly in the warp (offsets 1..16): every lane holds its warp's partial;
//  2. lanes 0..7 of warp w of CTA r st.async the partial into slot 8r+w of CTA 0..7's
//     shared memory, each store counted (16 B) on the receiving CTA's mbarrier;
//  3. every warp waits for its CTA's 64 slots (1024 B), then lane l adds slots 2l, 2l+1 and
//     an xor-butterfly over the lanes finishes the tree over the 64 (CTA, warp) leaves.
// No CTA or cluster barrier is needed; every warp of every CTA ends with the same bits.
// Slots and mbarriers are double-buffered by reduction parity: a CTA can only receive the
// data of reduction n+2 after all of its own warps have sent reduction n+1, i.e. after
// they finished reading the buffers of reduction n.
struct ClusterReducer {
    double2 (*slots)[64];
    uint64_t *bars;
    uint32_t rank;
    int warp, lane, par;
    uint32_t phase;  // bit p: parity of the next phase to wait for on bars[p]

    __device__ __forceinline__ double2 sum(double re, double im) {
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) {
            re = re + __shfl_xor_sync(0xffffffffu, re, h);
            im = im + __shfl_xor_sync(0xffffffffu, im, h);
        }
        if (lane < kImgsCtas) {
            const uint32_t dst = map_dsmem(smem_u32(&slots[par][rank * 8 + warp]), (uint32_t)lane);
            const uint32_t bar = map_dsmem(smem_u32(&bars[par]), (uint32_t)lane);
            st_async_v2(dst, re, im, bar);
        }
        mbar_wait_cluster(&bars[par], (phase >> par) & 1u);
        phase ^= 1u << par;
        if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&bars[par], 64 * 16);  // re-arm for n+2
        const double2 a = slots[par][2 * lane], b = slots[par][2 * lane + 1];
        double x = a.x + b.x, y = a.y + b.y;
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) {
            x = x + __shfl_xor_sync(0xffffffffu, x, h);
            y = y + __shfl_xor_sync(0xffffffffu, y, h);
        }
        par ^= 1;
        return make_double2(x, y);
    }
};

template <bool CPLX, int MAXV>
__device__ __forceinline__ double nrm_partial(const double2 (&v)[MAXV], const double *w, long long lane_g,
                                              long long nvec) {
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < MAXV; m++) {
        const long long u = lane_g + (long long)m * kLaneImgs;
        if (u < nvec) {  // CAC rule 4
            if (CPLX) {
                const double wu = w[u];
                double t = wu * v[m].x;
                acc = fma(t, v[m].x, acc);
                t = wu * v[m].y;
                acc = fma(t, v[m].y, acc);
            } else {
                double t = w[2 * u] * v[m].x;
                acc = fma(t, v[m].x, acc);
                t = w[2 * u + 1] * v[m].y;
                acc = fma(t, v[m].y, acc);
            }
        }
    }
    return acc;
}

template <bool CPLX, int MAXV>
__global__ void __cluster_dims__(kImgsCtas, 1, 1) __launch_bounds__(kImgsThreads, 1)
    k_imgs(const ImgsArgs a) {
    __shared__ double2 s_slots[2][64];
    __shared__ __align__(8) uint64_t s_bars[2];

    const int stop0 = a.st->stop;
    if (stop0) return;
    const long long k = a.st->k;
    const uint32_t rank = cluster_ctarank();
    const int tid = threadIdx.x;
    const long long lane_g = (long long)rank * kImgsThreads + tid;
    const long long nvec = a.nvec;
    const bool odd_tail = !CPLX && (a.N & 1);

    // ---- a3: pivot decision (identical in every CTA and on every rank) ------------------
    double m;
    long long J;
    int owner = 0;
    if (a.world == 1) {
        m = a.st->m_loc;
        J = a.st->j_loc;
    } else {
        m = -INFINITY;
        J = 0x7fffffffffffffffLL;
        for (int p = 0; p < a.world; p++) {
            const Rec *r = reinterpret_cast<const Rec *>(a.recv + (size_t)p * a.slot_bytes);
            if (rec_better(r->m, r->j, m, J)) {
                m = r->m;
                J = r->j;
                owner = p;
            }
        }
    }
    const double err = sqrt(fmax(m, 0.0));  // CAC rule 8
    int why = kStopNone;
    if (m == -INFINITY) why = kStopAll;
    else if (err < a.tol) why = kStopTol;
    else if (k == a.k_max) why = kStopKmax;

    if (tid == 0) {
        mbar_init(&s_bars[0], 1);
        mbar_init(&s_bars[1], 1);
        mbar_arrive_expect_tx(&s_bars[0], 64 * 16);
        mbar_arrive_expect_tx(&s_bars[1], 64 * 16);
    }
    // every CTA has read the state before rank 0 changes it, and every CTA's mbarriers are
    // initialised before any remote st.async can target them
    cluster_sync_all();
    const bool leader = (rank == 0 && tid == 0);
    if (leader) a.errors[k] = err;
    if (why != kStopNone) {
        if (leader) a.st->stop = why;
        return;
    }

    // ---- a5: Hoffmann IMGS (CAC rule 9) ---------------------------------------------
    const double2 *src = (a.world == 1)
                             ? a.S + (J - a.col_offset) * a.ldv
                             : reinterpret_cast<const double2 *>(a.recv + (size_t)owner * a.slot_bytes +
                                                                 sizeof(Rec));
    double2 v[MAXV];
#pragma unroll
    for (int mm = 0; mm < MAXV; mm++) {
        const long long u = lane_g + (long long)mm * kLaneImgs;
        v[mm] = (u < nvec) ? src[u] : make_double2(0.0, 0.0);
        if (odd_tail && u == nvec - 1) v[mm].y = 0.0;
    }

    ClusterReducer red{s_slots, s_bars, rank, tid >> 5, tid & 31, 0, 0u};
    const uint64_t keep = policy_evict_last();
    const double n0 = sqrt(red.sum(nrm_partial<CPLX, MAXV>(v, a.w, lane_g, nvec), 0.0).x);
    double n_prev = n0, nn = 0.0;
    int nu = 0;
    bool accepted = false;
    while (nu < kNuMax) {
        nu++;
        // prefetch basis vector 0
        double2 wq[MAXV], q[MAXV];
        if (k > 0) {
#pragma unroll
            for (int mm = 0; mm < MAXV; mm++) {
                const long long u = lane_g + (long long)mm * kLaneImgs;
                wq[mm] = (u < nvec) ? ld_keep(a.WQ + u, keep) : make_double2(0.0, 0.0);
                q[mm] = (u < nvec) ? ld_keep(a.Q + u, keep) : make_double2(0.0, 0.0);
            }
        }
        for (long long i = 0; i < k; i++) {
            double pr = 0.0, pi = 0.0;
#pragma unroll
            for (int mm = 0; mm < MAXV; mm++) {
                const long long u = lane_g + (long long)mm * kLaneImgs;
                if (u < nvec) {  // DOT(WQ_i, v), CAC rule 2
                    if (CPLX) {
                        pr = fma(wq[mm].x, v[mm].x, pr);
                        pr = fma(wq[mm].y, v[mm].y, pr);
                        pi = fma(wq[mm].x, v[mm].y, pi);
                        pi = fma(-wq[mm].y, v[mm].x, pi);
                    } else {
                        pr = fma(wq[mm].x, v[mm].x, pr);
                        pr = fma(wq[mm].y, v[mm].y, pr);
                    }
                }
            }
            // next basis vector's loads overlap the cluster reduction
            double2 wq_n[MAXV], q_n[MAXV];
            if (i + 1 < k) {
                const double2 *wqp = a.WQ + (i + 1) * a.ldq_v;
                const double2 *qp = a.Q + (i + 1) * a.ldq_v;
#pragma unroll
                for (int mm = 0; mm < MAXV; mm++) {
                    const long long u = lane_g + (long long)mm * kLaneImgs;
                    wq_n[mm] = (u < nvec) ? ld_keep(wqp + u, keep) : make_double2(0.0, 0.0);
                    q_n[mm] = (u < nvec) ? ld_keep(qp + u, keep) : make_double2(0.0, 0.0);
                }
            }
            const double2 c = red.sum(pr, pi);
#pragma unroll
            for (int mm = 0; mm < MAXV; mm++) {
                const long long u = lane_g + (long long)mm * kLaneImgs;
                if (u < nvec) {  // v <- v - c q_i
                    if (CPLX) {
                        double vr = v[mm].x, vi = v[mm].y;
                        vr = fma(-c.x, q[mm].x, vr);
                        vr = fma(c.y, q[mm].y, vr);
                        vi = fma(-c.x, q[mm].y, vi);
                        vi = fma(-c.y, q[mm].x, vi);
                        v[mm] = make_double2(vr, vi);
                    } else {
                        v[mm].x = fma(-c.x, q[mm].x, v[mm].x);
                        v[mm].y = fma(-c.x, q[mm].y, v[mm].y);
                    }
                }
            }
            if (i + 1 < k) {
#pragma unroll
                for (int mm = 0; mm < MAXV; mm++) {
                    wq[mm] = wq_n[mm];
                    q[mm] = q_n[mm];
                }
            }
        }
        nn = sqrt(red.sum(nrm_partial<CPLX, MAXV>(v, a.w, lane_g, nvec), 0.0).x);
        if (nn > n_prev / 2.0) {  // Hoffmann's test with kappa = 2
            accepted = true;
            break;
        }
        n_prev = nn;
    }
    const double delta = 1000.0 * 0x1p-52;
    if (!accepted || !(nn >= delta * n0) || nn == 0.0) {
        if (leader) {
            a.nu[k] = nu;
            a.st->stop = kStopRank;
        }
        return;
    }

    // ---- q_{k+1} = v / n, w o q_{k+1}; a6 bookkeeping -------------------------------
    double2 *qo = a.Q + k * a.ldq_v;
    double2 *wqo = a.WQ + k * a.ldq_v;
#pragma unroll
    for (int mm = 0; mm < MAXV; mm++) {
        const long long u = lane_g + (long long)mm * kLaneImgs;
        if (u < nvec) {
            const double2 qq = make_double2(v[mm].x / nn, v[mm].y / nn);
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
        const long long jl = J - a.col_offset;
        if (jl >= 0 && jl < a.M_loc) a.r2[jl] = -INFINITY;
        a.st->k = k + 1;
    }
}

int imgs_maxv(long long nvec) {
    const long long per = (nvec + kLaneImgs - 1) / kLaneImgs;
    if (per <= 1) return 1;
    if (per <= 2) return 2;
    if (per <= 4) return 4;
    if (per <= 8) return 8;
    if (per <= 16) return 16;
    return 0;
}

template <bool CPLX>
static cudaError_t launch_c(const ImgsArgs &a, cudaStream_t s) {
    switch (imgs_maxv(a.nvec)) {
        case 1: k_imgs<CPLX, 1><<<kImgsCtas, kImgsThreads, 0, s>>>(a); break;
        case 2: k_imgs<CPLX, 2><<<kImgsCtas, kImgsThreads, 0, s>>>(a); break;
        case 4: k_imgs<CPLX, 4><<<kImgsCtas, kImgsThreads, 0, s>>>(a); break;
        case 8: k_imgs<CPLX, 8><<<kImgsCtas, kImgsThreads, 0, s>>>(a); break;
        case 16: k_imgs<CPLX, 16><<<kImgsCtas, kImgsThreads, 0, s>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_imgs(const ImgsArgs &a, bool cplx, cudaStream_t s) {
    return cplx ? launch_c<true>(a, s) : launch_c<false>(a, s);
}

}  // namespace rbg
