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
// warp xor-butterfly, a tree over the 8 warps in shared memory, an all-to-all of the 8
// CTA partials through distributed shared memory and one cluster barrier, after which
// every CTA holds the bit-identical coefficient and updates its slice of v.  The next
// step's basis vectors are loaded before the reduction so the L2 latency overlaps it.
// The kernel is replicated on every GPU of a sharded run (no broadcast of q needed).
#include <cmath>

#include "kernels.h"

namespace rbg {

struct ClusterReducer {
    double2 (*s_warp)[8];
    double2 (*s_cta)[8];
    uint32_t rank;
    int tid, warp, lane, par;

    // Sum over the 2048 lanes with the balanced pairwise tree of CAC rule 3:
    // offsets 1..16 in the warp, 32..128 across the 8 warps, 256..1024 across the 8 CTAs.
    __device__ __forceinline__ double2 sum(double re, double im) {
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) {
            re = re + __shfl_xor_sync(0xffffffffu, re, h);
            im = im + __shfl_xor_sync(0xffffffffu, im, h);
        }
        if (lane == 0) s_warp[par][warp] = make_double2(re, im);
        __syncthreads();
        if (tid < kImgsCtas) {
            const double2 *p = s_warp[par];
            const double a = (p[0].x + p[1].x) + (p[2].x + p[3].x);
            const double b = (p[4].x + p[5].x) + (p[6].x + p[7].x);
            const double c = (p[0].y + p[1].y) + (p[2].y + p[3].y);
            const double d = (p[4].y + p[5].y) + (p[6].y + p[7].y);
            const uint32_t dst = map_dsmem(smem_u32(&s_cta[par][rank]), (uint32_t)tid);
            st_dsmem_v2(dst, a + b, c + d);
        }
        cluster_sync_all();
        const double2 *q = s_cta[par];
        const double x = ((q[0].x + q[1].x) + (q[2].x + q[3].x)) + ((q[4].x + q[5].x) + (q[6].x + q[7].x));
        const double y = ((q[0].y + q[1].y) + (q[2].y + q[3].y)) + ((q[4].y + q[5].y) + (q[6].y + q[7].y));
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
    __shared__ double2 s_warp[2][8];
    __shared__ double2 s_cta[2][8];

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

    cluster_sync_all();  // every CTA has read the state before rank 0 changes it
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

    ClusterReducer red{s_warp, s_cta, rank, tid, tid >> 5, tid & 31, 0};
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
                wq[mm] = (u < nvec) ? a.WQ[u] : make_double2(0.0, 0.0);
                q[mm] = (u < nvec) ? a.Q[u] : make_double2(0.0, 0.0);
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
                    wq_n[mm] = (u < nvec) ? wqp[u] : make_double2(0.0, 0.0);
                    q_n[mm] = (u < nvec) ? qp[u] : make_double2(0.0, 0.0);
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
            qo[u] = qq;
            if (CPLX) {
                const double wu = a.w[u];
                wqo[u] = make_double2(wu * qq.x, wu * qq.y);
            } else {
                wqo[u] = make_double2(a.w[2 * u] * qq.x, a.w[2 * u + 1] * qq.y);
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
