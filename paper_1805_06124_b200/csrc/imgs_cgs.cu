// imgs_cgs.cu -- the orthogonalisation step with Hoffmann's iterated CLASSICAL Gram-Schmidt
// ("CGSCI", kappa = 2), an option next to the paper's MGSCI (the paper points
// to the iterated Gram-Schmidt family of Hoffmann).
//
// MGS needs 2*nu*k dependent length-N reductions per new basis vector; CGS computes all k
// coefficients of a pass at once (c = Q^H W v, then v <- v - Q c), so a pass is two
// grid-wide phases instead of k cluster reductions.  Same acceptance test (n > n_prev / 2,
// nu <= 5, degeneracy n < 1000 * 2^-52 * n0) and the same pivot decision as k_imgs.
//
// Arithmetic contract (DESIGN.md CAC rule 11): every dot and norm uses L_C = 256 lanes (one
// CTA: vector u on lane u mod 256, lane-sequential fma, pairwise tree over the 256 lanes);
// the update of each element runs sequentially over i = 0..k-1 with the rule-9 fma pattern.
// One cooperative launch over the whole GPU; the norms are evaluated redundantly by every
// CTA (identical bits), so only the two phases of a pass need grid barriers.
#include <cooperative_groups.h>

#include <cmath>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace rbg {

constexpr int kCgsThreads = 256;  // L_C

// Sum over the 256 lanes of one CTA: xor-butterfly in the warp, pairwise tree over 8 warps.
__device__ __forceinline__ double2 cta_sum256(double re, double im, double2 *s_w) {
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) {
        re = re + __shfl_xor_sync(0xffffffffu, re, h);
        im = im + __shfl_xor_sync(0xffffffffu, im, h);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();  // s_w free for reuse
    if (lane == 0) s_w[warp] = make_double2(re, im);
    __syncthreads();
    const double x = ((s_w[0].x + s_w[1].x) + (s_w[2].x + s_w[3].x)) + ((s_w[4].x + s_w[5].x) + (s_w[6].x + s_w[7].x));
    const double y = ((s_w[0].y + s_w[1].y) + (s_w[2].y + s_w[3].y)) + ((s_w[4].y + s_w[5].y) + (s_w[6].y + s_w[7].y));
    return make_double2(x, y);
}

// x - c q (CAC rule 9 pattern; real: both components by the real c)
template <bool CPLX>
__device__ __forceinline__ double2 cgs_msub(double2 x, double2 c, double2 q) {
    if (CPLX) {
        x.x = fma(-c.x, q.x, x.x);
        x.x = fma(c.y, q.y, x.x);
        x.y = fma(-c.x, q.y, x.y);
        x.y = fma(-c.y, q.x, x.y);
    } else {
        x.x = fma(-c.x, q.x, x.x);
        x.y = fma(-c.x, q.y, x.y);
    }
    return x;
}

template <bool CPLX>
__device__ __forceinline__ void nrm_acc(double &acc, double2 x, double2 wv) {
    // wv = (w_u, w_u) complex, (w_2u, w_2u+1) real -- CAC rule 4
    double t = wv.x * x.x;
    acc = fma(t, x.x, acc);
    t = wv.y * x.y;
    acc = fma(t, x.y, acc);
}

template <bool CPLX>
__device__ __forceinline__ double2 wvec(const double *w, long long u) {
    if (CPLX) {
        const double wu = w[u];
        return make_double2(wu, wu);
    }
    return reinterpret_cast<const double2 *>(w)[u];
}

template <bool CPLX>
__device__ double nrm256(const double2 *v, const double *w, long long nvec, double2 *s_w) {
    constexpr int U = 8;  // independent loads in flight ahead of the sequential chain
    double acc = 0.0;
    long long u = threadIdx.x;
    for (; u + (U - 1) * kCgsThreads < nvec; u += U * kCgsThreads) {
        double2 x[U], wv[U];
#pragma unroll
        for (int t = 0; t < U; t++) {
            x[t] = v[u + t * kCgsThreads];
            wv[t] = wvec<CPLX>(w, u + t * kCgsThreads);
        }
#pragma unroll
        for (int t = 0; t < U; t++) nrm_acc<CPLX>(acc, x[t], wv[t]);
    }
    for (; u < nvec; u += kCgsThreads) nrm_acc<CPLX>(acc, v[u], wvec<CPLX>(w, u));
    return cta_sum256(acc, 0.0, s_w).x;
}

template <bool CPLX>
__device__ __forceinline__ void dot_acc(double &pr, double &pi, double2 e, double2 x) {
    if (CPLX) {
        pr = fma(e.x, x.x, pr);
        pr = fma(e.y, x.y, pr);
        pi = fma(e.x, x.y, pi);
        pi = fma(-e.y, x.x, pi);
    } else {
        pr = fma(e.x, x.x, pr);
        pr = fma(e.y, x.y, pr);
    }
}

template <bool CPLX>
__device__ double2 dot256(const double2 *wq, const double2 *v, long long nvec, double2 *s_w) {
    constexpr int U = 8;  // independent 16-byte loads in flight per operand
    double pr = 0.0, pi = 0.0;
    long long u = threadIdx.x;
    for (; u + (U - 1) * kCgsThreads < nvec; u += U * kCgsThreads) {  // CAC rule 2, in order
        double2 e[U], x[U];
#pragma unroll
        for (int t = 0; t < U; t++) {
            e[t] = wq[u + t * kCgsThreads];
            x[t] = v[u + t * kCgsThreads];
        }
#pragma unroll
        for (int t = 0; t < U; t++) dot_acc<CPLX>(pr, pi, e[t], x[t]);
    }
    for (; u < nvec; u += kCgsThreads) dot_acc<CPLX>(pr, pi, wq[u], v[u]);
    return cta_sum256(pr, pi, s_w);
}

template <bool CPLX>
__global__ void __launch_bounds__(kCgsThreads) k_imgs_cgs(const ImgsArgs a, double2 *vbuf, double2 *cbuf) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double2 s_w[8];
    const int stop0 = a.st->stop;
    if (stop0) {
        if (threadIdx.x == 0 && blockIdx.x == 0) {
            loop_exit(a.cond, a.use_cond);
            a.st->noop += 1;  // rbg_stats.noop_iters: iterations launched past the stop
        }
        return;
    }
    const long long k = a.st->k;
    const long long nvec = a.nvec;
    const bool odd_tail = !CPLX && (a.N & 1);
    const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;

    // ---- pivot decision (identical in every CTA) ------------------------------------
    double m;
    long long J;
    const double2 *src;
    pivot_decision(a, k, m, J, src);
    const double err = sqrt(fmax(m, 0.0));
    int why = kStopNone;
    if (m == -INFINITY) why = kStopAll;
    else if (err < a.tol) why = kStopTol;
    else if (k == a.k_max) why = kStopKmax;
    grid.sync();  // every CTA has read the state
    const bool leader = (blockIdx.x == 0 && threadIdx.x == 0);
    if (leader) a.errors[k] = err;
    if (why != kStopNone) {
        if (leader) {
            a.st->stop = why;
            loop_exit(a.cond, a.use_cond);
        }
        return;
    }

    for (long long u = gtid; u < nvec; u += nthr) {
        double2 x = a.peer_mine ? ld_cv(src + u) : src[u];
        if (odd_tail && u == nvec - 1) x.y = 0.0;
        vbuf[u] = x;
    }
    grid.sync();
    const double n0 = sqrt(nrm256<CPLX>(vbuf, a.w, nvec, s_w));
    double n_prev = n0, nn = 0.0;
    int nu = 0;
    bool accepted = false;
    while (nu < kNuMax) {
        nu++;
        // c_i = <q_i, v>_w for every i (one CTA per coefficient)
        for (long long i = blockIdx.x; i < k; i += gridDim.x) {
            const double2 c = dot256<CPLX>(a.WQ + i * a.ldq_v, vbuf, nvec, s_w);
            if (threadIdx.x == 0) cbuf[i] = c;
        }
        grid.sync();
        // v <- v - Q c, each element sequentially over i
        for (long long u = gtid; u < nvec; u += nthr) {
            double2 x = vbuf[u];
            constexpr int U = 16;  // basis loads in flight ahead of the sequential fma chain
            long long i = 0;
            for (; i + U <= k; i += U) {
                double2 q[U];
#pragma unroll
                for (int t = 0; t < U; t++) q[t] = a.Q[(i + t) * a.ldq_v + u];
#pragma unroll
                for (int t = 0; t < U; t++) x = cgs_msub<CPLX>(x, cbuf[i + t], q[t]);
            }
            for (; i < k; i++) x = cgs_msub<CPLX>(x, cbuf[i], a.Q[i * a.ldq_v + u]);
            vbuf[u] = x;
        }
        grid.sync();
        nn = sqrt(nrm256<CPLX>(vbuf, a.w, nvec, s_w));
        if (nn > n_prev / 2.0) {
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
            loop_exit(a.cond, a.use_cond);
        }
        return;
    }
    double2 *qo = a.Q + k * a.ldq_v, *wqo = a.WQ + k * a.ldq_v;
    for (long long u = gtid; u < nvec; u += nthr) {
        const double2 v = vbuf[u];
        const double2 qq = make_double2(v.x / nn, v.y / nn);
        qo[u] = qq;
        if (CPLX) {
            const double wu = a.w[u];
            wqo[u] = make_double2(wu * qq.x, wu * qq.y);
        } else {
            wqo[u] = make_double2(a.w[2 * u] * qq.x, a.w[2 * u + 1] * qq.y);
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

int cgs_grid(int num_sms) {
    // one CTA per SM (measured: grid barriers over 592 CTAs cost more than the extra waves)
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_imgs_cgs<true>, kCgsThreads, 0) != cudaSuccess)
        return num_sms;
    int p2 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2, k_imgs_cgs<false>, kCgsThreads, 0) == cudaSuccess && p2 < per_sm)
        per_sm = p2;
    if (per_sm > 1) per_sm = 1;  // one CTA per SM: the cheapest grid barrier
    const int g = per_sm * num_sms;
    return g < 1 ? 1 : g;
}

cudaError_t launch_imgs_cgs(const ImgsArgs &a, bool cplx, double2 *vbuf, double2 *cbuf, int grid, cudaStream_t s) {
    ImgsArgs aa = a;
    void *args[] = {&aa, &vbuf, &cbuf};
    return cudaLaunchCooperativeKernel(cplx ? (void *)k_imgs_cgs<true> : (void *)k_imgs_cgs<false>, grid, kCgsThreads,
                                       args, 0, s);
}

}  // namespace rbg
