/*
 * oracle/rbg_oracle.c -- CPU ORACLE for the RB-greedy / MGS-with-pivoting hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1805_06124_b200/, include/rbg.h, the CUDA kernels) never calls it, links it
 * or shares a line of code, header, table or constant generator with it.
 *
 * What it computes: Algorithm 3 "RB-greedy" of arXiv 1805.06124 with
 * the residual recurrence of Sec. 6.1.2 (Eqs. rec1/Residual) and the
 * Hoffmann iterated MGS ("MGSCI", kappa = 2) for the new basis vector.
 * Weighted inner product <x,y>_w = sum_i w_i conj(x_i) y_i (BASELINE.json north_star);
 * with w = 1 this is the paper's l2 problem, and in general it is the paper's problem on
 * W^{1/2} S (reading R6).
 *
 * Summation order.  Every dot product and weighted norm is evaluated in the order fixed
 * by DESIGN.md section "Canonical arithmetic contract" (CAC): element i of a length-N vector
 * belongs to lane (i / V) mod L (V = 1 complex, 2 real), a lane accumulates its elements in
 * increasing i with explicit fma(), and the L lane partials are combined by a balanced
 * pairwise tree in lane order.  L = 1 is the textbook sequential sum ("plain mode");
 * L = 32 for the column sweep and L = 2048 for IMGS is the "canonical mode" that the GPU
 * path must reproduce bit for bit.  The lane count is an argument here, never read from
 * the CUDA path.  Compile with -ffp-contract=off so that no a*b+c is fused except where
 * fma() is written.
 *
 * Pins: tests/test_oracle_pins.py (closed forms, Prop. 5.5 equivalence with Algorithm 2,
 * LAPACK xGEQP3, Cor. 5.6 brute force, Cor. 5.7 volume identity, error bound of the dot).
 * Parity unpinned: the exact pivot sequence once the residuals reach the recurrence's accuracy
 * floor (R8) and the exact k of a RANK stop (configs 0, 1, 4) are fixed only by the
 * summation order above -- the paper does not determine them; the plain-mode test reports
 * where two valid orders part.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_STOP_NONE 0
#define ORC_STOP_TOL 1
#define ORC_STOP_KMAX 2
#define ORC_STOP_RANK 3
#define ORC_STOP_ALL_SELECTED 4

#define ORC_KAPPA 2.0       /* Hoffmann MGSCI kappa = 2 */
#define ORC_NU_MAX 5        /* sweep cap, reading R7 */

static int is_pow2(int L) { return L >= 1 && (L & (L - 1)) == 0; }

/* Balanced pairwise tree over lanes in lane order: for h = 1,2,4,..,L/2,
 * p[l] <- p[l] + p[l+h] for l = 0 mod 2h.  Returns p[0].  (CAC rule 3) */
static double lane_tree(double *p, int L)
{
    for (int h = 1; h < L; h *= 2)
        for (int l = 0; l < L; l += 2 * h)
            p[l] = p[l] + p[l + h];
    return p[0];
}

/* DOT_L(xt, y) = sum_i conj(xt_i) * y_i  (CAC rule 2).  xt is the weighted basis vector
 * w o q (the weight is folded into xt, PAPER.md Eq. Residual with <.,.>_w).
 * Complex data are interleaved (re, im). */
void orc_dot(const double *xt, const double *y, int64_t n, int cplx, int L,
             double *re_out, double *im_out)
{
    double *pr = (double *)calloc((size_t)L, sizeof(double));
    double *pi = (double *)calloc((size_t)L, sizeof(double));
    if (cplx) {
        for (int64_t i = 0; i < n; i++) {
            int l = (int)(i % L);
            double a = xt[2 * i], b = xt[2 * i + 1];
            double x = y[2 * i], yy = y[2 * i + 1];
            pr[l] = fma(a, x, pr[l]);
            pr[l] = fma(b, yy, pr[l]);
            pi[l] = fma(a, yy, pi[l]);
            pi[l] = fma(-b, x, pi[l]);
        }
    } else {
        for (int64_t i = 0; i < n; i++) {
            int l = (int)((i / 2) % L);
            pr[l] = fma(xt[i], y[i], pr[l]);
        }
    }
    *re_out = lane_tree(pr, L);
    *im_out = cplx ? lane_tree(pi, L) : 0.0;
    free(pr);
    free(pi);
}

/* NRM_L(y) = sum_i w_i |y_i|^2  (CAC rule 4): t = w_i*x; acc = fma(t, x, acc) per
 * real component.  This is ||s_i||^2 of PAPER.md Eq. Residual in the w-norm. */
double orc_nrm(const double *y, const double *w, int64_t n, int cplx, int L)
{
    double *p = (double *)calloc((size_t)L, sizeof(double));
    if (cplx) {
        for (int64_t i = 0; i < n; i++) {
            int l = (int)(i % L);
            double t = w[i] * y[2 * i];
            p[l] = fma(t, y[2 * i], p[l]);
            t = w[i] * y[2 * i + 1];
            p[l] = fma(t, y[2 * i + 1], p[l]);
        }
    } else {
        for (int64_t i = 0; i < n; i++) {
            int l = (int)((i / 2) % L);
            double t = w[i] * y[i];
            p[l] = fma(t, y[i], p[l]);
        }
    }
    double r = lane_tree(p, L);
    free(p);
    return r;
}

/* |c|^2 (CAC rule 5) */
static double abs2(double re, double im, int cplx)
{
    return cplx ? fma(re, re, im * im) : re * re;
}

/*
 * Iterated modified Gram-Schmidt, Hoffmann "MGSCI" with kappa = 2 (
 * acceptance test and cap are DESIGN.md reading R7).
 *   v <- s_J; n0 = sqrt(NRM(v)); n_prev = n0
 *   repeat (nu = 1..NU_MAX):  for i = 1..k: c = <q_i, v>_w; coeff_i += c; v <- v - c q_i
 *                             n = sqrt(NRM(v)); accept if n > n_prev / kappa; n_prev = n
 *   degenerate (return 0) if never accepted or n < delta * n0, delta = 1000 * 2^-52
 *   q = v / n (componentwise IEEE division), wq = w o q.
 * Q, WQ: column-major, column i at Q + i*ldq (ldq in doubles).  v is overwritten.
 * Returns 1 on success (q, wq, *n_out, *nu_out, coeff set), 0 if degenerate.
 */
int orc_imgs(const double *Q, const double *WQ, int64_t ldq, int64_t k,
             double *v, const double *w, int64_t n, int cplx, int L,
             double *q_out, double *wq_out, double *coeff /* k (x2 if cplx), may be NULL */,
             double *n_out, int *nu_out)
{
    const double delta = 1000.0 * 0x1p-52;
    const int nv = cplx ? 2 : 1;
    double n0 = sqrt(orc_nrm(v, w, n, cplx, L));
    double n_prev = n0, nn = 0.0;
    int nu = 0, accepted = 0;
    if (coeff) memset(coeff, 0, sizeof(double) * (size_t)(k * nv));
    while (nu < ORC_NU_MAX) {
        nu++;
        for (int64_t i = 0; i < k; i++) {
            const double *q = Q + i * ldq, *wq = WQ + i * ldq;
            double cr, ci;
            orc_dot(wq, v, n, cplx, L, &cr, &ci);
            if (coeff) {
                coeff[i * nv] += cr;
                if (cplx) coeff[i * nv + 1] += ci;
            }
            if (cplx) {
                for (int64_t e = 0; e < n; e++) {
                    double qr = q[2 * e], qi = q[2 * e + 1];
                    double vr = v[2 * e], vi = v[2 * e + 1];
                    vr = fma(-cr, qr, vr);
                    vr = fma(ci, qi, vr);
                    vi = fma(-cr, qi, vi);
                    vi = fma(-ci, qr, vi);
                    v[2 * e] = vr;
                    v[2 * e + 1] = vi;
                }
            } else {
                for (int64_t e = 0; e < n; e++) v[e] = fma(-cr, q[e], v[e]);
            }
        }
        nn = sqrt(orc_nrm(v, w, n, cplx, L));
        if (nn > n_prev / ORC_KAPPA) { accepted = 1; break; }
        n_prev = nn;
    }
    *nu_out = nu;
    *n_out = nn;
    if (!accepted || !(nn >= delta * n0) || nn == 0.0) return 0;
    for (int64_t e = 0; e < n * nv; e++) q_out[e] = v[e] / nn;
    if (cplx) {
        for (int64_t e = 0; e < n; e++) {
            wq_out[2 * e] = w[e] * q_out[2 * e];
            wq_out[2 * e + 1] = w[e] * q_out[2 * e + 1];
        }
    } else {
        for (int64_t e = 0; e < n; e++) wq_out[e] = w[e] * q_out[e];
    }
    return 1;
}

/*
 * Iterated CLASSICAL Gram-Schmidt, Hoffmann "CGSCI" with kappa = 2 (the same family and
 * acceptance test as orc_imgs; DESIGN.md CAC rule 11): per sweep all
 * coefficients c_i = <q_i, v>_w are taken from the same v, then v <- v - sum_i c_i q_i
 * (per element, sequentially over i = 1..k).  Lanes L for every dot / norm.
 */
int orc_imgs_cgs(const double *Q, const double *WQ, int64_t ldq, int64_t k,
                 double *v, const double *w, int64_t n, int cplx, int L,
                 double *q_out, double *wq_out, double *n_out, int *nu_out)
{
    const double delta = 1000.0 * 0x1p-52;
    double *c = (double *)calloc((size_t)(2 * (k > 0 ? k : 1)), sizeof(double));
    double n0 = sqrt(orc_nrm(v, w, n, cplx, L));
    double n_prev = n0, nn = 0.0;
    int nu = 0, accepted = 0;
    while (nu < ORC_NU_MAX) {
        nu++;
        for (int64_t i = 0; i < k; i++) orc_dot(WQ + i * ldq, v, n, cplx, L, &c[2 * i], &c[2 * i + 1]);
        for (int64_t e = 0; e < n; e++) {
            if (cplx) {
                double vr = v[2 * e], vi = v[2 * e + 1];
                for (int64_t i = 0; i < k; i++) {
                    const double *q = Q + i * ldq;
                    double cr = c[2 * i], ci = c[2 * i + 1], qr = q[2 * e], qi = q[2 * e + 1];
                    vr = fma(-cr, qr, vr);
                    vr = fma(ci, qi, vr);
                    vi = fma(-cr, qi, vi);
                    vi = fma(-ci, qr, vi);
                }
                v[2 * e] = vr;
                v[2 * e + 1] = vi;
            } else {
                double x = v[e];
                for (int64_t i = 0; i < k; i++) x = fma(-c[2 * i], Q[i * ldq + e], x);
                v[e] = x;
            }
        }
        nn = sqrt(orc_nrm(v, w, n, cplx, L));
        if (nn > n_prev / ORC_KAPPA) { accepted = 1; break; }
        n_prev = nn;
    }
    free(c);
    *nu_out = nu;
    *n_out = nn;
    if (!accepted || !(nn >= delta * n0) || nn == 0.0) return 0;
    const int nv = cplx ? 2 : 1;
    for (int64_t e = 0; e < n * nv; e++) q_out[e] = v[e] / nn;
    if (cplx) {
        for (int64_t e = 0; e < n; e++) {
            wq_out[2 * e] = w[e] * q_out[2 * e];
            wq_out[2 * e + 1] = w[e] * q_out[2 * e + 1];
        }
    } else {
        for (int64_t e = 0; e < n; e++) wq_out[e] = w[e] * q_out[e];
    }
    return 1;
}

static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/*
 * RB-greedy, Algorithm 3, with the residual recurrence (PAPER.md:
 * 854-866) stored in place as r2_j <- r2_j - |c_kj|^2 (reading R5):
 *   r2_j = NRM(s_j) for all j; k = 0
 *   loop:
 *     (J, m) = argmax over unselected j of r2_j, ties -> lowest j (R9); none -> m = 0
 *     err_k = sqrt(max(m, 0))                     (sigma_hat_k, Cor. 5.6 PAPER.md:539-545)
 *     stop ALL_SELECTED if none unselected; TOL if err_k < tol (R2/R3); KMAX if k = k_max
 *     IMGS(s_J) -> q_{k+1}, or stop RANK if degenerate
 *     Pi_k = J; mark J selected (R10); k += 1
 *     for all j: c = <q_k, s_j>_w; R(k,j) = c; if j unselected: r2_j -= |c|^2
 * S: column-major, column j at S + j*lds (lds in doubles, >= N*(1+cplx)).
 * Outputs (caller-allocated): piv[k_max], Q/WQ[N*(1+cplx) x k_max] (ldq = N*(1+cplx)),
 * R[k_max x M] row-major (row stride M*(1+cplx) doubles), err[k_max+1], nu[k_max],
 * rdiag[k_max], r2[M].  t_sweep/t_imgs/t_iter (may be NULL): per-iteration seconds
 * (t_iter: pivot search + IMGS + sweep of iteration k).
 * L_S / L_I: lane counts for the sweep and for IMGS (powers of two).
 * max_iters >= 0 stops after that many completed iterations with stop = NONE (used to
 * time a bounded sample); pass -1 for no limit.  k0 >= 0 resumes from k0 iterations of
 * state held in the output arrays (enrichment); k0 < 0 starts fresh with sweep 0.
 * ortho: 0 = Hoffmann MGSCI (orc_imgs, the paper's), 1 = CGSCI (orc_imgs_cgs); L_I is the
 * lane count of whichever is used.
 * Returns k (basis size) or -1 on bad arguments.
 */
int64_t orc_greedy(const double *S, int64_t N, int64_t M, int64_t lds, const double *w,
                   int cplx, double tol, int64_t k_max, int L_S, int L_I, int nthreads,
                   int64_t max_iters, int64_t k0, int ortho, int explicit_mode,
                   int64_t *piv, double *Q, double *WQ, double *R, double *err, int *nu,
                   double *rdiag, double *r2, int *stop_out,
                   double *t_sweep, double *t_imgs, double *t_iter)
{
    if (N < 1 || M < 1 || k_max < 1 || !is_pow2(L_S) || !is_pow2(L_I)) return -1;
    const int nv = cplx ? 2 : 1;
    const int64_t ldq = N * nv;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    double *v = (double *)malloc(sizeof(double) * (size_t)ldq);
    /* explicit residuals (Algorithm 2 in-place updates; DESIGN.md CAC rule
     * 12): work on V = W^{1/2} S (sqrt(w_i) rounded once) with unit weights; the basis handed
     * back is Q = Q~ / W^{1/2}. */
    const double *w_true = w;
    double *V = NULL, *ones = NULL;
    if (explicit_mode) {
        V = (double *)malloc(sizeof(double) * (size_t)(ldq * M));
        ones = (double *)malloc(sizeof(double) * (size_t)N);
        for (int64_t i = 0; i < N; i++) ones[i] = 1.0;
        for (int64_t j = 0; j < M; j++)
            for (int64_t i = 0; i < N; i++) {
                double r = sqrt(w[i]);
                V[j * ldq + i * nv] = r * S[j * lds + i * nv];
                if (cplx) V[j * ldq + i * nv + 1] = r * S[j * lds + i * nv + 1];
            }
        S = V;
        lds = ldq;
        w = ones;
    }

    int64_t k = 0;
    if (k0 >= 0) {
        /* resume (enrichment): the caller's arrays hold k0 iterations of state and r2 holds
         * the residuals of all M columns; the loop continues at the pivot decision */
        k = k0;
    } else {
        /* sweep 0: r2_j = ||s_j||_w^2 */
#pragma omp parallel for schedule(static) if (M * N > 65536)
        for (int64_t j = 0; j < M; j++) r2[j] = orc_nrm(S + j * lds, w, N, cplx, L_S);
    }
    int stop = ORC_STOP_NONE;
    for (;;) {
        double t_it = now_s();
        /* pivot: argmax of r2 over unselected columns (selected hold -inf), lowest j on ties */
        int64_t J = -1;
        double m = -INFINITY;
        for (int64_t j = 0; j < M; j++)
            if (r2[j] > m) { m = r2[j]; J = j; }
        if (J < 0) m = 0.0;
        err[k] = sqrt(fmax(m, 0.0));
        if (J < 0) { stop = ORC_STOP_ALL_SELECTED; break; }
        if (err[k] < tol) { stop = ORC_STOP_TOL; break; }
        if (k == k_max) { stop = ORC_STOP_KMAX; break; }
        if (max_iters >= 0 && k == max_iters) { stop = ORC_STOP_NONE; break; }

        /* orthogonalize the pivot column */
        double ti = now_s();
        memcpy(v, S + J * lds, sizeof(double) * (size_t)ldq);
        double nrm;
        int nuk;
        int ok = ortho ? orc_imgs_cgs(Q, WQ, ldq, k, v, w, N, cplx, L_I, Q + k * ldq, WQ + k * ldq, &nrm, &nuk)
                       : orc_imgs(Q, WQ, ldq, k, v, w, N, cplx, L_I, Q + k * ldq, WQ + k * ldq, NULL, &nrm, &nuk);
        if (t_imgs) t_imgs[k] = now_s() - ti;
        if (!ok) { stop = ORC_STOP_RANK; break; }
        piv[k] = J;
        nu[k] = nuk;
        rdiag[k] = nrm;
        r2[J] = -INFINITY;
        k++;

        /* sweep: coefficients of every column against q_k and the residual update */
        double ts = now_s();
        const double *wq = WQ + (k - 1) * ldq;
        double *Rrow = R + (k - 1) * M * nv;
#pragma omp parallel for schedule(static) if (M * N > 65536)
        for (int64_t j = 0; j < M; j++) {
            double cr, ci;
            orc_dot(wq, S + j * lds, N, cplx, L_S, &cr, &ci);
            Rrow[j * nv] = cr;
            if (cplx) Rrow[j * nv + 1] = ci;
            if (r2[j] == -INFINITY) continue;
            if (!explicit_mode) {
                r2[j] = r2[j] - abs2(cr, ci, cplx);
            } else {
                /* v_j <- v_j - c q~_k (CAC rule 9 pattern), then r2_j = ||v_j||^2 */
                double *vj = V + j * lds;
                const double *q = Q + (k - 1) * ldq;
                if (cplx) {
                    for (int64_t e = 0; e < N; e++) {
                        double xr = vj[2 * e], xi = vj[2 * e + 1];
                        xr = fma(-cr, q[2 * e], xr);
                        xr = fma(ci, q[2 * e + 1], xr);
                        xi = fma(-cr, q[2 * e + 1], xi);
                        xi = fma(-ci, q[2 * e], xi);
                        vj[2 * e] = xr;
                        vj[2 * e + 1] = xi;
                    }
                } else {
                    for (int64_t e = 0; e < N; e++) vj[e] = fma(-cr, q[e], vj[e]);
                }
                r2[j] = orc_nrm(vj, w, N, cplx, L_S);
            }
        }
        if (t_sweep) t_sweep[k - 1] = now_s() - ts;
        if (t_iter) t_iter[k - 1] = now_s() - t_it;
    }
    free(v);
    if (explicit_mode) {
        for (int64_t i = 0; i < k; i++)
            for (int64_t e = 0; e < N; e++) {
                double r = sqrt(w_true[e]);
                Q[i * ldq + e * nv] = Q[i * ldq + e * nv] / r;
                if (cplx) Q[i * ldq + e * nv + 1] = Q[i * ldq + e * nv + 1] / r;
            }
        free(V);
        free(ones);
    }
    *stop_out = stop;
    return k;
}

/*
 * Out-of-sample validation (DESIGN.md NEXT f-1): for each column v_j of V,
 * the coefficients C(i,j) = <q_i, v_j>_w (i < k) and the squared projection error
 *   e2_j = NRM(v_j) - |C(0,j)|^2 - ... - |C(k-1,j)|^2   (subtracted in order i = 0..k-1),
 * i.e. exactly the residual recurrence the greedy applies to its own columns.
 * C: k x M_v row-major (row stride M_v elements); e2: M_v.
 */
void orc_validate(const double *WQ, int64_t ldq, int64_t k, const double *V, int64_t M_v, int64_t ldv,
                  const double *w, int64_t N, int cplx, int L_S, double *C, double *e2, int nthreads)
{
    const int nv = cplx ? 2 : 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(static) if (M_v * N > 65536)
    for (int64_t j = 0; j < M_v; j++) {
        const double *v = V + j * ldv;
        double acc = orc_nrm(v, w, N, cplx, L_S);
        for (int64_t i = 0; i < k; i++) {
            double cr, ci;
            orc_dot(WQ + i * ldq, v, N, cplx, L_S, &cr, &ci);
            C[(i * M_v + j) * nv] = cr;
            if (cplx) C[(i * M_v + j) * nv + 1] = ci;
            acc = acc - abs2(cr, ci, cplx);
        }
        e2[j] = acc;
    }
}

/*
 * Gram matrix of the coefficient block for Algorithm 4, reading R30:
 * G(a,b) = sum_j R(a,j) conj(R(b,j)) for the k x M block R (row-major, row stride M).
 * Order: the columns are cut into chunks of `chunk`; within a chunk the terms of each pair
 * are accumulated in increasing j with DOT rule 2 (x~ = R(b,:), y = R(a,:)); the chunk
 * partials are then added in chunk order; the diagonal's imaginary part is set to 0.
 * G: k x k column-major, complex interleaved.
 */
void orc_gram(const double *R, int64_t k, int64_t M, int cplx, int64_t chunk, double *G)
{
    const int nv = cplx ? 2 : 1;
#pragma omp parallel for schedule(dynamic) if (k * k * M > 1000000)
    for (int64_t a = 0; a < k; a++) {
        for (int64_t b = a; b < k; b++) {
            const double *ra = R + a * M * nv, *rb = R + b * M * nv;
            double gr = 0.0, gi = 0.0;
            for (int64_t j0 = 0; j0 < M; j0 += chunk) {
                const int64_t j1 = j0 + chunk < M ? j0 + chunk : M;
                double pr = 0.0, pi = 0.0;
                for (int64_t j = j0; j < j1; j++) {
                    if (cplx) {
                        double p = rb[2 * j], q = rb[2 * j + 1], x = ra[2 * j], y = ra[2 * j + 1];
                        pr = fma(p, x, pr);
                        pr = fma(q, y, pr);
                        pi = fma(p, y, pi);
                        pi = fma(-q, x, pi);
                    } else {
                        pr = fma(rb[j], ra[j], pr);
                    }
                }
                gr = gr + pr;
                gi = gi + pi;
            }
            if (a == b) gi = 0.0;  /* a Hermitian matrix has a real diagonal */
            G[2 * (a + b * k)] = gr;
            G[2 * (a + b * k) + 1] = gi;
            G[2 * (b + a * k)] = gr;
            G[2 * (b + a * k) + 1] = -gi;
        }
    }
}

/* complex helpers for the EIM oracle (R31): v - c*x (CAC rule 9) and a / b */
static void c_msub(double *vr, double *vi, double cr, double ci, double xr, double xi)
{
    double r = *vr, i = *vi;
    r = fma(-cr, xr, r);
    r = fma(ci, xi, r);
    i = fma(-cr, xi, i);
    i = fma(-ci, xr, i);
    *vr = r;
    *vi = i;
}

static void c_div(double ar, double ai, double br, double bi, double *qr, double *qi)
{
    double den = fma(br, br, bi * bi);
    *qr = fma(ar, br, ai * bi) / den;
    *qi = fma(ai, br, -(ar * bi)) / den;
}

/*
 * Greedy empirical interpolation nodes (the cited Alg. 5 is absent, so
 * the standard greedy EIM in residual form, reading R31):
 *   xi_1 = q_1, p_1 = argmax_i |xi_1(i)|^2
 *   for l = 2..k: c = T^{-1} q_l(P) by forward substitution (T_ab = xi_b(p_a), a >= b),
 *                 xi_l = q_l - sum_{b<l} c_b xi_b (sequential in b), p_l = argmax |xi_l|^2
 * ties -> lowest row.  Q: k basis vectors of N complex (interleaved; real data promoted with
 * zero imaginary parts).  nodes[k]; B (k x k column-major complex) = Q(nodes, :).
 * Returns 1, or 0 if a residual vanishes (degenerate basis).
 */
int orc_eim(const double *Q, int64_t k, int64_t N, int64_t *nodes, double *B)
{
    double *Xi = (double *)calloc((size_t)(2 * k * N), sizeof(double));
    double *T = (double *)calloc((size_t)(2 * k * k), sizeof(double));
    double *c = (double *)calloc((size_t)(2 * k), sizeof(double));
    int ok = 1;
    for (int64_t l = 0; l < k && ok; l++) {
        const double *q = Q + 2 * l * N;
        /* forward substitution, row by row, sequential in b */
        for (int64_t a = 0; a < l; a++) {
            double vr = q[2 * nodes[a]], vi = q[2 * nodes[a] + 1];
            for (int64_t b = 0; b < a; b++)
                c_msub(&vr, &vi, c[2 * b], c[2 * b + 1], T[2 * (a * k + b)], T[2 * (a * k + b) + 1]);
            c_div(vr, vi, T[2 * (a * k + a)], T[2 * (a * k + a) + 1], &c[2 * a], &c[2 * a + 1]);
        }
        /* residual and its argmax */
        double best = -1.0;
        int64_t p = 0;
        for (int64_t i = 0; i < N; i++) {
            double xr = q[2 * i], xi = q[2 * i + 1];
            for (int64_t b = 0; b < l; b++)
                c_msub(&xr, &xi, c[2 * b], c[2 * b + 1], Xi[2 * (b * N + i)], Xi[2 * (b * N + i) + 1]);
            Xi[2 * (l * N + i)] = xr;
            Xi[2 * (l * N + i) + 1] = xi;
            double m = fma(xr, xr, xi * xi);
            if (m > best) { best = m; p = i; }
        }
        if (!(best > 0.0)) { ok = 0; p = 0; }
        nodes[l] = p;
        for (int64_t b = 0; b <= l; b++) {
            T[2 * (l * k + b)] = Xi[2 * (b * N + p)];
            T[2 * (l * k + b) + 1] = Xi[2 * (b * N + p) + 1];
        }
    }
    if (ok)
        for (int64_t a = 0; a < k; a++)
            for (int64_t b = 0; b < k; b++) {
                B[2 * (a + b * k)] = Q[2 * (b * N + nodes[a])];
                B[2 * (a + b * k) + 1] = Q[2 * (b * N + nodes[a]) + 1];
            }
    free(Xi);
    free(T);
    free(c);
    return ok;
}
