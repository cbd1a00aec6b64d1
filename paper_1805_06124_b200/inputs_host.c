/* inputs_host.c -- host (OpenMP) generator of the synthetic chirp snapshots of BASELINE.json
 * configs 1-3: the input recipe only (readings R19-R22), no arithmetic of
 * the method.  It exists so that bench.py's reference arm (the CPU oracle) can time the full
 * 10,000 x 409,600 workload without numpy's single-threaded generation (~400 s); the tests
 * keep using inputs.chirp_columns (numpy).  Values agree with the numpy and device generators
 * to rounding (different libm), which a timing arm does not depend on.
 *
 *   h_j(t_i) = A(t_i) (1 + 0.3 chi_j cos 3 phi) exp(i (phi + psi_j)),  phi = q_j base(t_i),
 *   then h_j /= ||h_j||_w.
 * A and base are the row factors computed by inputs.py; S is M x N complex (interleaved re,
 * im), column j at S + 2 j N.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>

/* nthreads > 0: that many OpenMP threads (torchrun sets OMP_NUM_THREADS=1 for its workers) */
void rbg_inputs_chirp(double *S, int64_t N, int64_t M, const double *A, const double *base, const double *w,
                      const double *q, const double *chi, const double *psi, int spin, int nthreads)
{
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t j = 0; j < M; j++) {
        double *col = S + 2 * j * N;
        const double qj = q[j], cj = spin ? chi[j] : 0.0, pj = psi[j];
        double acc = 0.0;
        for (int64_t i = 0; i < N; i++) {
            const double phi = qj * base[i];
            double amp = A[i];
            if (spin) amp *= 1.0 + 0.3 * cj * cos(3.0 * phi);
            const double re = amp * cos(phi + pj), im = amp * sin(phi + pj);
            col[2 * i] = re;
            col[2 * i + 1] = im;
            acc += w[i] * (re * re + im * im);
        }
        const double inv = 1.0 / sqrt(acc);
        for (int64_t i = 0; i < 2 * N; i++) col[i] *= inv;
    }
}
