/*
 * rbg_gen.h -- device generator for the synthetic chirp snapshot matrix (bench input).
 *
 * Not part of the method.  Fills the complex column-major N x M block S (column j at
 * S + j*ld complex elements, device memory) with the chirp recipe of DESIGN.md "Inputs"
 * (BASELINE.json configs 1-3; stand-in for the paper's IMRPhenomPv2 waveforms,
 * PAPER.md:820-834):
 *     h_j(t_i) = A_i (1 + 0.3 chi_j cos(3 phi_ij)) exp(i (phi_ij + psi_j)),  phi_ij = q_j base_i
 * then scales each column to ||h_j||_w = 1.  A, base, w (N each) and q, chi, psi (M each)
 * are device arrays; chi may be NULL when spin = 0.  Enqueued on `stream` (cudaStream_t).
 * Returns 0 on success, 1 on bad arguments, 2 on a launch error.
 */
#ifndef RBG_GEN_H
#define RBG_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
int rbg_gen_chirp(void *S, int64_t N, int64_t M, int64_t ld, const double *A, const double *base,
                  const double *w, const double *q, const double *chi, const double *psi, int spin,
                  void *stream);
#ifdef __cplusplus
}
#endif
#endif
