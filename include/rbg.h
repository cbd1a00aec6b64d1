/*
 * rbg.h -- C ABI of the B200-native RB-greedy / pivoted-QR hot path (arXiv 1805.06124).
 *
 * The library computes, on one or more B200 GPUs, the reduced-basis greedy of
 * Algorithm 3, which Proposition 5.5 shows is
 * modified Gram-Schmidt with column pivoting (Algorithm 2), using the
 * residual recurrence of Sec. 6.1.2 and Hoffmann's iterated MGS with
 * kappa = 2 for each new basis vector:
 *
 *   r2_j = ||s_j||_w^2                                             (sweep 0)
 *   repeat:  (J, m) = argmax_j r2_j (ties: lowest global index)   (pivot search)
 *            err_k = sqrt(max(m, 0)); stop if err_k < tol, k = k_max, or all selected
 *            q_{k+1} = IMGS(s_J) against q_1..q_k; stop RANK if degenerate
 *            R(k+1, j) = <q_{k+1}, s_j>_w and r2_j -= |R(k+1, j)|^2 for every column
 *
 * with <x, y>_w = sum_i w_i conj(x_i) y_i.  Every floating-point result follows the
 * canonical arithmetic contract of DESIGN.md (lane counts L_S = 32 for the sweep and
 * L_I = 2048 for IMGS), so results are bit-reproducible and independent of the number of
 * GPUs the columns are sharded over.
 *
 * Conventions (all entry points):
 *  - Every call returns rbg_status; none aborts, throws or exits.  On failure a
 *    thread-local message is available from rbg_last_error().
 *  - Matrices are column-major.  A complex element is two doubles (re, im) interleaved.
 *    S is N x M with column j at S + j*ld elements; ld >= N.
 *  - Ownership: the library owns the context and every buffer it allocates; outputs are
 *    copied into caller-owned buffers.  A borrowed device S (rbg_desc.borrow = 1) must
 *    stay alive and unmodified until rbg_destroy.  The work buffers of rbg_validate,
 *    rbg_gram(_fold), rbg_reconstruct(_gram) and rbg_eim (up to 1 GB each) stay allocated in
 *    the context between calls and are released by rbg_destroy; a context is not thread-safe.
 *  - All GPU work is enqueued on one CUDA stream (rbg_desc.stream, or a stream the library
 *    creates).  Getters synchronise that stream.
 */
#ifndef RBG_H
#define RBG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rbg_ctx rbg_ctx;  /* opaque, owned by the library */

typedef enum { RBG_REAL_F64 = 1, RBG_COMPLEX_F64 = 2 } rbg_dtype;

typedef enum {
    RBG_OK = 0,
    RBG_EINVAL = 1,      /* bad argument (sizes, tol, weights, null pointer, alignment) */
    RBG_ENONFINITE = 2,  /* S holds NaN/Inf; message gives the first (row, col)         */
    RBG_ENOMEM = 3,      /* device or host allocation failed                           */
    RBG_ECUDA = 4,       /* CUDA runtime error                                         */
    RBG_ENCCL = 5,       /* NCCL missing or failed                                     */
    RBG_ESTATE = 6       /* call not valid in the context's current state              */
} rbg_status;

/* Why the greedy stopped.  Stop reasons are results, not errors. */
typedef enum {
    RBG_STOP_NONE = 0,          /* still running (or not started)                         */
    RBG_STOP_TOL = 1,           /* err_k < tol (Algorithm 3 loop test)      */
    RBG_STOP_KMAX = 2,          /* k = k_max basis vectors                                */
    RBG_STOP_RANK = 3,          /* IMGS found the pivot numerically in span(Q) (R7, R17)   */
    RBG_STOP_ALL_SELECTED = 4,  /* every column already selected                          */
    RBG_STOP_PEER_TIMEOUT = 5   /* comm = PEER: a rank's record did not arrive within
                                   rbg_desc.peer_timeout_ms; the outputs are incomplete     */
} rbg_stop;

typedef enum { RBG_MEM_HOST = 0, RBG_MEM_DEVICE = 1 } rbg_mem;

/* Column-sharded execution (the paper's MPI exchange):
 * NONE = one GPU owns all columns;
 * NCCL = ncclAllGather of {maxloc record, candidate column} per iteration;
 * EXTERNAL = the caller moves the exchange buffers itself between rbg_iter_local and
 *   rbg_iter_finish (used to run the sharded path on one GPU in tests);
 * PEER = no collective library: each rank's sweep kernel stores its 16-byte maxloc record into
 *   every rank's memory over NVLink (CUDA IPC mappings, release/acquire tags) and the
 *   replicated IMGS reads the winner's column from the owner's send slot over NVLink.  Needs
 *   rbg_peer_export + rbg_peer_connect (all ranks on one node, P2P-capable GPUs, world <= 8). */
typedef enum { RBG_COMM_NONE = 0, RBG_COMM_NCCL = 1, RBG_COMM_EXTERNAL = 2, RBG_COMM_PEER = 3 } rbg_comm;

/* Bytes of one rank's PEER handle blob (two cudaIpcMemHandle_t). */
#define RBG_PEER_HANDLE_BYTES 128

/* Orthogonalisation of each new basis vector: Hoffmann's iterated MODIFIED Gram-Schmidt
 * ("MGSCI", kappa = 2; the paper's choice) or iterated CLASSICAL
 * Gram-Schmidt ("CGSCI", kappa = 2; same acceptance test, all coefficients of a pass at once:
 * 2 grid-wide phases per pass instead of k dependent reductions). */
typedef enum { RBG_ORTHO_MGS = 0, RBG_ORTHO_CGS = 1 } rbg_ortho;

/* Column residuals: RECURRENCE = the paper's Eq. (Residual), r2_j <- r2_j - |c_kj|^2 with one
 * read of S per iteration (accuracy floor ~sqrt(eps) max||s||, reading R8);
 * EXPLICIT = Algorithm 2's in-place column updates v_j <- v_j - c_kj q_k with r2_j recomputed
 * from the updated column: floor ~eps max||s||, a read and a write of the
 * (library-owned, W^{1/2}-scaled) columns per iteration.  NEXT-row calls (validate, add_columns,
 * gram, reconstruct, eim) need RECURRENCE.  (DESIGN.md CAC rule 12.)          */
typedef enum { RBG_RESIDUAL_RECURRENCE = 0, RBG_RESIDUAL_EXPLICIT = 1 } rbg_residual;

typedef struct rbg_desc {
    const void *S;        /* N x M_loc snapshot block, column-major                      */
    rbg_mem S_mem;        /* where S lives                                               */
    int64_t N;            /* rows (grid points), >= 1                                    */
    int64_t M;            /* columns on this rank (M_loc), >= 1                          */
    int64_t ld;           /* column stride in elements, >= N (0 => N)                    */
    int borrow;           /* device S only: 1 = use in place (16-B aligned columns; real
                             dtype needs even ld), 0 = copy                              */
    const double *w;      /* N positive finite weights, NULL => all ones                 */
    rbg_mem w_mem;
    rbg_dtype dtype;
    double tol;           /* >= 0; stop when err_k < tol                                 */
    int64_t k_max;        /* 1 <= k_max <= N (k_max > M_global stops ALL_SELECTED)        */
    void *stream;         /* cudaStream_t to enqueue on (cudaStreamLegacy for the legacy
                             default stream); NULL => a library-owned stream             */
    int device;           /* CUDA ordinal; -1 => current device                          */
    int check_finite;     /* 1 (default) => scan S for NaN/Inf at create                 */
    rbg_comm comm;
    int rank, world;      /* this rank and the number of ranks (world = 1 unless sharded) */
    int64_t col_offset;   /* global index of local column 0                              */
    int64_t M_global;     /* total columns over all ranks (0 => M)                       */
    uint8_t nccl_id[128]; /* ncclUniqueId from rbg_get_unique_id on rank 0 (comm = NCCL) */
    rbg_ortho ortho;      /* orthogonalisation of the pivot column (default MGS)         */
    rbg_residual residual;/* how the column residuals are kept (default RECURRENCE)       */
    int64_t peer_timeout_ms; /* comm = PEER: stop PEER_TIMEOUT when a peer's record is this
                             late (0 => 60,000 ms)                                       */
} rbg_desc;

typedef struct rbg_stats {
    int64_t k;              /* basis vectors built                                      */
    int64_t sweeps;         /* coefficient sweeps timed (excluding sweep 0)              */
    double t_init_ms;       /* sweep 0 (norms)                                          */
    double t_sweep_ms;      /* sum over sweeps of the fused sweep kernel (T_pivot)       */
    double t_xchg_ms;       /* sum of exchange time (C_j); 0 on one GPU                  */
    double t_imgs_ms;       /* sum of pivot decision + IMGS (T_IMGS)                     */
    double t_total_ms;      /* first event to last event (T_j summed)      */
    double t_gap_ms;        /* launch gaps between iterations (part of C_j)              */
    int64_t noop_iters;     /* iterations launched after the stop decision (early-exit
                               kernels; 0 with rbg_run's device loop)                    */
} rbg_stats;

/* Fill *d with defaults: ld = 0, borrow = 0, w = NULL, device = -1, check_finite = 1,
 * comm = NONE, rank = 0, world = 1, col_offset = 0, M_global = 0, ortho = MGS,
 * residual = RECURRENCE. */
void rbg_desc_init(rbg_desc *d);

/* North-star entry point: host S (N x M, ld = N) and host w (NULL => ones).  The matrix
 * is copied to the current device.  Errors: EINVAL (N < 1, M < 1, k_max outside
 * [1, N], tol < 0 or NaN, w_i <= 0 or non-finite, unknown dtype, NULL S or ctx),
 * ENONFINITE (first NaN/Inf position in the message), ENOMEM, ECUDA. */
rbg_status rbg_create(rbg_ctx **ctx, const void *S, int64_t N, int64_t M, const double *w,
                      double tol, int64_t k_max, rbg_dtype dtype);

/* Extended create (memory space, borrowing, stream, device, sharding). */
rbg_status rbg_create_ex(rbg_ctx **ctx, const rbg_desc *desc);

/* ncclGetUniqueId (rank 0 calls it; the caller broadcasts the 128 bytes).  ENCCL if
 * libnccl.so.2 cannot be loaded. */
rbg_status rbg_get_unique_id(uint8_t out[128]);

/* Run the greedy to its stop reason (blocking).  ESTATE for comm = EXTERNAL. */
rbg_status rbg_run(rbg_ctx *ctx);

/* Enqueue up to n more iterations without synchronising (the first call also enqueues
 * sweep 0).  Iterations after the stop decision are no-ops on the device. */
rbg_status rbg_step(rbg_ctx *ctx, int64_t n);

/* Per-phase CUDA-event timing of subsequent iterations (0 = off, the default). */
rbg_status rbg_set_timing(rbg_ctx *ctx, int on);

/* Capture iterations into CUDA graphs of `batch` iterations (0 = plain launches). */
rbg_status rbg_set_graph_batch(rbg_ctx *ctx, int batch);

/* Synchronise the context's stream. */
rbg_status rbg_sync(rbg_ctx *ctx);

/* k = basis size, M_loc = local columns, why = stop reason (NONE while running). */
rbg_status rbg_result_info(rbg_ctx *ctx, int64_t *k, int64_t *M_loc, rbg_stop *why);

/* Outputs (replicated on every rank unless noted).  Host buffers unless on_device. */
rbg_status rbg_get_pivots(rbg_ctx *ctx, int64_t *out);        /* k global column ids   */
/* errors: err_0 .. err_k (k+1 entries) once the greedy stopped; k entries (err_0 .. err_{k-1})
 * while it is running or after PEER_TIMEOUT (the decision for err_k never ran).           */
rbg_status rbg_get_errors(rbg_ctx *ctx, double *out);
rbg_status rbg_get_nu(rbg_ctx *ctx, int32_t *out);            /* k IMGS sweep counts   */
rbg_status rbg_get_rdiag(rbg_ctx *ctx, double *out);          /* k IMGS norms R(i,i)   */
/* Q: N x k column-major, column i at out + i*ldq elements (ldq >= N).                   */
rbg_status rbg_get_basis(rbg_ctx *ctx, void *out, int64_t ldq, int on_device);
/* R: k x M_loc ROW-major, R(i, j) = <q_i, s_j>_w at out + i*ldr + j elements
 * (ldr >= M_loc); column-sharded over ranks.                                            */
rbg_status rbg_get_R(rbg_ctx *ctx, void *out, int64_t ldr, int on_device);
/* r2: M_loc squared residuals after the last sweep (selected columns = -inf).           */
rbg_status rbg_get_r2(rbg_ctx *ctx, double *out, int on_device);
rbg_status rbg_get_stats(rbg_ctx *ctx, rbg_stats *out);
/* Per-iteration phase times (timing mode): n entries each, any pointer may be NULL.     */
rbg_status rbg_get_timings(rbg_ctx *ctx, double *sweep_ms, double *xchg_ms, double *imgs_ms,
                           int64_t n);

/* Out-of-sample validation ("performs out-of-sample validation of the
 * resulting basis"; DESIGN.md NEXT f-1): for each column v_j of the N x M_v block V
 * (column stride ldv elements, 0 => N; host or device), the coefficients
 * C(i, j) = <q_i, v_j>_w against the current basis (i < k) and the projection error
 * err_j = sqrt(max(||v_j||_w^2 - sum_i |C(i,j)|^2, 0)) evaluated with the same per-column
 * arithmetic as the greedy's own residuals (sweep 0 + the coefficient recurrence; all k
 * coefficients of a column come from one blocked pass over V, bit-identical to one sweep per
 * basis vector).  A device V with column pitch equal to the library's padded layout (complex,
 * or real with N even, ldv = N) and 16-byte alignment is read in place, otherwise copied.
 * err: M_v doubles (may be NULL); C: k x M_v row-major with row stride ldc (may be NULL);
 * both on the device if out_on_device.  Blocking.  ENONFINITE if V holds NaN/Inf.         */
rbg_status rbg_validate(rbg_ctx *ctx, const void *V, int64_t M_v, int64_t ldv, rbg_mem V_mem, double *err,
                        void *C, int64_t ldc, int out_on_device);

/* Enrichment ("automatically enrich the basis by iterative refinement"):
 * append the N x M_f block F (column stride ldf, 0 => N) to the training columns of a
 * single-GPU context.  Their R rows and residuals are computed with the greedy's own
 * arithmetic, the pivot search restarts over all columns and a stopped greedy may continue
 * (rbg_run / rbg_step).  The caller's S is not copied (a borrowed S stays borrowed): appended
 * columns live in a library-owned second segment that the sweep streams after the first;
 * only R's rows (k_max x M) and the per-column vectors are reallocated.
 * ESTATE on sharded contexts (see rbg_add_columns_ex), and on a running greedy (started, no
 * stop decision yet: the sweep with q_{k-1} is still pending) -- run it to its stop first.
 * Blocking.                                                                                 */
rbg_status rbg_add_columns(rbg_ctx *ctx, const void *F, int64_t M_f, int64_t ldf, rbg_mem F_mem);
/* Enrichment of a column-sharded context (also valid on one GPU): every rank calls it, in the
 * same round, with its own failing columns (M_f >= 0; F may be NULL when M_f = 0).  They get
 * the global indices first_gid .. first_gid + M_f - 1, which must lie in [M_global,
 * M_global_new); M_global_new is the new total over all ranks (the same on every rank).  With
 * the ranks' appended blocks numbered in rank order (first_gid = old M_global + the counts of
 * the ranks before), the result equals one context enriched with the concatenated columns bit
 * for bit.  The pivot search restarts on every rank (its candidate published to the exchange
 * with a new record epoch) and a stopped greedy may continue.  first_gid < 0 and
 * M_global_new <= 0 select the single-GPU defaults (M_global, M_global + M_f).  ESTATE on a
 * running greedy, as rbg_add_columns.  Blocking.                                            */
rbg_status rbg_add_columns_ex(rbg_ctx *ctx, const void *F, int64_t M_f, int64_t ldf, rbg_mem F_mem, int64_t first_gid,
                              int64_t M_global_new);

/* Checkpoint / resume.  A checkpoint is the state the getters return once the
 * greedy stopped: k, pivots[k], errors[k+1] (err_k may be dropped), nu[k], rdiag[k], Q (N x k,
 * column stride ldq >= N), R (k x M row-major, row stride ldr >= M) and r2[M].  rbg_restore
 * loads it into a FRESH single-GPU context created on the same S and w (k < k_max, e.g. a run
 * continued to a larger k_max): w o Q is recomputed with the IMGS kernel's multiplication, the
 * pivot search runs over r2, and the next rbg_run / rbg_step begins at the decision for k --
 * the continued greedy equals an uninterrupted one bit for bit.  Arrays in host memory
 * (mem = HOST) or device memory (DEVICE).  EINVAL on bad sizes or pivots; ESTATE on a started,
 * sharded or explicit-residual context.  k = 0 restores nothing.  Blocking.                */
rbg_status rbg_restore(rbg_ctx *ctx, int64_t k, const int64_t *pivots, const double *errors, const int32_t *nu,
                       const double *rdiag, const void *Q, int64_t ldq, const void *R, int64_t ldr, const double *r2,
                       rbg_mem mem);

/* Gram matrix G = R R^H of the k x M coefficient block (k = basis size): k x k Hermitian,
 * column-major with leading dimension ldg >= k, complex (16-byte) entries even for a real
 * dtype.  Summation order: columns in chunks of 4096, each chunk one sequential fma chain,
 * chunks added in order (reading R30).  Single-GPU contexts (ESTATE otherwise).
 * Like rbg_reconstruct and rbg_gram_fold it reads R rows 0..k-1: ESTATE on a running greedy
 * (started, no stop decision yet), whose row k-1 is still pending.                        */
rbg_status rbg_gram(rbg_ctx *ctx, void *G, int64_t ldg, int on_device);

/* Algorithm 4 "Reconstruction": SVD of R(1:k, :) through its Gram
 * matrix (cyclic Jacobi on the GPU), sigma = singular values in descending order (k
 * entries, may be NULL), kr = #{sigma_i > tau2} capped at kr_max (0 => no cap), and the
 * reconstructed basis X = Q V(:, 1:kr) (N x kr column-major, leading dimension ldx >= N;
 * W-orthonormal; may be NULL).  Single-GPU contexts.  Blocking.                             */
rbg_status rbg_reconstruct(rbg_ctx *ctx, double tau2, int64_t kr_max, int64_t *kr, double *sigma, void *X,
                           int64_t ldx, int on_device);

/* Sharded Algorithm 4 (column-sharded contexts; any world size).  rbg_gram_fold: G (k x k
 * complex column-major, leading dimension ldg >= k, host or device) holds the Gram sum of the
 * previous ranks (zeros on rank 0) and is replaced by G + R_loc R_loc^H, this rank's columns
 * summed in chunks of 4096 local columns, each chunk added onto G in order (real and imaginary
 * parts independently, diagonal made real).  Folding the ranks in rank order gives exactly
 * rbg_gram of one context holding all columns when every rank's col_offset is a multiple of
 * 4096 (reading R33).  rbg_reconstruct_gram: Algorithm 4 from a given Hermitian G
 * (e.g. the folded one, identical on every rank) -- outputs as rbg_reconstruct.           */
rbg_status rbg_gram_fold(rbg_ctx *ctx, void *G, int64_t ldg, int on_device);
rbg_status rbg_reconstruct_gram(rbg_ctx *ctx, const void *G, int64_t ldg, int G_on_device, double tau2,
                                int64_t kr_max, int64_t *kr, double *sigma, void *X, int64_t ldx, int on_device);

/* Empirical interpolation nodes (standard greedy EIM in residual form,
 * DESIGN.md reading R31) for the current basis: nodes[k] row indices (distinct; ties -> lowest
 * row) and B = Q(nodes, :), the k x k node matrix (column-major, leading dimension ldb >= k,
 * complex 16-byte entries even for a real dtype; may be NULL).  Requires k <= 1024.  ESTATE
 * if an interpolation residual vanishes (degenerate basis).  Blocking.                      */
rbg_status rbg_eim(rbg_ctx *ctx, int64_t *nodes, void *B, int64_t ldb, int on_device);

/* Sharded path driven by the caller (comm = EXTERNAL).  One iteration is
 *   rbg_iter_local (sweep + maxloc + pack the local candidate into the send buffer),
 *   the caller's all-gather of send buffers into every rank's receive buffer
 *   (rank p's bytes at recv + p * bytes), then rbg_iter_finish (pivot decision + IMGS). */
rbg_status rbg_iter_local(rbg_ctx *ctx);
rbg_status rbg_iter_finish(rbg_ctx *ctx);
rbg_status rbg_xchg_buffers(rbg_ctx *ctx, void **send, void **recv, size_t *bytes_per_rank);
/* Convenience for tests: all-gather the send buffers of `world` EXTERNAL contexts on the
 * same device (device-to-device copies), ctxs[p] holding rank p. */
rbg_status rbg_emulate_allgather(rbg_ctx **ctxs, int world);

/* PEER exchange setup.  Every rank exports RBG_PEER_HANDLE_BYTES of CUDA-IPC handles (its
 * record array and send slots), the caller all-gathers them (rank order) and every rank
 * connects: peer buffers are mapped with cudaIpcOpenMemHandle (own buffers used directly).
 * Until connected, rbg_run / rbg_step return ESTATE (a one-rank PEER context is connected at
 * create).  ESTATE on a non-PEER context; ECUDA if a mapping fails.  The PEER iteration can
 * also be driven by rbg_iter_local / rbg_iter_finish (finish = wait for the records + IMGS). */
rbg_status rbg_peer_export(rbg_ctx *ctx, uint8_t out[RBG_PEER_HANDLE_BYTES]);
rbg_status rbg_peer_connect(rbg_ctx *ctx, const uint8_t *all_handles);
/* Tests on one GPU: wire `world` PEER contexts of this process (ctxs[p] = rank p, same
 * device and the same stream, else EINVAL) to each other's buffers directly.  Drive them with rbg_iter_local on every rank,
 * then rbg_iter_finish on every rank (stream order puts every record in place before any
 * rank waits: no kernel ever waits for one that has not been launched). */
rbg_status rbg_peer_connect_local(rbg_ctx **ctxs, int world);

/* Out-of-bounds write detection (compute-sanitizer is closed on the GPU pool): while on, every
 * device buffer the library allocates gets a 256-byte canary tail (0xA5), checked when the
 * buffer is freed; buffers allocated while off are unaffected. */
void rbg_debug_set_canary(int on);
/* Canary violations so far, after checking every live canaried buffer now (synchronises the
 * devices); if > 0, rbg_last_error() describes the first. */
int64_t rbg_debug_canary_violations(void);

/* Lane counts of the canonical arithmetic contract this build implements. */
void rbg_lanes(int *L_S, int *L_I);
const char *rbg_version(void);
const char *rbg_last_error(void);

/* NULL-safe; frees everything the library allocated for ctx. */
void rbg_destroy(rbg_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* RBG_H */
