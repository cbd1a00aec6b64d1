// kernels.h -- host-visible launch interface of the rbg device kernels (internal).
#pragma once
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include "common.cuh"

namespace rbg {

// Fused column sweep (a0 init norms / a2 coefficient sweep + residual update + maxloc).
struct SweepArgs {
    const double2 *S;      // snapshot block as 16-byte vectors, column j < M0 at S + j*ldv
    long long ldv;         // column stride in vectors
    const double2 *S1;     // columns appended by enrichment (j >= M0) at S1 + (j - M0)*nvec
    long long M0;          // columns of the first segment (== M when nothing was appended)
    long long M;           // local columns
    long long N;           // rows (elements)
    long long nvec;        // vectors per column: complex N, real ceil(N/2)
    const double *w;       // weights, zero padded to a multiple of 2 (+2)
    const double2 *WQ;     // weighted basis, column i at WQ + i*ldq_v
    long long ldq_v;
    double *R;             // k_max rows of ldr elements (16 B complex / 8 B real), row-major
    long long ldr;         // R row stride in elements (>= M)
    long long qi;          // >= 0: use basis vector qi and R row qi (validation); -1: q_{k-1}
    double2 *V;            // explicit mode: the columns updated in place (== S), else NULL
    double *r2;            // M
    DevState *st;
    Rec *recs;             // one record per CTA
    unsigned *ticket;      // last-CTA-done counter (returns to 0)
    unsigned long long *next_col;  // dynamic column counter of k_sweep_dyn (returns to 0)
    long long col_offset;  // global index of local column 0
    unsigned char *send;   // exchange slot of this rank (NULL on one GPU)
    // PEER exchange (peer_world > 0): every rank's record array, this rank's index, and the
    // byte size of one of the two send slots (the candidate goes to slot tag & 1)
    PeerRec *peer_in[kMaxPeers];
    int peer_world, peer_rank;
    size_t peer_slot;
    unsigned long long peer_epoch;  // bumped by every sharded rbg_add_columns_ex (record tags)
    const long long *gid;   // global index of each local column once columns were appended to a
                            // sharded context (sorted ascending), else NULL: col_offset + local
    cudaGraphConditionalHandle cond;  // rbg_run's device loop (loop_exit), valid when use_cond
    int use_cond;
    int pdl;  // launch as a programmatic dependent of the preceding kernel (k_sweep_dyn only)
    int tail_pf;  // k_sweep_dyn: warps out of columns prefetch the last columns into L2
    unsigned long long *tstamp;  // RBG_DEBUG_IMGS: %globaltimer when the last CTA finished (else NULL)
};

// Column j of the local snapshot block: the caller's matrix for j < M0, the library-owned
// segment of appended columns (enrichment) after it -- so an append never copies S.
__device__ __forceinline__ const double2 *scol(const double2 *S, long long ldv, const double2 *S1, long long M0,
                                               long long nvec, long long j) {
    return j < M0 ? S + j * ldv : S1 + (j - M0) * nvec;
}

// Global index of local column j (sweep records).
__device__ __forceinline__ long long global_col(const SweepArgs &a, long long j) {
    if (j == 0x7fffffffffffffffLL) return j;
    return a.gid ? a.gid[j] : j + a.col_offset;
}

// PEER record tag of the sweep / decision with basis size k.
__host__ __device__ inline unsigned long long peer_tag(unsigned long long epoch, long long k) {
    return (epoch << 32) | (unsigned long long)(k + 1);
}

// Pivot decision + iterated MGS (a3 finalize, a5, a6).
struct ImgsArgs {
    const double2 *S;
    long long ldv;
    const double2 *S1;  // appended columns (see SweepArgs)
    long long M0;
    long long N, nvec;
    const double *w;
    double2 *Q, *WQ;
    long long ldq_v;
    DevState *st;
    double *errors;        // k_max + 1
    long long *piv;        // k_max
    int *nu;               // k_max
    double *rdiag;         // k_max
    double *r2;            // M_loc
    long long k_max;
    double tol;
    long long col_offset, M_loc;
    int world;
    bool xchg;                  // decision from the exchanged records (any world size)
    const unsigned char *recv;  // world slots of xchg_slot_bytes(nvec)
    size_t slot_bytes;
    // PEER exchange: this rank's record array (written by every rank's sweep) and every
    // rank's two send slots (P2P-mapped); NULL otherwise
    const PeerRec *peer_mine;
    const unsigned char *peer_send[kMaxPeers];
    size_t peer_slot;
    const long long *gid;  // as SweepArgs::gid (the owner masks its selected local column)
    long long *trace;      // RBG_DEBUG_IMGS: per-phase clock64 of 32 MGS steps, then the
                           // %globaltimer of the kernel's phases at trace[257..] (else NULL)
    cudaGraphConditionalHandle cond;  // rbg_run's device loop (loop_exit), valid when use_cond
    int use_cond;
    int pdl;  // launch as a programmatic dependent of the preceding sweep (MGS kernel)
    const void *tm;  // host copy of the CUtensorMap of Q for the staged basis pipe, or NULL
    int use_tm;
};

// Local index of global column J on this rank, -1 if another rank owns it.
__device__ __forceinline__ long long local_col(const ImgsArgs &a, long long J) {
    if (!a.gid) {
        const long long jl = J - a.col_offset;
        return (jl >= 0 && jl < a.M_loc) ? jl : -1;
    }
    long long lo = 0, hi = a.M_loc;  // gid is sorted ascending: binary search
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (a.gid[mid] < J) lo = mid + 1;
        else hi = mid;
    }
    return (lo < a.M_loc && a.gid[lo] == J) ? lo : -1;
}

// Pivot decision (a3) from this rank's maxloc, the all-gathered slots (NCCL / EXTERNAL) or the
// PEER records; `src` = the pivot column (local S, a received slot, or the owner's send slot
// over NVLink, read with ld_cv).  Identical bits on every CTA and every rank.
__device__ __forceinline__ void pivot_decision(const ImgsArgs &a, long long k, double &m, long long &J,
                                               const double2 *&src) {
    if (a.peer_mine) {
        const int par = (int)((k + 1) & 1);
        m = -INFINITY;
        J = 0x7fffffffffffffffLL;
        int owner = 0;
        for (int p = 0; p < a.world; p++) {
            const PeerRec *r = a.peer_mine + par * a.world + p;
            const double rm = ld_relaxed_sys_f64(&r->m);
            const long long rj = ld_relaxed_sys_s64(&r->j);
            if (rec_better(rm, rj, m, J)) {
                m = rm;
                J = rj;
                owner = p;
            }
        }
        src = reinterpret_cast<const double2 *>(a.peer_send[owner] + (size_t)par * a.peer_slot + sizeof(Rec));
    } else if (!a.xchg) {
        m = a.st->m_loc;
        J = a.st->j_loc;
        src = scol(a.S, a.ldv, a.S1, a.M0, a.nvec, J - a.col_offset);
    } else {
        m = -INFINITY;
        J = 0x7fffffffffffffffLL;
        int owner = 0;
        for (int p = 0; p < a.world; p++) {
            const Rec *r = reinterpret_cast<const Rec *>(a.recv + (size_t)p * a.slot_bytes);
            if (rec_better(r->m, r->j, m, J)) {
                m = r->m;
                J = r->j;
                owner = p;
            }
        }
        src = reinterpret_cast<const double2 *>(a.recv + (size_t)owner * a.slot_bytes + sizeof(Rec));
    }
}

// PEER exchange wait (a4): until every rank's record of this iteration has arrived (tag), or
// timeout_ns passed (then stop = PEER_TIMEOUT).  One warp; no-op once stopped.
cudaError_t launch_peer_wait(const PeerRec *mine, int world, DevState *st, unsigned long long epoch, long long timeout_ns,
                             cudaGraphConditionalHandle cond, int use_cond, cudaStream_t s);
// Pivot search restart after columns were added to a sharded context: the local maxloc of r2
// (one CTA, the sweep's total order and global indices) into the state, the candidate column
// packed into the send slot and, on a PEER context, the record published to every rank.
cudaError_t launch_restart(const SweepArgs &a, bool cplx, cudaStream_t s);

struct SweepConfig {
    int grid, threads;
    size_t smem;
    bool esmem;  // basis vector staged in shared memory (else read through L1/L2)
    int unroll;  // 16-byte loads in flight per lane (4, 8, 12, 16)
};

SweepConfig sweep_config(bool cplx, bool init, long long nvec, int num_sms, int device);
cudaError_t launch_sweep(const SweepArgs &a, bool cplx, bool init, const SweepConfig &cfg,
                         cudaStream_t s);
int imgs_maxv(long long nvec);  // 0 if unsupported
// The tensor map (one CUtensorMap, 64-byte aligned) of Q for k_imgs' staged basis pipe;
// the basis allocations must extend imgs_basis_pad(nvec) vectors past k_max * ldq_v.
bool make_imgs_maps(const double2 *Q, long long nvec, long long ldq_v, long long k_max, void *map);
inline long long imgs_basis_pad(long long nvec) { return (long long)imgs_maxv(nvec) * kLaneImgs; }
// Hoffmann CGSCI variant (imgs_cgs.cu): cooperative grid, vbuf nvec vectors, cbuf k_max.
int cgs_grid(int num_sms);
cudaError_t launch_imgs_cgs(const ImgsArgs &a, bool cplx, double2 *vbuf, double2 *cbuf, int grid, cudaStream_t s);
cudaError_t launch_imgs(const ImgsArgs &a, bool cplx, cudaStream_t s);
// Explicit mode: V = W^{1/2} S and Q = Q~ / W^{1/2} (sweep.cu).
cudaError_t launch_scale_sqrtw(double2 *V, long long ldv, const double2 *S, long long lds, long long M, long long nvec,
                               long long N, const double *w, bool cplx, cudaStream_t s);
cudaError_t launch_unscale_sqrtw(double2 *Q, const double2 *Qt, long long k, long long nvec, const double *w, bool cplx,
                                 cudaStream_t s);
// WQ = w o Q for basis vectors 0..k-1 (rbg_restore), the IMGS kernel's multiplication.
cudaError_t launch_weight_basis(double2 *WQ, const double2 *Q, long long k, long long ldq_v, long long nvec,
                                const double *w, bool cplx, cudaStream_t s);
// Deterministic maxloc of r2[0..M) (value desc, index asc) into st->m_loc / st->j_loc.
cudaError_t launch_maxloc(const double *r2, long long M, long long col_offset, DevState *st,
                          cudaStream_t s);
// out[j] = sqrt(max(in[j], 0)) (CAC rule 8), j < M.
cudaError_t launch_sqrt_clamp(const double *in, double *out, long long M, cudaStream_t s);
// Algorithm 4 (recon.cu)
struct Rot;
constexpr long long kGramChunk = 4096;  // columns per Gram chunk (R30)
int gram_tile();  // pairs per k_gram tile side
cudaError_t launch_gram(const double *R, long long ldr, int k, long long M, bool cplx, double2 *P, long long chunk,
                        const int4 *items_d, int nitems, cudaStream_t s);
cudaError_t launch_gram_reduce(const double2 *P, long long nchunks, int k, int kp, const double2 *G0, double2 *G,
                               cudaStream_t s);
cudaError_t launch_jacobi(double2 *G, double2 *V, int kp, Rot *rots, unsigned long long *flags, int *sweeps,
                          int num_sms, cudaStream_t s);
cudaError_t launch_eig_sort(const double2 *G, int k, int kp, double tau2, int kr_max, int *order, double *sigma,
                            int *kr, cudaStream_t s);
cudaError_t launch_recon_x(const double2 *Q, long long ldq_v, long long nvec, int k, const double2 *V, int kp,
                           const int *order, int kr, double2 *X, long long ldx_v, bool cplx, cudaStream_t s);
size_t rot_bytes(int kp);
size_t jacobi_scratch_bytes(int kp);  // k_jacobi's per-pair 2 x 2 scratch
// Block Jacobi (k_bjacobi): kp = jacobi_pad(k) (a multiple of 32), scratch U per block pair.
int jacobi_pad(int k);
size_t bjacobi_scratch_bytes(int kp);
cudaError_t launch_bjacobi(double2 *G, double2 *V, int kp, double2 *Us, unsigned long long *flags, int *sweeps,
                           int num_sms, cudaStream_t s, unsigned long long *trace = nullptr);

// Greedy EIM nodes (eim.cu): nodes_d[k], B_d = Q(P, :) k x k column-major complex.
// coeff.cu: C(i, j) = <q_i, v_j>_w for i < k, j < M in one blocked pass over V, then
// r2_j -= |C(i, j)|^2 in order i (r2 may be null); bit-identical to k coefficient sweeps.
bool coeff_block_enabled();
cudaError_t launch_coeff_block(const double2 *V, long long ldv, long long M, const double2 *WQ, long long ldq_v,
                               long long k, long long nvec, long long N, bool cplx, double *C, long long ldc,
                               double *r2, cudaStream_t s);
struct ScratchPool;
cudaError_t run_eim(const double2 *Q, long long ldq_v, long long N, bool cplx, int k, long long *nodes_d, double2 *B_d,
                    int *status_d, cudaStream_t s, ScratchPool *pool = nullptr);

// Device allocations of the library (devmem.cu): cudaMalloc / cudaFree, with a checked
// 256-byte canary tail per buffer while canaries are on (rbg_debug_set_canary).
cudaError_t dmalloc(void **p, size_t bytes);
cudaError_t dfree(void *p);

// Reusable device work buffers of one context (devmem.cu): slot i is (re)allocated through
// dmalloc only when a call needs more than it holds, and freed with the context -- the
// NEXT-row calls (Gram, reconstruction, EIM) would otherwise cudaMalloc / cudaFree their
// buffers on every call (~2 ms of host time per call at k = 300).  Contents are not kept
// between calls; every user initialises what it reads, as with a fresh allocation.
struct ScratchPool {
    static constexpr int kSlots = 24;
    static constexpr size_t kMaxKeep = size_t(1) << 30;   // larger requests are not retained
    void *p[kSlots] = {};
    size_t bytes[kSlots] = {};
    cudaError_t get(int slot, size_t n, void **out);
    bool owns(const void *q) const {
        for (int i = 0; i < kSlots; i++)
            if (q && p[i] == q) return true;
        return false;
    }
    void release();
};
enum ScratchSlot {
    kScGramItems = 0, kScGramP, kScRecG, kScRecV, kScRecRots, kScRecFlags, kScRecSweeps, kScRecOrder,
    kScRecKr, kScRecSig, kScRecX, kScEimNodes, kScEimB, kScEimStatus, kScEimXi, kScEimT, kScEimTt,
    kScEimC, kScEimBm, kScEimBj, kScEimTicket, kScValR, kScValE2, kScValE
};
bool scratch_disabled();   // RBG_NO_SCRATCH: every work buffer from dmalloc, freed per call (A/B)
// The pool's slot, or a fresh dmalloc without a pool or above kMaxKeep; every salloc is paired
// with an sfree, which frees only what the pool does not hold.
template <class T>
cudaError_t salloc(ScratchPool *pool, int slot, T **p, size_t bytes) {
    void *q = nullptr;
    cudaError_t e = (pool && bytes <= ScratchPool::kMaxKeep && !scratch_disabled()) ? pool->get(slot, bytes, &q)
                                                                                     : dmalloc(&q, bytes);
    *p = static_cast<T *>(q);
    return e;
}
inline void sfree(ScratchPool *pool, void *p) {
    if (!pool || !pool->owns(p)) dfree(p);
}
template <class T>
inline cudaError_t dmalloc(T **p, size_t bytes) {
    return dmalloc(reinterpret_cast<void **>(p), bytes);
}
void debug_set_canary(bool on);
long long debug_canary_violations(std::string *msg);

// First non-finite entry of a device block: atomicMin of (col0 + col) * N + row into *out
// (which the caller sets to ~0 first).
cudaError_t launch_check_finite(const double2 *S, long long ldv, long long M, long long N,
                                long long nvec, bool cplx, unsigned long long *out,
                                cudaStream_t s, long long col0 = 0);

}  // namespace rbg
