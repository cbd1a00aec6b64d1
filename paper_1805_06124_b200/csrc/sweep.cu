// sweep.cu -- the fused column sweep: the pivot-search half of each RB-greedy iteration.
//
// PAPER.md:838-868 (Sec. 6.1.2): every iteration computes, for all M columns, the
// coefficient c_kj = <q_k, s_j> and the residual recurrence of Eq. (Residual)
//     sigma_hat_k^2(s_j) = ||s_j||^2 - sum_{i<=k} |c_ij|^2,
// then the argmax over j.  "The j-th pivot search has a constant complexity with an
// asymptotic FLOP count of O(2MN)" -- it streams all of S once and is HBM-bound.
//
// B200 design:
//  * one CTA per SM, 16 warps; the default kernel (k_sweep_dyn) hands columns to warps
//    dynamically (a grid-wide counter claimed one column ahead); k_sweep (the explicit-
//    residual mode's kernel, RBG_SWEEP_KIND=percol) gives each CTA a contiguous block;
//  * the weighted basis vector e~_k = w o q_k (N x 16 B, 160 KB at N = 10,000 complex) is
//    staged once per CTA into shared memory with TMA bulk copies (cp.async.bulk) on an
//    mbarrier;
//  * one warp per column (L_S = 32 lanes): lane l owns the 16-byte vectors u = l (mod 32)
//    of the column, streamed with 16-byte ld.global.nc.L1::no_allocate + L2 evict-first
//    through a register ring of U loads in flight per lane (U = 16 on the 10,000-row case:
//    128 KB outstanding per SM; the ring runs across column boundaries), accumulated with
//    explicit fma() in increasing u;
//  * xor-butterfly with ascending offsets (= the pairwise lane tree of the CAC);
//  * lane 0 writes R(k, j), updates r2_j in place, and the warp keeps its maxloc;
//  * per-CTA maxloc records, the last CTA to finish (atomic ticket) reduces them with the
//    total order (value desc, index asc) into the device state, and on a sharded run packs
//    the local candidate column into the exchange slot.
// Sweep 0 (INIT) is the same kernel with e~ = w and the weighted norm of CAC rule 4.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "kernels.h"

namespace rbg {

constexpr int kSweepThreads = 512;
constexpr int kSweepWarps = kSweepThreads / 32;
constexpr size_t kSmemLimit = 220 * 1024;
constexpr uint32_t kBulkChunk = 32 * 1024;

// Accumulate one 16-byte vector x of a column against the staged vector e (CAC rules 2, 4).
template <bool CPLX, bool INIT>
__device__ __forceinline__ void accum(double &re, double &im, const double2 x, const double2 e) {
    if (INIT) {
        // e = (w_{2u}, w_{2u+1}) for real, (w_u, -) for complex
        if (CPLX) {
            double t = e.x * x.x;
            re = fma(t, x.x, re);
            t = e.x * x.y;
            re = fma(t, x.y, re);
        } else {
            double t = e.x * x.x;
            re = fma(t, x.x, re);
            t = e.y * x.y;
            re = fma(t, x.y, re);
        }
    } else {
        if (CPLX) {
            re = fma(e.x, x.x, re);
            re = fma(e.y, x.y, re);
            im = fma(e.x, x.y, im);
            im = fma(-e.y, x.x, im);
        } else {
            re = fma(e.x, x.x, re);
            re = fma(e.y, x.y, re);
        }
    }
}

template <bool CPLX, bool INIT, bool ESMEM>
__device__ __forceinline__ double2 load_e(const double2 *E, const double *Ew, long long u) {
    if (INIT && CPLX) {
        // complex sweep 0 reads one weight per vector
        double wv = ESMEM ? Ew[u] : __ldg(Ew + u);
        return make_double2(wv, 0.0);
    }
    return ESMEM ? E[u] : __ldg(E + u);
}

// This sweep's send slot: PEER keeps two (by the parity of the record tag st->k + 1), so a
// slot is rewritten only after every peer has consumed it.
__device__ __forceinline__ unsigned char *send_slot(const SweepArgs &a) {
    if (a.peer_world == 0) return a.send;
    return a.send + (size_t)((a.st->k + 1) & 1) * a.peer_slot;
}

// CTA maxloc of the warps' bests, then the last CTA to finish (atomic ticket) reduces the
// per-CTA records with the total order into the device state and, on a sharded run, packs
// the local candidate column into the exchange slot.
template <bool CPLX>
__device__ __forceinline__ void sweep_finish(const SweepArgs &a, double best_m, long long best_j, bool odd_tail) {
    __shared__ double s_m[kSweepWarps];
    __shared__ long long s_j[kSweepWarps];
    __shared__ int s_last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long nvec = a.nvec;
    if (lane == 0) {
        s_m[warp] = best_m;
        s_j[warp] = best_j;
    }
    __syncthreads();
    if (tid == 0) {
        double bm = s_m[0];
        long long bj = s_j[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); w++)
            if (rec_better(s_m[w], s_j[w], bm, bj)) {
                bm = s_m[w];
                bj = s_j[w];
            }
        a.recs[blockIdx.x].m = bm;
        a.recs[blockIdx.x].j = bj;
        __threadfence();
        const unsigned t = atomicAdd(a.ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp == 0) {
        double bm = -INFINITY;
        long long bj = 0x7fffffffffffffffLL;
        for (int b = lane; b < (int)gridDim.x; b += 32) {
            const double m = __ldcg(&a.recs[b].m);
            const long long j = __ldcg(&a.recs[b].j);
            if (rec_better(m, j, bm, bj)) {
                bm = m;
                bj = j;
            }
        }
#pragma unroll
        for (int h = 16; h >= 1; h >>= 1) {  // exact: total order, any combine order
            const double om = __shfl_xor_sync(0xffffffffu, bm, h);
            const long long oj = __shfl_xor_sync(0xffffffffu, bj, h);
            if (rec_better(om, oj, bm, bj)) {
                bm = om;
                bj = oj;
            }
        }
        if (lane == 0) {
            const long long jg = global_col(a, bj);
            a.st->m_loc = bm;
            a.st->j_loc = jg;
            if (a.tstamp) *a.tstamp = globaltimer_ns();
            *a.ticket = 0u;
            if (a.next_col) *a.next_col = 0ull;  // every warp has taken its last column
            if (a.send) {
                Rec *h = reinterpret_cast<Rec *>(send_slot(a));
                h->m = bm;
                h->j = jg;
            }
            s_m[1] = bm;
            s_j[1] = jg;
            if (!a.send && bj >= 0 && bj < a.M) {
                // one GPU: the decision kernel's first read is this column (streamed with
                // evict-first a while ago): pull it into L2 now (16-byte aligned, whole column)
                const char *col = reinterpret_cast<const char *>(scol(a.S, a.ldv, a.S1, a.M0, a.nvec, bj));
                const size_t bytes = (size_t)nvec * 16;
                for (size_t off = 0; off < bytes; off += 32768)
                    prefetch_l2(col + off, (uint32_t)((bytes - off) < 32768 ? (bytes - off) : 32768));
            }
        }
        if (a.send) s_j[0] = bj;
    }
    if (a.send) {  // pack the local candidate column for the all-gather / the peers
        __syncthreads();
        const long long bj = s_j[0];
        double2 *dst = reinterpret_cast<double2 *>(send_slot(a) + sizeof(Rec));
        const bool valid = bj >= 0 && bj < a.M;
        for (long long u = tid; u < nvec; u += blockDim.x) {
            double2 x = valid ? scol(a.S, a.ldv, a.S1, a.M0, a.nvec, bj)[u] : make_double2(0.0, 0.0);
            if (odd_tail && u == nvec - 1) x.y = 0.0;
            dst[u] = x;
        }
        if (a.peer_world > 0) {
            // PEER: the column is in place (CTA barrier), make it and the record visible to
            // every GPU, then publish the record in every rank's array and release the tag
            __syncthreads();
            if (tid == 0) {
                const unsigned long long tag = peer_tag(a.peer_epoch, a.st->k);
                const int par = (int)((a.st->k + 1) & 1);
                __threadfence_system();
                for (int q = 0; q < a.peer_world; q++) {
                    PeerRec *r = a.peer_in[q] + par * a.peer_world + a.peer_rank;
                    st_relaxed_sys_f64(&r->m, s_m[1]);
                    st_relaxed_sys_s64(&r->j, s_j[1]);
                    st_release_sys(&r->tag, tag);
                }
            }
        }
    }
}

template <bool CPLX, bool INIT, bool ESMEM, int U>
__global__ void __launch_bounds__(kSweepThreads, 1) k_sweep(const SweepArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t mbar;

    const int stop = a.st->stop;
    if (stop) {
        if (threadIdx.x == 0 && blockIdx.x == 0) loop_exit(a.cond, a.use_cond);
        return;
    }
    // sweep uses q_{k-1} (k >= 1) unless INIT; a validation pass names its basis vector
    const long long k = a.qi >= 0 ? a.qi + 1 : a.st->k;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long nvec = a.nvec;
    const bool odd_tail = !CPLX && (a.N & 1);

    // ---- stage e~ (w o q_{k-1}, or w for sweep 0) ------------------------------------
    const double2 *Eg = INIT ? reinterpret_cast<const double2 *>(a.w) : a.WQ + (k - 1) * a.ldq_v;
    const double2 *E = Eg;
    const double *Ew = a.w;
    if (ESMEM) {
        const size_t bytes = (INIT && CPLX) ? ((size_t)nvec * 8 + 15) / 16 * 16 : (size_t)nvec * 16;
        if (tid == 0) {
            mbar_init(&mbar, 1);
            mbar_arrive_expect_tx(&mbar, (uint32_t)bytes);
            const unsigned char *src = reinterpret_cast<const unsigned char *>(Eg);
            for (size_t off = 0; off < bytes; off += kBulkChunk) {
                uint32_t n = (uint32_t)((bytes - off) < kBulkChunk ? (bytes - off) : kBulkChunk);
                bulk_g2s(smem + off, src + off, n, &mbar);
            }
        }
        __syncthreads();
        E = reinterpret_cast<const double2 *>(smem);
        Ew = reinterpret_cast<const double *>(smem);
    }

    // ---- columns of this CTA ------------------------------------------------------
    const long long c_begin = (long long)blockIdx.x * a.M / gridDim.x;
    const long long c_end = (long long)(blockIdx.x + 1) * a.M / gridDim.x;
    // explicit mode re-reads each column right after its first pass: keep the first pass's
    // lines in L2 (evict-last) and demote them on the re-read and the write-back (evict-first)
    const uint64_t pol = a.V ? policy_evict_last() : policy_evict_first();
    const uint64_t pol_done = policy_evict_first();

    double best_m = -INFINITY;
    long long best_j = 0x7fffffffffffffffLL;
    bool waited = !ESMEM;

    for (long long c = c_begin + warp; c < c_end; c += kSweepWarps) {
        const double2 *col = scol(a.S, a.ldv, a.S1, a.M0, a.nvec, c);
        double re = 0.0, im = 0.0;
        // ring of U 16-byte loads in flight per lane: slot t is consumed, then immediately
        // refilled with the vector U*32 further down the column
        double2 xr[U];
#pragma unroll
        for (int t = 0; t < U; t++) {
            const long long u = (long long)t * 32 + lane;
            xr[t] = (u < nvec) ? ld_stream(col + u, pol) : make_double2(0.0, 0.0);
        }
        if (!waited) {  // first column: loads are in flight, now wait for e~
            mbar_wait(&mbar, 0);
            waited = true;
        }
        for (long long base = 0; base < nvec; base += 32 * U) {
#pragma unroll
            for (int t = 0; t < U; t++) {
                const long long u = base + (long long)t * 32 + lane;
                double2 x = xr[t];
                const long long un = u + 32 * U;
                xr[t] = (un < nvec) ? ld_stream(col + un, pol) : make_double2(0.0, 0.0);
                if (u < nvec) {
                    if (odd_tail && u == nvec - 1) x.y = 0.0;  // row N is padding
                    accum<CPLX, INIT>(re, im, x, load_e<CPLX, INIT, ESMEM>(E, Ew, u));
                }
            }
        }
        // lane tree, ascending offsets (CAC rule 3)
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) {
            re = re + __shfl_xor_sync(0xffffffffu, re, h);
            if (CPLX && !INIT) im = im + __shfl_xor_sync(0xffffffffu, im, h);
        }
        double r2n;
        if (INIT) {
            r2n = re;
            if (lane == 0) a.r2[c] = r2n;
        } else if (a.V) {
            // explicit residuals (Algorithm 2, DESIGN.md CAC rule 12): v_j <- v_j - c q~_k in
            // place and r2_j = ||v_j||^2 recomputed from the updated column (second pass)
            const double old = a.r2[c];
            if (lane == 0) {
                if (CPLX) reinterpret_cast<double2 *>(a.R)[(k - 1) * a.ldr + c] = make_double2(re, im);
                else a.R[(k - 1) * a.ldr + c] = re;
            }
            r2n = old;
            if (old != -INFINITY) {
                double2 *vcol = a.V + c * a.ldv;
                double acc = 0.0;
                for (long long base = 0; base < nvec; base += 32 * 8) {
                    double2 xv[8];
#pragma unroll
                    for (int t = 0; t < 8; t++) {
                        const long long u = base + (long long)t * 32 + lane;
                        xv[t] = (u < nvec) ? ld_keep(vcol + u, pol_done) : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int t = 0; t < 8; t++) {
                        const long long u = base + (long long)t * 32 + lane;
                        if (u < nvec) {
                            double2 x = xv[t];
                            const double2 e = load_e<CPLX, false, ESMEM>(E, Ew, u);  // q~_k (w = 1)
                            if (CPLX) {
                                double xr = x.x, xi = x.y;
                                xr = fma(-re, e.x, xr);
                                xr = fma(im, e.y, xr);
                                xi = fma(-re, e.y, xi);
                                xi = fma(-im, e.x, xi);
                                x = make_double2(xr, xi);
                            } else {
                                x.x = fma(-re, e.x, x.x);
                                x.y = fma(-re, e.y, x.y);
                            }
                            if (odd_tail && u == nvec - 1) x.y = 0.0;
                            st_keep(vcol + u, x, pol_done);
                            acc = fma(x.x, x.x, acc);
                            acc = fma(x.y, x.y, acc);
                        }
                    }
                }
#pragma unroll
                for (int h = 1; h < 32; h <<= 1) acc = acc + __shfl_xor_sync(0xffffffffu, acc, h);
                r2n = acc;
            }
            if (lane == 0) a.r2[c] = r2n;
        } else {
            const double cc = CPLX ? fma(re, re, im * im) : re * re;  // CAC rule 5
            const double old = a.r2[c];
            r2n = old - cc;                                            // CAC rule 6
            if (lane == 0) {
                if (CPLX) {
                    reinterpret_cast<double2 *>(a.R)[(k - 1) * a.ldr + c] = make_double2(re, im);
                } else {
                    a.R[(k - 1) * a.ldr + c] = re;
                }
                a.r2[c] = r2n;
            }
        }
        if (r2n > best_m) {  // columns visited in increasing order: first max wins
            best_m = r2n;
            best_j = c;
        }
    }
    if (!waited) mbar_wait(&mbar, 0);  // never leave with a bulk copy in flight

    sweep_finish<CPLX>(a, best_m, best_j, odd_tail);
}

// Pivot search restart (sharded rbg_add_columns_ex): one CTA; thread t scans r2[t], r2[t + T],
// ... (increasing index: first max wins), warp maxloc, then sweep_finish (grid of one CTA: it
// is the last CTA) writes the state, packs the candidate and publishes the PEER record.
template <bool CPLX>
__global__ void __launch_bounds__(kSweepThreads, 1) k_restart(const SweepArgs a) {
    double bm = -INFINITY;
    long long bj = 0x7fffffffffffffffLL;
    for (long long j = threadIdx.x; j < a.M; j += blockDim.x) {
        const double m = a.r2[j];
        if (m > bm) {
            bm = m;
            bj = j;
        }
    }
    for (int h = 16; h >= 1; h >>= 1) {  // exact: total order
        const double om = __shfl_xor_sync(0xffffffffu, bm, h);
        const long long oj = __shfl_xor_sync(0xffffffffu, bj, h);
        if (rec_better(om, oj, bm, bj)) {
            bm = om;
            bj = oj;
        }
    }
    sweep_finish<CPLX>(a, bm, bj, !CPLX && (a.N & 1));
}

cudaError_t launch_restart(const SweepArgs &a, bool cplx, cudaStream_t s) {
    if (cplx) k_restart<true><<<1, kSweepThreads, 0, s>>>(a);
    else k_restart<false><<<1, kSweepThreads, 0, s>>>(a);
    return cudaGetLastError();
}

// Dynamically scheduled ring sweep (default for the recurrence): a ring of U loads in flight per
// lane that runs across column boundaries, and a warp's columns come from a grid-wide counter
// instead of a static block, so SMs that stream
// faster take more columns (ncu on the static kernel: SMs active 91.8-100 % of the launch,
// 95.6 % on average).  The first column of a warp is its global warp index; each later one is
// one atomicAdd (lane 0) taken a column ahead of use, so its latency never stalls the ring.  A
// warp's columns increase, so "first max wins" keeps the lowest index among a warp's ties and
// the CTA / grid maxloc uses the total order: results are bit-identical to k_sweep.  The
// counter (a.next_col) returns to 0 in the last CTA.
template <bool CPLX, bool INIT, bool ESMEM, int U>
__global__ void __launch_bounds__(kSweepThreads, 1) k_sweep_dyn(const SweepArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t mbar;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long nvec = a.nvec;
    const bool odd_tail = !CPLX && (a.N & 1);
    const uint64_t pol = policy_evict_first();
    const int nv = (int)nvec;
    const long long M = a.M;
    // the first column of this warp and its first group of U loads: the snapshot matrix is
    // never written by the greedy, so with a programmatic dependent launch these loads are in
    // flight while the predecessor (the decision / IMGS kernel) is still running
    long long colA = (long long)blockIdx.x * kSweepWarps + warp;
    double2 xr[U];
    {
        const double2 *lp = scol(a.S, a.ldv, a.S1, a.M0, a.nvec, colA) + lane;
#pragma unroll
        for (int t = 0; t < U; t++)
            xr[t] = (colA < M && t * 32 + lane < nv) ? ld_stream(lp + t * 32, pol) : make_double2(0.0, 0.0);
    }
    grid_dep_wait();  // the state, q_{k-1}, r2 and the column counter are the predecessor's
    if (a.st->stop) {
        if (threadIdx.x == 0 && blockIdx.x == 0) loop_exit(a.cond, a.use_cond);
        return;
    }
    grid_dep_launch();
    const long long k = a.qi >= 0 ? a.qi + 1 : a.st->k;

    const double2 *Eg = INIT ? reinterpret_cast<const double2 *>(a.w) : a.WQ + (k - 1) * a.ldq_v;
    const double2 *E = Eg;
    const double *Ew = a.w;
    if (ESMEM) {
        const size_t bytes = (INIT && CPLX) ? ((size_t)nvec * 8 + 15) / 16 * 16 : (size_t)nvec * 16;
        if (tid == 0) {
            mbar_init(&mbar, 1);
            mbar_arrive_expect_tx(&mbar, (uint32_t)bytes);
            const unsigned char *src = reinterpret_cast<const unsigned char *>(Eg);
            for (size_t off = 0; off < bytes; off += kBulkChunk) {
                uint32_t n = (uint32_t)((bytes - off) < kBulkChunk ? (bytes - off) : kBulkChunk);
                bulk_g2s(smem + off, src + off, n, &mbar);
            }
        }
        __syncthreads();
        E = reinterpret_cast<const double2 *>(smem);
        Ew = reinterpret_cast<const double *>(smem);
    }

    const int gpc = (int)((nvec + 32 * U - 1) / (32 * U));  // groups of U trips per column
    const long long nwg = (long long)gridDim.x * kSweepWarps;
    // column window of this warp: A = being consumed, B = next, pend = the one after (raw
    // counter value held by lane 0, shuffled out only at the next shift)
    unsigned long long raw = 0;
    if (lane == 0) raw = atomicAdd(a.next_col, 1ull);
    long long colB = (long long)__shfl_sync(0xffffffffu, raw, 0) + nwg;
    unsigned long long praw = 0;
    if (lane == 0) praw = atomicAdd(a.next_col, 1ull);

    // the issue cursor is always exactly one group ahead of the consume cursor (group cg of
    // colA): group cg + 1 of colA, or group 0 of colB when cg is colA's last group (group 0 of
    // colA was issued before grid_dep_wait)
    if (ESMEM) mbar_wait(&mbar, 0);

    double best_m = -INFINITY;
    long long best_j = 0x7fffffffffffffffLL;
    double re = 0.0, im = 0.0;
    int cg = 0;
    double old = (!INIT && colA < M) ? a.r2[colA] : 0.0;

    while (colA < M) {
        const bool last = cg + 1 == gpc;
        const long long lc = last ? colB : colA;
        const int lgrp = last ? 0 : cg + 1;
        const int lu0 = lgrp * 32 * U + lane;
        const int cu0 = cg * 32 * U + lane;
        const double2 *lp = scol(a.S, a.ldv, a.S1, a.M0, a.nvec, lc) + lu0;
        const bool lvalid = lc < M;
#pragma unroll
        for (int t = 0; t < U; t++) {
            double2 x = xr[t];
            xr[t] = (lvalid && lu0 + t * 32 < nv) ? ld_stream(lp + t * 32, pol) : make_double2(0.0, 0.0);
            const int u = cu0 + t * 32;
            if (u < nv) {
                if (odd_tail && u == nv - 1) x.y = 0.0;  // row N is padding
                accum<CPLX, INIT>(re, im, x, load_e<CPLX, INIT, ESMEM>(E, Ew, u));
            }
        }
        if (!last) {
            cg++;
            continue;
        }
        // column colA complete (warp-uniform)
        cg = 0;
        const long long c = colA;
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) {  // CAC rule 3
            re = re + __shfl_xor_sync(0xffffffffu, re, h);
            if (CPLX && !INIT) im = im + __shfl_xor_sync(0xffffffffu, im, h);
        }
        double r2n;
        if (INIT) {
            r2n = re;
            if (lane == 0) a.r2[c] = r2n;
        } else {
            const double cc = CPLX ? fma(re, re, im * im) : re * re;  // CAC rule 5
            r2n = old - cc;                                            // CAC rule 6
            if (lane == 0) {
                if (CPLX) reinterpret_cast<double2 *>(a.R)[(k - 1) * a.ldr + c] = make_double2(re, im);
                else a.R[(k - 1) * a.ldr + c] = re;
                a.r2[c] = r2n;
            }
            old = colB < M ? a.r2[colB] : 0.0;
        }
        if (r2n > best_m) {  // a warp's columns increase: first max wins
            best_m = r2n;
            best_j = c;
        }
        re = 0.0;
        im = 0.0;
        // shift the window: B becomes current, the pending column becomes B, take a new one
        colA = colB;
        colB = (long long)__shfl_sync(0xffffffffu, praw, 0) + nwg;
        if (lane == 0) praw = atomicAdd(a.next_col, 1ull);
    }
    // Tail: this warp's column claims are exhausted; colA is its first claim past M (claims are
    // handed out in order, so X = colA - M earlier claims were also past M).  The columns claimed
    // last, M-1, M-2, ..., are being started by their warps about now, and a lone warp streams
    // a column at its latency-bound rate: pull column 2M-1-colA (one per exhausted claim, the
    // last claimed first) into L2 so its owner's loads hit L2.  No arithmetic changes.
    // Only for columns of <= 64 KB (configs 0, 1, 4: a column is a few us of one warp's stream):
    // on config 2's 160 KB columns the owners are mid-column by then and a whole-column prefetch
    // re-reads their first part (ncu: +110 MB per sweep, no gain).
    if (a.tail_pf && lane == 0 && nvec * 16 <= 65536) {
        const long long P = 2 * M - 1 - colA;
        if (P >= 0 && P < M && P >= M - nwg) {
            const char *col = reinterpret_cast<const char *>(scol(a.S, a.ldv, a.S1, a.M0, a.nvec, P));
            const uint32_t bytes = (uint32_t)(nvec * 16);
            for (uint32_t off = 0; off < bytes; off += 32768)
                prefetch_l2(col + off, (bytes - off) < 32768u ? (bytes - off) : 32768u);
        }
    }
    sweep_finish<CPLX>(a, best_m, best_j, odd_tail);
}

SweepConfig sweep_config(bool cplx, bool init, long long nvec, int num_sms, int device) {
    SweepConfig c;
    c.threads = kSweepThreads;
    const size_t ebytes = (init && cplx) ? ((size_t)nvec * 8 + 15) / 16 * 16 : (size_t)nvec * 16;
    c.esmem = ebytes <= kSmemLimit;
    c.smem = c.esmem ? ebytes : 0;
    // at most two CTAs per SM when the staged vector is small enough; launch_t clamps this to
    // the kernel's real occupancy (a 512-thread CTA at 128 registers fills the register file)
    int per_sm = 1;
    if (c.smem * 2 + 4096 <= 227 * 1024) per_sm = 2;
    (void)device;
    c.grid = num_sms * per_sm;
    // loads in flight per lane: 16 (128 KB per SM outstanding) for the dynamically scheduled
    // ring (7.43-7.45 vs 7.42 TB/s for 12, profiles/r01/sweep_dyn_tuning.jsonl); the explicit
    // mode's per-column kernel caps it at 12
    const long long trips = (nvec + 31) / 32;
    c.unroll = trips >= 16 ? 16 : (trips >= 12 ? 12 : (trips >= 8 ? 8 : 4));
    if (const char *env = getenv("RBG_SWEEP_UNROLL")) {
        const int u = atoi(env);
        if (u == 4 || u == 8 || u == 12 || u == 16) c.unroll = u;
    }
    return c;
}

using SweepKernel = void (*)(const SweepArgs);

template <bool CPLX, bool INIT, bool ESMEM, int U>
static SweepKernel pick_kernel(bool dyn) {
    // the explicit mode (a.V) re-reads and rewrites each column: per-column loop of k_sweep;
    // the recurrence: the dynamically scheduled ring (k_sweep_dyn)
    return dyn ? k_sweep_dyn<CPLX, INIT, ESMEM, U> : k_sweep<CPLX, INIT, ESMEM, U>;
}

// CTAs of `kern` that fit on the device at once (occupancy x SMs), cached per kernel and
// shared-memory size; `cap` if the query fails.
static int resident_ctas(const void *kern, int threads, size_t smem, int cap) {
    static std::mutex mu;
    static std::map<std::pair<const void *, size_t>, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(kern, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int dev = 0, sms = 0, occ = 0;
    int r = cap;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) == cudaSuccess && occ > 0)
        r = sms * occ;
    cache[key] = r;
    return r;
}

template <bool CPLX, bool INIT, bool ESMEM>
static cudaError_t launch_t(const SweepArgs &a, const SweepConfig &cfg, cudaStream_t s) {
    // RBG_SWEEP_KIND = dyn (default) | percol (k_sweep, static column blocks; the explicit mode's kernel)
    const char *kind = getenv("RBG_SWEEP_KIND");
    const bool dyn = a.V == nullptr && a.next_col != nullptr && !(kind && std::strcmp(kind, "percol") == 0);
    auto kern = pick_kernel<CPLX, INIT, ESMEM, 4>(dyn);
    const int unroll = (a.V && cfg.unroll > 12) ? 12 : cfg.unroll;
    switch (unroll) {
        case 8: kern = pick_kernel<CPLX, INIT, ESMEM, 8>(dyn); break;
        case 12: kern = pick_kernel<CPLX, INIT, ESMEM, 12>(dyn); break;
        case 16: kern = pick_kernel<CPLX, INIT, ESMEM, 16>(dyn); break;
        default: break;
    }
    if (cfg.smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)cfg.smem);
        if (e != cudaSuccess) return e;
    }
    // no more CTAs than the columns can occupy (one warp per column at least): a small M
    // does not pay 296 CTAs' staging of e~ and a 296-record maxloc (same bits: the per-column
    // arithmetic does not depend on the grid and the maxloc is a total order); and no more than
    // one wave: CTAs of a second wave would find the dynamic column counter exhausted
    const long long need = (a.M + kSweepWarps - 1) / kSweepWarps;
    int grid = (int)(need < 1 ? 1 : (need < cfg.grid ? need : cfg.grid));
    grid = std::min(grid, resident_ctas((const void *)kern, cfg.threads, cfg.smem, cfg.grid));
    if (!(a.pdl && dyn && !INIT)) {
        kern<<<grid, cfg.threads, cfg.smem, s>>>(a);
        return cudaGetLastError();
    }
    // programmatic dependent launch: the first loads of S are issued while the preceding
    // decision / IMGS kernel finishes (k_sweep_dyn waits for it in grid_dep_wait)
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid, 1, 1);
    lc.blockDim = dim3(cfg.threads, 1, 1);
    lc.dynamicSmemBytes = cfg.smem;
    lc.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&lc, kern, a);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_sweep(const SweepArgs &a, bool cplx, bool init, const SweepConfig &cfg,
                         cudaStream_t s) {
    if (cplx) {
        if (init) return cfg.esmem ? launch_t<true, true, true>(a, cfg, s) : launch_t<true, true, false>(a, cfg, s);
        return cfg.esmem ? launch_t<true, false, true>(a, cfg, s) : launch_t<true, false, false>(a, cfg, s);
    }
    if (init) return cfg.esmem ? launch_t<false, true, true>(a, cfg, s) : launch_t<false, true, false>(a, cfg, s);
    return cfg.esmem ? launch_t<false, false, true>(a, cfg, s) : launch_t<false, false, false>(a, cfg, s);
}

// ------------------------------------------------------------------ explicit-mode helpers
// V = W^{1/2} S (per real component, sqrt(w_i) rounded once): the explicit mode works on the
// unweighted problem for S~ (reading R6).  V, S: M columns of nvec vectors (strides ldv, lds).
__global__ void k_scale_sqrtw(double2 *V, long long ldv, const double2 *S, long long lds, long long M,
                              long long nvec, long long N, const double *w, bool cplx) {
    const long long total = M * nvec;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const long long c = t / nvec, u = t - c * nvec;
        const double2 x = S[c * lds + u];
        double2 y;
        if (cplx) {
            const double r = sqrt(w[u]);
            y = make_double2(r * x.x, r * x.y);
        } else {
            y = make_double2(sqrt(w[2 * u]) * x.x, 2 * u + 1 < N ? sqrt(w[2 * u + 1]) * x.y : 0.0);
        }
        V[c * ldv + u] = y;
    }
}

cudaError_t launch_scale_sqrtw(double2 *V, long long ldv, const double2 *S, long long lds, long long M, long long nvec,
                               long long N, const double *w, bool cplx, cudaStream_t s) {
    k_scale_sqrtw<<<148 * 8, 256, 0, s>>>(V, ldv, S, lds, M, nvec, N, w, cplx);
    return cudaGetLastError();
}

// Q = Q~ / sqrt(w) per real component (the W-orthonormal basis of the explicit mode).
__global__ void k_unscale_sqrtw(double2 *Q, const double2 *Qt, long long k, long long nvec, const double *w, bool cplx) {
    const long long total = k * nvec;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const long long u = t % nvec;
        const double2 x = Qt[t];
        if (cplx) {
            const double r = sqrt(w[u]);
            Q[t] = make_double2(x.x / r, x.y / r);
        } else {
            // padding rows carry w = 0: keep them zero
            const double r0 = sqrt(w[2 * u]), r1 = sqrt(w[2 * u + 1]);
            Q[t] = make_double2(x.x / r0, r1 > 0.0 ? x.y / r1 : 0.0);
        }
    }
}

cudaError_t launch_unscale_sqrtw(double2 *Q, const double2 *Qt, long long k, long long nvec, const double *w, bool cplx,
                                 cudaStream_t s) {
    k_unscale_sqrtw<<<148 * 4, 256, 0, s>>>(Q, Qt, k, nvec, w, cplx);
    return cudaGetLastError();
}

// WQ = w o Q for k basis vectors (rbg_restore): per component the one multiplication the IMGS
// kernel performs when it stores q_{k+1} and w o q_{k+1}, so the bits are the ones IMGS writes.
__global__ void k_weight_basis(double2 *WQ, const double2 *Q, long long k, long long ldq_v, long long nvec,
                               const double *w, bool cplx) {
    const long long total = k * nvec;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const long long i = t / nvec, u = t - i * nvec;
        const double2 q = Q[i * ldq_v + u];
        WQ[i * ldq_v + u] = cplx ? make_double2(w[u] * q.x, w[u] * q.y) : make_double2(w[2 * u] * q.x, w[2 * u + 1] * q.y);
    }
}

cudaError_t launch_weight_basis(double2 *WQ, const double2 *Q, long long k, long long ldq_v, long long nvec,
                                const double *w, bool cplx, cudaStream_t s) {
    k_weight_basis<<<148 * 4, 256, 0, s>>>(WQ, Q, k, ldq_v, nvec, w, cplx);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ maxloc / sqrt helpers
// Used when columns are added to a context (enrichment): the pivot search over the whole
// residual vector without a sweep.  One CTA, total order, exact.
__global__ void __launch_bounds__(1024) k_maxloc(const double *r2, long long M, long long col_offset,
                                                 DevState *st) {
    __shared__ double s_m[32];
    __shared__ long long s_j[32];
    double bm = -INFINITY;
    long long bj = 0x7fffffffffffffffLL;
    for (long long j = threadIdx.x; j < M; j += blockDim.x) {
        const double m = r2[j];
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
    if ((threadIdx.x & 31) == 0) {
        s_m[threadIdx.x >> 5] = bm;
        s_j[threadIdx.x >> 5] = bj;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++)
            if (rec_better(s_m[w], s_j[w], bm, bj)) {
                bm = s_m[w];
                bj = s_j[w];
            }
        st->m_loc = bm;
        st->j_loc = (bj == 0x7fffffffffffffffLL) ? bj : bj + col_offset;
    }
}

cudaError_t launch_maxloc(const double *r2, long long M, long long col_offset, DevState *st, cudaStream_t s) {
    k_maxloc<<<1, 1024, 0, s>>>(r2, M, col_offset, st);
    return cudaGetLastError();
}

__global__ void k_sqrt_clamp(const double *in, double *out, long long M) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < M; j += (long long)gridDim.x * blockDim.x)
        out[j] = sqrt(fmax(in[j], 0.0));
}

cudaError_t launch_sqrt_clamp(const double *in, double *out, long long M, cudaStream_t s) {
    const long long blocks = (M + 255) / 256;
    k_sqrt_clamp<<<(unsigned)(blocks < 4096 ? (blocks > 0 ? blocks : 1) : 4096), 256, 0, s>>>(in, out, M);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ finiteness scan
__global__ void k_check_finite(const double2 *S, long long ldv, long long M, long long N,
                               long long nvec, bool cplx, unsigned long long *out, long long col0) {
    const long long total = M * nvec;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long c = t / nvec, u = t - c * nvec;
        const double2 x = S[c * ldv + u];
        long long row0 = cplx ? u : 2 * u;
        bool bad0 = !isfinite(x.x), bad1 = !isfinite(x.y);
        if (!cplx && row0 + 1 >= N) bad1 = false;  // padding row
        if (bad0 || bad1) {
            const long long row = cplx ? u : (bad0 ? row0 : row0 + 1);
            atomicMin(out, (unsigned long long)((c + col0) * N + row));
        }
    }
}

cudaError_t launch_check_finite(const double2 *S, long long ldv, long long M, long long N,
                                long long nvec, bool cplx, unsigned long long *out,
                                cudaStream_t s, long long col0) {
    k_check_finite<<<148 * 8, 256, 0, s>>>(S, ldv, M, N, nvec, cplx, out, col0);
    return cudaGetLastError();
}

}  // namespace rbg
