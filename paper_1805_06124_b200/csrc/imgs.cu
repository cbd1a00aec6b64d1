// imgs.cu -- pivot decision + iterated modified Gram-Schmidt (the orthogonalisation half).
//
// PAPER.md:871-883 (Sec. 6.1.2): "the newly selected pivot column is orthogonalized with
// respect to the existing basis set ... We use the iterative modified Gram-Schmidt (IMGS)
// algorithm of Hoffman (MGSCI with kappa = 2)".  Cost O(nu_j j N) with nu_j < 3 typically.
// Acceptance test, sweep cap and degeneracy threshold: DESIGN.md reading R7.
//
// B200 design: the method is a chain of 2*nu*k dependent
// reductions of length N, so the kernel is latency-bound.  It runs as ONE thread-block
// cluster of 16 CTAs x 128 lanes (+ a producer warp each; 8 x 256 with RBG_IMGS_CTAS=8),
// L_I = 2048 lanes; the candidate vector v lives in registers (vector u on lane u mod 2048);
// each MGS step is a lane-local fma chain, a warp xor-butterfly, a CTA pre-reduction, an
// all-to-all of the CTA partials through distributed shared memory (st.async + mbarrier
// transaction counts, no cluster barrier) and the cross-CTA tree evaluated by every thread,
// after which every CTA holds the bit-identical coefficient and updates its slice of v.  The
// slices of q_b are prefetched several steps ahead by TMA from a producer warp (one 4D
// tensor-map copy per stage) and w o q_b is formed in registers; for nvec <= 512 only the 1, 2
// or 4 CTAs that hold vectors run (same tree, same bits).  The kernel is replicated on every
// GPU of a sharded run (no broadcast of q needed).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "kernels.h"

namespace rbg {

// Sum over the 2048 lanes with the balanced pairwise tree of CAC rule 3 (ClusterReducer, the
// RBG_IMGS_PRE=0 variant; the default ClusterReducerPre below adds a CTA pre-reduction).
//  1. xor-butterfly in the warp (offsets 1..16): every lane holds its warp's partial;
//  2. lanes 0..CTAS-1 of warp w of CTA r st.async the partial into slot WPC r + w of every
//     CTA's shared memory (WPC warps per CTA), each store counted (16 B) on the receiving
//     CTA's mbarrier;
//  3. every warp waits for its CTA's 64 slots (1024 B), then lane l adds slots 2l, 2l+1 and
//     an xor-butterfly over the lanes finishes the tree over the 64 (CTA, warp) leaves.
// No CTA or cluster barrier is needed; every warp of every CTA ends with the same bits.
// Slots and mbarriers are double-buffered by reduction parity: a CTA can only receive the
// data of reduction n+2 after all of its own warps have sent reduction n+1, i.e. after
// they finished reading the buffers of reduction n.
#include <cstdio>
// Producer-side waits.  Built with -DRBG_DEBUG_WATCHDOG (protocol debugging only), a wait that
// exceeds ~2 s of clock64 prints where it hung and traps; release builds never trap (a trap is a
// sticky error that poisons the process's CUDA context, and preemption or time slicing can
// stretch a healthy wait).
#ifdef RBG_DEBUG_WATCHDOG
#define RBG_WATCHDOG(t0, ...)                              \
    do {                                                   \
        if (clock64() - (t0) > 4000000000LL) {             \
            printf(__VA_ARGS__);                           \
            __trap();                                      \
        }                                                  \
    } while (0)
#else
#define RBG_WATCHDOG(t0, ...) \
    do {                      \
    } while (0)
#endif

__device__ __forceinline__ void mbar_wait_guarded(uint64_t *bar, uint32_t parity, int code, long long st) {
    const long long t0 = clock64();
    (void)t0;
    while (!mbar_try_wait(bar, parity))
        RBG_WATCHDOG(t0, "IMGS HANG code %d rank %u tid %d step %lld parity %u\n", code, cluster_ctarank(), threadIdx.x,
                     st, parity);
}

template <int CTAS>
struct ClusterReducer {
    static constexpr int WPC = kLaneImgs / CTAS / 32;  // warps per CTA; CTAS * WPC = 64 leaves
    double2 (*slots)[64];
    uint64_t *bars;
    uint32_t rank;
    int warp, lane, par;
    uint32_t phase;  // bit p: parity of the next phase to wait for on bars[p]

    // start: this warp's partial leaves for every CTA; finish: wait for all 64, then the tree.
    // Work placed between the two (loads for the next steps) overlaps the DSMEM round trip.
    __device__ __forceinline__ void start(double re, double im) {
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) {
            re = re + __shfl_xor_sync(0xffffffffu, re, h);
            im = im + __shfl_xor_sync(0xffffffffu, im, h);
        }
        if (lane < CTAS) {
            const uint32_t dst = map_dsmem(smem_u32(&slots[par][rank * WPC + warp]), (uint32_t)lane);
            const uint32_t bar = map_dsmem(smem_u32(&bars[par]), (uint32_t)lane);
            st_async_v2(dst, re, im, bar);
        }
    }

    __device__ __forceinline__ double2 sum(double re, double im) {
        start(re, im);
        return finish();
    }

    __device__ __forceinline__ double2 finish() {
        mbar_wait(&bars[par], (phase >> par) & 1u);
        phase ^= 1u << par;
        // re-arm for n+2 by a lane that sent nothing: an arrive has release semantics, so a
        // sender's arrive would first wait for its own st.async to land in the remote CTA
        if (warp == 0 && lane == 31) mbar_arrive_expect_tx(&bars[par], 64 * 16);
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

// Variant with a CTA-level pre-reduction (PRE): the warp partials of a CTA are combined in
// shared memory behind a named barrier of the consumer warps (tree levels 6 .. 5 + log2 WPC),
// then warp 0's lanes st.async the CTA partial into slot `rank` of every CTA (CTAS messages
// per CTA instead of 64), and every warp finishes the tree over the CTAS partials in
// registers.  Same balanced pairwise tree over the 2048 lanes, same bits.  Slots and
// mbarriers double-buffered by parity as in ClusterReducer (a CTA's warp 0 sends reduction
// n + 1 only after all its warps passed the named barrier of n + 1, i.e. after they read the
// slots of reduction n).
template <int CTAS, int THREADS = kLaneImgs / CTAS>
struct ClusterReducerPre {
    static constexpr int WPC = THREADS / 32;
    double2 (*slots)[64];   // [parity][CTA]
    double2 (*wp)[32];      // [parity][warp]
    uint64_t *bars;
    uint32_t rank;
    int warp, lane, par;
    uint32_t phase;
    long long *sub = nullptr;  // RBG_DEBUG_IMGS: clocks after butterfly / CTA tree / remote wait
    double2 own{};             // CTAS == 1: the CTA partial is the sum (no exchange)

    __device__ __forceinline__ double2 sum(double re, double im) {
        start(re, im);
        return finish();
    }

    // start: warp butterfly, CTA pre-reduction, the CTA partial leaves for every CTA;
    // finish: wait for the CTAS partials, then the cross-CTA tree.  Work placed between the two
    // (loads for the next steps) overlaps the DSMEM round trip.
    __device__ __forceinline__ void start(double re, double im) {
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) {
            re = re + __shfl_xor_sync(0xffffffffu, re, h);
            im = im + __shfl_xor_sync(0xffffffffu, im, h);
        }
        if (sub) sub[0] = clock64();
        if (lane == 0) wp[par][warp] = make_double2(re, im);
        asm volatile("bar.sync 1, %0;" ::"r"(WPC * 32) : "memory");   // consumer warps only
        double2 t[WPC];
#pragma unroll
        for (int w = 0; w < WPC; w++) t[w] = wp[par][w];
#pragma unroll
        for (int h = 1; h < WPC; h <<= 1)
#pragma unroll
            for (int w = 0; w < WPC; w += 2 * h) t[w] = make_double2(t[w].x + t[w + h].x, t[w].y + t[w + h].y);
        if (sub) sub[1] = clock64();
        if constexpr (CTAS == 1) {
            own = t[0];  // every thread evaluated the CTA tree: nothing to exchange
            return;
        }
        if (warp == 0 && lane < CTAS) {
            const uint32_t dst = map_dsmem(smem_u32(&slots[par][rank]), (uint32_t)lane);
            const uint32_t bar = map_dsmem(smem_u32(&bars[par]), (uint32_t)lane);
            st_async_v2(dst, t[0].x, t[0].y, bar);
        }
    }

    __device__ __forceinline__ double2 finish() {
        if constexpr (CTAS == 1) {
            par ^= 1;
            return own;
        }
        mbar_wait(&bars[par], (phase >> par) & 1u);
        if (sub) sub[2] = clock64();
        phase ^= 1u << par;
        // re-arm for n+2 by a warp that sent nothing (warp 0 sends): an arrive has release
        // semantics and would first wait for the sender's own st.async to land remotely
        if (warp == WPC - 1 && lane == 31) mbar_arrive_expect_tx(&bars[par], CTAS * 16);
        // the tree over the CTAS CTA partials, evaluated by every thread from shared memory
        // (broadcast reads): leaf l = slots[par][l], pairwise with ascending offsets -- the
        // nodes of the former xor-butterfly, without its dependent shuffles
        double2 c[CTAS];
#pragma unroll
        for (int l = 0; l < CTAS; l++) c[l] = slots[par][l];
#pragma unroll
        for (int h = 1; h < CTAS; h <<= 1)
#pragma unroll
            for (int l = 0; l < CTAS; l += 2 * h) c[l] = make_double2(c[l].x + c[l + h].x, c[l].y + c[l + h].y);
        par ^= 1;
        return c[0];
    }
};

template <int CTAS, int T>
__device__ __forceinline__ ClusterReducerPre<CTAS, T> make_reducer(ClusterReducerPre<CTAS, T> *, double2 (*slots)[64],
                                                                 double2 (*wp)[32], uint64_t *bars, uint32_t rank,
                                                                 int warp, int lane) {
    return ClusterReducerPre<CTAS, T>{slots, wp, bars, rank, warp, lane, 0, 0u};
}
template <int CTAS>
__device__ __forceinline__ ClusterReducer<CTAS> make_reducer(ClusterReducer<CTAS> *, double2 (*slots)[64],
                                                             double2 (*)[32], uint64_t *bars, uint32_t rank, int warp,
                                                             int lane) {
    return ClusterReducer<CTAS>{slots, bars, rank, warp, lane, 0, 0u};
}

template <bool CPLX, int MAXV>
__device__ __forceinline__ void dot_partial(const double2 (&v)[MAXV], const double2 *wq, int stride, int nm,
                                            double &pr, double &pi) {
    pr = 0.0;
    pi = 0.0;
#pragma unroll
    for (int m = 0; m < MAXV; m++) {
        if (m < nm) {  // DOT(WQ_i, v), CAC rule 2
            const double2 e = wq[m * stride];
            if (CPLX) {
                pr = fma(e.x, v[m].x, pr);
                pr = fma(e.y, v[m].y, pr);
                pi = fma(e.x, v[m].y, pi);
                pi = fma(-e.y, v[m].x, pi);
            } else {
                pr = fma(e.x, v[m].x, pr);
                pr = fma(e.y, v[m].y, pr);
            }
        }
    }
}

template <bool CPLX, int MAXV>
__device__ __forceinline__ void axpy(double2 (&v)[MAXV], const double2 *q, int stride, int nm, double2 c) {
#pragma unroll
    for (int m = 0; m < MAXV; m++) {
        if (m < nm) {  // v <- v - c q_i, CAC rule 9
            const double2 qq = q[m * stride];
            if (CPLX) {
                double vr = v[m].x, vi = v[m].y;
                vr = fma(-c.x, qq.x, vr);
                vr = fma(c.y, qq.y, vr);
                vi = fma(-c.x, qq.y, vi);
                vi = fma(-c.y, qq.x, vi);
                v[m] = make_double2(vr, vi);
            } else {
                v[m].x = fma(-c.x, qq.x, v[m].x);
                v[m].y = fma(-c.x, qq.y, v[m].y);
            }
        }
    }
}

// Register-operand forms (the staged slices loaded ahead of the step that uses them).
template <bool CPLX, int MAXV>
__device__ __forceinline__ void dot_regs(const double2 (&v)[MAXV], const double2 (&e)[MAXV], int nm, double &pr,
                                         double &pi) {
    pr = 0.0;
    pi = 0.0;
#pragma unroll
    for (int m = 0; m < MAXV; m++) {
        if (m < nm) {  // DOT(WQ_i, v), CAC rule 2
            if (CPLX) {
                pr = fma(e[m].x, v[m].x, pr);
                pr = fma(e[m].y, v[m].y, pr);
                pi = fma(e[m].x, v[m].y, pi);
                pi = fma(-e[m].y, v[m].x, pi);
            } else {
                pr = fma(e[m].x, v[m].x, pr);
                pr = fma(e[m].y, v[m].y, pr);
            }
        }
    }
}

template <bool CPLX, int MAXV>
__device__ __forceinline__ void axpy_regs(double2 (&v)[MAXV], const double2 (&q)[MAXV], int nm, double2 c) {
#pragma unroll
    for (int m = 0; m < MAXV; m++) {
        if (m < nm) {  // v <- v - c q_i, CAC rule 9
            if (CPLX) {
                double vr = v[m].x, vi = v[m].y;
                vr = fma(-c.x, q[m].x, vr);
                vr = fma(c.y, q[m].y, vr);
                vi = fma(-c.x, q[m].y, vi);
                vi = fma(-c.y, q[m].x, vi);
                v[m] = make_double2(vr, vi);
            } else {
                v[m].x = fma(-c.x, q[m].x, v[m].x);
                v[m].y = fma(-c.x, q[m].y, v[m].y);
            }
        }
    }
}

template <int MAXV>
__device__ __forceinline__ void load_slice(double2 (&r)[MAXV], const double2 *p, int stride, int nm) {
#pragma unroll
    for (int m = 0; m < MAXV; m++) r[m] = (m < nm) ? p[m * stride] : make_double2(0.0, 0.0);
}

// The weights of this lane's vectors, held in registers for the whole kernel: (w_u, w_u) for
// complex data, (w_2u, w_2u+1) for real data packed in pairs -- so that w o q_b is formed from
// the staged q_b alone.  wr.x * q.x is the same IEEE product the kernel stores into WQ (a1), so
// the dot's operand has the same bits as the stored w o q_b and only Q needs staging.
template <bool CPLX, int MAXV>
__device__ __forceinline__ void load_weights(double2 (&wr)[MAXV], const double *w, int u0, int nm) {
#pragma unroll
    for (int m = 0; m < MAXV; m++) {
        const int u = u0 + m * kLaneImgs;
        if (m < nm) wr[m] = CPLX ? make_double2(w[u], w[u]) : make_double2(w[2 * u], w[2 * u + 1]);
        else wr[m] = make_double2(0.0, 0.0);
    }
}

template <int MAXV>
__device__ __forceinline__ void weigh(double2 (&e)[MAXV], const double2 (&wr)[MAXV], const double2 (&q)[MAXV]) {
#pragma unroll
    for (int m = 0; m < MAXV; m++) e[m] = make_double2(wr[m].x * q[m].x, wr[m].y * q[m].y);
}

// the weighted squared norm's lane partial, CAC rule 4 (w_u v.x v.x + w_u v.y v.y in this order)
template <int MAXV>
__device__ __forceinline__ double nrm_regs(const double2 (&v)[MAXV], const double2 (&wr)[MAXV], int nm) {
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < MAXV; m++) {
        if (m < nm) {
            double t = wr[m].x * v[m].x;
            acc = fma(t, v[m].x, acc);
            t = wr[m].y * v[m].y;
            acc = fma(t, v[m].y, acc);
        }
    }
    return acc;
}

// Basis-vector pipeline.  STAGED (D > 0): the CTA's slice of q_b (MAXV chunks of THREADS
// vectors: chunk m starts at vector 2048 m + THREADS rank) is prefetched up to D MGS steps
// ahead into shared memory by TMA issued by a dedicated producer warp (the last warp), one
// full-mbarrier (TMA bytes) and one empty-mbarrier (the consumer warps) per stage, so issuing
// copies never delays a warp on the reduction's critical path.  w o q_b is formed in registers
// (weigh), so only Q is staged: half the TMA bytes and half the shared-memory reads of staging
// both arrays (round 2).  D = 0: the slices of WQ and Q are loaded straight from global memory
// one step ahead (large N only).
// 4D tensor-map TMA: (x, rank, chunk, basis index) -> one CTA's MAXV chunk slices in one copy.
__device__ __forceinline__ void tma_4d_g2s(void *dst, const CUtensorMap *map, int x, int y, int z, int w, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
        : "memory");
}

template <int MAXV, int D, int THREADS>
struct BasisPipe {
    unsigned char *smem;
    uint64_t *full, *empty;
    const double2 *Q;
    long long ldq_v;
    int k, rank, nvec;
    // 16 x 128 lanes: one tensor-map copy per stage (tmQ views the basis as
    // [basis][chunk][rank][128 vectors]; the allocation is padded so that the box of the last
    // chunk stays in bounds, its vectors past nvec are never read); else MAXV bulk copies.
    // Per-SM TMA work is what limits the prefetch: with 10 bulk copies per stage a stage was
    // issued only ~1.3 us (~1.6 MGS steps) before it was needed (RBG_DEBUG_IMGS).
    const CUtensorMap *tmQ;

    static constexpr int kStageBytes = MAXV * THREADS * 16;

    __device__ __forceinline__ double2 *q_stage(long long s) const {
        return reinterpret_cast<double2 *>(smem + (size_t)(s % D) * kStageBytes);
    }

    __device__ void issue(long long s) const {  // one producer thread
        const int b = (int)(s % k);
        if (tmQ) {
            uint64_t *bar = &full[s % D];
            mbar_arrive_expect_tx(bar, (uint32_t)kStageBytes);
            tma_4d_g2s(q_stage(s), tmQ, 0, rank, 0, b, bar);
            return;
        }
        uint32_t bytes = 0;
        int len[MAXV];
#pragma unroll
        for (int m = 0; m < MAXV; m++) {
            const int u0 = m * kLaneImgs + rank * THREADS;
            const int l = nvec - u0;
            len[m] = l < 0 ? 0 : (l > THREADS ? THREADS : l);
            bytes += (uint32_t)len[m] * 16u;
        }
        uint64_t *bar = &full[s % D];
        mbar_arrive_expect_tx(bar, bytes);
        const double2 *q = Q + (long long)b * ldq_v;
        double2 *dq = q_stage(s);
#pragma unroll
        for (int m = 0; m < MAXV; m++) {
            if (len[m] > 0) {
                const int u0 = m * kLaneImgs + rank * THREADS;
                bulk_g2s(dq + m * THREADS, q + u0, (uint32_t)len[m] * 16u, bar);
            }
        }
    }

    // Producer loop: steps D.. until the consumers publish their final step count in *done
    // (>= 0); then wait for every copy still in flight so none outlives the CTA.
    __device__ void produce(long long issued, long long limit, volatile long long *done,
                            unsigned long long *tissue = nullptr) const {
        while (issued < limit) {
            const uint32_t par = (uint32_t)((issued / D - 1) & 1);
            bool ok = false;
            const long long tp = clock64();
            (void)tp;
            while (!(ok = mbar_try_wait(&empty[issued % D], par))) {
                if (*done >= 0) break;
                RBG_WATCHDOG(tp, "IMGS HANG producer rank %u issued %lld par %u\n", cluster_ctarank(), issued, par);
            }
            if (!ok) break;
            // RBG_DEBUG_IMGS: when stages 65..72 were issued (consumers need them at steps 64..71)
            if (tissue && issued >= 65 && issued < 73) tissue[issued - 65] = globaltimer_ns();
            issue(issued++);
        }
        long long consumed;
        const long long td = clock64();
        (void)td;
        while ((consumed = *done) < 0)
            RBG_WATCHDOG(td, "IMGS HANG producer waits for done, rank %u issued %lld\n", cluster_ctarank(), issued);
        for (long long s = consumed; s < issued; s++) mbar_wait_guarded(&full[s % D], (uint32_t)((s / D) & 1), 3, s);
    }
};

// THREADS: consumer lanes per CTA, kLaneImgs / CTAS -- or 128 with CTAS in {1, 2, 4} when all
// vectors sit in the first CTAS x 128 lanes (nvec <= 512, see launch_imgs): the lanes of the
// other CTAs of the 16 x 128 layout would hold only zeros, their CTA partials are +0 and the
// cross-CTA tree's nodes over them add +0 (x + 0 = x; no partial is ever -0), so the fewer-CTA
// tree gives the 2,048-lane tree's bits (CAC rule 3) with fewer DSMEM messages.
template <bool CPLX, int MAXV, int D, int CTAS, bool PRE, int THREADS = kLaneImgs / CTAS>
__global__ void __launch_bounds__(THREADS + 32, 1)
    k_imgs(const ImgsArgs a, const __grid_constant__ CUtensorMap tmQ) {
    constexpr int DD = D > 0 ? D : 1;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ double2 s_slots[2][64];
    __shared__ double2 s_wp[2][32];
    __shared__ __align__(8) uint64_t s_bars[2];
    __shared__ __align__(8) uint64_t s_full[DD], s_empty[DD];
    __shared__ long long s_done;
    __shared__ long long s_sub[3];  // RBG_DEBUG_IMGS sub-phase clocks (CTA 0, thread 0)

    // state written by the previous decision kernel (stop, k) and the basis q_1..q_k are final
    // before this kernel starts even as a programmatic dependent of the sweep (the sweep waits
    // for its predecessor before it lets this grid launch); the sweep's maxloc is read only
    // after grid_dep_wait
    const int stop0 = a.st->stop;
    if (stop0) {
        if (threadIdx.x == 0 && blockIdx.x == 0) {
            loop_exit(a.cond, a.use_cond);
            a.st->noop += 1;  // rbg_stats.noop_iters: iterations launched past the stop
        }
        return;
    }
    const long long k = a.st->k;
    const uint32_t rank = cluster_ctarank();
    const int tid = threadIdx.x;
    const bool producer = tid >= THREADS;   // the last warp (D > 0 only)
    // RBG_DEBUG_IMGS: %globaltimer of this kernel's phases (CTA 0, thread 0) at trace[257 + p]
    unsigned long long *ts = (a.trace && rank == 0 && tid == 0) ? reinterpret_cast<unsigned long long *>(a.trace) + 257 : nullptr;
    if (ts) ts[0] = globaltimer_ns();
    const int nvec = (int)a.nvec;
    const int u0 = (int)rank * THREADS + tid;                  // this lane's first vector
    const int nm = (!producer && u0 < nvec) ? (nvec - u0 + kLaneImgs - 1) / kLaneImgs : 0;
    const bool odd_tail = !CPLX && (a.N & 1);

    const BasisPipe<MAXV, DD, THREADS> pipe{dsm,       s_full, s_empty, a.Q, a.ldq_v, (int)k, (int)rank, nvec,
                                            a.use_tm ? &tmQ : nullptr};
    const long long limit = (long long)kNuMax * k;  // MGS steps that can ever be needed
    // stages issued before the cluster barrier (the rest by the producer loop, off the
    // critical path: each stage is 2 MAXV bulk copies issued by one thread)
    const long long first = k < a.k_max ? (limit < 2 ? limit : (DD < 2 ? DD : 2)) : 0;
    if (tid == 0) {
        mbar_init_nofence(&s_bars[0], 1);
        mbar_init_nofence(&s_bars[1], 1);
        fence_mbarrier_init();
        mbar_arrive_expect_tx(&s_bars[0], (PRE ? CTAS : 64) * 16);
        mbar_arrive_expect_tx(&s_bars[1], (PRE ? CTAS : 64) * 16);
        s_done = -1;
    }
    if (D > 0 && tid == THREADS) {
        for (int i = 0; i < DD; i++) {
            mbar_init_nofence(&s_full[i], 1);
            mbar_init_nofence(&s_empty[i], THREADS / 32);
        }
        fence_mbarrier_init();
        for (long long s = 0; s < first; s++) pipe.issue(s);
    }
    // every CTA has read the state before rank 0 changes it, and every CTA's mbarriers are
    // initialised before any remote st.async can target them
    cluster_sync_all();
    if (ts) ts[1] = globaltimer_ns();
    grid_dep_wait();
    if (ts) ts[2] = globaltimer_ns();

    // ---- a3: pivot decision (identical in every CTA and on every rank) ------------------
    double m;
    long long J;
    const double2 *src;
    pivot_decision(a, k, m, J, src);
    const double err = sqrt(fmax(m, 0.0));  // CAC rule 8
    int why = kStopNone;
    if (m == -INFINITY) why = kStopAll;
    else if (err < a.tol) why = kStopTol;
    else if (k == a.k_max) why = kStopKmax;

    const bool leader = (rank == 0 && tid == 0);
    if (leader) a.errors[k] = err;
    if (why != kStopNone) {
        if (leader) {
            a.st->stop = why;
            loop_exit(a.cond, a.use_cond);
        }
        if (D > 0 && tid == THREADS)  // no copy may outlive the CTA
            for (long long s = 0; s < first; s++) mbar_wait_guarded(&s_full[s], 0u, 4, s);
        return;
    }
    if (producer) {
        if (D > 0 && tid == THREADS)
            pipe.produce(first, limit, &s_done,
                         a.trace ? reinterpret_cast<unsigned long long *>(a.trace) + 320 + rank * 8 : nullptr);
        return;
    }

    // ---- a5: Hoffmann IMGS (CAC rule 9) ---------------------------------------------
    double2 v[MAXV];
#pragma unroll
    for (int mm = 0; mm < MAXV; mm++) {
        const int u = u0 + mm * kLaneImgs;
        v[mm] = (mm < nm) ? (a.peer_mine ? ld_cv(src + u) : src[u]) : make_double2(0.0, 0.0);
        if (odd_tail && u == nvec - 1) v[mm].y = 0.0;
    }

    const int warp = tid >> 5, lane = tid & 31;
    using Red = typename std::conditional<PRE, ClusterReducerPre<CTAS, THREADS>, ClusterReducer<CTAS>>::type;
    Red red = make_reducer(static_cast<Red *>(nullptr), s_slots, s_wp, s_bars, rank, warp, lane);
    const uint64_t keep = policy_evict_last();
    double2 wr[MAXV];
    load_weights<CPLX, MAXV>(wr, a.w, u0, nm);
    const double n0 = sqrt(red.sum(nrm_regs<MAXV>(v, wr, nm), 0.0).x);
    if (ts) ts[3] = globaltimer_ns();
    double n_prev = n0, nn = 0.0;
    int nu = 0;
    bool accepted = false;
    long long s = 0;  // MGS steps taken (basis index s mod k)
    // direct-load path (D == 0): one step of register prefetch
    double2 wq[MAXV], q[MAXV];
    if (D == 0 && k > 0) {
#pragma unroll
        for (int mm = 0; mm < MAXV; mm++) {
            wq[mm] = (mm < nm) ? ld_keep(a.WQ + u0 + mm * kLaneImgs, keep) : make_double2(0.0, 0.0);
            q[mm] = (mm < nm) ? ld_keep(a.Q + u0 + mm * kLaneImgs, keep) : make_double2(0.0, 0.0);
        }
    }
    // staged path: q_s and w o q_s are in registers before step s begins (stage s was read,
    // and released, while the partials of step s - 1 were in flight)
    double2 wqr[MAXV], qc[MAXV];
    if (D > 0 && k > 0) {
        mbar_wait(&s_full[0], 0u);
        load_slice<MAXV>(qc, pipe.q_stage(0) + tid, THREADS, nm);
        weigh<MAXV>(wqr, wr, qc);
        __syncwarp();
        if (lane == 31) mbar_arrive(&s_empty[0]);
    }
    // one MGS step of the staged path: q_s in qcur (and w o q_s in wqr) on entry; stage s + 1
    // lands in qnext (and w o q_{s+1} in wqr).  Slots past nm hold zeros in v, wr, wqr and the
    // staged slices, so the dot / axpy run over all MAXV slots without predicates: the extra
    // terms are fma(+-0, +-0, x) = x for x != 0 and +0 for x = +0, and no partial is ever -0
    // (each starts at +0), so the bits are those of the nm-term chains (CAC rules 2, 9).
    auto mgs_step = [&](double2 (&qcur)[MAXV], double2 (&qnext)[MAXV]) {
        double pr, pi;
        // RBG_DEBUG_IMGS: clock64 at the phase boundaries of steps 64..95 (CTA 0, tid 0)
        const bool tr = a.trace && rank == 0 && tid == 0 && s >= 64 && s < 96;
        // every CTA's %globaltimer at step start / partial sent / coefficient known for
        // steps 64..71 (trace[512 + (rank*8 + step)*4 + p]; p = 3: the next stage is in
        // shared memory): the cluster's critical path
        unsigned long long *gt = (a.trace && tid == 0 && s >= 64 && s < 72)
                                     ? reinterpret_cast<unsigned long long *>(a.trace) + 512 + (rank * 8 + (s - 64)) * 4
                                     : nullptr;
        if (gt) gt[0] = globaltimer_ns();
        const long long c0 = tr ? clock64() : 0;
        dot_regs<CPLX, MAXV>(v, wqr, MAXV, pr, pi);
        const long long c1 = tr ? clock64() : 0;
        // (shared, not a local array: a local array costs three stack stores per step)
        long long *sb = s_sub;
        if constexpr (PRE) red.sub = tr ? sb : nullptr;
        red.start(pr, pi);
        if (gt) gt[1] = globaltimer_ns();
        const long long c2 = tr ? clock64() : 0;
        // while the partials travel: stage s + 1 into registers, w o q_{s+1} formed, the
        // stage released (lane 31 never issues st.async, so its release-arrive does not
        // wait for a remote store).  (Loading the stage before the reduction instead: k = 299
        // IMGS 369 -> 387 us, no gain on the one-CTA path either.)
        if (s + 1 < limit) {
            mbar_wait(&s_full[(s + 1) % DD], (uint32_t)(((s + 1) / DD) & 1));
            load_slice<MAXV>(qnext, pipe.q_stage(s + 1) + tid, THREADS, nm);
            weigh<MAXV>(wqr, wr, qnext);
            __syncwarp();
            if (lane == 31) mbar_arrive(&s_empty[(s + 1) % DD]);
        }
        if (gt) gt[3] = globaltimer_ns();
        const long long c3 = tr ? clock64() : 0;
        const double2 c = red.finish();
        if (gt) gt[2] = globaltimer_ns();
        const long long c4 = tr ? clock64() : 0;
        axpy_regs<CPLX, MAXV>(v, qcur, MAXV, c);
        if (tr) {
            const long long c5 = clock64();
            long long *t = a.trace + (s - 64) * 8;
            t[0] = c0; t[1] = c1; t[2] = c2; t[3] = c3; t[4] = c4; t[5] = c5;
            t[6] = sb[1]; t[7] = sb[2];
        }
        s++;
    };
    double2 qb[MAXV];  // the other register buffer of the staged path (q_{s+1})
    while (nu < kNuMax) {
        nu++;
        if (D > 0) {
            // two steps per trip with the buffers' roles swapped: no register copies
            for (long long i = 0; i < k; i += 2) {
                mgs_step(qc, qb);
                if (i + 1 == k) {
#pragma unroll
                    for (int mm = 0; mm < MAXV; mm++) qc[mm] = qb[mm];  // odd k: once per pass
                    break;
                }
                mgs_step(qb, qc);
            }
        } else {
            for (long long i = 0; i < k; i++, s++) {
                double pr, pi;
                dot_partial<CPLX, MAXV>(v, wq, 1, nm, pr, pi);
                double2 wq_n[MAXV], q_n[MAXV];
                const long long bn = (i + 1 < k) ? i + 1 : 0;
                const double2 *wqp = a.WQ + bn * a.ldq_v + u0, *qp = a.Q + bn * a.ldq_v + u0;
#pragma unroll
                for (int mm = 0; mm < MAXV; mm++) {
                    wq_n[mm] = (mm < nm) ? ld_keep(wqp + mm * kLaneImgs, keep) : make_double2(0.0, 0.0);
                    q_n[mm] = (mm < nm) ? ld_keep(qp + mm * kLaneImgs, keep) : make_double2(0.0, 0.0);
                }
                const double2 c = red.sum(pr, pi);
                axpy<CPLX, MAXV>(v, q, 1, nm, c);
#pragma unroll
                for (int mm = 0; mm < MAXV; mm++) {
                    wq[mm] = wq_n[mm];
                    q[mm] = q_n[mm];
                }
            }
        }
        nn = sqrt(red.sum(nrm_regs<MAXV>(v, wr, nm), 0.0).x);
        if (nn > n_prev / 2.0) {  // Hoffmann's test with kappa = 2
            accepted = true;
            break;
        }
        n_prev = nn;
    }
    // release the producer: it drains the copies it issued past the stages the consumers read
    // (stages 0 .. s, or 0 .. limit - 1: stage s + 1 is read during step s, and once released the
    // producer may already have reused its slot, so those slots must not be waited on again)
    if (tid == 0) s_done = (k > 0 && s < limit) ? s + 1 : s;
    if (ts) ts[4] = globaltimer_ns();
    // the next sweep may now take the SMs this cluster does not use (earlier, its first loads
    // would compete with the latency-bound reductions for the memory system)
    grid_dep_launch();
    const double delta = 1000.0 * 0x1p-52;
    if (!accepted || !(nn >= delta * n0) || nn == 0.0) {
        if (leader) {
            a.nu[k] = nu;
            a.st->stop = kStopRank;
            loop_exit(a.cond, a.use_cond);
        }
        return;
    }

    // ---- q_{k+1} = v / n, w o q_{k+1}; a6 bookkeeping -------------------------------
    double2 *qo = a.Q + k * a.ldq_v;
    double2 *wqo = a.WQ + k * a.ldq_v;
#pragma unroll
    for (int mm = 0; mm < MAXV; mm++) {
        const int u = u0 + mm * kLaneImgs;
        if (mm < nm) {
            const double2 qq = make_double2(v[mm].x / nn, v[mm].y / nn);
            st_keep(qo + u, qq, keep);
            st_keep(wqo + u, make_double2(wr[mm].x * qq.x, wr[mm].y * qq.y), keep);
        }
    }
    if (leader) {
        if (ts) ts[5] = globaltimer_ns();
        a.piv[k] = J;
        a.nu[k] = nu;
        a.rdiag[k] = nn;
        const long long jl = local_col(a, J);
        if (jl >= 0) a.r2[jl] = -INFINITY;
        a.st->k = k + 1;
    }
}

// (MAXV, D): vectors per lane and prefetch depth, D * MAXV * 32 KB / CTAS of shared memory.
// The tensor map of Q for the 16 x 128 staged path (BasisPipe); false if not applicable.
bool make_imgs_maps(const double2 *Q, long long nvec, long long ldq_v, long long k_max, void *map) {
    const int maxv = imgs_maxv(nvec);
    if (maxv == 0 || maxv > 8 || getenv("RBG_IMGS_BULK")) return false;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    // (256 doubles = 128 vectors) x 16 ranks x maxv chunks (2,048 vectors apart) x k_max
    const cuuint64_t dims[4] = {256, 16, (cuuint64_t)maxv, (cuuint64_t)k_max};
    const cuuint64_t strides[3] = {2048, 32768, (cuuint64_t)ldq_v * 16};
    const cuuint32_t box[4] = {256, 1, (cuuint32_t)maxv, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return encode(static_cast<CUtensorMap *>(map), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double2 *>(Q), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int imgs_maxv(long long nvec) {
    const long long per = (nvec + kLaneImgs - 1) / kLaneImgs;
    if (per <= 6) return (int)(per < 1 ? 1 : per);
    if (per <= 8) return 8;
    if (per <= 12) return 12;
    if (per <= 16) return 16;
    return 0;
}

// Cluster size: 16 CTAs x 128 lanes (non-portable cluster) halves each SM's share of the
// per-step FP64 work and basis bytes against 8 x 256; L_I = 2048 and the reduction tree are
// the same, so the result bits are identical.  RBG_IMGS_CTAS=8 selects the portable size.
static int imgs_ctas() {
    static int c = 0;
    if (c == 0) {
        c = 16;
        if (const char *e = getenv("RBG_IMGS_CTAS"))
            if (atoi(e) == 8) c = 8;
    }
    return c;
}

// CTA pre-reduction before the cluster all-to-all (ClusterReducerPre, the default: 0.76-0.78
// vs 0.78-0.85 us per MGS step at k = 300); RBG_IMGS_PRE=0 selects the 64-message all-to-all.
// Same tree, same bits either way.
static bool imgs_pre() {
    static int p = -1;
    if (p < 0) {
        p = 1;
        if (const char *e = getenv("RBG_IMGS_PRE")) p = atoi(e) != 0;
    }
    return p != 0;
}

template <bool CPLX, int MAXV, int D, int CTAS>
static cudaError_t launch_md(const ImgsArgs &a, cudaStream_t s) {
    auto kern = imgs_pre() ? k_imgs<CPLX, MAXV, D, CTAS, true> : k_imgs<CPLX, MAXV, D, CTAS, false>;
    constexpr int THREADS = kLaneImgs / CTAS;
    const size_t smem = D > 0 ? (size_t)D * MAXV * THREADS * 16 : 0;
    cudaError_t e;
    if (smem > 0) {  // dynamic + static may pass 48 KB even when the dynamic part alone does not
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    if (CTAS > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CTAS, 1, 1);
    cfg.blockDim = dim3(THREADS + 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CTAS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic dependent launch after the sweep: the cluster's prologue (barriers, the
    // producer's first basis copies) runs while the sweep drains; grid_dep_wait before the
    // decision reads the sweep's maxloc
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 2 : 1;
    // the tensor map cuts 128-vector slices: the 16 x 128 staged path only
    ImgsArgs b = a;
    b.use_tm = (a.use_tm && a.tm && CTAS == 16 && D > 0) ? 1 : 0;
    const CUtensorMap *tm = static_cast<const CUtensorMap *>(a.tm);
    static const CUtensorMap zero{};
    e = cudaLaunchKernelEx(&cfg, kern, b, tm ? *tm : zero);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// Small N (nvec <= 512, one vector per lane): a cluster of CTAS in {1, 2, 4} CTAs x 128 lanes
// (the occupied lanes of the 16 x 128 layout; same tree, same bits), CTA pre-reduction,
// 16 basis stages of one bulk copy each.  RBG_IMGS_SMALL=0 keeps the 16-CTA cluster.
template <bool CPLX, int CTAS>
static cudaError_t launch_small(const ImgsArgs &a, cudaStream_t s) {
    constexpr int THREADS = 128, D = 16;
    auto kern = k_imgs<CPLX, 1, D, CTAS, true, THREADS>;
    const size_t smem = (size_t)D * THREADS * 16;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CTAS, 1, 1);
    cfg.blockDim = dim3(THREADS + 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CTAS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 2 : 1;
    ImgsArgs b = a;
    b.use_tm = 0;
    static const CUtensorMap zero{};
    e = cudaLaunchKernelEx(&cfg, kern, b, zero);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

static bool imgs_small() {
    static int v = -1;
    if (v < 0) {
        v = 1;
        if (const char *e = getenv("RBG_IMGS_SMALL")) v = atoi(e) != 0;
    }
    return v != 0;
}

template <bool CPLX, int CTAS>
static cudaError_t launch_c(const ImgsArgs &a, cudaStream_t s) {
    // prefetch depth: the same shared-memory budget per CTA at either cluster size
    constexpr int X = CTAS / 8;
    switch (imgs_maxv(a.nvec)) {
        case 1: return launch_md<CPLX, 1, 8 * X, CTAS>(a, s);
        case 2: return launch_md<CPLX, 2, 6 * X, CTAS>(a, s);
        case 3: return launch_md<CPLX, 3, 6 * X, CTAS>(a, s);
        case 4: return launch_md<CPLX, 4, 5 * X, CTAS>(a, s);
        case 5: return launch_md<CPLX, 5, 4 * X, CTAS>(a, s);
        case 6: return launch_md<CPLX, 6, 4 * X, CTAS>(a, s);
        case 8: return launch_md<CPLX, 8, 3 * X, CTAS>(a, s);
        case 12: return launch_md<CPLX, 12, 0, CTAS>(a, s);
        case 16: return launch_md<CPLX, 16, 0, CTAS>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_imgs(const ImgsArgs &a, bool cplx, cudaStream_t s) {
    if (a.nvec <= 512 && imgs_ctas() == 16 && imgs_small()) {
        const int c = a.nvec <= 128 ? 1 : (a.nvec <= 256 ? 2 : 4);
        if (c == 1) return cplx ? launch_small<true, 1>(a, s) : launch_small<false, 1>(a, s);
        if (c == 2) return cplx ? launch_small<true, 2>(a, s) : launch_small<false, 2>(a, s);
        return cplx ? launch_small<true, 4>(a, s) : launch_small<false, 4>(a, s);
    }
    if (imgs_ctas() == 16) return cplx ? launch_c<true, 16>(a, s) : launch_c<false, 16>(a, s);
    return cplx ? launch_c<true, 8>(a, s) : launch_c<false, 8>(a, s);
}

}  // namespace rbg
