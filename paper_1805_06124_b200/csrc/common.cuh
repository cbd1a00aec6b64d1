// common.cuh -- device-side types and PTX helpers shared by the rbg kernels (sm_100a).
//
// Arithmetic rule for every kernel in this directory: the canonical arithmetic contract
// of DESIGN.md.  The library is compiled with --fmad=false, so a*b+c is never fused
// behind our back; every fused multiply-add is an explicit fma().
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rbg {

constexpr int kLaneSweep = 32;      // L_S: one warp per column
constexpr int kLaneImgs = 2048;     // L_I: the IMGS cluster's lanes (16 CTAs x 128 by default,
                                    // 8 x 256 with RBG_IMGS_CTAS=8; same lanes, same tree)
constexpr int kNuMax = 5;           // IMGS sweep cap (R7)

constexpr int kStopNone = 0, kStopTol = 1, kStopKmax = 2, kStopRank = 3, kStopAll = 4, kStopPeer = 5;
constexpr int kMaxPeers = 8;        // ranks of a PEER exchange (one NVSwitch box)

// One maxloc record: 16 bytes, total order (m descending, j ascending).
struct __align__(16) Rec {
    double m;
    long long j;
};

__device__ __forceinline__ bool rec_better(double m1, long long j1, double m2, long long j2) {
    return (m1 > m2) || (m1 == m2 && j1 < j2);
}

// PEER exchange: rank p's sweep writes its local maxloc into slot
// (parity, p) of EVERY rank's record array over NVLink (P2P stores), then the tag with release
// semantics; tag = st->k + 1 of the sweep (unique per iteration), parity = tag & 1 (records of
// consecutive iterations never share a slot).
struct __align__(32) PeerRec {
    double m;
    long long j;                  // global column index
    unsigned long long tag;
    long long pad;
};

// Device-resident loop state (one per context).
struct DevState {
    long long k;        // basis vectors built so far
    int stop;           // rbg_stop
    int noop;           // decision/IMGS launches that found the greedy already stopped
    double m_loc;       // local maxloc after the last sweep
    long long j_loc;    // its GLOBAL column index
};

// Layout of one rank's slot in the exchange buffer: Rec header then the candidate column
// (N_pad elements), padded to 16 bytes.
__host__ __device__ inline size_t xchg_slot_bytes(long long nvec) {
    return sizeof(Rec) + (size_t)nvec * 16;
}

// ----------------------------------------------------------------------- PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Several initialisations, then one fence_mbarrier_init() (each fence is a cluster-scope release).
__device__ __forceinline__ void mbar_init_nofence(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbarrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// TMA bulk copy global -> shared (non-tensor), completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Cluster-scope acquire wait (data arriving from other CTAs through st.async).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 16-byte store into another CTA's shared memory, completion counted on that CTA's mbarrier.
__device__ __forceinline__ void st_async_v2(uint32_t dst, double a, double b, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
                 "d"(a), "d"(b), "r"(remote_bar)
                 : "memory");
}

// L2 evict-last policy for the basis vectors (re-read by every later IMGS).
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ double2 ld_keep(const double2 *p, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ void st_keep(double2 *p, double2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

// L2 evict-first policy for the streamed snapshot matrix (read exactly once per sweep).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 16-byte streaming load: non-coherent path, no L1 allocation, L2 evict-first.
__device__ __forceinline__ double2 ld_stream(const double2 *p, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}

// L2 prefetch of a global range (no destination, no completion tracking).
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// System-scope release store / acquire load (flags written and polled across GPUs).
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys_f64(double *p, double v) {
    asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_s64(long long *p, long long v) {
    asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_sys_f64(const double *p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ long long ld_relaxed_sys_s64(const long long *p) {
    long long v;
    asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// 16-byte load that bypasses L1 (data written by another GPU since the last kernel).
__device__ __forceinline__ double2 ld_cv(const double2 *p) {
    double2 r;
    asm volatile("ld.global.cv.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its predecessor runs;
// grid_dep_wait() blocks until the predecessor grid has completed and its writes are visible
// (a no-op without the attribute), grid_dep_launch() lets the successor start early.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// rbg_run's device-side loop: the iteration body is a CUDA-graph
// conditional WHILE node; whichever kernel records the stop decision (or first sees it) sets
// the loop condition to 0, so no iteration is launched after the stop.  use = 0 outside that
// graph (plain launches, graph batches): the handle is then not touched.
__device__ __forceinline__ void loop_exit(cudaGraphConditionalHandle h, int use) {
    if (use) cudaGraphSetConditional(h, 0u);
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

// Map a local shared address to the same offset in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t map_dsmem(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}

__device__ __forceinline__ void st_dsmem_v2(uint32_t addr, double a, double b) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a), "d"(b) : "memory");
}

}  // namespace rbg
