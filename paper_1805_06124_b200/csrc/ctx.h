// ctx.h -- internal to librbg: the context behind the opaque rbg_ctx of include/rbg.h and the
// helpers shared by the C-ABI translation units (api.cu: create / run / exchange / getters;
// api_next.cu: validation, enrichment, Gram, reconstruction, EIM).  Not installed.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys / ncu --nvtx, no-ops otherwise

#include "comm.h"
#include "kernels.h"
#include "rbg.h"

using namespace rbg;  // internal header: included only by the C-ABI translation units

namespace rbg_api {

extern thread_local std::string g_err;   // rbg_last_error()
rbg_status fail(rbg_status s, const char *fmt, ...);

#define CU(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(e_ == cudaErrorMemoryAllocation ? RBG_ENOMEM : RBG_ECUDA,             \
                        "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

#define TRY(call)                          \
    do {                                   \
        rbg_status s_ = (call);            \
        if (s_ != RBG_OK) return s_;       \
    } while (0)

struct PhaseEvents {
    cudaEvent_t e[4];
};

// NVTX range for the host-side enqueue of one phase (SURVEY §5 tracing)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};


}  // namespace rbg_api

struct rbg_ctx {
    using PhaseEvents = rbg_api::PhaseEvents;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool cplx = true;
    long long N = 0, M = 0, nvec = 0, ldv = 0, ldq_v = 0;
    size_t se = 16;  // bytes per element
    double2 *S = nullptr;   // the caller's columns 0..M0-1 (borrowed or a library copy)
    bool own_S = false;
    double2 *S1 = nullptr;  // columns M0..M-1 appended by enrichment (library-owned, pitch nvec)
    long long M0 = 0;
    double *w = nullptr;
    double2 *Q = nullptr, *WQ = nullptr;
    double *R = nullptr, *r2 = nullptr;
    long long ldr = 0;  // R row stride in elements (>= M: room for appended columns, rbg_add_columns)
    DevState *st = nullptr;
    double *errors = nullptr, *rdiag = nullptr;
    long long *piv = nullptr;
    int *nu = nullptr;
    Rec *recs = nullptr;
    unsigned *ticket = nullptr;
    unsigned long long *next_col = nullptr;  // dynamic column counter of the sweep
    double tol = 0.0;
    long long k_max = 0;
    rbg_comm comm = RBG_COMM_NONE;
    int rank = 0, world = 1;
    long long col_offset = 0, M_global = 0;
    unsigned char *send = nullptr, *recv = nullptr;
    size_t slot = 0;
    void *nccl = nullptr;
    int num_sms = 148;
    SweepConfig cfg_init{}, cfg_sweep{};
    bool started = false;
    bool local_pending = false;  // EXTERNAL: local done, finish not yet
    bool resume_pending = false; // columns were added: next iteration starts at the decision
    long long iters = 0;         // iterations enqueued
    bool timing = false;
    std::vector<PhaseEvents> ev;  // per iteration when timing
    std::vector<long long> ev_iter;
    int graph_batch = 0;
    cudaGraphExec_t graph = nullptr;
    // rbg_run's device loop: one iteration as the body of a conditional WHILE graph node; the
    // kernel that records the stop sets the condition to 0 (loop_exit), so the host neither
    // polls nor launches iterations past the stop.  in_while: capturing the body (kernels get
    // use_cond = 1).  while_failed: the graph could not be built here, rbg_run polls instead.
    cudaGraphExec_t while_exec = nullptr;
    cudaGraphConditionalHandle cond = 0;
    bool in_while = false;
    bool while_failed = false;
    bool stopped = false;        // the last rbg_run ended at a stop decision (host-side)
    cudaStream_t cap_stream = nullptr;   // graphs are captured here, launched on `stream`
    cudaStream_t poll_stream = nullptr;  // polled rbg_run: reads the stop flag between batches
    int *poll_h = nullptr;               // pinned host word for that read
    rbg_ortho ortho = RBG_ORTHO_MGS;
    alignas(64) unsigned char imgs_tm[128] = {};  // tensor map of Q (k_imgs' basis pipe)
    bool imgs_tm_ok = false;
    bool xmode = false;          // explicit residuals (Algorithm 2 updates)
    double *w_true = nullptr;    // explicit mode: the caller's weights (w holds ones)
    double2 *cgs_v = nullptr, *cgs_c = nullptr;
    int cgs_grid = 0;
    // PEER exchange: this rank's record array, every rank's record array and send slots
    // (own pointers or CUDA-IPC mappings), which of them were opened through IPC
    PeerRec *peer_in = nullptr;
    PeerRec *peer_rec[kMaxPeers] = {};
    unsigned char *peer_send[kMaxPeers] = {};
    bool peer_ipc[kMaxPeers] = {};
    bool peer_connected = false;
    long long peer_timeout_ns = 0;
    // sharded enrichment: global index of each local column (sorted) once columns were
    // appended, and the record-tag epoch (bumped by every sharded append)
    long long *gid = nullptr;
    unsigned long long epoch = 0;
    long long *imgs_trace = nullptr;  // RBG_DEBUG_IMGS=<iteration>: phase clocks of that IMGS
    long long trace_iter = -1;
    rbg::ScratchPool scratch;         // work buffers of the NEXT-row calls, kept between calls
};

namespace rbg_api {

// helpers (api.cu)
void free_ctx(rbg_ctx *c);
SweepArgs sweep_args(const rbg_ctx *c);
ImgsArgs imgs_args(const rbg_ctx *c);
rbg_status check_ctx(rbg_ctx *c);
rbg_status read_state(rbg_ctx *c, DevState *h);
rbg_status need_settled(const rbg_ctx *c, const DevState &h, const char *what);
rbg_status upload_block(rbg_ctx *c, const void *src, long long Mb, long long ld, rbg_mem mem, double2 **out,
                        bool *owned);  // *owned = false: a device block read in place
rbg_status coeff_passes(rbg_ctx *c, const double2 *V, long long Mv, double *R, long long ldr, double *r2,
                        long long k);

}  // namespace rbg_api
