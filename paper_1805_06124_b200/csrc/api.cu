// api.cu -- the C ABI (include/rbg.h): argument checking, device memory, the iteration
// loop (plain launches or CUDA-graph batches), sharded exchange, getters.  (The NEXT-row
// entry points live in api_next.cu; the context and shared helpers in ctx.h.)
//
// One iteration of Algorithm 3 is enqueued as three stream-ordered
// steps with no host synchronisation:
//     local  : fused sweep with q_{k-1} (sweep 0 = weighted norms) + local maxloc
//              [+ pack of the local candidate column, PEER: record stores to every rank]
//                                                                          -> sweep.cu
//     xchg   : PEER wait for the ranks' records (peer.cu) or ncclAllGather of one slot per
//              rank (comm.cpp); sharded runs only
//     finish : global pivot decision, stop test, IMGS of s_J -> q_k        -> imgs.cu
// The loop state (k, stop flag, maxloc) lives in device memory, so the host only
// enqueues; steps after the stop decision return immediately on the device.  The cost
// model T_j = T_pivot + T_IMGS + C_j is measured with CUDA events
// around the three steps when timing is on.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "ctx.h"

using namespace rbg;
using namespace rbg_api;

namespace rbg_api {

thread_local std::string g_err;

rbg_status fail(rbg_status s, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}


void free_ctx(rbg_ctx *c) {
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->imgs_trace) {  // RBG_DEBUG_IMGS: mean cycles per phase over the traced MGS steps
        long long t[32 * 8];
        if (cudaMemcpy(t, c->imgs_trace, sizeof t, cudaMemcpyDeviceToHost) == cudaSuccess && t[5] > 0) {
            // t: 0 step start, 1 after dot, 2 after reduction start (butterfly, CTA tree, send),
            // 3 after the loads overlapped with the round trip, 4 coefficient known, 5 after
            // axpy; 7 = remote partials arrived (PRE reducer)
            double ph[5] = {0, 0, 0, 0, 0}, step = 0, remote = 0;
            int n = 0;
            for (int i = 0; i < 32 && t[i * 8 + 5] > 0; i++, n++) {
                for (int p = 0; p < 5; p++) ph[p] += (double)(t[i * 8 + p + 1] - t[i * 8 + p]);
                if (t[i * 8 + 7]) remote += (double)(t[i * 8 + 7] - t[i * 8 + 3]);
                if (i + 1 < 32 && t[(i + 1) * 8] > 0) step += (double)(t[(i + 1) * 8] - t[i * 8]);
            }
            if (n > 1)
                fprintf(stderr, "rbg: imgs iteration %lld, %d steps: dot %.0f, reduce-start %.0f, overlapped loads %.0f, "
                                "reduce-finish %.0f (remote wait %.0f), axpy %.0f, step %.0f cycles\n",
                        c->trace_iter, n, ph[0] / n, ph[1] / n, ph[2] / n, ph[3] / n, remote / n, ph[4] / n,
                        step / (n - 1));
        }
        // every CTA's step timestamps (steps 64..71): send skew across CTAs and the latency from
        // the last CTA's send to each CTA's coefficient
        unsigned long long gt[16 * 8 * 4];
        if (cudaMemcpy(gt, c->imgs_trace + 512, sizeof gt, cudaMemcpyDeviceToHost) == cudaSuccess && gt[2]) {
            double skew = 0, lat = 0, busy = 0, step = 0;
            int n = 0;
            for (int st = 0; st < 8; st++) {
                unsigned long long smin = ~0ull, smax = 0, cmax = 0, c0max = 0;
                int have = 0;
                double b = 0;
                for (int r = 0; r < 16; r++) {
                    const unsigned long long *g = gt + (r * 8 + st) * 4;
                    if (!g[1]) continue;
                    have++;
                    smin = std::min(smin, g[1]);
                    smax = std::max(smax, g[1]);
                    cmax = std::max(cmax, g[2]);
                    c0max = std::max(c0max, g[0]);
                    b += (double)(g[1] - g[0]);
                }
                if (!have) continue;
                skew += (double)(smax - smin);
                lat += (double)(cmax - smax);
                if (st + 1 < 8) {
                    unsigned long long nmax = 0;
                    for (int r = 0; r < 16; r++) nmax = std::max(nmax, gt[(r * 8 + st + 1) * 4]);
                    if (nmax) step += (double)(nmax - c0max);
                }
                n++;
                busy += b / have;
            }
            if (n > 1) {
                fprintf(stderr, "rbg: imgs cluster (ns/step): send skew across CTAs %.0f, last send -> last coefficient %.0f, "
                                "step start -> send %.0f, step %.0f\n", skew / n, lat / n, busy / n, step / (n - 1));
                // per CTA: mean send time and coefficient time relative to the step's first send
                fprintf(stderr, "rbg: imgs per CTA (ns after the first send: send / stage ready / coefficient):");
                for (int r = 0; r < 16; r++) {
                    double ds = 0, dc = 0, dg = 0;
                    int m = 0;
                    for (int st = 0; st < 8; st++) {
                        unsigned long long smin = ~0ull;
                        for (int q = 0; q < 16; q++)
                            if (gt[(q * 8 + st) * 4 + 1]) smin = std::min(smin, gt[(q * 8 + st) * 4 + 1]);
                        const unsigned long long *g = gt + (r * 8 + st) * 4;
                        if (!g[1] || smin == ~0ull) continue;
                        ds += (double)(g[1] - smin);
                        dc += (double)(g[2] - smin);
                        dg += (double)(g[3] - smin);
                        m++;
                    }
                    if (m) fprintf(stderr, " %d:%.0f/%.0f/%.0f", r, ds / m, dg / m, dc / m);
                }
                fprintf(stderr, "\n");
                // producer: stage s+1 issued how long before the consumers had it (ns)
                unsigned long long ti[16 * 8];
                if (cudaMemcpy(ti, c->imgs_trace + 320, sizeof ti, cudaMemcpyDeviceToHost) == cudaSuccess) {
                    fprintf(stderr, "rbg: imgs per CTA stage s+1: issued -> ready (ns):");
                    for (int r = 0; r < 16; r++) {
                        double d = 0;
                        int m = 0;
                        for (int st = 0; st < 8; st++) {
                            const unsigned long long iss = ti[r * 8 + st], rdy = gt[(r * 8 + st) * 4 + 3];
                            if (iss && rdy) {
                                d += (double)(long long)(rdy - iss);
                                m++;
                            }
                        }
                        if (m) fprintf(stderr, " %d:%.0f", r, d / m);
                    }
                    fprintf(stderr, "\n");
                }
            }
        }
        // %globaltimer (ns): [256] sweep's last CTA done, [257] IMGS entry, [258] cluster synced,
        // [259] after grid_dep_wait, [260] n0 known, [261] MGS sweeps done, [262] q stored
        unsigned long long g[8];
        if (cudaMemcpy(g, c->imgs_trace + 256, sizeof g, cudaMemcpyDeviceToHost) == cudaSuccess && g[1] && g[6]) {
            auto d = [&](int a, int b) { return (g[a] && g[b]) ? (double)(long long)(g[b] - g[a]) * 1e-3 : -1.0; };
            fprintf(stderr, "rbg: imgs iteration %lld phases (us): sweep-end->entry %.2f, entry->cluster sync %.2f, "
                            "->grid_dep_wait %.2f, ->n0 %.2f, ->MGS done %.2f, ->q stored %.2f (entry->end %.2f)\n",
                    c->trace_iter, d(0, 1), d(1, 2), d(2, 3), d(3, 4), d(4, 5), d(5, 6), d(1, 6));
        }
        dfree(c->imgs_trace);
    }
    if (c->graph) cudaGraphExecDestroy(c->graph);
    if (c->while_exec) cudaGraphExecDestroy(c->while_exec);
    if (c->poll_stream) cudaStreamDestroy(c->poll_stream);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    if (c->poll_h) cudaFreeHost(c->poll_h);
    for (auto &p : c->ev)
        for (int i = 0; i < 4; i++) cudaEventDestroy(p.e[i]);
    if (c->nccl) nccl_destroy(c->nccl);
    for (int q = 0; q < kMaxPeers; q++)
        if (c->peer_ipc[q]) {
            cudaIpcCloseMemHandle(c->peer_rec[q]);
            cudaIpcCloseMemHandle(c->peer_send[q]);
        }
    dfree(c->peer_in);
    dfree(c->gid);
    if (c->own_S) dfree(c->S);
    dfree(c->S1);
    dfree(c->w);
    dfree(c->Q);
    dfree(c->WQ);
    dfree(c->R);
    dfree(c->r2);
    dfree(c->st);
    dfree(c->errors);
    dfree(c->rdiag);
    dfree(c->piv);
    dfree(c->nu);
    dfree(c->recs);
    dfree(c->ticket);
    dfree(c->next_col);
    dfree(c->send);
    dfree(c->recv);
    dfree(c->cgs_v);
    dfree(c->w_true);
    dfree(c->cgs_c);
    c->scratch.release();
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

// Programmatic dependent launches (sweep after the decision kernel, decision/IMGS after the
// sweep): not with per-phase events between the kernels (timing mode), and the IMGS side only
// on one GPU (its predecessor there is the sweep, never the exchange wait that can set stop).
static bool pdl_enabled(const rbg_ctx *c) {
    static const bool off = getenv("RBG_NO_PDL") != nullptr;
    return !off && !c->timing;
}

SweepArgs sweep_args(const rbg_ctx *c) {
    SweepArgs a;
    a.S = c->S;
    a.ldv = c->ldv;
    a.S1 = c->S1;
    a.M0 = c->M0;
    a.M = c->M;
    a.N = c->N;
    a.nvec = c->nvec;
    a.w = c->w;
    a.WQ = c->WQ;
    a.ldq_v = c->ldq_v;
    a.R = c->R;
    a.ldr = c->ldr;
    a.qi = -1;
    a.V = c->xmode ? c->S : nullptr;
    a.r2 = c->r2;
    a.st = c->st;
    a.recs = c->recs;
    a.ticket = c->ticket;
    a.next_col = c->next_col;
    a.col_offset = c->col_offset;
    a.send = c->comm != RBG_COMM_NONE ? c->send : nullptr;
    a.peer_world = 0;
    a.peer_rank = c->rank;
    a.peer_slot = c->slot;
    for (int q = 0; q < kMaxPeers; q++) a.peer_in[q] = nullptr;
    if (c->comm == RBG_COMM_PEER) {
        a.peer_world = c->world;
        for (int q = 0; q < c->world; q++) a.peer_in[q] = c->peer_rec[q];
    }
    a.peer_epoch = c->epoch;
    a.gid = c->gid;
    a.cond = c->cond;
    a.use_cond = c->in_while ? 1 : 0;
    a.pdl = pdl_enabled(c) ? 1 : 0;
    static const bool no_tail_pf = getenv("RBG_NO_TAIL_PF") != nullptr;
    a.tail_pf = no_tail_pf ? 0 : 1;
    a.tstamp = (c->imgs_trace && c->iters == c->trace_iter) ? reinterpret_cast<unsigned long long *>(c->imgs_trace) + 256
                                                          : nullptr;
    return a;
}

ImgsArgs imgs_args(const rbg_ctx *c) {
    ImgsArgs a;
    a.S = c->S;
    a.ldv = c->ldv;
    a.S1 = c->S1;
    a.M0 = c->M0;
    a.N = c->N;
    a.nvec = c->nvec;
    a.w = c->w;
    a.Q = c->Q;
    a.WQ = c->WQ;
    a.ldq_v = c->ldq_v;
    a.st = c->st;
    a.errors = c->errors;
    a.piv = c->piv;
    a.nu = c->nu;
    a.rdiag = c->rdiag;
    a.r2 = c->r2;
    a.k_max = c->k_max;
    a.tol = c->tol;
    a.col_offset = c->col_offset;
    a.M_loc = c->M;
    a.world = c->world;
    a.xchg = c->comm != RBG_COMM_NONE;
    a.recv = c->recv;
    a.slot_bytes = c->slot;
    a.peer_mine = c->comm == RBG_COMM_PEER ? c->peer_in : nullptr;
    a.peer_slot = c->slot;
    for (int q = 0; q < kMaxPeers; q++) a.peer_send[q] = q < c->world ? c->peer_send[q] : nullptr;
    a.gid = c->gid;
    a.trace = (c->imgs_trace && c->iters == c->trace_iter) ? c->imgs_trace : nullptr;
    a.cond = c->cond;
    a.use_cond = c->in_while ? 1 : 0;
    a.pdl = (pdl_enabled(c) && c->comm == RBG_COMM_NONE && c->started) ? 1 : 0;
    a.tm = c->imgs_tm_ok ? c->imgs_tm : nullptr;
    a.use_tm = c->imgs_tm_ok ? 1 : 0;
    return a;
}

rbg_status enqueue_local(rbg_ctx *c) {
    NvtxRange range("rbg.sweep");
    if (c->resume_pending) {  // r2 / R of the added columns are already up to date
        c->resume_pending = false;
        return RBG_OK;
    }
    const bool init = !c->started;
    CU(launch_sweep(sweep_args(c), c->cplx, init, init ? c->cfg_init : c->cfg_sweep, c->stream));
    c->started = true;
    return RBG_OK;
}

rbg_status enqueue_xchg(rbg_ctx *c) {
    NvtxRange range("rbg.exchange");
    if (c->comm == RBG_COMM_PEER) {
        CU(launch_peer_wait(c->peer_in, c->world, c->st, c->epoch, c->peer_timeout_ns, c->cond, c->in_while ? 1 : 0,
                            c->stream));
        return RBG_OK;
    }
    if (c->comm == RBG_COMM_NCCL) {
        const char *msg = nullptr;
        if (nccl_allgather_bytes(c->send, c->recv, c->slot, c->nccl, c->stream, &msg))
            return fail(RBG_ENCCL, "ncclAllGather: %s", msg ? msg : "?");
    }
    return RBG_OK;
}

rbg_status enqueue_finish(rbg_ctx *c) {
    NvtxRange range("rbg.imgs");
    if (c->ortho == RBG_ORTHO_CGS)
        CU(launch_imgs_cgs(imgs_args(c), c->cplx, c->cgs_v, c->cgs_c, c->cgs_grid, c->stream));
    else
        CU(launch_imgs(imgs_args(c), c->cplx, c->stream));
    return RBG_OK;
}

rbg_status enqueue_iteration(rbg_ctx *c) {
    NvtxRange range("rbg.iteration");
    PhaseEvents *pe = nullptr;
    if (c->timing) {
        PhaseEvents p;
        for (int i = 0; i < 4; i++) CU(cudaEventCreate(&p.e[i]));
        c->ev.push_back(p);
        c->ev_iter.push_back(c->iters);
        pe = &c->ev.back();
        CU(cudaEventRecord(pe->e[0], c->stream));
    }
    TRY(enqueue_local(c));
    if (pe) CU(cudaEventRecord(pe->e[1], c->stream));
    TRY(enqueue_xchg(c));
    if (pe) CU(cudaEventRecord(pe->e[2], c->stream));
    TRY(enqueue_finish(c));
    if (pe) CU(cudaEventRecord(pe->e[3], c->stream));
    c->iters++;
    return RBG_OK;
}

// Graphs are captured on a private stream (the caller's stream may be the legacy default
// stream, which cannot be captured) and launched on the context's stream.
struct CaptureStream {
    rbg_ctx *c;
    cudaStream_t keep;
    explicit CaptureStream(rbg_ctx *ctx) : c(ctx), keep(ctx->stream) { c->stream = c->cap_stream; }
    ~CaptureStream() { c->stream = keep; }
};

rbg_status build_graph(rbg_ctx *c) {
    if (c->graph) return RBG_OK;
    if (!c->cap_stream) CU(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g;
    rbg_status s = RBG_OK;
    cudaError_t e;
    {
        CaptureStream cs(c);
        CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < c->graph_batch && s == RBG_OK; i++) {
            s = enqueue_local(c);
            if (s == RBG_OK) s = enqueue_xchg(c);
            if (s == RBG_OK) s = enqueue_finish(c);
        }
        e = cudaStreamEndCapture(c->stream, &g);
    }
    if (s != RBG_OK) return s;
    CU(e);
    e = cudaGraphInstantiate(&c->graph, g, 0);
    cudaGraphDestroy(g);
    CU(e);
    return RBG_OK;
}

rbg_status enqueue_n(rbg_ctx *c, long long n) {
    while (n > 0) {
        if (!c->started || c->resume_pending || c->timing || c->graph_batch <= 0 || n < c->graph_batch) {
            TRY(enqueue_iteration(c));
            n--;
            continue;
        }
        TRY(build_graph(c));
        CU(cudaGraphLaunch(c->graph, c->stream));
        c->iters += c->graph_batch;
        n -= c->graph_batch;
    }
    return RBG_OK;
}

// rbg_run's device loop: a graph whose only node is a conditional WHILE node (condition 1 at
// launch) with one steady-state iteration -- sweep with q_{k-1} [+ exchange wait] + decision and
// IMGS -- as its body.  The kernels in the body carry the condition handle; the one that
// records the stop decision, or first finds the greedy stopped, sets it to 0 (loop_exit in
// common.cuh), so the loop ends after the stopping iteration: no host round trip per
// iteration and no launches past the stop.  NCCL's collective (its own kernels) and the
// per-phase timing events stay outside (rbg_run polls then), as does the IMGS debug trace.
bool while_supported(const rbg_ctx *c) {
    return !c->while_failed && !c->timing && !c->imgs_trace && (c->comm == RBG_COMM_NONE || c->comm == RBG_COMM_PEER) &&
           !getenv("RBG_NO_DEVICE_LOOP");
}

rbg_status build_while(rbg_ctx *c) {
    if (c->while_exec) return RBG_OK;
    if (!c->cap_stream) CU(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    CaptureStream cs(c);
    cudaGraph_t g = nullptr;
    CU(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    if (e == cudaSuccess) e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
    cudaGraph_t body = p.conditional.phGraph_out ? p.conditional.phGraph_out[0] : nullptr;
    if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    rbg_status s = RBG_OK;
    if (e == cudaSuccess) {
        c->cond = h;
        c->in_while = true;
        s = enqueue_local(c);
        if (s == RBG_OK) s = enqueue_xchg(c);
        if (s == RBG_OK) s = enqueue_finish(c);
        c->in_while = false;
        cudaGraph_t out = nullptr;
        const cudaError_t e2 = cudaStreamEndCapture(c->stream, &out);
        if (e2 != cudaSuccess) e = e2;
    }
    if (e == cudaSuccess && s == RBG_OK) e = cudaGraphInstantiate(&c->while_exec, g, 0);
    cudaGraphDestroy(g);
    if (s != RBG_OK) return s;
    if (e != cudaSuccess) {
        c->while_exec = nullptr;
        return fail(RBG_ECUDA, "device loop graph: %s", cudaGetErrorString(e));
    }
    return RBG_OK;
}

// Polled rbg_run (timing mode, NCCL, or no device loop): batches of `graph_batch` (default 16)
// iterations, one batch in flight ahead; before enqueuing the next batch the host reads the
// stop flag as of the end of the batch before (side stream, pinned word), so at most two
// batches run past the stop (as early-exit kernels).
rbg_status run_polled(rbg_ctx *c) {
    const long long B = c->graph_batch > 0 ? c->graph_batch : 16;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    rbg_status s = RBG_OK;
    cudaError_t e = cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
    long long b = 0;
    bool stopped = false;
    while (e == cudaSuccess && s == RBG_OK && !stopped && c->iters < c->k_max + 1) {
        s = enqueue_n(c, std::min<long long>(B, c->k_max + 1 - c->iters));
        if (s != RBG_OK) break;
        e = cudaEventRecord(ev[b & 1], c->stream);
        if (e == cudaSuccess && b > 0) {
            e = cudaStreamWaitEvent(c->poll_stream, ev[(b - 1) & 1], 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(c->poll_h, &c->st->stop, sizeof(int), cudaMemcpyDeviceToHost, c->poll_stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(c->poll_stream);
            stopped = e == cudaSuccess && *c->poll_h != 0;
        }
        b++;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    for (auto &x : ev)
        if (x) cudaEventDestroy(x);
    if (s != RBG_OK) return s;
    if (e != cudaSuccess) return fail(RBG_ECUDA, "rbg_run: %s", cudaGetErrorString(e));
    DevState h;
    TRY(read_state(c, &h));
    c->stopped = h.stop != 0 || c->iters >= c->k_max + 1;
    return RBG_OK;
}

rbg_status check_ctx(rbg_ctx *c) {
    if (!c) return fail(RBG_EINVAL, "null context");
    CU(cudaSetDevice(c->device));
    return RBG_OK;
}

rbg_status read_state(rbg_ctx *c, DevState *h) {
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaMemcpy(h, c->st, sizeof(DevState), cudaMemcpyDeviceToHost));
    return RBG_OK;
}

// Calls that read R (or change the column set) need every R row 0..k-1 filled: before the
// first iteration, after a stop decision, or after rbg_add_columns (rows computed for the new
// columns).  Between rbg_step calls of a running greedy the sweep with q_{k-1} is still
// pending, i.e. R row k-1 is zero and r2 lacks |c_{k-1,j}|^2.
rbg_status need_settled(const rbg_ctx *c, const DevState &h, const char *what) {
    if (c->local_pending) return fail(RBG_ESTATE, "%s inside an EXTERNAL/PEER iteration", what);
    if (c->started && h.stop == 0 && !c->resume_pending)
        return fail(RBG_ESTATE, "%s on a running greedy (k=%lld, no stop decision yet): run it to its stop first",
                    what, h.k);
    return RBG_OK;
}

// Device copy of a caller block in the library's column layout (nvec 16-byte vectors per
// column, zero padded), with the NaN/Inf scan.  *out is owned by the caller of this helper.
rbg_status upload_block(rbg_ctx *c, const void *src, long long Mb, long long ld, rbg_mem mem, double2 **out,
                        bool *owned) {
    *out = nullptr;
    *owned = false;
    if (!src || Mb < 1) return fail(RBG_EINVAL, "null block or no columns");
    if (ld == 0) ld = c->N;
    if (ld < c->N) return fail(RBG_EINVAL, "ld=%lld < N=%lld", ld, c->N);
    const size_t pitch = (size_t)c->nvec * 16, col_bytes = (size_t)c->N * c->se;
    // a device block already in the padded layout (16-byte aligned, column pitch nvec*16) is
    // read in place for the duration of the call; anything else is copied
    const bool borrow = mem == RBG_MEM_DEVICE && (size_t)ld * c->se == pitch && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    double2 *d = nullptr;
    cudaError_t e = cudaSuccess;
    if (borrow) {
        d = const_cast<double2 *>(static_cast<const double2 *>(src));
    } else {
        CU(dmalloc(&d, pitch * Mb));
        *owned = true;
        const cudaMemcpyKind kind = mem == RBG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        if (pitch != col_bytes) e = cudaMemsetAsync(d, 0, pitch * Mb, c->stream);
        if (e == cudaSuccess) e = cudaMemcpy2DAsync(d, pitch, src, (size_t)ld * c->se, col_bytes, Mb, kind, c->stream);
    }
    unsigned long long *bad = nullptr, hbad = ~0ull;
    if (e == cudaSuccess) e = dmalloc(&bad, sizeof *bad);
    if (e == cudaSuccess) e = cudaMemcpyAsync(bad, &hbad, sizeof hbad, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = launch_check_finite(d, c->nvec, Mb, c->N, c->nvec, c->cplx, bad, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    dfree(bad);
    if (e != cudaSuccess) {
        if (*owned) dfree(d);
        *owned = false;
        return fail(RBG_ECUDA, "uploading a column block: %s", cudaGetErrorString(e));
    }
    if (hbad != ~0ull) {
        if (*owned) dfree(d);
        *owned = false;
        return fail(RBG_ENONFINITE, "non-finite entry at (row %lld, col %lld)", (long long)(hbad % c->N),
                    (long long)(hbad / c->N));
    }
    *out = d;
    return RBG_OK;
}

// Sweep 0 and sweeps with q_0..q_{k-1} over an extra column block: exactly the per-column
// arithmetic the block would have received inside the greedy (R rows, recurrence r2).
rbg_status coeff_passes(rbg_ctx *c, const double2 *V, long long Mv, double *R, long long ldr, double *r2,
                        long long k) {
    DevState *vst = nullptr;
    Rec *recs = nullptr;
    unsigned *ticket = nullptr;
    const int grid = std::max(c->cfg_init.grid, c->cfg_sweep.grid);
    cudaError_t e = dmalloc(&vst, sizeof(DevState));
    if (e == cudaSuccess) e = dmalloc(&recs, sizeof(Rec) * grid);
    unsigned long long *ncol = nullptr;
    if (e == cudaSuccess) e = dmalloc(&ticket, sizeof(unsigned));
    if (e == cudaSuccess) e = dmalloc(&ncol, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemsetAsync(vst, 0, sizeof(DevState), c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(ticket, 0, sizeof(unsigned), c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(ncol, 0, sizeof(unsigned long long), c->stream);
    SweepArgs a = sweep_args(c);
    a.S = V;
    a.ldv = c->nvec;
    a.S1 = nullptr;
    a.M0 = Mv;
    a.M = Mv;
    a.R = R;
    a.ldr = ldr;
    a.r2 = r2;
    a.st = vst;
    a.recs = recs;
    a.ticket = ticket;
    a.next_col = ncol;
    a.col_offset = 0;
    a.send = nullptr;
    a.peer_world = 0;   // a block outside the training set: no exchange, its own indices
    a.gid = nullptr;
    a.qi = -1;
    if (e == cudaSuccess) e = launch_sweep(a, c->cplx, true, c->cfg_init, c->stream);
    if (coeff_block_enabled()) {  // one blocked pass for all k basis vectors (coeff.cu)
        if (e == cudaSuccess)
            e = launch_coeff_block(V, c->nvec, Mv, c->WQ, c->ldq_v, k, c->nvec, c->N, c->cplx, R, ldr, r2, c->stream);
    } else {
        for (long long i = 0; i < k && e == cudaSuccess; i++) {
            a.qi = i;
            e = launch_sweep(a, c->cplx, false, c->cfg_sweep, c->stream);
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    dfree(vst);
    dfree(recs);
    dfree(ticket);
    dfree(ncol);
    if (e != cudaSuccess) return fail(RBG_ECUDA, "coefficient passes: %s", cudaGetErrorString(e));
    return RBG_OK;
}


}  // namespace rbg_api

extern "C" {

void rbg_desc_init(rbg_desc *d) {
    if (!d) return;
    std::memset(d, 0, sizeof *d);
    d->S_mem = RBG_MEM_HOST;
    d->w_mem = RBG_MEM_HOST;
    d->dtype = RBG_COMPLEX_F64;
    d->device = -1;
    d->check_finite = 1;
    d->comm = RBG_COMM_NONE;
    d->world = 1;
    d->ortho = RBG_ORTHO_MGS;
    d->residual = RBG_RESIDUAL_RECURRENCE;
}

const char *rbg_last_error(void) { return g_err.c_str(); }

void rbg_debug_set_canary(int on) { debug_set_canary(on != 0); }

int64_t rbg_debug_canary_violations(void) {
    std::string msg;
    const long long n = debug_canary_violations(&msg);
    if (n) g_err = msg;
    return n;
}

void rbg_lanes(int *L_S, int *L_I) {
    if (L_S) *L_S = kLaneSweep;
    if (L_I) *L_I = kLaneImgs;
}

const char *rbg_version(void) { return "rbg 0.1 sm_100a L_S=32 L_I=2048 kappa=2 nu_max=5"; }

rbg_status rbg_get_unique_id(uint8_t out[128]) {
    if (!out) return fail(RBG_EINVAL, "null output");
    const char *msg = nullptr;
    if (nccl_get_unique_id(out, &msg)) return fail(RBG_ENCCL, "ncclGetUniqueId: %s", msg ? msg : "?");
    return RBG_OK;
}

rbg_status rbg_create_ex(rbg_ctx **out, const rbg_desc *d) {
    if (!out || !d) return fail(RBG_EINVAL, "null ctx or desc");
    *out = nullptr;
    if (!d->S) return fail(RBG_EINVAL, "null S");
    if (d->dtype != RBG_REAL_F64 && d->dtype != RBG_COMPLEX_F64) return fail(RBG_EINVAL, "unknown dtype %d", (int)d->dtype);
    if (d->N < 1 || d->M < 1) return fail(RBG_EINVAL, "N=%lld M=%lld must be >= 1", (long long)d->N, (long long)d->M);
    const long long ld = d->ld ? d->ld : d->N;
    if (ld < d->N) return fail(RBG_EINVAL, "ld=%lld < N=%lld", ld, (long long)d->N);
    if (!(d->tol >= 0.0) || std::isinf(d->tol)) return fail(RBG_EINVAL, "tol must be finite and >= 0");
    const int world = d->world < 1 ? 1 : d->world;
    if (d->rank < 0 || d->rank >= world) return fail(RBG_EINVAL, "rank %d outside [0, %d)", d->rank, world);
    const long long Mg = d->M_global ? d->M_global : d->M;
    if (world == 1 && (d->col_offset != 0 || Mg != d->M))
        return fail(RBG_EINVAL, "one rank must own all columns");
    if (d->col_offset < 0 || d->col_offset + d->M > Mg) return fail(RBG_EINVAL, "column range outside M_global");
    // k_max <= N (a basis of R^N); k_max > M is allowed (the greedy stops ALL_SELECTED, or
    // continues after rbg_add_columns)
    if (d->k_max < 1 || d->k_max > d->N)
        return fail(RBG_EINVAL, "k_max=%lld outside [1, N=%lld]", (long long)d->k_max, (long long)d->N);
    if (world > 1 && d->comm == RBG_COMM_NONE) return fail(RBG_EINVAL, "world > 1 needs comm NCCL, EXTERNAL or PEER");
    if (d->comm < RBG_COMM_NONE || d->comm > RBG_COMM_PEER) return fail(RBG_EINVAL, "unknown comm %d", (int)d->comm);
    if (d->comm == RBG_COMM_PEER && world > kMaxPeers)
        return fail(RBG_EINVAL, "PEER exchange supports at most %d ranks", kMaxPeers);
    if (d->ortho != RBG_ORTHO_MGS && d->ortho != RBG_ORTHO_CGS) return fail(RBG_EINVAL, "unknown ortho %d", (int)d->ortho);
    if (d->residual != RBG_RESIDUAL_RECURRENCE && d->residual != RBG_RESIDUAL_EXPLICIT)
        return fail(RBG_EINVAL, "unknown residual mode %d", (int)d->residual);
    const bool cplx = d->dtype == RBG_COMPLEX_F64;
    const long long nvec = cplx ? d->N : (d->N + 1) / 2;
    if (imgs_maxv(nvec) == 0) return fail(RBG_EINVAL, "N=%lld exceeds the IMGS register tile (max %d vectors)", (long long)d->N, 16 * kLaneImgs);

    // weights: validate on the host
    std::vector<double> wh(d->N, 1.0);
    if (d->w) {
        if (d->w_mem == RBG_MEM_DEVICE) {
            cudaError_t e = cudaMemcpy(wh.data(), d->w, sizeof(double) * d->N, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) return fail(RBG_ECUDA, "reading w: %s", cudaGetErrorString(e));
        } else {
            std::memcpy(wh.data(), d->w, sizeof(double) * d->N);
        }
        for (long long i = 0; i < d->N; i++)
            if (!(wh[i] > 0.0) || std::isinf(wh[i])) return fail(RBG_EINVAL, "w[%lld]=%g must be positive and finite", i, wh[i]);
    }
    if (d->S_mem == RBG_MEM_DEVICE && d->borrow) {
        if (reinterpret_cast<uintptr_t>(d->S) % 16) return fail(RBG_EINVAL, "borrowed S must be 16-byte aligned");
        if (!cplx && (ld % 2)) return fail(RBG_EINVAL, "borrowed real S needs an even ld");
    }

    rbg_ctx *c = new rbg_ctx();
    auto bail = [&](rbg_status s) {
        std::string keep = g_err;
        free_ctx(c);
        g_err = keep;
        return s;
    };
#define CUB(call)                                                                                    \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess)                                                                       \
            return bail(fail(e_ == cudaErrorMemoryAllocation ? RBG_ENOMEM : RBG_ECUDA, "%s: %s", #call, \
                             cudaGetErrorString(e_)));                                               \
    } while (0)

    if (d->device >= 0) c->device = d->device;
    else CUB(cudaGetDevice(&c->device));
    CUB(cudaSetDevice(c->device));
    CUB(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
    if (d->stream) c->stream = static_cast<cudaStream_t>(d->stream);
    else {
        CUB(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    c->cplx = cplx;
    c->se = cplx ? 16 : 8;
    c->N = d->N;
    c->M = d->M;
    c->M0 = d->M;
    c->nvec = nvec;
    c->ldq_v = nvec;
    c->tol = d->tol;
    c->k_max = d->k_max;
    c->comm = d->comm;
    c->rank = d->rank;
    c->world = world;
    c->col_offset = d->col_offset;
    c->M_global = Mg;

    // snapshot matrix.  A private copy is uploaded in chunks of ~1 GB on the context's stream;
    // the finiteness scan of each chunk runs on a second stream as soon as the chunk has landed
    // (it overlaps the next chunk's copy), and the verdict is read only at the end of create, so
    // the host-side allocations below overlap the upload too (the e2e bench's create is bounded
    // by the PCIe copy).
    const size_t col_bytes = (size_t)d->N * c->se;
    unsigned long long *bad = nullptr, hbad = ~0ull;
    struct FreeOnExit {  // the flag of a create that fails before the verdict is read
        unsigned long long *&p;
        ~FreeOnExit() {
            if (p) dfree(p);
        }
    } bad_guard{bad};
    if (d->check_finite) {  // first non-finite entry in column-major order, on the device
        CUB(dmalloc(&bad, sizeof *bad));
        CUB(cudaMemcpyAsync(bad, &hbad, sizeof hbad, cudaMemcpyHostToDevice, c->stream));
    }
    CUB(cudaStreamCreateWithFlags(&c->poll_stream, cudaStreamNonBlocking));
    if (d->S_mem == RBG_MEM_DEVICE && d->borrow) {
        c->S = const_cast<double2 *>(static_cast<const double2 *>(d->S));
        c->ldv = cplx ? ld : ld / 2;
        if (bad) CUB(launch_check_finite(c->S, c->ldv, c->M, c->N, nvec, cplx, bad, c->stream));
    } else {
        c->ldv = nvec;
        const size_t dst_pitch = (size_t)nvec * 16;
        CUB(dmalloc(&c->S, dst_pitch * d->M));
        c->own_S = true;
        if (dst_pitch != col_bytes) CUB(cudaMemsetAsync(c->S, 0, dst_pitch * d->M, c->stream));
        const cudaMemcpyKind kind = d->S_mem == RBG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        const bool flat = dst_pitch == col_bytes && (size_t)ld * c->se == col_bytes;
        long long per = std::max<long long>(1, (1LL << 30) / (long long)dst_pitch);   // columns per chunk
        if (const char *e = getenv("RBG_UPLOAD_CHUNK_COLS")) per = std::max<long long>(1, atoll(e));   // tests
        cudaEvent_t ev = nullptr;
        if (bad) CUB(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        for (long long c0 = 0; c0 < d->M; c0 += per) {
            const long long mc = std::min<long long>(per, d->M - c0);
            const char *src = static_cast<const char *>(d->S) + (size_t)c0 * ld * c->se;
            double2 *dst = c->S + (size_t)c0 * nvec;
            cudaError_t e = flat ? cudaMemcpyAsync(dst, src, col_bytes * mc, kind, c->stream)
                                 : cudaMemcpy2DAsync(dst, dst_pitch, src, (size_t)ld * c->se, col_bytes, mc, kind, c->stream);
            if (e == cudaSuccess && bad) e = cudaEventRecord(ev, c->stream);
            if (e == cudaSuccess && bad) e = cudaStreamWaitEvent(c->poll_stream, ev, 0);
            if (e == cudaSuccess && bad) e = launch_check_finite(dst, nvec, mc, c->N, nvec, cplx, bad, c->poll_stream, c0);
            if (e != cudaSuccess) {
                if (ev) cudaEventDestroy(ev);
                CUB(e);
            }
        }
        if (bad) {  // the context's stream continues after every chunk's scan
            cudaError_t e = cudaEventRecord(ev, c->poll_stream);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(c->stream, ev, 0);
            cudaEventDestroy(ev);
            CUB(e);
        }
    }
    if (bad) CUB(cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, c->stream));
    auto nonfinite = [&]() -> bool {  // after a synchronisation of c->stream
        if (!bad) return false;
        dfree(bad);
        bad = nullptr;
        return hbad != ~0ull;
    };
    auto nonfinite_fail = [&]() {
        return bail(fail(RBG_ENONFINITE, "non-finite S entry at (row %lld, col %lld)", (long long)(hbad % d->N),
                         (long long)(hbad / d->N) + d->col_offset));
    };

    // weights (zero padded), basis, coefficients, state
    std::vector<double> wpad(2 * nvec + 2, 0.0);
    std::memcpy(wpad.data(), wh.data(), sizeof(double) * d->N);
    c->xmode = d->residual == RBG_RESIDUAL_EXPLICIT;
    if (c->xmode) {
        // the kernels see V = W^{1/2} S with unit weights; w_true keeps the caller's weights
        CUB(dmalloc(&c->w_true, sizeof(double) * wpad.size()));
        CUB(cudaMemcpyAsync(c->w_true, wpad.data(), sizeof(double) * wpad.size(), cudaMemcpyHostToDevice, c->stream));
        double2 *V = nullptr;
        if (c->own_S) V = c->S;                               // scale the private copy in place
        else CUB(dmalloc(&V, (size_t)nvec * 16 * c->M));
        CUB(cudaStreamSynchronize(c->stream));  // the scan's verdict before S is scaled
        if (nonfinite()) return nonfinite_fail();
        CUB(launch_scale_sqrtw(V, nvec, c->S, c->ldv, c->M, nvec, c->N, c->w_true, cplx, c->stream));
        c->S = V;
        c->own_S = true;
        c->ldv = nvec;
        CUB(cudaStreamSynchronize(c->stream));
        std::vector<double> ones(2 * nvec + 2, 0.0);
        for (long long i = 0; i < d->N; i++) ones[i] = 1.0;
        wpad.swap(ones);
    }
    CUB(dmalloc(&c->w, sizeof(double) * wpad.size()));
    CUB(cudaMemcpyAsync(c->w, wpad.data(), sizeof(double) * wpad.size(), cudaMemcpyHostToDevice, c->stream));
    // + imgs_basis_pad: the IMGS tensor-map boxes of the last basis vector stay in bounds
    const size_t qbytes = ((size_t)c->k_max * nvec + (size_t)imgs_basis_pad(nvec)) * 16;
    CUB(dmalloc(&c->Q, qbytes));
    CUB(dmalloc(&c->WQ, qbytes));
    CUB(cudaMemsetAsync(c->Q, 0, qbytes, c->stream));
    CUB(cudaMemsetAsync(c->WQ, 0, qbytes, c->stream));
    c->imgs_tm_ok = make_imgs_maps(c->Q, nvec, c->ldq_v, c->k_max, c->imgs_tm);
    c->ldr = c->M;
    CUB(dmalloc(&c->R, (size_t)c->k_max * c->M * c->se));
    CUB(cudaMemsetAsync(c->R, 0, (size_t)c->k_max * c->M * c->se, c->stream));
    CUB(dmalloc(&c->r2, sizeof(double) * c->M));
    CUB(dmalloc(&c->st, sizeof(DevState)));
    CUB(cudaMemsetAsync(c->st, 0, sizeof(DevState), c->stream));
    CUB(dmalloc(&c->errors, sizeof(double) * (c->k_max + 1)));
    CUB(cudaMemsetAsync(c->errors, 0, sizeof(double) * (c->k_max + 1), c->stream));
    CUB(dmalloc(&c->rdiag, sizeof(double) * c->k_max));
    CUB(dmalloc(&c->piv, sizeof(long long) * c->k_max));
    CUB(dmalloc(&c->nu, sizeof(int) * c->k_max));
    CUB(cudaMemsetAsync(c->nu, 0, sizeof(int) * c->k_max, c->stream));
    c->ortho = d->ortho;
    if (c->ortho == RBG_ORTHO_CGS) {
        CUB(dmalloc(&c->cgs_v, (size_t)nvec * 16));
        CUB(dmalloc(&c->cgs_c, sizeof(double2) * (size_t)c->k_max));
        c->cgs_grid = cgs_grid(c->num_sms);
    }
    if (const char *ti = getenv("RBG_DEBUG_IMGS")) {
        c->trace_iter = atoll(ti);
        CUB(dmalloc(&c->imgs_trace, 1024 * sizeof(long long)));
        CUB(cudaMemsetAsync(c->imgs_trace, 0, 1024 * sizeof(long long), c->stream));
    }
    c->cfg_init = sweep_config(cplx, true, nvec, c->num_sms, c->device);
    c->cfg_sweep = sweep_config(cplx, false, nvec, c->num_sms, c->device);
    const int max_grid = std::max(c->cfg_init.grid, c->cfg_sweep.grid);
    CUB(dmalloc(&c->recs, sizeof(Rec) * max_grid));
    CUB(dmalloc(&c->ticket, sizeof(unsigned)));
    CUB(cudaMemsetAsync(c->ticket, 0, sizeof(unsigned), c->stream));
    CUB(dmalloc(&c->next_col, sizeof(unsigned long long)));
    CUB(cudaMemsetAsync(c->next_col, 0, sizeof(unsigned long long), c->stream));

    if (d->comm == RBG_COMM_PEER) {  // two send slots (by tag parity) + 2 x world records
        c->slot = (xchg_slot_bytes(nvec) + 15) / 16 * 16;
        CUB(dmalloc(&c->send, 2 * c->slot));
        CUB(cudaMemsetAsync(c->send, 0, 2 * c->slot, c->stream));
        CUB(dmalloc(&c->peer_in, sizeof(PeerRec) * 2 * world));
        CUB(cudaMemsetAsync(c->peer_in, 0, sizeof(PeerRec) * 2 * world, c->stream));  // tag 0: none yet
        c->peer_rec[c->rank] = c->peer_in;
        c->peer_send[c->rank] = c->send;
        c->peer_timeout_ns = (d->peer_timeout_ms > 0 ? d->peer_timeout_ms : 60000) * 1000000LL;
        c->peer_connected = world == 1;
    } else if (d->comm != RBG_COMM_NONE) {  // (world = 1 runs the same exchange path, e.g. in tests)
        c->slot = (xchg_slot_bytes(nvec) + 15) / 16 * 16;
        CUB(dmalloc(&c->send, c->slot));
        CUB(dmalloc(&c->recv, c->slot * world));
        CUB(cudaMemsetAsync(c->send, 0, c->slot, c->stream));
        CUB(cudaMemsetAsync(c->recv, 0, c->slot * world, c->stream));
        if (d->comm == RBG_COMM_NCCL) {
            const char *msg = nullptr;
            if (nccl_init(&c->nccl, world, d->rank, d->nccl_id, &msg))
                return bail(fail(RBG_ENCCL, "ncclCommInitRank: %s", msg ? msg : "?"));
        }
    }
    // rbg_run's helpers, allocated here so that no run pays cudaHostAlloc / stream creation
    // (both synchronise with the device) between its iterations
    CUB(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    CUB(cudaHostAlloc(&c->poll_h, sizeof(int), cudaHostAllocDefault));
    CUB(cudaStreamSynchronize(c->stream));
    if (nonfinite()) return nonfinite_fail();
#undef CUB
    *out = c;
    return RBG_OK;
}

rbg_status rbg_create(rbg_ctx **ctx, const void *S, int64_t N, int64_t M, const double *w, double tol,
                      int64_t k_max, rbg_dtype dtype) {
    rbg_desc d;
    rbg_desc_init(&d);
    d.S = S;
    d.N = N;
    d.M = M;
    d.w = w;
    d.tol = tol;
    d.k_max = k_max;
    d.dtype = dtype;
    return rbg_create_ex(ctx, &d);
}

rbg_status rbg_step(rbg_ctx *c, int64_t n) {
    TRY(check_ctx(c));
    if (c->comm == RBG_COMM_EXTERNAL) return fail(RBG_ESTATE, "EXTERNAL contexts use rbg_iter_local/finish");
    if (c->comm == RBG_COMM_PEER && !c->peer_connected) return fail(RBG_ESTATE, "PEER context not connected (rbg_peer_connect)");
    if (n < 0) return fail(RBG_EINVAL, "n < 0");
    return enqueue_n(c, n);
}

rbg_status rbg_run(rbg_ctx *c) {
    TRY(check_ctx(c));
    if (c->comm == RBG_COMM_EXTERNAL) return fail(RBG_ESTATE, "EXTERNAL contexts use rbg_iter_local/finish");
    if (c->comm == RBG_COMM_PEER && !c->peer_connected) return fail(RBG_ESTATE, "PEER context not connected (rbg_peer_connect)");
    if (c->local_pending) return fail(RBG_ESTATE, "rbg_run inside an iteration (rbg_iter_local pending)");
    if (c->stopped || c->iters >= c->k_max + 1) {  // a previous rbg_run saw the stop
        CU(cudaStreamSynchronize(c->stream));
        return RBG_OK;
    }
    // no host synchronisation here: iterations enqueued by rbg_step run first in stream order
    // (and a greedy they stopped makes the loop below exit at its first kernel)
    DevState h;
    if (while_supported(c)) {
        // sweep 0 (or the restart after rbg_add_columns) is a different kernel: one plain
        // iteration first, then the device loop over the steady-state body
        if (!c->started || c->resume_pending) TRY(enqueue_iteration(c));
        rbg_status s = build_while(c);
        if (s == RBG_OK) {
            CU(cudaGraphLaunch(c->while_exec, c->stream));
            TRY(read_state(c, &h));
            c->iters = h.k + 1;  // iterations 0..k ran; the loop ended at the stop decision
            c->stopped = true;
            return RBG_OK;
        }
        c->while_failed = true;  // e.g. a driver without conditional nodes: poll instead
    }
    return run_polled(c);
}

rbg_status rbg_set_timing(rbg_ctx *c, int on) {
    TRY(check_ctx(c));
    c->timing = on != 0;
    return RBG_OK;
}

rbg_status rbg_set_graph_batch(rbg_ctx *c, int batch) {
    TRY(check_ctx(c));
    if (batch < 0) return fail(RBG_EINVAL, "batch < 0");
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    c->graph_batch = batch;
    return RBG_OK;
}

rbg_status rbg_sync(rbg_ctx *c) {
    TRY(check_ctx(c));
    CU(cudaStreamSynchronize(c->stream));
    return RBG_OK;
}

rbg_status rbg_result_info(rbg_ctx *c, int64_t *k, int64_t *M_loc, rbg_stop *why) {
    TRY(check_ctx(c));
    DevState h;
    TRY(read_state(c, &h));
    if (k) *k = h.k;
    if (M_loc) *M_loc = c->M;
    if (why) *why = (rbg_stop)h.stop;
    return RBG_OK;
}

rbg_status rbg_get_pivots(rbg_ctx *c, int64_t *out) {
    TRY(check_ctx(c));
    if (!out) return fail(RBG_EINVAL, "null output");
    DevState h;
    TRY(read_state(c, &h));
    if (h.k) CU(cudaMemcpy(out, c->piv, sizeof(long long) * h.k, cudaMemcpyDeviceToHost));
    return RBG_OK;
}

rbg_status rbg_get_errors(rbg_ctx *c, double *out) {
    TRY(check_ctx(c));
    if (!out) return fail(RBG_EINVAL, "null output");
    DevState h;
    TRY(read_state(c, &h));
    // err_k exists once the decision kernel ran: not after PEER_TIMEOUT (the wait stopped first)
    const long long n = (h.stop && h.stop != kStopPeer) ? h.k + 1 : h.k;
    if (n) CU(cudaMemcpy(out, c->errors, sizeof(double) * n, cudaMemcpyDeviceToHost));
    return RBG_OK;
}

rbg_status rbg_get_nu(rbg_ctx *c, int32_t *out) {
    TRY(check_ctx(c));
    if (!out) return fail(RBG_EINVAL, "null output");
    DevState h;
    TRY(read_state(c, &h));
    if (h.k) CU(cudaMemcpy(out, c->nu, sizeof(int) * h.k, cudaMemcpyDeviceToHost));
    return RBG_OK;
}

rbg_status rbg_get_rdiag(rbg_ctx *c, double *out) {
    TRY(check_ctx(c));
    if (!out) return fail(RBG_EINVAL, "null output");
    DevState h;
    TRY(read_state(c, &h));
    if (h.k) CU(cudaMemcpy(out, c->rdiag, sizeof(double) * h.k, cudaMemcpyDeviceToHost));
    return RBG_OK;
}

rbg_status rbg_get_basis(rbg_ctx *c, void *out, int64_t ldq, int on_device) {
    TRY(check_ctx(c));
    if (!out || ldq < c->N) return fail(RBG_EINVAL, "null output or ldq < N");
    DevState h;
    TRY(read_state(c, &h));
    if (!h.k) return RBG_OK;
    const double2 *src = c->Q;
    double2 *tmp = nullptr;
    if (c->xmode) {  // Q = Q~ / W^{1/2}: the W-orthonormal basis of S
        CU(dmalloc(&tmp, (size_t)h.k * c->ldq_v * 16));
        cudaError_t e = launch_unscale_sqrtw(tmp, c->Q, h.k, c->ldq_v, c->w_true, c->cplx, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) {
            dfree(tmp);
            return fail(RBG_ECUDA, "basis unscale: %s", cudaGetErrorString(e));
        }
        src = tmp;
    }
    cudaError_t e = cudaMemcpy2D(out, (size_t)ldq * c->se, src, (size_t)c->ldq_v * 16, (size_t)c->N * c->se, h.k,
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
    dfree(tmp);
    if (e != cudaSuccess) return fail(RBG_ECUDA, "get_basis: %s", cudaGetErrorString(e));
    return RBG_OK;
}

rbg_status rbg_get_R(rbg_ctx *c, void *out, int64_t ldr, int on_device) {
    TRY(check_ctx(c));
    if (!out || ldr < c->M) return fail(RBG_EINVAL, "null output or ldr < M_loc");
    DevState h;
    TRY(read_state(c, &h));
    if (h.k)
        CU(cudaMemcpy2D(out, (size_t)ldr * c->se, c->R, (size_t)c->ldr * c->se, (size_t)c->M * c->se, h.k,
                        on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
    return RBG_OK;
}

rbg_status rbg_get_r2(rbg_ctx *c, double *out, int on_device) {
    TRY(check_ctx(c));
    if (!out) return fail(RBG_EINVAL, "null output");
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaMemcpy(out, c->r2, sizeof(double) * c->M, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
    return RBG_OK;
}

rbg_status rbg_get_timings(rbg_ctx *c, double *sweep_ms, double *xchg_ms, double *imgs_ms, int64_t n) {
    TRY(check_ctx(c));
    CU(cudaStreamSynchronize(c->stream));
    // sweep i uses q_i: the local step of iteration i+1; xchg/imgs i: iteration i
    for (int64_t i = 0; i < n; i++) {
        float ms;
        if (sweep_ms) {
            sweep_ms[i] = NAN;
            if ((size_t)(i + 1) < c->ev.size() && c->ev_iter[i + 1] == i + 1) {
                CU(cudaEventElapsedTime(&ms, c->ev[i + 1].e[0], c->ev[i + 1].e[1]));
                sweep_ms[i] = ms;
            }
        }
        if ((size_t)i < c->ev.size() && c->ev_iter[i] == i) {
            if (xchg_ms) {
                CU(cudaEventElapsedTime(&ms, c->ev[i].e[1], c->ev[i].e[2]));
                xchg_ms[i] = ms;
            }
            if (imgs_ms) {
                CU(cudaEventElapsedTime(&ms, c->ev[i].e[2], c->ev[i].e[3]));
                imgs_ms[i] = ms;
            }
        } else {
            if (xchg_ms) xchg_ms[i] = NAN;
            if (imgs_ms) imgs_ms[i] = NAN;
        }
    }
    return RBG_OK;
}

rbg_status rbg_get_stats(rbg_ctx *c, rbg_stats *o) {
    TRY(check_ctx(c));
    if (!o) return fail(RBG_EINVAL, "null output");
    DevState h;
    TRY(read_state(c, &h));
    std::memset(o, 0, sizeof *o);
    o->k = h.k;
    o->noop_iters = h.noop;
    // iterations with events, restricted to those that did work: 0..k
    const long long last = std::min<long long>(h.k, (long long)c->ev.size() - 1);
    float ms;
    bool first = true;
    cudaEvent_t e_first = nullptr, e_last = nullptr;
    for (long long t = 0; t <= last; t++) {
        if (c->ev_iter[t] != t) continue;
        const PhaseEvents &p = c->ev[t];
        if (t > 0 && c->ev_iter[t - 1] == t - 1) {
            CU(cudaEventElapsedTime(&ms, c->ev[t - 1].e[3], p.e[0]));
            o->t_gap_ms += ms;
        }
        CU(cudaEventElapsedTime(&ms, p.e[0], p.e[1]));
        if (t == 0) o->t_init_ms = ms;
        else {
            o->t_sweep_ms += ms;
            o->sweeps++;
        }
        CU(cudaEventElapsedTime(&ms, p.e[1], p.e[2]));
        o->t_xchg_ms += ms;
        CU(cudaEventElapsedTime(&ms, p.e[2], p.e[3]));
        o->t_imgs_ms += ms;
        if (first) {
            e_first = p.e[0];
            first = false;
        }
        e_last = p.e[3];
    }
    if (e_first && e_last) {
        CU(cudaEventElapsedTime(&ms, e_first, e_last));
        o->t_total_ms = ms;
    }
    return RBG_OK;
}

rbg_status rbg_iter_local(rbg_ctx *c) {
    TRY(check_ctx(c));
    if ((c->comm != RBG_COMM_EXTERNAL && c->comm != RBG_COMM_PEER) || c->local_pending)
        return fail(RBG_ESTATE, "iter_local out of order");
    if (c->comm == RBG_COMM_PEER && !c->peer_connected) return fail(RBG_ESTATE, "PEER context not connected");
    PhaseEvents *pe = nullptr;
    if (c->timing) {  // the same per-phase events as enqueue_iteration
        PhaseEvents p;
        for (int i = 0; i < 4; i++) CU(cudaEventCreate(&p.e[i]));
        c->ev.push_back(p);
        c->ev_iter.push_back(c->iters);
        pe = &c->ev.back();
        CU(cudaEventRecord(pe->e[0], c->stream));
    }
    TRY(enqueue_local(c));
    if (pe) CU(cudaEventRecord(pe->e[1], c->stream));
    c->local_pending = true;
    return RBG_OK;
}

rbg_status rbg_iter_finish(rbg_ctx *c) {
    TRY(check_ctx(c));
    if ((c->comm != RBG_COMM_EXTERNAL && c->comm != RBG_COMM_PEER) || !c->local_pending)
        return fail(RBG_ESTATE, "iter_finish out of order");
    const bool timed = c->timing && !c->ev.empty() && c->ev_iter.back() == c->iters;
    if (c->comm == RBG_COMM_PEER) TRY(enqueue_xchg(c));  // wait for the peers' records
    if (timed) CU(cudaEventRecord(c->ev.back().e[2], c->stream));
    TRY(enqueue_finish(c));
    if (timed) CU(cudaEventRecord(c->ev.back().e[3], c->stream));
    c->local_pending = false;
    c->iters++;
    return RBG_OK;
}

rbg_status rbg_xchg_buffers(rbg_ctx *c, void **send, void **recv, size_t *bytes) {
    TRY(check_ctx(c));
    if (send) *send = c->send;
    if (recv) *recv = c->recv;
    if (bytes) *bytes = c->slot;
    return RBG_OK;
}

rbg_status rbg_emulate_allgather(rbg_ctx **ctxs, int world) {
    if (!ctxs || world < 1) return fail(RBG_EINVAL, "bad context list");
    for (int p = 0; p < world; p++) {
        if (!ctxs[p] || ctxs[p]->world != world || ctxs[p]->rank != p || !ctxs[p]->send)
            return fail(RBG_EINVAL, "context %d is not rank %d of a %d-rank EXTERNAL group", p, p, world);
        CU(cudaSetDevice(ctxs[p]->device));
        CU(cudaStreamSynchronize(ctxs[p]->stream));
    }
    for (int p = 0; p < world; p++)
        for (int r = 0; r < world; r++)
            CU(cudaMemcpy(ctxs[p]->recv + (size_t)r * ctxs[p]->slot, ctxs[r]->send, ctxs[r]->slot,
                          cudaMemcpyDeviceToDevice));
    return RBG_OK;
}

rbg_status rbg_peer_export(rbg_ctx *c, uint8_t out[RBG_PEER_HANDLE_BYTES]) {
    TRY(check_ctx(c));
    if (!out) return fail(RBG_EINVAL, "null output");
    if (c->comm != RBG_COMM_PEER) return fail(RBG_ESTATE, "not a PEER context");
    cudaIpcMemHandle_t h[2];
    CU(cudaIpcGetMemHandle(&h[0], c->peer_in));
    CU(cudaIpcGetMemHandle(&h[1], c->send));
    static_assert(sizeof(cudaIpcMemHandle_t) * 2 == RBG_PEER_HANDLE_BYTES, "handle size");
    std::memcpy(out, h, sizeof h);
    return RBG_OK;
}

rbg_status rbg_peer_connect(rbg_ctx *c, const uint8_t *all) {
    TRY(check_ctx(c));
    if (!all) return fail(RBG_EINVAL, "null handle list");
    if (c->comm != RBG_COMM_PEER) return fail(RBG_ESTATE, "not a PEER context");
    if (c->peer_connected) return fail(RBG_ESTATE, "already connected");
    for (int q = 0; q < c->world; q++) {
        if (q == c->rank) continue;  // own buffers: direct pointers
        cudaIpcMemHandle_t h[2];
        std::memcpy(h, all + (size_t)q * RBG_PEER_HANDLE_BYTES, sizeof h);
        void *rec = nullptr, *snd = nullptr;
        CU(cudaIpcOpenMemHandle(&rec, h[0], cudaIpcMemLazyEnablePeerAccess));
        cudaError_t e = cudaIpcOpenMemHandle(&snd, h[1], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaIpcCloseMemHandle(rec);
            return fail(RBG_ECUDA, "cudaIpcOpenMemHandle (rank %d send slots): %s", q, cudaGetErrorString(e));
        }
        c->peer_rec[q] = static_cast<PeerRec *>(rec);
        c->peer_send[q] = static_cast<unsigned char *>(snd);
        c->peer_ipc[q] = true;
    }
    c->peer_connected = true;
    return RBG_OK;
}

rbg_status rbg_peer_connect_local(rbg_ctx **ctxs, int world) {
    if (!ctxs || world < 1 || world > kMaxPeers) return fail(RBG_EINVAL, "bad context list");
    for (int p = 0; p < world; p++)
        if (!ctxs[p] || ctxs[p]->comm != RBG_COMM_PEER || ctxs[p]->world != world || ctxs[p]->rank != p ||
            ctxs[p]->peer_connected && world > 1)
            return fail(RBG_EINVAL, "context %d is not an unconnected rank %d of a %d-rank PEER group", p, p, world);
    for (int p = 1; p < world; p++)  // one stream: rank p's wait never runs beside a sweep it waits for
        if (ctxs[p]->stream != ctxs[0]->stream || ctxs[p]->device != ctxs[0]->device)
            return fail(RBG_EINVAL, "local PEER contexts must share one device and one stream");
    for (int p = 0; p < world; p++) {
        for (int q = 0; q < world; q++) {
            ctxs[p]->peer_rec[q] = ctxs[q]->peer_in;
            ctxs[p]->peer_send[q] = ctxs[q]->send;
        }
        ctxs[p]->peer_connected = true;
    }
    return RBG_OK;
}

void rbg_destroy(rbg_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    free_ctx(c);
}

}  // extern "C"
