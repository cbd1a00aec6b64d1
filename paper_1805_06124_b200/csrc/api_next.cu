// api_next.cu -- the C-ABI entry points of the NEXT rows of SURVEY §8(f) on a context built
// by api.cu: out-of-sample validation and enrichment, Algorithm 4
// reconstruction through the Gram matrix, EIM nodes,
// and their column-sharded forms (R33, R34).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "ctx.h"

using namespace rbg;
using namespace rbg_api;

extern "C" {

rbg_status rbg_validate(rbg_ctx *c, const void *V, int64_t M_v, int64_t ldv, rbg_mem V_mem, double *err, void *C,
                        int64_t ldc, int out_on_device) {
    TRY(check_ctx(c));
    if (c->xmode) return fail(RBG_ESTATE, "not available with explicit residuals");
    if (C && ldc < M_v) return fail(RBG_EINVAL, "ldc < M_v");
    if (c->local_pending) return fail(RBG_ESTATE, "validate inside an EXTERNAL iteration");
    DevState h;
    TRY(read_state(c, &h));
    double2 *Vd = nullptr;
    bool v_owned = false;
    TRY(upload_block(c, V, M_v, ldv, V_mem, &Vd, &v_owned));
    const long long k = h.k;
    double *Rv = nullptr, *e2 = nullptr, *ed = nullptr;
    cudaError_t e = salloc(&c->scratch, kScValR, &Rv, (size_t)std::max<long long>(k, 1) * M_v * c->se);
    if (e == cudaSuccess) e = salloc(&c->scratch, kScValE2, &e2, sizeof(double) * M_v);
    if (e == cudaSuccess) e = salloc(&c->scratch, kScValE, &ed, sizeof(double) * M_v);
    rbg_status st = e == cudaSuccess ? coeff_passes(c, Vd, M_v, Rv, M_v, e2, k)
                                     : fail(RBG_ENOMEM, "validation buffers: %s", cudaGetErrorString(e));
    const cudaMemcpyKind kind = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (st == RBG_OK && err) {
        e = launch_sqrt_clamp(e2, ed, M_v, c->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(err, ed, sizeof(double) * M_v, kind, c->stream);
        if (e != cudaSuccess) st = fail(RBG_ECUDA, "validation errors: %s", cudaGetErrorString(e));
    }
    if (st == RBG_OK && C && k) {
        e = cudaMemcpy2DAsync(C, (size_t)ldc * c->se, Rv, (size_t)M_v * c->se, (size_t)M_v * c->se, k, kind, c->stream);
        if (e != cudaSuccess) st = fail(RBG_ECUDA, "validation coefficients: %s", cudaGetErrorString(e));
    }
    cudaStreamSynchronize(c->stream);
    if (v_owned) dfree(Vd);
    sfree(&c->scratch, Rv);
    sfree(&c->scratch, e2);
    sfree(&c->scratch, ed);
    return st;
}

rbg_status rbg_add_columns_ex(rbg_ctx *c, const void *F, int64_t M_f, int64_t ldf, rbg_mem F_mem, int64_t first_gid,
                              int64_t M_global_new) {
    TRY(check_ctx(c));
    if (c->xmode) return fail(RBG_ESTATE, "not available with explicit residuals");
    if (c->local_pending) return fail(RBG_ESTATE, "add_columns inside an EXTERNAL/PEER iteration");
    const bool sharded = c->comm != RBG_COMM_NONE;
    if (first_gid < 0) first_gid = c->M_global;
    if (M_global_new <= 0) M_global_new = c->M_global + M_f;
    if (M_f < 0 || (!sharded && M_f < 1)) return fail(RBG_EINVAL, "M_f < 1");
    if (first_gid < c->M_global || first_gid + M_f > M_global_new)
        return fail(RBG_EINVAL, "appended ids [%lld, %lld) must lie in [M_global=%lld, M_global_new=%lld)",
                    (long long)first_gid, (long long)(first_gid + M_f), c->M_global, (long long)M_global_new);
    if (!sharded && (first_gid != c->M_global || M_global_new != c->M_global + M_f))
        return fail(RBG_EINVAL, "a single-GPU context appends at the end (ids M_global..M_global+M_f)");
    DevState h;
    TRY(read_state(c, &h));
    TRY(need_settled(c, h, "add_columns"));
    const long long M0 = c->M, M1 = c->M + M_f;
    const long long ext0 = c->M - c->M0;  // columns already in the appended segment
    double2 *Fd = nullptr;
    bool f_owned = false;
    if (M_f > 0) TRY(upload_block(c, F, M_f, ldf, F_mem, &Fd, &f_owned));
    // The caller's columns stay where they are (a borrowed S is never copied): the appended
    // columns go to a library-owned second segment that the sweep streams after the first
    // (scol in kernels.h).  Only that segment, R (k_max x M row-major: rows get longer) and the
    // per-column vectors are reallocated.
    const size_t pitch = (size_t)c->nvec * 16;
    double2 *S1n = c->S1;
    double *R1 = c->R, *r21 = c->r2;
    long long *gid1 = c->gid;
    // R keeps a row stride with room for appended columns: an append within it writes the new
    // columns' rows in place; beyond it R is reallocated with 1/8 (>= 4,096 columns) of slack
    // and rows 0..k-1 copied (rows >= k are written by later sweeps before anything reads them)
    const bool grow_r = M1 > c->ldr;
    const long long ldr1 = grow_r ? M1 + std::max<long long>(M1 / 8, 4096) : c->ldr;
    cudaError_t e = cudaSuccess;
    if (M_f > 0) {
        S1n = nullptr;
        r21 = nullptr;
        e = dmalloc(&S1n, pitch * (ext0 + M_f));
        if (e == cudaSuccess && ext0) e = cudaMemcpyAsync(S1n, c->S1, pitch * ext0, cudaMemcpyDeviceToDevice, c->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(S1n + ext0 * c->nvec, Fd, pitch * M_f, cudaMemcpyDeviceToDevice, c->stream);
        if (grow_r) {
            R1 = nullptr;
            if (e == cudaSuccess) e = dmalloc(&R1, (size_t)c->k_max * ldr1 * c->se);
            if (e == cudaSuccess && h.k)
                e = cudaMemcpy2DAsync(R1, (size_t)ldr1 * c->se, c->R, (size_t)c->ldr * c->se, (size_t)M0 * c->se, h.k,
                                      cudaMemcpyDeviceToDevice, c->stream);
        }
        if (e == cudaSuccess) e = dmalloc(&r21, sizeof(double) * M1);
        if (e == cudaSuccess) e = cudaMemcpyAsync(r21, c->r2, sizeof(double) * M0, cudaMemcpyDeviceToDevice, c->stream);
        if (e == cudaSuccess && sharded) {
            // global indices: the rank's original block, earlier appends, then these columns
            std::vector<long long> g((size_t)M1);
            if (c->gid) e = cudaMemcpy(g.data(), c->gid, sizeof(long long) * M0, cudaMemcpyDeviceToHost);
            else
                for (long long j = 0; j < M0; j++) g[(size_t)j] = c->col_offset + j;
            for (long long j = 0; j < M_f; j++) g[(size_t)(M0 + j)] = first_gid + j;
            gid1 = nullptr;
            if (e == cudaSuccess) e = dmalloc(&gid1, sizeof(long long) * M1);
            if (e == cudaSuccess) e = cudaMemcpy(gid1, g.data(), sizeof(long long) * M1, cudaMemcpyHostToDevice);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    }
    if (f_owned) dfree(Fd);
    auto drop_new = [&]() {
        if (M_f > 0) {
            dfree(S1n);
            if (R1 != c->R) dfree(R1);
            dfree(r21);
            if (gid1 != c->gid) dfree(gid1);
        }
    };
    if (e != cudaSuccess) {
        drop_new();
        return fail(e == cudaErrorMemoryAllocation ? RBG_ENOMEM : RBG_ECUDA, "add_columns: %s", cudaGetErrorString(e));
    }
    if (c->started && M_f > 0) {
        // the new columns get R rows 0..k-1 and the recurrence residual, then the pivot
        // search restarts over all columns and the next iteration begins at the decision
        rbg_status st = coeff_passes(c, S1n + ext0 * c->nvec, M_f, R1 + (size_t)M0 * (c->se / 8), ldr1, r21 + M0, h.k);
        if (st != RBG_OK) {
            drop_new();
            return st;
        }
    }
    if (M_f > 0) {
        dfree(c->S1);
        if (R1 != c->R) dfree(c->R);
        dfree(c->r2);
        if (gid1 != c->gid) dfree(c->gid);
        c->S1 = S1n;
        c->R = R1;
        c->ldr = ldr1;
        c->r2 = r21;
        c->gid = gid1;
        c->M = M1;
    }
    c->M_global = M_global_new;
    for (auto &p : c->ev)
        for (int i = 0; i < 4; i++) cudaEventDestroy(p.e[i]);
    c->ev.clear();
    c->ev_iter.clear();
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    if (c->while_exec) {  // its kernels hold the old column pointers and record epoch
        cudaGraphExecDestroy(c->while_exec);
        c->while_exec = nullptr;
    }
    if (c->started) {
        CU(cudaMemsetAsync(&c->st->stop, 0, sizeof(int), c->stream));
        if (sharded) {
            // new record tags (the stopped decision's records have the old epoch), the local
            // candidate packed and, on PEER, published; the next iteration exchanges and decides
            c->epoch++;
            CU(launch_restart(sweep_args(c), c->cplx, c->stream));
        } else {
            CU(launch_maxloc(c->r2, M1, 0, c->st, c->stream));
        }
        c->resume_pending = true;
        c->stopped = false;
        c->iters = h.k;
    }
    CU(cudaStreamSynchronize(c->stream));
    return RBG_OK;
}

rbg_status rbg_restore(rbg_ctx *c, int64_t k, const int64_t *pivots, const double *errors, const int32_t *nu,
                       const double *rdiag, const void *Q, int64_t ldq, const void *R, int64_t ldr, const double *r2,
                       rbg_mem mem) {
    TRY(check_ctx(c));
    if (c->xmode) return fail(RBG_ESTATE, "not available with explicit residuals");
    if (c->comm != RBG_COMM_NONE) return fail(RBG_ESTATE, "restore needs a single-GPU context");
    if (c->started || c->iters) return fail(RBG_ESTATE, "restore into a fresh context only");
    if (k < 0 || k >= c->k_max || k > c->M)
        return fail(RBG_EINVAL, "k=%lld outside [0, k_max=%lld) or above M", (long long)k, c->k_max);
    if (k == 0) return RBG_OK;  // nothing to restore: the greedy starts with sweep 0
    if (!pivots || !errors || !nu || !rdiag || !Q || !R || !r2) return fail(RBG_EINVAL, "null state array");
    if (ldq < c->N || ldr < c->M) return fail(RBG_EINVAL, "ldq < N or ldr < M");
    std::vector<long long> hp((size_t)k);
    const cudaMemcpyKind kind = mem == RBG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CU(cudaMemcpy(hp.data(), pivots, sizeof(long long) * k,
                  mem == RBG_MEM_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
    for (long long i = 0; i < k; i++)
        if (hp[(size_t)i] < 0 || hp[(size_t)i] >= c->M) return fail(RBG_EINVAL, "pivot %lld out of range", hp[(size_t)i]);
    const size_t col = (size_t)c->N * c->se, pitch = (size_t)c->nvec * 16;
    cudaError_t e = cudaSuccess;
    if (pitch != col) e = cudaMemsetAsync(c->Q, 0, pitch * k, c->stream);  // real, odd N: padding row
    if (e == cudaSuccess) e = cudaMemcpy2DAsync(c->Q, pitch, Q, (size_t)ldq * c->se, col, k, kind, c->stream);
    if (e == cudaSuccess) e = launch_weight_basis(c->WQ, c->Q, k, c->ldq_v, c->nvec, c->w, c->cplx, c->stream);
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(c->R, (size_t)c->ldr * c->se, R, (size_t)ldr * c->se, (size_t)c->M * c->se, k, kind, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->r2, r2, sizeof(double) * c->M, kind, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->piv, pivots, sizeof(long long) * k, kind, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->errors, errors, sizeof(double) * k, kind, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->nu, nu, sizeof(int) * k, kind, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->rdiag, rdiag, sizeof(double) * k, kind, c->stream);
    DevState h{};
    h.k = k;
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->st, &h, sizeof h, cudaMemcpyHostToDevice, c->stream);
    // the pivot search over the restored residuals; the next iteration begins at the decision
    if (e == cudaSuccess) e = launch_maxloc(c->r2, c->M, 0, c->st, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(RBG_ECUDA, "restore: %s", cudaGetErrorString(e));
    c->started = true;
    c->resume_pending = true;
    c->stopped = false;
    c->iters = k;
    return RBG_OK;
}

rbg_status rbg_add_columns(rbg_ctx *c, const void *F, int64_t M_f, int64_t ldf, rbg_mem F_mem) {
    TRY(check_ctx(c));
    if (c->world != 1 || c->comm != RBG_COMM_NONE)
        return fail(RBG_ESTATE, "sharded contexts use rbg_add_columns_ex (global ids of the appended columns)");
    return rbg_add_columns_ex(c, F, M_f, ldf, F_mem, -1, 0);
}

namespace {
// G = G0 + R(0:k, :) R(0:k, :)^H into a zero-padded kp x kp column-major device buffer
// (G0: same layout, or NULL for zero; the running sum of the previous ranks when folding).
rbg_status gram_device(rbg_ctx *c, int k, int kp, const double2 *G0, double2 *G) {
    const long long nchunks = std::max<long long>(1, (c->M + kGramChunk - 1) / kGramChunk);
    const int nt = (k + gram_tile() - 1) / gram_tile();
    // work items {tile a, tile b, chunk}, heaviest tiles first (FMA count of the tile's 16-row
    // groups below k, the diagonal tiles' lower groups skipped), chunk-major within a class
    const int gs = gram_tile() / 16;
    auto groups = [&](int t) { return std::min(gs, (k - t * gram_tile() + 15) / 16); };
    std::vector<std::pair<int, int2>> tiles;  // (cost, tile)
    for (int a = 0; a < nt; a++)
        for (int b = a; b < nt; b++) {
            const int nu = groups(a), nv = groups(b);
            int cost = 0;
            for (int u = 0; u < nu; u++)
                for (int v = 0; v < nv; v++) cost += (a != b || v >= u) ? 1 : 0;
            tiles.push_back({cost, make_int2(a, b)});
        }
    std::stable_sort(tiles.begin(), tiles.end(), [](const auto &x, const auto &y) { return x.first > y.first; });
    std::vector<int4> items;
    for (size_t i = 0; i < tiles.size();) {
        size_t j = i;
        while (j < tiles.size() && tiles[j].first == tiles[i].first) j++;
        for (long long ch = 0; ch < nchunks; ch++)
            for (size_t t = i; t < j; t++) items.push_back(make_int4(tiles[t].second.x, tiles[t].second.y, (int)ch, 0));
        i = j;
    }
    int4 *items_d = nullptr;
    double2 *P = nullptr;
    cudaError_t e = salloc(&c->scratch, kScGramItems, &items_d, sizeof(int4) * items.size());
    if (e == cudaSuccess) e = salloc(&c->scratch, kScGramP, &P, sizeof(double2) * (size_t)nchunks * k * k);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(items_d, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess)
        e = launch_gram(c->R, c->ldr, k, c->M, c->cplx, P, kGramChunk, items_d, (int)items.size(), c->stream);
    if (e == cudaSuccess) e = launch_gram_reduce(P, nchunks, k, kp, G0, G, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    sfree(&c->scratch, items_d);
    sfree(&c->scratch, P);
    if (e != cudaSuccess) return fail(RBG_ECUDA, "gram: %s", cudaGetErrorString(e));
    return RBG_OK;
}
}  // namespace

rbg_status rbg_gram(rbg_ctx *c, void *G, int64_t ldg, int on_device) {
    TRY(check_ctx(c));
    if (c->xmode) return fail(RBG_ESTATE, "not available with explicit residuals");
    if (c->world != 1) return fail(RBG_ESTATE, "gram needs a single-GPU context");
    DevState h;
    TRY(read_state(c, &h));
    TRY(need_settled(c, h, "gram"));
    const int k = (int)h.k;
    if (!G || ldg < k) return fail(RBG_EINVAL, "null output or ldg < k");
    if (k == 0) return RBG_OK;
    const int kp = k + (k & 1);
    double2 *Gd = nullptr;
    CU(salloc(&c->scratch, kScRecG, &Gd, sizeof(double2) * (size_t)kp * kp));
    rbg_status st = gram_device(c, k, kp, nullptr, Gd);
    if (st == RBG_OK) {
        cudaError_t e = cudaMemcpy2D(G, (size_t)ldg * 16, Gd, (size_t)kp * 16, (size_t)k * 16, k,
                                     on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) st = fail(RBG_ECUDA, "gram copy: %s", cudaGetErrorString(e));
    }
    sfree(&c->scratch, Gd);
    return st;
}

rbg_status rbg_gram_fold(rbg_ctx *c, void *G, int64_t ldg, int on_device) {
    TRY(check_ctx(c));
    if (c->xmode) return fail(RBG_ESTATE, "not available with explicit residuals");
    DevState h;
    TRY(read_state(c, &h));
    TRY(need_settled(c, h, "gram_fold"));
    const int k = (int)h.k;
    if (!G || ldg < k) return fail(RBG_EINVAL, "null G or ldg < k");
    if (k == 0) return RBG_OK;
    const int kp = k + (k & 1);
    const cudaMemcpyKind in = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const cudaMemcpyKind out = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    double2 *G0 = nullptr, *G1 = nullptr;
    cudaError_t e = salloc(&c->scratch, kScRecG, &G0, sizeof(double2) * (size_t)kp * kp);
    if (e == cudaSuccess) e = salloc(&c->scratch, kScRecV, &G1, sizeof(double2) * (size_t)kp * kp);
    if (e == cudaSuccess) e = cudaMemsetAsync(G0, 0, sizeof(double2) * (size_t)kp * kp, c->stream);
    if (e == cudaSuccess) e = cudaMemcpy2DAsync(G0, (size_t)kp * 16, G, (size_t)ldg * 16, (size_t)k * 16, k, in, c->stream);
    rbg_status st = e == cudaSuccess ? gram_device(c, k, kp, G0, G1) : fail(RBG_ECUDA, "gram_fold: %s", cudaGetErrorString(e));
    if (st == RBG_OK) {
        e = cudaMemcpy2D(G, (size_t)ldg * 16, G1, (size_t)kp * 16, (size_t)k * 16, k, out);
        if (e != cudaSuccess) st = fail(RBG_ECUDA, "gram_fold copy: %s", cudaGetErrorString(e));
    }
    sfree(&c->scratch, G0);
    sfree(&c->scratch, G1);
    return st;
}

namespace {
// Algorithm 4 after the Gram matrix: Gin = NULL -> this context's R R^H; else the given k x k
// Hermitian matrix (leading dimension ldg, host or device), e.g. a sharded fold.
rbg_status reconstruct_impl(rbg_ctx *c, const void *Gin, int64_t ldg, int g_on_device, double tau2, int64_t kr_max,
                            int64_t *kr_out, double *sigma, void *X, int64_t ldx, int on_device) {
    TRY(check_ctx(c));
    if (c->xmode) return fail(RBG_ESTATE, "not available with explicit residuals");
    if (!Gin && c->world != 1) return fail(RBG_ESTATE, "reconstruct needs a single-GPU context (sharded: rbg_gram_fold + rbg_reconstruct_gram)");
    if (!(tau2 >= 0.0) || kr_max < 0) return fail(RBG_EINVAL, "tau2 < 0 or kr_max < 0");
    if (X && ldx < c->N) return fail(RBG_EINVAL, "ldx < N");
    DevState h;
    TRY(read_state(c, &h));
    if (!Gin) TRY(need_settled(c, h, "reconstruct"));
    const int k = (int)h.k;
    if (kr_out) *kr_out = 0;
    if (k == 0) return RBG_OK;
    // block Jacobi (default) pads to a multiple of 32; RBG_JACOBI=elem selects the element
    // cyclic Jacobi (pads to even)
    const char *jenv = getenv("RBG_JACOBI");
    const bool block = !(jenv && std::strcmp(jenv, "elem") == 0);
    const int kp = block ? jacobi_pad(k) : k + (k & 1);
    double2 *G = nullptr, *V = nullptr, *Xd = nullptr;
    Rot *rots = nullptr;
    unsigned long long *flags = nullptr;
    int *sweeps = nullptr, *order = nullptr, *krd = nullptr;
    double *sig = nullptr;
    ScratchPool *sp = &c->scratch;
    cudaError_t e = salloc(sp, kScRecG, &G, sizeof(double2) * (size_t)kp * kp);
    if (e == cudaSuccess) e = salloc(sp, kScRecV, &V, sizeof(double2) * (size_t)kp * kp);
    if (e == cudaSuccess) e = salloc(sp, kScRecRots, &rots, block ? bjacobi_scratch_bytes(kp) : jacobi_scratch_bytes(kp));
    if (e == cudaSuccess) e = salloc(sp, kScRecFlags, &flags, 3 * sizeof(unsigned long long));  // ratios + barrier
    if (e == cudaSuccess) e = salloc(sp, kScRecSweeps, &sweeps, sizeof(int));
    if (e == cudaSuccess) e = salloc(sp, kScRecOrder, &order, sizeof(int) * kp);
    if (e == cudaSuccess) e = salloc(sp, kScRecKr, &krd, sizeof(int));
    if (e == cudaSuccess) e = salloc(sp, kScRecSig, &sig, sizeof(double) * kp);
    rbg_status st = e == cudaSuccess ? RBG_OK : fail(RBG_ENOMEM, "reconstruct buffers: %s", cudaGetErrorString(e));
    if (st == RBG_OK && !Gin) st = gram_device(c, k, kp, nullptr, G);
    if (st == RBG_OK && Gin) {
        if (ldg < k) st = fail(RBG_EINVAL, "ldg < k");
        if (st == RBG_OK) e = cudaMemsetAsync(G, 0, sizeof(double2) * (size_t)kp * kp, c->stream);
        if (st == RBG_OK && e == cudaSuccess)
            e = cudaMemcpy2DAsync(G, (size_t)kp * 16, Gin, (size_t)ldg * 16, (size_t)k * 16, k,
                                  g_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream);
        if (st == RBG_OK && e != cudaSuccess) st = fail(RBG_ECUDA, "reconstruct upload: %s", cudaGetErrorString(e));
    }
    if (st == RBG_OK) {
        std::vector<double2> I((size_t)kp * kp, make_double2(0.0, 0.0));
        for (int i = 0; i < kp; i++) I[(size_t)i * kp + i] = make_double2(1.0, 0.0);
        e = cudaMemcpyAsync(V, I.data(), sizeof(double2) * I.size(), cudaMemcpyHostToDevice, c->stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(flags, 0, 3 * sizeof(unsigned long long), c->stream);
        if (e == cudaSuccess) {
            unsigned long long *trace = nullptr;  // RBG_DEBUG_JACOBI: phase timestamps of 8 rounds
            if (block && getenv("RBG_DEBUG_JACOBI") && dmalloc(&trace, 128 * sizeof(unsigned long long)) != cudaSuccess)
                trace = nullptr;
            if (trace) cudaMemsetAsync(trace, 0, 128 * sizeof(unsigned long long), c->stream);
            if (e == cudaSuccess)
                e = block ? launch_bjacobi(G, V, kp, reinterpret_cast<double2 *>(rots), flags, sweeps, c->num_sms,
                                           c->stream, trace)
                          : launch_jacobi(G, V, kp, rots, flags, sweeps, c->num_sms, c->stream);
            if (trace) {
                unsigned long long tt[128];
                cudaMemcpyAsync(tt, trace, sizeof tt, cudaMemcpyDeviceToHost, c->stream);
                cudaStreamSynchronize(c->stream);
                for (int r = 1; r < 8; r++)
                    fprintf(stderr, "rbg: bjacobi round %d: P1+bar %.1f us, P2+bar %.1f us, P3+bar %.1f us\n", r,
                            (tt[r * 4 + 1] - tt[r * 4]) * 1e-3, (tt[r * 4 + 2] - tt[r * 4 + 1]) * 1e-3,
                            (tt[r * 4 + 3] - tt[r * 4 + 2]) * 1e-3);
                for (int r = 1; r < 8; r++)
                    fprintf(stderr, "rbg: bjacobi round %d P1 (CTA 0): load+measure %.2f us, %d local rounds %.2f us, U store %.2f us\n",
                            r, (tt[64 + r * 4] - tt[r * 4]) * 1e-3, 31, (tt[64 + r * 4 + 1] - tt[64 + r * 4]) * 1e-3,
                            (tt[64 + r * 4 + 2] - tt[64 + r * 4 + 1]) * 1e-3);
                fprintf(stderr, "rbg: bjacobi max off-diagonal ratio per sweep:");
                for (int sw = 0; sw < 32 && tt[32 + sw]; sw++) {
                    double v;
                    std::memcpy(&v, &tt[32 + sw], sizeof v);
                    fprintf(stderr, " %.2e", v);
                }
                fprintf(stderr, "\n");
                dfree(trace);
            }
        }
        if (e == cudaSuccess)
            e = launch_eig_sort(G, k, kp, tau2, (int)std::min<int64_t>(kr_max ? kr_max : k, k), order, sig, krd,
                                c->stream);
        int kr = 0;
        if (e == cudaSuccess && getenv("RBG_DEBUG_JACOBI")) {
            int sw = 0;
            cudaMemcpyAsync(&sw, sweeps, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
            cudaStreamSynchronize(c->stream);
            fprintf(stderr, "rbg: jacobi (%s) k=%d kp=%d sweeps=%d\n", block ? "block" : "elem", k, kp, sw);
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(&kr, krd, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e == cudaSuccess && sigma) e = cudaMemcpy(sigma, sig, sizeof(double) * k, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && X && kr > 0) {
            e = salloc(sp, kScRecX, &Xd, (size_t)kr * c->nvec * 16);
            if (e == cudaSuccess)
                e = launch_recon_x(c->Q, c->ldq_v, c->nvec, k, V, kp, order, kr, Xd, c->nvec, c->cplx, c->stream);
            if (e == cudaSuccess)
                e = cudaMemcpy2DAsync(X, (size_t)ldx * c->se, Xd, (size_t)c->nvec * 16, (size_t)c->N * c->se, kr,
                                      on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        }
        if (e != cudaSuccess) st = fail(RBG_ECUDA, "reconstruct: %s", cudaGetErrorString(e));
        else if (kr_out) *kr_out = kr;
    }
    for (void *q : {(void *)G, (void *)V, (void *)Xd, (void *)rots, (void *)flags, (void *)sweeps, (void *)order,
                    (void *)krd, (void *)sig})
        sfree(sp, q);   // no-ops for what the context's pool keeps
    return st;
}

}  // namespace

rbg_status rbg_reconstruct(rbg_ctx *c, double tau2, int64_t kr_max, int64_t *kr_out, double *sigma, void *X,
                           int64_t ldx, int on_device) {
    return reconstruct_impl(c, nullptr, 0, 0, tau2, kr_max, kr_out, sigma, X, ldx, on_device);
}

rbg_status rbg_reconstruct_gram(rbg_ctx *c, const void *G, int64_t ldg, int g_on_device, double tau2, int64_t kr_max,
                                int64_t *kr_out, double *sigma, void *X, int64_t ldx, int on_device) {
    if (!G) return fail(RBG_EINVAL, "null G");
    return reconstruct_impl(c, G, ldg, g_on_device, tau2, kr_max, kr_out, sigma, X, ldx, on_device);
}

rbg_status rbg_eim(rbg_ctx *c, int64_t *nodes, void *B, int64_t ldb, int on_device) {
    TRY(check_ctx(c));
    if (c->xmode) return fail(RBG_ESTATE, "not available with explicit residuals");
    DevState h;
    TRY(read_state(c, &h));
    const int k = (int)h.k;
    if (k > 1024) return fail(RBG_EINVAL, "EIM supports k <= 1024 (k = %d)", k);
    if (B && ldb < k) return fail(RBG_EINVAL, "ldb < k");
    if (k == 0) return RBG_OK;
    long long *nd = nullptr;
    double2 *Bd = nullptr;
    int *status = nullptr, hs = 0;
    cudaError_t e = salloc(&c->scratch, kScEimNodes, &nd, sizeof(long long) * k);
    if (e == cudaSuccess) e = salloc(&c->scratch, kScEimB, &Bd, sizeof(double2) * (size_t)k * k);
    if (e == cudaSuccess) e = salloc(&c->scratch, kScEimStatus, &status, sizeof(int));
    if (e == cudaSuccess) e = run_eim(c->Q, c->ldq_v, c->N, c->cplx, k, nd, Bd, status, c->stream, &c->scratch);
    if (e == cudaSuccess) e = cudaMemcpy(&hs, status, sizeof(int), cudaMemcpyDeviceToHost);
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (e == cudaSuccess && nodes) e = cudaMemcpy(nodes, nd, sizeof(long long) * k, kind);
    if (e == cudaSuccess && B) e = cudaMemcpy2D(B, (size_t)ldb * 16, Bd, (size_t)k * 16, (size_t)k * 16, k, kind);
    sfree(&c->scratch, nd);
    sfree(&c->scratch, Bd);
    sfree(&c->scratch, status);
    if (e != cudaSuccess) return fail(RBG_ECUDA, "eim: %s", cudaGetErrorString(e));
    if (hs) return fail(RBG_ESTATE, "EIM residual vanished: the basis is numerically degenerate");
    return RBG_OK;
}

}  // extern "C"
