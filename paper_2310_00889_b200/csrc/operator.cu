// operator.cu -- the full operator apply slb_matvec (single GPU or one rank of many) and the
// NCCL communicator.
//
// Per apply on rank r:
//   [mobility] per-body projector reductions -> sigma' = sigma - L sigma, L sigma   (Eq. L)
//   upsample local panels, epilogue packs far-field source records into the GLOBAL dyn array
//   NCCL all-gather (in place) of the fine records + the coarse sigma'          (only exchange step)
//   far field: local targets x all M fine sources -> per-chunk partials        (Eq. e:nystrom-no-correction)
//   finalize: partials + folded near blocks E sigma' + c_I sigma' [+ L sigma]  (Eq. e:nystrom-correction,
//                                                                              P:L1750/1868/2009)
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy torch already loaded is reused).
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>
#include "operator_impl.cuh"

using namespace slb;

// In-place all-gather of per-panel data: rank r owns elements [E(ranges[r]), E(ranges[r+1])) with
// E(p) = p * per_panel (uniform) or off[p] * unit (ragged panels, off = node offsets).
// Runs for EVERY communicator, a one-rank one included (then NCCL's gather is an identity, but the
// offsets, counts and calls are the multi-rank ones).  SLB_FORCE_GROUPED_GATHER=1 (tests) takes the
// unequal-shard path (grouped in-place broadcasts) even when the shards are equal.
static bool force_grouped_gather() {
    static const bool v = [] { const char* e = getenv("SLB_FORCE_GROUPED_GATHER"); return e && e[0] == '1'; }();
    return v;
}

static slb_status allgather(slb_operator* op, double* buf, int64_t per_panel, cudaStream_t s,
                            const std::vector<int64_t>* off = nullptr, int64_t unit = 1) {
    slb_comm* c = op->comm;
    if (!c) return SLB_OK;
    NcclApi& A = nccl();
    auto E = [&](int64_t p) { return off ? (*off)[p] * unit : p * per_panel; };
    bool equal = !force_grouped_gather();
    for (int r = 1; r < c->nranks; ++r)
        if (E(op->ranges[r + 1]) - E(op->ranges[r]) != E(op->ranges[1]) - E(op->ranges[0])) equal = false;
    if (equal) {
        size_t cnt = (size_t)(E(op->ranges[1]) - E(op->ranges[0]));
        SLB_NCCL(A.AllGather(buf + E(op->ranges[c->rank]), buf, cnt, ncclDouble, c->comm, s));
        c->n_allgather++;
    } else {
        SLB_NCCL(A.GroupStart());
        for (int r = 0; r < c->nranks; ++r) {
            size_t cnt = (size_t)(E(op->ranges[r + 1]) - E(op->ranges[r]));
            if (cnt == 0) continue;
            double* p = buf + E(op->ranges[r]);
            SLB_NCCL(A.Broadcast(p, p, cnt, ncclDouble, r, c->comm, s));
            c->n_broadcast++;
        }
        SLB_NCCL(A.GroupEnd());
    }
    return SLB_OK;
}

static void free_op(slb_operator* op) {
    if (!op) return;
    if (op->nvls_on) nvls_free(&op->nvls); else cudaFree(op->dyn);
    cudaFree(op->barrier_d);
    cudaFree(op->geo); cudaFree(op->sc); cudaFree(op->coarse);
    cudaFree(op->partials); cudaFree(op->Lsig); cudaFree(op->nb0); cudaFree(op->bodyc);
    cudaFree(op->coef); cudaFree(op->sig_dev); cudaFree(op->u_dev); cudaFree(op->rec);
    cudaFree(op->cn0_d); cudaFree(op->fn0_d); cudaFree(op->lc0_d); cudaFree(op->lf0_d); cudaFree(op->boff_d);
    cudaFree(op->pbucket_d); cudaFree(op->bmeta_d);
    for (auto& b : op->buckets) { cudaFree(b.plist_d); cudaFree(b.ip_buf); }
    cudaFree(op->ip_buf);
    for (auto& g : op->apply_graphs) cudaGraphExecDestroy(g.exec);
    if (op->cap_stream) cudaStreamDestroy(op->cap_stream);
    for (auto& e : op->ev) if (e) cudaEventDestroy(e);
    if (op->graph) cudaGraphExecDestroy(op->graph);
    for (auto& w : op->ws) if (w) cudaStreamDestroy(w);
    for (auto& e : op->join) if (e) cudaEventDestroy(e);
    if (op->fork) cudaEventDestroy(op->fork);
    delete op;
}

extern "C" {

slb_status slb_comm_unique_id(unsigned char id[128]) {
    SLB_REQUIRE(id, SLB_ERR_INVALID_ARG, "null id");
    NcclApi& A = nccl();
    SLB_REQUIRE(A.ok, SLB_ERR_NCCL, "libnccl.so.2 could not be loaded");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    SLB_NCCL(A.GetUniqueId(&u));
    std::memcpy(id, &u, 128);
    return SLB_OK;
}

slb_status slb_comm_create(const unsigned char id[128], int nranks, int rank, slb_comm** out) {
    SLB_REQUIRE(id && out && nranks >= 1 && rank >= 0 && rank < nranks, SLB_ERR_INVALID_ARG, "bad args");
    NcclApi& A = nccl();
    SLB_REQUIRE(A.ok, SLB_ERR_NCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    slb_comm* c = new slb_comm;
    c->nranks = nranks;
    c->rank = rank;
    ncclResult_t r = A.CommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        set_error(std::string("ncclCommInitRank: ") + A.GetErrorString(r));
        delete c;
        return SLB_ERR_NCCL;
    }
    *out = c;
    return SLB_OK;
}

slb_status slb_comm_collective_counts(const slb_comm* c, long long out[3]) {
    SLB_REQUIRE(c && out, SLB_ERR_INVALID_ARG, "null argument");
    out[0] = c->n_allgather.load();
    out[1] = c->n_broadcast.load();
    out[2] = c->n_allreduce.load();
    return SLB_OK;
}

slb_status slb_comm_destroy(slb_comm* c) {
    if (!c) return SLB_OK;
    if (c->comm) nccl().CommDestroy(c->comm);
    delete c;
    return SLB_OK;
}

slb_status slb_operator_create(const slb_operator_desc* d, slb_comm* comm, slb_operator** out) {
    SLB_REQUIRE(d && out, SLB_ERR_INVALID_ARG, "null descriptor/out");
    *out = nullptr;
    SLB_REQUIRE(d->kernel == SLB_LAPLACE_DL || d->kernel == SLB_STOKES_SLDL, SLB_ERR_INVALID_ARG, "bad kernel");
    const bool rag = d->panel_nt || d->panel_mt;      // ragged: nt, mt ignored (per-panel tables)
    SLB_REQUIRE(d->ns >= 1 && d->ms >= 1 && (rag || (d->nt >= 2 && d->mt >= 2 && d->nt % 2 == 0)),
                SLB_ERR_INVALID_ARG, "bad grid");
    SLB_REQUIRE(d->ns <= SLB_MAX_NS && d->ms <= SLB_MAX_MS && (rag || (d->nt <= SLB_MAX_NT && d->mt <= SLB_MAX_MT)),
                SLB_ERR_UNSUPPORTED, "grid beyond compiled limits");
    SLB_REQUIRE(d->n_panels_global >= 1 && d->panel_begin >= 0 && d->panel_end >= d->panel_begin &&
                    d->panel_end <= d->n_panels_global,
                SLB_ERR_INVALID_ARG, "bad panel range");
    const int R = comm ? comm->nranks : 1;
    SLB_REQUIRE(R > 1 || (d->panel_begin == 0 && d->panel_end == d->n_panels_global), SLB_ERR_INVALID_ARG,
                "single-GPU operator must own all panels");
    SLB_REQUIRE(d->n_trg_local >= 0 && d->n_on_local >= 0 && d->n_on_local <= d->n_trg_local,
                SLB_ERR_INVALID_ARG, "bad target counts");
    SLB_REQUIRE(d->y_fine && d->n_fine && d->w_fine, SLB_ERR_INVALID_ARG, "null fine geometry");
    SLB_REQUIRE(d->n_trg_local == 0 || (d->x_trg && d->row_ptr), SLB_ERR_INVALID_ARG, "null targets/CSR");
    SLB_REQUIRE(check_sticky("slb_operator_create") == SLB_OK, SLB_ERR_CUDA, slb_last_error());
    SLB_REQUIRE(coincident_counter(), SLB_ERR_CUDA, "coincident counter allocation failed");   // before any capture

    slb_operator* op = new slb_operator;
    op->d = *d;
    op->comm = comm;
    op->sdim = op->tdim = (d->kernel == SLB_LAPLACE_DL) ? 1 : 3;
    if (d->kernel == SLB_LAPLACE_DL) op->kind = (d->eta_fine || d->eta > 0.0) ? FAR_LAPLACE_SLDL : FAR_LAPLACE;
    else op->kind = (d->eta_fine || d->eta > 0.0) ? FAR_STOKES_SLDL : FAR_STOKES_DL;
    op->ragged = d->panel_nt || d->panel_mt || d->panel_ns || d->panel_ms;
    if (op->ragged) {
        // (NEXT N4) per-panel orders: node offsets and one interpolation bucket per (ns, nt, ms, mt)
        if (!d->panel_nt != !d->panel_mt || !d->panel_ns != !d->panel_ms) {
            free_op(op);
            set_error("slb_operator_create: panel_nt/panel_mt and panel_ns/panel_ms come in pairs");
            return SLB_ERR_INVALID_ARG;
        }
        const int64_t P = d->n_panels_global;
        op->cn0.assign(P + 1, 0);
        op->fn0.assign(P + 1, 0);
        std::vector<int32_t> pb(P);
        for (int64_t k = 0; k < P; ++k) {
            const int nt = d->panel_nt ? d->panel_nt[k] : d->nt, mt = d->panel_mt ? d->panel_mt[k] : d->mt;
            const int ns = d->panel_ns ? d->panel_ns[k] : d->ns, ms = d->panel_ms ? d->panel_ms[k] : d->ms;
            if (!(nt >= 2 && nt % 2 == 0 && mt >= 2 && nt <= SLB_MAX_NT && mt <= SLB_MAX_MT && ns >= 1 && ms >= 1 &&
                  ns <= SLB_MAX_NS && ms <= SLB_MAX_MS)) {
                free_op(op);
                set_error("slb_operator_create: panel orders must be positive (N_th even) and within the compiled limits");
                return SLB_ERR_INVALID_ARG;
            }
            op->cn0[k + 1] = op->cn0[k] + (int64_t)ns * nt;
            op->fn0[k + 1] = op->fn0[k] + (int64_t)ms * mt;
            op->max_cols = std::max(op->max_cols, ns * nt * op->sdim);
            int b = 0;
            while (b < (int)op->buckets.size() && !(op->buckets[b].nt == nt && op->buckets[b].mt == mt &&
                                                    op->buckets[b].ns == ns && op->buckets[b].ms == ms))
                ++b;
            if (b == (int)op->buckets.size()) {
                op->buckets.emplace_back();
                slb_operator::Bucket& nb = op->buckets.back();
                nb.nt = nt;
                nb.mt = mt;
                nb.ns = ns;
                nb.ms = ms;
                if (!make_interp(ns, nt, ms, mt, &nb.ip, &nb.ip_buf)) {
                    free_op(op);
                    set_error("slb_operator_create: interpolation matrices: allocation failed");
                    return SLB_ERR_OOM;
                }
            }
            pb[k] = b;
            if (k >= d->panel_begin && k < d->panel_end) op->buckets[b].n_loc++;
        }
        op->ip = op->buckets[0].ip;
        op->Nn = 0;                              // no uniform panel size
        op->Mn = 0;
        op->M = op->fn0[P];
        op->P_loc = d->panel_end - d->panel_begin;
        op->N_loc = op->cn0[d->panel_end] - op->cn0[d->panel_begin];
        op->cols = 0;
        // device tables (setup; synchronous)
        const int64_t Pl = op->P_loc;
        std::vector<int64_t> lc(Pl + 1), lf(Pl + 1);
        for (int64_t q = 0; q <= Pl; ++q) {
            lc[q] = op->cn0[d->panel_begin + q] - op->cn0[d->panel_begin];
            lf[q] = op->fn0[d->panel_begin + q] - op->fn0[d->panel_begin];
        }
        bool okm = cudaMalloc(&op->cn0_d, sizeof(int64_t) * (P + 1)) == cudaSuccess &&
                   cudaMalloc(&op->fn0_d, sizeof(int64_t) * (P + 1)) == cudaSuccess &&
                   cudaMalloc(&op->lc0_d, sizeof(int64_t) * (Pl + 1)) == cudaSuccess &&
                   cudaMalloc(&op->lf0_d, sizeof(int64_t) * (Pl + 1)) == cudaSuccess &&
                   cudaMalloc(&op->pbucket_d, sizeof(int32_t) * P) == cudaSuccess;
        if (okm) {
            okm = cudaMemcpy(op->cn0_d, op->cn0.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(op->fn0_d, op->fn0.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(op->lc0_d, lc.data(), sizeof(int64_t) * (Pl + 1), cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(op->lf0_d, lf.data(), sizeof(int64_t) * (Pl + 1), cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(op->pbucket_d, pb.data(), sizeof(int32_t) * P, cudaMemcpyHostToDevice) == cudaSuccess;
            for (int bi = 0; bi < (int)op->buckets.size(); ++bi) {
                auto& b = op->buckets[bi];
                std::vector<int32_t> pl;
                for (int64_t q = 0; q < Pl; ++q)
                    if (pb[d->panel_begin + q] == bi) pl.push_back((int32_t)q);
                if (pl.empty()) continue;
                okm = okm && cudaMalloc(&b.plist_d, sizeof(int32_t) * pl.size()) == cudaSuccess;
                if (okm)
                    okm = cudaMemcpy(b.plist_d, pl.data(), sizeof(int32_t) * pl.size(), cudaMemcpyHostToDevice) ==
                          cudaSuccess;
            }
        }
        if (!okm) {
            free_op(op);
            set_error("slb_operator_create: allocating / copying the ragged tables failed");
            return SLB_ERR_OOM;
        }
    } else {
        if (!make_interp(d->ns, d->nt, d->ms, d->mt, &op->ip, &op->ip_buf)) {
            free_op(op);
            set_error("slb_operator_create: interpolation matrices: allocation failed");
            return SLB_ERR_OOM;
        }
        op->Nn = (int64_t)d->ns * d->nt;
        op->Mn = (int64_t)d->ms * d->mt;
        op->M = d->n_panels_global * op->Mn;
        op->P_loc = d->panel_end - d->panel_begin;
        op->N_loc = op->P_loc * op->Nn;
        op->cols = op->Nn * op->sdim;
    }
    op->plan = far_plan(op->M);
    {
        const char* e = getenv("SLB_FAR_PATH");
        // constant-bank path from M = 2^16 (measured: c3 far 7.15 vs 7.63 ms, c3v 9.05 vs 9.80 ms on the
        // TMA path); the choice depends on M only, so every rank of a sharded operator takes the same path
        op->use_const = e ? (std::string(e) == "const") : (op->M >= (int64_t(1) << 16));
        if (op->use_const) op->plan.n_chunks = far_const_bufs(op->M);
    }
    if (d->n_on_local > op->N_loc) {
        free_op(op);
        set_error("slb_operator_create: n_on_local exceeds the local node count");
        return SLB_ERR_INVALID_ARG;
    }
    if (d->n_bodies_local > 0 && far_scalar(op->kind)) {
        free_op(op);
        set_error("slb_operator_create: the projector needs the Stokes kernel");
        return SLB_ERR_INVALID_ARG;
    }
    cudaStream_t s = 0;
    auto fail = [&](slb_status st) { free_op(op); return st; };
#define OPCUDA(call)                                                                             \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess) {                                                                 \
            set_error(std::string("slb_operator_create: " #call ": ") + cudaGetErrorString(e_)); \
            return fail(e_ == cudaErrorMemoryAllocation ? SLB_ERR_OOM : SLB_ERR_CUDA);           \
        }                                                                                        \
    } while (0)
#define OPST(expr)                          \
    do {                                    \
        slb_status st_ = (expr);            \
        if (st_ != SLB_OK) return fail(st_); \
    } while (0)
    // rank panel ranges
    op->ranges.assign(R + 1, 0);
    if (!comm) {
        op->ranges[1] = d->n_panels_global;
    } else {                                      // every communicator (one rank included) gathers the ranges
        int64_t* dr = nullptr;
        OPCUDA(cudaMalloc(&dr, sizeof(int64_t) * 2 * R));
        int64_t mine[2] = {d->panel_begin, d->panel_end};
        OPCUDA(cudaMemcpy(dr + 2 * comm->rank, mine, sizeof(mine), cudaMemcpyHostToDevice));
        ncclResult_t r = nccl().AllGather(dr + 2 * comm->rank, dr, 2, ncclInt64, comm->comm, s);
        comm->n_allgather++;
        std::vector<int64_t> all(2 * R);
        cudaError_t e = cudaMemcpy(all.data(), dr, sizeof(int64_t) * 2 * R, cudaMemcpyDeviceToHost);
        cudaFree(dr);
        if (r != ncclSuccess || e != cudaSuccess) {
            set_error("slb_operator_create: gathering panel ranges failed");
            return fail(r != ncclSuccess ? SLB_ERR_NCCL : SLB_ERR_CUDA);
        }
        for (int q = 0; q < R; ++q) {
            if (all[2 * q] != op->ranges[q]) {
                set_error("slb_operator_create: rank panel ranges must be contiguous and ordered by rank");
                return fail(SLB_ERR_INVALID_ARG);
            }
            op->ranges[q + 1] = all[2 * q + 1];
        }
        if (op->ranges[R] != d->n_panels_global) {
            set_error("slb_operator_create: rank panel ranges do not cover all panels");
            return fail(SLB_ERR_INVALID_ARG);
        }
        for (int q = 1; q < R; ++q)
            if (op->ranges[q + 1] - op->ranges[q] != op->ranges[1] - op->ranges[0]) op->equal_shards = false;
    }
    const int64_t T = d->n_trg_local;
    const int64_t Mloc = op->ragged ? op->fn0[d->panel_end] - op->fn0[d->panel_begin] : op->P_loc * op->Mn;
    const int64_t n_coarse_global = op->ragged ? op->cn0[d->n_panels_global] * op->sdim : d->n_panels_global * op->cols;
    OPCUDA(cudaMalloc(&op->geo, sizeof(double) * op->M * 6));
    OPCUDA(cudaMalloc(&op->sc, sizeof(double) * std::max<int64_t>(Mloc, 1) * 4));
    // (NEXT N4) SLB_NVLS=1 with a communicator: the fine records live in a multicast object and the
    // upsample writes them through it (fused gather); needs the streaming upsample for every bucket
    {
        static const bool want = [] { const char* e = getenv("SLB_NVLS"); return e && e[0] == '1'; }();
        bool ok = want && comm && nvls_supported() && op->sc != nullptr;
        if (ok) {
            if (op->ragged) {
                for (auto& b : op->buckets)
                    if (b.n_loc && !upsample_streams(op->kind, b.ip, op->sdim, true, op->coarse, op->sc)) ok = false;
            } else {
                ok = upsample_streams(op->kind, op->ip, op->sdim, true, op->coarse, op->sc);
            }
        }
        if (ok && nvls_alloc(comm, sizeof(double) * op->M * 4, &op->nvls) == SLB_OK) {
            op->nvls_on = true;
            op->dyn = reinterpret_cast<double*>(op->nvls.uc_va);
            op->dyn_mc = reinterpret_cast<double*>(op->nvls.mc_va);
        } else {
            if (want)          // requested explicitly: say why the NCCL all-gather path is used instead
                fprintf(stderr, "slb: SLB_NVLS=1 but the multicast gather is unavailable (%s)\n",
                        !comm ? "no communicator" : !ok ? "device or upsample path unsupported" : slb_last_error());
            OPCUDA(cudaMalloc(&op->dyn, sizeof(double) * op->M * 4));
        }
    }
    OPCUDA(cudaMalloc(&op->coarse, sizeof(double) * n_coarse_global));
    OPCUDA(cudaMalloc(&op->partials, sizeof(double) * std::max<int64_t>(op->plan.n_chunks * T * op->tdim, 1)));
    OPCUDA(cudaMalloc(&op->sig_dev, sizeof(double) * std::max<int64_t>(op->N_loc * op->sdim, 1)));
    OPCUDA(cudaMalloc(&op->u_dev, sizeof(double) * std::max<int64_t>(T * op->tdim, 1)));
    OPCUDA(cudaMemset(op->dyn, 0, sizeof(double) * op->M * 4));
    OPCUDA(cudaMemset(op->coarse, 0, sizeof(double) * n_coarse_global));
    if (T > 0) OPST(csr_check(T, d->row_ptr, d->panel_idx, d->n_panels_global));
    const int64_t f0 = op->ragged ? op->fn0[d->panel_begin] : d->panel_begin * op->Mn;
    if (op->ragged && T > 0) {
        // block offsets in CSR order: block p = [tdim][ns nt_k sdim], k = panel_idx[p]
        int64_t nnz = 0;
        OPCUDA(cudaMemcpy(&nnz, d->row_ptr + T, sizeof(int64_t), cudaMemcpyDeviceToHost));
        std::vector<int32_t> pk(std::max<int64_t>(nnz, 1));
        if (nnz) OPCUDA(cudaMemcpy(pk.data(), d->panel_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
        std::vector<int64_t> bo(nnz + 1, 0);
        for (int64_t p = 0; p < nnz; ++p)
            bo[p + 1] = bo[p] + (int64_t)op->tdim * (op->cn0[pk[p] + 1] - op->cn0[pk[p]]) * op->sdim;
        op->blk_total = bo[nnz];
        OPCUDA(cudaMalloc(&op->boff_d, sizeof(int64_t) * (nnz + 1)));
        OPCUDA(cudaMemcpy(op->boff_d, bo.data(), sizeof(int64_t) * (nnz + 1), cudaMemcpyHostToDevice));
        std::vector<int64_t> bm(std::max<int64_t>(nnz, 1));
        for (int64_t p = 0; p < nnz; ++p)
            bm[p] = ((op->cn0[pk[p]] * op->sdim / 2) << 12) | ((op->cn0[pk[p] + 1] - op->cn0[pk[p]]) * op->sdim / 2);
        OPCUDA(cudaMalloc(&op->bmeta_d, sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
        OPCUDA(cudaMemcpy(op->bmeta_d, bm.data(), sizeof(int64_t) * nnz, cudaMemcpyHostToDevice));
    }
    OPST(pack_geo(op->kind, op->M, d->y_fine, d->n_fine, d->eta_fine, d->eta, op->geo, s));
    OPST(pack_scale(op->kind, Mloc, d->n_fine + 3 * f0, d->w_fine + f0, d->eta_fine ? d->eta_fine + f0 : nullptr,
                    d->eta, op->sc, s));
    if (!d->blocks_folded && T > 0 && d->blocks) {
        if (op->ragged) {
            for (int b = 0; b < (int)op->buckets.size(); ++b)
                OPST(fold_launch(op->kind, T, d->x_trg, d->row_ptr, d->panel_idx, op->buckets[b].ip, d->y_fine,
                                 d->n_fine, d->w_fine, d->eta_fine, d->eta, d->blocks, s, op->pbucket_d, b,
                                 op->fn0_d, op->boff_d));
        } else {
            OPST(fold_launch(op->kind, T, d->x_trg, d->row_ptr, d->panel_idx, op->ip, d->y_fine, d->n_fine,
                             d->w_fine, d->eta_fine, d->eta, d->blocks, s));
        }
    }
    // projector: body node offsets (local), moments, inverse inertia
    if (d->n_bodies_local > 0) {
        if (!(d->body_of_panel_local && d->y_coarse && d->w_coarse)) {
            set_error("slb_operator_create: projector needs body_of_panel_local, y_coarse, w_coarse");
            return fail(SLB_ERR_INVALID_ARG);
        }
        const int64_t nb = d->n_bodies_local;
        std::vector<int32_t> bop(op->P_loc);
        OPCUDA(cudaMemcpy(bop.data(), d->body_of_panel_local, sizeof(int32_t) * op->P_loc, cudaMemcpyDeviceToHost));
        std::vector<int64_t> nb0(nb + 1, 0);
        for (int64_t p = 0; p < op->P_loc; ++p) {
            int32_t b = bop[p];
            if (b < 0 || b >= nb || (p > 0 && b < bop[p - 1])) {
                set_error("slb_operator_create: body_of_panel_local must be nondecreasing in [0, n_bodies_local)");
                return fail(SLB_ERR_INVALID_ARG);
            }
            nb0[b + 1] += op->ragged ? op->cn0[d->panel_begin + p + 1] - op->cn0[d->panel_begin + p] : op->Nn;
        }
        for (int64_t b = 0; b < nb; ++b) nb0[b + 1] += nb0[b];
        for (int64_t b = 0; b < nb; ++b) op->max_nodes_body = std::max(op->max_nodes_body, nb0[b + 1] - nb0[b]);
        OPCUDA(cudaMalloc(&op->nb0, sizeof(int64_t) * (nb + 1)));
        OPCUDA(cudaMemcpy(op->nb0, nb0.data(), sizeof(int64_t) * (nb + 1), cudaMemcpyHostToDevice));
        OPCUDA(cudaMalloc(&op->bodyc, sizeof(double) * nb * 16));
        OPCUDA(cudaMalloc(&op->coef, sizeof(double) * nb * 6));
        OPCUDA(cudaMalloc(&op->Lsig, sizeof(double) * std::max<int64_t>(op->N_loc, 1) * 3));
        OPST(body_moments_launch(nb, op->nb0, d->y_coarse, d->w_coarse, op->bodyc, s));
        std::vector<double> mom(nb * 16);
        OPCUDA(cudaMemcpy(mom.data(), op->bodyc, sizeof(double) * nb * 16, cudaMemcpyDeviceToHost));
        std::vector<double> bc(nb * 16, 0.0);
        for (int64_t b = 0; b < nb; ++b) {
            const double* m = &mom[b * 16];
            double I[3][3] = {{m[4], m[5], m[6]}, {m[5], m[7], m[8]}, {m[6], m[8], m[9]}};
            double det = I[0][0] * (I[1][1] * I[2][2] - I[1][2] * I[2][1]) -
                         I[0][1] * (I[1][0] * I[2][2] - I[1][2] * I[2][0]) +
                         I[0][2] * (I[1][0] * I[2][1] - I[1][1] * I[2][0]);
            if (!(std::fabs(det) > 0.0) || !(m[0] > 0.0)) {
                set_error("slb_operator_create: singular body inertia");
                return fail(SLB_ERR_INVALID_ARG);
            }
            double* o = &bc[b * 16];
            o[0] = m[0]; o[1] = m[1]; o[2] = m[2]; o[3] = m[3];
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
                    // inverse = adj^T / det  (symmetric matrix)
                    o[4 + 3 * j + i] = (I[i1][j1] * I[i2][j2] - I[i1][j2] * I[i2][j1]) / det;
                }
        }
        OPCUDA(cudaMemcpy(op->bodyc, bc.data(), sizeof(double) * nb * 16, cudaMemcpyHostToDevice));
    }
    for (auto& e : op->ev) OPCUDA(cudaEventCreate(&e));
    if (T > 0) {
        int64_t nnz = 0;
        OPCUDA(cudaMemcpy(&nnz, d->row_ptr + T, sizeof(int64_t), cudaMemcpyDeviceToHost));
        const double bb = op->ragged ? (nnz ? op->blk_total * 8.0 / (double)nnz : 0.0)
                                     : (double)op->tdim * op->cols * 8.0;
        op->near_G = near_group_size(T, nnz, bb);
    }
    if (op->use_const) {
        OPCUDA(cudaMalloc(&op->rec, sizeof(double) * op->M * 10));
        for (auto& w : op->ws) OPCUDA(cudaStreamCreateWithFlags(&w, cudaStreamNonBlocking));
        OPCUDA(cudaEventCreateWithFlags(&op->fork, cudaEventDisableTiming));
        for (auto& e : op->join) OPCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        OPST(far_const_prepare());
        OPCUDA(cudaDeviceSynchronize());
        // Coincident-pair prescan (R14).  Targets and sources are fixed per operator, so whether any r = 0
        // pair exists is decided once: one checked far pass with zero strengths (dyn = 0 here) counts this
        // rank's pairs into a private counter.  With none, every apply uses the kernels without the select
        // and count (1.2 % faster on c4, bitwise-identical results); otherwise the checked kernels as before.
        const char* pe_env = getenv("SLB_CONST_PRESCAN");      // read per create (tests toggle it)
        const bool prescan = !(pe_env && pe_env[0] == '0');
        if (prescan && T > 0) {
            unsigned long long* cnt = nullptr;
            OPCUDA(cudaMalloc(&cnt, sizeof(unsigned long long)));
            cudaStream_t ps = nullptr;
            cudaError_t pe = cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking);
            slb_status st = (pe == cudaSuccess) ? SLB_OK : SLB_ERR_CUDA;
            if (st == SLB_OK && cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), ps) != cudaSuccess) st = SLB_ERR_CUDA;
            if (st == SLB_OK) st = pack_rec_launch(op->M, op->geo, op->dyn, op->rec, ps);
            if (st == SLB_OK) {
                ConstBankLock bank;
                st = bank.acquire(ps);
                int64_t nl = 0;
                if (st == SLB_OK)
                    st = far_const_issue(op->kind, op->M, T, d->x_trg, op->rec, op->partials, cnt, ps, op->ws, op->fork,
                                         op->join, &nl, true);
                g_launch_count += (unsigned long long)nl;
                if (st == SLB_OK) st = bank.release(ps);
            }
            unsigned long long h = 1;
            if (st == SLB_OK && (cudaStreamSynchronize(ps) != cudaSuccess ||
                                 cudaMemcpy(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess))
                st = SLB_ERR_CUDA;
            if (ps) cudaStreamDestroy(ps);
            cudaFree(cnt);
            OPST(st);
            op->prescan_pairs = h;
            op->far_check = (h != 0);
        }
        // capture the tile sequence once; if capture is not possible, slb_matvec issues it directly
        cudaStream_t cs = nullptr;
        OPCUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t g = nullptr;
        bool ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            slb_status st = far_const_issue(op->kind, op->M, T, d->x_trg, op->rec, op->partials, coincident_counter(),
                                            cs, op->ws, op->fork, op->join, &op->const_launches, op->far_check);
            cudaError_t e1 = cudaStreamEndCapture(cs, &g);
            ok = (st == SLB_OK && e1 == cudaSuccess && g != nullptr);
            if (ok) ok = cudaGraphInstantiate(&op->graph, g, 0) == cudaSuccess;
            if (g) cudaGraphDestroy(g);
        }
        cudaStreamDestroy(cs);
        if (!ok) {
            op->graph = nullptr;
            cudaGetLastError();            // clear the capture error; fall back to direct issue
        }
        op->const_launches = (T > 0) ? (op->M + far_const_tile(op->M) - 1) / far_const_tile(op->M) : 0;
    }
    OPCUDA(cudaDeviceSynchronize());
    OPST(check_launch("slb_operator_create"));
#undef OPCUDA
#undef OPST
    *out = op;
    return SLB_OK;
}

}  // extern "C"

// Stage 1 of an apply: the projector (mobility operators) and the upsample of the local panels into the
// fine source records (op->dyn at the rank's offset).  Returns where the later stages read sigma'.
struct PrepOut {
    const double* near_sig;
    const double* id_sig;
    const double* Lsig;
};
static slb_status prep_stage(slb_operator* op, const double* sigma_local, cudaStream_t s, PrepOut* po) {
    const slb_operator_desc& d = op->d;
    slb_status st;
    // local sigma' inside the global coarse buffer.  One GPU without the projector: the caller's sigma IS
    // sigma' and the finalize reads it in place (no copy).  With a communicator the upsample writes the
    // staged density into the global buffer as it reads it (fused copy), the projector writes sigma' there.
    double* sig_p = op->coarse + (op->ragged ? op->cn0[d.panel_begin] * op->sdim : d.panel_begin * op->cols);
    const double* up_src = sig_p;      // what the upsample reads
    const double* near_sig = op->coarse;
    const double* id_sig = sig_p;
    double* copy_out = nullptr;
    const double* Lsig = nullptr;
    if (d.n_bodies_local > 0) {
        st = proj_launch(d.n_bodies_local, op->nb0, d.y_coarse, d.w_coarse, op->bodyc, sigma_local, op->coef, sig_p,
                         op->Lsig, op->max_nodes_body, s);
        if (st != SLB_OK) return st;
        Lsig = op->Lsig;
    } else if (op->N_loc > 0) {
        up_src = sigma_local;
        if (!op->comm) {
            near_sig = sigma_local;
            id_sig = sigma_local;
        } else {
            bool fused = true;
            if (op->ragged) {
                for (auto& b : op->buckets)
                    if (b.n_loc && !upsample_streams(op->kind, b.ip, op->sdim, true, sigma_local, op->sc)) fused = false;
            } else {
                fused = upsample_streams(op->kind, op->ip, op->sdim, true, sigma_local, op->sc);
            }
            if (fused) {
                copy_out = sig_p;
            } else {
                SLB_CUDA(cudaMemcpyAsync(sig_p, sigma_local, sizeof(double) * op->N_loc * op->sdim,
                                         cudaMemcpyDeviceToDevice, s));
                up_src = sig_p;
            }
        }
    }
    if (op->ragged) {
        double* dyn_loc = op->dyn + op->fn0[d.panel_begin] * 4;
        double* mc_loc = op->nvls_on ? op->dyn_mc + op->fn0[d.panel_begin] * 4 : nullptr;
        for (auto& b : op->buckets) {
            if (!b.n_loc) continue;
            st = upsample_launch(op->kind, b.n_loc, b.ip, op->sdim, up_src, nullptr, op->sc, dyn_loc, s, b.plist_d,
                                 op->lc0_d, op->lf0_d, copy_out, mc_loc);
            if (st != SLB_OK) return st;
        }
    } else {
        st = upsample_launch(op->kind, op->P_loc, op->ip, op->sdim, up_src, nullptr, op->sc,
                             op->dyn + d.panel_begin * op->Mn * 4, s, nullptr, nullptr, nullptr, copy_out,
                             op->nvls_on ? op->dyn_mc + d.panel_begin * op->Mn * 4 : nullptr);
        if (st != SLB_OK) return st;
    }
    po->near_sig = near_sig;
    po->id_sig = id_sig;
    po->Lsig = Lsig;
    return SLB_OK;
}

// The apply itself.  captured: being recorded into the operator's whole-apply graph (the stage events
// become event-record nodes; the constant-bank tiles are recorded inline and the bank lock is taken by
// the caller around the graph launch).
static slb_status matvec_body(slb_operator* op, const double* sigma_local, double* u_local, cudaStream_t s,
                              bool captured) {
    const slb_operator_desc& d = op->d;
    auto rec_ev = [&](int q) {
        return captured ? cudaEventRecordWithFlags(op->ev[q], s, cudaEventRecordExternal) : cudaEventRecord(op->ev[q], s);
    };
    unsigned long long* zc = coincident_counter();
    SLB_REQUIRE(zc, SLB_ERR_CUDA, "coincident counter allocation failed");
    slb_status st;
    SLB_CUDA(rec_ev(0));
    PrepOut po;
    st = prep_stage(op, sigma_local, s, &po);
    if (st != SLB_OK) return st;
    const double* near_sig = po.near_sig;
    const double* id_sig = po.id_sig;
    const double* Lsig = po.Lsig;
    SLB_CUDA(rec_ev(1));
    if (op->nvls_on) {
        // the records reached every rank's copy through the multicast stores; a barrier makes sure all
        // ranks finished writing before any reads (a one-rank team needs none)
        if (op->comm->nranks > 1) {
            SLB_NCCL(nccl().AllReduce(op->coincident_dummy(), op->coincident_dummy(), 1, ncclInt32, ncclSum,
                                      op->comm->comm, s));
            op->comm->n_allreduce++;
        }
    } else {
        st = op->ragged ? allgather(op, op->dyn, 0, s, &op->fn0, 4) : allgather(op, op->dyn, op->Mn * 4, s);
        if (st != SLB_OK) return st;
    }
    st = op->ragged ? allgather(op, op->coarse, 0, s, &op->cn0, op->sdim) : allgather(op, op->coarse, op->cols, s);
    if (st != SLB_OK) return st;
    SLB_CUDA(rec_ev(2));
    if (op->use_const) {
        st = pack_rec_launch(op->M, op->geo, op->dyn, op->rec, s);
        if (st != SLB_OK) return st;
        if (captured) {                            // tiles recorded inline; the caller holds the bank lock
            int64_t nl = 0;
            st = far_const_issue(op->kind, op->M, d.n_trg_local, d.x_trg, op->rec, op->partials, zc, s, op->ws,
                                 op->fork, op->join, &nl, op->far_check);
            if (st != SLB_OK) return st;
            g_launch_count += (unsigned long long)nl;
        } else {
            ConstBankLock bank;                    // the __constant__ bank is one per device (slb.h)
            st = bank.acquire(s);
            if (st != SLB_OK) return st;
            if (op->graph) {
                SLB_CUDA(cudaGraphLaunch(op->graph, s));
                g_launch_count += (unsigned long long)op->const_launches;
            } else {
                int64_t nl = 0;
                st = far_const_issue(op->kind, op->M, d.n_trg_local, d.x_trg, op->rec, op->partials, zc, s, op->ws,
                                     op->fork, op->join, &nl, op->far_check);
                if (st != SLB_OK) return st;
                g_launch_count += (unsigned long long)nl;
            }
            st = bank.release(s);
            if (st != SLB_OK) return st;
        }
    } else {
        st = far_partials(op->kind, op->plan, d.n_trg_local, d.x_trg, op->geo, op->dyn, op->partials, zc, s);
        if (st != SLB_OK) return st;
    }
    SLB_CUDA(rec_ev(3));
    RagNear rag;
    if (op->ragged) {
        rag.cn0 = op->cn0_d;
        rag.boff = op->boff_d;
        rag.max_cols = op->max_cols;
        rag.bmeta = op->bmeta_d;
    }
    st = finalize_launch(op->plan, d.n_trg_local, op->tdim, (int)op->cols, op->partials, d.row_ptr, d.panel_idx,
                         d.blocks, near_sig, d.n_on_local, d.c_identity, id_sig, Lsig, u_local, op->near_G, s, rag);
    if (st != SLB_OK) return st;
    SLB_CUDA(rec_ev(4));
    op->timed = true;
    return SLB_OK;
}

static bool apply_graphs_enabled(const slb_operator* op) {
    static const bool on = [] { const char* e = getenv("SLB_APPLY_GRAPH"); return !(e && e[0] == '0'); }();
    return on && (!op->comm || op->comm->nranks == 1);
}

namespace slb {
slb_status matvec_direct(slb_operator* op, const double* sigma_local, double* u_local, cudaStream_t s) {
    return matvec_body(op, sigma_local, u_local, s, false);
}
}  // namespace slb

extern "C" {

// One apply.  The whole sequence (projector, upsample, gathers, far field, finalize, stage events) is
// recorded once per (sigma, u) pointer pair into a CUDA graph (a small LRU per operator) and replayed,
// so consecutive kernels run back to back without host launch gaps (single-rank operators; the first
// call with a new pair runs directly and initialises everything lazily created).
slb_status slb_matvec(slb_operator* op, const double* sigma_local, double* u_local, cudaStream_t s) {
    SLB_REQUIRE(op, SLB_ERR_INVALID_ARG, "null operator");
    SLB_REQUIRE((op->N_loc == 0 || sigma_local) && (op->d.n_trg_local == 0 || u_local), SLB_ERR_INVALID_ARG,
                "null density/output");
    SLB_REQUIRE(check_sticky("slb_matvec") == SLB_OK, SLB_ERR_CUDA, slb_last_error());
    SLB_REQUIRE(coincident_counter(), SLB_ERR_CUDA, "coincident counter allocation failed");
    if (!apply_graphs_enabled(op)) return matvec_body(op, sigma_local, u_local, s, false);
    slb_operator::ApplyGraph* hit = nullptr;
    for (auto& g : op->apply_graphs)
        if (g.sigma == sigma_local && g.u == u_local) hit = &g;
    if (!hit) {
        if (!op->seen_direct) {
            op->seen_direct = true;
            return matvec_body(op, sigma_local, u_local, s, false);
        }
        if (!op->cap_stream) SLB_CUDA(cudaStreamCreateWithFlags(&op->cap_stream, cudaStreamNonBlocking));
        const unsigned long long c0 = g_launch_count.load();
        cudaGraph_t g = nullptr;
        SLB_CUDA(cudaStreamBeginCapture(op->cap_stream, cudaStreamCaptureModeThreadLocal));
        slb_status st = matvec_body(op, sigma_local, u_local, op->cap_stream, true);
        cudaError_t e = cudaStreamEndCapture(op->cap_stream, &g);
        const unsigned long long nl = g_launch_count.load() - c0;
        g_launch_count -= nl;                      // recorded, not launched
        cudaGraphExec_t ex = nullptr;
        if (st == SLB_OK && e == cudaSuccess && g) e = cudaGraphInstantiate(&ex, g, 0);
        if (g) cudaGraphDestroy(g);
        if (st != SLB_OK || e != cudaSuccess || !ex) {
            cudaGetLastError();
            return matvec_body(op, sigma_local, u_local, s, false);   // capture not possible: direct issue
        }
        if (op->apply_graphs.size() >= 4) {
            cudaGraphExecDestroy(op->apply_graphs.front().exec);
            op->apply_graphs.erase(op->apply_graphs.begin());
        }
        op->apply_graphs.push_back({sigma_local, u_local, ex, nl});
        hit = &op->apply_graphs.back();
    }
    if (op->use_const) {
        ConstBankLock bank;
        slb_status st = bank.acquire(s);
        if (st != SLB_OK) return st;
        SLB_CUDA(cudaGraphLaunch(hit->exec, s));
        st = bank.release(s);
        if (st != SLB_OK) return st;
    } else {
        SLB_CUDA(cudaGraphLaunch(hit->exec, s));
    }
    g_launch_count += hit->launches;
    op->timed = true;
    return SLB_OK;
}

slb_status slb_matvec_host(slb_operator* op, const double* sigma_host, double* u_host, cudaStream_t s) {
    SLB_REQUIRE(op && sigma_host && u_host, SLB_ERR_INVALID_ARG, "null argument");
    SLB_CUDA(cudaMemcpyAsync(op->sig_dev, sigma_host, sizeof(double) * op->N_loc * op->sdim, cudaMemcpyHostToDevice, s));
    slb_status st = slb_matvec(op, op->sig_dev, op->u_dev, s);
    if (st != SLB_OK) return st;
    SLB_CUDA(cudaMemcpyAsync(u_host, op->u_dev, sizeof(double) * op->d.n_trg_local * op->tdim,
                             cudaMemcpyDeviceToHost, s));
    SLB_CUDA(cudaStreamSynchronize(s));
    return SLB_OK;
}

slb_status slb_operator_prepare(slb_operator* op, const double* sigma_local, cudaStream_t s) {
    SLB_REQUIRE(op, SLB_ERR_INVALID_ARG, "null operator");
    SLB_REQUIRE(op->N_loc == 0 || sigma_local, SLB_ERR_INVALID_ARG, "null density");
    SLB_REQUIRE(check_sticky("slb_operator_prepare") == SLB_OK, SLB_ERR_CUDA, slb_last_error());
    PrepOut po;
    return prep_stage(op, sigma_local, s, &po);
}

slb_status slb_operator_last_timings(slb_operator* op, float out_ms[4]) {
    SLB_REQUIRE(op && out_ms, SLB_ERR_INVALID_ARG, "null argument");
    for (int q = 0; q < 4; ++q) out_ms[q] = -1.0f;
    if (!op->timed) return SLB_OK;
    SLB_CUDA(cudaEventSynchronize(op->ev[4]));
    for (int q = 0; q < 4; ++q) SLB_CUDA(cudaEventElapsedTime(&out_ms[q], op->ev[q], op->ev[q + 1]));
    return SLB_OK;
}

int slb_operator_nvls(const slb_operator* op) { return (op && op->nvls_on) ? 1 : 0; }

int slb_operator_launches_per_matvec(const slb_operator* op) {
    if (!op) return -1;
    int n = 3;                                   // upsample, far, finalize
    if (op->ragged) {                            // one upsample per bucket with local panels
        n -= 1;
        for (auto& b : op->buckets) n += b.n_loc > 0;
    }
    if (op->use_const) n += 1 + (int)op->const_launches - 1;   // pack_rec + one launch per source tile
    if (op->d.n_bodies_local > 0) n += 2;        // projector coef + apply
    return n;
}

slb_status slb_operator_destroy(slb_operator* op) {
    free_op(op);
    return SLB_OK;
}

}  // extern "C"
