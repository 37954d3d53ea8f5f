// api.cu -- C-ABI entry points for the stand-alone steps of the operator apply, plus the
// error/status plumbing shared by the library.  See include/slb.h for the contract.
#include <atomic>
#include <cmath>
#include <string>
#include <array>
#include <memory>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>
#include "common.cuh"

namespace slb {

static thread_local std::string g_err;
std::atomic<unsigned long long> g_launch_count{0};

void set_error(const std::string& msg) { g_err = msg; }

slb_status check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(what) + ": " + cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? SLB_ERR_OOM : SLB_ERR_CUDA;
    }
    return SLB_OK;
}

slb_status check_sticky(const char* what) {
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) {
        set_error(std::string(what) + ": pending CUDA error: " + cudaGetErrorString(e));
        return SLB_ERR_CUDA;
    }
    return SLB_OK;
}

// Function-local static initialisers: thread-safe one-time initialisation (C++11).
int num_sms() {
    static const int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return n;
}

unsigned long long* coincident_counter() {
    // allocated on first use outside any stream capture (slb_operator_create calls it before it
    // captures); a failed attempt is not cached
    static std::mutex mu;
    static std::atomic<unsigned long long*> p{nullptr};
    unsigned long long* v = p.load();
    if (v) return v;
    std::lock_guard<std::mutex> lk(mu);
    if (p.load()) return p.load();
    unsigned long long* q = nullptr;
    if (cudaMalloc(&q, sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    if (cudaMemset(q, 0, sizeof(unsigned long long)) != cudaSuccess) { cudaFree(q); return nullptr; }
    p.store(q);
    return q;
}

// Opt a kernel in to the device's full dynamic shared memory once (the attribute is process-wide;
// setting it to the maximum once, under a lock, means no launch can lower it under another).
slb_status smem_optin(const void* fn) {
    static std::mutex mu;
    static std::set<const void*> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(fn)) return SLB_OK;
    int dev = 0, mx = 0;
    SLB_CUDA(cudaGetDevice(&dev));
    SLB_CUDA(cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    SLB_CUDA(cudaFuncGetAttributes(&fa, fn));          // dynamic limit = opt-in maximum - static shared
    SLB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fa.sharedSizeBytes));
    done.insert(fn);
    return SLB_OK;
}

}  // namespace slb

using namespace slb;

extern "C" {

int slb_abi_version(void) { return SLB_ABI_VERSION; }

const char* slb_last_error(void) { return g_err.c_str(); }

double slb_eta_cfie(double rho) {
    if (!(rho > 0.0 && rho < 1.0)) return NAN;
    return 1.0 / (2.0 * rho * std::log(1.0 / rho));
}

long long slb_coincident_count(void) {
    unsigned long long* p = coincident_counter();
    if (!p) return -1;
    unsigned long long v = 0;
    if (cudaMemcpy(&v, p, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return (long long)v;
}

void slb_coincident_reset(void) {
    unsigned long long* p = coincident_counter();
    if (p) cudaMemset(p, 0, sizeof(unsigned long long));
}

unsigned long long slb_launch_count(void) { return g_launch_count; }

slb_status slb_upsample(int64_t n_panels, int ns, int nt, int ms, int mt, int ncomp,
                        const double* sigma_coarse, double* sigma_fine, cudaStream_t s) {
    SLB_REQUIRE(n_panels >= 0, SLB_ERR_INVALID_ARG, "n_panels < 0");
    SLB_REQUIRE(ncomp == 1 || ncomp == 3, SLB_ERR_INVALID_ARG, "ncomp must be 1 or 3");
    SLB_REQUIRE(ns >= 1 && nt >= 2 && ms >= 1 && mt >= 2 && nt % 2 == 0, SLB_ERR_INVALID_ARG,
                "need ns, ms >= 1 and even nt >= 2");
    SLB_REQUIRE(ns <= SLB_MAX_NS && nt <= SLB_MAX_NT && ms <= SLB_MAX_MS && mt <= SLB_MAX_MT,
                SLB_ERR_UNSUPPORTED, "grid beyond compiled limits");
    if (n_panels == 0) return SLB_OK;
    SLB_REQUIRE(sigma_coarse && sigma_fine, SLB_ERR_INVALID_ARG, "null pointer");
    SLB_REQUIRE(check_sticky("slb_upsample") == SLB_OK, SLB_ERR_CUDA, slb_last_error());
    std::unique_ptr<InterpParams> ipp(new InterpParams);   // 29 KB: heap, per call (thread-safe)
    InterpParams& ip = *ipp;
    double* owned = nullptr;  // device copy of large interpolation matrices (freed after the launch)
    SLB_REQUIRE(make_interp(ns, nt, ms, mt, &ip, &owned), SLB_ERR_OOM, "interpolation matrices: allocation failed");
    slb_status st = upsample_launch(FAR_STOKES_SLDL, n_panels, ip, ncomp, sigma_coarse, sigma_fine, nullptr, nullptr, s);
    if (owned) { cudaStreamSynchronize(s); cudaFree(owned); }
    return st;
}

slb_status slb_upsample_ragged(int64_t n_panels, const int32_t* ns, const int32_t* nt, const int32_t* ms,
                               const int32_t* mt, int ncomp, const double* sigma_coarse, double* sigma_fine,
                               cudaStream_t s) {
    SLB_REQUIRE(n_panels >= 0, SLB_ERR_INVALID_ARG, "n_panels < 0");
    SLB_REQUIRE(ncomp == 1 || ncomp == 3, SLB_ERR_INVALID_ARG, "ncomp must be 1 or 3");
    if (n_panels == 0) return SLB_OK;
    SLB_REQUIRE(ns && nt && ms && mt && sigma_coarse && sigma_fine, SLB_ERR_INVALID_ARG, "null pointer");
    SLB_REQUIRE(check_sticky("slb_upsample_ragged") == SLB_OK, SLB_ERR_CUDA, slb_last_error());
    std::vector<int64_t> c0(n_panels + 1, 0), f0(n_panels + 1, 0);
    std::map<std::array<int, 4>, std::vector<int32_t>> groups;
    for (int64_t p = 0; p < n_panels; ++p) {
        SLB_REQUIRE(nt[p] >= 2 && nt[p] % 2 == 0 && nt[p] <= SLB_MAX_NT && mt[p] >= 2 && mt[p] <= SLB_MAX_MT &&
                        ns[p] >= 1 && ns[p] <= SLB_MAX_NS && ms[p] >= 1 && ms[p] <= SLB_MAX_MS,
                    SLB_ERR_INVALID_ARG, "panel orders must be positive (N_th even) and within the compiled limits");
        c0[p + 1] = c0[p] + (int64_t)ns[p] * nt[p];
        f0[p + 1] = f0[p] + (int64_t)ms[p] * mt[p];
        groups[{ns[p], nt[p], ms[p], mt[p]}].push_back((int32_t)p);
    }
    int64_t *c0d = nullptr, *f0d = nullptr;
    int32_t* pl = nullptr;
    slb_status st = SLB_OK;
    auto cleanup = [&]() { cudaFree(c0d); cudaFree(f0d); cudaFree(pl); };
    if (cudaMalloc(&c0d, sizeof(int64_t) * (n_panels + 1)) != cudaSuccess ||
        cudaMalloc(&f0d, sizeof(int64_t) * (n_panels + 1)) != cudaSuccess ||
        cudaMalloc(&pl, sizeof(int32_t) * n_panels) != cudaSuccess) {
        cleanup();
        set_error("slb_upsample_ragged: out of device memory");
        return SLB_ERR_OOM;
    }
    std::vector<int32_t> flat;
    for (auto& g : groups) flat.insert(flat.end(), g.second.begin(), g.second.end());
    if (cudaMemcpy(c0d, c0.data(), sizeof(int64_t) * (n_panels + 1), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(f0d, f0.data(), sizeof(int64_t) * (n_panels + 1), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(pl, flat.data(), sizeof(int32_t) * n_panels, cudaMemcpyHostToDevice) != cudaSuccess) {
        cleanup();
        set_error("slb_upsample_ragged: copying the panel tables failed");
        return SLB_ERR_CUDA;
    }
    std::unique_ptr<InterpParams> ipp(new InterpParams);
    InterpParams& ip = *ipp;
    std::vector<double*> owned;
    int64_t off = 0;
    for (auto& g : groups) {
        double* o = nullptr;
        if (!make_interp(g.first[0], g.first[1], g.first[2], g.first[3], &ip, &o)) {
            set_error("slb_upsample_ragged: interpolation matrices: allocation failed");
            st = SLB_ERR_OOM;
            break;
        }
        if (o) owned.push_back(o);
        st = upsample_launch(FAR_STOKES_SLDL, (int64_t)g.second.size(), ip, ncomp, sigma_coarse, sigma_fine,
                             nullptr, nullptr, s, pl + off, c0d, f0d);
        if (st != SLB_OK) break;
        off += (int64_t)g.second.size();
    }
    cudaError_t e = cudaStreamSynchronize(s);
    cleanup();
    for (double* o : owned) cudaFree(o);
    if (st == SLB_OK && e != cudaSuccess) {
        set_error(std::string("slb_upsample_ragged: ") + cudaGetErrorString(e));
        st = SLB_ERR_CUDA;
    }
    return st;
}

static slb_status farfield_common(FarKind kind, int64_t n_trg, const double* x, int64_t n_src,
                                  const double* y, const double* n, const double* w,
                                  const double* eta_src, double eta, const double* sigma, double* u,
                                  cudaStream_t s) {
    SLB_REQUIRE(n_trg >= 0 && n_src >= 0, SLB_ERR_INVALID_ARG, "negative size");
    if (n_trg == 0) return SLB_OK;
    SLB_REQUIRE(x && u, SLB_ERR_INVALID_ARG, "null target/output pointer");
    SLB_REQUIRE(n_src == 0 || (y && n && w && sigma), SLB_ERR_INVALID_ARG, "null source pointer");
    SLB_REQUIRE(check_sticky("farfield") == SLB_OK, SLB_ERR_CUDA, slb_last_error());
    unsigned long long* zc = coincident_counter();
    SLB_REQUIRE(zc, SLB_ERR_CUDA, "coincident counter allocation failed");
    const int tdim = far_scalar(kind) ? 1 : 3;
    FarPlan plan = far_plan(n_src);
    double *geo = nullptr, *sc = nullptr, *dyn = nullptr, *part = nullptr;
    const int64_t M = n_src > 0 ? n_src : 1;
    SLB_CUDA(cudaMallocAsync(&geo, sizeof(double) * M * 6, s));
    SLB_CUDA(cudaMallocAsync(&sc, sizeof(double) * M * 4, s));
    SLB_CUDA(cudaMallocAsync(&dyn, sizeof(double) * M * 4, s));
    SLB_CUDA(cudaMallocAsync(&part, sizeof(double) * plan.n_chunks * n_trg * tdim, s));
    slb_status st = SLB_OK;
    if (n_src > 0) {
        if (st == SLB_OK) st = pack_geo(kind, n_src, y, n, eta_src, eta, geo, s);
        if (st == SLB_OK) st = pack_scale(kind, n_src, n, w, eta_src, eta, sc, s);
        if (st == SLB_OK) st = pack_dyn(kind, n_src, sc, sigma, dyn, s);
    }
    if (st == SLB_OK) st = far_partials(kind, plan, n_trg, x, geo, dyn, part, zc, s);
    if (st == SLB_OK) st = far_reduce(plan, n_trg, tdim, part, u, s);
    cudaFreeAsync(geo, s);
    cudaFreeAsync(sc, s);
    cudaFreeAsync(dyn, s);
    cudaFreeAsync(part, s);
    return st;
}

slb_status slb_farfield_laplace_dl(int64_t n_trg, const double* x_trg, int64_t n_src, const double* y,
                                   const double* n, const double* w, const double* sigma, double* u,
                                   cudaStream_t s) {
    return farfield_common(FAR_LAPLACE, n_trg, x_trg, n_src, y, n, w, nullptr, 0.0, sigma, u, s);
}

slb_status slb_farfield_stokes_sldl(int64_t n_trg, const double* x_trg, int64_t n_src, const double* y,
                                    const double* n, const double* w, const double* eta_src, double eta,
                                    const double* sigma, double* u, cudaStream_t s) {
    SLB_REQUIRE(eta_src || eta >= 0.0, SLB_ERR_INVALID_ARG, "scalar eta must be >= 0");
    FarKind kind = (eta_src || eta > 0.0) ? FAR_STOKES_SLDL : FAR_STOKES_DL;
    return farfield_common(kind, n_trg, x_trg, n_src, y, n, w, eta_src, eta, sigma, u, s);
}

slb_status slb_nearcorr_apply(int64_t n_trg, int tdim, int sdim, int nodes_per_panel,
                              const int64_t* row_ptr, const int32_t* panel_idx, const double* blocks,
                              const double* sigma_coarse, double* u, cudaStream_t s) {
    SLB_REQUIRE(n_trg >= 0, SLB_ERR_INVALID_ARG, "n_trg < 0");
    SLB_REQUIRE((tdim == 1 || tdim == 3) && (sdim == 1 || sdim == 3), SLB_ERR_INVALID_ARG,
                "tdim and sdim must be 1 or 3");
    SLB_REQUIRE(nodes_per_panel > 0 && (nodes_per_panel * sdim) % 2 == 0, SLB_ERR_INVALID_ARG,
                "nodes_per_panel*sdim must be positive and even");
    if (n_trg == 0) return SLB_OK;
    SLB_REQUIRE(row_ptr && u, SLB_ERR_INVALID_ARG, "null pointer");
    SLB_REQUIRE(check_sticky("slb_nearcorr_apply") == SLB_OK, SLB_ERR_CUDA, slb_last_error());
    return near_apply_launch(n_trg, tdim, nodes_per_panel * sdim, row_ptr, panel_idx, blocks,
                             sigma_coarse, u, s);
}

slb_status slb_nearcorr_fold(slb_kernel kernel, int64_t n_trg, const double* x_trg, const int64_t* row_ptr,
                             const int32_t* panel_idx, int ns, int nt, int ms, int mt,
                             const double* y_fine, const double* n_fine, const double* w_fine,
                             const double* eta_fine, double eta, double* blocks, cudaStream_t s) {
    SLB_REQUIRE(kernel == SLB_LAPLACE_DL || kernel == SLB_STOKES_SLDL, SLB_ERR_INVALID_ARG, "bad kernel");
    SLB_REQUIRE(n_trg >= 0, SLB_ERR_INVALID_ARG, "n_trg < 0");
    SLB_REQUIRE(ns >= 1 && nt >= 2 && ms >= 1 && mt >= 2 && nt % 2 == 0, SLB_ERR_INVALID_ARG, "bad grid");
    SLB_REQUIRE(ns <= SLB_MAX_NS && nt <= SLB_MAX_NT && ms <= SLB_MAX_MS && mt <= SLB_MAX_MT,
                SLB_ERR_UNSUPPORTED, "grid beyond compiled limits");
    if (n_trg == 0) return SLB_OK;
    SLB_REQUIRE(x_trg && row_ptr && y_fine && n_fine && w_fine, SLB_ERR_INVALID_ARG, "null pointer");
    std::unique_ptr<InterpParams> ipp(new InterpParams);
    InterpParams& ip = *ipp;
    double* owned = nullptr;
    SLB_REQUIRE(make_interp(ns, nt, ms, mt, &ip, &owned), SLB_ERR_OOM, "interpolation matrices: allocation failed");
    FarKind kind = kernel == SLB_LAPLACE_DL ? ((eta_fine || eta > 0.0) ? FAR_LAPLACE_SLDL : FAR_LAPLACE)
                                            : ((eta_fine || eta > 0.0) ? FAR_STOKES_SLDL : FAR_STOKES_DL);
    slb_status st = fold_launch(kind, n_trg, x_trg, row_ptr, panel_idx, ip, y_fine, n_fine, w_fine, eta_fine, eta,
                                blocks, s);
    if (owned) { cudaStreamSynchronize(s); cudaFree(owned); }
    return st;
}

}  // extern "C"
