// gmres.cu -- (NEXT N2) restarted GMRES around slb_matvec.
//
// The paper solves its second-kind BIEs (Laplace CFIE P:L1750, Stokes CFIE P:L1868, projected
// mobility (K(I-L)+L) P:L2009) with GMRES; this is that solver around the
// operator apply.  GMRES(m) with classical Gram-Schmidt applied twice (CGS2: one fused multi-dot
// + one fused update per pass), Givens rotations and the small least-squares problem on the host.
// Every reduction has a fixed order (per-block tree -> fixed-order block sum on device -> NCCL
// all-reduce across ranks), so a solve is bitwise reproducible for a fixed number of ranks.
// Convergence: ||b - A x|| <= tol ||b||, the true residual re-evaluated at every restart.
#include <algorithm>
#include <cmath>
#include <vector>
#include "operator_impl.cuh"

namespace slb {

constexpr int kDotBlocks = 256;
constexpr int kDotThreads = 256;

// partial[i][blk] = sum over this block's grid-stride segment of V_i . w
__global__ void __launch_bounds__(kDotThreads) multidot_kernel(int64_t n, int k, const double* __restrict__ V,
                                                               int64_t ld, const double* __restrict__ w,
                                                               double* __restrict__ partial) {
    __shared__ double red[kDotThreads];
    const int i = blockIdx.y;
    const double* v = V + (int64_t)i * ld;
    double acc = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; e < n; e += (int64_t)gridDim.x * kDotThreads)
        acc = fma(v[e], w[e], acc);
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kDotThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[(int64_t)i * gridDim.x + blockIdx.x] = red[0];
}

// dots[i] = sum_b partial[i][b] in order
__global__ void sum_partials_kernel(int k, int nb, const double* __restrict__ partial, double* __restrict__ dots) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += partial[(int64_t)i * nb + b];
    dots[i] = s;
}

// w[e] += alpha * sum_{i<k} h[i] V_i[e]
__global__ void update_kernel(int64_t n, int k, const double* __restrict__ V, int64_t ld,
                              const double* __restrict__ h, double alpha, double* __restrict__ w) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < k; ++i) s = fma(h[i], V[(int64_t)i * ld + e], s);
        w[e] = fma(alpha, s, w[e]);
    }
}

// out = a * x + b * y
__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b,
                             const double* __restrict__ y, double* __restrict__ out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = a * x[e] + (y ? b * y[e] : 0.0);
}

struct Gm {
    slb_operator* op;
    cudaStream_t s;
    int64_t n;
    double *partial, *dots_d, *h_d;
    std::vector<double> dots_h;
    int nblk;

    slb_status dots(int k, const double* V, int64_t ld, const double* w, double* out) {
        dim3 grid(nblk, k);
        multidot_kernel<<<grid, kDotThreads, 0, s>>>(n, k, V, ld, w, partial);
        sum_partials_kernel<<<(k + 63) / 64, 64, 0, s>>>(k, nblk, partial, dots_d);
        g_launch_count += 2;
        if (op->comm) {                       // every communicator, one rank included (the path is exercised)
            NcclApi& A = nccl();
            SLB_NCCL(A.AllReduce(dots_d, dots_d, (size_t)k, ncclDouble, ncclSum, op->comm->comm, s));
            op->comm->n_allreduce++;
        }
        SLB_CUDA(cudaMemcpyAsync(out, dots_d, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
        SLB_CUDA(cudaStreamSynchronize(s));
        return check_launch("gmres dots");
    }
    slb_status update(int k, const double* V, int64_t ld, const double* h, double alpha, double* w) {
        SLB_CUDA(cudaMemcpyAsync(h_d, h, sizeof(double) * k, cudaMemcpyHostToDevice, s));
        update_kernel<<<num_sms() * 4, 256, 0, s>>>(n, k, V, ld, h_d, alpha, w);
        ++g_launch_count;
        SLB_CUDA(cudaStreamSynchronize(s));   // h_d is reused by the next call
        return check_launch("gmres update");
    }
    slb_status axpby(double a, const double* x, double b, const double* y, double* out) {
        axpby_kernel<<<num_sms() * 4, 256, 0, s>>>(n, a, x, b, y, out);
        ++g_launch_count;
        return check_launch("gmres axpby");
    }
};

}  // namespace slb

using namespace slb;

extern "C" slb_status slb_gmres(slb_operator* op, const double* rhs, double* x, int restart, int max_iters,
                                double tol, int* iters_out, double* relres_out, cudaStream_t s) {
    SLB_REQUIRE(op && rhs && x, SLB_ERR_INVALID_ARG, "null argument");
    SLB_REQUIRE(restart >= 1 && restart <= 512 && max_iters >= 1 && tol > 0.0, SLB_ERR_INVALID_ARG,
                "need 1 <= restart <= 512, max_iters >= 1, tol > 0");
    SLB_REQUIRE(op->d.n_trg_local == op->N_loc && op->d.n_on_local == op->N_loc, SLB_ERR_INVALID_ARG,
                "GMRES needs a square operator: targets must be exactly the local nodes");
    const int64_t n = op->N_loc * op->sdim;
    const int m = restart;
    Gm g;
    g.op = op;
    g.s = s;
    g.n = n;
    g.nblk = kDotBlocks;
    double *V = nullptr, *w = nullptr;
    const int64_t ld = std::max<int64_t>(n, 1);
    SLB_CUDA(cudaMallocAsync(&V, sizeof(double) * ld * (m + 1), s));
    SLB_CUDA(cudaMallocAsync(&w, sizeof(double) * ld, s));
    SLB_CUDA(cudaMallocAsync(&g.partial, sizeof(double) * (size_t)kDotBlocks * (m + 1), s));
    SLB_CUDA(cudaMallocAsync(&g.dots_d, sizeof(double) * (m + 1), s));
    SLB_CUDA(cudaMallocAsync(&g.h_d, sizeof(double) * (m + 1), s));
    std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), gv(m + 1), y(m), h(m + 1), h2(m + 1);
    slb_status st = SLB_OK;
    double bnorm = 0.0, relres = 1.0;
    int it = 0;
    auto cleanup = [&]() {
        cudaFreeAsync(V, s); cudaFreeAsync(w, s); cudaFreeAsync(g.partial, s);
        cudaFreeAsync(g.dots_d, s); cudaFreeAsync(g.h_d, s);
    };
#define GM(expr) do { st = (expr); if (st != SLB_OK) { cleanup(); return st; } } while (0)
    double d1;
    GM(g.dots(1, rhs, ld, rhs, &d1));
    bnorm = std::sqrt(d1);
    if (bnorm == 0.0) {
        GM(g.axpby(0.0, x, 0.0, nullptr, x));
        if (iters_out) *iters_out = 0;
        if (relres_out) *relres_out = 0.0;
        cleanup();
        return SLB_OK;
    }
    while (true) {
        // r = b - A x  into V_0
        GM(matvec_direct(op, x, w, s));
        GM(g.axpby(1.0, rhs, -1.0, w, V));
        double rr;
        GM(g.dots(1, V, ld, V, &rr));
        const double beta = std::sqrt(rr);
        relres = beta / bnorm;
        if (relres <= tol || it >= max_iters) break;
        GM(g.axpby(1.0 / beta, V, 0.0, nullptr, V));
        std::fill(gv.begin(), gv.end(), 0.0);
        gv[0] = beta;
        int j = 0;
        for (; j < m && it < max_iters; ++j, ++it) {
            GM(matvec_direct(op, V + (int64_t)j * ld, w, s));
            // CGS2
            GM(g.dots(j + 1, V, ld, w, h.data()));
            GM(g.update(j + 1, V, ld, h.data(), -1.0, w));
            GM(g.dots(j + 1, V, ld, w, h2.data()));
            GM(g.update(j + 1, V, ld, h2.data(), -1.0, w));
            for (int i = 0; i <= j; ++i) h[i] += h2[i];
            double ww;
            GM(g.dots(1, w, ld, w, &ww));
            const double hn = std::sqrt(ww);
            h[j + 1] = hn;
            if (hn > 0.0) GM(g.axpby(1.0 / hn, w, 0.0, nullptr, V + (int64_t)(j + 1) * ld));
            // Givens
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * h[i] + sn[i] * h[i + 1];
                h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
                h[i] = t;
            }
            const double den = std::hypot(h[j], h[j + 1]);
            cs[j] = den > 0.0 ? h[j] / den : 1.0;
            sn[j] = den > 0.0 ? h[j + 1] / den : 0.0;
            h[j] = den;
            h[j + 1] = 0.0;
            gv[j + 1] = -sn[j] * gv[j];
            gv[j] = cs[j] * gv[j];
            for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = h[i];
            if (std::fabs(gv[j + 1]) / bnorm <= tol || hn == 0.0) { ++j; ++it; break; }
        }
        // y = R^-1 g ; x += V y
        for (int i = j - 1; i >= 0; --i) {
            double t = gv[i];
            for (int l = i + 1; l < j; ++l) t -= H[(size_t)i * m + l] * y[l];
            y[i] = t / H[(size_t)i * m + i];
        }
        if (j > 0) GM(g.update(j, V, ld, y.data(), 1.0, x));
    }
#undef GM
    if (iters_out) *iters_out = it;
    if (relres_out) *relres_out = relres;
    cleanup();
    SLB_CUDA(cudaStreamSynchronize(s));
    return SLB_OK;
}

extern "C" slb_status slb_mobility_solve(slb_operator* mob, slb_operator* sl, const double* force_torque,
                                         double* rigid_out, double* sigma, int restart, int max_iters, double tol,
                                         int* iters_out, double* relres_out, cudaStream_t s) {
    SLB_REQUIRE(mob && sl && force_torque && rigid_out && sigma, SLB_ERR_INVALID_ARG, "null argument");
    const int64_t nb = mob->d.n_bodies_local;
    SLB_REQUIRE(!far_scalar(mob->kind) && nb > 0 && mob->bodyc, SLB_ERR_INVALID_ARG,
                "mob must be a Stokes operator with the rigid-motion projector");
    SLB_REQUIRE(!far_scalar(sl->kind) && sl->d.n_bodies_local == 0 && sl->N_loc == mob->N_loc &&
                    sl->d.n_trg_local == mob->d.n_trg_local,
                SLB_ERR_INVALID_ARG, "sl must be a Stokes operator (no projector) on the same nodes and targets");
    const int64_t n = mob->N_loc * 3;
    double *ft = nullptr, *nu = nullptr, *rhs = nullptr;
    slb_status st = SLB_OK;
    auto cleanup = [&]() { cudaFreeAsync(ft, s); cudaFreeAsync(nu, s); cudaFreeAsync(rhs, s); };
#define MS(expr) do { st = (expr); if (st != SLB_OK) { cleanup(); return st; } } while (0)
    SLB_CUDA(cudaMallocAsync(&ft, sizeof(double) * nb * 6, s));
    SLB_CUDA(cudaMallocAsync(&nu, sizeof(double) * std::max<int64_t>(n, 1), s));
    SLB_CUDA(cudaMallocAsync(&rhs, sizeof(double) * std::max<int64_t>(n, 1), s));
    SLB_CUDA(cudaMemcpyAsync(ft, force_torque, sizeof(double) * nb * 6, cudaMemcpyHostToDevice, s));
    // nu (completion flow), rhs = -S[nu]
    MS(completion_launch(nb, mob->nb0, mob->d.y_coarse, mob->bodyc, ft, nu, mob->max_nodes_body, s));
    MS(slb_matvec(sl, nu, rhs, s));
    Gm g;
    g.op = mob;
    g.s = s;
    g.n = n;
    MS(g.axpby(-1.0, rhs, 0.0, nullptr, rhs));
    // (K(I-L) + L) sigma = -S[nu]
    MS(slb_gmres(mob, rhs, sigma, restart, max_iters, tol, iters_out, relres_out, s));
    // V = -L sigma: rigid coefficients of L sigma per body, negated
    MS(proj_coef_launch(nb, mob->nb0, mob->d.y_coarse, mob->d.w_coarse, mob->bodyc, sigma, mob->coef, s));
    std::vector<double> c(nb * 6);
    SLB_CUDA(cudaMemcpyAsync(c.data(), mob->coef, sizeof(double) * nb * 6, cudaMemcpyDeviceToHost, s));
    SLB_CUDA(cudaStreamSynchronize(s));
    for (int64_t q = 0; q < nb * 6; ++q) rigid_out[q] = -c[q];
#undef MS
    cleanup();
    SLB_CUDA(cudaStreamSynchronize(s));
    return SLB_OK;
}
