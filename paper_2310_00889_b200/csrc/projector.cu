// projector.cu -- (a0) rigid-motion projector of the mobility operator (K(I - L) + L).
//
// PAPER.md Eq. L: L = sum_i v_i v_i^T, {v_i} an L2(dOmega)-orthonormal basis
// of the rigid motions v + omega x (x - x_b^c) on each body.  The orthogonal projector is
// unique, so instead of Gram-Schmidt (the oracle's route) it is evaluated in closed form
// (R12): with the w-centroid c_b, area A_b, inertia I_b = sum w (|d|^2 I - d d^T),
//   F_b = sum w sigma,  T_b = sum w d x sigma,  (L sigma)(y) = F_b / A_b + (I_b^-1 T_b) x (y - c_b).
// Per body: one CTA, fixed-order (strided + tree) reductions -> deterministic.
#include "common.cuh"

namespace slb {

template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double* red) {
    // red: [blockDim.x][NV]; result valid in thread 0
    const int tid = threadIdx.x;
#pragma unroll
    for (int q = 0; q < NV; ++q) red[tid * NV + q] = v[q];
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s)
#pragma unroll
            for (int q = 0; q < NV; ++q) red[tid * NV + q] += red[(tid + s) * NV + q];
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = red[q];
    __syncthreads();
}

// mom[b] = {A, c(3), I(6: xx xy xz yy yz zz)} ; two passes (centroid, then inertia)
__global__ void __launch_bounds__(256)
body_moments_kernel(const int64_t* __restrict__ nb0, const double* __restrict__ y,
                    const double* __restrict__ w, double* __restrict__ mom) {
    __shared__ double red[256 * 6];
    const int64_t b = blockIdx.x;
    const int64_t i0 = nb0[b], i1 = nb0[b + 1];
    double a[4] = {0, 0, 0, 0};
    for (int64_t q = i0 + threadIdx.x; q < i1; q += blockDim.x) {
        double ww = w[q];
        a[0] += ww; a[1] += ww * y[3 * q]; a[2] += ww * y[3 * q + 1]; a[3] += ww * y[3 * q + 2];
    }
    block_reduce<4>(a, red);
    const double A = a[0], c0 = a[1] / A, c1 = a[2] / A, c2 = a[3] / A;
    double I[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t q = i0 + threadIdx.x; q < i1; q += blockDim.x) {
        double ww = w[q];
        double d0 = y[3 * q] - c0, d1 = y[3 * q + 1] - c1, d2 = y[3 * q + 2] - c2;
        double dd = d0 * d0 + d1 * d1 + d2 * d2;
        I[0] += ww * (dd - d0 * d0); I[1] -= ww * d0 * d1; I[2] -= ww * d0 * d2;
        I[3] += ww * (dd - d1 * d1); I[4] -= ww * d1 * d2; I[5] += ww * (dd - d2 * d2);
    }
    block_reduce<6>(I, red);
    if (threadIdx.x == 0) {
        double* o = mom + b * 16;
        o[0] = A; o[1] = c0; o[2] = c1; o[3] = c2;
        for (int q = 0; q < 6; ++q) o[4 + q] = I[q];
    }
}

// bodyc[b] = {A, c(3), Iinv(9 row-major), pad(3)}
__global__ void __launch_bounds__(256)
proj_coef_kernel(const int64_t* __restrict__ nb0, const double* __restrict__ y,
                 const double* __restrict__ w, const double* __restrict__ bodyc,
                 const double* __restrict__ sigma, double* __restrict__ coef) {
    __shared__ double red[256 * 6];
    const int64_t b = blockIdx.x;
    const int64_t i0 = nb0[b], i1 = nb0[b + 1];
    const double* bc = bodyc + b * 16;
    const double c0 = bc[1], c1 = bc[2], c2 = bc[3];
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t q = i0 + threadIdx.x; q < i1; q += blockDim.x) {
        double ww = w[q];
        double s0 = sigma[3 * q], s1 = sigma[3 * q + 1], s2 = sigma[3 * q + 2];
        double d0 = y[3 * q] - c0, d1 = y[3 * q + 1] - c1, d2 = y[3 * q + 2] - c2;
        v[0] += ww * s0; v[1] += ww * s1; v[2] += ww * s2;
        v[3] += ww * (d1 * s2 - d2 * s1); v[4] += ww * (d2 * s0 - d0 * s2); v[5] += ww * (d0 * s1 - d1 * s0);
    }
    block_reduce<6>(v, red);
    if (threadIdx.x == 0) {
        const double A = bc[0];
        const double* Ii = bc + 4;
        double* o = coef + b * 6;
        o[0] = v[0] / A; o[1] = v[1] / A; o[2] = v[2] / A;
        for (int r = 0; r < 3; ++r) o[3 + r] = Ii[3 * r] * v[3] + Ii[3 * r + 1] * v[4] + Ii[3 * r + 2] * v[5];
    }
}

// L sigma = F/A + Omega x (y - c);  sigma' = sigma - L sigma
__global__ void __launch_bounds__(256)
proj_apply_kernel(const int64_t* __restrict__ nb0, const double* __restrict__ y,
                  const double* __restrict__ bodyc, const double* __restrict__ coef,
                  const double* __restrict__ sigma, double* __restrict__ sigma_p, double* __restrict__ Lsig) {
    const int64_t b = blockIdx.y;
    const int64_t q = nb0[b] + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nb0[b + 1]) return;
    const double* bc = bodyc + b * 16;
    const double* o = coef + b * 6;
    double d0 = y[3 * q] - bc[1], d1 = y[3 * q + 1] - bc[2], d2 = y[3 * q + 2] - bc[3];
    double l0 = o[0] + (o[4] * d2 - o[5] * d1);
    double l1 = o[1] + (o[5] * d0 - o[3] * d2);
    double l2 = o[2] + (o[3] * d1 - o[4] * d0);
    Lsig[3 * q] = l0; Lsig[3 * q + 1] = l1; Lsig[3 * q + 2] = l2;
    sigma_p[3 * q] = sigma[3 * q] - l0;
    sigma_p[3 * q + 1] = sigma[3 * q + 1] - l1;
    sigma_p[3 * q + 2] = sigma[3 * q + 2] - l2;
}

// completion-flow density nu = alpha + beta x (y - c) with int nu = F, int nu x (y - c) = T
// (P:L1903-1912).  c = w-centroid, so int (y - c) = 0:  alpha = F / A,  beta = -I^-1 T  (I as above).
__global__ void __launch_bounds__(256)
completion_kernel(const int64_t* __restrict__ nb0, const double* __restrict__ y, const double* __restrict__ bodyc,
                  const double* __restrict__ ft, double* __restrict__ nu) {
    const int64_t b = blockIdx.y;
    const int64_t q = nb0[b] + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nb0[b + 1]) return;
    const double* bc = bodyc + b * 16;
    const double* f = ft + b * 6;
    const double* Ii = bc + 4;
    const double A = bc[0];
    double be[3];
    for (int r = 0; r < 3; ++r) be[r] = -(Ii[3 * r] * f[3] + Ii[3 * r + 1] * f[4] + Ii[3 * r + 2] * f[5]);
    const double d0 = y[3 * q] - bc[1], d1 = y[3 * q + 1] - bc[2], d2 = y[3 * q + 2] - bc[3];
    nu[3 * q] = f[0] / A + (be[1] * d2 - be[2] * d1);
    nu[3 * q + 1] = f[1] / A + (be[2] * d0 - be[0] * d2);
    nu[3 * q + 2] = f[2] / A + (be[0] * d1 - be[1] * d0);
}

slb_status completion_launch(int64_t n_bodies, const int64_t* nb0, const double* y, const double* bodyc,
                             const double* ft, double* nu, int64_t max_nodes_per_body, cudaStream_t s) {
    if (n_bodies <= 0) return SLB_OK;
    dim3 grid((unsigned)((max_nodes_per_body + 255) / 256), (unsigned)n_bodies);
    completion_kernel<<<grid, 256, 0, s>>>(nb0, y, bodyc, ft, nu);
    ++g_launch_count;
    return check_launch("completion_kernel");
}

slb_status proj_coef_launch(int64_t n_bodies, const int64_t* nb0, const double* y, const double* w,
                            const double* bodyc, const double* sigma, double* coef, cudaStream_t s) {
    if (n_bodies <= 0) return SLB_OK;
    proj_coef_kernel<<<(unsigned)n_bodies, 256, 0, s>>>(nb0, y, w, bodyc, sigma, coef);
    ++g_launch_count;
    return check_launch("proj_coef_kernel");
}

slb_status body_moments_launch(int64_t n_bodies, const int64_t* nb0, const double* y, const double* w,
                               double* mom, cudaStream_t s) {
    if (n_bodies <= 0) return SLB_OK;
    body_moments_kernel<<<(unsigned)n_bodies, 256, 0, s>>>(nb0, y, w, mom);
    ++g_launch_count;
    return check_launch("body_moments_kernel");
}

slb_status proj_launch(int64_t n_bodies, const int64_t* nb0, const double* y, const double* w,
                       const double* bodyc, const double* sigma, double* coef, double* sigma_p,
                       double* Lsig, int64_t max_nodes_per_body, cudaStream_t s) {
    if (n_bodies <= 0) return SLB_OK;
    proj_coef_kernel<<<(unsigned)n_bodies, 256, 0, s>>>(nb0, y, w, bodyc, sigma, coef);
    ++g_launch_count;
    slb_status st = check_launch("proj_coef_kernel");
    if (st != SLB_OK) return st;
    dim3 grid((unsigned)((max_nodes_per_body + 255) / 256), (unsigned)n_bodies);
    proj_apply_kernel<<<grid, 256, 0, s>>>(nb0, y, bodyc, coef, sigma, sigma_p, Lsig);
    ++g_launch_count;
    return check_launch("proj_apply_kernel");
}

}  // namespace slb
