// upsample.cu -- (a) density upsampling, coarse Nystrom grid -> fine smooth-quadrature grid.
//
// Per panel and component: Sigma_f = P_s Sigma_c F_th^T  (separable; P_s: barycentric
// Lagrange in s, F_th: trigonometric interpolation in theta; §3.1).
// One CTA per panel; the panel's coarse density and the theta-contracted intermediate live in
// shared memory; P_s and F_th arrive as a __grid_constant__ kernel parameter.  When `dyn` is
// given, the epilogue writes the far-field source records directly (fused packing:
// g = e w sigma_f for Stokes, w sigma_f n/(4 pi) for Laplace), so the upsampled density never
// makes a separate round trip through HBM.  HBM-bound (AI ~3.4 flop/B); << 1% of the apply.
#include "common.cuh"

namespace slb {

__global__ void __launch_bounds__(128)
upsample_kernel(int kind, int nc, const __grid_constant__ InterpParams ip,
                const double* __restrict__ sc_in, double* __restrict__ sf_out,
                const double* __restrict__ scale, double* __restrict__ dyn) {
    extern __shared__ double sm[];
    const int ns = ip.ns, nt = ip.nt, ms = ip.ms, mt = ip.mt;
    const double* Ps = ip.v;             // [ms][ns]
    const double* F = ip.v + ms * ns;    // [mt][nt]
    const int64_t p = blockIdx.x;
    const int nin = ns * nt * nc;
    double* s_in = sm;                   // [ns][nt][nc]
    double* s_mid = sm + nin;            // [ns][mt][nc]
    const double* src = sc_in + p * nin;
    for (int q = threadIdx.x; q < nin; q += blockDim.x) s_in[q] = src[q];
    __syncthreads();
    // theta contraction: mid[i][b][c] = sum_j F[b][j] in[i][j][c]
    const int nmid = ns * mt * nc;
    for (int q = threadIdx.x; q < nmid; q += blockDim.x) {
        int c = q % nc, b = (q / nc) % mt, i = q / (nc * mt);
        double acc = 0.0;
        for (int j = 0; j < nt; ++j) acc = fma(F[b * nt + j], s_in[(i * nt + j) * nc + c], acc);
        s_mid[q] = acc;
    }
    __syncthreads();
    // s contraction + epilogue: out[a][b][c] = sum_i Ps[a][i] mid[i][b][c]
    const int nnode = ms * mt;
    for (int q = threadIdx.x; q < nnode; q += blockDim.x) {
        int a = q / mt, b = q % mt;
        double o[3] = {0.0, 0.0, 0.0};
        for (int i = 0; i < ns; ++i) {
            double pa = Ps[a * ns + i];
            for (int c = 0; c < nc; ++c) o[c] = fma(pa, s_mid[(i * mt + b) * nc + c], o[c]);
        }
        int64_t m = p * nnode + q;
        if (dyn) {
            double4 r;
            if (kind == FAR_LAPLACE) {
                r = make_double4(scale[3 * m] * o[0], scale[3 * m + 1] * o[0], scale[3 * m + 2] * o[0], 0.0);
            } else {
                double f = scale[m];
                r = make_double4(f * o[0], f * o[1], f * o[2], 0.0);
            }
            reinterpret_cast<double4*>(dyn)[m] = r;
        } else {
            for (int c = 0; c < nc; ++c) sf_out[m * nc + c] = o[c];
        }
    }
}

slb_status upsample_launch(FarKind kind, int64_t n_panels, const InterpParams& ip, int nc,
                           const double* sigma_coarse, double* sigma_fine, const double* sc,
                           double* dyn, cudaStream_t s) {
    if (n_panels <= 0) return SLB_OK;
    SLB_REQUIRE(n_panels <= 2147483647LL, SLB_ERR_UNSUPPORTED, "too many panels");
    size_t smem = sizeof(double) * (size_t)(ip.ns * ip.nt * nc + ip.ns * ip.mt * nc);
    static size_t smem_set = 0;
    if (smem > 48 * 1024 && smem > smem_set) {
        SLB_CUDA(cudaFuncSetAttribute(upsample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set = smem;
    }
    upsample_kernel<<<(unsigned)n_panels, 128, smem, s>>>((int)kind, nc, ip, sigma_coarse, sigma_fine, sc, dyn);
    ++g_launch_count;
    return check_launch("upsample_kernel");
}

}  // namespace slb
