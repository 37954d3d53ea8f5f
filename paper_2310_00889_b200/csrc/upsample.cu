// upsample.cu -- (a) density upsampling, coarse Nystrom grid -> fine smooth-quadrature grid.
//
// Per panel and component: Sigma_f = P_s Sigma_c F_th^T  (separable; P_s: barycentric
// Lagrange in s, F_th: trigonometric interpolation in theta; §3.1).
// Both contractions are dense GEMMs over stacked panels and run on the FP64 tensor cores
// (DMMA, mma.sync.aligned.m8n8k4.f64 -- tcgen05 has no f64 kind on sm_100a):
//   step 1:  T1[(i,c)][b] = sum_j Sigma[i][j][c] F[b][j]       M = N_s*ncomp, K = N_th, N = M_th
//   step 2:  O[a][(b,c)]  = sum_i P_s[a][i] T1[(i,c)][b]       M = M_s,       K = N_s,  N = M_th*ncomp
// One warp per panel; P_s and F_th (zero-padded to multiples of 8/4) live in shared memory,
// staged from the __grid_constant__ parameter once per CTA.  The epilogue either writes the
// plain fine density or packs the far-field source records directly (fused: g = e w sigma_f
// for Stokes, w sigma_f n/(4 pi) for Laplace), so sigma_f never round-trips through HBM.
// HBM-bound (AI ~3.4 flop/B separable); << 1% of the apply.
#include <algorithm>
#include "common.cuh"

namespace slb {

constexpr int kUpWarps = 4;

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ int rup(int v, int m) { return (v + m - 1) / m * m; }

// shared layout (doubles):
//   Ps  [msp][nsp]           (zero padded; msp = rup(ms,8), nsp = rup(ns,4))
//   F   [mtp][ntp]           (mtp = rup(mt,8), ntp = rup(nt,4))
//   per warp: sig [rowsp][ntp]  rows (i,c) padded to rup(ns*nc, 8)
//             T1  [nsp][mtp*nc] laid out as T1[i][(b,c)] (rows i padded to nsp, zero)
__global__ void __launch_bounds__(kUpWarps * 32)
upsample_dmma_kernel(int kind, int nc, int64_t n_panels, const __grid_constant__ InterpParams ip,
                     const double* __restrict__ sc_in, double* __restrict__ sf_out,
                     const double* __restrict__ scale, double* __restrict__ dyn) {
    extern __shared__ double sm[];
    const int ns = ip.ns, nt = ip.nt, ms = ip.ms, mt = ip.mt;
    const int nsp = rup(ns, 4), ntp = rup(nt, 4), msp = rup(ms, 8), mtp = rup(mt, 8);
    const int rows = ns * nc, rowsp = rup(rows, 8);
    const int ncol2 = mt * nc, ncol2p = rup(ncol2, 8);
    double* Ps = sm;                          // [msp][nsp]
    double* F = Ps + msp * nsp;               // [mtp][ntp]
    double* wbase = F + mtp * ntp;
    const int per_warp = rowsp * ntp + nsp * ncol2p;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* sig = wbase + warp * per_warp;    // [rowsp][ntp]
    double* T1 = sig + rowsp * ntp;           // [nsp][ncol2p]
    for (int q = threadIdx.x; q < msp * nsp; q += blockDim.x) {
        const int a = q / nsp, i = q % nsp;
        Ps[q] = (a < ms && i < ns) ? ip.v[a * ns + i] : 0.0;
    }
    for (int q = threadIdx.x; q < mtp * ntp; q += blockDim.x) {
        const int b = q / ntp, j = q % ntp;
        F[q] = (b < mt && j < nt) ? ip.v[ms * ns + b * nt + j] : 0.0;
    }
    __syncthreads();
    const int g = lane >> 2, tq = lane & 3;   // fragment coordinates
    const int nin = ns * nt * nc;
    for (int64_t p = (int64_t)blockIdx.x * kUpWarps + warp; p < n_panels; p += (int64_t)gridDim.x * kUpWarps) {
        // stage the panel's coarse density as sig[(i,c)][j] (zero padded)
        const double* src = sc_in + p * nin;
        for (int q = lane; q < rowsp * ntp; q += 32) sig[q] = 0.0;
        __syncwarp();
        for (int q = lane; q < nin; q += 32) {
            const int c = q % nc, j = (q / nc) % nt, i = q / (nc * nt);
            sig[(i * nc + c) * ntp + j] = src[q];
        }
        for (int q = lane; q < nsp * ncol2p; q += 32) T1[q] = 0.0;
        __syncwarp();
        // step 1: T1[(i,c)][b] = sum_j sig[(i,c)][j] F[b][j]
        for (int r0 = 0; r0 < rowsp; r0 += 8)
            for (int n0 = 0; n0 < mtp; n0 += 8) {
                double d0 = 0.0, d1 = 0.0;
                for (int k0 = 0; k0 < ntp; k0 += 4)
                    dmma_8x8x4(d0, d1, sig[(r0 + g) * ntp + k0 + tq], F[(n0 + g) * ntp + k0 + tq]);
                const int r = r0 + g;
                if (r < rows) {
                    const int i = r / nc, c = r % nc;
                    const int b0 = n0 + 2 * tq;
                    if (b0 < mt) T1[i * ncol2p + b0 * nc + c] = d0;
                    if (b0 + 1 < mt) T1[i * ncol2p + (b0 + 1) * nc + c] = d1;
                }
            }
        __syncwarp();
        // step 2: O[a][(b,c)] = sum_i Ps[a][i] T1[i][(b,c)]  + epilogue
        for (int a0 = 0; a0 < msp; a0 += 8)
            for (int n0 = 0; n0 < ncol2p; n0 += 8) {
                double d0 = 0.0, d1 = 0.0;
                for (int k0 = 0; k0 < nsp; k0 += 4)
                    dmma_8x8x4(d0, d1, Ps[(a0 + g) * nsp + k0 + tq], T1[(k0 + tq) * ncol2p + n0 + g]);
                const int a = a0 + g;
                if (a >= ms) continue;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = n0 + 2 * tq + h;
                    if (col >= ncol2) continue;
                    const int b = col / nc, c = col % nc;
                    const int64_t m = p * (int64_t)(ms * mt) + a * mt + b;
                    const double v = h ? d1 : d0;
                    if (dyn) {
                        if (kind == FAR_LAPLACE) {
                            dyn[m * 4] = scale[3 * m] * v;
                            dyn[m * 4 + 1] = scale[3 * m + 1] * v;
                            dyn[m * 4 + 2] = scale[3 * m + 2] * v;
                        } else {
                            dyn[m * 4 + c] = scale[m] * v;
                        }
                    } else {
                        sf_out[m * nc + c] = v;
                    }
                }
            }
        __syncwarp();
    }
}

slb_status upsample_launch(FarKind kind, int64_t n_panels, const InterpParams& ip, int nc,
                           const double* sigma_coarse, double* sigma_fine, const double* sc,
                           double* dyn, cudaStream_t s) {
    if (n_panels <= 0) return SLB_OK;
    auto rup_h = [](int v, int m) { return (v + m - 1) / m * m; };
    const int nsp = rup_h(ip.ns, 4), ntp = rup_h(ip.nt, 4), msp = rup_h(ip.ms, 8), mtp = rup_h(ip.mt, 8);
    const int rowsp = rup_h(ip.ns * nc, 8), ncol2p = rup_h(ip.mt * nc, 8);
    const size_t smem = sizeof(double) * ((size_t)msp * nsp + (size_t)mtp * ntp +
                                          (size_t)kUpWarps * (rowsp * ntp + nsp * ncol2p));
    SLB_REQUIRE(smem <= 227 * 1024, SLB_ERR_UNSUPPORTED, "upsample: grid too large for shared memory");
    static size_t smem_set = 0;
    if (smem > 48 * 1024 && smem > smem_set) {
        SLB_CUDA(cudaFuncSetAttribute(upsample_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set = smem;
    }
    const int64_t want = (n_panels + kUpWarps - 1) / kUpWarps;
    const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)num_sms() * 8);
    upsample_dmma_kernel<<<grid, kUpWarps * 32, smem, s>>>((int)kind, nc, n_panels, ip, sigma_coarse, sigma_fine, sc,
                                                           dyn);
    ++g_launch_count;
    return check_launch("upsample_dmma_kernel");
}

}  // namespace slb
