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
#include <cstdlib>
#include "common.cuh"

namespace slb {

constexpr int kUpWarps = 4;

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ int rup(int v, int m) { return (v + m - 1) / m * m; }
// shared-memory leading dimensions (doubles) that keep the DMMA fragment loads <= 2-way bank
// conflicted: rows indexed by the fragment's g (8 rows) want ld = 4 or 12 (mod 16); rows indexed by
// tq (4 rows, 8 consecutive g) want ld = 8 (mod 16)
__host__ __device__ __forceinline__ int ld_g(int x) { return (x % 16 == 0 || x % 16 == 8) ? x + 4 : x; }
__host__ __device__ __forceinline__ int ld_t(int x) { return (x % 16 == 0) ? x + 8 : x; }

// shared layout (doubles), one panel per CTA at a time:
//   Ps  [msp][ldp]           (zero padded; msp = rup(ms,8), nsp = rup(ns,4), ldp >= nsp)
//   F   [mtp][ldf]           (mtp = rup(mt,8), ntp = rup(nt,4), ldf >= ntp)
//   raw [ns][nt][nc]         the panel's coarse density as stored (A operand of step 1 read in place)
//   T1  [nsp][ld1]           T1[i][(b,c)] (rows i padded to nsp, zero)
//   O   [ms][mt][nc]         step-2 result, written to HBM as whole 32-byte records
// The CTA's warps split the 8x8 output tiles of both steps (a panel is 39 tiles at 10x12 -> 20x24,
// 224 at 12x64 -> 24x128), so large panels are not serialised on one warp.
// Ragged panels (NEXT N4): the launch covers the n_panels panels plist[0..n_panels) (NULL: 0..n-1)
// of one (nt, mt) bucket; c_off / f_off give each panel's first coarse / fine node (NULL: uniform).
__global__ void __launch_bounds__(kUpWarps * 32)
upsample_dmma_kernel(int kind, int nc, int64_t n_panels, const __grid_constant__ InterpParams ip,
                     const double* __restrict__ sc_in, double* __restrict__ sf_out,
                     const double* __restrict__ scale, double* __restrict__ dyn,
                     const int32_t* __restrict__ plist, const int64_t* __restrict__ c_off,
                     const int64_t* __restrict__ f_off, int orows, int gmats) {
    // orows: output rows (a) staged in O at a time (msp, or fewer multiples of 8 for very large grids);
    // gmats: read P_s and F_th from the (L1-cached) global copy instead of shared memory (largest grids)
    extern __shared__ double sm[];
    const int ns = ip.ns, nt = ip.nt, ms = ip.ms, mt = ip.mt;
    const int nsp = rup(ns, 4), ntp = rup(nt, 4), msp = rup(ms, 8), mtp = rup(mt, 8);
    const int rows = ns * nc, rowsp = rup(rows, 8);
    const int ncol2 = mt * nc, ncol2p = rup(ncol2, 8);
    const int ldp = ld_g(nsp), ldf = ld_g(ntp), ld1 = ld_t(ncol2p);
    const int nin = ns * nt * nc;
    const int nout = ms * mt;
    double* Ps = sm;                          // [msp][ldp]   (absent when gmats)
    double* F = Ps + (gmats ? 0 : msp * ldp); // [mtp][ldf]   (absent when gmats)
    double* raw = F + (gmats ? 0 : mtp * ldf);// [ns][nt][nc] (rup to 2)
    double* T1 = raw + ((nin + 1) & ~1);      // [nsp][ld1]
    double* O = T1 + nsp * ld1;               // [orows][mt][nc]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const double* V = ip.vg ? ip.vg : ip.v;
    if (!gmats) {
        for (int q = threadIdx.x; q < msp * ldp; q += blockDim.x) {
            const int a = q / ldp, i = q % ldp;
            Ps[q] = (a < ms && i < ns) ? V[a * ns + i] : 0.0;
        }
        for (int q = threadIdx.x; q < mtp * ldf; q += blockDim.x) {
            const int b = q / ldf, j = q % ldf;
            F[q] = (b < mt && j < nt) ? V[ms * ns + b * nt + j] : 0.0;
        }
    }
    // fragment loaders: F[b][j] and Ps[a][i], zero outside the matrices
    auto Fv = [&](int b, int j) -> double {
        return gmats ? ((b < mt && j < nt) ? __ldg(V + ms * ns + b * nt + j) : 0.0) : F[b * ldf + j];
    };
    auto Pv = [&](int a, int i) -> double {
        return gmats ? ((a < ms && i < ns) ? __ldg(V + a * ns + i) : 0.0) : Ps[a * ldp + i];
    };
    const int g = lane >> 2, tq = lane & 3;   // fragment coordinates
    const int nt1 = (rowsp / 8) * (mtp / 8);  // step-1 tiles
    const int nt2 = (msp / 8) * (ncol2p / 8); // step-2 tiles
    for (int64_t pl = blockIdx.x; pl < n_panels; pl += gridDim.x) {
        const int64_t p = plist ? (int64_t)plist[pl] : pl;
        const int64_t m0 = f_off ? f_off[p] : p * (int64_t)nout;
        // stage the panel's coarse density unchanged (contiguous, coalesced)
        const double* src = sc_in + (c_off ? c_off[p] * nc : p * nin);
        __syncthreads();                      // previous panel's O fully written out; Ps/F staged
        for (int q = threadIdx.x; q < nin; q += blockDim.x) raw[q] = __ldg(src + q);
        for (int q = threadIdx.x; q < nsp * ld1; q += blockDim.x) T1[q] = 0.0;
        __syncthreads();
        // step 1: T1[(i,c)][b] = sum_j sigma[i][j][c] F[b][j]   (A fragment read in place from raw)
        for (int tile = warp; tile < nt1; tile += nwarps) {
            const int r0 = (tile / (mtp / 8)) * 8, n0 = (tile % (mtp / 8)) * 8;
            const int r = r0 + g;
            const int rb = (r < rows) ? (r / nc) * nt * nc + (r % nc) : -1;   // raw index of (i, j = 0, c)
            double d0 = 0.0, d1 = 0.0;
            for (int k0 = 0; k0 < ntp; k0 += 4) {
                const int j = k0 + tq;
                const double av = (rb >= 0 && j < nt) ? raw[rb + j * nc] : 0.0;
                dmma_8x8x4(d0, d1, av, Fv(n0 + g, k0 + tq));
            }
            if (r < rows) {
                const int i = r / nc, c = r % nc;
                const int b0 = n0 + 2 * tq;
                if (b0 < mt) T1[i * ld1 + b0 * nc + c] = d0;
                if (b0 + 1 < mt) T1[i * ld1 + (b0 + 1) * nc + c] = d1;
            }
        }
        __syncthreads();
        // step 2: O[a][(b,c)] = sum_i Ps[a][i] T1[i][(b,c)], orows output rows at a time
        for (int ac = 0; ac < msp; ac += orows) {
            const int ntc = (min(orows, msp - ac) / 8) * (ncol2p / 8);
            for (int tile = warp; tile < ntc; tile += nwarps) {
                const int a0 = ac + (tile / (ncol2p / 8)) * 8, n0 = (tile % (ncol2p / 8)) * 8;
                double d0 = 0.0, d1 = 0.0;
                for (int k0 = 0; k0 < nsp; k0 += 4)
                    dmma_8x8x4(d0, d1, Pv(a0 + g, k0 + tq), T1[(k0 + tq) * ld1 + n0 + g]);
                const int a = a0 + g;
                if (a >= ms) continue;
                const int col = n0 + 2 * tq;
                if (col < ncol2) O[(a - ac) * ncol2 + col] = d0;
                if (col + 1 < ncol2) O[(a - ac) * ncol2 + col + 1] = d1;
            }
            __syncthreads();
            // epilogue: whole 32-byte source records {g, 0} per fine node (coalesced), or the plain values
            const int e0 = ac * mt, e1 = min(ac + orows, ms) * mt;
            if (dyn) {
                double2* D2 = reinterpret_cast<double2*>(dyn);
                for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
                    const int64_t m = m0 + e;
                    const int eo = e - e0;
                    double v0, v1, v2, v3 = 0.0;
                    if (far_scalar(kind)) {
                        const double v = O[eo];
                        v0 = scale[4 * m] * v; v1 = scale[4 * m + 1] * v; v2 = scale[4 * m + 2] * v;
                        v3 = scale[4 * m + 3] * v;
                    } else {
                        const double sc = scale[m];
                        v0 = sc * O[3 * eo]; v1 = sc * O[3 * eo + 1]; v2 = sc * O[3 * eo + 2];
                    }
                    D2[2 * m] = make_double2(v0, v1);
                    D2[2 * m + 1] = make_double2(v2, v3);
                }
            } else {
                for (int e = e0 * nc + threadIdx.x; e < e1 * nc; e += blockDim.x) sf_out[m0 * nc + e] = O[e - e0 * nc];
            }
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------------------------------------
// upsample_warp_kernel: the streaming form (round 2).  One WARP per panel, no CTA barriers in the
// panel loop; each warp double-buffers its panels: lane 0 issues TMA bulk copies (cp.async.bulk +
// mbarrier complete_tx) of the NEXT panel's coarse density and fine-node scales while the warp
// contracts the current one, so HBM latency is hidden behind the DMMA work.
//   step 1 (rows (i,c) stacked):  T1_c[i][b] = sum_j sigma[i][j][c] F[b][j]     M = N_s nc, K = N_th, N = M_th
//   step 2 (per c, shared A):     O_c[a][b]  = sum_i P_s[a][i] T1_c[i][b]        M = M_s,   K = N_s,  N = M_th
// Step 2 keeps the nc components of one output tile in registers, so a lane holds ALL components of
// two adjacent fine nodes (a0+g, b0+2tq..+1) and writes their 32-byte source records straight from
// the accumulators (8 rows x 256 contiguous bytes per warp store) -- no output staging in shared
// memory.  Optionally the staged coarse density is also written to `copy_out` (the global coarse
// buffer of a sharded operator), fusing the copy into the read.  P_s and F_th are staged per CTA
// from a global copy (coalesced), never from the kernel-parameter bank.
constexpr int kUpW = 8;   // warps per CTA (upper bound; fewer when the per-warp buffers are large)

struct UpWarpLayout {
    int nsp, ntp, msp, mtp, rows8, ldp, ldf, ldt;
    int nin2, nout, scl;       // doubles: coarse panel (even), fine nodes, scale doubles per node
    size_t cta_d, warp_d;      // doubles: per-CTA matrices, per-warp buffers
};

__host__ __device__ inline UpWarpLayout up_layout(int ns, int nt, int ms, int mt, int nc, int scl) {
    UpWarpLayout L;
    L.nsp = (ns + 3) / 4 * 4;
    L.ntp = (nt + 3) / 4 * 4;
    L.msp = (ms + 7) / 8 * 8;
    L.mtp = (mt + 7) / 8 * 8;
    L.rows8 = (ns * nc + 7) / 8 * 8;
    L.ldp = ld_g(L.nsp);
    L.ldf = ld_g(L.ntp);
    L.ldt = ld_t(L.mtp);
    L.nin2 = (ns * nt * nc + 1) & ~1;
    L.nout = ms * mt;
    L.scl = scl;
    L.cta_d = (size_t)L.msp * L.ldp + (size_t)L.mtp * L.ldf;
    // raw[2][nin2] + scale[2][nout*scl] + T1[nc][nsp][ldt]
    L.warp_d = 2 * (size_t)L.nin2 + 2 * (size_t)L.nout * scl + (size_t)nc * L.nsp * L.ldt;
    return L;
}

template <int NC>
__global__ void __launch_bounds__(kUpW * 32)
upsample_warp_kernel(int kind, int64_t n_panels, int ns, int nt, int ms, int mt, const double* __restrict__ mats,
                     const double* __restrict__ sc_in, double* __restrict__ sf_out,
                     const double* __restrict__ scale, double* __restrict__ dyn, double* __restrict__ copy_out,
                     const int32_t* __restrict__ plist, const int64_t* __restrict__ c_off,
                     const int64_t* __restrict__ f_off, double* __restrict__ dyn_mc) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bars[kUpW * 2];
    const int scl = scale ? (far_scalar(kind) ? 4 : 1) : 0;
    const UpWarpLayout L = up_layout(ns, nt, ms, mt, NC, scl);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double* Ps = sm;                                   // [msp][ldp]
    double* F = Ps + L.msp * L.ldp;                    // [mtp][ldf]
    double* wb = sm + L.cta_d + (size_t)warp * L.warp_d;
    double* raw = wb;                                  // [2][nin2]
    double* scs = raw + 2 * L.nin2;                    // [2][nout*scl]
    double* T1 = scs + 2 * (size_t)L.nout * scl;       // [NC][nsp][ldt]
    uint64_t* bar = bars + 2 * warp;
    for (int q = threadIdx.x; q < L.msp * L.ldp; q += blockDim.x) {
        const int a = q / L.ldp, i = q % L.ldp;
        Ps[q] = (a < ms && i < ns) ? mats[a * ns + i] : 0.0;
    }
    for (int q = threadIdx.x; q < L.mtp * L.ldf; q += blockDim.x) {
        const int b = q / L.ldf, j = q % L.ldf;
        F[q] = (b < mt && j < nt) ? mats[ms * ns + b * nt + j] : 0.0;
    }
    for (int q = lane; q < NC * L.nsp * L.ldt; q += 32) T1[q] = 0.0;   // K padding rows stay zero
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int nin = ns * nt * NC;
    const int64_t gw = (int64_t)blockIdx.x * nw + warp, stride = (int64_t)gridDim.x * nw;
    auto issue = [&](int64_t pl, int buf) {            // lane 0: TMA the panel's inputs into buffer buf
        const int64_t p = plist ? (int64_t)plist[pl] : pl;
        const int64_t m0 = f_off ? f_off[p] : p * (int64_t)L.nout;
        const double* src = sc_in + (c_off ? c_off[p] * NC : p * (int64_t)nin);
        const uint32_t b0 = (uint32_t)(nin * 8), b1 = (uint32_t)(L.nout * scl * 8);
        mbar_expect_tx(&bar[buf], b0 + b1);
        bulk_g2s(raw + buf * L.nin2, src, b0, &bar[buf]);
        if (scl) bulk_g2s(scs + (size_t)buf * L.nout * scl, scale + m0 * scl, b1, &bar[buf]);
    };
    if (lane == 0 && gw < n_panels) issue(gw, 0);
    const int g = lane >> 2, tq = lane & 3;
    const int rows = ns * NC;
    int it = 0;
    for (int64_t pl = gw; pl < n_panels; pl += stride, ++it) {
        const int buf = it & 1;
        const int64_t p = plist ? (int64_t)plist[pl] : pl;
        const int64_t m0 = f_off ? f_off[p] : p * (int64_t)L.nout;
        mbar_wait(&bar[buf], (uint32_t)((it >> 1) & 1));
        // the other buffer was consumed by the previous iteration (its last reads are ordered before
        // this __syncwarp): refill it with the next panel
        __syncwarp();
        if (lane == 0 && pl + stride < n_panels) {
            fence_proxy_async_smem();
            issue(pl + stride, buf ^ 1);
        }
        const double* R = raw + buf * L.nin2;
        const double* SC = scs + (size_t)buf * L.nout * scl;
        if (copy_out) {
            double* dst = copy_out + (c_off ? c_off[p] * NC : p * (int64_t)nin);
            for (int q = lane; q < nin; q += 32) dst[q] = R[q];
        }
        // step 1: T1_c[i][b], rows r = i*NC + c
        for (int r0 = 0; r0 < L.rows8; r0 += 8) {
            const int r = r0 + g;
            const int rb = (r < rows) ? (r / NC) * nt * NC + (r % NC) : -1;
            for (int n0 = 0; n0 < L.mtp; n0 += 8) {
                double d0 = 0.0, d1 = 0.0;
                for (int k0 = 0; k0 < L.ntp; k0 += 4) {
                    const int j = k0 + tq;
                    const double av = (rb >= 0 && j < nt) ? R[rb + j * NC] : 0.0;
                    dmma_8x8x4(d0, d1, av, F[(n0 + g) * L.ldf + k0 + tq]);
                }
                if (r < rows) {
                    double* T = T1 + ((r % NC) * L.nsp + r / NC) * L.ldt + n0 + 2 * tq;
                    T[0] = d0;
                    T[1] = d1;
                }
            }
        }
        __syncwarp();
        // step 2 + epilogue
        for (int a0 = 0; a0 < L.msp; a0 += 8) {
            for (int n0 = 0; n0 < L.mtp; n0 += 8) {
                double d0[NC], d1[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) d0[c] = d1[c] = 0.0;
                for (int k0 = 0; k0 < L.nsp; k0 += 4) {
                    const double av = Ps[(a0 + g) * L.ldp + k0 + tq];
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        dmma_8x8x4(d0[c], d1[c], av, T1[(c * L.nsp + k0 + tq) * L.ldt + n0 + g]);
                }
                const int a = a0 + g, b = n0 + 2 * tq;
                if (a >= ms || b >= mt) continue;
                const int e = a * mt + b;                  // node e and e + 1 (b + 1 < mt: mt even)
                const int64_t m = m0 + e;
                if (dyn) {
                    double v[8];
                    if (NC == 1) {
                        const double* s0 = SC + 4 * e;
                        for (int q = 0; q < 4; ++q) { v[q] = s0[q] * d0[0]; v[4 + q] = s0[4 + q] * d1[0]; }
                    } else {
                        const double s0 = SC[e], s1 = SC[e + 1];
                        v[0] = s0 * d0[0]; v[1] = s0 * d0[1]; v[2] = s0 * d0[NC - 1]; v[3] = 0.0;
                        v[4] = s1 * d1[0]; v[5] = s1 * d1[1]; v[6] = s1 * d1[NC - 1]; v[7] = 0.0;
                    }
                    if (dyn_mc) {                      // fused gather (N4): replicated into every rank's copy
                        for (int q = 0; q < 4; ++q) multimem_st2(dyn_mc + 4 * m + 2 * q, v[2 * q], v[2 * q + 1]);
                    } else {
                        double2* D2 = reinterpret_cast<double2*>(dyn) + 2 * m;
                        for (int q = 0; q < 4; ++q) D2[q] = make_double2(v[2 * q], v[2 * q + 1]);
                    }
                } else {
                    double* o = sf_out + m * NC;
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        o[c] = d0[c];
                        o[NC + c] = d1[c];
                    }
                }
            }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------------------------------------
// upsample_rec_kernel<NS, NT, MS, MT>: the Stokes record path (NC = 3, dyn records) with the grid fixed at
// compile time (the benchmark grids: 10x12 -> 20x24 for c4/c5, 10x16 -> 20x32, 12x20 -> 24x40), so every
// DMMA tile loop is unrolled and addressing is constant-folded.  Differences to the generic kernel: the
// fine-node scales are prefetched straight into registers (__ldg, issued before the contraction; no
// shared-memory buffer), which leaves ~12 KB of shared memory per warp and 16 warps per SM; the coarse
// density is still double-buffered by TMA bulk copies.

template <int NS, int NT, int MS, int MT, int WARPS, int ORD>
__global__ void __launch_bounds__(WARPS * 32)
upsample_rec_kernel(int64_t n_panels, const double* __restrict__ mats, const double* __restrict__ sc_in,
                    const double* __restrict__ scale, double* __restrict__ dyn, double* __restrict__ copy_out,
                    const int32_t* __restrict__ plist, const int64_t* __restrict__ c_off,
                    const int64_t* __restrict__ f_off, double* __restrict__ dyn_mc) {
    constexpr int NC = 3;
    constexpr int NSP = (NS + 3) / 4 * 4, NTP = (NT + 3) / 4 * 4, MSP = (MS + 7) / 8 * 8, MTP = (MT + 7) / 8 * 8;
    constexpr int ROWS = NS * NC, ROWS8 = (ROWS + 7) / 8 * 8;
    constexpr int LDP = (NSP % 16 == 0 || NSP % 16 == 8) ? NSP + 4 : NSP;
    constexpr int LDF = (NTP % 16 == 0 || NTP % 16 == 8) ? NTP + 4 : NTP;
    constexpr int LDT = (MTP % 16 == 0) ? MTP + 8 : MTP;
    constexpr int NIN = NS * NT * NC, NIN2 = (NIN + 1) & ~1, NOUT = MS * MT;
    constexpr int WARP_D = 2 * NIN2 + NC * NSP * LDT;
    constexpr int NA = MSP / 8, NB = MTP / 8;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bars[WARPS * 2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double* Ps = sm;                                   // [MSP][LDP]
    double* F = Ps + MSP * LDP;                        // [MTP][LDF]
    double* wb = F + MTP * LDF + (size_t)warp * WARP_D;
    double* raw = wb;                                  // [2][NIN2]
    double* T1 = raw + 2 * NIN2;                       // [NC][NSP][LDT]
    uint64_t* bar = bars + 2 * warp;
    for (int q = threadIdx.x; q < MSP * LDP; q += blockDim.x) {
        const int a = q / LDP, i = q % LDP;
        Ps[q] = (a < MS && i < NS) ? mats[a * NS + i] : 0.0;
    }
    for (int q = threadIdx.x; q < MTP * LDF; q += blockDim.x) {
        const int b = q / LDF, j = q % LDF;
        F[q] = (b < MT && j < NT) ? mats[MS * NS + b * NT + j] : 0.0;
    }
    for (int q = lane; q < NC * NSP * LDT; q += 32) T1[q] = 0.0;
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t gw = (int64_t)blockIdx.x * nw + warp, stride = (int64_t)gridDim.x * nw;
    auto issue = [&](int64_t pl, int buf) {
        const int64_t p = plist ? (int64_t)plist[pl] : pl;
        const double* src = sc_in + (c_off ? c_off[p] * NC : p * (int64_t)NIN);
        mbar_expect_tx(&bar[buf], (uint32_t)(NIN * 8));
        bulk_g2s(raw + buf * NIN2, src, (uint32_t)(NIN * 8), &bar[buf]);
    };
    // both buffers filled up front (a warp typically owns only 2-3 panels: no steady state to hide behind)
    if (lane == 0 && gw < n_panels) issue(gw, 0);
    if (lane == 0 && gw + stride < n_panels) issue(gw + stride, 1);
    const int g = lane >> 2, tq = lane & 3;
    int it = 0;
    for (int64_t pl = gw; pl < n_panels; pl += stride, ++it) {
        const int buf = it & 1;
        const int64_t p = plist ? (int64_t)plist[pl] : pl;
        const int64_t m0 = f_off ? f_off[p] : p * (int64_t)NOUT;
        // this lane's fine-node scales (2 adjacent nodes per output tile), loads in flight during the GEMMs
        double sc0[NA][NB], sc1[NA][NB];
        if (ORD == 0)
#pragma unroll
        for (int ta = 0; ta < NA; ++ta)
#pragma unroll
            for (int tb = 0; tb < NB; ++tb) {
                const int a = ta * 8 + g, b = tb * 8 + 2 * tq;
                if (a < MS && b < MT) {
                    const double2 v = __ldg(reinterpret_cast<const double2*>(scale + m0 + a * MT + b));
                    sc0[ta][tb] = v.x;
                    sc1[ta][tb] = v.y;
                } else {
                    sc0[ta][tb] = sc1[ta][tb] = 0.0;
                }
            }
        mbar_wait(&bar[buf], (uint32_t)((it >> 1) & 1));
        __syncwarp();
        const double* R = raw + buf * NIN2;
        if (copy_out) {
            double* dst = copy_out + (c_off ? c_off[p] * NC : p * (int64_t)NIN);
            for (int q = lane; q < NIN; q += 32) dst[q] = R[q];
        }
        // step 1: T1_c[i][b] = sum_j sigma[i][j][c] F[b][j], rows r = i NC + c
        if constexpr (ORD == 1) {
            // every fragment loaded before the first T1 store (the compiler cannot move shared loads across
            // shared stores it cannot disambiguate): all ROWS8/8 x MTP/8 output tiles are independent DMMA chains
            constexpr int NRT1 = ROWS8 / 8, NK1 = NTP / 4, NN1 = MTP / 8;
            double av[NRT1][NK1], bv[NN1][NK1], d0[NRT1][NN1], d1[NRT1][NN1];
#pragma unroll
            for (int rt = 0; rt < NRT1; ++rt) {
                const int r = rt * 8 + g;
                const int rb = (r < ROWS) ? (r / NC) * NT * NC + (r % NC) : 0;
#pragma unroll
                for (int kk = 0; kk < NK1; ++kk) {
                    const int j = kk * 4 + tq;
                    av[rt][kk] = (r < ROWS && j < NT) ? R[rb + j * NC] : 0.0;
                }
            }
#pragma unroll
            for (int nn = 0; nn < NN1; ++nn)
#pragma unroll
                for (int kk = 0; kk < NK1; ++kk) bv[nn][kk] = F[(nn * 8 + g) * LDF + kk * 4 + tq];
#pragma unroll
            for (int rt = 0; rt < NRT1; ++rt)
#pragma unroll
                for (int nn = 0; nn < NN1; ++nn) d0[rt][nn] = d1[rt][nn] = 0.0;
#pragma unroll
            for (int kk = 0; kk < NK1; ++kk)
#pragma unroll
                for (int rt = 0; rt < NRT1; ++rt)
#pragma unroll
                    for (int nn = 0; nn < NN1; ++nn) dmma_8x8x4(d0[rt][nn], d1[rt][nn], av[rt][kk], bv[nn][kk]);
#pragma unroll
            for (int rt = 0; rt < NRT1; ++rt) {
                const int r = rt * 8 + g;
                if (r < ROWS) {
#pragma unroll
                    for (int nn = 0; nn < NN1; ++nn) {
                        double* T = T1 + ((r % NC) * NSP + r / NC) * LDT + nn * 8 + 2 * tq;
                        T[0] = d0[rt][nn];
                        T[1] = d1[rt][nn];
                    }
                }
            }
        } else
#pragma unroll
        for (int r0 = 0; r0 < ROWS8; r0 += 8) {
            const int r = r0 + g;
            const int rb = (r < ROWS) ? (r / NC) * NT * NC + (r % NC) : 0;
#pragma unroll
            for (int n0 = 0; n0 < MTP; n0 += 8) {
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int k0 = 0; k0 < NTP; k0 += 4) {
                    const int j = k0 + tq;
                    const double av = (r < ROWS && j < NT) ? R[rb + j * NC] : 0.0;
                    dmma_8x8x4(d0, d1, av, F[(n0 + g) * LDF + k0 + tq]);
                }
                if (r < ROWS) {
                    double* T = T1 + ((r % NC) * NSP + r / NC) * LDT + n0 + 2 * tq;
                    T[0] = d0;
                    T[1] = d1;
                }
            }
        }
        __syncwarp();
        // raw[buf] fully consumed (step 1 and the copy): refill it with the panel after next
        if (lane == 0 && pl + 2 * stride < n_panels) {
            fence_proxy_async_smem();
            issue(pl + 2 * stride, buf);
        }
        // step 2 + epilogue: records {g, 0} of two adjacent nodes per lane straight from the accumulators
        double2* D2 = reinterpret_cast<double2*>(dyn);
        if constexpr (ORD == 1) {
            // fine-theta tile outer: each T1 fragment feeds all NA fine-s tiles (NA x NC independent DMMA chains,
            // a third of the T1 loads); this tile's scales are loaded first and land during the contraction
#pragma unroll
            for (int tb = 0; tb < NB; ++tb) {
                const int b = tb * 8 + 2 * tq;
                double s0[NA], s1[NA];
#pragma unroll
                for (int ta = 0; ta < NA; ++ta) {
                    const int a = ta * 8 + g;
                    if (a < MS && b < MT) {
                        const double2 v = __ldg(reinterpret_cast<const double2*>(scale + m0 + a * MT + b));
                        s0[ta] = v.x;
                        s1[ta] = v.y;
                    } else {
                        s0[ta] = s1[ta] = 0.0;
                    }
                }
                double d0[NA][NC], d1[NA][NC];
#pragma unroll
                for (int ta = 0; ta < NA; ++ta)
#pragma unroll
                    for (int c = 0; c < NC; ++c) d0[ta][c] = d1[ta][c] = 0.0;
#pragma unroll
                for (int k0 = 0; k0 < NSP; k0 += 4) {
                    double bv[NC];
#pragma unroll
                    for (int c = 0; c < NC; ++c) bv[c] = T1[(c * NSP + k0 + tq) * LDT + tb * 8 + g];
#pragma unroll
                    for (int ta = 0; ta < NA; ++ta) {
                        const double av = Ps[(ta * 8 + g) * LDP + k0 + tq];
#pragma unroll
                        for (int c = 0; c < NC; ++c) dmma_8x8x4(d0[ta][c], d1[ta][c], av, bv[c]);
                    }
                }
#pragma unroll
                for (int ta = 0; ta < NA; ++ta) {
                    const int a = ta * 8 + g;
                    if (a < MS && b < MT) {
                        const int64_t m = m0 + a * MT + b;
                        if (dyn_mc) {
                            double* o = dyn_mc + 4 * m;
                            multimem_st2(o, s0[ta] * d0[ta][0], s0[ta] * d0[ta][1]);
                            multimem_st2(o + 2, s0[ta] * d0[ta][2], 0.0);
                            multimem_st2(o + 4, s1[ta] * d1[ta][0], s1[ta] * d1[ta][1]);
                            multimem_st2(o + 6, s1[ta] * d1[ta][2], 0.0);
                        } else {
                            double2* o = D2 + 2 * m;
                            o[0] = make_double2(s0[ta] * d0[ta][0], s0[ta] * d0[ta][1]);
                            o[1] = make_double2(s0[ta] * d0[ta][2], 0.0);
                            o[2] = make_double2(s1[ta] * d1[ta][0], s1[ta] * d1[ta][1]);
                            o[3] = make_double2(s1[ta] * d1[ta][2], 0.0);
                        }
                    }
                }
            }
        } else
#pragma unroll
        for (int ta = 0; ta < NA; ++ta) {
#pragma unroll
            for (int tb = 0; tb < NB; ++tb) {
                double d0[NC], d1[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) d0[c] = d1[c] = 0.0;
#pragma unroll
                for (int k0 = 0; k0 < NSP; k0 += 4) {
                    const double av = Ps[(ta * 8 + g) * LDP + k0 + tq];
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        dmma_8x8x4(d0[c], d1[c], av, T1[(c * NSP + k0 + tq) * LDT + tb * 8 + g]);
                }
                const int a = ta * 8 + g, b = tb * 8 + 2 * tq;
                if (a < MS && b < MT) {
                    const int64_t m = m0 + a * MT + b;
                    const double s0 = sc0[ta][tb], s1 = sc1[ta][tb];
                    if (dyn_mc) {                      // fused gather (N4): replicated into every rank's copy
                        double* o = dyn_mc + 4 * m;
                        multimem_st2(o, s0 * d0[0], s0 * d0[1]);
                        multimem_st2(o + 2, s0 * d0[2], 0.0);
                        multimem_st2(o + 4, s1 * d1[0], s1 * d1[1]);
                        multimem_st2(o + 6, s1 * d1[2], 0.0);
                    } else {
                        double2* o = D2 + 2 * m;
                        o[0] = make_double2(s0 * d0[0], s0 * d0[1]);
                        o[1] = make_double2(s0 * d0[2], 0.0);
                        o[2] = make_double2(s1 * d1[0], s1 * d1[1]);
                        o[3] = make_double2(s1 * d1[2], 0.0);
                    }
                }
            }
        }
        __syncwarp();
    }
}

template <int NS, int NT, int MS, int MT>
static constexpr size_t rec_smem_bytes(int warps) {
    return sizeof(double) * ((size_t)((MS + 7) / 8 * 8) * (((NS + 3) / 4 * 4) % 16 == 0 || ((NS + 3) / 4 * 4) % 16 == 8
                                                              ? (NS + 3) / 4 * 4 + 4 : (NS + 3) / 4 * 4) +
                             (size_t)((MT + 7) / 8 * 8) * (((NT + 3) / 4 * 4) % 16 == 0 || ((NT + 3) / 4 * 4) % 16 == 8
                                                              ? (NT + 3) / 4 * 4 + 4 : (NT + 3) / 4 * 4) +
                             (size_t)warps * (2 * ((NS * NT * 3 + 1) & ~1) +
                                              3 * ((NS + 3) / 4 * 4) *
                                                  ((((MT + 7) / 8 * 8) % 16 == 0) ? (MT + 7) / 8 * 8 + 8 : (MT + 7) / 8 * 8)));
}

template <int NS, int NT, int MS, int MT, int WARPS>
static slb_status launch_rec(int64_t n_panels, const double* mats, const double* sc_in, const double* scale,
                             double* dyn, double* copy_out, const int32_t* plist, const int64_t* c_off,
                             const int64_t* f_off, cudaStream_t s, double* dyn_mc) {
    const size_t bytes = rec_smem_bytes<NS, NT, MS, MT>(WARPS);
    static const int ord = [] { const char* e = getenv("SLB_UPS_ORD"); return (e && e[0] == '0') ? 0 : 1; }();
    const void* fn = ord ? (const void*)upsample_rec_kernel<NS, NT, MS, MT, WARPS, 1>
                         : (const void*)upsample_rec_kernel<NS, NT, MS, MT, WARPS, 0>;
    { slb_status st_ = smem_optin(fn); if (st_ != SLB_OK) return st_; }
    int per_sm = 0;
    SLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, WARPS * 32, bytes));
    const unsigned grid = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((n_panels + WARPS - 1) / WARPS, (int64_t)num_sms() * std::max(1, per_sm)));
    if (ord)
        upsample_rec_kernel<NS, NT, MS, MT, WARPS, 1><<<grid, WARPS * 32, bytes, s>>>(n_panels, mats, sc_in, scale, dyn,
                                                                                     copy_out, plist, c_off, f_off, dyn_mc);
    else
        upsample_rec_kernel<NS, NT, MS, MT, WARPS, 0><<<grid, WARPS * 32, bytes, s>>>(n_panels, mats, sc_in, scale, dyn,
                                                                                     copy_out, plist, c_off, f_off, dyn_mc);
    ++g_launch_count;
    return check_launch("upsample_rec_kernel");
}

// the compiled grids; returns false when (ns, nt, ms, mt) is not one of them
static bool rec_supported(int ns, int nt, int ms, int mt) {
    return (ns == 10 && nt == 12 && ms == 20 && mt == 24) || (ns == 10 && nt == 16 && ms == 20 && mt == 32) ||
           (ns == 12 && nt == 20 && ms == 24 && mt == 40);
}

static slb_status rec_dispatch(const InterpParams& ip, int64_t n_panels, const double* sc_in, const double* scale,
                               double* dyn, double* copy_out, const int32_t* plist, const int64_t* c_off,
                               const int64_t* f_off, cudaStream_t s, double* dyn_mc) {
    static const int w8 = [] { const char* e = getenv("SLB_UPS_W8"); return (e && e[0] == '1') ? 1 : 0; }();
    if (ip.ns == 10 && ip.nt == 12 && w8)
        return launch_rec<10, 12, 20, 24, 8>(n_panels, ip.mats_d, sc_in, scale, dyn, copy_out, plist, c_off, f_off, s, dyn_mc);
    if (ip.ns == 10 && ip.nt == 12)
        return launch_rec<10, 12, 20, 24, 16>(n_panels, ip.mats_d, sc_in, scale, dyn, copy_out, plist, c_off, f_off, s, dyn_mc);
    if (ip.ns == 10 && ip.nt == 16)
        return launch_rec<10, 16, 20, 32, 8>(n_panels, ip.mats_d, sc_in, scale, dyn, copy_out, plist, c_off, f_off, s, dyn_mc);
    return launch_rec<12, 20, 24, 40, 8>(n_panels, ip.mats_d, sc_in, scale, dyn, copy_out, plist, c_off, f_off, s, dyn_mc);
}

// Per-warp buffers of the streaming kernel (doubles), or 0 when it does not apply (large grids).
static size_t up_warp_bytes(const InterpParams& ip, int nc, bool scaled, bool scalar, int* warps) {
    const UpWarpLayout L = up_layout(ip.ns, ip.nt, ip.ms, ip.mt, nc, scaled ? (scalar ? 4 : 1) : 0);
    const size_t cta = L.cta_d * 8, wb = L.warp_d * 8;
    int w = kUpW;
    while (w > 1 && cta + w * wb > 200 * 1024) --w;
    if (cta + w * wb > 200 * 1024 || w < 4) return 0;
    *warps = w;
    return cta + w * wb;
}

static bool upsample_legacy() {
    static const bool v = [] { const char* e = getenv("SLB_UPSAMPLE_LEGACY"); return e && e[0] == '1'; }();
    return v;
}

bool upsample_streams(FarKind kind, const InterpParams& ip, int nc, bool records, const double* sigma_coarse,
                      const double* sc) {
    int warps = 0;
    const bool aligned = ((uintptr_t)sigma_coarse % 16 == 0) && (!sc || (uintptr_t)sc % 16 == 0);
    return !upsample_legacy() && ip.mats_d && aligned && up_warp_bytes(ip, nc, records, far_scalar(kind), &warps) > 0;
}

slb_status upsample_launch(FarKind kind, int64_t n_panels, const InterpParams& ip, int nc,
                           const double* sigma_coarse, double* sigma_fine, const double* sc,
                           double* dyn, cudaStream_t s, const int32_t* plist, const int64_t* c_off,
                           const int64_t* f_off, double* copy_out, double* dyn_mc) {
    if (n_panels <= 0) return SLB_OK;
    int warps = 0;
    const size_t wsm = up_warp_bytes(ip, nc, dyn != nullptr, far_scalar(kind), &warps);
    static const bool generic = [] { const char* e = getenv("SLB_UPSAMPLE_GENERIC"); return e && e[0] == '1'; }();
    if (!generic && dyn && nc == 3 && !far_scalar(kind) && rec_supported(ip.ns, ip.nt, ip.ms, ip.mt) &&
        upsample_streams(kind, ip, nc, true, sigma_coarse, sc))
        return rec_dispatch(ip, n_panels, sigma_coarse, sc, dyn, copy_out, plist, c_off, f_off, s, dyn_mc);
    if (upsample_streams(kind, ip, nc, dyn != nullptr, sigma_coarse, sc)) {
        { slb_status st_ = smem_optin((const void*)upsample_warp_kernel<1>); if (st_ != SLB_OK) return st_; }
        { slb_status st_ = smem_optin((const void*)upsample_warp_kernel<3>); if (st_ != SLB_OK) return st_; }
        // a warp per panel up to the resident limit; beyond it the warps loop (and prefetch)
        const unsigned grid = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>((n_panels + warps - 1) / warps, (int64_t)num_sms() * (200 * 1024 / wsm)));
        if (nc == 1)
            upsample_warp_kernel<1><<<grid, warps * 32, wsm, s>>>((int)kind, n_panels, ip.ns, ip.nt, ip.ms, ip.mt,
                                                                  ip.mats_d, sigma_coarse, sigma_fine, sc, dyn,
                                                                  copy_out, plist, c_off, f_off, dyn_mc);
        else
            upsample_warp_kernel<3><<<grid, warps * 32, wsm, s>>>((int)kind, n_panels, ip.ns, ip.nt, ip.ms, ip.mt,
                                                                  ip.mats_d, sigma_coarse, sigma_fine, sc, dyn,
                                                                  copy_out, plist, c_off, f_off, dyn_mc);
        ++g_launch_count;
        return check_launch("upsample_warp_kernel");
    }
    SLB_REQUIRE(!dyn_mc, SLB_ERR_UNSUPPORTED, "fused multicast gather needs the streaming upsample");
    if (copy_out) {
        // legacy kernel: separate copy of the coarse density (contiguous for uniform panels / plist == NULL)
        SLB_REQUIRE(!plist, SLB_ERR_UNSUPPORTED, "fused coarse copy needs the streaming upsample");
        const int64_t nin = (int64_t)ip.ns * ip.nt * nc;
        SLB_CUDA(cudaMemcpyAsync(copy_out, sigma_coarse, sizeof(double) * nin * n_panels, cudaMemcpyDeviceToDevice, s));
    }
    auto rup_h = [](int v, int m) { return (v + m - 1) / m * m; };
    const int nsp = rup_h(ip.ns, 4), ntp = rup_h(ip.nt, 4), msp = rup_h(ip.ms, 8), mtp = rup_h(ip.mt, 8);
    const int ncol2p = rup_h(ip.mt * nc, 8);
    const int ldp = ld_g(nsp), ldf = ld_g(ntp), ld1 = ld_t(ncol2p);
    const int nin = ip.ns * ip.nt * nc;
    auto smem_of = [&](int orows, int gm) {
        return sizeof(double) * ((gm ? 0 : (size_t)msp * ldp + (size_t)mtp * ldf) + (size_t)((nin + 1) & ~1) +
                                 (size_t)nsp * ld1 + (size_t)orows * ip.mt * nc);
    };
    int orows = msp, gmats = 0;
    while (orows > 8 && smem_of(orows, 0) > 227 * 1024) orows -= 8;
    if (smem_of(orows, 0) > 227 * 1024) {           // largest grids: matrices from global memory
        gmats = 1;
        orows = msp;
        while (orows > 8 && smem_of(orows, 1) > 227 * 1024) orows -= 8;
    }
    const size_t smem = smem_of(orows, gmats);
    SLB_REQUIRE(smem <= 227 * 1024, SLB_ERR_UNSUPPORTED, "upsample: grid too large for shared memory");
    if (smem > 48 * 1024) {
        slb_status st_ = smem_optin((const void*)upsample_dmma_kernel);
        if (st_ != SLB_OK) return st_;
    }
    // one panel per CTA and pass; enough CTAs for every SM to hold several
    const unsigned grid = (unsigned)std::min<int64_t>(n_panels, (int64_t)num_sms() * 16);
    upsample_dmma_kernel<<<grid, kUpWarps * 32, smem, s>>>((int)kind, nc, n_panels, ip, sigma_coarse, sigma_fine, sc,
                                                           dyn, plist, c_off, f_off, orows, gmats);
    ++g_launch_count;
    return check_launch("upsample_dmma_kernel");
}

}  // namespace slb
