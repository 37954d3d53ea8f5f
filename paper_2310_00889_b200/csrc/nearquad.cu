// nearquad.cu -- (NEXT N1, setup) special-quadrature correction blocks.
//
// PAPER.md §3.2.3-3.2.4: for a target x near element Gamma_k (or on it), the
// correction E_ij(x) = (special quadrature of K against the interpolation basis) - G(x, y_ij) w_ij.
// This kernel computes the first part,
//     B_{t,k}[r][(i,j,c)] = int_{I_k} int_0^{2pi} K_rc(x_t - y(s,th); n(s,th)) l_i(s) C_j(th) J(s,th) dth ds,
// i.e. the exact action of the layer potential on the panel's interpolant (P:L1233-1239 with the
// adaptive rule written out), for every (target, near panel) pair of a CSR; the operator folds
// the smooth-rule part in at creation as for any B (E = B - G U).
//
// The paper's rules (toroidal Green's-function modal sums with generalized Chebyshev tables,
// App. B) are replaced by a singularity-resolving adaptive rule built on the fly:
//   * geometry y(s,th), y_s, y_th from the panel's coarse nodes by the same Lagrange x trig
//     interpolation the paper uses to represent the surface;
//   * closest point (t*, th*) by Gauss-Newton from the nearest node;
//   * quadtree cells in the locally scaled parameter plane (a = S_t (t - t*), b = S_th (th - th*)),
//     accepted when sqrt(d^2 + dist(cell)^2) >= beta * diag(cell) (flat-surface proxy), split otherwise;
//   * on-surface targets (d = 0): the four cells meeting at the node are integrated with the Duffy
//     transform (two triangles each, Jacobian u cancels the 1/r singularity), refined until their
//     aspect ratio and size are moderate;
//   * q x q Gauss-Legendre per regular cell, 2 q_d^2 nodes per Duffy cell; the contraction with the
//     basis is sum-factorized and runs on the FP64 tensor cores: regular cells are tensor grids in
//     (t, th) (Lagrange rows first, then the theta features: per-node cost NG ns (1 + nt / q)
//     instead of NG ns nt), each Duffy triangle is separable in one direction (factorized along it);
//   * the quadtree is built level by level across the CTA (block prefix sums place the cells).
// One CTA (8 or 16 warps by panel class) per target row; fixed summation order -> deterministic.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <memory>
#include <string>
#include <vector>
#include "common.cuh"

namespace slb {

constexpr int kQBatch = 128;     // minimum scratch region: kQBatch (NG + ns + ld_pad(nt)) doubles
constexpr int kMaxCells = 768;
constexpr int kMaxLevels = 64;    // quadtree depth bound
constexpr int kMaxNsQ = 32, kMaxNtQ = 64, kMaxQ = 24;

constexpr int kTri = kMaxNsQ * (kMaxNsQ + 1) / 2;   // GL tables for every n <= kMaxNsQ, at n (n-1) / 2
struct QuadParams {
    int ns, nt, q, qd;        // ns, nt: the largest panel orders of the launch (shared-memory layout)
    int region, nb, gp;       // per-node / per-cell scratch (doubles); regular cells per Bacc update / per phase
    double beta;
    double dl;                // weight of the double layer: 1, or 0 for the pure single layer (SLB_STOKES_SL)
    double tgl[kTri];         // GL nodes on [-1,1] of every order n: tgl[n (n-1)/2 + i]
    double lam[kTri];         // barycentric weights, same layout
    double gx[kMaxQ], gw[kMaxQ];        // q-point GL on [-1,1]
    double dx[kMaxQ], dw[kMaxQ];        // qd-point GL on [0,1]
};

struct Cell {
    double t0, t1, h0, h1;    // parameter rectangle (t in [-1,1], th relative to th*)
    int duffy;                // 0 regular; 1 Duffy with singular corner (t*, th*)
};
struct CellBox {              // accepted cell in shared memory; Duffy cells at the front, regular at the back
    double t0, t1, h0, h1;
};

// shared-memory leading dimension for a DMMA operand row of n doubles: = 8 (mod 16), so the four
// k-rows of an m8n8k4 B fragment fall into disjoint bank halves (2 wavefronts per load instead of 4)
__host__ __device__ constexpr int ld_pad(int n) { return ((n + 7) / 16) * 16 + 8; }

// Lagrange basis l_i(t) and l_i'(t) (barycentric second form + derivative formula)
// tg / lm: the panel order's GL nodes and barycentric weights (QuadParams tables)
__device__ void lagrange_eval(int n, const double* tg, const double* lm, double t, double* l, double* dl) {
    int hit = -1;
    for (int i = 0; i < n; ++i)
        if (fabs(t - tg[i]) < 1e-15) hit = i;
    if (hit >= 0) {
        // l_i(t_k) = delta; l_i'(t_k) = (lam_i/lam_k)/(t_k - t_i) (i != k), l_k'(t_k) = -sum_{i != k} l_i'(t_k)
        double s = 0.0;
        for (int i = 0; i < n; ++i) {
            l[i] = (i == hit) ? 1.0 : 0.0;
            if (i != hit) {
                dl[i] = (lm[i] / lm[hit]) / (tg[hit] - tg[i]);
                s += dl[i];
            }
        }
        dl[hit] = -s;
        return;
    }
    double den = 0.0, dden = 0.0;
    for (int i = 0; i < n; ++i) {
        const double c = lm[i] / (t - tg[i]);
        den += c;
        dden -= c / (t - tg[i]);
    }
    for (int i = 0; i < n; ++i) {
        const double c = lm[i] / (t - tg[i]);
        const double dc = -c / (t - tg[i]);
        l[i] = c / den;
        dl[i] = (dc * den - c * dden) / (den * den);
    }
}

// trig cardinal C_j(th) and C_j'(th), th_j = 2 pi j / N (real interpolant with the Nyquist cosine):
//   C_j = (1/N)[1 + 2 sum_{l=1}^{N/2-1} cos(l (th - th_j)) + cos(N (th - th_j) / 2)]
// with cos(l (th - th_j)) = cos(l th) cos(l th_j) + sin(l th) sin(l th_j): one sincos per point,
// cos / sin(l th) by rotation, cos / sin(l th_j) = TC / TS[(l j) mod N] (TC[m] = cos(2 pi m / N)),
// and cos(N (th - th_j)/2) = (-1)^j cos(N th / 2).  No division: exact at th = th_j.
__device__ void trig_eval(int N, double th, double* C, double* dC, const double* TC, const double* TS) {
    double c1, s1;
    sincos(th, &s1, &c1);
    double cl[kMaxNtQ / 2 + 1], sl[kMaxNtQ / 2 + 1];
    cl[0] = 1.0; sl[0] = 0.0;
    for (int l = 1; l <= N / 2; ++l) {
        cl[l] = cl[l - 1] * c1 - sl[l - 1] * s1;
        sl[l] = sl[l - 1] * c1 + cl[l - 1] * s1;
    }
    const double cN = cl[N / 2], sN = sl[N / 2];
    for (int j = 0; j < N; ++j) {
        double sv = 0.0, dv = 0.0;
        int idx = 0;
        for (int l = 1; l < N / 2; ++l) {
            idx += j;
            if (idx >= N) idx -= N;
            const double tc = TC[idx], ts = TS[idx];
            sv = fma(cl[l], tc, fma(sl[l], ts, sv));
            dv = fma((double)l, fma(cl[l], ts, -sl[l] * tc), dv);
        }
        const double sgn = (j & 1) ? -1.0 : 1.0;
        C[j] = (1.0 + 2.0 * sv + sgn * cN) / N;
        dC[j] = (2.0 * dv - 0.5 * N * sgn * sN) / N;
    }
}

// surface point and tangents from the panel's nodes Y[i][j][3]
__device__ void geom_eval(int ns, const double* tg, const double* lm, int nt, const double* Y, double t, double th,
                          double* y, double* yt, double* yh, double* lbuf, double* dlbuf, double* Cb, double* dCb,
                          const double* TC, const double* TS) {
    lagrange_eval(ns, tg, lm, t, lbuf, dlbuf);
    trig_eval(nt, th, Cb, dCb, TC, TS);
    for (int c = 0; c < 3; ++c) { y[c] = 0.0; yt[c] = 0.0; yh[c] = 0.0; }
    for (int i = 0; i < ns; ++i) {
        double a[3] = {0, 0, 0}, ad[3] = {0, 0, 0};
        for (int j = 0; j < nt; ++j) {
            const double* Yij = Y + (i * nt + j) * 3;
            for (int c = 0; c < 3; ++c) { a[c] = fma(Cb[j], Yij[c], a[c]); ad[c] = fma(dCb[j], Yij[c], ad[c]); }
        }
        for (int c = 0; c < 3; ++c) {
            y[c] = fma(lbuf[i], a[c], y[c]);
            yt[c] = fma(dlbuf[i], a[c], yt[c]);
            yh[c] = fma(lbuf[i], ad[c], yh[c]);
        }
    }
}

// trig cardinal functions without the per-panel cos/sin tables (closest-point pre-pass)
__device__ void trig_eval_direct(int N, double th, double* C, double* dC) {
    for (int j = 0; j < N; ++j) {
        const double p = th - 2.0 * kPi * j / N;
        double sv = 1.0, dv = 0.0, c1, s1;
        sincos(p, &s1, &c1);
        double ck = c1, sk = s1;
        for (int l = 1; l < N / 2; ++l) {
            sv += 2.0 * ck;
            dv -= 2.0 * l * sk;
            const double cn = ck * c1 - sk * s1, sn = sk * c1 + ck * s1;
            ck = cn; sk = sn;
        }
        sv += ck;
        dv -= 0.5 * N * sk;
        C[j] = sv / N;
        dC[j] = dv / N;
    }
}

// Closest point (t*, th*) of every off-surface (target, panel) pair by Gauss-Newton on
// |x - y(t, th)|^2 from the nearest node, one thread per CSR entry (setup pre-pass: keeps this
// serial iteration off the quadrature CTA's critical path).  cp[p] = {t*, th*}; singular pairs skipped.
__global__ void __launch_bounds__(128)
nearquad_cp_kernel(int64_t T, const double* __restrict__ x_trg, const int64_t* __restrict__ trg_node,
                   const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ panel_idx,
                   const double* __restrict__ y_coarse, const __grid_constant__ QuadParams P,
                   const int32_t* __restrict__ pnt, const int64_t* __restrict__ cn0,
                   const int32_t* __restrict__ pns, double* __restrict__ cp) {
    const int64_t nnz = row_ptr[T];
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nnz) return;
    int64_t lo = 0, hi = T - 1;                           // target t: row_ptr[t] <= p < row_ptr[t+1]
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (row_ptr[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const int64_t t = lo;
    const int64_t k = panel_idx[p];
    const int nt = pnt ? pnt[k] : P.nt, ns = pns ? pns[k] : P.ns, Nn = ns * nt;
    const int64_t c0 = cn0 ? cn0[k] : k * (int64_t)Nn;
    const int64_t node = trg_node ? trg_node[t] : -1;
    if (node >= c0 && node < c0 + Nn) return;              // singular: the node itself
    const double* tg = P.tgl + ns * (ns - 1) / 2;
    const double* lm = P.lam + ns * (ns - 1) / 2;
    const double* Y = y_coarse + c0 * 3;
    const double x0 = x_trg[3 * t], x1 = x_trg[3 * t + 1], x2 = x_trg[3 * t + 2];
    double best = 1e300, ts = 0.0, hs = 0.0;
    for (int i = 0; i < ns; ++i)
        for (int j = 0; j < nt; ++j) {
            const double* Yij = Y + (i * nt + j) * 3;
            const double d2 = (x0 - Yij[0]) * (x0 - Yij[0]) + (x1 - Yij[1]) * (x1 - Yij[1]) +
                              (x2 - Yij[2]) * (x2 - Yij[2]);
            if (d2 < best) { best = d2; ts = tg[i]; hs = 2.0 * kPi * j / nt; }
        }
    double lb[kMaxNsQ], dlb[kMaxNsQ], Cb[kMaxNtQ], dCb[kMaxNtQ];
    for (int it = 0; it < 12; ++it) {
        double y[3] = {0, 0, 0}, yt[3] = {0, 0, 0}, yh[3] = {0, 0, 0};
        lagrange_eval(ns, tg, lm, ts, lb, dlb);
        trig_eval_direct(nt, hs, Cb, dCb);
        for (int i = 0; i < ns; ++i) {
            double a[3] = {0, 0, 0}, ad[3] = {0, 0, 0};
            for (int j = 0; j < nt; ++j) {
                const double* Yij = Y + (i * nt + j) * 3;
                for (int c = 0; c < 3; ++c) { a[c] = fma(Cb[j], Yij[c], a[c]); ad[c] = fma(dCb[j], Yij[c], ad[c]); }
            }
            for (int c = 0; c < 3; ++c) {
                y[c] = fma(lb[i], a[c], y[c]);
                yt[c] = fma(dlb[i], a[c], yt[c]);
                yh[c] = fma(lb[i], ad[c], yh[c]);
            }
        }
        const double r[3] = {x0 - y[0], x1 - y[1], x2 - y[2]};
        const double a11 = yt[0] * yt[0] + yt[1] * yt[1] + yt[2] * yt[2];
        const double a22 = yh[0] * yh[0] + yh[1] * yh[1] + yh[2] * yh[2];
        const double a12 = yt[0] * yh[0] + yt[1] * yh[1] + yt[2] * yh[2];
        const double g1 = r[0] * yt[0] + r[1] * yt[1] + r[2] * yt[2];
        const double g2 = r[0] * yh[0] + r[1] * yh[1] + r[2] * yh[2];
        const double det = a11 * a22 - a12 * a12;
        if (!(det > 0.0)) break;
        double dt = (a22 * g1 - a12 * g2) / det, dh = (a11 * g2 - a12 * g1) / det;
        const double tn = fmin(1.0, fmax(-1.0, ts + dt));
        if (tn != ts + dt) dh = g2 / a22;                  // on the boundary: 1-D step in th
        dt = tn - ts;
        ts = tn;
        hs += dh;
        if (fabs(dt) + fabs(dh) < 1e-15) break;
    }
    cp[2 * p] = ts;
    cp[2 * p + 1] = hs;
}

// features of the trig cardinal basis at th (c1, s1 = cos th, sin th): C_j(th) = sum_m f_m(th) phi_m(th_j),
// f = (1, 2cos th, 2sin th, ..., 2cos (N/2-1)th, 2sin (N/2-1)th, cos(N th/2)) / N
__device__ __forceinline__ void trig_features(int nt, double c1, double s1, double* Cb) {
    const double invN = 1.0 / nt;
    Cb[0] = invN;
    double ck = c1, sk = s1;
    for (int l = 1; l < nt / 2; ++l) {
        Cb[2 * l - 1] = 2.0 * invN * ck;
        Cb[2 * l] = 2.0 * invN * sk;
        const double cn = ck * c1 - sk * s1;
        sk = sk * c1 + ck * s1;
        ck = cn;
    }
    Cb[nt - 1] = invN * ck;                   // ck = cos(N th / 2) here
}

__device__ __forceinline__ void point_kernel(int kind, const double* y, const double* yt, const double* yh, double W,
                                             double x0, double x1, double x2, double eta, double dlw, double* G);

// kernel x weight at one quadrature node (t given by its Lagrange values lb, dlb; angle th; rule
// weight W): surface point and tangents from the rings' Fourier modes FA / FB [ns][H][3] (modes <= K),
// outward normal (R8) n = y_th x y_t / |.|, J = |y_th x y_t|; G[NG] = K(x - y; n) W J.
__device__ __forceinline__ void node_kernel(int kind, int ns, int nt, int K, int H, const double* FA, const double* FB,
                                            const double* lb, const double* dlb, double c1, double s1, double W,
                                            double x0, double x1, double x2, double eta, double dlw, double* G) {
    double y[3] = {0, 0, 0}, yt[3] = {0, 0, 0}, yh[3] = {0, 0, 0};
    for (int i = 0; i < ns; ++i) {                // ring i at th, and d/dth, from its modes
        const double* Ai = FA + i * H * 3;
        const double* Bi = FB + i * H * 3;
        double R[3] = {Ai[0], Ai[1], Ai[2]}, dR[3] = {0, 0, 0};
        double ck = c1, sk = s1;
        for (int l = 1; l <= K; ++l) {
            const double f = (2 * l == nt) ? 1.0 : 2.0;
            for (int c = 0; c < 3; ++c) {
                R[c] = fma(f, fma(Ai[3 * l + c], ck, Bi[3 * l + c] * sk), R[c]);
                dR[c] = fma(f * l, fma(Bi[3 * l + c], ck, -Ai[3 * l + c] * sk), dR[c]);
            }
            const double cn = ck * c1 - sk * s1;
            sk = sk * c1 + ck * s1;
            ck = cn;
        }
        const double li = lb[i], dli = dlb[i];
        for (int c = 0; c < 3; ++c) {
            y[c] = fma(li, R[c], y[c]);
            yt[c] = fma(dli, R[c], yt[c]);
            yh[c] = fma(li, dR[c], yh[c]);
        }
    }
    point_kernel(kind, y, yt, yh, W, x0, x1, x2, eta, dlw, G);
}

// G[NG] = K(x - y; n) W J at a surface point y with tangents yt, yh (n = y_th x y_t / |.|, J = |.|)
__device__ __forceinline__ void point_kernel(int kind, const double* y, const double* yt, const double* yh, double W,
                                             double x0, double x1, double x2, double eta, double dlw, double* G) {
    const double cr[3] = {yh[1] * yt[2] - yh[2] * yt[1], yh[2] * yt[0] - yh[0] * yt[2],
                          yh[0] * yt[1] - yh[1] * yt[0]};
    const double J = sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
    const double nrm[3] = {cr[0] / J, cr[1] / J, cr[2] / J};
    const double r[3] = {x0 - y[0], x1 - y[1], x2 - y[2]};
    const double r2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
    const double wJ = W * J;
    const int NG = (kind == FAR_LAPLACE) ? 1 : 9;
    for (int q2 = 0; q2 < NG; ++q2) G[q2] = 0.0;
    if (r2 > 0.0) {
        const double ir = 1.0 / sqrt(r2);
        const double rn = r[0] * nrm[0] + r[1] * nrm[1] + r[2] * nrm[2];
        if (kind == FAR_LAPLACE) {
            G[0] = (dlw * rn * ir * ir * ir + eta * ir) / (4.0 * kPi) * wJ;
        } else {
            const double ir3 = ir * ir * ir;
            const double sl = eta / (8.0 * kPi), dl = dlw * 3.0 / (4.0 * kPi) * rn * ir3 * ir * ir;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b)
                    G[a * 3 + b] = (sl * ((a == b ? ir : 0.0) + r[a] * r[b] * ir3) + dl * r[a] * r[b]) * wJ;
        }
    }
}

// C(m, n) (+)= sum_{k < Kn} A(m, k) B(k, n) for m < M, n < N on the FP64 tensor cores (DMMA m8n8k4,
// K padded with zeros).  Row-dependent address parts are computed once per work unit: ra = arow(m),
// then A(m, k) = fa(ra, k); rc = crow(m), then C(m, n) = fc(rc, n) (a shared-memory reference).  Work
// unit of a warp: one 8-row strip x up to 8 column tiles, the A fragment loaded once per k-step.
// acc = false: C is overwritten.
template <int NT, int TPG = 8, class FRA, class FA, class FB, class FRC, class FC>
__device__ __forceinline__ void dmma_gemm(int M, int N, int Kn, bool acc, FRA arow, FA fa, FB fb, FRC crow, FC fc) {
    // TPG: column tiles per work unit (<= 8; fewer = more, smaller units for many warps)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, fg = lane >> 2, ftq = lane & 3;
    const int mtl = (M + 7) / 8, ntl = (N + 7) / 8, ngrp = (ntl + TPG - 1) / TPG;
    for (int u = warp; u < mtl * ngrp; u += NT / 32) {
        const int m0 = (u / ngrp) * 8, ct0 = (u % ngrp) * TPG, nct = min(TPG, ntl - ct0);
        const int row = m0 + fg;
        const bool rok = row < M;
        const int ra = rok ? arow(row) : 0, rc = rok ? crow(row) : 0;
        double d0[8], d1[8];
#pragma unroll
        for (int tn = 0; tn < 8; ++tn) {
            const int oc = (ct0 + tn) * 8 + 2 * ftq;           // output columns oc, oc+1 of row m0+fg
            d0[tn] = (acc && tn < nct && rok && oc < N) ? fc(rc, oc) : 0.0;
            d1[tn] = (acc && tn < nct && rok && oc + 1 < N) ? fc(rc, oc + 1) : 0.0;
        }
        for (int k0 = 0; k0 < Kn; k0 += 4) {
            const int k = k0 + ftq;
            const double a = (rok && k < Kn) ? fa(ra, k) : 0.0;
#pragma unroll
            for (int tn = 0; tn < 8; ++tn) {
                if (tn < nct) {                                  // warp-uniform
                    const int col = (ct0 + tn) * 8 + fg;         // B column of this lane
                    const double b = (k < Kn && col < N) ? fb(k, col) : 0.0;
                    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                        : "+d"(d0[tn]), "+d"(d1[tn]) : "d"(a), "d"(b));
                }
            }
        }
#pragma unroll
        for (int tn = 0; tn < 8; ++tn) {
            const int oc = (ct0 + tn) * 8 + 2 * ftq;
            if (tn < nct && rok && oc < N) fc(rc, oc) = d0[tn];
            if (tn < nct && rok && oc + 1 < N) fc(rc, oc + 1) = d1[tn];
        }
    }
}

// regular-cell scratch (doubles): U and C of nb cells (one Bacc update), per-phase tables of gp cells
// (gp divides nb), all q t rows at once; the rings alias U when gp == nb
__host__ __device__ inline int regular_need(int q, int ns, int nt, int NG, int nb, int gp) {
    const int u = ns * ld_pad(nb * q * NG), r = gp * 6 * ns * q;
    return nb * q * ld_pad(nt) + (gp == nb ? (u > r ? u : r) : u + r) + gp * q * (3 * ld_pad(ns) + ld_pad(q * NG));
}
// one cell per group, t rows in chunks: the chunk `ac` that fits `region` (< 1: does not fit)
__host__ __device__ inline int regular_chunk(int q, int ns, int nt, int NG, int region) {
    const int fixed = q * ld_pad(nt) + ns * ld_pad(q * NG) + 6 * ns * q;
    const int per_a = 3 * ld_pad(ns) + ld_pad(q * NG);
    const int ac = (region - fixed) / per_a;
    return ac < q ? ac : q;
}

// exclusive block-wide prefix sums of three per-thread counts (o*) and their totals (t*); all NT
// threads call it; sh: 3 NT / 32 ints of shared scratch
template <int NT>
__device__ __forceinline__ void block_scan3(int a, int b, int c, int& oa, int& ob, int& oc, int& ta, int& tb, int& tc,
                                            int* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int va = a, vb = b, vc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int xa = __shfl_up_sync(0xffffffffu, va, o), xb = __shfl_up_sync(0xffffffffu, vb, o),
                  xc = __shfl_up_sync(0xffffffffu, vc, o);
        if (lane >= o) { va += xa; vb += xb; vc += xc; }
    }
    if (lane == 31) { sh[3 * warp] = va; sh[3 * warp + 1] = vb; sh[3 * warp + 2] = vc; }
    __syncthreads();
    int pa = 0, pb = 0, pc = 0;
    ta = 0; tb = 0; tc = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        const int wa = sh[3 * w], wb = sh[3 * w + 1], wc = sh[3 * w + 2];
        if (w < warp) { pa += wa; pb += wb; pc += wc; }
        ta += wa; tb += wb; tc += wc;
    }
    oa = pa + va - a; ob = pb + vb - b; oc = pc + vc - c;
    __syncthreads();
}

// SLB_NQ_PROFILE (dev builds only): per-phase SM clocks of thread 0, summed over CTAs, printed by nearquad_run
#ifdef SLB_NQ_PROFILE
__device__ unsigned long long g_nq_prof[16], g_nq_cnt[4];
#define NQ_MARK(k)                                                                                       \
    if (threadIdx.x == 0) {                                                                              \
        const long long nq_now = clock64();                                                              \
        atomicAdd(&g_nq_prof[k], (unsigned long long)(nq_now - nq_tp));                                  \
        nq_tp = nq_now;                                                                                  \
    }
#else
#define NQ_MARK(k)
#endif

// (1) of nearquad_kernel: the Duffy cells of a singular pair (see the comment inside)
template <int NT>
__device__ __noinline__ void duffy_cells(int kind, int ns, int nt, int NG, int K, int H, const double* FA,
                                         const double* FB, const double* tg, const double* lm, const QuadParams& P,
                                         const CellBox* cells, int ncells, double ts, double hs, double x0, double x1,
                                         double x2, double eta, double* Gs, double* Bacc) {
    const int tid = threadIdx.x;
    double lb[kMaxNsQ], dlb[kMaxNsQ];
    // ---------------- (1) Duffy cells (on-surface targets): two triangles per cell, each a qd x qd
    // Gauss grid in (u, v) with the singular corner C0 = (ct, ch) at u = 0.  Neither is a tensor grid
    // in (t, th), but each is separable in one direction, and the contraction is factorized along it:
    //   triangle 0 (C0, (ot, ch), (ot, oh)):  t = ct + u At (row u only),     th = ch + u v Bh
    //     T[a][q2][j] = sum_b G[(a,b)][q2] C_j(th_ab)   (DFMA),  Bacc[i][(q2,j)] += sum_a l_i(t_a) T[a][(q2,j)]
    //   triangle 1 (C0, (ot, oh), (ct, oh)):  th = ch + u Ah (row u only),    t = ct + u At (1 - v)
    //     V[a][(i,q2)] = sum_b l_i(t_ab) G[(a,b)][q2] (DFMA),  Bacc[(i,q2)][j] += sum_a V[a][(i,q2)] C_j(th_a)
    // (second steps on DMMA), u rows in chunks that fit the scratch region.
    {
        const int qd = P.qd, ldC = ld_pad(nt), ldL = ld_pad(ns), ldT = ld_pad(NG * nt), ldV = ld_pad(ns * NG);
        const int r0 = qd * (ldC + NG) + ldL + ldT, r1 = qd * (ldL + NG) + ldC + ldV;   // doubles per u row
        const int nc0 = max(1, min(qd, P.region / r0)), nc1 = max(1, min(qd, P.region / r1));
        for (int dc = 0; dc < ncells; ++dc) {
            const CellBox c = cells[dc];
            // rectangle with the singular corner at (ts, 0): corner C0, opposite corners
            const double ct = (c.t0 == ts) ? c.t0 : c.t1, ch = (c.h0 == 0.0) ? c.h0 : c.h1;
            const double ot = (c.t0 == ts) ? c.t1 : c.t0, oh = (c.h0 == 0.0) ? c.h1 : c.h0;
            const double At = ot - ct, Bh = oh - ch, Wc = fabs(At * Bh);
            for (int tri = 0; tri < 2; ++tri) {
                const int nc = tri == 0 ? nc0 : nc1;
                for (int a0 = 0; a0 < qd; a0 += nc) {
                    const int na = min(nc, qd - a0);
                    // scratch: tri 0  Cn [na qd][ldC], Gn [na qd][NG], Lr [na][ldL], Tr [na][ldT]
                    //          tri 1  Ln [na qd][ldL], Gn [na qd][NG], Cr [na][ldC], Vr [na][ldV]
                    double* Xn = Gs;                                   // Cn or Ln
                    double* Gn = Xn + na * qd * (tri == 0 ? ldC : ldL);
                    double* Xr = Gn + na * qd * NG;                    // Lr or Cr
                    double* Yr = Xr + na * (tri == 0 ? ldL : ldC);     // Tr or Vr
                    for (int n = tid; n < na * qd; n += NT) {
                        const int a2 = n / qd, ib = n % qd, ia = a0 + a2;
                        const double u = P.dx[ia], v = P.dx[ib];
                        const double tt = tri == 0 ? ct + u * At : ct + u * At * (1.0 - v);
                        const double hh = tri == 0 ? ch + u * v * Bh : ch + u * Bh;
                        const double W = P.dw[ia] * P.dw[ib] * u * Wc;
                        lagrange_eval(ns, tg, lm, tt, lb, dlb);
                        double c1, s1;
                        sincos(hs + hh, &s1, &c1);
                        double G[9];
                        node_kernel(kind, ns, nt, K, H, FA, FB, lb, dlb, c1, s1, W, x0, x1, x2, eta, P.dl, G);
                        for (int q2 = 0; q2 < NG; ++q2) Gn[n * NG + q2] = G[q2];
                        if (tri == 0) {
                            trig_features(nt, c1, s1, Xn + n * ldC);
                            if (ib == 0) for (int i = 0; i < ns; ++i) Xr[a2 * ldL + i] = lb[i];
                        } else {
                            for (int i = 0; i < ns; ++i) Xn[n * ldL + i] = lb[i];
                            if (ib == 0) trig_features(nt, c1, s1, Xr + a2 * ldC);
                        }
                    }
                    __syncthreads();
                    if (tri == 0) {
                        // T[a][q2][j] = sum_b G[(a,b)][q2] C_j(th_ab): one (a, j) per thread, NG sums
                        for (int e = tid; e < na * nt; e += NT) {
                            const int a2 = e / nt, j = e % nt;
                            double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
                            for (int ib = 0; ib < qd; ++ib) {
                                const int n = a2 * qd + ib;
                                const double cj = Xn[n * ldC + j];
                                for (int q2 = 0; q2 < NG; ++q2) acc[q2] = fma(Gn[n * NG + q2], cj, acc[q2]);
                            }
                            for (int q2 = 0; q2 < NG; ++q2) Yr[a2 * ldT + q2 * nt + j] = acc[q2];
                        }
                    } else {
                        // V[a][(i,q2)] = sum_b l_i(t_ab) G[(a,b)][q2]: one (a, i) per thread, NG sums
                        for (int e = tid; e < na * ns; e += NT) {
                            const int a2 = e / ns, i = e % ns;
                            double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
                            for (int ib = 0; ib < qd; ++ib) {
                                const int n = a2 * qd + ib;
                                const double li = Xn[n * ldL + i];
                                for (int q2 = 0; q2 < NG; ++q2) acc[q2] = fma(Gn[n * NG + q2], li, acc[q2]);
                            }
                            for (int q2 = 0; q2 < NG; ++q2) Yr[a2 * ldV + i * NG + q2] = acc[q2];
                        }
                    }
                    __syncthreads();
                    if (tri == 0)
                        dmma_gemm<NT, 4>(ns, NG * nt, na, true,
                                      [&](int row) { return row; },
                                      [&](int ra, int k) { return Xr[k * ldL + ra]; },
                                      [&](int k, int col) { return Yr[k * ldT + col]; },
                                      [&](int row) { return row * (NG * nt); },
                                      [&](int rc, int col) -> double& { return Bacc[rc + col]; });
                    else
                        dmma_gemm<NT, 4>(ns * NG, nt, na, true,
                                      [&](int row) { return row; },
                                      [&](int ra, int k) { return Yr[k * ldV + ra]; },
                                      [&](int k, int col) { return Xr[k * ldC + col]; },
                                      [&](int row) { return row * nt; },
                                      [&](int rc, int col) -> double& { return Bacc[rc + col]; });
                    __syncthreads();
                }
            }
        }
    }
}

// NT threads per (target row) CTA: 256 (two CTAs per SM) for panel classes whose layout fits 113 KB,
// else 512 (one CTA per SM, 16 warps to hide the phase latencies)
template <int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 2 : 1)
nearquad_kernel(int kind, int64_t T, const double* __restrict__ x_trg, const int64_t* __restrict__ trg_node,
                const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ panel_idx,
                const double* __restrict__ y_coarse, const double* __restrict__ eta_panel,
                const __grid_constant__ QuadParams P, double* __restrict__ blocks, int* __restrict__ status,
                const int32_t* __restrict__ pnt, const int64_t* __restrict__ cn0, const int64_t* __restrict__ boff,
                const int32_t* __restrict__ pns, const double* __restrict__ cp,
                const int32_t* __restrict__ pclass, int cls) {
    extern __shared__ double sm[];
    // ragged (NEXT N4): panel k has pnt[k] angular nodes and starts at coarse node cn0[k]; block p at
    // boff[p]; the shared layout is sized for P.nt = the largest order.  NULL: uniform P.nt.
    const int nsm = P.ns, ntm = P.nt, Nnm = nsm * ntm;   // largest panel of the launch
    const int TD = (kind == FAR_LAPLACE) ? 1 : 3;
    const int NG = TD * TD;
    const int tid = threadIdx.x;
    // shared layout
    // Y: the panel's nodes [Nn][3] for the closest point; then (same region) the rings' Fourier
    // coefficients FA, FB [ns][nt/2+1][3] for the quadrature nodes
    const int Ysz = max(Nnm * 3, nsm * (ntm / 2 + 1) * 6);
    double* Y = sm;
    double* Bacc = Y + Ysz;                           // [NG*ns][nt]  (Fourier-space accumulator)
    double* Gs = Bacc + NG * Nnm;                     // scratch region: P.region doubles (level buffers of
                                                      // the quadtree, then the Duffy / regular-cell tables)
    double* TC = Gs + P.region;                       // [ntm] cos(2 pi m / nt) of the current panel
    double* TS = TC + ntm;                            // [ntm] sin(2 pi m / nt)
    CellBox* cells = reinterpret_cast<CellBox*>(TS + ntm);
    __shared__ double s_par[8];                       // t*, th*, d, St, Sh, node-singular flag
    __shared__ int s_ncell, s_ntot, s_nreg, s_fail, s_K, s_nlvl;
    __shared__ int s_scan[3 * (NT / 32)];
    __shared__ unsigned long long s_amax;
    // per-thread scratch for the interpolation (registers / local)
    double lb[kMaxNsQ], dlb[kMaxNsQ], Cb[kMaxNtQ], dCb[kMaxNtQ];

    const int64_t t = blockIdx.x;
    if (t >= T) return;
    const double x0 = x_trg[3 * t], x1 = x_trg[3 * t + 1], x2 = x_trg[3 * t + 2];
    const int64_t node = trg_node ? trg_node[t] : -1;
#ifdef SLB_NQ_PROFILE
    long long nq_tp = clock64();
#endif
    for (int64_t p = row_ptr[t]; p < row_ptr[t + 1]; ++p) {
        const int64_t k = panel_idx[p];
        if (pclass && pclass[k] != cls) continue;             // another size class's launch
        const int nt = pnt ? pnt[k] : ntm, ns = pns ? pns[k] : nsm, Nn = ns * nt;
        const double* tg = P.tgl + ns * (ns - 1) / 2;
        const double* lm = P.lam + ns * (ns - 1) / 2;
        const int64_t c0 = cn0 ? cn0[k] : k * (int64_t)Nn;
        // single-layer weight: Stokes eta_panel (or 1: pure S); Laplace eta_panel (combined field
        // D + eta S_L), else 0 (pure D) or 1 (pure S_L, P.dl = 0)
        const double eta = (kind == FAR_STOKES_SLDL) ? (eta_panel ? eta_panel[k] : 1.0)
                                                     : (eta_panel ? eta_panel[k] : (P.dl == 0.0 ? 1.0 : 0.0));
        for (int e = tid; e < Nn * 3; e += NT) Y[e] = y_coarse[c0 * 3 + e];
        for (int e = tid; e < nt; e += NT) sincos(2.0 * kPi * e / nt, &TS[e], &TC[e]);
        for (int e = tid; e < NG * Nn; e += NT) Bacc[e] = 0.0;
        __syncthreads();
        NQ_MARK(0);
        // ---------------- closest point and the cell list (thread 0)
        if (tid == 0) {
            s_fail = 0;
            const bool singular = (node >= c0 && node < c0 + Nn);
            double ts, hs;
            if (singular) {
                const int loc = (int)(node - c0);
                ts = tg[loc / nt];
                hs = 2.0 * kPi * (loc % nt) / nt;
            } else {                          // Gauss-Newton result of the pre-pass
                ts = cp[2 * p];
                hs = cp[2 * p + 1];
            }
            double y[3], yt[3], yh[3];
            geom_eval(ns, tg, lm, nt, Y, ts, hs, y, yt, yh, lb, dlb, Cb, dCb, TC, TS);
            const double d = singular ? 0.0
                                      : sqrt((x0 - y[0]) * (x0 - y[0]) + (x1 - y[1]) * (x1 - y[1]) +
                                             (x2 - y[2]) * (x2 - y[2]));
            const double St = sqrt(yt[0] * yt[0] + yt[1] * yt[1] + yt[2] * yt[2]);
            const double Sh = sqrt(yh[0] * yh[0] + yh[1] * yh[1] + yh[2] * yh[2]);
            s_par[0] = ts; s_par[1] = hs; s_par[2] = d; s_par[3] = St; s_par[4] = Sh;
            s_par[5] = singular ? 1.0 : 0.0;
            s_ncell = 0; s_nreg = 0; s_nlvl = 0;
        }
        __syncthreads();
        // ---------------- quadtree over the parameter rectangle [-1,1] x [hs - pi, hs + pi], split at
        // (ts, hs), level by level: one thread per cell of the level, accepted cells and children placed by
        // block-wide prefix sums (deterministic order).  Level buffers live in the scratch region.
        {
            const double ts = s_par[0], d = s_par[2], St = s_par[3], Sh = s_par[4];
            const bool singular = s_par[5] != 0.0;
            const int lmax = (int)((size_t)P.region * sizeof(double) / (2 * sizeof(Cell)));
            Cell* lvl[2] = {reinterpret_cast<Cell*>(Gs), reinterpret_cast<Cell*>(Gs) + lmax};
            if (tid == 0) {
                const double T0[2] = {-1.0, ts}, T1[2] = {ts, 1.0};
                const double H0[2] = {-kPi, 0.0}, H1[2] = {0.0, kPi};
                int n0 = 0;
                for (int a = 0; a < 2; ++a)
                    for (int b = 0; b < 2; ++b) {
                        if (T1[a] - T0[a] <= 0.0) continue;
                        Cell c;
                        c.t0 = T0[a]; c.t1 = T1[a]; c.h0 = H0[b]; c.h1 = H1[b];
                        c.duffy = singular ? 1 : 0;
                        lvl[0][n0++] = c;
                    }
                s_nlvl = n0;
            }
            __syncthreads();
            const double cap = 2.0 * Sh;   // ~ tube diameter: keeps the opposite wall resolved
            // distance used by the acceptance test: on the tube (radius ~ Sh) a target at distance d
            // from the surface puts the kernel's complex singularity in th at acosh(1 + d^2 / (2 Sh (Sh + d)))
            // from th*, closer than the flat proxy d / Sh (d = 2 rho: 1.1 instead of 2) -- use that strip
            // width so cells around th* resolve the kernel (tests/test_gpu_bvp.py: 1e-9 -> 1e-12)
            const double deff = (d > 0.0) ? Sh * acosh(1.0 + d * d / (2.0 * Sh * (Sh + d))) : 0.0;
            // theta width for which a q-point GL rule integrates the degree-k = nt/2 trigonometric
            // basis to the accuracy the distance criterion gives (~2.76^-2q at beta = 0.6): the GL
            // error for e^{ik th} on a half-width h is ~ (e k h / 4q)^2q, so k h <= 4q / (2.76 e) and
            // the width 2h <= 2.13 q / nt.  Without it, cells of moderate-distance targets spanning
            // half the circumference under-resolve cos(nt th / 2) (tests/test_gpu_bvp.py: 1e-7 -> 1e-12)
            const double hmax = 2.13 * P.q / nt;
            int cur = 0;
            for (int level = 0; level < kMaxLevels; ++level) {
                const int n = s_nlvl;
                if (n == 0 || s_fail) break;
                int nout = 0;                                     // children written so far (uniform)
                for (int base = 0; base < n; base += NT) {
                    const int i = base + tid;
                    int accd = 0, accr = 0, nch = 0;
                    Cell ch[4];
                    Cell c;
                    if (i < n) {
                        c = lvl[cur][i];
                        const double wa = (c.t1 - c.t0) * St, wb = (c.h1 - c.h0) * Sh;
                        const double diag = sqrt(wa * wa + wb * wb);
                        bool accept;
                        if (c.duffy) {
                            accept = (fmax(wa, wb) <= 2.5 * fmin(wa, wb)) && diag <= cap;
                        } else {
                            // distance from (t*, th*) to the cell in scaled coordinates, plus the normal offset
                            const double da = (c.t0 > ts) ? (c.t0 - ts) * St : ((c.t1 < ts) ? (ts - c.t1) * St : 0.0);
                            const double db = (c.h0 > 0.0) ? c.h0 * Sh : ((c.h1 < 0.0) ? -c.h1 * Sh : 0.0);
                            const double dist = sqrt(deff * deff + da * da + db * db);
                            if (da >= 2.0 * cap) {
                                // far along the fiber (more than two tube diameters): the whole cross-section
                                // is at true distance >= da - cap >= da / 2, so no size cap -- cells grow
                                // geometrically along t (slender panels, rho << panel length)
                                accept = fmax(0.5 * da, d) >= P.beta * diag;
                            } else {
                                accept = dist >= P.beta * diag && diag <= 2.0 * cap;
                            }
                        }
                        accept = accept && (c.h1 - c.h0) <= hmax;
                        if (accept) {
                            (c.duffy ? accd : accr) = 1;
                        } else {
                            // split: the longer side in two (or both if comparable); Duffy keeps its corner cell
                            const bool sa = wa >= 0.5 * wb, sb = wb >= 0.5 * wa || (c.h1 - c.h0) > hmax;
                            const double tm = 0.5 * (c.t0 + c.t1), hm = 0.5 * (c.h0 + c.h1);
                            const double ta[3] = {c.t0, sa ? tm : c.t1, c.t1};
                            const double ha[3] = {c.h0, sb ? hm : c.h1, c.h1};
                            for (int a = 0; a < (sa ? 2 : 1); ++a)
                                for (int b = 0; b < (sb ? 2 : 1); ++b) {
                                    Cell sc;
                                    sc.t0 = ta[a]; sc.t1 = ta[a + 1]; sc.h0 = ha[b]; sc.h1 = ha[b + 1];
                                    // the singular corner is (ts, 0): a sub-cell keeps Duffy if it touches it
                                    const bool touch = (sc.t0 == ts || sc.t1 == ts) && (sc.h0 == 0.0 || sc.h1 == 0.0);
                                    sc.duffy = c.duffy && touch;
                                    ch[nch++] = sc;
                                }
                        }
                    }
                    int od, orr, och, td, tr, tch;
                    block_scan3<NT>(accd, accr, nch, od, orr, och, td, tr, tch, s_scan);
                    const int nc0 = s_ncell, nr0 = s_nreg;                // before this chunk
                    if (nc0 + nr0 + td + tr > kMaxCells || nout + tch > lmax) {
                        if (tid == 0) s_fail = (nout + tch > lmax) ? 2 : 1;
                        __syncthreads();
                        break;
                    }
                    if (accd) cells[nc0 + od] = CellBox{c.t0, c.t1, c.h0, c.h1};
                    if (accr) cells[kMaxCells - 1 - (nr0 + orr)] = CellBox{c.t0, c.t1, c.h0, c.h1};
                    for (int k = 0; k < nch; ++k) lvl[cur ^ 1][nout + och + k] = ch[k];
                    __syncthreads();
                    if (tid == 0) { s_ncell = nc0 + td; s_nreg = nr0 + tr; }
                    nout += tch;
                    __syncthreads();
                }
                if (tid == 0) s_nlvl = s_fail ? 0 : nout;
                cur ^= 1;
                __syncthreads();
                if (level == kMaxLevels - 1 && s_nlvl > 0 && tid == 0) s_fail = 2;
            }
            if (tid == 0) s_ntot = s_ncell * 2 * P.qd * P.qd;
        }
        __syncthreads();
        NQ_MARK(1);
        if (s_fail) {
            if (tid == 0) atomicOr(status, s_fail);
            __syncthreads();
            continue;
        }
        const double ts = s_par[0], hs = s_par[1];
        const int ntot = s_ntot, nreg = s_nreg;   // Duffy-rule nodes, regular cells
#ifdef SLB_NQ_PROFILE
        if (tid == 0) {
            atomicAdd(&g_nq_cnt[0], (unsigned long long)s_nreg);
            atomicAdd(&g_nq_cnt[1], (unsigned long long)s_ntot);
            atomicAdd(&g_nq_cnt[2], 1ull);
        }
#endif
        // ---------------- Fourier coefficients of every GL ring of the panel (trig interpolant in th):
        //   ring(th) = A_0 + 2 sum_{l=1}^{N/2-1} (A_l cos l th + B_l sin l th) + A_{N/2} cos(N th / 2),
        //   A_l = (1/N) sum_j Y_j cos(l th_j), B_l = (1/N) sum_j Y_j sin(l th_j).  Modes above K (the
        //   last one with a coefficient > 1e-15 of the ring means; K = 1 for circular cross-sections)
        //   are dropped, so a node costs O(N_s K) instead of O(N_s N_th).
        const int H = nt / 2 + 1;
        double* FA = Y;                               // [ns][H][3]
        double* FB = Y + ns * H * 3;                  // [ns][H][3]
        if (tid == 0) { s_K = 0; s_amax = 0ull; }
        __syncthreads();
        for (int e = tid; e < ns * H * 3; e += NT) {
            const int c = e % 3, l = (e / 3) % H, i = e / (3 * H);
            const double* Yr = y_coarse + (c0 + (int64_t)i * nt) * 3 + c;
            double a = 0.0, b = 0.0;
            int idx = 0;
            for (int j = 0; j < nt; ++j) {
                a = fma(Yr[3 * j], TC[idx], a);
                b = fma(Yr[3 * j], TS[idx], b);
                idx += l;
                if (idx >= nt) idx -= nt;
            }
            FA[e] = a / nt;
            FB[e] = b / nt;
            if (l == 0) atomicMax(&s_amax, (unsigned long long)__double_as_longlong(fabs(a / nt)));
        }
        __syncthreads();
        {
            const double tol = 1e-15 * __longlong_as_double((long long)s_amax);
            for (int e = tid; e < ns * H * 3; e += NT) {
                const int l = (e / 3) % H;
                if (l > 0 && (fabs(FA[e]) > tol || fabs(FB[e]) > tol)) atomicMax(&s_K, l);
            }
        }
        __syncthreads();
        NQ_MARK(2);
        const int K = s_K;
        // Bacc layout [ns][NG][nt]: row (i, q2) holds the feature coefficients of l_i(t) C_m(th) for the
        // kernel component q2 -- so that the sum-factorized step (3b) below is ONE GEMM with N = NG nt.
        // ---------------- (1) Duffy cells (on-surface targets), in a function of its own (registers)
        duffy_cells<NT>(kind, ns, nt, NG, K, H, FA, FB, tg, lm, P, cells, ntot / (2 * P.qd * P.qd), ts, hs, x0, x1, x2,
                        eta, Gs, Bacc);
        NQ_MARK(3);
        // ---------------- (2) regular cells: q x q tensor Gauss grids, contraction sum-factorized
        //   U[i][(b,q2)]     = sum_a l_i(t_a) G[(a,b)][q2]       (GEMM: M = ns, N = q NG, K = q)
        //   Bacc[(i,q2)][j] += sum_b U[i][(b,q2)] C_j(th_b)      (GEMM: M = ns NG, N = nt, K = q)
        // i.e. q^2 NG ns + q NG ns nt multiply-adds per cell instead of q^2 NG ns nt.  Every phase
        // (tables: features and rings at the q theta nodes, Lagrange rows at the q t nodes; kernel at the
        // nodes; U) covers a group of P.gp cells, one entry per thread; the U and C of P.nb cells (a
        // multiple of gp) are stacked along K for one Bacc update.  All in the scratch region (Gs..).
        // Without room for one whole cell (nb = gp = 1 only) the t rows go in chunks of ac.
        {
            const int q = P.q, nk = P.nb, ng = P.gp;
            const int ldC = ld_pad(nt), ldL = ld_pad(ns), ldG = ld_pad(q * NG), ldU = ld_pad(nk * q * NG);
            const int ac = nk > 1 ? q : max(1, regular_chunk(q, ns, nt, NG, P.region));
            // rings alias U when a group fills U (U dead between the node phase and the U GEMM)
            const bool alias = ac == q && ng == nk;
            double* Cc = Gs;                          // [nk q][ldC]      features at the cells' th nodes
            double* Uc = Cc + nk * q * ldC;           // [ns][ldU]        (cell, b, q2)
            double* Rg = alias ? Uc : Uc + ns * ldU;  // [ng][ns][6][q]   rings and d/dth at the th nodes
            double* Lc = alias ? Uc + max(ns * ldU, ng * 6 * ns * q) : Rg + ng * 6 * ns * q;   // [ng][ac][ldL]
            double* dLc = Lc + ng * ac * ldL;         // [ng][ac][ldL]    l_i'(t_a)
            double* iXc = dLc + ng * ac * ldL;        // [ng][ac][ldL]    1 / (t_a - t_i)
            double* Gc = iXc + ng * ac * ldL;         // [ng][ac][ldG]    (b, q2): kernel x weight at the nodes
            const int nl = nt / 2;                    // feature pairs (cos l th, sin l th), l = 1 .. nt/2
            const int nparts = 4, lper = (nl + nparts - 1) / nparts;
            const CellBox* creg = cells + kMaxCells - 1;   // regular cell r: creg[-r]
            for (int g0 = 0; g0 < nreg; g0 += ng) {
                const int gn = min(ng, nreg - g0);
                for (int a0 = 0; a0 < q; a0 += ac) {
                    const int na = min(ac, q - a0);
                    if (a0 == 0) {
                        // features C[b][m] (trig_features layout) by (cell, b, quarter of the l range)
                        for (int e = tid; e < gn * q * nparts; e += NT) {
                            const int sl = e / (q * nparts), b2 = (e / nparts) % q;
                            const int l0 = 1 + (e % nparts) * lper, l1 = min(nl, l0 + lper - 1);
                            const CellBox c = creg[-(g0 + sl)];
                            const double th = hs + c.h0 + 0.5 * (c.h1 - c.h0) * (P.gx[b2] + 1.0);
                            double* Cr = Cc + (((g0 + sl) % nk) * q + b2) * ldC;
                            const double invN = 1.0 / nt;
                            if (l0 == 1) Cr[0] = invN;
                            if (l0 <= l1) {
                                double c1, s1, ck, sk;
                                sincos(th, &s1, &c1);
                                sincos(l0 * th, &sk, &ck);
                                for (int l = l0; l <= l1; ++l) {
                                    if (l < nl) { Cr[2 * l - 1] = 2.0 * invN * ck; Cr[2 * l] = 2.0 * invN * sk; }
                                    else Cr[nt - 1] = invN * ck;                  // l = N/2: cos(N th / 2)
                                    const double cn = ck * c1 - sk * s1;
                                    sk = sk * c1 + ck * s1;
                                    ck = cn;
                                }
                            }
                        }
                        // ring i at the q theta nodes from its Fourier modes (<= K): R_i(th_b), dR_i/dth (th_b)
                        for (int e = tid; e < gn * ns * q; e += NT) {
                            const int sl = e / (ns * q), i = (e / q) % ns, b2 = e % q;
                            const CellBox c = creg[-(g0 + sl)];
                            double c1, s1;
                            sincos(hs + c.h0 + 0.5 * (c.h1 - c.h0) * (P.gx[b2] + 1.0), &s1, &c1);
                            const double* Ai = FA + i * H * 3;
                            const double* Bi = FB + i * H * 3;
                            double R[3] = {Ai[0], Ai[1], Ai[2]}, dR[3] = {0, 0, 0};
                            double ck = c1, sk = s1;
                            for (int l = 1; l <= K; ++l) {
                                const double f = (2 * l == nt) ? 1.0 : 2.0;
                                for (int cc = 0; cc < 3; ++cc) {
                                    R[cc] = fma(f, fma(Ai[3 * l + cc], ck, Bi[3 * l + cc] * sk), R[cc]);
                                    dR[cc] = fma(f * l, fma(Bi[3 * l + cc], ck, -Ai[3 * l + cc] * sk), dR[cc]);
                                }
                                const double cn = ck * c1 - sk * s1;
                                sk = sk * c1 + ck * s1;
                                ck = cn;
                            }
                            double* Rs = Rg + sl * 6 * ns * q;
                            for (int cc = 0; cc < 3; ++cc) {
                                Rs[(i * 6 + cc) * q + b2] = R[cc];
                                Rs[(i * 6 + 3 + cc) * q + b2] = dR[cc];
                            }
                        }
                    }
                    // Lagrange rows, barycentric (as lagrange_eval): reciprocals of t_a - t_i first
                    for (int e = tid; e < gn * na * ns; e += NT) {
                        const int sl = e / (na * ns), a2 = (e / ns) % na, i = e % ns;
                        const CellBox c = creg[-(g0 + sl)];
                        const double X = (c.t0 + 0.5 * (c.t1 - c.t0) * (P.gx[a0 + a2] + 1.0)) - tg[i];
                        iXc[(sl * ac + a2) * ldL + i] = (fabs(X) < 1e-15) ? 0.0 : 1.0 / X;    // 0: t_a on node i
                    }
                    __syncthreads();
                    NQ_MARK(6);
                    for (int e = tid; e < gn * na * ns; e += NT) {
                        const int sl = e / (na * ns), a2 = (e / ns) % na, i = e % ns;
                        const double* iX = iXc + (sl * ac + a2) * ldL;
                        int hit = -1;
                        double den = 0.0, dden = 0.0;
                        for (int k = 0; k < ns; ++k) {
                            if (iX[k] == 0.0) hit = k;
                            const double ck = lm[k] * iX[k];
                            den += ck;
                            dden -= ck * iX[k];
                        }
                        double l, dl;
                        if (hit >= 0) {                   // t_a on a node: l = delta, l' by the node formula
                            l = (i == hit) ? 1.0 : 0.0;
                            if (i != hit) {
                                dl = (lm[i] / lm[hit]) / (tg[hit] - tg[i]);
                            } else {
                                dl = 0.0;
                                for (int k = 0; k < ns; ++k)
                                    if (k != hit) dl -= (lm[k] / lm[hit]) / (tg[hit] - tg[k]);
                            }
                        } else {
                            const double ci = lm[i] * iX[i], dci = -ci * iX[i], iden = 1.0 / den;
                            l = ci * iden;
                            dl = (dci * den - ci * dden) * iden * iden;
                        }
                        Lc[(sl * ac + a2) * ldL + i] = l;
                        dLc[(sl * ac + a2) * ldL + i] = dl;
                    }
                    __syncthreads();
                    NQ_MARK(7);
                    for (int n = tid; n < gn * na * q; n += NT) {
                        const int sl = n / (na * q), a2 = (n / q) % na, b2 = n % q;
                        const CellBox c = creg[-(g0 + sl)];
                        const double* la = Lc + (sl * ac + a2) * ldL;
                        const double* dla = dLc + (sl * ac + a2) * ldL;
                        const double* Rs = Rg + sl * 6 * ns * q + b2;
                        double y[3] = {0, 0, 0}, yt[3] = {0, 0, 0}, yh[3] = {0, 0, 0};
                        for (int i = 0; i < ns; ++i) {
                            const double li = la[i], dli = dla[i];
                            const double* Ri = Rs + i * 6 * q;
                            for (int cc = 0; cc < 3; ++cc) {
                                y[cc] = fma(li, Ri[cc * q], y[cc]);
                                yt[cc] = fma(dli, Ri[cc * q], yt[cc]);
                                yh[cc] = fma(li, Ri[(3 + cc) * q], yh[cc]);
                            }
                        }
                        const double W = P.gw[a0 + a2] * P.gw[b2] * (0.5 * (c.t1 - c.t0)) * (0.5 * (c.h1 - c.h0));
                        double G[9];
                        point_kernel(kind, y, yt, yh, W, x0, x1, x2, eta, P.dl, G);
                        double* Gn = Gc + (sl * ac + a2) * ldG + b2 * NG;
                        for (int q2 = 0; q2 < NG; ++q2) Gn[q2] = G[q2];
                    }
                    __syncthreads();
                    NQ_MARK(8);
                    for (int sl = 0; sl < gn; ++sl)
                        dmma_gemm<NT, NT == 512 ? 2 : 4>(ns, q * NG, na, a0 > 0,
                                      [&](int row) { return row; },
                                      [&](int ra, int k) { return Lc[(sl * ac + k) * ldL + ra]; },
                                      [&](int k, int col) { return Gc[(sl * ac + k) * ldG + col]; },
                                      [&](int row) { return row * ldU + ((g0 + sl) % nk) * q * NG; },
                                      [&](int rc2, int col) -> double& { return Uc[rc2 + col]; });
                    __syncthreads();
                    NQ_MARK(9);
                }
                if ((g0 + gn) % nk == 0 || g0 + gn == nreg) {
                    // 16 warps: half-width units balance the 18 row strips of a 16 x 64 panel
                    dmma_gemm<NT, NT == 512 ? 4 : 8>(ns * NG, nt, ((g0 + gn - 1) % nk + 1) * q, true,
                                  [&](int row) { return (row / NG) * ldU + row % NG; },
                                  [&](int ra, int k) { return Uc[ra + k * NG]; },
                                  [&](int k, int col) { return Cc[k * ldC + col]; },
                                  [&](int row) { return row * nt; },
                                  [&](int rc2, int col) -> double& { return Bacc[rc2 + col]; });
                    __syncthreads();
                    NQ_MARK(10);
                }
            }
        }
        // ---------------- write the block: [tdim][node (i,j)][sdim]
        // back from the feature basis to the nodal basis: B[(q2,i)][j] = sum_m Bacc[(q2,i)][m] phi_m(th_j),
        // phi = (1, cos th_j, sin th_j, ..., cos (N/2-1)th_j, sin (N/2-1)th_j, (-1)^j)
        double* Bp = blocks + (boff ? boff[p] : p * (int64_t)TD * Nn * TD);
        for (int o = tid; o < NG * Nn; o += NT) {
            const int q2 = o / Nn, ij = o % Nn, i = ij / nt, j = ij % nt;
            const double* Fr = Bacc + (i * NG + q2) * nt;
            double acc = Fr[0];
            int idx = 0;
            for (int l = 1; l < nt / 2; ++l) {
                idx += j;
                if (idx >= nt) idx -= nt;
                acc = fma(Fr[2 * l - 1], TC[idx], fma(Fr[2 * l], TS[idx], acc));
            }
            acc = fma((j & 1) ? -1.0 : 1.0, Fr[nt - 1], acc);
            const int a = q2 / TD, b = q2 % TD;
            Bp[(a * Nn + ij) * TD + b] = acc;
        }
        __syncthreads();
        NQ_MARK(5);
    }
}

}  // namespace slb

using namespace slb;

namespace slb {
slb_status nearquad_modal_run(slb_kernel kernel, int64_t n_trg, const double* x_trg, const int64_t* trg_node,
                              const int64_t* row_ptr, const int32_t* panel_idx, int ns_max, int nt_max,
                              const double* y_coarse, const double* eta_panel, double* blocks, cudaStream_t s,
                              const int32_t* pnt, const int64_t* cn0, const int64_t* boff, const int32_t* pns,
                              int ns_uniform, int nt_uniform);
}

// One launch per panel size class (ragged panels: the shared-memory layout is sized by the class's
// largest panel, so small panels keep several CTAs per SM -- c3v's 16 x 64 gap panels would otherwise
// force one CTA per SM on every target).  classes: (ns_max, nt_max) per class; pclass [P] or NULL.
static slb_status nearquad_run(slb_kernel kernel, int64_t n_trg, const double* x_trg, const int64_t* trg_node,
                               const int64_t* row_ptr, const int32_t* panel_idx, int ns, int nt,
                               const double* y_coarse, const double* eta_panel, int order, double beta,
                               double* blocks, cudaStream_t s, const int32_t* pnt, const int64_t* cn0,
                               const int64_t* boff, const int32_t* pns,
                               const std::vector<std::pair<int, int>>& classes = {}, const int32_t* pclass = nullptr) {
    std::unique_ptr<QuadParams> Pp(new QuadParams);      // 10 KB: heap, per call (thread-safe)
    QuadParams& P = *Pp;
    P.region = 0; P.nb = 1; P.gp = 1;
    P.ns = ns; P.nt = nt; P.q = order; P.qd = std::min(kMaxQ, order + 4); P.beta = beta;
    P.dl = (kernel == SLB_STOKES_SL || kernel == SLB_LAPLACE_SL) ? 0.0 : 1.0;
    double w[kMaxNsQ];
    for (int n = 2; n <= kMaxNsQ; ++n) {
        double* tg = P.tgl + n * (n - 1) / 2;
        double* lm = P.lam + n * (n - 1) / 2;
        gl_nodes(n, tg, w);
        for (int i = 0; i < n; ++i) {
            double pr = 1.0;
            for (int l = 0; l < n; ++l) if (l != i) pr *= (tg[i] - tg[l]);
            lm[i] = 1.0 / pr;
        }
    }
    gl_nodes(P.q, P.gx, P.gw);
    gl_nodes(P.qd, P.dx, P.dw);
    for (int a = 0; a < P.qd; ++a) { P.dx[a] = 0.5 * (P.dx[a] + 1.0); P.dw[a] *= 0.5; }
    const int TD = (kernel == SLB_LAPLACE_DL || kernel == SLB_LAPLACE_SL) ? 1 : 3;
    // shared layout per class: the scratch region holds the quadtree levels, Duffy u-row chunks or the regular-cell
    // tables of nb cells; nb (<= 4) as large as the CTA shape allows -- 256 threads and <= 113 KB (two
    // CTAs per SM) when the Duffy-only layout fits that, else 512 threads and <= 227 KB -- else one cell
    // per update with t rows in chunks
    struct Layout { int region, nb, gp, threads; size_t smem; };
    const int NGh = TD * TD;
    auto layout_of = [&](int ns_, int nt_) -> Layout {
        const size_t Nn = (size_t)ns_ * nt_;
        const size_t Ysz = std::max(Nn * 3, (size_t)ns_ * (nt_ / 2 + 1) * 6);
        const size_t base = sizeof(double) * (Ysz + (size_t)NGh * Nn + 2 * (size_t)nt_) + sizeof(CellBox) * kMaxCells;
        const int duffy = kQBatch * (NGh + ns_ + ld_pad(nt_));
        const bool small = base + sizeof(double) * duffy <= 113 * 1024;
        const size_t budget = small ? 113 * 1024 : 227 * 1024;
        const int threads = small ? 256 : 512;
        // SLB_NQ_NB: cap on the cells per group (tuning knob; read once, thread-safe static)
        static const int nb_max = [] {
            const char* e = getenv("SLB_NQ_NB");
            return e ? std::max(1, std::min(4, atoi(e))) : 4;
        }();
        // (cells per update, per phase): K-stacking first, then phase groups
        static const int cand[8][2] = {{4, 4}, {4, 2}, {3, 3}, {2, 2}, {4, 1}, {3, 1}, {2, 1}, {1, 1}};
        for (const auto& c : cand) {
            if (c[0] > nb_max) continue;
            const int region = std::max(duffy, regular_need(order, ns_, nt_, NGh, c[0], c[1]));
            if (base + sizeof(double) * region <= budget)
                return {region, c[0], c[1], threads, base + sizeof(double) * region};
        }
        return {duffy, 1, 1, threads, base + sizeof(double) * duffy};
    };
    std::vector<std::pair<int, int>> cls = classes.empty() ? std::vector<std::pair<int, int>>{{ns, nt}} : classes;
    size_t smem_max = 0;
    for (auto& c : cls) {
        const Layout L = layout_of(c.first, c.second);
        SLB_REQUIRE(L.smem <= 227 * 1024, SLB_ERR_UNSUPPORTED, "nearquad: shared memory");
        SLB_REQUIRE(regular_chunk(order, c.first, c.second, NGh, L.region) >= 1, SLB_ERR_UNSUPPORTED,
                    "nearquad: rule order too large for the panel grid");
        smem_max = std::max(smem_max, L.smem);
    }
    { slb_status st_ = smem_optin((const void*)nearquad_kernel<256>); if (st_ != SLB_OK) return st_; }
    { slb_status st_ = smem_optin((const void*)nearquad_kernel<512>); if (st_ != SLB_OK) return st_; }
    int* st = nullptr;
    SLB_CUDA(cudaMallocAsync(&st, sizeof(int), s));
    SLB_CUDA(cudaMemsetAsync(st, 0, sizeof(int), s));
    int64_t nnz = 0;
    SLB_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n_trg, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SLB_CUDA(cudaStreamSynchronize(s));
    double* cp = nullptr;
    SLB_CUDA(cudaMallocAsync(&cp, sizeof(double) * 2 * std::max<int64_t>(nnz, 1), s));
    if (nnz > 0) {
        nearquad_cp_kernel<<<(unsigned)((nnz + 127) / 128), 128, 0, s>>>(n_trg, x_trg, trg_node, row_ptr, panel_idx,
                                                                        y_coarse, P, pnt, cn0, pns, cp);
        ++g_launch_count;
    }
    const FarKind kind = (kernel == SLB_LAPLACE_DL || kernel == SLB_LAPLACE_SL) ? FAR_LAPLACE : FAR_STOKES_SLDL;
    slb_status r = SLB_OK;
    for (int c = 0; c < (int)cls.size() && r == SLB_OK; ++c) {
        P.ns = cls[c].first;
        P.nt = cls[c].second;
        const Layout L = layout_of(P.ns, P.nt);
        P.region = L.region;
        P.nb = L.nb;
        P.gp = L.gp;
        if (L.threads == 256)
            nearquad_kernel<256><<<(unsigned)n_trg, 256, L.smem, s>>>(
                (int)kind, n_trg, x_trg, trg_node, row_ptr, panel_idx, y_coarse, eta_panel, P, blocks, st, pnt, cn0,
                boff, pns, cp, pclass, c);
        else
            nearquad_kernel<512><<<(unsigned)n_trg, 512, L.smem, s>>>(
                (int)kind, n_trg, x_trg, trg_node, row_ptr, panel_idx, y_coarse, eta_panel, P, blocks, st, pnt, cn0,
                boff, pns, cp, pclass, c);
        ++g_launch_count;
        r = check_launch("nearquad_kernel");
    }
    int h = 0;
    if (r == SLB_OK) {
        cudaError_t e = cudaMemcpyAsync(&h, st, sizeof(int), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) { set_error(std::string("nearquad: ") + cudaGetErrorString(e)); r = SLB_ERR_CUDA; }
    }
#ifdef SLB_NQ_PROFILE
    {
        unsigned long long pr[16], cn[4];
        cudaMemcpyFromSymbol(pr, g_nq_prof, sizeof(pr));
        cudaMemcpyFromSymbol(cn, g_nq_cnt, sizeof(cn));
        fprintf(stderr, "nearquad profile (Mclk): setup %.0f tree %.0f modes %.0f duffy %.0f tables %.0f lagr %.0f nodes %.0f "
                "gemm1 %.0f gemm2 %.0f write %.0f | pairs %llu regular cells %llu duffy nodes %llu\n",
                pr[0] * 1e-6, pr[1] * 1e-6, pr[2] * 1e-6, pr[3] * 1e-6, pr[6] * 1e-6, pr[7] * 1e-6, pr[8] * 1e-6,
                pr[9] * 1e-6, pr[10] * 1e-6, pr[5] * 1e-6, cn[2], cn[0], cn[1]);
    }
#endif
    cudaFreeAsync(st, s);
    cudaFreeAsync(cp, s);
    if (r == SLB_OK && h) {
        set_error("nearquad: adaptive cell budget exceeded (target extremely close to a panel?)");
        r = SLB_ERR_UNSUPPORTED;
    }
    return r;
}

static slb_status nearquad_check(slb_kernel kernel, int64_t n_trg, int ns, int order, double beta) {
    SLB_REQUIRE(kernel == SLB_LAPLACE_DL || kernel == SLB_STOKES_SLDL || kernel == SLB_STOKES_SL ||
                    kernel == SLB_LAPLACE_SL,
                SLB_ERR_INVALID_ARG, "bad kernel");
    SLB_REQUIRE(n_trg >= 0 && ns >= 2, SLB_ERR_INVALID_ARG, "bad sizes");
    SLB_REQUIRE(ns <= kMaxNsQ, SLB_ERR_UNSUPPORTED, "panel grid too large for nearquad");
    SLB_REQUIRE(order == 0 || (order >= 4 && order <= kMaxQ && beta > 0.0), SLB_ERR_INVALID_ARG,
                "need order 0 (the paper's rule) or 4 <= order <= 24 with beta > 0");
    SLB_REQUIRE(n_trg <= 2147483647LL, SLB_ERR_UNSUPPORTED, "too many targets");
    return SLB_OK;
}

extern "C" slb_status slb_nearcorr_quad(slb_kernel kernel, int64_t n_trg, const double* x_trg, const int64_t* trg_node,
                                        const int64_t* row_ptr, const int32_t* panel_idx, int ns, int nt,
                                        const double* y_coarse, const double* eta_panel, int order, double beta,
                                        double* blocks, cudaStream_t s) {
    slb_status c = nearquad_check(kernel, n_trg, ns, order, beta);
    if (c != SLB_OK) return c;
    SLB_REQUIRE(nt >= 4 && nt % 2 == 0, SLB_ERR_INVALID_ARG, "bad sizes");
    SLB_REQUIRE(nt <= kMaxNtQ, SLB_ERR_UNSUPPORTED, "panel grid too large for nearquad");
    if (n_trg == 0) return SLB_OK;
    SLB_REQUIRE(x_trg && row_ptr && panel_idx && y_coarse && blocks, SLB_ERR_INVALID_ARG, "null pointer");
    SLB_REQUIRE(kernel != SLB_STOKES_SLDL || eta_panel, SLB_ERR_INVALID_ARG, "Stokes SL+DL needs eta_panel");
    if (order == 0)
        return nearquad_modal_run(kernel, n_trg, x_trg, trg_node, row_ptr, panel_idx, ns, nt, y_coarse, eta_panel, blocks,
                                  s, nullptr, nullptr, nullptr, nullptr, ns, nt);
    return nearquad_run(kernel, n_trg, x_trg, trg_node, row_ptr, panel_idx, ns, nt, y_coarse, eta_panel, order, beta,
                        blocks, s, nullptr, nullptr, nullptr, nullptr);
}

extern "C" slb_status slb_nearcorr_quad_ragged(slb_kernel kernel, int64_t n_trg, const double* x_trg,
                                               const int64_t* trg_node, const int64_t* row_ptr,
                                               const int32_t* panel_idx, int64_t n_panels, const int32_t* panel_ns,
                                               const int32_t* panel_nt, const double* y_coarse,
                                               const double* eta_panel, int order, double beta, double* blocks,
                                               cudaStream_t s) {
    slb_status c = nearquad_check(kernel, n_trg, 2, order, beta);
    if (c != SLB_OK) return c;
    if (n_trg == 0) return SLB_OK;
    SLB_REQUIRE(x_trg && row_ptr && panel_idx && y_coarse && blocks && panel_nt && panel_ns && n_panels > 0,
                SLB_ERR_INVALID_ARG, "null pointer");
    SLB_REQUIRE(kernel != SLB_STOKES_SLDL || eta_panel, SLB_ERR_INVALID_ARG, "Stokes SL+DL needs eta_panel");
    const int TD = (kernel == SLB_LAPLACE_DL || kernel == SLB_LAPLACE_SL) ? 1 : 3;
    std::vector<int64_t> c0(n_panels + 1, 0);
    int ntmax = 0, nsmax = 0;
    for (int64_t k = 0; k < n_panels; ++k) {
        SLB_REQUIRE(panel_nt[k] >= 4 && panel_nt[k] % 2 == 0 && panel_ns[k] >= 2, SLB_ERR_INVALID_ARG,
                    "bad panel orders");
        SLB_REQUIRE(panel_nt[k] <= kMaxNtQ && panel_ns[k] <= kMaxNsQ, SLB_ERR_UNSUPPORTED,
                    "panel grid too large for nearquad");
        c0[k + 1] = c0[k] + (int64_t)panel_ns[k] * panel_nt[k];
        ntmax = std::max(ntmax, (int)panel_nt[k]);
        nsmax = std::max(nsmax, (int)panel_ns[k]);
    }
    int64_t nnz = 0;
    SLB_CUDA(cudaStreamSynchronize(s));
    SLB_CUDA(cudaMemcpy(&nnz, row_ptr + n_trg, sizeof(int64_t), cudaMemcpyDeviceToHost));
    std::vector<int32_t> pk(std::max<int64_t>(nnz, 1));
    if (nnz) SLB_CUDA(cudaMemcpy(pk.data(), panel_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
    std::vector<int64_t> bo(nnz + 1, 0);
    for (int64_t p = 0; p < nnz; ++p) {
        SLB_REQUIRE(pk[p] >= 0 && pk[p] < n_panels, SLB_ERR_INVALID_ARG, "panel_idx entry outside [0, n_panels)");
        bo[p + 1] = bo[p] + (int64_t)TD * (c0[pk[p] + 1] - c0[pk[p]]) * TD;
    }
    // size classes by nodes per panel: <= 192, <= 512, larger (each launch sized by its largest panel)
    std::vector<int32_t> pc(n_panels);
    std::vector<std::pair<int, int>> classes(3, {2, 4});
    for (int64_t k = 0; k < n_panels; ++k) {
        const int nn = panel_ns[k] * panel_nt[k];
        const int c = nn <= 192 ? 0 : (nn <= 512 ? 1 : 2);
        pc[k] = c;
        classes[c].first = std::max(classes[c].first, (int)panel_ns[k]);
        classes[c].second = std::max(classes[c].second, (int)panel_nt[k]);
    }
    int32_t *pnt_d = nullptr, *pns_d = nullptr, *pc_d = nullptr;
    int64_t *c0_d = nullptr, *bo_d = nullptr;
    auto cleanup = [&]() { cudaFree(pnt_d); cudaFree(pns_d); cudaFree(c0_d); cudaFree(bo_d); cudaFree(pc_d); };
    if (cudaMalloc(&pnt_d, sizeof(int32_t) * n_panels) != cudaSuccess ||
        cudaMalloc(&pns_d, sizeof(int32_t) * n_panels) != cudaSuccess ||
        cudaMalloc(&c0_d, sizeof(int64_t) * (n_panels + 1)) != cudaSuccess ||
        cudaMalloc(&bo_d, sizeof(int64_t) * (nnz + 1)) != cudaSuccess ||
        cudaMalloc(&pc_d, sizeof(int32_t) * n_panels) != cudaSuccess) {
        cleanup();
        set_error("slb_nearcorr_quad_ragged: out of device memory");
        return SLB_ERR_OOM;
    }
    if (cudaMemcpy(pnt_d, panel_nt, sizeof(int32_t) * n_panels, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(pns_d, panel_ns, sizeof(int32_t) * n_panels, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c0_d, c0.data(), sizeof(int64_t) * (n_panels + 1), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(bo_d, bo.data(), sizeof(int64_t) * (nnz + 1), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(pc_d, pc.data(), sizeof(int32_t) * n_panels, cudaMemcpyHostToDevice) != cudaSuccess) {
        cleanup();
        set_error("slb_nearcorr_quad_ragged: copying the panel tables failed");
        return SLB_ERR_CUDA;
    }
    slb_status r = order == 0
                       ? nearquad_modal_run(kernel, n_trg, x_trg, trg_node, row_ptr, panel_idx, nsmax, ntmax, y_coarse,
                                            eta_panel, blocks, s, pnt_d, c0_d, bo_d, pns_d, nsmax, ntmax)
                       : nearquad_run(kernel, n_trg, x_trg, trg_node, row_ptr, panel_idx, nsmax, ntmax, y_coarse, eta_panel,
                                      order, beta, blocks, s, pnt_d, c0_d, bo_d, pns_d, classes, pc_d);
    cudaStreamSynchronize(s);
    cleanup();
    return r;
}
