// interp.cpp -- host construction of the upsampling operators U = P_s (x) F_th.
//
// PAPER.md §3.1: "barycentric Lagrange interpolation from the nodes of the
// containing panel in s [Berrut2004] and trigonometric interpolation in theta".
// Written independently of oracle/ (which uses the direct Lagrange product formula and the
// closed-form cardinal cot formula): here GL nodes come from a Newton iteration seeded by
// Tricomi's asymptotic formula, P_s from the barycentric (second) form, and F_th from the
// explicit real Fourier sum (reading R3).
#include <cmath>
#include <cstring>
#include <vector>
#include "common.cuh"

namespace slb {

void gl_nodes(int n, double* x, double* w) {
    // Legendre P_n and P_n' at z by the upward recurrence.
    auto legendre = [n](double z, double* pn, double* dpn) {
        double pm1 = 1.0, p = z;
        if (n == 0) { *pn = 1.0; *dpn = 0.0; return; }
        for (int k = 2; k <= n; ++k) {
            double pk = ((2 * k - 1) * z * p - (k - 1) * pm1) / k;
            pm1 = p;
            p = pk;
        }
        *pn = p;
        *dpn = n * (pm1 - z * p) / (1.0 - z * z);
    };
    for (int k = 1; k <= n; ++k) {
        // Tricomi: x_k ~ (1 - (n-1)/(8 n^3)) cos(pi (4k - 1) / (4n + 2)), k-th largest root
        double z = (1.0 - (n - 1.0) / (8.0 * n * n * n)) * std::cos(kPi * (4.0 * k - 1.0) / (4.0 * n + 2.0));
        double pn = 0, dpn = 1;
        for (int it = 0; it < 60; ++it) {
            legendre(z, &pn, &dpn);
            double dz = pn / dpn;
            z -= dz;
            if (std::fabs(dz) <= 1e-16 * (1.0 + std::fabs(z))) break;
        }
        legendre(z, &pn, &dpn);
        x[n - k] = z;                                   // ascending
        w[n - k] = 2.0 / ((1.0 - z * z) * dpn * dpn);
    }
}

void bary_matrix(int nf, const double* xs, int nt, const double* xt, double* P) {
    // barycentric weights lambda_i = 1 / prod_{l != i} (x_i - x_l)
    double lam[64];
    for (int i = 0; i < nf; ++i) {
        double p = 1.0;
        for (int l = 0; l < nf; ++l) if (l != i) p *= (xs[i] - xs[l]);
        lam[i] = 1.0 / p;
    }
    for (int m = 0; m < nt; ++m) {
        int hit = -1;
        for (int i = 0; i < nf; ++i) if (xt[m] == xs[i]) hit = i;
        if (hit >= 0) {
            for (int i = 0; i < nf; ++i) P[m * nf + i] = (i == hit) ? 1.0 : 0.0;
            continue;
        }
        double den = 0.0;
        for (int i = 0; i < nf; ++i) den += lam[i] / (xt[m] - xs[i]);
        for (int i = 0; i < nf; ++i) P[m * nf + i] = (lam[i] / (xt[m] - xs[i])) / den;
    }
}

void trig_matrix(int N, int M, double* F) {
    for (int b = 0; b < M; ++b)
        for (int j = 0; j < N; ++j) {
            double d = 2.0 * kPi * ((double)b / M - (double)j / N);
            double s = 1.0 + std::cos(0.5 * N * d);
            for (int l = 1; l < N / 2; ++l) s += 2.0 * std::cos(l * d);
            F[b * N + j] = s / N;
        }
}

bool make_interp(int ns, int nt, int ms, int mt, InterpParams* ip, double** owned) {
    if (ns < 1 || ms < 1 || nt < 2 || mt < 2 || (nt & 1) || ns > 64 || ms > 64) return false;
    ip->ns = ns; ip->nt = nt; ip->ms = ms; ip->mt = mt;
    ip->vg = nullptr;
    ip->mats_d = nullptr;
    double xs[64], ws[64], xf[64], wf[64];
    gl_nodes(ns, xs, ws);
    gl_nodes(ms, xf, wf);
    const int n = ms * ns + mt * nt;
    const bool fits = n <= kMaxInterp;
    if (fits) {
        bary_matrix(ns, xs, ms, xf, ip->v);
        trig_matrix(nt, mt, ip->v + ms * ns);
    }
    if (!owned) return fits;
    // device copy (always, when the caller can own one): the streaming upsample stages the matrices
    // from global memory; kernels that take them by value use it only when they exceed ip->v
    std::vector<double> h(n);
    bary_matrix(ns, xs, ms, xf, h.data());
    trig_matrix(nt, mt, h.data() + ms * ns);
    double* d = nullptr;
    if (cudaMalloc(&d, sizeof(double) * n) != cudaSuccess) return false;
    if (cudaMemcpy(d, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return false;
    }
    *owned = d;
    ip->mats_d = d;
    if (!fits) ip->vg = d;
    return true;
}

}  // namespace slb
