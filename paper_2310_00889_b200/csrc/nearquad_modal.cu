// nearquad_modal.cu -- (NEXT N1, setup) special-quadrature correction blocks by the paper's method.
//
// PAPER.md §3.2.2-3.2.4.  For a target x and an element Gamma_k the block is
//     B[r][(i,j,c)] = sum_m P_mi w_m h_j^{rc}(x, s_m)
// (the first term of the paper's E; the smooth-rule term -G w is folded in by the operator), with
//   * the ANGULAR integral done first (§3.2.2): at an s-node, the ring y(s, .) and the closest angle
//     th0 to x; an angular rule centred at th0 chosen by alpha = dist(x, ring) / ring radius
//     (P:L1111-1113); the modal sums (Eq. e:modal-greens-fn-coeff)
//         hhat_l = sum_m K(x - y(s, th_m)) J(s, th_m) omega_m e^{i l th_m},   l = 0 .. N/2
//     (hhat_{-l} = conj hhat_l) -- a GEMM over the rule's nodes on the FP64 tensor cores
//     (DMMA m8n8k4: rows = kernel components, K = angular nodes, columns = (cos, sin) of the modes) --
//     and the weights by the inverse DFT (Eq. e:modal-greens-fn-wts; R3's symmetric
//     Nyquist term): h_j = (1/N)[Re hhat_0 + 2 sum_{0<l<N/2} Re(hhat_l e^{-i l th_j}) + Re(hhat_{N/2} e^{-i N th_j/2})];
//   * the s integral (§3.2.3): off-surface targets -- adaptive Gauss-Legendre sub-panels of the element,
//     split until x lies outside the Bernstein rho = 2.5 ellipse of each sub-panel,
//     20 nodes per sub-panel (rho^-40 ~ 1e-16);
//   * on-surface (singular) targets (§3.2.4, the paper's panel fallback): sub-panels refined
//     dyadically towards s0 until they are ~rho/4 long, Gauss-Legendre on the panels not touching s0 and
//     a rule exact for p(s) log|s - s0| + q(s) (tools/gen_log_rule.py, nq_logrule.inc) on the two that do;
//   * P = barycentric Lagrange from the N_s GL nodes to the s-nodes, the block accumulated
//     as sum over s-nodes of (w_s l_i(s)) x h_j(s) (a rank-1 update per s-node).
// The paper's generalized-Chebyshev compression of the angular and singular rules (App. B) is replaced by
// the uncompressed rules it starts from: composite GL panels refined
// dyadically towards th0 down to the annulus size alpha (alpha < 1), the periodic trapezoidal rule with
// enough nodes for the strip of analyticity (alpha >= 1); the modes e^{i l th_m} are generated per node
// instead of stored with the rule.
// Accuracy detail: the target-to-surface vector is evaluated in difference form,
//     r = x - y(s, th) = sum_ij (x - y_ij) l_i(s) C_j(th),
// so its rounding error is eps |x - y_ij| ~ eps L, not eps |x|; for the element's own node the (i0, j0)
// term is exactly zero and l_i, C_j are evaluated to full relative accuracy from (s - s0, th - th0), so
// r is accurate relative to |r| arbitrarily close to the singular point (the double layer's (r.n)/|r|^3
// would otherwise turn eps |y| into an O(eps/|r|) error).
// One CTA per (target, element) pair, pairs handed out by an atomic counter (deterministic: each pair is
// computed by exactly one CTA in a fixed order).  Blocks: [tdim][N_s N_th sdim], unfolded B.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>
#include "common.cuh"

namespace slb {

#include "nq_logrule.inc"
#include "nq_chebrules.inc"

namespace nqm {

constexpr int kMaxNs = 32, kMaxNt = 64, kMaxL = kMaxNt / 2;
constexpr int kQs = 20;            // GL nodes per near-singular s sub-panel
constexpr int kQd = 16;            // GL nodes per dyadic panel of the singular s rule
constexpr int kQa = 16;            // GL nodes per angular panel
constexpr int kMaxSub = 160;       // s sub-panels per pair
constexpr int kNTrap = 6;          // trapezoidal brackets alpha in [2^j, 2^(j+1)), j = 0..5 (the last: alpha >= 32)
constexpr int kMaxK = 46;          // composite-GL brackets alpha in [2^-k, 2^(1-k)), k = 1..46
constexpr int kNRules = kNTrap + kMaxK;
constexpr int kNClass = 4;         // rule sets by N_th: <= 12, <= 24, <= 40, <= 64
constexpr int kChunk = 32;         // angular nodes per DMMA chunk
constexpr int kTri = kMaxNs * (kMaxNs + 1) / 2;
constexpr double kBernSum = 2.5 + 1.0 / 2.5;   // Bernstein rho = 2.5: |z - 1| + |z + 1| = rho + 1/rho

__host__ __device__ inline int lmax_of_class(int c) { return c == 0 ? 8 : c == 1 ? 14 : c == 2 ? 22 : 34; }
__host__ __device__ inline int class_of_nt(int nt) { return nt <= 12 ? 0 : nt <= 24 ? 1 : nt <= 40 ? 2 : 3; }

struct RuleSet {
    const double* th;              // angular nodes relative to th0
    const double* w;               // weights (0 on padding)
    const double* E;               // [node][lde]: cos(l th_m), sin(l th_m), l = 0 .. the class's largest N_th / 2
    int lde;
    int off[kNRules], cnt[kNRules];   // cnt: multiple of kChunk
};

struct Tables {
    double gx20[kQs], gw20[kQs], gx16[kQd], gw16[kQd];   // GL on [-1,1]
    double tgl[kTri], lam[kTri];                          // GL nodes / barycentric weights of every order <= 32
    RuleSet rs[kNClass];
};

struct Args {
    int kernel;                    // 1 Laplace D (+ eta S_L), 2 Stokes eta S + D, 3 Stokes eta S, 4 Laplace eta S_L
    int64_t T, nnz;
    const double* x;               // [T][3]
    const int64_t* trg_node;       // [T] or NULL
    const int64_t* row_ptr;        // [T+1]
    const int32_t* panel_idx;      // [nnz]
    const double* y;               // element nodes
    const int64_t* cn0;            // [P+1] first node of each element (NULL: uniform k ns nt)
    const int32_t* pns;            // [P] (NULL: uniform)
    const int32_t* pnt;
    int ns, nt;                    // uniform orders / launch maxima
    const int64_t* boff;           // [nnz+1] block offsets (NULL: p * blen)
    const double* eta_panel;       // [P] or NULL
    double eta_default, dl;
    double* blocks;
    unsigned long long* work;      // pair counter
    int* status;                   // 1: a pair exceeded the sub-panel budget
    int warps, ld_e;               // warps per CTA, E row stride
    double bern;                   // Bernstein sum rho + 1/rho of the s sub-panel test (rho = 2.5)
    int64_t p0, p1;                // this launch's pairs: plist[p0 .. p1) (plist NULL: the pair ids p0 .. p1)
    const int64_t* plist;
    double* pre;                   // [p1 - p0][4]: s-rule geometry from nq_srule_kernel (ts, dmin, |y_t|, rho)
    int64_t* prow;                 // [p1 - p0]: the pair's target row
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Lagrange basis l_i and derivative at s (n nodes tg, barycentric weights lam), with the node differences
// e_k = s - s_k computed as ds + (s0 - s_k) (ds = s - s0 exact for singular pairs, s0 = tg[i0]; i0 < 0: s0 = 0).
//   l_i = (lam_i / e_i) / sum_k (lam_k / e_k),    l_i' = l_i sum_{k != i} 1 / e_k   (l_i = prod_{k != i} ...)
// For singular pairs the i0 term is factored out (den' = lam_i0 + ds sum_{k != i0} lam_k / e_k = ds den), so
// l_i (i != i0) and l_i' keep full relative accuracy as ds -> 0 (no 1/ds - 1/ds cancellation).
__device__ void lagrange_bary(int n, const double* tg, const double* lam, double ds, int i0, double* l,
                              double* dl) {
    const double s0 = i0 >= 0 ? tg[i0] : 0.0;
    int hit = -1;
    for (int k = 0; k < n; ++k)
        if (ds + (s0 - tg[k]) == 0.0) hit = k;
    if (hit >= 0) {
        double sm = 0.0;
        for (int i = 0; i < n; ++i) {
            l[i] = i == hit ? 1.0 : 0.0;
            if (i != hit) {
                dl[i] = (lam[i] / lam[hit]) / (tg[hit] - tg[i]);
                sm += dl[i];
            }
        }
        dl[hit] = -sm;
        return;
    }
    if (i0 >= 0) {
        double den = 0.0, sinv = 0.0;                   // den' and sum_{k != i0} 1/e_k
        for (int k = 0; k < n; ++k) {
            if (k == i0) continue;
            const double e = ds + (s0 - tg[k]);
            den += lam[k] / e;
            sinv += 1.0 / e;
        }
        den = lam[i0] + ds * den;
        for (int i = 0; i < n; ++i) {
            if (i == i0) {
                l[i] = lam[i0] / den;
                dl[i] = l[i] * sinv;
            } else {
                const double e = ds + (s0 - tg[i]);
                const double q = (lam[i] / e) / den;    // = l_i / ds
                l[i] = q * ds;
                dl[i] = q + l[i] * (sinv - 1.0 / e);    // l_i (1/ds + sum_{k != i, i0} 1/e_k)
            }
        }
        return;
    }
    double den = 0.0, sinv = 0.0;
    for (int k = 0; k < n; ++k) {
        const double e = ds - tg[k];
        den += lam[k] / e;
        sinv += 1.0 / e;
    }
    for (int i = 0; i < n; ++i) {
        const double e = ds - tg[i];
        l[i] = (lam[i] / e) / den;
        dl[i] = l[i] * (sinv - 1.0 / e);
    }
}

// lagrange_bary with the n <= 32 nodes spread over the warp's lanes (lane i owns node i; the two sums by
// warp reductions).  Same formulas; only the summation order differs.
__device__ void lagrange_bary_warp(int lane, int n, const double* tg, const double* lam, double ds, int i0, double* l,
                                   double* dl) {
    const double s0 = i0 >= 0 ? tg[i0] : 0.0;
    const bool own = lane < n;
    const double e = own ? ds + (s0 - tg[lane]) : 1.0;
    const unsigned hitm = __ballot_sync(0xffffffffu, own && e == 0.0);
    if (hitm) {
        const int hit = 31 - __clz(hitm);                // the last such node (as the serial loop)
        double v = (own && lane != hit) ? (lam[lane] / lam[hit]) / (tg[hit] - tg[lane]) : 0.0;
        const double sm = wsum(v);
        if (own) {
            l[lane] = lane == hit ? 1.0 : 0.0;
            dl[lane] = lane == hit ? -sm : v;
        }
        return;
    }
    const bool term = own && lane != i0;                 // i0 < 0: every node
    const double den0 = wsum(term ? lam[lane] / e : 0.0);
    const double sinv = wsum(term ? 1.0 / e : 0.0);
    if (i0 >= 0) {
        const double den = lam[i0] + ds * den0;
        if (own) {
            if (lane == i0) {
                l[lane] = lam[i0] / den;
                dl[lane] = l[lane] * sinv;
            } else {
                const double q = (lam[lane] / e) / den;
                l[lane] = q * ds;
                dl[lane] = q + l[lane] * (sinv - 1.0 / e);
            }
        }
        return;
    }
    if (own) {
        l[lane] = (lam[lane] / e) / den0;
        dl[lane] = l[lane] * (sinv - 1.0 / e);
    }
}

// Cardinal C_j(th) and C_j'(th), th = th0 + dh (R3: C_N(phi) = sin(N phi/2) cot(phi/2) / N, phi = th - th_j).
// j0 >= 0 (singular pairs): th0 = th_{j0}, and the values are accurate RELATIVE to their size near th0:
//   * closer to th0 than to th_j (|dh| <= |phi|): sin(N phi/2) = (-1)^(j-j0) sin(N dh/2) from dh itself;
//   * j = j0, or phi small (near th_j): the Fourier sums C = (1 + 2 sum_l cos l phi + cos(N phi/2)) / N and
//     C' = -(2 sum_l l sin l phi + (N/2) sin(N phi/2)) / N (no N/phi - N/phi cancellation in C');
//   * otherwise the cot form with sin(N phi/2) evaluated directly.
__device__ __forceinline__ void cardinal_j(int N, int j, int j0, double th0, double dh, double sh, double ch,
                                           double* C, double* dC) {
    double phi = (j0 >= 0) ? dh + 2.0 * kPi * (double)(j0 - j) / N : (th0 + dh) - 2.0 * kPi * j / N;
    phi -= 2.0 * kPi * rint(phi / (2.0 * kPi));          // into (-pi, pi]; period 2 pi for even N
    double sp, cp;
    sincos(0.5 * phi, &sp, &cp);
    const bool near_j = fabs(sp) < 0.25 && (j0 < 0 || fabs(phi) < fabs(dh));
    if (j == j0 || near_j) {
        double s1, c1;
        sincos(phi, &s1, &c1);
        double cl = 1.0, sl = 0.0, v = 1.0, d = 0.0;
        for (int l = 1; l < N / 2; ++l) {
            const double cn = cl * c1 - sl * s1;
            sl = sl * c1 + cl * s1;
            cl = cn;
            v += 2.0 * cl;
            d -= 2.0 * l * sl;
        }
        const double cn = cl * c1 - sl * s1, sn = sl * c1 + cl * s1;   // l = N/2
        *C = (v + cn) / N;
        *dC = (d - 0.5 * N * sn) / N;
        return;
    }
    double sn, cn;
    if (j0 >= 0 && fabs(dh) <= fabs(phi)) {
        const double sg = ((j - j0) & 1) ? -1.0 : 1.0;
        sn = sg * sh;
        cn = sg * ch;
    } else {
        sincos(0.5 * N * phi, &sn, &cn);
    }
    const double cot = cp / sp;
    *C = sn * cot / N;
    *dC = (0.5 * N * cn * cot - 0.5 * sn / (sp * sp)) / N;
}

// Singular-pair form for a whole ring at once (j0 = the target's index, th = th_j0 + dh, |dh| < pi / N):
// sin(N phi_j / 2) = (-1)^(j - j0) sin(N dh / 2) and cot(phi_j / 2) = (cot b_j - t) / (1 + t cot b_j), with
// t = tan(dh / 2) and b_j = pi (j0 - j) / N, so each j costs one division and keeps full relative accuracy
// (|dh| < pi / N keeps every phi_j, j != j0, at least pi / N from 0); j = j0 takes the Fourier sums.
__device__ __forceinline__ void cardinal_ring_sing(int N, int j0, double dh, double sh, double ch, double t,
                                                   const double* scm, const double* D, const double* Dp,
                                                   double* r, double* rh, double* rs) {
    for (int c = 0; c < 3; ++c) { r[c] = 0.0; rh[c] = 0.0; rs[c] = 0.0; }
    for (int j = 0; j < N; ++j) {
        double C, dC;
        const int m = j0 - j;
        if (m == 0) {
            cardinal_j(N, j, j0, 0.0, dh, sh, ch, &C, &dC);
        } else {
            const double sb = scm[2 * (m + N - 1)], cb = scm[2 * (m + N - 1) + 1];   // sincospi(m / N)
            const double cotb = cb / sb;
            const double cot = (cotb - t) / (1.0 + t * cotb);          // cot((dh + 2 pi m / N) / 2)
            const double sg = (m & 1) ? -1.0 : 1.0;
            const double sn = sg * sh, cn = sg * ch;
            C = sn * cot / N;
            dC = (0.5 * N * cn * cot - 0.5 * sn * (1.0 + cot * cot)) / N;
        }
        for (int c = 0; c < 3; ++c) {
            r[c] += D[3 * j + c] * C;
            rh[c] += D[3 * j + c] * dC;
            rs[c] += Dp[3 * j + c] * C;
        }
    }
}

// The s-rule geometry of one (target, element) pair (one warp): for on-surface targets |y_t| and the ring
// radius |y_th| at the target node; otherwise the closest point (t*, th*) (the nearest node, then Gauss-Newton
// on |r(t, th)|^2 with t clamped to [-1, 1]), its distance and |y_t| there.  Dq: the element's nodes relative
// to the target ((i0, j0) zeroed for on-surface pairs); lg / dlg: the warp's Lagrange scratch.
__device__ void srule_geometry(int lane, int ns, int nt, const double* tg, const double* lam, const double* Dq,
                               double* lg, double* dlg, bool sing, int i0, int j0, double* out) {
    // geometry at (t, th): r = sum D_ij l_i C_j, r_t, r_th (warp-cooperative over j)
    auto eval_pt = [&](double t, double th, double* r, double* rt, double* rh) {
        lagrange_bary(ns, tg, lam, t, -1, lg, dlg);       // redundantly per lane (ns <= 32)
        double a[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int j = lane; j < nt; j += 32) {
            double C, dC;
            cardinal_j(nt, j, -1, th, 0.0, 0.0, 0.0, &C, &dC);
            double d[3] = {0, 0, 0}, dd[3] = {0, 0, 0};
            for (int i = 0; i < ns; ++i)
                for (int c = 0; c < 3; ++c) {
                    d[c] += Dq[3 * (i * nt + j) + c] * lg[i];
                    dd[c] += Dq[3 * (i * nt + j) + c] * dlg[i];
                }
            for (int c = 0; c < 3; ++c) {
                a[c] += d[c] * C;
                a[3 + c] += dd[c] * C;
                a[6 + c] += d[c] * dC;
            }
        }
        for (int c = 0; c < 3; ++c) {
            r[c] = wsum(a[c]);
            rt[c] = wsum(a[3 + c]);
            rh[c] = wsum(a[6 + c]);
        }
    };
    double ts = 0.0, hs = 0.0, dmin = 0.0, ytn = 1.0, rho = 1.0;
    if (sing) {
        double r[3], rt[3], rh[3];
        eval_pt(tg[i0], 2.0 * kPi * j0 / nt, r, rt, rh);
        ytn = sqrt(rt[0] * rt[0] + rt[1] * rt[1] + rt[2] * rt[2]);
        rho = sqrt(rh[0] * rh[0] + rh[1] * rh[1] + rh[2] * rh[2]);
        ts = tg[i0];
    } else {
        // closest point: the nearest node, then Gauss-Newton on |r(t, th)|^2 with t clamped to [-1, 1]
        double best = 1e300;
        int bq = 0;
        for (int q = lane; q < ns * nt; q += 32) {
            const double dd = Dq[3 * q] * Dq[3 * q] + Dq[3 * q + 1] * Dq[3 * q + 1] + Dq[3 * q + 2] * Dq[3 * q + 2];
            if (dd < best) { best = dd; bq = q; }
        }
        for (int o = 16; o; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
            if (ob < best || (ob == best && oq < bq)) { best = ob; bq = oq; }
        }
        ts = tg[bq / nt];
        hs = 2.0 * kPi * (bq % nt) / nt;
        double r[3], rt[3], rh[3];
        for (int it = 0; it < 40; ++it) {
            eval_pt(ts, hs, r, rt, rh);
            const double a11 = rt[0] * rt[0] + rt[1] * rt[1] + rt[2] * rt[2];
            const double a12 = rt[0] * rh[0] + rt[1] * rh[1] + rt[2] * rh[2];
            const double a22 = rh[0] * rh[0] + rh[1] * rh[1] + rh[2] * rh[2];
            // minimise |r|^2 with r = x - y: grad = 2 r.r_t, 2 r.r_h; GN step solves [a] delta = -(r.r_t, r.r_h)
            const double g1 = r[0] * rt[0] + r[1] * rt[1] + r[2] * rt[2];
            const double g2 = r[0] * rh[0] + r[1] * rh[1] + r[2] * rh[2];
            const double det = a11 * a22 - a12 * a12;
            double dt = -(a22 * g1 - a12 * g2) / det, dh = -(a11 * g2 - a12 * g1) / det;
            double tn = ts + dt;
            if (tn > 1.0 || tn < -1.0) {
                tn = tn > 1.0 ? 1.0 : -1.0;
                dh = -g2 / a22;
            }
            const double step = fabs(tn - ts) + fabs(dh);
            ts = tn;
            hs += dh;
            // the closest point only places the s sub-panels (Bernstein test) and sets dmin, which is
            // second order in the t error: 1e-12 is far below anything the partition can resolve
            // (a 1e-15 test never triggers when |hs| ~ pi rounds at ~4e-16 per step: 40 iterations)
            if (step < 1e-12) break;
        }
        eval_pt(ts, hs, r, rt, rh);
        dmin = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
        ytn = sqrt(rt[0] * rt[0] + rt[1] * rt[1] + rt[2] * rt[2]);
    }
    out[0] = ts; out[1] = dmin; out[2] = ytn; out[3] = rho;
}

// kernel matrix (rows a = target component, cols b = source component), times J omega
template <int KD>
__device__ __forceinline__ void kernel_vals(int kernel, const double r[3], const double n[3], double eta, double dl,
                                            double scale, double* V) {
    const double r2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
    const double ri = 1.0 / sqrt(r2);
    const double ri2 = ri * ri;
    const double rn = r[0] * n[0] + r[1] * n[1] + r[2] * n[2];
    if (KD == 1) {
        // Laplace: D = (r.n)/(4 pi |r|^3), S_L = 1/(4 pi |r|)
        const double d = (kernel == 4) ? 0.0 : rn * ri2 * ri;
        V[0] = (d + eta * ri) * (scale / (4.0 * kPi));
    } else {
        // Stokes: eta S + dl D, S = (I/|r| + r r^T/|r|^3)/(8 pi), D = (3/(4 pi)) (r.n) r r^T/|r|^5 (R1)
        const double a = eta * ri / (8.0 * kPi);
        const double b = eta * ri * ri2 / (8.0 * kPi) + dl * 3.0 / (4.0 * kPi) * rn * ri2 * ri2 * ri;
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int q = 0; q < 3; ++q) V[p * 3 + q] = ((p == q ? a : 0.0) + b * r[p] * r[q]) * scale;
    }
}

// shared memory layout (doubles) of one CTA
struct Smem {
    int ns, nt, W, ldE, rows, ldv;       // rows: DMMA rows (16 Stokes, 8 Laplace); ldv = rows + 4 (banks)
    size_t dq, bs, hb, wb, sub, trig, warp0, per_warp, total;
};

__host__ __device__ inline Smem smem_layout(int ns, int nt, int W, int ldE, int KD) {
    Smem S;
    S.ns = ns; S.nt = nt; S.W = W; S.ldE = ldE; S.rows = KD == 3 ? 16 : 8; S.ldv = S.rows + 4;
    const int kd2 = KD * KD, L = nt / 2;
    size_t o = 0;
    S.dq = o; o += (size_t)ns * nt * 3;                 // x - y_ij
    S.bs = o; o += (size_t)kd2 * ns * nt;               // block accumulator [r][i][j]
    S.hb = o; o += (size_t)W * kd2 * nt;                // h_j per warp slot
    S.wb = o; o += (size_t)W * ns;                      // w_s l_i(s) per warp slot
    S.sub = o; o += (size_t)kMaxSub * 3 + 8;            // sub-panels (a, b, type) + misc
    S.trig = o; o += (size_t)6 * nt;                   // sincospi(2q / nt), q < nt; sincospi(m / nt), |m| < nt
    o = (o + 1) & ~(size_t)1;
    S.warp0 = o;
    // per warp: ring D[nt][3], D'[nt][3], modes Rh[(L+1)][3][2], Rp[(L+1)][3][2], l[ns], dl[ns],
    //           V[kChunk][rows], the ghat staging [rows][ldE]
    size_t pw = (size_t)nt * 6 + (size_t)(L + 1) * 12 + 2 * ns + (size_t)kChunk * S.ldv + (size_t)S.rows * ldE;
    S.per_warp = (pw + 1) & ~(size_t)1;
    o += S.per_warp * W;
    S.total = o;
    return S;
}

// Pre-pass: the s-rule geometry of every pair of [p0, p1), one warp per pair (the Gauss-Newton closest point
// is serial per pair; done here at full occupancy instead of by one warp of the quadrature CTA while the
// others wait).  Per warp: the element's nodes relative to the target, Lagrange scratch.
__global__ void __launch_bounds__(128) nq_srule_kernel(const __grid_constant__ Args A, const __grid_constant__ Tables TB) {
    extern __shared__ __align__(16) double sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per_warp = A.ns * A.nt * 3 + 2 * A.ns;
    double* Dq = sm + (size_t)warp * per_warp;
    double* lg = Dq + A.ns * A.nt * 3;
    double* dlg = lg + A.ns;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t q = A.p0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; q < A.p1; q += nw) {
        const int64_t p = A.plist ? A.plist[q] : q;
        int64_t t = 0;
        if (lane == 0) {
            int64_t lo = 0, hi = A.T;                 // row t: row_ptr[t] <= p < row_ptr[t+1]
            while (hi - lo > 1) {
                const int64_t mid = (lo + hi) / 2;
                if (A.row_ptr[mid] <= p) lo = mid; else hi = mid;
            }
            t = lo;
        }
        t = __shfl_sync(0xffffffffu, t, 0);
        const int k = A.panel_idx[p];
        const int ns = A.pns ? A.pns[k] : A.ns, nt = A.pnt ? A.pnt[k] : A.nt;
        const int64_t n0 = A.cn0 ? A.cn0[k] : (int64_t)k * ns * nt;
        int i0 = -1, j0 = -1;
        const int64_t nd = A.trg_node ? A.trg_node[t] : -1;
        if (nd >= n0 && nd < n0 + (int64_t)ns * nt) {
            i0 = (int)((nd - n0) / nt);
            j0 = (int)((nd - n0) % nt);
        }
        const double x0 = A.x[3 * t], x1 = A.x[3 * t + 1], x2 = A.x[3 * t + 2];
        for (int q = lane; q < ns * nt; q += 32) {
            const double* yv = A.y + 3 * (n0 + q);
            Dq[3 * q] = x0 - yv[0];
            Dq[3 * q + 1] = x1 - yv[1];
            Dq[3 * q + 2] = x2 - yv[2];
        }
        __syncwarp();
        if (i0 >= 0 && lane == 0) {
            Dq[3 * (i0 * nt + j0)] = 0.0; Dq[3 * (i0 * nt + j0) + 1] = 0.0; Dq[3 * (i0 * nt + j0) + 2] = 0.0;
        }
        __syncwarp();
        double out[4];
        srule_geometry(lane, ns, nt, TB.tgl + ns * (ns - 1) / 2, TB.lam + ns * (ns - 1) / 2, Dq, lg, dlg, i0 >= 0,
                       i0, j0, out);
        if (lane == 0) {
            double* o = A.pre + 4 * (q - A.p0);
            o[0] = out[0]; o[1] = out[1]; o[2] = out[2]; o[3] = out[3];
            A.prow[q - A.p0] = t;
        }
        __syncwarp();
    }
}

// KD: kernel dimension (1 Laplace, 3 Stokes); NCT: 8-column DMMA tiles of the modal sums (covers the
// launch's largest N_th: 2 (N_th/2 + 1) columns), so the accumulators are sized per rule class.
template <int KD, int NCT>
__global__ void __launch_bounds__(256) nq_modal_kernel(const __grid_constant__ Args A, const __grid_constant__ Tables TB) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int64_t s_pair, s_q;
    __shared__ int s_info[8];
    __shared__ double s_real[16];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = A.warps;
    constexpr int kd2 = KD * KD;
    const int g = lane >> 2, tq = lane & 3;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const int64_t q = A.p0 + (int64_t)atomicAdd(A.work, 1ull);
            s_q = q;
            s_pair = q < A.p1 ? (A.plist ? A.plist[q] : q) : -1;
        }
        __syncthreads();
        const int64_t p = s_pair, qi = s_q - A.p0;      // qi: index into the pre-pass arrays
        if (p < 0) return;
        // ------------------------------------------------ pair setup
        if (threadIdx.x == 0) {
            const int64_t t = A.prow[qi];
            const int k = A.panel_idx[p];
            const int ns = A.pns ? A.pns[k] : A.ns, nt = A.pnt ? A.pnt[k] : A.nt;
            const int64_t n0 = A.cn0 ? A.cn0[k] : (int64_t)k * ns * nt;
            int i0 = -1, j0 = -1;
            const int64_t nd = A.trg_node ? A.trg_node[t] : -1;
            if (nd >= n0 && nd < n0 + (int64_t)ns * nt) {
                i0 = (int)((nd - n0) / nt);
                j0 = (int)((nd - n0) % nt);
            }
            s_info[0] = (int)t; s_info[1] = k; s_info[2] = ns; s_info[3] = nt; s_info[4] = i0; s_info[5] = j0;
            s_info[6] = (int)(t >> 31);
            s_real[0] = A.x[3 * t]; s_real[1] = A.x[3 * t + 1]; s_real[2] = A.x[3 * t + 2];
            s_real[3] = A.eta_panel ? A.eta_panel[k] : A.eta_default;
            reinterpret_cast<int64_t*>(s_real)[4] = n0;
        }
        __syncthreads();
        const int ns = s_info[2], nt = s_info[3], i0 = s_info[4], j0 = s_info[5];
        const bool sing = i0 >= 0;
        const double x0 = s_real[0], x1 = s_real[1], x2 = s_real[2], eta = s_real[3];
        const int64_t n0 = reinterpret_cast<const int64_t*>(s_real)[4];
        const int L = nt / 2;
        const Smem S = smem_layout(A.ns, A.nt, W, A.ld_e, KD);
        double* Dq = sm + S.dq;
        double* Bs = sm + S.bs;
        double* Hb = sm + S.hb;
        double* Wb = sm + S.wb;
        double* Sub = sm + S.sub;
        double* cs2 = sm + S.trig;               // [nt][2]: sincospi(2 q / nt) = (sin, cos)(2 pi q / nt)
        double* scm = cs2 + 2 * nt;              // [2 nt - 1][2]: sincospi(m / nt), m = 1 - nt .. nt - 1
        double* wbase = sm + S.warp0 + (size_t)warp * S.per_warp;
        double* Dr = wbase;                      // [nt][3]
        double* Dp = Dr + nt * 3;                // [nt][3]
        double* Rh = Dp + nt * 3;                // [(L+1)][3][2]
        double* Rp = Rh + (L + 1) * 6;           // [(L+1)][3][2]
        double* lg = Rp + (L + 1) * 6;           // [ns]
        double* dlg = lg + ns;                   // [ns]
        // V [kChunk][ldv] and E [kChunk][ldE] sit after the ring buffers sized for the launch maxima
        double* Vb = wbase + (size_t)A.nt * 6 + (size_t)(A.nt / 2 + 1) * 12 + 2 * A.ns;
        double* Eb = Vb + kChunk * S.ldv;
        const double* tg = TB.tgl + ns * (ns - 1) / 2;
        const double* lam = TB.lam + ns * (ns - 1) / 2;
        const RuleSet& RS = TB.rs[class_of_nt(nt)];
        const int ncol = 2 * (L + 1), nct = (ncol + 7) / 8;     // <= NCT
        constexpr int NRT = KD == 3 ? 2 : 1;                  // 8-row DMMA tiles (9 kernel components -> 16 rows)
        const int nrt = NRT;
        // element nodes relative to the target; block accumulator
        for (int q = threadIdx.x; q < ns * nt; q += blockDim.x) {
            const double* yv = A.y + 3 * (n0 + q);
            Dq[3 * q] = x0 - yv[0];
            Dq[3 * q + 1] = x1 - yv[1];
            Dq[3 * q + 2] = x2 - yv[2];
        }
        for (int q = threadIdx.x; q < kd2 * ns * nt; q += blockDim.x) Bs[q] = 0.0;
        for (int q = threadIdx.x; q < nt; q += blockDim.x) sincospi(2.0 * (double)q / nt, &cs2[2 * q], &cs2[2 * q + 1]);
        for (int q = threadIdx.x; q < 2 * nt - 1; q += blockDim.x)
            sincospi((double)(q - (nt - 1)) / nt, &scm[2 * q], &scm[2 * q + 1]);
        for (int q = lane; q < kChunk * S.ldv; q += 32) Vb[q] = 0.0;        // padded rows stay zero
        __syncthreads();
        if (sing && threadIdx.x == 0) {
            Dq[3 * (i0 * nt + j0)] = 0.0; Dq[3 * (i0 * nt + j0) + 1] = 0.0; Dq[3 * (i0 * nt + j0) + 2] = 0.0;
        }
        __syncthreads();
        // ------------------------------------------------ s rule (warp 0, from the pre-pass geometry)
        if (warp == 0) {
            const double* pg = A.pre + 4 * qi;
            const double ts = pg[0], dmin = pg[1], ytn = pg[2], rho = pg[3];
            if (lane == 0) {
                int nsub = 0, over = 0;
                auto push = [&](double a, double b, int type) {
                    if (nsub < kMaxSub) {
                        Sub[3 * nsub] = a; Sub[3 * nsub + 1] = b; Sub[3 * nsub + 2] = type;
                        ++nsub;
                    } else {
                        over = 1;
                    }
                };
                if (sing) {
                    // dyadic towards s0 down to ~rho/4 (parameter units), log rule on the two touching panels;
                    // the singular sub-panels store the OFFSET from s0 (exact near s0)
                    // log panel length: the s-structure of h_j near s0 lives on the scale rho / (N_th |y_s|)
                    // (C_j oscillates N_th / 2 times), so the panel shrinks with N_th (0.25 rho / |y_t| at N_th = 12)
                    const double hl = fmin(0.25, 3.0 / nt) * rho / ytn;
                    // left: offsets -(1 + s0) ... 0
                    {
                        double len = 1.0 + ts;
                        double e[64];
                        int ne = 0;
                        e[ne++] = -len;
                        double h = len;
                        while (h > hl && ne < 60) { h *= 0.5; e[ne++] = -h; }
                        for (int q = 0; q + 1 < ne; ++q) push(e[q], e[q + 1], 1);
                        push(e[ne - 1], 0.0, 3);                 // singular end at b = 0
                    }
                    {
                        double len = 1.0 - ts;
                        double e[64];
                        int ne = 0;
                        double h = len;
                        while (h > hl && ne < 60) { h *= 0.5; e[ne++] = h; }   // descending offsets
                        push(0.0, ne ? e[ne - 1] : len, 2);       // singular end at a = 0
                        for (int q = ne - 1; q > 0; --q) push(e[q], e[q - 1], 1);
                        if (ne) push(e[0], len, 1);
                    }
                } else {
                    // Bernstein rho = 2.5 test of the target's complex position ts + i d / |y_t|
                    const double del = dmin / ytn;
                    const double lim = A.bern;
                    double stk[2 * 64];
                    int top = 0;
                    stk[0] = -1.0; stk[1] = 1.0; top = 1;
                    while (top > 0) {
                        --top;
                        const double a = stk[2 * top], b = stk[2 * top + 1];
                        const double h = 0.5 * (b - a);
                        const double zr = (ts - 0.5 * (a + b)) / h, zi = del / h;
                        const double s1 = sqrt((zr - 1) * (zr - 1) + zi * zi) + sqrt((zr + 1) * (zr + 1) + zi * zi);
                        if (s1 >= lim || h < 1e-14 || top >= 62) {
                            push(a, b, 0);
                        } else {
                            const double m = 0.5 * (a + b);
                            stk[2 * top] = m; stk[2 * top + 1] = b; ++top;       // right below left
                            stk[2 * top] = a; stk[2 * top + 1] = m; ++top;
                        }
                    }
                }
                s_info[7] = nsub;
                if (over) atomicOr(A.status, 1);
            }
        }
        __syncthreads();
        const int nsub = s_info[7];

        // s-node count and the prefix of each sub-panel (every thread, from shared memory)
        auto nodes_of = [&](int type) { return type == 0 ? kQs : type == 1 ? kQd : kLogRuleN; };
        int nsn = 0;
        for (int q = 0; q < nsub; ++q) nsn += nodes_of((int)Sub[3 * q + 2]);
        // ------------------------------------------------ s-node batches: warp w takes node b0 + w
        for (int b0 = 0; b0 < nsn; b0 += W) {
            const int sn = b0 + warp;
            double* hw = Hb + (size_t)warp * kd2 * nt;
            double* ww = Wb + (size_t)warp * ns;
            if (sn < nsn) {
                // locate the sub-panel
                int q = 0, base = 0;
                while (base + nodes_of((int)Sub[3 * q + 2]) <= sn) { base += nodes_of((int)Sub[3 * q + 2]); ++q; }
                const int m = sn - base, type = (int)Sub[3 * q + 2];
                const double a = Sub[3 * q], b = Sub[3 * q + 1];
                double ds, wsn;              // ds: s - s0 (singular) or s itself
                if (type == 0) { ds = 0.5 * (a + b) + 0.5 * (b - a) * TB.gx20[m]; wsn = 0.5 * (b - a) * TB.gw20[m]; }
                else if (type == 1) { ds = 0.5 * (a + b) + 0.5 * (b - a) * TB.gx16[m]; wsn = 0.5 * (b - a) * TB.gw16[m]; }
                else if (type == 2) { ds = a + (b - a) * c_logrule_u[m]; wsn = (b - a) * c_logrule_w[m]; }
                else { ds = b - (b - a) * c_logrule_u[m]; wsn = (b - a) * c_logrule_w[m]; }
                // Lagrange basis at s (relative differences for singular pairs)
                lagrange_bary_warp(lane, ns, tg, lam, ds, sing ? i0 : -1, lg, dlg);
                __syncwarp();
                // ring D_j(s) = sum_i (x - y_ij) l_i(s), D'_j = sum_i (x - y_ij) l_i'(s)
                for (int e = lane; e < nt * 3; e += 32) {
                    const int j = e / 3, c = e % 3;
                    double v = 0.0, dv = 0.0;
                    for (int i = 0; i < ns; ++i) {
                        const double dq = Dq[3 * (i * nt + j) + c];
                        v += dq * lg[i];
                        dv += dq * dlg[i];
                    }
                    Dr[e] = v;
                    Dp[e] = dv;
                }
                for (int i = lane; i < ns; i += 32) ww[i] = wsn * lg[i];
                __syncwarp();
                // modes of the ring (non-singular geometry): Rh_l = (1/N) sum_j D_j e^{-i l th_j}
                int leff = 0;
                double th0 = 0.0, dist = 0.0, rr = 1.0;
                {
                    for (int e = lane; e < (L + 1) * 6; e += 32) {
                        const int l = e / 6, c = (e % 6) >> 1, im = e & 1, wh = 0;
                        (void)wh;
                        double v = 0.0, dv = 0.0;
                        for (int j = 0; j < nt; ++j) {
                            const int q2 = (l * j) % nt;
                            const double f = im ? -cs2[2 * q2] : cs2[2 * q2 + 1];
                            v += Dr[3 * j + c] * f;
                            dv += Dp[3 * j + c] * f;
                        }
                        Rh[e] = v / nt;
                        Rp[e] = dv / nt;
                    }
                    __syncwarp();
                    // significant modes (a circle: l <= 1)
                    // (fmax is exact, so the lane-parallel maxima equal the serial ones)
                    double mx = 0.0;
                    for (int e = lane; e < (L + 1) * 6; e += 32) mx = fmax(mx, fmax(fabs(Rh[e]), fabs(Rp[e])));
#pragma unroll
                    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    int lhi = 0;
                    for (int l = lane; l <= L; l += 32) {
                        double v = 0.0;
                        for (int e = 0; e < 6; ++e) v = fmax(v, fmax(fabs(Rh[6 * l + e]), fabs(Rp[6 * l + e])));
                        if (v > 1e-17 * mx) lhi = l;
                    }
                    leff = __reduce_max_sync(0xffffffffu, lhi);
                }
                if (!sing) {
                    // closest angle: 64 samples, then Newton on f = |r|^2 / 2 (all lanes, redundantly)
                    auto ring = [&](double th, double* r, double* rh, double* rhh) {
                        for (int c = 0; c < 3; ++c) { r[c] = Rh[c * 2]; rh[c] = 0.0; rhh[c] = 0.0; }
                        double s1, c1;
                        sincos(th, &s1, &c1);
                        double cl = 1.0, sl = 0.0;
                        for (int l = 1; l <= leff; ++l) {
                            const double cn = cl * c1 - sl * s1;
                            sl = sl * c1 + cl * s1;
                            cl = cn;
                            const double f = (2 * l == nt) ? 1.0 : 2.0;
                            for (int c = 0; c < 3; ++c) {
                                const double re = Rh[6 * l + 2 * c], im = Rh[6 * l + 2 * c + 1];
                                // Re((re + i im) e^{i l th}) = re cl - im sl
                                r[c] += f * (re * cl - im * sl);
                                rh[c] += f * l * (-re * sl - im * cl);
                                rhh[c] += f * l * l * (-re * cl + im * sl);
                            }
                        }
                    };
                    double best = 1e300, bth = 0.0;
                    for (int q2 = lane; q2 < 64; q2 += 32) {
                        const double th = 2.0 * kPi * q2 / 64.0;
                        double r[3], rh[3], rhh[3];
                        ring(th, r, rh, rhh);
                        const double dd = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
                        if (dd < best) { best = dd; bth = th; }
                    }
                    for (int o = 16; o; o >>= 1) {
                        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                        const double oth = __shfl_xor_sync(0xffffffffu, bth, o);
                        if (ob < best || (ob == best && oth < bth)) { best = ob; bth = oth; }
                    }
                    th0 = bth;
                    for (int it = 0; it < 30; ++it) {
                        double r[3], rh[3], rhh[3];
                        ring(th0, r, rh, rhh);
                        const double f1 = r[0] * rh[0] + r[1] * rh[1] + r[2] * rh[2];
                        const double f2 = rh[0] * rh[0] + rh[1] * rh[1] + rh[2] * rh[2] + r[0] * rhh[0] + r[1] * rhh[1] +
                                          r[2] * rhh[2];
                        double step = f2 > 0.0 ? -f1 / f2 : -f1 / (rh[0] * rh[0] + rh[1] * rh[1] + rh[2] * rh[2]);
                        const double lim2 = 0.5;
                        step = fmax(-lim2, fmin(lim2, step));
                        th0 += step;
                        if (fabs(step) < 1e-13) break;     // Newton: the remaining error is ~step^2
                    }
                    double r[3], rh[3], rhh[3];
                    ring(th0, r, rh, rhh);
                    dist = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
                    rr = sqrt(rh[0] * rh[0] + rh[1] * rh[1] + rh[2] * rh[2]);
                } else {
                    th0 = 2.0 * kPi * j0 / nt;
                    // r(th_j0) = D_j0; |r_th(th_j0)| with C_j'(th_k) = (-1)^(k-j) cot(pi (k - j)/N) / 2
                    double rh[3] = {0, 0, 0};
                    for (int j = 0; j < nt; ++j) {
                        if (j == j0) continue;
                        const double sg = ((j0 - j) & 1) ? -1.0 : 1.0;
                        const double sp = scm[2 * (j0 - j + nt - 1)], cp = scm[2 * (j0 - j + nt - 1) + 1];
                        const double dc = 0.5 * sg * cp / sp;
                        for (int c = 0; c < 3; ++c) rh[c] += Dr[3 * j + c] * dc;
                    }
                    dist = sqrt(Dr[3 * j0] * Dr[3 * j0] + Dr[3 * j0 + 1] * Dr[3 * j0 + 1] + Dr[3 * j0 + 2] * Dr[3 * j0 + 2]);
                    rr = sqrt(rh[0] * rh[0] + rh[1] * rh[1] + rh[2] * rh[2]);
                }
                // angular rule by alpha = dist / ring radius
                const double alpha = dist / rr;
                int rule;
                if (alpha >= 1.0) rule = min(kNTrap - 1, (int)floor(log2(alpha)));
                else rule = kNTrap - 1 + min(kMaxK, (int)floor(-log2(fmax(alpha, 1e-300))) + 1);
                const int roff = RS.off[rule], rcnt = RS.cnt[rule];

                // DMMA accumulators: hhat[row][col], col = 2 l + (0: cos, 1: sin)
                double acc[NRT][NCT][2];
#pragma unroll
                for (int a2 = 0; a2 < NRT; ++a2)
#pragma unroll
                    for (int c2 = 0; c2 < NCT; ++c2) acc[a2][c2][0] = acc[a2][c2][1] = 0.0;
                for (int c0 = 0; c0 < rcnt; c0 += kChunk) {
                    // node lane: geometry, kernel, modes
                    {
                        const double dh = RS.th[roff + c0 + lane], wq = RS.w[roff + c0 + lane];
                        double V[9];
                        double r[3], rh[3], rs[3];
                        const double th = th0 + dh;
                        double s1, c1;
                        sincos(th, &s1, &c1);
                        if (wq != 0.0) {
                            // the element's own node: relative-accuracy nodal geometry only where r is small
                            // (close ring and |dh| < 1); elsewhere the modes are accurate to eps |r|
                            // (within half a node spacing of th_j0: there every other j has |phi_j| > |dh|;
                            // beyond it |r| > ~rho pi / N and the modal form is accurate to ~eps N)
                            const bool nodal = sing && alpha < 0.5 && fabs(dh) < kPi / nt;
                            if (!nodal) {
                                for (int c = 0; c < 3; ++c) { r[c] = Rh[2 * c]; rh[c] = 0.0; rs[c] = Rp[2 * c]; }
                                double cl = 1.0, sl = 0.0;
                                for (int l = 1; l <= leff; ++l) {
                                    const double cn = cl * c1 - sl * s1;
                                    sl = sl * c1 + cl * s1;
                                    cl = cn;
                                    const double f = (2 * l == nt) ? 1.0 : 2.0;
                                    for (int c = 0; c < 3; ++c) {
                                        const double re = Rh[6 * l + 2 * c], im = Rh[6 * l + 2 * c + 1];
                                        r[c] += f * (re * cl - im * sl);
                                        rh[c] += f * l * (-re * sl - im * cl);
                                        const double pre = Rp[6 * l + 2 * c], pim = Rp[6 * l + 2 * c + 1];
                                        rs[c] += f * (pre * cl - pim * sl);
                                    }
                                }
                            } else {
                                double sh, ch;
                                sincos(0.5 * nt * dh, &sh, &ch);
                                cardinal_ring_sing(nt, j0, dh, sh, ch, tan(0.5 * dh), scm, Dr, Dp, r, rh, rs);
                            }
                            // y = x - r: y_th x y_s = r_th x r_s (outward, R8); J = |.|, n = ./J
                            const double cx = rh[1] * rs[2] - rh[2] * rs[1];
                            const double cy = rh[2] * rs[0] - rh[0] * rs[2];
                            const double cz = rh[0] * rs[1] - rh[1] * rs[0];
                            const double J = sqrt(cx * cx + cy * cy + cz * cz);
                            const double nv[3] = {cx / J, cy / J, cz / J};
                            kernel_vals<KD>(A.kernel, r, nv, eta, A.dl, J * wq, V);
                        } else {
#pragma unroll
                            for (int e = 0; e < 9; ++e) V[e] = 0.0;
                        }
                        double* vr = Vb + lane * S.ldv;
#pragma unroll
                        for (int e = 0; e < kd2; ++e) vr[e] = V[e];
                    }
                    __syncwarp();
                    // ghat[row][col] += sum_m V[m][row] E[m][col], E = the rule's stored modes e^{i l th_m} (th_m
                    // relative to th0; the rotation by e^{i l th0} is applied in the inverse DFT)
                    const double* Et = RS.E + (size_t)(roff + c0) * RS.lde;
#pragma unroll
                    for (int k0 = 0; k0 < kChunk; k0 += 4) {
                        const int mrow = k0 + tq;
                        double av[NRT];
#pragma unroll
                        for (int rt = 0; rt < NRT; ++rt) av[rt] = Vb[mrow * S.ldv + 8 * rt + g];
#pragma unroll
                        for (int ct = 0; ct < NCT; ++ct) {
                            if (ct < nct) {
                                const double bv = __ldg(Et + (size_t)mrow * RS.lde + 8 * ct + g);
#pragma unroll
                                for (int rt = 0; rt < NRT; ++rt) dmma(acc[rt][ct][0], acc[rt][ct][1], av[rt], bv);
                            }
                        }
                    }
                    __syncwarp();
                }
                // stage ghat in Eb as [row][ld_e], then the inverse DFT h_j (Eq. e:modal-greens-fn-wts) of
                // hhat_l = e^{i l th0} ghat_l: Re(hhat_l e^{-i l th_j}) = Re(ghat_l e^{-i l (th_j - th0)})
#pragma unroll
                for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
                    for (int ct = 0; ct < NCT; ++ct)
                        if (ct < nct) {
                            Eb[(8 * rt + g) * A.ld_e + 8 * ct + 2 * tq] = acc[rt][ct][0];
                            Eb[(8 * rt + g) * A.ld_e + 8 * ct + 2 * tq + 1] = acc[rt][ct][1];
                        }
                __syncwarp();
                double st0, ct0;
                sincos(th0, &st0, &ct0);
                for (int e = lane; e < kd2 * nt; e += 32) {
                    const int row = e / nt, j = e % nt;
                    const double* hh = Eb + row * A.ld_e;
                    const double sj = cs2[2 * j] * ct0 - cs2[2 * j + 1] * st0;      // sin(th_j - th0)
                    const double cj = cs2[2 * j + 1] * ct0 + cs2[2 * j] * st0;      // cos(th_j - th0)
                    double cl = 1.0, sl = 0.0, v = hh[0];
                    for (int l = 1; l <= L; ++l) {
                        const double cn = cl * cj - sl * sj;
                        sl = sl * cj + cl * sj;
                        cl = cn;
                        const double f = (2 * l == nt) ? 1.0 : 2.0;
                        v += f * (hh[2 * l] * cl + hh[2 * l + 1] * sl);
                    }
                    hw[e] = v / nt;
                }
            } else {
                for (int e = lane; e < kd2 * nt; e += 32) hw[e] = 0.0;
                for (int i = lane; i < ns; i += 32) ww[i] = 0.0;
            }
            __syncthreads();
            // B[row][i][j] += sum_w h_w[row][j] (w_s l_i)_w
            for (int e = threadIdx.x; e < kd2 * ns * nt; e += blockDim.x) {
                const int row = e / (ns * nt), i = (e / nt) % ns, j = e % nt;
                double v = Bs[e];
                for (int w2 = 0; w2 < W; ++w2) v += Hb[((size_t)w2 * kd2 + row) * nt + j] * Wb[(size_t)w2 * ns + i];
                Bs[e] = v;
            }
            __syncthreads();
        }
        // ------------------------------------------------ write the block [a][(i nt + j) KD + b]
        const int64_t bo = A.boff ? A.boff[p] : p * (int64_t)kd2 * ns * nt;
        for (int e = threadIdx.x; e < kd2 * ns * nt; e += blockDim.x) {
            const int row = e / (ns * nt), i = (e / nt) % ns, j = e % nt;
            const int a = row / KD, b = row % KD;
            A.blocks[bo + (int64_t)a * (ns * nt * KD) + (int64_t)(i * nt + j) * KD + b] = Bs[e];
        }
    }
}

// ------------------------------------------------------------------ host: rule tables, launch
struct RuleBuf {
    double* th = nullptr;
    double* w = nullptr;
    double* E = nullptr;
    int lde = 0;
    int off[kNRules], cnt[kNRules];
};

// Angular rules for modes up to lmax (the rules the paper's generalized-Chebyshev tables
// are built from):
//   j < kNTrap (alpha in [2^j, 2^(j+1))): periodic trapezoidal rule, M >= 37 / a + 2 lmax + 2 nodes, a =
//     acosh(1 + alpha^2 / (2 (1 + alpha))) the half-width of the strip of analyticity of G(x, y(th)) for a
//     circle of radius 1 and a target at distance alpha (e^{-a M} < 1e-16 after the modes);
//   k >= 1 (alpha in [2^-k, 2^(1-k))): 16-point GL on panels [0, 2^-k], [2^-k, 2^(1-k)], ... up to pi,
//     no panel longer than 16 / lmax (resolves e^{i lmax th}), mirrored to [-pi, 0].
// Every rule is padded with zero-weight nodes to a multiple of kChunk.
static void build_rules(int cls, int lmax, std::vector<double>& th, std::vector<double>& w, int* off, int* cnt) {
    static const bool composite = [] { const char* e = getenv("SLB_NQ_COMPOSITE"); return e && e[0] == '1'; }();
    double gx[kQa], gw[kQa];
    gl_nodes(kQa, gx, gw);
    auto pad = [&](int start) {
        while ((th.size() - start) % kChunk) { th.push_back(0.0); w.push_back(0.0); }
    };
    for (int j = 0; j < kNTrap; ++j) {
        const double al = std::ldexp(1.0, j);
        const double a = std::acosh(1.0 + al * al / (2.0 * (1.0 + al)));
        const int M = (int)std::ceil(37.0 / a) + 2 * lmax + 2;
        const int start = (int)th.size();
        off[j] = start;
        for (int m = 0; m < M; ++m) {
            th.push_back(2.0 * kPi * (m - M / 2) / M);
            w.push_back(2.0 * kPi / M);
        }
        pad(start);
        cnt[j] = (int)th.size() - start;
    }
    const double hcap = 16.0 / lmax;
    for (int k = 1; k <= kMaxK; ++k) {
        if (!composite && k <= kChebK && c_cheb_rule[cls][k - 1][1] > 0) {
            // the generalized Chebyshev rule of this class and bracket (App. B; tools/gen_cheb_rules.py), built on
            // (0, pi) for the even integrands and mirrored
            const int o = c_cheb_rule[cls][k - 1][0], n = c_cheb_rule[cls][k - 1][1];
            const int start = (int)th.size();
            off[kNTrap - 1 + k] = start;
            for (int sgn = -1; sgn <= 1; sgn += 2)
                for (int j = 0; j < n; ++j) {
                    th.push_back(sgn * c_cheb_th[o + j]);
                    w.push_back(c_cheb_w[o + j]);
                }
            pad(start);
            cnt[kNTrap - 1 + k] = (int)th.size() - start;
            continue;
        }
        const double al = std::ldexp(1.0, -k);
        std::vector<double> e{0.0, al};
        while (e.back() * 2.0 < kPi) e.push_back(e.back() * 2.0);
        if (kPi - e.back() < 0.25 * e.back()) e.back() = kPi; else e.push_back(kPi);
        std::vector<double> ed{0.0};
        for (size_t q = 1; q < e.size(); ++q) {
            const double len = e[q] - e[q - 1];
            const int np = std::max(1, (int)std::ceil(len / hcap - 1e-12));
            for (int r = 1; r <= np; ++r) ed.push_back(e[q - 1] + len * r / np);
        }
        ed.back() = kPi;
        const int start = (int)th.size();
        off[kNTrap - 1 + k] = start;
        for (int sgn = -1; sgn <= 1; sgn += 2)
            for (size_t q = 1; q < ed.size(); ++q) {
                const double c = 0.5 * (ed[q] + ed[q - 1]), h = 0.5 * (ed[q] - ed[q - 1]);
                for (int m = 0; m < kQa; ++m) {
                    th.push_back(sgn * (c + h * gx[m]));
                    w.push_back(h * gw[m]);
                }
            }
        pad(start);
        cnt[kNTrap - 1 + k] = (int)th.size() - start;
    }
}

static const RuleBuf* rules_for_class(int c) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, RuleBuf> cache;       // (device, class)
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, c});
    if (it != cache.end()) return &it->second;
    RuleBuf rb;
    std::vector<double> th, w;
    build_rules(c, lmax_of_class(c), th, w, rb.off, rb.cnt);
    // stored modes of every node ("precomputed and stored along with the quadrature rule")
    const int Lc = (c == 0 ? 12 : c == 1 ? 24 : c == 2 ? 40 : 64) / 2;
    rb.lde = (2 * (Lc + 1) + 7) / 8 * 8;
    std::vector<double> E(th.size() * rb.lde, 0.0);
    for (size_t m = 0; m < th.size(); ++m)
        for (int l = 0; 2 * l + 1 < rb.lde; ++l) {
            E[m * rb.lde + 2 * l] = std::cos(l * th[m]);
            E[m * rb.lde + 2 * l + 1] = std::sin(l * th[m]);
        }
    if (cudaMalloc(&rb.E, sizeof(double) * E.size()) != cudaSuccess ||
        cudaMemcpy(rb.E, E.data(), sizeof(double) * E.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return nullptr;
    if (cudaMalloc(&rb.th, sizeof(double) * th.size()) != cudaSuccess) return nullptr;
    if (cudaMalloc(&rb.w, sizeof(double) * w.size()) != cudaSuccess) { cudaFree(rb.th); return nullptr; }
    if (cudaMemcpy(rb.th, th.data(), sizeof(double) * th.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(rb.w, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(rb.th);
        cudaFree(rb.w);
        return nullptr;
    }
    return &(cache[{dev, c}] = rb);
}

}  // namespace nqm

// The paper's rule (order == 0 in slb_nearcorr_quad[_ragged]).  ns_max / nt_max: the launch's largest
// element; pns / pnt / cn0 / boff: device tables for ragged orders (NULL: uniform ns, nt).
slb_status nearquad_modal_run(slb_kernel kernel, int64_t n_trg, const double* x_trg, const int64_t* trg_node,
                              const int64_t* row_ptr, const int32_t* panel_idx, int ns_max, int nt_max,
                              const double* y_coarse, const double* eta_panel, double* blocks, cudaStream_t s,
                              const int32_t* pnt, const int64_t* cn0, const int64_t* boff, const int32_t* pns,
                              int ns_uniform, int nt_uniform) {
    using namespace nqm;
    SLB_REQUIRE(ns_max <= kMaxNs && nt_max <= kMaxNt, SLB_ERR_UNSUPPORTED, "nearquad (modal): element too large");
    std::unique_ptr<Tables> tb(new Tables);
    gl_nodes(kQs, tb->gx20, tb->gw20);
    gl_nodes(kQd, tb->gx16, tb->gw16);
    double w[kMaxNs];
    for (int n = 1; n <= kMaxNs; ++n) {
        double* tg = tb->tgl + n * (n - 1) / 2;
        double* lm = tb->lam + n * (n - 1) / 2;
        gl_nodes(n, tg, w);
        double mx = 0.0;
        for (int i = 0; i < n; ++i) {
            double pr = 1.0;
            for (int l = 0; l < n; ++l) if (l != i) pr *= (tg[i] - tg[l]);
            lm[i] = 1.0 / pr;
            mx = std::max(mx, std::fabs(lm[i]));
        }
        for (int i = 0; i < n; ++i) lm[i] /= mx;           // barycentric weights are defined up to scale
    }
    for (int c = 0; c < kNClass; ++c) {
        const RuleBuf* rb = rules_for_class(c);
        SLB_REQUIRE(rb, SLB_ERR_OOM, "nearquad (modal): rule tables");
        tb->rs[c].th = rb->th;
        tb->rs[c].w = rb->w;
        tb->rs[c].E = rb->E;
        tb->rs[c].lde = rb->lde;
        std::memcpy(tb->rs[c].off, rb->off, sizeof(rb->off));
        std::memcpy(tb->rs[c].cnt, rb->cnt, sizeof(rb->cnt));
    }
    const int KD = (kernel == SLB_LAPLACE_DL || kernel == SLB_LAPLACE_SL) ? 1 : 3;
    Args a;
    std::memset(&a, 0, sizeof(a));
    a.kernel = (int)kernel;
    a.T = n_trg;
    a.x = x_trg; a.trg_node = trg_node; a.row_ptr = row_ptr; a.panel_idx = panel_idx; a.y = y_coarse;
    a.cn0 = cn0; a.pns = pns; a.pnt = pnt;
    a.ns = pns ? ns_max : ns_uniform;
    a.nt = pnt ? nt_max : nt_uniform;
    a.boff = boff;
    a.eta_panel = eta_panel;
    a.eta_default = (kernel == SLB_STOKES_SL || kernel == SLB_LAPLACE_SL) ? 1.0 : 0.0;
    a.dl = (kernel == SLB_STOKES_SL || kernel == SLB_LAPLACE_SL) ? 0.0 : 1.0;
    a.blocks = blocks;
    {
        static const double rb = [] { const char* e = getenv("SLB_NQ_BERN_RHO"); return e ? atof(e) : 2.5; }();
        a.bern = rb + 1.0 / rb;          // SLB_NQ_BERN_RHO: tuning / accuracy studies only
    }
    int64_t nnz = 0;
    SLB_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n_trg, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SLB_CUDA(cudaStreamSynchronize(s));
    a.nnz = nnz;
    if (nnz == 0) return SLB_OK;
    // Segments of pairs with one launch configuration each.  Uniform orders: one segment, every pair.  Ragged
    // orders: the pairs grouped by the angular rule class of their element (N_th <= 12 / 24 / 40 / 64), each
    // group launched with its own accumulator width, shared-memory layout and CTA size, so the small elements
    // do not pay for the largest one (pair order inside a group: ascending, i.e. target-major).
    struct Seg { int64_t off, cnt; int ns, nt; };
    std::vector<Seg> segs;
    int64_t* plist_d = nullptr;
    if (pnt) {
        std::vector<int32_t> pidx(nnz);
        SLB_CUDA(cudaMemcpyAsync(pidx.data(), panel_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, s));
        SLB_CUDA(cudaStreamSynchronize(s));
        int32_t P = 0;
        for (int64_t q = 0; q < nnz; ++q) P = std::max(P, pidx[q] + 1);
        std::vector<int32_t> hnt(P), hns(P, ns_uniform);
        SLB_CUDA(cudaMemcpy(hnt.data(), pnt, sizeof(int32_t) * P, cudaMemcpyDeviceToHost));
        if (pns) SLB_CUDA(cudaMemcpy(hns.data(), pns, sizeof(int32_t) * P, cudaMemcpyDeviceToHost));
        std::vector<int64_t> order;
        order.reserve(nnz);
        for (int c = 0; c < kNClass; ++c) {
            Seg g{(int64_t)order.size(), 0, 1, 1};
            for (int64_t q = 0; q < nnz; ++q) {
                const int k = pidx[q];
                if (class_of_nt(hnt[k]) != c) continue;
                order.push_back(q);
                g.ns = std::max(g.ns, hns[k]);
                g.nt = std::max(g.nt, hnt[k]);
            }
            g.cnt = (int64_t)order.size() - g.off;
            if (g.cnt) segs.push_back(g);
        }
        SLB_CUDA(cudaMallocAsync(&plist_d, sizeof(int64_t) * nnz, s));
        SLB_CUDA(cudaMemcpyAsync(plist_d, order.data(), sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, s));
        SLB_CUDA(cudaStreamSynchronize(s));              // order is a host temporary
    } else {
        segs.push_back({0, nnz, a.ns, a.nt});
    }
    a.plist = plist_d;
    unsigned long long* work = nullptr;
    SLB_CUDA(cudaMallocAsync(&work, sizeof(unsigned long long) + sizeof(int) * 2, s));
    SLB_CUDA(cudaMemsetAsync(work, 0, sizeof(unsigned long long) + sizeof(int) * 2, s));
    a.work = work;
    a.status = reinterpret_cast<int*>(work + 1);
    // pre-pass geometry for pairs in chunks (32 + 8 bytes per pair)
    const int64_t chunk = std::min<int64_t>(nnz, (int64_t)1 << 22);
    SLB_CUDA(cudaMallocAsync(&a.pre, sizeof(double) * 4 * chunk, s));
    SLB_CUDA(cudaMallocAsync(&a.prow, sizeof(int64_t) * chunk, s));
    static const int w_env = [] { const char* e = getenv("SLB_NQ_WARPS"); return e ? atoi(e) : 8; }();
    slb_status r = SLB_OK;
    for (const Seg& g : segs) {
        if (r != SLB_OK) break;
        a.ns = g.ns;
        a.nt = g.nt;
        const int L = a.nt / 2;
        a.ld_e = (2 * (L + 1) + 7) / 8 * 8;
        int W = (w_env == 1 || w_env == 2 || w_env == 4 || w_env == 8) ? w_env : 8;   // tuning studies
        size_t bytes = 0;
        for (; W >= 1; W /= 2) {
            const Smem S = smem_layout(a.ns, a.nt, W, a.ld_e, KD);
            bytes = S.total * sizeof(double);
            if (bytes <= 200 * 1024) break;
        }
        SLB_REQUIRE(W >= 1, SLB_ERR_UNSUPPORTED, "nearquad (modal): shared memory");
        a.warps = W;
        const int nct_launch = (2 * (a.nt / 2 + 1) + 7) / 8;
        const int NCTc = nct_launch <= 2 ? 2 : nct_launch <= 4 ? 4 : nct_launch <= 6 ? 6 : 9;
        const void* fn;
#define NQ_FN(K, C) (const void*)nq_modal_kernel<K, C>
        if (KD == 3) fn = NCTc == 2 ? NQ_FN(3, 2) : NCTc == 4 ? NQ_FN(3, 4) : NCTc == 6 ? NQ_FN(3, 6) : NQ_FN(3, 9);
        else fn = NCTc == 2 ? NQ_FN(1, 2) : NCTc == 4 ? NQ_FN(1, 4) : NCTc == 6 ? NQ_FN(1, 6) : NQ_FN(1, 9);
#undef NQ_FN
        { slb_status st_ = smem_optin(fn); if (st_ != SLB_OK) return st_; }
        int per_sm = 0;
        SLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, W * 32, bytes));
        const void* fpre = (const void*)nq_srule_kernel;
        const size_t pre_bytes = sizeof(double) * 4 * ((size_t)a.ns * a.nt * 3 + 2 * a.ns);   // 4 warps
        { slb_status st_ = smem_optin(fpre); if (st_ != SLB_OK) return st_; }
        int pre_per_sm = 0;
        SLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pre_per_sm, fpre, 128, pre_bytes));
        for (int64_t c0 = g.off; c0 < g.off + g.cnt && r == SLB_OK; c0 += chunk) {
            a.p0 = c0;
            a.p1 = std::min<int64_t>(g.off + g.cnt, c0 + chunk);
            const int64_t np = a.p1 - a.p0;
            void* args[] = {(void*)&a, (void*)tb.get()};
            const int64_t gpre = std::min<int64_t>((np + 3) / 4, (int64_t)num_sms() * std::max(1, pre_per_sm));
            SLB_CUDA(cudaLaunchKernel(fpre, dim3((unsigned)gpre), dim3(128), args, pre_bytes, s));
            ++g_launch_count;
            r = check_launch("nq_srule_kernel");
            if (r != SLB_OK) break;
            SLB_CUDA(cudaMemsetAsync(work, 0, sizeof(unsigned long long), s));
            const int64_t grid = std::min<int64_t>(np, (int64_t)num_sms() * std::max(1, per_sm));
            SLB_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(W * 32), args, bytes, s));
            ++g_launch_count;
            r = check_launch("nq_modal_kernel");
        }
    }
    int h = 0;
    if (r == SLB_OK) {
        cudaError_t e = cudaMemcpyAsync(&h, a.status, sizeof(int), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) { set_error(std::string("nearquad (modal): ") + cudaGetErrorString(e)); r = SLB_ERR_CUDA; }
    }
    cudaFreeAsync(work, s);
    cudaFreeAsync(a.pre, s);
    cudaFreeAsync(a.prow, s);
    if (plist_d) cudaFreeAsync(plist_d, s);
    if (r == SLB_OK && h) {
        set_error("nearquad (modal): s sub-panel budget exceeded (target extremely close to an element)");
        r = SLB_ERR_UNSUPPORTED;
    }
    return r;
}

}  // namespace slb
