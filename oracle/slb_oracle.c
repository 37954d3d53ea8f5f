/*
 * slb_oracle.c -- plain, slow, obviously-correct CPU oracle of the slender-body
 * Nystrom operator apply (arXiv 2310.00889).  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 * it.  It shares no code, header, table or constant generator with the CUDA library
 * (paper_2310_00889_b200/csrc); neither includes the other.
 *
 * fp64 throughout; compiled WITHOUT -ffast-math and with -ffp-contract=off so every
 * operation is a plain IEEE operation in the order written.  Sums over sources are
 * Neumaier-compensated and run in ascending source order.
 *
 * What it computes (SURVEY.md §8(c) "Definition"):
 *
 *   u_t = c_I [t < n_on] sigma'_t                                       (a5)
 *       + sum_m K(x_t - y_m; n_m) w_m (U sigma')_m                       (a1 + a3; r = 0 -> 0)
 *       + sum_{k in near(t)} [ B_{t,k} sigma'_k
 *                              - sum_{m in fine(k)} K(x_t - y_m; n_m) w_m (U sigma')_m ]   (a4)
 *       [+ (L sigma)_t for the mobility operator, with sigma' = sigma - L sigma]           (a0)
 *
 * Citations (PAPER.md line numbers, P:L):
 *   Gauss-Legendre nodes on panels ............... §3.1
 *   Lagrange interpolation in s, trig in theta ... §3.1, P:L790-796 (readings R3, R4, R5)
 *   smooth Nystrom rule .......................... Eq. e:nystrom-no-correction
 *   local corrections ............................ Eq. e:nystrom-correction, P:L935-961,
 *                                                  E = sum P w h - G w
 *   Laplace DL kernel dG/dn_y .................... P:L1442-1443 (reading R2)
 *   Stokes SL kernel ............................. Eq. e:stokes-sl
 *   Stokes DL kernel ............................. Eq. e:stokes-dl, P:L551 with sign reading R1
 *   CFIE operators ............................... P:L1750 (Laplace), P:L1868 (Stokes),
 *                                                  P:L2009 (mobility, (K(I-L)+L))
 *   projector L = sum v_i v_i^T, Gram-Schmidt .... Eq. L
 *   eta = 1/(2 rho log rho^-1) ................... P:L1750, P:L1868 (reading R11)
 *
 * Pins for every function: tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.14159265358979323846

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------ */
/* Compensated (Neumaier) accumulator                                  */
/* ------------------------------------------------------------------ */
typedef struct { double s, c; } or_acc;

static void acc_add(or_acc* a, double v) {
    double t = a->s + v;
    if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v;
    else                       a->c += (v - t) + a->s;
    a->s = t;
}
static double acc_val(const or_acc* a) { return a->s + a->c; }

/* ------------------------------------------------------------------ */
/* Gauss-Legendre: Newton iteration on the Legendre three-term recurrence */
/* ------------------------------------------------------------------ */
void or_gauss_legendre(int n, double* x, double* w) {
    for (int i = 0; i < n; ++i) {
        /* i-th root counted from the right end: cos(pi (i + 3/4) / (n + 1/2)) */
        double z = cos(OR_PI * (i + 0.75) / (n + 0.5));
        double dp = 1.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = z;                 /* P_0, P_1 */
            for (int k = 1; k < n; ++k) {            /* (k+1) P_{k+1} = (2k+1) z P_k - k P_{k-1} */
                double p2 = ((2.0 * k + 1.0) * z * p1 - k * p0) / (k + 1.0);
                p0 = p1; p1 = p2;
            }
            if (n == 1) { p0 = 1.0; p1 = z; }
            dp = n * (z * p1 - p0) / (z * z - 1.0);  /* P_n' */
            double dz = p1 / dp;
            z -= dz;
            if (fabs(dz) < 1e-17) break;
        }
        /* recompute derivative at the converged root */
        double p0 = 1.0, p1 = z;
        for (int k = 1; k < n; ++k) {
            double p2 = ((2.0 * k + 1.0) * z * p1 - k * p0) / (k + 1.0);
            p0 = p1; p1 = p2;
        }
        if (n == 1) p0 = 1.0;
        dp = n * (z * p1 - p0) / (z * z - 1.0);
        /* store ascending: root i from the right goes to slot n-1-i */
        x[n - 1 - i] = z;
        w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
}

/* P[m][i] = prod_{l != i} (t_m - s_l) / (s_i - s_l): Lagrange basis by the direct
 * product formula (not barycentric), from nodes s[0..nf) to points t[0..nt). */
void or_lagrange_matrix(int nf, const double* s, int nt, const double* t, double* P) {
    for (int m = 0; m < nt; ++m)
        for (int i = 0; i < nf; ++i) {
            double v = 1.0;
            for (int l = 0; l < nf; ++l)
                if (l != i) v *= (t[m] - s[l]) / (s[i] - s[l]);
            P[(size_t)m * nf + i] = v;
        }
}

/* F[m][j] = C_N(theta'_m - theta_j), theta_j = 2 pi j / N, theta'_m = 2 pi m / M,
 * C_N(th) = sin(N th / 2) cot(th / 2) / N, C_N(0) = 1 (reading R3, N even). */
void or_trig_matrix(int N, int M, double* F) {
    for (int m = 0; m < M; ++m)
        for (int j = 0; j < N; ++j) {
            double v;
            if ((long)m * N == (long)j * M) v = 1.0;
            else {
                double th = 2.0 * OR_PI * ((double)m / M - (double)j / N);
                v = sin(N * th / 2.0) / tan(th / 2.0) / N;
            }
            F[(size_t)m * N + j] = v;
        }
}

/* sigma_f[p][ms][mt][c] = sum_i sum_j Ps[ms][i] F[mt][j] sigma_c[p][i][j][c] */
void or_upsample(long n_panels, int ns, int nt, int ms, int mt, int nc,
                 const double* sigma_c, double* sigma_f) {
    double* sg = malloc(sizeof(double) * ns);
    double* wg = malloc(sizeof(double) * ns);
    double* sf = malloc(sizeof(double) * ms);
    double* wf = malloc(sizeof(double) * ms);
    double* Ps = malloc(sizeof(double) * ms * ns);
    double* F = malloc(sizeof(double) * mt * nt);
    or_gauss_legendre(ns, sg, wg);
    or_gauss_legendre(ms, sf, wf);
    or_lagrange_matrix(ns, sg, ms, sf, Ps);
    or_trig_matrix(nt, mt, F);
    #pragma omp parallel for schedule(static)
    for (long p = 0; p < n_panels; ++p)
        for (int a = 0; a < ms; ++a)
            for (int b = 0; b < mt; ++b)
                for (int c = 0; c < nc; ++c) {
                    or_acc acc = {0, 0};
                    for (int i = 0; i < ns; ++i)
                        for (int j = 0; j < nt; ++j)
                            acc_add(&acc, Ps[a * ns + i] * F[b * nt + j] *
                                          sigma_c[(((size_t)p * ns + i) * nt + j) * nc + c]);
                    sigma_f[(((size_t)p * ms + a) * mt + b) * nc + c] = acc_val(&acc);
                }
    free(sg); free(wg); free(sf); free(wf); free(Ps); free(F);
}

/* Ragged grids (NEXT N4; §3.1: element k has N_s^(k) x N_th^(k) nodes):
 * panel k's coarse block starts at node sum_{k'<k} ns[k'] nt[k'], its fine block at
 * sum_{k'<k} ms[k'] mt[k']; each panel is interpolated with its own (ns, nt, ms, mt) matrices. */
void or_upsample_ragged(long n_panels, const int* ns, const int* nt, const int* ms, const int* mt, int nc,
                        const double* sigma_c, double* sigma_f) {
    long* c0 = malloc(sizeof(long) * (n_panels + 1));
    long* f0 = malloc(sizeof(long) * (n_panels + 1));
    c0[0] = f0[0] = 0;
    for (long p = 0; p < n_panels; ++p) {
        c0[p + 1] = c0[p] + (long)ns[p] * nt[p];
        f0[p + 1] = f0[p] + (long)ms[p] * mt[p];
    }
    #pragma omp parallel for schedule(dynamic, 1)
    for (long p = 0; p < n_panels; ++p)
        or_upsample(1, ns[p], nt[p], ms[p], mt[p], nc, sigma_c + c0[p] * nc, sigma_f + f0[p] * nc);
    free(c0); free(f0);
}

/* ------------------------------------------------------------------ */
/* Kernels, written out as their matrices.  r = x - y (target minus source).  */
/* ------------------------------------------------------------------ */
/* Laplace double layer dG/dn_y = (r.n) / (4 pi |r|^3)   (R2) */
double or_laplace_dl(const double r[3], const double n[3]) {
    double rr = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    double rn = r[0] * n[0] + r[1] * n[1] + r[2] * n[2];
    return rn / (4.0 * OR_PI * rr * rr * rr);
}

/* Laplace single layer 1/(4 pi |r|) -- used by the Green's identity pin */
double or_laplace_sl(const double r[3]) {
    double rr = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    return 1.0 / (4.0 * OR_PI * rr);
}

/* Stokes single layer S = (1/8pi)(I/|r| + r r^T/|r|^3)   (Eq. e:stokes-sl) */
void or_stokes_sl(const double r[3], double S[9]) {
    double rr = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            S[i * 3 + j] = ((i == j ? 1.0 : 0.0) / rr + r[i] * r[j] / (rr * rr * rr)) / (8.0 * OR_PI);
}

/* Stokes double layer D = +(3/4pi)(r.n) r r^T/|r|^5   (Eq. e:stokes-dl, sign R1) */
void or_stokes_dl(const double r[3], const double n[3], double D[9]) {
    double rr = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    double rn = r[0] * n[0] + r[1] * n[1] + r[2] * n[2];
    double r5 = rr * rr * rr * rr * rr;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            D[i * 3 + j] = 3.0 / (4.0 * OR_PI) * rn * r[i] * r[j] / r5;
}

/* Combined kernel matrix K = eta S + D (Stokes, kind 2), or the Laplace combined field
 * D + eta S_L (kind 1, 1x1 in K[0]; eta = 0: the Laplace DL).  kind 3 = Laplace SL. */
void or_kernel_matrix(int kind, const double r[3], const double n[3], double eta, double K[9]) {
    if (kind == 1) { K[0] = or_laplace_dl(r, n) + eta * or_laplace_sl(r); return; }
    if (kind == 3) { K[0] = or_laplace_sl(r); return; }
    double S[9], D[9];
    or_stokes_sl(r, S);
    or_stokes_dl(r, n, D);
    for (int q = 0; q < 9; ++q) K[q] = eta * S[q] + D[q];
}

static int kind_dim(int kind) { return kind == 2 ? 3 : 1; }

/* one target, sources [m0, m1): adds K w sigma into acc[dim] (r = 0 pairs skipped) */
static void far_range(int kind, const double* x, long m0, long m1, const double* y,
                      const double* nrm, const double* w, const double* eta,
                      const double* sig, or_acc* acc) {
    int d = kind_dim(kind);
    double K[9];
    for (long m = m0; m < m1; ++m) {
        double r[3] = {x[0] - y[3 * m], x[1] - y[3 * m + 1], x[2] - y[3 * m + 2]};
        if (r[0] == 0.0 && r[1] == 0.0 && r[2] == 0.0) continue;
        or_kernel_matrix(kind, r, nrm ? nrm + 3 * m : r, eta ? eta[m] : 0.0, K);
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j)
                acc_add(&acc[i], K[i * d + j] * w[m] * sig[m * d + j]);
    }
}

/* u_t = sum_m K(x_t - y_m; n_m) w_m sigma_m  (Eq. e:nystrom-no-correction) */
void or_farfield(int kind, long T, const double* x, long M, const double* y,
                 const double* nrm, const double* w, const double* eta,
                 const double* sig, double* u) {
    int d = kind_dim(kind);
    #pragma omp parallel for schedule(dynamic, 4)
    for (long t = 0; t < T; ++t) {
        or_acc acc[3] = {{0, 0}, {0, 0}, {0, 0}};
        far_range(kind, x + 3 * t, 0, M, y, nrm, w, eta, sig, acc);
        for (int i = 0; i < d; ++i) u[t * d + i] = acc_val(&acc[i]);
    }
}

/* ------------------------------------------------------------------ */
/* Synthetic special-quadrature block entries: SplitMix64 at a counter (R10) */
/* ------------------------------------------------------------------ */
uint64_t or_splitmix64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double or_block_entry(uint64_t seed, uint64_t flat, double s_blk) {
    double u = (double)(or_splitmix64(seed, flat) >> 11) * (1.0 / 9007199254740992.0);
    return ((2.0 * u - 1.0) * 1.7320508075688772) * s_blk;
}

void or_block_entries(uint64_t seed, uint64_t first, long count, double s_blk, double* out) {
    for (long q = 0; q < count; ++q) out[q] = or_block_entry(seed, first + (uint64_t)q, s_blk);
}

/* ------------------------------------------------------------------ */
/* Rigid-motion projector L = sum_i v_i v_i^T (Eq. L):     */
/* per body, 3 translations + 3 rotations e_a x (y - y_ref), orthonormalised */
/* by (modified) Gram-Schmidt in the surface L2 inner product <f,g> = sum w f.g. */
/* ------------------------------------------------------------------ */
void or_projector(long n_nodes, const double* y, const double* w, const int* body_of_node,
                  int n_bodies, const double* sigma, double* Lsigma) {
    for (int b = 0; b < n_bodies; ++b) {
        long cnt = 0;
        double ref[3] = {0, 0, 0};
        for (long q = 0; q < n_nodes; ++q)
            if (body_of_node[q] == b) { cnt++; for (int a = 0; a < 3; ++a) ref[a] += y[3 * q + a]; }
        if (!cnt) continue;
        for (int a = 0; a < 3; ++a) ref[a] /= (double)cnt;     /* unweighted node mean */
        long* idx = malloc(sizeof(long) * cnt);
        long c = 0;
        for (long q = 0; q < n_nodes; ++q) if (body_of_node[q] == b) idx[c++] = q;
        double* V = calloc((size_t)6 * cnt * 3, sizeof(double));   /* V[i][node][3] */
        for (long q = 0; q < cnt; ++q) {
            const double* yy = y + 3 * idx[q];
            double d[3] = {yy[0] - ref[0], yy[1] - ref[1], yy[2] - ref[2]};
            for (int a = 0; a < 3; ++a) V[((size_t)a * cnt + q) * 3 + a] = 1.0;
            /* e_a x d */
            double* r0 = V + ((size_t)3 * cnt + q) * 3;  /* e_x x d = (0, -d_z, d_y) */
            r0[0] = 0; r0[1] = -d[2]; r0[2] = d[1];
            double* r1 = V + ((size_t)4 * cnt + q) * 3;  /* e_y x d = (d_z, 0, -d_x) */
            r1[0] = d[2]; r1[1] = 0; r1[2] = -d[0];
            double* r2 = V + ((size_t)5 * cnt + q) * 3;  /* e_z x d = (-d_y, d_x, 0) */
            r2[0] = -d[1]; r2[1] = d[0]; r2[2] = 0;
        }
        for (int i = 0; i < 6; ++i) {
            double* vi = V + (size_t)i * cnt * 3;
            for (int j = 0; j < i; ++j) {          /* modified Gram-Schmidt */
                double* vj = V + (size_t)j * cnt * 3;
                or_acc ip = {0, 0};
                for (long q = 0; q < cnt; ++q)
                    for (int a = 0; a < 3; ++a) acc_add(&ip, w[idx[q]] * vi[3 * q + a] * vj[3 * q + a]);
                double p = acc_val(&ip);
                for (long q = 0; q < cnt; ++q)
                    for (int a = 0; a < 3; ++a) vi[3 * q + a] -= p * vj[3 * q + a];
            }
            or_acc nn = {0, 0};
            for (long q = 0; q < cnt; ++q)
                for (int a = 0; a < 3; ++a) acc_add(&nn, w[idx[q]] * vi[3 * q + a] * vi[3 * q + a]);
            double nrm = sqrt(acc_val(&nn));
            for (long q = 0; q < cnt * 3; ++q) vi[q] /= nrm;
        }
        /* L sigma = sum_i v_i <v_i, sigma>_w */
        double coef[6];
        for (int i = 0; i < 6; ++i) {
            const double* vi = V + (size_t)i * cnt * 3;
            or_acc ip = {0, 0};
            for (long q = 0; q < cnt; ++q)
                for (int a = 0; a < 3; ++a) acc_add(&ip, w[idx[q]] * vi[3 * q + a] * sigma[3 * idx[q] + a]);
            coef[i] = acc_val(&ip);
        }
        for (long q = 0; q < cnt; ++q)
            for (int a = 0; a < 3; ++a) {
                or_acc s = {0, 0};
                for (int i = 0; i < 6; ++i) acc_add(&s, coef[i] * V[((size_t)i * cnt + q) * 3 + a]);
                Lsigma[3 * idx[q] + a] = acc_val(&s);
            }
        free(V); free(idx);
    }
}

/* eta = 1 / (2 rho log(1/rho))  (natural log, R11) */
double or_eta_cfie(double rho) { return 1.0 / (2.0 * rho * log(1.0 / rho)); }

/* ------------------------------------------------------------------ */
/* Full operator rows                                                  */
/* ------------------------------------------------------------------ */
typedef struct {
    int kind;               /* 1 Laplace DL, 2 Stokes eta S + D */
    int ns, nt, ms, mt;
    long n_panels;
    long n_trg, n_on;
    double c_identity;
    const double* x_trg;    /* [T][3] */
    const double* y_f;      /* [M][3] fine nodes */
    const double* n_f;
    const double* w_f;
    const double* eta_f;    /* [M] (Stokes) */
    const long* row_ptr;    /* [T+1] */
    const int* panel_idx;   /* [nnz] */
    uint64_t blk_seed;
    double s_blk;
    const double* blocks;   /* optional explicit blocks [nnz][tdim][Nn*sdim]; NULL -> seeded */
    /* projector (mobility operator); n_bodies = 0 disables */
    int n_bodies;
    const int* body_of_node;   /* [N] */
    const double* y_c;         /* [N][3] */
    const double* w_c;         /* [N] */
    /* ragged orders per panel (NEXT N4), or NULL: every panel has (ns, nt, ms, mt) */
    const int* panel_nt;       /* [n_panels] */
    const int* panel_mt;       /* [n_panels] */
    const int* panel_ns;       /* [n_panels] */
    const int* panel_ms;       /* [n_panels] */
} or_problem;

/* node offsets of panel k (coarse c0, fine f0), k = 0..n_panels */
static void or_offsets(const or_problem* pb, long* c0, long* f0) {
    c0[0] = f0[0] = 0;
    for (long k = 0; k < pb->n_panels; ++k) {
        int nt = pb->panel_nt ? pb->panel_nt[k] : pb->nt;
        int mt = pb->panel_mt ? pb->panel_mt[k] : pb->mt;
        int ns = pb->panel_ns ? pb->panel_ns[k] : pb->ns;
        int ms = pb->panel_ms ? pb->panel_ms[k] : pb->ms;
        c0[k + 1] = c0[k] + (long)ns * nt;
        f0[k + 1] = f0[k] + (long)ms * mt;
    }
}

/* Precompute sigma' (= sigma or sigma - L sigma), its fine upsample, and L sigma. */
void or_prepare(const or_problem* pb, const double* sigma, double* sigma_p,
                double* sigma_f, double* Lsigma) {
    int d = kind_dim(pb->kind);
    long* c0 = malloc(sizeof(long) * (pb->n_panels + 1));
    long* f0 = malloc(sizeof(long) * (pb->n_panels + 1));
    or_offsets(pb, c0, f0);
    long N = c0[pb->n_panels];
    if (pb->n_bodies > 0) {
        or_projector(N, pb->y_c, pb->w_c, pb->body_of_node, pb->n_bodies, sigma, Lsigma);
        for (long q = 0; q < N * d; ++q) sigma_p[q] = sigma[q] - Lsigma[q];
    } else {
        for (long q = 0; q < N * d; ++q) { sigma_p[q] = sigma[q]; if (Lsigma) Lsigma[q] = 0.0; }
    }
    if (pb->panel_nt || pb->panel_ns) {
        int* a[4];
        for (int q = 0; q < 4; ++q) a[q] = malloc(sizeof(int) * pb->n_panels);
        for (long k = 0; k < pb->n_panels; ++k) {
            a[0][k] = pb->panel_ns ? pb->panel_ns[k] : pb->ns;
            a[1][k] = pb->panel_nt ? pb->panel_nt[k] : pb->nt;
            a[2][k] = pb->panel_ms ? pb->panel_ms[k] : pb->ms;
            a[3][k] = pb->panel_mt ? pb->panel_mt[k] : pb->mt;
        }
        or_upsample_ragged(pb->n_panels, a[0], a[1], a[2], a[3], d, sigma_p, sigma_f);
        for (int q = 0; q < 4; ++q) free(a[q]);
    } else
        or_upsample(pb->n_panels, pb->ns, pb->nt, pb->ms, pb->mt, d, sigma_p, sigma_f);
    free(c0); free(f0);
}

/* u for the listed global target rows; near-correction smooth re-sum done literally. */
void or_apply_rows(const or_problem* pb, const double* sigma_p, const double* sigma_f,
                   const double* Lsigma, long n_rows, const long* rows, double* u,
                   double* u_far, double* u_near) {
    int d = kind_dim(pb->kind);
    long* c0 = malloc(sizeof(long) * (pb->n_panels + 1));
    long* f0 = malloc(sizeof(long) * (pb->n_panels + 1));
    or_offsets(pb, c0, f0);
    long M = f0[pb->n_panels];
    /* first flat entry of every near block: block p = [d][N_n^(k) d], k = panel_idx[p] */
    long nnz = pb->row_ptr[pb->n_trg];
    long* b0 = malloc(sizeof(long) * (nnz + 1));
    b0[0] = 0;
    for (long p = 0; p < nnz; ++p) {
        long k = pb->panel_idx[p];
        b0[p + 1] = b0[p] + (long)d * (c0[k + 1] - c0[k]) * d;
    }
    #pragma omp parallel for schedule(dynamic, 1)
    for (long q = 0; q < n_rows; ++q) {
        long t = rows[q];
        const double* x = pb->x_trg + 3 * t;
        or_acc far[3] = {{0, 0}, {0, 0}, {0, 0}};
        far_range(pb->kind, x, 0, M, pb->y_f, pb->n_f, pb->w_f, pb->eta_f, sigma_f, far);
        or_acc nr[3] = {{0, 0}, {0, 0}, {0, 0}};
        for (long p = pb->row_ptr[t]; p < pb->row_ptr[t + 1]; ++p) {
            long k = pb->panel_idx[p];
            long Nn = c0[k + 1] - c0[k];
            /* + B_{t,k} sigma'_k */
            for (int i = 0; i < d; ++i)
                for (long col = 0; col < Nn * d; ++col) {
                    long flat = b0[p] + i * Nn * d + col;
                    double b = pb->blocks ? pb->blocks[flat]
                                          : or_block_entry(pb->blk_seed, (uint64_t)flat, pb->s_blk);
                    acc_add(&nr[i], b * sigma_p[c0[k] * d + col]);
                }
            /* - smooth contribution of panel k's fine nodes (already inside the far sum) */
            or_acc sm[3] = {{0, 0}, {0, 0}, {0, 0}};
            far_range(pb->kind, x, f0[k], f0[k + 1], pb->y_f, pb->n_f, pb->w_f, pb->eta_f,
                      sigma_f, sm);
            for (int i = 0; i < d; ++i) acc_add(&nr[i], -acc_val(&sm[i]));
        }
        for (int i = 0; i < d; ++i) {
            double fv = acc_val(&far[i]), nv = acc_val(&nr[i]);
            double id = 0.0;
            if (t < pb->n_on) {
                id = pb->c_identity * sigma_p[t * d + i];
                if (pb->n_bodies > 0 && Lsigma) id += Lsigma[t * d + i];
            }
            or_acc tot = {0, 0};
            acc_add(&tot, fv); acc_add(&tot, nv); acc_add(&tot, id);
            u[q * d + i] = acc_val(&tot);
            if (u_far) u_far[q * d + i] = fv;
            if (u_near) u_near[q * d + i] = nv;
        }
    }
    free(c0); free(f0); free(b0);
}

/* Near correction alone with explicit blocks (pin P11: gather-apply == dense product). */
void or_nearcorr_apply(long T, int tdim, int sdim, int nodes_per_panel, const long* row_ptr,
                       const int* panel_idx, const double* blocks, const double* sigma_c,
                       double* u) {
    long cols = (long)nodes_per_panel * sdim;
    #pragma omp parallel for schedule(static)
    for (long t = 0; t < T; ++t)
        for (int i = 0; i < tdim; ++i) {
            or_acc a = {0, 0};
            acc_add(&a, u[t * tdim + i]);
            for (long p = row_ptr[t]; p < row_ptr[t + 1]; ++p) {
                long k = panel_idx[p];
                for (long c = 0; c < cols; ++c)
                    acc_add(&a, blocks[(p * tdim + i) * cols + c] * sigma_c[k * cols + c]);
            }
            u[t * tdim + i] = acc_val(&a);
        }
}
