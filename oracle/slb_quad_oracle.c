/*
 * slb_quad_oracle.c -- plain CPU oracle of the special-quadrature correction blocks (NEXT N1).
 * TEST INFRASTRUCTURE ONLY (same rules as slb_oracle.c: only tests/, smoke() and bench.py's
 * cpu_baseline leg may load it; it shares no code, header or table with the CUDA library).
 *
 * What it computes -- the plain definition of the special-quadrature part of the local
 * correction (PAPER.md Eq. e:nystrom-correction P:L935-941 and the E formulas P:L1233-1239,
 * P:L1344-1351, whose first term is the exact action of the layer potential of element k on
 * the element's interpolation basis):
 *
 *   B_{t,k}[r][(i,j,c)] = int_{-1}^{1} int_{0}^{2pi} K_rc(x_t - y(t,th); n(t,th)) l_i(t) C_j(th) J(t,th) dth dt
 *
 *   y(t,th)  = sum_ij y_ij l_i(t) C_j(th)        the element's surface interpolant from its nodes
 *                                                 (Lagrange in s on the GL nodes, trig in th)
 *   l_i      = Lagrange basis on the N_s GL nodes of [-1,1], direct product formula
 *   C_j(th)  = (1/N)[1 + 2 sum_{l=1}^{N/2-1} cos l(th - th_j) + cos (N/2)(th - th_j)]   (reading R3, R4)
 *   J        = |y_t x y_th|,  n = (y_th x y_t) / J  (outward, reading R8)
 *   K        = eta S + D (Stokes, D with sign R1), D + eta S_L (Laplace), S or S_L (pure single layers)
 *
 * How: iterated (nested) adaptive Gauss-Kronrod (G7/K15) -- the inner integral in th for each
 * outer node t, then the outer integral in t -- each split at the target's closest point on the
 * element (found by dense sampling + Gauss-Newton) and graded dyadically towards it, refined
 * until |K15 - G7| is below tol times the integral's scale.  A target that is node (i0, j0) of the
 * element itself (on-surface, singular) is integrated instead over the 4 parameter rectangles
 * meeting at (t_i0, th_j0), each split into 2 triangles and mapped by the Duffy transform
 * (Jacobian u cancels the 1/r singularity), then the same nested adaptive rule in (u, v).
 * No tables, no blocking, no fusion: every quadrature point evaluates the definition above.
 *
 * Pins (tests/test_oracle_pins.py, "N1"): jump relations (Gauss's law -1/2 on the surface,
 * -1 / 0 off it), Prop. 1 (Stokes DL of rigid motions), Stokes S[n] = 0,
 * Green's representation on and off the surface (Eq. e:greens-rep), the paper's
 * convergence table t:conv-biest as an upper bound, and the identity term of the
 * full operator (c_I = 1/2 with sigma' != 0).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define Q_PI 3.14159265358979323846
#define Q_MAXN 64
#define Q_MAXDEPTH 48

void or_gauss_legendre(int n, double* x, double* w);                           /* slb_oracle.c */
void or_kernel_matrix(int kind, const double r[3], const double n[3], double eta, double K[9]);

/* ------------------------------------------------------------------ */
/* element geometry                                                    */
/* ------------------------------------------------------------------ */
typedef struct {
    int ns, nt;
    const double* yc;             /* [ns][nt][3] */
    double tg[Q_MAXN];            /* GL nodes of [-1,1] */
    double ec[Q_MAXN / 2 + 1][Q_MAXN], es[Q_MAXN / 2 + 1][Q_MAXN];   /* cos / sin(l th_j) */
} qpanel;

static void qpanel_init(qpanel* P, int ns, int nt, const double* yc) {
    double w[Q_MAXN];
    P->ns = ns;
    P->nt = nt;
    P->yc = yc;
    or_gauss_legendre(ns, P->tg, w);
    for (int l = 0; l <= nt / 2; ++l)
        for (int j = 0; j < nt; ++j) {
            double th = 2.0 * Q_PI * j / nt;
            P->ec[l][j] = cos(l * th);
            P->es[l][j] = sin(l * th);
        }
}

/* Lagrange basis and derivative, direct product formulas.  Evaluated in long double: the geometry built
 * from them feeds (r.n) = O(|r|^2) of the double layer near the surface, whose absolute accuracy the
 * pins and the parity tests need beyond what eps-level basis values give. */
typedef long double qreal;

static void lagrange_ld(const qpanel* P, qreal t, qreal* l, qreal* dl) {
    int n = P->ns;
    for (int i = 0; i < n; ++i) {
        qreal p = 1.0L;
        for (int k = 0; k < n; ++k)
            if (k != i) p *= (t - (qreal)P->tg[k]) / ((qreal)P->tg[i] - (qreal)P->tg[k]);
        l[i] = p;
        qreal d = 0.0L;
        for (int m = 0; m < n; ++m) {
            if (m == i) continue;
            qreal q = 1.0L / ((qreal)P->tg[i] - (qreal)P->tg[m]);
            for (int k = 0; k < n; ++k)
                if (k != i && k != m) q *= (t - (qreal)P->tg[k]) / ((qreal)P->tg[i] - (qreal)P->tg[k]);
            d += q;
        }
        dl[i] = d;
    }
}

static void lagrange(const qpanel* P, double t, double* l, double* dl) {
    qreal L[Q_MAXN], D[Q_MAXN];
    lagrange_ld(P, t, L, D);
    for (int i = 0; i < P->ns; ++i) { l[i] = (double)L[i]; dl[i] = (double)D[i]; }
}

/* trig cardinal functions C_j(th) and C_j'(th) from the Fourier-sum definition (R3), long double:
 * cos l(th - th_j), sin l(th - th_j) evaluated directly at the difference */
static void cardinal_ld(const qpanel* P, qreal th, qreal* C, qreal* dC) {
    int N = P->nt;
    for (int j = 0; j < N; ++j) {
        qreal phi = th - 2.0L * 3.141592653589793238462643383279502884L * j / N;
        qreal c1 = cosl(phi), s1 = sinl(phi), cl = 1.0L, sl = 0.0L;
        qreal v = 1.0L, d = 0.0L;
        for (int l = 1; l < N / 2; ++l) {          /* cos, sin of l phi by the angle-addition recurrence */
            qreal cn = cl * c1 - sl * s1;
            sl = sl * c1 + cl * s1;
            cl = cn;
            v += 2.0L * cl;
            d -= 2.0L * l * sl;
        }
        v += cosl(0.5L * N * phi);
        d -= 0.5L * N * sinl(0.5L * N * phi);
        C[j] = v / N;
        dC[j] = d / N;
    }
}

static void cardinal(const qpanel* P, double th, double* C, double* dC) {
    qreal c[Q_MAXN], d[Q_MAXN];
    cardinal_ld(P, th, c, d);
    for (int j = 0; j < P->nt; ++j) { C[j] = (double)c[j]; dC[j] = (double)d[j]; }
}

typedef struct {
    double l[Q_MAXN], dl[Q_MAXN], C[Q_MAXN], dC[Q_MAXN];
    double y[3], yt[3], yh[3], n[3], J;
    double rel[3];                /* y - xref (eval_point_x), long-double accumulated */
} qpoint;

/* Surface point and tangents.  xref: evaluate them from the node positions relative to xref (y_ij - xref;
 * the interpolant reproduces constants, so y - xref, y_t, y_th are the same functions), which keeps their
 * rounding error at eps |y_ij - xref| ~ eps L instead of eps |y| -- the normal of a near-singular
 * double-layer integrand enters through (r.n) = O(|r|^2) and needs that.  xref = NULL: absolute. */
static void eval_point_x(const qpanel* P, const double* xref, double t, double th, qpoint* q) {
    qreal L[Q_MAXN], DL[Q_MAXN], C[Q_MAXN], DC[Q_MAXN];
    lagrange_ld(P, t, L, DL);
    cardinal_ld(P, th, C, DC);
    const double z[3] = {0.0, 0.0, 0.0};
    const double* o = xref ? xref : z;
    qreal y[3] = {0, 0, 0}, yt[3] = {0, 0, 0}, yh[3] = {0, 0, 0};
    for (int i = 0; i < P->ns; ++i)
        for (int j = 0; j < P->nt; ++j) {
            const double* v = P->yc + 3 * (i * P->nt + j);
            for (int a = 0; a < 3; ++a) {
                const qreal dv = (qreal)v[a] - (qreal)o[a];
                y[a] += dv * L[i] * C[j];
                yt[a] += dv * DL[i] * C[j];
                yh[a] += dv * L[i] * DC[j];
            }
        }
    for (int i = 0; i < P->ns; ++i) { q->l[i] = (double)L[i]; q->dl[i] = (double)DL[i]; }
    for (int j = 0; j < P->nt; ++j) { q->C[j] = (double)C[j]; q->dC[j] = (double)DC[j]; }
    for (int a = 0; a < 3; ++a) {
        q->y[a] = (double)(y[a] + (qreal)o[a]);
        q->yt[a] = (double)yt[a];
        q->yh[a] = (double)yh[a];
        q->rel[a] = (double)y[a];                 /* y - xref */
    }
    qreal c[3] = {yh[1] * yt[2] - yh[2] * yt[1], yh[2] * yt[0] - yh[0] * yt[2], yh[0] * yt[1] - yh[1] * yt[0]};
    qreal J = sqrtl(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    q->J = (double)J;
    for (int a = 0; a < 3; ++a) q->n[a] = (double)(c[a] / J);
}

static void eval_point(const qpanel* P, double t, double th, qpoint* q) { eval_point_x(P, NULL, t, th, q); }

/* ------------------------------------------------------------------ */
/* kernels by slb_kernel id: 1 Laplace D (+ eta S_L), 2 Stokes eta S + D, 3 Stokes S, 4 Laplace S_L */
/* ------------------------------------------------------------------ */
static int kdim(int kernel) { return (kernel == 2 || kernel == 3) ? 3 : 1; }

static void kernel_eval(int kernel, const double r[3], const double n[3], double eta, double K[9]) {
    static const double zero[3] = {0.0, 0.0, 0.0};
    switch (kernel) {
        case 1: or_kernel_matrix(1, r, n, eta, K); break;            /* D + eta S_L */
        case 2: or_kernel_matrix(2, r, n, eta, K); break;            /* eta S + D */
        case 3: or_kernel_matrix(2, r, zero, eta, K); break;         /* eta S (D of n = 0 vanishes) */
        default: or_kernel_matrix(3, r, n, 0.0, K); K[0] *= eta; break;   /* eta S_L */
    }
}

/* ------------------------------------------------------------------ */
/* vector adaptive Gauss-Kronrod G7/K15                                */
/* ------------------------------------------------------------------ */
static const double XK[8] = {0.991455371120812639206854697526329, 0.949107912342758524526189684047851,
                             0.864864423359769072789712788640926, 0.741531185599394439863864773280788,
                             0.586087235467691130294144845693013, 0.405845151377397166906606412076961,
                             0.207784955007898467600689403773245, 0.000000000000000000000000000000000};
static const double WK[8] = {0.022935322010529224963732008058970, 0.063092092629978553290700663189204,
                             0.104790010322250183839876322541518, 0.140653259715525918745189590510238,
                             0.169004726639267902826583426598550, 0.190350578064785409913256402421014,
                             0.204432940075298892414161999234649, 0.209482141084727828012999174891714};
static const double WG[4] = {0.129484966168869693270611432679082, 0.279705391489276667901467771423780,
                             0.381830050505118944950369775488975, 0.417959183673469387755102040816327};

typedef void (*qfun)(void* ctx, double x, double* out);

/* one GK15 panel: res = K15 (nv values); returns the QUADPACK-style error estimate
 * max_c E_c min(1, (200 E_c / A_c)^1.5), E_c = |K15_c - G7_c|, A_c = h sum_k wk |f_c(x_k)|;
 * *abs_out = max_c A_c. */
static double gk15(qfun f, void* ctx, int nv, double a, double b, double* res, double* tmp, double* abs_out) {
    double c = 0.5 * (a + b), h = 0.5 * (b - a);
    double* g = tmp + nv;
    double* ab = tmp + 2 * nv;
    for (int v = 0; v < nv; ++v) { res[v] = 0.0; g[v] = 0.0; ab[v] = 0.0; }
    for (int k = 0; k < 8; ++k) {
        int npt = (k == 7) ? 1 : 2;
        for (int s = 0; s < npt; ++s) {
            double x = (s == 0) ? c - h * XK[k] : c + h * XK[k];
            f(ctx, x, tmp);
            for (int v = 0; v < nv; ++v) {
                res[v] += WK[k] * tmp[v];
                ab[v] += WK[k] * fabs(tmp[v]);
                if (k % 2 == 1) g[v] += WG[k / 2] * tmp[v];      /* Gauss nodes are the odd Kronrod ones */
            }
        }
    }
    /* the QUADPACK heuristic E min(1, (200 E / A)^1.5) per component (E, A of the same component),
     * then the maximum over components */
    double e = 0.0, A = 0.0;
    for (int v = 0; v < nv; ++v) {
        res[v] *= h;
        g[v] *= h;
        double d = fabs(res[v] - g[v]);
        double av = fabs(h) * ab[v];
        if (av > 0.0 && d > 0.0) {
            double q = pow(200.0 * d / av, 1.5);
            if (q < 1.0) d *= q;
        }
        d -= 50.0 * 2.2e-16 * av;          /* what remains above this component's rounding floor */
        if (d > e) e = d;
        if (av > A) A = av;
    }
    *abs_out = A;
    return e;
}

/* Global adaptive integration (QUADPACK qag strategy) of f over [bp[0], bp[nb]] starting from
 * the panels of bp: bisect the panel with the largest error estimate until the summed estimate
 * is <= tol * S (S = max_c |integral_c| estimated on the initial panels), a panel's estimate being
 * what is left above each component's rounding floor (50 eps int |f_c|), or 4000 panels.  The result is summed in panel order
 * (deterministic).  out[nv] written. */
typedef struct { double a, b, err, A; int live; } qpan;

static void adapt(qfun f, void* ctx, int nv, const double* bp, int nb, double tol, double* out) {
    const int cap = 4000;
    qpan* pan = (qpan*)malloc(sizeof(qpan) * cap);
    double* R = (double*)malloc(sizeof(double) * (size_t)nv * cap);     /* per-panel results */
    double* tmp = (double*)malloc(sizeof(double) * nv * 3);
    int np = 0;
    double E = 0.0;
    double* net = (double*)calloc((size_t)nv, sizeof(double));
    for (int q = 0; q < nb && np < cap; ++q) {
        if (!(bp[q + 1] > bp[q])) continue;
        pan[np].a = bp[q];
        pan[np].b = bp[q + 1];
        pan[np].err = gk15(f, ctx, nv, bp[q], bp[q + 1], R + (size_t)np * nv, tmp, &pan[np].A);
        pan[np].live = 1;
        for (int v = 0; v < nv; ++v) net[v] += R[(size_t)np * nv + v];
        if (pan[np].err > 0.0) E += pan[np].err;
        ++np;
    }
    /* scale: the largest |integral| (max-norm of the result), not the integral of |f| */
    double S = 0.0;
    for (int v = 0; v < nv; ++v) if (fabs(net[v]) > S) S = fabs(net[v]);
    free(net);
    if (S == 0.0) S = 1e-300;
    while (E > tol * S && np < cap) {
        int w = -1;
        for (int q = 0; q < np; ++q)
            if (pan[q].live && (w < 0 || pan[q].err > pan[w].err)) w = q;
        if (w < 0) break;
        if (pan[w].err <= 0.0 || (pan[w].b - pan[w].a) < 1e-15 * (bp[nb] - bp[0])) {
            pan[w].live = 0;             /* at the rounding floor: keep it, stop refining it */
            continue;
        }
        double a = pan[w].a, b = pan[w].b, m = 0.5 * (a + b);
        E -= fmax(pan[w].err, 0.0);
        /* left half replaces w, right half appended; order restored by sorting on a at the end */
        pan[w].b = m;
        pan[w].err = gk15(f, ctx, nv, a, m, R + (size_t)w * nv, tmp, &pan[w].A);
        pan[np].a = m;
        pan[np].b = b;
        pan[np].live = 1;
        pan[np].err = gk15(f, ctx, nv, m, b, R + (size_t)np * nv, tmp, &pan[np].A);
        E += fmax(pan[w].err, 0.0) + fmax(pan[np].err, 0.0);
        ++np;
    }
    /* sum in ascending a (deterministic order independent of the refinement history) */
    for (int v = 0; v < nv; ++v) out[v] = 0.0;
    char* used = (char*)calloc((size_t)(np > 0 ? np : 1), 1);
    for (int k = 0; k < np; ++k) {
        int w = -1;
        for (int q = 0; q < np; ++q)
            if (!used[q] && (w < 0 || pan[q].a < pan[w].a)) w = q;
        used[w] = 1;
        for (int v = 0; v < nv; ++v) out[v] += R[(size_t)w * nv + v];
    }
    free(used);
    free(tmp);
    free(R);
    free(pan);
}

/* breakpoints on [a, b] graded dyadically towards p in [a, b] down to a smallest gap hmin */
static int graded(double a, double b, double p, double hmin, double* bp) {
    int n = 0;
    double lo[80], hi[80];
    int nl = 0, nh = 0;
    for (double h = (p - a) / 2; h > hmin && nl < 78; h /= 2) lo[nl++] = p - h;
    for (double h = (b - p) / 2; h > hmin && nh < 78; h /= 2) hi[nh++] = p + h;
    bp[n++] = a;
    for (int q = 0; q < nl; ++q) if (lo[q] > bp[n - 1]) bp[n++] = lo[q];
    if (p > bp[n - 1] && p < b) bp[n++] = p;
    for (int q = nh - 1; q >= 0; --q) if (hi[q] > bp[n - 1] && hi[q] < b) bp[n++] = hi[q];
    bp[n++] = b;
    return n - 1;       /* panels */
}

/* ------------------------------------------------------------------ */
/* the block integrand                                                 */
/* ------------------------------------------------------------------ */
typedef struct {
    const qpanel* P;
    int kernel, d;
    double eta, x[3];
    double tol;
    /* nested (off-element) integration */
    double t_cur;          /* outer node for the inner integral */
    double th_split, hmin_th;
    int nH;                /* d*d*nt */
    double* Hbuf;
    /* singular (Duffy) integration */
    double t0, th0, A, B;  /* corner, signed extents */
    int i0, j0;            /* the corner node */
    int tri;               /* 0: (A u, B u v), 1: (A u v, B u) */
    double u_cur;
} qctx;

/* inner integrand (th at fixed t): H[r][c][j] = K_rc J C_j */
static void f_inner(void* vc, double th, double* out) {
    qctx* c = (qctx*)vc;
    qpoint q;
    eval_point_x(c->P, c->x, c->t_cur, th, &q);
    /* r = x - y from the node positions relative to x, accumulated in long double */
    double r[3] = {-q.rel[0], -q.rel[1], -q.rel[2]};
    double K[9];
    kernel_eval(c->kernel, r, q.n, c->eta, K);
    int d = c->d, N = c->P->nt;
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b)
            for (int j = 0; j < N; ++j) out[(a * d + b) * N + j] = K[a * d + b] * q.J * q.C[j];
}

/* outer integrand (t): B[r][(i,j,c)] = l_i(t) H[r][c][j](t) */
static void f_outer(void* vc, double t, double* out) {
    qctx* c = (qctx*)vc;
    c->t_cur = t;
    double bp[200];
    int nb = graded(c->th_split - Q_PI, c->th_split + Q_PI, c->th_split, c->hmin_th, bp);
    adapt(f_inner, c, c->nH, bp, nb, c->tol * 0.1, c->Hbuf);
    double l[Q_MAXN], dl[Q_MAXN];
    lagrange(c->P, t, l, dl);
    int d = c->d, N = c->P->nt, ns = c->P->ns;
    for (int a = 0; a < d; ++a)
        for (int i = 0; i < ns; ++i)
            for (int j = 0; j < N; ++j)
                for (int b = 0; b < d; ++b)
                    out[a * (ns * N * d) + (i * N + j) * d + b] = l[i] * c->Hbuf[(a * d + b) * N + j];
}

/* r = x - y(t0 + dt, th0 + dh) for the element's own node x = y_{i0 j0}, in the cancellation-free
 * difference form r = sum_ij (x - y_ij) l_i(t) C_j(th) (partition of unity): the (i0, j0) term is
 * exactly 0 and every other term is a node difference times a basis value that is computed to full
 * RELATIVE accuracy from (dt, dh) -- l_i by the product formula with t - t_k = dt + (t0 - t_k), C_j by
 * the cardinal form sin(N phi/2) cot(phi/2)/N with sin(N (th - th_j)/2) = (-1)^(j0-j) sin(N dh/2).
 * (Evaluated naively, x - y has an absolute rounding error ~eps |y|, which the double layer's
 * (r.n)/|r|^3 turns into an O(eps/|r|) error near the node.) */
static void r_singular(const qctx* c, double dt, double dh, const double* Cnaive, double r[3]) {
    const qpanel* P = c->P;
    int ns = P->ns, N = P->nt, i0 = c->i0, j0 = c->j0;
    double l[Q_MAXN], C[Q_MAXN];
    for (int i = 0; i < ns; ++i) {
        double p = 1.0;
        for (int k = 0; k < ns; ++k)
            if (k != i) p *= (dt + (P->tg[i0] - P->tg[k])) / (P->tg[i] - P->tg[k]);
        l[i] = p;
    }
    double sh = sin(0.5 * N * dh);
    for (int j = 0; j < N; ++j) {
        double phi = dh + 2.0 * Q_PI * (j0 - j) / N;      /* th - th_j */
        if (j == j0) {
            double h = 0.5 * dh;
            C[j] = (fabs(h) < 1e-8) ? 1.0 : sh / tan(h) / N;
        } else if (fabs(sin(0.5 * phi)) < 1e-3) {
            C[j] = Cnaive[j];              /* next to another node (far from the target): 0 * inf form */
        } else {
            double sg = ((j0 - j) % 2 == 0) ? 1.0 : -1.0;
            C[j] = sg * sh / tan(0.5 * phi) / N;
        }
    }
    r[0] = r[1] = r[2] = 0.0;
    for (int i = 0; i < ns; ++i)
        for (int j = 0; j < N; ++j) {
            if (i == i0 && j == j0) continue;
            const double* v = P->yc + 3 * (i * N + j);
            for (int a = 0; a < 3; ++a) r[a] += (c->x[a] - v[a]) * l[i] * C[j];
        }
}

/* Duffy triangle, inner variable v at fixed u */
static void f_duffy_inner(void* vc, double v, double* out) {
    qctx* c = (qctx*)vc;
    double u = c->u_cur;
    double dt = c->tri == 0 ? c->A * u : c->A * u * v;
    double dh = c->tri == 0 ? c->B * u * v : c->B * u;
    double t = c->t0 + dt, th = c->th0 + dh;
    qpoint q;
    eval_point_x(c->P, c->x, t, th, &q);
    double r[3];
    r_singular(c, dt, dh, q.C, r);
    double K[9];
    kernel_eval(c->kernel, r, q.n, c->eta, K);
    double jac = fabs(c->A * c->B) * u;
    int d = c->d, N = c->P->nt, ns = c->P->ns;
    for (int a = 0; a < d; ++a)
        for (int i = 0; i < ns; ++i)
            for (int j = 0; j < N; ++j)
                for (int b = 0; b < d; ++b)
                    out[a * (ns * N * d) + (i * N + j) * d + b] = K[a * d + b] * q.J * jac * q.l[i] * q.C[j];
}

static void f_duffy_outer(void* vc, double u, double* out) {
    qctx* c = (qctx*)vc;
    c->u_cur = u;
    double bp[2] = {0.0, 1.0};
    int nv = c->d * c->d * c->P->ns * c->P->nt;
    adapt(f_duffy_inner, c, nv, bp, 1, c->tol * 0.1, out);
}

/* closest point of x on the element (t clamped to [-1,1]): dense sampling + Gauss-Newton */
static void closest(const qpanel* P, const double x[3], double* t_out, double* th_out, double* d_out) {
    double best = 1e300, bt = 0.0, bh = 0.0;
    qpoint q;
    for (int a = 0; a <= 64; ++a)
        for (int b = 0; b < 128; ++b) {
            double t = -1.0 + 2.0 * a / 64.0, th = 2.0 * Q_PI * b / 128.0;
            eval_point(P, t, th, &q);
            double r[3] = {x[0] - q.y[0], x[1] - q.y[1], x[2] - q.y[2]};
            double dd = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
            if (dd < best) { best = dd; bt = t; bh = th; }
        }
    for (int it = 0; it < 60; ++it) {
        eval_point(P, bt, bh, &q);
        double r[3] = {x[0] - q.y[0], x[1] - q.y[1], x[2] - q.y[2]};
        double a11 = 0, a12 = 0, a22 = 0, g1 = 0, g2 = 0;
        for (int k = 0; k < 3; ++k) {
            a11 += q.yt[k] * q.yt[k]; a12 += q.yt[k] * q.yh[k]; a22 += q.yh[k] * q.yh[k];
            g1 += r[k] * q.yt[k]; g2 += r[k] * q.yh[k];
        }
        double det = a11 * a22 - a12 * a12;
        double dt = (a22 * g1 - a12 * g2) / det, dh = (a11 * g2 - a12 * g1) / det;
        double tn = bt + dt;
        if (tn > 1.0 || tn < -1.0) {             /* on the edge: th only */
            tn = tn > 1.0 ? 1.0 : -1.0;
            dh = g2 / a22;
        }
        bt = tn;
        bh += dh;
    }
    eval_point(P, bt, bh, &q);
    double r[3] = {x[0] - q.y[0], x[1] - q.y[1], x[2] - q.y[2]};
    *t_out = bt;
    *th_out = bh;
    *d_out = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
}

/* One block: kernel (slb_kernel id), target x, element nodes yc [ns][nt][3], single-layer weight
 * eta, singular node (i0, j0) of this element or i0 < 0, relative tolerance tol.
 * B [tdim][ns*nt*sdim] written. */
void or_nearquad_block(int kernel, const double* x, int ns, int nt, const double* yc, double eta, int i0, int j0,
                       double tol, double* B) {
    qpanel* P = (qpanel*)malloc(sizeof(qpanel));
    qpanel_init(P, ns, nt, yc);
    qctx c;
    memset(&c, 0, sizeof(c));
    c.P = P;
    c.kernel = kernel;
    c.d = kdim(kernel);
    c.eta = eta;
    c.tol = tol;
    for (int a = 0; a < 3; ++a) c.x[a] = x[a];
    int nv = c.d * c.d * ns * nt;
    c.nH = c.d * c.d * nt;
    c.Hbuf = (double*)malloc(sizeof(double) * (c.nH + 1));
    if (i0 < 0) {
        double ts, hs, dist;
        closest(P, x, &ts, &hs, &dist);
        qpoint q;
        eval_point(P, ts, hs, &q);
        double nyt = sqrt(q.yt[0] * q.yt[0] + q.yt[1] * q.yt[1] + q.yt[2] * q.yt[2]);
        double nyh = sqrt(q.yh[0] * q.yh[0] + q.yh[1] * q.yh[1] + q.yh[2] * q.yh[2]);
        c.th_split = hs;
        c.hmin_th = 0.25 * dist / nyh;
        if (c.hmin_th < 1e-15) c.hmin_th = 1e-15;
        double bp[200];
        double hmin_t = 0.25 * dist / nyt;
        if (hmin_t < 1e-15) hmin_t = 1e-15;
        int nb = graded(-1.0, 1.0, ts, hmin_t, bp);
        adapt(f_outer, &c, nv, bp, nb, tol, B);
    } else {
        double* tmp = (double*)malloc(sizeof(double) * nv);
        for (int v = 0; v < nv; ++v) B[v] = 0.0;
        c.t0 = P->tg[i0];
        c.th0 = 2.0 * Q_PI * j0 / nt;
        c.i0 = i0;
        c.j0 = j0;
        for (int rect = 0; rect < 4; ++rect) {
            c.A = (rect & 1) ? (1.0 - c.t0) : (-1.0 - c.t0);
            c.B = (rect & 2) ? Q_PI : -Q_PI;
            for (int tri = 0; tri < 2; ++tri) {
                c.tri = tri;
                double bp[2] = {0.0, 1.0};
                adapt(f_duffy_outer, &c, nv, bp, 1, tol, tmp);
                for (int v = 0; v < nv; ++v) B[v] += tmp[v];
            }
        }
        free(tmp);
    }
    free(c.Hbuf);
    free(P);
}

/* All CSR pairs (OpenMP over pairs): the same arguments as slb_nearcorr_quad (uniform orders).
 * trg_node[t] = global coarse node id of target t if it is a node (on-surface), else -1; a pair is
 * singular when that node belongs to the pair's element.  eta_panel may be NULL (weight 1 for the
 * single layers, 0 for Laplace D).  blocks [nnz][tdim][ns*nt*sdim] written. */
void or_nearquad(int kernel, long n_trg, const double* x, const long* trg_node, const long* row_ptr,
                 const int* panel_idx, int ns, int nt, const double* y_coarse, const double* eta_panel,
                 double tol, double* blocks) {
    int d = kdim(kernel);
    long blen = (long)d * d * ns * nt;
    long nnz = row_ptr[n_trg];
    #pragma omp parallel for schedule(dynamic, 1)
    for (long p = 0; p < nnz; ++p) {
        long t = 0;
        while (row_ptr[t + 1] <= p) ++t;                 /* row of pair p */
        int k = panel_idx[p];
        int i0 = -1, j0 = -1;
        long nd = trg_node ? trg_node[t] : -1;
        if (nd >= 0 && nd / ((long)ns * nt) == k) {
            long loc = nd % ((long)ns * nt);
            i0 = (int)(loc / nt);
            j0 = (int)(loc % nt);
        }
        double eta = eta_panel ? eta_panel[k] : ((kernel == 3 || kernel == 4) ? 1.0 : 0.0);
        or_nearquad_block(kernel, x + 3 * t, ns, nt, y_coarse + (long)k * ns * nt * 3, eta, i0, j0, tol,
                          blocks + p * blen);
    }
}
