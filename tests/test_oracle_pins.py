"""Oracle pins: the CPU oracle checked against what the paper and mathematics fix
(pins P1-P13).  CPU only (-m "not gpu").

Each pin is chosen so that a plausible slip (dropped term, wrong sign/index, transposed
operand, wrong normal orientation or Nyquist convention) fails at least one of them.
Pin geometries: the refined torus 'REF' (R=1, rho=0.1, 256 x 10 x 48, coarse = fine).
"""
import os

import numpy as np
import pytest

import oracle as O
from synth import pin_torus, make_config, torus_body, discretize, random_rotation
from synth.rng import splitmix64

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FOUR_PI = 4 * np.pi


@pytest.fixture(scope="module")
def ref():
    return pin_torus()


def _interior_exterior():
    ph = np.array([0.1, 1.3, 2.9, 4.4, 5.9])
    on_c = np.stack([np.cos(ph), np.sin(ph), 0 * ph], 1)                      # centerline
    off = np.stack([(1 + 0.05) * np.cos(ph + .3), (1 + .05) * np.sin(ph + .3), 0 * ph], 1)  # 0.5 rho
    off2 = np.stack([np.cos(ph + .7), np.sin(ph + .7), 0.05 + 0 * ph], 1)
    xin = np.concatenate([on_c, off, off2])
    xout = np.array([[0, 0, 0.0], [2, 0, 0], [0, 0, 0.5], [1.3, 0.2, 0.1], [0.5, 0.5, -0.2],
                     [1.0, 0.0, 0.2], [-3, 1, 2]])
    return xin, xout


# ---------------------------------------------------------------- P1 kernel point values
def test_p1_kernel_point_values():
    e = np.array([1.0, 0, 0])
    assert O.kernel_matrix(1, e, e) == pytest.approx(1 / FOUR_PI, rel=1e-15)
    assert O.kernel_matrix(3, e) == pytest.approx(0.07957747154594767, rel=1e-15)
    S = O.kernel_matrix(2, e, np.zeros(3), eta=1.0)
    np.testing.assert_allclose(S, np.diag([1 / FOUR_PI, 1 / (8 * np.pi), 1 / (8 * np.pi)]), rtol=1e-15)
    D = O.kernel_matrix(2, e, e, eta=0.0)                                           # P:L551 (R1 sign)
    expect = np.zeros((3, 3))
    expect[0, 0] = 0.238732414637843
    np.testing.assert_allclose(D, expect, rtol=1e-14, atol=0)


# ---------------------------------------------------------------- P2 Gauss's law
def test_p2_gauss_law_laplace_dl(ref):
    _, g = ref
    xin, xout = _interior_exterior()
    u = O.farfield(1, np.concatenate([xin, xout]), g.y, g.n, g.w, np.ones(g.w.size))
    np.testing.assert_allclose(u[:len(xin)], -1.0, rtol=0, atol=1e-13)
    np.testing.assert_allclose(u[len(xin):], 0.0, rtol=0, atol=1e-13)


# ---------------------------------------------------------------- P3 Stokes DL, constant density
def test_p3_stokes_dl_constant_density(ref):
    _, g = ref
    xin, xout = _interior_exterior()
    X = np.concatenate([xin, xout])
    zero = np.zeros(g.w.size)
    for c in np.eye(3):
        u = O.farfield(2, X, g.y, g.n, g.w, np.tile(c, (g.w.size, 1)), eta=zero)
        np.testing.assert_allclose(u[:len(xin)], -np.tile(c, (len(xin), 1)), rtol=0, atol=1e-12)
        np.testing.assert_allclose(u[len(xin):], 0.0, rtol=0, atol=1e-12)


# ---------------------------------------------------------------- P4 Stokes DL, rigid motion
def test_p4_stokes_dl_rigid_motion(ref):
    _, g = ref
    xin, xout = _interior_exterior()
    X = np.concatenate([xin, xout])
    a = np.array([0.3, -1.1, 0.7])
    om = np.array([0.9, 0.2, -0.5])
    c = np.array([0.2, 0.1, -0.3])
    v = a + np.cross(om, g.y - c)
    u = O.farfield(2, X, g.y, g.n, g.w, v, eta=np.zeros(g.w.size))
    vx = a + np.cross(om, xin - c)
    np.testing.assert_allclose(u[:len(xin)], -vx, rtol=0, atol=1e-11)
    np.testing.assert_allclose(u[len(xin):], 0.0, rtol=0, atol=1e-11)


# ---------------------------------------------------------------- P5 Stokeslet flux
def test_p5_stokes_sl_of_normal_vanishes(ref):
    _, g = ref
    xin, xout = _interior_exterior()
    X = np.concatenate([xin, xout])
    u = O.farfield(2, X, g.y, np.zeros_like(g.n), g.w, g.n, eta=np.ones(g.w.size))
    np.testing.assert_allclose(u, 0.0, rtol=0, atol=1e-12)


# ---------------------------------------------------------------- P6 symmetry / reciprocity
def test_p6_stokeslet_symmetry_and_reciprocity():
    rng = np.random.default_rng(6)
    for _ in range(20):
        r = rng.standard_normal(3)
        S = O.kernel_matrix(2, r, np.zeros(3), eta=1.0)
        Sm = O.kernel_matrix(2, -r, np.zeros(3), eta=1.0)
        assert np.array_equal(S, S.T) and np.array_equal(S, Sm)
    b, g = pin_torus(P=6, Ns=6, Nt=8)
    sig = rng.standard_normal(g.y.shape)
    tau = rng.standard_normal(g.y.shape)
    z = np.zeros_like(g.n)
    one = np.ones(g.w.size)
    us = O.farfield(2, g.y, g.y, z, g.w, sig, eta=one)    # targets = sources, r = 0 skipped
    ut = O.farfield(2, g.y, g.y, z, g.w, tau, eta=one)
    lhs = np.sum(g.w[:, None] * tau * us)
    rhs = np.sum(g.w[:, None] * sig * ut)
    assert abs(lhs - rhs) <= 1e-13 * max(abs(lhs), abs(rhs))
    # the DL is NOT reciprocal in this sense: guards against a transposed operand
    ud = O.farfield(2, g.y, g.y, g.n, g.w, sig, eta=0 * one)
    udt = O.farfield(2, g.y, g.y, g.n, g.w, tau, eta=0 * one)
    assert abs(np.sum(g.w[:, None] * tau * ud) - np.sum(g.w[:, None] * sig * udt)) > 1e-6


# ---------------------------------------------------------------- P7 upsampling exactness
@pytest.mark.parametrize("ns,nt", [(10, 12), (10, 16), (12, 20), (5, 4)])
def test_p7_upsample_exactness(ns, nt):
    ms, mt = 2 * ns, 2 * nt
    P = 3
    sc, _ = O.gauss_legendre(ns)
    sf, _ = O.gauss_legendre(ms)
    rng = np.random.default_rng(7)
    coef = rng.standard_normal((P, ns))            # degree ns-1 polynomial per panel
    ac = rng.standard_normal(nt // 2)
    bc = rng.standard_normal(nt // 2)
    ny = rng.standard_normal()

    def field(p, t, th):
        poly = np.polynomial.polynomial.polyval(t, coef[p])
        trig = sum(ac[l] * np.cos(l * th) + bc[l] * np.sin(l * th) for l in range(nt // 2))
        trig = trig + ny * np.cos(nt * th / 2)      # Nyquist cosine (R3)
        return poly * trig

    thc = 2 * np.pi * np.arange(nt) / nt
    thf = 2 * np.pi * np.arange(mt) / mt
    c = np.stack([field(p, sc[:, None], thc[None, :]) for p in range(P)])
    f = np.stack([field(p, sf[:, None], thf[None, :]) for p in range(P)])
    for nc in (1, 3):
        cc = np.repeat(c[..., None], nc, axis=-1) * (1 + np.arange(nc))
        ff = np.repeat(f[..., None], nc, axis=-1) * (1 + np.arange(nc))
        out = O.upsample(cc.reshape(-1), P, ns, nt, ms, mt, nc).reshape(ff.shape)
        np.testing.assert_allclose(out, ff, rtol=0, atol=1e-13 * np.abs(ff).max())
    F = O.trig_matrix(nt, mt)
    np.testing.assert_allclose(F[0::2], np.eye(nt), atol=1e-14)
    # the sine Nyquist mode is invisible on the grid and must interpolate to 0, not sin
    s_ny = np.sin(nt * thc / 2)
    assert np.abs(F @ s_ny).max() < 1e-13


def test_gauss_legendre_exactness():
    for n in (1, 2, 5, 10, 12, 20, 24, 40):
        x, w = O.gauss_legendre(n)
        assert np.all(np.diff(x) > 0)
        for k in range(2 * n):
            exact = 0.0 if k % 2 else 2.0 / (k + 1)
            assert abs(np.dot(w, x ** k) - exact) < 5e-15 * (1 + k)
        if 2 <= n <= 12:   # degree 2n is NOT integrated exactly (error ~ 2^(2n+1)(n!)^4/((2n+1)((2n)!)^2))
            assert abs(np.dot(w, x ** (2 * n)) - 2.0 / (2 * n + 1)) > 1e-12


# ---------------------------------------------------------------- P8 weights & geometry
@pytest.mark.parametrize("name", ["c1", "c3"])
def test_p8_weights_geometry(name):
    pr = make_config(name)
    rho = 0.1 if name == "c1" else 0.05
    area = 4 * np.pi ** 2 * 1.0 * rho * pr.n_bodies
    for w, y, n in ((pr.w_c, pr.y_c, pr.n_c), (pr.w_f, pr.y_f, pr.n_f)):
        assert abs(w.sum() - area) <= 1e-14 * area
        assert np.abs((w[:, None] * n).sum(0)).max() <= 1e-13
        cen = (w[:, None] * y).sum(0) / w.sum()
        np.testing.assert_allclose(cen, pr.body_center.mean(0), atol=1e-13)


# ---------------------------------------------------------------- P9 Green's identity
def test_p9_green_identity_laplace():
    b, g = pin_torus(R=1.0, rho=0.25, P=192, Ns=10, Nt=64)
    x0 = np.array([1.0, 2.0, 3.0])
    d = g.y - x0
    rr = np.sqrt((d * d).sum(1))
    u = 1 / (FOUR_PI * rr)
    dudn = -(d * g.n).sum(1) / (FOUR_PI * rr ** 3)
    ph = np.linspace(0, 2 * np.pi, 7)[:-1] + 0.2
    X = np.concatenate([np.stack([np.cos(ph), np.sin(ph), 0 * ph], 1),
                        np.stack([1.1 * np.cos(ph), 1.1 * np.sin(ph), 0.05 + 0 * ph], 1)])
    S = O.farfield(3, X, g.y, None, g.w, dudn)
    D = O.farfield(1, X, g.y, g.n, g.w, u)
    exact = 1 / (FOUR_PI * np.sqrt(((X - x0) ** 2).sum(1)))
    np.testing.assert_allclose(S - D, exact, rtol=1e-12, atol=0)


def test_p9b_laplace_combined_field_kernel():
    """the combined Laplace kernel D + eta S_L (kind 1 with eta, the CFIE of P:L1750) against Green's
    identity: with zero normals and eta = 1 it is S_L, with eta = 0 it is D; and for a general eta it
    is exactly the sum (u = S[du/dn] - D[u] inside)"""
    b, g = pin_torus(R=1.0, rho=0.25, P=192, Ns=10, Nt=64)
    x0 = np.array([1.0, 2.0, 3.0])
    d = g.y - x0
    rr = np.sqrt((d * d).sum(1))
    u = 1 / (FOUR_PI * rr)
    dudn = -(d * g.n).sum(1) / (FOUR_PI * rr ** 3)
    ph = np.linspace(0, 2 * np.pi, 5)[:-1] + 0.4
    X = np.stack([1.05 * np.cos(ph), 1.05 * np.sin(ph), 0.1 + 0 * ph], 1)
    one = np.ones(g.w.size)
    S = O.farfield(1, X, g.y, np.zeros_like(g.n), g.w, dudn, eta=one)
    D = O.farfield(1, X, g.y, g.n, g.w, u, eta=0 * one)
    exact = 1 / (FOUR_PI * np.sqrt(((X - x0) ** 2).sum(1)))
    np.testing.assert_allclose(S - D, exact, rtol=1e-12, atol=0)
    eta = 0.7
    C = O.farfield(1, X, g.y, g.n, g.w, u, eta=eta * one)
    SL = O.farfield(3, X, g.y, None, g.w, u)
    np.testing.assert_allclose(C, D + eta * SL, rtol=1e-13, atol=0)


# ---------------------------------------------------------------- P10 brute-force adaptive
def test_p10_bruteforce_adaptive_quadrature():
    from scipy.integrate import quad
    P, ns, nt = 4, 10, 16
    b = torus_body(1.0, 0.25, (0.1, -0.2, 0.05), random_rotation(np.random.default_rng(10)))
    gc = discretize(b, P, ns, nt)
    gf = discretize(b, P, 2 * ns, 2 * nt)
    # band-limited density: a degree-9 polynomial in s times a trig polynomial in theta
    pc = np.array([0.3, -1.0, 0.5, 0.25, -0.6, 0.1, 0.05, -0.02, 0.01, 0.003])

    def sig(s, th):
        return np.polynomial.polynomial.polyval(s, pc) * (1 + 0.5 * np.cos(th) - 0.3 * np.sin(2 * th))

    sc = sig(gc.s, gc.th)
    sf = O.upsample(sc, P, ns, nt, 2 * ns, 2 * nt, 1)
    X = np.array([[0.1, -0.2, 0.05], [2.4, 0.3, -0.4], [0.5, 1.9, 1.2]])
    u = O.farfield(1, X, gf.y, gf.n, gf.w, sf)

    H = 1e-30

    def integrand(s, th, x):
        y = b.surface(np.array([s]), np.array([th]))[0]
        ys = b.surface(np.array([s + 1j * H]), np.array([th + 0j]))[0].imag / H
        yt = b.surface(np.array([s + 0j]), np.array([th + 1j * H]))[0].imag / H
        cr = np.cross(yt, ys)
        r = x - y
        return (r @ cr) / (FOUR_PI * np.linalg.norm(r) ** 3) * sig(s, th)

    for t in range(len(X)):
        tot = 0.0
        for k in range(P):
            inner = lambda s: quad(lambda th: integrand(s, th, X[t]), 0, 2 * np.pi,
                                   epsabs=1e-15, epsrel=1e-14, limit=200)[0]
            tot += quad(inner, k / P, (k + 1) / P, epsabs=1e-15, epsrel=1e-14, limit=200)[0]
        assert abs(u[t] - tot) <= 1e-12 * max(1.0, abs(tot)), (t, u[t], tot)


def test_p10s_bruteforce_adaptive_quadrature_stokes():
    """P10 for the Stokes eta S + D far sum (R1 sign) with a NON-rigid band-limited 3-vector density,
    against nested adaptive Gauss-Kronrod (scipy quad_vec) over the exact surface; every component of
    S and D enters (a dropped rr^T term, a transposed D or a wrong eta placement fails)."""
    from scipy.integrate import quad_vec
    P, ns, nt = 4, 10, 16
    eta = 0.8
    b = torus_body(1.0, 0.25, (-0.1, 0.15, 0.05), random_rotation(np.random.default_rng(13)))
    gc = discretize(b, P, ns, nt)
    gf = discretize(b, P, 2 * ns, 2 * nt)
    pc = [np.array([0.3, -1.0, 0.5, 0.25, -0.6, 0.1]), np.array([-0.7, 0.2, 0.9, -0.3, 0.05, 0.02]),
          np.array([0.1, 0.4, -0.8, 0.6, -0.2, -0.04])]
    tc = [(0.5, -0.3, 0.2), (-0.4, 0.6, 0.1), (0.25, 0.35, -0.45)]

    def sig(s, th):
        s, th = np.asarray(s), np.asarray(th)
        return np.stack([np.polynomial.polynomial.polyval(s, pc[c]) *
                         (1 + tc[c][0] * np.cos(th) + tc[c][1] * np.sin(2 * th) + tc[c][2] * np.cos(3 * th))
                         for c in range(3)], -1)

    sc = sig(gc.s, gc.th)
    sf = O.upsample(sc.reshape(-1), P, ns, nt, 2 * ns, 2 * nt, 3)
    X = np.array([[-0.1, 0.15, 0.05], [2.3, -0.5, 0.6]])
    u = O.farfield(2, X, gf.y, gf.n, gf.w, sf, eta=np.full(gf.w.size, eta))
    H = 1e-30

    def integrand(s, th, x):
        y = b.surface(np.array([s]), np.array([th]))[0]
        ys = b.surface(np.array([s + 1j * H]), np.array([th + 0j]))[0].imag / H
        yt = b.surface(np.array([s + 0j]), np.array([th + 1j * H]))[0].imag / H
        cr = np.cross(yt, ys)
        J = np.linalg.norm(cr)
        nn = cr / J
        r = x - y
        rr = np.linalg.norm(r)
        S = (np.eye(3) / rr + np.outer(r, r) / rr ** 3) / (8 * np.pi)          # Eq. e:stokes-sl
        D = 3.0 / FOUR_PI * (r @ nn) * np.outer(r, r) / rr ** 5                 # P:L551, sign R1
        return (eta * S + D) @ sig(s, th) * J

    for t in range(len(X)):
        tot = np.zeros(3)
        for k in range(P):
            inner = lambda s: quad_vec(lambda th: integrand(s, th, X[t]), 0, 2 * np.pi,
                                       epsabs=1e-15, epsrel=1e-14)[0]
            tot += quad_vec(inner, k / P, (k + 1) / P, epsabs=1e-15, epsrel=1e-14)[0]
        assert np.abs(u[t] - tot).max() <= 1e-12 * max(1.0, np.abs(tot).max()), (t, u[t], tot)


# ---------------------------------------------------------------- P11 near apply == dense
def test_p11_near_apply_equals_dense():
    pr = make_config("c1")
    nb = pr.nnz * pr.block_len
    B = O.block_entries(pr.blk_seed, 0, nb, pr.s_blk).reshape(pr.nnz, pr.tdim, pr.Nn * pr.sdim)
    cols = pr.P * pr.Nn * pr.sdim
    dense = np.zeros((pr.T * pr.tdim, cols))
    for t in range(pr.T):
        for p in range(pr.row_ptr[t], pr.row_ptr[t + 1]):
            k = pr.panel_idx[p]
            dense[t * pr.tdim:(t + 1) * pr.tdim, k * pr.Nn * pr.sdim:(k + 1) * pr.Nn * pr.sdim] += B[p]
    sig = pr.sigma.reshape(-1)
    u = O.nearcorr_apply(pr.T, pr.tdim, pr.sdim, pr.Nn, pr.row_ptr, pr.panel_idx, B, sig,
                         np.zeros(pr.T * pr.tdim))
    np.testing.assert_allclose(u, dense @ sig, rtol=0, atol=1e-13)
    # the literal near term of the full operator: dense B sigma - smooth re-sum over near panels
    orc = O.Oracle(pr)
    rows = np.arange(0, pr.T, 37)
    _, uf, un = orc.apply_rows(pr.sigma, rows, parts=True)
    sf = O.upsample(pr.sigma.reshape(-1), pr.P, pr.Ns, pr.Nt, pr.Ms, pr.Mt, 1)
    for q, t in enumerate(rows):
        ks = pr.panel_idx[pr.row_ptr[t]:pr.row_ptr[t + 1]]
        m = np.concatenate([np.arange(k * pr.Mn, (k + 1) * pr.Mn) for k in ks]) if ks.size else np.zeros(0, int)
        sm = O.farfield(1, pr.x_trg[t:t + 1], pr.y_f[m], pr.n_f[m], pr.w_f[m], sf[m])[0] if m.size else 0.0
        expect = (dense[t] @ sig) - sm
        assert abs(un[q, 0] - expect) <= 1e-13 * (1 + abs(expect))
        # far + near == far over the NON-near panels + B sigma
        keep = np.setdiff1d(np.arange(pr.M), m)
        ffar = O.farfield(1, pr.x_trg[t:t + 1], pr.y_f[keep], pr.n_f[keep], pr.w_f[keep], sf[keep])[0]
        assert abs((uf[q, 0] + un[q, 0]) - (ffar + dense[t] @ sig)) <= 1e-12 * (1 + abs(ffar))


# ---------------------------------------------------------------- P12 invariances
def test_p12_invariances():
    rng = np.random.default_rng(12)
    b, g = pin_torus(P=8, Ns=8, Nt=12)
    X = rng.uniform(-1.5, 1.5, (9, 3))
    sig1 = rng.standard_normal(g.w.size)
    sig3 = rng.standard_normal(g.y.shape)
    tau3 = rng.standard_normal(g.y.shape)
    eta = np.full(g.w.size, 2.5)
    uL = O.farfield(1, X, g.y, g.n, g.w, sig1)
    uS = O.farfield(2, X, g.y, g.n, g.w, sig3, eta=eta)
    # linearity
    a, c = 0.7, -1.3
    lin = O.farfield(2, X, g.y, g.n, g.w, a * sig3 + c * tau3, eta=eta)
    np.testing.assert_allclose(lin, a * uS + c * O.farfield(2, X, g.y, g.n, g.w, tau3, eta=eta),
                               rtol=0, atol=1e-13 * np.abs(uS).max() * 10)
    # translation
    s = np.array([3.0, -2.0, 0.5])
    np.testing.assert_allclose(O.farfield(1, X + s, g.y + s, g.n, g.w, sig1), uL, rtol=1e-11, atol=1e-14)
    # rotation: Laplace invariant, Stokes rotates with the density
    Q = random_rotation(rng)
    np.testing.assert_allclose(O.farfield(1, X @ Q.T, g.y @ Q.T, g.n @ Q.T, g.w, sig1), uL,
                               rtol=1e-11, atol=1e-13)
    uSr = O.farfield(2, X @ Q.T, g.y @ Q.T, g.n @ Q.T, g.w, sig3 @ Q.T, eta=eta)
    np.testing.assert_allclose(uSr, uS @ Q.T, rtol=1e-11, atol=1e-13)
    # scale x -> lam x, w -> lam^2 w: Laplace DL invariant, Stokes SL x lam, DL invariant
    lam = 2.5
    np.testing.assert_allclose(O.farfield(1, lam * X, lam * g.y, g.n, lam ** 2 * g.w, sig1), uL,
                               rtol=1e-12, atol=1e-14)
    uSL = O.farfield(2, X, g.y, g.n, g.w, sig3, eta=eta) - O.farfield(2, X, g.y, g.n, g.w, sig3, eta=0 * eta)
    uSL2 = (O.farfield(2, lam * X, lam * g.y, g.n, lam ** 2 * g.w, sig3, eta=eta)
            - O.farfield(2, lam * X, lam * g.y, g.n, lam ** 2 * g.w, sig3, eta=0 * eta))
    np.testing.assert_allclose(uSL2, lam * uSL, rtol=1e-11, atol=1e-13)
    uDL = O.farfield(2, X, g.y, g.n, g.w, sig3, eta=0 * eta)
    np.testing.assert_allclose(O.farfield(2, lam * X, lam * g.y, g.n, lam ** 2 * g.w, sig3, eta=0 * eta),
                               uDL, rtol=1e-11, atol=1e-13)


# ---------------------------------------------------------------- P13 projector
def test_p13_projector_identities():
    pr = make_config("c4", n_loops=3, panels=8)
    body = np.repeat(pr.body_of_panel, pr.Nn)
    rng = np.random.default_rng(13)
    sig = rng.standard_normal((pr.N, 3))
    L = lambda s: O.projector(pr.y_c, pr.w_c, body, pr.n_bodies, s)
    Ls = L(sig)
    np.testing.assert_allclose(L(Ls), Ls, atol=1e-12)
    ip = np.sum(pr.w_c[:, None] * Ls * (sig - Ls))
    assert abs(ip) <= 1e-12 * np.sum(pr.w_c[:, None] * sig * sig)
    # rigid motions (different per body) are fixed
    v = np.zeros_like(sig)
    for bb in range(pr.n_bodies):
        m = body == bb
        a, om, c = rng.standard_normal(3), rng.standard_normal(3), rng.standard_normal(3)
        v[m] = a + np.cross(om, pr.y_c[m] - c)
    np.testing.assert_allclose(L(v), v, atol=1e-12)
    # rank 6 per body
    E = np.stack([L(rng.standard_normal((pr.N, 3))).reshape(-1) for _ in range(30)], 1)
    s = np.linalg.svd(E, compute_uv=False)
    assert np.sum(s > 1e-8 * s[0]) == 6 * pr.n_bodies


def test_mobility_operator_rigid_density_is_fixed():
    """(K(I-L)+L) v = v for a rigid v, whatever the blocks: (I-L)v = 0 (Eq. e:new-mobility-bie)."""
    pr = make_config("c4", n_loops=2, panels=6)
    body = np.repeat(pr.body_of_panel, pr.Nn)
    rng = np.random.default_rng(14)
    v = np.zeros((pr.N, 3))
    for bb in range(pr.n_bodies):
        m = body == bb
        v[m] = rng.standard_normal(3) + np.cross(rng.standard_normal(3), pr.y_c[m])
    orc = O.Oracle(pr)
    rows = np.arange(0, pr.n_on, 53)
    u = orc.apply_rows(v, rows)
    np.testing.assert_allclose(u, v[rows], atol=1e-12)


# ---------------------------------------------------------------- RNG & constants
def test_splitmix64_golden():
    lines = [l.split() for l in open(os.path.join(GOLD, "splitmix64_vigna.txt")) if not l.startswith("#")]
    seed = int(lines[0][1])
    vals = [int(l[0]) for l in lines[1:]]
    for i, v in enumerate(vals):
        assert O.splitmix64(seed, i) == v
        assert splitmix64(seed, i) == v


def test_block_entry_statistics():
    s_blk = 1 / 120
    x = O.block_entries(12345, 0, 200000, s_blk)
    assert abs(x.mean()) < 5 * s_blk / np.sqrt(x.size)
    assert abs(x.std() / s_blk - 1) < 0.01
    assert np.abs(x).max() <= np.sqrt(3) * s_blk


def test_eta_printed_values():
    for l in open(os.path.join(GOLD, "paper_constants.txt")):
        if l.startswith("#") or not l.strip():
            continue
        name, rho, val, tol, _ = l.split()
        assert abs(O.eta_cfie(float(rho)) - float(val)) <= float(tol) * float(val)


# ---------------------------------------------------------------- N4: ragged angular orders
# PAPER.md §3.1: element k carries its own N_th^(k).  The oracle's ragged bookkeeping
# (per-panel interpolation, node / fine / block offsets) is pinned by exactness, by the physics of
# a ragged refined torus, and by an independent dense assembly from the generator's offsets.
@pytest.mark.parametrize("ragged_ns", [False, True])
def test_n4_ragged_upsample_exactness(ragged_ns):
    nts = np.array([12, 4, 20, 8, 12, 16])
    nss = np.array([10, 6, 12, 10, 16, 8]) if ragged_ns else np.full(6, 10)
    mts, mss = 2 * nts, 2 * nss
    rng = np.random.default_rng(11)
    cs, fs = [], []
    for p, (ns, nt, ms, mt) in enumerate(zip(nss, nts, mss, mts)):
        coef = rng.standard_normal(ns)                 # degree ns-1 polynomial in t
        a = rng.standard_normal(nt // 2)
        b = rng.standard_normal(nt // 2)
        ny = rng.standard_normal()
        sc, _ = O.gauss_legendre(int(ns))
        sf, _ = O.gauss_legendre(int(ms))
        f = lambda t, th: np.polynomial.polynomial.polyval(t, coef) * (
            sum(a[l] * np.cos(l * th) + b[l] * np.sin(l * th) for l in range(nt // 2)) + ny * np.cos(nt * th / 2))
        cs.append(f(sc[:, None], 2 * np.pi * np.arange(nt)[None, :] / nt).reshape(-1))
        fs.append(f(sf[:, None], 2 * np.pi * np.arange(mt)[None, :] / mt).reshape(-1))
    c, f = np.concatenate(cs), np.concatenate(fs)
    for nc in (1, 3):
        out = O.upsample_ragged(np.repeat(c[:, None], nc, 1) * (1 + np.arange(nc)), nss, nts, mss, mts, nc)
        np.testing.assert_allclose(out.reshape(-1, nc), np.repeat(f[:, None], nc, 1) * (1 + np.arange(nc)),
                                   rtol=0, atol=1e-13 * np.abs(f).max())


def test_n4_ragged_gauss_law():
    """Laplace DL of sigma = 1 on a refined torus whose panels alternate N_th in {32, 48, 64}:
    -1 inside, 0 outside.  sigma_f comes from the oracle's ragged upsample."""
    from synth.geometry import discretize_ragged
    b = torus_body(1.0, 0.1)
    P = 192
    nts = np.array([32, 48, 64])[np.arange(P) % 3]
    g = discretize_ragged(b, P, 10, 2 * nts)
    sf = O.upsample_ragged(np.ones(10 * int(nts.sum())), 10, nts, 10, 2 * nts, 1)   # ms = ns: identity in s
    assert np.abs(sf - 1).max() < 1e-14
    xin, xout = _interior_exterior()
    u = O.farfield(1, np.concatenate([xin, xout]), g.y, g.n, g.w, sf)
    np.testing.assert_allclose(u[:len(xin)], -1.0, rtol=0, atol=1e-12)
    np.testing.assert_allclose(u[len(xin):], 0.0, rtol=0, atol=1e-12)


def test_n4_ragged_uniform_reduces_to_uniform():
    """all N_th^(k) equal: the ragged bookkeeping must give the uniform operator bit for bit"""
    pr = make_config("c2", panels=6)
    import copy
    rg = copy.deepcopy(pr)
    rg.panel_nt = np.full(pr.P, pr.Nt, np.int32)
    rows = np.arange(0, pr.T, 7)
    a = O.Oracle(pr).apply_rows(pr.sigma, rows)
    b = O.Oracle(rg).apply_rows(rg.sigma, rows)
    assert np.array_equal(a, b)


def test_n4_ragged_operator_vs_dense_assembly():
    """c3v (ragged): near term = dense B sigma (blocks placed from the GENERATOR's offsets and the
    generator's counter rule) minus the far sum over the near panels' fine nodes; far + near =
    far over the non-near panels + B sigma."""
    from synth.rng import block_entries_array
    pr = make_config("c3v", panels=8)
    assert pr.ragged and len(set(pr.panel_nt.tolist())) > 1 and len(set(pr.panel_ns.tolist())) > 1
    no, fo, bo = pr.node_off(), pr.fine_off(), pr.blk_off()
    d = pr.sdim
    orc = O.Oracle(pr)
    rows = np.arange(0, pr.T, 97)
    sp, sf, _ = orc.prepare(pr.sigma)
    _, uf, un = orc.apply_rows(pr.sigma, rows, parts=True, prepared=(sp, sf, None))
    # fine density: per-panel uniform upsample with that panel's orders
    nsk, ntk = pr.ns_of_panel(), pr.nt_of_panel()
    sf_ref = np.concatenate([O.upsample(pr.sigma[no[k]:no[k + 1]].reshape(-1), 1, int(nsk[k]), int(ntk[k]),
                                        2 * int(nsk[k]), 2 * int(ntk[k]), d) for k in range(pr.P)]).reshape(-1, d)
    np.testing.assert_array_equal(sf.reshape(-1, d), sf_ref)
    for q, t in enumerate(rows):
        bsig = np.zeros(d)
        ms = []
        for p in range(pr.row_ptr[t], pr.row_ptr[t + 1]):
            k = pr.panel_idx[p]
            nn = no[k + 1] - no[k]
            B = block_entries_array(pr.blk_seed, np.arange(bo[p], bo[p + 1]), pr.s_blk).reshape(d, nn * d)
            bsig += B @ pr.sigma[no[k]:no[k + 1]].reshape(-1)
            ms.append(np.arange(fo[k], fo[k + 1]))
        m = np.concatenate(ms)
        eta = pr.eta_f
        sm = O.farfield(2, pr.x_trg[t:t + 1], pr.y_f[m], pr.n_f[m], pr.w_f[m], sf_ref[m], eta=eta[m])[0]
        np.testing.assert_allclose(un[q], bsig - sm, rtol=0, atol=1e-12 * (1 + np.abs(bsig).max()))
        keep = np.setdiff1d(np.arange(pr.M), m)
        ffar = O.farfield(2, pr.x_trg[t:t + 1], pr.y_f[keep], pr.n_f[keep], pr.w_f[keep], sf_ref[keep],
                          eta=eta[keep])[0]
        np.testing.assert_allclose(uf[q] + un[q], ffar + bsig, rtol=0, atol=1e-11 * (1 + np.abs(ffar).max()))


def test_graded_panels_geometry_and_gauss_law():
    """adaptive (non-uniform) panels in s: the generator's weights still integrate the
    torus area exactly and the Laplace DL of 1 is -1 inside / 0 outside"""
    from synth.geometry import discretize, panel_arclength
    b = torus_body(1.0, 0.1)
    P = 320
    h = np.geomspace(1.0, 2.5, P // 2)
    br = np.concatenate([[0.0], np.cumsum(np.concatenate([h, h[::-1]]))])
    br /= br[-1]
    g = discretize(b, P, 10, 48, br)
    assert abs(g.w.sum() - 4 * np.pi ** 2 * 0.1) < 1e-13
    assert abs(panel_arclength(b, P, br).sum() - 2 * np.pi) < 1e-13
    xin, xout = _interior_exterior()
    u = O.farfield(1, np.concatenate([xin, xout]), g.y, g.n, g.w, np.ones(g.w.size))
    np.testing.assert_allclose(u[:len(xin)], -1.0, rtol=0, atol=1e-11)
    np.testing.assert_allclose(u[len(xin):], 0.0, rtol=0, atol=1e-11)
