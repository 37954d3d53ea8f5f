"""(NEXT N1) Special-quadrature correction blocks computed on the GPU (slb_nearcorr_quad).

Pins that do not come from the implementation itself:
  * physics: with the special blocks the discrete operator satisfies the jump relations the paper
    relies on -- Laplace (I/2 + D)[1] = 0 on the surface and D[1] = -1 / 0 just inside / outside
    (P:L1455-1460); Stokes (I/2 + D)[v] = 0 for rigid v (Prop. 1) and D[v] = -v / 0 off it;
  * an independent integrator: B sigma for sample (target, panel) pairs -- singular (target on the
    panel) and near-singular -- against scipy adaptive Gauss-Kronrod in polar coordinates around
    the closest point on the EXACT analytic surface (the GPU uses the interpolated surface).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_torus_problem, torus_body  # noqa: E402

QUAD = dict(order=0)   # the paper's rule (modal angular sums, Bernstein s-panels, singular log rule)


def cu(a, dt=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to("cuda", dt or torch.float64)


def _skip():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def near_surface_targets(R=1.0, rho=0.1, n=24, seed=3):
    """points at 0.5, 0.9, 0.99 rho (inside) and 1.01, 1.1, 1.5 rho (outside) from the centerline"""
    rng = np.random.default_rng(seed)
    out, inside = [], []
    for f in (0.5, 0.9, 0.99, 1.01, 1.1, 1.5):
        for _ in range(n // 6):
            ph, th = rng.uniform(0, 2 * np.pi, 2)
            c = np.array([R * np.cos(ph), R * np.sin(ph), 0.0])
            er = np.array([np.cos(ph), np.sin(ph), 0.0])
            out.append(c + f * rho * (np.cos(th) * np.array([0, 0, 1.0]) + np.sin(th) * er))
            inside.append(f < 1)
    return np.array(out), np.array(inside)


def test_laplace_gauss_law_with_special_blocks():
    _skip()
    from harness import DeviceProblem
    X, inside = near_surface_targets()
    pr = make_torus_problem(panels=16, extra_targets=X)
    dp = DeviceProblem(pr, quad=QUAD)
    u = dp.matvec(cu(np.ones((pr.N, 1)))).cpu().numpy()[:, 0]
    dp.close()
    on = u[:pr.n_on]                         # (I/2 + D)[1] = 1/2 - 1/2 = 0
    off = u[pr.n_on:]                        # c_I = 0 off the surface: D[1] = -1 inside, 0 outside
    assert np.abs(on).max() < 1e-9, np.abs(on).max()
    np.testing.assert_allclose(off, np.where(inside, -1.0, 0.0), atol=1e-9)


@pytest.mark.parametrize("mode", ["translation", "rotation"])
def test_stokes_dl_rigid_motion_with_special_blocks(mode):
    _skip()
    from harness import DeviceProblem
    X, inside = near_surface_targets(seed=4)
    pr = make_torus_problem(panels=16, kernel=2, eta=0.0, extra_targets=X)
    rng = np.random.default_rng(9)
    if mode == "translation":
        a = rng.standard_normal(3)
        v = np.tile(a, (pr.N, 1))
        vx = np.tile(a, (X.shape[0], 1))
    else:
        om, c = rng.standard_normal(3), rng.standard_normal(3) * 0.2
        v = np.cross(om, pr.y_c - c)
        vx = np.cross(om, X - c)
    dp = DeviceProblem(pr, quad=QUAD)
    u = dp.matvec(cu(v)).cpu().numpy()
    dp.close()
    assert np.abs(u[:pr.n_on]).max() < 1e-8 * np.abs(v).max()        # (I/2 + D) v = 0  (Prop. 1)
    np.testing.assert_allclose(u[pr.n_on:], np.where(inside[:, None], -vx, 0.0), atol=1e-8 * np.abs(v).max())


# panel grids x rule orders that take every shared-memory layout of the regular-cell path (see
# nearquad_run's layout_of): t rows in chunks (12 x 20 and 8 x 8 at order 24, 256 threads), groups of 4
# cells (10 x 12 at order 6), 512-thread CTAs with groups of 2 (16 x 64 at order 14) and the rings
# kept apart from U (Laplace 16 x 64 at order 24: 4 cells per update, 2 per phase)
LAYOUTS = [(2, 12, 20, 24, 1e-9), (2, 8, 8, 24, 1e-9), (2, 10, 12, 6, 1e-5), (2, 16, 64, 14, 1e-9),
           (1, 16, 64, 24, 1e-9)]


@pytest.mark.parametrize("kernel,Ns,Nt,order,tol", LAYOUTS)
def test_jump_relations_across_layouts(kernel, Ns, Nt, order, tol):
    """the same jump relations as above for each layout variant (tolerance from the rule's
    ~2.76^(-2q) accuracy at beta = 0.6): Laplace (I/2 + D)[1] = 0, D[1] = -1 / 0; Stokes (I/2 + D)[v] = 0,
    D[v] = -v / 0 for a rigid translation v"""
    _skip()
    from harness import DeviceProblem
    X, inside = near_surface_targets(seed=5)
    pr = make_torus_problem(panels=16, Ns=Ns, Nt=Nt, kernel=kernel, eta=0.0 if kernel == 2 else None,
                            extra_targets=X)
    a = np.array([0.3, -1.0, 0.7])[:pr.sdim] if kernel == 2 else np.ones(1)
    v = np.tile(a, (pr.N, 1))
    dp = DeviceProblem(pr, quad=dict(order=order, beta=0.6))
    u = dp.matvec(cu(v)).cpu().numpy()
    dp.close()
    assert np.abs(u[:pr.n_on]).max() < tol, np.abs(u[:pr.n_on]).max()
    exp = np.where(inside[:, None], -np.tile(a, (X.shape[0], 1)), 0.0)
    np.testing.assert_allclose(u[pr.n_on:], exp, atol=tol)


# ------------------------------------------------------------------ independent integrator
def _exact_panel_integral(body, P, k, Ns, Nt, sig_panel, x, kind, eta, t0=None, h0=None):
    """int int K(x - y(t,th)) sigma_interp(t,th) J dt dth over panel k, t in [-1,1] local, polar
    coordinates around (t0, h0) (the singular node or the closest point), scipy adaptive GK
    (quad_vec: all components share one adaptive subdivision, max-norm error control)."""
    H = 1e-30
    tg, _ = O.gauss_legendre(Ns)

    def surf(t, th):
        s = (k + (t + 1) / 2) / P
        return body.surface(np.array([s]), np.array([th]))[0]

    def frame(t, th):
        y = surf(t, th)
        yt = body.surface(np.array([(k + (t + 1j * H + 1) / 2) / P]), np.array([th + 0j]))[0].imag / H
        yh = body.surface(np.array([(k + (t + 1) / 2) / P + 0j]), np.array([th + 1j * H]))[0].imag / H
        cr = np.cross(yh, yt)
        J = np.linalg.norm(cr)
        return y, cr / J, J, yt, yh

    def basis(t, th):
        lt = O.lagrange_matrix(tg, np.array([t]))[0]
        ph = th - 2 * np.pi * np.arange(Nt) / Nt
        with np.errstate(divide="ignore", invalid="ignore"):
            C = np.where(np.abs(np.sin(ph / 2)) < 1e-15, 1.0, np.sin(Nt * ph / 2) / np.tan(ph / 2) / Nt)
        return np.outer(lt, C)

    def F(t, th):
        y, n, J, _, _ = frame(t, th)
        r = x - y
        rr = np.linalg.norm(r)
        s = np.tensordot(basis(t, th), sig_panel, axes=([0, 1], [0, 1]))      # sigma_interp
        if kind == 1:
            return (r @ n) / (4 * np.pi * rr ** 3) * s * J
        S = (np.eye(3) / rr + np.outer(r, r) / rr ** 3) / (8 * np.pi)
        D = 3 / (4 * np.pi) * (r @ n) * np.outer(r, r) / rr ** 5
        return (eta * S + D) @ s * J

    _, _, _, yt, yh = frame(t0, h0)
    St, Sh = np.linalg.norm(yt), np.linalg.norm(yh)
    amin, amax, bmin, bmax = (-1 - t0) * St, (1 - t0) * St, -np.pi * Sh, np.pi * Sh

    def R(phi):
        c, s = np.cos(phi), np.sin(phi)
        rs = []
        if c > 1e-300: rs.append(amax / c)
        if c < -1e-300: rs.append(amin / c)
        if s > 1e-300: rs.append(bmax / s)
        if s < -1e-300: rs.append(bmin / s)
        return min(rs)

    corners = sorted(np.mod([np.arctan2(b, a) for a in (amin, amax) for b in (bmin, bmax)], 2 * np.pi))
    from scipy.integrate import quad_vec

    def inner(phi):     # all components at once: one adaptive rule per ray
        c, s = np.cos(phi), np.sin(phi)
        g = lambda rho: np.atleast_1d(F(t0 + rho * c / St, h0 + rho * s / Sh)) * rho / (St * Sh)
        return quad_vec(g, 0, R(phi), epsabs=1e-13, epsrel=1e-11, norm="max", limit=200)[0]
    return quad_vec(inner, 0, 2 * np.pi, points=corners, epsabs=1e-13, epsrel=1e-10, norm="max", limit=400)[0]


@pytest.mark.parametrize("kind", [1, 2])
def test_blocks_vs_independent_integrator(kind):
    _skip()
    import paper_2310_00889_b200 as S
    pr = make_torus_problem(panels=12, kernel=kind, extra_targets=np.array([[1.0, 0.0, 0.112], [0.0, 1.003, 0.1]]))
    body = torus_body(1.0, 0.1)
    rng = np.random.default_rng(2)
    d = pr.sdim
    sig = rng.standard_normal((pr.N, d))
    Nn = pr.Nn
    # sample pairs: a node target on its own panel (singular), a node target on the neighbour panel,
    # and the two off-surface targets on their nearest panel
    t_sing = 3 * Nn + 4 * pr.Nt + 5                 # node (i=4, j=5) of panel 3
    t_edge = 3 * Nn + 9 * pr.Nt + 2                 # last GL ring of panel 3, evaluated on panel 4
    pairs = [(t_sing, 3), (t_edge, 4), (pr.n_on, None), (pr.n_on + 1, None)]
    rows, pids = [], []
    for t, k in pairs:
        ks = pr.panel_idx[pr.row_ptr[t]:pr.row_ptr[t + 1]]
        if k is None:
            dist = [np.min(np.linalg.norm(pr.y_c[kk * Nn:(kk + 1) * Nn] - pr.x_trg[t], axis=1)) for kk in ks]
            k = int(ks[int(np.argmin(dist))])
        assert k in ks
        rows.append(t)
        pids.append(k)
    rp = np.arange(len(rows) + 1, dtype=np.int64)
    trg_node = np.array([t if t < pr.n_on else -1 for t in rows], np.int64)
    blocks = torch.empty(len(rows) * pr.block_len, dtype=torch.float64, device="cuda")
    eta_panel = cu(pr.eta_body[pr.body_of_panel]) if kind == 2 else None
    S.slb_nearcorr_quad(kind, cu(pr.x_trg[rows]), cu(rp, torch.int64), cu(np.array(pids, np.int32), torch.int32),
                        pr.Ns, pr.Nt, cu(pr.y_c.reshape(pr.P, Nn, 3)), blocks, trg_node=cu(trg_node, torch.int64),
                        eta_panel=eta_panel, **QUAD)
    B = blocks.cpu().numpy().reshape(len(rows), d, Nn * d)
    eta = pr.eta_body[0] if kind == 2 else 0.0
    for q, (t, k) in enumerate(zip(rows, pids)):
        sp = sig[k * Nn:(k + 1) * Nn].reshape(pr.Ns, pr.Nt, d)
        got = B[q] @ sig[k * Nn:(k + 1) * Nn].reshape(-1)
        if t < pr.n_on and t // Nn == k:
            loc = t - k * Nn
            tg, _ = O.gauss_legendre(pr.Ns)
            t0, h0 = tg[loc // pr.Nt], 2 * np.pi * (loc % pr.Nt) / pr.Nt
        else:   # closest point on the exact surface (dense sampling + local refinement)
            tt = np.linspace(-1, 1, 201)
            hh = np.linspace(0, 2 * np.pi, 400, endpoint=False)
            Tg, Hg = np.meshgrid(tt, hh, indexing="ij")
            Y = body.surface(((k + (Tg + 1) / 2) / pr.P).reshape(-1), Hg.reshape(-1))
            i = np.argmin(np.linalg.norm(Y - pr.x_trg[t], axis=1))
            t0, h0 = Tg.reshape(-1)[i], Hg.reshape(-1)[i]
            from scipy.optimize import minimize
            res = minimize(lambda z: np.linalg.norm(body.surface(np.array([(k + (np.clip(z[0], -1, 1) + 1) / 2) / pr.P]),
                                                                 np.array([z[1]]))[0] - pr.x_trg[t]),
                           [t0, h0], method="Nelder-Mead", options=dict(xatol=1e-12, fatol=1e-15))
            t0, h0 = float(np.clip(res.x[0], -1, 1)), float(res.x[1])
        ref = _exact_panel_integral(body, pr.P, k, pr.Ns, pr.Nt, sp, pr.x_trg[t], kind, eta, t0, h0)
        err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-3)
        assert err < 1e-8, (t, k, got, ref, err)


# ------------------------------------------------------------------ edge cases of the entry point
def _torus_inputs(pr):
    rp = cu(pr.row_ptr, torch.int64)
    pi = cu(pr.panel_idx, torch.int32)
    return cu(pr.x_trg), rp, pi, cu(pr.y_c)


def test_nearcorr_quad_edge_cases():
    """empty CSR rows leave the blocks untouched; bad orders / panel grids are rejected with the
    library's error codes; a target 1e-12 rho off the surface (but off the nodes) either gets finite
    blocks or a clean 'cell budget' error -- never NaN, never a hang"""
    _skip()
    import paper_2310_00889_b200 as S
    from paper_2310_00889_b200 import SlbError
    pr = make_torus_problem(panels=6, Ns=8, Nt=8)
    x, rp, pi, y = _torus_inputs(pr)
    # every row empty
    rp0 = torch.zeros_like(rp)
    blocks = torch.full((8,), 7.0, dtype=torch.float64, device="cuda")
    S.slb_nearcorr_quad(1, x, rp0, pi[:1], pr.Ns, pr.Nt, y, blocks)
    assert torch.all(blocks == 7.0)
    nb = pr.n_blocks_entries()
    blocks = torch.empty(nb, dtype=torch.float64, device="cuda")
    for order in (3, 25):
        with pytest.raises(SlbError, match="INVALID_ARG|order"):
            S.slb_nearcorr_quad(1, x, rp, pi, pr.Ns, pr.Nt, y, blocks, order=order)
    with pytest.raises(SlbError, match="UNSUPPORTED|too large"):
        S.slb_nearcorr_quad(1, x, rp, pi, pr.Ns, 66, y, blocks)
    # a target just off the surface, between nodes, against its own panel (no trg_node: off-surface)
    body = torus_body(1.0, 0.1)
    s0, th0 = (0.5 + 0.37) / 6, 0.41                          # inside panel 0, between its nodes
    p0 = body.surface(np.array([s0]), np.array([th0]))[0]
    c0 = body.surface(np.array([s0]), np.array([th0 + np.pi]))[0]
    nrm = (p0 - c0) / np.linalg.norm(p0 - c0)                 # outward (circular cross-section)
    xt = cu((p0 + 1e-12 * 0.1 * nrm)[None, :])
    rp1 = cu(np.array([0, 1]), torch.int64)
    pi1 = cu(np.array([0]), torch.int32)
    b1 = torch.empty(pr.Ns * pr.Nt, dtype=torch.float64, device="cuda")
    for order in (0, 14):
        try:
            S.slb_nearcorr_quad(1, xt, rp1, pi1, pr.Ns, pr.Nt, y, b1, order=order)
        except SlbError as e:
            assert "budget" in str(e) or "UNSUPPORTED" in str(e), e
        else:
            assert torch.isfinite(b1).all()
