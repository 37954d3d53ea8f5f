"""(NEXT N1 + N2) The whole GPU path against numbers the paper prints: the sedimentation speed
of a ring, PAPER.md Table t:conv-sbt (values in tests/golden/ring_sedimentation.txt).

Problem: torus R = 1, minor radius rho, axial force F = (0,0,-1), zero torque,
unit viscosity, no slip.  Stokes mobility CFIE, Eq. e:new-mobility-bie:

    (K (I - L) + L) sigma = -S[nu],       K = I/2 + D + eta S,  eta = 1/(2 rho ln(1/rho))
    nu = alpha + beta x (x - c),  int nu = F, int nu x (x - c) = T   (completion flow, P:L1903-1912:
                                                                       a 6x6 system on the surface rule)
    V = -L sigma                                                      (Eq. e:recover-rigidbody-motion)

Everything that touches the operator runs on the GPU through libslb: the special-quadrature
blocks (slb_nearcorr_quad), the operator applies (slb_matvec) and the solve (slb_gmres).
S[nu] uses linearity in eta: S = K_{eta=1} - K_{eta=0} (both without the projector).  V is read
off with the oracle's projector (test infrastructure).  The expected speeds are the paper's
(reference values accurate to 13 digits; the paper's own BIE errors are 1e-14 .. 9e-13).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def golden():
    out = {}
    for line in open(os.path.join(HERE, "golden", "ring_sedimentation.txt")):
        if line.strip() and not line.startswith("#"):
            rho, u, _ = line.split()
            out[float(rho)] = float(u)
    return out


def completion_density(y, w, center, F, Tq):
    """nu = alpha + beta x (y - c) with int nu = F, int nu x (y - c) = Tq, 6x6 solve."""
    d = y - center
    A = np.zeros((6, 6))
    # unknowns (alpha, beta); rows: force (3), torque (3)
    e = np.eye(3)
    for k in range(3):
        nu_a = np.tile(e[k], (y.shape[0], 1))                 # d nu / d alpha_k
        nu_b = np.cross(e[k], d)                               # d nu / d beta_k
        for col, nu in ((k, nu_a), (3 + k, nu_b)):
            A[:3, col] = (w[:, None] * nu).sum(0)
            A[3:, col] = (w[:, None] * np.cross(nu, d)).sum(0)
    ab = np.linalg.solve(A, np.concatenate([F, Tq]))
    return ab[:3] + np.cross(ab[3:], d)


def sedimentation_speed(rho, panels, Ns=10, Nt=12, order=0, beta=0.6, tol=1e-14):
    import oracle as O
    from harness import DeviceProblem
    from synth import make_torus_problem

    quad = dict(order=order, beta=beta)
    pr = make_torus_problem(rho=rho, panels=panels, Ns=Ns, Nt=Nt, kernel=2)
    nu = completion_density(pr.y_c, pr.w_c, np.zeros(3), np.array([0.0, 0.0, -1.0]), np.zeros(3))
    nu_d = torch.from_numpy(np.ascontiguousarray(nu)).cuda()
    Knu = []
    for e in (1.0, 0.0):
        p = make_torus_problem(rho=rho, panels=panels, Ns=Ns, Nt=Nt, kernel=2, eta=e)
        dp = DeviceProblem(p, quad=quad)
        Knu.append(dp.matvec(nu_d).clone())
        dp.close()
    rhs = (Knu[1] - Knu[0]).contiguous()                       # -S[nu]
    pr.projector = True
    dp = DeviceProblem(pr, quad=quad)
    x, it, rr = dp.op.gmres(rhs, restart=100, max_iters=500, tol=tol)
    torch.cuda.synchronize()
    dp.close()
    sig = x.cpu().numpy()
    V = -O.projector(pr.y_c, pr.w_c, np.zeros(pr.N, np.int32), 1, sig)
    return V, it, rr, pr


# (rho, panels, N_theta): coarse grids of the kind the paper uses for these rings
CASES = [(1e-1, 16, 12), (1e-2, 24, 12), (1e-3, 24, 8), (1e-4, 24, 8), (1e-5, 24, 8)]
TOL = {1e-1: 1e-12, 1e-2: 5e-12, 1e-3: 5e-12, 1e-4: 1e-11, 1e-5: 2e-9}   # measured 1e-14 .. 4e-10


@pytest.mark.parametrize("rho,panels,nt", CASES)
def test_ring_sedimentation_speed(rho, panels, nt):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    U_exact = golden()[rho]
    V, it, rr, pr = sedimentation_speed(rho, panels, Nt=nt)
    assert rr < 1e-13, (it, rr)
    # the recovered rigid motion is a pure downward translation (symmetry)
    Vz = V[:, 2]
    assert np.abs(V[:, :2]).max() < 1e-10 * abs(Vz).max()
    assert np.ptp(Vz) < 1e-10 * abs(Vz).max()
    U = -float(np.average(Vz, weights=pr.w_c))
    err = abs(U - U_exact) / U_exact
    print(f"rho={rho:g} P={panels} Nt={nt} N={pr.N} gmres it={it} U={U:.15e} exact={U_exact:.15e} rel.err={err:.2e}")
    assert err < TOL[rho], (U, U_exact, err)


# ------------------------------------------------------------------ the library's mobility solve
def _mobility_ops(pr, quad):
    from harness import DeviceProblem
    p = __import__("copy").copy(pr)
    p.projector = True
    return DeviceProblem(p, quad=quad), DeviceProblem(pr, quad=quad, single_layer=True)


@pytest.mark.parametrize("rho,panels,nt", [(1e-1, 16, 12), (1e-2, 24, 12)])
def test_mobility_solve_ring_sedimentation(rho, panels, nt):
    """slb_mobility_solve (completion flow + S apply + GMRES + V = -L sigma inside libslb) gives the
    paper's sedimentation speed (Table t:conv-sbt)"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from synth import make_torus_problem
    pr = make_torus_problem(rho=rho, panels=panels, Nt=nt, kernel=2)
    mob, sl = _mobility_ops(pr, dict(order=0))
    rig, sig, it, rr = mob.op.mobility_solve(sl.op, [[0, 0, -1.0, 0, 0, 0]], tol=1e-14)
    mob.close(); sl.close()
    U = -rig[0, 2]
    ex = golden()[rho]
    assert np.abs(rig[0, [0, 1, 3, 4, 5]]).max() < 1e-10 * abs(U)      # pure translation along the axis
    assert abs(U - ex) / ex < TOL[rho], (U, ex, it, rr)


def test_mobility_solve_two_bodies_matches_assembled():
    """two close rings, random forces and torques: the library's solve equals the same solve
    assembled step by step outside it (6x6 completion systems, K_1 - K_0 for S, GMRES, and V read
    with the oracle's Gram-Schmidt projector)"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle as O
    from harness import DeviceProblem
    from synth import make_config
    quad = dict(order=0)
    pr = make_config("c3", panels=10)                  # two tori, gap r/20, per-body eta
    rng = np.random.default_rng(3)
    ft = rng.standard_normal((2, 6))
    body = np.repeat(pr.body_of_panel, np.diff(pr.node_off()))
    cent = np.array([np.average(pr.y_c[body == b], axis=0, weights=pr.w_c[body == b]) for b in range(2)])
    mob, sl = _mobility_ops(pr, quad)
    rig, sig, it, rr = mob.op.mobility_solve(sl.op, ft, tol=1e-13)
    mob.close(); sl.close()
    # assembled
    nu = np.zeros((pr.N, 3))
    for b in range(2):
        m = body == b
        nu[m] = completion_density(pr.y_c[m], pr.w_c[m], cent[b], ft[b, :3], ft[b, 3:])
    nu_d = torch.from_numpy(nu).cuda()
    import copy
    Knu = []
    for e in (1.0, 0.0):
        p = copy.copy(pr)
        p.eta_f = np.full_like(pr.eta_f, e)
        p.eta_body = np.full_like(pr.eta_body, e)
        dp = DeviceProblem(p, quad=quad)
        Knu.append(dp.matvec(nu_d).clone())
        dp.close()
    p = copy.copy(pr)
    p.projector = True
    dp = DeviceProblem(p, quad=quad)
    x, it2, rr2 = dp.op.gmres((Knu[1] - Knu[0]).contiguous(), restart=100, max_iters=1000, tol=1e-13)
    dp.close()
    V = -O.projector(pr.y_c, pr.w_c, body.astype(np.int32), 2, x.cpu().numpy())
    for b in range(2):
        m = np.nonzero(body == b)[0]
        d = pr.y_c[m] - cent[b]
        Vb = rig[b, :3] + np.cross(rig[b, 3:], d)                 # library's rigid motion at the nodes
        np.testing.assert_allclose(Vb, V[m], rtol=0, atol=1e-9 * np.abs(V).max())


def test_ring_sedimentation_graded_ragged_mesh():
    """adaptive-style mesh: geometrically graded panels in s and mixed N_th per panel;
    the paper's sedimentation speed at rho = 1e-2 must still come out (Table t:conv-sbt)"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle as O
    from harness import DeviceProblem
    from synth import make_torus_problem
    rho, P = 1e-2, 24
    h = np.geomspace(1.0, 3.0, P // 2)
    br = np.concatenate([[0.0], np.cumsum(np.concatenate([h, h[::-1]]))])
    br /= br[-1]
    nts = np.array([12, 8] * (P // 2), np.int32)
    quad = dict(order=0)
    mk = lambda **kw: make_torus_problem(rho=rho, panels=P, kernel=2, nt_panels=nts, breaks=br, **kw)
    pr = mk()
    nu = completion_density(pr.y_c, pr.w_c, np.zeros(3), np.array([0.0, 0.0, -1.0]), np.zeros(3))
    mob, sl = _mobility_ops(pr, quad)
    rig, sig, it, rr = mob.op.mobility_solve(sl.op, [[0, 0, -1.0, 0, 0, 0]], tol=1e-14)
    mob.close(); sl.close()
    U = -rig[0, 2]
    ex = golden()[rho]
    assert abs(U - ex) / ex < 5e-12, (U, ex, it, rr)
