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


def sedimentation_speed(rho, panels, Ns=10, Nt=12, order=14, beta=0.6, tol=1e-14):
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
