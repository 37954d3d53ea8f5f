"""Laplace single layer on the GPU: the combined field D + eta S_L of the Laplace CFIE
(PAPER.md Eq. e:laplace-bie-new) through the operator, against the oracle; and the paper's
Green's representation convergence table (Table t:conv-biest, P:L2085-2114,
tests/golden/greens_rep_conv_biest.txt) reproduced with special-quadrature blocks:

    on the surface  u = u/2 + S_L[du/dn] - D[u]   (Eq. e:greens-rep),  u = G(x - x0), x0 = (1,2,3)
    e_inf = max |S_L[du/dn] - (1/2 + D)[u]|  over the nodes.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_config, make_torus_problem  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
FOUR_PI = 4 * np.pi


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.float64)


def _skip():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("eta", [0.7, 3.0])
@pytest.mark.parametrize("path", ["const", "tma"])
def test_laplace_combined_field_parity(eta, path, monkeypatch):
    """c1 (torus, 960 nodes + 200 off-surface targets) with the Laplace CFIE kernel D + eta S_L"""
    _skip()
    monkeypatch.setenv("SLB_FAR_PATH", path)
    from harness import DeviceProblem
    pr = make_config("c1")
    pr.eta_f = np.full_like(pr.eta_f, eta)
    pr.eta_body = np.full_like(pr.eta_body, eta)
    dp = DeviceProblem(pr)
    u = dp.matvec().cpu().numpy()[:, 0]
    dp.close()
    ref = O.Oracle(pr).apply_rows(pr.sigma, np.arange(pr.T))[:, 0]
    assert np.abs(u - ref).max() / np.abs(ref).max() <= 1e-12


def golden():
    rows = []
    for line in open(os.path.join(HERE, "golden", "greens_rep_conv_biest.txt")):
        if line.strip() and not line.startswith("#"):
            f = line.split()
            rows.append((int(f[0]), int(f[1]), int(f[2]), float(f[3])))
    return rows


def greens_rep_error(P, nt, order=0, beta=0.6):
    from harness import DeviceProblem
    quad = dict(order=order, beta=beta)
    pr = make_torus_problem(R=1.0, rho=0.25, panels=P, Ns=10, Nt=nt, kernel=1)
    x0 = np.array([1.0, 2.0, 3.0])
    d = pr.y_c - x0
    rr = np.sqrt((d * d).sum(1))
    u = 1.0 / (FOUR_PI * rr)
    dudn = -(d * pr.n_c).sum(1) / (FOUR_PI * rr ** 3)
    dl = DeviceProblem(pr, quad=quad)                         # (1/2 + D)
    A = dl.matvec(cu(u[:, None])).cpu().numpy()[:, 0]
    dl.close()
    sl = DeviceProblem(pr, quad=quad, single_layer=True)      # S_L
    B = sl.matvec(cu(dudn[:, None])).cpu().numpy()[:, 0]
    sl.close()
    return np.abs(B - A).max(), pr.N


@pytest.mark.parametrize("row", range(4))
def test_greens_representation_convergence_table(row):
    """our e_inf at the paper's discretizations (N_elem, N_s = 10, N_theta) is at most the paper's
    CSBQ error (times 2, plus 1e-12): the same Nystrom discretization converges as printed"""
    _skip()
    n_unk, P, nt, e_paper = golden()[row]
    e, N = greens_rep_error(P, nt)
    assert N == n_unk
    print(f"N={N} P={P} Nt={nt}: e_inf = {e:.2e} (paper {e_paper:.1e})")
    assert e <= 2.0 * e_paper + 1e-12, (e, e_paper)
