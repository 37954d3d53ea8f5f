"""(NEXT N4) Ragged angular orders on the GPU: element k carries its own N_th^(k)
(§3.1; the close-touching mesh is adaptive in N_th up to 88).

Parity against the CPU oracle (whose ragged bookkeeping is pinned in test_oracle_pins.py) on the
same seeded inputs at the north_star tolerance, plus physics with the special-quadrature blocks
and the paper's ring sedimentation speed on a ragged mesh."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_config, make_torus_problem  # noqa: E402

TOL = 1e-12


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def cu(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_00889_b200 as S
    return S


@pytest.mark.parametrize("nc", [1, 3])
@pytest.mark.parametrize("ragged_ns", [False, True])
def test_upsample_ragged_parity(S, nc, ragged_ns):
    rng = np.random.default_rng(5 + nc)
    nts = rng.choice([4, 8, 12, 20, 40, 64], size=37).astype(np.int32)
    nss = rng.choice([4, 10, 12, 16], size=37).astype(np.int32) if ragged_ns else np.full(37, 10, np.int32)
    mts, mss = 2 * nts, 2 * nss
    sc = rng.standard_normal(int((nss.astype(np.int64) * nts).sum()) * nc)
    g = S.slb_upsample_ragged(cu(sc), nss, nts, mss, mts, nc).cpu().numpy()
    ref = O.upsample_ragged(sc, nss, nts, mss, mts, nc)
    assert rel(g, ref) <= TOL


def _vs_oracle(pr, rows=None, **kw):
    from harness import DeviceProblem
    dp = DeviceProblem(pr, **kw)
    u = dp.matvec().cpu().numpy().reshape(pr.T, pr.tdim)
    u2 = dp.matvec().cpu().numpy().reshape(pr.T, pr.tdim)
    dp.close()
    rows = np.arange(pr.T) if rows is None else rows
    ref = O.Oracle(pr).apply_rows(pr.sigma, rows)
    return rel(u[rows], ref), u, u2


@pytest.mark.parametrize("kw", [dict(panels=8), dict(panels=12)])
@pytest.mark.parametrize("path", ["const", "tma"])
def test_matvec_ragged_parity_small(S, kw, path, monkeypatch):
    monkeypatch.setenv("SLB_FAR_PATH", path)
    pr = make_config("c3v", **kw)
    assert pr.ragged and len(set(pr.panel_nt.tolist())) > 1 and len(set(pr.ns_of_panel().tolist())) > 1
    err, u, u2 = _vs_oracle(pr)
    assert err <= TOL, err
    assert np.array_equal(u, u2)


def test_matvec_ragged_parity_full_size_sampled(S):
    pr = make_config("c3v")
    rng = np.random.default_rng(4)
    gap = np.argsort(np.abs(pr.x_trg[:, 0] - 1.05125))[:48]          # targets at the close-touching gap
    nn = np.diff(pr.row_ptr)
    rows = np.unique(np.concatenate([gap, rng.choice(pr.T, 160, replace=False), np.argsort(nn)[-16:],
                                     [0, pr.T - 1]]))
    err, _, _ = _vs_oracle(pr, rows)
    assert err <= TOL, err


def test_matvec_ragged_mobility_parity(S):
    """ragged torus with the rigid-motion projector (K(I-L) + L); rigid densities are fixed points"""
    nts = np.array([8, 12, 16, 12] * 3, np.int32)
    pr = make_torus_problem(rho=0.1, panels=12, kernel=2, nt_panels=nts)
    pr.projector = True
    err, u, _ = _vs_oracle(pr)
    assert err <= TOL, err
    from harness import DeviceProblem
    rng = np.random.default_rng(2)
    v = rng.standard_normal(3) + np.cross(rng.standard_normal(3), pr.y_c)
    dp = DeviceProblem(pr)
    np.testing.assert_allclose(dp.matvec(cu(v)).cpu().numpy(), v, atol=1e-12)
    dp.close()


def test_ragged_equal_orders_match_uniform_bitwise(S):
    """panel_nt all equal to Nt: the ragged engine returns the uniform operator's u bit for bit"""
    import copy
    from harness import DeviceProblem
    pr = make_config("c2", panels=8)
    rg = copy.deepcopy(pr)
    rg.panel_nt = np.full(pr.P, pr.Nt, np.int32)
    a = DeviceProblem(pr).matvec().cpu().numpy()
    b = DeviceProblem(rg).matvec().cpu().numpy()
    assert np.array_equal(a, b)


def test_gmres_ragged_manufactured(S):
    from harness import DeviceProblem
    pr = make_config("c3v", panels=6)
    # the synthetic B entries (R10) are random, not a quadrature: at the close-touching gap with
    # wide blocks they make I/2 + K far from well-conditioned; shrink them (both sides read s_blk)
    pr.s_blk *= 0.05
    rng = np.random.default_rng(8)
    xs = rng.standard_normal(pr.sigma.shape)
    b = O.Oracle(pr).apply_rows(xs, np.arange(pr.T)).reshape(pr.sigma.shape)
    dp = DeviceProblem(pr)
    x, it, rr = dp.op.gmres(cu(b), restart=80, max_iters=2000, tol=1e-13)
    dp.close()
    assert rr <= 1e-13, (it, rr)
    assert np.abs(x.cpu().numpy() - xs).max() / np.abs(xs).max() <= 1e-9


# ------------------------------------------------------------------ with special-quadrature blocks (N1)
@pytest.mark.parametrize("order", [0, 10], ids=["paper_modal", "adaptive2d"])
def test_ragged_quad_blocks_equal_orders_match_uniform(S, order):
    """slb_nearcorr_quad_ragged with all orders equal reproduces the uniform blocks bit for bit"""
    import paper_2310_00889_b200 as P
    pr = make_torus_problem(panels=8, kernel=2)
    x = cu(pr.x_trg)
    rp, pi = cu(pr.row_ptr, torch.int64), cu(pr.panel_idx, torch.int32)
    tn = cu(np.arange(pr.T), torch.int64)
    eta = cu(pr.eta_body[pr.body_of_panel])
    b1 = torch.empty(pr.nnz * pr.block_len, dtype=torch.float64, device="cuda")
    b2 = torch.empty_like(b1)
    P.slb_nearcorr_quad(2, x, rp, pi, pr.Ns, pr.Nt, cu(pr.y_c), b1, trg_node=tn, eta_panel=eta, order=order)
    P.slb_nearcorr_quad(2, x, rp, pi, pr.Ns, pr.Nt, cu(pr.y_c), b2, trg_node=tn, eta_panel=eta, order=order,
                        panel_nt=np.full(pr.P, pr.Nt))
    assert torch.equal(b1, b2)


def test_ragged_gauss_law_with_special_blocks(S):
    """Laplace (I/2 + D)[1] = 0 on a ragged torus, D[1] = -1 / 0 just inside / outside"""
    from harness import DeviceProblem
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_nearquad import near_surface_targets
    X, inside = near_surface_targets(seed=6)
    nts = np.array([12, 16, 20, 16] * 4, np.int32)
    pr = make_torus_problem(panels=16, extra_targets=X, nt_panels=nts)
    dp = DeviceProblem(pr, quad=dict(order=0))
    u = dp.matvec(cu(np.ones((pr.N, 1)))).cpu().numpy()[:, 0]
    dp.close()
    assert np.abs(u[:pr.n_on]).max() < 1e-9
    np.testing.assert_allclose(u[pr.n_on:], np.where(inside, -1.0, 0.0), atol=1e-9)


def test_ragged_ring_sedimentation(S):
    """the paper's sedimenting ring (Table t:conv-sbt, rho = 1e-2) on a mesh with alternating N_th"""
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_sedimentation import golden, completion_density
    from harness import DeviceProblem
    rho, P = 1e-2, 24
    nts = np.array([8, 12] * (P // 2), np.int32)
    quad = dict(order=0)
    pr = make_torus_problem(rho=rho, panels=P, kernel=2, nt_panels=nts)
    nu = completion_density(pr.y_c, pr.w_c, np.zeros(3), np.array([0.0, 0.0, -1.0]), np.zeros(3))
    Knu = []
    for e in (1.0, 0.0):
        p = make_torus_problem(rho=rho, panels=P, kernel=2, eta=e, nt_panels=nts)
        dp = DeviceProblem(p, quad=quad)
        Knu.append(dp.matvec(cu(nu)).clone())
        dp.close()
    pr.projector = True
    dp = DeviceProblem(pr, quad=quad)
    x, it, rr = dp.op.gmres((Knu[1] - Knu[0]).contiguous(), restart=100, max_iters=500, tol=1e-14)
    dp.close()
    V = -O.projector(pr.y_c, pr.w_c, np.zeros(pr.N, np.int32), 1, x.cpu().numpy())
    U = -float(np.average(V[:, 2], weights=pr.w_c))
    ex = golden()[rho]
    assert abs(U - ex) / ex < 5e-12, (U, ex, it, rr)
