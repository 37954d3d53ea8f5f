"""Pins of the N1 oracle (oracle/slb_quad_oracle.c: special-quadrature blocks by nested adaptive
Gauss-Kronrod + Duffy), CPU only.  None of these compares the oracle with itself: each checks a
value the paper or the mathematics fixes.

  * Gauss's law for the Laplace DL with unit density over a closed surface (jump relations,
    PAPER.md P:L1455-1460): D[1] = -1 inside, 0 outside, -1/2 on the surface (principal value at
    a node, the singular Duffy path), including targets 1e-3 rho from the surface;
  * Prop. 1 (proof P:L3038-3047): the Stokes DL of a rigid motion v is -v inside, 0
    outside, -v/2 on the surface;
  * S[n] = 0 for the Stokes single layer (divergence theorem), on and off the surface;
  * Green's representation (Eq. e:greens-rep): S_L[du/dn] - D[u] = u inside, u/2 on the
    surface, for u = G(x - x0), x0 outside;
  * the identity term of the full operator with sigma' = 1 != 0: c_I sigma + far + (B - smooth) =
    0 at the nodes (exterior limit) -- a wrong c_I fails;
  * the paper's convergence table t:conv-biest as an upper bound, through the full
    operator with the oracle's blocks.

The torus is R = 1 with 16 panels x 10 GL nodes: the panels' Lagrange interpolants then meet to
~1e-14, so the interpolated surface is closed to the tolerance the identities are checked at."""
import os

import numpy as np
import pytest

import oracle as O
from synth import make_torus_problem

FOUR_PI = 4 * np.pi
HERE = os.path.dirname(os.path.abspath(__file__))


def _all_panel_blocks(pr, kernel, X, node_of=None, eta=None):
    """blocks of every panel for targets X (rows), CSR = all panels per row"""
    T = len(X)
    rp = np.arange(T + 1, dtype=np.int64) * pr.P
    pidx = np.tile(np.arange(pr.P, dtype=np.int32), T)
    tn = None if node_of is None else np.asarray(node_of, np.int64)
    ep = None if eta is None else np.full(pr.P, eta)
    B = O.nearquad(kernel, np.asarray(X), rp, pidx, pr.Ns, pr.Nt, pr.y_c, trg_node=tn, eta_panel=ep)
    return B.reshape(T, pr.P, B.shape[1], B.shape[2])


def _apply_all(B, sig, pr):
    """sum_k B_{t,k} sigma_k  for each target row"""
    d = B.shape[2]
    s = sig.reshape(pr.P, pr.Nn * d)
    return np.einsum("tkrc,kc->tr", B, s)


def _torus():
    return make_torus_problem(R=1.0, rho=0.25, panels=16, Ns=10, Nt=12, kernel=1)


def _targets(pr, rho=0.25):
    """interior / exterior points near the surface (0.5 rho, 1 - 1e-3 rho / 1 + 1e-3 rho, 1.5 rho from the
    centerline), and three node targets"""
    ph = np.array([0.3, 2.0, 4.1])
    th = np.array([0.7, 2.9, 5.0])
    pts, inside = [], []
    for f in (0.5, 1 - 1e-3, 1 + 1e-3, 1.5):
        for a, b in zip(ph, th):
            er = np.array([np.cos(a), np.sin(a), 0.0])
            pts.append(np.array([np.cos(a), np.sin(a), 0.0]) + f * rho * (np.cos(b) * er + np.sin(b) * np.array([0, 0, 1.0])))
            inside.append(f < 1)
    nodes = [5 * pr.Nn + 3 * pr.Nt + 4, 11 * pr.Nn + 9 * pr.Nt + 0, 0 * pr.Nn + 0 * pr.Nt + 7]
    return np.array(pts), np.array(inside), nodes


def test_n1_gauss_law_on_and_off_surface():
    pr = _torus()
    X, inside, nodes = _targets(pr)
    Xall = np.concatenate([X, pr.y_c[nodes]])
    node_of = [-1] * len(X) + nodes
    B = _all_panel_blocks(pr, 1, Xall, node_of)
    u = _apply_all(B, np.ones(pr.N), pr)[:, 0]
    np.testing.assert_allclose(u[:len(X)], np.where(inside, -1.0, 0.0), rtol=0, atol=1e-12)
    np.testing.assert_allclose(u[len(X):], -0.5, rtol=0, atol=1e-12)       # principal value on the surface


def test_n1_stokes_rigid_motion_prop1():
    pr = make_torus_problem(R=1.0, rho=0.25, panels=16, Ns=10, Nt=12, kernel=2, eta=0.0)
    X, inside, nodes = _targets(pr)
    a = np.array([0.3, -0.7, 0.5])
    w = np.array([0.2, 0.4, -0.9])
    c = np.array([0.05, -0.1, 0.2])
    v = a + np.cross(w, pr.y_c - c)
    Xall = np.concatenate([X, pr.y_c[nodes]])
    B = _all_panel_blocks(pr, 2, Xall, [-1] * len(X) + nodes, eta=0.0)
    u = _apply_all(B, v, pr)
    vx = a + np.cross(w, Xall - c)
    exp = np.concatenate([np.where(inside[:, None], -vx[:len(X)], 0.0), -0.5 * vx[len(X):]])
    np.testing.assert_allclose(u, exp, rtol=0, atol=1e-12 * np.abs(vx).max())


def test_n1_stokes_single_layer_of_normal_vanishes():
    pr = make_torus_problem(R=1.0, rho=0.25, panels=16, Ns=10, Nt=12, kernel=2, eta=1.0)
    X, _, nodes = _targets(pr)
    Xall = np.concatenate([X, pr.y_c[nodes]])
    B = _all_panel_blocks(pr, 3, Xall, [-1] * len(X) + nodes, eta=1.0)
    u = _apply_all(B, pr.n_c, pr)
    # scale: the single layer of |sigma| = 1 is O(rho log) ~ 0.1; S[n] must vanish to rounding
    assert np.abs(u).max() <= 1e-12, np.abs(u).max()


def test_n1_greens_representation_on_and_off_surface():
    # N_th = 24, N_s = 12: the densities u, du/dn are interpolated to ~1e-13 (at N_th = 12 their trig
    # interpolation error alone is ~1e-8)
    pr = make_torus_problem(R=1.0, rho=0.25, panels=16, Ns=12, Nt=24, kernel=1)
    X, inside, nodes = _targets(pr)
    Xin = X[inside]
    Xall = np.concatenate([Xin, pr.y_c[nodes]])
    node_of = [-1] * len(Xin) + nodes
    x0 = np.array([1.0, 2.0, 3.0])
    d = pr.y_c - x0
    rr = np.sqrt((d * d).sum(1))
    u = 1.0 / (FOUR_PI * rr)
    dudn = -(d * pr.n_c).sum(1) / (FOUR_PI * rr ** 3)
    BD = _all_panel_blocks(pr, 1, Xall, node_of)
    BS = _all_panel_blocks(pr, 4, Xall, node_of, eta=1.0)
    rep = _apply_all(BS, dudn, pr)[:, 0] - _apply_all(BD, u, pr)[:, 0]
    ux = 1.0 / (FOUR_PI * np.linalg.norm(Xall - x0, axis=1))
    exp = np.concatenate([ux[:len(Xin)], 0.5 * ux[len(Xin):]])
    np.testing.assert_allclose(rep, exp, rtol=1e-11, atol=0)


def _quad_blocks_for_rows(pr, kernel, rows, eta_panel=None):
    """full-CSR block array with the oracle's special-quadrature blocks on the given rows (zero elsewhere)"""
    blen = pr.block_len
    blocks = np.zeros(pr.nnz * blen)
    sub_rp = np.concatenate([[0], np.cumsum(pr.row_ptr[rows + 1] - pr.row_ptr[rows])]).astype(np.int64)
    sub_pi = np.concatenate([pr.panel_idx[pr.row_ptr[t]:pr.row_ptr[t + 1]] for t in rows]).astype(np.int32)
    tn = np.where(rows < pr.n_on, rows, -1)
    B = O.nearquad(kernel, pr.x_trg[rows], sub_rp, sub_pi, pr.Ns, pr.Nt, pr.y_c, trg_node=tn, eta_panel=eta_panel)
    for q, t in enumerate(rows):
        a, b = pr.row_ptr[t], pr.row_ptr[t + 1]
        blocks[a * blen:b * blen] = B[sub_rp[q]:sub_rp[q + 1]].reshape(-1)
    return blocks


def test_n1_identity_term_of_full_operator():
    """(1/2 + D)[1] = 0 at every node through the FULL oracle operator: c_I sigma' (sigma' = 1) + smooth far
    sum over all panels + (B - smooth) over the near panels; B from the N1 oracle.  c_I = 1/2 is the only
    value that gives 0 (c_I = 0 or 1 leave -1/2 / +1/2)."""
    pr = make_torus_problem(R=1.0, rho=0.1, panels=16, Ns=10, Nt=12, kernel=1)
    rows = np.array([3, pr.Nn * 7 + 45, pr.Nn * 15 + pr.Nn - 1])
    blocks = _quad_blocks_for_rows(pr, 1, rows)
    u = O.Oracle(pr, blocks=blocks).apply_rows(np.ones(pr.N), rows)[:, 0]
    assert pr.c_identity == 0.5
    np.testing.assert_allclose(u, 0.0, atol=1e-11)


def _golden():
    out = []
    for line in open(os.path.join(HERE, "golden", "greens_rep_conv_biest.txt")):
        if line.strip() and not line.startswith("#"):
            f = line.split()
            out.append((int(f[0]), int(f[1]), int(f[2]), float(f[3])))
    return out


@pytest.mark.parametrize("row", [0, 1])
def test_n1_greens_rep_convergence_table_bound(row):
    """Table t:conv-biest: on the surface S_L[du/dn] - (1/2 + D)[u] = 0 through the full
    oracle operator (smooth far rule + N1 blocks on the near panels), e_inf over sampled nodes at most
    the paper's printed error at the same (N_elem, N_s = 10, N_theta)."""
    n_unk, P, nt, e_paper = _golden()[row]
    pr = make_torus_problem(R=1.0, rho=0.25, panels=P, Ns=10, Nt=nt, kernel=1)
    assert pr.N == n_unk
    rng = np.random.default_rng(row)
    rows = np.sort(rng.choice(pr.N, 10, replace=False))
    x0 = np.array([1.0, 2.0, 3.0])
    d = pr.y_c - x0
    rr = np.sqrt((d * d).sum(1))
    u = 1.0 / (FOUR_PI * rr)
    dudn = -(d * pr.n_c).sum(1) / (FOUR_PI * rr ** 3)
    A = O.Oracle(pr, blocks=_quad_blocks_for_rows(pr, 1, rows)).apply_rows(u, rows)[:, 0]      # (1/2 + D)[u]
    import copy
    ps = copy.copy(pr)                       # pure S_L: zero normals, eta = 1, no identity term
    ps.n_f = np.zeros_like(pr.n_f)
    ps.eta_f = np.ones_like(pr.eta_f)
    ps.c_identity = 0.0
    S = O.Oracle(ps, blocks=_quad_blocks_for_rows(pr, 4, rows, eta_panel=np.ones(pr.P))).apply_rows(dudn, rows)[:, 0]
    e = np.abs(S - A).max()
    print(f"N={pr.N}: e_inf(sampled) = {e:.2e} (paper {e_paper:.1e})")
    assert e <= e_paper, (e, e_paper)
