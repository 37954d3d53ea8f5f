"""(NEXT N1) GPU special-quadrature blocks (slb_nearcorr_quad) against the CPU oracle
(oracle/slb_quad_oracle.c, nested adaptive Gauss-Kronrod + Duffy; pinned in test_oracle_n1_pins.py),
element by element, on the same seeded geometry:

  * singular pairs (a node target on its own element),
  * near-singular on-surface pairs (a node of the neighbouring element; across the gap of the two close
    tori of c3, distance rho/20),
  * off-surface targets at 1e-3 rho, 0.1 rho and 0.5 rho from the surface, inside and outside,

on c2 (trefoil, varying radius, 10 x 16), c3 (12 x 20, two tori at gap rho/20), c3v's largest class
(16 x 64) and a Laplace torus.  Metric per block: max |B_gpu - B_oracle| / max |B_oracle|.
Tolerance: TOL = 1e-12 (the north_star's), the oracle being accurate to ~1e-14 (its pins)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_config, make_torus_problem  # noqa: E402

TOL = 1e-12


def cu(a, dt=None):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt or torch.float64)


def _skip():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _off_surface(pr, k, fracs, rho):
    """points off the surface near element k: along the outward normal of node (ns/2, j) at distance f rho"""
    Nn, nt = pr.Nn, pr.Nt
    out = []
    for q, f in enumerate(fracs):
        nd = k * Nn + (pr.Ns // 2) * nt + (3 * q) % nt
        out.append(pr.y_c[nd] + f * rho * pr.n_c[nd])
    return np.array(out)


def _pairs(pr, rho, extra_k=0):
    """(target x, target node id or -1, element) triples"""
    Nn, nt = pr.Nn, pr.Nt
    P = pr.P
    k = extra_k
    trip = []
    for (i, j) in [(0, 0), (pr.Ns // 2, nt // 3), (pr.Ns - 1, nt - 1)]:
        nd = k * Nn + i * nt + j
        trip.append((pr.y_c[nd], nd, k))                    # singular
    nd = ((k + 1) % P) * Nn + 0 * nt + 2                      # first ring of the next element, on element k
    trip.append((pr.y_c[nd], nd, k))
    nd = ((k - 1) % P) * Nn + (pr.Ns - 1) * nt + 5            # last ring of the previous element
    trip.append((pr.y_c[nd], nd, k))
    for x in _off_surface(pr, k, [1e-3, -1e-3, 0.1, -0.1, 0.5, -0.5], rho):
        trip.append((x, -1, k))
    return trip


def _run(kernel, pr, trip, eta_panel, method=None, **kw):
    import paper_2310_00889_b200 as S
    X = np.array([t[0] for t in trip])
    nodes = np.array([t[1] for t in trip], np.int64)
    pid = np.array([t[2] for t in trip], np.int32)
    rp = np.arange(len(trip) + 1, dtype=np.int64)
    d = 3 if kernel in (2, 3) else 1
    blen = d * d * pr.Nn
    blocks = torch.empty(len(trip) * blen, dtype=torch.float64, device="cuda")
    args = dict(trg_node=cu(nodes, torch.int64), eta_panel=None if eta_panel is None else cu(eta_panel))
    args.update(kw)
    S.slb_nearcorr_quad(kernel, cu(X), cu(rp, torch.int64), cu(pid, torch.int32), pr.Ns, pr.Nt,
                        cu(pr.y_c.reshape(pr.P, pr.Nn, 3)), blocks, **args)
    got = blocks.cpu().numpy().reshape(len(trip), d, pr.Nn * d)
    ref = O.nearquad(kernel, X, rp, pid, pr.Ns, pr.Nt, pr.y_c, trg_node=nodes, eta_panel=eta_panel)
    errs = [np.abs(got[q] - ref[q]).max() / np.abs(ref[q]).max() for q in range(len(trip))]
    return np.array(errs)


CASES = [
    ("torus_laplace", lambda: make_torus_problem(R=1.0, rho=0.1, panels=12, Ns=10, Nt=12, kernel=1), 1, 0.1),
    ("torus_laplace_sl", lambda: make_torus_problem(R=1.0, rho=0.1, panels=12, Ns=10, Nt=12, kernel=1), 4, 0.1),
    ("torus_stokes_dl", lambda: make_torus_problem(R=1.0, rho=0.1, panels=12, Ns=10, Nt=12, kernel=2, eta=0.0), 2, 0.1),
    ("torus_stokes_sl", lambda: make_torus_problem(R=1.0, rho=0.1, panels=12, Ns=10, Nt=12, kernel=2), 3, 0.1),
    ("c2_stokes", lambda: make_config("c2", panels=32), 2, None),
    ("c3_stokes", lambda: make_config("c3", panels=64), 2, 0.05),
]


@pytest.mark.parametrize("name,mk,kernel,rho", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("order", [0, 14], ids=["paper_modal", "adaptive2d_q14"])
def test_nearquad_blocks_vs_oracle(name, mk, kernel, rho, order):
    _skip()
    pr = mk()
    if rho is None:                                     # trefoil: radius at the element's midpoint
        rho = 0.05 * (1 + 0.3 * np.cos(6 * np.pi * (3.5 / pr.P)))
    k = 0 if name == "c3_stokes" else 3                 # c3: element 0 of torus 0 faces the gap
    trip = _pairs(pr, rho, extra_k=k)
    if name == "c3_stokes":                             # across the gap (rho/20): the other torus' closest node
        Nn = pr.Nn
        y1 = pr.y_c[pr.P // 2 * Nn:]
        d0 = np.linalg.norm(y1[:, None, :] - pr.y_c[None, 0:Nn, :], axis=-1).min(1)
        nd = int(np.argmin(d0)) + pr.P // 2 * Nn
        trip.append((pr.y_c[nd], nd, 0))
    eta = pr.eta_body[pr.body_of_panel] if kernel in (2, 3) else None
    errs = _run(kernel, pr, trip, eta, order=order, beta=0.6)
    print(name, order, " ".join(f"{e:.1e}" for e in errs))
    # the paper's rule (order 0) at the north_star tolerance; the generic 2-D rule of round 1 is held
    # to what its acceptance test supports (it is kept for comparison, N1)
    assert errs.max() <= (TOL if order == 0 else 1e-9), errs


def test_nearquad_blocks_vs_oracle_c3v_ragged():
    """c3v's ragged elements (N4): the 16 x 64 gap elements and a 12 x 12 outer element, through
    slb_nearcorr_quad_ragged -- singular, neighbour-node, across-the-gap and off-surface pairs."""
    _skip()
    import paper_2310_00889_b200 as S
    pr = make_config("c3v", panels=64)
    no = pr.node_off()
    pns, pnt = pr.ns_of_panel(), pr.nt_of_panel()
    big = int(np.argmax(pns * pnt))                     # a 16 x 64 element at the gap
    small = int(np.argmin(pns * pnt))                   # a 12 x 12 element away from it
    trip = []
    for k in (big, small):
        ns, nt = int(pns[k]), int(pnt[k])
        for (i, j) in [(0, 0), (ns // 2, nt // 3), (ns - 1, nt - 1)]:
            nd = no[k] + i * nt + j
            trip.append((pr.y_c[nd], nd, k))
        kn = (k + 1) % pr.P if (k + 1) % (pr.P // 2) else k - 1
        nd = no[kn] + 2
        trip.append((pr.y_c[nd], nd, k))
        for q, f in enumerate([1e-3, -1e-3, 0.1, -0.5]):
            nd = no[k] + (ns // 2) * nt + (5 * q) % nt
            trip.append((pr.y_c[nd] + f * 0.05 * pr.n_c[nd], -1, k))
    y1 = pr.y_c[no[pr.P // 2]:]                        # the other torus' node closest to the gap element
    d0 = np.linalg.norm(y1 - pr.y_c[no[big]:no[big + 1]].mean(0), axis=1)
    nd = int(np.argmin(d0)) + no[pr.P // 2]
    trip.append((pr.y_c[nd], nd, big))
    X = np.array([t[0] for t in trip])
    nodes = np.array([t[1] for t in trip], np.int64)
    pid = np.array([t[2] for t in trip], np.int32)
    rp = np.arange(len(trip) + 1, dtype=np.int64)
    sizes = [9 * int(pns[k] * pnt[k]) for k in pid]
    off = np.concatenate([[0], np.cumsum(sizes)])
    blocks = torch.empty(int(off[-1]), dtype=torch.float64, device="cuda")
    eta = pr.eta_body[pr.body_of_panel]
    S.slb_nearcorr_quad(2, cu(X), cu(rp, torch.int64), cu(pid, torch.int32), pr.Ns, pr.Nt, cu(pr.y_c), blocks,
                        trg_node=cu(nodes, torch.int64), eta_panel=cu(eta), order=0, panel_nt=pnt, panel_ns=pns)
    got = blocks.cpu().numpy()
    errs = []
    for q, (x, nd, k) in enumerate(trip):
        ns, nt = int(pns[k]), int(pnt[k])
        yk = pr.y_c[no[k]:no[k + 1]].reshape(ns, nt, 3)
        node = ((nd - no[k]) // nt, (nd - no[k]) % nt) if no[k] <= nd < no[k + 1] else None
        ref = O.nearquad_block(2, x, yk, eta=float(eta[k]), node=node)
        errs.append(np.abs(got[off[q]:off[q + 1]] - ref.reshape(-1)).max() / np.abs(ref).max())
    errs = np.array(errs)
    print("c3v", " ".join(f"{e:.1e}" for e in errs))
    assert errs.max() <= TOL, errs
