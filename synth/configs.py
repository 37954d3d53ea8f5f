"""The five BASELINE.json workloads as seeded synthetic problems.

Seed = 2310_00889 + config index (PCG64 via numpy.random.default_rng).  Every array
is what the operator takes as input; nothing here evaluates the operator.

  c1  Laplace DL, torus R=1 rho=0.1, 8 x 10 x 12 -> 2x upsampled, T = 960 nodes + 200 points
  c2  Stokes eta S + D, trefoil (R17) rho(s)=0.05(1+0.3cos 6 pi s), 32 x 10 x 16
  c3  Stokes, two tori R=1 rho=0.05 at gap 0.0025 (R19), 64 x 12 x 20 each
  c3v c3's geometry with per-panel N_th in {12, 24, 40, 64} by distance to the gap (NEXT N4)
  c4  Stokes mobility (K(I-L)+L), 64 random loops in [0,8]^3, 32 x 10 x 12 each
  c5  Stokes, 512 loops R=1 rho=0.05 in [0,16]^3, 9 x 10 x 12 each (R16); c5alt: 36 panels
"""
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .geometry import (Body, torus_body, trefoil_body, discretize, discretize_ragged, random_rotation,
                       panel_arclength, centerline_min_distance)
from .nearlist import build_near_csr

BASE_SEED = 2310_00889
LAPLACE_DL = 1
STOKES_SLDL = 2


def eta_cfie_input(rho: float) -> float:
    """CFIE single-layer scaling 1/(2 rho ln(1/rho)) (Eqs. e:laplace-bie-new P:L1750,
    e:stokes-bie-new P:L1868).  Supplied to BOTH sides as part of the operator's
    definition (the C library exports its own slb_eta_cfie, tested against this)."""
    return 1.0 / (2.0 * rho * np.log(1.0 / rho))


@dataclass
class Problem:
    name: str
    kernel: int                 # LAPLACE_DL or STOKES_SLDL
    seed: int
    Ns: int
    Nt: int
    Ms: int
    Mt: int
    n_bodies: int
    panels_per_body: List[int]
    body_of_panel: np.ndarray   # [P] int32
    # coarse (Nystrom) grid, layout [panel][i][j]
    y_c: np.ndarray
    n_c: np.ndarray
    w_c: np.ndarray
    # fine (smooth-quadrature) grid, same panels, layout [panel][m_s][m_t]
    y_f: np.ndarray
    n_f: np.ndarray
    w_f: np.ndarray
    eta_f: np.ndarray           # [M] CFIE eta of the source's body (0 for Laplace DL)
    eta_body: np.ndarray        # [n_bodies]
    x_trg: np.ndarray           # [T,3]; first n_on are the coarse nodes in node order
    n_on: int
    c_identity: float
    sigma: np.ndarray           # [N, sdim] coarse density
    row_ptr: np.ndarray         # [T+1] int64
    panel_idx: np.ndarray       # [nnz] int32, ascending per row
    blk_seed: int
    s_blk: float
    projector: bool = False
    panel_len: Optional[np.ndarray] = None
    body_center: Optional[np.ndarray] = None
    extra: dict = field(default_factory=dict)
    # ragged orders (NEXT N4): N_th^(k) and/or N_s^(k) per panel; fine orders
    # M_th^(k) = q_th N_th^(k), M_s^(k) = q_s N_s^(k) with q_th = Mt // Nt, q_s = Ms // Ns (Ns, Nt, Ms, Mt
    # then hold the base orders).  None: every panel has the base order.
    panel_nt: Optional[np.ndarray] = None
    panel_ns: Optional[np.ndarray] = None

    @property
    def ragged(self):
        return self.panel_nt is not None or self.panel_ns is not None

    def nt_of_panel(self):
        return self.panel_nt.astype(np.int64) if self.panel_nt is not None else np.full(self.P, self.Nt, np.int64)

    def mt_of_panel(self):
        return self.nt_of_panel() * (self.Mt // self.Nt) if self.ragged else np.full(self.P, self.Mt, np.int64)

    def ns_of_panel(self):
        return self.panel_ns.astype(np.int64) if self.panel_ns is not None else np.full(self.P, self.Ns, np.int64)

    def ms_of_panel(self):
        return self.ns_of_panel() * (self.Ms // self.Ns) if self.ragged else np.full(self.P, self.Ms, np.int64)

    def node_off(self):
        """[P+1] first coarse node of each panel"""
        return np.concatenate([[0], np.cumsum(self.ns_of_panel() * self.nt_of_panel())]).astype(np.int64)

    def fine_off(self):
        """[P+1] first fine node of each panel"""
        return np.concatenate([[0], np.cumsum(self.ms_of_panel() * self.mt_of_panel())]).astype(np.int64)

    def blk_off(self):
        """[nnz+1] first entry of each near block [t_dim][N_n^(k) s_dim] in the flat block array"""
        nn = self.ns_of_panel() * self.nt_of_panel()
        bl = self.tdim * self.sdim * nn[self.panel_idx]
        return np.concatenate([[0], np.cumsum(bl)]).astype(np.int64)

    def n_blocks_entries(self):
        return int(self.blk_off()[-1]) if self.ragged else self.nnz * self.block_len

    @property
    def P(self):
        return int(self.body_of_panel.shape[0])

    @property
    def sdim(self):
        return 1 if self.kernel == LAPLACE_DL else 3

    @property
    def tdim(self):
        return self.sdim

    @property
    def Nn(self):
        assert not self.ragged, "ragged problem: use node_off()"
        return self.Ns * self.Nt

    @property
    def Mn(self):
        assert not self.ragged, "ragged problem: use fine_off()"
        return self.Ms * self.Mt

    @property
    def N(self):
        return int(self.node_off()[-1]) if self.ragged else self.P * self.Nn

    @property
    def M(self):
        return int(self.fine_off()[-1]) if self.ragged else self.P * self.Mn

    @property
    def T(self):
        return int(self.x_trg.shape[0])

    @property
    def nnz(self):
        return int(self.panel_idx.shape[0])

    @property
    def block_len(self):
        assert not self.ragged, "ragged problem: use blk_off()"
        return self.tdim * self.Nn * self.sdim

    def pairs(self):
        return self.T * self.M


def _assemble(name, kernel, seed, bodies: List[Body], P_per_body, Ns, Nt, q=(2, 2),
              extra_targets=None, c1_rule=False, projector=False, rng=None, nt_panels=None, ns_panels=None,
              breaks=None):
    """nt_panels / ns_panels: optional lists (per body) of per-panel angular / GL orders (ragged,
    NEXT N4); Nt, Ns are then the base orders and q the fine factors of every panel.  breaks: optional
    list (per body) of panel breakpoints in s (adaptive panels); default uniform."""
    Ms, Mt = q[0] * Ns, q[1] * Nt
    breaks = breaks if breaks is not None else [None] * len(bodies)
    ragged = nt_panels is not None or ns_panels is not None
    if ragged:
        nt_panels = nt_panels if nt_panels is not None else [np.full(P, Nt) for P in P_per_body]
        ns_panels = ns_panels if ns_panels is not None else [np.full(P, Ns) for P in P_per_body]
        coarse = [discretize_ragged(b, P, np.asarray(ns), nt, br)
                  for b, P, ns, nt, br in zip(bodies, P_per_body, ns_panels, nt_panels, breaks)]
        fine = [discretize_ragged(b, P, q[0] * np.asarray(ns), q[1] * np.asarray(nt), br)
                for b, P, ns, nt, br in zip(bodies, P_per_body, ns_panels, nt_panels, breaks)]
    else:
        coarse = [discretize(b, P, Ns, Nt, br) for b, P, br in zip(bodies, P_per_body, breaks)]
        fine = [discretize(b, P, Ms, Mt, br) for b, P, br in zip(bodies, P_per_body, breaks)]
    cat = lambda L, a: np.ascontiguousarray(np.concatenate([getattr(g, a) for g in L], axis=0))
    y_c, n_c, w_c = cat(coarse, "y"), cat(coarse, "n"), cat(coarse, "w")
    y_f, n_f, w_f = cat(fine, "y"), cat(fine, "n"), cat(fine, "w")
    body_of_panel = np.concatenate([np.full(P, b, np.int32) for b, P in enumerate(P_per_body)])
    Ptot = int(body_of_panel.shape[0])
    panel_nt = None if not ragged else np.concatenate([np.asarray(v, np.int32) for v in nt_panels])
    panel_ns = None if not ragged else np.concatenate([np.asarray(v, np.int32) for v in ns_panels])
    nt_k = np.full(Ptot, Nt, np.int64) if panel_nt is None else panel_nt.astype(np.int64)
    ns_k = np.full(Ptot, Ns, np.int64) if panel_ns is None else panel_ns.astype(np.int64)
    node_off = np.concatenate([[0], np.cumsum(ns_k * nt_k)])
    fine_per_panel = q[0] * ns_k * q[1] * nt_k
    if kernel == STOKES_SLDL:
        eta_body = np.array([eta_cfie_input(b.rho_min) for b in bodies])
    else:
        eta_body = np.zeros(len(bodies))
    eta_f = np.repeat(eta_body[body_of_panel], fine_per_panel).astype(np.float64)
    n_on = y_c.shape[0]
    x_trg = y_c.copy()
    if extra_targets is not None:
        x_trg = np.ascontiguousarray(np.concatenate([x_trg, extra_targets], axis=0))
    sdim = 1 if kernel == LAPLACE_DL else 3
    sigma = rng.standard_normal((y_c.shape[0], sdim))
    L = np.concatenate([panel_arclength(b, P, br) for b, P, br in zip(bodies, P_per_body, breaks)])
    # first node of every GL ring: its centerline point and radius (ragged-safe: panels with fewer
    # rings repeat their first ring, which leaves the min over rings unchanged)
    nsmax = int(ns_k.max())
    ii = np.arange(nsmax)[None, :]
    ring_first = (node_off[:-1, None] + np.where(ii < ns_k[:, None], ii, 0) * nt_k[:, None]).reshape(-1)
    ring_xc = cat(coarse, "xc")[ring_first].reshape(Ptot, nsmax, 3)
    s_all = np.concatenate([g.s for g in coarse])
    S_ring = s_all[ring_first].reshape(Ptot, nsmax)
    rho_ring = np.empty((Ptot, nsmax))
    for bi, b in enumerate(bodies):
        m = body_of_panel == bi
        rho_ring[m] = np.broadcast_to(b.rho(S_ring[m]), (int(m.sum()), nsmax))
    own = np.full(x_trg.shape[0], -1, np.int64)
    own[:n_on] = np.repeat(np.arange(Ptot), ns_k * nt_k)
    forced = None
    if c1_rule:
        # config 1 node targets: panels {k-1, k, k+1} mod P of their own body (R15)
        P0 = P_per_body[0]
        k = np.repeat(np.arange(P0), Ns * Nt)
        forced = np.stack([(k - 1) % P0, k, (k + 1) % P0], axis=1)
    if not ragged:
        y_panels = y_c.reshape(Ptot, Ns * Nt, 3)
    else:   # pad every panel to the largest node count with copies of its first node (min unchanged)
        nmax = int((ns_k * nt_k).max())
        j = np.arange(nmax)[None, :]
        idx = node_off[:-1, None] + np.where(j < (ns_k * nt_k)[:, None], j, 0)
        y_panels = y_c[idx]
    row_ptr, panel_idx = build_near_csr(x_trg, y_panels, ring_xc, rho_ring, L, own, forced_rows=forced)
    # coincident-pair guard (R14): no target may sit on a fine source
    _assert_separated(x_trg, y_f)
    blk_seed = (seed * 0x9E3779B1 + 0xB10C) & ((1 << 64) - 1)
    s_blk = 1.0 / (Ns * Nt)
    centers = np.array([b.center for b in bodies])
    return Problem(name=name, kernel=kernel, seed=seed, Ns=Ns, Nt=Nt, Ms=Ms, Mt=Mt,
                   n_bodies=len(bodies), panels_per_body=list(P_per_body),
                   body_of_panel=body_of_panel, y_c=y_c, n_c=n_c, w_c=w_c, y_f=y_f, n_f=n_f,
                   w_f=w_f, eta_f=eta_f, eta_body=eta_body, x_trg=x_trg, n_on=n_on,
                   c_identity=0.5, sigma=sigma, row_ptr=row_ptr, panel_idx=panel_idx,
                   blk_seed=blk_seed, s_blk=s_blk, projector=projector, panel_len=L,
                   body_center=centers, panel_nt=panel_nt,
                   panel_ns=panel_ns if (panel_ns is not None and np.any(panel_ns != Ns)) else None)


def _assert_separated(x, y, tol=1e-9):
    from scipy.spatial import cKDTree
    d, _ = cKDTree(y).query(x, k=1)
    assert d.min() > tol, f"target coincides with a fine source (min dist {d.min():.3e})"


def _place_loops(rng, n, R_of, rho_of, lo_hi_of, gap_of, max_tries=200000):
    bodies = []
    tries = 0
    while len(bodies) < n:
        tries += 1
        if tries > max_tries:
            raise RuntimeError("loop placement failed")
        R, rho = R_of(), rho_of()
        Q = random_rotation(rng)
        ax = Q[:, 2]
        half = R * np.sqrt(np.clip(1 - ax ** 2, 0, 1)) + rho
        lo, hi = lo_hi_of(half)
        if np.any(hi <= lo):
            continue
        c = lo + (hi - lo) * rng.random(3)
        cand = torus_body(R, rho, c, Q)
        cand.extra_R = R
        ok = True
        for b in bodies:
            if np.linalg.norm(b.center - c) > R + b.extra_R + rho + b.rho_min + gap_of(rho, b.rho_min):
                continue
            d = centerline_min_distance(cand, b)
            if d - rho - b.rho_min < gap_of(rho, b.rho_min) + 1e-3:
                ok = False
                break
        if ok:
            bodies.append(cand)
    return bodies, tries


CONFIGS = ("c1", "c2", "c3", "c3v", "c4", "c5", "c5alt")


def make_torus_problem(R=1.0, rho=0.1, panels=12, Ns=10, Nt=12, kernel=LAPLACE_DL, eta=None, extra_targets=None,
                       seed_offset=0, nt_panels=None, ns_panels=None, breaks=None):
    """Single torus (axis z, centre 0) with the 2 L_k near rule -- pin problems for the special
    quadrature (N1).  eta=None -> the CFIE value 1/(2 rho ln(1/rho)) for Stokes, the pure DL for
    Laplace; an explicit eta sets the single-layer weight of either kernel (0 -> pure DL)."""
    seed = BASE_SEED + 100 + seed_offset
    rng = np.random.default_rng(seed)
    b = torus_body(R, rho)
    pr = _assemble("torus", kernel, seed, [b], [panels], Ns, Nt, extra_targets=extra_targets, rng=rng,
                   nt_panels=None if nt_panels is None else [np.asarray(nt_panels)],
                   ns_panels=None if ns_panels is None else [np.asarray(ns_panels)],
                   breaks=None if breaks is None else [np.asarray(breaks)])
    if eta is not None:       # Stokes eta S + D, or the Laplace combined field D + eta S_L
        pr.eta_body[:] = eta
        pr.eta_f[:] = eta
    return pr


def make_config(name: str, **kw) -> Problem:
    """Build one of the BASELINE configs.  Keyword overrides shrink a config for tests
    (n_loops, panels) while keeping its shape and recipe."""
    idx = {"c1": 0, "c2": 1, "c3": 2, "c3v": 2, "c4": 3, "c5": 4, "c5alt": 4}[name]
    seed = BASE_SEED + idx + kw.pop("seed_offset", 0)
    rng = np.random.default_rng(seed)
    if name == "c1":
        P = kw.get("panels", 8)
        b = torus_body(1.0, 0.1)
        nextra = kw.get("n_extra", 200)
        extra = rng.uniform(-1.5, 1.5, size=(nextra, 3))
        return _assemble(name, LAPLACE_DL, seed, [b], [P], 10, 12, extra_targets=extra,
                         c1_rule=True, rng=rng)
    if name == "c2":
        P = kw.get("panels", 32)
        return _assemble(name, STOKES_SLDL, seed, [trefoil_body()], [P], 10, 16, rng=rng)
    if name == "c3":
        P = kw.get("panels", 64)
        rho, gap = 0.05, 0.0025
        b0 = torus_body(1.0, rho, (0.0, 0.0, 0.0))
        b1 = torus_body(1.0, rho, (2.0 + 2 * rho + gap, 0.0, 0.0))
        return _assemble(name, STOKES_SLDL, seed, [b0, b1], [P, P], 12, 20, rng=rng)
    if name == "c3v":
        # c3 with per-panel orders (NEXT N4; the paper's close-touching mesh is adaptive in N_th up
        # to 88): N_th by the distance from the panel's centerline midpoint to the other
        # ring's centerline -- 64 within 0.15, 40 within 0.4, 24 within 0.8, else 12; N_s = 16 within
        # 0.4, else 12 (base 12 x 12, q = 2)
        P = kw.get("panels", 64)
        rho, gap = 0.05, 0.0025
        c1x = 2.0 + 2 * rho + gap
        b0 = torus_body(1.0, rho, (0.0, 0.0, 0.0))
        b1 = torus_body(1.0, rho, (c1x, 0.0, 0.0))
        mid = (np.arange(P) + 0.5) / P
        nts, nss = [], []
        for b, other in ((b0, b1), (b1, b0)):
            xm = b.xc(mid)
            so = np.arange(720) / 720
            d = np.min(np.linalg.norm(xm[:, None, :] - other.xc(so)[None, :, :], axis=-1), axis=1)
            nts.append(np.select([d < 0.15, d < 0.4, d < 0.8], [64, 40, 24], 12).astype(np.int32))
            nss.append(np.where(d < 0.4, 16, 12).astype(np.int32))      # N_s^(k): 16 at the gap
        return _assemble(name, STOKES_SLDL, seed, [b0, b1], [P, P], 12, 12, rng=rng, nt_panels=nts, ns_panels=nss)
    if name == "c4":
        n = kw.get("n_loops", 64)
        P = kw.get("panels", 32)
        box = kw.get("box", 8.0)
        bodies, tries = _place_loops(
            rng, n, lambda: rng.uniform(0.8, 1.2), lambda: rng.uniform(0.02, 0.05),
            lambda half: (half, box - half), lambda ra, rb: 0.5 * min(ra, rb))
        pr = _assemble(name, STOKES_SLDL, seed, bodies, [P] * n, 10, 12, projector=True, rng=rng)
        pr.extra["placement_tries"] = tries
        return pr
    if name in ("c5", "c5alt"):
        n = kw.get("n_loops", 512)
        P = kw.get("panels", 9 if name == "c5" else 36)
        box = kw.get("box", 16.0)
        bodies, tries = _place_loops(
            rng, n, lambda: 1.0, lambda: 0.05,
            lambda half: (np.full(3, 1.05), np.full(3, box - 1.05)), lambda ra, rb: 0.025)
        pr = _assemble(name, STOKES_SLDL, seed, bodies, [P] * n, 10, 12, rng=rng)
        pr.extra["placement_tries"] = tries
        return pr
    raise ValueError(name)


def pin_torus(R=1.0, rho=0.1, P=256, Ns=10, Nt=48, center=(0.0, 0.0, 0.0), Q=None):
    """Refined 'pin geometry' (SURVEY §0.6, §8c 'REF'): coarse = fine (q = 1)."""
    b = torus_body(R, rho, center, Q)
    return b, discretize(b, P, Ns, Nt)
