"""Slender-body geometry and its panel x Fourier discretisation (input generation).

Follows PAPER.md §3.1:
  * surface map  y(s,th) = x_c(s) + rho(s) [e1(s) cos th + e2(s) sin th],  e2 = t_hat x e1
    (Eq. e:surface-coord);
  * panels I_k = [k/P, (k+1)/P) (uniform), N_s Gauss-Legendre nodes in s
    (ascending) x N_th uniform nodes th_j = 2 pi j / N_th (R4);
  * far-field weights w_ij = J_ij * w^(GL,k)_i * 2 pi / N_th with J = |y_s x y_th|
    (P:L870-876), J taken w.r.t. s in [0,1) (R7);
  * outward normal n = (y_th x y_s)/|y_th x y_s| (R8; asserted n.(y - x_c) > 0).

Derivatives y_s, y_th are computed by complex-step differentiation of the analytic map,
exact to rounding, so coarse and fine grids are both sampled from the exact surface
(R7: fine geometry is not interpolated).  Frames: tori use the body axis as e1, the
trefoil uses e1 = normalize(z - (z.t)t) (R18); any smooth frame is admissible.
"""
from dataclasses import dataclass
from typing import Callable

import numpy as np

_H = 1e-30  # complex-step size


def gauss_legendre_np(n: int):
    """GL nodes (ascending) and weights on [-1,1] (numpy's library routine)."""
    x, w = np.polynomial.legendre.leggauss(n)
    return x, w


def _cross(a, b):
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)


def _normalize(v):
    # analytic (no conj): valid under complex-step perturbation
    return v / np.sqrt(np.sum(v * v, axis=-1, keepdims=True))


@dataclass
class Body:
    """A closed slender loop: centerline x_c(s), its derivative, radius rho(s), frame e1(s)."""
    xc: Callable
    dxc: Callable
    rho: Callable
    e1: Callable
    rho_min: float
    kind: str = "loop"
    center: np.ndarray = None
    axis: np.ndarray = None

    def surface(self, s, th):
        s = np.asarray(s)
        th = np.asarray(th)
        xc = self.xc(s)
        t = _normalize(self.dxc(s))
        e1 = self.e1(s, t)
        e2 = _cross(t, e1)
        r = self.rho(s)[..., None]
        return xc + r * (e1 * np.cos(th)[..., None] + e2 * np.sin(th)[..., None])


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniform random rotation from a normalised Gaussian quaternion."""
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    a, b, c, d = q
    return np.array([[a*a + b*b - c*c - d*d, 2*(b*c - a*d), 2*(b*d + a*c)],
                     [2*(b*c + a*d), a*a - b*b + c*c - d*d, 2*(c*d - a*b)],
                     [2*(b*d - a*c), 2*(c*d + a*b), a*a - b*b - c*c + d*d]])


def torus_body(R: float, rho: float, center=(0.0, 0.0, 0.0), Q=None) -> Body:
    """Circular loop of major radius R, constant tube radius rho, axis Q z, centred at center."""
    Q = np.eye(3) if Q is None else np.asarray(Q, dtype=np.float64)
    c = np.asarray(center, dtype=np.float64)
    ax = Q[:, 2].copy()

    def xc(s):
        ph = 2 * np.pi * s
        loc = np.stack([R * np.cos(ph), R * np.sin(ph), 0 * ph], axis=-1)
        return c + loc @ Q.T

    def dxc(s):
        ph = 2 * np.pi * s
        loc = np.stack([-R * np.sin(ph), R * np.cos(ph), 0 * ph], axis=-1) * (2 * np.pi)
        return loc @ Q.T

    def rhof(s):
        return rho + 0 * s

    def e1(s, t):
        return np.broadcast_to(ax, t.shape) + 0 * t

    return Body(xc, dxc, rhof, e1, rho_min=rho, kind="torus", center=c, axis=ax)


def trefoil_body() -> Body:
    """Config-2 fiber: trefoil centerline, rho(s) = 0.05 (1 + 0.3 cos 6 pi s)."""
    def xc(s):
        ph = 2 * np.pi * s
        a = 1 + 0.4 * np.cos(3 * ph)
        return np.stack([a * np.cos(2 * ph), a * np.sin(2 * ph), 0.4 * np.sin(3 * ph)], axis=-1)

    def dxc(s):
        ph = 2 * np.pi * s
        a = 1 + 0.4 * np.cos(3 * ph)
        da = -1.2 * np.sin(3 * ph)
        d = np.stack([da * np.cos(2 * ph) - 2 * a * np.sin(2 * ph),
                      da * np.sin(2 * ph) + 2 * a * np.cos(2 * ph),
                      1.2 * np.cos(3 * ph)], axis=-1)
        return d * (2 * np.pi)

    def rhof(s):
        return 0.05 * (1 + 0.3 * np.cos(6 * np.pi * s))

    def e1(s, t):
        z = np.zeros(t.shape, dtype=t.dtype)
        z[..., 2] = 1.0
        return _normalize(z - np.sum(z * t, axis=-1, keepdims=True) * t)

    return Body(xc, dxc, rhof, e1, rho_min=0.035, kind="trefoil",
                center=np.zeros(3), axis=np.array([0.0, 0.0, 1.0]))


@dataclass
class Grid:
    """Nodes of one body on one (N_s, N_th) grid, layout [panel][i (s)][j (th)]."""
    y: np.ndarray      # [P*Ns*Nt, 3]
    n: np.ndarray      # [P*Ns*Nt, 3] outward unit normal
    w: np.ndarray      # [P*Ns*Nt]    far-field quadrature weight
    J: np.ndarray      # [P*Ns*Nt]    surface Jacobian wrt (s, th)
    s: np.ndarray      # [P*Ns*Nt]    parameter s of the node
    th: np.ndarray     # [P*Ns*Nt]    parameter th of the node
    xc: np.ndarray     # [P*Ns*Nt, 3] centerline point of the node's ring
    P: int
    Ns: int
    Nt: int


def _breaks(P, breaks):
    """panel breakpoints in s: uniform [k/P, (k+1)/P) unless given (P+1 increasing values 0 .. 1)"""
    if breaks is None:
        return np.arange(P + 1) / P
    b = np.asarray(breaks, dtype=np.float64)
    assert b.shape == (P + 1,) and b[0] == 0.0 and b[-1] == 1.0 and np.all(np.diff(b) > 0)
    return b


def discretize(body: Body, P: int, Ns: int, Nt: int, breaks=None) -> Grid:
    """breaks: optional panel breakpoints in s (adaptive panels); default uniform"""
    t, wgl = gauss_legendre_np(Ns)
    b = _breaks(P, breaks)
    a, h = b[:-1, None], (b[1:] - b[:-1])[:, None]
    s = a + h * (t[None, :] + 1) / 2                           # [P, Ns]
    th = 2 * np.pi * np.arange(Nt) / Nt                        # [Nt]
    S = np.broadcast_to(s[:, :, None], (P, Ns, Nt)).reshape(-1)
    TH = np.broadcast_to(th[None, None, :], (P, Ns, Nt)).reshape(-1)
    y = body.surface(S, TH)
    ys = body.surface(S + 1j * _H, TH.astype(np.complex128)).imag / _H
    yt = body.surface(S.astype(np.complex128), TH + 1j * _H).imag / _H
    cr = _cross(yt, ys)
    J = np.sqrt(np.sum(cr * cr, axis=-1))
    n = cr / J[:, None]
    wpan = np.broadcast_to((wgl[None, :] * h / 2)[:, :, None], (P, Ns, Nt)).reshape(-1)
    w = J * wpan * (2 * np.pi / Nt)
    xc = body.xc(S)
    assert np.all(np.sum(n * (y - xc), axis=-1) > 0), "normals must point outward (S:L34)"
    return Grid(y=np.ascontiguousarray(y), n=np.ascontiguousarray(n), w=np.ascontiguousarray(w),
                J=J, s=S.copy(), th=TH.copy(), xc=xc, P=P, Ns=Ns, Nt=Nt)


def discretize_ragged(body: Body, P: int, Ns, nt_panels, breaks=None) -> Grid:
    """Per-panel orders (§3.1: element k has N_s^(k) x N_th^(k) nodes).
    Ns: int or [P] array; nt_panels: [P].  Layout [panel][i][j], panel k contributing
    N_s^(k) N_th^(k) nodes; the node recipe per panel is discretize()'s.  Grid.Ns/Nt are 0 (ragged)."""
    nt_panels = np.asarray(nt_panels, dtype=np.int64)
    ns_panels = np.broadcast_to(np.asarray(Ns, dtype=np.int64), (P,))
    assert nt_panels.shape == (P,) and np.all(nt_panels % 2 == 0) and np.all(nt_panels >= 2)
    assert np.all(ns_panels >= 1)
    cache = {}
    fields = ("y", "n", "w", "J", "s", "th", "xc")
    out = {f: [] for f in fields}
    for k in range(P):
        ns, nt = int(ns_panels[k]), int(nt_panels[k])
        if (ns, nt) not in cache:
            cache[(ns, nt)] = discretize(body, P, ns, nt, breaks)
        g = cache[(ns, nt)]
        a, b = k * ns * nt, (k + 1) * ns * nt
        for f in fields:
            out[f].append(getattr(g, f)[a:b])
    cat = {f: np.ascontiguousarray(np.concatenate(out[f], axis=0)) for f in fields}
    return Grid(P=P, Ns=0, Nt=0, **cat)


def panel_arclength(body: Body, P: int, breaks=None) -> np.ndarray:
    """Centerline arc length of each panel by 16-point GL."""
    t, wgl = gauss_legendre_np(16)
    b = _breaks(P, breaks)
    a, h = b[:-1, None], (b[1:] - b[:-1])[:, None]
    s = a + h * (t[None, :] + 1) / 2
    sp = np.sqrt(np.sum(body.dxc(s) ** 2, axis=-1))
    return np.sum(sp * wgl[None, :] * h / 2, axis=1)


def centerline_min_distance(a: Body, b: Body, nsamp: int = 160) -> float:
    """Sampled minimum distance between two centerlines (placement rejection test).

    Coarse sampling, then a 41x41 refinement around the best sample.  For unit-scale
    loops the result overestimates the true minimum by < 1e-3; callers add that margin.
    """
    s = np.arange(nsamp) / nsamp
    pa = a.xc(s)
    pb = b.xc(s)
    d2 = ((pa[:, None, 0] - pb[None, :, 0]) ** 2 + (pa[:, None, 1] - pb[None, :, 1]) ** 2
          + (pa[:, None, 2] - pb[None, :, 2]) ** 2)
    i, j = np.unravel_index(np.argmin(d2), d2.shape)
    ss = (i + np.linspace(-1, 1, 41)) / nsamp
    tt = (j + np.linspace(-1, 1, 41)) / nsamp
    qa, qb = a.xc(ss), b.xc(tt)
    d2f = ((qa[:, None, 0] - qb[None, :, 0]) ** 2 + (qa[:, None, 1] - qb[None, :, 1]) ** 2
           + (qa[:, None, 2] - qb[None, :, 2]) ** 2)
    return float(np.sqrt(min(d2.min(), d2f.min())))
