"""CPU oracle for the slender-body Nystrom operator apply -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs may import this package.  The product path (paper_2310_00889_b200) never imports
it and shares no code with it.  The arithmetic lives in slb_oracle.c (plain C, fp64,
no fast-math, no FMA contraction, Neumaier-compensated sums); this module only builds
it with gcc and marshals numpy arrays through ctypes.

Parity status per function:
  or_gauss_legendre, or_lagrange_matrix, or_trig_matrix, or_upsample  -- pinned (P7, exactness)
  or_farfield (Laplace DL, Stokes eta S + D)                            -- pinned (P1-P6, P9, P10, P12)
  or_projector                                                          -- pinned (P13)
  or_nearquad_block / or_nearquad (N1 special-quadrature blocks)       -- pinned (jump relations, Prop. 1,
      S[n] = 0, Green's representation, Table t:conv-biest bound, identity term; test_oracle_pins "N1")
  or_apply_rows (full operator)                                         -- pinned via its parts + P11;
      the synthetic B-block VALUES are "parity unpinned" (no paper value exists).
"""
import ctypes
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "slb_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "slb_quad_oracle.c")]
_SO = os.path.join(_HERE, "libslb_oracle.so")
_lib = None

CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11"]


def build(force=False):
    if force or not os.path.exists(_SO) or any(os.path.getmtime(_SO) < os.path.getmtime(f) for f in _SRCS):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO, *_SRCS, "-lm"])
    return _SO


class OrProblem(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("ns", ctypes.c_int), ("nt", ctypes.c_int),
                ("ms", ctypes.c_int), ("mt", ctypes.c_int), ("n_panels", ctypes.c_long),
                ("n_trg", ctypes.c_long), ("n_on", ctypes.c_long), ("c_identity", ctypes.c_double),
                ("x_trg", ctypes.c_void_p), ("y_f", ctypes.c_void_p), ("n_f", ctypes.c_void_p),
                ("w_f", ctypes.c_void_p), ("eta_f", ctypes.c_void_p), ("row_ptr", ctypes.c_void_p),
                ("panel_idx", ctypes.c_void_p), ("blk_seed", ctypes.c_uint64),
                ("s_blk", ctypes.c_double), ("blocks", ctypes.c_void_p), ("n_bodies", ctypes.c_int),
                ("body_of_node", ctypes.c_void_p), ("y_c", ctypes.c_void_p), ("w_c", ctypes.c_void_p),
                ("panel_nt", ctypes.c_void_p), ("panel_mt", ctypes.c_void_p),
                ("panel_ns", ctypes.c_void_p), ("panel_ms", ctypes.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        L.or_gauss_legendre.argtypes = [ctypes.c_int, P, P]
        L.or_lagrange_matrix.argtypes = [ctypes.c_int, P, ctypes.c_int, P, P]
        L.or_trig_matrix.argtypes = [ctypes.c_int, ctypes.c_int, P]
        L.or_upsample.argtypes = [ctypes.c_long] + [ctypes.c_int] * 5 + [P, P]
        L.or_upsample_ragged.argtypes = [ctypes.c_long, P, P, P, P, ctypes.c_int, P, P]
        L.or_kernel_matrix.argtypes = [ctypes.c_int, P, P, ctypes.c_double, P]
        L.or_farfield.argtypes = [ctypes.c_int, ctypes.c_long, P, ctypes.c_long, P, P, P, P, P, P]
        L.or_splitmix64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.or_splitmix64.restype = ctypes.c_uint64
        L.or_block_entry.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double]
        L.or_block_entry.restype = ctypes.c_double
        L.or_block_entries.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_long,
                                       ctypes.c_double, P]
        L.or_projector.argtypes = [ctypes.c_long, P, P, P, ctypes.c_int, P, P]
        L.or_eta_cfie.argtypes = [ctypes.c_double]
        L.or_eta_cfie.restype = ctypes.c_double
        L.or_prepare.argtypes = [ctypes.POINTER(OrProblem), P, P, P, P]
        L.or_apply_rows.argtypes = [ctypes.POINTER(OrProblem), P, P, P, ctypes.c_long, P, P, P, P]
        L.or_nearcorr_apply.argtypes = [ctypes.c_long, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        P, P, P, P, P]
        L.or_nearquad_block.argtypes = [ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P, ctypes.c_double,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_double, P]
        L.or_nearquad.argtypes = [ctypes.c_int, ctypes.c_long, P, P, P, P, ctypes.c_int, ctypes.c_int, P, P,
                                  ctypes.c_double, P]
        L.or_num_threads.restype = ctypes.c_int
        L.or_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


def num_threads():
    return lib().or_num_threads()


def set_num_threads(n):
    lib().or_set_num_threads(int(n))


def gauss_legendre(n):
    x = np.empty(n)
    w = np.empty(n)
    lib().or_gauss_legendre(n, _p(x), _p(w))
    return x, w


def lagrange_matrix(s_from, s_to):
    s_from, s_to = _c(s_from), _c(s_to)
    P = np.empty((s_to.size, s_from.size))
    lib().or_lagrange_matrix(s_from.size, _p(s_from), s_to.size, _p(s_to), _p(P))
    return P


def trig_matrix(N, M):
    F = np.empty((M, N))
    lib().or_trig_matrix(N, M, _p(F))
    return F


def upsample(sigma_c, n_panels, ns, nt, ms, mt, nc):
    sigma_c = _c(sigma_c)
    out = np.empty(n_panels * ms * mt * nc)
    lib().or_upsample(n_panels, ns, nt, ms, mt, nc, _p(sigma_c), _p(out))
    return out.reshape(n_panels * ms * mt, nc) if nc > 1 else out


def upsample_ragged(sigma_c, ns_panels, nt_panels, ms_panels, mt_panels, nc):
    """per-panel orders (NEXT N4): panel k is ns[k] x nt[k] -> ms[k] x mt[k] (ints broadcast)"""
    nt = _c(nt_panels, np.int32)
    P = nt.size
    ns = _c(np.broadcast_to(np.asarray(ns_panels), (P,)), np.int32)
    ms = _c(np.broadcast_to(np.asarray(ms_panels), (P,)), np.int32)
    mt = _c(np.broadcast_to(np.asarray(mt_panels), (P,)), np.int32)
    sigma_c = _c(sigma_c)
    out = np.empty(int((ms.astype(np.int64) * mt).sum()) * nc)
    lib().or_upsample_ragged(P, _p(ns), _p(nt), _p(ms), _p(mt), nc, _p(sigma_c), _p(out))
    return out


def kernel_matrix(kind, r, n=(0.0, 0.0, 0.0), eta=0.0):
    r = _c(r)
    n = _c(n)
    K = np.zeros(9)
    lib().or_kernel_matrix(kind, _p(r), _p(n), float(eta), _p(K))
    return K[0] if kind in (1, 3) else K.reshape(3, 3)


def farfield(kind, x, y, n, w, sigma, eta=None):
    """kind 1: Laplace D + eta S_L (eta None: D); 2: Stokes eta S + D; 3: Laplace SL.  r = 0 skipped."""
    x, y, w, sigma = _c(x), _c(y), _c(w), _c(sigma)
    n = _c(n) if n is not None else None
    eta = _c(eta) if eta is not None else None
    d = 3 if kind == 2 else 1
    u = np.empty(x.shape[0] * d)
    lib().or_farfield(kind, x.shape[0], _p(x), y.shape[0], _p(y), _p(n), _p(w), _p(eta),
                      _p(sigma), _p(u))
    return u.reshape(-1, d) if d == 3 else u


def splitmix64(seed, i):
    return int(lib().or_splitmix64(seed, i))


def block_entries(seed, first, count, s_blk):
    out = np.empty(count)
    lib().or_block_entries(seed, first, count, s_blk, _p(out))
    return out


def projector(y, w, body_of_node, n_bodies, sigma):
    y, w, sigma = _c(y), _c(w), _c(sigma)
    b = _c(body_of_node, np.int32)
    out = np.empty_like(sigma)
    lib().or_projector(y.shape[0], _p(y), _p(w), _p(b), int(n_bodies), _p(sigma), _p(out))
    return out


def eta_cfie(rho):
    return lib().or_eta_cfie(rho)


def nearcorr_apply(T, tdim, sdim, nodes_per_panel, row_ptr, panel_idx, blocks, sigma_c, u):
    row_ptr, panel_idx = _c(row_ptr, np.int64), _c(panel_idx, np.int32)
    blocks, sigma_c = _c(blocks), _c(sigma_c)
    u = _c(u).copy()
    lib().or_nearcorr_apply(T, tdim, sdim, nodes_per_panel, _p(row_ptr), _p(panel_idx),
                            _p(blocks), _p(sigma_c), _p(u))
    return u


def nearquad_block(kernel, x, y_panel, eta=0.0, node=None, tol=1e-13):
    """(N1) Special-quadrature block of one element by nested adaptive Gauss-Kronrod (slb_quad_oracle.c).
    kernel: slb_kernel id (1 Laplace D + eta S_L, 2 Stokes eta S + D, 3 Stokes eta S, 4 Laplace eta S_L);
    y_panel [ns][nt][3]; node = (i0, j0) if x is that node of the element (singular), else None.
    Returns B [tdim][ns*nt*sdim]."""
    y = _c(y_panel)
    ns, nt = y.shape[0], y.shape[1]
    d = 3 if kernel in (2, 3) else 1
    B = np.empty((d, ns * nt * d))
    i0, j0 = node if node is not None else (-1, -1)
    lib().or_nearquad_block(kernel, _p(_c(x)), ns, nt, _p(y), float(eta), int(i0), int(j0), float(tol), _p(B))
    return B


def nearquad(kernel, x_trg, row_ptr, panel_idx, ns, nt, y_coarse, trg_node=None, eta_panel=None, tol=1e-13):
    """(N1) All CSR pairs, same arguments as slb_nearcorr_quad (uniform orders).  Returns blocks [nnz][tdim][cols]."""
    x, rp, pi = _c(x_trg), _c(row_ptr, np.int64), _c(panel_idx, np.int32)
    yc = _c(y_coarse)
    tn = None if trg_node is None else _c(trg_node, np.int64)
    ep = None if eta_panel is None else _c(eta_panel)
    d = 3 if kernel in (2, 3) else 1
    out = np.empty((int(rp[-1]), d, ns * nt * d))
    lib().or_nearquad(kernel, x.shape[0], _p(x), _p(tn), _p(rp), _p(pi), ns, nt, _p(yc), _p(ep), float(tol),
                      _p(out))
    return out


class Oracle:
    """Full operator of a synth.Problem, evaluated row by row."""

    def __init__(self, pr, blocks=None):
        self.pr = pr
        self._keep = dict(x=_c(pr.x_trg), y_f=_c(pr.y_f), n_f=_c(pr.n_f), w_f=_c(pr.w_f),
                          eta_f=_c(pr.eta_f), row_ptr=_c(pr.row_ptr, np.int64),
                          panel_idx=_c(pr.panel_idx, np.int32),
                          blocks=None if blocks is None else _c(blocks),
                          body=_c(np.repeat(pr.body_of_panel, np.diff(pr.node_off())), np.int32),
                          y_c=_c(pr.y_c), w_c=_c(pr.w_c),
                          pnt=_c(pr.nt_of_panel(), np.int32) if pr.ragged else None,
                          pmt=_c(pr.mt_of_panel(), np.int32) if pr.ragged else None,
                          pns=_c(pr.ns_of_panel(), np.int32) if pr.ragged else None,
                          pms=_c(pr.ms_of_panel(), np.int32) if pr.ragged else None)
        k = self._keep
        self.s = OrProblem(kind=pr.kernel, ns=pr.Ns, nt=pr.Nt, ms=pr.Ms, mt=pr.Mt,
                           n_panels=pr.P, n_trg=pr.T, n_on=pr.n_on, c_identity=pr.c_identity,
                           x_trg=_p(k["x"]), y_f=_p(k["y_f"]), n_f=_p(k["n_f"]), w_f=_p(k["w_f"]),
                           eta_f=_p(k["eta_f"]), row_ptr=_p(k["row_ptr"]),
                           panel_idx=_p(k["panel_idx"]), blk_seed=pr.blk_seed, s_blk=pr.s_blk,
                           blocks=_p(k["blocks"]), n_bodies=pr.n_bodies if pr.projector else 0,
                           body_of_node=_p(k["body"]), y_c=_p(k["y_c"]), w_c=_p(k["w_c"]),
                           panel_nt=_p(k["pnt"]), panel_mt=_p(k["pmt"]),
                           panel_ns=_p(k["pns"]), panel_ms=_p(k["pms"]))

    def prepare(self, sigma):
        pr = self.pr
        d = pr.sdim
        sigma = _c(sigma).reshape(pr.N, d)
        sp = np.empty_like(sigma)
        sf = np.empty((pr.M, d))
        Ls = np.empty_like(sigma)
        lib().or_prepare(ctypes.byref(self.s), _p(sigma), _p(sp), _p(sf), _p(Ls))
        return sp, sf, Ls

    def apply_rows(self, sigma, rows, parts=False, prepared=None):
        pr = self.pr
        d = pr.sdim
        sp, sf, Ls = prepared if prepared is not None else self.prepare(sigma)
        rows = _c(rows, np.int64)
        u = np.empty((rows.size, d))
        uf = np.empty((rows.size, d))
        un = np.empty((rows.size, d))
        lib().or_apply_rows(ctypes.byref(self.s), _p(sp), _p(sf), _p(Ls), rows.size, _p(rows),
                            _p(u), _p(uf), _p(un))
        if parts:
            return u, uf, un
        return u
