"""Thin Python binding of libslb's C-ABI (include/slb.h), same names as the C entry points.

Argument marshalling only: torch supplies device memory and the current CUDA stream; every
step of the operator runs in the library's CUDA kernels.  There is no CPU fallback: a missing
library, a CPU tensor or a wrong dtype raises.
"""
import ctypes

import torch

from ._native import lib, check, OperatorDesc, SlbError

LAPLACE_DL = 1
STOKES_SLDL = 2
STOKES_SL = 3        # slb_nearcorr_quad only: pure single-layer blocks


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t, name, dtype=torch.float64, allow_none=False):
    if t is None:
        if allow_none:
            return None
        raise SlbError(f"{name} is required")
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise SlbError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise SlbError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise SlbError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def slb_abi_version():
    return lib().slb_abi_version()


def slb_eta_cfie(rho):
    return lib().slb_eta_cfie(float(rho))


def slb_coincident_count():
    return lib().slb_coincident_count()


def slb_coincident_reset():
    lib().slb_coincident_reset()


def slb_launch_count():
    return int(lib().slb_launch_count())


def slb_upsample(sigma_coarse, n_panels, ns, nt, ms, mt, ncomp, out=None):
    if out is None:
        out = torch.empty(n_panels * ms * mt * ncomp, dtype=torch.float64, device=sigma_coarse.device)
    check(lib().slb_upsample(n_panels, ns, nt, ms, mt, ncomp, _dev(sigma_coarse, "sigma_coarse"),
                             _dev(out, "sigma_fine"), _stream()))
    return out


def _host_i32(a, name):
    import numpy as np
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    if arr.ndim != 1:
        raise SlbError(f"{name} must be a 1-D integer array")
    return arr


def slb_upsample_ragged(sigma_coarse, ns_panels, nt_panels, ms_panels, mt_panels, ncomp, out=None):
    """(NEXT N4) per-panel orders: panel p is ns[p] x nt[p] -> ms[p] x mt[p] (host int arrays; a
    scalar ns / ms applies to every panel)."""
    import numpy as np
    nt = _host_i32(nt_panels, "nt_panels")
    P = nt.size
    ns = _host_i32(np.broadcast_to(np.asarray(ns_panels), (P,)), "ns_panels")
    ms = _host_i32(np.broadcast_to(np.asarray(ms_panels), (P,)), "ms_panels")
    mt = _host_i32(np.broadcast_to(np.asarray(mt_panels), (P,)), "mt_panels")
    if out is None:
        out = torch.empty(int((ms.astype("int64") * mt).sum()) * ncomp, dtype=torch.float64,
                          device=sigma_coarse.device)
    vp = lambda a: ctypes.c_void_p(a.ctypes.data)
    check(lib().slb_upsample_ragged(P, vp(ns), vp(nt), vp(ms), vp(mt), ncomp, _dev(sigma_coarse, "sigma_coarse"),
                                    _dev(out, "sigma_fine"), _stream()))
    return out


def slb_farfield_laplace_dl(x_trg, y, n, w, sigma, out=None):
    T = x_trg.shape[0]
    if out is None:
        out = torch.empty(T, dtype=torch.float64, device=x_trg.device)
    check(lib().slb_farfield_laplace_dl(T, _dev(x_trg, "x_trg"), y.shape[0], _dev(y, "y"), _dev(n, "n"),
                                        _dev(w, "w"), _dev(sigma, "sigma"), _dev(out, "u"), _stream()))
    return out


def slb_farfield_stokes_sldl(x_trg, y, n, w, sigma, eta_src=None, eta=0.0, out=None):
    T = x_trg.shape[0]
    if out is None:
        out = torch.empty((T, 3), dtype=torch.float64, device=x_trg.device)
    check(lib().slb_farfield_stokes_sldl(T, _dev(x_trg, "x_trg"), y.shape[0], _dev(y, "y"), _dev(n, "n"),
                                         _dev(w, "w"), _dev(eta_src, "eta_src", allow_none=True), float(eta),
                                         _dev(sigma, "sigma"), _dev(out, "u"), _stream()))
    return out


def slb_nearcorr_apply(row_ptr, panel_idx, blocks, sigma_coarse, u, tdim, sdim, nodes_per_panel):
    T = row_ptr.shape[0] - 1
    check(lib().slb_nearcorr_apply(T, tdim, sdim, nodes_per_panel, _dev(row_ptr, "row_ptr", torch.int64),
                                   _dev(panel_idx, "panel_idx", torch.int32), _dev(blocks, "blocks"),
                                   _dev(sigma_coarse, "sigma_coarse"), _dev(u, "u"), _stream()))
    return u


def slb_nearcorr_fold(kernel, x_trg, row_ptr, panel_idx, ns, nt, ms, mt, y_fine, n_fine, w_fine, blocks,
                      eta_fine=None, eta=0.0):
    T = row_ptr.shape[0] - 1
    check(lib().slb_nearcorr_fold(kernel, T, _dev(x_trg, "x_trg"), _dev(row_ptr, "row_ptr", torch.int64),
                                  _dev(panel_idx, "panel_idx", torch.int32), ns, nt, ms, mt,
                                  _dev(y_fine, "y_fine"), _dev(n_fine, "n_fine"), _dev(w_fine, "w_fine"),
                                  _dev(eta_fine, "eta_fine", allow_none=True), float(eta),
                                  _dev(blocks, "blocks"), _stream()))
    return blocks


def slb_nearcorr_quad(kernel, x_trg, row_ptr, panel_idx, ns, nt, y_coarse, blocks, trg_node=None, eta_panel=None,
                      order=12, beta=0.6, panel_nt=None, panel_ns=None):
    """Special-quadrature blocks B for the CSR pairs (unfolded), written into `blocks`.
    panel_nt / panel_ns (host int arrays [n_panels]): ragged orders (NEXT N4); nt / ns then ignored."""
    import numpy as np
    T = row_ptr.shape[0] - 1
    if panel_nt is not None or panel_ns is not None:
        P = len(panel_nt) if panel_nt is not None else len(panel_ns)
        pnt = _host_i32(panel_nt if panel_nt is not None else np.full(P, nt), "panel_nt")
        pns = _host_i32(panel_ns if panel_ns is not None else np.full(P, ns), "panel_ns")
        check(lib().slb_nearcorr_quad_ragged(kernel, T, _dev(x_trg, "x_trg"),
                                             _dev(trg_node, "trg_node", torch.int64, True),
                                             _dev(row_ptr, "row_ptr", torch.int64),
                                             _dev(panel_idx, "panel_idx", torch.int32), P,
                                             ctypes.c_void_p(pns.ctypes.data),
                                             ctypes.c_void_p(pnt.ctypes.data), _dev(y_coarse, "y_coarse"),
                                             _dev(eta_panel, "eta_panel", allow_none=True), int(order), float(beta),
                                             _dev(blocks, "blocks"), _stream()))
        return blocks
    check(lib().slb_nearcorr_quad(kernel, T, _dev(x_trg, "x_trg"), _dev(trg_node, "trg_node", torch.int64, True),
                                  _dev(row_ptr, "row_ptr", torch.int64), _dev(panel_idx, "panel_idx", torch.int32),
                                  ns, nt, _dev(y_coarse, "y_coarse"), _dev(eta_panel, "eta_panel", allow_none=True),
                                  int(order), float(beta), _dev(blocks, "blocks"), _stream()))
    return blocks


def slb_fill_blocks(seed, first, count, s_blk, out):
    check(lib().slb_fill_blocks(ctypes.c_uint64(seed), ctypes.c_uint64(first), count, float(s_blk),
                                _dev(out, "blocks"), _stream()))
    return out


def slb_near_build(x_trg, y_nodes, radius, own_panel=None):
    """Near-list CSR on the GPU (R15): returns (row_ptr int64 [T+1], panel_idx int32 [nnz])."""
    T = x_trg.shape[0]
    P, Nn = y_nodes.shape[0], y_nodes.shape[1]
    row_ptr = torch.empty(T + 1, dtype=torch.int64, device=x_trg.device)
    nnz = ctypes.c_int64(0)
    args = (T, _dev(x_trg, "x_trg"), P, Nn, _dev(y_nodes, "y_nodes"), _dev(radius, "radius"),
            _dev(own_panel, "own_panel", torch.int64, allow_none=True), _dev(row_ptr, "row_ptr", torch.int64))
    check(lib().slb_near_build(*args, None, 0, ctypes.byref(nnz), _stream()))
    panel_idx = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=x_trg.device)
    check(lib().slb_near_build(*args, _dev(panel_idx, "panel_idx", torch.int32), panel_idx.numel(),
                               ctypes.byref(nnz), _stream()))
    return row_ptr, panel_idx[:nnz.value]


def slb_bench_dfma(iters=20000):
    g = ctypes.c_double(0.0)
    check(lib().slb_bench_dfma(int(iters), ctypes.byref(g), _stream()))
    return g.value


class Comm:
    """NCCL communicator (one process per GPU); the 128-byte id travels through torch.distributed."""

    def __init__(self, nranks, rank, group=None):
        import torch.distributed as dist
        idbuf = (ctypes.c_ubyte * 128)()
        if rank == 0:
            check(lib().slb_comm_unique_id(idbuf))
        t = torch.tensor(list(bytes(idbuf)), dtype=torch.uint8,
                         device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.broadcast(t, src=0, group=group)
        raw = bytes(t.cpu().tolist())
        idbuf = (ctypes.c_ubyte * 128).from_buffer_copy(raw)
        h = ctypes.c_void_p()
        check(lib().slb_comm_create(idbuf, nranks, rank, ctypes.byref(h)))
        self.h = h
        self.nranks, self.rank = nranks, rank

    def collective_counts(self):
        """(allgather, broadcast, allreduce) NCCL calls issued through this communicator."""
        out = (ctypes.c_longlong * 3)()
        check(lib().slb_comm_collective_counts(self.h, out))
        return {"allgather": out[0], "broadcast": out[1], "allreduce": out[2]}

    def close(self):
        if self.h:
            lib().slb_comm_destroy(self.h)
            self.h = None


class Operator:
    """slb_operator: the full operator apply on this rank.  Tensors passed in are borrowed
    (kept alive by this object).  blocks are folded in place (E = B - G U) unless folded=True."""

    def __init__(self, *, kernel, ns, nt, ms, mt, n_panels_global, panel_begin, panel_end, x_trg, n_on,
                 y_fine, n_fine, w_fine, row_ptr, panel_idx, blocks, c_identity=0.5, eta_fine=None, eta=0.0,
                 folded=False, n_bodies=0, body_of_panel=None, y_coarse=None, w_coarse=None, comm=None,
                 panel_nt=None, panel_mt=None, panel_ns=None, panel_ms=None):
        """panel_nt / panel_mt, panel_ns / panel_ms (host int arrays [n_panels_global]): ragged orders (NEXT N4)."""
        self._keep = [x_trg, y_fine, n_fine, w_fine, eta_fine, row_ptr, panel_idx, blocks, body_of_panel,
                      y_coarse, w_coarse]
        d = OperatorDesc()
        d.kernel, d.ns, d.nt, d.ms, d.mt = kernel, ns, nt, ms, mt
        d.n_panels_global, d.panel_begin, d.panel_end = n_panels_global, panel_begin, panel_end
        d.n_trg_local, d.n_on_local, d.c_identity = x_trg.shape[0], n_on, float(c_identity)
        d.x_trg = _dev(x_trg, "x_trg")
        d.y_fine, d.n_fine, d.w_fine = _dev(y_fine, "y_fine"), _dev(n_fine, "n_fine"), _dev(w_fine, "w_fine")
        d.eta_fine = _dev(eta_fine, "eta_fine", allow_none=True)
        d.eta = float(eta)
        d.row_ptr = _dev(row_ptr, "row_ptr", torch.int64)
        d.panel_idx = _dev(panel_idx, "panel_idx", torch.int32)
        d.blocks = _dev(blocks, "blocks")
        d.blocks_folded = 1 if folded else 0
        d.n_bodies_local = int(n_bodies)
        if n_bodies:
            d.body_of_panel_local = _dev(body_of_panel, "body_of_panel", torch.int32)
            d.y_coarse, d.w_coarse = _dev(y_coarse, "y_coarse"), _dev(w_coarse, "w_coarse")
        if (panel_nt is None) != (panel_mt is None) or (panel_ns is None) != (panel_ms is None):
            raise SlbError("panel_nt/panel_mt and panel_ns/panel_ms must be given in pairs")
        import numpy as np
        P = n_panels_global
        nn = np.full(P, ns, dtype=np.int64) * np.full(P, nt, dtype=np.int64)
        if panel_nt is not None:
            pnt, pmt = _host_i32(panel_nt, "panel_nt"), _host_i32(panel_mt, "panel_mt")
            self._keep += [pnt, pmt]
            d.panel_nt, d.panel_mt = pnt.ctypes.data, pmt.ctypes.data
            nn = nn // nt * pnt.astype(np.int64)
        if panel_ns is not None:
            pns, pms = _host_i32(panel_ns, "panel_ns"), _host_i32(panel_ms, "panel_ms")
            self._keep += [pns, pms]
            d.panel_ns, d.panel_ms = pns.ctypes.data, pms.ctypes.data
            nn = nn // ns * pns.astype(np.int64)
        self.n_loc_nodes = int(nn[panel_begin:panel_end].sum())
        self.desc = d
        self.kernel = kernel
        self.tdim = 1 if kernel == LAPLACE_DL else 3
        self.n_trg = x_trg.shape[0]
        self.comm = comm
        h = ctypes.c_void_p()
        check(lib().slb_operator_create(ctypes.byref(d), comm.h if comm is not None else None, ctypes.byref(h)))
        self.h = h

    def matvec(self, sigma_local, out=None):
        if out is None:
            out = torch.empty((self.n_trg, self.tdim), dtype=torch.float64, device=sigma_local.device)
        check(lib().slb_matvec(self.h, _dev(sigma_local, "sigma_local"), _dev(out, "u_local"), _stream()))
        return out

    def matvec_host(self, sigma_host, out_host):
        """Host-buffer variant (torch CPU tensors, ideally pinned): copies inside the call."""
        for t, nm in ((sigma_host, "sigma_host"), (out_host, "u_host")):
            if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
                raise SlbError(f"{nm} must be a contiguous float64 CPU tensor")
        check(lib().slb_matvec_host(self.h, ctypes.c_void_p(sigma_host.data_ptr()),
                                    ctypes.c_void_p(out_host.data_ptr()), _stream()))
        return out_host

    def gmres(self, rhs, x0=None, restart=50, max_iters=1000, tol=1e-12):
        """Solve A x = rhs with slb_gmres; returns (x, iterations, relative residual)."""
        x = torch.zeros_like(rhs) if x0 is None else x0.clone()
        it = ctypes.c_int(0)
        rr = ctypes.c_double(0.0)
        check(lib().slb_gmres(self.h, _dev(rhs, "rhs"), _dev(x, "x"), int(restart), int(max_iters), float(tol),
                              ctypes.byref(it), ctypes.byref(rr), _stream()))
        return x, it.value, rr.value

    def mobility_solve(self, sl, force_torque, sigma0=None, restart=100, max_iters=1000, tol=1e-12):
        """slb_mobility_solve: force_torque [n_bodies][6] (host, F and T about each body's centroid) ->
        (rigid [n_bodies][6] = (v, omega), sigma, iterations, relative residual).  `sl` is the
        single-layer Operator on the same nodes."""
        import numpy as np
        ft = np.ascontiguousarray(np.asarray(force_torque, dtype=np.float64).reshape(-1, 6))
        rig = np.empty_like(ft)
        x = torch.zeros((self.n_loc_nodes, 3), dtype=torch.float64, device="cuda") if sigma0 is None \
            else sigma0.clone()
        it = ctypes.c_int(0)
        rr = ctypes.c_double(0.0)
        check(lib().slb_mobility_solve(self.h, sl.h, ctypes.c_void_p(ft.ctypes.data), ctypes.c_void_p(rig.ctypes.data),
                                       _dev(x, "sigma"), int(restart), int(max_iters), float(tol), ctypes.byref(it),
                                       ctypes.byref(rr), _stream()))
        return rig, x, it.value, rr.value

    def prepare(self, sigma_local):
        """Stage 1 of an apply alone (projector + upsample into the fine records), for kernel timing."""
        check(lib().slb_operator_prepare(self.h, _dev(sigma_local, "sigma"), _stream()))

    def timings(self):
        arr = (ctypes.c_float * 4)()
        check(lib().slb_operator_last_timings(self.h, arr))
        return list(arr)

    def launches_per_matvec(self):
        return lib().slb_operator_launches_per_matvec(self.h)

    def uses_nvls(self):
        """True when the fine records are gathered through a multicast object (NEXT N4, SLB_NVLS=1)."""
        return bool(lib().slb_operator_nvls(self.h))

    def close(self):
        if self.h:
            lib().slb_operator_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
