"""Glue shared by tests and bench.py: turns a seeded synth.Problem into the device inputs
of one rank's slb_operator (no method arithmetic here: slicing, copying, seeded fill)."""
import numpy as np
import torch

from paper_2310_00889_b200 import Operator, partition_panels, slb_fill_blocks, slb_nearcorr_quad


def local_rows(pr, rank, nranks):
    """Global target ids owned by `rank`, the panel range, and n_on_local."""
    ranges = partition_panels(pr.P, nranks, pr.body_of_panel, whole_bodies=pr.projector)
    pb, pe = ranges[rank]
    no = pr.node_off()
    rows = np.arange(no[pb], no[pe], dtype=np.int64)
    if rank == 0 and pr.T > pr.n_on:
        rows = np.concatenate([rows, np.arange(pr.n_on, pr.T, dtype=np.int64)])
    return rows, pb, pe, int(no[pe] - no[pb]), ranges


def _segments(rows):
    """Contiguous runs [a, b) of a sorted-by-construction row list."""
    if rows.size == 0:
        return []
    br = np.nonzero(np.diff(rows) != 1)[0] + 1
    starts = np.concatenate([[0], br])
    ends = np.concatenate([br, [rows.size]])
    return [(int(rows[s]), int(rows[e - 1]) + 1) for s, e in zip(starts, ends)]


class DeviceProblem:
    def __init__(self, pr, rank=0, nranks=1, device="cuda", fold=True, comm=None, blocks=None, quad=None,
                 slice_only=False, single_layer=False):
        """blocks: None -> seeded synthetic B (R10); quad=dict(order=.., beta=..) -> special-quadrature
        B computed on the GPU by slb_nearcorr_quad (N1).
        slice_only: a ONE-GPU operator over rank `rank`'s target rows of an `nranks` partition with all
        source panels (no communicator, identity term off) -- the per-rank compute of the sharded
        operator, for timing projections (tools/scaling_projection.py).
        single_layer: the pure single layer (Stokes S or Laplace S_L) on the same nodes (eta = 1, zero
        normals, no identity term, no projector; quad blocks with SLB_STOKES_SL / SLB_LAPLACE_SL) --
        e.g. the `sl` of slb_mobility_solve."""
        if single_layer:
            import copy
            pr = copy.copy(pr)
            pr.n_f = np.zeros_like(pr.n_f)
            pr.eta_f = np.ones_like(pr.eta_f)
            pr.eta_body = np.ones_like(pr.eta_body)
            pr.c_identity = 0.0
            pr.projector = False
        self.pr = pr
        rows, pb, pe, n_on, ranges = local_rows(pr, rank, nranks)
        if slice_only:
            pb, pe, n_on = 0, pr.P, 0
        self.rows, self.pb, self.pe, self.n_on, self.ranges = rows, pb, pe, n_on, ranges
        dev = torch.device(device)
        f64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
        rp = pr.row_ptr
        cnt = rp[rows + 1] - rp[rows]
        row_ptr = np.zeros(rows.size + 1, np.int64)
        np.cumsum(cnt, out=row_ptr[1:])
        segs = _segments(rows)
        pidx = np.concatenate([pr.panel_idx[rp[a]:rp[b]] for a, b in segs]) if segs else np.zeros(0, np.int32)
        self.nnz = int(row_ptr[-1])
        bo = pr.blk_off()                      # global block offsets (ragged-safe)
        n_entries = int(sum(bo[rp[b]] - bo[rp[a]] for a, b in segs))
        self.n_entries = n_entries
        if quad is not None:
            self.blocks = torch.empty(max(n_entries, 2), dtype=torch.float64, device=dev)
        elif blocks is None:
            self.blocks = torch.empty(max(n_entries, 2), dtype=torch.float64, device=dev)
            off = 0
            for a, b in segs:
                n = int(bo[rp[b]] - bo[rp[a]])
                if n:
                    slb_fill_blocks(pr.blk_seed, int(bo[rp[a]]), n, pr.s_blk, self.blocks[off:off + n])
                off += n
        else:
            self.blocks = blocks
        self.x_trg = f64(pr.x_trg[rows])
        if quad is not None and self.nnz > 0:
            trg_node = torch.from_numpy(np.where(rows < pr.n_on, rows, -1).astype(np.int64)).to(dev)
            eta_panel = f64(pr.eta_body[pr.body_of_panel]) if (pr.kernel == 2 or np.any(pr.eta_body != 0)) else None
            rp_d = torch.from_numpy(row_ptr).to(dev)
            pi_d = torch.from_numpy(np.ascontiguousarray(pidx, dtype=np.int32)).to(dev)
            qk = (3 if pr.kernel == 2 else 4) if single_layer else pr.kernel
            slb_nearcorr_quad(qk, self.x_trg, rp_d, pi_d, pr.Ns, pr.Nt, f64(pr.y_c),
                              self.blocks, trg_node=trg_node, eta_panel=None if single_layer else eta_panel, order=quad.get("order", 0),
                              beta=quad.get("beta", 0.6), panel_nt=pr.nt_of_panel() if pr.ragged else None,
                              panel_ns=pr.ns_of_panel() if pr.ragged else None)
        self.y_f, self.n_f, self.w_f = f64(pr.y_f), f64(pr.n_f), f64(pr.w_f)
        # pure double layer (all eta = 0) runs the DL kernel: eta_fine must then be NULL
        self.eta_f = f64(pr.eta_f) if np.any(pr.eta_f != 0) else None
        self.row_ptr = torch.from_numpy(row_ptr).to(dev)
        self.panel_idx = torch.from_numpy(np.ascontiguousarray(pidx, dtype=np.int32)).to(dev)
        no = pr.node_off()
        sig = pr.sigma.reshape(pr.N, pr.sdim)[no[pb]:no[pe]]
        self.sigma = f64(sig)
        nb = 0
        bop = y_c = w_c = None
        if pr.projector:
            b_loc = pr.body_of_panel[pb:pe]
            nb = int(b_loc.max() - b_loc.min() + 1) if b_loc.size else 0
            bop = torch.from_numpy((b_loc - (b_loc.min() if b_loc.size else 0)).astype(np.int32)).to(dev)
            y_c = f64(pr.y_c[no[pb]:no[pe]])
            w_c = f64(pr.w_c[no[pb]:no[pe]])
        self.op = Operator(kernel=pr.kernel, ns=pr.Ns, nt=pr.Nt, ms=pr.Ms, mt=pr.Mt, n_panels_global=pr.P,
                           panel_begin=pb, panel_end=pe, x_trg=self.x_trg, n_on=n_on, y_fine=self.y_f,
                           n_fine=self.n_f, w_fine=self.w_f, row_ptr=self.row_ptr, panel_idx=self.panel_idx,
                           blocks=self.blocks, c_identity=0.0 if slice_only else pr.c_identity,
                           eta_fine=self.eta_f, eta=0.0,
                           folded=not fold, n_bodies=nb, body_of_panel=bop, y_coarse=y_c, w_coarse=w_c,
                           comm=comm, panel_nt=pr.nt_of_panel() if pr.ragged else None,
                           panel_mt=pr.mt_of_panel() if pr.ragged else None,
                           panel_ns=pr.ns_of_panel() if pr.ragged else None,
                           panel_ms=pr.ms_of_panel() if pr.ragged else None)

    def matvec(self, sigma=None, out=None):
        return self.op.matvec(self.sigma if sigma is None else sigma, out)

    def close(self):
        self.op.close()
