"""Example: the sedimentation speed of a slender ring (PAPER.md Table t:conv-sbt) with the library's
public API on one B200 -- special-quadrature blocks, the mobility operator and slb_mobility_solve.

    python examples/sedimenting_ring.py [rho] [panels] [N_theta]

Steps (all on the GPU through libslb): geometry (nodes, normals, weights on the coarse and the 2x
fine grid) -> near lists (slb_near_build) -> special-quadrature blocks for the CFIE kernel and for
the pure single layer (slb_nearcorr_quad) -> two operators (slb_operator_create: the mobility
operator K(I-L)+L and the single layer S) -> slb_mobility_solve -> rigid velocity.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_00889_b200 as slb  # noqa: E402
from synth import make_torus_problem  # noqa: E402  (geometry and near-list generator)


def cu(a, dt=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)


def main():
    rho = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    Nt = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    eta = slb.slb_eta_cfie(rho)                                   # 1 / (2 rho ln(1/rho))
    pr = make_torus_problem(rho=rho, panels=P, Nt=Nt, kernel=slb.STOKES_SLDL)
    x = cu(pr.x_trg)
    # near lists on the GPU: panels within 2 panel lengths of a target, plus the target's own panel
    own = cu(np.repeat(np.arange(pr.P), pr.Nn), torch.int64)
    row_ptr, panel_idx = slb.slb_near_build(x, cu(pr.y_c.reshape(pr.P, pr.Nn, 3)), cu(2 * pr.panel_len), own)
    nnz = panel_idx.numel()
    node = cu(np.arange(pr.N), torch.int64)                       # every target is a node (on-surface)

    def operator(kernel_quad, eta_fine, normals, c_identity, projector):
        blocks = torch.empty(nnz * 3 * pr.Nn * 3, dtype=torch.float64, device="cuda")
        slb.slb_nearcorr_quad(kernel_quad, x, row_ptr, panel_idx, pr.Ns, pr.Nt, cu(pr.y_c), blocks, trg_node=node,
                              eta_panel=cu(np.full(pr.P, eta)) if kernel_quad == slb.STOKES_SLDL else None,
                              order=14, beta=0.6)
        kw = {}
        if projector:
            kw = dict(n_bodies=1, body_of_panel=torch.zeros(pr.P, dtype=torch.int32, device="cuda"),
                      y_coarse=cu(pr.y_c), w_coarse=cu(pr.w_c))
        return slb.Operator(kernel=slb.STOKES_SLDL, ns=pr.Ns, nt=pr.Nt, ms=pr.Ms, mt=pr.Mt, n_panels_global=pr.P,
                            panel_begin=0, panel_end=pr.P, x_trg=x, n_on=pr.N, y_fine=cu(pr.y_f), n_fine=normals,
                            w_fine=cu(pr.w_f), row_ptr=row_ptr, panel_idx=panel_idx, blocks=blocks,
                            c_identity=c_identity, eta_fine=eta_fine, **kw), blocks

    mob, b1 = operator(slb.STOKES_SLDL, cu(np.full(pr.M, eta)), cu(pr.n_f), 0.5, True)      # K(I-L) + L
    sl, b2 = operator(slb.STOKES_SL, cu(np.ones(pr.M)), cu(np.zeros_like(pr.n_f)), 0.0, False)  # S
    rigid, sigma, iters, relres = mob.mobility_solve(sl, [[0, 0, -1.0, 0, 0, 0]], tol=1e-13)
    U = -rigid[0, 2]
    print(f"rho = {rho:g}: {pr.N * 3} unknowns, GMRES {iters} iterations (residual {relres:.1e}); "
          f"sedimentation speed U = {U:.15f}")
    print("paper (Table t:conv-sbt): 0.0614921383598558 (rho 0.1), 0.0909845223245838 (rho 0.01)")
    mob.close()
    sl.close()


if __name__ == "__main__":
    main()
