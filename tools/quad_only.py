"""One special-quadrature call (slb_nearcorr_quad, NEXT N1) on a workload -- for ncu captures.
usage: python tools/quad_only.py [c3v] [order]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_00889_b200 as S  # noqa: E402
from synth import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3v"
order = int(sys.argv[2]) if len(sys.argv) > 2 else 14
pr = make_config(name)
cu = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
trg_node = cu(np.where(np.arange(pr.T) < pr.n_on, np.arange(pr.T), -1).astype(np.int64), torch.int64)
eta_panel = cu(pr.eta_body[pr.body_of_panel]) if pr.kernel == 2 else None
blocks = torch.empty(pr.n_blocks_entries(), dtype=torch.float64, device="cuda")
rag = dict(panel_nt=pr.nt_of_panel(), panel_ns=pr.ns_of_panel()) if pr.ragged else {}
S.slb_nearcorr_quad(pr.kernel, cu(pr.x_trg), cu(pr.row_ptr, torch.int64), cu(pr.panel_idx, torch.int32), pr.Ns, pr.Nt,
                    cu(pr.y_c), blocks, trg_node=trg_node, eta_panel=eta_panel, order=order, beta=0.6, **rag)
torch.cuda.synchronize()
print("ok", name, order, float(blocks.abs().sum()))
