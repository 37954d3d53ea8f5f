"""N1 timing helper: slb_nearcorr_quad (paper's rule) on one workload, device time; optional ncu target."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_00889_b200 as S
from synth import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
pr = make_config(name)
cu = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
x = cu(pr.x_trg)
tn = cu(np.where(np.arange(pr.T) < pr.n_on, np.arange(pr.T), -1).astype(np.int64), torch.int64)
eta = cu(pr.eta_body[pr.body_of_panel])
blocks = torch.empty(pr.n_blocks_entries(), dtype=torch.float64, device="cuda")
rp, pi = cu(pr.row_ptr, torch.int64), cu(pr.panel_idx, torch.int32)
rag = dict(panel_nt=pr.nt_of_panel(), panel_ns=pr.ns_of_panel()) if pr.ragged else {}
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S.slb_nearcorr_quad(pr.kernel, x, rp, pi, pr.Ns, pr.Nt, cu(pr.y_c), blocks, trg_node=tn, eta_panel=eta, order=0, **rag)
    torch.cuda.synchronize()
    print(name, "seconds", time.perf_counter() - t0, "unknowns/s", pr.N * pr.sdim / (time.perf_counter() - t0), flush=True)
