"""Development aid: dump GPU special-quadrature blocks (order 0) of c3's parity-test pairs to gpurun_out/."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2310_00889_b200 as S
from synth import make_config
import test_gpu_nearquad_parity as T

pr = make_config('c3')
trip = T._pairs(pr, 0.05, extra_k=0)
X = np.array([t[0] for t in trip]); nodes = np.array([t[1] for t in trip], np.int64); pid = np.array([t[2] for t in trip], np.int32)
rp = np.arange(len(trip) + 1, dtype=np.int64)
blocks = torch.empty(len(trip) * 9 * pr.Nn, dtype=torch.float64, device="cuda")
S.slb_nearcorr_quad(2, T.cu(X), T.cu(rp, torch.int64), T.cu(pid, torch.int32), pr.Ns, pr.Nt, T.cu(pr.y_c.reshape(pr.P, pr.Nn, 3)),
                    blocks, trg_node=T.cu(nodes, torch.int64), eta_panel=T.cu(pr.eta_body[pr.body_of_panel]), order=0)
np.save('gpurun_out/r02f/c3_blocks.npy', blocks.cpu().numpy().reshape(len(trip), 3, -1))
