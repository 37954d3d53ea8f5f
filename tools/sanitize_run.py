"""Tiny end-to-end exercise of every libslb kernel, for compute-sanitizer (dev tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import make_config  # noqa: E402
from harness import DeviceProblem  # noqa: E402
import paper_2310_00889_b200 as S  # noqa: E402

cu = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
for path in ("tma", "const"):
    os.environ["SLB_FAR_PATH"] = path
    for name, kw in (("c1", dict(panels=2, n_extra=7)), ("c4", dict(n_loops=2, panels=3)), ("c2", dict(panels=3))):
        pr = make_config(name, **kw)
        dp = DeviceProblem(pr)
        u = dp.matvec()
        if pr.T == pr.N:
            dp.op.gmres(u.clone(), restart=5, max_iters=12, tol=1e-8)
        dp.close()
pr = make_config("c2", panels=3)
S.slb_upsample(cu(pr.sigma), pr.P, pr.Ns, pr.Nt, pr.Ms, pr.Mt, 3)
S.slb_farfield_stokes_sldl(cu(pr.x_trg[:37]), cu(pr.y_f), cu(pr.n_f), cu(pr.w_f), cu(pr.sigma.repeat(4, 0)[:pr.M]),
                           eta_src=cu(pr.eta_f))
S.slb_near_build(cu(pr.x_trg), cu(pr.y_c.reshape(pr.P, pr.Nn, 3)), cu(2 * pr.panel_len))
torch.cuda.synchronize()
print("sanitize_run ok")
