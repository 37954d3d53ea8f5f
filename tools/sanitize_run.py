"""Tiny end-to-end exercise of every libslb kernel, for compute-sanitizer (dev tool; the shared
GPU pool does not allow compute-sanitizer, so this is for a local machine):
    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_run.py
Run it a second time with SLB_NEAR_CHUNKED_UNIFORM=1 (read once per process) to send the
uniform blocks through the chunked near stream.  Covers both far paths, uniform and ragged (N4) meshes, the chunked near stream, the fold, GMRES,
the special-quadrature blocks (N1) for all four kernels, the near-list build (N3), the projector
and slb_mobility_solve."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import make_config, make_torus_problem  # noqa: E402
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
S.slb_upsample_ragged(cu(pr.sigma[:pr.Nn * 2]), [pr.Ns, pr.Ns], [pr.Nt, pr.Nt], pr.Ms, [pr.Mt, pr.Mt], 3)
# ragged mesh (N4), both kernels; special-quadrature blocks (N1) for DL / SLDL / SL kernels
rag = dict(panels=4, nt_panels=np.array([12, 8, 16, 8]), ns_panels=np.array([10, 8, 10, 6]))
for kernel in (1, 2):
    for path in ("tma", "const"):
        os.environ["SLB_FAR_PATH"] = path
        pr = make_torus_problem(rho=0.1, kernel=kernel, eta=0.5, **rag)
        dp = DeviceProblem(pr, quad=dict(order=6, beta=0.6))
        u = dp.matvec()
        dp.op.gmres(u.clone(), restart=5, max_iters=8, tol=1e-8)
        dp.close()
        sl = DeviceProblem(pr, quad=dict(order=6, beta=0.6), single_layer=True)
        sl.matvec()
        sl.close()
# projector + mobility solve on a small uniform torus
import copy  # noqa: E402
pr = make_torus_problem(rho=0.1, panels=4, Nt=8, kernel=2)
p = copy.copy(pr)
p.projector = True
mob, sl = DeviceProblem(p, quad=dict(order=6, beta=0.6)), DeviceProblem(pr, quad=dict(order=6, beta=0.6), single_layer=True)
mob.op.mobility_solve(sl.op, [[0, 0, -1.0, 0, 0, 0]], restart=5, max_iters=8, tol=1e-8)
mob.close(); sl.close()
torch.cuda.synchronize()
print("sanitize_run ok")
