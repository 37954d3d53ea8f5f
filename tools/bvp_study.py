"""Resolution study of the exterior Dirichlet CFIE check (tests/test_gpu_bvp.py)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_bvp import exterior_targets, line_source_field, cu  # noqa: E402
from harness import DeviceProblem  # noqa: E402
from synth import make_torus_problem  # noqa: E402

for spec in sys.argv[1:]:
    f = spec.split(":")
    kernel, rho, P, Nt, order = int(f[0]), float(f[1]), int(f[2]), int(f[3]), int(f[4])
    beta = float(f[5]) if len(f) > 5 else 0.6
    quad = dict(order=order, beta=beta)
    eta = 1.0 / (2 * rho * np.log(1 / rho))
    X = exterior_targets(1.0, rho)
    pr = make_torus_problem(rho=rho, panels=P, Nt=Nt, kernel=kernel, eta=eta)
    u0 = line_source_field(pr.y_c, 1.0, kernel)
    u0 = u0[:, None] if kernel == 1 else u0
    exact = line_source_field(X, 1.0, kernel)
    dp = DeviceProblem(pr, quad=quad)
    sig, it, rr = dp.op.gmres(cu(u0), restart=100, max_iters=500, tol=1e-14)
    dp.close()
    pe = make_torus_problem(rho=rho, panels=P, Nt=Nt, kernel=kernel, eta=eta, extra_targets=X)
    ev = DeviceProblem(pe, quad=quad)
    u = ev.matvec(sig).cpu().numpy()[pe.n_on:]
    ev.close()
    u = u[:, 0] if kernel == 1 else u
    err = np.abs(u - exact).reshape(len(X), -1).max(1) / np.abs(exact).max()
    d = np.hypot(np.hypot(X[:, 0], X[:, 1]) - 1.0, X[:, 2]) / rho
    print(f"{spec}: N={pr.N} it={it} err={err.max():.2e}  err(d<2rho)={err[d < 2].max():.2e} err(d>2rho)={err[d >= 2].max():.2e}", flush=True)
    nn = np.diff(pe.row_ptr)[pe.n_on:]
    for q in np.argsort(err)[-6:]:
        print(f"    target {q}: d/rho={d[q]:.2f} |x|={np.linalg.norm(X[q]):.3f} near panels={nn[q]} err={err[q]:.2e}")
