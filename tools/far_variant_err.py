"""Parity of the operator apply against the CPU oracle for the far-kernel variant selected by
SLB_CONST_VARIANT (dev tool): prints the relative max-norm error on c3 (close tori, sampled rows near the
gap), c2 and a reduced c4 with the constant-bank far path forced."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SLB_FAR_PATH"] = "const"
import oracle
from synth import make_config
from harness import DeviceProblem

for name, kw in (("c3", {}), ("c2", {}), ("c4", dict(n_loops=4, panels=8))):
    pr = make_config(name, **kw)
    rng = np.random.default_rng(3)
    if name == "c3":
        gap = np.argsort(np.abs(pr.x_trg[:, 0] - 1.05125))[:64]
        rows = np.unique(np.concatenate([gap, rng.choice(pr.T, 192, replace=False)]))
    else:
        rows = np.unique(rng.choice(pr.T, min(pr.T, 512), replace=False))
    dp = DeviceProblem(pr)
    u = dp.matvec().cpu().numpy().reshape(pr.T, pr.tdim)
    ref = oracle.Oracle(pr).apply_rows(pr.sigma, rows)
    err = float(np.abs(u[rows] - ref).max() / np.abs(ref).max())
    print(f"variant {os.environ.get('SLB_CONST_VARIANT', '0')} {name}: rel max-norm err vs oracle {err:.3e}", flush=True)
    dp.close()
