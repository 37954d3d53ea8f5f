"""Resolution study for the sedimenting-ring check (PAPER.md Table t:conv-sbt):
runs tests/test_gpu_sedimentation.sedimentation_speed on the GPU and prints the error against
the paper's U_exact.

usage: python tools/ring_sedimentation.py rho:panels:Nt[:order] [...]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from test_gpu_sedimentation import golden, sedimentation_speed  # noqa: E402

if __name__ == "__main__":
    G = golden()
    for spec in sys.argv[1:] or ["0.1:16:12"]:
        f = spec.split(":")
        rho, P, Nt = float(f[0]), int(f[1]), int(f[2])
        order = int(f[3]) if len(f) > 3 else 14
        t0 = time.time()
        V, it, rr, pr = sedimentation_speed(rho, P, Nt=Nt, order=order)
        U = -float(np.average(V[:, 2], weights=pr.w_c))
        ex = G[rho]
        print(f"rho={rho:g} P={P} Nt={Nt} order={order} N={pr.N} it={it} rr={rr:.1e} U={U:.15e} "
              f"exact={ex:.15e} rel.err={abs(U - ex) / ex:.2e} rot/trans={np.abs(V[:, :2]).max() / abs(V[:, 2]).max():.1e} "
              f"({time.time() - t0:.1f}s)", flush=True)
