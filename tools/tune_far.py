"""Far-field kernel tuning sweep (dev tool): times slb_farfield_stokes_sldl on a c4-sized
random problem for the variant selected by SLB_FAR_VARIANT.  Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_00889_b200 as S  # noqa: E402

T = int(os.environ.get("TUNE_T", 147456))
M = int(os.environ.get("TUNE_M", 983040))
kind = os.environ.get("TUNE_KIND", "sldl")
rng = np.random.default_rng(0)
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
x = cu(rng.uniform(0, 8, (T, 3)))
y = cu(rng.uniform(0, 8, (M, 3)))
n = rng.standard_normal((M, 3))
n = cu(n / np.linalg.norm(n, axis=1, keepdims=True))
w = cu(rng.uniform(1e-4, 2e-4, M))
sig = cu(rng.standard_normal((M, 3)))
eta = cu(rng.uniform(3, 4, M))
u = torch.empty((T, 3), dtype=torch.float64, device="cuda")
f = lambda: S.slb_farfield_stokes_sldl(x, y, n, w, sig, eta_src=cu_eta, out=u)
cu_eta = eta if kind == "sldl" else None
f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
tf = T * M * 39 / (ms * 1e-3) / 1e12
print(json.dumps({"variant": int(os.environ.get("SLB_FAR_VARIANT", 0)), "T": T, "M": M, "ms": ms,
                  "tflops": tf, "frac": tf / 37.22496, "gpairs": T * M / ms / 1e6}))
