"""Near-list build time (N3) on the GPU: the Morton-sorted search (default) vs the O(T P) all-panel scan
(SLB_NEAR_SCAN=1), R15 radius 2 L_k, own panels; prints one JSON line per config.
usage: python tools/nearlist_bench.py c5 [c5alt ...]   (set SLB_NEAR_SCAN=1 in the environment for the scan)"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_00889_b200 import slb_near_build  # noqa: E402
from synth import make_config  # noqa: E402

for name in sys.argv[1:]:
    pr = make_config(name)
    cu = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
    x, y, r = cu(pr.x_trg), cu(pr.y_c.reshape(pr.P, pr.Nn, 3)), cu(2.0 * pr.panel_len)
    own = cu(np.repeat(np.arange(pr.P), pr.Nn).astype(np.int64), torch.int64)
    slb_near_build(x, y, r, own)                            # warm-up (module load, allocator)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        rp, pi = slb_near_build(x, y, r, own)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ok = np.array_equal(rp.cpu().numpy(), pr.row_ptr) and np.array_equal(pi.cpu().numpy(), pr.panel_idx)
    print(json.dumps({"config": name, "method": "scan" if os.environ.get("SLB_NEAR_SCAN") == "1" else "morton",
                      "targets": pr.T, "panels": pr.P, "nnz": int(pi.numel()), "seconds_min": min(ts),
                      "bit_exact_vs_generator": bool(ok)}), flush=True)
