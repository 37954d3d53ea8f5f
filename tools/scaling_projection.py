"""Projected strong scaling of the operator apply from per-rank slices timed on ONE GPU.

The sharded operator does, per rank and apply: its own panels' upsample, one
in-place all-gather of the fine density (+ coarse sigma'), then far field and near correction
for its own target rows against ALL sources -- no other exchange.  Each rank's compute is
therefore an independent one-GPU job: the operator over that rank's target rows with all source
panels (harness.DeviceProblem(slice_only=True)).  This tool times every rank's slice for
N = 1, 2, 4, 8 on one B200 (CUDA events, 3 warm-up applies) and reports

    T_proj(N) = max_r T_slice(r, N) + T_gather(N),
    T_gather(N) = (N - 1)/N * gathered bytes / B_nvlink     (model; B_nvlink = 700 GB/s effective)

It is a PROJECTION (no multi-GPU box in this run): the bench's measured N-GPU number comes from
bench.py under torchrun.  The slice includes the full-size upsample (all panels; a rank upsamples
1/N of them) and omits the O(N) identity term -- both < 0.01 % of the apply.

usage: python tools/scaling_projection.py [config] [steps] > out.json
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from harness import DeviceProblem  # noqa: E402
from synth import make_config  # noqa: E402

B_NVLINK = 700e9


def time_slice(pr, rank, nranks, steps):
    dp = DeviceProblem(pr, rank=rank, nranks=nranks, slice_only=True)
    sig = torch.from_numpy(np.ascontiguousarray(pr.sigma.reshape(pr.N, pr.sdim))).cuda()
    for _ in range(3):
        u = dp.matvec(sig)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        dp.matvec(sig, out=u)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    rows = int(dp.rows.size)
    nnz = dp.nnz
    dp.close()
    del dp, u
    torch.cuda.empty_cache()
    return ms, rows, nnz


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    pr = make_config(name)
    gathered = pr.M * 4 * 8 + pr.N * pr.sdim * 8          # fine records {g, 0} + coarse sigma'
    out = {"config": name, "what": "projected strong scaling from per-rank slices timed on one B200",
           "gather_model": f"(N-1)/N x {gathered} B / {B_NVLINK / 1e9:.0f} GB/s", "N": {}}
    t1 = None
    for N in (1, 2, 4, 8):
        slices = [time_slice(pr, r, N, steps) for r in range(N)]
        ms = [s[0] for s in slices]
        tg = (N - 1) / N * gathered / B_NVLINK * 1e3
        tp = max(ms) + tg
        if N == 1:
            t1 = tp
        out["N"][N] = {"slice_ms": ms, "rows": [s[1] for s in slices], "nnz": [s[2] for s in slices],
                       "gather_ms_model": tg, "t_proj_ms": tp, "speedup": t1 / tp, "efficiency": t1 / tp / N}
        print(json.dumps({N: out["N"][N]}), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
