"""Helper for test_gpu_comm.py (run in a subprocess so NCCL_DEBUG / SLB_FORCE_GROUPED_GATHER take
effect before NCCL and libslb read them).

One process, one GPU, a one-rank NCCL communicator: builds the communicator-free operator and the
communicator operator for a few configs, applies both, runs GMRES through both, and prints one JSON
line with the bitwise comparisons and the collective counts libslb reports."""
import json
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [("c1", {}), ("c4", dict(n_loops=3, panels=6)), ("c3v", dict(panels=8)),
         ("c2", dict(panels=8))]


def main():
    from harness import DeviceProblem
    from paper_2310_00889_b200 import Comm
    from synth import make_config

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    comm = Comm(1, 0)
    from paper_2310_00889_b200._native import lib
    res = {"cases": {}, "nvls_supported": bool(lib().slb_nvls_supported())}
    for name, kw in CASES:
        pr = make_config(name, **kw)
        plain = DeviceProblem(pr)
        u0 = plain.matvec().clone()
        c0 = comm.collective_counts()
        dp = DeviceProblem(pr, comm=comm)
        c1 = comm.collective_counts()
        u1 = dp.matvec().clone()
        u2 = dp.matvec().clone()
        torch.cuda.synchronize()
        c2 = comm.collective_counts()
        r = {"equal_first": bool(torch.equal(u0, u1)), "equal_second": bool(torch.equal(u1, u2)),
             "finite": bool(torch.isfinite(u1).all()),
             "create": {k: c1[k] - c0[k] for k in c0}, "two_applies": {k: c2[k] - c1[k] for k in c1},
             "nvls": dp.op.uses_nvls()}
        if pr.T == pr.n_on:                                      # square: GMRES through both
            rng = np.random.default_rng(3)
            b = torch.from_numpy(rng.standard_normal(pr.sigma.shape)).cuda()
            xa, ita, rra = plain.op.gmres(b.clone(), restart=30, max_iters=60, tol=1e-12)
            c3 = comm.collective_counts()
            xb, itb, rrb = dp.op.gmres(b.clone(), restart=30, max_iters=60, tol=1e-12)
            c4 = comm.collective_counts()
            r["gmres"] = {"iters": [ita, itb], "equal": bool(torch.equal(xa, xb)) and ita == itb and rra == rrb,
                          "collectives": {k: c4[k] - c3[k] for k in c3}}
        res["cases"][name] = r
        dp.close()
        plain.close()
    comm.close()
    dist.destroy_process_group()
    print("RESULT " + json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
