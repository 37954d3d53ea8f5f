"""The NCCL path of slb_matvec on one GPU.

A one-rank communicator runs the same code as the multi-GPU operator: libslb dlopens NCCL,
the 128-byte id travels through torch.distributed, slb_operator_create all-gathers the panel
ranges and every apply runs the in-place ncclAllGather of the fine (and coarse) density.  With
one rank the gather is an identity, so the result must equal the communicator-free operator
bit for bit.  (Two ranks cannot share one GPU under NCCL; the multi-rank partition and layout
are covered on CPU by test_multirank_gloo.py.)
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c4", dict(n_loops=3, panels=6))])
def test_single_rank_nccl_operator_matches_plain(name, kw):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    from harness import DeviceProblem
    from paper_2310_00889_b200 import Comm
    from synth import make_config

    pr = make_config(name, **kw)
    plain = DeviceProblem(pr)
    u0 = plain.matvec().clone()
    plain.close()

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = Comm(1, 0)
        dp = DeviceProblem(pr, comm=comm)
        u1 = dp.matvec().clone()
        u2 = dp.matvec().clone()          # a second apply reuses the gathered buffers
        torch.cuda.synchronize()
        dp.close()
        comm.close()
    finally:
        dist.destroy_process_group()
    assert torch.equal(u0, u1)
    assert torch.equal(u1, u2)
    assert np.isfinite(u1.cpu().numpy()).all()
