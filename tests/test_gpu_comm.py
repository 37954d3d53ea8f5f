"""The NCCL data plane of slb_matvec / slb_gmres, executed on one GPU.

A one-rank communicator runs every collective the multi-GPU operator runs -- no `nranks == 1`
short-circuit remains in libslb: the create-time ncclAllGather of the rank panel ranges, the two
in-place ncclAllGathers per apply (fine source records, coarse density), the grouped in-place
ncclBroadcasts that replace them for unequal shards (forced here with SLB_FORCE_GROUPED_GATHER=1),
and the ncclAllReduce of the GMRES dot products.  With one rank each collective is an identity,
so results must equal the communicator-free operator bit for bit.  Evidence that the calls really
went through NCCL: libslb's own per-communicator call counts, and NCCL's INFO log of the
collectives (NCCL_DEBUG=INFO, NCCL_DEBUG_SUBSYS=COLL), which names each AllGather / Broadcast /
AllReduce.  (Two NCCL ranks cannot share one GPU; the multi-rank partition and layout arithmetic
is covered on CPU by test_multirank_gloo.py.)
"""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(tmp_path, grouped, nvls=False):
    log = tmp_path / f"nccl_{'grouped' if grouped else 'equal'}.%h.%p.log"
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="COLL", NCCL_DEBUG_FILE=str(log),
               SLB_FORCE_GROUPED_GATHER="1" if grouped else "0", SLB_NVLS="1" if nvls else "0")
    r = subprocess.run([sys.executable, os.path.join(HERE, "nccl_one_rank.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")][-1]
    res = json.loads(line[len("RESULT "):])
    res["stderr"] = r.stderr[-2000:]
    text = "".join(p.read_text(errors="replace") for p in tmp_path.glob(f"nccl_{'grouped' if grouped else 'equal'}.*"))
    return res, text


@pytest.mark.parametrize("grouped", [False, True], ids=["allgather", "grouped_broadcast"])
def test_one_rank_nccl_collectives_bitwise(tmp_path, grouped):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    res, log = _run(tmp_path, grouped)
    for name, r in res["cases"].items():
        assert r["equal_first"] and r["equal_second"] and r["finite"], (name, r)
        # create: the panel-range gather (always an AllGather)
        assert r["create"]["allgather"] == 1, (name, r)
        # two applies: fine records + coarse density per apply
        if grouped:
            assert r["two_applies"]["broadcast"] == 4 and r["two_applies"]["allgather"] == 0, (name, r)
        else:
            assert r["two_applies"]["allgather"] == 4 and r["two_applies"]["broadcast"] == 0, (name, r)
        if "gmres" in r:
            g = r["gmres"]
            assert g["equal"], (name, g)
            assert g["collectives"]["allreduce"] >= g["iters"][1] > 0, (name, g)
    # NCCL's own log of the calls
    assert "AllGather" in log, log[-2000:]
    assert "AllReduce" in log, log[-2000:]
    if grouped:
        assert "Broadcast" in log, log[-2000:]


def test_one_rank_fused_multicast_gather_bitwise(tmp_path):
    """(NEXT N4) SLB_NVLS=1: the fine records live in a one-device multicast object and the upsample
    epilogue writes them with multimem.st (the switch-replicated store); the per-apply all-gather of the
    records is gone (only the coarse-density gather remains: 2 AllGathers for two applies, not 4), and
    every result equals the communicator-free operator bit for bit.  Multi-rank replication itself needs
    an NVSwitch box with several GPUs (N4)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    res, _ = _run(tmp_path, False, nvls=True)
    if not res["nvls_supported"]:
        # e.g. this pool's boxes: the attribute says supported but cuMulticastCreate returns
        # CUDA_ERROR_INVALID_VALUE for every team size / handle type (tools/nvls_probe.py)
        pytest.skip("multicast objects cannot be created on this device (see tools/nvls_probe.py)")
    for name, r in res["cases"].items():
        assert r["nvls"], (name, r, res["stderr"])
        assert r["equal_first"] and r["equal_second"] and r["finite"], (name, r)
        assert r["two_applies"]["allgather"] == 2 and r["two_applies"]["broadcast"] == 0, (name, r)
        if "gmres" in r:
            assert r["gmres"]["equal"], (name, r["gmres"])
