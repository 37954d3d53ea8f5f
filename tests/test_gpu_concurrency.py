"""SURVEY §8(b) concurrency contract: distinct operators may be applied concurrently.

The large-M far field stages source tiles in the device's one __constant__ bank; libslb
serialises every user of the bank (host lock + device event chain, slb.h "Concurrency").  Two
DIFFERENT operators on that path (forced with SLB_FAR_PATH=const at creation) are applied
(i) interleaved on two streams from one thread and (ii) from two host threads on their own
streams; every result must be bitwise equal to the sequential apply."""
import os
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ops():
    from harness import DeviceProblem
    from synth import make_config
    old = os.environ.get("SLB_FAR_PATH")
    os.environ["SLB_FAR_PATH"] = "const"
    try:
        a = DeviceProblem(make_config("c4", n_loops=8, panels=16))      # mobility, M = 61,440
        b = DeviceProblem(make_config("c3", panels=24))                 # two close tori, M = 46,080
    finally:
        if old is None:
            del os.environ["SLB_FAR_PATH"]
        else:
            os.environ["SLB_FAR_PATH"] = old
    return a, b


def test_two_operators_two_streams_bitwise():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a, b = _ops()
    ua = a.matvec().clone()
    ub = b.matvec().clone()
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs_a = [torch.empty_like(ua) for _ in range(6)]
    outs_b = [torch.empty_like(ub) for _ in range(6)]
    torch.cuda.synchronize()
    for i in range(6):
        with torch.cuda.stream(s1):
            a.matvec(out=outs_a[i])
        with torch.cuda.stream(s2):
            b.matvec(out=outs_b[i])
    torch.cuda.synchronize()
    for i in range(6):
        assert torch.equal(outs_a[i], ua), i
        assert torch.equal(outs_b[i], ub), i
    a.close()
    b.close()


def test_two_operators_two_threads_bitwise():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a, b = _ops()
    ua = a.matvec().clone()
    ub = b.matvec().clone()
    torch.cuda.synchronize()
    errs, res = [], {}

    def work(dp, key, n):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            outs = []
            with torch.cuda.stream(s):
                for _ in range(n):
                    outs.append(dp.matvec().clone())
            s.synchronize()
            res[key] = outs
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    ts = [threading.Thread(target=work, args=(a, "a", 5)), threading.Thread(target=work, args=(b, "b", 5))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    assert all(torch.equal(u, ua) for u in res["a"])
    assert all(torch.equal(u, ub) for u in res["b"])
    assert np.isfinite(ua.cpu().numpy()).all() and np.isfinite(ub.cpu().numpy()).all()
    a.close()
    b.close()
