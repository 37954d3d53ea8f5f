"""slb_operator_prepare (apply stage 1 alone: projector + upsample into the fine records), the call bench.py
times for the upsample roofline.  It must launch exactly the stage-1 kernels and leave the operator valid:
any number of prepares followed by an apply gives the same result, bit for bit, as the apply alone."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("spec", [("c1", {}), ("c4", {"n_loops": 4, "panels": 8}), ("c3v", {})])
def test_prepare_then_apply_bitwise(spec):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_00889_b200 as S
    from harness import DeviceProblem
    from synth import make_config
    name, kw = spec
    dp = DeviceProblem(make_config(name, **kw))
    u_ref = dp.matvec().clone()
    n0 = S.slb_launch_count()
    for _ in range(3):
        dp.op.prepare(dp.sigma)
    torch.cuda.synchronize()
    per_prepare = (S.slb_launch_count() - n0) / 3
    assert per_prepare >= 1
    assert per_prepare < dp.op.launches_per_matvec()          # no gather, far field or finalize
    # a different density through prepare, then the apply of the original: the apply redoes stage 1
    dp.op.prepare(torch.randn_like(dp.sigma))
    u = dp.matvec()
    torch.cuda.synchronize()
    assert torch.equal(u, u_ref), (name, float((u - u_ref).abs().max()))
    dp.close()
