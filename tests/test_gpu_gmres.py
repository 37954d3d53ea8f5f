"""(NEXT N2) GMRES around slb_matvec: manufactured solutions whose right-hand sides come from
the CPU oracle's operator, so the GPU solve is checked against the oracle (not against itself)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_config  # noqa: E402


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.float64)


@pytest.mark.parametrize("name,kw", [("c1", dict(n_extra=0)), ("c2", dict(panels=8)),
                                     ("c4", dict(n_loops=2, panels=6)), ("c3", dict(panels=6))])
def test_gmres_manufactured_solution(name, kw):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from harness import DeviceProblem
    pr = make_config(name, **kw)
    rng = np.random.default_rng(5)
    xs = rng.standard_normal(pr.sigma.shape)
    b = O.Oracle(pr).apply_rows(xs, np.arange(pr.T)).reshape(pr.sigma.shape)   # b = A x* (oracle)
    dp = DeviceProblem(pr)
    x, it, rr = dp.op.gmres(cu(b), restart=60, max_iters=2000, tol=1e-13)
    x = x.cpu().numpy()
    assert rr <= 1e-13, (it, rr)
    err = np.abs(x - xs).max() / np.abs(xs).max()
    assert err <= 1e-9, (err, it)
    # reproducible
    x2, it2, rr2 = dp.op.gmres(cu(b), restart=60, max_iters=2000, tol=1e-13)
    assert it2 == it and np.array_equal(x2.cpu().numpy(), x)
    dp.close()


def test_gmres_zero_rhs_and_exact_guess():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from harness import DeviceProblem
    pr = make_config("c2", panels=4)
    dp = DeviceProblem(pr)
    x, it, rr = dp.op.gmres(cu(np.zeros(pr.sigma.shape)))
    assert it == 0 and rr == 0 and float(x.abs().max()) == 0.0
    b = dp.matvec(cu(pr.sigma))
    x, it, rr = dp.op.gmres(b.clone(), x0=cu(pr.sigma), tol=1e-10)
    assert it == 0 and rr <= 1e-10
    dp.close()
