"""(NEXT N3) GPU near-list construction vs the input generator's CPU rule (R15):
integer output, so the CSR must match bit for bit on every config."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import make_config  # noqa: E402


def cu(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c2", {}), ("c3", {}), ("c4", {}), ("c5", dict(n_loops=64, box=8.0)),
                                     ("c5", {})])
def test_near_build_matches_generator(name, kw):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_00889_b200 import slb_near_build
    pr = make_config(name, **kw)
    radius = cu(2.0 * pr.panel_len)
    y = cu(pr.y_c.reshape(pr.P, pr.Nn, 3))
    if name == "c1":   # node targets follow the forced {k-1,k,k+1} rule; compare the off-surface rows
        rows = np.arange(pr.n_on, pr.T)
        own = None
    else:
        rows = np.arange(pr.T)
        own = cu(np.repeat(np.arange(pr.P), pr.Nn).astype(np.int64), torch.int64)
    rp, pi = slb_near_build(cu(pr.x_trg[rows]), y, radius, own)
    rp, pi = rp.cpu().numpy(), pi.cpu().numpy()
    ref_rp = pr.row_ptr[rows[0]:rows[-1] + 2] - pr.row_ptr[rows[0]]
    ref_pi = pr.panel_idx[pr.row_ptr[rows[0]]:pr.row_ptr[rows[-1] + 1]]
    assert np.array_equal(rp, ref_rp)
    assert np.array_equal(pi, ref_pi)


def test_near_build_edge_cases():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_00889_b200 import slb_near_build
    y = cu(np.random.default_rng(0).standard_normal((3, 4, 3)))
    # no targets
    rp, pi = slb_near_build(cu(np.zeros((0, 3))), y, cu(np.ones(3)))
    assert rp.cpu().tolist() == [0] and pi.numel() == 0
    # far target: empty row; own panel forced even when far
    x = cu(np.array([[100.0, 0, 0], [100.0, 0, 0]]))
    rp, pi = slb_near_build(x, y, cu(np.ones(3)), cu(np.array([-1, 2]), torch.int64))
    assert rp.cpu().tolist() == [0, 0, 1] and pi.cpu().tolist() == [2]


def test_near_build_ragged_by_padding():
    """ragged panels (N4, c3v): pad each panel's nodes to the widest panel with copies of its first
    node (the min over nodes is unchanged) -- bit-exact against the generator's CSR"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_00889_b200 import slb_near_build
    pr = make_config("c3v", panels=16)
    no = pr.node_off()
    cnt = np.diff(no)
    j = np.arange(cnt.max())[None, :]
    idx = no[:-1, None] + np.where(j < cnt[:, None], j, 0)
    own = np.repeat(np.arange(pr.P), cnt).astype(np.int64)
    rp, pi = slb_near_build(cu(pr.x_trg), cu(pr.y_c[idx]), cu(2.0 * pr.panel_len), cu(own, torch.int64))
    assert np.array_equal(rp.cpu().numpy(), pr.row_ptr)
    assert np.array_equal(pi.cpu().numpy(), pr.panel_idx)


@pytest.mark.parametrize("frac", [0.25, 3.0])
def test_near_build_other_radius_rule_vs_brute_force(frac):
    """the Morton search is rule-independent: a different per-element radius (frac * L_k, e.g. a
    tolerance-based near region) against a plain CPU brute force of the same predicate
    sqrt(min_j ((dx^2 + dy^2) + dz^2)) < r_k, bit for bit, plus extra targets far outside the nodes' box"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_00889_b200 import slb_near_build
    pr = make_config("c4", n_loops=6, panels=8)
    rng = np.random.default_rng(4)
    r = frac * pr.panel_len * rng.uniform(0.5, 1.5, pr.P)
    x = np.concatenate([pr.x_trg, rng.uniform(-3, 11, size=(500, 3))])
    own = np.concatenate([np.repeat(np.arange(pr.P), pr.Nn), -np.ones(500, np.int64)]).astype(np.int64)
    Y = pr.y_c.reshape(pr.P, pr.Nn, 3)
    rp, pi = slb_near_build(cu(x), cu(Y), cu(r), cu(own, torch.int64))
    rp, pi = rp.cpu().numpy(), pi.cpu().numpy()
    for t in range(0, x.shape[0], 7):                       # every 7th row (brute force is O(P Nn) per row)
        d = x[t][None, None, :] - Y
        m = np.sqrt(np.min((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2], axis=1))
        ks = set(np.nonzero(m < r)[0].tolist())
        if own[t] >= 0:
            ks.add(int(own[t]))
        assert pi[rp[t]:rp[t + 1]].tolist() == sorted(ks), t
