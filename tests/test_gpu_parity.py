"""GPU parity: every C-ABI step and the composed slb_matvec against the CPU oracle on the same
seeded inputs (relative max-norm <= 1e-12, north_star), plus bit-exact integer/byte work,
edge cases and determinism.  Runs on a B200 through libslb.so (-m gpu)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_config, pin_torus  # noqa: E402

TOL = 1e-12


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_00889_b200 as S
    S.slb_abi_version()
    return S


def cu(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


# ------------------------------------------------------------------ (a) upsample
@pytest.mark.parametrize("ns,nt,P,nc", [(10, 12, 8, 1), (10, 16, 7, 3), (12, 20, 5, 3), (10, 12, 1, 3),
                                        (5, 4, 3, 1), (10, 12, 300, 3)])
def test_upsample_parity(S, ns, nt, P, nc):
    rng = np.random.default_rng(ns * 100 + nt + P)
    sc = rng.standard_normal(P * ns * nt * nc)
    ms, mt = 2 * ns, 2 * nt
    g = S.slb_upsample(cu(sc), P, ns, nt, ms, mt, nc).cpu().numpy()
    ref = O.upsample(sc, P, ns, nt, ms, mt, nc).reshape(-1)
    assert rel(g, ref) <= TOL


def test_upsample_unequal_factors(S):
    rng = np.random.default_rng(3)
    sc = rng.standard_normal(4 * 10 * 12 * 3)
    g = S.slb_upsample(cu(sc), 4, 10, 12, 20, 12, 3).cpu().numpy()   # q = (2, 1)
    assert rel(g, O.upsample(sc, 4, 10, 12, 20, 12, 3).reshape(-1)) <= TOL


# ------------------------------------------------------------------ (b) far field
def _far_case(kind, T, M, seed, eta_mode="array", zero_normals=False):
    rng = np.random.default_rng(seed)
    b, g = pin_torus(P=max(1, M // 120 + 1), Ns=10, Nt=12)
    y, n, w = g.y[:M], g.n[:M], g.w[:M]
    if zero_normals:
        n = np.zeros_like(n)
    x = rng.uniform(-1.5, 1.5, (T, 3))
    d = 1 if kind == 1 else 3
    sig = rng.standard_normal((M, d)) if d == 3 else rng.standard_normal(M)
    eta = rng.uniform(1.0, 5.0, M)
    return x, y, n, w, sig, eta


@pytest.mark.parametrize("T,M", [(1160, 3840), (1, 1), (37, 257), (1000, 40000), (3000, 600000), (33, 0)])
def test_farfield_laplace_parity(S, T, M):
    x, y, n, w, sig, _ = _far_case(1, T, M, T + M)
    u = S.slb_farfield_laplace_dl(cu(x), cu(y.reshape(-1, 3)), cu(n.reshape(-1, 3)), cu(w), cu(sig)).cpu().numpy()
    if M == 0:
        assert np.all(u == 0)
        return
    ref = O.farfield(1, x, y, n, w, sig)
    assert rel(u, ref) <= TOL


@pytest.mark.parametrize("T,M,mode", [(513, 3840, "array"), (40, 20480, "scalar"), (700, 70001, "array"),
                                      (129, 5000, "dl"), (64, 2600, "sl"), (2000, 600000, "array")])
def test_farfield_stokes_parity(S, T, M, mode):
    x, y, n, w, sig, eta = _far_case(2, T, M, 7 * T + M, zero_normals=(mode == "sl"))
    args = dict(eta_src=cu(eta)) if mode in ("array", "sl") else dict(eta=(3.3 if mode == "scalar" else 0.0))
    u = S.slb_farfield_stokes_sldl(cu(x), cu(y), cu(n), cu(w), cu(sig), **args).cpu().numpy()
    eta_or = eta if mode in ("array", "sl") else np.full(M, 3.3 if mode == "scalar" else 0.0)
    ref = O.farfield(2, x, y, n, w, sig, eta=eta_or)
    assert rel(u, ref) <= TOL


def test_farfield_coincident_pairs_skipped_and_counted(S):
    b, g = pin_torus(P=4, Ns=6, Nt=8)
    rng = np.random.default_rng(5)
    sig = rng.standard_normal(g.y.shape)
    eta = np.full(g.w.size, 2.0)
    S.slb_coincident_reset()
    u = S.slb_farfield_stokes_sldl(cu(g.y), cu(g.y), cu(g.n), cu(g.w), cu(sig), eta_src=cu(eta)).cpu().numpy()
    assert S.slb_coincident_count() == g.w.size
    ref = O.farfield(2, g.y, g.y, g.n, g.w, sig, eta=eta)
    assert np.all(np.isfinite(u)) and rel(u, ref) <= TOL


def test_farfield_gauss_law_on_gpu(S):
    """The GPU far field reproduces Gauss's law (-1 inside, 0 outside) on the pin torus."""
    b, g = pin_torus()
    x = np.array([[1.0, 0, 0], [0, 1.05, 0], [0, 0, 0], [2.0, 0, 0]])
    u = S.slb_farfield_laplace_dl(cu(x), cu(g.y), cu(g.n), cu(g.w), cu(np.ones(g.w.size))).cpu().numpy()
    np.testing.assert_allclose(u, [-1, -1, 0, 0], atol=1e-13)


# ------------------------------------------------------------------ (c) near correction
def test_fill_blocks_bit_exact(S):
    for seed, first, count in [(12345, 0, 100003), (2**63 + 17, 10**12, 4097)]:
        g = torch.empty(count, dtype=torch.float64, device="cuda")
        S.slb_fill_blocks(seed, first, count, 1 / 120, g)
        ref = O.block_entries(seed, first, count, 1 / 120)
        assert np.array_equal(g.cpu().numpy().view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_nearcorr_apply_parity(S, name):
    pr = make_config(name)
    rng = np.random.default_rng(11)
    B = rng.standard_normal(pr.nnz * pr.block_len)
    u0 = rng.standard_normal(pr.T * pr.tdim)
    sig = pr.sigma.reshape(-1)
    u = cu(u0)
    S.slb_nearcorr_apply(cu(pr.row_ptr, torch.int64), cu(pr.panel_idx, torch.int32), cu(B), cu(sig), u,
                         pr.tdim, pr.sdim, pr.Nn)
    ref = O.nearcorr_apply(pr.T, pr.tdim, pr.sdim, pr.Nn, pr.row_ptr, pr.panel_idx, B, sig, u0)
    assert rel(u.cpu().numpy(), ref) <= TOL
    if name == "c1":
        assert np.any(np.diff(pr.row_ptr) == 0)   # empty rows covered


# ------------------------------------------------------------------ full operator
def _matvec_vs_oracle(S, pr, rows=None, fold=True):
    from harness import DeviceProblem
    dp = DeviceProblem(pr, fold=fold)
    u = dp.matvec().cpu().numpy().reshape(pr.T, pr.tdim)
    rows = np.arange(pr.T) if rows is None else rows
    ref = O.Oracle(pr).apply_rows(pr.sigma, rows)
    err = rel(u[rows], ref)
    u2 = dp.matvec().cpu().numpy().reshape(pr.T, pr.tdim)
    dp.close()
    return err, u, u2


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c2", {}), ("c4", dict(n_loops=4, panels=8)),
                                     ("c5", dict(n_loops=6, panels=9, box=6.0)), ("c3", dict(panels=16))])
def test_matvec_parity_small(S, name, kw):
    pr = make_config(name, **kw)
    err, u, u2 = _matvec_vs_oracle(S, pr)
    assert err <= TOL, err
    assert np.array_equal(u, u2)            # bitwise deterministic


def test_matvec_parity_c3_sampled(S):
    pr = make_config("c3")
    rng = np.random.default_rng(3)
    # worst near-gap targets (largest x on torus 0 / smallest on torus 1) + random rows
    gap = np.argsort(np.abs(pr.x_trg[:, 0] - 1.05125))[:64]
    rows = np.unique(np.concatenate([gap, rng.choice(pr.T, 448, replace=False)]))
    err, _, _ = _matvec_vs_oracle(S, pr, rows)
    assert err <= TOL, err


def test_matvec_unfolded_blocks_are_B(S):
    """Without folding, the apply uses B directly: u(fold=False) - u(fold=True) = smooth near part."""
    pr = make_config("c1")
    _, u_f, _ = _matvec_vs_oracle(S, pr, rows=np.arange(3), fold=True)
    orc = O.Oracle(pr)
    _, uf, un = orc.apply_rows(pr.sigma, np.arange(pr.T), parts=True)
    from harness import DeviceProblem
    dp = DeviceProblem(pr, fold=False)
    u_nf = dp.matvec().cpu().numpy().reshape(pr.T, 1)
    dp.close()
    nb = O.block_entries(pr.blk_seed, 0, pr.nnz * pr.block_len, pr.s_blk)
    bs = O.nearcorr_apply(pr.T, 1, 1, pr.Nn, pr.row_ptr, pr.panel_idx, nb, pr.sigma.reshape(-1), np.zeros(pr.T))
    smooth = bs - un[:, 0]
    assert rel((u_nf - u_f)[:, 0], smooth) <= 1e-11


def test_matvec_target_partition_bitwise(S):
    """Per-target sums do not depend on which targets share a launch (multi-GPU determinism):
    an operator over any subset of the targets returns bit-identical rows."""
    from harness import DeviceProblem
    from paper_2310_00889_b200 import Operator, slb_fill_blocks
    pr = make_config("c2")
    pr.c_identity = 0.0          # identity rows are rank-local by construction; compare the sums
    full = DeviceProblem(pr).matvec().cpu().numpy()
    blen = pr.block_len
    for lo, hi in ((0, 1234), (1234, 5120), (777, 778)):
        idx = np.arange(lo, hi)
        rp = np.concatenate([[0], np.cumsum(np.diff(pr.row_ptr)[idx])]).astype(np.int64)
        pidx = pr.panel_idx[pr.row_ptr[lo]:pr.row_ptr[hi]].astype(np.int32)
        a, b = pr.row_ptr[lo], pr.row_ptr[hi]
        blocks = torch.empty(int(b - a) * blen, dtype=torch.float64, device="cuda")
        slb_fill_blocks(pr.blk_seed, int(a) * blen, int(b - a) * blen, pr.s_blk, blocks)
        op = Operator(kernel=pr.kernel, ns=pr.Ns, nt=pr.Nt, ms=pr.Ms, mt=pr.Mt, n_panels_global=pr.P,
                      panel_begin=0, panel_end=pr.P, x_trg=cu(pr.x_trg[idx]), n_on=0, y_fine=cu(pr.y_f),
                      n_fine=cu(pr.n_f), w_fine=cu(pr.w_f), row_ptr=cu(rp, torch.int64),
                      panel_idx=cu(pidx, torch.int32), blocks=blocks, eta_fine=cu(pr.eta_f), c_identity=0.0)
        u = op.matvec(cu(pr.sigma)).cpu().numpy()
        assert np.array_equal(u, full[idx])
        op.close()


def test_matvec_host_variant(S):
    from harness import DeviceProblem
    pr = make_config("c2")
    dp = DeviceProblem(pr)
    ud = dp.matvec().cpu().numpy()
    sh = torch.from_numpy(pr.sigma.copy()).pin_memory()
    uh = torch.empty((pr.T, 3), dtype=torch.float64).pin_memory()
    dp.op.matvec_host(sh, uh)
    assert np.array_equal(uh.numpy(), ud)
    t = dp.op.timings()
    assert all(v >= 0 for v in t)
    dp.close()


def test_rigid_density_fixed_by_mobility_operator(S):
    from harness import DeviceProblem
    pr = make_config("c4", n_loops=3, panels=8)
    body = np.repeat(pr.body_of_panel, pr.Nn)
    rng = np.random.default_rng(1)
    v = np.zeros((pr.N, 3))
    for b in range(pr.n_bodies):
        m = body == b
        v[m] = rng.standard_normal(3) + np.cross(rng.standard_normal(3), pr.y_c[m])
    dp = DeviceProblem(pr)
    u = dp.matvec(cu(v)).cpu().numpy()
    np.testing.assert_allclose(u, v, atol=1e-12)
    dp.close()


# ------------------------------------------------------------------ full-size configs (sampled rows)
@pytest.mark.parametrize("name", ["c4", "c5"])
def test_matvec_parity_full_size_sampled(S, name):
    pr = make_config(name)
    rng = np.random.default_rng(99)
    nn = np.diff(pr.row_ptr)
    rows = np.unique(np.concatenate([rng.choice(pr.T, 96, replace=False), np.argsort(nn)[-16:],
                                     np.array([0, pr.T - 1])]))
    err, u, _ = _matvec_vs_oracle(S, pr, rows)
    assert err <= TOL, err


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c2", dict(panels=4)), ("c4", dict(n_loops=2, panels=8)),
                                     ("c5", dict(n_loops=3, panels=9, box=5.0))])
@pytest.mark.parametrize("path", ["const", "tma"])
def test_matvec_both_far_paths(S, name, kw, path, monkeypatch):
    """Both far-field engines (constant-bank tiles / TMA smem ring) on small problems, including
    fewer source tiles than constant buffers (c2 with 4 panels: 10240 sources = 52 tiles; c1)."""
    monkeypatch.setenv("SLB_FAR_PATH", path)
    pr = make_config(name, **kw)
    err, u, u2 = _matvec_vs_oracle(S, pr)
    assert err <= TOL, err
    assert np.array_equal(u, u2)


def test_const_path_fewer_tiles_than_buffers(S, monkeypatch):
    monkeypatch.setenv("SLB_FAR_PATH", "const")
    pr = make_config("c1", panels=1, n_extra=5)      # 1 panel: 480 fine sources = 3 tiles < 4 buffers
    err, u, _ = _matvec_vs_oracle(S, pr)
    assert err <= TOL, err


def test_const_path_coincident_pairs(S, monkeypatch):
    """r = 0 pairs on the constant-bank far path (R14): contribute 0, are counted, parity holds."""
    monkeypatch.setenv("SLB_FAR_PATH", "const")
    pr = make_config("c2", panels=4)
    pr.x_trg = pr.x_trg.copy()
    far_src = [int(np.argmax(np.linalg.norm(pr.y_f - pr.x_trg[t], axis=1))) for t in (7, 300)]
    pr.x_trg[7] = pr.y_f[far_src[0]]          # two targets moved onto far fine sources
    pr.x_trg[300] = pr.y_f[far_src[1]]
    S.slb_coincident_reset()
    err, u, u2 = _matvec_vs_oracle(S, pr)
    assert err <= TOL, err
    assert np.array_equal(u, u2)
    assert S.slb_coincident_count() >= 4      # 2 pairs x 2 applies (more if a moved target is near-listed)
    S.slb_coincident_reset()


def test_const_path_prescan_is_bitwise_neutral(S, monkeypatch):
    """Create-time coincident-pair prescan: without r = 0 pairs the applies use the unchecked far kernels;
    results are bit for bit those of the checked kernels (SLB_CONST_PRESCAN=0), and nothing is counted."""
    from harness import DeviceProblem
    monkeypatch.setenv("SLB_FAR_PATH", "const")
    pr = make_config("c4", n_loops=2, panels=8)
    out = {}
    S.slb_coincident_reset()
    for flag in ("1", "0"):
        monkeypatch.setenv("SLB_CONST_PRESCAN", flag)
        dp = DeviceProblem(pr)
        out[flag] = dp.matvec().cpu().numpy()
        dp.close()
    assert np.array_equal(out["1"], out["0"])
    assert S.slb_coincident_count() == 0


def test_operator_rejects_bad_csr(S):
    from paper_2310_00889_b200 import Operator, SlbError
    pr = make_config("c2", panels=4)
    rp = pr.row_ptr.copy()
    pi = pr.panel_idx.copy()
    pi[5] = pr.P + 3                          # panel id out of range
    blocks = torch.zeros(pr.nnz * pr.block_len, dtype=torch.float64, device="cuda")
    kw = dict(kernel=pr.kernel, ns=pr.Ns, nt=pr.Nt, ms=pr.Ms, mt=pr.Mt, n_panels_global=pr.P, panel_begin=0,
              panel_end=pr.P, x_trg=cu(pr.x_trg), n_on=pr.n_on, y_fine=cu(pr.y_f), n_fine=cu(pr.n_f),
              w_fine=cu(pr.w_f), blocks=blocks, eta_fine=cu(pr.eta_f))
    with pytest.raises(SlbError, match="panel_idx"):
        Operator(row_ptr=cu(rp, torch.int64), panel_idx=cu(pi, torch.int32), **kw)
    rp2 = rp.copy()
    rp2[10] = rp2[11] + 1                     # non-monotone
    with pytest.raises(SlbError, match="row_ptr"):
        Operator(row_ptr=cu(rp2, torch.int64), panel_idx=cu(pr.panel_idx, torch.int32), **kw)
    with pytest.raises(SlbError):
        S.slb_farfield_stokes_sldl(cu(pr.x_trg), cu(pr.y_f), cu(pr.n_f), cu(pr.w_f), cu(np.zeros((pr.M, 3))), eta=-1.0)


# ------------------------------------------------------------------ edge cases: limits, empty operators
@pytest.mark.parametrize("ns,nt,ms,mt", [(32, 64, 64, 128), (32, 2, 1, 2), (1, 2, 64, 128)])
def test_upsample_compiled_limits(S, ns, nt, ms, mt):
    """the largest grids the header allows (SLB_MAX_NS/NT/MS/MT) and degenerate 1-node / 2-angle
    panels: interpolation matrices beyond the kernel-parameter budget live in a device buffer"""
    rng = np.random.default_rng(ns + nt + ms)
    P, nc = 3, 3
    sc = rng.standard_normal(P * ns * nt * nc)
    g = S.slb_upsample(cu(sc), P, ns, nt, ms, mt, nc).cpu().numpy()
    assert rel(g, O.upsample(sc, P, ns, nt, ms, mt, nc).reshape(-1)) <= TOL


def test_upsample_beyond_limits_rejected(S):
    from paper_2310_00889_b200 import SlbError
    with pytest.raises(SlbError, match="UNSUPPORTED"):
        S.slb_upsample(cu(np.zeros(33 * 4)), 1, 33, 4, 66, 8, 1)


def test_operator_without_targets(S):
    """a rank may own sources but no targets (T_local = 0): the apply is a no-op that still runs"""
    from paper_2310_00889_b200 import Operator
    pr = make_config("c2", panels=4)
    op = Operator(kernel=pr.kernel, ns=pr.Ns, nt=pr.Nt, ms=pr.Ms, mt=pr.Mt, n_panels_global=pr.P, panel_begin=0,
                  panel_end=pr.P, x_trg=torch.zeros((0, 3), dtype=torch.float64, device="cuda"), n_on=0,
                  y_fine=cu(pr.y_f), n_fine=cu(pr.n_f), w_fine=cu(pr.w_f),
                  row_ptr=torch.zeros(1, dtype=torch.int64, device="cuda"),
                  panel_idx=torch.zeros(1, dtype=torch.int32, device="cuda"),
                  blocks=torch.zeros(2, dtype=torch.float64, device="cuda"), eta_fine=cu(pr.eta_f), c_identity=0.0)
    u = op.matvec(cu(pr.sigma))
    torch.cuda.synchronize()
    assert u.shape == (0, 3)
    op.close()


def test_zero_density_gives_zero(S):
    from harness import DeviceProblem
    pr = make_config("c4", n_loops=2, panels=6)
    dp = DeviceProblem(pr)
    u = dp.matvec(cu(np.zeros_like(pr.sigma))).cpu().numpy()
    dp.close()
    assert np.all(u == 0.0)


@pytest.mark.parametrize("nn", [12 * 32, 16 * 64])
def test_nearcorr_apply_wide_stokes_blocks(S, nn):
    """Wide Stokes blocks (12 x 32 and 16 x 64 panels: 27-74 KB per block) stream through the chunked
    ring in the stand-alone slb_nearcorr_apply (they used to return UNSUPPORTED)."""
    rng = np.random.default_rng(12)
    T, P = 37, 5
    cnt = rng.integers(0, 4, size=T)
    row_ptr = np.zeros(T + 1, np.int64)
    np.cumsum(cnt, out=row_ptr[1:])
    pidx = np.concatenate([np.sort(rng.choice(P, c, replace=False)) for c in cnt]).astype(np.int32)
    nnz = int(row_ptr[-1])
    B = rng.standard_normal(nnz * 3 * nn * 3)
    sig = rng.standard_normal(P * nn * 3)
    u0 = rng.standard_normal(T * 3)
    u = cu(u0)
    S.slb_nearcorr_apply(cu(row_ptr, torch.int64), cu(pidx, torch.int32), cu(B), cu(sig), u, 3, 3, nn)
    ref = O.nearcorr_apply(T, 3, 3, nn, row_ptr, pidx, B, sig, u0)
    assert rel(u.cpu().numpy(), ref) <= TOL
