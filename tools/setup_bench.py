"""Throughput of the setup steps and the solve around the operator (NEXT rows N1-N3) on one B200.

For each workload: GPU near-list build (N3, slb_near_build), special-quadrature correction
blocks (N1, slb_nearcorr_quad) by the paper's rule (order 0) and the round-1 generic 2-D rule (order 14),
with their accuracy against the CPU oracle on 24 sampled blocks, operator creation (packing + fold
E = B - G U), and a GMRES solve (N2, slb_gmres) of the CFIE with the special blocks.  Every
time is CUDA-event (device) time after one warm-up call; rates are in the paper's units
(unknowns per second of quadrature setup, P:L2315 / P:L2353 / P:L2527 / P:L2629).

usage: python tools/setup_bench.py [names...]   (default: torus torus_slender c2 c3 c3v) -> JSON lines
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2310_00889_b200 as S  # noqa: E402
from harness import DeviceProblem  # noqa: E402
from synth import make_config, make_torus_problem  # noqa: E402


def cu(a, dt=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)


def timed(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        out = fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def problem(name):
    if name == "torus":
        return make_torus_problem(rho=0.1, panels=16, kernel=2)
    if name == "torus_slender":
        return make_torus_problem(rho=1e-3, panels=24, Nt=8, kernel=2)
    return make_config(name)


def run(name):
    pr = problem(name)
    d = pr.sdim
    no = pr.node_off()
    cnt = np.diff(no)
    res = {"workload": name, "nodes": pr.N, "unknowns": pr.N * d, "panels": pr.P,
           "grid": [pr.Ns, pr.Nt] if not pr.ragged else "ragged (N_s, N_th)", "near_pairs": pr.nnz,
           "block_entries": pr.n_blocks_entries()}
    # N3: near lists on the GPU (2 L_k rule + own panel); ragged panels padded with their first node
    own_h = np.full(pr.T, -1, np.int64)
    own_h[:pr.n_on] = np.repeat(np.arange(pr.P), cnt)
    own = cu(own_h, torch.int64)
    j = np.arange(cnt.max())[None, :]
    ypad = pr.y_c[no[:-1, None] + np.where(j < cnt[:, None], j, 0)]
    x, y, rad = cu(pr.x_trg), cu(ypad), cu(2.0 * pr.panel_len)
    ms, (rp, pi) = timed(lambda: S.slb_near_build(x, y, rad, own))
    res["near_build_ms"] = ms
    res["near_build_target_panel_tests_per_s"] = pr.T * pr.P / (ms * 1e-3)
    # N1: special-quadrature blocks, two rule orders
    trg_node = cu(np.where(np.arange(pr.T) < pr.n_on, np.arange(pr.T), -1).astype(np.int64), torch.int64)
    eta_panel = cu(pr.eta_body[pr.body_of_panel]) if pr.kernel == 2 else None
    blocks = torch.empty(pr.n_blocks_entries(), dtype=torch.float64, device="cuda")
    rp_d, pi_d = cu(pr.row_ptr, torch.int64), cu(pr.panel_idx, torch.int32)
    rag = dict(panel_nt=pr.nt_of_panel(), panel_ns=pr.ns_of_panel()) if pr.ragged else {}
    # sampled pairs for the accuracy column: max |B - B_oracle| / max |B_oracle| per block
    import oracle as O
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(pr.nnz, min(24, pr.nnz), replace=False))
    bo = pr.blk_off()
    rows = np.searchsorted(pr.row_ptr, sample, side="right") - 1
    refs = []
    for p, t in zip(sample, rows):
        k = int(pr.panel_idx[p])
        nsk, ntk = int(pr.ns_of_panel()[k]), int(pr.nt_of_panel()[k])
        yk = pr.y_c[no[k]:no[k + 1]].reshape(nsk, ntk, 3)
        node = None
        if t < pr.n_on and no[k] <= t < no[k + 1]:
            node = ((t - no[k]) // ntk, (t - no[k]) % ntk)
        eta = float(pr.eta_body[pr.body_of_panel[k]]) if pr.kernel == 2 else 0.0
        refs.append(O.nearquad_block(pr.kernel, pr.x_trg[t], yk, eta=eta, node=node))
    for order, label in ((0, "paper_modal"), (14, "adaptive2d_q14")):
        ms, _ = timed(lambda: S.slb_nearcorr_quad(pr.kernel, x, rp_d, pi_d, pr.Ns, pr.Nt, cu(pr.y_c), blocks,
                                                  trg_node=trg_node, eta_panel=eta_panel, order=order, beta=0.6,
                                                  **rag))
        res[f"quad_{label}_ms"] = ms
        res[f"quad_{label}_unknowns_per_s"] = pr.N * d / (ms * 1e-3)
        res[f"quad_{label}_blocks_per_s"] = pr.nnz / (ms * 1e-3)
        bh = blocks.cpu().numpy()
        errs = [float(np.abs(bh[bo[p]:bo[p + 1]] - ref.reshape(-1)).max() / np.abs(ref).max())
                for p, ref in zip(sample, refs)]
        res[f"quad_{label}_max_rel_err_vs_oracle"] = max(errs)
    del blocks
    torch.cuda.empty_cache()
    # operator creation with the special blocks (fold included) and one apply
    quad = dict(order=0)
    t0 = time.perf_counter()
    dp = DeviceProblem(pr, quad=quad)
    torch.cuda.synchronize()
    res["operator_create_s_incl_quad"] = time.perf_counter() - t0
    ms, _ = timed(lambda: dp.matvec(), reps=5)
    res["matvec_ms"] = ms
    # N2: GMRES on the CFIE with a smooth right-hand side (a rigid translation field)
    rhs = cu(np.tile(np.array([1.0, 0.5, -0.25])[:d], (pr.T, 1)))
    t0 = time.perf_counter()
    xs, it, rr = dp.op.gmres(rhs, restart=100, max_iters=600, tol=1e-12)
    torch.cuda.synchronize()
    res["gmres_s"] = time.perf_counter() - t0
    res["gmres_iters"] = it
    res["gmres_rel_residual"] = rr
    res["gmres_ms_per_iter"] = res["gmres_s"] * 1e3 / max(it, 1)
    dp.close()
    return res


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["torus", "torus_slender", "c2", "c3", "c3v"]:
        print(json.dumps(run(nm)), flush=True)
