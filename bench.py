"""Benchmark of the slender-body Nystrom operator apply (arXiv 2310.00889) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

A step is one full operator apply (slb_matvec): projector (mobility configs), upsample, NCCL
all-gather (N > 1), far field, folded near correction, identity term.  Default workload: config
5 (512 loops, the config the north_star's throughput and scaling targets are quoted on).
N > 1: launched by torchrun, one rank per GPU, panels/targets sharded, strong scaling.
Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (the reference arm of
this tier) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 BIE matvecs/s & G pair-interactions/s; % of FP64 peak / HBM BW"
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12     # derived: SMs x FP64 FMA lanes x 2 x max SM clock
FLOPS_PER_PAIR = {1: 20, 2: 39}                        # algorithmic, FMA = 2


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def setup_dist(args):
    """World from torchrun's env.  `--gpus N` (N > 1) without WORLD_SIZE re-launches this script
    under torch.distributed.run with N ranks (one per GPU); fewer visible GPUs than N is an error."""
    if "WORLD_SIZE" not in os.environ:
        n = args.gpus if args.gpus is not None else 1
        if n > 1:
            if args.impl == "ours":
                import torch
                have = torch.cuda.device_count()
                if have < n:
                    sys.stderr.write(f"bench.py: --gpus {n} requested but only {have} CUDA device(s) are visible\n")
                    sys.exit(2)
            import socket
            so = socket.socket()
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
            so.close()
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                   "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
            sys.stdout.flush()
            os.execv(sys.executable, cmd)
        return 1, 0, 0
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus is not None and args.gpus != world:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    if args.impl == "ours":
        import torch
        if torch.cuda.device_count() <= local:
            sys.stderr.write(f"bench.py: rank {rank} (LOCAL_RANK {local}) has no GPU: "
                             f"{torch.cuda.device_count()} visible\n")
            sys.exit(2)
    return world, rank, local


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline_run(pr, seconds_target=15.0, rows_n=None, gpu_u=None):
    """Time the oracle as it stands on a bounded row sample; extrapolate to one full apply.
    gpu_u (the GPU apply's output for all T rows, N = 1): also compare the sampled rows with it --
    the bench's parity number comes from this leg, the one place bench.py runs the oracle."""
    import oracle
    thr = oracle.num_threads()
    orc = oracle.Oracle(pr)
    t0 = time.perf_counter()
    prep = orc.prepare(pr.sigma)
    t_prep = time.perf_counter() - t0
    rng = np.random.default_rng(7)
    if rows_n is None:
        # calibrate on a few rows, then size the sample to ~seconds_target
        probe = rng.choice(pr.T, min(pr.T, max(4, thr)), replace=False)
        t0 = time.perf_counter()
        orc.apply_rows(pr.sigma, probe, prepared=prep)
        per = (time.perf_counter() - t0) / probe.size
        rows_n = int(min(pr.T, max(thr, seconds_target / max(per, 1e-9))))
    rows = np.sort(rng.choice(pr.T, rows_n, replace=False))
    t0 = time.perf_counter()
    ref = orc.apply_rows(pr.sigma, rows, prepared=prep)
    t_rows = time.perf_counter() - t0
    t_full = t_prep + t_rows * pr.T / rows.size
    parity = None
    if gpu_u is not None:
        got = np.asarray(gpu_u).reshape(pr.T, -1)[rows]
        parity = float(np.abs(got - ref.reshape(got.shape)).max() / np.abs(ref).max())
    return {"value": 1.0 / t_full, "parity_rows": int(rows.size), "parity_rel_err": parity, "unit": "matvec/s", "cores": thr, "kind": "oracle", "cpu_model": _cpu_model(),
            "nproc": os.cpu_count(),
            "sample": (f"{rows.size} of {pr.T} target rows of {pr.name} (full operator per row: far sum over "
                       f"{pr.M} fine sources + literal near correction + identity), plus the O(N) "
                       f"prepare (projector/upsample, {t_prep:.2f}s); extrapolated linearly in T"),
            "seconds": t_prep + t_rows, "pairs_per_s": pr.pairs() / t_full}


def l2_note(pr):
    """Timing rule: inputs larger than L2 between timed iterations (stated per workload; identical in
    both arms' config)."""
    big = pr.M * 80 + pr.n_blocks_entries() * 8
    return (f"inputs larger than L2 (fine sources {pr.M * 80 / 1e6:.0f} MB, near blocks "
            f"{pr.n_blocks_entries() * 8 / 1e9:.1f} GB)" if big > 126e6 else
            f"inputs {big / 1e6:.1f} MB < 126 MB L2: L2-resident between applies (small config)")


def config_info(pr, world):
    return {"workload": pr.name, "kernel": "laplace_dl" if pr.kernel == 1 else "stokes_sl+dl",
            "operator": "K(I-L)+L mobility" if pr.projector else ("I/2 + D" if pr.kernel == 1 else "I/2 + D + eta S"),
            "bodies": pr.n_bodies, "panels": pr.P,
            "coarse_grid": [pr.Ns, pr.Nt] if not pr.ragged else
            [pr.Ns, {int(k): int(v) for k, v in zip(*np.unique(pr.panel_nt, return_counts=True))}],
            "fine_grid": [pr.Ms, pr.Mt] if not pr.ragged else [pr.Ms, f"{pr.Mt // pr.Nt} x N_th per panel"],
            "nodes": pr.N, "unknowns": pr.N * pr.sdim, "fine_sources": pr.M, "targets": pr.T,
            "pairs_per_apply": pr.pairs(), "near_blocks": pr.nnz,
            "block_shape": [pr.tdim, pr.Nn * pr.sdim] if not pr.ragged else [pr.tdim, "N_n^(k) s_dim (ragged)"],
            "parallelism": f"targets sharded over {world} GPU(s), all-gather of fine density",
            "l2": l2_note(pr), "seed": pr.seed}


def run_reference(args, world, rank):
    from synth import make_config
    if rank != 0:
        return
    pr = make_config(args.config)
    vals = []
    res = None
    for i in range(args.warmup + args.steps):
        res = cpu_baseline_run(pr, seconds_target=args.ref_seconds, rows_n=None if i == 0 else res_rows)
        res_rows = int(res["sample"].split(" of ")[0])
        if i >= args.warmup:
            vals.append(res["value"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "matvec/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_info(pr, world),
            "cpu_baseline": {"value": v, "unit": "matvec/s", "cores": res["cores"], "kind": "oracle",
                             "sample": res["sample"], "cpu_model": res.get("cpu_model"), "nproc": res.get("nproc")},
            "e2e": {"value": v, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("SLB_BENCH_CONFIG", "c5"))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    args = ap.parse_args()
    world, rank, local = setup_dist(args)
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    from synth import make_config
    from harness import DeviceProblem
    import paper_2310_00889_b200 as S

    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = S.Comm(world, rank)
    t_setup = time.perf_counter()
    pr = make_config(args.config)
    t_gen = time.perf_counter() - t_setup
    dp = DeviceProblem(pr, rank=rank, nranks=world, comm=comm)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        u = dp.matvec()
    barrier()
    u = torch.empty((dp.rows.size, pr.tdim), dtype=torch.float64, device="cuda")
    n_launch0 = S.slb_launch_count()
    stage = []
    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local]
                    if os.environ.get("CUDA_VISIBLE_DEVICES") else local)
    with ClockSampler(gpu_index) as clk:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            dp.matvec(out=u)
            stage.append(dp.op.timings())      # stage events on the launching stream (syncs the step)
        e1.record(stream)
        barrier()
    n_launch = S.slb_launch_count() - n_launch0
    ms = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    st = np.array(stage)                        # [K][4] ms: prep+upsample, allgather, far, finalize
    st_mean = st.mean(0)
    far_ms = st_mean[2]
    fin_ms = st_mean[3]

    # the upsample (+projector) kernels alone: K back-to-back launches of apply stage 1 (slb_operator_prepare),
    # CUDA events on the launching stream -- the kernels' own duration, without the in-apply stage events' launch
    # gap (stage_ms keeps the in-apply figure)
    barrier()
    k_up = 50
    u0 = torch.cuda.Event(enable_timing=True)
    u1 = torch.cuda.Event(enable_timing=True)
    dp.op.prepare(dp.sigma)
    u0.record(stream)
    for _ in range(k_up):
        dp.op.prepare(dp.sigma)
    u1.record(stream)
    barrier()
    up_kernel_ms = u0.elapsed_time(u1) / k_up

    # e2e through the public API with host buffers (H2D sigma, D2H u inside the timed region)
    no, fo = pr.node_off(), pr.fine_off()
    sig_h = torch.from_numpy(pr.sigma.reshape(pr.N, pr.sdim)[no[dp.pb]:no[dp.pe]].copy()).pin_memory()
    u_h = torch.empty((dp.rows.size, pr.tdim), dtype=torch.float64).pin_memory()
    e2e_steps = max(1, min(args.steps, 5))
    barrier()
    h0 = torch.cuda.Event(enable_timing=True)
    h1 = torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for _ in range(e2e_steps):
        dp.op.matvec_host(sig_h, u_h)
    h1.record(stream)
    barrier()
    e2e_ms = torch.tensor([h0.elapsed_time(h1) / e2e_steps], dtype=torch.float64, device="cuda")
    h2d = torch.tensor([sig_h.numel() * 8, u_h.numel() * 8], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(h2d)
    # roofline quantities per rank -> report rank 0's (targets are balanced)
    T_loc = dp.rows.size
    far_flops = T_loc * pr.M * FLOPS_PER_PAIR[pr.kernel]
    near_bytes = dp.n_entries * 8 + dp.nnz * 4 + T_loc * 8 * (pr.tdim + 2)
    n_loc_nodes = int(no[dp.pe] - no[dp.pb])
    m_loc = int(fo[dp.pe] - fo[dp.pb])
    # upsample (+projector) algorithmic bytes: the coarse density read once (+ the projector's second read
    # and its sigma', L sigma writes), the fine-node scales read (1 double per node Stokes, 4 Laplace), the
    # 32-byte source records written
    up_bytes = (n_loc_nodes * pr.sdim * 8 * (1 + (3 if pr.projector else 0)) + m_loc * 8 * (4 if pr.kernel == 1 else 1)
                + m_loc * 32)
    dfma = None
    if rank == 0:
        try:
            dfma = S.slb_bench_dfma(200000) / 1e3
        except Exception:
            dfma = None
    cpu_base = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_base = cpu_baseline_run(pr, seconds_target=args.ref_seconds, gpu_u=u.cpu().numpy())
        parity = {"rel_err": cpu_base.pop("parity_rel_err"), "rows": cpu_base.pop("parity_rows"),
                  "against": "CPU oracle on the cpu_baseline row sample"}
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"traffic_{pr.name}.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("far_kernel_dram_bytes_per_launch")
        except Exception:
            traffic = None
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    clocks = clk.summary()
    if rank == 0:
        far_tf = far_flops / (far_ms * 1e-3) / 1e12
        near_gbs = near_bytes / (fin_ms * 1e-3) / 1e9
        value = 1e3 / ms_max
        line = {
            "metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_info(pr, world),
            "pairs_per_s": pr.pairs() * value,
            "roofline": {"bound": "alu", "kernel": "far_const_kernel (FP64 DFMA pipe; far_kernel below M = 2^16)", "achieved": far_tf,
                         "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": far_tf / FP64_PEAK_TFLOPS,
                         "traffic": traffic,
                         "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1965 MHz (no FP64 entry in "
                                        "MEASURED_PEAKS.json)",
                         "dfma_microbench_tflops": dfma,
                         "frac_of_dfma_microbench": (far_tf / dfma) if dfma else None,
                         "flops_per_pair": FLOPS_PER_PAIR[pr.kernel], "launch_ms": far_ms,
                         "share_of_step": far_ms / ms},
            "roofline_near": {"bound": "hbm", "kernel": "finalize_kernel (near blocks + chunk reduce)",
                              "achieved": near_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": near_gbs / hbm_peak,
                              "bytes_per_launch": near_bytes, "launch_ms": fin_ms},
            "roofline_upsample": {"bound": "hbm", "kernel": "upsample_rec_kernel / upsample_warp_kernel (+ projector; DMMA m8n8k4, TMA-fed)",
                                  "achieved": up_bytes / (up_kernel_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                                  "frac": up_bytes / (up_kernel_ms * 1e-3) / 1e9 / hbm_peak,
                                  "bytes_per_launch": up_bytes, "launch_ms": up_kernel_ms,
                                  "timing": "50 back-to-back launches of apply stage 1 (slb_operator_prepare), CUDA events",
                                  "in_apply_stage_ms": st_mean[0],
                                  "frac_in_apply_stage": up_bytes / (st_mean[0] * 1e-3) / 1e9 / hbm_peak},
            "stage_ms": {"projector_upsample": st_mean[0], "allgather": st_mean[1], "far": far_ms,
                         "finalize_near": fin_ms},
            "cpu_baseline": cpu_base,
            "e2e": {"value": 1e3 / float(e2e_ms.item()), "unit": "matvec/s",
                    "h2d_bytes_per_step": int(h2d[0].item()), "d2h_bytes_per_step": int(h2d[1].item())},
            "gpu_launches": int(n_launch),
            "gpu_launches_per_step": dp.op.launches_per_matvec(),
            "clocks": clocks,
            "parity_sampled": parity,
            "setup_s": t_setup, "gen_s": t_gen,
        }
        print(json.dumps(line), flush=True)
    dp.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
