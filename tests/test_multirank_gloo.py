"""Multi-rank host logic on CPU (gloo, world_size 2): the target/panel partition and the
all-gather layout used by slb_matvec.  Each rank upsamples only its own
panels, the shards are all-gathered into the global fine-source order, and each rank evaluates
its own target rows; the gathered rows must equal the single-process operator bit for bit.
The arithmetic on each rank is the oracle's (tests may call it); what is under test is the
partition (paper_2310_00889_b200.shard), the row assignment (harness.local_rows) and the
gathered layout."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_00889_b200.shard import partition_panels


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, kw, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from synth import make_config
        from harness import local_rows
        pr = make_config(name, **kw)
        rows, pb, pe, n_on, ranges = local_rows(pr, rank, world)
        d = pr.sdim
        orc = O.Oracle(pr)
        # sigma' on local panels (projector is per body; bodies are whole on a rank)
        sp_full, _, Ls_full = orc.prepare(pr.sigma)
        no, fo = pr.node_off(), pr.fine_off()          # panel -> node offsets (ragged-safe)
        sp_loc = sp_full[no[pb]:no[pe]]
        if pr.ragged:
            sf_loc = O.upsample_ragged(sp_loc.reshape(-1), pr.ns_of_panel()[pb:pe], pr.nt_of_panel()[pb:pe],
                                       pr.ms_of_panel()[pb:pe], pr.mt_of_panel()[pb:pe], d).reshape(-1, d)
        else:
            sf_loc = O.upsample(sp_loc.reshape(-1), pe - pb, pr.Ns, pr.Nt, pr.Ms, pr.Mt, d).reshape(-1, d)
        assert sf_loc.shape[0] == fo[pe] - fo[pb]
        # all-gather (variable counts: pad to the max shard, as a grouped broadcast would place them)
        maxn = max(int(fo[e] - fo[b]) for b, e in ranges)
        buf = torch.zeros(maxn * d, dtype=torch.float64)
        buf[:sf_loc.size] = torch.from_numpy(sf_loc.reshape(-1))
        parts = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
        sf = np.concatenate([p.numpy()[:int(fo[e] - fo[b]) * d] for p, (b, e) in zip(parts, ranges)]).reshape(-1, d)
        # this rank's rows with the gathered fine density
        u_loc = orc.apply_rows(pr.sigma, rows, prepared=(sp_full, sf, Ls_full))
        out = [None] * world
        dist.all_gather_object(out, (rows, u_loc, (pb, pe)))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c4", dict(n_loops=3, panels=6)), ("c2", dict(panels=9)),
                                     ("c3v", dict(panels=6))])
def test_two_rank_partition_matches_single(name, kw):
    import oracle as O
    from synth import make_config
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, kw, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pr = make_config(name, **kw)
    rows = np.concatenate([o[0] for o in out])
    assert np.array_equal(np.sort(rows), np.arange(pr.T))          # every target exactly once
    # panel ranges contiguous, ordered, covering
    rg = [o[2] for o in out]
    assert rg[0][0] == 0 and rg[-1][1] == pr.P and all(rg[i][1] == rg[i + 1][0] for i in range(world - 1))
    if pr.projector:   # whole bodies per rank
        for b, e in rg:
            assert b == 0 or pr.body_of_panel[b] != pr.body_of_panel[b - 1]
    u = np.concatenate([o[1] for o in out])
    ref = O.Oracle(pr).apply_rows(pr.sigma, rows)
    assert np.array_equal(u, ref)


def test_partition_panels_properties():
    for n, R in [(8, 1), (8, 8), (4608, 8), (9, 2), (2048, 3), (1, 1), (5, 8)]:
        rg = partition_panels(n, R)
        assert rg[0][0] == 0 and rg[-1][1] == n
        assert all(rg[i][1] == rg[i + 1][0] for i in range(R - 1))
        sizes = [e - b for b, e in rg]
        assert max(sizes) - min(sizes) <= 1
    bop = np.repeat(np.arange(64), 32)
    rg = partition_panels(bop.size, 8, bop, whole_bodies=True)
    assert all(b % 32 == 0 for b, _ in rg) and [e - b for b, e in rg] == [256] * 8
