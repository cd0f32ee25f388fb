"""CPU, world_size 2 over gloo: the multi-GPU plumbing of the start-sharded
pipeline -- shard partition, the per-sweep candidate
all-gather, the np.argmin min-loc rule across shards, and the padded
all-gather of per-start outputs.  The device kernels themselves are covered
by the -m gpu shard-emulation tests (tests/test_gpu_pso.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_28770_b200 import driver, engine

        N, d = 11, 3
        lo, hi = engine.shard_bounds(N, rank, world)
        # every shard proposes its best personal best [f, idx, x...]
        rng = np.random.default_rng(rank)
        f = [3.0, 1.0][rank]
        cand = torch.tensor([f, float(lo + 1)] + rng.uniform(size=d).tolist(),
                            dtype=torch.float64)
        g = engine.gather_candidates(cand).reshape(world, d + 2)
        win = engine.resolve_minloc([(row[0].item(), row[1].item()) for row in g])
        # ties: equal f on both ranks -> the lower global index must win
        tie = torch.tensor([2.0, float(lo + 2)], dtype=torch.float64)
        tg = engine.gather_candidates(tie).reshape(world, 2)
        twin = engine.resolve_minloc(tg.tolist())
        # empty shard (idx = -1) never wins; NaN wins (np.argmin)
        e = torch.tensor([-5.0, -1.0] if rank == 0 else [7.0, float(lo)], dtype=torch.float64)
        ewin = engine.resolve_minloc(engine.gather_candidates(e).reshape(world, 2).tolist())
        nan = torch.tensor([float("nan") if rank == 1 else 0.0, float(lo)], dtype=torch.float64)
        nwin = engine.resolve_minloc(engine.gather_candidates(nan).reshape(world, 2).tolist())
        # padded all-gather of per-start SoA outputs (ragged last shard)
        n = hi - lo
        xs = torch.arange(lo, hi, dtype=torch.float64).repeat(d, 1) + 100 * torch.arange(d)[:, None]
        per = -(-N // world)
        gx = driver._gather_rows(xs, per, world, None)[:, :N]
        # the peer-memory exchange setup is agreed: without device memory
        # (this CPU box) every rank gets None and falls back to the collective
        xg = engine.PsoExchange.get(None, torch.device("cpu"), d)
        q.put((rank, lo, hi, g.numpy().copy(), win, twin, ewin, nwin, gx.numpy().copy(),
               xg is None))
    finally:
        dist.destroy_process_group()


def test_two_rank_plumbing():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, lo0, hi0, g0, w0, t0, e0, n0, x0, f0), (r1, lo1, hi1, g1, w1, t1, e1, n1, x1, f1) = out
    assert (lo0, hi0, lo1, hi1) == (0, 6, 6, 11)
    assert np.array_equal(g0, g1)                 # identical gathered candidates on every rank
    assert w0 == w1 == 7                          # rank 1's f=1.0 at global index 6+1
    assert t0 == t1 == 2                          # tie f=2.0: lower global index (0+2) wins
    assert e0 == e1 == 6                          # empty shard ignored
    assert n0 == n1 == 6                          # NaN wins like np.argmin
    want = np.arange(11)[None, :] + 100 * np.arange(3)[:, None]
    assert np.array_equal(x0, want) and np.array_equal(x1, want)
    assert f0 and f1                              # exchange unavailable on both: fallback


def test_resolve_minloc_matches_np_argmin():
    from paper_2603_28770_b200.engine import resolve_minloc

    rng = np.random.default_rng(0)
    for _ in range(200):
        v = rng.integers(0, 4, size=7).astype(float)
        if rng.random() < 0.2:
            v[rng.integers(0, 7)] = np.nan
        assert resolve_minloc(list(zip(v, range(7)))) == int(np.argmin(v))
