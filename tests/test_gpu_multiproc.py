"""The multi-process (one process per GPU) path of zeus_run, run for real with
two processes on one GPU over gloo (the round's GPU box has one B200; on an
8-GPU node the same code runs one process per device over NCCL).

* start sharding: per_run / best / tallies of a 2-rank run are bit-identical
  to the 1-process run (starts depend only on (seed, global
  index), the per-sweep barrier is an all-gather + np.argmin min-loc);
* the same with the per-sweep barrier fused into the sweep kernels as a
  peer-memory exchange over CUDA IPC (ZEUS_PSO_EXCHANGE=peer);
* the cross-process early-stop block (driver.py:137-202: one counter and flag
  for the whole pool): a convergence counted in one process stops the other
  process's starts, through CUDA IPC-mapped device memory and system-scope
  atomics.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(z, case):
    if case in ("shard", "shard_peer"):
        return z.rastrigin, z.ZeusConfig(N=4099, dim=10, range=(-5.12, 5.12), iter_pso=5,
                                         iter_bfgs=2000, seed=11, deterministic=True)
    return z.rastrigin, z.ZeusConfig(N=20000, dim=2, range=(-5.12, 5.12), iter_pso=2,
                                     iter_bfgs=1000, required_c=100, workers=2, seed=5)


def _worker(rank, world, port, q, case, gather="root"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    if case == "shard_peer":
        os.environ["ZEUS_PSO_EXCHANGE"] = "peer"  # barrier fused into the sweeps over IPC
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2603_28770_b200 as z
        from paper_2603_28770_b200 import engine
        from paper_2603_28770_b200.linesearch import LineSearchParams

        dev = torch.device("cuda", 0)
        if case == "ipc":
            blk = engine.StopBlock.get(None, dev)
            blk.arm(None, dev)
            P = engine.bfgs_params(1e-6, 1000, LineSearchParams())
            if rank == 1:
                # 64 starts already at the Rosenbrock minimum: converged at k = 0;
                # the 5th convergence raises the shared flag
                x0 = torch.ones((2, 64), dtype=torch.float64, device=dev)
                out = engine.BfgsBuffers.allocate(2, 64, dev)
                engine.run_bfgs(0, x0, P, out, dev, required_c=5, stop=(blk.counter, blk.flag))
                torch.cuda.synchronize()
            dist.barrier()
            res = None
            if rank == 0:
                # far from the minimum: would need many iterations, but the flag
                # raised by the OTHER process stops every start at the first probe
                x0 = torch.full((2, 256), -3.0, dtype=torch.float64, device=dev)
                out = engine.BfgsBuffers.allocate(2, 256, dev)
                engine.run_bfgs(0, x0, P, out, dev, required_c=5, stop=(blk.counter, blk.flag))
                torch.cuda.synchronize()
                res = (out.status.cpu().numpy(), out.iterations.cpu().numpy())
            q.put((rank, res))
            dist.barrier()
            return
        fn, cfg = _cfg(z, case)
        r = z.zeus_run(fn, cfg, gather=gather)
        pr = r.per_run
        lo, _ = engine.shard_bounds(cfg.N, rank, world)
        q.put((rank, pr.x_final.copy(), pr.f_final.copy(), pr.status_codes.copy(),
               pr.iterations.copy(), pr.grad_norm.copy(), r.best, r.converged_count,
               r.pso_best_before_bfgs, lo))
    finally:
        dist.destroy_process_group()


def _run(case, world=2, gather="root"):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, case, gather))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=600) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("case,world,gather", [("shard", 2, "all"), ("shard_peer", 2, "all"),
                                               ("shard", 4, "root"), ("shard_peer", 4, "root")])
def test_multi_process_run_is_bit_identical_to_one(z, case, world, gather):
    """2 and 4 processes on the one GPU: per_run, best, tallies and the PSO
    best bit-identical to the one-process run.  `shard_peer`: the per-sweep
    barrier runs inside the sweep kernels as a peer-memory exchange between
    the processes (IPC-mapped blocks, system-scope release/acquire flags)
    instead of the all-gather.  gather="all": every rank holds all N
    outcomes; gather="root" (the default): rank 0 holds all N, every other
    rank its own shard, and every rank the global best."""
    fn, cfg = _cfg(z, "shard")
    one = z.zeus_run(fn, cfg)
    for rank, x, f, s, k, gn, best, conv, psob, lo in _run(case, world, gather):
        full = gather == "all" or rank == 0
        sl = slice(0, cfg.N) if full else slice(lo, lo + len(s))
        assert full == (len(s) == cfg.N), (rank, len(s))
        assert np.array_equal(x, one.per_run.x_final[sl]), rank
        assert np.array_equal(f, one.per_run.f_final[sl], equal_nan=True)
        assert np.array_equal(s, one.per_run.status_codes[sl])
        assert np.array_equal(k, one.per_run.iterations[sl])
        assert best == one.best and conv == one.converged_count
        assert psob == one.pso_best_before_bfgs


def test_stop_block_is_shared_across_processes():
    (_, _), (_, _) = out = _run("ipc")
    status, iters = out[0][1]
    assert np.all(status == 2) and np.all(iters == 0)   # every start 'stopped' at k = 0


def test_two_process_early_stop_semantics(z):
    fn, cfg = _cfg(z, "stop")
    out = _run("stop")
    r0, r1 = out
    assert np.array_equal(r0[3][r1[9]:], r1[3])  # rank 1 holds its shard of rank 0's table
    assert r0[6] == r1[6]                        # the same global best on both ranks
    x, f, s, k, gn, bf, conv = r0[1], r0[2], r0[3], r0[4], r0[5], r0[6], r0[7]
    assert len(s) == cfg.N                        # parallel mode: every start reported
    assert conv == int(np.sum(s == 0)) and conv >= cfg.required_c
    assert np.sum(s == 2) > 0                     # the rest were stopped
    unstarted = (s == 2) & (k == 0)
    assert np.all(np.isinf(gn[unstarted]))        # never-started runs: |g| = inf
    # converged <=> |g| < theta, except runs stopped at the probe that precedes
    # the convergence test (bfgs.py:115-121): those keep their small |g|
    assert np.array_equal(s == 0, (gn < cfg.theta) & (s != 2))
    # both shards were stopped by the one shared flag (each half has stopped runs)
    half = (cfg.N + 1) // 2
    assert np.any(s[:half] == 2) and np.any(s[half:] == 2)


@pytest.mark.parametrize("exchange", ["collective", "peer"])
def test_bench_two_ranks_prints_one_line(exchange):
    """bench.py's N > 1 path (the driver's scaling run) end to end: two ranks
    under torch.distributed.run on the one GPU (gloo; collective barrier or
    the IPC peer exchange): every collective is taken by both ranks, rank 0
    alone prints one JSON line with n_gpus = 2 and the whole-job count."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ZEUS_BENCH_DEVICE="0", ZEUS_BENCH_BACKEND="gloo",
               ZEUS_PSO_EXCHANGE=exchange)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--config", "c1", "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "start-sharded x2"
    assert d["gpu_launches"] > 0 and d["roofline"]["achieved"] > 0
    assert d["value"] > 0 and d["e2e"]["value"] > 0
