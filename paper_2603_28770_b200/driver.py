"""End-to-end pipeline (driver.py of the reference) on B200.

``zeus_run(f, cfg)`` keeps the reference's signature, configuration and result
record.  Internally: the swarm lives in HBM (SoA), PSO init + ``iter_pso``
sweeps run as sm_100a kernels with a device min-loc barrier after each sweep,
then one persistent BFGS kernel refines every particle's final position
(driver.py:244) with forward-AD gradients, Armijo search and the rank-2
update fused on chip, then a device reduction yields ``best`` and the status
tallies.  Under ``torch.distributed`` (one process per GPU, NCCL) the starts
are sharded in contiguous global-index blocks and the only data-path
collective is the per-sweep all-gather of each shard's best candidate.
"""

from __future__ import annotations

import logging
import math
import time
import weakref
from dataclasses import dataclass, field, replace
from typing import Callable, Iterator, Optional, Sequence

import numpy as np
import torch

from . import _capi, _device, engine
from .bfgs import CONVERGED, DOMAIN_ERROR, STATUSES, BfgsOutcome
from .linesearch import LineSearchParams
from .objectives import objective_id
from .pso import PsoParams
from .streams import make_start_streams

__all__ = [
    "ZeusConfig",
    "ZeusResult",
    "RunStats",
    "NoValidOptimumError",
    "OutcomeList",
    "zeus_run",
    "reduce_best",
    "make_start_streams",
]

log = logging.getLogger(__name__)


class NoValidOptimumError(RuntimeError):
    """Every launched run ended in a domain error; no optimum to report
    (driver.py:45-46)."""


@dataclass
class ZeusConfig:
    """All pipeline hyperparameters (driver.py:49-95), same fields, defaults
    and validation as the reference."""

    N: int
    dim: int
    range: tuple[float, float]
    iter_pso: int = 5
    iter_bfgs: int = 1000
    iter_ls: int = 20
    theta: float = 1e-6
    required_c: int | None = None
    pso: PsoParams = field(default_factory=PsoParams)
    ls: LineSearchParams = field(default_factory=LineSearchParams)
    seed: int = 0
    workers: int = 0
    deterministic: bool = False

    def __post_init__(self):
        if self.N < 1:
            raise ValueError("N must be at least 1")
        if self.dim < 1:
            raise ValueError("dim must be at least 1")
        lower, upper = self.range
        if not lower < upper:
            raise ValueError("range requires lower < upper")
        if self.required_c is None:
            self.required_c = self.N
        if not 1 <= self.required_c <= self.N:
            raise ValueError("required_c must be in [1, N]")
        if min(self.iter_pso, self.iter_bfgs) < 0:
            raise ValueError("iteration budgets must be non-negative")
        if self.theta <= 0.0:
            raise ValueError("theta must be positive")
        if self.workers < 0:
            raise ValueError("workers must be non-negative")
        self.pso = replace(self.pso, iter_pso=self.iter_pso)
        self.ls = replace(self.ls, iter_ls=self.iter_ls)


@dataclass
class RunStats:
    """Per-start work counters returned by the BFGS kernel (host copies, in
    per_run order): they feed the algorithmic-FLOP roofline."""

    iterations: np.ndarray
    ls_trials: np.ndarray
    grad_evals: np.ndarray
    status_counts: dict
    pso_time: float = 0.0       # device seconds, PSO init + sweeps + barriers
    bfgs_time: float = 0.0      # device seconds, the persistent BFGS kernel
    reduce_time: float = 0.0    # device seconds, reduce_best (+ collectives)
    kernel_launches: int = 0    # our kernels launched by this call
    n_within: int | None = None  # zeus_run(within=(optimum, radius)): starts inside


@dataclass
class ZeusResult:
    """Outcome of one pipeline execution (driver.py:98-112).

    The first five fields are the reference's.  ``device_time`` (kernels +
    collectives, CUDA events) and ``stats`` are additions with defaults.
    """

    best: BfgsOutcome
    per_run: Sequence[BfgsOutcome]
    converged_count: int
    wall_time: float
    pso_best_before_bfgs: float
    device_time: float | None = None
    stats: RunStats | None = None


class OutcomeList(Sequence):
    """Lazy ``Sequence[BfgsOutcome]`` over host SoA copies of the per-start
    outputs: 1M frozen dataclasses would cost seconds of CPython time, so an
    entry is materialised on access.  Compares equal to a list of outcomes."""

    def __init__(self, x: np.ndarray, f: np.ndarray, gn: np.ndarray, it: np.ndarray,
                 st: np.ndarray, length: int | None = None):
        self._x, self._f, self._gn, self._it, self._st = x, f, gn, it, st
        self._n = len(f) if length is None else int(length)

    def __len__(self) -> int:
        return self._n

    def _one(self, i: int) -> BfgsOutcome:
        return BfgsOutcome(x_final=tuple(self._x[i].tolist()), f_final=float(self._f[i]),
                           grad_norm=float(self._gn[i]), iterations=int(self._it[i]),
                           status=STATUSES[int(self._st[i])])

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._one(k) for k in range(*i.indices(self._n))]
        if i < 0:
            i += self._n
        if not 0 <= i < self._n:
            raise IndexError(i)
        return self._one(i)

    def __iter__(self) -> Iterator[BfgsOutcome]:
        for i in range(self._n):
            yield self._one(i)

    def __eq__(self, other) -> bool:
        if not isinstance(other, Sequence) or len(other) != self._n:
            return NotImplemented if not isinstance(other, Sequence) else False
        return all(a == b for a, b in zip(self, other))

    def __repr__(self) -> str:
        return f"OutcomeList(n={self._n})"

    # columnar views (numpy), in per_run order
    @property
    def x_final(self) -> np.ndarray:
        return self._x[: self._n]

    @property
    def f_final(self) -> np.ndarray:
        return self._f[: self._n]

    @property
    def grad_norm(self) -> np.ndarray:
        return self._gn[: self._n]

    @property
    def iterations(self) -> np.ndarray:
        return self._it[: self._n]

    @property
    def status_codes(self) -> np.ndarray:
        return self._st[: self._n]


def reduce_best(outcomes: Sequence[BfgsOutcome]) -> tuple[BfgsOutcome, int]:
    """Minimum f_final among non-domain-error, non-NaN outcomes, lowest index
    on ties (driver.py:115-134).  Raises NoValidOptimumError if none."""
    if isinstance(outcomes, OutcomeList):
        f, st = outcomes.f_final, outcomes.status_codes
        valid = (st != STATUSES.index(DOMAIN_ERROR)) & ~np.isnan(f)
        if not valid.any():
            raise NoValidOptimumError("all runs ended in domain errors")
        idx = int(np.flatnonzero(valid)[np.argmin(f[valid])])
        return outcomes[idx], idx
    best: BfgsOutcome | None = None
    best_index = -1
    for i, outcome in enumerate(outcomes):
        if outcome.status == DOMAIN_ERROR or math.isnan(outcome.f_final):
            continue
        if best is None or outcome.f_final < best.f_final:
            best = outcome
            best_index = i
    if best is None:
        raise NoValidOptimumError("all runs ended in domain errors")
    return best, best_index


def _peer_exchange(process_group, world: int) -> bool:
    """Fuse the multi-GPU PSO barrier into the sweep kernels (peer-memory
    exchange) when the ranks' devices can map each other: NCCL groups of at
    most 8 ranks.  ZEUS_PSO_EXCHANGE=collective forces the all-gather path,
    =peer forces the exchange (e.g. gloo ranks sharing one GPU)."""
    import os

    mode = os.environ.get("ZEUS_PSO_EXCHANGE", "auto")
    if mode == "collective" or world > 8:
        return False
    if mode == "peer":
        return True
    return not engine._host_backend(process_group)


def _broadcast_best(per_run, bidx: int, owner: int, d: int, group, dev) -> BfgsOutcome:
    """The best outcome from the rank whose table holds it (group rank
    ``owner`` always does: it ran that start) to every rank."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    row = torch.zeros(d + 4, dtype=torch.float64)
    if rank == owner:
        o = per_run[bidx]
        row[:d] = torch.tensor(o.x_final, dtype=torch.float64)
        row[d:] = torch.tensor([o.f_final, o.grad_norm, o.iterations, STATUSES.index(o.status)],
                               dtype=torch.float64)
    src = dist.get_global_rank(group, owner) if group is not None else owner
    if not engine._host_backend(group):
        row = row.to(dev)
    dist.broadcast(row, src=src, group=group)
    r = row.cpu().numpy()
    return BfgsOutcome(x_final=tuple(float(v) for v in r[:d]), f_final=float(r[d]),
                       grad_norm=float(r[d + 1]), iterations=int(r[d + 2]),
                       status=STATUSES[int(r[d + 3])])


_PINNED: dict = {}
_IN_USE = (lambda: True)


class _HostTable:
    """A page-locked host table for a run's results and a weak reference to
    the numpy array the run's per_run views (None: free)."""

    __slots__ = ("t", "ref")

    def __init__(self, t):
        self.t, self.ref = t, None

    def hold(self, arr: np.ndarray) -> np.ndarray:
        self.ref = weakref.ref(arr)
        return arr


def _pinned(shape: tuple, dtype) -> _HostTable:
    """Fresh page-locked allocations cost ~0.5 ms per MB (measured: 52-150 ms
    for a 109 MB table), more than the copy itself, so the tables are pooled
    and a table is reused once no result views it any more."""
    pool = _PINNED.setdefault((shape, dtype), [])
    for e in pool:
        if e.ref is None or e.ref() is None:
            e.ref = _IN_USE  # until the caller hands its views out (hold) or releases it
            return e
    # touched once on the host: the kernels write these rows directly, and a
    # first touch from the device is paid inside the run (measured: +300 ms
    # in the BFGS kernel for a fresh 436 MB table)
    e = _HostTable(torch.zeros(shape, dtype=dtype, pin_memory=True))
    e.ref = _IN_USE
    pool.append(e)
    if len(pool) > 4:  # bounded: the oldest table stays with whichever result views it
        pool.pop(0)
    return e


def _host_device_ptr(t: torch.Tensor) -> int:
    """Device address of a page-locked host tensor (zeus_host_device_ptr)."""
    import ctypes

    p = ctypes.c_void_p()
    _capi.check(_capi.lib().zeus_host_device_ptr(t.data_ptr(), ctypes.byref(p)),
                "host_device_ptr")
    return int(p.value)


def _stop_wave(cfg: ZeusConfig, required_c: int) -> int:
    """First launch size of the parallel early-stop mode: the reference's
    pool has `workers` runs in flight at a time (driver.py:184-201), and at
    least required_c starts must run to reach the target."""
    return max(int(required_c), int(cfg.workers), 1)


def _gather_mode(gather) -> str:
    if gather is True or gather == "all":
        return "all"
    if gather is False or gather == "local":
        return "local"
    if gather == "root":
        return "root"
    raise ValueError("gather must be 'root', 'all' (True) or False")


def _dist_world(process_group):
    if not torch.distributed.is_available() or not torch.distributed.is_initialized():
        return 0, 1
    return (torch.distributed.get_rank(process_group),
            torch.distributed.get_world_size(process_group))


def _gather_rows(t: torch.Tensor, per: int, world: int, group) -> torch.Tensor:
    """All-gather equal-size padded shards along the last dim."""
    lead = t.shape[:-1]
    pad = torch.zeros(*lead, per, dtype=t.dtype, device=t.device)
    pad[..., : t.shape[-1]] = t
    flat = pad.reshape(-1, per).contiguous()
    out = engine.all_gather_flat(flat.view(-1), group).view((world,) + tuple(flat.shape))
    # [world][rows][per] -> [rows][world*per]
    return out.permute(1, 0, 2).reshape(*lead, world * per)


def _zeus_run_devices(obj, cfg: ZeusConfig, devs, starts, within, t0) -> ZeusResult:
    """zeus_run over several GPUs from ONE process (``devices=``): shard g of
    G runs on devs[g] on a stream of its own.  The PSO barrier is
    the peer-memory exchange inside the sweep kernels (blocks addressed
    directly, peer access enabled between the devices), the early-stop
    counter/flag (workers > 0) is one block on devs[0] reached by every
    device, and the per-shard results are merged on the host in global start
    order -- the same per-start results as one GPU.  Every
    shard's PSO is enqueued before anything else, so no host call can wait on
    a device that waits on a shard not yet launched."""
    G = len(devs)
    N, d = cfg.N, cfg.dim
    required_c = N if cfg.deterministic else int(cfg.required_c)
    early = required_c < N
    device_stop = early and cfg.workers > 0
    launches0 = engine.LAUNCHES[0]
    if starts is not None:
        pts = np.asarray(starts, dtype=np.float64)
        if pts.shape != (N, d):
            raise ValueError(f"starts must have shape ({N}, {d})")
    stop = None
    if device_stop:
        blk = engine.StopBlock.local(devs)
        blk.reset_now(devs[0])
        stop = (blk.counter, blk.flag)
    xgs = engine.PsoExchange.local(devs, d) if starts is None else None
    sh = []
    for g, dev in enumerate(devs):  # ---- phase 1: every shard's PSO (driver.py:236-241)
        lo, hi = engine.shard_bounds(N, g, G)
        n = hi - lo
        # one stream per shard (after the device's pending work): shards that
        # share a device must not queue behind each other's exchange waits
        stream = torch.cuda.Stream(dev)
        stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.device(dev), torch.cuda.stream(stream):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record(stream)
            if starts is None:
                shard = engine.SwarmShard(obj, d, max(n, 1), lo, cfg.seed, dev)
                shard.run_xchg(xgs[g], n, cfg.range[0], cfg.range[1], cfg.pso.w,
                               cfg.pso.c1_pso, cfg.pso.c2_pso, cfg.iter_pso)
                x0, gbest = shard.x[:, :n], shard.gbest
            else:
                x0 = (_device.to_soa(pts[lo:hi], dev) if n > 0 else
                      torch.empty((d, 0), device=dev, dtype=torch.float64))
                shard, gbest = None, None
            ev[1].record(stream)
        sh.append(dict(dev=dev, lo=lo, n=n, stream=stream, ev=ev, shard=shard, x0=x0,
                       gbest=gbest))
    params = engine.bfgs_params(cfg.theta, cfg.iter_bfgs, cfg.ls)
    L = _capi.lib()
    for c in sh:  # ---- phase 2: BFGS, reduction, packing, D2H (all asynchronous)
        dev, n, lo = c["dev"], c["n"], c["lo"]
        with torch.cuda.device(dev), torch.cuda.stream(c["stream"]):
            out = engine.BfgsBuffers.allocate(d, n, dev)
            if n > 0:
                x0 = c["x0"]
                engine.run_bfgs(obj, x0.contiguous() if x0.stride(0) != x0.shape[1] else x0,
                                params, out, dev, required_c=required_c, stop=stop,
                                wave=_stop_wave(cfg, required_c) if stop is not None else 0)
            c["ev"][2].record(c["stream"])
            best = torch.empty(2, dtype=torch.float64, device=dev)
            tallies = torch.zeros(4, dtype=torch.int64, device=dev)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            if n > 0:
                ws = _device.workspace(L.zeus_argmin_workspace_bytes(n), dev)
                _capi.check(L.zeus_reduce_best(n, lo, out.f_final.data_ptr(),
                                               out.status.data_ptr(), best.data_ptr(),
                                               tallies.data_ptr(), ws.data_ptr(),
                                               _device.stream_ptr(dev)), "reduce_best")
                engine.LAUNCHES[0] += 2
                if within is not None:
                    opt = torch.tensor([float(v) for v in within[0]], dtype=torch.float64,
                                       device=dev)
                    _capi.check(L.zeus_count_within(d, n, out.x_final.data_ptr(),
                                                    out.x_final.shape[1], opt.data_ptr(),
                                                    float(within[1]), cnt.data_ptr(),
                                                    _device.stream_ptr(dev)), "count_within")
                    engine.LAUNCHES[0] += 1
            else:
                best[0], best[1] = math.nan, -1.0
            c["ev"][3].record(c["stream"])
            fpack = torch.empty((n, d + 2), dtype=torch.float64, device=dev)
            ipack = torch.empty((n, 4), dtype=torch.int32, device=dev)
            spack = torch.empty(8, dtype=torch.float64, device=dev)
            _capi.check(L.zeus_pack_results(
                out.c_struct(n), d, n, fpack.data_ptr(), ipack.data_ptr(), tallies.data_ptr(),
                c["gbest"].data_ptr() if c["gbest"] is not None else None, best.data_ptr(), 2,
                spack.data_ptr(), _device.stream_ptr(dev)), "pack_results")
            engine.LAUNCHES[0] += 1
            if within is not None:
                spack[7] = cnt[0]
            c["fe"] = _pinned(tuple(fpack.shape), torch.float64)  # (copied out below)
            c["ie"] = _pinned(tuple(ipack.shape), torch.int32)
            c["fh"], c["ih"] = c["fe"].t, c["ie"].t
            c["sh"] = torch.empty(8, dtype=torch.float64, pin_memory=True)
            c["fh"].copy_(fpack, non_blocking=True)
            c["ih"].copy_(ipack, non_blocking=True)
            c["sh"].copy_(spack, non_blocking=True)
    for c in sh:
        c["stream"].synchronize()
    for xg in xgs or ():
        xg.check()
    fnp = np.concatenate([c["fh"].numpy() for c in sh])
    inp = np.concatenate([c["ih"].numpy() for c in sh])
    for c in sh:  # the host tables were copied out: free for the next run
        c["fe"].ref = c["ie"].ref = None
    shs = np.stack([c["sh"].numpy() for c in sh])
    x_host = fnp[:, :d]
    f_h, gn_h = fnp[:, d], fnp[:, d + 1]
    it_h, st_h, ls_h, ge_h = inp[:, 0], inp[:, 1].astype(np.uint8), inp[:, 2], inp[:, 3]
    m = len(f_h)
    converged_count = int(shs[:, 0].sum())
    n_in = int(shs[:, 7].sum()) if within is not None else None
    if early and not device_stop:
        # sequential semantics (driver.py:205-217): cut after the required_c-th convergence
        conv = np.flatnonzero(st_h == 0)
        if len(conv) >= required_c:
            m = int(conv[required_c - 1]) + 1
        converged_count = int(np.count_nonzero(st_h[:m] == 0))
        valid = (st_h[:m] != 3) & ~np.isnan(f_h[:m])
        if not valid.any():
            raise NoValidOptimumError("all runs ended in domain errors")
        bidx = int(np.flatnonzero(valid)[np.argmin(f_h[:m][valid])])
        if within is not None:
            tgt = np.asarray([float(v) for v in within[0]], dtype=np.float64)
            n_in = int(np.count_nonzero(np.linalg.norm(x_host[:m] - tgt, axis=1) < within[1]))
    else:
        bidx = engine.resolve_minloc(shs[:, 5:7].tolist())
        if bidx < 0:
            raise NoValidOptimumError("all runs ended in domain errors")
    per_run = OutcomeList(x_host, f_h, gn_h, it_h, st_h, length=m)

    def span(a: int, b: int) -> float:  # slowest shard between two of its events
        return max(c["ev"][a].elapsed_time(c["ev"][b]) for c in sh) / 1e3

    stats = RunStats(iterations=it_h[:m], ls_trials=ls_h[:m], grad_evals=ge_h[:m],
                     status_counts={s: int(np.count_nonzero(st_h[:m] == k))
                                    for k, s in enumerate(STATUSES)},
                     pso_time=span(0, 1), bfgs_time=span(1, 2), reduce_time=span(2, 3),
                     kernel_launches=engine.LAUNCHES[0] - launches0, n_within=n_in)
    return ZeusResult(best=per_run[bidx], per_run=per_run, converged_count=converged_count,
                      wall_time=time.perf_counter() - t0, pso_best_before_bfgs=float(shs[0, 4]),
                      device_time=span(0, 3), stats=stats)


def check_objective_device(obj, dev) -> None:
    """A DeviceObjective's NVRTC module and data live on the device it was
    built for; launching it on another device would cross contexts."""
    if obj.device.index != torch.device(dev).index:
        raise ValueError(f"DeviceObjective {obj.name!r} was compiled for cuda:{obj.device.index}, "
                         f"not cuda:{torch.device(dev).index}: build it with device=")


def zeus_run(f: Callable[[Sequence], object], cfg: ZeusConfig, *, device=None,
             process_group=None, starts: Optional[np.ndarray] = None,
             gather="root", within=None, devices=None) -> ZeusResult:
    """Run the full pipeline on registered objective ``f`` (driver.py:220-265).

    Extensions (keyword-only, defaults reproduce the reference):
      device        CUDA device for this process (default: current).
      process_group torch.distributed group to shard starts over (default:
                    the world group when torch.distributed is initialised).
      starts        host-supplied BFGS starts [N][dim]: skips PSO (used to
                    decouple BFGS parity from PSO libm flips).
      gather        several ranks: "root" (default) gives group rank 0, the
                    caller's process, per_run over all N starts and the
                    other ranks their own shard; "all" (or True) gives every
                    rank all N; False keeps per_run local to each shard.
                    ``best`` is the global best on every rank.
      within        (optimum, radius): count the starts whose final point lies
                    within radius of optimum on device (bench.py:131-141),
                    reported as stats.n_within (summed over ranks).
      devices       several GPUs from THIS process: an int (the first n
                    devices) or a sequence of device indices / torch devices
                    (one start shard per entry).  Same per-start results as
                    one GPU; no torch.distributed needed.

    Early stop: ``deterministic`` or ``required_c == N`` runs every start.
    ``workers == 0`` with ``required_c < N`` reproduces the reference's
    sequential semantics exactly (per_run is the prefix ending at the
    required_c-th convergence; every start is independent so the prefix is
    computed, then cut).  ``workers > 0`` uses the device stop protocol:
    converged starts bump a device counter, the start that reaches
    ``required_c`` raises a flag polled at the top of every iteration, and the
    rest end ``stopped`` (timing-dependent, as in the reference).
    """
    t0 = time.perf_counter()
    obj = objective_id(f, cfg.dim)
    if within is not None and len(within[0]) != cfg.dim:
        raise ValueError("within: optimum must have dim coordinates")
    if devices is not None:
        if isinstance(devices, int):
            devices = list(range(devices))
        devs = [d if isinstance(d, torch.device) else torch.device("cuda", int(d))
                for d in devices]
        if not devs or any(d.type != "cuda" for d in devs):
            raise ValueError("devices: one or more CUDA devices")
        if _dist_world(process_group)[1] > 1:
            raise ValueError("devices= runs in one process; do not combine with a process group")
        for d_ in devs:
            _device.require_device(d_)
        if len(devs) > 1:
            if not isinstance(obj, int) and len({d_.index for d_ in devs}) > 1:
                raise NotImplementedError(
                    "a user objective is compiled for one device: run one process per GPU "
                    "(torchrun) to use several GPUs")
            if not isinstance(obj, int):
                check_objective_device(obj, devs[0])
            return _zeus_run_devices(obj, cfg, devs, starts, within, t0)
        device = devs[0]
    dev = _device.require_device(device)
    if not isinstance(obj, int):
        check_objective_device(obj, dev)
    rank, world = _dist_world(process_group)
    N, d = cfg.N, cfg.dim
    lo, hi = engine.shard_bounds(N, rank, world)
    n = hi - lo
    required_c = N if cfg.deterministic else int(cfg.required_c)
    early = required_c < N
    device_stop = early and cfg.workers > 0
    stream = torch.cuda.current_stream(dev)
    ev_start, ev_pso, ev_bfgs, ev_end = (torch.cuda.Event(enable_timing=True) for _ in range(4))
    launches0 = engine.LAUNCHES[0]
    ev_start.record(stream)

    # ---- PSO phase (driver.py:236-241)
    pso_best = math.nan
    xchg = None
    if starts is None:
        shard = engine.SwarmShard(obj, d, max(n, 1), lo, cfg.seed, dev)
        lower, upper = cfg.range
        if world == 1:
            # one GPU: the barrier is the shard's own candidate -> fused sweeps
            shard.run_local(lower, upper, cfg.pso.w, cfg.pso.c1_pso, cfg.pso.c2_pso,
                            cfg.iter_pso)
        elif _peer_exchange(process_group, world) and \
                (xchg := engine.PsoExchange.get(process_group, dev, d)) is not None:
            # several GPUs: the barrier is fused into every sweep launch as a
            # peer-memory exchange of the shard candidates (no NCCL per sweep)
            shard.run_xchg(xchg, n, lower, upper, cfg.pso.w, cfg.pso.c1_pso, cfg.pso.c2_pso,
                           cfg.iter_pso)
        else:
            barrier = (engine.local_barrier if world == 1 else
                       engine.make_dist_barrier(process_group))
            if n > 0:
                shard.init(lower, upper)
            else:
                shard.cand.zero_()
                shard.cand[1] = -1.0
            barrier(shard)
            for _ in range(cfg.iter_pso):
                if n > 0:
                    shard.sweep(cfg.pso.w, cfg.pso.c1_pso, cfg.pso.c2_pso)
                barrier(shard)
        x0 = shard.x[:, :n]
        gbest = shard.gbest
    else:
        pts = np.asarray(starts, dtype=np.float64)
        if pts.shape != (N, d):
            raise ValueError(f"starts must have shape ({N}, {d})")
        x0 = _device.to_soa(pts[lo:hi], dev) if n > 0 else torch.empty((d, 0), device=dev,
                                                                        dtype=torch.float64)
        gbest = None

    ev_pso.record(stream)
    # ---- multistart BFGS (driver.py:243-249)
    out = engine.BfgsBuffers.allocate(d, n, dev)
    # one process: the kernels write every start's outcome straight into
    # page-locked host rows as the start finishes (zeus_bfgs_out.rows), so no
    # pack and no copy follow the run; several ranks pack on the device and
    # gather instead
    direct = world == 1 and n > 0
    if direct:
        fe, ie = _pinned((n, d + 2), torch.float64), _pinned((n, 4), torch.int32)
        out.rows = (_host_device_ptr(fe.t), d + 2, _host_device_ptr(ie.t))
    params = engine.bfgs_params(cfg.theta, cfg.iter_bfgs, cfg.ls)
    stop = None
    if device_stop and world == 1:
        stop = (torch.zeros(1, dtype=torch.int64, device=dev),
                torch.zeros(1, dtype=torch.int32, device=dev))
    elif device_stop:
        # one counter/flag for every GPU of the group (driver.py:137-202)
        blk = engine.StopBlock.get(process_group, dev)
        blk.arm(process_group, dev)
        stop = (blk.counter, blk.flag)
    if n > 0:
        engine.run_bfgs(obj, x0.contiguous() if x0.stride(0) != x0.shape[1] else x0, params,
                        out, dev, required_c=required_c, stop=stop,
                        wave=_stop_wave(cfg, required_c) if stop is not None else 0)

    ev_bfgs.record(stream)
    # ---- reduction (driver.py:250-251) on device
    L = _capi.lib()
    best_dev = torch.empty(2, dtype=torch.float64, device=dev)
    tallies = torch.zeros(4, dtype=torch.int64, device=dev)
    ws = _device.workspace(L.zeus_argmin_workspace_bytes(max(n, 1)), dev)
    if n > 0:
        _capi.check(L.zeus_reduce_best(n, lo, out.f_final.data_ptr(), out.status.data_ptr(),
                                       best_dev.data_ptr(), tallies.data_ptr(), ws.data_ptr(),
                                       _device.stream_ptr(dev)), "reduce_best")
        engine.LAUNCHES[0] += 2
    else:
        best_dev[0] = math.nan
        best_dev[1] = -1.0
    n_within = None
    if within is not None:
        opt = torch.tensor([float(v) for v in within[0]], dtype=torch.float64, device=dev)
        if opt.numel() != d:
            raise ValueError("within: optimum must have dim coordinates")
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        if n > 0:
            _capi.check(L.zeus_count_within(d, n, out.x_final.data_ptr(), out.x_final.shape[1],
                                            opt.data_ptr(), float(within[1]), cnt.data_ptr(),
                                            _device.stream_ptr(dev)), "count_within")
            engine.LAUNCHES[0] += 1
        if world > 1:
            engine.all_reduce_sum(cnt, group=process_group)
        n_within = cnt
    if world > 1:
        best_dev = engine.gather_candidates(best_dev, process_group)  # resolved on the host
        engine.all_reduce_sum(tallies, group=process_group)
    ev_end.record(stream)

    # ---- results to host (part of the end-to-end wall time): two row-major
    # tables ([n][d + 2] f64: x, f, |g|; [n][4] i32: k, status, trials,
    # gradients) -- one process: already written to page-locked host memory
    # by the BFGS kernels; several ranks: packed on the device, gathered, and
    # copied with one asynchronous D2H each.  The host arrays are views.
    # Several ranks: the packed shards (padded to ceil(N / world) rows) are
    # gathered to group rank 0 (gather="root", the caller's copy) or to every
    # rank (gather="all" / True); gather=False keeps the local shard.
    mode = _gather_mode(gather)
    if early and not device_stop and mode == "root":
        mode = "all"  # the sequential prefix cut needs the whole table on every rank
    per = -(-N // world)
    npack = 0 if direct else (per if world > 1 else n)
    fpack = torch.empty((npack, d + 2), dtype=torch.float64, device=dev)
    ipack = torch.empty((npack, 4), dtype=torch.int32, device=dev)
    # scalars in one small table: tallies[4], the PSO best f, every rank's [f, idx]
    spack = torch.empty(5 + best_dev.numel(), dtype=torch.float64, device=dev)
    _capi.check(L.zeus_pack_results(
        out.c_struct(n), d, 0 if direct else n, fpack.data_ptr(), ipack.data_ptr(),
        tallies.data_ptr(), gbest.data_ptr() if gbest is not None else None,
        best_dev.data_ptr(), best_dev.numel(), spack.data_ptr(), _device.stream_ptr(dev)),
        "pack_results")
    engine.LAUNCHES[0] += 1
    base = lo
    if world > 1 and mode == "local":
        fpack, ipack = fpack[:n], ipack[:n]
    elif world > 1:
        if mode == "all":
            gf = engine.all_gather_flat(fpack.view(-1), process_group)
            gi = engine.all_gather_flat(ipack.view(-1), process_group)
        else:
            gf = engine.gather_root_flat(fpack.view(-1), process_group)
            gi = engine.gather_root_flat(ipack.view(-1), process_group)
        if gf is not None:  # this rank holds the whole table
            fpack = gf.view(world * per, d + 2)[:N]
            ipack = gi.view(world * per, 4)[:N]
            base = 0
        else:
            fpack, ipack = fpack[:n], ipack[:n]
    if not direct:
        fe, ie = _pinned(tuple(fpack.shape), torch.float64), _pinned(tuple(ipack.shape), torch.int32)
        fe.t.copy_(fpack, non_blocking=True)
        ie.t.copy_(ipack, non_blocking=True)
    fh, ih = fe.t, ie.t
    sh = spack.cpu().numpy()
    best_host = sh[5:]  # (world > 1: every rank's [f, idx])
    stream.synchronize()
    if xchg is not None:
        xchg.check()
    device_time = ev_start.elapsed_time(ev_end) / 1e3
    fnp, inp = fe.hold(fh.numpy()), ie.hold(ih.numpy())
    x_host = fnp[:, :d]
    host = [fnp[:, d], fnp[:, d + 1], inp[:, 0], inp[:, 1].astype(np.uint8), inp[:, 2],
            inp[:, 3]]
    tallies_host = sh[0:4].astype(np.int64)
    pso_best = float(sh[4])
    f_h, gn_h, it_h, st_h, ls_h, ge_h = host
    m = len(f_h)
    converged_count = int(tallies_host[0])
    if early and not device_stop:
        # sequential semantics (driver.py:205-217): cut after the required_c-th convergence
        conv = np.flatnonzero(st_h == 0)
        if base == 0 and len(conv) >= required_c:
            m = int(conv[required_c - 1]) + 1
        converged_count = int(np.count_nonzero(st_h[:m] == 0))
        valid = (st_h[:m] != 3) & ~np.isnan(f_h[:m])
        if not valid.any():
            raise NoValidOptimumError("all runs ended in domain errors")
        bidx = int(np.flatnonzero(valid)[np.argmin(f_h[:m][valid])])
    else:
        gidx = engine.resolve_minloc(best_host.reshape(-1, 2).tolist())
        if gidx < 0:
            raise NoValidOptimumError("all runs ended in domain errors")
        bidx = gidx - base
    per_run = OutcomeList(x_host, f_h, gn_h, it_h, st_h, length=m)
    n_in = None if n_within is None else int(n_within.item())
    if n_within is not None and m < len(f_h):
        # sequential early stop reports a prefix: count inside it (host columns)
        tgt = np.asarray([float(v) for v in within[0]], dtype=np.float64)
        n_in = int(np.count_nonzero(np.linalg.norm(x_host[:m] - tgt, axis=1) < within[1]))
    if world > 1 and not (early and not device_stop):
        # the global best on every rank: its owner broadcasts the row
        best = _broadcast_best(per_run, bidx, gidx // per, d, process_group, dev)
    else:
        best = per_run[bidx]
    stats = RunStats(iterations=it_h[:m], ls_trials=ls_h[:m], grad_evals=ge_h[:m],
                     status_counts={s: int(np.count_nonzero(st_h[:m] == k))
                                    for k, s in enumerate(STATUSES)},
                     pso_time=ev_start.elapsed_time(ev_pso) / 1e3,
                     bfgs_time=ev_pso.elapsed_time(ev_bfgs) / 1e3,
                     reduce_time=ev_bfgs.elapsed_time(ev_end) / 1e3,
                     kernel_launches=engine.LAUNCHES[0] - launches0,
                     n_within=n_in)
    return ZeusResult(best=best, per_run=per_run, converged_count=converged_count,
                      wall_time=time.perf_counter() - t0, pso_best_before_bfgs=pso_best,
                      device_time=device_time, stats=stats)
