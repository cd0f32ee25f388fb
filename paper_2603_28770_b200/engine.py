"""Device engine: launches the sm_100a kernels for one shard of the swarm.

A *shard* is the contiguous block of global particle / start indices
[i0, i0 + n) owned by one GPU (one process per GPU).  Everything a shard
computes is a pure function of (seed, global index, gbest history), so any
sharding of the same problem yields bit-identical per-start results
(SURVEY.md section 8(e)); the only exchange is the per-sweep global best.

Buffers (HBM, SoA, float64):
  x, v, p   [d][n]   positions / velocities / personal bests (ld = n)
  pval      [n]
  cand      [d + 2]  this shard's best personal best  [f, idx, x...]
  gX        [d]      global best position of the previous barrier
  gbest     [2]      [f, idx] of the global best
  BFGS outputs: x_final [d][n], f_final, grad_norm [n] f64, iterations,
  ls_trials, grad_evals [n] i32, status [n] u8.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Optional

import torch

from . import _capi, _device


# Kernels launched through this module (bench.py reports the count inside its
# timed region as gpu_launches).
LAUNCHES = [0]


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Global index range [lo, hi) owned by ``rank`` of ``world``
    (contiguous blocks of ceil(n / world))."""
    per = -(-n // world)
    lo = min(n, rank * per)
    hi = min(n, lo + per)
    return lo, hi


@dataclass
class BfgsBuffers:
    x_final: torch.Tensor
    f_final: torch.Tensor
    grad_norm: torch.Tensor
    iterations: torch.Tensor
    status: torch.Tensor
    ls_trials: torch.Tensor
    grad_evals: torch.Tensor

    @classmethod
    def allocate(cls, d: int, n: int, device) -> "BfgsBuffers":
        f64 = torch.float64
        return cls(
            x_final=torch.empty((d, max(n, 1)), dtype=f64, device=device),
            f_final=torch.empty(max(n, 1), dtype=f64, device=device),
            grad_norm=torch.empty(max(n, 1), dtype=f64, device=device),
            iterations=torch.empty(max(n, 1), dtype=torch.int32, device=device),
            status=torch.empty(max(n, 1), dtype=torch.uint8, device=device),
            ls_trials=torch.empty(max(n, 1), dtype=torch.int32, device=device),
            grad_evals=torch.empty(max(n, 1), dtype=torch.int32, device=device),
        )

    # optional host-ready rows (zeus_bfgs_out.rows / irows): device addresses
    # of [n][ld_rows] f64 and [n][4] i32 tables, set by zeus_run
    rows: Optional[tuple] = None

    def c_struct(self, n: int, lo: int = 0) -> _capi.BfgsOut:
        """The C view of starts [lo, lo + n) (same row stride)."""
        rows_ptr, ld_rows, irows_ptr = self.rows or (None, 0, None)
        return _capi.BfgsOut(
            x_final=self.x_final.data_ptr() + 8 * lo, ld_out=self.x_final.shape[1],
            f_final=self.f_final.data_ptr() + 8 * lo,
            grad_norm=self.grad_norm.data_ptr() + 8 * lo,
            iterations=self.iterations.data_ptr() + 4 * lo, status=self.status.data_ptr() + lo,
            ls_trials=self.ls_trials.data_ptr() + 4 * lo,
            grad_evals=self.grad_evals.data_ptr() + 4 * lo,
            rows=rows_ptr + 8 * lo * ld_rows if rows_ptr else None, ld_rows=ld_rows,
            irows=irows_ptr + 16 * lo if irows_ptr else None)


def bfgs_params(theta: float, iter_bfgs: int, ls) -> _capi.BfgsParams:
    return _capi.BfgsParams(theta=float(theta), iter_bfgs=int(iter_bfgs), iter_ls=int(ls.iter_ls),
                            c1_armijo=float(ls.c1_armijo), alpha0=float(ls.alpha0),
                            shrink=float(ls.shrink))


def run_bfgs(obj: int, x0: torch.Tensor, params: _capi.BfgsParams, out: BfgsBuffers,
             device, required_c: int = 0, stop=None,
             ws: Optional[torch.Tensor] = None, wave: int = 0) -> None:
    """Multistart BFGS over the SoA starts ``x0`` [d][n] (bfgs.py:80-156).
    ``stop`` = (counter, flag) as tensors or raw device addresses (the
    cross-process StopBlock).

    ``wave`` > 0 (parallel early stop, driver.py:153-202): the starts run in
    consecutive launches of wave, 2 wave, 4 wave, ... starts, like the
    reference's pool that starts a run only when a worker frees up: once the
    stop flag is set, the starts of later launches end at their first probe
    -- status stopped, iterations 0, grad_norm inf, f_final = f(x0), the
    reference's never-started outcome -- instead of all N running at once."""
    d, n = x0.shape
    if n == 0:
        return
    if stop is not None and 0 < wave < n:
        if ws is None:
            ws = _device.workspace(_capi.lib().zeus_bfgs_workspace_bytes(d, n)
                                   if isinstance(obj, int) else
                                   _capi.lib().zeus_user_bfgs_workspace_bytes(), device)
        lo, size = 0, wave
        while lo < n:
            m = min(size, n - lo)
            _run_bfgs_slice(obj, x0, params, out, device, required_c, stop, ws, lo, m)
            lo += m
            size *= 2
        return
    _run_bfgs_slice(obj, x0, params, out, device, required_c, stop, ws, 0, n)


def _run_bfgs_slice(obj, x0, params, out, device, required_c, stop, ws, lo, n):
    d = x0.shape[0]
    xs = x0.narrow(1, lo, n)
    L = _capi.lib()
    counter = flag = None
    if stop is not None:
        counter, flag = (v if isinstance(v, int) else v.data_ptr() for v in stop)
    if not isinstance(obj, int):  # user objective (plugin.DeviceObjective)
        if ws is None:
            ws = _device.workspace(L.zeus_user_bfgs_workspace_bytes(), device)
        sp = _device.stream_ptr(device)
        obj.bind(sp)
        _capi.check(L.zeus_user_bfgs(obj.handle, n, xs.data_ptr(), xs.stride(0), params,
                                     int(required_c), counter, flag, out.c_struct(n, lo),
                                     ws.data_ptr(), sp), "bfgs (user objective)")
        LAUNCHES[0] += 1
        return
    if ws is None:
        ws = _device.workspace(L.zeus_bfgs_workspace_bytes(d, n), device)
    _capi.check(L.zeus_bfgs(obj, d, n, xs.data_ptr(), xs.stride(0), params, int(required_c),
                            counter, flag, out.c_struct(n, lo), ws.data_ptr(),
                            _device.stream_ptr(device)), "bfgs")
    # small d: thread-per-start tier, warp-per-start tier for starts still
    # running at k1t, CTA-team tier for those still running at k1 (bfgs.cu)
    if d <= 16:
        k1 = int(os.environ.get("ZEUS_K1", "48"))
        k1t = int(os.environ.get("ZEUS_K1T", "0" if d <= 4 else "16"))
        thread = os.environ.get("ZEUS_NO_THREAD", "0") in ("", "0")
        warp = not thread or (k1t > 0 and params.iter_bfgs > k1t)
        LAUNCHES[0] += int(thread) + int(warp) + int(warp and k1 > 0 and params.iter_bfgs > k1)
    else:
        LAUNCHES[0] += 1


class SwarmShard:
    """PSO state of one shard on one device (pso.py:47-70 SwarmState, SoA)."""

    def __init__(self, obj: int, d: int, n: int, i0: int, seed: int, device):
        self.obj, self.d, self.n, self.i0 = obj, d, n, i0
        self.seed = int(seed) & (2**64 - 1)
        self.device = device
        f64 = torch.float64
        self.x = torch.empty((d, n), dtype=f64, device=device)
        self.v = torch.empty((d, n), dtype=f64, device=device)
        self.p = torch.empty((d, n), dtype=f64, device=device)
        self.pval = torch.empty(n, dtype=f64, device=device)
        self.cand = torch.empty(d + 2, dtype=f64, device=device)
        self.gX = torch.empty(d, dtype=f64, device=device)
        self.gbest = torch.empty(2, dtype=f64, device=device)
        self.ws = _device.workspace(_capi.lib().zeus_pso_workspace_bytes(n), device)
        self.sweeps_done = 0

    def _stream(self) -> int:
        return _device.stream_ptr(self.device)

    def init(self, lower: float, upper: float) -> None:
        """init_swarm (pso.py:79-120) for this shard."""
        L = _capi.lib()
        tail = (self.n, self.i0, self.seed, float(lower), float(upper), self.x.data_ptr(),
                self.v.data_ptr(), self.p.data_ptr(), self.pval.data_ptr(), self.n,
                self.cand.data_ptr(), self.ws.data_ptr(), self._stream())
        if isinstance(self.obj, int):
            _capi.check(L.zeus_pso_init(self.obj, self.d, *tail), "pso_init")
        else:
            self.obj.bind(self._stream())
            _capi.check(L.zeus_user_pso_init(self.obj.handle, *tail), "pso_init (user)")
        LAUNCHES[0] += 2
        self.sweeps_done = 0

    def sweep(self, w: float, c1: float, c2: float) -> None:
        """One update_swarm sweep (pso.py:123-164) using gX of the previous barrier."""
        tail = (self.n, self.i0, self.seed, self.sweeps_done, float(w), float(c1), float(c2),
                self.x.data_ptr(), self.v.data_ptr(), self.p.data_ptr(), self.pval.data_ptr(),
                self.n, self.gX.data_ptr(), self.cand.data_ptr(), self.ws.data_ptr(),
                self._stream())
        if isinstance(self.obj, int):
            _capi.check(_capi.lib().zeus_pso_sweep(self.obj, self.d, *tail), "pso_sweep")
        else:
            _capi.check(_capi.lib().zeus_user_pso_sweep(self.obj.handle, *tail),
                        "pso_sweep (user)")
        LAUNCHES[0] += 2
        self.sweeps_done += 1

    def _fused(self, n: int, lower: float, upper: float, w: float, c1: float, c2: float,
               iter_pso: int, xg: "PsoExchange | None") -> None:
        L = _capi.lib()
        common = (int(n), self.i0, self.seed, float(lower), float(upper), float(w), float(c1),
                  float(c2), int(iter_pso), self.x.data_ptr(), self.v.data_ptr(),
                  self.p.data_ptr(), self.pval.data_ptr(), self.n, self.cand.data_ptr(),
                  self.gX.data_ptr(), self.gbest.data_ptr(), self.ws.data_ptr())
        xargs = (xg.block, xg.world, xg.seq) if xg is not None else (None, 1, 1)
        if not isinstance(self.obj, int):
            self.obj.bind(self._stream())
            _capi.check(L.zeus_user_pso_run(self.obj.handle, *common, *xargs, self._stream()),
                        "pso_run (user)")
        elif xg is not None:
            _capi.check(L.zeus_pso_run_xchg(self.obj, self.d, *common, *xargs, self._stream()),
                        "pso_run_xchg")
        else:
            _capi.check(L.zeus_pso_run(self.obj, self.d, *common, self._stream()), "pso_run")
        if xg is not None:
            xg.seq += int(iter_pso) + 1
        LAUNCHES[0] += 1 + int(iter_pso)
        self.sweeps_done = int(iter_pso)

    def run_local(self, lower: float, upper: float, w: float, c1: float, c2: float,
                  iter_pso: int) -> None:
        """init + iter_pso sweeps + the barrier after each, when this shard is
        the whole swarm (one GPU): one fused launch per sweep (zeus_pso_run)."""
        self._fused(self.n, lower, upper, w, c1, c2, iter_pso, None)

    def run_xchg(self, xg: "PsoExchange", n: int, lower: float, upper: float, w: float,
                 c1: float, c2: float, iter_pso: int) -> None:
        """init + iter_pso sweeps of this rank's shard (n real starts, may be
        0) with the cross-GPU barrier fused into every launch (peer-memory
        exchange, zeus_pso_run_xchg): same results as init/sweep + an
        all-gather + select, without a collective launch per sweep."""
        self._fused(n, lower, upper, w, c1, c2, iter_pso, xg)

    def select(self, cands: torch.Tensor, ncand: int) -> None:
        """Global best across shard candidates (np.argmin order, pso.py:73-76)."""
        _capi.check(_capi.lib().zeus_minloc_select(
            self.d, ncand, cands.data_ptr(), self.gX.data_ptr(), self.gbest.data_ptr(),
            self._stream()), "minloc_select")
        LAUNCHES[0] += 1


Barrier = Callable[[SwarmShard], None]


def local_barrier(shard: SwarmShard) -> None:
    """Single-shard barrier: the shard's candidate is the global best."""
    shard.select(shard.cand, 1)


def _host_backend(group) -> bool:
    """gloo (CPU tests, or several processes sharing one GPU) moves CUDA
    tensors through host memory; NCCL collectives run on device."""
    import torch.distributed as dist

    return dist.get_backend(group) == "gloo"


def all_gather_flat(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather equal-size 1-D shards: [world * len(t)] in rank order."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    src = t.contiguous()
    if _host_backend(group) and src.is_cuda:
        out = torch.empty(world * src.numel(), dtype=src.dtype)
        dist.all_gather_into_tensor(out, src.cpu(), group=group)
        return out.to(src.device)
    out = torch.empty(world * src.numel(), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return out


def gather_root_flat(t: torch.Tensor, group=None):
    """Gather equal-size 1-D shards to group rank 0 only: rank 0 gets
    [world * len(t)] in rank order, the other ranks None (one collective,
    no redundant copies of the whole table on every rank)."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dst = dist.get_global_rank(group, 0) if group is not None else 0
    src = t.contiguous()
    host = _host_backend(group) and src.is_cuda
    if host:
        src = src.cpu()
    parts = [torch.empty_like(src) for _ in range(world)] if rank == 0 else None
    dist.gather(src, parts, dst=dst, group=group)
    if rank != 0:
        return None
    out = torch.cat(parts)
    return out.to(t.device) if host else out


def all_reduce_sum(t: torch.Tensor, group=None) -> None:
    """In-place sum over ranks (status tallies)."""
    import torch.distributed as dist

    if _host_backend(group) and t.is_cuda:
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)


def gather_candidates(cand: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather each shard's candidate vector (any device / backend):
    returns [world * len(cand)] in rank order."""
    return all_gather_flat(cand, group)


class StopBlock:
    """The early-stop counter and flag shared by every rank of a process
    group (driver.py:137-202: the pool's Value('q') counter and Value('i')
    flag).  Group rank 0 allocates 64 B of its device memory and exports a
    CUDA IPC handle; the other ranks map it (peer access over NVLink, or the
    same device when several processes share one GPU).  The BFGS kernels bump
    the counter with system-scope atomics and poll the flag with volatile
    loads, so a convergence on any GPU stops every GPU.  One block per
    (group, device), kept for the life of the process."""

    _cache: dict = {}

    def __init__(self, ptr: int, owner: bool):
        self.ptr, self.owner = ptr, owner

    @property
    def counter(self) -> int:
        return self.ptr

    @property
    def flag(self) -> int:
        return self.ptr + 8

    @classmethod
    def get(cls, group, device) -> "StopBlock":
        import ctypes

        import torch.distributed as dist

        key = (id(group), device.index)
        blk = cls._cache.get(key)
        if blk is not None:
            return blk
        L = _capi.lib()
        rank = dist.get_rank(group)
        src = dist.get_global_rank(group, 0) if group is not None else 0
        handle = ctypes.create_string_buffer(64)
        ptr = ctypes.c_void_p()
        ok = True
        if rank == 0:
            ok = L.zeus_stop_block_create(ctypes.byref(ptr), handle) == 0
        box = [bytes(handle.raw) if (rank == 0 and ok) else None]
        dist.broadcast_object_list(box, src=src, group=group)
        if rank != 0:
            ok = box[0] is not None and L.zeus_stop_block_open(box[0], ctypes.byref(ptr)) == 0
        # agreed outcome: a rank that cannot map the block must not leave the
        # others waiting in arm()'s barriers -- every rank raises together
        votes = [None] * dist.get_world_size(group)
        dist.all_gather_object(votes, bool(ok), group=group)
        if not all(votes):
            why = L.zeus_last_error().decode(errors="replace") if not ok else "a peer rank failed"
            if ok and ptr.value:
                L.zeus_stop_block_close(ptr.value, int(rank == 0))
            raise RuntimeError(
                "cross-GPU early stop (workers > 0, required_c < N) needs every rank to map "
                f"rank 0's stop block over CUDA IPC / peer access ({why}); run with "
                "workers=0 (sequential semantics, exact) or deterministic=True")
        blk = cls(int(ptr.value), rank == 0)
        cls._cache[key] = blk
        return blk

    @classmethod
    def local(cls, devices) -> "StopBlock":
        """The stop block of a single-process multi-GPU run: 64 B on the
        first device, reached from the others through peer access."""
        import ctypes

        key = ("local", tuple(int(v.index) for v in devices))
        blk = cls._cache.get(key)
        if blk is not None:
            return blk
        L = _capi.lib()
        idx = sorted({int(v.index) for v in devices})
        for a in idx:
            _capi.check(L.zeus_enable_peer_access(a, int(devices[0].index)), "peer access")
        ptr, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
        with torch.cuda.device(devices[0]):
            _capi.check(L.zeus_stop_block_create(ctypes.byref(ptr), handle), "stop block create")
        blk = cls(int(ptr.value), True)
        cls._cache[key] = blk
        return blk

    def reset_now(self, device) -> None:
        """Zero counter and flag before any shard launches (single process)."""
        stream = torch.cuda.current_stream(device)
        _capi.check(_capi.lib().zeus_stop_block_reset(self.ptr, stream.cuda_stream),
                    "stop block reset")
        stream.synchronize()

    def arm(self, group, device) -> None:
        """Zero counter and flag once no rank still runs a previous call's
        kernel, and before any rank launches the next one."""
        import torch.distributed as dist

        dist.barrier(group=group)
        if self.owner:
            stream = torch.cuda.current_stream(device)
            _capi.check(_capi.lib().zeus_stop_block_reset(self.ptr, stream.cuda_stream),
                        "stop block reset")
            stream.synchronize()
        dist.barrier(group=group)


class PsoExchange:
    """The per-sweep global-best exchange of a multi-GPU PSO phase, done over
    peer memory inside the sweep kernels (csrc/pso_kernels.cuh xchg_barrier;
    the reference's per-sweep reduction across shards, pso.py:73-76).  Every
    rank allocates its exchange block (own cudaMalloc), the IPC handles are
    all-gathered once, each rank maps its peers' blocks (NVLink/NVSwitch peer
    access) and uploads the descriptor.  ``seq`` numbers the exchanges; all
    ranks advance it identically (iter_pso + 1 per PSO phase).  One exchange
    per (group, device, d), kept for the life of the process."""

    _cache: dict = {}

    def __init__(self, block: int, d: int, rank: int, world: int, opened=()):
        self.block, self.d, self.rank, self.world = block, d, rank, world
        self.opened = list(opened)
        self.seq = 1

    @classmethod
    def get(cls, group, device, d: int) -> "PsoExchange | None":
        """The group's exchange for dimension d, or None on EVERY rank when
        any rank cannot map its peers' blocks (the caller then uses the
        collective barrier; the decision is agreed, so no rank waits on an
        exchange the others skip)."""
        import ctypes
        import logging

        import torch.distributed as dist

        key = (id(group), device.index, d)
        if key in cls._cache:
            return cls._cache[key]
        L = _capi.lib()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        nbytes = L.zeus_pso_xchg_bytes(d, world)
        handle = ctypes.create_string_buffer(64)
        mine = ctypes.c_void_p()
        ok = nbytes > 0 and L.zeus_ipc_alloc(nbytes, ctypes.byref(mine), handle) == 0
        handles = [None] * world
        dist.all_gather_object(handles, bytes(handle.raw) if ok else None, group=group)
        bases, opened = [], []
        ok = ok and all(h is not None for h in handles)
        for q in range(world):
            if not ok:
                break
            if q == rank:
                bases.append(int(mine.value))
                continue
            ptr = ctypes.c_void_p()
            if L.zeus_ipc_open(handles[q], ctypes.byref(ptr)) != 0:
                ok = False
                break
            bases.append(int(ptr.value))
            opened.append(int(ptr.value))
        xg = None
        if ok:
            xg = cls(int(mine.value), d, rank, world, opened)
            ok = L.zeus_pso_xchg_setup(xg.block, d, rank, world,
                                       (ctypes.c_void_p * world)(*bases),
                                       _device.stream_ptr(device)) == 0
        votes = [None] * world
        dist.all_gather_object(votes, bool(ok), group=group)  # also: every block zeroed
        if not all(votes):
            for p in opened:
                L.zeus_ipc_close(p, 0)
            if mine.value:
                L.zeus_ipc_close(mine.value, 1)
            logging.getLogger(__name__).warning(
                "peer-memory PSO exchange unavailable (%s); using the collective barrier",
                L.zeus_last_error().decode(errors="replace") if not ok else "a peer rank failed")
            xg = None
        cls._cache[key] = xg
        return xg

    @classmethod
    def local(cls, devices, d: int) -> list:
        """One exchange per shard of a SINGLE-process multi-GPU run (one shard
        per entry of ``devices``; a device may repeat, its shards then run on
        separate streams): every block lives on its shard's device and is
        addressed directly -- peer access enabled between every pair of
        distinct devices, no IPC.  Cached per (devices, d)."""
        import ctypes

        key = ("local", tuple(int(v.index) for v in devices), d)
        if key in cls._cache:
            return cls._cache[key]
        L = _capi.lib()
        world = len(devices)
        nbytes = L.zeus_pso_xchg_bytes(d, world)
        if nbytes == 0:
            raise ValueError(f"the PSO exchange supports 1..8 shards, not {world}")
        idx = sorted({int(v.index) for v in devices})
        for a in idx:
            for b in idx:
                _capi.check(L.zeus_enable_peer_access(a, b), f"peer access {a} -> {b}")
        blocks = []
        for dev in devices:
            ptr, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
            with torch.cuda.device(dev):
                _capi.check(L.zeus_ipc_alloc(nbytes, ctypes.byref(ptr), handle),
                            "exchange alloc")
            blocks.append(int(ptr.value))
        out = [cls(blocks[r], d, r, world) for r in range(world)]
        for xg, dev in zip(out, devices):
            with torch.cuda.device(dev):
                xg._setup(blocks, dev)
        cls._cache[key] = out
        return out

    @classmethod
    def emulated(cls, device, d: int, world: int) -> list:
        """``world`` fresh exchanges on ONE device (tests of the kernel
        protocol: each shard on its own stream)."""
        key = ("local", (int(device.index),) * world, d)
        cls._cache.pop(key, None)
        return cls.local([device] * world, d)

    def _setup(self, bases, device) -> None:
        import ctypes

        arr = (ctypes.c_void_p * self.world)(*bases)
        _capi.check(_capi.lib().zeus_pso_xchg_setup(self.block, self.d, self.rank, self.world,
                                                    arr, _device.stream_ptr(device)),
                    "pso exchange setup")

    def check(self) -> None:
        """Raise if a peer never arrived at an exchange (the kernel's 20 s
        bound; the swarm results of that call are invalid)."""
        import ctypes

        flag = ctypes.c_uint(0)
        _capi.check(_capi.lib().zeus_pso_xchg_status(self.block, self.d, self.world,
                                                     ctypes.byref(flag)), "pso exchange status")
        if flag.value:
            raise RuntimeError("multi-GPU PSO exchange timed out: a peer rank did not arrive")


def resolve_minloc(pairs) -> int:
    """np.argmin order over gathered (f, global_idx) pairs, idx < 0 = empty
    shard: the first NaN wins, else the smallest f, ties to the lowest index.
    Returns the winning global index or -1.  (Host mirror of the device rule
    in csrc/zeus_common.cuh argmin_better, used for the final `best`.)"""
    import math

    best_f, best_i = 0.0, -1
    for f, i in pairs:
        i = int(i)
        if i < 0:
            continue
        if best_i < 0:
            best_f, best_i = f, i
            continue
        fn, bn = math.isnan(f), math.isnan(best_f)
        if fn or bn:
            if (fn and bn and i < best_i) or (fn and not bn):
                best_f, best_i = f, i
        elif f < best_f or (f == best_f and i < best_i):
            best_f, best_i = f, i
    return best_i


def make_dist_barrier(group=None) -> Barrier:
    """Multi-GPU barrier: all-gather every shard's [f, idx, x] candidate over
    NCCL (one collective per sweep) and select the np.argmin winner on device."""
    import torch.distributed as dist

    world = dist.get_world_size(group)

    def barrier(shard: SwarmShard) -> None:
        shard.select(gather_candidates(shard.cand, group), world)

    return barrier
