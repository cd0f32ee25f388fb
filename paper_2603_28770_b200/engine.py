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

    def c_struct(self, n: int) -> _capi.BfgsOut:
        return _capi.BfgsOut(
            x_final=self.x_final.data_ptr(), ld_out=self.x_final.shape[1],
            f_final=self.f_final.data_ptr(), grad_norm=self.grad_norm.data_ptr(),
            iterations=self.iterations.data_ptr(), status=self.status.data_ptr(),
            ls_trials=self.ls_trials.data_ptr(), grad_evals=self.grad_evals.data_ptr())


def bfgs_params(theta: float, iter_bfgs: int, ls) -> _capi.BfgsParams:
    return _capi.BfgsParams(theta=float(theta), iter_bfgs=int(iter_bfgs), iter_ls=int(ls.iter_ls),
                            c1_armijo=float(ls.c1_armijo), alpha0=float(ls.alpha0),
                            shrink=float(ls.shrink))


def run_bfgs(obj: int, x0: torch.Tensor, params: _capi.BfgsParams, out: BfgsBuffers,
             device, required_c: int = 0, stop: Optional[tuple[torch.Tensor, torch.Tensor]] = None,
             ws: Optional[torch.Tensor] = None) -> None:
    """Multistart BFGS over the SoA starts ``x0`` [d][n] (bfgs.py:80-156)."""
    d, n = x0.shape
    if n == 0:
        return
    L = _capi.lib()
    if ws is None:
        ws = _device.workspace(L.zeus_bfgs_workspace_bytes(d, n), device)
    counter = flag = None
    if stop is not None:
        counter, flag = stop[0].data_ptr(), stop[1].data_ptr()
    _capi.check(L.zeus_bfgs(obj, d, n, x0.data_ptr(), x0.stride(0), params, int(required_c),
                            counter, flag, out.c_struct(n), ws.data_ptr(),
                            _device.stream_ptr(device)), "bfgs")
    # small d: warp kernel + the CTA-team kernel for promoted stragglers
    k1 = int(os.environ.get("ZEUS_K1", "48"))
    LAUNCHES[0] += 2 if (d <= 16 and k1 > 0 and params.iter_bfgs > k1) else 1


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
        _capi.check(_capi.lib().zeus_pso_init(
            self.obj, self.d, self.n, self.i0, self.seed, float(lower), float(upper),
            self.x.data_ptr(), self.v.data_ptr(), self.p.data_ptr(), self.pval.data_ptr(),
            self.n, self.cand.data_ptr(), self.ws.data_ptr(), self._stream()), "pso_init")
        LAUNCHES[0] += 2
        self.sweeps_done = 0

    def sweep(self, w: float, c1: float, c2: float) -> None:
        """One update_swarm sweep (pso.py:123-164) using gX of the previous barrier."""
        _capi.check(_capi.lib().zeus_pso_sweep(
            self.obj, self.d, self.n, self.i0, self.seed, self.sweeps_done, float(w), float(c1),
            float(c2), self.x.data_ptr(), self.v.data_ptr(), self.p.data_ptr(),
            self.pval.data_ptr(), self.n, self.gX.data_ptr(), self.cand.data_ptr(),
            self.ws.data_ptr(), self._stream()), "pso_sweep")
        LAUNCHES[0] += 2
        self.sweeps_done += 1

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


def gather_candidates(cand: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather each shard's candidate vector (any device / backend):
    returns [world * len(cand)] in rank order."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    gathered = torch.empty(world * cand.numel(), dtype=cand.dtype, device=cand.device)
    dist.all_gather_into_tensor(gathered, cand.contiguous(), group=group)
    return gathered


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
