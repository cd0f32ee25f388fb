"""Quasi-Newton local minimisation (bfgs.py of the reference) on the device.

``bfgs_run`` and ``hessian_update`` keep the reference signatures and
semantics; both run on the GPU (csrc/bfgs.cu, csrc/blocks.cu).  Inside
``zeus_run`` one persistent kernel runs every start (see engine.run_bfgs).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _capi, _device, engine
from .linesearch import LineSearchParams
from .objectives import objective_id

__all__ = [
    "CONVERGED",
    "DIVERGED",
    "STOPPED",
    "DOMAIN_ERROR",
    "STATUSES",
    "CURVATURE_FLOOR",
    "BfgsOutcome",
    "hessian_update",
    "bfgs_run",
]

CONVERGED = "converged"
DIVERGED = "diverged"
STOPPED = "stopped"
DOMAIN_ERROR = "domain_error"
STATUSES = (CONVERGED, DIVERGED, STOPPED, DOMAIN_ERROR)  # index == device status code

CURVATURE_FLOOR = 1e-12  # bfgs.py:40


@dataclass(frozen=True)
class BfgsOutcome:
    """Terminal state of one local minimisation (bfgs.py:43-56)."""

    x_final: tuple[float, ...]
    f_final: float
    grad_norm: float
    iterations: int
    status: str


def hessian_update(H: np.ndarray, dx: np.ndarray, dg: np.ndarray) -> np.ndarray:
    """Rank-two inverse-Hessian update (bfgs.py:59-77) on the device.

    Returns ``H`` itself (the same object) when the curvature guard
    ``dx.dg <= 1e-12 |dx| |dg|`` skips the update; inputs are never mutated.
    """
    Hn = np.asarray(H, dtype=np.float64)
    dxn = np.asarray(dx, dtype=np.float64).ravel()
    dgn = np.asarray(dg, dtype=np.float64).ravel()
    d = dxn.shape[0]
    dev = _device.require_device()
    Ht = torch.from_numpy(np.ascontiguousarray(Hn).copy()).to(dev)
    a = torch.from_numpy(dxn.copy()).to(dev)
    b = torch.from_numpy(dgn.copy()).to(dev)
    upd = torch.empty(1, dtype=torch.uint8, device=dev)
    _capi.check(_capi.lib().zeus_hessian_update(d, 1, Ht.data_ptr(), a.data_ptr(), b.data_ptr(),
                                                upd.data_ptr(), _device.stream_ptr(dev)),
                "hessian_update")
    if not bool(upd.item()):
        return H
    return Ht.cpu().numpy()


def _single(obj: int, x0: np.ndarray, theta: float, iter_bfgs: int, ls: LineSearchParams,
            dev) -> BfgsOutcome:
    d = x0.shape[0]
    xs = torch.from_numpy(x0.reshape(d, 1).copy()).to(dev)
    out = engine.BfgsBuffers.allocate(d, 1, dev)
    engine.run_bfgs(obj, xs, engine.bfgs_params(theta, iter_bfgs, ls), out, dev)
    return BfgsOutcome(
        x_final=tuple(out.x_final[:, 0].cpu().tolist()),
        f_final=float(out.f_final[0].item()),
        grad_norm=float(out.grad_norm[0].item()),
        iterations=int(out.iterations[0].item()),
        status=STATUSES[int(out.status[0].item())],
    )


def bfgs_run(
    f: Callable[[Sequence], object],
    x0: Sequence[float],
    theta: float,
    iter_bfgs: int,
    ls: LineSearchParams | None = None,
    stop_probe: Optional[Callable[[], bool]] = None,
) -> BfgsOutcome:
    """Minimise registered objective ``f`` from ``x0`` (bfgs.py:80-156).

    ``stop_probe`` is read at the top of every iteration, before any gradient
    work, exactly as often as the reference reads it: the device run is
    deterministic, so the run is executed once, the probe is replayed over its
    iteration tops, and if it fires at top ``j`` the state after ``j``
    iterations is reproduced by re-running with the cap set to ``j``.
    """
    if theta <= 0.0:
        raise ValueError("theta must be positive")
    if iter_bfgs < 0:
        raise ValueError("iter_bfgs must be non-negative")
    if ls is None:
        ls = LineSearchParams()
    x = np.asarray(x0, dtype=np.float64).ravel()
    obj = objective_id(f, x.shape[0])
    dev = _device.require_device()
    if not isinstance(obj, int):
        from .driver import check_objective_device

        check_objective_device(obj, dev)
    full = _single(obj, x, theta, iter_bfgs, ls, dev)
    if stop_probe is None:
        return full
    # the reference reads the probe at tops 0..K (K = full.iterations)
    for j in range(full.iterations + 1):
        if stop_probe():
            if j == 0:
                return BfgsOutcome(x_final=tuple(x.tolist()), f_final=_f_at(obj, x, dev),
                                   grad_norm=math.inf, iterations=0, status=STOPPED)
            part = _single(obj, x, theta, j, ls, dev)
            return BfgsOutcome(x_final=part.x_final, f_final=part.f_final,
                               grad_norm=part.grad_norm, iterations=j, status=STOPPED)
    return full


def _f_at(obj, x: np.ndarray, dev) -> float:
    if not isinstance(obj, int):  # user objective
        return float(obj.values(x.reshape(1, -1))[0])
    xs = torch.from_numpy(x.reshape(-1, 1).copy()).to(dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    _capi.check(_capi.lib().zeus_objective_value(obj, x.shape[0], 1, xs.data_ptr(), 1,
                                                 out.data_ptr(), _device.stream_ptr(dev)),
                "objective")
    return float(out.item())
