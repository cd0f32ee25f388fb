"""Armijo backtracking line search (linesearch.py of the reference).

``armijo_search`` runs the reference's trial schedule on the device
(csrc/blocks.cu); inside ``zeus_run`` the same search is fused into the BFGS
kernel (csrc/bfgs.cu) and never leaves the SM.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch

from . import _capi, _device
from .objectives import objective_id

__all__ = ["LineSearchParams", "armijo_search"]

log = logging.getLogger(__name__)


@dataclass(frozen=True)
class LineSearchParams:
    """Step-halving schedule and acceptance constant (linesearch.py:16-37)."""

    c1_armijo: float = 0.3
    alpha0: float = 1.0
    iter_ls: int = 20
    shrink: float = 0.5

    def __post_init__(self):
        if not 0.0 < self.c1_armijo < 1.0:
            raise ValueError("c1_armijo must be in (0, 1)")
        if not 0.0 < self.shrink < 1.0:
            raise ValueError("shrink must be in (0, 1)")
        if self.alpha0 <= 0.0:
            raise ValueError("alpha0 must be positive")
        if self.iter_ls < 1:
            raise ValueError("iter_ls must be a positive integer")


def _params(ls: LineSearchParams, theta: float = 1e-6, iter_bfgs: int = 0) -> _capi.BfgsParams:
    return _capi.BfgsParams(theta=theta, iter_bfgs=iter_bfgs, iter_ls=ls.iter_ls,
                            c1_armijo=ls.c1_armijo, alpha0=ls.alpha0, shrink=ls.shrink)


def armijo_search(
    f: Callable[[Sequence[float]], float],
    x: np.ndarray,
    p: np.ndarray,
    g: np.ndarray,
    f0: float,
    params: LineSearchParams,
) -> float:
    """First alpha in alpha0 * shrink**k (k = 0..iter_ls) with
    f(x + alpha p) <= f0 + c1 alpha (g . p); the last trial if none passes
    (linesearch.py:40-71)."""
    x = np.asarray(x, dtype=np.float64)
    p = np.asarray(p, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    d = x.shape[0]
    obj = objective_id(f, d)
    ddir = float(np.dot(g, p))
    if ddir >= 0.0:
        log.debug("line search entered with non-descent direction (g.p=%g)", ddir)
    dev = _device.require_device()
    xs = torch.from_numpy(x.reshape(d, 1).copy()).to(dev)
    ps = torch.from_numpy(p.reshape(d, 1).copy()).to(dev)
    gs = torch.from_numpy(g.reshape(d, 1).copy()).to(dev)
    f0s = torch.tensor([float(f0)], dtype=torch.float64, device=dev)
    alpha = torch.empty(1, dtype=torch.float64, device=dev)
    trials = torch.empty(1, dtype=torch.int32, device=dev)
    P = _params(params)
    sp = _device.stream_ptr(dev)
    if not isinstance(obj, int):  # user objective (plugin.DeviceObjective)
        from .autodiff import DomainError

        obj.bind(sp)
        _capi.check(_capi.lib().zeus_user_armijo(obj.handle, 1, xs.data_ptr(), ps.data_ptr(),
                                                 gs.data_ptr(), 1, f0s.data_ptr(), P,
                                                 alpha.data_ptr(), trials.data_ptr(), sp),
                    "armijo_search (user objective)")
        if int(trials.item()) < 0:  # the reference lets the DomainError propagate
            raise DomainError(f"{obj.name}: evaluation left the domain in the line search")
        return float(alpha.item())
    _capi.check(_capi.lib().zeus_armijo(obj, d, 1, xs.data_ptr(), ps.data_ptr(), gs.data_ptr(),
                                        1, f0s.data_ptr(), P, alpha.data_ptr(),
                                        trials.data_ptr(), sp),
                "armijo_search")
    return float(alpha.item())
