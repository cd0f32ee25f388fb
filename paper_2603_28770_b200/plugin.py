"""User-defined objectives on the GPU path.

The reference accepts any Python callable written against its generic-scalar
contract (pkg/README.md:70-87): the same code runs on floats and on ``Dual``
numbers.  Kernels cannot run Python, so a user objective here is the same
idea written as device source, compiled at run time with NVRTC for sm_100a
together with the framework's own PSO and BFGS kernels
(csrc/plugin.cu, contract in csrc/user_objective.cuh)::

    from paper_2603_28770_b200 import DeviceObjective, ZeusConfig, zeus_run

    f = DeviceObjective('''
    template <class T, class X>
    __device__ T objective(const X& x, int d, const double* data, bool& err) {
      T total = 0.0;
      for (int i = 0; i < d; ++i) total = total + x(i) * x(i) - zu::cos(3.0 * x(i));
      return total;
    }''', dim=4)
    res = zeus_run(f, ZeusConfig(N=4096, dim=4, range=(-3.0, 3.0)))

``zu::cos / sin / exp / sqrt / log / pow / div`` are the zeus.autodiff helpers
(the last four take ``err`` and raise the reference's DomainError cases), and
``data`` is an optional constant array (``data=`` below).  Gradients are
forward-mode: one seeded Dual pass per coordinate, like the reference's
forward_gradient.  ``dim`` <= 128 (BFGS: one thread per start up to 16,
one warp per start above).  A DomainError anywhere in a BFGS run gives the
``domain_error`` status exactly where the reference would.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
from typing import Sequence

import numpy as np

from . import _capi

__all__ = ["DeviceObjective", "MAX_DIM"]

MAX_DIM = 128
CSRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc")
_CACHE: dict = {}  # (device, sha1(source), dim) -> handle


class DeviceObjective:
    """A user objective compiled for the GPU.  Callable like the registered
    objectives (``f(x) -> float``, evaluated on the device) and accepted by
    ``zeus_run`` / ``bfgs_run``."""

    def __init__(self, source: str, dim: int, data: Sequence[float] | None = None,
                 name: str = "user_objective", device=None):
        import torch

        from . import _device

        if not 1 <= int(dim) <= MAX_DIM:
            raise ValueError(f"user objectives support 1 <= dim <= {MAX_DIM}")
        self.source, self.dim, self.name = source, int(dim), name
        self.__name__ = name
        self.device = _device.require_device(device)
        L = _capi.lib()
        key = (self.device.index, hashlib.sha1(source.encode()).hexdigest(), self.dim,
               os.environ.get("ZEUS_USER_WARP", ""))
        handle = _CACHE.get(key)
        if handle is None:
            h = ctypes.c_void_p()
            with torch.cuda.device(self.device):
                rc = L.zeus_user_compile(source.encode(), self.dim, CSRC.encode(),
                                         ctypes.byref(h))
            if rc != 0:
                log = L.zeus_user_compile_log().decode(errors="replace")
                msg = L.zeus_last_error().decode(errors="replace")
                raise ValueError(f"user objective {name!r} does not compile: {msg}\n{log}")
            handle = h.value
            _CACHE[key] = handle
        self.handle = handle
        self.data = None
        if data is not None:
            arr = np.ascontiguousarray(np.asarray(data, dtype=np.float64).ravel())
            self.data = torch.from_numpy(arr).to(self.device)

    def bind(self, stream_ptr: int) -> None:
        """Point the module's `data` at this objective's array (one module may
        serve several DeviceObjective instances with different data)."""
        ptr = self.data.data_ptr() if self.data is not None else None
        _capi.check(_capi.lib().zeus_user_set_data(self.handle, ptr, stream_ptr),
                    "user objective data")

    def values(self, points) -> np.ndarray:
        """f at each row of ``points`` [n][dim] (NaN where it raises)."""
        import torch

        from . import _device

        pts = np.asarray(points, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != self.dim:
            raise ValueError(f"points must have shape (n, {self.dim})")
        n = pts.shape[0]
        x = _device.to_soa(pts, self.device)
        f = torch.empty(max(n, 1), dtype=torch.float64, device=self.device)
        sp = _device.stream_ptr(self.device)
        self.bind(sp)
        _capi.check(_capi.lib().zeus_user_value(self.handle, n, x.data_ptr(), max(n, 1),
                                                f.data_ptr(), sp), "user objective value")
        return f[:n].cpu().numpy()

    def __call__(self, x: Sequence[float]) -> float:
        from .autodiff import DomainError

        v = float(self.values([list(map(float, x))])[0])
        if np.isnan(v):
            raise DomainError(f"{self.name}: evaluation left the domain")
        return v

    def __repr__(self) -> str:
        return f"DeviceObjective({self.name!r}, dim={self.dim})"
