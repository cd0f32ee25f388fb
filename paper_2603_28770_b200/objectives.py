"""Objective registry (objectives.py:116-221 of the reference) backed by device
functors.

The four registered functions keep their reference names and call signature
``f(x: Sequence[float]) -> float``; calling one evaluates it on the GPU
(csrc/objectives.cuh), with the reference's operation order.  ``zeus_run`` and
the other drivers never call them: they map the callable to its device
objective id (``objective_id``) and fuse the evaluation into the kernels.
The reference's own functions (``zeus.objectives.rosenbrock`` ...) are accepted
too, so code written against the reference switches by changing the import.
Unregistered Python callables raise -- there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

from . import _capi

__all__ = [
    "ObjectiveSpec",
    "rosenbrock",
    "rastrigin",
    "ackley",
    "goldstein_price",
    "get_objective",
    "objective_names",
    "objective_id",
]


def _evaluate(obj_id: int, x: Sequence[float]) -> float:
    import torch

    from . import _device
    from .autodiff import Dual

    if any(isinstance(v, Dual) for v in x):
        return _evaluate_dual(obj_id, x)
    vals = [float(v) for v in x]
    dev = _device.require_device()
    xs = torch.tensor(vals, dtype=torch.float64, device=dev).reshape(len(vals), 1)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    _capi.check(_capi.lib().zeus_objective_value(obj_id, len(vals), 1, xs.data_ptr(), 1,
                                                 out.data_ptr(), _device.stream_ptr(dev)),
                "objective")
    return float(out.item())


def _evaluate_dual(obj_id: int, x: Sequence) -> object:
    """The objective on Dual numbers (the reference's functions are generic
    over float / Dual, objectives.py:33-113): the real part is the float
    evaluation (bit for bit, as in the reference), the dual part the
    directional derivative grad f . t from the device's forward-mode gradient
    (summed in coordinate order; the reference propagates tangents through
    the expression instead, so it can differ in the last bits).  DomainError
    where the reference's Dual evaluation raises (Ackley's sqrt at sum x^2 = 0,
    autodiff.py:207-213) -- whatever the tangents."""
    import numpy as np

    from .autodiff import DomainError, Dual
    from . import autodiff

    reals = [float(v.real) if isinstance(v, Dual) else float(v) for v in x]
    tans = [float(v.dual) if isinstance(v, Dual) else 0.0 for v in x]
    f = _evaluate(obj_id, reals)
    fn = {_capi.OBJ_ROSENBROCK: rosenbrock, _capi.OBJ_RASTRIGIN: rastrigin,
          _capi.OBJ_ACKLEY: ackley, _capi.OBJ_GOLDSTEIN_PRICE: goldstein_price}[obj_id]
    g, err = autodiff.gradients(fn, np.asarray([reals]))
    if err[0]:
        raise DomainError("the Dual evaluation leaves the domain (autodiff.py:207-216)")
    dual = 0.0
    for gi, ti in zip(g[0].tolist(), tans):
        dual += gi * ti
    return Dual(f, dual)


def rosenbrock(x: Sequence[float]) -> float:
    """sum_{i<n-1} (1 - x_i)^2 + 100 (x_{i+1} - x_i^2)^2 (objectives.py:33-45)."""
    return _evaluate(_capi.OBJ_ROSENBROCK, x)


def rastrigin(x: Sequence[float]) -> float:
    """10 n + sum_i (x_i^2 - 10 cos(2 pi x_i)) (objectives.py:48-61)."""
    return _evaluate(_capi.OBJ_RASTRIGIN, x)


def ackley(x: Sequence[float]) -> float:
    """-20 exp(-0.2 sqrt(mean x^2)) - exp(mean cos 2 pi x) + e + 20 (objectives.py:64-85)."""
    return _evaluate(_capi.OBJ_ACKLEY, x)


def goldstein_price(x: Sequence[float]) -> float:
    """Goldstein-Price, 2-D only (objectives.py:88-113)."""
    if len(x) != 2:
        raise ValueError("goldstein_price is defined for exactly 2 dimensions")
    return _evaluate(_capi.OBJ_GOLDSTEIN_PRICE, x)


@dataclass(frozen=True)
class ObjectiveSpec:
    """A registered objective with its search box and known optimum
    (objectives.py:116-139)."""

    name: str
    fn: Callable[[Sequence], object]
    dim: int
    lower: float
    upper: float
    optimum_x: tuple[float, ...] | None = None
    optimum_f: float | None = None
    gradient_continuous: bool = True

    def __post_init__(self):
        if not self.lower < self.upper:
            raise ValueError("objective range requires lower < upper")
        if self.dim < 1:
            raise ValueError("objective dimension must be >= 1")


# objectives.py:145-182 (boxes, optima, dimension rules)
_REGISTRY: dict[str, dict] = {
    "rosenbrock": dict(fn=rosenbrock, obj_id=_capi.OBJ_ROSENBROCK, min_dim=2, fixed_dim=None,
                       lower=-5.0, upper=5.0, optimum=lambda dim: ((1.0,) * dim, 0.0),
                       gradient_continuous=True),
    "rastrigin": dict(fn=rastrigin, obj_id=_capi.OBJ_RASTRIGIN, min_dim=1, fixed_dim=None,
                      lower=-5.12, upper=5.12, optimum=lambda dim: ((0.0,) * dim, 0.0),
                      gradient_continuous=True),
    "ackley": dict(fn=ackley, obj_id=_capi.OBJ_ACKLEY, min_dim=1, fixed_dim=None,
                   lower=-5.0, upper=5.0, optimum=lambda dim: ((0.0,) * dim, 0.0),
                   gradient_continuous=False),
    "goldstein_price": dict(fn=goldstein_price, obj_id=_capi.OBJ_GOLDSTEIN_PRICE, min_dim=2,
                            fixed_dim=2, lower=-2.0, upper=2.0,
                            optimum=lambda dim: ((0.0, -1.0), 3.0), gradient_continuous=True),
}


def objective_names() -> list[str]:
    """Names accepted by :func:`get_objective` (objectives.py:185-187)."""
    return sorted(_REGISTRY)


def get_objective(name: str, dim: int = 2) -> ObjectiveSpec:
    """Look up a registered objective (objectives.py:190-221).

    Raises KeyError for an unknown name, ValueError for an unsupported dim.
    """
    try:
        entry = _REGISTRY[name]
    except KeyError:
        raise KeyError(
            f"unknown objective {name!r}; known: {', '.join(objective_names())}"
        ) from None
    fixed = entry["fixed_dim"]
    if fixed is not None and dim != fixed:
        raise ValueError(f"{name} is only defined for dim={fixed}")
    if dim < entry["min_dim"]:
        raise ValueError(f"{name} requires dim >= {entry['min_dim']}")
    opt_x, opt_f = entry["optimum"](dim)
    return ObjectiveSpec(name=name, fn=entry["fn"], dim=dim, lower=entry["lower"],
                         upper=entry["upper"], optimum_x=opt_x, optimum_f=opt_f,
                         gradient_continuous=entry["gradient_continuous"])


def objective_id(f, dim: int | None = None):
    """Device objective id of a registered callable (a ``DeviceObjective``
    user plug-in is returned as itself: the engine launches its NVRTC
    module instead of the built-in kernels).

    Accepts this package's functions, ``ObjectiveSpec`` objects, registry
    names, and the reference package's own functions (matched by module and
    name, ``zeus.objectives.<name>``).  Any other callable is a user
    objective: with ``dim`` it is traced into a DeviceObjective (trace.py);
    kernels cannot run Python and there is no CPU fallback.  Goldstein-Price at ``dim != 2`` raises ``ValueError`` like the
    reference's evaluation would (objectives.py:92-93).
    """
    from .plugin import DeviceObjective

    if isinstance(f, ObjectiveSpec) and isinstance(f.fn, DeviceObjective):
        f = f.fn
    if isinstance(f, DeviceObjective):  # user objective: the plugin stands in for the id
        if dim is not None and dim != f.dim:
            raise ValueError(f"{f.name} was compiled for dim={f.dim}, not {dim}")
        return f
    name = None
    if isinstance(f, ObjectiveSpec):
        name = f.name
    elif isinstance(f, str):
        name = f if f in _REGISTRY else None
    else:
        for key, entry in _REGISTRY.items():
            if f is entry["fn"]:
                name = key
                break
        if name is None and getattr(f, "__module__", None) == "zeus.objectives":
            cand = getattr(f, "__name__", None)
            name = cand if cand in _REGISTRY else None
    if name is None:
        if callable(f) and dim is not None:
            # a generic Python objective (pkg/README.md:70-87): traced once into
            # device source and compiled with NVRTC (trace.py); a callable that
            # cannot be traced raises TraceError (a NotImplementedError)
            from .trace import traced_objective

            return traced_objective(f, int(dim))
        raise NotImplementedError(
            f"objective {getattr(f, '__name__', f)!r} is not a registered device objective "
            f"({', '.join(objective_names())}) and no dimension was given to trace it; "
            f"there is no CPU fallback")
    if name == "goldstein_price" and dim is not None and dim != 2:
        raise ValueError("goldstein_price is defined for exactly 2 dimensions")
    return int(_REGISTRY[name]["obj_id"])
