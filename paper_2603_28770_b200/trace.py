"""Python objectives on the device: trace a generic-scalar callable into
device source (the reference's objective contract, pkg/README.md:70-87).

The reference evaluates any Python callable ``f(x: list) -> scalar`` written
once over floats and ``Dual`` numbers (zeus/autodiff.py) -- arithmetic plus
the helpers ``exp, cos, sin, sqrt, log, powf``.  Kernels cannot run Python,
so instead of a CPU fallback such a callable is run ONCE on symbolic scalars:
every arithmetic operation it performs on a coordinate (in Python's own
evaluation order, constants folded exactly as Python folds them) becomes one
node of an expression DAG, and the DAG is emitted as the straight-line
``objective<T, X>`` of a DeviceObjective (csrc/user_objective.cuh), compiled
with NVRTC for sm_100a (-fmad=false: one IEEE rounding per Python operation,
like CPython floats).  The same source then runs on doubles for values and on
Dual numbers for gradients, with the reference's DomainError loci
(division by zero, sqrt / log / pow domains) mapped to ``err``.

What cannot be traced raises ``TraceError`` (a NotImplementedError): control
flow that depends on a coordinate's value (``if x[0] > 0``, ``math.isfinite``
of a traced value, ``float(x[i])``) and calls into ``math`` on traced values
(use the zeus.autodiff helpers, as the reference's contract asks).  Side
effects run once, at trace time.
"""

from __future__ import annotations

import math
from typing import Callable, Sequence

__all__ = ["Sym", "TraceError", "trace_source", "traced_objective"]


class TraceError(NotImplementedError):
    """The callable cannot be compiled for the device by tracing."""


class Sym:
    """A traced scalar: one node of the objective's expression DAG."""

    __slots__ = ("op", "args", "value", "uid")
    _next = 0

    def __init__(self, op: str, args=(), value=None):
        self.op, self.args, self.value = op, tuple(args), value
        Sym._next += 1
        self.uid = Sym._next

    # ---- arithmetic (Python evaluation order is the emission order) --------
    def __add__(self, o):
        return _bin("+", self, o)

    def __radd__(self, o):
        return _bin("+", o, self)

    def __sub__(self, o):
        return _bin("-", self, o)

    def __rsub__(self, o):
        return _bin("-", o, self)

    def __mul__(self, o):
        return _bin("*", self, o)

    def __rmul__(self, o):
        return _bin("*", o, self)

    def __truediv__(self, o):
        return _bin("/", self, o)

    def __rtruediv__(self, o):
        return _bin("/", o, self)

    def __pow__(self, o):
        return _bin("pow", self, o)

    def __rpow__(self, o):
        return _bin("pow", o, self)

    def __neg__(self):
        return Sym("neg", (self,))

    def __pos__(self):
        return self

    # ---- what a straight-line program cannot express ----------------------
    def _branch(self, *_):
        raise TraceError("the objective branches on (or converts) a coordinate-dependent "
                         "value; device objectives are traced as straight-line code")

    __lt__ = __le__ = __gt__ = __ge__ = __bool__ = __float__ = __int__ = __index__ = _branch
    __abs__ = __round__ = __floor__ = __ceil__ = __mod__ = __floordiv__ = _branch

    def __eq__(self, o):  # identity only (containers, caches); no value semantics
        if isinstance(o, Sym):
            return self is o
        self._branch()

    __hash__ = object.__hash__

    def __repr__(self):
        return f"Sym({self.op}#{self.uid})"


def _num(v):
    if isinstance(v, Sym):
        return v
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        try:
            import numpy as np

            if isinstance(v, np.floating | np.integer):
                return Sym("const", value=float(v))
        except ImportError:  # pragma: no cover
            pass
        raise TraceError(f"unsupported operand {type(v).__name__} in a traced objective")
    return Sym("const", value=float(v))


def _bin(op, a, b):
    return Sym(op, (_num(a), _num(b)))


def unary(name: str, x):
    """exp / cos / sin / sqrt / log of a traced value (zeus.autodiff helpers)."""
    return Sym(name, (_num(x),))


def finite_check(x):
    """x, raising the device ``err`` (-> DomainError) when its value is not
    finite (fitting.py:112-117's non-finite prediction check)."""
    return Sym("finite", (_num(x),)) if isinstance(x, Sym) else x


def _lit(v: float) -> str:
    if math.isnan(v):
        return "__longlong_as_double(0x7ff8000000000000LL)"
    if math.isinf(v):
        return "__longlong_as_double(0x%016xLL)" % (0x7FF0000000000000 | (1 << 63 if v < 0 else 0))
    return f"{v.hex()}"  # exact C++17 hexadecimal floating literal


def coordinates(dim: int) -> list:
    """The traced coordinates x(0) .. x(dim - 1)."""
    return [Sym("x", value=i) for i in range(dim)]


def trace_source(f: Callable[[Sequence], object], dim: int, name: str = "traced") -> str:
    """Device source of ``f`` at dimension ``dim`` (raises TraceError)."""
    try:
        out = f(coordinates(dim))
    except TraceError:
        raise
    except (TypeError, ValueError, AttributeError) as e:
        raise TraceError(f"{name}: tracing failed ({type(e).__name__}: {e})") from None
    return source_of(out, dim, name)


def source_of(out, dim: int, name: str = "traced") -> str:
    """Straight-line device source computing the traced value ``out``."""
    if isinstance(out, Sym):
        root = out
    else:
        try:
            root = _num(out)
        except TraceError:
            raise TraceError(f"{name}: returned {type(out).__name__}, not a scalar") from None
    lines, names = [], {}

    def emit(n: Sym) -> str:
        stack = [(n, False)]
        while stack:
            node, ready = stack.pop()
            if node.uid in names:
                continue
            if node.op == "const":
                # a plain double: Dual (op) double follows the reference's
                # scalar rules (autodiff.py: Dual * float -> (r c, d c)), not
                # the Dual (op) Dual ones
                names[node.uid] = _lit(node.value)
                continue
            if node.op == "x":
                v = f"v{len(lines)}"
                lines.append(f"  const T {v} = x({node.value});")
                names[node.uid] = v
                continue
            if not ready:
                stack.append((node, True))
                for a in reversed(node.args):
                    if a.uid not in names:
                        stack.append((a, False))
                continue
            a = [names[x.uid] for x in node.args]
            if node.op in "+-*":
                e = f"{a[0]} {node.op} {a[1]}"
            elif node.op == "/":
                e = f"zu::div({a[0]}, {a[1]}, err)"
            elif node.op == "pow":
                e = f"zu::pow({a[0]}, {a[1]}, err)"
            elif node.op == "neg":
                e = f"-{a[0]}"
            elif node.op in ("sqrt", "log"):
                e = f"zu::{node.op}({a[0]}, err)"
            elif node.op == "finite":
                lines.append(f"  if (!isfinite(zeus::real_of({a[0]}))) err = true;")
                names[node.uid] = a[0]
                continue
            else:  # exp, cos, sin
                e = f"zu::{node.op}({a[0]})"
            v = f"v{len(lines)}"
            lines.append(f"  const T {v} = {e};")
            names[node.uid] = v
        return names[n.uid]

    ret = emit(root)
    body = "\n".join(lines)
    return (f"// traced from Python callable {name!r} at dim {dim} "
            f"({len(lines)} operations, Python evaluation order)\n"
            "template <class T, class X>\n"
            "__device__ T objective(const X& x, int d, const double* data, bool& err) {\n"
            f"{body}\n  return {ret};\n}}\n")


_TRACED: dict = {}


def traced_objective(f: Callable[[Sequence], object], dim: int, device=None):
    """The DeviceObjective compiled from ``f`` at ``dim`` (cached per
    callable, dimension and device)."""
    from . import _device
    from .plugin import DeviceObjective

    dev = _device.require_device(device)
    key = (id(f), dim, dev.index)
    hit = _TRACED.get(key)
    if hit is not None and hit[0] is f:
        return hit[1]
    name = getattr(f, "__name__", "objective")
    obj = DeviceObjective(trace_source(f, dim, name), dim=dim, name=name, device=dev)
    _TRACED[key] = (f, obj)
    return obj
