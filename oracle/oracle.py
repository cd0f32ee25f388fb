"""TEST INFRASTRUCTURE ONLY: ctypes wrapper over oracle/liboracle.so.

The CPU restatement of the reference hot path (see zeus_oracle.c).  Imported
only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg, as a
checker / baseline -- never by the product package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

OBJ_IDS = {"rosenbrock": 0, "rastrigin": 1, "ackley": 2, "goldstein_price": 3}
STATUS_NAMES = ("converged", "diverged", "stopped", "domain_error")

_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64


class Outcome(ctypes.Structure):
    _fields_ = [
        ("f_final", ctypes.c_double),
        ("grad_norm", ctypes.c_double),
        ("iterations", ctypes.c_int64),
        ("status", ctypes.c_int64),
        ("ls_trials", ctypes.c_int64),
        ("grad_evals", ctypes.c_int64),
    ]


def build() -> str:
    """Compile liboracle.so with oracle/Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_philox_u64.restype = _u64
        L.oracle_philox_u64.argtypes = [_u64, _u64, _u64]
        L.oracle_draw_uniform.argtypes = [_u64, _u64, _u64, _i64, ctypes.c_double,
                                          ctypes.c_double, _dp]
        L.oracle_objective.restype = ctypes.c_double
        L.oracle_objective.argtypes = [ctypes.c_int, _dp, ctypes.c_int]
        L.oracle_gradient.restype = ctypes.c_int
        L.oracle_gradient.argtypes = [ctypes.c_int, _dp, ctypes.c_int, _dp]
        L.oracle_argmin.restype = _i64
        L.oracle_argmin.argtypes = [_dp, _i64]
        L.oracle_pso_init.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _u64,
                                      ctypes.c_double, ctypes.c_double,
                                      _dp, _dp, _dp, _dp, _dp, _dp]
        L.oracle_pso_sweep.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _u64,
                                       ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, _dp, _dp, _dp, _dp, _dp, _dp]
        L.oracle_armijo.restype = ctypes.c_double
        L.oracle_armijo.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp, _dp,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_int, ctypes.c_double, _dp, _dp,
                                    ctypes.POINTER(ctypes.c_int)]
        L.oracle_hessian_update.restype = ctypes.c_int
        L.oracle_hessian_update.argtypes = [ctypes.c_int, _dp, _dp, _dp]
        L.oracle_bfgs_run.argtypes = [ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double,
                                      ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int, ctypes.c_double,
                                      ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(Outcome), _dp]
        L.oracle_bfgs_batch.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _dp,
                                        ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_int, ctypes.POINTER(Outcome), _dp]
        L.oracle_bfgs_batch_jitter.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _dp,
                                               ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                               ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                               ctypes.c_int, _u64, ctypes.POINTER(Outcome), _dp]
        L.oracle_zeus_run.restype = _i64
        L.oracle_zeus_run.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _u64, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int, ctypes.c_double, ctypes.c_int, _dp, _dp, _dp,
                                      _dp, _dp, _dp, ctypes.POINTER(Outcome), _dp]
        L.oracle_reduce_best.restype = _i64
        L.oracle_reduce_best.argtypes = [ctypes.POINTER(Outcome), _i64]
        _LIB = L
    return _LIB


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _obj(name_or_id) -> int:
    return OBJ_IDS[name_or_id] if isinstance(name_or_id, str) else int(name_or_id)


def philox_u64(seed: int, i: int, k: int) -> int:
    return int(lib().oracle_philox_u64(seed & (2**64 - 1), i, k))


def draw_uniform(seed: int, i: int, k0: int, count: int, low: float, high: float):
    out = np.empty(count)
    lib().oracle_draw_uniform(seed & (2**64 - 1), i, k0, count, low, high, _p(out))
    return out


def objective(obj, x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().oracle_objective(_obj(obj), _p(x), len(x)))


def gradient(obj, x):
    """Returns (grad, domain_error)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    g = np.empty(len(x))
    err = lib().oracle_gradient(_obj(obj), _p(x), len(x), _p(g))
    return g, bool(err)


@dataclass
class Swarm:
    positions: np.ndarray
    velocities: np.ndarray
    personal_best_pos: np.ndarray
    personal_best_val: np.ndarray
    global_best_pos: np.ndarray
    global_best_val: float


def pso(obj, d: int, n: int, seed: int, lower: float, upper: float, sweeps: int,
        w=0.5, c1=1.2, c2=1.5) -> Swarm:
    x = np.empty((n, d)); v = np.empty((n, d)); p = np.empty((n, d))
    pv = np.empty(n); gX = np.empty(d); gF = ctypes.c_double()
    L = lib()
    L.oracle_pso_init(_obj(obj), d, n, seed & (2**64 - 1), lower, upper, _p(x), _p(v),
                      _p(p), _p(pv), _p(gX), ctypes.byref(gF))
    for s in range(sweeps):
        L.oracle_pso_sweep(_obj(obj), d, n, seed & (2**64 - 1), s, w, c1, c2, _p(x),
                           _p(v), _p(p), _p(pv), _p(gX), ctypes.byref(gF))
    return Swarm(x, v, p, pv, gX, gF.value)


def armijo(obj, x, p, g, f0, c1=0.3, alpha0=1.0, iter_ls=20, shrink=0.5):
    x = np.ascontiguousarray(x, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    xt = np.empty(len(x)); ft = ctypes.c_double(); tr = ctypes.c_int()
    a = lib().oracle_armijo(_obj(obj), len(x), _p(x), _p(p), _p(g), f0, c1, alpha0,
                            iter_ls, shrink, _p(xt), ctypes.byref(ft), ctypes.byref(tr))
    return a, tr.value


def hessian_update(H, dx, dg):
    H2 = np.array(H, dtype=np.float64, order="C", copy=True)
    dx = np.ascontiguousarray(dx, dtype=np.float64)
    dg = np.ascontiguousarray(dg, dtype=np.float64)
    updated = lib().oracle_hessian_update(len(dx), _p(H2), _p(dx), _p(dg))
    return H2, bool(updated)


@dataclass
class BfgsResult:
    x_final: np.ndarray
    f_final: np.ndarray
    grad_norm: np.ndarray
    iterations: np.ndarray
    status: np.ndarray
    ls_trials: np.ndarray
    grad_evals: np.ndarray


def bfgs_batch(obj, x0, theta=1e-6, iter_bfgs=1000, c1=0.3, alpha0=1.0, iter_ls=20,
               shrink=0.5, threads=None, jitter_seed=0) -> BfgsResult:
    """bfgs_run over the rows of x0.  ``jitter_seed`` != 0 selects the
    rounding-jitter model (zeus_oracle.c): every objective value and gradient
    component of row i moved by -1/0/+1 ulp from a per-row stream -- used
    only by the parity certificates, never as a reference outcome."""
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    n, d = x0.shape
    out = (Outcome * n)()
    xf = np.empty((n, d))
    if threads is None:
        threads = os.cpu_count() or 1
    lib().oracle_bfgs_batch_jitter(_obj(obj), d, n, _p(x0), theta, iter_bfgs, c1, alpha0,
                                   iter_ls, shrink, threads, jitter_seed & (2**64 - 1), out,
                                   _p(xf))
    arr = np.frombuffer(out, dtype=np.dtype([(f, "f8" if f in ("f_final", "grad_norm")
                                               else "i8") for f, _ in Outcome._fields_]))
    return BfgsResult(xf, arr["f_final"].copy(), arr["grad_norm"].copy(),
                      arr["iterations"].copy(), arr["status"].copy(),
                      arr["ls_trials"].copy(), arr["grad_evals"].copy())


def reduce_best(f_final, status) -> int:
    best = -1
    for i, (f, s) in enumerate(zip(f_final, status)):
        if s == 3 or np.isnan(f):
            continue
        if best < 0 or f < f_final[best]:
            best = i
    return best


def zeus_run(obj, d: int, n: int, seed: int, lower: float, upper: float, iter_pso: int,
             iter_bfgs: int, theta=1e-6, threads=None, w=0.5, c1_pso=1.2, c2_pso=1.5,
             c1_ls=0.3, alpha0=1.0, iter_ls=20, shrink=0.5, return_swarm=False):
    """Deterministic zeus_run (driver.py:220-265, required_c = N): PSO on one
    thread (as the reference), BFGS on a pthread pool.  Returns
    (converged_count, best_index, pso_best, BfgsResult) (+ the final Swarm
    when ``return_swarm``)."""
    if threads is None:
        threads = os.cpu_count() or 1
    x = np.empty((n, d)); v = np.empty((n, d)); p = np.empty((n, d)); pv = np.empty(n)
    gX = np.empty(d); pb = ctypes.c_double()
    out = (Outcome * n)()
    xf = np.empty((n, d))
    best = lib().oracle_zeus_run(_obj(obj), d, n, seed & (2**64 - 1), lower, upper, iter_pso,
                                 w, c1_pso, c2_pso, theta, iter_bfgs, c1_ls, alpha0, iter_ls,
                                 shrink, threads, _p(x), _p(v), _p(p), _p(pv), _p(gX),
                                 ctypes.byref(pb), out, _p(xf))
    arr = np.frombuffer(out, dtype=np.dtype([(f, "f8" if f in ("f_final", "grad_norm")
                                               else "i8") for f, _ in Outcome._fields_]))
    res = BfgsResult(xf, arr["f_final"].copy(), arr["grad_norm"].copy(),
                     arr["iterations"].copy(), arr["status"].copy(),
                     arr["ls_trials"].copy(), arr["grad_evals"].copy())
    ret = (int(np.sum(res.status == 0)), int(best), pb.value, res)
    if return_swarm:
        ret += (Swarm(x, v, p, pv, gX, pb.value),)
    return ret
