"""Algorithmic FLOP model of the BFGS hot path ('Roofline').

Convention: +, -, *, /, sqrt count 1, an FMA counts 2, each
libm cos/sin/exp call counts 1, negations count 0; redundant work earns no
credit.  Per BFGS iteration

    F_iter = F_grad + T * F_trial + F_lin,
    F_trial = C_val + 2d + 3          (trial point x + a p, Armijo test)
    F_lin   = 6 d^2 + 18 d            (one matvec, symmetric rank-2 update, dots)

and per start  G * F_grad + sum(T) * F_trial + K * F_lin + C_val(x0), with K,
G, T taken from the per-start counters the kernel returns.

Two gradient conventions are reported:
  * 'minimal' (headline): the sparse-tangent forward mode this kernel runs --
    only the terms that contain x_i carry a tangent, the value sweep is the
    line search's last trial (no re-evaluation): F_grad = C_tan_sparse.
  * 'generic': value sweep + d full tangent passes,
    F_grad = C_val + d * C_tan; the reference's own algorithm.
"""

from __future__ import annotations

import numpy as np

# per-objective constants: (C_val(d), C_tan_full(d), C_tan_sparse(d))
_CONSTS = {
    0: (lambda d: 8 * (d - 1), lambda d: 13 * (d - 1), lambda d: 21 * (d - 1) + d),   # rosenbrock
    1: (lambda d: 6 * d + 1, lambda d: 8 * d - 1, lambda d: 6 * d),                   # rastrigin
    2: (lambda d: 5 * d + 10, lambda d: 7 * d + 7, lambda d: 15 * d + 10),            # ackley
    3: (lambda d: 38, lambda d: 60, lambda d: 120),                                    # goldstein
}


def flops(obj: int, d: int, iterations: np.ndarray, ls_trials: np.ndarray,
          grad_evals: np.ndarray, convention: str = "minimal") -> float:
    """Total algorithmic FLOPs of a BFGS launch from its per-start counters."""
    c_val, c_tan_full, c_tan_sparse = (f(d) for f in _CONSTS[obj])
    if convention == "minimal":
        f_grad = c_tan_sparse
    elif convention == "generic":
        f_grad = c_val + d * c_tan_full
    else:
        raise ValueError(convention)
    f_trial = c_val + 2 * d + 3
    f_lin = 6 * d * d + 18 * d
    K = float(np.sum(iterations, dtype=np.int64))
    G = float(np.sum(grad_evals, dtype=np.int64))
    T = float(np.sum(ls_trials, dtype=np.int64))
    n = len(iterations)
    return G * f_grad + T * f_trial + K * f_lin + n * c_val
