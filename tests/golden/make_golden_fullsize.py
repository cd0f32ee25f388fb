"""Golden outcomes at the BASELINE sizes, produced by the REFERENCE itself.

Run in the build container (where /root/reference exists; ~1 h on 8 cores):

    python tests/golden/make_golden_fullsize.py [tag ...]

For every configuration below it runs the reference's own PSO
(`zeus.init_swarm` + `zeus.update_swarm`, pso.py:79-164) over the FULL swarm
(every particle, every sweep), then the reference's `zeus.bfgs_run`
(bfgs.py:80-156) from the final positions (driver.py:244) of a strided subset
of starts i = j * stride, on a process pool (the reference's own parallel
path is a fork pool of bfgs_run calls, driver.py:153-202).  It writes
`fullsize_<tag>.npz` next to this file:

    idx        the start indices checked
    x0         the reference's final swarm positions at idx (the BFGS starts)
    pos_sha    sha256 of the full [N][d] final position array (C order)
    gF, gX     the swarm's global best after the sweeps
    x, f, gn, k, s   bfgs_run outcome per checked start (s: 0 converged,
                     1 diverged, 2 stopped, 3 domain_error)

Nothing on the GPU box reads /root/reference: the tests regenerate the swarm
on the device (and with the oracle), check it against pos_sha / x0 / gF, and
compare the per-start outcomes with these fixtures.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

BOXES = {"rosenbrock": (-5.0, 5.0), "rastrigin": (-5.12, 5.12), "ackley": (-5.0, 5.0)}
STATUS = ("converged", "diverged", "stopped", "domain_error")

# tag: (objective, d, N, seed, iter_pso, cap, number of starts checked)
CASES = {
    "c2": ("rastrigin", 10, 65536, 42, 20, 2000, 8192),      # BASELINE config 2
    "c3": ("ackley", 50, 262144, 42, 5, 1000, 2048),         # config 3
    "t50r": ("rastrigin", 50, 131072, 42, 5, 2000, 2048),    # T50, one GPU's shard
    "t50b": ("rosenbrock", 50, 131072, 42, 5, 2000, 1024),
    "c4": ("rosenbrock", 100, 131072, 42, 5, 2000, 48),      # config 4, one GPU's shard
    "c5_s20": ("rastrigin", 20, 4096, 42, 20, 2000, 1024),   # config 5 (trade-off sweep)
    "c5_s5_k128": ("rastrigin", 20, 4096, 42, 5, 128, 1024),
    "c5_s100_k16": ("rastrigin", 20, 4096, 42, 100, 16, 1024),
}

_FN = None
_CAP = None


def _init(name, cap):
    global _FN, _CAP
    sys.path.insert(0, REF)
    import zeus.objectives as zo

    _FN = getattr(zo, name)
    _CAP = cap


def _one(x0):
    import zeus

    o = zeus.bfgs_run(_FN, list(x0), theta=1e-6, iter_bfgs=_CAP)
    return (np.asarray(o.x_final, dtype=np.float64), o.f_final, o.grad_norm, o.iterations,
            STATUS.index(o.status))


def make(tag: str) -> None:
    sys.path.insert(0, REF)
    import zeus
    import zeus.objectives as zo

    name, d, n, seed, sweeps, cap, count = CASES[tag]
    fn = getattr(zo, name)
    t0 = time.time()
    st = zeus.make_start_streams(seed, n, d)
    state = zeus.init_swarm(fn, n, BOXES[name], st, dim=d)
    for _ in range(sweeps):
        zeus.update_swarm(state, fn, zeus.PsoParams(), st)
    pos = np.ascontiguousarray(state.positions, dtype=np.float64)
    t1 = time.time()
    idx = np.arange(0, n, n // count)[:count]
    with Pool(os.cpu_count(), initializer=_init, initargs=(name, cap)) as pool:
        out = pool.map(_one, list(pos[idx]), chunksize=1)
    t2 = time.time()
    np.savez_compressed(
        os.path.join(HERE, f"fullsize_{tag}.npz"),
        idx=idx.astype(np.int64), x0=pos[idx], pos_sha=hashlib.sha256(pos.tobytes()).hexdigest(),
        gF=float(state.global_best_val), gX=np.asarray(state.global_best_pos, dtype=np.float64),
        x=np.array([o[0] for o in out]), f=np.array([o[1] for o in out]),
        gn=np.array([o[2] for o in out]), k=np.array([o[3] for o in out], dtype=np.int64),
        s=np.array([o[4] for o in out], dtype=np.int64),
        meta=np.array([name, d, n, seed, sweeps, cap], dtype=object).astype(str))
    print(f"{tag}: PSO {t1 - t0:.1f} s, BFGS on {len(idx)} starts {t2 - t1:.1f} s", flush=True)


if __name__ == "__main__":
    for t in (sys.argv[1:] or list(CASES)):
        make(t)
