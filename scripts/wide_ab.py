"""A/B of BFGS kernel builds under full load: SM-cycles per start-iteration.

    ZEUS_LIB=variants/lib_x.so python scripts/wide_ab.py [name d N ...]

Runs one deterministic zeus_run per (objective, d, N) after a warm-up and
prints the BFGS kernel time, iterations, trials per iteration and the
SM-cycles one start-iteration costs (kernel time x clock x SMs / total
iterations), plus the minimal-FLOP roofline fraction (roofline.py) against
36.7 TFLOP/s.  Also prints a checksum of the per-start results so two builds
of the same numerics can be compared."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2603_28770_b200 as z
from paper_2603_28770_b200 import roofline

args = sys.argv[1:] or ["rosenbrock", "50", "131072", "rastrigin", "50", "131072",
                        "ackley", "50", "131072", "rosenbrock", "100", "16384"]
sms = torch.cuda.get_device_properties(0).multi_processor_count
ids = {"rosenbrock": 0, "rastrigin": 1, "ackley": 2}
for k in range(0, len(args), 3):
    name, d, n = args[k], int(args[k + 1]), int(args[k + 2])
    spec = z.get_objective(name, d)
    cfg = z.ZeusConfig(N=n, dim=d, range=(spec.lower, spec.upper), iter_pso=5, iter_bfgs=2000,
                       seed=42, deterministic=True)
    z.zeus_run(spec.fn, cfg)
    best = None
    for rep in range(3):
        r = z.zeus_run(spec.fn, cfg)
        t = r.stats.bfgs_time
        best = t if best is None else min(best, t)
    st = r.stats
    K = int(np.sum(st.iterations, dtype=np.int64))
    fl = roofline.flops(ids[name], d, st.iterations, st.ls_trials, st.grad_evals)
    print(json.dumps({"obj": name, "d": d, "N": n, "bfgs_ms": best * 1e3,
                      "sm_cycles_per_start_iter": best * 1.965e9 * sms / K,
                      "iter_mean": K / n, "trials_per_iter": float(st.ls_trials.sum() / K),
                      "frac": fl / best / 1e12 / 36.7,
                      "converged": r.converged_count,
                      "x_checksum": float(np.nansum(r.per_run.x_final))}), flush=True)
