"""Per-phase cycles of the BFGS kernels under FULL load (throughput view).

    ZEUS_LIB=variants/lib_timing.so python scripts/phase_probe.py rosenbrock 50 16384 5

Runs one deterministic zeus_run and divides each phase's summed clock64()
deltas (lane 0 / thread 0 of every start) by the total iterations: the mean
wall-clock latency of one start-iteration's phases while the SM is shared
with the other resident starts.  Also prints iterations, trials/iteration and
the SM-cycles per start-iteration implied by the kernel time."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2603_28770_b200 as z
from paper_2603_28770_b200 import _capi

obj, d, N, sweeps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cap = int(sys.argv[5]) if len(sys.argv) > 5 else 2000
spec = z.get_objective(obj, d)
cfg = z.ZeusConfig(N=N, dim=d, range=(spec.lower, spec.upper), iter_pso=sweeps, iter_bfgs=cap,
                   seed=42, deterministic=True)
L = _capi.lib()
timing = hasattr(L, "zeus_debug_team_phase_cycles")
buf = (ctypes.c_ulonglong * 16)()
z.zeus_run(spec.fn, cfg)  # warm-up
torch.cuda.synchronize()
if timing:
    L.zeus_debug_phase_cycles(buf, 1)
    L.zeus_debug_team_phase_cycles(buf, 1)
res = z.zeus_run(spec.fn, cfg)
torch.cuda.synchronize()
it = res.stats.iterations.astype(np.int64)
K = int(it.sum())
sms = torch.cuda.get_device_properties(0).multi_processor_count
clk = 1.965e9
out = {"objective": obj, "d": d, "N": N, "iterations_total": K,
       "iter_mean": float(it.mean()), "iter_max": int(it.max()),
       "trials_per_iter": float(res.stats.ls_trials.sum() / max(K, 1)),
       "bfgs_ms": res.stats.bfgs_time * 1e3,
       "sm_cycles_per_start_iter": res.stats.bfgs_time * clk * sms / max(K, 1)}
if timing:
    L.zeus_debug_phase_cycles(buf, 0)
    wn = ["line search", "gradient", "H pass", "reduce8+p'", "ddir+swap", "prologue"]
    out["warp_phase_cycles_per_iter"] = {n: round(buf[i] / max(K, 1)) for i, n in enumerate(wn)}
    L.zeus_debug_team_phase_cycles(buf, 0)
    tn = ["line search", "gradient", "H pass", "reduce8+p'", "ddir"]
    out["team_phase_cycles_per_iter"] = {n: round(buf[i] / max(K, 1)) for i, n in enumerate(tn)}
print(json.dumps(out))
