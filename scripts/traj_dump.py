"""Trajectory of chosen starts under the current library (ZEUS_LIB for A/B):
x_final / f / |g| after caps j = 0, step, 2 step, ... (deterministic kernels:
the capped run's state is the full run's state after j iterations).
    python scripts/traj_dump.py OUT.npz name d N sweeps seed step jmax index [index ...]"""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2603_28770_b200 as z
from paper_2603_28770_b200 import engine
from paper_2603_28770_b200.linesearch import LineSearchParams
out, name, d, n, sweeps, seed, step, jmax = sys.argv[1], sys.argv[2], *map(int, sys.argv[3:9])
idx = [int(v) for v in sys.argv[9:]]
spec = z.get_objective(name, d)
dev = torch.device("cuda", 0)
sh = engine.SwarmShard({"rosenbrock": 0, "rastrigin": 1, "ackley": 2}[name], d, n, 0, seed, dev)
sh.run_local(spec.lower, spec.upper, 0.5, 1.2, 1.5, sweeps)
x0 = sh.x.cpu().numpy()[:, idx]  # [d][k]
res = {}
for j in range(0, jmax + 1, step):
    xs = torch.from_numpy(np.ascontiguousarray(x0)).to(dev)
    o = engine.BfgsBuffers.allocate(d, len(idx), dev)
    engine.run_bfgs(engine.objective_id(spec.fn, d) if hasattr(engine, "objective_id") else
                    {"rosenbrock": 0, "rastrigin": 1, "ackley": 2}[name], xs,
                    engine.bfgs_params(1e-6, j, LineSearchParams()), o, dev)
    res[j] = (o.x_final.cpu().numpy().T.copy(), o.f_final.cpu().numpy().copy(),
              o.grad_norm.cpu().numpy().copy(), o.iterations.cpu().numpy().copy())
js = sorted(res)
np.savez(out, j=np.array(js), x=np.stack([res[j][0] for j in js]), f=np.stack([res[j][1] for j in js]),
         g=np.stack([res[j][2] for j in js]), k=np.stack([res[j][3] for j in js]))
print(out, "done")
