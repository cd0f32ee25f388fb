"""Robustness probe: tiny / 1M-start / every-objective zeus_run calls and
NaN / inf host-supplied starts (wall time printed per call)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, paper_2603_28770_b200 as z
for name, d, N in (("rastrigin", 1, 1), ("rastrigin", 1, 1000), ("rosenbrock", 2, 1 << 20),
                   ("rastrigin", 50, 1 << 20), ("ackley", 2, 77777), ("goldstein_price", 2, 5)):
    spec = z.get_objective(name, d)
    cfg = z.ZeusConfig(N=N, dim=d, range=(spec.lower, spec.upper), iter_pso=5, iter_bfgs=2000,
                       seed=1, deterministic=True)
    t = time.perf_counter()
    r = z.zeus_run(spec.fn, cfg)
    print(name, d, N, "conv", r.converged_count, "best", r.best.f_final, "wall %.3f s" % (time.perf_counter() - t))
# NaN / inf starts
cfg = z.ZeusConfig(N=4, dim=3, range=(-5.0, 5.0), iter_bfgs=100, deterministic=True)
st = np.array([[np.nan, 0, 0], [np.inf, 1, 1], [1, 1, 1], [0.5, 0.5, 0.5]])
r = z.zeus_run(z.rosenbrock, cfg, starts=st)
print("nan starts:", [o.status for o in r.per_run], r.best.f_final)
