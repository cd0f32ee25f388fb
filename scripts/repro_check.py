"""Run one zeus_run twice and compare per-start outcomes bitwise (races show as
differences), printing the starts that differ or fail:
    python scripts/repro_check.py name d N [sweeps cap seed]"""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2603_28770_b200 as z
name, d, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
sweeps, cap, seed = (int(v) for v in (sys.argv[4:7] + ["5", "2000", "42"][len(sys.argv[4:7]):]))
spec = z.get_objective(name, d)
cfg = z.ZeusConfig(N=n, dim=d, range=(spec.lower, spec.upper), iter_pso=sweeps, iter_bfgs=cap,
                   seed=seed, deterministic=True)
runs = [z.zeus_run(spec.fn, cfg) for _ in range(2)]
a, b = (r.per_run for r in runs)
same = np.array_equal(a.x_final, b.x_final, equal_nan=True) and np.array_equal(a.status_codes, b.status_codes)
bad = np.flatnonzero(a.status_codes != 0)
print(name, d, n, "reproducible" if same else "NOT REPRODUCIBLE", "non-converged:", bad[:10],
      [(int(a.iterations[i]), float(a.grad_norm[i])) for i in bad[:5]])
if not same:
    diff = np.flatnonzero(np.any(a.x_final != b.x_final, axis=1))
    print("differing starts", diff[:20], len(diff))
