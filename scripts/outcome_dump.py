"""Dump per-start outcomes of one zeus_run (for A/B of library builds, ZEUS_LIB):
    python scripts/outcome_dump.py OUT.npz name d N [sweeps cap seed]"""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2603_28770_b200 as z
out, name, d, n = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
sweeps, cap, seed = (int(v) for v in (sys.argv[5:8] + ["5", "2000", "42"][len(sys.argv[5:8]):]))
spec = z.get_objective(name, d)
cfg = z.ZeusConfig(N=n, dim=d, range=(spec.lower, spec.upper), iter_pso=sweeps, iter_bfgs=cap,
                   seed=seed, deterministic=True)
r = z.zeus_run(spec.fn, cfg, starts=None)
pr = r.per_run
np.savez(out, x=pr.x_final, f=pr.f_final, gn=pr.grad_norm, k=pr.iterations, s=pr.status_codes)
print(out, "converged", r.converged_count, "statuses", np.bincount(pr.status_codes, minlength=4))
