import sys, traceback, os; sys.path.insert(0, '.')
print("start", flush=True)
import paper_2603_28770_b200 as z
print("imported", flush=True)
try:
    spec = z.get_objective("ackley", 50)
    cfg = z.ZeusConfig(N=8, dim=50, range=(spec.lower, spec.upper), iter_pso=2, iter_bfgs=60, seed=1, deterministic=True)
    print("running", flush=True)
    r = z.zeus_run(spec.fn, cfg); print("ok", r.converged_count, r.best.f_final, flush=True)
except BaseException as e:
    traceback.print_exc(); sys.stdout.flush()
