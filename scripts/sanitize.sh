#!/bin/bash
# memcheck + racecheck + synccheck of every kernel family on small configs
# (race detection): thread / warp / CTA-team tiers (d <= 16, with
# promotions), warp kernel (d = 24), wide kernel W = 1 (d = 40, 50) and W = 2
# (d = 70, 100), fused PSO, the early-stop protocol, a user plug-in.
mkdir -p gpurun_out
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, paper_2603_28770_b200 as z
for name, d, n, cap, workers in (("rastrigin", 10, 300, 120, 0), ("rosenbrock", 2, 64, 60, 0),
                                 ("rosenbrock", 24, 8, 60, 0), ("ackley", 50, 8, 60, 0),
                                 ("rastrigin", 40, 5, 60, 0), ("rosenbrock", 100, 3, 60, 0),
                                 ("rastrigin", 70, 3, 60, 0), ("goldstein_price", 2, 33, 60, 0),
                                 ("rastrigin", 10, 200, 60, 2), ("rosenbrock", 50, 8, 60, 2)):
    spec = z.get_objective(name, d)
    cfg = z.ZeusConfig(N=n, dim=d, range=(spec.lower, spec.upper), iter_pso=2, iter_bfgs=cap,
                       seed=1, deterministic=workers == 0, required_c=2 if workers else None,
                       workers=workers)
    r = z.zeus_run(spec.fn, cfg)
    print(name, d, r.converged_count, r.best.f_final)
f = z.DeviceObjective("""
template <class T, class X>
__device__ T objective(const X& x, int d, const double* data, bool& err) {
  T s = 0.0;
  for (int i = 0; i < d; ++i) s = s + data[i] * x(i) * x(i) - zu::cos(3.0 * x(i));
  return s;
}""", dim=3, data=[1.0, 2.0, 3.0])
r = z.zeus_run(f, z.ZeusConfig(N=100, dim=3, range=(-2.0, 2.0), iter_pso=2, iter_bfgs=60, seed=2))
print("plugin", r.converged_count, r.best.f_final)
PY
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san.py > gpurun_out/$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/$tool.txt
  tail -6 gpurun_out/$tool.txt
done
