#!/bin/bash
# memcheck + racecheck + synccheck of every kernel family on small configs
# (race detection): thread / warp / CTA-team tiers (d <= 16, with
# promotions), warp kernel (d = 24), wide kernel W = 1 (d = 20 with the
# reference-order folds, 40, 50 in TMEM) and W = 2 (d = 70, 100 in TMEM with
# two starts per CTA), fused PSO, the early-stop protocol, user plug-ins (thread and
# warp kernels), the multi-GPU PSO peer exchange (3 emulated ranks).
mkdir -p gpurun_out
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, paper_2603_28770_b200 as z
for name, d, n, cap, workers in (("rastrigin", 10, 300, 120, 0), ("rosenbrock", 2, 64, 60, 0),
                                 ("rosenbrock", 24, 8, 60, 0), ("ackley", 50, 8, 60, 0),
                                 ("rastrigin", 40, 5, 60, 0), ("rosenbrock", 100, 3, 60, 0),
                                 ("rastrigin", 70, 3, 60, 0), ("goldstein_price", 2, 33, 60, 0),
                                 ("rastrigin", 20, 9, 60, 0), ("rosenbrock", 20, 9, 60, 0),
                                 ("rosenbrock", 100, 5, 60, 2),
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
# user objective on the warp kernel (d > 16)
f = z.DeviceObjective(f.source, dim=24, data=[1.0 + 0.1 * i for i in range(24)])
r = z.zeus_run(f, z.ZeusConfig(N=8, dim=24, range=(-2.0, 2.0), iter_pso=2, iter_bfgs=60, seed=2))
print("plugin d=24", r.converged_count, r.best.f_final)
# multi-GPU PSO peer exchange, 3 ranks emulated on one device (one stream each)
import torch
from paper_2603_28770_b200 import engine
dev = torch.device("cuda", 0)
xgs = engine.PsoExchange.emulated(dev, 10, 3)
streams = [torch.cuda.Stream(dev) for _ in range(3)]
shards = []
for q in range(3):
    a, b = engine.shard_bounds(700, q, 3)
    shards.append((engine.SwarmShard(1, 10, b - a, a, 5, dev), b - a))
torch.cuda.synchronize()
for q, (sh, nq) in enumerate(shards):
    with torch.cuda.stream(streams[q]):
        sh.run_xchg(xgs[q], nq, -5.12, 5.12, 0.5, 1.2, 1.5, 3)
torch.cuda.synchronize()
print("exchange", [float(sh.gbest[0]) for sh, _ in shards])
PY
# synccheck flags every tcgen05.alloc (a bare alloc/dealloc kernel included:
# csrc/tools/tmem_synccheck.cu), so it runs on the shared-memory kernels
# (ZEUS_NO_TMEM=1); memcheck and racecheck cover the TMEM kernels too
for tool in memcheck racecheck synccheck; do
  env=""; [ $tool = synccheck ] && env="ZEUS_NO_TMEM=1"
  timeout 1200 env $env compute-sanitizer --tool $tool --print-limit 20 python /tmp/san.py > gpurun_out/$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/$tool.txt
  tail -6 gpurun_out/$tool.txt
done
