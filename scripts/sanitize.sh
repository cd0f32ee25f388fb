#!/bin/bash
# memcheck + racecheck of the hot kernels on small configs (race detection)
mkdir -p gpurun_out
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, paper_2603_28770_b200 as z
for name, d, n in (("rastrigin", 10, 96), ("rosenbrock", 2, 64), ("ackley", 50, 8), ("rosenbrock", 100, 3), ("rastrigin", 40, 5), ("goldstein_price", 2, 33)):
    spec = z.get_objective(name, d)
    cfg = z.ZeusConfig(N=n, dim=d, range=(spec.lower, spec.upper), iter_pso=2, iter_bfgs=60, seed=1, deterministic=True)
    r = z.zeus_run(spec.fn, cfg)
    print(name, d, r.converged_count, r.best.f_final)
PY
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python /tmp/san.py > gpurun_out/memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python /tmp/san.py > gpurun_out/racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck.txt
tail -12 gpurun_out/memcheck.txt; tail -12 gpurun_out/racecheck.txt
