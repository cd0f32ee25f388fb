"""PSO phase timing + swarm digest for A/B of two libzeus builds.

  ZEUS_LIB=/path/to/lib.so python scripts/pso_ab.py > out.json

For each (objective, d, N, sweeps): device time of init + sweeps (one fused
zeus_pso_run call, CUDA events, median of 5 after 2 warm-ups) and a sha256
of the final swarm (x, v, p, pval, gX, gbest) so two builds can be compared
bit for bit."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_28770_b200 as z  # noqa: E402
from paper_2603_28770_b200 import engine  # noqa: E402

CASES = [("rastrigin", 10, 65536, 20), ("rastrigin", 20, 1024, 100), ("rastrigin", 20, 65536, 100),
         ("rastrigin", 20, 1 << 20, 20), ("rosenbrock", 50, 1 << 20, 5), ("rastrigin", 50, 1 << 20, 5),
         ("ackley", 50, 262144, 5), ("rosenbrock", 100, 131072, 5), ("rosenbrock", 2, 1024, 20),
         ("goldstein_price", 2, 4096, 20), ("rastrigin", 7, 5000, 9), ("ackley", 33, 3001, 7)]
dev = torch.device("cuda", 0)
for name, d, n, sw in CASES:
    spec = z.get_objective(name, d)
    oid = z.objective_id(spec.fn)
    sh = engine.SwarmShard(oid, d, n, 0, 42, dev)
    ts = []
    for rep in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        sh.run_local(spec.lower, spec.upper, 0.5, 1.2, 1.5, sw)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    h = hashlib.sha256()
    for t in (sh.x, sh.v, sh.p, sh.pval, sh.gX, sh.gbest):
        h.update(t.cpu().numpy().tobytes())
    ms = sorted(ts[2:])[len(ts[2:]) // 2]
    print(json.dumps({"case": f"{name} d={d} N={n} sweeps={sw}", "ms": ms,
                      "us_per_sweep": ms * 1e3 / (sw + 1), "sha": h.hexdigest()[:16]}), flush=True)
