"""Wall vs device time of zeus_run calls (the bench's L2 flush between calls):
how much of the end-to-end time lies outside the device window, and (with
`profile`) where that host time goes.

    python scripts/e2e_probe.py [c2|c3|t50b] [profile]"""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2603_28770_b200 as z
CFG = {"c2": ("rastrigin", 10, 65536, 20, 2000, (-5.12, 5.12)),
       "c3": ("ackley", 50, 262144, 5, 1000, (-5.0, 5.0)),
       "t50b": ("rosenbrock", 50, 1 << 20, 5, 2000, (-5.0, 5.0))}
name = next((a for a in sys.argv[1:] if a in CFG), "c2")
obj, d, n, sweeps, cap, box = CFG[name]
fn = getattr(z, obj)
cfg = lambda s: z.ZeusConfig(N=n, dim=d, range=box, iter_pso=sweeps, iter_bfgs=cap, seed=s,
                             deterministic=True)
r = None
for s in range(3): r = z.zeus_run(fn, cfg(1000 + s))  # (held: the result-table pool's steady state)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
rows = []
for s in range(6):
    flush.fill_(1.0); torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = z.zeus_run(fn, cfg(42 + s))
    t1 = time.perf_counter()
    rows.append(((t1 - t0) * 1e3, r.device_time * 1e3, r.stats.pso_time * 1e3, r.stats.bfgs_time * 1e3, r.stats.reduce_time * 1e3))
print("per call (wall, device) ms:", [(round(w, 1), round(dv, 1)) for w, dv, *_ in rows])
a = np.array(rows).mean(0)
print("%s: wall %.3f device %.3f (pso %.3f bfgs %.3f reduce %.3f) -> outside device window %.3f ms" % (name, a[0], a[1], a[2], a[3], a[4], a[0] - a[1]))
if "profile" in sys.argv:  # where the host time goes
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for s in range(4):
        flush.fill_(1.0); torch.cuda.synchronize()
        r = z.zeus_run(fn, cfg(50 + s))
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)
