"""Wall vs device time of config-2 zeus_run calls (the bench's L2 flush between
calls): how much of the end-to-end time lies outside the device window."""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2603_28770_b200 as z
cfg = lambda s: z.ZeusConfig(N=65536, dim=10, range=(-5.12, 5.12), iter_pso=20, iter_bfgs=2000, seed=s, deterministic=True)
for s in range(3): z.zeus_run(z.rastrigin, cfg(1000 + s))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
rows = []
for s in range(6):
    flush.fill_(1.0); torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = z.zeus_run(z.rastrigin, cfg(42 + s))
    t1 = time.perf_counter()
    rows.append(((t1 - t0) * 1e3, r.device_time * 1e3, r.stats.pso_time * 1e3, r.stats.bfgs_time * 1e3, r.stats.reduce_time * 1e3))
a = np.array(rows).mean(0)
print("wall %.3f device %.3f (pso %.3f bfgs %.3f reduce %.3f) -> outside device window %.3f ms" % (a[0], a[1], a[2], a[3], a[4], a[0] - a[1]))
if len(sys.argv) > 1 and sys.argv[1] == "profile":  # where the host time goes
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for s in range(4):
        flush.fill_(1.0); torch.cuda.synchronize()
        z.zeus_run(z.rastrigin, cfg(50 + s))
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
