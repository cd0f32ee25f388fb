"""Where config 2's end-to-end time goes beyond the device time: wall vs
device per zeus_run with the bench's L2 flush, with / without the NVML clock
sampler thread, and a per-section host timeline of one call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_28770_b200 as z
import bench

cfg = lambda s: z.ZeusConfig(N=65536, dim=10, range=(-5.12, 5.12), iter_pso=20, iter_bfgs=2000,
                             seed=s, deterministic=True)
dev = torch.device("cuda", 0)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for s in range(3):
    z.zeus_run(z.rastrigin, cfg(1000 + s))
for sampler in (False, True):
    rows = []
    ctx = bench.ClockSampler(0) if sampler else None
    if ctx: ctx.__enter__()
    for s in range(8):
        flush.fill_(float(s)); torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = z.zeus_run(z.rastrigin, cfg(42 + s))
        t1 = time.perf_counter()
        rows.append(((t1 - t0) * 1e3, r.wall_time * 1e3, r.device_time * 1e3))
    if ctx: ctx.__exit__(None, None, None)
    a = np.array(rows)
    print("sampler" if sampler else "no sampler", "outer wall %.3f  wall %.3f  device %.3f  gap %.3f ms" %
          tuple(list(a.mean(0)) + [a[:, 1].mean() - a[:, 2].mean()]))
