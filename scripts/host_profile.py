"""Host-side cost of one zeus_run (config 2): wall vs device time and the
top Python functions (cProfile) -- what separates e2e from the device rate."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_28770_b200 as z
cfg = z.ZeusConfig(N=65536, dim=10, range=(-5.12, 5.12), iter_pso=20, iter_bfgs=2000, seed=42,
                   deterministic=True)
for _ in range(3):
    z.zeus_run(z.rastrigin, cfg)
torch.cuda.synchronize()
walls, devs = [], []
for _ in range(5):
    r = z.zeus_run(z.rastrigin, cfg)
    walls.append(r.wall_time); devs.append(r.device_time)
print("wall ms", [round(w * 1e3, 2) for w in walls], "device ms", [round(d * 1e3, 2) for d in devs])
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    z.zeus_run(z.rastrigin, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
