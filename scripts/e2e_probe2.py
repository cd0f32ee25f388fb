"""Exposed host time of one config-2 zeus_run: call -> first launch, and
final synchronize -> return (the device is idle in both)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_28770_b200 as z
from paper_2603_28770_b200 import engine

marks = {}
orig_fused = engine.SwarmShard._fused
def fused(self, *a, **k):
    marks.setdefault("launch", time.perf_counter())
    return orig_fused(self, *a, **k)
engine.SwarmShard._fused = fused
orig_sync = torch.cuda.Stream.synchronize
def sync(self):
    r = orig_sync(self)
    marks["synced"] = time.perf_counter()
    return r
torch.cuda.Stream.synchronize = sync

cfg = lambda s: z.ZeusConfig(N=65536, dim=10, range=(-5.12, 5.12), iter_pso=20, iter_bfgs=2000,
                             seed=s, deterministic=True)
for s in range(3):
    z.zeus_run(z.rastrigin, cfg(1000 + s))
pre, post, tot = [], [], []
for s in range(8):
    torch.cuda.synchronize()
    marks.clear()
    t0 = time.perf_counter()
    r = z.zeus_run(z.rastrigin, cfg(42 + s))
    t1 = time.perf_counter()
    pre.append((marks["launch"] - t0) * 1e3); post.append((t1 - marks["synced"]) * 1e3)
    tot.append((t1 - t0) * 1e3)
print("pre-launch ms %.3f  post-sync ms %.3f  total %.3f" % (np.mean(pre), np.mean(post), np.mean(tot)))
import cProfile, pstats
marks.clear()
pr = cProfile.Profile()
for s in range(5):
    torch.cuda.synchronize(); marks.clear()
    pr.enable(); z.zeus_run(z.rastrigin, cfg(42 + s)); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
