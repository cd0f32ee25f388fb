"""Per-iteration latency of ONE straggler start (runs to the cap) alone on
the GPU: the quantity that sets time-to-solution for config 2."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_28770_b200 as z
from paper_2603_28770_b200 import engine
from paper_2603_28770_b200.linesearch import LineSearchParams

obj, d, N, sweeps, cap = sys.argv[1] if len(sys.argv) > 1 else "rastrigin", 10, 65536, 20, 2000
if len(sys.argv) > 2: d = int(sys.argv[2]); N = int(sys.argv[3]); sweeps = int(sys.argv[4])
spec = z.get_objective(obj, d)
cfg = z.ZeusConfig(N=N, dim=d, range=(spec.lower, spec.upper), iter_pso=sweeps, iter_bfgs=cap, seed=42, deterministic=True)
res = z.zeus_run(spec.fn, cfg)
it = res.per_run.iterations
order = np.argsort(-it)
print("iterations: p50 %d p99 %d p99.9 %d max %d; n at cap %d" % (np.median(it), np.percentile(it, 99), np.percentile(it, 99.9), it.max(), int(np.sum(it >= cap))))
ls = res.stats.ls_trials
print("trials/iter mean %.2f; straggler trials/iter %.2f" % (ls.sum() / max(1, it.sum()), ls[order[0]] / max(1, it[order[0]])))
# rebuild the starts (final swarm positions) and time the worst start alone
dev = torch.device("cuda", 0)
sh = engine.SwarmShard(z.objective_id(spec.fn), d, N, 0, 42, dev)
sh.init(spec.lower, spec.upper); engine.local_barrier(sh)
for _ in range(sweeps): sh.sweep(0.5, 1.2, 1.5); engine.local_barrier(sh)
x0 = sh.x[:, order[:1]].contiguous()
out = engine.BfgsBuffers.allocate(d, 1, dev)
P = engine.bfgs_params(1e-6, cap, LineSearchParams())
import ctypes
from paper_2603_28770_b200 import _capi
L = _capi.lib()
timing = hasattr(L, "zeus_debug_phase_cycles")
buf = (ctypes.c_ulonglong * 16)()
for rep in range(3):
    if timing:
        torch.cuda.synchronize(); L.zeus_debug_phase_cycles(buf, 1); L.zeus_debug_team_phase_cycles(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); engine.run_bfgs(z.objective_id(spec.fn), x0, P, out, dev); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
k = int(out.iterations[0].item())
if timing:
    L.zeus_debug_phase_cycles(buf, 0)
    names = ["line search (rest)", "gradient", "H pass", "8-value reduction+p'", "ddir+swap",
             "prologue", "LS setup", "bar A", "g.p reduction (warp 0)", "bar B (helpers' term pass)", "folds"]
    print("warp phase cycles per iteration:", {n: round(buf[i] / max(k, 1)) for i, n in enumerate(names)})
    L.zeus_debug_team_phase_cycles(buf, 0)
    tn = ["line search", "gradient", "H pass", "8-value reduction+p'", "ddir"]
    print("team phase cycles total (per iteration of k):", {n: round(buf[i] / max(k, 1)) for i, n in enumerate(tn)})
print(json.dumps({"objective": obj, "d": d, "straggler_iterations": k, "ms": ms, "us_per_iteration": ms * 1e3 / max(k, 1),
                  "cycles_per_iteration_at_1965MHz": ms * 1e-3 * 1.965e9 / max(k, 1)}))
