"""Benchmark: BFGS starts converged per second (and time to solution) on the
north-star workload T50 -- 1,048,576-start 50-D Rosenbrock + 1,048,576-start
50-D Rastrigin (BASELINE.json north_star) -- on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config t50|t50b|t50r|c1|c2|c3|c4|c5]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...

A step is one full zeus_run (PSO init + sweeps + multistart BFGS + reduction,
results to host) per problem of the workload.  T50 and config 4 are fixed
1,048,576-start problems: N GPUs split the starts (strong scaling; at N = 8
each GPU owns the 131,072 starts BASELINE quotes).  Configs 1-3 are
single-GPU problems (weak scaling: the per-GPU share is fixed).  Config 5 is
the paper's trade-off grid (Rastrigin d=20, PSO sweeps x starts x BFGS depth);
its step runs every grid point.

`value`  = converged starts / device time (CUDA events from the first PSO
           kernel to the final reduction; max over ranks per problem).
`e2e`    = the same through the public API (zeus_run's wall time, which
           includes the device-to-host copy of every start's x, f, |g|, k,
           status); the call's inputs are scalars (objective, config, seed).
`roofline` = the dominant BFGS kernel's algorithmic FP64 rate (per-start
           counters the kernel returns; paper_2603_28770_b200/roofline.py)
           over the measured DFMA peak; `traffic` = its DRAM bytes per launch
           from the committed ncu capture (profiles/ncu_summary.json).
`cpu_baseline` = the reference algorithm's CPU restatement (oracle/, C,
           every host thread) on a bounded sample of the same workload.
--impl reference prints the same line for that CPU arm (rank 0 only).
L2 (126 MB) is flushed between problems; every problem's inputs and
outputs are larger than L2 anyway.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BFGS starts converged/sec"
OBJ_IDS = {"rosenbrock": 0, "rastrigin": 1, "ackley": 2, "goldstein_price": 3}
BOX = {"rosenbrock": (-5.0, 5.0), "rastrigin": (-5.12, 5.12), "ackley": (-5.0, 5.0)}
M = 1 << 20


def P(obj, d, n, sweeps, cap, sample):
    """One problem: n starts (total for strong scaling, per GPU for weak),
    `sample` = starts per step of the CPU arm's bounded sample."""
    return dict(obj=obj, d=d, n=n, sweeps=sweeps, cap=cap, sample=sample)


CONFIGS = {
    # north star: both 50-D problems, 1M starts each
    "t50": dict(problems=[P("rosenbrock", 50, M, 5, 2000, 1024),
                          P("rastrigin", 50, M, 5, 2000, 2048)], scaling="strong"),
    "t50b": dict(problems=[P("rosenbrock", 50, M, 5, 2000, 1024)], scaling="strong"),
    "t50r": dict(problems=[P("rastrigin", 50, M, 5, 2000, 2048)], scaling="strong"),
    "c1": dict(problems=[P("rosenbrock", 2, 1024, 10, 1000, 1024)], scaling="weak"),
    "c2": dict(problems=[P("rastrigin", 10, 65536, 20, 2000, 65536)], scaling="weak"),
    "c3": dict(problems=[P("ackley", 50, 262144, 5, 1000, 4096)], scaling="weak"),
    "c4": dict(problems=[P("rosenbrock", 100, M, 5, 2000, 96)], scaling="strong"),
    # config 5: the trade-off grid; the CPU arm samples N <= 2^14
    "c5": dict(problems=[P("rastrigin", 20, n, s, k, min(n, 1 << 12))
                         for s in (0, 5, 20, 100) for n in (1 << 10, 1 << 12, 1 << 14, 1 << 16,
                                                             1 << 18, M)
                         for k in (16, 128, 1024)], scaling="strong"),
}


def problem_name(p):
    return (f"{p['obj']} d={p['d']}, {p['n']:,} starts, {p['sweeps']} PSO sweeps, "
            f"BFGS cap {p['cap']}")


def global_n(cfg, p, world):
    return p["n"] if cfg["scaling"] == "strong" else p["n"] * world


def config_dict(name, world):
    """The `config` object of BOTH arms' lines (identical by construction)."""
    cfg = CONFIGS[name]
    probs = cfg["problems"]
    if name == "c5":
        work = ("config 5 trade-off grid: rastrigin d=20, PSO sweeps {0,5,20,100} x starts "
                "{2^10..2^20} x BFGS cap {16,128,1024} (72 zeus_run calls per step)")
    else:
        work = " + ".join(problem_name(dict(p, n=global_n(cfg, p, world))) for p in probs)
    per = ", ".join(f"{-(-global_n(cfg, p, world) // world):,}" for p in probs[:2])
    return {"workload": work, "name": name, "scaling": cfg["scaling"],
            "starts_per_gpu": per, "parallelism": f"start-sharded x{world}",
            "theta": 1e-6, "seed": "42+step",
            "l2": "flushed between problems (inputs and outputs > 126 MB L2)"}


def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        import psutil

        phys = psutil.cpu_count(logical=False)
    except Exception:
        phys = None
    return {"model": model, "physical_cores": phys, "logical_cpus": os.cpu_count()}


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self.nvml = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            # NVML queries take the driver's lock: sampled sparsely so they do
            # not stall the measured calls' own CUDA API calls (a 5 ms period
            # added ~10 ms per call to config 2's end-to-end time)
            self._stop.wait(0.05)

    def __enter__(self):
        if self.nvml:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nvml:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def ncu_traffic(config, obj, d):
    """DRAM bytes per launch of the problem's BFGS kernel in the committed ncu
    capture of this config (profiles/ncu_summary.json), or None."""
    try:
        s = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        return s[config]["kernels"][f"{obj}{d}"]["dram_bytes_per_launch"]
    except Exception:
        return None


def measure_fp64_peak(torch, dev):
    """DFMA microbenchmark (csrc/measure.cu): the FP64 roofline denominator
    (MEASURED_PEAKS.json has no FP64 figure)."""
    import ctypes

    from paper_2603_28770_b200 import _capi

    L = _capi.lib()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sink = torch.empty(sms * 8, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    flops = ctypes.c_double()
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _capi.check(L.zeus_bench_dfma(sms * 8, 256, 4096, sink.data_ptr(), ctypes.byref(flops),
                                      stream.cuda_stream))
        e1.record(stream)
        e1.synchronize()
        best = max(best, flops.value / (e0.elapsed_time(e1) / 1e3))
    return best / 1e12


# ---------------------------------------------------------------- CPU arm

def cpu_sample(cfg_name, seed, world=1):
    """The reference algorithm on host cores (oracle/zeus_oracle.c: PSO on one
    thread as the reference, BFGS on a pthread pool over every host thread):
    one deterministic zeus_run per problem on its bounded sample of starts.
    Each problem's count and time are scaled from its sample to its
    workload size, so a multi-problem rate weighs the problems as the GPU
    arm's workload does.  Returns (converged, seconds) extrapolated, the
    seconds actually spent, and the thread count."""
    from oracle import oracle as O

    cfg = CONFIGS[cfg_name]
    threads = os.cpu_count() or 1
    conv = secs = spent = 0.0
    for p in cfg["problems"]:
        lo, hi = BOX[p["obj"]]
        t0 = time.perf_counter()
        c, _, _, _ = O.zeus_run(p["obj"], p["d"], p["sample"], seed, lo, hi, p["sweeps"],
                                p["cap"], threads=threads)
        t = time.perf_counter() - t0
        scale = global_n(cfg, p, world) / p["sample"]
        conv += c * scale
        secs += t * scale
        spent += t
    return conv, secs, spent, threads


def sample_desc(cfg_name):
    probs = CONFIGS[cfg_name]["problems"]
    if cfg_name == "c5":
        return ("every config-5 grid point with N capped at 4,096 starts (same sweeps and "
                "caps), one deterministic oracle zeus_run each")
    return ("per step: " + " + ".join(f"{p['obj']} d={p['d']} on {p['sample']:,} starts"
                                      for p in probs) +
            " (own swarm of that size, same PSO sweeps and BFGS cap, deterministic) through "
            "oracle/zeus_oracle.c; each problem's count and time scaled to its workload size "
            "(the per-start cost is size-independent)")


def python_reference(cfg_name):
    """The reference package itself (baseline/_ref, installed offline from
    /root/reference) on a tiny sample: zeus.zeus_run with workers = physical
    cores (its own fork pool), deterministic.  None when not installed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "zeus")):
        return None
    sys.path.insert(0, ref)
    try:
        import psutil
        import zeus
    except Exception as e:  # pragma: no cover
        return {"unavailable": str(e)}
    workers = psutil.cpu_count(logical=False) or 1
    conv = secs = starts = 0
    probs = CONFIGS[cfg_name]["problems"]
    if cfg_name == "c5":
        probs = [p for p in probs if p["n"] == 1 << 10 and p["sweeps"] == 5]
    for p in probs:
        n = 32 if p["d"] >= 50 else min(p["n"], 1024)
        fn = getattr(zeus.objectives, p["obj"])
        cfg = zeus.ZeusConfig(N=n, dim=p["d"], range=BOX[p["obj"]], iter_pso=p["sweeps"],
                              iter_bfgs=p["cap"], seed=42, workers=workers, deterministic=True)
        t0 = time.perf_counter()
        r = zeus.zeus_run(fn, cfg)
        secs += time.perf_counter() - t0
        conv += r.converged_count
        starts += n
    return {"value": conv / secs, "unit": "starts/s", "cores": workers,
            "sample": f"{starts} starts through zeus.zeus_run (the reference package, "
                      f"workers={workers}, deterministic)", "seconds": secs}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return  # the CPU arm is one host's figure; other ranks exit without work
    from oracle import oracle as O

    O.build()
    for s in range(args.warmup):
        cpu_sample(args.config, 1000 + s, world)
    conv = secs = spent = 0.0
    for s in range(args.steps):
        c, t, sp, threads = cpu_sample(args.config, 42 + s, world)
        conv += c
        secs += t
        spent += sp
    value = conv / secs
    info = cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "starts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": spent / args.steps * 1e3, "higher_is_better": True,
        "scaling": CONFIGS[args.config]["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Philox(seed, start) starts, seed 42+step)",
        "config": config_dict(args.config, world),
        "cpu_baseline": {"value": value, "unit": "starts/s", "cores": threads, "kind": "port",
                         "sample": sample_desc(args.config), "cpu": info},
        "e2e": {"value": value, "unit": "starts/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if args.config != "c5":  # the whole workload on these host cores, extrapolated
        line["time_to_solution_s_extrapolated"] = secs / args.steps
    if not args.no_python_reference:
        line["python_reference"] = python_reference(args.config)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="t50")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-python-reference", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2603_28770_b200 as z
    from paper_2603_28770_b200 import engine, roofline

    # test hooks: ZEUS_BENCH_DEVICE pins every rank to one GPU and
    # ZEUS_BENCH_BACKEND=gloo lets several ranks share it (exercises the N > 1
    # path on a one-GPU box); the driver's runs use neither
    local = int(os.environ.get("ZEUS_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("ZEUS_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, **({"device_id": dev} if backend == "nccl" else {}))
    cfg = CONFIGS[args.config]
    probs = cfg["problems"]

    def run(p, seed):
        N = global_n(cfg, p, world)
        zc = z.ZeusConfig(N=N, dim=p["d"], range=BOX[p["obj"]], iter_pso=p["sweeps"],
                          iter_bfgs=p["cap"], seed=seed, deterministic=True)
        return z.zeus_run(getattr(z, p["obj"]), zc)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    peak = measure_fp64_peak(torch, dev)
    # warm-up holds each result until the next call returns, as the timed
    # loop does, so zeus_run's pool of page-locked result tables (the kernels
    # write into them directly) reaches its steady state before timing
    held = None
    for s in range(args.warmup):
        for p in probs:
            held = run(p, 1000 + s)
    del held
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # rec[step][problem] = per-rank numbers
    recs = []
    with ClockSampler(local) as clocks:
        t_bracket = time.perf_counter()
        for s in range(args.steps):
            row = []
            for p in probs:
                flush.fill_(float(s))  # evict L2 (> 126 MB) between problems
                torch.cuda.synchronize()
                res = run(p, 42 + s)
                st = res.stats
                oid = OBJ_IDS[p["obj"]]
                # this rank's own starts (rank 0 holds every start's counters)
                N = global_n(cfg, p, world)
                lo, hi = engine.shard_bounds(N, rank, world)
                sl = slice(lo, hi) if len(st.iterations) == N else slice(None)
                it, ls, ge = st.iterations[sl], st.ls_trials[sl], st.grad_evals[sl]
                row.append(dict(
                    conv=res.converged_count, dev=res.device_time, wall=res.wall_time,
                    bfgs=st.bfgs_time, pso=st.pso_time,
                    flops=roofline.flops(oid, p["d"], it, ls, ge),
                    flops_generic=roofline.flops(oid, p["d"], it, ls, ge, "generic"),
                    launches=st.kernel_launches,
                    iters=float(np.sum(it, dtype=np.int64)),
                    trials=float(np.sum(ls, dtype=np.int64)),
                    d2h=len(res.per_run) * (p["d"] * 8 + 8 + 8 + 4 + 4 + 4 + 4)))
            recs.append(row)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        bracket = time.perf_counter() - t_bracket

    def maxrank(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.cpu().numpy()

    def sumrank(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t)
        return t.cpu().numpy()

    K, NP = args.steps, len(probs)
    flat = lambda key: [recs[s][j][key] for s in range(K) for j in range(NP)]  # noqa: E731
    dev_t = maxrank(flat("dev")).reshape(K, NP)
    wall_t = maxrank(flat("wall")).reshape(K, NP)
    bfgs_t = maxrank(flat("bfgs")).reshape(K, NP)
    pso_t = maxrank(flat("pso")).reshape(K, NP)
    bracket = float(maxrank([bracket])[0])
    # kernel rates: this rank's FLOPs over this rank's kernel time, summed over ranks
    fl = sumrank(flat("flops")).reshape(K, NP)
    flg = sumrank(flat("flops_generic")).reshape(K, NP)
    bfgs_sum = sumrank(flat("bfgs")).reshape(K, NP)
    iters = sumrank(flat("iters")).reshape(K, NP)
    trials = sumrank(flat("trials")).reshape(K, NP)
    conv = np.array(flat("conv"), dtype=np.float64).reshape(K, NP)  # global counts
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # dominant kernel: the problem with the largest BFGS time
    j_dom = int(np.argmax(bfgs_t.sum(axis=0)))
    pd = probs[j_dom]
    # achieved = algorithmic FLOPs of that kernel's launches / their duration,
    # per GPU (every rank's FLOPs over every rank's kernel time) vs a GPU's peak
    ach = float(fl[:, j_dom].sum() / bfgs_sum[:, j_dom].sum() / 1e12)
    ach_g = float(flg[:, j_dom].sum() / bfgs_sum[:, j_dom].sum() / 1e12)
    per_problem = []
    for j, p in enumerate(probs):
        a = float(fl[:, j].sum() / bfgs_sum[:, j].sum() / 1e12)
        per_problem.append({
            "problem": problem_name(dict(p, n=global_n(cfg, p, world))),
            "value": float(conv[:, j].sum() / dev_t[:, j].sum()),
            "e2e": float(conv[:, j].sum() / wall_t[:, j].sum()),
            "time_to_solution_s": float(dev_t[:, j].mean()),
            "bfgs_s": float(bfgs_t[:, j].mean()), "pso_s": float(pso_t[:, j].mean()),
            "converged_per_step": float(conv[:, j].mean()),
            "iterations_mean": float(iters[:, j].mean() / global_n(cfg, p, world)),
            "trials_per_iteration": float(trials[:, j].sum() / max(1.0, iters[:, j].sum())),
            "roofline": {"bound": "fp64", "achieved": a, "peak": peak, "unit": "TFLOP/s",
                         "frac": a / peak,
                         "traffic": ncu_traffic(args.config, p["obj"], p["d"])}})
    if args.config == "c5":
        per_problem = [dict(pp, sweeps=p["sweeps"], starts=p["n"], cap=p["cap"])
                       for pp, p in zip(per_problem, probs)]
    total_dev = float(dev_t.sum())
    line = {
        "metric": METRIC,
        "value": float(conv.sum() / total_dev),
        "unit": "starts/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": total_dev / K * 1e3,
        "higher_is_better": True,
        "scaling": cfg["scaling"],
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (Philox(seed, start) starts, seed 42+step)",
        "config": config_dict(args.config, world),
        "time_to_solution_s": float(dev_t.sum(axis=1).mean()),
        "bracket_ms_per_step": bracket / K * 1e3,
        "converged_per_step": float(conv.sum() / K),
        "e2e": {"value": float(conv.sum() / wall_t.sum()), "unit": "starts/s",
                "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": int(sum(recs[0][j]["d2h"] for j in range(NP))),
                "path": "zeus_run(f, ZeusConfig(...)) wall time per problem, every start's "
                        "outcome (x_final, f, |g|, k, status, counters) delivered to host "
                        "memory (one GPU: written by the BFGS kernels into page-locked, "
                        "device-mapped host rows as each start finishes; several ranks: "
                        "packed, gathered and copied D2H); d2h_bytes_per_step = those rows",
                "inputs": "the call's inputs are (objective, config, seed): kernel arguments "
                          "only; the swarm is generated on the device by the reference's "
                          "Philox stream (SURVEY S1), so no input bytes cross PCIe"},
        "gpu_launches": int(sum(r["launches"] for row in recs for r in row)),
        "roofline": {"bound": "fp64",
                     "kernel": f"BFGS kernel of {pd['obj']} d={pd['d']} (the step's "
                               "largest; profiles/*_launches.txt)",
                     "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                     "traffic": ncu_traffic(args.config, pd["obj"], pd["d"]),
                     "peak_source": "measured DFMA microbenchmark (csrc/measure.cu) on this "
                                    "GPU; MEASURED_PEAKS.json has no FP64 figure",
                     "flop_convention": "minimal sparse-tangent (paper_2603_28770_b200/"
                                        "roofline.py); achieved_generic = SURVEY 8(d) generic",
                     "achieved_generic_convention": ach_g},
        "problems": per_problem,
        "clocks": clocks.summary(),
    }
    if not args.no_cpu_baseline and world == 1:  # the CPU baseline is an N = 1 figure
        c, secs, _, threads = cpu_sample(args.config, 42)
        line["cpu_baseline"] = {"value": c / secs, "unit": "starts/s", "cores": threads,
                                "kind": "port", "sample": sample_desc(args.config),
                                "cpu": cpu_info()}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
