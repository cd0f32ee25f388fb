"""Benchmark: BFGS starts converged per second on BASELINE config 2
(Rastrigin d=10, 65,536 starts per GPU, 20 PSO sweeps, BFGS cap 2,000).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...

A step is one full zeus_run (PSO init + 20 sweeps + multistart BFGS +
reduction) over the step's starts; per-GPU work is fixed (weak scaling, each
rank owns 65,536 starts of a 65,536 x N swarm).  `value` is converged starts
per second of device time (CUDA events, max over ranks); `e2e` is the same
metric through the public API with the per-start results copied back to host
memory every step.  L2 is flushed (256 MiB write) between steps, outside the
per-step event window.  --impl reference times the reference algorithm's CPU
restatement (oracle/, C, all host threads) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

from dataclasses import replace

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (objective, d, starts per GPU, iter_pso, cap, box)
    "c2": ("rastrigin", 10, 65536, 20, 2000, (-5.12, 5.12)),
    "c1": ("rosenbrock", 2, 1024, 10, 1000, (-5.0, 5.0)),
    "c3": ("ackley", 50, 262144, 5, 1000, (-5.0, 5.0)),
    # north-star targets: 1,048,576 starts on 8 GPUs = 131,072 per GPU
    "t50r": ("rastrigin", 50, 131072, 5, 2000, (-5.12, 5.12)),
    "t50b": ("rosenbrock", 50, 131072, 5, 2000, (-5.0, 5.0)),
    # BASELINE config 4: 1,048,576 starts over 8 GPUs = 131,072 per GPU
    "c4": ("rosenbrock", 100, 131072, 5, 2000, (-5.0, 5.0)),
}
METRIC = "BFGS starts converged/sec"
OBJ_IDS = {"rosenbrock": 0, "rastrigin": 1, "ackley": 2, "goldstein_price": 3}


def workload_name(cfg_name, world):
    obj, d, n, sweeps, cap, _ = CONFIGS[cfg_name]
    return (f"{obj} d={d}, {n * world:,} starts ({n:,}/GPU), {sweeps} PSO sweeps, "
            f"BFGS cap {cap}")


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
            self._stop.wait(0.005)

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


def _ncu_traffic(config):
    """DRAM bytes per launch of the config's BFGS kernels from the committed
    ncu capture (profiles/ncu_summary.json), or None."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))[config][
            "dram_bytes_per_launch"]
    except Exception:
        return None


def measure_fp64_peak(torch, dev):
    """DFMA microbenchmark (csrc/measure.cu): the FP64 roofline denominator."""
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


def cpu_reference_run(cfg_name, world, seed):
    """The reference algorithm on host cores (oracle/, C, pthreads): one full
    deterministic zeus_run of the workload.  Returns (converged, seconds)."""
    from oracle import oracle as O

    obj, d, n, sweeps, cap, (lo, hi) = CONFIGS[cfg_name]
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    conv, _, _, _ = O.zeus_run(obj, d, n * world, seed, lo, hi, sweeps, cap, threads=threads)
    return conv, time.perf_counter() - t0, threads


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O

    O.build()
    # each step times a bounded sample: the one-GPU share of the workload
    # (the CPU rate is size-independent; N x the work would take minutes)
    for s in range(args.warmup):
        cpu_reference_run(args.config, 1, 42 + s)
    conv = secs = 0.0
    for s in range(args.steps):
        c, t, threads = cpu_reference_run(args.config, 1, 42 + s)
        conv += c
        secs += t
    value = conv / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "starts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (Philox starts)",
        "config": {"workload": workload_name(args.config, world), "seed": "42+step"},
        "cpu_baseline": {"value": value, "unit": "starts/s", "cores": threads, "kind": "port",
                         "sample": workload_name(args.config, 1) + " per step (the one-GPU "
                                   "share of the workload), deterministic (required_c=N); PSO "
                                   "on one thread as in the reference, BFGS on a pthread pool"},
        "e2e": {"value": value, "unit": "starts/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-north-star", action="store_true",
                    help="skip the T50 (1M-start 50-D) roofline lines")
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
    from paper_2603_28770_b200 import roofline

    # test hooks: ZEUS_BENCH_DEVICE pins every rank to one GPU and
    # ZEUS_BENCH_BACKEND=gloo lets several ranks share it (exercises the N > 1
    # path on a one-GPU box); the driver's runs use neither
    local = int(os.environ.get("ZEUS_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("ZEUS_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, **({"device_id": dev} if backend == "nccl" else {}))
    obj_name, d, n_per, sweeps, cap, box = CONFIGS[args.config]
    N = n_per * world
    fn = getattr(z, obj_name)

    def run(seed):
        cfg = z.ZeusConfig(N=N, dim=d, range=box, iter_pso=sweeps, iter_bfgs=cap, seed=seed,
                           deterministic=True)
        return z.zeus_run(fn, cfg)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    peak = measure_fp64_peak(torch, dev)
    for s in range(args.warmup):
        run(1000 + s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    records = []
    with ClockSampler(local) as clocks:
        t_bracket = time.perf_counter()
        for s in range(args.steps):
            flush.fill_(float(s))  # evict L2 (> 126 MB) between steps
            torch.cuda.synchronize()
            res = run(42 + s)
            st = res.stats
            fl = roofline.flops(OBJ_IDS[obj_name], d, st.iterations, st.ls_trials, st.grad_evals)
            flg = roofline.flops(OBJ_IDS[obj_name], d, st.iterations, st.ls_trials,
                                 st.grad_evals, "generic")
            records.append(dict(conv=res.converged_count, dev=res.device_time,
                                wall=res.wall_time, bfgs=st.bfgs_time, pso=st.pso_time,
                                flops=fl, flops_generic=flg, launches=st.kernel_launches,
                                d2h=len(res.per_run) * (d * 8 + 8 + 8 + 4 + 1 + 4 + 4)))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        bracket = time.perf_counter() - t_bracket

    # max over ranks of every per-step time
    def maxrank(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.cpu().numpy()

    # north-star workloads: 1M-start 50-D Rastrigin and
    # Rosenbrock, 131,072 starts per GPU (weak scaling to 8 GPUs), one timed
    # run each after one warm-up, FP64 roofline of the BFGS kernel
    ns = None
    if not args.no_north_star and args.config == "c2":
        ns = {}
        for key in ("t50b", "t50r"):
            o_name, dd, nn, sw, cp, bx = CONFIGS[key]
            cfg_ns = z.ZeusConfig(N=nn * world, dim=dd, range=bx, iter_pso=sw, iter_bfgs=cp,
                                  seed=7, deterministic=True)
            z.zeus_run(getattr(z, o_name), replace(cfg_ns, seed=8))
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            r = z.zeus_run(getattr(z, o_name), cfg_ns)
            st = r.stats
            fl = roofline.flops(OBJ_IDS[o_name], dd, st.iterations, st.ls_trials, st.grad_evals)
            bt = float(maxrank([st.bfgs_time])[0])
            dt = float(maxrank([r.device_time])[0])
            ach = fl / st.bfgs_time / 1e12
            ns[key] = {"workload": workload_name(key, world), "value": r.converged_count / dt,
                       "unit": "starts/s", "time_to_solution_s": dt, "bfgs_s": bt,
                       "converged": r.converged_count,
                       "iterations_mean": float(np.mean(st.iterations)),
                       "trials_per_iteration": float(np.sum(st.ls_trials) /
                                                     max(1, np.sum(st.iterations))),
                       "roofline": {"bound": "fp64", "achieved": ach, "peak": peak,
                                    "unit": "TFLOP/s", "frac": ach / peak,
                                    "traffic": _ncu_traffic(key),
                                    "flop_convention": "minimal sparse-tangent"}}

    dev_t = maxrank([r["dev"] for r in records])
    wall_t = maxrank([r["wall"] for r in records])
    bfgs_t = maxrank([r["bfgs"] for r in records])
    bracket = float(maxrank([bracket])[0])
    pso_t = maxrank([r["pso"] for r in records])  # every collective before rank 0 goes on alone
    conv = sum(r["conv"] for r in records)  # global counts (tallies are all-reduced)
    flops_local = sum(r["flops"] for r in records)
    flops_generic = sum(r["flops_generic"] for r in records)
    bfgs_local = sum(r["bfgs"] for r in records)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    achieved = flops_local / bfgs_local / 1e12  # this rank's kernel, TFLOP/s
    traffic = _ncu_traffic(args.config)
    line = {
        "metric": METRIC,
        "value": conv / float(np.sum(dev_t)),
        "unit": "starts/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": float(np.mean(dev_t)) * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (Philox(seed, start) starts, seed 42+step)",
        "config": {"workload": workload_name(args.config, world), "starts_per_gpu": n_per,
                   "parallelism": f"start-sharded x{world}", "l2": "flushed between steps"},
        "time_to_solution_s": float(np.mean(dev_t)),
        "bfgs_ms_per_step": float(np.mean(bfgs_t)) * 1e3,
        "pso_ms_per_step": float(np.mean(pso_t)) * 1e3,
        "bracket_ms_per_step": bracket / args.steps * 1e3,
        "converged_per_step": conv / args.steps,
        "e2e": {"value": conv / float(np.sum(wall_t)), "unit": "starts/s",
                "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": int(records[0]["d2h"]),
                "path": "zeus_run(rastrigin, ZeusConfig(...)) wall time, per-start results "
                        "(x_final, f, |g|, k, status, counters) copied to host every step",
                "inputs": "the call's inputs are (objective, config, seed): kernel arguments "
                          "only; the swarm is generated on the device from the seed by the "
                          "reference's Philox stream (SURVEY S1), as the reference does on "
                          "the host, so no input bytes cross PCIe"},
        "gpu_launches": int(sum(r["launches"] for r in records)),
        "roofline": {"bound": "fp64",
                     "kernel": "BFGS tiers of the step (bfgs_thread -> bfgs_warp -> CTA-team "
                               "straggler kernel); see profiles/*_launches.txt for the shares",
                     "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "peak_source": "measured DFMA microbenchmark (csrc/measure.cu) on this GPU",
                     "flop_convention": "minimal sparse-tangent (paper_2603_28770_b200/roofline.py)",
                     "achieved_generic_convention": flops_generic / bfgs_local / 1e12},
        "clocks": clocks.summary(),
    }
    if ns is not None:
        line["north_star"] = ns
    if not args.no_cpu_baseline and world == 1:  # the CPU baseline is an N = 1 figure
        c, secs, threads = cpu_reference_run(args.config, world, 42)
        line["cpu_baseline"] = {"value": c / secs, "unit": "starts/s", "cores": threads,
                                "kind": "port",
                                "sample": "one full deterministic run of the workload "
                                          "(seed 42) through oracle/ (C restatement)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
