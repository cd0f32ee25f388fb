"""Turn one gpurun call's ncu output into committed summaries under profiles/.

    python scripts/summarize_profiles.py <tag> --config t50 [--rep R.ncu-rep ...]
                                          [--launches launches.csv]

Writes
  profiles/<tag>_<config>_launches.txt  per-kernel totals of the launch list
                                (ncu --metrics gpu__time_duration.sum
                                --clock-control none) of one bench step of the
                                config, with each kernel's share
  profiles/<tag>_<config>_ncu_<kernel>.txt  key metrics of each `ncu --set
                                full` capture (FP64 pipe, issue, DRAM bytes,
                                stalls)
  profiles/ncu_summary.json     {config: {"kernels": {"<objective><d>":
                                {dram_bytes_per_launch, kernels, sources}}}}
                                read by bench.py for roofline.traffic: each
                                BFGS capture is keyed by the config's problem
                                with that objective (the small-d tiers of one
                                problem are summed: one zeus_run launches
                                them in sequence)
"""

from __future__ import annotations

import argparse
import collections
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__average_warp_latency_per_inst_issued.ratio",
    "sm__cycles_elapsed.avg.per_second",
]
STALLS = "smsp__average_warps_issue_stalled_"


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, mi, ui = (h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Name",
                                            "Metric Unit"))
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                 "nsecond": 1e-3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0] if "<" not in r[ki] else r[ki][: r[ki].index(">") + 1]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", "")) * scale
    return agg


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    res = []
    for row in r[2:]:
        d = dict(zip(h, row))
        m = {"kernel": d["Kernel Name"], "grid": d["Grid Size"], "block": d["Block Size"]}
        for k in KEYS:
            if k in d:
                m[k] = (d[k], u[h.index(k)])
        stalls = {k[len(STALLS):].replace("_per_issue_active.ratio", ""): float(d[k])
                  for k in h if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio")
                  and d[k] not in ("", "n/a")}
        m["stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        res.append(m)
    return res


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--config", required=True)
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--launches", default=None)
    args = ap.parse_args()
    sys.path.insert(0, ROOT)
    from bench import CONFIGS

    probs = CONFIGS[args.config]["problems"]
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    base = f"{args.tag}_{args.config}"
    if args.launches and os.path.exists(args.launches):
        agg = launches(args.launches)
        # bench.py's DFMA peak probe runs before the timed steps: not part of a step
        agg = collections.OrderedDict((k, v) for k, v in agg.items() if "dfma" not in k)
        tot = sum(v[1] for v in agg.values())
        lines = [f"# {base}: ncu --metrics gpu__time_duration.sum --clock-control none of one "
                 f"bench.py step (cold-cache, serialised; shares, not absolutes, compare)",
                 f"# {'launches':>8} {'total_us':>12} {'share':>6}  kernel"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"  {n:8d} {t:12.1f} {100 * t / tot:5.1f}%  {k}")
        open(os.path.join(prof, f"{base}_launches.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    summ_path = os.path.join(prof, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    entry = {"kernels": {}}
    for rep in args.rep:
        for m in raw_metrics(rep):
            kname = m["kernel"].split("(")[0]
            short = kname.replace("void ", "").replace("zeus::", "")
            lines = [f"# {base}: ncu --set full --clock-control none of {short}",
                     f"grid {m['grid']} block {m['block']}"]
            for k in KEYS:
                if k in m:
                    lines.append(f"{k} = {m[k][0]} {m[k][1]}")
            lines.append("top stalls (warps per issue-active cycle): " +
                         ", ".join(f"{k} {v:.3f}" for k, v in m["stalls"].items()))
            safe = "".join(c if c.isalnum() else "_" for c in short)[:60].strip("_")
            fn = os.path.join(prof, f"{base}_ncu_{safe}.txt")
            open(fn, "w").write("\n".join(lines) + "\n")
            print("\n".join(lines))
            if "dram__bytes_read.sum" not in m or not short.startswith("bfgs"):
                continue
            obj = short[short.index("<") + 1:].split(",")[0].split(">")[0].strip().lower()
            dims = {p["d"] for p in probs if p["obj"] == obj}
            if len(dims) != 1 or "nan" in m["dram__bytes_read.sum"][0]:
                continue
            key = f"{obj}{dims.pop()}"
            rd = to_bytes(*m["dram__bytes_read.sum"])
            wr = to_bytes(*m["dram__bytes_write.sum"])
            e = entry["kernels"].setdefault(key, {"dram_bytes_per_launch": 0.0, "kernels": [],
                                                  "sources": []})
            e["kernels"].append(short)
            e["dram_bytes_per_launch"] += rd + wr
            e["sources"].append(os.path.basename(fn))
    if entry["kernels"]:  # merge per problem: a new capture replaces that problem's entry
        cur = summ.get(args.config)
        if not isinstance(cur, dict) or not isinstance(cur.get("kernels"), dict):
            cur = {"kernels": {}}
        cur["kernels"].update(entry["kernels"])
        summ[args.config] = cur
    json.dump(summ, open(summ_path, "w"), indent=1)


if __name__ == "__main__":
    sys.exit(main())
