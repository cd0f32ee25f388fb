"""Experiment harness on the GPU path (the reference's zeus/bench.py, SURVEY.md
8(f) row 2): plan files -> grids of zeus_run calls -> one record per run,
streamed as JSON lines and written as the reference's fixed-header CSV.

The record schema, plan syntax, seed rule (rep r runs seed base + r), CSV
header and JSONL round trip are the reference's (bench.py:56-141,
bench.py:166-395), so result files of both implementations are
interchangeable.  What moves to the device: every pipeline run, and the two
per-run metrics over all N starts -- ``n_correct`` (starts whose final point
lies within CORRECT_RADIUS of the known optimum, bench.py:113-126) is counted
by a kernel (zeus_count_within) on the device copy of the final points before
they leave HBM; ``euclid_error`` is the best point's distance.
"""

from __future__ import annotations

import configparser
import dataclasses
import json
import math
import statistics
from dataclasses import dataclass, replace
from pathlib import Path
from typing import Callable, Iterable, Sequence

import numpy as np

from .bfgs import CONVERGED, DIVERGED, DOMAIN_ERROR, STOPPED, BfgsOutcome
from .driver import OutcomeList, ZeusConfig, ZeusResult, zeus_run
from .linesearch import LineSearchParams
from .objectives import ObjectiveSpec, get_objective
from .pso import PsoParams

__all__ = [
    "CSV_HEADER", "CORRECT_RADIUS", "STRICT_RADIUS", "RunRecord", "ExperimentPlan",
    "PlanEntry", "PlanError", "parse_plan", "run_experiment", "emit_results",
    "read_records", "count_within", "euclidean_error", "speedup_study", "SpeedupRow",
    "ackley_audit", "AckleyAudit",
]

CORRECT_RADIUS = 0.5     # bench.py:49-53: "correct" local solution radius
STRICT_RADIUS = 1e-6

# column order of the reference's CSV (bench.py:56-75); best_point is JSONL-only
CSV_COLUMNS = ("experiment", "objective", "dim", "N", "iter_pso", "iter_bfgs", "required_c",
               "seed", "rep", "wall_time_s", "best_f", "euclid_error", "n_correct",
               "converged", "diverged", "stopped", "domain_error")
CSV_HEADER = ",".join(CSV_COLUMNS)


class PlanError(ValueError):
    """Malformed or inconsistent plan file (bench.py:78-79)."""


def _csv_cell(v) -> str:
    return repr(v) if isinstance(v, float) else str(v)


@dataclass(frozen=True)
class RunRecord:
    """One pipeline execution's metrics (bench.py:82-121)."""

    experiment: str
    objective: str
    dim: int
    N: int
    iter_pso: int
    iter_bfgs: int
    required_c: int
    seed: int
    rep: int
    wall_time_s: float
    best_f: float
    best_point: tuple[float, ...]
    euclid_error: float
    n_correct: int
    converged: int
    diverged: int
    stopped: int
    domain_error: int

    def csv_row(self) -> str:
        return ",".join(_csv_cell(getattr(self, c)) for c in CSV_COLUMNS)

    def to_json(self) -> str:
        d = dataclasses.asdict(self)
        d["best_point"] = list(self.best_point)
        return json.dumps(d)

    @classmethod
    def from_json(cls, line: str) -> "RunRecord":
        d = json.loads(line)
        d["best_point"] = tuple(d["best_point"])
        return cls(**d)


def euclidean_error(point: Sequence[float], optimum: Sequence[float]) -> float:
    """|point - optimum|_2 (bench.py:124-128)."""
    diff = np.asarray(point, dtype=float) - np.asarray(optimum, dtype=float)
    return float(np.linalg.norm(diff))


def count_within(outcomes: Iterable[BfgsOutcome], optimum: Sequence[float],
                 radius: float = CORRECT_RADIUS) -> int:
    """Outcomes whose final point is strictly within ``radius`` of ``optimum``
    (bench.py:131-141).  A per_run of zeus_run is counted column-wise from its
    host SoA copy (no per-outcome objects); zeus_run itself counts on device
    when given ``within=`` (see run_experiment)."""
    target = np.asarray(optimum, dtype=float)
    if isinstance(outcomes, OutcomeList):
        x = outcomes.x_final
        if len(x) == 0:
            return 0
        return int(np.count_nonzero(np.linalg.norm(x - target[None, :], axis=1) < radius))
    return sum(1 for o in outcomes
               if float(np.linalg.norm(np.asarray(o.x_final) - target)) < radius)


@dataclass(frozen=True)
class PlanEntry:
    """A grid point: experiment id, objective, configuration (bench.py:144-150)."""

    experiment: str
    spec: ObjectiveSpec
    config: ZeusConfig


@dataclass
class ExperimentPlan:
    """Expanded plan (bench.py:153-166)."""

    entries: list[PlanEntry]
    repetitions: int
    base_seed: int
    output: Path | None = None

    def __post_init__(self):
        if self.repetitions < 1:
            raise PlanError("repetitions must be at least 1")
        if not self.entries:
            raise PlanError("plan has no experiments")


# plan keys by value type (bench.py:169-176)
_INT = frozenset({"dim", "N", "iter_pso", "iter_bfgs", "iter_ls", "required_c", "workers"})
_FLOAT = frozenset({"theta", "lower", "upper", "w", "c1_pso", "c2_pso", "c1_armijo",
                    "alpha0", "shrink"})
_BOOL = frozenset({"deterministic"})
_GRIDDABLE = _INT | _FLOAT | {"objective"}
_ALLOWED = _GRIDDABLE | _BOOL
_PLAN_SECTION_KEYS = frozenset({"repetitions", "output"})
_TRUE, _FALSE = ("true", "yes", "on", "1"), ("false", "no", "off", "0")


def _value(key: str, text: str):
    if key in _INT:
        return int(text)
    if key in _FLOAT:
        return float(text)
    if key in _BOOL:
        t = text.strip().lower()
        if t in _TRUE:
            return True
        if t in _FALSE:
            return False
        raise PlanError(f"not a boolean: {text!r}")
    return text.strip()


def _grid_points(section: str, raw: dict[str, str]) -> list[tuple[str, dict]]:
    """Cartesian expansion of one experiment section; labels list the varied
    keys in file order, e.g. ``name[N=1000,dim=5]`` (bench.py:196-228)."""
    bad = sorted(set(raw) - _ALLOWED)
    if bad:
        raise PlanError(f"[{section}] has unknown keys: {', '.join(bad)}")
    if "objective" not in raw:
        raise PlanError(f"[{section}] is missing the 'objective' key")
    fixed, axes = {}, []
    for key, text in raw.items():
        vals = [_value(key, part.strip()) for part in text.split(",") if part.strip()]
        if not vals:
            raise PlanError(f"[{section}] key {key!r} has no value")
        if len(vals) == 1:
            fixed[key] = vals[0]
        elif key in _GRIDDABLE:
            axes.append((key, vals))
        else:
            raise PlanError(f"[{section}] key {key!r} cannot take a value list")
    points = [({}, [])]
    for key, vals in axes:
        points = [({**chosen, key: v}, label + [f"{key}={v}"])
                  for chosen, label in points for v in vals]
    return [(section + (f"[{','.join(label)}]" if label else ""), {**fixed, **chosen})
            for chosen, label in points]


def _entry(experiment: str, point: dict, seed: int) -> PlanEntry:
    p = dict(point)
    spec = get_objective(p.pop("objective"), p.pop("dim", 2))
    box = (p.pop("lower", spec.lower), p.pop("upper", spec.upper))
    pso = PsoParams(**{k: p.pop(k) for k in ("w", "c1_pso", "c2_pso") if k in p})
    ls = LineSearchParams(**{k: p.pop(k) for k in ("c1_armijo", "alpha0", "shrink") if k in p})
    cfg = ZeusConfig(N=p.pop("N", 1024), dim=spec.dim, range=box, seed=seed, pso=pso, ls=ls, **p)
    return PlanEntry(experiment=experiment, spec=spec, config=cfg)


def parse_plan(path, base_seed: int, output=None) -> ExperimentPlan:
    """Load and expand an INI plan (bench.py:231-283): one optional ``[plan]``
    section (repetitions, output) plus one section per experiment; the seed
    comes from the caller, never the file."""
    cp = configparser.ConfigParser(interpolation=None)
    cp.optionxform = str  # N and n are different keys
    if not cp.read(str(path)):
        raise OSError(f"cannot read plan file: {path}")
    reps = 1
    if cp.has_section("plan"):
        head = dict(cp.items("plan"))
        bad = sorted(set(head) - _PLAN_SECTION_KEYS)
        if bad:
            raise PlanError(f"[plan] has unknown keys: {', '.join(bad)}")
        reps = int(head.get("repetitions", 1))
        if output is None:
            output = head.get("output")
    entries = [_entry(name, point, base_seed)
               for section in cp.sections() if section != "plan"
               for name, point in _grid_points(section, dict(cp.items(section)))]
    return ExperimentPlan(entries=entries, repetitions=reps, base_seed=base_seed,
                          output=None if output is None else Path(output))


def _record(entry: PlanEntry, rep: int, result: ZeusResult) -> RunRecord:
    spec, cfg = entry.spec, entry.config
    counts = (result.stats.status_counts if result.stats is not None else
              {s: sum(1 for o in result.per_run if o.status == s)
               for s in (CONVERGED, DIVERGED, STOPPED, DOMAIN_ERROR)})
    if spec.optimum_x is None:
        err, n_ok = math.nan, 0
    else:
        err = euclidean_error(result.best.x_final, spec.optimum_x)
        n_ok = (result.stats.n_within if result.stats is not None
                and result.stats.n_within is not None
                else count_within(result.per_run, spec.optimum_x))
    return RunRecord(
        experiment=entry.experiment, objective=spec.name, dim=cfg.dim, N=cfg.N,
        iter_pso=cfg.iter_pso, iter_bfgs=cfg.iter_bfgs, required_c=cfg.required_c,
        seed=cfg.seed, rep=rep, wall_time_s=result.wall_time, best_f=result.best.f_final,
        best_point=result.best.x_final, euclid_error=err, n_correct=int(n_ok),
        converged=counts[CONVERGED], diverged=counts[DIVERGED], stopped=counts[STOPPED],
        domain_error=counts[DOMAIN_ERROR])


def run_experiment(plan: ExperimentPlan,
                   progress: Callable[[RunRecord], None] | None = None) -> list[RunRecord]:
    """Run every grid point ``plan.repetitions`` times, one pipeline at a time
    (bench.py:344-376); records are appended to ``<output>.jsonl`` as they
    complete, so an interrupted run keeps what finished."""
    records: list[RunRecord] = []
    sink = None
    if plan.output is not None:
        plan.output.parent.mkdir(parents=True, exist_ok=True)
        sink = open(plan.output.with_suffix(".jsonl"), "a")
    try:
        for entry in plan.entries:
            for rep in range(plan.repetitions):
                cfg = replace(entry.config, seed=plan.base_seed + rep)
                within = None
                if entry.spec.optimum_x is not None:
                    within = (entry.spec.optimum_x, CORRECT_RADIUS)
                result = zeus_run(entry.spec.fn, cfg, within=within)
                rec = _record(replace(entry, config=cfg), rep, result)
                records.append(rec)
                if sink is not None:
                    sink.write(rec.to_json() + "\n")
                    sink.flush()
                if progress is not None:
                    progress(rec)
    finally:
        if sink is not None:
            sink.close()
    return records


def emit_results(records: Sequence[RunRecord], fmt: str, path) -> Path:
    """``csv`` (fixed header, no best_point) or ``jsonl`` / ``json-lines``
    (bench.py:379-395)."""
    fmt = "jsonl" if fmt == "json-lines" else fmt
    if fmt not in ("csv", "jsonl"):
        raise ValueError(f"unknown results format: {fmt!r}")
    path = Path(path)
    lines = ([CSV_HEADER] + [r.csv_row() for r in records] if fmt == "csv"
             else [r.to_json() for r in records])
    path.write_text("".join(line + "\n" for line in lines))
    return path


def read_records(path) -> list[RunRecord]:
    """Records back from a JSON-lines file (bench.py:398-407)."""
    with open(path) as fh:
        return [RunRecord.from_json(line) for line in (raw.strip() for raw in fh) if line]


@dataclass(frozen=True)
class SpeedupRow:
    workers: int
    wall_time: float
    speedup: float


def speedup_study(f: Callable, cfg: ZeusConfig, worker_counts: Sequence[int],
                  repetitions: int = 5) -> list[SpeedupRow]:
    """Median wall time per worker count and speedup vs 1 worker
    (bench.py:417-449).  On the GPU path ``workers`` only selects the device
    early-stop protocol (workers > 0), so the rows measure that protocol's
    cost, not a process pool."""
    if repetitions < 5:
        raise ValueError("speedup_study needs at least 5 repetitions")
    counts = list(worker_counts)
    if 1 not in counts:
        counts = [1] + counts
    med = {}
    for w in counts:
        run_cfg = replace(cfg, workers=w, deterministic=False)
        med[w] = statistics.median(zeus_run(f, run_cfg).wall_time for _ in range(repetitions))
    return [SpeedupRow(workers=w, wall_time=med[w], speedup=med[1] / med[w]) for w in counts]


@dataclass
class AckleyAudit:
    """The two populations that show the gradient test misfiring on Ackley
    (bench.py:452-466)."""

    result: ZeusResult
    diverged_near_origin: list[tuple[int, float]]
    converged_high: list[tuple[int, float]]

    @property
    def flagged(self) -> bool:
        return bool(self.diverged_near_origin) and bool(self.converged_high)


def ackley_audit(n: int = 1000, seed: int = 0, theta: float = 1e-6, iter_bfgs: int = 150,
                 workers: int = 0, near_radius: float = 0.1,
                 high_value: float = 1.0) -> AckleyAudit:
    """2-D Ackley without PSO (bench.py:469-503): runs that reach the origin
    exhaust the budget (no derivative at the minimum) while runs caught in
    outer local minima report convergence at f > 1."""
    spec = get_objective("ackley", 2)
    cfg = ZeusConfig(N=n, dim=2, range=(spec.lower, spec.upper), iter_pso=0,
                     iter_bfgs=iter_bfgs, theta=theta, required_c=n, seed=seed, workers=workers)
    result = zeus_run(spec.fn, cfg)
    pr = result.per_run
    dist = np.linalg.norm(pr.x_final, axis=1)
    st, f = pr.status_codes, pr.f_final
    near = np.flatnonzero((st == 1) & (dist < near_radius))
    high = np.flatnonzero((st == 0) & ~(dist < near_radius) & (f > high_value))
    return AckleyAudit(result=result,
                       diverged_near_origin=[(int(i), float(dist[i])) for i in near],
                       converged_high=[(int(i), float(f[i])) for i in high])
