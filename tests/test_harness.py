"""Experiment harness + CLI on the GPU path (the reference's bench.py / cli.py,
SURVEY.md 8(f) rows 2 and 4).  CPU tests: plan parsing and grid expansion,
record formats (the reference's CSV header and JSONL schema), metrics, CLI
exit codes.  GPU tests: a plan run end to end, the device n_correct count, the
CLI commands."""

import json
import math

import numpy as np
import pytest

from paper_2603_28770_b200 import bench, cli
from paper_2603_28770_b200.bfgs import BfgsOutcome

# the reference's header (zeus/bench.py:56-76), verbatim
REF_HEADER = ("experiment,objective,dim,N,iter_pso,iter_bfgs,required_c,seed,rep,wall_time_s,"
              "best_f,euclid_error,n_correct,converged,diverged,stopped,domain_error")


def _plan(tmp_path, text):
    p = tmp_path / "plan.ini"
    p.write_text(text)
    return p


def test_csv_header_matches_reference():
    assert bench.CSV_HEADER == REF_HEADER


def test_grid_expansion_labels_and_seeds(tmp_path):
    p = _plan(tmp_path, "[plan]\nrepetitions = 3\noutput = out/res\n\n"
                        "[scan]\nobjective = rastrigin\ndim = 2, 5\nN = 100, 200\niter_pso = 4\n"
                        "deterministic = yes\n\n[one]\nobjective = rosenbrock\n")
    plan = bench.parse_plan(p, base_seed=7)
    names = [e.experiment for e in plan.entries]
    assert names == ["scan[dim=2,N=100]", "scan[dim=2,N=200]", "scan[dim=5,N=100]",
                     "scan[dim=5,N=200]", "one"]
    assert plan.repetitions == 3 and plan.base_seed == 7 and str(plan.output) == "out/res"
    e = plan.entries[3].config
    assert (e.dim, e.N, e.iter_pso, e.deterministic, e.seed) == (5, 200, 4, True, 7)
    assert plan.entries[4].config.N == 1024 and plan.entries[4].config.dim == 2
    assert plan.entries[4].config.range == (-5.0, 5.0)


@pytest.mark.parametrize("text,err", [
    ("[a]\ndim = 2\n", "missing the 'objective'"),
    ("[a]\nobjective = rastrigin\nbogus = 1\n", "unknown keys"),
    ("[a]\nobjective = rastrigin\ndeterministic = yes, no\n", "cannot take a value list"),
    ("[a]\nobjective = rastrigin\ndeterministic = maybe\n", "not a boolean"),
    ("[plan]\nrepetitions = 0\n[a]\nobjective = rastrigin\n", "at least 1"),
    ("[plan]\nrepetitions = 1\n", "no experiments"),
    ("[plan]\nrounds = 2\n[a]\nobjective = rastrigin\n", "unknown keys"),
])
def test_plan_errors(tmp_path, text, err):
    with pytest.raises(bench.PlanError, match=err):
        bench.parse_plan(_plan(tmp_path, text), base_seed=0)


def test_plan_unreadable(tmp_path):
    with pytest.raises(OSError):
        bench.parse_plan(tmp_path / "missing.ini", base_seed=0)


def _record(**kw):
    base = dict(experiment="e", objective="rastrigin", dim=2, N=10, iter_pso=1, iter_bfgs=5,
                required_c=10, seed=3, rep=0, wall_time_s=0.25, best_f=1e-9,
                best_point=(0.1, -0.2), euclid_error=0.2236, n_correct=7, converged=9,
                diverged=1, stopped=0, domain_error=0)
    base.update(kw)
    return bench.RunRecord(**base)


def test_record_formats_round_trip(tmp_path):
    recs = [_record(), _record(rep=1, best_f=float("nan"), euclid_error=math.nan)]
    csv = bench.emit_results(recs, "csv", tmp_path / "r.csv").read_text().splitlines()
    assert csv[0] == REF_HEADER
    assert csv[1] == "e,rastrigin,2,10,1,5,10,3,0,0.25,1e-09,0.2236,7,9,1,0,0"
    jl = bench.emit_results(recs, "json-lines", tmp_path / "r.jsonl")
    back = bench.read_records(jl)
    assert back[0] == recs[0] and back[1].rep == 1 and math.isnan(back[1].best_f)
    assert json.loads(jl.read_text().splitlines()[0])["best_point"] == [0.1, -0.2]
    with pytest.raises(ValueError):
        bench.emit_results(recs, "xml", tmp_path / "r.xml")


def test_metrics():
    assert bench.euclidean_error((3.0, 4.0), (0.0, 0.0)) == 5.0
    outs = [BfgsOutcome(x_final=(0.1, 0.1), f_final=0.0, grad_norm=0.0, iterations=1,
                        status="converged"),
            BfgsOutcome(x_final=(0.5, 0.0), f_final=0.0, grad_norm=0.0, iterations=1,
                        status="converged"),   # exactly on the radius: not within
            BfgsOutcome(x_final=(2.0, 0.0), f_final=0.0, grad_norm=0.0, iterations=1,
                        status="diverged")]
    assert bench.count_within(outs, (0.0, 0.0)) == 1
    assert bench.count_within(outs, (0.0, 0.0), radius=3.0) == 3


def test_cli_config_errors(capsys):
    assert cli.main([]) == cli.EXIT_CONFIG                       # usage error -> 1, not 2
    assert cli.main(["run", "--objective", "nope"]) == cli.EXIT_CONFIG
    assert cli.main(["run", "--objective", "goldstein_price", "--dim", "3"]) == cli.EXIT_CONFIG
    assert cli.main(["fit"]) == cli.EXIT_CONFIG                  # needs --data or --demo
    assert cli.main(["bench", "--plan", "/nonexistent.ini", "--seed", "1"]) == cli.EXIT_IO


@pytest.mark.gpu
def test_run_experiment_on_gpu(tmp_path, z):
    p = _plan(tmp_path, f"[plan]\nrepetitions = 2\noutput = {tmp_path}/res\n\n"
                        "[r]\nobjective = rastrigin\ndim = 2, 3\nN = 500\niter_pso = 3\n"
                        "iter_bfgs = 200\ndeterministic = true\n")
    plan = bench.parse_plan(p, base_seed=11)
    seen = []
    recs = bench.run_experiment(plan, progress=seen.append)
    assert len(recs) == 4 and seen == recs
    assert [r.seed for r in recs] == [11, 12, 11, 12]
    for r in recs:
        cfg = z.ZeusConfig(N=500, dim=r.dim, range=(-5.12, 5.12), iter_pso=3, iter_bfgs=200,
                           seed=r.seed, deterministic=True)
        res = z.zeus_run(z.rastrigin, cfg)
        # device n_correct == the reference's per-outcome definition
        assert r.n_correct == bench.count_within(list(res.per_run), (0.0,) * r.dim)
        assert r.best_f == res.best.f_final
        assert r.converged + r.diverged + r.stopped + r.domain_error == 500
        assert r.euclid_error == bench.euclidean_error(res.best.x_final, (0.0,) * r.dim)
    assert bench.read_records(tmp_path / "res.jsonl") == recs


@pytest.mark.gpu
def test_cli_run_and_audit(capsys):
    assert cli.main(["run", "--objective", "rastrigin", "--dim", "3", "--N", "256",
                     "--seed", "4", "--json"]) == cli.EXIT_OK
    out = json.loads(capsys.readouterr().out)
    assert out["launched"] == 256 and len(out["best_x"]) == 3 and "euclid_error" in out
    assert cli.main(["ackley-audit", "--N", "400", "--seed", "1"]) == cli.EXIT_OK
    text = capsys.readouterr().out
    assert "runs diverged" in text and "audit " in text


@pytest.mark.gpu
def test_ackley_audit_populations():
    au = bench.ackley_audit(n=1000, seed=0)
    pr = au.result.per_run
    for i, dist in au.diverged_near_origin:
        assert pr[i].status == "diverged" and dist < 0.1
    for i, f in au.converged_high:
        assert pr[i].status == "converged" and f > 1.0
    assert au.flagged


def test_config5_tradeoff_plan_parses():
    """BASELINE config 5's grid as a harness plan (plans/tradeoff-c5.ini):
    PSO sweeps {0,5,20,100} x starts 2^10..2^20 x BFGS depth {16,128,1024}."""
    import os

    from paper_2603_28770_b200 import bench as hb

    path = os.path.join(os.path.dirname(hb.__file__), "plans", "tradeoff-c5.ini")
    plan = hb.parse_plan(path, 42)
    assert len(plan.entries) == 72
    grid = {(e.config.iter_pso, e.config.N, e.config.iter_bfgs) for e in plan.entries}
    assert grid == {(s, n, k) for s in (0, 5, 20, 100) for n in (2**10, 2**12, 2**14, 2**16,
                                                                  2**18, 2**20)
                    for k in (16, 128, 1024)}
    assert all(e.config.deterministic and e.spec.dim == 20 for e in plan.entries)
