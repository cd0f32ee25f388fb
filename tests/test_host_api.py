"""CPU: the drop-in boundary -- the C-ABI library loads and exports every
symbol include/zeus_b200.h declares, and the host-side mirror of the
reference's API keeps its names, dataclasses, validation and errors
(driver.py:49-95, pso.py:24-44, linesearch.py:16-37, objectives.py:185-221).
No compute call is made here."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "zeus_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(zeus_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2603_28770_b200 import _capi

    L = _capi.lib()
    declared = _header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_capi.EXPORTED_SYMBOLS) == declared
    assert L.zeus_abi_version() == _capi.ABI_VERSION == 2
    assert L.zeus_pso_workspace_bytes(1000) >= 16


def test_library_is_sm100a():
    import subprocess

    from paper_2603_28770_b200 import _capi

    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_public_namespace_matches_reference():
    import paper_2603_28770_b200 as z

    reference_all = ["Dual", "DomainError", "forward_gradient", "BfgsOutcome", "bfgs_run",
                     "hessian_update", "CONVERGED", "DIVERGED", "STOPPED", "DOMAIN_ERROR",
                     "LineSearchParams", "armijo_search", "PsoParams", "SwarmState",
                     "init_swarm", "update_swarm", "ObjectiveSpec", "get_objective",
                     "objective_names", "ZeusConfig", "ZeusResult", "zeus_run", "reduce_best",
                     "make_start_streams", "NoValidOptimumError", "__version__"]
    missing = [n for n in reference_all if not hasattr(z, n)]
    assert missing == []
    from paper_2603_28770_b200 import autodiff

    for n in ("Dual", "DomainError", "exp", "cos", "sin", "sqrt", "log", "powf",
              "forward_gradient"):   # zeus/autodiff.py:19-29
        assert hasattr(autodiff, n), n
    assert (z.CONVERGED, z.DIVERGED, z.STOPPED, z.DOMAIN_ERROR) == (
        "converged", "diverged", "stopped", "domain_error")


def test_config_validation(z):
    cfg = z.ZeusConfig(N=12, dim=2, range=(-1.0, 1.0))
    assert cfg.required_c == 12
    for kw in (dict(N=0), dict(range=(1.0, -1.0)), dict(required_c=5), dict(theta=0.0),
               dict(workers=-1), dict(iter_pso=-1)):
        args = dict(N=4, dim=2, range=(-1.0, 1.0))
        args.update(kw)
        with pytest.raises(ValueError):
            z.ZeusConfig(**args)
    cfg = z.ZeusConfig(N=4, dim=2, range=(-1.0, 1.0), iter_pso=7, iter_ls=9)
    assert cfg.pso.iter_pso == 7 and cfg.ls.iter_ls == 9


def test_param_validation(z):
    p = z.PsoParams()
    assert (p.w, p.c1_pso, p.c2_pso) == (0.5, 1.2, 1.5)
    z.PsoParams(w=0.0, c1_pso=0.0, c2_pso=0.0)
    with pytest.raises(ValueError):
        z.PsoParams(w=-0.1)
    ls = z.LineSearchParams()
    assert (ls.c1_armijo, ls.alpha0, ls.iter_ls, ls.shrink) == (0.3, 1.0, 20, 0.5)
    for kw in (dict(c1_armijo=0.0), dict(c1_armijo=1.0), dict(shrink=1.5), dict(iter_ls=0),
               dict(alpha0=0.0)):
        with pytest.raises(ValueError):
            z.LineSearchParams(**kw)


def test_registry(z):
    assert z.objective_names() == ["ackley", "goldstein_price", "rastrigin", "rosenbrock"]
    spec = z.get_objective("rastrigin", 3)
    assert (spec.lower, spec.upper, spec.optimum_x, spec.optimum_f) == (-5.12, 5.12,
                                                                         (0.0,) * 3, 0.0)
    assert z.get_objective("goldstein_price", 2).optimum_x == (0.0, -1.0)
    assert not z.get_objective("ackley", 2).gradient_continuous
    with pytest.raises(KeyError):
        z.get_objective("sphere")
    with pytest.raises(ValueError):
        z.get_objective("goldstein_price", 3)
    with pytest.raises(ValueError):
        z.get_objective("rosenbrock", 1)


def test_objective_mapping(z):
    from paper_2603_28770_b200 import _capi

    assert z.objective_id(z.rosenbrock) == _capi.OBJ_ROSENBROCK
    assert z.objective_id(z.get_objective("ackley", 4)) == _capi.OBJ_ACKLEY
    assert z.objective_id("goldstein_price", 2) == _capi.OBJ_GOLDSTEIN_PRICE

    def rastrigin(x):  # the reference's function, recognised by module + name
        return 0.0
    rastrigin.__module__ = "zeus.objectives"
    assert z.objective_id(rastrigin) == _capi.OBJ_RASTRIGIN
    with pytest.raises(NotImplementedError):
        z.objective_id(lambda x: 0.0)
    with pytest.raises(ValueError):
        z.objective_id(z.goldstein_price, 3)


def test_reduce_best_on_lists(z):
    def outcome(f, status=z.CONVERGED):
        return z.BfgsOutcome(x_final=(0.0,), f_final=f, grad_norm=0.0, iterations=1,
                             status=status)
    only = outcome(3.0)
    assert z.reduce_best([only]) == (only, 0)
    a, b = outcome(1.0), outcome(1.0)
    best, idx = z.reduce_best([a, b])
    assert best is a and idx == 0
    bad, good = outcome(-100.0, z.DOMAIN_ERROR), outcome(5.0)
    assert z.reduce_best([bad, good]) == (good, 1)
    assert z.reduce_best([outcome(float("nan")), good]) == (good, 1)
    with pytest.raises(z.NoValidOptimumError):
        z.reduce_best([outcome(1.0, z.DOMAIN_ERROR)])
    with pytest.raises(z.NoValidOptimumError):
        z.reduce_best([])


def test_outcome_list_semantics(z):
    x = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    f = np.array([2.0, 1.0, 1.0])
    gn = np.array([1e-7, 1e-8, 0.5])
    it = np.array([3, 4, 5], dtype=np.int32)
    st = np.array([0, 0, 1], dtype=np.uint8)
    ol = z.OutcomeList(x, f, gn, it, st)
    assert len(ol) == 3
    assert ol[1] == z.BfgsOutcome((3.0, 4.0), 1.0, 1e-8, 4, "converged")
    assert ol[-1].status == "diverged"
    assert ol == list(ol) and ol[0:2] == [ol[0], ol[1]]
    assert z.reduce_best(ol) == (ol[1], 1)
    short = z.OutcomeList(x, f, gn, it, st, length=2)
    assert len(short) == 2 and list(short.iterations) == [3, 4]
    with pytest.raises(IndexError):
        ol[3]


@pytest.mark.parametrize("n,world", [(10, 3), (1, 8), (65536, 8), (7, 7), (1000, 1)])
def test_shard_bounds_partition(n, world):
    from paper_2603_28770_b200.engine import shard_bounds

    covered = []
    for r in range(world):
        lo, hi = shard_bounds(n, r, world)
        assert 0 <= lo <= hi <= n
        covered.extend(range(lo, hi))
    assert covered == list(range(n))


def test_no_cpu_fallback_without_gpu(z):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_28770_b200._capi import ZeusNativeError

    cfg = z.ZeusConfig(N=4, dim=2, range=(-1.0, 1.0))
    with pytest.raises(ZeusNativeError):
        z.zeus_run(z.rosenbrock, cfg)
    with pytest.raises(ZeusNativeError):
        z.rosenbrock([1.0, 1.0])


def test_abi_structs_match_the_header(tmp_path):
    """The ctypes mirrors of zeus_bfgs_out / zeus_bfgs_params have the C
    layout of include/zeus_b200.h (size and every field offset, compiled
    with the host C compiler): a drift would hand the kernels garbage
    pointers."""
    import ctypes
    import subprocess

    from paper_2603_28770_b200 import _capi

    fields = {"zeus_bfgs_out": [f for f, _ in _capi.BfgsOut._fields_],
              "zeus_bfgs_params": [f for f, _ in _capi.BfgsParams._fields_]}
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "zeus_b200.h"', 'int main(void) {']
    for st, fs in fields.items():
        src.append(f'  printf("{st} %zu\\n", sizeof({st}));')
        src += [f'  printf("{st}.{f} %zu\\n", offsetof({st}, {f}));' for f in fs]
    src.append("  return 0;\n}")
    c = tmp_path / "abi.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)],
                   check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True,
                                                       text=True, check=True).stdout.splitlines())
    for st, cls in (("zeus_bfgs_out", _capi.BfgsOut), ("zeus_bfgs_params", _capi.BfgsParams)):
        assert int(got[st]) == ctypes.sizeof(cls), st
        for f in fields[st]:
            assert int(got[f"{st}.{f}"]) == getattr(cls, f).offset, (st, f)


def test_early_stop_waves_cover_every_start(monkeypatch):
    """run_bfgs in the parallel early-stop mode (driver.py:153-202 pool
    semantics): launches of wave, 2 wave, 4 wave, ... starts, contiguous and
    covering [0, n) exactly once."""
    import torch

    from paper_2603_28770_b200 import engine

    calls = []
    monkeypatch.setattr(engine, "_run_bfgs_slice",
                        lambda obj, x0, params, out, device, rc, stop, ws, lo, m:
                        calls.append((lo, m)))
    monkeypatch.setattr(engine._device, "workspace", lambda nbytes, dev: None)

    class _L:
        @staticmethod
        def zeus_bfgs_workspace_bytes(d, n):
            return 0

    monkeypatch.setattr(engine._capi, "lib", lambda: _L)
    x0 = torch.zeros((3, 1000), dtype=torch.float64)
    engine.run_bfgs(0, x0, None, None, "cpu", required_c=5, stop=(0, 0), wave=7)
    assert [m for _, m in calls] == [7, 14, 28, 56, 112, 224, 448, 111]
    assert calls[0][0] == 0 and all(a + m == b for (a, m), (b, _) in zip(calls, calls[1:]))
    assert sum(m for _, m in calls) == 1000
    calls.clear()
    engine.run_bfgs(0, x0, None, None, "cpu", required_c=5, stop=None, wave=7)
    assert calls == [(0, 1000)]  # no stop block: one launch
