"""CPU: the oracle (oracle/zeus_oracle.c) pinned against golden vectors that
the REFERENCE produced (tests/golden/make_golden.py).

Bit-exact: Philox draws (streams.py), objective values (objectives.py),
forward-AD gradients (autodiff.py), PSO swarms (pso.py), Armijo step
(linesearch.py).  Tolerance (OpenBLAS summation order is implementation
defined): hessian_update and bfgs_run outcomes, SURVEY.md 8(c).
"""

import numpy as np
import pytest

from conftest import BOXES


def test_philox_raw_and_uniform_bit_exact(golden, oracle):
    g = golden("philox")
    for a, seed in enumerate(g["seeds"]):
        for b, i in enumerate(g["parts"]):
            raw = [oracle.philox_u64(int(seed), int(i), k) for k in range(g["raw"].shape[2])]
            assert raw == [int(v) for v in g["raw"][a, b]]
            u0 = oracle.draw_uniform(int(seed), int(i), 0, 13, -5.12, 5.12)
            u1 = oracle.draw_uniform(int(seed), int(i), 13, 13, -10.24, 10.24)
            assert np.array_equal(u0, g["uniform"][a, b, 0])
            assert np.array_equal(u1, g["uniform"][a, b, 1])


def _objective_cases(g):
    return sorted({k.rsplit("_", 1)[0] for k in g.files})


def test_objective_values_and_gradients_bit_exact(golden, oracle):
    g = golden("objectives")
    cases = _objective_cases(g)
    assert len(cases) >= 14
    for case in cases:
        name = case.rsplit("_", 1)[0]
        X, F, G, E = g[case + "_x"], g[case + "_f"], g[case + "_g"], g[case + "_err"]
        for x, f, gr, e in zip(X, F, G, E):
            assert oracle.objective(name, x) == f, (case, x)
            go, err = oracle.gradient(name, x)
            assert err == bool(e), (case, x)
            if not e:
                assert np.array_equal(go, gr), (case, x)


def test_ackley_domain_error_locus(oracle):
    # sqrt'(0): raises at the origin and where sum x^2 underflows to 0
    assert oracle.gradient("ackley", [0.0, 0.0])[1]
    assert oracle.gradient("ackley", [1e-170, 0.0])[1]
    assert not oracle.gradient("ackley", [1e-150, 0.0])[1]


def _pso_tags(g):
    tags = set()
    for k in g.files:
        parts = k.split("_")
        # name may contain '_' (goldstein_price); the tag is name_d_n_seed_sweeps
        for cut in range(2, len(parts)):
            tag = "_".join(parts[:cut])
            if tag + "_gF" in g.files:
                tags.add(tag)
    return sorted(tags)


def _parse_tag(tag, nfields):
    parts = tag.split("_")
    return ["_".join(parts[: len(parts) - nfields])] + [int(p) for p in parts[-nfields:]]


def test_pso_bit_exact(golden, oracle):
    g = golden("pso")
    tags = _pso_tags(g)
    assert len(tags) == 5
    for tag in tags:
        name, d, n, seed, sweeps = _parse_tag(tag, 4)
        lo, hi = BOXES[name]
        init = oracle.pso(name, d, n, seed, lo, hi, 0)
        assert np.array_equal(init.positions, g[tag + "_init_x"])
        assert np.array_equal(init.velocities, g[tag + "_init_v"])
        assert np.array_equal(init.personal_best_val, g[tag + "_init_pval"])
        assert np.array_equal(init.global_best_pos, g[tag + "_init_gX"])
        sw = oracle.pso(name, d, n, seed, lo, hi, sweeps)
        assert np.array_equal(sw.positions, g[tag + "_x"]), tag
        assert np.array_equal(sw.velocities, g[tag + "_v"]), tag
        assert np.array_equal(sw.personal_best_pos, g[tag + "_p"]), tag
        assert np.array_equal(sw.personal_best_val, g[tag + "_pval"]), tag
        assert np.array_equal(sw.global_best_pos, g[tag + "_gX"]), tag
        assert sw.global_best_val == float(g[tag + "_gF"])


def test_armijo_bit_exact(golden, oracle):
    g = golden("linesearch")
    for name, x, p, gr, f0, alpha in zip(g["name"], g["x"], g["p"], g["g"], g["f0"],
                                         g["alpha"]):
        a, trials = oracle.armijo(str(name), x, p, gr, float(f0))
        assert a == alpha
        assert 1 <= trials <= 21


def test_hessian_update_matches_reference(golden, oracle):
    g = golden("hessian")
    for H, dx, dg, out, updated in zip(g["H"], g["dx"], g["dg"], g["out"], g["updated"]):
        H2, upd = oracle.hessian_update(H, dx, dg)
        assert upd == bool(updated)
        # V H V^T through OpenBLAS vs naive loops: relative 1e-13
        assert np.max(np.abs(H2 - out)) <= 1e-13 * np.max(np.abs(out))
        assert np.array_equal(H2, H2.T)


def _bfgs_tags(g):
    return sorted(k[: -len("_starts")] for k in g.files if k.endswith("_starts"))


def test_bfgs_outcomes_match_reference(golden, oracle):
    """statuses identical, |dx|_inf <= 1e-6,
    |df| <= 1e-10 max(1,|f|); iteration counts are reported, not gated."""
    g = golden("bfgs")
    tags = _bfgs_tags(g)
    assert len(tags) == 6
    for tag in tags:
        name, d, n, seed, sweeps, cap = _parse_tag(tag, 5)
        r = oracle.bfgs_batch(name, g[tag + "_starts"], iter_bfgs=cap)
        assert np.array_equal(r.status, g[tag + "_s"]), tag
        ref_x, ref_f = g[tag + "_x"], g[tag + "_f"]
        both_nan = np.isnan(ref_x) & np.isnan(r.x_final)
        dx = np.where(both_nan, 0.0, np.abs(r.x_final - ref_x))
        assert np.max(dx) <= 1e-6, tag
        fin = ~np.isnan(ref_f)
        assert np.array_equal(np.isnan(r.f_final), ~fin)
        # converged starts: 1e-10 relative; starts that hit the cap oscillating
        # around Ackley's kink (|grad| ~ 2.8 at the origin) only agree to 1e-6
        tol = np.where(g[tag + "_s"] == 1, 1e-6, 1e-10)[fin]
        assert np.all(np.abs(r.f_final[fin] - ref_f[fin]) <= tol * np.maximum(1, np.abs(ref_f[fin])))
        best = oracle.reduce_best(r.f_final, r.status)
        assert abs(r.f_final[best] - float(g[tag + "_best_f"])) <= 1e-10 * max(1, abs(r.f_final[best]))


def test_bfgs_classic_rosenbrock(golden, oracle):
    g = golden("bfgs")
    r = oracle.bfgs_batch("rosenbrock", np.array([[-1.2, 1.0]]), iter_bfgs=10_000)
    assert r.status[0] == 0
    assert np.max(np.abs(r.x_final[0] - g["classic_x"])) <= 1e-6
    assert abs(int(r.iterations[0]) - int(g["classic_k"])) <= 3


@pytest.mark.parametrize("name,d", [("rosenbrock", 3), ("rastrigin", 4), ("ackley", 3)])
def test_gradient_agrees_with_central_differences(oracle, name, d):
    rng = np.random.default_rng(20240917)
    lo, hi = BOXES[name]
    for _ in range(50):
        x = rng.uniform(lo, hi, d)
        gr, err = oracle.gradient(name, x)
        assert not err
        for i in range(d):
            h = 1e-6
            xp, xm = x.copy(), x.copy()
            xp[i] += h
            xm[i] -= h
            fd = (oracle.objective(name, xp) - oracle.objective(name, xm)) / (2 * h)
            assert abs(gr[i] - fd) <= max(1e-8, 1e-5 * abs(fd))
