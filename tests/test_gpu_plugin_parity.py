"""User objectives against the REFERENCE's own outcomes (tests/golden/plugin.npz,
made by tests/golden/make_golden_plugin.py running the reference):

* generic Python closures (the reference test-suite's shifted_sphere, the
  README's cos objective) given to zeus_run as plain callables: traced into
  device source (trace.py) and run by the plug-in kernels;
* the spectrum fit (fitting.fit, fitting.py:235-294) on the reference
  test-suite's Poisson and noiseless data sets, with the chi-square traced
  from the model's generic ``predict`` and with the hand-written device
  source of the same model.

Bar: the full-size parity gate of tests/conftest.py (statuses, minimisers
within 1e-6, f within 1e-10; flips only for starts stalled near theta).
"""

import numpy as np
import pytest

from conftest import GOLDEN, gate

pytestmark = pytest.mark.gpu


def golden():
    import os

    return np.load(os.path.join(GOLDEN, "plugin.npz"))


class Ref:
    def __init__(self, g, tag):
        self.x_final, self.f_final, self.grad_norm = g[f"{tag}_x"], g[f"{tag}_f"], g[f"{tag}_gn"]
        self.iterations, self.status = g[f"{tag}_k"], g[f"{tag}_s"]


class Dev:
    def __init__(self, pr):
        self.x_final, self.f_final, self.grad_norm = pr.x_final, pr.f_final, pr.grad_norm
        self.iterations, self.status_codes = pr.iterations, pr.status_codes.astype(np.int64)


def shifted_sphere(x):  # the reference test-suite's closure (tests/test_driver.py)
    total = 0.0
    for i, v in enumerate(x):
        d = v - 0.5 * (i + 1)
        total = total + d * d
    return total


def wavy(x):  # pkg/README.md:72-82, through this package's generic cos
    from paper_2603_28770_b200.autodiff import cos

    total = 0.0
    for v in x:
        total = total + v * v - cos(3.0 * v)
    return total


@pytest.mark.parametrize("tag,fn,d,rng,seed", [("sphere", shifted_sphere, 4, (-3.0, 3.0), 7),
                                              ("wavy", wavy, 6, (-3.0, 3.0), 11)])
def test_python_closure_matches_reference(z, tag, fn, d, rng, seed):
    g = golden()
    cfg = z.ZeusConfig(N=512, dim=d, range=rng, iter_pso=5, iter_bfgs=400, seed=seed,
                       deterministic=True)
    res = z.zeus_run(fn, cfg)   # a plain Python callable: traced, compiled, run on device
    assert abs(res.pso_best_before_bfgs - float(g[f"{tag}_pso_best"])) <= \
        1e-12 * max(1.0, abs(float(g[f"{tag}_pso_best"])))
    gate(f"{tag} (traced closure) vs reference", Dev(res.per_run), Ref(g, tag), 0)


@pytest.mark.parametrize("tag", ["fitp", "fitn"])
@pytest.mark.parametrize("traced", [True, False])
def test_spectrum_fit_matches_reference(z, tag, traced):
    from dataclasses import replace

    from paper_2603_28770_b200 import fitting

    g = golden()
    model = fitting.falling_spectrum(6000.0)
    if traced:
        model = replace(model, device_source=None)  # chi-square traced from predict()
    data = fitting.BinnedDataset(bin_edges=np.linspace(1200.0, 4800.0, 41),
                                 counts=g[f"{tag}_counts"])
    fo = fitting.fit(model, data, [1.0, 0.0, 0.0], [1000.0, 20.0, 10.0], seed=5)
    theta_ref, chi2_ref = g[f"{tag}_theta"], float(g[f"{tag}_chi2"])
    print(f"\n{tag} traced={traced}: theta {fo.theta} vs {tuple(theta_ref)}, chi2 "
          f"{fo.chi_square!r} vs {chi2_ref!r}, statuses {np.bincount(fo.result.per_run.status_codes, minlength=4)}")
    assert np.allclose(fo.theta, theta_ref, rtol=1e-6, atol=1e-6)
    assert abs(fo.chi_square - chi2_ref) <= 1e-8 * max(1.0, chi2_ref)
    unstable = g[f"{tag}_ref_unstable"]
    gate(f"{tag} fit (traced={traced}) vs reference", Dev(fo.result.per_run), Ref(g, tag),
         int(unstable.sum()), ref_unstable=unstable)


def test_untraceable_closure_raises(z):
    """Value-dependent control flow cannot become device code: a clear
    NotImplementedError, never a CPU fallback."""
    def branchy(x):
        return x[0] * x[0] if x[0] > 0 else -x[0]

    cfg = z.ZeusConfig(N=8, dim=2, range=(-1.0, 1.0), iter_pso=1, iter_bfgs=10)
    with pytest.raises(NotImplementedError, match="straight-line"):
        z.zeus_run(branchy, cfg)


def test_traced_rosenbrock_is_the_registered_one(z, oracle):
    """The reference's Rosenbrock text (objectives.py:33-45) as a plain Python
    closure, traced: swarm and BFGS outcomes bit-identical to the registered
    kernel's and equal to the oracle's."""
    def rosenbrock(x):
        total = 0.0
        for i in range(len(x) - 1):
            a = 1.0 - x[i]
            b = x[i + 1] - x[i] * x[i]
            total = total + (a * a + 100.0 * (b * b))
        return total

    cfg = z.ZeusConfig(N=2048, dim=5, range=(-5.0, 5.0), iter_pso=5, iter_bfgs=1000, seed=3,
                       deterministic=True)
    a = z.zeus_run(rosenbrock, cfg)
    b = z.zeus_run(z.rosenbrock, cfg)
    assert a.pso_best_before_bfgs == b.pso_best_before_bfgs
    assert np.array_equal(a.per_run.status_codes, b.per_run.status_codes)
    assert np.max(np.abs(a.per_run.x_final - b.per_run.x_final)) <= 1e-6
    sw = oracle.pso("rosenbrock", 5, 2048, 3, -5.0, 5.0, 5)
    assert a.pso_best_before_bfgs == sw.global_best_val
    g = z.forward_gradient(rosenbrock, [0.3, -0.2, 1.1, 0.7, 0.05])
    g_ref, _ = oracle.gradient("rosenbrock", [0.3, -0.2, 1.1, 0.7, 0.05])
    assert np.array_equal(g, g_ref)
