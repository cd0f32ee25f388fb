"""User objectives as device plug-ins (the reference's
generic-scalar contract, pkg/README.md:70-87) and the GPU fitting module
(the reference's fitting.py) built on them.

CPU tests: dataset handling / validation (no device needed).  GPU tests:
NVRTC compile + value kernel vs numpy, zeus_run on a plug-in that restates a
registered objective (same PSO swarm bit for bit, same statuses, minimisers
within the stated tolerance), DomainError -> domain_error, compile errors,
the chi^2 spectrum fit recovering the generating parameters, CLI `fit`."""

import math

import numpy as np
import pytest

from conftest import assert_outcomes_close
from paper_2603_28770_b200 import cli, fitting

RASTRIGIN_SRC = """
template <class T, class X>
__device__ T objective(const X& x, int d, const double* data, bool& err) {
  T total = 10.0 * d;  // objectives.py:48-61, reference order
  for (int i = 0; i < d; ++i) total = total + (x(i) * x(i) - 10.0 * zu::cos(zeus::two_pi() * x(i)));
  return total;
}
"""

WAVY_SRC = """
template <class T, class X>
__device__ T objective(const X& x, int d, const double* data, bool& err) {
  T total = 0.0;
  for (int i = 0; i < d; ++i) total = total + data[i] * x(i) * x(i) - zu::cos(3.0 * x(i));
  return total;
}
"""


# ---- CPU: datasets -----------------------------------------------------------
def test_dataset_validation_and_io(tmp_path):
    d = fitting.BinnedDataset(bin_edges=[0, 1, 2, 4], counts=[0, 4, 9])
    assert np.array_equal(d.sigma, [1.0, 2.0, 3.0]) and d.n_bins == 3
    assert np.array_equal(d.centers, [0.5, 1.5, 3.0])
    for bad in (dict(bin_edges=[0, 1], counts=[1, 2]), dict(bin_edges=[0, 2, 1], counts=[1, 2]),
                dict(bin_edges=[0, 1, 2], counts=[1, -1]),
                dict(bin_edges=[0, 1, 2], counts=[1, 1], sigma=[1, 0])):
        with pytest.raises(ValueError):
            fitting.BinnedDataset(**bad)
    p = tmp_path / "d.txt"
    fitting.save_dataset(d, p)
    back = fitting.load_dataset(p)
    assert np.array_equal(back.bin_edges, d.bin_edges) and np.array_equal(back.sigma, d.sigma)
    p.write_text("# comment\n0, 1, 5\n1 2 6 # trailing\n\n2 3 7\n")
    assert np.array_equal(fitting.load_dataset(p).counts, [5, 6, 7])
    p.write_text("0 1 5\n1.5 2 6\n")
    with pytest.raises(ValueError, match="contiguous"):
        fitting.load_dataset(p)
    p.write_text("0 1 5\n1 2\n")
    with pytest.raises(ValueError, match="columns"):
        fitting.load_dataset(p)


def test_falling_spectrum_host_model():
    m = fitting.falling_spectrum(6000.0)
    v = m.predict((50.0, 10.0, 5.0), 3000.0)
    assert v == pytest.approx(50.0 * 0.5 ** 10 * 0.5 ** -5)
    with pytest.raises(Exception):
        m.predict((50.0, 10.0, 5.0), 7000.0)


# ---- GPU --------------------------------------------------------------------
@pytest.mark.gpu
def test_plugin_values_and_data(z):
    coef = [1.0, 2.0, 0.5]
    f = z.DeviceObjective(WAVY_SRC, dim=3, data=coef, name="wavy")
    pts = np.random.default_rng(0).uniform(-2, 2, size=(500, 3))
    want = np.sum(np.array(coef) * pts * pts - np.cos(3.0 * pts), axis=1)
    got = f.values(pts)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
    assert f([0.0, 0.0, 0.0]) == -3.0


@pytest.mark.gpu
def test_plugin_matches_registered_objective(z):
    """A plug-in restating Rastrigin: identical PSO swarm (same kernels, same
    op order), identical statuses, minimisers within the stated tolerance."""
    f = z.DeviceObjective(RASTRIGIN_SRC, dim=6, name="rastrigin_plugin")
    cfg = z.ZeusConfig(N=2048, dim=6, range=(-5.12, 5.12), iter_pso=5, iter_bfgs=2000, seed=3,
                       deterministic=True)
    a = z.zeus_run(f, cfg)
    b = z.zeus_run(z.rastrigin, cfg)
    assert a.pso_best_before_bfgs == b.pso_best_before_bfgs
    pa, pb = a.per_run, b.per_run
    assert_outcomes_close(pa.x_final, pa.f_final, pa.status_codes, pb.x_final, pb.f_final,
                          pb.status_codes, "plugin vs registered", pb.grad_norm)
    pts = np.random.default_rng(1).uniform(-5, 5, size=(64, 6))
    assert np.array_equal(f.values(pts),
                          np.array([z.rastrigin(list(p)) for p in pts]))


@pytest.mark.gpu
def test_plugin_domain_error_and_compile_error(z):
    src = """
template <class T, class X>
__device__ T objective(const X& x, int d, const double* data, bool& err) {
  return zu::sqrt(x(0) * x(0) + x(1) * x(1), err);   // Ackley-like kink at 0
}"""
    f = z.DeviceObjective(src, dim=2, name="cone")
    out = z.bfgs_run(f, [0.0, 0.0], theta=1e-6, iter_bfgs=50)
    assert out.status == z.DOMAIN_ERROR and out.iterations == 0 and out.grad_norm == math.inf
    out = z.bfgs_run(f, [1.0, 1.0], theta=1e-6, iter_bfgs=50)
    assert out.status in (z.DOMAIN_ERROR, z.DIVERGED, z.CONVERGED)
    with pytest.raises(ValueError, match="does not compile"):
        z.DeviceObjective("this is not C++", dim=2)
    with pytest.raises(ValueError):
        z.DeviceObjective(src, dim=129)
    g = z.forward_gradient(f, [3.0, 4.0])        # d|x|/dx = x / |x|
    assert np.allclose(g, [0.6, 0.8], rtol=0, atol=1e-15)
    with pytest.raises(z.DomainError):
        z.forward_gradient(f, [0.0, 0.0])          # sqrt'(0), like the reference


@pytest.mark.gpu
def test_plugin_gradient_and_line_search_match_registered(z):
    f = z.DeviceObjective(RASTRIGIN_SRC, dim=4, name="rastrigin_plugin")
    rng = np.random.default_rng(5)
    for _ in range(20):
        x = rng.uniform(-4, 4, 4)
        g_user = z.forward_gradient(f, x)
        g_reg = z.forward_gradient(z.rastrigin, x)
        assert np.array_equal(g_user, g_reg)        # same Dual rules, same order
        p = -g_reg
        ls = z.LineSearchParams()
        assert z.armijo_search(f, x, p, g_reg, z.rastrigin(list(x)), ls) == \
            z.armijo_search(z.rastrigin, x, p, g_reg, z.rastrigin(list(x)), ls)


@pytest.mark.gpu
def test_spectrum_fit_recovers_parameters():
    model = fitting.falling_spectrum(scale=6000.0)
    edges = np.linspace(1200.0, 4800.0, 41)
    truth = (50.0, 10.0, 5.0)
    data = fitting.generate_spectrum_data(model, truth, edges)  # noiseless
    out = fitting.fit(model, data, [1, 0, 0], [1000, 20, 10], seed=0)
    assert out.chi_square < 1e-6
    assert np.allclose(out.theta, truth, rtol=1e-3)
    assert np.max(np.abs(out.pulls)) < 1e-3


@pytest.mark.gpu
def test_cli_fit_demo(tmp_path, capsys):
    rep = tmp_path / "fit.txt"
    assert cli.main(["fit", "--demo", "--report", str(rep)]) == cli.EXIT_OK
    text = rep.read_text()
    assert text.startswith("model: falling_spectrum\nbins: 40\n") and "chi_square:" in text
    assert "of pulls within +-2" in capsys.readouterr().out


@pytest.mark.gpu
def test_plugin_fused_and_peer_exchange_pso(z):
    """A user objective through the fused PSO launches, alone and with the
    multi-GPU peer-memory exchange (3 shards emulated on one device, one
    stream each): the same swarm as the registered objective's single run."""
    import torch

    from paper_2603_28770_b200 import engine

    dev = torch.device("cuda", 0)
    f = z.DeviceObjective(RASTRIGIN_SRC, dim=6, name="rastrigin_plugin")
    n, sweeps = 3000, 5
    ref = engine.SwarmShard(1, 6, n, 0, 9, dev)
    ref.run_local(-5.12, 5.12, 0.5, 1.2, 1.5, sweeps)
    one = engine.SwarmShard(f, 6, n, 0, 9, dev)
    one.run_local(-5.12, 5.12, 0.5, 1.2, 1.5, sweeps)
    for t in ("x", "v", "p", "pval", "gX", "gbest"):
        assert torch.equal(getattr(one, t), getattr(ref, t)), t
    xgs = engine.PsoExchange.emulated(dev, 6, 3)
    streams = [torch.cuda.Stream(dev) for _ in range(3)]
    shards = []
    for r in range(3):
        a, b = engine.shard_bounds(n, r, 3)
        shards.append((engine.SwarmShard(f, 6, b - a, a, 9, dev), a, b))
    torch.cuda.synchronize()
    for r, (s, a, b) in enumerate(shards):
        with torch.cuda.stream(streams[r]):
            s.run_xchg(xgs[r], b - a, -5.12, 5.12, 0.5, 1.2, 1.5, sweeps)
    torch.cuda.synchronize()
    for (s, a, b), xg in zip(shards, xgs):
        xg.check()
        assert torch.equal(s.gX, ref.gX) and torch.equal(s.gbest, ref.gbest)
        assert torch.equal(s.x, ref.x[:, a:b])


SQRT_WELL_SRC = """
template <class T, class X>
__device__ T objective(const X& x, int d, const double* data, bool& err) {
  // defined for x0 >= -1 only: trials that step past it raise DomainError
  T s = -4.0 * zu::sqrt(x(0) + 1.0, err);
  for (int i = 0; i < d; ++i) s = s + (x(i) - 0.5) * (x(i) - 0.5) - zu::cos(2.0 * x(i));
  return s;
}
"""


@pytest.mark.gpu
@pytest.mark.parametrize("d", [24, 40, 100])
def test_plugin_warp_kernel_matches_registered(z, d):
    """d > 16: the user objective runs on the warp-per-start kernel (NVRTC
    instance of bfgs_warp.cuh); restating Rastrigin it gives the registered
    objective's swarm bit for bit and the same statuses / minimisers."""
    f = z.DeviceObjective(RASTRIGIN_SRC, dim=d, name=f"rastrigin_plugin_{d}")
    n = 256 if d < 100 else 64
    cfg = z.ZeusConfig(N=n, dim=d, range=(-5.12, 5.12), iter_pso=3, iter_bfgs=1000, seed=4,
                       deterministic=True)
    a = z.zeus_run(f, cfg)
    b = z.zeus_run(z.rastrigin, cfg)
    assert a.pso_best_before_bfgs == b.pso_best_before_bfgs
    pa, pb = a.per_run, b.per_run
    assert_outcomes_close(pa.x_final, pa.f_final, pa.status_codes, pb.x_final, pb.f_final,
                          pb.status_codes, f"plugin d={d} vs registered", pb.grad_norm)


@pytest.mark.gpu
def test_plugin_warp_kernel_domain_errors_match_thread_kernel(z, monkeypatch):
    """The warp kernel's speculative line search reports a DomainError only
    when the sequential search would reach the raising trial: on a function
    with a domain edge, every start's status, iteration count and counters
    equal the thread-per-start kernel's (which evaluates trials in order)."""
    d = 8
    rng = np.random.default_rng(2)
    x0 = rng.uniform(-1.0, 2.0, size=(512, d))
    x0[:, 0] = rng.uniform(-0.999, -0.5, size=512)   # close to the edge x0 = -1
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("ZEUS_USER_WARP", mode)
        f = z.DeviceObjective(SQRT_WELL_SRC, dim=d, name=f"sqrt_well_{mode}")
        cfg = z.ZeusConfig(N=512, dim=d, range=(-1.0, 2.0), iter_pso=0, iter_bfgs=500, seed=0,
                           deterministic=True)
        res[mode] = z.zeus_run(f, cfg, starts=x0)
    t, w = res["0"], res["1"]
    st_t, st_w = t.per_run.status_codes, w.per_run.status_codes
    assert np.sum(st_t == 3) > 0                        # domain_error: the edge is hit
    assert np.array_equal(st_t, st_w)
    assert np.array_equal(t.per_run.iterations, w.per_run.iterations)
    assert np.array_equal(t.stats.ls_trials, w.stats.ls_trials)
    assert np.array_equal(t.stats.grad_evals, w.stats.grad_evals)
    assert_outcomes_close(w.per_run.x_final, w.per_run.f_final, st_w, t.per_run.x_final,
                          t.per_run.f_final, st_t, "warp vs thread kernel", t.per_run.grad_norm)
