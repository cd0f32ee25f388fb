"""GPU parity of multistart BFGS (bfgs.py:80-156) against the reference's
golden outcomes and the oracle, from identical starts.

Tolerance (stated in tests/conftest.py): statuses identical;
|x - x_ref|_inf <= 1e-6 (1e-5 for converged starts: theta / lambda_min);
|f - f_ref| <= 1e-10 max(1,|f_ref|) (1e-6 for runs that hit the cap);
escaping capped runs gate only the status; iteration counts are reported as
a |dk| histogram, not gated.
"""

import math

import numpy as np
import pytest
import torch

from conftest import BOXES, assert_outcomes_close

pytestmark = pytest.mark.gpu

OBJ = {"rosenbrock": 0, "rastrigin": 1, "ackley": 2, "goldstein_price": 3}


def device_bfgs(name, starts, cap, theta=1e-6):
    from paper_2603_28770_b200 import engine
    from paper_2603_28770_b200.linesearch import LineSearchParams

    dev = torch.device("cuda", 0)
    starts = np.asarray(starts, dtype=np.float64)
    n, d = starts.shape
    x0 = torch.from_numpy(np.ascontiguousarray(starts.T)).to(dev)
    out = engine.BfgsBuffers.allocate(d, n, dev)
    engine.run_bfgs(OBJ[name], x0, engine.bfgs_params(theta, cap, LineSearchParams()), out, dev)
    return dict(x=out.x_final.cpu().numpy().T, f=out.f_final.cpu().numpy(),
                gn=out.grad_norm.cpu().numpy(), k=out.iterations.cpu().numpy(),
                s=out.status.cpu().numpy().astype(np.int64),
                ls=out.ls_trials.cpu().numpy(), ng=out.grad_evals.cpu().numpy())


def check(dev, ref_x, ref_f, ref_s, ref_k, label, ref_gn=None):
    dx = assert_outcomes_close(dev["x"], dev["f"], dev["s"], ref_x, ref_f, ref_s, label, ref_gn)
    dk = np.abs(dev["k"].astype(np.int64) - np.asarray(ref_k, dtype=np.int64))
    print(f"{label}: {len(ref_s)} starts, max|dx| {dx.max():.2e}, |dk| mean {dk.mean():.2f} "
          f"max {dk.max()}, bit-identical x {np.mean(np.all(dev['x'] == ref_x, axis=1)):.2f}")


def test_matches_reference_golden(golden):
    g = golden("bfgs")
    for tag in sorted(k[: -len("_starts")] for k in g.files if k.endswith("_starts")):
        parts = tag.split("_")
        name = "_".join(parts[:-5])
        cap = int(parts[-1])
        dev = device_bfgs(name, g[tag + "_starts"], cap)
        check(dev, g[tag + "_x"], g[tag + "_f"], g[tag + "_s"], g[tag + "_k"], tag, g[tag + "_gn"])
        assert np.array_equal(dev["s"] == 0, dev["gn"] < 1e-6)  # converged <=> |g| < theta


@pytest.mark.parametrize("name,d,n,cap", [
    ("rastrigin", 10, 512, 2000), ("rosenbrock", 10, 64, 2000), ("ackley", 10, 128, 1000),
    ("rosenbrock", 50, 16, 2000), ("ackley", 50, 64, 1000), ("rastrigin", 50, 24, 2000),
    ("goldstein_price", 2, 256, 1000), ("rosenbrock", 2, 1024, 1000),
    ("rastrigin", 200, 4, 2000),   # H in HBM (d too large for shared memory)
    # warp-per-start throughput kernel (32 < d <= 64): register/shared H split,
    # ragged second column set (d not a multiple of 32), both edges of the range
    ("rosenbrock", 33, 16, 2000), ("rastrigin", 33, 32, 2000), ("ackley", 40, 32, 1000),
    ("rosenbrock", 64, 8, 2000), ("rastrigin", 64, 16, 2000), ("ackley", 64, 16, 1000),
    # two warps per start (64 < d <= 128): cross-warp reductions / neighbours
    ("rastrigin", 65, 8, 2000), ("rosenbrock", 100, 4, 2000), ("ackley", 100, 8, 1000),
    # (rastrigin d=128 with 4 starts has one start whose 150-iteration path
    # ends one basin over for the CTA-team kernel and this one alike: chaotic
    # at that size, so the 16-start case is the one pinned here)
    ("rastrigin", 128, 16, 2000), ("rosenbrock", 97, 4, 2000),
    ("rosenbrock", 129, 2, 2000),  # past the wide kernel: warp kernel, H in smem
])
def test_matches_oracle(oracle, name, d, n, cap):
    lo, hi = BOXES[name]
    starts = oracle.pso(name, d, n, 3, lo, hi, 2).positions
    ref = oracle.bfgs_batch(name, starts, iter_bfgs=cap)
    dev = device_bfgs(name, starts, cap)
    check(dev, ref.x_final, ref.f_final, ref.status, ref.iterations, f"{name} d={d}",
          ref.grad_norm)
    assert np.all(dev["ls"] >= dev["k"])            # >= 1 trial per iteration
    assert np.all(dev["ng"] <= dev["k"] + 1)


@pytest.mark.parametrize("name,d,n", [("rosenbrock", 50, 64), ("rastrigin", 50, 128),
                                       ("ackley", 50, 128), ("rosenbrock", 37, 64),
                                       ("rastrigin", 61, 64), ("ackley", 33, 64),
                                       ("rosenbrock", 100, 16), ("rastrigin", 90, 32),
                                       ("ackley", 70, 32)])
def test_wide_kernel_shapes_match_oracle(oracle, name, d, n):
    """The warp-per-start kernels (bfgs_wide.cu, one warp for d <= 64, two
    for d <= 128) over ragged shapes, against the oracle from identical
    starts, under the full-size parity bar (tests/conftest.py gate)."""
    from conftest import gate

    lo, hi = BOXES[name]
    starts = oracle.pso(name, d, n, 5, lo, hi, 3).positions
    ref = oracle.bfgs_batch(name, starts, iter_bfgs=2000)
    dev = device_bfgs(name, starts, 2000)

    class D:
        x_final, f_final, grad_norm = dev["x"], dev["f"], dev["gn"]
        iterations, status_codes = dev["k"], dev["s"]

    gate(f"wide {name} d={d}", D, ref, 0, cert=(oracle, name, starts, 2000))


def test_hand_traces(z, golden):
    out = z.bfgs_run(z.rosenbrock, [1.0, 1.0], theta=1e-6, iter_bfgs=100)
    assert (out.status, out.iterations, out.x_final) == (z.CONVERGED, 0, (1.0, 1.0))
    out = z.bfgs_run(z.rosenbrock, [-1.2, 1.0], theta=1e-6, iter_bfgs=10_000)
    assert out.status == z.CONVERGED
    assert math.dist(out.x_final, (1.0, 1.0)) < 1e-4
    assert np.max(np.abs(np.array(out.x_final) - golden("bfgs")["classic_x"])) <= 1e-6
    out = z.bfgs_run(z.rosenbrock, [-1.2, 1.0], theta=1e-6, iter_bfgs=3)
    assert (out.status, out.iterations) == (z.DIVERGED, 3) and out.grad_norm >= 1e-6
    out = z.bfgs_run(z.ackley, [0.0, 0.0], theta=1e-6, iter_bfgs=100)
    assert (out.status, out.iterations, out.x_final) == (z.DOMAIN_ERROR, 0, (0.0, 0.0))
    assert out.grad_norm == math.inf and out.f_final == pytest.approx(0.0, abs=1e-12)


def test_converged_iff_gradient_below_theta(z):
    rng = np.random.default_rng(12)
    for _ in range(20):
        x0 = rng.uniform(-5.0, 5.0, 2)
        cap = int(rng.integers(0, 30))
        out = z.bfgs_run(z.rosenbrock, x0, theta=1e-6, iter_bfgs=cap)
        assert (out.status == z.CONVERGED) == (out.grad_norm < 1e-6)
        assert out.iterations <= cap


def test_stop_probe_semantics(z):
    out = z.bfgs_run(z.rastrigin, [3.0, 4.0], theta=1e-6, iter_bfgs=100, stop_probe=lambda: True)
    assert (out.status, out.iterations, out.x_final) == (z.STOPPED, 0, (3.0, 4.0))
    assert out.grad_norm == math.inf
    probes = 0

    def probe():
        nonlocal probes
        probes += 1
        return probes > 1

    out = z.bfgs_run(z.rosenbrock, [8.0, -3.0], theta=1e-16, iter_bfgs=1000, stop_probe=probe)
    assert (out.status, out.iterations) == (z.STOPPED, 1)
    full = z.bfgs_run(z.rosenbrock, [8.0, -3.0], theta=1e-16, iter_bfgs=1)
    assert out.x_final == full.x_final and out.grad_norm == full.grad_norm


def test_validation(z):
    with pytest.raises(ValueError):
        z.bfgs_run(z.rastrigin, [1.0], theta=0.0, iter_bfgs=10)
    with pytest.raises(ValueError):
        z.bfgs_run(z.rastrigin, [1.0], theta=1e-6, iter_bfgs=-1)
    # a plain callable is traced into device source (trace.py) and runs
    out = z.bfgs_run(lambda x: x[0] * x[0], [1.0], theta=1e-6, iter_bfgs=10)
    assert out.status == z.CONVERGED and out.x_final == (0.0,)

    def branchy(x):  # data-dependent control flow cannot be traced
        return x[0] if x[0] > 0 else -x[0]

    with pytest.raises(NotImplementedError):
        z.bfgs_run(branchy, [1.0], theta=1e-6, iter_bfgs=10)


def test_sqrt_free_convergence_and_guard_decisions(tmp_path):
    """The iteration tests decided without square roots (|g|^2 <= gsq_max,
    the squared curvature guard with its exact near-tie fallback) take the
    reference's decisions for every input: millions of random, boundary,
    ulp-neighbour, zero, inf and NaN cases on the device.  Same tool: the
    one-polynomial cos_fast equals sincos_fast's cosine bit for bit."""
    import os
    import subprocess

    from paper_2603_28770_b200 import _capi

    csrc = os.path.join(os.path.dirname(_capi.__file__), "csrc")
    exe = tmp_path / "guard_check"
    subprocess.run(["nvcc", "-O3", "-fmad=false", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-I", csrc, "-o", str(exe), os.path.join(csrc, "tools", "guard_check.cu")],
                   check=True, capture_output=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("name,d,n", [("rastrigin", 10, 2048), ("rosenbrock", 4, 1024),
                                      ("ackley", 6, 1024), ("rastrigin", 24, 128)])
@pytest.mark.parametrize("cap", [0, 1, 15, 16, 17, 47, 48, 49])
def test_caps_at_the_tier_boundaries(oracle, name, d, n, cap):
    """The small-d tiers hand a start over at k1t = 16 (thread -> warp) and
    k1 = 48 (warp -> CTA team).  With the cap on either side of a hand-over
    (and caps 0 / 1) every start ends converged (|g| < theta) or diverged at
    exactly k = cap -- a start whose cap equals a hand-over iteration stops,
    it is not handed over.  Against the oracle: caps 0 / 1 exactly (status,
    k, gradient and trial counts); later caps for every start whose uncapped
    run converges at the same iteration on both sides (iteration counts are
    not gated in general: a rounding-level difference can flip one Armijo
    decision and reroute a Rastrigin path): its status at this cap is then
    fixed -- converged iff its uncapped k <= cap -- and both must show it."""
    lo, hi = BOXES[name]
    starts = oracle.pso(name, d, n, 5, lo, hi, 1).positions
    ref = oracle.bfgs_batch(name, starts, iter_bfgs=cap)
    dev = device_bfgs(name, starts, cap)
    s, k, gn = dev["s"], dev["k"], dev["gn"]
    assert set(np.unique(s)) <= {0, 1}
    assert np.all(k[s == 1] == cap) and np.all(k <= cap)
    assert np.array_equal(s == 0, gn < 1e-6)
    if cap <= 1:
        check(dev, ref.x_final, ref.f_final, ref.status, ref.iterations, f"{name} cap={cap}",
              ref.grad_norm)
        assert np.array_equal(k, ref.iterations) and np.array_equal(dev["ng"], ref.grad_evals)
        assert np.array_equal(dev["ls"], ref.ls_trials)
        return
    full_ref = oracle.bfgs_batch(name, starts, iter_bfgs=2000)
    full_dev = device_bfgs(name, starts, 2000)
    same = (full_ref.status == 0) & (full_dev["s"] == 0) & (full_ref.iterations == full_dev["k"])
    # (d > 16 folds f in tree order, not the reference's: more paths reroute)
    assert same.mean() > (0.8 if d <= 16 else 0.4), same.mean()
    want = np.where(full_ref.iterations <= cap, 0, 1)
    assert np.array_equal(s[same], want[same]), np.flatnonzero(s[same] != want[same])[:10]
    assert np.array_equal(ref.status[same], want[same])
    assert np.array_equal(k[same], np.minimum(full_ref.iterations, cap)[same])


def test_theta_and_line_search_extremes(oracle):
    """theta so large every start converges at k = 0 (one gradient, no
    trial); iter_ls = 1 (two trials at most: alpha0, then the shrunk step
    taken whatever its value) against the oracle over the first iterations
    (longer iter_ls = 1 Rastrigin runs are chaotic: near-full steps)."""
    from paper_2603_28770_b200 import engine
    from paper_2603_28770_b200.linesearch import LineSearchParams

    lo, hi = BOXES["rastrigin"]
    starts = oracle.pso("rastrigin", 10, 512, 7, lo, hi, 1).positions
    dev = device_bfgs("rastrigin", starts, 100, theta=1e10)
    assert np.all(dev["s"] == 0) and np.all(dev["k"] == 0) and np.all(dev["ls"] == 0)
    assert np.all(dev["ng"] == 1)
    d_ = torch.device("cuda", 0)
    x0 = torch.from_numpy(np.ascontiguousarray(starts.T)).to(d_)
    for cap in (1, 2, 3):
        ref = oracle.bfgs_batch("rastrigin", starts, iter_bfgs=cap, iter_ls=1)
        out = engine.BfgsBuffers.allocate(10, 512, d_)
        engine.run_bfgs(1, x0, engine.bfgs_params(1e-6, cap, LineSearchParams(iter_ls=1)), out,
                        d_)
        got = dict(x=out.x_final.cpu().numpy().T, f=out.f_final.cpu().numpy(),
                   s=out.status.cpu().numpy().astype(np.int64), k=out.iterations.cpu().numpy())
        check(got, ref.x_final, ref.f_final, ref.status, ref.iterations, f"iter_ls=1 cap={cap}",
              ref.grad_norm)
        assert np.array_equal(out.ls_trials.cpu().numpy(), ref.ls_trials)
        assert np.all(ref.ls_trials <= 2 * cap)
