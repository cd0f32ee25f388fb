"""Full-size parity at every BASELINE configuration (
north_star: "per-start convergence flags must be identical", minimisers
within the stated FP64 tolerance).

Three implementations of the same algorithm take part:

* the REFERENCE itself (pure Python, numpy/OpenBLAS), run in the build
  container by tests/golden/make_golden_fullsize.py: its own PSO over the full
  swarm, then its own bfgs_run on a strided subset of the final positions;
  the outcomes are the committed fixtures tests/golden/fullsize_<tag>.npz;
* the ORACLE (oracle/zeus_oracle.c, the reference restated in C with glibc
  libm and sequential dot products; test infrastructure);
* the DEVICE path (the product kernels, through zeus_run).

Per configuration: the device swarm (every particle, every sweep, at the
configuration's full size or its one-GPU shard) must equal the reference's
bit for bit (sha256 of the whole [N][d] position array, the global best),
and the device's per-start BFGS outcomes are compared with the reference's
and, on larger subsets, with the oracle's.

Why the flag bar is stated against a noise floor.  The reference's dot
products and its V H V^T update go through OpenBLAS, whose summation order
is implementation-defined; the oracle uses sequential order.  From the SAME
starts the oracle and the reference disagree on some statuses: a start whose
|g| stalls at ~1-5e-6 (the f resolution of a Rastrigin local minimum: the
Armijo decrease is a few ulps of f) converges on one side and hits the cap
on the other (config 2: 2 of 8,192 starts; config 5 at cap 16: 35 of 1,024).
No implementation can be flag-identical to the reference without reproducing
OpenBLAS's order, so the bar here is:

  * every start the two sides agree on: |x - x_ref|_inf <= 1e-6 and
    |f - f_ref| <= 1e-10 max(1, |f_ref|) (conftest.assert_outcomes_close);
  * every status flip is a rounding-floor flip: both sides end with
    |g| < 1e-4 = 100 theta;
  * the device's disagreements with the reference number at most the
    oracle's on the same starts plus a statistical margin (2 x + 2); flips
    and different minima are listed start by start.
"""

import hashlib
import os

import numpy as np
import pytest
import torch

from conftest import BOXES, GOLDEN, Sub, disagreements, gate, xdiff

pytestmark = pytest.mark.gpu

OBJ = {"rosenbrock": 0, "rastrigin": 1, "ackley": 2, "goldstein_price": 3}
TAGS = ["c2", "c3", "t50r", "t50b", "c4", "c5_s20", "c5_s5_k128", "c5_s100_k16"]


def device_swarm(name, d, n, seed, sweeps):
    from paper_2603_28770_b200 import engine

    dev = torch.device("cuda", 0)
    lo, hi = BOXES[name]
    s = engine.SwarmShard(OBJ[name], d, n, 0, seed, dev)
    s.run_local(lo, hi, 0.5, 1.2, 1.5, sweeps)
    torch.cuda.synchronize()
    return dict(x=s.x.cpu().numpy().T, v=s.v.cpu().numpy().T, p=s.p.cpu().numpy().T,
                pval=s.pval.cpu().numpy(), gX=s.gX.cpu().numpy(), gF=float(s.gbest[0]))


def check_swarm(label, dev, ref):
    """Positions, velocities and personal bests bit-identical for every
    particle; pval (= f(pbest), the device cos / exp vs glibc's) within
    1e-13 relative; the global best bit-identical."""
    xvp = (np.all(dev["x"] == ref.positions, axis=1) & np.all(dev["v"] == ref.velocities, axis=1)
           & np.all(dev["p"] == ref.personal_best_pos, axis=1))
    rel = xdiff(dev["pval"], ref.personal_best_val) / np.maximum(1, np.abs(ref.personal_best_val))
    print(f"\n[parity] {label} swarm: x/v/pbest bit-identical {xvp.sum()}/{len(xvp)}; pval "
          f"bit-identical {np.sum(dev['pval'] == ref.personal_best_val)}, max rel {rel.max():.2e}")
    assert xvp.all(), np.flatnonzero(~xvp)[:10]
    assert rel.max() <= 1e-13
    assert np.array_equal(dev["gX"], ref.global_best_pos), label
    assert dev["gF"] == ref.global_best_val, label


class Golden:
    def __init__(self, tag):
        g = np.load(os.path.join(GOLDEN, f"fullsize_{tag}.npz"))
        name, d, n, seed, sweeps, cap = (str(v) for v in g["meta"])
        self.name, self.d, self.n, self.seed = name, int(d), int(n), int(seed)
        self.sweeps, self.cap = int(sweeps), int(cap)
        self.idx, self.x0 = g["idx"], g["x0"]
        self.pos_sha, self.gF, self.gX = str(g["pos_sha"]), float(g["gF"]), g["gX"]
        self.x_final, self.f_final, self.grad_norm = g["x"], g["f"], g["gn"]
        self.iterations, self.status = g["k"], g["s"]


@pytest.mark.parametrize("tag", TAGS)
def test_against_reference_fixtures(z, oracle, tag):
    """Device vs the reference's own outcomes (and the oracle's noise floor on
    the same starts): full-size swarm bit-identical, per-start outcomes
    under the stated bar."""
    g = Golden(tag)
    lo, hi = BOXES[g.name]
    dev = device_swarm(g.name, g.d, g.n, g.seed, g.sweeps)
    assert hashlib.sha256(np.ascontiguousarray(dev["x"]).tobytes()).hexdigest() == g.pos_sha
    assert dev["gF"] == g.gF and np.array_equal(dev["gX"], g.gX)
    assert np.array_equal(dev["x"][g.idx], g.x0)
    spec = z.get_objective(g.name, g.d)
    res = z.zeus_run(spec.fn, z.ZeusConfig(N=g.n, dim=g.d, range=(lo, hi), iter_pso=g.sweeps,
                                           iter_bfgs=g.cap, seed=g.seed, deterministic=True))
    assert res.pso_best_before_bfgs == g.gF
    ora = oracle.bfgs_batch(g.name, g.x0, iter_bfgs=g.cap)
    f_o, b_o = disagreements(ora.status, ora.x_final, ora.grad_norm, g.status, g.x_final,
                             g.grad_norm)
    print(f"\n[parity] {tag}: oracle vs reference: {len(f_o)} flips, {len(b_o)} different "
          f"minima of {len(g.idx)}")
    gate(f"{tag} device vs reference ({len(g.idx)} starts of {g.n})", Sub(res.per_run, g.idx), g,
         len(f_o) + len(b_o), cert=(oracle, g.name, g.x0, g.cap))


@pytest.mark.parametrize("name,d,n,sweeps,cap,seed", [
    ("rosenbrock", 2, 1024, 10, 1000, 42),     # config 1
    ("rastrigin", 10, 65536, 20, 2000, 42),    # config 2
])
def test_small_configs_every_start_vs_oracle(z, oracle, name, d, n, sweeps, cap, seed):
    """Configs 1 and 2 end to end on EVERY start: zeus_run vs the oracle's
    zeus_run (PSO + BFGS)."""
    lo, hi = BOXES[name]
    conv, best, pso_best, ref, sw = oracle.zeus_run(name, d, n, seed, lo, hi, sweeps, cap,
                                                    return_swarm=True)
    check_swarm(f"{name} d={d}", device_swarm(name, d, n, seed, sweeps), sw)
    spec = z.get_objective(name, d)
    res = z.zeus_run(spec.fn, z.ZeusConfig(N=n, dim=d, range=(lo, hi), iter_pso=sweeps,
                                           iter_bfgs=cap, seed=seed, deterministic=True))
    assert res.pso_best_before_bfgs == pso_best
    # config 2's oracle-vs-reference floor: 2 flips in 8,192 (fixture c2) -> 16 per 65,536
    rep = gate(f"{name} d={d} N={n} device vs oracle", Sub(res.per_run), ref,
               0 if d == 2 else 16, cert=(oracle, name, sw.positions, cap))
    assert abs(res.converged_count - conv) <= rep["flips"]
    assert abs(res.best.f_final - ref.f_final[best]) <= 1e-10 * max(1, abs(ref.f_final[best]))


@pytest.mark.parametrize("name,d,n,sweeps,cap,stride,floor", [
    ("ackley", 50, 262144, 5, 1000, 8, 0),        # config 3: 32,768 starts
    ("rastrigin", 50, 131072, 5, 2000, 16, 0),    # T50 Rastrigin, one GPU's shard: 8,192
    ("rosenbrock", 50, 131072, 5, 2000, 16, 0),   # T50 Rosenbrock: 8,192
    ("rosenbrock", 100, 131072, 5, 2000, 256, 0),  # config 4 shard: 512
])
def test_wide_configs_vs_oracle(z, oracle, name, d, n, sweeps, cap, stride, floor):
    """The 50-D / 100-D configurations on larger strided subsets than the
    reference fixtures hold: the oracle (the slow side is its O(d^3)
    update) vs the full device pipeline."""
    lo, hi = BOXES[name]
    sw = oracle.pso(name, d, n, 42, lo, hi, sweeps)
    check_swarm(f"{name} d={d} N={n}", device_swarm(name, d, n, 42, sweeps), sw)
    idx = np.arange(0, n, stride)
    ref = oracle.bfgs_batch(name, sw.positions[idx], iter_bfgs=cap)
    spec = z.get_objective(name, d)
    res = z.zeus_run(spec.fn, z.ZeusConfig(N=n, dim=d, range=(lo, hi), iter_pso=sweeps,
                                           iter_bfgs=cap, seed=42, deterministic=True))
    assert res.pso_best_before_bfgs == sw.global_best_val
    gate(f"{name} d={d} N={n} device vs oracle ({len(idx)} strided)", Sub(res.per_run, idx), ref,
         floor, cert=(oracle, name, sw.positions[idx], cap))


@pytest.mark.parametrize("sweeps,cap", [(20, 2000), (0, 2000), (5, 1024), (5, 128), (100, 16)])
def test_config5_every_start_vs_oracle(z, oracle, sweeps, cap):
    """Config 5 (the paper's trade-off sweep, Rastrigin d=20: the warp-kernel
    path for 16 < d <= 32) on every one of 4,096 starts, uncapped and at
    the sweep's BFGS depths.  Floors: the oracle-vs-reference counts of the
    c5 fixtures (1,024 starts) scaled to 4,096."""
    n, d = 4096, 20
    lo, hi = BOXES["rastrigin"]
    conv, best, pso_best, ref, sw = oracle.zeus_run("rastrigin", d, n, 42, lo, hi, sweeps, cap,
                                                    return_swarm=True)
    check_swarm(f"c5 sweeps={sweeps}", device_swarm("rastrigin", d, n, 42, sweeps), sw)
    res = z.zeus_run(z.rastrigin, z.ZeusConfig(N=n, dim=d, range=(lo, hi), iter_pso=sweeps,
                                               iter_bfgs=cap, seed=42, deterministic=True))
    floor = {16: 35 * 4}.get(cap, 4)
    gate(f"c5 rastrigin d=20 sweeps={sweeps} cap={cap} device vs oracle", Sub(res.per_run), ref,
         floor, cert=(oracle, "rastrigin", sw.positions, cap))
