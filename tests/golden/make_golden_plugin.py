"""Golden outcomes of USER objectives, produced by the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_plugin.py

* two Python closures through the reference's zeus_run (driver.py:220-265):
  the reference test-suite's shifted_sphere (tests/test_driver.py) and the
  README's generic objective with cos (pkg/README.md:72-82);
* the reference's fitting.fit (fitting.py:235-294) on a small Poisson
  falling-spectrum dataset with its default multistart configuration.

Writes plugin.npz next to this file (per-start x, f, |g|, k, status, the PSO
best, and for the fit theta / chi-square / the dataset).  The GPU tests run
the same closures through this package (traced into device source) and
compare (tests/test_gpu_plugin_parity.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
STATUS = ("converged", "diverged", "stopped", "domain_error")


def shifted_sphere(x):
    total = 0.0
    for i, v in enumerate(x):
        d = v - 0.5 * (i + 1)
        total = total + d * d
    return total


def make_wavy(cos):
    def wavy(x):
        total = 0.0
        for v in x:
            total = total + v * v - cos(3.0 * v)
        return total
    return wavy


CASES = {  # name: (dim, N, range, iter_pso, iter_bfgs, seed)
    "sphere": (4, 512, (-3.0, 3.0), 5, 400, 7),
    "wavy": (6, 512, (-3.0, 3.0), 5, 400, 11),
}
# the reference test-suite's spectrum fits (tests/test_fitting.py:135-157):
# Poisson-fluctuated (rng 99) and noiseless data, its bounds and seed
FIT = dict(scale=6000.0, theta=(50.0, 10.0, 5.0), edges=np.linspace(1200.0, 4800.0, 41),
           lower=(1.0, 0.0, 0.0), upper=(1000.0, 20.0, 10.0), seed=5)


def perturbed(x0, k, seed):
    """k copies of x0, each coordinate moved by -1, 0 or +1 ulp at random."""
    rng = np.random.default_rng(seed)
    x0 = np.asarray(x0, dtype=np.float64)
    steps = rng.integers(-1, 2, size=(k, len(x0)))
    up, dn = np.nextafter(x0, np.inf), np.nextafter(x0, -np.inf)
    return np.where(steps > 0, up, np.where(steps < 0, dn, x0))


def reference_unstable(zeus, f, cfg, outcomes, k=16):
    """The reference's OWN rounding-level noise floor on these starts: for
    every start that did not end in a domain error, run the reference's
    bfgs_run (bfgs.py:80-156) from k starts within 1 ulp of it; the start is
    unstable when any of those runs changes status or lands > 1e-6 away.
    Starts are the reference's final swarm (driver.py:236-245)."""
    from zeus.linesearch import LineSearchParams

    streams = zeus.make_start_streams(cfg.seed, cfg.N, cfg.dim)
    state = zeus.init_swarm(f, cfg.N, cfg.range, streams, dim=cfg.dim)
    for _ in range(cfg.iter_pso):
        zeus.update_swarm(state, f, cfg.pso, streams)
    starts = np.asarray(state.positions, dtype=np.float64)
    ls = cfg.ls if hasattr(cfg, "ls") else LineSearchParams()
    unstable = np.zeros(cfg.N, dtype=bool)
    for i, o in enumerate(outcomes):
        if o.status == "domain_error":
            continue
        for xs in perturbed(starts[i], k, i):
            r = zeus.bfgs_run(f, list(xs), cfg.theta, cfg.iter_bfgs, ls)
            if r.status != o.status or np.max(np.abs(np.subtract(r.x_final, o.x_final))) > 1e-6:
                unstable[i] = True
                break
    return starts, unstable


def main() -> None:
    sys.path.insert(0, REF)
    import zeus
    from zeus import fitting
    from zeus.autodiff import cos

    out = {}
    for name, (d, n, rng, sweeps, cap, seed) in CASES.items():
        fn = shifted_sphere if name == "sphere" else make_wavy(cos)
        cfg = zeus.ZeusConfig(N=n, dim=d, range=rng, iter_pso=sweeps, iter_bfgs=cap, seed=seed,
                              deterministic=True)
        r = zeus.zeus_run(fn, cfg)
        out[f"{name}_x"] = np.array([o.x_final for o in r.per_run])
        out[f"{name}_f"] = np.array([o.f_final for o in r.per_run])
        out[f"{name}_gn"] = np.array([o.grad_norm for o in r.per_run])
        out[f"{name}_k"] = np.array([o.iterations for o in r.per_run])
        out[f"{name}_s"] = np.array([STATUS.index(o.status) for o in r.per_run])
        out[f"{name}_pso_best"] = np.float64(r.pso_best_before_bfgs)
        print(name, r.converged_count, r.best.f_final)
    model = fitting.falling_spectrum(FIT["scale"])
    for tag, rng in (("fitp", np.random.default_rng(99)), ("fitn", None)):
        data = fitting.generate_spectrum_data(model, FIT["theta"], FIT["edges"], rng=rng)
        fo = fitting.fit(model, data, FIT["lower"], FIT["upper"], seed=FIT["seed"])
        pr = fo.result.per_run
        # the fit's scaled objective and default config (fitting.py:250-280)
        objective = fitting.chi_square_objective(model, data)
        lo, span = FIT["lower"], [u - l for l, u in zip(FIT["lower"], FIT["upper"])]

        def scaled(u, objective=objective, lo=lo, span=span):
            return objective([a + ui * s for ui, a, s in zip(u, lo, span)])

        cfg = zeus.ZeusConfig(N=256, dim=3, range=(0.0, 1.0), iter_pso=10, iter_bfgs=600,
                              iter_ls=40, theta=1e-8, seed=FIT["seed"])
        starts, unstable = reference_unstable(zeus, scaled, cfg, pr)
        out[f"{tag}_starts"] = starts
        out[f"{tag}_ref_unstable"] = unstable
        print(tag, "reference-unstable starts:", np.flatnonzero(unstable))
        out.update({f"{tag}_counts": data.counts, f"{tag}_theta": np.array(fo.theta),
                    f"{tag}_chi2": np.float64(fo.chi_square),
                    f"{tag}_x": np.array([o.x_final for o in pr]),
                    f"{tag}_f": np.array([o.f_final for o in pr]),
                    f"{tag}_gn": np.array([o.grad_norm for o in pr]),
                    f"{tag}_k": np.array([o.iterations for o in pr]),
                    f"{tag}_s": np.array([STATUS.index(o.status) for o in pr]),
                    f"{tag}_pso_best": np.float64(fo.result.pso_best_before_bfgs)})
        print(tag, fo.theta, fo.chi_square, fo.result.converged_count,
              np.bincount([STATUS.index(o.status) for o in pr], minlength=4))
    np.savez_compressed(os.path.join(HERE, "plugin.npz"), **out)


if __name__ == "__main__":
    main()
