"""Generate golden vectors by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (pure Python +
numpy) and writes small .npz fixtures next to this
file.  The fixtures are committed; nothing on the GPU box reads
/root/reference.  Each block names the reference function it exercises.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    import zeus
    from zeus import bfgs as zb
    from zeus import objectives as zo

    fns = {"rosenbrock": zo.rosenbrock, "rastrigin": zo.rastrigin,
           "ackley": zo.ackley, "goldstein_price": zo.goldstein_price}
    boxes = {"rosenbrock": (-5.0, 5.0), "rastrigin": (-5.12, 5.12),
             "ackley": (-5.0, 5.0), "goldstein_price": (-2.0, 2.0)}

    # ---- streams.py:21-54: numpy Philox(key=[seed, i]) raw u64 + uniforms
    seeds = [0, 42, 2024, -17, 2**63 + 5, 7]
    parts = [0, 1, 7, 1000, 2**20 - 1]
    raw = np.zeros((len(seeds), len(parts), 23), dtype=np.uint64)
    uni = np.zeros((len(seeds), len(parts), 2, 13))
    for a, s in enumerate(seeds):
        for b, i in enumerate(parts):
            st = zeus.make_start_streams(s, i + 1, 3)
            raw[a, b] = st.generator(i).bit_generator.random_raw(23)
            st2 = zeus.make_start_streams(s, i + 1, 3)
            uni[a, b, 0] = st2.draw_uniform(i, -5.12, 5.12, 13)  # k = 0..12
            uni[a, b, 1] = st2.draw_uniform(i, -10.24, 10.24, 13)  # k = 13..25
    np.savez_compressed(os.path.join(HERE, "philox.npz"),
                        seeds=np.array([s & (2**64 - 1) for s in seeds], dtype=np.uint64),
                        parts=np.array(parts, dtype=np.uint64), raw=raw, uniform=uni)

    # ---- objectives.py:33-113 values + autodiff.py:243-266 gradients
    rng = np.random.default_rng(20240917)
    obj_out = {}
    for name, fn in fns.items():
        dims = [2] if name == "goldstein_price" else [1, 2, 3, 10, 50]
        if name == "rosenbrock":
            dims = [2, 3, 10, 50]
        for d in dims:
            lo, hi = boxes[name]
            pts = rng.uniform(lo, hi, (40, d))
            special = []
            if name in ("rastrigin", "ackley"):
                special = [np.zeros(d), np.ones(d), np.full(d, 1e-170)]
            if name == "rosenbrock":
                special = [np.ones(d), np.zeros(d), np.full(d, 1e3)]
            if name == "goldstein_price":
                special = [np.array([0.0, -1.0]), np.array([1.0, 1.0]), np.zeros(2)]
            pts = np.vstack([pts] + [s[None] for s in special])
            vals = np.array([fn(p.tolist()) for p in pts])
            grads = np.zeros_like(pts)
            errs = np.zeros(len(pts), dtype=np.int8)
            for k, p in enumerate(pts):
                try:
                    grads[k] = zeus.forward_gradient(fn, p.tolist())
                except zeus.DomainError:
                    errs[k] = 1
                    grads[k] = np.nan
            obj_out[f"{name}_{d}_x"] = pts
            obj_out[f"{name}_{d}_f"] = vals
            obj_out[f"{name}_{d}_g"] = grads
            obj_out[f"{name}_{d}_err"] = errs
    np.savez_compressed(os.path.join(HERE, "objectives.npz"), **obj_out)

    # ---- pso.py:79-164: swarm states after init and k sweeps
    pso_cases = [("rosenbrock", 4, 30, 0, 10), ("rastrigin", 3, 40, 7, 5),
                 ("ackley", 5, 20, 123, 3), ("goldstein_price", 2, 16, 5, 4),
                 ("rastrigin", 10, 64, 42, 20)]
    pso_out = {}
    for name, d, n, seed, sweeps in pso_cases:
        st = zeus.make_start_streams(seed, n, d)
        state = zeus.init_swarm(fns[name], n, boxes[name], st, dim=d)
        tag = f"{name}_{d}_{n}_{seed}_{sweeps}"
        pso_out[tag + "_init_x"] = state.positions.copy()
        pso_out[tag + "_init_v"] = state.velocities.copy()
        pso_out[tag + "_init_pval"] = state.personal_best_val.copy()
        pso_out[tag + "_init_gX"] = state.global_best_pos.copy()
        for _ in range(sweeps):
            zeus.update_swarm(state, fns[name], zeus.PsoParams(), st)
        pso_out[tag + "_x"] = state.positions
        pso_out[tag + "_v"] = state.velocities
        pso_out[tag + "_p"] = state.personal_best_pos
        pso_out[tag + "_pval"] = state.personal_best_val
        pso_out[tag + "_gX"] = state.global_best_pos
        pso_out[tag + "_gF"] = np.array(state.global_best_val)
    np.savez_compressed(os.path.join(HERE, "pso.npz"), **pso_out)

    # ---- linesearch.py:40-71 on registered objectives along -g
    ls_out = {"name": [], "x": [], "p": [], "g": [], "f0": [], "alpha": []}
    rng = np.random.default_rng(5)
    for name in ("rosenbrock", "rastrigin", "ackley"):
        for _ in range(20):
            d = 4
            lo, hi = boxes[name]
            x = rng.uniform(lo, hi, d)
            g = zeus.forward_gradient(fns[name], x.tolist())
            p = -g * rng.uniform(0.2, 3.0)
            f0 = fns[name](x.tolist())
            a = zeus.armijo_search(fns[name], x, p, g, f0, zeus.LineSearchParams())
            for key, val in (("name", name), ("x", x), ("p", p), ("g", g),
                             ("f0", f0), ("alpha", a)):
                ls_out[key].append(val)
    np.savez_compressed(os.path.join(HERE, "linesearch.npz"),
                        name=np.array(ls_out["name"]), x=np.array(ls_out["x"]),
                        p=np.array(ls_out["p"]), g=np.array(ls_out["g"]),
                        f0=np.array(ls_out["f0"]), alpha=np.array(ls_out["alpha"]))

    # ---- bfgs.py:59-77 hessian_update on SPD inputs
    rng = np.random.default_rng(2718)
    hu = {"H": [], "dx": [], "dg": [], "out": [], "updated": []}
    for _ in range(60):
        d = 5
        A = rng.normal(size=(d, d))
        H = A @ A.T + d * np.eye(d)
        dx = rng.normal(size=d)
        dg = rng.normal(size=d)
        out = zb.hessian_update(H, dx, dg)
        hu["H"].append(H); hu["dx"].append(dx); hu["dg"].append(dg)
        hu["out"].append(out); hu["updated"].append(out is not H)
    np.savez_compressed(os.path.join(HERE, "hessian.npz"),
                        **{k: np.array(v) for k, v in hu.items()})

    # ---- bfgs.py:80-156 outcomes from reference PSO starts + classic start
    bf = {}
    status_code = {"converged": 0, "diverged": 1, "stopped": 2, "domain_error": 3}
    bfgs_cases = [("rosenbrock", 2, 64, 0, 10, 1000), ("rastrigin", 10, 32, 42, 20, 2000),
                  ("ackley", 10, 24, 3, 5, 1000), ("goldstein_price", 2, 32, 9, 3, 1000),
                  ("rosenbrock", 10, 8, 1, 0, 2000), ("ackley", 2, 48, 11, 5, 150)]
    for name, d, n, seed, sweeps, cap in bfgs_cases:
        cfg = zeus.ZeusConfig(N=n, dim=d, range=boxes[name], iter_pso=sweeps,
                              iter_bfgs=cap, seed=seed, deterministic=True)
        res = zeus.zeus_run(fns[name], cfg)
        st = zeus.make_start_streams(seed, n, d)
        state = zeus.init_swarm(fns[name], n, boxes[name], st, dim=d)
        for _ in range(sweeps):
            zeus.update_swarm(state, fns[name], zeus.PsoParams(), st)
        tag = f"{name}_{d}_{n}_{seed}_{sweeps}_{cap}"
        bf[tag + "_starts"] = state.positions
        bf[tag + "_x"] = np.array([o.x_final for o in res.per_run])
        bf[tag + "_f"] = np.array([o.f_final for o in res.per_run])
        bf[tag + "_gn"] = np.array([o.grad_norm for o in res.per_run])
        bf[tag + "_k"] = np.array([o.iterations for o in res.per_run])
        bf[tag + "_s"] = np.array([status_code[o.status] for o in res.per_run])
        bf[tag + "_best_f"] = np.array(res.best.f_final)
        bf[tag + "_pso_best"] = np.array(res.pso_best_before_bfgs)
        bf[tag + "_converged"] = np.array(res.converged_count)
    out = zeus.bfgs_run(zo.rosenbrock, [-1.2, 1.0], theta=1e-6, iter_bfgs=10_000)
    bf["classic_x"] = np.array(out.x_final)
    bf["classic_f"] = np.array(out.f_final)
    bf["classic_k"] = np.array(out.iterations)
    np.savez_compressed(os.path.join(HERE, "bfgs.npz"), **bf)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
