"""Where does a start's device trajectory leave the oracle's?

    python scripts/divergence_probe.py NAME D N SWEEPS CAP INDEX [INDEX ...]

Regenerates the swarm (seed 42) with the oracle, takes the final positions
of the given start indices, and runs BFGS with caps j = 0, 1, 2, ... on the
device (the product kernels, one start per launch) and in the oracle.  Both
are deterministic, so the state after j iterations is the capped run's
x_final.  Prints per iteration the relative |dx|, the trial counts and
whether the device / oracle f agree, up to the first large departure.
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2603_28770_b200 import engine  # noqa: E402
from paper_2603_28770_b200.linesearch import LineSearchParams  # noqa: E402

OBJ = {"rosenbrock": 0, "rastrigin": 1, "ackley": 2}
BOX = {"rosenbrock": (-5.0, 5.0), "rastrigin": (-5.12, 5.12), "ackley": (-5.0, 5.0)}


def dev_run(name, x0, cap):
    dev = torch.device("cuda", 0)
    d = len(x0)
    xs = torch.from_numpy(np.ascontiguousarray(x0.reshape(d, 1))).to(dev)
    out = engine.BfgsBuffers.allocate(d, 1, dev)
    engine.run_bfgs(OBJ[name], xs, engine.bfgs_params(1e-6, cap, LineSearchParams()), out, dev)
    return (out.x_final.cpu().numpy()[:, 0], float(out.f_final[0]), float(out.grad_norm[0]),
            int(out.iterations[0]), int(out.status[0]), int(out.ls_trials[0]))


def main():
    name, d, n, sweeps, cap = sys.argv[1], *map(int, sys.argv[2:6])
    idxs = [int(v) for v in sys.argv[6:]]
    lo, hi = BOX[name]
    sw = O.pso(name, d, n, 42, lo, hi, sweeps)
    for i in idxs:
        x0 = sw.positions[i]
        full_o = O.bfgs_batch(name, x0[None], iter_bfgs=cap)
        full_d = dev_run(name, x0, cap)
        print(f"== {name} d={d} start {i}: oracle k={full_o.iterations[0]} f={full_o.f_final[0]!r} "
              f"| device k={full_d[3]} f={full_d[1]!r} status {full_d[4]}")
        prev_t = 0
        prev_to = 0
        maxj = int(os.environ.get("MAXJ", cap))
        for j in range(0, min(maxj, cap, max(full_o.iterations[0], full_d[3])) + 1):
            o = O.bfgs_batch(name, x0[None], iter_bfgs=j)
            dv = dev_run(name, x0, j)
            rel = np.max(np.abs(dv[0] - o.x_final[0])) / max(1e-300, np.max(np.abs(o.x_final[0])))
            to = int(o.ls_trials[0])
            print(f"  k={j:4d} rel|dx|={rel:.3e} f dev {dv[1]!r} oracle {o.f_final[0]!r} "
                  f"trials dev {dv[5] - prev_t} oracle {to - prev_to} |g| dev {dv[2]:.3e} "
                  f"oracle {o.grad_norm[0]:.3e}")
            prev_t, prev_to = dv[5], to
            if rel > 1e-3:
                break


if __name__ == "__main__":
    main()
