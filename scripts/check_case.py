"""Diagnose one oracle-parity case: per-start |dx|, statuses, iterations for
the default kernels and the team kernel (ZEUS_NO_WIDE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import BOXES, xdiff
from oracle import oracle as O
import test_gpu_bfgs as T
name, d, n, cap = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
lo, hi = BOXES[name]
starts = O.pso(name, d, n, 3, lo, hi, 2).positions
ref = O.bfgs_batch(name, starts, iter_bfgs=cap)
for tag in ("default", "team"):
    if tag == "team": os.environ["ZEUS_NO_WIDE"] = "1"
    dev = T.device_bfgs(name, starts, cap)
    dx = np.max(xdiff(dev["x"], ref.x_final), axis=1)
    print(tag, "dx", np.array2string(dx, precision=2), "status", dev["s"], ref.status,
          "k", dev["k"], ref.iterations, "f", dev["f"], ref.f_final)
