"""Compare two traj_dump.py files (e.g. two library builds) start by start:
where the trajectories part and whether one of them escapes.
    python scripts/traj_cmp.py A.npz B.npz"""
import sys
import numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for s in range(a['f'].shape[1]):
    print("start column", s)
    for t, j in enumerate(a['j']):
        rel = np.max(np.abs(a['x'][t, s] - b['x'][t, s])) / max(1e-300, np.max(np.abs(b['x'][t, s])))
        if t % 5 == 0 or rel > 1e-2:
            print(f"  j={j:5d} rel|dx|={rel:.2e} f {a['f'][t, s]:.6e} / {b['f'][t, s]:.6e} "
                  f"|g| {a['g'][t, s]:.3e} / {b['g'][t, s]:.3e}")
        if rel > 1e-1 and a['f'][t, s] > 10 * max(b['f'][t, s], 1):
            break
