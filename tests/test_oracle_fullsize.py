"""The oracle against the reference's own full-size outcomes (CPU; the
fixtures are tests/golden/fullsize_<tag>.npz, made by running the reference
itself: tests/golden/make_golden_fullsize.py).

* PSO: the oracle's swarm over the FULL swarm of every BASELINE
  configuration (65,536 - 262,144 particles, every sweep) is the
  reference's bit for bit (sha256 of the [N][d] positions, the global best);
* BFGS from the same starts: the oracle-vs-reference noise floor (status
  flips from OpenBLAS vs sequential summation order; the GPU parity tests
  are gated against it), every disagreement a start stalled near theta and
  certified at the rounding level (the oracle from a start within 1 ulp
  reaches the reference's outcome, or its own outcome changes).
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import BOXES, GOLDEN, FLOOR_GN, assert_outcomes_close, certify, disagreements

TAGS = ["c2", "c3", "t50r", "t50b", "c4", "c5_s20", "c5_s5_k128", "c5_s100_k16"]
# oracle-vs-reference disagreements measured on the committed fixtures
FLOOR = {"c2": 2, "c4": 1, "c5_s100_k16": 35}


def load(tag):
    g = np.load(os.path.join(GOLDEN, f"fullsize_{tag}.npz"))
    name, d, n, seed, sweeps, cap = (str(v) for v in g["meta"])
    return g, name, int(d), int(n), int(seed), int(sweeps), int(cap)


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_swarm_is_the_reference_swarm(oracle, tag):
    g, name, d, n, seed, sweeps, cap = load(tag)
    lo, hi = BOXES[name]
    sw = oracle.pso(name, d, n, seed, lo, hi, sweeps)
    assert hashlib.sha256(np.ascontiguousarray(sw.positions).tobytes()).hexdigest() == \
        str(g["pos_sha"])
    assert sw.global_best_val == float(g["gF"]) and np.array_equal(sw.global_best_pos, g["gX"])
    assert np.array_equal(sw.positions[g["idx"]], g["x0"])


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_bfgs_vs_reference(oracle, tag):
    g, name, d, n, seed, sweeps, cap = load(tag)
    r = oracle.bfgs_batch(name, g["x0"], iter_bfgs=cap)
    flips, basins = disagreements(r.status, r.x_final, r.grad_norm, g["s"], g["x"], g["gn"])
    print(f"\n{tag}: oracle vs reference on {len(g['idx'])} starts: {len(flips)} flips, "
          f"{len(basins)} different minima")
    assert len(basins) == 0
    assert len(flips) == FLOOR.get(tag, 0)
    assert np.all(np.maximum(r.grad_norm[flips], g["gn"][flips]) < FLOOR_GN)
    for i in flips:
        assert certify(oracle, name, g["x0"][i], cap, int(g["s"][i]), g["x"][i]) is not None
    keep = np.ones(len(r.status), dtype=bool)
    keep[flips] = False
    assert_outcomes_close(r.x_final[keep], r.f_final[keep], r.status[keep], g["x"][keep],
                          g["f"][keep], g["s"][keep], tag, g["gn"][keep])
