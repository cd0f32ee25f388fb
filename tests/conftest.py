"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built
libzeus_sm100.so; `-m "not gpu"` tests run on CPU only."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

BOXES = {"rosenbrock": (-5.0, 5.0), "rastrigin": (-5.12, 5.12), "ackley": (-5.0, 5.0),
         "goldstein_price": (-2.0, 2.0)}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libzeus_sm100.so")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name + ".npz"))
    return load


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O


@pytest.fixture(scope="session")
def z():
    import paper_2603_28770_b200 as z

    return z


def xdiff(a, b):
    """|a - b| elementwise; equal values (incl. +-inf) and NaN/NaN pairs and
    pairs of non-finite values count as 0 (runs that blew up on both sides)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_nf = ~np.isfinite(a) & ~np.isfinite(b)
    with np.errstate(invalid="ignore"):
        d = np.abs(a - b)
    return np.where((a == b) | both_nf, 0.0, np.where(np.isnan(d), np.inf, d))


# Stated FP64 tolerance for per-start outcomes from identical starts
# (DESIGN.md 'Parity'): x within 1e-6 -- relaxed to 1e-5 for
# CONVERGED starts, because the stopping rule |g| < theta = 1e-6 only pins the
# minimiser to theta / lambda_min(Hessian) (Rosenbrock at (1,1): 2.5e-6), so
# two exact-arithmetic-equivalent trajectories may stop at different points of
# that ball; f within 1e-10 max(1,|f|) (1e-6 for runs that hit the cap at a
# gradient kink).
X_TOL, X_TOL_CONVERGED = 1e-6, 1e-5


def assert_outcomes_close(x, f, s, ref_x, ref_f, ref_s, label="", ref_gn=None):
    """Statuses identical; x / f within the stated tolerance.  Runs that hit
    the cap while ESCAPING (reference |g| >= 1e3, e.g. Goldstein-Price
    trajectories thrown to |x| ~ 1e5 with f ~ 1e23) are chaotic: only their
    status is gated."""
    s = np.asarray(s)
    ref_s = np.asarray(ref_s)
    assert np.array_equal(s, ref_s), (label, np.flatnonzero(s != ref_s)[:10])
    escaped = np.zeros(len(ref_s), dtype=bool)
    if ref_gn is not None:
        escaped = (ref_s == 1) & ~(np.asarray(ref_gn) < 1e3)
    keep = ~escaped
    x, f, s = np.asarray(x)[keep], np.asarray(f)[keep], s[keep]
    ref_x, ref_f, ref_s = np.asarray(ref_x)[keep], np.asarray(ref_f)[keep], ref_s[keep]
    dx = np.max(xdiff(x, ref_x), axis=1)
    tol = np.where(ref_s == 0, X_TOL_CONVERGED, X_TOL)
    bad = np.flatnonzero(dx > tol)
    assert bad.size == 0, (label, bad[:10], dx[bad[:10]])
    fin = np.isfinite(ref_f)
    assert np.array_equal(np.isfinite(f), fin), label
    ftol = np.where(ref_s == 1, 1e-6, 1e-10)[fin]
    df = xdiff(np.asarray(f)[fin], np.asarray(ref_f)[fin])
    assert np.all(df <= ftol * np.maximum(1, np.abs(np.asarray(ref_f)[fin]))), label
    return dx
