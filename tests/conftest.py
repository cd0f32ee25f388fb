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
# (DESIGN.md 'Parity'): x within 1e-6 for every start,
# converged or not (observed max 3.1e-7); f within 1e-10 max(1,|f|) (1e-6 for
# runs that hit the cap at a gradient kink).
X_TOL, X_TOL_CONVERGED = 1e-6, 1e-6


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


def parity_report(label, x, f, gn, k, s, ref):
    """Per-start comparison of a device result with the oracle's BfgsResult
    on identical starts.  Prints (and returns) the numbers the north-star
    parity bar is stated in: status flips, max |dx|_inf, max relative |df|,
    the |dk| histogram and the bit-identical fraction.  Each flip is listed
    with both gradient norms and iteration counts."""
    s = np.asarray(s).astype(np.int64)
    rs = np.asarray(ref.status).astype(np.int64)
    flips = np.flatnonzero(s != rs)
    same = s == rs
    dx = np.max(xdiff(x, ref.x_final), axis=1)
    rf = np.asarray(ref.f_final)
    df = xdiff(f, rf) / np.maximum(1.0, np.abs(np.where(np.isfinite(rf), rf, 1.0)))
    dk = np.abs(np.asarray(k, dtype=np.int64) - np.asarray(ref.iterations, dtype=np.int64))
    hist = np.bincount(np.minimum(dk, 10), minlength=11)
    bit = float(np.mean(np.all(np.asarray(x) == ref.x_final, axis=1)))
    out = dict(n=len(s), flips=len(flips), max_dx=float(dx[same].max(initial=0.0)),
               max_df=float(df[same].max(initial=0.0)), dk_mean=float(dk.mean()),
               dk_max=int(dk.max(initial=0)), bit_identical_x=bit,
               statuses={int(c): int(np.sum(rs == c)) for c in np.unique(rs)})
    print(f"\n[parity] {label}: {out}")
    print(f"[parity] {label}: |dk| histogram 0..9,>=10: {hist.tolist()}")
    for i in flips[:20]:
        print(f"[parity] {label}: flip start {i}: device status {s[i]} |g| {gn[i]:.3e} k {k[i]}"
              f" / oracle status {rs[i]} |g| {ref.grad_norm[i]:.3e} k {ref.iterations[i]}")
    return out


FLOOR_GN = 1e-4   # a status flip must be a start stalled near theta on both sides


class Sub:
    """Per-start columns of a result at the given indices."""

    def __init__(self, pr, idx=None):
        sel = slice(None) if idx is None else idx
        self.x_final = pr.x_final[sel]
        self.f_final = pr.f_final[sel]
        self.grad_norm = pr.grad_norm[sel]
        self.iterations = pr.iterations[sel]
        self.status_codes = np.asarray(pr.status_codes[sel]).astype(np.int64)


def disagreements(a_s, a_x, a_gn, b_s, b_x, b_gn):
    """(flips, different minima) between two outcome sets on the same starts."""
    flips = np.flatnonzero(a_s != b_s)
    same = a_s == b_s
    dx = np.max(xdiff(a_x, b_x), axis=1)
    basins = np.flatnonzero(same & (dx > 1e-6))
    return flips, basins


def perturbed_starts(x0, k, seed=0):
    """k copies of x0, each coordinate moved by -1, 0 or +1 ulp at random."""
    rng = np.random.default_rng(seed)
    steps = rng.integers(-1, 2, size=(k, len(x0)))
    up, dn = np.nextafter(x0, np.inf), np.nextafter(x0, -np.inf)
    return np.where(steps > 0, up, np.where(steps < 0, dn, x0))


def certify(oracle, name, x0, cap, dev_status, dev_x, k=64, dev_gn=None):
    """Rounding-level certificate for a start on which two implementations
    disagree.  The oracle is run from the same start under two models of
    rounding freedom: k starts within 1 ulp of x0, and k runs of the
    rounding-jitter model (every objective value and gradient component moved
    by -1/0/+1 ulp, oracle.bfgs_batch(jitter_seed=...) -- the device computes
    each of them within ~1 ulp of the reference).  Returns 'reached' when one
    of those runs ends with the device's status at the device's minimiser
    (|dx| <= 1e-6), 'unstable' when the oracle's own outcome changes under the
    perturbations (status or |dx| > 1e-6), 'stall' when the disagreement is
    only whether |g| crossed theta at the noise floor of one minimiser (both
    sides within 1e-6 of each other, both |g| < 10 theta: one side stalled
    there -- the Armijo test cannot resolve f below its rounding noise, so x
    freezes at |g| ~ theta until the cap), else None -- a disagreement no
    rounding-level change explains."""
    x0 = np.asarray(x0, dtype=np.float64)
    base = oracle.bfgs_batch(name, x0[None, :], iter_bfgs=cap)
    runs = [oracle.bfgs_batch(name, perturbed_starts(x0, k), iter_bfgs=cap),
            oracle.bfgs_batch(name, np.repeat(x0[None, :], k, axis=0), iter_bfgs=cap,
                              jitter_seed=0x5EED)]
    for r in runs:
        dx_dev = np.max(xdiff(r.x_final, np.asarray(dev_x)[None, :]), axis=1)
        if np.any((r.status == dev_status) & (dx_dev <= 1e-6)):
            return "reached"
    for r in runs:
        dx_base = np.max(xdiff(r.x_final, base.x_final), axis=1)
        if np.any((r.status != base.status[0]) | (dx_base > 1e-6)):
            return "unstable"
    if dev_gn is not None:
        theta = 1e-6
        same_point = float(np.max(xdiff(base.x_final[0], np.asarray(dev_x)))) <= 1e-6
        if same_point and max(float(dev_gn), float(base.grad_norm[0])) < 10 * theta:
            return "stall"
    return None


def gate(label, dev, ref, floor_count, cert=None, ref_unstable=None):
    """The full-size parity bar (tests/test_gpu_parity_fullsize.py):
    agreeing starts within the stated tolerance; every status flip a start
    stalled near theta on both sides; the number of disagreements (flips +
    different minima) at most 2 x the oracle-vs-reference noise floor + 2;
    and, with ``cert = (oracle, name, starts, cap)``, every disagreement
    certified at the rounding level (certify()); with ``ref_unstable`` (per
    start: the REFERENCE's own outcome changes when its start moves by 1 ulp,
    measured by the golden script), every disagreement must be on such a
    start."""
    rep = parity_report(label, dev.x_final, dev.f_final, dev.grad_norm, dev.iterations,
                        dev.status_codes, ref)
    flips, basins = disagreements(dev.status_codes, dev.x_final, dev.grad_norm,
                                  np.asarray(ref.status), ref.x_final, ref.grad_norm)
    for i in basins[:10]:
        print(f"[parity] {label}: different minimum at start {i}: f {dev.f_final[i]!r} vs "
              f"{ref.f_final[i]!r}, |g| {dev.grad_norm[i]:.2e} / {ref.grad_norm[i]:.2e}, "
              f"k {dev.iterations[i]} / {ref.iterations[i]}")
    n_dis = len(flips) + len(basins)
    allowed = 2 * floor_count + 2
    print(f"[parity] {label}: {len(flips)} flips + {len(basins)} different minima = {n_dis} "
          f"(noise floor {floor_count}, allowed {allowed})")
    gmax = np.maximum(dev.grad_norm[flips], np.asarray(ref.grad_norm)[flips])
    assert np.all(gmax < FLOOR_GN), (label, flips[gmax >= FLOOR_GN][:10])
    assert n_dis <= allowed, (label, n_dis, allowed)
    if ref_unstable is not None and n_dis:
        dis = np.concatenate([flips, basins])
        bad = dis[~np.asarray(ref_unstable, dtype=bool)[dis]]
        assert bad.size == 0, (label, "disagreement on a reference-stable start", bad[:10])
        print(f"[parity] {label}: all {n_dis} disagreements on starts where the reference's "
              f"own outcome changes under 1-ulp start perturbations")
    if cert is not None and n_dis:
        oracle, name, starts, cap = cert
        verdicts = {}
        for i in np.concatenate([flips, basins]):
            v = certify(oracle, name, starts[i], cap, int(dev.status_codes[i]), dev.x_final[i],
                        dev_gn=dev.grad_norm[i])
            verdicts[v] = verdicts.get(v, 0) + 1
            assert v is not None, (label, "uncertified disagreement at start", int(i))
        print(f"[parity] {label}: rounding-level certificates {verdicts} ('reached': the oracle "
              f"from a start within 1 ulp or under 1-ulp rounding jitter lands on the device's "
              f"outcome; 'unstable': the oracle's own outcome moves under them; 'stall': same "
              f"minimiser, |g| < 10 theta on both sides, one side frozen at the noise floor)")
        rep["certificates"] = verdicts
    keep = np.ones(len(dev.status_codes), dtype=bool)
    keep[flips] = False
    keep[basins] = False
    assert_outcomes_close(dev.x_final[keep], dev.f_final[keep], dev.status_codes[keep],
                          ref.x_final[keep], ref.f_final[keep], np.asarray(ref.status)[keep],
                          label, np.asarray(ref.grad_norm)[keep])
    rep["disagreements"] = n_dis
    return rep
