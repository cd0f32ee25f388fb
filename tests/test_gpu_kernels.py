"""GPU parity: Philox streams, objective values, forward-AD gradients, Armijo
and the inverse-Hessian update, through the C ABI, against the reference's
golden vectors and the oracle.

Tolerances: Philox draws bit-exact; Rosenbrock and
Goldstein-Price values / gradients bit-exact (no libm, no contraction);
Rastrigin / Ackley use CUDA cos/sin/exp (<= 2 ulp from glibc), so values are
checked to 1e-12 max(1,|f|) and gradients to 1e-12 max(1,|g|_inf).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL_LIBM = 1e-12


def _lib():
    from paper_2603_28770_b200 import _capi
    return _capi.lib(), _capi


def _stream():
    return torch.cuda.current_stream().cuda_stream


def test_philox_streams_match_reference_golden(golden, z):
    g = golden("philox")
    for a, seed in enumerate(g["seeds"]):
        for b, i in enumerate(g["parts"]):
            st = z.make_start_streams(int(seed), int(i) + 1, 3)
            u0 = st.draw_uniform(int(i), -5.12, 5.12, 13)
            u1 = st.draw_uniform(int(i), -10.24, 10.24, 13)
            assert np.array_equal(u0, g["uniform"][a, b, 0])
            assert np.array_equal(u1, g["uniform"][a, b, 1])


def test_philox_batch_matches_oracle_bitwise(oracle):
    L, capi = _lib()
    seed, i0, n, k0, count = 2**63 + 5, 1_000_000, 512, 37, 41
    out = torch.empty(n * count, dtype=torch.float64, device="cuda")
    capi.check(L.zeus_philox_uniform(seed, i0, n, k0, count, -3.0, 7.5, out.data_ptr(), _stream()))
    got = out.cpu().numpy().reshape(n, count)
    for r in range(0, n, 37):
        ref = oracle.draw_uniform(seed, i0 + r, k0, count, -3.0, 7.5)
        assert np.array_equal(got[r], ref)


def _device_values(obj, X):
    L, capi = _lib()
    n, d = X.shape
    xs = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    f = torch.empty(n, dtype=torch.float64, device="cuda")
    capi.check(L.zeus_objective_value(obj, d, n, xs.data_ptr(), n, f.data_ptr(), _stream()))
    g = torch.empty((d, n), dtype=torch.float64, device="cuda")
    e = torch.empty(n, dtype=torch.uint8, device="cuda")
    capi.check(L.zeus_objective_gradient(obj, d, n, xs.data_ptr(), n, g.data_ptr(), e.data_ptr(),
                                         _stream()))
    return f.cpu().numpy(), g.cpu().numpy().T, e.cpu().numpy().astype(bool)


OBJ = {"rosenbrock": 0, "rastrigin": 1, "ackley": 2, "goldstein_price": 3}


def test_objectives_and_gradients_match_reference_golden(golden):
    g = golden("objectives")
    cases = sorted({k.rsplit("_", 1)[0] for k in g.files})
    exact = total = 0
    for case in cases:
        name = case.rsplit("_", 1)[0]
        X, F, G, E = g[case + "_x"], g[case + "_f"], g[case + "_g"], g[case + "_err"]
        f, gr, err = _device_values(OBJ[name], X)
        assert np.array_equal(err, E.astype(bool)), case
        ok = ~E.astype(bool)
        if name in ("rosenbrock", "goldstein_price"):
            assert np.array_equal(f, F), case
            assert np.array_equal(gr[ok], G[ok]), case
        else:
            assert np.all(np.abs(f - F) <= TOL_LIBM * np.maximum(1, np.abs(F))), case
            scale = np.maximum(1, np.max(np.abs(G[ok]), axis=1, keepdims=True))
            assert np.all(np.abs(gr[ok] - G[ok]) <= TOL_LIBM * scale), case
        exact += int(np.sum(f == F))
        total += len(F)
    print(f"objective values bit-identical to the reference: {exact}/{total}")


def test_rastrigin_ackley_bulk_against_oracle(oracle):
    rng = np.random.default_rng(7)
    for name, d in (("rastrigin", 10), ("ackley", 50), ("rosenbrock", 100)):
        X = rng.uniform(-5.0, 5.0, (300, d))
        f, gr, err = _device_values(OBJ[name], X)
        assert not err.any()
        for i in range(0, 300, 7):
            fo = oracle.objective(name, X[i])
            go, _ = oracle.gradient(name, X[i])
            assert abs(f[i] - fo) <= TOL_LIBM * max(1, abs(fo))
            assert np.max(np.abs(gr[i] - go)) <= TOL_LIBM * max(1, np.max(np.abs(go)))
            if name == "rosenbrock":
                assert f[i] == fo and np.array_equal(gr[i], go)


def test_ackley_domain_error_locus(z):
    with pytest.raises(z.DomainError):
        z.forward_gradient(z.ackley, [0.0, 0.0])
    with pytest.raises(z.DomainError):
        z.forward_gradient(z.ackley, [1e-170, 0.0])
    z.forward_gradient(z.ackley, [1e-150, 0.0])


def test_forward_gradient_hand_values(z):
    assert z.forward_gradient(z.rosenbrock, [1.0, 1.0]).tolist() == [0.0, 0.0]
    assert z.forward_gradient(z.rosenbrock, [0.0, 0.0]).tolist() == [-2.0, 0.0]
    for dim in (1, 2, 5):
        assert z.forward_gradient(z.rastrigin, [0.0] * dim).tolist() == [0.0] * dim
    assert z.rosenbrock([1.0, 1.0, 1.0, 1.0]) == 0.0
    assert z.rosenbrock([-1.0, 1.0]) == 4.0
    assert z.goldstein_price([0.0, -1.0]) == 3.0
    assert z.goldstein_price([1.0, 1.0]) == 1876.0
    assert z.ackley([1.0, 1.0]) == pytest.approx(3.62538493844036, rel=1e-12)
    assert z.rastrigin([1.0, 1.0]) == pytest.approx(2.0, abs=1e-12)


def test_armijo_matches_reference_golden(golden, z):
    g = golden("linesearch")
    for name, x, p, gr, f0, alpha in zip(g["name"], g["x"], g["p"], g["g"], g["f0"], g["alpha"]):
        fn = getattr(z, str(name))
        a = z.armijo_search(fn, x, p, gr, float(f0), z.LineSearchParams())
        assert a == alpha


def test_hessian_update_matches_reference_golden(golden, z):
    g = golden("hessian")
    for H, dx, dg, out, updated in zip(g["H"], g["dx"], g["dg"], g["out"], g["updated"]):
        H_in = H.copy()
        got = z.hessian_update(H, dx, dg)
        assert np.array_equal(H, H_in)  # inputs never mutated
        if not updated:
            assert got is H
            continue
        assert np.max(np.abs(got - out)) <= 1e-12 * np.max(np.abs(out))
        assert np.array_equal(got, got.T)
        np.linalg.cholesky(got)


def test_hessian_update_guards(z):
    H = np.array([[2.0, 0.3], [0.3, 1.0]])
    assert z.hessian_update(H, np.array([1.0, 0.0]), np.array([0.0, 1.0])) is H
    I3 = np.eye(3)
    assert z.hessian_update(I3, np.array([1.0, 0.0, 0.0]), np.array([-1.0, 0.5, 0.0])) is I3
    upd = z.hessian_update(np.eye(2), np.array([1.0, 0.0]), np.array([2.0, 0.0]))
    assert np.allclose(upd, np.diag([0.5, 1.0]), atol=1e-15)
    assert np.array_equal(z.hessian_update(np.eye(2), np.array([1.0, 0.0]),
                                           np.array([1.0, 0.0])), np.eye(2))


def test_registered_objectives_on_dual_numbers(z, oracle):
    """The registered functions are generic over float / Dual like the
    reference's (objectives.py:33-113): the real part of a Dual evaluation is
    the float evaluation bit for bit; the dual part is grad f . t; Ackley's
    sqrt'(0) raises DomainError whatever the tangents (autodiff.py:207-213)."""
    rng = np.random.default_rng(11)
    for fn, dim, (lo, hi) in [(z.rosenbrock, 4, (-5.0, 5.0)), (z.rastrigin, 4, (-5.12, 5.12)),
                              (z.ackley, 4, (-5.0, 5.0)), (z.goldstein_price, 2, (-2.0, 2.0))]:
        for _ in range(5):
            x = rng.uniform(lo, hi, dim).tolist()
            t = rng.uniform(-1.0, 1.0, dim).tolist()
            plain = fn(x)
            dual = fn([z.Dual(v, w) for v, w in zip(x, t)])
            assert dual.real == plain, fn.__name__
            g = z.forward_gradient(fn, x)
            assert dual.dual == pytest.approx(float(np.dot(g, t)), rel=1e-12, abs=1e-12)
    assert z.ackley([0.0, 0.0]) == pytest.approx(0.0, abs=1e-12)
    with pytest.raises(z.DomainError):
        z.ackley([z.Dual(0.0, 1.0), z.Dual(0.0, 0.0)])
    with pytest.raises(z.DomainError):
        z.ackley([z.Dual(0.0, 0.0), z.Dual(0.0, 0.0)])
