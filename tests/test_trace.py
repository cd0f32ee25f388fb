"""Host side of user objectives (CPU): the tracer's code generation and
refusals, and the host Dual / generic helpers of the reference's scalar
contract (autodiff.py:62-240)."""

import math

import numpy as np
import pytest

from paper_2603_28770_b200 import autodiff as ad
from paper_2603_28770_b200.trace import TraceError, trace_source


def test_emission_follows_python_order():
    def f(x):
        total = 0.0
        for i, v in enumerate(x):
            d = v - 0.5 * (i + 1)
            total = total + d * d
        return total
    src = trace_source(f, 2)
    body = [l.strip() for l in src.splitlines() if l.strip().startswith("const T")]
    assert body == ["const T v0 = x(0);", "const T v1 = v0 - 0x1.0000000000000p-1;",
                    "const T v2 = v1 * v1;", "const T v3 = 0x0.0p+0 + v2;",
                    "const T v4 = x(1);", "const T v5 = v4 - 0x1.0000000000000p+0;",
                    "const T v6 = v5 * v5;", "const T v7 = v3 + v6;"]
    assert src.rstrip().endswith("return v7;\n}") or "return v7;" in src


def test_helpers_and_domain_checks_are_emitted():
    src = trace_source(lambda x: ad.sqrt(x[0] * x[0] + 1.0) / x[1] + ad.log(x[1])
                       + ad.powf(2.0, x[0]) + ad.exp(-x[0]) * ad.cos(x[1]), 2)
    for frag in ("zu::sqrt(", "err)", "zu::div(", "zu::log(", "zu::pow(", "zu::exp(", "zu::cos("):
        assert frag in src
    assert "0x1.0000000000000p+1" in src   # 2.0 as an exact hex literal


def test_constants_and_constant_objectives():
    assert "return 0x1.c000000000000p+2;" in trace_source(lambda x: 7.0, 3)
    assert "-0x0.0p+0" in trace_source(lambda x: x[0] * -0.0, 1)


@pytest.mark.parametrize("bad", [lambda x: x[0] if x[0] > 0 else -x[0],
                                 lambda x: math.cos(x[0]),
                                 lambda x: float(x[0]),
                                 lambda x: abs(x[0])])
def test_untraceable_callables_raise(bad):
    with pytest.raises(TraceError):
        trace_source(bad, 2)
    assert issubclass(TraceError, NotImplementedError)


def test_dual_arithmetic_rules():
    a, b = ad.Dual(3.0, 1.0), ad.Dual(2.0, -0.5)
    for got, want in [(a + b, (5.0, 0.5)), (a - b, (1.0, 1.5)), (a * b, (6.0, 3.0 * -0.5 + 2.0)),
                      (2.0 - a, (-1.0, -1.0)), (a * 4, (12.0, 4.0)), (1.0 + a, (4.0, 1.0)),
                      (a / b, (1.5, (1.0 * 2.0 - 3.0 * -0.5) / 4.0)),
                      (6.0 / a, (2.0, -6.0 * 1.0 / 9.0)), (-a, (-3.0, -1.0)),
                      (a ** 2, (9.0, 2 * 3.0 * 1.0)), (a ** 0.5, (math.sqrt(3.0), 0.5 * 3.0 ** -0.5))]:
        assert (got.real, got.dual) == pytest.approx(want, rel=0, abs=1e-15), (got, want)
    assert a > b and b < 2.5 and a >= 3.0 and not a < b


def test_dual_domain_errors():
    z = ad.Dual(0.0, 1.0)
    for f in (lambda: ad.sqrt(z), lambda: ad.sqrt(ad.Dual(-1.0, 0.0)), lambda: ad.log(z),
              lambda: 1.0 / z, lambda: ad.Dual(1.0, 1.0) / 0.0, lambda: z ** -1,
              lambda: ad.Dual(-2.0, 1.0) ** 0.5, lambda: ad.sqrt(-1.0), lambda: ad.log(0.0),
              lambda: ad.powf(-2.0, 0.5), lambda: ad.powf(0.0, -1.0)):
        with pytest.raises(ad.DomainError):
            f()
    assert ad.sqrt(0.0) == 0.0
    assert ad.exp(1e6) == math.inf and ad.exp(ad.Dual(1e6, 1.0)).real == math.inf
    assert ad.powf(1e300, 2.0) == math.inf and ad.powf(-1e300, 3.0) == -math.inf


def test_elementary_dual_rules():
    x = ad.Dual(0.7, 2.0)
    assert (ad.cos(x).real, ad.cos(x).dual) == (math.cos(0.7), -math.sin(0.7) * 2.0)
    assert (ad.sin(x).real, ad.sin(x).dual) == (math.sin(0.7), math.cos(0.7) * 2.0)
    e = ad.exp(x)
    assert (e.real, e.dual) == (math.exp(0.7), math.exp(0.7) * 2.0)
    assert ad.log(x).dual == 2.0 / 0.7
    p = ad.powf(2.0, x)   # exp(x log 2)
    assert p.real == math.exp(x.real * math.log(2.0))


def test_streams_generator_view():
    from paper_2603_28770_b200.streams import make_start_streams

    st = make_start_streams(42, 4, 3)
    st._offset[2] = 5
    g = st.generator(2)
    ref = np.random.Generator(np.random.Philox(key=np.array([42, 2], dtype=np.uint64)))
    ref.bit_generator.random_raw(5)
    assert np.array_equal(g.uniform(0.0, 1.0, 9), ref.uniform(0.0, 1.0, 9))
