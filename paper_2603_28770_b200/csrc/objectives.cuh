// objectives.cuh -- device objectives and lane-mapped forward-mode AD.
//
// Each registered objective of the reference (objectives.py:33-113) is written
// ONCE as a template over the scalar type, mirroring the Python text operation
// by operation, and instantiated with `double` (values) and `Dual` (tangents).
// `Dual` reproduces autodiff.py:62-240 rule by rule (including the
// scalar-on-the-left forms and the sqrt'(0) DomainError), and the library is
// built with -fmad=false, so a value evaluation here is the reference's float
// evaluation up to libm ulps (bit-exact for Rosenbrock / Goldstein-Price).
//
// Gradients (autodiff.py:243-266 forward_gradient seeds coordinate i and
// re-evaluates the whole objective).  Every registered objective is a
// sequential fold over "terms", and a term that does not touch x_i carries a
// zero tangent, which adds exactly nothing to the fold.  So the reference's
// tangent for coordinate i equals the fold of the tangents of the terms that
// contain x_i -- O(1) terms instead of O(d).  Lanes own coordinates: lane i
// seeds its own tangent and evaluates only its terms in Dual arithmetic; the
// value sweep (real parts of shared accumulators, e.g. Ackley's two sums) is
// computed once per start and broadcast.
#pragma once
#include "zeus_common.cuh"
#include "zeus_trig.cuh"

namespace zeus {

// ---- dual numbers (autodiff.py:62-173) ------------------------------------
struct Dual {
  double r, d;
  Dual() = default;
  // a float constant is a Dual with zero tangent (autodiff.py:66-68)
  __host__ __device__ constexpr Dual(double v) : r(v), d(0.0) {}
  __host__ __device__ constexpr Dual(double rv, double dv) : r(rv), d(dv) {}
};
__device__ __forceinline__ Dual operator+(Dual a, Dual b) { return {a.r + b.r, a.d + b.d}; }
__device__ __forceinline__ Dual operator+(Dual a, double s) { return {a.r + s, a.d}; }
__device__ __forceinline__ Dual operator+(double s, Dual a) { return {a.r + s, a.d}; }
__device__ __forceinline__ Dual operator-(Dual a, Dual b) { return {a.r - b.r, a.d - b.d}; }
__device__ __forceinline__ Dual operator-(Dual a, double s) { return {a.r - s, a.d}; }
__device__ __forceinline__ Dual operator-(double s, Dual a) { return {s - a.r, -a.d}; }
__device__ __forceinline__ Dual operator*(Dual a, Dual b) {
  return {a.r * b.r, a.r * b.d + a.d * b.r};
}
__device__ __forceinline__ Dual operator*(Dual a, double s) { return {a.r * s, a.d * s}; }
__device__ __forceinline__ Dual operator*(double s, Dual a) { return {a.r * s, a.d * s}; }
__device__ __forceinline__ Dual operator/(Dual a, double s) { return {a.r / s, a.d / s}; }

// Math policies for the transcendental calls.  Fast: branch-free sincos
// (zeus_trig.cuh) valid on |x| <= kTrigMax, raising `oor` outside so the
// caller can re-evaluate the whole batch with Precise (CUDA libm) -- keeping
// the hot loops branch-free lets independent terms interleave.
struct FastMath {
  __device__ static __forceinline__ double cos(double x, bool& oor) {
    oor |= !trig_in_range(x);
    return cos_fast(x);  // == sincos_fast(x).c, one polynomial chain
  }
  __device__ static __forceinline__ SinCos sincos(double x, bool& oor) {
    oor |= !trig_in_range(x);
    return sincos_fast(x);
  }
};
struct PreciseMath {
  __device__ static __forceinline__ double cos(double x, bool&) { return ::cos(x); }
  __device__ static __forceinline__ SinCos sincos(double x, bool&) {
    SinCos r;
    ::sincos(x, &r.s, &r.c);
    return r;
  }
};
// Single-call policy (PSO, thread-sequential code): fast path, libm fallback.
struct AutoMath {
  __device__ static __forceinline__ double cos(double x, bool&) {
    return trig_in_range(x) ? cos_fast(x) : ::cos(x);
  }
  __device__ static __forceinline__ SinCos sincos(double x, bool&) {
    if (trig_in_range(x)) return sincos_fast(x);
    SinCos r;
    ::sincos(x, &r.s, &r.c);
    return r;
  }
};

// Elementary functions: `err` is raised where autodiff.py raises DomainError.
__device__ __forceinline__ double gexp(double x, bool&) { return exp(x); }
__device__ __forceinline__ Dual gexp(Dual x, bool&) {
  const double v = exp(x.r);
  return {v, v * x.d};
}
template <class M>
__device__ __forceinline__ double gcos(double x, bool& oor) { return M::cos(x, oor); }
template <class M>
__device__ __forceinline__ Dual gcos(Dual x, bool& oor) {
  const SinCos sc = M::sincos(x.r, oor);  // one reduction serves value and tangent
  return {sc.c, (-sc.s) * x.d};
}
// float path only rejects negatives; Dual path also rejects 0 (autodiff.py:198-216)
__device__ __forceinline__ double gsqrt(double x, bool& err) {
  if (x < 0.0) err = true;
  return sqrt(x);
}
__device__ __forceinline__ Dual gsqrt(Dual x, bool& err) {
  if (x.r < 0.0 || x.r == 0.0) {
    err = true;
    return {0.0, 0.0};
  }
  const double v = sqrt(x.r);
  return {v, x.d / (2.0 * v)};
}

template <class T>
__device__ __forceinline__ double tangent(const T&) { return 0.0; }
template <>
__device__ __forceinline__ double tangent<Dual>(const Dual& v) { return v.d; }

// ---------------------------------------------------------------------------
// Objective interface (all static):
//   NACC                      number of sequential accumulators (1 or 2)
//   nterms(d)                 terms folded into the accumulators
//   init(a, d)                accumulator a's initial float value
//   term<M>(X, j, d, t[NACC], oor)   term j (X(j) -> coordinate j), math policy M
//   finish(acc[NACC], d, err)
//   grad<M>(X, i, d, acc, err, oor)  d f / d x_i from the Dual rules (see header)
//   KT, term_tan<M>(X, j, d, t[NACC], tan[KT], oor)
//                             term j's value AND its tangents w.r.t. the
//                             coordinates it contains (one Dual pass per
//                             coordinate; sin comes free with the cos)
//   grad_from_tan(TA, i, d, acc, err)  d f / d x_i assembled from the stored
//                             term tangents TA(j, k) -- the fold of the
//                             non-zero tangents in the reference's order
// ---------------------------------------------------------------------------

// objectives.py:33-45  (total = total + (a*a + 100*(b*b)), a = 1-x_i, b = x_{i+1}-x_i^2)
struct Rosenbrock {
  static constexpr bool kOorIsError = false;  // oor = trig range, not a DomainError
  static constexpr int kId = ZEUS_OBJ_ROSENBROCK;
  static constexpr int NACC = 1;
  __host__ __device__ static constexpr int nterms(int d) { return d - 1; }
  __device__ static double init(int, int) { return 0.0; }
  template <class T>
  __device__ static T term2(T xj, T xj1) {
    const T a = 1.0 - xj;
    const T b = xj1 - xj * xj;
    return a * a + 100.0 * (b * b);
  }
  template <class M = AutoMath, class X>
  __device__ static void term(const X& x, int j, int, double t[1], bool&) {
    t[0] = term2<double>(x(j), x(j + 1));
  }
  __device__ static double finish(const double acc[1], int, bool&) { return acc[0]; }
  static constexpr int KT = 2;  // d term_j / d x_j, d term_j / d x_{j+1}
  template <class M, class X>
  __device__ static void term_tan(const X& x, int j, int, double t[1], double tan[2], bool&) {
    const double xj = x(j), xj1 = x(j + 1);
    const Dual e0 = term2<Dual>(Dual{xj, 1.0}, Dual{xj1, 0.0});
    const Dual e1 = term2<Dual>(Dual{xj, 0.0}, Dual{xj1, 1.0});
    t[0] = e0.r;
    tan[0] = e0.d;
    tan[1] = e1.d;
  }
  template <class TA>
  __device__ static double grad_from_tan(const TA& tan, int i, int d, const double*, bool&) {
    double g = 0.0;
    bool any = false;
    if (i >= 1) {
      g = tan(i - 1, 1);
      any = true;
    }
    if (i + 1 < d) {
      const double t = tan(i, 0);
      g = any ? g + t : t;
    }
    return g;
  }
  template <class M = AutoMath, class X>
  __device__ static double grad(const X& x, int i, int d, const double*, bool&, bool&) {
    // seed x_i: term i-1 sees it as x_{j+1}, term i as x_j
    const double xi = x(i);
    double g = 0.0;
    bool any = false;
    if (i >= 1) {
      g = term2<Dual>(Dual{x(i - 1), 0.0}, Dual{xi, 1.0}).d;
      any = true;
    }
    if (i + 1 < d) {
      const double t = term2<Dual>(Dual{xi, 1.0}, Dual{x(i + 1), 0.0}).d;
      g = any ? g + t : t;
    }
    return g;
  }
};

// objectives.py:48-61  (total = 10 d; total = total + (x*x - 10 cos(2 pi x)))
struct Rastrigin {
  static constexpr bool kOorIsError = false;  // oor = trig range, not a DomainError
  static constexpr int kId = ZEUS_OBJ_RASTRIGIN;
  static constexpr int NACC = 1;
  __host__ __device__ static constexpr int nterms(int d) { return d; }
  __device__ static double init(int, int d) { return 10.0 * d; }
  template <class M, class T>
  __device__ static T term1(T xi, bool& oor) {
    return xi * xi - 10.0 * gcos<M>(two_pi() * xi, oor);
  }
  template <class M = AutoMath, class X>
  __device__ static void term(const X& x, int j, int, double t[1], bool& oor) {
    t[0] = term1<M, double>(x(j), oor);
  }
  __device__ static double finish(const double acc[1], int, bool&) { return acc[0]; }
  template <class M = AutoMath, class X>
  __device__ static double grad(const X& x, int i, int, const double*, bool&, bool& oor) {
    return term1<M, Dual>(Dual{x(i), 1.0}, oor).d;
  }
  static constexpr int KT = 1;
  template <class M, class X>
  __device__ static void term_tan(const X& x, int j, int, double t[1], double tan[1],
                                  bool& oor) {
    const Dual e = term1<M, Dual>(Dual{x(j), 1.0}, oor);
    t[0] = e.r;
    tan[0] = e.d;
  }
  template <class TA>
  __device__ static double grad_from_tan(const TA& tan, int i, int, const double*, bool&) {
    return tan(i, 0);
  }
};

// objectives.py:64-85
struct Ackley {
  static constexpr bool kOorIsError = false;  // oor = trig range, not a DomainError
  static constexpr int kId = ZEUS_OBJ_ACKLEY;
  static constexpr int NACC = 2;  // sum_sq, sum_cos
  __host__ __device__ static constexpr int nterms(int d) { return d; }
  __device__ static double init(int, int) { return 0.0; }
  template <class M, class T>
  __device__ static void terms(T xi, T& sq, T& cs, bool& oor) {
    sq = xi * xi;
    cs = gcos<M>(two_pi() * xi, oor);
  }
  template <class M = AutoMath, class X>
  __device__ static void term(const X& x, int j, int, double t[2], bool& oor) {
    terms<M, double>(x(j), t[0], t[1], oor);
  }
  template <class T>
  __device__ static T outer(T sum_sq, T sum_cos, int d, bool& err) {
    return -20.0 * gexp(-0.2 * gsqrt(sum_sq / (double)d, err), err) -
           gexp(sum_cos / (double)d, err) + kE + 20.0;
  }
  // Out-of-line copies for the one-warp-per-start kernels (bfgs_wide.cu): one
  // copy of the exp / sqrt chains in the instruction cache instead of one
  // per call site -- the inlined d = 50 kernel stalled on instruction fetch
  // (ncu no_instruction 2.7 warps per issue): 1,091 -> 1,026 SM-cycles per
  // start-iteration at d = 50, 3,903 -> 3,744 at d = 100, same results.  The
  // small-d kernels keep the inline form (4-7% faster there).
  __device__ __noinline__ static double finish_ool(const double acc[2], int d, bool& err) {
    return outer<double>(acc[0], acc[1], d, err);
  }
  template <class TA>
  __device__ __noinline__ static double grad_from_tan_ool(const TA& tan, int i, int d,
                                                          const double* acc, bool& err) {
    return outer<Dual>(Dual{acc[0], tan(i, 0)}, Dual{acc[1], tan(i, 1)}, d, err).d;
  }
  __device__ static double finish(const double acc[2], int d, bool& err) {
    return outer<double>(acc[0], acc[1], d, err);
  }
  template <class M = AutoMath, class X>
  __device__ static double grad(const X& x, int i, int d, const double* acc, bool& err,
                                bool& oor) {
    Dual sq, cs;
    terms<M, Dual>(Dual{x(i), 1.0}, sq, cs, oor);
    // real parts: the full sequential sums; tangents: the only non-zero term
    return outer<Dual>(Dual{acc[0], sq.d}, Dual{acc[1], cs.d}, d, err).d;
  }
  static constexpr int KT = 2;  // d(x_j^2)/dx_j, d cos(2 pi x_j)/dx_j
  template <class M, class X>
  __device__ static void term_tan(const X& x, int j, int, double t[2], double tan[2],
                                  bool& oor) {
    Dual sq, cs;
    terms<M, Dual>(Dual{x(j), 1.0}, sq, cs, oor);
    t[0] = sq.r;
    t[1] = cs.r;
    tan[0] = sq.d;
    tan[1] = cs.d;
  }
  template <class TA>
  __device__ static double grad_from_tan(const TA& tan, int i, int d, const double* acc,
                                         bool& err) {
    return outer<Dual>(Dual{acc[0], tan(i, 0)}, Dual{acc[1], tan(i, 1)}, d, err).d;
  }
};

// objectives.py:88-113 (d == 2 only; validated on the host)
struct GoldsteinPrice {
  static constexpr bool kOorIsError = false;  // oor = trig range, not a DomainError
  static constexpr int kId = ZEUS_OBJ_GOLDSTEIN_PRICE;
  static constexpr int NACC = 1;
  __host__ __device__ static constexpr int nterms(int) { return 1; }
  __device__ static double init(int, int) { return 0.0; }
  template <class T>
  __device__ static T eval(T x1, T x2) {
    const T s = x1 + x2 + 1.0;
    const T first = 1.0 + s * s *
                              (19.0 - 14.0 * x1 + 3.0 * x1 * x1 - 14.0 * x2 +
                               6.0 * x1 * x2 + 3.0 * x2 * x2);
    const T t = 2.0 * x1 - 3.0 * x2;
    const T second = 30.0 + t * t *
                                (18.0 - 32.0 * x1 + 12.0 * x1 * x1 + 48.0 * x2 -
                                 36.0 * x1 * x2 + 27.0 * x2 * x2);
    return first * second;
  }
  template <class M = AutoMath, class X>
  __device__ static void term(const X& x, int, int, double t[1], bool&) {
    t[0] = eval<double>(x(0), x(1));
  }
  // the single "term" is the whole value: 0.0 + v == v for every v but -0.0,
  // and GP is >= 3 on its domain; finish returns the term itself.
  __device__ static double finish(const double acc[1], int, bool&) { return acc[0]; }
  template <class M = AutoMath, class X>
  __device__ static double grad(const X& x, int i, int, const double*, bool&, bool&) {
    return i == 0 ? eval<Dual>(Dual{x(0), 1.0}, Dual{x(1), 0.0}).d
                  : eval<Dual>(Dual{x(0), 0.0}, Dual{x(1), 1.0}).d;
  }
  static constexpr int KT = 2;  // both partials of the single term
  template <class M, class X>
  __device__ static void term_tan(const X& x, int, int, double t[1], double tan[2], bool&) {
    const Dual e0 = eval<Dual>(Dual{x(0), 1.0}, Dual{x(1), 0.0});
    const Dual e1 = eval<Dual>(Dual{x(0), 0.0}, Dual{x(1), 1.0});
    t[0] = e0.r;
    tan[0] = e0.d;
    tan[1] = e1.d;
  }
  template <class TA>
  __device__ static double grad_from_tan(const TA& tan, int i, int, const double*, bool&) {
    return tan(0, i);
  }
};

// ---- accessors ------------------------------------------------------------
// Tangent slot k of term j for batch row b (buffer [KT][rows][tstride]).
struct TanRow {
  const double* T;
  int rows, tstride, b;
  __device__ __forceinline__ double operator()(int j, int k) const {
    return T[(k * rows + b) * tstride + j];
  }
};
struct StridedX {
  const double* p;
  long long stride;
  __device__ __forceinline__ double operator()(int j) const { return p[(long long)j * stride]; }
};
struct DenseX {
  const double* p;
  __device__ __forceinline__ double operator()(int j) const { return p[j]; }
};

// Sequential (reference-order) value of one point, one thread.
template <class Obj, class X>
__device__ __forceinline__ double value_seq(const X& x, int d, double acc[Obj::NACC],
                                            bool& err) {
#pragma unroll
  for (int a = 0; a < Obj::NACC; ++a) acc[a] = Obj::init(a, d);
  const int nt = Obj::nterms(d);
  bool oor = false;
  for (int j = 0; j < nt; ++j) {
    double t[Obj::NACC];
    Obj::template term<AutoMath>(x, j, d, t, oor);
#pragma unroll
    for (int a = 0; a < Obj::NACC; ++a) acc[a] = acc[a] + t[a];
  }
  return Obj::finish(acc, d, err);
}

#ifndef __CUDACC_RTC__
// Dispatch helper: calls F::template run<Obj>(args...) for the objective id.
template <class F, class... A>
__host__ int dispatch_objective(int obj, A&&... args) {
  switch (obj) {
    case ZEUS_OBJ_ROSENBROCK: return F::template run<Rosenbrock>(args...);
    case ZEUS_OBJ_RASTRIGIN: return F::template run<Rastrigin>(args...);
    case ZEUS_OBJ_ACKLEY: return F::template run<Ackley>(args...);
    case ZEUS_OBJ_GOLDSTEIN_PRICE: return F::template run<GoldsteinPrice>(args...);
    default: return ZEUS_ERR_ARGUMENT;
  }
}

#endif  // __CUDACC_RTC__

}  // namespace zeus
