// user_objective.cuh -- what a user objective's device source sees (the GPU
// counterpart of the reference's "generic scalar" contract, pkg/README.md:70-87
// and zeus/autodiff.py): a plugin is C++ source for
//
//     template <class T, class X>
//     __device__ T objective(const X& x, int d, const double* data, bool& err);
//
// generic over T in {double, zeus::Dual}; x(i) returns coordinate i as a T,
// `data` is the plugin's constant array (e.g. binned counts), and `err` must
// be raised where the reference raises DomainError (the zu:: helpers below do
// it for you).  The same text is evaluated on doubles for values and on Dual
// numbers for forward-mode gradients (one seeded pass per coordinate, the
// reference's forward_gradient, autodiff.py:243-266).  It is compiled at run
// time with NVRTC for sm_100a together with the framework's PSO and BFGS
// kernels (plugin.cu).
#pragma once
#include "objectives.cuh"

namespace zeus {

// ---- the rest of the Dual arithmetic (autodiff.py:62-173) -----------------
__device__ __forceinline__ Dual operator-(Dual a) { return {-a.r, -a.d}; }
__device__ __forceinline__ Dual operator/(Dual a, Dual b) {
  return {a.r / b.r, (a.d * b.r - a.r * b.d) / (b.r * b.r)};
}
__device__ __forceinline__ Dual operator/(double s, Dual b) {
  return {s / b.r, -s * b.d / (b.r * b.r)};
}
// comparisons use real parts only (autodiff.py:163-173)
__device__ __forceinline__ double real_of(double v) { return v; }
__device__ __forceinline__ double real_of(Dual v) { return v.r; }

}  // namespace zeus

// zu:: the generic elementary functions of zeus.autodiff for plugin sources
namespace zu {
using zeus::Dual;

__device__ __forceinline__ double cos(double x) {
  bool o = false;
  return zeus::AutoMath::cos(x, o);
}
__device__ __forceinline__ Dual cos(Dual x) {  // (cos r, -sin r * d)
  bool o = false;
  const zeus::SinCos sc = zeus::AutoMath::sincos(x.r, o);
  return {sc.c, (-sc.s) * x.d};
}
__device__ __forceinline__ double sin(double x) {
  bool o = false;
  return zeus::AutoMath::sincos(x, o).s;
}
__device__ __forceinline__ Dual sin(Dual x) {  // (sin r, cos r * d)
  bool o = false;
  const zeus::SinCos sc = zeus::AutoMath::sincos(x.r, o);
  return {sc.s, sc.c * x.d};
}
// exp overflows to +inf, never raises (autodiff.py:37-43, 176-181)
__device__ __forceinline__ double exp(double x) { return ::exp(x); }
__device__ __forceinline__ Dual exp(Dual x) {
  const double v = ::exp(x.r);
  return {v, v * x.d};
}
// sqrt: value raises below 0, the Dual also at 0 (autodiff.py:198-216)
__device__ __forceinline__ double sqrt(double x, bool& err) {
  if (x < 0.0) err = true;
  return ::sqrt(x);
}
__device__ __forceinline__ Dual sqrt(Dual x, bool& err) {
  if (x.r < 0.0 || x.r == 0.0) {
    err = true;
    return {0.0, 0.0};
  }
  const double v = ::sqrt(x.r);
  return {v, x.d / (2.0 * v)};
}
// log requires x > 0 (autodiff.py:219-227)
__device__ __forceinline__ double log(double x, bool& err) {
  if (x <= 0.0) err = true;
  return ::log(x);
}
__device__ __forceinline__ Dual log(Dual x, bool& err) {
  if (x.r <= 0.0) {
    err = true;
    return {0.0, 0.0};
  }
  return {::log(x.r), x.d / x.r};
}
// division with the reference's zero checks (autodiff.py:108-131)
template <class A, class B>
__device__ __forceinline__ auto div(A a, B b, bool& err) -> decltype(a / b) {
  if (zeus::real_of(b) == 0.0) err = true;
  return a / b;
}
// powf(base, exponent) (autodiff.py:230-240, Dual.__pow__ 133-161)
__device__ __forceinline__ double pow(double b, double e, bool& err) {
  // math.pow raises ValueError (-> DomainError, autodiff.py:46-58) for a
  // fractional power of a negative base and for a zero base with a negative
  // exponent; overflow follows IEEE to +-inf like _safe_pow
  const double r = ::pow(b, e);
  if ((b < 0.0 && e != ::floor(e)) || (b == 0.0 && e < 0.0)) err = true;
  return r;
}
__device__ __forceinline__ Dual pow(Dual b, double e, bool& err) {
  if (e == ::floor(e)) {
    const int n = (int)e;
    if (b.r == 0.0 && n < 1) err = true;
    return {::pow(b.r, (double)n), n == 0 ? 0.0 : n * ::pow(b.r, (double)(n - 1)) * b.d};
  }
  if (b.r <= 0.0) err = true;
  return {::pow(b.r, e), e * ::pow(b.r, e - 1.0) * b.d};
}
__device__ __forceinline__ Dual pow(Dual b, Dual e, bool& err) { return exp(e * log(b, err)); }
__device__ __forceinline__ Dual pow(double b, Dual e, bool& err) {
  return exp(e * log(b, err));
}

}  // namespace zu
