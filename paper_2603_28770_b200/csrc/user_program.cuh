// user_program.cuh -- the tail of a user objective's NVRTC program
// (plugin.cu): adapts the user's `objective<T>(x, d, data, err)` to the
// framework's objective interface (objectives.cuh) and pulls in the PSO and
// thread-per-start (d <= 16) and warp-per-start (d > 16) BFGS kernels, which
// NVRTC then instantiates for UserObj.
// Compiled only by NVRTC, with -DZEUS_USER_D=<d> (the problem dimension, so
// every per-coordinate array is sized exactly).
#pragma once
#include "bfgs_thread.cuh"
#include "bfgs_warp.cuh"
#include "pso_kernels.cuh"

namespace zeus {

__device__ const double* zeus_user_data;  // plugin data array (set by the host)

// coordinate k seeded: x(i) as a Dual with tangent [i == k]
template <class X>
struct SeedX {
  const X& x;
  int k;
  __device__ __forceinline__ Dual operator()(int i) const { return Dual{x(i), i == k ? 1.0 : 0.0}; }
};
struct PlainX {
  const double* p;
  __device__ __forceinline__ double operator()(int i) const { return p[i]; }
};

// The whole objective is one "term"; its tangents are the d partials from d
// seeded Dual passes (the reference's forward_gradient).  Domain errors come
// back through the `oor` flag (kOorIsError) for the thread-per-start kernel,
// and through two extra tangent slots for the warp-per-start kernel (d > 16),
// whose speculative batches must tell which trial raised: slot d = the
// gradient (or the value) raised, slot d + 1 = the value raised (its term
// value is then NaN).  Either way the BFGS kernel turns them into the
// domain_error status at the old iterate, as bfgs.py does.
struct UserObj {
  static constexpr int kId = 100;
  static constexpr int NACC = 1;
  static constexpr int KT = ZEUS_USER_D + 2;
  static constexpr bool kOorIsError = true;
  __host__ __device__ static int nterms(int) { return 1; }
  __device__ static double init(int, int) { return 0.0; }
  __device__ static double finish(const double acc[1], int, bool&) { return acc[0]; }
  template <class M = AutoMath, class X>
  __device__ static void term(const X& x, int, int d, double t[1], bool& oor) {
    t[0] = objective<double>(x, d, zeus_user_data, oor);
  }
  template <class M, class X>
  __device__ static void term_tan(const X& x, int, int d, double t[1], double tan[KT], bool& oor) {
    bool ev = false, eg = false;
    const double f = objective<double>(x, d, zeus_user_data, ev);
    t[0] = ev ? __longlong_as_double(0x7ff8000000000000LL) : f;
#pragma unroll 1
    for (int k = 0; k < KT - 2; ++k)
      tan[k] = k < d ? objective<Dual>(SeedX<X>{x, k}, d, zeus_user_data, eg).d : 0.0;
    tan[KT - 2] = tan[KT - 1] = 0.0;
    tan[d] = (ev || eg) ? 1.0 : 0.0;
    tan[d + 1] = ev ? 1.0 : 0.0;
    oor = oor || ev || eg;
  }
  template <class TA>
  __device__ static double grad_from_tan(const TA& tan, int i, int d, const double*, bool& err) {
    if (tan(0, d) != 0.0) err = true;
    return tan(0, i);
  }
  template <class TA>
  __device__ static bool value_error(const TA& tan, int d) {
    return tan(0, d + 1) != 0.0;
  }
};

// f of n points (SoA [d][ldx]); NaN where the objective raises DomainError
__global__ void user_value_kernel(int d, int64_t n, const double* x, int64_t ldx, double* f) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xs[ZEUS_USER_D];
  for (int k = 0; k < d; ++k) xs[k] = x[(int64_t)k * ldx + i];
  bool err = false;
  double t[1];
  UserObj::term(PlainX{xs}, 0, d, t, err);
  f[i] = err ? __longlong_as_double(0x7ff8000000000000LL) : t[0];
}

// forward_gradient (autodiff.py:243-266) of n points: d seeded Dual passes
__global__ void user_gradient_kernel(int d, int64_t n, const double* x, int64_t ldx, double* g,
                                     uint8_t* domain_error) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xs[ZEUS_USER_D];
  for (int k = 0; k < d; ++k) xs[k] = x[(int64_t)k * ldx + i];
  bool err = false;
  for (int k = 0; k < d; ++k)
    g[(int64_t)k * ldx + i] = objective<Dual>(SeedX<PlainX>{PlainX{xs}, k}, d, zeus_user_data, err).d;
  domain_error[i] = err ? 1 : 0;
}

// armijo_search (linesearch.py:40-71) on n problems; trials = -1 where the
// objective raised DomainError (the reference propagates the exception)
__global__ void user_armijo_kernel(int d, int64_t n, const double* x, const double* p,
                                   const double* g, int64_t ld, const double* f0, double c1,
                                   double alpha0, int iter_ls, double shrink, double* alpha_out,
                                   int32_t* trials_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ddir = 0.0;  // np.dot(g, p), sequential order
  for (int k = 0; k < d; ++k) ddir = ddir + g[(int64_t)k * ld + i] * p[(int64_t)k * ld + i];
  double alpha = alpha0, xt[ZEUS_USER_D];
  int t = 0;
  bool err = false;
  for (;; ++t) {
    for (int k = 0; k < d; ++k) xt[k] = x[(int64_t)k * ld + i] + alpha * p[(int64_t)k * ld + i];
    const double ft = objective<double>(PlainX{xt}, d, zeus_user_data, err);
    if (err) break;
    if (ft <= f0[i] + c1 * alpha * ddir) break;  // NaN fails
    if (t >= iter_ls) break;
    alpha *= shrink;
  }
  alpha_out[i] = alpha;
  trials_out[i] = err ? -1 : t + 1;
}

}  // namespace zeus
