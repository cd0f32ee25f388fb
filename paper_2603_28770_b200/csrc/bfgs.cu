// bfgs.cu -- multistart BFGS (bfgs.py:80-156) on sm_100a, generic-d kernel.
//
// Persistent kernel, one warp per start: a warp pops start indices from a
// device work counter and runs the whole local minimisation without leaving
// the SM -- forward-AD gradient (autodiff.py:243), Armijo backtracking
// (linesearch.py:40), curvature-guarded rank-2 inverse-Hessian update
// (bfgs.py:59) and the convergence / cap / stop tests (bfgs.py:115-130).
//
// Lane mapping: lane l owns coordinates j = l, l+32, ... and the matching
// columns of H.  Vectors live in the warp's shared-memory slice so any lane
// can read neighbours (Rosenbrock couples x_j and x_{j+1}).  H is d x d,
// column j owned by lane j%32: the matvec u_j = sum_i H_ij dg_i and the
// update H_ij += dx_i a_j + u_i b_j  (a_j = c dx_j - rho u_j, b_j = -rho dx_j,
// the O(d^2) form of V H V^T + rho dx dx^T) read dx_i / u_i as shared-memory
// broadcasts.  One matvec per iteration: with u = H dg the next direction
// needs H' g', which is formed from the same column pass.
//
// Objective values keep the reference's sequential summation order (terms
// computed lane-parallel into shared memory, then folded in index order by
// every lane), so f is bit-identical to the reference wherever libm agrees.
#include <algorithm>

#include "objectives.cuh"
#include "zeus_internal.h"

namespace zeus {

struct BfgsArgs {
  int d;
  int64_t n;
  const double* x0;
  int64_t ldx;
  double theta;
  int cap;
  int iter_ls;
  double c1, alpha0, shrink;
  long long required_c;
  unsigned long long* stop_counter;
  int* stop_flag;
  zeus_bfgs_out out;
  unsigned long long* work;
  double* h_global;  // non-null: H lives in HBM/L2 (d too large for smem)
  int warp_doubles;  // shared-memory doubles per warp
};

constexpr int kBfgsWarps = 4;

template <class Obj>
__device__ __forceinline__ double warp_value(const double* xs, int d, double* terms,
                                             double* acc, int lane) {
  const int nt = Obj::nterms(d);
  const DenseX X{xs};
  for (int j = lane; j < nt; j += 32) {
    double t[Obj::NACC];
    Obj::term(X, j, d, t);
#pragma unroll
    for (int a = 0; a < Obj::NACC; ++a) terms[a * d + j] = t[a];
  }
  __syncwarp();
#pragma unroll
  for (int a = 0; a < Obj::NACC; ++a) {
    double s = Obj::init(a, d);
    for (int j = 0; j < nt; ++j) s = s + terms[a * d + j];
    acc[a] = s;
  }
  __syncwarp();
  bool err = false;
  return Obj::finish(acc, d, err);
}

// Gradient at xs given the accumulators of the value sweep at the same point.
// Returns false (uniformly across the warp) on a DomainError.
template <class Obj>
__device__ __forceinline__ bool warp_gradient(const double* xs, int d, const double* acc,
                                              double* g, int lane) {
  const DenseX X{xs};
  bool err = false;
  for (int i = lane; i < d; i += 32) g[i] = Obj::grad(X, i, d, acc, err);
  __syncwarp();
  return !__any_sync(kFull, err);
}

__device__ __forceinline__ double warp_dot(const double* a, const double* b, int d, int lane) {
  double s = 0.0;
  for (int j = lane; j < d; j += 32) s = fma(a[j], b[j], s);
  return warp_sum(s);
}

template <class Obj>
__device__ void bfgs_one(const BfgsArgs& A, long long s, int lane, double* H, double* x,
                         double* g, double* p, double* xn, double* gn, double* dx, double* dg,
                         double* u, double* terms) {
  const int d = A.d;
  for (int j = lane; j < d; j += 32) x[j] = A.x0[(int64_t)j * A.ldx + s];
  for (int i = 0; i < d; ++i)
    for (int j = lane; j < d; j += 32) H[(int64_t)i * d + j] = (i == j) ? 1.0 : 0.0;
  __syncwarp();

  double acc[Obj::NACC], acc_n[Obj::NACC];
  double f0 = warp_value<Obj>(x, d, terms, acc, lane);  // f(x0): also f_final for k=0 exits
  int k = 0, status = ZEUS_DIVERGED, ls_trials = 0, grads = 0;
  double gnorm = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  bool have_grad = false;

  for (;;) {
    if (A.stop_flag && *(volatile int*)A.stop_flag) {
      status = ZEUS_STOPPED;
      break;
    }
    if (!have_grad) {
      ++grads;
      if (!warp_gradient<Obj>(x, d, acc, g, lane)) {
        status = ZEUS_DOMAIN_ERROR;
        break;
      }
      have_grad = true;
      gnorm = sqrt(warp_dot(g, g, d, lane));
    }
    if (gnorm < A.theta) {
      status = ZEUS_CONVERGED;
      break;
    }
    if (k >= A.cap) {
      status = ZEUS_DIVERGED;
      break;
    }
    // p = -(H g)   (bfgs.py:131)
    for (int j = lane; j < d; j += 32) {
      double t = 0.0;
      for (int i = 0; i < d; ++i) t = fma(H[(int64_t)i * d + j], g[i], t);
      p[j] = -t;
    }
    __syncwarp();
    // Armijo backtracking (linesearch.py:60-71); f0 is the cached f(x)
    const double ddir = warp_dot(g, p, d, lane);
    double alpha = A.alpha0, ft = 0.0;
    int t = 0;
    for (;; ++t) {
      for (int j = lane; j < d; j += 32) xn[j] = x[j] + alpha * p[j];
      __syncwarp();
      ft = warp_value<Obj>(xn, d, terms, acc_n, lane);
      if (ft <= f0 + A.c1 * alpha * ddir) break;
      if (t >= A.iter_ls) break;
      alpha *= A.shrink;
    }
    ls_trials += t + 1;
    // gradient at x_new = x + alpha p (bfgs.py:135-136)
    ++grads;
    if (!warp_gradient<Obj>(xn, d, acc_n, gn, lane)) {
      status = ZEUS_DOMAIN_ERROR;
      break;
    }
    // hessian_update(H, x_new - x, g_new - g)   (bfgs.py:59-77, 140)
    double c_dd = 0.0, c_xx = 0.0, c_gg = 0.0;
    for (int j = lane; j < d; j += 32) {
      const double a = xn[j] - x[j], b = gn[j] - g[j];
      dx[j] = a;
      dg[j] = b;
      c_dd = fma(a, b, c_dd);
      c_xx = fma(a, a, c_xx);
      c_gg = fma(b, b, c_gg);
    }
    const double curv = warp_sum(c_dd);
    const double ndx = sqrt(warp_sum(c_xx)), ndg = sqrt(warp_sum(c_gg));
    __syncwarp();
    if (!(curv <= kCurvatureFloor * ndx * ndg)) {
      const double rho = 1.0 / curv;
      double dgu = 0.0;
      for (int j = lane; j < d; j += 32) {
        double t2 = 0.0;
        for (int i = 0; i < d; ++i) t2 = fma(H[(int64_t)i * d + j], dg[i], t2);
        u[j] = t2;
        dgu = fma(dg[j], t2, dgu);
      }
      dgu = warp_sum(dgu);
      __syncwarp();
      const double cc = fma(rho * rho, dgu, rho);
      for (int j = lane; j < d; j += 32) {
        const double aj = fma(cc, dx[j], -rho * u[j]);
        const double bj = -rho * dx[j];
        for (int i = 0; i < d; ++i) {
          double* h = H + (int64_t)i * d + j;
          *h = fma(dx[i], aj, fma(u[i], bj, *h));
        }
      }
      __syncwarp();
    }
    // x, g <- x_new, g_new  (bfgs.py:141-145)
    double* tmp = x;
    x = xn;
    xn = tmp;
    tmp = g;
    g = gn;
    gn = tmp;
    f0 = ft;
#pragma unroll
    for (int a = 0; a < Obj::NACC; ++a) acc[a] = acc_n[a];
    gnorm = sqrt(warp_dot(g, g, d, lane));
    ++k;
    __syncwarp();
  }

  // outputs; f_final = f(x) is the cached value of the current iterate
  const zeus_bfgs_out& o = A.out;
  for (int j = lane; j < d; j += 32) o.x_final[(int64_t)j * o.ld_out + s] = x[j];
  if (lane == 0) {
    o.f_final[s] = f0;
    o.grad_norm[s] = gnorm;
    o.iterations[s] = k;
    o.status[s] = (uint8_t)status;
    if (o.ls_trials) o.ls_trials[s] = ls_trials;
    if (o.grad_evals) o.grad_evals[s] = grads;
    if (status == ZEUS_CONVERGED && A.stop_counter) {
      const unsigned long long old = atomicAdd(A.stop_counter, 1ull);
      if ((long long)old + 1 == A.required_c) atomicExch(A.stop_flag, 1);
    }
  }
  __syncwarp();
}

template <class Obj>
__global__ void __launch_bounds__(kBfgsWarps * 32) bfgs_warp_kernel(BfgsArgs A) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int d = A.d;
  double* base = sm + (size_t)wib * A.warp_doubles;
  double *H, *vec;
  if (A.h_global) {
    H = A.h_global + ((size_t)blockIdx.x * (blockDim.x >> 5) + wib) * (size_t)d * d;
    vec = base;
  } else {
    H = base;
    vec = base + (size_t)d * d;
  }
  double *x = vec, *g = x + d, *p = g + d, *xn = p + d, *gn = xn + d, *dx = gn + d,
         *dg = dx + d, *u = dg + d, *terms = u + d;
  for (;;) {
    long long s = 0;
    if (lane == 0) s = (long long)atomicAdd(A.work, 1ull);
    s = __shfl_sync(kFull, s, 0);
    if (s >= A.n) break;
    bfgs_one<Obj>(A, s, lane, H, x, g, p, xn, gn, dx, dg, u, terms);
  }
}

// ---- sizing --------------------------------------------------------------
constexpr size_t kSmemLimit = 227 * 1024;
constexpr size_t kWsHeader = 256;

static inline int vec_doubles(int d) { return (8 + 2) * d; }  // 8 vectors + NACC<=2 term rows
struct BfgsPlan {
  int wpb;      // warps per block
  bool smem_h;  // H in shared memory
};
static inline BfgsPlan bfgs_plan(int d) {
  const size_t per_warp = ((size_t)d * d + vec_doubles(d)) * sizeof(double);
  int wpb = (int)std::min<size_t>(kBfgsWarps, kSmemLimit / per_warp);
  if (wpb >= 1) return {wpb, true};
  return {kBfgsWarps, false};
}
static inline int global_h_blocks(int sms) { return sms * 2; }

struct BfgsLaunch {
  template <class Obj>
  static int run(BfgsArgs A, cudaStream_t s) {
    const int d = A.d;
    const BfgsPlan plan = bfgs_plan(d);
    A.warp_doubles = vec_doubles(d) + (plan.smem_h ? d * d : 0);
    const size_t smem = (size_t)A.warp_doubles * sizeof(double) * plan.wpb;
    if (smem > kSmemLimit)
      return set_error(ZEUS_ERR_UNSUPPORTED, "bfgs: d=%d needs %zu B smem", d, smem);
    auto kern = bfgs_warp_kernel<Obj>;
    int rc = check_cuda(
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
        "cudaFuncSetAttribute");
    if (rc) return rc;
    int per_sm = 0;
    rc = check_cuda(
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, plan.wpb * 32, smem),
        "occupancy");
    if (rc) return rc;
    const int sms = current_sm_count();
    if (per_sm < 1 || sms < 1) return set_error(ZEUS_ERR_UNSUPPORTED, "bfgs: kernel does not fit");
    int grid = per_sm * sms;
    if (!plan.smem_h) grid = std::min(grid, global_h_blocks(sms));
    const int64_t need = (A.n + plan.wpb - 1) / plan.wpb;
    if (grid > need) grid = (int)std::max<int64_t>(1, need);
    kern<<<grid, plan.wpb * 32, smem, s>>>(A);
    return check_launch("bfgs_warp_kernel");
  }
};

}  // namespace zeus

using namespace zeus;

extern "C" {

size_t zeus_bfgs_workspace_bytes(int d, int64_t n) {
  (void)n;
  if (d < 1 || bfgs_plan(d).smem_h) return kWsHeader;
  int sms = current_sm_count();
  if (sms < 1) sms = 148;
  return kWsHeader + (size_t)global_h_blocks(sms) * kBfgsWarps * (size_t)d * d * sizeof(double);
}

int zeus_bfgs(int obj, int d, int64_t n, const double* x0, int64_t ldx,
              const zeus_bfgs_params* P, int64_t required_c, unsigned long long* stop_counter,
              int* stop_flag, zeus_bfgs_out* out, void* workspace, void* stream) {
  if (d < 1 || n < 0 || ldx < n || !P || !out || !workspace ||
      (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2) || (n > 0 && (!x0 || !out->x_final ||
      !out->f_final || !out->grad_norm || !out->iterations || !out->status)) ||
      out->ld_out < n || !(P->theta > 0.0) || P->iter_bfgs < 0 || P->iter_ls < 1 ||
      ((stop_counter == nullptr) != (stop_flag == nullptr)))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_bfgs: bad arguments");
  if (n == 0) return ZEUS_OK;
  cudaStream_t s = as_stream(stream);
  BfgsArgs A{};
  A.d = d;
  A.n = n;
  A.x0 = x0;
  A.ldx = ldx;
  A.theta = P->theta;
  A.cap = P->iter_bfgs;
  A.iter_ls = P->iter_ls;
  A.c1 = P->c1_armijo;
  A.alpha0 = P->alpha0;
  A.shrink = P->shrink;
  A.required_c = required_c;
  A.stop_counter = stop_counter;
  A.stop_flag = stop_flag;
  A.out = *out;
  A.work = (unsigned long long*)workspace;
  A.h_global = bfgs_plan(d).smem_h ? nullptr : (double*)((char*)workspace + kWsHeader);
  int rc = check_cuda(cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), s), "memset");
  if (rc) return rc;
  rc = dispatch_objective<BfgsLaunch>(obj, A, s);
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
}

}  // extern "C"
