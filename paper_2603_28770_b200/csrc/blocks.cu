// blocks.cu -- batched building blocks behind the reference's public helpers:
// armijo_search (linesearch.py:40-71) and hessian_update (bfgs.py:59-77).
// One thread per independent problem; these serve the drop-in API surface
// and the parity tests, the fused hot path lives in bfgs.cu.
#include "objectives.cuh"
#include "zeus_internal.h"

namespace zeus {

// The trial point is materialised in a per-thread scratch column of `xt`
// (SoA [d][ld]) so objectives can read neighbours.
template <class Obj>
__global__ void armijo_kernel(int d, int64_t n, const double* x, const double* p,
                              const double* g, int64_t ld, const double* f0, double c1,
                              double alpha0, int iter_ls, double shrink, double* xt,
                              double* alpha_out, int32_t* trials_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ddir = 0.0;  // np.dot(g, p): sequential order
  for (int k = 0; k < d; ++k) ddir = ddir + g[k * ld + i] * p[k * ld + i];
  const double fx = f0[i];
  double alpha = alpha0;
  int t = 0;
  for (;; ++t) {
    for (int k = 0; k < d; ++k) xt[k * ld + i] = x[k * ld + i] + alpha * p[k * ld + i];
    double acc[Obj::NACC];
    bool err = false;
    const double ft = value_seq<Obj>(StridedX{xt + i, ld}, d, acc, err);
    if (ft <= fx + c1 * alpha * ddir) break;
    if (t >= iter_ls) break;
    alpha *= shrink;
  }
  alpha_out[i] = alpha;
  if (trials_out) trials_out[i] = t + 1;
}

struct ArmijoLaunch {
  template <class Obj>
  static int run(int d, int64_t n, const double* x, const double* p, const double* g,
                 int64_t ld, const double* f0, const zeus_bfgs_params* P, double* alpha,
                 int32_t* trials, cudaStream_t s) {
    double* xt = nullptr;
    int rc = check_cuda(cudaMallocAsync((void**)&xt, sizeof(double) * (size_t)d * ld, s),
                        "cudaMallocAsync");
    if (rc) return rc;
    const int B = 128;
    armijo_kernel<Obj><<<(unsigned)((n + B - 1) / B), B, 0, s>>>(
        d, n, x, p, g, ld, f0, P->c1_armijo, P->alpha0, P->iter_ls, P->shrink, xt, alpha,
        trials);
    rc = check_launch("armijo_kernel");
    cudaFreeAsync(xt, s);
    return rc;
  }
};

// O(d^2) form of V H V^T + rho dx dx^T (bfgs.py:72-77): with u = H dg,
// H' = H - rho (dx u^T + u dx^T) + (rho^2 dg.u + rho) dx dx^T; the upper
// triangle is computed once and mirrored, so H' is exactly symmetric like the
// reference's 0.5 (U + U^T).
__global__ void hessian_update_kernel(int d, int64_t n, double* H, const double* dx,
                                      const double* dg, uint8_t* updated) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= n) return;
  double* h = H + b * (int64_t)d * d;
  const double* a = dx + b * d;
  const double* c = dg + b * d;
  double curv = 0.0, na = 0.0, nc = 0.0;
  for (int k = 0; k < d; ++k) {
    curv = curv + a[k] * c[k];
    na = na + a[k] * a[k];
    nc = nc + c[k] * c[k];
  }
  if (curv <= kCurvatureFloor * sqrt(na) * sqrt(nc)) {  // bfgs.py:69-71
    if (updated) updated[b] = 0;
    return;
  }
  const double rho = 1.0 / curv;
  double ubuf[256];  // u = H dg from the OLD H (d <= 256, checked on the host)
  double dgu = 0.0;
  for (int i = 0; i < d; ++i) {
    double ui = 0.0;
    for (int j = 0; j < d; ++j) ui = fma(h[i * d + j], c[j], ui);
    ubuf[i] = ui;
    dgu = fma(c[i], ui, dgu);
  }
  const double cc = fma(rho * rho, dgu, rho);
  for (int i = 0; i < d; ++i)
    for (int j = i; j < d; ++j) {
      const double v = h[i * d + j] + (cc * a[i] * a[j] - rho * (a[i] * ubuf[j] + ubuf[i] * a[j]));
      h[i * d + j] = v;
      h[j * d + i] = v;
    }
  if (updated) updated[b] = 1;
}

}  // namespace zeus

using namespace zeus;

extern "C" {

int zeus_armijo(int obj, int d, int64_t n, const double* x, const double* p, const double* g,
                int64_t ld, const double* f0, const zeus_bfgs_params* P, double* alpha,
                int32_t* trials, void* stream) {
  if (d < 1 || n < 0 || ld < n || !P || P->iter_ls < 1 || !(P->alpha0 > 0.0) ||
      (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_armijo: bad arguments");
  if (n == 0) return ZEUS_OK;
  const int rc = dispatch_objective<ArmijoLaunch>(obj, d, n, x, p, g, ld, f0, P, alpha, trials,
                                                  as_stream(stream));
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
}

int zeus_hessian_update(int d, int64_t n, double* H, const double* dx, const double* dg,
                        uint8_t* updated, void* stream) {
  if (d < 1 || d > 256 || n < 0 || (n > 0 && (!H || !dx || !dg)))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_hessian_update: bad arguments (d <= 256)");
  if (n == 0) return ZEUS_OK;
  const int B = 64;
  hessian_update_kernel<<<(unsigned)((n + B - 1) / B), B, 0, as_stream(stream)>>>(d, n, H, dx,
                                                                                  dg, updated);
  return check_launch("hessian_update_kernel");
}

}  // extern "C"
