// pso.cu -- host launch + C ABI of the particle-swarm phase (pso.py:79-164);
// the kernels are in pso_kernels.cuh.
#include "pso_kernels.cuh"
#include "zeus_internal.h"

namespace zeus {

struct PsoInitLaunch {
  template <class Obj>
  static int run(int d, int64_t n, int64_t i0, uint64_t seed, double lower, double upper,
                 double* x, double* v, double* p, double* pval, int64_t ld, double* cand,
                 void* ws, cudaStream_t s) {
    const int nb = (int)((n + kPsoBlock - 1) / kPsoBlock);
    double* blk_f = (double*)ws;
    long long* blk_i = (long long*)(blk_f + nb);
    const double range = upper - lower;
    const double vr = upper - lower;  // vel_range (pso.py:101)
    const double vlow = -vr, vrange = vr - (-vr);
    pso_init_kernel<Obj><<<nb, kPsoBlock, 0, s>>>(d, n, i0, seed, lower, range, vlow, vrange,
                                                  x, v, p, pval, ld, blk_f, blk_i);
    int rc = check_launch("pso_init_kernel");
    if (rc) return rc;
    pso_finalize_kernel<<<1, kPsoBlock, 0, s>>>(d, nb, i0, p, ld, blk_f, blk_i, cand);
    return check_launch("pso_finalize_kernel");
  }
};

struct PsoSweepLaunch {
  template <class Obj>
  static int run(int d, int64_t n, int64_t i0, uint64_t seed, int sweep, double w, double c1,
                 double c2, double* x, double* v, double* p, double* pval, int64_t ld,
                 const double* gX, double* cand, void* ws, cudaStream_t s) {
    const int nb = (int)((n + kPsoBlock - 1) / kPsoBlock);
    double* blk_f = (double*)ws;
    long long* blk_i = (long long*)(blk_f + nb);
    const uint64_t k0 = (uint64_t)(2 * d) * (uint64_t)(sweep + 1);
    pso_sweep_kernel<Obj><<<nb, kPsoBlock, 0, s>>>(d, n, i0, seed, k0, w, c1, c2, x, v, p,
                                                   pval, ld, gX, blk_f, blk_i);
    int rc = check_launch("pso_sweep_kernel");
    if (rc) return rc;
    pso_finalize_kernel<<<1, kPsoBlock, 0, s>>>(d, nb, i0, p, ld, blk_f, blk_i, cand);
    return check_launch("pso_finalize_kernel");
  }
};

}  // namespace zeus

using namespace zeus;

extern "C" {

size_t zeus_pso_workspace_bytes(int64_t n) {
  const int64_t nb = (n + kPsoBlock - 1) / kPsoBlock;
  return (size_t)(nb < 1 ? 1 : nb) * (sizeof(double) + sizeof(long long));
}

int zeus_pso_init(int obj, int d, int64_t n, int64_t i0, uint64_t seed, double lower,
                  double upper, double* x, double* v, double* pbest, double* pval, int64_t ld,
                  double* cand, void* workspace, void* stream) {
  if (d < 1 || n < 1 || i0 < 0 || ld < n || !(lower < upper) || !x || !v || !pbest || !pval ||
      !cand || !workspace || (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_pso_init: bad arguments");
  const int rc = dispatch_objective<PsoInitLaunch>(obj, d, n, i0, seed, lower, upper, x, v,
                                                   pbest, pval, ld, cand, workspace,
                                                   as_stream(stream));
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
}

int zeus_pso_sweep(int obj, int d, int64_t n, int64_t i0, uint64_t seed, int sweep, double w,
                   double c1, double c2, double* x, double* v, double* pbest, double* pval,
                   int64_t ld, const double* gX, double* cand, void* workspace, void* stream) {
  if (d < 1 || n < 1 || i0 < 0 || ld < n || sweep < 0 || !x || !v || !pbest || !pval || !gX ||
      !cand || !workspace || (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_pso_sweep: bad arguments");
  const int rc = dispatch_objective<PsoSweepLaunch>(obj, d, n, i0, seed, sweep, w, c1, c2, x,
                                                    v, pbest, pval, ld, gX, cand, workspace,
                                                    as_stream(stream));
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
}

}  // extern "C"
