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
                                                  x, v, p, pval, ld, blk_f, blk_i, nullptr,
                                                  nullptr, nullptr, nullptr);
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
                                                   pval, ld, gX, blk_f, blk_i, nullptr, nullptr,
                                                   nullptr, nullptr);
    int rc = check_launch("pso_sweep_kernel");
    if (rc) return rc;
    pso_finalize_kernel<<<1, kPsoBlock, 0, s>>>(d, nb, i0, p, ld, blk_f, blk_i, cand);
    return check_launch("pso_finalize_kernel");
  }
};

// The whole PSO phase of one shard that is the whole swarm (one GPU): init +
// iter_pso sweeps, each ONE launch whose last block reduces the candidate and
// writes the global best (pso.py:73-76 over one shard), no host round trips.
struct PsoRunLaunch {
  template <class Obj>
  static int run(int d, int64_t n, int64_t i0, uint64_t seed, double lower, double upper,
                 double w, double c1, double c2, int iter_pso, double* x, double* v, double* p,
                 double* pval, int64_t ld, double* cand, double* gX, double* gbest, void* ws,
                 cudaStream_t s) {
    const int nb = (int)((n + kPsoBlock - 1) / kPsoBlock);
    double* blk_f = (double*)ws;
    long long* blk_i = (long long*)(blk_f + nb);
    unsigned* done = (unsigned*)(blk_i + nb);
    int rc = check_cuda(cudaMemsetAsync(done, 0, sizeof(unsigned), s), "memset(pso done)");
    if (rc) return rc;
    const double range = upper - lower, vr = upper - lower;  // pso.py:101
    pso_init_kernel<Obj><<<nb, kPsoBlock, 0, s>>>(d, n, i0, seed, lower, range, -vr,
                                                  vr - (-vr), x, v, p, pval, ld, blk_f, blk_i,
                                                  done, cand, gX, gbest);
    rc = check_launch("pso_init_kernel(fused)");
    for (int sw = 0; sw < iter_pso && !rc; ++sw) {
      const uint64_t k0 = (uint64_t)(2 * d) * (uint64_t)(sw + 1);
      pso_sweep_kernel<Obj><<<nb, kPsoBlock, 0, s>>>(d, n, i0, seed, k0, w, c1, c2, x, v, p,
                                                     pval, ld, gX, blk_f, blk_i, done, cand, gX,
                                                     gbest);
      rc = check_launch("pso_sweep_kernel(fused)");
    }
    return rc;
  }
};

}  // namespace zeus

using namespace zeus;

extern "C" {

size_t zeus_pso_workspace_bytes(int64_t n) {
  const int64_t nb = (n + kPsoBlock - 1) / kPsoBlock;
  // block partials + the fused barrier's ticket counter (zeus_pso_run)
  return (size_t)(nb < 1 ? 1 : nb) * (sizeof(double) + sizeof(long long)) + 16;
}

int zeus_pso_run(int obj, int d, int64_t n, int64_t i0, uint64_t seed, double lower,
                 double upper, double w, double c1, double c2, int iter_pso, double* x,
                 double* v, double* pbest, double* pval, int64_t ld, double* cand, double* gX,
                 double* gbest, void* workspace, void* stream) {
  if (d < 1 || n < 1 || i0 < 0 || ld < n || !(lower < upper) || iter_pso < 0 || !x || !v ||
      !pbest || !pval || !cand || !gX || !gbest || !workspace ||
      (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_pso_run: bad arguments");
  const int rc = dispatch_objective<PsoRunLaunch>(obj, d, n, i0, seed, lower, upper, w, c1, c2,
                                                  iter_pso, x, v, pbest, pval, ld, cand, gX,
                                                  gbest, workspace, as_stream(stream));
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
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
