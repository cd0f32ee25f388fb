/* zeus_oracle.h -- TEST INFRASTRUCTURE ONLY (see zeus_oracle.c header).
 * CPU restatement of the reference hot path; never linked by the product. */
#ifndef ZEUS_ORACLE_H
#define ZEUS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* objective ids: same enum as include/zeus_b200.h */
#define ZEUS_OBJ_ROSENBROCK 0
#define ZEUS_OBJ_RASTRIGIN 1
#define ZEUS_OBJ_ACKLEY 2
#define ZEUS_OBJ_GOLDSTEIN_PRICE 3

/* status codes (bfgs.py:32-35) */
#define ZEUS_CONVERGED 0
#define ZEUS_DIVERGED 1
#define ZEUS_STOPPED 2
#define ZEUS_DOMAIN_ERROR 3

#define ZEUS_CURVATURE_FLOOR 1e-12 /* bfgs.py:40 */

typedef struct {
  double f_final;
  double grad_norm;
  int64_t iterations;
  int64_t status;
  int64_t ls_trials;
  int64_t grad_evals;
} zeus_oracle_outcome;

void oracle_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]);
uint64_t oracle_philox_u64(uint64_t seed, uint64_t i, uint64_t k);
void oracle_draw_uniform(uint64_t seed, uint64_t i, uint64_t k0, int64_t count,
                         double low, double high, double *out);
double oracle_objective(int obj, const double *x, int d);
int oracle_gradient(int obj, const double *x, int d, double *grad);
int64_t oracle_argmin(const double *v, int64_t n);
void oracle_pso_init(int obj, int d, int64_t n, uint64_t seed, double lower, double upper,
                     double *x, double *v, double *pbest, double *pval, double *gX, double *gF);
void oracle_pso_sweep(int obj, int d, int64_t n, uint64_t seed, int sweep, double w,
                      double c1, double c2, double *x, double *v, double *pbest,
                      double *pval, double *gX, double *gF);
double oracle_armijo(int obj, int d, const double *x, const double *p, const double *g,
                     double f0, double c1, double alpha0, int iter_ls, double shrink,
                     double *xt, double *ft, int *trials);
int oracle_hessian_update(int d, double *H, const double *dx, const double *dg);
void oracle_bfgs_run(int obj, int d, const double *x0, double theta, int iter_bfgs,
                     double c1, double alpha0, int iter_ls, double shrink,
                     volatile const int *stop_flag, zeus_oracle_outcome *out,
                     double *x_final);
void oracle_bfgs_batch(int obj, int d, int64_t n, const double *x0, double theta,
                       int iter_bfgs, double c1, double alpha0, int iter_ls, double shrink,
                       int threads, zeus_oracle_outcome *out, double *x_final);
/* the batch with the rounding-jitter model (zeus_oracle.c; seed 0 = exact) */
void oracle_bfgs_batch_jitter(int obj, int d, int64_t n, const double *x0, double theta,
                              int iter_bfgs, double c1, double alpha0, int iter_ls,
                              double shrink, int threads, uint64_t jitter_seed,
                              zeus_oracle_outcome *out, double *x_final);
int64_t oracle_reduce_best(const zeus_oracle_outcome *out, int64_t n);
int64_t oracle_zeus_run(int obj, int d, int64_t n, uint64_t seed, double lower, double upper,
                        int iter_pso, double w, double c1_pso, double c2_pso, double theta,
                        int iter_bfgs, double c1_ls, double alpha0, int iter_ls,
                        double shrink, int threads, double *x, double *v, double *pbest,
                        double *pval, double *gX, double *pso_best,
                        zeus_oracle_outcome *out, double *x_final);

#ifdef __cplusplus
}
#endif
#endif
