/*
 * zeus_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, scalar restatement of the reference (arxiv/paper_2603_28770,
 * "Zeus", /root/reference/pkg/src/zeus) hot path.  It exists to CHECK the
 * CUDA product path and to time the reference algorithm on host cores
 * (bench.py --impl reference / cpu_baseline).  Only tests/, __graft_entry__.smoke()
 * and bench.py's CPU-baseline leg may load it; the product path never does.
 *
 * Pinning: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py).  Philox draws, PSO swarms, objective values
 * and forward-AD gradients are pinned BIT-EXACT (same glibc libm, same
 * operation order, compiled with -ffp-contract=off).  The reference's BLAS
 * calls (np.dot / H @ g / V @ H @ V.T, OpenBLAS) have an implementation
 * defined summation order, so armijo/hessian_update/bfgs_run are pinned to a
 * stated tolerance instead.
 *
 * Every function cites the reference file:line it restates.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "zeus_oracle.h"

/* ------------------------------------------------------------------------ */
/* Rounding-jitter model (certificates only, tests/conftest.py certify()).   */
/* The device path computes every objective value and gradient component    */
/* within ~1 ulp of the reference (its sincos is <= 1 ulp from glibc, d > 16 */
/* folds are trees) and updates H by an algebraically identical O(d^2) form */
/* (bfgs.py:72-77 rounds differently).  With a non-zero jitter seed,         */
/* oracle_bfgs_batch_jitter moves each objective value, gradient component, */
/* direction component and updated H element (symmetrically) of start i by  */
/* -1, 0 or +1 ulp, drawn from a per-start splitmix64 stream: one sample of */
/* that rounding freedom.  Off (the default) the oracle is the exact        */
/* restatement.                                                             */
/* ------------------------------------------------------------------------ */
static __thread uint64_t jit_state; /* 0: off */

static inline uint64_t splitmix64(uint64_t *s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static inline double jitter(double v) {
  if (!jit_state || !isfinite(v)) return v;
  switch (splitmix64(&jit_state) & 3u) {
    case 1: return nextafter(v, INFINITY);
    case 2: return nextafter(v, -INFINITY);
    default: return v;
  }
}

/* ------------------------------------------------------------------------ */
/* Philox4x64-10 (numpy bit generator used by streams.py:36-45)             */
/* ------------------------------------------------------------------------ */

#define PHILOX_M0 0xD2E7470EE14C6C93ULL
#define PHILOX_M1 0xCA5A826395121157ULL
#define PHILOX_W0 0x9E3779B97F4A7C15ULL
#define PHILOX_W1 0xBB67AE8584CAA73BULL

void oracle_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2],
                          uint64_t out[4]) {
  uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint64_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += PHILOX_W0;
      k1 += PHILOX_W1;
    }
    unsigned __int128 p0 = (unsigned __int128)PHILOX_M0 * c0;
    unsigned __int128 p1 = (unsigned __int128)PHILOX_M1 * c2;
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* u64 draw number k of particle i's stream: numpy Philox(key=[seed, i]) starts
 * with counter 0 and an empty 4-word buffer, and increments the counter BEFORE
 * each block (streams.py:36-37 -> numpy philox_next64), so block b = k/4 uses
 * ctr = (b+1, 0, 0, 0) with carry. */
uint64_t oracle_philox_u64(uint64_t seed, uint64_t i, uint64_t k) {
  uint64_t b = k >> 2;
  uint64_t ctr[4] = {b + 1, (b + 1 == 0) ? 1u : 0u, 0, 0};
  uint64_t key[2] = {seed, i};
  uint64_t out[4];
  oracle_philox4x64_10(ctr, key, out);
  return out[k & 3];
}

/* numpy Generator.uniform(low, high): low + (high-low) * ((u64>>11) * 2^-53)
 * (streams.py:41-45); one multiply then one add, no FMA. */
static inline double uniform_from_u64(uint64_t u, double low, double range) {
  double unit = (double)(u >> 11) * (1.0 / 9007199254740992.0);
  return low + range * unit;
}

void oracle_draw_uniform(uint64_t seed, uint64_t i, uint64_t k0, int64_t count,
                         double low, double high, double *out) {
  double range = high - low;
  for (int64_t c = 0; c < count; ++c)
    out[c] = uniform_from_u64(oracle_philox_u64(seed, i, k0 + (uint64_t)c), low,
                              range);
}

/* ------------------------------------------------------------------------ */
/* Dual numbers (autodiff.py:62-240), reproduced operation by operation.     */
/* ------------------------------------------------------------------------ */

typedef struct {
  double r, d;
} dual;

static inline dual D(double r, double d) {
  dual z = {r, d};
  return z;
}
/* Dual + Dual (autodiff.py:80-85) */
static inline dual d_add(dual a, dual b) { return D(a.r + b.r, a.d + b.d); }
/* Dual + scalar and scalar + Dual (__radd__ = __add__, autodiff.py:83-87) */
static inline dual d_adds(dual a, double s) { return D(a.r + s, a.d); }
/* Dual - Dual (autodiff.py:89-94) */
static inline dual d_sub(dual a, dual b) { return D(a.r - b.r, a.d - b.d); }
/* scalar - Dual (__rsub__, autodiff.py:96-99) */
static inline dual d_rsubs(double s, dual a) { return D(s - a.r, -a.d); }
/* Dual * Dual (autodiff.py:101-107) */
static inline dual d_mul(dual a, dual b) {
  return D(a.r * b.r, a.r * b.d + a.d * b.r);
}
/* Dual * scalar and scalar * Dual (__rmul__ = __mul__, autodiff.py:108-111) */
static inline dual d_muls(dual a, double s) { return D(a.r * s, a.d * s); }
/* Dual / scalar (autodiff.py:119-123); divisor never zero here */
static inline dual d_divs(dual a, double s) { return D(a.r / s, a.d / s); }

/* exp overflows to +inf without raising (autodiff.py:37-43, 176-181) */
static inline dual d_exp(dual a) {
  double v = exp(a.r);
  return D(v, v * a.d);
}
/* cos: (cos r, (-sin r) * d) (autodiff.py:184-188) */
static inline dual d_cos(dual a) { return D(cos(a.r), (-sin(a.r)) * a.d); }
/* sqrt raises DomainError at r < 0 and at r == 0 (autodiff.py:198-213) */
static inline dual d_sqrt(dual a, int *domain_error) {
  if (a.r < 0.0 || a.r == 0.0) {
    *domain_error = 1;
    return D(NAN, NAN);
  }
  double v = sqrt(a.r);
  return D(v, a.d / (2.0 * v));
}

/* ------------------------------------------------------------------------ */
/* Objectives (objectives.py:33-113): float path and Dual path.              */
/* ------------------------------------------------------------------------ */

#define TWO_PI (2.0 * M_PI) /* objectives.py:30 */

/* objectives.py:33-45 */
static double rosenbrock_f(const double *x, int d) {
  double total = 0.0;
  for (int i = 0; i < d - 1; ++i) {
    double a = 1.0 - x[i];
    double b = x[i + 1] - x[i] * x[i];
    total = total + (a * a + 100.0 * (b * b));
  }
  return total;
}
static dual rosenbrock_d(const dual *x, int d, int *err) {
  (void)err;
  /* total starts as the float 0.0; float + Dual -> Dual.__radd__ */
  dual total = D(0.0, 0.0);
  int first = 1;
  for (int i = 0; i < d - 1; ++i) {
    dual a = d_rsubs(1.0, x[i]);
    dual b = d_sub(x[i + 1], d_mul(x[i], x[i]));
    dual term = d_add(d_mul(a, a), d_muls(d_mul(b, b), 100.0));
    if (first) {
      total = d_adds(term, 0.0);
      first = 0;
    } else {
      total = d_add(total, term);
    }
  }
  return total;
}

/* objectives.py:48-61 */
static double rastrigin_f(const double *x, int d) {
  double total = 10.0 * d;
  for (int i = 0; i < d; ++i) {
    double xi = x[i];
    total = total + (xi * xi - 10.0 * cos(TWO_PI * xi));
  }
  return total;
}
static dual rastrigin_d(const dual *x, int d, int *err) {
  (void)err;
  double t0 = 10.0 * d;
  dual total = D(t0, 0.0);
  for (int i = 0; i < d; ++i) {
    dual xi = x[i];
    dual term = d_sub(d_mul(xi, xi), d_muls(d_cos(d_muls(xi, TWO_PI)), 10.0));
    if (i == 0)
      total = d_adds(term, t0);
    else
      total = d_add(total, term);
  }
  return total;
}

/* objectives.py:64-85 */
static double ackley_f(const double *x, int d) {
  double sum_sq = 0.0, sum_cos = 0.0;
  for (int i = 0; i < d; ++i) {
    double xi = x[i];
    sum_sq = sum_sq + xi * xi;
    sum_cos = sum_cos + cos(TWO_PI * xi);
  }
  /* float-path sqrt only rejects negatives (autodiff.py:214-216) */
  return -20.0 * exp(-0.2 * sqrt(sum_sq / d)) - exp(sum_cos / d) + M_E + 20.0;
}
static dual ackley_d(const dual *x, int d, int *err) {
  dual sum_sq = D(0.0, 0.0), sum_cos = D(0.0, 0.0);
  for (int i = 0; i < d; ++i) {
    dual xi = x[i];
    dual sq = d_mul(xi, xi);
    dual cs = d_cos(d_muls(xi, TWO_PI));
    if (i == 0) {
      sum_sq = d_adds(sq, 0.0);
      sum_cos = d_adds(cs, 0.0);
    } else {
      sum_sq = d_add(sum_sq, sq);
      sum_cos = d_add(sum_cos, cs);
    }
  }
  dual s = d_sqrt(d_divs(sum_sq, (double)d), err);
  if (*err) return D(NAN, NAN);
  dual a = d_muls(d_exp(d_muls(s, -0.2)), -20.0);
  dual b = d_exp(d_divs(sum_cos, (double)d));
  return d_adds(d_adds(d_sub(a, b), M_E), 20.0);
}

/* objectives.py:88-113 (d == 2 only; caller validates) */
static double goldstein_price_f(const double *x, int d) {
  (void)d;
  double x1 = x[0], x2 = x[1];
  double s = x1 + x2 + 1.0;
  double first = 1.0 + s * s *
                           (19.0 - 14.0 * x1 + 3.0 * x1 * x1 - 14.0 * x2 +
                            6.0 * x1 * x2 + 3.0 * x2 * x2);
  double t = 2.0 * x1 - 3.0 * x2;
  double second = 30.0 + t * t *
                             (18.0 - 32.0 * x1 + 12.0 * x1 * x1 + 48.0 * x2 -
                              36.0 * x1 * x2 + 27.0 * x2 * x2);
  return first * second;
}
static dual goldstein_price_d(const dual *x, int d, int *err) {
  (void)d;
  (void)err;
  dual x1 = x[0], x2 = x[1];
  dual s = d_adds(d_add(x1, x2), 1.0);
  /* 19.0 - 14.0*x1 + 3.0*x1*x1 - 14.0*x2 + 6.0*x1*x2 + 3.0*x2*x2 (left fold) */
  dual p = d_rsubs(19.0, d_muls(x1, 14.0));
  p = d_add(p, d_mul(d_muls(x1, 3.0), x1));
  p = d_sub(p, d_muls(x2, 14.0));
  p = d_add(p, d_mul(d_muls(x1, 6.0), x2));
  p = d_add(p, d_mul(d_muls(x2, 3.0), x2));
  dual first = d_adds(d_mul(d_mul(s, s), p), 1.0);
  dual t = d_sub(d_muls(x1, 2.0), d_muls(x2, 3.0));
  dual q = d_rsubs(18.0, d_muls(x1, 32.0));
  q = d_add(q, d_mul(d_muls(x1, 12.0), x1));
  q = d_add(q, d_muls(x2, 48.0));
  q = d_sub(q, d_mul(d_muls(x1, 36.0), x2));
  q = d_add(q, d_mul(d_muls(x2, 27.0), x2));
  dual second = d_adds(d_mul(d_mul(t, t), q), 30.0);
  return d_mul(first, second);
}

double oracle_objective(int obj, const double *x, int d) {
  switch (obj) {
    case ZEUS_OBJ_ROSENBROCK: return rosenbrock_f(x, d);
    case ZEUS_OBJ_RASTRIGIN: return rastrigin_f(x, d);
    case ZEUS_OBJ_ACKLEY: return ackley_f(x, d);
    case ZEUS_OBJ_GOLDSTEIN_PRICE: return goldstein_price_f(x, d);
    default: return NAN;
  }
}

static dual objective_dual(int obj, const dual *x, int d, int *err) {
  switch (obj) {
    case ZEUS_OBJ_ROSENBROCK: return rosenbrock_d(x, d, err);
    case ZEUS_OBJ_RASTRIGIN: return rastrigin_d(x, d, err);
    case ZEUS_OBJ_ACKLEY: return ackley_d(x, d, err);
    case ZEUS_OBJ_GOLDSTEIN_PRICE: return goldstein_price_d(x, d, err);
    default: *err = 1; return D(NAN, NAN);
  }
}

/* forward_gradient (autodiff.py:243-266): d passes, seeding coordinate i's
 * tangent with 1.0 and resetting it afterwards.  Returns 1 on DomainError. */
int oracle_gradient(int obj, const double *x, int d, double *grad) {
  dual xd_stack[64];
  dual *xd = d <= 64 ? xd_stack : (dual *)malloc(sizeof(dual) * (size_t)d);
  for (int i = 0; i < d; ++i) xd[i] = D(x[i], 0.0);
  int err = 0;
  for (int i = 0; i < d && !err; ++i) {
    xd[i].d = 1.0;
    dual res = objective_dual(obj, xd, d, &err);
    grad[i] = res.d;
    xd[i].d = 0.0;
  }
  if (xd != xd_stack) free(xd);
  return err;
}

/* ------------------------------------------------------------------------ */
/* PSO (pso.py:73-164)                                                       */
/* ------------------------------------------------------------------------ */

/* np.argmin semantics: first NaN if any, else first minimum (pso.py:73-76). */
int64_t oracle_argmin(const double *v, int64_t n) {
  int64_t best = 0;
  for (int64_t i = 0; i < n; ++i)
    if (isnan(v[i])) return i;
  for (int64_t i = 1; i < n; ++i)
    if (v[i] < v[best]) best = i;
  return best;
}

static void reduce_global_best(int d, int64_t n, const double *pbest,
                               const double *pval, double *gX, double *gF,
                               int64_t *gidx) {
  int64_t b = oracle_argmin(pval, n);
  memcpy(gX, pbest + b * d, sizeof(double) * (size_t)d);
  *gF = pval[b];
  if (gidx) *gidx = b;
}

/* init_swarm (pso.py:79-120).  Arrays are row-major [n][d] like the reference.
 * Draw order per particle: k in [0,d) positions, [d,2d) velocities. */
void oracle_pso_init(int obj, int d, int64_t n, uint64_t seed, double lower,
                     double upper, double *x, double *v, double *pbest,
                     double *pval, double *gX, double *gF) {
  double vr = upper - lower;
  for (int64_t i = 0; i < n; ++i) {
    oracle_draw_uniform(seed, (uint64_t)i, 0, d, lower, upper, x + i * d);
    oracle_draw_uniform(seed, (uint64_t)i, (uint64_t)d, d, -vr, vr, v + i * d);
    pval[i] = oracle_objective(obj, x + i * d, d);
  }
  memcpy(pbest, x, sizeof(double) * (size_t)(n * d));
  reduce_global_best(d, n, pbest, pval, gX, gF, NULL);
}

/* update_swarm (pso.py:123-164) for 0-based sweep index s: draws
 * k in [2d(s+1), 2d(s+2)), first d = r1, next d = r2. */
void oracle_pso_sweep(int obj, int d, int64_t n, uint64_t seed, int sweep,
                      double w, double c1, double c2, double *x, double *v,
                      double *pbest, double *pval, double *gX, double *gF) {
  double *g = (double *)malloc(sizeof(double) * (size_t)d);
  double *r = (double *)malloc(sizeof(double) * (size_t)(2 * d));
  memcpy(g, gX, sizeof(double) * (size_t)d); /* previous barrier's best */
  uint64_t k0 = (uint64_t)(2 * d) * (uint64_t)(sweep + 1);
  for (int64_t i = 0; i < n; ++i) {
    oracle_draw_uniform(seed, (uint64_t)i, k0, 2 * d, 0.0, 1.0, r);
    double *xi = x + i * d, *vi = v + i * d, *pi = pbest + i * d;
    for (int k = 0; k < d; ++k) {
      /* numpy: w*v + c1*r1*(p-x) + c2*r2*(g-x), left to right, no FMA */
      double nv = w * vi[k] + c1 * r[k] * (pi[k] - xi[k]) +
                  c2 * r[d + k] * (g[k] - xi[k]);
      vi[k] = nv;
      xi[k] = xi[k] + nv;
    }
    double f = oracle_objective(obj, xi, d);
    if (f < pval[i]) {
      pval[i] = f;
      memcpy(pi, xi, sizeof(double) * (size_t)d);
    }
  }
  reduce_global_best(d, n, pbest, pval, gX, gF, NULL);
  free(g);
  free(r);
}

/* ------------------------------------------------------------------------ */
/* Line search (linesearch.py:40-71)                                         */
/* ------------------------------------------------------------------------ */

static double dot(const double *a, const double *b, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += a[i] * b[i];
  return s;
}

double oracle_armijo(int obj, int d, const double *x, const double *p,
                     const double *g, double f0, double c1, double alpha0,
                     int iter_ls, double shrink, double *xt, double *ft,
                     int *trials) {
  double ddir = dot(g, p, d);
  double alpha = alpha0;
  for (int k = 0; k < iter_ls + 1; ++k) {
    for (int j = 0; j < d; ++j) xt[j] = x[j] + alpha * p[j];
    double f = jitter(oracle_objective(obj, xt, d));
    *ft = f;
    *trials = k + 1;
    if (f <= f0 + c1 * alpha * ddir) return alpha;
    if (k < iter_ls) alpha *= shrink;
  }
  return alpha;
}

/* ------------------------------------------------------------------------ */
/* Inverse-Hessian update (bfgs.py:59-77): V H V^T + rho dx dx^T, then       */
/* 0.5 (U + U^T).  Returns 0 when the curvature guard skipped the update     */
/* (H untouched), 1 otherwise.                                              */
/* ------------------------------------------------------------------------ */

int oracle_hessian_update(int d, double *H, const double *dx, const double *dg) {
  double curvature = dot(dx, dg, d);
  double ndx = sqrt(dot(dx, dx, d)), ndg = sqrt(dot(dg, dg, d));
  if (curvature <= ZEUS_CURVATURE_FLOOR * ndx * ndg) return 0;
  double rho = 1.0 / curvature;
  size_t dd = (size_t)d * (size_t)d;
  double *V = (double *)malloc(sizeof(double) * dd);
  double *VT = (double *)malloc(sizeof(double) * dd);
  double *T = (double *)malloc(sizeof(double) * dd);
  double *U = (double *)malloc(sizeof(double) * dd);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      V[i * d + j] = (i == j ? 1.0 : 0.0) - rho * (dx[i] * dg[j]);
      VT[j * d + i] = V[i * d + j];
    }
  /* T = V @ H and U = T @ V^T.  Each element is the k-ordered sum
   * ((0 + a_0 b_0) + a_1 b_1) + ... exactly as a dot-product loop would form
   * it; the loops run i-k-j so the j loop is a plain (vectorisable) axpy that
   * does not reorder any element's additions. */
  for (size_t e = 0; e < dd; ++e) T[e] = 0.0;
  for (int i = 0; i < d; ++i)
    for (int k = 0; k < d; ++k) {
      double a = V[i * d + k];
      const double *Hk = H + (size_t)k * d;
      double *Ti = T + (size_t)i * d;
      for (int j = 0; j < d; ++j) Ti[j] += a * Hk[j];
    }
  for (size_t e = 0; e < dd; ++e) U[e] = 0.0;
  for (int i = 0; i < d; ++i)
    for (int k = 0; k < d; ++k) {
      double a = T[i * d + k];
      const double *Vk = VT + (size_t)k * d;
      double *Ui = U + (size_t)i * d;
      for (int j = 0; j < d; ++j) Ui[j] += a * Vk[j];
    }
  for (int i = 0; i < d; ++i) /* + rho dx dx^T */
    for (int j = 0; j < d; ++j) U[i * d + j] = U[i * d + j] + rho * (dx[i] * dx[j]);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) H[i * d + j] = 0.5 * (U[i * d + j] + U[j * d + i]);
  free(V);
  free(VT);
  free(T);
  free(U);
  return 1;
}

/* ------------------------------------------------------------------------ */
/* bfgs_run (bfgs.py:80-156)                                                 */
/* ------------------------------------------------------------------------ */

void oracle_bfgs_run(int obj, int d, const double *x0, double theta,
                     int iter_bfgs, double c1, double alpha0, int iter_ls,
                     double shrink, volatile const int *stop_flag,
                     zeus_oracle_outcome *out, double *x_final) {
  size_t bytes = sizeof(double) * (size_t)d;
  double *x = (double *)malloc(bytes), *g = (double *)malloc(bytes);
  double *p = (double *)malloc(bytes), *xn = (double *)malloc(bytes);
  double *gn = (double *)malloc(bytes), *dx = (double *)malloc(bytes);
  double *dg = (double *)malloc(bytes);
  double *H = (double *)calloc((size_t)d * (size_t)d, sizeof(double));
  for (int i = 0; i < d; ++i) H[i * d + i] = 1.0;
  memcpy(x, x0, bytes);
  int have_grad = 0, k = 0, status = ZEUS_DIVERGED;
  int64_t ls_trials = 0, grads = 0;
  double gnorm = INFINITY;
  for (;;) {
    if (stop_flag && *stop_flag) {
      status = ZEUS_STOPPED;
      break;
    }
    if (!have_grad) {
      ++grads;
      if (oracle_gradient(obj, x, d, g)) {
        status = ZEUS_DOMAIN_ERROR;
        break;
      }
      for (int i = 0; i < d; ++i) g[i] = jitter(g[i]);
      have_grad = 1;
      gnorm = sqrt(dot(g, g, d));
    }
    if (gnorm < theta) {
      status = ZEUS_CONVERGED;
      break;
    }
    if (k >= iter_bfgs) {
      status = ZEUS_DIVERGED;
      break;
    }
    for (int i = 0; i < d; ++i) p[i] = jitter(-dot(H + (size_t)i * d, g, d));
    double f0 = jitter(oracle_objective(obj, x, d));
    double ft;
    int trials;
    oracle_armijo(obj, d, x, p, g, f0, c1, alpha0, iter_ls, shrink, xn, &ft,
                  &trials);
    ls_trials += trials;
    ++grads;
    if (oracle_gradient(obj, xn, d, gn)) {
      status = ZEUS_DOMAIN_ERROR;
      break;
    }
    for (int i = 0; i < d; ++i) gn[i] = jitter(gn[i]);
    for (int i = 0; i < d; ++i) {
      dx[i] = xn[i] - x[i];
      dg[i] = gn[i] - g[i];
    }
    if (oracle_hessian_update(d, H, dx, dg) && jit_state)
      for (int i = 0; i < d; ++i)
        for (int j = i; j < d; ++j) H[i * d + j] = H[j * d + i] = jitter(H[i * d + j]);
    memcpy(x, xn, bytes);
    memcpy(g, gn, bytes);
    gnorm = sqrt(dot(g, g, d));
    ++k;
  }
  out->f_final = oracle_objective(obj, x, d);
  out->grad_norm = gnorm;
  out->iterations = k;
  out->status = status;
  out->ls_trials = ls_trials;
  out->grad_evals = grads;
  memcpy(x_final, x, bytes);
  free(x); free(g); free(p); free(xn); free(gn); free(dx); free(dg); free(H);
}

/* ------------------------------------------------------------------------ */
/* Batch BFGS over starts with a pthread pool (the reference's fork pool,    */
/* driver.py:153-202, as threads).  Deterministic: no early stop.           */
/* ------------------------------------------------------------------------ */

typedef struct {
  int obj, d, iter_bfgs, iter_ls;
  double theta, c1, alpha0, shrink;
  int64_t n;
  const double *x0; /* [n][d] */
  double *x_final;  /* [n][d] */
  zeus_oracle_outcome *out;
  int64_t next;
  uint64_t jitter_seed; /* 0: exact restatement */
  pthread_mutex_t lock;
} batch_ctx;

static void *batch_worker(void *arg) {
  batch_ctx *c = (batch_ctx *)arg;
  for (;;) {
    pthread_mutex_lock(&c->lock);
    int64_t lo = c->next;
    int64_t hi = lo + 4 < c->n ? lo + 4 : c->n;
    c->next = hi;
    pthread_mutex_unlock(&c->lock);
    if (lo >= c->n) break;
    for (int64_t i = lo; i < hi; ++i) {
      uint64_t js = c->jitter_seed ^ ((uint64_t)i * 0xd1342543de82ef95ull);
      jit_state = c->jitter_seed ? (splitmix64(&js) | 1u) : 0u;
      oracle_bfgs_run(c->obj, c->d, c->x0 + i * c->d, c->theta, c->iter_bfgs,
                      c->c1, c->alpha0, c->iter_ls, c->shrink, NULL,
                      c->out + i, c->x_final + i * c->d);
    }
  }
  jit_state = 0;
  return NULL;
}

void oracle_bfgs_batch(int obj, int d, int64_t n, const double *x0,
                       double theta, int iter_bfgs, double c1, double alpha0,
                       int iter_ls, double shrink, int threads,
                       zeus_oracle_outcome *out, double *x_final) {
  oracle_bfgs_batch_jitter(obj, d, n, x0, theta, iter_bfgs, c1, alpha0, iter_ls, shrink,
                           threads, 0, out, x_final);
}

void oracle_bfgs_batch_jitter(int obj, int d, int64_t n, const double *x0,
                              double theta, int iter_bfgs, double c1, double alpha0,
                              int iter_ls, double shrink, int threads, uint64_t jitter_seed,
                              zeus_oracle_outcome *out, double *x_final) {
  batch_ctx c;
  c.jitter_seed = jitter_seed;
  c.obj = obj; c.d = d; c.iter_bfgs = iter_bfgs; c.iter_ls = iter_ls;
  c.theta = theta; c.c1 = c1; c.alpha0 = alpha0; c.shrink = shrink;
  c.n = n; c.x0 = x0; c.x_final = x_final; c.out = out; c.next = 0;
  pthread_mutex_init(&c.lock, NULL);
  if (threads < 1) threads = 1;
  pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, batch_worker, &c);
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
  pthread_mutex_destroy(&c.lock);
}

/* reduce_best (driver.py:115-134): strict '<' in index order over outcomes
 * that are not domain errors and whose f_final is not NaN.  -1 if none. */
int64_t oracle_reduce_best(const zeus_oracle_outcome *out, int64_t n) {
  int64_t best = -1;
  for (int64_t i = 0; i < n; ++i) {
    if (out[i].status == ZEUS_DOMAIN_ERROR || isnan(out[i].f_final)) continue;
    if (best < 0 || out[i].f_final < out[best].f_final) best = i;
  }
  return best;
}

/* zeus_run in deterministic mode (driver.py:220-265 with required_c = N):
 * PSO is single-threaded by design (driver.py:237-240); BFGS runs on the pool.
 * Returns the best index (or -1).  x/v/pbest/pval are caller scratch [n][d]. */
int64_t oracle_zeus_run(int obj, int d, int64_t n, uint64_t seed, double lower,
                        double upper, int iter_pso, double w, double c1_pso,
                        double c2_pso, double theta, int iter_bfgs,
                        double c1_ls, double alpha0, int iter_ls, double shrink,
                        int threads, double *x, double *v, double *pbest,
                        double *pval, double *gX, double *pso_best,
                        zeus_oracle_outcome *out, double *x_final) {
  double gF;
  oracle_pso_init(obj, d, n, seed, lower, upper, x, v, pbest, pval, gX, &gF);
  for (int s = 0; s < iter_pso; ++s)
    oracle_pso_sweep(obj, d, n, seed, s, w, c1_pso, c2_pso, x, v, pbest, pval,
                     gX, &gF);
  *pso_best = gF;
  oracle_bfgs_batch(obj, d, n, x, theta, iter_bfgs, c1_ls, alpha0, iter_ls,
                    shrink, threads, out, x_final);
  return oracle_reduce_best(out, n);
}
