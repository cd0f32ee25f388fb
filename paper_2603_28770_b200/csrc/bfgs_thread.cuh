// bfgs_thread.cuh -- multistart BFGS (bfgs.py:80-156) for small d, one THREAD
// per start (d <= 16).
//
// At d = 10 a warp-per-start kernel keeps 10 of 32 lanes busy; here every
// lane runs its own start, so every FP64 instruction does useful work and no
// shuffle or barrier sits on an iteration's path.  Per thread:
//   * x, p, g in registers (fully unrolled over the compile-time bound D >= d,
//     predicated past d);
//   * the inverse Hessian H (bfgs.py:59-77) as its packed upper triangle
//     (D (D + 1) / 2 doubles -- H stays exactly symmetric, like the
//     reference's 0.5 (H + H^T)) in shared memory, interleaved by thread
//     (element e of thread t at e * NT + t: conflict-free);
//   * Armijo trials (linesearch.py:60-71) one at a time, value-only terms
//     folded in the reference's sequential order, so f is bit-identical to the
//     reference wherever libm agrees; the warp runs as many trial rounds as
//     its slowest start needs;
//   * the gradient at the accepted point from one forward-mode term-tangent
//     pass (autodiff.py:243-266 restricted to the terms that contain x_i);
//   * u = H dg and w = H g' from the packed triangle, then the rank-2 update
//     H += dx a^T + u b^T applied in place (the O(d^2) form of bfgs.py:72-77)
//     and p' = -H' g' from the identity used by the warp kernels.
// A start still running at iteration k1 is handed to the CTA-team resume
// kernel through the shared carry-record format (bfgs_common.cuh), so the few
// starts that run to the cap (config 2: ~10 of 65,536) get 8 warps each.
#pragma once
#include "bfgs_common.cuh"

namespace zeus {

namespace {

constexpr int kThreadBlock = 64;

template <int D>
__host__ __device__ constexpr int tri_size() { return D * (D + 1) / 2; }
// packed index of (i, j), i <= j
__host__ __device__ constexpr int tri(int D, int i, int j) { return i * D - i * (i - 1) / 2 + (j - i); }

}  // namespace

template <class Obj, int D>
struct ThreadStart {
  static constexpr int NA = Obj::NACC;
  static constexpr int KT = Obj::KT;
  double* Hs;  // this thread's packed triangle: element e at Hs[e * kThreadBlock]

  __device__ __forceinline__ double& H(int e) const { return Hs[e * kThreadBlock]; }

  // f at x + alpha p (alpha == 0 -> x itself is NOT special-cased: callers pass
  // the point through xs directly) -- value-only terms, reference-order fold.
  template <class M>
  __device__ __forceinline__ double value(int d, const double (&xs)[D + 1], double acc[NA],
                                          bool& oor, bool& err) const {
    const int nt = Obj::nterms(d);
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = Obj::init(a, d);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (j < nt) {
        double t[NA];
        Obj::template term<M>([&](int q) { return xs[q]; }, j, d, t, oor);
#pragma unroll
        for (int a = 0; a < NA; ++a) acc[a] = acc[a] + t[a];
      }
    }
    return Obj::finish(acc, d, err);
  }

  // value + gradient at xs from one term-tangent pass
  template <class M>
  __device__ __forceinline__ double value_grad(int d, const double (&xs)[D + 1], double acc[NA],
                                               double (&gout)[D + 1], bool& oor,
                                               bool& err) const {
    const int nt = Obj::nterms(d);
    double tn[D + 1][KT];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = Obj::init(a, d);
#pragma unroll
    for (int j = 0; j <= D; ++j)
#pragma unroll
      for (int k = 0; k < KT; ++k) tn[j][k] = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (j < nt) {
        double t[NA];
        Obj::template term_tan<M>([&](int q) { return xs[q]; }, j, d, t, tn[j], oor);
#pragma unroll
        for (int a = 0; a < NA; ++a) acc[a] = acc[a] + t[a];
      }
    }
    bool ferr = false;
    const double f = Obj::finish(acc, d, ferr);
    auto TA = [&](int j, int k) { return tn[j][k]; };
#pragma unroll
    for (int i = 0; i < D; ++i) {
      gout[i] = 0.0;
      if (i < d) gout[i] = Obj::grad_from_tan(TA, i, d, acc, err);
    }
    gout[D] = 0.0;
    return f;
  }

  __device__ void run(const BfgsArgs& A, long long s) {
    const int d = A.d;
    double x[D + 1], p[D + 1], g[D + 1];
    double acc[NA];
    double f0 = 0.0;
    int k = 0, status = ZEUS_DIVERGED, ls_trials = 0, grads = 0, prev_trials = 1;
    double gsq = __longlong_as_double(0x7ff0000000000000LL);  // |g|^2 (|g| = inf: no gradient)
    double ddir = 0.0;

#pragma unroll
    for (int j = 0; j <= D; ++j) x[j] = p[j] = g[j] = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (j < d) x[j] = A.x0[(int64_t)j * A.ldx + s];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = i; j < D; ++j) H(tri(D, i, j)) = i == j ? 1.0 : 0.0;

    {  // f(x0), stop probe, first gradient; p = -g (H0 = I)
      bool oor = false, err = false;
      double gx[D + 1];
      f0 = value_grad<FastMath>(d, x, acc, gx, oor, err);
      if constexpr (Obj::kOorIsError) {  // user objective: oor is a DomainError
        if (oor) {
          bool verr = false, fe = false;
          double av[NA];
          const double fv = value<FastMath>(d, x, av, verr, fe);
          f0 = verr ? __longlong_as_double(0x7ff8000000000000LL) : fv;  // f(x) raised: NaN
          err = true;
        }
      } else if (oor) {
        oor = false;
        err = false;
        f0 = value_grad<PreciseMath>(d, x, acc, gx, oor, err);
      }
      if (A.stop_flag && *(volatile int*)A.stop_flag) {
        status = ZEUS_STOPPED;
        goto done;
      }
      ++grads;
      if (err) {
        status = ZEUS_DOMAIN_ERROR;
        goto done;
      }
      double gg = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        g[j] = gx[j];
        p[j] = -gx[j];
        gg = fma(gx[j], gx[j], gg);
      }
      gsq = gg;
      ddir = -gg;
    }

    for (;;) {
      if (gsq <= A.gsq_max) {  // |g| < theta (bfgs.py:118)
        status = ZEUS_CONVERGED;
        break;
      }
      if (k >= A.cap) {
        status = ZEUS_DIVERGED;
        break;
      }
      if (A.k1 > 0 && k == A.k1) {  // straggler: hand over to the CTA-team resume kernel
        promote(A, s, x, p, g, f0, acc, gsq, ddir, k, ls_trials, grads, prev_trials);
        return;
      }
      // ---- Armijo backtracking (linesearch.py:60-71), one trial at a time
      double alpha = A.alpha0, f_new = 0.0, acc_new[NA];
      int t = 0;
      bool trial_err = false;
      for (;; ++t) {
        double xt[D + 1];
#pragma unroll
        for (int j = 0; j <= D; ++j) xt[j] = x[j] + alpha * p[j];
        bool oor = false, ferr = false;
        double fb = value<FastMath>(d, xt, acc_new, oor, ferr);
        if constexpr (Obj::kOorIsError) {
          if (oor) {  // DomainError inside the line search (bfgs.py: domain_error)
            trial_err = true;
            break;
          }
        } else if (oor) {
          fb = value<PreciseMath>(d, xt, acc_new, oor, ferr);
        }
        if (fb <= f0 + A.c1 * alpha * ddir || t >= A.iter_ls) {  // NaN fails
          f_new = fb;
          break;
        }
        alpha = alpha * A.shrink;
      }
      if (trial_err) {
        status = ZEUS_DOMAIN_ERROR;
        break;
      }
      ls_trials += t + 1;
      prev_trials = t + 1;

      // ---- x_new and the gradient there; DomainError leaves x, k unchanged
      double xn[D + 1], gn[D + 1];
#pragma unroll
      for (int j = 0; j <= D; ++j) xn[j] = x[j] + alpha * p[j];
      ++grads;
      {
        bool oor = false, err = false;
        double accg[NA];
        value_grad<FastMath>(d, xn, accg, gn, oor, err);
        if constexpr (Obj::kOorIsError) {
          err = err || oor;
        } else if (oor) {
          oor = false;
          err = false;
          value_grad<PreciseMath>(d, xn, accg, gn, oor, err);
        }
        if (err) {
          status = ZEUS_DOMAIN_ERROR;
          break;
        }
      }
      // ---- u = H dg, w = H g' from the packed triangle; dots
      double dx[D + 1], dg[D + 1], u[D + 1], w[D + 1];
#pragma unroll
      for (int j = 0; j <= D; ++j) {
        dx[j] = xn[j] - x[j];
        dg[j] = gn[j] - g[j];
        u[j] = w[j] = 0.0;
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
#pragma unroll
        for (int j = i; j < D; ++j) {
          if (j < d) {
            const double h = H(tri(D, i, j));
            u[i] = fma(h, dg[j], u[i]);
            w[i] = fma(h, gn[j], w[i]);
            if (j != i) {
              u[j] = fma(h, dg[i], u[j]);
              w[j] = fma(h, gn[i], w[j]);
            }
          }
        }
      }
      double gg = 0.0, curv = 0.0, dxdx = 0.0, dgdg = 0.0, dgu = 0.0, ug = 0.0, xg = 0.0, wg = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        gg = fma(gn[j], gn[j], gg);
        curv = fma(dx[j], dg[j], curv);
        dxdx = fma(dx[j], dx[j], dxdx);
        dgdg = fma(dg[j], dg[j], dgdg);
        dgu = fma(dg[j], u[j], dgu);
        ug = fma(u[j], gn[j], ug);
        xg = fma(dx[j], gn[j], xg);
        wg = fma(w[j], gn[j], wg);
      }
      (void)wg;
      const bool upd = curvature_update(curv, dxdx, dgdg);  // bfgs.py:69-71
      double pd = 0.0;
      if (upd) {
        const double rho = 1.0 / curv;
        const double cc = fma(rho * rho, dgu, rho);
        // p' = -(w - rho dx (u.g') - rho u (dx.g') + c dx (dx.g'))
#pragma unroll
        for (int j = 0; j < D; ++j) {
          p[j] = -(w[j] + fma(dx[j], fma(cc, xg, -rho * ug), -rho * xg * u[j]));
          pd = fma(gn[j], p[j], pd);
        }
        // H += dx a^T + u b^T, a = c dx - rho u, b = -rho dx (upper triangle)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          if (j < d) {
            const double aj = fma(cc, dx[j], -rho * u[j]), bj = -rho * dx[j];
#pragma unroll
            for (int i = 0; i <= j; ++i) {
              double& h = H(tri(D, i, j));
              h = fma(dx[i], aj, fma(u[i], bj, h));
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < D; ++j) {
          p[j] = -w[j];
          pd = fma(gn[j], p[j], pd);
        }
      }
#pragma unroll
      for (int j = 0; j <= D; ++j) {
        x[j] = xn[j];
        g[j] = gn[j];
      }
      f0 = f_new;
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[a] = acc_new[a];
      gsq = gg;
      ddir = pd;  // np.dot(g, p) of the next line search
      ++k;
      if (A.stop_flag && *(volatile int*)A.stop_flag) {
        status = ZEUS_STOPPED;
        break;
      }
    }

  done:
    const zeus_bfgs_out& o = A.out;
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (j < d) o.x_final[(int64_t)j * o.ld_out + s] = x[j];
    if (o.rows) {
#pragma unroll
      for (int j = 0; j < D; ++j)
        if (j < d) o.rows[(int64_t)s * o.ld_rows + j] = x[j];
    }
    write_row_tail(o, s, d, f0, sqrt(gsq), k, status, ls_trials, grads);
    o.f_final[s] = f0;
    o.grad_norm[s] = sqrt(gsq);
    o.iterations[s] = k;
    o.status[s] = (uint8_t)status;
    if (o.ls_trials) o.ls_trials[s] = ls_trials;
    if (o.grad_evals) o.grad_evals[s] = grads;
    if (status == ZEUS_CONVERGED && A.stop_counter) {
      const unsigned long long old = atomicAdd_system(A.stop_counter, 1ull);
      if ((long long)old + 1 == A.required_c) atomicExch_system(A.stop_flag, 1);
    }
  }

  // carry record (bfgs_common.cuh): H written in full, both triangles
  __device__ void promote(const BfgsArgs& A, long long s, const double (&x)[D + 1],
                          const double (&p)[D + 1], const double (&g)[D + 1], double f0,
                          const double acc[NA], double gsq, double ddir, int k, int ls_trials,
                          int grads, int prev_trials) const {
    const int d = A.d;
    const unsigned long long slot = atomicAdd(A.promo_count, 1ull);
    double* rec = A.carry + (size_t)slot * A.carry_stride;
    rec[0] = (double)s;
    rec[1] = k;
    rec[2] = ls_trials;
    rec[3] = grads;
    rec[4] = prev_trials;
    rec[5] = f0;
    rec[6] = acc[0];
    rec[7] = NA > 1 ? acc[NA - 1] : 0.0;
    rec[8] = gsq;
    rec[9] = ddir;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (j < d) {
        rec[kCarryHead + j] = x[j];
        rec[kCarryHead + d + j] = g[j];
        rec[kCarryHead + 2 * d + j] = p[j];
      }
    }
    double* Hr = rec + kCarryHead + 3 * d;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = i; j < D; ++j)
        if (j < d) {
          const double h = H(tri(D, i, j));
          Hr[(int64_t)i * d + j] = h;
          Hr[(int64_t)j * d + i] = h;
        }
  }
};

template <class Obj, int D>
__global__ void __launch_bounds__(kThreadBlock) bfgs_thread_kernel(BfgsArgs A) {
  extern __shared__ double sm[];
  ThreadStart<Obj, D> T;
  T.Hs = sm + threadIdx.x;
  for (;;) {
    const long long s = (long long)atomicAdd(A.work, 1ull);
    if (s >= A.n) break;
    T.run(A, s);
  }
}

}  // namespace zeus
