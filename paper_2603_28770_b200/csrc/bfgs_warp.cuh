// bfgs_warp.cuh -- device code of the warp-per-start BFGS kernel (bfgs.cu
// holds its host launch, the tier orchestration and the C ABI).  A header so
// that the NVRTC program of a user objective (plugin.cu, user_program.cuh)
// instantiates the same kernel for d > 16.  Design notes: bfgs.cu.
#pragma once
#include "bfgs_common.cuh"

namespace zeus {

// Named-barrier helpers for the helper-warp mode.  Warp 0 and the helpers
// meet at barrier 1 from different code locations, so these are the
// NON-aligned forms (barrier.sync / barrier.red): bar.sync is
// barrier.sync.aligned, which requires every thread to execute the same
// instruction (compute-sanitizer synccheck flags it).
__device__ __forceinline__ void bar1(int n) {
  asm volatile("barrier.sync 1, %0;" ::"r"(n) : "memory");
}
__device__ __forceinline__ bool bar1_or(int n, bool v) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\t"
      "barrier.red.or.pred q, 1, %2, p;\n\tselp.s32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((int)v), "r"(n)
      : "memory");
  return r != 0;
}

// Task published by the driving warp to its helper warps (NH > 0).
struct HelperTask {
  int B;      // trials in the batch (0: evaluate x itself); -1: exit
  int xsel;   // which smem buffer holds the current x (x / xn swap)
};

// NH == 0: one warp per start, blocks of kBfgsWarps independent warps.
// NH  > 0: one start per CTA of 1 + NH warps; warp 0 runs the iteration and
//          the NH helper warps only evaluate the speculative term batches
//          (promoted stragglers: the batch work spreads over 32 (1+NH) lanes
//          while everything else stays warp-synchronous in warp 0).
template <class Obj, int DR, int NH = 0>
struct BfgsWarp {
  static constexpr int NT = 32 * (NH + 1);
  // shared-memory vectors of this warp (each d doubles unless noted)
  double *x, *xn, *p, *g, *gn, *row4, *T;
  double* H;  // smem / global H (DR == 0)
  const double* alpha_tab;
  HelperTask* task;
  double* xbuf[2];  // the two x buffers (helper mode needs to name them)
  TermIdx tix;      // helper mode: this thread's term-pass indices (fixed per kernel)
#ifdef ZEUS_PHASE_TIMING
  long long _pt;  // phase clock (scripts/latency_probe.py)
#endif

  // Evaluate a batch: NH == 0 -> eval_batch over the warp; NH > 0 -> publish
  // the task (batch_publish), the NH helper warps run the term pass while
  // warp 0 does work that needs no trial result (the run loop: the previous
  // iteration's g.p reduction and the pending rank-2 update of H), then warp
  // 0 waits for the terms and folds (batch_finish).
  __device__ __forceinline__ void batch_publish(int B) {
    const int lane = threadIdx.x & 31;  // (warp 0: == threadIdx.x)
    (void)lane;
    if (lane == 0) {
      task->B = B;
      task->xsel = (x == xbuf[0]) ? 0 : 1;
    }
    __syncwarp();
    PHASE(6);  // batch setup (alpha table, task)
    bar1(NT);  // A: task, x, p, alphas visible to the helpers
    PHASE(7);  // barrier A
  }
  __device__ __forceinline__ double batch_finish(const BfgsArgs& A, int B, int d, int lane,
                                                 double acc[Obj::NACC]) {
    PHASE(8);  // warp 0's own work during the batch
    const bool any_oor = bar1_or(NT, false);
    PHASE(9);  // barrier B (waits for the helpers' terms)
    if (any_oor) bar1(NT);  // the helpers re-evaluate with libm
    const int nt = Obj::nterms(d);
    const int nb = B > 0 ? B : 1;
    double f = 0.0;
    if (lane < nb) {
#pragma unroll
      for (int a = 0; a < Obj::NACC; ++a) {
        const double* row = T + (a * A.bmax + lane) * A.tstride;
        acc[a] = seq_fold<DR>(row, nt, Obj::init(a, d));
      }
      bool err = false;
      f = Obj::finish(acc, d, err);
    }
    __syncwarp();
    PHASE(10);  // reference-order folds
    return f;
  }
  __device__ __forceinline__ double evalb(const BfgsArgs& A, int B, const double* alphas, int d,
                                          double* TT, int lane, double acc[Obj::NACC]) {
    if constexpr (NH == 0) {
      return eval_batch<Obj>(B, alphas, d, x, p, T, TT, A.tstride, A.bmax, lane, acc);
    } else {
      batch_publish(B);
      return batch_finish(A, B, d, lane, acc);
    }
  }

  __device__ __forceinline__ double alpha_at(const BfgsArgs& A, int t) const {
    if (t < A.nalpha) return alpha_tab[t];
    double a = alpha_tab[A.nalpha - 1];
    for (int k = A.nalpha - 1; k < t; ++k) a *= A.shrink;
    return a;
  }

  // Write the carry record of a start that reached iteration k1 (layout in
  // bfgs_common.cuh); the pending lazy rank-2 update is applied first so the
  // record holds H_k itself.
  __device__ void promote(const BfgsArgs& A, long long s, int lane, double* hreg, bool pending,
                          double aj, double bj, double f0, const double* acc, double gsq,
                          double ddir, int k, int ls_trials, int grads, int prev_trials) {
    const int d = A.d;
    unsigned long long slot = 0;
    if (lane == 0) slot = atomicAdd(A.promo_count, 1ull);
    slot = __shfl_sync(kFull, slot, 0);
    double* rec = A.carry + (size_t)slot * A.carry_stride;
    if (lane == 0) {
      rec[0] = (double)s;
      rec[1] = k;
      rec[2] = ls_trials;
      rec[3] = grads;
      rec[4] = prev_trials;
      rec[5] = f0;
      rec[6] = acc[0];
      rec[7] = Obj::NACC > 1 ? acc[Obj::NACC - 1] : 0.0;
      rec[8] = gsq;
      rec[9] = ddir;
    }
    for (int j = lane; j < d; j += 32) {
      rec[kCarryHead + j] = x[j];
      rec[kCarryHead + d + j] = g[j];
      rec[kCarryHead + 2 * d + j] = p[j];
    }
    if constexpr (DR > 0) {
      double* Hr = rec + kCarryHead + 3 * d;
      if (lane < d) {
#pragma unroll
        for (int i = 0; i < DR; ++i) {
          if (i < d) {
            double h = hreg[i];
            if (pending) h = fma(row4[4 * i + 2], aj, fma(row4[4 * i + 3], bj, h));
            Hr[(int64_t)i * d + lane] = h;
          }
        }
      }
    }
    __syncwarp();
  }

  // Fresh start s from x0, or (rec != nullptr, helper mode) resume a start
  // promoted by the warp kernel from its carry record (bfgs_common.cuh).
  __device__ void run(const BfgsArgs& A, long long s, int lane, const double* rec = nullptr) {
#ifdef ZEUS_PHASE_TIMING
    _pt = clock64();
#endif
    const int d = A.d;
    const int C = (d + 31) >> 5;  // columns per lane
    double hreg[DR > 0 ? DR : 1];
    // lane-local state of the owned columns: previous update coefficients
    double a_col[DR > 0 ? 1 : kMaxC], b_col[DR > 0 ? 1 : kMaxC];
#pragma unroll
    for (int c = 0; c < (DR > 0 ? 1 : kMaxC); ++c) a_col[c] = b_col[c] = 0.0;
    double acc[Obj::NACC];
    double* TT = T + Obj::NACC * A.bmax * A.tstride;  // term tangents [KT][bmax][tstride]
    double* atab = TT + Obj::KT * A.bmax * A.tstride;  // per-warp alpha window (32)
    const int bdef = max(1, 32 / max(Obj::nterms(d), 1));  // trials filling one warp
    atab[lane] = alpha_at(A, lane);
    int atab_t0 = 0;
    __syncwarp();
    double f0 = 0.0;
    int k = 0, status = ZEUS_DIVERGED, ls_trials = 0, grads = 0, prev_trials = 1;
    double gsq = __longlong_as_double(0x7ff0000000000000LL);  // |g|^2 (|g| = inf: no gradient)
    double ddir = 0.0, pd_part = 0.0;
    bool pending = false, ddir_pending = false;

    for (int i = d + lane; i < DR; i += 32)  // zero padding rows of row4
      row4[4 * i] = row4[4 * i + 1] = row4[4 * i + 2] = row4[4 * i + 3] = 0.0;
    if (rec) {
      k = (int)rec[1];
      ls_trials = (int)rec[2];
      grads = (int)rec[3];
      prev_trials = (int)rec[4];
      f0 = rec[5];
      acc[0] = rec[6];
      if (Obj::NACC > 1) acc[Obj::NACC - 1] = rec[7];
      gsq = rec[8];
      ddir = rec[9];
      for (int j = lane; j < d; j += 32) {
        x[j] = rec[kCarryHead + j];
        g[j] = rec[kCarryHead + d + j];
        p[j] = rec[kCarryHead + 2 * d + j];
      }
      if constexpr (DR > 0) {
        const double* Hr = rec + kCarryHead + 3 * d;
#pragma unroll
        for (int i = 0; i < DR; ++i) hreg[i] = (i < d && lane < d) ? Hr[(int64_t)i * d + lane] : 0.0;
      }
      __syncwarp();
      goto iterate;
    }

    for (int j = lane; j < d; j += 32) x[j] = A.x0[(int64_t)j * A.ldx + s];
    if constexpr (DR > 0) {
#pragma unroll
      for (int i = 0; i < DR; ++i) hreg[i] = (i == lane) ? 1.0 : 0.0;
    } else {
      for (int i = 0; i < d; ++i)
        for (int j = lane; j < d; j += 32) H[(int64_t)i * A.ldh + j] = (i == j) ? 1.0 : 0.0;
    }
    __syncwarp();

    f0 = evalb(A, 0, nullptr, d, TT, lane, acc);
    f0 = __shfl_sync(kFull, f0, 0);
#pragma unroll
    for (int a = 0; a < Obj::NACC; ++a) acc[a] = __shfl_sync(kFull, acc[a], 0);

    // ---- iteration 0 prologue: stop probe, first gradient, p = -g
    if (A.stop_flag && *(volatile int*)A.stop_flag) {
      status = ZEUS_STOPPED;
      goto done;
    }
    {
      ++grads;
      bool err = false;
      double part = 0.0;
      const TanRow tan0{TT, A.bmax, A.tstride, 0};
      for (int j = lane; j < d; j += 32) {
        const double gj = Obj::grad_from_tan(tan0, j, d, acc, err);
        g[j] = gj;
        p[j] = -gj;  // H0 = I: -(I @ g) is exact
        part = fma(gj, gj, part);
      }
      if (__any_sync(kFull, err)) {
        status = ZEUS_DOMAIN_ERROR;
        goto done;
      }
      const double gg = warp_sum(part);
      gsq = gg;
      ddir = -gg;  // g . (-g)
      __syncwarp();
    }

    PHASE(5);  // prologue: loads, H = I, f(x0), first gradient
  iterate:
    for (;;) {
      if (gsq <= A.gsq_max) {  // |g| < theta (bfgs.py:118), no sqrt on the path
        status = ZEUS_CONVERGED;
        break;
      }
      if (k >= A.cap) {
        status = ZEUS_DIVERGED;
        break;
      }
      if constexpr (DR > 0 && NH == 0) {
        if (A.k1 > 0 && k == A.k1) {  // straggler: hand over to the helper-warp kernel
          promote(A, s, lane, hreg, pending, a_col[0], b_col[0], f0, acc, gsq, ddir, k,
                  ls_trials, grads, prev_trials);
          return;
        }
      }
      // ---- speculative batched Armijo search (linesearch.py:60-71)
      int t_acc = -1;
      bool ls_err = false;  // user objective: DomainError inside the line search
      double f_new = 0.0, acc_new[Obj::NACC];
      int src_row = 0;  // batch row of the accepted trial (its tangents in TT)
      {
        int t0 = 0;
        int B = min(max(prev_trials, bdef), A.bmax);
        for (;;) {
          B = min(B, A.iter_ls + 1 - t0);
          if (t0 != atab_t0) {  // the window's step lengths (t0 = 0: kept from the last round)
            atab[lane] = alpha_at(A, t0 + lane);
            atab_t0 = t0;
            __syncwarp();
          }
          double accb[Obj::NACC];
          // Armijo threshold of this lane's trial (same ops, same order):
          // formed before the batch in warp mode (its latency hides behind
          // the term pass); after it in helper mode, where g.p itself is
          // reduced during the batch
          double thr = 0.0, fb;
          if constexpr (NH == 0) {
            thr = f0 + A.c1 * atab[lane] * ddir;
            fb = evalb(A, B, atab, d, TT, lane, accb);
          } else {
            batch_publish(B);
            if (ddir_pending) {  // g.p of this line search, reduced during the batch
              ddir = warp_sum_n<(DR > 0 && DR <= 16) ? 16 : 32>(pd_part);
              ddir_pending = false;
            }
            if constexpr (DR > 0) {
              if (pending) {  // the previous iteration's rank-2 update of H, also
                const double aj = a_col[0], bj = b_col[0];  // during the batch
#pragma unroll
                for (int i = 0; i < DR; ++i) {
                  const double2 r1 = *reinterpret_cast<const double2*>(row4 + 4 * i + 2);
                  hreg[i] = fma(r1.x, aj, fma(r1.y, bj, hreg[i]));
                }
                pending = false;
              }
            }
            thr = f0 + A.c1 * atab[lane] * ddir;  // also inside the batch window
            fb = batch_finish(A, B, d, lane, accb);
          }
          bool pass = false;
          if (lane < B) pass = fb <= thr;  // NaN fails
          const unsigned m = __ballot_sync(kFull, pass);
          if constexpr (Obj::kOorIsError) {
            // user objective: a trial whose value raised DomainError ends the
            // run (bfgs.py: domain_error) if the sequential search reaches it,
            // i.e. no earlier trial of the batch passed
            const bool verr =
                lane < B && Obj::value_error(TanRow{TT, A.bmax, A.tstride, lane}, d);
            const unsigned me = __ballot_sync(kFull, verr);
            if (me && !(m & ((me & (0u - me)) - 1u))) {
              ls_err = true;
              break;
            }
          }
          int src = -1;
          if (m) {
            src = __ffs(m) - 1;
          } else if (t0 + B > A.iter_ls) {
            src = B - 1;  // fell through: the last trial (shrink^iter_ls)
          }
          if (src >= 0) {
            t_acc = t0 + src;
            src_row = src;
            f_new = __shfl_sync(kFull, fb, src);
#pragma unroll
            for (int a = 0; a < Obj::NACC; ++a) acc_new[a] = __shfl_sync(kFull, accb[a], src);
            const double alpha = __shfl_sync(kFull, lane < B ? atab[lane] : 0.0, src);
            for (int j = lane; j < d; j += 32) xn[j] = x[j] + alpha * p[j];
            break;
          }
          t0 += B;
          B = min(2 * B, A.bmax);
        }
      }
      PHASE(0);  // line search (term pass + folds + ballot + x_new)
      if (ls_err) {
        status = ZEUS_DOMAIN_ERROR;
        break;
      }
      ls_trials += t_acc + 1;
      prev_trials = t_acc + 1;
      __syncwarp();

      // ---- gradient at x_new (bfgs.py:136); DomainError leaves x, k unchanged
      ++grads;
      double part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      {
        bool err = false;
        const TanRow tanr{TT, A.bmax, A.tstride, src_row};
        for (int j = lane; j < d; j += 32) {
          const double gj = Obj::grad_from_tan(tanr, j, d, acc_new, err);
          const double dgj = gj - g[j];
          gn[j] = gj;
          row4[4 * j + 0] = dgj;
          row4[4 * j + 1] = gj;
        }
        if (__any_sync(kFull, err)) {
          status = ZEUS_DOMAIN_ERROR;
          break;
        }
      }
      __syncwarp();

      PHASE(1);  // gradient
      // ---- fused pass over H: lazy rank-2 update, u = H dg, w = H g'
      double u_own[DR > 0 ? 1 : kMaxC], w_own[DR > 0 ? 1 : kMaxC];
      if constexpr (DR > 0) {
        // straight-line over DR rows (row4 zero-padded past d: every load is
        // issued up front), four accumulator chains of DR / 4
        double uq[4] = {0.0, 0.0, 0.0, 0.0}, wq[4] = {0.0, 0.0, 0.0, 0.0};
        const double aj = a_col[0], bj = b_col[0];
#pragma unroll
        for (int i = 0; i < DR; ++i) {
          const double2 r0 = *reinterpret_cast<const double2*>(row4 + 4 * i);
          const double2 r1 = *reinterpret_cast<const double2*>(row4 + 4 * i + 2);
          double h = hreg[i];
          if constexpr (NH == 0) {  // (helper mode applied it during the batch)
            const double upd = fma(r1.x, aj, fma(r1.y, bj, h));
            h = pending ? upd : h;
            hreg[i] = h;
          }
          uq[i & 3] = fma(h, r0.x, uq[i & 3]);
          wq[i & 3] = fma(h, r0.y, wq[i & 3]);
        }
        u_own[0] = (uq[0] + uq[1]) + (uq[2] + uq[3]);
        w_own[0] = (wq[0] + wq[1]) + (wq[2] + wq[3]);
      } else {
        for (int c = 0; c < C; ++c) {
          const int j = lane + 32 * c;
          double u0 = 0.0, u1 = 0.0, w0 = 0.0, w1 = 0.0;
          if (j < d) {
            const double aj = a_col[c], bj = b_col[c];
            double* col = H + j;
            int i = 0;
            for (; i + 1 < d; i += 2) {
              const double2 ra = *reinterpret_cast<const double2*>(row4 + 4 * i);
              const double2 rb = *reinterpret_cast<const double2*>(row4 + 4 * i + 4);
              double ha = col[(int64_t)i * A.ldh], hb = col[(int64_t)(i + 1) * A.ldh];
              if (pending) {
                const double2 sa = *reinterpret_cast<const double2*>(row4 + 4 * i + 2);
                const double2 sb = *reinterpret_cast<const double2*>(row4 + 4 * i + 6);
                ha = fma(sa.x, aj, fma(sa.y, bj, ha));
                hb = fma(sb.x, aj, fma(sb.y, bj, hb));
                col[(int64_t)i * A.ldh] = ha;
                col[(int64_t)(i + 1) * A.ldh] = hb;
              }
              u0 = fma(ha, ra.x, u0);
              w0 = fma(ha, ra.y, w0);
              u1 = fma(hb, rb.x, u1);
              w1 = fma(hb, rb.y, w1);
            }
            if (i < d) {
              const double2 ra = *reinterpret_cast<const double2*>(row4 + 4 * i);
              double ha = col[(int64_t)i * A.ldh];
              if (pending) {
                const double2 sa = *reinterpret_cast<const double2*>(row4 + 4 * i + 2);
                ha = fma(sa.x, aj, fma(sa.y, bj, ha));
                col[(int64_t)i * A.ldh] = ha;
              }
              u0 = fma(ha, ra.x, u0);
              w0 = fma(ha, ra.y, w0);
            }
          }
          u_own[c] = u0 + u1;
          w_own[c] = w0 + w1;
        }
      }

      PHASE(2);  // H pass
      // ---- one 8-value reduction: norms, curvature and the p' scalars
      {
        for (int c = 0; c < C; ++c) {
          const int j = lane + 32 * c;
          if (j >= d) break;
          const double dxj = xn[j] - x[j], dgj = row4[4 * j], gj = gn[j];
          const double uj = u_own[DR > 0 ? 0 : c], wj = w_own[DR > 0 ? 0 : c];
          part[0] = fma(gj, gj, part[0]);
          part[1] = fma(dxj, dgj, part[1]);
          part[2] = fma(dxj, dxj, part[2]);
          part[3] = fma(dgj, dgj, part[3]);
          part[4] = fma(dgj, uj, part[4]);
          part[5] = fma(uj, gj, part[5]);
          part[6] = fma(dxj, gj, part[6]);
          part[7] = fma(wj, gj, part[7]);
        }
        warp_sum8<(DR > 0 && DR <= 16) ? 16 : 32>(part);
      }
      const double curv = part[1];
      // 1/curv issued next to the guard (straight-line), so the two overlap
      const double rinv = 1.0 / curv;
      pending = curvature_update_sl(curv, part[2], part[3]);  // bfgs.py:69-71
      double pd = 0.0;
      __syncwarp();  // row4 (dx/u of the previous iteration) fully consumed
      {
        const double rho = pending ? rinv : 0.0;
        const double cc = pending ? fma(rho * rho, part[4], rho) : 0.0;
        const double ug = part[5], xg = part[6];
        for (int c = 0; c < C; ++c) {
          const int j = lane + 32 * c;
          if (j >= d) break;
          const double dxj = xn[j] - x[j];
          const double uj = u_own[DR > 0 ? 0 : c], wj = w_own[DR > 0 ? 0 : c];
          double pj = -wj;
          if (pending) {
            // p' = -(w - rho dx (u.g') - rho u (dx.g') + c dx (dx.g'))
            pj = -(wj + fma(dxj, fma(cc, xg, -rho * ug), -rho * xg * uj));
            const double aj = fma(cc, dxj, -rho * uj), bj = -rho * dxj;
            if constexpr (DR > 0) {
              a_col[0] = aj;
              b_col[0] = bj;
            } else {
              a_col[c] = aj;
              b_col[c] = bj;
            }
            row4[4 * j + 2] = dxj;
            row4[4 * j + 3] = uj;
          }
          p[j] = pj;
          pd = fma(gn[j], pj, pd);
        }
      }
      PHASE(3);  // 8-value reduction + p' + update coefficients
      // x, g <- x_new, g_new (bfgs.py:141-145)
      {
        double* t = x;
        x = xn;
        xn = t;
        t = g;
        g = gn;
        gn = t;
      }
      f0 = f_new;
#pragma unroll
      for (int a = 0; a < Obj::NACC; ++a) acc[a] = acc_new[a];
      gsq = part[0];
      // np.dot(g, p) of the next line search: in helper mode the reduction
      // runs during the next batch (evalb), here only the lane partial
      if constexpr (NH > 0) {
        pd_part = pd;
        ddir_pending = true;
      } else {
        ddir = warp_sum_n<(DR > 0 && DR <= 16) ? 16 : 32>(pd);
      }
      PHASE(4);  // ddir reduction + swap
      ++k;
      __syncwarp();
      if (A.stop_flag && *(volatile int*)A.stop_flag) {
        status = ZEUS_STOPPED;
        break;
      }
    }

  done:
    const zeus_bfgs_out& o = A.out;
    for (int j = lane; j < d; j += 32) o.x_final[(int64_t)j * o.ld_out + s] = x[j];
    if (o.rows)
      for (int j = lane; j < d; j += 32) o.rows[(int64_t)s * o.ld_rows + j] = x[j];
    if (lane == 0) {
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
    __syncwarp();
  }
};

template <class Obj, int DR, int NH = 0>
__global__ void __launch_bounds__(NH > 0 ? 32 * (NH + 1) : kBfgsWarps * 32,
                                  NH > 0 ? 1 : (DR > 0 ? ZEUS_MINB : 1))
    bfgs_warp_kernel(BfgsArgs A) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int d = A.d;
  // block-shared alpha table: alpha0 * shrink^t by repeated multiplication,
  // exactly as linesearch.py:70 updates alpha
  double* alpha_tab = sm;
  if (threadIdx.x == 0) {
    double a = A.alpha0;
    for (int t = 0; t < A.nalpha; ++t) {
      alpha_tab[t] = a;
      a *= A.shrink;
    }
  }
  __syncthreads();
  // one slice per warp (NH == 0) or one slice per CTA (NH > 0)
  double* base = sm + A.nalpha + (NH > 0 ? (size_t)0 : (size_t)wib * A.warp_doubles);
  BfgsWarp<Obj, DR, NH> W;
  W.alpha_tab = alpha_tab;
  double* v = base;
  if constexpr (DR == 0) {
    if (A.h_global) {
      W.H = A.h_global + ((size_t)blockIdx.x * (blockDim.x >> 5) + wib) * (size_t)d * A.ldh;
    } else {
      W.H = v;
      v += hsize(d, A.ldh);
    }
  } else {
    W.H = nullptr;
  }
  W.row4 = v;  // [max(d,DR)][4] = {dg, g', dx_prev, u_prev}; 16-B aligned (offsets even)
  v += 4 * (DR > d ? DR : d);
  W.x = v;
  v += d;
  W.xn = v;
  v += d;
  W.p = v;
  v += d;
  W.g = v;
  v += d;
  W.gn = v;
  v += d;
  W.T = v;
  W.xbuf[0] = W.x;
  W.xbuf[1] = W.xn;
  if constexpr (NH > 0)  // the helper warps alone cover a batch (warp 0 reduces g.p meanwhile)
    W.tix = term_idx<32 * NH>(Obj::nterms(d) > 0 ? Obj::nterms(d) : 1,
                              (int)threadIdx.x - 32);
  W.task = reinterpret_cast<HelperTask*>(sm + A.nalpha + A.warp_doubles);

  if constexpr (NH == 0) {
    const long long nwork = A.resume ? (long long)*A.in_count : A.n;
    for (;;) {
      long long s = 0;
      if (lane == 0) s = (long long)atomicAdd(A.resume ? A.in_taken : A.work, 1ull);
      s = __shfl_sync(kFull, s, 0);
      if (s >= nwork) break;
      BfgsWarp<Obj, DR, NH> w = W;  // fresh pointer set per start (run() swaps x/xn, g/gn)
      if (A.resume) {  // a start promoted by the thread-per-start kernel
        const double* rec = A.carry_in + (size_t)s * A.carry_stride;
        w.run(A, (long long)rec[0], lane, rec);
      } else {
        w.run(A, s, lane);
      }
    }
  } else if (wib == 0) {  // driving warp
    const long long nwork = A.resume ? (long long)*A.in_count : A.n;
    for (;;) {
      long long w = 0;
      if (lane == 0) w = (long long)atomicAdd(A.resume ? A.in_taken : A.work, 1ull);
      w = __shfl_sync(kFull, w, 0);
      if (w >= nwork) break;
      BfgsWarp<Obj, DR, NH> wk = W;
      if (A.resume) {
        const double* rec = A.carry_in + (size_t)w * A.carry_stride;
        wk.run(A, (long long)rec[0], lane, rec);
      } else {
        wk.run(A, w, lane);
      }
    }
    if (lane == 0) W.task->B = -1;
    __syncwarp();
    bar1(32 * (NH + 1));  // A: release the helpers
  } else {  // helper warps: evaluate term batches until told to exit
    const int tid = threadIdx.x;
    const int nt = Obj::nterms(d);
    double* TT = W.T + Obj::NACC * A.bmax * A.tstride;
    const double* atab = TT + Obj::KT * A.bmax * A.tstride;
    for (;;) {
      bar1(32 * (NH + 1));  // A
      const int B = W.task->B;
      if (B < 0) break;
      const double* x = W.xbuf[W.task->xsel];
      const int total = (B > 0 ? B : 1) * nt;
      bool oor = false;
      if (total > 0)
        term_pass<Obj, FastMath, 32 * NH>(B, nt, total, atab, d, x, W.p, W.T, TT, A.tstride,
                                          A.bmax, tid - 32, oor, &W.tix);
      if (bar1_or(32 * (NH + 1), oor)) {  // B
        if (total > 0)
          term_pass<Obj, PreciseMath, 32 * NH>(B, nt, total, atab, d, x, W.p, W.T, TT,
                                               A.tstride, A.bmax, tid - 32, oor, &W.tix);
        bar1(32 * (NH + 1));
      }
    }
  }
}

}  // namespace zeus
