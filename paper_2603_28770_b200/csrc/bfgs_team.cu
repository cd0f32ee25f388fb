// bfgs_team.cu -- multistart BFGS (bfgs.py:80-156), one CTA per start.
//
// For 32 < d <= 128 a start gets a whole CTA: thread t owns column j of the
// inverse Hessian H (bfgs.py:59-77) and keeps its rows in REGISTERS
// (h[R]; for d > 64 two threads split a column's rows, S = 2), so the fused
// per-iteration pass (lazy rank-2 update + u = H dg + w = H g') runs from the
// register file with shared-memory broadcasts of the row values -- no H
// traffic at all.  Everything else is spread over the CTA:
//   * speculative line search: the B x nterms objective terms of a batch of
//     Armijo trials are distributed over all NT threads; each trial's terms
//     are folded by one warp (tree) or, for d <= 16, by one thread in the
//     reference's sequential order;
//   * gradient (lane-mapped forward-mode duals) by the column threads;
//   * the 8 scalars of an iteration in one CTA reduction (warp butterflies +
//     a fixed-order cross-warp sum, identical on every thread).
// One start per CTA at a time; CTAs are persistent and pop starts from the
// device work counter.  The iteration algebra is the one of bfgs.cu.
#include "bfgs_common.cuh"

namespace zeus {

#ifdef ZEUS_PHASE_TIMING
__device__ unsigned long long zeus_team_phase_cycles[8];
#define TPHASE(i)                                                                      \
  do {                                                                                 \
    const long long _n = clock64();                                                    \
    if (tid == 0) atomicAdd(&zeus_team_phase_cycles[i], (unsigned long long)(_n - _tp)); \
    _tp = _n;                                                                          \
  } while (0)
#define TPHASE_T0() long long _tp = clock64()
#else
#define TPHASE(i)
#define TPHASE_T0()
#endif

namespace {

// CTA-wide sum of 8 values, identical on every thread (fixed order).  When
// only warp 0 holds data (`w0only`: all column owners are in warp 0) the
// other warps skip the butterfly and the cross-warp adds.
template <int NW>
__device__ __forceinline__ void cta_sum8(double v[8], double* red, int lane, int warp,
                                         bool w0only) {
  if (!w0only || warp == 0) {
    warp_sum8(v);
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) red[warp * 8 + q] = v[q];
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    double s = red[q];
    if (!w0only) {
#pragma unroll
      for (int w = 1; w < NW; ++w) s += red[w * 8 + q];
    }
    v[q] = s;
  }
  __syncthreads();
}

template <int NW>
__device__ __forceinline__ double cta_sum1(double v, double* red, int lane, int warp,
                                           bool w0only) {
  if (!w0only || warp == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (lane == 0) red[warp] = v;
  }
  __syncthreads();
  double s = red[0];
  if (!w0only) {
#pragma unroll
    for (int w = 1; w < NW; ++w) s += red[w];
  }
  __syncthreads();
  return s;
}

}  // namespace

// Shared-memory layout of one CTA (one start), in doubles.
struct TeamSmem {
  double *alpha_tab, *x, *xn, *p, *g, *gn, *row4, *T, *TT, *atab, *fval, *accv, *red;
  unsigned* pass_mask;
  long long* start;
};

template <class Obj, int NW, int R, int S>
struct BfgsTeam {
  static constexpr int NT = NW * 32;
  TeamSmem sm;

  __device__ __forceinline__ double alpha_at(const BfgsArgs& A, int t) const {
    if (t < A.nalpha) return sm.alpha_tab[t];
    double a = sm.alpha_tab[A.nalpha - 1];
    for (int k = A.nalpha - 1; k < t; ++k) a *= A.shrink;
    return a;
  }

  // Fold trial b's terms; returns f on the folding thread (thread b for the
  // sequential fold, lane 0 of warp b % NW for the tree fold).  Results go
  // to fval[b], accv[b][a].
  __device__ __forceinline__ void fold(const BfgsArgs& A, int nb, int d, int tid, int lane,
                                       int warp) {
    const int nt = Obj::nterms(d);
    if (d <= 16) {  // reference order: bit-identical f
      if (tid < nb) {
        double acc[Obj::NACC];
#pragma unroll
        for (int a = 0; a < Obj::NACC; ++a) {
          const double* row = sm.T + (a * A.bmax + tid) * A.tstride;
          double s = Obj::init(a, d);
          for (int j = 0; j < nt; ++j) s = s + row[j];
          acc[a] = s;
          sm.accv[tid * 2 + a] = s;
        }
        bool err = false;
        sm.fval[tid] = Obj::finish(acc, d, err);
      }
    } else {  // warp tree: lane sums j = lane, lane+32, ... then butterfly
      for (int b = warp; b < nb; b += NW) {
        double acc[Obj::NACC];
#pragma unroll
        for (int a = 0; a < Obj::NACC; ++a) {
          const double* row = sm.T + (a * A.bmax + b) * A.tstride;
          double s = 0.0;
          for (int j = lane; j < nt; j += 32) s += row[j];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
          acc[a] = Obj::init(a, d) + s;
        }
        if (lane == 0) {
#pragma unroll
          for (int a = 0; a < Obj::NACC; ++a) sm.accv[b * 2 + a] = acc[a];
          bool err = false;
          sm.fval[b] = Obj::finish(acc, d, err);
        }
      }
    }
  }

  // Fresh start s (rec == nullptr) or resume from a carry record written by
  // the warp kernel at iteration k1 (rec != nullptr; s is read from it).
  __device__ void run(const BfgsArgs& A, long long s, int tid, const double* rec) {
    TPHASE_T0();
    const int d = A.d;
    const int lane = tid & 31, warp = tid >> 5;
    // column role
    int col, split;
    if constexpr (S == 1) {
      col = tid;
      split = 0;
    } else {
      col = warp * 16 + (lane & 15);
      split = lane >> 4;
    }
    const bool has_col = col < d;
    const bool primary = has_col && split == 0;
    const int row0 = split * R;
    const bool w0only = S == 1 && d <= 32;

    double h[R];
    double aj = 0.0, bj = 0.0;  // pending rank-2 coefficients of my column
    for (int i = d + tid; i < R * S; i += NT) {  // zero padding rows of row4
      sm.row4[4 * i] = sm.row4[4 * i + 1] = sm.row4[4 * i + 2] = sm.row4[4 * i + 3] = 0.0;
    }
    double *x = sm.x, *xn = sm.xn, *g = sm.g, *gn = sm.gn;
    const int nt = Obj::nterms(d);
    double acc[Obj::NACC];
    double f0;
    int k = 0, status = ZEUS_DIVERGED, ls_trials = 0, grads = 0, prev_trials = 1;
    double gnorm = __longlong_as_double(0x7ff0000000000000LL);
    double ddir = 0.0;
    bool pending = false;

    if (rec) {  // ---- resume (carry layout in bfgs_common.cuh)
      k = (int)rec[1];
      ls_trials = (int)rec[2];
      grads = (int)rec[3];
      prev_trials = (int)rec[4];
      f0 = rec[5];
#pragma unroll
      for (int a = 0; a < Obj::NACC; ++a) acc[a] = rec[6 + a];
      gnorm = sqrt(rec[8]);  // the record carries |g|^2
      ddir = rec[9];
      if (primary) {
        x[col] = rec[kCarryHead + col];
        g[col] = rec[kCarryHead + d + col];
        sm.p[col] = rec[kCarryHead + 2 * d + col];
      }
      const double* Hr = rec + kCarryHead + 3 * d;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = row0 + r;
        h[r] = (has_col && i < d) ? Hr[(int64_t)i * d + col] : 0.0;
      }
      __syncthreads();
      goto iterate;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) h[r] = (row0 + r == col) ? 1.0 : 0.0;
    if (primary) x[col] = A.x0[(int64_t)col * A.ldx + s];
    __syncthreads();

    // f(x0)
    {
      bool oor = false;
      if (nt > 0) term_pass<Obj, FastMath, NT>(0, nt, nt, nullptr, d, x, sm.p, sm.T, sm.TT,
                                                A.tstride, A.bmax, tid, oor);
      if (__syncthreads_or(oor))
        term_pass<Obj, PreciseMath, NT>(0, nt, nt, nullptr, d, x, sm.p, sm.T, sm.TT,
                                        A.tstride, A.bmax, tid, oor);
      fold(A, 1, d, tid, lane, warp);
      __syncthreads();
      f0 = sm.fval[0];
#pragma unroll
      for (int a = 0; a < Obj::NACC; ++a) acc[a] = sm.accv[a];
    }

    if (A.stop_flag && __syncthreads_or(tid == 0 && *(volatile int*)A.stop_flag)) {
      status = ZEUS_STOPPED;
      goto done;
    }
    {  // first gradient; p = -g (H0 = I)
      ++grads;
      bool err = false;
      double part = 0.0;
      if (primary) {
        const double gj = Obj::grad_from_tan(TanRow{sm.TT, A.bmax, A.tstride, 0}, col, d, acc, err);
        g[col] = gj;
        sm.p[col] = -gj;
        part = gj * gj;
      }
      if (__syncthreads_or(err)) {
        status = ZEUS_DOMAIN_ERROR;
        goto done;
      }
      const double gg = cta_sum1<NW>(part, sm.red, lane, warp, w0only);
      gnorm = sqrt(gg);
      ddir = -gg;
    }

  iterate:
#ifdef ZEUS_PHASE_TIMING
    _tp = clock64();
#endif
    for (;;) {
      if (gnorm < A.theta) {
        status = ZEUS_CONVERGED;
        break;
      }
      if (k >= A.cap) {
        status = ZEUS_DIVERGED;
        break;
      }
      // ---- speculative batched Armijo search (linesearch.py:60-71)
      int t_acc, src_row = 0;
      double f_new, acc_new[Obj::NACC], alpha;
      {
        int t0 = 0;
        int B = min(max(prev_trials, max(1, NT / max(nt, 1))), A.bmax);
        for (;;) {
          B = min(B, A.iter_ls + 1 - t0);
          if (tid < B) sm.atab[tid] = alpha_at(A, t0 + tid);
          if (tid == 0) *sm.pass_mask = 0u;
          __syncthreads();
          const int total = B * nt;
          bool oor = false;
          if (total > 0)
            term_pass<Obj, FastMath, NT>(B, nt, total, sm.atab, d, x, sm.p, sm.T, sm.TT,
                                         A.tstride, A.bmax, tid, oor);
          if (__syncthreads_or(oor))
            term_pass<Obj, PreciseMath, NT>(B, nt, total, sm.atab, d, x, sm.p, sm.T, sm.TT,
                                            A.tstride, A.bmax, tid, oor);
          fold(A, B, d, tid, lane, warp);
          __syncthreads();
          if (tid < B) {
            const double fb = sm.fval[tid];
            if (fb <= f0 + A.c1 * sm.atab[tid] * ddir) atomicOr(sm.pass_mask, 1u << tid);
          }
          __syncthreads();
          const unsigned m = *sm.pass_mask;
          int src = -1;
          if (m) src = __ffs(m) - 1;
          else if (t0 + B > A.iter_ls) src = B - 1;  // fell through: last trial
          if (src >= 0) {
            t_acc = t0 + src;
            src_row = src;
            f_new = sm.fval[src];
#pragma unroll
            for (int a = 0; a < Obj::NACC; ++a) acc_new[a] = sm.accv[src * 2 + a];
            alpha = sm.atab[src];
            break;
          }
          t0 += B;
          B = min(2 * B, A.bmax);
          __syncthreads();  // atab / pass_mask reuse
        }
      }
      TPHASE(0);
      ls_trials += t_acc + 1;
      prev_trials = t_acc + 1;
      // ---- x_new and the gradient there, assembled from the accepted trial's
      // term tangents (computed in the term pass); DomainError leaves x, k
      ++grads;
      {
        bool err = false;
        if (primary) {
          xn[col] = x[col] + alpha * sm.p[col];
          const double gj =
              Obj::grad_from_tan(TanRow{sm.TT, A.bmax, A.tstride, src_row}, col, d, acc_new, err);
          gn[col] = gj;
          sm.row4[4 * col + 0] = gj - g[col];
          sm.row4[4 * col + 1] = gj;
        }
        if (__syncthreads_or(err)) {
          status = ZEUS_DOMAIN_ERROR;
          break;
        }
      }

      TPHASE(1);
      // ---- fused register pass over my column: lazy update, u = H dg, w = H g'
      double u = 0.0, w = 0.0;
      {
        // straight-line over R rows: row4 is zero-padded beyond d, so rows past
        // d contribute nothing and need no guard; the lazy update is a select
        double u0 = 0.0, u1 = 0.0, w0 = 0.0, w1 = 0.0;
        const double* rp = sm.row4 + 4 * row0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double2 ra = *reinterpret_cast<const double2*>(rp + 4 * r);
          const double2 rb = *reinterpret_cast<const double2*>(rp + 4 * r + 2);
          const double upd = fma(rb.x, aj, fma(rb.y, bj, h[r]));
          const double hv = pending ? upd : h[r];
          h[r] = hv;
          if (r & 1) {
            u1 = fma(hv, ra.x, u1);
            w1 = fma(hv, ra.y, w1);
          } else {
            u0 = fma(hv, ra.x, u0);
            w0 = fma(hv, ra.y, w0);
          }
        }
        u = u0 + u1;
        w = w0 + w1;
      }
      if constexpr (S == 2) {
        u += __shfl_xor_sync(kFull, u, 16);
        w += __shfl_xor_sync(kFull, w, 16);
      }

      TPHASE(2);
      // ---- one CTA reduction of the 8 iteration scalars
      double part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      double dxj = 0.0;
      if (has_col) dxj = xn[col] - x[col];
      if (primary) {
        const double dgj = sm.row4[4 * col], gj = gn[col];
        part[0] = gj * gj;
        part[1] = dxj * dgj;
        part[2] = dxj * dxj;
        part[3] = dgj * dgj;
        part[4] = dgj * u;
        part[5] = u * gj;
        part[6] = dxj * gj;
        part[7] = w * gj;
      }
      cta_sum8<NW>(part, sm.red, lane, warp, w0only);  // ends with __syncthreads: row4 consumed
      const double curv = part[1];
      const double ndx = sqrt(part[2]), ndg = sqrt(part[3]);
      pending = !(curv <= kCurvatureFloor * ndx * ndg);  // bfgs.py:69-71
      double pd = 0.0;
      {
        const double rho = pending ? 1.0 / curv : 0.0;
        const double cc = pending ? fma(rho * rho, part[4], rho) : 0.0;
        const double ug = part[5], xg = part[6];
        if (has_col && pending) {
          aj = fma(cc, dxj, -rho * u);
          bj = -rho * dxj;
        }
        if (primary) {
          double pj = -w;
          if (pending) {
            pj = -(w + fma(dxj, fma(cc, xg, -rho * ug), -rho * xg * u));
            sm.row4[4 * col + 2] = dxj;
            sm.row4[4 * col + 3] = u;
          }
          sm.p[col] = pj;
          pd = gn[col] * pj;
        }
      }
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
      gnorm = sqrt(part[0]);
      TPHASE(3);
      ddir = cta_sum1<NW>(pd, sm.red, lane, warp, w0only);  // syncs: p / row4 visible
      TPHASE(4);
      ++k;
      if (A.stop_flag && __syncthreads_or(tid == 0 && *(volatile int*)A.stop_flag)) {
        status = ZEUS_STOPPED;
        break;
      }
    }

  done:
    const zeus_bfgs_out& o = A.out;
    if (primary) o.x_final[(int64_t)col * o.ld_out + s] = x[col];
    if (tid == 0) {
      o.f_final[s] = f0;
      o.grad_norm[s] = gnorm;
      o.iterations[s] = k;
      o.status[s] = (uint8_t)status;
      if (o.ls_trials) o.ls_trials[s] = ls_trials;
      if (o.grad_evals) o.grad_evals[s] = grads;
      if (status == ZEUS_CONVERGED && A.stop_counter) {
        const unsigned long long old = atomicAdd_system(A.stop_counter, 1ull);
        if ((long long)old + 1 == A.required_c) atomicExch_system(A.stop_flag, 1);
      }
    }
    __syncthreads();
  }
};

template <class Obj, int NW, int R, int S>
__global__ void __launch_bounds__(NW * 32, 1) bfgs_team_kernel(BfgsArgs A) {
  extern __shared__ double smem[];
  const int tid = threadIdx.x;
  const int d = A.d;
  TeamSmem sm;
  double* v = smem;
  sm.alpha_tab = v;
  v += A.nalpha;
  sm.row4 = v;  // 16-B aligned: nalpha is even; R*S rows (zero padding past d)
  v += 4 * R * S;
  sm.x = v;
  v += d;
  sm.xn = v;
  v += d;
  sm.p = v;
  v += d;
  sm.g = v;
  v += d;
  sm.gn = v;
  v += d;
  sm.T = v;
  v += Obj::NACC * A.bmax * A.tstride;
  sm.TT = v;
  v += Obj::KT * A.bmax * A.tstride;
  sm.atab = v;
  v += 32;
  sm.fval = v;
  v += 32;
  sm.accv = v;
  v += 64;
  sm.red = v;
  v += 8 * NW;
  sm.pass_mask = reinterpret_cast<unsigned*>(v);
  sm.start = reinterpret_cast<long long*>(v + 1);
  if (tid == 0) {
    double a = A.alpha0;
    for (int t = 0; t < A.nalpha; ++t) {
      sm.alpha_tab[t] = a;
      a *= A.shrink;
    }
  }
  BfgsTeam<Obj, NW, R, S> T{sm};
  const long long nwork = A.resume ? (long long)*A.in_count : A.n;
  for (;;) {
    if (tid == 0)
      *sm.start = (long long)atomicAdd(A.resume ? A.in_taken : A.work, 1ull);
    __syncthreads();
    const long long w = *sm.start;
    __syncthreads();
    if (w >= nwork) break;
    if (A.resume) {
      const double* rec = A.carry_in + (size_t)w * A.carry_stride;
      T.run(A, (long long)rec[0], tid, rec);
    } else {
      T.run(A, w, tid, nullptr);
    }
  }
}

namespace {

constexpr int kTeamTermCap = 1024;

size_t team_smem_bytes(int d, int rows, int nacc, int kt, int nw, int bmax, int tstride,
                       int nalpha) {
  return sizeof(double) * ((size_t)nalpha + 4 * (size_t)rows + 5 * (size_t)d +
                           (size_t)(nacc + kt) * bmax * tstride + 32 + 32 + 64 + 8 * nw + 2);
}

template <class Obj, int NW, int R, int S>
int launch_shape(BfgsArgs A, cudaStream_t s) {
  const int nt = std::max(1, Obj::nterms(A.d));
  A.tstride = nt | 1;
  A.bmax = std::max(1, std::min(32, kTeamTermCap / nt));
  A.nalpha = kAlphaTable;
  const size_t smem =
      team_smem_bytes(A.d, R * S, Obj::NACC, Obj::KT, NW, A.bmax, A.tstride, A.nalpha);
  auto kern = bfgs_team_kernel<Obj, NW, R, S>;
  int rc = check_cuda(
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
      "cudaFuncSetAttribute(team)");
  if (rc) return rc;
  int per_sm = 0;
  rc = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem),
                  "occupancy(team)");
  if (rc) return rc;
  const int sms = current_sm_count();
  if (per_sm < 1 || sms < 1) return set_error(ZEUS_ERR_UNSUPPORTED, "bfgs team: does not fit");
  int64_t grid = (int64_t)per_sm * sms;
  if (!A.resume && grid > A.n) grid = A.n;
  kern<<<(unsigned)grid, NW * 32, smem, s>>>(A);
  return check_launch("bfgs_team_kernel");
}

struct TeamLaunch {
  template <class Obj>
  static int run(BfgsArgs A, cudaStream_t s) {
    const int d = A.d;
    if (A.resume) {  // stragglers of the warp kernel (d <= 16): 8 warps per start
      if (d <= 16) return launch_shape<Obj, 8, 16, 1>(A, s);
      return set_error(ZEUS_ERR_UNSUPPORTED, "team resume: d=%d > 16", d);
    }
    if constexpr (Obj::kId == ZEUS_OBJ_GOLDSTEIN_PRICE) {
      return set_error(ZEUS_ERR_UNSUPPORTED, "team: goldstein_price is 2-D");
    } else {
      if (d <= 48) return launch_shape<Obj, 2, 48, 1>(A, s);
      if (d <= 50) return launch_shape<Obj, 2, 50, 1>(A, s);
      if (d <= 64) return launch_shape<Obj, 2, 64, 1>(A, s);
      if (d <= 100) return launch_shape<Obj, 7, 50, 2>(A, s);
      if (d <= 128) return launch_shape<Obj, 8, 64, 2>(A, s);
      return set_error(ZEUS_ERR_UNSUPPORTED, "team: d=%d > 128", d);
    }
  }
};

}  // namespace

#ifdef ZEUS_PHASE_TIMING
int team_phase_cycles(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, zeus_team_phase_cycles, 8 * sizeof(unsigned long long)) != cudaSuccess)
    return -2;
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(zeus_team_phase_cycles, z, sizeof(z));
  }
  return 0;
}
#endif

bool bfgs_team_covers(int obj, int d) {
  return obj != ZEUS_OBJ_GOLDSTEIN_PRICE && d > 32 && d <= 128;
}

int launch_bfgs_team(int obj, BfgsArgs A, cudaStream_t s) {
  return dispatch_objective<TeamLaunch>(obj, A, s);
}

}  // namespace zeus
