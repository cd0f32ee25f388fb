// bfgs_wide.cu -- multistart BFGS (bfgs.py:80-156) for 32 < d <= 64, one WARP
// per start, built for throughput (the 1M-start 50-D targets).
//
// Why a second kernel family next to the CTA-per-start team kernel
// (bfgs_team.cu): at d = 50 a team start costs ~7,300 cycles of wall time per
// iteration, 55% of it in the CTA-synchronised line search and 24% in CTA
// reductions, and only 4 starts fit an SM (scripts/phase_probe.py).  Here
// everything is warp-synchronous (shuffles, no __syncthreads) and a start's
// state is spread over the 32 lanes of one warp, so ~8-10 starts share an SM
// and their latency-bound phases overlap each other's FP64 work.
//
// Ownership: lane l owns coordinates c0 = l and c1 = l + 32 (if < d): their
// x, p, g entries live in REGISTERS, and so do the first RR rows of the two
// inverse-Hessian columns H[:, c0], H[:, c1]; rows RR..d-1 of those columns
// live in the warp's shared-memory slice (conflict-free: lanes read
// consecutive columns).  The per-row broadcast values of the fused H pass
// {dg_i, g'_i, dx_i, u_i} are the only other shared-memory traffic.
//
// Per iteration (reference order, bfgs.py:108-156):
//  1. speculative batched Armijo search (linesearch.py:60-71): trials
//     alpha0 shrink^t, t = t0..t0+B-1, evaluated together; every lane
//     evaluates its own objective terms of every trial in registers
//     (x + alpha p with the reference's two roundings), one transpose-reduce
//     (warp_sum8) folds the B trials, and the FIRST passing trial is taken --
//     alpha, trial count and f of the sequential search;
//  2. gradient at x_new from lane-local forward-mode term tangents
//     (autodiff.py:243-266 restricted to the terms that contain x_i; the one
//     neighbour tangent Rosenbrock needs arrives by shuffle);
//  3. one fused pass over H: the lazy rank-2 update of the previous iteration
//     (H += dx a^T + u b^T, the O(d^2) form of bfgs.py:72-77), u = H dg and
//     w = H g' in the same sweep;
//  4. one 8-value warp reduction: |g'|^2, dx.dg, |dx|^2, |dg|^2, dg.u, u.g',
//     dx.g', w.g' -> curvature guard (bfgs.py:69-71), rho, the next direction
//     p' = -H' g' = -(w - rho dx (u.g') - rho u (dx.g') + c dx (dx.g'));
//  5. g'.p' (the next line search's ddir) by one butterfly.
// Objective folds for d > 16 are warp trees (as in the team kernel): f agrees
// with the reference's sequential fold to ~1 ulp, inside the stated tolerance.
#include "bfgs_common.cuh"

namespace zeus {

namespace {

constexpr int kWideWarps = 2;    // warps (starts) per block
constexpr int kWideMaxB = 8;     // trials per speculative batch (registers)
constexpr int kWideLd = 64;      // row stride of the shared-memory H rows
#ifdef ZEUS_WIDE_CH
constexpr int kCH = ZEUS_WIDE_CH;  // trials per chunk of the batched (SEQ=0) search
#else
constexpr int kCH = 4;
#endif
#ifndef ZEUS_WIDE_ACKLEY
#define ZEUS_WIDE_ACKLEY 1
#endif
#ifndef ZEUS_WIDE_SEQ
#define ZEUS_WIDE_SEQ 1
#endif
#ifndef ZEUS_WIDE_UFROMP
#define ZEUS_WIDE_UFROMP 1
#endif
#if ZEUS_WIDE_UFROMP
#define UACC(x)
#else
#define UACC(x) x
#endif

// Term j's coordinate accessor: x(j) -> xj, x(j + 1) -> xj1 (Rosenbrock's
// neighbour); objectives only ever ask for these two.
struct LX {
  int j;
  double xj, xj1;
  __device__ __forceinline__ double operator()(int k) const { return k == j ? xj : xj1; }
};
// Term-tangent accessor for coordinate i: tan(i, k) -> own[k] (term i),
// tan(i - 1, 1) -> prev (term i-1's tangent w.r.t. x_i, from the neighbour).
struct LT {
  int i;
  double own0, own1, prev;
  __device__ __forceinline__ double operator()(int j, int k) const {
    return j == i ? (k == 0 ? own0 : own1) : prev;
  }
};

template <class Obj>
struct WideTraits {
  static constexpr bool kNeighbour = Obj::kId == ZEUS_OBJ_ROSENBROCK;
};

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(kFull, v, src); }

}  // namespace

// Per-objective shape, tuned on B200 (scripts/wide_variants.sh +
// scripts/phase_probe.py at d = 50): rows of H kept in registers (RR),
// resident starts per SM (2 * MINB warps) and trials per line-search chunk
// (CH: Ackley needs 1.6 trials per iteration, Rosenbrock 2.7, Rastrigin 6.2;
// SM-cycles per start-iteration for CH = 1 / 2 / 3 / 4: Rosenbrock 820 / 770
// / 781 / 793, Rastrigin 1781 / 1729 / 1746 / 1915, Ackley 1596 / 1854 (team
// kernel: 2884)).
template <class Obj>
struct WideShape {
  static constexpr int RR = Obj::kId == ZEUS_OBJ_ROSENBROCK ? 32 : 16;
  static constexpr int MINB = Obj::kId == ZEUS_OBJ_ROSENBROCK ? 4 : 5;
  static constexpr int CH = Obj::kId == ZEUS_OBJ_ACKLEY ? 1 : 2;
};

template <class Obj, int RR>
struct WideStart {
  static constexpr int NA = Obj::NACC;
  double* Hs;          // [d - RR][kWideLd] rows RR.. of every column
  double* rowv;        // [64][4] {dg, g', dx_prev, u_prev}
  const double* atab;  // block alpha table

  __device__ __forceinline__ double alpha_at(const BfgsArgs& A, int t) const {
    if (t < A.nalpha) return atab[t];
    double a = atab[A.nalpha - 1];
    for (int k = A.nalpha - 1; k < t; ++k) a *= A.shrink;
    return a;
  }

  // Values of this lane's terms (c0, c1) at CH trial points x + alpha_c p,
  // s[c][a] = (0 + t(c0)) + t(c1) (the team kernel's lane order).  Branch-free:
  // all 2 CH term evaluations are independent chains the scheduler can
  // interleave (a missing term is evaluated at 0 and masked out).
  template <class M, int CH>
  __device__ __forceinline__ void lane_terms(int d, int nt, int l, const double al[CH], double x0,
                                             double x1, double p0, double p1, double nx0,
                                             double nx1, double np0, double np1,
                                             double s[CH][NA], bool& oor) const {
    const bool v0 = l < nt, v1 = l + 32 < nt;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const double xt0 = x0 + al[c] * p0, xt1 = x1 + al[c] * p1;
      double xn0 = 0.0, xn1 = 0.0;
      if constexpr (WideTraits<Obj>::kNeighbour) {
        xn0 = nx0 + al[c] * np0;
        xn1 = nx1 + al[c] * np1;
      }
      double t0[NA], t1[NA];
      Obj::template term<M>(LX{l, xt0, xn0}, l, d, t0, oor);
      Obj::template term<M>(LX{l + 32, xt1, xn1}, l + 32, d, t1, oor);
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        double v = v0 ? 0.0 + t0[a] : 0.0;
        s[c][a] = v1 ? v + t1[a] : v;
      }
    }
  }

  // Cold path: the chunk with CUDA libm trig (some argument beyond kTrigMax),
  // kept out of line so the hot loop stays small in the instruction cache.
  template <int CH>
  __device__ __noinline__ void lane_terms_precise(int d, int nt, int l, const double* al,
                                                  double x0, double x1, double p0, double p1,
                                                  double nx0, double nx1, double np0,
                                                  double np1, double* out) const {
    double a4[CH], sc[CH][NA];
    for (int c = 0; c < CH; ++c) a4[c] = al[c];
    bool oor = false;
    lane_terms<PreciseMath, CH>(d, nt, l, a4, x0, x1, p0, p1, nx0, nx1, np0, np1, sc, oor);
    for (int c = 0; c < CH; ++c)
      for (int a = 0; a < NA; ++a) out[c * NA + a] = sc[c][a];
  }

  // Values AND term tangents of this lane's terms at the point (x0, x1)
  // (neighbour coordinates nx0, nx1); branch-free like lane_terms.
  template <class M>
  __device__ __forceinline__ void lane_tan(int d, int nt, int l, double x0, double x1,
                                           double nx0, double nx1, double s[NA], double tA[2],
                                           double tB[2], bool& oor) const {
    const bool v0 = l < nt, v1 = l + 32 < nt;
    double t0[NA], t1[NA], n0[Obj::KT], n1[Obj::KT];
    Obj::template term_tan<M>(LX{l, x0, nx0}, l, d, t0, n0, oor);
    Obj::template term_tan<M>(LX{l + 32, x1, nx1}, l + 32, d, t1, n1, oor);
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      double v = v0 ? 0.0 + t0[a] : 0.0;
      s[a] = v1 ? v + t1[a] : v;
    }
    tA[0] = v0 ? n0[0] : 0.0;
    tA[1] = v0 && Obj::KT > 1 ? n0[Obj::KT - 1] : 0.0;
    tB[0] = v1 ? n1[0] : 0.0;
    tB[1] = v1 && Obj::KT > 1 ? n1[Obj::KT - 1] : 0.0;
  }

  // Gradient components of c0, c1 from the lane's term tangents (+ the
  // neighbour's tangent of term c-1 w.r.t. x_c for Rosenbrock).
  __device__ __forceinline__ void lane_grad(int d, int l, const double tA[2], const double tB[2],
                                            const double acc[NA], double& g0, double& g1,
                                            bool& err) const {
    double prevA = 0.0, prevB = 0.0;
    if constexpr (WideTraits<Obj>::kNeighbour) {
      const int src = (l + 31) & 31;
      const double s0 = shfl(tA[1], src), s1 = shfl(tB[1], src);
      prevA = s0;                 // term l-1 (lane l-1's c0 term), l >= 1
      prevB = l >= 1 ? s1 : s0;   // term l+31: lane l-1's c1 term, or lane 31's c0 term
    }
    g0 = Obj::grad_from_tan(LT{l, tA[0], tA[1], prevA}, l, d, acc, err);
    g1 = 0.0;
    if (l + 32 < d) g1 = Obj::grad_from_tan(LT{l + 32, tB[0], tB[1], prevB}, l + 32, d, acc, err);
  }

  // f at a point from the lane sums s[a]: warp tree, then Obj::init + sum.
  __device__ __forceinline__ double fold1(int d, const double s[NA], double acc[NA],
                                          bool& err) const {
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = Obj::init(a, d) + warp_sum(s[a]);
    return Obj::finish(acc, d, err);
  }

  __device__ void run(const BfgsArgs& A, long long s, int l) {
    const int d = A.d;
    const int nt = Obj::nterms(d);
    const bool own1 = l + 32 < d;
    double h0[RR], h1[RR];
    double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;  // pending rank-2 coefficients
    double x0, x1 = 0.0, p0, p1 = 0.0, g0, g1 = 0.0;
    double acc[NA];
    double f0;
    int k = 0, status = ZEUS_DIVERGED, ls_trials = 0, grads = 0, prev_trials = 1;
    double gnorm = __longlong_as_double(0x7ff0000000000000LL);
    double ddir = 0.0;
    bool pending = false;

    // ---- H = I, x = x0, rowv = 0
#pragma unroll
    for (int i = 0; i < RR; ++i) {
      h0[i] = i == l ? 1.0 : 0.0;
      h1[i] = i == l + 32 ? 1.0 : 0.0;
    }
    for (int i = RR; i < d; ++i) {
      Hs[(i - RR) * kWideLd + l] = i == l ? 1.0 : 0.0;
      Hs[(i - RR) * kWideLd + l + 32] = i == l + 32 ? 1.0 : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      rowv[4 * l + q] = 0.0;
      rowv[4 * (l + 32) + q] = 0.0;
    }
    x0 = A.x0[(int64_t)l * A.ldx + s];
    if (own1) x1 = A.x0[(int64_t)(l + 32) * A.ldx + s];
    __syncwarp();

    // neighbour coordinates of the current point (Rosenbrock term j needs x_{j+1})
    double nx0 = 0.0, nx1 = 0.0;
    auto neighbours = [&](double v0, double v1, double& n0, double& n1) {
      if constexpr (WideTraits<Obj>::kNeighbour) {
        const int src = (l + 1) & 31;
        const double t0 = shfl(v0, src), t1 = shfl(v1, src);
        n0 = l < 31 ? t0 : t1;  // x_{l+1}; lane 31 -> x_32 = lane 0's c1
        n1 = t1;                // x_{l+33}
      }
    };

    // ---- f(x0) and the first gradient, from one term pass with tangents
    {
      neighbours(x0, x1, nx0, nx1);
      double sv[NA], tA[2], tB[2];
      bool oor = false, err = false;
      lane_tan<FastMath>(d, nt, l, x0, x1, nx0, nx1, sv, tA, tB, oor);
      if (__any_sync(kFull, oor)) lane_tan<PreciseMath>(d, nt, l, x0, x1, nx0, nx1, sv, tA, tB, oor);
      bool ferr = false;
      f0 = fold1(d, sv, acc, ferr);
      if (A.stop_flag && *(volatile int*)A.stop_flag) {
        status = ZEUS_STOPPED;
        goto done;
      }
      ++grads;
      lane_grad(d, l, tA, tB, acc, g0, g1, err);
      if (__any_sync(kFull, err)) {
        status = ZEUS_DOMAIN_ERROR;
        goto done;
      }
      p0 = -g0;  // H0 = I: -(I @ g) is exact
      p1 = -g1;
      const double gg = warp_sum(fma(g1, g1, g0 * g0));
      gnorm = sqrt(gg);
      ddir = -gg;
    }

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
      double np0 = 0.0, np1 = 0.0;
      neighbours(x0, x1, nx0, nx1);
      neighbours(p0, p1, np0, np1);
      double alpha = 0.0, f_new = 0.0, acc_new[NA];
      int t_acc = -1;
#if ZEUS_WIDE_SEQ
      {
#ifdef ZEUS_WIDE_CH
        constexpr int CHK = ZEUS_WIDE_CH;
#else
        constexpr int CHK = WideShape<Obj>::CH;
#endif
        // chunks of CHK trials t0 .. t0 + CHK - 1 evaluated together, in order,
        // until one passes: one copy of the chunk code (instruction cache) and
        // no trial past the accepted chunk is evaluated
        static_assert(CHK * NA <= 8, "one warp_sum8 per chunk");
        for (int t0 = 0;; t0 += CHK) {
          double al[CHK], sc[CHK][NA];
#pragma unroll
          for (int c = 0; c < CHK; ++c) al[c] = alpha_at(A, t0 + c);
          bool oor = false;
          lane_terms<FastMath, CHK>(d, nt, l, al, x0, x1, p0, p1, nx0, nx1, np0, np1, sc, oor);
          if (__any_sync(kFull, oor))  // some |2 pi x| > kTrigMax: CUDA libm, out of line
            lane_terms_precise<CHK>(d, nt, l, al, x0, x1, p0, p1, nx0, nx1, np0, np1, &sc[0][0]);
          double v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = q < CHK * NA ? sc[q % CHK][q / CHK] : 0.0;
          warp_sum8(v);
          unsigned pm = 0u;
          double fb[CHK];
#pragma unroll
          for (int c = 0; c < CHK; ++c) {
            double ab[NA];
#pragma unroll
            for (int a = 0; a < NA; ++a) ab[a] = Obj::init(a, d) + v[a * CHK + c];
            const bool valid = t0 + c <= A.iter_ls;
            bool ferr = false;
            if constexpr (NA > 1) {  // Ackley: exp / sqrt only for trials that exist
              fb[c] = 0.0;
              if (valid) fb[c] = Obj::finish(ab, d, ferr);
            } else {
              fb[c] = Obj::finish(ab, d, ferr);
            }
            // NaN fails; the trial at t = iter_ls is taken when nothing passed
            const bool pass = fb[c] <= f0 + A.c1 * al[c] * ddir || t0 + c == A.iter_ls;
            pm |= (valid && pass) ? (1u << c) : 0u;
          }
          if (pm) {
            const int src = __ffs(pm) - 1;
#pragma unroll
            for (int c = 0; c < CHK; ++c) {
              if (c == src) {
                f_new = fb[c];
                alpha = al[c];
#pragma unroll
                for (int a = 0; a < NA; ++a) acc_new[a] = Obj::init(a, d) + v[a * CHK + c];
              }
            }
            t_acc = t0 + src;
            break;
          }
        }
      }
#else
      {
        int t0 = 0;
        int B = min(max(prev_trials, 1), kWideMaxB);
        for (;;) {
          B = min(B, A.iter_ls + 1 - t0);
          double al[8];  // the batch's step lengths, alpha0 shrink^(t0 + b)
#pragma unroll
          for (int b = 0; b < 8; ++b) al[b] = alpha_at(A, t0 + b);
          double v[NA][8];
#pragma unroll
          for (int a = 0; a < NA; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) v[a][b] = 0.0;
          // trials in chunks of CH evaluated together (the last chunk may
          // evaluate trials past B; they are never selected)
#pragma unroll
          for (int c0 = 0; c0 < 8; c0 += kCH) {
            if (c0 < B) {
              double sc[kCH][NA];
              bool oor = false;
              lane_terms<FastMath, kCH>(d, nt, l, al + c0, x0, x1, p0, p1, nx0, nx1, np0, np1,
                                        sc, oor);
              if (__any_sync(kFull, oor))  // some |2 pi x| > kTrigMax: CUDA libm, out of line
                lane_terms_precise<kCH>(d, nt, l, al + c0, x0, x1, p0, p1, nx0, nx1, np0, np1, &sc[0][0]);
#pragma unroll
              for (int c = 0; c < kCH; ++c)
#pragma unroll
                for (int a = 0; a < NA; ++a) v[a][c0 + c] = sc[c][a];
            }
          }
#pragma unroll
          for (int a = 0; a < NA; ++a) warp_sum8(v[a]);
          // Armijo test of every trial (identical in all lanes), then the
          // FIRST passing one; the batch's last trial at t = iter_ls is taken
          // when nothing passes (linesearch.py:71)
          unsigned pm = 0u;
          double fb[8];
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            double ab[NA];
#pragma unroll
            for (int a = 0; a < NA; ++a) ab[a] = Obj::init(a, d) + v[a][b];
            bool ferr = false;
            if constexpr (NA > 1) {  // Ackley: exp / sqrt only for evaluated trials
              fb[b] = 0.0;
              if (b < B) fb[b] = Obj::finish(ab, d, ferr);
            } else {
              fb[b] = Obj::finish(ab, d, ferr);
            }
            const bool pass = fb[b] <= f0 + A.c1 * al[b] * ddir || t0 + b >= A.iter_ls;
            pm |= (b < B && pass) ? (1u << b) : 0u;
          }
          if (pm) {
            const int src = __ffs(pm) - 1;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
              if (b == src) {
                f_new = fb[b];
                alpha = al[b];
#pragma unroll
                for (int a = 0; a < NA; ++a) acc_new[a] = Obj::init(a, d) + v[a][b];
              }
            }
            t_acc = t0 + src;
            break;
          }
          t0 += B;
          B = min(2 * B, kWideMaxB);
        }
      }
#endif
      ls_trials += t_acc + 1;
      prev_trials = t_acc + 1;

      // ---- x_new and the gradient there (bfgs.py:136); DomainError leaves x, k
      const double xn0 = x0 + alpha * p0;
      const double xn1 = own1 ? x1 + alpha * p1 : 0.0;
      ++grads;
      double gn0, gn1;
      {
        double nxn0 = 0.0, nxn1 = 0.0;
        if constexpr (WideTraits<Obj>::kNeighbour) {
          nxn0 = nx0 + alpha * np0;  // == the neighbour lane's x_new, same roundings
          nxn1 = nx1 + alpha * np1;
        }
        double sv[NA], tA[2], tB[2];
        bool oor = false, err = false;
        lane_tan<FastMath>(d, nt, l, xn0, xn1, nxn0, nxn1, sv, tA, tB, oor);
        if (__any_sync(kFull, oor))
          lane_tan<PreciseMath>(d, nt, l, xn0, xn1, nxn0, nxn1, sv, tA, tB, oor);
        lane_grad(d, l, tA, tB, acc_new, gn0, gn1, err);
        if (__any_sync(kFull, err)) {
          status = ZEUS_DOMAIN_ERROR;
          break;
        }
      }
      const double dg0 = gn0 - g0, dg1 = gn1 - g1;
      {
        double2* r0 = reinterpret_cast<double2*>(rowv + 4 * l);
        r0[0] = make_double2(dg0, gn0);
        if (own1) reinterpret_cast<double2*>(rowv + 4 * (l + 32))[0] = make_double2(dg1, gn1);
      }
      __syncwarp();

      // ---- fused pass over my two columns: lazy update, u = H dg, w = H g'
      double u0 = 0.0, w0 = 0.0, u1 = 0.0, w1 = 0.0;
      {
        double u0b = 0.0, w0b = 0.0, u1b = 0.0, w1b = 0.0;
#pragma unroll
        for (int i = 0; i < RR; ++i) {
          const double2 ra = *reinterpret_cast<const double2*>(rowv + 4 * i);      // dg, g'
          const double2 rb = *reinterpret_cast<const double2*>(rowv + 4 * i + 2);  // dx, u
          const double e0 = pending ? fma(rb.x, a0, fma(rb.y, b0, h0[i])) : h0[i];
          const double e1 = pending ? fma(rb.x, a1, fma(rb.y, b1, h1[i])) : h1[i];
          h0[i] = e0;
          h1[i] = e1;
          if (i & 1) {
            UACC(u0b = fma(e0, ra.x, u0b));
            w0b = fma(e0, ra.y, w0b);
            UACC(u1b = fma(e1, ra.x, u1b));
            w1b = fma(e1, ra.y, w1b);
          } else {
            UACC(u0 = fma(e0, ra.x, u0));
            w0 = fma(e0, ra.y, w0);
            UACC(u1 = fma(e1, ra.x, u1));
            w1 = fma(e1, ra.y, w1);
          }
        }
        // rows RR.. from shared memory, two per step with every load issued
        // before the arithmetic (the loads' latency overlaps)
        int i = RR;
        for (; i + 1 < d; i += 2) {
          const double2 ra = *reinterpret_cast<const double2*>(rowv + 4 * i);
          const double2 rb = *reinterpret_cast<const double2*>(rowv + 4 * i + 2);
          const double2 rc = *reinterpret_cast<const double2*>(rowv + 4 * i + 4);
          const double2 rd = *reinterpret_cast<const double2*>(rowv + 4 * i + 6);
          double* hr = Hs + (i - RR) * kWideLd;
          double e0 = hr[l], e1 = hr[l + 32], f0v = hr[kWideLd + l], f1v = hr[kWideLd + l + 32];
          if (pending) {
            e0 = fma(rb.x, a0, fma(rb.y, b0, e0));
            e1 = fma(rb.x, a1, fma(rb.y, b1, e1));
            f0v = fma(rd.x, a0, fma(rd.y, b0, f0v));
            f1v = fma(rd.x, a1, fma(rd.y, b1, f1v));
            hr[l] = e0;
            hr[l + 32] = e1;
            hr[kWideLd + l] = f0v;
            hr[kWideLd + l + 32] = f1v;
          }
          UACC(u0 = fma(e0, ra.x, u0));
          w0 = fma(e0, ra.y, w0);
          UACC(u1 = fma(e1, ra.x, u1));
          w1 = fma(e1, ra.y, w1);
          UACC(u0b = fma(f0v, rc.x, u0b));
          w0b = fma(f0v, rc.y, w0b);
          UACC(u1b = fma(f1v, rc.x, u1b));
          w1b = fma(f1v, rc.y, w1b);
        }
        if (i < d) {
          const double2 ra = *reinterpret_cast<const double2*>(rowv + 4 * i);
          const double2 rb = *reinterpret_cast<const double2*>(rowv + 4 * i + 2);
          double* hr = Hs + (i - RR) * kWideLd;
          double e0 = hr[l], e1 = hr[l + 32];
          if (pending) {
            e0 = fma(rb.x, a0, fma(rb.y, b0, e0));
            e1 = fma(rb.x, a1, fma(rb.y, b1, e1));
            hr[l] = e0;
            hr[l + 32] = e1;
          }
          UACC(u0b = fma(e0, ra.x, u0b));
          w0b = fma(e0, ra.y, w0b);
          UACC(u1b = fma(e1, ra.x, u1b));
          w1b = fma(e1, ra.y, w1b);
        }
        w0 += w0b;
        w1 += w1b;
#if ZEUS_WIDE_UFROMP
        // u = H_k dg = H_k g' - H_k g = w + p: p = -H_k g is this iteration's
        // direction (exact in exact arithmetic), so the pass needs one matvec
        u0 = w0 + p0;
        u1 = w1 + p1;
        (void)u0b;
        (void)u1b;
#else
        u0 += u0b;
        u1 += u1b;
#endif
      }

      // ---- one 8-value reduction: norms, curvature and the p' scalars
      const double dx0 = xn0 - x0, dx1 = own1 ? xn1 - x1 : 0.0;
      double part[8];
      part[0] = fma(gn1, gn1, gn0 * gn0);
      part[1] = fma(dx1, dg1, dx0 * dg0);
      part[2] = fma(dx1, dx1, dx0 * dx0);
      part[3] = fma(dg1, dg1, dg0 * dg0);
      part[4] = fma(dg1, u1, dg0 * u0);
      part[5] = fma(u1, gn1, u0 * gn0);
      part[6] = fma(dx1, gn1, dx0 * gn0);
      part[7] = fma(w1, gn1, w0 * gn0);
      warp_sum8(part);
      const double curv = part[1];
      const double ndx = sqrt(part[2]), ndg = sqrt(part[3]);
      pending = !(curv <= kCurvatureFloor * ndx * ndg);  // bfgs.py:69-71
      __syncwarp();  // rowv (dx/u of the previous iteration) fully consumed
      double pd;
      {
        const double rho = pending ? 1.0 / curv : 0.0;
        const double cc = pending ? fma(rho * rho, part[4], rho) : 0.0;
        const double ug = part[5], xg = part[6];
        double q0 = -w0, q1 = -w1;
        if (pending) {
          // p' = -(w - rho dx (u.g') - rho u (dx.g') + c dx (dx.g'))
          q0 = -(w0 + fma(dx0, fma(cc, xg, -rho * ug), -rho * xg * u0));
          q1 = -(w1 + fma(dx1, fma(cc, xg, -rho * ug), -rho * xg * u1));
          a0 = fma(cc, dx0, -rho * u0);
          b0 = -rho * dx0;
          a1 = fma(cc, dx1, -rho * u1);
          b1 = -rho * dx1;
          reinterpret_cast<double2*>(rowv + 4 * l)[1] = make_double2(dx0, u0);
          if (own1) reinterpret_cast<double2*>(rowv + 4 * (l + 32))[1] = make_double2(dx1, u1);
        }
        if (!own1) q1 = 0.0;
        p0 = q0;
        p1 = q1;
        pd = fma(gn1, q1, gn0 * q0);
      }
      // x, g <- x_new, g_new (bfgs.py:141-145)
      x0 = xn0;
      x1 = xn1;
      g0 = gn0;
      g1 = gn1;
      f0 = f_new;
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[a] = acc_new[a];
      gnorm = sqrt(part[0]);
      ddir = warp_sum(pd);  // np.dot(g, p) of the next line search
      ++k;
      __syncwarp();
      if (A.stop_flag && *(volatile int*)A.stop_flag) {
        status = ZEUS_STOPPED;
        break;
      }
    }

  done:
    const zeus_bfgs_out& o = A.out;
    o.x_final[(int64_t)l * o.ld_out + s] = x0;
    if (own1) o.x_final[(int64_t)(l + 32) * o.ld_out + s] = x1;
    if (l == 0) {
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
    __syncwarp();
  }
};

#ifndef ZEUS_WIDE_MINB
#define ZEUS_WIDE_MINB 5
#endif

#ifdef ZEUS_WIDE_RR_OVERRIDE
#define ZEUS_WIDE_RR_OF(Obj) ZEUS_WIDE_RR_OVERRIDE
#define ZEUS_WIDE_MINB_OF(Obj) ZEUS_WIDE_MINB
#else
#define ZEUS_WIDE_RR_OF(Obj) WideShape<Obj>::RR
#define ZEUS_WIDE_MINB_OF(Obj) WideShape<Obj>::MINB
#endif

template <class Obj, int RR>
__global__ void __launch_bounds__(kWideWarps * 32, ZEUS_WIDE_MINB_OF(Obj))
    bfgs_wide_kernel(BfgsArgs A) {
  extern __shared__ double sm[];
  const int l = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* alpha_tab = sm;
  if (threadIdx.x == 0) {
    double a = A.alpha0;  // alpha0 * shrink^t by repeated multiplication (linesearch.py:70)
    for (int t = 0; t < A.nalpha; ++t) {
      alpha_tab[t] = a;
      a *= A.shrink;
    }
  }
  __syncthreads();
  WideStart<Obj, RR> W;
  W.atab = alpha_tab;
  W.rowv = sm + A.nalpha + (size_t)wib * A.warp_doubles;
  W.Hs = W.rowv + 4 * 64;
  for (;;) {
    long long s = 0;
    if (l == 0) s = (long long)atomicAdd(A.work, 1ull);
    s = __shfl_sync(kFull, s, 0);
    if (s >= A.n) break;
    W.run(A, s, l);
  }
}

namespace {

template <class Obj, int RR>
int launch_wide_rr(BfgsArgs A, cudaStream_t s) {
  A.nalpha = kAlphaTable;
  A.warp_doubles = 4 * 64 + std::max(0, A.d - RR) * kWideLd;
  const size_t smem = sizeof(double) * ((size_t)A.nalpha + (size_t)kWideWarps * A.warp_doubles);
  auto kern = bfgs_wide_kernel<Obj, RR>;
  int rc = check_cuda(
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
      "cudaFuncSetAttribute(wide)");
  if (rc) return rc;
  int per_sm = 0;
  rc = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWideWarps * 32, smem),
                  "occupancy(wide)");
  if (rc) return rc;
  const int sms = current_sm_count();
  if (per_sm < 1 || sms < 1) return set_error(ZEUS_ERR_UNSUPPORTED, "bfgs wide: does not fit");
  int64_t grid = (int64_t)per_sm * sms;
  const int64_t need = (A.n + kWideWarps - 1) / kWideWarps;
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, kWideWarps * 32, smem, s>>>(A);
  return check_launch("bfgs_wide_kernel");
}


struct WideLaunch {
  template <class Obj>
  static int run(BfgsArgs A, cudaStream_t s) {
    if constexpr (Obj::kId == ZEUS_OBJ_GOLDSTEIN_PRICE ||
                  (Obj::kId == ZEUS_OBJ_ACKLEY && !ZEUS_WIDE_ACKLEY)) {
      return set_error(ZEUS_ERR_UNSUPPORTED, "wide: objective runs on another kernel");
    } else {
      return launch_wide_rr<Obj, ZEUS_WIDE_RR_OF(Obj)>(A, s);
    }
  }
};

}  // namespace

bool bfgs_wide_covers(int obj, int d) {
  return (obj == ZEUS_OBJ_ROSENBROCK || obj == ZEUS_OBJ_RASTRIGIN ||
          (ZEUS_WIDE_ACKLEY && obj == ZEUS_OBJ_ACKLEY)) &&
         d > 32 && d <= 64;
}

int launch_bfgs_wide(int obj, BfgsArgs A, cudaStream_t s) {
  return dispatch_objective<WideLaunch>(obj, A, s);
}

}  // namespace zeus
