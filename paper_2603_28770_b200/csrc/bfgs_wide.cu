// bfgs_wide.cu -- multistart BFGS (bfgs.py:80-156) for 32 < d <= 128, one or
// two WARPS per start, built for throughput (the 1M-start 50-D targets and
// config 4's 100-D Rosenbrock).
//
// Why not one CTA per start (the round-1 design, measured and retired): at
// d = 50 such a start costs ~7,300 cycles of wall time per
// iteration, 55% of it in the CTA-synchronised line search and 24% in CTA
// reductions, and only 4 starts fit an SM (scripts/phase_probe.py).  Here a
// start's state is spread over the lanes of W = 1 warp (d <= 64) or W = 2
// warps (d <= 128); W = 1 is synchronised by shuffles only, W = 2 adds one
// 64-thread barrier per reduction, so several starts share an SM and their
// latency-bound phases overlap each other's FP64 work.
//
// Ownership: lane l of warp w owns coordinates c0 = 64 w + l and c1 = c0 + 32
// (if < d): their x, p, g entries live in REGISTERS, and so do the first RR
// rows of the two inverse-Hessian columns H[:, c0], H[:, c1]; rows RR..d-1 of
// those columns live in the start's shared-memory slice (conflict-free: lanes
// read consecutive columns).  At d = 50 (T50, Rosenbrock and Rastrigin) the
// H elements are instead distributed by the BLOCK layout (WideStart) over
// registers and TENSOR MEMORY (tmem.cuh: each thread's elements in its own
// TMEM lane, 4-warp CTAs, 4 per SM, 128 columns each).  The per-row broadcast
// values of the fused H pass {g'_i, dx_i, u_i} (three [64 W] arrays, read two
// rows per 16-byte load) are the only other shared-memory traffic.
//
// Per iteration (reference order, bfgs.py:108-156):
//  1. Armijo search (linesearch.py:60-71) in chunks of CH trials
//     alpha0 shrink^t evaluated together and tested in order until one passes:
//     every lane evaluates its own objective terms of the chunk's trials in
//     registers (x + alpha p with the reference's two roundings), one
//     transpose-reduce folds them, and the FIRST passing trial is taken --
//     alpha, trial count and f of the sequential search;
//  2. gradient at x_new from lane-local forward-mode term tangents
//     (autodiff.py:243-266 restricted to the terms that contain x_i; the one
//     neighbour tangent Rosenbrock needs arrives by shuffle);
//  3. one fused pass over H: the lazy rank-2 update of the previous iteration
//     (H += dx a^T + u b^T, the O(d^2) form of bfgs.py:72-77) and w = H g' in
//     the same sweep; u = H dg = w + p (p = -H g is this iteration's
//     direction), so one matvec per pass;
//  4. one 8-value reduction: |g'|^2, dx.dg, |dx|^2, |dg|^2, dg.u, u.g',
//     dx.g', w.g' -> curvature guard (bfgs.py:69-71), rho, the next direction
//     p' = -H' g' = -(w - rho dx (u.g') - rho u (dx.g') + c dx (dx.g'));
//  5. g'.p' (the next line search's ddir) by one butterfly.
// Objective folds for d > 16 are trees: f agrees with
// the reference's sequential fold to ~1 ulp, inside the stated tolerance.
#include <cstdlib>

#include "bfgs_common.cuh"
#include "tmem.cuh"

namespace zeus {

namespace {

constexpr int kWideThreads = 64;  // block: 2 warps = 2 starts (W = 1) or 1 start (W = 2)
// TMEM kernels: CTAs of 4 warps (warp w on TMEM lane quarter w) -- four
// starts of one warp (d = 50) or two starts of two warps (d = 100) --
// WideShape::TM_CTAS per SM, the SM's 512 TMEM columns split between them
constexpr int kTmWarps = 4;

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
  // the objective evaluates trig (a fast-path range fallback is possible) /
  // can raise a DomainError (Ackley's sqrt'(0), autodiff.py:207-213); without
  // them the team votes on oor / err are skipped (a barrier each at W = 2)
  static constexpr bool kTrig = Obj::kId == ZEUS_OBJ_RASTRIGIN || Obj::kId == ZEUS_OBJ_ACKLEY;
  static constexpr bool kErr = Obj::kId == ZEUS_OBJ_ACKLEY;
};

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(kFull, v, src); }

// f from the folded accumulators / gradient component from term tangents;
// Ackley's out-of-line copies (objectives.cuh) keep the kernels' code small
template <class Obj>
__device__ __forceinline__ double wfinish(const double* acc, int d, bool& err) {
  if constexpr (Obj::kId == ZEUS_OBJ_ACKLEY) return Obj::finish_ool(acc, d, err);
  else return Obj::finish(acc, d, err);
}
template <class Obj, class TA>
__device__ __forceinline__ double wgrad(const TA& tan, int i, int d, const double* acc, bool& err) {
  if constexpr (Obj::kId == ZEUS_OBJ_ACKLEY) return Obj::grad_from_tan_ool(tan, i, d, acc, err);
  else return Obj::grad_from_tan(tan, i, d, acc, err);
}
__device__ __forceinline__ double shfl_xor(double v, int m) { return __shfl_xor_sync(kFull, v, m); }

}  // namespace

// Shape, tuned on B200 (scripts/wide_variants.sh + scripts/phase_probe.py at
// d = 50): rows of H kept in registers (RR), resident blocks per SM (MINB; 2
// warps each), trials per line-search chunk (CH: Ackley needs 1.6 trials per
// iteration, Rosenbrock 2.7, Rastrigin 6.2; SM-cycles per start-iteration for
// CH = 1 / 2 / 3 / 4: Rosenbrock 820 / 770 / 781 / 793, Rastrigin 1781 / 1729
// / 1746 / 1915, Ackley 1596 / 1854 (team kernel: 2884)) and shared-memory H
// rows per step of the fused pass (SR).
template <class Obj, int W>
struct WideShape {
  // W = 1: 20 register rows at 168 registers = 3 warps per SMSP (12 starts/SM;
  // the per-SMSP register file caps 3 warps at 168); measured at d = 50
  // (SM-cycles/start-iteration, RR/MINB/SR): Rosenbrock 772 (32/4/4) -> 713
  // (20/6/2), Rastrigin 1688 -> 1556, Ackley 1331 -> 1320.  W = 2 (d <= 128):
  // 32 rows, 4 blocks/SM, four shared-memory rows per step (2: 11% slower).
  static constexpr int RR = W > 1 ? 32 : 20;
#ifdef ZEUS_WIDE_MINB_OVERRIDE
  static constexpr int MINB = ZEUS_WIDE_MINB_OVERRIDE;
#else
  static constexpr int MINB = W > 1 ? 4 : 6;
#endif
  static constexpr int CH = Obj::kId == ZEUS_OBJ_ACKLEY ? 1 : 2;
  // TMEM kernel (d = 50, the block layout of WideStart): TM_CTAS 4-warp CTAs
  // per SM (4 = 16 warps: <= 128 registers per thread, all 512 TMEM columns
  // allocated), RR_TM of a lane's 25 block rows in registers, the rest in
  // TMEM.  Measured at d = 50 (SM-cycles per start-iteration): the split
  // layout that preceded it (column l + half a column + 4 rows per lane,
  // 80 elements) Rosenbrock 508 at 3 CTAs / 36 register elements, 476 at
  // 4 / 16; Rastrigin 1,153 / 1,087; this layout Rosenbrock 448 (RR 7),
  // 454 (5), 492 (9), 516 (11); Rastrigin 1,062 (5), 1,070 (7), 1,085 (9);
  // 3 CTAs (168 registers, RR 9): 484 / 1,173.
  static constexpr bool kRosen = Obj::kId == ZEUS_OBJ_ROSENBROCK;
#ifdef ZEUS_WIDE_TM_CTAS
  static constexpr int TM_CTAS = ZEUS_WIDE_TM_CTAS;
#else
  static constexpr int TM_CTAS = W > 1 ? 2 : 4;  // d = 100: 8 warps, 256 columns per CTA
#endif
  static constexpr int TM_COLS = 512 / TM_CTAS;  // TMEM columns per CTA (= per warp)
#ifdef ZEUS_WIDE_RR_TM
  static constexpr int RR_TM = ZEUS_WIDE_RR_TM;
#else
  static constexpr int RR_TM = W > 1 ? 8 : (kRosen ? 7 : 5);
#endif
  // d = 20 (config 5, sequential folds): trials per chunk and resident
  // 2-warp blocks per SM, measured (SM-cycles per start-iteration, CH / MINB):
  // Rastrigin 960 (2 / 6), 878 (3 / 6), 909 (4 / 6), 1,026 (4 / 8);
  // Rosenbrock 314 (2 / 6), 295 (2 / 8), 322 (3 / 6); the warp kernel
  // (bfgs_warp.cuh) it replaces: 1,348 / 512
#ifdef ZEUS_WIDE_SEQ_CH
  static constexpr int SEQ_CH = ZEUS_WIDE_SEQ_CH;
#else
  static constexpr int SEQ_CH = kRosen ? 2 : 3;
#endif
#ifdef ZEUS_WIDE_SEQ_MINB
  static constexpr int SEQ_MINB = ZEUS_WIDE_SEQ_MINB;
#else
  static constexpr int SEQ_MINB = kRosen ? 8 : 6;
#endif
#ifdef ZEUS_WIDE_SMEM_STEP
  static constexpr int SR = ZEUS_WIDE_SMEM_STEP;
#else
  static constexpr int SR = W > 1 ? 4 : 2;  // shared-memory rows per step (<= 4)
#endif
};

// Shared-memory slice of one start, in doubles: rowv [4][64W] (g', dx, u and
// a spare row), H rows
// [d - RR][64W], exchange scratch (W > 1): two reduction buffers [2][W][8],
// boundary values x, p, tangent [3][W].
__host__ __device__ inline int wide_slot_doubles(int d, int rr, int w) {
  return 4 * 64 * w + (d > rr ? d - rr : 0) * 64 * w + (w > 1 ? 16 * w + 3 * w : 0);
}

// D > 0: the kernel compiled for that dimension (row loops fully unrolled,
// shared-memory offsets immediate); D = 0: any 32 < d <= 64 W at run time.
template <class Obj, int RR, int W, int D, bool TM = false>
struct WideStart {
  static constexpr int NA = Obj::NACC;
  static constexpr int LD = 64 * W;  // row stride of the shared-memory H rows
  // TM (d = 50): the BLOCK layout.  Lane l owning columns l and l + 32
  // would leave 14 of a warp's 64 column slots empty at d = 50, and one load
  // of a row value would serve one or two elements per lane.  Instead lane
  // l = 16 q + p keeps rows 2 r + q (r = 0..24) of columns 3 p .. 3 p + 2
  // (columns 0..47) plus rows (l & 15) + 16 t (t = 0..3) of column
  // 48 + (l >> 4): 79 elements, no dead slot, and one load of a row value
  // (g', dx, u: 16 contiguous bytes for the two parities, one shared-memory
  // wavefront) serves three columns.  The update coefficients of every
  // column are in shared memory (written by the owners); the column sums
  // are completed over the two parities by one shuffle and handed to the
  // owners through the spare rowv row.  RR block rows in registers, the
  // other NT3 in Tensor Memory.
  static constexpr bool BLK3 = TM;
  // SEQ (one warp, d <= 32: config 5's d = 20): objective values are folded in
  // the reference's sequential order (a Python left fold, objectives.py:
  // 40-85) instead of a tree, so f at identical x is the reference's f bit
  // for bit (Rosenbrock) and Armijo decisions at the noise floor |g| ~ theta
  // follow the reference's; the terms go through the spare rowv row and lane
  // q folds value q.
  static constexpr bool SEQ = W == 1 && D > 0 && D <= 32;
  // SEQ: trials per chunk -- the CH folds run in parallel lanes, so a wider
  // chunk means fewer sequential fold rounds per iteration (WideShape)
  static constexpr int kSeqCH = NA == 1 ? WideShape<Obj, 1>::SEQ_CH : 1;
  static_assert(!TM || (W == 1 && D == 50) || (W == 2 && D == 100),
                "TMEM kernels: the block layout at d = 50 (one warp) / 100 (two warps)");
  // d = 100 (W = 2): lane L = 32 w + l keeps rows 2 r + q (r = 0..49, q =
  // bit 4 of l) of columns 3 p .. 3 p + 2, p = 16 w + (l & 15) (columns
  // 0..95), plus rows (L & 15) + 16 t (t = 0..6) of column 96 + (L >> 4)
  static constexpr int NRW = D / 2;              // block rows per lane
  static constexpr int XT = (D + 15) / 16;       // rows per lane of the extra columns
  static constexpr int NT3 = BLK3 ? NRW - RR : 0;  // block rows in TMEM
  static constexpr int TMA = WideShape<Obj, W>::TM_COLS;
  static_assert(!BLK3 || (NT3 % 2 == 0 && 6 * NT3 <= TMA), "block layout");
  // several starts per CTA (d = 100): per-start named barriers
  static constexpr bool MULTI = TM && W > 1;
  static constexpr int H0N = BLK3 ? 1 : RR;  // register arrays of the pass
  static constexpr int H1N = BLK3 ? 3 * RR + XT : SEQ ? 1 : RR;  // SEQ: no column c1
  uint32_t tm = 0;     // TM: this thread's TMEM column base (lane = its thread)
  double* Hs;          // [d - RR][LD] rows RR.. of every column of the start
  double* rowv;        // [4][64 W]: g' | dx_prev | u_prev | w (TM); TM: + [64][2] (a, b)
  double* xch;         // W > 1: [2][W][8] reductions, then xb[W], pb[W], tb[W]
  const double* atab;  // block alpha table
  int wi = 0;          // warp index within the start (0 .. W-1)
  int slot = 0;        // reduction double-buffer
  int bar_id = 0;      // MULTI: the start's named barrier (1 + its slot in the CTA)

  __device__ __forceinline__ double alpha_at(const BfgsArgs& A, int t) const {
    if (t < A.nalpha) return atab[t];
    double a = atab[A.nalpha - 1];
    for (int k = A.nalpha - 1; k < t; ++k) a *= A.shrink;
    return a;
  }

  // ---- team primitives (W == 1: the warp itself) -------------------------
  __device__ __forceinline__ void team_sync() const {
    if constexpr (MULTI) {
      asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "n"(32 * W) : "memory");
    } else if constexpr (W > 1) {
      __syncthreads();
    } else {
      __syncwarp();
    }
  }
  __device__ __forceinline__ bool team_any(bool b) const {
    if constexpr (MULTI) {
      int r;
      asm volatile(
          "{\n .reg .pred p, q;\n setp.ne.s32 p, %1, 0;\n bar.red.or.pred q, %2, %3, p;\n"
          " selp.s32 %0, 1, 0, q;\n}\n"
          : "=r"(r)
          : "r"((int)b), "r"(bar_id), "n"(32 * W)
          : "memory");
      return r != 0;
    } else if constexpr (W > 1) {
      return __syncthreads_or(b);
    } else {
      return __any_sync(kFull, b);
    }
  }
  // 8 values summed over the team, identical in every lane of every warp
  // (warp transpose-reduce, then the W warp totals in warp order)
  __device__ __forceinline__ void team_sum8(double v[8], int l) {
    warp_sum8(v);
    if constexpr (W > 1) {
      double* r = xch + slot * 8 * W;
      slot ^= 1;  // the next call's buffer: a warp cannot be two calls ahead
      if (l == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) r[wi * 8 + q] = v[q];
      }
      team_sync();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double s = r[q];
#pragma unroll
        for (int w = 1; w < W; ++w) s += r[w * 8 + q];
        v[q] = s;
      }
    }
  }
  // SEQ: values v[0 .. nv) (nv <= 4: rows 3..4 of the slot hold 4 x 32 terms), each
  // lane's term of value q, folded as init[q] + t_0 + t_1 + ... + t_{nt-1}
  // (left to right), identical in every lane
  __device__ __forceinline__ void seq_fold(double v[8], const double init[8], int nv, int l,
                                           int nt) const {
    double* T = rowv + 3 * LD;
    __syncwarp();  // the previous fold's readers are done
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < nv && l < nt) T[q * 32 + l] = v[q];
    __syncwarp();
    double sacc = 0.0;
    if (l < nv) {
      double t[D > 0 ? D : 1];
#pragma unroll
      for (int j = 0; j < (D > 0 ? D : 1); ++j) t[j] = j < nt ? T[l * 32 + j] : 0.0;
      sacc = init[0];
#pragma unroll
      for (int q = 1; q < 4; ++q)
        if (l == q) sacc = init[q];
#pragma unroll
      for (int j = 0; j < (D > 0 ? D : 1); ++j) {
        if (j >= nt) break;
        sacc = sacc + t[j];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < nv) v[q] = shfl(sacc, q);
  }

  // v[0..3] summed over the team (one transpose-reduce: 10 shuffles)
  __device__ __forceinline__ void team_sum4(double v[8], int l) {
    warp_sum4(v);
    if constexpr (W > 1) {
      double* r = xch + slot * 8 * W;
      slot ^= 1;
      if (l == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) r[wi * 8 + q] = v[q];
      }
      team_sync();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double s = r[q];
#pragma unroll
        for (int w = 1; w < W; ++w) s += r[w * 8 + q];
        v[q] = s;
      }
    }
  }
  // v[0], v[1] summed over the team (butterflies: 10 shuffles instead of 17)
  __device__ __forceinline__ void team_sum2(double v[8], int l) {
    v[0] = warp_sum(v[0]);
    v[1] = warp_sum(v[1]);
    if constexpr (W > 1) {
      double* r = xch + slot * 8 * W;
      slot ^= 1;
      if (l == 0) {
        r[wi * 8] = v[0];
        r[wi * 8 + 1] = v[1];
      }
      team_sync();
      double s0 = r[0], s1 = r[1];
#pragma unroll
      for (int w = 1; w < W; ++w) {
        s0 += r[w * 8];
        s1 += r[w * 8 + 1];
      }
      v[0] = s0;
      v[1] = s1;
    }
  }
  __device__ __forceinline__ double team_sum(double v, int l) {
    v = warp_sum(v);
    if constexpr (W > 1) {
      double* r = xch + slot * 8 * W;
      slot ^= 1;
      if (l == 0) r[wi * 8] = v;
      team_sync();
      double s = r[0];
#pragma unroll
      for (int w = 1; w < W; ++w) s += r[w * 8];
      v = s;
    }
    return v;
  }

  // Values of this lane's terms (c0, c1) at CH trial points x + alpha_c p,
  // s[c][a] = (0 + t(c0)) + t(c1) (the team kernel's lane order).  Branch-free:
  // all 2 CH term evaluations are independent chains the scheduler can
  // interleave (a missing term is evaluated at 0 and masked out).
  // W = 1 with d fixed: every lane's first term exists (c0 < 32 <= nt)
  static constexpr bool kAllC0 = W == 1 && D > 0 && Obj::nterms(D) >= 32;

  template <class M, int CH>
  __device__ __forceinline__ void lane_terms(int d, int nt, int c0, const double al[CH],
                                             double x0, double x1, double p0, double p1,
                                             double nx0, double nx1, double np0, double np1,
                                             double s[CH][NA], bool& oor) const {
    const int c1 = c0 + 32;
    const bool v0 = kAllC0 || c0 < nt, v1 = c1 < nt;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const double xt0 = x0 + al[c] * p0, xt1 = x1 + al[c] * p1;
      double xn0 = 0.0, xn1 = 0.0;
      if constexpr (WideTraits<Obj>::kNeighbour) {
        xn0 = nx0 + al[c] * np0;
        xn1 = nx1 + al[c] * np1;
      }
      double t0[NA], t1[NA];
      Obj::template term<M>(LX{c0, xt0, xn0}, c0, d, t0, oor);
      Obj::template term<M>(LX{c1, xt1, xn1}, c1, d, t1, oor);
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
  __device__ __noinline__ void lane_terms_precise(int d, int nt, int c0, const double* al,
                                                  double x0, double x1, double p0, double p1,
                                                  double nx0, double nx1, double np0,
                                                  double np1, double* out) const {
    double a4[CH], sc[CH][NA];
    for (int c = 0; c < CH; ++c) a4[c] = al[c];
    bool oor = false;
    lane_terms<PreciseMath, CH>(d, nt, c0, a4, x0, x1, p0, p1, nx0, nx1, np0, np1, sc, oor);
    for (int c = 0; c < CH; ++c)
      for (int a = 0; a < NA; ++a) out[c * NA + a] = sc[c][a];
  }

  // Values AND term tangents of this lane's terms at the point (x0, x1)
  // (neighbour coordinates nx0, nx1); branch-free like lane_terms.
  template <class M>
  __device__ __forceinline__ void lane_tan(int d, int nt, int c0, double x0, double x1,
                                           double nx0, double nx1, double s[NA], double tA[2],
                                           double tB[2], bool& oor) const {
    const int c1 = c0 + 32;
    const bool v0 = kAllC0 || c0 < nt, v1 = c1 < nt;
    double t0[NA], t1[NA], n0[Obj::KT], n1[Obj::KT];
    Obj::template term_tan<M>(LX{c0, x0, nx0}, c0, d, t0, n0, oor);
    Obj::template term_tan<M>(LX{c1, x1, nx1}, c1, d, t1, n1, oor);
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

  // Cold path of lane_tan (some |2 pi x| > kTrigMax: CUDA libm), out of line
  // so the hot loop's code stays small in the instruction cache.
  __device__ __noinline__ void lane_tan_precise(int d, int nt, int c0, double x0, double x1,
                                                double nx0, double nx1, double* s, double* tA,
                                                double* tB) const {
    double sv[NA], a[2], b[2];
    bool oor = false;
    lane_tan<PreciseMath>(d, nt, c0, x0, x1, nx0, nx1, sv, a, b, oor);
    for (int q = 0; q < NA; ++q) s[q] = sv[q];
    tA[0] = a[0], tA[1] = a[1], tB[0] = b[0], tB[1] = b[1];
  }

  // Gradient components of c0, c1 from the lane's term tangents (+ the
  // neighbour's tangent of term c-1 w.r.t. x_c for Rosenbrock; across the
  // warp boundary it comes through the exchange scratch).
  __device__ __forceinline__ void lane_grad(int d, int l, int c0, const double tA[2],
                                            const double tB[2], const double acc[NA],
                                            double& g0, double& g1, bool& err) {
    const int c1 = c0 + 32;
    double prevA = 0.0, prevB = 0.0;
    if constexpr (WideTraits<Obj>::kNeighbour) {
      const int src = (l + 31) & 31;
      const double s0 = shfl(tA[1], src), s1 = shfl(tB[1], src);
      prevA = s0;                 // term c0-1 (lane l-1's c0 term), l >= 1
      prevB = l >= 1 ? s1 : s0;   // term c1-1: lane l-1's c1 term, or lane 31's c0 term
      if constexpr (W > 1) {      // term 64w - 1: the previous warp's lane 31 c1 term
        double* tb = xch + 16 * W + 2 * W;
        if (l == 31) tb[wi] = tB[1];
        team_sync();
        if (l == 0 && wi > 0) prevA = tb[wi - 1];
      }
    }
    g0 = 0.0;
    if ((W == 1 && D > 32) || c0 < d) g0 = wgrad<Obj>(LT{c0, tA[0], tA[1], prevA}, c0, d, acc, err);
    g1 = 0.0;
    if (c1 < d) g1 = wgrad<Obj>(LT{c1, tB[0], tB[1], prevB}, c1, d, acc, err);
  }

  // neighbour coordinates (Rosenbrock term j needs x_{j+1}) of two lane
  // vectors (x and p); the last lane's c1 neighbour is the next warp's c0
  __device__ __forceinline__ void neighbours2(int l, double x0, double x1, double p0, double p1,
                                              double& nx0, double& nx1, double& np0,
                                              double& np1) {
    if constexpr (WideTraits<Obj>::kNeighbour) {
      const int src = (l + 1) & 31;
      const double tx0 = shfl(x0, src), tx1 = shfl(x1, src);
      const double tp0 = shfl(p0, src), tp1 = shfl(p1, src);
      nx0 = l < 31 ? tx0 : tx1;  // x_{c0+1}; lane 31 -> lane 0's c1
      np0 = l < 31 ? tp0 : tp1;
      nx1 = tx1;                 // x_{c1+1}; lane 31 -> next warp (below)
      np1 = tp1;
      if constexpr (W > 1) {
        double* xb = xch + 16 * W;
        double* pb = xb + W;
        if (l == 0) {
          xb[wi] = x0;
          pb[wi] = p0;
        }
        team_sync();
        if (l == 31) {
          nx1 = wi + 1 < W ? xb[wi + 1] : 0.0;
          np1 = wi + 1 < W ? pb[wi + 1] : 0.0;
        }
      }
    }
  }

  // BLK3 pass: the lazy rank-2 update of the lane's 79 elements and their
  // matvec partials; returns w = H g' for the lane's coordinates c0, c1.
  __device__ __forceinline__ void hpass_blk3(int l, double (&h1)[H1N], int c0, int c1,
                                             bool own1, double& w0, double& w1) const {
    const int L = 32 * wi + l;
    const int q = (l >> 4) & 1, pq = 16 * wi + (l & 15), rC0 = L & 15, cX = 48 * W + (L >> 4);
    const double* CF = rowv + 4 * LD;  // (a, b) by column
    double a[3], b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double2 ab = *reinterpret_cast<const double2*>(CF + 2 * (3 * pq + k));
      a[k] = ab.x;
      b[k] = ab.y;
    }
    const double2 abC = *reinterpret_cast<const double2*>(CF + 2 * cX);
    const double aC = abC.x, bC = abC.y;
    const double* G = rowv + q;
    const double* DX = rowv + LD + q;
    const double* U = rowv + 2 * LD + q;
    double w[3] = {0.0, 0.0, 0.0}, wc[2] = {0.0, 0.0};
#pragma unroll
    for (int r = 0; r < RR; ++r) {  // register rows: row 2 r + q
      const double g = G[2 * r], x = DX[2 * r], u = U[2 * r];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        h1[3 * r + k] = fma(x, a[k], fma(u, b[k], h1[3 * r + k]));
        w[k] = fma(h1[3 * r + k], g, w[k]);
      }
    }
#pragma unroll
    for (int t = 0; t < XT; ++t) {  // the extra column's rows: 16 consecutive rows per load
      const int r = rC0 + 16 * t;
      h1[3 * RR + t] = fma(rowv[LD + r], aC, fma(rowv[2 * LD + r], bC, h1[3 * RR + t]));
      wc[t & 1] = fma(h1[3 * RR + t], rowv[r], wc[t & 1]);
    }
    tmem::wait_st();
#ifndef ZEUS_WIDE_B3_NR
#define ZEUS_WIDE_B3_NR 2
#endif
    constexpr int NR = ZEUS_WIDE_B3_NR;  // TMEM rows per wait (3 NR elements)
    static_assert(NT3 % NR == 0, "whole TMEM groups");
#pragma unroll
    for (int r0 = RR; r0 < NRW; r0 += NR) {
      double gr[NR], xr[NR], ur[NR];
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        gr[j] = G[2 * (r0 + j)];
        xr[j] = DX[2 * (r0 + j)];
        ur[j] = U[2 * (r0 + j)];
      }
      const uint32_t ta = tm + 6 * (r0 - RR);
      tmem::D2 e[3 * NR];
#pragma unroll
      for (int j = 0; j < 3 * NR; ++j) tmem::ld2(ta + 2 * j, e[j]);
      tmem::wait_ld_n(e);
#pragma unroll
      for (int j = 0; j < NR; ++j) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double v = fma(xr[j], a[k], fma(ur[j], b[k], e[3 * j + k].v()));
          tmem::st2(ta + 6 * j + 2 * k, v);
          w[k] = fma(v, gr[j], w[k]);
        }
      }
    }
    // column sums over the two row parities (lanes l, l ^ 16)
#pragma unroll
    for (int k = 0; k < 3; ++k) w[k] += shfl_xor(w[k], 16);
    double* wv = rowv + 3 * LD;  // the spare row: w by column
    if (q == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) wv[3 * pq + k] = w[k];
    }
    double c = wc[0] + wc[1];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) c += shfl_xor(c, o);
    if (rC0 == 0) wv[cX] = c;
    team_sync();
    w0 = wv[c0];
    w1 = own1 ? wv[c1] : 0.0;
  }

  __device__ void run(const BfgsArgs& A, long long s, int l) {
    const int d = D > 0 ? D : A.d;
    const int nt = Obj::nterms(d);
    const int c0 = 64 * wi + l, c1 = c0 + 32;
    const bool own0 = (W == 1 && D > 32) || c0 < d, own1 = c1 < d;
    // h0 / h1: rows 0..RR-1 of the columns c0 / c1; TM: h1 = the block's
    // register rows [RR][3] then the 4 C rows
    double h0[H0N], h1[H1N];
    double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;  // pending rank-2 coefficients
    double x0 = 0.0, x1 = 0.0, p0 = 0.0, p1 = 0.0, g0 = 0.0, g1 = 0.0;
    double acc[NA];
    double f0;
    int k = 0, status = ZEUS_DIVERGED, ls_trials = 0, grads = 0;
    // |g|^2 (+inf before the first gradient): |g| < theta <=> |g|^2 <= gsq_max,
    // so the square root is taken once, for the output (bfgs.py:118)
    double gsq = __longlong_as_double(0x7ff0000000000000LL);
    double ddir = 0.0;
    // this lane's share of the next line search's g.p, reduced together with
    // the first trial chunk's objective terms (the same tree as a separate
    // warp sum: bitwise the same ddir, one reduction chain less per iteration)
    double pd_part = 0.0;
    bool pending = false;

    // ---- H = I, x = x0, rowv = 0
    if constexpr (BLK3) {
      const int L = 32 * wi + l;
      const int q = (l >> 4) & 1, pq = 16 * wi + (l & 15), cC = 48 * W + (L >> 4), rC0 = L & 15;
#pragma unroll
      for (int r = 0; r < NRW; ++r) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double e = 2 * r + q == 3 * pq + k ? 1.0 : 0.0;
          if (r < RR) {
            h1[3 * r + k] = e;
          } else {
            tmem::st2(tm + 6 * (r - RR) + 2 * k, e);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < XT; ++t) h1[3 * RR + t] = rC0 + 16 * t == cC ? 1.0 : 0.0;
      rowv[4 * LD + 2 * c0] = 0.0;  // column coefficients (a, b) by column
      rowv[4 * LD + 2 * c0 + 1] = 0.0;
      rowv[4 * LD + 2 * c1] = 0.0;
      rowv[4 * LD + 2 * c1 + 1] = 0.0;
    } else {
#pragma unroll
      for (int i = 0; i < RR; ++i) {
        h0[i] = i == c0 ? 1.0 : 0.0;
        if constexpr (!SEQ) h1[i] = i == c1 ? 1.0 : 0.0;
      }
      for (int i = RR; i < d; ++i) {
        Hs[(i - RR) * LD + c0] = i == c0 ? 1.0 : 0.0;
        Hs[(i - RR) * LD + c1] = i == c1 ? 1.0 : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      rowv[q * LD + c0] = 0.0;
      rowv[q * LD + c1] = 0.0;
    }
    if (own0) x0 = A.x0[(int64_t)c0 * A.ldx + s];
    if (own1) x1 = A.x0[(int64_t)c1 * A.ldx + s];
    team_sync();

    double nx0 = 0.0, nx1 = 0.0, np0 = 0.0, np1 = 0.0;

    // ---- f(x0) and the first gradient, from one term pass with tangents
    {
      neighbours2(l, x0, x1, 0.0, 0.0, nx0, nx1, np0, np1);
      double sv[NA], tA[2], tB[2];
      bool oor = false, err = false;
      lane_tan<FastMath>(d, nt, c0, x0, x1, nx0, nx1, sv, tA, tB, oor);
      if (WideTraits<Obj>::kTrig && team_any(oor))
        lane_tan_precise(d, nt, c0, x0, x1, nx0, nx1, sv, tA, tB);
#pragma unroll
      if constexpr (SEQ) {
        double v[8], in[8];
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          v[a] = sv[a];
          in[a] = Obj::init(a, d);
        }
        seq_fold(v, in, NA, l, nt);
#pragma unroll
        for (int a = 0; a < NA; ++a) acc[a] = v[a];
      } else {
#pragma unroll
        for (int a = 0; a < NA; ++a) acc[a] = Obj::init(a, d) + team_sum(sv[a], l);
      }
      bool ferr = false;
      f0 = wfinish<Obj>(acc, d, ferr);
      if (A.stop_flag && team_any(*(volatile int*)A.stop_flag != 0)) {
        status = ZEUS_STOPPED;
        goto done;
      }
      ++grads;
      lane_grad(d, l, c0, tA, tB, acc, g0, g1, err);
      if (WideTraits<Obj>::kErr && team_any(err)) {
        status = ZEUS_DOMAIN_ERROR;
        goto done;
      }
      p0 = -g0;  // H0 = I: -(I @ g) is exact
      p1 = -g1;
      const double gpart = fma(g1, g1, g0 * g0);
      const double gg = team_sum(gpart, l);
      gsq = gg;
      pd_part = -gpart;  // p = -g: sums to -gg exactly (rounding is sign-symmetric)
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
      // ---- Armijo search (linesearch.py:60-71): chunks of CH trials
      // t0 .. t0 + CH - 1 evaluated together, in order, until one passes
      neighbours2(l, x0, x1, p0, p1, nx0, nx1, np0, np1);
      double alpha = 0.0, f_new = 0.0, acc_new[NA];
      int t_acc = -1;
      {
#ifdef ZEUS_WIDE_CH  // (variant builds; kept only where a slot for g.p remains)
        constexpr int CH = ZEUS_WIDE_CH * NA < 8 ? ZEUS_WIDE_CH : WideShape<Obj, W>::CH;
#else
        constexpr int CH = SEQ ? kSeqCH : WideShape<Obj, W>::CH;
#endif
        static_assert(CH * NA <= 8, "one reduction per chunk");
        for (int t0 = 0;; t0 += CH) {
          double al[CH], sc[CH][NA];
          if (t0 == 0) {  // alpha0 shrink^c by the table's own repeated products
            double a = A.alpha0;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              al[c] = a;
              a *= A.shrink;
            }
          } else {
#pragma unroll
            for (int c = 0; c < CH; ++c) al[c] = alpha_at(A, t0 + c);
          }
          bool oor = false;
          lane_terms<FastMath, CH>(d, nt, c0, al, x0, x1, p0, p1, nx0, nx1, np0, np1, sc, oor);
          if (WideTraits<Obj>::kTrig && team_any(oor))  // some |2 pi x| > kTrigMax: libm
            lane_terms_precise<CH>(d, nt, c0, al, x0, x1, p0, p1, nx0, nx1, np0, np1,
                                   &sc[0][0]);
          double v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = q < CH * NA ? sc[q % CH][q / CH] : 0.0;
          static_assert(CH * NA < 8, "a slot for g.p");
          if constexpr (SEQ) {
            static_assert(!SEQ || CH * NA <= 4, "four fold rows");
            if (t0 == 0) ddir = warp_sum(pd_part);  // (a tree, like OpenBLAS's ddot)
            double in[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) in[q] = Obj::init(q / CH, d);
            seq_fold(v, in, CH * NA, l, nt);
          } else if (t0 == 0) {  // g.p rides with the first chunk (slot CH * NA)
            v[CH * NA] = pd_part;
            if constexpr (CH * NA + 1 <= 4) {
              team_sum4(v, l);
            } else {
              team_sum8(v, l);
            }
            ddir = v[CH * NA];
          } else if constexpr (CH * NA <= 2) {
            team_sum2(v, l);  // butterflies (+ the warp totals for W = 2)
          } else if constexpr (CH * NA <= 4) {
            team_sum4(v, l);  // transpose-reduce
          } else {
            team_sum8(v, l);
          }
          unsigned pm = 0u;
          double fb[CH];
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            double ab[NA];
#pragma unroll
            for (int a = 0; a < NA; ++a) ab[a] = SEQ ? v[a * CH + c] : Obj::init(a, d) + v[a * CH + c];
            const bool valid = t0 + c <= A.iter_ls;
            bool ferr = false;
            if constexpr (NA > 1) {  // Ackley: exp / sqrt only for trials that exist
              fb[c] = 0.0;
              if (valid) fb[c] = wfinish<Obj>(ab, d, ferr);
            } else {
              fb[c] = wfinish<Obj>(ab, d, ferr);
            }
            // NaN fails; the trial at t = iter_ls is taken when nothing passed
            const bool pass = fb[c] <= f0 + A.c1 * al[c] * ddir || t0 + c == A.iter_ls;
            pm |= (valid && pass) ? (1u << c) : 0u;
          }
          if (pm) {
            const int src = __ffs(pm) - 1;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              if (c == src) {
                f_new = fb[c];
                alpha = al[c];
#pragma unroll
                for (int a = 0; a < NA; ++a)
                  acc_new[a] = SEQ ? v[a * CH + c] : Obj::init(a, d) + v[a * CH + c];
              }
            }
            t_acc = t0 + src;
            break;
          }
        }
      }
      ls_trials += t_acc + 1;

      // ---- x_new and the gradient there (bfgs.py:136); DomainError leaves x, k
      const double xn0 = own0 ? x0 + alpha * p0 : 0.0;
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
        lane_tan<FastMath>(d, nt, c0, xn0, xn1, nxn0, nxn1, sv, tA, tB, oor);
        if (WideTraits<Obj>::kTrig && team_any(oor))
          lane_tan_precise(d, nt, c0, xn0, xn1, nxn0, nxn1, sv, tA, tB);
        lane_grad(d, l, c0, tA, tB, acc_new, gn0, gn1, err);
        if (WideTraits<Obj>::kErr && team_any(err)) {
          status = ZEUS_DOMAIN_ERROR;
          break;
        }
      }
      const double dg0 = gn0 - g0, dg1 = gn1 - g1;
      if (own0) rowv[c0] = gn0;
      if (own1) rowv[c1] = gn1;
      team_sync();

      // ---- fused pass over my two columns: the lazy rank-2 update of the
      // previous iteration (coefficients zero when its curvature guard
      // skipped it: no select in the pass) and w = H g' (u = w + p below).
      // Four accumulators per column (rows i mod 4) so a warp keeps 8
      // independent DFMA chains in flight; rows come in pairs, one 16-byte
      // load of each of g', dx, u per pair.
      double u0 = 0.0, w0 = 0.0, u1 = 0.0, w1 = 0.0;
      {
        const double* G = rowv;
        const double* DX = rowv + LD;
        const double* U = rowv + 2 * LD;
        double wa[4] = {0.0, 0.0, 0.0, 0.0}, wb[4] = {0.0, 0.0, 0.0, 0.0};
        static_assert(BLK3 || RR % 2 == 0, "register rows in pairs");
        if constexpr (BLK3) {
          hpass_blk3(l, h1, c0, c1, own1, w0, w1);
        } else {
#pragma unroll
        for (int i = 0; i < RR; i += 2) {
          const double2 g2 = *reinterpret_cast<const double2*>(G + i);
          const double2 x2 = *reinterpret_cast<const double2*>(DX + i);
          const double2 u2 = *reinterpret_cast<const double2*>(U + i);
          h0[i] = fma(x2.x, a0, fma(u2.x, b0, h0[i]));
          h0[i + 1] = fma(x2.y, a0, fma(u2.y, b0, h0[i + 1]));
          wa[i & 3] = fma(h0[i], g2.x, wa[i & 3]);
          wa[(i + 1) & 3] = fma(h0[i + 1], g2.y, wa[(i + 1) & 3]);
          if constexpr (!SEQ) {  // (SEQ: d <= 32, no second column)
            h1[i] = fma(x2.x, a1, fma(u2.x, b1, h1[i]));
            h1[i + 1] = fma(x2.y, a1, fma(u2.y, b1, h1[i + 1]));
            wb[i & 3] = fma(h1[i], g2.x, wb[i & 3]);
            wb[(i + 1) & 3] = fma(h1[i + 1], g2.y, wb[(i + 1) & 3]);
          }
        }
        {
          // rows RR.. from shared memory, SR per step with every load issued
          // before the arithmetic (the loads' latency overlaps)
          constexpr int SR = WideShape<Obj, W>::SR;  // shared-memory rows per step
          static_assert(SR == 2 || SR == 4, "rows in pairs, four accumulators per column");
          int i = RR;
  #pragma unroll
          for (; i + SR - 1 < (D > 0 ? D : d); i += SR) {
            double2 g2[SR / 2], x2[SR / 2], u2[SR / 2];
            double e0[SR], e1[SR];
            double* hr = Hs + (i - RR) * LD;
  #pragma unroll
            for (int r = 0; r < SR / 2; ++r) {
              g2[r] = *reinterpret_cast<const double2*>(G + i + 2 * r);
              x2[r] = *reinterpret_cast<const double2*>(DX + i + 2 * r);
              u2[r] = *reinterpret_cast<const double2*>(U + i + 2 * r);
            }
  #pragma unroll
            for (int r = 0; r < SR; ++r) {
              e0[r] = hr[r * LD + c0];
              e1[r] = hr[r * LD + c1];
            }
  #pragma unroll
            for (int r = 0; r < SR; ++r) {
              const double xr = (r & 1) ? x2[r / 2].y : x2[r / 2].x;
              const double ur = (r & 1) ? u2[r / 2].y : u2[r / 2].x;
              const double gr = (r & 1) ? g2[r / 2].y : g2[r / 2].x;
              e0[r] = fma(xr, a0, fma(ur, b0, e0[r]));
              e1[r] = fma(xr, a1, fma(ur, b1, e1[r]));
              hr[r * LD + c0] = e0[r];
              hr[r * LD + c1] = e1[r];
              wa[r] = fma(e0[r], gr, wa[r]);
              wb[r] = fma(e1[r], gr, wb[r]);
            }
          }
  #pragma unroll 1
          for (; i < (D > 0 ? D : d); ++i) {  // (the < SR remainder rows)
            double* hr = Hs + (i - RR) * LD;
            const double e0 = fma(DX[i], a0, fma(U[i], b0, hr[c0]));
            const double e1 = fma(DX[i], a1, fma(U[i], b1, hr[c1]));
            hr[c0] = e0;
            hr[c1] = e1;
            wa[0] = fma(e0, G[i], wa[0]);
            wb[0] = fma(e1, G[i], wb[0]);
          }
        }
        w0 = (wa[0] + wa[1]) + (wa[2] + wa[3]);
        w1 = (wb[0] + wb[1]) + (wb[2] + wb[3]);
        }
        // u = H_k dg = H_k g' - H_k g = w + p: p = -H_k g is this iteration's
        // direction (exact in exact arithmetic), so the pass needs one matvec
        u0 = w0 + p0;
        u1 = w1 + p1;
        if (!own0) u0 = w0 = 0.0;
        if (!own1) u1 = w1 = 0.0;
      }

      // ---- one 8-value reduction: norms, curvature and the p' scalars
      const double dx0 = own0 ? xn0 - x0 : 0.0, dx1 = own1 ? xn1 - x1 : 0.0;
      double part[8];
      part[0] = fma(gn1, gn1, gn0 * gn0);
      part[1] = fma(dx1, dg1, dx0 * dg0);
      part[2] = fma(dx1, dx1, dx0 * dx0);
      part[3] = fma(dg1, dg1, dg0 * dg0);
      part[4] = fma(dg1, u1, dg0 * u0);
      part[5] = fma(u1, gn1, u0 * gn0);
      part[6] = fma(dx1, gn1, dx0 * gn0);
      part[7] = fma(w1, gn1, w0 * gn0);
      team_sum8(part, l);  // W > 1: its barrier also ends every read of rowv
      const double curv = part[1];
      // 1/curv issued next to the guard's straight-line form (the same
      // decision as the reference expression, without its square roots)
      const double rinv = 1.0 / curv;
      pending = curvature_update_sl(curv, part[2], part[3]);  // bfgs.py:69-71
      if constexpr (W == 1) __syncwarp();  // rowv (dx/u of the previous iteration) consumed
      {
        const double rho = pending ? rinv : 0.0;
        const double cc = pending ? fma(rho * rho, part[4], rho) : 0.0;
        const double ug = part[5], xg = part[6];
        double q0 = -w0, q1 = -w1;
        a0 = b0 = a1 = b1 = 0.0;  // skipped update (bfgs.py:69-71): the pass adds 0
        double rx0 = 0.0, ru0 = 0.0, rx1 = 0.0, ru1 = 0.0;
        if (pending) {
          // p' = -(w - rho dx (u.g') - rho u (dx.g') + c dx (dx.g'))
          q0 = -(w0 + fma(dx0, fma(cc, xg, -rho * ug), -rho * xg * u0));
          q1 = -(w1 + fma(dx1, fma(cc, xg, -rho * ug), -rho * xg * u1));
          a0 = fma(cc, dx0, -rho * u0);
          b0 = -rho * dx0;
          a1 = fma(cc, dx1, -rho * u1);
          b1 = -rho * dx1;
          rx0 = dx0, ru0 = u0, rx1 = dx1, ru1 = u1;
        }
        if (own0) {
          rowv[LD + c0] = rx0;
          rowv[2 * LD + c0] = ru0;
        }
        if (own1) {
          rowv[LD + c1] = rx1;
          rowv[2 * LD + c1] = ru1;
        }
        if constexpr (BLK3) {  // the pass reads every column's (a, b) here
          *reinterpret_cast<double2*>(rowv + 4 * LD + 2 * c0) = make_double2(a0, b0);
          if (own1) *reinterpret_cast<double2*>(rowv + 4 * LD + 2 * c1) = make_double2(a1, b1);
        }
        if (!own0) q0 = 0.0;
        if (!own1) q1 = 0.0;
        p0 = q0;
        p1 = q1;
        pd_part = fma(gn1, q1, gn0 * q0);
      }
      // x, g <- x_new, g_new (bfgs.py:141-145)
      x0 = xn0;
      x1 = xn1;
      g0 = gn0;
      g1 = gn1;
      f0 = f_new;
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[a] = acc_new[a];
      gsq = part[0];
      ++k;
      if constexpr (W == 1) __syncwarp();
      if (A.stop_flag && team_any(*(volatile int*)A.stop_flag != 0)) {
        status = ZEUS_STOPPED;
        break;
      }
    }

  done:
    const zeus_bfgs_out& o = A.out;
    if (own0) o.x_final[(int64_t)c0 * o.ld_out + s] = x0;
    if (own1) o.x_final[(int64_t)c1 * o.ld_out + s] = x1;
    if (o.rows) {
      if (own0) o.rows[(int64_t)s * o.ld_rows + c0] = x0;
      if (own1) o.rows[(int64_t)s * o.ld_rows + c1] = x1;
    }
    if (wi == 0 && l == 0) {
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
    team_sync();
  }
};

template <class Obj, int RR, int W, int D, bool TM>
__global__ void __launch_bounds__(TM ? 32 * kTmWarps : kWideThreads,
                                  TM ? WideShape<Obj, W>::TM_CTAS
                                     : (W == 1 && D > 0 && D <= 32) ? WideShape<Obj, 1>::SEQ_MINB
                                                                    : WideShape<Obj, W>::MINB)
    bfgs_wide_kernel(BfgsArgs A) {
  extern __shared__ double sm[];
  const int l = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* alpha_tab = sm;
  __shared__ uint32_t tm_slot;
  if (threadIdx.x == 0) {
    double a = A.alpha0;  // alpha0 * shrink^t by repeated multiplication (linesearch.py:70)
    for (int t = 0; t < A.nalpha; ++t) {
      alpha_tab[t] = a;
      a *= A.shrink;
    }
  }
  if constexpr (TM) {
    if (wib == 0) tmem::alloc(&tm_slot, WideShape<Obj, W>::TM_COLS);
    tmem::fence_before_sync();
  }
  __syncthreads();
  WideStart<Obj, RR, W, D, TM> S;
  if constexpr (TM) {
    tmem::fence_after_sync();
    // this warp's lane quarter (TMEM address: lane << 16 | column)
    S.tm = tm_slot + ((uint32_t)(wib & 3) * 32u << 16);
  }
  const int start_slot = wib / W;  // W = 1: independent starts per block
  S.wi = wib % W;
  S.atab = alpha_tab;
  S.rowv = sm + A.nalpha + (size_t)start_slot * A.warp_doubles;
  S.Hs = S.rowv + 4 * 64 * W;
  // TM: rowv, the (a, b) by column and then the exchange scratch
  S.xch = TM ? S.rowv + 6 * 64 * W : S.Hs + (size_t)(A.d > RR ? A.d - RR : 0) * 64 * W;
  S.bar_id = 1 + start_slot;  // (used when several multi-warp starts share the CTA)
  __shared__ long long next[kTmWarps];
  for (;;) {
    long long s = 0;
    if constexpr (W == 1) {
      if (l == 0) s = (long long)atomicAdd(A.work, 1ull);
      s = __shfl_sync(kFull, s, 0);
    } else {
      if (S.wi == 0 && l == 0) next[start_slot] = (long long)atomicAdd(A.work, 1ull);
      S.team_sync();
      s = next[start_slot];
      S.team_sync();
    }
    if (s >= A.n) break;
    S.run(A, s, l);
  }
  if constexpr (TM) {
    tmem::wait_st();
    tmem::fence_before_sync();
    __syncthreads();
    if (wib == 0) tmem::dealloc(tm_slot, WideShape<Obj, W>::TM_COLS);
  }
}

namespace {

template <class Obj, int RR, int W, int D, bool TM = false>
int launch_wide(BfgsArgs A, cudaStream_t s) {
  A.nalpha = kAlphaTable;
  const int threads = TM ? 32 * kTmWarps : kWideThreads;
  // per start: rowv only (TM: the H rows are in Tensor Memory), else the full slice
  // (d <= 32: 64 more doubles, the SEQ folds' second scratch row)
  // TM: rowv [4][64 W] + (a, b) by column [64 W][2] + the W > 1 exchange scratch
  A.warp_doubles = TM ? ((6 * 64 * W + (W > 1 ? 19 * W : 0) + 1) & ~1)
                      : wide_slot_doubles(A.d, RR, W) + (A.d <= 32 ? 64 : 0);
  const int starts_per_block = threads / 32 / W;
  const size_t smem =
      sizeof(double) * ((size_t)A.nalpha + (size_t)starts_per_block * A.warp_doubles);
  auto kern = bfgs_wide_kernel<Obj, RR, W, D, TM>;
  int rc = check_cuda(
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
      "cudaFuncSetAttribute(wide)");
  if (rc) return rc;
  int per_sm = 0;
  rc = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem),
                  "occupancy(wide)");
  if (rc) return rc;
  // TM: the CTAs per SM whose TMEM allocations fit the SM's 512 columns (the
  // occupancy API reports 1 for kernels that allocate TMEM)
  if (TM) per_sm = WideShape<Obj, W>::TM_CTAS;
  const int sms = current_sm_count();
  if (per_sm < 1 || sms < 1) return set_error(ZEUS_ERR_UNSUPPORTED, "bfgs wide: does not fit");
  int64_t grid = (int64_t)per_sm * sms;
  const int64_t need = (A.n + starts_per_block - 1) / starts_per_block;
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, threads, smem, s>>>(A);
  return check_launch("bfgs_wide_kernel");
}

#ifdef ZEUS_WIDE_RR_OVERRIDE
#define ZEUS_WIDE_RR_OF(Obj, W) ZEUS_WIDE_RR_OVERRIDE
#else
#define ZEUS_WIDE_RR_OF(Obj, W) WideShape<Obj, W>::RR
#endif

struct WideLaunch {
  template <class Obj>
  static int run(BfgsArgs A, cudaStream_t s) {
    if constexpr (Obj::kId == ZEUS_OBJ_GOLDSTEIN_PRICE) {
      return set_error(ZEUS_ERR_UNSUPPORTED, "wide: goldstein_price is 2-D");
    } else {
      // the BASELINE dimensions get kernels compiled for them (T50 and
      // config 3: d = 50; config 4: d = 100); any other 32 < d <= 128 runs
      // the generic build.  d = 50: the block layout with the H elements
      // beyond the register rows in Tensor Memory (SM-cycles per
      // start-iteration, TMEM block layout / shared-memory rows: Rosenbrock
      // 448 / 628, Rastrigin 1,062 / 1,251, Ackley 1,120 / 1,341)
#ifndef ZEUS_WIDE_NO_TMEM
      // (ZEUS_NO_TMEM=1: the shared-memory kernels, for compute-sanitizer's
      // synccheck, which flags every tcgen05.alloc -- csrc/tools/tmem_synccheck.cu)
      const char* no_tm = getenv("ZEUS_NO_TMEM");
      const bool tmem_ok = !(no_tm && no_tm[0] && no_tm[0] != '0');
      if (A.d == 50 && tmem_ok) return launch_wide<Obj, WideShape<Obj, 1>::RR_TM, 1, 50, true>(A, s);
#endif
      if constexpr (Obj::kId != ZEUS_OBJ_ACKLEY)  // config 5 (Ackley: the warp kernel)
        if (A.d == 20) return launch_wide<Obj, 20, 1, 20>(A, s);
      if (A.d == 50) return launch_wide<Obj, ZEUS_WIDE_RR_OF(Obj, 1), 1, 50>(A, s);
      if (A.d <= 64) return launch_wide<Obj, ZEUS_WIDE_RR_OF(Obj, 1), 1, 0>(A, s);
#ifndef ZEUS_WIDE_NO_TMEM
      if (A.d == 100 && tmem_ok) return launch_wide<Obj, WideShape<Obj, 2>::RR_TM, 2, 100, true>(A, s);
#endif
      if (A.d == 100) return launch_wide<Obj, ZEUS_WIDE_RR_OF(Obj, 2), 2, 100>(A, s);
      return launch_wide<Obj, ZEUS_WIDE_RR_OF(Obj, 2), 2, 0>(A, s);
    }
  }
};

}  // namespace

bool bfgs_wide_covers(int obj, int d) {
  return obj != ZEUS_OBJ_GOLDSTEIN_PRICE &&
         ((d > 32 && d <= 128) || (d == 20 && obj != ZEUS_OBJ_ACKLEY));
}

int launch_bfgs_wide(int obj, BfgsArgs A, cudaStream_t s) {
  return dispatch_objective<WideLaunch>(obj, A, s);
}

}  // namespace zeus
