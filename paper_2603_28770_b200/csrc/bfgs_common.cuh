// bfgs_common.cuh -- pieces shared by the BFGS kernel families (thread, warp
// and CTA-helper tiers in bfgs.cu / bfgs_thread.cu, the wide kernels in
// bfgs_wide.cu): launch arguments, the trial-point accessor, the speculative
// term pass, gradient helpers.
#pragma once
#ifndef __CUDACC_RTC__
#include <algorithm>
#endif

#include "objectives.cuh"
#ifndef __CUDACC_RTC__
#include "zeus_internal.h"
#endif

namespace zeus {

struct BfgsArgs {
  int d;
  int64_t n;
  const double* x0;
  int64_t ldx;
  double theta;
  // largest double q with sqrt(q) < theta (sqrt is correctly rounded and
  // monotone, so |g| < theta <=> |g|^2 <= gsq_max): the convergence test
  // without a sqrt on the iteration's critical path (thread / warp tiers)
  double gsq_max;
  int cap;
  int iter_ls;
  double c1, alpha0, shrink;
  long long required_c;
  unsigned long long* stop_counter;
  int* stop_flag;
  zeus_bfgs_out out;
  unsigned long long* work;
  double* h_global;  // non-null: H lives in HBM/L2 (d too large for smem)
  int warp_doubles;  // shared-memory doubles per warp
  int ldh;           // row stride of an smem/global H
  int tstride;       // term-buffer row stride (odd, >= nterms)
  int bmax;          // max trials per speculative batch
  int nalpha;        // alpha table length (block smem)
  // straggler promotion (small d): a start still running at iteration k1 is
  // handed from one tier to the next through a carry record
  int k1;                          // 0: never promote
  double* carry;                   // [capacity][carry_stride] state records
  int carry_stride;                // doubles per record
  unsigned long long* promo_count; // records written to `carry`
  // resume mode: the kernel consumes carry records written by the previous
  // tier (thread kernel -> warp kernel -> helper-warp kernel)
  const double* carry_in;
  unsigned long long* in_count;    // records available in carry_in
  unsigned long long* in_taken;    // records claimed
  int resume;                      // 1 = consume carry_in records
};

// Carry record layout (doubles): [0] start index, [1] k, [2] ls_trials,
// [3] grads, [4] prev_trials, [5] f0, [6..7] acc, [8] |g|^2, [9] ddir,
// then x[d], g[d], p[d], H[d][d] (row-major, the pending rank-2 update applied).
constexpr int kCarryHead = 10;

#ifndef __CUDACC_RTC__
// host: BfgsArgs::gsq_max for theta (NaN / <= 0: never converges)
inline double gsq_max_for(double theta) {
  if (!(theta > 0.0)) return -1.0;
  if (isinf(theta)) return 1.7976931348623157e308;
  double q = theta * theta;
  while (q > 0.0 && !(sqrt(q) < theta)) q = nextafter(q, 0.0);
  for (;;) {
    const double up = nextafter(q, 1.0 / 0.0);
    if (!(sqrt(up) < theta)) break;
    q = up;
  }
  return q;
}
#endif
__host__ __device__ inline int carry_stride_for(int d) { return kCarryHead + 3 * d + d * d; }

constexpr int kBfgsWarps = 4;
#ifndef ZEUS_TERM_UNROLL
#define ZEUS_TERM_UNROLL 1
#endif
#ifndef ZEUS_MINB
#define ZEUS_MINB 4
#endif
constexpr int kU = ZEUS_TERM_UNROLL;  // independent objective terms per lane per step

// Optional per-phase cycle accounting (build with -DZEUS_PHASE_TIMING): lane 0
// of every warp adds clock64() deltas into zeus_phase_cycles[] (diagnostics
// for the latency probe, scripts/latency_probe.py; off in normal builds).
#ifdef ZEUS_PHASE_TIMING
__device__ unsigned long long zeus_phase_cycles[16];
#define PHASE_T0() long long _pt = clock64()
#define PHASE(i)                                                  \
  do {                                                            \
    __syncwarp();                                                 \
    const long long _n = clock64();                               \
    if (lane == 0) atomicAdd(&zeus_phase_cycles[i], (unsigned long long)(_n - _pt)); \
    _pt = _n;                                                     \
  } while (0)
#else
#define PHASE_T0()
#define PHASE(i)
#endif
constexpr int kTermCap = 320;   // objective terms per speculative batch
constexpr int kAlphaTable = 64;
constexpr int kMaxC = 32;       // columns per lane in the smem / HBM path: d <= 1024

// H slice size in doubles, kept even so the row4 double2 loads stay 16-B aligned
__host__ __device__ inline size_t hsize(int d, int ldh) { return ((size_t)d * ldh + 1) & ~(size_t)1; }


// The optional host-ready row of start s (zeus_bfgs_out.rows / irows): its
// scalar tail (x is written by the coordinate owners next to x_final).
__device__ __forceinline__ void write_row_tail(const zeus_bfgs_out& o, long long s, int d,
                                               double f, double gn, int k, int status,
                                               int ls_trials, int grads) {
  if (!o.rows) return;
  double* r = o.rows + s * o.ld_rows;
  r[d] = f;
  r[d + 1] = gn;
  *reinterpret_cast<int4*>(o.irows + 4 * s) = make_int4(k, status, ls_trials, grads);
}

// Trial-point accessor: coordinate j of x + alpha p (reference: x + alpha*p,
// numpy multiply then add, no contraction).
struct TrialX {
  const double* x;
  const double* p;
  double alpha;
  __device__ __forceinline__ double operator()(int j) const { return x[j] + alpha * p[j]; }
};

// Sum of 8 values over a warp, identical in every lane: a transpose-reduce
// (each level halves the values a lane carries: 4+2+1+1+1 shuffles) followed
// by 8 broadcasts -- 17 double shuffles instead of 40 for 8 butterflies.
// 8 warp sums at once by a transpose-reduce (7 shuffles + 8 broadcasts
// instead of 40).  LANES = 16: only lanes 0..15 hold non-zero values (d <= 16
// column owners), one butterfly level less.  Every lane receives all 8 sums.
template <int LANES = 32>
__device__ __forceinline__ void warp_sum8(double v[8]) {
  static_assert(LANES == 32 || LANES == 16, "warp_sum8: 16 or 32 lanes");
  constexpr int S = LANES / 2;  // first butterfly distance
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & S, b3 = lane & (S / 2), b2 = lane & (S / 4);
  double w4[4], w2[2];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double send = b4 ? v[q] : v[q + 4];
    const double keep = b4 ? v[q + 4] : v[q];
    w4[q] = keep + __shfl_xor_sync(kFull, send, S);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const double send = b3 ? w4[q] : w4[q + 2];
    const double keep = b3 ? w4[q + 2] : w4[q];
    w2[q] = keep + __shfl_xor_sync(kFull, send, S / 2);
  }
  double w1 = (b2 ? w2[1] : w2[0]) + __shfl_xor_sync(kFull, b2 ? w2[0] : w2[1], S / 4);
#pragma unroll
  for (int o = S / 8; o > 0; o >>= 1) w1 += __shfl_xor_sync(kFull, w1, o);
  // lane l now holds value index b2 + 2 b3 + 4 b4
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int src = ((q >> 2) & 1) * S | ((q >> 1) & 1) * (S / 2) | (q & 1) * (S / 4);
    v[q] = __shfl_sync(kFull, w1, src);
  }
}

// 4 warp sums at once (transpose-reduce: 2+1+3 shuffles + 4 broadcasts
// instead of 20 for 4 butterflies), identical in every lane.  Each total is
// bitwise the butterfly warp_sum's: the pairing tree (xor 16, 8, 4, 2, 1) is
// the same, only which lane carries which partial differs.
__device__ __forceinline__ void warp_sum4(double v[4]) {
  const int lane = threadIdx.x & 31;
  const bool b16 = lane & 16, b8 = lane & 8;
  double w2[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const double send = b16 ? v[q] : v[q + 2];
    const double keep = b16 ? v[q + 2] : v[q];
    w2[q] = keep + __shfl_xor_sync(kFull, send, 16);
  }
  double w1 = (b8 ? w2[1] : w2[0]) + __shfl_xor_sync(kFull, b8 ? w2[0] : w2[1], 8);
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) w1 += __shfl_xor_sync(kFull, w1, o);
  // lane l now holds value index b8 + 2 b16
#pragma unroll
  for (int q = 0; q < 4; ++q) v[q] = __shfl_sync(kFull, w1, ((q >> 1) & 1) * 16 | (q & 1) * 8);
}

// Warp sum when only lanes 0..LANES-1 hold non-zero values; all lanes get it.
template <int LANES>
__device__ __forceinline__ double warp_sum_n(double v) {
#pragma unroll
  for (int o = LANES / 2; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  if constexpr (LANES < 32) v = __shfl_sync(kFull, v, 0);
  return v;
}

// Term pass of a batch: (trial b, term j) pairs q = b * nt + j are spread over
// the lanes, four independent terms per lane per step (their libm chains
// overlap); (b, j) advance incrementally, no integer division per term.
// Thread -> first (trial, term) item and the per-step increments of a term
// pass; fixed for a kernel (d fixed), so helper CTAs compute it once.
struct TermIdx {
  int b0, j0, step_b, step_j;
};
template <int NTH>
__device__ __forceinline__ TermIdx term_idx(int nt, int lane) {
  const int step_b = NTH / nt;
  const int b = lane / nt;
  return TermIdx{b, lane - b * nt, step_b, NTH - step_b * nt};
}

template <class Obj, class M, int NTH = 32>
__device__ __forceinline__ void term_pass(int B, int nt, int total, const double* alpha_of,
                                          int d, const double* x, const double* p, double* T,
                                          double* TT, int tstride, int rows, int lane,
                                          bool& oor, const TermIdx* pre = nullptr) {
  const TermIdx ix = pre ? *pre : term_idx<NTH>(nt, lane);
  const int step_b = ix.step_b, step_j = ix.step_j;
  int b = ix.b0, j = ix.j0;
  for (int q0 = lane; q0 < total; q0 += NTH * kU) {
    double t[kU][Obj::NACC], tn[kU][Obj::KT];
    int bb[kU], jj[kU];
#pragma unroll
    for (int r = 0; r < kU; ++r) {
      bb[r] = b;
      jj[r] = j;
      if (q0 + NTH * r < total) {
        if (B > 0) {
          Obj::template term_tan<M>(TrialX{x, p, alpha_of[b]}, j, d, t[r], tn[r], oor);
        } else {
          Obj::template term_tan<M>(DenseX{x}, j, d, t[r], tn[r], oor);
        }
      }
      j += step_j;
      b += step_b;
      while (j >= nt) {  // at most once when NTH >= nt
        j -= nt;
        ++b;
      }
    }
#pragma unroll
    for (int r = 0; r < kU; ++r) {
      if (q0 + NTH * r < total) {
#pragma unroll
        for (int a = 0; a < Obj::NACC; ++a) T[(a * rows + bb[r]) * tstride + jj[r]] = t[r][a];
#pragma unroll
        for (int k = 0; k < Obj::KT; ++k) TT[(k * rows + bb[r]) * tstride + jj[r]] = tn[r][k];
      }
    }
  }
}

// Reference-order fold s + row[0] + row[1] + ... of nt <= MAXT terms with
// every load issued before the add chain (MAXT == 0: runtime loop).
template <int MAXT>
__device__ __forceinline__ double seq_fold(const double* row, int nt, double s) {
  if constexpr (MAXT > 0) {
    double v[MAXT];
#pragma unroll
    for (int j = 0; j < MAXT; ++j) v[j] = j < nt ? row[j] : 0.0;
#pragma unroll
    for (int j = 0; j < MAXT; ++j) {  // the add chain is nt long, not MAXT
      if (j >= nt) break;
      s = s + v[j];
    }
  } else {
    for (int j = 0; j < nt; ++j) s = s + row[j];
  }
  return s;
}

// Evaluate B trial points x + alpha_of[b] p (values AND term tangents);
// lane b < B returns trial b's value and accumulators (reference-order fold).
// B == 0 evaluates x itself.
template <class Obj, int MAXT = 0>
__device__ __forceinline__ double eval_batch(int B, const double* alpha_of, int d,
                                             const double* x, const double* p, double* T,
                                             double* TT, int tstride, int rows, int lane,
                                             double acc[Obj::NACC]) {
  const int nt = Obj::nterms(d);
  const int nb = B > 0 ? B : 1;
  const int total = nb * nt;
  if (total > 0) {
    bool oor = false;
    term_pass<Obj, FastMath>(B, nt, total, alpha_of, d, x, p, T, TT, tstride, rows, lane, oor);
    if (__any_sync(kFull, oor))  // some |2 pi x| > kTrigMax: redo with CUDA libm
      term_pass<Obj, PreciseMath>(B, nt, total, alpha_of, d, x, p, T, TT, tstride, rows, lane,
                                  oor);
  }
  __syncwarp();
  double f = 0.0;
  if (lane < nb) {
#pragma unroll
    for (int a = 0; a < Obj::NACC; ++a) {
      const double* row = T + (a * rows + lane) * tstride;
      acc[a] = seq_fold<MAXT>(row, nt, Obj::init(a, d));
    }
    bool err = false;
    f = Obj::finish(acc, d, err);
  }
  __syncwarp();
  return f;
}

// Gradient component j at xs (fast trig, libm fallback decided warp-wide).
template <class Obj>
__device__ __forceinline__ double grad_at(const double* xs, int j, int d, const double* acc,
                                          bool& err, bool slow) {
  bool oor = false;
  return slow ? Obj::template grad<PreciseMath>(DenseX{xs}, j, d, acc, err, oor)
              : Obj::template grad<FastMath>(DenseX{xs}, j, d, acc, err, oor);
}
template <class Obj>
__device__ __forceinline__ bool grad_needs_slow(const double* xs, int d, int lane) {
  bool oor = false;
  for (int j = lane; j < d; j += 32) oor |= !trig_in_range(kTwoPi * xs[j]);
  return __any_sync(kFull, oor);
}


#ifndef __CUDACC_RTC__
// Launch of the thread-per-start kernel for d <= 16 (bfgs_thread.cu).
int launch_bfgs_thread(int obj, BfgsArgs A, cudaStream_t s);
bool bfgs_thread_covers(int obj, int d);

// Launch of the warp-per-start throughput kernel for 32 < d <= 64 (bfgs_wide.cu).
int launch_bfgs_wide(int obj, BfgsArgs A, cudaStream_t s);
bool bfgs_wide_covers(int obj, int d);

#endif  // __CUDACC_RTC__

}  // namespace zeus
