// zeus_common.cuh -- shared device helpers for the sm_100a Zeus kernels.
//
// The whole library is compiled with -fmad=false: every a*b+c in this tree
// rounds twice, exactly like CPython floats / numpy ufuncs in the reference
// (pso.py:150-157, objectives.py:40-113, linesearch.py:66-67).  Where the
// BFGS linear algebra wants fused multiply-adds (the reference's OpenBLAS
// order is implementation-defined anyway) they are written as explicit fma().
#pragma once
#ifdef __CUDACC_RTC__
// NVRTC (user objectives, plugin.cu): no host headers
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#else
#include <cuda_runtime.h>
#include <stdint.h>
#endif

#include "../../include/zeus_b200.h"

namespace zeus {

constexpr double kTwoPi = 2.0 * 3.141592653589793;  // objectives.py:30 (2.0*math.pi)
constexpr double kE = 2.718281828459045;             // math.e
constexpr double kCurvatureFloor = 1e-12;            // bfgs.py:40

// The curvature guard of bfgs.py:69-71, update <=> !(curv <= floor*|dx|*|dg|)
// with |dx| = sqrt(dxdx), |dg| = sqrt(dgdg), decided without the two square
// roots whenever the squared comparison is clear by a margin far above its
// rounding error (curv^2 vs floor^2 dxdx dgdg, all normal and finite); only
// the near-tie (and under/overflow) case evaluates the reference expression.
// Same decision as the reference expression for every input.
__device__ __forceinline__ bool curvature_update(double curv, double dxdx, double dgdg) {
  constexpr double kMin = 2.2250738585072014e-308, kMax = 1e300;
  const double q = curv * curv;
  const double t = (kCurvatureFloor * kCurvatureFloor) * dxdx;  // every partial normal
  const double r = t * dgdg;
  const bool normal = t >= kMin && t <= kMax && r >= kMin && r <= kMax && q >= kMin && q <= kMax;
  // floor*|dx|*|dg| is finite and >= 0 for finite norms (NaN / inf fall through)
  if (curv <= 0.0 && dxdx <= 1e300 && dgdg <= 1e300) return false;
  if (normal) {
    if (q > r * (1.0 + 1e-9)) return true;
    if (q < r * (1.0 - 1e-9)) return false;
  }
  return !(curv <= kCurvatureFloor * sqrt(dxdx) * sqrt(dgdg));
}
// The same decision with the common case in straight-line code (selects), so
// its arithmetic can interleave with an independent computation issued next
// to it (the 1/curvature division of the BFGS update); only a near tie or an
// out-of-range operand takes the branch to the reference expression.
__device__ __forceinline__ bool curvature_update_sl(double curv, double dxdx, double dgdg) {
  constexpr double kMin = 2.2250738585072014e-308, kMax = 1e300;
  const double q = curv * curv;
  const double t = (kCurvatureFloor * kCurvatureFloor) * dxdx;
  const double r = t * dgdg;
  const bool normal = t >= kMin && t <= kMax && r >= kMin && r <= kMax && q >= kMin && q <= kMax;
  const bool nonpos = curv <= 0.0 && dxdx <= 1e300 && dgdg <= 1e300;
  const bool up = normal && q > r * (1.0 + 1e-9);
  const bool dn = normal && q < r * (1.0 - 1e-9);
  if (nonpos || up || dn) return up && !nonpos;
  return !(curv <= kCurvatureFloor * sqrt(dxdx) * sqrt(dgdg));
}
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// Philox4x64-10, bit-exact with numpy's Philox(key=[seed, i])
// (streams.py:36-45).  u64 draw k of particle i lives in block k/4, which is
// generated from counter (k/4 + 1, 0, 0, 0): numpy increments the counter
// before producing each block.  64x64->128 products via __umul64hi.
// ---------------------------------------------------------------------------
struct Philox4x64 {
  static constexpr uint64_t M0 = 0xD2E7470EE14C6C93ULL;
  static constexpr uint64_t M1 = 0xCA5A826395121157ULL;
  static constexpr uint64_t W0 = 0x9E3779B97F4A7C15ULL;
  static constexpr uint64_t W1 = 0xBB67AE8584CAA73BULL;

  __device__ __forceinline__ static void block(uint64_t b, uint64_t k0, uint64_t k1,
                                               uint64_t out[4]) {
    uint64_t c0 = b + 1, c1 = (b + 1 == 0) ? 1 : 0, c2 = 0, c3 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      if (r) {
        k0 += W0;
        k1 += W1;
      }
      const uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
      const uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
      const uint64_t n0 = hi1 ^ c1 ^ k0;
      const uint64_t n2 = hi0 ^ c3 ^ k1;
      c0 = n0;
      c1 = lo1;
      c2 = n2;
      c3 = lo0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
  }
};

// Sequential reader of one particle's stream: caches the current 4-word block.
struct PhiloxCursor {
  uint64_t seed, key1, cur = ~0ull;
  uint64_t buf[4];
  __device__ PhiloxCursor(uint64_t s, uint64_t i) : seed(s), key1(i) {}
  __device__ __forceinline__ uint64_t at(uint64_t k) {
    const uint64_t b = k >> 2;
    if (b != cur) {
      Philox4x64::block(b, seed, key1, buf);
      cur = b;
    }
    // dynamic register indexing avoided with a select chain
    const unsigned q = (unsigned)(k & 3);
    return q == 0 ? buf[0] : q == 1 ? buf[1] : q == 2 ? buf[2] : buf[3];
  }
};

// numpy next_double: (u64 >> 11) * 2^-53; Generator.uniform: low + range*u
// (no FMA: -fmad=false).
__device__ __forceinline__ double unit_double(uint64_t u) {
  return (double)(u >> 11) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double uniform_draw(uint64_t u, double low, double range) {
  return low + range * unit_double(u);
}

// np.argmin ordering on (value, index): first NaN wins, else smaller value,
// ties to the lower index (pso.py:73-76).  `idx < 0` marks an empty slot.
__device__ __forceinline__ bool argmin_better(double fa, long long ia, double fb,
                                              long long ib) {
  if (ib < 0) return ia >= 0;
  if (ia < 0) return false;
  const bool na = isnan(fa), nb = isnan(fb);
  if (na || nb) return na && nb ? ia < ib : na;
  if (fa < fb) return true;
  if (fb < fa) return false;
  return ia < ib;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Block-wide argmin of (f, idx) pairs; result valid in thread 0.
template <int BLOCK>
__device__ __forceinline__ void block_argmin(double& f, long long& idx) {
  __shared__ double sf[BLOCK / 32];
  __shared__ long long si[BLOCK / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double of = __shfl_down_sync(kFull, f, o);
    const long long oi = __shfl_down_sync(kFull, idx, o);
    if (argmin_better(of, oi, f, idx)) {
      f = of;
      idx = oi;
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    sf[w] = f;
    si[w] = idx;
  }
  __syncthreads();
  if (w == 0) {
    f = lane < BLOCK / 32 ? sf[lane] : 0.0;
    idx = lane < BLOCK / 32 ? si[lane] : -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double of = __shfl_down_sync(kFull, f, o);
      const long long oi = __shfl_down_sync(kFull, idx, o);
      if (argmin_better(of, oi, f, idx)) {
        f = of;
        idx = oi;
      }
    }
  }
}

}  // namespace zeus
