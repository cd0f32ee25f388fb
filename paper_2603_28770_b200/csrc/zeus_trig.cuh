// zeus_trig.cuh -- branch-free double sincos for the objective kernels.
//
// CUDA's cos/sin carry a Payne-Hanek slow path behind a branch, so several
// independent calls in one thread cannot be interleaved by the scheduler;
// the speculative line search evaluates up to 21 x d cosines per iteration
// and was latency-bound on exactly that.  Here the reduction is a 3-constant
// Cody-Waite reduction (exact first step, FMA-exact tail; valid for
// |x| <= kTrigMax, quotient < 2^17) and
// the kernels are the fdlibm / musl __sin / __cos minimax polynomials; both
// polynomials are evaluated and the quadrant selects, so there is no branch.
// Outside |x| <= kTrigMax callers fall back to the libm path (see FastMath).
//
// Accuracy: the reduced argument is carried as a double-double and the
// leading polynomial terms are formed with exact-product corrections, so the
// result is correctly rounded except within a small fraction of an ulp of a
// rounding boundary; near a zero of the function the absolute error stays
// below 1e-27 (what matters inside a sum of terms).
// The GPU parity tests compare objective values built on it against the
// reference / oracle (glibc) values.
//
// Code generation: the polynomial and reduction constants live in a
// __constant__ table, so every DFMA/DMUL takes its constant as a c[] bank
// operand (immediates would be staged through UMOV pairs -- extra issue
// slots and false dependencies on the few uniform registers, which kept
// independent sincos chains from interleaving); rint and the quadrant come
// from one DADD with 1.5 * 2^52 (no FRND / F2I conversion instructions).
#pragma once

#ifndef __CUDACC__
#include <cmath>
#ifndef __host__
#define __host__
#endif
#ifndef __device__
#define __device__
#endif
#ifndef __forceinline__
#define __forceinline__ inline
#endif
#endif

namespace zeus {

constexpr double kTrigMax = 1.0e5;

#ifdef __CUDACC__
// [0] 2/pi, [1..3] pi/2 = PIO2_1 + 1T + 1TT, [4..9] S1..S6, [10..15] C1..C6,
// [16] 2 pi (objectives.py:30 _TWO_PI = 2.0 * math.pi, exact doubling)
static __constant__ double kSinCosTab[17] = {
    0.6366197723675814,    1.5707963267341256,        6.077100506506192e-11,
    3.5215598651832e-27,   -1.66666666666666324348e-01, 8.33333333332248946124e-03,
    -1.98412698298579493134e-04, 2.75573137070700676789e-06, -2.50507602534068634195e-08,
    1.58969099521155010221e-10,  4.16666666666666019037e-02, -1.38888888888741095749e-03,
    2.48015872894767294178e-05,  -2.75573143513906633035e-07, 2.08757232129817482790e-09,
    -1.13596475577881948265e-11, 6.283185307179586};
#endif

// 2 pi as a constant-bank operand on the device (see "Code generation")
__host__ __device__ __forceinline__ double two_pi() {
#ifdef __CUDA_ARCH__
  return kSinCosTab[16];
#else
  return 6.283185307179586;
#endif
}

struct SinCos {
  double s, c;
};

__host__ __device__ __forceinline__ SinCos sincos_fast(double x) {
#ifdef __CUDA_ARCH__
  const double INV_PIO2 = kSinCosTab[0], PIO2_1 = kSinCosTab[1], PIO2_1T = kSinCosTab[2],
               PIO2_1TT = kSinCosTab[3];
  const double S1 = kSinCosTab[4], S2 = kSinCosTab[5], S3 = kSinCosTab[6], S4 = kSinCosTab[7],
               S5 = kSinCosTab[8], S6 = kSinCosTab[9];
  const double C1 = kSinCosTab[10], C2 = kSinCosTab[11], C3 = kSinCosTab[12],
               C4 = kSinCosTab[13], C5 = kSinCosTab[14], C6 = kSinCosTab[15];
  // rint(x * 2/pi) by the 1.5 * 2^52 shifter (round-half-even, |.| < 2^51);
  // the integer's low bits sit in the low mantissa word
  const double shifted = x * INV_PIO2 + 6755399441055744.0;
  const double fn = shifted - 6755399441055744.0;
  const int q = __double2loint(shifted) & 3;
#else
  constexpr double INV_PIO2 = 0.6366197723675814;  // 0x3fe45f306dc9c883
  // pi/2 = PIO2_1 (33 bits: fn * PIO2_1 is exact for |fn| < 2^20) + 1T + 1TT
  constexpr double PIO2_1 = 1.5707963267341256;     // 0x3ff921fb54400000
  constexpr double PIO2_1T = 6.077100506506192e-11;  // 0x3dd0b4611a626331
  constexpr double PIO2_1TT = 3.5215598651832e-27;   // 0x3a71701b839a2520
  // fdlibm k_sin.c / k_cos.c coefficients (Sun Microsystems, public domain)
  constexpr double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
                   S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
                   S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
  constexpr double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
                   C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
                   C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
  const double fn = std::nearbyint(x * INV_PIO2);
  const int q = (int)fn & 3;
#endif
  // reduced argument as a double-double rh + rl (|fn| < 2^17 here)
  const double r0 = x - fn * PIO2_1;  // exact (Sterbenz)
  const double p = fn * PIO2_1T;
  const double pe = fma(fn, PIO2_1T, -p);  // exact product error
  const double rh = r0 - p;
  const double bb = rh - r0;
  const double rl = ((r0 - (rh - bb)) + (-p - bb)) - pe - fn * PIO2_1TT;  // TwoSum error
  // z = (rh + rl)^2 as z + zl
  const double z = rh * rh;
  const double zl = fma(rh, rh, -z) + 2.0 * rh * rl;
  const double w = z * z;
  // sin: rh + S1 rh^3 (double-double) + rh^5 P(z) + rl (1 - z/2)
  const double c3 = z * rh, c3l = fma(z, rh, -c3) + zl * rh;
  const double t1 = c3 * S1, t1l = fma(c3, S1, -t1) + c3l * S1;
  const double sh = rh + t1, sl = t1 - (sh - rh);  // Fast2Sum, |rh| >= |t1|
  const double s5 = c3 * z * fma(z * w, fma(z, S6, S5), fma(z, fma(z, S4, S3), S2));
  const double s = sh + (sl + (t1l + s5 + rl * fma(-0.5, z, 1.0)));
  // cos: 1 - z/2 (exact split) + C1 z^2 (double-double) + z^3 Q(z)
  const double hz = 0.5 * z, a = 1.0 - hz, al = (1.0 - a) - hz;
  const double w_l = fma(z, z, -w) + 2.0 * z * zl;
  const double t2 = w * C1, t2l = fma(w, C1, -t2) + w_l * C1;
  const double ch = a + t2, cl = t2 - (ch - a);  // |a| >= 0.69 > |t2|
  const double c6 = w * z * fma(w * z, fma(z, C6, C5), fma(z, fma(z, C4, C3), C2));
  const double c = ch + (cl + (al - 0.5 * zl + t2l + c6));
  SinCos out;
  out.s = (q == 0) ? s : (q == 1) ? c : (q == 2) ? -s : -c;
  out.c = (q == 0) ? c : (q == 1) ? -s : (q == 2) ? -c : s;
  // tiny arguments: sin x = x (keeps the sign of zero), cos x = 1 (selects,
  // no branch: keeps independent calls interleavable)
  const double ax = x < 0 ? -x : x;
  const bool tiny = ax < 1.4901161193847656e-08;  // 2^-26
  out.s = tiny ? x : out.s;
  out.c = tiny ? 1.0 : out.c;
  return out;
}

// cos alone, bit-identical to sincos_fast(x).c with ONE polynomial chain:
// cos x is +-cos r (q even) or -+sin r (q odd), and the two double-double
// kernels above share their shape -- head + leading correction (rh / 1 - z/2
// with c3 S1 / w C1), a tail polynomial and a low-order term -- so the
// parity of q selects the operands and constants of one evaluation, each
// sum keeping its own kernel's association.  Half the FP64 work of the pair
// for the value-only calls (line-search trials, PSO sweeps).
__host__ __device__ __forceinline__ double cos_fast(double x) {
#ifdef __CUDA_ARCH__
  const double INV_PIO2 = kSinCosTab[0], PIO2_1 = kSinCosTab[1], PIO2_1T = kSinCosTab[2],
               PIO2_1TT = kSinCosTab[3];
  const double shifted = x * INV_PIO2 + 6755399441055744.0;
  const double fn = shifted - 6755399441055744.0;
  const int q = __double2loint(shifted) & 3;
  const bool odd = q & 1;
  const double K1 = odd ? kSinCosTab[4] : kSinCosTab[10], K2 = odd ? kSinCosTab[5] : kSinCosTab[11],
               K3 = odd ? kSinCosTab[6] : kSinCosTab[12], K4 = odd ? kSinCosTab[7] : kSinCosTab[13],
               K5 = odd ? kSinCosTab[8] : kSinCosTab[14], K6 = odd ? kSinCosTab[9] : kSinCosTab[15];
#else
  constexpr double INV_PIO2 = 0.6366197723675814, PIO2_1 = 1.5707963267341256,
                   PIO2_1T = 6.077100506506192e-11, PIO2_1TT = 3.5215598651832e-27;
  const double fn = std::nearbyint(x * INV_PIO2);
  const int q = (int)fn & 3;
  const bool odd = q & 1;
  const double K1 = odd ? -1.66666666666666324348e-01 : 4.16666666666666019037e-02,
               K2 = odd ? 8.33333333332248946124e-03 : -1.38888888888741095749e-03,
               K3 = odd ? -1.98412698298579493134e-04 : 2.48015872894767294178e-05,
               K4 = odd ? 2.75573137070700676789e-06 : -2.75573143513906633035e-07,
               K5 = odd ? -2.50507602534068634195e-08 : 2.08757232129817482790e-09,
               K6 = odd ? 1.58969099521155010221e-10 : -1.13596475577881948265e-11;
#endif
  const double r0 = x - fn * PIO2_1;
  const double p = fn * PIO2_1T;
  const double pe = fma(fn, PIO2_1T, -p);
  const double rh = r0 - p;
  const double bb = rh - r0;
  const double rl = ((r0 - (rh - bb)) + (-p - bb)) - pe - fn * PIO2_1TT;
  const double z = rh * rh;
  const double zl = fma(rh, rh, -z) + 2.0 * rh * rl;
  const double w = z * z;
  // q odd: the sin kernel (head rh, m = c3 = z rh, ml = fma(z, rh, -c3) +
  // zl rh); q even: the cos kernel (head a = 1 - z/2, m = w = z z, ml =
  // fma(z, z, -w) + (2 z) zl) -- selects, no branch
  const double hz = 0.5 * z, a = 1.0 - hz, al = (1.0 - a) - hz;
  const double u = odd ? rh : z, vv = odd ? rh : 2.0 * z;
  const double head = odd ? rh : a;
  const double m = z * u;
  const double ml = fma(z, u, -m) + zl * vv;
  const double e = odd ? rl * fma(-0.5, z, 1.0) : al - 0.5 * zl;
  const double t = m * K1, tl = fma(m, K1, -t) + ml * K1;
  const double hh = head + t, ll = t - (hh - head);
  const double tail = m * z * fma(z * w, fma(z, K6, K5), fma(z, fma(z, K4, K3), K2));
  // sin: (t1l + s5) + rl (1 - z/2);  cos: ((al - zl/2) + t2l) + c6
  const double a1 = odd ? tl : e, a2 = odd ? tail : tl, a3 = odd ? e : tail;
  double r = hh + (ll + ((a1 + a2) + a3));
  r = (q == 1 || q == 2) ? -r : r;
  const double ax = x < 0 ? -x : x;
  return ax < 1.4901161193847656e-08 ? 1.0 : r;  // tiny: cos x = 1
}

__host__ __device__ __forceinline__ bool trig_in_range(double x) {
  return x <= kTrigMax && x >= -kTrigMax;  // false for NaN too
}

}  // namespace zeus
