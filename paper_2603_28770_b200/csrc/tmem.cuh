// tmem.cuh -- Tensor Memory (TMEM) as per-thread private storage for the
// wide BFGS kernel's inverse-Hessian rows (sm_100a: tcgen05.alloc / ld / st).
//
// TMEM is 128 lanes x 512 columns x 32 bit per SM; warp w of a CTA reaches
// lanes 32 (w % 4) .. 32 (w % 4) + 31, so with 4-warp CTAs every thread owns
// the columns of "its" lane: [base, base + ncols) of the CTA's allocation.
// A .32x32b.x16 access moves 16 consecutive 32-bit columns (8 doubles) per
// thread.  Measured on B200 (csrc/tools/tmem_probe.cu): one .x16 load + wait
// 17 cycles for a warp alone; read-modify-write of 64-128 words per thread
// at 8-16 warps/SM 570-760 B/clk/SM, against the 128 B/clk/SM shared-memory
// data path that bound the shared-memory layout.  Accesses here are .x2 (one
// double = its own register pair): the .x16 vector forms made ptxas shuffle
// registers into and out of the 16-register operand blocks (~200 moves per
// BFGS iteration, measured), a hand-written asm chunk fared worse, and .x4
// (one row's two columns per access) traded the 64 saved accesses for ~100
// register moves around the 4-register operands (Rosenbrock d = 50 +2%); in the block
// layout one .x8 + one .x4 access per two-row group measured +4% too.
#pragma once
#include <cstdint>

namespace zeus {
namespace tmem {

// One warp of the CTA allocates ncols (power of two, >= 32) columns and
// writes the base address to *slot (shared memory); every thread reads it
// after the fence / barrier / fence sequence (tmem_base()).
__device__ __forceinline__ void alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(slot)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void dealloc(uint32_t base, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "r"(ncols));
}
__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// 4 doubles (8 columns) of this thread's lane at column address `a`
__device__ __forceinline__ void st4d(uint32_t a, double v0, double v1, double v2, double v3) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(a),
      "r"(__double2loint(v0)), "r"(__double2hiint(v0)), "r"(__double2loint(v1)),
      "r"(__double2hiint(v1)), "r"(__double2loint(v2)), "r"(__double2hiint(v2)),
      "r"(__double2loint(v3)), "r"(__double2hiint(v3))
      : "memory");
}

// One double (2 columns) per access: the .x2 vector is the double's own
// register pair, so no register shuffling around the access.  ld_issue2 /
// wait_ld8 / value2: issue up to 8 loads, one wait tying their registers,
// then read them.
struct D2 {
  uint32_t lo, hi;
  __device__ __forceinline__ double v() const { return __hiloint2double(hi, lo); }
};
__device__ __forceinline__ void ld2(uint32_t a, D2& d) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(d.lo), "=r"(d.hi) : "r"(a));
}
template <int N>
__device__ __forceinline__ void wait_ld_n(D2 (&d)[N]) {
  static_assert(N == 12 || N == 8 || N == 6 || N == 4, "wait_ld_n: 4, 6, 8 or 12 doubles");
  if constexpr (N == 12)
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(d[0].lo), "+r"(d[0].hi), "+r"(d[1].lo), "+r"(d[1].hi), "+r"(d[2].lo),
                   "+r"(d[2].hi), "+r"(d[3].lo), "+r"(d[3].hi), "+r"(d[4].lo), "+r"(d[4].hi),
                   "+r"(d[5].lo), "+r"(d[5].hi), "+r"(d[6].lo), "+r"(d[6].hi), "+r"(d[7].lo),
                   "+r"(d[7].hi), "+r"(d[8].lo), "+r"(d[8].hi), "+r"(d[9].lo), "+r"(d[9].hi),
                   "+r"(d[10].lo), "+r"(d[10].hi), "+r"(d[11].lo), "+r"(d[11].hi)
                 :
                 : "memory");
  else if constexpr (N == 6)
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(d[0].lo), "+r"(d[0].hi), "+r"(d[1].lo), "+r"(d[1].hi), "+r"(d[2].lo),
                   "+r"(d[2].hi), "+r"(d[3].lo), "+r"(d[3].hi), "+r"(d[4].lo), "+r"(d[4].hi),
                   "+r"(d[5].lo), "+r"(d[5].hi)
                 :
                 : "memory");
  else if constexpr (N == 8)
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(d[0].lo), "+r"(d[0].hi), "+r"(d[1].lo), "+r"(d[1].hi), "+r"(d[2].lo),
                   "+r"(d[2].hi), "+r"(d[3].lo), "+r"(d[3].hi), "+r"(d[4].lo), "+r"(d[4].hi),
                   "+r"(d[5].lo), "+r"(d[5].hi), "+r"(d[6].lo), "+r"(d[6].hi), "+r"(d[7].lo),
                   "+r"(d[7].hi)
                 :
                 : "memory");
  else
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(d[0].lo), "+r"(d[0].hi), "+r"(d[1].lo), "+r"(d[1].hi), "+r"(d[2].lo),
                   "+r"(d[2].hi), "+r"(d[3].lo), "+r"(d[3].hi)
                 :
                 : "memory");
}
__device__ __forceinline__ void st2(uint32_t a, double v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n" ::"r"(a),
               "r"(__double2loint(v)), "r"(__double2hiint(v))
               : "memory");
}

__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

}  // namespace tmem
}  // namespace zeus
