// measure.cu -- FP64 roofline denominator: a DFMA throughput microbenchmark.
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the BFGS kernel is
// bound by the FP64 pipe, so bench.py measures its peak on the box with this
// kernel (8 independent FMA chains per thread, no memory traffic).
#include "zeus_internal.h"

namespace zeus {

__global__ void dfma_peak_kernel(long long iters, double seed, double* sink) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4,
         a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999999, c = 1e-9;
  for (long long i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) sink[blockIdx.x] = s;  // keep the chains alive
}

}  // namespace zeus

using namespace zeus;

extern "C" {

int zeus_bench_dfma(int blocks, int threads, long long iters, double* sink,
                    double* flops_out, void* stream) {
  if (blocks < 1 || threads < 32 || threads > 1024 || iters < 1 || !sink || !flops_out)
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_bench_dfma: bad arguments");
  dfma_peak_kernel<<<blocks, threads, 0, as_stream(stream)>>>(iters, 1.0, sink);
  *flops_out = 2.0 * 32.0 * (double)iters * (double)blocks * (double)threads;
  return check_launch("dfma_peak_kernel");
}

}  // extern "C"
