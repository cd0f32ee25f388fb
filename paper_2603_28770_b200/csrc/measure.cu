// measure.cu -- FP64 roofline denominator: a DFMA throughput microbenchmark.
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the BFGS kernel is
// bound by the FP64 pipe, so bench.py measures its peak on the box with this
// kernel (8 independent FMA chains per thread, no memory traffic).
#include "zeus_internal.h"
#include "zeus_trig.cuh"

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

// ---- dependent-chain latencies (one warp), cycles per operation ----------
namespace zeus {
__global__ void latency_kernel(double seed, long long* out, double* sink) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = seed + lane;
  sm[lane + 32] = seed;
  __syncwarp();
  double a = seed + lane, b = 1.0000001, c = 1e-9;
  const int N = 256;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) a = fma(a, b, c);
  t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / N;
  // DADD chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) a = a + c;
  t1 = clock64();
  if (lane == 0) out[1] = (t1 - t0) / N;
  // SHFL (double) chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1);
  t1 = clock64();
  if (lane == 0) out[2] = (t1 - t0) / N;
  // LDS dependent chain (index from loaded value)
  int idx = lane;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) idx = ((int)sm[idx & 63]) & 63;
  t1 = clock64();
  if (lane == 0) out[3] = (t1 - t0) / N;
  // sqrt chain
  double s = a + 2.0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) s = sqrt(s) + 1.5;
  t1 = clock64();
  if (lane == 0) out[4] = (t1 - t0) / 64;
  // division chain
  double q = a + 3.0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) q = 1.0 / q + 2.0;
  t1 = clock64();
  if (lane == 0) out[5] = (t1 - t0) / 64;
  // cos (CUDA libm) chain
  double cc = a;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) cc = cos(cc) + 0.5;
  t1 = clock64();
  if (lane == 0) out[6] = (t1 - t0) / 64;
  // __syncwarp + ballot round trip
  unsigned m = 0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) m += __ballot_sync(0xffffffffu, (a + m) > 0.5);
  t1 = clock64();
  if (lane == 0) out[7] = (t1 - t0) / N;
  // branch-free sincos chain, then 4 independent chains (ILP)
  double f1 = a;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) f1 = sincos_fast(f1).c + 0.5;
  t1 = clock64();
  if (lane == 0) out[8] = (t1 - t0) / 64;
  double g1 = a, g2 = a + 1, g3 = a + 2, g4 = a + 3;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
    g1 = sincos_fast(g1).c + 0.5;
    g2 = sincos_fast(g2).c + 0.5;
    g3 = sincos_fast(g3).c + 0.5;
    g4 = sincos_fast(g4).c + 0.5;
  }
  t1 = clock64();
  if (lane == 0) out[9] = (t1 - t0) / 64;
  sink[lane] = a + s + q + cc + idx + m + f1 + g1 + g2 + g3 + g4;
}
}  // namespace zeus

extern "C" int zeus_bench_latency(long long* out_host, void* stream) {
  long long* d = nullptr;
  double* sink = nullptr;
  cudaMalloc(&d, 10 * sizeof(long long));
  cudaMalloc(&sink, 32 * sizeof(double));
  zeus::latency_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(1.25, d, sink);
  int rc = zeus::check_launch("latency_kernel");
  cudaMemcpy(out_host, d, 10 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  cudaFree(sink);
  return rc;
}
