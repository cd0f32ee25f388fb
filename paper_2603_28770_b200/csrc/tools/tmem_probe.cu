// tmem_probe.cu -- B200 microbenchmark (diagnostic tool, not product code):
// per-thread private storage in TMEM vs shared memory, the question being
// whether the inverse-Hessian rows of the wide BFGS kernel that do not fit in
// registers are cheaper to stream through tcgen05.ld / tcgen05.st than
// through LDS / STS.
//
// Each thread owns NW 32-bit words (NW / 2 doubles) and per pass reads all of
// them, adds a constant, writes them back (the H pass's read-modify-write).
// Reports bytes moved per SM-cycle (read + write) for CTAs of 4 warps, B CTAs
// per SM.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int NW>
__global__ void __launch_bounds__(128) tmem_rmw(int passes, unsigned long long* cyc, float* sink) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  constexpr int NCOL = NW <= 32 ? 32 : NW <= 64 ? 64 : NW <= 128 ? 128 : 256;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&taddr_s)), "n"(NCOL));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = taddr_s + ((uint32_t)(warp & 3) * 32u << 16);
  float acc = 0.f;
  // initialise
  {
    uint32_t r[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) r[q] = __float_as_uint((float)(threadIdx.x + q));
#pragma unroll
    for (int c = 0; c < NW; c += 16)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(base + c),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
  }
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < passes; ++it) {
    // all loads of the pass issued before one wait (as the H pass would)
    uint32_t r[NW];
#pragma unroll
    for (int c = 0; c < NW; c += 16)
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[c + 0]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]), "=r"(r[c + 5]),
            "=r"(r[c + 6]), "=r"(r[c + 7]), "=r"(r[c + 8]), "=r"(r[c + 9]), "=r"(r[c + 10]), "=r"(r[c + 11]),
            "=r"(r[c + 12]), "=r"(r[c + 13]), "=r"(r[c + 14]), "=r"(r[c + 15])
          : "r"(base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int q = 0; q < NW; ++q) r[q] = __float_as_uint(__uint_as_float(r[q]) + 1.0f);
#pragma unroll
    for (int c = 0; c < NW; c += 16)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(base + c),
          "r"(r[c + 0]), "r"(r[c + 1]), "r"(r[c + 2]), "r"(r[c + 3]), "r"(r[c + 4]), "r"(r[c + 5]), "r"(r[c + 6]),
          "r"(r[c + 7]), "r"(r[c + 8]), "r"(r[c + 9]), "r"(r[c + 10]), "r"(r[c + 11]), "r"(r[c + 12]),
          "r"(r[c + 13]), "r"(r[c + 14]), "r"(r[c + 15]));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  const unsigned long long t1 = clock64();
  {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(base));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int q = 0; q < 16; ++q) acc += __uint_as_float(r[q]);
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr_s), "n"(NCOL));
}

// the same read-modify-write on a per-thread shared-memory slice (doubles,
// lane-consecutive: conflict-free, like the wide kernel's H rows)
template <int NW>
__global__ void __launch_bounds__(128) smem_rmw(int passes, unsigned long long* cyc, float* sink) {
  extern __shared__ double sh[];
  constexpr int ND = NW / 2;
  double* my = sh + threadIdx.x;
  for (int q = 0; q < ND; ++q) my[q * 128] = threadIdx.x + q;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < passes; ++it) {
#pragma unroll
    for (int c = 0; c < ND; c += 8) {
      double r[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = my[(c + q) * 128];
#pragma unroll
      for (int q = 0; q < 8; ++q) my[(c + q) * 128] = r[q] + 1.0;
    }
  }
  const unsigned long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = (float)my[0];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


// Latency of one tcgen05.ld.32x32b.x16 -> wait::ld round trip (one warp
// alone), and of st -> ld of the same columns.
__global__ void __launch_bounds__(128) tmem_lat(unsigned long long* out) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&taddr_s)), "n"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = taddr_s;
  uint32_t r[16];
  for (int q = 0; q < 16; ++q) r[q] = q;
  unsigned long long tl = 0, tsl = 0, tw = 0;
  if (warp == 0) {
    for (int it = 0; it < 64; ++it) {
      unsigned long long t0 = clock64();
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(base));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" : "+r"(r[0]), "+r"(r[15]) :: "memory");
      unsigned long long t1 = clock64();
      r[0] += 1;
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(base),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
      unsigned long long t2 = clock64();
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      unsigned long long t3 = clock64();
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(base));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" : "+r"(r[0]), "+r"(r[15]) :: "memory");
      unsigned long long t4 = clock64();
      if (it >= 8) { tl += t1 - t0; tw += t3 - t2; tsl += t4 - t3; }
    }
  }
  if (threadIdx.x == 0) { out[0] = tl / 56; out[1] = tw / 56; out[2] = tsl / 56; out[3] = r[0] + r[15]; }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr_s), "n"(32));
}

template <int NW, bool TM>
int run(int ctas_per_sm, int sms) {
  const int passes = 2000, grid = ctas_per_sm * sms;
  unsigned long long* cyc;
  float* sink;
  CK(cudaMalloc(&cyc, grid * sizeof(unsigned long long)));
  CK(cudaMalloc(&sink, grid * 128 * sizeof(float)));
  size_t smem = TM ? 0 : (size_t)NW / 2 * 128 * sizeof(double);
  if (!TM) CK(cudaFuncSetAttribute(smem_rmw<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int rep = 0; rep < 2; ++rep) {
    if (TM) tmem_rmw<NW><<<grid, 128>>>(passes, cyc, sink);
    else smem_rmw<NW><<<grid, 128, smem>>>(passes, cyc, sink);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
  }
  unsigned long long* h = new unsigned long long[grid];
  CK(cudaMemcpy(h, cyc, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  double mx = 0, mean = 0;
  for (int i = 0; i < grid; ++i) { mx = h[i] > mx ? h[i] : mx; mean += h[i]; }
  mean /= grid;
  // bytes per SM: ctas_per_sm CTAs x 128 threads x NW words x 4 B x 2 (read + write) x passes
  const double bytes = (double)ctas_per_sm * 128 * NW * 4 * 2 * passes;
  printf("%s NW=%3d words/thread  CTAs/SM=%d (%2d warps/SM): %.1f B/clk/SM (read+write), %.2f clk per thread-word RMW (mean %.0f, max %.0f cycles)\n",
         TM ? "TMEM" : "SMEM", NW, ctas_per_sm, 4 * ctas_per_sm, bytes / mx,
         mx / ((double)passes * NW), mean, mx);
  delete[] h;
  cudaFree(cyc);
  cudaFree(sink);
  return 0;
}

int main() {
  int sms = 0;
  {
    unsigned long long* o;
    CK(cudaMalloc(&o, 4 * sizeof(unsigned long long)));
    tmem_lat<<<1, 128>>>(o);
    CK(cudaDeviceSynchronize());
    unsigned long long h[4];
    CK(cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost));
    printf("one warp: ld.x16 + wait::ld %llu clk; wait::st after st.x16 %llu clk; ld.x16 + wait::ld after a waited st %llu clk\n",
           h[0], h[1], h[2]);
    cudaFree(o);
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, true>(1, sms);
  run<64, true>(2, sms);
  run<64, true>(4, sms);
  run<128, true>(1, sms);
  run<128, true>(3, sms);
  run<128, true>(4, sms);
  run<64, false>(1, sms);
  run<64, false>(3, sms);
  run<64, false>(4, sms);
  run<128, false>(1, sms);
  run<128, false>(3, sms);
  return 0;
}
