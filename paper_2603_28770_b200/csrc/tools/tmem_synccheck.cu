// tmem_synccheck.cu -- diagnostic (not product code): is compute-sanitizer's
// synccheck "Barrier error ... Missing init" on the TMEM kernels a property
// of tcgen05.alloc itself?  The kernel below only allocates, fences,
// synchronises and frees Tensor Memory, exactly as bfgs_wide_kernel does.
//   nvcc -gencode arch=compute_100a,code=sm_100a tmem_synccheck.cu -o t
//   compute-sanitizer --tool synccheck ./t
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(128) alloc_only(int* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&slot)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (threadIdx.x == 0) out[blockIdx.x] = (int)slot;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(slot), "n"(128));
}

int main() {
  int* o;
  cudaMalloc(&o, 4 * sizeof(int));
  alloc_only<<<4, 128>>>(o);
  cudaError_t e = cudaDeviceSynchronize();
  int h[4];
  cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  printf("alloc_only: %s, TMEM bases %d %d %d %d\n", cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
  return e == cudaSuccess ? 0 : 1;
}
