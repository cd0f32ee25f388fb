// bfgs_thread.cu -- host launch of the thread-per-start BFGS tier (kernels in
// bfgs_thread.cuh).
#include "bfgs_thread.cuh"

namespace zeus {

namespace {

template <class Obj, int D>
int launch_thread_d(BfgsArgs A, cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)tri_size<D>() * kThreadBlock;
  auto kern = bfgs_thread_kernel<Obj, D>;
  int rc = check_cuda(
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
      "cudaFuncSetAttribute(thread)");
  if (rc) return rc;
  int per_sm = 0;
  rc = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreadBlock, smem),
                  "occupancy(thread)");
  if (rc) return rc;
  const int sms = current_sm_count();
  if (per_sm < 1 || sms < 1) return set_error(ZEUS_ERR_UNSUPPORTED, "bfgs thread: does not fit");
  int64_t grid = (int64_t)per_sm * sms;
  const int64_t need = (A.n + kThreadBlock - 1) / kThreadBlock;
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, kThreadBlock, smem, s>>>(A);
  return check_launch("bfgs_thread_kernel");
}

struct ThreadLaunch {
  template <class Obj>
  static int run(BfgsArgs A, cudaStream_t s) {
    const int d = A.d;
    if constexpr (Obj::kId == ZEUS_OBJ_GOLDSTEIN_PRICE) {
      return launch_thread_d<Obj, 2>(A, s);
    } else {
      if (d <= 2) return launch_thread_d<Obj, 2>(A, s);
      if (d <= 4) return launch_thread_d<Obj, 4>(A, s);
      if (d <= 8) return launch_thread_d<Obj, 8>(A, s);
      if (d <= 10) return launch_thread_d<Obj, 10>(A, s);
      if (d <= 16) return launch_thread_d<Obj, 16>(A, s);
      return set_error(ZEUS_ERR_UNSUPPORTED, "bfgs thread: d=%d > 16", d);
    }
  }
};

}  // namespace

bool bfgs_thread_covers(int obj, int d) { return d >= 1 && d <= 16; }

int launch_bfgs_thread(int obj, BfgsArgs A, cudaStream_t s) {
  return dispatch_objective<ThreadLaunch>(obj, A, s);
}

}  // namespace zeus
