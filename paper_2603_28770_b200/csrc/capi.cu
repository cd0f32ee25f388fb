// capi.cu -- library plumbing plus the small kernels behind the C ABI:
// Philox uniforms (streams.py), batched objective values / gradients
// (objectives.py, autodiff.py), reduce_best (driver.py:115-134) and the
// cross-shard min-loc select (pso.py:73-76 across GPUs).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "objectives.cuh"
#include "zeus_internal.h"

namespace zeus {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int current_sm_count() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return sms;
}

// ---------------------------------------------------------------------------
__global__ void philox_uniform_kernel(uint64_t seed, int64_t i0, int64_t n, uint64_t k0,
                                      int64_t count, double low, double range, double* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * count) return;
  const int64_t r = t / count, c = t % count;
  uint64_t buf[4];
  const uint64_t k = k0 + (uint64_t)c;
  Philox4x64::block(k >> 2, seed, (uint64_t)(i0 + r), buf);
  const unsigned q = (unsigned)(k & 3);
  const uint64_t u = q == 0 ? buf[0] : q == 1 ? buf[1] : q == 2 ? buf[2] : buf[3];
  out[t] = uniform_draw(u, low, range);
}

template <class Obj>
__global__ void objective_value_kernel(int d, int64_t n, const double* x, int64_t ldx,
                                       double* f) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc[Obj::NACC];
  bool err = false;
  const double v = value_seq<Obj>(StridedX{x + i, ldx}, d, acc, err);
  f[i] = err ? __longlong_as_double(0x7ff8000000000000LL) : v;
}

template <class Obj>
__global__ void objective_gradient_kernel(int d, int64_t n, const double* x, int64_t ldx,
                                          double* g, uint8_t* domain_error) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const StridedX X{x + i, ldx};
  double acc[Obj::NACC];
  bool err = false;
  value_seq<Obj>(X, d, acc, err);  // real parts shared by every tangent pass
  err = false;
  for (int k = 0; k < d; ++k) {
    bool oor = false;
    const double gk = Obj::template grad<AutoMath>(X, k, d, acc, err, oor);
    g[(int64_t)k * ldx + i] = err ? __longlong_as_double(0x7ff8000000000000LL) : gk;
  }
  if (domain_error) domain_error[i] = err ? 1 : 0;
}

struct ValueLaunch {
  template <class Obj>
  static int run(int d, int64_t n, const double* x, int64_t ldx, double* f, cudaStream_t s) {
    const int B = 128;
    objective_value_kernel<Obj><<<(unsigned)((n + B - 1) / B), B, 0, s>>>(d, n, x, ldx, f);
    return check_launch("objective_value_kernel");
  }
};
struct GradientLaunch {
  template <class Obj>
  static int run(int d, int64_t n, const double* x, int64_t ldx, double* g, uint8_t* e,
                 cudaStream_t s) {
    const int B = 128;
    objective_gradient_kernel<Obj>
        <<<(unsigned)((n + B - 1) / B), B, 0, s>>>(d, n, x, ldx, g, e);
    return check_launch("objective_gradient_kernel");
  }
};

// ---------------------------------------------------------------------------
// reduce_best (driver.py:115-134): valid = status != domain_error && !isnan(f)
constexpr int kArgminBlock = 256;
constexpr int kArgminMaxBlocks = 1024;

__global__ void reduce_best_partial(int64_t n, int64_t i0, const double* f,
                                    const uint8_t* status, double* pf, long long* pi,
                                    unsigned long long* tallies) {
  __shared__ unsigned int cnt[4];
  if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
  __syncthreads();
  double bf = 0.0;
  long long bi = -1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t st = status[i];
    if (st < 4) atomicAdd(&cnt[st], 1u);
    const double v = f[i];
    if (st == ZEUS_DOMAIN_ERROR || isnan(v)) continue;
    if (argmin_better(v, i0 + i, bf, bi)) {
      bf = v;
      bi = i0 + i;
    }
  }
  block_argmin<kArgminBlock>(bf, bi);
  if (threadIdx.x == 0) {
    pf[blockIdx.x] = bf;
    pi[blockIdx.x] = bi;
  }
  __syncthreads();
  if (threadIdx.x < 4 && tallies && cnt[threadIdx.x])
    atomicAdd(&tallies[threadIdx.x], (unsigned long long)cnt[threadIdx.x]);
}

__global__ void reduce_best_final(int nb, const double* pf, const long long* pi, double* best) {
  double bf = 0.0;
  long long bi = -1;
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (argmin_better(pf[b], pi[b], bf, bi)) {
      bf = pf[b];
      bi = pi[b];
    }
  block_argmin<kArgminBlock>(bf, bi);
  if (threadIdx.x == 0) {
    best[0] = bi < 0 ? __longlong_as_double(0x7ff8000000000000LL) : bf;
    best[1] = (double)bi;
  }
}

// ---------------------------------------------------------------------------
// min-loc across shards: cands[c] = [f, idx, x...]; np.argmin order.
__global__ void minloc_select_kernel(int d, int ncand, const double* cands, double* gX,
                                     double* gbest) {
  __shared__ int win;
  if (threadIdx.x < 32) {
    double bf = 0.0;
    long long bi = -1;
    int bc = -1;
    for (int c = threadIdx.x; c < ncand; c += 32) {
      const double f = cands[(int64_t)c * (d + 2)];
      const long long idx = (long long)cands[(int64_t)c * (d + 2) + 1];
      if (idx >= 0 && argmin_better(f, idx, bf, bi)) {
        bf = f;
        bi = idx;
        bc = c;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double of = __shfl_down_sync(kFull, bf, o);
      const long long oi = __shfl_down_sync(kFull, bi, o);
      const int oc = __shfl_down_sync(kFull, bc, o);
      if (argmin_better(of, oi, bf, bi)) {
        bf = of;
        bi = oi;
        bc = oc;
      }
    }
    if (threadIdx.x == 0) {
      win = bc;
      gbest[0] = bf;
      gbest[1] = (double)bi;
    }
  }
  __syncthreads();
  if (win < 0) return;
  for (int k = threadIdx.x; k < d; k += blockDim.x) gX[k] = cands[(int64_t)win * (d + 2) + 2 + k];
}

// bench.py:131-141 count_within over SoA final points: |x_i - optimum|_2 < radius
__global__ void count_within_kernel(int d, int64_t n, const double* x, int64_t ldx,
                                    const double* opt, double radius, unsigned long long* count) {
  unsigned c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double e = x[(int64_t)k * ldx + i] - opt[k];
      s = s + e * e;
    }
    c += sqrt(s) < radius ? 1u : 0u;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

// Result hand-off (driver.py:244-265 returns per_run as a list of outcomes):
// the per-start SoA outputs packed into two row-major host-ready tables in one
// pass -- fpack[i][0..d) = x_final, [d] = f_final, [d + 1] = grad_norm;
// ipack[i] = {iterations, status, ls_trials, grad_evals} -- plus the scalar
// table spack = {tallies[4], pso best f, best[0 .. nbest)}.  A 32-start x 32-
// column tile goes through shared memory so the SoA reads (along starts) and
// the row writes (along columns) are both coalesced.
constexpr int kPackTile = 32;
__global__ void pack_results_kernel(zeus_bfgs_out o, int d, int64_t n, double* fpack,
                                    int32_t* ipack, const unsigned long long* tallies,
                                    const double* gbest, const double* best, int nbest,
                                    double* spack) {
  __shared__ double tile[kPackTile][kPackTile + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const int cols = d + 2;
  for (int64_t i0 = (int64_t)blockIdx.x * kPackTile; i0 < n; i0 += (int64_t)gridDim.x * kPackTile) {
    for (int k0 = 0; k0 < cols; k0 += kPackTile) {
      for (int r = ty; r < kPackTile; r += blockDim.y) {  // r: column, tx: start
        const int k = k0 + r;
        const int64_t i = i0 + tx;
        double v = 0.0;
        if (i < n && k < cols)
          v = k < d ? o.x_final[(int64_t)k * o.ld_out + i] : (k == d ? o.f_final[i] : o.grad_norm[i]);
        tile[r][tx] = v;
      }
      __syncthreads();
      for (int r = ty; r < kPackTile; r += blockDim.y) {  // r: start, tx: column
        const int64_t i = i0 + r;
        const int k = k0 + tx;
        if (i < n && k < cols) fpack[i * cols + k] = tile[tx][r];
      }
      __syncthreads();
    }
    const int t = ty * kPackTile + tx;
    if (t < kPackTile && i0 + t < n) {
      const int64_t i = i0 + t;
      int4 q;
      q.x = o.iterations[i];
      q.y = (int)o.status[i];
      q.z = o.ls_trials ? o.ls_trials[i] : 0;
      q.w = o.grad_evals ? o.grad_evals[i] : 0;
      reinterpret_cast<int4*>(ipack)[i] = q;
    }
  }
  if (spack && blockIdx.x == 0 && ty == 0) {
    if (tx < 4) spack[tx] = tallies ? (double)tallies[tx] : 0.0;
    if (tx == 4) spack[4] = gbest ? gbest[0] : __longlong_as_double(0x7ff8000000000000LL);
    for (int j = tx; j < nbest; j += kPackTile) spack[5 + j] = best[j];
  }
}

}  // namespace zeus

using namespace zeus;

extern "C" {

int zeus_abi_version(void) { return ZEUS_ABI_VERSION; }

const char* zeus_last_error(void) { return g_err; }

int zeus_sm_count(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return -1;
  return sms;
}

int zeus_philox_uniform(uint64_t seed, int64_t i0, int64_t n, uint64_t k0, int64_t count,
                        double low, double high, double* out, void* stream) {
  if (n < 0 || count < 0 || i0 < 0 || (!out && n * count > 0))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_philox_uniform: bad arguments");
  if (n * count == 0) return ZEUS_OK;
  const double range = high - low;  // numpy: range = high - low
  const int B = 256;
  const int64_t total = n * count;
  philox_uniform_kernel<<<(unsigned)((total + B - 1) / B), B, 0, as_stream(stream)>>>(
      seed, i0, n, k0, count, low, range, out);
  return check_launch("philox_uniform_kernel");
}

int zeus_objective_value(int obj, int d, int64_t n, const double* x, int64_t ldx, double* f,
                         void* stream) {
  if (d < 1 || n < 0 || ldx < n || (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_objective_value: bad arguments (obj=%d d=%d)",
                     obj, d);
  if (n == 0) return ZEUS_OK;
  const int rc = dispatch_objective<ValueLaunch>(obj, d, n, x, ldx, f, as_stream(stream));
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
}

int zeus_objective_gradient(int obj, int d, int64_t n, const double* x, int64_t ldx,
                            double* grad, uint8_t* domain_error, void* stream) {
  if (d < 1 || n < 0 || ldx < n || (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_objective_gradient: bad arguments");
  if (n == 0) return ZEUS_OK;
  const int rc =
      dispatch_objective<GradientLaunch>(obj, d, n, x, ldx, grad, domain_error, as_stream(stream));
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
}

size_t zeus_argmin_workspace_bytes(int64_t n) {
  (void)n;
  return (size_t)kArgminMaxBlocks * (sizeof(double) + sizeof(long long));
}

int zeus_reduce_best(int64_t n, int64_t i0, const double* f_final, const uint8_t* status,
                     double* best, unsigned long long* tallies, void* workspace,
                     void* stream) {
  if (n < 0 || !best || !workspace) return set_error(ZEUS_ERR_ARGUMENT, "zeus_reduce_best");
  cudaStream_t s = as_stream(stream);
  double* pf = (double*)workspace;
  long long* pi = (long long*)(pf + kArgminMaxBlocks);
  int nb = (int)((n + kArgminBlock - 1) / kArgminBlock);
  if (nb < 1) nb = 1;
  if (nb > kArgminMaxBlocks) nb = kArgminMaxBlocks;
  reduce_best_partial<<<nb, kArgminBlock, 0, s>>>(n, i0, f_final, status, pf, pi, tallies);
  int rc = check_launch("reduce_best_partial");
  if (rc) return rc;
  reduce_best_final<<<1, kArgminBlock, 0, s>>>(nb, pf, pi, best);
  return check_launch("reduce_best_final");
}

int zeus_minloc_select(int d, int ncand, const double* cands, double* gX, double* gbest,
                       void* stream) {
  if (d < 1 || ncand < 1 || !cands || !gX || !gbest)
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_minloc_select: bad arguments");
  minloc_select_kernel<<<1, 128, 0, as_stream(stream)>>>(d, ncand, cands, gX, gbest);
  return check_launch("minloc_select_kernel");
}

int zeus_count_within(int d, int64_t n, const double* x, int64_t ldx, const double* optimum,
                      double radius, unsigned long long* count, void* stream) {
  if (d < 1 || n < 0 || ldx < n || !optimum || !count || (n > 0 && !x))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_count_within: bad arguments");
  if (n == 0) return ZEUS_OK;
  const int B = 256;
  int sms = current_sm_count();
  const int64_t want = (n + B - 1) / B, cap = (int64_t)(sms > 0 ? sms : 148) * 8;
  count_within_kernel<<<(unsigned)(want < cap ? want : cap), B, 0, as_stream(stream)>>>(
      d, n, x, ldx, optimum, radius, count);
  return check_launch("count_within_kernel");
}

int zeus_pack_results(const zeus_bfgs_out* out, int d, int64_t n, double* fpack, int32_t* ipack,
                      const unsigned long long* tallies, const double* gbest, const double* best,
                      int nbest, double* spack, void* stream) {
  if (!out || d < 1 || n < 0 || nbest < 0 || (n > 0 && (!fpack || !ipack || !out->x_final ||
      !out->f_final || !out->grad_norm || !out->iterations || !out->status)) ||
      (spack && nbest > 0 && !best) || (n > 0 && out->ld_out < n) ||
      ((uintptr_t)ipack & 15) != 0)
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_pack_results: bad arguments");
  if (n == 0 && !spack) return ZEUS_OK;
  int sms = current_sm_count();
  const int64_t want = (n + kPackTile - 1) / kPackTile, cap = (int64_t)(sms > 0 ? sms : 148) * 16;
  int64_t grid = want < cap ? want : cap;
  if (grid < 1) grid = 1;
  pack_results_kernel<<<(unsigned)grid, dim3(kPackTile, 8), 0, as_stream(stream)>>>(
      *out, d, n, fpack, ipack, tallies, gbest, best, nbest, spack);
  return check_launch("pack_results_kernel");
}

int zeus_host_device_ptr(void* host, void** dev) {
  if (!host || !dev) return set_error(ZEUS_ERR_ARGUMENT, "zeus_host_device_ptr");
  return check_cuda(cudaHostGetDevicePointer(dev, host, 0), "cudaHostGetDevicePointer");
}

// ---- cross-process early-stop block (driver.py:153-177 across GPUs) --------
// 64 bytes of cudaMalloc'ed device memory: counter (u64) at 0, flag (i32) at 8.
// Its own allocation, so the IPC handle maps exactly this block (torch's
// caching allocator would hand out an offset into a larger segment).
int zeus_ipc_alloc(size_t bytes, void** dptr, unsigned char* handle) {
  if (!dptr || !handle || bytes == 0) return set_error(ZEUS_ERR_ARGUMENT, "zeus_ipc_alloc");
  void* p = nullptr;
  int rc = check_cuda(cudaMalloc(&p, bytes), "cudaMalloc(ipc block)");
  if (rc) return rc;
  rc = check_cuda(cudaMemset(p, 0, bytes), "cudaMemset(ipc block)");
  cudaIpcMemHandle_t h;
  if (!rc) rc = check_cuda(cudaIpcGetMemHandle(&h, p), "cudaIpcGetMemHandle");
  if (rc) {
    cudaFree(p);
    return rc;
  }
  memcpy(handle, &h, sizeof(h));
  *dptr = p;
  return ZEUS_OK;
}

int zeus_ipc_open(const unsigned char* handle, void** dptr) {
  if (!dptr || !handle) return set_error(ZEUS_ERR_ARGUMENT, "zeus_ipc_open");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return check_cuda(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess),
                    "cudaIpcOpenMemHandle");
}

int zeus_ipc_close(void* dptr, int owner) {
  if (!dptr) return ZEUS_OK;
  return owner ? check_cuda(cudaFree(dptr), "cudaFree(ipc block)")
               : check_cuda(cudaIpcCloseMemHandle(dptr), "cudaIpcCloseMemHandle");
}

// Kernels running on `device` may then load / store / atomically update
// memory of `peer` (NVLink / NVSwitch), as the single-process multi-GPU run
// needs for its exchange and stop blocks.  device == peer is a no-op.
int zeus_enable_peer_access(int device, int peer) {
  if (device < 0 || peer < 0) return set_error(ZEUS_ERR_ARGUMENT, "zeus_enable_peer_access");
  if (device == peer) return ZEUS_OK;
  int can = 0;
  int rc = check_cuda(cudaDeviceCanAccessPeer(&can, device, peer), "cudaDeviceCanAccessPeer");
  if (rc) return rc;
  if (!can)
    return set_error(ZEUS_ERR_UNSUPPORTED, "device %d cannot access device %d", device, peer);
  int cur = 0;
  rc = check_cuda(cudaGetDevice(&cur), "cudaGetDevice");
  if (rc) return rc;
  rc = check_cuda(cudaSetDevice(device), "cudaSetDevice");
  if (!rc) {
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled)
      (void)cudaGetLastError();  // clear the sticky-free status
    else
      rc = check_cuda(e, "cudaDeviceEnablePeerAccess");
  }
  cudaSetDevice(cur);
  return rc;
}

int zeus_stop_block_create(void** dptr, unsigned char* handle) {
  return zeus_ipc_alloc(ZEUS_STOP_BLOCK_BYTES, dptr, handle);
}

int zeus_stop_block_open(const unsigned char* handle, void** dptr) {
  return zeus_ipc_open(handle, dptr);
}

int zeus_stop_block_close(void* dptr, int owner) { return zeus_ipc_close(dptr, owner); }

int zeus_stop_block_reset(void* dptr, void* stream) {
  if (!dptr) return set_error(ZEUS_ERR_ARGUMENT, "zeus_stop_block_reset");
  return check_cuda(cudaMemsetAsync(dptr, 0, 16, as_stream(stream)), "reset stop block");
}

}  // extern "C"
