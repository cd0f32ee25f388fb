// plugin.cu -- user-defined objectives on the GPU path (
// the reference accepts any generic-scalar Python callable, pkg/README.md:70-87).
//
// A plugin is device source for `objective<T>(x, d, data, err)` (contract in
// user_objective.cuh).  zeus_user_compile builds ONE NVRTC program per
// (source, d): user_objective.cuh + the user text + user_program.cuh, which
// instantiates the framework's own PSO kernels (pso_kernels.cuh) and
// thread-per-start BFGS kernel (bfgs_thread.cuh) for the adapter UserObj, at
// -arch=sm_100a with -fmad=false like the rest of the library.  The module is
// loaded into the current context and launched with the driver API; the
// kernels' host-side logic (grid sizing, candidates, work counters) mirrors
// pso.cu / bfgs_thread.cu.  d <= 16 (the thread-per-start tier; H lives in
// shared memory).
#include <cuda.h>
#include <nvrtc.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "bfgs_plan.h"
#include "zeus_internal.h"

namespace zeus {
namespace {

constexpr int kUserMaxD = 128;
constexpr int kUserThreadMaxD = 16;  // d <= 16: thread per start; above: warp per start
constexpr int kPsoBlockU = 256;   // pso_kernels.cuh kPsoBlock
constexpr int kThreadBlockU = 64; // bfgs_thread.cuh kThreadBlock
constexpr size_t kUserWsHeader = 256;

struct UserPlugin {
  CUmodule mod = nullptr;
  CUfunction pso_init = nullptr, pso_sweep = nullptr, pso_finalize = nullptr, bfgs = nullptr,
             value = nullptr, gradient = nullptr, armijo = nullptr;
  CUdeviceptr data_sym = 0;
  int d = 0;
  bool warp = false;  // bfgs = the warp-per-start kernel (d > kUserThreadMaxD)
  BfgsPlan plan{};    // its sizing
};

// Sizing of the warp-per-start kernel for a user objective: one term with
// d + 2 tangent slots (user_program.cuh); H in registers (DR = the plan's
// bucket, d <= 32) or in the shared-memory slice (d <= 128 always fits one
// warp per CTA).  The NVRTC instance uses the plan's DR.
BfgsPlan user_warp_plan(int d) { return bfgs_plan(d, 1, 1, 0, d + 2); }
int user_warp_dr(int d) { return user_warp_plan(d).dr; }

// per-thread log of the last failed compile (zeus_user_compile_log)
thread_local std::string g_log;

// Driver-API entry points resolved through the runtime (no link-time
// dependency on libcuda.so, so the library still loads on a host without a
// driver -- the CPU tests check its exported symbols).
struct Drv {
  decltype(&cuModuleLoadData) ModuleLoadData = nullptr;
  decltype(&cuModuleGetFunction) ModuleGetFunction = nullptr;
  decltype(&cuModuleGetGlobal) ModuleGetGlobal = nullptr;
  decltype(&cuModuleUnload) ModuleUnload = nullptr;
  decltype(&cuFuncSetAttribute) FuncSetAttribute = nullptr;
  decltype(&cuLaunchKernel) LaunchKernel = nullptr;
  decltype(&cuMemcpyHtoDAsync) MemcpyHtoDAsync = nullptr;
  decltype(&cuMemsetD8Async) MemsetD8Async = nullptr;
  decltype(&cuOccupancyMaxActiveBlocksPerMultiprocessor) Occupancy = nullptr;
  decltype(&cuGetErrorString) GetErrorString = nullptr;
  bool ok = false;
};

template <class F>
bool resolve(const char* name, F& fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  fn = reinterpret_cast<F>(p);
  return true;
}

const Drv& drv() {
  static Drv D = [] {
    Drv d;
    d.ok = resolve("cuModuleLoadData", d.ModuleLoadData) &&
           resolve("cuModuleGetFunction", d.ModuleGetFunction) &&
           resolve("cuModuleGetGlobal", d.ModuleGetGlobal) &&
           resolve("cuModuleUnload", d.ModuleUnload) &&
           resolve("cuFuncSetAttribute", d.FuncSetAttribute) &&
           resolve("cuLaunchKernel", d.LaunchKernel) &&
           resolve("cuMemcpyHtoDAsync", d.MemcpyHtoDAsync) &&
           resolve("cuMemsetD8Async", d.MemsetD8Async) &&
           resolve("cuOccupancyMaxActiveBlocksPerMultiprocessor", d.Occupancy) &&
           resolve("cuGetErrorString", d.GetErrorString);
    return d;
  }();
  return D;
}

int cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return ZEUS_OK;
  const char* msg = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &msg);
  return set_error(ZEUS_ERR_CUDA, "%s: %s", what, msg ? msg : "?");
}

int rtc_check(nvrtcResult r, const char* what) {
  if (r == NVRTC_SUCCESS) return ZEUS_OK;
  return set_error(ZEUS_ERR_CUDA, "%s: %s", what, nvrtcGetErrorString(r));
}

}  // namespace
}  // namespace zeus

using namespace zeus;

extern "C" {

const char* zeus_user_compile_log(void) { return g_log.c_str(); }

int zeus_user_compile(const char* source, int d, const char* include_dir, void** handle) {
  if (!source || !include_dir || !handle || d < 1 || d > kUserMaxD)
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_user_compile: bad arguments (d=%d, max %d)", d,
                     kUserMaxD);
  // the runtime API owns the context (torch / cudaSetDevice); make it current
  int rc = check_cuda(cudaFree(nullptr), "cudaFree(0)");
  if (rc) return rc;
  if (!drv().ok) return set_error(ZEUS_ERR_CUDA, "driver API entry points unavailable");
  std::string prog = "#include \"user_objective.cuh\"\n#line 1 \"user_objective\"\n";
  prog += source;
  prog += "\n#include \"user_program.cuh\"\n";
  nvrtcProgram p;
  rc = rtc_check(nvrtcCreateProgram(&p, prog.c_str(), "zeus_user.cu", 0, nullptr, nullptr),
                 "nvrtcCreateProgram");
  if (rc) return rc;
  char dflag[32], iflag[4096];
  snprintf(dflag, sizeof dflag, "-DZEUS_USER_D=%d", d);
  snprintf(iflag, sizeof iflag, "-I%s", include_dir);
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false",
                        "-lineinfo", dflag, iflag};
  // ZEUS_USER_WARP=1: warp per start for every d (tests compare the two kernels)
  const char* force = getenv("ZEUS_USER_WARP");
  const bool warp = d > kUserThreadMaxD || (force && force[0] == '1');
  const std::string k_bfgs =
      warp ? "zeus::bfgs_warp_kernel<zeus::UserObj, " + std::to_string(user_warp_dr(d)) + ", 0>"
           : "zeus::bfgs_thread_kernel<zeus::UserObj, " + std::to_string(d) + ">";
  const char* names[] = {"zeus::pso_init_kernel<zeus::UserObj>",
                         "zeus::pso_sweep_kernel<zeus::UserObj>", "zeus::pso_finalize_kernel",
                         k_bfgs.c_str(), "zeus::user_value_kernel",
                         "zeus::user_gradient_kernel", "zeus::user_armijo_kernel"};
  constexpr int kNames = 7;
  for (const char* nm : names) nvrtcAddNameExpression(p, nm);
  const nvrtcResult cres = nvrtcCompileProgram(p, (int)(sizeof opts / sizeof opts[0]), opts);
  size_t log_n = 0;
  nvrtcGetProgramLogSize(p, &log_n);
  g_log.assign(log_n, '\0');
  if (log_n) nvrtcGetProgramLog(p, &g_log[0]);
  if (cres != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&p);
    return set_error(ZEUS_ERR_ARGUMENT, "user objective failed to compile (see compile log): %s",
                     g_log.substr(0, 400).c_str());
  }
  size_t cubin_n = 0;
  rc = rtc_check(nvrtcGetCUBINSize(p, &cubin_n), "nvrtcGetCUBINSize");
  std::vector<char> cubin(cubin_n);
  if (!rc) rc = rtc_check(nvrtcGetCUBIN(p, cubin.data()), "nvrtcGetCUBIN");
  const char* lowered[kNames] = {};
  for (int i = 0; i < kNames && !rc; ++i)
    rc = rtc_check(nvrtcGetLoweredName(p, names[i], &lowered[i]), "nvrtcGetLoweredName");
  UserPlugin* up = nullptr;
  if (!rc) {
    up = new UserPlugin();
    up->d = d;
    rc = cu_check(drv().ModuleLoadData(&up->mod, cubin.data()), "cuModuleLoadData");
    CUfunction* fs[kNames] = {&up->pso_init, &up->pso_sweep, &up->pso_finalize, &up->bfgs,
                              &up->value, &up->gradient, &up->armijo};
    for (int i = 0; i < kNames && !rc; ++i)
      rc = cu_check(drv().ModuleGetFunction(fs[i], up->mod, lowered[i]), "cuModuleGetFunction");
    size_t sym_n = 0;
    if (!rc)
      rc = cu_check(drv().ModuleGetGlobal(&up->data_sym, &sym_n, up->mod, "_ZN4zeus14zeus_user_dataE"),
                    "cuModuleGetGlobal(zeus_user_data)");
    up->warp = warp;
    if (warp) {
      up->plan = user_warp_plan(d);
      if (!up->plan.smem_h && up->plan.dr == 0)
        rc = set_error(ZEUS_ERR_UNSUPPORTED, "user objective d=%d: H does not fit in smem", d);
    }
    if (!rc) {
      const int smem = warp ? (int)up->plan.smem
                            : (int)(sizeof(double) * (size_t)(d * (d + 1) / 2) * kThreadBlockU);
      rc = cu_check(drv().FuncSetAttribute(up->bfgs, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                       smem),
                    "cuFuncSetAttribute");
    }
  }
  nvrtcDestroyProgram(&p);
  if (rc) {
    if (up) {
      if (up->mod) drv().ModuleUnload(up->mod);
      delete up;
    }
    return rc;
  }
  *handle = up;
  return ZEUS_OK;
}

int zeus_user_free(void* handle) {
  UserPlugin* up = (UserPlugin*)handle;
  if (!up) return ZEUS_OK;
  int rc = ZEUS_OK;
  if (up->mod) rc = cu_check(drv().ModuleUnload(up->mod), "cuModuleUnload");
  delete up;
  return rc;
}

int zeus_user_dim(void* handle) { return handle ? ((UserPlugin*)handle)->d : -1; }

// data: device array the objective reads as `data` (may be NULL)
int zeus_user_set_data(void* handle, const double* data, void* stream) {
  UserPlugin* up = (UserPlugin*)handle;
  if (!up) return set_error(ZEUS_ERR_ARGUMENT, "zeus_user_set_data: null handle");
  const double* v = data;
  return cu_check(drv().MemcpyHtoDAsync(up->data_sym, &v, sizeof(v), (CUstream)stream),
                  "set zeus_user_data");
}

int zeus_user_value(void* handle, int64_t n, const double* x, int64_t ldx, double* f,
                    void* stream) {
  UserPlugin* up = (UserPlugin*)handle;
  if (!up || n < 0 || ldx < n || (n > 0 && (!x || !f)))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_user_value: bad arguments");
  if (n == 0) return ZEUS_OK;
  int d = up->d;
  void* args[] = {&d, &n, &x, &ldx, &f};
  const unsigned nb = (unsigned)((n + 127) / 128);
  return cu_check(drv().LaunchKernel(up->value, nb, 1, 1, 128, 1, 1, 0, (CUstream)stream, args,
                                 nullptr),
                  "user_value_kernel");
}

int zeus_user_gradient(void* handle, int64_t n, const double* x, int64_t ldx, double* grad,
                       uint8_t* domain_error, void* stream) {
  UserPlugin* up = (UserPlugin*)handle;
  if (!up || n < 0 || ldx < n || (n > 0 && (!x || !grad || !domain_error)))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_user_gradient: bad arguments");
  if (n == 0) return ZEUS_OK;
  int d = up->d;
  void* args[] = {&d, &n, &x, &ldx, &grad, &domain_error};
  return cu_check(drv().LaunchKernel(up->gradient, (unsigned)((n + 127) / 128), 1, 1, 128, 1, 1, 0,
                                     (CUstream)stream, args, nullptr),
                  "user_gradient_kernel");
}

int zeus_user_armijo(void* handle, int64_t n, const double* x, const double* p, const double* g,
                     int64_t ld, const double* f0, const zeus_bfgs_params* P, double* alpha,
                     int32_t* trials, void* stream) {
  UserPlugin* up = (UserPlugin*)handle;
  if (!up || n < 0 || ld < n || !P || (n > 0 && (!x || !p || !g || !f0 || !alpha || !trials)))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_user_armijo: bad arguments");
  if (n == 0) return ZEUS_OK;
  int d = up->d;
  double c1 = P->c1_armijo, a0 = P->alpha0, sh = P->shrink;
  int il = P->iter_ls;
  void* args[] = {&d, &n, &x, &p, &g, &ld, &f0, &c1, &a0, &il, &sh, &alpha, &trials};
  return cu_check(drv().LaunchKernel(up->armijo, (unsigned)((n + 127) / 128), 1, 1, 128, 1, 1, 0,
                                     (CUstream)stream, args, nullptr),
                  "user_armijo_kernel");
}

static int finalize(UserPlugin* up, int nb, int64_t i0, double* p, int64_t ld, double* blk_f,
                    long long* blk_i, double* cand, CUstream s) {
  int d = up->d;
  void* args[] = {&d, &nb, &i0, &p, &ld, &blk_f, &blk_i, &cand};
  return cu_check(drv().LaunchKernel(up->pso_finalize, 1, 1, 1, kPsoBlockU, 1, 1, 0, s, args, nullptr),
                  "pso_finalize_kernel(user)");
}

int zeus_user_pso_init(void* handle, int64_t n, int64_t i0, uint64_t seed, double lower,
                       double upper, double* x, double* v, double* pbest, double* pval,
                       int64_t ld, double* cand, void* workspace, void* stream) {
  UserPlugin* up = (UserPlugin*)handle;
  if (!up || n < 1 || i0 < 0 || ld < n || !(lower < upper) || !x || !v || !pbest || !pval ||
      !cand || !workspace)
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_user_pso_init: bad arguments");
  int d = up->d;
  int nb = (int)((n + kPsoBlockU - 1) / kPsoBlockU);
  double* blk_f = (double*)workspace;
  long long* blk_i = (long long*)(blk_f + nb);
  double range = upper - lower, vr = upper - lower;  // pso.py:101
  double vlow = -vr, vrange = vr - (-vr);
  void* none = nullptr;
  unsigned long long seq = 0;  // no peer exchange on this path
  void* args[] = {&d, &n, &i0, &seed, &lower, &range, &vlow, &vrange, &x, &v, &pbest, &pval,
                  &ld, &blk_f, &blk_i, &none, &none, &none, &none, &none, &seq};
  int rc = cu_check(drv().LaunchKernel(up->pso_init, nb, 1, 1, kPsoBlockU, 1, 1, 0, (CUstream)stream,
                                   args, nullptr),
                    "pso_init_kernel(user)");
  if (rc) return rc;
  return finalize(up, nb, i0, pbest, ld, blk_f, blk_i, cand, (CUstream)stream);
}

int zeus_user_pso_sweep(void* handle, int64_t n, int64_t i0, uint64_t seed, int sweep, double w,
                        double c1, double c2, double* x, double* v, double* pbest, double* pval,
                        int64_t ld, const double* gX, double* cand, void* workspace,
                        void* stream) {
  UserPlugin* up = (UserPlugin*)handle;
  if (!up || n < 1 || i0 < 0 || ld < n || sweep < -1 || !x || !v || !pbest || !pval || !gX ||
      !cand || !workspace)
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_user_pso_sweep: bad arguments");
  int d = up->d;
  int nb = (int)((n + kPsoBlockU - 1) / kPsoBlockU);
  double* blk_f = (double*)workspace;
  long long* blk_i = (long long*)(blk_f + nb);
  uint64_t k0 = (uint64_t)(2 * d) * (uint64_t)(sweep + 1);
  void* none = nullptr;
  unsigned long long seq = 0;  // no peer exchange on this path
  void* args[] = {&d, &n, &i0, &seed, &k0, &w, &c1, &c2, &x, &v, &pbest, &pval, &ld, &gX,
                  &blk_f, &blk_i, &none, &none, &none, &none, &none, &seq};
  int rc = cu_check(drv().LaunchKernel(up->pso_sweep, nb, 1, 1, kPsoBlockU, 1, 1, 0,
                                   (CUstream)stream, args, nullptr),
                    "pso_sweep_kernel(user)");
  if (rc) return rc;
  return finalize(up, nb, i0, pbest, ld, blk_f, blk_i, cand, (CUstream)stream);
}

// The fused PSO phase of a user objective (zeus_pso_run / zeus_pso_run_xchg
// with the NVRTC-compiled kernels): init + iter_pso sweeps, one launch each,
// the last block writes the barrier's result; xchg_block != NULL adds the
// multi-GPU peer-memory exchange (exchanges seq0 ...).
int zeus_user_pso_run(void* handle, int64_t n, int64_t i0, uint64_t seed, double lower,
                      double upper, double w, double c1, double c2, int iter_pso, double* x,
                      double* v, double* pbest, double* pval, int64_t ld, double* cand,
                      double* gX, double* gbest, void* workspace, void* xchg_block, int world,
                      unsigned long long seq0, void* stream) {
  UserPlugin* up = (UserPlugin*)handle;
  if (!up || n < 0 || (n == 0 && !xchg_block) || i0 < 0 || ld < n || ld < 1 ||
      !(lower < upper) || iter_pso < 0 || !x || !v || !pbest || !pval || !cand || !gX ||
      !gbest || !workspace || (xchg_block && (world < 1 || world > 8 || seq0 < 1)))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_user_pso_run: bad arguments");
  int d = up->d;
  CUstream s = (CUstream)stream;
  int nb = n > 0 ? (int)((n + kPsoBlockU - 1) / kPsoBlockU) : 1;
  double* blk_f = (double*)workspace;
  long long* blk_i = (long long*)(blk_f + nb);
  unsigned* done = (unsigned*)(blk_i + nb);
  void* xg = xchg_block ? (char*)xchg_block + xchg_desc_offset(d, world) : nullptr;
  int rc = check_cuda(cudaMemsetAsync(done, 0, sizeof(unsigned), (cudaStream_t)stream),
                      "memset(pso done)");
  if (rc) return rc;
  double range = upper - lower, vr = upper - lower;  // pso.py:101
  double vlow = -vr, vrange = vr - (-vr);
  unsigned long long seq = seq0;
  void* a_init[] = {&d, &n, &i0, &seed, &lower, &range, &vlow, &vrange, &x, &v, &pbest, &pval,
                    &ld, &blk_f, &blk_i, &done, &cand, &gX, &gbest, &xg, &seq};
  rc = cu_check(drv().LaunchKernel(up->pso_init, nb, 1, 1, kPsoBlockU, 1, 1, 0, s, a_init,
                                   nullptr),
                "pso_init_kernel(user, fused)");
  for (int sw = 0; sw < iter_pso && !rc; ++sw) {
    uint64_t k0 = (uint64_t)(2 * d) * (uint64_t)(sw + 1);
    unsigned long long sq = seq0 + 1 + (unsigned)sw;
    void* a_sw[] = {&d, &n, &i0, &seed, &k0, &w, &c1, &c2, &x, &v, &pbest, &pval, &ld, &gX,
                    &blk_f, &blk_i, &done, &cand, &gX, &gbest, &xg, &sq};
    rc = cu_check(drv().LaunchKernel(up->pso_sweep, nb, 1, 1, kPsoBlockU, 1, 1, 0, s, a_sw,
                                     nullptr),
                  "pso_sweep_kernel(user, fused)");
  }
  return rc;
}

size_t zeus_user_bfgs_workspace_bytes(void) { return kUserWsHeader; }

int zeus_user_bfgs(void* handle, int64_t n, const double* x0, int64_t ldx,
                   const zeus_bfgs_params* P, int64_t required_c,
                   unsigned long long* stop_counter, int* stop_flag, zeus_bfgs_out* out,
                   void* workspace, void* stream) {
  UserPlugin* up = (UserPlugin*)handle;
  if (!up || n < 0 || ldx < n || !P || !out || !workspace || (n > 0 && (!x0 || !out->x_final ||
      !out->f_final || !out->grad_norm || !out->iterations || !out->status)) ||
      out->ld_out < n || !(P->theta > 0.0) || P->iter_bfgs < 0 || P->iter_ls < 1 ||
      !(P->alpha0 > 0.0) || ((stop_counter == nullptr) != (stop_flag == nullptr)))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_user_bfgs: bad arguments");
  if (n == 0) return ZEUS_OK;
  CUstream s = (CUstream)stream;
  BfgsArgs A{};
  A.d = up->d;
  A.n = n;
  A.x0 = x0;
  A.ldx = ldx;
  A.theta = P->theta;
  A.gsq_max = gsq_max_for(P->theta);
  A.cap = P->iter_bfgs;
  A.iter_ls = P->iter_ls;
  A.c1 = P->c1_armijo;
  A.alpha0 = P->alpha0;
  A.shrink = P->shrink;
  A.required_c = required_c;
  A.stop_counter = stop_counter;
  A.stop_flag = stop_flag;
  A.out = *out;
  A.work = (unsigned long long*)workspace;
  int rc = cu_check(drv().MemsetD8Async((CUdeviceptr)workspace, 0, 8, s), "memset(work)");
  if (rc) return rc;
  int block = kThreadBlockU, smem = 0;
  if (up->warp) {  // warp per start: no promotion tiers (k1 = 0), H in smem
    const BfgsPlan& Pl = up->plan;
    A.warp_doubles = (int)Pl.warp_doubles;
    A.ldh = Pl.ldh;
    A.tstride = Pl.tstride;
    A.bmax = Pl.bmax;
    A.nalpha = Pl.nalpha;
    block = Pl.wpb * 32;
    smem = (int)Pl.smem;
  } else {
    smem = (int)(sizeof(double) * (size_t)(up->d * (up->d + 1) / 2) * kThreadBlockU);
  }
  int per_sm = 0;
  rc = cu_check(drv().Occupancy(&per_sm, up->bfgs, block, smem), "occupancy(user bfgs)");
  if (rc) return rc;
  const int sms = current_sm_count();
  if (per_sm < 1 || sms < 1) return set_error(ZEUS_ERR_UNSUPPORTED, "user bfgs: does not fit");
  int64_t grid = (int64_t)per_sm * sms;
  const int64_t per_block = up->warp ? block / 32 : kThreadBlockU;
  const int64_t need = (n + per_block - 1) / per_block;
  if (grid > need) grid = need;
  void* args[] = {&A};
  return cu_check(drv().LaunchKernel(up->bfgs, (unsigned)grid, 1, 1, block, 1, 1, smem, s,
                                     args, nullptr),
                  up->warp ? "bfgs_warp_kernel(user)" : "bfgs_thread_kernel(user)");
}

}  // extern "C"
