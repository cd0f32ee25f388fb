// pso.cu -- host launch + C ABI of the particle-swarm phase (pso.py:79-164);
// the kernels are in pso_kernels.cuh.
#include "pso_kernels.cuh"
#include "zeus_internal.h"

namespace zeus {

// Block partials a shard's workspace holds: enough for the tiled sweep's
// smallest tile (16 particles per CTA) and for the one-thread-per-particle
// kernels (kPsoBlock per CTA).
static int64_t pso_partials_max(int64_t n) {
  const int64_t nb = (n + 15) / 16;
  return nb < 1 ? 1 : nb;
}

// One sweep launch: the tiled kernel for d <= kStreamMax (every registered
// objective's sweep), else one thread per particle.  Returns the grid size
// (= the number of block partials written).
template <class Obj>
static int launch_sweep(int d, int64_t n, int64_t i0, uint64_t seed, uint64_t k0, double w,
                        double c1, double c2, double* x, double* v, double* p, double* pval,
                        int64_t ld, const double* gX, double* blk_f, long long* blk_i,
                        unsigned* done, double* cand, double* gX_out, double* gbest_out,
                        const PsoXchg* xg, unsigned long long seq, cudaStream_t s) {
  if (d <= kStreamMax) {
    static const bool attr = [] {
      return cudaFuncSetAttribute(pso_sweep_tiled_kernel<Obj>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  64 * 1024) == cudaSuccess;
    }();
    (void)attr;
    const int P = 1 << pso_tile_log2(d);
    const int nb = n > 0 ? (int)((n + P - 1) / P) : 1;
    // programmatic dependent launch: this sweep's draw pass overlaps the tail
    // of the previous PSO kernel on the stream (pso_tiled_body).  Not with a
    // peer exchange: there the previous sweep's last CTA waits for the other
    // ranks' sweeps, and ranks sharing a GPU (emulated shards, several
    // processes on one device) would find SM slots held by CTAs of the next
    // sweep waiting on that CTA -- measured: the 8-rank exchange test times out
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(nb);
    lc.blockDim = dim3(kPsoBlock);
    lc.dynamicSmemBytes = pso_tile_smem(d);
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = xg ? 0 : 1;
    cudaLaunchKernelEx(&lc, pso_sweep_tiled_kernel<Obj>, d, n, i0, seed, k0, w, c1, c2, x, v, p,
                       pval, ld, gX, blk_f, blk_i, done, cand, gX_out, gbest_out, xg, seq);
    return nb;
  }
  const int nb = n > 0 ? (int)((n + kPsoBlock - 1) / kPsoBlock) : 1;
  pso_sweep_kernel<Obj><<<nb, kPsoBlock, 0, s>>>(d, n, i0, seed, k0, w, c1, c2, x, v, p, pval,
                                                 ld, gX, blk_f, blk_i, done, cand, gX_out,
                                                 gbest_out, xg, seq);
  return nb;
}

// init_swarm launch: the tiled kernel for d <= kStreamMax, else one thread
// per particle.  Returns the grid size.
template <class Obj>
static int launch_init(int d, int64_t n, int64_t i0, uint64_t seed, double lower, double range,
                       double vlow, double vrange, double* x, double* v, double* p,
                       double* pval, int64_t ld, double* blk_f, long long* blk_i,
                       unsigned* done, double* cand, double* gX_out, double* gbest_out,
                       const PsoXchg* xg, unsigned long long seq, cudaStream_t s) {
  if (d <= kStreamMax) {
    static const bool attr = [] {
      return cudaFuncSetAttribute(pso_init_tiled_kernel<Obj>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  64 * 1024) == cudaSuccess;
    }();
    (void)attr;
    const int P = 1 << pso_tile_log2(d);
    const int nb = n > 0 ? (int)((n + P - 1) / P) : 1;
    pso_init_tiled_kernel<Obj><<<nb, kPsoBlock, pso_tile_smem(d), s>>>(
        d, n, i0, seed, lower, range, vlow, vrange, x, v, p, pval, ld, blk_f, blk_i, done, cand,
        gX_out, gbest_out, xg, seq);
    return nb;
  }
  const int nb = n > 0 ? (int)((n + kPsoBlock - 1) / kPsoBlock) : 1;
  pso_init_kernel<Obj><<<nb, kPsoBlock, 0, s>>>(d, n, i0, seed, lower, range, vlow, vrange, x,
                                                v, p, pval, ld, blk_f, blk_i, done, cand, gX_out,
                                                gbest_out, xg, seq);
  return nb;
}

struct PsoInitLaunch {
  template <class Obj>
  static int run(int d, int64_t n, int64_t i0, uint64_t seed, double lower, double upper,
                 double* x, double* v, double* p, double* pval, int64_t ld, double* cand,
                 void* ws, cudaStream_t s) {
    double* blk_f = (double*)ws;
    long long* blk_i = (long long*)(blk_f + pso_partials_max(n));
    const double range = upper - lower;
    const double vr = upper - lower;  // vel_range (pso.py:101)
    const double vlow = -vr, vrange = vr - (-vr);
    const int nb = launch_init<Obj>(d, n, i0, seed, lower, range, vlow, vrange, x, v, p, pval,
                                    ld, blk_f, blk_i, nullptr, nullptr, nullptr, nullptr,
                                    nullptr, 0ull, s);
    int rc = check_launch("pso_init_kernel");
    if (rc) return rc;
    pso_finalize_kernel<<<1, kPsoBlock, 0, s>>>(d, nb, i0, p, ld, blk_f, blk_i, cand);
    return check_launch("pso_finalize_kernel");
  }
};

struct PsoSweepLaunch {
  template <class Obj>
  static int run(int d, int64_t n, int64_t i0, uint64_t seed, int sweep, double w, double c1,
                 double c2, double* x, double* v, double* p, double* pval, int64_t ld,
                 const double* gX, double* cand, void* ws, cudaStream_t s) {
    double* blk_f = (double*)ws;
    long long* blk_i = (long long*)(blk_f + pso_partials_max(n));
    const uint64_t k0 = (uint64_t)(2 * d) * (uint64_t)(sweep + 1);
    const int nb = launch_sweep<Obj>(d, n, i0, seed, k0, w, c1, c2, x, v, p, pval, ld, gX, blk_f,
                                     blk_i, nullptr, nullptr, nullptr, nullptr, nullptr, 0ull, s);
    int rc = check_launch("pso_sweep_kernel");
    if (rc) return rc;
    pso_finalize_kernel<<<1, kPsoBlock, 0, s>>>(d, nb, i0, p, ld, blk_f, blk_i, cand);
    return check_launch("pso_finalize_kernel");
  }
};

// The whole PSO phase of a shard: init + iter_pso sweeps, each ONE launch
// whose last block reduces the candidate and writes the global best -- over
// this shard alone when it is the whole swarm (one GPU, pso.py:73-76 over one
// shard), or over every rank's shard through the peer-memory exchange `xg`
// (exchange seq0, seq0+1, ...) -- no host round trips, no NCCL launches.
// n == 0 (an empty shard of a multi-GPU run) launches one idle block that
// still takes part in the exchange.
struct PsoRunLaunch {
  template <class Obj>
  static int run(int d, int64_t n, int64_t i0, uint64_t seed, double lower, double upper,
                 double w, double c1, double c2, int iter_pso, double* x, double* v, double* p,
                 double* pval, int64_t ld, double* cand, double* gX, double* gbest, void* ws,
                 const PsoXchg* xg, unsigned long long seq0, cudaStream_t s) {
    double* blk_f = (double*)ws;
    long long* blk_i = (long long*)(blk_f + pso_partials_max(n));
    unsigned* done = (unsigned*)(blk_i + pso_partials_max(n));
    int rc = check_cuda(cudaMemsetAsync(done, 0, sizeof(unsigned), s), "memset(pso done)");
    if (rc) return rc;
    const double range = upper - lower, vr = upper - lower;  // pso.py:101
    launch_init<Obj>(d, n, i0, seed, lower, range, -vr, vr - (-vr), x, v, p, pval, ld, blk_f,
                     blk_i, done, cand, gX, gbest, xg, seq0, s);
    rc = check_launch("pso_init_kernel(fused)");
    for (int sw = 0; sw < iter_pso && !rc; ++sw) {
      const uint64_t k0 = (uint64_t)(2 * d) * (uint64_t)(sw + 1);
      launch_sweep<Obj>(d, n, i0, seed, k0, w, c1, c2, x, v, p, pval, ld, gX, blk_f, blk_i,
                        done, cand, gX, gbest, xg, seq0 + 1 + (unsigned)sw, s);
      rc = check_launch("pso_sweep_kernel(fused)");
    }
    return rc;
  }
};

// Exchange block of one rank: [2][world][d+2] f64 slots, [2][world] u64
// flags, a u32 timeout word (padded to 8 B), then the PsoXchg descriptor.
static size_t xchg_slots_bytes(int d, int world) {
  return (size_t)2 * world * (d + 2) * sizeof(double);
}
size_t xchg_desc_offset(int d, int world) {
  return xchg_slots_bytes(d, world) + (size_t)2 * world * 8 + 8;
}

}  // namespace zeus

using namespace zeus;

extern "C" {

size_t zeus_pso_workspace_bytes(int64_t n) {
  // block partials (as many as the tiled sweep's smallest tile leaves) +
  // the fused barrier's ticket counter (zeus_pso_run)
  return (size_t)pso_partials_max(n) * (sizeof(double) + sizeof(long long)) + 16;
}

int zeus_pso_run(int obj, int d, int64_t n, int64_t i0, uint64_t seed, double lower,
                 double upper, double w, double c1, double c2, int iter_pso, double* x,
                 double* v, double* pbest, double* pval, int64_t ld, double* cand, double* gX,
                 double* gbest, void* workspace, void* stream) {
  if (d < 1 || n < 1 || i0 < 0 || ld < n || !(lower < upper) || iter_pso < 0 || !x || !v ||
      !pbest || !pval || !cand || !gX || !gbest || !workspace ||
      (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_pso_run: bad arguments");
  const PsoXchg* none = nullptr;
  const int rc = dispatch_objective<PsoRunLaunch>(obj, d, n, i0, seed, lower, upper, w, c1, c2,
                                                  iter_pso, x, v, pbest, pval, ld, cand, gX,
                                                  gbest, workspace, none, 0ull,
                                                  as_stream(stream));
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
}

size_t zeus_pso_xchg_bytes(int d, int world) {
  if (d < 1 || world < 1 || world > kXchgMaxRanks) return 0;
  return xchg_desc_offset(d, world) + sizeof(PsoXchg);
}

int zeus_pso_xchg_setup(void* block, int d, int rank, int world, void* const* bases,
                        void* stream) {
  if (!block || !bases || d < 1 || world < 1 || world > kXchgMaxRanks || rank < 0 ||
      rank >= world || bases[rank] != block)
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_pso_xchg_setup: bad arguments");
  PsoXchg h;
  memset(&h, 0, sizeof(h));
  for (int q = 0; q < world; ++q) {
    if (!bases[q]) return set_error(ZEUS_ERR_ARGUMENT, "zeus_pso_xchg_setup: null peer block");
    h.cand[q] = (double*)bases[q];
    h.flag[q] = (unsigned long long*)((char*)bases[q] + xchg_slots_bytes(d, world));
  }
  h.timeout = (unsigned*)((char*)block + xchg_slots_bytes(d, world) + (size_t)2 * world * 8);
  h.rank = rank;
  h.world = world;
  cudaStream_t s = as_stream(stream);
  int rc = check_cuda(cudaMemsetAsync(block, 0, xchg_desc_offset(d, world), s),
                      "memset(pso exchange)");
  if (!rc)
    rc = check_cuda(cudaMemcpyAsync((char*)block + xchg_desc_offset(d, world), &h, sizeof(h),
                                    cudaMemcpyHostToDevice, s),
                    "upload(pso exchange descriptor)");
  if (!rc) rc = check_cuda(cudaStreamSynchronize(s), "pso exchange setup");
  return rc;
}

int zeus_pso_xchg_status(const void* block, int d, int world, unsigned* timed_out) {
  if (!block || !timed_out || d < 1 || world < 1 || world > kXchgMaxRanks)
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_pso_xchg_status: bad arguments");
  return check_cuda(cudaMemcpy(timed_out,
                               (const char*)block + xchg_slots_bytes(d, world) +
                                   (size_t)2 * world * 8,
                               sizeof(unsigned), cudaMemcpyDeviceToHost),
                    "read pso exchange status");
}

int zeus_pso_run_xchg(int obj, int d, int64_t n, int64_t i0, uint64_t seed, double lower,
                      double upper, double w, double c1, double c2, int iter_pso, double* x,
                      double* v, double* pbest, double* pval, int64_t ld, double* cand,
                      double* gX, double* gbest, void* workspace, void* xchg_block, int world,
                      unsigned long long seq0, void* stream) {
  if (d < 1 || n < 0 || i0 < 0 || ld < n || ld < 1 || !(lower < upper) || iter_pso < 0 || !x ||
      !v || !pbest || !pval || !cand || !gX || !gbest || !workspace || !xchg_block ||
      world < 1 || world > kXchgMaxRanks || seq0 < 1 ||
      (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_pso_run_xchg: bad arguments");
  const PsoXchg* xg = (const PsoXchg*)((char*)xchg_block + xchg_desc_offset(d, world));
  const int rc = dispatch_objective<PsoRunLaunch>(obj, d, n, i0, seed, lower, upper, w, c1, c2,
                                                  iter_pso, x, v, pbest, pval, ld, cand, gX,
                                                  gbest, workspace, xg, seq0,
                                                  as_stream(stream));
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
}

int zeus_pso_init(int obj, int d, int64_t n, int64_t i0, uint64_t seed, double lower,
                  double upper, double* x, double* v, double* pbest, double* pval, int64_t ld,
                  double* cand, void* workspace, void* stream) {
  if (d < 1 || n < 1 || i0 < 0 || ld < n || !(lower < upper) || !x || !v || !pbest || !pval ||
      !cand || !workspace || (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_pso_init: bad arguments");
  const int rc = dispatch_objective<PsoInitLaunch>(obj, d, n, i0, seed, lower, upper, x, v,
                                                   pbest, pval, ld, cand, workspace,
                                                   as_stream(stream));
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
}

int zeus_pso_sweep(int obj, int d, int64_t n, int64_t i0, uint64_t seed, int sweep, double w,
                   double c1, double c2, double* x, double* v, double* pbest, double* pval,
                   int64_t ld, const double* gX, double* cand, void* workspace, void* stream) {
  if (d < 1 || n < 1 || i0 < 0 || ld < n || sweep < -1 || !x || !v || !pbest || !pval || !gX ||
      !cand || !workspace || (obj == ZEUS_OBJ_GOLDSTEIN_PRICE && d != 2))
    return set_error(ZEUS_ERR_ARGUMENT, "zeus_pso_sweep: bad arguments");
  const int rc = dispatch_objective<PsoSweepLaunch>(obj, d, n, i0, seed, sweep, w, c1, c2, x,
                                                    v, pbest, pval, ld, gX, cand, workspace,
                                                    as_stream(stream));
  if (rc == ZEUS_ERR_ARGUMENT) return set_error(rc, "unknown objective id %d", obj);
  return rc;
}

}  // extern "C"
