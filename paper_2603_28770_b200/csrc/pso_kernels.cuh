// pso_kernels.cuh -- device code of the particle-swarm phase (pso.py:79-164):
// included by pso.cu (registered objectives) and by the NVRTC program of a
// user objective (plugin.cu), which instantiates the same kernels.
//
// One thread per particle; swarm arrays are SoA [d][ld] so that coordinate k
// of consecutive particles is one coalesced 256-B transaction per warp.  The
// uniform draws come straight from the counter-based Philox stream of the
// particle's GLOBAL index (no RNG state in HBM); every update is evaluated
// in the reference's numpy order without contraction, so the swarm is
// bit-identical to init_swarm/update_swarm whenever libm agrees (always for
// Rosenbrock and Goldstein-Price).  The objective is folded in the same pass
// that produces x' (no second read of the position), then the personal best
// is updated under the strict '<' rule and a warp-shuffle + shared-memory
// block argmin leaves one (f, index) per block; a tiny finalize kernel turns
// those into this shard's candidate [f, idx, x...] (pso.py:73-76).
#pragma once
#include "objectives.cuh"

namespace zeus {

constexpr int kPsoBlock = 256;

// Streaming accumulator: feeds coordinates in order, reproduces value_seq.
// Generic accumulator (user objectives, d <= kStreamMax): buffers the
// coordinates, evaluates Obj's sequential value at the end.
constexpr int kStreamMax = 128;
template <class Obj>
struct StreamAcc {
  double xs[kStreamMax];
  int k = 0;
  __device__ void push(double x) { xs[k++] = x; }
  __device__ double result(int d) {
    double acc[Obj::NACC];
    bool err = false;
    const double f = value_seq<Obj>(DenseX{xs}, d, acc, err);
    return err ? __longlong_as_double(0x7ff8000000000000LL) : f;
  }
};

template <>
struct StreamAcc<Rosenbrock> {
  double total = 0.0, prev = 0.0;
  int k = 0;
  __device__ void push(double x) {
    if (k > 0) total = total + Rosenbrock::term2<double>(prev, x);
    prev = x;
    ++k;
  }
  __device__ double result(int) { return total; }
};
template <>
struct StreamAcc<Rastrigin> {
  double total;
  __device__ explicit StreamAcc(int d = 0) : total(10.0 * d) {}
  __device__ void push(double x) {
    bool oor = false;
    total = total + Rastrigin::term1<AutoMath, double>(x, oor);
  }
  __device__ double result(int) { return total; }
};
template <>
struct StreamAcc<Ackley> {
  double sq = 0.0, cs = 0.0;
  __device__ void push(double x) {
    double a, b;
    bool oor = false;
    Ackley::terms<AutoMath, double>(x, a, b, oor);
    sq = sq + a;
    cs = cs + b;
  }
  __device__ double result(int d) {
    bool err = false;
    return Ackley::outer<double>(sq, cs, d, err);
  }
};
template <>
struct StreamAcc<GoldsteinPrice> {
  double x1 = 0.0, v = 0.0;
  int k = 0;
  __device__ void push(double x) {
    if (k == 0) x1 = x;
    else v = GoldsteinPrice::eval<double>(x1, x);
    ++k;
  }
  __device__ double result(int) { return v; }
};

template <class Obj>
__device__ __forceinline__ StreamAcc<Obj> make_acc(int d) {
  if constexpr (Obj::kId == ZEUS_OBJ_RASTRIGIN) return StreamAcc<Obj>(d);
  else return StreamAcc<Obj>();
}

// Reduce block partials -> this shard's candidate [f, idx, pbest[:, idx]];
// with gX / gbest (one shard: the candidate IS the global best, pso.py:73-76)
// also the barrier's result.  Partials are read with __ldcg (written by
// other SMs in the fused path).
__device__ __forceinline__ void finalize_body(int d, int nb, int64_t i0,
                                              const double* __restrict__ p, int64_t ld,
                                              const double* blk_f, const long long* blk_i,
                                              double* cand, double* gX, double* gbest) {
  __shared__ long long win;
  double bf = 0.0;
  long long bi = -1;
  for (int b = threadIdx.x; b < nb; b += kPsoBlock) {
    const double fb = __ldcg(blk_f + b);
    const long long ib = __ldcg(blk_i + b);
    if (argmin_better(fb, ib, bf, bi)) {
      bf = fb;
      bi = ib;
    }
  }
  block_argmin<kPsoBlock>(bf, bi);
  if (threadIdx.x == 0) {
    win = bi;
    cand[0] = bf;
    cand[1] = (double)bi;
    if (gbest) {
      gbest[0] = bf;
      gbest[1] = (double)bi;
    }
  }
  __syncthreads();
  const long long li = win - i0;  // win < 0: empty shard, slot never selected
  for (int k = threadIdx.x; k < d; k += kPsoBlock) {
    const double v = win < 0 ? 0.0 : __ldcg(p + (int64_t)k * ld + li);
    cand[2 + k] = v;
    if (gX) gX[k] = v;
  }
}

__global__ void __launch_bounds__(kPsoBlock)
    pso_finalize_kernel(int d, int nb, int64_t i0, const double* __restrict__ p, int64_t ld,
                        const double* blk_f, const long long* blk_i, double* cand) {
  finalize_body(d, nb, i0, p, ld, blk_f, blk_i, cand, nullptr, nullptr);
}

// Cross-GPU barrier over peer memory (world > 1): every rank's exchange
// block holds two phases of [world][d+2] candidate slots plus [world] u64
// sequence flags; the descriptor below carries every rank's block as mapped
// into this process (CUDA IPC over NVLink/NVSwitch; plain pointers when the
// shards share a device).  The last block of a sweep stores this shard's
// candidate into slot (phase, rank) of EVERY rank, fences at system scope,
// release-stores seq into each rank's flag (phase, rank), then spins on its
// own flags until all world slots carry seq and picks the global best from
// its local copy in np.argmin order (pso.py:73-76) -- the per-sweep
// all-gather + select done inside the sweep kernel, no NCCL launch, no host.
// Two phases suffice: a rank can only publish sweep s+2 (same phase as s)
// after every rank published s+1, i.e. after every rank finished reading s.
constexpr int kXchgMaxRanks = 8;
struct PsoXchg {
  double* cand[kXchgMaxRanks];              // rank q's slots [2][world][d+2]
  unsigned long long* flag[kXchgMaxRanks];  // rank q's flags [2][world]
  unsigned* timeout;                        // this rank's: set if a peer never arrived
  int rank, world;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __noinline__ void xchg_barrier(const PsoXchg* __restrict__ xg, unsigned long long seq,
                                          int d, const double* cand, double* gX,
                                          double* gbest) {
  __shared__ int win;
  const int W = xg->world, r = xg->rank, ph = (int)(seq & 1), stride = d + 2;
  for (int e = threadIdx.x; e < W * stride; e += kPsoBlock) {
    const int q = e / stride, k = e - q * stride;
    xg->cand[q][(int64_t)(ph * W + r) * stride + k] = __ldcg(cand + k);
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < W) {
    st_release_sys(xg->flag[threadIdx.x] + ph * W + r, seq);
    const unsigned long long* f = xg->flag[r] + ph * W + threadIdx.x;
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(f) != seq) {
      __nanosleep(128);
      if (global_ns() - t0 > 20000000000ull) {  // 20 s: a peer died; report, don't hang
        atomicExch(xg->timeout, 1u);
        break;
      }
    }
  }
  __syncthreads();
  const double* mine = xg->cand[r] + (int64_t)ph * W * stride;
  if (threadIdx.x == 0) {
    double bf = 0.0;
    long long bi = -1;
    int bc = 0;
    for (int q = 0; q < W; ++q) {
      const double f = __ldcv(mine + (int64_t)q * stride);
      const long long idx = (long long)__ldcv(mine + (int64_t)q * stride + 1);
      if (argmin_better(f, idx, bf, bi)) {
        bf = f;
        bi = idx;
        bc = q;
      }
    }
    win = bc;
    gbest[0] = bf;
    gbest[1] = (double)bi;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < d; k += kPsoBlock)
    gX[k] = __ldcv(mine + (int64_t)win * stride + 2 + k);
}

// Fused barrier (`done` != nullptr): the last block to finish reduces every
// block's partial into the candidate (and, for one shard, the global best;
// with `xg`, the global best over every rank's shard via xchg_barrier), so a
// sweep is one launch.  Every block's writes are fenced before its ticket.
__device__ __forceinline__ void fused_finalize(unsigned* done, int d, int64_t i0, const double* p,
                                               int64_t ld, const double* blk_f,
                                               const long long* blk_i, double* cand, double* gX,
                                               double* gbest, const PsoXchg* xg,
                                               unsigned long long seq) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    if (xg) {
      finalize_body(d, (int)gridDim.x, i0, p, ld, blk_f, blk_i, cand, nullptr, nullptr);
      __syncthreads();
      xchg_barrier(xg, seq, d, cand, gX, gbest);
    } else {
      finalize_body(d, (int)gridDim.x, i0, p, ld, blk_f, blk_i, cand, gX, gbest);
    }
    if (threadIdx.x == 0) *done = 0u;  // ready for the next launch
  }
}

// init_swarm: positions U[lo,hi)^d from draws 0..d-1, velocities U[-vr,vr)^d
// from draws d..2d-1 (pso.py:101-109); pbest = x; pval = f(x).
template <class Obj>
__global__ void __launch_bounds__(kPsoBlock)
    pso_init_kernel(int d, int64_t n, int64_t i0, uint64_t seed, double lower, double range,
                    double vlow, double vrange, double* __restrict__ x, double* __restrict__ v,
                    double* __restrict__ p, double* __restrict__ pval, int64_t ld,
                    double* blk_f, long long* blk_i, unsigned* done, double* cand,
                    double* gX_out, double* gbest_out, const PsoXchg* xg,
                    unsigned long long seq) {
  const int64_t i = blockIdx.x * (int64_t)kPsoBlock + threadIdx.x;
  double bf = 0.0;
  long long bi = -1;
  if (i < n) {
    PhiloxCursor cur(seed, (uint64_t)(i0 + i));
    StreamAcc<Obj> acc = make_acc<Obj>(d);
    for (int k = 0; k < d; ++k) {
      const double xk = uniform_draw(cur.at((uint64_t)k), lower, range);
      x[(int64_t)k * ld + i] = xk;
      p[(int64_t)k * ld + i] = xk;
      acc.push(xk);
    }
    for (int k = 0; k < d; ++k)
      v[(int64_t)k * ld + i] = uniform_draw(cur.at((uint64_t)(d + k)), vlow, vrange);
    const double f = acc.result(d);
    pval[i] = f;
    bf = f;
    bi = i0 + i;
  }
  block_argmin<kPsoBlock>(bf, bi);
  if (threadIdx.x == 0) {
    blk_f[blockIdx.x] = bf;
    blk_i[blockIdx.x] = bi;
  }
  if (done) {
    __syncthreads();  // block_argmin's shared scratch is reused by the finalize
    fused_finalize(done, d, i0, p, ld, blk_f, blk_i, cand, gX_out, gbest_out, xg, seq);
  }
}

// update_swarm sweep s: r1 = draws 2d(s+1)+k, r2 = draws 2d(s+1)+d+k;
// v' = w v + c1 r1 (p - x) + c2 r2 (g - x); x' = x + v' (pso.py:143-163).
template <class Obj>
__global__ void __launch_bounds__(kPsoBlock)
    pso_sweep_kernel(int d, int64_t n, int64_t i0, uint64_t seed, uint64_t k0, double w,
                     double c1, double c2, double* __restrict__ x, double* __restrict__ v,
                     double* __restrict__ p, double* __restrict__ pval, int64_t ld,
                     const double* gX, double* blk_f, long long* blk_i, unsigned* done,
                     double* cand, double* gX_out, double* gbest_out, const PsoXchg* xg,
                     unsigned long long seq) {
  const int64_t i = blockIdx.x * (int64_t)kPsoBlock + threadIdx.x;
  double bf = 0.0;
  long long bi = -1;
  if (i < n) {
    PhiloxCursor c_r1(seed, (uint64_t)(i0 + i)), c_r2(seed, (uint64_t)(i0 + i));
    StreamAcc<Obj> acc = make_acc<Obj>(d);
    for (int k = 0; k < d; ++k) {
      const double r1 = uniform_draw(c_r1.at(k0 + (uint64_t)k), 0.0, 1.0);
      const double r2 = uniform_draw(c_r2.at(k0 + (uint64_t)(d + k)), 0.0, 1.0);
      const int64_t o = (int64_t)k * ld + i;
      const double xk = x[o], vk = v[o], pk = p[o], gk = gX[k];
      const double nv = w * vk + c1 * r1 * (pk - xk) + c2 * r2 * (gk - xk);
      const double nx = xk + nv;
      v[o] = nv;
      x[o] = nx;
      acc.push(nx);
    }
    const double f = acc.result(d);
    double best = pval[i];
    if (f < best) {  // strict: ties keep the old personal best (pso.py:161)
      best = f;
      pval[i] = f;
      for (int k = 0; k < d; ++k) p[(int64_t)k * ld + i] = x[(int64_t)k * ld + i];
    }
    bf = best;
    bi = i0 + i;
  }
  block_argmin<kPsoBlock>(bf, bi);
  if (threadIdx.x == 0) {
    blk_f[blockIdx.x] = bf;
    blk_i[blockIdx.x] = bi;
  }
  if (done) {
    __syncthreads();  // block_argmin's shared scratch is reused by the finalize
    fused_finalize(done, d, i0, p, ld, blk_f, blk_i, cand, gX_out, gbest_out, xg, seq);
  }
}

}  // namespace zeus
