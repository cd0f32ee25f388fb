// pso_kernels.cuh -- device code of the particle-swarm phase (pso.py:79-164):
// included by pso.cu (registered objectives) and by the NVRTC program of a
// user objective (plugin.cu), which instantiates the same kernels.
//
// Registered objectives (d <= kStreamMax) run the TILED kernels at the end of
// this file (a CTA owns 16-64 particles and spreads draws, updates and
// objective terms over its threads); pso_init_kernel / pso_sweep_kernel below
// are one thread per particle (user objectives, larger d).  Swarm arrays are
// SoA [d][ld] so that coordinate k of consecutive particles is one coalesced
// transaction per warp.  The
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
  // partials in batches of 8 loads in flight (the tiled sweep leaves up to
  // n / 16 of them; this loop is the serial tail of every sweep)
  for (int b0 = threadIdx.x; b0 < nb; b0 += 8 * kPsoBlock) {
    double fb[8];
    long long ib[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int b = b0 + u * kPsoBlock;
      fb[u] = b < nb ? __ldcg(blk_f + b) : 0.0;
      ib[u] = b < nb ? __ldcg(blk_i + b) : -1;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (argmin_better(fb[u], ib[u], bf, bi)) {
        bf = fb[u];
        bi = ib[u];
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

// Tiled sweep (registered objectives, d <= kStreamMax): one CTA owns P
// particles and spreads the sweep's independent work over all its threads
// instead of running d coordinates one after another in one thread:
//   1. draws: the 2d draws of sweep s are counters [k0, k0 + 2d) of each
//      particle's stream (r1 of coordinate k = counter k0 + k, r2 = k0 + d + k);
//      task (particle, Philox block) computes one Philox4x64-10 block, so
//      each block is generated once (the per-particle cursors of
//      pso_sweep_kernel generate the block straddling r1 / r2 twice);
//   2. update: task (particle, coordinate) loads x, v, p, forms v', x' in
//      the reference's order (the same expression as pso_sweep_kernel) and
//      stores them -- coordinate k of P consecutive particles is one
//      coalesced segment;
//   3. terms: task (particle, term) evaluates the objective's term on the new
//      coordinates (the same term functions StreamAcc calls: the libm-heavy
//      part in parallel);
//   4. fold: thread j adds particle j's terms in coordinate order (the
//      reference's left fold, StreamAcc's value bit for bit), applies the
//      strict '<' personal-best rule; improved particles' p rows are then
//      written by all threads, coalesced.
// Objectives without a term form (PsoTerms<Obj>::NT == 0) fold StreamAcc
// over the new coordinates in step 4 instead.
// Shared memory: draws [2d][P] (reused for the terms) + positions [d][P]
// doubles + P flags.  P = 2^LP.
__host__ __device__ __forceinline__ int pso_tile_log2(int d) {
  return d <= 32 ? 6 : d <= 64 ? 5 : 4;
}
__host__ __device__ __forceinline__ size_t pso_tile_smem(int d) {
  const int P = 1 << pso_tile_log2(d);
  return (size_t)3 * d * P * sizeof(double) + (size_t)P * sizeof(int);
}

// Term form of the registered objectives' sequential value (value_seq):
// NT accumulators; term(k) of the NEW coordinates xs (column j, stride P);
// fold(t) adds them in coordinate order from the reference's initial values.
template <class Obj>
struct PsoTerms {
  static constexpr int NT = 0;
};
template <>
struct PsoTerms<Rastrigin> {
  static constexpr int NT = 1;
  static constexpr int K0 = 0;  // first coordinate with a term
  __device__ static void term(const double* xs, int k, int P, double* t) {
    bool oor = false;
    t[0] = Rastrigin::term1<AutoMath, double>(xs[k * P], oor);
  }
  __device__ static double fold(const double* t, int d, int P) {
    double total = 10.0 * d;
    for (int k = 0; k < d; ++k) total = total + t[k * P];
    return total;
  }
};
template <>
struct PsoTerms<Rosenbrock> {
  static constexpr int NT = 1;
  static constexpr int K0 = 1;  // term k couples x[k-1], x[k]
  __device__ static void term(const double* xs, int k, int P, double* t) {
    t[0] = Rosenbrock::term2<double>(xs[(k - 1) * P], xs[k * P]);
  }
  __device__ static double fold(const double* t, int d, int P) {
    double total = 0.0;
    for (int k = 1; k < d; ++k) total = total + t[k * P];
    return total;
  }
};
template <>
struct PsoTerms<Ackley> {
  static constexpr int NT = 2;
  static constexpr int K0 = 0;
  __device__ static void term(const double* xs, int k, int P, double* t) {
    bool oor = false;
    Ackley::terms<AutoMath, double>(xs[k * P], t[0], t[1], oor);
  }
  __device__ static double fold(const double* t, int d, int P) {
    double sq = 0.0, cs = 0.0;
    for (int k = 0; k < d; ++k) {
      sq = sq + t[k * P];
      cs = cs + t[(d + k) * P];
    }
    bool err = false;
    return Ackley::outer<double>(sq, cs, d, err);
  }
};

// INIT: init_swarm in the same four passes (draws 0 .. 2d-1: x from draws
// k, v from draws d + k, pso.py:101-109; p = x, pval = f).  Otherwise sweep
// s (draws k0 = 2d(s+1) ..).  a0..a3: (lower, range, vlow, vrange) for INIT,
// (w, c1, c2, -) for a sweep.
template <class Obj, bool INIT>
__device__ __forceinline__ void pso_tiled_body(int d, int64_t n, int64_t i0, uint64_t seed,
                                               uint64_t k0, double a0, double a1, double a2,
                                               double a3, double* __restrict__ x,
                                               double* __restrict__ v, double* __restrict__ p,
                                               double* __restrict__ pval, int64_t ld,
                                               const double* gX, double* blk_f,
                                               long long* blk_i, unsigned* done, double* cand,
                                               double* gX_out, double* gbest_out,
                                               const PsoXchg* xg, unsigned long long seq) {
  using T = PsoTerms<Obj>;
  // programmatic dependent launch (pso.cu launch_pso_tiled): the next sweep
  // may be scheduled as soon as every CTA of this one is resident; it
  // generates its draws (pass 1: no global reads) while this one finishes,
  // then waits (griddepcontrol.wait: this grid complete, its writes visible)
  // before touching the swarm.  Both are no-ops for an ordinary launch.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ double pso_tile_sm[];
  const int LP = pso_tile_log2(d), P = 1 << LP, PM = P - 1;
  double* rs = pso_tile_sm;     // [2d][P] uniform draws, then [NT d][P] terms
  double* xs = rs + 2 * d * P;  // [d][P] new positions
  int* improved = (int*)(xs + d * P);
  const int64_t base = (int64_t)blockIdx.x * P;
  const int np = n > base ? (int)min((int64_t)P, n - base) : 0;
  const uint64_t kend = k0 + 2 * (uint64_t)d;
  const uint64_t b0 = k0 >> 2;
  const int nblk = (int)(((kend - 1) >> 2) - b0 + 1);
  for (int u = threadIdx.x; u < (nblk << LP); u += kPsoBlock) {
    const int j = u & PM, q = u >> LP;
    if (j < np) {
      uint64_t o[4];
      Philox4x64::block(b0 + q, seed, (uint64_t)(i0 + base + j), o);
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const uint64_t c = ((b0 + q) << 2) + m;
        // uniform_draw(u, 0, 1) == unit_double(u) exactly (0 + 1 * r, r >= 0)
        if (c >= k0 && c < kend) rs[((int)(c - k0) << LP) + j] = unit_double(o[m]);
      }
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  for (int u = threadIdx.x; u < (d << LP); u += kPsoBlock) {
    const int j = u & PM, k = u >> LP;
    if (j < np) {
      const double r1 = rs[u], r2 = rs[(d << LP) + u];
      const int64_t o = (int64_t)k * ld + base + j;
      if constexpr (INIT) {  // low + range * r, as uniform_draw
        const double xk = a0 + a1 * r1;
        x[o] = xk;
        p[o] = xk;
        v[o] = a2 + a3 * r2;
        xs[u] = xk;
      } else {
        const double xk = x[o], vk = v[o], pk = p[o], gk = gX[k];
        const double nv = a0 * vk + a1 * r1 * (pk - xk) + a2 * r2 * (gk - xk);
        const double nx = xk + nv;
        v[o] = nv;
        x[o] = nx;
        xs[u] = nx;
      }
    }
  }
  __syncthreads();
  if constexpr (T::NT > 0) {
    for (int u = threadIdx.x + (T::K0 << LP); u < (d << LP); u += kPsoBlock) {
      const int j = u & PM, k = u >> LP;
      if (j < np) {
        double t[T::NT];
        T::term(xs + j, k, P, t);
#pragma unroll
        for (int a = 0; a < T::NT; ++a) rs[((a * d) << LP) + u] = t[a];
      }
    }
    __syncthreads();
  }
  double bf = 0.0;
  long long bi = -1;
  if (threadIdx.x < P) {
    const int j = threadIdx.x;
    int imp = 0;
    if (j < np) {
      double f;
      if constexpr (T::NT > 0) {
        f = T::fold(rs + j, d, P);
      } else {
        StreamAcc<Obj> acc = make_acc<Obj>(d);
        for (int k = 0; k < d; ++k) acc.push(xs[(k << LP) + j]);
        f = acc.result(d);
      }
      double best;
      if constexpr (INIT) {
        best = f;
        pval[base + j] = f;
      } else {
        best = pval[base + j];
        if (f < best) {  // strict: ties keep the old personal best (pso.py:161)
          best = f;
          pval[base + j] = f;
          imp = 1;
        }
      }
      bf = best;
      bi = i0 + base + j;
    }
    improved[j] = imp;
  }
  __syncthreads();
  if constexpr (!INIT) {
    for (int u = threadIdx.x; u < (d << LP); u += kPsoBlock) {
      const int j = u & PM, k = u >> LP;
      if (improved[j]) p[(int64_t)k * ld + base + j] = xs[u];
    }
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

template <class Obj>
__global__ void __launch_bounds__(kPsoBlock)
    pso_sweep_tiled_kernel(int d, int64_t n, int64_t i0, uint64_t seed, uint64_t k0, double w,
                           double c1, double c2, double* __restrict__ x,
                           double* __restrict__ v, double* __restrict__ p,
                           double* __restrict__ pval, int64_t ld, const double* gX,
                           double* blk_f, long long* blk_i, unsigned* done, double* cand,
                           double* gX_out, double* gbest_out, const PsoXchg* xg,
                           unsigned long long seq) {
  pso_tiled_body<Obj, false>(d, n, i0, seed, k0, w, c1, c2, 0.0, x, v, p, pval, ld, gX, blk_f,
                             blk_i, done, cand, gX_out, gbest_out, xg, seq);
}

template <class Obj>
__global__ void __launch_bounds__(kPsoBlock)
    pso_init_tiled_kernel(int d, int64_t n, int64_t i0, uint64_t seed, double lower,
                          double range, double vlow, double vrange, double* __restrict__ x,
                          double* __restrict__ v, double* __restrict__ p,
                          double* __restrict__ pval, int64_t ld, double* blk_f,
                          long long* blk_i, unsigned* done, double* cand, double* gX_out,
                          double* gbest_out, const PsoXchg* xg, unsigned long long seq) {
  pso_tiled_body<Obj, true>(d, n, i0, seed, 0, lower, range, vlow, vrange, x, v, p, pval, ld,
                            nullptr, blk_f, blk_i, done, cand, gX_out, gbest_out, xg, seq);
}

}  // namespace zeus
