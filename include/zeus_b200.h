/*
 * zeus_b200.h -- C ABI of libzeus_sm100.so, the B200 (sm_100a) implementation
 * of the reference's multistart optimizer hot path (arxiv/paper_2603_28770,
 * "Zeus"; reference package /root/reference/pkg/src/zeus).
 *
 * Conventions
 *  - Plain C types only: device pointers are raw CUDA device addresses (from
 *    torch tensors or cudaMalloc), owned by the caller; `stream` is a
 *    cudaStream_t passed as void*.  Every call is asynchronous on `stream`.
 *  - Point sets are SoA, coordinate-major: coordinate k of point i is
 *    x[k * ld + i]  (ld >= n).  This is what makes PSO loads coalesced.
 *  - Return value: 0 on success, < 0 on error (ZEUS_ERR_*); the message is
 *    available from zeus_last_error() on the calling host thread.  No C++
 *    exception crosses this boundary.
 *  - Objective ids follow the reference registry (objectives.py:145-182).
 *  - Status codes follow bfgs.py:32-35.
 *
 * Each entry point names the reference interface it replaces (file:line,
 * relative to /root/reference/pkg/src/zeus/).
 */
#ifndef ZEUS_B200_H
#define ZEUS_B200_H

#ifndef __CUDACC_RTC__
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define ZEUS_ABI_VERSION 2

/* objective ids (objectives.py:145-182 _REGISTRY) */
#define ZEUS_OBJ_ROSENBROCK 0
#define ZEUS_OBJ_RASTRIGIN 1
#define ZEUS_OBJ_ACKLEY 2
#define ZEUS_OBJ_GOLDSTEIN_PRICE 3

/* BFGS statuses (bfgs.py:32-35) */
#define ZEUS_CONVERGED 0
#define ZEUS_DIVERGED 1
#define ZEUS_STOPPED 2
#define ZEUS_DOMAIN_ERROR 3

/* error codes */
#define ZEUS_OK 0
#define ZEUS_ERR_ARGUMENT (-1)
#define ZEUS_ERR_CUDA (-2)
#define ZEUS_ERR_WORKSPACE (-3)
#define ZEUS_ERR_UNSUPPORTED (-4)

/* Per-start BFGS outputs (bfgs.py:43-56 BfgsOutcome, plus work counters the
 * roofline accounting needs).  Every pointer is a device array of n entries
 * except x_final (SoA, [d][ld_out]).  Counters may be NULL. */
typedef struct zeus_bfgs_out {
  double *x_final;      /* BfgsOutcome.x_final, SoA [d][ld_out]           */
  int64_t ld_out;
  double *f_final;      /* BfgsOutcome.f_final (NaN if f raised)          */
  double *grad_norm;    /* BfgsOutcome.grad_norm (+inf if none computed)  */
  int32_t *iterations;  /* BfgsOutcome.iterations                         */
  uint8_t *status;      /* BfgsOutcome.status (ZEUS_CONVERGED ...)        */
  int32_t *ls_trials;   /* objective evaluations spent in line searches   */
  int32_t *grad_evals;  /* forward-AD gradient evaluations                */
  /* Optional (NULL: not written): every start's outcome also as host-ready
   * rows, the zeus_pack_results layout -- rows[s * ld_rows + k] = x_final[k]
   * (k < d), [d] = f_final, [d + 1] = grad_norm; irows[4 s .. 4 s + 3] =
   * (iterations, status, ls_trials, grad_evals), 16-byte aligned.  They may
   * be page-locked host memory (device address from zeus_host_device_ptr):
   * each start's outcome then reaches the host as the start finishes, with
   * no pack kernel and no copy after the run. */
  double *rows;
  int64_t ld_rows;
  int32_t *irows;
} zeus_bfgs_out;

/* BFGS / line-search hyper-parameters: bfgs_run(theta, iter_bfgs) bfgs.py:80-87,
 * LineSearchParams linesearch.py:16-37. */
typedef struct zeus_bfgs_params {
  double theta;
  int32_t iter_bfgs;
  int32_t iter_ls;
  double c1_armijo;
  double alpha0;
  double shrink;
} zeus_bfgs_params;

#ifndef __CUDACC_RTC__  /* NVRTC (user-objective programs) sees only the types above */
/* ---- library ---------------------------------------------------------- */
int zeus_abi_version(void);
const char *zeus_last_error(void);
/* device properties used for persistent-grid sizing; -1 on error */
int zeus_sm_count(int device);

/* ---- counter-based streams: streams.py:21-54 (ParticleStreams.draw_uniform,
 * numpy Philox(key=[seed, i]) + Generator.uniform).  out[r * count + c] is
 * draw k0 + c of particle i0 + r, i.e. row-major [n][count]. */
int zeus_philox_uniform(uint64_t seed, int64_t i0, int64_t n, uint64_t k0, int64_t count,
                        double low, double high, double *out, void *stream);

/* ---- objectives: objectives.py:33-113 (values) and autodiff.py:243-266
 * forward_gradient.  x is SoA [d][ldx]; f[n]; grad SoA [d][ldx];
 * domain_error[n] = 1 where the reference raises DomainError. */
int zeus_objective_value(int obj, int d, int64_t n, const double *x, int64_t ldx,
                         double *f, void *stream);
int zeus_objective_gradient(int obj, int d, int64_t n, const double *x, int64_t ldx,
                            double *grad, uint8_t *domain_error, void *stream);

/* ---- PSO: pso.py:79-164.  The swarm shard is particles [i0, i0+n) of the
 * global swarm (streams are keyed by the GLOBAL index, so any sharding gives
 * bit-identical particles).  x, v, pbest are SoA [d][ld]; pval[n].
 * After init / each sweep the kernel leaves this shard's best personal best
 * in `cand` = [f, (double)global_index, x_0 .. x_{d-1}]  (d + 2 doubles).
 * workspace: zeus_pso_workspace_bytes(n). */
size_t zeus_pso_workspace_bytes(int64_t n);
/* init_swarm (pso.py:79-120) */
int zeus_pso_init(int obj, int d, int64_t n, int64_t i0, uint64_t seed, double lower,
                  double upper, double *x, double *v, double *pbest, double *pval,
                  int64_t ld, double *cand, void *workspace, void *stream);
/* update_swarm (pso.py:123-164) for 0-based sweep `sweep`, reading the
 * previous barrier's global best gX[d] (pso.py:143).  Sweep s draws r1, r2
 * from the particle streams' positions 2d(s+1) .. 2d(s+2)-1 (after init's 2d
 * draws); sweep = -1 draws from the streams' start (a swarm that was not made
 * by init_swarm, fresh streams). */
int zeus_pso_sweep(int obj, int d, int64_t n, int64_t i0, uint64_t seed, int sweep,
                   double w, double c1, double c2, double *x, double *v, double *pbest,
                   double *pval, int64_t ld, const double *gX, double *cand,
                   void *workspace, void *stream);
/* The whole PSO phase when this shard is the whole swarm (one GPU): init_swarm
 * + iter_pso update_swarm sweeps with the global-best barrier after each
 * (pso.py:79-164, driver.py:236-241), 1 + iter_pso launches; the last block of
 * every launch reduces the candidate and writes gX[d], gbest[2] = {f, index}
 * (the barrier's result for the next sweep).  Same results as zeus_pso_init /
 * zeus_pso_sweep + zeus_minloc_select(ncand = 1). */
int zeus_pso_run(int obj, int d, int64_t n, int64_t i0, uint64_t seed, double lower,
                 double upper, double w, double c1, double c2, int iter_pso, double *x,
                 double *v, double *pbest, double *pval, int64_t ld, double *cand, double *gX,
                 double *gbest, void *workspace, void *stream);
/* Multi-GPU PSO phase with the global-best barrier done INSIDE each sweep
 * kernel over peer memory (pso.py:73-76 + driver.py:236-241 across shards; the
 * reference's per-sweep host reduction, replaced here by NVLink stores): each
 * rank owns an exchange block of zeus_pso_xchg_bytes(d, world) bytes
 * (zeus_ipc_alloc; peers map it with zeus_ipc_open), initialised once by
 * zeus_pso_xchg_setup with every rank's block as mapped in this process
 * (bases[world], bases[rank] == block).  zeus_pso_run_xchg then runs init +
 * iter_pso sweeps of this rank's shard [i0, i0 + n) (n may be 0); the last
 * block of each launch publishes the shard candidate to every rank, waits
 * for all ranks' candidates of the same exchange and writes the np.argmin
 * winner to gX[d] / gbest[2].  Exchanges are numbered seq0, seq0 + 1, ...,
 * seq0 + iter_pso; every rank passes the same seq0 (>= 1), and the next call
 * continues the numbering at seq0 + iter_pso + 1.  A peer that never arrives
 * within 20 s sets the timeout word (zeus_pso_xchg_status) instead of
 * hanging.  world <= 8.  Results identical to zeus_pso_init / zeus_pso_sweep
 * + an all-gather + zeus_minloc_select over the same shards. */
size_t zeus_pso_xchg_bytes(int d, int world);
int zeus_pso_xchg_setup(void *block, int d, int rank, int world, void *const *bases,
                        void *stream);
int zeus_pso_xchg_status(const void *block, int d, int world, unsigned *timed_out);
int zeus_pso_run_xchg(int obj, int d, int64_t n, int64_t i0, uint64_t seed, double lower,
                      double upper, double w, double c1, double c2, int iter_pso, double *x,
                      double *v, double *pbest, double *pval, int64_t ld, double *cand,
                      double *gX, double *gbest, void *workspace, void *xchg_block, int world,
                      unsigned long long seq0, void *stream);
/* _reduce_global_best across shards (pso.py:73-76): cands[ncand][d+2] from
 * every shard (e.g. an NCCL all-gather); writes the np.argmin winner to
 * gX[d] and gbest[2] = {f, (double)global_index}. */
int zeus_minloc_select(int d, int ncand, const double *cands, double *gX, double *gbest,
                       void *stream);

/* ---- multistart BFGS: bfgs.py:80-156 bfgs_run over n independent starts,
 * with autodiff.py:243 gradients, linesearch.py:40 Armijo search and
 * bfgs.py:59 inverse-Hessian update fused in one persistent kernel.
 * x0 is SoA [d][ldx] (for zeus_run: the final swarm positions, driver.py:244).
 * Early stop (driver.py:153-177): if `stop_counter`/`stop_flag` are non-NULL,
 * each converged start atomically increments *stop_counter and the one that
 * reaches `required_c` sets *stop_flag = 1; every start polls *stop_flag at
 * the top of each iteration (bfgs.py:115-117) and ends `stopped`.
 * workspace: zeus_bfgs_workspace_bytes(d, n). */
size_t zeus_bfgs_workspace_bytes(int d, int64_t n);
int zeus_bfgs(int obj, int d, int64_t n, const double *x0, int64_t ldx,
              const zeus_bfgs_params *params, int64_t required_c,
              unsigned long long *stop_counter, int *stop_flag, zeus_bfgs_out *out,
              void *workspace, void *stream);

/* ---- reduce_best + converged_count: driver.py:115-134, 251.  Strict '<' over
 * starts whose status != DOMAIN_ERROR and f is not NaN, lowest index on ties.
 * best[2] = {f, (double)(i0 + index)} or {NaN, -1} when none is valid;
 * tallies[4] += per-status counts.  workspace: zeus_argmin_workspace_bytes(n). */
size_t zeus_argmin_workspace_bytes(int64_t n);
int zeus_reduce_best(int64_t n, int64_t i0, const double *f_final, const uint8_t *status,
                     double *best, unsigned long long *tallies, void *workspace,
                     void *stream);

/* ---- building blocks exposed for the reference's public helpers --------- */
/* armijo_search (linesearch.py:40-71) on n independent problems: x, p, g SoA
 * [d][ld]; f0[n]; alpha[n]; trials[n] = objective evaluations used. */
int zeus_armijo(int obj, int d, int64_t n, const double *x, const double *p,
                const double *g, int64_t ld, const double *f0, const zeus_bfgs_params *params,
                double *alpha, int32_t *trials, void *stream);
/* hessian_update (bfgs.py:59-77) on n problems: H[n][d][d] row-major (in
 * place), dx/dg [n][d]; updated[n] = 0 where the curvature guard skipped. */
int zeus_hessian_update(int d, int64_t n, double *H, const double *dx, const double *dg,
                        uint8_t *updated, void *stream);

/* ---- measurement ------------------------------------------------------- */
/* FP64 FMA throughput microbenchmark (the roofline denominator for the BFGS
 * kernel; MEASURED_PEAKS.json has no FP64 figure).  Launches blocks x threads
 * threads each running `iters` x 32 independent DFMAs; *flops_out receives
 * the FLOP count of the launch (time it with events on `stream`).
 * sink: device scratch of >= blocks doubles. */
int zeus_bench_dfma(int blocks, int threads, long long iters, double *sink, double *flops_out,
                    void *stream);

/* ---- experiment metrics: bench.py:131-141 count_within on device.
 * *count += number of points i (SoA x [d][ldx]) with |x_i - optimum|_2 < radius
 * (optimum: device array of d doubles; *count is accumulated, zero it first). */
int zeus_count_within(int d, int64_t n, const double *x, int64_t ldx, const double *optimum,
                      double radius, unsigned long long *count, void *stream);

/* ---- result hand-off: driver.py:244-265 (per_run, converged_count, best).
 * Packs the per-start SoA outputs of zeus_bfgs into host-ready row-major
 * tables in one kernel: fpack [n][d + 2] f64 = (x_final[0..d), f_final,
 * grad_norm); ipack [n][4] i32 = (iterations, status, ls_trials, grad_evals)
 * (16-byte aligned; NULL counters read as 0).  If spack is not NULL it also
 * receives {tallies[0..4) (zeus_reduce_best's status counts), gbest[0] (the
 * PSO global best f, NaN if gbest is NULL), best[0..nbest)} -- so one D2H of
 * each table hands a whole run to the host. */
int zeus_pack_results(const zeus_bfgs_out *out, int d, int64_t n, double *fpack, int32_t *ipack,
                      const unsigned long long *tallies, const double *gbest, const double *best,
                      int nbest, double *spack, void *stream);
/* Device address of page-locked host memory (cudaHostGetDevicePointer), for
 * zeus_bfgs_out.rows / irows. */
int zeus_host_device_ptr(void *host, void **dev);

/* ---- cross-GPU early stop: driver.py:137-202 (_init_worker / _run_parallel's
 * shared Value('q') counter and Value('i') flag, one per pool).  Here the pool
 * is one process per GPU: rank 0 creates a stop block in its device memory and
 * exports a CUDA IPC handle (ZEUS_IPC_HANDLE_BYTES opaque bytes, sent to the
 * other ranks by the host, e.g. torch.distributed.broadcast_object_list); the
 * other ranks open it and every rank passes (block, block + 8) as
 * zeus_bfgs's stop_counter / stop_flag.  The BFGS kernels use system-scope
 * atomics and volatile flag loads, so the counter is coherent across GPUs
 * over NVLink / NVSwitch.  Layout: u64 counter at offset 0, i32 flag at 8. */
/* device memory of its own cudaMalloc (so an IPC handle maps exactly it),
 * zeroed; handle: ZEUS_IPC_HANDLE_BYTES.  zeus_ipc_open maps a peer's block
 * (peer access enabled lazily); zeus_ipc_close frees (owner) or unmaps. */
int zeus_ipc_alloc(size_t bytes, void **block, unsigned char *handle);
int zeus_ipc_open(const unsigned char *handle, void **block);
int zeus_ipc_close(void *block, int owner);
/* Let kernels on `device` access memory of `peer` (cudaDeviceEnablePeerAccess;
 * already enabled is not an error): the single-process multi-GPU run maps its
 * exchange and stop blocks this way instead of through IPC handles. */
int zeus_enable_peer_access(int device, int peer);
#define ZEUS_STOP_BLOCK_BYTES 64
#define ZEUS_IPC_HANDLE_BYTES 64
int zeus_stop_block_create(void **block, unsigned char *handle);
int zeus_stop_block_open(const unsigned char *handle, void **block);
/* owner = 1 frees the block (creator), 0 unmaps an opened handle */
int zeus_stop_block_close(void *block, int owner);
/* zero counter and flag on `stream` (call before the ranks launch) */
int zeus_stop_block_reset(void *block, void *stream);

/* ---- user objectives: the reference's generic-scalar user callables
 * (pkg/README.md:70-87, autodiff.py) as device source, compiled at run time
 * with NVRTC together with this library's PSO and thread-per-start BFGS
 * kernels.  Contract of `source`: csrc/user_objective.cuh.  1 <= d <= 128
 * (BFGS: thread per start for d <= 16, the warp-per-start kernel above).
 * include_dir: the csrc/ directory holding the kernel headers.  The handle
 * is bound to the CUDA context current at compile time. */
int zeus_user_compile(const char *source, int d, const char *include_dir, void **handle);
const char *zeus_user_compile_log(void); /* NVRTC log of the last compile on this thread */
int zeus_user_free(void *handle);
int zeus_user_dim(void *handle);
/* the objective's `data` argument (device array or NULL); stream-ordered */
int zeus_user_set_data(void *handle, const double *data, void *stream);
/* objectives.py-style evaluation of n points (SoA [d][ldx]); NaN where the
 * objective raises DomainError */
int zeus_user_value(void *handle, int64_t n, const double *x, int64_t ldx, double *f,
                    void *stream);
/* forward_gradient (autodiff.py:243-266) / armijo_search (linesearch.py:40-71)
 * on n points -- as zeus_objective_gradient / zeus_armijo; trials[i] = -1
 * where the objective raised DomainError inside the search */
int zeus_user_gradient(void *handle, int64_t n, const double *x, int64_t ldx, double *grad,
                       uint8_t *domain_error, void *stream);
int zeus_user_armijo(void *handle, int64_t n, const double *x, const double *p, const double *g,
                     int64_t ld, const double *f0, const zeus_bfgs_params *params, double *alpha,
                     int32_t *trials, void *stream);
/* init_swarm / update_swarm (pso.py:79-164) -- as zeus_pso_init/_sweep */
int zeus_user_pso_init(void *handle, int64_t n, int64_t i0, uint64_t seed, double lower,
                       double upper, double *x, double *v, double *pbest, double *pval,
                       int64_t ld, double *cand, void *workspace, void *stream);
int zeus_user_pso_sweep(void *handle, int64_t n, int64_t i0, uint64_t seed, int sweep,
                        double w, double c1, double c2, double *x, double *v, double *pbest,
                        double *pval, int64_t ld, const double *gX, double *cand,
                        void *workspace, void *stream);
/* zeus_pso_run (xchg_block == NULL; n >= 1) / zeus_pso_run_xchg (exchange
 * block of zeus_pso_xchg_bytes(d, world), set up as above) for a user
 * objective. */
int zeus_user_pso_run(void *handle, int64_t n, int64_t i0, uint64_t seed, double lower,
                      double upper, double w, double c1, double c2, int iter_pso, double *x,
                      double *v, double *pbest, double *pval, int64_t ld, double *cand,
                      double *gX, double *gbest, void *workspace, void *xchg_block, int world,
                      unsigned long long seq0, void *stream);
/* bfgs_run over n starts (bfgs.py:80-156) -- as zeus_bfgs */
size_t zeus_user_bfgs_workspace_bytes(void);
int zeus_user_bfgs(void *handle, int64_t n, const double *x0, int64_t ldx,
                   const zeus_bfgs_params *params, int64_t required_c,
                   unsigned long long *stop_counter, int *stop_flag, zeus_bfgs_out *out,
                   void *workspace, void *stream);

#endif /* __CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif
#endif /* ZEUS_B200_H */
