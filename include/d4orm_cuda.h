/*
 * d4orm_cuda.h — the drop-in C-ABI boundary of the B200 denoise-step path.
 *
 * The reference (D4orm, /root/reference/proj) has no FFI: its operator
 * boundary is the C++ function
 *     DenoiseResult run_denoising(const JointControls& base, const Scenario&,
 *                                 const DynamicsModel&, const NoiseSchedule&,
 *                                 const DenoiserConfig&, double dt)
 *     (proj/include/d4orm/denoiser.hpp:68-70, proj/src/denoiser.cpp:119-184)
 * plus the public sub-operators it is built from (denoiser.hpp:44-58,
 * dynamics.hpp:148-155, reward.hpp:49-51).  Each entry point below replaces one
 * of them; the C++ drop-in in include/d4orm/*.hpp (same names and signatures as
 * the reference headers) is a thin layer over these calls that turns status
 * codes back into the reference's exception types and messages.
 *
 * Conventions: plain pointers and sizes, host memory, column-major fp64 exactly
 * as the reference's Eigen matrices (u: (R*du) x T -> element (k*du+d, t) at
 * t*R*du + k*du + d).  Every call returns D4ORM_OK or an error code; the
 * message is available from d4orm_cuda_last_error(ctx).  A context owns one
 * GPU stream and is used by one host thread at a time (the reference's
 * run_denoising is re-entrant per call).
 */
#ifndef D4ORM_CUDA_H
#define D4ORM_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  D4ORM_OK = 0,
  D4ORM_E_INVALID = 1,  /* std::invalid_argument in the reference */
  D4ORM_E_RUNTIME = 2,  /* std::runtime_error (non-finite state / reward) */
  D4ORM_E_CUDA = 3,
  D4ORM_E_NCCL = 4,
  D4ORM_E_UNSUPPORTED = 5
};

/* ModelKind (dynamics.hpp:11) + the BASELINE extensions. */
enum {
  D4ORM_DIFFDRIVE = 0,
  D4ORM_HOLO2D = 1,
  D4ORM_HOLO3D = 2,
  D4ORM_HOLO2D_VEL = 3,
  D4ORM_HOLO3D_VEL = 4,
  D4ORM_UNICYCLE = 5
};

enum { D4ORM_FROM_SCRATCH = 0, D4ORM_DEFORMATION = 1 };   /* DenoiseMode, denoiser.hpp:14-17 */
enum { D4ORM_NOISE_PHILOX = 0, D4ORM_NOISE_HOST = 1 };    /* K1 in-HBM Philox | host buffer */
enum { D4ORM_PREC_F32 = 0, D4ORM_PREC_F64 = 1 };          /* throughput | parity arithmetic */

/* Problem = Scenario (scenario.hpp:17-30) + DynamicsModel (dynamics.hpp:22-34)
 * + RewardConfig (reward.hpp:13-19) + the rollout dt/horizon. */
typedef struct {
  int kind;
  int dx, du, pdim;       /* must match kind */
  int robots;             /* R */
  int horizon;            /* T */
  double dt;
  double lower[3], upper[3];
  const double* starts;   /* dx x R column-major (Scenario::starts) */
  const double* goals;    /* pdim x R (Scenario::goals) */
  int n_obstacles;
  const double* obs_centers; /* pdim x O */
  const double* obs_radii;   /* O */
  double w_t, epsilon, robot_radius, goal_tolerance, obstacle_weight;
  double effort_weight;   /* extension; 0 = reference reward */
} d4orm_problem;

/* DenoiserConfig (denoiser.hpp:19-27); `batch` is BASELINE's "N samples". */
typedef struct {
  int steps;
  int64_t batch;
  double lambda;
  double alpha_bar_final;
  uint64_t seed;
  int mode;
  /* NoiseSchedule::alpha_bar (steps+1 values, alpha_bar[0] = 1), or NULL for
   * make_schedule(steps, alpha_bar_final) (schedule.cpp:9-27). */
  const double* alpha_bar;
} d4orm_denoiser_config;

/* DenoiseStepRecord (denoiser.hpp:29-34) */
typedef struct {
  int step;
  double best_reward, mean_reward, weight_entropy;
} d4orm_trace_rec;

/* Host noise provider for D4ORM_NOISE_HOST: fill dst (count x elems fp64,
 * row = sample m0+j) with the standard normals of denoising step `step`.
 * Return 0 on success. */
typedef int (*d4orm_noise_fn)(void* user, int step, int64_t m0, int64_t count, int64_t elems,
                              double* dst);

typedef struct d4orm_cuda_ctx d4orm_cuda_ctx;

/* ---- lifetime ---------------------------------------------------------- */
/* One context per (process, GPU).  world > 1 shards the samples across ranks;
 * nccl_id is the 128-byte ncclUniqueId rank 0 created (d4orm_cuda_nccl_id),
 * broadcast by the caller.  world == 1: nccl_id may be NULL. */
int d4orm_cuda_create(int device, int rank, int world, const void* nccl_id, d4orm_cuda_ctx** out);
/* world > 1 without NCCL (nccl_id NULL): the step's two all-gathers (rewards,
 * chunk-tree roots) go through fn, which must block until `gathered`
 * (world x bytes, rank order) holds every rank's `local` block and return 0
 * (e.g. MPI_Allgather, or torch.distributed over gloo).  Runs of such a
 * context launch no CUDA graphs (the exchange is a host call mid-step).  The
 * per-rank batch must be 256 x a power of two samples whenever world > 1. */
typedef int (*d4orm_exchange_fn)(void* user, const void* local, int64_t bytes, void* gathered);
int d4orm_cuda_set_exchange_fn(d4orm_cuda_ctx* ctx, d4orm_exchange_fn fn, void* user);
int d4orm_cuda_nccl_id(void* out128);
void d4orm_cuda_destroy(d4orm_cuda_ctx* ctx);
const char* d4orm_cuda_last_error(const d4orm_cuda_ctx* ctx);
const char* d4orm_cuda_version(void);

/* ---- configuration ------------------------------------------------------- */
/* validate_scenario-style checks (scenario.cpp:46-108 subset used by the path)
 * then upload to HBM. */
int d4orm_cuda_set_problem(d4orm_cuda_ctx* ctx, const d4orm_problem* problem);
int d4orm_cuda_set_options(d4orm_cuda_ctx* ctx, int precision, int noise_source, int use_graphs);
int d4orm_cuda_set_noise_fn(d4orm_cuda_ctx* ctx, d4orm_noise_fn fn, void* user);

/* ---- the path: run_denoising (denoiser.cpp:119-184) ----------------------- */
/* base: (R*du) x T; out_variable: (R*du) x T; trace: config->steps records
 * (may be NULL).  Errors mirror the reference's messages. */
int d4orm_cuda_run_denoising(d4orm_cuda_ctx* ctx, const double* base, const d4orm_denoiser_config* config,
                             double* out_variable, d4orm_trace_rec* trace);

/* ---- the caller of the path: the anytime loop solve (optimizer.cpp:49-102) --
 * Every iteration runs on the device: seed and key table (K7), the denoising
 * steps, the final fp64 rollout of base + delta, total_reward / objective /
 * check_success and best-trajectory tracking (K6).  Philox mode replays one
 * CUDA graph per iteration; the host reads back one record per iteration
 * (stop_on_success and the deadline are decided as in optimizer.cpp:91-92).
 * Replaces d4orm::solve (optimizer.hpp:31-32) for its caller run_trial
 * (bench.cpp:61) / cmd_solve (tools/main.cpp:338). */
typedef int (*d4orm_iteration_fn)(void* user, int iteration, uint64_t seed_it);
typedef struct {
  int max_iterations;               /* OptimizerConfig::max_iterations (>= 1) */
  int stop_on_success;              /* OptimizerConfig::stop_on_success */
  double deadline_seconds;          /* <= 0: no deadline */
  d4orm_denoiser_config denoiser;   /* mode is forced to Deformation (optimizer.cpp:23) */
  /* optional, called before iteration it (1-based) with seed_it =
   * mix_seed(denoiser.seed, it): host-noise providers reseed here.  Non-zero
   * aborts the solve. */
  d4orm_iteration_fn on_iteration;
  void* on_iteration_user;
} d4orm_solve_config;

/* IterationStats (result.hpp) */
typedef struct {
  double reward, objective;
  int success;
  double elapsed;                   /* seconds since the solve started */
} d4orm_iteration_rec;

/* ---- the paper's baselines on the same kernels (baselines.cpp:99-173) ------
 * MPPI: samples mean + sigma*z, softmax weights (score_weights), mc_average;
 * CEM: samples mean + std.*z, the elite fraction by a stable descending sort
 * of the rewards (select_elites), diagonal Gaussian refit with a std floor.
 * Every iteration (one CUDA graph in Philox mode) ends with K6 on the mean:
 * fp64 rollout, total_reward / objective / check_success, best tracking.
 * Host noise: the provider's `step` is the iteration (stream
 * mix_seed(seed, it, m)).  Replace mppi_solve / cem_solve (baselines.hpp:46-50). */
typedef struct {                    /* MppiConfig (baselines.hpp:16-27); horizon/dt from the problem */
  int64_t batch;
  double lambda, sigma;
  int iterations;
  uint64_t seed;
  int stop_on_success;
  double deadline_seconds;          /* <= 0: none */
} d4orm_mppi_config;

typedef struct {                    /* CemConfig (baselines.hpp:31-43) */
  int64_t batch;
  double elite_fraction, initial_std, min_std;
  int iterations;
  uint64_t seed;
  int stop_on_success;
  double deadline_seconds;
} d4orm_cem_config;

/* best_states: (R*dx) x (T+1); best_controls: (R*du) x (T+1) (column T zero);
 * per_iteration: max_iterations records; traces: max_iterations x steps
 * records (may be NULL).  *success = check_success(best trajectory). */
int d4orm_cuda_solve(d4orm_cuda_ctx* ctx, const d4orm_solve_config* config, double* best_states,
                     double* best_controls, d4orm_iteration_rec* per_iteration, d4orm_trace_rec* traces,
                     int* iterations_used, double* best_reward, int* success);
int d4orm_cuda_mppi_solve(d4orm_cuda_ctx* ctx, const d4orm_mppi_config* config, double* best_states,
                          double* best_controls, d4orm_iteration_rec* per_iteration, int* iterations_used,
                          double* best_reward, int* success);
int d4orm_cuda_cem_solve(d4orm_cuda_ctx* ctx, const d4orm_cem_config* config, double* best_states,
                         double* best_controls, d4orm_iteration_rec* per_iteration, int* iterations_used,
                         double* best_reward, int* success);

/* ---- per-stage entry points (parity) -------------------------------------- */
/* One denoising step i (loop body denoiser.cpp:152-180) from a given variable;
 * noise (batch x elems, fp64) or NULL for Philox. Outputs may be NULL. */
int d4orm_cuda_denoise_step(d4orm_cuda_ctx* ctx, const double* base, const double* variable_in,
                            const double* noise, int i, const d4orm_denoiser_config* config,
                            double* variable_out, double* rewards, double* weights, d4orm_trace_rec* rec);
/* rollout (dynamics.cpp:122-169) + total_reward (reward.cpp:67-130) of `count`
 * candidate control sequences u (count x (R*du*T)).  states: count x (R*dx)x(T+1),
 * controls: count x (R*du)x(T+1); counts: count x 2 (conflict, obstacle
 * robot-steps).  Any output may be NULL. */
int d4orm_cuda_rollout_fitness(d4orm_cuda_ctx* ctx, const double* u, int64_t count, double* states,
                               double* controls, double* rewards, int64_t* counts);
/* score_weights (denoiser.cpp:50-90) + entropy (:24-30). trace4 = {best, mean, entropy}. */
int d4orm_cuda_score_weights(d4orm_cuda_ctx* ctx, const double* rewards, int64_t m, double lambda,
                             double* weights, double* trace3);
/* mc_average (denoiser.cpp:92-108): out = sum_m weights[m] * samples[m] over
 * m sample rows of `elems` values (m x elems fp64, any layout the caller
 * shares between rows), after the reference's |sum(w) - 1| <= 1e-9 check
 * (D4ORM_E_INVALID "mc_average: weights must sum to 1").  K5a + K5b in the
 * context's precision: each 256-row chunk summed in ascending m, the chunk
 * partials combined by a fixed pairwise tree (fp64: within rounding of the
 * reference's sequential sum).  Needs no problem. */
int d4orm_cuda_weighted_mean(d4orm_cuda_ctx* ctx, const double* samples, const double* weights, int64_t m,
                             int64_t elems, double* out);
/* K1: the Philox normals of (seed, step) for samples [m0, m0+count). */
int d4orm_cuda_philox_noise(d4orm_cuda_ctx* ctx, uint64_t seed, int step, int64_t m0, int64_t count,
                            float* out);

/* ---- device-resident benchmarking ----------------------------------------- */
/* Prepare a device-resident run (base uploaded once), then time `steps`
 * denoising steps after `warmup` untimed ones, with CUDA events on the
 * context's stream.  Fills ms_total and, if non-NULL, per-kernel average
 * milliseconds kernel_ms[6] = {K1 noise, K2+K3 rollout+fitness, K4 weights,
 * K5 partial, K5 tree} (measured in a separate instrumented pass), and in
 * kernel_ms[5] the mean number of this rank's samples with a non-zero weight
 * in that pass (the z rows K5's partial pass reads; zero weights are skipped). */
int d4orm_cuda_bench_steps(d4orm_cuda_ctx* ctx, const double* base, const d4orm_denoiser_config* config,
                           int warmup, int steps, double* ms_total, double* kernel_ms);
/* Number of this library's kernel launches per denoising step (graph nodes). */
int d4orm_cuda_launches_per_step(const d4orm_cuda_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif
