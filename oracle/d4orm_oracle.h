/*
 * d4orm_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C fp64 restatement of the reference's denoise-step path (D4orm,
 * /root/reference/proj).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it, and only as the checker or
 * the CPU baseline — never as the product path.  The product (the CUDA library
 * under paper_2503_12204_b200/) never links or calls this code.
 *
 * Parity pin: every function below is checked (tests/test_oracle_pin.py)
 *   (1) against the SPEC.md worked examples (the only known-answer values the
 *       reference holds; its proj/tests/ is empty), and
 *   (2) bitwise against oracle/_ref/libd4orm_ref.so — the reference's own
 *       proj/src/{dynamics,reward,schedule,denoiser,optimizer,scenario}.cpp
 *       compiled from /root/reference against our Eigen-subset header
 *       (oracle/eigen_shim), see oracle/Makefile.
 *
 * Layouts follow the reference (column-major Eigen::MatrixXd):
 *   controls u      : (R*du) x T   -> element (k*du+d, t) at t*R*du + k*du + d
 *   states          : (R*dx) x (T+1)
 *   starts          : dx x R,  goals: pdim x R,  obstacle centres: pdim x O
 */
#ifndef D4ORM_ORACLE_H
#define D4ORM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Model kinds.  0..2 are the reference's ModelKind (dynamics.hpp:11); 3..5 are
 * the BASELINE extensions added through the reference's own extension point, a
 * derivative functor plugged into detail::rk4_with (dynamics.hpp:121-130). */
enum {
  OR_DIFFDRIVE = 0,  /* [x,y,theta,v], u=[omega,a]      dynamics.hpp:81-93  */
  OR_HOLO2D = 1,     /* [x,y,vx,vy],   u=[ax,ay]        dynamics.hpp:95-106 */
  OR_HOLO3D = 2,     /* [p(3),v(3)],   u=a(3)           dynamics.hpp:108-119 */
  OR_HOLO2D_VEL = 3, /* [x,y],         u=[vx,vy]  xdot=u   (extension) */
  OR_HOLO3D_VEL = 4, /* [x,y,z],       u=v(3)     xdot=u   (extension) */
  OR_UNICYCLE = 5    /* [x,y,theta],   u=[v,omega]         (extension) */
};

typedef struct {
  int kind, dx, du, pdim;
  int robots;  /* R */
  int horizon; /* T */
  double dt;
  double lower[3], upper[3];  /* control box, du entries */
  const double* starts;       /* dx x R */
  const double* goals;        /* pdim x R */
  int n_obstacles;
  const double* obs_centers;  /* pdim x O */
  const double* obs_radii;    /* O */
  /* RewardConfig (reward.hpp:13-19) */
  double w_t, epsilon, robot_radius, goal_tolerance, obstacle_weight;
} or_problem;

typedef struct {
  int steps;            /* reference N (DenoiserConfig::steps) */
  int64_t batch;        /* reference M (DenoiserConfig::batch) = BASELINE "N samples" */
  double lambda;
  double alpha_bar_final;
  uint64_t seed;
  int mode;             /* 0 = FromScratch, 1 = Deformation (denoiser.hpp:14-17) */
  int workers;          /* 0 = all hardware threads (parallel.hpp:12-16) */
} or_denoiser_config;

typedef struct {
  int step;
  double best_reward, mean_reward, weight_entropy;
} or_trace_rec;

/* ---- rng.hpp:10-40 ---- */
uint64_t or_splitmix64(uint64_t x);
uint64_t or_mix_seed(uint64_t a, uint64_t b);
uint64_t or_mix_seed3(uint64_t a, uint64_t b, uint64_t c);
void or_normal_fill(uint64_t stream_seed, double* out, int64_t count);
/* Noise of denoising step i for samples [m0, m0+count): sample m's (R*du)xT
 * block (elems doubles) from NormalStream(mix_seed(seed, i, m)) — exactly what
 * sample_batch draws (denoiser.cpp:39-43).  out is count x elems. */
void or_step_noise(uint64_t seed, int i, int64_t m0, int64_t count, int64_t elems, double* out,
                   int workers);
void or_step_noise_f32(uint64_t seed, int i, int64_t m0, int64_t count, int64_t elems,
                       float* out, int workers);

/* ---- schedule.cpp:9-36 ---- */
int or_make_schedule(int steps, double alpha_bar_final, double* alpha_bar /* steps+1 */,
                     double* alpha /* steps, may be NULL */);
void or_sampling_spread(const double* alpha_bar, int i, double* mean_scale, double* std_dev);

/* ---- dynamics.hpp / dynamics.cpp ---- */
int or_model_dims(int kind, int* dx, int* du, int* pdim);
void or_derivative(int kind, const double* x, const double* u, double* xdot);
void or_rk4_step(int kind, const double* x, const double* u, double dt, double* out);
/* Returns 0, or 1 on a non-finite state (bad_robot/bad_step set as in
 * dynamics.cpp:81-84, step counted from 1).  controls_out may be NULL. */
int or_rollout(const or_problem* p, const double* u, double* states, double* controls_out,
               int* bad_robot, int* bad_step);

/* ---- reward.cpp ---- */
/* total_reward (reward.cpp:67-130).  Optional counts: robot-steps (t>=1) with an
 * inter-robot conflict and with an obstacle hit. Returns 0, or 2 if a robot
 * starts on its goal. */
int or_total_reward(const or_problem* p, const double* states, double* reward,
                    int64_t* n_conflict, int64_t* n_obstacle);
double or_objective(const or_problem* p, const double* states);
/* check_success (reward.cpp:162-200); returns 1 on success, 0 on failure and
 * writes the reference's violation message into msg. */
int or_check_success(const or_problem* p, const double* states, char* msg, int msg_len);

/* ---- denoiser.cpp ---- */
/* score_weights (denoiser.cpp:50-90).  Returns 0, 1 on bad args, 2+j on a
 * non-finite reward j (clamped to INT32_MAX). */
int or_score_weights(const double* rewards, int64_t m, double lambda, double* weights);
double or_weight_entropy(const double* weights, int64_t m);

/* One denoising step i (the body of the loop at denoiser.cpp:152-180).
 *   variable (in/out): (R*du) x T
 *   noise: if non-NULL, count=batch blocks to use instead of the NormalStream
 *          draws (host-supplied noise; must equal or_step_noise output to match
 *          the reference); if NULL the oracle draws them itself.
 *   rewards_out / weights_out (batch) and rec may be NULL.
 * Returns 0 or a nonzero error (see or_last_error()). */
int or_denoise_step(const or_problem* p, const double* base, const double* alpha_bar,
                    const or_denoiser_config* cfg, int i, double* variable, const double* noise,
                    double* rewards_out, double* weights_out, or_trace_rec* rec);

/* mc_average (denoiser.cpp:92-108): samples M x elems, ascending-m sum.
 * Returns 0, or 4 when |Σw − 1| > 1e-9. */
int or_mc_average(const double* samples, const double* w, int64_t M, int64_t elems, double* out);
/* sample_batch (denoiser.cpp:39-46) + mc_average + denoise_step (:110-117)
 * for given weights: out = update_scale · Σ_m w_m (mean_scale·variable + std·z_m). */
int or_weighted_update(const double* variable, const double* noise, const double* w, int64_t M, int64_t elems,
                       double mean_scale, double std_dev, double update_scale, double* out);

/* run_denoising (denoiser.cpp:119-184).  trace has cfg->steps records. */
int or_run_denoising(const or_problem* p, const double* base, const or_denoiser_config* cfg,
                     double* variable_out, or_trace_rec* trace);

typedef struct {
  int max_iterations;
  int stop_on_success;
  double deadline_seconds; /* <= 0: none */
} or_optimizer_config;

typedef struct {
  double reward, objective;
  int success;
  double wall_seconds;
} or_iteration_stats;

/* solve (optimizer.cpp:48-102).  best_states: (R*dx)x(T+1); per_iteration and
 * traces (max_iterations*steps) may be NULL.  Returns iterations used (>0) or
 * a negative error. */
int or_solve(const or_problem* p, const or_denoiser_config* dcfg, const or_optimizer_config* ocfg,
             double* best_states, double* best_controls, double* best_reward, int* success,
             or_iteration_stats* per_iteration, or_trace_rec* traces);

/* ---- baselines.cpp (MPPI / CEM in the joint control space) ---- */
typedef struct {           /* MppiConfig (baselines.hpp:16-27); horizon/dt from the problem */
  int64_t batch;
  double lambda, sigma;
  int iterations;
  uint64_t seed;
  int stop_on_success;
  double deadline_seconds; /* <= 0: none */
  int workers;
} or_mppi_config;

typedef struct {           /* CemConfig (baselines.hpp:31-43) */
  int64_t batch;
  double elite_fraction, initial_std, min_std;
  int iterations;
  uint64_t seed;
  int stop_on_success;
  double deadline_seconds;
  int workers;
} or_cem_config;

/* select_elites (baselines.cpp:86-97): `count` indices, ascending. */
int or_select_elites(const double* rewards, int64_t m, int count, int* out);
/* mppi_solve / cem_solve (baselines.cpp:99-173).  Same outputs as or_solve;
 * returns iterations used (> 0) or -1. */
int or_mppi_solve(const or_problem* p, const or_mppi_config* c, double* best_states, double* best_controls,
                  double* best_reward, int* success, or_iteration_stats* per_it);
int or_cem_solve(const or_problem* p, const or_cem_config* c, double* best_states, double* best_controls,
                 double* best_reward, int* success, or_iteration_stats* per_it);

const char* or_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
