/*
 * d4orm_oracle.c — TEST INFRASTRUCTURE ONLY (see d4orm_oracle.h).
 *
 * fp64 CPU restatement of the reference's denoise-step path.  Every function
 * cites the reference file:line it follows; evaluation order is kept exactly
 * (sequential reductions, Eigen's elementwise expression order, no FMA
 * contraction: build with -ffp-contract=off like the reference's x86-64
 * baseline build, proj/CMakeLists.txt:8-15).
 */
#define _GNU_SOURCE
#include "d4orm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

static __thread char g_err[512];

static void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

const char* or_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ rng */

/* rng.hpp:10-15 */
uint64_t or_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* rng.hpp:17-19 */
uint64_t or_mix_seed(uint64_t a, uint64_t b) {
  return or_splitmix64(or_splitmix64(a) ^ (0x9e3779b97f4a7c15ull + b));
}

/* rng.hpp:21-23 */
uint64_t or_mix_seed3(uint64_t a, uint64_t b, uint64_t c) {
  return or_mix_seed(or_mix_seed(a, b), c);
}

/* std::mt19937_64 — output fixed by the C++ standard [rand.eng.mers]. */
typedef struct {
  uint64_t mt[312];
  int idx;
  int saved_available;
  double saved;
} normal_stream;

static void mt_seed(normal_stream* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  s->idx = 312;
  s->saved_available = 0;
  s->saved = 0.0;
}

static uint64_t mt_next(normal_stream* s) {
  if (s->idx >= 312) {
    const uint64_t upper = 0xffffffff80000000ull, lower = 0x7fffffffull;
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (s->mt[i] & upper) | (s->mt[(i + 1) % 312] & lower);
      uint64_t v = s->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ull) v ^= 0xb5026f5aa96619e9ull;
      s->mt[i] = v;
    }
    s->idx = 0;
  }
  uint64_t z = s->mt[s->idx++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71d67fffeda60000ull;
  z ^= (z << 37) & 0xfff7eee000000000ull;
  z ^= z >> 43;
  return z;
}

/* std::generate_canonical<double, 53>(mt19937_64) as implemented by libstdc++
 * (bits/random.tcc): one 64-bit draw, divided by 2^64, clamped below 1. */
static double canonical(normal_stream* s) {
  double r = (double)mt_next(s) / 18446744073709551616.0;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r;
}

/* std::normal_distribution<double>(0,1)::operator() as implemented by
 * libstdc++ (Marsaglia polar method, the second deviate cached). The reference
 * reaches it via NormalStream (rng.hpp:27-40); the algorithm is
 * implementation-defined, so this mirrors the toolchain the reference is built
 * with here (g++ 13 / libstdc++), pinned bitwise against oracle/_ref. */
static double normal_next(normal_stream* s) {
  double ret;
  if (s->saved_available) {
    s->saved_available = 0;
    ret = s->saved;
  } else {
    double x, y, r2;
    do {
      x = 2.0 * canonical(s) - 1.0;
      y = 2.0 * canonical(s) - 1.0;
      r2 = x * x + y * y;
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = sqrt(-2.0 * log(r2) / r2);
    s->saved = x * mult;
    s->saved_available = 1;
    ret = y * mult;
  }
  return ret * 1.0 + 0.0;
}

/* NormalStream::fill (rng.hpp:33-35) */
void or_normal_fill(uint64_t stream_seed, double* out, int64_t count) {
  normal_stream s;
  mt_seed(&s, stream_seed);
  for (int64_t i = 0; i < count; ++i) out[i] = normal_next(&s);
}

/* ------------------------------------------------------------ parallel_for */

/* parallel.hpp:12-16 */
static int resolve_workers(int workers) {
  if (workers > 0) return workers;
  long hw = sysconf(_SC_NPROCESSORS_ONLN);
  return hw <= 0 ? 1 : (int)hw;
}

typedef void (*pf_fn)(int64_t i, void* ctx);
typedef struct {
  int64_t count;
  int w, workers;
  pf_fn fn;
  void* ctx;
} pf_job;

static void* pf_thread(void* arg) {
  pf_job* j = (pf_job*)arg;
  for (int64_t i = j->w; i < j->count; i += j->workers) j->fn(i, j->ctx);
  return NULL;
}

/* parallel.hpp:21-45 — indices interleaved i = w, w+W, ...; results owned per
 * index, so they never depend on the worker count. */
static void parallel_for(int64_t count, int workers, pf_fn fn, void* ctx) {
  if (count <= 0) return;
  workers = resolve_workers(workers);
  if (workers > count) workers = (int)count;
  if (workers <= 1) {
    for (int64_t i = 0; i < count; ++i) fn(i, ctx);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * workers);
  pf_job* jobs = (pf_job*)malloc(sizeof(pf_job) * workers);
  for (int w = 0; w < workers; ++w) {
    jobs[w] = (pf_job){count, w, workers, fn, ctx};
    pthread_create(&th[w], NULL, pf_thread, &jobs[w]);
  }
  for (int w = 0; w < workers; ++w) pthread_join(th[w], NULL);
  free(th);
  free(jobs);
}

typedef struct {
  uint64_t seed;
  int i;
  int64_t m0, elems;
  double* out64;
  float* out32;
} noise_ctx;

static void noise_one(int64_t j, void* c) {
  noise_ctx* n = (noise_ctx*)c;
  const uint64_t ss = or_mix_seed3(n->seed, (uint64_t)n->i, (uint64_t)(n->m0 + j));
  if (n->out64) {
    or_normal_fill(ss, n->out64 + j * n->elems, n->elems);
  } else {
    normal_stream s;
    mt_seed(&s, ss);
    float* o = n->out32 + j * n->elems;
    for (int64_t e = 0; e < n->elems; ++e) o[e] = (float)normal_next(&s);
  }
}

/* denoiser.cpp:39-43 (normal_matrix with stream mix_seed(seed, i, m)) */
void or_step_noise(uint64_t seed, int i, int64_t m0, int64_t count, int64_t elems, double* out,
                   int workers) {
  noise_ctx c = {seed, i, m0, elems, out, NULL};
  parallel_for(count, workers, noise_one, &c);
}

void or_step_noise_f32(uint64_t seed, int i, int64_t m0, int64_t count, int64_t elems,
                       float* out, int workers) {
  noise_ctx c = {seed, i, m0, elems, NULL, out};
  parallel_for(count, workers, noise_one, &c);
}

/* ------------------------------------------------------------- schedule */

/* schedule.cpp:9-27 */
int or_make_schedule(int steps, double alpha_bar_final, double* alpha_bar, double* alpha) {
  if (steps < 1) {
    set_err("make_schedule: steps must be >= 1, got %d", steps);
    return 1;
  }
  if (!(alpha_bar_final > 0.0) || !(alpha_bar_final < 1.0)) {
    set_err("make_schedule: alpha_bar_final must lie in (0, 1), got %f", alpha_bar_final);
    return 1;
  }
  alpha_bar[0] = 1.0;
  for (int i = 1; i <= steps; ++i) {
    alpha_bar[i] = pow(alpha_bar_final, (double)i / steps);
    if (alpha) alpha[i - 1] = alpha_bar[i] / alpha_bar[i - 1];
  }
  return 0;
}

/* schedule.cpp:29-36 */
void or_sampling_spread(const double* alpha_bar, int i, double* mean_scale, double* std_dev) {
  const double ab = alpha_bar[i];
  *mean_scale = 1.0 / sqrt(ab);
  *std_dev = sqrt(1.0 / ab - 1.0);
}

/* ------------------------------------------------------------- dynamics */

int or_model_dims(int kind, int* dx, int* du, int* pdim) {
  static const int DX[6] = {4, 4, 6, 2, 3, 3};
  static const int DU[6] = {2, 2, 3, 2, 3, 2};
  static const int PD[6] = {2, 2, 3, 2, 3, 2};
  if (kind < 0 || kind > 5) return 1;
  *dx = DX[kind];
  *du = DU[kind];
  *pdim = PD[kind];
  return 0;
}

/* Derivative functors: dynamics.hpp:81-93 (DiffDrive), :95-106 (Holo2D),
 * :108-119 (Holo3D); the three extensions follow the same pattern. */
void or_derivative(int kind, const double* x, const double* u, double* f) {
  switch (kind) {
    case OR_DIFFDRIVE: {
      const double theta = x[2], v = x[3];
      f[0] = v * cos(theta);
      f[1] = v * sin(theta);
      f[2] = u[0];
      f[3] = u[1];
      break;
    }
    case OR_HOLO2D:
      f[0] = x[2]; f[1] = x[3]; f[2] = u[0]; f[3] = u[1];
      break;
    case OR_HOLO3D:
      f[0] = x[3]; f[1] = x[4]; f[2] = x[5]; f[3] = u[0]; f[4] = u[1]; f[5] = u[2];
      break;
    case OR_HOLO2D_VEL:
      f[0] = u[0]; f[1] = u[1];
      break;
    case OR_HOLO3D_VEL:
      f[0] = u[0]; f[1] = u[1]; f[2] = u[2];
      break;
    case OR_UNICYCLE: {
      const double theta = x[2];
      f[0] = u[0] * cos(theta);
      f[1] = u[0] * sin(theta);
      f[2] = u[1];
      break;
    }
  }
}

/* detail::rk4_with (dynamics.hpp:123-130), Eigen's lazy expressions evaluated
 * per element in source order:
 *   k2 = f(x + (0.5*dt)*k1), k3 = f(x + (0.5*dt)*k2), k4 = f(x + dt*k3)
 *   out = x + (dt/6)*(((k1 + 2*k2) + 2*k3) + k4)                          */
void or_rk4_step(int kind, const double* x, const double* u, double dt, double* out) {
  int dx, du, pd;
  or_model_dims(kind, &dx, &du, &pd);
  double k1[6], k2[6], k3[6], k4[6], tmp[6];
  const double h = 0.5 * dt;
  or_derivative(kind, x, u, k1);
  for (int j = 0; j < dx; ++j) tmp[j] = x[j] + h * k1[j];
  or_derivative(kind, tmp, u, k2);
  for (int j = 0; j < dx; ++j) tmp[j] = x[j] + h * k2[j];
  or_derivative(kind, tmp, u, k3);
  for (int j = 0; j < dx; ++j) tmp[j] = x[j] + dt * k3[j];
  or_derivative(kind, tmp, u, k4);
  const double s = dt / 6.0;
  for (int j = 0; j < dx; ++j) out[j] = x[j] + s * (((k1[j] + 2.0 * k2[j]) + 2.0 * k3[j]) + k4[j]);
}

/* rollout (dynamics.cpp:122-169) + rollout_robot<DX,DU> (dynamics.cpp:65-87):
 * clamp = raw.cwiseMax(lower).cwiseMin(upper), stored as the executed control;
 * RK4; non-finite check naming robot k and step t+1. */
int or_rollout(const or_problem* p, const double* u, double* states, double* controls_out,
               int* bad_robot, int* bad_step) {
  const int R = p->robots, T = p->horizon, dx = p->dx, du = p->du;
  if (controls_out) memset(controls_out, 0, sizeof(double) * (size_t)R * du * (T + 1));
  for (int k = 0; k < R; ++k) {
    double x[6], xn[6], uc[3];
    for (int j = 0; j < dx; ++j) x[j] = p->starts[k * dx + j];
    for (int j = 0; j < dx; ++j) states[(size_t)k * dx + j] = x[j];
    for (int t = 0; t < T; ++t) {
      const double* raw = u + (size_t)t * R * du + (size_t)k * du;
      for (int d = 0; d < du; ++d) {
        double v = raw[d];
        v = (v < p->lower[d]) ? p->lower[d] : v;  /* std::max(v, lower) */
        v = (p->upper[d] < v) ? p->upper[d] : v;  /* std::min(v, upper) */
        uc[d] = v;
        if (controls_out) controls_out[(size_t)t * R * du + (size_t)k * du + d] = v;
      }
      or_rk4_step(p->kind, x, uc, p->dt, xn);
      for (int j = 0; j < dx; ++j) {
        if (!isfinite(xn[j])) {
          if (bad_robot) *bad_robot = k;
          if (bad_step) *bad_step = t + 1;
          set_err("rollout: non-finite state for robot %d at step %d", k, t + 1);
          return 1;
        }
      }
      for (int j = 0; j < dx; ++j) {
        x[j] = xn[j];
        states[(size_t)(t + 1) * R * dx + (size_t)k * dx + j] = x[j];
      }
    }
  }
  return 0;
}

/* --------------------------------------------------------------- reward */

static double start_goal_distance(const or_problem* p, int k) {
  double s = 0.0;
  for (int j = 0; j < p->pdim; ++j) {
    const double d = p->starts[(size_t)k * p->dx + j] - p->goals[(size_t)k * p->pdim + j];
    s += d * d;
  }
  return sqrt(s);
}

/* total_reward (reward.cpp:67-130): hoisted start distances (:79-86), t-major
 * k-minor sum (:88-129), pair test with break at the first hit (:99-110),
 * obstacle test with break (:112-125), divide by n*H (:129). */
int or_total_reward(const or_problem* p, const double* states, double* reward,
                    int64_t* n_conflict, int64_t* n_obstacle) {
  const int n = p->robots, H = p->horizon, pd = p->pdim, dx = p->dx;
  const double margin = 2.0 * p->robot_radius + p->epsilon;
  const double margin_sq = margin * margin;
  double sd[256];
  double* start_dist = n <= 256 ? sd : (double*)malloc(sizeof(double) * n);
  for (int k = 0; k < n; ++k) {
    start_dist[k] = start_goal_distance(p, k);
    if (!(start_dist[k] > 0.0)) {
      set_err("total_reward: robot %d starts on its goal (degenerate scenario)", k);
      if (start_dist != sd) free(start_dist);
      return 2;
    }
  }
  int64_t nc = 0, no = 0;
  double sum = 0.0;
  for (int t = 1; t <= H; ++t) {
    const double* col = states + (size_t)t * n * dx;
    for (int k = 0; k < n; ++k) {
      double gsq = 0.0;
      for (int j = 0; j < pd; ++j) {
        const double d = col[k * dx + j] - p->goals[(size_t)k * pd + j];
        gsq += d * d;
      }
      double value = 1.0 - sqrt(gsq) / start_dist[k];
      for (int l = 0; l < n; ++l) {
        if (l == k) continue;
        double psq = 0.0;
        for (int j = 0; j < pd; ++j) {
          const double d = col[k * dx + j] - col[l * dx + j];
          psq += d * d;
        }
        if (psq <= margin_sq) {
          value -= p->w_t;
          ++nc;
          break;
        }
      }
      for (int o = 0; o < p->n_obstacles; ++o) {
        double osq = 0.0;
        for (int j = 0; j < pd; ++j) {
          const double d = col[k * dx + j] - p->obs_centers[(size_t)o * pd + j];
          osq += d * d;
        }
        const double limit = p->obs_radii[o] + p->robot_radius;
        if (osq <= limit * limit) {
          value -= p->obstacle_weight;
          ++no;
          break;
        }
      }
      sum += value;
    }
  }
  if (start_dist != sd) free(start_dist);
  *reward = sum / ((double)n * H);
  if (n_conflict) *n_conflict = nc;
  if (n_obstacle) *n_obstacle = no;
  return 0;
}

/* objective (reward.cpp:136-156) */
double or_objective(const or_problem* p, const double* states) {
  const int n = p->robots, H = p->horizon, pd = p->pdim, dx = p->dx;
  const double tol_sq = p->goal_tolerance * p->goal_tolerance;
  long hits = 0;
  for (int t = 1; t <= H; ++t) {
    for (int k = 0; k < n; ++k) {
      double g = 0.0;
      for (int j = 0; j < pd; ++j) {
        const double d = states[(size_t)t * n * dx + (size_t)k * dx + j] - p->goals[(size_t)k * pd + j];
        g += d * d;
      }
      if (g <= tol_sq) ++hits;
    }
  }
  return (double)hits / ((double)n * H);
}

/* check_success (reward.cpp:162-200) — strict 2R_a at every step incl. t=0,
 * obstacles, then the terminal goal ball. */
int or_check_success(const or_problem* p, const double* states, char* msg, int msg_len) {
  const int n = p->robots, H = p->horizon, pd = p->pdim, dx = p->dx;
  const double safety_sq = 4.0 * p->robot_radius * p->robot_radius;
  char local[256];
  if (!msg) { msg = local; msg_len = sizeof local; }
  msg[0] = 0;
  for (int t = 0; t <= H; ++t) {
    const double* col = states + (size_t)t * n * dx;
    for (int k = 0; k < n; ++k) {
      for (int l = k + 1; l < n; ++l) {
        double s = 0.0;
        for (int j = 0; j < pd; ++j) {
          const double d = col[k * dx + j] - col[l * dx + j];
          s += d * d;
        }
        if (s <= safety_sq) {
          snprintf(msg, msg_len, "safety: robots %d and %d within 2*R_a at step %d", k, l, t);
          return 0;
        }
      }
      for (int o = 0; o < p->n_obstacles; ++o) {
        double s = 0.0;
        for (int j = 0; j < pd; ++j) {
          const double d = col[k * dx + j] - p->obs_centers[(size_t)o * pd + j];
          s += d * d;
        }
        const double limit = p->obs_radii[o] + p->robot_radius;
        if (s <= limit * limit) {
          snprintf(msg, msg_len, "obstacle: robot %d hits obstacle %d at step %d", k, o, t);
          return 0;
        }
      }
    }
  }
  for (int k = 0; k < n; ++k) {
    double s = 0.0;
    for (int j = 0; j < pd; ++j) {
      const double d = states[(size_t)H * n * dx + (size_t)k * dx + j] - p->goals[(size_t)k * pd + j];
      s += d * d;
    }
    const double end_dist = sqrt(s);
    if (end_dist > p->goal_tolerance) {
      snprintf(msg, msg_len, "terminal: robot %d ends %f m from its goal (tolerance %f)", k,
               end_dist, p->goal_tolerance);
      return 0;
    }
  }
  return 1;
}

/* ------------------------------------------------------------- denoiser */

/* score_weights (denoiser.cpp:50-90) */
int or_score_weights(const double* rewards, int64_t m, double lambda, double* w) {
  if (m < 2) {
    set_err("score_weights: need at least 2 rewards");
    return 1;
  }
  if (!(lambda > 0.0)) {
    set_err("score_weights: lambda must be positive");
    return 1;
  }
  for (int64_t j = 0; j < m; ++j) {
    if (!isfinite(rewards[j])) {
      set_err("score_weights: non-finite reward for sample %lld", (long long)j);
      return j + 2 > 0x7fffffff ? 0x7fffffff : (int)(j + 2);
    }
  }
  double mean = 0.0;
  for (int64_t j = 0; j < m; ++j) mean += rewards[j];
  mean /= (double)m;
  double var = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double d = rewards[j] - mean;
    var += d * d;
  }
  const double std_dev = sqrt(var / (double)m);
  if (std_dev < 1e-8) {
    for (int64_t j = 0; j < m; ++j) w[j] = 1.0 / (double)m;
    return 0;
  }
  double max_scaled = -INFINITY;
  for (int64_t j = 0; j < m; ++j) {
    w[j] = (rewards[j] - mean) / std_dev / lambda;
    max_scaled = max_scaled < w[j] ? w[j] : max_scaled; /* std::max(max, w) */
  }
  double sum = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    w[j] = exp(w[j] - max_scaled);
    sum += w[j];
  }
  for (int64_t j = 0; j < m; ++j) w[j] /= sum;
  return 0;
}

/* weight_entropy (denoiser.cpp:24-30) */
double or_weight_entropy(const double* w, int64_t m) {
  double h = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    if (w[j] > 0.0) h -= w[j] * log(w[j]);
  }
  return h;
}

typedef struct {
  const or_problem* p;
  const double* base;
  const double* variable;
  const double* noise;  /* batch x elems, or NULL */
  double* samples;      /* batch x elems */
  double* rewards;
  double mean_scale, std_dev;
  uint64_t seed;
  int i, deform;
  int64_t elems;
  int* failed;          /* per-sample error flags */
  char (*errs)[160];
} step_ctx;

static void sample_one(int64_t m, void* c) {
  step_ctx* s = (step_ctx*)c;
  double* out = s->samples + m * s->elems;
  /* sample_batch (denoiser.cpp:39-46): mean_scale*current + std*z */
  if (s->noise) {
    memcpy(out, s->noise + m * s->elems, sizeof(double) * (size_t)s->elems);
  } else {
    or_normal_fill(or_mix_seed3(s->seed, (uint64_t)s->i, (uint64_t)m), out, s->elems);
  }
  for (int64_t e = 0; e < s->elems; ++e) out[e] = s->mean_scale * s->variable[e] + s->std_dev * out[e];
}

static void evaluate_one(int64_t m, void* c) {
  step_ctx* s = (step_ctx*)c;
  const or_problem* p = s->p;
  const double* smp = s->samples + m * s->elems;
  double* cand = (double*)malloc(sizeof(double) * (size_t)s->elems);
  double* states = (double*)malloc(sizeof(double) * (size_t)p->robots * p->dx * (p->horizon + 1));
  /* denoiser.cpp:158-160: candidate = base + sample (Deformation) | sample */
  for (int64_t e = 0; e < s->elems; ++e) cand[e] = s->deform ? s->base[e] + smp[e] : smp[e];
  int br = 0, bs = 0;
  if (or_rollout(p, cand, states, NULL, &br, &bs) != 0) {
    s->failed[m] = 1;
    snprintf(s->errs[m], 160, "rollout: non-finite state for robot %d at step %d", br, bs);
  } else if (or_total_reward(p, states, &s->rewards[m], NULL, NULL) != 0) {
    s->failed[m] = 1;
    snprintf(s->errs[m], 160, "%s", g_err);
  }
  free(cand);
  free(states);
}

/* One iteration of the loop body at denoiser.cpp:152-180. */
int or_denoise_step(const or_problem* p, const double* base, const double* alpha_bar,
                    const or_denoiser_config* cfg, int i, double* variable, const double* noise,
                    double* rewards_out, double* weights_out, or_trace_rec* rec) {
  const int64_t M = cfg->batch;
  const int64_t elems = (int64_t)p->robots * p->du * p->horizon;
  step_ctx s;
  memset(&s, 0, sizeof s);
  s.p = p;
  s.base = base;
  s.variable = variable;
  s.noise = noise;
  s.seed = cfg->seed;
  s.i = i;
  s.deform = cfg->mode == 1;
  s.elems = elems;
  or_sampling_spread(alpha_bar, i, &s.mean_scale, &s.std_dev);
  s.samples = (double*)malloc(sizeof(double) * (size_t)(M * elems));
  s.rewards = rewards_out ? rewards_out : (double*)malloc(sizeof(double) * (size_t)M);
  s.failed = (int*)calloc((size_t)M, sizeof(int));
  s.errs = (char (*)[160])calloc((size_t)M, 160);
  double* w = weights_out ? weights_out : (double*)malloc(sizeof(double) * (size_t)M);
  int rc = 0;
  if (!s.samples || !s.failed || !s.errs) {
    set_err("or_denoise_step: out of memory");
    rc = 1;
    goto done;
  }
  parallel_for(M, cfg->workers, sample_one, &s);
  parallel_for(M, cfg->workers, evaluate_one, &s);
  for (int64_t m = 0; m < M; ++m) {
    if (s.failed[m]) { /* first exception by index (parallel.hpp:31-44 keeps the first thrown) */
      set_err("run_denoising: sample %lld at step %d: %s", (long long)m, i, s.errs[m]);
      rc = 3;
      goto done;
    }
  }
  rc = or_score_weights(s.rewards, M, cfg->lambda, w);
  if (rc) goto done;
  {
    /* mc_average (denoiser.cpp:92-108): check sum, ascending-m accumulation */
    double sum = 0.0;
    for (int64_t m = 0; m < M; ++m) sum += w[m];
    if (fabs(sum - 1.0) > 1e-9) {
      set_err("mc_average: weights must sum to 1");
      rc = 4;
      goto done;
    }
    double* acc = (double*)calloc((size_t)elems, sizeof(double));
    for (int64_t m = 0; m < M; ++m) {
      const double* smp = s.samples + m * elems;
      const double wm = w[m];
      for (int64_t e = 0; e < elems; ++e) acc[e] = acc[e] + wm * smp[e];
    }
    /* denoise_step (denoiser.cpp:110-117) */
    const double scale = sqrt(alpha_bar[i - 1]);
    for (int64_t e = 0; e < elems; ++e) variable[e] = scale * acc[e];
    free(acc);
  }
  if (rec) {
    /* trace (denoiser.cpp:172-179) */
    double best = s.rewards[0], mean = 0.0;
    for (int64_t m = 0; m < M; ++m) {
      best = best < s.rewards[m] ? s.rewards[m] : best;
      mean += s.rewards[m];
    }
    mean /= (double)M;
    rec->step = i;
    rec->best_reward = best;
    rec->mean_reward = mean;
    rec->weight_entropy = or_weight_entropy(w, M);
  }
done:
  free(s.samples);
  if (!rewards_out) free(s.rewards);
  if (!weights_out) free(w);
  free(s.failed);
  free(s.errs);
  return rc;
}

/* mc_average (denoiser.cpp:92-108): |Σw − 1| ≤ 1e-9, then out = Σ_m w_m·sample_m
 * accumulated in ascending m, one element at a time. */
int or_mc_average(const double* samples, const double* w, int64_t M, int64_t elems, double* out) {
  double sum = 0.0;
  for (int64_t m = 0; m < M; ++m) sum += w[m];
  if (fabs(sum - 1.0) > 1e-9) {
    set_err("mc_average: weights must sum to 1");
    return 4;
  }
  for (int64_t e = 0; e < elems; ++e) out[e] = 0.0;
  for (int64_t m = 0; m < M; ++m) {
    const double* smp = samples + m * elems;
    const double wm = w[m];
    for (int64_t e = 0; e < elems; ++e) out[e] = out[e] + wm * smp[e];
  }
  return 0;
}

/* The tail of one denoising step for given weights: sample_batch
 * (denoiser.cpp:39-46, sample_m = mean_scale·variable + std·z_m) formed one
 * sample at a time, mc_average (:92-108) in ascending m, then denoise_step
 * (:110-117) variable' = update_scale·average.  Same arithmetic as
 * or_denoise_step's tail without holding the M sample matrices. */
int or_weighted_update(const double* variable, const double* noise, const double* w, int64_t M, int64_t elems,
                       double mean_scale, double std_dev, double update_scale, double* out) {
  double sum = 0.0;
  for (int64_t m = 0; m < M; ++m) sum += w[m];
  if (fabs(sum - 1.0) > 1e-9) {
    set_err("mc_average: weights must sum to 1");
    return 4;
  }
  double* acc = (double*)calloc((size_t)elems, sizeof(double));
  for (int64_t m = 0; m < M; ++m) {
    const double* z = noise + m * elems;
    const double wm = w[m];
    for (int64_t e = 0; e < elems; ++e) {
      const double smp = mean_scale * variable[e] + std_dev * z[e];
      acc[e] = acc[e] + wm * smp;
    }
  }
  for (int64_t e = 0; e < elems; ++e) out[e] = update_scale * acc[e];
  free(acc);
  return 0;
}

/* run_denoising (denoiser.cpp:119-184) */
int or_run_denoising(const or_problem* p, const double* base, const or_denoiser_config* cfg,
                     double* variable, or_trace_rec* trace) {
  if (cfg->batch < 2) { set_err("run_denoising: batch must be >= 2"); return 1; }
  if (!(cfg->lambda > 0.0)) { set_err("run_denoising: lambda must be > 0"); return 1; }
  const int64_t elems = (int64_t)p->robots * p->du * p->horizon;
  double* ab = (double*)malloc(sizeof(double) * (size_t)(cfg->steps + 1));
  int rc = or_make_schedule(cfg->steps, cfg->alpha_bar_final, ab, NULL);
  if (rc) { free(ab); return rc; }
  if (cfg->mode == 1) {
    memset(variable, 0, sizeof(double) * (size_t)elems);
  } else {
    /* step index 0 stream is free for the initial draw (denoiser.cpp:141-145) */
    or_normal_fill(or_mix_seed3(cfg->seed, 0, 0), variable, elems);
  }
  for (int i = cfg->steps; i >= 1; --i) {
    rc = or_denoise_step(p, base, ab, cfg, i, variable, NULL, NULL, NULL,
                         trace ? &trace[cfg->steps - i] : NULL);
    if (rc) break;
  }
  free(ab);
  return rc;
}

/* ------------------------------------------------------------ optimizer */

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + ts.tv_nsec * 1e-9;
}

/* solve (optimizer.cpp:48-102) with iterate_impl (optimizer.cpp:19-29). */
int or_solve(const or_problem* p, const or_denoiser_config* dcfg, const or_optimizer_config* ocfg,
             double* best_states, double* best_controls, double* best_reward, int* success,
             or_iteration_stats* per_iteration, or_trace_rec* traces) {
  if (ocfg->max_iterations < 1) { set_err("solve: max_iterations must be >= 1"); return -1; }
  if (p->horizon < 2) { set_err("solve: horizon must be >= 2"); return -1; }
  const int R = p->robots, T = p->horizon;
  const size_t ns = (size_t)R * p->dx * (T + 1), nc = (size_t)R * p->du * (T + 1);
  const size_t elems = (size_t)R * p->du * T;
  double* states = (double*)malloc(sizeof(double) * ns);
  double* controls = (double*)malloc(sizeof(double) * nc);
  double* base = (double*)malloc(sizeof(double) * elems);
  double* delta = (double*)malloc(sizeof(double) * elems);
  const double t0 = now_s();
  int used = 0, rc = 0, best_it = -1;
  memset(base, 0, sizeof(double) * elems);
  if (or_rollout(p, base, states, controls, NULL, NULL)) { rc = -1; goto out; }
  for (int it = 1; it <= ocfg->max_iterations; ++it) {
    or_denoiser_config c = *dcfg;
    c.mode = 1;
    c.seed = or_mix_seed(dcfg->seed, (uint64_t)it);
    memcpy(base, controls, sizeof(double) * elems); /* executed_controls: leftCols(H) */
    rc = or_run_denoising(p, base, &c, delta, traces ? traces + (size_t)(it - 1) * dcfg->steps : NULL);
    if (rc) { rc = -1; goto out; }
    for (size_t e = 0; e < elems; ++e) delta[e] = base[e] + delta[e];
    if (or_rollout(p, delta, states, controls, NULL, NULL)) { rc = -1; goto out; }
    double reward;
    or_total_reward(p, states, &reward, NULL, NULL);
    const double quality = or_objective(p, states);
    const int ok = or_check_success(p, states, NULL, 0);
    if (per_iteration) per_iteration[it - 1] = (or_iteration_stats){reward, quality, ok, now_s() - t0};
    used = it;
    if (best_it < 0 || reward > *best_reward) {
      *best_reward = reward;
      memcpy(best_states, states, sizeof(double) * ns);
      if (best_controls) memcpy(best_controls, controls, sizeof(double) * nc);
      best_it = it;
    }
    if (ocfg->stop_on_success && ok) break;
    if (ocfg->deadline_seconds > 0 && now_s() - t0 >= ocfg->deadline_seconds) break;
  }
  *success = or_check_success(p, best_states, NULL, 0);
  rc = used;
out:
  free(states);
  free(controls);
  free(base);
  free(delta);
  return rc;
}

/* ------------------------------------------------------------ baselines */
/* MPPI and CEM in the joint control space (baselines.cpp:19-173): the same
 * rollout / total_reward / score_weights / mc_average pieces, no schedule. */

typedef struct {
  const or_problem* p;
  const double* mean;
  const double* stdv;   /* CEM: per-element std; NULL → MPPI scalar sigma */
  double sigma;
  uint64_t seed;
  int it;
  int64_t elems;
  double* samples;      /* batch x elems */
  double* rewards;
  int* failed;
  char (*errs)[160];
} base_ctx;

static void base_sample_one(int64_t m, void* c) {
  base_ctx* b = (base_ctx*)c;
  double* out = b->samples + m * b->elems;
  /* normal_matrix with stream mix_seed(seed, iteration, m) (baselines.cpp:116-119,152-155) */
  or_normal_fill(or_mix_seed3(b->seed, (uint64_t)b->it, (uint64_t)m), out, b->elems);
  for (int64_t e = 0; e < b->elems; ++e)  /* mean.u + sigma*z | mean.u + std.cwiseProduct(z) */
    out[e] = b->stdv ? b->mean[e] + b->stdv[e] * out[e] : b->mean[e] + b->sigma * out[e];
}

static void base_eval_one(int64_t m, void* c) {  /* evaluate_batch (baselines.cpp:30-38) */
  base_ctx* b = (base_ctx*)c;
  const or_problem* p = b->p;
  double* states = (double*)malloc(sizeof(double) * (size_t)p->robots * p->dx * (p->horizon + 1));
  int br = 0, bs = 0;
  if (or_rollout(p, b->samples + m * b->elems, states, NULL, &br, &bs) != 0) {
    b->failed[m] = 1;
    snprintf(b->errs[m], 160, "rollout: non-finite state for robot %d at step %d", br, bs);
  } else if (or_total_reward(p, states, &b->rewards[m], NULL, NULL) != 0) {
    b->failed[m] = 1;
    snprintf(b->errs[m], 160, "%s", g_err);
  }
  free(states);
}

static int base_evaluate(base_ctx* b, int64_t M, int workers) {
  parallel_for(M, workers, base_sample_one, b);
  parallel_for(M, workers, base_eval_one, b);
  for (int64_t m = 0; m < M; ++m)
    if (b->failed[m]) { set_err("%s", b->errs[m]); return 1; }
  return 0;
}

/* run_anytime's per-iteration bookkeeping (baselines.cpp:45-75) on `mean`. */
typedef struct {
  double* states;
  double* controls;
  int best_it, used;
  double t0;
} anytime_ctx;

static int anytime_record(const or_problem* p, anytime_ctx* a, const double* mean, int it,
                          double* best_states, double* best_controls, double* best_reward,
                          or_iteration_stats* per_it, int* ok_out) {
  const size_t ns = (size_t)p->robots * p->dx * (p->horizon + 1), nc = (size_t)p->robots * p->du * (p->horizon + 1);
  if (or_rollout(p, mean, a->states, a->controls, NULL, NULL)) return 1;
  double reward;
  or_total_reward(p, a->states, &reward, NULL, NULL);
  const double quality = or_objective(p, a->states);
  const int ok = or_check_success(p, a->states, NULL, 0);
  if (per_it) per_it[it - 1] = (or_iteration_stats){reward, quality, ok, now_s() - a->t0};
  a->used = it;
  if (a->best_it < 0 || reward > *best_reward) {
    *best_reward = reward;
    memcpy(best_states, a->states, sizeof(double) * ns);
    if (best_controls) memcpy(best_controls, a->controls, sizeof(double) * nc);
    a->best_it = it;
  }
  *ok_out = ok;
  return 0;
}

static int check_base_problem(const or_problem* p, int64_t batch, const char* what) {
  if (p->horizon < 2) { set_err("%s: horizon must be >= 2", what); return 1; }
  if (!(p->dt > 0.0)) { set_err("%s: dt must be positive", what); return 1; }
  if (batch < 2) { set_err("%s: batch must be >= 2", what); return 1; }
  return 0;
}

static const double* g_elite_r;
static int elite_cmp(const void* a, const void* b) {  /* reward descending, index ascending */
  const int i = *(const int*)a, j = *(const int*)b;
  const double ri = g_elite_r[i], rj = g_elite_r[j];
  if (ri > rj) return -1;
  if (rj > ri) return 1;
  return (i > j) - (i < j);
}
static int int_cmp(const void* a, const void* b) {
  const int i = *(const int*)a, j = *(const int*)b;
  return (i > j) - (i < j);
}

/* select_elites (baselines.cpp:86-97): stable sort by reward descending (ties →
 * lower index first), keep `count`, return them in ascending index order. */
int or_select_elites(const double* rewards, int64_t m, int count, int* out) {
  if (count < 1 || count > m) { set_err("select_elites: elite count out of range"); return 1; }
  int* order = (int*)malloc(sizeof(int) * (size_t)m);
  for (int64_t i = 0; i < m; ++i) order[i] = (int)i;
  g_elite_r = rewards;  /* not re-entrant: test infrastructure */
  qsort(order, (size_t)m, sizeof(int), elite_cmp);
  qsort(order, (size_t)count, sizeof(int), int_cmp);
  memcpy(out, order, sizeof(int) * (size_t)count);
  free(order);
  return 0;
}

/* mppi_solve (baselines.cpp:99-129) */
int or_mppi_solve(const or_problem* p, const or_mppi_config* c, double* best_states, double* best_controls,
                  double* best_reward, int* success, or_iteration_stats* per_it) {
  if (check_base_problem(p, c->batch, "mppi_solve")) return -1;
  if (!(c->sigma > 0.0)) { set_err("mppi_solve: sigma must be positive"); return -1; }
  if (c->iterations < 1) { set_err("mppi_solve: iterations must be >= 1"); return -1; }
  const int64_t M = c->batch, E = (int64_t)p->robots * p->du * p->horizon;
  double* mean = (double*)calloc((size_t)E, sizeof(double));
  double* w = (double*)malloc(sizeof(double) * (size_t)M);
  base_ctx b = {p, mean, NULL, c->sigma, c->seed, 0, E, (double*)malloc(sizeof(double) * (size_t)(M * E)),
                (double*)malloc(sizeof(double) * (size_t)M), (int*)calloc((size_t)M, sizeof(int)),
                (char (*)[160])calloc((size_t)M, 160)};
  anytime_ctx a = {(double*)malloc(sizeof(double) * (size_t)p->robots * p->dx * (p->horizon + 1)),
                   (double*)malloc(sizeof(double) * (size_t)p->robots * p->du * (p->horizon + 1)), -1, 0, now_s()};
  int rc = 0;
  for (int it = 1; it <= c->iterations; ++it) {
    b.it = it;
    if (base_evaluate(&b, M, c->workers)) { rc = -1; break; }
    if (or_score_weights(b.rewards, M, c->lambda, w)) { rc = -1; break; }
    double sum = 0.0;  /* mc_average (denoiser.cpp:92-108) */
    for (int64_t m = 0; m < M; ++m) sum += w[m];
    if (fabs(sum - 1.0) > 1e-9) { set_err("mc_average: weights must sum to 1"); rc = -1; break; }
    memset(mean, 0, sizeof(double) * (size_t)E);
    for (int64_t m = 0; m < M; ++m)
      for (int64_t e = 0; e < E; ++e) mean[e] = mean[e] + w[m] * b.samples[m * E + e];
    int ok = 0;
    if (anytime_record(p, &a, mean, it, best_states, best_controls, best_reward, per_it, &ok)) { rc = -1; break; }
    if (c->stop_on_success && ok) break;
    if (c->deadline_seconds > 0 && now_s() - a.t0 >= c->deadline_seconds) break;
  }
  if (rc == 0) {
    *success = or_check_success(p, best_states, NULL, 0);
    rc = a.used;
  }
  free(mean); free(w); free(b.samples); free(b.rewards); free(b.failed); free(b.errs);
  free(a.states); free(a.controls);
  return rc;
}

/* cem_solve (baselines.cpp:131-173) */
int or_cem_solve(const or_problem* p, const or_cem_config* c, double* best_states, double* best_controls,
                 double* best_reward, int* success, or_iteration_stats* per_it) {
  if (check_base_problem(p, c->batch, "cem_solve")) return -1;
  if (!(c->elite_fraction > 0.0) || !(c->elite_fraction < 1.0)) {
    set_err("cem_solve: elite_fraction must lie in (0, 1)");
    return -1;
  }
  const int k = (int)(c->elite_fraction * (double)c->batch);
  if (k < 1) { set_err("cem_solve: elite_fraction * batch must be >= 1"); return -1; }
  if (!(c->initial_std > 0.0) || !(c->min_std > 0.0)) { set_err("cem_solve: stds must be positive"); return -1; }
  if (c->iterations < 1) { set_err("cem_solve: iterations must be >= 1"); return -1; }
  const int64_t M = c->batch, E = (int64_t)p->robots * p->du * p->horizon;
  double* mean = (double*)calloc((size_t)E, sizeof(double));
  double* stdv = (double*)malloc(sizeof(double) * (size_t)E);
  double* nm = (double*)malloc(sizeof(double) * (size_t)E);
  double* var = (double*)malloc(sizeof(double) * (size_t)E);
  int* el = (int*)malloc(sizeof(int) * (size_t)k);
  for (int64_t e = 0; e < E; ++e) stdv[e] = c->initial_std;
  base_ctx b = {p, mean, stdv, 0.0, c->seed, 0, E, (double*)malloc(sizeof(double) * (size_t)(M * E)),
                (double*)malloc(sizeof(double) * (size_t)M), (int*)calloc((size_t)M, sizeof(int)),
                (char (*)[160])calloc((size_t)M, 160)};
  anytime_ctx a = {(double*)malloc(sizeof(double) * (size_t)p->robots * p->dx * (p->horizon + 1)),
                   (double*)malloc(sizeof(double) * (size_t)p->robots * p->du * (p->horizon + 1)), -1, 0, now_s()};
  int rc = 0;
  for (int it = 1; it <= c->iterations; ++it) {
    b.it = it;
    if (base_evaluate(&b, M, c->workers)) { rc = -1; break; }
    if (or_select_elites(b.rewards, M, k, el)) { rc = -1; break; }
    memset(nm, 0, sizeof(double) * (size_t)E);
    for (int j = 0; j < k; ++j)
      for (int64_t e = 0; e < E; ++e) nm[e] = nm[e] + b.samples[(int64_t)el[j] * E + e];
    for (int64_t e = 0; e < E; ++e) nm[e] = nm[e] / (double)k;
    memset(var, 0, sizeof(double) * (size_t)E);
    for (int j = 0; j < k; ++j)
      for (int64_t e = 0; e < E; ++e) {
        const double d = b.samples[(int64_t)el[j] * E + e] - nm[e];
        var[e] = var[e] + d * d;
      }
    for (int64_t e = 0; e < E; ++e) {
      var[e] = var[e] / (double)k;
      const double s = sqrt(var[e]);
      stdv[e] = s < c->min_std ? c->min_std : s;  /* cwiseSqrt().cwiseMax(min_std) */
    }
    memcpy(mean, nm, sizeof(double) * (size_t)E);
    int ok = 0;
    if (anytime_record(p, &a, mean, it, best_states, best_controls, best_reward, per_it, &ok)) { rc = -1; break; }
    if (c->stop_on_success && ok) break;
    if (c->deadline_seconds > 0 && now_s() - a.t0 >= c->deadline_seconds) break;
  }
  if (rc == 0) {
    *success = or_check_success(p, best_states, NULL, 0);
    rc = a.used;
  }
  free(mean); free(stdv); free(nm); free(var); free(el);
  free(b.samples); free(b.rewards); free(b.failed); free(b.errs);
  free(a.states); free(a.controls);
  return rc;
}
