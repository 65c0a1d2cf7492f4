// k_outcome.cuh — the anytime iteration's tail on the device (K6, K7).
//
// K7 k_iter_begin  starts iteration `it` of solve (optimizer.cpp:66-80): the
//                  base is the executed controls of the current trajectory,
//                  the variable restarts at zero (Deformation), the Philox key
//                  table is re-derived for seed_it = mix_seed(seed, it)
//                  (optimizer.cpp:76) — all from device state, so one CUDA
//                  graph replays every iteration.
// K6 k_outcome     iterate_impl's tail and the bookkeeping of solve
//                  (optimizer.cpp:25-28,80-93): updated = base + Δ, fp64
//                  rollout with the reference's clamp and RK4
//                  (dynamics.cpp:65-87), total_reward (reward.cpp:67-130, the
//                  reference's t-major / k-minor summation order), objective
//                  (reward.cpp:136-156), check_success (reward.cpp:162-200),
//                  best-trajectory tracking, per-iteration record.
//
// One CTA: the trajectory is a single (T+1)·R·dx object; every per-(t, k)
// quantity is computed in parallel, the order-sensitive sums by one thread.
#pragma once

#include "d4orm_common.cuh"

namespace d4k {

__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t mix_seed_dev(uint64_t a, uint64_t b) {  // rng.hpp:17-23
  return splitmix64_dev(splitmix64_dev(a) ^ (0x9E3779B97F4A7C15ull + b));
}

// Device state of a solve: counters and the best-so-far scalars.
struct SolveState {
  int iter;          // iterations finished
  int best_iter;     // -1 before the first
  int success;       // of the latest iteration
  int pad;
  double best_reward;
  uint64_t seed;     // config.denoiser.seed
};

template <typename S>
struct IterBeginParams {
  const double* cur_ctrl;  // [T][R][du] executed controls of the current trajectory
  S* base;                 // [E]
  S* msv;                  // [E]
  S* bm;                   // [E] or null (fp64 path)
  double* var;             // [E]
  int64_t E;
  uint2* keys;             // [N+1]
  int N;
  const SolveState* st;
  unsigned long long* err;
};

template <typename S>
__global__ void k_iter_begin(const IterBeginParams<S> p) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t e = i0; e < p.E; e += stride) {
    const S b = (S)p.cur_ctrl[e];
    p.base[e] = b;
    p.var[e] = 0.0;  // Deformation: the variable starts at zero (denoiser.cpp:137-140)
    p.msv[e] = S(0);
    if (p.bm) p.bm[e] = b;
  }
  if (i0 <= p.N) {
    const uint64_t seed_it = mix_seed_dev(p.st->seed, (uint64_t)(p.st->iter + 1));
    const uint64_t v = mix_seed_dev(seed_it, (uint64_t)i0);
    p.keys[i0] = make_uint2((uint32_t)v, (uint32_t)(v >> 32));
  }
  if (i0 == 0) *p.err = ~0ull;
}

struct OutcomeParams {
  const double* ctrl_in;   // [T][R][du] base: current executed controls (solve) | zeros (MPPI / CEM)
  double* ctrl;            // [T][R][du] out: the new executed controls (may alias ctrl_in)
  const double* var;       // [E] Δ
  const double* starts;    // [R][dx]
  const double* goals;     // [R][pd]
  const double* obs_c;     // [O][pd]
  const double* obs_r;     // [O]
  double lower[3], upper[3];
  double dt;
  int R, T, O;
  double w_t, epsilon, robot_radius, goal_tol, w_o, w_e;
  double* states;          // [T+1][R][dx] scratch: the iteration's trajectory
  double* vals;            // [T][R] per-(t, k) reward terms
  double* best_states;     // [T+1][R][dx]
  double* best_ctrl;       // [T+1][R][du] (column T zero)
  double* rec;             // [max_iter][4]: reward, objective, success, -
  SolveState* st;
  int step_key;            // error key marking the final rollout (host: kOutcomeKey)
  unsigned long long* err;
};

template <int KIND>
__global__ void __launch_bounds__(256) k_outcome(const OutcomeParams p) {
  constexpr int DX = ModelDims<KIND>::DX, DU = ModelDims<KIND>::DU, PD = ModelDims<KIND>::PD;
  const int R = p.R, T = p.T, tid = threadIdx.x, nt = blockDim.x;
  __shared__ int s_fail, s_hits, s_bad;
  __shared__ double s_reward;
  __shared__ int s_better;
  if (tid == 0) {
    s_fail = 0;
    s_hits = 0;
    s_bad = 0;
  }
  __syncthreads();
  // ---- rollout of base + Δ (dynamics.cpp:65-87), one thread per robot
  for (int k = tid; k < R; k += nt) {
    double x[DX];
#pragma unroll
    for (int j = 0; j < DX; ++j) x[j] = p.starts[k * DX + j];
#pragma unroll
    for (int j = 0; j < DX; ++j) p.states[(size_t)k * DX + j] = x[j];
    bool bad = false;
    for (int t = 0; t < T; ++t) {
      double u[DU];
      const size_t e = ((size_t)t * R + k) * DU;
#pragma unroll
      for (int d = 0; d < DU; ++d) {
        double v = xadd(p.ctrl_in[e + d], p.var[e + d]);  // base_controls.u + denoised.variable.u
        v = (v < p.lower[d]) ? p.lower[d] : v;         // cwiseMax(lower)
        v = (p.upper[d] < v) ? p.upper[d] : v;         // cwiseMin(upper)
        u[d] = v;
        p.ctrl[e + d] = v;                             // the executed control
      }
      rk4<KIND, double>(x, u, p.dt, 0.5 * p.dt, p.dt / 6.0);
      bool fin = true;
#pragma unroll
      for (int j = 0; j < DX; ++j) fin = fin && isfinite(x[j]);
      if (!fin && !bad) {
        bad = true;
        atomicMin(p.err, ((unsigned long long)p.step_key << 52) | ((unsigned long long)k << 10) |
                             (unsigned long long)(t + 1));
        atomicExch(&s_bad, 1);
      }
#pragma unroll
      for (int j = 0; j < DX; ++j) p.states[((size_t)(t + 1) * R + k) * DX + j] = x[j];
    }
  }
  __syncthreads();
  if (s_bad) return;  // the host reports the rollout error
  const double m = xadd(xmul(2.0, p.robot_radius), p.epsilon);  // 2R_a + ε
  const double m2 = xmul(m, m);
  const double safety = xmul(xmul(4.0, p.robot_radius), p.robot_radius);
  const double tol2 = xmul(p.goal_tol, p.goal_tol);
  auto pos = [&](int t, int k, int j) { return p.states[((size_t)t * R + k) * DX + j]; };
  auto sq = [&](double acc, double d) { return xadd(acc, xmul(d, d)); };
  // ---- per-(t, k) reward terms, objective hits, success checks
  for (int idx = tid; idx < (T + 1) * R; idx += nt) {
    const int t = idx / R, k = idx - t * R;
    double gsq = 0.0;
#pragma unroll
    for (int j = 0; j < PD; ++j) gsq = sq(gsq, xsub(pos(t, k, j), p.goals[k * PD + j]));
    if (t >= 1) {
      // total_reward term (reward.cpp:92-125): goal progress, first conflicting
      // partner, first overlapping obstacle
      double sd = 0.0;
#pragma unroll
      for (int j = 0; j < PD; ++j) sd = sq(sd, xsub(p.starts[k * DX + j], p.goals[k * PD + j]));
      double v = xsub(1.0, sqrt(gsq) / sqrt(sd));
      for (int l = 0; l < R; ++l) {
        if (l == k) continue;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < PD; ++j) s = sq(s, xsub(pos(t, k, j), pos(t, l, j)));
        if (s <= m2) {
          v = xsub(v, p.w_t);
          break;
        }
      }
      for (int o = 0; o < p.O; ++o) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < PD; ++j) s = sq(s, xsub(pos(t, k, j), p.obs_c[o * PD + j]));
        const double lim = xadd(p.obs_r[o], p.robot_radius);
        if (s <= xmul(lim, lim)) {
          v = xsub(v, p.w_o);
          break;
        }
      }
      p.vals[(size_t)(t - 1) * R + k] = v;
      if (gsq <= tol2) atomicAdd(&s_hits, 1);  // objective (reward.cpp:136-156)
    }
    // check_success (reward.cpp:162-200): strict 2R_a separation and no obstacle
    // overlap at every t (t = 0 included), terminal goal ball
    for (int l = k + 1; l < R; ++l) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < PD; ++j) s = sq(s, xsub(pos(t, k, j), pos(t, l, j)));
      if (s <= safety) atomicExch(&s_fail, 1);
    }
    for (int o = 0; o < p.O; ++o) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < PD; ++j) s = sq(s, xsub(pos(t, k, j), p.obs_c[o * PD + j]));
      const double lim = xadd(p.obs_r[o], p.robot_radius);
      if (s <= xmul(lim, lim)) atomicExch(&s_fail, 1);
    }
    if (t == T && sqrt(gsq) > p.goal_tol) atomicExch(&s_fail, 1);
  }
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;  // reward.cpp: t-major, k-minor accumulation
    for (int e = 0; e < T * R; ++e) sum = xadd(sum, p.vals[e]);
    if (p.w_e != 0.0) {  // effort extension, as the host total_reward
      double ef = 0.0;
      for (int e = 0; e < T * R * DU; ++e) ef = xadd(ef, xmul(p.ctrl[e], p.ctrl[e]));
      sum = xsub(sum, xmul(p.w_e, ef));
    }
    const double reward = sum / ((double)R * (double)T);
    const double quality = (double)s_hits / ((double)R * (double)T);
    const int it = p.st->iter;  // 0-based index of this iteration
    p.rec[4 * it + 0] = reward;
    p.rec[4 * it + 1] = quality;
    p.rec[4 * it + 2] = s_fail ? 0.0 : 1.0;
    p.rec[4 * it + 3] = 0.0;
    const bool better = p.st->best_iter < 0 || reward > p.st->best_reward;
    if (better) {
      p.st->best_reward = reward;
      p.st->best_iter = it;
    }
    p.st->success = s_fail ? 0 : 1;
    p.st->iter = it + 1;
    s_reward = reward;
    s_better = better ? 1 : 0;
  }
  __syncthreads();
  if (s_better) {
    for (int e = tid; e < (T + 1) * R * DX; e += nt) p.best_states[e] = p.states[e];
    for (int e = tid; e < (T + 1) * R * DU; e += nt) p.best_ctrl[e] = e < T * R * DU ? p.ctrl[e] : 0.0;
  }
}

// K8: start of an MPPI / CEM iteration (baselines.cpp:116-119,152-155): the
// Philox key of iteration it = mix_seed(seed, it), so sample m's noise is the
// counter stream (·, m, k) of that key — the analogue of the reference's
// NormalStream(mix_seed(seed, it, m)).
__global__ void k_baseline_begin(uint2* keys, const SolveState* st, unsigned long long* err) {
  if (threadIdx.x == 0) {
    const uint64_t v = mix_seed_dev(st->seed, (uint64_t)(st->iter + 1));
    keys[0] = make_uint2((uint32_t)v, (uint32_t)(v >> 32));
    *err = ~0ull;
  }
}

// CEM elite selection (select_elites, baselines.cpp:86-97): `order` is the
// stable descending sort of the rewards (ties keep the lower index first), so
// the first k entries are the elites; their weight is 1, every other 0 (the
// elite sum is divided by k in the tree, as new_mean /= elite_count).
__global__ void k_elite_weights(const int* __restrict__ order, int64_t M, int64_t k, double* __restrict__ w64,
                                float* __restrict__ w32) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < M) {
    const int m = order[j];
    w64[m] = j < k ? 1.0 : 0.0;
    w32[m] = j < k ? 1.0f : 0.0f;
  }
}

// Sort input: rewards with −0 folded into +0 (the reference's `>` treats them
// as equal; radix keys would not) and the sample indices.
__global__ void k_sort_prep(const double* __restrict__ r, int64_t M, double* __restrict__ keys, int* __restrict__ idx) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < M) {
    keys[j] = r[j] + 0.0;
    idx[j] = (int)j;
  }
}

}  // namespace d4k
