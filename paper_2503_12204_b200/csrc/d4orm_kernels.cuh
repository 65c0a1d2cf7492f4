// d4orm_kernels.cuh — the five sm_100a kernels of the denoise-step hot path.
//
//   K1    k_philox_noise     counter-based Philox4x32-10 + Box-Muller → z[m][t][k][d]
//   K2+K3 k_rollout_fitness  fused rollout + team fitness → reward[m]   (k23.cuh)
//   K4    k_score_weights    z-scored softmax weights (fp64), entropy, best/mean
//   K5    k_wmean_partial    streaming weighted mean over [chunk of m] × E
//         k_wmean_regen      the same partials, the noise regenerated (no z rows)
//         k_wmean_tree       deterministic pairwise tree over chunk partials +
//                            the update var ← √ᾱ_{i−1} · Σ_m w_m sample_m
//
// Reference semantics: denoiser.cpp:152-180 (loop body), denoiser.cpp:50-108
// (score_weights, mc_average), schedule.cpp:29-36, denoiser.cpp:110-117.
#pragma once

#include <cooperative_groups.h>

#include "d4orm_common.cuh"
#include "k23.cuh"

namespace d4k {

constexpr int kThreads = 256;

// ------------------------------------------------------------------ K1 noise
// Standalone Philox generator (d4orm_common.cuh for the counter mapping):
// thread = (robot k, group g) of one sample row; grid.y strides samples.  The
// fp32 hot path draws the same normals inside K2+K3 instead (fused), so this
// kernel serves the fp64 path, tests and d4orm_cuda_philox_noise.
template <typename S>
__global__ void __launch_bounds__(kThreads) k_philox_noise(S* __restrict__ z, int64_t count, int R, int T, int DU,
                                                           int64_t m0, const uint2* __restrict__ keys, int step) {
  const uint2 key = keys[step];
  const int G = (T * DU + 3) >> 2;  // groups per robot
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * G) return;
  const int k = idx / G, g = idx - k * G;
  for (int64_t ml = blockIdx.y; ml < count; ml += gridDim.y) {
    const float4 v = philox_normals(key, (uint64_t)(m0 + ml), (uint32_t)k, (uint32_t)g);
    const float vv[4] = {v.x, v.y, v.z, v.w};
    S* row = z + ml * (int64_t)T * R * DU;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = 4 * g + j;
      if (n < T * DU) {
        const int t = n / DU, d = n - t * DU;
        row[((int64_t)t * R + k) * DU + d] = (S)vv[j];
      }
    }
  }
}

// ------------------------------------------------------------ K4 weights
// fp32 weights drive the fp32 weighted mean (K5), which skips samples whose
// w32 is 0.  A sample's w32 is zeroed when its weight lies below an adaptive
// floor: the largest power of two 2^-b such that the weights below it provably
// add up to at most 2^-24 of the total — half an ulp of the fp32 weights' sum (≈ 1), a
// mass the fp32 weights K5 consumes cannot resolve (round 1 used 2^-30; 2^-24 keeps
// 25 % instead of 42 % of C5's samples over a run: −5 % per step, K5a −40 %)
// (was: 1e-9 — far below the fp32 sum's own
// rounding).  The proof is a count histogram over octaves: e = exp(s − s_max)
// ∈ [2^-(b+1), 2^-b) falls in bin b (bin 128: e < 2^-128), and bins ≥ b hold at
// most Σ c_b'·2^-b' of Σe.  Integer counts → deterministic, identical on every
// rank.  (At C5 this keeps ≈ 41 % of the samples, against 59 % for a fixed
// 2^-48 floor — which gave the same 2^-30 bound only at M = 2^18.)
// Where K5a reads every row anyway (small E, z in L2) the histogram is not
// built and the fixed floor 2^-48 of the largest weight applies (bound
// M·2^-48 of the total).
constexpr double kW32Floor = 3.5527136788005009e-15;  // 2^-48
constexpr int kWBins = 129;
#ifndef D4K_W32_MASS_LOG2
#define D4K_W32_MASS_LOG2 24
#endif
constexpr double kW32Mass = 1.0 / (double)(1ull << D4K_W32_MASS_LOG2);  // 2^-24
constexpr int kWScratch = 6 * 160 + 80;               // grid folds + the bin counts (as doubles)

__device__ __forceinline__ int wbin(double e) {  // e ∈ (0, 1]: octave below the max
  if (!(e >= 0x1p-128)) return 128;
  const int ex = (int)((__double_as_longlong(e) >> 52) & 0x7ff) - 1023;  // ilogb, e normal
  const int b = ex >= -1 ? 0 : -ex - 1;
  D4K_CHECK(b >= 0 && b < kWBins);
  return b;
}

// Floor from the bin counts, by one warp (all 32 lanes; the same fixed-order
// arithmetic on every CTA and rank): U(b) = Σ_{b' ≥ b} c_b'·2^-b' as a suffix
// scan (5 bins per lane, then across lanes), floor = 2^-b* for the smallest
// b* ≥ 1 with U(b*) ≤ kW32Mass·Σe (0 if none).
__device__ __forceinline__ double w32_floor_warp(const unsigned* c, double sum_e) {
  constexpr int PER = 5;  // 32·5 ≥ kWBins
  const int lane = threadIdx.x & 31;
  const double bound = kW32Mass * sum_e;
  double m[PER], loc = 0.0;
#pragma unroll
  for (int j = PER - 1; j >= 0; --j) {
    const int b = lane * PER + j;
    if (b < kWBins) loc += (double)c[b] * __longlong_as_double((long long)(1023 - b) << 52);  // c·2^-b
    m[j] = loc;
  }
  double x = loc;  // Σ over lanes ≥ lane
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_down_sync(0xffffffffu, x, o);
    if (lane + o < 32) x += y;
  }
  double above = __shfl_down_sync(0xffffffffu, x, 1);
  if (lane == 31) above = 0.0;
  int best = 1 << 30;
#pragma unroll
  for (int j = PER - 1; j >= 0; --j) {
    const int b = lane * PER + j;
    if (b >= 1 && b < kWBins && m[j] + above <= bound) best = b;
  }
  best = __reduce_min_sync(0xffffffffu, best);
  return best < kWBins ? __longlong_as_double((long long)(1023 - best) << 52) : 0.0;
}

// One count into bin b, aggregated over the warp's lanes that share the bin.
__device__ __forceinline__ void hist_add(unsigned* h, int b) {
  const unsigned peers = __match_any_sync(__activemask(), b);
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[b], (unsigned)__popc(peers));
}

struct WeightParams {
  const double* reward;  // [M] all samples (global)
  int64_t M;
  double lambda;
  double* w64;           // [M]
  float* w32;            // [M]
  double* trace;         // [4]: step, best, mean, entropy
  int step;
  unsigned long long* err;  // set on non-finite reward
  int adaptive;             // 1: the adaptive w32 floor (K5 skips zero weights); 0: the fixed 2^-48 one
};

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((tid & 31) == 0) sh[tid >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (tid == 0) {
    for (int w = 0; w < NT / 32; ++w) r += sh[w];
    sh[NT / 32] = r;
  }
  __syncthreads();
  r = sh[NT / 32];
  __syncthreads();
  return r;
}

template <int NT>
__device__ __forceinline__ double block_max(double v, double* sh) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((tid & 31) == 0) sh[tid >> 5] = v;
  __syncthreads();
  if (tid == 0) {
    double r = sh[0];
    for (int w = 1; w < NT / 32; ++w) r = fmax(r, sh[w]);
    sh[NT / 32] = r;
  }
  __syncthreads();
  const double r = sh[NT / 32];
  __syncthreads();
  return r;
}

// score_weights (denoiser.cpp:50-90) + trace (denoiser.cpp:172-179) as one
// cooperative grid of G CTAs (grid.sync between the four reduction phases).
// Every thread keeps its ≤ PER rewards in registers (one load pass, all in
// flight), CTA partials go to `scratch` and every CTA folds the G partials in
// the same fixed order — bitwise reproducible and identical on every rank.
constexpr int kWThreads = 1024;  // PER (rewards per thread) is 2 or 16, see the launch

// N reductions with one grid barrier: v[i] is summed, or max-ed where MAXMASK
// has bit i.  Fixed fold order (warp tree, CTA tree, CTAs in index order).
// CL = false: the CTA partials go through `scratch` (global) and a cooperative
// grid barrier.  CL = true (the whole grid is one thread-block cluster, ≤ 8
// CTAs): through each CTA's shared `cl` slots and a cluster barrier, read over
// distributed shared memory in the same CTA order — the same numbers.
template <int N, int MAXMASK, bool CL = false>
__device__ __forceinline__ void grid_fold_n(double* v, double* sh, double* scratch, int slot, double* cl = nullptr) {
  namespace cg = cooperative_groups;
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const bool mx = (MAXMASK >> i) & 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, v[i], o);
      v[i] = mx ? fmax(v[i], u) : v[i] + u;
    }
    if ((tid & 31) == 0) sh[i * 32 + (tid >> 5)] = v[i];
  }
  __syncthreads();
  if (tid < 32) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const bool mx = (MAXMASK >> i) & 1;
      double r = sh[i * 32 + tid];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, r, o);
        r = mx ? fmax(r, u) : r + u;
      }
      if (tid == 0) {
        if constexpr (CL) cl[slot + i] = r;
        else scratch[(slot + i) * gridDim.x + blockIdx.x] = r;
      }
    }
  }
  if constexpr (CL) {
    cg::this_cluster().sync();  // (distinct slots per fold: no later overwrite)
    cg::cluster_group cluster = cg::this_cluster();
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const bool mx = (MAXMASK >> i) & 1;
      double r = cluster.map_shared_rank(cl, 0u)[slot + i];
      for (unsigned b = 1; b < gridDim.x; ++b) {
        const double u = cluster.map_shared_rank(cl, b)[slot + i];
        r = mx ? fmax(r, u) : r + u;
      }
      v[i] = r;
    }
  } else {
    if (gridDim.x > 1) cg::this_grid().sync();  // cooperative launch only when G > 1
    else __syncthreads();
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const bool mx = (MAXMASK >> i) & 1;
      double r = scratch[(slot + i) * gridDim.x];
      for (unsigned b = 1; b < gridDim.x; ++b) {
        const double u = scratch[(slot + i) * gridDim.x + b];
        r = mx ? fmax(r, u) : r + u;
      }
      v[i] = r;
    }
  }
  __syncthreads();
}

template <int NT, int kWPer, bool CL>
__device__ __forceinline__ void score_weights_grid_body(const WeightParams& p, double* scratch) {
  static_assert(NT == kWThreads, "k_score_weights_grid block size");
  __shared__ double sh[3 * 32];
  __shared__ unsigned s_hist[kWBins];
  __shared__ double s_floor;
  __shared__ double cl[6];  // CL: this CTA's fold partials (slots 0..5)
  unsigned* g_hist = CL ? nullptr : reinterpret_cast<unsigned*>(scratch + 6 * 160);
  if (threadIdx.x < kWBins) {
    s_hist[threadIdx.x] = 0u;
    if (!CL && blockIdx.x == 0) g_hist[threadIdx.x] = 0u;  // added to only after two grid barriers
  }
  const int64_t stride = (int64_t)gridDim.x * kWThreads;
  const int64_t g0 = (int64_t)blockIdx.x * kWThreads + threadIdx.x;
  double r[kWPer];
  double s = 0.0, best = -INFINITY;
  bool finite = true;
#pragma unroll
  for (int q = 0; q < kWPer; ++q) {
    const int64_t j = g0 + q * stride;
    r[q] = j < p.M ? p.reward[j] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < kWPer; ++q) {
    if (g0 + q * stride < p.M) {
      finite = finite && isfinite(r[q]);
      s += r[q];
      best = fmax(best, r[q]);
    }
  }
  // three grid barriers in all: {non-finite count, Σr, max r}, {Σ(r−mean)²}, {Σe, Σe·s}
  double f3[3] = {finite ? 0.0 : 1.0, s, best};
  grid_fold_n<3, 4, CL>(f3, sh, scratch, 0, cl);
  const double nf = f3[0];
  if (nf != 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicMin(p.err, 0xFFFFFFFFFFFFFFFEull);
    return;  // (CL: the caller's final cluster barrier keeps the slots alive)
  }
  const double mean = f3[1] / (double)p.M;
  best = f3[2];
  double v = 0.0;
#pragma unroll
  for (int q = 0; q < kWPer; ++q) {
    if (g0 + q * stride < p.M) {
      const double d = r[q] - mean;
      v += d * d;
    }
  }
  double f1[1] = {v};
  grid_fold_n<1, 0, CL>(f1, sh, scratch, 3, cl);
  const double std_dev = sqrt(f1[0] / (double)p.M);
  const bool head = blockIdx.x == 0 && threadIdx.x == 0;
  if (std_dev < 1e-8) {  // degenerate batch → uniform (denoiser.cpp:74-77)
    const double u = 1.0 / (double)p.M;
#pragma unroll
    for (int q = 0; q < kWPer; ++q) {
      const int64_t j = g0 + q * stride;
      if (j < p.M) {
        p.w64[j] = u;
        p.w32[j] = (float)u;
      }
    }
    if (head) {
      p.trace[0] = p.step;
      p.trace[1] = best;
      p.trace[2] = mean;
      p.trace[3] = -(double)p.M * u * log(u);
    }
    return;
  }
  // (r−mean)/std/λ as one multiply; max of the scaled values = scaled max
  // (denoiser.cpp:78-82); log w = (s − s_max) − log Σ for the entropy.
  const double inv = 1.0 / (std_dev * p.lambda);
  const double max_scaled = (best - mean) * inv;
  double e[kWPer];
  double sum = 0.0, es = 0.0;
#pragma unroll
  for (int q = 0; q < kWPer; ++q) {
    e[q] = 0.0;
    if (g0 + q * stride < p.M) {
      r[q] = (r[q] - mean) * inv - max_scaled;  // now the shifted exponent
      e[q] = exp(r[q]);
      sum += e[q];
      es += e[q] * r[q];
      if (p.adaptive) hist_add(s_hist, wbin(e[q]));
    }
  }
  __syncthreads();
  if (!CL && p.adaptive && threadIdx.x < kWBins && s_hist[threadIdx.x])
    atomicAdd(&g_hist[threadIdx.x], s_hist[threadIdx.x]);
  double f2[2] = {sum, es};
  grid_fold_n<2, 0, CL>(f2, sh, scratch, 4, cl);  // (its barrier also completes g_hist / every s_hist)
  sum = f2[0];
  double floor32 = kW32Floor;
  if (p.adaptive) {
    if constexpr (CL) {  // the cluster's integer counts summed over DSMEM (order-free)
      __shared__ unsigned s_tot[kWBins];
      if (threadIdx.x < kWBins) {
        namespace cg = cooperative_groups;
        cg::cluster_group cluster = cg::this_cluster();
        unsigned t = 0;
        for (unsigned b = 0; b < gridDim.x; ++b) t += cluster.map_shared_rank(s_hist, b)[threadIdx.x];
        s_tot[threadIdx.x] = t;
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        const double fl = w32_floor_warp(s_tot, sum);
        if (threadIdx.x == 0) s_floor = fl;
      }
      __syncthreads();
      floor32 = s_floor;
    } else {
      if (threadIdx.x < kWBins) s_hist[threadIdx.x] = __ldcg(&g_hist[threadIdx.x]);
      __syncthreads();
      if (threadIdx.x < 32) {
        const double f = w32_floor_warp(s_hist, sum);
        if (threadIdx.x == 0) s_floor = f;
      }
      __syncthreads();
      floor32 = s_floor;
    }
  }
  const double rsum = 1.0 / sum, lsum = log(sum);
  // entropy −Σ w·log w with log w = s − log Σe: log Σe − Σe·s / Σe (terms with
  // e = 0 contribute 0, as the w > 0 guard of denoiser.cpp:24-30)
  const double h = lsum - f2[1] / sum;
#pragma unroll
  for (int q = 0; q < kWPer; ++q) {
    const int64_t j = g0 + q * stride;
    if (j < p.M) {
      const double w = e[q] * rsum;
      p.w64[j] = w;
      p.w32[j] = e[q] >= floor32 ? (float)w : 0.f;  // adaptive floor (kW32Mass)
    }
  }
  if (head) {
    p.trace[0] = p.step;
    p.trace[1] = best;
    p.trace[2] = mean;
    p.trace[3] = h;
  }
}

template <int NT, int kWPer>
__global__ void __launch_bounds__(NT) k_score_weights_grid(const WeightParams p, double* scratch) {
  pdl_wait();
  score_weights_grid_body<NT, kWPer, false>(p, scratch);
}

// The same as one thread-block cluster of G ≤ 8 CTAs (M ≤ 8·2048: C3, C4):
// cluster barriers and DSMEM instead of a cooperative grid's global scratch
// and grid barriers — the same fold order, so the same weights.
template <int NT, int kWPer>
__global__ void __launch_bounds__(NT) k_score_weights_cluster(const WeightParams p) {
  pdl_wait();
  score_weights_grid_body<NT, kWPer, true>(p, nullptr);
  cooperative_groups::this_cluster().sync();  // every CTA's shared slots stay alive until all have read them
}

// Small batches (M ≤ 8192, C1 and C2): the same computation in ONE CTA of
// 1024 threads, PER ≤ 8 rewards per thread in registers, folds through shared
// memory — no cooperative launch, no grid barriers, no global scratch round
// trips (C1 step 29.1 → 26.9 µs).  Fixed fold order (warp tree, then warp 0 over
// the 32 warp partials): deterministic, identical on every rank.
template <int N, int MAXMASK, int NT = kWThreads>
__device__ __forceinline__ void cta_fold_n(double* v, double* sh) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const bool mx = (MAXMASK >> i) & 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, v[i], o);
      v[i] = mx ? fmax(v[i], u) : v[i] + u;
    }
    if (lane == 0) sh[i * 32 + wid] = v[i];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const bool mx = (MAXMASK >> i) & 1;
      double r = lane < NT / 32 ? sh[i * 32 + lane] : (mx ? -INFINITY : 0.0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, r, o);
        r = mx ? fmax(r, u) : r + u;
      }
      if (lane == 0) sh[96 + i] = r;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = sh[96 + i];
  __syncthreads();
}

// The body, shared with the fused small-batch step tail (k_small_step_tail):
// `writer` CTAs write w64 / w32 / trace / the error word; s_w32 (optional,
// shared memory) receives the fp32 weights.  Returns false on a non-finite
// reward.  sh: 3·32 + 4 doubles, s_hist: kWBins.
template <int NT, int PER>
__device__ __forceinline__ bool score_weights_cta_body(const WeightParams& p, bool writer, float* s_w32, double* sh,
                                                       unsigned* s_hist, double* s_floor_p) {
  double& s_floor = *s_floor_p;
  const int tid = threadIdx.x;
  if (tid < kWBins) s_hist[tid] = 0u;
  double r[PER];
  double s = 0.0, best = -INFINITY;
  bool finite = true;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int64_t j = tid + (int64_t)q * NT;
    r[q] = j < p.M ? p.reward[j] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (tid + (int64_t)q * NT < p.M) {
      finite = finite && isfinite(r[q]);
      s += r[q];
      best = fmax(best, r[q]);
    }
  }
  double f3[3] = {finite ? 0.0 : 1.0, s, best};
  cta_fold_n<3, 4, NT>(f3, sh);
  if (f3[0] != 0.0) {
    if (writer && tid == 0) atomicMin(p.err, 0xFFFFFFFFFFFFFFFEull);
    return false;
  }
  const double mean = f3[1] / (double)p.M;
  best = f3[2];
  double v = 0.0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (tid + (int64_t)q * NT < p.M) {
      const double d = r[q] - mean;
      v += d * d;
    }
  }
  double f1[1] = {v};
  cta_fold_n<1, 0, NT>(f1, sh);
  const double std_dev = sqrt(f1[0] / (double)p.M);
  if (std_dev < 1e-8) {  // degenerate batch → uniform (denoiser.cpp:74-77)
    const double u = 1.0 / (double)p.M;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int64_t j = tid + (int64_t)q * NT;
      if (j < p.M) {
        if (writer) {
          p.w64[j] = u;
          p.w32[j] = (float)u;
        }
        if (s_w32) s_w32[j] = (float)u;
      }
    }
    if (writer && tid == 0) {
      p.trace[0] = p.step;
      p.trace[1] = best;
      p.trace[2] = mean;
      p.trace[3] = -(double)p.M * u * log(u);
    }
    return true;
  }
  const double inv = 1.0 / (std_dev * p.lambda);
  const double max_scaled = (best - mean) * inv;
  double sum = 0.0, es = 0.0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (tid + (int64_t)q * NT < p.M) {
      const double a = (r[q] - mean) * inv - max_scaled;  // shifted exponent
      const double e = exp(a);
      sum += e;
      es += e * a;
      r[q] = e;
      if (p.adaptive) hist_add(s_hist, wbin(e));
    }
  }
  double f2[2] = {sum, es};
  cta_fold_n<2, 0, NT>(f2, sh);  // (its barriers also complete s_hist)
  sum = f2[0];
  double floor32 = kW32Floor;
  if (p.adaptive) {
    if (tid < 32) {
      const double f = w32_floor_warp(s_hist, sum);
      if (tid == 0) s_floor = f;
    }
    __syncthreads();
    floor32 = s_floor;
  }
  const double rsum = 1.0 / sum;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int64_t j = tid + (int64_t)q * NT;
    if (j < p.M) {
      const double w = r[q] * rsum;
      const float w32 = r[q] >= floor32 ? (float)w : 0.f;  // adaptive floor (kW32Mass)
      if (writer) {
        p.w64[j] = w;
        p.w32[j] = w32;
      }
      if (s_w32) s_w32[j] = w32;
    }
  }
  if (writer && tid == 0) {
    p.trace[0] = p.step;
    p.trace[1] = best;
    p.trace[2] = mean;
    p.trace[3] = log(sum) - f2[1] / sum;
  }
  return true;
}

template <int NT, int PER>
__global__ void __launch_bounds__(NT, 1) k_score_weights_cta(const WeightParams p) {
  pdl_wait();
  __shared__ double sh[3 * 32 + 4];
  __shared__ unsigned s_hist[kWBins];
  __shared__ double s_floor;
  score_weights_cta_body<NT, PER>(p, true, nullptr, sh, s_hist, &s_floor);
}

// Single-CTA variant (kept for d4orm_cuda_score_weights on arbitrary M).
template <int NT>
__global__ void __launch_bounds__(NT) k_score_weights(const WeightParams p) {
  pdl_wait();
  __shared__ double sh[NT / 32 + 1];
  const int tid = threadIdx.x;
  const int64_t per = (p.M + NT - 1) / NT;
  const int64_t b = tid * per, e = b + per < p.M ? b + per : p.M;
  double s = 0.0, best = -INFINITY;
  bool finite = true;
  for (int64_t j = b; j < e; ++j) {
    const double r = p.reward[j];
    finite = finite && isfinite(r);
    s += r;
    best = fmax(best, r);
  }
  const int nonfinite = __syncthreads_or(!finite);
  if (nonfinite) {
    if (tid == 0) atomicMin(p.err, 0xFFFFFFFFFFFFFFFEull);
    return;
  }
  const double total = block_sum<NT>(s, sh);
  const double mean = total / (double)p.M;
  best = block_max<NT>(best, sh);
  double v = 0.0;
  for (int64_t j = b; j < e; ++j) {
    const double d = p.reward[j] - mean;
    v += d * d;
  }
  const double var = block_sum<NT>(v, sh);
  const double std_dev = sqrt(var / (double)p.M);
  if (std_dev < 1e-8) {  // degenerate batch → uniform (denoiser.cpp:74-77)
    const double u = 1.0 / (double)p.M;
    for (int64_t j = b; j < e; ++j) {
      p.w64[j] = u;
      p.w32[j] = (float)u;
    }
    if (tid == 0) {
      p.trace[0] = p.step;
      p.trace[1] = best;
      p.trace[2] = mean;
      p.trace[3] = -(double)p.M * u * log(u);
    }
    return;
  }
  // max of the scaled values = the scaled max (monotone), denoiser.cpp:78-82.
  // (r−mean)/std/λ as one multiply by 1/(std·λ); normalisation by 1/Σ; the
  // entropy uses log w = (s − s_max) − log Σ, so no per-sample log (all equal
  // to the reference's expressions up to fp64 rounding).
  const double inv = 1.0 / (std_dev * p.lambda);
  const double max_scaled = (best - mean) * inv;
  double sum = 0.0;
  for (int64_t j = b; j < e; ++j) {
    const double w = exp((p.reward[j] - mean) * inv - max_scaled);
    p.w64[j] = w;
    sum += w;
  }
  sum = block_sum<NT>(sum, sh);
  const double rsum = 1.0 / sum, lsum = log(sum);
  double h = 0.0;
  for (int64_t j = b; j < e; ++j) {
    const double w = p.w64[j] * rsum;
    p.w64[j] = w;
    p.w32[j] = (float)w;
    if (w > 0.0) h -= w * (((p.reward[j] - mean) * inv - max_scaled) - lsum);
  }
  h = block_sum<NT>(h, sh);
  if (tid == 0) {
    p.trace[0] = p.step;
    p.trace[1] = best;
    p.trace[2] = mean;
    p.trace[3] = h;
  }
}

// ---------------------------------------------------- K5 weighted mean
// Partial of Σ_m w_m·sample_m over one chunk of kPartSub·kPartLanes samples,
// sample_m = msv + sd·z_m (denoiser.cpp:44-45, mc_average :104-106).
// CTA = kPartGroups element groups (4 consecutive elements each) × kPartSub
// sub-ranges: a thread accumulates its kPartLanes samples (ascending m, all
// loads in flight at once — this kernel is HBM-latency/bandwidth bound and
// streams z exactly once), then the kPartSub sub-partials are combined by a
// fixed pairwise tree in shared memory.  The order is fixed by the chunk, so
// the result is deterministic and independent of how samples are sharded.
// Two fixed CTA shapes, chosen per problem by E (so the order is still fixed
// for a given problem and sharding): small E splits the chunk across 16
// sub-ranges to expose parallelism; large E already has enough CTAs along E and
// keeps one sequential 256-sample walk per thread (best streaming efficiency).
constexpr int kChunkSamples = 256;
constexpr int kPartBatch = 8;  // loads in flight per thread (16 with 2 resident CTAs: C2/C3 K5a 26.5 µs; 8 with 4: 22.5 µs)
template <int SUB>
struct PartShape {
  static constexpr int GROUPS = SUB == 1 ? 256 : 16;
  static constexpr int LANES = kChunkSamples / SUB;
  static constexpr int THREADS = GROUPS * SUB;
};

template <typename S>
struct PartArgs {
  const S* z;        // [M][E] noise of this rank's samples
  const S* msv;      // [E] mean-scaled variable (sample = msv + sd·z)
  S sd;              // scalar std, or
  const S* sdv;      // [E] per-element std (CEM), else null
  const S* nm;       // DEV: [E] the new mean (CEM variance pass)
  int64_t M, elems;
  S* partial;        // [chunks][E]
  int reverse = 0;   // walk the chunks last-first (the z rows K2+K3 wrote last are the ones still in L2)
};

// DEV = 0: Σ_m w_m·sample_m (mc_average, denoiser.cpp:92-108; CEM's elite sum
// with w ∈ {0, 1}).  DEV = 1: Σ_m w_m·(sample_m − nm)² (CEM's variance,
// baselines.cpp:162-167; zero-weight samples are skipped as the reference only
// visits the elites).
template <typename S, typename W, int SUB, int DEV>
__global__ void __launch_bounds__(PartShape<SUB>::THREADS, (SUB > 1 && sizeof(S) == 4) ? 4 : 1) k_wmean_partial(const PartArgs<S> a,
                                                                           const W* __restrict__ w) {
  pdl_wait();
  constexpr int kPartGroups = PartShape<SUB>::GROUPS, kPartSub = SUB, kPartLanes = PartShape<SUB>::LANES;
  __shared__ S red[kPartSub][kPartGroups][4];
  const S* __restrict__ z = a.z;
  const int64_t M = a.M, elems = a.elems;
  const int g = threadIdx.x % kPartGroups, sr = threadIdx.x / kPartGroups;
  const int64_t e0 = ((int64_t)blockIdx.x * kPartGroups + g) * 4;
  const int64_t c = a.reverse ? (int64_t)gridDim.y - 1 - blockIdx.y : (int64_t)blockIdx.y;
  const int64_t mb = c * (kPartSub * kPartLanes) + (int64_t)sr * kPartLanes;
  const int n = e0 < elems ? (elems - e0 < 4 ? (int)(elems - e0) : 4) : 0;
  // large E (fp32): the CTA first compacts its chunk's non-zero weights (in
  // ascending sample order, so the sum is the same) into shared memory; the
  // walk then issues only the z loads that count, back to back
  __shared__ int s_idx[SUB == 1 ? kPartLanes : 1];
  __shared__ float s_w[SUB == 1 ? kPartLanes : 1];
  __shared__ int s_cnt[SUB == 1 ? kPartLanes / 32 + 1 : 1];
  if constexpr (SUB == 1 && std::is_same<S, float>::value) {
    static_assert(PartShape<SUB>::THREADS == kPartLanes, "one weight per thread");
    const int64_t m = mb + threadIdx.x;
    const float wm = m < M ? (float)w[m] : 0.f;
    const bool nz = wm != 0.f;
    const unsigned bal = __ballot_sync(0xffffffffu, nz);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) s_cnt[wid] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < kPartLanes / 32; ++i) {
      off += i < wid ? s_cnt[i] : 0;
      tot += s_cnt[i];
    }
    if (nz) {
      const int pos = off + __popc(bal & ((1u << lane) - 1u));
      D4K_CHECK(pos >= 0 && pos < kPartLanes);
      s_idx[pos] = threadIdx.x;
      s_w[pos] = wm;
    }
    if (threadIdx.x == 0) s_cnt[kPartLanes / 32] = tot;
    __syncthreads();
  }
  S acc[4] = {S(0), S(0), S(0), S(0)};
  if (n > 0) {
    // (constant-index loops with predication keep these in registers)
    S mv[4] = {S(0), S(0), S(0), S(0)}, sv[4], nv[4] = {S(0), S(0), S(0), S(0)};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sv[j] = a.sd;
      if (j < n) {
        mv[j] = a.msv[e0 + j];
        if (a.sdv) sv[j] = a.sdv[e0 + j];
        if (DEV) nv[j] = a.nm[e0 + j];
      }
    }
    auto term = [&](S wm, S zv, int j) -> S {  // fp32: fused; the weight multiplies the (squared) sample
      const S smp = fmaf(sv[j], zv, mv[j]);
      if constexpr (DEV) {
        const S d = smp - nv[j];
        return wm * (d * d);
      } else {
        return wm * smp;
      }
    };
    bool vec = false;
    if constexpr (std::is_same<S, float>::value) vec = n == 4 && (elems & 3) == 0;
    if (vec) {
      if constexpr (std::is_same<S, float>::value && SUB == 1) {
        // large E: one streaming walk per thread over the compacted rows
        const float4* zp = reinterpret_cast<const float4*>(z + mb * elems + e0);
        const int64_t stride = elems / 4;
        const int nnz = s_cnt[kPartLanes / 32];
#pragma unroll 4
        for (int q = 0; q < nnz; ++q) {
          const float wm = s_w[q];
          const float4 v = __ldcs(zp + (int64_t)s_idx[q] * stride);
          if constexpr (DEV) {
            acc[0] += term(wm, v.x, 0);
            acc[1] += term(wm, v.y, 1);
            acc[2] += term(wm, v.z, 2);
            acc[3] += term(wm, v.w, 3);
          } else {
            acc[0] = fmaf(wm, fmaf(sv[0], v.x, mv[0]), acc[0]);
            acc[1] = fmaf(wm, fmaf(sv[1], v.y, mv[1]), acc[1]);
            acc[2] = fmaf(wm, fmaf(sv[2], v.z, mv[2]), acc[2]);
            acc[3] = fmaf(wm, fmaf(sv[3], v.w, mv[3]), acc[3]);
          }
        }
      } else if constexpr (std::is_same<S, float>::value) {
        for (int q0 = 0; q0 < kPartLanes; q0 += kPartBatch) {
          float4 v[kPartBatch];
          float wv[kPartBatch];
#pragma unroll
          for (int q = 0; q < kPartBatch; ++q) {
            const int64_t m = mb + q0 + q;
            // (small E: L2-resident, so loads are issued unconditionally — a
            // weight-dependent load would serialise two round trips)
            if (m < M) {
              v[q] = __ldcs(reinterpret_cast<const float4*>(z + m * elems + e0));
              wv[q] = (float)__ldg(w + m);
            } else {
              v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
              wv[q] = 0.f;
            }
          }
#pragma unroll
          for (int q = 0; q < kPartBatch; ++q) {
            if constexpr (DEV) {
              acc[0] += term(wv[q], v[q].x, 0);
              acc[1] += term(wv[q], v[q].y, 1);
              acc[2] += term(wv[q], v[q].z, 2);
              acc[3] += term(wv[q], v[q].w, 3);
            } else {
              acc[0] = fmaf(wv[q], fmaf(sv[0], v[q].x, mv[0]), acc[0]);
              acc[1] = fmaf(wv[q], fmaf(sv[1], v[q].y, mv[1]), acc[1]);
              acc[2] = fmaf(wv[q], fmaf(sv[2], v[q].z, mv[2]), acc[2]);
              acc[3] = fmaf(wv[q], fmaf(sv[3], v[q].w, mv[3]), acc[3]);
            }
          }
        }
      }
    } else {
      // reference arithmetic (fp64 parity path; also ragged fp32 tails)
      for (int q = 0; q < kPartLanes; ++q) {
        const int64_t m = mb + q;
        if (m >= M) break;
        const S wm = (S)w[m];
        if (DEV && wm == S(0)) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j >= n) break;
          const S smp = xadd(mv[j], xmul(sv[j], z[m * elems + e0 + j]));
          if constexpr (DEV) {
            const S d = xsub(smp, nv[j]);
            acc[j] = xadd(acc[j], xmul(wm, xmul(d, d)));
          } else {
            acc[j] = xadd(acc[j], xmul(wm, smp));
          }
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) red[sr][g][j] = acc[j];
  __syncthreads();
  // pairwise over the sub-ranges: strides 1, 2, ... (fixed order)
#pragma unroll
  for (int s = 1; s < kPartSub; s <<= 1) {
    if ((sr & (2 * s - 1)) == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) red[sr][g][j] = xadd(red[sr][g][j], red[sr + s][g][j]);
    }
    __syncthreads();
  }
  if (sr == 0 && n > 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < n) a.partial[c * elems + e0 + j] = red[0][g][j];
  }
}

// K5a, regenerating variant (fp32, Philox noise).  A sample's noise is a pure
// function of (key, m, k, n) (the counter mapping above), so instead of reading
// back the z rows K2+K3 would have stored, the weighted mean draws the normals
// again for the samples that keep a weight: K2+K3 skips its z stores
// (FitParams::z_keep == 2) and no z buffer is round-tripped through HBM.
// Thread = one Philox group (robot k, normals n = 4g..4g+3 of its stream, i.e.
// the elements ((n/du)·R + k)·du + n%du) × one sub-range of the 256-sample
// chunk.  The chunk's non-zero weights are compacted in ascending m first; every
// per-element sum is the same ascending-m fmaf chain, and the sub-range split /
// pairwise tree are k_wmean_partial's (SUB = 1 for large E, 16 for small E), so
// the partials equal the stored-z path's bit for bit (a zero weight adds an
// exact 0 there).
struct RegenArgs {
  const float* msv;  // [E] mean-scaled variable (sample = msv + sd·z)
  float sd;
  int64_t M, m_global0, elems;
  int R, T, du;
  const uint2* keys;
  int step;
  float* partial;  // [chunks][E]
};

#ifdef D4K_REGEN_MINB  // experiment knob: resident CTAs per SM the kernel is register-capped for
#define D4K_REGEN_LB __launch_bounds__(256, D4K_REGEN_MINB)
#else
#define D4K_REGEN_LB __launch_bounds__(256)
#endif
template <int SUB>
__global__ void D4K_REGEN_LB k_wmean_regen(const RegenArgs a, const float* __restrict__ w) {
  pdl_wait();
  constexpr int GROUPS = 256 / SUB, LANES = 256 / SUB;
  __shared__ float red[SUB][GROUPS][4];
  __shared__ int2 s_iw[256];  // compacted (sample offset in the chunk, fp32 weight bits)
  __shared__ int s_pos[257];
  __shared__ int s_cnt[8];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t c = blockIdx.y, mc = c * 256;
  // compaction: s_pos[i] = non-zero weights before sample i of the chunk
  {
    const int64_t m = mc + tid;
    const float wm = m < a.M ? w[m] : 0.f;
    const bool nz = wm != 0.f;
    const unsigned bal = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) s_cnt[wid] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      off += i < wid ? s_cnt[i] : 0;
      tot += s_cnt[i];
    }
    const int pos = off + __popc(bal & ((1u << lane) - 1u));
    D4K_CHECK(pos >= 0 && pos < 256 && tot <= 256);
    s_pos[tid] = pos;
    if (nz) s_iw[pos] = make_int2(tid, __float_as_int(wm));
    if (tid == 0) s_pos[256] = tot;
    __syncthreads();
  }
  const int g = tid % GROUPS, sr = tid / GROUPS;
  const int G = (a.T * a.du + 3) >> 2;  // Philox groups per robot
  const int gi = blockIdx.x * GROUPS + g;
  const int k = gi / G, gg = gi - k * G;
  const int nmax = a.T * a.du;
  int64_t e[4];
  float mv[4] = {0.f, 0.f, 0.f, 0.f};
  bool ok[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int n = 4 * gg + j;
    ok[j] = k < a.R && n < nmax;
    const int t = n / a.du, d = n - t * a.du;
    e[j] = ((int64_t)t * a.R + k) * a.du + d;
    if (ok[j]) mv[j] = a.msv[e[j]];
  }
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  // the round keys in (vector) registers, derived once: a warp-uniform key
  // would be re-derived in uniform registers on every draw
  uint2 key = a.keys[a.step];
  key.x = __shfl_sync(0xffffffffu, key.x, 0);
  key.y = __shfl_sync(0xffffffffu, key.y, 0);
  if (k < a.R) {
    const PhiloxKeys ks(key);
    const float sd = a.sd;
    const int q0 = s_pos[sr * LANES], q1 = s_pos[(sr + 1) * LANES];
    // chunks start at multiples of 256 samples (a rank's first sample too), so
    // m = mg + offset never carries into the counter's high word
    const uint64_t mg = (uint64_t)(a.m_global0 + mc);
    D4K_CHECK((mg & 255u) == 0 && q0 >= 0 && q1 <= 256);
    const uint32_t m_hi = (uint32_t)(mg >> 32), m_lo = (uint32_t)mg;
#pragma unroll 4
    for (int q = q0; q < q1; ++q) {
      const int2 iw = s_iw[q];  // one LDS.64: offset + weight
      const float wm = __int_as_float(iw.y);
      const float4 v = philox_normals(ks, m_hi, m_lo + (uint32_t)iw.x, (uint32_t)k, (uint32_t)gg);
      acc[0] = fmaf(wm, fmaf(sd, v.x, mv[0]), acc[0]);
      acc[1] = fmaf(wm, fmaf(sd, v.y, mv[1]), acc[1]);
      acc[2] = fmaf(wm, fmaf(sd, v.z, mv[2]), acc[2]);
      acc[3] = fmaf(wm, fmaf(sd, v.w, mv[3]), acc[3]);
    }
  }
  if constexpr (SUB > 1) {
#pragma unroll
    for (int j = 0; j < 4; ++j) red[sr][g][j] = acc[j];
    __syncthreads();
#pragma unroll
    for (int s = 1; s < SUB; s <<= 1) {  // k_wmean_partial's pairwise order
      if ((sr & (2 * s - 1)) == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) red[sr][g][j] = red[sr][g][j] + red[sr + s][g][j];
      }
      __syncthreads();
    }
    if (sr == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = red[0][g][j];
    }
  }
  if (sr == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (ok[j]) a.partial[c * a.elems + e[j]] = acc[j];
  }
}

// What the tree does with the total of each element.
enum { FIN_UPDATE = 0, FIN_CEM_MEAN = 1, FIN_CEM_VAR = 2 };
template <typename S>
struct TreeFinal {
  int mode;
  // FIN_UPDATE (denoise_step, denoiser.cpp:110-117; MPPI with unit scales):
  //   var ← scale·avg, msv ← next_ms·var, bm ← base + msv
  double scale, next_ms;
  double* var;
  S* msv;
  const S* base;
  S* bm;
  // CEM (baselines.cpp:157-170): FIN_CEM_MEAN  nm ← total / k;
  //   FIN_CEM_VAR  std ← max(√(total / k), min_std), mean ← nm
  double kdiv, min_std;
  double* nm64;
  S* nm_s;
  const S* nm_in;
  double* std64;
  S* sdv;
};

// What K5b does with element e's total (see TreeFinal).
template <typename S>
__device__ __forceinline__ void tree_finalize(const TreeFinal<S>& f, int64_t e, S total) {
  if (f.mode == FIN_UPDATE) {
    const double nv = f.scale * (double)total;
    f.var[e] = nv;
    const S m = (S)(f.next_ms * nv);
    f.msv[e] = m;
    if (f.bm) f.bm[e] = f.base[e] + m;
  } else if (f.mode == FIN_CEM_MEAN) {
    const double nm = (double)total / f.kdiv;  // new_mean /= elite_count
    f.nm64[e] = nm;
    f.nm_s[e] = (S)nm;
  } else {
    const double sd = sqrt((double)total / f.kdiv);  // variance /= k; cwiseSqrt
    const double s = sd < f.min_std ? f.min_std : sd;  // cwiseMax(min_std)
    f.std64[e] = s;
    f.sdv[e] = (S)s;
    f.var[e] = f.nm64[e];  // mean.u = new_mean
    f.msv[e] = f.nm_s[e];
    if (f.bm) f.bm[e] = f.base[e] + f.nm_s[e];
  }
}

// Pairwise (binary-counter) sum of the chunk partials — a balanced binary tree
// when the chunk count is a power of two, so a rank owning an aligned block of
// chunks computes exactly one subtree and results are identical for any GPU
// count.  Then the finalisation `f` (see TreeFinal).
template <typename S>
__global__ void __launch_bounds__(kThreads) k_wmean_tree(const S* __restrict__ partial, int64_t nchunks,
                                                         int64_t elems, const TreeFinal<S> f,
                                                         S* __restrict__ root_out) {
  pdl_wait();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= elems) return;
  S stack[40];
  int top = 0;
  // whole blocks of 8 chunks: their perfect 8-leaf subtree in registers, then
  // the binary counter over blocks (the same tree as leaf by leaf: every block
  // starts at a multiple of 8, where the leaf counter's low 3 bits are 0)
  const int64_t nblk = nchunks / 8;
  for (int64_t b = 0; b < nblk; ++b) {
    S v8[8];  // eight loads in flight
#pragma unroll
    for (int j = 0; j < 8; ++j) v8[j] = partial[(8 * b + j) * elems + e];
    S v = xadd(xadd(xadd(v8[0], v8[1]), xadd(v8[2], v8[3])), xadd(xadd(v8[4], v8[5]), xadd(v8[6], v8[7])));
    for (int64_t k = b; k & 1; k >>= 1) v = xadd(stack[--top], v);  // merge equal-size subtrees
    D4K_CHECK(top >= 0 && top < 40);
    stack[top++] = v;
  }
  for (int64_t cnt = 8 * nblk; cnt < nchunks; ++cnt) {  // leaves past the last whole block
    S v = partial[cnt * elems + e];
    for (int64_t k = cnt; k & 1; k >>= 1) v = xadd(stack[--top], v);
    D4K_CHECK(top >= 0 && top < 40);
    stack[top++] = v;
  }
  S total = stack[--top];
  while (top > 0) total = xadd(stack[--top], total);
  if (root_out) {
    root_out[e] = total;
    return;
  }
  tree_finalize(f, e, total);
}

// K5b with the 8-leaf block roots in parallel: P threads per element compute
// the roots of blocks j, j + P, … (each exactly k_wmean_tree's 8-leaf subtree)
// into shared memory, then one thread per element runs k_wmean_tree's binary
// counter over the roots in block order, the leaves past the last whole block,
// and the finalisation — the same additions in the same order, so bitwise
// k_wmean_tree; P× the loads in flight (C4: 12 CTAs of 64-deep serial walks →
// 96 CTAs).  Dynamic shared memory: (256 / P) · nblk values.
template <typename S>
__global__ void __launch_bounds__(kThreads) k_wmean_tree_par(const S* __restrict__ partial, int64_t nchunks,
                                                             int64_t elems, const TreeFinal<S> f, S* __restrict__ root_out,
                                                             int P) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char tree_smem[];
  S* roots = reinterpret_cast<S*>(tree_smem);
  const int EB = kThreads / P;
  // element index fastest: a warp reads 32 consecutive elements of one partial row (one
  // 128-byte line per load; with the block index fastest a warp touched 8 rows × 16 bytes),
  // and roots are stored [block][element] so neither pass has bank conflicts
  const int el = threadIdx.x % EB, j = threadIdx.x / EB;
  const int64_t e = (int64_t)blockIdx.x * EB + el;
  const int64_t nblk = nchunks / 8;
  if (e < elems) {
    for (int64_t b = j; b < nblk; b += P) {
      S v8[8];  // eight loads in flight
#pragma unroll
      for (int q = 0; q < 8; ++q) v8[q] = partial[(8 * b + q) * elems + e];
      roots[(size_t)b * EB + el] =
          xadd(xadd(xadd(v8[0], v8[1]), xadd(v8[2], v8[3])), xadd(xadd(v8[4], v8[5]), xadd(v8[6], v8[7])));
    }
  }
  __syncthreads();
  if (e >= elems || j != 0) return;
  S stack[40];
  int top = 0;
  for (int64_t b = 0; b < nblk; ++b) {
    S v = roots[(size_t)b * EB + el];
    for (int64_t k = b; k & 1; k >>= 1) v = xadd(stack[--top], v);  // merge equal-size subtrees
    D4K_CHECK(top >= 0 && top < 40);
    stack[top++] = v;
  }
  for (int64_t cnt = 8 * nblk; cnt < nchunks; ++cnt) {  // leaves past the last whole block
    S v = partial[cnt * elems + e];
    for (int64_t k = cnt; k & 1; k >>= 1) v = xadd(stack[--top], v);
    D4K_CHECK(top >= 0 && top < 40);
    stack[top++] = v;
  }
  S total = stack[--top];
  while (top > 0) total = xadd(stack[--top], total);
  if (root_out) {
    root_out[e] = total;
    return;
  }
  tree_finalize(f, e, total);
}

// ------------------------------------------------- fused small-batch step tail
// For latency-bound batches (M ≤ 2048 samples, fp32, stored z, one rank — C1)
// the step's K4 → K5a → K5b chain is one launch of a thread-block-cluster
// grid: CTA (x, c) owns elements [64x, 64x + 64) of chunk c, and the cluster
// spans the chunks (≤ 8).  Every CTA computes the z-scored softmax weights of
// all M rewards itself (score_weights_cta_body — the standalone K4's
// arithmetic; CTA (0, 0) writes w64 / w32 / trace), then its chunk partial
// exactly as k_wmean_partial<float, float, 16, 0> (16 sub-ranges of 16
// samples, fmaf chains, pairwise combine) into its shared memory; after a
// cluster barrier the cluster's rank-0 CTA reads the chunk partials over
// distributed shared memory and folds them exactly as k_wmean_tree (8-leaf
// blocks, binary counter), then the FIN_UPDATE.  Bitwise the three-kernel
// path's result (tests/test_gpu_tail.py); two launches fewer per step.
constexpr int kTailMaxChunks = 8;
struct TailArgs {
  WeightParams wp;
  const float* z;    // [M][E] this step's noise
  const float* msv;  // [E]
  float sd;
  int64_t E, nchunks;
  TreeFinal<float> fin;
};

template <int PER>
__global__ void __launch_bounds__(256, 1) k_small_step_tail(const TailArgs a) {
  pdl_wait();
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double sh[3 * 32 + 4];
  __shared__ unsigned s_hist[kWBins];
  __shared__ double s_floor;
  __shared__ float s_w32[256 * PER];
  __shared__ float red[16][16][4];
  __shared__ float s_part[64];
  const bool ok = score_weights_cta_body<256, PER>(a.wp, blockIdx.x == 0 && blockIdx.y == 0, s_w32, sh, s_hist,
                                                   &s_floor);
  const int64_t M = a.wp.M, E = a.E;
  const int64_t c = blockIdx.y;  // this CTA's chunk = its rank in the cluster
  D4K_CHECK(a.nchunks >= 1 && a.nchunks <= kTailMaxChunks && (int)cluster.block_index().y == (int)c);
  const int g = threadIdx.x % 16, sr = threadIdx.x / 16;
  const int64_t e0 = ((int64_t)blockIdx.x * 16 + g) * 4;
  const bool live = ok && e0 < E;  // E % 4 == 0 (host): a live group has 4 elements
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (live) {
    const float sd = a.sd;
    float mv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) mv[j] = a.msv[e0 + j];
    const int64_t mb = c * 256 + (int64_t)sr * 16;
    float4 v[16];
    float wv[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int64_t m = mb + q;
      if (m < M) {
        v[q] = __ldcs(reinterpret_cast<const float4*>(a.z + m * E + e0));
        wv[q] = s_w32[m];
      } else {
        v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        wv[q] = 0.f;
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      acc[0] = fmaf(wv[q], fmaf(sd, v[q].x, mv[0]), acc[0]);
      acc[1] = fmaf(wv[q], fmaf(sd, v[q].y, mv[1]), acc[1]);
      acc[2] = fmaf(wv[q], fmaf(sd, v[q].z, mv[2]), acc[2]);
      acc[3] = fmaf(wv[q], fmaf(sd, v[q].w, mv[3]), acc[3]);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) red[sr][g][j] = acc[j];
  __syncthreads();
#pragma unroll
  for (int s = 1; s < 16; s <<= 1) {  // k_wmean_partial's pairwise order
    if ((sr & (2 * s - 1)) == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) red[sr][g][j] = red[sr][g][j] + red[sr + s][g][j];
    }
    __syncthreads();
  }
  if (sr == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) s_part[g * 4 + j] = red[0][g][j];
  }
  cluster.sync();  // every chunk partial of this element block is in its CTA's shared memory
  const int t = threadIdx.x;
  const int64_t e = (int64_t)blockIdx.x * 64 + t;
  if (ok && c == 0 && t < 64 && e < E) {
    // k_wmean_tree's order over the chunk partials (read over DSMEM), then the update
    float stack[4];
    int top = 0;
    auto leaf = [&](int64_t ch) { return cluster.map_shared_rank(s_part, (unsigned)ch)[t]; };
    const int64_t nblk = a.nchunks / 8;
    for (int64_t b = 0; b < nblk; ++b) {
      float v8[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v8[j] = leaf(8 * b + j);
      float v = ((v8[0] + v8[1]) + (v8[2] + v8[3])) + ((v8[4] + v8[5]) + (v8[6] + v8[7]));
      for (int64_t k = b; k & 1; k >>= 1) v = stack[--top] + v;
      D4K_CHECK(top >= 0 && top < 4);
      stack[top++] = v;
    }
    for (int64_t cnt = 8 * nblk; cnt < a.nchunks; ++cnt) {
      float v = leaf(cnt);
      for (int64_t k = cnt; k & 1; k >>= 1) v = stack[--top] + v;
      D4K_CHECK(top >= 0 && top < 4);
      stack[top++] = v;
    }
    float total = stack[--top];
    while (top > 0) total = stack[--top] + total;
    const TreeFinal<float>& f = a.fin;  // FIN_UPDATE (the host selects this kernel for it only)
    const double nv = f.scale * (double)total;
    f.var[e] = nv;
    const float m = (float)(f.next_ms * nv);
    f.msv[e] = m;
    if (f.bm) f.bm[e] = f.base[e] + m;
  }
  cluster.sync();  // keep every CTA's shared partials alive until rank 0 has read them
}

template <typename S>
__global__ void k_init_var(const double* __restrict__ var, double ms, S* __restrict__ msv, const S* __restrict__ base,
                           S* __restrict__ bm, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) {
    const S m = (S)(ms * var[e]);
    msv[e] = m;
    if (bm) bm[e] = base[e] + m;
  }
}

}  // namespace d4k
