// K2+K3, time-segmented variant for latency-bound launches of the velocity-input
// kinds (fp32): rollout + fitness with each robot's horizon split over
// kSegs = 8 threads.
//
// The regular kernel (k23.cuh) walks a robot's T steps in one thread, so a
// launch with few samples (C1: 1024 samples × 4 robots = 32 CTAs) is bound by
// that serial chain, not by any throughput.  For ẋ = u the state is a prefix
// sum, x_t = x_0 + Σ_{τ<t} dt·u_τ (the fp32 closed form of rk4_with for these
// kinds, dynamics.hpp:123-130), so the chain splits:
//   1. thread (sample, robot k, segment j) draws its segment's normals
//      (Philox, the same counter mapping as K1 / the fused draw: group
//      n/4 of robot k's stream, n = t·du + d) or reads them (host noise),
//      clamps u = clamp(bm + sd·z) (dynamics.cpp:72, stored as executed),
//      and forms the local prefix q_t = Σ_{segment τ ≤ t} dt·u_τ;
//   2. an exclusive scan of the segment totals across the 8 lanes gives the
//      offset x_0 + Σ_{earlier segments}; states x_{t+1} = offset + q_t go to
//      shared memory, the goal term 1 − ‖x − g‖/‖s − g‖ (reward.cpp:92-96) is
//      accumulated on the way;
//   3. after one barrier, each thread tests its robot's states in its segment
//      against every other robot (‖Δp‖² ≤ (2R_a + ε)², reward.cpp:99-108, the
//      direct form) and every obstacle (reward.cpp:110-124, the expanded form
//      of the regular kernel) — a robot-step counts once per kind;
//   4. a fixed-order reduction per sample writes the reward.
// The positions differ from the serial chain's only by fp32 association
// (x_0 + (Σ…) instead of ((x_0 + dt·u_0) + dt·u_1) …); the decisions and the
// reward are checked against the fp64 oracle and against the regular kernel
// in tests/test_gpu_seg.py.
#include "k_seg.cuh"

#include <cstdlib>

#include "d4orm_common.cuh"
#include "k23.cuh"

namespace d4k {

constexpr int kSegMaxL = 16;   // steps per segment (T ≤ 128 at 8 segments)

// kSegs threads per robot (a shuffle group): 8.  16 (knob D4ORM_SEGS=16, where
// the horizon splits into whole Philox groups) halves each thread's serial
// chain but was measured slower on C1 (0.0164 → 0.0214 ms per step: twice the
// CTAs, and the per-thread pair loop does not shrink with the segment).
template <int PD, int NOISE, int kSegs>
__global__ void __launch_bounds__(128) k_rollout_fitness_seg(const __grid_constant__ FitParams<float> p) {
  pdl_wait();
  constexpr int DU = PD;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* pos = reinterpret_cast<float*>(smem_raw);  // [spc][T+1][R][PD]
  const int R = p.R, T = p.T, L = T / kSegs;
  const int per_sample = R * kSegs, spc = blockDim.x / per_sample;
  const int tid = threadIdx.x, s = tid / per_sample, r = tid - s * per_sample;
  const int k = r / kSegs, j = r - k * kSegs;
  const int64_t m = (int64_t)blockIdx.x * spc + s;
  const bool live = s < spc && m < p.M;
  float* P = pos + (size_t)s * (T + 1) * R * PD;
  double* red = reinterpret_cast<double*>(pos + (size_t)spc * (T + 1) * R * PD);  // [8] warp goal / effort sums
  int* cnt = reinterpret_cast<int*>(red + 8);                                     // [8] warp counts

  // ---- 1. noise, controls, local prefix (states → shared as q_t for now)
  float q[PD], eff = 0.f;
#pragma unroll
  for (int d = 0; d < PD; ++d) q[d] = 0.f;
  const int t0 = j * L;
  if (live) {
    const float* bm = p.bm + ((size_t)t0 * R + k) * DU;
    const int RDU = R * DU;
    float bq[kSegMaxL * DU];  // base + msv, loaded first: the draws hide the latency
#pragma unroll
    for (int i = 0; i < kSegMaxL; ++i)
      if (i < L)
#pragma unroll
        for (int d = 0; d < DU; ++d) bq[i * DU + d] = __ldg(bm + i * RDU + d);
    float z[kSegMaxL * DU];
    if constexpr (NOISE == 1) {
      const uint2 key = p.keys[p.step];
      const uint64_t mg = (uint64_t)(p.m_global0 + m);
#pragma unroll
      for (int g = 0; g < kSegMaxL * DU / 4; ++g) {
        if (g < L * DU / 4) {
          const float4 v = philox_normals(key, mg, (uint32_t)k, (uint32_t)(t0 * DU / 4 + g));
          z[4 * g] = v.x;
          z[4 * g + 1] = v.y;
          z[4 * g + 2] = v.z;
          z[4 * g + 3] = v.w;
        }
      }
      if (p.z_keep != 2) {  // z rows for K5a (it regenerates them when z_keep == 2)
        float* zs = p.z_store + (size_t)m * T * RDU + ((size_t)t0 * R + k) * DU;
#pragma unroll
        for (int i = 0; i < kSegMaxL; ++i)
          if (i < L)
#pragma unroll
            for (int d = 0; d < DU; ++d) zs[i * RDU + d] = z[i * DU + d];
      }
    } else {
      const float* zr = p.z + (size_t)m * T * RDU + ((size_t)t0 * R + k) * DU;
#pragma unroll
      for (int i = 0; i < kSegMaxL; ++i)
        if (i < L)
#pragma unroll
          for (int d = 0; d < DU; ++d) z[i * DU + d] = __ldg(zr + i * RDU + d);
    }
#pragma unroll
    for (int i = 0; i < kSegMaxL; ++i) {
      if (i < L) {
#pragma unroll
        for (int d = 0; d < DU; ++d) {
          const float u = fminf(fmaxf(fmaf(p.sd, z[i * DU + d], bq[i * DU + d]), p.lower[d]), p.upper[d]);
          eff = fmaf(u, u, eff);
          q[d] = fmaf(p.dt, u, q[d]);
          P[((size_t)(t0 + i + 1) * R + k) * PD + d] = q[d];
        }
      }
    }
  }
  // ---- 2. offsets: x_0 + exclusive scan of the segment totals (8-lane groups)
  float off[PD];
#pragma unroll
  for (int d = 0; d < PD; ++d) {
    float incl = q[d];
#pragma unroll
    for (int o = 1; o < kSegs; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, incl, o, kSegs);
      if (j >= o) incl += y;
    }
    const float excl = __shfl_up_sync(0xffffffffu, incl, 1, kSegs);
    off[d] = (live ? p.starts[(size_t)k * PD + d] : 0.f) + (j > 0 ? excl : 0.f);
  }
  float gsd = 0.f;
  int bad_t = 0x3ff;
  if (live) {
    if (j == 0) {
#pragma unroll
      for (int d = 0; d < PD; ++d) P[(size_t)k * PD + d] = off[d];
    }
    const float ginv = p.inv_dstart[k];
    float gl[PD];
#pragma unroll
    for (int d = 0; d < PD; ++d) gl[d] = p.goals[(size_t)k * PD + d];
    for (int i = 0; i < L; ++i) {
      float* x = P + ((size_t)(t0 + i + 1) * R + k) * PD;
      float d2 = 0.f;
      bool fin = true;
#pragma unroll
      for (int d = 0; d < PD; ++d) {
        const float v = off[d] + x[d];
        x[d] = v;
        fin = fin && isfinite(v);
        const float e = v - gl[d];
        d2 = fmaf(e, e, d2);
      }
      if (!fin && bad_t == 0x3ff) bad_t = t0 + i + 1;
      gsd = fmaf(sqrt_approx(d2), ginv, gsd);
    }
    if (bad_t != 0x3ff) {  // first non-finite state of robot k (dynamics.cpp:81-84)
      const unsigned long long key = ((unsigned long long)p.step_key << 52) |
                                     ((unsigned long long)(p.m_global0 + m) << 20) |
                                     ((unsigned long long)k << 10) | (unsigned long long)bad_t;
      atomicMin(p.err, key);
    }
  }
  __syncthreads();
  // ---- 3. pair and obstacle tests for robot k's states in this segment
  int nc = 0, no = 0;
  if (live) {
    for (int i = 0; i < L; ++i) {
      const float* row = P + (size_t)(t0 + i + 1) * R * PD;
      float a[PD];
#pragma unroll
      for (int d = 0; d < PD; ++d) a[d] = row[k * PD + d];
      // direct form as the pair-list path: ‖Δp‖² − m²↑ < 0 ⟺ ‖Δp‖² ≤ m² (m²↑ =
      // the float after m², FitParams::margin_sq)
      bool hit = false;
      for (int l = 0; l < R; ++l) {
        float t = -p.margin_sq;
#pragma unroll
        for (int d = PD - 1; d >= 0; --d) {
          const float e = a[d] - row[l * PD + d];
          t = fmaf(e, e, t);
        }
        hit = hit || (l != k && t < 0.f);
      }
      nc += hit ? 1 : 0;
      // expanded form as the tile path: (|c|² − L²↑ + |a|²) − 2c·a < 0
      float a2 = 0.f;
#pragma unroll
      for (int d = 0; d < PD; ++d) a2 = fmaf(a[d], a[d], a2);
      bool ob = false;
      for (int o = 0; o < p.n_obs; ++o) {
        const float4 c = __ldg(reinterpret_cast<const float4*>(p.obs) + o);
        float v = c.w + a2;
        v = fmaf(c.x, a[0], v);
        v = fmaf(c.y, a[1], v);
        if constexpr (PD == 3) v = fmaf(c.z, a[2], v);
        ob = ob || v < 0.f;
      }
      no += ob ? 1 : 0;
    }
  }
  // ---- 4. per-sample fixed-order reduction: a shuffle tree per warp (a warp
  // never spans two samples: per_sample is 8·R ∈ {8, …, 128}), then the
  // sample's warps in index order
  double g = live ? (double)L - (double)gsd : 0.0, ef = live ? (double)eff : 0.0;
  int ncs = nc, nos = no;
  const int width = per_sample < 32 ? per_sample : 32;
  for (int o = width / 2; o > 0; o >>= 1) {
    g += __shfl_down_sync(0xffffffffu, g, o, width);
    ef += __shfl_down_sync(0xffffffffu, ef, o, width);
    ncs += __shfl_down_sync(0xffffffffu, ncs, o, width);
    nos += __shfl_down_sync(0xffffffffu, nos, o, width);
  }
  const int lane = tid & 31, w = tid >> 5;
  if (per_sample > 32) {
    if (lane == 0) {
      red[w] = g;
      red[4 + w] = ef;
      cnt[2 * w] = ncs;
      cnt[2 * w + 1] = nos;
    }
    __syncthreads();
    if (r == 0) {
      for (int q = 1; q < per_sample / 32; ++q) {
        g += red[w + q];
        ef += red[4 + w + q];
        ncs += cnt[2 * (w + q)];
        nos += cnt[2 * (w + q) + 1];
      }
    }
  }
  if (live && r == 0) {
    double value = g - p.w_t * (double)ncs - p.w_o * (double)nos;
    if (p.w_e != 0.0) value -= p.w_e * ef;
    p.reward[m] = value / ((double)R * (double)T);
    if (p.counts) {
      p.counts[2 * m] = ncs;
      p.counts[2 * m + 1] = nos;
    }
  }
}

namespace {
bool segs_ok(int segs, int R, int T, int du) {
  if (R < 1 || R * segs > 128 || 128 % (R * segs) != 0) return false;
  if (T % segs != 0 || T / segs > kSegMaxL) return false;
  return ((T / segs) * du) % 4 == 0;  // segments start on a Philox group
}
int segs_for(int R, int T, int du) {
  if (const char* e = std::getenv("D4ORM_SEGS")) {
    const int v = std::atoi(e);
    if ((v == 8 || v == 16) && segs_ok(v, R, T, du)) return v;
  }
  return 8;
}
}  // namespace

size_t seg_smem_bytes(int R, int T, int pdim) {
  const int spc = 128 / (R * segs_for(R, T, pdim));
  return (size_t)spc * (T + 1) * R * pdim * sizeof(float) + 8 * sizeof(double) + 8 * sizeof(int);
}

bool seg_supported(int kind, int R, int T, int du) {
  if (kind != HOLO2D_VEL && kind != HOLO3D_VEL) return false;
  return segs_ok(8, R, T, du);  // R ∈ {1, 2, 4, 8, 16}, T % 8 == 0, T ≤ 128
}

cudaError_t launch_seg(int kind, bool philox, int64_t M, cudaStream_t st, const FitParams<float>& f) {
  const int du = kind == HOLO3D_VEL ? 3 : 2;
  const int segs = segs_for(f.R, f.T, du);
  const int spc = 128 / (f.R * segs);
  const dim3 grid((unsigned)((M + spc - 1) / spc));
  const size_t smem = seg_smem_bytes(f.R, f.T, du);
  auto go = [&](auto k) { return launch_step(k, grid, dim3(128), smem, st, false, f); };
  if (kind == HOLO2D_VEL) {
    if (segs == 16) return philox ? go(k_rollout_fitness_seg<2, 1, 16>) : go(k_rollout_fitness_seg<2, 0, 16>);
    return philox ? go(k_rollout_fitness_seg<2, 1, 8>) : go(k_rollout_fitness_seg<2, 0, 8>);
  }
  if (segs == 16) return philox ? go(k_rollout_fitness_seg<3, 1, 16>) : go(k_rollout_fitness_seg<3, 0, 16>);
  return philox ? go(k_rollout_fitness_seg<3, 1, 8>) : go(k_rollout_fitness_seg<3, 0, 8>);
}

}  // namespace d4k
