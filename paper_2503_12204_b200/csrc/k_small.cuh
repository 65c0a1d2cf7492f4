// k_small.cuh — K2+K3 for small teams (R ≤ 16: BASELINE C2, C3, C4) on the
// production path (fp32, Philox noise drawn in registers, scalar std).
//
// These launches are one-wave problems: 131 072 robot threads = 1024 CTAs of
// 128.  The general kernel (k_rollout_fitness<float, KIND, 8, 2, 1>) is capped
// at 96 registers there and spills (120–168 B of stack), so 5 CTAs per SM are
// resident: 740 slots, 1.38 waves, the second wave 38 % full.  This kernel is
// the same arithmetic — fused_block for the rollout, item_f32 (robot tiles of
// 8, expanded-form pair tests) for the fitness, 16-step chunks — with nothing
// else in it, so that it fits 7 CTAs per SM (72 registers): 1036 slots, every
// CTA of C2–C4 resident in one wave at 28 warps per SM.  LEAN instantiations drop
// the effort accumulation (effort_weight = 0) and, where K5a regenerates the
// noise (C4), the z-store code.
//
// Same chunk length and fold order as the general kernel: rewards and counts are
// bitwise equal to it (tests/test_gpu_small.py; the effort sum of the
// two-control kinds differs by fp32 association where effort_weight ≠ 0).
#pragma once

#include "k23.cuh"

namespace d4k {

#ifndef D4K_SMALL_THREADS
#define D4K_SMALL_THREADS 128
#endif
constexpr int kSmallThreads = D4K_SMALL_THREADS, kSmallTC = 16, kSmallTB = 8;
#ifndef D4K_SMALL_KPF
#define D4K_SMALL_KPF 8
#endif
#ifndef D4K_SMALL_MINB
#define D4K_SMALL_MINB (7 * 128 / D4K_SMALL_THREADS)
#endif

template <int PD>
__host__ __device__ inline size_t small_smem_bytes(int RP, int n_obs) {
  const int spc = kSmallThreads / RP;
  size_t pos = (size_t)PD * spc * kSmallTC * (RP + 2) * sizeof(float);
  const size_t red = 2 * (size_t)kSmallThreads * sizeof(double) + 2 * (size_t)kSmallThreads * sizeof(int);
  size_t b = ((pos > red ? pos : red) + 15) & ~size_t(15);
  b += (size_t)4 * (n_obs + 1) * sizeof(float);
  return (b + 15) & ~size_t(15);
}

template <int KIND, int RP, int LEAN>  // LEAN bit 0: no effort accumulation, bit 1: no z-store code
__global__ void __launch_bounds__(kSmallThreads, D4K_SMALL_MINB) k_rollout_fitness_small(const __grid_constant__ FitParams<float> p) {
  pdl_wait();
  constexpr int DX = ModelDims<KIND>::DX, DU = ModelDims<KIND>::DU, PD = ModelDims<KIND>::PD;
  constexpr int TB = kSmallTB, TC = kSmallTC, spc = kSmallThreads / RP, RS = RP + 2, nthreads = kSmallThreads;
  constexpr int KPF = D4K_SMALL_KPF;
  static_assert(RP % TB == 0 && RP <= 16 && TC % KPF == 0 && (KPF * DU) % 4 == 0 && TC % RP == 0, "shape");
  constexpr int ipt = TC / RP;  // fitness items per thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int R = p.R, T = p.T;

  FitSmem<float> sm;
  sm.npd = PD;
  sm.RS = RS;
  sm.TC = TC;
  sm.spc = spc;
  sm.Rp = RP;
  sm.nthreads = nthreads;
  sm.pos = reinterpret_cast<float*>(smem_raw);
  {
    constexpr size_t pos_b = (size_t)PD * spc * TC * RS * sizeof(float);
    constexpr size_t red_b = 2 * (size_t)nthreads * sizeof(double) + 2 * (size_t)nthreads * sizeof(int);
    sm.obs = reinterpret_cast<float*>(smem_raw + (((pos_b > red_b ? pos_b : red_b) + 15) & ~size_t(15)));
  }
  sm.goal = sm.inv = sm.ocl = sm.bb = sm.opl = nullptr;
  sm.key = nullptr;
  sm.pbox = nullptr;
  for (int j = tid; j < 4 * (p.n_obs + 1); j += nthreads) sm.obs[j] = p.obs[j];  // (−2c, |c|²−L²↑), pad row

  // ---- phase-A identity: (sample sA, robot kA)
  const int sA = tid / RP, kA = tid % RP;
  const int64_t mA = (int64_t)blockIdx.x * spc + sA;
  const bool liveA = mA < p.M;
  const bool robotA = liveA && kA < R;
  float x[DX];
#pragma unroll
  for (int j = 0; j < DX; ++j) x[j] = robotA ? p.starts[kA * DX + j] : 0.f;
  if (liveA && kA >= R) {  // padding robots: parked far apart, never counted
    for (int tc = 0; tc < TC; ++tc) {
      sm.row(0, sA, tc)[kA] = 1.0e6f + 1.0e3f * (float)kA;
      sm.row(1, sA, tc)[kA] = -1.0e6f - 1.0e3f * (float)kA;
      if constexpr (PD == 3) sm.row(2, sA, tc)[kA] = 1.0e6f;
    }
  }
  float effort = 0.f, eff32 = 0.f, goalA = 0.f;
  float ng[3] = {0.f, 0.f, 0.f}, ginv = 0.f;
  if (robotA) {
#pragma unroll
    for (int c = 0; c < PD; ++c) ng[c] = -p.goals[kA * PD + c];
    ginv = p.inv_dstart[kA];
  }
  const int RDU = R * DU;
  float* zst = p.z_store + (liveA ? mA : 0) * (int64_t)T * RDU;
  const uint2 key = p.keys[p.step];

  // ---- phase-B identity: ipt consecutive (sample, step) items per thread
  const int item0 = tid * ipt;
  const int sB = item0 / TC;
  const int64_t mB = (int64_t)blockIdx.x * spc + sB;
  const bool liveB = mB < p.M;
  int nconf = 0, nobs = 0;

  __syncthreads();

  for (int t0 = 0; t0 < T; t0 += TC) {
    // ===== phase A: integrate the chunk's steps
    const int nsteps = t0 + TC < T ? TC : T - t0;
    if (robotA) {
      float x0[DX];
#pragma unroll
      for (int q = 0; q < DX; ++q) x0[q] = x[q];
      const int64_t e0 = ((int64_t)t0 * R + kA) * DU;
      const float* bmp = p.bm + e0;
      float* zp = zst + e0;
      float* px = sm.row(0, sA, 0) + kA;
      float* py = sm.row(1, sA, 0) + kA;
      float* pz = PD == 3 ? sm.row(2, sA, 0) + kA : px;
      float chk = 0.f, gsd = 0.f;
      float4 bx;
      for (int tc = 0; tc < nsteps; tc += KPF) {
        const int nb = nsteps - tc;
        const uint32_t g0 = (uint32_t)((t0 + tc) * DU / 4);
        if (nb >= KPF)
          fused_block<KIND, true, false, false, KPF, 0, !(LEAN & 1), !(LEAN & 2)>(p, KPF, bmp, nullptr, zp, RDU, (uint64_t)(p.m_global0 + mA), kA, g0, key,
                                                     px, py, pz, RS, x, eff32, chk, ng, ginv, gsd, bx);
        else
          fused_block<KIND, false, false, false, KPF, 0, !(LEAN & 1), !(LEAN & 2)>(p, nb, bmp, nullptr, zp, RDU, (uint64_t)(p.m_global0 + mA), kA, g0,
                                                      key, px, py, pz, RS, x, eff32, chk, ng, ginv, gsd, bx);
        bmp += KPF * RDU;
        zp += KPF * RDU;
        px += KPF * RS;
        py += KPF * RS;
        pz += KPF * RS;
      }
      goalA += (float)nsteps - gsd;
      // state = position (velocity-input kinds): a NaN/inf state reaches the goal
      // distance, so the goal sum carries it (k23.cuh rollout_fused)
      if constexpr (DX == PD) chk = gsd * 0.f;
      if (!(chk == 0.f)) rollout_check<KIND>(p, kA, p.m_global0 + mA, t0, nsteps, x0, zst);
    }
    effort += eff32;
    eff32 = 0.f;
    __syncthreads();

    // ===== phase B: fitness of the steps just integrated
    if (liveB) {
#pragma unroll
      for (int j = 0; j < ipt; ++j) {
        const int tc = item0 + j - sB * TC;
        if (t0 + tc >= T) break;
        uint32_t cm[1] = {0u};
        item_f32<PD, TB, 1, false>(sm, sB, tc, R, p.n_obs, p.margin_sq, p.cull_margin, 0, 1, nullptr, cm, &nobs);
        nconf += __popc(cm[0] & ((1u << R) - 1u));
      }
    }
    __syncthreads();
  }

  // ---- per-sample deterministic reduction (the order of k_rollout_fitness)
  double* red = reinterpret_cast<double*>(smem_raw);  // aliases pos (dead now)
  double* eff = red + nthreads;
  int* cnt = reinterpret_cast<int*>(eff + nthreads);
  red[tid] = robotA ? (double)goalA : 0.0;
  eff[tid] = robotA ? (double)effort : 0.0;
  cnt[2 * tid] = liveB ? nconf : 0;
  cnt[2 * tid + 1] = liveB ? nobs : 0;
  __syncthreads();
  if (liveA && kA == 0) {  // first thread of the sample
    const int first = sA * RP;
    double g = 0.0;
    long long nc = 0, no = 0;
    for (int q = 0; q < RP; ++q) {
      g += red[first + q];
      nc += cnt[2 * (first + q)];
      no += cnt[2 * (first + q) + 1];
    }
    double value = g - p.w_t * (double)nc - p.w_o * (double)no;
    if (p.w_e != 0.0) {  // effort extension
      double es = 0.0;
      for (int k = 0; k < R; ++k) es += eff[first + k];
      value -= p.w_e * es;
    }
    p.reward[mA] = value / ((double)R * (double)T);
    if (p.counts) {
      p.counts[2 * mA] = (int)nc;
      p.counts[2 * mA + 1] = (int)no;
    }
  }
}

// Launch (grid = ⌈M / spc⌉ CTAs of 128 threads); rp = robot lanes per sample (8 or 16).
template <int KIND>
cudaError_t launch_small(int rp, cudaStream_t st, const FitParams<float>& p) {
  constexpr int PD = ModelDims<KIND>::PD;
  const size_t smem = small_smem_bytes<PD>(rp, p.n_obs);
  const int spc = kSmallThreads / rp;
  const dim3 grid((unsigned)((p.M + spc - 1) / spc));
  auto launch = [&](auto fn) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return launch_step(fn, grid, dim3(kSmallThreads), smem, st, false, p);
  };
  // the reference's reward (effort_weight = 0) compiles the effort accumulation out; a launch
  // whose K5a regenerates the noise (z_keep == 2, e.g. C4) also the z-store code
  const int lean = p.w_e != 0.0 ? 0 : (p.z_keep == 2 ? 3 : 1);
  if (rp == 16) {
    if (lean == 3) return launch(k_rollout_fitness_small<KIND, 16, 3>);
    if (lean == 1) return launch(k_rollout_fitness_small<KIND, 16, 1>);
    return launch(k_rollout_fitness_small<KIND, 16, 0>);
  }
  if (rp == 8) {
    if (lean == 3) return launch(k_rollout_fitness_small<KIND, 8, 3>);
    if (lean == 1) return launch(k_rollout_fitness_small<KIND, 8, 1>);
    return launch(k_rollout_fitness_small<KIND, 8, 0>);
  }
  return cudaErrorInvalidValue;
}

}  // namespace d4k
