// k_pl32.cuh — K2+K3 for planar teams of 33–64 robots on the production path
// (fp32, Philox noise drawn in registers, scalar std): the pair-list fitness of
// k23.cuh on 32-step chunks, one sample per 64-thread CTA, 11 CTAs per SM.
//
// k_rollout_fitness<…, PL> keeps a 64-step position tile per sample (71 KB per
// 128-thread CTA) and 168 registers: 3 CTAs = 12 warps per SM, and ncu shows it
// latency-bound there (issue 55 %, top stall "wait", no pipe above 40 %).  Here
// the tile is one 32-step warp window (19.5 KB per sample) and the dedicated
// kernel needs 79 registers with 8-step rollout blocks, so 11 CTAs = 22 warps
// are resident: C5 K2+K3 18.9 → 13.9 ms (history in DESIGN.md §3 / §7).
//
//  phase A  thread = robot: 32 steps in blocks of 8 (fused_block of k23.cuh:
//           Philox draws, controls, RK4, goal term, swept box); the row stride
//           of base + mean-scaled variable is a compile-time constant when
//           R = 64 (RFULL: no 64-bit address arithmetic per load).  LEAN
//           launches (the reference's reward, K5a regenerating the noise,
//           culling on) carry no effort accumulation, no z-store code and no
//           culling-off paths.
//  phase B  the window is shared by the sample's two warps: lane = step in both,
//           warp h votes and tests the pair-pair offsets d ≡ h + 1 (mod 2), the
//           obstacles o ≡ h (mod 2) and the own pairs l ≡ h (mod 2); warp 1
//           leaves its conflict / obstacle masks in shared memory and warp 0 ORs
//           and counts them after the phase barrier (a robot-step in conflict
//           with several others counts once, reward.cpp:104-110).  Votes test
//           this pair's two robot boxes (not their union) against the partner
//           pair's union box / the obstacle's box.
//
// The ranking (x strips of 8, y inside) is renewed every 64 steps and the
// per-robot fp32 goal / effort partials are folded every 64 steps, exactly as
// the 64-step kernel does, and all culling is exact, so rewards and counts are
// bitwise those of k_rollout_fitness<float, KIND, 16, 2, 1, true>
// (tests/test_gpu_pl32.py; the effort sum differs by fp32 association where
// effort_weight ≠ 0).
#pragma once

#include "k23.cuh"

namespace d4k {

#ifndef D4K_PL32_SPC
#define D4K_PL32_SPC 1  // samples per CTA (64 threads each)
#endif
constexpr int kPl32Spc = D4K_PL32_SPC, kPl32Threads = 64 * kPl32Spc, kPl32TC = 32, kPl32Rp = 64, kPl32RS = 66;
#ifndef D4K_PL32_KPF
#define D4K_PL32_KPF 8
#endif
#ifndef D4K_PL32_STRIP
#define D4K_PL32_STRIP 8  // robots per x strip of the ranking (y order inside a strip)
#endif
#ifndef D4K_PL32_RANK
#define D4K_PL32_RANK 64  // steps between rankings (a multiple of 32)
#endif
#ifndef D4K_PL32_MINB
#define D4K_PL32_MINB (11 / D4K_PL32_SPC)
#endif

struct Pl32Smem {
  float* pos;     // [2 planes][spc samples][32 steps][66]
  int* key;       // [spc][64] ranking keys (aliases pbox)
  float4* rbox;   // [spc][64] robot swept boxes of the window (lo.x, lo.y, hi.x, hi.y)
  float4* pbox;   // [spc][64] inflated pair boxes, stored twice (index l and l + 32: no wrap); a sample's two
                  // warps both write it — the same values — and each reads after its own writes
  uint4* msk;     // [spc][32 lanes] warp 1's (conflict, obstacle) masks
  float* opl;     // [O][8] FitParams::obs_pl
  __device__ __forceinline__ float* row(int c, int s, int tc) const {
    D4K_CHECK(c >= 0 && c < 2 && s >= 0 && s < kPl32Spc && tc >= 0 && tc < kPl32TC);
    return pos + ((c * kPl32Spc + s) * kPl32TC + tc) * kPl32RS;
  }
};

__host__ __device__ inline size_t pl32_smem_bytes(int n_obs) {
  size_t b = (size_t)2 * kPl32Spc * kPl32TC * kPl32RS * sizeof(float);  // pos (33 792 B; the final reduction aliases it)
  b += (size_t)kPl32Spc * kPl32Rp * sizeof(float4);                       // rbox
  b += (size_t)kPl32Spc * 64 * sizeof(float4);                            // pbox (the ranking keys alias it)
  b += (size_t)kPl32Spc * 32 * sizeof(uint4);                             // msk
  b += (size_t)8 * (n_obs > 0 ? n_obs : 1) * sizeof(float);               // opl
  return (b + 15) & ~size_t(15);
}

__device__ __forceinline__ int top_bit(uint32_t v) {  // index of the highest set bit (v ≠ 0): one FLO
  int r;
  asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// Half h of one (sample, 32-step window) item: called by all 32 lanes of a warp,
// lane = step.  Returns the conflict / obstacle bits (bit = column) this half finds.
template <bool CULLC>  // CULLC: culling known on at compile time (production); else `cull_rt` decides
__device__ __forceinline__ void item_pl32(const Pl32Smem& sm, int s, int h, int n_obs, float m2u, float cmh,
                                          bool cull_rt, uint64_t& conf, uint64_t& obsm) {
  const bool cull = CULLC || cull_rt;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const float* X = sm.row(0, s, lane);
  const float* Y = sm.row(1, s, lane);
  const float4* rb = sm.rbox + s * kPl32Rp;
  float4* pb = sm.pbox + s * 64;
  const uint64_t nm2 = pack2(-m2u, -m2u);
  D4K_CHECK(s >= 0 && s < kPl32Spc && (h == 0 || h == 1) && n_obs >= 0);
  const float4 b0 = rb[2 * lane], b1 = rb[2 * lane + 1];
  // the pair's union box grown by half the margin: what the partners' votes test against
  const float4 Ai = make_float4(fminf(b0.x, b1.x) - cmh, fminf(b0.y, b1.y) - cmh, fmaxf(b0.z, b1.z) + cmh,
                                fmaxf(b0.w, b1.w) + cmh);
  // the robots' own boxes grown by half the margin (the votes test them against
  // the partner pair's union box, not union against union: a pair whose union
  // meets only the gap between this pair's two robots is no candidate)
  const float4 b0i = make_float4(b0.x - cmh, b0.y - cmh, b0.z + cmh, b0.w + cmh);
  const float4 b1i = make_float4(b1.x - cmh, b1.y - cmh, b1.z + cmh, b1.w + cmh);
  pb[lane] = Ai;
  pb[lane + 32] = Ai;
  {  // the pairs' own tests (2l, 2l+1): both warps vote, warp h tests the pairs l ≡ h (mod 2)
    uint32_t bits = 0x55555555u << h;
    if (cull) bits &= __ballot_sync(full, boxes_meet(b0i, b1i));
    while (bits) {
      const int l = top_bit(bits);
      bits ^= 1u << l;
      const float2 x = *reinterpret_cast<const float2*>(X + 2 * l);
      const float2 y = *reinterpret_cast<const float2*>(Y + 2 * l);
      const float dx = x.y - x.x, dy = y.y - y.x;
      const float t = fmaf(dx, dx, fmaf(dy, dy, -m2u));
      if (t < 0.f) conf |= 3ull << (2 * l);
    }
  }
  __syncwarp();
  // pair-pair blocks (l, l + d mod 32) for this half's offsets d = 2i + 1 + h
  // (h = 0: 1, 3, …, 15; h = 1: 2, 4, …, 16, d = 16 once per pair): the ballots
  // first (independent loads and votes), then the live blocks
  uint32_t lv[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int d = 2 * i + 1 + h;
    if (cull) {
      D4K_CHECK(lane + d < 64);
      const float4 B = pb[lane + d];
      lv[i] = __ballot_sync(full, (d < 16 || lane < 16) && (boxes_meet(b0i, B) || boxes_meet(b1i, B)));
    } else {
      lv[i] = d < 16 ? full : 0xffffu;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int d = 2 * i + 1 + h;
    uint32_t live = lv[i];
    while (live) {
      const int l1 = top_bit(live);
      live ^= 1u << l1;
      pl_block(X, Y, l1, (l1 + d) & 31, nm2, conf);
    }
  }
  // obstacles o ≡ h (mod 2): pair boxes vs the obstacles' inflated boxes, eight ballots at a time
  for (int o0 = h; o0 < n_obs; o0 += 16) {
    uint32_t ov[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int o = o0 + 2 * q;
      ov[q] = 0;
      if (o < n_obs) {
        // the pair's two robot boxes, not their union: an obstacle in the gap between the two is no candidate
        const float4 ob = *reinterpret_cast<const float4*>(sm.opl + 8 * o + 4);
        ov[q] = cull ? __ballot_sync(full, boxes_meet(b0, ob) || boxes_meet(b1, ob)) : full;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t live = ov[q];
      if (!live) continue;
      const float4 oc = *reinterpret_cast<const float4*>(sm.opl + 8 * (o0 + 2 * q));  // cx, cy, −L²↑
      const uint64_t cx = pack2(oc.x, oc.x), cy = pack2(oc.y, oc.y), nl = pack2(oc.z, oc.z);
      while (live) {
        const int l = top_bit(live);
        live ^= 1u << l;
        const uint64_t xa = *reinterpret_cast<const uint64_t*>(X + 2 * l);
        const uint64_t ya = *reinterpret_cast<const uint64_t*>(Y + 2 * l);
        uint64_t t = ffma2_sq(fsub2(xa, cx), nl);
        t = ffma2_sq(fsub2(ya, cy), t);
        if ((int)(lo32(t) | hi32(t)) < 0)
          obsm |= (uint64_t)((lo32(t) >> 31) | ((hi32(t) >> 31) << 1)) << (2 * l);
      }
    }
  }
}

template <int KIND, bool RFULL, bool LEAN>
__global__ void __launch_bounds__(kPl32Threads, D4K_PL32_MINB) k_rollout_fitness_pl32(const __grid_constant__ FitParams<float> p) {
  pdl_wait();
  constexpr int DX = ModelDims<KIND>::DX, DU = ModelDims<KIND>::DU, PD = ModelDims<KIND>::PD;
  static_assert(PD == 2 && DU == 2, "pair-list path: planar two-control kinds");
  constexpr int KPF = D4K_PL32_KPF, TC = kPl32TC, Rp = kPl32Rp, spc = kPl32Spc, nthreads = kPl32Threads;
  constexpr int RDUC = RFULL ? Rp * DU : 0;
  static_assert(TC % KPF == 0 && (KPF * DU) % 4 == 0, "block depth");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int R = RFULL ? Rp : p.R, T = p.T;

  Pl32Smem sm;
  sm.pos = reinterpret_cast<float*>(smem_raw);
  sm.rbox = reinterpret_cast<float4*>(sm.pos + 2 * spc * TC * kPl32RS);
  sm.pbox = sm.rbox + spc * Rp;
  // the ranking keys live in the pair-box array: keys are written and read between the
  // end-of-window barrier and phase A, pair boxes between the phase barriers
  sm.key = reinterpret_cast<int*>(sm.pbox);
  sm.msk = reinterpret_cast<uint4*>(sm.pbox + spc * 64);
  sm.opl = reinterpret_cast<float*>(sm.msk + spc * 32);
  for (int j = tid; j < 8 * p.n_obs; j += nthreads) sm.opl[j] = p.obs_pl[j];  // (c, −L²↑, box)

  // ---- phase-A identity: (sample sA, robot kA)
  const int sA = tid >> 6, kA = tid & 63;
  const int64_t mA = (int64_t)blockIdx.x * spc + sA;
  const bool liveA = mA < p.M;
  const bool robotA = liveA && kA < R;
  float x[DX];
#pragma unroll
  for (int j = 0; j < DX; ++j) x[j] = robotA ? p.starts[kA * DX + j] : 0.f;
  if (liveA && kA >= R) {  // padding robots: parked far apart, never counted; empty window box
    for (int tc = 0; tc < TC; ++tc) {
      sm.row(0, sA, tc)[kA] = 1.0e6f + 1.0e3f * (float)kA;
      sm.row(1, sA, tc)[kA] = -1.0e6f - 1.0e3f * (float)kA;
    }
    sm.rbox[sA * Rp + kA] = empty_box();
  }
  float effort = 0.f, eff32 = 0.f, goalA = 0.f, gsd = 0.f;
  float ng[2] = {0.f, 0.f}, ginv = 0.f;
  if (robotA) {
    ng[0] = -p.goals[kA * PD];
    ng[1] = -p.goals[kA * PD + 1];
    ginv = p.inv_dstart[kA];
  }
  const int RDU = R * DU;
  float* zst = p.z_store + (liveA ? mA : 0) * (int64_t)T * RDU;
  const uint2 key = p.keys[p.step];

  // ---- phase-B identity: warp w = (sample sB, half hB), lane = step of the window
  const int wB = tid >> 5, sB = wB >> 1, hB = wB & 1, lane = tid & 31;
  const int64_t mB = (int64_t)blockIdx.x * spc + sB;
  const uint64_t real = R >= 64 ? ~0ull : ((1ull << R) - 1ull);
  int nconf = 0, nobs = 0;
  int rA = kA;
  int period0 = 0;  // first step of the current 64-step fold period

  __syncthreads();

  for (int t0 = 0; t0 < T; t0 += TC) {
    // ===== every 64 steps: rank the sample's robots by x (strips of D4K_PL32_STRIP), then by y
    // inside a strip, so column pairs (2l, 2l+1) are neighbours in both coordinates
    if ((t0 % D4K_PL32_RANK) == 0) {
      // keys are 31-bit unsigned (order-preserving float bits >> 1, low 6 bits = lane: unique),
      // so "k < me" is the top bit of k − me: two instructions per key (IADD + LEA.HI into
      // one of four independent counters) instead of a compare-select chain
      if (liveA) {
        int xi = __float_as_int(x[0]);
        xi ^= (xi >> 31) & 0x7fffffff;
        const uint32_t xu = robotA ? (((uint32_t)xi ^ 0x80000000u) >> 1) : 0x7fffffffu;  // padding sorts last
        sm.key[tid] = (int)((xu & ~63u) | (uint32_t)kA);
      }
      __syncthreads();
      if (robotA) {
        const uint32_t me = (uint32_t)sm.key[tid];
        const uint4* kv = reinterpret_cast<const uint4*>(sm.key + sA * Rp);
        uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll 4
        for (int j = 0; j < Rp / 4; ++j) {
          const uint4 v = kv[j];
          r0 += (v.x - me) >> 31;
          r1 += (v.y - me) >> 31;
          r2 += (v.z - me) >> 31;
          r3 += (v.w - me) >> 31;
        }
        rA = (int)((r0 + r1) + (r2 + r3));
      }
      __syncthreads();
      uint32_t me = 0;
      if (liveA) {
        int yi = __float_as_int(x[1]);
        yi ^= (yi >> 31) & 0x7fffffff;
        const uint32_t yu = (uint32_t)yi ^ 0x80000000u;
        me = robotA ? (((yu >> 10) << 6) | (uint32_t)kA) : (0x7fffffc0u | (uint32_t)kA);
        D4K_CHECK(rA >= 0 && rA < Rp);
        sm.key[sA * Rp + rA] = (int)me;
      }
      __syncthreads();
      if (robotA) {
        const uint4* kv = reinterpret_cast<const uint4*>(sm.key + sA * Rp + (rA & ~(D4K_PL32_STRIP - 1)));
        uint32_t r0 = (uint32_t)(rA & ~(D4K_PL32_STRIP - 1)), r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
        for (int j = 0; j < D4K_PL32_STRIP / 4; ++j) {
          const uint4 v = kv[j];
          r0 += (v.x - me) >> 31;
          r1 += (v.y - me) >> 31;
          r2 += (v.z - me) >> 31;
          r3 += (v.w - me) >> 31;
        }
        rA = (int)((r0 + r1) + (r2 + r3));
      }
    }
    // ===== phase A: integrate the window's steps
    const int nsteps = t0 + TC < T ? TC : T - t0;
    if (robotA) {
      float x0[DX];
#pragma unroll
      for (int q = 0; q < DX; ++q) x0[q] = x[q];
      const int64_t e0 = ((int64_t)t0 * R + kA) * DU;
      const float* bmp = p.bm + e0;
      float* zp = zst + e0;
      float* px = sm.row(0, sA, 0) + rA;
      float* py = sm.row(1, sA, 0) + rA;
      float chk = 0.f;
      float4 bx = empty_box();
      D4K_CHECK(rA >= 0 && rA < Rp);
      for (int tc = 0; tc < nsteps; tc += KPF) {
        const int nb = nsteps - tc;
        const uint32_t g0 = (uint32_t)((t0 + tc) * DU / 4);
        if (nb >= KPF)
          fused_block<KIND, true, false, true, KPF, RDUC, !LEAN, !LEAN>(p, KPF, bmp, nullptr, zp, RDU, (uint64_t)(p.m_global0 + mA), kA, g0,
                                                          key, px, py, px, kPl32RS, x, eff32, chk, ng, ginv, gsd, bx);
        else
          fused_block<KIND, false, false, true, KPF, RDUC, !LEAN, !LEAN>(p, nb, bmp, nullptr, zp, RDU, (uint64_t)(p.m_global0 + mA), kA,
                                                           g0, key, px, py, px, kPl32RS, x, eff32, chk, ng, ginv, gsd, bx);
        bmp += KPF * RDU;
        zp += KPF * RDU;
        px += KPF * kPl32RS;
        py += KPF * kPl32RS;
      }
      D4K_CHECK(sA * Rp + rA < spc * Rp);
      sm.rbox[sA * Rp + rA] = bx;
      // state = position (velocity-input kinds): a NaN/inf state reaches the goal
      // distance, so the goal sum carries it (k23.cuh rollout_fused)
      if constexpr (DX == PD) chk = gsd * 0.f;
      if (!(chk == 0.f)) rollout_check<KIND>(p, kA, p.m_global0 + mA, t0, nsteps, x0, zst);
      if (((t0 + TC) & 63) == 0 || t0 + TC >= T) {  // fold the fp32 partials of this 64-step period
        goalA += (float)(t0 + nsteps - period0) - gsd;
        gsd = 0.f;
        effort += eff32;
        eff32 = 0.f;
        period0 = t0 + nsteps;
      }
    }
    __syncthreads();

    // ===== phase B: this warp's half of the window's fitness
    uint64_t conf = 0, obsm = 0;
    if (mB < p.M) {
      item_pl32<LEAN>(sm, sB, hB, p.n_obs, p.margin_sq, 0.5f * p.cull_margin, p.cull != 0, conf, obsm);
      if (hB == 1) sm.msk[sB * 32 + lane] = make_uint4(lo32(conf), hi32(conf), lo32(obsm), hi32(obsm));
    }
    __syncthreads();
    if (hB == 0 && mB < p.M && t0 + lane < T) {
      const uint4 o = sm.msk[sB * 32 + lane];
      conf |= (uint64_t)o.x | ((uint64_t)o.y << 32);
      obsm |= (uint64_t)o.z | ((uint64_t)o.w << 32);
      nconf += __popcll(conf & real);
      nobs += __popcll(obsm & real);
    }
  }

  // ---- per-sample deterministic reduction (the order of k_rollout_fitness)
  __syncthreads();
  double* red = reinterpret_cast<double*>(smem_raw);  // aliases pos (dead now)
  double* eff = red + nthreads;
  int* cnt = reinterpret_cast<int*>(eff + nthreads);
  red[tid] = robotA ? (double)goalA : 0.0;
  eff[tid] = robotA ? (double)effort : 0.0;
  cnt[2 * tid] = nconf;
  cnt[2 * tid + 1] = nobs;
  __syncthreads();
  if (mB < p.M && tid == sB * Rp) {  // first thread of the sample
    const int first = sB * Rp;
    double g = 0.0;
    long long nc = 0, no = 0;
    for (int q = 0; q < Rp; ++q) {
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
    p.reward[mB] = value / ((double)R * (double)T);
    if (p.counts) {
      p.counts[2 * mB] = (int)nc;
      p.counts[2 * mB + 1] = (int)no;
    }
  }
}

// Launch (grid = ⌈M / spc⌉ CTAs of 64·spc threads).  Planar two-control kinds only.
template <int KIND>
cudaError_t launch_pl32(cudaStream_t st, const FitParams<float>& p) {
  if constexpr (ModelDims<KIND>::PD == 2 && ModelDims<KIND>::DU == 2) {
    const size_t smem = pl32_smem_bytes(p.n_obs);
    const dim3 grid((unsigned)((p.M + kPl32Spc - 1) / kPl32Spc));
    auto launch = [&](auto fn) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
      if (e != cudaSuccess) return e;
      return launch_step(fn, grid, dim3(kPl32Threads), smem, st, false, p);
    };
    // LEAN: the reference's reward (effort_weight = 0) on a launch whose K5a regenerates the
    // noise (z_keep == 2), culling on — no effort accumulation and no z-store code in the
    // rollout block, no culling-off paths in the votes
    if (p.w_e == 0.0 && p.z_keep == 2 && p.cull != 0) {
      if (p.R == kPl32Rp) return launch(k_rollout_fitness_pl32<KIND, true, true>);
      return launch(k_rollout_fitness_pl32<KIND, false, true>);
    }
    if (p.R == kPl32Rp) return launch(k_rollout_fitness_pl32<KIND, true, false>);
    return launch(k_rollout_fitness_pl32<KIND, false, false>);
  } else {
    return cudaErrorInvalidValue;
  }
}

}  // namespace d4k
