// d4orm_kernels.cuh — the five sm_100a kernels of the denoise-step hot path.
//
//   K1 k_philox_noise      counter-based Philox4x32-10 + Box-Muller → z[m][t][k][d]
//   K2+K3 k_rollout_fitness fused rollout (RK4, clamp) + team fitness (goal,
//                           effort, obstacle, O(R²T) pair terms) → reward[m]
//   K4 k_score_weights     z-scored softmax weights (fp64), entropy, best/mean
//   K5 k_wmean_partial     streaming weighted mean over [chunk of m] × E
//      k_wmean_tree        deterministic pairwise tree over chunk partials +
//                          the denoise update var ← √ᾱ_{i−1} · Σ_m w_m sample_m
//
// Reference semantics: denoiser.cpp:152-180 (loop body), dynamics.cpp:65-87,
// dynamics.hpp:81-130 (rollout/RK4), reward.cpp:67-130 (total_reward),
// denoiser.cpp:50-108 (score_weights, mc_average), schedule.cpp:29-36.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <type_traits>

namespace d4k {

constexpr int kThreads = 256;

enum Kind { DIFFDRIVE = 0, HOLO2D = 1, HOLO3D = 2, HOLO2D_VEL = 3, HOLO3D_VEL = 4, UNICYCLE = 5 };

template <int KIND>
struct ModelDims;
template <> struct ModelDims<DIFFDRIVE> { static constexpr int DX = 4, DU = 2, PD = 2; };
template <> struct ModelDims<HOLO2D> { static constexpr int DX = 4, DU = 2, PD = 2; };
template <> struct ModelDims<HOLO3D> { static constexpr int DX = 6, DU = 3, PD = 3; };
template <> struct ModelDims<HOLO2D_VEL> { static constexpr int DX = 2, DU = 2, PD = 2; };
template <> struct ModelDims<HOLO3D_VEL> { static constexpr int DX = 3, DU = 3, PD = 3; };
template <> struct ModelDims<UNICYCLE> { static constexpr int DX = 3, DU = 2, PD = 2; };

// ---------------------------------------------------------------- scalar ops
// fp64 (parity) mode evaluates every expression exactly as the reference's
// x86-64 build does: separately rounded mul/add, never contracted to FMA.
// fp32 (throughput) mode lets the compiler contract freely.
template <typename S> __device__ __forceinline__ S xmul(S a, S b);
template <typename S> __device__ __forceinline__ S xadd(S a, S b);
template <> __device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ float xmul(float a, float b) { return a * b; }
template <> __device__ __forceinline__ float xadd(float a, float b) { return a + b; }
template <typename S> __device__ __forceinline__ S xsub(S a, S b) { return xadd(a, -b); }

__device__ __forceinline__ void xsincos(double a, double* s, double* c) { sincos(a, s, c); }
__device__ __forceinline__ void xsincos(float a, float* s, float* c) { sincosf(a, s, c); }
__device__ __forceinline__ double xsqrt(double a) { return sqrt(a); }
__device__ __forceinline__ float xsqrt(float a) { return sqrtf(a); }

// Derivative functors (dynamics.hpp:81-119 and the three BASELINE extensions).
template <int KIND, typename S>
__device__ __forceinline__ void deriv(const S* x, const S* u, S* f) {
  if constexpr (KIND == DIFFDRIVE) {
    S sn, cs;
    xsincos(x[2], &sn, &cs);
    f[0] = xmul(x[3], cs);
    f[1] = xmul(x[3], sn);
    f[2] = u[0];
    f[3] = u[1];
  } else if constexpr (KIND == HOLO2D) {
    f[0] = x[2]; f[1] = x[3]; f[2] = u[0]; f[3] = u[1];
  } else if constexpr (KIND == HOLO3D) {
    f[0] = x[3]; f[1] = x[4]; f[2] = x[5]; f[3] = u[0]; f[4] = u[1]; f[5] = u[2];
  } else if constexpr (KIND == HOLO2D_VEL) {
    f[0] = u[0]; f[1] = u[1];
  } else if constexpr (KIND == HOLO3D_VEL) {
    f[0] = u[0]; f[1] = u[1]; f[2] = u[2];
  } else {  // UNICYCLE
    S sn, cs;
    xsincos(x[2], &sn, &cs);
    f[0] = xmul(u[0], cs);
    f[1] = xmul(u[0], sn);
    f[2] = u[1];
  }
}

// detail::rk4_with (dynamics.hpp:123-130), element order as Eigen evaluates it.
template <int KIND, typename S>
__device__ __forceinline__ void rk4(S* x, const S* u, S dt, S half_dt, S dt6) {
  constexpr int DX = ModelDims<KIND>::DX;
  S k1[DX], k2[DX], k3[DX], k4[DX], tmp[DX];
  deriv<KIND>(x, u, k1);
#pragma unroll
  for (int j = 0; j < DX; ++j) tmp[j] = xadd(x[j], xmul(half_dt, k1[j]));
  deriv<KIND>(tmp, u, k2);
#pragma unroll
  for (int j = 0; j < DX; ++j) tmp[j] = xadd(x[j], xmul(half_dt, k2[j]));
  deriv<KIND>(tmp, u, k3);
#pragma unroll
  for (int j = 0; j < DX; ++j) tmp[j] = xadd(x[j], xmul(dt, k3[j]));
  deriv<KIND>(tmp, u, k4);
#pragma unroll
  for (int j = 0; j < DX; ++j) {
    const S acc = xadd(xadd(xadd(k1[j], xmul(S(2), k2[j])), xmul(S(2), k3[j])), k4[j]);
    x[j] = xadd(x[j], xmul(dt6, acc));
  }
}

// ------------------------------------------------------------------ K1 noise
// Philox4x32-10 (Salmon et al., SC'11).  Key = (seed_it, step i) mixed by
// splitmix64; counter = (group q, global sample m lo, m hi, 0).  Every normal is
// a pure function of (seed, i, m, element), so any sample sharding across GPUs
// sees the identical noise.
struct Philox {
  static __device__ __forceinline__ uint4 round(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  static __device__ __forceinline__ uint4 gen(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

__device__ __forceinline__ float u01_open(uint32_t x) {  // (0, 1]
  return (float)(x >> 8) * (1.0f / 16777216.0f) + (1.0f / 16777216.0f);
}

__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
  const float r = sqrtf(-2.0f * __logf(u01_open(a)));
  float s, c;
  __sincosf(6.28318530717958647692f * u01_open(b), &s, &c);
  return make_float2(r * c, r * s);
}

template <typename S>
__global__ void __launch_bounds__(kThreads) k_philox_noise(S* __restrict__ z, int64_t count, int64_t elems,
                                                           int64_t m0, const uint2* __restrict__ keys, int step) {
  const uint2 key = keys[step];
  // one thread per group of 4 consecutive elements of one sample
  const int64_t groups_per_sample = (elems + 3) / 4;
  const int64_t total = count * groups_per_sample;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ml = g / groups_per_sample;
    const int64_t q = g - ml * groups_per_sample;
    const uint64_t m = (uint64_t)(m0 + ml);
    const uint4 r = Philox::gen(make_uint4((uint32_t)q, (uint32_t)m, (uint32_t)(m >> 32), 0u), key);
    const float2 a = box_muller(r.x, r.y), b = box_muller(r.z, r.w);
    S* out = z + ml * elems + q * 4;
    if constexpr (std::is_same<S, float>::value) {
      if ((elems & 3) == 0) {
        *reinterpret_cast<float4*>(out) = make_float4(a.x, a.y, b.x, b.y);
        continue;
      }
    }
    const float v[4] = {a.x, a.y, b.x, b.y};
    const int64_t n = elems - q * 4 < 4 ? elems - q * 4 : 4;
    for (int j = 0; j < n; ++j) out[j] = (S)v[j];
  }
}

// ------------------------------------------------- K2+K3 rollout + fitness
template <typename S>
struct FitParams {
  const S* z;            // [M][T][R][du] this rank's samples (row m - m0)
  const S* base;         // [T][R][du]
  const S* msv;          // [T][R][du] mean_scale * variable
  S sd;                  // sampling std
  const S* starts;       // [R][dx]
  const S* goals;        // [R][pd]
  const S* inv_dstart;   // [R]   1/‖start-goal‖ (fp32) or ‖start-goal‖ (fp64: divide)
  const S* obs;          // [O][4]: cx, cy, cz, -(r+R_a)^2 (fp32: nudged up) / (r+R_a)^2 (fp64)
  int n_obs;
  S lower[3], upper[3];
  S dt, half_dt, dt6;
  S neg_margin_sq;       // fp32: -(nextafter((2R_a+eps)^2)), fp64: (2R_a+eps)^2
  double w_t, w_o, w_e;  // safety, obstacle, effort weights
  int R, Rp, T, TC, spc;
  int64_t M;             // samples in this launch
  int64_t m_global0;     // global index of row 0 (error keys)
  int step_key;          // (N - i) for the error key
  double* reward;        // [M]
  int* counts;           // [M][2] conflict / obstacle robot-steps, or null
  S* states_out;         // [M][T+1][R][dx] or null (parity)
  S* controls_out;       // [M][T+1][R][du] or null (parity)
  unsigned long long* err;  // min error key
};

__device__ __forceinline__ uint64_t pack2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ uint64_t fadd2_b(float a, uint64_t b) {  // (a,a) + b
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pack2(a, a)), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t ffma2_sq(uint64_t a, uint64_t c) {  // a*a + c
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(d) : "l"(a), "l"(c));
  return d;
}
__device__ __forceinline__ uint32_t lo32(uint64_t v) { return (uint32_t)v; }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return (uint32_t)(v >> 32); }

// Pair test, fp32 throughput form.  t = dx² + dy² [+ dz²] − m²↑ evaluated as
// fma(dx,dx, fma(dy,dy, −m²↑)); its sign bit is set iff the pair is within the
// margin (m²↑ = next float above m², so d² == m² counts, matching `<=`).  Two
// pairs per packed f32x2 instruction (FADD2/FFMA2).
template <int PD>
__device__ __forceinline__ uint64_t pair2_f32(float nxa, float nya, float nza, uint64_t xb, uint64_t yb,
                                              uint64_t zb, uint64_t nm2) {
  const uint64_t dx = fadd2_b(nxa, xb);
  const uint64_t dy = fadd2_b(nya, yb);
  uint64_t t;
  if constexpr (PD == 3) {
    const uint64_t dz = fadd2_b(nza, zb);
    t = ffma2_sq(dz, nm2);
    t = ffma2_sq(dy, t);
  } else {
    t = ffma2_sq(dy, nm2);
  }
  return ffma2_sq(dx, t);
}

template <int PD>
__device__ __forceinline__ uint32_t pair1_f32(float xa, float ya, float za, float xb, float yb, float zb, float nm2) {
  const float dx = xb - xa, dy = yb - ya;
  float t;
  if constexpr (PD == 3) {
    const float dz = zb - za;
    t = fmaf(dy, dy, fmaf(dz, dz, nm2));
  } else {
    t = fmaf(dy, dy, nm2);
  }
  return __float_as_uint(fmaf(dx, dx, t));
}

// Pair test, fp64 parity form: exactly reward.cpp:100-106 (sequential squared
// distance, `<=`), returning an all-ones word on a hit.
template <int PD>
__device__ __forceinline__ uint32_t pair1_f64(double xa, double ya, double za, double xb, double yb, double zb,
                                              double m2) {
  double s = 0.0;
  double d = __dadd_rn(xa, -xb);
  s = __dadd_rn(s, __dmul_rn(d, d));
  d = __dadd_rn(ya, -yb);
  s = __dadd_rn(s, __dmul_rn(d, d));
  if constexpr (PD == 3) {
    d = __dadd_rn(za, -zb);
    s = __dadd_rn(s, __dmul_rn(d, d));
  }
  return s <= m2 ? 0xffffffffu : 0u;
}

// Shared-memory position tile: pos[s][k][tc] per coordinate, row stride TC+1
// (odd → conflict-free both for the robot-major writes of the rollout phase
// and the time-major reads of the fitness phase).
template <typename S, int PD>
struct PosSmem {
  S* base;
  int Rp, TC, spc;
  __device__ __forceinline__ S* at(int c, int s, int k, int tc) const {
    return base + (((size_t)c * spc + s) * Rp + k) * (TC + 1) + tc;
  }
};

// Tile of TB robots × one (sample, t) item, held in registers.
template <typename S, int PD, int TB>
struct Tile {
  S x[TB], y[TB], z[PD == 3 ? TB : 1];
  __device__ __forceinline__ void load(const PosSmem<S, PD>& ps, int s, int k0, int tc) {
#pragma unroll
    for (int j = 0; j < TB; ++j) {
      x[j] = *ps.at(0, s, k0 + j, tc);
      y[j] = *ps.at(1, s, k0 + j, tc);
      if constexpr (PD == 3) z[j] = *ps.at(2, s, k0 + j, tc);
    }
  }
};

// Off-diagonal tile pair A×B: TB² pair tests; fa/fb collect sign-bit flags.
template <int PD, int TB>
__device__ __forceinline__ void tile_pairs_f32(const Tile<float, PD, TB>& A, const Tile<float, PD, TB>& B, float nm2,
                                               uint32_t* fa, uint32_t* fb) {
  uint64_t xb[TB / 2], yb[TB / 2], zb[TB / 2];
#pragma unroll
  for (int j = 0; j < TB / 2; ++j) {
    xb[j] = pack2(B.x[2 * j], B.x[2 * j + 1]);
    yb[j] = pack2(B.y[2 * j], B.y[2 * j + 1]);
    if constexpr (PD == 3) zb[j] = pack2(B.z[2 * j], B.z[2 * j + 1]); else zb[j] = 0;
  }
  const uint64_t nm2p = pack2(nm2, nm2);
#pragma unroll
  for (int i = 0; i < TB; i += 2) {
    const float nx0 = -A.x[i], ny0 = -A.y[i], nz0 = PD == 3 ? -A.z[i] : 0.f;
    const float nx1 = -A.x[i + 1], ny1 = -A.y[i + 1], nz1 = PD == 3 ? -A.z[i + 1] : 0.f;
#pragma unroll
    for (int j = 0; j < TB / 2; ++j) {
      const uint64_t t0 = pair2_f32<PD>(nx0, ny0, nz0, xb[j], yb[j], zb[j], nm2p);
      const uint64_t t1 = pair2_f32<PD>(nx1, ny1, nz1, xb[j], yb[j], zb[j], nm2p);
      fa[i] |= lo32(t0) | hi32(t0);
      fa[i + 1] |= lo32(t1) | hi32(t1);
      fb[2 * j] |= lo32(t0) | lo32(t1);
      fb[2 * j + 1] |= hi32(t0) | hi32(t1);
    }
  }
}

// Diagonal tile A×A: the TB(TB−1)/2 pairs inside the tile.
template <int PD, int TB>
__device__ __forceinline__ void tile_self_f32(const Tile<float, PD, TB>& A, float nm2, uint32_t* fa) {
  if constexpr (TB >= 4) {
    // 2x2 blocks above the diagonal, packed two at a time
    const uint64_t nm2p = pack2(nm2, nm2);
#pragma unroll
    for (int i = 0; i < TB; i += 2) {
      const float nx0 = -A.x[i], ny0 = -A.y[i], nz0 = PD == 3 ? -A.z[i] : 0.f;
      const float nx1 = -A.x[i + 1], ny1 = -A.y[i + 1], nz1 = PD == 3 ? -A.z[i + 1] : 0.f;
#pragma unroll
      for (int j = i + 2; j < TB; j += 2) {
        const uint64_t xb = pack2(A.x[j], A.x[j + 1]), yb = pack2(A.y[j], A.y[j + 1]);
        const uint64_t zb = PD == 3 ? pack2(A.z[j], A.z[j + 1]) : 0ull;
        const uint64_t t0 = pair2_f32<PD>(nx0, ny0, nz0, xb, yb, zb, nm2p);
        const uint64_t t1 = pair2_f32<PD>(nx1, ny1, nz1, xb, yb, zb, nm2p);
        fa[i] |= lo32(t0) | hi32(t0);
        fa[i + 1] |= lo32(t1) | hi32(t1);
        fa[j] |= lo32(t0) | lo32(t1);
        fa[j + 1] |= hi32(t0) | hi32(t1);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < TB; i += 2) {  // the pairs (i, i+1) on the diagonal
    const uint32_t t = pair1_f32<PD>(A.x[i], A.y[i], PD == 3 ? A.z[i] : 0.f, A.x[i + 1], A.y[i + 1],
                                     PD == 3 ? A.z[i + 1] : 0.f, nm2);
    fa[i] |= t;
    fa[i + 1] |= t;
  }
}

template <int PD, int TB>
__device__ __forceinline__ void tile_pairs_f64(const Tile<double, PD, TB>& A, const Tile<double, PD, TB>& B, double m2,
                                               uint32_t* fa, uint32_t* fb) {
#pragma unroll
  for (int i = 0; i < TB; ++i) {
#pragma unroll
    for (int j = 0; j < TB; ++j) {
      const uint32_t t = pair1_f64<PD>(A.x[i], A.y[i], PD == 3 ? A.z[i] : 0.0, B.x[j], B.y[j],
                                       PD == 3 ? B.z[j] : 0.0, m2);
      fa[i] |= t;
      fb[j] |= t;
    }
  }
}

template <int PD, int TB>
__device__ __forceinline__ void tile_self_f64(const Tile<double, PD, TB>& A, double m2, uint32_t* fa) {
#pragma unroll
  for (int i = 0; i < TB; ++i) {
#pragma unroll
    for (int j = i + 1; j < TB; ++j) {
      const uint32_t t = pair1_f64<PD>(A.x[i], A.y[i], PD == 3 ? A.z[i] : 0.0, A.x[j], A.y[j],
                                       PD == 3 ? A.z[j] : 0.0, m2);
      fa[i] |= t;
      fa[j] |= t;
    }
  }
}

template <int TB>
__device__ __forceinline__ uint32_t sign_mask(const uint32_t* f) {
  uint32_t m = 0;
#pragma unroll
  for (int j = TB - 1; j >= 0; --j) m = __funnelshift_l(f[j], m, 1);  // m = (m << 1) | sign(f[j])
  return m;
}

// Fused K2+K3.  CTA = `spc` samples; time is processed in chunks of TC steps:
//   phase A (thread = (sample, robot)): roll TC steps forward in registers,
//            writing positions to shared memory;
//   phase B (thread = (sample, t) items): goal + obstacle terms and all
//            unordered robot pairs of that time step from shared memory.
// Reward per sample = (Σ goal − w_t·#conflict − w_o·#obstacle − w_e·effort)/(R·T),
// reduced in a fixed order (deterministic; reward.cpp:67-130 up to rounding).
template <typename S, int KIND, int TB, int MAXW>
__global__ void __launch_bounds__(kThreads, 1) k_rollout_fitness(const FitParams<S> p) {
  constexpr int DX = ModelDims<KIND>::DX, DU = ModelDims<KIND>::DU, PD = ModelDims<KIND>::PD;
  constexpr bool F32 = std::is_same<S, float>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int R = p.R, Rp = p.Rp, TC = p.TC, spc = p.spc, T = p.T;
  const int nthreads = spc * Rp;

  // shared: positions | goals | inv_dstart | obstacles | reduction scratch
  PosSmem<S, PD> ps{reinterpret_cast<S*>(smem_raw), Rp, TC, spc};
  S* sgoal = ps.base + (size_t)PD * spc * Rp * (TC + 1);
  S* sinv = sgoal + (size_t)Rp * PD;
  S* sobs = sinv + Rp;
  double* sred = reinterpret_cast<double*>(sobs + (size_t)4 * p.n_obs + 2);  // 8-byte aligned below
  sred = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sred) + 15) & ~uintptr_t(15));
  double* seff = sred + kThreads;
  int* scnt = reinterpret_cast<int*>(seff + kThreads);

  for (int j = tid; j < Rp * PD; j += blockDim.x) sgoal[j] = j < R * PD ? p.goals[j] : S(0);
  for (int j = tid; j < Rp; j += blockDim.x) sinv[j] = j < R ? p.inv_dstart[j] : S(1);
  for (int j = tid; j < 4 * p.n_obs; j += blockDim.x) sobs[j] = p.obs[j];

  // ---- phase-A identity
  const int sA = tid / Rp, kA = tid % Rp;
  const int64_t mA = (int64_t)blockIdx.x * spc + sA;
  const bool liveA = tid < nthreads && mA < p.M;
  const bool robotA = liveA && kA < R;
  S x[DX];
#pragma unroll
  for (int j = 0; j < DX; ++j) x[j] = robotA ? p.starts[kA * DX + j] : S(0);
  double effort = 0.0;
  const S* zrow = p.z + (liveA ? mA : 0) * (int64_t)T * R * DU;
  bool bad = false;
  if (robotA && p.states_out) {
    S* so = p.states_out + mA * (int64_t)(T + 1) * R * DX + (int64_t)kA * DX;
#pragma unroll
    for (int j = 0; j < DX; ++j) so[j] = x[j];
  }

  // ---- phase-B identity: items (s, tc), ipt per thread, all of one sample
  // TC >= Rp: TC = Rp*ipt items per sample, ipt consecutive items per thread;
  // TC <  Rp: one item per thread for the first spc*TC threads.
  const int NI = spc * TC;
  const int ipt = TC >= Rp ? TC / Rp : 1;
  const int item0 = TC >= Rp ? tid * ipt : tid;
  const int sB = item0 / TC;
  const int64_t mB = (int64_t)blockIdx.x * spc + sB;
  const bool liveB = item0 < NI && mB < p.M && tid < nthreads;
  double gsum = 0.0;
  int nconf = 0, nobs = 0;
  const int ntiles = Rp / TB;
  const uint32_t last_valid = (R % 32) == 0 ? 0xffffffffu : ((1u << (R % 32)) - 1u);

  __syncthreads();

  for (int t0 = 0; t0 < T; t0 += TC) {
    // ===== phase A: integrate TC steps
    if (liveA) {
      if (robotA) {
        for (int tc = 0; tc < TC; ++tc) {
          const int t = t0 + tc;
          if (t >= T) break;
          S u[DU];
          const int64_t e = ((int64_t)t * R + kA) * DU;
#pragma unroll
          for (int d = 0; d < DU; ++d) {
            // sample = mean_scale*var + std*z (denoiser.cpp:44-45); candidate = base + sample (:158-159)
            const S smp = xadd(__ldg(p.msv + e + d), xmul(p.sd, __ldg(zrow + e + d)));
            S v = xadd(__ldg(p.base + e + d), smp);
            v = (v < p.lower[d]) ? p.lower[d] : v;  // cwiseMax(lower)
            v = (p.upper[d] < v) ? p.upper[d] : v;  // cwiseMin(upper)
            u[d] = v;
            effort += (double)(v * v);
          }
          rk4<KIND>(x, u, p.dt, p.half_dt, p.dt6);
          bool fin = true;
#pragma unroll
          for (int j = 0; j < DX; ++j) fin = fin && isfinite(x[j]);
          if (!fin && !bad) {
            bad = true;
            const unsigned long long key = ((unsigned long long)p.step_key << 52) |
                                           ((unsigned long long)(p.m_global0 + mA) << 20) |
                                           ((unsigned long long)kA << 10) | (unsigned long long)(t + 1);
            atomicMin(p.err, key);
          }
          *ps.at(0, sA, kA, tc) = x[0];
          *ps.at(1, sA, kA, tc) = x[1];
          if constexpr (PD == 3) *ps.at(2, sA, kA, tc) = x[2];
          if (p.states_out) {
            S* so = p.states_out + (mA * (int64_t)(T + 1) + t + 1) * R * DX + (int64_t)kA * DX;
#pragma unroll
            for (int j = 0; j < DX; ++j) so[j] = x[j];
          }
          if (p.controls_out) {
            S* co = p.controls_out + (mA * (int64_t)(T + 1) + t) * R * DU + (int64_t)kA * DU;
#pragma unroll
            for (int d = 0; d < DU; ++d) co[d] = u[d];
          }
        }
      } else {
        // padding robots: parked far away at distinct points, never counted
        for (int tc = 0; tc < TC; ++tc) {
          *ps.at(0, sA, kA, tc) = S(1.0e6) + S(1.0e3) * S(kA);
          *ps.at(1, sA, kA, tc) = S(-1.0e6) - S(1.0e3) * S(kA);
          if constexpr (PD == 3) *ps.at(2, sA, kA, tc) = S(1.0e6);
        }
      }
    }
    __syncthreads();

    // ===== phase B: fitness of the TC time steps just integrated
    if (liveB) {
      for (int j = 0; j < ipt; ++j) {
        const int item = item0 + j;
        const int tc = item - sB * TC;
        if (t0 + tc >= T) break;
        uint32_t cm[MAXW];
#pragma unroll
        for (int w = 0; w < MAXW; ++w) cm[w] = 0;
        S gitem = S(0);
        for (int a = 0; a < ntiles; ++a) {
          Tile<S, PD, TB> A;
          A.load(ps, sB, a * TB, tc);
          uint32_t fa[TB];
#pragma unroll
          for (int q = 0; q < TB; ++q) fa[q] = 0;
          // goal + obstacle terms of tile A's robots (reward.cpp:92-97, :112-125)
          uint32_t om = 0;
#pragma unroll
          for (int q = 0; q < TB; ++q) {
            const int k = a * TB + q;
            if (k < R) {
              const S gx = xsub(A.x[q], sgoal[k * PD + 0]);
              const S gy = xsub(A.y[q], sgoal[k * PD + 1]);
              S g2 = xadd(xmul(gx, gx), xmul(gy, gy));
              if constexpr (PD == 3) {
                const S gz = xsub(A.z[q], sgoal[k * PD + 2]);
                g2 = xadd(g2, xmul(gz, gz));
              }
              if constexpr (F32) {
                gitem += 1.0f - xsqrt(g2) * sinv[k];
              } else {
                gitem = xadd(gitem, xsub(S(1), xsqrt(g2) / sinv[k]));
              }
              uint32_t of = 0;
              for (int o = 0; o < p.n_obs; ++o) {
                const S* ob = sobs + 4 * o;
                if constexpr (F32) {
                  of |= pair1_f32<PD>(A.x[q], A.y[q], PD == 3 ? A.z[q] : 0.f, ob[0], ob[1], ob[2], ob[3]);
                } else {
                  of |= pair1_f64<PD>(A.x[q], A.y[q], PD == 3 ? A.z[q] : 0.0, ob[0], ob[1], ob[2], ob[3]);
                }
              }
              om |= (of >> 31) << q;
            }
          }
          nobs += __popc(om);
          if constexpr (F32) tile_self_f32<PD, TB>(A, p.neg_margin_sq, fa);
          else tile_self_f64<PD, TB>(A, p.neg_margin_sq, fa);
          for (int b = a + 1; b < ntiles; ++b) {
            Tile<S, PD, TB> B;
            B.load(ps, sB, b * TB, tc);
            uint32_t fb[TB];
#pragma unroll
            for (int q = 0; q < TB; ++q) fb[q] = 0;
            if constexpr (F32) tile_pairs_f32<PD, TB>(A, B, p.neg_margin_sq, fa, fb);
            else tile_pairs_f64<PD, TB>(A, B, p.neg_margin_sq, fa, fb);
            const uint32_t mb = sign_mask<TB>(fb);
            const int wb = (b * TB) >> 5, sh = (b * TB) & 31;
#pragma unroll
            for (int w = 0; w < MAXW; ++w)
              if (w == wb) cm[w] |= mb << sh;
          }
          const uint32_t ma = sign_mask<TB>(fa);
          const int wa = (a * TB) >> 5, sha = (a * TB) & 31;
#pragma unroll
          for (int w = 0; w < MAXW; ++w)
            if (w == wa) cm[w] |= ma << sha;
        }
        int c = 0;
#pragma unroll
        for (int w = 0; w < MAXW; ++w) {
          const int k0 = w * 32;
          if (k0 < R) c += __popc(k0 + 32 <= R ? cm[w] : (cm[w] & last_valid));
        }
        nconf += c;
        gsum += (double)gitem;
      }
    }
    __syncthreads();
  }

  // ---- per-sample deterministic reduction (phase-B items, then effort)
  sred[tid] = liveB ? gsum : 0.0;
  seff[tid] = robotA ? effort : 0.0;
  scnt[2 * tid] = liveB ? nconf : 0;
  scnt[2 * tid + 1] = liveB ? nobs : 0;
  __syncthreads();
  if (liveB && item0 == sB * TC) {  // first phase-B thread of the sample
    const int nt = TC >= Rp ? Rp : TC;          // phase-B threads per sample
    const int first = TC >= Rp ? sB * Rp : sB * TC;
    double g = 0.0;
    long long nc = 0, no = 0;
    for (int q = 0; q < nt; ++q) {
      g += sred[first + q];
      nc += scnt[2 * (first + q)];
      no += scnt[2 * (first + q) + 1];
    }
    double value = g - p.w_t * (double)nc - p.w_o * (double)no;
    if (p.w_e != 0.0) {  // effort extension: w_e · Σ_{t,k} ‖u‖²
      double eff = 0.0;
      for (int k = 0; k < R; ++k) eff += seff[sB * Rp + k];
      value -= p.w_e * eff;
    }
    p.reward[mB] = value / ((double)R * (double)T);
    if (p.counts) {
      p.counts[2 * mB] = (int)nc;
      p.counts[2 * mB + 1] = (int)no;
    }
  }
}

// ------------------------------------------------------------ K4 weights
struct WeightParams {
  const double* reward;  // [M] all samples (global)
  int64_t M;
  double lambda;
  double* w64;           // [M]
  float* w32;            // [M]
  double* trace;         // [4]: step, best, mean, entropy
  int step;
  double* stats;         // [4] scratch: mean, std, max_scaled, sum
  unsigned long long* err;  // set on non-finite reward
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

// score_weights (denoiser.cpp:50-90) + trace (denoiser.cpp:172-179), one CTA.
// Each thread owns a contiguous slice, reductions are fixed-order.
template <int NT>
__global__ void __launch_bounds__(NT) k_score_weights(const WeightParams p) {
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
  if (std_dev < 1e-8) {
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
  // max of scaled values = scaled max (monotone), as denoiser.cpp:78-82
  const double max_scaled = (best - mean) / std_dev / p.lambda;
  double sum = 0.0;
  for (int64_t j = b; j < e; ++j) {
    const double w = exp((p.reward[j] - mean) / std_dev / p.lambda - max_scaled);
    p.w64[j] = w;
    sum += w;
  }
  sum = block_sum<NT>(sum, sh);
  double h = 0.0;
  for (int64_t j = b; j < e; ++j) {
    const double w = p.w64[j] / sum;
    p.w64[j] = w;
    p.w32[j] = (float)w;
    if (w > 0.0) h -= w * log(w);
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
// Partial of Σ_m w_m·sample_m over one chunk of CH samples (ascending m) for
// 4 consecutive elements per thread; sample_m = msv + sd·z_m (denoiser.cpp:44-45,
// mc_average :104-106).
template <typename S, typename W>
__global__ void __launch_bounds__(kThreads) k_wmean_partial(const S* __restrict__ z, const W* __restrict__ w,
                                                            const S* __restrict__ msv, S sd, int64_t M,
                                                            int64_t elems, int ch, S* __restrict__ partial) {
  const int64_t e0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int64_t c = blockIdx.y;
  const int64_t mb = c * ch, me = mb + ch < M ? mb + ch : M;
  if (e0 >= elems) return;
  const int n = elems - e0 < 4 ? (int)(elems - e0) : 4;
  S acc[4] = {S(0), S(0), S(0), S(0)};
  S mv[4] = {S(0), S(0), S(0), S(0)};
  for (int j = 0; j < n; ++j) mv[j] = msv[e0 + j];
  if constexpr (std::is_same<S, float>::value) {
    if (n == 4 && (elems & 3) == 0) {
      const float4* zp = reinterpret_cast<const float4*>(z + mb * elems + e0);
      const int64_t stride = elems / 4;
      int64_t m = mb;
#pragma unroll 4
      for (; m < me; ++m) {
        const float4 v = __ldcs(zp);
        zp += stride;
        const float wm = (float)__ldg(w + m);
        acc[0] = fmaf(wm, fmaf(sd, v.x, mv[0]), acc[0]);
        acc[1] = fmaf(wm, fmaf(sd, v.y, mv[1]), acc[1]);
        acc[2] = fmaf(wm, fmaf(sd, v.z, mv[2]), acc[2]);
        acc[3] = fmaf(wm, fmaf(sd, v.w, mv[3]), acc[3]);
      }
      *reinterpret_cast<float4*>(partial + c * elems + e0) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      return;
    }
  }
  for (int64_t m = mb; m < me; ++m) {
    const W wm = w[m];
    for (int j = 0; j < n; ++j) {
      const S smp = xadd(mv[j], xmul(sd, z[m * elems + e0 + j]));
      acc[j] = xadd(acc[j], xmul((S)wm, smp));
    }
  }
  for (int j = 0; j < n; ++j) partial[c * elems + e0 + j] = acc[j];
}

// Pairwise (binary-counter) sum of the chunk partials — a balanced binary tree
// when the chunk count is a power of two, so a rank owning an aligned block of
// chunks computes exactly one subtree: results are identical for any GPU count.
// Then var ← √ᾱ_{i−1}·avg (denoise_step, denoiser.cpp:110-117) and the next
// step's mean-scaled variable msv ← mean_scale_{i−1}·var.
template <typename S>
__global__ void __launch_bounds__(kThreads) k_wmean_tree(const S* __restrict__ partial, int64_t nchunks,
                                                         int64_t elems, double scale, double next_ms,
                                                         double* __restrict__ var, S* __restrict__ msv,
                                                         S* __restrict__ root_out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= elems) return;
  S stack[40];
  int64_t cnt = 0;
  int top = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    S v = partial[c * elems + e];
    // merge equal-size subtrees: number of merges = trailing ones of cnt
    int64_t k = cnt;
    while (k & 1) {
      v = xadd(stack[--top], v);
      k >>= 1;
    }
    stack[top++] = v;
    ++cnt;
  }
  S total = stack[--top];
  while (top > 0) total = xadd(stack[--top], total);
  if (root_out) {
    root_out[e] = total;
    return;
  }
  const double nv = scale * (double)total;
  var[e] = nv;
  msv[e] = (S)(next_ms * nv);
}

}  // namespace d4k
