// k23.cuh — K2+K3: fused rollout + team fitness, one kernel.
//
// CTA = `spc` samples × Rp robot lanes (blockDim = spc·Rp ≤ 256, usually 128,
// several CTAs resident per SM).  Time advances in chunks of TC steps:
//
//  phase A  thread = (sample, robot): TC RK4 steps in registers
//           (dynamics.cpp:65-87 / dynamics.hpp:123-130), controls formed as
//           clamp(base + mean_scale·var + std·z) (denoiser.cpp:44-45,158-159)
//           with an 8-deep register prefetch ring on the HBM noise stream;
//           positions → shared memory, one robot-contiguous row per (sample, t).
//  phase B  thread = (sample, t) item: goal + obstacle terms for every robot
//           and all R(R−1)/2 unordered pair tests of that time step
//           (reward.cpp:88-127).  fp32: tiles of TB robots, A rows streamed
//           against a register-resident B tile, two pair tests per packed
//           FADD2/FFMA2 instruction; a conflict is the sign bit of
//           d² − m²↑, OR-ed into per-robot flags (3 issue slots per pair).
//           fp64 (parity): the reference's own loops, exact `<=` tests.
//
// reward[m] = (Σ goal − w_t·#conflict robot-steps − w_o·#obstacle robot-steps
//              − w_e·Σ‖u‖²) / (R·T), reduced in a fixed order.
#pragma once

#include "d4orm_common.cuh"

namespace d4k {

constexpr int kFitMaxThreads = 128;
constexpr int kObsBuckets = 64;  // x-buckets of the obstacle culling table
#ifndef D4K_KPF
#define D4K_KPF 8
#endif
constexpr int kPF = D4K_KPF;  // rollout block depth (time steps): Philox draws in flight per thread
// The fused-noise rollout's block depth per kind: 16 steps for the two-control
// kinds (C5 K2+K3 19.28 → 18.97 ms, C2 0.110 → 0.108 ms), 8 for du = 3 (16
// measured +18 µs on C4: 48 normals in flight spill)
template <int KIND>
constexpr int kPFf = ModelDims<KIND>::DU == 3 ? kPF : 2 * kPF;
#ifndef D4K_MINB16
#define D4K_MINB16 3  // resident CTAs per SM the 16-robot-tile kernels are register-capped for
#endif
#ifndef D4K_MINB8
#define D4K_MINB8 5   // ... and the small-tile (R <= 16) kernels
#endif

template <typename S>
struct FitParams {
  const S* z;            // [M][T][R][du] (row 0 = global sample m_global0)
  const S* base;         // [T][R][du]   (fp64 path)
  const S* msv;          // [T][R][du]   mean_scale·variable (fp64 path)
  const S* bm;           // [T][R][du]   base + msv (fp32 path)
  S sd;                  // sampling std of this step
  const S* sdv;          // CEM: per-element std [T][R][du] (replaces sd), else null
  const S* starts;       // [R][dx]
  const S* goals;        // [R][pd]
  const S* inv_dstart;   // [R]  fp32: 1/‖start−goal‖; fp64: ‖start−goal‖ (divide)
  const S* obs;          // [O+1][4] fp32: −2c, |c|²−(r+R_a)²↑ (row O: never-hit pad) | fp64: c, (r+R_a)²
  const S* obs_cull;     // fp32: obstacle x-bucket table (kObsBuckets, see upload_problem), obstacles sorted by left end
  S cull_margin;         // fp32: separation (m) beyond which a pair cannot be in conflict, with rounding slack
  int cull;              // fp32: rank robots by x per chunk and cull tile pairs / obstacles (≥ 3 tiles)
  const float* obs_pl;   // fp32 pair-list path: [O][8] (cx, cy, −L²↑, 0, box lo.x, lo.y, hi.x, hi.y)
  int z_keep;            // fused noise: z stores with an L2 evict_last hint (1: z fits in L2, K5a reads
                         // it there) or evict_first (0: z ≫ L2, stream it out); 2: no z stores at all
                         // (K5a regenerates the normals, k_wmean_regen)
  int n_obs;
  S lower[3], upper[3];
  S dt, half_dt, dt6;
  S margin_sq;           // fp32: −(2R_a+ε)²↑ ; fp64: (2R_a+ε)²
  double w_t, w_o, w_e;
  int R, Rp, T, TC, spc;
  int64_t M;             // samples in this launch
  int64_t m_global0;     // global index of row 0 (error keys)
  int step_key;          // N − i (error key)
  double* reward;        // [M]
  int* counts;           // [M][2] or null
  S* states_out;         // [M][T+1][R][dx] or null
  S* controls_out;       // [M][T+1][R][du] or null
  unsigned long long* err;
  // fused-noise mode (NOISE >= 1; 2 = with sdv): Philox key table, this step, z written for K5
  const uint2* keys;
  int step;
  S* z_store;            // [M][T][R][du]
};

template <typename S>
struct FitSmem {
  S* pos;     // [PD][spc][TC][RS]; fp32: robot k's column is its rank in the chunk's x order
  S* goal;    // fp64: [PD][Rp] goal
  S* inv;     // fp64: [2·Rp] (‖s−g‖, valid)
  S* obs;     // [O+1][4]
  S* ocl;     // fp32: obstacle x-bucket table (FitParams::obs_cull): {x0, 1/w, -, -} + [kObsBuckets][2] int
  int* key;   // fp32: [spc][Rp] chunk sort keys (x order)
  float* bb;  // fp32: [2·ntiles][nthreads] per-item tile x-extent (lo, hi)
  float4* pbox;  // fp32 pair-list path: [spc][TC/32][Rp] robot window boxes (lo.x, lo.y, hi.x, hi.y)
  float* opl;    // fp32 pair-list path: FitParams::obs_pl
  // the final reduction arrays alias `pos` (dead after the last chunk)
  double* red;   // [nthreads]
  double* eff;   // [nthreads]
  int* cnt;      // [2·nthreads]
  int RS, TC, spc, Rp, nthreads, npd = 3;
  __device__ __forceinline__ S* row(int c, int s, int tc) const {
    D4K_CHECK(c >= 0 && c < npd && s >= 0 && s < spc && tc >= 0 && tc < TC);
    return pos + ((size_t)(c * spc + s) * TC + tc) * RS;
  }
};

template <typename S>
__host__ __device__ inline size_t fit_smem_bytes(int PD, int spc, int TC, int Rp, int nobs, int nthreads, int TB,
                                                 bool pl = false) {
  const int RS = Rp + 2;
  size_t pos = (size_t)PD * spc * TC * RS * sizeof(S);
  const size_t red = 2 * (size_t)nthreads * sizeof(double) + 2 * (size_t)nthreads * sizeof(int);
  size_t b = ((pos > red ? pos : red) + 15) & ~size_t(15);
  b += (size_t)4 * (nobs + 1) * sizeof(S);
  if (sizeof(S) == 8) {
    b += (size_t)PD * Rp * sizeof(S) + 2 * (size_t)Rp * sizeof(S);
  } else if (pl) {  // key, robot window boxes, obstacle table
    b += (size_t)spc * Rp * sizeof(int);
    b = (b + 15) & ~size_t(15);
    b += (size_t)spc * (TC / 32) * Rp * sizeof(float4) + (size_t)8 * nobs * sizeof(float);
  } else {
    b += (size_t)(4 + 2 * kObsBuckets) * sizeof(float) + (size_t)spc * Rp * sizeof(int) +
         (size_t)2 * (Rp / TB) * nthreads * sizeof(float);
  }
  return (b + 15) & ~size_t(15);
}

// ---------------------------------------------------------------- fp32 tiles
template <int PD>
__device__ __forceinline__ uint64_t pair2_f32(float nxa, float nya, float nza, uint64_t xb, uint64_t yb, uint64_t zb,
                                              uint64_t nm2) {
  const uint64_t dx = fadd2_b(nxa, xb);
  const uint64_t dy = fadd2_b(nya, yb);
  uint64_t t;
  if constexpr (PD == 3) {
    t = ffma2_sq(fadd2_b(nza, zb), nm2);
    t = ffma2_sq(dy, t);
  } else {
    t = ffma2_sq(dy, nm2);
  }
  return ffma2_sq(dx, t);
}

template <int PD>
__device__ __forceinline__ uint32_t pair1_f32(float xa, float ya, float za, float xb, float yb, float zb, float nm2) {
  const float dx = xb - xa, dy = yb - ya;
  float t = fmaf(dy, dy, nm2);
  if constexpr (PD == 3) t = fmaf(zb - za, zb - za, t);
  return __float_as_uint(fmaf(dx, dx, t));
}

template <int TB>
__device__ __forceinline__ uint32_t sign_mask(const uint32_t* f) {
  uint32_t m = 0;
#pragma unroll
  for (int j = TB - 1; j >= 0; --j) m = __funnelshift_l(f[j], m, 1);  // (m << 1) | sign(f[j])
  return m;
}

template <int PD, int TB>
struct PackedTile {
  uint64_t x[TB / 2], y[TB / 2], z[PD == 3 ? TB / 2 : 1];
  __device__ __forceinline__ void load(const float* X, const float* Y, const float* Z, int k0) {
#pragma unroll
    for (int j = 0; j < TB / 2; ++j) {
      x[j] = *reinterpret_cast<const uint64_t*>(X + k0 + 2 * j);
      y[j] = *reinterpret_cast<const uint64_t*>(Y + k0 + 2 * j);
      if constexpr (PD == 3) z[j] = *reinterpret_cast<const uint64_t*>(Z + k0 + 2 * j);
    }
  }
};

// Column side of a tile-pair task: robots [k0, k0+TB) as −2·p and |p|²−m²↑,
// register-resident; the row side is streamed from shared memory.
template <int PD, int TB>
struct ColTile {
  uint64_t x[TB / 2], y[TB / 2], z[PD == 3 ? TB / 2 : 1], n[TB / 2];
  __device__ __forceinline__ void load(const float* X, const float* Y, const float* Z, int k0, float m2u) {
    const uint64_t m2n = pack2(-2.0f, -2.0f);
#pragma unroll
    for (int j = 0; j < TB / 2; ++j) {
      const uint64_t bx = *reinterpret_cast<const uint64_t*>(X + k0 + 2 * j);
      const uint64_t by = *reinterpret_cast<const uint64_t*>(Y + k0 + 2 * j);
      uint64_t n2 = fmul2(bx, bx);
      n2 = ffma2_sq(by, n2);
      if constexpr (PD == 3) {
        const uint64_t bz = *reinterpret_cast<const uint64_t*>(Z + k0 + 2 * j);
        n2 = ffma2_sq(bz, n2);
        z[j] = fmul2(bz, m2n);
      }
      x[j] = fmul2(bx, m2n);
      y[j] = fmul2(by, m2n);
      n[j] = fadd2_b(-m2u, n2);
    }
  }
};

// Expanded-form test of two row robots (scalars) against column pair j:
// t = |a|² + (|b|² − m²↑) − 2·a·b, sign bit set ⟺ within the margin.
template <int PD, int TB>
__device__ __forceinline__ void row_pair_vs_col(const ColTile<PD, TB>& C, int j, float2 ax, float2 ay, float2 az,
                                                float n0, float n1, uint64_t& t0, uint64_t& t1) {
  t0 = fadd2_b(n0, C.n[j]);
  t1 = fadd2_b(n1, C.n[j]);
  t0 = ffma2(pack2(ax.x, ax.x), C.x[j], t0);
  t1 = ffma2(pack2(ax.y, ax.y), C.x[j], t1);
  t0 = ffma2(pack2(ay.x, ay.x), C.y[j], t0);
  t1 = ffma2(pack2(ay.y, ay.y), C.y[j], t1);
  if constexpr (PD == 3) {
    t0 = ffma2(pack2(az.x, az.x), C.z[j], t0);
    t1 = ffma2(pack2(az.y, az.y), C.z[j], t1);
  }
}

template <int MAXW>
__device__ __forceinline__ void or_mask(uint32_t* cm, int k0, uint32_t bits) {
  const int w = k0 >> 5, sh = k0 & 31;
#pragma unroll
  for (int q = 0; q < MAXW; ++q)
    if (q == w) cm[q] |= bits << sh;
}

// Obstacle index range [ob, oe) that can meet the x-range [xlo, xhi]: two
// lookups in the host-built bucket table (obstacles sorted by the left end of
// their culling interval; each entry keeps one bucket of slack on both sides,
// so float rounding of the bucket index cannot drop an obstacle).
__device__ __forceinline__ void obstacle_range(const float* ocl, int n_obs, float xlo, float xhi, int* ob, int* oe) {
  const int* tab = reinterpret_cast<const int*>(ocl + 4);
  const float fl = (xlo - ocl[0]) * ocl[1], fh = (xhi - ocl[0]) * ocl[1];
  *ob = !(fl >= 1.0f) ? 0 : tab[2 * min((int)fl, kObsBuckets - 1)];
  *oe = !(fh < (float)(kObsBuckets - 1)) ? n_obs : tab[2 * max((int)fh, 0) + 1];
}

// One (sample, t) item in fp32, shared by Q threads: thread q takes the tasks
// of the (a ≤ b) tile-pair enumeration with index ≡ q (mod Q); diagonal tasks
// also carry tile a's obstacle terms.  Adds obstacle robot-steps to *nobs and
// OR-s conflict flags into cm (merged across the Q lanes and counted by the
// caller).  The goal terms are accumulated by the rollout (phase A).
//
// Distance tests use the expanded form  t = |a|² + (|b|² − m²↑) − 2·a·b, three
// packed FP instructions per two tests (FADD2 of the norms, then one FFMA2 per
// coordinate against the −2-scaled partner) instead of four for the direct
// form; the sign bit of t is the (fp32-approximate) `<=` decision of
// reward.cpp:106,120.  Obstacles: t = |p|² + (|c|² − L²↑) − 2·p·c, with the
// obstacle's −2c and |c|²−L²↑ precomputed.
//
// Culling (exact): robot columns are in x order (ranked at the chunk start),
// so tiles are x-strips.  A tile pair whose x-extents are more than
// cull_margin apart cannot hold a conflict; it is skipped when that holds for
// every item of the warp.  Likewise only obstacles whose x-interval can meet
// the strip's extent (warp union) are tested.  The slack in cull_margin and
// in the obstacle intervals exceeds the expanded form's rounding error, so the
// skipped tests are ones that would have come out negative anyway.
template <int PD, int TB, int MAXW, bool CULL>
__device__ __forceinline__ void item_f32(const FitSmem<float>& sm, int s, int tc, int R, int n_obs, float m2u,
                                         float cmg, int q, int Q, float* bbp, uint32_t* cm, int* nobs) {
  constexpr bool cull = CULL;
  const float* X = sm.row(0, s, tc);
  const float* Y = sm.row(1, s, tc);
  const float* Z = PD == 3 ? sm.row(2, s, tc) : X;
  const int ntiles = sm.Rp / TB;
  const int bbs = sm.nthreads;
  // Lanes of one item run the same task kind in lockstep (no divergence):
  // diagonal tiles a ≡ q (mod Q), then off-diagonal task k ≡ q (mod Q).
  for (int a = q; a < ntiles; a += Q) {
    {
      // ---------------- diagonal task (a, a): extent + obstacles + inner pairs
      {
        PackedTile<PD, TB> A;
        A.load(X, Y, Z, a * TB);
        uint64_t NA[TB / 2];
        // x-extent of each half tile (robot pairs [h·JH, (h+1)·JH)) and of the tile
#ifndef D4K_OBS_PARTS
#define D4K_OBS_PARTS 2
#endif
        // obstacle culling parts per tile: NPART groups of JH robot pairs
        constexpr int NPART = (TB / 2) >= D4K_OBS_PARTS ? D4K_OBS_PARTS : (TB / 2);
        constexpr int JH = (TB / 2) / NPART;
        float hlo[NPART], hhi[NPART];
#pragma unroll
        for (int h = 0; h < NPART; ++h) {
          hlo[h] = INFINITY;
          hhi[h] = -INFINITY;
        }
#pragma unroll
        for (int j = 0; j < TB / 2; ++j) {
          uint64_t n2 = fmul2(A.x[j], A.x[j]);
          n2 = ffma2_sq(A.y[j], n2);
          if constexpr (PD == 3) n2 = ffma2_sq(A.z[j], n2);
          NA[j] = n2;
          const int h = j / JH;
          hlo[h] = fminf(hlo[h], fminf(lo_f(A.x[j]), hi_f(A.x[j])));
          hhi[h] = fmaxf(hhi[h], fmaxf(lo_f(A.x[j]), hi_f(A.x[j])));
        }
        float xlo = hlo[0], xhi = hhi[0];
#pragma unroll
        for (int h = 1; h < NPART; ++h) {
          xlo = fminf(xlo, hlo[h]);
          xhi = fmaxf(xhi, hhi[h]);
        }
        if (cull) {
          bbp[(2 * a) * bbs] = xlo;
          bbp[(2 * a + 1) * bbs] = xhi;
        }
        // obstacle terms (reward.cpp:112-125).  Culling: per half tile, only the
        // obstacles whose x-interval meets the half's extent (warp union).
        uint32_t olo[TB / 2], ohi[TB / 2];
#pragma unroll
        for (int j = 0; j < TB / 2; ++j) olo[j] = ohi[j] = 0;
        auto obstacle_block = [&](int ob, int oe, auto j0_tag, auto jn_tag) {
          constexpr int J0 = decltype(j0_tag)::value, JN = decltype(jn_tag)::value;
          for (int o = ob; o < oe; o += 2) {
            const float4 b0 = *reinterpret_cast<const float4*>(sm.obs + 4 * o);      // −2c, |c|²−L²↑
            const float4 b1 = *reinterpret_cast<const float4*>(sm.obs + 4 * o + 4);  // row O: never hits
#pragma unroll
            for (int j = J0; j < JN; ++j) {
              uint64_t t0 = fadd2_b(b0.w, NA[j]);
              uint64_t t1 = fadd2_b(b1.w, NA[j]);
              t0 = ffma2(A.x[j], pack2(b0.x, b0.x), t0);
              t1 = ffma2(A.x[j], pack2(b1.x, b1.x), t1);
              t0 = ffma2(A.y[j], pack2(b0.y, b0.y), t0);
              t1 = ffma2(A.y[j], pack2(b1.y, b1.y), t1);
              if constexpr (PD == 3) {
                t0 = ffma2(A.z[j], pack2(b0.z, b0.z), t0);
                t1 = ffma2(A.z[j], pack2(b1.z, b1.z), t1);
              }
              olo[j] |= lo32(t0) | lo32(t1);
              ohi[j] |= hi32(t0) | hi32(t1);
            }
          }
        };
        if constexpr (CULL) {
          if (n_obs > 0) {
            const unsigned am = __activemask();
            int ob[NPART], oe[NPART];
#pragma unroll
            for (int h = 0; h < NPART; ++h) {
              obstacle_range(sm.ocl, n_obs, hlo[h], hhi[h], &ob[h], &oe[h]);
              ob[h] = __reduce_min_sync(am, ob[h]);
              oe[h] = __reduce_max_sync(am, oe[h]);
            }
            obstacle_block(ob[0], oe[0], std::integral_constant<int, 0>{}, std::integral_constant<int, JH>{});
            if constexpr (NPART > 1)
              obstacle_block(ob[1], oe[1], std::integral_constant<int, JH>{}, std::integral_constant<int, 2 * JH>{});
            if constexpr (NPART > 2)
              obstacle_block(ob[2], oe[2], std::integral_constant<int, 2 * JH>{}, std::integral_constant<int, 3 * JH>{});
            if constexpr (NPART > 3)
              obstacle_block(ob[3], oe[3], std::integral_constant<int, 3 * JH>{}, std::integral_constant<int, 4 * JH>{});
          }
        } else {
          obstacle_block(0, n_obs, std::integral_constant<int, 0>{}, std::integral_constant<int, TB / 2>{});
        }
        uint32_t om = 0;  // bit 2j / 2j+1: robot pair j's obstacle hits (one funnel shift per bit)
#pragma unroll
        for (int j = TB / 2 - 1; j >= 0; --j) {
          om = __funnelshift_l(ohi[j], om, 1);
          om = __funnelshift_l(olo[j], om, 1);
        }
        const int kv = R - a * TB;  // valid robots in this tile
        *nobs += __popc(kv >= 32 ? om : (om & ((1u << (kv > 0 ? kv : 0)) - 1u)));
        // pairs inside tile a, from the tile already in registers: columns as
        // −2·p and |p|²−m²↑, rows as scalars
        ColTile<PD, TB> C;
        const uint64_t m2n = pack2(-2.0f, -2.0f);
#pragma unroll
        for (int j = 0; j < TB / 2; ++j) {
          C.x[j] = fmul2(A.x[j], m2n);
          C.y[j] = fmul2(A.y[j], m2n);
          if constexpr (PD == 3) C.z[j] = fmul2(A.z[j], m2n);
          C.n[j] = fadd2_b(-m2u, NA[j]);
        }
        uint32_t f[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) f[k] = 0;
#pragma unroll
        for (int i = 0; i < TB / 2; ++i) {
          const float2 ax = make_float2(lo_f(A.x[i]), hi_f(A.x[i]));
          const float2 ay = make_float2(lo_f(A.y[i]), hi_f(A.y[i]));
          const float2 az = PD == 3 ? make_float2(lo_f(A.z[i]), hi_f(A.z[i])) : make_float2(0.f, 0.f);
          const float n0 = lo_f(NA[i]), n1 = hi_f(NA[i]);
#pragma unroll
          for (int j = i + 1; j < TB / 2; ++j) {
            uint64_t t0, t1;
            row_pair_vs_col<PD, TB>(C, j, ax, ay, az, n0, n1, t0, t1);
            f[2 * i] |= lo32(t0) | hi32(t0);
            f[2 * i + 1] |= lo32(t1) | hi32(t1);
            f[2 * j] |= lo32(t0) | lo32(t1);
            f[2 * j + 1] |= hi32(t0) | hi32(t1);
          }
          // the pair (2i, 2i+1) itself
          float t = fmaf(-2.0f * ax.x, ax.y, n0 + (n1 - m2u));
          t = fmaf(-2.0f * ay.x, ay.y, t);
          if constexpr (PD == 3) t = fmaf(-2.0f * az.x, az.y, t);
          f[2 * i] |= __float_as_uint(t);
          f[2 * i + 1] |= __float_as_uint(t);
        }
        or_mask<MAXW>(cm, a * TB, sign_mask<TB>(f));
      }
    }
  }
  const int n_off = ntiles * (ntiles - 1) / 2;
  if (cull && Q > 1 && n_off > 0) __syncwarp(__activemask());  // tile extents written by the item's other lanes
  int k = 0;
  for (int a = 0; a < ntiles - 1; ++a)
  for (int b = a + 1; b < ntiles; ++b, ++k) {
    // ---------------- off-diagonal task k = (a, b), a < b; this lane's when k ≡ q (mod Q)
    if (Q > 1 && k % Q != q) continue;
    if (cull) {
      const bool apart = bbp[(2 * a + 1) * bbs] + cmg < bbp[(2 * b) * bbs] ||
                         bbp[(2 * b + 1) * bbs] + cmg < bbp[(2 * a) * bbs];
      if (__all_sync(__activemask(), apart)) continue;
    }
    {
      ColTile<PD, TB> C;
      C.load(X, Y, Z, b * TB, m2u);
      uint32_t fb[TB];
#pragma unroll
      for (int k = 0; k < TB; ++k) fb[k] = 0;
      uint32_t ma = 0;
      // row culling: a row pair whose x lies outside tile b's extent ± margin
      // (for every item of the warp) cannot conflict with any column
      const float blo = cull ? bbp[(2 * b) * bbs] - cmg : -INFINITY;
      const float bhi = cull ? bbp[(2 * b + 1) * bbs] + cmg : INFINITY;
#pragma unroll 2
      for (int i = 0; i < TB / 2; ++i) {
        const float2 ax = *reinterpret_cast<const float2*>(X + a * TB + 2 * i);
        if (cull) {
          const bool far = (ax.x < blo || ax.x > bhi) && (ax.y < blo || ax.y > bhi);
          if (__all_sync(__activemask(), far)) continue;
        }
        const float2 ay = *reinterpret_cast<const float2*>(Y + a * TB + 2 * i);
        const float2 az = PD == 3 ? *reinterpret_cast<const float2*>(Z + a * TB + 2 * i) : make_float2(0.f, 0.f);
        const float n0 = fmaf(ax.x, ax.x, fmaf(ay.x, ay.x, az.x * az.x));
        const float n1 = fmaf(ax.y, ax.y, fmaf(ay.y, ay.y, az.y * az.y));
        uint32_t fa0 = 0, fa1 = 0;
#pragma unroll
        for (int j = 0; j < TB / 2; ++j) {
          uint64_t t0, t1;
          row_pair_vs_col<PD, TB>(C, j, ax, ay, az, n0, n1, t0, t1);
          fa0 |= lo32(t0) | hi32(t0);
          fa1 |= lo32(t1) | hi32(t1);
          fb[2 * j] |= lo32(t0) | lo32(t1);
          fb[2 * j + 1] |= hi32(t0) | hi32(t1);
        }
        ma |= ((fa0 >> 31) | ((fa1 >> 31) << 1)) << (2 * i);
      }
      or_mask<MAXW>(cm, a * TB, ma);
      or_mask<MAXW>(cm, b * TB, sign_mask<TB>(fb));
    }
  }
}

// ------------------------------------------------------- fp32 pair-list path
// Rp = 64 robots as 32 column pairs (2l, 2l+1); a warp is one sample's 32
// consecutive steps (TC = 64: two warp windows per chunk).  Phase A leaves each
// robot's bounding box over the window (its swept box); the chunk ranking
// (x strips of 16, y inside a strip) pairs robots that are close.  Per window
// the warp first decides which pair-pair blocks can hold a conflict — swept
// pair boxes within the margin, one lane per pair, one ballot per offset d of
// the circular enumeration (l, l + d mod 32) — then every lane tests only
// those blocks at its own step: 4 tests per block in the direct form
// t = Δx² + Δy² − m²↑ (8 packed FP2 ops), sign bit ⇔ the reference's `<=`
// (reward.cpp:106).  Obstacles likewise: pair boxes vs the obstacles'
// inflated boxes, then t = |p − c|² − L²↑ (reward.cpp:120).  The culling is
// exact: swept boxes contain every position of the window and the margin
// carries a rounding slack (cull_margin), so a skipped block holds no hit.
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ bool boxes_meet(float4 a, float4 b) {  // (lo.x, lo.y, hi.x, hi.y)
  return a.z >= b.x && b.z >= a.x && a.w >= b.y && b.w >= a.y;
}

// Pair (2l, 2l+1) vs pair (2j, 2j+1) at one step: conflict bits of the four
// robots OR-ed into `conf` (bit = column).  Hits are rare: the bit assembly
// is behind a branch on "any test of this lane hit".
__device__ __forceinline__ void pl_block(const float* X, const float* Y, int l, int j, uint64_t nm2, uint64_t& conf) {
  const uint64_t xa = *reinterpret_cast<const uint64_t*>(X + 2 * l);
  const uint64_t ya = *reinterpret_cast<const uint64_t*>(Y + 2 * l);
  const uint64_t xb = *reinterpret_cast<const uint64_t*>(X + 2 * j);
  const uint64_t yb = *reinterpret_cast<const uint64_t*>(Y + 2 * j);
  uint64_t t0 = ffma2_sq(fsub2(xb, pack2(lo_f(xa), lo_f(xa))), nm2);
  uint64_t t1 = ffma2_sq(fsub2(xb, pack2(hi_f(xa), hi_f(xa))), nm2);
  t0 = ffma2_sq(fsub2(yb, pack2(lo_f(ya), lo_f(ya))), t0);
  t1 = ffma2_sq(fsub2(yb, pack2(hi_f(ya), hi_f(ya))), t1);
  const uint32_t r0 = lo32(t0) | hi32(t0), r1 = lo32(t1) | hi32(t1);
  if ((int)(r0 | r1) < 0) {
    const uint32_t c0 = lo32(t0) | lo32(t1), c1 = hi32(t0) | hi32(t1);
    const uint64_t rb = (r0 >> 31) | ((r1 >> 31) << 1), cb = (c0 >> 31) | ((c1 >> 31) << 1);
    conf |= (rb << (2 * l)) | (cb << (2 * j));
  }
}

// One (sample, t) item of the pair-list path: conflict and obstacle bits per
// column.  Called by all 32 lanes of a warp (one sample, one window); lanes
// whose step lies beyond the horizon run along and the caller drops them.
__device__ __forceinline__ void item_pl(const FitSmem<float>& sm, int s, int tc, int n_obs, float m2u, float cmh,
                                        bool cull, uint64_t& conf, uint64_t& obsm) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const float* X = sm.row(0, s, tc);
  const float* Y = sm.row(1, s, tc);
  float4* pb = sm.pbox + (size_t)(s * (sm.TC / 32) + (tc >> 5)) * sm.Rp;
  const uint64_t nm2 = pack2(-m2u, -m2u);
  const float4 b0 = pb[2 * lane], b1 = pb[2 * lane + 1];
  const float4 A = make_float4(fminf(b0.x, b1.x), fminf(b0.y, b1.y), fmaxf(b0.z, b1.z), fmaxf(b0.w, b1.w));
  const float4 Ai = make_float4(A.x - cmh, A.y - cmh, A.z + cmh, A.w + cmh);
  // the pair's own test (2l, 2l+1)
  uint32_t bits = full;
  if (cull) {
    const float4 b0i = make_float4(b0.x - cmh, b0.y - cmh, b0.z + cmh, b0.w + cmh);
    const float4 b1i = make_float4(b1.x - cmh, b1.y - cmh, b1.z + cmh, b1.w + cmh);
    bits = __ballot_sync(full, boxes_meet(b0i, b1i));
  }
  __syncwarp();
  pb[lane] = Ai;  // pair boxes replace the robot boxes (this warp's window only)
  __syncwarp();
  while (bits) {
    const int l = __ffs(bits) - 1;
    bits &= bits - 1u;
    const float2 x = *reinterpret_cast<const float2*>(X + 2 * l);
    const float2 y = *reinterpret_cast<const float2*>(Y + 2 * l);
    const float dx = x.y - x.x, dy = y.y - y.x;
    const float t = fmaf(dx, dx, fmaf(dy, dy, -m2u));
    if (t < 0.f) conf |= 3ull << (2 * l);
  }
  // pair-pair blocks (l, l + d mod 32), d = 1..16 (d = 16 once per pair):
  // all 16 ballots first (independent loads and votes), then the blocks
  // (pairing two blocks per iteration, or four, measured slower: code size)
  uint32_t lv[16];
#pragma unroll
  for (int d = 1; d <= 16; ++d) {
    if (cull) {
      const float4 B = pb[(lane + d) & 31];
      lv[d - 1] = __ballot_sync(full, (d < 16 || lane < 16) && boxes_meet(Ai, B));
    } else {
      lv[d - 1] = d < 16 ? full : 0xffffu;
    }
  }
#pragma unroll
  for (int d = 1; d <= 16; ++d) {
    uint32_t live = lv[d - 1];
    while (live) {
      const int l1 = __ffs(live) - 1;
      live &= live - 1u;
      pl_block(X, Y, l1, (l1 + d) & 31, nm2, conf);
    }
  }
  // obstacles: pair boxes vs the obstacles' inflated boxes, eight ballots at a time
  for (int o0 = 0; o0 < n_obs; o0 += 8) {
    uint32_t ov[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int o = o0 + q;
      ov[q] = 0;
      if (o < n_obs)
        ov[q] = cull ? __ballot_sync(full, boxes_meet(A, *reinterpret_cast<const float4*>(sm.opl + 8 * o + 4))) : full;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t live = ov[q];
      if (!live) continue;
      const float4 oc = *reinterpret_cast<const float4*>(sm.opl + 8 * (o0 + q));  // cx, cy, −L²↑
      const uint64_t cx = pack2(oc.x, oc.x), cy = pack2(oc.y, oc.y), nl = pack2(oc.z, oc.z);
      while (live) {
        const int l = __ffs(live) - 1;
        live &= live - 1u;
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

// One (sample, t) item in fp64: the reference's loops (reward.cpp:88-127) on
// shared-memory positions, exact `<=` tests; returns Σ goal terms.
template <int PD>
__device__ __forceinline__ double item_f64(const FitSmem<double>& sm, int s, int tc, int R, int n_obs, double m2,
                                           int* nconf, int* nobs) {
  const double* X = sm.row(0, s, tc);
  const double* Y = sm.row(1, s, tc);
  const double* Z = PD == 3 ? sm.row(2, s, tc) : X;
  double g = 0.0;
  for (int k = 0; k < R; ++k) {
    double gsq = 0.0, d;
    d = __dadd_rn(X[k], -sm.goal[k]);
    gsq = __dadd_rn(gsq, __dmul_rn(d, d));
    d = __dadd_rn(Y[k], -sm.goal[sm.Rp + k]);
    gsq = __dadd_rn(gsq, __dmul_rn(d, d));
    if constexpr (PD == 3) {
      d = __dadd_rn(Z[k], -sm.goal[2 * sm.Rp + k]);
      gsq = __dadd_rn(gsq, __dmul_rn(d, d));
    }
    g = __dadd_rn(g, __dadd_rn(1.0, -(sqrt(gsq) / sm.inv[2 * k])));
    for (int l = 0; l < R; ++l) {
      if (l == k) continue;
      double s2 = 0.0;
      d = __dadd_rn(X[k], -X[l]);
      s2 = __dadd_rn(s2, __dmul_rn(d, d));
      d = __dadd_rn(Y[k], -Y[l]);
      s2 = __dadd_rn(s2, __dmul_rn(d, d));
      if constexpr (PD == 3) {
        d = __dadd_rn(Z[k], -Z[l]);
        s2 = __dadd_rn(s2, __dmul_rn(d, d));
      }
      if (s2 <= m2) {
        ++*nconf;
        break;
      }
    }
    for (int o = 0; o < n_obs; ++o) {
      const double* ob = sm.obs + 4 * o;
      double s2 = 0.0;
      d = __dadd_rn(X[k], -ob[0]);
      s2 = __dadd_rn(s2, __dmul_rn(d, d));
      d = __dadd_rn(Y[k], -ob[1]);
      s2 = __dadd_rn(s2, __dmul_rn(d, d));
      if constexpr (PD == 3) {
        d = __dadd_rn(Z[k], -ob[2]);
        s2 = __dadd_rn(s2, __dmul_rn(d, d));
      }
      if (s2 <= ob[3]) {
        ++*nobs;
        break;
      }
    }
  }
  return g;
}

// ------------------------------------------------- fp32 fused rollout (phase A)
// Goal term of reward.cpp:92-97 for the robot a phase-A thread owns:
// accumulates ‖p − g‖ / ‖start − g‖ (ng = −g, ginv = 1/‖start − g‖).
template <int PD>
__device__ __forceinline__ void goal_acc(const float* x, const float* ng, float ginv, float& gsd) {
  // (x, y) − goal and its squares as packed pairs: FADD2 + FMUL2 + FADD
  const uint64_t dxy = fadd2(pack2(x[0], x[1]), pack2(ng[0], ng[1]));
  const uint64_t sq = fmul2(dxy, dxy);
  float d2 = lo_f(sq) + hi_f(sq);
  if constexpr (PD == 3) {
    const float dz = x[2] + ng[2];
    d2 = fmaf(dz, dz, d2);
  }
  gsd = fmaf(sqrt_approx(d2), ginv, gsd);
}

// Chunk sort key of a robot: its x in an order-preserving integer form, low
// bits replaced by the lane so keys are unique (the order only steers the
// culling; ties and near-ties may go either way).  Padding lanes sort last.
__device__ __forceinline__ int chunk_key(float x, int k, int Rp2, bool real) {
  int i = __float_as_int(x);
  i ^= (i >> 31) & 0x7fffffff;
  if (!real) i = 0x7fffffff;
  return (i & ~(Rp2 - 1)) | k;
}
// One robot's `nsteps` steps of a chunk: the block's base+msv loads are issued
// first, the Philox draws (in registers) hide their latency, z is written once
// for K5, then the RK4 steps run; positions go to the chunk's shared rows.
// Pointers advance by a stride per step (no per-step 64-bit index math).  The
// returned value is 0 unless some state went non-finite (NaN/inf propagate
// through fma(x, 0, acc)); the caller then replays the chunk exactly.
template <int KIND, bool FULL, bool SDV, bool PLB, int KPFT = kPFf<KIND>, int RDUC = 0, bool EFFORT = true,
          bool ZSTORE = true>
__device__ __forceinline__ void fused_block(const FitParams<float>& p, int nb, const float* bmp, const float* sdp,
                                            float* zp, int RDU_rt,
                                            uint64_t m, int kA, uint32_t g0, uint2 key, float* px, float* py, float* pz,
                                            int RS, float* x, float& eff32, float& chk, const float* ng, float ginv,
                                            float& gsd, float4& bx) {
  constexpr int DX = ModelDims<KIND>::DX, DU = ModelDims<KIND>::DU, PD = ModelDims<KIND>::PD;
  constexpr int KPF = KPFT;  // block depth (steps); RDUC: the row stride R·du when known at compile time
  const int RDU = RDUC ? RDUC : RDU_rt;
  float bq[KPF][DU], sq[SDV ? KPF : 1][DU];
#pragma unroll
  for (int j = 0; j < KPF; ++j) {
    if (FULL || j < nb) {
      if constexpr (DU == 2) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(bmp + j * RDU));
        bq[j][0] = v.x;
        bq[j][1] = v.y;
      } else {
#pragma unroll
        for (int d = 0; d < DU; ++d) bq[j][d] = __ldg(bmp + j * RDU + d);
      }
      if constexpr (SDV) {
#pragma unroll
        for (int d = 0; d < DU; ++d) sq[j][d] = __ldg(sdp + j * RDU + d);
      }
    }
  }
  float nz[KPF * DU];
#pragma unroll
  for (int g = 0; g < KPF * DU / 4; ++g) {
#ifdef D4K_EXPERIMENT_CHEAP_RNG
    const float h = __uint_as_float(((key.x ^ (uint32_t)m * 0x9E3779B9u ^ kA * 0x85EBCA6Bu ^ (g0 + g) * 0xC2B2AE35u) >> 9) | 0x3f800000u) - 1.5f;
    const float4 v = make_float4(h, -h, 0.5f * h, -0.5f * h);
#else
    const float4 v = philox_normals(key, m, (uint32_t)kA, g0 + g);
#endif
    nz[4 * g] = v.x;
    nz[4 * g + 1] = v.y;
    nz[4 * g + 2] = v.z;
    nz[4 * g + 3] = v.w;
  }
  if constexpr (ZSTORE) {  // ZSTORE = false: launches whose K5a regenerates the noise (z_keep == 2) carry no store code
    uint64_t zpol;  // L2 policy of the z stores (FitParams::z_keep)
    if (p.z_keep == 1) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(zpol));
    else asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(zpol));
  #pragma unroll
    for (int j = 0; j < KPF; ++j) {
      if (p.z_keep == 2) break;  // K5a regenerates the noise
      if (FULL || j < nb) {
        if constexpr (DU == 2) {
          asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(zp + j * RDU), "f"(nz[2 * j]),
                       "f"(nz[2 * j + 1]), "l"(zpol) : "memory");
        } else {
  #pragma unroll
          for (int d = 0; d < DU; ++d)
            asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(zp + j * RDU + d), "f"(nz[j * DU + d]),
                         "l"(zpol) : "memory");
        }
      }
    }
  }
  // two-control kinds: the control pair, its effort and (velocity input) the
  // position update as packed FFMA2 — the same per-lane fma as the scalar form
  constexpr bool PK = DU == 2 && !SDV;
  uint64_t eff2 = 0;
#pragma unroll
  for (int j = 0; j < KPF; ++j) {
    if (FULL || j < nb) {
      float u[DU];
      if constexpr (PK) {
        // base + (mean_scale·var + std·z), clamped; FMNMX equals cwiseMax/Min
        // here because NaN inputs are rejected on the host before launch
        const uint64_t v = ffma2(pack2(p.sd, p.sd), pack2(nz[2 * j], nz[2 * j + 1]), pack2(bq[j][0], bq[j][1]));
        u[0] = fminf(fmaxf(lo_f(v), p.lower[0]), p.upper[0]);
        u[1] = fminf(fmaxf(hi_f(v), p.lower[1]), p.upper[1]);
        const uint64_t uc = pack2(u[0], u[1]);
        if constexpr (EFFORT) eff2 = ffma2(uc, uc, eff2);
        if constexpr (KIND == HOLO2D_VEL) {  // rk4: x + dt·u (fp32 velocity-input closed form)
          const uint64_t xn = ffma2(pack2(p.dt, p.dt), uc, pack2(x[0], x[1]));
          x[0] = lo_f(xn);
          x[1] = hi_f(xn);
        } else {
          rk4<KIND>(x, u, p.dt, p.half_dt, p.dt6);
        }
      } else {
#pragma unroll
        for (int d = 0; d < DU; ++d) {
          const float sdj = SDV ? sq[SDV ? j : 0][d] : p.sd;
          u[d] = fminf(fmaxf(fmaf(sdj, nz[j * DU + d], bq[j][d]), p.lower[d]), p.upper[d]);
          if constexpr (EFFORT) eff32 = fmaf(u[d], u[d], eff32);
        }
        rk4<KIND>(x, u, p.dt, p.half_dt, p.dt6);
      }
      if constexpr (DX != PD) {  // state beyond the position: its own NaN/inf watch
        float s = x[0];
#pragma unroll
        for (int q = 1; q < DX; ++q) s += x[q];
        chk = fmaf(s, 0.f, chk);
      }
      goal_acc<PD>(x, ng, ginv, gsd);
      px[j * RS] = x[0];
      py[j * RS] = x[1];
      if constexpr (PD == 3) pz[j * RS] = x[2];
      if constexpr (PLB) {  // pair-list path: the robot's swept box over the warp window
        bx.x = fminf(bx.x, x[0]);
        bx.y = fminf(bx.y, x[1]);
        bx.z = fmaxf(bx.z, x[0]);
        bx.w = fmaxf(bx.w, x[1]);
      }
    }
  }
  if constexpr (PK) eff32 += lo_f(eff2) + hi_f(eff2);
}

__device__ __forceinline__ float4 empty_box() { return make_float4(INFINITY, INFINITY, -INFINITY, -INFINITY); }

template <int KIND, bool SDV, bool PL>
__device__ __forceinline__ float rollout_fused(const FitParams<float>& p, const FitSmem<float>& sm, int sA, int kA,
                                               int rA, int64_t m, int t0, int nsteps, float* x, float* zrow, uint2 key,
                                               float& eff32, const float* ng, float ginv, float& gsd) {
  constexpr int DU = ModelDims<KIND>::DU, PD = ModelDims<KIND>::PD;
  constexpr int KPF = kPFf<KIND>;
  const int RDU = p.R * DU;
  const int64_t e0 = ((int64_t)t0 * p.R + kA) * DU;
  const float* bmp = p.bm + e0;
  const float* sdp = SDV ? p.sdv + e0 : nullptr;
  float* zp = zrow + e0;
  float* px = sm.row(0, sA, 0) + rA;
  float* py = sm.row(1, sA, 0) + rA;
  float* pz = PD == 3 ? sm.row(2, sA, 0) + rA : px;
  const int RS = sm.RS;
  float chk = 0.f;
  float4 bx = empty_box();
  float4* pbw = PL ? sm.pbox + (size_t)sA * (sm.TC / 32) * sm.Rp + rA : nullptr;  // window 0 box slot
  D4K_CHECK(rA >= 0 && rA < sm.Rp && nsteps >= 1 && nsteps <= sm.TC);
  for (int tc = 0; tc < nsteps; tc += KPF) {
    const int nb = nsteps - tc;
    const uint32_t g0 = (uint32_t)((t0 + tc) * DU / 4);
    if (nb >= KPF) {
      fused_block<KIND, true, SDV, PL>(p, KPF, bmp, sdp, zp, RDU, (uint64_t)m, kA, g0, key, px, py, pz, RS, x, eff32, chk,
                                       ng, ginv, gsd, bx);
    } else {
      fused_block<KIND, false, SDV, PL>(p, nb, bmp, sdp, zp, RDU, (uint64_t)m, kA, g0, key, px, py, pz, RS, x, eff32,
                                        chk, ng, ginv, gsd, bx);
    }
    if constexpr (PL) {
      if (((tc + KPF) & 31) == 0 || tc + KPF >= nsteps) {  // end of a warp window (or of the steps)
        D4K_CHECK(pbw < sm.pbox + (size_t)(sA + 1) * (sm.TC / 32) * sm.Rp);
        *pbw = bx;
        pbw += sm.Rp;
        bx = empty_box();
      }
    }
    bmp += KPF * RDU;
    if constexpr (SDV) sdp += KPF * RDU;
    zp += KPF * RDU;
    px += KPF * RS;
    py += KPF * RS;
    pz += KPF * RS;
  }
  if constexpr (PL) {  // windows past the horizon: empty boxes
    for (float4* e = sm.pbox + (size_t)(sA + 1) * (sm.TC / 32) * sm.Rp + rA; pbw < e; pbw += sm.Rp) *pbw = empty_box();
  }
  // state = position (velocity-input kinds): a NaN/inf state reaches the goal
  // distance, so the goal sum (ginv > 0: start ≠ goal is validated) carries it
  if constexpr (ModelDims<KIND>::DX == PD) return gsd * 0.f;
  return chk;
}

// Exact replay of a chunk whose states went non-finite (rare): the same
// controls from the stored z, first failing (robot, step) reported as in
// dynamics.cpp:81-84.
template <int KIND>
__device__ __noinline__ void rollout_check(const FitParams<float>& p, int kA, int64_t m, int t0, int nsteps,
                                           const float* x_in, const float* zrow) {
  constexpr int DX = ModelDims<KIND>::DX, DU = ModelDims<KIND>::DU;
  float x[DX];
  for (int q = 0; q < DX; ++q) x[q] = x_in[q];
  for (int tc = 0; tc < nsteps; ++tc) {
    const int t = t0 + tc;
    const int64_t e = ((int64_t)t * p.R + kA) * DU;
    float u[DU];
    for (int d = 0; d < DU; ++d) {
      float zv;
      if (p.z_keep == 2) {  // z not stored: the same Philox draw as the fused block
        const int n = t * DU + d;
        const float4 v = philox_normals(p.keys[p.step], (uint64_t)m, (uint32_t)kA, (uint32_t)(n >> 2));
        const int l = n & 3;
        zv = l == 0 ? v.x : l == 1 ? v.y : l == 2 ? v.z : v.w;
      } else {
        zv = zrow[e + d];
      }
      u[d] = fminf(fmaxf(fmaf(p.sdv ? p.sdv[e + d] : p.sd, zv, p.bm[e + d]), p.lower[d]), p.upper[d]);
    }
    rk4<KIND>(x, u, p.dt, p.half_dt, p.dt6);
    bool fin = true;
    for (int q = 0; q < DX; ++q) fin = fin && isfinite(x[q]);
    if (!fin) {
      const unsigned long long key = ((unsigned long long)p.step_key << 52) | ((unsigned long long)m << 20) |
                                     ((unsigned long long)kA << 10) | (unsigned long long)(t + 1);
      atomicMin(p.err, key);
      return;
    }
  }
}

template <typename S, int KIND, int TB, int MAXW, int NOISE, bool PL = false>
__global__ void __launch_bounds__(kFitMaxThreads, TB >= 16 ? D4K_MINB16 : D4K_MINB8) k_rollout_fitness(const __grid_constant__ FitParams<S> p) {
  pdl_wait();
  static_assert(!PL || (std::is_same<S, float>::value && ModelDims<KIND>::PD == 2 && MAXW == 2),
                "pair-list path: fp32, planar kinds, Rp = 64");
  constexpr int DX = ModelDims<KIND>::DX, DU = ModelDims<KIND>::DU, PD = ModelDims<KIND>::PD;
  constexpr bool F32 = std::is_same<S, float>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // the pair-list instantiation has a fixed shape (Rp = TC = 64, 2 samples per
  // 128-thread CTA): compile-time constants for all identity / index math
  const int tid = threadIdx.x, nthreads = PL ? 128 : blockDim.x;
  const int R = p.R, Rp = PL ? 64 : p.Rp, TC = PL ? 64 : p.TC, spc = PL ? 2 : p.spc, T = p.T;

  FitSmem<S> sm;
  sm.npd = PD;
  sm.RS = Rp + 2;
  sm.TC = TC;
  sm.spc = spc;
  sm.Rp = Rp;
  sm.nthreads = nthreads;
  sm.pos = reinterpret_cast<S*>(smem_raw);
  {
    const size_t pos_b = (size_t)PD * spc * TC * sm.RS * sizeof(S);
    const size_t red_b = 2 * (size_t)nthreads * sizeof(double) + 2 * (size_t)nthreads * sizeof(int);
    sm.red = reinterpret_cast<double*>(smem_raw);  // aliases pos: used after the last chunk only
    sm.eff = sm.red + nthreads;
    sm.cnt = reinterpret_cast<int*>(sm.eff + nthreads);
    sm.obs = reinterpret_cast<S*>(smem_raw + (((pos_b > red_b ? pos_b : red_b) + 15) & ~size_t(15)));
  }
  if constexpr (F32 && PL) {
    sm.key = reinterpret_cast<int*>(sm.obs + 4 * (p.n_obs + 1));
    // plain pointer arithmetic on the shared base (an integer round trip would
    // lose the address space: generic LD/ST instead of LDS/STS); key is 16-B
    // aligned and spc·Rp = 128 ints, so pbox is too
    sm.pbox = reinterpret_cast<float4*>(sm.key + spc * Rp);
    sm.opl = reinterpret_cast<float*>(sm.pbox + (size_t)spc * (TC / 32) * Rp);
    sm.bb = sm.ocl = nullptr;
    sm.goal = sm.inv = nullptr;
    for (int j = tid; j < 8 * p.n_obs; j += nthreads) sm.opl[j] = p.obs_pl[j];  // (c, −L²↑, box)
  } else if constexpr (F32) {
    sm.key = reinterpret_cast<int*>(sm.obs + 4 * (p.n_obs + 1));  // 16-B aligned (Rp % 4 == 0)
    sm.bb = reinterpret_cast<float*>(sm.key + spc * Rp);
    sm.ocl = sm.bb + 2 * (Rp / TB) * nthreads;
    sm.goal = sm.inv = nullptr;
    for (int j = tid; j < 4 * (p.n_obs + 1); j += nthreads) sm.obs[j] = p.obs[j];  // (−2c, |c|²−L²↑), pad row
    for (int j = tid; j < 4 + 2 * kObsBuckets; j += nthreads) sm.ocl[j] = p.obs_cull[j];
  } else {
    sm.goal = sm.obs + 4 * (p.n_obs + 1);
    sm.inv = sm.goal + (size_t)PD * Rp;
    sm.ocl = nullptr;
    sm.key = nullptr;
    sm.bb = nullptr;
    for (int j = tid; j < PD * Rp; j += nthreads) {
      const int c = j / Rp, k = j % Rp;
      sm.goal[j] = k < R ? p.goals[k * PD + c] : S(0);
    }
    for (int k = tid; k < Rp; k += nthreads) {  // interleaved (‖s−g‖, valid)
      sm.inv[2 * k] = k < R ? p.inv_dstart[k] : S(1);
      sm.inv[2 * k + 1] = k < R ? S(1) : S(0);
    }
    for (int j = tid; j < 4 * p.n_obs; j += nthreads) sm.obs[j] = p.obs[j];  // (c, L²)
  }

  // ---- phase-A identity: (sample sA, robot kA)
  const int sA = tid / Rp, kA = tid % Rp;
  const int64_t mA = (int64_t)blockIdx.x * spc + sA;
  const bool liveA = mA < p.M;
  const bool robotA = liveA && kA < R;
  S x[DX];
#pragma unroll
  for (int j = 0; j < DX; ++j) x[j] = robotA ? p.starts[kA * DX + j] : S(0);
  if (liveA && kA >= R) {  // padding robots: parked far apart, never counted
    for (int tc = 0; tc < TC; ++tc) {
      sm.row(0, sA, tc)[kA] = S(1.0e6) + S(1.0e3) * S(kA);
      sm.row(1, sA, tc)[kA] = S(-1.0e6) - S(1.0e3) * S(kA);
      if constexpr (PD == 3) sm.row(2, sA, tc)[kA] = S(1.0e6);
    }
  }
  if (robotA && p.states_out) {
    S* so = p.states_out + mA * (int64_t)(T + 1) * R * DX + (int64_t)kA * DX;
#pragma unroll
    for (int j = 0; j < DX; ++j) so[j] = x[j];
  }
  const S* zrow = p.z + (liveA ? mA : 0) * (int64_t)T * R * DU;
  // per-robot accumulators across chunks: fp32 on the throughput path (no
  // fp64 adds, no spills in the chunk loop), fp64 on the parity path
  using Acc = typename std::conditional<F32, float, double>::type;
  Acc effort = Acc(0);
  float eff32 = 0.f;
  bool bad = false;
  // fp32: the robot's goal term is accumulated here (Σ ‖p−g‖/‖s−g‖ per chunk)
  float ng[3] = {0.f, 0.f, 0.f}, ginv = 0.f;
  Acc goalA = Acc(0);
  if (F32 && robotA) {
#pragma unroll
    for (int c = 0; c < PD; ++c) ng[c] = -(float)p.goals[kA * PD + c];
    ginv = (float)p.inv_dstart[kA];
  }
  int Rp2 = 1;
  while (Rp2 < Rp) Rp2 <<= 1;

  // NOISE == 0: prefetch ring over the HBM noise stream + base/mean-scaled
  // variable (L2-resident).  NOISE == 1: the noise is drawn here in registers
  // (Philox, d4orm_common.cuh) block by block and written once for K5.  Both
  // are chunk-local, so they hold no registers during the fitness phase.
  S zq[kPF][DU], bq[kPF][DU], mq[kPF][F32 ? 1 : DU], sq[kPF][DU];
  S* zst = NOISE >= 1 ? p.z_store + (liveA ? mA : 0) * (int64_t)T * R * DU : nullptr;
  const uint2 key = NOISE >= 1 ? p.keys[p.step] : make_uint2(0u, 0u);
  auto fetch = [&](int t, int t_end, int slot) {
    if (NOISE == 0 && robotA && t < t_end) {
      const int64_t e = ((int64_t)t * R + kA) * DU;
#pragma unroll
      for (int d = 0; d < DU; ++d) {
        zq[slot][d] = __ldcs(zrow + e + d);
        sq[slot][d] = p.sdv ? __ldg(p.sdv + e + d) : p.sd;
        if constexpr (F32) {
          bq[slot][d] = __ldg(p.bm + e + d);
        } else {
          bq[slot][d] = __ldg(p.base + e + d);
          mq[slot][d] = __ldg(p.msv + e + d);
        }
      }
    }
  };
  // ---- phase-B identity.  TC >= Rp: ipt consecutive items per thread;
  // TC < Rp: each item is shared by Q = Rp/TC adjacent threads (task split).
  // Either way the threads of sample s are [s·Rp, (s+1)·Rp).
  const int ipt = TC >= Rp ? TC / Rp : 1;
  const int Q = TC >= Rp ? 1 : Rp / TC;
  const int qB = TC >= Rp ? 0 : tid % Q;
  const int item0 = TC >= Rp ? tid * ipt : tid / Q;
  const int sB = item0 / TC;
  const int64_t mB = (int64_t)blockIdx.x * spc + sB;
  const bool liveB = item0 < spc * TC && mB < p.M;
  double gsum = 0.0;
  int nconf = 0, nobs = 0;

  __syncthreads();

  for (int t0 = 0; t0 < T; t0 += TC) {
    // ===== fp32: rank the sample's robots by x at the chunk start; a robot's
    // positions go to column rA, so TB-robot tiles are x-strips (culling)
    int rA = kA;
    if (F32 && (p.cull || PL)) {
      if (liveA) sm.key[tid] = chunk_key((float)x[0], kA, Rp2, robotA);
      __syncthreads();
      if (robotA) {
        const int me = sm.key[tid];
        const int4* kv = reinterpret_cast<const int4*>(sm.key + sA * Rp);
        int r = 0;
        for (int j = 0; j < Rp / 4; ++j) {
          const int4 v = kv[j];
          r += (v.x < me) + (v.y < me) + (v.z < me) + (v.w < me);
        }
        rA = r;
      }
      if constexpr (PL) {
        // second level: y order inside each 16-robot x strip, so column pairs
        // (2l, 2l+1) are neighbours in both coordinates (padding stays last)
        // (keys stored at the x-rank slot: a strip's 16 keys are contiguous)
        __syncthreads();
        int me = 0;
        if (liveA) {
          int yi = __float_as_int((float)x[1]);
          yi ^= (yi >> 31) & 0x7fffffff;
          const uint32_t yu = (uint32_t)yi ^ 0x80000000u;
          me = robotA ? (int)(((yu >> 10) << 6) | (uint32_t)kA) : (int)(0x7fffffc0u | (uint32_t)kA);
          D4K_CHECK(rA >= 0 && rA < Rp);
          sm.key[sA * Rp + rA] = me;
        }
        __syncthreads();
        if (robotA) {
          const int4* kv = reinterpret_cast<const int4*>(sm.key + sA * Rp + (rA & ~15));
          int r = rA & ~15;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int4 v = kv[j];
            r += (v.x < me) + (v.y < me) + (v.z < me) + (v.w < me);
          }
          rA = r;
        }
        if (liveA && !robotA) {  // padding columns (rank = lane): empty window boxes
          for (int w = 0; w < TC / 32; ++w) sm.pbox[((size_t)sA * (TC / 32) + w) * Rp + kA] = empty_box();
        }
      }
    }
    // ===== phase A: integrate TC steps
    if constexpr (NOISE >= 1) {
      if (robotA) {
        const int nsteps = t0 + TC < T ? TC : T - t0;
        float x0[DX];
#pragma unroll
        for (int q = 0; q < DX; ++q) x0[q] = x[q];
        float gsd = 0.f;
        const float chk = rollout_fused<KIND, NOISE == 2, PL>(p, sm, sA, kA, rA, p.m_global0 + mA, t0, nsteps, x, zst, key, eff32,
                                              ng, ginv, gsd);
        goalA += (Acc)nsteps - (Acc)gsd;
        if (!(chk == 0.f)) rollout_check<KIND>(p, kA, p.m_global0 + mA, t0, nsteps, x0, zst);
      }
    } else if (robotA) {
      float gsd = 0.f;
      const int t_end = t0 + TC < T ? t0 + TC : T;
      float4 bxA = empty_box();  // pair-list path: swept box of the warp window
      float4* pbwA = PL ? sm.pbox + (size_t)sA * (TC / 32) * Rp + rA : nullptr;
#pragma unroll
      for (int j = 0; j < kPF; ++j) fetch(t0 + j, t_end, j);
      for (int tc = 0; tc < TC; tc += kPF) {
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
          const int t = t0 + tc + j;
          if (t < T) {
            S u[DU];
#pragma unroll
            for (int d = 0; d < DU; ++d) {
              S v;
              if constexpr (F32) {
                // base + (mean_scale·var + std·z), clamped (FMNMX; NaN inputs are
                // rejected on the host before launch, so this equals cwiseMax/Min)
                v = fminf(fmaxf(fmaf(sq[j][d], zq[j][d], bq[j][d]), p.lower[d]), p.upper[d]);
              } else {
                v = xadd(bq[j][d], xadd(mq[j][d], xmul(sq[j][d], zq[j][d])));
                v = (v < p.lower[d]) ? p.lower[d] : v;  // cwiseMax(lower), dynamics.cpp:78
                v = (p.upper[d] < v) ? p.upper[d] : v;  // cwiseMin(upper)
              }
              u[d] = v;
              eff32 = fmaf(v, v, eff32);  // effort extension (w_e·Σ‖u‖²)
            }
            fetch(t + kPF, t_end, j);
            rk4<KIND>(x, u, p.dt, p.half_dt, p.dt6);
            bool fin = true;
#pragma unroll
            for (int q = 0; q < DX; ++q) fin = fin && isfinite(x[q]);
            if (!fin && !bad) {
              bad = true;
              const unsigned long long key = ((unsigned long long)p.step_key << 52) |
                                             ((unsigned long long)(p.m_global0 + mA) << 20) |
                                             ((unsigned long long)kA << 10) | (unsigned long long)(t + 1);
              atomicMin(p.err, key);
            }
            if constexpr (F32) goal_acc<PD>(x, ng, ginv, gsd);
            D4K_CHECK(rA >= 0 && rA < Rp);
            sm.row(0, sA, tc + j)[rA] = x[0];
            sm.row(1, sA, tc + j)[rA] = x[1];
            if constexpr (PD == 3) sm.row(2, sA, tc + j)[rA] = x[2];
            if constexpr (PL) {
              bxA.x = fminf(bxA.x, (float)x[0]);
              bxA.y = fminf(bxA.y, (float)x[1]);
              bxA.z = fmaxf(bxA.z, (float)x[0]);
              bxA.w = fmaxf(bxA.w, (float)x[1]);
              if (((tc + j + 1) & 31) == 0 || t + 1 == t_end) {
                *pbwA = bxA;
                pbwA += Rp;
                bxA = empty_box();
              }
            }
            if (NOISE == 0 && p.states_out) {
              S* so = p.states_out + (mA * (int64_t)(T + 1) + t + 1) * R * DX + (int64_t)kA * DX;
#pragma unroll
              for (int q = 0; q < DX; ++q) so[q] = x[q];
            }
            if (NOISE == 0 && p.controls_out) {
              S* co = p.controls_out + (mA * (int64_t)(T + 1) + t) * R * DU + (int64_t)kA * DU;
#pragma unroll
              for (int d = 0; d < DU; ++d) co[d] = u[d];
            }
          }
        }
      }
      if constexpr (F32) goalA += (Acc)(t_end - t0) - (Acc)gsd;
      if constexpr (PL) {  // windows past the horizon: empty boxes
        for (float4* e = sm.pbox + (size_t)(sA + 1) * (TC / 32) * Rp + rA; pbwA < e; pbwA += Rp) *pbwA = empty_box();
      }
    }
    effort += (Acc)eff32;  // per-chunk fp32 partial → the cross-chunk accumulator
    eff32 = 0.f;
    __syncthreads();

    // ===== phase B: fitness of the TC steps just integrated
#ifdef D4K_EXPERIMENT_SKIP_B
    const bool runB = p.n_obs < 0;
#else
    constexpr bool runB = true;
#endif
    if (PL && runB && mB < p.M) {
      // pair-list path: the warp is one sample's 32-step window; lanes past the
      // horizon run the warp-collective loops and are dropped here
      if constexpr (PL) {
        const int tc = item0 - sB * TC;
        if (t0 + (tc & ~31) < T) {
          uint64_t conf = 0, obsm = 0;
          item_pl(sm, sB, tc, p.n_obs, p.margin_sq, 0.5f * p.cull_margin, p.cull != 0, conf, obsm);
          if (t0 + tc < T) {
            const uint64_t real = R >= 64 ? ~0ull : ((1ull << R) - 1ull);
            nconf += __popcll(conf & real);
            nobs += __popcll(obsm & real);
          }
        }
      }
    } else if (liveB && runB) {
      for (int j = 0; j < ipt; ++j) {
        const int tc = item0 + j - sB * TC;
        if (t0 + tc >= T) break;
        if constexpr (F32) {
          uint32_t cm[MAXW];
#pragma unroll
          for (int w = 0; w < MAXW; ++w) cm[w] = 0;
          if (p.cull)
            item_f32<PD, TB, MAXW, true>(sm, sB, tc, R, p.n_obs, p.margin_sq, p.cull_margin, qB, Q,
                                         sm.bb + (tid - qB), cm, &nobs);
          else
            item_f32<PD, TB, MAXW, false>(sm, sB, tc, R, p.n_obs, p.margin_sq, p.cull_margin, qB, Q,
                                          sm.bb + (tid - qB), cm, &nobs);
          // merge the Q lanes' conflict flags (adjacent lanes, same item)
          for (int off = 1; off < Q; off <<= 1) {
#pragma unroll
            for (int w = 0; w < MAXW; ++w) cm[w] |= __shfl_xor_sync(__activemask(), cm[w], off);
          }
          if (qB == 0) {
#pragma unroll
            for (int w = 0; w < MAXW; ++w) {
              const int kv = R - 32 * w;
              if (kv > 0) nconf += __popc(kv >= 32 ? cm[w] : (cm[w] & ((1u << kv) - 1u)));
            }
          }
        } else if (qB == 0) {
          gsum += item_f64<PD>(sm, sB, tc, R, p.n_obs, p.margin_sq, &nconf, &nobs);
        }
      }
    }
    __syncthreads();
  }

  // ---- per-sample deterministic reduction
  sm.red[tid] = (liveB ? gsum : 0.0) + (robotA ? (double)goalA : 0.0);  // fp32 goal terms come from phase A
  sm.eff[tid] = robotA ? (double)effort : 0.0;
  sm.cnt[2 * tid] = liveB ? nconf : 0;
  sm.cnt[2 * tid + 1] = liveB ? nobs : 0;
  __syncthreads();
  if (liveB && tid == sB * Rp) {  // first thread of the sample
    const int nt = Rp;
    const int first = sB * Rp;
    double g = 0.0;
    long long nc = 0, no = 0;
    for (int q = 0; q < nt; ++q) {
      g += sm.red[first + q];
      nc += sm.cnt[2 * (first + q)];
      no += sm.cnt[2 * (first + q) + 1];
    }
    double value = g - p.w_t * (double)nc - p.w_o * (double)no;
    if (p.w_e != 0.0) {  // effort extension
      double eff = 0.0;
      for (int k = 0; k < R; ++k) eff += sm.eff[sB * Rp + k];
      value -= p.w_e * eff;
    }
    p.reward[mB] = value / ((double)R * (double)T);
    if (p.counts) {
      p.counts[2 * mB] = (int)nc;
      p.counts[2 * mB + 1] = (int)no;
    }
  }
}

}  // namespace d4k
