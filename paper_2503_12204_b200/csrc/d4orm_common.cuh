// d4orm_common.cuh — model kinds, reference-exact scalar arithmetic, RK4.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <type_traits>
#include <utility>

// Checked builds (-DD4K_CHECKED: libd4orm_b200_checked.so, run over
// tools/sanitize.py by tests/test_gpu_checked.py): device-side bounds checks
// on the shared-memory tiles, the pair-list window boxes, K4's octave bins,
// K5a's compaction and K5b's stack.  (compute-sanitizer is not available on
// the GPU pool; these are the repo's own substitute.)  No-ops otherwise.
#ifdef D4K_CHECKED
#define D4K_CHECK(cond)                                                                                   \
  do {                                                                                                    \
    if (!(cond)) {                                                                                        \
      printf("d4k check failed: %s:%d: %s (block %d,%d thread %d)\n", __FILE__, __LINE__, #cond,         \
             (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);                                         \
      __trap();                                                                                           \
    }                                                                                                     \
  } while (0)
#else
#define D4K_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace d4k {

// ------------------------------------------------- programmatic dependent launch
// The four kernels of a denoising step form a strict chain (K2+K3 → K4 → K5a →
// K5b → next step's K2+K3).  They are launched with programmatic stream
// serialization (sm_90+), so a kernel is scheduled while its predecessor's last
// blocks drain instead of after the grid-completion round trip; each waits in
// pdl_wait() — before touching anything its predecessor writes — until the
// predecessor grid has completed and its memory is visible.  Knob D4ORM_PDL=0.
// (An early griddepcontrol.launch_dependents at block start was measured
// slightly slower: C1 0.0187 -> 0.0196 ms, C4 0.152 -> 0.154 ms.)
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("D4ORM_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// Launch a step kernel (PDL when enabled; the cooperative attribute for grid-
// synchronising kernels, which are launched without PDL).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_step(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               bool cooperative, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  if (cooperative) {
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
  } else {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = (cooperative || pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fn, std::forward<Args>(args)...);
}

// ... as a grid of thread-block clusters (cluster = `cluster` CTAs)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_step_cluster(void (*fn)(KArgs...), dim3 grid, dim3 block, dim3 cluster, cudaStream_t st,
                                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster.x;
  at[0].val.clusterDim.y = cluster.y;
  at[0].val.clusterDim.z = cluster.z;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, fn, std::forward<Args>(args)...);
}

enum Kind { DIFFDRIVE = 0, HOLO2D = 1, HOLO3D = 2, HOLO2D_VEL = 3, HOLO3D_VEL = 4, UNICYCLE = 5 };

template <int KIND>
struct ModelDims;
template <> struct ModelDims<DIFFDRIVE> { static constexpr int DX = 4, DU = 2, PD = 2; };
template <> struct ModelDims<HOLO2D> { static constexpr int DX = 4, DU = 2, PD = 2; };
template <> struct ModelDims<HOLO3D> { static constexpr int DX = 6, DU = 3, PD = 3; };
template <> struct ModelDims<HOLO2D_VEL> { static constexpr int DX = 2, DU = 2, PD = 2; };
template <> struct ModelDims<HOLO3D_VEL> { static constexpr int DX = 3, DU = 3, PD = 3; };
template <> struct ModelDims<UNICYCLE> { static constexpr int DX = 3, DU = 2, PD = 2; };

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

// fp32 throughput path: sin/cos with a two-constant Cody-Waite reduction to
// [−π, π] and the MUFU approximations there (abs. error ≈ 2^-21 for any
// heading the rollouts reach).  NaN/inf headings stay non-finite.
__device__ __forceinline__ void fast_sincos(float a, float* s, float* c) {
  const float q = rintf(a * 0.159154943091895335769f);  // a / 2π
  float r = fmaf(q, -6.28318548202514648438f, a);       // float(2π) = 2π + 1.7484555e-7
  r = fmaf(q, 1.74845553e-7f, r);
  __sincosf(r, s, c);
}

// detail::rk4_with (dynamics.hpp:123-130), element order as Eigen evaluates it:
//   k2 = f(x + (0.5dt)k1), k3 = f(x + (0.5dt)k2), k4 = f(x + dt·k3)
//   x' = x + (dt/6)·(((k1 + 2k2) + 2k3) + k4)
template <int KIND, typename S>
__device__ __forceinline__ void rk4(S* x, const S* u, S dt, S half_dt, S dt6) {
  constexpr int DX = ModelDims<KIND>::DX;
  if constexpr (std::is_same<S, float>::value && (KIND == HOLO2D_VEL || KIND == HOLO3D_VEL)) {
    // fp32 throughput path, velocity-input models: the derivative is u at all
    // four stages, so RK4 is x + dt·u (one FFMA; equal in exact arithmetic to
    // the staged expression the fp64 path evaluates).
#pragma unroll
    for (int j = 0; j < DX; ++j) x[j] = fmaf(dt, u[j], x[j]);
    return;
  }
  if constexpr (std::is_same<S, float>::value && (KIND == UNICYCLE || KIND == DIFFDRIVE)) {
    // fp32 throughput path, heading kinds: the derivative depends on (θ, v)
    // only, and the θ/v components of x + (dt/2)·k1 and x + (dt/2)·k2 are the
    // same numbers (both derivatives are the held controls), so k3 = k2:
    // three distinct headings θ, θ + (dt/2)ω, θ + dt·ω, one fast sincos each.
    constexpr bool UNI = KIND == UNICYCLE;
    const float w = UNI ? u[1] : u[0];                 // heading rate ω
    const float v1 = UNI ? u[0] : x[3];                // speed at stages 1, 2 (= 3), 4
    const float v2 = UNI ? u[0] : x[3] + half_dt * u[1];
    const float v4 = UNI ? u[0] : x[3] + dt * u[1];
    float s1, c1, s2, c2, s4, c4;
    fast_sincos(x[2], &s1, &c1);
    fast_sincos(x[2] + half_dt * w, &s2, &c2);
    fast_sincos(x[2] + dt * w, &s4, &c4);
    const float kx2 = v2 * c2, ky2 = v2 * s2;
    x[0] = x[0] + dt6 * (((v1 * c1 + 2.f * kx2) + 2.f * kx2) + v4 * c4);
    x[1] = x[1] + dt6 * (((v1 * s1 + 2.f * ky2) + 2.f * ky2) + v4 * s4);
    x[2] = x[2] + dt6 * (((w + 2.f * w) + 2.f * w) + w);
    if constexpr (!UNI) x[3] = x[3] + dt6 * (((u[1] + 2.f * u[1]) + 2.f * u[1]) + u[1]);
    return;
  }
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

// ---------------------------------------------------------- packed f32x2
// sm_100 packed FP32 (FADD2 / FFMA2 / FMUL2): two lanes per instruction, the
// scalar operand broadcast from one register.
__device__ __forceinline__ uint64_t pack2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {  // MUFU.SQRT (fp32 throughput path)
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lo_f(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi_f(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint32_t lo32(uint64_t v) { return (uint32_t)v; }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return (uint32_t)(v >> 32); }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fadd2_b(float a, uint64_t b) { return fadd2(pack2(a, a), b); }  // (a,a)+b
__device__ __forceinline__ uint64_t ffma2_sq(uint64_t a, uint64_t c) {                               // a*a + c
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(d) : "l"(a), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {  // a*b + c
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// ------------------------------------------------------------ Philox noise
// Philox4x32-10 (Salmon et al., SC'11) + Box-Muller.  Noise of denoising step
// i is keyed by keys[i] = mix_seed(seed_it, i).  For sample m and robot k the
// normals form one sequence n = t·du + d (t < T, d < du); group g = n/4 is
// Philox(counter = (k, g, m_hi, m_lo)), lanes n%4.  (The words that vary
// along a draw loop — g along a rollout thread's steps, m_lo along the weighted
// mean's samples — sit in the two XOR-only slots of round 1 (y, w), so the
// compiler folds round 1 and half of rounds 2–3 into per-thread constants: 34
// instead of 37–40 integer ops per group.)  Each normal is a pure
// function of (seed, i, m, k, t, d): identical under any sharding of samples,
// and a rollout thread owning robot k draws its own stream with no redundancy.
#ifndef D4K_PHILOX_ROUNDS
#define D4K_PHILOX_ROUNDS 10
#endif
struct Philox {
  static __device__ __forceinline__ uint4 round(uint4 c, uint2 k) {
    // one IMAD.WIDE.U32 per 32x32→64 product (hi and lo together)
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    return make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k.x, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k.y,
                      (uint32_t)p0);
  }
  static __device__ __forceinline__ uint4 gen(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < D4K_PHILOX_ROUNDS; ++r) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

// (2k+1)·2^-24 for k = x >> 9: strictly inside (0, 1) and exact.  Built from the
// bits as [1,2) − (1 − 2^-24): one LOP3 + one FADD.
__device__ __forceinline__ float u01_open(uint32_t x) {
  return __uint_as_float((x >> 9) | 0x3f800000u) - 0.99999994039535522461f;
}

// Box-Muller on the MUFU unit: r = √(−2 ln u) as √(−2 ln2 · log2 u), and the
// angle 2π·u folded into one FFMA on the [1, 2) bit pattern.
__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
  float l2;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(u01_open(a)));
  const float r = sqrt_approx(l2 * -1.38629436111989061883f);  // −2 ln u > 0
  const float f = __uint_as_float((b >> 9) | 0x3f800000u);     // 1 + k·2^-23
  float s, c;
  __sincosf(fmaf(f, 6.28318530717958647692f, -6.28318530717958647692f), &s, &c);  // 2π·k·2^-23
  const uint64_t z = fmul2(pack2(r, r), pack2(c, s));  // r·cos, r·sin in one FMUL2
  return make_float2(lo_f(z), hi_f(z));
}

// Round keys of Philox::gen, precomputed once (a loop drawing many groups under
// one key keeps them in registers instead of re-deriving the schedule per draw).
struct PhiloxKeys {
  uint2 rk[D4K_PHILOX_ROUNDS];
  __device__ __forceinline__ explicit PhiloxKeys(uint2 k) {
#pragma unroll
    for (int r = 0; r < D4K_PHILOX_ROUNDS; ++r) {
      rk[r] = k;
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
  }
  __device__ __forceinline__ uint4 gen(uint4 c) const {
#pragma unroll
    for (int r = 0; r < D4K_PHILOX_ROUNDS; ++r) c = Philox::round(c, rk[r]);
    return c;
  }
};

__device__ __forceinline__ float4 philox_normals(uint2 key, uint64_t m, uint32_t k, uint32_t g) {
  const uint4 r = Philox::gen(make_uint4(k, g, (uint32_t)(m >> 32), (uint32_t)m), key);
  const float2 a = box_muller(r.x, r.y), b = box_muller(r.z, r.w);
  return make_float4(a.x, a.y, b.x, b.y);
}

// philox_normals with a precomputed key schedule (same numbers)
__device__ __forceinline__ float4 philox_normals(const PhiloxKeys& ks, uint64_t m, uint32_t k, uint32_t g) {
  const uint4 r = ks.gen(make_uint4(k, g, (uint32_t)(m >> 32), (uint32_t)m));
  const float2 a = box_muller(r.x, r.y), b = box_muller(r.z, r.w);
  return make_float4(a.x, a.y, b.x, b.y);
}
// ... with the sample index as its two counter words (m = m_hi·2^32 + m_lo)
__device__ __forceinline__ float4 philox_normals(const PhiloxKeys& ks, uint32_t m_hi, uint32_t m_lo, uint32_t k,
                                                 uint32_t g) {
  const uint4 r = ks.gen(make_uint4(k, g, m_hi, m_lo));
  const float2 a = box_muller(r.x, r.y), b = box_muller(r.z, r.w);
  return make_float4(a.x, a.y, b.x, b.y);
}

}  // namespace d4k
