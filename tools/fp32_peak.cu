// FP32 pipe microbenchmark for the roofline denominator ("measure an
// FP32 FMA microbenchmark plus SM count and clocks on the box").
// Reports, per instruction form, sustained throughput over the whole GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// 3-register FFMA, 8 independent chains.
__global__ void k_ffma(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
  float bb = b + threadIdx.x * 1e-9f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, bb);
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5f) out[0] = s;
}

// Packed FFMA2 (sm_100 f32x2), 8 independent chains of float2.
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long x[8];
  float2 av = make_float2(a, a + threadIdx.x * 1e-9f), bv = make_float2(b, b);
  unsigned long long ar = *reinterpret_cast<unsigned long long*>(&av);
  unsigned long long br = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int j = 0; j < 8; ++j) { float2 v = make_float2(threadIdx.x * 1e-3f + j, j); x[j] = *reinterpret_cast<unsigned long long*>(&v); }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = ffma2(x[j], ar, br);
  }
  float s = 0; for (int j = 0; j < 8; ++j) { float2 v = *reinterpret_cast<float2*>(&x[j]); s += v.x + v.y; }
  if (s == 1234.5f) out[0] = s;
}

// Pair-test proxy: per 2 pairs FADD2,FADD2,FFMA2,FFMA2 + one LOP3 (sign-AND flags).
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__global__ void k_pair(float* out, float a, float b) {
  unsigned long long px[4], py[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 v = make_float2(threadIdx.x * 1e-3f + j, j * 0.5f); px[j] = *reinterpret_cast<unsigned long long*>(&v);
    float2 w = make_float2(j * 0.25f, threadIdx.x * 2e-3f); py[j] = *reinterpret_cast<unsigned long long*>(&w);
  }
  float2 kv = make_float2(a, a), mv = make_float2(b, b);
  unsigned long long kx = *reinterpret_cast<unsigned long long*>(&kv), m2 = *reinterpret_cast<unsigned long long*>(&mv);
  unsigned int f0 = 0xffffffffu, f1 = 0xffffffffu;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      unsigned long long dx = fadd2(kx, px[j]);
      unsigned long long dy = fadd2(kx, py[j]);
      unsigned long long t = ffma2(dy, dy, m2);
      t = ffma2(dx, dx, t);
      unsigned int lo = (unsigned int)t, hi = (unsigned int)(t >> 32);
      f0 &= lo & hi;
      px[j] ^= (unsigned long long)(f0 & 1u);  // keep loop-carried, cheap
    }
    kx += 0x100000001ull;
  }
  if ((f0 ^ f1) == 77u) out[0] = 1.f;
}

__global__ void k_mufu(float* out, float a) {
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j + 1.f;
  for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __logf(x[j] + a);
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f}\n", p.name, p.multiProcessorCount, clk_khz / 1e3);
  float* out; CK(cudaMalloc(&out, 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  for (int threads : {256, 512, 1024}) {
    for (int occ : {4, 8}) {
      int blocks = sms * occ * 256 / threads; if (blocks < sms) blocks = sms;
      double lanes = (double)blocks * threads;
      // warm
      k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f); CK(cudaDeviceSynchronize());
      float ms;
      cudaEventRecord(e0); k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double ffma = lanes * ITERS * 8 * 2 / (ms * 1e-3) / 1e12;
      cudaEventRecord(e0); k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double ffma2v = lanes * ITERS * 8 * 4 / (ms * 1e-3) / 1e12;
      cudaEventRecord(e0); k_pair<<<blocks, threads>>>(out, 0.5f, -0.2f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double pairs = lanes * ITERS * 4 * 2 / (ms * 1e-3) / 1e12;  // Tpairs/s
      cudaEventRecord(e0); k_mufu<<<blocks, threads>>>(out, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double mufu = lanes * (ITERS / 8) * 8 / (ms * 1e-3) / 1e12;
      printf("{\"threads\": %d, \"blocks\": %d, \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, \"pair_proxy_tpairs_s\": %.3f, \"pair_proxy_tflops_at6\": %.2f, \"mufu_lg2_tops\": %.3f}\n",
             threads, blocks, ffma, ffma2v, pairs, pairs * 6, mufu);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
