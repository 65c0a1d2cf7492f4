// k23_launch.cuh — launch glue for the fused rollout+fitness kernel (K2+K3).
// Instantiated per model kind in k23_k<kind>.cu so the 6 kinds × {f32,f64} ×
// robot-tile × noise-source variants compile in parallel.  Fused Philox noise
// (NOISE=1, and NOISE=2 with CEM's per-element std) exists for fp32 only; the
// fp64 parity path reads z from HBM.
#pragma once

#include "d4orm_kernels.cuh"
#include "k_pl32.cuh"
#include "k_small.cuh"

namespace d4k {

template <typename S, int KIND, int TB, int MAXW, int NOISE, bool PL = false>
cudaError_t launch_k23_tb(dim3 grid, int threads, size_t smem, cudaStream_t st, const FitParams<S>& p) {
  auto fn = k_rollout_fitness<S, KIND, TB, MAXW, NOISE, PL>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_step(fn, grid, dim3(threads), smem, st, false, p);
}

template <typename S, int KIND, int NOISE>
cudaError_t launch_k23_n(int tb, int maxw, bool pl, dim3 grid, int threads, size_t smem, cudaStream_t st,
                         const FitParams<S>& p) {
  if (pl) {  // pair-list fitness: fp32, planar kinds, Rp = 64
    if constexpr (std::is_same<S, float>::value && ModelDims<KIND>::PD == 2) {
      if (tb == 16 && maxw == 2) return launch_k23_tb<S, KIND, 16, 2, NOISE, true>(grid, threads, smem, st, p);
    }
    return cudaErrorInvalidValue;
  }
  if (maxw <= 2) {
    switch (tb) {
      case 4: return launch_k23_tb<S, KIND, 4, 2, NOISE>(grid, threads, smem, st, p);
      case 8: return launch_k23_tb<S, KIND, 8, 2, NOISE>(grid, threads, smem, st, p);
      case 16: return launch_k23_tb<S, KIND, 16, 2, NOISE>(grid, threads, smem, st, p);
      default: return cudaErrorInvalidValue;
    }
  }
  if (tb == 16) return launch_k23_tb<S, KIND, 16, 8, NOISE>(grid, threads, smem, st, p);
  return cudaErrorInvalidValue;
}

template <typename S, int KIND>
cudaError_t launch_k23(int tb, int maxw, int noise, bool pl, dim3 grid, int threads, size_t smem, cudaStream_t st,
                       const FitParams<S>& p) {
  if constexpr (std::is_same<S, float>::value) {
    if (noise && p.sdv) return launch_k23_n<S, KIND, 2>(tb, maxw, pl, grid, threads, smem, st, p);  // CEM
    if (noise) return launch_k23_n<S, KIND, 1>(tb, maxw, pl, grid, threads, smem, st, p);
  } else {
    if (noise || pl) return cudaErrorInvalidValue;
  }
  return launch_k23_n<S, KIND, 0>(tb, maxw, pl, grid, threads, smem, st, p);
}

#define D4K_INSTANTIATE_K23(KIND)                                                                      \
  template cudaError_t launch_k23<float, KIND>(int, int, int, bool, dim3, int, size_t, cudaStream_t,   \
                                               const FitParams<float>&);                                \
  template cudaError_t launch_k23<double, KIND>(int, int, int, bool, dim3, int, size_t, cudaStream_t,  \
                                                const FitParams<double>&);                               \
  template cudaError_t launch_pl32<KIND>(cudaStream_t, const FitParams<float>&);                       \
  template cudaError_t launch_small<KIND>(int, cudaStream_t, const FitParams<float>&);

}  // namespace d4k
