// Launcher of the time-segmented K2+K3 variant (k_seg.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace d4k {
template <typename S>
struct FitParams;
// kind ∈ {HOLO2D_VEL, HOLO3D_VEL}, R ∈ {1, 2, 4, 8, 16}, T % 8 == 0, T ≤ 128,
// segments aligned to Philox groups ((T/8)·du % 4 == 0)
bool seg_supported(int kind, int R, int T, int du);
size_t seg_smem_bytes(int R, int T, int pdim);
cudaError_t launch_seg(int kind, bool philox, int64_t M, cudaStream_t st, const FitParams<float>& f);
}  // namespace d4k
