#pragma once
// GPU execution options for the drop-in (kept out of the reference structs so
// their signatures stay unchanged).  Per host thread; the defaults come from
// D4ORM_DEVICE / D4ORM_PRECISION=f32|f64 / D4ORM_NOISE=philox|host /
// D4ORM_GRAPHS=0|1 (for callers compiled unchanged against the reference headers).
#include "../d4orm_cuda.h"

namespace d4orm {

struct GpuOptions {
  int device{0};
  int precision{D4ORM_PREC_F32};  // D4ORM_PREC_F64: the reference's arithmetic (parity)
  bool host_noise{false};         // true: the reference's NormalStream draws (correctness mode)
  bool graphs{true};
};

void set_gpu_options(const GpuOptions& options);
GpuOptions gpu_options();

}  // namespace d4orm
