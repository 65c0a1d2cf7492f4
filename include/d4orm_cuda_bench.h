/*
 * d4orm_cuda_bench.h — measurement helpers (not part of the drop-in boundary).
 */
#ifndef D4ORM_CUDA_BENCH_H
#define D4ORM_CUDA_BENCH_H
#ifdef __cplusplus
extern "C" {
#endif
/* Sustained FP32 throughput of this GPU (TFLOP/s, FMA = 2 flops): packed
 * FFMA2 chains over all SMs, best of `reps`.  The roofline denominator for the
 * CUDA-core kernels (K2+K3), measured on the box that runs the bench. */
int d4orm_cuda_fp32_peak(int device, int reps, double* tflops, double* sm_clock_mhz);
#ifdef __cplusplus
}
#endif
#endif
