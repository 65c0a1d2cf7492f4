/*
 * d4orm_cuda_bench.h — measurement helpers (not part of the drop-in boundary).
 */
#ifndef D4ORM_CUDA_BENCH_H
#define D4ORM_CUDA_BENCH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* Sustained FP32 throughput of this GPU (TFLOP/s, FMA = 2 flops): packed
 * FFMA2 chains over all SMs, best of `reps`.  The roofline denominator for the
 * CUDA-core kernels (K2+K3), measured on the box that runs the bench. */
int d4orm_cuda_fp32_peak(int device, int reps, double* tflops, double* sm_clock_mhz);
/* Which fp32 fitness form K2+K3 runs for the context's problem: 1 = pair list
 * (planar teams of 33..64 robots), 0 = robot tiles, -1 = no problem set. */
struct d4orm_cuda_ctx;
int d4orm_cuda_fitness_path(const struct d4orm_cuda_ctx* ctx);
/* Which K2+K3 kernel the context's last fitness launch (or captured step) used:
 * 0 = k_rollout_fitness, 1 = the time-segmented kernel, 2 = the 32-step-window
 * pair-list kernel (k_rollout_fitness_pl32), -1 = none yet. */
int d4orm_cuda_last_fit_kernel(const struct d4orm_cuda_ctx* ctx);
/* How the context's last run formed the weighted mean (K5a): 1 = regenerated
 * the Philox noise (no z rows stored, k_wmean_regen), 0 = read the z rows
 * K2+K3 stored, -1 = no run yet. */
int d4orm_cuda_k5_regen(const struct d4orm_cuda_ctx* ctx);
/* The fp32 weights K4 left for K5 (after d4orm_cuda_score_weights or a step):
 * w64 cast to float, zero below the adaptive floor (weights whose total is at
 * most 2^-30 of the sum).  m = how many to copy. */
int d4orm_cuda_last_w32(struct d4orm_cuda_ctx* ctx, float* out, int64_t m);
#ifdef __cplusplus
}
#endif
#endif
