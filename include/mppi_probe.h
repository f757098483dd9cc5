/*
 * mppi_probe.h — FP32 peak probe used by bench.py for the rollout kernel's ALU roofline
 * denominator (libmppi_probe.so; not part of the MPPI step).
 *
 * mppi_probe_fp32 launches `blocks` x `threads` threads on the current device; each thread runs
 * `iters` iterations of 16 independent dependent chains of FFMA (packed = 0) or FFMA2
 * (packed = 1, sm_100 `fma.rn.f32x2`, two FMAs per instruction).  FLOPs counted = 2 per FMA.
 * Synchronous; times with CUDA events on the legacy stream.  Returns 0 on success, else the
 * CUDA error code.  tflops_out: HOST double, achieved TFLOP/s; ms_out: HOST double or NULL.
 */
#ifndef MPPI_PROBE_H
#define MPPI_PROBE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
int mppi_probe_fp32(int packed, int blocks, int threads, int iters, double* tflops_out,
                    double* ms_out);

/*
 * mppi_probe_bm32 — runs the device BM32 transform of the noise contract (
 * PAPER.md:101, eps standard normal) on the index range [first, first + count), for the
 * exhaustive GPU-vs-oracle test (tests/test_gpu_bm32_exhaustive.py).  Test infrastructure.
 *   kind 0 (radius): index n < 2^23, input word w = (n << 9) | (uint32(n * 0x9E3779B9) >> 23);
 *                    out0[i] = r(w) for n = first + i.
 *   kind 1 (angle):  index n < 2^24, input word w = (n << 8) | (uint32(n * 0x9E3779B9) >> 24);
 *                    out0[i] = sin theta(w), out1[i] = cos theta(w).
 *   packed = 0: the scalar device functions (bm32_radius, bm32_sincos); packed = 1: the FP32x2
 *   twins (bm32_radius_x2, bm32_sincos_x2), lane a on index i and lane b on index i + ceil(count/2).
 * out0/out1: DEVICE fp32 arrays of length count (caller-owned).  Synchronous on the legacy stream.
 * Returns 0, -1 for an invalid argument (range past the domain, NULL output), else the CUDA
 * error code.
 */
int mppi_probe_bm32(int kind, int packed, uint32_t first, uint32_t count, float* out0,
                    float* out1);
#ifdef __cplusplus
}
#endif
#endif
