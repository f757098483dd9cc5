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
#ifdef __cplusplus
extern "C" {
#endif
int mppi_probe_fp32(int packed, int blocks, int threads, int iters, double* tflops_out,
                    double* ms_out);
#ifdef __cplusplus
}
#endif
#endif
