// fp32_probe.cu — FFMA / FFMA2 throughput probe (the ALU roofline denominator of bench.py).
#include <cuda_runtime.h>

#include "mppi_probe.h"

namespace {

__global__ void ffma_probe(float* out, int iters, float b, float c) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-7f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2_probe(float* out, int iters, float b, float c) {
    float2 a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = make_float2(threadIdx.x * 1e-7f + i, i * 0.5f);
    const float2 B = make_float2(b, b), Cc = make_float2(c, c);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = __ffma2_rn(a[i], B, Cc);
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

extern "C" int mppi_probe_fp32(int packed, int blocks, int threads, int iters, double* tflops_out,
                               double* ms_out) {
    float* out = nullptr;
    cudaError_t e = cudaMalloc(&out, (size_t)blocks * threads * sizeof(float));
    if (e != cudaSuccess) return (int)e;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    // warm-up launch, then the timed one
    for (int rep = 0; rep < 2; ++rep) {
        if (rep == 1) cudaEventRecord(a);
        if (packed) ffma2_probe<<<blocks, threads>>>(out, iters, 0.999999f, 1e-6f);
        else ffma_probe<<<blocks, threads>>>(out, iters, 0.999999f, 1e-6f);
    }
    cudaEventRecord(b);
    e = cudaEventSynchronize(b);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    if (e != cudaSuccess) return (int)e;
    const double fmas = (double)blocks * threads * iters * 16.0 * (packed ? 2.0 : 1.0);
    if (tflops_out) *tflops_out = 2.0 * fmas / (ms * 1e-3) / 1e12;
    if (ms_out) *ms_out = ms;
    return 0;
}
