// bm32_probe.cu — evaluates the device BM32 transform (csrc/noise.cuh) over caller-chosen index
// ranges so a test can compare every radius input (2^23) and every angle index (2^24) bitwise
// with the oracle ("standard normal" eps).  Test
// infrastructure of the GPU side: it runs exactly the device functions the rollout and noise
// kernels call (bm32_radius / bm32_sincos and their packed FP32x2 twins), nothing else.
#include <cuda_runtime.h>

#include <cstdint>

#include "mppi_probe.h"
#include "noise.cuh"

namespace {

// Input word of index i: the index in the bits BM32 reads (w >> 9 for the radius, w >> 8 for the
// angle) and arbitrary low bits (a multiplicative hash of i), which the transform must ignore.
__device__ __forceinline__ uint32_t salt(uint32_t i, int shift) {
    return (i * 0x9E3779B9u) >> (32 - shift);
}

__global__ void bm32_radius_probe(uint32_t first, uint32_t count, int packed, float* out) {
    const uint32_t half = (count + 1) / 2;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (!packed) {
        if (i >= count) return;
        const uint32_t n = first + i;
        out[i] = mppi::bm32_radius((n << 9) | salt(n, 9));
        return;
    }
    // packed: lane a takes index i, lane b index i + half (two unrelated inputs per thread)
    if (i >= half) return;
    const uint32_t ia = i, ib = i + half < count ? i + half : i;
    const uint32_t na = first + ia, nb = first + ib;
    const float2 r = mppi::bm32_radius_x2((na << 9) | salt(na, 9), (nb << 9) | salt(nb, 9));
    out[ia] = r.x;
    if (ib != ia) out[ib] = r.y;
}

__global__ void bm32_angle_probe(uint32_t first, uint32_t count, int packed, float* sn, float* cs) {
    const uint32_t half = (count + 1) / 2;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (!packed) {
        if (i >= count) return;
        const uint32_t n = first + i;
        const float2 v = mppi::bm32_sincos((n << 8) | salt(n, 8));
        sn[i] = v.x;
        cs[i] = v.y;
        return;
    }
    if (i >= half) return;
    const uint32_t ia = i, ib = i + half < count ? i + half : i;
    const uint32_t na = first + ia, nb = first + ib;
    float2 s, c;
    mppi::bm32_sincos_x2((na << 8) | salt(na, 8), (nb << 8) | salt(nb, 8), s, c);
    sn[ia] = s.x;
    cs[ia] = c.x;
    if (ib != ia) {
        sn[ib] = s.y;
        cs[ib] = c.y;
    }
}

}  // namespace

extern "C" int mppi_probe_bm32(int kind, int packed, uint32_t first, uint32_t count, float* out0,
                               float* out1) {
    if (count == 0) return 0;
    const int threads = 256;
    const uint32_t work = packed ? (count + 1) / 2 : count;
    const uint32_t blocks = (work + threads - 1) / threads;
    if (kind == 0) {
        if (!out0 || (uint64_t)first + count > (1u << 23)) return -1;
        bm32_radius_probe<<<blocks, threads>>>(first, count, packed, out0);
    } else if (kind == 1) {
        if (!out0 || !out1 || (uint64_t)first + count > (1u << 24)) return -1;
        bm32_angle_probe<<<blocks, threads>>>(first, count, packed, out0, out1);
    } else {
        return -1;
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return (int)e;
}
