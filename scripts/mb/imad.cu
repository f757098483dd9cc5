#include <cstdint>
#include <cstdio>
#define M0 0xD2511F53u
#define M1 0xCD9E8D57u
template <int V>
__global__ void philox_bench(uint32_t* out, int iters, uint32_t seed) {
    uint32_t c0 = threadIdx.x + blockIdx.x * blockDim.x, c1 = seed, c2 = 3, c3 = 4;
    uint32_t k0 = seed * 7, k1 = 11;
    uint32_t acc = 0; const uint32_t seedz = seed >> 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            uint32_t h0, l0, h1, l1;
            if (V == 0) {
                uint64_t p0 = (uint64_t)M0 * c0, p1 = (uint64_t)M1 * c2;
                h0 = p0 >> 32; l0 = (uint32_t)p0; h1 = p1 >> 32; l1 = (uint32_t)p1;
            } else if (V == 1) {
                asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(h0) : "r"(c0), "r"(M0));
                asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(l0) : "r"(c0), "r"(M0));
                asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(h1) : "r"(c2), "r"(M1));
                asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(l1) : "r"(c2), "r"(M1));
            } else if (V == 2) {
                h0 = __umulhi(c0, M0); h1 = __umulhi(c2, M1);
                asm("mad.lo.u32 %0, %1, %2, %1;" : "=r"(l0) : "r"(c0), "n"(M0 - 1));
                asm("mad.lo.u32 %0, %1, %2, %1;" : "=r"(l1) : "r"(c2), "n"(M1 - 1));
            } else {
                h0 = __umulhi(c0, M0); h1 = __umulhi(c2, M1);
                l0 = c0 * (M0 ^ seedz); l1 = c2 * (M1 ^ seedz);
            }
            uint32_t n0 = h1 ^ c1 ^ k0, n2 = h0 ^ c3 ^ k1;
            c0 = n0; c1 = l1; c2 = n2; c3 = l0;
            k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
        }
        acc += c0 ^ c1 ^ c2 ^ c3;
        c0 += it;
    }
    out[threadIdx.x + blockIdx.x * blockDim.x] = acc;
}
template __global__ void philox_bench<0>(uint32_t*, int, uint32_t);
template __global__ void philox_bench<1>(uint32_t*, int, uint32_t);
template __global__ void philox_bench<2>(uint32_t*, int, uint32_t);
template __global__ void philox_bench<3>(uint32_t*, int, uint32_t);

int main() {
    uint32_t* d;
    const int blocks = 148 * 8, threads = 256, iters = 4000;
    cudaMalloc(&d, blocks * threads * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        for (int v = 0; v < 4; ++v) {
            auto k = v == 0 ? philox_bench<0> : v == 1 ? philox_bench<1> : v == 2 ? philox_bench<2> : philox_bench<3>;
            k<<<blocks, threads>>>(d, 100, 1);
            cudaEventRecord(a);
            k<<<blocks, threads>>>(d, iters, 1);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double rounds = (double)blocks * threads * iters * 10;
            // 2 mulhilo per round
            printf("V%d %.3f ms  %.3f Tmulhilo/s  %.2f cycles/warp-mulhilo/SMSP @1.965GHz\n", v, ms,
                   2 * rounds / ms / 1e9, (ms * 1e-3 * 1.965e9 * 148 * 4) / (2 * rounds / 32));
        }
    }
    return 0;
}
