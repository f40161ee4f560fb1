// Peak probe for the "alu" roofline of the base case (SURVEY.md §8(d),
// "Integer MAD: LP_peak = SMs x r_LP x f_SM ... Measure it"): each thread
// runs 8 independent 3-word accumulators through the same
// mad.lo.cc / madc.hi.cc / addc sequence the schoolbook kernel issues per
// limb product.
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/toomgpu.h"

namespace {
constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) k_probe(uint32_t seed, uint32_t* sink) {
    uint32_t c0[kChains], c1[kChains], c2[kChains], a[kChains];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int j = 0; j < kChains; ++j) { c0[j] = t + j; c1[j] = 0; c2[j] = 0; a[j] = seed * (j + 3) + t; }
    uint32_t b = seed ^ t;
#pragma unroll 1
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int j = 0; j < kChains; ++j) {
            asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
                         "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
                         "addc.u32 %2, %2, 0;"
                         : "+r"(c0[j]), "+r"(c1[j]), "+r"(c2[j]) : "r"(a[j]), "r"(b));
        }
        b += 0x9E3779B9u;
    }
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < kChains; ++j) acc ^= c0[j] ^ c1[j] ^ c2[j];
    if (acc == 0x12345678u) sink[0] = acc;
}
}  // namespace

extern "C" double toom_probe_limb_products(double* ms, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return -1; }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t* sink = nullptr;
    if (cudaMalloc(&sink, 4) != cudaSuccess) { cudaGetLastError(); return -1; }
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_probe<<<blocks, threads, 0, st>>>(1u, sink);   // warm-up
    cudaEventRecord(a, st);
    for (int r = 0; r < 5; ++r) k_probe<<<blocks, threads, 0, st>>>(r + 2u, sink);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float t = 0;
    cudaEventElapsedTime(&t, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (cudaGetLastError() != cudaSuccess) return -1;
    if (ms) *ms = t;
    const double lp = 5.0 * blocks * threads * (double)kIters * kChains;
    return lp / (t * 1e-3);
}
