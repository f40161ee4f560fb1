// Peak probes for the "alu" roofline of the base case (SURVEY.md §8(d),
// "Integer MAD: LP_peak = SMs x r_LP x f_SM ... Measure it").
//   toom_probe_limb_products: the issue rate of the 32x32->64 integer MAD
//     (mad.wide.u32 -> IMAD.WIDE.U32), 8 independent 64-bit chains per thread:
//     one limb-product per instruction, the machine's limb-product peak.
//   toom_probe_carry_chain: 8 independent 3-word accumulators through the
//     mad.lo.cc / madc.hi.cc / addc sequence the schoolbook kernel issues per
//     limb product (carry-flag chains; reported for context).
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
__global__ void __launch_bounds__(256) k_probe_wide(uint32_t seed, uint32_t* sink) {
    unsigned long long acc[kChains];
    uint32_t a[kChains];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int j = 0; j < kChains; ++j) { acc[j] = t + j; a[j] = seed * (j + 3) + t; }
    uint32_t b = seed ^ t;
#pragma unroll 1
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int j = 0; j < kChains; ++j)
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[j]) : "r"(a[j]), "r"(b));
        b += 0x9E3779B9u;
    }
    unsigned long long x = 0;
#pragma unroll
    for (int j = 0; j < kChains; ++j) x ^= acc[j];
    if (x == 0x123456789ull) sink[0] = (uint32_t)x;
}

template <class K>
static double run_probe(K kern, double ops_per_thread_iter, double* ms, cudaStream_t st) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return -1; }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t* sink = nullptr;
    if (cudaMalloc(&sink, 4) != cudaSuccess) { cudaGetLastError(); return -1; }
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<blocks, threads, 0, st>>>(1u, sink);   // warm-up
    cudaEventRecord(a, st);
    for (int r = 0; r < 5; ++r) kern<<<blocks, threads, 0, st>>>(r + 2u, sink);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float t = 0;
    cudaEventElapsedTime(&t, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (cudaGetLastError() != cudaSuccess) return -1;
    if (ms) *ms = t;
    const double lp = 5.0 * blocks * threads * (double)kIters * ops_per_thread_iter;
    return lp / (t * 1e-3);
}
}  // namespace

extern "C" double toom_probe_limb_products(double* ms, void* stream) {
    return run_probe(k_probe_wide, kChains, ms, (cudaStream_t)stream);
}

extern "C" double toom_probe_carry_chain(double* ms, void* stream) {
    return run_probe(k_probe, kChains, ms, (cudaStream_t)stream);
}
