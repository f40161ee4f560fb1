// Peak probes for the "alu" roofline of the base case (SURVEY.md §8(d),
// "Integer MAD: LP_peak = SMs x r_LP x f_SM ... Measure it").
//   toom_probe_limb_products: the issue rate of the 32x32->64 integer MAD
//     (mad.wide.u32 -> IMAD.WIDE.U32), 8 independent 64-bit chains per thread:
//     one limb-product per instruction, the machine's limb-product peak.
//   toom_probe_carry_chain: 8 x 8 product-scanning (Comba) schoolbook products
//     on the mad.lo.cc / madc.hi.cc / addc sequence the base-case kernels
//     issue per limb product (reported for context).
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/toomgpu.h"

namespace {
constexpr int kChains = 8;
constexpr int kIters = 4096;

// the base case's own instruction pattern: product-scanning (Comba) 8 x 8
// limb products per iteration on mad.lo.cc / madc.hi.cc / addc, as the
// schoolbook kernels issue them (ptxas: IMAD.WIDE.U32 with a carry-out
// predicate into the column pair + IADD3.X collecting two carries)
constexpr int kComba = 8;
__global__ void __launch_bounds__(256) k_probe(uint32_t seed, uint32_t* sink) {
    uint32_t a[kComba], b[kComba];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int j = 0; j < kComba; ++j) { a[j] = seed * (j + 3) + t; b[j] = (seed ^ t) * (2 * j + 1); }
    uint32_t sum = 0;
#pragma unroll 1
    for (int it = 0; it < kIters / kComba; ++it) {
        uint32_t c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
        for (int k = 0; k < 2 * kComba - 1; ++k) {
#pragma unroll
            for (int i = (k < kComba ? 0 : k - kComba + 1); i <= (k < kComba ? k : kComba - 1); ++i)
                asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
                             "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
                             "addc.u32 %2, %2, 0;"
                             : "+r"(c0), "+r"(c1), "+r"(c2) : "r"(a[i]), "r"(b[k - i]));
            sum ^= c0;
            c0 = c1; c1 = c2; c2 = 0;
        }
        sum += c0;
#pragma unroll
        for (int j = 0; j < kComba; ++j) a[j] += sum;   // next operands depend on this product
    }
    if (sum == 0x12345678u) sink[0] = sum;
}
// (written in C: ptxas turns `acc += (u64)a * b` into ONE IMAD.WIDE.U32 with a
// 64-bit accumulate, while inline `mad.wide.u32` asm was split into a zero-
// addend IMAD.WIDE + IADD3 + IMAD.X, three instructions per limb-product,
// which made the round-1 probe issue-bound at 20.7 LP/clk/SM instead of
// measuring the pipe; profiles/r02_probe_sass.txt.)  Two products per chain
// and iteration, 16 IMAD.WIDE per loop trip.
__global__ void __launch_bounds__(256) k_probe_wide(uint32_t seed, uint32_t* sink) {
    unsigned long long acc[kChains];
    uint32_t a[kChains];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int j = 0; j < kChains; ++j) { acc[j] = t + j; a[j] = seed * (j + 3) + t; }
    uint32_t b = seed ^ t, c = b * 7u;
#pragma unroll 1
    for (int it = 0; it < kIters / 2; ++it) {
#pragma unroll
        for (int j = 0; j < kChains; ++j) {
            acc[j] += (unsigned long long)a[j] * b;
            acc[j] += (unsigned long long)a[j] * c;
        }
        b += 0x9E3779B9u;
        c ^= b;
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
