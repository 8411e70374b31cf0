// pipe_rates.cuh -- microbenchmark for the roofline denominator of SURVEY 8(d):
// the sustained thread-level instruction rate of the DPX / integer pipes on every SM.
//
// Each thread runs 8 independent dependency chains of one instruction kind; 1024 threads per SM
// (2 CTAs of 512) keep every scheduler supplied.  The host times `iters` rounds of 8 x 32 chained
// instructions with CUDA events and divides.  clock64 deltas give the average SM clock.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace swb {

enum PipeOp : int {
    kOpViaddmnmx16 = 0,
    kOpVimnmx3_16 = 1,
    kOpViadd16 = 2,
    kOpViaddmnmx32 = 3,
    kOpPrmt = 4,
    kOpImad = 5,
    kOpMixAluFma = 6,
    kOpCount = 7
};

constexpr int kPipeChains = 8;
constexpr int kPipeUnroll = 32;

template <int OP>
__device__ __forceinline__ uint32_t pipe_step(uint32_t x, uint32_t c0, uint32_t c1) {
    if (OP == kOpViaddmnmx16) return __viaddmax_s16x2(x, c0, c1);
    if (OP == kOpVimnmx3_16) return __vimax3_s16x2_relu(x, c0, c1);
    if (OP == kOpViadd16) return __vadd2(x, c0);
    if (OP == kOpViaddmnmx32) return static_cast<uint32_t>(__viaddmax_s32(static_cast<int>(x), static_cast<int>(c0), static_cast<int>(c1)));
    if (OP == kOpPrmt) {
        uint32_t d;
        asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(c0), "r"(c1));
        return d;
    }
    // IMAD with a run-time multiplier so that ptxas cannot turn it into an add on the ALU pipe
    uint32_t d;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(c0), "r"(c1));
    return d;
}

template <int OP>
__global__ void __launch_bounds__(512, 2) pipe_rate_kernel(uint32_t* sink, unsigned long long* cycles,
                                                           uint32_t c0, uint32_t c1, int iters) {
    uint32_t x[kPipeChains];
#pragma unroll
    for (int i = 0; i < kPipeChains; ++i) x[i] = threadIdx.x * 2654435761u + i;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < kPipeUnroll; ++u) {
#pragma unroll
            for (int i = 0; i < kPipeChains; ++i) {
                if (OP == kOpMixAluFma) {
                    // even chains on the ALU/DPX pipe, odd chains on the FMA pipe
                    if (i & 1) x[i] = pipe_step<kOpImad>(x[i], c0 | 1u, c1);
                    else x[i] = pipe_step<kOpViaddmnmx16>(x[i], c0, c1);
                } else {
                    x[i] = pipe_step<OP>(x[i], c0, c1);
                }
            }
        }
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < kPipeChains; ++i) acc ^= x[i];
    if (acc == 0x12345678u) sink[0] = acc;   // keep the chains alive
    if (threadIdx.x == 0) atomicMax(cycles, static_cast<unsigned long long>(t1 - t0));
}

}  // namespace swb
