// tools/lat_probe.cu -- what bounds ONE warp on sm_100a?  Dependent-issue latency of the DPX instructions of the
// recurrence, the issue rate of a single warp with K independent chains, and the clocks per chunk of the narrow
// 8 x 8 block sweep (kernels.cuh: sweep_unit_narrow_s16) run by one warp alone on an SM with no global hand-off.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2203_11100_b200/csrc tools/lat_probe.cu -o /tmp/lat_probe
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "kernels.cuh"

using namespace swb;

enum Op { kAddMax, kMax3, kAdd, kTriple };

template <int OP, int K>
__global__ void chain_kernel(uint32_t* sink, long long* clocks, uint32_t a, uint32_t b, int iters) {
    uint32_t x[K];
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = threadIdx.x * 2654435761u + i;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 32; ++u) {
#pragma unroll
            for (int i = 0; i < K; ++i) {
                if (OP == kAddMax) x[i] = __viaddmax_s16x2(x[i], a, b);
                if (OP == kMax3) x[i] = __vimax3_s16x2_relu(x[i], a, b);
                if (OP == kAdd) x[i] = __vadd2(x[i], a);
                if (OP == kTriple) {   // E -> H -> Hm: the chain of one cell
                    const uint32_t e = __viaddmax_s16x2(b, a, x[i]);
                    const uint32_t h = __vimax3_s16x2_relu(e, a, b);
                    x[i] = __vadd2(h, a);
                }
            }
        }
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) acc ^= x[i];
    if (acc == 0x12345678u) sink[0] = acc;
    if (threadIdx.x == 0) clocks[blockIdx.x] = t1 - t0;
}

template <int OP, int K>
void run_chain(const char* name, int warps) {
    uint32_t* sink;
    long long* clocks;
    cudaMalloc(&sink, 64);
    cudaMalloc(&clocks, 8);
    const int iters = 2000;
    chain_kernel<OP, K><<<1, 32 * warps>>>(sink, clocks, 0xfffefffeu, 0x00030003u, iters);
    chain_kernel<OP, K><<<1, 32 * warps>>>(sink, clocks, 0xfffefffeu, 0x00030003u, iters);
    long long c = 0;
    cudaMemcpy(&c, clocks, 8, cudaMemcpyDeviceToHost);
    const double n = double(iters) * 32 * K * (OP == kTriple ? 3 : 1);
    std::printf("%-10s chains=%d warps/SM=%2d : %6.2f clk per instruction of a warp (%.2f per chain step)\n", name, K, warps, c / n,
                c / (double(iters) * 32));
    cudaFree(sink), cudaFree(clocks);
}

// One warp (or `warps` warps, each its own copy) sweeps a narrow tile over n_chunks chunks: no producer, no consumer.
__global__ void __launch_bounds__(512, 1) narrow_kernel(WaveParams p, long long* clocks) {
    extern __shared__ __align__(16) uint8_t smem_prof[];
    const uint32_t n16 = kProfRows * p.pstride / 16;
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) reinterpret_cast<uint4*>(smem_prof)[i] = reinterpret_cast<const uint4*>(p.prof8)[i];
    __syncthreads();
    const GroupDesc gd = p.groups[0];
    const long long t0 = clock64();
    const uint32_t best = sweep_unit_narrow_s16(p, reinterpret_cast<const int8_t*>(smem_prof), gd, 0, 1, nullptr, nullptr, threadIdx.x & 31);
    const long long t1 = clock64();
    if (best == 0x12345678u) p.slot_scores[0] = best;
    if ((threadIdx.x & 31) == 0) clocks[threadIdx.x >> 5] = t1 - t0;
}

__global__ void __launch_bounds__(512, 1) wide_kernel(WaveParams p, long long* clocks) {
    extern __shared__ __align__(16) uint8_t smem_prof[];
    const uint32_t n16 = kProfRows * p.pstride / 16;
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) reinterpret_cast<uint4*>(smem_prof)[i] = reinterpret_cast<const uint4*>(p.prof8)[i];
    __syncthreads();
    const GroupDesc gd = p.groups[0];
    const long long t0 = clock64();
    const uint32_t best = sweep_unit_s16<32, 2, 1, false>(p, reinterpret_cast<const int8_t*>(smem_prof), gd, 0, 1, 1, nullptr, nullptr, threadIdx.x & 31, 0,
                                                           gd.n_chunks, nullptr);
    const long long t1 = clock64();
    if (best == 0x12345678u) p.slot_scores[0] = best;
    if ((threadIdx.x & 31) == 0) clocks[threadIdx.x >> 5] = t1 - t0;
}

int main() {
    run_chain<kAddMax, 1>("VIADDMNMX", 1);
    run_chain<kMax3, 1>("VIMNMX3", 1);
    run_chain<kAdd, 1>("VIADD.16x2", 1);
    run_chain<kTriple, 1>("E->H->Hm", 1);
    run_chain<kTriple, 2>("E->H->Hm", 1);
    run_chain<kTriple, 4>("E->H->Hm", 1);
    run_chain<kTriple, 8>("E->H->Hm", 1);
    run_chain<kAddMax, 2>("VIADDMNMX", 1);
    run_chain<kAddMax, 4>("VIADDMNMX", 1);
    run_chain<kAddMax, 8>("VIADDMNMX", 1);
    run_chain<kAddMax, 8>("VIADDMNMX", 4);
    run_chain<kAddMax, 8>("VIADDMNMX", 8);
    run_chain<kAddMax, 8>("VIADDMNMX", 16);
    run_chain<kAdd, 8>("VIADD.16x2", 1);
    run_chain<kAdd, 8>("VIADD.16x2", 4);

    // the narrow sweep
    const uint32_t n_chunks = 2000;
    std::vector<uint8_t> codes(static_cast<size_t>(n_chunks) * 512);
    for (size_t i = 0; i < codes.size(); ++i) codes[i] = static_cast<uint8_t>((i * 2654435761u >> 13) % 20);
    const uint32_t pstride = 48;   // 32 columns + 16
    std::vector<int8_t> prof(kProfRows * pstride);
    for (size_t i = 0; i < prof.size(); ++i) prof[i] = static_cast<int8_t>(10 + static_cast<int>((i * 40503u >> 7) % 15) - 4);
    GroupDesc gd{};
    gd.chunk_base = 0, gd.n_chunks = n_chunks, gd.first_slot = 0;
    uint8_t* d_codes;
    int8_t* d_prof;
    GroupDesc* d_gd;
    int32_t* d_scores;
    long long* d_clocks;
    cudaMalloc(&d_codes, codes.size());
    cudaMalloc(&d_prof, prof.size());
    cudaMalloc(&d_gd, sizeof(gd));
    cudaMalloc(&d_scores, 256);
    cudaMalloc(&d_clocks, 16 * 8);
    cudaMemcpy(d_codes, codes.data(), codes.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_prof, prof.data(), prof.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_gd, &gd, sizeof(gd), cudaMemcpyHostToDevice);
    WaveParams p{};
    p.codes = reinterpret_cast<const uint4*>(d_codes);
    p.groups = d_gd;
    p.n_groups = 1;
    p.prof8 = d_prof;
    p.pstride = pstride;
    p.n_tiles = 1, p.n_tiles_narrow = 1;
    p.slot_scores = d_scores;
    p.neg_open2 = 0xfff6fff6u, p.neg_ext2 = 0xfffefffeu;
    for (int warps : {1, 4, 8, 16}) {
        long long c[16] = {};
        for (int rep = 0; rep < 2; ++rep) narrow_kernel<<<1, 32 * warps, kProfRows * pstride>>>(p, d_clocks);
        cudaMemcpy(c, d_clocks, sizeof(c), cudaMemcpyDeviceToHost);
        std::printf("narrow 8x8 block sweep, %2d warps on the SM: %7.1f clk per chunk (%.1f per row)\n", warps, double(c[0]) / n_chunks,
                    double(c[0]) / n_chunks / 8);
        for (int rep = 0; rep < 2; ++rep) wide_kernel<<<1, 32 * warps, kProfRows * pstride>>>(p, d_clocks);
        cudaMemcpy(c, d_clocks, sizeof(c), cudaMemcpyDeviceToHost);
        std::printf("32-column sweep,        %2d warps on the SM: %7.1f clk per chunk (%.1f per row)\n", warps, double(c[0]) / n_chunks,
                    double(c[0]) / n_chunks / 8);
    }
    std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
