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

// What does a global store cost a lone warp?  Per iteration: 64 independent-ish DPX instructions (8 chains x 8) and
// `kStores` stores of 8 bytes per lane (256 B per warp, coalesced), to addresses that advance like a link buffer's.
enum StoreKind { kStWeak, kStStrong, kStCg, kStShared };
template <int KIND, int kStores>
__global__ void store_cost_kernel(unsigned long long* out, uint32_t* sink, long long* clocks, uint32_t a, uint32_t b, int iters) {
    __shared__ unsigned long long sm[8 * 32];
    uint32_t x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 2654435761u + i;
    unsigned long long* o = out + threadIdx.x;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = __viaddmax_s16x2(x[i], a, b);
#pragma unroll
        for (int r = 0; r < kStores; ++r) {
            const unsigned long long v = (static_cast<unsigned long long>(x[r & 7]) << 32) | x[(r + 1) & 7];
            if (KIND == kStWeak) o[r * 32] = v;
            if (KIND == kStStrong) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(o + r * 32), "l"(v));
            if (KIND == kStCg) asm volatile("st.global.cg.u64 [%0], %1;" ::"l"(o + r * 32), "l"(v));
            if (KIND == kStShared) sm[r * 32 + threadIdx.x] = v;
        }
        o += 8 * 32;
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= x[i];
    if (acc == 0x12345678u) sink[0] = acc + static_cast<uint32_t>(sm[threadIdx.x]);
    if (threadIdx.x == 0) clocks[0] = t1 - t0;
}

template <int KIND, int kStores>
void run_store(const char* name, unsigned long long* buf) {
    uint32_t* sink;
    long long* clocks;
    cudaMalloc(&sink, 64);
    cudaMalloc(&clocks, 8);
    const int iters = 4000;
    for (int rep = 0; rep < 2; ++rep) store_cost_kernel<KIND, kStores><<<1, 32>>>(buf, sink, clocks, 0xfffefffeu, 0x00030003u, iters);
    long long c = 0;
    cudaMemcpy(&c, clocks, 8, cudaMemcpyDeviceToHost);
    std::printf("64 DPX instr + %d %-22s stores per iteration: %7.1f clk per iteration\n", kStores, name, double(c) / iters);
    cudaFree(sink), cudaFree(clocks);
}

// Latency of ld.relaxed.gpu on lines another SM has just written (a link buffer's situation): CTA 0 fills `n` words of 8
// bytes per lane with st.relaxed.gpu and raises a flag; CTA 1 (another SM) then chases a dependent chain of loads
// through them; for comparison CTA 0 afterwards chases through its own lines.
__global__ void link_latency_kernel(unsigned long long* buf, uint32_t* flag, int n, long long* clocks) {
    const uint32_t lane = threadIdx.x;
    if (blockIdx.x == 0) {
        for (int i = 0; i < n; ++i) {
            const unsigned long long next = static_cast<unsigned long long>((i + 1) % n);
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(buf + static_cast<size_t>(i) * 32 + lane), "l"(next));
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(flag, 1u);
    }
    if (lane == 0) while (atomicAdd(flag, 0u) == 0u) __nanosleep(100);
    __syncwarp();
    if (blockIdx.x == 1) __nanosleep(2000);
    unsigned long long at = 0;
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(at) : "l"(buf + at * 32 + lane));
    const long long t1 = clock64();
    if (lane == 0) clocks[blockIdx.x] = (t1 - t0) + (at == 12345 ? 1 : 0);
}

// One warp (or `warps` warps, each its own copy) sweeps a narrow tile over n_chunks chunks: no producer, no consumer.
template <int T>
__global__ void __launch_bounds__(128, 1) narrow_kernel(WaveParams p, long long* clocks) {
    extern __shared__ __align__(128) uint8_t smem_prof[];
    const uint32_t n16 = kProfRows * p.pstride / 16;
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) reinterpret_cast<uint4*>(smem_prof)[i] = reinterpret_cast<const uint4*>(p.prof8)[i];
    __shared__ uint32_t consts[2];
    if (threadIdx.x == 0) consts[0] = p.neg_open2, consts[1] = p.neg_ext2;
    __syncthreads();
    NarrowWarp nw{consts};
    const GroupDesc gd = p.groups[0];
    const long long t0 = clock64();
    const uint32_t best = sweep_unit_narrow_s16<T, false>(p, reinterpret_cast<const int8_t*>(smem_prof), gd, 0, 1, nullptr, threadIdx.x & 31, nw);
    const long long t1 = clock64();
    if (best == 0x12345678u) p.slot_scores[0] = best;
    if ((threadIdx.x & 31) == 0) clocks[threadIdx.x >> 5] = t1 - t0;
}

// A chain of n_tiles narrow tiles, one warp per CTA (= per SM), handing rows over through link buffers in global memory.
template <int T>
__global__ void __launch_bounds__(128, 1) narrow_chain_kernel(WaveParams p, uint8_t* links, uint32_t n_tiles, long long* clocks) {
    extern __shared__ __align__(128) uint8_t smem_prof[];
    const uint32_t n16 = kProfRows * p.pstride / 16;
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) reinterpret_cast<uint4*>(smem_prof)[i] = reinterpret_cast<const uint4*>(p.prof8)[i];
    __shared__ uint32_t consts[2];
    if (threadIdx.x == 0) consts[0] = p.neg_open2, consts[1] = p.neg_ext2;
    __syncthreads();
    NarrowWarp nw{consts};
    const GroupDesc gd = p.groups[0];
    const uint32_t tile = blockIdx.x;
    const long long t0 = clock64();
    const uint32_t best = sweep_unit_narrow_s16<T, false>(p, reinterpret_cast<const int8_t*>(smem_prof), gd, tile, n_tiles, links, threadIdx.x & 31, nw);
    const long long t1 = clock64();
    if (best == 0x12345678u) p.slot_scores[0] = best;
    if ((threadIdx.x & 31) == 0) clocks[blockIdx.x] = t1 - t0;
}

// The same chain with a helper warp per tile (warp 4, the compute warp's scheduler): rings in shared memory.
template <int T>
__global__ void __launch_bounds__(256, 1) narrow_helper_chain_kernel(WaveParams p, uint8_t* links, uint32_t n_tiles, long long* clocks) {
    extern __shared__ __align__(128) uint8_t smem_prof[];
    const uint32_t n16 = kProfRows * p.pstride / 16;
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) reinterpret_cast<uint4*>(smem_prof)[i] = reinterpret_cast<const uint4*>(p.prof8)[i];
    __shared__ uint32_t consts[2];
    if (threadIdx.x == 0) consts[0] = p.neg_open2, consts[1] = p.neg_ext2;
    const uint32_t stage = smem_u32(smem_prof) + 4096;
    for (uint32_t i = threadIdx.x; i < kNarrowPairBytes / 16; i += blockDim.x)
        sts128v(stage + i * 16, make_uint4(kNarrowEmptyWord, kNarrowEmptyWord, kNarrowEmptyWord, kNarrowEmptyWord));
    __syncthreads();
    NarrowWarp nw{consts};
    nw.in_ring = stage, nw.out_ring = stage + kNarrowRingSlots * kNarrowChunkBytes;
    const GroupDesc gd = p.groups[0];
    const uint32_t tile = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 4) narrow_helper_unit(links, gd.n_chunks, tile, n_tiles, lane, nw);
    if (warp != 0) return;
    const long long t0 = clock64();
    const uint32_t best = sweep_unit_narrow_s16<T, true>(p, reinterpret_cast<const int8_t*>(smem_prof), gd, tile, n_tiles, links, lane, nw);
    const long long t1 = clock64();
    if (best == 0x12345678u) p.slot_scores[0] = best;
    if (lane == 0) clocks[blockIdx.x] = t1 - t0;
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

    {
        unsigned long long* buf;
        cudaMalloc(&buf, 4000ull * 8 * 32 * 8 + 4096);
        run_store<kStWeak, 0>("(none)", buf);
        run_store<kStWeak, 1>("weak global", buf);
        run_store<kStWeak, 4>("weak global", buf);
        run_store<kStWeak, 8>("weak global", buf);
        run_store<kStStrong, 8>("st.relaxed.gpu", buf);
        run_store<kStCg, 8>("st.global.cg", buf);
        run_store<kStShared, 8>("shared", buf);
        cudaFree(buf);
    }
    {
        unsigned long long* buf;
        uint32_t* flag;
        long long* d_c;
        const int n = 4096;
        cudaMalloc(&buf, static_cast<size_t>(n) * 32 * 8);
        cudaMalloc(&flag, 4);
        cudaMalloc(&d_c, 16 * 8);
        cudaFuncSetAttribute(link_latency_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 << 10);
        for (int grid : {2, 8, 75, 148}) {   // the reader is always CTA 1; more CTAs only spread the placement
            cudaMemset(flag, 0, 4);
            link_latency_kernel<<<grid, 32, 120 << 10>>>(buf, flag, n, d_c);
            long long c[2] = {};
            cudaMemcpy(c, d_c, sizeof(c), cudaMemcpyDeviceToHost);
            std::printf("ld.relaxed.gpu latency (grid %3d): lines written by this SM %6.1f clk, by another SM %6.1f clk\n", grid, double(c[0]) / n,
                        double(c[1]) / n);
        }
        cudaFree(buf), cudaFree(flag), cudaFree(d_c);
    }
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
    for (int warps : {1, 4}) {
        long long c[16] = {};
        for (int rep = 0; rep < 2; ++rep) narrow_kernel<8><<<1, 32 * warps, kProfRows * pstride>>>(p, d_clocks);
        cudaMemcpy(c, d_clocks, sizeof(c), cudaMemcpyDeviceToHost);
        std::printf("narrow 8x8 block sweep, %2d warps on the SM: %7.1f clk per chunk (%.1f per row)\n", warps, double(c[0]) / n_chunks,
                    double(c[0]) / n_chunks / 8);
        for (int rep = 0; rep < 2; ++rep) narrow_kernel<4><<<1, 32 * warps, kProfRows * pstride>>>(p, d_clocks);
        cudaMemcpy(c, d_clocks, sizeof(c), cudaMemcpyDeviceToHost);
        std::printf("narrow 8x4 block sweep, %2d warps on the SM: %7.1f clk per chunk (%.1f per row)\n", warps, double(c[0]) / n_chunks,
                    double(c[0]) / n_chunks / 8);
        for (int rep = 0; rep < 2; ++rep) wide_kernel<<<1, 32 * warps, kProfRows * pstride>>>(p, d_clocks);
        cudaMemcpy(c, d_clocks, sizeof(c), cudaMemcpyDeviceToHost);
        std::printf("32-column sweep,        %2d warps on the SM: %7.1f clk per chunk (%.1f per row)\n", warps, double(c[0]) / n_chunks,
                    double(c[0]) / n_chunks / 8);
    }
    {
        // chains of tiles over link buffers: tile 0 alone with its stores (nobody reads), then 2, 8 and 36 tiles
        const uint32_t max_tiles = 36;
        uint8_t* d_links;
        const size_t link_bytes = static_cast<size_t>(max_tiles) * n_chunks * kNarrowChunkBytes;
        cudaMalloc(&d_links, link_bytes);
        long long* d_c;
        cudaMalloc(&d_c, 64 * 8);
        cudaFuncSetAttribute(narrow_chain_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 << 10);
        cudaFuncSetAttribute(narrow_chain_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 << 10);
        for (uint32_t tiles : {1u, 2u, 8u, 36u}) {
            for (int t = 0; t < 2; ++t) {
                long long c[64] = {};
                cudaMemset(d_links, 0x80, link_bytes);
                // tiles == 1: the producer writes into link 0 and nobody consumes (n_tiles = 2, grid 1); 120 KB of dynamic
                // shared memory: one CTA per SM
                const uint32_t n_tiles = tiles == 1 ? 2 : tiles, grid = tiles == 1 ? 1 : tiles;
                if (t == 0) narrow_chain_kernel<8><<<grid, 32, 120 << 10>>>(p, d_links, n_tiles, d_c);
                else narrow_chain_kernel<4><<<grid, 32, 120 << 10>>>(p, d_links, n_tiles, d_c);
                cudaMemcpy(c, d_c, sizeof(c), cudaMemcpyDeviceToHost);
                std::printf("chain of %2u narrow tiles (T=%d): clk per chunk of tile 0 %7.1f, tile 1 %7.1f, last tile %7.1f  %s\n", tiles, t == 0 ? 8 : 4,
                            double(c[0]) / n_chunks, double(c[grid > 1 ? 1 : 0]) / n_chunks, double(c[grid - 1]) / n_chunks,
                            cudaGetErrorString(cudaGetLastError()));
                cudaMemset(d_links, 0x80, link_bytes);
                cudaFuncSetAttribute(narrow_helper_chain_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 << 10);
                cudaFuncSetAttribute(narrow_helper_chain_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 << 10);
                if (t == 0) narrow_helper_chain_kernel<8><<<grid, 160, 120 << 10>>>(p, d_links, n_tiles, d_c);
                else narrow_helper_chain_kernel<4><<<grid, 160, 120 << 10>>>(p, d_links, n_tiles, d_c);
                cudaMemcpy(c, d_c, sizeof(c), cudaMemcpyDeviceToHost);
                std::printf("   with helper warps             : clk per chunk of tile 0 %7.1f, tile 1 %7.1f, last tile %7.1f  %s\n",
                            double(c[0]) / n_chunks, double(c[grid > 1 ? 1 : 0]) / n_chunks, double(c[grid - 1]) / n_chunks,
                            cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
