// kernels.cuh -- hand-written sm_100a kernels of the SW#db scoring path.
//
// All kernels compute the recurrence of the reference's detail::local_score_rows
// (align.hpp:42-64) in a shifted but algebraically identical form:
//
//   stored per cell:  Hm = H - open            (so both uses of "H - open" are free)
//   profile entries:  sub' = M[s][q] + open    (so diag + sub = Hm_diag + sub')
//   E (reference gap_h, along the query), F (reference gap_v, along the subject), and the
//   boundaries H = 0, gap = -inf become Hm = -open, E = F = -open: the first real cell then gets
//   max(0 - open, -open - extend) = -open, the value the reference's -inf sentinel yields
//   (align.hpp:51-55).  Nothing can drop below -open - extend, so nothing wraps on the low side.
//
//   per cell:   E  = max(E - ext, Hm_left)            VIADDMNMX        (__viaddmax)
//               F  = max(F - ext, Hm_up)              VIADDMNMX
//               H  = max(0, Hm_diag + sub', E, F)     VIADDMNMX.RELU + VIMNMX.RELU
//               Hm = H - open                         VIADD
//               best = max(best, H)                   VIMNMX3 per two cells
//
// Padding (rows past a sequence's end, columns past the query's end, lanes with no sequence) uses
// substitution score 0: every padded cell is bounded by an earlier real cell, so `best` is
// unaffected, and a pad row applied to the initial state leaves it unchanged.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "pack.hpp"
#include "scan_plan.hpp"

namespace swb {

constexpr int kProfRows = 25;        // 24 symbols + the pad row
#ifndef SWB_INTER_TILE
#define SWB_INTER_TILE 32
#endif
#ifndef SWB_INTER_THREADS
#define SWB_INTER_THREADS 512
#endif
constexpr int kInterTile = SWB_INTER_TILE;        // query columns held in registers per pass (multiple of 8)
constexpr int kInterThreads = SWB_INTER_THREADS;  // persistent CTA: 16 warps, four per SMSP
constexpr int kNarrowThreads = 128;               // wavefront CTAs of narrow units next to the pipeline: one warp per SMSP
constexpr int kIntraDelta = 64;      // step offset between neighbouring warps of an intra-task CTA
constexpr int kIntraRing = 128;      // rows of border ring buffer between neighbouring warps
constexpr int kIntraMaxWarps = 8;

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// ------------------------------------------------------------------------------------------------
// Query profile (scoring.hpp:199-215 restated for the device layouts).
//   prof8  [25][pstride]            int8   sub' for the inter-task kernels, column-contiguous
//   prof8i [25][n_lane_tiles][8]    int8   the same, re-tiled so that an intra-task lane's T<=8
//                                          columns are one aligned 8-byte word
//   prof32 / prof32i                int32  the wide variants (matrices that do not fit int8)
// ------------------------------------------------------------------------------------------------
struct ProfileParams {
    const uint8_t* query;    // m codes
    const int32_t* matrix;   // 24x24, [subject*24 + query]
    uint32_t m;
    int32_t shift_main;      // added to every entry of prof8 (open for the s16 kernel, c for the u16 kernel)
    int32_t shift_intra;     // added to every entry of prof8i / prof32i (open)
    uint32_t pstride;        // bytes (int8) / elements (int32) per row of the column-contiguous form
    uint32_t intra_t;        // columns per lane in the intra-task kernel (<= 8)
    uint32_t n_lane_tiles;   // number of 8-slot words per row of the re-tiled form
    int8_t* prof8;
    int8_t* prof8i;
    int32_t* prof32;
    int32_t* prof32i;
};

__global__ void build_profile_kernel(ProfileParams p) {
    const uint32_t per_row = p.pstride;
    const uint32_t total = kProfRows * per_row;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t s = i / per_row, j = i % per_row;
        int32_t v = p.shift_main;  // pad row / pad column: substitution 0
        if (s < kAlphabet && j < p.m) v = p.matrix[s * kAlphabet + p.query[j]] + p.shift_main;
        if (p.prof8) p.prof8[i] = static_cast<int8_t>(v);
        if (p.prof32) p.prof32[i] = v;
    }
    const uint32_t per_row_i = p.n_lane_tiles * 8;
    const uint32_t total_i = kProfRows * per_row_i;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total_i; i += gridDim.x * blockDim.x) {
        const uint32_t s = i / per_row_i, rem = i % per_row_i;
        const uint32_t tile = rem / 8, k = rem % 8;
        const uint32_t j = tile * p.intra_t + k;
        int32_t v = p.shift_intra;
        if (s < kAlphabet && k < p.intra_t && j < p.m) v = p.matrix[s * kAlphabet + p.query[j]] + p.shift_intra;
        if (p.prof8i) p.prof8i[i] = static_cast<int8_t>(v);
        if (p.prof32i) p.prof32i[i] = v;
    }
}

// ------------------------------------------------------------------------------------------------
// The hot kernel: packed-int16 DPX tile-wavefront over interleaved groups.
//
// Work decomposition.  A group (64 sequences, R padded rows) times the query's n_tiles tiles of 32
// columns is cut into units of consecutive tiles: tiles_per_unit = clamp(unit_target / R, 1,
// n_tiles), so short groups are one unit (pure inter-task: one warp scores 64 sequences end to
// end) while a long group becomes up to n_tiles units that different warps -- on any SM -- work on
// at the same time, each one tile (stripe) behind its left neighbour: the anti-diagonal wavefront
// of the reference's intra-task kernel (align.hpp:194-226) at warp granularity.  Units are handed
// out by one global ticket counter in (group, tile) order with groups sorted longest first, so a
// unit's left neighbour always holds an earlier ticket and is already running: waiting on it
// cannot deadlock, and the longest groups start first (LPT).
//
// Data flow.  Each thread carries two sequences in the int16 halves of every DPX word and keeps
// Hm and F of its 32 columns in registers.  The (Hm, E) of a tile's last column goes, row by row,
// through a database-shaped border array (8 B per row per thread, coalesced, double-buffered by
// tile parity, L2-resident between neighbouring units).  A unit publishes the rows completed in
// its last tile after every chunk of 8 rows (fence + store); the unit to its right polls that
// counter before the chunk's first border load.  Border loads bypass L1 (ld.global.cg) because the
// producer may sit on another SM.  The int8 profile lives in shared memory with a row stride of
// 16 (mod 128) bytes so that the 25 rows spread over the banks.
//
// Exactness.  Additions wrap (VIADD.16x2 / VIADDMNMX do not saturate), so a lane is trusted only
// if its best never exceeded limit = 32767 - max(matrix): H grows by at most max(matrix) per step,
// hence no wrap can precede a value above the limit.  Scores above the limit are re-run in int32
// by the intra-task kernel below -- the reference's contract for saturated lanes
// (align.hpp:149-153).
// ------------------------------------------------------------------------------------------------
struct WaveParams {
    const uint4* codes;
    const GroupDesc* groups;
    uint32_t n_groups;
    const uint32_t* unit_start;   // [n_groups + 1] first unit of each group
    const uint8_t* group_mode;    // [n_groups] GroupMode
    const uint32_t* vstate_off;   // [n_groups] first vstate slot of a kGroupRowBlock group (slots of one tile each)
    uint4* vstate;                // register-state hand-over between row blocks
    uint32_t n_units;
    uint32_t n_tiles_narrow;      // ceil(m / narrow_tile): tiles of a kGroupNarrow group
    const int8_t* prof8;
    uint32_t pstride;
    uint32_t n_tiles;             // ceil(m / T)
    uint2* border0;
    uint2* border1;
    int32_t* slot_scores;         // [n_groups*64], zeroed per search, updated with atomicMax
    uint32_t* progress;           // [n_units], zeroed per search
    uint32_t* ticket;
    uint32_t neg_open2;           // (-open, -open) packed
    uint32_t neg_ext2;            // (-extend, -extend) packed
    // narrow units only (behind the fields every variant reads: ptxas's allocation of the plain sweep proved sensitive
    // even to the parameter layout)
    uint32_t narrow_tile;         // 8 or 4 columns
    uint32_t narrow_staged;       // 1: narrow units hand over through link buffers of their own (short queries);
                                  // 0: through the border arrays like every other tile (deep wavefronts: many narrow tiles)
    uint32_t narrow_helpers;      // 1: CTAs of 8 warps, warps 0-3 take units, warps 4-7 carry their narrow units' blocks between the
                                  // link buffers and rings in shared memory (narrow_stage_off: where those start)
    uint32_t narrow_stage_off;
    uint8_t* nlinks;              // link buffers of the narrow groups (vstate_off[g]: first row slot, 256 B each, of group g's links)
};

// A group is either one unit (all tiles, one warp) or n_tiles units (one tile each, a wavefront of
// cooperating warps); the host decides per search (unit_budget in cabi.cu) and the kernel reads the
// decision back from unit_start.

// Cross-CTA hand-off through a progress counter (PTX memory model, scope .gpu).
//   producer: its 32 lanes store the guarded rows (weak stores), __syncwarp, then lane 0 publishes the counter with
//             st.release.gpu -- cumulative over the other lanes' stores through the barrier.
//   consumer: polls with ld.relaxed.gpu (an acquire load makes ptxas emit CCTL.IVALL, an L1 invalidate, per poll:
//             4.6 % of all stall samples when every poll was an acquire) and, once the wanted value has been seen,
//             reads the counter ONE more time with ld.acquire.gpu.  The counter only grows, so that load observes
//             the same or a later release: release -> acquire synchronises, and every later load of the guarded rows
//             (by lane 0 in program order, by the other lanes after the __syncwarp that follows) happens after the
//             producer's stores.  One acquire per completed wait, none per poll.
__device__ __forceinline__ uint32_t ld_poll(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Wait until *p >= need; returns an acquired value (>= need).  Called by one lane; the caller follows with __syncwarp.
__device__ __forceinline__ uint32_t wait_progress(const uint32_t* p, uint32_t need) {
    while (ld_poll(p) < need) __nanosleep(64);
    return ld_acquire_gpu(p);
}

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One unit: tiles [t0, t1) of `n_tiles` tiles of width T over all rows of group `gd`.
//   dep  progress counter of the unit to the left (nullptr: none), pub: this unit's counter (nullptr: no consumer)
//   D    border look-ahead in rows (a power of two <= 8), P: publish progress every P chunks
//   kRowBlock  the unit is a block of rows [chunk_lo, chunk_hi) swept over ALL tiles; the register state (Hm, F of
//        the 32 columns, plus the corner value) of every tile is handed from the block above through `vstate`
//        (one slot of kVStateWords x 32 lanes per tile), and dep / pub count completed TILES instead of rows.
constexpr uint32_t kVStateWords = 2 * kInterTile + 4;   // Hm + F of the tile's columns, the corner, padded to uint4

template <int T, int D, int P, bool kRowBlock>
__device__ __forceinline__ uint32_t sweep_unit_s16(const WaveParams& p, const int8_t* prof, const GroupDesc& gd,
                                                   uint32_t t0, uint32_t t1, uint32_t n_tiles, const uint32_t* dep,
                                                   uint32_t* pub, uint32_t lane, uint32_t chunk_lo, uint32_t chunk_hi,
                                                   uint4* vstate) {
    static_assert(T % 8 == 0, "tile width must be a multiple of 8 columns");
    static_assert(!kRowBlock || T == kInterTile, "row blocks hand over exactly kInterTile columns of state");
    const uint32_t NO = p.neg_open2, NE = p.neg_ext2;
    const uint32_t rows = chunk_hi * kRowsPerChunk;     // one past the last row this unit touches
    const uint4* gcodes = p.codes + gd.chunk_base * 32 + lane;
    const size_t brow0 = static_cast<size_t>(gd.chunk_base) * kRowsPerChunk * 32 + lane;
    uint32_t best = 0;

    for (uint32_t tile = t0; tile < t1; ++tile) {
        const int8_t* ptile = prof + tile * T;
        const bool first = tile == 0, last = tile + 1 == n_tiles;
        const bool wait = !kRowBlock && dep != nullptr && tile == t0;
        const bool publish = !kRowBlock && pub != nullptr && tile + 1 == t1;
        const uint2* bin = ((tile & 1) ? p.border0 : p.border1) + brow0;
        uint2* bout = ((tile & 1) ? p.border1 : p.border0) + brow0;

        uint32_t Hm[T], F[T];
        uint32_t diag_in = NO;
        if (kRowBlock && dep != nullptr) {
            // the block above must have finished this tile; then take over its register state
            if (lane == 0) wait_progress(dep, tile + 1);
            __syncwarp();
            const uint4* slot = vstate + static_cast<size_t>(tile) * (kVStateWords / 4) * 32 + lane;
#pragma unroll
            for (int i = 0; i < T / 4; ++i) {
                const uint4 a = __ldcg(slot + i * 32), b = __ldcg(slot + (T / 4 + i) * 32);
                Hm[4 * i] = a.x, Hm[4 * i + 1] = a.y, Hm[4 * i + 2] = a.z, Hm[4 * i + 3] = a.w;
                F[4 * i] = b.x, F[4 * i + 1] = b.y, F[4 * i + 2] = b.z, F[4 * i + 3] = b.w;
            }
            diag_in = __ldcg(slot + (2 * T / 4) * 32).x;
        } else {
#pragma unroll
            for (int k = 0; k < T; ++k) Hm[k] = NO, F[k] = NO;
        }
        uint4 cw = chunk_lo < chunk_hi ? __ldg(gcodes + static_cast<size_t>(chunk_lo) * 32) : make_uint4(0, 0, 0, 0);
        // inbound border rows are fetched D rows ahead of their use (q[i]: row = i mod D); a waiting tile stays
        // far enough behind its producer that this look-ahead never reads an unpublished row
        uint2 q[D];
#pragma unroll
        for (int i = 0; i < D; ++i) q[i] = make_uint2(NO, NO);
        uint32_t known = 0;   // producer progress observed so far

        for (uint32_t chunk = chunk_lo; chunk < chunk_hi; ++chunk) {
            const uint4 cur = cw;
            if (chunk + 1 < chunk_hi) cw = __ldg(gcodes + static_cast<size_t>(chunk + 1) * 32);
            const size_t row0 = static_cast<size_t>(chunk) * kRowsPerChunk;
            if (wait) {
                const uint32_t need = min(rows, static_cast<uint32_t>(row0) + kRowsPerChunk + D);
                if (P == 1) {          // the producer publishes every chunk: poll every chunk, keep no state
                    if (lane == 0) wait_progress(dep, need);
                    __syncwarp();
                } else if (known < need) {
                    if (lane == 0) known = wait_progress(dep, need);
                    known = __shfl_sync(0xffffffffu, known, 0);
                }
            }
            if (!first && chunk == chunk_lo) {
#pragma unroll
                for (int i = 0; i < D; ++i) q[i] = __ldcg(bin + (row0 + i) * 32);   // a chunk has 8 >= D rows
            }
#pragma unroll
            for (int r = 0; r < static_cast<int>(kRowsPerChunk); ++r) {
                const uint32_t wa = r < 4 ? cur.x : cur.y;
                const uint32_t wb = r < 4 ? cur.z : cur.w;
                const uint32_t a1 = (wa >> (8 * (r & 3))) & 0xffu;
                const uint32_t a2 = (wb >> (8 * (r & 3))) & 0xffu;
                const int8_t* pa = ptile + a1 * p.pstride;
                const int8_t* pb = ptile + a2 * p.pstride;
                uint32_t wA[T / 4], wB[T / 4];
                if (T % 16 == 0) {
#pragma unroll
                    for (int i = 0; i < T / 16; ++i) {
                        const uint4 va = reinterpret_cast<const uint4*>(pa)[i], vb = reinterpret_cast<const uint4*>(pb)[i];
                        wA[4 * i] = va.x, wA[4 * i + 1] = va.y, wA[4 * i + 2] = va.z, wA[4 * i + 3] = va.w;
                        wB[4 * i] = vb.x, wB[4 * i + 1] = vb.y, wB[4 * i + 2] = vb.z, wB[4 * i + 3] = vb.w;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < T / 8; ++i) {
                        const uint2 va = reinterpret_cast<const uint2*>(pa)[i], vb = reinterpret_cast<const uint2*>(pb)[i];
                        wA[2 * i] = va.x, wA[2 * i + 1] = va.y;
                        wB[2 * i] = vb.x, wB[2 * i + 1] = vb.y;
                    }
                }
                const size_t row = row0 + r;
                const uint2 bi = q[r % D];
                if (!first && row + D < rows) q[r % D] = __ldcg(bin + (row + D) * 32);
                uint32_t hl = bi.x;   // Hm of the column left of the tile, this row
                uint32_t E = bi.y;
                uint32_t diag = diag_in;
                diag_in = hl;
#pragma unroll
                for (int k = 0; k < T; k += 2) {
                    const uint32_t s0 = prmt(wA[k / 4], wB[k / 4], (k & 3) == 0 ? 0xC480u : 0xE6A2u);
                    const uint32_t s1 = prmt(wA[k / 4], wB[k / 4], (k & 3) == 0 ? 0xD591u : 0xF7B3u);
                    // cell k
                    E = __viaddmax_s16x2(E, NE, hl);
                    F[k] = __viaddmax_s16x2(F[k], NE, Hm[k]);
                    const uint32_t d0 = __vadd2(diag, s0);
                    const uint32_t h0 = __vimax3_s16x2_relu(d0, E, F[k]);
                    diag = Hm[k];
                    hl = __vadd2(h0, NO);
                    Hm[k] = hl;
                    // cell k+1
                    E = __viaddmax_s16x2(E, NE, hl);
                    F[k + 1] = __viaddmax_s16x2(F[k + 1], NE, Hm[k + 1]);
                    const uint32_t d1 = __vadd2(diag, s1);
                    const uint32_t h1 = __vimax3_s16x2_relu(d1, E, F[k + 1]);
                    diag = Hm[k + 1];
                    hl = __vadd2(h1, NO);
                    Hm[k + 1] = hl;
                    // The running maximum is taken over the diagonal terms d, not over H: a cell whose H comes
                    // from E or F is dominated by an earlier cell (gaps only subtract), so max(H) == max(0, max(d)).
                    // Giving d this second use also makes the compiler keep the packed add as VIADD.16x2 (FMA
                    // pipe) + one VIMNMX3 instead of VIADDMNMX + VIMNMX (two ALU-pipe instructions).
                    best = __vimax3_s16x2(best, d0, d1);
                }
                if (!last) bout[row * 32] = make_uint2(hl, E);
            }
            if (publish && ((chunk + 1) % P == 0 || chunk + 1 == chunk_hi)) {
                __syncwarp();
                if (lane == 0) st_release(pub, static_cast<uint32_t>(row0) + kRowsPerChunk);
            }
        }
        if (kRowBlock && pub != nullptr) {
            // hand this tile's register state to the block below, then count the tile as done
            uint4* slot = vstate + static_cast<size_t>(tile) * (kVStateWords / 4) * 32 + lane;
#pragma unroll
            for (int i = 0; i < T / 4; ++i) {
                slot[i * 32] = make_uint4(Hm[4 * i], Hm[4 * i + 1], Hm[4 * i + 2], Hm[4 * i + 3]);
                slot[(T / 4 + i) * 32] = make_uint4(F[4 * i], F[4 * i + 1], F[4 * i + 2], F[4 * i + 3]);
            }
            slot[(2 * T / 4) * 32] = make_uint4(diag_in, 0, 0, 0);
            __syncwarp();
            if (lane == 0) st_release(pub, tile + 1);
        }
    }
    return best;
}

// Narrow units (kGroupNarrow): one tile of T = 8 or 4 columns over all rows of a very tall group, for searches whose
// duration is bounded by that group's chain of rows (short query, 35,213-residue sequence).  A block of 8 rows x T
// columns is swept in ANTI-DIAGONAL order: cell (r, c) needs (r-1, c), (r, c-1) and (r-1, c-1), all on the two previous
// anti-diagonals, so the cells of an anti-diagonal are independent and a block's dependent chain is 8 + T - 1 cell steps
// instead of 8 T (the reference's intra-task schedule, align.hpp:194-226, inside one thread).  Everything is unrolled:
// Hm and F live per column, E and the left neighbour's Hm per row, and d[r] holds the diagonal term of row r's next cell,
// formed from Hm[c] = H(r-1, c) before cell (r, c) overwrites that register.  A warp alone on its scheduler then runs at
// its issue rate (tools/lat_probe.cu: dependent DPX instructions issue 4 clk apart, independent ones 2 clk apart; 760 clk
// per 8 x 8 block and 390 per 8 x 4 block, i.e. 95 / 49 clk per row against 365 for the 32-column sweep), so such units
// want a scheduler of their own: wavefront_s16_kernel hands its first round of units out statically, one per SM at a
// time, and the host gives it CTAs of 4 warps.
//
// Hand-off between neighbouring tiles (one warp each, usually on different SMs): the DATA IS THE FLAG.  Every (Hm, E)
// border entry is one 8-byte word per lane and row in a link buffer of its own (one region per group and tile boundary,
// written once and read once per search, laid out [block][row pair][lane][2 rows] so that a warp's access is 512
// contiguous bytes), which holds kNarrowEmpty wherever nothing has been produced yet.  The producer stores a block's rows
// with four st.relaxed.gpu.v2.u64; the consumer reads them with ld.relaxed.gpu.v2.u64 a block ahead of their use, asks
// again while a word's Hm half still reads as empty, and stores kNarrowEmpty back once it has the value, which leaves the
// buffer ready for the next search (the next writer of that word is a later kernel on the stream).  Every 64-bit element
// of these accesses is a strong, naturally aligned operation at gpu scope on one location: single-copy atomic and
// race-free under the PTX memory model, and nothing else is published through it, so the path needs no fence, no
// progress counter and no L1 invalidate.  That is what makes it fast, not only clean: measured on the B200
// (tools/lat_probe.cu, profiles/r02_summary.md) a membar.gpu behind st.release.gpu or a fence.proxy.async costs the
// issuing warp 750-850 clk -- two blocks of a 4-column tile -- and slows the other warps of its SM as well (a variant
// with TMA staging and one release / acquire per 8 blocks ran 960 clk per block alone and 1,600 with four warps per SM).
// kNarrowEmpty cannot be a value: its halves are -32,640, below anything a trusted lane holds (>= -open - ext >= -254);
// a lane that has wrapped (its score is already above the trust limit and will be re-run in int32) could produce the
// pattern by accident, so the producer nudges exactly that Hm word by one -- garbage stays garbage.
constexpr unsigned long long kNarrowEmpty = 0x8080808080808080ull;   // what cudaMemset(0x80) leaves
constexpr uint32_t kNarrowEmptyWord = 0x80808080u;                    // the test looks at the Hm word (the low one)
constexpr uint32_t kNarrowLagBlocks = 4;                              // a tile (re)starts this many blocks behind its producer

static_assert(kNarrowChunkBytes == kRowsPerChunk * 32 * 8, "scan_plan.hpp and the packed layout disagree on the block of border rows");

// Two rows of a lane (16 bytes) at a time: each 64-bit element is a strong relaxed access of its own.
__device__ __forceinline__ void ld_link2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
__device__ __forceinline__ void st_link2(unsigned long long* p, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b));
}
__device__ __forceinline__ bool link_empty(unsigned long long v) { return static_cast<uint32_t>(v) == kNarrowEmptyWord; }

// Per-warp state of the narrow units.
struct NarrowWarp {
    const uint32_t* consts;   // (neg_open2, neg_ext2) in shared memory
    uint32_t in_ring = 0;     // kRings: shared-memory address of the pair's inbound / outbound ring of blocks
    uint32_t out_ring = 0;
    uint32_t mailbox = 0;     // and of the mailbox through which the compute warp tells its helper what to carry
    uint32_t posted = 0;      // commands posted so far
};

// With a helper warp (kRings): the compute warp of a narrow unit never touches global memory for its hand-off.  Its
// partner on the same scheduler -- warp w + 4 of the CTA -- carries the blocks between the link buffers in global memory
// (same strong relaxed accesses, same "data is the flag" protocol as above) and two rings of kNarrowRingSlots blocks in
// shared memory, where the flag is again the data: a slot whose Hm words read kNarrowEmpty is free / not yet filled.  The
// compute warp waits 30 clk for a shared-memory load instead of 310 for L2, packs and checks nothing for the far side, and
// the helper's waiting costs its scheduler nothing but an occasional poll.
constexpr uint32_t kNarrowRingSlots = 4;
constexpr uint32_t kNarrowPairBytes = 2 * kNarrowRingSlots * kNarrowChunkBytes + 64;   // in ring, out ring, mailbox
static_assert(kNarrowPairBytes == kNarrowPairBytesHost, "scan_plan.hpp and kernels.cuh disagree on a pair's shared memory");
struct NarrowMail {           // compute warp -> helper
    uint32_t cmd;             // incremented by the compute warp once the fields below describe a new unit (0: nothing yet)
    uint32_t done;            // set to cmd by the helper when it has carried the unit's last block
    uint32_t kind;            // 1: a narrow unit, 0: leave
    uint32_t n_chunks, tile, n_tiles;
    uint32_t link_lo, link_hi;   // the group's link buffers (64-bit address)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint4 lds128v(uint32_t a) {
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128v(uint32_t a, uint4 v) {
    asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}
__device__ __forceinline__ uint32_t lds32v(uint32_t a) {
    uint32_t v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts32v(uint32_t a, uint32_t v) { asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(a), "r"(v)); }

// The helper's side of one narrow unit: blocks of the inbound link -> the in ring, blocks of the out ring -> the outbound
// link, each as far as its source has them and its target has room; neither direction ever blocks the other.
__device__ __forceinline__ void narrow_helper_unit(uint8_t* link_base, uint32_t n_chunks, uint32_t tile, uint32_t n_tiles, uint32_t lane,
                                                   const NarrowWarp& nw) {
    constexpr size_t kBlockWords = kNarrowChunkBytes / 8;
    const size_t link_words = static_cast<size_t>(n_chunks) * kBlockWords;
    unsigned long long* const links = reinterpret_cast<unsigned long long*>(link_base);
    const bool has_in = tile > 0, has_out = tile + 1 < n_tiles;
    unsigned long long* lin = links + (static_cast<size_t>(tile) - (has_in ? 1 : 0)) * link_words + lane * 2;
    unsigned long long* lout = links + static_cast<size_t>(tile) * link_words + lane * 2;
    const uint4 empty4 = make_uint4(kNarrowEmptyWord, kNarrowEmptyWord, kNarrowEmptyWord, kNarrowEmptyWord);
    uint32_t bi = 0, bo = 0;
    // outbound: a block the compute warp has completed -> the link buffer; false: nothing there yet
    auto try_out = [&]() -> bool {
        if (!has_out || bo >= n_chunks) return false;
        const uint32_t slot = nw.out_ring + (bo % kNarrowRingSlots) * kNarrowChunkBytes + lane * 16;
        uint4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = lds128v(slot + i * 512);
        bool valid = true;
#pragma unroll
        for (int i = 0; i < 4; ++i) valid &= v[i].x != kNarrowEmptyWord && v[i].z != kNarrowEmptyWord;
        if (!__all_sync(0xffffffffu, valid)) return false;
#pragma unroll
        for (int i = 0; i < 4; ++i) sts128v(slot + i * 512, empty4);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            st_link2(lout + i * 64, (static_cast<unsigned long long>(v[i].y) << 32) | v[i].x, (static_cast<unsigned long long>(v[i].w) << 32) | v[i].z);
        lout += kBlockWords;
        ++bo;
        return true;
    };
    // inbound: TWO blocks are on request at any time, each into registers of its own (ga: the block to move next, gb: the
    // one after it, then the roles swap), so that an answer that came too early costs one more round trip for that block
    // only, and the stream is not paced by one L2 round trip per block
    unsigned long long ga[8], gb[8];
    auto request = [&](unsigned long long(&g)[8], uint32_t block) {
        const unsigned long long* at = lin + static_cast<size_t>(min(block, n_chunks - 1)) * kBlockWords;
#pragma unroll
        for (int i = 0; i < 4; ++i) ld_link2(at + i * 64, g[2 * i], g[2 * i + 1]);
    };
    // block bi is in g (or on its way): into the in ring if it is all there and the slot is free
    auto try_in = [&](unsigned long long(&g)[8]) -> bool {
        bool valid = true;
#pragma unroll
        for (int i = 0; i < 8; ++i) valid &= !link_empty(g[i]);
        if (!__all_sync(0xffffffffu, valid)) {
            request(g, bi);   // not all there yet: ask again
            return false;
        }
        const uint32_t slot = nw.in_ring + (bi % kNarrowRingSlots) * kNarrowChunkBytes + lane * 16;
        if (!__all_sync(0xffffffffu, lds32v(slot + 3 * 512 + 8) == kNarrowEmptyWord)) return false;   // the slot's last word: not free yet
#pragma unroll
        for (int i = 0; i < 4; ++i)
            sts128v(slot + i * 512, make_uint4(static_cast<uint32_t>(g[2 * i]), static_cast<uint32_t>(g[2 * i] >> 32),
                                               static_cast<uint32_t>(g[2 * i + 1]), static_cast<uint32_t>(g[2 * i + 1] >> 32)));
        unsigned long long* at = lin + static_cast<size_t>(bi) * kBlockWords;
#pragma unroll
        for (int i = 0; i < 4; ++i) st_link2(at + i * 64, kNarrowEmpty, kNarrowEmpty);
        ++bi;
        request(g, bi + 1);   // the other register set holds block bi now
        return true;
    };
    if (has_in) {
        request(ga, 0);
        request(gb, 1);
        while (bi < n_chunks) {
            while (!try_in(ga))
                if (!try_out()) __nanosleep(40);
            try_out();
            if (bi >= n_chunks) break;
            while (!try_in(gb))
                if (!try_out()) __nanosleep(40);
            try_out();
        }
    }
    // (a short back-off: spinning without it takes issue slots from the compute warp on the same scheduler -- 680 against 637
    // clk per block for a tile that only sends)
    while (has_out && bo < n_chunks)
        if (!try_out()) __nanosleep(40);
}

// kFirst / kLast (tile 0 / the last tile) are compile-time, so that a tile without an inbound or outbound link carries
// none of its code and the block loop's body is straight-line code apart from the rare "a row has not arrived yet".
template <int T, bool kFirst, bool kLast, bool kRings>
__device__ __forceinline__ uint32_t sweep_narrow_tile_s16(const WaveParams& p, const int8_t* prof, const GroupDesc& gd, uint32_t tile,
                                                          uint8_t* link_base, uint32_t lane, NarrowWarp& nw) {
    constexpr int R = static_cast<int>(kRowsPerChunk);
    static_assert((T == 8 || T == 4) && R == 8, "the block sweep is written for 8 rows x 8 or 4 columns");
    using ProfWord = typename std::conditional<T == 8, uint2, uint32_t>::type;   // a row's T int8 entries
    // The two packed constants are read back from shared memory (written by the kernel from its parameters): taken from the
    // parameters directly ptxas keeps them as 16-bit halves in uniform registers and, in a loop under this register
    // pressure, rebuilds the vector operand with a PRMT in front of every VIADDMNMX and VIADD that uses them (+47
    // instructions per 8 x 4 block; a shuffle does not hide the uniformity, a load does).
    const uint32_t NO = *reinterpret_cast<const volatile uint32_t*>(nw.consts), NE = *reinterpret_cast<const volatile uint32_t*>(nw.consts + 1);
    const uint32_t n_chunks = gd.n_chunks;
    if (n_chunks == 0) return 0;
    constexpr size_t kBlockWords = kNarrowChunkBytes / 8;
    const size_t link_words = static_cast<size_t>(n_chunks) * kBlockWords;   // one link: every block of the group
    const uint4* gcodes = p.codes + gd.chunk_base * 32 + lane;
    const int8_t* ptile = prof + tile * T;
    // link t: tile t -> tile t + 1; both pointers advance a block per iteration; a lane's rows 2i, 2i + 1 at [i][lane]
    unsigned long long* const links = reinterpret_cast<unsigned long long*>(link_base);
    const unsigned long long* lin = links + (static_cast<size_t>(tile) - (kFirst ? 0 : 1)) * link_words + lane * 2;
    unsigned long long* lout = links + static_cast<size_t>(tile) * link_words + lane * 2;
    const unsigned long long* const lin_end = lin + (static_cast<size_t>(n_chunks) - 1) * kBlockWords;   // the last block
    auto next_block = [&](const unsigned long long* at) { return at < lin_end ? at + kBlockWords : lin_end; };
    auto request = [&](unsigned long long(&q)[R], const unsigned long long* at) {
#pragma unroll
        for (int i = 0; i < R / 2; ++i) ld_link2(at + i * 64, q[2 * i], q[2 * i + 1]);
    };
    // wait until the producer is kNarrowLagBlocks ahead of block `at` (or done), so that from there on a request made a
    // block ahead finds its rows: at the start, and again whenever the tile has caught up with its producer
    auto fall_back = [&](const unsigned long long* at) {
        const unsigned long long* probe = at;
#pragma unroll
        for (uint32_t i = 0; i < kNarrowLagBlocks; ++i) probe = next_block(probe);
        unsigned long long a, b;
        for (;;) {
            ld_link2(probe + 3 * 64, a, b);
            if (!link_empty(b)) break;   // the block's last row
            __nanosleep(200);
        }
    };

    uint32_t Hm[T], F[T];
#pragma unroll
    for (int k = 0; k < T; ++k) Hm[k] = NO, F[k] = NO;
    uint32_t diag_in = NO, best = 0;
    // Inbound rows are requested at the start of the block BEFORE the one that uses them, into registers of their own, and
    // take the place of the current ones at its end: a block (400+ clk) covers the L2 round trip (~310 clk), and the copy
    // at the end never waits.  (Requests further ahead were tried: the values are then live across the loop's back edge in
    // registers ptxas does not load into directly, and its copies wait for the load.)
    unsigned long long q[R], qn[R];
    const unsigned long long edge = (static_cast<unsigned long long>(NO) << 32) | NO;
#pragma unroll
    for (int i = 0; i < R; ++i) q[i] = qn[i] = edge;
    if (!kFirst && !kRings) {
        fall_back(lin);
        request(q, lin);
    }
    const uint4 empty4 = make_uint4(kNarrowEmptyWord, kNarrowEmptyWord, kNarrowEmptyWord, kNarrowEmptyWord);
    auto profile_rows = [&](const uint4& w, ProfWord* pa, ProfWord* pb) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            // residue r of either sequence: one PRMT each (byte r & 3 of the word, zero-extended)
            const uint32_t a1 = prmt(r < 4 ? w.x : w.y, 0, 0x4440u | (r & 3));
            const uint32_t a2 = prmt(r < 4 ? w.z : w.w, 0, 0x4440u | (r & 3));
            pa[r] = *reinterpret_cast<const ProfWord*>(ptile + a1 * p.pstride);
            pb[r] = *reinterpret_cast<const ProfWord*>(ptile + a2 * p.pstride);
        }
    };
    auto codes_of = [&](uint32_t chunk) { return __ldg(gcodes + static_cast<size_t>(min(chunk, n_chunks - 1)) * 32); };
    ProfWord na[R], nb[R];                       // the profile rows of the block about to be computed
    profile_rows(codes_of(0), na, nb);
    // the residues of the next odd / even block: loaded three blocks ahead into registers of their own (the loop is unrolled
    // by two for that: rotating one set through another would wait for the load at the rotation)
    uint4 cb = codes_of(1), ca = codes_of(2);

    auto step = [&](uint4& cnext, uint32_t chunk) {
        ProfWord pa[R], pb[R];
#pragma unroll
        for (int r = 0; r < R; ++r) pa[r] = na[r], pb[r] = nb[r];
        // substitution word of (row r, column c): the two sequences' int8 entries, sign-extended into the halves
        auto sub = [&](int r, int c) {
            const uint32_t sel = (c & 3) == 0 ? 0xC480u : (c & 3) == 1 ? 0xD591u : (c & 3) == 2 ? 0xE6A2u : 0xF7B3u;
            if constexpr (T == 8) return prmt(c < 4 ? pa[r].x : pa[r].y, c < 4 ? pb[r].x : pb[r].y, sel);
            else return prmt(pa[r], pb[r], sel);
        };
        if (!kFirst && kRings) {
            // this block's rows from the in ring (the helper warp brings them): wait until every word is there, take them,
            // give the slot back
            const uint32_t slot = nw.in_ring + (chunk % kNarrowRingSlots) * kNarrowChunkBytes + lane * 16;
            uint4 v[R / 2];
            for (;;) {
#pragma unroll
                for (int i = 0; i < R / 2; ++i) v[i] = lds128v(slot + i * 512);
                bool valid = true;
#pragma unroll
                for (int i = 0; i < R / 2; ++i) valid &= v[i].x != kNarrowEmptyWord && v[i].z != kNarrowEmptyWord;
                if (valid) break;
                __nanosleep(20);
            }
#pragma unroll
            for (int i = 0; i < R / 2; ++i) sts128v(slot + i * 512, empty4);
#pragma unroll
            for (int i = 0; i < R / 2; ++i)
                q[2 * i] = (static_cast<unsigned long long>(v[i].y) << 32) | v[i].x, q[2 * i + 1] = (static_cast<unsigned long long>(v[i].w) << 32) | v[i].z;
        }
        if (!kFirst && !kRings) {
            request(qn, next_block(lin));   // the next block's rows (past the end: the last block's again, unused)
            // this block's rows, requested a block ago.  A missing one means the tile has caught up with its producer:
            // it falls back by kNarrowLagBlocks instead of trailing it row by row, then asks for both blocks again
            bool missing = false;
#pragma unroll
            for (int i = 0; i < R; ++i) missing |= link_empty(q[i]);
            if (missing) {
                fall_back(lin);
                request(q, lin);
                request(qn, next_block(lin));
            }
#pragma unroll
            for (int i = 0; i < R / 2; ++i) st_link2(const_cast<unsigned long long*>(lin) + i * 64, kNarrowEmpty, kNarrowEmpty);
        }
        uint32_t E[R], hl[R], d[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            hl[r] = static_cast<uint32_t>(q[r]), E[r] = static_cast<uint32_t>(q[r] >> 32);
            d[r] = __vadd2(r == 0 ? diag_in : static_cast<uint32_t>(q[r - 1]), sub(r, 0));   // diagonal of column 0: the row above's inbound Hm
        }
        diag_in = static_cast<uint32_t>(q[R - 1]);
        // the next block's profile rows and the residues three blocks on travel while this one is computed (past the end:
        // the last block's again, unused); tile 0 reads the residues from HBM for everyone behind it, well ahead
        profile_rows(cnext, na, nb);
        cnext = codes_of(chunk + 3);
        if (kFirst) asm volatile("prefetch.global.L2 [%0];" ::"l"(gcodes + static_cast<size_t>(min(chunk + 32, n_chunks - 1)) * 32));
        uint32_t pend = 0;
        bool have = false;
#pragma unroll
        for (int dd = 0; dd < R + T - 1; ++dd) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int c = dd - r;
                if (c < 0 || c >= T) continue;
                E[r] = __viaddmax_s16x2(E[r], NE, hl[r]);
                F[c] = __viaddmax_s16x2(F[c], NE, Hm[c]);
                const uint32_t dcur = d[r];
                if (c + 1 < T) d[r] = __vadd2(Hm[c], sub(r, c + 1));
                hl[r] = __vadd2(__vimax3_s16x2_relu(dcur, E[r], F[c]), NO);
                Hm[c] = hl[r];
                // running maximum over the diagonal terms (exact, see sweep_unit_s16): one VIMNMX3 per two cells
                if (have) best = __vimax3_s16x2(best, pend, dcur), have = false;
                else pend = dcur, have = true;
            }
        }
        if (!kLast && kRings) {
            // outbound: into the out ring once its slot is free (the helper warp takes it from there)
            const uint32_t slot = nw.out_ring + (chunk % kNarrowRingSlots) * kNarrowChunkBytes + lane * 16;
            while (lds32v(slot + 3 * 512 + 8) != kNarrowEmptyWord) __nanosleep(20);
#pragma unroll
            for (int i = 0; i < R / 2; ++i) {
                const uint32_t h0 = hl[2 * i] == kNarrowEmptyWord ? kNarrowEmptyWord + 1 : hl[2 * i];
                const uint32_t h1 = hl[2 * i + 1] == kNarrowEmptyWord ? kNarrowEmptyWord + 1 : hl[2 * i + 1];
                sts128v(slot + i * 512, make_uint4(h0, E[2 * i], h1, E[2 * i + 1]));
            }
        }
        if (!kLast && !kRings) {
#pragma unroll
            for (int i = 0; i < R / 2; ++i) {
                // only a lane that has already wrapped can hold the "empty" pattern: nudge it, garbage stays garbage
                const uint32_t h0 = hl[2 * i] == kNarrowEmptyWord ? kNarrowEmptyWord + 1 : hl[2 * i];
                const uint32_t h1 = hl[2 * i + 1] == kNarrowEmptyWord ? kNarrowEmptyWord + 1 : hl[2 * i + 1];
                st_link2(lout + i * 64, (static_cast<unsigned long long>(E[2 * i]) << 32) | h0,
                         (static_cast<unsigned long long>(E[2 * i + 1]) << 32) | h1);
            }
            lout += kBlockWords;
        }
        if (!kFirst && !kRings) {
            lin = next_block(lin);
#pragma unroll
            for (int i = 0; i < R; ++i) q[i] = qn[i];
        }
    };
    for (uint32_t chunk = 0; chunk < n_chunks; chunk += 2) {
        step(cb, chunk);
        if (chunk + 1 < n_chunks) step(ca, chunk + 1);
    }
    return best;
}

template <int T, bool kRings>
__device__ __forceinline__ uint32_t sweep_unit_narrow_s16(const WaveParams& p, const int8_t* prof, const GroupDesc& gd, uint32_t tile,
                                                          uint32_t n_tiles, uint8_t* link_base, uint32_t lane, NarrowWarp& nw) {
    const bool first = tile == 0, last = tile + 1 == n_tiles;
    if (first) return last ? sweep_narrow_tile_s16<T, true, true, kRings>(p, prof, gd, tile, link_base, lane, nw)
                           : sweep_narrow_tile_s16<T, true, false, kRings>(p, prof, gd, tile, link_base, lane, nw);
    return last ? sweep_narrow_tile_s16<T, false, true, kRings>(p, prof, gd, tile, link_base, lane, nw)
                : sweep_narrow_tile_s16<T, false, false, kRings>(p, prof, gd, tile, link_base, lane, nw);
}

// Group modes (GroupMode, kNarrowTile): scan_plan.hpp, where the host decides them per search.

// kNarrow: compile the 8-column path in.  Searches without narrow groups (all long queries) launch the variant
// without it, whose register allocation is not disturbed by the second sweep.
template <bool kSmemProfile, int T, int kThreads, bool kNarrow, bool kRowBlocks>
__global__ void __launch_bounds__(kThreads, 1) wavefront_s16_kernel(WaveParams p) {
    extern __shared__ __align__(16) uint8_t smem_prof[];
    struct NoNarrow {};
    typename std::conditional<kNarrow, NarrowWarp, NoNarrow>::type nw{};
    if constexpr (kNarrow) {
        __shared__ uint32_t narrow_consts[2];   // sweep_narrow_tile_s16 reads its packed constants from here
        if (threadIdx.x == 0) narrow_consts[0] = p.neg_open2, narrow_consts[1] = p.neg_ext2;
        nw.consts = narrow_consts;
        if (p.narrow_helpers) {
            // rings (all slots empty) and mailboxes of the four compute / helper pairs
            const uint32_t stage = smem_u32(smem_prof) + p.narrow_stage_off;
            for (uint32_t i = threadIdx.x; i < 4 * kNarrowPairBytes / 16; i += blockDim.x) {
                const uint32_t off = i * 16, in_pair = off % kNarrowPairBytes;
                const uint32_t fill = in_pair < kNarrowPairBytes - 64 ? kNarrowEmptyWord : 0u;
                sts128v(stage + off, make_uint4(fill, fill, fill, fill));
            }
            const uint32_t base = stage + ((threadIdx.x >> 5) & 3) * kNarrowPairBytes;
            nw.in_ring = base;
            nw.out_ring = base + kNarrowRingSlots * kNarrowChunkBytes;
            nw.mailbox = nw.out_ring + kNarrowRingSlots * kNarrowChunkBytes;
        }
        __syncthreads();
    }

    const int8_t* prof;
    if (kSmemProfile) {
        const uint32_t n16 = kProfRows * p.pstride / 16;
        const uint4* src = reinterpret_cast<const uint4*>(p.prof8);
        uint4* dst = reinterpret_cast<uint4*>(smem_prof);
        for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
        __syncthreads();
        prof = reinterpret_cast<const int8_t*>(smem_prof);
    } else {
        prof = p.prof8;
    }

    const uint32_t lane = threadIdx.x & 31;
    bool helpers = false;
    if constexpr (kNarrow) {
        helpers = p.narrow_helpers != 0;
        if (helpers && (threadIdx.x >> 5) >= 4) {
            // a helper warp: carries the blocks of whatever narrow unit its compute warp (warp - 4, same scheduler) posts
            for (uint32_t seen = 0;;) {
                uint32_t cmd;
                while ((cmd = lds32v(nw.mailbox)) == seen) __nanosleep(100);
                seen = cmd;
                if (lds32v(nw.mailbox + 8) == 0) return;
                const uint32_t n_chunks = lds32v(nw.mailbox + 12), tile = lds32v(nw.mailbox + 16), n_tiles = lds32v(nw.mailbox + 20);
                const unsigned long long link = (static_cast<unsigned long long>(lds32v(nw.mailbox + 28)) << 32) | lds32v(nw.mailbox + 24);
                narrow_helper_unit(reinterpret_cast<uint8_t*>(link), n_chunks, tile, n_tiles, lane, nw);
                __syncwarp();
                if (lane == 0) sts32v(nw.mailbox + 4, cmd);
            }
        }
    }
    const uint32_t n_compute = helpers ? 4u : blockDim.x >> 5;   // warps that take units

    // First round: static, unit (warp, CTA) -> warp x gridDim + CTA, so that consecutive units -- the tiles of the
    // tallest groups, whose warps are bound by their own chain -- start on different SMs instead of on the sixteen warps
    // of whichever CTA came up first.  After that, tickets.  Either way a unit's producer (the unit before it) is held
    // by a resident warp or was handed out earlier: waiting on it cannot deadlock (the grid never exceeds the SM count).
    const uint32_t static_units = gridDim.x * n_compute;
    for (uint32_t round = 0;; ++round) {
        uint32_t u = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
        if (round > 0) {
            if (lane == 0) u = static_units + atomicAdd(p.ticket, 1u);
            u = __shfl_sync(0xffffffffu, u, 0);
        }
        if (u >= p.n_units) break;

        // group of this unit: largest g with unit_start[g] <= u
        uint32_t lo = 0, hi = p.n_groups;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(p.unit_start + mid) <= u) lo = mid;
            else hi = mid;
        }
        const uint32_t g = lo;
        const GroupDesc gd = p.groups[g];
        const uint32_t u0 = __ldg(p.unit_start + g);
        const uint32_t mode = p.group_mode[g];
        const uint32_t n_tiles = mode == kGroupNarrow ? p.n_tiles_narrow : p.n_tiles;
        uint32_t best;
        if (kRowBlocks && mode == kGroupRowBlock) {
            // unit b of nb: chunks [b * per, min((b + 1) * per, n_chunks)), all tiles
            const uint32_t nb = __ldg(p.unit_start + g + 1) - u0, b = u - u0;
            const uint32_t per = (gd.n_chunks + nb - 1) / nb;
            const uint32_t lo_c = min(gd.n_chunks, b * per), hi_c = min(gd.n_chunks, lo_c + per);
            const uint32_t* dep = b > 0 ? p.progress + (u - 1) : nullptr;
            uint32_t* pub = b + 1 < nb ? p.progress + u : nullptr;
            uint4* vs = p.vstate + static_cast<size_t>(p.vstate_off[g]) * (kVStateWords / 4) * 32;
            best = sweep_unit_s16<T, 2, 1, true>(p, prof, gd, 0, n_tiles, n_tiles, dep, pub, lane, lo_c, hi_c, vs);
        } else {
            const uint32_t t0 = mode == kGroupSingle ? 0 : u - u0;
            const uint32_t t1 = mode == kGroupSingle ? n_tiles : t0 + 1;
            const uint32_t* dep = t0 > 0 ? p.progress + (u - 1) : nullptr;
            uint32_t* pub = t1 < n_tiles ? p.progress + u : nullptr;
            bool narrow_done = false;
            if constexpr (kNarrow) {
                if (mode == kGroupNarrow) {
                    // (the link-buffer forms are only compiled where the host can choose them: profile in shared memory, and the
                    // helper form only into the build for CTAs of 4 + 4 warps -- each form is eight instantiations of the sweep)
                    if (kSmemProfile && kThreads == 2 * kNarrowThreads && p.narrow_staged && helpers) {
                        // tell the helper warp what to carry (once it is done with the unit before), then sweep on the rings
                        uint8_t* links = p.nlinks + static_cast<size_t>(p.vstate_off[g]) * 256;
                        while (lds32v(nw.mailbox + 4) != nw.posted) __nanosleep(40);
                        ++nw.posted;
                        if (lane == 0) {
                            const unsigned long long link = reinterpret_cast<unsigned long long>(links);
                            sts32v(nw.mailbox + 8, 1u), sts32v(nw.mailbox + 12, gd.n_chunks), sts32v(nw.mailbox + 16, t0);
                            sts32v(nw.mailbox + 20, n_tiles), sts32v(nw.mailbox + 24, static_cast<uint32_t>(link));
                            sts32v(nw.mailbox + 28, static_cast<uint32_t>(link >> 32));
                            sts32v(nw.mailbox, nw.posted);
                        }
                        best = p.narrow_tile == 4 ? sweep_unit_narrow_s16<4, true>(p, prof, gd, t0, n_tiles, links, lane, nw)
                                                  : sweep_unit_narrow_s16<8, true>(p, prof, gd, t0, n_tiles, links, lane, nw);
                    } else if (kSmemProfile && p.narrow_staged) {
                        uint8_t* links = p.nlinks + static_cast<size_t>(p.vstate_off[g]) * 256;
                        best = p.narrow_tile == 4 ? sweep_unit_narrow_s16<4, false>(p, prof, gd, t0, n_tiles, links, lane, nw)
                                                  : sweep_unit_narrow_s16<8, false>(p, prof, gd, t0, n_tiles, links, lane, nw);
                    } else {
                        // a deep wavefront of 8-column tiles (long query): rows fetched 8 ahead, progress published every 4 chunks
                        best = sweep_unit_s16<kNarrowTile, 8, 4, false>(p, prof, gd, t0, t1, n_tiles, dep, pub, lane, 0, gd.n_chunks, nullptr);
                    }
                    narrow_done = true;
                }
            }
            if (!narrow_done)
                best = sweep_unit_s16<T, 2, 1, false>(p, prof, gd, t0, t1, n_tiles, dep, pub, lane, 0, gd.n_chunks, nullptr);
        }

        // halves -> slots (lane, lane+32); the maximum over the group's units
        const int32_t sa = static_cast<int32_t>(best & 0xffffu);
        const int32_t sb = static_cast<int32_t>(best >> 16);
        const uint32_t slot_a = gd.first_slot + lane;
        if (sa) atomicMax(p.slot_scores + slot_a, sa);
        if (sb) atomicMax(p.slot_scores + slot_a + 32, sb);
    }
    if constexpr (kNarrow) {
        if (helpers) {   // send the helper warp home (once it is done with the last unit)
            while (lds32v(nw.mailbox + 4) != nw.posted) __nanosleep(40);
            if (lane == 0) sts32v(nw.mailbox + 8, 0u), sts32v(nw.mailbox, nw.posted + 1);
        }
    }
}

// Slots whose packed-int16 score is above the trust limit -> list for the int32 re-run.
__global__ void collect_flagged_kernel(const int32_t* slot_scores, uint32_t n_slots, int32_t limit,
                                       uint32_t* list, uint32_t* count) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_slots; i += gridDim.x * blockDim.x)
        if (slot_scores[i] > limit) list[atomicAdd(count, 1u)] = i;
}

// ------------------------------------------------------------------------------------------------
// Intra-task kernel (int32, warp shuffles): one CTA per sequence (align.hpp:166-229 re-designed).
// Used for (a) the exact re-run of lanes flagged by the int16 kernel (align.hpp:149-153), (b)
// swb_score_pair / sw_score_wavefront, (c) every sequence in "wide" mode (matrix + open outside
// int8), where the packed kernel does not apply.
//
// The query is striped over lanes, T (<= 8) columns per lane, 32*T per warp, W warps side by side
// (W*32*T columns per pass).  Lane l of warp w handles subject row  d - w*Delta - l  at step d:
// an anti-diagonal wavefront.  The (Hm, E) border of a lane's last column moves to its right
// neighbour with one __shfl_up per step; between warps it goes through a shared-memory ring
// (written by lane 31, read by the next warp's lane 0 >= 33 steps later, one __syncthreads every
// 32 steps); between passes it goes through a per-CTA border row in global memory.
// The diagonal seed is the previous step's inbound Hm, exactly the reference's diag_seed
// (align.hpp:223).  Rows outside [0, n) are pad rows: before the start they leave the initial
// state untouched, after the end they cannot raise `best`.
// ------------------------------------------------------------------------------------------------
struct IntraParams {
    const uint8_t* codes;       // interleaved group layout, as bytes
    const GroupDesc* groups;
    const uint32_t* slot_len;
    const uint32_t* list;       // slots to score; nullptr = every slot 0..n_slots-1
    const uint32_t* list_count; // device count for `list`
    uint32_t n_slots;
    const void* profi;          // prof8i or prof32i
    uint32_t n_lane_tiles;      // 8-slot words per profile row
    uint32_t n_passes;
    uint2* border0;             // [gridDim.x][border_rows]
    uint2* border1;
    uint64_t border_rows;
    int32_t* slot_scores;
    int32_t open, ext;
};

// A lane meets its subject's residues in order, one per step: they come as 8-byte words (8 consecutive rows of the
// interleaved layout), requested four steps before the first of them is needed, and the int8 profile entries of the
// lane's own columns (25 symbols x 8 B) are staged in shared memory once per pass -- without either, every step waited
// for two dependent global loads (2,600 clk per step instead of ~200: the int32 re-run of three 8,000-residue hits cost
// 47 ms next to a 160 ms scan).
template <int T, typename PT>
__global__ void __launch_bounds__(32 * kIntraMaxWarps) intra_s32_kernel(IntraParams p) {
    __shared__ uint2 ring[kIntraMaxWarps][kIntraRing];
    __shared__ int32_t warp_best[kIntraMaxWarps];
    extern __shared__ __align__(16) uint8_t intra_dyn[];   // int8 profile: [25][blockDim.x] uint2, this pass's columns
    uint2* const sprof = reinterpret_cast<uint2*>(intra_dyn);

    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int32_t NO = -p.open, NE = -p.ext;
    const PT* prof = static_cast<const PT*>(p.profi);
    const uint32_t row_words = p.n_lane_tiles * 8;
    const uint32_t count = p.list ? *p.list_count : p.n_slots;
    uint2* const my_b0 = p.border0 + static_cast<size_t>(blockIdx.x) * p.border_rows;
    uint2* const my_b1 = p.border1 + static_cast<size_t>(blockIdx.x) * p.border_rows;

    for (uint32_t item = blockIdx.x; item < count; item += gridDim.x) {
        const uint32_t slot = p.list ? p.list[item] : item;
        const int64_t n = p.slot_len[slot];
        const GroupDesc gd = p.groups[slot / kGroupSeqs];
        const uint32_t sl = slot % kGroupSeqs;
        // residues 8w .. 8w + 7 of this sequence: the 8-byte word seq8[w * 64]
        const uint2* seq8 = reinterpret_cast<const uint2*>(p.codes + (static_cast<size_t>(gd.chunk_base) * 32 + (sl & 31)) * 16 + (sl >> 5) * 8);
        const int64_t n_words = gd.n_chunks;

        int32_t best = 0;
        const int64_t steps = n + 31 + static_cast<int64_t>(kIntraDelta) * (W - 1);

        for (uint32_t pass = 0; pass < p.n_passes && n > 0; ++pass) {
            const uint32_t lane_tile = (pass * W + w) * 32 + lane;   // which T-column stripe this lane owns
            const bool tile_valid = lane_tile < p.n_lane_tiles;
            const PT* ptile = prof + static_cast<size_t>(tile_valid ? lane_tile : 0) * 8;
            const bool first = pass == 0, last = pass + 1 == p.n_passes;
            const uint2* bin = (pass & 1) ? my_b0 : my_b1;
            uint2* bout = (pass & 1) ? my_b1 : my_b0;

            int32_t Hm[T], F[T];
#pragma unroll
            for (int k = 0; k < T; ++k) Hm[k] = NO, F[k] = NO;
            int32_t diag_in = NO, out_h = NO, out_e = NO;

            __syncthreads();   // ring, border rows and the profile slice are reused across passes and items
            if (sizeof(PT) == 1) {
                for (uint32_t sym = 0; sym < kProfRows; ++sym)
                    sprof[sym * blockDim.x + threadIdx.x] = *reinterpret_cast<const uint2*>(ptile + static_cast<size_t>(sym) * row_words);
                __syncthreads();
            }

            const int64_t r0 = -static_cast<int64_t>(w) * kIntraDelta - lane;   // this lane's row at step 0
            uint2 cur8 = make_uint2(0, 0), nxt8 = __ldg(seq8);
            // the previous pass's border rows (warp 0, lane 0 needs row d at step d): fetched 32 rows at a time by the whole
            // warp, a batch ahead, and handed to lane 0 by shuffle -- a load per step would stall the leading warp, and with
            // it the whole wavefront, for an L2 round trip at every step of every pass but the first
            const bool from_pass = w == 0 && !first;
            uint2 bq = make_uint2(0, 0), bq_next = make_uint2(0, 0);
            if (from_pass && lane < n) bq_next = bin[lane];
            for (int64_t d = 0; d < steps; ++d) {
                const int64_t r = d + r0;
                const bool in_range = r >= 0 && r < n;
                if ((r & 7) == 0) cur8 = nxt8;
                if ((r & 7) == 4) {
                    const int64_t wi = (r >> 3) + 1;
                    if (wi >= 0 && wi < n_words) nxt8 = __ldg(seq8 + wi * 64);
                }
                const uint32_t byte = ((r & 4) ? cur8.y : cur8.x) >> (8 * (static_cast<uint32_t>(r) & 3u)) & 0xffu;
                const uint32_t a = (in_range && tile_valid) ? byte : kPadCode;

                // inbound border: from the left lane (previous step), the left warp's ring, the
                // previous pass's global row, or the matrix edge
                int32_t in_h = __shfl_up_sync(0xffffffffu, out_h, 1);
                int32_t in_e = __shfl_up_sync(0xffffffffu, out_e, 1);
                if (lane == 0) {
                    in_h = NO, in_e = NO;
                    if (in_range) {
                        if (w > 0) {
                            const uint2 v = ring[w][r & (kIntraRing - 1)];
                            in_h = static_cast<int32_t>(v.x), in_e = static_cast<int32_t>(v.y);
                        }
                    }
                }
                if (from_pass) {
                    if ((d & 31) == 0) {
                        bq = bq_next;
                        const int64_t ahead = d + 32 + lane;
                        if (ahead < n) bq_next = bin[ahead];
                    }
                    const uint32_t vx = __shfl_sync(0xffffffffu, bq.x, static_cast<int>(d & 31));
                    const uint32_t vy = __shfl_sync(0xffffffffu, bq.y, static_cast<int>(d & 31));
                    if (lane == 0 && in_range) in_h = static_cast<int32_t>(vx), in_e = static_cast<int32_t>(vy);
                }

                int32_t sub[T];
                if (sizeof(PT) == 1) {
                    const uint2 v = sprof[a * blockDim.x + threadIdx.x];
#pragma unroll
                    for (int k = 0; k < T; ++k) {
                        const uint32_t word = k < 4 ? v.x : v.y;
                        const uint32_t sel = (k & 3) == 0 ? 0x8880u : (k & 3) == 1 ? 0x9991u : (k & 3) == 2 ? 0xAAA2u : 0xBBB3u;
                        sub[k] = static_cast<int32_t>(prmt(word, 0, sel));
                    }
                } else {
                    const int4* q = reinterpret_cast<const int4*>(ptile + static_cast<size_t>(a) * row_words);
                    const int4 v0 = q[0];
                    const int4 v1 = T > 4 ? q[1] : make_int4(0, 0, 0, 0);
                    const int32_t all[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                    for (int k = 0; k < T; ++k) sub[k] = all[k];
                }

                int32_t hl = in_h, E = in_e;
                int32_t diag = diag_in;
                diag_in = in_h;
#pragma unroll
                for (int k = 0; k < T; ++k) {
                    E = __viaddmax_s32(E, NE, hl);
                    F[k] = __viaddmax_s32(F[k], NE, Hm[k]);
                    const int32_t h = __vimax3_s32_relu(diag + sub[k], E, F[k]);
                    diag = Hm[k];
                    hl = h + NO;
                    Hm[k] = hl;
                    best = max(best, h);
                }
                out_h = hl, out_e = E;

                if (lane == 31 && in_range) {
                    if (w + 1 < W) ring[w + 1][r & (kIntraRing - 1)] = make_uint2(hl, E);
                    else if (!last) bout[r] = make_uint2(hl, E);
                }
                if (W > 1 && (d & 31) == 31) __syncthreads();
            }
        }

#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
        __syncthreads();
        if (lane == 0) warp_best[w] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (uint32_t i = 1; i < W; ++i) best = max(best, warp_best[i]);
            p.slot_scores[slot] = best;
        }
    }
}

// ------------------------------------------------------------------------------------------------
// Traceback on the GPU (sw_align_traceback, align.hpp:254-353) -- SURVEY 8(f) rank 2.  Runs after scoring on the
// <= top_k surviving hits, outside the measured region, but it is on by default (scheduler.hpp:27) and on the host
// it costs more than the whole search for long pairs.
//
// traceback_fill_kernel: one CTA per pair (all pairs of a search in one launch), the intra-task wavefront of intra_s32_kernel (8 columns per lane) that
// additionally writes one direction byte per cell with the reference's encoding and tie-breaking
// (align.hpp:269-305): bits 0-1 where H came from (0 stop, 1 diagonal, 2 gap along the query, 3 gap along the
// subject, later ones winning only on strict improvement), bit 2 / bit 3 set when that gap is an extension (a tie
// between opening and extending counts as opening).  The end point is the first maximum in (subject row, query
// column) order (align.hpp:308).  Layout: dir[(t - 1) * pitch + (q - 1)], pitch = m rounded up to 8, so that a
// lane's 8 columns are one aligned 8-byte store.
// traceback_walk_kernel: one warp follows the path backwards; diagonal runs are followed 32 cells per step.
// ------------------------------------------------------------------------------------------------
struct TracebackJob {
    uint64_t codes_off;   // byte offset of the subject's first residue in the interleaved layout
    uint64_t dir_off;     // byte offset of this pair's direction matrix
    uint64_t border_off;  // element offset of this pair's per-pass border rows
    uint64_t ops_off;     // byte offset of this pair's (reversed) edit script
    uint32_t n;           // subject length
    uint32_t result_off;  // index of this pair's 8-int result record
};

struct TracebackParams {
    const uint8_t* codes;      // interleaved group layout of the resident database
    const uint8_t* query;      // m codes
    const TracebackJob* jobs;  // one per CTA
    uint32_t m;
    const void* profi;         // prof8i or prof32i, re-tiled with 8 columns per lane tile
    uint32_t n_lane_tiles;
    uint32_t n_passes;
    uint2* border0;
    uint2* border1;
    uint8_t* dir;
    uint32_t pitch;            // m rounded up to 8
    int32_t open, ext;
    int32_t* result;           // per job: [0] score, [1] end row t (1-based), [2] end column q (1-based), [3] n_ops,
                               //          [4] query_begin, [5] subject_begin
    uint8_t* ops_reversed;     // walk output, last operation first
};

template <typename PT>
__global__ void __launch_bounds__(32 * kIntraMaxWarps) traceback_fill_kernel(TracebackParams p) {
    constexpr int T = 8;
    __shared__ uint2 ring[kIntraMaxWarps][kIntraRing];
    __shared__ int32_t red_score[kIntraMaxWarps * 32];
    __shared__ uint32_t red_t[kIntraMaxWarps * 32], red_q[kIntraMaxWarps * 32];

    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int32_t NO = -p.open, NE = -p.ext;
    const PT* prof = static_cast<const PT*>(p.profi);
    const uint32_t row_words = p.n_lane_tiles * 8;
    const TracebackJob job = p.jobs[blockIdx.x];
    const int64_t n = job.n;
    const uint8_t* seq = p.codes + job.codes_off;
    uint8_t* const dir = p.dir + job.dir_off;
    const int64_t steps = n + 31 + static_cast<int64_t>(kIntraDelta) * (W - 1);

    int32_t best = 0;
    uint32_t best_t = 0, best_q = 0;

    for (uint32_t pass = 0; pass < p.n_passes; ++pass) {
        const uint32_t lane_tile = (pass * W + w) * 32 + lane;
        const bool tile_valid = lane_tile < p.n_lane_tiles;
        const PT* ptile = prof + static_cast<size_t>(tile_valid ? lane_tile : 0) * 8;
        const uint32_t col0 = lane_tile * T;                 // 0-based query column of this lane's first cell
        const bool first = pass == 0, last = pass + 1 == p.n_passes;
        const uint2* bin = ((pass & 1) ? p.border0 : p.border1) + job.border_off;
        uint2* bout = ((pass & 1) ? p.border1 : p.border0) + job.border_off;

        int32_t Hm[T], F[T];
#pragma unroll
        for (int k = 0; k < T; ++k) Hm[k] = NO, F[k] = NO;
        int32_t diag_in = NO, out_h = NO, out_e = NO;
        __syncthreads();

        for (int64_t d = 0; d < steps; ++d) {
            const int64_t r = d - static_cast<int64_t>(w) * kIntraDelta - lane;
            const bool in_range = r >= 0 && r < n;
            const uint32_t a = (in_range && tile_valid) ? seq[(r >> 3) * 512 + (r & 7)] : kPadCode;

            int32_t in_h = __shfl_up_sync(0xffffffffu, out_h, 1);
            int32_t in_e = __shfl_up_sync(0xffffffffu, out_e, 1);
            if (lane == 0) {
                in_h = NO, in_e = NO;
                if (in_range) {
                    if (w > 0) {
                        const uint2 v = ring[w][r & (kIntraRing - 1)];
                        in_h = static_cast<int32_t>(v.x), in_e = static_cast<int32_t>(v.y);
                    } else if (!first) {
                        const uint2 v = bin[r];
                        in_h = static_cast<int32_t>(v.x), in_e = static_cast<int32_t>(v.y);
                    }
                }
            }

            int32_t sub[T];
            if (sizeof(PT) == 1) {
                const uint2 v = *reinterpret_cast<const uint2*>(ptile + static_cast<size_t>(a) * row_words);
#pragma unroll
                for (int k = 0; k < T; ++k) {
                    const uint32_t word = k < 4 ? v.x : v.y;
                    const uint32_t sel = (k & 3) == 0 ? 0x8880u : (k & 3) == 1 ? 0x9991u : (k & 3) == 2 ? 0xAAA2u : 0xBBB3u;
                    sub[k] = static_cast<int32_t>(prmt(word, 0, sel));
                }
            } else {
                const int4* q4 = reinterpret_cast<const int4*>(ptile + static_cast<size_t>(a) * row_words);
                const int4 v0 = q4[0], v1 = q4[1];
                const int32_t all[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                for (int k = 0; k < T; ++k) sub[k] = all[k];
            }

            int32_t hl = in_h, E = in_e;
            int32_t diag = diag_in;
            diag_in = in_h;
            uint32_t dlo = 0, dhi = 0;   // 8 direction bytes
#pragma unroll
            for (int k = 0; k < T; ++k) {
                uint32_t flags = 0;
                const int32_t e_ext = E + NE;                 // extend the gap along the query
                if (hl < e_ext) flags |= 4u;                  // opening (hl = H_left - open) loses strictly
                E = max(hl, e_ext);
                const int32_t f_ext = F[k] + NE;              // extend the gap along the subject
                if (Hm[k] < f_ext) flags |= 8u;
                F[k] = max(Hm[k], f_ext);
                int32_t h = 0;
                uint32_t from = 0;
                const int32_t paired = diag + sub[k];         // sub = matrix + open, diag = H_diag - open
                if (paired > h) h = paired, from = 1u;
                if (E > h) h = E, from = 2u;
                if (F[k] > h) h = F[k], from = 3u;
                const uint32_t byte = flags | from;
                if (k < 4) dlo |= byte << (8 * k);
                else dhi |= byte << (8 * (k - 4));
                diag = Hm[k];
                hl = h + NO;
                Hm[k] = hl;
                // first maximum in (row, column) order (align.hpp:308).  A thread meets its cells pass by pass, so a
                // later pass can reach an equal score at an EARLIER row: ties are broken by position, not by arrival
                if (in_range && col0 + k < p.m) {
                    const uint32_t ct = static_cast<uint32_t>(r) + 1, cq = col0 + k + 1;
                    if (h > best || (h == best && h > 0 && (ct < best_t || (ct == best_t && cq < best_q)))) best = h, best_t = ct, best_q = cq;
                }
            }
            out_h = hl, out_e = E;

            if (in_range && tile_valid)
                *reinterpret_cast<uint2*>(dir + static_cast<size_t>(r) * p.pitch + col0) = make_uint2(dlo, dhi);
            if (lane == 31 && in_range) {
                if (w + 1 < W) ring[w + 1][r & (kIntraRing - 1)] = make_uint2(hl, E);
                else if (!last) bout[r] = make_uint2(hl, E);
            }
            if (W > 1 && (d & 31) == 31) __syncthreads();
        }
    }

    // end point: maximum score, then smallest row, then smallest column == first maximum in row-major order
    red_score[threadIdx.x] = best, red_t[threadIdx.x] = best_t, red_q[threadIdx.x] = best_q;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t i = 1; i < blockDim.x; ++i) {
            const bool better = red_score[i] > best ||
                                (red_score[i] == best && best > 0 &&
                                 (red_t[i] < best_t || (red_t[i] == best_t && red_q[i] < best_q)));
            if (better) best = red_score[i], best_t = red_t[i], best_q = red_q[i];
        }
        int32_t* result = p.result + static_cast<size_t>(job.result_off) * 8;
        result[0] = best, result[1] = static_cast<int32_t>(best_t), result[2] = static_cast<int32_t>(best_q);
    }
}

__global__ void __launch_bounds__(32) traceback_walk_kernel(TracebackParams p) {
    const uint32_t lane = threadIdx.x;
    const TracebackJob job = p.jobs[blockIdx.x];
    int32_t* const result = p.result + static_cast<size_t>(job.result_off) * 8;
    const uint8_t* const dir = p.dir + job.dir_off;
    const uint8_t* const seq = p.codes + job.codes_off;
    uint8_t* const ops = p.ops_reversed + job.ops_off;
    const int32_t score = result[0];
    uint32_t t = static_cast<uint32_t>(result[1]), q = static_cast<uint32_t>(result[2]);   // 1-based
    uint32_t n_ops = 0;
    if (score > 0) {
        enum { kCell = 0, kGapQ = 1, kGapS = 2 };
        int where = kCell;
        for (bool walking = true; walking;) {
            if (where == kCell) {
                // speculate that the next 32 cells up the diagonal are all "from diagonal"
                uint32_t byte = 0;
                const bool inside = t > lane && q > lane;
                if (inside) byte = dir[static_cast<size_t>(t - lane - 1) * p.pitch + (q - lane - 1)];
                const bool is_diag = inside && (byte & 3u) == 1u;
                const uint32_t not_diag = ~__ballot_sync(0xffffffffu, is_diag);
                const uint32_t run = not_diag ? __ffs(not_diag) - 1 : 32;   // lanes 0..run-1 are diagonal moves
                if (lane < run) {
                    const uint8_t qc = p.query[q - lane - 1];
                    const uint32_t row = t - lane - 1;
                    const uint8_t sc = seq[(row >> 3) * 512 + (row & 7)];
                    ops[n_ops + lane] = qc == sc ? 0 : 1;                                // match : substitute
                }
                n_ops += run, t -= run, q -= run;
                if (run < 32) {
                    // the cell at the end of the run is not diagonal (or is outside the matrix)
                    const uint32_t stop_byte = __shfl_sync(0xffffffffu, byte, run);
                    const bool stop_inside = __shfl_sync(0xffffffffu, static_cast<int>(inside), run) != 0;
                    const uint32_t from = stop_inside ? (stop_byte & 3u) : 0u;
                    if (from == 0) walking = false;
                    else where = from == 2 ? kGapQ : kGapS;
                }
            } else {
                // gap runs are short: one cell per step
                const uint32_t byte = dir[static_cast<size_t>(t - 1) * p.pitch + (q - 1)];
                if (where == kGapQ) {
                    if (lane == 0) ops[n_ops] = 3;   // del: a query residue against a gap
                    ++n_ops, --q;
                    if (!(byte & 4u)) where = kCell;
                } else {
                    if (lane == 0) ops[n_ops] = 2;   // insert: a subject residue against a gap
                    ++n_ops, --t;
                    if (!(byte & 8u)) where = kCell;
                }
            }
        }
    }
    if (lane == 0) {
        result[3] = static_cast<int32_t>(n_ops);
        result[4] = static_cast<int32_t>(q);   // query_begin (0-based, half-open)
        result[5] = static_cast<int32_t>(t);   // subject_begin
    }
}

// ------------------------------------------------------------------------------------------------
// Score gather (merge_results, scheduler.hpp:106-117, without the full sort).
//   key = (score << 32) | (0xFFFFFFFF - db_index): descending key order == (score desc, index asc).
//   0 is never a valid key (db_index < 2^32 - 1), so it pads.
// select: every block bitonic-sorts a slice of 4096 keys in shared memory and emits its top k;
// rounds repeat until one block remains.  k <= 1024 here; larger k takes the full bitonic sort.
// ------------------------------------------------------------------------------------------------
constexpr int kSelectSlice = 4096;
constexpr int kSelectThreads = 1024;
constexpr uint32_t kSelectMaxK = 1024;

__global__ void build_keys_kernel(const int32_t* slot_scores, const uint32_t* slot_index, uint32_t n_slots,
                                  uint64_t* keys) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_slots; i += gridDim.x * blockDim.x) {
        const uint32_t idx = slot_index[i];
        keys[i] = idx == kNoSequence
                      ? 0ull
                      : (static_cast<uint64_t>(static_cast<uint32_t>(slot_scores[i])) << 32) | (0xFFFFFFFFu - idx);
    }
}

__global__ void scatter_scores_kernel(const int32_t* slot_scores, const uint32_t* slot_index, uint32_t n_slots,
                                      int32_t* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_slots; i += gridDim.x * blockDim.x) {
        const uint32_t idx = slot_index[i];
        if (idx != kNoSequence) out[idx] = slot_scores[i];
    }
}

// Sort `s` (kSelectSlice keys in shared memory) descending.
__device__ __forceinline__ void bitonic_sort_desc(uint64_t* s) {
    for (uint32_t size = 2; size <= kSelectSlice; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (uint32_t t = threadIdx.x; t < kSelectSlice / 2; t += blockDim.x) {
                const uint32_t lo = 2 * t - (t & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool desc = (lo & size) == 0;
                const uint64_t a = s[lo], b = s[hi];
                if ((a < b) == desc) s[lo] = b, s[hi] = a;
            }
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSelectThreads) select_topk_kernel(const uint64_t* in, uint64_t n, uint32_t k,
                                                                      uint64_t* out) {
    __shared__ uint64_t s[kSelectSlice];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSelectSlice;
    for (uint32_t i = threadIdx.x; i < kSelectSlice; i += blockDim.x) s[i] = base + i < n ? in[base + i] : 0ull;
    bitonic_sort_desc(s);
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) out[static_cast<uint64_t>(blockIdx.x) * k + i] = s[i];
}

// Full descending bitonic sort in global memory for k > kSelectMaxK (n padded to a power of two).
__global__ void bitonic_step_kernel(uint64_t* keys, uint64_t n_pow2, uint64_t size, uint64_t stride) {
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < n_pow2 / 2;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t lo = 2 * t - (t & (stride - 1));
        const uint64_t hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const uint64_t a = keys[lo], b = keys[hi];
        if ((a < b) == desc) keys[lo] = b, keys[hi] = a;
    }
}

}  // namespace swb
