// duo.cuh -- the on-chip tile pipeline for two STREAMS of queries at once.
//
// pipeline_s16_kernel packs two database sequences into the int16 halves of every DPX word; the two halves then
// need two different profile rows (one per residue), and one PRMT per pair of cells stitches the two int8
// entries into a substitution word: 4.5 ALU-pipe instructions per two cells, the pipe that bounds the kernel.
// Here the halves are two QUERIES against the same sequence: same residue, same column, so the profile can hold
// the finished s16x2 word (query A's entry in the low half, query B's in the high half) and the PRMT disappears:
// 3.5 ALU-pipe instructions per two cells.  A thread now carries one sequence; an item is one half (32 sequences)
// of an interleaved group of 64.
//
// Everything else is pipeline.cuh's design: slot stream over a CTA's 16 warps, border rings in shared memory, the
// link into warp 0 through global memory for queries of more than 16 tiles, items by ticket.  One difference: the
// 4-byte profile of a long query does not fit shared memory, so each warp keeps only the slice of its current tile
// (25 rows x 32 columns, 3.6 KB) and reloads it at every slot start; shared-memory use no longer depends on m.
//
// Streams.  Each half is not one query but a STREAM of queries laid end to end, every query starting on a tile
// boundary (DuoTile): at a query's first tile the inbound border of that half is reset to the matrix edge, and at
// the end of every tile the half's running maximum goes to the score array of the query the tile belongs to.  A
// batch of queries of any lengths is dealt over the two streams so that they end up equally long, and the only
// padding left is each query's last tile (swb_search_many; the pad columns carry substitution score 0, which cannot
// raise a score).
#pragma once
#include "pipeline.cuh"

namespace swb {

// (An 8-byte layout, [column pair][symbol] x 2 words read with LDS.64, was built and measured: 42 instead of 67 shared-memory
// wavefronts per row of 32 columns, bit-exact, and 3 % slower -- 7,239 against 7,455 GCUPS on the sweep: the 8 extra issue
// slots per row cost more than the wavefronts saved; profiles/r02_summary.md.)
constexpr uint32_t kDuoRowWords = kInterTile + 4;                 // 36 words = 144 B: rows 16 B apart modulo 128
constexpr uint32_t kDuoSliceWords = kProfRows * kDuoRowWords;     // one tile's profile slice: 900 words
constexpr uint32_t kDuoSliceBytes = (kDuoSliceWords * 4 + 255) & ~255u;

constexpr uint32_t kDuoNone = 0xFFFFFFFFu;

// One 32-column tile of the two streams.
struct DuoTile {
    uint32_t qa, qb;          // query (number within the scan) the low / high half belongs to, kDuoNone: padding
    uint32_t reset;           // bit 0 / bit 1: the low / high half starts a query here
    uint32_t a_off, a_left;   // low half: offset of the tile's first column in the scan's concatenated query codes,
    uint32_t b_off, b_left;   // and how many real columns are left from there (0: padding); same for the high half
    uint32_t reserved;
};

// prof2[tile][symbol][36]: word c = (M[s][a_c] + open) | (M[s][b_c] + open) << 16 for the tile's columns c < 32;
// pad rows, pad columns (past a query's end) and the 4 filler words carry `open` (substitution score 0).
struct DuoProfileParams {
    const uint8_t* codes;     // the scan's queries, concatenated
    const DuoTile* tiles;
    const int32_t* matrix;
    int32_t shift;
    uint32_t n_tiles;
    uint32_t* prof2;
};

__global__ void build_duo_profile_kernel(DuoProfileParams p) {
    const uint32_t total = p.n_tiles * kDuoSliceWords;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t tile = i / kDuoSliceWords, rem = i % kDuoSliceWords;
        const uint32_t s = rem / kDuoRowWords, c = rem % kDuoRowWords;
        const DuoTile td = p.tiles[tile];
        int32_t va = p.shift, vb = p.shift;
        if (s < kAlphabet && c < kInterTile) {
            if (c < td.a_left) va += p.matrix[s * kAlphabet + p.codes[td.a_off + c]];
            if (c < td.b_left) vb += p.matrix[s * kAlphabet + p.codes[td.b_off + c]];
        }
        p.prof2[i] = (static_cast<uint32_t>(va) & 0xffffu) | (static_cast<uint32_t>(vb) << 16);
    }
}

struct DuoParams {
    const uint4* codes;
    const GroupDesc* groups;
    uint32_t n_items;         // whole items: 2 x groups, item i = half (i & 1) of group (i >> 1), longest first;
                              // pass items: 2 x groups x n_passes
    uint32_t pass_items;      // 1: an item is ONE PASS (16 tiles) of a half-group; consecutive passes of a half-group may
                              // run on different CTAs, linked through the global border rows and `progress`
    uint32_t n_passes;        // ceil(n_tiles / 16)
    uint32_t window;          // pass items are handed out pass-major within windows of this many half-groups
    uint32_t* progress;       // [2 x groups][n_passes]: chunks the pass's last warp has published, zeroed per scan
    const uint32_t* prof2;
    const DuoTile* tiles;     // [n_tiles]
    uint32_t n_tiles;         // tiles of the longer stream
    uint32_t ring_chunks;
    uint32_t lag_div;
    uint2* border0;           // database-shaped border rows for the link into warp 0: half 0 / half 1 of a group
    uint2* border1;
    int32_t* scores;          // [queries of the scan][n_slots], zeroed per scan, updated with atomicMax
    uint32_t n_slots;
    uint32_t* ticket;
    uint32_t neg_open2, neg_ext2;
    unsigned long long* stats;   // SWB_PIPE_STATS builds: [cta][warp][4] clocks waited on input / output / item fetch, total
};

// kPassItems: compile the pass-item form (DuoParams::pass_items); the whole-item form keeps its register allocation.
template <int T, int kThreads, bool kPassItems>
__global__ void __launch_bounds__(kThreads, 1) duo_pipeline_kernel(DuoParams p) {
    static_assert(T == 32, "the slice layout assumes 32-column tiles");
    extern __shared__ __align__(256) uint8_t smem[];
    PipeCtl* ctl = reinterpret_cast<PipeCtl*>(smem);
    uint8_t* slices = smem + sizeof(PipeCtl);
    uint8_t* rings = slices + kPipeWarps * kDuoSliceBytes;
    {
        uint32_t* c = reinterpret_cast<uint32_t*>(ctl);
        for (uint32_t i = threadIdx.x; i < sizeof(PipeCtl) / 4; i += kThreads) c[i] = 0;
        __syncthreads();
    }

    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t next = (warp + 1) % kPipeWarps;
    const bool wrap = p.n_tiles > kPipeWarps;
    const uint32_t NO = p.neg_open2, NE = p.neg_ext2;
    const uint32_t ring_mask = p.ring_chunks - 1;
    const uint32_t ring_bytes = p.ring_chunks * kPipeChunkBytes;
    const uint8_t* ring_in = rings + warp * ring_bytes + lane * 8;
    const uint32_t ring_stage = static_cast<uint32_t>(__cvta_generic_to_shared(rings)) + lane * 16;
    uint8_t* ring_out = rings + next * ring_bytes + lane * 8;
    uint32_t* const slice = reinterpret_cast<uint32_t*>(slices + warp * kDuoSliceBytes);
    uint32_t in_pos = 0, out_pos = 0;

#ifdef SWB_PIPE_STATS
    long long w_in = 0, w_out = 0, w_item = 0;
    const long long t_begin = clock64();
#define SWB_STAT(acc, stmt) { const long long t0__ = clock64(); stmt; acc += clock64() - t0__; }
#else
#define SWB_STAT(acc, stmt) { stmt; }
#endif
    const uint32_t n_half_groups = kPassItems ? p.n_items / p.n_passes : p.n_items;
    for (uint32_t slot = warp;; slot += kPipeWarps) {
        const uint32_t tiles_per_item = kPassItems ? kPipeWarps : p.n_tiles;
        const uint32_t item = slot / tiles_per_item;
        uint32_t tile = slot - item * tiles_per_item;
        uint32_t it;
        SWB_STAT(w_item, it = pipe_item(p.ticket, p.n_items, 0u, ctl, item, lane));
        if (it == kPipeEnd) break;
        if (lane == 0) ctl->warp_item[warp] = item;
        uint32_t hg = it, pass = 0;
        if (kPassItems) {
            // ticket -> (half-group, pass): pass-major within a window of half-groups, so that by the time pass p + 1 of
            // a half-group is handed out its pass p has been running for a whole window of tickets
            const uint32_t per_window = p.window * p.n_passes;
            const uint32_t w = it / per_window, r = it - w * per_window;
            const uint32_t in_window = min(p.window, n_half_groups - w * p.window);
            pass = r / in_window;
            hg = w * p.window + (r - pass * in_window);
            tile += pass * kPipeWarps;
            if (tile >= p.n_tiles) continue;   // the last pass is shorter: nothing for this warp
        }
        const uint32_t half = hg & 1;
        const GroupDesc gd = p.groups[hg >> 1];
        const bool first = tile == 0, last = tile + 1 == p.n_tiles;
        // pass items: the link into the pass's first warp comes from another item (maybe another CTA)
        const bool wrap_in = kPassItems ? (warp == 0 && pass > 0) : (wrap && warp == 0);
        const bool wrap_out = kPassItems ? (next == 0 && !last) : (wrap && next == 0);
        const uint32_t* prog_in = p.progress + static_cast<size_t>(hg) * p.n_passes + (pass ? pass - 1 : 0);
        uint32_t* prog_out = p.progress + static_cast<size_t>(hg) * p.n_passes + pass;
        const DuoTile td = p.tiles[tile];
        // a half that starts a query here takes the matrix edge instead of its left neighbour's border
        const uint32_t keep = ((td.reset & 1u) ? 0u : 0x0000FFFFu) | ((td.reset & 2u) ? 0u : 0xFFFF0000u);
        const uint32_t edge = NO & ~keep;
        const uint4* gcodes = p.codes + gd.chunk_base * 32 + lane;
        uint2* const gb = (half ? p.border1 : p.border0) + gd.chunk_base * kRowsPerChunk * 32;
        uint8_t* gborder = reinterpret_cast<uint8_t*>(gb + lane);
        const uint8_t* gstage = reinterpret_cast<const uint8_t*>(gb) + lane * 16;
        const uint32_t in_end = in_pos + gd.n_chunks;
        const uint32_t lag = max(1u, min(p.ring_chunks - 1, gd.n_chunks / p.lag_div));

        // this tile's profile slice -> the warp's private shared-memory copy
        {
            const uint4* src = reinterpret_cast<const uint4*>(p.prof2 + static_cast<size_t>(tile) * kDuoSliceWords);
            uint4* dst = reinterpret_cast<uint4*>(slice);
            __syncwarp();
            for (uint32_t i = lane; i < kDuoSliceWords / 4; i += 32) dst[i] = __ldg(src + i);
            __syncwarp();
        }

        uint32_t Hm[T], F[T];
#pragma unroll
        for (int k = 0; k < T; ++k) Hm[k] = NO, F[k] = NO;
        uint32_t diag_in = NO, best = 0;
        uint4 cw = __ldg(gcodes);
        const uint32_t in_base = in_pos;
        uint32_t staged = in_pos;
        uint32_t seen = in_pos;   // pass items: the inbound link's published position, as last ACQUIRED

        for (uint32_t chunk = 0; chunk < gd.n_chunks; ++chunk) {
            const uint4 cur = cw;
            if (chunk + 1 < gd.n_chunks) cw = __ldg(gcodes + static_cast<size_t>(chunk + 1) * 32);
            if (!first) {
                if (wrap_in) {
                    // published chunks of the inbound link, as a position on it: the ring's head counter, or (pass
                    // items) the producing pass's progress counter in global memory
                    // Pass items: relaxed polls, and ONE ld.acquire.gpu per observed advance (kernels.cuh, wait_progress):
                    // rows are only ever staged up to an acquired value of the counter, so every cp.async below is
                    // ordered after the producing warp's stores + st.release.gpu.  All lanes do the same loads.
                    auto published = [&]() {
                        if (!kPassItems) return lds_acquire(&ctl->head[0]);
                        if (in_base + ld_poll(prog_in) > seen) seen = in_base + ld_acquire_gpu(prog_in);
                        return seen;
                    };
                    if (staged == in_pos) {
                        const uint32_t need = min(in_pos + 2, in_end);
                        SWB_STAT(w_in, while (published() < need) __nanosleep(kPipePollNs));
                        stage_chunk(ring_stage + (staged & ring_mask) * kPipeChunkBytes,
                                    gstage + static_cast<size_t>(staged - in_base) * kPipeChunkBytes);
                        asm volatile("cp.async.commit_group;" ::: "memory");
                        ++staged;
                    }
                    // chunk in_pos must have landed; the one behind it may stay in flight (one commit group per chunk)
                    if (staged - in_pos >= 2) asm volatile("cp.async.wait_group 1;" ::: "memory");
                    else asm volatile("cp.async.wait_group 0;" ::: "memory");
                    __syncwarp();
                    // keep up to two chunks requested beyond the current one (ring of 4; one beyond for a ring of 2)
                    const uint32_t upto = min(min(published(), in_end), in_pos + min(3u, p.ring_chunks));
                    if (staged < upto) {
                        stage_chunk(ring_stage + (staged & ring_mask) * kPipeChunkBytes,
                                    gstage + static_cast<size_t>(staged - in_base) * kPipeChunkBytes);
                        asm volatile("cp.async.commit_group;" ::: "memory");
                        ++staged;
                    }
                    if (staged < upto) {
                        stage_chunk(ring_stage + (staged & ring_mask) * kPipeChunkBytes,
                                    gstage + static_cast<size_t>(staged - in_base) * kPipeChunkBytes);
                        asm volatile("cp.async.commit_group;" ::: "memory");
                        ++staged;
                    }
                } else {
                    const uint32_t need = min(chunk == 0 ? in_pos + lag : in_pos + 1, in_end);
                    SWB_STAT(w_in, while (lds_acquire(&ctl->head[warp]) < need) __nanosleep(kPipePollNs));
                }
            }
            if (!last && !wrap_out)
                SWB_STAT(w_out, while (out_pos - lds_acquire(&ctl->tail[next]) >= p.ring_chunks) __nanosleep(kPipePollNs));
            const uint2* bin = reinterpret_cast<const uint2*>(ring_in + (in_pos & ring_mask) * kPipeChunkBytes);
            uint8_t* bout = wrap_out ? gborder + static_cast<size_t>(chunk) * kPipeChunkBytes
                                     : ring_out + (out_pos & ring_mask) * kPipeChunkBytes;
            const uint32_t r_lo = half ? cur.z : cur.x, r_hi = half ? cur.w : cur.y;   // this half's 8 residues
            // Two rows at a time, the second one column behind the first: its cell (r+1, k) needs (r, k) and (r, k-1),
            // which the first row has just produced, and the two E -> H -> Hm chains are independent of each other,
            // which doubles the instructions a warp can have in flight (the chains, not the ALU pipe, were what
            // the single-row sweep waited on).  Both rows update Hm[k] and F[k] in place, the second after the first.
#pragma unroll
            for (int rp = 0; rp < static_cast<int>(kRowsPerChunk); rp += 2) {
                const uint32_t aA = ((rp < 4 ? r_lo : r_hi) >> (8 * (rp & 3))) & 0xffu;
                const uint32_t aB = ((rp + 1 < 4 ? r_lo : r_hi) >> (8 * ((rp + 1) & 3))) & 0xffu;
                const uint4* prowA = reinterpret_cast<const uint4*>(slice + aA * kDuoRowWords);
                const uint4* prowB = reinterpret_cast<const uint4*>(slice + aB * kDuoRowWords);
                uint2 biA = make_uint2(NO, NO), biB = make_uint2(NO, NO);
                if (!first) {
                    biA = bin[rp * 32], biB = bin[(rp + 1) * 32];
                    biA.x = (biA.x & keep) | edge, biA.y = (biA.y & keep) | edge;
                    biB.x = (biB.x & keep) | edge, biB.y = (biB.y & keep) | edge;
                }
                uint32_t hlA = biA.x, EA = biA.y, hlB = biB.x, EB = biB.y;
                uint4 swA = prowA[0], swB = prowB[0];
                uint32_t dA = __vadd2(diag_in, swA.x);   // (row A, column 0): diagonal = the previous row's inbound Hm
                uint32_t dB = __vadd2(hlA, swB.x);       // (row B, column 0): diagonal = row A's inbound Hm
                diag_in = hlB;
                uint32_t seenA = 0;
#pragma unroll
                for (int k = 0; k <= T; ++k) {
                    // row A, column k
                    if (k < T) {
                        const uint32_t sA = (k & 3) == 3 ? 0u : (k & 3) == 0 ? swA.y : (k & 3) == 1 ? swA.z : swA.w;   // column k + 1's word
                        EA = __viaddmax_s16x2(EA, NE, hlA);
                        F[k] = __viaddmax_s16x2(F[k], NE, Hm[k]);
                        const uint32_t dcur = dA;
                        if ((k & 3) == 3) {
                            if (k + 1 < T) {
                                swA = prowA[(k + 1) / 4];
                                dA = __vadd2(Hm[k], swA.x);
                            }
                        } else {
                            dA = __vadd2(Hm[k], sA);
                        }
                        hlA = __vadd2(__vimax3_s16x2_relu(dcur, EA, F[k]), NO);
                        Hm[k] = hlA;
                        if (k == 0) best = __vmaxs2(best, dcur);
                        else seenA = dcur;
                    }
                    // row B, column k - 1
                    if (k >= 1) {
                        const int c = k - 1;
                        const uint32_t sB = (c & 3) == 3 ? 0u : (c & 3) == 0 ? swB.y : (c & 3) == 1 ? swB.z : swB.w;
                        EB = __viaddmax_s16x2(EB, NE, hlB);
                        F[c] = __viaddmax_s16x2(F[c], NE, Hm[c]);
                        const uint32_t dcur = dB;
                        if ((c & 3) == 3) {
                            if (c + 1 < T) {
                                swB = prowB[(c + 1) / 4];
                                dB = __vadd2(Hm[c], swB.x);
                            }
                        } else {
                            dB = __vadd2(Hm[c], sB);
                        }
                        hlB = __vadd2(__vimax3_s16x2_relu(dcur, EB, F[c]), NO);
                        Hm[c] = hlB;
                        // the running maximum over the diagonal terms (exact, see sweep_unit_s16): one VIMNMX3 per two cells
                        best = k < T ? __vimax3_s16x2(best, seenA, dcur) : __vmaxs2(best, dcur);
                    }
                }
                if (!last) {
                    *reinterpret_cast<uint2*>(bout + rp * 256) = make_uint2(hlA, EA);
                    *reinterpret_cast<uint2*>(bout + (rp + 1) * 256) = make_uint2(hlB, EB);
                }
            }
            __syncwarp();
            if (!first) {
                ++in_pos;
                if (lane == 0 && !wrap_in) sts_release(&ctl->tail[warp], in_pos);
            }
            if (!last) {
                ++out_pos;
                if (lane == 0) {
                    if (wrap_out && kPassItems) st_release(prog_out, chunk + 1);   // release.gpu: the rows are in L2 first
                    else {
                        if (wrap_out) __threadfence();
                        sts_release(&ctl->head[next], out_pos);
                    }
                }
            }
        }

        // halves -> this lane's sequence against the two queries this tile belongs to
        const int32_t sa = static_cast<int32_t>(best & 0xffffu);
        const int32_t sb = static_cast<int32_t>(best >> 16);
        const uint32_t sl = gd.first_slot + half * 32 + lane;
        if (sa && td.qa != kDuoNone) atomicMax(p.scores + static_cast<size_t>(td.qa) * p.n_slots + sl, sa);
        if (sb && td.qb != kDuoNone) atomicMax(p.scores + static_cast<size_t>(td.qb) * p.n_slots + sl, sb);
    }
    if (lane == 0) ctl->warp_item[warp] = kPipeEnd;
#ifdef SWB_PIPE_STATS
    if (lane == 0 && p.stats) {
        unsigned long long* o = p.stats + (static_cast<size_t>(blockIdx.x) * kPipeWarps + warp) * 4;
        o[0] = w_in, o[1] = w_out, o[2] = w_item, o[3] = clock64() - t_begin;
    }
#endif
#undef SWB_STAT
}

}  // namespace swb
