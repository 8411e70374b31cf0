// pipeline.cuh -- the on-chip tile pipeline: packed-int16 DPX scan whose tile borders never leave the SM.
//
// Same arithmetic, same thread mapping and same inner loop as wavefront_s16_kernel (kernels.cuh): one thread
// carries two sequences in the int16 halves of every DPX word and keeps Hm and F of a 32-column query tile in
// registers.  What changes is who works on what.  In the wavefront kernel every warp sweeps its own group and
// hands the (Hm, E) of a tile's last column to the next tile through a database-shaped array in global memory:
// 16 bytes of traffic per row, tile and lane, ~100 GB per search on a Swiss-Prot-sized database, far beyond
// what L2 can hold (profiles/traffic.json).  Here the 16 warps of a CTA work on the SAME group at the same
// time, on consecutive tiles, each a few rows behind its left neighbour, and the border rows travel through
// small rings in shared memory.  HBM sees the residues (once per CTA pass; L1 serves the other 15 warps) and
// two atomics per sequence and tile -- nothing else.
//
// Slot stream.  A CTA takes items (= groups, longest first) from a global ticket counter.  The tiles of its
// successive items form one continuous stream of slots,  slot = item * n_tiles + tile,  and warp w processes
// the slots congruent to w modulo 16, in order.  Slot s reads its inbound border from the ring filled by slot
// s - 1 (the warp to its left, cyclically) and writes its outbound border into the ring of the warp to its
// right.  Because the stream is continuous there is no pipeline fill or drain per group: a warp that finishes
// tile t of one group goes straight on to its next slot, which may belong to the next group.  A query with
// more than 16 tiles wraps around: warp 15 feeds warp 0, which takes it up once its previous tile is done; the
// ring's back-pressure holds the producers until then and in steady state all 16 warps are busy.
//
// Flow control.  Each ring has a head (chunks of 8 rows produced) and a tail (chunks consumed) in shared
// memory; a producer waits for space, a consumer for data, once per chunk.  Dependencies always point to an
// earlier slot, every warp processes its slots in order and all 16 warps are resident, so the slot with the
// lowest index among the unfinished ones can always advance: no deadlock.
//
// Items are fetched on demand, in order, under a CTA-local lock (the first warp that needs item j fetches it);
// once the ticket counter runs past the end every later item is the end marker and warps leave when they
// meet it.
#pragma once
#include "kernels.cuh"

namespace swb {

constexpr uint32_t kPipeWarps = kInterThreads / 32;
constexpr uint32_t kPipeItemRing = 64;                   // CTA-local ring of fetched items
constexpr uint32_t kPipeChunkBytes = kRowsPerChunk * 32 * 8;   // one chunk of border rows: 8 rows x 32 lanes x (Hm, E)
constexpr uint32_t kPipeEnd = 0xFFFFFFFFu;
#ifndef SWB_PIPE_POLL_NS
#define SWB_PIPE_POLL_NS 20
#endif
constexpr uint32_t kPipePollNs = SWB_PIPE_POLL_NS;   // back-off between two looks at a ring counter

struct PipeParams {
    const uint4* codes;
    const GroupDesc* groups;
    uint32_t group_first;     // items are the groups [group_first, group_first + n_items), longest first
    uint32_t n_items;
    const int8_t* prof8;
    uint32_t pstride;
    uint32_t prof_bytes;      // 25 * pstride rounded up to 256
    uint32_t n_tiles;         // ceil(m / 32)
    uint32_t ring_chunks;     // capacity of each ring in chunks (power of two >= 2)
    uint32_t lag_div;         // start lag of a tile = group chunks / lag_div, clamped to [1, ring_chunks - 1]
    uint2* border;            // database-shaped border rows (8 B per row and lane) for the link into warp 0
    int32_t* slot_scores;
    uint32_t* ticket;
    uint32_t neg_open2, neg_ext2;
    unsigned long long* stats;   // SWB_PIPE_STATS builds: [cta][warp][4] clocks waited on input / output / item fetch, total
};

struct PipeCtl {
    uint32_t head[kPipeWarps];        // chunks produced into the ring that warp w reads
    uint32_t tail[kPipeWarps];        // chunks warp w has consumed from it
    uint32_t warp_item[kPipeWarps];   // item each warp is working on (kPipeEnd once it has left)
    uint32_t fetched;                 // items fetched so far
    uint32_t lock;
    uint32_t pad[14];
    uint32_t item_group[kPipeItemRing];
};

__device__ __forceinline__ uint32_t lds_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))) : "memory");
    return v;
}
// One chunk of border rows (2 KB, contiguous in both places) global -> shared, asynchronously; 64 B per lane.
__device__ __forceinline__ void stage_chunk(uint32_t dst, const uint8_t* src) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + i * 512), "l"(src + i * 512) : "memory");
}

// A border row from either link: a shared-memory ring or (warp 0) global memory written by another warp of this
// CTA; generic address, served by L2 when global.
__device__ __forceinline__ uint2 ld_border(const uint8_t* p) {
    uint2 v;
    asm volatile("ld.relaxed.gpu.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void sts_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "r"(v) : "memory");
}

// Item `item` of this CTA -> first_id + its ticket (tickets 0 .. n_items - 1 are handed out once each, GPU-wide), or
// kPipeEnd.  Called by whole warps; lane 0 does the work.
__device__ __forceinline__ uint32_t pipe_item(uint32_t* ticket, uint32_t n_items, uint32_t first_id, PipeCtl* ctl, uint32_t item,
                                              uint32_t lane) {
    uint32_t g = 0;
    if (lane == 0) {
        while (lds_acquire(&ctl->fetched) <= item) {
            if (atomicCAS(&ctl->lock, 0u, 1u) == 0u) {
                const uint32_t f = lds_acquire(&ctl->fetched);
                if (f <= item) {
                    // the entry being overwritten belonged to item f - kPipeItemRing: every warp must be past it
                    if (f >= kPipeItemRing)
                        for (uint32_t w = 0; w < kPipeWarps; ++w)
                            for (;;) {
                                const uint32_t at = lds_relaxed(&ctl->warp_item[w]);   // kPipeEnd: the warp has left
                                if (at == kPipeEnd || at + kPipeItemRing > f) break;
                                __nanosleep(100);
                            }
                    const uint32_t t = atomicAdd(ticket, 1u);
                    ctl->item_group[f % kPipeItemRing] = t < n_items ? first_id + t : kPipeEnd;
                    sts_release(&ctl->fetched, f + 1);
                }
                sts_release(&ctl->lock, 0u);
            } else {
                __nanosleep(100);
            }
        }
        g = ctl->item_group[item % kPipeItemRing];
    }
    return __shfl_sync(0xffffffffu, g, 0);
}

// kSlice: the query's profile does not fit shared memory next to the rings (m beyond ~6,500): every warp keeps the 25 x 32 B
// slice of its current tile only (rows kPipeSliceStride apart) and reloads it from the profile in global memory at every slot
// start, as the two-stream kernel does (scan_plan.hpp: pipe_rings_for).  prof_bytes is then the 16 slices' size.
template <int T, int kThreads, bool kSlice>
__global__ void __launch_bounds__(kThreads, 1) pipeline_s16_kernel(PipeParams p) {
    static_assert(T % 16 == 0, "tile width must be a multiple of 16 columns");
    static_assert(!kSlice || T == 32, "the slice layout assumes 32-column tiles");
    static_assert(kThreads == kPipeWarps * 32, "CTA shape");
    static_assert(kPipeWarps == kPipeWarpsHost && kProfRows * kPipeSliceStride <= kPipeSliceBytes, "slice geometry");
    extern __shared__ __align__(256) uint8_t smem[];
    int8_t* prof = reinterpret_cast<int8_t*>(smem);
    PipeCtl* ctl = reinterpret_cast<PipeCtl*>(smem + p.prof_bytes);
    uint8_t* rings = smem + p.prof_bytes + sizeof(PipeCtl);

    {
        if (!kSlice) {
            const uint32_t n16 = kProfRows * p.pstride / 16;
            const uint4* src = reinterpret_cast<const uint4*>(p.prof8);
            uint4* dst = reinterpret_cast<uint4*>(smem);
            for (uint32_t i = threadIdx.x; i < n16; i += kThreads) dst[i] = src[i];
        }
        uint32_t* c = reinterpret_cast<uint32_t*>(ctl);
        for (uint32_t i = threadIdx.x; i < sizeof(PipeCtl) / 4; i += kThreads) c[i] = 0;
        __syncthreads();
    }

    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t next = (warp + 1) % kPipeWarps;
    // The link into warp 0 closes the cycle of 16 warps.  A smem ring there would deadlock on groups taller
    // than the rings' total capacity (warp 0 cannot start tile 16 before it has finished tile 0, and could
    // not finish it with every ring downstream full), so this one link goes through the database-shaped border
    // array in global memory: unbounded, flow-controlled by its head counter only.  It carries 1/16 of the
    // border rows and is read back one pass later from L2.
    // Queries of at most 16 tiles never put two tiles of one group on the same warp, so there the cycle cannot
    // close and all 16 links are rings.
    const bool wrap = p.n_tiles > kPipeWarps;
    const bool wrap_in = wrap && warp == 0, wrap_out = wrap && next == 0;
    const uint32_t NO = p.neg_open2, NE = p.neg_ext2;
    const uint32_t ring_mask = p.ring_chunks - 1;
    const uint32_t ring_bytes = p.ring_chunks * kPipeChunkBytes;
    const uint8_t* ring_in = rings + warp * ring_bytes + lane * 8;
    const uint32_t ring_stage = static_cast<uint32_t>(__cvta_generic_to_shared(rings)) + lane * 16;   // warp 0's ring, as a copy target
    uint8_t* ring_out = rings + next * ring_bytes + lane * 8;
    uint32_t in_pos = 0, out_pos = 0;   // chunks consumed from the inbound / produced into the outbound link so far

#ifdef SWB_PIPE_STATS
    long long w_in = 0, w_out = 0, w_item = 0;
    const long long t_begin = clock64();
#define SWB_STAT(acc, stmt) { const long long t0__ = clock64(); stmt; acc += clock64() - t0__; }
#else
#define SWB_STAT(acc, stmt) { stmt; }
#endif
    for (uint32_t slot = warp;; slot += kPipeWarps) {
        const uint32_t item = slot / p.n_tiles, tile = slot - item * p.n_tiles;
        uint32_t g;
        SWB_STAT(w_item, g = pipe_item(p.ticket, p.n_items, p.group_first, ctl, item, lane));
        if (g == kPipeEnd) break;
        if (lane == 0) ctl->warp_item[warp] = item;
        const GroupDesc gd = p.groups[g];
        const bool first = tile == 0, last = tile + 1 == p.n_tiles;
        const int8_t* ptile = kSlice ? prof + (threadIdx.x >> 5) * kPipeSliceBytes : prof + tile * T;
        const uint32_t pstr = kSlice ? kPipeSliceStride : p.pstride;
        if (kSlice) {
            // this tile's 25 rows x 32 B -> the warp's own slice (50 loads of 16 B over the warp)
            __syncwarp();
            for (uint32_t i = lane; i < kProfRows * 2; i += 32) {
                const uint32_t row = i >> 1, part = i & 1;
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.prof8 + static_cast<size_t>(row) * p.pstride + tile * T) + part);
                reinterpret_cast<uint4*>(const_cast<int8_t*>(ptile) + row * kPipeSliceStride)[part] = v;
            }
            __syncwarp();
        }
        const uint4* gcodes = p.codes + gd.chunk_base * 32 + lane;
        uint8_t* gborder = reinterpret_cast<uint8_t*>(p.border + gd.chunk_base * kRowsPerChunk * 32 + lane);
        const uint8_t* gstage = reinterpret_cast<const uint8_t*>(p.border + gd.chunk_base * kRowsPerChunk * 32) + lane * 16;
        const uint32_t in_end = in_pos + gd.n_chunks;
        const uint32_t lag = max(1u, min(p.ring_chunks - 1, gd.n_chunks / p.lag_div));

        uint32_t Hm[T], F[T];
#pragma unroll
        for (int k = 0; k < T; ++k) Hm[k] = NO, F[k] = NO;
        uint32_t diag_in = NO, best = 0;
        uint4 cw = __ldg(gcodes);
        const uint32_t in_base = in_pos;   // link position of this slot's chunk 0
        uint32_t staged = in_pos;          // warp 0: chunks of the global link already requested into its ring

        for (uint32_t chunk = 0; chunk < gd.n_chunks; ++chunk) {
            const uint4 cur = cw;
            if (chunk + 1 < gd.n_chunks) cw = __ldg(gcodes + static_cast<size_t>(chunk + 1) * 32);
            if (!first) {
                if (wrap_in) {
                    // Warp 0 leads the pipeline: whenever it stalls, the fifteen warps behind it run dry one after
                    // the other.  Its inbound rows come from global memory, so they are staged into its (otherwise
                    // unused) ring with cp.async one chunk ahead and read from shared memory like everyone else's.
                    if (staged == in_pos) {
                        // nothing in flight (start of a slot, or the producer is close): wait until two chunks are
                        // published, so that from here on the next chunk can always be requested while this one is
                        // being consumed
                        const uint32_t need = min(in_pos + 2, in_end);
                        SWB_STAT(w_in, while (lds_acquire(&ctl->head[0]) < need) __nanosleep(kPipePollNs));
                        stage_chunk(ring_stage + (staged & ring_mask) * kPipeChunkBytes,
                                    gstage + static_cast<size_t>(staged - in_base) * kPipeChunkBytes);
                        ++staged;
                    }
                    asm volatile("cp.async.wait_all;" ::: "memory");
                    __syncwarp();
                    if (staged < in_end && lds_acquire(&ctl->head[0]) > staged) {
                        stage_chunk(ring_stage + (staged & ring_mask) * kPipeChunkBytes,
                                    gstage + static_cast<size_t>(staged - in_base) * kPipeChunkBytes);
                        ++staged;
                    }
                } else {
                    // A tile starts `lag` chunks behind its left neighbour: a cushion against scheduling jitter.
                    const uint32_t need = min(chunk == 0 ? in_pos + lag : in_pos + 1, in_end);
                    SWB_STAT(w_in, while (lds_acquire(&ctl->head[warp]) < need) __nanosleep(kPipePollNs));
                }
            }
            if (!last && !wrap_out)
                SWB_STAT(w_out, while (out_pos - lds_acquire(&ctl->tail[next]) >= p.ring_chunks) __nanosleep(kPipePollNs));
            const uint2* bin = reinterpret_cast<const uint2*>(ring_in + (in_pos & ring_mask) * kPipeChunkBytes);
            uint8_t* bout = wrap_out ? gborder + static_cast<size_t>(chunk) * kPipeChunkBytes
                                     : ring_out + (out_pos & ring_mask) * kPipeChunkBytes;
            uint2 bnext = make_uint2(NO, NO);
            if (!first) bnext = bin[0];
            // the first 16 columns' profile bytes of a row are loaded while the previous row is computed
            const int8_t* pa_next = ptile + (cur.x & 0xffu) * pstr;
            const int8_t* pb_next = ptile + (cur.z & 0xffu) * pstr;
            uint4 va_next = *reinterpret_cast<const uint4*>(pa_next), vb_next = *reinterpret_cast<const uint4*>(pb_next);
#pragma unroll
            for (int r = 0; r < static_cast<int>(kRowsPerChunk); ++r) {
                const int8_t* pa = pa_next;
                const int8_t* pb = pb_next;
                uint32_t wA[T / 4], wB[T / 4];
                wA[0] = va_next.x, wA[1] = va_next.y, wA[2] = va_next.z, wA[3] = va_next.w;
                wB[0] = vb_next.x, wB[1] = vb_next.y, wB[2] = vb_next.z, wB[3] = vb_next.w;
#pragma unroll
                for (int i = 1; i < T / 16; ++i) {
                    const uint4 va = reinterpret_cast<const uint4*>(pa)[i], vb = reinterpret_cast<const uint4*>(pb)[i];
                    wA[4 * i] = va.x, wA[4 * i + 1] = va.y, wA[4 * i + 2] = va.z, wA[4 * i + 3] = va.w;
                    wB[4 * i] = vb.x, wB[4 * i + 1] = vb.y, wB[4 * i + 2] = vb.z, wB[4 * i + 3] = vb.w;
                }
                if (r + 1 < static_cast<int>(kRowsPerChunk)) {
                    const uint32_t wa = r + 1 < 4 ? cur.x : cur.y;
                    const uint32_t wb = r + 1 < 4 ? cur.z : cur.w;
                    pa_next = ptile + ((wa >> (8 * ((r + 1) & 3))) & 0xffu) * pstr;
                    pb_next = ptile + ((wb >> (8 * ((r + 1) & 3))) & 0xffu) * pstr;
                    va_next = *reinterpret_cast<const uint4*>(pa_next);
                    vb_next = *reinterpret_cast<const uint4*>(pb_next);
                }
                const uint2 bi = bnext;   // this row's inbound border, loaded while the previous row was computed
                if (!first && r + 1 < static_cast<int>(kRowsPerChunk)) bnext = bin[(r + 1) * 32];
                uint32_t hl = bi.x;   // Hm of the column left of the tile, this row
                uint32_t E = bi.y;
                // d of a column is formed from the OLD Hm of the column to its left, i.e. before that register is
                // overwritten in place: every Hm[k] and F[k] then stays in one physical register for the whole
                // chunk and the compiler needs no moves to rotate them
                uint32_t d = __vadd2(diag_in, prmt(wA[0], wB[0], 0xC480u));
                diag_in = hl;
#pragma unroll
                for (int k = 0; k < T; k += 2) {
                    const uint32_t s1 = prmt(wA[k / 4], wB[k / 4], (k & 3) == 0 ? 0xD591u : 0xF7B3u);
                    // cell k
                    E = __viaddmax_s16x2(E, NE, hl);
                    F[k] = __viaddmax_s16x2(F[k], NE, Hm[k]);
                    const uint32_t d0 = d;
                    const uint32_t d1 = __vadd2(Hm[k], s1);
                    hl = __vadd2(__vimax3_s16x2_relu(d0, E, F[k]), NO);
                    Hm[k] = hl;
                    // cell k+1
                    E = __viaddmax_s16x2(E, NE, hl);
                    F[k + 1] = __viaddmax_s16x2(F[k + 1], NE, Hm[k + 1]);
                    if (k + 2 < T)
                        d = __vadd2(Hm[k + 1], prmt(wA[(k + 2) / 4], wB[(k + 2) / 4], ((k + 2) & 3) == 0 ? 0xC480u : 0xE6A2u));
                    hl = __vadd2(__vimax3_s16x2_relu(d1, E, F[k + 1]), NO);
                    Hm[k + 1] = hl;
                    best = __vimax3_s16x2(best, d0, d1);   // see sweep_unit_s16: max over the diagonal terms is exact
                }
                if (!last) *reinterpret_cast<uint2*>(bout + r * 256) = make_uint2(hl, E);
            }
            __syncwarp();
            if (!first) {
                ++in_pos;
                if (lane == 0 && !wrap_in) sts_release(&ctl->tail[warp], in_pos);
            }
            if (!last) {
                ++out_pos;
                if (lane == 0) {
                    if (wrap_out) __threadfence();   // the rows must be in L2 before warp 0 is told about them
                    sts_release(&ctl->head[next], out_pos);
                }
            }
        }

        const int32_t sa = static_cast<int32_t>(best & 0xffffu);
        const int32_t sb = static_cast<int32_t>(best >> 16);
        const uint32_t slot_a = gd.first_slot + lane;
        if (sa) atomicMax(p.slot_scores + slot_a, sa);
        if (sb) atomicMax(p.slot_scores + slot_a + 32, sb);
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
