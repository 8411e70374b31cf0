// scan_plan.hpp -- host-only: how one search is divided between the two scan kernels and into work units.
//
// Replaces the reference's chunk lists (detail::make_chunks, scheduler.hpp:130-138: short chunks of
// lane_width*16 sequences, long chunks of one) and its two worker pools (scheduler.hpp:200-213).  Pure
// arithmetic on the packed database's group table; no CUDA, so the CPU test-suite exercises it through
// swb_scan_plan (tests/test_host.py).
//
// Work is counted in row-tiles (one row of one 32-column tile for a group of 64 sequences).
//
// 1. Division of labour (pipeline.cuh).  The on-chip pipeline gives a group one CTA, so a group whose rows
//    exceed about a third of a CTA's fair share of the database would unbalance it: those few tall groups at
//    the head of the sorted list stay with the wavefront kernel, which spreads a group over warps of many SMs,
//    and run next to the pipeline on `wave_sms` SMs of their own.  Queries of fewer than 9 tiles (little border
//    traffic to save, chains too short to keep 16 warps in step) stay with the wavefront kernel entirely unless the
//    search is chain-bound (then separating the tall groups onto SMs of their own is what pays: m = 144 on
//    Swiss-Prot 7.7 -> 6.0 ms); so do databases with fewer than two groups per SM.
// 2. Unit policy of the wavefront kernel (kernels.cuh, GroupMode).  `fair` is one warp's share of its groups.
//      single    the default: one warp scores the group's 64 sequences end to end;
//      split     a group whose sweep exceeds `budget` is cut so that no unit dominates the makespan and there
//                are enough units for every warp, either
//                  by tile   (wavefront of warps, each 2 chunks behind its left neighbour:
//                             efficiency rows / (rows + 16 (tiles - 1))), or
//                  by rows   (blocks of rows, each one tile behind the block above:
//                             efficiency tiles / (tiles + blocks - 1)),
//                whichever wastes less;
//      narrow    even a tile-split group's per-tile chain (rows x 32 columns, strictly sequential in one
//                thread, ~900 clk per row when the SM empties out, against ~1600 clk per row-tile of saturated
//                throughput) would take more than about half the whole search: 8-column tiles cut that chain
//                four-fold.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "pack.hpp"

namespace swb {

// Group modes of the wavefront kernel, decided per search and uploaded next to unit_start.
enum GroupMode : uint8_t {
    kGroupSingle = 0,   // one unit: all tiles of width T, one warp
    kGroupSplit = 1,    // one unit per tile of width T: a wavefront of warps
    kGroupNarrow = 2,   // one unit per tile of width 8: a wavefront with a 4x shorter per-row chain, for groups whose
                        // rows x T sequential chain would otherwise outlast the whole search (short query, very
                        // long sequences)
    kGroupRowBlock = 3  // units are blocks of rows, each swept over all tiles one tile behind the block above; the
                        // efficient split when the query has many tiles and the group few rows (long queries,
                        // small per-GPU shards)
};
constexpr int kNarrowTile = 8;          // columns of a narrow tile ...
constexpr int kNarrowTileFine = 4;      // ... or of a fine one, for the most chain-bound searches
constexpr uint32_t kNarrowChunkBytes = 8 * 32 * 8;   // a block of border rows in a narrow link buffer: 8 rows x 32 lanes x 8 B
constexpr uint32_t kNarrowPairBytesHost = 2 * 4 * kNarrowChunkBytes + 64;   // = kNarrowPairBytes (kernels.cuh): a compute / helper pair's rings

enum ScanPolicy : int { kScanAuto = 0, kScanPipeline = 1, kScanWavefront = 2 };   // = swb_scan_policy

// Tuning knobs; the defaults were measured on B200 (profiles/r01_summary.md), the environment overrides them.
struct ScanKnobs {
    double unit_budget = 0.0;        // SWB200_UNIT_BUDGET: fraction of a warp's fair share above which a group is split (0: automatic)
    bool row_blocks = true;          // SWB200_ROWBLOCKS=0 disables the row-block split
    double narrow_chain = 0.9;       // SWB200_NARROW: a group goes to 8-column tiles when its rows exceed this x fair
    bool pipe = true;                // SWB200_PIPE=0: never use the pipeline under the automatic policy
    uint32_t pipe_min_tiles = 9;     // SWB200_PIPE_MINTILES: fewer tiles -> wavefront kernel only, unless chain-bound
    double pipe_chain = 1.2;         // SWB200_PIPE_CHAIN: chain-bound when max_rows > this x a warp's fair share of the search
    double pipe_tall = 0.35;         // SWB200_PIPE_TALL: groups taller than this x a CTA's fair share of rows go to the wavefront kernel
    double pipe_tall_small = 0.6;    // SWB200_PIPE_TALL_SMALL: ... x this on databases of fewer than 32 groups per SM (shards)
    double wave_margin = 1.25;       // SWB200_PIPE_WAVE_MARGIN: wavefront SMs = its share of the rows x this ...
    double wave_margin_near = 1.6;   // SWB200_PIPE_WAVE_MARGIN_NEAR: ... x this when the search is close to chain-bound ...
    double wave_margin_chain = 2.0;  // SWB200_PIPE_WAVE_MARGIN_CHAIN: ... or x this when chain-bound (its SMs are then
                                     // busy for the whole search whatever their number: +15 % at m = 375, -2 % at m = 1000)
    uint32_t pipe_ring_cap = 4;      // SWB200_PIPE_RING: chunks per shared-memory ring at most (power of two)
    uint32_t pipe_lag_div = 24;      // SWB200_PIPE_LAGDIV: a tile starts group_chunks / this chunks behind its neighbour
    double duo_ratio = 0.75;         // SWB200_DUO: swb_search_many lays its queries out as two streams per scan (duo.cuh); a scan
                                     // is kept when its shorter stream has at least this fraction of the longer one's tiles (the
                                     // two-stream kernel is ~15 % faster per padded cell: below 0.74 the padding eats the gain);
                                     // > 1: never
    uint32_t duo_stream_tiles = 704; // SWB200_DUO_TILES: tiles per stream of a shared scan at most (a tall group's item must not outlast the scan)
    uint32_t duo_pass_items = 1;     // SWB200_DUO_PASS: shared scans hand out one pass (16 tiles) of a half-group per item:
                                     // 1 (default) where whole items do not fit, 2 always, 0 ("off") never
    uint32_t duo_window_mb = 128;    // SWB200_DUO_WINDOW_MB: pass items are handed out pass-major within windows of half-groups whose
                                     // border rows (256 B per database row) stay under this many MB, i.e. resident in L2
    double duo_tall = 1.0;           // SWB200_DUO_TALL: ... and the tallest group's rows x SMs stay under this x the database's rows x 2
                                     // (a half-group is one CTA's item: it must fit that CTA's fair share of the scan)
    double duo_min_groups_per_sm = 2.0; // SWB200_DUO_MINGROUPS: ... and the database has at least this many groups per SM
    double narrow_fine = 8.0;        // SWB200_NARROW_FINE: narrow tiles are 4 columns instead of 8 when the tallest group's rows exceed
                                     // this x a warp's fair share of the search (an 8-column chain, ~95 clk per row, would still be
                                     // about half the search)
    bool narrow_helpers = true;      // SWB200_NARROW_HELPERS=0: narrow units without helper warps (link buffers read by the unit itself)
    double narrow_sms = 0.5;         // SWB200_NARROW_SMS: next to the pipeline, narrow units get a scheduler each (4 warps per SM) on at
                                     // most this fraction of the SMs
    uint64_t narrow_link_rows = 24u << 20; // SWB200_NARROW_LINKROWS: row slots (256 B each) of narrow link buffers at most (6 GiB)
    uint32_t wave_threads = 0;       // SWB200_WAVE_THREADS: CTA size of the wavefront kernel (128, 256 or 512; 0: automatic)
    double wave_thin = 4.0;          // SWB200_WAVE_THIN: next to the pipeline, the wavefront kernel runs 8 warps per SM instead of
                                     // 16 when max_rows exceeds this x a warp's fair share of the search, and 4 warps beyond 1.5 x
                                     // this: its SMs then hold little besides the longest group's chain, which runs faster with
                                     // fewer warps per scheduler (1/8 Swiss-Prot, m = 1000: 8.3 -> 6.4 ms)

    static ScanKnobs from_env() {
        ScanKnobs k;
        auto num = [](const char* name, double fallback) {
            const char* e = std::getenv(name);
            const double v = e ? std::atof(e) : 0.0;
            return v > 0.0 ? v : fallback;
        };
        auto off = [](const char* name) {
            const char* e = std::getenv(name);
            return e && std::string(e) == "0";
        };
        k.unit_budget = num("SWB200_UNIT_BUDGET", 0.0);
        k.row_blocks = !off("SWB200_ROWBLOCKS");
        k.narrow_chain = num("SWB200_NARROW", k.narrow_chain);
        k.pipe = !off("SWB200_PIPE");
        k.pipe_min_tiles = static_cast<uint32_t>(num("SWB200_PIPE_MINTILES", k.pipe_min_tiles));
        k.pipe_chain = num("SWB200_PIPE_CHAIN", k.pipe_chain);
        k.pipe_tall = num("SWB200_PIPE_TALL", k.pipe_tall);
        k.pipe_tall_small = num("SWB200_PIPE_TALL_SMALL", k.pipe_tall_small);
        k.wave_margin = num("SWB200_PIPE_WAVE_MARGIN", k.wave_margin);
        k.wave_margin_chain = num("SWB200_PIPE_WAVE_MARGIN_CHAIN", k.wave_margin_chain);
        k.wave_margin_near = num("SWB200_PIPE_WAVE_MARGIN_NEAR", k.wave_margin_near);
        k.pipe_ring_cap = std::max<uint32_t>(2, static_cast<uint32_t>(num("SWB200_PIPE_RING", k.pipe_ring_cap)));
        k.pipe_lag_div = std::max<uint32_t>(1, static_cast<uint32_t>(num("SWB200_PIPE_LAGDIV", k.pipe_lag_div)));
        k.wave_thin = num("SWB200_WAVE_THIN", k.wave_thin);
        k.wave_threads = static_cast<uint32_t>(num("SWB200_WAVE_THREADS", 0.0));
        k.narrow_fine = num("SWB200_NARROW_FINE", k.narrow_fine);
        k.narrow_helpers = !off("SWB200_NARROW_HELPERS");
        k.narrow_sms = num("SWB200_NARROW_SMS", k.narrow_sms);
        k.narrow_link_rows = static_cast<uint64_t>(num("SWB200_NARROW_LINKROWS", static_cast<double>(k.narrow_link_rows)));
        k.duo_ratio = num("SWB200_DUO", k.duo_ratio);
        k.duo_stream_tiles = std::max<uint32_t>(16, static_cast<uint32_t>(num("SWB200_DUO_TILES", k.duo_stream_tiles)));
        k.duo_tall = num("SWB200_DUO_TALL", k.duo_tall);
        k.duo_window_mb = std::max<uint32_t>(1, static_cast<uint32_t>(num("SWB200_DUO_WINDOW_MB", k.duo_window_mb)));
        if (const char* e = std::getenv("SWB200_DUO_PASS")) k.duo_pass_items = std::string(e) == "off" ? 0u : static_cast<uint32_t>(std::atoi(e));
        k.duo_min_groups_per_sm = num("SWB200_DUO_MINGROUPS", k.duo_min_groups_per_sm);
        return k;
    }
};

struct ScanShape {
    const GroupDesc* groups = nullptr;   // sorted by rows, longest first
    uint32_t n_groups = 0;
    uint64_t padded_rows = 0;            // sum of the groups' padded rows
    uint32_t n_tiles = 0;                // ceil(m / 32)
    uint32_t query_len = 0;              // m
    uint32_t sm_count = 0;
    uint32_t warps_per_cta = 16;
    bool s16 = true;                     // the packed int16 kernels scan (row blocks, narrow tiles, pipeline exist there only)
    int policy = kScanAuto;
    uint32_t pipe_rings = 0;             // chunks per ring that fit next to this query's profile (< 2: no pipeline)
    size_t narrow_room = 0;              // shared memory left next to the profile for the helper warps' rings (wavefront kernel)
};

struct ScanPlan {
    uint32_t pipe_first = 0;   // groups [pipe_first, n_groups) go through the on-chip pipeline, [0, pipe_first) through the wavefront kernel
    uint32_t wave_sms = 0;     // SMs the wavefront kernel gets
    uint32_t wave_threads = 512; // its CTA size
    uint32_t n_units = 0;      // wavefront units
    uint64_t vstate_slots = 0; // tiles of register state handed between row blocks
    uint32_t narrow_tile = kNarrowTile;   // columns of a narrow tile (8 or 4)
    uint32_t n_tiles_narrow = 0;          // ceil(m / narrow_tile)
    uint64_t link_rows = 0;    // row slots of the narrow groups' link buffers (vstate_off[g]: a narrow group's first one)
    bool narrow_staged = false;     // narrow units hand over through link buffers of their own (kernels.cuh: the data is the flag)
    bool narrow_helpers = false;    // ... carried by helper warps through rings in shared memory (CTAs of 4 + 4 warps)
    bool any_narrow = false, any_rowblock = false, chain_bound = false;
    uint32_t n_split = 0, n_narrow = 0, n_rowblock = 0;   // groups per mode (the rest of [0, pipe_first) is single)
    uint64_t wave_rows = 0;    // padded rows of the wavefront kernel's groups
};

// unit_start [n_groups + 1], vstate_off [n_groups], modes [n_groups] are filled for every group (pipeline groups: 0).
inline ScanPlan plan_scan(const ScanShape& in, const ScanKnobs& k, uint32_t* unit_start, uint32_t* vstate_off, uint8_t* modes) {
    ScanPlan pl;
    const uint32_t n_groups = in.n_groups, n_tiles = in.n_tiles;
    auto rows_of = [&](uint32_t g) { return static_cast<uint64_t>(in.groups[g].n_chunks) * kRowsPerChunk; };
    const uint32_t max_rows = n_groups ? static_cast<uint32_t>(rows_of(0)) : 0;

    // ---- 1. which kernel ------------------------------------------------------------------------------------
    pl.pipe_first = n_groups;
    pl.wave_sms = in.sm_count;
    pl.wave_rows = in.padded_rows;
    const double fair_all = static_cast<double>(in.padded_rows) * n_tiles / (static_cast<double>(in.sm_count) * in.warps_per_cta);
    pl.chain_bound = static_cast<double>(max_rows) > k.pipe_chain * fair_all;
    // Narrow units come in two forms.  With link buffers of their own (kernels.cuh: the data is the flag, no fences) a block
    // costs half as much, but every tile runs kNarrowLagBlocks + 1 blocks behind its left neighbour and the links take
    // 256 B per row and tile boundary: that form is for wavefronts that are shallow against the tallest group (short
    // queries), in 4-column tiles for the most chain-bound searches.  Deep wavefronts (many 8-column tiles: long queries)
    // keep the classic hand-over through the border arrays and progress counters.
    pl.narrow_tile = static_cast<double>(max_rows) > k.narrow_fine * fair_all ? kNarrowTileFine : kNarrowTile;
    pl.n_tiles_narrow = (in.query_len + pl.narrow_tile - 1) / pl.narrow_tile;
    // (narrow_room > 0: the profile is in shared memory -- the kernel builds for a profile in global memory carry the classic form only)
    pl.narrow_staged = in.narrow_room > 0 && max_rows / kRowsPerChunk >= 32ull * pl.n_tiles_narrow;
    if (!pl.narrow_staged && pl.narrow_tile != kNarrowTile) {
        pl.narrow_tile = kNarrowTile;
        pl.n_tiles_narrow = (in.query_len + pl.narrow_tile - 1) / pl.narrow_tile;
        pl.narrow_staged = in.narrow_room > 0 && max_rows / kRowsPerChunk >= 32ull * pl.n_tiles_narrow;
    }
    const bool can_pipe = in.s16 && in.pipe_rings >= 2 && n_groups > 0;
    if (can_pipe && in.policy == kScanPipeline) {
        pl.pipe_first = 0;
        pl.wave_sms = 0;
        pl.wave_rows = 0;
    } else if (can_pipe && in.policy == kScanAuto && k.pipe && (n_tiles >= k.pipe_min_tiles || pl.chain_bound) &&
               n_groups >= 2 * in.sm_count) {
        const uint64_t fair_cta = in.padded_rows / in.sm_count;   // rows per CTA
        // (a smaller shard has fewer groups per CTA to balance with, but its wavefront share grows with every group that is
        // called tall: 0.6 of a CTA's share below 32 groups per SM -- 1/8 Swiss-Prot, m = 3564: 18.1 -> 16.9 ms)
        const double tall_fraction = n_groups < 32 * in.sm_count ? k.pipe_tall_small : k.pipe_tall;
        const uint64_t tall = std::max<uint64_t>(256, static_cast<uint64_t>(tall_fraction * static_cast<double>(fair_cta)));
        uint32_t g = 0;
        uint64_t rows_wave = 0;
        while (g < n_groups && rows_of(g) > tall) rows_wave += rows_of(g++);
        pl.pipe_first = g;
        pl.wave_rows = rows_wave;
        if (g == 0) {
            pl.wave_sms = 0;
        } else {
            const double share = static_cast<double>(rows_wave) / static_cast<double>(in.padded_rows);
            // chain-bound searches give the wavefront kernel twice its share; searches close to it (the tallest group's rows
            // above 1.0 x a warp's fair share: long queries on a 1/8 shard) 1.6 x -- m = 5478 on 1/8 Swiss-Prot 29.7 -> 27.4 ms
            // (long queries only: at 23 tiles, m = 729 on the whole database, the same ratio loses 2 % with the larger share)
            const double near_chain = static_cast<double>(max_rows) > 1.0 * fair_all && n_tiles >= 64 ? k.wave_margin_near : k.wave_margin;
            const double margin = pl.chain_bound ? k.wave_margin_chain : near_chain;
            pl.wave_sms = static_cast<uint32_t>(std::ceil(share * margin * in.sm_count));
            pl.wave_sms = std::max<uint32_t>(1, std::min<uint32_t>(pl.wave_sms, in.sm_count - 1));
        }
    }

    // ---- 2. units of the wavefront kernel's groups [0, pipe_first) ---------------------------------------------
    const uint32_t n_wave = pl.pipe_first;
    const uint64_t total_row_tiles = pl.wave_rows * n_tiles;
    pl.wave_threads = in.warps_per_cta * 32;
    if (k.wave_threads) {
        pl.wave_threads = k.wave_threads;   // tuning override
    } else if (pl.pipe_first < n_groups && pl.pipe_first > 0) {
        const double chain = static_cast<double>(max_rows) / std::max(fair_all, 1.0);
        if (chain >= 1.5 * k.wave_thin) pl.wave_threads = std::min<uint32_t>(pl.wave_threads, 128);
        else if (chain >= k.wave_thin) pl.wave_threads = std::min<uint32_t>(pl.wave_threads, 256);
    }
    const uint64_t warps = static_cast<uint64_t>(std::max<uint32_t>(pl.wave_sms, 1)) * (pl.wave_threads / 32);
    const uint64_t fair = total_row_tiles / warps;
    // With plenty of groups per warp (a whole Swiss-Prot on one GPU: 3.7) only units larger than about three
    // quarters of a warp's fair share need cutting -- LPT order fills the rest; a small shard with fewer groups
    // than warps has to be cut finer to give every warp several units.
    const double auto_fraction = std::min(0.75, std::max(0.08, static_cast<double>(n_wave) / (4.0 * static_cast<double>(warps))));
    const double fraction = k.unit_budget > 0.0 ? k.unit_budget : auto_fraction;
    const uint64_t budget = std::max<uint64_t>(2048, static_cast<uint64_t>(fraction * static_cast<double>(fair)));
    const uint64_t narrow_rows = std::max<uint64_t>(2048, static_cast<uint64_t>(k.narrow_chain * static_cast<double>(fair)));
    // Groups are sorted longest first: narrow tiles are needed iff the first group needs them.  The kernel variant
    // that carries both extra paths spills registers in the common 32-column sweep (about 12 % slower), so a search
    // that needs narrow tiles cuts its other large groups by rows only if cutting them by tile instead would waste
    // more than that (small shards, long queries).
    const bool narrow_ok = in.s16 && pl.n_tiles_narrow > 1;
    const bool narrow_needed = narrow_ok && n_wave && rows_of(0) > narrow_rows;
    bool row_blocks_ok = in.s16 && k.row_blocks;
    auto split_shape = [&](uint32_t g, double* eff_tiles, double* eff_rows) {   // -> row blocks of >= 2 chunks, ~budget row-tiles each
        const uint64_t chunks = in.groups[g].n_chunks, rows = rows_of(g), work = rows * n_tiles;
        *eff_tiles = static_cast<double>(rows) / static_cast<double>(rows + 16 * (n_tiles - 1));
        const uint64_t blocks = std::min<uint64_t>((work + budget - 1) / budget, std::max<uint64_t>(chunks / 2, 1));
        *eff_rows = static_cast<double>(n_tiles) / static_cast<double>(n_tiles + blocks - 1);
        return blocks;
    };
    if (row_blocks_ok && narrow_needed) {
        double wasted = 0.0;   // extra warp time of tile-splitting where row blocks would have been chosen
        for (uint32_t g = 0; g < n_wave; ++g) {
            const uint64_t rows = rows_of(g), work = rows * n_tiles;
            if (work <= budget || n_tiles < 2 || rows > narrow_rows) continue;
            double eff_tiles, eff_rows;
            const uint64_t blocks = split_shape(g, &eff_tiles, &eff_rows);
            if (blocks >= 2 && eff_rows > eff_tiles) wasted += static_cast<double>(work) * (1.0 / eff_tiles - 1.0 / eff_rows);
        }
        row_blocks_ok = wasted > 0.12 * static_cast<double>(total_row_tiles);
    }
    for (uint32_t g = n_wave; g < n_groups; ++g) unit_start[g] = 0, vstate_off[g] = 0, modes[g] = kGroupSingle;
    for (uint32_t g = 0; g < n_wave; ++g) {
        unit_start[g] = pl.n_units;
        vstate_off[g] = 0;
        const uint64_t rows = rows_of(g), work = rows * n_tiles;
        uint8_t mode = kGroupSingle;
        uint32_t units = 1;
        bool took_vstate = false;
        if (work > budget && n_tiles > 1) {
            mode = kGroupSplit;
            units = n_tiles;
            double eff_tiles, eff_rows;
            const uint64_t blocks = split_shape(g, &eff_tiles, &eff_rows);
            if (row_blocks_ok && blocks >= 2 && eff_rows > eff_tiles) {
                mode = kGroupRowBlock;
                units = static_cast<uint32_t>(blocks);
                vstate_off[g] = static_cast<uint32_t>(pl.vstate_slots);
                pl.vstate_slots += n_tiles;
                took_vstate = true;
            }
        }
        const uint64_t links = pl.narrow_staged ? rows * (pl.n_tiles_narrow - 1) : 0;   // a link buffer per tile boundary
        if (narrow_ok && rows > narrow_rows && pl.link_rows + links <= k.narrow_link_rows &&
            pl.link_rows + links < (1ull << 32)) {
            if (took_vstate) pl.vstate_slots -= n_tiles;
            mode = kGroupNarrow;
            units = pl.n_tiles_narrow;
            vstate_off[g] = static_cast<uint32_t>(pl.link_rows);
            pl.link_rows += links;
        }
        modes[g] = mode;
        pl.n_split += mode == kGroupSplit;
        pl.n_narrow += mode == kGroupNarrow;
        pl.n_rowblock += mode == kGroupRowBlock;
        pl.n_units += units;
    }
    pl.any_narrow = pl.n_narrow > 0;
    pl.any_rowblock = pl.n_rowblock > 0;
    if (pl.any_narrow && pl.narrow_staged && pl.pipe_first < n_groups && pl.narrow_tile == kNarrowTileFine) {
        // The most chain-bound searches (those that take 4-column tiles): narrow units are bound by their own chain and run
        // it fastest alone on a scheduler (tools/lat_probe.cu: 760 clk per 8 x 8 block with one warp per scheduler, 1,336
        // with two): 4 warps per CTA, and SMs for the first round of units.  Where the chain is a smaller part of the
        // search (a whole Swiss-Prot on one GPU, m = 144: 5 x a warp's fair share) the SMs are worth more to the pipeline.
        pl.wave_threads = 128;   // = kNarrowThreads (kernels.cuh)
        // ... and, where their rings fit next to the profile, a helper warp per unit on the same scheduler that carries its
        // blocks between global and shared memory (4 + 4 warps per CTA): the unit itself then never waits for L2
        if (k.narrow_helpers && in.narrow_room >= 4 * kNarrowPairBytesHost) {
            pl.narrow_helpers = true;
            pl.wave_threads = 256;
        }
        const uint32_t want = (pl.n_units + 3) / 4;
        const uint32_t cap = std::max<uint32_t>(pl.wave_sms, static_cast<uint32_t>(k.narrow_sms * in.sm_count));
        pl.wave_sms = std::max(pl.wave_sms, std::min(want, cap));
        pl.wave_sms = std::max<uint32_t>(1, std::min<uint32_t>(pl.wave_sms, in.sm_count - 1));
    }
    // The thinnest CTA shape (4 warps) serves the chains only while (nearly) every unit of the wavefronts has a warp: units that
    // wait for a ticket stall the tiles behind them (1/8 Swiss-Prot, m = 1000: 346 units on 43 x 4 warps 6.8 ms, on 43 x 8 warps
    // 5.4 ms); beyond 8 warps per CTA the chains themselves slow down more than that
    if (pl.any_narrow && !pl.narrow_helpers && !k.wave_threads)
        while (pl.wave_threads < 256 && 20ull * pl.wave_sms * (pl.wave_threads / 32) < 19ull * pl.n_units) pl.wave_threads *= 2;
    unit_start[n_wave] = pl.n_units;
    for (uint32_t g = n_wave + 1; g <= n_groups; ++g) unit_start[g] = pl.n_units;
    return pl;
}

// ---- batches of queries (swb_search_many) -------------------------------------------------------------------------

// One shared scan: the two streams of queries (numbers into the caller's arrays), each in the order they are laid out.
struct DuoScan {
    std::vector<uint32_t> a, b;
    uint32_t tiles_a = 0, tiles_b = 0;
};

inline uint32_t tiles_of(uint32_t m) { return (m + 31) / 32; }

// How shared scans hand out their work.  Whole items (a half-group with all its tiles on one CTA) are the faster form,
// but the tallest half-group must fit a CTA's fair share of the scan; small shards of a database with a few very long
// sequences do not satisfy that (one 35,213-row item would outlast the scan several times), and take pass items:
// one pass of 16 tiles per item, pass-major over the whole shard, so that a tall half-group's passes run on many CTAs
// one behind the other (3 % slower per cell, but 48 instead of 35 TCUPS-equivalent on eight 1/8 shards of Swiss-Prot).
enum SharedScanMode : int { kSharedNone = 0, kSharedWhole = 1, kSharedPass = 2 };

inline SharedScanMode shared_scan_mode(const ScanKnobs& k, uint32_t n_groups, uint32_t max_rows, uint64_t padded_rows, uint32_t sm_count) {
    if (k.duo_ratio > 1.0) return kSharedNone;
    if (static_cast<double>(n_groups) < k.duo_min_groups_per_sm * static_cast<double>(sm_count)) return kSharedNone;
    const bool whole_fits = static_cast<double>(max_rows) * sm_count <= k.duo_tall * 2.0 * static_cast<double>(padded_rows);
    if (k.duo_pass_items >= 2) return kSharedPass;
    if (whole_fits) return kSharedWhole;
    return k.duo_pass_items >= 1 ? kSharedPass : kSharedNone;
}

// Deals the queries of a batch over shared scans: longest first, each to the shortest stream so far, so that the two
// streams of a scan end up equally long.  A scan whose streams differ too much (the padding would eat the two-stream
// kernel's ~15 % advantage) or that is too short to keep the pipeline busy is dissolved again: its queries go one by
// one.  `single` receives every query that is not part of a scan (empty queries, and all of them when !enabled).
inline void plan_batch(const ScanKnobs& k, SharedScanMode mode, const uint32_t* lens, uint32_t n_queries, std::vector<DuoScan>& scans,
                       std::vector<uint32_t>& single) {
    const bool enabled = mode != kSharedNone;
    // pass items need more than one pass; whole items the pipeline's usual minimum
    const uint32_t min_tiles = mode == kSharedPass ? 17u : k.pipe_min_tiles;
    scans.clear();
    single.clear();
    std::vector<uint32_t> eligible;
    for (uint32_t q = 0; q < n_queries; ++q) (enabled && lens[q] > 0 ? eligible : single).push_back(q);
    if (eligible.size() < 2) {
        single.insert(single.end(), eligible.begin(), eligible.end());
        std::sort(single.begin(), single.end());
        return;
    }
    std::stable_sort(eligible.begin(), eligible.end(), [&](uint32_t x, uint32_t y) { return lens[x] > lens[y]; });
    uint64_t total_tiles = 0;
    for (uint32_t q : eligible) total_tiles += tiles_of(lens[q]);
    const uint32_t n_scans = static_cast<uint32_t>((total_tiles + 2ull * k.duo_stream_tiles - 1) / (2ull * k.duo_stream_tiles));
    scans.resize(n_scans);
    for (uint32_t q : eligible) {
        DuoScan* best = nullptr;
        bool high = false;
        uint32_t least = ~0u;
        for (DuoScan& sc : scans) {
            if (sc.tiles_a < least) least = sc.tiles_a, best = &sc, high = false;
            if (sc.tiles_b < least) least = sc.tiles_b, best = &sc, high = true;
        }
        (high ? best->b : best->a).push_back(q);
        (high ? best->tiles_b : best->tiles_a) += tiles_of(lens[q]);
    }
    // then split each scan's queries as evenly as possible: subset sum over their tile counts (a few hundred
    // tiles per scan at most, so the table is tiny)
    for (DuoScan& sc : scans) {
        std::vector<uint32_t> members(sc.a);
        members.insert(members.end(), sc.b.begin(), sc.b.end());
        std::stable_sort(members.begin(), members.end(), [&](uint32_t x, uint32_t y) { return lens[x] > lens[y]; });
        const uint32_t total = sc.tiles_a + sc.tiles_b;
        // ok[s]: some subset of the members seen so far has s tiles; reach[s]: the member that first made it so (sums
        // are walked downwards, so ok[s - t] still refers to the members before the current one)
        std::vector<uint32_t> reach(total / 2 + 1, 0);
        std::vector<uint8_t> ok(total / 2 + 1, 0);
        ok[0] = 1;
        for (size_t i = 0; i < members.size(); ++i) {
            const uint32_t t = tiles_of(lens[members[i]]);
            for (uint32_t sum = total / 2; sum >= t; --sum)
                if (!ok[sum] && ok[sum - t]) {
                    ok[sum] = 1;
                    reach[sum] = static_cast<uint32_t>(i);
                }
        }
        uint32_t best = total / 2;
        while (best > 0 && !ok[best]) --best;
        std::vector<uint8_t> in_a(members.size(), 0);
        for (uint32_t sum = best; sum > 0;) {
            const uint32_t i = reach[sum];
            in_a[i] = 1;
            sum -= tiles_of(lens[members[i]]);
        }
        sc.a.clear(), sc.b.clear();
        sc.tiles_a = sc.tiles_b = 0;
        for (size_t i = 0; i < members.size(); ++i) {
            (in_a[i] ? sc.a : sc.b).push_back(members[i]);
            (in_a[i] ? sc.tiles_a : sc.tiles_b) += tiles_of(lens[members[i]]);
        }
    }
    std::vector<DuoScan> kept;
    for (DuoScan& sc : scans) {
        const uint32_t lo = std::min(sc.tiles_a, sc.tiles_b), hi = std::max(sc.tiles_a, sc.tiles_b);
        if (lo == 0 || static_cast<double>(lo) < k.duo_ratio * static_cast<double>(hi) || hi < min_tiles) {
            single.insert(single.end(), sc.a.begin(), sc.a.end());
            single.insert(single.end(), sc.b.begin(), sc.b.end());
        } else {
            kept.push_back(std::move(sc));
        }
    }
    scans.swap(kept);
    std::sort(single.begin(), single.end());
}

// Capacity of each border ring (chunks, a power of two) that fits next to a profile of `prof_bytes` in
// `smem_optin` bytes of shared memory; < 2: the pipeline cannot run.  fixed_bytes: the pipeline's control block.
inline uint32_t ring_chunks_for(size_t prof_bytes, size_t smem_optin, size_t fixed_bytes, size_t ring_chunk_bytes_all_warps,
                                uint32_t cap) {
    const size_t fixed = ((prof_bytes + 255) & ~size_t(255)) + fixed_bytes;
    if (fixed >= smem_optin) return 0;
    const size_t room = (smem_optin - fixed) / ring_chunk_bytes_all_warps;
    if (room < 1) return 0;
    uint32_t c = 1;
    while (c * 2 <= room && c * 2 <= cap) c *= 2;
    return c;
}

// The pipeline kernel keeps the query's whole int8 profile in shared memory while at least two chunks per ring fit next to
// it (m up to ~6,500); beyond that each warp keeps only the slice of its current tile (25 rows x 32 B, kPipeSliceStride apart,
// reloaded at every slot start), the rings get their full capacity and shared memory no longer depends on m.
// SWB200_PIPE_SLICES=1 takes the slice form for every query (measurement).
constexpr uint32_t kPipeSliceStride = 48;     // bytes between the rows of a warp's slice: 16-byte groups 3 apart modulo 8
constexpr uint32_t kPipeSliceBytes = 1280;    // 25 rows x 48 B, rounded up to 256
constexpr uint32_t kPipeWarpsHost = 16;
struct PipeRings {
    uint32_t chunks = 0;      // capacity of each ring; < 2: the pipeline cannot run
    bool slices = false;      // per-warp tile slices instead of the whole profile
    size_t prof_bytes = 0;    // shared memory in front of the control block
};
inline PipeRings pipe_rings_for(size_t prof_bytes, size_t smem_optin, size_t fixed_bytes, size_t ring_chunk_bytes_all_warps,
                                uint32_t cap) {
    static const bool force = [] {
        const char* e = std::getenv("SWB200_PIPE_SLICES");
        return e != nullptr && *e == '1';
    }();
    PipeRings r;
    r.prof_bytes = (prof_bytes + 255) & ~size_t(255);
    r.chunks = ring_chunks_for(prof_bytes, smem_optin, fixed_bytes, ring_chunk_bytes_all_warps, cap);
    if (r.chunks < 2 || force) {
        r.slices = true;
        r.prof_bytes = static_cast<size_t>(kPipeWarpsHost) * kPipeSliceBytes;
        r.chunks = ring_chunks_for(r.prof_bytes, smem_optin, fixed_bytes, ring_chunk_bytes_all_warps, cap);
    }
    return r;
}

// Row stride of the int8 profile: columns padded to whole 32-column tiles, then to 16 (mod 128) bytes so that the
// 25 rows spread over the shared-memory banks.
inline uint32_t profile_stride(uint32_t m, uint32_t tile) {
    const uint32_t mpad = std::max<uint32_t>(tile, (m + tile - 1) / tile * tile);
    return mpad + ((16 + 128 - (mpad % 128)) % 128);
}

}  // namespace swb
