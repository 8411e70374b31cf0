// cabi.cu -- the C-ABI of include/swb200.h: handles, orchestration, launches.
//
// Host flow of one search (replaces scheduler.hpp:188-244):
//   validate -> upload query + matrix + unit table -> build_profile_kernel -> packed-int16
//   tile-wavefront kernel over all groups -> collect + int32 re-run of lanes above the trust limit
//   -> key build -> top-k select -> download k hits.
// Everything runs on one stream per handle; no host synchronisation happens between the upload and
// the final download.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/swb200.h"
#include "kernels.cuh"
#include "pack.hpp"
#include "pipe_rates.cuh"

using namespace swb;

namespace {

thread_local std::string g_error;

swb_status fail(swb_status st, const std::string& msg) {
    g_error = msg;
    return st;
}

#define SWB_CUDA(expr)                                                                           \
    do {                                                                                         \
        cudaError_t e__ = (expr);                                                                \
        if (e__ != cudaSuccess)                                                                  \
            return fail(SWB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__));      \
    } while (0)

template <class T>
swb_status dev_alloc(T** ptr, size_t count, uint64_t* tally) {
    *ptr = nullptr;
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    SWB_CUDA(cudaMalloc(reinterpret_cast<void**>(ptr), bytes));
    if (tally) *tally += bytes;
    return SWB_OK;
}

inline uint32_t pack16(int32_t v) {
    const uint32_t h = static_cast<uint32_t>(v) & 0xffffu;
    return h | (h << 16);
}

enum { EV_START = 0, EV_UP, EV_SCAN, EV_RESCORE, EV_TOPK, EV_END, EV_COUNT };

enum MainKernel { kMainNone = 0, kMainS16 = 1 };

struct QueryPlan {
    int main = kMainNone;     // which packed kernel scans the database (none: int32 intra kernel for everything)
    bool wide = false;        // the int32 intra kernel needs the int32 profile (matrix + open outside int8)
    bool may_overflow = true; // a score above `limit` is possible at all
    int32_t limit = 0;
    int32_t open = 0, ext = 0;
    uint32_t m = 0;
    uint32_t tile = kInterTile; // query columns per register tile of the packed kernel
    uint32_t threads = kInterThreads;
    uint32_t pstride = 0;       // inter profile row stride
    uint32_t intra_t = 8, n_lane_tiles = 0, intra_w = 1, intra_passes = 0;
};

}  // namespace

struct swb_db {
    int device = 0;
    cudaStream_t own_stream = nullptr, stream = nullptr;
    int sm_count = 0;
    size_t smem_optin = 0;
    std::mutex mu;
    uint64_t device_bytes = 0;
    bool force_intra = false;   // swb_score_pair: score with the intra-task kernel only

    // database (metadata stays on the host, bulk arrays live on the device only)
    PackedDb meta;
    uint32_t n_slots = 0;
    uint32_t max_rows = 0;      // padded rows of the longest group
    uint8_t* d_codes = nullptr;
    GroupDesc* d_groups = nullptr;
    uint32_t* d_slot_index = nullptr;
    uint32_t* d_slot_len = nullptr;

    // work buffers
    uint2 *d_border0 = nullptr, *d_border1 = nullptr;      // wavefront kernel, database-shaped
    uint2 *d_iborder0 = nullptr, *d_iborder1 = nullptr;    // intra kernel, [ctas][max_rows]
    uint32_t intra_ctas = 0;
    int32_t* d_slot_scores = nullptr;
    uint32_t* d_flag_list = nullptr;
    uint32_t* d_counters = nullptr;   // [0] ticket, [1] flag count
    uint32_t* d_unit_start = nullptr;
    uint8_t* d_group_mode = nullptr;
    uint32_t* d_vstate_off = nullptr;
    uint4* d_vstate = nullptr;
    size_t vstate_cap = 0;
    uint32_t* d_progress = nullptr;
    size_t progress_cap = 0;
    uint64_t* d_keys = nullptr;
    uint64_t* d_sel[2] = {nullptr, nullptr};
    size_t sel_cap = 0;
    uint64_t* d_sort = nullptr;
    size_t sort_cap = 0;
    int32_t* d_all_scores = nullptr;

    // query side
    uint32_t query_cap = 0;
    uint8_t* d_query = nullptr;
    int32_t* d_matrix = nullptr;
    int8_t *d_prof8 = nullptr, *d_prof8i = nullptr;
    int32_t* d_prof32i = nullptr;
    size_t prof8_cap = 0, prof8i_cap = 0, prof32i_cap = 0;

    uint8_t* h_stage = nullptr;   // pinned: matrix + query + unit table up, keys down
    size_t stage_cap = 0;
    uint32_t* h_counters = nullptr;   // pinned copy of d_counters
    cudaEvent_t ev[EV_COUNT] = {};
    uint32_t launches = 0;
    uint32_t last_units = 0;
    uint32_t last_tile = kInterTile;
    std::vector<uint32_t> slot_of;   // db_index -> slot (built on the first traceback request)
    bool smem_attr_set = false;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

swb_status ensure_stage(swb_db* db, size_t bytes) {
    if (bytes <= db->stage_cap) return SWB_OK;
    if (db->h_stage) cudaFreeHost(db->h_stage);
    db->h_stage = nullptr;
    db->stage_cap = 0;
    const size_t cap = std::max<size_t>(bytes * 2, 1 << 16);
    SWB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&db->h_stage), cap));
    db->stage_cap = cap;
    return SWB_OK;
}

template <class T>
swb_status ensure_dev(T** ptr, size_t* cap, size_t need, uint64_t* tally) {
    if (need <= *cap) return SWB_OK;
    if (*ptr) {
        cudaFree(*ptr);
        *tally -= *cap * sizeof(T);
    }
    *ptr = nullptr;
    *cap = 0;
    const size_t want = need + need / 4 + 256;
    swb_status st = dev_alloc(ptr, want, tally);
    if (st != SWB_OK) return st;
    *cap = want;
    return SWB_OK;
}

swb_status check_scoring_args(const uint8_t* query, uint32_t m, const int32_t* matrix, int32_t open,
                              int32_t ext) {
    if (!matrix) return fail(SWB_ERR_INVALID, "matrix is null");
    if (m && !query) return fail(SWB_ERR_INVALID, "query is null");
    // GapModel's invariant and message (scoring.hpp:50-53)
    if (ext < 0 || open < ext) return fail(SWB_ERR_INVALID, "gap model requires open >= extend >= 0");
    // QueryProfile's check and message (scoring.hpp:203-205)
    for (uint32_t j = 0; j < m; ++j)
        if (query[j] >= kAlphabet) return fail(SWB_ERR_RANGE, "query code outside matrix alphabet");
    int32_t lo = matrix[0], hi = matrix[0];
    for (int i = 1; i < 576; ++i) lo = std::min(lo, matrix[i]), hi = std::max(hi, matrix[i]);
    if (lo < -(1 << 20) || hi > (1 << 20) || open > (1 << 28))
        return fail(SWB_ERR_UNSUPPORTED, "matrix entries beyond +-2^20 or gap open beyond 2^28");
    return SWB_OK;
}

// Fraction of a warp's fair share of the search above which a group is split into a wavefront.
double unit_budget_fraction() {
    static const double f = [] {
        const char* e = std::getenv("SWB200_UNIT_BUDGET");
        const double v = e ? std::atof(e) : 0.0;
        return v > 0.0 ? v : 0.0;   // 0: automatic (see score_core)
    }();
    return f;
}

bool row_blocks_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SWB200_ROWBLOCKS");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

// A group goes to 8-column tiles when its rows exceed this fraction of a warp's fair share (in row-tiles).
double narrow_chain_fraction() {
    static const double f = [] {
        const char* e = std::getenv("SWB200_NARROW");
        const double v = e ? std::atof(e) : 0.0;
        return v > 0.0 ? v : 0.9;
    }();
    return f;
}

QueryPlan make_plan(const swb_db* db, uint32_t m, const int32_t* matrix, int32_t open, int32_t ext) {
    QueryPlan pl;
    pl.m = m;
    pl.open = open;
    pl.ext = ext;
    int32_t lo = matrix[0], hi = matrix[0];
    for (int i = 1; i < 576; ++i) lo = std::min(lo, matrix[i]), hi = std::max(hi, matrix[i]);
    const int32_t top = std::max(hi, 0);
    // int8 profile shifted by `open` (s16 kernel and the int8 flavour of the intra kernel)
    const bool fits8 = (lo + open >= -128) && (hi + open <= 127) && (open <= 127);
    pl.wide = !fits8;
    static const bool force_intra_env = [] {
        const char* e = std::getenv("SWB200_KERNEL");
        return e && std::string(e) == "intra";
    }();
    pl.main = (fits8 && !db->force_intra && !force_intra_env) ? kMainS16 : kMainNone;
    pl.limit = 32767 - top;
    const uint64_t reach = static_cast<uint64_t>(top) * std::min<uint64_t>(m, db->meta.max_length);
    pl.may_overflow = reach > static_cast<uint64_t>(pl.limit);

    pl.tile = kInterTile;
    pl.threads = kInterThreads;
    // wavefront profile stride: columns padded to whole tiles, then to 16 (mod 128) bytes
    const uint32_t mpad = std::max<uint32_t>(pl.tile, (m + pl.tile - 1) / pl.tile * pl.tile);
    pl.pstride = mpad + ((16 + 128 - (mpad % 128)) % 128);

    // intra-task geometry: T columns per lane (4..8), W warps per CTA, passes
    uint64_t best_cols = ~0ull;
    for (uint32_t t = 4; t <= 8; ++t) {
        const uint32_t tiles = (std::max<uint32_t>(m, 1) + t - 1) / t;
        const uint32_t w = std::min<uint32_t>(kIntraMaxWarps, (tiles + 31) / 32);
        const uint32_t passes = (tiles + 32 * w - 1) / (32 * w);
        const uint64_t cols = static_cast<uint64_t>(passes) * w * 32 * t;
        if (cols <= best_cols) {
            best_cols = cols;
            pl.intra_t = t;
            pl.n_lane_tiles = tiles;
            pl.intra_w = w;
            pl.intra_passes = passes;
        }
    }
    return pl;
}

template <int T, typename PT>
void launch_intra(const IntraParams& ip, uint32_t ctas, uint32_t warps, cudaStream_t s) {
    intra_s32_kernel<T, PT><<<ctas, warps * 32, 0, s>>>(ip);
}

template <typename PT>
void launch_intra_t(uint32_t t, const IntraParams& ip, uint32_t ctas, uint32_t warps, cudaStream_t s) {
    switch (t) {
        case 4: launch_intra<4, PT>(ip, ctas, warps, s); break;
        case 5: launch_intra<5, PT>(ip, ctas, warps, s); break;
        case 6: launch_intra<6, PT>(ip, ctas, warps, s); break;
        case 7: launch_intra<7, PT>(ip, ctas, warps, s); break;
        default: launch_intra<8, PT>(ip, ctas, warps, s); break;
    }
}

// Launch the int32 intra-task kernel over `list` (nullptr = every slot).
swb_status run_intra(swb_db* db, const QueryPlan& pl, const uint32_t* list, cudaStream_t s) {
    swb_status st;
    if (!db->intra_ctas) {
        // per-CTA border rows are only touched when the query needs more than one pass, but the
        // allocation is sized once for the worst case
        const uint64_t rows = std::max<uint32_t>(db->max_rows, 1);
        uint64_t ctas = (512ull << 20) / (rows * 16);
        ctas = std::min<uint64_t>(static_cast<uint64_t>(db->sm_count) * 8, std::max<uint64_t>(8, ctas));
        ctas = std::min<uint64_t>(ctas, std::max<uint32_t>(db->n_slots, 1));
        if ((st = dev_alloc(&db->d_iborder0, rows * ctas, &db->device_bytes)) != SWB_OK) return st;
        if ((st = dev_alloc(&db->d_iborder1, rows * ctas, &db->device_bytes)) != SWB_OK) return st;
        db->intra_ctas = static_cast<uint32_t>(ctas);
    }
    IntraParams ip{};
    ip.codes = db->d_codes;
    ip.groups = db->d_groups;
    ip.slot_len = db->d_slot_len;
    ip.list = list;
    ip.list_count = db->d_counters + 1;
    ip.n_slots = db->n_slots;
    ip.profi = pl.wide ? static_cast<const void*>(db->d_prof32i) : static_cast<const void*>(db->d_prof8i);
    ip.n_lane_tiles = pl.n_lane_tiles;
    ip.n_passes = pl.intra_passes;
    ip.border0 = db->d_iborder0;
    ip.border1 = db->d_iborder1;
    ip.border_rows = std::max<uint32_t>(db->max_rows, 1);
    ip.slot_scores = db->d_slot_scores;
    ip.open = pl.open;
    ip.ext = pl.ext;
    if (pl.wide) launch_intra_t<int32_t>(pl.intra_t, ip, db->intra_ctas, pl.intra_w, s);
    else launch_intra_t<int8_t>(pl.intra_t, ip, db->intra_ctas, pl.intra_w, s);
    ++db->launches;
    return SWB_OK;
}

// Scores every local sequence; results land in d_slot_scores.  Asynchronous on db->stream.
swb_status score_core(swb_db* db, const uint8_t* query, uint32_t m, const int32_t* matrix, int32_t open,
                      int32_t ext) {
    cudaStream_t s = db->stream;
    const QueryPlan pl = make_plan(db, m, matrix, open, ext);
    db->launches = 0;
    db->last_units = 0;
    db->last_tile = pl.tile;
    SWB_CUDA(cudaEventRecord(db->ev[EV_START], s));
    SWB_CUDA(cudaMemsetAsync(db->d_slot_scores, 0, std::max<size_t>(db->n_slots, 1) * sizeof(int32_t), s));
    SWB_CUDA(cudaMemsetAsync(db->d_counters, 0, 4 * sizeof(uint32_t), s));

    if (m == 0 || db->meta.n_local == 0) {
        // empty query: every score is 0 (align.hpp:45,100,172)
        for (int e = EV_UP; e <= EV_RESCORE; ++e) SWB_CUDA(cudaEventRecord(db->ev[e], s));
        return SWB_OK;
    }

    const uint32_t n_groups = static_cast<uint32_t>(db->meta.groups.size());
    const bool packed = pl.main != kMainNone;

    // ---- stage matrix + query (+ the unit table of the wavefront kernel) and upload -----------------
    const size_t off_query = 576 * sizeof(int32_t);
    const size_t off_units = (off_query + m + 15) & ~size_t(15);
    const size_t off_vsoff = off_units + (static_cast<size_t>(n_groups) + 1) * sizeof(uint32_t);
    const size_t off_modes = off_vsoff + static_cast<size_t>(n_groups) * sizeof(uint32_t);
    const size_t stage_bytes = off_modes + n_groups;
    swb_status st = ensure_stage(db, stage_bytes);
    if (st != SWB_OK) return st;
    if (m > db->query_cap) {
        if (db->d_query) cudaFree(db->d_query);
        db->d_query = nullptr;
        st = dev_alloc(&db->d_query, static_cast<size_t>(m) * 2, &db->device_bytes);
        if (st != SWB_OK) return st;
        db->query_cap = m * 2;
    }
    std::memcpy(db->h_stage, matrix, off_query);
    std::memcpy(db->h_stage + off_query, query, m);
    const uint32_t n_tiles = (m + pl.tile - 1) / pl.tile;
    const uint32_t n_tiles_narrow = (m + kNarrowTile - 1) / kNarrowTile;
    uint32_t n_units = 0;
    bool any_narrow = false, any_rowblock = false;
    uint64_t vstate_slots = 0;
    if (packed) {
        // Unit policy (see kernels.cuh, GroupMode).  Work is counted in row-tiles (one row of one T-column tile);
        // `fair` is one warp's share of the whole search.
        //   single    the default: one warp scores the group's 64 sequences end to end;
        //   split     a group whose sweep exceeds `budget` is cut so that no unit dominates the makespan and there
        //             are enough units for every warp, either
        //               by tile   (wavefront of warps, each 2 chunks behind its left neighbour:
        //                          efficiency rows / (rows + 16 (tiles - 1))), or
        //               by rows   (blocks of rows, each one tile behind the block above:
        //                          efficiency tiles / (tiles + blocks - 1)),
        //             whichever wastes less;
        //   narrow    even a tile-split group's per-tile chain (rows x T columns, strictly sequential in one thread,
        //             ~900 clk per row when the SM empties out, against ~1600 clk per row-tile of saturated
        //             throughput) would take more than about half the whole search: 8-column tiles cut that chain
        //             four-fold.
        // Row blocks and narrow tiles exist in the s16 kernel only.
        uint32_t* us = reinterpret_cast<uint32_t*>(db->h_stage + off_units);
        uint32_t* vso = reinterpret_cast<uint32_t*>(db->h_stage + off_vsoff);
        uint8_t* modes = db->h_stage + off_modes;
        const uint64_t total_row_tiles = db->meta.padded_rows * n_tiles;
        const uint64_t warps = static_cast<uint64_t>(db->sm_count) * (pl.threads / 32);
        const uint64_t fair = total_row_tiles / warps;
        // With plenty of groups per warp (a whole Swiss-Prot on one GPU: 3.7) only units larger than about
        // three quarters of a warp's fair share need cutting -- LPT order fills the rest; a small shard with fewer
        // groups than warps has to be cut finer to give every warp several units.
        const double auto_fraction = std::min(0.75, std::max(0.08, static_cast<double>(n_groups) / (4.0 * static_cast<double>(warps))));
        const double fraction = unit_budget_fraction() > 0.0 ? unit_budget_fraction() : auto_fraction;
        const uint64_t budget = std::max<uint64_t>(2048, static_cast<uint64_t>(fraction * static_cast<double>(fair)));
        const uint64_t narrow_rows = std::max<uint64_t>(2048, static_cast<uint64_t>(narrow_chain_fraction() * fair));
        const bool s16 = pl.main == kMainS16;
        // groups are sorted longest first: narrow tiles are needed iff the first group needs them.  The kernel
        // variant that carries both extra paths spills registers in the common 32-column sweep, so a search that
        // needs narrow tiles cuts its other large groups by tile rather than by rows.
        const bool narrow_needed = s16 && n_groups && n_tiles_narrow > 1 &&
                                   static_cast<uint64_t>(db->meta.groups[0].n_chunks) * kRowsPerChunk > narrow_rows;
        const bool row_blocks_ok = s16 && row_blocks_enabled() && !narrow_needed;
        for (uint32_t g = 0; g < n_groups; ++g) {
            us[g] = n_units;
            vso[g] = 0;
            const uint64_t chunks = db->meta.groups[g].n_chunks;
            const uint64_t rows = chunks * kRowsPerChunk;
            const uint64_t work = rows * n_tiles;
            uint8_t mode = kGroupSingle;
            uint32_t units = 1;
            if (work > budget && n_tiles > 1) {
                mode = kGroupSplit;
                units = n_tiles;
                const double eff_tiles = static_cast<double>(rows) / static_cast<double>(rows + 16 * (n_tiles - 1));
                // row blocks of at least 2 chunks, about `budget` row-tiles each
                const uint64_t blocks = std::min<uint64_t>((work + budget - 1) / budget, std::max<uint64_t>(chunks / 2, 1));
                const double eff_rows = static_cast<double>(n_tiles) / static_cast<double>(n_tiles + blocks - 1);
                if (row_blocks_ok && blocks >= 2 && eff_rows > eff_tiles) {
                    mode = kGroupRowBlock;
                    units = static_cast<uint32_t>(blocks);
                    vso[g] = static_cast<uint32_t>(vstate_slots);
                    vstate_slots += n_tiles;
                    any_rowblock = true;
                }
            }
            if (s16 && rows > narrow_rows && n_tiles_narrow > 1) {
                if (mode == kGroupRowBlock) vstate_slots -= n_tiles;
                mode = kGroupNarrow;
                units = n_tiles_narrow;
            }
            modes[g] = mode;
            any_narrow |= mode == kGroupNarrow;
            n_units += units;
        }
        us[n_groups] = n_units;
        SWB_CUDA(cudaMemcpyAsync(db->d_unit_start, us, (static_cast<size_t>(n_groups) + 1) * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, s));
        SWB_CUDA(cudaMemcpyAsync(db->d_group_mode, modes, std::max<size_t>(n_groups, 1), cudaMemcpyHostToDevice, s));
        SWB_CUDA(cudaMemcpyAsync(db->d_vstate_off, vso, std::max<size_t>(n_groups, 1) * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, s));
        if (any_rowblock) {
            const size_t need = static_cast<size_t>(vstate_slots) * (kVStateWords / 4) * 32;
            if ((st = ensure_dev(&db->d_vstate, &db->vstate_cap, need, &db->device_bytes)) != SWB_OK) return st;
        }
        if ((st = ensure_dev(&db->d_progress, &db->progress_cap, n_units, &db->device_bytes)) != SWB_OK) return st;
        SWB_CUDA(cudaMemsetAsync(db->d_progress, 0, static_cast<size_t>(n_units) * sizeof(uint32_t), s));
        db->last_units = n_units;
    }
    SWB_CUDA(cudaMemcpyAsync(db->d_matrix, db->h_stage, off_query, cudaMemcpyHostToDevice, s));
    SWB_CUDA(cudaMemcpyAsync(db->d_query, db->h_stage + off_query, m, cudaMemcpyHostToDevice, s));

    const size_t prof_elems = static_cast<size_t>(kProfRows) * pl.pstride;
    const size_t profi_elems = static_cast<size_t>(kProfRows) * pl.n_lane_tiles * 8;
    ProfileParams pp{};
    pp.query = db->d_query;
    pp.matrix = db->d_matrix;
    pp.m = m;
    pp.shift_main = open;
    pp.shift_intra = open;
    pp.pstride = pl.pstride;
    pp.intra_t = pl.intra_t;
    pp.n_lane_tiles = pl.n_lane_tiles;
    if (packed) {
        if ((st = ensure_dev(&db->d_prof8, &db->prof8_cap, prof_elems, &db->device_bytes)) != SWB_OK) return st;
        pp.prof8 = db->d_prof8;
    }
    if (!pl.wide) {
        if ((st = ensure_dev(&db->d_prof8i, &db->prof8i_cap, profi_elems, &db->device_bytes)) != SWB_OK) return st;
        pp.prof8i = db->d_prof8i;
    } else {
        if ((st = ensure_dev(&db->d_prof32i, &db->prof32i_cap, profi_elems, &db->device_bytes)) != SWB_OK) return st;
        pp.prof32i = db->d_prof32i;
    }
    build_profile_kernel<<<64, 256, 0, s>>>(pp);
    ++db->launches;
    SWB_CUDA(cudaEventRecord(db->ev[EV_UP], s));

    // ---- the scan ------------------------------------------------------------------------------------
    if (packed) {
        WaveParams wp{};
        wp.codes = reinterpret_cast<const uint4*>(db->d_codes);
        wp.groups = db->d_groups;
        wp.n_groups = n_groups;
        wp.unit_start = db->d_unit_start;
        wp.group_mode = db->d_group_mode;
        wp.vstate_off = db->d_vstate_off;
        wp.vstate = db->d_vstate;
        wp.n_units = n_units;
        wp.n_tiles_narrow = n_tiles_narrow;
        wp.prof8 = db->d_prof8;
        wp.pstride = pl.pstride;
        wp.n_tiles = n_tiles;
        wp.border0 = db->d_border0;
        wp.border1 = db->d_border1;
        wp.slot_scores = db->d_slot_scores;
        wp.progress = db->d_progress;
        wp.ticket = db->d_counters;
        wp.neg_open2 = pack16(-open);
        wp.neg_ext2 = pack16(-ext);
        const size_t smem = prof_elems;
        const uint32_t warps_per_cta = pl.threads / 32;
        const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(db->sm_count, (n_units + warps_per_cta - 1) / warps_per_cta));
        const bool in_smem = smem <= db->smem_optin;
        {
#define SWB_LAUNCH_S16(NARROW, RB)                                                                                 \
    {                                                                                                              \
        if (in_smem) {                                                                                             \
            SWB_CUDA(cudaFuncSetAttribute(wavefront_s16_kernel<true, kInterTile, kInterThreads, NARROW, RB>,       \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,                             \
                                          static_cast<int>(db->smem_optin)));                                      \
            wavefront_s16_kernel<true, kInterTile, kInterThreads, NARROW, RB><<<grid, kInterThreads, smem, s>>>(wp); \
        } else {                                                                                                   \
            wavefront_s16_kernel<false, kInterTile, kInterThreads, NARROW, RB><<<grid, kInterThreads, 0, s>>>(wp); \
        }                                                                                                          \
    }
            // the narrow-tile and row-block paths are only compiled into the variants that need them, so that the
            // plain 32-column sweep keeps its register allocation
            if (any_narrow && any_rowblock) SWB_LAUNCH_S16(true, true)
            else if (any_narrow) SWB_LAUNCH_S16(true, false)
            else if (any_rowblock) SWB_LAUNCH_S16(false, true)
            else SWB_LAUNCH_S16(false, false)
#undef SWB_LAUNCH_S16
        }
        ++db->launches;
    }
    SWB_CUDA(cudaEventRecord(db->ev[EV_SCAN], s));

    // ---- int32: re-run of lanes above the trust limit, or everything when the packed path is out ----
    if (!packed) {
        if ((st = run_intra(db, pl, nullptr, s)) != SWB_OK) return st;
    } else if (pl.may_overflow) {
        collect_flagged_kernel<<<std::max(1u, std::min(1024u, (db->n_slots + 255) / 256)), 256, 0, s>>>(
            db->d_slot_scores, db->n_slots, pl.limit, db->d_flag_list, db->d_counters + 1);
        ++db->launches;
        if ((st = run_intra(db, pl, db->d_flag_list, s)) != SWB_OK) return st;
    }
    SWB_CUDA(cudaEventRecord(db->ev[EV_RESCORE], s));
    SWB_CUDA(cudaGetLastError());
    return SWB_OK;
}

// Descending top-k of n device keys; result pointer (k entries, zero padded) in *out.
swb_status select_topk(swb_db* db, const uint64_t* d_in, uint64_t n, uint32_t k, const uint64_t** out) {
    cudaStream_t s = db->stream;
    swb_status st;
    if (k <= kSelectMaxK) {
        const uint64_t first_blocks = std::max<uint64_t>(1, (n + kSelectSlice - 1) / kSelectSlice);
        const size_t need = static_cast<size_t>(first_blocks) * k;
        if (need > db->sel_cap) {
            for (auto& p : db->d_sel) {
                if (p) cudaFree(p);
                p = nullptr;
            }
            for (auto& p : db->d_sel)
                if ((st = dev_alloc(&p, need, &db->device_bytes)) != SWB_OK) return st;
            db->sel_cap = need;
        }
        const uint64_t* in = d_in;
        int which = 0;
        for (;;) {
            const uint64_t blocks = std::max<uint64_t>(1, (n + kSelectSlice - 1) / kSelectSlice);
            select_topk_kernel<<<static_cast<unsigned>(blocks), kSelectThreads, 0, s>>>(in, n, k, db->d_sel[which]);
            ++db->launches;
            in = db->d_sel[which];
            n = blocks * k;
            which ^= 1;
            if (blocks == 1) break;
        }
        *out = in;
        return SWB_OK;
    }
    // k > 1024: full bitonic sort of the zero-padded key array
    uint64_t pow2 = 2;
    while (pow2 < n) pow2 <<= 1;
    if (pow2 > db->sort_cap) {
        if (db->d_sort) cudaFree(db->d_sort);
        db->d_sort = nullptr;
        if ((st = dev_alloc(&db->d_sort, pow2, &db->device_bytes)) != SWB_OK) return st;
        db->sort_cap = pow2;
    }
    SWB_CUDA(cudaMemsetAsync(db->d_sort, 0, pow2 * sizeof(uint64_t), s));
    SWB_CUDA(cudaMemcpyAsync(db->d_sort, d_in, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(4096, std::max<uint64_t>(1, pow2 / 2 / 256)));
    for (uint64_t size = 2; size <= pow2; size <<= 1)
        for (uint64_t stride = size >> 1; stride > 0; stride >>= 1) {
            bitonic_step_kernel<<<grid, 256, 0, s>>>(db->d_sort, pow2, size, stride);
            ++db->launches;
        }
    *out = db->d_sort;
    return SWB_OK;
}

void fill_stats(swb_db* db, uint32_t m, swb_stats* st) {
    if (!st) return;
    std::memset(st, 0, sizeof(*st));
    st->lane_scored = db->meta.n_short;
    st->wavefront_scored = db->meta.n_long;
    st->chunks_claimed = db->last_units ? db->last_units : db->meta.n_local;
    st->rescored_i32 = db->h_counters ? db->h_counters[1] : 0;
    st->cells = static_cast<uint64_t>(m) * db->meta.residues;
    const uint64_t mpad = (static_cast<uint64_t>(m) + db->last_tile - 1) / db->last_tile * db->last_tile;
    st->padded_cells = mpad * db->meta.padded_rows * kGroupSeqs;
    st->kernel_launches = db->launches;
    auto span = [&](int a, int b) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, db->ev[a], db->ev[b]);
        return ms;
    };
    st->ms_setup = span(EV_START, EV_UP);
    st->ms_scan = span(EV_UP, EV_SCAN);
    st->ms_rescore = span(EV_SCAN, EV_RESCORE);
    st->ms_topk = span(EV_RESCORE, EV_TOPK);
    st->ms_total = span(EV_START, EV_END);
}

swb_status upload_db(swb_db* db) {
    PackedDb& m = db->meta;
    db->n_slots = static_cast<uint32_t>(m.groups.size() * kGroupSeqs);
    db->max_rows = m.groups.empty() ? 0 : m.groups[0].n_chunks * kRowsPerChunk;
    uint64_t* tally = &db->device_bytes;
    swb_status st;
#define ALLOC_COPY(dptr, vec)                                                                        \
    if ((st = dev_alloc(&(dptr), (vec).size(), tally)) != SWB_OK) return st;                         \
    if (!(vec).empty())                                                                              \
        SWB_CUDA(cudaMemcpy((dptr), (vec).data(), (vec).size() * sizeof((vec)[0]), cudaMemcpyHostToDevice));
    ALLOC_COPY(db->d_codes, m.codes);
    ALLOC_COPY(db->d_groups, m.groups);
    ALLOC_COPY(db->d_slot_index, m.slot_index);
    ALLOC_COPY(db->d_slot_len, m.slot_len);
#undef ALLOC_COPY
    const size_t brows = static_cast<size_t>(m.total_chunks) * kRowsPerChunk * 32 + 64;
    if ((st = dev_alloc(&db->d_border0, brows, tally)) != SWB_OK) return st;
    if ((st = dev_alloc(&db->d_border1, brows, tally)) != SWB_OK) return st;
    if ((st = dev_alloc(&db->d_slot_scores, db->n_slots, tally)) != SWB_OK) return st;
    if ((st = dev_alloc(&db->d_flag_list, db->n_slots, tally)) != SWB_OK) return st;
    if ((st = dev_alloc(&db->d_counters, 4, tally)) != SWB_OK) return st;
    if ((st = dev_alloc(&db->d_unit_start, m.groups.size() + 1, tally)) != SWB_OK) return st;
    if ((st = dev_alloc(&db->d_group_mode, m.groups.size() + 1, tally)) != SWB_OK) return st;
    if ((st = dev_alloc(&db->d_vstate_off, m.groups.size() + 1, tally)) != SWB_OK) return st;
    if ((st = dev_alloc(&db->d_keys, db->n_slots, tally)) != SWB_OK) return st;
    if ((st = dev_alloc(&db->d_matrix, 576, tally)) != SWB_OK) return st;
    // the bulk host copy is no longer needed
    std::vector<uint8_t>().swap(m.codes);
    return SWB_OK;
}

// Stream, events and pinned staging of a fresh handle.
swb_status init_handle_resources(swb_db* db) {
    if (cudaStreamCreateWithFlags(&db->own_stream, cudaStreamNonBlocking) != cudaSuccess)
        return fail(SWB_ERR_CUDA, "cudaStreamCreate failed");
    db->stream = db->own_stream;
    for (auto& ev : db->ev)
        if (cudaEventCreate(&ev) != cudaSuccess) return fail(SWB_ERR_CUDA, "cudaEventCreate failed");
    if (cudaMallocHost(reinterpret_cast<void**>(&db->h_counters), 4 * sizeof(uint32_t)) != cudaSuccess)
        return fail(SWB_ERR_CUDA, "cudaMallocHost failed");
    std::memset(db->h_counters, 0, 4 * sizeof(uint32_t));
    return SWB_OK;
}

swb_status create_from(const SeqSource& src, uint64_t threshold, int32_t device, uint32_t rank,
                       uint32_t count, swb_db** out) {
    if (!out) return fail(SWB_ERR_INVALID, "out is null");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(SWB_ERR_CUDA, "no CUDA device available (this library has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(SWB_ERR_INVALID, "device index out of range");
    auto* db = new swb_db();
    db->device = device;
    bool bad = false;
    const std::string err = pack_database(src, threshold, rank, count, db->meta, &bad);
    if (!err.empty()) {
        delete db;
        return fail(bad ? SWB_ERR_RANGE : SWB_ERR_INVALID, err);
    }
    DeviceGuard guard(device);
    cudaDeviceProp prop{};
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) {
        delete db;
        return fail(SWB_ERR_CUDA, cudaGetErrorString(e));
    }
    if (prop.major < 10) {
        delete db;
        return fail(SWB_ERR_CUDA, "device is not sm_100-class; this library is built for sm_100a only");
    }
    db->sm_count = prop.multiProcessorCount;
    db->smem_optin = prop.sharedMemPerBlockOptin;
    swb_status st = init_handle_resources(db);
    if (st == SWB_OK) st = upload_db(db);
    if (st != SWB_OK) {
        const std::string keep = g_error;
        swb_db_destroy(db);
        g_error = keep;
        return st;
    }
    *out = db;
    return SWB_OK;
}

swb_status search_keys_locked(swb_db* db, const uint8_t* query, uint32_t m, const int32_t* matrix,
                              int32_t open, int32_t ext, uint32_t top_k, const uint64_t** d_out) {
    swb_status st = score_core(db, query, m, matrix, open, ext);
    if (st != SWB_OK) return st;
    cudaStream_t s = db->stream;
    if (db->n_slots) {
        build_keys_kernel<<<std::max(1u, std::min(1024u, (db->n_slots + 255) / 256)), 256, 0, s>>>(
            db->d_slot_scores, db->d_slot_index, db->n_slots, db->d_keys);
        ++db->launches;
    }
    st = select_topk(db, db->d_keys, db->n_slots, top_k, d_out);
    if (st != SWB_OK) return st;
    SWB_CUDA(cudaEventRecord(db->ev[EV_TOPK], s));
    return SWB_OK;
}

}  // namespace

extern "C" {

const char* swb_last_error(void) { return g_error.c_str(); }
const char* swb_version(void) { return "swb200 0.1 (sm_100a)"; }

swb_status swb_device_count(int32_t* count) {
    if (!count) return fail(SWB_ERR_INVALID, "count is null");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        *count = 0;
        return fail(SWB_ERR_CUDA, "cudaGetDeviceCount failed");
    }
    *count = n;
    return SWB_OK;
}

swb_status swb_db_create(const uint8_t* const* seqs, const uint32_t* lens, uint32_t n, uint64_t length_threshold,
                         int32_t device, uint32_t shard_rank, uint32_t shard_count, swb_db** out) {
    if (n && (!seqs || !lens)) return fail(SWB_ERR_INVALID, "seqs/lens are null");
    SeqSource src;
    static const uint8_t* const kNoPtrs[1] = {nullptr};
    static const uint32_t kNoLens[1] = {0};
    src.ptrs = n ? seqs : kNoPtrs;
    src.lens = n ? lens : kNoLens;
    src.n = n;
    return create_from(src, length_threshold, device, shard_rank, shard_count, out);
}

swb_status swb_db_create_flat(const uint8_t* codes, const uint64_t* offsets, uint32_t n, uint64_t length_threshold,
                              int32_t device, uint32_t shard_rank, uint32_t shard_count, swb_db** out) {
    if (!offsets) return fail(SWB_ERR_INVALID, "offsets is null");
    if (n && offsets[n] && !codes) return fail(SWB_ERR_INVALID, "codes is null");
    for (uint32_t i = 0; i < n; ++i)
        if (offsets[i + 1] < offsets[i]) return fail(SWB_ERR_INVALID, "offsets must be non-decreasing");
    SeqSource src;
    src.flat = codes;
    src.offsets = offsets;
    src.n = n;
    return create_from(src, length_threshold, device, shard_rank, shard_count, out);
}

namespace {
struct PackedFileHeader {
    char magic[8];              // "SWB200DB"
    uint32_t version;           // 1
    uint32_t n_total, n_local, n_short, n_long, shard_rank, shard_count, max_length;
    uint64_t residues, padded_rows, total_chunks, length_threshold, n_groups, codes_bytes;
};
constexpr uint32_t kPackedFileVersion = 1;
}  // namespace

swb_status swb_db_save(swb_db* db, const char* path) {
    if (!db || !path) return fail(SWB_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    const PackedDb& m = db->meta;
    PackedFileHeader h{};
    std::memcpy(h.magic, "SWB200DB", 8);
    h.version = kPackedFileVersion;
    h.n_total = m.n_total, h.n_local = m.n_local, h.n_short = m.n_short, h.n_long = m.n_long;
    h.shard_rank = m.shard_rank, h.shard_count = m.shard_count, h.max_length = m.max_length;
    h.residues = m.residues, h.padded_rows = m.padded_rows, h.total_chunks = m.total_chunks;
    h.length_threshold = m.length_threshold, h.n_groups = m.groups.size();
    h.codes_bytes = static_cast<uint64_t>(m.total_chunks) * 32 * 16;
    std::vector<uint8_t> codes(h.codes_bytes);
    if (h.codes_bytes) SWB_CUDA(cudaMemcpy(codes.data(), db->d_codes, h.codes_bytes, cudaMemcpyDeviceToHost));
    FILE* f = std::fopen(path, "wb");
    if (!f) return fail(SWB_ERR_INVALID, std::string("cannot open ") + path + " for writing");
    bool ok = std::fwrite(&h, sizeof(h), 1, f) == 1;
    auto put = [&](const void* data, size_t bytes) { ok = ok && (bytes == 0 || std::fwrite(data, 1, bytes, f) == bytes); };
    put(m.groups.data(), m.groups.size() * sizeof(GroupDesc));
    put(m.slot_index.data(), m.slot_index.size() * sizeof(uint32_t));
    put(m.slot_len.data(), m.slot_len.size() * sizeof(uint32_t));
    put(codes.data(), codes.size());
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return fail(SWB_ERR_INVALID, std::string("short write to ") + path);
    return SWB_OK;
}

swb_status swb_db_load(const char* path, int32_t device, swb_db** out) {
    if (!path || !out) return fail(SWB_ERR_INVALID, "null argument");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(SWB_ERR_CUDA, "no CUDA device available (this library has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(SWB_ERR_INVALID, "device index out of range");
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(SWB_ERR_INVALID, std::string("cannot open ") + path);
    PackedFileHeader h{};
    bool ok = std::fread(&h, sizeof(h), 1, f) == 1 && std::memcmp(h.magic, "SWB200DB", 8) == 0 &&
              h.version == kPackedFileVersion && h.codes_bytes == h.total_chunks * 32 * 16 &&
              h.n_groups <= (1ull << 32) / kGroupSeqs && h.n_local <= h.n_groups * kGroupSeqs;
    auto* db = new swb_db();
    db->device = device;
    PackedDb& m = db->meta;
    if (ok) {
        m.n_total = h.n_total, m.n_local = h.n_local, m.n_short = h.n_short, m.n_long = h.n_long;
        m.shard_rank = h.shard_rank, m.shard_count = h.shard_count, m.max_length = h.max_length;
        m.residues = h.residues, m.padded_rows = h.padded_rows, m.total_chunks = h.total_chunks;
        m.length_threshold = h.length_threshold;
        m.groups.resize(h.n_groups);
        m.slot_index.resize(h.n_groups * kGroupSeqs);
        m.slot_len.resize(h.n_groups * kGroupSeqs);
        m.codes.resize(h.codes_bytes);
        auto get = [&](void* data, size_t bytes) { ok = ok && (bytes == 0 || std::fread(data, 1, bytes, f) == bytes); };
        get(m.groups.data(), m.groups.size() * sizeof(GroupDesc));
        get(m.slot_index.data(), m.slot_index.size() * sizeof(uint32_t));
        get(m.slot_len.data(), m.slot_len.size() * sizeof(uint32_t));
        get(m.codes.data(), m.codes.size());
        // the tables must be consistent with the header before anything is trusted on the device
        uint64_t chunks = 0;
        for (const GroupDesc& g : m.groups) {
            ok = ok && g.chunk_base == chunks;
            chunks += g.n_chunks;
        }
        ok = ok && chunks == h.total_chunks;
        for (uint8_t c : m.codes) ok = ok && c <= kPadCode;
    }
    std::fclose(f);
    if (!ok) {
        delete db;
        return fail(SWB_ERR_INVALID, std::string(path) + " is not a valid swb200 packed database (version 1)");
    }
    DeviceGuard guard(device);
    cudaDeviceProp prop{};
    swb_status st = SWB_OK;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) st = fail(SWB_ERR_CUDA, "cudaGetDeviceProperties failed");
    if (st == SWB_OK) {
        db->sm_count = prop.multiProcessorCount;
        db->smem_optin = prop.sharedMemPerBlockOptin;
        st = init_handle_resources(db);
    }
    if (st == SWB_OK) st = upload_db(db);
    if (st != SWB_OK) {
        const std::string keep = g_error;
        swb_db_destroy(db);
        g_error = keep;
        return st;
    }
    *out = db;
    return SWB_OK;
}

void swb_db_destroy(swb_db* db) {
    if (!db) return;
    {
        DeviceGuard guard(db->device);
        if (db->own_stream) cudaStreamSynchronize(db->own_stream);
        void* ptrs[] = {db->d_codes,      db->d_groups,   db->d_slot_index, db->d_slot_len,    db->d_border0,
                        db->d_border1,    db->d_iborder0, db->d_iborder1,   db->d_slot_scores, db->d_flag_list,
                        db->d_counters,   db->d_unit_start, db->d_group_mode, db->d_vstate_off, db->d_vstate, db->d_progress, db->d_keys,        db->d_sel[0],
                        db->d_sel[1],     db->d_sort,     db->d_all_scores, db->d_query,       db->d_matrix,
                        db->d_prof8,      db->d_prof8i,   db->d_prof32i};
        for (void* p : ptrs)
            if (p) cudaFree(p);
        if (db->h_stage) cudaFreeHost(db->h_stage);
        if (db->h_counters) cudaFreeHost(db->h_counters);
        for (auto& ev : db->ev)
            if (ev) cudaEventDestroy(ev);
        if (db->own_stream) cudaStreamDestroy(db->own_stream);
    }
    delete db;
}

swb_status swb_db_info_get(const swb_db* db, swb_db_info* info) {
    if (!db || !info) return fail(SWB_ERR_INVALID, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->n_total = db->meta.n_total;
    info->n_local = db->meta.n_local;
    info->n_short = db->meta.n_short;
    info->n_long = db->meta.n_long;
    info->n_groups = static_cast<uint32_t>(db->meta.groups.size());
    info->max_length = db->meta.max_length;
    info->shard_rank = db->meta.shard_rank;
    info->shard_count = db->meta.shard_count;
    info->residues = db->meta.residues;
    info->padded_residues = db->meta.padded_rows * kGroupSeqs;
    info->device_bytes = db->device_bytes;
    info->length_threshold = db->meta.length_threshold;
    info->device = db->device;
    return SWB_OK;
}

swb_status swb_db_set_stream(swb_db* db, void* cuda_stream) {
    if (!db) return fail(SWB_ERR_INVALID, "db is null");
    std::lock_guard<std::mutex> lock(db->mu);
    db->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : db->own_stream;
    return SWB_OK;
}

swb_status swb_search_keys(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                           int32_t gap_open, int32_t gap_extend, uint32_t top_k, uint64_t* host_keys,
                           void** device_keys, swb_stats* stats) {
    if (!db) return fail(SWB_ERR_INVALID, "db is null");
    // SearchConfig::validate's message (scheduler.hpp:34)
    if (top_k < 1) return fail(SWB_ERR_INVALID, "top_k must be >= 1");
    swb_status st = check_scoring_args(query, query_len, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    // never select more than the shard holds (plus zero padding up to top_k on the host side)
    const uint64_t n_keys = db->meta.n_local;
    const uint32_t k_eff = static_cast<uint32_t>(std::min<uint64_t>(top_k, std::max<uint64_t>(n_keys, 1)));
    const uint64_t* d_top = nullptr;
    st = search_keys_locked(db, query, query_len, matrix, gap_open, gap_extend, k_eff, &d_top);
    if (st != SWB_OK) return st;
    cudaStream_t s = db->stream;
    if (host_keys) {
        st = ensure_stage(db, static_cast<size_t>(k_eff) * sizeof(uint64_t));
        if (st != SWB_OK) return st;
        SWB_CUDA(cudaMemcpyAsync(db->h_stage, d_top, static_cast<size_t>(k_eff) * sizeof(uint64_t),
                                 cudaMemcpyDeviceToHost, s));
    }
    SWB_CUDA(cudaMemcpyAsync(db->h_counters, db->d_counters, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SWB_CUDA(cudaEventRecord(db->ev[EV_END], s));
    SWB_CUDA(cudaStreamSynchronize(s));
    if (host_keys) {
        std::memcpy(host_keys, db->h_stage, static_cast<size_t>(k_eff) * sizeof(uint64_t));
        for (uint32_t i = k_eff; i < top_k; ++i) host_keys[i] = 0;
    }
    if (device_keys) *device_keys = (k_eff == top_k) ? const_cast<uint64_t*>(d_top) : nullptr;
    fill_stats(db, query_len, stats);
    return SWB_OK;
}

swb_status swb_search(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix, int32_t gap_open,
                      int32_t gap_extend, uint32_t top_k, swb_hit* hits, uint32_t* n_hits, swb_stats* stats) {
    if (!hits || !n_hits) return fail(SWB_ERR_INVALID, "hits/n_hits are null");
    if (top_k < 1) return fail(SWB_ERR_INVALID, "top_k must be >= 1");
    if (!db) return fail(SWB_ERR_INVALID, "db is null");
    const uint64_t n_keys = db->meta.n_local;
    const uint32_t k_eff = static_cast<uint32_t>(std::min<uint64_t>(top_k, std::max<uint64_t>(n_keys, 1)));
    std::vector<uint64_t> keys(k_eff);
    swb_status st = swb_search_keys(db, query, query_len, matrix, gap_open, gap_extend, k_eff, keys.data(), nullptr, stats);
    if (st != SWB_OK) return st;
    uint32_t cnt = 0;
    for (uint32_t i = 0; i < k_eff; ++i) {
        if (!keys[i]) break;
        hits[cnt].db_index = 0xFFFFFFFFu - static_cast<uint32_t>(keys[i] & 0xFFFFFFFFu);
        hits[cnt].score = static_cast<int32_t>(keys[i] >> 32);
        ++cnt;
    }
    *n_hits = cnt;
    return SWB_OK;
}

swb_status swb_score_all(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix, int32_t gap_open,
                         int32_t gap_extend, int32_t* scores, swb_stats* stats) {
    if (!db || !scores) return fail(SWB_ERR_INVALID, "null argument");
    swb_status st = check_scoring_args(query, query_len, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    st = score_core(db, query, query_len, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    cudaStream_t s = db->stream;
    const uint32_t n_total = db->meta.n_total;
    if (!db->d_all_scores)
        if ((st = dev_alloc(&db->d_all_scores, n_total, &db->device_bytes)) != SWB_OK) return st;
    // entries of other shards must stay untouched: stage the caller's values first
    SWB_CUDA(cudaMemcpyAsync(db->d_all_scores, scores, static_cast<size_t>(n_total) * sizeof(int32_t),
                             cudaMemcpyHostToDevice, s));
    if (db->n_slots) {
        scatter_scores_kernel<<<std::max(1u, std::min(1024u, (db->n_slots + 255) / 256)), 256, 0, s>>>(
            db->d_slot_scores, db->d_slot_index, db->n_slots, db->d_all_scores);
        ++db->launches;
    }
    SWB_CUDA(cudaEventRecord(db->ev[EV_TOPK], s));
    SWB_CUDA(cudaMemcpyAsync(scores, db->d_all_scores, static_cast<size_t>(n_total) * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, s));
    SWB_CUDA(cudaMemcpyAsync(db->h_counters, db->d_counters, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SWB_CUDA(cudaEventRecord(db->ev[EV_END], s));
    SWB_CUDA(cudaStreamSynchronize(s));
    fill_stats(db, query_len, stats);
    return SWB_OK;
}

swb_status swb_merge_keys(const uint64_t* keys, uint64_t n, int32_t keys_on_device, int32_t device, uint32_t top_k,
                          swb_hit* hits, uint32_t* n_hits) {
    if (!hits || !n_hits) return fail(SWB_ERR_INVALID, "hits/n_hits are null");
    if (top_k < 1) return fail(SWB_ERR_INVALID, "top_k must be >= 1");
    if (n && !keys) return fail(SWB_ERR_INVALID, "keys is null");
    *n_hits = 0;
    if (n == 0) return SWB_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(SWB_ERR_CUDA, "no CUDA device available (this library has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(SWB_ERR_INVALID, "device index out of range");
    DeviceGuard guard(device);
    // a scratch handle gives select_topk its buffers and stream
    swb_db tmp;
    tmp.device = device;
    SWB_CUDA(cudaStreamCreateWithFlags(&tmp.own_stream, cudaStreamNonBlocking));
    tmp.stream = tmp.own_stream;
    uint64_t* d_in = nullptr;
    swb_status st = SWB_OK;
    std::vector<uint64_t> top;
    const uint32_t k_eff = static_cast<uint32_t>(std::min<uint64_t>(top_k, n));
    do {
        const uint64_t* src = keys;
        if (!keys_on_device) {
            if ((st = dev_alloc(&d_in, n, &tmp.device_bytes)) != SWB_OK) break;
            if (cudaMemcpyAsync(d_in, keys, n * sizeof(uint64_t), cudaMemcpyHostToDevice, tmp.stream) != cudaSuccess) {
                st = fail(SWB_ERR_CUDA, "cudaMemcpyAsync failed");
                break;
            }
            src = d_in;
        }
        const uint64_t* d_top = nullptr;
        if ((st = select_topk(&tmp, src, n, k_eff, &d_top)) != SWB_OK) break;
        top.resize(k_eff);
        if (cudaMemcpyAsync(top.data(), d_top, k_eff * sizeof(uint64_t), cudaMemcpyDeviceToHost, tmp.stream) != cudaSuccess ||
            cudaStreamSynchronize(tmp.stream) != cudaSuccess) {
            st = fail(SWB_ERR_CUDA, std::string("merge: ") + cudaGetErrorString(cudaGetLastError()));
            break;
        }
    } while (false);
    if (d_in) cudaFree(d_in);
    for (auto& p : tmp.d_sel)
        if (p) cudaFree(p);
    if (tmp.d_sort) cudaFree(tmp.d_sort);
    cudaStreamDestroy(tmp.own_stream);
    tmp.own_stream = nullptr;
    if (st != SWB_OK) return st;
    uint32_t cnt = 0;
    for (uint32_t i = 0; i < k_eff; ++i) {
        if (!top[i]) break;
        hits[cnt].db_index = 0xFFFFFFFFu - static_cast<uint32_t>(top[i] & 0xFFFFFFFFu);
        hits[cnt].score = static_cast<int32_t>(top[i] >> 32);
        ++cnt;
    }
    *n_hits = cnt;
    return SWB_OK;
}

swb_status swb_score_batch(const uint8_t* query, uint32_t query_len, const uint8_t* const* subjects,
                           const uint32_t* lens, uint32_t count, uint32_t lane_width, const int32_t* matrix,
                           int32_t gap_open, int32_t gap_extend, int32_t device, int32_t* out) {
    // align.hpp:93-95, same messages
    if (lane_width < 1) return fail(SWB_ERR_INVALID, "lane_width must be >= 1");
    if (count > lane_width) return fail(SWB_ERR_INVALID, "more subjects than lanes");
    if (!out) return fail(SWB_ERR_INVALID, "out is null");
    if (count && (!subjects || !lens)) return fail(SWB_ERR_INVALID, "subjects/lens are null");
    swb_status st = check_scoring_args(query, query_len, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    for (uint32_t l = 0; l < lane_width; ++l) out[l] = 0;
    // Null lanes are padding (align.hpp:126,148): they are packed as empty sequences and their
    // score (0) is simply not reported back.
    std::vector<const uint8_t*> ptrs(count);
    std::vector<uint32_t> ls(count);
    for (uint32_t i = 0; i < count; ++i) {
        ptrs[i] = subjects[i];
        ls[i] = subjects[i] ? lens[i] : 0;
    }
    if (count == 0 || query_len == 0) return SWB_OK;
    swb_db* db = nullptr;
    // threshold = infinity: every lane goes through the inter-task kernel, whatever its length
    st = swb_db_create(ptrs.data(), ls.data(), count, ~0ull, device, 0, 1, &db);
    if (st != SWB_OK) return st;
    std::vector<int32_t> scores(count, 0);
    st = swb_score_all(db, query, query_len, matrix, gap_open, gap_extend, scores.data(), nullptr);
    const std::string keep = g_error;
    swb_db_destroy(db);
    g_error = keep;
    if (st != SWB_OK) return st;
    for (uint32_t i = 0; i < count; ++i) out[i] = subjects[i] ? scores[i] : 0;
    return SWB_OK;
}

swb_status swb_score_pair(const uint8_t* query, uint32_t query_len, const uint8_t* subject, uint32_t subject_len,
                          const int32_t* matrix, int32_t gap_open, int32_t gap_extend, uint64_t chunk_width,
                          int32_t device, int32_t* score) {
    // align.hpp:169, same message
    if (chunk_width < 1) return fail(SWB_ERR_INVALID, "chunk_width must be >= 1");
    if (!score) return fail(SWB_ERR_INVALID, "score is null");
    if (subject_len && !subject) return fail(SWB_ERR_INVALID, "subject is null");
    swb_status st = check_scoring_args(query, query_len, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    *score = 0;
    if (query_len == 0 || subject_len == 0) return SWB_OK;
    swb_db* db = nullptr;
    const uint8_t* ptrs[1] = {subject};
    const uint32_t ls[1] = {subject_len};
    // threshold = 0 routes the sequence to the intra-task pool (scheduler.hpp:59-62); force_intra makes
    // the warp-shuffle wavefront kernel score it (one CTA for the one pair)
    st = swb_db_create(ptrs, ls, 1, 0, device, 0, 1, &db);
    if (st != SWB_OK) return st;
    db->force_intra = true;
    int32_t out[1] = {0};
    st = swb_score_all(db, query, query_len, matrix, gap_open, gap_extend, out, nullptr);
    const std::string keep = g_error;
    swb_db_destroy(db);
    g_error = keep;
    if (st != SWB_OK) return st;
    *score = out[0];
    return SWB_OK;
}

swb_status swb_db_align_hits(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                             int32_t gap_open, int32_t gap_extend, const swb_hit* hits, uint32_t n_hits,
                             uint64_t memory_cap, swb_alignment* out, uint8_t* ops, const uint64_t* ops_offset) {
    if (!db) return fail(SWB_ERR_INVALID, "db is null");
    if (n_hits && (!hits || !out || !ops_offset)) return fail(SWB_ERR_INVALID, "null argument");
    swb_status st = check_scoring_args(query, query_len, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    cudaStream_t s = db->stream;

    if (db->slot_of.empty() && db->meta.n_total) {      // db_index -> slot, built on first use
        db->slot_of.assign(db->meta.n_total, kNoSequence);
        for (uint32_t slot = 0; slot < db->meta.slot_index.size(); ++slot)
            if (db->meta.slot_index[slot] != kNoSequence) db->slot_of[db->meta.slot_index[slot]] = slot;
    }

    const uint64_t m = query_len;
    const uint32_t pitch = (query_len + 7) / 8 * 8;
    std::vector<TracebackJob> jobs;
    std::vector<uint32_t> job_hit;
    uint64_t dir_bytes = 0, border_elems = 0, ops_bytes = 0;
    for (uint32_t i = 0; i < n_hits; ++i) {
        std::memset(&out[i], 0, sizeof(out[i]));
        const uint32_t idx = hits[i].db_index;
        if (idx >= db->meta.n_total || db->slot_of[idx] == kNoSequence)
            return fail(SWB_ERR_INVALID, "hit " + std::to_string(i) + " does not belong to this shard");
        const uint32_t slot = db->slot_of[idx];
        const uint64_t n = db->meta.slot_len[slot];
        if (m == 0 || n == 0) continue;                                     // align.hpp:260: empty alignment
        const uint64_t cells = (m + 1) * (n + 1);                           // align.hpp:262-267
        if (cells / (m + 1) != n + 1 || cells > memory_cap) {
            out[i].score = hits[i].score;
            out[i].capped = 1;
            continue;
        }
        const GroupDesc& gd = db->meta.groups[slot / kGroupSeqs];
        const uint32_t sl = slot % kGroupSeqs;
        TracebackJob job{};
        job.codes_off = (static_cast<uint64_t>(gd.chunk_base) * 32 + (sl & 31)) * 16 + (sl >> 5) * 8;
        job.dir_off = dir_bytes;
        job.border_off = border_elems;
        job.ops_off = ops_bytes;
        job.n = static_cast<uint32_t>(n);
        job.result_off = static_cast<uint32_t>(jobs.size());
        dir_bytes += static_cast<uint64_t>(pitch) * n;
        border_elems += n;
        ops_bytes += (m + n + 63) & ~63ull;
        jobs.push_back(job);
        job_hit.push_back(i);
    }
    if (jobs.empty()) return SWB_OK;

    const QueryPlan pl = make_plan(db, query_len, matrix, gap_open, gap_extend);
    const uint32_t n_lane_tiles = (query_len + 7) / 8;
    const uint32_t warps = std::min<uint32_t>(kIntraMaxWarps, (n_lane_tiles + 31) / 32);
    const uint32_t passes = (n_lane_tiles + 32 * warps - 1) / (32 * warps);
    const size_t profi_elems = static_cast<size_t>(kProfRows) * n_lane_tiles * 8;

    uint8_t *d_dir = nullptr, *d_ops = nullptr, *d_query = nullptr;
    int32_t *d_result = nullptr, *d_prof32 = nullptr;
    uint2 *d_b0 = nullptr, *d_b1 = nullptr;
    int8_t* d_prof8 = nullptr;
    TracebackJob* d_jobs = nullptr;
    std::vector<int32_t> results(jobs.size() * 8, 0);
    std::vector<uint8_t> reversed(ops_bytes);
    st = [&]() -> swb_status {
        swb_status e;
        if ((e = dev_alloc(&d_dir, dir_bytes, nullptr)) != SWB_OK) return e;
        if ((e = dev_alloc(&d_ops, ops_bytes, nullptr)) != SWB_OK) return e;
        if ((e = dev_alloc(&d_result, results.size(), nullptr)) != SWB_OK) return e;
        if ((e = dev_alloc(&d_b0, border_elems, nullptr)) != SWB_OK) return e;
        if ((e = dev_alloc(&d_b1, border_elems, nullptr)) != SWB_OK) return e;
        if ((e = dev_alloc(&d_query, m, nullptr)) != SWB_OK) return e;
        if ((e = dev_alloc(&d_jobs, jobs.size(), nullptr)) != SWB_OK) return e;
        if (!pl.wide) { if ((e = dev_alloc(&d_prof8, profi_elems, nullptr)) != SWB_OK) return e; }
        else { if ((e = dev_alloc(&d_prof32, profi_elems, nullptr)) != SWB_OK) return e; }
        SWB_CUDA(cudaMemcpyAsync(d_query, query, m, cudaMemcpyHostToDevice, s));
        SWB_CUDA(cudaMemcpyAsync(db->d_matrix, matrix, 576 * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        SWB_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), jobs.size() * sizeof(TracebackJob), cudaMemcpyHostToDevice, s));
        SWB_CUDA(cudaMemsetAsync(d_result, 0, results.size() * sizeof(int32_t), s));
        ProfileParams pp{};
        pp.query = d_query;
        pp.matrix = db->d_matrix;
        pp.m = query_len;
        pp.shift_main = gap_open;
        pp.shift_intra = gap_open;
        pp.pstride = 0;                 // only the re-tiled form is needed
        pp.intra_t = 8;
        pp.n_lane_tiles = n_lane_tiles;
        pp.prof8i = d_prof8;
        pp.prof32i = d_prof32;
        build_profile_kernel<<<64, 256, 0, s>>>(pp);
        TracebackParams tp{};
        tp.codes = db->d_codes;
        tp.query = d_query;
        tp.jobs = d_jobs;
        tp.m = query_len;
        tp.profi = pl.wide ? static_cast<const void*>(d_prof32) : static_cast<const void*>(d_prof8);
        tp.n_lane_tiles = n_lane_tiles;
        tp.n_passes = passes;
        tp.border0 = d_b0;
        tp.border1 = d_b1;
        tp.dir = d_dir;
        tp.pitch = pitch;
        tp.open = gap_open;
        tp.ext = gap_extend;
        tp.result = d_result;
        tp.ops_reversed = d_ops;
        const unsigned grid = static_cast<unsigned>(jobs.size());
        if (pl.wide) traceback_fill_kernel<int32_t><<<grid, warps * 32, 0, s>>>(tp);
        else traceback_fill_kernel<int8_t><<<grid, warps * 32, 0, s>>>(tp);
        traceback_walk_kernel<<<grid, 32, 0, s>>>(tp);
        SWB_CUDA(cudaMemcpyAsync(results.data(), d_result, results.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SWB_CUDA(cudaMemcpyAsync(reversed.data(), d_ops, ops_bytes, cudaMemcpyDeviceToHost, s));
        SWB_CUDA(cudaStreamSynchronize(s));
        SWB_CUDA(cudaGetLastError());
        return SWB_OK;
    }();
    for (void* ptr : {static_cast<void*>(d_dir), static_cast<void*>(d_ops), static_cast<void*>(d_result),
                      static_cast<void*>(d_b0), static_cast<void*>(d_b1), static_cast<void*>(d_prof8),
                      static_cast<void*>(d_prof32), static_cast<void*>(d_query), static_cast<void*>(d_jobs)})
        if (ptr) cudaFree(ptr);
    if (st != SWB_OK) return st;

    for (size_t j = 0; j < jobs.size(); ++j) {
        const uint32_t i = job_hit[j];
        const int32_t* r = &results[j * 8];
        out[i].score = r[0];
        if (r[0] <= 0) continue;
        out[i].query_begin = static_cast<uint64_t>(r[4]);
        out[i].query_end = static_cast<uint64_t>(r[2]);
        out[i].subject_begin = static_cast<uint64_t>(r[5]);
        out[i].subject_end = static_cast<uint64_t>(r[1]);
        out[i].n_ops = static_cast<uint64_t>(r[3]);
        if (ops) {
            const uint64_t room = ops_offset[i + 1] - ops_offset[i];
            const uint8_t* src = reversed.data() + jobs[j].ops_off;
            const uint64_t count = static_cast<uint64_t>(r[3]);
            for (uint64_t k = 0; k < count && k < room; ++k) ops[ops_offset[i] + k] = src[count - 1 - k];
        }
    }
    return SWB_OK;
}

swb_status swb_align_traceback(const uint8_t* query, uint32_t query_len, const uint8_t* subject, uint32_t subject_len,
                               const int32_t* matrix, int32_t gap_open, int32_t gap_extend, uint64_t memory_cap,
                               int32_t device, swb_alignment* out, uint8_t* ops, uint64_t ops_capacity) {
    if (!out) return fail(SWB_ERR_INVALID, "out is null");
    if (subject_len && !subject) return fail(SWB_ERR_INVALID, "subject is null");
    swb_status st = check_scoring_args(query, query_len, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    std::memset(out, 0, sizeof(*out));
    const uint64_t m = query_len, n = subject_len;
    if (m == 0 || n == 0) return SWB_OK;                                  // align.hpp:260
    swb_hit hit{0, 0};
    const uint64_t cells = (m + 1) * (n + 1);                             // align.hpp:262-267
    if (cells / (m + 1) != n + 1 || cells > memory_cap) {
        st = swb_score_pair(query, query_len, subject, subject_len, matrix, gap_open, gap_extend, 1, device, &hit.score);
        if (st != SWB_OK) return st;
        out->score = hit.score;
        out->capped = 1;
        return SWB_OK;
    }
    swb_db* db = nullptr;
    const uint8_t* ptrs[1] = {subject};
    const uint32_t ls[1] = {subject_len};
    st = swb_db_create(ptrs, ls, 1, 0, device, 0, 1, &db);
    if (st != SWB_OK) return st;
    const uint64_t offsets[2] = {0, ops_capacity};
    st = swb_db_align_hits(db, query, query_len, matrix, gap_open, gap_extend, &hit, 1, memory_cap, out, ops, offsets);
    const std::string keep = g_error;
    swb_db_destroy(db);
    g_error = keep;
    return st;
}

swb_status swb_shard_assignment(const uint32_t* lens, uint32_t n, uint64_t length_threshold, uint32_t shard_count,
                                uint32_t* shard_of) {
    if (n && (!lens || !shard_of)) return fail(SWB_ERR_INVALID, "null argument");
    if (shard_count < 1) return fail(SWB_ERR_INVALID, "shard_count must be >= 1");
    std::vector<const uint8_t*> ptrs(std::max<uint32_t>(n, 1), nullptr);
    SeqSource src;
    src.ptrs = ptrs.data();
    src.lens = lens;
    src.n = n;
    std::vector<uint32_t> result;
    shard_assignment(src, length_threshold, shard_count, result);
    for (uint32_t i = 0; i < n; ++i) shard_of[i] = result[i];
    return SWB_OK;
}

}  // extern "C"

// ---- pipe-rate microbenchmark -------------------------------------------------------------------
template <int OP>
static swb_status run_pipe(int sm_count, double seconds, double* rate_ginst, double* clock_mhz) {
    uint32_t* sink = nullptr;
    unsigned long long* cyc = nullptr;
    SWB_CUDA(cudaMalloc(&sink, 64));
    SWB_CUDA(cudaMalloc(&cyc, sizeof(unsigned long long)));
    cudaEvent_t a, b;
    SWB_CUDA(cudaEventCreate(&a));
    SWB_CUDA(cudaEventCreate(&b));
    const int grid = sm_count * 2, block = 512;
    int iters = 2000;
    double ms = 0;
    for (int attempt = 0; attempt < 6; ++attempt) {
        SWB_CUDA(cudaMemset(cyc, 0, sizeof(unsigned long long)));
        pipe_rate_kernel<OP><<<grid, block>>>(sink, cyc, 0xfffefffeu, 0x00030003u, iters);   // warm-up
        SWB_CUDA(cudaMemset(cyc, 0, sizeof(unsigned long long)));
        SWB_CUDA(cudaEventRecord(a));
        pipe_rate_kernel<OP><<<grid, block>>>(sink, cyc, 0xfffefffeu, 0x00030003u, iters);
        SWB_CUDA(cudaEventRecord(b));
        SWB_CUDA(cudaEventSynchronize(b));
        float fms = 0;
        SWB_CUDA(cudaEventElapsedTime(&fms, a, b));
        ms = fms;
        if (ms >= seconds * 1000.0 * 0.5 || iters > (1 << 28)) break;
        const double scale = std::min(64.0, std::max(2.0, seconds * 1000.0 / std::max(ms, 1e-3)));
        iters = static_cast<int>(iters * scale);
    }
    unsigned long long cycles = 0;
    SWB_CUDA(cudaMemcpy(&cycles, cyc, sizeof(cycles), cudaMemcpyDeviceToHost));
    const double inst = static_cast<double>(grid) * block * static_cast<double>(iters) * kPipeChains * kPipeUnroll;
    *rate_ginst = inst / (ms * 1e-3) / 1e9;
    *clock_mhz = static_cast<double>(cycles) / (ms * 1e-3) / 1e6;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    cudaFree(cyc);
    return SWB_OK;
}

extern "C" {

swb_status swb_measure_pipe_rates(int32_t device, double seconds, swb_pipe_rates* out) {
    if (!out) return fail(SWB_ERR_INVALID, "out is null");
    std::memset(out, 0, sizeof(*out));
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(SWB_ERR_CUDA, "no CUDA device available");
    if (device < 0 || device >= ndev) return fail(SWB_ERR_INVALID, "device index out of range");
    DeviceGuard guard(device);
    cudaDeviceProp prop{};
    SWB_CUDA(cudaGetDeviceProperties(&prop, device));
    out->sm_count = prop.multiProcessorCount;
    // half of the budget goes to the instruction the roofline is defined on, best of two runs (the first launch
    // after an idle period can still see the clock ramping); the rest is shared by the other probes
    const double each = std::max(0.02, seconds * 0.5 / (kOpCount - 1));
    double clk = 0, clk_sum = 0;
    swb_status st;
    for (int rep = 0; rep < 2; ++rep) {
        double rate = 0, c = 0;
        if ((st = run_pipe<kOpViaddmnmx16>(prop.multiProcessorCount, std::max(0.02, seconds * 0.25), &rate, &c)) != SWB_OK) return st;
        if (rate > out->viaddmnmx_s16x2) out->viaddmnmx_s16x2 = rate, clk_sum = c;
    }
    if ((st = run_pipe<kOpVimnmx3_16>(prop.multiProcessorCount, each, &out->vimnmx3_s16x2, &clk)) != SWB_OK) return st;
    if ((st = run_pipe<kOpViadd16>(prop.multiProcessorCount, each, &out->viadd_16x2, &clk)) != SWB_OK) return st;
    if ((st = run_pipe<kOpViaddmnmx32>(prop.multiProcessorCount, each, &out->viaddmnmx_s32, &clk)) != SWB_OK) return st;
    if ((st = run_pipe<kOpPrmt>(prop.multiProcessorCount, each, &out->prmt, &clk)) != SWB_OK) return st;
    if ((st = run_pipe<kOpImad>(prop.multiProcessorCount, each, &out->imad, &clk)) != SWB_OK) return st;
    if ((st = run_pipe<kOpMixAluFma>(prop.multiProcessorCount, each, &out->mix_alu_fma, &clk)) != SWB_OK) return st;
    out->sm_clock_mhz = clk_sum;
    return SWB_OK;
}

}  // extern "C"

#include "multi.inl"
