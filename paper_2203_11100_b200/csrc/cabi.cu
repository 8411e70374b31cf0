// cabi.cu -- the C-ABI of include/swb200.h: handles, orchestration, launches.
//
// Host flow of one search (replaces scheduler.hpp:188-244):
//   validate -> upload query + matrix + unit table -> build_profile_kernel -> packed-int16
//   tile-wavefront kernel over all groups -> collect + int32 re-run of lanes above the trust limit
//   -> key build -> top-k select -> download k hits.
// Everything runs on one stream per handle; no host synchronisation happens between the upload and
// the final download.
//
// One translation unit, split by topic:
//   plan.inl     per-search decisions (which kernel, profile geometry, unit policy knobs)
//   handle.inl   shard handle lifetime, upload of the packed database, statistics
//   scan.inl     score_core (upload, profile, unit table, scan, re-run) and the top-k select
//   duo.inl      shared scans of swb_search_many: two streams of queries per scan
//   persist.inl  swb_db_save / swb_db_load
//   pairs.inl    swb_merge_keys, swb_score_batch, swb_score_pair, swb_db_align_hits, swb_align_traceback
//   pipe.inl     swb_measure_pipe_rates
//   multi.inl    several GPUs in one process (NCCL)
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/swb200.h"
#include "kernels.cuh"
#include "pipeline.cuh"
#include "duo.cuh"
#include "pack.hpp"
#include "pipe_rates.cuh"
#include "scan_plan.hpp"

static_assert(swb::kScanAuto == SWB_SCAN_AUTO && swb::kScanPipeline == SWB_SCAN_PIPELINE && swb::kScanWavefront == SWB_SCAN_WAVEFRONT,
              "scan_plan.hpp and swb200.h disagree on the scan policies");

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

// ---- block cache of the ad-hoc entry points ------------------------------------------------------------------------
// swb_score_pair / swb_score_batch / swb_align_traceback / swb_merge_keys build a handle per call (the reference's
// sw_score_scalar, sw_score_batch, sw_align_traceback take plain sequences, align.hpp:42,91,166,262): some thirty
// cudaMalloc / cudaFree and three cudaMallocHost per call cost milliseconds, the kernels microseconds.  While such a call
// runs (BlockCacheScope on its thread) device and pinned blocks up to kCacheBlockMax come out of size classes (powers of two)
// kept per device and go back there instead of to the driver, up to kCacheBytesMax per device.  Handles of resident
// databases (swb_db_create & co.) do not use it.  A block is only handed back after the device went idle (release_block
// synchronises unless the caller just did), so reuse needs no stream ordering.
constexpr size_t kCacheBlockMax = 8u << 20;
constexpr size_t kCacheBytesMax = 256u << 20;

struct BlockCache {
    struct Class {
        std::vector<void*> dev, host;
    };
    std::mutex mu;
    std::unordered_map<void*, uint32_t> owned;          // block -> (device << 8) | (host ? 0x80 : 0) | log2(size)
    std::unordered_map<uint32_t, Class> classes;        // (device << 8) | log2(size)
    std::unordered_map<int, size_t> cached_bytes;       // per device, blocks lying in `classes`
};

BlockCache& block_cache() {   // leaked on purpose: no CUDA call from a static destructor
    static BlockCache* c = new BlockCache();
    return *c;
}

thread_local int t_cache_scope = 0;

struct BlockCacheScope {
    BlockCacheScope() { ++t_cache_scope; }
    ~BlockCacheScope() { --t_cache_scope; }
    BlockCacheScope(const BlockCacheScope&) = delete;
    BlockCacheScope& operator=(const BlockCacheScope&) = delete;
};

inline uint32_t size_class(size_t bytes) {
    uint32_t lg = 9;   // 512 B: the smallest class
    while ((size_t(1) << lg) < bytes) ++lg;
    return lg;
}

// nullptr: not served from the cache (scope not active, block too large, nothing cached and the driver refused)
void* cached_block(size_t bytes, bool host) {
    static const bool off = std::getenv("SWB200_NO_BLOCK_CACHE") != nullptr;   // measurement: every block from the driver
    if (!t_cache_scope || off || bytes > kCacheBlockMax) return nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    const uint32_t lg = size_class(bytes);
    const uint32_t key = (static_cast<uint32_t>(dev) << 8) | lg;
    BlockCache& c = block_cache();
    {
        std::lock_guard<std::mutex> lock(c.mu);
        auto it = c.classes.find(key);
        if (it != c.classes.end()) {
            auto& list = host ? it->second.host : it->second.dev;
            if (!list.empty()) {
                void* p = list.back();
                list.pop_back();
                c.cached_bytes[dev] -= size_t(1) << lg;
                return p;
            }
        }
    }
    void* p = nullptr;
    const cudaError_t e = host ? cudaMallocHost(&p, size_t(1) << lg) : cudaMalloc(&p, size_t(1) << lg);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    std::lock_guard<std::mutex> lock(c.mu);
    c.owned[p] = key | (host ? 0x80u : 0u);
    return p;
}

// Blocks of the cache go back to their class, others to the driver.  idle: the caller has synchronised every stream that
// touched the block (cudaFree would have waited for the device by itself).
void release_block(void* p, bool host, bool idle = false) {
    if (!p) return;
    BlockCache& c = block_cache();
    uint32_t tag = 0;
    bool ours = false;
    {
        std::lock_guard<std::mutex> lock(c.mu);
        auto it = c.owned.find(p);
        if (it != c.owned.end()) ours = true, tag = it->second;
    }
    if (!ours) {
        if (host) cudaFreeHost(p);
        else cudaFree(p);
        return;
    }
    if (!idle) cudaDeviceSynchronize();
    const int dev = static_cast<int>(tag >> 8);
    const size_t bytes = size_t(1) << (tag & 0x7fu);
    {
        std::lock_guard<std::mutex> lock(c.mu);
        size_t& cached = c.cached_bytes[dev];
        if (cached + bytes <= kCacheBytesMax) {
            auto& cl = c.classes[tag & ~0x80u];
            (host ? cl.host : cl.dev).push_back(p);
            cached += bytes;
            return;
        }
        c.owned.erase(p);
    }
    if (host) cudaFreeHost(p);
    else cudaFree(p);
}

inline void dev_free(void* p, bool idle = false) { release_block(p, false, idle); }
inline void host_free(void* p, bool idle = false) { release_block(p, true, idle); }

swb_status host_alloc(void** ptr, size_t bytes) {
    if ((*ptr = cached_block(bytes, true)) != nullptr) return SWB_OK;
    SWB_CUDA(cudaMallocHost(ptr, bytes));
    return SWB_OK;
}

template <class T>
swb_status dev_alloc(T** ptr, size_t count, uint64_t* tally) {
    *ptr = nullptr;
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if ((*ptr = static_cast<T*>(cached_block(bytes, false))) == nullptr)
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
    cudaStream_t side_stream = nullptr;   // the pipeline kernel, next to the wavefront kernel on `stream`
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool pipe_attr_set = false;
    int scan_policy = SWB_SCAN_AUTO;
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
    uint8_t* d_nlinks = nullptr;   // narrow groups' link buffers (kernels.cuh: 256 B per row and tile boundary)
    size_t nlinks_cap = 0;
    uint64_t* d_keys = nullptr;
    uint64_t* d_sel[2] = {nullptr, nullptr};
    size_t sel_cap = 0;
    uint64_t* d_sort = nullptr;
    size_t sort_cap = 0;
    int32_t* d_all_scores = nullptr;
    // shared scans of swb_search_many (duo.cuh)
    int32_t* d_multi_scores = nullptr;   // [queries of the scan][n_slots]
    size_t multi_scores_cap = 0;
    uint8_t* d_multi_codes = nullptr;    // the scan's queries, concatenated
    size_t multi_codes_cap = 0;
    uint8_t* d_duo_tiles = nullptr;      // DuoTile[n_tiles]
    size_t duo_tiles_cap = 0;
    uint32_t* d_prof2 = nullptr;
    size_t prof2_cap = 0;
    uint32_t* d_duo_progress = nullptr;  // pass items: [half-groups][passes]
    size_t duo_progress_cap = 0;
    bool duo_attr_set = false;

    // query side
    uint32_t query_cap = 0;
    uint8_t* d_query = nullptr;
    int32_t* d_matrix = nullptr;
    int8_t *d_prof8 = nullptr, *d_prof8i = nullptr;
    int32_t* d_prof32i = nullptr;
    size_t prof8_cap = 0, prof8i_cap = 0, prof32i_cap = 0;

    uint8_t* h_stage = nullptr;   // pinned: matrix + query + unit table up, keys down
    size_t stage_cap = 0;
    size_t stage_base = 0;        // offset of the current query's staging area (swb_search_many pipelines several)
    std::vector<cudaEvent_t> many_events;   // per-query start/end events of swb_search_many
    uint32_t* h_counters = nullptr;   // pinned copy of d_counters
    uint64_t* h_merge = nullptr;      // pinned: merged keys down (swb_db_merge_keys)
    uint32_t merge_cap = 0;
    cudaEvent_t ev[EV_COUNT] = {};
    bool async_pending = false;   // swb_search_keys_device: a search is enqueued whose inputs still sit in h_stage
    uint32_t launches = 0;        // of the current search
    uint32_t launches_total = 0;  // of all earlier ones
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
    if (db->h_stage) host_free(db->h_stage);
    db->h_stage = nullptr;
    db->stage_cap = 0;
    const size_t cap = std::max<size_t>(bytes * 2, 1 << 16);
    swb_status st = host_alloc(reinterpret_cast<void**>(&db->h_stage), cap);
    if (st != SWB_OK) return st;
    db->stage_cap = cap;
    return SWB_OK;
}

template <class T>
swb_status ensure_dev(T** ptr, size_t* cap, size_t need, uint64_t* tally) {
    if (need <= *cap) return SWB_OK;
    if (*ptr) {
        dev_free(*ptr);
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

#include "plan.inl"
#include "handle.inl"
#include "scan.inl"
#include "duo.inl"

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

#include "persist.inl"

void swb_db_destroy(swb_db* db) {
    if (!db) return;
    {
        DeviceGuard guard(db->device);
        if (db->own_stream) cudaStreamSynchronize(db->own_stream);
        if (db->side_stream) cudaStreamSynchronize(db->side_stream);
        void* ptrs[] = {db->d_codes,      db->d_groups,   db->d_slot_index, db->d_slot_len,    db->d_border0,
                        db->d_border1,    db->d_iborder0, db->d_iborder1, db->d_multi_scores, db->d_multi_codes, db->d_duo_tiles, db->d_prof2, db->d_duo_progress,   db->d_slot_scores, db->d_flag_list,
                        db->d_counters,   db->d_unit_start, db->d_group_mode, db->d_vstate_off, db->d_vstate, db->d_progress, db->d_nlinks, db->d_keys,        db->d_sel[0],
                        db->d_sel[1],     db->d_sort,     db->d_all_scores, db->d_query,       db->d_matrix,
                        db->d_prof8,      db->d_prof8i,   db->d_prof32i};
        // (both streams are idle: blocks of the ad-hoc entry points' cache can go straight back to it)
        for (void* p : ptrs)
            if (p) dev_free(p, true);
        host_free(db->h_stage, true);
        host_free(db->h_counters, true);
        host_free(db->h_merge, true);
        for (auto& ev : db->ev)
            if (ev) cudaEventDestroy(ev);
        for (auto& ev : db->many_events) cudaEventDestroy(ev);
        if (db->own_stream) cudaStreamDestroy(db->own_stream);
        if (db->side_stream) cudaStreamDestroy(db->side_stream);
        if (db->ev_fork) cudaEventDestroy(db->ev_fork);
        if (db->ev_join) cudaEventDestroy(db->ev_join);
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
    info->kernel_launches_total = db->launches_total + db->launches;
    return SWB_OK;
}

swb_status swb_db_set_scan_policy(swb_db* db, int32_t policy) {
    if (!db) return fail(SWB_ERR_INVALID, "db is null");
    if (policy < SWB_SCAN_AUTO || policy > SWB_SCAN_WAVEFRONT) return fail(SWB_ERR_INVALID, "unknown scan policy");
    std::lock_guard<std::mutex> lock(db->mu);
    db->scan_policy = policy;
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

swb_status swb_search_keys_device(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                                  int32_t gap_open, int32_t gap_extend, uint32_t top_k, uint64_t* device_keys_out) {
    if (!db) return fail(SWB_ERR_INVALID, "db is null");
    if (top_k < 1) return fail(SWB_ERR_INVALID, "top_k must be >= 1");
    if (!device_keys_out) return fail(SWB_ERR_INVALID, "device_keys_out is null");
    swb_status st = check_scoring_args(query, query_len, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    const uint64_t n_keys = db->meta.n_local;
    const uint32_t k_eff = static_cast<uint32_t>(std::min<uint64_t>(top_k, std::max<uint64_t>(n_keys, 1)));
    const uint64_t* d_top = nullptr;
    st = search_keys_locked(db, query, query_len, matrix, gap_open, gap_extend, k_eff, &d_top);
    if (st != SWB_OK) return st;
    cudaStream_t s = db->stream;
    if (k_eff < top_k) SWB_CUDA(cudaMemsetAsync(device_keys_out, 0, static_cast<size_t>(top_k) * sizeof(uint64_t), s));
    SWB_CUDA(cudaMemcpyAsync(device_keys_out, d_top, static_cast<size_t>(k_eff) * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    SWB_CUDA(cudaMemcpyAsync(db->h_counters, db->d_counters, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SWB_CUDA(cudaEventRecord(db->ev[EV_END], s));
    db->async_pending = true;
    return SWB_OK;
}

swb_status swb_db_merge_keys(swb_db* db, const uint64_t* device_keys, uint64_t n, uint32_t top_k, swb_hit* hits,
                             uint32_t* n_hits, uint32_t query_len, swb_stats* stats) {
    if (!db) return fail(SWB_ERR_INVALID, "db is null");
    if (!hits || !n_hits) return fail(SWB_ERR_INVALID, "hits/n_hits are null");
    if (top_k < 1) return fail(SWB_ERR_INVALID, "top_k must be >= 1");
    if (n && !device_keys) return fail(SWB_ERR_INVALID, "device_keys is null");
    *n_hits = 0;
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    cudaStream_t s = db->stream;
    const uint32_t k_eff = static_cast<uint32_t>(std::min<uint64_t>(top_k, n));
    // the keys come down next to, not over, the pending search's inputs: a second pinned buffer of their own
    if (k_eff > db->merge_cap) {
        host_free(db->h_merge);
        db->h_merge = nullptr, db->merge_cap = 0;
        swb_status hst = host_alloc(reinterpret_cast<void**>(&db->h_merge), static_cast<size_t>(k_eff) * 2 * sizeof(uint64_t));
        if (hst != SWB_OK) return hst;
        db->merge_cap = k_eff * 2;
    }
    if (k_eff) {
        const uint64_t* d_top = nullptr;
        const uint32_t launches_before = db->launches;
        swb_status st = select_topk(db, device_keys, n, k_eff, &d_top);
        if (st != SWB_OK) return st;
        db->launches = launches_before;   // the merge's launches are not the search's
        db->launches_total += 1;
        SWB_CUDA(cudaMemcpyAsync(db->h_merge, d_top, static_cast<size_t>(k_eff) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    }
    SWB_CUDA(cudaStreamSynchronize(s));
    db->async_pending = false;
    uint32_t cnt = 0;
    for (uint32_t i = 0; i < k_eff && db->h_merge[i]; ++i, ++cnt) {
        hits[cnt].db_index = 0xFFFFFFFFu - static_cast<uint32_t>(db->h_merge[i] & 0xFFFFFFFFu);
        hits[cnt].score = static_cast<int32_t>(db->h_merge[i] >> 32);
    }
    *n_hits = cnt;
    fill_stats(db, query_len, stats);
    return SWB_OK;
}

// All scores of two queries from one scan, before any int32 re-run (tests/manual/duo_experiment.py: kernel parity and timing).
swb_status swb_score_all_duo(swb_db* db, const uint8_t* qa, uint32_t ma, const uint8_t* qb, uint32_t mb, const int32_t* matrix,
                             int32_t gap_open, int32_t gap_extend, int32_t* scores_a, int32_t* scores_b, swb_stats* stats) {
    if (!db || !scores_a || !scores_b) return fail(SWB_ERR_INVALID, "null argument");
    swb_status st = check_scoring_args(qa, ma, matrix, gap_open, gap_extend);
    if (st == SWB_OK) st = check_scoring_args(qb, mb, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    if (ma == 0 || mb == 0) return fail(SWB_ERR_INVALID, "empty query");
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    const QueryPlan pl = make_plan(db, std::max(ma, mb), matrix, gap_open, gap_extend);
    if (pl.main != kMainS16) return fail(SWB_ERR_UNSUPPORTED, "the shared scan needs the packed int16 path");
    const uint8_t* two[2] = {qa, qb};
    const uint32_t two_len[2] = {ma, mb};
    DuoScan scan;
    scan.a = {0};
    scan.b = {1};
    scan.tiles_a = tiles_of(ma);
    scan.tiles_b = tiles_of(mb);
    std::vector<uint32_t> order, code_off;
    st = score_streams_core(db, two, two_len, scan, matrix, gap_open, gap_extend, order, code_off);
    if (st != SWB_OK) return st;
    cudaStream_t s = db->stream;
    const uint32_t n_total = db->meta.n_total;
    if (!db->d_all_scores)
        if ((st = dev_alloc(&db->d_all_scores, n_total, &db->device_bytes)) != SWB_OK) return st;
    const unsigned blocks = std::max(1u, std::min(1024u, (db->n_slots + 255) / 256));
    int32_t* outs[2] = {scores_a, scores_b};
    for (int q = 0; q < 2; ++q) {
        SWB_CUDA(cudaMemcpyAsync(db->d_all_scores, outs[q], static_cast<size_t>(n_total) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        if (db->n_slots)
            scatter_scores_kernel<<<blocks, 256, 0, s>>>(db->d_multi_scores + static_cast<size_t>(q) * db->n_slots, db->d_slot_index,
                                                          db->n_slots, db->d_all_scores);
        SWB_CUDA(cudaMemcpyAsync(outs[q], db->d_all_scores, static_cast<size_t>(n_total) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    }
    SWB_CUDA(cudaEventRecord(db->ev[EV_TOPK], s));
    SWB_CUDA(cudaEventRecord(db->ev[EV_END], s));
    SWB_CUDA(cudaStreamSynchronize(s));
    fill_stats(db, ma + mb, stats);
    return SWB_OK;
}

swb_status swb_search_many(swb_db* db, const uint8_t* const* queries, const uint32_t* query_lens, uint32_t n_queries,
                           const int32_t* matrix, int32_t gap_open, int32_t gap_extend, uint32_t top_k, swb_hit* hits,
                           uint32_t* n_hits, float* ms_per_query) {
    if (!db) return fail(SWB_ERR_INVALID, "db is null");
    if (top_k < 1) return fail(SWB_ERR_INVALID, "top_k must be >= 1");
    if (n_queries && (!queries || !query_lens || !hits || !n_hits)) return fail(SWB_ERR_INVALID, "null argument");
    swb_status st;
    for (uint32_t q = 0; q < n_queries; ++q)
        if ((st = check_scoring_args(queries[q], query_lens[q], matrix, gap_open, gap_extend)) != SWB_OK) return st;
    if (n_queries == 0) return SWB_OK;
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    cudaStream_t s = db->stream;
    const uint64_t n_keys = db->meta.n_local;
    const uint32_t k_eff = static_cast<uint32_t>(std::min<uint64_t>(top_k, std::max<uint64_t>(n_keys, 1)));
    const size_t n_groups = db->meta.groups.size();

    // Queries share database scans where that pays (duo.inl): the rest go one by one.
    struct Job {
        int scan;        // >= 0: shared scan number; -1: a single-query scan of `query`
        uint32_t query;
    };
    std::vector<DuoScan> scans;
    std::vector<uint32_t> single;
    plan_batch(scan_knobs(), duo_mode(db, matrix, gap_open, gap_extend), query_lens, n_queries, scans, single);
    std::vector<Job> jobs;
    for (size_t i = 0; i < scans.size(); ++i) jobs.push_back(Job{static_cast<int>(i), 0});
    for (uint32_t q : single) jobs.push_back(Job{-1, q});

    // one staging area per job (inputs up) and per query (keys down), sized up front: the pinned buffer must not
    // move while copies are in flight
    std::vector<size_t> in_off(jobs.size()), out_off(n_queries);
    size_t total = 0;
    for (size_t j = 0; j < jobs.size(); ++j) {
        in_off[j] = total;
        size_t need = 576 * sizeof(int32_t) + 256 + (n_groups + 1) * 9;
        if (jobs[j].scan >= 0) {
            const DuoScan& sc = scans[jobs[j].scan];
            for (uint32_t q : sc.a) need += (query_lens[q] + 15) & ~15u;
            for (uint32_t q : sc.b) need += (query_lens[q] + 15) & ~15u;
            need += static_cast<size_t>(std::max(sc.tiles_a, sc.tiles_b)) * sizeof(DuoTile);
        } else {
            need += query_lens[jobs[j].query];
        }
        total += (need + 255) & ~size_t(255);
    }
    for (uint32_t q = 0; q < n_queries; ++q) {
        out_off[q] = total;
        total += (static_cast<size_t>(k_eff) * sizeof(uint64_t) + 16 + 255) & ~size_t(255);
    }
    if ((st = ensure_stage(db, total)) != SWB_OK) return st;
    while (db->many_events.size() < 2 * jobs.size()) {
        cudaEvent_t ev;
        SWB_CUDA(cudaEventCreate(&ev));
        db->many_events.push_back(ev);
    }
    auto keys_down = [&](uint32_t q, const uint64_t* d_top) {
        if (cudaMemcpyAsync(db->h_stage + out_off[q], d_top, static_cast<size_t>(k_eff) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s) !=
            cudaSuccess)
            st = fail(SWB_ERR_CUDA, "cudaMemcpyAsync failed");
    };
    // jobs are issued back to back on the stream: the host prepares the next one (unit table, launches) while the
    // GPU still scans, and nothing synchronises until the last one is in flight
    std::vector<uint32_t> scan_queries, code_off;
    for (size_t j = 0; j < jobs.size() && st == SWB_OK; ++j) {
        db->stage_base = in_off[j];
        cudaEventRecord(db->many_events[2 * j], s);
        const uint64_t* d_top = nullptr;
        if (jobs[j].scan < 0) {
            const uint32_t q = jobs[j].query;
            st = search_keys_locked(db, queries[q], query_lens[q], matrix, gap_open, gap_extend, k_eff, &d_top);
            if (st == SWB_OK) keys_down(q, d_top);
        } else {
            st = score_streams_core(db, queries, query_lens, scans[jobs[j].scan], matrix, gap_open, gap_extend, scan_queries, code_off);
            for (size_t i = 0; i < scan_queries.size() && st == SWB_OK; ++i) {
                const uint32_t q = scan_queries[i];
                st = finish_duo_query(db, db->d_multi_codes + code_off[i], query_lens[q], matrix, gap_open, gap_extend,
                                      db->d_multi_scores + i * static_cast<size_t>(db->n_slots), k_eff, &d_top);
                if (st == SWB_OK) keys_down(q, d_top);
            }
        }
        cudaEventRecord(db->many_events[2 * j + 1], s);
    }
    db->stage_base = 0;
    const cudaError_t sync = cudaStreamSynchronize(s);
    if (st != SWB_OK) return st;
    if (sync != cudaSuccess) return fail(SWB_ERR_CUDA, cudaGetErrorString(sync));
    for (uint32_t q = 0; q < n_queries; ++q) {
        const uint64_t* keys = reinterpret_cast<const uint64_t*>(db->h_stage + out_off[q]);
        uint32_t cnt = 0;
        for (uint32_t i = 0; i < k_eff && keys[i]; ++i, ++cnt) {
            hits[static_cast<size_t>(q) * top_k + cnt].db_index = 0xFFFFFFFFu - static_cast<uint32_t>(keys[i] & 0xFFFFFFFFu);
            hits[static_cast<size_t>(q) * top_k + cnt].score = static_cast<int32_t>(keys[i] >> 32);
        }
        n_hits[q] = cnt;
    }
    if (ms_per_query)
        for (size_t j = 0; j < jobs.size(); ++j) {
            // a shared scan's time is split between its queries in proportion to their lengths
            float ms = 0.f;
            cudaEventElapsedTime(&ms, db->many_events[2 * j], db->many_events[2 * j + 1]);
            if (jobs[j].scan < 0) {
                ms_per_query[jobs[j].query] = ms;
                continue;
            }
            const DuoScan& sc = scans[jobs[j].scan];
            double columns = 0.0;
            for (uint32_t q : sc.a) columns += query_lens[q];
            for (uint32_t q : sc.b) columns += query_lens[q];
            for (const std::vector<uint32_t>* stream : {&sc.a, &sc.b})
                for (uint32_t q : *stream) ms_per_query[q] = static_cast<float>(ms * query_lens[q] / std::max(columns, 1.0));
        }
    return SWB_OK;
}

// The scores behind swb_search_many: the batch goes through the same plan (shared scans of two streams where they
// apply, single scans for the rest) and the same kernels, and every query's whole score vector comes back in
// database order -- what the parity tests compare with the oracle (scheduler.hpp:179-183: "sequential scalar scan").
swb_status swb_score_many(swb_db* db, const uint8_t* const* queries, const uint32_t* query_lens, uint32_t n_queries,
                          const int32_t* matrix, int32_t gap_open, int32_t gap_extend, int32_t* scores, int32_t* scan_of_query,
                          uint32_t* rescored_i32) {
    if (!db) return fail(SWB_ERR_INVALID, "db is null");
    if (n_queries && (!queries || !query_lens || !scores)) return fail(SWB_ERR_INVALID, "null argument");
    swb_status st;
    for (uint32_t q = 0; q < n_queries; ++q)
        if ((st = check_scoring_args(queries[q], query_lens[q], matrix, gap_open, gap_extend)) != SWB_OK) return st;
    if (n_queries == 0) return SWB_OK;
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    cudaStream_t s = db->stream;
    const size_t n_groups = db->meta.groups.size();
    const uint32_t n_total = db->meta.n_total;
    std::vector<DuoScan> scans;
    std::vector<uint32_t> single;
    plan_batch(scan_knobs(), duo_mode(db, matrix, gap_open, gap_extend), query_lens, n_queries, scans, single);
    size_t stage = 576 * sizeof(int32_t) + 256 + (n_groups + 1) * 9;
    uint32_t longest = 0;
    for (uint32_t q = 0; q < n_queries; ++q) longest = std::max(longest, query_lens[q]);
    stage += longest;
    for (const DuoScan& sc : scans) {
        size_t need = 576 * sizeof(int32_t) + 256 + static_cast<size_t>(std::max(sc.tiles_a, sc.tiles_b)) * sizeof(DuoTile);
        for (uint32_t q : sc.a) need += (query_lens[q] + 15) & ~15u;
        for (uint32_t q : sc.b) need += (query_lens[q] + 15) & ~15u;
        stage = std::max(stage, need);
    }
    if ((st = ensure_stage(db, stage)) != SWB_OK) return st;
    if (!db->d_all_scores)
        if ((st = dev_alloc(&db->d_all_scores, n_total, &db->device_bytes)) != SWB_OK) return st;
    const unsigned blocks = std::max(1u, std::min(1024u, (db->n_slots + 255) / 256));
    // one query's slot scores -> database order -> the caller's row (entries of other shards stay as they were)
    auto deliver = [&](uint32_t q, const int32_t* slot_scores) -> swb_status {
        int32_t* row = scores + static_cast<size_t>(q) * n_total;
        SWB_CUDA(cudaMemcpyAsync(db->d_all_scores, row, static_cast<size_t>(n_total) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        if (db->n_slots) {
            scatter_scores_kernel<<<blocks, 256, 0, s>>>(slot_scores, db->d_slot_index, db->n_slots, db->d_all_scores);
            ++db->launches;
        }
        SWB_CUDA(cudaMemcpyAsync(row, db->d_all_scores, static_cast<size_t>(n_total) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SWB_CUDA(cudaMemcpyAsync(db->h_counters, db->d_counters, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SWB_CUDA(cudaStreamSynchronize(s));   // the staging area is reused by the next job
        if (rescored_i32) rescored_i32[q] = db->h_counters[1];
        return SWB_OK;
    };
    std::vector<uint32_t> scan_queries, code_off;
    for (size_t i = 0; i < scans.size(); ++i) {
        if ((st = score_streams_core(db, queries, query_lens, scans[i], matrix, gap_open, gap_extend, scan_queries, code_off)) != SWB_OK)
            return st;
        for (size_t j = 0; j < scan_queries.size(); ++j) {
            const uint32_t q = scan_queries[j];
            int32_t* slot_scores = db->d_multi_scores + j * static_cast<size_t>(db->n_slots);
            SWB_CUDA(cudaMemsetAsync(db->d_counters + 1, 0, sizeof(uint32_t), s));
            if ((st = rescore_duo_query(db, db->d_multi_codes + code_off[j], query_lens[q], matrix, gap_open, gap_extend, slot_scores)) != SWB_OK)
                return st;
            if ((st = deliver(q, slot_scores)) != SWB_OK) return st;
            if (scan_of_query) scan_of_query[q] = static_cast<int32_t>(i);
        }
    }
    for (uint32_t q : single) {
        if ((st = score_core(db, queries[q], query_lens[q], matrix, gap_open, gap_extend)) != SWB_OK) return st;
        if ((st = deliver(q, db->d_slot_scores)) != SWB_OK) return st;
        if (scan_of_query) scan_of_query[q] = -1;
    }
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

#include "pairs.inl"

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

swb_status swb_scan_plan(const uint32_t* lens, uint32_t n, uint64_t length_threshold, uint32_t shard_rank,
                         uint32_t shard_count, uint32_t query_len, uint32_t sm_count, int32_t policy,
                         swb_scan_plan_info* out) {
    if (!out || (n && !lens)) return fail(SWB_ERR_INVALID, "null argument");
    if (shard_count < 1 || shard_rank >= shard_count) return fail(SWB_ERR_INVALID, "shard_rank must be < shard_count");
    if (sm_count < 1) return fail(SWB_ERR_INVALID, "sm_count must be >= 1");
    if (policy < SWB_SCAN_AUTO || policy > SWB_SCAN_WAVEFRONT) return fail(SWB_ERR_INVALID, "unknown scan policy");
    std::memset(out, 0, sizeof(*out));
    SeqSource src;
    static const uint32_t kNoLens[1] = {0};
    src.lens = n ? lens : kNoLens;
    src.n = n;
    std::vector<GroupDesc> groups;
    uint64_t padded_rows = 0;
    group_table(src, length_threshold, shard_rank, shard_count, groups, &padded_rows);
    const uint32_t n_groups = static_cast<uint32_t>(groups.size());
    out->n_groups = n_groups;
    if (query_len == 0 || n_groups == 0) return SWB_OK;
    constexpr size_t kSmemOptinB200 = 227 * 1024;
    ScanShape shape;
    shape.groups = groups.data();
    shape.n_groups = n_groups;
    shape.padded_rows = padded_rows;
    shape.n_tiles = (query_len + kInterTile - 1) / kInterTile;
    shape.query_len = query_len;
    {
        const size_t prof_bytes = static_cast<size_t>(kProfRows) * profile_stride(query_len, kInterTile);
        const size_t used = ((prof_bytes + 127) & ~size_t(127)) + 1024;
        shape.narrow_room = used < kSmemOptinB200 ? kSmemOptinB200 - used : 0;
    }
    shape.sm_count = sm_count;
    shape.warps_per_cta = kInterThreads / 32;
    shape.policy = policy;
    shape.pipe_rings = pipe_rings_for(static_cast<size_t>(kProfRows) * profile_stride(query_len, kInterTile), kSmemOptinB200,
                                      sizeof(PipeCtl), static_cast<size_t>(kPipeWarps) * kPipeChunkBytes, scan_knobs().pipe_ring_cap).chunks;
    std::vector<uint32_t> us(static_cast<size_t>(n_groups) + 1), vso(n_groups);
    std::vector<uint8_t> modes(n_groups);
    const ScanPlan sp = plan_scan(shape, scan_knobs(), us.data(), vso.data(), modes.data());
    out->n_tiles = shape.n_tiles;
    out->pipeline_groups = n_groups - sp.pipe_first;
    out->wavefront_groups = sp.pipe_first;
    out->wavefront_sms = sp.wave_sms;
    out->wavefront_units = sp.n_units;
    out->split_groups = sp.n_split;
    out->narrow_groups = sp.n_narrow;
    out->rowblock_groups = sp.n_rowblock;
    out->ring_chunks = shape.pipe_rings;
    out->chain_bound = sp.chain_bound ? 1 : 0;
    out->narrow_tile = sp.narrow_tile;
    out->wavefront_threads = sp.wave_threads;
    out->narrow_link_bytes = sp.link_rows * 256;
    out->wavefront_rows = sp.wave_rows;
    out->pipeline_rows = padded_rows - sp.wave_rows;
    return SWB_OK;
}

swb_status swb_batch_plan(const uint32_t* lens, uint32_t n, uint64_t length_threshold, uint32_t shard_rank, uint32_t shard_count,
                          const uint32_t* query_lens, uint32_t n_queries, uint32_t sm_count, int32_t* scan_of_query,
                          int32_t* stream_of_query) {
    if ((n && !lens) || (n_queries && (!query_lens || !scan_of_query || !stream_of_query))) return fail(SWB_ERR_INVALID, "null argument");
    if (shard_count < 1 || shard_rank >= shard_count) return fail(SWB_ERR_INVALID, "shard_rank must be < shard_count");
    if (sm_count < 1) return fail(SWB_ERR_INVALID, "sm_count must be >= 1");
    SeqSource src;
    static const uint32_t kNoLens[1] = {0};
    src.lens = n ? lens : kNoLens;
    src.n = n;
    std::vector<GroupDesc> groups;
    uint64_t padded_rows = 0;
    group_table(src, length_threshold, shard_rank, shard_count, groups, &padded_rows);
    const uint32_t max_rows = groups.empty() ? 0 : groups[0].n_chunks * kRowsPerChunk;
    const SharedScanMode enabled = shared_scan_mode(scan_knobs(), static_cast<uint32_t>(groups.size()), max_rows, padded_rows, sm_count);
    std::vector<DuoScan> scans;
    std::vector<uint32_t> single;
    plan_batch(scan_knobs(), enabled, query_lens, n_queries, scans, single);
    for (uint32_t q : single) scan_of_query[q] = -1, stream_of_query[q] = -1;
    for (size_t i = 0; i < scans.size(); ++i) {
        for (uint32_t q : scans[i].a) scan_of_query[q] = static_cast<int32_t>(i), stream_of_query[q] = 0;
        for (uint32_t q : scans[i].b) scan_of_query[q] = static_cast<int32_t>(i), stream_of_query[q] = 1;
    }
    return SWB_OK;
}

}  // extern "C"

#include "pipe.inl"
#include "multi.inl"
