// multi.inl -- several GPUs of one box driven from one process (included by cabi.cu).
//
// The database is dealt over the devices by residue count (pack.hpp: snake deal of the
// length-sorted pools).  A search runs every shard concurrently (one host thread per shard, each
// on its shard's own stream), each producing its top-k as packed keys on its device.  The only
// exchange is k x 8 bytes per shard: one ncclAllGather over NVLink (ncclCommInitAll communicator,
// grouped call), after which shard 0 selects the global top-k from the G x k gathered keys.
// NCCL is loaded with dlopen only when two or more distinct devices are used, so a single-GPU
// process never needs it.  Shards that share a device (used to exercise the sharding logic on a
// one-GPU box) cannot form an NCCL communicator (NCCL rejects duplicate devices), so their keys
// are gathered with device-to-device copies on that device instead.

namespace {

struct NcclApi {
    void* handle = nullptr;
    int (*CommInitAll)(void**, int, const int*) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;

    bool load(std::string* why) {
        if (handle) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            handle = dlopen(name, RTLD_NOW | RTLD_LOCAL);
            if (handle) break;
        }
        if (!handle) {
            *why = std::string("cannot load libnccl: ") + dlerror();
            return false;
        }
        CommInitAll = reinterpret_cast<decltype(CommInitAll)>(dlsym(handle, "ncclCommInitAll"));
        CommDestroy = reinterpret_cast<decltype(CommDestroy)>(dlsym(handle, "ncclCommDestroy"));
        GroupStart = reinterpret_cast<decltype(GroupStart)>(dlsym(handle, "ncclGroupStart"));
        GroupEnd = reinterpret_cast<decltype(GroupEnd)>(dlsym(handle, "ncclGroupEnd"));
        AllGather = reinterpret_cast<decltype(AllGather)>(dlsym(handle, "ncclAllGather"));
        GetErrorString = reinterpret_cast<decltype(GetErrorString)>(dlsym(handle, "ncclGetErrorString"));
        if (!CommInitAll || !CommDestroy || !GroupStart || !GroupEnd || !AllGather || !GetErrorString) {
            *why = "libnccl is missing a required symbol";
            return false;
        }
        return true;
    }
};

constexpr int kNcclUint64 = 5;   // ncclUint64 (nccl.h)

// One persistent host thread per shard: a search hands every worker its shard's job and waits for all of them,
// instead of creating and joining G threads per call (the reference does the latter, scheduler.hpp:218-229).
class ShardPool {
public:
    explicit ShardPool(size_t n) : jobs_(n), busy_(n, false) {
        for (size_t r = 0; r < n; ++r) threads_.emplace_back([this, r] { loop(r); });
    }
    ~ShardPool() {
        {
            std::lock_guard<std::mutex> lock(mu_);
            stop_ = true;
        }
        wake_.notify_all();
        for (auto& t : threads_) t.join();
    }
    // fn(r) on worker r for every r, concurrently; returns when all are done
    void run(const std::function<void(size_t)>& fn) {
        {
            std::lock_guard<std::mutex> lock(mu_);
            for (size_t r = 0; r < jobs_.size(); ++r) jobs_[r] = &fn, busy_[r] = true;
            pending_ = jobs_.size();
        }
        wake_.notify_all();
        std::unique_lock<std::mutex> lock(mu_);
        done_.wait(lock, [this] { return pending_ == 0; });
    }

private:
    void loop(size_t r) {
        for (;;) {
            const std::function<void(size_t)>* job = nullptr;
            {
                std::unique_lock<std::mutex> lock(mu_);
                wake_.wait(lock, [&] { return stop_ || busy_[r]; });
                if (stop_) return;
                job = jobs_[r];
            }
            (*job)(r);
            {
                std::lock_guard<std::mutex> lock(mu_);
                busy_[r] = false;
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    std::mutex mu_;
    std::condition_variable wake_, done_;
    std::vector<const std::function<void(size_t)>*> jobs_;
    std::vector<bool> busy_;
    size_t pending_ = 0;
    bool stop_ = false;
    std::vector<std::thread> threads_;
};

}  // namespace

struct swb_mdb {
    std::vector<swb_db*> shards;
    std::vector<int> devices;
    bool distinct = true;
    NcclApi nccl;
    std::vector<void*> comms;
    std::vector<uint64_t*> d_gather;   // per shard: G * k_cap keys on that shard's device
    std::vector<uint64_t*> d_send;     // per shard: k_cap keys
    uint32_t k_cap = 0;
    std::unique_ptr<ShardPool> pool;   // one worker per shard, created with the first multi-shard search
    std::mutex mu;
};

namespace {

swb_status mdb_build(const SeqSource& src, uint64_t threshold, const int32_t* devices, uint32_t n_devices,
                     swb_mdb** out) {
    if (!out) return fail(SWB_ERR_INVALID, "out is null");
    *out = nullptr;
    if (n_devices < 1 || !devices) return fail(SWB_ERR_INVALID, "at least one device is required");
    auto* mdb = new swb_mdb();
    mdb->devices.assign(devices, devices + n_devices);
    std::vector<int> sorted(mdb->devices);
    std::sort(sorted.begin(), sorted.end());
    mdb->distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    mdb->shards.assign(n_devices, nullptr);

    // pack + upload the shards concurrently (each on its own device)
    std::vector<swb_status> sts(n_devices, SWB_OK);
    std::vector<std::string> errs(n_devices);
    std::vector<std::thread> pool;
    for (uint32_t r = 0; r < n_devices; ++r)
        pool.emplace_back([&, r] {
            sts[r] = create_from(src, threshold, devices[r], r, n_devices, &mdb->shards[r]);
            if (sts[r] != SWB_OK) errs[r] = g_error;
        });
    for (auto& t : pool) t.join();
    for (uint32_t r = 0; r < n_devices; ++r)
        if (sts[r] != SWB_OK) {
            const swb_status st = sts[r];
            const std::string msg = errs[r];
            swb_mdb_destroy(mdb);
            return fail(st, msg);
        }

    // SWB200_FORCE_NCCL=1: a communicator even for one device, so that the NCCL branch (dlopen, ncclCommInitAll, the grouped
    // all-gather on the shards' streams) can be exercised on a box with a single GPU
    static const bool force_nccl = [] {
        const char* e = std::getenv("SWB200_FORCE_NCCL");
        return e && *e == '1';
    }();
    if ((n_devices > 1 || force_nccl) && mdb->distinct) {
        std::string why;
        if (!mdb->nccl.load(&why)) {
            swb_mdb_destroy(mdb);
            return fail(SWB_ERR_NCCL, why);
        }
        mdb->comms.assign(n_devices, nullptr);
        const int rc = mdb->nccl.CommInitAll(mdb->comms.data(), static_cast<int>(n_devices), mdb->devices.data());
        if (rc != 0) {
            const std::string msg = std::string("ncclCommInitAll: ") + mdb->nccl.GetErrorString(rc);
            mdb->comms.clear();
            swb_mdb_destroy(mdb);
            return fail(SWB_ERR_NCCL, msg);
        }
    }
    *out = mdb;
    return SWB_OK;
}

swb_status mdb_ensure_buffers(swb_mdb* mdb, uint32_t k) {
    if (k <= mdb->k_cap) return SWB_OK;
    const size_t G = mdb->shards.size();
    for (size_t r = 0; r < mdb->d_gather.size(); ++r) {
        DeviceGuard guard(mdb->devices[r]);
        if (mdb->d_gather[r]) cudaFree(mdb->d_gather[r]);
        if (mdb->d_send[r]) cudaFree(mdb->d_send[r]);
    }
    mdb->d_gather.assign(G, nullptr);
    mdb->d_send.assign(G, nullptr);
    mdb->k_cap = 0;
    for (size_t r = 0; r < G; ++r) {
        DeviceGuard guard(mdb->devices[r]);
        SWB_CUDA(cudaMalloc(reinterpret_cast<void**>(&mdb->d_gather[r]), G * k * sizeof(uint64_t)));
        SWB_CUDA(cudaMalloc(reinterpret_cast<void**>(&mdb->d_send[r]), static_cast<size_t>(k) * sizeof(uint64_t)));
    }
    mdb->k_cap = k;
    return SWB_OK;
}

}  // namespace

extern "C" {

swb_status swb_mdb_create_flat(const uint8_t* codes, const uint64_t* offsets, uint32_t n, uint64_t length_threshold,
                               const int32_t* devices, uint32_t n_devices, swb_mdb** out) {
    if (!offsets) return fail(SWB_ERR_INVALID, "offsets is null");
    for (uint32_t i = 0; i < n; ++i)
        if (offsets[i + 1] < offsets[i]) return fail(SWB_ERR_INVALID, "offsets must be non-decreasing");
    SeqSource src;
    src.flat = codes;
    src.offsets = offsets;
    src.n = n;
    return mdb_build(src, length_threshold, devices, n_devices, out);
}

swb_status swb_mdb_create(const uint8_t* const* seqs, const uint32_t* lens, uint32_t n, uint64_t length_threshold,
                          const int32_t* devices, uint32_t n_devices, swb_mdb** out) {
    if (n && (!seqs || !lens)) return fail(SWB_ERR_INVALID, "seqs/lens are null");
    static const uint8_t* const kNoPtrs[1] = {nullptr};
    static const uint32_t kNoLens[1] = {0};
    SeqSource src;
    src.ptrs = n ? seqs : kNoPtrs;
    src.lens = n ? lens : kNoLens;
    src.n = n;
    return mdb_build(src, length_threshold, devices, n_devices, out);
}

// A packed file (swb_pack_file / swb_db_save, one shard holding the whole database) as a one-device swb_mdb, so that
// the drop-in's run_search can start from the file instead of parsing and packing (fasta.hpp:80-86).
swb_status swb_mdb_load(const char* path, int32_t device, swb_mdb** out) {
    if (!out) return fail(SWB_ERR_INVALID, "out is null");
    *out = nullptr;
    swb_db* db = nullptr;
    const swb_status st = swb_db_load(path, device, &db);
    if (st != SWB_OK) return st;
    if (db->meta.shard_count != 1) {
        swb_db_destroy(db);
        return fail(SWB_ERR_INVALID, std::string(path) + " holds one shard of several; swb_mdb_load needs an unsharded file");
    }
    auto* mdb = new swb_mdb();
    mdb->devices.assign(1, device);
    mdb->shards.assign(1, db);
    *out = mdb;
    return SWB_OK;
}

void swb_mdb_destroy(swb_mdb* mdb) {
    if (!mdb) return;
    for (size_t r = 0; r < mdb->comms.size(); ++r)
        if (mdb->comms[r]) mdb->nccl.CommDestroy(mdb->comms[r]);
    for (size_t r = 0; r < mdb->d_gather.size(); ++r) {
        DeviceGuard guard(mdb->devices[r]);
        if (mdb->d_gather[r]) cudaFree(mdb->d_gather[r]);
        if (mdb->d_send[r]) cudaFree(mdb->d_send[r]);
    }
    for (swb_db* db : mdb->shards) swb_db_destroy(db);
    delete mdb;
}

swb_status swb_mdb_align_hits(swb_mdb* mdb, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                              int32_t gap_open, int32_t gap_extend, const swb_hit* hits, uint32_t n_hits,
                              uint64_t memory_cap, swb_alignment* out, uint8_t* ops, const uint64_t* ops_offset) {
    if (!mdb) return fail(SWB_ERR_INVALID, "mdb is null");
    if (n_hits && (!hits || !out || !ops_offset)) return fail(SWB_ERR_INVALID, "null argument");
    const size_t G = mdb->shards.size();
    if (G == 1)
        return swb_db_align_hits(mdb->shards[0], query, query_len, matrix, gap_open, gap_extend, hits, n_hits, memory_cap,
                                 out, ops, ops_offset);
    // route every hit to the shard that holds it
    for (size_t r = 0; r < G; ++r) {
        swb_db* db = mdb->shards[r];
        {
            std::lock_guard<std::mutex> lock(db->mu);
            if (db->slot_of.empty() && db->meta.n_total) {
                db->slot_of.assign(db->meta.n_total, kNoSequence);
                for (uint32_t slot = 0; slot < db->meta.slot_index.size(); ++slot)
                    if (db->meta.slot_index[slot] != kNoSequence) db->slot_of[db->meta.slot_index[slot]] = slot;
            }
        }
        std::vector<swb_hit> mine;
        std::vector<uint32_t> where;
        std::vector<uint64_t> offs(1, 0);
        for (uint32_t i = 0; i < n_hits; ++i) {
            if (hits[i].db_index < db->meta.n_total && db->slot_of[hits[i].db_index] != kNoSequence) {
                mine.push_back(hits[i]);
                where.push_back(i);
                offs.push_back(offs.back() + (ops_offset[i + 1] - ops_offset[i]));
            }
        }
        if (mine.empty()) continue;
        std::vector<swb_alignment> part(mine.size());
        std::vector<uint8_t> part_ops(std::max<uint64_t>(offs.back(), 1));
        const swb_status st = swb_db_align_hits(db, query, query_len, matrix, gap_open, gap_extend, mine.data(),
                                                static_cast<uint32_t>(mine.size()), memory_cap, part.data(),
                                                ops ? part_ops.data() : nullptr, offs.data());
        if (st != SWB_OK) return st;
        for (size_t j = 0; j < mine.size(); ++j) {
            out[where[j]] = part[j];
            if (ops) std::memcpy(ops + ops_offset[where[j]], part_ops.data() + offs[j], std::min<uint64_t>(part[j].n_ops, offs[j + 1] - offs[j]));
        }
    }
    return SWB_OK;
}

// A batch of queries on every shard at once (one host thread per shard, each running swb_search_many: shared scans
// where they apply), then a host-side merge per query: top-k of the union = top-k of the per-shard top-k's
// (scheduler.hpp:106-117; the order on packed keys is exactly (score desc, db_index asc)).  n_queries x k x G keys
// are a few kilobytes, so unlike the per-search path this needs no collective.
swb_status swb_mdb_search_many(swb_mdb* mdb, const uint8_t* const* queries, const uint32_t* query_lens, uint32_t n_queries,
                               const int32_t* matrix, int32_t gap_open, int32_t gap_extend, uint32_t top_k, swb_hit* hits,
                               uint32_t* n_hits, float* ms_per_query) {
    if (!mdb) return fail(SWB_ERR_INVALID, "mdb is null");
    if (top_k < 1) return fail(SWB_ERR_INVALID, "top_k must be >= 1");
    if (n_queries && (!queries || !query_lens || !hits || !n_hits)) return fail(SWB_ERR_INVALID, "null argument");
    const size_t G = mdb->shards.size();
    if (G == 1)
        return swb_search_many(mdb->shards[0], queries, query_lens, n_queries, matrix, gap_open, gap_extend, top_k, hits, n_hits,
                               ms_per_query);
    std::lock_guard<std::mutex> lock(mdb->mu);
    std::vector<swb_status> sts(G, SWB_OK);
    std::vector<std::string> errs(G);
    std::vector<std::vector<swb_hit>> shard_hits(G, std::vector<swb_hit>(static_cast<size_t>(n_queries) * top_k));
    std::vector<std::vector<uint32_t>> shard_counts(G, std::vector<uint32_t>(n_queries, 0));
    std::vector<std::vector<float>> shard_ms(G, std::vector<float>(n_queries, 0.f));
    if (!mdb->pool) mdb->pool.reset(new ShardPool(G));
    mdb->pool->run([&](size_t r) {
        sts[r] = swb_search_many(mdb->shards[r], queries, query_lens, n_queries, matrix, gap_open, gap_extend, top_k,
                                 shard_hits[r].data(), shard_counts[r].data(), shard_ms[r].data());
        if (sts[r] != SWB_OK) errs[r] = g_error;
    });
    for (size_t r = 0; r < G; ++r)
        if (sts[r] != SWB_OK) return fail(sts[r], "shard " + std::to_string(r) + ": " + errs[r]);
    std::vector<uint64_t> keys;
    for (uint32_t q = 0; q < n_queries; ++q) {
        keys.clear();
        for (size_t r = 0; r < G; ++r)
            for (uint32_t i = 0; i < shard_counts[r][q]; ++i) {
                const swb_hit& h = shard_hits[r][static_cast<size_t>(q) * top_k + i];
                keys.push_back((static_cast<uint64_t>(static_cast<uint32_t>(h.score)) << 32) | (0xFFFFFFFFu - h.db_index));
            }
        std::sort(keys.begin(), keys.end(), std::greater<uint64_t>());
        const uint32_t cnt = static_cast<uint32_t>(std::min<size_t>(keys.size(), top_k));
        for (uint32_t i = 0; i < cnt; ++i) {
            hits[static_cast<size_t>(q) * top_k + i].db_index = 0xFFFFFFFFu - static_cast<uint32_t>(keys[i] & 0xFFFFFFFFu);
            hits[static_cast<size_t>(q) * top_k + i].score = static_cast<int32_t>(keys[i] >> 32);
        }
        n_hits[q] = cnt;
        if (ms_per_query) {
            ms_per_query[q] = 0.f;
            for (size_t r = 0; r < G; ++r) ms_per_query[q] = std::max(ms_per_query[q], shard_ms[r][q]);   // shards run side by side
        }
    }
    return SWB_OK;
}

uint32_t swb_mdb_shard_count(const swb_mdb* mdb) { return mdb ? static_cast<uint32_t>(mdb->shards.size()) : 0; }

swb_db* swb_mdb_shard(swb_mdb* mdb, uint32_t i) {
    return (mdb && i < mdb->shards.size()) ? mdb->shards[i] : nullptr;
}

swb_status swb_mdb_search(swb_mdb* mdb, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                          int32_t gap_open, int32_t gap_extend, uint32_t top_k, swb_hit* hits, uint32_t* n_hits,
                          swb_stats* stats) {
    if (!mdb) return fail(SWB_ERR_INVALID, "mdb is null");
    if (!hits || !n_hits) return fail(SWB_ERR_INVALID, "hits/n_hits are null");
    if (top_k < 1) return fail(SWB_ERR_INVALID, "top_k must be >= 1");
    const size_t G = mdb->shards.size();
    if (G == 1 && mdb->comms.empty())
        return swb_search(mdb->shards[0], query, query_len, matrix, gap_open, gap_extend, top_k, hits, n_hits, stats);
    swb_status st = check_scoring_args(query, query_len, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;

    std::lock_guard<std::mutex> lock(mdb->mu);
    // no shard can contribute more than the whole database holds
    const uint32_t n_total = mdb->shards[0]->meta.n_total;
    const uint32_t k = static_cast<uint32_t>(std::min<uint64_t>(top_k, std::max<uint32_t>(n_total, 1)));
    if ((st = mdb_ensure_buffers(mdb, k)) != SWB_OK) return st;

    // 1. every shard enqueues its search on its own stream (one persistent worker per shard: the host-side preparation
    //    runs side by side); the k keys land in d_send on the shard's device, nothing synchronises yet
    std::vector<swb_status> sts(G, SWB_OK);
    std::vector<std::string> errs(G);
    if (!mdb->pool) mdb->pool.reset(new ShardPool(G));
    mdb->pool->run([&](size_t r) {
        sts[r] = swb_search_keys_device(mdb->shards[r], query, query_len, matrix, gap_open, gap_extend, k, mdb->d_send[r]);
        if (sts[r] != SWB_OK) errs[r] = g_error;
    });
    for (size_t r = 0; r < G; ++r)
        if (sts[r] != SWB_OK) return fail(sts[r], errs[r]);

    // 2. exchange: k keys per shard, enqueued behind each shard's search on its stream
    if (mdb->distinct) {
        int rc = mdb->nccl.GroupStart();
        for (size_t r = 0; r < G && rc == 0; ++r) {
            DeviceGuard guard(mdb->devices[r]);
            rc = mdb->nccl.AllGather(mdb->d_send[r], mdb->d_gather[r], k, kNcclUint64, mdb->comms[r], mdb->shards[r]->stream);
        }
        const int rc_end = mdb->nccl.GroupEnd();
        if (rc == 0) rc = rc_end;
        if (rc != 0) return fail(SWB_ERR_NCCL, std::string("ncclAllGather: ") + mdb->nccl.GetErrorString(rc));
    } else {
        // shards that share a device (tests on a one-GPU box): device-to-device copies on shard 0's stream, each
        // behind the event that ends its shard's search
        DeviceGuard guard(mdb->devices[0]);
        for (size_t r = 0; r < G; ++r) {
            if (r) SWB_CUDA(cudaStreamWaitEvent(mdb->shards[0]->stream, mdb->shards[r]->ev[EV_END], 0));
            SWB_CUDA(cudaMemcpyPeerAsync(mdb->d_gather[0] + r * k, mdb->devices[0], mdb->d_send[r], mdb->devices[r],
                                         k * sizeof(uint64_t), mdb->shards[0]->stream));
        }
    }

    // 3. global select on shard 0's stream: the one device-to-host copy (k hits) and, for shard 0, the one
    //    synchronisation; the other shards only have to finish before their statistics are read
    std::vector<swb_stats> sstats(G);
    st = swb_db_merge_keys(mdb->shards[0], mdb->d_gather[0], G * k, top_k, hits, n_hits, query_len, &sstats[0]);
    if (st != SWB_OK) return st;
    for (size_t r = 1; r < G; ++r) {
        swb_db* db = mdb->shards[r];
        std::lock_guard<std::mutex> shard_lock(db->mu);
        DeviceGuard guard(db->device);
        SWB_CUDA(cudaStreamSynchronize(db->stream));
        db->async_pending = false;
        fill_stats(db, query_len, &sstats[r]);
    }
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        for (size_t r = 0; r < G; ++r) {
            stats->lane_scored += sstats[r].lane_scored;
            stats->wavefront_scored += sstats[r].wavefront_scored;
            stats->chunks_claimed += sstats[r].chunks_claimed;
            stats->rescored_i32 += sstats[r].rescored_i32;
            stats->cells += sstats[r].cells;
            stats->padded_cells += sstats[r].padded_cells;
            stats->kernel_launches += sstats[r].kernel_launches;
            stats->ms_total = std::max(stats->ms_total, sstats[r].ms_total);
            stats->ms_setup = std::max(stats->ms_setup, sstats[r].ms_setup);
            stats->ms_scan = std::max(stats->ms_scan, sstats[r].ms_scan);
            stats->ms_rescore = std::max(stats->ms_rescore, sstats[r].ms_rescore);
            stats->ms_topk = std::max(stats->ms_topk, sstats[r].ms_topk);
        }
    }
    return SWB_OK;
}

}  // extern "C"
