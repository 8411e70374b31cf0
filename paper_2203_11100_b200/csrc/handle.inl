// handle.inl -- lifetime of a shard handle: upload of the packed database, stream/events, statistics.
// Included by cabi.cu inside its anonymous namespace.

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

// codes_src: the interleaved residues when they are not in meta.codes (a memory-mapped packed file, persist.inl).
swb_status upload_db(swb_db* db, const uint8_t* codes_src = nullptr, size_t codes_bytes = 0) {
    PackedDb& m = db->meta;
    db->n_slots = static_cast<uint32_t>(m.groups.size() * kGroupSeqs);
    db->max_rows = m.groups.empty() ? 0 : m.groups[0].n_chunks * kRowsPerChunk;
    uint64_t* tally = &db->device_bytes;
    swb_status st;
#define ALLOC_COPY(dptr, vec)                                                                        \
    if ((st = dev_alloc(&(dptr), (vec).size(), tally)) != SWB_OK) return st;                         \
    if (!(vec).empty())                                                                              \
        SWB_CUDA(cudaMemcpy((dptr), (vec).data(), (vec).size() * sizeof((vec)[0]), cudaMemcpyHostToDevice));
    if (codes_src) {
        if ((st = dev_alloc(&db->d_codes, codes_bytes, tally)) != SWB_OK) return st;
        if (codes_bytes) {
            // pin the mapping for the copy where the driver allows it (read-only mapping); else a pageable copy
            const bool pinned = cudaHostRegister(const_cast<uint8_t*>(codes_src), codes_bytes, cudaHostRegisterReadOnly) == cudaSuccess;
            if (!pinned) cudaGetLastError();
            const cudaError_t e = cudaMemcpy(db->d_codes, codes_src, codes_bytes, cudaMemcpyHostToDevice);
            if (pinned) cudaHostUnregister(const_cast<uint8_t*>(codes_src));
            if (e != cudaSuccess) return fail(SWB_ERR_CUDA, std::string("upload of the packed residues: ") + cudaGetErrorString(e));
        }
    } else {
        ALLOC_COPY(db->d_codes, m.codes);
    }
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
    if (cudaStreamCreateWithFlags(&db->side_stream, cudaStreamNonBlocking) != cudaSuccess)
        return fail(SWB_ERR_CUDA, "cudaStreamCreate failed");
    if (cudaEventCreateWithFlags(&db->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&db->ev_join, cudaEventDisableTiming) != cudaSuccess)
        return fail(SWB_ERR_CUDA, "cudaEventCreate failed");
    for (auto& ev : db->ev)
        if (cudaEventCreate(&ev) != cudaSuccess) return fail(SWB_ERR_CUDA, "cudaEventCreate failed");
    if (host_alloc(reinterpret_cast<void**>(&db->h_counters), 4 * sizeof(uint32_t)) != SWB_OK)
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
    // three attributes, not cudaGetDeviceProperties: that call costs milliseconds, and the pair / batch entry points
    // build a handle per call
    int major = 0, sms = 0, smem_optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) {
        delete db;
        return fail(SWB_ERR_CUDA, cudaGetErrorString(e));
    }
    if (major < 10) {
        delete db;
        return fail(SWB_ERR_CUDA, "device is not sm_100-class; this library is built for sm_100a only");
    }
    db->sm_count = sms;
    db->smem_optin = static_cast<size_t>(smem_optin);
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
