// pairs.inl -- entry points that score ad-hoc subjects or trace alignments back: swb_merge_keys, swb_score_batch,
// swb_score_pair, swb_db_align_hits, swb_align_traceback.  Included by cabi.cu inside extern "C".

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
    BlockCacheScope cache;
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
    cudaStreamSynchronize(tmp.own_stream);
    dev_free(d_in, true);
    for (auto& p : tmp.d_sel) dev_free(p, true);
    dev_free(tmp.d_sort, true);
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
    BlockCacheScope cache;
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
    BlockCacheScope cache;
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

// Direction matrices of all hits of one call live on the device at once: memory_cap bounds each pair (align.hpp:262-267), this
// bounds their sum -- beyond it the hits are traced back in several rounds (large top_k with long query and subjects).
static uint64_t traceback_round_bytes() {   // SWB200_TRACEBACK_ROUND_KB (tests: a tiny value forces several rounds)
    static const uint64_t bytes = [] {
        const char* e = std::getenv("SWB200_TRACEBACK_ROUND_KB");
        const long long kb = e ? std::atoll(e) : 0;
        return kb > 0 ? static_cast<uint64_t>(kb) << 10 : 6ull << 30;
    }();
    return bytes;
}

static swb_status align_hits_locked(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix, int32_t gap_open,
                                    int32_t gap_extend, const swb_hit* hits, uint32_t n_hits, uint64_t memory_cap, swb_alignment* out,
                                    uint8_t* ops, const uint64_t* ops_offset);

swb_status swb_db_align_hits(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                             int32_t gap_open, int32_t gap_extend, const swb_hit* hits, uint32_t n_hits,
                             uint64_t memory_cap, swb_alignment* out, uint8_t* ops, const uint64_t* ops_offset) {
    if (!db) return fail(SWB_ERR_INVALID, "db is null");
    if (n_hits && (!hits || !out || !ops_offset)) return fail(SWB_ERR_INVALID, "null argument");
    swb_status st = check_scoring_args(query, query_len, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    return align_hits_locked(db, query, query_len, matrix, gap_open, gap_extend, hits, n_hits, memory_cap, out, ops, ops_offset);
}

static swb_status align_hits_locked(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix, int32_t gap_open,
                                    int32_t gap_extend, const swb_hit* hits, uint32_t n_hits, uint64_t memory_cap, swb_alignment* out,
                                    uint8_t* ops, const uint64_t* ops_offset) {
    swb_status st = SWB_OK;
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
    if (dir_bytes > traceback_round_bytes() && n_hits > 1) {
        // too much for one round: the two halves of the hit list one after the other (ops_offset holds absolute offsets)
        const uint32_t half = n_hits / 2;
        st = align_hits_locked(db, query, query_len, matrix, gap_open, gap_extend, hits, half, memory_cap, out, ops, ops_offset);
        if (st != SWB_OK) return st;
        return align_hits_locked(db, query, query_len, matrix, gap_open, gap_extend, hits + half, n_hits - half, memory_cap, out + half, ops,
                                 ops_offset + half);
    }

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
    cudaStreamSynchronize(s);   // (after an error the stream may still be busy with these blocks)
    for (void* ptr : {static_cast<void*>(d_dir), static_cast<void*>(d_ops), static_cast<void*>(d_result),
                      static_cast<void*>(d_b0), static_cast<void*>(d_b1), static_cast<void*>(d_prof8),
                      static_cast<void*>(d_prof32), static_cast<void*>(d_query), static_cast<void*>(d_jobs)})
        dev_free(ptr, true);
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
    BlockCacheScope cache;
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
