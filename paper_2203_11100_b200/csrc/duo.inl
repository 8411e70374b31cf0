// duo.inl -- two queries per scan (duo.cuh): host side.  Included by cabi.cu inside extern "C".

namespace {

// Scores every local sequence against both queries; results land in d_slot_scores (a) and d_slot_scores2 (b).
// Asynchronous on db->stream.  Requires the packed int16 path (matrix + open within int8).
swb_status score_duo_core(swb_db* db, const uint8_t* qa, uint32_t ma, const uint8_t* qb, uint32_t mb, const int32_t* matrix,
                          int32_t open, int32_t ext) {
    cudaStream_t s = db->stream;
    swb_status st;
    const uint32_t m = std::max(ma, mb);
    const uint32_t n_tiles = (m + kInterTile - 1) / kInterTile;
    const uint32_t n_groups = static_cast<uint32_t>(db->meta.groups.size());
    db->launches_total += db->launches;
    db->launches = 0;
    db->last_tile = kInterTile;
    if (!db->d_slot_scores2)
        if ((st = dev_alloc(&db->d_slot_scores2, db->n_slots, &db->device_bytes)) != SWB_OK) return st;
    SWB_CUDA(cudaEventRecord(db->ev[EV_START], s));
    SWB_CUDA(cudaMemsetAsync(db->d_slot_scores, 0, std::max<size_t>(db->n_slots, 1) * sizeof(int32_t), s));
    SWB_CUDA(cudaMemsetAsync(db->d_slot_scores2, 0, std::max<size_t>(db->n_slots, 1) * sizeof(int32_t), s));
    SWB_CUDA(cudaMemsetAsync(db->d_counters, 0, 4 * sizeof(uint32_t), s));

    // stage matrix + both queries
    const size_t off_qa = 576 * sizeof(int32_t), off_qb = off_qa + ((ma + 15) & ~15u);
    if ((st = ensure_stage(db, db->stage_base + off_qb + mb + 16)) != SWB_OK) return st;
    uint8_t* const stage = db->h_stage + db->stage_base;
    std::memcpy(stage, matrix, off_qa);
    std::memcpy(stage + off_qa, qa, ma);
    std::memcpy(stage + off_qb, qb, mb);
    if (ma > db->query_cap) {
        if (db->d_query) cudaFree(db->d_query);
        db->d_query = nullptr;
        if ((st = dev_alloc(&db->d_query, static_cast<size_t>(ma) * 2, &db->device_bytes)) != SWB_OK) return st;
        db->query_cap = ma * 2;
    }
    if (mb > db->query2_cap) {
        if (db->d_query2) cudaFree(db->d_query2);
        db->d_query2 = nullptr;
        if ((st = dev_alloc(&db->d_query2, static_cast<size_t>(mb) * 2, &db->device_bytes)) != SWB_OK) return st;
        db->query2_cap = mb * 2;
    }
    SWB_CUDA(cudaMemcpyAsync(db->d_matrix, stage, off_qa, cudaMemcpyHostToDevice, s));
    SWB_CUDA(cudaMemcpyAsync(db->d_query, stage + off_qa, ma, cudaMemcpyHostToDevice, s));
    SWB_CUDA(cudaMemcpyAsync(db->d_query2, stage + off_qb, mb, cudaMemcpyHostToDevice, s));

    if ((st = ensure_dev(&db->d_prof2, &db->prof2_cap, static_cast<size_t>(n_tiles) * kDuoSliceWords, &db->device_bytes)) != SWB_OK)
        return st;
    DuoProfileParams pp{};
    pp.qa = db->d_query;
    pp.qb = db->d_query2;
    pp.ma = ma;
    pp.mb = mb;
    pp.matrix = db->d_matrix;
    pp.shift = open;
    pp.n_tiles = n_tiles;
    pp.prof2 = db->d_prof2;
    build_duo_profile_kernel<<<64, 256, 0, s>>>(pp);
    ++db->launches;
    SWB_CUDA(cudaEventRecord(db->ev[EV_UP], s));

    DuoParams dp{};
    dp.codes = reinterpret_cast<const uint4*>(db->d_codes);
    dp.groups = db->d_groups;
    dp.n_items = n_groups * 2;
    dp.prof2 = db->d_prof2;
    dp.n_tiles = n_tiles;
    dp.ring_chunks = scan_knobs().pipe_ring_cap >= 4 ? 4 : 2;
    dp.lag_div = scan_knobs().pipe_lag_div;
    dp.border0 = db->d_border0;
    dp.border1 = db->d_border1;
    dp.scores_a = db->d_slot_scores;
    dp.scores_b = db->d_slot_scores2;
    dp.ticket = db->d_counters + 2;
    dp.neg_open2 = pack16(-open);
    dp.neg_ext2 = pack16(-ext);
    const size_t smem = sizeof(PipeCtl) + static_cast<size_t>(kPipeWarps) * kDuoSliceBytes +
                        static_cast<size_t>(kPipeWarps) * dp.ring_chunks * kPipeChunkBytes;
    if (!db->duo_attr_set) {
        SWB_CUDA(cudaFuncSetAttribute(duo_pipeline_kernel<kInterTile, kInterThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(db->smem_optin)));
        db->duo_attr_set = true;
    }
    const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(static_cast<uint32_t>(db->sm_count), dp.n_items));
    duo_pipeline_kernel<kInterTile, kInterThreads><<<grid, kInterThreads, smem, s>>>(dp);
    ++db->launches;
    SWB_CUDA(cudaEventRecord(db->ev[EV_SCAN], s));
    SWB_CUDA(cudaEventRecord(db->ev[EV_RESCORE], s));
    SWB_CUDA(cudaGetLastError());
    return SWB_OK;
}

// After score_duo_core: exact re-run of one query's flagged lanes, its keys and its top k.  `q_dev` is the query's
// device copy, `scores` its slot scores.
swb_status finish_duo_query(swb_db* db, const uint8_t* q_dev, uint32_t m, const int32_t* matrix, int32_t open, int32_t ext,
                            int32_t* scores, uint32_t top_k, const uint64_t** d_out) {
    cudaStream_t s = db->stream;
    swb_status st;
    const QueryPlan pl = make_plan(db, m, matrix, open, ext);
    if (pl.may_overflow) {
        // the int32 kernel's profile of this query, then the flagged lanes (align.hpp:149-153)
        const size_t profi_elems = static_cast<size_t>(kProfRows) * pl.n_lane_tiles * 8;
        if ((st = ensure_dev(&db->d_prof8i, &db->prof8i_cap, profi_elems, &db->device_bytes)) != SWB_OK) return st;
        ProfileParams pp{};
        pp.query = q_dev;
        pp.matrix = db->d_matrix;
        pp.m = m;
        pp.shift_main = open;
        pp.shift_intra = open;
        pp.pstride = 0;
        pp.intra_t = pl.intra_t;
        pp.n_lane_tiles = pl.n_lane_tiles;
        pp.prof8i = db->d_prof8i;
        build_profile_kernel<<<64, 256, 0, s>>>(pp);
        SWB_CUDA(cudaMemsetAsync(db->d_counters + 1, 0, sizeof(uint32_t), s));
        collect_flagged_kernel<<<std::max(1u, std::min(1024u, (db->n_slots + 255) / 256)), 256, 0, s>>>(
            scores, db->n_slots, pl.limit, db->d_flag_list, db->d_counters + 1);
        db->launches += 2;
        if ((st = run_intra(db, pl, db->d_flag_list, s, scores)) != SWB_OK) return st;
    }
    build_keys_kernel<<<std::max(1u, std::min(1024u, (db->n_slots + 255) / 256)), 256, 0, s>>>(scores, db->d_slot_index, db->n_slots,
                                                                                            db->d_keys);
    ++db->launches;
    return select_topk(db, db->d_keys, db->n_slots, top_k, d_out);
}

// Can this pair of queries share one scan?
bool duo_applies(const swb_db* db, uint32_t ma, uint32_t mb, const int32_t* matrix, int32_t open, int32_t ext) {
    const ScanKnobs& k = scan_knobs();
    const uint32_t lo = std::min(ma, mb), hi = std::max(ma, mb);
    if (k.duo_ratio > 1.0 || lo == 0 || static_cast<double>(lo) < k.duo_ratio * static_cast<double>(hi)) return false;
    if ((hi + kInterTile - 1) / kInterTile < k.pipe_min_tiles) return false;   // short queries: chains, not throughput
    if (db->scan_policy != SWB_SCAN_AUTO || db->force_intra) return false;
    if (static_cast<double>(db->meta.groups.size()) < k.duo_min_groups_per_sm * static_cast<double>(db->sm_count)) return false;
    return make_plan(db, hi, matrix, open, ext).main == kMainS16;
}

}  // namespace

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
    if (pl.main != kMainS16) return fail(SWB_ERR_UNSUPPORTED, "the two-query scan needs the packed int16 path");
    st = score_duo_core(db, qa, ma, qb, mb, matrix, gap_open, gap_extend);
    if (st != SWB_OK) return st;
    cudaStream_t s = db->stream;
    const uint32_t n_total = db->meta.n_total;
    if (!db->d_all_scores)
        if ((st = dev_alloc(&db->d_all_scores, n_total, &db->device_bytes)) != SWB_OK) return st;
    const unsigned blocks = std::max(1u, std::min(1024u, (db->n_slots + 255) / 256));
    int32_t* outs[2] = {scores_a, scores_b};
    int32_t* srcs[2] = {db->d_slot_scores, db->d_slot_scores2};
    for (int q = 0; q < 2; ++q) {
        SWB_CUDA(cudaMemcpyAsync(db->d_all_scores, outs[q], static_cast<size_t>(n_total) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        if (db->n_slots) scatter_scores_kernel<<<blocks, 256, 0, s>>>(srcs[q], db->d_slot_index, db->n_slots, db->d_all_scores);
        SWB_CUDA(cudaMemcpyAsync(outs[q], db->d_all_scores, static_cast<size_t>(n_total) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    }
    SWB_CUDA(cudaEventRecord(db->ev[EV_TOPK], s));
    SWB_CUDA(cudaEventRecord(db->ev[EV_END], s));
    SWB_CUDA(cudaStreamSynchronize(s));
    fill_stats(db, ma + mb, stats);
    return SWB_OK;
}
