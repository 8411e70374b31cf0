// duo.inl -- two streams of queries per scan (duo.cuh): host side.  Included by cabi.cu inside its anonymous namespace.

inline SharedScanMode shared_mode(const swb_db* db) {
    return shared_scan_mode(scan_knobs(), static_cast<uint32_t>(db->meta.groups.size()), db->max_rows, db->meta.padded_rows,
                            static_cast<uint32_t>(db->sm_count));
}

// Scores every local sequence against every query of the scan; query number `scan_queries[i]` (a's members first, then
// b's) gets the score array d_multi_scores + i * n_slots and the device copy d_multi_codes + code_off[i].
// Asynchronous on db->stream.  Requires the packed int16 path (matrix + open within int8).
swb_status score_streams_core(swb_db* db, const uint8_t* const* queries, const uint32_t* lens, const DuoScan& scan,
                              const int32_t* matrix, int32_t open, int32_t ext, std::vector<uint32_t>& scan_queries,
                              std::vector<uint32_t>& code_off) {
    cudaStream_t s = db->stream;
    swb_status st;
    if ((st = settle_async(db)) != SWB_OK) return st;
    const uint32_t n_tiles = std::max(scan.tiles_a, scan.tiles_b);
    const uint32_t n_groups = static_cast<uint32_t>(db->meta.groups.size());
    scan_queries.clear();
    scan_queries.insert(scan_queries.end(), scan.a.begin(), scan.a.end());
    scan_queries.insert(scan_queries.end(), scan.b.begin(), scan.b.end());
    const uint32_t nq = static_cast<uint32_t>(scan_queries.size());
    db->launches_total += db->launches;
    db->launches = 0;
    db->last_tile = kInterTile;
    db->last_units = n_groups * 2;

    // ---- staging: matrix | concatenated codes | tile table ---------------------------------------------------------
    code_off.assign(nq, 0);
    size_t codes_bytes = 0;
    for (uint32_t i = 0; i < nq; ++i) {
        code_off[i] = static_cast<uint32_t>(codes_bytes);
        codes_bytes += (lens[scan_queries[i]] + 15) & ~15u;
    }
    const size_t off_codes = 576 * sizeof(int32_t);
    const size_t off_tiles = (off_codes + codes_bytes + 31) & ~size_t(31);
    const size_t stage_bytes = off_tiles + static_cast<size_t>(n_tiles) * sizeof(DuoTile);
    if ((st = ensure_stage(db, db->stage_base + stage_bytes)) != SWB_OK) return st;
    uint8_t* const stage = db->h_stage + db->stage_base;
    std::memcpy(stage, matrix, off_codes);
    for (uint32_t i = 0; i < nq; ++i) std::memcpy(stage + off_codes + code_off[i], queries[scan_queries[i]], lens[scan_queries[i]]);
    DuoTile* tiles = reinterpret_cast<DuoTile*>(stage + off_tiles);
    for (uint32_t t = 0; t < n_tiles; ++t) tiles[t] = DuoTile{kDuoNone, kDuoNone, 3u, 0, 0, 0, 0, 0};
    auto lay_out = [&](const std::vector<uint32_t>& stream, uint32_t first_local, bool high) {
        uint32_t t = 0;
        for (size_t k = 0; k < stream.size(); ++k) {
            const uint32_t local = first_local + static_cast<uint32_t>(k), m = lens[stream[k]];
            for (uint32_t c = 0; c < m; c += kInterTile, ++t) {
                DuoTile& td = tiles[t];
                (high ? td.qb : td.qa) = local;
                (high ? td.b_off : td.a_off) = code_off[local] + c;
                (high ? td.b_left : td.a_left) = m - c;
                if (c) td.reset &= high ? ~2u : ~1u;   // only a query's first tile starts from the matrix edge
            }
        }
    };
    lay_out(scan.a, 0, false);
    lay_out(scan.b, static_cast<uint32_t>(scan.a.size()), true);

    if ((st = ensure_dev(&db->d_multi_codes, &db->multi_codes_cap, codes_bytes + 64, &db->device_bytes)) != SWB_OK) return st;
    if ((st = ensure_dev(&db->d_duo_tiles, &db->duo_tiles_cap, static_cast<size_t>(n_tiles) * sizeof(DuoTile), &db->device_bytes)) != SWB_OK)
        return st;
    if ((st = ensure_dev(&db->d_multi_scores, &db->multi_scores_cap, static_cast<size_t>(nq) * std::max<uint32_t>(db->n_slots, 1),
                         &db->device_bytes)) != SWB_OK)
        return st;
    if ((st = ensure_dev(&db->d_prof2, &db->prof2_cap, static_cast<size_t>(n_tiles) * kDuoSliceWords, &db->device_bytes)) != SWB_OK)
        return st;
    // pass items: one item per half-group and pass of 16 tiles, pass-major over the whole shard (duo.cuh)
    const bool pass_items = shared_mode(db) == kSharedPass && n_tiles > kPipeWarps;
    const uint32_t n_passes = (n_tiles + kPipeWarps - 1) / kPipeWarps;
    const size_t progress_counters = static_cast<size_t>(n_groups) * 2 * n_passes;
    if (pass_items && (st = ensure_dev(&db->d_duo_progress, &db->duo_progress_cap, progress_counters, &db->device_bytes)) != SWB_OK)
        return st;
    SWB_CUDA(cudaEventRecord(db->ev[EV_START], s));   // every allocation is above this line: none inside the timed scan
    SWB_CUDA(cudaMemsetAsync(db->d_multi_scores, 0, static_cast<size_t>(nq) * std::max<uint32_t>(db->n_slots, 1) * sizeof(int32_t), s));
    SWB_CUDA(cudaMemsetAsync(db->d_counters, 0, 4 * sizeof(uint32_t), s));
    SWB_CUDA(cudaMemcpyAsync(db->d_matrix, stage, off_codes, cudaMemcpyHostToDevice, s));
    SWB_CUDA(cudaMemcpyAsync(db->d_multi_codes, stage + off_codes, codes_bytes, cudaMemcpyHostToDevice, s));
    SWB_CUDA(cudaMemcpyAsync(db->d_duo_tiles, tiles, static_cast<size_t>(n_tiles) * sizeof(DuoTile), cudaMemcpyHostToDevice, s));

    DuoProfileParams pp{};
    pp.codes = db->d_multi_codes;
    pp.tiles = reinterpret_cast<const DuoTile*>(db->d_duo_tiles);
    pp.matrix = db->d_matrix;
    pp.shift = open;
    pp.n_tiles = n_tiles;
    pp.prof2 = db->d_prof2;
    build_duo_profile_kernel<<<128, 256, 0, s>>>(pp);
    ++db->launches;
    SWB_CUDA(cudaEventRecord(db->ev[EV_UP], s));

    DuoParams dp{};
    dp.codes = reinterpret_cast<const uint4*>(db->d_codes);
    dp.groups = db->d_groups;
    dp.n_items = n_groups * 2;
    if (pass_items) {
        dp.pass_items = 1;
        dp.n_passes = n_passes;
        // Pass-major WITHIN WINDOWS of half-groups: a pass writes one border row per database row of its half-group
        // (256 B) and the next pass reads it back, so what is in flight between two passes is the window's rows x 256 B.
        // Handing the passes out over the whole shard at once (the first version) made that the whole shard -- 200 MB on a
        // 1/8 Swiss-Prot, against 126 MB of L2: 19 GB of DRAM traffic per sweep, 37 x the algorithmic bytes.  A window is
        // as many half-groups (longest first) as keep that under duo_window_mb, but at least one per SM, so that the next
        // pass of a half-group still goes to another CTA while its previous pass runs.
        {
            const uint64_t budget_rows = static_cast<uint64_t>(scan_knobs().duo_window_mb) * (1u << 20) / 256;
            uint64_t rows = 0;
            uint32_t fit = 0;
            while (fit < n_groups && rows + 2ull * db->meta.groups[fit].n_chunks * kRowsPerChunk <= budget_rows)
                rows += 2ull * db->meta.groups[fit++].n_chunks * kRowsPerChunk;
            dp.window = std::min<uint32_t>(n_groups * 2, std::max<uint32_t>(2 * fit, static_cast<uint32_t>(db->sm_count + 1) & ~1u));
        }
        dp.n_items = n_groups * 2 * dp.n_passes;
        SWB_CUDA(cudaMemsetAsync(db->d_duo_progress, 0, progress_counters * sizeof(uint32_t), s));
        dp.progress = db->d_duo_progress;
    }
    dp.prof2 = db->d_prof2;
    dp.tiles = reinterpret_cast<const DuoTile*>(db->d_duo_tiles);
    dp.n_tiles = n_tiles;
    dp.ring_chunks = scan_knobs().pipe_ring_cap >= 4 ? 4 : 2;
    dp.lag_div = scan_knobs().pipe_lag_div;
    dp.border0 = db->d_border0;
    dp.border1 = db->d_border1;
    dp.scores = db->d_multi_scores;
    dp.n_slots = db->n_slots;
    dp.ticket = db->d_counters + 2;
    dp.neg_open2 = pack16(-open);
    dp.neg_ext2 = pack16(-ext);
    const size_t smem = sizeof(PipeCtl) + static_cast<size_t>(kPipeWarps) * kDuoSliceBytes +
                        static_cast<size_t>(kPipeWarps) * dp.ring_chunks * kPipeChunkBytes;
    if (!db->duo_attr_set) {
        SWB_CUDA(cudaFuncSetAttribute(duo_pipeline_kernel<kInterTile, kInterThreads, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(db->smem_optin)));
        SWB_CUDA(cudaFuncSetAttribute(duo_pipeline_kernel<kInterTile, kInterThreads, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(db->smem_optin)));
        db->duo_attr_set = true;
    }
    const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(static_cast<uint32_t>(db->sm_count), dp.n_items));
#ifdef SWB_PIPE_STATS
    dp.stats = pipe_stats_buffer(s);
#endif
    if (dp.pass_items) duo_pipeline_kernel<kInterTile, kInterThreads, true><<<grid, kInterThreads, smem, s>>>(dp);
    else duo_pipeline_kernel<kInterTile, kInterThreads, false><<<grid, kInterThreads, smem, s>>>(dp);
    ++db->launches;
#ifdef SWB_PIPE_STATS
    report_pipe_stats("two-stream", dp.stats, grid, n_tiles, s);
#endif
    SWB_CUDA(cudaEventRecord(db->ev[EV_SCAN], s));
    SWB_CUDA(cudaEventRecord(db->ev[EV_RESCORE], s));
    SWB_CUDA(cudaGetLastError());
    return SWB_OK;
}

// After score_streams_core: exact re-run of one query's flagged lanes (align.hpp:149-153).  `q_dev` is the query's
// device copy, `scores` its slot scores.
swb_status rescore_duo_query(swb_db* db, const uint8_t* q_dev, uint32_t m, const int32_t* matrix, int32_t open, int32_t ext,
                             int32_t* scores) {
    cudaStream_t s = db->stream;
    swb_status st;
    const QueryPlan pl = make_plan(db, m, matrix, open, ext);
    if (!pl.may_overflow) return SWB_OK;
    // the int32 kernel's profile of this query, then the flagged lanes
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
    return run_intra(db, pl, db->d_flag_list, s, scores);
}

// ... and then its keys and its top k.
swb_status finish_duo_query(swb_db* db, const uint8_t* q_dev, uint32_t m, const int32_t* matrix, int32_t open, int32_t ext,
                            int32_t* scores, uint32_t top_k, const uint64_t** d_out) {
    cudaStream_t s = db->stream;
    const swb_status st = rescore_duo_query(db, q_dev, m, matrix, open, ext, scores);
    if (st != SWB_OK) return st;
    build_keys_kernel<<<std::max(1u, std::min(1024u, (db->n_slots + 255) / 256)), 256, 0, s>>>(scores, db->d_slot_index, db->n_slots,
                                                                                            db->d_keys);
    ++db->launches;
    return select_topk(db, db->d_keys, db->n_slots, top_k, d_out);
}

// Can queries of a batch share scans on this handle, and in which form?  (The rest is plan_batch in scan_plan.hpp.)
SharedScanMode duo_mode(const swb_db* db, const int32_t* matrix, int32_t open, int32_t ext) {
    if (db->scan_policy != SWB_SCAN_AUTO || db->force_intra) return kSharedNone;
    if (make_plan(db, 64, matrix, open, ext).main != kMainS16) return kSharedNone;
    return shared_mode(db);
}
