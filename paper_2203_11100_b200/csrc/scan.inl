// scan.inl -- one search on one shard: upload, profile, unit table, packed scan, int32 re-run, top-k select.
// Included by cabi.cu inside its anonymous namespace.

void launch_pipeline(const PipeParams& qp, bool slices, uint32_t grid, size_t smem, cudaStream_t s) {
    if (slices) pipeline_s16_kernel<kInterTile, kInterThreads, true><<<grid, kInterThreads, smem, s>>>(qp);
    else pipeline_s16_kernel<kInterTile, kInterThreads, false><<<grid, kInterThreads, smem, s>>>(qp);
}

template <int T, typename PT>
void launch_intra(const IntraParams& ip, uint32_t ctas, uint32_t warps, cudaStream_t s) {
    // the int8 flavour stages each lane's 25 profile words in shared memory: 200 B per thread, 50 KB for 8 warps
    const size_t smem = sizeof(PT) == 1 ? static_cast<size_t>(kProfRows) * warps * 32 * sizeof(uint2) : 0;
    if (smem > 48 * 1024)   // per device, so not remembered: the call is cheap
        cudaFuncSetAttribute(intra_s32_kernel<T, PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    intra_s32_kernel<T, PT><<<ctas, warps * 32, smem, s>>>(ip);
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
swb_status run_intra(swb_db* db, const QueryPlan& pl, const uint32_t* list, cudaStream_t s, int32_t* slot_scores = nullptr) {
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
    ip.slot_scores = slot_scores ? slot_scores : db->d_slot_scores;
    ip.open = pl.open;
    ip.ext = pl.ext;
    if (pl.wide) launch_intra_t<int32_t>(pl.intra_t, ip, db->intra_ctas, pl.intra_w, s);
    else launch_intra_t<int8_t>(pl.intra_t, ip, db->intra_ctas, pl.intra_w, s);
    ++db->launches;
    return SWB_OK;
}

#ifdef SWB_PIPE_STATS
// Debug builds only (SWB_PIPE_STATS): where do the warps of a pipeline kernel wait?  [cta][warp][4] clocks.
unsigned long long* pipe_stats_buffer(cudaStream_t s) {
    static unsigned long long* d_stats = nullptr;
    if (!d_stats) cudaMalloc(&d_stats, sizeof(unsigned long long) * 4 * kPipeWarps * 1024);
    cudaMemsetAsync(d_stats, 0, sizeof(unsigned long long) * 4 * kPipeWarps * 1024, s);
    return d_stats;
}

void report_pipe_stats(const char* what, const unsigned long long* d_stats, uint32_t grid, uint32_t n_tiles, cudaStream_t s) {
    std::vector<unsigned long long> h(static_cast<size_t>(grid) * kPipeWarps * 4);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), d_stats, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double tot[kPipeWarps][4] = {};
    for (uint32_t c = 0; c < grid; ++c)
        for (uint32_t w = 0; w < kPipeWarps; ++w)
            for (int k = 0; k < 4; ++k) tot[w][k] += static_cast<double>(h[(static_cast<size_t>(c) * kPipeWarps + w) * 4 + k]);
    std::fprintf(stderr, "%s stats tiles=%u grid=%u: warp  wait_in%%  wait_out%%  item%%  (of the warp's lifetime)\n", what, n_tiles, grid);
    double sum_in = 0, sum_out = 0;
    for (uint32_t w = 0; w < kPipeWarps; ++w) {
        std::fprintf(stderr, "   %2u  %6.2f  %6.2f  %6.2f   life %.2f ms\n", w, 100 * tot[w][0] / tot[w][3], 100 * tot[w][1] / tot[w][3],
                     100 * tot[w][2] / tot[w][3], tot[w][3] / grid / 1.9e6);
        sum_in += 100 * tot[w][0] / tot[w][3] / kPipeWarps, sum_out += 100 * tot[w][1] / tot[w][3] / kPipeWarps;
    }
    std::fprintf(stderr, "   mean wait_in %.2f%% wait_out %.2f%%\n", sum_in, sum_out);
}
#endif

constexpr size_t kWaveStaticSmem = 1024;   // the wavefront kernel's own static shared memory, rounded up generously

// The wavefront kernel.  The narrow-tile and row-block paths are only compiled into the variants that need them, so
// that the plain 32-column sweep keeps its register allocation; a profile too large for shared memory is read from
// global memory.
swb_status launch_wavefront(swb_db* db, const WaveParams& wp, uint32_t grid, uint32_t threads, size_t smem, bool narrow,
                            bool rowblock, cudaStream_t s) {
    constexpr size_t kStaticSmem = kWaveStaticSmem;
    const bool in_smem = smem + kStaticSmem <= db->smem_optin;
#define SWB_LAUNCH_S16(THREADS, NARROW, RB)                                                                        \
    {                                                                                                              \
        if (in_smem) {                                                                                             \
            SWB_CUDA(cudaFuncSetAttribute(wavefront_s16_kernel<true, kInterTile, THREADS, NARROW, RB>,             \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,                             \
                                          static_cast<int>(db->smem_optin - kStaticSmem)));                        \
            wavefront_s16_kernel<true, kInterTile, THREADS, NARROW, RB><<<grid, threads, smem, s>>>(wp);            \
        } else {                                                                                                   \
            wavefront_s16_kernel<false, kInterTile, THREADS, NARROW, RB><<<grid, threads, 0, s>>>(wp);              \
        }                                                                                                          \
    }
    // CTAs of 4 or 8 warps (narrow units next to the pipeline, one or two warps per scheduler) get builds of their own,
    // whose register budget is not the 128 of a 16-warp CTA
    if (narrow && threads <= kNarrowThreads) {
        if (rowblock) SWB_LAUNCH_S16(kNarrowThreads, true, true)
        else SWB_LAUNCH_S16(kNarrowThreads, true, false)
    } else if (narrow && threads <= 2 * kNarrowThreads) {
        if (rowblock) SWB_LAUNCH_S16(2 * kNarrowThreads, true, true)
        else SWB_LAUNCH_S16(2 * kNarrowThreads, true, false)
    } else if (narrow && rowblock) SWB_LAUNCH_S16(kInterThreads, true, true)
    else if (narrow) SWB_LAUNCH_S16(kInterThreads, true, false)
    else if (rowblock) SWB_LAUNCH_S16(kInterThreads, false, true)
    else SWB_LAUNCH_S16(kInterThreads, false, false)
#undef SWB_LAUNCH_S16
    ++db->launches;
    return SWB_OK;
}

// Scores every local sequence; results land in d_slot_scores.  Asynchronous on db->stream.
// A search enqueued by swb_search_keys_device may still be reading its inputs from the pinned staging buffer.
swb_status settle_async(swb_db* db) {
    if (db->async_pending) {
        SWB_CUDA(cudaStreamSynchronize(db->stream));
        db->async_pending = false;
    }
    return SWB_OK;
}

swb_status score_core(swb_db* db, const uint8_t* query, uint32_t m, const int32_t* matrix, int32_t open,
                      int32_t ext) {
    cudaStream_t s = db->stream;
    {
        const swb_status settled = settle_async(db);
        if (settled != SWB_OK) return settled;
    }
    const QueryPlan pl = make_plan(db, m, matrix, open, ext);
    db->launches_total += db->launches;
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
    swb_status st = ensure_stage(db, db->stage_base + stage_bytes);   // a no-op inside swb_search_many (pre-sized)
    if (st != SWB_OK) return st;
    uint8_t* const stage = db->h_stage + db->stage_base;
    if (m > db->query_cap) {
        if (db->d_query) dev_free(db->d_query);
        db->d_query = nullptr;
        st = dev_alloc(&db->d_query, static_cast<size_t>(m) * 2, &db->device_bytes);
        if (st != SWB_OK) return st;
        db->query_cap = m * 2;
    }
    std::memcpy(stage, matrix, off_query);
    std::memcpy(stage + off_query, query, m);
    const uint32_t n_tiles = (m + pl.tile - 1) / pl.tile;
    uint32_t n_tiles_narrow = (m + kNarrowTile - 1) / kNarrowTile, narrow_tile = kNarrowTile;
    bool narrow_staged = false, narrow_helpers = false;
    uint32_t n_units = 0;
    uint32_t pipe_first = n_groups;   // groups [pipe_first, n_groups) go through the on-chip pipeline
    uint32_t wave_sms = static_cast<uint32_t>(db->sm_count);   // SMs the wavefront kernel gets
    uint32_t wave_threads = kInterThreads;                      // and its CTA size
    const size_t prof_elems = static_cast<size_t>(kProfRows) * pl.pstride;
    const PipeRings pipe_ring_plan = pipe_ring_chunks(db, prof_elems);
    const uint32_t pipe_rings = pipe_ring_plan.chunks;
    bool any_narrow = false, any_rowblock = false;
    if (packed) {
        // which kernel scans which groups, and the wavefront kernel's units: scan_plan.hpp
        uint32_t* us = reinterpret_cast<uint32_t*>(stage + off_units);
        uint32_t* vso = reinterpret_cast<uint32_t*>(stage + off_vsoff);
        uint8_t* modes = stage + off_modes;
        ScanShape shape;
        shape.groups = db->meta.groups.data();
        shape.n_groups = n_groups;
        shape.padded_rows = db->meta.padded_rows;
        shape.n_tiles = n_tiles;
        shape.query_len = m;
        shape.sm_count = static_cast<uint32_t>(db->sm_count);
        shape.warps_per_cta = pl.threads / 32;
        shape.s16 = pl.main == kMainS16;
        shape.policy = db->scan_policy;
        shape.pipe_rings = pipe_rings;
        {
            const size_t used = ((prof_elems + 127) & ~size_t(127)) + kWaveStaticSmem;
            shape.narrow_room = used < db->smem_optin ? db->smem_optin - used : 0;
        }
        const ScanPlan sp = plan_scan(shape, scan_knobs(), us, vso, modes);
        pipe_first = sp.pipe_first;
        wave_sms = sp.wave_sms;
        wave_threads = sp.wave_threads;
        n_units = sp.n_units;
        any_narrow = sp.any_narrow;
        any_rowblock = sp.any_rowblock;
        n_tiles_narrow = sp.n_tiles_narrow;
        narrow_tile = sp.narrow_tile;
        narrow_staged = sp.narrow_staged;
        narrow_helpers = sp.narrow_helpers && sp.any_narrow;
        if (any_narrow && narrow_staged && sp.link_rows * 256 > db->nlinks_cap) {
            // link buffers of the narrow groups (256 B per row and tile boundary): every word holds kNarrowEmpty between
            // searches -- the consumers give them back
            if ((st = ensure_dev(&db->d_nlinks, &db->nlinks_cap, static_cast<size_t>(sp.link_rows) * 256, &db->device_bytes)) != SWB_OK) return st;
            SWB_CUDA(cudaMemsetAsync(db->d_nlinks, 0x80, db->nlinks_cap, s));
        }
        SWB_CUDA(cudaMemcpyAsync(db->d_unit_start, us, (static_cast<size_t>(n_groups) + 1) * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, s));
        SWB_CUDA(cudaMemcpyAsync(db->d_group_mode, modes, std::max<size_t>(n_groups, 1), cudaMemcpyHostToDevice, s));
        SWB_CUDA(cudaMemcpyAsync(db->d_vstate_off, vso, std::max<size_t>(n_groups, 1) * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, s));
        if (any_rowblock) {
            const size_t need = static_cast<size_t>(sp.vstate_slots) * (kVStateWords / 4) * 32;
            if ((st = ensure_dev(&db->d_vstate, &db->vstate_cap, need, &db->device_bytes)) != SWB_OK) return st;
        }
        if ((st = ensure_dev(&db->d_progress, &db->progress_cap, n_units, &db->device_bytes)) != SWB_OK) return st;
        if (n_units) SWB_CUDA(cudaMemsetAsync(db->d_progress, 0, static_cast<size_t>(n_units) * sizeof(uint32_t), s));
        db->last_units = n_units + (n_groups - pipe_first);
    }
    SWB_CUDA(cudaMemcpyAsync(db->d_matrix, stage, off_query, cudaMemcpyHostToDevice, s));
    SWB_CUDA(cudaMemcpyAsync(db->d_query, stage + off_query, m, cudaMemcpyHostToDevice, s));

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
    // Pipeline groups run on a second stream next to the wavefront kernel's tall groups; the SMs the wavefront
    // kernel used join the pipeline's item queue when it is done (a second, small pipeline launch behind it).
    const uint32_t n_pipe_items = n_groups - pipe_first;
    PipeParams qp{};
    size_t pipe_smem = 0;
    if (packed && n_pipe_items) {
        qp.codes = reinterpret_cast<const uint4*>(db->d_codes);
        qp.groups = db->d_groups;
        qp.group_first = pipe_first;
        qp.n_items = n_pipe_items;
        qp.prof8 = db->d_prof8;
        qp.pstride = pl.pstride;
        qp.prof_bytes = static_cast<uint32_t>(pipe_ring_plan.prof_bytes);   // the whole profile, or 16 tile slices
        qp.n_tiles = n_tiles;
        qp.ring_chunks = pipe_rings;
        qp.lag_div = scan_knobs().pipe_lag_div;
        qp.border = db->d_border0;
        qp.slot_scores = db->d_slot_scores;
        qp.ticket = db->d_counters + 2;
        qp.neg_open2 = pack16(-open);
        qp.neg_ext2 = pack16(-ext);
        pipe_smem = qp.prof_bytes + sizeof(PipeCtl) + static_cast<size_t>(kPipeWarps) * qp.ring_chunks * kPipeChunkBytes;
        if (!db->pipe_attr_set) {
            SWB_CUDA(cudaFuncSetAttribute(pipeline_s16_kernel<kInterTile, kInterThreads, false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(db->smem_optin)));
            SWB_CUDA(cudaFuncSetAttribute(pipeline_s16_kernel<kInterTile, kInterThreads, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(db->smem_optin)));
            db->pipe_attr_set = true;
        }
        const uint32_t wave_grid = pipe_first ? wave_sms : 0;
        const uint32_t side_grid = std::min<uint32_t>(static_cast<uint32_t>(db->sm_count) - wave_grid, n_pipe_items);
#ifdef SWB_PIPE_STATS
        qp.stats = pipe_stats_buffer(s);
#endif
        if (wave_grid) {
            SWB_CUDA(cudaEventRecord(db->ev_fork, s));
            SWB_CUDA(cudaStreamWaitEvent(db->side_stream, db->ev_fork, 0));
            launch_pipeline(qp, pipe_ring_plan.slices, side_grid, pipe_smem, db->side_stream);
            SWB_CUDA(cudaEventRecord(db->ev_join, db->side_stream));
        } else {
            launch_pipeline(qp, pipe_ring_plan.slices, side_grid, pipe_smem, s);
        }
        ++db->launches;
    }
    if (packed && pipe_first) {
        WaveParams wp{};
        wp.codes = reinterpret_cast<const uint4*>(db->d_codes);
        wp.groups = db->d_groups;
        wp.n_groups = pipe_first;
        wp.unit_start = db->d_unit_start;
        wp.group_mode = db->d_group_mode;
        wp.vstate_off = db->d_vstate_off;
        wp.vstate = db->d_vstate;
        wp.n_units = n_units;
        wp.n_tiles_narrow = n_tiles_narrow;
        wp.narrow_tile = narrow_tile;
        wp.nlinks = db->d_nlinks;
        wp.narrow_staged = narrow_staged ? 1u : 0u;
        wp.narrow_helpers = narrow_helpers ? 1u : 0u;
        wp.narrow_stage_off = static_cast<uint32_t>((prof_elems + 127) & ~size_t(127));
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
        const uint32_t warps_per_cta = narrow_helpers ? 4 : wave_threads / 32;   // warps that take units
        const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(wave_sms, (n_units + warps_per_cta - 1) / warps_per_cta));
        const size_t wave_smem = narrow_helpers ? wp.narrow_stage_off + 4 * static_cast<size_t>(kNarrowPairBytes) : prof_elems;
        if ((st = launch_wavefront(db, wp, grid, wave_threads, wave_smem, any_narrow, any_rowblock, s)) != SWB_OK) return st;
        if (n_pipe_items) {
            // the wavefront kernel's SMs are free now: let them help with whatever pipeline items are left
            launch_pipeline(qp, pipe_ring_plan.slices, grid, pipe_smem, s);
            ++db->launches;
            SWB_CUDA(cudaStreamWaitEvent(s, db->ev_join, 0));
        }
    }
#ifdef SWB_PIPE_STATS
    if (packed && n_pipe_items)
        report_pipe_stats("pipeline", qp.stats, std::min<uint32_t>(static_cast<uint32_t>(db->sm_count) - (pipe_first ? wave_sms : 0), n_pipe_items),
                          n_tiles, s);
#endif
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
                if (p) dev_free(p);
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
        if (db->d_sort) dev_free(db->d_sort);
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
