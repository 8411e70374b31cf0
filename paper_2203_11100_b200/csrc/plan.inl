// plan.inl -- per-search decisions: arithmetic width, profile geometry, intra-task geometry (the division of the
// scan into kernels and units is scan_plan.hpp).
// Included by cabi.cu inside its anonymous namespace.

// Policy knobs (defaults + environment overrides), read once.
const ScanKnobs& scan_knobs() {
    static const ScanKnobs k = ScanKnobs::from_env();
    return k;
}

// Capacity of each border ring of the pipeline kernel next to a profile of `prof_elems` bytes; < 2: it cannot run.
PipeRings pipe_ring_chunks(const swb_db* db, size_t prof_elems) {
    return pipe_rings_for(prof_elems, db->smem_optin, sizeof(PipeCtl), static_cast<size_t>(kPipeWarps) * kPipeChunkBytes,
                          scan_knobs().pipe_ring_cap);
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
    pl.pstride = profile_stride(m, pl.tile);

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
