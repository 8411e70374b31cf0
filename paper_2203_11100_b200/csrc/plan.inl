// plan.inl -- per-search decisions: which kernel scans the database, profile geometry, unit policy knobs.
// Included by cabi.cu inside its anonymous namespace.

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

// The on-chip tile pipeline (pipeline.cuh) scans the database unless SWB200_PIPE=0.
bool pipe_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SWB200_PIPE");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

double env_number(const char* name, double fallback) {
    const char* e = std::getenv(name);
    const double v = e ? std::atof(e) : 0.0;
    return v > 0.0 ? v : fallback;
}

// Queries with fewer tiles than this stay with the wavefront kernel.
uint32_t pipe_min_tiles() {
    static const uint32_t v = static_cast<uint32_t>(env_number("SWB200_PIPE_MINTILES", 9));
    return v;
}

// A search is chain-bound when max_rows > this factor x a warp's fair share of the search (row-tiles).
double pipe_chain_factor() {
    static const double v = env_number("SWB200_PIPE_CHAIN", 1.2);
    return v;
}

// A group taller than this fraction of a CTA's fair share of rows stays with the wavefront kernel.
double pipe_tall_fraction() {
    static const double v = env_number("SWB200_PIPE_TALL", 0.35);
    return v;
}

double pipe_wave_margin_chain() {
    static const double v = env_number("SWB200_PIPE_WAVE_MARGIN_CHAIN", 2.0);
    return v;
}

// SMs for the wavefront kernel = its share of the rows x this margin (the one above when chain-bound).
double pipe_wave_margin() {
    static const double v = env_number("SWB200_PIPE_WAVE_MARGIN", 1.25);
    return v;
}

uint32_t pipe_lag_div() {
    static const uint32_t d = [] {
        const char* e = std::getenv("SWB200_PIPE_LAGDIV");
        const int v = e ? std::atoi(e) : 0;
        return v >= 1 ? static_cast<uint32_t>(v) : 24u;
    }();
    return d;
}

// Capacity of each border ring (chunks, a power of two) that fits next to the profile; < 2: the pipeline cannot run.
uint32_t pipe_ring_chunks(const swb_db* db, size_t prof_elems) {
    static const uint32_t cap = [] {
        const char* e = std::getenv("SWB200_PIPE_RING");
        const int v = e ? std::atoi(e) : 0;
        return v >= 2 ? static_cast<uint32_t>(v) : 4u;
    }();
    const size_t fixed = ((prof_elems + 255) & ~size_t(255)) + sizeof(PipeCtl);
    if (fixed >= db->smem_optin) return 0;
    const size_t room = (db->smem_optin - fixed) / (static_cast<size_t>(kPipeWarps) * kPipeChunkBytes);
    uint32_t c = 1;
    while (c * 2 <= room && c * 2 <= cap) c *= 2;
    return room >= 1 ? c : 0;
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
