// persist.inl -- the packed shard as a versioned file (swb_db_save / swb_db_load).  Included by cabi.cu inside extern "C".

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
