// persist.inl -- the packed shard as a versioned file (swb_db_save / swb_db_load).  Included by cabi.cu inside extern "C".
// Replaces the reference's load path for repeated runs (fasta.hpp:80-86: parse + encode, single-threaded) -- SURVEY 8(f) rank 4.

namespace {
struct PackedFileHeader {
    char magic[8];              // "SWB200DB"
    uint32_t version;           // 2
    uint32_t n_total, n_local, n_short, n_long, shard_rank, shard_count, max_length;
    uint64_t residues, padded_rows, total_chunks, length_threshold, n_groups, codes_bytes;
    uint64_t names_bytes;       // optional trailing section: uint64 offsets[n_total + 1], then the sequence headers (0: none)
};
constexpr uint32_t kPackedFileVersion = 2;
static_assert(sizeof(PackedFileHeader) == 96, "packed file header layout (include/swsearch/packed.hpp reads the same bytes)");
}  // namespace

namespace {
swb_status write_packed(const PackedDb& m, const uint8_t* codes, const char* const* names, const char* path) {
    PackedFileHeader h{};
    std::memcpy(h.magic, "SWB200DB", 8);
    h.version = kPackedFileVersion;
    h.n_total = m.n_total, h.n_local = m.n_local, h.n_short = m.n_short, h.n_long = m.n_long;
    h.shard_rank = m.shard_rank, h.shard_count = m.shard_count, h.max_length = m.max_length;
    h.residues = m.residues, h.padded_rows = m.padded_rows, h.total_chunks = m.total_chunks;
    h.length_threshold = m.length_threshold, h.n_groups = m.groups.size();
    h.codes_bytes = static_cast<uint64_t>(m.total_chunks) * 32 * 16;
    std::vector<uint64_t> name_off;
    if (names) {
        name_off.assign(static_cast<size_t>(m.n_total) + 1, 0);
        for (uint32_t i = 0; i < m.n_total; ++i) name_off[i + 1] = name_off[i] + (names[i] ? std::strlen(names[i]) : 0);
        h.names_bytes = name_off.size() * sizeof(uint64_t) + name_off.back();
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) return fail(SWB_ERR_INVALID, std::string("cannot open ") + path + " for writing");
    bool ok = std::fwrite(&h, sizeof(h), 1, f) == 1;
    auto put = [&](const void* data, size_t bytes) { ok = ok && (bytes == 0 || std::fwrite(data, 1, bytes, f) == bytes); };
    put(m.groups.data(), m.groups.size() * sizeof(GroupDesc));
    put(m.slot_index.data(), m.slot_index.size() * sizeof(uint32_t));
    put(m.slot_len.data(), m.slot_len.size() * sizeof(uint32_t));
    put(codes, h.codes_bytes);
    if (names) {
        put(name_off.data(), name_off.size() * sizeof(uint64_t));
        for (uint32_t i = 0; i < m.n_total; ++i) put(names[i], static_cast<size_t>(name_off[i + 1] - name_off[i]));
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return fail(SWB_ERR_INVALID, std::string("short write to ") + path);
    return SWB_OK;
}

swb_status pack_to_file(const SeqSource& src, uint64_t threshold, uint32_t rank, uint32_t count, const char* const* names,
                        const char* path) {
    if (!path) return fail(SWB_ERR_INVALID, "path is null");
    try {
        PackedDb m;
        bool bad = false;
        const std::string err = pack_database(src, threshold, rank, count, m, &bad);
        if (!err.empty()) return fail(bad ? SWB_ERR_RANGE : SWB_ERR_INVALID, err);
        return write_packed(m, m.codes.data(), names, path);
    } catch (const std::bad_alloc&) {
        return fail(SWB_ERR_INTERNAL, "out of host memory packing the database");
    }
}
}  // namespace

swb_status swb_db_save(swb_db* db, const char* path) {
    if (!db || !path) return fail(SWB_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lock(db->mu);
    DeviceGuard guard(db->device);
    const size_t bytes = static_cast<size_t>(db->meta.total_chunks) * 32 * 16;
    try {
        std::vector<uint8_t> codes(bytes);
        if (bytes) SWB_CUDA(cudaMemcpy(codes.data(), db->d_codes, bytes, cudaMemcpyDeviceToHost));
        return write_packed(db->meta, codes.data(), nullptr, path);
    } catch (const std::bad_alloc&) {
        return fail(SWB_ERR_INTERNAL, "out of host memory saving the database");
    }
}

// Pack on the host and write the file, without touching a GPU (the `swsearch pack` command; a build machine needs no
// device).  Same layout and content as swb_db_create + swb_db_save.
swb_status swb_pack_file(const uint8_t* const* seqs, const uint32_t* lens, uint32_t n, uint64_t length_threshold,
                         uint32_t shard_rank, uint32_t shard_count, const char* const* names, const char* path) {
    if (n && (!seqs || !lens)) return fail(SWB_ERR_INVALID, "seqs/lens are null");
    static const uint8_t* const kNoPtrs[1] = {nullptr};
    static const uint32_t kNoLens[1] = {0};
    SeqSource src;
    src.ptrs = n ? seqs : kNoPtrs;
    src.lens = n ? lens : kNoLens;
    src.n = n;
    return pack_to_file(src, length_threshold, shard_rank, shard_count, names, path);
}

swb_status swb_pack_file_flat(const uint8_t* codes, const uint64_t* offsets, uint32_t n, uint64_t length_threshold,
                              uint32_t shard_rank, uint32_t shard_count, const char* const* names, const char* path) {
    if (!offsets) return fail(SWB_ERR_INVALID, "offsets is null");
    if (n && offsets[n] && !codes) return fail(SWB_ERR_INVALID, "codes is null");
    for (uint32_t i = 0; i < n; ++i)
        if (offsets[i + 1] < offsets[i]) return fail(SWB_ERR_INVALID, "offsets must be non-decreasing");
    SeqSource src;
    src.flat = codes;
    src.offsets = offsets;
    src.n = n;
    return pack_to_file(src, length_threshold, shard_rank, shard_count, names, path);
}

// Loading trusts nothing it has not checked: the file is mapped read-only, its size must match what the header
// implies (which also bounds every table by the file size), every table is validated against the invariants the
// kernels rely on, and the counters of the header are recomputed from the tables and must agree -- a stale or damaged
// file is rejected instead of producing out-of-bounds accesses or wrapped int16 scores (an understated max_length
// would skip the int32 re-run).  The residues go from the mapping straight to the device.
swb_status swb_db_load(const char* path, int32_t device, swb_db** out) {
    if (!path || !out) return fail(SWB_ERR_INVALID, "null argument");
    *out = nullptr;
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) return fail(SWB_ERR_INVALID, std::string("cannot open ") + path);
    struct stat sb {};
    if (::fstat(fd, &sb) != 0 || sb.st_size < static_cast<off_t>(sizeof(PackedFileHeader))) {
        ::close(fd);
        return fail(SWB_ERR_INVALID, std::string(path) + " is not a valid swb200 packed database (too short)");
    }
    const size_t file_bytes = static_cast<size_t>(sb.st_size);
    void* map = ::mmap(nullptr, file_bytes, PROT_READ, MAP_PRIVATE, fd, 0);
    ::close(fd);
    if (map == MAP_FAILED) return fail(SWB_ERR_INVALID, std::string("cannot map ") + path);
    ::madvise(map, file_bytes, MADV_SEQUENTIAL);
    struct Unmap {
        void* p;
        size_t n;
        ~Unmap() { ::munmap(p, n); }
    } unmap{map, file_bytes};
    const uint8_t* base = static_cast<const uint8_t*>(map);
    auto invalid = [&](const char* why) {
        return fail(SWB_ERR_INVALID, std::string(path) + " is not a valid swb200 packed database (version 2): " + why);
    };

    PackedFileHeader h;
    std::memcpy(&h, base, sizeof(h));
    if (std::memcmp(h.magic, "SWB200DB", 8) != 0 || h.version != kPackedFileVersion) return invalid("magic / version");
    // sizes: everything is bounded by the file size before anything is allocated
    if (h.n_groups > file_bytes / sizeof(GroupDesc) || h.total_chunks > file_bytes / 512) return invalid("table sizes beyond the file");
    const uint64_t n_slots = h.n_groups * kGroupSeqs;
    const uint64_t tables = sizeof(PackedFileHeader) + h.n_groups * sizeof(GroupDesc) + 2 * n_slots * sizeof(uint32_t) + h.total_chunks * 512;
    if (h.codes_bytes != h.total_chunks * 512 || tables > file_bytes || file_bytes - tables != h.names_bytes || n_slots > 0xFFFFFFFFull)
        return invalid("sizes do not add up");
    if (h.names_bytes && h.names_bytes < (static_cast<uint64_t>(h.n_total) + 1) * sizeof(uint64_t)) return invalid("names section too short");
    if (h.shard_count < 1 || h.shard_rank >= h.shard_count) return invalid("shard rank / count");
    const GroupDesc* groups = reinterpret_cast<const GroupDesc*>(base + sizeof(PackedFileHeader));
    const uint32_t* slot_index = reinterpret_cast<const uint32_t*>(groups + h.n_groups);
    const uint32_t* slot_len = slot_index + n_slots;
    const uint8_t* codes = reinterpret_cast<const uint8_t*>(slot_len + n_slots);

    swb_db* db = nullptr;
    try {
        // groups: contiguous chunks, slots in order, longest first (the kernels size borders by groups[0] and the
        // ticket order relies on it)
        uint64_t chunks = 0, padded_rows = 0;
        for (uint64_t g = 0; g < h.n_groups; ++g) {
            const GroupDesc& gd = groups[g];
            if (gd.chunk_base != chunks || gd.first_slot != g * kGroupSeqs) return invalid("group table is not contiguous");
            if (g && gd.n_chunks > groups[g - 1].n_chunks) return invalid("groups are not sorted longest first");
            chunks += gd.n_chunks;
            padded_rows += static_cast<uint64_t>(gd.n_chunks) * kRowsPerChunk;
        }
        if (chunks != h.total_chunks) return invalid("chunk count");
        // slots: every db_index at most once and below n_total; lengths within the group's rows
        std::vector<uint8_t> seen((static_cast<size_t>(h.n_total) + 7) / 8, 0);
        uint64_t n_local = 0, n_short = 0, n_long = 0, residues = 0;
        uint32_t max_length = 0;
        for (uint64_t slot = 0; slot < n_slots; ++slot) {
            const uint32_t idx = slot_index[slot], len = slot_len[slot];
            const uint64_t rows = static_cast<uint64_t>(groups[slot / kGroupSeqs].n_chunks) * kRowsPerChunk;
            if (idx == kNoSequence) {
                if (len != 0) return invalid("an unused slot has a length");
                continue;
            }
            if (idx >= h.n_total) return invalid("db_index beyond n_total");
            if (seen[idx >> 3] & (1u << (idx & 7))) return invalid("a db_index occurs twice");
            seen[idx >> 3] |= static_cast<uint8_t>(1u << (idx & 7));
            if (len > rows) return invalid("a sequence is longer than its group's rows");
            ++n_local;
            (len < h.length_threshold ? n_short : n_long) += 1;
            residues += len;
            max_length = std::max(max_length, len);
        }
        // the header's counters are derived data: recomputed, and a disagreement means a stale or edited file
        if (n_local != h.n_local || n_short != h.n_short || n_long != h.n_long || residues != h.residues ||
            max_length != h.max_length || padded_rows != h.padded_rows)
            return invalid("header counters disagree with the tables");
        // residue codes index the 25-row profile in shared memory
        uint8_t worst = 0;
        for (uint64_t i = 0; i < h.codes_bytes; ++i) worst = std::max(worst, codes[i]);
        if (worst > kPadCode) return invalid("residue code beyond the alphabet");

        // the file is sound; from here on a device is needed (host-only validation above is what the CPU tests reach)
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            return fail(SWB_ERR_CUDA, "no CUDA device available (this library has no CPU fallback)");
        if (device < 0 || device >= ndev) return fail(SWB_ERR_INVALID, "device index out of range");
        db = new swb_db();
        db->device = device;
        PackedDb& m = db->meta;
        m.n_total = h.n_total, m.n_local = h.n_local, m.n_short = h.n_short, m.n_long = h.n_long;
        m.shard_rank = h.shard_rank, m.shard_count = h.shard_count, m.max_length = max_length;
        m.residues = residues, m.padded_rows = padded_rows, m.total_chunks = h.total_chunks;
        m.length_threshold = h.length_threshold;
        m.groups.assign(groups, groups + h.n_groups);
        m.slot_index.assign(slot_index, slot_index + n_slots);
        m.slot_len.assign(slot_len, slot_len + n_slots);
    } catch (const std::bad_alloc&) {
        delete db;
        return fail(SWB_ERR_INTERNAL, std::string("out of host memory loading ") + path);
    }

    DeviceGuard guard(device);
    cudaDeviceProp prop{};
    swb_status st = SWB_OK;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) st = fail(SWB_ERR_CUDA, "cudaGetDeviceProperties failed");
    if (st == SWB_OK && prop.major < 10) st = fail(SWB_ERR_CUDA, "device is not sm_100-class; this library is built for sm_100a only");
    if (st == SWB_OK) {
        db->sm_count = prop.multiProcessorCount;
        db->smem_optin = prop.sharedMemPerBlockOptin;
        st = init_handle_resources(db);
    }
    if (st == SWB_OK) st = upload_db(db, codes, h.codes_bytes);
    if (st != SWB_OK) {
        const std::string keep = g_error;
        swb_db_destroy(db);
        g_error = keep;
        return st;
    }
    *out = db;
    return SWB_OK;
}
