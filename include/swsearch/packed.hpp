// swsearch/packed.hpp -- the packed on-disk database: what a process loads instead of parsing,
// encoding, sorting and packing a FASTA file again (the reference's load path, fasta.hpp:80-86, is single-threaded
// parse + encode on every start; the GPU drop-in adds a sort + interleave on top).
//
//   save_packed_database(db, path, threshold)   pack on the host, write residues + index tables + headers (no GPU)
//   load_packed_database(path, threshold*)      the SequenceDatabase back -- headers and residues de-interleaved
//                                               straight from the file, no text parsing
//   open_packed_database(path)                  load_packed_database + gpu::attach_packed: the file's residues go
//                                               from the mapping to the device as they are, run_search finds the
//                                               packed copy already resident
//
// The file format is documented in include/swb200.h (swb_pack_file); the device-side loader (swb_db_load) validates
// every table before anything reaches a kernel.
#pragma once

#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "swb200.h"
#include "swsearch/errors.hpp"
#include "swsearch/gpu.hpp"
#include "swsearch/sequence.hpp"

namespace swsearch {

namespace detail {
struct PackedHeader {   // the first 96 bytes of the file, little-endian (swb200.h)
    char magic[8];
    std::uint32_t version, n_total, n_local, n_short, n_long, shard_rank, shard_count, max_length;
    std::uint64_t residues, padded_rows, total_chunks, length_threshold, n_groups, codes_bytes, names_bytes;
};
static_assert(sizeof(PackedHeader) == 96, "packed file header");
struct PackedGroup {
    std::uint64_t chunk_base;
    std::uint32_t n_chunks, first_slot;
};
}  // namespace detail

/// Pack `db` for the given routing threshold and write it, headers included.  Host only.
inline void save_packed_database(const SequenceDatabase& db, const std::filesystem::path& path, std::size_t length_threshold) {
    std::vector<const std::uint8_t*> rows(db.sequences.size());
    std::vector<std::uint32_t> lengths(db.sequences.size());
    std::vector<const char*> names(db.sequences.size());
    for (std::size_t i = 0; i < rows.size(); ++i) {
        rows[i] = db.sequences[i].codes.data();
        lengths[i] = static_cast<std::uint32_t>(db.sequences[i].codes.size());
        names[i] = db.sequences[i].header.c_str();
    }
    const swb_status st = swb_pack_file(rows.data(), lengths.data(), static_cast<std::uint32_t>(rows.size()),
                                        static_cast<std::uint64_t>(length_threshold), 0, 1, names.data(), path.string().c_str());
    if (st == SWB_ERR_INVALID && std::string(swb_last_error()).rfind("cannot open", 0) == 0) throw io_error(swb_last_error());
    if (st == SWB_ERR_INVALID && std::string(swb_last_error()).rfind("short write", 0) == 0) throw io_error(swb_last_error());
    gpu::check(st);
}

/// The database a packed file was made from: same sequences in the same order, same headers.
inline SequenceDatabase load_packed_database(const std::filesystem::path& path, std::size_t* length_threshold = nullptr) {
    std::ifstream file(path, std::ios::binary);
    if (!file) throw io_error("cannot open " + path.string());
    detail::PackedHeader h{};
    file.read(reinterpret_cast<char*>(&h), sizeof(h));
    if (!file || std::memcmp(h.magic, "SWB200DB", 8) != 0 || h.version != 2)
        throw format_error(path.string() + " is not a swb200 packed database (version 2)");
    if (h.shard_count != 1 || h.n_local != h.n_total)
        throw format_error(path.string() + " holds one shard of a database, not a whole one");
    const std::uint64_t n_slots = h.n_groups * 64;
    const std::uint64_t size = std::filesystem::file_size(path);
    const std::uint64_t tables = sizeof(h) + h.n_groups * sizeof(detail::PackedGroup) + 2 * n_slots * 4 + h.codes_bytes;
    if (h.codes_bytes != h.total_chunks * 512 || tables > size || size - tables != h.names_bytes ||
        (h.names_bytes != 0 && h.names_bytes < (std::uint64_t(h.n_total) + 1) * 8))
        throw format_error(path.string() + ": sizes in the header do not match the file");
    std::vector<detail::PackedGroup> groups(h.n_groups);
    std::vector<std::uint32_t> slot_index(n_slots), slot_len(n_slots);
    std::vector<std::uint8_t> codes(h.codes_bytes);
    file.read(reinterpret_cast<char*>(groups.data()), static_cast<std::streamsize>(groups.size() * sizeof(detail::PackedGroup)));
    file.read(reinterpret_cast<char*>(slot_index.data()), static_cast<std::streamsize>(n_slots * 4));
    file.read(reinterpret_cast<char*>(slot_len.data()), static_cast<std::streamsize>(n_slots * 4));
    file.read(reinterpret_cast<char*>(codes.data()), static_cast<std::streamsize>(codes.size()));
    std::vector<std::uint64_t> name_off;
    std::string blob;
    if (h.names_bytes) {
        name_off.resize(std::size_t(h.n_total) + 1);
        file.read(reinterpret_cast<char*>(name_off.data()), static_cast<std::streamsize>(name_off.size() * 8));
        blob.resize(h.names_bytes - name_off.size() * 8);
        file.read(blob.data(), static_cast<std::streamsize>(blob.size()));
    }
    if (!file) throw io_error(path.string() + ": read failure");

    SequenceDatabase db;
    db.sequences.resize(h.n_total);
    std::vector<bool> filled(h.n_total, false);
    for (std::uint64_t slot = 0; slot < n_slots; ++slot) {
        const std::uint32_t idx = slot_index[slot], len = slot_len[slot];
        if (idx == 0xFFFFFFFFu) continue;
        const detail::PackedGroup& g = groups[slot / 64];
        if (idx >= h.n_total || filled[idx] || len > std::uint64_t(g.n_chunks) * 8 || (g.chunk_base + g.n_chunks) * 512 > codes.size())
            throw format_error(path.string() + ": damaged index tables");
        filled[idx] = true;
        // residue r of slot s: codes[((chunk_base + r/8)*32 + s%32)*16 + (s/32)*8 + r%8]
        const std::uint32_t s = static_cast<std::uint32_t>(slot % 64);
        const std::uint8_t* src = codes.data() + (g.chunk_base * 32 + s % 32) * 16 + (s / 32) * 8;
        auto& out = db.sequences[idx].codes;
        out.resize(len);
        for (std::uint32_t r0 = 0; r0 < len; r0 += 8)
            std::memcpy(out.data() + r0, src + std::size_t(r0 / 8) * 512, std::min<std::uint32_t>(8, len - r0));
        db.total_residues += len;
        if (len > db.max_length) db.max_length = len;
    }
    for (std::uint32_t i = 0; i < h.n_total; ++i) {
        if (!filled[i]) throw format_error(path.string() + ": a sequence is missing from the index tables");
        if (!name_off.empty()) {
            if (name_off[i + 1] < name_off[i] || name_off[i + 1] > blob.size()) throw format_error(path.string() + ": damaged names section");
            db.sequences[i].header.assign(blob, name_off[i], name_off[i + 1] - name_off[i]);
        }
    }
    if (length_threshold != nullptr) *length_threshold = static_cast<std::size_t>(h.length_threshold);
    return db;
}

/// Host copy + device copy from one file.  The database is returned behind a pointer because the resident cache is
/// keyed by the object's address (gpu.hpp); searches must use config.length_threshold == *length_threshold.
inline std::unique_ptr<SequenceDatabase> open_packed_database(const std::filesystem::path& path, std::size_t* length_threshold = nullptr) {
    std::size_t threshold = 0;
    auto db = std::make_unique<SequenceDatabase>(load_packed_database(path, &threshold));
    gpu::attach_packed(*db, threshold, path.string());
    if (length_threshold != nullptr) *length_threshold = threshold;
    return db;
}

}  // namespace swsearch
