// swsearch/gpu.hpp -- glue between the swsearch C++ API and the C-ABI of libswb200.so (include/swb200.h).
//
// New state the reference does not have: the packed, device-resident copy of a SequenceDatabase.  The reference's
// run_search takes the database by const reference on every call (scheduler.hpp:184) and re-partitions it each time
// (scheduler.hpp:189); packing and uploading 200 MB per query would dwarf the search, so the packed copy is cached
// per (database object, length_threshold) on first use and reused.  A database is "immutable after load"
// (sequence.hpp:28); a cheap fingerprint (addresses, totals, 64 fully hashed sample sequences) still guards against a
// re-allocated or re-filled object.  It cannot see an in-place edit of a residue outside the sample: a caller that
// edits a database calls gpu::release(db) afterwards, or sets SWB200_VERIFY_DB=1 to have every call hash every residue.
// At most SWB200_CACHE_ENTRIES (default 4) packed databases stay resident, least recently used out first.
//
//   SWB200_DEVICES   comma-separated CUDA device indices to shard over, or "all" (default: all visible devices)
//
// Nothing in here computes scores on the CPU; without a usable GPU every call throws std::runtime_error.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "swb200.h"
#include "swsearch/scoring.hpp"
#include "swsearch/sequence.hpp"

namespace swsearch::gpu {

/// Non-zero status -> the exception family the reference would have thrown (error conventions).
inline void check(swb_status status) {
    if (status == SWB_OK) return;
    const std::string message = swb_last_error();
    if (status == SWB_ERR_INVALID) throw std::invalid_argument(message);
    if (status == SWB_ERR_RANGE) throw std::out_of_range(message);
    throw std::runtime_error("swb200: " + message);
}

/// Devices searches are sharded over.
inline const std::vector<std::int32_t>& devices() {
    static const std::vector<std::int32_t> list = [] {
        std::int32_t visible = 0;
        check(swb_device_count(&visible));
        if (visible < 1) throw std::runtime_error("swb200: no CUDA device visible (there is no CPU fallback)");
        std::vector<std::int32_t> chosen;
        const char* env = std::getenv("SWB200_DEVICES");
        if (env != nullptr && *env != '\0' && std::string(env) != "all") {
            std::string item;
            for (const char* p = env;; ++p) {
                if (*p == ',' || *p == '\0') {
                    if (!item.empty()) chosen.push_back(static_cast<std::int32_t>(std::stoi(item)));
                    item.clear();
                    if (*p == '\0') break;
                } else {
                    item.push_back(*p);
                }
            }
        }
        if (chosen.empty())
            for (std::int32_t d = 0; d < visible; ++d) chosen.push_back(d);
        return chosen;
    }();
    return list;
}

inline const std::int32_t* matrix_table(const ScoringMatrix& matrix) { return matrix.row(0); }   // 576 contiguous scores

namespace detail {

struct Fingerprint {
    std::size_t count = 0;
    std::uint64_t residues = 0;
    std::uint64_t sample = 0;
    const void* storage = nullptr;
    bool operator==(const Fingerprint& o) const {
        return count == o.count && residues == o.residues && sample == o.sample && storage == o.storage;
    }
};

inline std::uint64_t mix(std::uint64_t h, std::uint64_t v) { return (h ^ v) * 1099511628211ull; }

inline std::uint64_t hash_codes(std::uint64_t h, const std::vector<std::uint8_t>& codes) {
    h = mix(h, codes.size());
    for (std::uint8_t c : codes) h = mix(h, c);
    return h;
}

// O(1) per call (it runs on every run_search): the element count, the address of the sequence array, the totals
// and a sample of 64 sequences -- their lengths, the addresses of their residues and their full contents.
inline Fingerprint fingerprint(const SequenceDatabase& db) {
    Fingerprint f;
    f.count = db.sequences.size();
    f.storage = db.sequences.data();
    f.residues = db.total_residues;
    f.sample = mix(1469598103934665603ull, db.max_length);
    const std::size_t stride = f.count / 64 + 1;
    for (std::size_t i = 0; i < f.count; i += stride) {
        const auto& codes = db.sequences[i].codes;
        f.sample = mix(f.sample, static_cast<std::uint64_t>(reinterpret_cast<std::uintptr_t>(codes.data())));
        f.sample = hash_codes(f.sample, codes);
    }
    return f;
}

// Every residue of the database (tens of milliseconds for Swiss-Prot): taken when a database is packed, and checked
// again on every call only when SWB200_VERIFY_DB=1 -- for callers that edit residues in place although a database
// is documented as immutable after load (sequence.hpp:28); everyone else calls gpu::release(db) after an edit.
inline std::uint64_t content_hash(const SequenceDatabase& db) {
    std::uint64_t h = 1469598103934665603ull;
    for (const auto& seq : db.sequences) h = hash_codes(h, seq.codes);
    return h;
}

inline bool verify_every_call() {
    static const bool on = [] {
        const char* e = std::getenv("SWB200_VERIFY_DB");
        return e != nullptr && *e == '1';
    }();
    return on;
}

inline std::size_t cache_capacity() {   // SWB200_CACHE_ENTRIES: packed databases kept resident at most (default 4)
    static const std::size_t cap = [] {
        const char* e = std::getenv("SWB200_CACHE_ENTRIES");
        const long v = e ? std::atol(e) : 0;
        return static_cast<std::size_t>(v > 0 ? v : 4);
    }();
    return cap;
}

struct Cached {
    swb_mdb* handle = nullptr;
    Fingerprint print;
    std::uint64_t content = 0;
    std::uint64_t last_use = 0;
};

// The registry is created on first use and never destroyed: its handles own CUDA streams, events and NCCL
// communicators, and tearing those down from a static destructor runs after the CUDA runtime may already be gone.
// The process exit reclaims the device memory; gpu::release / release_all free it earlier.
struct Registry {
    std::mutex lock;
    std::map<std::pair<const SequenceDatabase*, std::size_t>, Cached> entries;
    std::uint64_t clock = 0;
};

inline Registry& registry() {
    static Registry* instance = new Registry();
    return *instance;
}

}  // namespace detail

/// The packed multi-GPU copy of `db` for this threshold; built (packed, sharded, uploaded) on first use.  At most
/// cache_capacity() databases stay resident: the least recently used one is dropped when another is packed, so
/// temporaries (a loop or a property test creating databases at ever new addresses) cannot pile up on the device.
inline swb_mdb* resident(const SequenceDatabase& db, std::size_t length_threshold) {
    detail::Registry& reg = detail::registry();
    std::lock_guard<std::mutex> guard(reg.lock);
    const auto key = std::make_pair(&db, length_threshold);
    const detail::Fingerprint now = detail::fingerprint(db);
    auto found = reg.entries.find(key);
    if (found != reg.entries.end()) {
        if (found->second.print == now && (!detail::verify_every_call() || found->second.content == detail::content_hash(db))) {
            found->second.last_use = ++reg.clock;
            return found->second.handle;
        }
        swb_mdb_destroy(found->second.handle);      // the object changed under us: repack
        reg.entries.erase(found);
    }
    while (reg.entries.size() >= detail::cache_capacity()) {
        auto oldest = reg.entries.begin();
        for (auto it = reg.entries.begin(); it != reg.entries.end(); ++it)
            if (it->second.last_use < oldest->second.last_use) oldest = it;
        swb_mdb_destroy(oldest->second.handle);
        reg.entries.erase(oldest);
    }
    std::vector<const std::uint8_t*> rows(db.sequences.size());
    std::vector<std::uint32_t> lengths(db.sequences.size());
    for (std::size_t i = 0; i < rows.size(); ++i) {
        rows[i] = db.sequences[i].codes.data();
        lengths[i] = static_cast<std::uint32_t>(db.sequences[i].codes.size());
    }
    const auto& devs = devices();
    swb_mdb* handle = nullptr;
    check(swb_mdb_create(rows.data(), lengths.data(), static_cast<std::uint32_t>(rows.size()),
                         static_cast<std::uint64_t>(length_threshold), devs.data(),
                         static_cast<std::uint32_t>(devs.size()), &handle));
    reg.entries[key] = detail::Cached{handle, now, detail::verify_every_call() ? detail::content_hash(db) : 0, ++reg.clock};
    return handle;
}

/// A packed file written by `swsearch pack` / swb_pack_file stands in for `db`'s device copy: nothing is parsed,
/// sorted or packed (replaces fasta.hpp:80-86 + the pack for every run after the first).  `db` still supplies
/// headers and residues for reporting and must be the database the file was packed from (count is checked).
inline swb_mdb* attach_packed(const SequenceDatabase& db, std::size_t length_threshold, const std::string& path) {
    detail::Registry& reg = detail::registry();
    std::lock_guard<std::mutex> guard(reg.lock);
    const auto key = std::make_pair(&db, length_threshold);
    auto found = reg.entries.find(key);
    if (found != reg.entries.end()) {
        swb_mdb_destroy(found->second.handle);
        reg.entries.erase(found);
    }
    swb_mdb* handle = nullptr;
    check(swb_mdb_load(path.c_str(), devices().front(), &handle));
    swb_db_info info{};
    check(swb_db_info_get(swb_mdb_shard(handle, 0), &info));
    if (info.n_total != db.sequences.size() || info.length_threshold != length_threshold || info.shard_count != 1) {
        swb_mdb_destroy(handle);
        throw std::invalid_argument("packed database " + path + " does not belong to this database / threshold");
    }
    reg.entries[key] = detail::Cached{handle, detail::fingerprint(db), detail::verify_every_call() ? detail::content_hash(db) : 0, ++reg.clock};
    return handle;
}

/// Drop the device copy of one database (all thresholds) / of every database.
inline void release(const SequenceDatabase& db) {
    detail::Registry& reg = detail::registry();
    std::lock_guard<std::mutex> guard(reg.lock);
    for (auto it = reg.entries.begin(); it != reg.entries.end();) {
        if (it->first.first == &db) {
            swb_mdb_destroy(it->second.handle);
            it = reg.entries.erase(it);
        } else {
            ++it;
        }
    }
}

inline void release_all() {
    detail::Registry& reg = detail::registry();
    std::lock_guard<std::mutex> guard(reg.lock);
    for (auto& kv : reg.entries) swb_mdb_destroy(kv.second.handle);
    reg.entries.clear();
}

}  // namespace swsearch::gpu
