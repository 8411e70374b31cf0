// swsearch/gpu.hpp -- glue between the swsearch C++ API and the C-ABI of libswb200.so (include/swb200.h).
//
// New state the reference does not have: the packed, device-resident copy of a SequenceDatabase.  The reference's
// run_search takes the database by const reference on every call (scheduler.hpp:184) and re-partitions it each time
// (scheduler.hpp:189); packing and uploading 200 MB per query would dwarf the search, so the packed copy is cached
// per (database object, length_threshold) on first use and reused.  A database is "immutable after load"
// (sequence.hpp:28); a cheap fingerprint still guards against a mutated or re-allocated object.
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

// O(1) per call (it runs on every run_search): the element count, the address of the sequence array and a
// sample of 64 sequences (length, first and last residue, address of the residues).
inline Fingerprint fingerprint(const SequenceDatabase& db) {
    Fingerprint f;
    f.count = db.sequences.size();
    f.storage = db.sequences.data();
    f.residues = db.total_residues;
    const std::size_t stride = f.count / 64 + 1;
    for (std::size_t i = 0; i < f.count; i += stride) {
        const auto& codes = db.sequences[i].codes;
        f.sample = f.sample * 1099511628211ull + codes.size() * 131u +
                   static_cast<std::uint64_t>(reinterpret_cast<std::uintptr_t>(codes.data()));
        if (!codes.empty()) f.sample = f.sample * 31u + codes.front() * 7u + codes.back();
    }
    return f;
}

struct Cached {
    swb_mdb* handle = nullptr;
    Fingerprint print;
};

struct Registry {
    std::mutex lock;
    std::map<std::pair<const SequenceDatabase*, std::size_t>, Cached> entries;
    ~Registry() {
        for (auto& kv : entries) swb_mdb_destroy(kv.second.handle);
    }
};

inline Registry& registry() {
    static Registry instance;
    return instance;
}

}  // namespace detail

/// The packed multi-GPU copy of `db` for this threshold; built (packed, sharded, uploaded) on first use.
inline swb_mdb* resident(const SequenceDatabase& db, std::size_t length_threshold) {
    detail::Registry& reg = detail::registry();
    std::lock_guard<std::mutex> guard(reg.lock);
    const auto key = std::make_pair(&db, length_threshold);
    const detail::Fingerprint now = detail::fingerprint(db);
    auto found = reg.entries.find(key);
    if (found != reg.entries.end()) {
        if (found->second.print == now) return found->second.handle;
        swb_mdb_destroy(found->second.handle);      // the object changed under us: repack
        reg.entries.erase(found);
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
    reg.entries[key] = detail::Cached{handle, now};
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
