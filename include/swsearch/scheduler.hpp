// swsearch/scheduler.hpp -- database search (drop-in for the reference's scheduler.hpp:20-251).
//
// run_search keeps its signature and its contract -- the result equals a sequential scalar scan followed by the
// (score desc, index asc) sort and truncation to top_k, whatever the worker / lane / chunk settings
// (scheduler.hpp:179-183) -- but the region between "profile built" and "hits merged" (scheduler.hpp:189-244)
// runs on the GPUs: the database is packed once and kept resident (gpu.hpp), every search is one call into the C-ABI
// (swb_mdb_search), and the top-k comes back already ordered.  worker_count, lane_width, chunk_width and
// cpu_pool_threads are validated and otherwise ignored: they never changed results (scheduler.hpp:18-19).
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <vector>

#include "swsearch/align.hpp"
#include "swsearch/gpu.hpp"
#include "swsearch/scoring.hpp"
#include "swsearch/sequence.hpp"

namespace swsearch {

/// Search knobs.  Only top_k and length_threshold (which pool a sequence is accounted to) are semantically live.
struct SearchConfig {
    std::size_t worker_count = 1;
    std::size_t lane_width = 8;
    std::size_t chunk_width = 64;
    std::size_t length_threshold = 3000;   // residues; sequences this long or longer form the intra-task pool
    std::size_t top_k = 10;
    std::size_t cpu_pool_threads = 1;
    bool compute_alignments = true;
    std::size_t traceback_memory_cap = std::size_t{256} << 20;

    void validate() const {
        auto at_least_one = [](std::size_t v, const char* what) {
            if (v < 1) throw std::invalid_argument(std::string(what) + " must be >= 1");
        };
        at_least_one(worker_count, "worker_count");
        at_least_one(lane_width, "lane_width");
        at_least_one(chunk_width, "chunk_width");
        at_least_one(top_k, "top_k");
    }
};

enum class KernelRoute : std::uint8_t { inter_task, intra_task };

/// [begin, end) positions of one routing pool.
struct WorkChunk {
    std::uint32_t begin = 0;
    std::uint32_t end = 0;
    KernelRoute route = KernelRoute::inter_task;
};

/// Database indices by route: shorter than the threshold -> inter-task pool, otherwise intra-task pool.
struct DatabasePartition {
    std::vector<std::uint32_t> short_pool;
    std::vector<std::uint32_t> long_pool;
};

inline DatabasePartition partition_database(const SequenceDatabase& db, std::size_t threshold) {
    DatabasePartition pools;
    const auto count = static_cast<std::uint32_t>(db.num_sequences());
    for (std::uint32_t index = 0; index < count; ++index)
        (db.sequences[index].length() < threshold ? pools.short_pool : pools.long_pool).push_back(index);
    return pools;
}

/// A fixed list of chunks, each handed out exactly once to whoever asks first.
class ChunkQueue {
public:
    explicit ChunkQueue(std::vector<WorkChunk> chunks) : items_(std::move(chunks)) {}

    std::optional<WorkChunk> claim() {
        const std::size_t ticket = cursor_.fetch_add(1, std::memory_order_relaxed);
        if (ticket < items_.size()) return items_[ticket];
        return std::nullopt;
    }

    std::size_t size() const { return items_.size(); }

private:
    std::vector<WorkChunk> items_;
    std::atomic<std::size_t> cursor_{0};
};

/// One scored database sequence.  Equality ignores the alignment.
struct Hit {
    std::uint32_t db_index = 0;
    AlignScore score;
    std::optional<Alignment> alignment;

    bool operator==(const Hit& other) const { return db_index == other.db_index && score == other.score; }
};

/// Hits by score descending, then database index ascending, at most top_k of them.
struct RankedResults {
    std::vector<Hit> hits;

    bool operator==(const RankedResults& other) const { return hits == other.hits; }
};

/// Merge partial hit lists into the global order and truncate (host utility; the GPU search does not need it).
inline RankedResults merge_results(std::vector<std::vector<Hit>> partials, std::size_t top_k) {
    RankedResults merged;
    std::size_t total = 0;
    for (const auto& part : partials) total += part.size();
    merged.hits.reserve(total);
    for (auto& part : partials)
        for (Hit& hit : part) merged.hits.push_back(std::move(hit));
    auto ranks_before = [](const Hit& a, const Hit& b) {
        return a.score.value > b.score.value || (a.score.value == b.score.value && a.db_index < b.db_index);
    };
    const std::size_t keep = std::min(top_k, merged.hits.size());
    std::partial_sort(merged.hits.begin(), merged.hits.begin() + static_cast<std::ptrdiff_t>(keep), merged.hits.end(),
                      ranks_before);
    merged.hits.resize(keep);
    return merged;
}

/// How a search was executed.
struct SearchStats {
    std::size_t lane_scored = 0;        // sequences of the inter-task pool
    std::size_t wavefront_scored = 0;   // sequences of the intra-task pool
    std::size_t chunks_claimed = 0;     // work units handed out on the GPUs
};

namespace detail {

inline std::vector<WorkChunk> make_chunks(std::size_t pool_size, std::size_t chunk_len, KernelRoute route) {
    std::vector<WorkChunk> chunks;
    if (chunk_len == 0) return chunks;
    chunks.reserve((pool_size + chunk_len - 1) / chunk_len);
    for (std::size_t begin = 0; begin < pool_size; begin += chunk_len)
        chunks.push_back(WorkChunk{static_cast<std::uint32_t>(begin),
                                   static_cast<std::uint32_t>(std::min(pool_size, begin + chunk_len)), route});
    return chunks;
}

}  // namespace detail

namespace detail {

/// Tracebacks of all surviving hits, on the GPU, straight from the resident database (scheduler.hpp:246-249).
inline void attach_alignments(const EncodedSequence& query, const SequenceDatabase& db, const ScoringMatrix& matrix,
                              const GapModel& gaps, const SearchConfig& config, swb_mdb* resident, RankedResults& results) {
    if (config.compute_alignments && !results.hits.empty()) {
        // all surviving hits are traced back on the GPU in one go, straight from the resident database
        const std::size_t count = results.hits.size();
        std::vector<swb_hit> raw_hits(count);
        std::vector<std::uint64_t> offsets(count + 1, 0);
        for (std::size_t i = 0; i < count; ++i) {
            raw_hits[i] = swb_hit{results.hits[i].db_index, results.hits[i].score.value};
            offsets[i + 1] = offsets[i] + query.length() + db.sequences[results.hits[i].db_index].length();
        }
        std::vector<swb_alignment> raw(count);
        std::vector<std::uint8_t> scripts(std::max<std::uint64_t>(offsets[count], 1));
        gpu::check(swb_mdb_align_hits(resident, query.codes.data(), static_cast<std::uint32_t>(query.length()),
                                      gpu::matrix_table(matrix), gaps.open(), gaps.extend(), raw_hits.data(),
                                      static_cast<std::uint32_t>(count), config.traceback_memory_cap, raw.data(),
                                      scripts.data(), offsets.data()));
        for (std::size_t i = 0; i < count; ++i) {
            Alignment a;
            a.score = {raw[i].score};
            a.capped = raw[i].capped != 0;
            a.query_begin = raw[i].query_begin, a.query_end = raw[i].query_end;
            a.subject_begin = raw[i].subject_begin, a.subject_end = raw[i].subject_end;
            a.ops.resize(raw[i].n_ops);
            for (std::size_t k = 0; k < a.ops.size(); ++k) a.ops[k] = static_cast<EditOp>(scripts[offsets[i] + k]);
            results.hits[i].alignment = std::move(a);
        }
    }
}

}  // namespace detail

/// Search one query against the whole database on the GPUs.
inline RankedResults run_search(const EncodedSequence& query, const SequenceDatabase& db, const ScoringMatrix& matrix,
                                const GapModel& gaps, const SearchConfig& config, SearchStats* stats = nullptr) {
    config.validate();
    for (std::uint8_t code : query.codes)    // what QueryProfile's constructor rejects in the reference
        if (code >= ScoringMatrix::size) throw std::out_of_range("query code outside matrix alphabet");

    RankedResults results;
    swb_mdb* resident = gpu::resident(db, config.length_threshold);
    const std::size_t want = std::min<std::size_t>(config.top_k, db.num_sequences());
    if (want > 0) {
        std::vector<swb_hit> hits(want);
        std::uint32_t found = 0;
        swb_stats report{};
        gpu::check(swb_mdb_search(resident, query.codes.data(), static_cast<std::uint32_t>(query.length()),
                                  gpu::matrix_table(matrix), gaps.open(), gaps.extend(),
                                  static_cast<std::uint32_t>(want), hits.data(), &found, &report));
        results.hits.resize(found);
        for (std::uint32_t i = 0; i < found; ++i) {
            results.hits[i].db_index = hits[i].db_index;
            results.hits[i].score = {hits[i].score};
        }
        if (stats != nullptr) {
            stats->lane_scored += report.lane_scored;
            stats->wavefront_scored += report.wavefront_scored;
            stats->chunks_claimed += report.chunks_claimed;
        }
    }

    detail::attach_alignments(query, db, matrix, gaps, config, resident, results);
    return results;
}

/// Several queries against the same database: the same results as a loop over run_search (which is what the
/// reference's callers write), but issued to the GPU as one batch -- searches overlap each other's
/// host preparation, and the queries share database scans as two streams (swb_search_many; on every GPU at once
/// when the database is sharded over several, swb_mdb_search_many).
inline std::vector<RankedResults> run_search_batch(const std::vector<EncodedSequence>& queries, const SequenceDatabase& db,
                                                   const ScoringMatrix& matrix, const GapModel& gaps,
                                                   const SearchConfig& config, SearchStats* stats = nullptr) {
    config.validate();
    for (const EncodedSequence& query : queries)
        for (std::uint8_t code : query.codes)
            if (code >= ScoringMatrix::size) throw std::out_of_range("query code outside matrix alphabet");
    std::vector<RankedResults> all(queries.size());
    swb_mdb* resident = gpu::resident(db, config.length_threshold);
    const std::size_t want = std::min<std::size_t>(config.top_k, db.num_sequences());
    if (queries.empty()) return all;
    if (want == 0) {
        for (std::size_t q = 0; q < queries.size(); ++q) all[q] = run_search(queries[q], db, matrix, gaps, config, stats);
        return all;
    }
    std::vector<const std::uint8_t*> rows(queries.size());
    std::vector<std::uint32_t> lengths(queries.size());
    for (std::size_t q = 0; q < queries.size(); ++q) {
        rows[q] = queries[q].codes.data();
        lengths[q] = static_cast<std::uint32_t>(queries[q].length());
    }
    std::vector<swb_hit> hits(queries.size() * want);
    std::vector<std::uint32_t> found(queries.size(), 0);
    gpu::check(swb_mdb_search_many(resident, rows.data(), lengths.data(), static_cast<std::uint32_t>(queries.size()),
                                   gpu::matrix_table(matrix), gaps.open(), gaps.extend(), static_cast<std::uint32_t>(want),
                                   hits.data(), found.data(), nullptr));
    swb_db_info info{};   // counters for SearchStats: summed over the shards
    for (std::uint32_t r = 0; r < swb_mdb_shard_count(resident); ++r) {
        swb_db_info one{};
        gpu::check(swb_db_info_get(swb_mdb_shard(resident, r), &one));
        info.n_short += one.n_short, info.n_long += one.n_long, info.n_groups += one.n_groups;
    }
    for (std::size_t q = 0; q < queries.size(); ++q) {
        all[q].hits.resize(found[q]);
        for (std::uint32_t i = 0; i < found[q]; ++i) {
            all[q].hits[i].db_index = hits[q * want + i].db_index;
            all[q].hits[i].score = {hits[q * want + i].score};
        }
        if (stats != nullptr) {
            stats->lane_scored += info.n_short;
            stats->wavefront_scored += info.n_long;
            stats->chunks_claimed += info.n_groups;
        }
        detail::attach_alignments(queries[q], db, matrix, gaps, config, resident, all[q]);
    }
    return all;
}

}  // namespace swsearch
