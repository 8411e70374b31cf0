// tests/cpp/batch_unit.cpp -- GPU check of swsearch::run_search_batch: identical to a loop over run_search
// (ranked lists and edit scripts), on a database large enough for the queries to share scans.  Run a second time
// with SWB200_DEVICES=0,0 it covers the sharded flavour (swb_mdb_search_many).
#include <cstdio>
#include <random>

#include "swsearch/scheduler.hpp"

using namespace swsearch;

static EncodedSequence random_sequence(std::mt19937_64& rng, std::size_t n) {
    EncodedSequence s;
    s.codes.resize(n);
    for (auto& c : s.codes) c = static_cast<std::uint8_t>(rng() % 20);
    return s;
}

int main() {
    std::mt19937_64 rng(0x5357444200ull + 99);
    SequenceDatabase db;
    const std::size_t n = 24000;   // 375 groups of 64: more than two per SM, so the batch may pair queries
    db.sequences.reserve(n);
    for (std::size_t i = 0; i < n; ++i) {
        db.sequences.push_back(random_sequence(rng, 40 + rng() % 500));
        db.total_residues += db.sequences.back().length();
        db.max_length = std::max<std::size_t>(db.max_length, db.sequences.back().length());
    }
    std::vector<EncodedSequence> queries;
    for (std::size_t m : {300u, 330u, 90u, 700u, 650u, 0u, 1200u}) queries.push_back(random_sequence(rng, m));
    for (std::size_t q = 0; q < queries.size(); ++q)          // plant a copy of every query
        if (queries[q].length()) db.sequences[100 + 37 * q].codes = queries[q].codes;

    const ScoringMatrix& matrix = blosum62();
    const GapModel gaps(10, 2);
    int failures = 0;
    for (bool alignments : {false, true}) {
        SearchConfig config;
        config.top_k = 5;
        config.compute_alignments = alignments;
        SearchStats batch_stats, loop_stats;
        const std::vector<RankedResults> batch = run_search_batch(queries, db, matrix, gaps, config, &batch_stats);
        for (std::size_t q = 0; q < queries.size(); ++q) {
            const RankedResults one = run_search(queries[q], db, matrix, gaps, config, &loop_stats);
            bool same = one.hits.size() == batch[q].hits.size();
            for (std::size_t i = 0; same && i < one.hits.size(); ++i) {
                same = one.hits[i] == batch[q].hits[i];
                if (same && alignments)
                    same = one.hits[i].alignment.has_value() && batch[q].hits[i].alignment.has_value() &&
                           one.hits[i].alignment->ops == batch[q].hits[i].alignment->ops &&
                           one.hits[i].alignment->query_begin == batch[q].hits[i].alignment->query_begin &&
                           one.hits[i].alignment->subject_end == batch[q].hits[i].alignment->subject_end;
            }
            if (queries[q].length() && (one.hits.empty() || one.hits[0].db_index != 100 + 37 * q)) same = false;
            if (!same) {
                std::printf("FAIL: query %zu (m=%zu, alignments=%d)\n", q, queries[q].length(), int(alignments));
                ++failures;
            }
        }
        if (batch_stats.lane_scored != loop_stats.lane_scored || batch_stats.wavefront_scored != loop_stats.wavefront_scored) {
            std::printf("FAIL: stats differ\n");
            ++failures;
        }
    }
    gpu::release_all();
    std::printf(failures ? "batch_unit: %d failure(s)\n" : "batch_unit: ok\n", failures);
    return failures ? 1 : 0;
}
