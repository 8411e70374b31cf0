// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI window onto the *unmodified* reference implementation.  It is compiled straight from
// the headers where they lie (/root/reference/proj/include/swsearch/*.hpp, force-including
// oracle/ref_compat.h for the one construct g++ rejects) into oracle/_ref/libswref.so by
// oracle/Makefile.  Nothing of the reference is copied into this repository; this file only
// *calls* it.  Users: tests/ (to pin the C restatement in oracle/sw_oracle.c and the CUDA path),
// tests/golden/make_golden.py (fixture generation) and bench.py's cpu_baseline / --impl reference
// leg.  The product library (libswb200.so) never links or loads this.
//
// Every export returns 0 on success; 1 = std::invalid_argument, 2 = std::out_of_range,
// 3 = anything else.  The message is kept per thread (swref_last_error).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "swsearch/align.hpp"
#include "swsearch/scheduler.hpp"
#include "swsearch/scoring.hpp"
#include "swsearch/sequence.hpp"

namespace {

thread_local std::string g_error;

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_error.clear();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_error = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_error = e.what();
        return 3;
    } catch (...) {
        g_error = "unknown exception";
        return 3;
    }
}

swsearch::ScoringMatrix matrix_from(const std::int32_t* table) {
    swsearch::ScoringMatrix mat("shim");
    for (unsigned a = 0; a < 24; ++a)
        for (unsigned b = 0; b < 24; ++b)
            mat.set(static_cast<std::uint8_t>(a), static_cast<std::uint8_t>(b), table[a * 24 + b]);
    return mat;
}

swsearch::EncodedSequence seq_from(const std::uint8_t* codes, std::uint64_t len) {
    swsearch::EncodedSequence s;
    if (len) s.codes.assign(codes, codes + len);
    return s;
}

}  // namespace

extern "C" {

const char* swref_last_error() { return g_error.c_str(); }

// The reference's built-in table (scoring.hpp:65-101), so fixtures never retype it.
int swref_blosum62(std::int32_t* out576) {
    return guarded([&] {
        const swsearch::ScoringMatrix& mat = swsearch::blosum62();
        for (unsigned a = 0; a < 24; ++a)
            for (unsigned b = 0; b < 24; ++b)
                out576[a * 24 + b] = mat.score(static_cast<std::uint8_t>(a), static_cast<std::uint8_t>(b));
    });
}

// align.hpp:69-78
int swref_score_scalar(const std::uint8_t* q, std::uint32_t m, const std::uint8_t* s, std::uint32_t n,
                       const std::int32_t* matrix, std::int32_t open, std::int32_t extend,
                       std::int32_t* out) {
    return guarded([&] {
        const auto mat = matrix_from(matrix);
        const swsearch::GapModel gaps(open, extend);
        *out = swsearch::sw_score_scalar(seq_from(q, m), seq_from(s, n), mat, gaps).value;
    });
}

// align.hpp:91-159.  subjects[i] may be null (a padding lane).  out has lane_width entries.
int swref_score_batch(const std::uint8_t* q, std::uint32_t m, const std::uint8_t* const* subjects,
                      const std::uint32_t* lens, std::uint32_t count, std::uint32_t lane_width,
                      const std::int32_t* matrix, std::int32_t open, std::int32_t extend,
                      std::int32_t* out) {
    return guarded([&] {
        const auto mat = matrix_from(matrix);
        const swsearch::GapModel gaps(open, extend);
        const auto profile = swsearch::make_profile(mat, seq_from(q, m));
        std::vector<swsearch::EncodedSequence> owned(count);
        swsearch::LaneBatch batch;
        batch.lane_width = lane_width;
        for (std::uint32_t i = 0; i < count; ++i) {
            if (subjects[i]) {
                owned[i] = seq_from(subjects[i], lens[i]);
                batch.subjects.push_back(&owned[i]);
            } else {
                batch.subjects.push_back(nullptr);
            }
        }
        const auto scores = swsearch::sw_score_batch(profile, batch, gaps);
        for (std::size_t i = 0; i < scores.size(); ++i) out[i] = scores[i].value;
    });
}

// align.hpp:166-229
int swref_score_wavefront(const std::uint8_t* q, std::uint32_t m, const std::uint8_t* s,
                          std::uint32_t n, const std::int32_t* matrix, std::int32_t open,
                          std::int32_t extend, std::uint64_t chunk_width, std::int32_t* out) {
    return guarded([&] {
        const auto mat = matrix_from(matrix);
        const swsearch::GapModel gaps(open, extend);
        *out = swsearch::sw_score_wavefront(seq_from(q, m), seq_from(s, n), mat, gaps, chunk_width)
                   .value;
    });
}

// sequence.hpp:30-35 -- a database built from flat codes + (n+1) offsets.
void* swref_db_create(const std::uint8_t* codes, const std::uint64_t* offsets, std::uint32_t n) {
    auto* db = new swsearch::SequenceDatabase();
    db->sequences.resize(n);
    for (std::uint32_t i = 0; i < n; ++i) {
        const std::uint64_t len = offsets[i + 1] - offsets[i];
        if (len) db->sequences[i].codes.assign(codes + offsets[i], codes + offsets[i + 1]);
        db->total_residues += len;
        db->max_length = std::max<std::size_t>(db->max_length, len);
    }
    return db;
}

void swref_db_destroy(void* db) { delete static_cast<swsearch::SequenceDatabase*>(db); }

// scheduler.hpp:184-251 with compute_alignments=false (the timed region).
// stats3 = {lane_scored, wavefront_scored, chunks_claimed}; out_* hold up to top_k entries.
int swref_run_search(void* dbh, const std::uint8_t* q, std::uint32_t m, const std::int32_t* matrix,
                     std::int32_t open, std::int32_t extend, std::uint64_t worker_count,
                     std::uint64_t lane_width, std::uint64_t chunk_width,
                     std::uint64_t length_threshold, std::uint64_t top_k,
                     std::uint64_t cpu_pool_threads, std::uint32_t* out_index,
                     std::int32_t* out_score, std::uint32_t* out_count, std::uint64_t* stats3) {
    return guarded([&] {
        const auto& db = *static_cast<swsearch::SequenceDatabase*>(dbh);
        const auto mat = matrix_from(matrix);
        const swsearch::GapModel gaps(open, extend);
        swsearch::SearchConfig cfg;
        cfg.worker_count = worker_count;
        cfg.lane_width = lane_width;
        cfg.chunk_width = chunk_width;
        cfg.length_threshold = length_threshold;
        cfg.top_k = top_k;
        cfg.cpu_pool_threads = cpu_pool_threads;
        cfg.compute_alignments = false;
        swsearch::SearchStats st;
        const auto res = swsearch::run_search(seq_from(q, m), db, mat, gaps, cfg, &st);
        *out_count = static_cast<std::uint32_t>(res.hits.size());
        for (std::size_t i = 0; i < res.hits.size(); ++i) {
            out_index[i] = res.hits[i].db_index;
            out_score[i] = res.hits[i].score.value;
        }
        if (stats3) {
            stats3[0] = st.lane_scored;
            stats3[1] = st.wavefront_scored;
            stats3[2] = st.chunks_claimed;
        }
    });
}

// scheduler.hpp:106-117 on (index, score) partial lists laid end to end; part_sizes has n_parts entries.
int swref_merge_results(const std::uint32_t* index, const std::int32_t* score,
                        const std::uint64_t* part_sizes, std::uint32_t n_parts, std::uint64_t top_k,
                        std::uint32_t* out_index, std::int32_t* out_score, std::uint64_t* out_count) {
    return guarded([&] {
        std::vector<std::vector<swsearch::Hit>> partials(n_parts);
        std::size_t pos = 0;
        for (std::uint32_t p = 0; p < n_parts; ++p)
            for (std::uint64_t i = 0; i < part_sizes[p]; ++i, ++pos)
                partials[p].push_back({index[pos], {score[pos]}, std::nullopt});
        const auto res = swsearch::merge_results(std::move(partials), top_k);
        *out_count = res.hits.size();
        for (std::size_t i = 0; i < res.hits.size(); ++i) {
            out_index[i] = res.hits[i].db_index;
            out_score[i] = res.hits[i].score.value;
        }
    });
}

// align.hpp:254-353.  bounds4 = {query_begin, query_end, subject_begin, subject_end};
// ops receives at most ops_cap edit ops (align.hpp:236 numbering); *n_ops is the true count.
int swref_traceback(const std::uint8_t* q, std::uint32_t m, const std::uint8_t* s, std::uint32_t n,
                    const std::int32_t* matrix, std::int32_t open, std::int32_t extend,
                    std::uint64_t memory_cap, std::uint64_t* bounds4, std::int32_t* score,
                    std::int32_t* capped, std::uint8_t* ops, std::uint64_t ops_cap,
                    std::uint64_t* n_ops, std::int32_t* rescored) {
    return guarded([&] {
        const auto mat = matrix_from(matrix);
        const swsearch::GapModel gaps(open, extend);
        const auto qs = seq_from(q, m);
        const auto ss = seq_from(s, n);
        const auto al = swsearch::sw_align_traceback(qs, ss, mat, gaps, memory_cap);
        bounds4[0] = al.query_begin;
        bounds4[1] = al.query_end;
        bounds4[2] = al.subject_begin;
        bounds4[3] = al.subject_end;
        *score = al.score.value;
        *capped = al.capped ? 1 : 0;
        *n_ops = al.ops.size();
        for (std::size_t i = 0; i < al.ops.size() && i < ops_cap; ++i)
            ops[i] = static_cast<std::uint8_t>(al.ops[i]);
        if (rescored) *rescored = swsearch::rescore_alignment(al, qs, ss, mat, gaps);
    });
}

}  // extern "C"
