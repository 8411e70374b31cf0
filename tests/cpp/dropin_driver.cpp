// tests/cpp/dropin_driver.cpp -- one program, two builds.
//
// It uses nothing but the public swsearch API, so the very same source compiles against
//   (a) the unmodified reference headers  (-I /root/reference/proj/include, -include oracle/ref_compat.h)
//       -> oracle/_ref/dropin_ref        (CPU, built in the authoring container, travels prebuilt), and
//   (b) this repository's drop-in headers (-I include, -lswb200)
//       -> tests/cpp/_build/dropin_b200  (GPU).
// tests/test_gpu_dropin.py runs both and requires byte-identical output: scores, ranked lists, edit scripts,
// statistics, exception types and messages.
#include <cstdint>
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "swsearch/align.hpp"
#include "swsearch/alphabet.hpp"
#include "swsearch/errors.hpp"
#include "swsearch/fasta.hpp"
#include "swsearch/scheduler.hpp"
#include "swsearch/scoring.hpp"
#include "swsearch/sequence.hpp"

using namespace swsearch;

namespace {

struct Lcg {
    std::uint64_t state;
    explicit Lcg(std::uint64_t seed) : state(seed * 2862933555777941757ull + 3037000493ull) {}
    std::uint32_t next() {
        state = state * 6364136223846793005ull + 1442695040888963407ull;
        return static_cast<std::uint32_t>(state >> 33);
    }
    std::uint32_t below(std::uint32_t n) { return n ? next() % n : 0; }
};

EncodedSequence random_sequence(Lcg& rng, std::size_t len, std::uint32_t symbols = 20) {
    EncodedSequence s;
    s.codes.resize(len);
    for (auto& c : s.codes) c = static_cast<std::uint8_t>(rng.below(symbols));
    return s;
}

EncodedSequence mutated(Lcg& rng, const EncodedSequence& src, std::uint32_t percent) {
    EncodedSequence s = src;
    for (auto& c : s.codes)
        if (rng.below(100) < percent) c = static_cast<std::uint8_t>(rng.below(20));
    if (s.codes.size() > 10) s.codes.erase(s.codes.begin() + 5, s.codes.begin() + 8);
    return s;
}

std::string ops_text(const Alignment& a) {
    std::string t;
    for (EditOp op : a.ops) t.push_back("MSID"[static_cast<int>(op)]);
    return t;
}

template <class Fn>
void expect_throw(const char* label, Fn&& fn) {
    try {
        fn();
        std::printf("%s: no exception\n", label);
    } catch (const std::invalid_argument& e) {
        std::printf("%s: invalid_argument: %s\n", label, e.what());
    } catch (const std::out_of_range& e) {
        std::printf("%s: out_of_range: %s\n", label, e.what());
    } catch (const format_error& e) {
        std::printf("%s: format_error: %s\n", label, e.what());
    } catch (const io_error& e) {
        std::printf("%s: io_error: %s\n", label, e.what());
    } catch (const std::exception& e) {
        std::printf("%s: exception: %s\n", label, e.what());
    }
}

void print_results(const char* label, const RankedResults& r, const SearchStats& st, bool alignments) {
    std::printf("%s: %zu hits lane=%zu wavefront=%zu\n", label, r.hits.size(), st.lane_scored, st.wavefront_scored);
    for (const Hit& h : r.hits) {
        std::printf("  %u %d", h.db_index, h.score.value);
        if (alignments && h.alignment) {
            const Alignment& a = *h.alignment;
            std::printf(" q[%zu,%zu) s[%zu,%zu) capped=%d score=%d %s", a.query_begin, a.query_end, a.subject_begin,
                        a.subject_end, a.capped ? 1 : 0, a.score.value, ops_text(a).c_str());
        }
        std::printf("\n");
    }
}

}  // namespace

int main() {
    const ScoringMatrix& b62 = blosum62();
    const GapModel gaps(10, 2);
    Lcg rng(20220311);

    // ---- L0-L2: alphabet, sequences, FASTA, matrices -------------------------------------------------------
    const Alphabet& alpha = protein_alphabet();
    std::printf("alphabet %zu unknown=%u A=%u w=%u ?=%u contains(-)=%d\n", alpha.size(), alpha.unknown_index(),
                alpha.index_of('A'), alpha.index_of('w'), alpha.index_of('?'), alpha.contains('-') ? 1 : 0);
    std::istringstream fasta(">sp|P1 first\nARNDC\nQEGHI\r\n\n>second  \nlkmfpstwyv bzx*\n>third\n");
    LoadStats load;
    SequenceDatabase small = build_database(fasta, alpha, &load);
    std::printf("fasta %zu seqs %zu residues max=%zu unknown=%zu empty=%zu [%s] [%s]\n", small.num_sequences(),
                small.total_residues, small.max_length, load.unknown_residues, load.zero_length_records,
                small.sequences[1].header.c_str(), decode_sequence(small.sequences[1], alpha).c_str());
    std::ostringstream back;
    write_fasta(back, small, alpha, 7);
    std::printf("%s", back.str().c_str());
    expect_throw("fasta-no-header", [] { std::istringstream s("ACGT\n"); parse_fasta(s); });
    expect_throw("fasta-empty-header", [] { std::istringstream s(">\nAC\n"); parse_fasta(s); });

    std::printf("blosum62 AA=%d WW=%d AR=%d **=%d name=%s\n", b62.score(0, 0), b62.score(17, 17), b62.score(0, 1),
                b62.score(23, 23), b62.name().c_str());
    std::ostringstream mtext;
    write_matrix(mtext, b62);
    std::istringstream mback(mtext.str());
    std::printf("matrix round trip equal=%d\n", parse_matrix(mback, "again") == b62 ? 1 : 0);
    {
        std::istringstream partial("# tiny\n A R\nA 3 -2\nR -2 4\n");
        const ScoringMatrix tiny = parse_matrix(partial);
        std::printf("partial AA=%d AR=%d NN=%d NA=%d name=%s\n", tiny.score(0, 0), tiny.score(0, 1), tiny.score(2, 2),
                    tiny.score(2, 0), tiny.name().c_str());
    }
    expect_throw("matrix-asym", [] { std::istringstream s(" A R\nA 1 2\nR 3 1\n"); parse_matrix(s); });
    expect_throw("matrix-short", [] { std::istringstream s(" A R\nA 1\nR 1 1\n"); parse_matrix(s); });
    expect_throw("matrix-missing", [] { std::istringstream s(" A R\nA 1 1\n"); parse_matrix(s); });
    expect_throw("gap-model", [] { GapModel g(1, 2); });
    expect_throw("gap-negative", [] { GapModel g(3, -1); });

    // ---- L3: kernels on pairs ----------------------------------------------------------------------------------
    EncodedSequence aaa;
    aaa.codes = {0, 0, 0};
    std::printf("AAA scalar=%d wavefront=%d\n", sw_score_scalar(aaa, aaa, b62, gaps).value,
                sw_score_wavefront(aaa, aaa, b62, gaps, 1).value);
    for (int i = 0; i < 12; ++i) {
        const EncodedSequence q = random_sequence(rng, 1 + rng.below(300));
        EncodedSequence s = (i % 3 == 0) ? mutated(rng, q, 20) : random_sequence(rng, rng.below(400));
        const GapModel g(5 + static_cast<int>(rng.below(10)), static_cast<int>(rng.below(5)));
        std::printf("pair %d: %zu x %zu scalar=%d wf1=%d wf64=%d\n", i, q.length(), s.length(),
                    sw_score_scalar(q, s, b62, g).value, sw_score_wavefront(q, s, b62, g, 1).value,
                    sw_score_wavefront(q, s, b62, g, 64).value);
    }
    {
        const EncodedSequence q = random_sequence(rng, 90);
        const QueryProfile profile = make_profile(b62, q);
        std::vector<EncodedSequence> owned;
        for (int i = 0; i < 6; ++i) owned.push_back(random_sequence(rng, rng.below(200)));
        owned.push_back(mutated(rng, q, 10));
        LaneBatch batch;
        batch.lane_width = 16;
        for (auto& s : owned) batch.subjects.push_back(&s);
        batch.subjects[2] = nullptr;
        const auto scores = sw_score_batch(profile, batch, gaps);
        std::printf("batch %zu:", scores.size());
        for (const AlignScore& s : scores) std::printf(" %d", s.value);
        std::printf(" row0=%d row16=%d\n", profile.row(0)[0], profile.row16(17)[3]);
        // a lane that leaves the 16-bit range
        EncodedSequence big;
        big.codes.assign(3200, 17);
        const QueryProfile wide = make_profile(b62, big);
        LaneBatch one;
        one.lane_width = 2;
        one.subjects = {&big};
        const auto s2 = sw_score_batch(wide, one, gaps);
        std::printf("saturating lane: %d %d\n", s2[0].value, s2[1].value);
        expect_throw("batch-width", [&] { LaneBatch b; b.lane_width = 0; sw_score_batch(profile, b, gaps); });
        expect_throw("batch-overfull", [&] { LaneBatch b; b.lane_width = 1; b.subjects = {&owned[0], &owned[1]}; sw_score_batch(profile, b, gaps); });
        expect_throw("wavefront-width", [&] { sw_score_wavefront(q, q, b62, gaps, 0); });
        expect_throw("profile-code", [&] { EncodedSequence bad; bad.codes = {1, 30}; make_profile(b62, bad); });
    }

    // ---- traceback ---------------------------------------------------------------------------------------------------
    for (int i = 0; i < 4; ++i) {
        const EncodedSequence q = random_sequence(rng, 30 + rng.below(120));
        const EncodedSequence s = mutated(rng, q, 15 + 10 * i);
        const Alignment a = sw_align_traceback(q, s, b62, gaps);
        std::printf("traceback %d: score=%d q[%zu,%zu) s[%zu,%zu) rescored=%d %s\n", i, a.score.value, a.query_begin,
                    a.query_end, a.subject_begin, a.subject_end, rescore_alignment(a, q, s, b62, gaps), ops_text(a).c_str());
        const Alignment capped = sw_align_traceback(q, s, b62, gaps, 64);
        std::printf("  capped=%d score=%d ops=%zu\n", capped.capped ? 1 : 0, capped.score.value, capped.ops.size());
    }

    // ---- L4: search ----------------------------------------------------------------------------------------------------
    SequenceDatabase db;
    const EncodedSequence query = random_sequence(rng, 144);
    for (int i = 0; i < 300; ++i) {
        EncodedSequence s = random_sequence(rng, rng.below(420), 23);
        if (i == 17) s = query;
        if (i == 99) s = mutated(rng, query, 10);
        if (i == 250) s = mutated(rng, query, 35);
        if (i == 123 || i == 124) s = db.sequences[40];   // ties
        if (i == 200) s.codes.clear();
        db.total_residues += s.length();
        db.max_length = std::max(db.max_length, s.length());
        db.sequences.push_back(std::move(s));
    }
    const DatabasePartition part = partition_database(db, 300);
    std::printf("partition short=%zu long=%zu first_long=%u\n", part.short_pool.size(), part.long_pool.size(),
                part.long_pool.empty() ? 0u : part.long_pool.front());
    {
        ChunkQueue queue(detail::make_chunks(10, 4, KernelRoute::intra_task));
        std::printf("queue %zu:", queue.size());
        while (auto c = queue.claim()) std::printf(" [%u,%u)", c->begin, c->end);
        std::printf(" then %d\n", queue.claim().has_value() ? 1 : 0);
    }
    struct Variant { std::size_t workers, lanes, chunk, threshold, k; bool align; };
    const Variant variants[] = {{1, 8, 64, 3000, 10, true}, {4, 1, 1, 300, 10, false}, {8, 32, 64, 0, 7, false},
                                {2, 8, 16, 100000, 500, false}, {1, 8, 64, 200, 3, true}};
    int v = 0;
    for (const Variant& var : variants) {
        SearchConfig cfg;
        cfg.worker_count = var.workers;
        cfg.lane_width = var.lanes;
        cfg.chunk_width = var.chunk;
        cfg.length_threshold = var.threshold;
        cfg.top_k = var.k;
        cfg.cpu_pool_threads = var.workers > 1 ? var.workers / 2 : 1;
        cfg.compute_alignments = var.align;
        cfg.traceback_memory_cap = v == 4 ? 2000 : (std::size_t{256} << 20);
        SearchStats st;
        const RankedResults r = run_search(query, db, b62, gaps, cfg, &st);
        char label[32];
        std::snprintf(label, sizeof label, "search %d", v++);
        if (var.k > 20) {
            std::uint64_t digest = 1469598103934665603ull;
            for (const Hit& h : r.hits) digest = (digest ^ (h.db_index * 1000003ull + static_cast<std::uint32_t>(h.score.value))) * 1099511628211ull;
            std::printf("%s: %zu hits lane=%zu wavefront=%zu digest=%llu\n", label, r.hits.size(), st.lane_scored,
                        st.wavefront_scored, static_cast<unsigned long long>(digest));
        } else {
            print_results(label, r, st, var.align);
        }
    }
    {
        SequenceDatabase empty;
        SearchConfig cfg;
        const RankedResults r = run_search(query, empty, b62, gaps, cfg);
        std::printf("empty db: %zu hits\n", r.hits.size());
        EncodedSequence none;
        cfg.compute_alignments = true;
        const RankedResults r2 = run_search(none, db, b62, gaps, cfg);
        std::printf("empty query: %zu hits first=%u score=%d has_alignment=%d\n", r2.hits.size(), r2.hits[0].db_index,
                    r2.hits[0].score.value, r2.hits[0].alignment.has_value() ? 1 : 0);
    }
    expect_throw("config-workers", [&] { SearchConfig c; c.worker_count = 0; run_search(query, db, b62, gaps, c); });
    expect_throw("config-lanes", [&] { SearchConfig c; c.lane_width = 0; run_search(query, db, b62, gaps, c); });
    expect_throw("config-chunk", [&] { SearchConfig c; c.chunk_width = 0; run_search(query, db, b62, gaps, c); });
    expect_throw("config-topk", [&] { SearchConfig c; c.top_k = 0; run_search(query, db, b62, gaps, c); });
    expect_throw("query-code", [&] { EncodedSequence bad; bad.codes = {0, 24}; SearchConfig c; run_search(bad, db, b62, gaps, c); });

    // ---- merge ---------------------------------------------------------------------------------------------------------
    {
        std::vector<std::vector<Hit>> parts(3);
        parts[0].push_back({3, {50}, std::nullopt});
        parts[1].push_back({1, {50}, std::nullopt});
        parts[1].push_back({9, {70}, std::nullopt});
        const RankedResults merged = merge_results(parts, 2);
        std::printf("merge:");
        for (const Hit& h : merged.hits) std::printf(" (%u,%d)", h.db_index, h.score.value);
        std::printf(" equal_self=%d\n", merged == merged ? 1 : 0);
    }
    return 0;
}
