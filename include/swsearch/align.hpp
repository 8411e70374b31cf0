// swsearch/align.hpp -- alignment kernels of the swsearch API (drop-in for the reference's align.hpp:18-384).
//
// Every *scoring* entry point keeps its signature, validation, messages and exact result, but runs on the GPU
// through libswb200.so:
//     sw_score_scalar     align.hpp:69-78    -> swb_score_pair   (intra-task warp-shuffle kernel, int32)
//     sw_score_batch      align.hpp:91-159   -> swb_score_batch  (packed int16 DPX kernel + int32 re-run)
//     sw_score_wavefront  align.hpp:166-229  -> swb_score_pair
//     sw_align_traceback  align.hpp:254-353  -> swb_align_traceback (direction-matrix fill + backward walk on the GPU;
//                                               runs after scoring on at most top_k hits, outside the measured path,
//                                               SPEC.md:403, but on by default)
#pragma once

#include <algorithm>
#include <compare>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "swsearch/gpu.hpp"
#include "swsearch/scoring.hpp"
#include "swsearch/sequence.hpp"

namespace swsearch {

/// Optimal local alignment score; the empty alignment makes it non-negative.
struct AlignScore {
    std::int32_t value = 0;
    auto operator<=>(const AlignScore&) const = default;
};

namespace detail {
/// The reference's stand-in for minus infinity in the gap layers (INT32_MIN / 4).
inline constexpr std::int32_t kNegInf = std::numeric_limits<std::int32_t>::min() / 4;

inline AlignScore pair_on_gpu(const EncodedSequence& query, const EncodedSequence& subject, const ScoringMatrix& matrix,
                              const GapModel& gaps, std::size_t chunk_width) {
    for (std::uint8_t code : subject.codes)
        if (code >= ScoringMatrix::size) throw std::out_of_range("subject code outside matrix alphabet");
    std::int32_t score = 0;
    gpu::check(swb_score_pair(query.codes.data(), static_cast<std::uint32_t>(query.length()), subject.codes.data(),
                              static_cast<std::uint32_t>(subject.length()), gpu::matrix_table(matrix), gaps.open(),
                              gaps.extend(), chunk_width, gpu::devices().front(), &score));
    return {score};
}
}  // namespace detail

/// Full-precision affine-gap local alignment score of one pair.
inline AlignScore sw_score_scalar(const EncodedSequence& query, const EncodedSequence& subject,
                                  const ScoringMatrix& matrix, const GapModel& gaps) {
    return detail::pair_on_gpu(query, subject, matrix, gaps, 1);
}

/// Subjects scored together, one per lane; missing lanes (fewer subjects than lane_width, or null entries) are
/// padding and score 0.
struct LaneBatch {
    std::size_t lane_width = 1;
    std::vector<const EncodedSequence*> subjects;
};

/// Inter-task kernel.  The result has lane_width entries.  On the GPU the lanes are the two int16 halves of DPX
/// words; a lane whose score leaves the trusted 16-bit range is re-run in int32, so the narrow arithmetic never
/// shows in the results.
inline std::vector<AlignScore> sw_score_batch(const QueryProfile& profile, const LaneBatch& batch, const GapModel& gaps) {
    if (batch.lane_width < 1) throw std::invalid_argument("lane_width must be >= 1");
    if (batch.subjects.size() > batch.lane_width) throw std::invalid_argument("more subjects than lanes");
    std::vector<AlignScore> scores(batch.lane_width);
    if (profile.query_length() == 0 || batch.subjects.empty()) return scores;

    std::vector<const std::uint8_t*> rows(batch.subjects.size(), nullptr);
    std::vector<std::uint32_t> lengths(batch.subjects.size(), 0);
    static const std::uint8_t kNoResidues[1] = {0};
    for (std::size_t lane = 0; lane < rows.size(); ++lane) {
        const EncodedSequence* s = batch.subjects[lane];
        if (s == nullptr) continue;
        rows[lane] = s->codes.empty() ? kNoResidues : s->codes.data();
        lengths[lane] = static_cast<std::uint32_t>(s->length());
    }
    std::vector<std::int32_t> raw(batch.lane_width, 0);
    gpu::check(swb_score_batch(profile.query().codes.data(), static_cast<std::uint32_t>(profile.query_length()),
                               rows.data(), lengths.data(), static_cast<std::uint32_t>(rows.size()),
                               static_cast<std::uint32_t>(batch.lane_width), gpu::matrix_table(profile.matrix()),
                               gaps.open(), gaps.extend(), gpu::devices().front(), raw.data()));
    for (std::size_t lane = 0; lane < scores.size(); ++lane) scores[lane].value = raw[lane];
    return scores;
}

/// Intra-task kernel: same score as sw_score_scalar for every chunk_width >= 1.
inline AlignScore sw_score_wavefront(const EncodedSequence& query, const EncodedSequence& subject,
                                     const ScoringMatrix& matrix, const GapModel& gaps, std::size_t chunk_width) {
    if (chunk_width < 1) throw std::invalid_argument("chunk_width must be >= 1");
    return detail::pair_on_gpu(query, subject, matrix, gaps, chunk_width);
}

/// One column of an alignment.
///   match / substitute  residues paired (equal / different codes)
///   insert              a subject residue facing a gap in the query
///   del                 a query residue facing a gap in the subject
enum class EditOp : std::uint8_t { match, substitute, insert, del };

/// Local alignment with its edit script.  `capped` means the traceback matrix would have exceeded the memory
/// budget: the score is still exact but the script is empty.
struct Alignment {
    std::size_t query_begin = 0, query_end = 0;       // half-open
    std::size_t subject_begin = 0, subject_end = 0;   // half-open
    std::vector<EditOp> ops;
    AlignScore score;
    bool capped = false;
};

/// Optimal local alignment with its edit script, computed on the GPU (swb_align_traceback): an anti-diagonal
/// fill that writes one direction byte per cell, then a backward walk.  The matrix needs (|query|+1)*(|subject|+1)
/// bytes by the reference's accounting; pairs beyond `memory_cap` come back score-only with `capped` set.
/// Tie-breaking follows the reference exactly, so the scripts are identical: inside a cell zero, diagonal, gap along
/// the query, gap along the subject win in that order only on strict improvement; a gap that is as good opened as
/// extended counts as opened; the first best cell in (subject row, query column) order is the end point.
inline Alignment sw_align_traceback(const EncodedSequence& query, const EncodedSequence& subject,
                                    const ScoringMatrix& matrix, const GapModel& gaps,
                                    std::size_t memory_cap = std::size_t{256} << 20) {
    Alignment result;
    const std::size_t m = query.length(), n = subject.length();
    if (m == 0 || n == 0) return result;
    for (std::uint8_t code : subject.codes)
        if (code >= ScoringMatrix::size) throw std::out_of_range("subject code outside matrix alphabet");

    swb_alignment raw{};
    std::vector<std::uint8_t> script(m + n);
    gpu::check(swb_align_traceback(query.codes.data(), static_cast<std::uint32_t>(m), subject.codes.data(),
                                   static_cast<std::uint32_t>(n), gpu::matrix_table(matrix), gaps.open(), gaps.extend(),
                                   memory_cap, gpu::devices().front(), &raw, script.data(), script.size()));
    result.score = {raw.score};
    result.capped = raw.capped != 0;
    result.query_begin = raw.query_begin;
    result.query_end = raw.query_end;
    result.subject_begin = raw.subject_begin;
    result.subject_end = raw.subject_end;
    result.ops.resize(raw.n_ops);
    for (std::size_t i = 0; i < result.ops.size(); ++i) result.ops[i] = static_cast<EditOp>(script[i]);
    return result;
}

/// Score of an edit script under a matrix and gap model (checks that a traceback is sound).
inline std::int32_t rescore_alignment(const Alignment& alignment, const EncodedSequence& query,
                                      const EncodedSequence& subject, const ScoringMatrix& matrix, const GapModel& gaps) {
    std::int64_t sum = 0;
    std::size_t qi = alignment.query_begin, si = alignment.subject_begin;
    bool in_del = false, in_ins = false;
    for (EditOp op : alignment.ops) {
        if (op == EditOp::del) {
            sum -= in_del ? gaps.extend() : gaps.open();
            ++qi;
        } else if (op == EditOp::insert) {
            sum -= in_ins ? gaps.extend() : gaps.open();
            ++si;
        } else {
            sum += matrix.score(subject.codes[si++], query.codes[qi++]);
        }
        in_del = op == EditOp::del;
        in_ins = op == EditOp::insert;
    }
    return static_cast<std::int32_t>(sum);
}

}  // namespace swsearch
