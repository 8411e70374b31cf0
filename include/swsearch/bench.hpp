// swsearch/bench.hpp -- the paper's measurement protocol.
//
// The reference ships this module as specification only (no code exists under proj/), so there is nothing to be
// drop-in compatible with beyond the names, formulas and CSV schema the SPEC fixes:
//   measure_gcups     gcups = query_length x db_residues / (elapsed x 1e9)
//   run_benchmark     one discarded warm-up, then `repetitions` timed run_search calls per query;
//                     every repetition's RankedResults must equal the first (determinism_error)
//   sweep_parameter   one benchmark per lane_width / chunk_width value, argmax flagged
//   emit_csv          query_id,query_length,repetitions,mean_gcups,min_gcups,max_gcups,stddev_gcups
//                     and parameter,value,mean_gcups,is_best
// Timed region: run_search with compute_alignments = false (scoring + scheduling + merge); database load/packing
// and traceback are excluded -- the packed device copy is built by the warm-up run.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <iomanip>
#include <ostream>
#include <sstream>
#include <string>
#include <vector>

#include "swsearch/errors.hpp"
#include "swsearch/scheduler.hpp"

namespace swsearch {

struct GcupsMeasure {
    std::size_t query_length = 0;
    std::size_t db_residues = 0;
    double elapsed = 0.0;   // seconds
    double gcups = 0.0;
};

/// GCUPS of one timed search.  elapsed must be positive.
inline GcupsMeasure measure_gcups(std::size_t query_length, std::size_t db_residues, double elapsed) {
    if (!(elapsed > 0.0)) throw measurement_error("elapsed time must be positive");
    GcupsMeasure m;
    m.query_length = query_length;
    m.db_residues = db_residues;
    m.elapsed = elapsed;
    m.gcups = static_cast<double>(query_length) * static_cast<double>(db_residues) / (elapsed * 1e9);
    return m;
}

struct BenchRow {
    std::size_t query_id = 0;
    std::size_t query_length = 0;
    std::size_t repetitions = 0;
    double mean_gcups = 0.0, min_gcups = 0.0, max_gcups = 0.0, stddev_gcups = 0.0;   // sample (n-1) deviation
};

enum class SweepParameter { lane_width, chunk_width };

struct SweepRow {
    SweepParameter parameter = SweepParameter::lane_width;
    std::size_t value = 0;
    double mean_gcups = 0.0;
    bool is_best = false;
};

struct BenchEnvironment {
    std::size_t worker_count = 0, lane_width = 0, chunk_width = 0, length_threshold = 0, top_k = 0;
    std::size_t db_sequences = 0, db_residues = 0, db_max_length = 0;
};

struct BenchReport {
    std::vector<BenchRow> rows;
    std::vector<SweepRow> sweep;
    BenchEnvironment environment;
};

/// Seconds on a monotonic clock; injectable so that the timing isolation can be tested with a fake clock.
using BenchClock = std::function<double()>;

inline double steady_seconds() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

/// The paper's protocol: for every query one discarded warm-up, then `repetitions` timed searches.
inline BenchReport run_benchmark(const std::vector<EncodedSequence>& queries, const SequenceDatabase& db,
                                 const ScoringMatrix& matrix, const GapModel& gaps, SearchConfig config,
                                 std::size_t repetitions = 20, const BenchClock& clock = steady_seconds,
                                 std::size_t warmup_runs = 1) {
    if (repetitions < 1) throw std::invalid_argument("repetitions must be >= 1");
    config.compute_alignments = false;   // traceback is outside the timed region
    BenchReport report;
    report.environment = BenchEnvironment{config.worker_count, config.lane_width,   config.chunk_width,
                                          config.length_threshold, config.top_k,    db.num_sequences(),
                                          db.total_residues,      db.max_length};
    std::size_t residues = 0;
    for (const EncodedSequence& s : db.sequences) residues += s.length();

    for (std::size_t id = 0; id < queries.size(); ++id) {
        const EncodedSequence& query = queries[id];
        // the reference result every repetition is compared with; it doubles as the first (discarded) warm-up
        const RankedResults first = run_search(query, db, matrix, gaps, config);
        for (std::size_t w = 1; w < warmup_runs; ++w) run_search(query, db, matrix, gaps, config);
        BenchRow row;
        row.query_id = id;
        row.query_length = query.length();
        row.repetitions = repetitions;
        double sum = 0.0, sum_sq = 0.0;
        for (std::size_t rep = 0; rep < repetitions; ++rep) {
            const double t0 = clock();
            const RankedResults again = run_search(query, db, matrix, gaps, config);
            const double elapsed = clock() - t0;
            if (!(again == first))
                throw determinism_error("query " + std::to_string(id) + ": repetition " + std::to_string(rep) +
                                        " returned different results");
            const double g = measure_gcups(query.length(), residues, elapsed).gcups;
            sum += g;
            sum_sq += g * g;
            row.min_gcups = rep == 0 ? g : std::min(row.min_gcups, g);
            row.max_gcups = rep == 0 ? g : std::max(row.max_gcups, g);
        }
        const double n = static_cast<double>(repetitions);
        row.mean_gcups = sum / n;
        row.stddev_gcups = repetitions > 1 ? std::sqrt(std::max(0.0, (sum_sq - sum * sum / n) / (n - 1.0))) : 0.0;
        report.rows.push_back(row);
    }
    return report;
}

/// One benchmark per value of lane_width or chunk_width; the best mean is flagged.  On the GPU path these knobs
/// are result- and (by design) performance-invisible; the sweep exists for protocol parity.
inline std::vector<SweepRow> sweep_parameter(SweepParameter parameter, const std::vector<std::size_t>& values,
                                             const SearchConfig& fixed, const std::vector<EncodedSequence>& queries,
                                             const SequenceDatabase& db, const ScoringMatrix& matrix, const GapModel& gaps,
                                             std::size_t repetitions = 20, const BenchClock& clock = steady_seconds) {
    if (values.empty()) throw std::invalid_argument("sweep needs at least one value");
    std::vector<SweepRow> table;
    for (std::size_t value : values) {
        SearchConfig cfg = fixed;
        (parameter == SweepParameter::lane_width ? cfg.lane_width : cfg.chunk_width) = value;
        const BenchReport report = run_benchmark(queries, db, matrix, gaps, cfg, repetitions, clock);
        double mean = 0.0;
        for (const BenchRow& row : report.rows) mean += row.mean_gcups;
        if (!report.rows.empty()) mean /= static_cast<double>(report.rows.size());
        table.push_back(SweepRow{parameter, value, mean, false});
    }
    std::size_t best = 0;
    for (std::size_t i = 1; i < table.size(); ++i)
        if (table[i].mean_gcups > table[best].mean_gcups) best = i;
    table[best].is_best = true;
    return table;
}

namespace detail {
inline std::string csv_field(const std::string& text) {   // RFC 4180 quoting
    if (text.find_first_of(",\"\r\n") == std::string::npos) return text;
    std::string quoted = "\"";
    for (char c : text) {
        if (c == '"') quoted += '"';
        quoted += c;
    }
    return quoted + "\"";
}
}  // namespace detail

/// query rows, then (if present) the sweep table, each with its header row.
inline void emit_csv(const BenchReport& report, std::ostream& sink) {
    sink << "query_id,query_length,repetitions,mean_gcups,min_gcups,max_gcups,stddev_gcups\n";
    sink << std::setprecision(9);
    for (const BenchRow& row : report.rows)
        sink << row.query_id << ',' << row.query_length << ',' << row.repetitions << ',' << row.mean_gcups << ','
             << row.min_gcups << ',' << row.max_gcups << ',' << row.stddev_gcups << '\n';
    if (!report.sweep.empty()) {
        sink << "parameter,value,mean_gcups,is_best\n";
        for (const SweepRow& row : report.sweep)
            sink << detail::csv_field(row.parameter == SweepParameter::lane_width ? "lane_width" : "chunk_width") << ','
                 << row.value << ',' << row.mean_gcups << ',' << (row.is_best ? 1 : 0) << '\n';
    }
    if (!sink) throw io_error("CSV: stream write failure");
}

}  // namespace swsearch
