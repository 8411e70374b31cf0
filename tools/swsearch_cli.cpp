// tools/swsearch_cli.cpp -- command-line front end.  Spec-only in the
// reference; built here on the drop-in headers, so every search runs on the GPU(s).
//
//   swsearch search -q query.fa -d db.fa [options]     ranked hits (rank, header, score, alignment summary)
//   swsearch bench  -q query.fa -d db.fa [options]     CSV per SPEC.md:414 (20 repetitions by default)
//   swsearch sweep  -q query.fa -d db.fa --param lane_width|chunk_width --values 4,8,16 [options]
//   swsearch stats  -d db.fa                           "<n> sequences, <r> residues, max <l>"
//   swsearch pack   -d db.fa -o db.swb [--threshold N] pack once on the host (no GPU): sorted, interleaved, with headers
//   ... --packed db.swb instead of -d db.fa            search / bench / sweep / stats straight from the packed file:
//                                                      no FASTA parsing, no sort, no pack
//
// Exit codes: 0 ok, 2 usage, 3 I/O, 4 format, 5 determinism violation, 1 anything else.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "swsearch/bench.hpp"
#include "swsearch/fasta.hpp"
#include "swsearch/packed.hpp"
#include "swsearch/scheduler.hpp"

using namespace swsearch;

namespace {

struct usage_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct CliInvocation {
    std::string command, query_path, db_path, packed_path, matrix = "BLOSUM62", output;
    bool threshold_given = false;
    std::int32_t gap_open = 10, gap_extend = 2;
    SearchConfig config;
    std::size_t repetitions = 20;
    std::string sweep_param = "lane_width";
    std::vector<std::size_t> sweep_values;
    bool help = false;
};

const char* kUsage =
    "usage: swsearch <search|bench|sweep|stats|pack> (-d DB.fa | --packed DB.swb) [-q QUERY.fa] [options]\n"
    "  -q, --query PATH        query FASTA (search, bench, sweep)\n"
    "  -d, --db PATH           database FASTA\n"
    "  --packed PATH           packed database written by 'swsearch pack' (instead of -d)\n"
    "  --matrix NAME|PATH      BLOSUM62 (default) or an NCBI-format matrix file\n"
    "  --gap-open N            default 10\n"
    "  --gap-extend N          default 2\n"
    "  -T, --workers N         accepted for compatibility (results never depend on it)\n"
    "  --lane-width N          accepted for compatibility\n"
    "  --chunk-width N         accepted for compatibility\n"
    "  --threshold N           length routing threshold, default 3000\n"
    "  --top-k N               default 10\n"
    "  --no-align              skip the traceback of the reported hits\n"
    "  --repetitions N         bench/sweep, default 20\n"
    "  --param NAME            sweep: lane_width | chunk_width\n"
    "  --values A,B,C          sweep values\n"
    "  -o, --output PATH       write results there instead of stdout\n"
    "  -h, --help\n";

std::size_t number(const std::string& flag, const std::string& text) {
    try {
        std::size_t used = 0;
        const long long v = std::stoll(text, &used);
        if (used != text.size() || v < 0) throw std::invalid_argument(text);
        return static_cast<std::size_t>(v);
    } catch (const std::exception&) {
        throw usage_error("non-numeric value for " + flag + ": '" + text + "'");
    }
}

CliInvocation parse_args(const std::vector<std::string>& argv) {
    CliInvocation inv;
    std::size_t i = 0;
    if (!argv.empty() && argv[0][0] != '-') inv.command = argv[i++];
    for (; i < argv.size(); ++i) {
        const std::string& flag = argv[i];
        auto value = [&]() -> const std::string& {
            if (i + 1 >= argv.size()) throw usage_error("missing value for " + flag);
            return argv[++i];
        };
        if (flag == "-h" || flag == "--help") inv.help = true;
        else if (flag == "-q" || flag == "--query") inv.query_path = value();
        else if (flag == "-d" || flag == "--db") inv.db_path = value();
        else if (flag == "--packed") inv.packed_path = value();
        else if (flag == "--matrix") inv.matrix = value();
        else if (flag == "--gap-open") inv.gap_open = static_cast<std::int32_t>(number(flag, value()));
        else if (flag == "--gap-extend") inv.gap_extend = static_cast<std::int32_t>(number(flag, value()));
        else if (flag == "-T" || flag == "--workers") inv.config.worker_count = number(flag, value());
        else if (flag == "--lane-width") inv.config.lane_width = number(flag, value());
        else if (flag == "--chunk-width") inv.config.chunk_width = number(flag, value());
        else if (flag == "--threshold") inv.config.length_threshold = number(flag, value()), inv.threshold_given = true;
        else if (flag == "--top-k") inv.config.top_k = number(flag, value());
        else if (flag == "--no-align") inv.config.compute_alignments = false;
        else if (flag == "--repetitions") inv.repetitions = number(flag, value());
        else if (flag == "--param") inv.sweep_param = value();
        else if (flag == "--values") {
            std::stringstream list(value());
            for (std::string item; std::getline(list, item, ',');) inv.sweep_values.push_back(number(flag, item));
        } else if (flag == "-o" || flag == "--output") inv.output = value();
        else throw usage_error("unknown flag '" + flag + "'");
    }
    if (inv.help) return inv;
    if (inv.command != "search" && inv.command != "bench" && inv.command != "sweep" && inv.command != "stats" && inv.command != "pack")
        throw usage_error("expected a command: search, bench, sweep, stats or pack");
    if (inv.command == "pack") {
        if (inv.db_path.empty() || inv.output.empty()) throw usage_error("pack needs a FASTA database (-d) and an output file (-o)");
        return inv;
    }
    if (inv.db_path.empty() == inv.packed_path.empty()) throw usage_error("exactly one of -d and --packed is required");
    if (inv.command != "stats" && inv.query_path.empty()) throw usage_error("a query (-q) is required");
    if (inv.command == "sweep") {
        if (inv.sweep_param != "lane_width" && inv.sweep_param != "chunk_width")
            throw usage_error("--param must be lane_width or chunk_width");
        if (inv.sweep_values.empty()) throw usage_error("--values is required for sweep");
    }
    return inv;
}

void print_alignment(std::ostream& out, const Alignment& a, const EncodedSequence& q, const EncodedSequence& s) {
    // compact three-line display, 60 columns per block
    const Alphabet& alpha = protein_alphabet();
    std::string top, mid, bottom;
    std::size_t qi = a.query_begin, si = a.subject_begin;
    for (EditOp op : a.ops) {
        switch (op) {
        case EditOp::match: top += alpha.symbol(q.codes[qi++]); mid += '|'; bottom += alpha.symbol(s.codes[si++]); break;
        case EditOp::substitute: top += alpha.symbol(q.codes[qi++]); mid += '.'; bottom += alpha.symbol(s.codes[si++]); break;
        case EditOp::insert: top += '-'; mid += ' '; bottom += alpha.symbol(s.codes[si++]); break;
        case EditOp::del: top += alpha.symbol(q.codes[qi++]); mid += ' '; bottom += '-'; break;
        }
    }
    for (std::size_t at = 0; at < top.size(); at += 60)
        out << "    " << top.substr(at, 60) << "\n    " << mid.substr(at, 60) << "\n    " << bottom.substr(at, 60) << "\n";
}

int run(const CliInvocation& inv_in, std::ostream& out) {
    CliInvocation inv = inv_in;
    std::unique_ptr<SequenceDatabase> holder;
    if (!inv.packed_path.empty()) {
        // stats needs the host copy only; everything else also wants the device copy, made from the same file
        std::size_t threshold = 0;
        if (inv.command == "stats") holder = std::make_unique<SequenceDatabase>(load_packed_database(inv.packed_path, &threshold));
        else holder = open_packed_database(inv.packed_path, &threshold);
        if (inv.threshold_given && inv.config.length_threshold != threshold)
            throw usage_error("--threshold " + std::to_string(inv.config.length_threshold) + " differs from the threshold the file was packed with (" +
                              std::to_string(threshold) + ")");
        inv.config.length_threshold = threshold;
    } else {
        holder = std::make_unique<SequenceDatabase>(load_database(inv.db_path));
    }
    const SequenceDatabase& db = *holder;
    if (inv.command == "stats") {
        out << db.num_sequences() << " sequences, " << db.total_residues << " residues, max " << db.max_length << "\n";
        return 0;
    }
    const ScoringMatrix matrix = inv.matrix == "BLOSUM62" ? blosum62() : load_matrix(inv.matrix);
    const GapModel gaps(inv.gap_open, inv.gap_extend);
    const SequenceDatabase queries = load_database(inv.query_path);

    if (inv.command == "search") {
        for (const EncodedSequence& query : queries.sequences) {
            const RankedResults results = run_search(query, db, matrix, gaps, inv.config);
            out << "query " << query.header << " (" << query.length() << " residues): " << results.hits.size() << " hits\n";
            std::size_t rank = 1;
            for (const Hit& hit : results.hits) {
                const EncodedSequence& subject = db.sequences[hit.db_index];
                out << "  " << rank++ << "\t" << subject.header << "\t" << hit.score.value;
                if (hit.alignment) {
                    const Alignment& a = *hit.alignment;
                    if (a.capped) out << "\t(alignment capped)";
                    else out << "\tq[" << a.query_begin << "," << a.query_end << ") s[" << a.subject_begin << "," << a.subject_end << ") " << a.ops.size() << " columns";
                }
                out << "\n";
                if (hit.alignment && !hit.alignment->capped) print_alignment(out, *hit.alignment, query, subject);
            }
        }
        return 0;
    }
    BenchReport report;
    if (inv.command == "bench") {
        report = run_benchmark(queries.sequences, db, matrix, gaps, inv.config, inv.repetitions);
    } else {
        const SweepParameter param = inv.sweep_param == "lane_width" ? SweepParameter::lane_width : SweepParameter::chunk_width;
        report.sweep = sweep_parameter(param, inv.sweep_values, inv.config, queries.sequences, db, matrix, gaps, inv.repetitions);
    }
    emit_csv(report, out);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const CliInvocation inv = parse_args(std::vector<std::string>(argv + 1, argv + argc));
        if (inv.help) {
            std::cout << kUsage;
            return 0;
        }
        if (inv.command == "pack") {
            const SequenceDatabase db = load_database(inv.db_path);
            save_packed_database(db, inv.output, inv.config.length_threshold);
            std::cout << "packed " << db.num_sequences() << " sequences, " << db.total_residues << " residues (threshold "
                      << inv.config.length_threshold << ") -> " << inv.output << "\n";
            return 0;
        }
        if (inv.output.empty()) return run(inv, std::cout);
        std::ofstream file(inv.output);
        if (!file) throw io_error("cannot open " + inv.output);
        return run(inv, file);
    } catch (const usage_error& e) {
        std::cerr << "swsearch: " << e.what() << "\n" << kUsage;
        return 2;
    } catch (const io_error& e) {
        std::cerr << "swsearch: " << e.what() << "\n";
        return 3;
    } catch (const format_error& e) {
        std::cerr << "swsearch: " << e.what() << "\n";
        return 4;
    } catch (const determinism_error& e) {
        std::cerr << "swsearch: determinism violation: " << e.what() << "\n";
        return 5;
    } catch (const std::exception& e) {
        std::cerr << "swsearch: " << e.what() << "\n";
        return 1;
    }
}
