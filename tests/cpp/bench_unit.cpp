// tests/cpp/bench_unit.cpp -- CPU-only checks of swsearch/bench.hpp against the SPEC's examples.
#include <cmath>
#include <cstdio>
#include <sstream>

#include "swsearch/bench.hpp"

using namespace swsearch;

int main() {
    int failures = 0;
    auto check = [&](bool ok, const char* what) {
        if (!ok) {
            std::printf("FAIL: %s\n", what);
            ++failures;
        }
    };
    const GcupsMeasure one = measure_gcups(144, 204173280, 1.0);
    check(std::fabs(one.gcups - 29.40095232) < 1e-6, "144 x 204173280 / 1 s = 29.400... GCUPS");
    check(measure_gcups(0, 204173280, 1.0).gcups == 0.0, "zero query length -> 0 GCUPS");
    check(std::fabs(measure_gcups(144, 1000, 2.0).gcups * 2 - measure_gcups(144, 1000, 1.0).gcups) < 1e-15,
          "doubling elapsed halves gcups");
    check(std::fabs(one.gcups * one.elapsed * 1e9 - 144.0 * 204173280.0) / (144.0 * 204173280.0) < 1e-9, "formula identity");
    for (double bad : {0.0, -1.0}) {
        bool threw = false;
        try {
            measure_gcups(1, 1, bad);
        } catch (const measurement_error&) {
            threw = true;
        }
        check(threw, "elapsed <= 0 -> measurement_error");
    }
    BenchReport empty;
    std::ostringstream a;
    emit_csv(empty, a);
    check(a.str() == "query_id,query_length,repetitions,mean_gcups,min_gcups,max_gcups,stddev_gcups\n", "empty report -> header only");
    BenchReport r;
    r.rows.push_back(BenchRow{0, 144, 20, 29.5, 29.0, 30.0, 0.25});
    r.sweep.push_back(SweepRow{SweepParameter::chunk_width, 64, 12.5, true});
    std::ostringstream b;
    emit_csv(r, b);
    check(b.str() == "query_id,query_length,repetitions,mean_gcups,min_gcups,max_gcups,stddev_gcups\n"
                     "0,144,20,29.5,29,30,0.25\nparameter,value,mean_gcups,is_best\nchunk_width,64,12.5,1\n",
          "one row + one sweep point");
    check(detail::csv_field("a,b\"c") == "\"a,b\"\"c\"", "RFC 4180 quoting");
    std::printf(failures ? "bench_unit: %d failure(s)\n" : "bench_unit: ok\n", failures);
    return failures ? 1 : 0;
}
