// ref_callers_main.cpp -- runs the reference's OWN L4 callers on the GPU.
//
// Linked with /root/reference/proj/src/bench.cpp (run_suite, emit_csv) and
// /root/reference/proj/src/checks.cpp (verify_strategies,
// check_cell_coverage, ltm_exactness_sweep), compiled UNMODIFIED against
// include/trigrid_compat/trigrid/*.hpp -> include/trigrid_b200.hpp (namespace
// trigrid) and libtrigrid_b200.so.  Built by tests/test_cpp_dropin.py (or
// tests/cpp/build_ref_callers.sh) here, where /root/reference exists; the
// binary travels to the GPU box.
//
//   ref_callers verify <which> <n_max> <rho>    -> verify_strategies lines, exit 0 iff all ok
//   ref_callers suite <kernel> <csv> N...       -> run_suite (all strategies, d=3, reps=3,
//                                                  verify_cap=4096), CSV to <csv>
//   ref_callers sweep <n_blocks>                -> ltm_exactness_sweep per engine (repair off)
//   ref_callers perpass <N> <rho>               -> launch_count(rec) per_pass stats
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "trigrid/bench.hpp"
#include "trigrid/checks.hpp"

using namespace trigrid;

int main(int argc, char** argv) {
    if (argc >= 5 && std::strcmp(argv[1], "verify") == 0) {
        const VerifySummary s = verify_strategies(argv[2], std::strtoull(argv[3], nullptr, 10),
                                                  (std::uint32_t)std::strtoul(argv[4], nullptr, 10));
        for (const std::string& l : s.lines) std::printf("%s\n", l.c_str());
        std::printf("verify %s\n", s.ok ? "OK" : "FAILED");
        return s.ok ? 0 : 1;
    }
    if (argc >= 5 && std::strcmp(argv[1], "suite") == 0) {
        BenchConfig cfg;
        cfg.strategies = all_strategies();
        for (int a = 4; a < argc; ++a) cfg.n_values.push_back(std::strtoull(argv[a], nullptr, 10));
        cfg.kernel = std::strcmp(argv[2], "edm") == 0 ? KernelSpec::Kind::Edm : KernelSpec::Kind::Dummy;
        cfg.features = 3;
        cfg.repetitions = 3;
        cfg.verify_cap = 4096;
        const SuiteResult r = run_suite(cfg);
        emit_csv(r.records, argv[3]);
        for (const std::string& s : r.skipped) std::printf("skipped %s\n", s.c_str());
        std::printf("records %zu all_verified %d\n", r.records.size(), (int)r.all_verified);
        return r.all_verified ? 0 : 1;
    }
    if (argc >= 3 && std::strcmp(argv[1], "sweep") == 0) {
        const std::uint64_t nb = std::strtoull(argv[2], nullptr, 10);
        for (const SqrtVariant v : {SqrtVariant::NativeSingle, SqrtVariant::NewtonRaphson, SqrtVariant::Reciprocal,
                                    SqrtVariant::ExactInteger})
            for (const bool diag : {true, false}) {
                const ExactnessResult e = ltm_exactness_sweep(nb, engine_for(v), diag);
                std::printf("%s %d %llu %llu %llu\n", to_string(v), (int)diag, (unsigned long long)e.checked,
                            (unsigned long long)e.mismatches, (unsigned long long)e.first_mismatch);
            }
        return 0;
    }
    if (argc >= 4 && std::strcmp(argv[1], "perpass") == 0) {
        const std::uint64_t n = std::strtoull(argv[2], nullptr, 10);
        const std::uint32_t rho = (std::uint32_t)std::strtoul(argv[3], nullptr, 10);
        const AnyStrategy s = make_strategy(*parse_strategy("rec"), ProblemSize{n, rho});
        std::vector<std::uint32_t> counts(tri_count(n, true), 0);
        std::vector<DispatchStats> pp;
        const DispatchStats t = launch_count(s, counts, {0, &pp});
        for (const DispatchStats& p : pp)
            std::printf("pass %llu %llu %llu %llu\n", (unsigned long long)p.blocks_launched,
                        (unsigned long long)p.blocks_discarded, (unsigned long long)p.threads_discarded,
                        (unsigned long long)p.wall_time_ns);
        std::printf("total %llu %llu %llu\n", (unsigned long long)t.blocks_launched,
                    (unsigned long long)t.blocks_discarded, (unsigned long long)t.threads_discarded);
        std::uint64_t bad = 0;
        for (const std::uint32_t c : counts) bad += c != 1;
        std::printf("bad %llu\n", (unsigned long long)bad);
        return bad ? 1 : 0;
    }
    std::fprintf(stderr, "usage: ref_callers verify|suite|sweep|perpass ...\n");
    return 2;
}
