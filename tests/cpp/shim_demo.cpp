// shim_demo.cpp -- a reference-style C++ caller of the B200 library through
// include/trigrid_b200.hpp (the code a user of trigrid::launch_edm writes,
// namespace swapped).  Built and run by tests/test_cpp_shim.py.
//
//   shim_demo host            -- host-only API checks (no GPU needed)
//   shim_demo edm N d out.bin -- launch_edm on the GPU, raw packed fp32 to out.bin
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "trigrid_b200.hpp"

namespace tb = trigrid_b200;

static int host_checks() {
    int fails = 0;
    auto expect = [&](bool c, const char* what) {
        if (!c) {
            std::printf("FAIL %s\n", what);
            ++fails;
        }
    };
    expect(tb::tri_count(4) == 10, "tri_count(4)");
    expect(tb::tri_linear_index({2, 1}) == 4, "tri_linear_index(2,1)");
    expect(tb::grid_side_balanced(1920) == 1358, "grid_side_balanced(1920)");
    expect(tb::ltm_map(4, tb::SqrtEngine::reciprocal()) == tb::TriCoord{2, 1}, "ltm_map(4)");
    expect(tb::ltm_map(1844159, tb::SqrtEngine::reciprocal()) == tb::TriCoord{1919, 1919}, "ltm_map(1844159)");
    expect(tb::count_wasted(tb::StrategyKind::BoundingBox, 1920) == 1842240, "count_wasted(bb,1920)");
    expect(!tb::parse_strategy("zz").has_value(), "parse_strategy(zz)");
    bool threw = false;
    try {
        tb::make_strategy(*tb::parse_strategy("rec"), tb::ProblemSize{100, 16});
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, "rec N=100 throws invalid_argument");
    threw = false;
    try {
        tb::tri_linear_index({1, 2});
    } catch (const std::out_of_range&) {
        threw = true;
    }
    expect(threw, "tri_linear_index j>i throws out_of_range");
    threw = false;
    try {
        tb::ProblemSize(0, 16);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, "ProblemSize(0) throws");
    std::printf(fails ? "host checks FAILED\n" : "host checks ok\n");
    return fails ? 1 : 0;
}

int main(int argc, char** argv) {
    if (argc >= 2 && std::strcmp(argv[1], "host") == 0) return host_checks();
    if (argc >= 5 && std::strcmp(argv[1], "edm") == 0) {
        const std::uint64_t n = std::strtoull(argv[2], nullptr, 10);
        const std::uint32_t d = (std::uint32_t)std::strtoul(argv[3], nullptr, 10);
        const tb::PointSet pts = tb::gen_points(n, d, 42);
        const tb::AnyStrategy s = tb::make_strategy(*tb::parse_strategy("ltm-r"), tb::ProblemSize{n, 16});
        tb::PackedEdm out = tb::PackedEdm::zeros(n);
        const tb::DispatchStats st = tb::launch_edm(s, pts, out);
        std::printf("launched %llu discarded %llu threads_discarded %llu\n",
                    (unsigned long long)st.blocks_launched, (unsigned long long)st.blocks_discarded,
                    (unsigned long long)st.threads_discarded);
        std::FILE* f = std::fopen(argv[4], "wb");
        std::fwrite(out.values.data(), sizeof(float), out.values.size(), f);
        std::fclose(f);
        std::printf("coverage %d\n", (int)tb::coverage_ok(s));
        return 0;
    }
    std::fprintf(stderr, "usage: shim_demo host | edm N d out.bin\n");
    return 2;
}
