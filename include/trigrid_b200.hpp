// trigrid_b200.hpp -- header-only C++ drop-in over the C-ABI (trigrid_b200.h).
//
// Mirrors the reference's C++ engine surface so a caller of
//   /root/reference/proj/include/trigrid/engine.hpp:59-78     (launch_*)
//   /root/reference/proj/include/trigrid/strategies.hpp:393-400 (make_strategy)
//   /root/reference/proj/include/trigrid/edm.hpp:13-53        (PointSet, PackedEdm)
// switches by changing the include and the namespace (trigrid -> trigrid_b200).
// Same names, argument meaning and exception classes (std::invalid_argument,
// std::out_of_range, std::runtime_error); the work runs on a B200.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "trigrid_b200.h"

namespace trigrid_b200 {

inline void check(tg_status s) {
    if (s == TG_OK) return;
    const std::string msg = tg_last_error();
    switch (s) {
        case TG_EINVAL: throw std::invalid_argument(msg);
        case TG_ERANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

// tri.hpp:11-41
inline constexpr std::uint64_t kMaxElems = std::uint64_t{1} << 20;
struct TriCoord {
    std::uint64_t i = 0, j = 0;
    friend bool operator==(const TriCoord&, const TriCoord&) = default;
};
class ProblemSize {
public:
    ProblemSize(std::uint64_t elems, std::uint32_t rho) : elems_(elems), rho_(rho) {
        if (elems == 0) throw std::invalid_argument("ProblemSize: N must be >= 1");
        if (elems > kMaxElems) throw std::invalid_argument("ProblemSize: N exceeds the 2^20 cap");
        if (rho == 0) throw std::invalid_argument("ProblemSize: rho must be >= 1");
    }
    std::uint64_t elems() const noexcept { return elems_; }
    std::uint32_t rho() const noexcept { return rho_; }
    std::uint64_t blocks() const noexcept { return (elems_ + rho_ - 1) / rho_; }

private:
    std::uint64_t elems_;
    std::uint32_t rho_;
};
inline std::uint64_t tri_count(std::uint64_t n, bool with_diag = true) { return tg_tri_count(n, with_diag); }
inline std::uint64_t tri_linear_index(TriCoord c) {
    std::uint64_t v;
    check(tg_tri_linear_index(c.i, c.j, &v));
    return v;
}
inline std::uint64_t grid_side_balanced(std::uint64_t n) {
    std::uint64_t v;
    check(tg_grid_side_balanced(n, &v));
    return v;
}

// strategies.hpp:27-36, strategies.cpp:19-28
struct StrategyId {
    tg_strategy id = TG_BB;
    friend bool operator==(const StrategyId&, const StrategyId&) = default;
};
inline std::optional<StrategyId> parse_strategy(std::string_view name) noexcept {
    tg_strategy s;
    if (tg_parse_strategy(std::string(name).c_str(), &s) != TG_OK) return std::nullopt;
    return StrategyId{s};
}

// AnyStrategy / make_strategy (strategies.hpp:393-400): the strategy plus its
// problem size; construction validates exactly like the reference's
// constructors (e.g. rec throws when N != m*2^k).
struct AnyStrategy {
    StrategyId id;
    ProblemSize size;
};
inline AnyStrategy make_strategy(const StrategyId& id, ProblemSize size) {
    tg_dispatch_stats st;
    check(tg_dispatch_stats_for(id.id, size.elems(), size.rho(), 0, 1, &st));
    return AnyStrategy{id, size};
}

inline TriCoord ltm_map(std::uint64_t lambda, int engine = 2, bool with_diag = true) {
    TriCoord c;
    check(tg_ltm_map(lambda, engine, with_diag, &c.i, &c.j));
    return c;
}

// edm.hpp:13-49
struct PointSet {
    std::uint64_t count = 0;
    std::uint32_t features = 0;
    std::vector<float> data;
};
inline PointSet gen_points(std::uint64_t n, std::uint32_t d, std::uint64_t seed) {
    PointSet p{n, d, std::vector<float>(n * d)};
    check(tg_gen_points_host(n, d, seed, p.data.data(), -1));
    return p;
}
struct PackedEdm {
    std::uint64_t count = 0;
    std::vector<float> values;
    static PackedEdm zeros(std::uint64_t n) { return {n, std::vector<float>(tri_count(n, true), 0.0f)}; }
    float at(std::uint64_t i, std::uint64_t j) const { return values[tri_linear_index({i, j})]; }
};

// engine.hpp:19-37
struct DispatchStats {
    std::uint64_t blocks_launched = 0, blocks_discarded = 0, threads_discarded = 0, wall_time_ns = 0;
};
struct LaunchOptions {
    unsigned workers = 0;  // accepted for source compatibility; the GPU ignores it
    int device = -1;
    tg_mode mode = TG_MODE_AUTO;
};

inline DispatchStats to_stats(const tg_dispatch_stats& s) {
    return {s.blocks_launched, s.blocks_discarded, s.threads_discarded, s.wall_time_ns};
}

// launch_edm (engine.cpp:157-175): same validation, host buffers in/out.
inline DispatchStats launch_edm(const AnyStrategy& strategy, const PointSet& points, PackedEdm& out,
                                const LaunchOptions& opt = {}) {
    const std::uint64_t n = strategy.size.elems();
    if (points.count != n)
        throw std::invalid_argument("launch_edm: point count does not match the strategy's N");
    if (points.features < 1 || points.features > 4)
        throw std::invalid_argument("launch_edm: features must be in [1, 4]");
    if (points.data.size() != points.count * points.features)
        throw std::invalid_argument("launch_edm: point data size mismatch");
    if (out.count != n || out.values.size() != tri_count(n, true))
        throw std::invalid_argument("launch_edm: output buffer is not N(N+1)/2 packed cells");
    tg_launch_opts o;
    tg_launch_opts_init(&o);
    o.device = opt.device;
    o.mode = opt.mode;
    tg_dispatch_stats st;
    check(tg_edm_strategy_host(strategy.id.id, points.data.data(), n, points.features,
                               strategy.size.rho(), out.values.data(), &o, &st));
    return to_stats(st);
}

// check_cell_coverage (checks.cpp:16-38) -> bool, on device.
inline bool coverage_ok(const AnyStrategy& strategy, int device = -1) {
    int ok = 0;
    check(tg_coverage_ok(strategy.id.id, strategy.size.elems(), strategy.size.rho(), device, &ok));
    return ok != 0;
}

// count_wasted (engine.cpp:205-217)
inline std::uint64_t count_wasted(const StrategyId& id, std::uint64_t n) {
    std::uint64_t v;
    check(tg_count_wasted(id.id, n, &v));
    return v;
}

}  // namespace trigrid_b200
