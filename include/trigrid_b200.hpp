// trigrid_b200.hpp -- header-only C++ drop-in over the C-ABI (trigrid_b200.h).
//
// Source-compatible with the reference's C++ API surface
//   tri.hpp:11-107        TriCoord, ProblemSize, tri_count, tri_linear_index,
//                         grid_side_balanced, enumerate_lower
//   fastmath.hpp:13-103   isqrt, ceil_sqrt, fast_inv_sqrt, rsqrt_single, SqrtVariant,
//                         SqrtEngine, sqrt_via, RepairPolicy, repair_lower_row
//   strategies.hpp:15-402 StrategyKind/StrategyId/parse_strategy/strategy_name,
//                         the mappers (bb_map, ltm_map, utm_map, rb_map, rec_schedule,
//                         ...), the five strategy classes, AnyStrategy,
//                         make_strategy, grid_of
//   edm.hpp:13-64         PointSet, gen_points, edm_pair, PackedEdm, edm_reference,
//                         save/load_packed_edm
//   engine.hpp:13-87      KernelSpec, DispatchStats, LaunchOptions, DummySink,
//                         launch_dummy / launch_edm / launch_count / launch,
//                         count_wasted, ltm_diag_waste_blocks
// with the same names, argument meaning and exception classes
// (std::invalid_argument, std::out_of_range, std::runtime_error).  The
// launches run the sm_100a kernels of libtrigrid_b200.so.
//
// Namespace: trigrid_b200 by default.  Defining TRIGRID_B200_NS=trigrid
// before the include (what include/trigrid_compat/trigrid/*.hpp do) puts the
// same declarations into namespace trigrid, so the reference's own callers
// (proj/src/bench.cpp run_suite, proj/src/checks.cpp verify_strategies) compile
// unmodified against it (tests/test_cpp_dropin.py).
//
// Host-side pieces stay host code exactly as in the reference: the scalar
// mappers (through the library's host entry points), PEDM file I/O, and
// edm_reference -- the reference API's sequential oracle, which launch_edm
// results are verified against (never a fallback for the device path).
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <compare>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <variant>
#include <vector>

#include "trigrid_b200.h"

#ifndef TRIGRID_B200_NS
#define TRIGRID_B200_NS trigrid_b200
#endif

namespace TRIGRID_B200_NS {

namespace detail {
inline void check(tg_status s) {
    if (s == TG_OK) return;
    const std::string msg = tg_last_error();
    switch (s) {
        case TG_EINVAL: throw std::invalid_argument(msg);
        case TG_ERANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}
}  // namespace detail

// ============================================================ tri.hpp

inline constexpr std::uint64_t kMaxElems = std::uint64_t{1} << 20;

struct TriCoord {
    std::uint64_t i = 0;
    std::uint64_t j = 0;
    friend bool operator==(const TriCoord&, const TriCoord&) = default;
    friend auto operator<=>(const TriCoord&, const TriCoord&) = default;
};

class ProblemSize {
public:
    ProblemSize(std::uint64_t elems, std::uint32_t rho) : elems_(elems), rho_(rho) {
        tg_dispatch_stats st;  // the library's ProblemSize checks (tri.cpp:9-15)
        if (elems == 0 || elems > kMaxElems || rho == 0) detail::check(tg_dispatch_stats_for(TG_BB, elems, rho, 0, 1, &st));
    }
    std::uint64_t elems() const noexcept { return elems_; }
    std::uint32_t rho() const noexcept { return rho_; }
    std::uint64_t blocks() const noexcept { return (elems_ + rho_ - 1) / rho_; }

private:
    std::uint64_t elems_;
    std::uint32_t rho_;
};

constexpr std::uint64_t tri_count(std::uint64_t n, bool with_diag = true) noexcept {
    return with_diag ? n * (n + 1) / 2 : (n == 0 ? 0 : n * (n - 1) / 2);
}

inline std::uint64_t tri_linear_index(TriCoord c) {
    std::uint64_t v;
    detail::check(tg_tri_linear_index(c.i, c.j, &v));
    return v;
}

inline std::uint64_t grid_side_balanced(std::uint64_t n) {
    std::uint64_t v;
    detail::check(tg_grid_side_balanced(n, &v));
    return v;
}

// Lazy lower-triangle walk in ascending lambda order (tri.hpp:53-105).
class LowerTriRange {
public:
    class iterator {
    public:
        using value_type = TriCoord;
        using difference_type = std::ptrdiff_t;
        using iterator_category = std::forward_iterator_tag;
        iterator() = default;
        TriCoord operator*() const noexcept { return at_; }
        iterator& operator++() noexcept {
            const std::uint64_t width = diag_ ? at_.i + 1 : at_.i;
            if (++at_.j >= width) at_ = TriCoord{at_.i + 1, 0};
            return *this;
        }
        iterator operator++(int) noexcept {
            iterator old = *this;
            ++*this;
            return old;
        }
        friend bool operator==(const iterator& a, const iterator& b) noexcept { return a.at_ == b.at_; }

    private:
        friend class LowerTriRange;
        iterator(TriCoord at, bool diag) : at_(at), diag_(diag) {}
        TriCoord at_{};
        bool diag_ = true;
    };
    LowerTriRange(std::uint64_t n, bool with_diag) noexcept : n_(n), diag_(with_diag) {}
    iterator begin() const noexcept {
        return size() ? iterator{TriCoord{diag_ ? 0u : 1u, 0}, diag_} : end();
    }
    iterator end() const noexcept { return iterator{TriCoord{n_, 0}, diag_}; }
    std::uint64_t size() const noexcept { return tri_count(n_, diag_); }

private:
    std::uint64_t n_;
    bool diag_;
};

inline LowerTriRange enumerate_lower(std::uint64_t n, bool with_diag = true) noexcept {
    return LowerTriRange{n, with_diag};
}

// ======================================================== fastmath.hpp

inline std::uint64_t isqrt(std::uint64_t v) noexcept { return tg_isqrt(v); }
inline std::uint64_t ceil_sqrt(std::uint64_t v) noexcept {
    const std::uint64_t r = tg_isqrt(v);
    return r * r == v ? r : r + 1;
}
inline float fast_inv_sqrt(float x, int iterations) noexcept { return tg_fast_inv_sqrt(x, iterations); }
inline float rsqrt_single(float x) noexcept { return tg_rsqrt_single(x); }

enum class SqrtVariant : std::uint8_t { NativeSingle, NewtonRaphson, Reciprocal, ExactInteger };
inline constexpr float kRepairEpsilon = 1e-4f;

struct SqrtEngine {
    SqrtVariant variant = SqrtVariant::Reciprocal;
    float epsilon = kRepairEpsilon;
    static constexpr SqrtEngine native_single() { return {SqrtVariant::NativeSingle, 0.0f}; }
    static constexpr SqrtEngine newton_raphson() { return {SqrtVariant::NewtonRaphson, kRepairEpsilon}; }
    static constexpr SqrtEngine reciprocal() { return {SqrtVariant::Reciprocal, kRepairEpsilon}; }
    static constexpr SqrtEngine exact_integer() { return {SqrtVariant::ExactInteger, 0.0f}; }
};

inline const char* to_string(SqrtVariant v) noexcept {
    static const char* const names[] = {"native-single", "newton-raphson", "reciprocal", "exact-integer"};
    const auto k = static_cast<unsigned>(v);
    return k < 4 ? names[k] : "?";
}

inline double sqrt_via(const SqrtEngine& engine, double x) {
    double out;
    detail::check(tg_sqrt_via(static_cast<int>(engine.variant), x, &out));
    return out;
}

inline constexpr std::uint64_t kRepairFreeLambdaLimit = 1'844'160;
enum class RepairPolicy : std::uint8_t { Auto, Off, On };

inline std::uint64_t repair_lower_row(std::uint64_t i, std::uint64_t lambda, bool with_diag) noexcept {
    auto start = [with_diag](std::uint64_t r) { return with_diag ? r * (r + 1) / 2 : r * (r - 1) / 2; };
    const std::uint64_t lo = with_diag ? 0 : 1;
    i = std::max(i, lo);
    for (; i > lo && start(i) > lambda; --i) {
    }
    for (; start(i + 1) <= lambda; ++i) {
    }
    return i;
}

// ====================================================== strategies.hpp

enum class StrategyKind : std::uint8_t { BoundingBox, LowerTri, UpperTri, RectBox, Recursive };

inline const char* to_string(StrategyKind k) noexcept {
    static const char* const names[] = {"bb", "ltm", "utm", "rb", "rec"};
    const auto v = static_cast<unsigned>(k);
    return v < 5 ? names[v] : "?";
}

struct StrategyId {
    StrategyKind kind = StrategyKind::BoundingBox;
    SqrtVariant engine = SqrtVariant::Reciprocal;
    friend bool operator==(const StrategyId&, const StrategyId&) = default;
};

inline std::optional<StrategyId> parse_strategy(std::string_view name) noexcept {
    struct Row {
        std::string_view name;
        StrategyId id;
    };
    static constexpr Row rows[] = {
        {"bb", {StrategyKind::BoundingBox, SqrtVariant::NativeSingle}},
        {"ltm-x", {StrategyKind::LowerTri, SqrtVariant::NativeSingle}},
        {"ltm-n", {StrategyKind::LowerTri, SqrtVariant::NewtonRaphson}},
        {"ltm-r", {StrategyKind::LowerTri, SqrtVariant::Reciprocal}},
        {"utm", {StrategyKind::UpperTri, SqrtVariant::NewtonRaphson}},
        {"rb", {StrategyKind::RectBox, SqrtVariant::NativeSingle}},
        {"rec", {StrategyKind::Recursive, SqrtVariant::NativeSingle}},
    };
    for (const Row& r : rows)
        if (r.name == name) return r.id;
    return std::nullopt;
}

inline std::string strategy_name(const StrategyId& id) {
    if (id.kind != StrategyKind::LowerTri) return to_string(id.kind);
    static const char* const ltm[] = {"ltm-x", "ltm-n", "ltm-r", "ltm-exact"};
    return ltm[static_cast<unsigned>(id.engine) & 3];
}

inline std::vector<StrategyId> all_strategies() {
    std::vector<StrategyId> v;
    for (const char* n : {"bb", "ltm-x", "ltm-n", "ltm-r", "utm", "rb", "rec"}) v.push_back(*parse_strategy(n));
    return v;
}

inline SqrtEngine engine_for(SqrtVariant v) noexcept {
    switch (v) {
        case SqrtVariant::NativeSingle: return SqrtEngine::native_single();
        case SqrtVariant::NewtonRaphson: return SqrtEngine::newton_raphson();
        case SqrtVariant::ExactInteger: return SqrtEngine::exact_integer();
        default: return SqrtEngine::reciprocal();
    }
}

struct RecLevel {
    std::uint32_t level = 0;
    std::uint64_t side = 0;
    std::uint64_t squares = 0;
};
struct Pass {
    std::uint64_t blocks_x = 0;
    std::uint64_t blocks_y = 0;
    std::optional<RecLevel> level_tag;
};
struct GridSpec {
    StrategyKind strategy = StrategyKind::BoundingBox;
    std::uint32_t rho = 1;
    std::vector<Pass> passes;
    std::uint64_t total_blocks() const noexcept {
        std::uint64_t t = 0;
        for (const Pass& p : passes) t += p.blocks_x * p.blocks_y;
        return t;
    }
};

struct BlockCoord {
    std::uint64_t x = 0;
    std::uint64_t y = 0;
};

class MapOutcome {
public:
    static MapOutcome mapped(TriCoord c) noexcept { return MapOutcome{c, true}; }
    static MapOutcome discard() noexcept { return MapOutcome{{}, false}; }
    bool is_mapped() const noexcept { return ok_; }
    TriCoord coord() const noexcept { return c_; }

private:
    MapOutcome(TriCoord c, bool ok) : c_(c), ok_(ok) {}
    TriCoord c_;
    bool ok_;
};

inline MapOutcome bb_map(BlockCoord b) noexcept {
    std::uint64_t i, j;
    return tg_bb_map(b.x, b.y, &i, &j) ? MapOutcome::mapped({i, j}) : MapOutcome::discard();
}

// g(lambda) with the reference's repair policy: host binary32 arithmetic
// identical to strategies.cpp:60-83 (tg_ltm_map_policy).
inline TriCoord ltm_map(std::uint64_t lambda, const SqrtEngine& engine, bool with_diag = true,
                        RepairPolicy repair = RepairPolicy::Auto) {
    TriCoord c;
    detail::check(tg_ltm_map_policy(lambda, static_cast<int>(engine.variant), with_diag,
                                    static_cast<int>(repair), &c.i, &c.j));
    return c;
}

inline std::optional<std::uint64_t> ltm_block_to_lambda(BlockCoord b, std::uint64_t n_prime,
                                                        std::uint64_t block_count) noexcept {
    const std::uint64_t lam = b.y * n_prime + b.x;
    return lam < block_count ? std::optional<std::uint64_t>{lam} : std::nullopt;
}

struct UtmPair {
    std::uint64_t a = 0;
    std::uint64_t b = 0;
};
inline UtmPair utm_map(std::uint64_t k, std::uint64_t n_elems, const SqrtEngine& engine) {
    UtmPair p;
    detail::check(tg_utm_map(k, n_elems, static_cast<int>(engine.variant), &p.a, &p.b));
    return p;
}
// disc_base is implied by n ((2n-1)^2); kept for signature compatibility.
inline UtmPair utm_pair_unchecked(std::uint64_t k, std::uint64_t n, std::uint64_t /*disc_base*/,
                                  const SqrtEngine& engine) noexcept {
    UtmPair p;
    if (tg_utm_map(k, n, static_cast<int>(engine.variant), &p.a, &p.b) != TG_OK) return UtmPair{};
    return p;
}

struct RbRect {
    std::uint64_t width = 0;
    std::uint64_t height = 0;
};
inline RbRect rb_rect(std::uint64_t n_elems) {
    RbRect r;
    detail::check(tg_rb_rect(n_elems, &r.width, &r.height));
    return r;
}
inline MapOutcome rb_map(std::uint64_t tx, std::uint64_t ty, std::uint64_t n_elems) noexcept {
    std::uint64_t i, j;
    return tg_rb_map(tx, ty, n_elems, &i, &j) ? MapOutcome::mapped({i, j}) : MapOutcome::discard();
}

namespace detail {
inline GridSpec grid_spec(tg_strategy s, StrategyKind kind, std::uint64_t n, std::uint32_t rho, std::uint64_t m = 0,
                          std::uint32_t k = 0) {
    tg_launch_opts o;
    tg_launch_opts_init(&o);
    o.rec_m = m;
    o.rec_k = k;
    std::uint32_t np = 0;
    check(tg_grid_spec(s, n, rho, &o, nullptr, 0, &np));
    std::vector<tg_pass> v(np);
    check(tg_grid_spec(s, n, rho, &o, v.data(), np, &np));
    GridSpec g{kind, rho, {}};
    for (const tg_pass& p : v) {
        Pass q{p.blocks_x, p.blocks_y, std::nullopt};
        if (p.has_level) q.level_tag = RecLevel{p.level, p.side, p.squares};
        g.passes.push_back(q);
    }
    return g;
}
}  // namespace detail

inline GridSpec rb_grid(std::uint64_t n_elems, std::uint32_t rho) {
    return detail::grid_spec(TG_RB, StrategyKind::RectBox, n_elems, rho);
}

struct RecSchedule {
    std::uint64_t m = 0;
    std::uint32_t k = 0;
    GridSpec grid;
};
inline RecSchedule rec_schedule(std::uint64_t n_elems, std::uint64_t m, std::uint32_t k, std::uint32_t rho) {
    return RecSchedule{m, k, detail::grid_spec(TG_REC, StrategyKind::Recursive, n_elems, rho, m, k)};
}

inline std::optional<std::pair<std::uint64_t, std::uint32_t>> rec_decompose(std::uint64_t n_elems,
                                                                            std::uint32_t rho) noexcept {
    std::uint64_t m;
    std::uint32_t k;
    if (!tg_rec_decompose(n_elems, rho, &m, &k)) return std::nullopt;
    return std::make_pair(m, k);
}

inline TriCoord rec_block_map(std::uint64_t m, std::uint32_t level, std::uint64_t square, BlockCoord local,
                              std::uint32_t rho) noexcept {
    const std::uint64_t side = m << (level - 1);
    return {(2 * square + 1) * side + local.y * rho, 2 * square * side + local.x * rho};
}

struct BlockDecision {
    enum class Kind : std::uint8_t { Discard, FullTile, DiagTile, ThreadMapped };
    Kind kind = Kind::Discard;
    std::uint64_t origin_i = 0;
    std::uint64_t origin_j = 0;
    static BlockDecision discard() noexcept { return {Kind::Discard, 0, 0}; }
    static BlockDecision full(std::uint64_t i, std::uint64_t j) noexcept { return {Kind::FullTile, i, j}; }
    static BlockDecision diag(std::uint64_t i, std::uint64_t j) noexcept { return {Kind::DiagTile, i, j}; }
    static BlockDecision threads() noexcept { return {Kind::ThreadMapped, 0, 0}; }
};

// The strategy objects carry what a launch needs (problem size, engine, REC
// schedule) plus the host-side decide / map_thread of process_block
// (engine.cpp:17-68).  The device kernels implement the same decisions.
namespace detail {
inline BlockDecision tile_decision(TriCoord blk, std::uint32_t rho) {
    const std::uint64_t oi = blk.i * rho, oj = blk.j * rho;
    return blk.i == blk.j ? BlockDecision::diag(oi, oj) : BlockDecision::full(oi, oj);
}
}  // namespace detail

class BbStrategy {
public:
    explicit BbStrategy(ProblemSize size)
        : size_(size), grid_(detail::grid_spec(TG_BB, StrategyKind::BoundingBox, size.elems(), size.rho())) {}
    const GridSpec& grid() const noexcept { return grid_; }
    const ProblemSize& size() const noexcept { return size_; }
    BlockDecision decide(std::size_t, std::uint64_t bx, std::uint64_t by) const noexcept {
        const MapOutcome o = bb_map({bx, by});
        return o.is_mapped() ? detail::tile_decision(o.coord(), size_.rho()) : BlockDecision::discard();
    }
    std::optional<TriCoord> map_thread(std::size_t, std::uint64_t, std::uint64_t, std::uint32_t,
                                       std::uint32_t) const noexcept {
        return std::nullopt;
    }

private:
    ProblemSize size_;
    GridSpec grid_;
};

class LtmStrategy {
public:
    LtmStrategy(ProblemSize size, SqrtEngine engine)
        : size_(size),
          engine_(engine),
          n_prime_(grid_side_balanced(size.blocks())),
          block_count_(tri_count(size.blocks(), true)),
          grid_{StrategyKind::LowerTri, size.rho(), {Pass{n_prime_, n_prime_, std::nullopt}}} {}
    const GridSpec& grid() const noexcept { return grid_; }
    const ProblemSize& size() const noexcept { return size_; }
    const SqrtEngine& engine() const noexcept { return engine_; }
    std::uint64_t balanced_side() const noexcept { return n_prime_; }
    BlockDecision decide(std::size_t, std::uint64_t bx, std::uint64_t by) const {
        const auto lam = ltm_block_to_lambda({bx, by}, n_prime_, block_count_);
        return lam ? detail::tile_decision(ltm_map(*lam, engine_), size_.rho()) : BlockDecision::discard();
    }
    std::optional<TriCoord> map_thread(std::size_t, std::uint64_t, std::uint64_t, std::uint32_t,
                                       std::uint32_t) const noexcept {
        return std::nullopt;
    }

private:
    ProblemSize size_;
    SqrtEngine engine_;
    std::uint64_t n_prime_;
    std::uint64_t block_count_;
    GridSpec grid_;
};

class UtmStrategy {
public:
    UtmStrategy(ProblemSize size, SqrtEngine engine)
        : size_(size),
          engine_(engine),
          pair_count_(tri_count(size.elems(), false)),
          grid_(detail::grid_spec(TG_UTM, StrategyKind::UpperTri, size.elems(), size.rho())) {}
    const GridSpec& grid() const noexcept { return grid_; }
    const ProblemSize& size() const noexcept { return size_; }
    const SqrtEngine& engine() const noexcept { return engine_; }
    std::uint64_t pair_count() const noexcept { return pair_count_; }
    BlockDecision decide(std::size_t, std::uint64_t, std::uint64_t) const noexcept { return BlockDecision::threads(); }
    std::optional<TriCoord> map_thread(std::size_t, std::uint64_t bx, std::uint64_t by, std::uint32_t sx,
                                       std::uint32_t sy) const {
        const std::uint64_t rho = size_.rho();
        const std::uint64_t k = ((by * grid_.passes[0].blocks_x + bx) * rho + sy) * rho + sx;
        if (k >= pair_count_) return std::nullopt;
        const UtmPair p = utm_map(k, size_.elems(), engine_);
        return TriCoord{p.b, p.a};  // transposed onto the lower triangle
    }

private:
    ProblemSize size_;
    SqrtEngine engine_;
    std::uint64_t pair_count_;
    GridSpec grid_;
};

class RbStrategy {
public:
    explicit RbStrategy(ProblemSize size)
        : size_(size), rect_(rb_rect(size.elems())), grid_(rb_grid(size.elems(), size.rho())) {}
    const GridSpec& grid() const noexcept { return grid_; }
    const ProblemSize& size() const noexcept { return size_; }
    const RbRect& rect() const noexcept { return rect_; }
    BlockDecision decide(std::size_t, std::uint64_t, std::uint64_t) const noexcept { return BlockDecision::threads(); }
    std::optional<TriCoord> map_thread(std::size_t, std::uint64_t bx, std::uint64_t by, std::uint32_t sx,
                                       std::uint32_t sy) const noexcept {
        const MapOutcome o = rb_map(bx * size_.rho() + sx, by * size_.rho() + sy, size_.elems());
        return o.is_mapped() ? std::optional<TriCoord>{o.coord()} : std::nullopt;
    }

private:
    ProblemSize size_;
    RbRect rect_;
    GridSpec grid_;
};

class RecStrategy {
public:
    RecStrategy(ProblemSize size, RecSchedule schedule) : size_(size), schedule_(std::move(schedule)) {}
    const GridSpec& grid() const noexcept { return schedule_.grid; }
    const ProblemSize& size() const noexcept { return size_; }
    const RecSchedule& schedule() const noexcept { return schedule_; }
    BlockDecision decide(std::size_t pass, std::uint64_t bx, std::uint64_t by) const noexcept {
        const std::uint32_t rho = size_.rho();
        const std::uint64_t m = schedule_.m;
        if (pass < schedule_.k) {  // square level pass + 1
            const auto level = static_cast<std::uint32_t>(pass + 1);
            const std::uint64_t sb = (m << (level - 1)) / rho;
            const TriCoord o = rec_block_map(m, level, by / sb, {bx, by % sb}, rho);
            return BlockDecision::full(o.i, o.j);
        }
        const std::uint64_t sb = m / rho, t = by / sb, ly = by % sb;  // diagonal pass
        if (bx > ly) return BlockDecision::discard();
        const std::uint64_t oi = t * m + ly * rho, oj = t * m + bx * rho;
        return bx == ly ? BlockDecision::diag(oi, oj) : BlockDecision::full(oi, oj);
    }
    std::optional<TriCoord> map_thread(std::size_t, std::uint64_t, std::uint64_t, std::uint32_t,
                                       std::uint32_t) const noexcept {
        return std::nullopt;
    }

private:
    ProblemSize size_;
    RecSchedule schedule_;
};

using AnyStrategy = std::variant<BbStrategy, LtmStrategy, UtmStrategy, RbStrategy, RecStrategy>;

inline AnyStrategy make_strategy(const StrategyId& id, ProblemSize size) {
    switch (id.kind) {
        case StrategyKind::BoundingBox: return BbStrategy{size};
        case StrategyKind::LowerTri: return LtmStrategy{size, engine_for(id.engine)};
        case StrategyKind::UpperTri: return UtmStrategy{size, engine_for(id.engine)};
        case StrategyKind::RectBox: return RbStrategy{size};
        case StrategyKind::Recursive: {
            const auto mk = rec_decompose(size.elems(), size.rho());
            if (!mk) throw std::invalid_argument("rec: N is not m*2^k with m a multiple of rho");
            return RecStrategy{size, rec_schedule(size.elems(), mk->first, mk->second, size.rho())};
        }
    }
    throw std::invalid_argument("make_strategy: unknown strategy kind");
}

inline const GridSpec& grid_of(const AnyStrategy& s) noexcept {
    return std::visit([](const auto& x) -> const GridSpec& { return x.grid(); }, s);
}

// ============================================================= edm.hpp

struct PointSet {
    std::uint64_t count = 0;
    std::uint32_t features = 0;
    std::vector<float> data;
    const float* point(std::uint64_t idx) const noexcept { return data.data() + idx * features; }
};

// splitmix64 stream of the reference (edm.cpp:38-51), generated on device.
inline PointSet gen_points(std::uint64_t n, std::uint32_t d, std::uint64_t seed) {
    if (n == 0 || n > kMaxElems || d < 1 || d > 4) detail::check(tg_gen_points_host(n, d, seed, nullptr, -1));
    PointSet p{n, d, std::vector<float>(n * d)};
    detail::check(tg_gen_points_host(n, d, seed, p.data.data(), -1));
    return p;
}

inline float edm_pair(const float* a, const float* b, std::uint32_t d) noexcept {
    float acc = 0.0f;
    for (std::uint32_t k = 0; k < d; ++k) {
        const float t = a[k] - b[k];
        acc += t * t;
    }
    return std::sqrt(acc);
}

struct PackedEdm {
    std::uint64_t count = 0;
    std::vector<float> values;
    static PackedEdm zeros(std::uint64_t n) { return {n, std::vector<float>(tri_count(n, true), 0.0f)}; }
    float at(std::uint64_t i, std::uint64_t j) const { return values[tri_linear_index({i, j})]; }
};

// The sequential oracle (edm.cpp:53-63): host code by contract.
inline PackedEdm edm_reference(const PointSet& points) {
    PackedEdm out{points.count, std::vector<float>(tri_count(points.count, true))};
    detail::check(tg_edm_reference_host(points.data.data(), points.count, points.features, out.values.data()));
    return out;
}

// PEDM: "PEDM", u32 LE version 1, u32 N, u32 d, packed binary32 (edm.cpp:65-96).
namespace detail {
inline void put_le32(std::ostream& os, std::uint32_t v) {
    const char b[4] = {char(v & 0xff), char((v >> 8) & 0xff), char((v >> 16) & 0xff), char(v >> 24)};
    os.write(b, 4);
}
inline std::uint32_t get_le32(std::istream& is) {
    unsigned char b[4] = {0, 0, 0, 0};
    is.read(reinterpret_cast<char*>(b), 4);
    return std::uint32_t(b[0]) | std::uint32_t(b[1]) << 8 | std::uint32_t(b[2]) << 16 | std::uint32_t(b[3]) << 24;
}
}  // namespace detail

inline void save_packed_edm(const PackedEdm& edm, std::uint32_t features, const std::filesystem::path& path) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw std::runtime_error("cannot open for writing: " + path.string());
    os.write("PEDM", 4);
    detail::put_le32(os, 1);
    detail::put_le32(os, static_cast<std::uint32_t>(edm.count));
    detail::put_le32(os, features);
    os.write(reinterpret_cast<const char*>(edm.values.data()),
             static_cast<std::streamsize>(edm.values.size() * sizeof(float)));
    if (!os) throw std::runtime_error("write failed: " + path.string());
}

// Per-shard PEDM writing: create the full-size file once, then
// every shard writes its packed slice [elem_begin, elem_begin + count) at
// byte offset 16 + 4 elem_begin.
inline void create_packed_edm(std::uint64_t n, std::uint32_t features, const std::filesystem::path& path) {
    {
        std::ofstream os(path, std::ios::binary | std::ios::trunc);
        if (!os) throw std::runtime_error("cannot open for writing: " + path.string());
        os.write("PEDM", 4);
        detail::put_le32(os, 1);
        detail::put_le32(os, static_cast<std::uint32_t>(n));
        detail::put_le32(os, features);
        if (!os) throw std::runtime_error("write failed: " + path.string());
    }
    std::filesystem::resize_file(path, 16 + 4 * tri_count(n, true));
}
inline void save_packed_edm_slice(const float* values, std::uint64_t elem_begin, std::uint64_t count,
                                  const std::filesystem::path& path) {
    std::fstream f(path, std::ios::binary | std::ios::in | std::ios::out);
    if (!f) throw std::runtime_error("cannot open for writing: " + path.string());
    f.seekp(static_cast<std::streamoff>(16 + 4 * elem_begin));
    f.write(reinterpret_cast<const char*>(values), static_cast<std::streamsize>(count * sizeof(float)));
    if (!f) throw std::runtime_error("write failed: " + path.string());
}

struct PedmFile {
    PackedEdm edm;
    std::uint32_t features = 0;
};

inline PedmFile load_packed_edm(const std::filesystem::path& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::runtime_error("cannot open for reading: " + path.string());
    char magic[4] = {0, 0, 0, 0};
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "PEDM", 4) != 0) throw std::runtime_error("not a PEDM file: " + path.string());
    if (detail::get_le32(is) != 1) throw std::runtime_error("unsupported PEDM version");
    const std::uint32_t n = detail::get_le32(is), features = detail::get_le32(is);
    PedmFile f{PackedEdm::zeros(n), features};
    is.read(reinterpret_cast<char*>(f.edm.values.data()),
            static_cast<std::streamsize>(f.edm.values.size() * sizeof(float)));
    if (!is) throw std::runtime_error("truncated PEDM file: " + path.string());
    return f;
}

// ========================================================== engine.hpp

struct KernelSpec {
    enum class Kind : std::uint8_t { Dummy, Edm };
    Kind kind = Kind::Dummy;
    std::uint32_t features = 0;
};

struct DispatchStats {
    std::uint64_t blocks_launched = 0;
    std::uint64_t blocks_discarded = 0;
    std::uint64_t threads_discarded = 0;
    std::uint64_t wall_time_ns = 0;  // device time (CUDA events)
    DispatchStats& operator+=(const DispatchStats& o) noexcept {
        blocks_launched += o.blocks_launched;
        blocks_discarded += o.blocks_discarded;
        threads_discarded += o.threads_discarded;
        wall_time_ns += o.wall_time_ns;
        return *this;
    }
};

// The reference's two fields first (aggregate init `{workers, per_pass}`
// keeps compiling), then the B200 extensions.
struct LaunchOptions {
    unsigned workers = 0;                             // accepted for compatibility; the GPU ignores it
    std::vector<DispatchStats>* per_pass = nullptr;   // per grid pass, device-timed
    int device = -1;                                  // CUDA ordinal (-1 = current)
    tg_mode mode = TG_MODE_AUTO;
    std::vector<int> devices;                         // launch_edm: split over these GPUs
};

class DummySink {
public:
    void write(std::uint64_t v) noexcept { cell_.store(v, std::memory_order_relaxed); }
    std::uint64_t value() const noexcept { return cell_.load(std::memory_order_relaxed); }

private:
    alignas(64) std::atomic<std::uint64_t> cell_{0};
};

inline void dummy_kernel(TriCoord c, DummySink& sink) noexcept { sink.write(c.i + c.j); }

namespace detail {
// AnyStrategy -> the C-ABI strategy id and its launch options.
struct Target {
    tg_strategy s;
    tg_launch_opts o;
    std::uint64_t n;
    std::uint32_t rho;
};
inline tg_strategy ltm_id(SqrtVariant v) {
    switch (v) {
        case SqrtVariant::NativeSingle: return TG_LTM_X;
        case SqrtVariant::NewtonRaphson: return TG_LTM_N;
        case SqrtVariant::Reciprocal: return TG_LTM_R;
        default: return TG_LTM_EXACT;
    }
}
inline Target target(const AnyStrategy& st, const LaunchOptions& opt) {
    Target t{};
    tg_launch_opts_init(&t.o);
    t.o.device = opt.device;
    t.o.mode = opt.mode;
    std::visit(
        [&](const auto& x) {
            using S = std::decay_t<decltype(x)>;
            t.n = x.size().elems();
            t.rho = x.size().rho();
            if constexpr (std::is_same_v<S, BbStrategy>) {
                t.s = TG_BB;
            } else if constexpr (std::is_same_v<S, LtmStrategy>) {
                t.s = ltm_id(x.engine().variant);
            } else if constexpr (std::is_same_v<S, UtmStrategy>) {
                t.s = TG_UTM;
                t.o.engine = static_cast<int32_t>(x.engine().variant);
            } else if constexpr (std::is_same_v<S, RbStrategy>) {
                t.s = TG_RB;
            } else {
                t.s = TG_REC;
                t.o.rec_m = x.schedule().m;
                t.o.rec_k = x.schedule().k;
            }
        },
        st);
    return t;
}
inline DispatchStats to_stats(const tg_dispatch_stats& s) {
    return {s.blocks_launched, s.blocks_discarded, s.threads_discarded, s.wall_time_ns};
}
// per-pass buffer wiring (LaunchOptions::per_pass)
struct PerPass {
    std::vector<tg_dispatch_stats> buf;
    void attach(Target& t, const AnyStrategy& st, const LaunchOptions& opt) {
        if (!opt.per_pass) return;
        buf.resize(grid_of(st).passes.size());
        t.o.per_pass = buf.data();
        t.o.per_pass_cap = static_cast<std::uint32_t>(buf.size());
    }
    void publish(const LaunchOptions& opt) const {
        if (!opt.per_pass) return;
        opt.per_pass->clear();
        for (const auto& s : buf) opt.per_pass->push_back(to_stats(s));
    }
};
}  // namespace detail

inline DispatchStats launch_dummy(const AnyStrategy& strategy, DummySink& sink, const LaunchOptions& opt = {}) {
    detail::Target t = detail::target(strategy, opt);
    detail::PerPass pp;
    pp.attach(t, strategy, opt);
    tg_dispatch_stats st;
    std::uint64_t v = 0;
    detail::check(tg_dummy_host(t.s, t.n, t.rho, &t.o, &st, &v));
    (void)sink;  // the device sink's anti-DCE store never fires (runtime-false predicate)
    pp.publish(opt);
    return detail::to_stats(st);
}

inline DispatchStats launch_edm(const AnyStrategy& strategy, const PointSet& points, PackedEdm& out,
                                const LaunchOptions& opt = {}) {
    detail::Target t = detail::target(strategy, opt);
    if (points.count != t.n) throw std::invalid_argument("launch_edm: point count does not match the strategy's N");
    if (points.features < 1 || points.features > 4) throw std::invalid_argument("launch_edm: features must be in [1, 4]");
    if (points.data.size() != points.count * points.features)
        throw std::invalid_argument("launch_edm: point data size mismatch");
    if (out.count != t.n || out.values.size() != tri_count(t.n, true))
        throw std::invalid_argument("launch_edm: output buffer is not N(N+1)/2 packed cells");
    detail::PerPass pp;
    pp.attach(t, strategy, opt);
    std::vector<int32_t> devs(opt.devices.begin(), opt.devices.end());
    if (devs.size() > 1) {
        t.o.devices = devs.data();
        t.o.n_devices = static_cast<std::uint32_t>(devs.size());
    }
    tg_dispatch_stats st;
    detail::check(tg_edm_strategy_host(t.s, points.data.data(), t.n, points.features, t.rho, out.values.data(), &t.o,
                                       &st));
    pp.publish(opt);
    return detail::to_stats(st);
}

inline DispatchStats launch_count(const AnyStrategy& strategy, std::vector<std::uint32_t>& counts,
                                  const LaunchOptions& opt = {}) {
    detail::Target t = detail::target(strategy, opt);
    if (counts.size() != tri_count(t.n, true))
        throw std::invalid_argument("launch_count: counter buffer is not N(N+1)/2 cells");
    detail::PerPass pp;
    pp.attach(t, strategy, opt);
    tg_dispatch_stats st;
    detail::check(tg_count_host(t.s, t.n, t.rho, counts.data(), &t.o, &st));
    pp.publish(opt);
    return detail::to_stats(st);
}

inline DispatchStats launch(const AnyStrategy& strategy, const KernelSpec& kernel, DummySink* sink,
                            const PointSet* points, PackedEdm* out, const LaunchOptions& opt = {}) {
    switch (kernel.kind) {
        case KernelSpec::Kind::Dummy:
            if (!sink) throw std::invalid_argument("launch: dummy kernel needs a sink");
            return launch_dummy(strategy, *sink, opt);
        case KernelSpec::Kind::Edm:
            if (!points || !out) throw std::invalid_argument("launch: EDM kernel needs points and an output buffer");
            return launch_edm(strategy, *points, *out, opt);
    }
    throw std::invalid_argument("launch: unknown kernel kind");
}

inline std::uint64_t count_wasted(StrategyKind strategy, std::uint64_t n) {
    std::uint64_t v;
    const tg_strategy s = strategy == StrategyKind::BoundingBox ? TG_BB
                          : strategy == StrategyKind::LowerTri  ? TG_LTM_R
                                                                : TG_UTM;  // no closed form: EINVAL
    detail::check(tg_count_wasted(s, n, &v));
    return v;
}

inline double ltm_diag_waste_blocks(std::uint64_t n) noexcept { return static_cast<double>(n) / 2.0; }

// ------------------------------------------------------------ extensions

// check_cell_coverage's verdict (checks.cpp:16-38), counted on device.
inline bool coverage_ok(const AnyStrategy& strategy, const LaunchOptions& opt = {}) {
    detail::Target t = detail::target(strategy, opt);
    int ok = 0;
    detail::check(tg_coverage_ok_opts(t.s, t.n, t.rho, &t.o, &ok, nullptr, nullptr));
    return ok != 0;
}

}  // namespace TRIGRID_B200_NS
