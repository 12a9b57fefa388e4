// trigrid_b200.cu -- host side of the C-ABI (include/trigrid_b200.h):
// validation with the reference's error classes, closed-form DispatchStats,
// lambda-range sharding, launch planning for the GRID and SPAN kernels, and
// the pipelined host-buffer drop-ins.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <numeric>

#include "../../include/trigrid_b200.h"
#include "tg_gram.cuh"
#include "tg_kernels.cuh"

using namespace tg;

namespace {

constexpr uint64_t kMaxElems = uint64_t{1} << 20;  // tri.hpp:11

thread_local std::string g_err;
thread_local uint64_t g_launches = 0;

tg_status fail(tg_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

#define TG_CUDA(expr)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            (void)cudaGetLastError();                                                   \
            return fail(e_ == cudaErrorMemoryAllocation ? TG_ENOMEM : TG_ECUDA,         \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));            \
        }                                                                               \
    } while (0)

#define TG_TRY(expr)                   \
    do {                               \
        tg_status s_ = (expr);         \
        if (s_ != TG_OK) return s_;    \
    } while (0)

uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

bool is_ltm(tg_strategy s) { return s >= TG_LTM_X && s <= TG_LTM_EXACT; }
int ltm_engine(tg_strategy s) {
    switch (s) {
        case TG_LTM_X: return kNative;
        case TG_LTM_N: return kNewton;
        case TG_LTM_R: return kReciprocal;
        default: return kExact;
    }
}

// A strategy instance: make_strategy(StrategyId, ProblemSize) (strategies.cpp:
// 192-208) plus the RecStrategy schedule (m, k) a caller may pick
// (rec_schedule, strategies.cpp:116-140) and the UTM engine.
struct Problem {
    tg_strategy s;
    uint64_t n;
    uint32_t rho;
    uint64_t m = 0;  // REC
    uint32_t k = 0;
    int engine = kNewton;  // UTM (parse_strategy("utm"), strategies.cpp:24)
};

// ProblemSize (tri.cpp:9-15) plus the per-strategy constructors' checks.
tg_status make_problem(tg_strategy s, uint64_t n, uint32_t rho, const tg_launch_opts* o, Problem* P) {
    if (n == 0) return fail(TG_EINVAL, "ProblemSize: N must be >= 1");
    if (n > kMaxElems) return fail(TG_EINVAL, "ProblemSize: N exceeds the 2^20 cap");
    if (rho == 0) return fail(TG_EINVAL, "ProblemSize: rho must be >= 1");
    if ((int)s < 0 || (int)s > (int)TG_REC) return fail(TG_EINVAL, "make_strategy: unknown strategy kind");
    if (s == TG_RB && n < 2) return fail(TG_EINVAL, "rb_rect: N must be >= 2");
    *P = Problem{s, n, rho};
    if (s == TG_UTM && o && o->engine >= 0) {
        if (o->engine > 3) return fail(TG_EINVAL, "make_strategy: unknown sqrt engine");
        P->engine = o->engine;
    }
    if (s == TG_REC) {
        if (o && (o->rec_m || o->rec_k)) {  // rec_schedule's own checks (strategies.cpp:118-124)
            if (o->rec_k < 1 || o->rec_k > 40) return fail(TG_EINVAL, "rec_schedule: k must be in [1, 40]");
            if (o->rec_m == 0 || o->rec_m % rho != 0)
                return fail(TG_EINVAL, "rec_schedule: m must be a positive multiple of rho");
            if (o->rec_m > (kMaxElems >> 1) || n != (o->rec_m << o->rec_k))
                return fail(TG_EINVAL, "rec_schedule: N must equal m*2^k");
            P->m = o->rec_m;
            P->k = o->rec_k;
        } else if (!rec_decompose(n, rho, &P->m, &P->k)) {
            return fail(TG_EINVAL, "rec: N is not m*2^k with m a multiple of rho");
        }
    }
    return TG_OK;
}

tg_status validate_problem(tg_strategy s, uint64_t n, uint32_t rho) {
    Problem P;
    return make_problem(s, n, rho, nullptr, &P);
}

// ------------------------------------------------------------ sharding

// Block-row bounds of G lambda-range shards: rows[g] is the block row whose
// start T(r) is nearest to g*T(nb)/G.
std::vector<uint64_t> shard_rows(uint64_t nb, uint32_t G) {
    std::vector<uint64_t> rows(G + 1, 0);
    const uint64_t total = tri(nb);
    rows[G] = nb;
    for (uint32_t g = 1; g < G; ++g) {
        const uint64_t target = (uint64_t)((unsigned __int128)total * g / G);
        const uint64_t r = fix_row(ltm_row_guess(target, kExact, true), target, true);
        const uint64_t lo = tri(r), hi = tri(r + 1);
        uint64_t b = (target - lo <= hi - target) ? r : r + 1;
        b = std::min(std::max(b, rows[g - 1]), nb);
        rows[g] = b;
    }
    return rows;
}

// --------------------------------------------------- closed-form stats

// threads filtered inside the surviving tiles of block rows [b0, b1)
// (process_block FullTile/DiagTile, engine.cpp:26-55).
uint64_t tile_threads_discarded(uint64_t n, uint64_t rho, uint64_t b0, uint64_t b1) {
    const uint64_t nb = ceil_div(n, rho);
    uint64_t t = 0;
    const uint64_t full_rows_end = std::min(b1, nb - 1);
    if (full_rows_end > b0) t += (full_rows_end - b0) * (rho * (rho - 1) / 2);
    if (b1 == nb && nb - 1 >= b0) {  // last block row, r valid cell rows
        const uint64_t b = nb - 1, r = n - rho * b;
        uint64_t diag = 0;
        for (uint64_t dy = 0; dy < r; ++dy) diag += rho - dy - 1;
        if (r < rho) diag += rho * (rho - r);
        const uint64_t full = (r < rho) ? b * rho * (rho - r) : 0;
        t += diag + full;
    }
    return t;
}

// Block-row window of shard `shard` of G: block rows [b0, b1), cell rows [r_lo, r_hi).
struct Window {
    uint64_t b0, b1, r_lo, r_hi;
};
Window window_of(const Problem& P, uint32_t shard, uint32_t G) {
    const auto rows = shard_rows(ceil_div(P.n, P.rho), G);
    Window w{rows[shard], rows[shard + 1], 0, 0};
    w.r_lo = std::min<uint64_t>(P.n, w.b0 * P.rho);
    w.r_hi = std::min<uint64_t>(P.n, w.b1 * P.rho);
    return w;
}

// REC grid passes in the reference's order (rec_schedule, strategies.cpp:
// 116-140): levels 1..k (square side m 2^(l-1), 2^(k-l) squares), then the
// diagonal pass (level 0: 2^k triangles of side m).
struct RecPassInfo {
    uint32_t level;
    uint64_t side, sb, count;  // count = squares or triangles
};
std::vector<RecPassInfo> rec_passes(const Problem& P) {
    std::vector<RecPassInfo> v;
    for (uint32_t level = 1; level <= P.k; ++level) {
        const uint64_t side = P.m << (level - 1);
        v.push_back({level, side, side / P.rho, 1ull << (P.k - level)});
    }
    v.push_back({0, P.m, P.m / P.rho, 1ull << P.k});
    return v;
}

// Global block row of pass-local block row `by` (strictly increasing in by).
uint64_t rec_row_of(const RecPassInfo& q, uint64_t by) {
    if (q.level == 0) return by;  // triangle t at block row t sb
    const uint64_t sq = by / q.sb, ly = by % q.sb;
    return (2 * sq + 1) * q.sb + ly;  // rec_block_map (strategies.hpp:214-220)
}
// First pass-local block row whose global row is >= X.
uint64_t rec_row_lower_bound(const RecPassInfo& q, uint64_t X) {
    uint64_t lo = 0, hi = q.sb * q.count;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (rec_row_of(q, mid) >= X) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// RB rect block rows whose direct (level 0) / folded (level 1) part meets cell rows [r_lo, r_hi).
void rb_row_ranges(const Problem& P, const Window& w, uint64_t* y) {
    const uint64_t n = P.n, rho = P.rho, even = (n % 2 == 0);
    const uint64_t h = even ? n + 1 : n, hb = ceil_div(h, rho);
    if (w.r_hi <= w.r_lo) {
        y[0] = y[1] = y[2] = y[3] = 0;
        return;
    }
    // direct part: row i = ty - even
    y[0] = std::min(hb, (w.r_lo + even) / rho);
    y[1] = std::min(hb, ceil_div(w.r_hi + even, rho));
    // folded part: row i = n - 1 - ty, ty in [n - r_hi, n - r_lo)
    y[2] = std::min(hb, (n - w.r_hi) / rho);
    y[3] = std::min(hb, ceil_div(n - w.r_lo, rho));
}

// What run_strategy tallies (engine.cpp:70-136), closed form, for the whole
// domain or one shard; per_pass (optional) gets one entry per grid pass.
tg_status stats_for(const Problem& P, uint32_t shard, uint32_t shards, tg_dispatch_stats* st,
                    std::vector<tg_dispatch_stats>* per_pass = nullptr) {
    const uint64_t n = P.n, rho = P.rho;
    *st = tg_dispatch_stats{0, 0, 0, 0};
    if (per_pass) per_pass->clear();
    const uint64_t nb = ceil_div(n, rho);
    const uint32_t G = shards == 0 ? 1 : shards;
    if (shard >= G) return fail(TG_EINVAL, "shard_index must be < shard_count");
    const Window w = window_of(P, shard, G);
    const tg_strategy s = P.s;
    if (s == TG_BB || is_ltm(s)) {
        const uint64_t b0 = w.b0, b1 = w.b1;
        if (s == TG_BB) {
            const uint64_t W = b1, H = b1 - b0;
            st->blocks_launched = W * H;
            // sum over grid rows y in [b0, b1) of the W - 1 - y blocks with x > y
            st->blocks_discarded = H * (H - (H > 0 ? 1 : 0)) / 2;
        } else {
            const uint64_t L = tri(b1) - tri(b0);
            const uint64_t side = L ? ceil_sqrt(L) : 0;
            st->blocks_launched = side * side;
            st->blocks_discarded = side * side - L;
        }
        st->threads_discarded = (b1 > b0) ? tile_threads_discarded(n, rho, b0, b1) : 0;
    } else if (s == TG_UTM) {
        if (G == 1) {
            const uint64_t pairs = tri_nd(n), tpb = rho * rho;
            const uint64_t blocks = pairs == 0 ? 1 : ceil_div(pairs, tpb);
            st->blocks_launched = blocks;
            st->threads_discarded = blocks * tpb - pairs;
        } else {  // shard: the rho x rho tiles of its rows the span walk visits (no reference counterpart)
            const uint64_t H = w.b1 - w.b0;
            st->blocks_launched = w.b0 * H + tri(H);
        }
    } else if (s == TG_RB) {
        const uint64_t wd = (n % 2 == 0) ? n / 2 : (n + 1) / 2, h = (n % 2 == 0) ? n + 1 : n;
        const uint64_t gx = ceil_div(wd, rho), gy = ceil_div(h, rho);
        if (G == 1) {
            st->blocks_launched = gx * gy;
            st->threads_discarded = gx * gy * rho * rho - wd * h;
        } else {  // shard: rect blocks whose direct or folded part meets its rows
            uint64_t y[4];
            rb_row_ranges(P, w, y);
            const uint64_t lo = std::max(y[0], y[2]), hi = std::min(y[1], y[3]);
            st->blocks_launched = gx * ((y[1] - y[0]) + (y[3] - y[2]) - (hi > lo ? hi - lo : 0));
        }
    } else {  // REC: per pass, the pass-local block rows inside the window
        for (const RecPassInfo& q : rec_passes(P)) {
            const uint64_t y0 = rec_row_lower_bound(q, w.b0), y1 = rec_row_lower_bound(q, w.b1);
            tg_dispatch_stats ps{(y1 - y0) * q.sb, 0, 0, 0};
            if (q.level == 0) {  // diagonal pass: BB inside each m-triangle
                for (uint64_t by = y0; by < y1; ++by) ps.blocks_discarded += q.sb - 1 - by % q.sb;
                ps.threads_discarded = (y1 - y0) * (rho * (rho - 1) / 2);
            }
            st->blocks_launched += ps.blocks_launched;
            st->blocks_discarded += ps.blocks_discarded;
            st->threads_discarded += ps.threads_discarded;
            if (per_pass) per_pass->push_back(ps);
        }
        return TG_OK;
    }
    if (per_pass) per_pass->push_back(*st);
    (void)nb;
    return TG_OK;
}

tg_status stats_for(tg_strategy s, uint64_t n, uint32_t rho, uint32_t shard, uint32_t shards,
                    tg_dispatch_stats* st) {
    Problem P;
    TG_TRY(make_problem(s, n, rho, nullptr, &P));
    return stats_for(P, shard, shards, st);
}

// ------------------------------------------------------- device context

struct Buf {
    void* p = nullptr;
    size_t cap = 0;
};

struct DeviceCtx {
    std::mutex mu;       // guards the cached buffers / internal streams of the host drop-ins
    std::mutex init_mu;  // one-time initialisation (and the per-device kernel attributes below)
    std::atomic<bool> init{false};
    int dev = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;       // internal compute stream (host drop-ins)
    cudaStream_t copy_stream = nullptr;  // D2H pipeline
    cudaStream_t copy_stream2 = nullptr; // second D2H stream (alternating 256 MB sub-copies)
    unsigned long long* scratch = nullptr;  // [0] sink [1] bad [2] first [3] hits (host drop-ins, under mu)
    Buf bufs[4];  // [0] pts [1] out (host drop-ins) [2] counts [3] gen
    cudaEvent_t ev[34];
    // per-device kernel attributes / occupancies (function attributes are per device)
    std::atomic<bool> attr_wide2{false}, attr_gram{false}, attr_gram2{false};
    std::atomic<int> occ_wide2{-1}, occ_edm{-1}, occ_write{-1};
};

DeviceCtx g_ctx[64];

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per device and kernel.
template <class K>
tg_status ensure_smem_attr(DeviceCtx* c, std::atomic<bool>& done, K* kernel, size_t bytes) {
    if (done.load(std::memory_order_acquire)) return TG_OK;
    std::lock_guard<std::mutex> lk(c->init_mu);
    if (!done.load(std::memory_order_relaxed)) {
        TG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        done.store(true, std::memory_order_release);
    }
    return TG_OK;
}

template <class K>
int occupancy(std::atomic<int>& slot, K* kernel, int threads, size_t smem) {
    int v = slot.load(std::memory_order_relaxed);
    if (v < 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, threads, smem) != cudaSuccess) {
            (void)cudaGetLastError();
            v = 1;
        }
        slot.store(std::max(v, 1), std::memory_order_relaxed);
    }
    return std::max(v, 1);
}

tg_status ensure_buf(Buf& b, size_t bytes) {
    if (b.cap >= bytes) return TG_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    TG_CUDA(cudaMalloc(&b.p, std::max<size_t>(bytes, 256)));
    b.cap = std::max<size_t>(bytes, 256);
    return TG_OK;
}

// Stream-ordered scratch for one launch (cudaMallocAsync from the device's
// default pool, which keeps the memory between launches): the Gram operands,
// the feature-major points, the classify verdict and the persistent unit
// counter are private to the launch, so concurrent launches on other streams
// / host threads never share them.
struct Scratch {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    Scratch() = default;
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    ~Scratch() {
        if (p) cudaFreeAsync(p, st);
    }
};

tg_status scratch_alloc(Scratch& s, size_t bytes, cudaStream_t st) {
    s.st = st;
    TG_CUDA(cudaMallocAsync(&s.p, std::max<size_t>(bytes, 256), st));
    return TG_OK;
}

// Restores the caller's current device when an entry point returns (get_ctx
// switches to the launch's device).
struct DevGuard {
    int prev = -1;
    DevGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            (void)cudaGetLastError();
            prev = -1;
        }
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

tg_status get_ctx(int device, DeviceCtx** out) {
    int dev = device;
    if (dev < 0) TG_CUDA(cudaGetDevice(&dev));
    if (dev >= 64) return fail(TG_EINVAL, "device ordinal out of range");
    TG_CUDA(cudaSetDevice(dev));
    DeviceCtx& c = g_ctx[dev];
    if (c.init.load(std::memory_order_acquire)) {
        *out = &c;
        return TG_OK;
    }
    std::lock_guard<std::mutex> lk(c.init_mu);  // not c.mu: callers may hold c.mu
    if (!c.init.load(std::memory_order_relaxed)) {
        c.dev = dev;
        TG_CUDA(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev));
        TG_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        TG_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
        TG_CUDA(cudaStreamCreateWithFlags(&c.copy_stream2, cudaStreamNonBlocking));
        TG_CUDA(cudaMalloc(&c.scratch, 256));
        for (auto& e : c.ev) TG_CUDA(cudaEventCreate(&e));
        cudaMemPool_t pool;  // keep stream-ordered scratch cached between launches
        TG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t keep = ~0ull;
        TG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        c.init.store(true, std::memory_order_release);
    }
    *out = &c;
    return TG_OK;
}

// --------------------------------------------------------- span planning

// Chunk slots per lane of the d <= 4 EDM span kernel: 2 (1 KB contiguous per
// warp and row, C = 16 blocks per unit at rho = 16) measured 1.51 ms vs
// 1.55 ms for 1 slot at N=65536 in two same-session A/B runs.
int span_slots() {
    static int p = [] {
        const char* e = std::getenv("TG_SPAN_SLOTS");
        return (e && std::atoi(e) == 1) ? 1 : 2;
    }();
    return p;
}


// Strategies / rho with a span form (row tiles; utm: super-block slabs):
// every strategy with rho % 4 == 0.
bool span_eligible(tg_strategy s, uint32_t rho) {
    (void)s;
    return rho % 4 == 0 && rho <= 128;
}
// Bodies restricted to the square-tile strategies (16-row tiles at block-row
// multiples: the d > 4 kernels, the collision kernel).
bool square_tiles(tg_strategy s) { return s == TG_BB || is_ltm(s) || s == TG_REC; }

// UTM super-block side in run widths: about 4 super-block rows per launch,
// within [16, 64].  utm_pair orders the super-blocks column by column, so the
// 32-byte sectors split across a vertical super-block boundary are completed
// long after their first half was written: evicted half-written sectors cost
// a DRAM read-modify-write (ncu: the UTM write kernel reads 20.8 MB vs 2.4 MB
// for LTM).  Fewer, wider super-blocks at large N: A/B at N=65536 (runs 16 /
// 32 / 64 / 128): write 1.488 / 1.425 / 1.370 / 1.347 ms, EDM 1.607 / 1.59 /
// 1.578 / 1.621 ms.  A/B: TG_UTM_RUNS.
uint64_t utm_runs(uint64_t n, uint64_t run_cols) {
    static int env = [] {
        const char* e = std::getenv("TG_UTM_RUNS");
        return e ? std::max(1, std::atoi(e)) : 0;
    }();
    if (env) return (uint64_t)env;
    return std::min<uint64_t>(64, std::max<uint64_t>(16, ceil_div(n, 4 * run_cols)));
}

tg_status plan_span_c(const Problem& P, const Window& w, uint32_t C, SpanGeom* g, int only_pass);

// LTM span units: row-aligned lambda segments (default) or, A/B
// TG_LTM_ROWS=0, runs of C consecutive lambda that may cross row ends.
bool ltm_row_units() {
    static bool v = [] {
        const char* e = std::getenv("TG_LTM_ROWS");
        return !e || std::atoi(e) != 0;
    }();
    return v;
}

// Live units a launch should have at least: ~16 warps' worth per SM.  A small
// problem planned with the default C (16 blocks per warp) leaves most SMs idle
// and each warp on a long serial run walk (N=1024 LTM: 133 warps, 56 us vs
// 15 us for BB), so C shrinks until the launch has this many units that do
// work.  Counted on LIVE blocks (BB's discarded x > y blocks excluded): with
// the grid count BB kept twice LTM's run length at the same N and LTM's
// 16-column runs at N=2048 left 7/8 of the lanes idle (CUDA-graph replay:
// LTM write 18.5 us vs BB 12.7 us at N=2048, 20.5 vs 13.7 us at N=4096).
uint64_t min_span_units() {  // A/B: TG_SPAN_MIN_UNITS
    static uint64_t v = [] {
        const char* e = std::getenv("TG_SPAN_MIN_UNITS");
        return e ? (uint64_t)std::atoll(e) : (uint64_t)148 * 16;
    }();
    return v;
}

// Grid blocks of the launch that emit tiles (BB: the y >= x half; LTM: the
// lambda range without the balanced-grid padding; the pass-table and UTM
// plans have no discarded units).
uint64_t live_span_blocks(const SpanGeom& g) {
    if (g.strat == kSpanBB) return tri(g.W) - tri(g.b0);
    if (g.strat == kSpanLTM) return g.lam1 - g.lam0;
    return g.units * g.C;
}

// Geometry for the window's block rows; `adaptive` lets C shrink for small
// problems (the one-CTA-per-run d > 4 kernel needs the fixed C).  only_pass
// (REC, >= 0): plan that grid pass alone (LaunchOptions::per_pass timing).
// A/B: TG_SPAN_PERM=f (f in (0, 1), e.g. 0.618) runs the units in the order
// u -> (u * p) % units, p ~ f * units coprime to units; 0 / unset = identity.
double span_perm_frac() {
    static double v = [] {
        const char* e = std::getenv("TG_SPAN_PERM");
        return e ? std::atof(e) : 0.0;
    }();
    return v;
}

void set_span_perm(SpanGeom* g) {
    g->perm = 0;
    const double f = span_perm_frac();
    if (f <= 0.0 || f >= 1.0 || g->units < 3 || g->units > 0xffffffffull) return;
    uint64_t p = std::max<uint64_t>(1, (uint64_t)(f * (double)g->units));
    while (std::gcd(p, g->units) != 1) ++p;
    g->perm = p;
}

tg_status plan_span(const Problem& P, const Window& w, uint32_t C, SpanGeom* g, bool adaptive = true,
                    int only_pass = -1) {
    TG_TRY(plan_span_c(P, w, C, g, only_pass));
    const uint64_t min_units = min_span_units();
    const uint64_t live = live_span_blocks(*g);
    if (adaptive && C > 1 && ceil_div(live, C) < min_units) {
        const uint32_t c2 = (uint32_t)std::max<uint64_t>(1, live / min_units);
        if (c2 < C) TG_TRY(plan_span_c(P, w, c2, g, only_pass));
    }
    set_span_perm(g);
    return TG_OK;
}

void add_pass(SpanGeom* g, uint64_t& unit, uint64_t y0, uint64_t y1, uint64_t sb, uint64_t side, uint32_t level,
              uint32_t C) {
    SpanPass& q = g->pass[g->npass++];
    q.unit_begin = unit;
    q.y0 = y0;
    q.sb = sb;
    q.side = side;
    q.level = level;
    q.cu = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(C, sb));
    q.upr = (uint32_t)ceil_div(sb, q.cu);
    unit += (y1 > y0 ? y1 - y0 : 0) * q.upr;
}

tg_status plan_span_c(const Problem& P, const Window& w, uint32_t C, SpanGeom* g, int only_pass) {
    std::memset(g, 0, sizeof(*g));
    const uint64_t n = P.n, rho = P.rho, b0 = w.b0, b1 = w.b1;
    g->one = 1.0f;
    g->rho = P.rho;
    g->C = C;
    g->n = n;
    g->b0 = b0;
    g->r_lo = w.r_lo;
    g->r_hi = w.r_hi;
    const tg_strategy s = P.s;
    if (s == TG_BB) {
        g->strat = kSpanBB;
        g->W = b1;
        g->vb_count = b1 * (b1 - b0);
        g->units = ceil_div(g->vb_count, C);
    } else if (is_ltm(s)) {
        g->strat = kSpanLTM;
        g->engine = ltm_engine(s);
        g->lam0 = tri(b0);
        g->lam1 = tri(b1);
        const uint64_t L = g->lam1 - g->lam0;
        const uint64_t side = L ? ceil_sqrt(L) : 0;
        g->vb_count = side * side;  // balanced grid (tri.cpp:23-26) incl. padding
        g->units = ceil_div(g->vb_count, C);
        g->b1 = b1;
        if (ltm_row_units()) {  // row-aligned lambda segments: U(r) units before block row r
            auto U = [C](uint64_t r) {
                const uint64_t q = r / C, t = r % C;
                return C * (q * (q + 1) / 2) + t * (q + 1);
            };
            g->ltm_rows = 1;
            g->ubase = U(b0);
            g->units = U(b1) - U(b0);
        }
    } else if (s == TG_REC) {
        g->strat = kSpanREC;
        g->m = P.m;
        // unit order: the diagonal pass and the small low levels first (many
        // short runs, slow warps) so they do not form the launch's tail; the big
        // square passes, whose units are uniform full runs, come last (the
        // passes are independent).  A pass narrower than C blocks gets units of
        // one block row (cu = sb).
        const auto qs = rec_passes(P);
        uint64_t unit = 0;
        for (size_t t = 0; t < qs.size(); ++t) {
            const size_t pi = (t == 0) ? qs.size() - 1 : t - 1;  // diag, level 1, ..., level k
            if (only_pass >= 0 && (size_t)only_pass != pi) continue;
            const RecPassInfo& q = qs[pi];
            const uint64_t y0 = rec_row_lower_bound(q, b0), y1 = rec_row_lower_bound(q, b1);
            add_pass(g, unit, y0, y1, q.sb, q.side, q.level, C);
        }
        g->units = unit;
    } else if (s == TG_RB) {
        g->strat = kSpanRB;
        const uint64_t wd = (n % 2 == 0) ? n / 2 : (n + 1) / 2;
        uint64_t y[4];
        rb_row_ranges(P, w, y);
        uint64_t unit = 0;
        if (y[0] < y[3] && y[2] < y[1]) {
            // the direct and folded rect-row ranges overlap (always for the whole
            // domain): one pass over their union, each unit emitting both of its
            // complementary parts (clipped to the window), so no unit is empty
            add_pass(g, unit, std::min(y[0], y[2]), std::max(y[1], y[3]), ceil_div(wd, rho), 0, 2, C);
        } else {
            add_pass(g, unit, y[0], y[1], ceil_div(wd, rho), 0, 0, C);  // direct part
            add_pass(g, unit, y[2], y[3], ceil_div(wd, rho), 0, 1, C);  // folded part
        }
        g->units = unit;
    } else if (s == TG_UTM) {
        g->strat = kSpanUTM;
        g->engine = P.engine;
        // super-blocks of W = utm_runs() run widths (C rho columns each); one
        // unit per 16-row x run tile
        const uint64_t runs = utm_runs(n, (uint64_t)C * rho), S = (uint64_t)C * rho * runs, R0 = std::min(n, b0 * rho);
        const uint64_t He = w.r_hi - R0;
        g->W = S;
        g->ur = runs;
        g->H = ceil_div(He, S);
        g->rect_blocks = ceil_div(He, 16) * runs;  // units per rectangle strip
        g->u_rect = ceil_div(R0, S) * g->rect_blocks;
        g->upb = ceil_div(S, 16) * runs;
        g->tri_blocks = tri(g->H);  // = T_nodiag(H + 1) pairs of the super-block-level UTM
        g->disc = (2 * g->H + 1) * (2 * g->H + 1);
        g->units = g->u_rect + g->tri_blocks * g->upb;
    } else {
        return fail(TG_EINVAL, "span mode: unknown strategy");
    }
    return TG_OK;
}

uint64_t span_grid(const SpanGeom& g, bool persistent, int sms, int occ, int warps_per_cta = kWarpsPerCta) {
    const uint64_t need = ceil_div(g.units, (uint64_t)warps_per_cta);
    if (need == 0) return 0;
    uint64_t grid = need;
    if (persistent) grid = std::min<uint64_t>(need, (uint64_t)sms * std::max(occ, 1));
    return std::min<uint64_t>(grid, 0x7fffffffull);
}

int span_packed() {
    static int v = [] {
        const char* e = std::getenv("TG_SPAN_PACKED");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

template <int D, int P, bool PK>
tg_status launch_span_edm_t(const SpanGeom& g, OutWin ow, const float* pts, float* out,
                            const unsigned int* flag, cudaStream_t st, bool persistent, int sms) {
    int occ = 1;
    Scratch qs;  // persistent launches: a per-launch zeroed unit counter (stream-ordered, private)
    unsigned long long* queue = nullptr;
    if (persistent) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, span_edm_kernel<D, P, PK>, kEdmWarps * 32, 0) !=
            cudaSuccess)
            occ = 1;
        TG_TRY(scratch_alloc(qs, sizeof(unsigned long long), st));
        queue = static_cast<unsigned long long*>(qs.p);
        TG_CUDA(cudaMemsetAsync(queue, 0, sizeof(unsigned long long), st));
    }
    const uint64_t grid = span_grid(g, persistent, sms, occ, kEdmWarps);
    if (!grid) return TG_OK;
    span_edm_kernel<D, P, PK><<<(unsigned)grid, kEdmWarps * 32, 0, st>>>(g, ow, pts, out, flag, queue);
    ++g_launches;
    TG_CUDA(cudaGetLastError());
    return TG_OK;
}

// The A/B variants (1 chunk slot per lane, scalar instead of f32x2 row pairs)
// are compiled only into -DTG_AB_VARIANTS=1 builds (build.py --variant): they
// triple the compile time of the default library for switches that lost.
#ifndef TG_AB_VARIANTS
#define TG_AB_VARIANTS 0
#endif

template <int P, bool PK>
tg_status launch_span_edm_pk(uint32_t d, const SpanGeom& g, OutWin ow, const float* pts, float* out,
                             const unsigned int* flag, cudaStream_t st, bool persistent, int sms) {
    switch (d) {
        case 1: return launch_span_edm_t<1, P, PK>(g, ow, pts, out, flag, st, persistent, sms);
        case 2: return launch_span_edm_t<2, P, PK>(g, ow, pts, out, flag, st, persistent, sms);
        case 3: return launch_span_edm_t<3, P, PK>(g, ow, pts, out, flag, st, persistent, sms);
        case 4: return launch_span_edm_t<4, P, PK>(g, ow, pts, out, flag, st, persistent, sms);
    }
    return fail(TG_EINVAL, "span EDM supports d in [1, 4]");
}

tg_status launch_span_edm(uint32_t d, const SpanGeom& g, OutWin ow, const float* pts, float* out,
                          const unsigned int* flag, cudaStream_t st, bool persistent, int sms) {
    const bool pk = span_packed() != 0, two = span_slots() == 2;
#if TG_AB_VARIANTS
    if (!pk) return two ? launch_span_edm_pk<2, false>(d, g, ow, pts, out, flag, st, persistent, sms)
                        : launch_span_edm_pk<1, false>(d, g, ow, pts, out, flag, st, persistent, sms);
    if (!two) return launch_span_edm_pk<1, true>(d, g, ow, pts, out, flag, st, persistent, sms);
#else
    if (!pk || !two) return fail(TG_EINVAL, "TG_SPAN_PACKED=0 / TG_SPAN_SLOTS=1 need a -DTG_AB_VARIANTS=1 build");
#endif
    return launch_span_edm_pk<2, true>(d, g, ow, pts, out, flag, st, persistent, sms);
}

// A/B switch: TG_WIDE_V1=1 keeps the first d > 4 kernel (per-run transposed staging).
bool wide_v1() {
    static bool v = [] {
        const char* e = std::getenv("TG_WIDE_V1");
        return e && std::atoi(e) != 0;
    }();
    return v;
}

// d > 4, version 2: feature-major copy of the points + pipelined two-runs-per-CTA kernel.
tg_status launch_wide2_edm(uint32_t d, const SpanGeom& g, OutWin ow, const float* pts, float* out,
                           const unsigned int* flag, cudaStream_t st, bool persistent, int sms, DeviceCtx* c) {
    const uint64_t n = g.n;
    const uint64_t n_pad = ceil_div(n + kW2Cols, kW2Cols) * kW2Cols;  // a run's 128 columns / 16 rows stay in range
    const uint32_t d_pad = (uint32_t)ceil_div(d, kW2K) * kW2K;
    Scratch sp;
    TG_TRY(scratch_alloc(sp, (size_t)n_pad * d_pad * sizeof(float), st));
    float* ptsT = static_cast<float*>(sp.p);
    transpose_points_kernel<<<dim3((unsigned)(n_pad / 32), (unsigned)ceil_div(d_pad, 32)), dim3(32, 8), 0, st>>>(
        pts, n, d, n_pad, d_pad, ptsT);
    const size_t smem = kW2Groups * kW2GroupFloats * sizeof(float);
    TG_TRY(ensure_smem_attr(c, c->attr_wide2, wide2_edm_kernel, smem));
    const int occ = occupancy(c->occ_wide2, wide2_edm_kernel, kW2Threads, smem);
    const uint64_t grid =
        std::min<uint64_t>(ceil_div(g.units, kW2Groups), (uint64_t)sms * std::max(occ, 1) * (persistent ? 1 : 64));
    if (!grid) return TG_OK;
    wide2_edm_kernel<<<(unsigned)grid, kW2Threads, smem, st>>>(g, ow, ptsT, n_pad, d_pad / kW2K, out, flag);
    g_launches += 2;
    TG_CUDA(cudaGetLastError());
    return TG_OK;
}

// d > 4: CTA-per-run tiled kernel (rho == 16, runs of <= 128 columns).
tg_status launch_wide_edm(uint32_t d, const SpanGeom& g, OutWin ow, const float* pts, float* out,
                          const unsigned int* flag, cudaStream_t st, bool persistent, int sms, DeviceCtx* c) {
    if (g.rho != 16 || g.C != (wide_v1() ? 8u : 8u * kW2CH)) return fail(TG_EINVAL, "wide EDM span kernel needs rho == 16");
    if (!wide_v1()) return launch_wide2_edm(d, g, ow, pts, out, flag, st, persistent, sms, c);
    uint64_t grid = std::min<uint64_t>(g.units, 0x7fffffffull);
    if (persistent) {
        int occ = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wide_edm_kernel, 256, 0) != cudaSuccess) occ = 1;
        grid = std::min<uint64_t>(grid, (uint64_t)sms * std::max(occ, 1));
    }
    if (!grid) return TG_OK;
    wide_edm_kernel<<<(unsigned)grid, 256, 0, st>>>(g, ow, pts, d, out, flag);
    ++g_launches;
    TG_CUDA(cudaGetLastError());
    return TG_OK;
}

// Gram-trick EDM on tcgen05 (tg_gram.cuh) over the block rows [b0, b1) of
// the rho-block triangle: 128-row tiles covering those rows, tile lambda
// range [T(ty0), T(ty1)), rows and elements clipped to the window.
tg_status launch_gram_edm(uint64_t n, uint32_t d, uint32_t rho, uint64_t b0, uint64_t b1, OutWin ow,
                          const float* pts, float* out, float* norms, cudaStream_t st, DeviceCtx* c) {
    const int sms = c->sms;
    TG_TRY(ensure_smem_attr(c, c->attr_gram, gram_edm_kernel, kGSmemBytes));
    const uint64_t r0 = std::min<uint64_t>(n, b0 * rho), r1 = std::min<uint64_t>(n, b1 * rho);
    if (r1 <= r0) return TG_OK;
    GramGeom g{};
    g.n = n;
    g.d = d;
    g.nt = (uint32_t)ceil_div(n, kGT);
    const uint64_t ty0 = r0 / kGT, ty1 = ceil_div(r1, kGT);
    g.t0 = tri(ty0);
    g.t1 = tri(ty1);
    g.r0 = r0;
    g.r1 = r1;
    g.e_base = ow.e_base;
    g.e_end = ow.e_end;
    const uint64_t tiles = g.t1 - g.t0;
    const uint64_t grid = std::min<uint64_t>(tiles, (uint64_t)sms);
    g.per_cta = ceil_div(tiles, grid);
    const uint64_t nb = std::min<uint64_t>(ceil_div(n, 256), (uint64_t)sms * 8);
    gram_norms_kernel<<<(unsigned)nb, 256, 0, st>>>(pts, n, d, norms);
    ++g_launches;
    gram_edm_kernel<<<(unsigned)ceil_div(tiles, g.per_cta), kGThreads, kGSmemBytes, st>>>(g, pts, norms, out);
    ++g_launches;
    TG_CUDA(cudaGetLastError());
    return TG_OK;
}

// A/B switch: TG_GRAM_V1=1 forces the first (unpipelined 3xTF32) Gram kernel.
bool gram_v1() {
    static bool v = [] {
        const char* e = std::getenv("TG_GRAM_V1");
        return e && std::atoi(e) != 0;
    }();
    return v;
}

// Pipelined fp16-split Gram EDM (tg_gram.cuh v2), any d (row tile resident for d <= 128, streamed above): prep (norms,
// max |x|) -> split (hi/lo operands in UMMA layout) -> warp-specialised kernel.
tg_status launch_gram2_edm(uint64_t n, uint32_t d, uint32_t rho, uint64_t b0, uint64_t b1, OutWin ow,
                           const float* pts, float* out, DeviceCtx* c, cudaStream_t st) {
    TG_TRY(ensure_smem_attr(c, c->attr_gram2, gram2_edm_kernel, kG2SmemMax));
    const uint64_t r0 = std::min<uint64_t>(n, b0 * rho), r1 = std::min<uint64_t>(n, b1 * rho);
    if (r1 <= r0) return TG_OK;
    const uint32_t nk = (uint32_t)ceil_div(d, 64);
    const uint64_t nt = ceil_div(n, kGT), n_pad = nt * kGT;
    const uint64_t a_bytes = nt * nk * (uint64_t)kG2Slice;
    const uint64_t bslice = (nt * 16 + 1) * (uint64_t)kG2Group;
    const uint64_t b_bytes = nk * 2 * bslice;
    Scratch sn, so;
    // norms | per-point scale factors | per-point max |x| bits, (n_pad + 8) each
    TG_TRY(scratch_alloc(sn, 3 * (n_pad + 8) * sizeof(float), st));
    TG_TRY(scratch_alloc(so, a_bytes + b_bytes + 256, st));
    float* norms = static_cast<float*>(sn.p);
    float* facs = norms + (n_pad + 8);
    unsigned int* pmax = reinterpret_cast<unsigned int*>(facs + (n_pad + 8));
    uint8_t* opA = static_cast<uint8_t*>(so.p);
    uint8_t* opB = opA + a_bytes;
    unsigned int* bits = reinterpret_cast<unsigned int*>(opB + b_bytes);  // max |x|, ~min nonzero point max
    TG_CUDA(cudaMemsetAsync(bits, 0, 2 * sizeof(unsigned int), st));
    const unsigned pb = (unsigned)std::min<uint64_t>(ceil_div(n_pad + 8, 256), (uint64_t)c->sms * 8);
    gram_prep_kernel<<<pb, 256, 0, st>>>(pts, n, n_pad + 8, d, norms, pmax, bits);
    const unsigned sb = (unsigned)std::min<uint64_t>(ceil_div((n_pad + 8) * nk * 8, 256), (uint64_t)c->sms * 16);
    gram_split_kernel<<<sb, 256, 0, st>>>(pts, n, n_pad, d, nk, bits, pmax, facs, opA, opB, bslice);
    Gram2Geom g{};
    g.n = n;
    g.nk = nk;
    g.bslice = bslice;
    g.a_stream = nk > (uint32_t)kG2MaxNk ? 1u : 0u;
    g.stage = g2_stage_bytes(g.a_stream != 0);
    g.ring = 2;
    while (g.ring < 8 && g2_smem_bytes(nk, g.ring + 1, g.a_stream != 0) <= kG2SmemMax) ++g.ring;
    if (g2_smem_bytes(nk, g.ring, g.a_stream != 0) > kG2SmemMax) return fail(TG_EINVAL, "gram: shared memory plan");
    const uint64_t ty0 = r0 / kGT, ty1 = ceil_div(r1, kGT);
    g.t0 = tri(ty0);
    g.t1 = tri(ty1);
    g.r0 = r0;
    g.r1 = r1;
    g.e_base = ow.e_base;
    g.e_end = ow.e_end;
    const uint64_t tiles = g.t1 - g.t0;
    const uint64_t grid = std::min<uint64_t>(tiles, (uint64_t)c->sms);
    g.per_cta = ceil_div(tiles, grid);
    gram2_edm_kernel<<<(unsigned)ceil_div(tiles, g.per_cta), kG2Threads, g2_smem_bytes(nk, g.ring, g.a_stream != 0), st>>>(
        g, opA, opB, norms, facs, bits, out);
    g_launches += 3;
    TG_CUDA(cudaGetLastError());
    return TG_OK;
}

tg_status launch_classify(const float* pts, uint64_t count, unsigned int* flag, cudaStream_t st, int sms) {
    TG_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned int), st));
    const uint64_t blocks = std::min<uint64_t>(ceil_div(count, 256), (uint64_t)sms * 4);
    classify_points_kernel<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, 0, st>>>(pts, count, flag);
    ++g_launches;
    TG_CUDA(cudaGetLastError());
    return TG_OK;
}

template <int P, int OP>
tg_status launch_span_write_p(const SpanGeom& g, OutWin ow, uint32_t* out, cudaStream_t st,
                              bool persistent, int sms) {
    int occ = 1;
    if (persistent &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, span_write_kernel<P, OP>, kWarpsPerCta * 32, 0) !=
            cudaSuccess)
        occ = 1;
    const uint64_t grid = span_grid(g, persistent, sms, occ);
    if (!grid) return TG_OK;
    span_write_kernel<P, OP><<<(unsigned)grid, kWarpsPerCta * 32, 0, st>>>(g, ow, out);
    ++g_launches;
    TG_CUDA(cudaGetLastError());
    return TG_OK;
}

// Chunk slots per lane of the write kernel: 2 (1 KB contiguous per warp and
// row) measured 1.27 ms vs 1.50 ms for 1 slot at N=65536 (profiles/r1d_*).
int write_slots() {
    static int v = [] {
        const char* e = std::getenv("TG_WRITE_SLOTS");
        return (e && std::atoi(e) == 1) ? 1 : 2;
    }();
    return v;
}

tg_status launch_span_write(const SpanGeom& g, OutWin ow, uint32_t* out, cudaStream_t st,
                            bool persistent, int sms) {
#if TG_AB_VARIANTS
    if (write_slots() == 1) return launch_span_write_p<1, kOpWrite>(g, ow, out, st, persistent, sms);
#else
    if (write_slots() == 1) return fail(TG_EINVAL, "TG_WRITE_SLOTS=1 needs a -DTG_AB_VARIANTS=1 build");
#endif
    return launch_span_write_p<2, kOpWrite>(g, ow, out, st, persistent, sms);
}

// Span COUNT: +1 per cell of every owned chunk (same walk as the write kernel).
tg_status launch_span_count(const SpanGeom& g, OutWin ow, uint32_t* out, cudaStream_t st, bool persistent,
                            int sms) {
    return launch_span_write_p<2, kOpCount>(g, ow, out, st, persistent, sms);
}

// --------------------------------------------------------- grid planning

std::vector<GridGeom> plan_grid(const Problem& P) {
    const tg_strategy s = P.s;
    const uint64_t n = P.n;
    const uint32_t rho = P.rho;
    std::vector<GridGeom> passes;
    GridGeom g{};
    g.rho = rho;
    g.n = n;
    const uint64_t nb = ceil_div(n, rho);
    if (s == TG_BB) {
        g.strat = kGridBB;
        g.blocks_x = nb;
        g.vb_count = nb * nb;
        passes.push_back(g);
    } else if (is_ltm(s)) {
        g.strat = kGridLTM;
        g.engine = ltm_engine(s);
        const uint64_t side = ceil_sqrt(tri(nb));
        g.blocks_x = side;
        g.vb_count = side * side;
        g.lam_count = tri(nb);
        passes.push_back(g);
    } else if (s == TG_UTM) {
        g.strat = kGridUTM;
        g.engine = P.engine;  // newton unless the StrategyId says otherwise (strategies.cpp:24)
        g.pairs = tri_nd(n);
        g.disc_base = (2 * n - 1) * (2 * n - 1);
        const uint64_t tpb = (uint64_t)rho * rho;
        g.vb_count = g.pairs == 0 ? 1 : ceil_div(g.pairs, tpb);
        g.blocks_x = g.vb_count;
        passes.push_back(g);
    } else if (s == TG_RB) {
        g.strat = kGridRB;
        const uint64_t w = (n % 2 == 0) ? n / 2 : (n + 1) / 2, h = (n % 2 == 0) ? n + 1 : n;
        g.blocks_x = ceil_div(w, rho);
        g.vb_count = g.blocks_x * ceil_div(h, rho);
        passes.push_back(g);
    } else {  // REC: k square passes + 1 diagonal pass, one launch each
        const uint64_t m = P.m;
        const uint32_t k = P.k;
        g.m = m;
        for (uint32_t level = 1; level <= k; ++level) {
            GridGeom p = g;
            p.strat = kGridRECSq;
            p.side = m << (level - 1);
            p.sb = p.side / rho;
            p.blocks_x = p.sb;
            p.vb_count = p.sb * p.sb * (1ull << (k - level));
            passes.push_back(p);
        }
        GridGeom p = g;
        p.strat = kGridRECDiag;
        p.side = m;
        p.sb = m / rho;
        p.blocks_x = p.sb;
        p.vb_count = p.sb * p.sb * (1ull << k);
        passes.push_back(p);
    }
    return passes;
}

// One launch per grid pass (run_strategy's pass loop, engine.cpp:87-133);
// marks (optional, passes.size() + 1 events) bracket the passes for per-pass
// device times.
template <class Body>
tg_status launch_grid(const std::vector<GridGeom>& passes, Body body, cudaStream_t st,
                      const std::vector<cudaEvent_t>* marks = nullptr) {
    for (size_t p = 0; p < passes.size(); ++p) {
        const GridGeom& g = passes[p];
        if (marks) TG_CUDA(cudaEventRecord((*marks)[p], st));
        if (g.vb_count == 0) continue;
        const uint32_t threads = std::min<uint32_t>(g.rho * g.rho, 1024);
        const uint64_t blocks = std::min<uint64_t>(g.vb_count, 0x7fffffffull);
        grid_kernel<Body><<<(unsigned)blocks, threads, 0, st>>>(g, body);
        ++g_launches;
        TG_CUDA(cudaGetLastError());
    }
    if (marks) TG_CUDA(cudaEventRecord(marks->back(), st));
    return TG_OK;
}

template <class T>
tg_status launch_diag_fill(T* out, uint64_t n, bool write_table, cudaStream_t st, int sms) {
    const uint64_t blocks = std::min<uint64_t>(ceil_div(n, 256), (uint64_t)sms * 4);
    diag_fill_kernel<T><<<(unsigned)blocks, 256, 0, st>>>(out, n, write_table ? 1 : 0);
    ++g_launches;
    TG_CUDA(cudaGetLastError());
    return TG_OK;
}

// ------------------------------------------------------------- timing

struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t st;
    bool on;
    Timer(cudaStream_t s, bool enable) : st(s), on(enable) {
        if (on) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, st);
        }
    }
    tg_status finish(tg_dispatch_stats* stats) {
        if (!on) return TG_OK;
        TG_CUDA(cudaEventRecord(b, st));
        TG_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        TG_CUDA(cudaEventElapsedTime(&ms, a, b));
        if (stats) stats->wall_time_ns = (uint64_t)std::llround((double)ms * 1e6);
        return TG_OK;
    }
    ~Timer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

tg_launch_opts default_opts() {
    tg_launch_opts o;
    tg_launch_opts_init(&o);
    return o;
}

bool resolve_span(const tg_launch_opts& o, tg_strategy s, uint32_t rho, bool body_ok) {
    if (o.mode == TG_MODE_GRID) return false;
    const bool ok = body_ok && span_eligible(s, rho);
    return o.mode == TG_MODE_SPAN ? true : ok;
}

// A/B switch: TG_COLLIDE_V1=1 keeps the first span collision kernel (one pair per lane per word).
bool collide_v1() {
    static bool v = [] {
        const char* e = std::getenv("TG_COLLIDE_V1");
        return e && std::atoi(e) != 0;
    }();
    return v;
}

// A/B switch: TG_COLLIDE_V2=1 keeps the second span collision kernel (unpaired operands, select trees).
bool collide_v2() {
    static bool v = [] {
        const char* e = std::getenv("TG_COLLIDE_V2");
        return e && std::atoi(e) != 0;
    }();
    return v;
}

// The td-kernel launch behind tg_launch (launch_dummy / launch_edm /
// launch_count / launch, engine.cpp:150-203) for a validated problem.  Per-pass
// device times go to o.per_pass (LaunchOptions::per_pass, engine.cpp:87-133):
// REC's passes are then launched one by one, bracketed by events.
tg_status launch_impl(tg_kernel kernel, const Problem& P, uint32_t d, const float* pts, void* out,
                      const tg_launch_opts& o, tg_dispatch_stats* stats) {
    const tg_strategy s = P.s;
    const uint64_t n = P.n;
    const uint32_t rho = P.rho;
    const uint32_t G = o.shard_count == 0 ? 1 : o.shard_count;
    tg_dispatch_stats st_local;
    std::vector<tg_dispatch_stats> pp;
    TG_TRY(stats_for(P, o.shard_index, G, &st_local, &pp));
    if (o.per_pass && o.per_pass_cap < pp.size())
        return fail(TG_EINVAL, "per_pass: buffer holds fewer entries than the strategy's grid passes");
    auto report = [&](bool timed_passes) {
        if (stats) *stats = st_local;
        if (o.per_pass) {
            for (size_t p = 0; p < pp.size(); ++p) {
                if (!timed_passes) pp[p].wall_time_ns = pp.size() == 1 ? st_local.wall_time_ns : 0;
                o.per_pass[p] = pp[p];
            }
        }
        return TG_OK;
    };
    if (G > 1 && kernel != TG_KERNEL_DUMMY) {
        uint64_t eb, ee;
        TG_TRY(tg_shard_elems(n, rho, o.shard_index, G, 1, &eb, &ee));
        if (ee == eb) return report(false);  // empty shard (more shards than block rows): nothing to do
    }
    if (kernel == TG_KERNEL_EDM) {
        if (d < 1) return fail(TG_EINVAL, "launch_edm: features must be >= 1");
        if (!pts || !out) return fail(TG_EINVAL, "launch: EDM kernel needs points and an output buffer");
        if (reinterpret_cast<uintptr_t>(pts) % 16 != 0)
            return fail(TG_EINVAL, "launch_edm: device points must be 16-byte aligned");
    }
    if ((kernel == TG_KERNEL_WRITE || kernel == TG_KERNEL_COUNT) && !out)
        return fail(TG_EINVAL, "launch: output buffer is NULL");
    if (kernel == TG_KERNEL_EDM || kernel == TG_KERNEL_WRITE) {
        if (reinterpret_cast<uintptr_t>(out) % 16 != 0)
            return fail(TG_EINVAL, "launch: device output must be 16-byte aligned");
    }
    if ((int)kernel < 0 || (int)kernel > (int)TG_KERNEL_COUNT) return fail(TG_EINVAL, "launch: unknown kernel kind");
    DeviceCtx* c;
    TG_TRY(get_ctx(o.device, &c));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(o.stream);
    const Window w = window_of(P, o.shard_index, G);
    const OutWin ow{tri(w.r_lo), tri(w.r_hi)};
    if (o.mode == TG_MODE_GRAM) {
        if (kernel != TG_KERNEL_EDM) return fail(TG_EINVAL, "gram mode computes the EDM only");
        if (!(is_ltm(s) || s == TG_BB))
            return fail(TG_EINVAL, "gram mode tiles the triangle by g(lambda) (bb / ltm-* strategies)");
        Timer timer(st, !o.async);
        if (!gram_v1()) {
            TG_TRY(launch_gram2_edm(n, d, rho, w.b0, w.b1, ow, pts, static_cast<float*>(out), c, st));
        } else {
            Scratch sn;
            TG_TRY(scratch_alloc(sn, n * sizeof(float), st));
            TG_TRY(launch_gram_edm(n, d, rho, w.b0, w.b1, ow, pts, static_cast<float*>(out),
                                   static_cast<float*>(sn.p), st, c));
        }
        TG_TRY(timer.finish(&st_local));
        return report(false);
    }
    // the dummy kernel runs in span form only on request: AUTO keeps the
    // paper's one-thread-per-cell dummy so the mapping comparison (I vs BB)
    // of the reference protocol stays within one execution shape
    const bool body_span = (kernel == TG_KERNEL_EDM && (d <= 4 || (rho == 16 && square_tiles(s)))) ||
                           kernel == TG_KERNEL_WRITE || kernel == TG_KERNEL_COUNT ||
                           (kernel == TG_KERNEL_DUMMY && o.mode == TG_MODE_SPAN);
    const bool span = resolve_span(o, s, rho, body_span);
    if (span && !(body_span && span_eligible(s, rho)))
        return fail(TG_EINVAL, "span mode needs rho % 4 == 0, rho <= 128 and an edm (d <= 4; d > 4 with "
                               "rho == 16 for bb/ltm-*/rec), write, count or dummy body");
    if (G > 1 && !span) return fail(TG_EINVAL, "sharded launches run in span mode");

    const bool timed_passes = o.per_pass && !o.async && pp.size() > 1;
    std::vector<cudaEvent_t> marks;
    struct EvGuard {
        std::vector<cudaEvent_t>& v;
        ~EvGuard() {
            for (auto e : v) cudaEventDestroy(e);
        }
    } evg{marks};
    if (timed_passes) {
        marks.resize(pp.size() + 1);
        for (auto& e : marks) TG_CUDA(cudaEventCreate(&e));
    }
    Timer timer(st, !o.async);
    if (span) {
        const bool wide = kernel == TG_KERNEL_EDM && d > 4;
        const int slots = wide ? (wide_v1() ? 1 : kW2CH)
                               : ((kernel == TG_KERNEL_WRITE || kernel == TG_KERNEL_COUNT) ? write_slots()
                                                                                              : span_slots());
        const uint32_t C = std::max<uint32_t>(1, (uint32_t)(128 * slots) / rho);
        Scratch fs;
        unsigned int* flag = nullptr;
        if (kernel == TG_KERNEL_EDM) {  // per-launch classify verdict (stream-ordered, private)
            TG_TRY(scratch_alloc(fs, sizeof(unsigned int), st));
            flag = static_cast<unsigned int*>(fs.p);
            TG_TRY(launch_classify(pts, n * d, flag, st, c->sms));
        }
        // REC with per-pass timing: one launch per grid pass, reference order
        const int npl = (timed_passes && s == TG_REC) ? (int)pp.size() : 1;
        for (int pl = 0; pl < npl; ++pl) {
            SpanGeom g;
            TG_TRY(plan_span(P, w, C, &g, !wide, npl > 1 ? pl : -1));
            if (timed_passes) TG_CUDA(cudaEventRecord(marks[pl], st));
            if (kernel == TG_KERNEL_EDM) {
                if (d <= 4) {
                    TG_TRY(launch_span_edm(d, g, ow, pts, static_cast<float*>(out), flag, st, o.persistent != 0,
                                           c->sms));
                } else {
                    TG_TRY(launch_wide_edm(d, g, ow, pts, static_cast<float*>(out), flag, st, o.persistent != 0,
                                           c->sms, c));
                }
            } else if (kernel == TG_KERNEL_DUMMY) {
                auto* sink = o.sink ? static_cast<unsigned long long*>(o.sink) : c->scratch;
                const uint64_t grid = span_grid(g, o.persistent != 0, c->sms, 8);
                if (grid) {
                    span_dummy_kernel<<<(unsigned)grid, kWarpsPerCta * 32, 0, st>>>(g, sink, o.sentinel);
                    ++g_launches;
                    TG_CUDA(cudaGetLastError());
                }
            } else if (kernel == TG_KERNEL_COUNT) {
                TG_TRY(launch_span_count(g, ow, static_cast<uint32_t*>(out), st, o.persistent != 0, c->sms));
            } else {
                TG_TRY(launch_span_write(g, ow, static_cast<uint32_t*>(out), st, o.persistent != 0, c->sms));
            }
        }
        if (timed_passes) {
            if (npl == 1)  // single span launch for a multi-pass grid: time it as a whole
                for (size_t p = 1; p < marks.size() - 1; ++p) TG_CUDA(cudaEventRecord(marks[p], st));
            TG_CUDA(cudaEventRecord(marks.back(), st));
        }
    } else {
        const auto passes = plan_grid(P);
        const std::vector<cudaEvent_t>* mk = timed_passes ? &marks : nullptr;
        switch (kernel) {
            case TG_KERNEL_EDM:
                TG_TRY(launch_grid(passes, EdmBody{pts, static_cast<float*>(out), d}, st, mk));
                if (s == TG_UTM) TG_TRY(launch_diag_fill(static_cast<float*>(out), n, false, st, c->sms));
                break;
            case TG_KERNEL_WRITE:
                TG_TRY(launch_grid(passes, WriteBody{static_cast<uint32_t*>(out)}, st, mk));
                if (s == TG_UTM) TG_TRY(launch_diag_fill(static_cast<uint32_t*>(out), n, true, st, c->sms));
                break;
            case TG_KERNEL_COUNT:
                TG_TRY(launch_grid(passes, CountBody{static_cast<uint32_t*>(out)}, st, mk));
                break;
            default: {  // TG_KERNEL_DUMMY
                auto* sink = o.sink ? static_cast<unsigned long long*>(o.sink) : c->scratch;
                TG_TRY(launch_grid(passes, DummyBody{sink, o.sentinel}, st, mk));
                break;
            }
        }
    }
    TG_TRY(timer.finish(&st_local));
    if (timed_passes) {
        for (size_t p = 0; p < pp.size(); ++p) {
            float ms = 0;
            TG_CUDA(cudaEventElapsedTime(&ms, marks[p], marks[p + 1]));
            pp[p].wall_time_ns = (uint64_t)std::llround((double)ms * 1e6);
        }
    }
    return report(timed_passes);
}

}  // namespace

// ======================================================================
extern "C" {

void tg_launch_opts_init(tg_launch_opts* o) {
    std::memset(o, 0, sizeof(*o));
    o->device = -1;
    o->mode = TG_MODE_AUTO;
    o->sentinel = ~0ull;
    o->engine = -1;
}

const char* tg_last_error(void) { return g_err.c_str(); }
int tg_api_version(void) { return TG_API_VERSION; }
uint64_t tg_last_launch_count(void) { return g_launches; }

uint64_t tg_tri_count(uint64_t n, int with_diag) { return tri_count(n, with_diag != 0); }

tg_status tg_tri_linear_index(uint64_t i, uint64_t j, uint64_t* out) {
    if (j > i) return fail(TG_ERANGE, "tri_linear_index: j > i is outside the lower triangle");
    *out = i * (i + 1) / 2 + j;
    return TG_OK;
}

tg_status tg_grid_side_balanced(uint64_t n, uint64_t* out) {
    if (n == 0) return fail(TG_EINVAL, "grid_side_balanced: n must be >= 1");
    *out = ceil_sqrt(tri(n));
    return TG_OK;
}

uint64_t tg_isqrt(uint64_t v) { return isqrt(v); }
float tg_fast_inv_sqrt(float x, int iterations) { return fast_inv_sqrt(x, iterations); }
float tg_rsqrt_single(float x) { return 1.0f / std::sqrt(x); }

tg_status tg_sqrt_via(int engine, double x, double* out) {
    if (std::isnan(x) || std::isinf(x) || x < 0.0)
        return fail(TG_EINVAL, "sqrt_via: x must be finite and non-negative");
    switch (engine) {
        case kNative: *out = (double)std::sqrt((float)x); return TG_OK;
        case kNewton:
            if (x == 0.0) return fail(TG_EINVAL, "sqrt_via: NewtonRaphson requires x > 0");
            *out = (double)engine_sqrt(kNewton, (float)x);
            return TG_OK;
        case kReciprocal:
            if (x == 0.0) return fail(TG_EINVAL, "sqrt_via: Reciprocal requires x > 0");
            *out = (double)engine_sqrt(kReciprocal, (float)x);
            return TG_OK;
        case kExact:
            if (x != std::floor(x) || x > 0x1p53)
                return fail(TG_EINVAL, "sqrt_via: ExactInteger requires an integral x");
            *out = (double)isqrt((uint64_t)x);
            return TG_OK;
    }
    return fail(TG_EINVAL, "sqrt_via: unknown engine variant");
}

tg_status tg_ltm_map(uint64_t lambda, int engine, int with_diag, uint64_t* i, uint64_t* j) {
    if (engine < 0 || engine > 3) return fail(TG_EINVAL, "ltm_map: unknown engine");
    const Coord c = ltm_map(lambda, engine, with_diag != 0);
    *i = c.i;
    *j = c.j;
    return TG_OK;
}

int tg_bb_map(uint64_t x, uint64_t y, uint64_t* i, uint64_t* j) {
    if (x > y) return 0;
    *i = y;
    *j = x;
    return 1;
}

tg_status tg_utm_map(uint64_t k, uint64_t n, int engine, uint64_t* a, uint64_t* b) {
    if (n < 2 || k >= tri_nd(n)) return fail(TG_ERANGE, "utm_map: k outside [0, N(N-1)/2)");
    const Coord p = utm_pair(k, n, (2 * n - 1) * (2 * n - 1), engine);
    *a = p.i;
    *b = p.j;
    return TG_OK;
}

tg_status tg_rb_rect(uint64_t n, uint64_t* w, uint64_t* h) {
    if (n < 2) return fail(TG_EINVAL, "rb_rect: N must be >= 2");
    if (n % 2 == 0) {
        *w = n / 2;
        *h = n + 1;
    } else {
        *w = (n + 1) / 2;
        *h = n;
    }
    return TG_OK;
}

int tg_rb_map(uint64_t tx, uint64_t ty, uint64_t n, uint64_t* i, uint64_t* j) {
    Coord c;
    if (!rb_map(tx, ty, n, &c)) return 0;
    *i = c.i;
    *j = c.j;
    return 1;
}

int tg_rec_decompose(uint64_t n, uint32_t rho, uint64_t* m, uint32_t* k) {
    if (rho == 0) return 0;
    return rec_decompose(n, rho, m, k) ? 1 : 0;
}

tg_status tg_count_wasted(tg_strategy s, uint64_t n, uint64_t* out) {
    if (n == 0) return fail(TG_EINVAL, "count_wasted: n must be >= 1");
    if (s == TG_BB) {
        *out = n * (n - 1) / 2;
        return TG_OK;
    }
    if (is_ltm(s)) {
        const uint64_t side = ceil_sqrt(tri(n));
        *out = side * side - tri(n);
        return TG_OK;
    }
    return fail(TG_EINVAL, "count_wasted: no closed form for this strategy");
}

double tg_ltm_diag_waste_blocks(uint64_t n) { return static_cast<double>(n) / 2.0; }

tg_status tg_improvement_model(double beta, double tau, double n, double* out) {
    if (!(beta > 0.0) || !(tau > 0.0))
        return fail(TG_EINVAL, "improvement_model: beta and tau must be positive");
    if (!(n >= 1.0)) return fail(TG_EINVAL, "improvement_model: n must be >= 1");
    *out = 2.0 * beta * n * n / (tau * n * n + tau * n);
    return TG_OK;
}

tg_status tg_parse_strategy(const char* name, tg_strategy* out) {
    static const char* names[] = {"bb", "ltm-x", "ltm-n", "ltm-r", "ltm-exact", "utm", "rb", "rec"};
    if (name)
        for (int t = 0; t < 8; ++t)
            if (std::strcmp(name, names[t]) == 0) {
                *out = (tg_strategy)t;
                return TG_OK;
            }
    return fail(TG_EINVAL, std::string("unknown strategy '") + (name ? name : "") + "'");
}

tg_status tg_dispatch_stats_for(tg_strategy s, uint64_t n, uint32_t rho, uint32_t shard_index,
                                uint32_t shard_count, tg_dispatch_stats* out) {
    return stats_for(s, n, rho, shard_index, shard_count, out);
}

tg_status tg_shard_rows(uint64_t n, uint32_t rho, uint32_t shard_count, uint64_t* rows) {
    if (n == 0 || rho == 0 || shard_count == 0) return fail(TG_EINVAL, "tg_shard_rows: bad arguments");
    const auto r = shard_rows(ceil_div(n, rho), shard_count);
    std::copy(r.begin(), r.end(), rows);
    return TG_OK;
}

tg_status tg_shard_elems(uint64_t n, uint32_t rho, uint32_t shard_index, uint32_t shard_count,
                         int with_diag, uint64_t* begin, uint64_t* end) {
    const uint32_t G = shard_count == 0 ? 1 : shard_count;
    if (n == 0 || rho == 0 || shard_index >= G) return fail(TG_EINVAL, "tg_shard_elems: bad arguments");
    const auto r = shard_rows(ceil_div(n, rho), G);
    const uint64_t i0 = std::min<uint64_t>(n, r[shard_index] * rho);
    const uint64_t i1 = std::min<uint64_t>(n, r[shard_index + 1] * rho);
    *begin = tri_count(i0, with_diag != 0);
    *end = tri_count(i1, with_diag != 0);
    return TG_OK;
}

tg_status tg_launch(tg_kernel kernel, tg_strategy s, uint64_t n, uint32_t d, uint32_t rho,
                    const float* pts, void* out, const tg_launch_opts* opts,
                    tg_dispatch_stats* stats) {
    g_launches = 0;
    const tg_launch_opts o = opts ? *opts : default_opts();
    Problem P;
    TG_TRY(make_problem(s, n, rho, &o, &P));
    DevGuard guard;
    return launch_impl(kernel, P, d, pts, out, o, stats);
}

tg_status tg_collide(tg_strategy s, uint64_t n, uint32_t rho, const float* spheres, float r_max,
                     uint32_t* bits, uint64_t* hits, const tg_launch_opts* opts,
                     tg_dispatch_stats* stats) {
    g_launches = 0;
    const tg_launch_opts o = opts ? *opts : default_opts();
    Problem P;
    TG_TRY(make_problem(s, n, rho, &o, &P));
    if (!spheres || !bits || !hits) return fail(TG_EINVAL, "collide: NULL buffer");
    if (reinterpret_cast<uintptr_t>(spheres) % 16 != 0)
        return fail(TG_EINVAL, "collide: spheres must be 16-byte aligned");
    const uint32_t G = o.shard_count == 0 ? 1 : o.shard_count;
    tg_dispatch_stats st_local;
    TG_TRY(stats_for(P, o.shard_index, G, &st_local));
    DevGuard guard;
    DeviceCtx* c;
    TG_TRY(get_ctx(o.device, &c));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(o.stream);
    const bool ok_span = span_eligible(s, rho) && (square_tiles(s) || s == TG_RB);
    const bool span = resolve_span(o, s, rho, ok_span);
    if (span && !ok_span) return fail(TG_EINVAL, "span collide needs bb/ltm-*/rec/rb and rho % 4 == 0");
    if (G > 1 && !span) return fail(TG_EINVAL, "sharded launches run in span mode");
    uint64_t p0, p1;
    TG_TRY(tg_shard_elems(n, rho, o.shard_index, G, 0, &p0, &p1));
    Timer timer(st, !o.async);
    TG_CUDA(cudaMemsetAsync(hits, 0, sizeof(uint64_t), st));
    if (span) {
        const Window w = window_of(P, o.shard_index, G);
        SpanGeom g;
        TG_TRY(plan_span(P, w, std::max<uint32_t>(1, (collide_v1() ? 128 : 32 * TG_COLLIDE_SLOTS) / rho), &g));
        const uint64_t grid = span_grid(g, o.persistent != 0, c->sms, 8);
        if (grid && collide_v1()) {
            span_collide_kernel<<<(unsigned)grid, kWarpsPerCta * 32, 0, st>>>(
                g, p0, p1, reinterpret_cast<const float4*>(spheres), r_max, bits,
                reinterpret_cast<unsigned long long*>(hits));
            ++g_launches;
            TG_CUDA(cudaGetLastError());
        } else if (grid) {
            // partial words at row-segment ends are OR-ed into a zeroed table
            TG_CUDA(cudaMemsetAsync(bits, 0, ceil_div(p1 - p0, 32) * 4, st));
            const uint64_t grid2 = span_grid(g, o.persistent != 0, c->sms, 32, kCollideWarps);
            const float4* sph4 = reinterpret_cast<const float4*>(spheres);
            unsigned long long* h = reinterpret_cast<unsigned long long*>(hits);
            if (collide_v2()) {
                span_collide2_kernel<TG_COLLIDE_SLOTS><<<(unsigned)grid2, kCollideWarps * 32, 0, st>>>(
                    g, p0, sph4, r_max, bits, h);
                ++g_launches;
            } else {
                // pre-paired column operands (qa, qb: 2 x 16 B per sphere), private to the launch
                Scratch sq;
                TG_TRY(scratch_alloc(sq, (size_t)n * 2 * sizeof(float4), st));
                float4* qa = static_cast<float4*>(sq.p);
                float4* qb = qa + n;
                collide_pairs_prep_kernel<<<(unsigned)std::min<uint64_t>(ceil_div(n, 256), (uint64_t)c->sms * 8), 256, 0,
                                            st>>>(sph4, n, r_max, qa, qb);
                span_collide3_kernel<TG_COLLIDE_SLOTS><<<(unsigned)grid2, kCollideWarps * 32, 0, st>>>(
                    g, p0, sph4, qa, qb, r_max, bits, h);
                g_launches += 2;
            }
            TG_CUDA(cudaGetLastError());
        }
    } else {
        TG_CUDA(cudaMemsetAsync(bits, 0, ceil_div(p1 - p0, 32) * 4, st));
        TG_TRY(launch_grid(plan_grid(P),
                           CollideBody{reinterpret_cast<const float4*>(spheres), r_max, bits,
                                       reinterpret_cast<unsigned long long*>(hits)},
                           st));
    }
    TG_TRY(timer.finish(&st_local));
    if (stats) *stats = st_local;
    return TG_OK;
}

}  // extern "C"

namespace {

// One device's part of tg_edm_strategy_host: lambda-range shard `shard` of G
// of problem P, host points in, the shard's packed slice out (host).  The
// kernel runs in block-row pieces whose D2H copies overlap the next piece.
tg_status edm_host_shard(const Problem& P, const float* pts, uint32_t d, float* out, const tg_launch_opts& o,
                         int device, uint32_t shard, uint32_t G, uint64_t* wall_ns) {
    const uint64_t n = P.n;
    const uint32_t rho = P.rho;
    DeviceCtx* c;
    TG_TRY(get_ctx(device, &c));
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t st = (o.stream && o.n_devices <= 1) ? reinterpret_cast<cudaStream_t>(o.stream) : c->stream;
    const bool span = resolve_span(o, P.s, rho, true);
    if (G > 1 && !span) return fail(TG_EINVAL, "sharded launches run in span mode");
    if (span && !span_eligible(P.s, rho))
        return fail(TG_EINVAL, "span mode needs rho % 4 == 0 and rho <= 128");
    const Window w = window_of(P, shard, G);
    const uint64_t b0 = w.b0, b1 = w.b1;
    const uint64_t eb = tri(w.r_lo), ee = tri(w.r_hi);
    const uint64_t elems = ee - eb;
    *wall_ns = 0;
    if (elems == 0) return TG_OK;
    TG_TRY(ensure_buf(c->bufs[0], n * d * sizeof(float)));
    TG_TRY(ensure_buf(c->bufs[1], elems * sizeof(float)));
    float* d_pts = static_cast<float*>(c->bufs[0].p);
    float* d_out = static_cast<float*>(c->bufs[1].p);

    TG_CUDA(cudaEventRecord(c->ev[32], st));
    TG_CUDA(cudaMemcpyAsync(d_pts, pts, n * d * sizeof(float), cudaMemcpyHostToDevice, st));
    if (span) {
        Scratch fs;
        TG_TRY(scratch_alloc(fs, sizeof(unsigned int), st));
        unsigned int* flag = static_cast<unsigned int*>(fs.p);
        TG_TRY(launch_classify(d_pts, n * d, flag, st, c->sms));
        // Copy pipeline: pieces of block rows (row windows: every strategy's
        // piece q writes exactly the packed rows of its window), each piece's
        // D2H overlapping the next piece's kernel.
        const uint64_t bytes = elems * sizeof(float);
        uint32_t Q = (uint32_t)std::min<uint64_t>(16, std::max<uint64_t>(1, bytes >> 28));
        Q = (uint32_t)std::min<uint64_t>(Q, std::max<uint64_t>(1, b1 - b0));
        std::vector<uint64_t> pr(Q + 1);  // piece bounds: [b0, b1) split by element count
        pr[0] = b0;
        pr[Q] = b1;
        for (uint32_t q = 1; q < Q; ++q) {
            const uint64_t target = tri(b0) + (tri(b1) - tri(b0)) * q / Q;
            uint64_t r = fix_row(ltm_row_guess(target, kExact, true), target, true);
            pr[q] = std::min(std::max(r, pr[q - 1]), b1);
        }
        const uint32_t C = std::max<uint32_t>(1, (uint32_t)(128 * span_slots()) / rho);
        const OutWin ow{eb, ee};
        uint64_t lo = 0, sub_k = 0;
        for (uint32_t q = 0; q < Q; ++q) {
            const Window wq{pr[q], pr[q + 1], std::min<uint64_t>(n, pr[q] * rho), std::min<uint64_t>(n, pr[q + 1] * rho)};
            SpanGeom g;
            TG_TRY(plan_span(P, wq, C, &g));
            TG_TRY(launch_span_edm(d, g, ow, d_pts, d_out, flag, st, o.persistent != 0, c->sms));
            TG_CUDA(cudaEventRecord(c->ev[q], st));
            const uint64_t piece_end = tri(wq.r_hi) - eb;
            const uint64_t hi = (q + 1 == Q) ? elems : std::min<uint64_t>(elems, (piece_end + 3) & ~3ull);
            if (hi > lo) {
                // 256 MB sub-copies alternating two streams: 56 vs 52 GB/s for one
                // 8.6 GB copy on B200 PCIe Gen5 x16 (scripts/d2h_probe.py)
                TG_CUDA(cudaStreamWaitEvent(c->copy_stream, c->ev[q], 0));
                TG_CUDA(cudaStreamWaitEvent(c->copy_stream2, c->ev[q], 0));
                constexpr uint64_t kSub = (256ull << 20) / sizeof(float);
                for (uint64_t a = lo; a < hi; a += kSub) {
                    const uint64_t bnd = std::min<uint64_t>(hi, a + kSub);
                    TG_CUDA(cudaMemcpyAsync(out + a, d_out + a, (bnd - a) * sizeof(float), cudaMemcpyDeviceToHost,
                                            (sub_k++ & 1) ? c->copy_stream2 : c->copy_stream));
                }
                lo = hi;
            }
        }
        TG_CUDA(cudaEventRecord(c->ev[33], st));
    } else {
        TG_TRY(launch_grid(plan_grid(P), EdmBody{d_pts, d_out, d}, st));
        if (P.s == TG_UTM) TG_TRY(launch_diag_fill(d_out, n, false, st, c->sms));
        TG_CUDA(cudaEventRecord(c->ev[33], st));
        TG_CUDA(cudaStreamWaitEvent(c->copy_stream, c->ev[33], 0));
        TG_CUDA(cudaMemcpyAsync(out, d_out, elems * sizeof(float), cudaMemcpyDeviceToHost, c->copy_stream));
    }
    TG_CUDA(cudaStreamSynchronize(c->copy_stream));
    TG_CUDA(cudaStreamSynchronize(c->copy_stream2));
    TG_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    TG_CUDA(cudaEventElapsedTime(&ms, c->ev[32], c->ev[33]));
    *wall_ns = (uint64_t)std::llround((double)ms * 1e6);
    return TG_OK;
}

// Coverage verdict of one count table on device: cells of the window that
// are not touched exactly once (0 on the diagonal for a no-diagonal domain).
tg_status check_counts(DeviceCtx* c, cudaStream_t st, const uint32_t* counts, uint64_t n, bool with_diag,
                       uint64_t* bad, uint64_t* first) {
    unsigned long long init[2] = {0, ~0ull};
    TG_CUDA(cudaMemcpyAsync(c->scratch + 1, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const uint64_t blocks = std::min<uint64_t>(ceil_div(tri(n), 256), (uint64_t)c->sms * 16);
    check_counts_kernel<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, 0, st>>>(counts, n, with_diag ? 1 : 0,
                                                                                  c->scratch + 1, c->scratch + 2);
    ++g_launches;
    TG_CUDA(cudaGetLastError());
    unsigned long long res[2];
    TG_CUDA(cudaMemcpyAsync(res, c->scratch + 1, sizeof(res), cudaMemcpyDeviceToHost, st));
    TG_CUDA(cudaStreamSynchronize(st));
    *bad = res[0];
    *first = res[1];
    return TG_OK;
}

}  // namespace

extern "C" {

tg_status tg_edm_strategy_host(tg_strategy s, const float* pts, uint64_t n, uint32_t d,
                               uint32_t rho, float* out, const tg_launch_opts* opts,
                               tg_dispatch_stats* stats) {
    g_launches = 0;
    const tg_launch_opts o = opts ? *opts : default_opts();
    Problem P;
    TG_TRY(make_problem(s, n, rho, &o, &P));
    if (d < 1 || d > 4) return fail(TG_EINVAL, "launch_edm: features must be in [1, 4]");
    if (!pts || !out) return fail(TG_EINVAL, "launch: EDM kernel needs points and an output buffer");
    const uint32_t G = o.shard_count == 0 ? 1 : o.shard_count;
    tg_dispatch_stats st_local;
    TG_TRY(stats_for(P, o.shard_index, G, &st_local));
    DevGuard guard;
    if (o.n_devices <= 1) {
        const int dev = (o.n_devices == 1 && o.devices) ? o.devices[0] : o.device;
        TG_TRY(edm_host_shard(P, pts, d, out, o, dev, o.shard_index, G, &st_local.wall_time_ns));
        if (stats) *stats = st_local;
        return TG_OK;
    }
    // several devices: shard g of n_devices on devices[g], each copying its
    // slice out over its own link, in parallel host threads
    if (G > 1) return fail(TG_EINVAL, "edm_strategy: n_devices > 1 splits the whole domain (shard_count must be 0/1)");
    if (!o.devices) return fail(TG_EINVAL, "edm_strategy: n_devices > 1 needs a devices array");
    const uint32_t D = o.n_devices;
    TG_TRY(stats_for(P, 0, 1, &st_local));
    std::vector<tg_status> rc(D, TG_OK);
    std::vector<std::string> err(D);
    std::vector<uint64_t> wall(D, 0);
    std::vector<std::thread> th;
    for (uint32_t g = 0; g < D; ++g) {
        th.emplace_back([&, g] {
            const Window w = window_of(P, g, D);
            rc[g] = edm_host_shard(P, pts, d, out + tri(w.r_lo), o, o.devices[g], g, D, &wall[g]);
            if (rc[g] != TG_OK) err[g] = g_err;
        });
    }
    for (auto& t : th) t.join();
    for (uint32_t g = 0; g < D; ++g)
        if (rc[g] != TG_OK) return fail(rc[g], "device " + std::to_string(o.devices[g]) + ": " + err[g]);
    st_local.wall_time_ns = *std::max_element(wall.begin(), wall.end());
    if (stats) *stats = st_local;
    return TG_OK;
}

tg_status tg_coverage_ok_opts(tg_strategy s, uint64_t n, uint32_t rho, const tg_launch_opts* opts, int* ok,
                              uint64_t* bad, uint64_t* first_bad) {
    g_launches = 0;
    tg_launch_opts o = opts ? *opts : default_opts();
    Problem P;
    TG_TRY(make_problem(s, n, rho, &o, &P));
    o.shard_index = 0;
    o.shard_count = 1;
    o.async = 0;
    o.per_pass = nullptr;
    DevGuard guard;
    DeviceCtx* c;
    TG_TRY(get_ctx(o.device, &c));
    std::lock_guard<std::mutex> lk(c->mu);
    o.device = c->dev;
    o.stream = c->stream;
    const uint64_t cells = tri(n);
    TG_TRY(ensure_buf(c->bufs[2], cells * sizeof(uint32_t)));
    uint32_t* counts = static_cast<uint32_t*>(c->bufs[2].p);
    TG_CUDA(cudaMemsetAsync(counts, 0, cells * sizeof(uint32_t), c->stream));
    const uint64_t launches0 = g_launches;
    TG_TRY(launch_impl(TG_KERNEL_COUNT, P, 0, nullptr, counts, o, nullptr));
    uint64_t nbad, first;
    TG_TRY(check_counts(c, c->stream, counts, n, s != TG_UTM, &nbad, &first));
    g_launches += launches0;
    *ok = nbad == 0 ? 1 : 0;
    if (bad) *bad = nbad;
    if (first_bad) *first_bad = first;
    return TG_OK;
}

tg_status tg_coverage_ok(tg_strategy s, uint64_t n, uint32_t rho, int device, int* ok) {
    tg_launch_opts o = default_opts();
    o.device = device;
    return tg_coverage_ok_opts(s, n, rho, &o, ok, nullptr, nullptr);
}

tg_status tg_count_host(tg_strategy s, uint64_t n, uint32_t rho, uint32_t* counts, const tg_launch_opts* opts,
                        tg_dispatch_stats* stats) {
    g_launches = 0;
    tg_launch_opts o = opts ? *opts : default_opts();
    Problem P;
    TG_TRY(make_problem(s, n, rho, &o, &P));
    if (!counts) return fail(TG_EINVAL, "launch_count: NULL counter buffer");
    if (o.shard_count > 1) return fail(TG_EINVAL, "launch_count: the host counter vector covers the whole domain");
    DevGuard guard;
    DeviceCtx* c;
    TG_TRY(get_ctx(o.device, &c));
    std::lock_guard<std::mutex> lk(c->mu);
    o.device = c->dev;
    o.stream = c->stream;
    o.async = 0;
    const uint64_t bytes = tri(n) * sizeof(uint32_t);
    TG_TRY(ensure_buf(c->bufs[2], bytes));
    uint32_t* d = static_cast<uint32_t*>(c->bufs[2].p);
    TG_CUDA(cudaMemcpyAsync(d, counts, bytes, cudaMemcpyHostToDevice, c->stream));
    TG_TRY(launch_impl(TG_KERNEL_COUNT, P, 0, nullptr, d, o, stats));
    TG_CUDA(cudaMemcpyAsync(counts, d, bytes, cudaMemcpyDeviceToHost, c->stream));
    TG_CUDA(cudaStreamSynchronize(c->stream));
    return TG_OK;
}

tg_status tg_dummy_host(tg_strategy s, uint64_t n, uint32_t rho, const tg_launch_opts* opts,
                        tg_dispatch_stats* stats, uint64_t* sink_value) {
    g_launches = 0;
    tg_launch_opts o = opts ? *opts : default_opts();
    Problem P;
    TG_TRY(make_problem(s, n, rho, &o, &P));
    DevGuard guard;
    DeviceCtx* c;
    TG_TRY(get_ctx(o.device, &c));
    std::lock_guard<std::mutex> lk(c->mu);
    o.device = c->dev;
    o.stream = c->stream;
    o.async = 0;
    o.sink = c->scratch + 4;
    TG_CUDA(cudaMemsetAsync(c->scratch + 4, 0, sizeof(unsigned long long), c->stream));
    TG_TRY(launch_impl(TG_KERNEL_DUMMY, P, 0, nullptr, nullptr, o, stats));
    unsigned long long v = 0;
    TG_CUDA(cudaMemcpyAsync(&v, c->scratch + 4, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
    TG_CUDA(cudaStreamSynchronize(c->stream));
    if (sink_value) *sink_value = v;
    return TG_OK;
}

// edm_reference (edm.cpp:53-63): sequential by contract -- host binary32
// arithmetic in edm_pair's order (each op separately rounded; the translation
// unit is compiled without FMA contraction for host code, see build.py).
tg_status tg_edm_reference_host(const float* pts, uint64_t n, uint32_t d, float* out) {
    if (n == 0) return fail(TG_EINVAL, "ProblemSize: N must be >= 1");
    if (d == 0) return fail(TG_EINVAL, "edm_reference: features must be >= 1");
    if (!pts || !out) return fail(TG_EINVAL, "edm_reference: NULL buffer");
    uint64_t e = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const float* a = pts + i * d;
        for (uint64_t j = 0; j <= i; ++j, ++e) {
            const float* b = pts + j * d;
            float sum = 0.0f;
            for (uint32_t k = 0; k < d; ++k) {
                const float diff = fsub(a[k], b[k]);
                sum = fadd(sum, fmul(diff, diff));
            }
            out[e] = std::sqrt(sum);
        }
    }
    return TG_OK;
}

tg_status tg_grid_spec(tg_strategy s, uint64_t n, uint32_t rho, const tg_launch_opts* opts, tg_pass* passes,
                       uint32_t cap, uint32_t* npass) {
    Problem P;
    TG_TRY(make_problem(s, n, rho, opts, &P));
    std::vector<tg_pass> v;
    const uint64_t nb = ceil_div(n, rho);
    if (s == TG_BB) {
        v.push_back({nb, nb, 0, 0, 0, 0});
    } else if (is_ltm(s)) {
        const uint64_t side = ceil_sqrt(tri(nb));
        v.push_back({side, side, 0, 0, 0, 0});
    } else if (s == TG_UTM) {
        const uint64_t pairs = tri_nd(n), tpb = (uint64_t)rho * rho;
        v.push_back({pairs == 0 ? 1 : ceil_div(pairs, tpb), 1, 0, 0, 0, 0});
    } else if (s == TG_RB) {
        const uint64_t wd = (n % 2 == 0) ? n / 2 : (n + 1) / 2, h = (n % 2 == 0) ? n + 1 : n;
        v.push_back({ceil_div(wd, rho), ceil_div(h, rho), 0, 0, 0, 0});
    } else {
        for (const RecPassInfo& q : rec_passes(P)) v.push_back({q.sb, q.sb * q.count, 1, q.level, q.side, q.count});
    }
    if (npass) *npass = (uint32_t)v.size();
    if (passes) {
        if (cap < v.size()) return fail(TG_EINVAL, "grid_spec: pass buffer too small");
        std::copy(v.begin(), v.end(), passes);
    }
    return TG_OK;
}

tg_status tg_ltm_map_policy(uint64_t lambda, int engine, int with_diag, int repair, uint64_t* i, uint64_t* j) {
    if (engine < 0 || engine > 3) return fail(TG_EINVAL, "ltm_map: unknown engine");
    if (repair < 0 || repair > 2) return fail(TG_EINVAL, "ltm_map: unknown repair policy");
    const bool wd = with_diag != 0;
    uint64_t r = ltm_row_guess(lambda, engine, wd);
    // RepairPolicy Auto: repair only at lambda >= kRepairFreeLambdaLimit (fastmath.hpp:82-88)
    if (engine != kExact && (repair == 2 || (repair == 0 && lambda >= 1844160ull))) r = fix_row(r, lambda, wd);
    *i = r;
    *j = lambda - row_start(r, wd);
    return TG_OK;
}

tg_status tg_dispatch_stats_opts(tg_strategy s, uint64_t n, uint32_t rho, const tg_launch_opts* opts,
                                 tg_dispatch_stats* out) {
    const tg_launch_opts o = opts ? *opts : default_opts();
    Problem P;
    TG_TRY(make_problem(s, n, rho, &o, &P));
    std::vector<tg_dispatch_stats> pp;
    TG_TRY(stats_for(P, o.shard_index, o.shard_count == 0 ? 1 : o.shard_count, out, &pp));
    if (o.per_pass) {
        if (o.per_pass_cap < pp.size()) return fail(TG_EINVAL, "per_pass: buffer too small");
        std::copy(pp.begin(), pp.end(), o.per_pass);
    }
    return TG_OK;
}

tg_status tg_lambda_sweep(int engine, int with_diag, int fixup, uint64_t begin, uint64_t end,
                          int device, uint64_t* mismatches, uint64_t* first) {
    g_launches = 0;
    if (engine < 0 || engine > 3) return fail(TG_EINVAL, "lambda_sweep: unknown engine");
    if (end < begin) return fail(TG_EINVAL, "lambda_sweep: end < begin");
    if (end > (1ull << 40)) return fail(TG_EINVAL, "lambda_sweep: end beyond 2^40");
    DeviceCtx* c;
    TG_TRY(get_ctx(device, &c));
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t st = c->stream;
    unsigned long long init[2] = {0, ~0ull};
    TG_CUDA(cudaMemcpyAsync(c->scratch + 1, init, sizeof(init), cudaMemcpyHostToDevice, st));
    if (end > begin) {
        const uint64_t blocks = std::min<uint64_t>(ceil_div(end - begin, 256), (uint64_t)c->sms * 32);
        lambda_sweep_kernel<<<(unsigned)blocks, 256, 0, st>>>(engine, with_diag, fixup, begin, end,
                                                              c->scratch + 1, c->scratch + 2);
        ++g_launches;
        TG_CUDA(cudaGetLastError());
    }
    unsigned long long res[2];
    TG_CUDA(cudaMemcpyAsync(res, c->scratch + 1, sizeof(res), cudaMemcpyDeviceToHost, st));
    TG_CUDA(cudaStreamSynchronize(st));
    *mismatches = res[0];
    *first = res[1];
    return TG_OK;
}

tg_status tg_sqrt_selftest(uint32_t lo, uint32_t hi, int device, uint64_t* mismatches) {
    g_launches = 0;
    DeviceCtx* c;
    TG_TRY(get_ctx(device, &c));
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t st = c->stream;
    TG_CUDA(cudaMemsetAsync(c->scratch + 1, 0, sizeof(unsigned long long), st));
    if (hi > lo) {
        const uint64_t blocks = std::min<uint64_t>(ceil_div((uint64_t)hi - lo, 256), (uint64_t)c->sms * 32);
        sqrt_selftest_kernel<<<(unsigned)blocks, 256, 0, st>>>(lo, hi, c->scratch + 1);
        ++g_launches;
        TG_CUDA(cudaGetLastError());
    }
    unsigned long long r;
    TG_CUDA(cudaMemcpyAsync(&r, c->scratch + 1, sizeof(r), cudaMemcpyDeviceToHost, st));
    TG_CUDA(cudaStreamSynchronize(st));
    *mismatches = r;
    return TG_OK;
}

tg_status tg_gen_values(uint64_t count, uint64_t seed, float* out, const tg_launch_opts* opts) {
    g_launches = 0;
    const tg_launch_opts o = opts ? *opts : default_opts();
    if (!out) return fail(TG_EINVAL, "gen_values: NULL output");
    DeviceCtx* c;
    TG_TRY(get_ctx(o.device, &c));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(o.stream);
    if (count) {
        const uint64_t blocks = std::min<uint64_t>(ceil_div(count, 256), (uint64_t)c->sms * 16);
        gen_points_kernel<<<(unsigned)blocks, 256, 0, st>>>(count, seed, out);
        ++g_launches;
        TG_CUDA(cudaGetLastError());
    }
    if (!o.async) TG_CUDA(cudaStreamSynchronize(st));
    return TG_OK;
}

tg_status tg_gen_points_host(uint64_t n, uint32_t d, uint64_t seed, float* out, int device) {
    if (n == 0) return fail(TG_EINVAL, "gen_points: N must be >= 1");
    if (n > kMaxElems) return fail(TG_EINVAL, "gen_points: N exceeds the 2^20 cap");
    if (d < 1 || d > 4) return fail(TG_EINVAL, "gen_points: d must be in [1, 4]");
    DeviceCtx* c;
    TG_TRY(get_ctx(device, &c));
    std::lock_guard<std::mutex> lk(c->mu);
    TG_TRY(ensure_buf(c->bufs[3], n * d * sizeof(float)));
    tg_launch_opts o = default_opts();
    o.device = c->dev;
    o.stream = c->stream;
    o.async = 1;
    TG_TRY(tg_gen_values(n * d, seed, static_cast<float*>(c->bufs[3].p), &o));
    TG_CUDA(cudaMemcpyAsync(out, c->bufs[3].p, n * d * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    TG_CUDA(cudaStreamSynchronize(c->stream));
    return TG_OK;
}

}  // extern "C"

// A/B instrumentation of the Gram kernel (TG_G2_PROF=1 builds only; zeros otherwise)
extern "C" int tg_debug_g2_prof(unsigned long long* out16, int reset) {
#if TG_G2_PROF
    if (cudaMemcpyFromSymbol(out16, tg::tg_g2_prof, 16 * sizeof(unsigned long long)) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(tg::tg_g2_prof, z, sizeof(z));
    }
    return 0;
#else
    for (int k = 0; k < 16; ++k) out16[k] = 0;
    (void)reset;
    return 1;
#endif
}
