/*
 * trigrid_b200.h -- C-ABI of the B200-native triangular-domain library
 * (libtrigrid_b200.so, sm_100a).
 *
 * This is the "thin C-ABI layer in proj/bindings" that the reference's
 * C++ API and pybind module reach the GPU through.  Plain pointers and sizes
 * only; no torch or C++ types.  Every entry point names the reference
 * interface it replaces (/root/reference/proj/<file>:<line>).
 * shows the pybind / ctypes bindings a maintainer adds on the reference side.
 *
 * Errors: every call returns a tg_status.  The reference throws
 *   std::invalid_argument -> TG_EINVAL   (pybind: ValueError)
 *   std::out_of_range     -> TG_ERANGE   (pybind: IndexError)
 *   std::runtime_error    -> TG_ERUNTIME (pybind: RuntimeError)
 * plus TG_ECUDA / TG_ENOMEM for device failures; tg_last_error() returns a
 * thread-local message for the last failing call on this thread.
 *
 * Memory: tg_launch / tg_collide take DEVICE pointers and enqueue on
 * opts->stream (default: the legacy default stream of opts->device); they
 * synchronise before returning unless opts->async is set.  The *_host entry
 * points take HOST pointers (pinned for full PCIe speed) and are synchronous,
 * exactly like the reference's CPU calls.
 */
#ifndef TRIGRID_B200_H_
#define TRIGRID_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_API_VERSION 2

typedef enum {
    TG_OK = 0,
    TG_EINVAL = 1,   /* std::invalid_argument */
    TG_ERANGE = 2,   /* std::out_of_range */
    TG_ERUNTIME = 3, /* std::runtime_error */
    TG_ECUDA = 4,    /* CUDA runtime / launch failure */
    TG_ENOMEM = 5    /* device or pinned allocation failed */
} tg_status;

/* Mapping strategies: parse_strategy names bb, ltm-x, ltm-n, ltm-r, utm, rb,
 * rec (strategies.cpp:19-28) plus ltm-exact (strategy_name, :32-41). */
typedef enum {
    TG_BB = 0,
    TG_LTM_X = 1,     /* g(lambda), sqrtf                      */
    TG_LTM_N = 2,     /* g(lambda), 0x5f3759df + 3 Newton steps */
    TG_LTM_R = 3,     /* g(lambda), rsqrtf (MUFU.RSQ)           */
    TG_LTM_EXACT = 4, /* g(lambda), integer sqrt                */
    TG_UTM = 5,
    TG_RB = 6,
    TG_REC = 7
} tg_strategy;

/* td-kernel bodies. */
typedef enum {
    TG_KERNEL_DUMMY = 0, /* launch_dummy  engine.cpp:150-155: mapping cost only */
    TG_KERNEL_WRITE = 1, /* packed u32 i+j (the dummy kernel made HBM-visible)  */
    TG_KERNEL_EDM = 2,   /* launch_edm    engine.cpp:157-175: packed fp32 EDM   */
    TG_KERNEL_COUNT = 3  /* launch_count  engine.cpp:177-188: u32 += 1 per cell (span: per cell of
                            every owned 16-byte chunk -- the exactly-once check of the span rule) */
} tg_kernel;

/* Execution mode. */
typedef enum {
    TG_MODE_AUTO = 0, /* span when the strategy/rho/body allow it (every strategy: rho % 4 == 0,
                         rho <= 128; bodies edm d <= 4, write, count;
                         d > 4 and collide: bb, ltm-*, rec), else grid */
    TG_MODE_GRID = 1, /* paper-faithful: one CTA of rho*rho threads per grid block, one cell per thread */
    TG_MODE_SPAN = 2, /* B200: warp per run of consecutive blocks, 128-bit owned-chunk stores */
    TG_MODE_GRAM = 3  /* EDM only: Gram trick on tcgen05 (fp16 hi/lo split, kind::f16, any d),
                         stated tolerance
                         |d^2 - d_exact^2| <= 2^-17 (|x_i|^2 + |x_j|^2), diagonal 0; not bit-exact.
                         Any magnitude spread: one power-of-two operand scale when the per-point
                         max |x| spans <= 2^20, per-point scales beyond (finite inputs) */
} tg_mode;

/* Mirrors trigrid::DispatchStats field for field (engine.hpp:19-32).
 * wall_time_ns is DEVICE time (CUDA events around the kernel launches). */
typedef struct {
    uint64_t blocks_launched;
    uint64_t blocks_discarded;
    uint64_t threads_discarded;
    uint64_t wall_time_ns;
} tg_dispatch_stats;

/* Mirrors trigrid::LaunchOptions (engine.hpp:34-37) for a device. */
typedef struct {
    int32_t device;        /* CUDA ordinal; -1 = current device */
    uint32_t mode;         /* tg_mode */
    void* stream;          /* cudaStream_t; NULL = default stream */
    uint32_t async;        /* 1: do not synchronise before returning (stats.wall_time_ns = 0) */
    uint32_t persistent;   /* span mode: 1 = persistent grid (148 x occupancy CTAs) */
    uint32_t shard_index;  /* lambda-range shard g of shard_count (block-row slices, tg_shard_rows) */
    uint32_t shard_count;  /* 0 or 1 = whole domain */
    uint64_t sentinel;     /* dummy kernel: runtime value i+j is compared with (never matches) */
    void* sink;            /* dummy kernel: optional device u64 sink (else internal) */
    /* ---- API version 2 */
    uint64_t rec_m;        /* REC schedule N = m * 2^k (rec_schedule, strategies.cpp:116-140);
                              0 = the largest-k decomposition of make_strategy (rec_decompose) */
    uint32_t rec_k;
    int32_t engine;        /* UTM sqrt engine (StrategyId{UpperTri, engine}, strategies.hpp:27-31):
                              0 native, 1 newton, 2 reciprocal, 3 exact; -1 = newton (parse_strategy("utm")) */
    tg_dispatch_stats* per_pass;  /* LaunchOptions::per_pass (engine.hpp:36, engine.cpp:87-133): when
                                     non-NULL, one entry per grid pass (tg_grid_spec order), each pass
                                     launched and device-timed on its own */
    uint32_t per_pass_cap;        /* entries available at per_pass */
    uint32_t n_devices;           /* host drop-ins: 0/1 = `device` only; > 1 = split the lambda range
                                     into n_devices shards, one per devices[g], each copying its
                                     packed slice out over its own PCIe link */
    const int32_t* devices;
} tg_launch_opts;

/* One grid pass (trigrid::Pass + RecLevel, strategies.hpp:40-60). */
typedef struct {
    uint64_t blocks_x;
    uint64_t blocks_y;
    uint32_t has_level;  /* REC passes carry a level tag */
    uint32_t level;      /* 0 = diagonal pass */
    uint64_t side;
    uint64_t squares;
} tg_pass;

void tg_launch_opts_init(tg_launch_opts* o);

/* ------------------------------------------------------------ geometry */

/* tri_count (tri.hpp:39-41). */
uint64_t tg_tri_count(uint64_t n, int with_diag);
/* tri_linear_index (tri.cpp:17-21); TG_ERANGE when j > i. */
tg_status tg_tri_linear_index(uint64_t i, uint64_t j, uint64_t* out);
/* grid_side_balanced (tri.cpp:23-26); TG_EINVAL when n == 0. */
tg_status tg_grid_side_balanced(uint64_t n, uint64_t* out);
/* isqrt (fastmath.cpp:8-16). */
uint64_t tg_isqrt(uint64_t v);
/* fast_inv_sqrt (fastmath.hpp:22-34) and rsqrt_single (fastmath.hpp:39), host binary32. */
float tg_fast_inv_sqrt(float x, int iterations);
float tg_rsqrt_single(float x);
/* sqrt_via (fastmath.cpp:33-59): engine 0 native, 1 newton, 2 reciprocal, 3 exact. */
tg_status tg_sqrt_via(int engine, double x, double* out);
/* ltm_map (strategies.cpp:60-83): g(lambda) -> (i, j); exact for every lambda. */
tg_status tg_ltm_map(uint64_t lambda, int engine, int with_diag, uint64_t* i, uint64_t* j);
/* bb_map (strategies.hpp:94-97): returns 1 mapped / 0 discarded. */
int tg_bb_map(uint64_t x, uint64_t y, uint64_t* i, uint64_t* j);
/* utm_map (strategies.cpp:85-91): TG_ERANGE outside [0, N(N-1)/2). */
tg_status tg_utm_map(uint64_t k, uint64_t n, int engine, uint64_t* a, uint64_t* b);
/* rb_rect (strategies.cpp:93-97): TG_EINVAL when N < 2. */
tg_status tg_rb_rect(uint64_t n, uint64_t* width, uint64_t* height);
/* rb_map (strategies.hpp:182-193): returns 1 mapped / 0 discarded. */
int tg_rb_map(uint64_t tx, uint64_t ty, uint64_t n, uint64_t* i, uint64_t* j);
/* rec_decompose (strategies.cpp:142-151): returns 1 found / 0 none. */
int tg_rec_decompose(uint64_t n, uint32_t rho, uint64_t* m, uint32_t* k);
/* count_wasted (engine.cpp:205-217): bb and ltm-* only, else TG_EINVAL. */
tg_status tg_count_wasted(tg_strategy s, uint64_t n, uint64_t* out);
/* ltm_diag_waste_blocks (engine.hpp:87, engine.cpp:219-221): n / 2, the LTM
 * diagonal blocks' half-empty share counted in blocks. */
double tg_ltm_diag_waste_blocks(uint64_t n);
/* improvement_model (bench.cpp:138-144). */
tg_status tg_improvement_model(double beta, double tau, double n, double* out);
/* Strategy name <-> id (parse_strategy strategies.cpp:19-28 + "ltm-exact"). */
tg_status tg_parse_strategy(const char* name, tg_strategy* out);

/* grid_of / rec_schedule / rb_grid (strategies.hpp:393-400, strategies.cpp:107-140): the
 * strategy's grid passes.  opts supplies rec_m/rec_k (may be NULL).  *npass is set even when
 * cap is too small (then TG_EINVAL). */
tg_status tg_grid_spec(tg_strategy s, uint64_t n, uint32_t rho, const tg_launch_opts* opts, tg_pass* passes,
                       uint32_t cap, uint32_t* npass);

/* ltm_map with the reference's RepairPolicy (strategies.cpp:60-83, fastmath.hpp:84-103):
 * repair 0 = Auto (repair for lambda >= 1,844,160), 1 = Off (float row only), 2 = On.
 * Host binary32 arithmetic identical to the reference (engine 2 = 1/sqrtf). */
tg_status tg_ltm_map_policy(uint64_t lambda, int engine, int with_diag, int repair, uint64_t* i, uint64_t* j);

/* Closed-form DispatchStats of a launch (what run_strategy tallies,
 * engine.cpp:70-136) for the whole domain or one shard. */
tg_status tg_dispatch_stats_for(tg_strategy s, uint64_t n, uint32_t rho, uint32_t shard_index,
                                uint32_t shard_count, tg_dispatch_stats* out);
/* Same with a full option set (rec_m/rec_k, shard); per-pass stats into opts->per_pass when set. */
tg_status tg_dispatch_stats_opts(tg_strategy s, uint64_t n, uint32_t rho, const tg_launch_opts* opts,
                                 tg_dispatch_stats* out);

/* Lambda-range sharding across G devices (new): block-row bounds
 * rows[0..G] with rows[0] = 0, rows[G] = ceil(N/rho); shard g owns block rows
 * [rows[g], rows[g+1]) = packed elements [T(rho*rows[g]), T(min(N, rho*rows[g+1]))). */
tg_status tg_shard_rows(uint64_t n, uint32_t rho, uint32_t shard_count, uint64_t* rows);
/* Element range [begin, end) of shard g in the with-diagonal (with_diag=1)
 * or no-diagonal (with_diag=0, collision table) packed layout. */
tg_status tg_shard_elems(uint64_t n, uint32_t rho, uint32_t shard_index, uint32_t shard_count,
                         int with_diag, uint64_t* begin, uint64_t* end);

/* -------------------------------------------------------- device kernels */

/* The td-kernel launch: launch_dummy / launch_edm / launch_count / launch
 * (engine.hpp:59-78, engine.cpp:150-203) on a B200.
 *   pts : device float[N*d] row-major (EDM only; 16-byte aligned), d >= 1
 *   out : EDM   -> device float[shard elems]  (packed lambda order, engine.hpp:62-64)
 *         WRITE -> device uint32[shard elems] (i+j)
 *         COUNT -> device uint32[shard elems] (T(N) unsharded), incremented (caller zeroes)
 *         DUMMY -> ignored (see opts->sink)
 * Unlike the reference, EDM accepts any d >= 1 (the reference caps d at 4,
 * engine.cpp:162-163); d in {1,2,3,4} use the register-window span kernel. */
tg_status tg_launch(tg_kernel kernel, tg_strategy s, uint64_t n, uint32_t d, uint32_t rho,
                    const float* pts, void* out, const tg_launch_opts* opts,
                    tg_dispatch_stats* stats);

/* Collision table (new td-kernel; semantics in DESIGN.md, oracle
 * trigrid_oracle.c:or_collide_reference).  spheres: device float[N*4]
 * (x, y, z, u), radius u*r_max.  bits: device uint32[ceil(shard pairs/32)]
 * (pair p = i(i-1)/2 + j - shard_begin at bit p%32 of word p/32; zero bits
 * past the end).  hits: device uint64 accumulated (caller zeroes). */
tg_status tg_collide(tg_strategy s, uint64_t n, uint32_t rho, const float* spheres, float r_max,
                     uint32_t* bits, uint64_t* hits, const tg_launch_opts* opts,
                     tg_dispatch_stats* stats);

/* ------------------------------------------------------- host drop-ins */

/* _trigrid.edm_strategy (bindings/module.cpp:149-161): host points in, host
 * packed fp32 out (out must hold T(N) floats, or the shard's elements when
 * shard_count > 1).  The copy-out is pipelined against the kernel in
 * block-row pieces; pass pinned memory for full PCIe bandwidth. */
tg_status tg_edm_strategy_host(tg_strategy s, const float* pts, uint64_t n, uint32_t d,
                               uint32_t rho, float* out, const tg_launch_opts* opts,
                               tg_dispatch_stats* stats);

/* _trigrid.coverage_ok (bindings/module.cpp:163-172) / check_cell_coverage
 * (checks.cpp:16-38): 1 when every domain cell is touched exactly once
 * (no-diagonal domain for utm), computed with the COUNT kernel on device. */
tg_status tg_coverage_ok(tg_strategy s, uint64_t n, uint32_t rho, int device, int* ok);
/* Same with options: mode (AUTO = the kernel shape EDM/write launches use, SPAN checks the
 * owned-chunk rule of the span kernels, GRID the paper-faithful kernel), rec_m/rec_k, engine;
 * bad (may be NULL) = number of wrong cells, first_bad (may be NULL) = first wrong element. */
tg_status tg_coverage_ok_opts(tg_strategy s, uint64_t n, uint32_t rho, const tg_launch_opts* opts, int* ok,
                              uint64_t* bad, uint64_t* first_bad);

/* launch_count (engine.cpp:177-188) with the reference's HOST counter vector: counts (host
 * uint32[T(N)]) are incremented in place by the COUNT kernel on device. */
tg_status tg_count_host(tg_strategy s, uint64_t n, uint32_t rho, uint32_t* counts, const tg_launch_opts* opts,
                        tg_dispatch_stats* stats);

/* launch_dummy (engine.cpp:150-155) from the host: the dummy kernel on device, synchronous;
 * *sink_value = the device sink's value after the launch (the anti-DCE store never fires for
 * the default sentinel, so it stays as it was: 0). */
tg_status tg_dummy_host(tg_strategy s, uint64_t n, uint32_t rho, const tg_launch_opts* opts,
                        tg_dispatch_stats* stats, uint64_t* sink_value);

/* edm_reference (edm.cpp:53-63): the reference API's SEQUENTIAL oracle, i.e. host code by
 * contract (every pair j <= i in row-major order, binary32 edm_pair arithmetic, any d).  It is
 * what launch_edm results are verified against (run_suite, bench.cpp:80-108) -- never a
 * fallback for the device path. */
tg_status tg_edm_reference_host(const float* pts, uint64_t n, uint32_t d, float* out);

/* ltm_exactness_sweep (checks.cpp:81-95) generalised: on device, for every
 * lambda in [begin, end) compare the g(lambda) row (float guess only when
 * fixup == 0, guess + integer fix-up when fixup == 1) with isqrt(8L+1).
 * Outputs the mismatch count and the first mismatching lambda (UINT64_MAX). */
tg_status tg_lambda_sweep(int engine, int with_diag, int fixup, uint64_t begin, uint64_t end,
                          int device, uint64_t* mismatches, uint64_t* first);

/* Self-test of the kernel's fast correctly-rounded sqrt against __fsqrt_rn
 * over every binary32 bit pattern in [lo_bits, hi_bits). */
tg_status tg_sqrt_selftest(uint32_t lo_bits, uint32_t hi_bits, int device, uint64_t* mismatches);

/* gen_points (edm.cpp:38-51) on device: the first `count` values of the
 * splitmix64 stream from `seed` (N x d points = N*d values; the stream is
 * shape-invariant).  out: device float[count]. */
tg_status tg_gen_values(uint64_t count, uint64_t seed, float* out, const tg_launch_opts* opts);
/* _trigrid.gen_points (bindings/module.cpp:135-143): host float[n*d], with
 * the reference's checks (N in [1, 2^20], d in [1, 4]); generated on device. */
tg_status tg_gen_points_host(uint64_t n, uint32_t d, uint64_t seed, float* out, int device);

/* Number of kernels the last tg_* call on this thread launched. */
uint64_t tg_last_launch_count(void);

const char* tg_last_error(void);
int tg_api_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TRIGRID_B200_H_ */
