// tg_mapping.cuh -- block/thread mapping functions of the triangular domain,
// shared by host geometry code and the sm_100a kernels.
//
// Reference semantics (all citations /root/reference/proj/...):
//   tri_count            include/trigrid/tri.hpp:39-41
//   packed index         src/tri.cpp:17-21, src/engine.cpp:173,185
//   isqrt / ceil_sqrt    src/fastmath.cpp:8-21
//   fast_inv_sqrt        include/trigrid/fastmath.hpp:22-34
//   g(lambda) ltm_map    src/strategies.cpp:60-83 (+ repair fastmath.hpp:93-103)
//   bb_map               include/trigrid/strategies.hpp:94-97
//   utm_pair_unchecked   include/trigrid/strategies.hpp:128-166
//   rb_map               include/trigrid/strategies.hpp:182-193
//   rec_block_map        include/trigrid/strategies.hpp:214-220
//
// B200 design notes.  g(lambda) keeps the paper's float square-root row guess
// (sqrtf / 0x5f3759df Newton / MUFU rsqrt) but ALWAYS finishes with an exact
// 64-bit integer fix-up walk, so (i, j) is exact for every lambda instead of
// the reference's "exact below 1,844,160, repaired above" policy.  The
// fix-up is the same walk as repair_lower_row; for lambda < 2^40 it moves at
// most one row (proved exhaustively for lambda < 2^32 on device by
// tg_lambda_sweep, tests/test_gpu_sweep.py).
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define TG_HD __host__ __device__ __forceinline__
#else
#define TG_HD inline
#endif

#if defined(__CUDA_ARCH__)
#include <cuda_runtime.h>
#else
#include <cmath>
#include <cstring>
#endif

namespace tg {

// Square-root engines (SqrtVariant order, fastmath.hpp:41-46).
enum Engine : int { kNative = 0, kNewton = 1, kReciprocal = 2, kExact = 3 };

TG_HD uint64_t tri(uint64_t n) { return n * (n + 1) / 2; }                // with diagonal
TG_HD uint64_t tri_nd(uint64_t n) { return n * (n - (n > 0 ? 1 : 0)) / 2; }  // no diagonal
TG_HD uint64_t tri_count(uint64_t n, bool with_diag) { return with_diag ? tri(n) : tri_nd(n); }

// Exact floor sqrt of a 64-bit integer (double guess + integer fix-up).
TG_HD uint64_t isqrt(uint64_t v) {
    if (v == 0) return 0;
#if defined(__CUDA_ARCH__)
    uint64_t r = (uint64_t)__dsqrt_rn((double)v);
#else
    uint64_t r = (uint64_t)std::sqrt((double)v);
#endif
    while (r > 0 && (r > 0xffffffffull || r * r > v)) --r;
    while ((r + 1) <= 0xffffffffull && (r + 1) * (r + 1) <= v) ++r;
    return r;
}

TG_HD uint64_t ceil_sqrt(uint64_t v) {
    const uint64_t r = isqrt(v);
    return r * r == v ? r : r + 1;
}

TG_HD uint32_t f2u(float f) {
#if defined(__CUDA_ARCH__)
    return __float_as_uint(f);
#else
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
#endif
}
TG_HD float u2f(uint32_t u) {
#if defined(__CUDA_ARCH__)
    return __uint_as_float(u);
#else
    float f;
    std::memcpy(&f, &u, 4);
    return f;
#endif
}

// Explicitly rounded binary32 ops: never contracted into FMA, so the device
// reproduces the reference's SSE scalar arithmetic bit for bit.
TG_HD float fmul(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fmul_rn(a, b);
#else
    volatile float r = a * b;
    return r;
#endif
}
TG_HD float fadd(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fadd_rn(a, b);
#else
    volatile float r = a + b;
    return r;
#endif
}
TG_HD float fsub(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fsub_rn(a, b);
#else
    volatile float r = a - b;
    return r;
#endif
}
TG_HD float fsqrt(float a) {
#if defined(__CUDA_ARCH__)
    return __fsqrt_rn(a);
#else
    return std::sqrt(a);
#endif
}

// fastmath.hpp:22-34 -- same grouping y*(1.5f - half_x*(y*y)).
TG_HD float fast_inv_sqrt(float x, int iterations) {
    uint32_t bits = f2u(x);
    bits = 0x5f3759dfu - (bits >> 1);
    float y = u2f(bits);
    const float half_x = fmul(0.5f, x);
    for (int k = 0; k < iterations; ++k) y = fmul(y, fsub(1.5f, fmul(half_x, fmul(y, y))));
    return y;
}

// The engine's binary32 sqrt.  kReciprocal is the device rsqrt (MUFU.RSQ) on
// the GPU -- the paper's LTM-R -- and the reference's 1/sqrt stand-in
// (fastmath.hpp:39) on the host.
TG_HD float engine_sqrt(int engine, float xf) {
    switch (engine) {
        case kNative: return fsqrt(xf);
        case kNewton: return fmul(xf, fast_inv_sqrt(xf, 3));
        default:
#if defined(__CUDA_ARCH__)
        {
            // MUFU.RSQ directly: every argument here is >= 0.25 (g(lambda))
            // or >= 1 (utm discriminant), so rsqrtf's denormal rescaling is
            // dead code and this is bit-identical to rsqrtf.
            float y;
            asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(xf));
            return fmul(xf, y);
        }
#else
            return fmul(xf, 1.0f / std::sqrt(xf));
#endif
    }
}

TG_HD float engine_epsilon(int engine) {
    return (engine == kNewton || engine == kReciprocal) ? 1e-4f : 0.0f;  // fastmath.hpp:50
}

// Row start of the lower-triangular domain.
TG_HD uint64_t row_start(uint64_t r, bool with_diag) {
    return with_diag ? r * (r + 1) / 2 : r * (r - 1) / 2;
}

// The integer fix-up (repair_lower_row, fastmath.hpp:93-103).
TG_HD uint64_t fix_row(uint64_t i, uint64_t lambda, bool with_diag) {
    const uint64_t min_row = with_diag ? 0 : 1;
    if (i < min_row) i = min_row;
    while (i > min_row && row_start(i, with_diag) > lambda) --i;
    while (row_start(i + 1, with_diag) <= lambda) ++i;
    return i;
}

// Float row guess of g(lambda) before any fix-up (strategies.cpp:69-77).
TG_HD uint64_t ltm_row_guess(uint64_t lambda, int engine, bool with_diag) {
    if (engine == kExact) {
        const uint64_t root = isqrt(8 * lambda + 1);
        return with_diag ? (root - 1) / 2 : (root + 1) / 2;
    }
    const float xf = (float)(0.25 + 2.0 * (double)lambda);
    const float s = engine_sqrt(engine, xf);
    const float arg = fadd(with_diag ? fsub(s, 0.5f) : fadd(s, 0.5f), engine_epsilon(engine));
#if defined(__CUDA_ARCH__)
    long long row = (long long)floorf(arg);
#else
    long long row = (long long)std::floor(arg);
#endif
    return row < 0 ? 0 : (uint64_t)row;
}

// g(lambda): exact (i, j) for every lambda (float guess + integer fix-up).
struct Coord {
    uint64_t i, j;
};
TG_HD Coord ltm_map(uint64_t lambda, int engine, bool with_diag) {
    const uint64_t i = fix_row(ltm_row_guess(lambda, engine, with_diag), lambda, with_diag);
    return {i, lambda - row_start(i, with_diag)};
}

// Upper-triangular pair (a, b), 0-based, a < b (strategies.hpp:128-166).
// disc_base = (2N-1)^2.
TG_HD Coord utm_pair(uint64_t k, uint64_t n, uint64_t disc_base, int engine) {
    const uint64_t disc = disc_base - 8 * k;
    float s;
    if (engine == kExact) s = (float)isqrt(disc);
    else s = engine_sqrt(engine, (float)disc);
    long long a = (long long)(((double)(2 * n + 1) - (double)s) * 0.5);
    if (a < 1) a = 1;
    if (a > (long long)n - 1) a = (long long)n - 1;
    uint64_t ua = (uint64_t)a;
#define TG_ROW_OFF(r) (((r) - 1) * (2 * n - (r)) / 2)
    while (ua > 1 && TG_ROW_OFF(ua) > k) --ua;
    while (ua < n - 1 && TG_ROW_OFF(ua + 1) <= k) ++ua;
    const uint64_t b = (ua + 1) + k - TG_ROW_OFF(ua);
#undef TG_ROW_OFF
    return {ua - 1, b - 1};
}

// Rectangular-box fold (strategies.hpp:182-193). Returns false on discard.
TG_HD bool rb_map(uint64_t tx, uint64_t ty, uint64_t n, Coord* c) {
    if (n % 2 == 0) {
        if (tx >= n / 2 || ty >= n + 1) return false;
        if (tx + 1 <= ty) { *c = {ty - 1, tx}; return true; }
        *c = {n - ty - 1, n - tx - 1};
        return true;
    }
    if (tx >= (n + 1) / 2 || ty >= n) return false;
    if (tx <= ty) { *c = {ty, tx}; return true; }
    *c = {n - ty - 1, n - tx};
    return true;
}

// Largest-k decomposition N = m 2^k, m a multiple of rho (strategies.cpp:142-151).
TG_HD bool rec_decompose(uint64_t n, uint32_t rho, uint64_t* m, uint32_t* k) {
    bool found = false;
    for (uint32_t kk = 1; kk <= 40 && (1ull << kk) <= n; ++kk) {
        if (n % (1ull << kk) != 0) continue;
        const uint64_t mm = n >> kk;
        if (mm % rho == 0) { *m = mm; *k = kk; found = true; }
    }
    return found;
}

}  // namespace tg
