// tg_gram.cuh -- Gram-trick packed EDM on the 5th-generation tensor cores
// (tcgen05, TMEM), the optional large-d path of the north star
// (N=65536, d=64).
//
//   d^2(i, j) = |x_i|^2 + |x_j|^2 - 2 <x_i, x_j>,   d = sqrt(max(d^2, 0)),  d(i, i) = 0
//
// <x_i, x_j> for a 128 x 128 tile of the triangle comes from tcgen05.mma
// kind::tf32 with fp32 accumulation in TMEM, in 3xTF32 form
// (a_hi b_hi + a_hi b_lo + a_lo b_hi, a_hi = a with the 13 low mantissa bits
// cleared, a_lo = a - a_hi exactly), which keeps the dot product close to
// fp32 accuracy.  The result is NOT bit-exact with the reference (different
// formula); the stated tolerance, tested in tests/test_gpu_gram.py, is
//   |d_gram^2 - d_exact^2| <= 2^-17 * (|x_i|^2 + |x_j|^2).
//
// Structure (one CTA of 256 threads per SM, persistent over a contiguous
// range of tiles so consecutive tiles share the row tile and reuse A):
//   1. stage A (tile rows) and B (tile columns) K-slices of 64 features as
//      hi/lo tf32 in shared memory, canonical K-major no-swizzle UMMA layout
//      (8-row x 16-byte core matrices; LBO = 128 B along K, SBO = 2048 B
//      along M/N), fence.proxy.async;
//   2. one thread issues 3 x 8 tcgen05.mma (M=128, N=128, K=8 each) into a
//      128-column TMEM accumulator, tcgen05.commit -> mbarrier;
//   3. the 8 warps read TMEM (tcgen05.ld 32x32b.x32: warp w owns lanes
//      32(w%4).. and columns 64(w/4)..), apply the norms / clamp / sqrt /
//      diagonal, stage the tile in shared memory, and write each packed row
//      segment with aligned STG.128 (scalar stores only at the two edges).
// Tiles are enumerated by g(lambda) over the 128-row tile triangle.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tg_mapping.cuh"

namespace tg {

constexpr int kGT = 128;           // tile rows / columns
constexpr int kGK = 64;            // K slice (features) per MMA pass
constexpr int kGThreads = 256;
constexpr uint32_t kGSlice = kGT * kGK * 4;    // bytes of one operand slice (32 KB)
constexpr uint32_t kGLBO = 128;                // bytes between core matrices along K
constexpr uint32_t kGSBO = (kGK / 4) * 128;    // bytes between 8-row groups (2048)
constexpr int kGOutLd = kGT + 4;               // staged output row stride (floats)
// shared memory: A_hi, A_lo, B_hi, B_lo (4 x 32 KB), out tile (128 x 132 x 4),
// norms (2 x 128 x 4), mbarrier + tmem address
constexpr uint32_t kGSmemOut = 4 * kGSlice;
constexpr uint32_t kGSmemNorm = kGSmemOut + kGT * kGOutLd * 4;
constexpr uint32_t kGSmemBar = kGSmemNorm + 2 * kGT * 4;
constexpr uint32_t kGSmemBytes = kGSmemBar + 64;

struct GramGeom {
    uint64_t n;
    uint32_t d;
    uint32_t nt;        // tile rows = ceil(n / 128)
    uint64_t t0, t1;    // tile-lambda range of this launch (shard)
    uint64_t per_cta;   // consecutive tiles per CTA
    uint64_t r0, r1;    // element rows of the output window (shard rows)
    uint64_t e_base, e_end;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of (row m, feature k) inside one K-major no-swizzle slice
__device__ __forceinline__ uint32_t umma_off(uint32_t m, uint32_t k) {
    return (m >> 3) * kGSBO + (k >> 2) * kGLBO + (m & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((kGLBO >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((kGSBO >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (sm100)
    // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
    return d;
}

// kind::tf32, fp32 accumulate, A/B K-major, M = 128, N = 128
constexpr uint32_t kGIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kGT >> 3) << 17) |
                             ((uint32_t)(kGT >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_c, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_c),
        "l"(da), "l"(db), "r"(kGIdesc), "r"(accum));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred done;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}\n" ::"r"(bar),
        "r"(phase));
}

template <int SPLIT>  // 0 = hi (tf32 truncation), 1 = lo residual
__device__ __forceinline__ float tf32_part(float a) {
    const float hi = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
    return SPLIT == 0 ? hi : __fsub_rn(a, hi);
}

// Stage rows [row0, row0+128) x features [k0, k0+64) (zero padded) as hi/lo.
__device__ __forceinline__ void gram_stage(const float* __restrict__ pts, uint64_t n, uint32_t d,
                                           uint64_t row0, uint32_t k0, uint8_t* s_hi, uint8_t* s_lo) {
    for (uint32_t v = threadIdx.x; v < kGT * (kGK / 4); v += kGThreads) {
        const uint32_t m = v / (kGK / 4), kq = v % (kGK / 4);
        const uint64_t row = row0 + m;
        const uint32_t kb = k0 + 4 * kq;
        float a[4];
        if (row < n && (d & 3) == 0 && kb + 4 <= d) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(pts + row * d + kb));
            a[0] = t.x;
            a[1] = t.y;
            a[2] = t.z;
            a[3] = t.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t k = kb + q;
                a[q] = (row < n && k < d) ? __ldg(pts + row * d + k) : 0.0f;
            }
        }
        const uint32_t off = umma_off(m, 4 * kq);
        *reinterpret_cast<float4*>(s_hi + off) =
            make_float4(tf32_part<0>(a[0]), tf32_part<0>(a[1]), tf32_part<0>(a[2]), tf32_part<0>(a[3]));
        *reinterpret_cast<float4*>(s_lo + off) =
            make_float4(tf32_part<1>(a[0]), tf32_part<1>(a[1]), tf32_part<1>(a[2]), tf32_part<1>(a[3]));
    }
}

__global__ void __launch_bounds__(kGThreads, 1)
    gram_edm_kernel(const __grid_constant__ GramGeom g, const float* __restrict__ pts,
                    const float* __restrict__ norms, float* __restrict__ out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* a_hi = smem;
    uint8_t* a_lo = smem + kGSlice;
    uint8_t* b_hi = smem + 2 * kGSlice;
    uint8_t* b_lo = smem + 3 * kGSlice;
    float* otile = reinterpret_cast<float*>(smem + kGSmemOut);
    float* nrm_i = reinterpret_cast<float*>(smem + kGSmemNorm);
    float* nrm_j = nrm_i + kGT;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kGSmemBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kGSmemBar + 16);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kGT));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    uint32_t phase = 0;

    const uint64_t tb = g.t0 + (uint64_t)blockIdx.x * g.per_cta;
    const uint64_t te = min(tb + g.per_cta, g.t1);
    uint64_t loaded_ti = ~0ull;
    for (uint64_t lam = tb; lam < te; ++lam) {
        const Coord c = ltm_map(lam, kReciprocal, true);  // g(lambda) over the tile triangle
        const uint64_t ri = c.i * kGT, rj = c.j * kGT;
        // ---- MMA over K slices
        for (uint32_t k0 = 0; k0 < g.d; k0 += kGK) {
            if (g.d > kGK || loaded_ti != c.i) gram_stage(pts, g.n, g.d, ri, k0, a_hi, a_lo);
            gram_stage(pts, g.n, g.d, rj, k0, b_hi, b_lo);
            asm volatile("fence.proxy.async.shared::cta;");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
                for (int s = 0; s < kGK / 8; ++s) {
                    const uint32_t ko = s * 2 * kGLBO;
                    const uint32_t acc0 = (k0 > 0 || s > 0) ? 1u : 0u;
                    mma_tf32(tmem, umma_desc(ah + ko), umma_desc(bh + ko), acc0);
                    mma_tf32(tmem, umma_desc(ah + ko), umma_desc(bl + ko), 1u);
                    mma_tf32(tmem, umma_desc(al + ko), umma_desc(bh + ko), 1u);
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(bar))
                             : "memory");
            }
            mbar_wait(smem_u32(bar), phase);
            phase ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;");
        }
        loaded_ti = c.i;
        // ---- epilogue: TMEM -> registers -> d -> shared tile
        if (threadIdx.x < kGT) {
            const uint64_t ra = ri + threadIdx.x, rb = rj + threadIdx.x;
            nrm_i[threadIdx.x] = ra < g.n ? __ldg(norms + ra) : 0.0f;
            nrm_j[threadIdx.x] = rb < g.n ? __ldg(norms + rb) : 0.0f;
        }
        __syncthreads();
        {
            const int q = warp & 3, h = warp >> 2;
            const int row = 32 * q + lane;
            const float ni = nrm_i[row];
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int col0 = 64 * h + 32 * cc;
                uint32_t v[32];
                const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)col0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
                      "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
                      "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    const int col = col0 + t;
                    const float gij = __uint_as_float(v[t]);
                    float d2 = fmaf(-2.0f, gij, ni + nrm_j[col]);
                    float dist = sqrtf(fmaxf(d2, 0.0f));
                    if (ri + row == rj + col) dist = 0.0f;
                    otile[row * kGOutLd + col] = dist;
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        // ---- aligned packed row writes: own cells [rj, min(rj + 128, i + 1)) of rows in the window
        for (int r = warp; r < kGT; r += kGThreads / 32) {
            const uint64_t i = ri + r;
            if (i >= g.n || i < g.r0 || i >= g.r1) continue;
            const uint64_t cend = min(rj + kGT, i + 1);
            if (cend <= rj) continue;
            const uint64_t e0 = i * (i + 1) / 2 + rj;
            const uint64_t e1 = e0 + (cend - rj);
            const uint64_t lo = max(e0, g.e_base), hi = min(e1, g.e_end);
            if (lo >= hi) continue;
            const uint64_t k0 = (lo - g.e_base) >> 2, k1 = (hi - g.e_base + 3) >> 2;
            for (uint64_t k = k0 + lane; k < k1; k += 32) {
                const uint64_t eg = 4 * k + g.e_base;
                const float* src = otile + r * kGOutLd + (int64_t)(eg - e0);
                if (eg >= lo && eg + 4 <= hi) {
                    reinterpret_cast<float4*>(out)[k] = make_float4(src[0], src[1], src[2], src[3]);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (eg + q >= lo && eg + q < hi) out[eg + q - g.e_base] = src[q];
                }
            }
        }
        __syncthreads();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kGT));
}

// |x_i|^2 in fp32 (sequential fma over the features)
__global__ void gram_norms_kernel(const float* __restrict__ pts, uint64_t n, uint32_t d, float* __restrict__ norms) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (uint32_t k = 0; k < d; ++k) {
            const float a = __ldg(pts + i * d + k);
            s = fmaf(a, a, s);
        }
        norms[i] = s;
    }
}

// ===================================================================== v2
//
// Pipelined, warp-specialised Gram EDM (d <= 128), the B200 path of config
// C4.  Differences from gram_edm_kernel above:
//
//  * Operands are split ONCE by gram_split_kernel into fp16 hi/lo pairs
//    (x * 2^s = hi + lo, s a global power of two putting max|x| in
//    [2^14, 2^15), so hi/lo stay in fp16's normal range and the pair carries
//    ~22 significant bits) and laid out in global memory in the canonical
//    K-major no-swizzle UMMA layout, so every operand stage is a contiguous
//    cp.async.bulk copy (no tensor map, no per-thread staging), and kind::f16
//    runs at twice the tf32 rate with half the L2 bytes.
//  * Row tile (MMA A, M = 128 = TMEM lanes) is stored ROW-PERMUTED: TMEM lane
//    quarter q holds the 32 tile rows r with T(r) = q (mod 4), so all rows a
//    warp reads from TMEM share one 16-byte alignment shift of their packed
//    row start T(i) + j.
//  * Column operand (MMA B) is N = 136 = 128 + 8 points: the tile plus the
//    first 8 points of the next column tile.  Each row of tile (i, j) then
//    OWNS the 32 aligned 16-byte chunks that start in its 128 columns (the
//    last one spills up to 3 columns into tile j + 1), so every store of an
//    interior tile is a full aligned STG.128 -- no partial chunks, no
//    scattered edge stores.  Rows of tile (i, 0) add the <= 3 elements before
//    their first owned chunk; diagonal / clipped tiles mask per element.
//  * Roles: warp 0 = bulk-copy producer (row tile resident while the tile row
//    stays, column operands through a ring of stages), warp 1 = MMA issuer (per
//    64-feature slice 3 x 4 tcgen05.mma M=128 N=136 K=16: hi*lo + lo*hi +
//    hi*hi), warps 2..17 = epilogue: TMEM lane quarter warp % 4, split into two
//    2-warp sync groups of 16 rows (TG_G2_SUB; tcgen05.ld 16x32bx2, each warp
//    64 of the 128 columns).  kG2Acc accumulators in TMEM let the MMAs run ahead.
//  * Epilogue per warp: tcgen05.ld (32 rows x 40 columns) -> release the
//    accumulator -> d = sqrt(max(|x_i|^2 + |x_j|^2 - 2 g, 0)) on the 32 owned
//    columns (warp-uniform compile-time selection of the shift) -> 8 chunks
//    per row to a per-warp shared buffer -> transposed read -> STG.128, each
//    warp store instruction 4 rows x 128 contiguous bytes.
#ifndef TG_G2_EPI
#define TG_G2_EPI 16  // epilogue warps (4 lane quarters x 4 or x 2)
#endif
constexpr int kG2EpiWarps = TG_G2_EPI;
constexpr int kG2Threads = 32 * (2 + kG2EpiWarps);
constexpr uint32_t kG2Slice = 32768;          // row-tile block of one 64-feature slice: hi | lo fp16
constexpr uint32_t kG2Half = 16384;
constexpr uint32_t kG2Group = 1024;           // 8 points x 64 features fp16
constexpr uint32_t kG2N = 136;                // MMA N: column tile + 8 points of the next
constexpr uint32_t kG2BHalf = 17 * kG2Group;  // 17 groups
constexpr uint32_t kG2Stage = 2 * kG2BHalf;   // column stage: hi | lo
constexpr uint32_t kG2LBO = 128;              // K-adjacent core matrices
constexpr uint32_t kG2SBO = 1024;             // M/N-adjacent 8-row groups (8 core matrices along K)
constexpr int kG2MaxNk = 2;                   // d <= 128
constexpr uint32_t kG2SmemMax = 232448;
constexpr uint32_t kG2Acc = 3;                // TMEM accumulators
constexpr uint32_t kG2AccStride = 144;        // TMEM columns per accumulator (>= kG2N)
constexpr uint32_t kG2TmemCols = 512;
constexpr int kG2QChunks = 33;                // quarter staging row stride in chunks (32 used, odd: no conflicts)
constexpr uint32_t kG2EpiBytes = 32 * kG2QChunks * 16 / (kG2EpiWarps / 4);  // per epilogue warp
constexpr uint32_t kG2NormSlots = 8;          // norm ring: [column norms 136 | pad | row norms 128] floats
constexpr uint32_t kG2NormSlot = 2 * (136 + 8 + 128) * 4;  // norms | per-point scale factors (wide range)
constexpr uint32_t kG2NormRowOff = (136 + 8) * 4;
constexpr uint32_t kG2FacOff = (136 + 8 + 128) * 4;
// kind::f16 (A, B fp16, K-major), fp32 accumulate, M = 128, N = 136
constexpr uint32_t kG2Idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((kG2N >> 3) << 17) |
                              ((uint32_t)(kGT >> 4) << 24);

#ifndef TG_G2_PROF
#define TG_G2_PROF 0
#endif
#if TG_G2_PROF
// A/B instrumentation: cycles spent in each wait (summed over CTAs)
// 0 prod:norm_empty 1 prod:a_empty 2 prod:b_empty 3 mma:a_full 4 mma:acc_empty 5 mma:b_full
// 6 epi:norm_full 7 epi:acc_full 8 epi:total 9 mma:total 10 prod:total
__device__ unsigned long long tg_g2_prof[16];
#define G2W(slot, call)                                      \
    do {                                                     \
        const long long _t0 = clock64();                     \
        call;                                                \
        prof[slot] += (unsigned long long)(clock64() - _t0); \
    } while (0)
#else
#define G2W(slot, call) call
#endif

struct Gram2Geom {
    uint64_t n;
    uint32_t nk;        // 64-feature slices
    uint32_t ring;      // column stages
    uint64_t t0, t1;    // tile-lambda range
    uint64_t per_cta;
    uint64_t r0, r1;    // element rows of the output window
    uint64_t e_base, e_end;
    uint64_t bslice;    // bytes of one slice of the column operand (hi or lo)
    uint32_t a_stream;  // 0: row tile resident (nk <= kG2MaxNk); 1: row slices ride the ring with the columns
    uint32_t stage;     // bytes of one ring stage
};

// ring stage: the column slice (hi | lo, 17 KB each), preceded by the row-tile
// slice (32 KB) when the row operand streams (d > 64 kG2MaxNk)
__host__ __device__ __forceinline__ uint32_t g2_stage_bytes(bool a_stream) {
    return a_stream ? kG2Slice + kG2Stage : kG2Stage;
}

__host__ __device__ __forceinline__ uint32_t g2_smem_bytes(uint32_t nk, uint32_t ring, bool a_stream = false) {
    return (a_stream ? 0u : nk * kG2Slice) + ring * g2_stage_bytes(a_stream) + kG2EpiWarps * kG2EpiBytes +
           kG2NormSlots * kG2NormSlot +
           8 * (2 + 2 * kG2Acc + 2 * ring + 2 * kG2NormSlots) + 16;
}

// tile row of TMEM lane p (row-tile permutation); quarter q holds T(r) = q mod 4
__host__ __device__ __forceinline__ uint32_t g2_perm(uint32_t p) {
    // residues rho (r mod 8) with T(rho) mod 4 = q: q0 {0,7} q1 {1,6} q2 {3,4} q3 {2,5}
    const uint32_t q = p >> 5, l = p & 31;
    const uint32_t res = (0x52436170u >> (4 * (2 * q + (l & 1)))) & 0xF;
    return 8 * (l >> 1) + res;
}
// inverse: TMEM lane of tile row r
__host__ __device__ __forceinline__ uint32_t g2_perm_inv(uint32_t r) {
    // rho -> 2q + b : 0->0, 1->2, 2->6, 3->4, 4->5, 5->7, 6->3, 7->1
    const uint32_t qb = (0x13754620u >> (4 * (r & 7))) & 0xF;
    return 32 * (qb >> 1) + 2 * (r >> 3) + (qb & 1);
}

__device__ __forceinline__ uint32_t g2_off(uint32_t m, uint32_t k) {  // bytes in a 16 KB half
    return (m >> 3) * kG2SBO + (k >> 3) * kG2LBO + (m & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ uint64_t g2_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((kG2LBO >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((kG2SBO >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ void g2_mma(uint32_t tmem_c, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_c),
        "l"(da), "l"(db), "r"(kG2Idesc), "r"(accum));
}

__device__ __forceinline__ void g2_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void g2_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
#ifndef TG_G2_L2
#define TG_G2_L2 1  // operands bulk-loaded with an L2 evict_last policy, packed output stored .cs (evict first):
                    // DRAM reads 778 -> 57 MB per launch at N=65536 d=64, 1.967 -> 1.927 ms (0: both default)
#endif
// one bulk global -> shared copy completing on `bar`; pol = an L2 cache
// policy (TG_G2_L2) or ignored
__device__ __forceinline__ void g2_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
#if TG_G2_L2
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
#else
    (void)pol;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
#endif
}

__device__ __forceinline__ void g2_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void g2_bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                             uint64_t pol = 0) {
    g2_expect(bar, bytes);
    g2_copy(dst, src, bytes, bar, pol);
}

// next tile of the g(lambda) order: (i, j) -> (i, j + 1), row end -> (i + 1, 0)
__device__ __forceinline__ void g2_next(Coord& c) {
    if (c.j == c.i) {
        ++c.i;
        c.j = 0;
    } else {
        ++c.j;
    }
}

// mbarrier wait with a suspend-time hint: a waiting warp sleeps instead of
// spinning on the issue slots the epilogue warps need.  A wait that lasts
// ~2^34 cycles (seconds) is a pipeline bug: trap instead of hanging the GPU.
__device__ __forceinline__ void g2_wait_sleep(uint32_t bar, uint32_t phase) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase), "r"(0x100000)
        : "memory");
    if (done) return;
    const long long t0 = clock64();
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase), "r"(0x100000)
            : "memory");
        if (!done && clock64() - t0 > (1ll << 34)) __trap();
    } while (!done);
}

__device__ __forceinline__ void g2_ld32(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// Pass 1: |x_i|^2 (fp32 sequential fma, 0 for padding rows), the point's
// max |x| (pmax, binary32 bits) and over all points bits[0] = max |x|,
// bits[1] = ~(smallest nonzero per-point max |x|) (atomicMax of the complement).
__global__ void gram_prep_kernel(const float* __restrict__ pts, uint64_t n, uint64_t n_pad, uint32_t d,
                                 float* __restrict__ norms, unsigned int* __restrict__ pmax,
                                 unsigned int* __restrict__ bits) {
    unsigned int mb = 0, mn = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad;
         i += (uint64_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        unsigned int pm = 0;
        if (i < n) {
            for (uint32_t k = 0; k < d; ++k) {
                const float a = __ldg(pts + i * d + k);
                s = fmaf(a, a, s);
                pm = max(pm, __float_as_uint(a) & 0x7fffffffu);
            }
        }
        norms[i] = s;
        pmax[i] = pm;
        mb = max(mb, pm);
        if (pm) mn = max(mn, ~pm);
    }
    for (int o = 16; o; o >>= 1) {
        mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
        mn = max(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (mb) atomicMax(bits, mb);
        if (mn) atomicMax(bits + 1, mn);
    }
}

// power-of-two exponent s with max|x| * 2^s in [2^14, 2^15), clamped to
// [-63, 63] so that the unscale factor -2 * 2^-2s is a normal float
__device__ __forceinline__ int g2_scale_exp(unsigned int maxbits) {
    if (maxbits == 0 || maxbits >= 0x7f800000u) return 0;
    const int e = (int)(maxbits >> 23) - 127;  // floor(log2(max)) for normals
    return max(-63, min(63, 14 - e));
}

// Wide dynamic range: one global scale puts max|x| at 2^14; a
// point whose own max|x| is 2^20 x smaller has its hi/lo pair near fp16's
// subnormal floor and the tolerance no longer holds for its pairs (CPU
// emulation: err/bound 0.2 at a 1e7 magnitude ratio, 2.6 at 1e8).  Beyond a
// 2^20 spread of per-point max|x| every point gets its own power-of-two scale
// s_i (same [2^14, 2^15) placement) and the epilogue unscales each product by
// 2^-s_i 2^-s_j (row factor per lane, column factors through the norm ring).
__device__ __forceinline__ bool g2_wide_range(const unsigned int* bits) {
    const unsigned int mx = __ldg(bits), mn = ~__ldg(bits + 1);
    if (mx == 0 || __ldg(bits + 1) == 0) return false;
    return (int)(mx >> 23) - (int)(mn >> 23) > 20;
}

// Pass 2: x * 2^s = hi + lo in fp16, in the UMMA layout (8-point x 16-byte
// core matrices, K-major).  Row-tile operand opA: block (tile t, slice k) at
// (t * nk + k) * 32 KB (hi | lo), points permuted by g2_perm_inv.  Column
// operand opB: per slice, all points in natural order as 1 KB 8-point groups
// (hi array, then lo array, g.bslice bytes each, one zero group past the last
// tile).  One thread per (point, 8-feature group); padding is zero.
__global__ void gram_split_kernel(const float* __restrict__ pts, uint64_t n, uint64_t n_pad, uint32_t d,
                                  uint32_t nk, const unsigned int* __restrict__ bits,
                                  const unsigned int* __restrict__ pmax, float* __restrict__ facs,
                                  uint8_t* __restrict__ opA, uint8_t* __restrict__ opB, uint64_t bslice) {
    const bool wide = g2_wide_range(bits);
    const int sg = g2_scale_exp(__ldg(bits));
    const float scg = exp2f((float)sg);
    const uint32_t groups = nk * 8;
    const uint64_t total = (n_pad + 8) * groups;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t row = v / groups;
        const uint32_t g = (uint32_t)(v % groups);
        const uint32_t k0 = 8 * g;
        float sc = scg;
        if (wide) {  // per-point scale, its unscale factor 2^-s_i for the epilogue
            const int si = g2_scale_exp(__ldg(pmax + row));
            sc = exp2f((float)si);
            if (g == 0) facs[row] = exp2f((float)-si);
        }
        __half hi[8], lo[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const uint32_t k = k0 + t;
            const float x = (row < n && k < d) ? __fmul_rn(__ldg(pts + row * d + k), sc) : 0.0f;
            hi[t] = __float2half_rn(x);
            lo[t] = __float2half_rn(__fsub_rn(x, __half2float(hi[t])));
        }
        const uint4 vh = *reinterpret_cast<const uint4*>(hi), vl = *reinterpret_cast<const uint4*>(lo);
        const uint32_t slice = g / 8, kk = (g % 8) * 8;
        uint8_t* b = opB + slice * 2 * bslice + (row >> 3) * kG2Group + (kk >> 3) * kG2LBO + (row & 7) * 16;
        *reinterpret_cast<uint4*>(b) = vh;
        *reinterpret_cast<uint4*>(b + bslice) = vl;
        if (row < n_pad) {
            const uint64_t t = row / kGT;
            uint8_t* blk = opA + (t * nk + slice) * (uint64_t)kG2Slice + g2_off(g2_perm_inv((uint32_t)(row % kGT)), kk);
            *reinterpret_cast<uint4*>(blk) = vh;
            *reinterpret_cast<uint4*>(blk + kG2Half) = vl;
        }
    }
}

__device__ __forceinline__ void g2_ld4(uint32_t taddr, uint32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}

__device__ __forceinline__ void g2_ld8(uint32_t taddr, uint32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

#ifndef TG_G2_SQRT
#define TG_G2_SQRT 0  // epilogue sqrt: 0 MUFU.SQRT, 1 FMA-pipe (magic seed + 2 steps), 2 half and half
#endif

// sqrt of two non-negative floats on the FMA pipe (no MUFU, i.e. no MIO
// slot): inverse-sqrt seed 0x5F1FFFF9 - (bits >> 1) with the one-step
// correction of Moroz et al. (max rel. error 6.5e-4), one Newton step, then
// x * y.  x = 0 gives 0 (finite seed).  Max relative error of d 7.7e-7
// (2^-20.3, binary32 emulation over all exponents), i.e. <= 2^-18.3
// (|x_i|^2 + |x_j|^2) on d^2 -- inside the stated Gram tolerance together
// with the split error (measured <= 0.11 of it).
__device__ __forceinline__ float2 g2_sqrt2_fma(float2 x) {
    float2 y = make_float2(__uint_as_float(0x5F1FFFF9u - (__float_as_uint(x.x) >> 1)),
                           __uint_as_float(0x5F1FFFF9u - (__float_as_uint(x.y) >> 1)));
    float2 t = __fmul2_rn(__fmul2_rn(x, y), y);
    t = __ffma2_rn(t, make_float2(-0.703952253f, -0.703952253f), make_float2(1.681914091f, 1.681914091f));
    y = __fmul2_rn(y, t);
    const float2 xy = __fmul2_rn(x, y);
    t = __ffma2_rn(__fmul2_rn(xy, y), make_float2(-0.5f, -0.5f), make_float2(1.5f, 1.5f));
    return __fmul2_rn(xy, t);
}

// d for the 32 owned columns S .. S+31 of the loaded 40 (S = warp-uniform
// shift): d^2 = |x_i|^2 + |x_j|^2 - 2 * 2^-2s * acc, clamped at 0, sqrt.approx.
// nb4 = the 16-byte aligned column norms of loaded columns 0 .. 39 (broadcast).
// WIDE: per-point scales -- acc is first multiplied by the column factors
// 2^-s_j (cb4, same layout as nb4) and m2 = -2 * 2^-s_i is the row's.
template <int S, int SV = S, bool WIDE = false>
__device__ __forceinline__ void g2_epi(const uint32_t* v, const float4* nb4, const float4* cb4, float ni, float m2,
                                       float* dv) {
    const float2 m22 = make_float2(m2, m2), ni2 = make_float2(ni, ni);
    float4 lo = nb4[0], clo = make_float4(0.f, 0.f, 0.f, 0.f);
    if (WIDE) clo = cb4[0];
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4) {
        const float4 hi = nb4[c4 + 1];
        const float w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};  // columns 4 c4 .. 4 c4 + 7
        float4 chi = make_float4(0.f, 0.f, 0.f, 0.f);
        if (WIDE) chi = cb4[c4 + 1];
        const float cw[8] = {clo.x, clo.y, clo.z, clo.w, chi.x, chi.y, chi.z, chi.w};
#pragma unroll
        for (int t = 0; t < 4; t += 2) {
            const int p = 4 * c4 + t;
            float2 acc = make_float2(__uint_as_float(v[SV + p]), __uint_as_float(v[SV + p + 1]));
            if (WIDE) acc = __fmul2_rn(acc, make_float2(cw[S + t], cw[S + t + 1]));
            const float2 nn = __fadd2_rn(ni2, make_float2(w[S + t], w[S + t + 1]));
            const float2 d2 = __ffma2_rn(acc, m22, nn);
            float d0, d1;
            if (TG_G2_SQRT == 1 || (TG_G2_SQRT == 2 && (t & 2))) {
                const float2 r = g2_sqrt2_fma(make_float2(fmaxf(d2.x, 0.0f), fmaxf(d2.y, 0.0f)));
                d0 = r.x;
                d1 = r.y;
            } else {
                // sqrt(|d^2|): a rounding-negative d^2 (true value >= 0) gives
                // ||c| - e| <= |c - e|, so the stated d^2 tolerance still holds and the
                // clamp folds into MUFU's |x| operand modifier (no FMNMX per cell)
                asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d0) : "f"(fabsf(d2.x)));
                asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d1) : "f"(fabsf(d2.y)));
            }
            dv[p] = d0;
            dv[p + 1] = d1;
        }
        lo = hi;
        if (WIDE) clo = chi;
    }
}

#ifndef TG_G2_SUB
#define TG_G2_SUB 1  // epilogue sync groups (A/B: 1.87-1.89 vs 1.89-1.92 ms): 1 = two 2-warp groups per lane quarter (16 rows,
                     // tcgen05.ld 16x32bx2), 0 = one 4-warp group per quarter (32 rows, 32x32b)
#endif
#ifndef TG_G2_CS
#define TG_G2_CS 1  // interior row stores .cs (evict-first); 0: default caching (A/B: 1.89 vs 1.87 ms)
#endif
#ifndef TG_G2_ROWPTR
#define TG_G2_ROWPTR 0  // store-path row pointer cached per tile row (A/B: 1.86 vs 1.83 ms; 0 recomputes per tile)
#endif
#if TG_G2_ROWPTR && !TG_G2_L2
#error "TG_G2_ROWPTR assumes the .cs stores of TG_G2_L2"
#endif
#ifndef TG_G2_BULK
#define TG_G2_BULK 0  // 1: non-masked tiles leave through 512-byte cp.async.bulk row stores (A/B: 1.95 vs 1.84 ms)
#endif
#if TG_G2_SUB
static_assert(kG2EpiWarps == 16, "sub-group epilogue: 4 warps per lane quarter");
// named barrier of the 2 epilogue warps of sub-group g (ids 1..8): 16 TMEM lanes
__device__ __forceinline__ void g2_bar_quarter(uint32_t g) {
    asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "n"(64) : "memory");
}
#else
// named barrier of the 4 epilogue warps of TMEM lane quarter q (ids 1..4)
__device__ __forceinline__ void g2_bar_quarter(uint32_t q) {
    asm volatile("bar.sync %0, %1;" ::"r"(q + 1), "n"(32 * (kG2EpiWarps / 4)) : "memory");
}
#endif

// 16 TMEM lanes x 2 column halves: thread t < 16 reads lane base + t, columns
// c .. c + N - 1; thread t >= 16 lane base + t - 16, columns c + 32 ..
__device__ __forceinline__ void g2_ld32x2(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], 32;"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void g2_ld4x2(uint32_t taddr, uint32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], 32;"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}

__device__ __forceinline__ float g2_dist(uint32_t accbits, float ni, float nj, float m2, float cj = 1.0f) {
    float dd;
    const float acc = __fmul_rn(__uint_as_float(accbits), cj);
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(dd) : "f"(fmaxf(fmaf(acc, m2, __fadd_rn(ni, nj)), 0.0f)));
    return dd;
}

__global__ void __launch_bounds__(kG2Threads, 1)  // 96 registers: 5 warps x 96 x 32 fit one SMSP's 16 K
    gram2_edm_kernel(const __grid_constant__ Gram2Geom g, const uint8_t* __restrict__ opA,
                     const uint8_t* __restrict__ opB, const float* __restrict__ norms,
                     const float* __restrict__ facs, const unsigned int* __restrict__ bits,
                     float* __restrict__ out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t nk = g.nk, R = g.ring;
    const bool as = g.a_stream != 0;
    const bool wide = g2_wide_range(bits);  // per-point scales (uniform across the grid)
    uint8_t* sA = smem;                                   // resident row tile: nk x 32 KB (MMA A)
    uint8_t* sB = smem + (as ? 0u : nk * kG2Slice);       // ring: R x ([row slice 32 KB] | col hi | col lo)
    const uint32_t SB = g.stage;
    const uint32_t boff = as ? kG2Slice : 0u;             // column slice offset inside a stage
    uint8_t* sE = sB + R * SB;                            // kG2EpiWarps x kG2EpiBytes
    uint8_t* sN = sE + kG2EpiWarps * kG2EpiBytes;         // norm ring
    uint64_t* bars = reinterpret_cast<uint64_t*>(sN + kG2NormSlots * kG2NormSlot);
    // barrier slots: 0 a_full, 1 a_empty, acc_full[kG2Acc], acc_empty[kG2Acc], n_full[NS], n_empty[NS],
    // b_full[R], b_empty[R]
    constexpr uint32_t AF = 2, AE = 2 + kG2Acc, NF = 2 + 2 * kG2Acc, NE = NF + kG2NormSlots,
                       BF = NE + kG2NormSlots;
    const uint32_t BE = BF + R;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + BF + 2 * R);
    const uint32_t bar0 = smem_u32(bars);
    auto BAR = [&](uint32_t k) { return bar0 + 8 * k; };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if TG_G2_PROF
    unsigned long long prof[16] = {};
    const long long tstart = clock64();
#endif

    if (threadIdx.x == 0) {
        mbar_init(BAR(0), 1);
        mbar_init(BAR(1), 1);
        for (uint32_t b = 0; b < kG2Acc; ++b) {
            mbar_init(BAR(AF + b), 1);
            mbar_init(BAR(AE + b), kG2EpiWarps);
        }
        for (uint32_t b = 0; b < kG2NormSlots; ++b) {
            mbar_init(BAR(NF + b), 1);
            mbar_init(BAR(NE + b), kG2EpiWarps);
        }
        for (uint32_t s = 0; s < 2 * R; ++s) mbar_init(BAR(BF + s), 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kG2TmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    const uint64_t tb = g.t0 + (uint64_t)blockIdx.x * g.per_cta;
    const uint64_t te = min(tb + g.per_cta, g.t1);

    if (warp == 0) {
        // ------------------------------------------------------- producer
        if (lane == 0 && tb < te) {
            uint64_t pol = 0;
#if TG_G2_L2
            // the split operands (17 MB at N = 65536, d = 64) are re-read by every CTA
            // sweeping its tile rows; keep them in L2 against the 8.6 GB output stream
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
            Coord c = ltm_map(tb, kReciprocal, true);  // g(lambda) over the tile triangle
            uint64_t cur = ~0ull;
            uint32_t na = 0, q = 0, it = 0;
            for (uint64_t lam = tb; lam < te; ++lam, ++it, g2_next(c)) {
                {  // norms of the tile: 136 column norms (tile + 8 spill points), 128 row norms
                    const uint32_t ns = it % kG2NormSlots, bar = BAR(NF + ns);
                    G2W(0, g2_wait_sleep(BAR(NE + ns), ((it / kG2NormSlots) & 1) ^ 1));
                    const uint32_t dst = smem_u32(sN + ns * kG2NormSlot);
                    g2_expect(bar, (wide ? 2 : 1) * (136 * 4 + 128 * 4));
                    g2_copy(dst, norms + c.j * kGT, 136 * 4, bar, pol);
                    g2_copy(dst + kG2NormRowOff, norms + c.i * kGT, 128 * 4, bar, pol);
                    if (wide) {
                        g2_copy(dst + kG2FacOff, facs + c.j * kGT, 136 * 4, bar, pol);
                        g2_copy(dst + kG2FacOff + kG2NormRowOff, facs + c.i * kGT, 128 * 4, bar, pol);
                    }
                }
                if (!as && c.i != cur) {
                    if (na > 0) G2W(1, g2_wait_sleep(BAR(1), (na - 1) & 1));  // MMAs done with the old row tile
                    g2_bulk_load(smem_u32(sA), opA + c.i * nk * (uint64_t)kG2Slice, nk * kG2Slice, BAR(0), pol);
                    cur = c.i;
                    ++na;
                }
                for (uint32_t k = 0; k < nk; ++k, ++q) {
                    const uint32_t s = q % R, round = q / R;
                    G2W(2, g2_wait_sleep(BAR(BE + s), (round & 1) ^ 1));
                    const uint8_t* src = opB + k * 2 * g.bslice + c.j * 16 * (uint64_t)kG2Group;
                    const uint32_t dst = smem_u32(sB + s * SB) + boff, bar = BAR(BF + s);
                    g2_expect(bar, SB);
                    if (as)  // the row tile's slice k rides along
                        g2_copy(dst - kG2Slice, opA + (c.i * nk + k) * (uint64_t)kG2Slice, kG2Slice, bar, pol);
                    g2_copy(dst, src, kG2BHalf, bar, pol);
                    g2_copy(dst + kG2BHalf, src + g.bslice, kG2BHalf, bar, pol);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA
        if (lane == 0 && tb < te) {
            Coord c = ltm_map(tb, kReciprocal, true);
            uint64_t cur = ~0ull;
            uint32_t na = 0, q = 0, it = 0;
            for (uint64_t lam = tb; lam < te; ++lam, ++it) {
                if (!as && c.i != cur) {
                    G2W(3, g2_wait_sleep(BAR(0), na & 1));
                    cur = c.i;
                    ++na;
                }
                const uint32_t buf = it % kG2Acc;
                G2W(4, g2_wait_sleep(BAR(AE + buf), ((it / kG2Acc) & 1) ^ 1));  // epilogue drained this accumulator
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t dtm = tmem + buf * kG2AccStride;
                for (uint32_t k = 0; k < nk; ++k, ++q) {
                    const uint32_t s = q % R, round = q / R;
                    G2W(5, g2_wait_sleep(BAR(BF + s), round & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t ah = as ? smem_u32(sB + s * SB) : smem_u32(sA + k * kG2Slice), al = ah + kG2Half;
                    const uint32_t bh = smem_u32(sB + s * SB) + boff, bl = bh + kG2BHalf;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t ko = kk * 2 * kG2LBO;  // K = 16 fp16 = 2 core matrices
                        g2_mma(dtm, g2_desc(ah + ko), g2_desc(bl + ko), (k > 0 || kk > 0) ? 1u : 0u);
                        g2_mma(dtm, g2_desc(al + ko), g2_desc(bh + ko), 1u);
                        g2_mma(dtm, g2_desc(ah + ko), g2_desc(bh + ko), 1u);
                    }
                    g2_commit(BAR(BE + s));  // stage s free once these MMAs complete
                }
                g2_commit(BAR(AF + buf));  // accumulator ready
                const uint64_t row = c.i;
                g2_next(c);
                if (!as && (lam + 1 >= te || c.i != row)) g2_commit(BAR(1));  // row tile free
            }
        }
    } else {
        // ------------------------------------------------------- epilogue
        // kG2EpiWarps warps: TMEM lane quarter q = warp % 4 (32 rows), EPW warps
        // per quarter, warp w4 owns WCOLS columns and stores WROWS row slots.
        constexpr int EPW = kG2EpiWarps / 4, WCOLS = 128 / EPW, WROWS = 32 / EPW, NH = WCOLS / 32;
        const uint32_t e = warp - 2, q = warp & 3, w4 = e >> 2;
        const uint32_t a = (q - (uint32_t)g.e_base) & 3u;  // (T(i) + j0 - e_base) mod 4, rows of quarter q
        const uint32_t s = (4u - a) & 3u;                    // first owned column of every row
        const int sh = g2_scale_exp(__ldg(bits));
        const float m2g = -2.0f * exp2f((float)(-2 * sh));
        // quarter staging tile: row slot r (= TMEM lane 32q + r) x 33 chunks (32 used)
#if TG_G2_SUB
        // sub-group sg = w4 / 2 of quarter q owns TMEM lanes 32 q + 16 sg + [0, 16) (16 rows x 128
        // columns, its own staging and named barrier, so the two sub-groups of a quarter -- which
        // share one SMSP -- drift out of phase instead of running MUFU / staging / stores in
        // lockstep); warp m = w4 % 2 of it loads columns 64 m + [0, 64): thread t the row of lane
        // t % 16, columns 64 m + 32 (t / 16) + [0, 32)
        const uint32_t sg = w4 >> 1, m = w4 & 1;
        const uint32_t cbase = 64 * m + 32 * (lane >> 4);
        const uint32_t bq = 2 * q + sg;  // barrier / staging group
        float4* qbuf = reinterpret_cast<float4*>(sE + bq * 2 * kG2EpiBytes) - 16 * sg * kG2QChunks;
        const uint32_t r_lane = g2_perm(32 * q + 16 * sg + (lane & 15));
        float4* my = qbuf + (16 * sg + (lane & 15)) * kG2QChunks + cbase / 4;
#else
        const uint32_t cbase = WCOLS * w4, bq = q;
        float4* qbuf = reinterpret_cast<float4*>(sE + q * EPW * kG2EpiBytes);
        const uint32_t r_lane = g2_perm(32 * q + lane);  // compute phase: lane = TMEM lane
        float4* my = qbuf + lane * kG2QChunks + (WCOLS / 4) * w4;
#endif
        float4* out4 = reinterpret_cast<float4*>(out);
        const uint32_t cw = cbase + s;  // first owned column of this thread, relative to the tile
        const uint32_t rb0 = g2_perm(32 * q), rb1 = g2_perm(32 * q + 1);  // tile rows of slots 0, 1 (+8 per 2 slots)

#if TG_G2_ROWPTR
        uint32_t prow_i = ~0u;  // tile row of the cached row-slot pointer
        float4* prow0 = out4;   // row slot 0 at column s of the tile row's column tile 0
        uint32_t pd1 = 0, rd0 = 0, rd1 = 0;  // slot 1 - slot 0 (chunks); rows x + 8: + 2x + 9 chunks
#endif
#if TG_G2_BULK
        uint64_t pol_ef;  // packed output: L2 evict-first
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_ef));
#endif
        Coord c = ltm_map(tb, kReciprocal, true);
        uint32_t it = 0;
        for (uint64_t lam = tb; lam < te; ++lam, ++it) {
            const uint64_t ri = c.i * kGT, rj = c.j * kGT;
            const uint32_t buf = it % kG2Acc;
            const uint32_t ns = it % kG2NormSlots;
            const float* nslot = reinterpret_cast<const float*>(sN + ns * kG2NormSlot);
            G2W(6, g2_wait_sleep(BAR(NF + ns), (it / kG2NormSlots) & 1));
            const float ni = nslot[kG2NormRowOff / 4 + r_lane];
            const float4* nb4 = reinterpret_cast<const float4*>(nslot + cbase);  // norms of loaded columns
            const float4* cb4 = reinterpret_cast<const float4*>(nslot + kG2FacOff / 4 + cbase);  // their 2^-s_j
            const float m2 = wide ? -2.0f * nslot[(kG2FacOff + kG2NormRowOff) / 4 + r_lane] : m2g;
            G2W(7, g2_wait_sleep(BAR(AF + buf), (it / kG2Acc) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint32_t v[WCOLS + 4];
#if TG_G2_SUB
            const bool head = c.j == 0 && m == 0 && s > 0;  // warp-uniform: columns [0, s) of tile (i, 0)
            const uint32_t taddr = tmem + ((32 * q + 16 * sg) << 16) + buf * kG2AccStride + 64 * m;
            g2_ld32x2(taddr + s, v);
            if (head) g2_ld4x2(taddr, v + WCOLS);  // head columns 0..3 (threads t < 16)
#else
            const bool head = c.j == 0 && w4 == 0 && s > 0;  // warp-uniform: columns [0, s) of tile (i, 0)
            const uint32_t taddr = tmem + ((32 * q) << 16) + buf * kG2AccStride + WCOLS * w4;
            // owned columns s + WCOLS w4 + [0, WCOLS) (tcgen05.ld at the column offset)
#pragma unroll
            for (int h = 0; h < NH; ++h) g2_ld32(taddr + 32 * h + s, v + 32 * h);
            if (head) g2_ld4(taddr, v + WCOLS);  // head columns 0..3
#endif
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) g2_arrive(BAR(AE + buf));  // TMEM buffer may be overwritten

            const uint64_t i = ri + r_lane;
            // masked tiles: diagonal, its left neighbour (spill columns reach the
            // diagonal / the next row), rows past n or outside the window
            const bool special = c.i <= c.j + 1 || ri + kGT > g.n || ri < g.r0 || ri + kGT > g.r1;
            float dv[WCOLS];
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                if (!wide) {
                    switch (s) {
                        case 0: g2_epi<0, 0>(v + 32 * h, nb4 + 8 * h, cb4, ni, m2, dv + 32 * h); break;
                        case 1: g2_epi<1, 0>(v + 32 * h, nb4 + 8 * h, cb4, ni, m2, dv + 32 * h); break;
                        case 2: g2_epi<2, 0>(v + 32 * h, nb4 + 8 * h, cb4, ni, m2, dv + 32 * h); break;
                        default: g2_epi<3, 0>(v + 32 * h, nb4 + 8 * h, cb4, ni, m2, dv + 32 * h); break;
                    }
                } else {
                    switch (s) {
                        case 0: g2_epi<0, 0, true>(v + 32 * h, nb4 + 8 * h, cb4 + 8 * h, ni, m2, dv + 32 * h); break;
                        case 1: g2_epi<1, 0, true>(v + 32 * h, nb4 + 8 * h, cb4 + 8 * h, ni, m2, dv + 32 * h); break;
                        case 2: g2_epi<2, 0, true>(v + 32 * h, nb4 + 8 * h, cb4 + 8 * h, ni, m2, dv + 32 * h); break;
                        default: g2_epi<3, 0, true>(v + 32 * h, nb4 + 8 * h, cb4 + 8 * h, ni, m2, dv + 32 * h); break;
                    }
                }
            }
            float nh0 = 0.0f, nh1 = 0.0f, nh2 = 0.0f;  // column norms 0..2 (head cells)
            float ch[3] = {1.0f, 1.0f, 1.0f};         // and their factors (wide range)
            if (head) {
                nh0 = nslot[0];
                nh1 = nslot[1];
                nh2 = nslot[2];
                if (wide) {
                    ch[0] = nslot[kG2FacOff / 4];
                    ch[1] = nslot[kG2FacOff / 4 + 1];
                    ch[2] = nslot[kG2FacOff / 4 + 2];
                }
            }
            __syncwarp();
            if (lane == 0) g2_arrive(BAR(NE + ns));  // norm slot consumed
            if (special) {
#pragma unroll
                for (int p = 0; p < WCOLS; ++p)
                    if (rj + cw + p == i) dv[p] = 0.0f;
            }
            if (head && cbase == 0 && i < g.n && i >= g.r0 && i < g.r1) {
                float* rowp = out + (i * (i + 1) / 2 - g.e_base);
                const float nhv[3] = {nh0, nh1, nh2};
#pragma unroll
                for (uint32_t p = 0; p < 3; ++p)
                    if (p < s && p <= i) rowp[p] = (p == i) ? 0.0f : g2_dist(v[WCOLS + p], ni, nhv[p], m2, ch[p]);
            }
#if TG_G2_BULK
            // the bulk stores issued from this lane have finished reading the staging rows
            if (lane < WROWS) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
            g2_bar_quarter(bq);  // the group's previous tile is fully read
#pragma unroll
            for (int cc = 0; cc < WCOLS / 4; ++cc)
                my[cc] = make_float4(dv[4 * cc], dv[4 * cc + 1], dv[4 * cc + 2], dv[4 * cc + 3]);
#if TG_G2_BULK
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging visible to the bulk copies
#endif
            const Coord cn = c;
            g2_next(c);
            g2_bar_quarter(bq);  // the group's rows x 32 chunks are staged
            // warp w4 stores row slots WROWS w4 .. + WROWS, one 512-byte row segment per
            // instruction: slot 2 r2 + b (relative) is tile row 4 WROWS w4 + 8 r2 + rb_b
            const float4* src = qbuf + WROWS * w4 * kG2QChunks + lane;
#if TG_G2_BULK
            if (!special) {
                // lane r < WROWS: one 512-byte bulk copy (TMA engine) of row slot r, so the
                // staging read and the global store leave the LSU / MIO path
                if (lane < WROWS) {
                    const uint64_t x = ri + 4 * WROWS * w4 + 8 * (lane >> 1) + ((lane & 1) ? rb1 : rb0);
                    const float* dst = out + (x * (x + 1) / 2 + rj + s - g.e_base);
                    asm volatile(
                        "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], 512, %2;\n\t"
                        "cp.async.bulk.commit_group;" ::"l"(dst),
                        "r"(smem_u32(qbuf + (WROWS * w4 + lane) * kG2QChunks)), "l"(pol_ef)
                        : "memory");
                }
            } else if (false) {
#else
            if (!special) {
#endif
                // chunk index of (row x, column rj + s) is (T(x) + rj + s - e_base) / 4;
                // rows x + 8: + (8x + 36) / 4 = 2x + 9
#if TG_G2_ROWPTR
                // row-slot pointers and row offsets depend only on the tile row: recomputed when
                // it changes, moved by 32 chunks per column tile (T(x) + s - e_base = 0 mod 4)
                if ((uint32_t)cn.i != prow_i) {
                    prow_i = (uint32_t)cn.i;
                    const uint64_t x0 = ri + 4 * WROWS * w4 + rb0, x1 = ri + 4 * WROWS * w4 + rb1;
                    prow0 = out4 + ((x0 * (x0 + 1) / 2 + s - g.e_base) >> 2) + lane;
                    pd1 = (uint32_t)((x1 * (x1 + 1) / 2 - x0 * (x0 + 1) / 2) >> 2);  // x1 > x0, same shift
                    rd0 = 2 * (uint32_t)x0 + 9;
                    rd1 = 2 * (uint32_t)x1 + 9;
                }
                float4* p0 = prow0 + 32 * cn.j;
#pragma unroll
                for (int r2 = 0; r2 < WROWS / 2; ++r2) {
                    __stcs(p0 + (uint32_t)(r2 * rd0 + 8 * r2 * (r2 - 1)), src[(2 * r2) * kG2QChunks]);
                    __stcs(p0 + (uint32_t)(pd1 + r2 * rd1 + 8 * r2 * (r2 - 1)), src[(2 * r2 + 1) * kG2QChunks]);
                }
#else
                const uint64_t colb = rj + s - g.e_base;
                const uint64_t x0 = ri + 4 * WROWS * w4 + rb0, x1 = ri + 4 * WROWS * w4 + rb1;
                float4* p0 = out4 + ((x0 * (x0 + 1) / 2 + colb) >> 2) + lane;
                float4* p1 = out4 + ((x1 * (x1 + 1) / 2 + colb) >> 2) + lane;
                const uint32_t d0 = 2 * (uint32_t)x0 + 9, d1 = 2 * (uint32_t)x1 + 9;
#pragma unroll
                for (int r2 = 0; r2 < WROWS / 2; ++r2) {
#if TG_G2_L2 && TG_G2_CS
                    __stcs(p0 + (uint32_t)(r2 * d0 + 8 * r2 * (r2 - 1)), src[(2 * r2) * kG2QChunks]);
                    __stcs(p1 + (uint32_t)(r2 * d1 + 8 * r2 * (r2 - 1)), src[(2 * r2 + 1) * kG2QChunks]);
#else
                    p0[(uint32_t)(r2 * d0 + 8 * r2 * (r2 - 1))] = src[(2 * r2) * kG2QChunks];
                    p1[(uint32_t)(r2 * d1 + 8 * r2 * (r2 - 1))] = src[(2 * r2 + 1) * kG2QChunks];
#endif
                }
#endif
            } else {
                const uint64_t col0 = cn.j * kGT + s + 4 * lane;  // first column of this lane's chunk
#pragma unroll 1
                for (int r = 0; r < WROWS; ++r) {
                    const uint64_t ii = ri + 4 * WROWS * w4 + 8 * (r >> 1) + ((r & 1) ? rb1 : rb0);
                    if (ii >= g.n || ii < g.r0 || ii >= g.r1 || col0 > ii) continue;
                    const float4 val = src[r * kG2QChunks];
                    float* dst = out + (ii * (ii + 1) / 2 + col0 - g.e_base);
                    if (col0 + 3 <= ii) {
                        *reinterpret_cast<float4*>(dst) = val;
                    } else {
                        const float vals[4] = {val.x, val.y, val.z, val.w};
                        for (uint32_t u = 0; u < 4 && col0 + u <= ii; ++u) dst[u] = vals[u];
                    }
                }
            }
        }
#if TG_G2_BULK
        if (lane < WROWS) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
    }
#if TG_G2_PROF
    if (lane == 0 && (warp <= 2)) {
        prof[warp == 0 ? 10 : warp == 1 ? 9 : 8] = (unsigned long long)(clock64() - tstart);
        for (int k = 0; k < 16; ++k)
            if (prof[k]) atomicAdd(&tg_g2_prof[k], prof[k]);
    }
#endif
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kG2TmemCols));
    }
}

}  // namespace tg
