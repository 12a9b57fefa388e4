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
//    K-major no-swizzle UMMA layout, one 32 KB (hi 16 KB | lo 16 KB) block per
//    (128-row tile, 64-feature slice).  A tile's operand is therefore one
//    contiguous cp.async.bulk copy (no tensor map, no per-thread staging), and
//    kind::f16 runs at twice the tf32 rate with half the L2 bytes.
//  * The A copy (tile rows) is stored ROW-PERMUTED: TMEM lane quarter q holds
//    the 32 tile rows r with T(r) = q (mod 4).  The packed element T(i) + j of
//    every row a warp reads from TMEM then has the same 16-byte alignment
//    shift, so the realignment of a row segment onto aligned float4 chunks is a
//    warp-uniform compile-time register selection (no divergence).
//  * Roles: warp 0 = bulk-copy producer (A resident while the tile row stays,
//    B through a ring of 32 KB stages), warp 1 = MMA issuer (3 x 4
//    tcgen05.mma M=128 N=128 K=16 per 64-feature slice: hi*hi + hi*lo + lo*hi),
//    warps 2..9 = epilogue (lane quarter warp % 4, column half).  The fp32
//    accumulator is double-buffered in TMEM (2 x 128 columns), so the MMAs of
//    tile t+1 run under the epilogue / HBM stores of tile t.
//  * Epilogue per warp: 32 rows x 64 columns: tcgen05.ld -> release the TMEM
//    buffer -> d = sqrt(max(|x_i|^2 + |x_j|^2 - 2 g, 0)) -> realigned chunks
//    to a per-warp shared buffer (32 rows x 17 chunks, conflict-free) ->
//    transposed read -> STG.128 of every full 16-byte chunk, lanes on
//    consecutive chunks of a row (coalesced); scalar stores only for the two
//    partial chunks at the ends of each 64-column row segment.
constexpr int kG2Threads = 320;               // 10 warps
constexpr uint32_t kG2Slice = 32768;          // one (tile, 64-feature slice): hi | lo fp16
constexpr uint32_t kG2Half = 16384;
constexpr uint32_t kG2LBO = 128;              // K-adjacent core matrices
constexpr uint32_t kG2SBO = 1024;             // M-adjacent 8-row groups (8 core matrices along K)
constexpr int kG2Chunks = 17;                 // 16-byte chunks per staged 64-column row segment
constexpr uint32_t kG2EpiBytes = 32 * kG2Chunks * 16;  // per epilogue warp
constexpr int kG2MaxNk = 2;                   // d <= 128
// kind::f16 (A, B fp16, K-major), fp32 accumulate, M = 128, N = 128
constexpr uint32_t kG2Idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(kGT >> 3) << 17) |
                              ((uint32_t)(kGT >> 4) << 24);

struct Gram2Geom {
    uint64_t n;
    uint32_t nk;        // 64-feature slices
    uint32_t ring;      // B stages
    uint64_t t0, t1;    // tile-lambda range
    uint64_t per_cta;
    uint64_t r0, r1;    // element rows of the output window
    uint64_t e_base, e_end;
};

// tile row of TMEM lane p (A row permutation); quarter q holds T(r) = q mod 4
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
__device__ __forceinline__ void g2_bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// Pass 1: |x_i|^2 (fp32 sequential fma, 0 for padding rows) and max |x|.
__global__ void gram_prep_kernel(const float* __restrict__ pts, uint64_t n, uint64_t n_pad, uint32_t d,
                                 float* __restrict__ norms, unsigned int* __restrict__ maxbits) {
    unsigned int mb = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad;
         i += (uint64_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        if (i < n) {
            for (uint32_t k = 0; k < d; ++k) {
                const float a = __ldg(pts + i * d + k);
                s = fmaf(a, a, s);
                mb = max(mb, __float_as_uint(a) & 0x7fffffffu);
            }
        }
        norms[i] = s;
    }
    for (int o = 16; o; o >>= 1) mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
    if ((threadIdx.x & 31) == 0 && mb) atomicMax(maxbits, mb);
}

// power-of-two exponent s with max|x| * 2^s in [2^14, 2^15), clamped to
// [-63, 63] so that the unscale factor -2 * 2^-2s is a normal float
__device__ __forceinline__ int g2_scale_exp(unsigned int maxbits) {
    if (maxbits == 0 || maxbits >= 0x7f800000u) return 0;
    const int e = (int)(maxbits >> 23) - 127;  // floor(log2(max)) for normals
    return max(-63, min(63, 14 - e));
}

// Pass 2: x * 2^s = hi + lo in fp16, written to opA (row-permuted) and opB
// (natural) in the UMMA layout: block (tile t, slice k) at ((t * nk + k) * 32 KB),
// hi at +0, lo at +16 KB.  One thread per (row, 8-feature group).
__global__ void gram_split_kernel(const float* __restrict__ pts, uint64_t n, uint64_t n_pad, uint32_t d,
                                  uint32_t nk, const unsigned int* __restrict__ maxbits,
                                  uint8_t* __restrict__ opA, uint8_t* __restrict__ opB) {
    const float sc = exp2f((float)g2_scale_exp(__ldg(maxbits)));
    const uint32_t groups = nk * 8;
    const uint64_t total = n_pad * groups;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t row = v / groups;
        const uint32_t g = (uint32_t)(v % groups);
        const uint32_t k0 = 8 * g;
        __half hi[8], lo[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const uint32_t k = k0 + t;
            const float x = (row < n && k < d) ? __fmul_rn(__ldg(pts + row * d + k), sc) : 0.0f;
            hi[t] = __float2half_rn(x);
            lo[t] = __float2half_rn(__fsub_rn(x, __half2float(hi[t])));
        }
        const uint64_t t = row / kGT;
        const uint32_t r = (uint32_t)(row % kGT), slice = g / 8, kk = (g % 8) * 8;
        const uint64_t blk = (t * nk + slice) * (uint64_t)kG2Slice;
        const uint4 vh = *reinterpret_cast<const uint4*>(hi), vl = *reinterpret_cast<const uint4*>(lo);
        const uint32_t ob = g2_off(r, kk), oa = g2_off(g2_perm_inv(r), kk);
        *reinterpret_cast<uint4*>(opB + blk + ob) = vh;
        *reinterpret_cast<uint4*>(opB + blk + kG2Half + ob) = vl;
        *reinterpret_cast<uint4*>(opA + blk + oa) = vh;
        *reinterpret_cast<uint4*>(opA + blk + kG2Half + oa) = vl;
    }
}

// Realign 64 row values onto 17 aligned chunks (segment start at position A
// of chunk 0) and stage them: chunk c holds positions 4c - A + [0, 4).
template <int A>
__device__ __forceinline__ void g2_stage_row(const float* v, float4* row_buf) {
#pragma unroll
    for (int c = 0; c < kG2Chunks; ++c) {
        float e[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int p = 4 * c - A + t;
            e[t] = (p >= 0 && p < 64) ? v[p] : 0.0f;
        }
        row_buf[c] = make_float4(e[0], e[1], e[2], e[3]);
    }
}

__global__ void __launch_bounds__(kG2Threads, 1)
    gram2_edm_kernel(const __grid_constant__ Gram2Geom g, const uint8_t* __restrict__ opA,
                     const uint8_t* __restrict__ opB, const float* __restrict__ norms,
                     const unsigned int* __restrict__ maxbits, float* __restrict__ out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t nk = g.nk, R = g.ring;
    uint8_t* sA = smem;                                   // nk x 32 KB
    uint8_t* sB = smem + nk * kG2Slice;                   // R x 32 KB
    uint8_t* sE = sB + R * kG2Slice;                      // 8 x kG2EpiBytes
    uint64_t* bars = reinterpret_cast<uint64_t*>(sE + 8 * kG2EpiBytes);
    // barrier slots: 0 a_full, 1 a_empty, 2..3 acc_full, 4..5 acc_empty, 6.. b_full[R], 6+R.. b_empty[R]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6 + 2 * R);
    const uint32_t bar0 = smem_u32(bars);
    auto BAR = [&](uint32_t k) { return bar0 + 8 * k; };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(BAR(0), 1);
        mbar_init(BAR(1), 1);
        mbar_init(BAR(2), 1);
        mbar_init(BAR(3), 1);
        mbar_init(BAR(4), 8);
        mbar_init(BAR(5), 8);
        for (uint32_t s = 0; s < 2 * R; ++s) mbar_init(BAR(6 + s), 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(256));
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
        if (lane == 0) {
            uint64_t cur = ~0ull;
            uint32_t na = 0, q = 0;
            for (uint64_t lam = tb; lam < te; ++lam) {
                const Coord c = ltm_map(lam, kReciprocal, true);
                if (c.i != cur) {
                    if (na > 0) mbar_wait(BAR(1), (na - 1) & 1);  // MMAs done with the old A
                    g2_bulk_load(smem_u32(sA), opA + c.i * nk * (uint64_t)kG2Slice, nk * kG2Slice, BAR(0));
                    cur = c.i;
                    ++na;
                }
                for (uint32_t k = 0; k < nk; ++k, ++q) {
                    const uint32_t s = q % R, round = q / R;
                    mbar_wait(BAR(6 + R + s), (round & 1) ^ 1);
                    g2_bulk_load(smem_u32(sB + s * kG2Slice), opB + (c.j * nk + k) * (uint64_t)kG2Slice, kG2Slice,
                                 BAR(6 + s));
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA
        if (lane == 0) {
            uint64_t cur = ~0ull;
            uint32_t na = 0, q = 0, it = 0;
            for (uint64_t lam = tb; lam < te; ++lam, ++it) {
                const Coord c = ltm_map(lam, kReciprocal, true);
                if (c.i != cur) {
                    mbar_wait(BAR(0), na & 1);
                    cur = c.i;
                    ++na;
                }
                const uint32_t buf = it & 1;
                mbar_wait(BAR(4 + buf), ((it >> 1) & 1) ^ 1);  // epilogue drained this accumulator
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t dtm = tmem + buf * kGT;
                for (uint32_t k = 0; k < nk; ++k, ++q) {
                    const uint32_t s = q % R, round = q / R;
                    mbar_wait(BAR(6 + s), round & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t ah = smem_u32(sA + k * kG2Slice), al = ah + kG2Half;
                    const uint32_t bh = smem_u32(sB + s * kG2Slice), bl = bh + kG2Half;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t ko = kk * 2 * kG2LBO;  // K = 16 fp16 = 2 core matrices
                        g2_mma(dtm, g2_desc(ah + ko), g2_desc(bl + ko), (k > 0 || kk > 0) ? 1u : 0u);
                        g2_mma(dtm, g2_desc(al + ko), g2_desc(bh + ko), 1u);
                        g2_mma(dtm, g2_desc(ah + ko), g2_desc(bh + ko), 1u);
                    }
                    g2_commit(BAR(6 + R + s));  // stage s free once these MMAs complete
                }
                g2_commit(BAR(2 + buf));  // accumulator ready
                bool last_of_row = lam + 1 >= te;
                if (!last_of_row) last_of_row = ltm_map(lam + 1, kReciprocal, true).i != c.i;
                if (last_of_row) g2_commit(BAR(1));  // A free
            }
        }
    } else {
        // ------------------------------------------------------- epilogue
        const uint32_t q = warp & 3, h = (warp - 2) >> 2;
        const int sh = g2_scale_exp(__ldg(maxbits));
        const float m2 = -2.0f * exp2f((float)(-2 * sh));
        const uint32_t a = (uint32_t)(q - (uint32_t)g.e_base) & 3u;  // warp-uniform alignment shift
        float4* wbuf = reinterpret_cast<float4*>(sE + (warp - 2) * kG2EpiBytes);
        const uint32_t r_lane = g2_perm(32 * q + lane);
        uint32_t it = 0;
        for (uint64_t lam = tb; lam < te; ++lam, ++it) {
            const Coord c = ltm_map(lam, kReciprocal, true);
            const uint64_t ri = c.i * kGT, rj = c.j * kGT;
            const uint32_t buf = it & 1;
            mbar_wait(BAR(2 + buf), (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint32_t v[64];
            const uint32_t taddr = tmem + ((32 * q) << 16) + buf * kGT + 64 * h;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                  "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                  "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(taddr));
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]),
                  "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]),
                  "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]),
                  "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]),
                  "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
                : "r"(taddr + 32));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) g2_arrive(BAR(4 + buf));  // TMEM buffer may be overwritten

            const uint64_t i = ri + r_lane;
            const uint64_t j0 = rj + 64 * h;
            const bool special = c.i == c.j || ri + kGT > g.n || ri < g.r0 || ri + kGT > g.r1;
            const float ni = __ldg(norms + i);  // norms are zero-padded to whole tiles
            float dv[64];
            const float4* nj4 = reinterpret_cast<const float4*>(norms + j0);
#pragma unroll
            for (int c4 = 0; c4 < 16; ++c4) {
                const float4 nj = __ldg(nj4 + c4);
                const float njv[4] = {nj.x, nj.y, nj.z, nj.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float d2 = fmaf(__uint_as_float(v[4 * c4 + t]), m2, __fadd_rn(ni, njv[t]));
                    float dd;
                    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(dd) : "f"(fmaxf(d2, 0.0f)));
                    dv[4 * c4 + t] = dd;
                }
            }
            if (special) {
#pragma unroll
                for (int cc = 0; cc < 64; ++cc)
                    if (j0 + cc == i) dv[cc] = 0.0f;
            }
            float4* my = wbuf + lane * kG2Chunks;
            switch (a) {
                case 0: g2_stage_row<0>(dv, my); break;
                case 1: g2_stage_row<1>(dv, my); break;
                case 2: g2_stage_row<2>(dv, my); break;
                default: g2_stage_row<3>(dv, my); break;
            }
            // float4 index of chunk 0 of this lane's row segment
            const uint64_t kbase = (i * (i + 1) / 2 + j0 - g.e_base - a) >> 2;
            __syncwarp();
#pragma unroll 1
            for (int s = 0; s < kG2Chunks; ++s) {
                const uint32_t idx = 32 * s + lane;
                const uint32_t row = idx / kG2Chunks, cch = idx - row * kG2Chunks;
                const float4 val = wbuf[idx];
                const uint64_t kb = __shfl_sync(0xffffffffu, (unsigned long long)kbase, row);
                const uint64_t ii = ri + g2_perm(32 * q + row);
                float* dst = out + 4 * (kb + cch);
                const int p0 = 4 * (int)cch - (int)a;  // segment position of element 0
                bool ok[4];
                bool all = true;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int p = p0 + t;
                    bool o = p >= 0 && p < 64;
                    if (special) {
                        const uint64_t jj = j0 + (uint64_t)p;
                        o = o && jj <= ii && ii < g.n && ii >= g.r0 && ii < g.r1;
                    }
                    ok[t] = o;
                    all = all && o;
                }
                if (all) {
                    *reinterpret_cast<float4*>(dst) = val;
                } else {
                    if (ok[0]) dst[0] = val.x;
                    if (ok[1]) dst[1] = val.y;
                    if (ok[2]) dst[2] = val.z;
                    if (ok[3]) dst[3] = val.w;
                }
            }
            __syncwarp();
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    }
}

}  // namespace tg
