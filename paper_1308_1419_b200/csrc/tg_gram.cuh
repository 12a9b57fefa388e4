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

}  // namespace tg
