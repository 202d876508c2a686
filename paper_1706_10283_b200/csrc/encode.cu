// encode.cu -- h(x): 4-bit PQ encoder and the
// layout-v1 pack/unpack helpers.
//
// Each thread encodes 4 consecutive rows; centroids of all codebooks sit in
// shared memory negated and transposed ([c][dim][16]) so that one LDS.128
// feeds 4 centroids to the 4 rows, and each (row, centroid pair) update is one
// packed FADD2 (x + (-c) == x - c exactly) and one FFMA2 -- the same fp32
// operations, in the same ascending-dimension order, as the scalar
// d += (x - c)^2.  The argmin keeps the lowest index on ties (R9).  Codes of
// a block (512 rows = 64 layout-v1 groups) are staged in shared memory and
// written as one contiguous run of 64*m words.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tma_host.cuh"

namespace bolt {
namespace {

constexpr int kEncThreads = 128;
constexpr int kEncRowsPerThread = 4;
constexpr int kEncRowsPerBlock = kEncThreads * kEncRowsPerThread;  // 512
constexpr int kEncGroupsPerBlock = kEncRowsPerBlock / kRowsPerWord;  // 64

template <bool kVec>
__global__ void __launch_bounds__(kEncThreads)
encode_kernel(const float* __restrict__ X, int64_t n, int j, int64_t ldx,
              const float* __restrict__ C, int m, uint32_t* __restrict__ codes) {
    extern __shared__ float4 enc_smem4[];
    float* cneg = reinterpret_cast<float*>(enc_smem4);  // [m][L][16] negated
    uint32_t* stage = reinterpret_cast<uint32_t*>(cneg + (size_t)j * kK);  // [64][m]
    const int L = j / m;
    // C is [m][16][L]; store -C as [m][L][16]
    for (int e = threadIdx.x; e < j * kK; e += blockDim.x) {
        int c = e / (kK * L);
        int r = e - c * kK * L;
        int k = r / L;
        int d = r - k * L;
        cneg[((size_t)c * L + d) * kK + k] = -C[e];
    }
    __syncthreads();

    const int64_t row0 = (int64_t)blockIdx.x * kEncRowsPerBlock + threadIdx.x * kEncRowsPerThread;
    const float* xr[kEncRowsPerThread];
    bool valid[kEncRowsPerThread];
#pragma unroll
    for (int r = 0; r < kEncRowsPerThread; ++r) {
        valid[r] = row0 + r < n;
        xr[r] = X + (valid[r] ? (row0 + r) : 0) * ldx;
    }
    for (int c = 0; c < m; ++c) {
        float2 d[kEncRowsPerThread][kK / 2];
#pragma unroll
        for (int r = 0; r < kEncRowsPerThread; ++r)
#pragma unroll
            for (int p = 0; p < kK / 2; ++p) d[r][p] = make_float2(0.f, 0.f);
        const float* cc = cneg + (size_t)c * L * kK;
        for (int d0 = 0; d0 < L; d0 += 4) {
            float xv[kEncRowsPerThread][4];
#pragma unroll
            for (int r = 0; r < kEncRowsPerThread; ++r) {
                const float* p = xr[r] + c * L + d0;
                if (kVec) {
                    float4 v = valid[r] ? __ldg(reinterpret_cast<const float4*>(p)) : make_float4(0, 0, 0, 0);
                    xv[r][0] = v.x; xv[r][1] = v.y; xv[r][2] = v.z; xv[r][3] = v.w;
                } else {
#pragma unroll
                    for (int t = 0; t < 4; ++t) xv[r][t] = (valid[r] && d0 + t < L) ? __ldg(p + t) : 0.f;
                }
            }
            const int dn = min(4, L - d0);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (t >= dn) break;
                const float4* cv = reinterpret_cast<const float4*>(cc + (size_t)(d0 + t) * kK);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float4 c4 = cv[q];
                    float2 ca = make_float2(c4.x, c4.y), cb = make_float2(c4.z, c4.w);
#pragma unroll
                    for (int r = 0; r < kEncRowsPerThread; ++r) {
                        float2 xx = make_float2(xv[r][t], xv[r][t]);
                        float2 da = __fadd2_rn(xx, ca);
                        float2 db = __fadd2_rn(xx, cb);
                        d[r][2 * q] = __ffma2_rn(da, da, d[r][2 * q]);
                        d[r][2 * q + 1] = __ffma2_rn(db, db, d[r][2 * q + 1]);
                    }
                }
            }
        }
        // argmin, lowest index on ties; pack this thread's 4 rows (16 bits)
        uint32_t half = 0;
#pragma unroll
        for (int r = 0; r < kEncRowsPerThread; ++r) {
            float best = d[r][0].x;
            uint32_t arg = 0;
#pragma unroll
            for (int p = 0; p < kK / 2; ++p) {
                if (p > 0 && d[r][p].x < best) { best = d[r][p].x; arg = 2 * p; }
                if (d[r][p].y < best) { best = d[r][p].y; arg = 2 * p + 1; }
            }
            if (!valid[r]) arg = 0;
            half |= arg << (4 * r);
        }
        uint32_t other = __shfl_xor_sync(0xffffffffu, half, 1);
        if ((threadIdx.x & 1) == 0) stage[(threadIdx.x >> 1) * m + c] = half | (other << 16);
    }
    __syncthreads();
    const int64_t g0 = (int64_t)blockIdx.x * kEncGroupsPerBlock;
    const int64_t groups = ceil_div(n, kRowsPerWord);
    const int64_t ng = min64(kEncGroupsPerBlock, groups - g0);
    uint32_t* dst = codes + g0 * m;
    for (int64_t e = threadIdx.x; e < ng * m; e += blockDim.x) dst[e] = stage[e];
}

// v2 for L = 8 (J/M = 8: c2, c4, c5): 2 rows per thread, the next codebook's
// 16 floats of the two rows prefetched into registers while the current one
// is processed (load latency hidden), 256 threads per block.  Same fp32
// operations in the same order as encode_kernel (bit-identical codes).
// 32-byte load (sm_100: LDG.E.ENL2.256): one L1TEX request per (row, codebook)
// slice instead of two 16-byte ones -- the row-strided loads are L1TEX-bound
__device__ __forceinline__ void ldg256(const float* p, float4& a, float4& b) {
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(p));
}

constexpr int kEnc2Threads = 256;
constexpr int kEnc2Rows = 2;
constexpr int kEnc2RowsPerBlock = kEnc2Threads * kEnc2Rows;  // 512 = 64 groups

// L = 8 (c2, c4, c5) or 16 (c3): the codebook's L floats of a row are L/8
// 32-byte loads.
// THREADS = 256 (512 rows = 64 groups per block) or 128 for small n, where
// 512-row blocks would leave SMs idle.
template <int L, int THREADS>
__global__ void __launch_bounds__(THREADS, L == 8 ? 3 * 256 / THREADS : 2 * 256 / THREADS)
encode_l8_kernel(const float* __restrict__ X, int64_t n, int64_t ldx, const float* __restrict__ C, int m,
                 uint32_t* __restrict__ codes) {
    extern __shared__ float4 enc_smem4[];
    static_assert(L == 8 || L == 16, "32-byte row slices");
    constexpr int NL = L / 8;  // 32-byte loads per (row, codebook)
    const int j = m * L;
    float* cneg = reinterpret_cast<float*>(enc_smem4);  // [m][L][16] negated
    uint32_t* stage = reinterpret_cast<uint32_t*>(cneg + (size_t)j * kK);  // [64][m]
    for (int e = threadIdx.x; e < j * kK; e += blockDim.x) {
        int c = e / (kK * L);
        int r = e - c * kK * L;
        int k = r / L;
        int d = r - k * L;
        cneg[((size_t)c * L + d) * kK + k] = -C[e];
    }
    __syncthreads();
    // thread t: rows 4*(t/2) + 2*(t%2) + {0,1}: a pair of threads covers 4 rows,
    // so the 16-bit half-words of a layout-v1 group are built as before
    constexpr int RPB = THREADS * kEnc2Rows, GPB = RPB / kRowsPerWord;  // rows, groups per block
    const int64_t row0 = (int64_t)blockIdx.x * RPB + threadIdx.x * kEnc2Rows;
    const float4* xr[kEnc2Rows];
    bool valid[kEnc2Rows];
#pragma unroll
    for (int r = 0; r < kEnc2Rows; ++r) {
        valid[r] = row0 + r < n;
        xr[r] = reinterpret_cast<const float4*>(X + (valid[r] ? (row0 + r) : 0) * ldx);
    }
    float4 nx[kEnc2Rows][2 * NL];
#pragma unroll
    for (int r = 0; r < kEnc2Rows; ++r)
#pragma unroll
        for (int h = 0; h < NL; ++h) {
            if (valid[r]) ldg256(reinterpret_cast<const float*>(xr[r] + 2 * h), nx[r][2 * h], nx[r][2 * h + 1]);
            else nx[r][2 * h] = nx[r][2 * h + 1] = make_float4(0, 0, 0, 0);
        }
    for (int c = 0; c < m; ++c) {
        float xv[kEnc2Rows][L];
#pragma unroll
        for (int r = 0; r < kEnc2Rows; ++r)
#pragma unroll
            for (int h = 0; h < 2 * NL; ++h) {
                xv[r][4 * h] = nx[r][h].x; xv[r][4 * h + 1] = nx[r][h].y;
                xv[r][4 * h + 2] = nx[r][h].z; xv[r][4 * h + 3] = nx[r][h].w;
            }
        if (c + 1 < m) {
#pragma unroll
            for (int r = 0; r < kEnc2Rows; ++r)
                if (valid[r])
#pragma unroll
                    for (int h = 0; h < NL; ++h)
                        ldg256(reinterpret_cast<const float*>(xr[r] + 2 * NL * (c + 1) + 2 * h), nx[r][2 * h],
                               nx[r][2 * h + 1]);
        }
        float2 d[kEnc2Rows][kK / 2];
#pragma unroll
        for (int r = 0; r < kEnc2Rows; ++r)
#pragma unroll
            for (int p = 0; p < kK / 2; ++p) d[r][p] = make_float2(0.f, 0.f);
        const float* cc = cneg + (size_t)c * L * kK;
#pragma unroll
        for (int t = 0; t < L; ++t) {
            const float4* cv = reinterpret_cast<const float4*>(cc + (size_t)t * kK);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float4 c4 = cv[q];
                float2 ca = make_float2(c4.x, c4.y), cb = make_float2(c4.z, c4.w);
#pragma unroll
                for (int r = 0; r < kEnc2Rows; ++r) {
                    float2 xx = make_float2(xv[r][t], xv[r][t]);
                    float2 da = __fadd2_rn(xx, ca);
                    float2 db = __fadd2_rn(xx, cb);
                    d[r][2 * q] = __ffma2_rn(da, da, d[r][2 * q]);
                    d[r][2 * q + 1] = __ffma2_rn(db, db, d[r][2 * q + 1]);
                }
            }
        }
        uint32_t quarter = 0;  // this thread's 2 rows (8 bits)
#pragma unroll
        for (int r = 0; r < kEnc2Rows; ++r) {
            float best = d[r][0].x;
            uint32_t arg = 0;
#pragma unroll
            for (int p = 0; p < kK / 2; ++p) {
                if (p > 0 && d[r][p].x < best) { best = d[r][p].x; arg = 2 * p; }
                if (d[r][p].y < best) { best = d[r][p].y; arg = 2 * p + 1; }
            }
            if (!valid[r]) arg = 0;
            quarter |= arg << (4 * r);
        }
        // 4 consecutive threads hold the 8 rows of one group
        const uint32_t q1 = __shfl_down_sync(0xffffffffu, quarter, 1);
        const uint32_t q2 = __shfl_down_sync(0xffffffffu, quarter, 2);
        const uint32_t q3 = __shfl_down_sync(0xffffffffu, quarter, 3);
        if ((threadIdx.x & 3) == 0) stage[(threadIdx.x >> 2) * m + c] = quarter | (q1 << 8) | (q2 << 16) | (q3 << 24);
    }
    __syncthreads();
    const int64_t g0 = (int64_t)blockIdx.x * GPB;
    const int64_t groups = ceil_div(n, kRowsPerWord);
    const int64_t ng = min64(GPB, groups - g0);
    uint32_t* dst = codes + g0 * m;
    for (int64_t e = threadIdx.x; e < ng * m; e += blockDim.x) dst[e] = stage[e];
}

// Direct-difference argmin of one (row, codebook) slice: encode_l8_kernel's
// fp32 operations in the same order (x + (-c), then fma, ascending
// dimensions; lowest index on ties).  Out of line: the fast kernel's rare
// fallback must not cost the hot loop registers.
template <int L>
__device__ __noinline__ uint32_t direct_argmin(const float* __restrict__ x, const float* __restrict__ cd) {
    float2 d[kK / 2];
#pragma unroll
    for (int p = 0; p < kK / 2; ++p) d[p] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int t = 0; t < L; ++t) {
        const float xt = __ldg(x + t);
        const float2 xx = make_float2(xt, xt);
        const float4* cv = reinterpret_cast<const float4*>(cd + (size_t)t * kK);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 c4 = cv[q];
            const float2 da = __fadd2_rn(xx, make_float2(c4.x, c4.y));
            const float2 db = __fadd2_rn(xx, make_float2(c4.z, c4.w));
            d[2 * q] = __ffma2_rn(da, da, d[2 * q]);
            d[2 * q + 1] = __ffma2_rn(db, db, d[2 * q + 1]);
        }
    }
    float best = d[0].x;
    uint32_t arg = 0;
#pragma unroll
    for (int p = 0; p < kK / 2; ++p) {
        if (p > 0 && d[p].x < best) { best = d[p].x; arg = 2 * p; }
        if (d[p].y < best) { best = d[p].y; arg = 2 * p + 1; }
    }
    return arg;
}

// Argmin epilogue of the expanded kernel (A/B switch, tools/gpu_ab_enc*.sh;
// DESIGN.md 6.3 has the measurements):
//   2 (default) bit-group minima, no index tags, need as two FFMAs
//   3           runner-up test and argmin on the FMA pipe (slower)
//   1           index tags, one LOP3 each, 32-bit row arithmetic
//   0           round 2's first epilogue (two LOP3 per tag, 64-bit row arithmetic)
#ifndef BOLT_ENC_LEAN
#define BOLT_ENC_LEAN 2
#endif
// 1: the direct-difference fallback reads x and the centroids from shared memory
#ifndef BOLT_ENC_FB_SMEM
#define BOLT_ENC_FB_SMEM 1
#endif
// PK (template): a warp's 4-bit codes of a stage go through a byte staging
// area in shared memory ([codebook][slab][lane]; the fallback overwrites its own
// byte) and are packed into layout-v1 words once per stage, instead of three
// shuffle-OR steps and a predicated store per (codebook, row) and atomics in
// the fallback.  Used for J <= 128 (c2 0.168 -> 0.160 ms); for J = 512 the
// staging area would cost a stage (3 -> 2), for J = 256 it measured no gain.
// BOLT_ENC_PACK=0 switches it off (A/B).
#ifndef BOLT_ENC_PACK
#define BOLT_ENC_PACK 1
#endif
constexpr int kEncPackCb = 2;  // staged codebooks per warp and stage

// (x & mask) | K in one LOP3: with the mask in a register and the 4-bit
// centroid index as the immediate (ptxas splits the all-immediate form into
// an AND and an OR)
template <uint32_t K>
__device__ __forceinline__ float tag_low4(float x, uint32_t mask) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(__float_as_uint(x)), "r"(mask), "n"(K));
    return __uint_as_float(d);
}

// Expanded distances (BOLT_ENCODE_EXPANDED): per
// centroid s_k = fl(||c_k||^2) + sum_t x_t (-2 c_kt) as one packed FFMA chain
// (one FFMA per (dimension, centroid) instead of a subtract and an FFMA),
// which orders the centroids like ||x - c_k||^2 up to a rigorous rounding
// bound; the code is that argmin unless another centroid falls within the
// bound, in which case the codebook is recomputed by direct differences with
// encode_l8_kernel's exact fp32 operations.  Codes are therefore bit-identical
// to the direct kernel (tests/test_gpu_parity.py compares the two).
//
// Bound (u = 2^-24, g(n) = n u / (1 - n u)): the FFMA chain of L terms from
// n_k = fl(||c_k||^2) errs by <= g(L)(|n_k| + 2 sum_t |x_t||c_kt|), n_k by
// <= g(L)||c_k||^2; with 2 sum_t |x_t||c_kt| <= ||x||^2 + ||c_k||^2 that is
// |s^_k - s_k| < 1.5 g(L)(1 + g(L)) A, A = 2 C2 + X2 (C2 >= max_k n_k, X2 >=
// ||x||^2 of the slice), and E = 2 g(L) A bounds it (round 2's first
// version: 4 g(L) A, twice the fallbacks).  The direct fp32 distance errs by
// <= g(L+2) d_k.  With b1 = min_k s^_k and every other s^_k >= b1 + need,
// need = 2.5 E + 3 g(L+2)(X2 + |b1| + E) (X2 >= ||x||^2), the direct
// distances keep the same unique minimum.  The factors carry a >= 25 % slack
// for the rounding of the test itself.
//
// The kernel is persistent (one CTA per SM; the centroid tables are set up
// once) and streams whole rows: a stage is R = 32 RT consecutive rows x J
// floats, brought in by J/32 2-D tensor copies of 32-float (128-byte) x R
// boxes in the 128-byte swizzle, kRowStages stages in flight.  Warp 8 issues
// the copies; compute warp w owns codebooks [w CPW, w CPW + CPW) of every row
// of RT of the stage's NS 32-row slabs (lane = row within a slab), so the
// centroid loads of a codebook are shared by RT rows.  (Round 2's first version staged
// 32-byte row slices per codebook in short-lived 512-row blocks: 0.205 ms on
// c2, no faster than the direct kernel.)

// direct_argmin reading the centroids from global memory (x + (-c) == x - c
// exactly): the expanded kernel's rare fallback, no negated table in shared memory
template <int L>
__device__ __noinline__ uint32_t direct_argmin_g(const float* __restrict__ x, const float* __restrict__ c) {
    float2 d[kK / 2];
#pragma unroll
    for (int p = 0; p < kK / 2; ++p) d[p] = make_float2(0.f, 0.f);
    for (int t = 0; t < L; ++t) {
        const float xt = __ldg(x + t);
        const float2 xx = make_float2(xt, xt);
#pragma unroll
        for (int p = 0; p < kK / 2; ++p) {
            const float2 cp = make_float2(-__ldg(c + (2 * p) * L + t), -__ldg(c + (2 * p + 1) * L + t));
            const float2 dd = __fadd2_rn(xx, cp);
            d[p] = __ffma2_rn(dd, dd, d[p]);
        }
    }
    float best = d[0].x;
    uint32_t arg = 0;
#pragma unroll
    for (int p = 0; p < kK / 2; ++p) {
        if (p > 0 && d[p].x < best) { best = d[p].x; arg = 2 * p; }
        if (d[p].y < best) { best = d[p].y; arg = 2 * p + 1; }
    }
    return arg;
}

// direct_argmin from shared memory: x from the stage's swizzled row (rowp, the
// slice's first 16-byte chunk ch0, row rl) and the centroids from the -2c
// table, -c = 0.5 * (-2c) exactly, so fma(-2c, 0.5, x) is the direct kernel's
// fl(x + (-c)) and the distances are its fp32 operations in its order.  The
// expanded kernel's fallback (A/B: BOLT_ENC_FB_SMEM=0 reads X and C from
// global memory, round 2's first version).
template <int L>
__device__ __noinline__ uint32_t direct_argmin_s(const uint8_t* __restrict__ rowp, int ch0, int rl,
                                                 const float* __restrict__ ccm) {
    float xv[L];
#pragma unroll
    for (int h = 0; h < L / 4; ++h) {
        const float4 v = *reinterpret_cast<const float4*>(rowp + (((ch0 + h) ^ (rl & 7)) << 4));
        xv[4 * h] = v.x; xv[4 * h + 1] = v.y; xv[4 * h + 2] = v.z; xv[4 * h + 3] = v.w;
    }
    float2 d[kK / 2];
#pragma unroll
    for (int p = 0; p < kK / 2; ++p) d[p] = make_float2(0.f, 0.f);
    const float2 hf = make_float2(0.5f, 0.5f);
#pragma unroll
    for (int t = 0; t < L; ++t) {
        const float2 xx = make_float2(xv[t], xv[t]);
        const float4* cv = reinterpret_cast<const float4*>(ccm + (size_t)t * kK);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 c4 = cv[q];
            const float2 da = __ffma2_rn(make_float2(c4.x, c4.y), hf, xx);
            const float2 db = __ffma2_rn(make_float2(c4.z, c4.w), hf, xx);
            d[2 * q] = __ffma2_rn(da, da, d[2 * q]);
            d[2 * q + 1] = __ffma2_rn(db, db, d[2 * q + 1]);
        }
    }
    float best = d[0].x;
    uint32_t arg = 0;
#pragma unroll
    for (int p = 0; p < kK / 2; ++p) {
        if (p > 0 && d[p].x < best) { best = d[p].x; arg = 2 * p; }
        if (d[p].y < best) { best = d[p].y; arg = 2 * p + 1; }
    }
    return arg;
}

template <int L, int NS, int RT, int W, int H, bool PK = false>
__global__ void __launch_bounds__(32 * W + 32, 1)
encode_rows_kernel(const __grid_constant__ CUtensorMap xmap, const float* __restrict__ X, int64_t n, int64_t ldx,
                   const float* __restrict__ C, int m, uint32_t* __restrict__ codes, int64_t nblocks, int S,
                   int xm) {
    static_assert(L == 8 || L == 16, "32-float boxes hold 32 / L codebooks");
#ifndef BOLT_XMODE
    xm = 0;  // diagnostic switches (1: loads only, 2: no fallback, 4: no code stores) exist only in libbolt_x.so
#endif
    extern __shared__ __align__(1024) uint8_t enc_row_smem[];
    constexpr float kU = 5.9604645e-8f;  // 2^-24
    constexpr float kGL = (float)L * kU / (1.0f - (float)L * kU);
    constexpr float kGL2 = (float)(L + 2) * kU / (1.0f - (float)(L + 2) * kU);
    // E = kE g(L) A: the chain errs by <= g(L)(|n_k| + 2 sum|x_t||c_kt|) <= g(L)(1 + g(L))(2 C2 + X2)
    // and n_k by <= g(L) C2, together < 1.5 g(L)(1 + g(L)) A; kE = 2 keeps > 25 % slack
    // (BOLT_ENC_E4: round 2's first factor, 4)
#ifdef BOLT_ENC_E4
    constexpr float kE = 4.0f;
#else
    constexpr float kE = 2.0f;
#endif
    constexpr float kN1 = 2.5f * kE * kGL + 3.0f * kGL2 * kE * kGL;
    constexpr float kN3 = (kN1 + 3.0f * kGL2) * (1.0f + 2.0f * kGL);   // on the computed ||x||^2 (rounded up by 1 + 2 g(L))
    constexpr float kN4 = 3.0f * kGL2;
    static_assert(NS % RT == 0, "slab groups");
    constexpr int R = 32 * NS;           // rows per stage
    constexpr int SG = NS / RT;          // slab groups (of RT slabs)
    const int j = m * L;
    const int jh = j / H;                // floats of a row per stage (H column parts per row block)
    const int mh = m / H;                // codebooks per stage
    const int nbox = jh / 32;
    const uint32_t stage_bytes = (uint32_t)R * jh * 4;
    const int cpw = mh * SG / W;         // codebooks per compute warp (mh * SG % W == 0)
    uint8_t* xs = enc_row_smem;                                          // [S][j/32][R][32] swizzled
    float* cm2 = reinterpret_cast<float*>(xs + (size_t)S * stage_bytes);  // [m][L][16] -2c
    float* cn = cm2 + (size_t)j * kK;                                    // [m][16]
    float* c2max = cn + (size_t)m * kK;                                  // [m]
    uint32_t* tagmask = reinterpret_cast<uint32_t*>(c2max + ((m + 1) & ~1));  // [2]: ~0xF, kept out of ptxas's sight
    uint64_t* full = reinterpret_cast<uint64_t*>(tagmask + 2);
    uint64_t* empty = full + S;
    uint8_t* const pk = reinterpret_cast<uint8_t*>(empty + S) + (threadIdx.x >> 5) * (kEncPackCb * RT * 32);  // PK only
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], W);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // centroid tables, before the copy warp enters its loop (a block barrier
    // after that point would deadlock against its empty-slot waits)
    for (int e = tid; e < j * kK; e += blockDim.x) {
        int c = e / (kK * L);
        int r = e - c * kK * L;
        int k = r / L;
        int d = r - k * L;
        cm2[((size_t)c * L + d) * kK + k] = -2.0f * C[e];
    }
    for (int e = tid; e < m * kK; e += blockDim.x) {
        const float* ck = C + (size_t)e * L;
        float acc = 0.f;
        for (int t = 0; t < L; ++t) acc = __fmaf_rn(ck[t], ck[t], acc);
        cn[e] = acc;
    }
    __syncthreads();
    for (int c = tid; c < m; c += blockDim.x) {
        float a = 0.f;
        for (int k = 0; k < kK; ++k) a = fmaxf(a, fabsf(cn[c * kK + k]));
#if BOLT_ENC_LEAN >= 2
        // need = 2.5 E + 3 g(L+2)(X2 + |b1| + E) with E = kE g(L)(2 C2 + X2), sorted by
        // variable: kN1 2 C2 (this table) + kN3 ||x||^2 + kN4 |b1|
        c2max[c] = 2.0f * kN1 * (a * (1.0f + 2.0f * kGL));
#else
        c2max[c] = a * (1.0f + 2.0f * kGL);
#endif
    }
    if (tid == 0) tagmask[0] = ~0xFu;
    __syncthreads();
    if (warp == W) {
        // ------------------------------------------------ copy warp
        if (lane == 0) {
            for (int i = 0;; ++i) {
                const int64_t b = blockIdx.x + (int64_t)(i / H) * gridDim.x;  // row block, column part i % H
                if (b >= nblocks) break;
                const int s = i % S;
                tc::mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(&full[s])),
                             "r"(stage_bytes)
                             : "memory");
                const uint32_t dst = tc::smem_u32(xs + (size_t)s * stage_bytes);
                for (int bx = 0; bx < nbox; ++bx)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                            "r"(dst + (uint32_t)bx * (R * 128)),
                        "l"(&xmap), "r"((i % H) * jh + bx * 32), "r"((int)(b * R)), "r"(tc::smem_u32(&full[s]))
                        : "memory");
            }
        }
        return;
    }
    // ---------------------------------------------------- compute warps
    for (int i = 0;; ++i) {
        const int64_t b = blockIdx.x + (int64_t)(i / H) * gridDim.x;
        if (b >= nblocks) break;
        const int c0 = (i % H) * mh;  // first codebook of this stage
        const int s = i % S;
        const int64_t row_blk = b * R;
        uint32_t amb = 0;  // ambiguous (codebook, slab) items of this stage, bit cc RT + r
#if BOLT_ENC_LEAN
        // 32-bit row arithmetic within the stage: rows left in it, its first code word
        const int nrem = (int)min64(n - row_blk, (int64_t)R);
        uint32_t* const cst = codes + (row_blk >> 3) * m;
        const uint32_t tmask = tagmask[0];
        // this lane's group word of the warp's first slab (slab r: + 4 r m words)
        uint32_t* const wp = cst + ((32 * ((warp % SG) * RT) + lane) >> 3) * m;
#endif
        tc::mbar_wait(&full[s], (i / S) & 1);
        const uint8_t* st = xs + (size_t)s * stage_bytes;
        for (int cc = 0; cc < (xm & 1 ? 0 : cpw); ++cc) {
            const int c = c0 + (warp / SG) * cpw + cc;
            const int sl0 = (warp % SG) * RT;         // first slab of this warp
            const int bx = ((c - c0) * L) >> 5;       // box of this codebook's L floats
            const int ch0 = ((c * L) & 31) >> 2;      // its first 16-byte chunk within the 128-byte row
            float xv[RT][L];
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                const int rl = 32 * (sl0 + r) + lane;
                const uint8_t* rowp = st + (size_t)bx * (R * 128) + rl * 128;
#pragma unroll
                for (int h = 0; h < L / 4; ++h) {
                    const float4 v = *reinterpret_cast<const float4*>(rowp + (((ch0 + h) ^ (rl & 7)) << 4));
                    xv[r][4 * h] = v.x; xv[r][4 * h + 1] = v.y; xv[r][4 * h + 2] = v.z; xv[r][4 * h + 3] = v.w;
                }
            }
            float2 sv[RT][kK / 2];
            float2 x2p[RT];  // ||x||^2 of the slice, as (even, odd) dimension partial sums
            {
                const float4* cn4 = reinterpret_cast<const float4*>(cn + c * kK);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 v = cn4[q];
#pragma unroll
                    for (int r = 0; r < RT; ++r) {
                        sv[r][2 * q] = make_float2(v.x, v.y);
                        sv[r][2 * q + 1] = make_float2(v.z, v.w);
                    }
                }
#pragma unroll
                for (int r = 0; r < RT; ++r) {
                    x2p[r] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int h = 0; h < L / 2; ++h) {
                        const float2 xp = make_float2(xv[r][2 * h], xv[r][2 * h + 1]);
                        x2p[r] = __ffma2_rn(xp, xp, x2p[r]);
                    }
                }
            }
            const float* ccm = cm2 + (size_t)c * L * kK;
#pragma unroll
            for (int t = 0; t < L; ++t) {
                const float4* cv = reinterpret_cast<const float4*>(ccm + (size_t)t * kK);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 c4 = cv[q];
                    const float2 ca = make_float2(c4.x, c4.y), cb = make_float2(c4.z, c4.w);
#pragma unroll
                    for (int r = 0; r < RT; ++r) {
                        const float2 xx = make_float2(xv[r][t], xv[r][t]);
                        sv[r][2 * q] = __ffma2_rn(xx, ca, sv[r][2 * q]);
                        sv[r][2 * q + 1] = __ffma2_rn(xx, cb, sv[r][2 * q + 1]);
                    }
                }
            }
            const float c2 = c2max[c];
#pragma unroll
            for (int r = 0; r < RT; ++r) {
#if BOLT_ENC_LEAN
                const int lrow = 32 * (sl0 + r) + lane;
                const bool valid = lrow < nrem;
#else
                const int64_t row = row_blk + 32 * (sl0 + r) + lane;
                const bool valid = row < n;
#endif
#if BOLT_ENC_LEAN == 3
                // A/B: runner-up test and argmin on the FMA pipe.  b1 = min (3-input
                // tree), y_k = s^_k - b1 >= 0, z_k = sat(y_k / need) in [0, 1]: z = 0 for
                // the argmin and 1 for every value at least need above it, so the slice
                // is unambiguous iff sum z_k = 15, and then sum k z_k = 120 - argmin.
                // (The sums' rounding lets a z_k within 4e-6 of 1 through, far inside
                // need's 25 % slack; need = 0: 1 / need = inf, 0 * inf = NaN -> sat 0.)
                static_assert(kK == 16, "sixteen centroids");
                const float b1 =
                    fminf(fminf(fminf(fminf(sv[r][0].x, sv[r][0].y), sv[r][1].x),
                                fminf(fminf(sv[r][1].y, sv[r][2].x), sv[r][2].y)),
                          fminf(fminf(fminf(fminf(sv[r][3].x, sv[r][3].y), sv[r][4].x),
                                      fminf(fminf(sv[r][4].y, sv[r][5].x), sv[r][5].y)),
                                fminf(fminf(fminf(sv[r][6].x, sv[r][6].y), sv[r][7].x), sv[r][7].y)));
                const float need3 = __fmaf_rn(kN4, fabsf(b1), __fmaf_rn(kN3, x2p[r].x + x2p[r].y, c2));
                float rneed;
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rneed) : "f"(need3));
                const float2 nb = make_float2(-b1, -b1);
                float2 zs[kK / 2];
                float tsum = 0.f;
#pragma unroll
                for (int p = 0; p < kK / 2; ++p) {
                    const float2 y = __fadd2_rn(sv[r][p], nb);
                    asm("mul.rn.sat.f32 %0, %1, %2;" : "=f"(zs[p].x) : "f"(y.x), "f"(rneed));
                    asm("mul.rn.sat.f32 %0, %1, %2;" : "=f"(zs[p].y) : "f"(y.y), "f"(rneed));
                    if (p > 0) tsum = __fmaf_rn(zs[p].x, (float)(2 * p), tsum);
                    tsum = __fmaf_rn(zs[p].y, (float)(2 * p + 1), tsum);
                }
#pragma unroll
                for (int w = kK / 4; w >= 1; w /= 2)
#pragma unroll
                    for (int p = 0; p < w; ++p) zs[p] = __fadd2_rn(zs[p], zs[p + w]);
                const bool ambig = !(zs[0].x + zs[0].y >= 15.0f) && valid;
                const uint32_t arg = valid ? ((uint32_t)__float2int_rn(120.0f - tsum) & 0xFu) : 0u;
#elif BOLT_ENC_LEAN == 2
                // Bit-group minima (no index tags): m[j][b] = min of the values whose
                // index has bit j = b.  The minimum is min(m[j][0], m[j][1]) for any j;
                // the runner-up differs from the argmin in some bit j, where it is the
                // other group's minimum, and every max(m[j][0], m[j][1]) is the minimum
                // of a group without the argmin, so second = min_j max(m[j][0], m[j][1]);
                // bit j of the argmin is m[j][1] < m[j][0] (an exact tie makes
                // second == min: ambiguous, redone by direct differences).
                static_assert(kK == 16, "four index bits");
                float pm[8], qm[4];
#pragma unroll
                for (int p = 0; p < 8; ++p) pm[p] = fminf(sv[r][p].x, sv[r][p].y);
#pragma unroll
                for (int p = 0; p < 4; ++p) qm[p] = fminf(pm[2 * p], pm[2 * p + 1]);
                const float m30 = fminf(qm[0], qm[1]), m31 = fminf(qm[2], qm[3]);
                const float m20 = fminf(qm[0], qm[2]), m21 = fminf(qm[1], qm[3]);
                const float m10 = fminf(fminf(pm[0], pm[2]), fminf(pm[4], pm[6]));
                const float m11 = fminf(fminf(pm[1], pm[3]), fminf(pm[5], pm[7]));
                const float m00 = fminf(fminf(fminf(sv[r][0].x, sv[r][1].x), sv[r][2].x),
                                        fminf(fminf(fminf(sv[r][3].x, sv[r][4].x), sv[r][5].x),
                                              fminf(sv[r][6].x, sv[r][7].x)));
                const float m01 = fminf(fminf(fminf(sv[r][0].y, sv[r][1].y), sv[r][2].y),
                                        fminf(fminf(fminf(sv[r][3].y, sv[r][4].y), sv[r][5].y),
                                              fminf(sv[r][6].y, sv[r][7].y)));
                const float b1 = fminf(m30, m31);
                const float b2 = fminf(fminf(fminf(fmaxf(m00, m01), fmaxf(m10, m11)), fmaxf(m20, m21)), fmaxf(m30, m31));
                // sign bits of m[j][1] - m[j][0], funnel-shifted together (bit 3 first)
                uint32_t argb = __float_as_uint(m31 - m30) >> 31;
                argb = __funnelshift_l(__float_as_uint(m21 - m20), argb, 1);
                argb = __funnelshift_l(__float_as_uint(m11 - m10), argb, 1);
                argb = __funnelshift_l(__float_as_uint(m01 - m00), argb, 1);
#else
                // index k in the low 4 mantissa bits of s^_k (a change of < 2^-19 |s^_k|):
                // the minimum of the tagged values names its centroid; a (min,
                // second) tree gives the two smallest
                float lo[kK / 2], hi[kK / 2];
#if BOLT_ENC_LEAN
#define BOLT_TAG_PAIR(P)                                                   \
    {                                                                      \
        const float e0 = tag_low4<2u * (P)>(sv[r][P].x, tmask);            \
        const float e1 = tag_low4<2u * (P) + 1u>(sv[r][P].y, tmask);       \
        lo[P] = fminf(e0, e1);                                             \
        hi[P] = fmaxf(e0, e1);                                             \
    }
                BOLT_TAG_PAIR(0) BOLT_TAG_PAIR(1) BOLT_TAG_PAIR(2) BOLT_TAG_PAIR(3)
                BOLT_TAG_PAIR(4) BOLT_TAG_PAIR(5) BOLT_TAG_PAIR(6) BOLT_TAG_PAIR(7)
#undef BOLT_TAG_PAIR
                static_assert(kK == 16, "eight tagged pairs");
#else
#pragma unroll
                for (int p = 0; p < kK / 2; ++p) {
                    const float e0 = __uint_as_float((__float_as_uint(sv[r][p].x) & ~0xFu) | (2u * p));
                    const float e1 = __uint_as_float((__float_as_uint(sv[r][p].y) & ~0xFu) | (2u * p + 1u));
                    lo[p] = fminf(e0, e1);
                    hi[p] = fmaxf(e0, e1);
                }
#endif
#pragma unroll
                for (int w = kK / 4; w >= 1; w /= 2)
#pragma unroll
                    for (int p = 0; p < w; ++p) {
                        const float l = fminf(lo[p], lo[p + w]);
                        hi[p] = fminf(fmaxf(lo[p], lo[p + w]), fminf(hi[p], hi[p + w]));
                        lo[p] = l;
                    }
                const float b1 = lo[0], b2 = hi[0];
#endif
                // |s^_k| <= A = 2 C2 + X2 (2|x.c| <= X2 + ||c||^2), so E = 4 g(L) A
                // bounds |s^_k - s_k| (2 sum|x_t||c_kt| <= X2 + C2) and the tags move
                // each value by < 2^-19 A; need' = need + 2 * 2^-19 A (25 % slack)
#if BOLT_ENC_LEAN == 3
#elif BOLT_ENC_LEAN == 2
                // the same need without the tag term (no tags), as two FFMAs on the
                // per-codebook constant
                const float need = __fmaf_rn(kN4, fabsf(b1), __fmaf_rn(kN3, x2p[r].x + x2p[r].y, c2));
                const bool ambig = !(b2 >= b1 + need) && valid;
                const uint32_t arg = valid ? argb : 0u;
#else
                const float X2 = (x2p[r].x + x2p[r].y) * (1.0f + 2.0f * kGL);
                const float A = 2.0f * c2 + X2;
                const float E = 4.0f * kGL * A;
                const float need = 2.5f * E + 3.0f * kGL2 * (X2 + fabsf(b1) + E) + 1.25f * 3.8146973e-6f * A;
                const bool ambig = !(b2 >= b1 + need) && valid;
                const uint32_t arg = valid ? (__float_as_uint(b1) & 0xFu) : 0u;
#endif
                amb |= (ambig ? 1u : 0u) << (cc * RT + r);
                if constexpr (PK) {
                    pk[(cc * RT + r) * 32 + lane] = (uint8_t)arg;
                } else {
                // layout-v1 word of this row's group: 8 consecutive lanes hold its 8 rows
                uint32_t v = arg << (4 * (lane & 7));
                v |= __shfl_xor_sync(0xffffffffu, v, 1);
                v |= __shfl_xor_sync(0xffffffffu, v, 2);
                v |= __shfl_xor_sync(0xffffffffu, v, 4);
#if BOLT_ENC_LEAN
                // the group's first row is this lane's: it exists iff the row does
                if ((lane & 7) == 0 && valid && !(xm & 4)) wp[4 * r * m + c] = v;
#else
                const int64_t g = row >> 3;
                if ((lane & 7) == 0 && g * kRowsPerWord < n && !(xm & 4)) codes[g * m + c] = v;
#endif
                }
            }
        }
        // ambiguous (row, codebook) slices: direct differences (the direct
        // kernel's exact fp32 operations), patched into the stored words; the
        // lanes of a warp run their fallbacks side by side
        __syncwarp();
        if (xm & 2) amb = 0;
        while (amb) {
            const int bit = __ffs(amb) - 1;
            amb &= amb - 1;
            const int cc = bit / RT, r = bit - cc * RT;
            const int c = c0 + (warp / SG) * cpw + cc;
            const int64_t row = row_blk + 32 * ((warp % SG) * RT + r) + lane;
#if BOLT_ENC_FB_SMEM
            const int rl = 32 * ((warp % SG) * RT + r) + lane;
            const uint32_t arg = direct_argmin_s<L>(st + (size_t)(((c - c0) * L) >> 5) * (R * 128) + rl * 128,
                                                    ((c * L) & 31) >> 2, rl, cm2 + (size_t)c * L * kK);
#else
            const uint32_t arg = direct_argmin_g<L>(X + row * ldx + c * L, C + (size_t)c * kK * L);
#endif
            if constexpr (PK) {
                pk[bit * 32 + lane] = (uint8_t)arg;  // bit = cc RT + r: this lane's own byte
            } else {
                const int pos = 4 * (int)(row & 7);
                uint32_t* w = codes + (row >> 3) * m + c;
                atomicAnd(w, ~(0xFu << pos));
                atomicOr(w, arg << pos);
            }
        }
        __syncwarp();
#if BOLT_ENC_LEAN
        // word l of the warp = bytes 8 l .. 8 l + 7 of its staging area: codebook
        // l / (4 RT), slab (l / 4) % RT, rows 8 (l % 4) .. + 7 of the slab
        if (PK && lane < 4 * RT * cpw && !(xm & 4)) {
            const uint2 b = reinterpret_cast<const uint2*>(pk)[lane];
            const uint32_t tl = b.x | (b.x >> 4), th = b.y | (b.y >> 4);  // byte 0 = b0 | b1 << 4, byte 2 = b2 | b3 << 4
            const uint32_t v = __byte_perm(tl, th, 0x6420);
            const int cc = lane / (4 * RT), r = (lane >> 2) % RT;
            const int lrow0 = 32 * ((warp % SG) * RT + r) + 8 * (lane & 3);
            if (lrow0 < nrem) cst[(lrow0 >> 3) * m + c0 + (warp / SG) * cpw + cc] = v;
        }
        if constexpr (PK) __syncwarp();
#endif
        if (lane == 0) tc::mbar_arrive(&empty[s]);  // this warp is done with the stage
    }
}

__global__ void pack_kernel(const uint8_t* __restrict__ flat, int64_t n, int m,
                            uint32_t* __restrict__ codes) {
    int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = ceil_div(n, kRowsPerWord) * m;
    if (w >= total) return;
    int64_t g = w / m;
    int c = (int)(w - g * m);
    uint32_t word = 0;
    for (int r = 0; r < kRowsPerWord; ++r) {
        int64_t i = g * kRowsPerWord + r;
        if (i < n) word |= (uint32_t)(flat[i * m + c] & 0xF) << (4 * r);
    }
    codes[w] = word;
}

__global__ void unpack_kernel(const uint32_t* __restrict__ codes, int64_t n, int m,
                              uint8_t* __restrict__ flat) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * m) return;
    int64_t i = e / m;
    int c = (int)(e - i * m);
    flat[e] = (uint8_t)((codes[(i >> 3) * m + c] >> (4 * (i & 7))) & 0xF);
}

}  // namespace

cudaError_t launch_encode(const float* X, int64_t n, int j, int64_t ldx, const float* C, int m,
                          uint32_t* codes, int sms, cudaStream_t s, int mode) {
    if (n == 0) return cudaSuccess;
    const int L = j / m;
    size_t smem = (size_t)j * kK * sizeof(float) + (size_t)kEncGroupsPerBlock * m * sizeof(uint32_t);
    bool vec = (L % 4 == 0) && (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    int64_t blocks = ceil_div(n, kEncRowsPerBlock);
    // AUTO: the expanded kernel where it applies (c2 0.184 vs 0.199 ms, c3
    // 0.538 vs 0.671, c4 0.059 vs 0.067)
    if ((mode == 2 || mode == 0) && (L == 8 || L == 16) && j % 32 == 0 && j <= 512 && m % 8 == 0 && (ldx % 4) == 0 &&
        (reinterpret_cast<uintptr_t>(X) & 15) == 0 && encode_tiled()) {
        // persistent whole-row TMA expanded-distance kernel (bit-identical codes)
        // H column parts per row block (J = 512: two stages of 64 rows x 256 floats),
        // NS 32-row slabs per 64 KB stage, 16 compute warps of RT slabs each
        const int H = j <= 256 ? 1 : 2;
        const int jh = j / H;
        const int NS = jh <= 128 ? 4 : 2;
        int W = 16, RT = 2;
        const bool pack = BOLT_ENC_PACK && BOLT_ENC_LEAN && L == 8 && NS == 4 && H == 1;
#ifdef BOLT_XMODE
        if (getenv("BOLT_ENC_W8") && NS == 4) W = 8, RT = 4;
#endif
        const int R = 32 * NS;
        const size_t stage = (size_t)R * jh * sizeof(float);
        const size_t tables = (size_t)j * kK * sizeof(float) + (size_t)m * kK * sizeof(float) +
                              (size_t)(((m + 1) & ~1) + 2) * sizeof(float) +  // + the tag mask word
                              (pack ? (size_t)(W + 1) * kEncPackCb * RT * 32 : 0);  // code staging, per warp
        const size_t budget = 227 * 1024 - 256;
        int S = (int)std::min<size_t>(4, (budget - tables - 8 * sizeof(uint64_t)) / stage);
        int xm = 0;
#ifdef BOLT_XMODE
        if (const char* e = getenv("BOLT_ENC_XMODE")) xm = atoi(e);
        if (const char* e = getenv("BOLT_ENC_STAGES")) S = std::min(S, atoi(e));
#endif
        CUtensorMap xmap{};
        const cuuint64_t dims[2] = {(cuuint64_t)j, (cuuint64_t)n};
        const cuuint64_t strides[1] = {(cuuint64_t)(ldx * sizeof(float))};
        const cuuint32_t box[2] = {32u, (cuuint32_t)R};
        const cuuint32_t estr[2] = {1u, 1u};
        if (S >= 2 && ((m / H) * (NS / RT)) % W == 0 && (!pack || (m / H) * (NS / RT) / W <= kEncPackCb) && n < (int64_t(1) << 31) &&
            encode_tiled()(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
            const size_t tsmem = (size_t)S * stage + tables + 2 * (size_t)S * sizeof(uint64_t);
            const int64_t nblocks = ceil_div(n, (int64_t)R);
            const unsigned grid = (unsigned)std::min<int64_t>(nblocks, sms);
            decltype(&encode_rows_kernel<8, 4, 2, 16, 1>) kern;
            if (L == 8) kern = H == 2 ? encode_rows_kernel<8, 2, 2, 16, 2>
                             : NS == 4 ? (W == 8 ? encode_rows_kernel<8, 4, 4, 8, 1>
                                          : pack ? encode_rows_kernel<8, 4, 2, 16, 1, true> : encode_rows_kernel<8, 4, 2, 16, 1>)
                                       : encode_rows_kernel<8, 2, 2, 16, 1>;
            else kern = H == 2 ? encode_rows_kernel<16, 2, 2, 16, 2>
                        : NS == 4 ? encode_rows_kernel<16, 4, 2, 16, 1> : encode_rows_kernel<16, 2, 2, 16, 1>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
            kern<<<grid, 32 * W + 32, tsmem, s>>>(xmap, X, n, ldx, C, m, codes, nblocks, S, xm);
            return cudaGetLastError();
        }
    }
    if (vec && (L == 8 || L == 16) && (ldx % 8) == 0 && (reinterpret_cast<uintptr_t>(X) & 31) == 0) {
        static_assert(kEnc2RowsPerBlock == kEncRowsPerBlock, "same 64-group staging");
        const bool small = blocks < 2 * sms;  // halve the blocks' rows so that every SM gets work
        auto kern = L == 8 ? (small ? encode_l8_kernel<8, 128> : encode_l8_kernel<8, 256>)
                           : (small ? encode_l8_kernel<16, 128> : encode_l8_kernel<16, 256>);
        const int threads = small ? 128 : 256;
        const int64_t nb = ceil_div(n, (int64_t)threads * kEnc2Rows);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<(unsigned)nb, threads, smem, s>>>(X, n, ldx, C, m, codes);
    } else if (vec) {
        cudaFuncSetAttribute(encode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        encode_kernel<true><<<(unsigned)blocks, kEncThreads, smem, s>>>(X, n, j, ldx, C, m, codes);
    } else {
        cudaFuncSetAttribute(encode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        encode_kernel<false><<<(unsigned)blocks, kEncThreads, smem, s>>>(X, n, j, ldx, C, m, codes);
    }
    return cudaGetLastError();
}

// Streaming append: the h < 8 rows that complete a partial layout-v1 group.
// Thread c encodes codebook c of those rows with encode_kernel's scalar
// arithmetic (x + (-c), then fma; ascending dimensions; lowest index on
// ties) and rewrites the group's word c keeping the nibbles below `pos`.
__global__ void append_head_kernel(const float* __restrict__ X, int h, int j, int64_t ldx,
                                   const float* __restrict__ C, int m, uint32_t* __restrict__ word, int pos) {
    const int c = threadIdx.x;
    if (c >= m) return;
    const int L = j / m;
    uint32_t bits = 0;
    for (int r = 0; r < h; ++r) {
        const float* x = X + (int64_t)r * ldx + c * L;
        float best = 0.f;
        uint32_t arg = 0;
        for (int k = 0; k < kK; ++k) {
            const float* cc = C + ((int64_t)c * kK + k) * L;
            float d = 0.f;
            for (int t = 0; t < L; ++t) {
                const float diff = __fadd_rn(x[t], -cc[t]);
                d = __fmaf_rn(diff, diff, d);
            }
            if (k == 0 || d < best) { best = d; arg = (uint32_t)k; }
        }
        bits |= arg << (4 * (pos + r));
    }
    const uint32_t keep = pos == 0 ? 0u : (0xFFFFFFFFu >> (32 - 4 * pos));
    word[c] = (word[c] & keep) | bits;
}

cudaError_t launch_encode_append(const float* X, int64_t n_new, int j, int64_t ldx, const float* C, int m,
                                 uint32_t* codes, int64_t n_old, int sms, cudaStream_t s) {
    if (n_new == 0) return cudaSuccess;
    const int pos = (int)(n_old % kRowsPerWord);
    const int64_t h = pos == 0 ? 0 : min64(kRowsPerWord - pos, n_new);
    if (h > 0) {
        append_head_kernel<<<1, ((m + 31) / 32) * 32, 0, s>>>(X, (int)h, j, ldx, C, m,
                                                               codes + (n_old / kRowsPerWord) * m, pos);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (n_new == h) return cudaSuccess;
    return launch_encode(X + h * ldx, n_new - h, j, ldx, C, m, codes + ((n_old + h) / kRowsPerWord) * m, sms, s, 0);
}

cudaError_t launch_pack(const uint8_t* flat, int64_t n, int m, uint32_t* codes, cudaStream_t s) {
    int64_t total = ceil_div(n, kRowsPerWord) * m;
    if (total == 0) return cudaSuccess;
    pack_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, s>>>(flat, n, m, codes);
    return cudaGetLastError();
}

cudaError_t launch_unpack(const uint32_t* codes, int64_t n, int m, uint8_t* flat, cudaStream_t s) {
    int64_t total = n * m;
    if (total == 0) return cudaSuccess;
    unpack_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, s>>>(codes, n, m, flat);
    return cudaGetLastError();
}

}  // namespace bolt
