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
// <= g(L)||c_k||^2, so |s^_k - s_k| <= E = 4 g(L)(C2 + 2 AX) with C2 >= max_k
// n_k and AX = sum_t |x_t| max_k |c_kt|.  The direct fp32 distance errs by
// <= g(L+2) d_k.  With b1 = min_k s^_k and every other s^_k >= b1 + need,
// need = 2.5 E + 3 g(L+2)(X2 + |b1| + E) (X2 >= ||x||^2), the direct
// distances keep the same unique minimum.  The factors carry a >= 25 % slack
// for the rounding of the test itself.
//
// The kernel stages the row slices of a codebook in shared memory by 2-D
// tensor copies (one 256-row x 32-byte box per half block) instead of
// register loads (a register-loading version of the same arithmetic ran at
// 0.24 ms on c2, its loads exposed; ncu profiles/r2/ncu_full_enc_*.txt).
// Warp 8 issues the copies kEncStages slices ahead; warps 0-7 (thread t =
// local rows t and t + 256) rank the centroids and pack the layout-v1 words
// with shuffles.  Measured c2: 0.205 ms against the direct kernel's 0.199 --
// no faster, so it is the explicit variant, not the default.
constexpr int kEncStages = 4;
constexpr int kTmaRows = 512;               // rows per block
constexpr int kTmaWorkers = 256;            // compute threads (2 rows each)

template <int L>
__global__ void __launch_bounds__(kTmaWorkers + 32, 2)
encode_tma_kernel(const __grid_constant__ CUtensorMap xmap, const float* __restrict__ X, int64_t n, int64_t ldx,
                  const float* __restrict__ C, int m, uint32_t* __restrict__ codes) {
    static_assert(L == 8, "32-byte row slices");
    extern __shared__ __align__(1024) uint8_t enc_tma_smem[];
    constexpr float kU = 5.9604645e-8f;  // 2^-24
    constexpr float kGL = (float)L * kU / (1.0f - (float)L * kU);
    constexpr float kGL2 = (float)(L + 2) * kU / (1.0f - (float)(L + 2) * kU);
    constexpr int SLICE = kTmaRows * L * 4;  // bytes of one codebook's row slices
    const int j = m * L;
    float* xs = reinterpret_cast<float*>(enc_tma_smem);                 // [S][512][L]
    float* cneg = xs + kEncStages * kTmaRows * L;                        // [m][L][16] -c
    float* cm2 = cneg + (size_t)j * kK;                                  // [m][L][16] -2c
    float* cn = cm2 + (size_t)j * kK;                                    // [m][16]
    float* amax = cn + (size_t)m * kK;                                   // [m][L]
    float* c2max = amax + (size_t)j;                                     // [m]
    uint32_t* stage = reinterpret_cast<uint32_t*>(c2max + ((m + 3) & ~3));  // [64][m]
    uint64_t* full = reinterpret_cast<uint64_t*>(stage + (size_t)(kTmaRows / kRowsPerWord) * m + 2);  // 8 B aligned
    full = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(full) + 7) & ~uintptr_t(7));
    uint64_t* empty = full + kEncStages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t row_blk = (int64_t)blockIdx.x * kTmaRows;
    if (tid == 0) {
        for (int i = 0; i < kEncStages; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], kTmaWorkers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // centroid tables (all threads), before the copy warp enters its loop: a
    // block barrier after that point would deadlock against its empty-slot waits
    for (int e = tid; e < j * kK; e += blockDim.x) {
        int c = e / (kK * L);
        int r = e - c * kK * L;
        int k = r / L;
        int d = r - k * L;
        cneg[((size_t)c * L + d) * kK + k] = -C[e];
        cm2[((size_t)c * L + d) * kK + k] = -2.0f * C[e];
    }
    for (int e = tid; e < m * kK; e += blockDim.x) {
        const float* ck = C + (size_t)e * L;
        float acc = 0.f;
        for (int t = 0; t < L; ++t) acc = __fmaf_rn(ck[t], ck[t], acc);
        cn[e] = acc;
    }
    for (int e = tid; e < j; e += blockDim.x) {
        const int c = e / L, t = e - c * L;
        float a = 0.f;
        for (int k = 0; k < kK; ++k) a = fmaxf(a, fabsf(C[((size_t)c * kK + k) * L + t]));
        amax[e] = a;
    }
    __syncthreads();
    for (int c = tid; c < m; c += blockDim.x) {
        float a = 0.f;
        for (int k = 0; k < kK; ++k) a = fmaxf(a, fabsf(cn[c * kK + k]));
        c2max[c] = a * (1.0f + 2.0f * kGL);
    }
    __syncthreads();
    if (warp == kTmaWorkers / 32) {
        // ------------------------------------------------ copy warp
        if (lane == 0) {
            for (int c = 0; c < m; ++c) {
                const int s = c % kEncStages;
                tc::mbar_wait(&empty[s], ((c / kEncStages) & 1) ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(&full[s])),
                             "r"(SLICE)
                             : "memory");
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                            "r"(tc::smem_u32(xs + ((size_t)s * kTmaRows + h * 256) * L)),
                        "l"(&xmap), "r"(c * L), "r"((int)(row_blk + h * 256)), "r"(tc::smem_u32(&full[s]))
                        : "memory");
            }
        }
        return;
    }
    // ---------------------------------------------------- compute warps
    uint64_t amb[2] = {0ull, 0ull};
    const bool valid[2] = {row_blk + tid < n, row_blk + tid + 256 < n};
    for (int c = 0; c < m; ++c) {
        const int s = c % kEncStages;
        tc::mbar_wait(&full[s], (c / kEncStages) & 1);
        float xv[2][L];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const float4* xp = reinterpret_cast<const float4*>(xs + ((size_t)s * kTmaRows + tid + 256 * r) * L);
            const float4 a0 = xp[0], a1 = xp[1];
            xv[r][0] = a0.x; xv[r][1] = a0.y; xv[r][2] = a0.z; xv[r][3] = a0.w;
            xv[r][4] = a1.x; xv[r][5] = a1.y; xv[r][6] = a1.z; xv[r][7] = a1.w;
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[s]);  // the slice is in registers
        float2 sv[2][kK / 2];
        float2 xa[2];
        {
            const float4* cn4 = reinterpret_cast<const float4*>(cn + c * kK);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 v = cn4[q];
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    sv[r][2 * q] = make_float2(v.x, v.y);
                    sv[r][2 * q + 1] = make_float2(v.z, v.w);
                }
            }
            xa[0] = xa[1] = make_float2(0.f, 0.f);
        }
        const float* cc = cm2 + (size_t)c * L * kK;
        const float* am = amax + c * L;
#pragma unroll
        for (int t = 0; t < L; ++t) {
            const float4* cv = reinterpret_cast<const float4*>(cc + (size_t)t * kK);
            const float at = am[t];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float4 c4 = cv[q];
                float2 ca = make_float2(c4.x, c4.y), cb = make_float2(c4.z, c4.w);
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    float2 xx = make_float2(xv[r][t], xv[r][t]);
                    sv[r][2 * q] = __ffma2_rn(xx, ca, sv[r][2 * q]);
                    sv[r][2 * q + 1] = __ffma2_rn(xx, cb, sv[r][2 * q + 1]);
                }
            }
#pragma unroll
            for (int r = 0; r < 2; ++r)
                xa[r] = __ffma2_rn(make_float2(xv[r][t], fabsf(xv[r][t])), make_float2(xv[r][t], at), xa[r]);
        }
        const float c2 = c2max[c];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            float mn[kK / 2];
#pragma unroll
            for (int p = 0; p < kK / 2; ++p) mn[p] = fminf(sv[r][p].x, sv[r][p].y);
#pragma unroll
            for (int w = kK / 4; w >= 1; w /= 2)
#pragma unroll
                for (int p = 0; p < w; ++p) mn[p] = fminf(mn[p], mn[p + w]);
            const float b1 = mn[0];
            const float E = 4.0f * kGL * (c2 + 2.0f * xa[r].y * (1.0f + 2.0f * kGL));
            const float need = 2.5f * E + 3.0f * kGL2 * (xa[r].x * (1.0f + 2.0f * kGL) + fabsf(b1) + E);
            const float thr = b1 + need;
            uint32_t bl[kK / 2];
#pragma unroll
            for (int p = 0; p < kK / 2; ++p)
                bl[p] = ((sv[r][p].x < thr ? 1u : 0u) | (sv[r][p].y < thr ? 2u : 0u)) << (2 * p);
#pragma unroll
            for (int w = kK / 4; w >= 1; w /= 2)
#pragma unroll
                for (int p = 0; p < w; ++p) bl[p] |= bl[p + w];
            const uint32_t below = bl[0];
            uint32_t arg = __ffs(below) - 1;
            if (__popc(below) != 1 && valid[r]) amb[r] |= 1ull << c;
            if (!valid[r]) arg = 0;
            // layout-v1 word of this row's group: 8 consecutive lanes hold its 8 rows
            uint32_t v = (arg & 0xFu) << (4 * (tid & 7));
            v |= __shfl_xor_sync(0xffffffffu, v, 1);
            v |= __shfl_xor_sync(0xffffffffu, v, 2);
            v |= __shfl_xor_sync(0xffffffffu, v, 4);
            if ((tid & 7) == 0) stage[((tid + 256 * r) >> 3) * m + c] = v;
        }
    }
    // ambiguous (row, codebook) slices: direct differences, patched into the staged words
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        while (amb[r]) {
            const int c = __ffsll((long long)amb[r]) - 1;
            amb[r] &= amb[r] - 1;
            const uint32_t arg = direct_argmin<L>(X + (row_blk + tid + 256 * r) * ldx + c * L, cneg + (size_t)c * L * kK);
            const int pos = 4 * (tid & 7);
            uint32_t* w = stage + ((tid + 256 * r) >> 3) * m + c;
            atomicAnd(w, ~(0xFu << pos));
            atomicOr(w, arg << pos);
        }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kTmaWorkers) : "memory");
    const int64_t g0 = (int64_t)blockIdx.x * (kTmaRows / kRowsPerWord);
    const int64_t groups = ceil_div(n, kRowsPerWord);
    const int64_t ng = min64(kTmaRows / kRowsPerWord, groups - g0);
    uint32_t* dst = codes + g0 * m;
    for (int64_t e = tid; e < ng * m; e += kTmaWorkers) dst[e] = stage[e];
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
    if (mode == 2 && L == 8 && (ldx % 4) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 && encode_tiled()) {
        // TMA-staged expanded-distance kernel (bit-identical codes)
        CUtensorMap xmap{};
        const cuuint64_t dims[2] = {(cuuint64_t)j, (cuuint64_t)n};
        const cuuint64_t strides[1] = {(cuuint64_t)(ldx * sizeof(float))};
        const cuuint32_t box[2] = {(cuuint32_t)L, 256u};
        const cuuint32_t estr[2] = {1u, 1u};
        if (encode_tiled()(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
            const size_t tsmem = (size_t)kEncStages * kTmaRows * L * sizeof(float) + 2 * (size_t)j * kK * sizeof(float) +
                                 (size_t)m * kK * sizeof(float) + (size_t)j * sizeof(float) +
                                 (size_t)((m + 3) & ~3) * sizeof(float) +
                                 ((size_t)(kTmaRows / kRowsPerWord) * m + 2) * sizeof(uint32_t) + 8 +
                                 2 * kEncStages * sizeof(uint64_t);
            cudaFuncSetAttribute(encode_tma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
            encode_tma_kernel<8><<<(unsigned)ceil_div(n, kTmaRows), kTmaWorkers + 32, tsmem, s>>>(xmap, X, n, ldx, C, m,
                                                                                                codes);
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
