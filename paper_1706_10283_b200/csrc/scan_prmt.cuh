// scan_prmt.cu -- d^: the Bolt scan on CUDA cores with PRMT byte permutes.
//
// PAPER.md L264 performs "V lookups for V consecutive h(x)" with an in-register
// 16-entry byte shuffle (vpshufb).  The sm_100a analogue used here is PRMT:
// one PRMT looks up 4 rows' codes (4 selector nibbles) in an 8-byte table
// {hi, lo}.  A 16-entry u8 table is split by nibble -- lo4[i] = beta[i] & 15,
// hi4[i] = beta[i] >> 4 -- so every table byte is < 128.  Then
//   PRMT(T0, T1, w)          returns T[c]   for codes c < 8, and 0 for c >= 8
//   PRMT(T2, T3, w ^ 0x8888) returns T[c]   for codes c >= 8, and 0 for c < 8
// because a selector nibble with bit 3 set replicates the (zero) sign bit of
// the addressed byte.  The two results are simply added, and because every
// lookup is <= 15 the four byte lanes can accumulate 16 codebooks without
// overflow.  Every 16 codebooks the byte sums are widened into packed u16
// pairs: acc = lo_sum + 16 * hi_sum, exact for M <= 64 (<= 16320, R11).
//
// Cost per (query, codebook, 8 rows): 8 PRMT + 4 IADD3 (+ 2 broadcast LDS.128
// of the split table), i.e. 1.5 integer instructions per lookup.
//
// Layout v1 (R12): lane = one group of 8 rows, word c holds codebook c.
#pragma once
#include "common.cuh"
#include "topk_list.cuh"

namespace bolt {
namespace pscan {

inline int pick_qt(int64_t nq) { return nq >= 8 ? 8 : nq >= 4 ? 4 : nq >= 2 ? 2 : 1; }

constexpr int kScanThreads = 128;   // 4 warps
constexpr int kWarps = kScanThreads / 32;
constexpr int kChunk = 16;          // codebooks per byte-accumulation chunk

// Split quantized tables of queries [q0, q0+qt) into nibble tables in smem:
// tab[(ql*m + c)*2 + 0] = lo4 (uint4: bytes 0-15), [...+1] = hi4.
__device__ __forceinline__ void load_split_tables(const uint8_t* __restrict__ qluts, int64_t nq,
                                                  int m, int64_t q0, int qt, uint4* tab) {
    for (int e = threadIdx.x; e < qt * m; e += blockDim.x) {
        int ql = e / m;
        int c = e - ql * m;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (q0 + ql < nq) v = __ldg(reinterpret_cast<const uint4*>(qluts + ((q0 + ql) * m + c) * kK));
        uint4 lo = make_uint4(v.x & 0x0F0F0F0Fu, v.y & 0x0F0F0F0Fu, v.z & 0x0F0F0F0Fu, v.w & 0x0F0F0F0Fu);
        uint4 hi = make_uint4((v.x >> 4) & 0x0F0F0F0Fu, (v.y >> 4) & 0x0F0F0F0Fu,
                              (v.z >> 4) & 0x0F0F0F0Fu, (v.w >> 4) & 0x0F0F0F0Fu);
        tab[2 * e] = lo;
        tab[2 * e + 1] = hi;
    }
}

// Load up to kChunk code words of group g starting at codebook c0.
__device__ __forceinline__ void load_words(const uint32_t* __restrict__ codes, int64_t g, int m,
                                           int c0, int cn, bool vec, uint32_t (&w)[kChunk]) {
    const uint32_t* p = codes + g * m + c0;
    if (vec) {
#pragma unroll
        for (int t = 0; t < kChunk / 4; ++t) {
            if (4 * t < cn) {
                uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + t);
                w[4 * t] = v.x; w[4 * t + 1] = v.y; w[4 * t + 2] = v.z; w[4 * t + 3] = v.w;
            } else {
                w[4 * t] = w[4 * t + 1] = w[4 * t + 2] = w[4 * t + 3] = 0;
            }
        }
    } else {
#pragma unroll
        for (int t = 0; t < kChunk; ++t) w[t] = t < cn ? __ldg(p + t) : 0u;
    }
}

// Accumulate one chunk of codebooks for QT queries into packed u16 totals
// tot[q][0..3] = rows (0,2), (1,3), (4,6), (5,7).
template <int QT>
__device__ __forceinline__ void scan_chunk(const uint32_t (&w)[kChunk], int cn, int c0, int m,
                                           const uint4* __restrict__ tab, uint32_t (&tot)[QT][4]) {
#pragma unroll
    for (int q = 0; q < QT; ++q) {
        uint32_t aL0 = 0, aH0 = 0, aL1 = 0, aH1 = 0;
#pragma unroll
        for (int t = 0; t < kChunk; ++t) {
            if (t < cn) {
                const uint32_t s0 = w[t];
                const uint32_t x0 = s0 ^ 0x88888888u;
                const uint32_t s1 = s0 >> 16;
                const uint32_t x1 = x0 >> 16;
                const uint4 lo = tab[2 * (q * m + c0 + t)];
                const uint4 hi = tab[2 * (q * m + c0 + t) + 1];
                aL0 += prmt(lo.x, lo.y, s0) + prmt(lo.z, lo.w, x0);
                aH0 += prmt(hi.x, hi.y, s0) + prmt(hi.z, hi.w, x0);
                aL1 += prmt(lo.x, lo.y, s1) + prmt(lo.z, lo.w, x1);
                aH1 += prmt(hi.x, hi.y, s1) + prmt(hi.z, hi.w, x1);
            }
        }
        tot[q][0] += (aL0 & 0x00FF00FFu) + ((aH0 & 0x00FF00FFu) << 4);
        tot[q][1] += ((aL0 >> 8) & 0x00FF00FFu) + (((aH0 >> 8) & 0x00FF00FFu) << 4);
        tot[q][2] += (aL1 & 0x00FF00FFu) + ((aH1 & 0x00FF00FFu) << 4);
        tot[q][3] += ((aL1 >> 8) & 0x00FF00FFu) + (((aH1 >> 8) & 0x00FF00FFu) << 4);
    }
}

template <int QT>
__device__ __forceinline__ void scan_group_rt(const uint32_t* __restrict__ codes, int64_t g, int m,
                                              bool vec, const uint4* __restrict__ tab,
                                              uint32_t (&tot)[QT][4]) {
#pragma unroll
    for (int q = 0; q < QT; ++q) tot[q][0] = tot[q][1] = tot[q][2] = tot[q][3] = 0;
    for (int c0 = 0; c0 < m; c0 += kChunk) {
        const int cn = min(kChunk, m - c0);
        uint32_t w[kChunk];
        load_words(codes, g, m, c0, cn, vec, w);
        scan_chunk<QT>(w, cn, c0, m, tab, tot);
    }
}

// Compile-time M (multiple of 4): codebook-outer / query-inner so that the
// selectors of a word are computed once for all QT queries, with no
// predication in the fully unrolled body.
template <int QT, int M>
__device__ __forceinline__ void scan_group_ct(const uint32_t* __restrict__ codes, int64_t g,
                                              const uint4* __restrict__ tab, uint32_t (&tot)[QT][4]) {
    static_assert(M % 4 == 0, "compile-time M must be a multiple of 4");
    constexpr int NCH = (M + kChunk - 1) / kChunk;
    const uint4* p = reinterpret_cast<const uint4*>(codes + g * M);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        constexpr int CN0 = M < kChunk ? M : kChunk;
        uint32_t w[kChunk];
#pragma unroll
        for (int t = 0; t < CN0 / 4; ++t) {
            const uint4 v = __ldg(p + ch * (kChunk / 4) + t);
            w[4 * t] = v.x; w[4 * t + 1] = v.y; w[4 * t + 2] = v.z; w[4 * t + 3] = v.w;
        }
        uint32_t aL0[QT], aH0[QT], aL1[QT], aH1[QT];
#pragma unroll
        for (int q = 0; q < QT; ++q) aL0[q] = aH0[q] = aL1[q] = aH1[q] = 0;
#pragma unroll
        for (int t = 0; t < CN0; ++t) {
            const uint32_t s0 = w[t];
            const uint32_t x0 = s0 ^ 0x88888888u;
            const uint32_t s1 = s0 >> 16;
            const uint32_t x1 = x0 >> 16;
#pragma unroll
            for (int q = 0; q < QT; ++q) {
                const uint4 lo = tab[2 * (q * M + ch * kChunk + t)];
                const uint4 hi = tab[2 * (q * M + ch * kChunk + t) + 1];
                aL0[q] += prmt(lo.x, lo.y, s0) + prmt(lo.z, lo.w, x0);
                aH0[q] += prmt(hi.x, hi.y, s0) + prmt(hi.z, hi.w, x0);
                aL1[q] += prmt(lo.x, lo.y, s1) + prmt(lo.z, lo.w, x1);
                aH1[q] += prmt(hi.x, hi.y, s1) + prmt(hi.z, hi.w, x1);
            }
        }
#pragma unroll
        for (int q = 0; q < QT; ++q) {
            const uint32_t f0 = (aL0[q] & 0x00FF00FFu) + ((aH0[q] & 0x00FF00FFu) << 4);
            const uint32_t f1 = ((aL0[q] >> 8) & 0x00FF00FFu) + (((aH0[q] >> 8) & 0x00FF00FFu) << 4);
            const uint32_t f2 = (aL1[q] & 0x00FF00FFu) + ((aH1[q] & 0x00FF00FFu) << 4);
            const uint32_t f3 = ((aL1[q] >> 8) & 0x00FF00FFu) + (((aH1[q] >> 8) & 0x00FF00FFu) << 4);
            if (ch == 0) {
                tot[q][0] = f0; tot[q][1] = f1; tot[q][2] = f2; tot[q][3] = f3;
            } else {
                tot[q][0] += f0; tot[q][1] += f1; tot[q][2] += f2; tot[q][3] += f3;
            }
        }
    }
}

// MC = 0: runtime m; otherwise m == MC at compile time.
template <int QT, int MC>
__device__ __forceinline__ void scan_group(const uint32_t* __restrict__ codes, int64_t g, int m,
                                           bool vec, const uint4* __restrict__ tab,
                                           uint32_t (&tot)[QT][4]) {
    if constexpr (MC == 0)
        scan_group_rt<QT>(codes, g, m, vec, tab, tot);
    else
        scan_group_ct<QT, MC>(codes, g, tab, tot);
}

// value of row r (0..7) from the packed totals
__device__ __forceinline__ uint32_t row_value(const uint32_t (&t)[4], int r) {
    const uint32_t pair = t[(r >> 2) * 2 + (r & 1)];
    return (r & 2) ? (pair >> 16) : (pair & 0xFFFFu);
}

// ------------------------------------------------------------ full output
template <int QT, int MC, bool kDequant>
__global__ void __launch_bounds__(kScanThreads)
scan_full_kernel(ScanArgs a, uint16_t* __restrict__ out16, float* __restrict__ out32, int64_t ldo,
                 float inv_a, float b_sum) {
    extern __shared__ uint4 full_tab[];
    const int64_t q0 = (int64_t)blockIdx.y * QT;
    load_split_tables(a.qluts, a.nq, a.m, q0, QT, full_tab);
    __syncthreads();
    const int64_t g = (int64_t)blockIdx.x * kScanThreads + threadIdx.x;
    if (g >= a.groups) return;
    const bool vec = (a.m % 4) == 0;
    uint32_t tot[QT][4];
    scan_group<QT, MC>(a.codes, g, a.m, vec, full_tab, tot);
    const int qn = (int)min64(QT, a.nq - q0);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int64_t i = g * 8 + r;
        if (i >= a.n) break;
        if (kDequant) {
            float* o = out32 + i * ldo + q0;
#pragma unroll
            for (int q = 0; q < QT; ++q)
                if (q < qn) o[q] = fmaf((float)row_value(tot[q], r), inv_a, b_sum);
        } else {
            uint16_t* o = out16 + i * ldo + q0;
#pragma unroll
            for (int q = 0; q < QT; ++q)
                if (q < qn) o[q] = (uint16_t)row_value(tot[q], r);
        }
    }
}

// ---------------------------------------------------------------- top-k
// One group-scan step of the top-k kernel: compile-time M, loop over pairs of
// codebooks (one 8-byte load of the lane's two code words, prefetched one
// iteration ahead), QT queries unrolled inside.  The loop body is kept small
// (about 230 instructions) so it stays in the instruction cache.  With
// kImad the byte accumulations run on the FMA pipe (IMAD with a runtime 1)
// so that the ALU pipe only carries the PRMTs.
__device__ __forceinline__ uint32_t add2(uint32_t acc, uint32_t p, uint32_t q, uint32_t one, bool imad) {
    if (imad) {
        uint32_t d;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(p), "r"(one), "r"(acc));
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(q), "r"(one), "r"(d));
        return d;
    }
    return acc + p + q;
}

template <int QT, int M, bool kImad>
__device__ __forceinline__ void scan_group_loop(const uint2* __restrict__ wp, const uint4* __restrict__ tab,
                                                uint32_t one, uint32_t (&tot)[QT][4]) {
    uint32_t aL0[QT], aH0[QT], aL1[QT], aH1[QT];
#pragma unroll
    for (int q = 0; q < QT; ++q) {
        aL0[q] = aH0[q] = aL1[q] = aH1[q] = 0;
        tot[q][0] = tot[q][1] = tot[q][2] = tot[q][3] = 0;
    }
    uint2 wn = __ldg(wp);
#pragma unroll 1
    for (int t = 0; t < M; t += 2) {
        const uint2 w = wn;
        if (t + 2 < M) wn = __ldg(wp + (t >> 1) + 1);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t s0 = h ? w.y : w.x;
            const uint32_t x0 = s0 ^ 0x88888888u;
            const uint32_t s1 = s0 >> 16;
            const uint32_t x1 = x0 >> 16;
            const uint4* tp = tab + 2 * (t + h);
#pragma unroll
            for (int q = 0; q < QT; ++q) {
                const uint4 lo = tp[2 * q * M];
                const uint4 hi = tp[2 * q * M + 1];
                aL0[q] = add2(aL0[q], prmt(lo.x, lo.y, s0), prmt(lo.z, lo.w, x0), one, kImad);
                aH0[q] = add2(aH0[q], prmt(hi.x, hi.y, s0), prmt(hi.z, hi.w, x0), one, kImad);
                aL1[q] = add2(aL1[q], prmt(lo.x, lo.y, s1), prmt(lo.z, lo.w, x1), one, kImad);
                aH1[q] = add2(aH1[q], prmt(hi.x, hi.y, s1), prmt(hi.z, hi.w, x1), one, kImad);
            }
        }
        if (((t + 2) & (kChunk - 1)) == 0 || t + 2 == M) {
#pragma unroll
            for (int q = 0; q < QT; ++q) {
                tot[q][0] += (aL0[q] & 0x00FF00FFu) + ((aH0[q] & 0x00FF00FFu) << 4);
                tot[q][1] += ((aL0[q] >> 8) & 0x00FF00FFu) + (((aH0[q] >> 8) & 0x00FF00FFu) << 4);
                tot[q][2] += (aL1[q] & 0x00FF00FFu) + ((aH1[q] & 0x00FF00FFu) << 4);
                tot[q][3] += ((aL1[q] >> 8) & 0x00FF00FFu) + (((aH1[q] >> 8) & 0x00FF00FFu) << 4);
                aL0[q] = aH0[q] = aL1[q] = aH1[q] = 0;
            }
        }
    }
}

// Persistent grid: warp tasks (query tile x row partition) are dealt round
// robin to all resident warps.  Per-warp shared memory: the QT nibble-split
// tables [QT][M][2] uint4 and QT sorted key lists of k entries.
template <int QT, int M, bool kImad>
__global__ void __launch_bounds__(kScanThreads, 4)
topk_prmt_kernel(ScanArgs a, int k, int metric, int64_t index_base, int parts, int64_t gpp, int tiles,
                 uint64_t* __restrict__ part_keys, uint32_t one) {
    extern __shared__ uint4 topk_smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint4* tab = topk_smem + warp * (QT * M * 2);
    uint64_t* lists = reinterpret_cast<uint64_t*>(topk_smem + kWarps * QT * M * 2) + warp * QT * k;
    const uint32_t flip = metric == BOLT_DOT ? 0xFFFFFFFFu : 0u;  // kv = 0xFFFF - acc for dot
    const int64_t ntasks = (int64_t)tiles * parts;
    for (int64_t task = (int64_t)blockIdx.x * kWarps + warp; task < ntasks;
         task += (int64_t)gridDim.x * kWarps) {
        const int tile = (int)(task % tiles);
        const int part = (int)(task / tiles);
        const int64_t q0 = (int64_t)tile * QT;
        __syncwarp();
        for (int e = lane; e < QT * M; e += 32) {
            const int ql = e / M;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (q0 + ql < a.nq) v = __ldg(reinterpret_cast<const uint4*>(a.qluts + ((q0 + ql) * M + (e - ql * M)) * kK));
            tab[2 * e] = make_uint4(v.x & 0x0F0F0F0Fu, v.y & 0x0F0F0F0Fu, v.z & 0x0F0F0F0Fu, v.w & 0x0F0F0F0Fu);
            tab[2 * e + 1] = make_uint4((v.x >> 4) & 0x0F0F0F0Fu, (v.y >> 4) & 0x0F0F0F0Fu,
                                        (v.z >> 4) & 0x0F0F0F0Fu, (v.w >> 4) & 0x0F0F0F0Fu);
        }
        for (int e = lane; e < QT * k; e += 32) lists[e] = ~0ull;
        __syncwarp();
        uint32_t thr[QT];
#pragma unroll
        for (int q = 0; q < QT; ++q) thr[q] = kNotFull;
        const int64_t gbeg = (int64_t)part * gpp;
        const int64_t gend = min64(a.groups, gbeg + gpp);
        for (int64_t gs = gbeg; gs < gend; gs += 32) {
            const int64_t g = gs + lane;
            const bool gvalid = g < gend;
            const uint2* wp = reinterpret_cast<const uint2*>(a.codes + (gvalid ? g : gbeg) * M);
            uint32_t tot[QT][4];
            scan_group_loop<QT, M, kImad>(wp, tab, one, tot);
            const int nrows = gvalid ? (int)min64(8, a.n - g * 8) : 0;
#pragma unroll
            for (int q = 0; q < QT; ++q) {
                bool flag;
                if (thr[q] == kNotFull) {
                    flag = nrows > 0;
                } else {
                    const uint32_t tp = thr[q] | (thr[q] << 16);
                    uint32_t f = 0;
#pragma unroll
                    for (int t = 0; t < 4; ++t) f |= vminu2(tot[q][t] ^ flip, tp) ^ tp;
                    flag = f != 0 && nrows > 0;
                }
                if (__any_sync(0xffffffffu, flag))
                    thr[q] = wl_insert_group(lists + q * k, k, tot[q][0], tot[q][1], tot[q][2], tot[q][3], flip,
                                             nrows, thr[q], (uint64_t)(index_base + g * 8), lane);
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < QT; ++q) {
            if (q0 + q >= a.nq) break;
            uint64_t* dst = part_keys + ((int64_t)part * a.nq + q0 + q) * k;
            for (int p = lane; p < k; p += 32) dst[p] = lists[q * k + p];
        }
    }
}

// Runtime-M fallback (any m): one task per warp of the old non-persistent
// form, used for M not in {8, 16, 32, 64}.
template <int QT>
__global__ void __launch_bounds__(kScanThreads)
topk_prmt_rt_kernel(ScanArgs a, int k, int metric, int64_t index_base, int parts, int64_t gpp, int tiles,
                    uint64_t* __restrict__ part_keys) {
    extern __shared__ uint4 topk_smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int m = a.m;
    uint4* tab = topk_smem + warp * (QT * m * 2);
    uint64_t* lists = reinterpret_cast<uint64_t*>(topk_smem + kWarps * QT * m * 2) + warp * QT * k;
    const uint32_t flip = metric == BOLT_DOT ? 0xFFFFFFFFu : 0u;
    const int64_t ntasks = (int64_t)tiles * parts;
    for (int64_t task = (int64_t)blockIdx.x * kWarps + warp; task < ntasks;
         task += (int64_t)gridDim.x * kWarps) {
        const int tile = (int)(task % tiles);
        const int part = (int)(task / tiles);
        const int64_t q0 = (int64_t)tile * QT;
        __syncwarp();
        for (int e = lane; e < QT * m; e += 32) {
            const int ql = e / m;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (q0 + ql < a.nq) v = __ldg(reinterpret_cast<const uint4*>(a.qluts + ((q0 + ql) * m + (e - ql * m)) * kK));
            tab[2 * e] = make_uint4(v.x & 0x0F0F0F0Fu, v.y & 0x0F0F0F0Fu, v.z & 0x0F0F0F0Fu, v.w & 0x0F0F0F0Fu);
            tab[2 * e + 1] = make_uint4((v.x >> 4) & 0x0F0F0F0Fu, (v.y >> 4) & 0x0F0F0F0Fu,
                                        (v.z >> 4) & 0x0F0F0F0Fu, (v.w >> 4) & 0x0F0F0F0Fu);
        }
        for (int e = lane; e < QT * k; e += 32) lists[e] = ~0ull;
        __syncwarp();
        uint32_t thr[QT];
#pragma unroll
        for (int q = 0; q < QT; ++q) thr[q] = kNotFull;
        const int64_t gbeg = (int64_t)part * gpp;
        const int64_t gend = min64(a.groups, gbeg + gpp);
        const bool vec = (m % 4) == 0;
        for (int64_t gs = gbeg; gs < gend; gs += 32) {
            const int64_t g = gs + lane;
            const bool gvalid = g < gend;
            uint32_t tot[QT][4];
            scan_group_rt<QT>(a.codes, gvalid ? g : gbeg, m, vec, tab, tot);
            const int nrows = gvalid ? (int)min64(8, a.n - g * 8) : 0;
#pragma unroll
            for (int q = 0; q < QT; ++q) {
                bool flag = nrows > 0;
                if (thr[q] != kNotFull) {
                    const uint32_t tp = thr[q] | (thr[q] << 16);
                    uint32_t f = 0;
#pragma unroll
                    for (int t = 0; t < 4; ++t) f |= vminu2(tot[q][t] ^ flip, tp) ^ tp;
                    flag = f != 0 && nrows > 0;
                }
                if (__any_sync(0xffffffffu, flag))
                    thr[q] = wl_insert_group(lists + q * k, k, tot[q][0], tot[q][1], tot[q][2], tot[q][3], flip,
                                             nrows, thr[q], (uint64_t)(index_base + g * 8), lane);
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < QT; ++q) {
            if (q0 + q >= a.nq) break;
            uint64_t* dst = part_keys + ((int64_t)part * a.nq + q0 + q) * k;
            for (int p = lane; p < k; p += 32) dst[p] = lists[q * k + p];
        }
    }
}

template <int QT, int MC>
inline cudaError_t launch_full_t(const ScanArgs& a, uint16_t* out16, float* out32, int64_t ldo, float inv_a,
                          float b_sum, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(a.groups, kScanThreads), (unsigned)ceil_div(a.nq, QT));
    size_t smem = (size_t)QT * a.m * 2 * sizeof(uint4);
    if (out32)
        scan_full_kernel<QT, MC, true><<<grid, kScanThreads, smem, s>>>(a, out16, out32, ldo, inv_a, b_sum);
    else
        scan_full_kernel<QT, MC, false><<<grid, kScanThreads, smem, s>>>(a, out16, out32, ldo, inv_a, b_sum);
    return cudaGetLastError();
}

template <int QT>
cudaError_t launch_full_qt(const ScanArgs& a, uint16_t* out16, float* out32, int64_t ldo, float inv_a,
                           float b_sum, cudaStream_t s) {
    switch (a.m) {
        case 8: return launch_full_t<QT, 8>(a, out16, out32, ldo, inv_a, b_sum, s);
        case 16: return launch_full_t<QT, 16>(a, out16, out32, ldo, inv_a, b_sum, s);
        case 32: return launch_full_t<QT, 32>(a, out16, out32, ldo, inv_a, b_sum, s);
        case 64: return launch_full_t<QT, 64>(a, out16, out32, ldo, inv_a, b_sum, s);
        default: return launch_full_t<QT, 0>(a, out16, out32, ldo, inv_a, b_sum, s);
    }
}

#ifndef BOLT_PRMT_IMAD
#define BOLT_PRMT_IMAD 1
#endif

inline size_t topk_smem_bytes(int qt, int m, int k) {
    return (size_t)kWarps * ((size_t)qt * m * 2 * sizeof(uint4) + (size_t)qt * k * sizeof(uint64_t));
}

template <int QT, int M>
inline cudaError_t launch_topk_t(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                                 uint64_t* part_keys, int sms, cudaStream_t s) {
    const int64_t gpp = ceil_div(a.groups, parts);
    const int tiles = (int)ceil_div(a.nq, QT);
    const int64_t tasks = (int64_t)tiles * parts;
    const size_t smem = topk_smem_bytes(QT, M ? M : a.m, k);
    const int64_t blocks = min64(ceil_div(tasks, kWarps), (int64_t)sms * 4);
    if constexpr (M == 0) {
        cudaFuncSetAttribute(topk_prmt_rt_kernel<QT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        topk_prmt_rt_kernel<QT><<<(unsigned)blocks, kScanThreads, smem, s>>>(a, k, metric, index_base, parts, gpp,
                                                                           tiles, part_keys);
    } else {
        constexpr bool kImad = BOLT_PRMT_IMAD != 0;
        cudaFuncSetAttribute(topk_prmt_kernel<QT, M, kImad>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        topk_prmt_kernel<QT, M, kImad><<<(unsigned)blocks, kScanThreads, smem, s>>>(
            a, k, metric, index_base, parts, gpp, tiles, part_keys, 1u);
    }
    return cudaGetLastError();
}

template <int QT>
inline cudaError_t launch_topk_qt(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                                  uint64_t* part_keys, int sms, cudaStream_t s) {
    switch (a.m) {
        case 8: return launch_topk_t<QT, 8>(a, k, metric, index_base, parts, part_keys, sms, s);
        case 16: return launch_topk_t<QT, 16>(a, k, metric, index_base, parts, part_keys, sms, s);
        case 32: return launch_topk_t<QT, 32>(a, k, metric, index_base, parts, part_keys, sms, s);
        case 64: return launch_topk_t<QT, 64>(a, k, metric, index_base, parts, part_keys, sms, s);
        default: return launch_topk_t<QT, 0>(a, k, metric, index_base, parts, part_keys, sms, s);
    }
}

}  // namespace pscan

// explicit per-QT entry points (one translation unit each)
template <int QT>
cudaError_t prmt_full_entry(const ScanArgs& a, uint16_t* out16, float* out32, int64_t ldo, float inv_a, float b_sum, cudaStream_t s);
template <int QT>
cudaError_t prmt_topk_entry(const ScanArgs& a, int k, int metric, int64_t index_base, int parts, uint64_t* part_keys, int sms, cudaStream_t s);
}  // namespace bolt
