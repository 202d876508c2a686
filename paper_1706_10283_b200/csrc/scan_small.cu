// scan_small.cu -- fused scan + top-k for small query batches (nq < 64):
// the HBM-bound regime of BASELINE north_star ("achieved HBM GB/s ... for
// small query batches").
//
// Same arithmetic as scan_prmt.cuh (PAPER.md L264's in-register 16-entry
// lookup as PRMT on nibble-split tables, exact u16 sums), organised for
// memory-level parallelism: every lane (one 8-row layout-v1 group) holds the
// M code words of its current group AND of its next group in registers, so a
// warp keeps 2 x 32 x 4M bytes of codes in flight; the codebook loop is fully
// unrolled.  Top-k: a warp-private sorted list per query in shared memory
// (topk_list.cuh) plus one shared threshold per query in global memory (the
// best k-th value any warp holds, published with red.max on 0xFFFF - value),
// so that a warp whose own list is still filling already filters with the
// other warps' bound.  The partial lists of all warps are merged by
// launch_merge_many (topk.cu), which keeps only keys within the k-th smallest
// list head.
//
// The ALU pipe carries only the PRMTs and one LOP3 per code word: the
// byte-lane sums, the high-half selectors (word >> 16 as mul.hi by a runtime
// 2^16) and the widening shifts run as IMADs on the FMA pipe (runtime
// constants keep ptxas from turning them back into ALU shifts/adds).
#include "scan_prmt.cuh"

namespace bolt {
namespace small {

constexpr int kThreads = 256;  // 8 warps
constexpr int kWarpsPB = kThreads / 32;
constexpr int kBlocksPerSM = 2;
constexpr int kMaxSlots = 32;  // minima slots per query (k <= 32)
#ifndef BOLT_SMALL_EARLY
#define BOLT_SMALL_EARLY 4  // sweep Q = 2, 4, 8: 0.508, 0.945, 1.752 -> 0.493, 0.920, 1.731 ms (every iteration: Q = 1 0.29 -> 0.44)
#endif

#ifndef BOLT_SMALL_IADD3
#define BOLT_SMALL_IADD3 0
#endif

template <int QT, int M>
__device__ __forceinline__ void load_group(const uint32_t* __restrict__ codes, int64_t g, bool valid,
                                           uint4 (&w)[M / 4]) {
    const uint4* p = reinterpret_cast<const uint4*>(codes + g * M);
#pragma unroll
    for (int i = 0; i < M / 4; ++i) w[i] = valid ? __ldg(p + i) : make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t imul_hi(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// Packed u16 totals tot[q][0..3] = rows (0,2), (1,3), (4,6), (5,7) of the group.
// one = 1, hi16 = 2^16, hi24 = 2^24, sixteen = 16 (runtime values; mul.hi by 2^(32-s) = >> s).
template <int QT, int M>
__device__ __forceinline__ void group_sums(const uint4 (&w)[M / 4], const uint4* __restrict__ tab,
                                           uint32_t one, uint32_t hi16, uint32_t hi24, uint32_t sixteen,
                                           uint32_t (&tot)[QT][4]) {
    constexpr int CH = pscan::kChunk;  // byte lanes hold <= 16 lookups of <= 15
#pragma unroll
    for (int c0 = 0; c0 < M; c0 += CH) {
        uint32_t aL0[QT], aH0[QT], aL1[QT], aH1[QT];
#pragma unroll
        for (int q = 0; q < QT; ++q) aL0[q] = aH0[q] = aL1[q] = aH1[q] = 0;
#pragma unroll
        for (int t = c0; t < c0 + CH && t < M; ++t) {
            const uint4 wv = w[t / 4];
            const uint32_t s0 = (t & 3) == 0 ? wv.x : (t & 3) == 1 ? wv.y : (t & 3) == 2 ? wv.z : wv.w;
            const uint32_t x0 = s0 ^ 0x88888888u;
            const uint32_t s1 = imul_hi(s0, hi16);  // s0 >> 16 on the FMA pipe
            const uint32_t x1 = s1 ^ 0x8888u;        // (s0 ^ 0x88888888) >> 16 on the ALU (balances the pipes)
#pragma unroll
            for (int q = 0; q < QT; ++q) {
                const uint4 lo = tab[2 * (q * M + t)];
                const uint4 hi = tab[2 * (q * M + t) + 1];
#if BOLT_SMALL_IADD3
                // A/B: the two halves' lookups added by one 3-input ALU add each
                // (4 IADD3 instead of 8 FMA-pipe IMADs per code word)
                aL0[q] = aL0[q] + prmt(lo.x, lo.y, s0) + prmt(lo.z, lo.w, x0);
                aH0[q] = aH0[q] + prmt(hi.x, hi.y, s0) + prmt(hi.z, hi.w, x0);
                aL1[q] = aL1[q] + prmt(lo.x, lo.y, s1) + prmt(lo.z, lo.w, x1);
                aH1[q] = aH1[q] + prmt(hi.x, hi.y, s1) + prmt(hi.z, hi.w, x1);
#else
                aL0[q] = imad(prmt(lo.z, lo.w, x0), one, imad(prmt(lo.x, lo.y, s0), one, aL0[q]));
                aH0[q] = imad(prmt(hi.z, hi.w, x0), one, imad(prmt(hi.x, hi.y, s0), one, aH0[q]));
                aL1[q] = imad(prmt(lo.z, lo.w, x1), one, imad(prmt(lo.x, lo.y, s1), one, aL1[q]));
                aH1[q] = imad(prmt(hi.z, hi.w, x1), one, imad(prmt(hi.x, hi.y, s1), one, aH1[q]));
#endif
            }
        }
#pragma unroll
        for (int q = 0; q < QT; ++q) {
            // widen byte lanes: acc = lo + 16 * hi per u16 pair
            const uint32_t f0 = imad(aH0[q] & 0x00FF00FFu, sixteen, aL0[q] & 0x00FF00FFu);
            const uint32_t f1 = imad(imul_hi(aH0[q], hi24) & 0x00FF00FFu, sixteen, imul_hi(aL0[q], hi24) & 0x00FF00FFu);
            const uint32_t f2 = imad(aH1[q] & 0x00FF00FFu, sixteen, aL1[q] & 0x00FF00FFu);
            const uint32_t f3 = imad(imul_hi(aH1[q], hi24) & 0x00FF00FFu, sixteen, imul_hi(aL1[q], hi24) & 0x00FF00FFu);
            if (c0 == 0) {
                tot[q][0] = f0; tot[q][1] = f1; tot[q][2] = f2; tot[q][3] = f3;
            } else {
                tot[q][0] = imad(f0, one, tot[q][0]); tot[q][1] = imad(f1, one, tot[q][1]);
                tot[q][2] = imad(f2, one, tot[q][2]); tot[q][3] = imad(f3, one, tot[q][3]);
            }
        }
    }
}

// One query's packed totals (tab_q = its nibble-split tables [M][2]).
template <int M>
__device__ __forceinline__ void group_sums1(const uint4 (&w)[M / 4], const uint4* __restrict__ tab_q, uint32_t one,
                                            uint32_t hi16, uint32_t hi24, uint32_t sixteen, uint32_t (&tot)[4]) {
    uint32_t t2[1][4];
    group_sums<1, M>(w, tab_q, one, hi16, hi24, sixteen, t2);
#pragma unroll
    for (int i = 0; i < 4; ++i) tot[i] = t2[0][i];
}

// While a warp's list is still filling: the k-th smallest of the 32 lanes'
// group minima.  Those k minima are k distinct rows, so it bounds the k-th
// best key of the warp's rows and only rows at or below it need inserting
// (instead of all 256 rows of the iteration).  0xFFFF if fewer than k lanes
// hold rows.  Bitonic sort of the 32 lane values by shuffles.
__device__ __forceinline__ uint32_t fill_bound(const uint32_t (&t)[4], uint32_t flip, int nrows, int k, int lane) {
    uint32_t mn = 0x10000u;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const uint32_t pair = t[(r >> 2) * 2 + (r & 1)] ^ flip;
        const uint32_t kv = (r & 2) ? (pair >> 16) : (pair & 0xFFFFu);
        if (r < nrows) mn = min(mn, kv);
    }
    uint32_t v = mn;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, v, stride);
            const bool up = ((lane & size) == 0) == ((lane & stride) == 0);
            v = up ? min(v, o) : max(v, o);
        }
    const uint32_t kth = __shfl_sync(0xffffffffu, v, k - 1);
    return kth > 0xFFFFu ? 0xFFFFu : kth;
}

// Block b = (query tile b % tiles, row block b / tiles); its 8 warps scan
// 8 consecutive group ranges.  Each warp keeps one sorted list per query in
// shared memory; at the end the block merges its 8 lists per query into one
// output list (part index b / tiles).  The query loop is rolled and the
// codebook loop unrolled, so the body stays in the instruction cache for
// any QT.  gthr_inv[q] = 0xFFFF - (best k-th value of any warp).
template <int QT, int M>
__global__ void __launch_bounds__(kThreads, kBlocksPerSM)
topk_small_kernel(ScanArgs a, int k, int metric, int64_t index_base, int tiles, int64_t gpw,
                  uint64_t* __restrict__ part_keys, uint32_t* __restrict__ gthr_inv, uint32_t one) {
    extern __shared__ uint4 small_smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int tile = (int)(blockIdx.x % tiles);
    const int64_t blk = blockIdx.x / tiles;  // output list index
    const int64_t q0 = (int64_t)tile * QT;
    uint4* tab = small_smem;  // [QT][M][2], shared by the block
    uint64_t* lists = reinterpret_cast<uint64_t*>(small_smem + QT * M * 2) + warp * QT * k;
    uint32_t* qstate = reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(small_smem + QT * M * 2) +
                                                   kWarpsPB * QT * k) + warp * 3 * QT;  // [QT] pub, shr, pub min
    // minima slots: gslot[q][s] = 0xFFFF - min over the warps of slot s of their
    // best value.  k slots filled by k distinct warps = k distinct rows, so
    // the largest slot value bounds the k-th best key of the union of all
    // warps' rows (much tighter than any single warp's k-th).
    uint32_t* gslot = gthr_inv + a.nq;
    const int myslot = (int)((blk * kWarpsPB + warp) % k);
    const uint32_t flip = metric == BOLT_DOT ? 0xFFFFFFFFu : 0u;  // kv = 0xFFFF - acc for dot (R13)
    for (int e = threadIdx.x; e < QT * M; e += kThreads) {
        const int ql = e / M;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (q0 + ql < a.nq) v = __ldg(reinterpret_cast<const uint4*>(a.qluts + ((q0 + ql) * M + (e - ql * M)) * kK));
        tab[2 * e] = make_uint4(v.x & 0x0F0F0F0Fu, v.y & 0x0F0F0F0Fu, v.z & 0x0F0F0F0Fu, v.w & 0x0F0F0F0Fu);
        tab[2 * e + 1] = make_uint4((v.x >> 4) & 0x0F0F0F0Fu, (v.y >> 4) & 0x0F0F0F0Fu,
                                    (v.z >> 4) & 0x0F0F0F0Fu, (v.w >> 4) & 0x0F0F0F0Fu);
    }
    for (int e = lane; e < QT * k; e += 32) lists[e] = ~0ull;
    for (int q = lane; q < QT; q += 32) {
        qstate[q] = kNotFull;
        qstate[QT + q] = q0 + q < a.nq ? 0xFFFFu - gthr_inv[q0 + q] + 1u : 0u;  // shared bound + 1 (0x10000 = none)
        qstate[2 * QT + q] = kNotFull;
    }
    __syncthreads();
    const int64_t gbeg = (blk * kWarpsPB + warp) * gpw;
    const int64_t gend = min64(a.groups, gbeg + gpw);
    uint4 wnext[M / 4];
    load_group<QT, M>(a.codes, gbeg + lane, gbeg + lane < gend, wnext);
    for (int64_t gs = gbeg; gs < gend; gs += 32) {
        const int64_t g = gs + lane;
        uint4 w[M / 4];
#pragma unroll
        for (int i = 0; i < M / 4; ++i) w[i] = wnext[i];
        load_group<QT, M>(a.codes, g + 32, g + 32 < gend, wnext);
        const int nrows = g < gend ? (int)min64(8, a.n - g * 8) : 0;
        // shared bounds re-read every iteration while they are still loose (the
        // first BOLT_SMALL_EARLY iterations of a warp), then every 8
        const int64_t it = (gs - gbeg) >> 5;
        const bool refresh = it < BOLT_SMALL_EARLY || (it & 7) == 0;
#pragma unroll 1
        for (int q = 0; q < QT; ++q) {
            if (q0 + q >= a.nq) break;
            uint32_t tot[4];
            group_sums1<M>(w, tab + 2 * q * M, one, one << 16, one << 24, one << 4, tot);
            uint64_t* list = lists + q * k;
            uint32_t shr = qstate[QT + q];
            if (refresh) {
                uint32_t gv, sv = 0xFFFFu;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gv) : "l"(gthr_inv + q0 + q));
                if (k <= kMaxSlots) {
                    uint32_t slot = 0;
                    if (lane < k)
                        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(slot)
                                     : "l"(gslot + (q0 + q) * kMaxSlots + lane));
                    sv = lane < k ? 0xFFFFu - slot : 0u;  // empty slot (0) -> 0xFFFF: no bound
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) sv = max(sv, __shfl_xor_sync(0xffffffffu, sv, off));
                }
                shr = min(min(shr, 0xFFFFu - gv + 1u), sv + 1u);
                qstate[QT + q] = shr;
            }
            // candidates: kv <= min(own k-th, shared bound); equal values may
            // still win on index, so the list compares full keys
            const uint32_t own = wl_threshold(list, k);
            uint32_t thr = min(own, shr - 1u);
            if (own == kNotFull && k <= 32) thr = min(thr, fill_bound(tot, flip, nrows, k, lane));
            bool flag = nrows > 0;
            if (thr < 0xFFFFu) {
                const uint32_t tp = (thr + 1) | ((thr + 1) << 16);  // kv <= thr <=> min(kv, thr+1) != thr+1
                uint32_t f = 0;
#pragma unroll
                for (int t = 0; t < 4; ++t) f |= vminu2(tot[t] ^ flip, tp) ^ tp;
                flag = flag && f != 0;
            }
            if (__any_sync(0xffffffffu, flag)) {
                const uint32_t nown = wl_insert_group(list, k, tot[0], tot[1], tot[2], tot[3], flip, nrows, thr,
                                                      (uint64_t)(index_base + g * 8), lane);
                const uint32_t nmin = (uint32_t)(list[0] >> 48);  // list[0] != ~0 after an insert
                if (nown < qstate[q] || (k <= kMaxSlots && nmin < qstate[2 * QT + q])) {
                    __syncwarp();
                    if (lane == 0) {
                        if (nown < qstate[q]) {
                            qstate[q] = nown;
                            asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(gthr_inv + q0 + q),
                                         "r"(0xFFFFu - nown)
                                         : "memory");
                        }
                        if (k <= kMaxSlots && nmin < qstate[2 * QT + q]) {
                            qstate[2 * QT + q] = nmin;
                            asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;"
                                         ::"l"(gslot + (q0 + q) * kMaxSlots + myslot), "r"(0xFFFFu - nmin)
                                         : "memory");
                        }
                    }
                    __syncwarp();
                }
            }
        }
    }
    __syncthreads();
    // block merge: warp w merges query w, w + 8, ... over the 8 warps' lists
    const uint64_t* all = reinterpret_cast<const uint64_t*>(small_smem + QT * M * 2);
    for (int q = warp; q < QT; q += kWarpsPB) {
        if (q0 + q >= a.nq) break;
        uint64_t* dst = part_keys + (blk * a.nq + q0 + q) * k;
        int head[kWarpsPB];  // per list read position, identical in every lane
#pragma unroll
        for (int l = 0; l < kWarpsPB; ++l) head[l] = 0;
        for (int r = 0; r < k; ++r) {
            // lane l < 8 proposes list l's head; warp min (keys are unique)
            uint64_t best = ~0ull;
            int bl = -1;
#pragma unroll
            for (int l = 0; l < kWarpsPB; ++l) {
                const uint64_t h = head[l] < k ? all[(l * QT + q) * k + head[l]] : ~0ull;
                if (h < best) { best = h; bl = l; }
            }
            if (lane == 0) dst[r] = best;
#pragma unroll
            for (int l = 0; l < kWarpsPB; ++l) head[l] += (l == bl);
        }
    }
}

// Queries per block tile: the one with the least padded work, ceil(nq / QT) QT
// queries at a per-query cost measured on 10^8 rows (0.29, 0.255, 0.24, 0.203
// ms for QT = 1, 2, 4, 8; more queries per tile share each code-word load).
inline int pick_qt(int64_t nq) {
    constexpr int qt[4] = {1, 2, 4, 8};
    constexpr double cost[4] = {1.43, 1.26, 1.18, 1.0};
    int best = 1;
    double bc = 1e300;
    for (int i = 0; i < 4; ++i) {
        const double c = (double)ceil_div(nq, qt[i]) * qt[i] * cost[i];
        if (c < bc - 1e-9) { bc = c; best = qt[i]; }
    }
    return best;
}

template <int QT, int M>
cudaError_t launch_qm(const ScanArgs& a, int k, int metric, int64_t index_base, int parts, uint64_t* part_keys,
                      uint32_t* gthr, cudaStream_t s) {
    const int tiles = (int)ceil_div(a.nq, QT);
    const int64_t gpw = ceil_div(ceil_div(a.groups, (int64_t)parts * kWarpsPB), 32) * 32;
    const size_t smem = (size_t)QT * M * 2 * sizeof(uint4) + (size_t)kWarpsPB * QT * k * sizeof(uint64_t) +
                        (size_t)kWarpsPB * 3 * QT * sizeof(uint32_t);
    auto kern = topk_small_kernel<QT, M>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<(unsigned)((int64_t)tiles * parts), kThreads, smem, s>>>(a, k, metric, index_base, tiles, gpw, part_keys,
                                                                   gthr, 1u);
    return cudaGetLastError();
}

template <int QT>
cudaError_t launch_q(const ScanArgs& a, int k, int metric, int64_t index_base, int parts, uint64_t* part_keys,
                     uint32_t* gthr, cudaStream_t s) {
    switch (a.m) {
        case 8: return launch_qm<QT, 8>(a, k, metric, index_base, parts, part_keys, gthr, s);
        case 16: return launch_qm<QT, 16>(a, k, metric, index_base, parts, part_keys, gthr, s);
        case 32: return launch_qm<QT, 32>(a, k, metric, index_base, parts, part_keys, gthr, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace small

int topk_small_supported(int64_t n, int m, int64_t nq, int k) {
    return n >= 1 && nq >= 1 && nq < 64 && k >= 1 && k <= kMaxK && (m == 8 || m == 16 || m == 32);
}

// One output list per block: all blocks resident at once (two per SM),
// split over the query tiles, each warp at least 8 iterations of 32 groups.
int topk_small_parts(int64_t n, int m, int64_t nq, int k, int num_sms) {
    (void)m;
    (void)k;
    const int64_t tiles = ceil_div(nq, small::pick_qt(nq));
    const int64_t blocks = (int64_t)num_sms * small::kBlocksPerSM;
    const int64_t by_work = ceil_div(ceil_div(n, 8), (int64_t)small::kWarpsPB * 32 * 8);
    return (int)max64(1, min64(max64(blocks / tiles, 1), by_work));
}

// part_keys: parts*nq*k keys followed by nq u32 shared thresholds and nq x 32
// u32 minima slots (zeroed here).
cudaError_t launch_topk_small(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                              uint64_t* part_keys, cudaStream_t s) {
    uint32_t* gthr = reinterpret_cast<uint32_t*>(part_keys + (size_t)parts * a.nq * k);
    cudaError_t e = cudaMemsetAsync(gthr, 0, (size_t)a.nq * (1 + small::kMaxSlots) * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    switch (small::pick_qt(a.nq)) {
        case 8: return small::launch_q<8>(a, k, metric, index_base, parts, part_keys, gthr, s);
        case 4: return small::launch_q<4>(a, k, metric, index_base, parts, part_keys, gthr, s);
        case 2: return small::launch_q<2>(a, k, metric, index_base, parts, part_keys, gthr, s);
        default: return small::launch_q<1>(a, k, metric, index_base, parts, part_keys, gthr, s);
    }
}

}  // namespace bolt
