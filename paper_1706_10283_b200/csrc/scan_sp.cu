// scan_sp.cu -- the Bolt scan + fused top-k as a 2:4-SPARSE tcgen05
// contraction (sm_100a).
//
// The scan sum acc(i, q) = sum_c beta[q][c][code(i, c)]
// is the integer product D[i][q] = sum_{c,k} A[i][16c + k] * B[q][16c + k]
// with A = one-hot(codes) and B = the u8 tables.  A one-hot 16-byte
// row has one non-zero, so every group of 4 consecutive K elements holds at
// most one: A is 2:4 structured-sparse, and tcgen05.mma.sp.kind::i8 takes it
// compressed to K/2 bytes plus 4 bits of metadata per group.  A sparse
// instruction covers K = 64 (four codebooks) in the cycles a dense one needs
// for K = 32 (measured: 128 cycles per instruction for a CTA pair, M = 256,
// N = 256, both; profiles/r2/probe_mma_sp.txt), so the contraction runs at
// twice the dense int8 rate.  The sums are the same exact integers as the
// PRMT scan (every product is 0 or a table entry, every sum <= 255 M).
//
// The sparse operand is A, so vectors sit on the MMA's M side and queries on
// N (the orientation of the full-output kernel): a CTA pair (cta_group::2)
// computes 256 vectors (128 per CTA = its TMEM lanes) x kNQ = 224 queries per
// tile; each CTA holds the tables of 112 queries (its half of B) and the
// compressed one-hot of its 128 vectors.  TMEM: two 224-column accumulators
// (448 columns) + the metadata ring (M/2 columns per stage) in the last 64.
//
// Operand encoding (probe: profiles/r2/probe_sp_layout.txt): codebook c of a
// vector covers logical K [16c, 16c + 16) = groups 4c .. 4c + 3; its
// compressed 8 bytes hold two bytes per group, and the group's metadata
// nibble = (idx1 << 2) | idx0 gives the two positions.  For code x the group
// x >> 2 stores value 1 at position x & 3: nibble 0x4 (0,1) / 0x9 (1,2) /
// 0xE (2,3) with the 1 in the first slot, or 0xE with the 1 in the second
// slot for x & 3 == 3; every other group stores (0, 0) with nibble 0x4.
// Metadata of one K = 64 instruction = 64 bits per row = TMEM columns
// (2 ks, 2 ks + 1) of the row's lane, group g at bits 4g.
//
// Warp roles: epilogue 0-7 (warp w: TMEM lane quadrant w % 4 = 32 vectors,
// query half w / 4 = 112 queries, packed u16 pairs in 56 registers),
// producers 8-11 (thread = vector: compressed one-hot into shared memory,
// metadata into TMEM with tcgen05.st), MMA issuer 12 (leader CTA).
//
// Top-k (k <= KMAX <= 32): one sorted list of 32-bit keys (kv' << IDX_BITS |
// local vector index, kv' = acc for L2, 255 M - acc for dot) per (warp,
// query) in shared memory; a warp inserts its candidates warp-cooperatively
// (lane l holds slot l), one query at a time, in lane = vector index order.
// Candidates: kv' < thr(q) = min(own list's k-th value, shared bound + 1);
// the filter is one packed IADD per two queries against per-warp threshold
// words in shared memory (broadcast reads), AND-reduced per lane.  The shared
// bound is the minimum over all lists of the query of their k-th value
// (inverted in a global word, red.max), re-read every 4 tiles.  Lists: 8 per
// query per row partition (2 CTAs x 4 quadrants), merged by merge_many_kernel.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace bolt {
#ifdef BOLT_PROFILE
// diagnostic counters of this kernel (libbolt_prof.so): read through bolt_debug_counters, slots 16..23
__device__ unsigned long long g_sp_counters[16];
#define SP_COUNT(i, v) atomicAdd(&g_sp_counters[(i)], (unsigned long long)(v))
#else
#define SP_COUNT(i, v) ((void)0)
#endif
namespace sp {

using namespace tc;

constexpr int kNQ = 224;                 // queries per MMA tile (N) of the large-batch instantiation
constexpr int kVT = 256;                 // vectors per MMA tile (M, 128 per CTA)
constexpr int kProdWarps = 4;           // thread = vector
constexpr int kProducers = kProdWarps * 32;
constexpr int kEpiWarps = 8;
constexpr int kEpilogue = kEpiWarps * 32;
constexpr int kMmaWarp = kEpiWarps + kProdWarps;  // MMA issuer (leader CTA, one thread)
constexpr int kThreads = (kMmaWarp + 1) * 32;
constexpr int kRefresh = 4;              // tiles between reads of the shared thresholds
constexpr uint32_t kNone = 0x7FFFu;      // "no threshold": every kv' <= 255 * 64 < 0x7FFF
constexpr int kGroupRegs = 8;            // slow-path granularity: 8 registers = 16 queries
constexpr int kScrStride = 9;            // words per thread of the slow-path scratch (odd: conflict-free)

template <int M, int KMAX, int NQ_ = kNQ>
struct Cfg {
    static constexpr int NQ = NQ_;                  // queries per tile (N): 224, or 64 / 32 for small batches
    static constexpr int NQH = NQ / 2;              // query rows of B per CTA
    static constexpr int QW = NQ / 2;               // queries per epilogue warp (column half)
    static constexpr int NR = QW / 2;               // packed registers per epilogue thread
    static constexpr int NG = NR / kGroupRegs;      // slow-path groups of 16 queries per warp
    static constexpr int META0 = 2 * NQ;            // TMEM: accumulators [0, 2 NQ), metadata ring after
    static_assert(QW % 16 == 0 && NR % kGroupRegs == 0, "whole 16-query groups per warp");
    static constexpr int K = 16 * M;                // logical K bytes per row
    static constexpr int KC = 8 * M;                // compressed A bytes per vector
    static constexpr int B_BYTES = NQH * K;        // tables of this CTA's queries
    static constexpr int A_BYTES = 128 * KC;        // one stage: compressed one-hot of 128 vectors
    static constexpr int META_COLS = M / 2;         // TMEM metadata columns per stage
    static constexpr int LIST_BYTES = kEpiWarps * QW * KMAX * 4;
    static constexpr int TQ_BYTES = kEpiWarps * QW * 4;   // per-warp query thresholds (kv')
    static constexpr int NT_BYTES = kEpiWarps * NR * 4;   // per-warp packed filter words
    static constexpr int SCR_BYTES = kEpilogue * kScrStride * 4;  // slow path: one group's sums per thread
    static constexpr int FIXED = B_BYTES + LIST_BYTES + TQ_BYTES + NT_BYTES + SCR_BYTES + 256;
    static constexpr int S_SMEM = (227 * 1024 - FIXED) / A_BYTES;
    static constexpr int S_TMEM = (512 - META0) / META_COLS;
    static constexpr int S0 = S_SMEM < S_TMEM ? S_SMEM : S_TMEM;
    static constexpr int STAGES = S0 > 8 ? 8 : S0;
    static_assert(STAGES >= 2, "no room for a double-buffered stage");
    static constexpr int KSTEPS = M / 4;            // sparse instructions (K = 64) per tile
    static constexpr int VAL_BITS = M <= 8 ? 11 : (M <= 16 ? 12 : 13);
    static constexpr int IDX_BITS = 31 - VAL_BITS;
    static constexpr int64_t MAX_RANGE = int64_t(1) << IDX_BITS;
    static constexpr uint32_t KVMAX = 255u * M;
    static constexpr int A_OFF = B_BYTES;
    static constexpr int LIST_OFF = A_OFF + STAGES * A_BYTES;
    static constexpr int TQ_OFF = LIST_OFF + LIST_BYTES;
    static constexpr int NT_OFF = TQ_OFF + TQ_BYTES;
    static constexpr int SCR_OFF = NT_OFF + NT_BYTES;
    static constexpr int BAR_OFF = SCR_OFF + SCR_BYTES;
    static constexpr int SMEM = BAR_OFF + 256;
    // instruction descriptor: D s32, A/B u8, K-major, N = 224, M = 256, sparse (bit 2)
    static constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(NQ >> 3) << 17) | ((uint32_t)(256 >> 4) << 24) | 4u;
};

__device__ __forceinline__ void mma_sp_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t meta, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(meta)
        : "memory");
}

template <int N>
__device__ __forceinline__ void tmem_st_meta(uint32_t taddr, const uint32_t (&v)[N]) {
    if constexpr (N == 2) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(v[0]), "r"(v[1])
                     : "memory");
    } else if constexpr (N == 4) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]),
                     "r"(v[1]), "r"(v[2]), "r"(v[3])
                     : "memory");
    } else if constexpr (N == 8) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
    } else {
        static_assert(N == 16, "metadata of 4 .. 32 codebooks");
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15, %16};" ::"r"(taddr),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
            : "memory");
    }
}

// Metadata of one codebook's four groups (16 bits) for code x (x = 16: an
// all-zero row): 0x4 everywhere, group x >> 2 gets {0x4, 0x9, 0xE, 0xE}[x & 3].
__device__ __forceinline__ uint32_t meta16(uint32_t x) {
    const uint32_t delta = (0xAAD0u >> (4 * (x & 3))) & 0xFu;  // nibble ^ 0x4
    return (0x4444u ^ (delta << (4 * (x >> 2)))) & 0xFFFFu;
}
// Compressed 8 bytes of one codebook as (lo, hi) words: byte 2 (x >> 2) + (x & 3 == 3) = 1.
__device__ __forceinline__ void comp8(uint32_t x, uint32_t& lo, uint32_t& hi) {
    const uint32_t s = ((x >> 2) << 4) + (((x & 3) + 1) & 4) * 2;  // bit offset of the 1
    lo = shl_clamp(1u, s);
    hi = shl_clamp(1u, s - 32u);
}

// Threshold (kv', exclusive) -> half of a packed filter word: L2 d = p + w
// (bit 15 set <=> p >= thr), dot d = w - p (bit 15 set <=> p <= KVMAX - thr).
template <bool kDot, uint32_t KVMAX>
__device__ __forceinline__ uint32_t filter_half(uint32_t thr) {
    return kDot ? (KVMAX + 0x8000u - thr) : (0x8000u - thr);
}

// Slow path of one group of 16 queries (one compact, non-inlined copy of the
// code: an inlined per-query body made the kernel ~300 KB of SASS and
// thrashed the instruction cache).  scr: this thread's 8 packed sums of the
// group (stride-9 rows, conflict-free), NT / TQ / L: the warp's filter
// words, thresholds and lists; qrem = queries of the warp below nq.
template <typename C, bool kDot, int KMAX>
__device__ __noinline__ void slow_group(const uint32_t* __restrict__ scr, int g, uint32_t vl, bool vvalid, int k,
                                        uint32_t* L, uint32_t* TQ, uint32_t* NT, uint32_t* gthr, int64_t qrem,
                                        int lane) {
    uint32_t m16 = 0;  // candidate bits of the group's 16 queries
#pragma unroll
    for (int j = 0; j < kGroupRegs; ++j) {
        const uint32_t w = NT[kGroupRegs * g + j];
        const uint32_t pv = scr[j];
        const uint32_t d = kDot ? w - pv : pv + w;
        const uint32_t f = ~d & 0x80008000u;
        m16 |= (((f >> 15) & 1u) | (f >> 30)) << (2 * j);
    }
    if (!vvalid) m16 = 0;
    uint32_t u = __reduce_or_sync(0xffffffffu, m16);
    if (lane == 0) SP_COUNT(1, __popc(u));  // (query, warp-tile) pairs with candidates
    while (u) {
        const int b = __ffs(u) - 1;
        u &= u - 1;
        const int q = kGroupRegs * 2 * g + b;  // query of the warp
        uint32_t bal = __ballot_sync(0xffffffffu, (m16 >> b) & 1u);
        if (lane == 0) SP_COUNT(2, __popc(bal));  // candidates
        const uint32_t v = (scr[b >> 1] >> (16 * (b & 1))) & 0xFFFFu;
        const uint32_t key = ((kDot ? C::KVMAX - v : v) << C::IDX_BITS) | vl;
        uint32_t* Lq = L + q * KMAX;
        uint32_t cur = lane < KMAX ? Lq[lane] : 0xFFFFFFFFu;
        bool changed = false;
        while (bal) {
            const int src = __ffs(bal) - 1;
            bal &= bal - 1;
            const uint32_t c = __shfl_sync(0xffffffffu, key, src);
            const uint32_t kth = __shfl_sync(0xffffffffu, cur, k - 1);
            if (c >= kth) continue;  // full key: ties go to the lower index
            const int pos = __popc(__ballot_sync(0xffffffffu, lane < k && cur < c));
            const uint32_t prev = __shfl_up_sync(0xffffffffu, cur, 1);
            cur = lane == pos ? c : ((lane > pos && lane < k) ? prev : cur);
            changed = true;
        }
        if (changed) {
            if (lane < KMAX) Lq[lane] = cur;
            const uint32_t kth = __shfl_sync(0xffffffffu, cur, k - 1);
            if (lane == 0) SP_COUNT(3, 1);  // list changes
            if (kth != 0xFFFFFFFFu && lane == 0) {
                const uint32_t own = kth >> C::IDX_BITS;
                const uint32_t t0 = min(TQ[q], own);
                TQ[q] = t0;
                const int hh = 16 * (q & 1);
                NT[q >> 1] = (NT[q >> 1] & ~(0xFFFFu << hh)) | (filter_half<kDot, C::KVMAX>(t0) << hh);
                if (q < qrem)
                    asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(gthr + q), "r"(0xFFFFu - own)
                                 : "memory");
            }
            __syncwarp();
        }
    }
}

template <int M, bool kDot, int KMAX, int NQ>
__global__ void __launch_bounds__(kThreads, 1)
topk_sp_kernel(ScanArgs a, int k, int64_t index_base, int64_t vpp, int tiles_q, uint64_t* __restrict__ part_keys,
               uint32_t* __restrict__ gthr_inv, int xmode) {
#ifndef BOLT_XMODE
    xmode = 0;  // diagnostic stage switches exist only in libbolt_x.so (tools/)
#endif
    using C = Cfg<M, KMAX, NQ>;
    constexpr int S = C::STAGES;
    constexpr int kNQH = C::NQH, kQW = C::QW, kNR = C::NR, kNG = C::NG, kMetaCol0 = C::META0;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sB = smem;
    uint8_t* sA = smem + C::A_OFF;
    uint32_t* lists_all = reinterpret_cast<uint32_t*>(smem + C::LIST_OFF);
    uint32_t* tq_all = reinterpret_cast<uint32_t*>(smem + C::TQ_OFF);
    uint32_t* nt_all = reinterpret_cast<uint32_t*>(smem + C::NT_OFF);
    uint32_t* scr_all = reinterpret_cast<uint32_t*>(smem + C::SCR_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* tfull = bars + 2 * S;
    uint64_t* tempty = bars + 2 * S + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int unit = (int)(blockIdx.x >> 1);
    const int tq = unit % tiles_q;
    const int part = unit / tiles_q;
    const int64_t qt0 = (int64_t)tq * NQ;            // first query of the tile
    const int64_t q0 = qt0 + rank * kNQH;             // this CTA's B rows
    const int64_t vbeg = (int64_t)part * vpp;
    const int64_t vend = min64(a.n, vbeg + vpp);
    const int ntiles = vend > vbeg ? (int)ceil_div(vend - vbeg, kVT) : 0;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 2 * kProdWarps);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 2 * kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= kEpiWarps && warp < kMmaWarp) {
        // ------------------------------------------------------ producers
        const int t = threadIdx.x - kEpilogue;
        const int v = t;                        // vector v of the CTA's 128 = TMEM lane v
        // B: this CTA's 112 queries, 16-byte unit (c, q) -> c * (112 * 16) + (q / 8) * 128 + (q % 8) * 16
        for (int u = t; u < kNQH * M; u += kProducers) {
            const int c = u / kNQH, q = u % kNQH;
            const bool ok = q0 + q < a.nq;
            const uint8_t* src = a.qluts + ((ok ? q0 + q : 0) * M + c) * kK;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                             smem_u32(sB + c * (kNQH * 16) + (q >> 3) * 128 + (q & 7) * 16)),
                         "l"(src), "r"(ok ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        constexpr int NW4 = M / 4;  // uint4 code-word loads per vector
        const uint32_t sh = (v & 7) * 4;
        const uint32_t tm_meta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + kMetaCol0;
        auto load_words = [&](int tile, uint4 (&w)[NW4]) {
            const int64_t g = (vbeg + (int64_t)tile * kVT + rank * 128 + v) >> 3;
#pragma unroll
            for (int i = 0; i < NW4; ++i)
                w[i] = g < a.groups ? __ldg(reinterpret_cast<const uint4*>(a.codes + g * M) + i) : make_uint4(0, 0, 0, 0);
        };
        auto produce = [&](int tile, const uint4 (&cur)[NW4]) {
            const int s = tile % S;
#ifdef BOLT_PROFILE
            const long long tw0 = clock64();
#endif
            mbar_wait(&empty[s], ((tile / S) & 1) ^ 1);
#ifdef BOLT_PROFILE
            const long long tw1 = clock64();
            if (t == 0) { SP_COUNT(8, tw1 - tw0); SP_COUNT(12, 1); }
#endif
            const bool valid = vbeg + (int64_t)tile * kVT + rank * 128 + v < vend;
            if (xmode & 2) {  // diagnostic: keep the stage's stale operands
                __syncwarp();
                if (lane == 0) {
                    if (rank == 0) mbar_arrive(&full[s]);
                    else mbar_arrive_remote_cta(&full[s], 0);
                }
                return;
            }
            uint8_t* b = sA + s * C::A_BYTES + (v >> 3) * 128 + (v & 7) * 16;
            uint32_t meta[M / 2];
#pragma unroll
            for (int i = 0; i < NW4; ++i) {
                const uint32_t ws[4] = {cur[i].x, cur[i].y, cur[i].z, cur[i].w};
#pragma unroll
                for (int j = 0; j < 4; j += 2) {
                    const uint32_t x0 = valid ? (ws[j] >> sh) & 0xFu : 16u;
                    const uint32_t x1 = valid ? (ws[j + 1] >> sh) & 0xFu : 16u;
                    uint32_t l0, h0, l1, h1;
                    comp8(x0, l0, h0);
                    comp8(x1, l1, h1);
                    const int ch = (4 * i + j) / 2;  // 16-byte chunk = codebooks 2 ch, 2 ch + 1
                    *reinterpret_cast<uint4*>(b + ch * (128 * 16)) = make_uint4(l0, h0, l1, h1);
                    meta[ch] = meta16(x0) | (meta16(x1) << 16);
                }
            }
            fence_proxy_async();
            if (!(xmode & 8)) {  // diagnostic 8: stale metadata (no tcgen05.st)
                tmem_st_meta<M / 2>(tm_meta + s * C::META_COLS, meta);
                tmem_wait_st();
            }
            tc_fence_before();
            __syncwarp();
#ifdef BOLT_PROFILE
            if (t == 0) SP_COUNT(9, clock64() - tw1);
#endif
            if (lane == 0) {
                if (rank == 0) mbar_arrive(&full[s]);
                else mbar_arrive_remote_cta(&full[s], 0);
            }
        };
        constexpr int D = M <= 16 ? 3 : 2;  // tiles of code words in flight
        uint4 pre[D][NW4];
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (j < ntiles) load_words(j, pre[j]);
        for (int t0 = 0; t0 < ntiles; t0 += D) {
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const int tile = t0 + j;
                if (tile < ntiles) {
                    produce(tile, pre[j]);
                    if (tile + D < ntiles) load_words(tile + D, pre[j]);
                }
            }
        }
    } else if (warp < kEpiWarps) {
        // ------------------------------------------------------- epilogue
        const int quad = warp & 3, half = warp >> 2;
        const int64_t qw0 = qt0 + half * kQW;  // first query of this warp
        uint32_t* L = lists_all + warp * kQW * KMAX;  // [112][KMAX]
        uint32_t* TQ = tq_all + warp * kQW;           // [112] thresholds (kv', exclusive)
        uint32_t* NT = nt_all + warp * kNR;           // [56] packed filter words
        for (int e = lane; e < kQW * KMAX; e += 32) L[e] = 0xFFFFFFFFu;
        // thresholds: own k-th (from the list) and the shared word; queries past nq never qualify
        auto refresh = [&]() {
            __syncwarp();
#pragma unroll
            for (int r = 0; r < (kQW + 31) / 32; ++r) {
                const int q = lane + 32 * r;
                if (q < kQW) {
                    const bool ok = qw0 + q < a.nq;
                    uint32_t gw = 0;
                    if (ok) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gw) : "l"(gthr_inv + qw0 + q));
                    const uint32_t own = L[q * KMAX + k - 1];
                    const uint32_t ov = own == 0xFFFFFFFFu ? kNone : own >> C::IDX_BITS;
                    const uint32_t sv = gw ? min(0xFFFFu - gw + 1u, kNone) : kNone;
                    TQ[q] = ok ? min(ov, sv) : 0u;
                }
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < (kNR + 31) / 32; ++r) {
                const int i = lane + 32 * r;
                if (i < kNR)
                    NT[i] = filter_half<kDot, C::KVMAX>(TQ[2 * i]) | (filter_half<kDot, C::KVMAX>(TQ[2 * i + 1]) << 16);
            }
            __syncwarp();
        };
        refresh();
        const uint32_t tlane = (uint32_t)(quad * 32) << 16;
#ifdef BOLT_PROFILE
        long long e_last = 0;
#endif
        for (int tile = 0; tile < ntiles; ++tile) {
            const int d = tile & 1;
#ifdef BOLT_PROFILE
            const long long e0 = clock64();
            if (threadIdx.x == 0 && tile > 0) SP_COUNT(15, e0 - e_last);
#endif
            mbar_wait(&tfull[d], (tile >> 1) & 1);
#ifdef BOLT_PROFILE
            const long long e1 = clock64();
            e_last = e1;
            if (threadIdx.x == 0) SP_COUNT(14, e1 - e0);
#endif
            tc_fence_after();
            uint32_t p[kNR];
            {
                const uint32_t ta = tmem + tlane + (uint32_t)(d * NQ + half * kQW);
#pragma unroll
                for (int c = 0; c < kQW / 32; ++c) {
                    uint32_t r[16];
                    tmem_ld16p(ta + c * 32, r);
#pragma unroll
                    for (int i = 0; i < 16; ++i) p[c * 16 + i] = r[i];
                }
                if constexpr (kQW % 32 == 16) {
                    uint32_t r8[8];
                    tmem_ld8p(ta + (kQW / 32) * 32, r8);
#pragma unroll
                    for (int i = 0; i < 8; ++i) p[(kQW / 32) * 16 + i] = r8[i];
                }
                tmem_wait_ld();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0) mbar_arrive(&tempty[d]);
                else mbar_arrive_cluster_relaxed(&tempty[d], 0);
            }
            if (xmode & 1) continue;  // diagnostic: load + release only
            if (tile > 0 && tile % kRefresh == 0) refresh();
            const int vl = tile * kVT + (int)rank * 128 + quad * 32 + lane;  // local vector index
            const bool vvalid = vbeg + vl < vend;
            // filter: one packed add per two queries, AND-reduced per group of 16 queries
            uint32_t gacc[kNG];
#pragma unroll
            for (int g = 0; g < kNG; ++g) gacc[g] = 0xFFFFFFFFu;
#pragma unroll
            for (int i = 0; i < kNR; i += 4) {
                const uint4 w = *reinterpret_cast<const uint4*>(NT + i);
                const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) gacc[(i + j) / kGroupRegs] &= kDot ? ww[j] - p[i + j] : p[i + j] + ww[j];
            }
            if (xmode & 4) {  // diagnostic: filter only
                if ((gacc[0] & gacc[kNG - 1]) == 0x12345678u) L[0] = gacc[0];
                continue;
            }
            uint32_t gm = 0;  // groups with a candidate in some lane (warp-uniform)
#pragma unroll
            for (int g = 0; g < kNG; ++g)
                gm |= (__any_sync(0xffffffffu, vvalid && (gacc[g] & 0x80008000u) != 0x80008000u) ? 1u : 0u) << g;
            if (lane == 0) {
                SP_COUNT(4, 1);            // warp-tiles
                SP_COUNT(0, __popc(gm));   // group entries
                if (tile < 16) SP_COUNT(5, __popc(gm));
                else if (tile < 128) SP_COUNT(6, __popc(gm));
                else SP_COUNT(7, __popc(gm));
            }
            if (!gm) continue;
            uint32_t* scr = scr_all + threadIdx.x * kScrStride;
#pragma unroll
            for (int g = 0; g < kNG; ++g) {
                if (!((gm >> g) & 1u)) continue;
#pragma unroll
                for (int j = 0; j < kGroupRegs; ++j) scr[j] = p[kGroupRegs * g + j];
                slow_group<C, kDot, KMAX>(scr, g, (uint32_t)vl, vvalid, k, L, TQ, NT, gthr_inv + qw0, a.nq - qw0, lane);
            }
        }
        __syncwarp();
        // lists -> part_keys[((part * 2 + rank) * 4 + quad)][query][k]
        const int64_t li = ((int64_t)part * 2 + rank) * 4 + quad;
        for (int q = 0; q < kQW; ++q) {
            if (qw0 + q >= a.nq) break;
            if (lane < k) {
                const uint32_t key = L[q * KMAX + lane];
                uint64_t out = ~0ull;
                if (key != 0xFFFFFFFFu) {
                    const uint32_t kvp = key >> C::IDX_BITS;
                    const uint32_t kv64 = kDot ? 0xFFFFu - (C::KVMAX - kvp) : kvp;  // (R13) 0xFFFF - acc
                    out = make_key(kv64, (uint64_t)(index_base + vbeg + (key & ((1u << C::IDX_BITS) - 1u))));
                }
                part_keys[(li * a.nq + qw0 + q) * k + lane] = out;
            }
        }
    } else if (warp == kMmaWarp && rank == 0) {
        // ------------------------------------------- MMA issuer (leader CTA)
        if (lane == 0) {
            const uint32_t a_base = smem_u32(sA);
            const uint32_t b_base = smem_u32(sB);
            for (int tile = 0; tile < ntiles; ++tile) {
                const int s = tile % S, d = tile & 1;
                mbar_wait_cluster(&full[s], (tile / S) & 1);
                mbar_wait_cluster(&tempty[d], ((tile >> 1) & 1) ^ 1);
                tc_fence_after();
#pragma unroll
                for (int ks = 0; ks < C::KSTEPS; ++ks) {
                    // A: compressed chunks 2 ks, 2 ks + 1 of the stage; B: table chunks 4 ks .. 4 ks + 3
                    const uint64_t ad = smem_desc(a_base + s * C::A_BYTES + 2 * ks * (128 * 16), 128 * 16, 128);
                    const uint64_t bd = smem_desc(b_base + 4 * ks * (kNQH * 16), kNQH * 16, 128);
                    mma_sp_pair(tmem + (uint32_t)(d * NQ), ad, bd,
                                tmem + (uint32_t)(kMetaCol0 + s * C::META_COLS + 2 * ks), C::IDESC, ks > 0 ? 1u : 0u);
                }
                mma_commit_pair(&empty[s]);
                mma_commit_pair(&tfull[d]);
            }
        }
        __syncwarp();
    }
    tc_fence_before();
    cluster_sync();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

template <int M, bool kDot, int KMAX, int NQ>
cudaError_t launch_mk(const ScanArgs& a, int k, int64_t index_base, int rparts, uint64_t* part_keys, uint32_t* gthr,
                      cudaStream_t s) {
    using C = Cfg<M, KMAX, NQ>;
    const int tiles_q = (int)ceil_div(a.nq, NQ);
    const int64_t vpp = ceil_div(ceil_div(a.n, rparts), 8) * 8;
    auto kern = topk_sp_kernel<M, kDot, KMAX, NQ>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * tiles_q * rparts));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int xmode = 0;
#ifdef BOLT_XMODE
    if (const char* x = getenv("BOLT_TC_XMODE")) xmode = atoi(x);
#endif
    cudaError_t e = cudaMemsetAsync(gthr, 0, (size_t)a.nq * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, kern, a, k, index_base, vpp, tiles_q, part_keys, gthr, xmode);
}

template <int M, int NQ>
cudaError_t launch_mq(const ScanArgs& a, int k, int metric, int64_t index_base, int rparts, uint64_t* part_keys,
                      uint32_t* gthr, cudaStream_t s) {
    const bool dot = metric == BOLT_DOT;
    if (k <= 4 && NQ == kNQ)
        return dot ? launch_mk<M, true, 4, NQ>(a, k, index_base, rparts, part_keys, gthr, s)
                   : launch_mk<M, false, 4, NQ>(a, k, index_base, rparts, part_keys, gthr, s);
    if (k <= 16 || M > 16)
        return dot ? launch_mk<M, true, 16, NQ>(a, k, index_base, rparts, part_keys, gthr, s)
                   : launch_mk<M, false, 16, NQ>(a, k, index_base, rparts, part_keys, gthr, s);
    if constexpr (M <= 16)
        return dot ? launch_mk<M, true, 32, NQ>(a, k, index_base, rparts, part_keys, gthr, s)
                   : launch_mk<M, false, 32, NQ>(a, k, index_base, rparts, part_keys, gthr, s);
    return cudaErrorInvalidValue;
}

// queries per tile: 32 or 64 for small batches (N = the batch, padded), else 224
inline int pick_nq(int64_t nq) { return nq <= 32 ? 32 : (nq <= 64 ? 64 : kNQ); }

template <int M>
cudaError_t launch_m(const ScanArgs& a, int k, int metric, int64_t index_base, int rparts, uint64_t* part_keys,
                     uint32_t* gthr, cudaStream_t s) {
    switch (pick_nq(a.nq)) {
        case 32: return launch_mq<M, 32>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        case 64: return launch_mq<M, 64>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        default: return launch_mq<M, kNQ>(a, k, metric, index_base, rparts, part_keys, gthr, s);
    }
}

}  // namespace sp

int topk_sp_supported(int64_t n, int m, int64_t nq, int k) {
    (void)nq;
    return n >= 1 && k >= 1 && (m == 8 || m == 16 || m == 32) && k <= (m == 32 ? 16 : 32);
}

// 8 lists per query per row partition (2 CTAs x 4 lane quadrants); partitions
// fill >= 4 waves of SM pairs, each within the local index range
int topk_sp_parts(int64_t n, int m, int64_t nq, int k, int num_sms) {
    (void)k;
    const int64_t tiles_q = ceil_div(nq, sp::pick_nq(nq));
    const int64_t max_range = m == 8 ? sp::Cfg<8, 4>::MAX_RANGE : (m == 16 ? sp::Cfg<16, 4>::MAX_RANGE
                                                                          : sp::Cfg<32, 4>::MAX_RANGE);
    int rparts = choose_parts(tiles_q, ceil_div(n, 8), num_sms / 2, (int64_t)256 * 16 / 8);
    rparts = (int)max64(rparts, ceil_div(n, max_range - 8));
    return 8 * rparts;
}

// part_keys: parts * nq * k keys followed by nq u32 shared thresholds
cudaError_t launch_topk_sp(const ScanArgs& a, int k, int metric, int64_t index_base, int parts, uint64_t* part_keys,
                           cudaStream_t s) {
    uint32_t* gthr = reinterpret_cast<uint32_t*>(part_keys + (size_t)parts * a.nq * k);
    const int rparts = parts / 8;
    switch (a.m) {
        case 8: return sp::launch_m<8>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        case 16: return sp::launch_m<16>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        case 32: return sp::launch_m<32>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace bolt

namespace bolt {
void sp_debug_counters(uint64_t* out8) {
#ifdef BOLT_PROFILE
    unsigned long long h[16] = {};
    cudaMemcpyFromSymbol(h, g_sp_counters, sizeof(h));
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_sp_counters, z, sizeof(z));
    for (int i = 0; i < 8; ++i) out8[i] = h[i];
    fflush(stdout);
    printf("sp timing: prod_wait_empty/tile %.0f prod_work/tile %.0f mma_wait_full/tile %.0f mma_wait_tempty/tile %.0f "
           "epi_wait_tfull/tile %.0f epi_work/tile %.0f (cycles, per CTA-tile)\n",
           (double)h[8] / (h[12] + 1e-9), (double)h[9] / (h[12] + 1e-9), (double)h[10] / (h[13] + 1e-9),
           (double)h[11] / (h[13] + 1e-9), (double)h[14] / (h[12] + 1e-9), (double)h[15] / (h[12] + 1e-9));
    fflush(stdout);
#else
    for (int i = 0; i < 8; ++i) out8[i] = 0;
#endif
}
}  // namespace bolt
