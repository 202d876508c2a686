// scan_tc.cu -- the Bolt scan as a tcgen05 tensor-core contraction (sm_100a).
//
// The scan sum acc(i, q) = sum_c beta[q][c][code(i, c)]
// equals the integer matrix product
//     D[q][i] = sum_{c, k} A[q][16c + k] * B[i][16c + k],
// A = the u8 tables (row = query, K = 16 M bytes, exactly the [q][c][16]
// layout), B = one-hot(codes) (B[i][16c + k] = 1 iff code(i, c) = k).
// Every product is 0 or a table entry and every sum is <= 255 M, so
// tcgen05.mma.kind::i8 (u8 x u8 -> s32 in TMEM) is exact: this is the same
// integer as the PRMT scan, bit for bit.  It executes 16x the algorithmic
// lookups, at tensor-core rate.
//
// A CTA pair (cluster of 2, cta_group::2) computes 256 queries x 256
// vectors per MMA tile: CTA r holds queries [128r, 128r+128) of the query
// tile (its half of A) and vectors [128r, 128r+128) of each vector tile (its
// half of B); its TMEM receives its 128 queries x all 256 vectors.  So each
// SM expands only 128 one-hot vectors per 1024-cycle MMA tile.
//   warps 0-3   producers: stage A once (16-byte units, K-major "interleave"
//               layout), then expand each vector tile's codes into the one-hot
//               B half in shared memory (one aligned 16-byte store per
//               (vector, codebook)), STAGES-deep ring.
//   warps 4-11  epilogue: thread = query (TMEM lane), two warps per lane
//               quadrant splitting the 256 columns; tcgen05.ld .pack::16b the
//               sums, packed u16x2 min/max tree against the query's running
//               top-k threshold, rare inserts into a register top-k list.
//   warp  12    MMA issuer (leader CTA, one thread): M/2 tcgen05.mma
//               (K = 32 bytes each) into one of two TMEM accumulators; commits
//               multicast to both CTAs' mbarriers.
// Shared-memory operand layout (both K-major, SWIZZLE_NONE): the 16-byte
// chunk j of row r lives at j * (rows * 16) + (r / 8) * 128 + (r % 8) * 16,
// so SBO (next 8 rows) = 128 B and LBO (next 16-byte K chunk) = rows * 16 B.
#include <cuda.h>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tma_host.cuh"
#include "topk_list.cuh"

namespace bolt {
#ifdef BOLT_PROFILE
__device__ unsigned long long g_counters[kNumCounters];
#endif

#ifdef BOLT_XMODE
// per-tile clock64 timeline of CTA 0 (BOLT_TC_XMODE & 64; tools/ only)
// [rank][tile][col] for the two CTAs of cluster 0
constexpr int kTraceTiles = 512, kTraceCols = 40;
__device__ unsigned long long g_trace[2 * kTraceTiles * kTraceCols];
#define BOLT_TRACE(tile, col)                                                               \
    do {                                                                                    \
        if ((xmode & 64) && blockIdx.x < 2 && (tile) < kTraceTiles)                         \
            g_trace[(blockIdx.x * kTraceTiles + (tile)) * kTraceCols + (col)] = clock64();  \
    } while (0)
#else
#define BOLT_TRACE(tile, col) ((void)0)
#endif

void sp_debug_counters(uint64_t* out8);  // scan_sp.cu

int tc_debug_counters(uint64_t* out, int n) {
    const int nc = n < kNumCounters ? n : kNumCounters;
#ifdef BOLT_PROFILE
    unsigned long long h[kNumCounters] = {};
    cudaMemcpyFromSymbol(h, g_counters, sizeof(h));
    unsigned long long z[kNumCounters] = {};
    cudaMemcpyToSymbol(g_counters, z, sizeof(z));
    for (int i = 0; i < nc; ++i) out[i] = h[i];
    uint64_t sp8[8];
    sp_debug_counters(sp8);
    for (int i = 16; i < nc; ++i) out[i] = out[i] ? out[i] : sp8[i - 16];
#else
    for (int i = 0; i < nc; ++i) out[i] = 0;
#endif
    if (n <= kNumCounters) return nc;
#ifdef BOLT_XMODE
    const int nt = n - kNumCounters < 2 * kTraceTiles * kTraceCols ? n - kNumCounters : 2 * kTraceTiles * kTraceCols;
    cudaMemcpyFromSymbol(out + kNumCounters, g_trace, nt * sizeof(uint64_t));
    return kNumCounters + nt;
#else
    return nc;
#endif
}

namespace tc {

constexpr int kQM = 128;                 // queries per CTA = TMEM lanes (MMA M = 256 per pair)
constexpr int kProdWarps = 4;            // thread = vector (NH = 128 per CTA)
constexpr int kProducers = kProdWarps * 32;
constexpr int kEpiWarps = 8;             // two warps per TMEM lane quadrant (column halves)
constexpr int kEpilogue = kEpiWarps * 32;
constexpr int kMmaWarp = kProdWarps + kEpiWarps;
// Warp roles by index: epilogue 0-7, producers 8-11, MMA issuer 12.  The
// SMSP schedulers favour higher warp ids, so the producers, whose one-hot
// stages gate the MMA, win issue slots over the epilogue's filter work.
constexpr int kThreads = (kMmaWarp + 1) * 32;
constexpr int kPrefetch = 3;             // tiles of code words in flight per producer thread
#ifndef BOLT_TC_KMAX10
#define BOLT_TC_KMAX10 1  // k <= 10: 10-slot register lists (c2 scan 1.705 -> 1.687 ms)
#endif
#ifndef BOLT_TC_ONECAND
#define BOLT_TC_ONECAND 1  // slow path: a lone candidate taken from the chunk minimum, no scratch round trip (c2 scan 1.679 -> 1.633 ms)
#endif
#ifndef BOLT_TC_MASK_ADD
#define BOLT_TC_MASK_ADD 1  // candidate mask: one add per register, values < 2^15 (c2 scan 1.643 -> 1.623 ms)
#endif
#ifndef BOLT_TC_MINMAX_INSERT
#define BOLT_TC_MINMAX_INSERT 1  // min/max bubble insert (c2 scan 1.687 -> 1.678 ms)
#endif
// u32 words of shared scratch per epilogue thread: top-k parks 32 u16 values
// (80-byte rows: 16-byte aligned, conflict-free); full output stages a 32-row x
// 128-byte block per warp (4 KB)
constexpr int kScratchStrideTopk = 20;
constexpr int kScratchStrideFull = 32;
constexpr int kUnionParts = 8;           // top-k: finished partitions whose lists seed a unit's bound
constexpr int kGroupUnionParts = 16;     // ... lists of 32 (k > 32): sampled, so more lists pay
constexpr int kUnionMinTiles = 256;      // ... only for units this long (the read costs ~50 tiles' time)
constexpr int kUnionGroups = 2;          // top-k: groups of lists of the union bound (epilogue; 5 measured no better)
static_assert(kUnionGroups == 2 || kUnionGroups == 5, "2 or 5 union groups (load widths)");
constexpr int kStorePieces = 2;          // full output: TMA stores per 32-row x 128-byte warp block
#ifndef BOLT_TC_STORE_HINT
#define BOLT_TC_STORE_HINT 1  // evict-first L2 policy on the full-output TMA stores (c4 u16 0.066 -> 0.059 ms, fp32 0.090 -> 0.087)
#endif

// QROWS: query rows of the table buffer per CTA (kQM, or kNQ/2 in the
// swapped top-k); LIST_BYTES: the swapped top-k's per-warp lists (else the
// scratch rows of the other modes)
// PAIR: cta_group::2 (a CTA pair shares each 256-vector tile, 128 queries per
// CTA) or cta_group::1 (one CTA, 128 queries, expands all 256 vectors)
template <int M, bool kFull = false, int QROWS = kQM, int LIST_BYTES = 0, bool PAIR = true>
struct Cfg {
    static constexpr int SCRATCH_STRIDE = kFull ? kScratchStrideFull : kScratchStrideTopk;
    static constexpr int K = 16 * M;                      // bytes per row
    static constexpr int N = 256;                         // vectors per MMA tile
    static constexpr int NH = PAIR ? N / 2 : N;           // vectors whose one-hot this CTA holds
    static constexpr int QR = QROWS;
    static constexpr int A_BYTES = QROWS * K;
    static constexpr int B_BYTES = NH * K;                // one stage of this CTA's half of B
    static constexpr int SCRATCH_BYTES = LIST_BYTES ? LIST_BYTES : kEpilogue * SCRATCH_STRIDE * 4;
    static constexpr int STAGES_RAW = (227 * 1024 - 256 - A_BYTES - SCRATCH_BYTES) / B_BYTES;
    static constexpr int STAGES = STAGES_RAW > 5 ? 5 : STAGES_RAW;
    static_assert(STAGES >= 2, "shared memory too small for a double-buffered B tile");
    static constexpr int KSTEPS = K / 32;
    static constexpr int TMEM_COLS = 512;                  // 2 x 256-column accumulators
    // 32-bit epilogue keys: kv' <= 255 M needs VAL_BITS, the rest (to 31 bits) index the pair's range
    static constexpr int VAL_BITS = M <= 8 ? 11 : (M <= 16 ? 12 : 13);
    static constexpr int IDX_BITS = 31 - VAL_BITS;
    static constexpr int64_t MAX_RANGE = int64_t(1) << IDX_BITS;
    static constexpr uint32_t KVMAX = 255u * M;
    // dynamic smem: A | B[STAGES] | scratch | barriers
    static constexpr int SCRATCH_OFF = A_BYTES + STAGES * B_BYTES;
    static constexpr int BAR_OFF = SCRATCH_OFF + SCRATCH_BYTES;
    static constexpr int SMEM = BAR_OFF + 256;
    // instruction descriptor: D s32 (bits 4-5 = 2), A/B u8 (format 0), K-major,
    // N >> 3 at bit 17, M >> 4 at bit 24 (M = 256 for the pair)
    static constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)((PAIR ? 256 : 128) >> 4) << 24);
    // swapped top-k: M = 256 vectors (A = one-hot), N = 2 QROWS queries (B = tables)
    static constexpr uint32_t IDESC_SW = (2u << 4) | ((uint32_t)((2 * QROWS) >> 3) << 17) |
                                         ((uint32_t)(256 >> 4) << 24);
};

// Register-resident sorted top-k list of one thread with 32-bit keys
// (kv' << IDX_BITS) | local index (kv' = acc for L2, 255 M - acc for dot, so
// smaller is better in both cases; local = vector index within the CTA's
// range), right-aligned in KMAX slots: slots [0, KMAX-k) hold 0 (every key
// passes through them), slots [KMAX-k, KMAX) the k best keys ascending, so
// the k-th best is always slot KMAX-1.  Keys are unique, so an insert is a
// branch-free bubble pass of min/max pairs.
template <int KMAX>
struct RegList {
    uint32_t v[KMAX];
    __device__ __forceinline__ void init(int k) {
#pragma unroll
        for (int i = 0; i < KMAX; ++i) v[i] = i < KMAX - k ? 0u : 0xFFFFFFFFu;
    }
    // Insert c, evicting the largest key.  All comparisons against the old
    // list are independent, then each slot selects its old value, c, or its
    // left neighbour (depth 3, instead of a KMAX-long min/max chain: the
    // slow path is latency-bound).
    __device__ __forceinline__ void insert(uint32_t c) {
#if BOLT_TC_MINMAX_INSERT
        // v'[i] = max(v[i-1], min(v[i], c)): each slot from the old values
        // only (depth 2, one min and one max per slot)
#pragma unroll
        for (int i = KMAX - 1; i > 0; --i) v[i] = max(v[i - 1], min(v[i], c));
        v[0] = min(v[0], c);
#else
        bool lt[KMAX];
#pragma unroll
        for (int i = 0; i < KMAX; ++i) lt[i] = v[i] < c;
#pragma unroll
        for (int i = KMAX - 1; i > 0; --i) v[i] = lt[i] ? v[i] : (lt[i - 1] ? c : v[i - 1]);
        v[0] = lt[0] ? v[0] : c;
#endif
    }
    __device__ __forceinline__ uint32_t threshold(int idx_bits) const {
        return v[KMAX - 1] == 0xFFFFFFFFu ? kNotFull : (v[KMAX - 1] >> idx_bits);
    }
    // value of the entry in slot `pos` (kNotFull if empty); select chain, no local memory
    __device__ __forceinline__ uint32_t value_at(int pos, int idx_bits) const {
        uint32_t r = 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < KMAX; ++i) r = i == pos ? v[i] : r;
        return r == 0xFFFFFFFFu ? kNotFull : (r >> idx_bits);
    }
};

}  // namespace tc
}  // namespace bolt

namespace bolt {
namespace tc {

// Candidate mask of 32 packed u16 sums p[16] (value j = half j&1 of p[j>>1])
// against the threshold: SWAR compare of both halves (values and threshold
// < 2^15), flags gathered with PRMT.  Bit 8k + i of the result <-> value
// 4i + k.
template <bool kDot>
__device__ __forceinline__ uint32_t candidate_mask(const uint32_t (&p)[16], uint32_t tp) {
    uint32_t nm = 0;  // 1 = not a candidate
#if BOLT_TC_MASK_ADD
    // values < 2^15: p | 0x80008000 == p + 0x80008000, so the per-half
    // compare is one add of a lane constant
    const uint32_t cadd = 0x80008000u - tp;
#endif
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#if BOLT_TC_MASK_ADD
        const uint32_t d0 = kDot ? ((tp | 0x80008000u) - p[2 * i]) : (p[2 * i] + cadd);
        const uint32_t d1 = kDot ? ((tp | 0x80008000u) - p[2 * i + 1]) : (p[2 * i + 1] + cadd);
#else
        const uint32_t d0 = kDot ? ((tp | 0x80008000u) - p[2 * i]) : ((p[2 * i] | 0x80008000u) - tp);
        const uint32_t d1 = kDot ? ((tp | 0x80008000u) - p[2 * i + 1]) : ((p[2 * i + 1] | 0x80008000u) - tp);
#endif
        const uint32_t x = __byte_perm(d0, d1, 0x7531);  // flags at bits 7, 15, 23, 31
        nm |= (x >> (7 - i)) & (0x01010101u << i);
    }
    return ~nm;
}

// Full-output mode (kOut = 1: u16 sums, 2: fp32 acc / a + sum b):
// out[i * ldo + q] for database vector i and query q.
struct FullOut {
    void* out;
    int64_t ldo;
    float inv_a, b_sum;
    int vec;  // rows 16 B aligned: vector stores
    int tma;  // store the staged blocks with TMA (omap valid; partitions are whole 256-row tiles)
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t smem, int x, int y) {
#if BOLT_TC_STORE_HINT
    // evict-first L2 policy for the streamed output (drains in issue order)
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(map),
                 "r"(smem), "r"(x), "r"(y), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem), "r"(x), "r"(y)
                 : "memory");
#endif
}

// ------------------------------------------------ swapped top-k epilogue
// kOut = 3: vectors on the MMA M side (A = one-hot, 128 per CTA = TMEM
// lanes), queries on N (B = tables of kNQ queries, kNQ/2 per CTA), so a
// small query batch does not pad the MMA to 256 queries.  Warp (quad, half)
// owns vectors 32 quad .. of its CTA (one per lane) and queries
// [half QW, half QW + QW) of the tile (QW = kNQ / 2, registers).  One sorted
// list of k <= 32 32-bit keys (kv' << IDX_BITS | local vector index) per
// (warp, query) in shared memory; a packed SWAR test against per-query
// thresholds (own k-th value, the query's shared word) finds candidates, and
// the warp inserts them one at a time (lane l holds entry l).  Lists of a
// query: 8 per CTA pair and row partition, merged afterwards.
template <typename C, bool kDot, int kNQ>
__device__ __forceinline__ void epilogue_swapped(const ScanArgs& a, int k, int64_t index_base, int64_t vbeg,
                                                 int64_t vend, int ntiles, int part, int tq, uint32_t rank,
                                                 int warp, int lane, uint32_t tmem, uint64_t* tfull,
                                                 uint64_t* tempty, uint32_t* lists, uint64_t* part_keys,
                                                 uint32_t* gthr_inv, int xmode) {
    constexpr int QW = kNQ / 2;  // queries per warp
    constexpr int NR = QW / 2;   // packed registers
    constexpr int NW = (QW + 31) / 32;
    const int quad = warp & 3, half = warp >> 2;
    uint32_t* lst = lists + warp * QW * 32;  // [QW][32]
    const int64_t qb = (int64_t)tq * kNQ + half * QW;  // first query of this warp
    for (int e = lane; e < QW * 32; e += 32) lst[e] = 0xFFFFFFFFu;
    __syncwarp();
    // thresholds in kv' units (candidate iff kv' < thr); 0x7FFF = none (every
    // value < 0x7FFF), 0 for queries past nq (never a candidate)
    uint32_t thrp[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        const uint32_t lo = qb + 2 * i < a.nq ? 0x7FFFu : 0u, hi = qb + 2 * i + 1 < a.nq ? 0x7FFFu : 0u;
        thrp[i] = lo | (hi << 16);
    }
    uint32_t gw[NW];  // shared words (inverted 0xFFFF - T) of queries qb + lane + 32 w
#pragma unroll
    for (int w = 0; w < NW; ++w) gw[w] = 0;
    const uint32_t tlane = (uint32_t)(quad * 32) << 16;
    const uint32_t kvmax2 = C::KVMAX | (C::KVMAX << 16);
    for (int tile = 0; tile < ntiles; ++tile) {
        const int d = tile & 1;
        mbar_wait(&tfull[d], (tile >> 1) & 1);
        tc_fence_after();
        uint32_t p[NR];
        const uint32_t ta = tmem + tlane + (uint32_t)(d * kNQ + half * QW);
        if (xmode & 8) {  // diagnostic: no TMEM reads
#pragma unroll
            for (int i = 0; i < NR; ++i) p[i] = 0x7FFF7FFFu;
        } else if constexpr (QW == 16) {
            uint32_t r[8];
            tmem_ld8p(ta, r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i) p[i] = r[i];
        } else {
#pragma unroll
            for (int c = 0; c < QW / 32; ++c) {
                uint32_t r[16];
                tmem_ld16p(ta + c * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 16; ++i) p[c * 16 + i] = r[i];
            }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            if (rank == 0) mbar_arrive(&tempty[d]);
            else mbar_arrive_cluster_relaxed(&tempty[d], 0);
        }
        if (xmode & 1) continue;  // diagnostic: load + release only
        const int64_t vl = (int64_t)tile * C::N + rank * C::NH + quad * 32 + lane;  // local vector index
        const bool vvalid = vbeg + vl < vend;
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            if (kDot) p[i] = kvmax2 - p[i];  // kv' = KVMAX - acc per half (no borrow: acc <= KVMAX)
            if (!vvalid) p[i] = 0x7FFF7FFFu;
        }
        // shared thresholds: re-read every 8 tiles, folded into thrp
        if ((tile & 7) == 7) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const int64_t q = qb + lane + 32 * w;
                uint32_t v = 0;
                if (lane + 32 * w < QW && q < a.nq)
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gthr_inv + q));
                gw[w] = v;
            }
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                // own k-th values from the lists (shared-memory broadcast reads)
                const uint32_t k0 = lst[(2 * i) * 32 + k - 1], k1 = lst[(2 * i + 1) * 32 + k - 1];
                const uint32_t o0 = k0 == 0xFFFFFFFFu ? 0x7FFFu : k0 >> C::IDX_BITS;
                const uint32_t o1 = k1 == 0xFFFFFFFFu ? 0x7FFFu : k1 >> C::IDX_BITS;
                const uint32_t s0 = __shfl_sync(0xffffffffu, gw[(2 * i) / 32], (2 * i) % 32);
                const uint32_t s1 = __shfl_sync(0xffffffffu, gw[(2 * i + 1) / 32], (2 * i + 1) % 32);
                const uint32_t t0 = min(o0, s0 ? 0xFFFFu - s0 + 1u : 0x7FFFu);
                const uint32_t t1 = min(o1, s1 ? 0xFFFFu - s1 + 1u : 0x7FFFu);
                const uint32_t lo = qb + 2 * i < a.nq ? t0 : 0u, hi = qb + 2 * i + 1 < a.nq ? t1 : 0u;
                thrp[i] = lo | (hi << 16);
            }
        }
        // fast test: bit 15 / 31 of (p | 0x80008000) - thr clear <=> that half is a candidate
        uint32_t all = 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < NR; ++i) all &= (p[i] | 0x80008000u) - thrp[i];
        if (!__any_sync(0xffffffffu, (all & 0x80008000u) != 0x80008000u)) continue;
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const uint32_t dd = (p[i] | 0x80008000u) - thrp[i];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t cand = __ballot_sync(0xffffffffu, !(dd & (0x8000u << (16 * h))));
                if (!cand) continue;
                const int q = 2 * i + h;
                uint32_t* L = lst + q * 32;
                const uint32_t key = (((p[i] >> (16 * h)) & 0xFFFFu) << C::IDX_BITS) | (uint32_t)vl;
                uint32_t kth = 0;
                while (cand) {
                    const int src = __ffs(cand) - 1;
                    cand &= cand - 1;
                    const uint32_t c = __shfl_sync(0xffffffffu, key, src);
                    const uint32_t cur = L[lane];
                    kth = __shfl_sync(0xffffffffu, cur, k - 1);
                    if (c >= kth) continue;
                    const uint32_t prev = __shfl_up_sync(0xffffffffu, cur, 1);
                    const int pos = __popc(__ballot_sync(0xffffffffu, lane < k && cur < c));
                    const uint32_t nw = lane == pos ? c : (lane > pos ? prev : cur);
                    __syncwarp();
                    if (lane < k) L[lane] = nw;
                    __syncwarp();
                    kth = __shfl_sync(0xffffffffu, nw, k - 1);
                }
                if (kth != 0xFFFFFFFFu) {
                    const uint32_t okv = kth >> C::IDX_BITS;
                    const uint32_t old = (thrp[i] >> (16 * h)) & 0xFFFFu;
                    if (okv < old) {
                        thrp[i] = (thrp[i] & ~(0xFFFFu << (16 * h))) | (okv << (16 * h));
                        if (lane == 0 && qb + q < a.nq)
                            asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(gthr_inv + qb + q),
                                         "r"(0xFFFFu - okv)
                                         : "memory");
                    }
                }
            }
        }
    }
    __syncwarp();
    // lists -> part_keys[((part * 2 + rank) * 4 + quad)][query][k]
    const int64_t li = ((int64_t)part * 2 + rank) * 4 + quad;
    for (int q = 0; q < QW; ++q) {
        if (qb + q >= a.nq) break;
        if (lane < k) {
            const uint32_t key = lst[q * 32 + lane];
            uint64_t out = ~0ull;
            if (key != 0xFFFFFFFFu) {
                const uint32_t kvp = key >> C::IDX_BITS;
                const uint32_t kv64 = kDot ? 0xFFFFu - (C::KVMAX - kvp) : kvp;
                out = make_key(kv64, (uint64_t)(index_base + vbeg + (key & ((1u << C::IDX_BITS) - 1u))));
            }
            part_keys[(li * a.nq + qb + q) * k + lane] = out;
        }
    }
}

template <int M, bool kDot, int KMAX, int kOut = 0, bool kGroup = false, int kNQ = 0, bool kPairT = true>
__global__ void __launch_bounds__(kThreads, 1)
topk_tc_kernel(ScanArgs a, int k, int64_t index_base, int64_t vpp, int tiles_q, uint64_t* __restrict__ part_keys,
               uint32_t* __restrict__ gthr_inv, int xmode, FullOut fo, const __grid_constant__ CUtensorMap omap) {
#ifndef BOLT_XMODE
#ifdef BOLT_XCONST
    xmode = BOLT_XCONST;  // diagnostic builds with one stage switch compiled in as a constant (tools/)
#else
    xmode = 0;  // diagnostic stage switches exist only in libbolt_x.so (tools/)
#endif
#endif
    using C = Cfg<M, (kOut == 1 || kOut == 2), (kOut == 3 ? kNQ / 2 : kQM),
                  (kOut == 3 ? kEpiWarps * (kNQ / 2) * 32 * 4 : 0), kPairT>;
    static_assert(kPairT || kOut == 0, "single-CTA tiles only for the top-k");
    constexpr int S = C::STAGES;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::A_BYTES;
    uint32_t* scratch_all = reinterpret_cast<uint32_t*>(smem + C::SCRATCH_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* full = bars;                 // [S]  leader: producers of both CTAs -> MMA
    uint64_t* empty = bars + S;            // [S]  both: MMA commit -> producers
    uint64_t* tfull = bars + 2 * S;        // [2]  both: MMA commit -> epilogue
    uint64_t* tempty = bars + 2 * S + 2;   // [2]  leader: epilogues of both CTAs -> MMA
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = kPairT ? cluster_rank() : 0u;
    const int unit = kPairT ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int tq = unit % tiles_q;
    const int part = unit / tiles_q;
    const int64_t q0 = (int64_t)tq * (kPairT ? 2 : 1) * C::QR + rank * C::QR;  // this CTA's queries
    const int64_t vbeg = (int64_t)part * vpp;
    const int64_t vend = min64(a.n, vbeg + vpp);
    const int ntiles = vend > vbeg ? (int)ceil_div(vend - vbeg, C::N) : 0;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], (kPairT ? 2 : 1) * kProdWarps);  // one arrive per producer warp of both CTAs
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], (kPairT ? 2 : 1) * kEpiWarps);  // one arrive per epilogue warp of both CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        if constexpr (kPairT) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"((uint32_t)C::TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"((uint32_t)C::TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    if constexpr (kPairT) cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const long long tk0 = BOLT_CLOCK();

    if (warp >= kEpiWarps && warp < kMmaWarp) {
        // ------------------------------------------------------ producers
        const int t = threadIdx.x - kEpilogue;
        // A: this CTA's queries, 16-byte unit (c, q) -> c*(QR*16) + (q/8)*128 + (q%8)*16,
        // as asynchronous copies (LDGSTS) issued back to back -- a dependent
        // load/store loop took ~10 us per unit for 64 KB of tables -- with
        // zero fill past nq; completed below before the first full arrive
        for (int u = t; u < C::QR * M; u += kProducers) {
            const int c = u / C::QR, q = u % C::QR;
            const bool ok = q0 + q < a.nq;
            const uint8_t* src = a.qluts + ((ok ? q0 + q : 0) * M + c) * kK;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                             smem_u32(sA + c * (C::QR * 16) + (q >> 3) * 128 + (q & 7) * 16)),
                         "l"(src), "r"(ok ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        // Thread t expands vector v = t of each tile: its M code words (the
        // same for the 8 vectors of a layout-v1 group, one broadcast load)
        // are fetched from global memory a tile ahead, so no producer barrier
        // is needed; each warp arrives on the stage's full barrier on its own.
        constexpr int VPT = C::NH / kProducers;     // vectors per producer thread (1 pair, 2 single)
        static_assert(VPT * kProducers == C::NH, "whole vectors per producer thread");
        constexpr int MH = M;                       // codebooks per producer thread
        constexpr int NW4 = MH / 4;                 // uint4 loads per vector
        constexpr int ch = 0;
        const uint32_t sh = (t & 7) * 4;            // kProducers % 8 == 0: the same for every vector of t
        // 8 * code = bits 3..6 of the word rotated right by sh - 3 (one funnel shift + mask)
        const uint32_t rot = (sh - 3u) & 31u;
        auto load_words = [&](int tile, uint4 (&w)[VPT][NW4]) {
#pragma unroll
            for (int u = 0; u < VPT; ++u) {
                const int64_t g = (vbeg + (int64_t)tile * C::N + rank * C::NH + t + u * kProducers) >> 3;
#pragma unroll
                for (int i = 0; i < NW4; ++i)
                    w[u][i] = g < a.groups ? __ldg(reinterpret_cast<const uint4*>(a.codes + g * M + ch * MH) + i)
                                           : make_uint4(0, 0, 0, 0);
            }
        };
        // one tile of expansion: wait for the stage, write the one-hot rows,
        // publish them to the async proxy and arrive on the stage's full barrier
        auto produce = [&](int tile, const uint4 (&cur)[VPT][NW4]) {
            const int s = tile % S;
            long long tw0 = BOLT_CLOCK();
            mbar_wait(&empty[s], ((tile / S) & 1) ^ 1);
            if (lane == 0) BOLT_TRACE(tile, 3 + t / 32);
            if (t == 0) BOLT_PROF_ADD(0, BOLT_CLOCK() - tw0);  // producer waits on empty
            const int64_t hb = vbeg + (int64_t)tile * C::N + rank * C::NH;  // first vector of this half
#pragma unroll
            for (int u = 0; u < VPT; ++u) {
                const int v = t + u * kProducers;
                uint8_t* b = sB + s * C::B_BYTES + ch * MH * (C::NH * 16) + v * 16;
                if (xmode & 2) {
                    // diagnostic: keep the stage's stale one-hot rows
                } else if (hb + C::NH <= vend) {
#pragma unroll
                    for (int i = 0; i < NW4; ++i) {
                        const uint32_t ws[4] = {cur[u][i].x, cur[u][i].y, cur[u][i].z, cur[u][i].w};
#pragma unroll
                        for (int j = 0; j < 4 && 4 * i + j < MH; ++j)
                            *reinterpret_cast<uint4*>(b + (4 * i + j) * (C::NH * 16)) =
                                one_hot16_s(__funnelshift_r(ws[j], ws[j], rot) & 0x78u);
                    }
                } else {  // last, partial tile: rows past the range are all-zero
                    const bool valid = hb + v < vend;
#pragma unroll
                    for (int i = 0; i < NW4; ++i) {
                        const uint32_t ws[4] = {cur[u][i].x, cur[u][i].y, cur[u][i].z, cur[u][i].w};
#pragma unroll
                        for (int j = 0; j < 4 && 4 * i + j < MH; ++j)
                            *reinterpret_cast<uint4*>(b + (4 * i + j) * (C::NH * 16)) =
                                one_hot16_s(valid ? (__funnelshift_r(ws[j], ws[j], rot) & 0x78u) : 128u);
                    }
                }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                BOLT_TRACE(tile, 7 + t / 32);
                if (rank == 0) mbar_arrive(&full[s]);
                else mbar_arrive_remote_cta(&full[s], 0);
            }
        };
        // code words prefetched kPrefetch tiles ahead (a register ring indexed
        // statically by unrolling the tile loop), issued after each arrive
        constexpr int D = VPT == 1 ? kPrefetch : 2;
        uint4 pre[D][VPT][NW4];
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
      if constexpr (kOut == 3) {
        epilogue_swapped<C, kDot, kNQ>(a, k, index_base, vbeg, vend, ntiles, part, tq, rank, warp, lane, tmem, tfull,
                                       tempty, scratch_all, part_keys, gthr_inv, xmode);
      } else {
        // ------------------------------------------------------- epilogue
        const int quad = warp & 3;                 // TMEM lanes 32*quad .. (warp % 4 rule)
        const int half = warp >> 2;                // column half of the tile
        const int q = quad * 32 + lane;            // query row of this CTA
        constexpr int kCols = C::N / 2;
        uint32_t* scratch = scratch_all + threadIdx.x * C::SCRATCH_STRIDE;
        RegList<KMAX> list;
        list.init(k);
        // Thresholds in kv' units.  own = k-th key of this list; shared =
        // min over every list of this query (all CTAs), kept in global memory
        // as 0xFFFF - T so that a zeroed word means "none" (T = 0xFFFF).  A
        // value can reach the global top-k only if kv' < own and kv' <= T.
        uint32_t own = kNotFull;
        uint32_t published = kNotFull;
        // Union bound over G = min(k, kUnionGroups) groups of lists: the lists
        // of a query (id 2 part + half, all disjoint vectors) are dealt into G
        // groups by id mod G; each publishes its j-th value, j = ceil(k / G),
        // into its group's word (minimum).  If every group's best list holds
        // j values <= x, the union holds >= G j >= k of them, so the largest
        // group minimum is a valid threshold.  G = 2 (the column halves, j =
        // ceil(k/2)); G = 5 (j = 2 at k = 10), better in an order-statistics
        // simulation, measured no fewer slow-path entries on c2 and a slower
        // scan.  Inverted words gthr_inv[hoff + 8q + g], hoff =
        // nq rounded up to a multiple of 4.
        const int hG = k < kUnionGroups ? k : kUnionGroups;
        const int hj = (k + hG - 1) / hG;
        const int hpos = KMAX - k + hj - 1;
        const int hgrp = (2 * part + half) % hG;
        uint32_t published_h = hG > 1 ? kNotFull : 0u;
        bool changed = false;  // list changed since the half bound was last published
        const bool qvalid = q0 + q < a.nq;
        uint32_t* gq = gthr_inv + (qvalid ? q0 + q : 0);
        uint32_t thr = kNotFull;
        uint32_t* gh = gthr_inv + ((a.nq + 3) & ~int64_t(3)) + 8 * (qvalid ? q0 + q : 0);  // 16 B aligned
        // kGroup (lists of 32 for a final k <= 32 G, G = a.noshare): a list's
        // 32nd value bounds only 32 values, so the lists of a query are dealt
        // into G groups (list id mod G) and each group keeps the minimum of its
        // lists' 32nd values (inverted word gthr_inv[4q + g]); the G group minima
        // come from G distinct lists, so >= 32 G >= k values lie at or below
        // their maximum, which bounds the k-th best.
        constexpr bool share = !kGroup;
        const int ngrp = kGroup ? a.noshare : 0;  // compile-time 0 outside the large-k instantiations
        uint32_t* gg = gthr_inv + 4 * (qvalid ? q0 + q : 0);
        const int grp = kGroup ? (2 * part + half) % ngrp : 0;
        uint32_t g_next = 0;                    // inverted shared threshold (0 = none yet), fetched a tile ahead
        uint32_t gw[kUnionGroups] = {};         // inverted union-group words, fetched a tile ahead
        uint32_t gs[4] = {0u, 0u, 0u, 0u};      // group words (kGroup)
        auto load_union = [&]() {
            if constexpr (kUnionGroups == 2) {
                asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];" : "=r"(gw[0]), "=r"(gw[1]) : "l"(gh));
            } else {
                asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(gw[0]), "=r"(gw[1]), "=r"(gw[2]), "=r"(gw[3])
                             : "l"(gh));
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gw[4]) : "l"(gh + 4));
            }
        };
        // Finished partitions' lists (done[p][tq] == number of CTAs of a
        // unit): their keys are final, every entry is a distinct row, so the
        // k-th smallest value of their union bounds this query's k-th best --
        // for units of later waves, the exact k-th of 20-80 % of the rows,
        // much tighter than any single list's k-th.  Read once, at unit start.
        // (c2: scan 1.78 -> 1.73 ms)
        // [rparts][tiles_q] after the threshold words (k <= 32: k-th words +
        // union-group rows; lists of 32: the [nq][4] group words)
        uint32_t* done = gthr_inv + (kGroup ? 4 * a.nq : ((a.nq + 3) & ~int64_t(3)) + 8 * a.nq);
        if (share && kOut == 0 && qvalid && part > 0 && ntiles >= kUnionMinTiles) {
            RegList<KMAX> ul;
            ul.init(k);
            // the first kUnionParts partitions (they finish first); any subset of
            // finished lists bounds, and more than 16 lists cost more to read
            // than they tighten (c3's 80 partitions: 0.33 -> 0.53 ms reading all)
            for (int pp = 0; pp < min(part, kUnionParts); ++pp) {
                uint32_t dn;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(dn) : "l"(done + (int64_t)pp * tiles_q + tq));
                if (dn != (kPairT ? 2u : 1u)) continue;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint64_t* src = part_keys + ((int64_t)(2 * pp + hh) * a.nq + q0 + q) * k;
                    for (int i = 0; i < k; ++i) {
                        const uint64_t key = src[i];
                        if (key == ~0ull) break;
                        const uint32_t kv64 = (uint32_t)(key >> 48);
                        const uint32_t kvp = kDot ? C::KVMAX - (0xFFFFu - kv64) : kv64;
                        if (kvp + 1u >= ul.v[KMAX - 1]) break;  // sorted list: the rest is no better
                        ul.insert(kvp + 1u);  // + 1: value 0 must not meet the 0 padding slots
                    }
                }
            }
            if (ul.v[KMAX - 1] != 0xFFFFFFFFu) {
                const uint32_t tu = ul.v[KMAX - 1] - 1u;  // k-th smallest value of the union
                asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(gq), "r"(0xFFFFu - tu) : "memory");
            }
        }
        // Lists of 32 (k > 32, R = 32 G rows needed): the same union, sampled --
        // each finished list contributes its values at positions 4i + 3 (i < 8),
        // each standing for 4 distinct rows at or below it, so the (R / 4)-th
        // smallest sample bounds the R-th best value; folded into every group
        // word (max_g min(G_g, T) = min(max_g G_g, T), still a valid bound).
        if (kGroup && kOut == 0 && qvalid && part > 0 && ntiles >= kUnionMinTiles) {
            RegList<32> ul;
            ul.init(8 * ngrp);  // R / 4 = 8 G samples
            for (int pp = 0; pp < min(part, kGroupUnionParts); ++pp) {
                uint32_t dn;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(dn) : "l"(done + (int64_t)pp * tiles_q + tq));
                if (dn != (kPairT ? 2u : 1u)) continue;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint64_t* src = part_keys + ((int64_t)(2 * pp + hh) * a.nq + q0 + q) * k;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint64_t key = src[4 * i + 3];
                        if (key == ~0ull) break;
                        const uint32_t kv64 = (uint32_t)(key >> 48);
                        const uint32_t kvp = kDot ? C::KVMAX - (0xFFFFu - kv64) : kv64;
                        if (kvp + 1u >= ul.v[31]) break;  // sorted list: the rest is no better
                        ul.insert(kvp + 1u);
                    }
                }
            }
            if (ul.v[31] != 0xFFFFFFFFu) {
                const uint32_t tu = ul.v[31] - 1u;
                for (int g = 0; g < ngrp; ++g)
                    asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(gg + g), "r"(0xFFFFu - tu) : "memory");
            }
        }
        if (share) {
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g_next) : "l"(gq));
            load_union();
        }
        const uint32_t tlane = (uint32_t)(quad * 32) << 16;
        for (int tile = 0; tile < ntiles; ++tile) {
            const int d = tile & 1;
            long long tw0 = BOLT_CLOCK();
            mbar_wait(&tfull[d], (tile >> 1) & 1);
            if (lane == 0) BOLT_TRACE(tile, 11 + warp);
            if (threadIdx.x == 0) BOLT_PROF_ADD(1, BOLT_CLOCK() - tw0);  // epilogue waits on tfull
            tc_fence_after();
            // copy this warp's 128 columns out of TMEM (packed u16 pairs) and
            // release the accumulator at once, so that a slow filter pass on
            // this warp never holds the MMA back
            uint32_t p[4][16];
            if (xmode & 8) {  // diagnostic: no TMEM reads
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int i = 0; i < 16; ++i) p[c][i] = 0xFFFFFFFFu;
            } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                tmem_ld16p(tmem + tlane + (uint32_t)(d * C::N + half * kCols + c * 32), p[c]);
            tmem_wait_ld();
            }
            if (threadIdx.x == 0) BOLT_PROF_ADD(2, BOLT_CLOCK() - tw0);  // wait + TMEM load
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                BOLT_TRACE(tile, 19 + warp);
                if (rank == 0) mbar_arrive(&tempty[d]);
                else mbar_arrive_cluster_relaxed(&tempty[d], 0);
            }
            const long long tp0 = BOLT_CLOCK();
            if (xmode & 1) continue;  // diagnostic: load + release only
            if constexpr (kOut != 0) {
                // Full output, swapped roles: this thread = database vector (TMEM
                // lane), registers = 128 consecutive queries of its output row.
                // Each 128-byte row segment (32 fp32 / 64 u16 queries) is written
                // whole: the warp stages its 32 rows x 128 B block in shared
                // memory (16-byte units XOR-swizzled by row, conflict-free both
                // ways) and reads it back so that each 16-byte global store
                // instruction covers 4 rows x 128 contiguous bytes.
                const int64_t vrow0 = vbeg + (int64_t)tile * C::N + rank * C::NH + quad * 32;  // warp's first row
                const int64_t qb = (int64_t)tq * 2 * kQM + half * kCols;  // first query of this warp
                uint4* stg = reinterpret_cast<uint4*>(scratch_all) + (warp & 7) * 256;  // 32 rows x 8 units
                constexpr int kEsz = kOut == 1 ? 2 : 4;
                constexpr int kQPU = 16 / kEsz;         // queries per 16-byte unit
                constexpr int kSeg = 8 * kQPU;          // queries per 128-byte segment
#pragma unroll
                for (int sg = 0; sg < kCols / kSeg; ++sg) {
                    // this lane's row: 8 units of the segment, computed before the
                    // staging block is reclaimed (overlaps the previous stores' reads)
                    uint4 us[8];
#pragma unroll
                    for (int f = 0; f < 8; ++f) {
                        uint4 u;
                        if (kOut == 1) {
                            const int c = (sg * kSeg + f * 8) / 32, i = ((sg * kSeg + f * 8) % 32) / 2;
                            u = make_uint4(p[c][i], p[c][i + 1], p[c][i + 2], p[c][i + 3]);
                        } else {
                            const int c = (sg * kSeg + f * 4) / 32, i = ((sg * kSeg + f * 4) % 32) / 2;
                            float fv[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                // exact u16 -> fp32: bits 0x4B00xxxx = 2^23 + x, minus 2^23
                                const uint32_t bits = __byte_perm(p[c][i + e / 2], 0x4B000000u, (e & 1) ? 0x7632 : 0x7610);
                                fv[e] = fmaf(__uint_as_float(bits) - 8388608.0f, fo.inv_a, fo.b_sum);
                            }
                            u = make_uint4(__float_as_uint(fv[0]), __float_as_uint(fv[1]), __float_as_uint(fv[2]),
                                           __float_as_uint(fv[3]));
                        }
                        us[f] = u;
                    }
                    if (fo.tma) {
                        // kStorePieces TMA stores per segment, one per row slice of the
                        // warp's 32 x 128-byte block (the staging layout is the tensor
                        // map's 128-byte swizzle): a slice is rewritten only once its
                        // store of the previous segment has been read (wait_group.read
                        // kStorePieces - 1), so stores stay in flight while the next
                        // slice is staged
#pragma unroll
                        for (int hh = 0; hh < kStorePieces; ++hh) {
                            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kStorePieces - 1) : "memory");
                            __syncwarp();
                            if (lane / (32 / kStorePieces) == hh) {
#pragma unroll
                                for (int f = 0; f < 8; ++f) stg[lane * 8 + (f ^ (lane & 7))] = us[f];
                            }
                            fence_proxy_async();
                            __syncwarp();
                            if (lane == 0) {
                                tma_store_2d(&omap, smem_u32(stg + hh * (256 / kStorePieces)), (int)(qb + sg * kSeg),
                                             (int)(vrow0 + (32 / kStorePieces) * hh));
                                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                            }
                        }
                        continue;
                    }
#pragma unroll
                    for (int f = 0; f < 8; ++f) stg[lane * 8 + (f ^ (lane & 7))] = us[f];
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = 4 * i + (lane >> 3), f = lane & 7;
                        const uint4 u = stg[r * 8 + (f ^ (r & 7))];
                        const int64_t vi = vrow0 + r;
                        const int64_t q = qb + sg * kSeg + f * kQPU;  // first query of the unit
                        if (vi < vend) {
                            char* dst = static_cast<char*>(fo.out) + (vi * fo.ldo + q) * kEsz;
                            if (fo.vec && q + kQPU <= a.nq) {
                                *reinterpret_cast<uint4*>(dst) = u;
                            } else {
                                const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                                for (int e = 0; e < kQPU; ++e)
                                    if (q + e < a.nq) {
                                        if (kOut == 1) reinterpret_cast<uint16_t*>(dst)[e] = (uint16_t)(w[e / 2] >> (16 * (e & 1)));
                                        else reinterpret_cast<uint32_t*>(dst)[e] = w[e];
                                    }
                            }
                        }
                    }
                    __syncwarp();
                }
                if (lane == 0) BOLT_TRACE(tile, 27 + warp);
                continue;
            }
            // shared threshold: use the value fetched one tile ago, prefetch the next
            if constexpr (kGroup) {
                // bound = max over the G groups = 0xFFFF - min of the inverted words
                uint32_t gmin = gs[0];
#pragma unroll
                for (int g = 1; g < 4; ++g) gmin = g < ngrp ? min(gmin, gs[g]) : gmin;
                g_next = gmin;
                asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];" : "=r"(gs[0]), "=r"(gs[1]) : "l"(gg));
                asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];" : "=r"(gs[2]), "=r"(gs[3]) : "l"(gg + 2));
            }
            uint32_t hmin = gw[0];  // groups >= hG hold no list: they do not bound (treated as 0xFFFF)
#pragma unroll
            for (int g = 1; g < kUnionGroups; ++g) hmin = min(hmin, g < hG ? gw[g] : 0xFFFFu);
            thr = min(min(own, 0xFFFFu - g_next + 1u), 0xFFFFu - hmin + 1u);
            if (tile >= 1 && thr > 0xFFFFu) BOLT_PROF_WARP(17, 1);  // lanes without a threshold after tile 0
            if (tile == 1) BOLT_PROF_ADD(18, thr);
            if (share) {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g_next) : "l"(gq));
                load_union();
            }
            const int tbl = tile * C::N;  // local index of the tile's first vector
            const int nvalid = (int)min64(C::N, vend - vbeg - tbl);
            // packed u16x2 tree over the warp's 128 columns; the four chunk
            // (32-column) minima route the slow path
            uint32_t cb[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t g[6];
#pragma unroll
                for (int i = 0; i < 5; ++i)
                    g[i] = kDot ? __vimax3_u16x2(p[c][3 * i], p[c][3 * i + 1], p[c][3 * i + 2])
                                : __vimin3_u16x2(p[c][3 * i], p[c][3 * i + 1], p[c][3 * i + 2]);
                g[5] = p[c][15];
                cb[c] = kDot ? __vmaxu2(__vimax3_u16x2(g[0], g[1], g[2]), __vimax3_u16x2(g[3], g[4], g[5]))
                             : __vminu2(__vimin3_u16x2(g[0], g[1], g[2]), __vimin3_u16x2(g[3], g[4], g[5]));
            }
            const uint32_t u = kDot ? __vimax3_u16x2(cb[0], cb[1], __vmaxu2(cb[2], cb[3]))
                                    : __vimin3_u16x2(cb[0], cb[1], __vminu2(cb[2], cb[3]));
            const uint32_t best = kDot ? max(u & 0xFFFFu, u >> 16) : min(u & 0xFFFFu, u >> 16);
            const uint32_t kvbest = kDot ? C::KVMAX - best : best;
            const bool tail = nvalid < C::N;
            if (xmode & 4) {  // diagnostic: filter only, never the slow path
                if (kvbest == 0xFFFFFFFFu) list.insert(kvbest);
                if (lane == 0) BOLT_TRACE(tile, 27 + warp);
                continue;
            }
            if (kvbest < thr || tail) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int col = half * kCols + c * 32;
                    const uint32_t cbest = kDot ? max(cb[c] & 0xFFFFu, cb[c] >> 16) : min(cb[c] & 0xFFFFu, cb[c] >> 16);
                    const int nleft = nvalid - col;
                    if ((kDot ? C::KVMAX - cbest : cbest) >= thr && nleft >= 32) continue;
                    BOLT_PROF_WARP(9, 1);   // lane slow-path entries
                    BOLT_PROF_WARP(11, 0);  // warp-chunk slow-path entries
                    BOLT_PROF_WARP(tile < 8 ? 12 : tile < 64 ? 13 : tile < 256 ? 14 : 15, 0);  // ... by tile index
                    // slow path (lane-divergent): candidate mask, values parked in
                    // this thread's scratch row, per-lane loop over its candidates
                    uint32_t mask = thr == kNotFull ? 0xFFFFFFFFu
                                                    : candidate_mask<kDot>(p[c], (kDot ? C::KVMAX - thr : thr) * 0x10001u);
#if BOLT_TC_ONECAND
                    // one candidate: it is the chunk's best value (every other
                    // value is at or above thr), so no scratch round trip
                    if ((mask & (mask - 1)) == 0) {
                        if (mask) {
                            const int bpos = __ffs(mask) - 1;
                            const int j = 4 * (bpos & 7) + (bpos >> 3);
                            const uint32_t kv = kDot ? C::KVMAX - cbest : cbest;
                            const uint32_t key = (kv << C::IDX_BITS) | (uint32_t)(tbl + col + j);
                            if (key < list.v[KMAX - 1] && j < nleft) {
                                list.insert(key);
                                own = list.threshold(C::IDX_BITS);
                                thr = min(thr, own);
                                changed = true;
                            }
                        }
                        continue;
                    }
#endif
                    uint4* sv = reinterpret_cast<uint4*>(scratch);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        sv[i] = make_uint4(p[c][4 * i], p[c][4 * i + 1], p[c][4 * i + 2], p[c][4 * i + 3]);
                    // The mask's bit order is not column order (bit 8i + r <->
                    // column 4r + i), so a candidate may follow a higher-index
                    // one of the same chunk.  Its own-list test is therefore on
                    // the full 32-bit key (value, then index), never the value
                    // alone: a lower index with the k-th key's value still
                    // displaces it.  The shared bounds (kv <= T) already hold
                    // for every mask bit.
                    while (mask) {
                        BOLT_PROF_WARP(16, 0);  // warp iterations of the candidate loop
                        const int bpos = __ffs(mask) - 1;
                        mask &= mask - 1;
                        const int j = 4 * (bpos & 7) + (bpos >> 3);
                        const uint32_t v = (scratch[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu;
                        const uint32_t kv = kDot ? C::KVMAX - v : v;
                        const uint32_t key = (kv << C::IDX_BITS) | (uint32_t)(tbl + col + j);
                        if (key < list.v[KMAX - 1] && j < nleft) {
                            list.insert(key);
                            own = list.threshold(C::IDX_BITS);
                            thr = min(thr, own);
                            changed = true;
                            BOLT_PROF_WARP(10, 1);  // inserts
                        }
                    }
                }
            }
            __syncwarp();  // reconverge before the next tile's .aligned tcgen05.ld
            if (lane == 0) BOLT_PROF_ADD(8, BOLT_CLOCK() - tp0);  // processing cycles (all warps)
            if (lane == 0) BOLT_TRACE(tile, 27 + warp);
            if (own < published && qvalid) {
                published = own;
                asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(kGroup ? gg + grp : gq), "r"(0xFFFFu - own)
                             : "memory");
            }
            if (changed && qvalid && share) {
                changed = false;
                const uint32_t own_h = list.value_at(hpos, C::IDX_BITS);
                if (own_h < published_h) {  // published_h = 0 for k == 1 (the union bound is own)
                    published_h = own_h;
                    asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(gh + hgrp), "r"(0xFFFFu - own_h)
                                 : "memory");
                }
            }
        }
        if (kOut != 0 && fo.tma && lane == 0)  // TMA stores of this warp complete before exit
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        if (kOut == 0 && q0 + q < a.nq) {
            uint64_t* dst = part_keys + ((int64_t)(2 * part + half) * a.nq + q0 + q) * k;
#pragma unroll
            for (int i = 0; i < KMAX; ++i) {
                if (i >= KMAX - k) {
                    const uint32_t key = list.v[i];
                    uint64_t out = ~0ull;
                    if (key != 0xFFFFFFFFu) {
                        const uint32_t kvp = key >> C::IDX_BITS;
                        const uint32_t kv64 = kDot ? 0xFFFFu - (C::KVMAX - kvp) : kvp;  // (R13) 0xFFFF - acc
                        out = make_key(kv64, (uint64_t)(index_base + vbeg + (key & ((1u << C::IDX_BITS) - 1u))));
                    }
                    dst[i - (KMAX - k)] = out;
                }
            }
        }
        if (kOut == 0) {
            // this CTA's lists are written: count it in done[part][tq] (release)
            asm volatile("bar.sync 1, %0;" ::"n"(kEpilogue) : "memory");
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(done + (int64_t)part * tiles_q + tq, 1u);
            }
        }
      }
    } else if (warp == kMmaWarp && rank == 0) {
        // ------------------------------------------- MMA issuer (leader CTA)
        if (lane == 0) {
            const uint32_t a_base = smem_u32(sA);
            const uint32_t b_base = smem_u32(sB);
            for (int tile = 0; tile < ntiles; ++tile) {
                const int s = tile % S, d = tile & 1;
                long long t0 = BOLT_CLOCK();
                mbar_wait_cluster(&full[s], (tile / S) & 1);
                long long t1 = BOLT_CLOCK();
                mbar_wait_cluster(&tempty[d], ((tile >> 1) & 1) ^ 1);
                long long t2 = BOLT_CLOCK();
                BOLT_PROF_ADD(3, t1 - t0);  // MMA waits on full
                BOLT_TRACE(tile, 0);
                BOLT_PROF_ADD(4, t2 - t1);  // MMA waits on tempty
                BOLT_TRACE(tile, 1);
                BOLT_PROF_ADD(5, 1);        // tiles
                tc_fence_after();
                const uint32_t bs = b_base + s * C::B_BYTES;
#pragma unroll
                for (int ks = 0; ks < C::KSTEPS; ++ks) {
                    // K step ks covers 16-byte chunks 2ks, 2ks+1 (same offsets in the peer CTA)
                    const uint64_t ad = smem_desc(a_base + 2 * ks * (C::QR * 16), C::QR * 16, 128);
                    const uint64_t bd = smem_desc(bs + 2 * ks * (C::NH * 16), C::NH * 16, 128);
                    // top-k: D[query][vector] (A = tables); full output: the roles swap,
                    // D[vector][query] (A = one-hot), so that an epilogue thread owns
                    // consecutive queries of one output row
                    if (kOut == 0 && !kPairT)
                        mma_i8_single(tmem + (uint32_t)(d * C::N), ad, bd, C::IDESC, ks > 0 ? 1u : 0u);
                    else if (kOut == 0) mma_i8_pair(tmem + (uint32_t)(d * C::N), ad, bd, C::IDESC, ks > 0 ? 1u : 0u);
                    else if (kOut == 3)
                        mma_i8_pair(tmem + (uint32_t)(d * kNQ), bd, ad, C::IDESC_SW, ks > 0 ? 1u : 0u);
                    else mma_i8_pair(tmem + (uint32_t)(d * C::N), bd, ad, C::IDESC, ks > 0 ? 1u : 0u);
                }
                if constexpr (kPairT) {
                    mma_commit_pair(&empty[s]);
                    mma_commit_pair(&tfull[d]);
                } else {
                    mma_commit_single(&empty[s]);
                    mma_commit_single(&tfull[d]);
                }
                BOLT_TRACE(tile, 2);
            }
        }
        __syncwarp();
    }
    if (threadIdx.x == 0) BOLT_PROF_ADD(6, BOLT_CLOCK() - tk0);   // CTA main-loop cycles
    if (threadIdx.x == 0) BOLT_PROF_ADD(7, 1);                    // CTAs
    tc_fence_before();
    if constexpr (kPairT) cluster_sync();  // all MMAs done and consumed in both CTAs
    else __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        if constexpr (kPairT)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                         "r"((uint32_t)C::TMEM_COLS)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                         "r"((uint32_t)C::TMEM_COLS)
                         : "memory");
    }
}

template <int M, bool kDot, int KMAX, int kOut = 0, bool kGroup = false, int kNQ = 0, bool kPairT = true>
cudaError_t launch_mk(const ScanArgs& a, int k, int64_t index_base, int rparts, uint64_t* part_keys,
                      uint32_t* gthr, cudaStream_t s, FullOut fo = FullOut{},
                      const CUtensorMap& omap = CUtensorMap{}) {
    using C = Cfg<M, (kOut == 1 || kOut == 2), (kOut == 3 ? kNQ / 2 : kQM),
                  (kOut == 3 ? kEpiWarps * (kNQ / 2) * 32 * 4 : 0), kPairT>;
    const int tiles_q = (int)ceil_div(a.nq, (kPairT ? 2 : 1) * C::QR);
    // full output with TMA stores: partitions of whole 256-vector tiles, so that
    // a tile's 256 rows never reach into the next partition
    const int64_t vpp = fo.tma ? ceil_div(ceil_div(a.n, rparts), C::N) * C::N : ceil_div(ceil_div(a.n, rparts), 8) * 8;
    auto kern = topk_tc_kernel<M, kDot, KMAX, kOut, kGroup, kNQ, kPairT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)((kPairT ? 2 : 1) * tiles_q * rparts));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = kPairT ? 1 : 0;  // single-CTA tiles: no cluster
    int xmode = 0;
#ifdef BOLT_XMODE
    if (const char* x = getenv("BOLT_TC_XMODE")) xmode = atoi(x);
#endif
    // shared thresholds: [nq] k-th-value words, then (16 B aligned) [nq][8] union-group words
    if (kOut == 3) {  // swapped top-k: [nq] k-th-value words
        cudaError_t e = cudaMemsetAsync(gthr, 0, (size_t)a.nq * sizeof(uint32_t), s);
        if (e != cudaSuccess) return e;
    } else if (kOut == 0 && kGroup) {  // large k: [nq][4] group words instead, then the done counters
        const int64_t tq_count = ceil_div(a.nq, (kPairT ? 2 : 1) * C::QR);
        cudaError_t e = cudaMemsetAsync(gthr, 0, (size_t)(a.nq * 4 + rparts * tq_count) * sizeof(uint32_t), s);
        if (e != cudaSuccess) return e;
    } else if (kOut == 0 && !(xmode & 16)) {  // diagnostic 16: keep caller-prefilled shared thresholds
        const int64_t hoff = (a.nq + 3) & ~int64_t(3);
        const int64_t tq_count = ceil_div(a.nq, (kPairT ? 2 : 1) * C::QR);
        cudaError_t e = cudaMemsetAsync(gthr, 0, (size_t)(hoff + 8 * a.nq + rparts * tq_count) * sizeof(uint32_t), s);
        if (e != cudaSuccess) return e;
    }
    return cudaLaunchKernelEx(&cfg, kern, a, k, index_base, vpp, tiles_q, part_keys, gthr, xmode, fo, omap);
}

// full [n][nq] output: u16 sums (out32 == nullptr) or fp32 dequantised
template <int M>
cudaError_t launch_full_m(const ScanArgs& a, int rparts, FullOut fo, const CUtensorMap& omap, bool f32,
                          cudaStream_t s) {
    return f32 ? launch_mk<M, false, 4, 2>(a, 1, 0, rparts, nullptr, nullptr, s, fo, omap)
               : launch_mk<M, false, 4, 1>(a, 1, 0, rparts, nullptr, nullptr, s, fo, omap);
}

using bolt::encode_tiled;

template <int M, bool kPairT>
cudaError_t launch_mp(const ScanArgs& a, int k, int metric, int64_t index_base, int rparts, uint64_t* part_keys,
                      uint32_t* gthr, cudaStream_t s) {
    const bool dot = metric == BOLT_DOT;
    // register list capacity: smallest of {4, 10, 12, 16, 32} >= k (bubble cost ~ 3 KMAX)
    if (k <= 4)
        return dot ? launch_mk<M, true, 4, 0, false, 0, kPairT>(a, k, index_base, rparts, part_keys, gthr, s)
                   : launch_mk<M, false, 4, 0, false, 0, kPairT>(a, k, index_base, rparts, part_keys, gthr, s);
#if BOLT_TC_KMAX10
    if (k <= 10)
        return dot ? launch_mk<M, true, 10, 0, false, 0, kPairT>(a, k, index_base, rparts, part_keys, gthr, s)
                   : launch_mk<M, false, 10, 0, false, 0, kPairT>(a, k, index_base, rparts, part_keys, gthr, s);
#endif
    if (k <= 12)
        return dot ? launch_mk<M, true, 12, 0, false, 0, kPairT>(a, k, index_base, rparts, part_keys, gthr, s)
                   : launch_mk<M, false, 12, 0, false, 0, kPairT>(a, k, index_base, rparts, part_keys, gthr, s);
    if (k <= 16)
        return dot ? launch_mk<M, true, 16, 0, false, 0, kPairT>(a, k, index_base, rparts, part_keys, gthr, s)
                   : launch_mk<M, false, 16, 0, false, 0, kPairT>(a, k, index_base, rparts, part_keys, gthr, s);
    if constexpr (kPairT)
        if (a.noshare > 0)  // lists of 32 for k > 32: group-shared thresholds
            return dot ? launch_mk<M, true, 32, 0, true>(a, k, index_base, rparts, part_keys, gthr, s)
                       : launch_mk<M, false, 32, 0, true>(a, k, index_base, rparts, part_keys, gthr, s);
    return dot ? launch_mk<M, true, 32, 0, false, 0, kPairT>(a, k, index_base, rparts, part_keys, gthr, s)
               : launch_mk<M, false, 32, 0, false, 0, kPairT>(a, k, index_base, rparts, part_keys, gthr, s);
}

// Single-CTA tiles (cta_group::1, 128 queries per CTA) for batches of at
// most 128 queries: a 128-query pair tile would be half padding, and a
// K = 32 step costs the same ~133 cycles per SM for 128 query rows either
// way, so one CTA per 256-vector tile doubles the vectors per SM.
// M <= 16 only: a 256-vector stage of M = 32 one-hot is 128 KB (no double buffer).
inline bool tc_single(int64_t nq, int m, int k, int noshare) {
#ifdef BOLT_XMODE
    if (getenv("BOLT_TC_NO_SINGLE")) return false;  // diagnostic A/B (tools/)
#endif
    return nq <= kQM && m <= 16 && k <= 32 && noshare == 0;
}

template <int M>
cudaError_t launch_m(const ScanArgs& a, int k, int metric, int64_t index_base, int rparts, uint64_t* part_keys,
                     uint32_t* gthr, cudaStream_t s) {
    if constexpr (M <= 16)
        if (tc_single(a.nq, M, k, a.noshare))
            return launch_mp<M, false>(a, k, metric, index_base, rparts, part_keys, gthr, s);
    return launch_mp<M, true>(a, k, metric, index_base, rparts, part_keys, gthr, s);
}

}  // namespace tc

int scan_tc_supported(int64_t n, int m, int64_t nq) {
    return n >= 1 && nq >= 1 && (m == 8 || m == 16 || m == 32);
}

// Full-output scan on the tensor cores (same pipeline as the top-k scan; the
// epilogue stores every sum).  Row partitions fill the SM pairs as for top-k.
cudaError_t launch_scan_tc(const ScanArgs& a, uint16_t* out16, float* out32, int64_t ldo, float inv_a, float b_sum,
                           int sms, cudaStream_t s) {
    // one wave of long units: the per-unit prologue (barriers, TMEM, the
    // query tables) would dominate short ones
    const int64_t tiles_q = ceil_div(a.nq, 2 * tc::kQM);
    const int64_t pairs = sms / 2;
    int rparts = (int)max64(1, min64(pairs / max64(tiles_q, 1), ceil_div(a.groups, 32)));
#ifdef BOLT_XMODE
    if (const char* e = getenv("BOLT_TC_RPARTS")) rparts = atoi(e);  // diagnostic sweeps (tools/)
#endif
    void* out = out32 ? static_cast<void*>(out32) : static_cast<void*>(out16);
    const int esz = out32 ? 4 : 2;
    const int vec = (reinterpret_cast<uintptr_t>(out) % 16 == 0) && ((ldo * esz) % 16 == 0);
    // TMA stores of the staged 32-row x 128-byte blocks: a 2-D tensor map over
    // out [n][nq] (row stride ldo) with the 128-byte swizzle of the staging
    // layout; the hardware clips rows >= n and queries >= nq
    CUtensorMap omap{};
    int tma = 0;
    if (vec && encode_tiled()) {
        const cuuint64_t dims[2] = {(cuuint64_t)a.nq, (cuuint64_t)a.n};
        const cuuint64_t strides[1] = {(cuuint64_t)(ldo * esz)};
        const cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)(32 / tc::kStorePieces)};  // a row slice of a warp's block
        const cuuint32_t estr[2] = {1u, 1u};
        tma = encode_tiled()(&omap, out32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, out,
                             dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    tc::FullOut fo{out, ldo, inv_a, b_sum, vec, tma};
    switch (a.m) {
        case 8: return tc::launch_full_m<8>(a, rparts, fo, omap, out32 != nullptr, s);
        case 16: return tc::launch_full_m<16>(a, rparts, fo, omap, out32 != nullptr, s);
        case 32: return tc::launch_full_m<32>(a, rparts, fo, omap, out32 != nullptr, s);
        default: return cudaErrorInvalidValue;
    }
}

int topk_tc_supported(int64_t n, int m, int64_t nq, int k) {
    (void)nq;
    // k <= 32: register lists of k; 32 < k <= 128: lists of 32 + exactness check (api.cu)
    return n >= 1 && k >= 1 && k <= kMaxK && (m == 8 || m == 16 || m == 32);
}

// Units = query tiles (256 per CTA pair, 128 per single CTA) x row partitions, the
// partition count chosen so units fill whole waves of SM pairs (>= 4
// waves), with at least 16 vector tiles per unit and each unit's range
// within the epilogue's local index bits.  Two partial lists per unit (the
// two column-half epilogue warps).
int topk_tc_parts(int64_t n, int m, int64_t nq, int k, int num_sms) {
    const bool single = tc::tc_single(nq, m, k, k > 32 ? 1 : 0);  // k > 32: pair lists of 32 (api.cu)
    const int64_t tiles_q = ceil_div(nq, (single ? 1 : 2) * tc::kQM);
    const int64_t max_range = m == 8 ? tc::Cfg<8>::MAX_RANGE : (m == 16 ? tc::Cfg<16>::MAX_RANGE : tc::Cfg<32>::MAX_RANGE);
    // finer units where one query tile spans the batch (measured: DESIGN.md §6.1 "Unit count")
    const int64_t W = single ? 4 * num_sms : (m == 32 && tiles_q == 1 ? num_sms : num_sms / 2);
    int rparts = choose_parts(tiles_q, ceil_div(n, 8), W, (int64_t)256 * 16 / 8);
    rparts = (int)max64(rparts, ceil_div(n, max_range - 8));
    return 2 * rparts;
}

namespace tc {

// Swapped top-k (kOut = 3): small query batches, vectors on the MMA's M side.
template <int M, int kNQ>
cudaError_t launch_sw_q(const ScanArgs& a, int k, int metric, int64_t index_base, int rparts, uint64_t* part_keys,
                        uint32_t* gthr, cudaStream_t s) {
    return metric == BOLT_DOT ? launch_mk<M, true, 4, 3, false, kNQ>(a, k, index_base, rparts, part_keys, gthr, s)
                              : launch_mk<M, false, 4, 3, false, kNQ>(a, k, index_base, rparts, part_keys, gthr, s);
}
template <int M>
cudaError_t launch_sw_m(const ScanArgs& a, int k, int metric, int64_t index_base, int rparts, uint64_t* part_keys,
                        uint32_t* gthr, cudaStream_t s) {
    if (a.nq <= 32) return launch_sw_q<M, 32>(a, k, metric, index_base, rparts, part_keys, gthr, s);
    if (a.nq <= 64) return launch_sw_q<M, 64>(a, k, metric, index_base, rparts, part_keys, gthr, s);
    return launch_sw_q<M, 128>(a, k, metric, index_base, rparts, part_keys, gthr, s);
}

}  // namespace tc

int topk_tcs_supported(int64_t n, int m, int64_t nq, int k) {
    return n >= 1 && nq >= 1 && nq <= 128 && k >= 1 && k <= 32 && (m == 8 || m == 16 || m == 32);
}

// 8 lists per query per row partition (2 CTAs x 4 quads); one wave of pairs
// or more, each partition within the local index range
int topk_tcs_parts(int64_t n, int m, int64_t nq, int k, int num_sms) {
    (void)nq;
    (void)k;
    const int64_t max_range = m == 8 ? tc::Cfg<8>::MAX_RANGE : (m == 16 ? tc::Cfg<16>::MAX_RANGE : tc::Cfg<32>::MAX_RANGE);
    int rparts = choose_parts(1, ceil_div(n, 8), num_sms / 2, (int64_t)256 * 16 / 8);
    rparts = (int)max64(rparts, ceil_div(n, max_range - 8));
    return 8 * rparts;
}

// part_keys: parts*nq*k keys followed by nq u32 shared thresholds
cudaError_t launch_topk_tcs(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                            uint64_t* part_keys, cudaStream_t s) {
    uint32_t* gthr = reinterpret_cast<uint32_t*>(part_keys + (size_t)parts * a.nq * k);
    const int rparts = parts / 8;
    switch (a.m) {
        case 8: return tc::launch_sw_m<8>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        case 16: return tc::launch_sw_m<16>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        case 32: return tc::launch_sw_m<32>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        default: return cudaErrorInvalidValue;
    }
}

// part_keys holds parts*nq*k keys followed by nq u32 shared thresholds.
cudaError_t launch_topk_tc(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                           uint64_t* part_keys, int sms, cudaStream_t s) {
    (void)sms;
    const int rparts = parts / 2;
    uint32_t* gthr = reinterpret_cast<uint32_t*>(part_keys + (size_t)parts * a.nq * k);
    switch (a.m) {
        case 8: return tc::launch_m<8>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        case 16: return tc::launch_m<16>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        case 32: return tc::launch_m<32>(a, k, metric, index_base, rparts, part_keys, gthr, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace bolt
