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
// Per CTA (one per SM): a tile of 128 queries (MMA M) against a contiguous
// range of database vectors in tiles of N vectors (N = 256 for M <= 16).
//   warps 0-3  producers: stage A once (16-byte units, K-major "interleave"
//              layout), then expand each vector tile's codes into the one-hot
//              B tile in shared memory (one aligned 16-byte store per
//              (vector, codebook)), double-buffered.
//   warp  8    MMA issuer (one thread): M/2 x tcgen05.mma (K = 32 bytes each)
//              into one of two TMEM accumulators, commit to mbarriers.
//   warps 4-7  epilogue: thread = query (TMEM lane); tcgen05.ld the N sums,
//              min/max-reduce against the query's running top-k threshold,
//              rare inserts into the query's sorted key list (shared memory).
// Shared-memory operand layout (both K-major, SWIZZLE_NONE): the 16-byte
// chunk j of row r lives at j * (rows * 16) + (r / 8) * 128 + (r % 8) * 16,
// so SBO (next 8 rows) = 128 B and LBO (next 16-byte K chunk) = rows * 16 B.
#include "common.cuh"
#include "topk_list.cuh"

namespace bolt {
namespace tc {

constexpr int kQM = 128;                 // queries per tile = MMA M = TMEM lanes
constexpr int kProducers = 128;
constexpr int kEpiWarps = 8;             // two warps per TMEM lane quadrant (column halves)
constexpr int kEpilogue = kEpiWarps * 32;
constexpr int kMmaWarp = 4 + kEpiWarps;
constexpr int kThreads = (kMmaWarp + 1) * 32;  // 4 producer + 8 epilogue + 1 MMA warp
constexpr int kMaxTopk = 32;

template <int M>
struct Cfg {
    static constexpr int K = 16 * M;                        // bytes per row
    static constexpr int N = (4096 / M) < 256 ? (4096 / M) : 256;  // vectors per tile
    static constexpr int A_BYTES = kQM * K;
    static constexpr int B_BYTES = N * K;
    static constexpr int KSTEPS = K / 32;
    static constexpr int TMEM_COLS = 2 * N <= 32 ? 32 : (2 * N <= 64 ? 64 : (2 * N <= 128 ? 128 : (2 * N <= 256 ? 256 : 512)));
    // dynamic smem: A | B0 | B1 | code stages [2][N*M/8] u32 | barriers
    static constexpr int STAGE_OFF = A_BYTES + 2 * B_BYTES;
    static constexpr int BAR_OFF = STAGE_OFF + 2 * N * M / 2;
    static constexpr int SMEM = BAR_OFF + 128;
    // instruction descriptor: D s32 (bits 4-5 = 2), A/B u8 (format 0), K-major,
    // N >> 3 at bit 17, M >> 4 at bit 24
    static constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kQM >> 4) << 24);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major SWIZZLE_NONE shared-memory matrix descriptor (sm_100 version 1)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32-bit shift with PTX clamping (shift amounts >= 32, including "negative"
// ones seen as unsigned, give 0)
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t s) {
    uint32_t d;
    asm("shl.b32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(s));
    return d;
}
// one-hot of a 4-bit code as 16 bytes: byte `code` = 1 (s = 8 * code)
__device__ __forceinline__ uint4 one_hot16_s(uint32_t s) {
    return make_uint4(shl_clamp(1u, s), shl_clamp(1u, s - 32u), shl_clamp(1u, s - 64u), shl_clamp(1u, s - 96u));
}

__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
    return r;
}

// Register-resident sorted top-k list of one thread, right-aligned in KMAX
// slots: slots [0, KMAX-k) hold 0 (passes every key through), slots
// [KMAX-k, KMAX) the k best keys ascending, so the k-th best is always
// slot KMAX-1.  Insert = one branch-free bubble pass.
template <int KMAX>
struct RegList {
    uint64_t v[KMAX];
    __device__ __forceinline__ void init(int k) {
#pragma unroll
        for (int i = 0; i < KMAX; ++i) v[i] = i < KMAX - k ? 0ull : ~0ull;
    }
    __device__ __forceinline__ void insert(uint64_t c) {
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
            const bool lt = v[i] < c;
            const uint64_t lo = lt ? v[i] : c;
            c = lt ? c : v[i];
            v[i] = lo;
        }
    }
    __device__ __forceinline__ uint32_t threshold() const {
        return v[KMAX - 1] == ~0ull ? kNotFull : (uint32_t)(v[KMAX - 1] >> 48);
    }
};

}  // namespace tc
}  // namespace bolt

namespace bolt {
namespace tc {

template <int M, bool kDot, int KMAX>
__global__ void __launch_bounds__(kThreads, 1)
topk_tc_kernel(ScanArgs a, int k, int64_t index_base, int parts, int64_t vpp, int tiles_q,
               uint64_t* __restrict__ part_keys) {
    using C = Cfg<M>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::A_BYTES;
    uint32_t* stages = reinterpret_cast<uint32_t*>(smem + C::STAGE_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* full = bars;            // [2] producers -> MMA (count 128)
    uint64_t* empty = bars + 2;       // [2] MMA commit -> producers
    uint64_t* tfull = bars + 4;       // [2] MMA commit -> epilogue
    uint64_t* tempty = bars + 6;      // [2] epilogue -> MMA (count 128)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int unit = blockIdx.x;
    const int tq = unit % tiles_q;
    const int part = unit / tiles_q;
    const int64_t q0 = (int64_t)tq * kQM;
    const int64_t vbeg = (int64_t)part * vpp;
    const int64_t vend = min64(a.n, vbeg + vpp);
    const int ntiles = vend > vbeg ? (int)ceil_div(vend - vbeg, C::N) : 0;

    if (threadIdx.x == 0) {
        mbar_init(&full[0], kProducers);
        mbar_init(&full[1], kProducers);
        mbar_init(&empty[0], 1);
        mbar_init(&empty[1], 1);
        mbar_init(&tfull[0], 1);
        mbar_init(&tfull[1], 1);
        mbar_init(&tempty[0], kEpilogue);
        mbar_init(&tempty[1], kEpilogue);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"((uint32_t)C::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
        // ------------------------------------------------------ producers
        const int t = threadIdx.x;
        // A: query tables, 16-byte unit (c, q) -> c * (128*16) + (q/8)*128 + (q%8)*16
        for (int u = t; u < kQM * M; u += kProducers) {
            const int c = u / kQM, q = u % kQM;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (q0 + q < a.nq) v = __ldg(reinterpret_cast<const uint4*>(a.qluts + ((q0 + q) * M + c) * kK));
            *reinterpret_cast<uint4*>(sA + c * (kQM * 16) + (q >> 3) * 128 + (q & 7) * 16) = v;
        }
        // codes of a tile = N/8 groups x M words, contiguous: one uint4 per thread
        constexpr int kChunks = C::N * M / 32;  // uint4 per tile (<= 128)
        static_assert(kChunks <= kProducers, "tile code block must fit one uint4 per producer");
        const int64_t words_total = a.groups * M;
        auto load_chunk = [&](int tile) -> uint4 {
            const int64_t w0 = ((vbeg + (int64_t)tile * C::N) >> 3) * M + (int64_t)t * 4;
            if (t < kChunks && w0 < words_total) return __ldg(reinterpret_cast<const uint4*>(a.codes + w0));
            return make_uint4(0, 0, 0, 0);
        };
        uint4 pre = ntiles > 0 ? load_chunk(0) : make_uint4(0, 0, 0, 0);
        constexpr int kVecPerThread = C::N / kProducers > 0 ? C::N / kProducers : 1;
        for (int tile = 0; tile < ntiles; ++tile) {
            const int s = tile & 1;
            mbar_wait(&empty[s], ((tile >> 1) & 1) ^ 1);
            uint32_t* stage = stages + s * (C::N * M / 8);
            if (t < kChunks) reinterpret_cast<uint4*>(stage)[t] = pre;
            asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
            if (tile + 1 < ntiles) pre = load_chunk(tile + 1);
            uint8_t* b = sB + s * C::B_BYTES;
            const int64_t tb = vbeg + (int64_t)tile * C::N;
#pragma unroll
            for (int h = 0; h < kVecPerThread; ++h) {
                const int v = t + h * kProducers;
                if (v >= C::N) break;
                const bool valid = tb + v < vend;
                const uint32_t* wv = stage + (v >> 3) * M;
                const uint32_t sh = (v & 7) * 4;
#pragma unroll
                for (int c4 = 0; c4 < M; c4 += 4) {
                    const uint4 w = *reinterpret_cast<const uint4*>(wv + c4);
                    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t sbits = valid ? ((ws[j] >> sh) & 0xFu) * 8u : 128u;  // 128 -> zeros
                        *reinterpret_cast<uint4*>(b + (c4 + j) * (C::N * 16) + v * 16) = one_hot16_s(sbits);
                    }
                }
            }
            fence_proxy_async();
            mbar_arrive(&full[s]);
        }
    } else if (warp < 4 + kEpiWarps) {
        // ------------------------------------------------------- epilogue
        const int quad = warp & 3;                 // TMEM lanes 32*quad .. (warp % 4 rule)
        const int half = (warp - 4) >> 2;          // column half of the tile
        const int q = quad * 32 + lane;            // query row of the tile
        constexpr int kCols = C::N / 2;
        RegList<KMAX> list;
        list.init(k);
        uint32_t thr = kNotFull;
        const uint32_t tlane = (uint32_t)(quad * 32) << 16;
        for (int tile = 0; tile < ntiles; ++tile) {
            const int d = tile & 1;
            mbar_wait(&tfull[d], (tile >> 1) & 1);
            tc_fence_after();
            const int64_t tb = vbeg + (int64_t)tile * C::N;
            const int nvalid = (int)min64(C::N, vend - tb);
#pragma unroll 1
            for (int col = half * kCols; col < (half + 1) * kCols; col += 32) {
                const uint32_t tcol = tmem + tlane + (uint32_t)(d * C::N + col);
                uint32_t r[32];
                tmem_ld32(tcol, r);
                tmem_wait_ld();
                // tree reduction on a copy: best (smallest kv) of the 32 columns
                uint32_t t[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) t[j] = kDot ? max(r[j], r[j + 16]) : min(r[j], r[j + 16]);
#pragma unroll
                for (int w = 8; w > 0; w >>= 1)
#pragma unroll
                    for (int j = 0; j < w; ++j) t[j] = kDot ? max(t[j], t[j + w]) : min(t[j], t[j + w]);
                const uint32_t kvbest = kDot ? 0xFFFFu - t[0] : t[0];
                const bool trig = kvbest < thr || col + 32 > nvalid;
                if (!__any_sync(0xffffffffu, trig)) continue;
                // slow path: per-lane candidate columns, then a warp-uniform walk
                // over the union re-reading single TMEM columns
                uint32_t mask = 0;
                if (trig) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t kv = kDot ? 0xFFFFu - r[j] : r[j];
                        mask |= (kv < thr && col + j < nvalid) ? (1u << j) : 0u;
                    }
                }
                uint32_t wm = __reduce_or_sync(0xffffffffu, mask);
                while (wm) {
                    const int j = __ffs(wm) - 1;
                    wm &= wm - 1;
                    const uint32_t v = tmem_ld1(tcol + j);
                    tmem_wait_ld();
                    const uint32_t kv = kDot ? 0xFFFFu - v : v;
                    if (((mask >> j) & 1u) && kv < thr) {
                        list.insert(make_key(kv, (uint64_t)(index_base + tb + col + j)));
                        thr = list.threshold();
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[d]);
        }
        if (q0 + q < a.nq) {
            uint64_t* dst = part_keys + ((int64_t)(2 * part + half) * a.nq + q0 + q) * k;
#pragma unroll
            for (int i = 0; i < KMAX; ++i)
                if (i >= KMAX - k) dst[i - (KMAX - k)] = list.v[i];
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t a_base = smem_u32(sA);
            const uint32_t b_base = smem_u32(sB);
            for (int tile = 0; tile < ntiles; ++tile) {
                const int s = tile & 1, d = tile & 1;
                mbar_wait(&full[s], (tile >> 1) & 1);
                mbar_wait(&tempty[d], ((tile >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t bs = b_base + s * C::B_BYTES;
#pragma unroll
                for (int ks = 0; ks < C::KSTEPS; ++ks) {
                    // K step ks covers 16-byte chunks 2ks, 2ks+1
                    const uint64_t ad = smem_desc(a_base + 2 * ks * (kQM * 16), kQM * 16, 128);
                    const uint64_t bd = smem_desc(bs + 2 * ks * (C::N * 16), C::N * 16, 128);
                    mma_i8(tmem + (uint32_t)(d * C::N), ad, bd, C::IDESC, ks > 0 ? 1u : 0u);
                }
                mma_commit(&empty[s]);
                mma_commit(&tfull[d]);
            }
        }
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS)
                     : "memory");
    }
}

template <int M, bool kDot, int KMAX>
cudaError_t launch_mk(const ScanArgs& a, int k, int64_t index_base, int rparts, uint64_t* part_keys,
                      cudaStream_t s) {
    using C = Cfg<M>;
    const int tiles_q = (int)ceil_div(a.nq, kQM);
    const int64_t vpp = ceil_div(ceil_div(a.n, rparts), 8) * 8;
    const unsigned grid = (unsigned)(tiles_q * rparts);
    cudaFuncSetAttribute(topk_tc_kernel<M, kDot, KMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    topk_tc_kernel<M, kDot, KMAX><<<grid, kThreads, C::SMEM, s>>>(a, k, index_base, rparts, vpp, tiles_q,
                                                                 part_keys);
    return cudaGetLastError();
}

template <int M>
cudaError_t launch_m(const ScanArgs& a, int k, int metric, int64_t index_base, int rparts, uint64_t* part_keys,
                     cudaStream_t s) {
    const bool dot = metric == BOLT_DOT;
    if (k <= 16)
        return dot ? launch_mk<M, true, 16>(a, k, index_base, rparts, part_keys, s)
                   : launch_mk<M, false, 16>(a, k, index_base, rparts, part_keys, s);
    return dot ? launch_mk<M, true, 32>(a, k, index_base, rparts, part_keys, s)
               : launch_mk<M, false, 32>(a, k, index_base, rparts, part_keys, s);
}

}  // namespace tc

int topk_tc_supported(int64_t n, int m, int64_t nq, int k) {
    (void)nq;
    return n >= 1 && k >= 1 && k <= tc::kMaxTopk && (m == 8 || m == 16 || m == 32);
}

// One CTA per SM; units = query tiles x row partitions, the partition count
// chosen so the unit count fills whole waves of the SMs (>= 4 waves), with at
// least 16 vector tiles per unit.
int topk_tc_parts(int64_t n, int m, int64_t nq, int k, int num_sms) {
    (void)k;
    const int64_t tiles_q = ceil_div(nq, tc::kQM);
    const int N = m == 8 ? tc::Cfg<8>::N : (m == 16 ? tc::Cfg<16>::N : tc::Cfg<32>::N);
    // two partial lists per row partition (the two column-half epilogue warps)
    return 2 * choose_parts(tiles_q, ceil_div(n, 8), num_sms, (int64_t)N * 16 / 8);
}

cudaError_t launch_topk_tc(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                           uint64_t* part_keys, int sms, cudaStream_t s) {
    (void)sms;
    const int rparts = parts / 2;
    switch (a.m) {
        case 8: return tc::launch_m<8>(a, k, metric, index_base, rparts, part_keys, s);
        case 16: return tc::launch_m<16>(a, k, metric, index_base, rparts, part_keys, s);
        case 32: return tc::launch_m<32>(a, k, metric, index_base, rparts, part_keys, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace bolt
