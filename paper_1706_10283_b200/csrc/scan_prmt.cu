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
#include "common.cuh"

namespace bolt {
namespace {

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
__device__ __forceinline__ void scan_group(const uint32_t* __restrict__ codes, int64_t g, int m,
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

// value of row r (0..7) from the packed totals
__device__ __forceinline__ uint32_t row_value(const uint32_t (&t)[4], int r) {
    const uint32_t pair = t[(r >> 2) * 2 + (r & 1)];
    return (r & 2) ? (pair >> 16) : (pair & 0xFFFFu);
}

// ------------------------------------------------------------ full output
template <int QT, bool kDequant>
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
    scan_group<QT>(a.codes, g, a.m, vec, full_tab, tot);
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
// A sorted key list of up to 32*KPL entries spread over the warp: position
// p = j*32 + lane lives in v[j] of that lane.
template <int KPL>
struct WarpList {
    uint64_t v[KPL];

    __device__ __forceinline__ void init() {
#pragma unroll
        for (int j = 0; j < KPL; ++j) v[j] = ~0ull;
    }
    __device__ __forceinline__ uint64_t at(int p) const {  // warp-uniform p
        uint64_t x = v[0];
#pragma unroll
        for (int j = 1; j < KPL; ++j)
            if ((p >> 5) == j) x = v[j];
        return __shfl_sync(0xffffffffu, x, p & 31);
    }
    // insert warp-uniform key c, keeping the first k positions sorted
    __device__ __forceinline__ void insert(uint64_t c, int k, int lane) {
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < KPL; ++j) cnt += __popc(__ballot_sync(0xffffffffu, v[j] < c));
        if (cnt >= k) return;
        uint64_t up[KPL];
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            uint64_t u = __shfl_up_sync(0xffffffffu, v[j], 1);
            uint64_t prev_last = j > 0 ? __shfl_sync(0xffffffffu, v[j > 0 ? j - 1 : 0], 31) : ~0ull;
            up[j] = lane == 0 ? prev_last : u;
        }
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            const int p = j * 32 + lane;
            v[j] = p < cnt ? v[j] : (p == cnt ? c : up[j]);
        }
    }
};

template <int QT, int KPL>
__global__ void __launch_bounds__(kScanThreads)
topk_prmt_kernel(ScanArgs a, int k, int metric, int64_t index_base, int parts,
                 int64_t groups_per_part, uint64_t* __restrict__ part_keys) {
    extern __shared__ uint4 topk_tab[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t q0 = (int64_t)blockIdx.y * QT;
    load_split_tables(a.qluts, a.nq, a.m, q0, QT, topk_tab);
    __syncthreads();
    const int part = blockIdx.x * kWarps + warp;
    if (part >= parts) return;
    const int64_t gbeg = (int64_t)part * groups_per_part;
    const int64_t gend = min64(a.groups, gbeg + groups_per_part);
    const bool vec = (a.m % 4) == 0;
    const uint32_t flip = metric == BOLT_DOT ? 0xFFFFFFFFu : 0u;  // kv = 0xFFFF - acc for dot

    WarpList<KPL> list[QT];
    uint32_t thr[QT];  // value part of the k-th key, 0x10000 while the list is not full
#pragma unroll
    for (int q = 0; q < QT; ++q) {
        list[q].init();
        thr[q] = 0x10000u;
    }
    for (int64_t gs = gbeg; gs < gend; gs += 32) {
        const int64_t g = gs + lane;
        const bool gvalid = g < gend;
        uint32_t tot[QT][4];
        scan_group<QT>(a.codes, gvalid ? g : gbeg, a.m, vec, topk_tab, tot);
        // number of valid rows of this lane's group
        const int nrows = gvalid ? (int)min64(8, a.n - g * 8) : 0;
#pragma unroll
        for (int q = 0; q < QT; ++q) {
            uint32_t flag = 0;
            if (thr[q] > 0xFFFFu) {
                flag = nrows > 0;
            } else {
                const uint32_t tp = thr[q] | (thr[q] << 16);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const uint32_t mn = vminu2(tot[q][t] ^ flip, tp);
                    flag |= mn ^ tp;
                }
                flag = flag != 0 && nrows > 0;
            }
            if (__ballot_sync(0xffffffffu, flag) == 0) continue;
            // slow path: candidate rows of this lane (kv < thr, or list not full)
            uint32_t pend = 0;
            if (flag) {
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const uint32_t kv = (row_value(tot[q], r) ^ flip) & 0xFFFFu;
                    if (r < nrows && kv < thr[q]) pend |= 1u << r;
                }
            }
            // insert candidates row slot by row slot (static r keeps tot[] in registers)
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint32_t kv = (row_value(tot[q], r) ^ flip) & 0xFFFFu;
                const uint64_t mine = make_key(kv, (uint64_t)(index_base + g * 8 + r));
                unsigned b = __ballot_sync(0xffffffffu, (pend >> r) & 1u);
                while (b) {
                    const int src = __ffs(b) - 1;
                    b &= b - 1;
                    list[q].insert(__shfl_sync(0xffffffffu, mine, src), k, lane);
                }
            }
            const uint64_t kth = list[q].at(k - 1);
            thr[q] = kth == ~0ull ? 0x10000u : (uint32_t)(kth >> 48);
        }
    }
    // write this warp's partial lists
#pragma unroll
    for (int q = 0; q < QT; ++q) {
        if (q0 + q >= a.nq) break;
        uint64_t* dst = part_keys + ((int64_t)part * a.nq + q0 + q) * k;
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            const int p = j * 32 + lane;
            if (p < k) dst[p] = list[q].v[j];
        }
    }
}

template <int QT>
cudaError_t launch_full_qt(const ScanArgs& a, uint16_t* out16, float* out32, int64_t ldo, float inv_a,
                           float b_sum, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(a.groups, kScanThreads), (unsigned)ceil_div(a.nq, QT));
    size_t smem = (size_t)QT * a.m * 2 * sizeof(uint4);
    if (out32)
        scan_full_kernel<QT, true><<<grid, kScanThreads, smem, s>>>(a, out16, out32, ldo, inv_a, b_sum);
    else
        scan_full_kernel<QT, false><<<grid, kScanThreads, smem, s>>>(a, out16, out32, ldo, inv_a, b_sum);
    return cudaGetLastError();
}

int pick_qt(int64_t nq) { return nq >= 8 ? 8 : nq >= 4 ? 4 : nq >= 2 ? 2 : 1; }
int pick_kpl(int k) { return k <= 32 ? 1 : k <= 64 ? 2 : 4; }

template <int QT, int KPL>
cudaError_t launch_topk_t(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                          uint64_t* part_keys, cudaStream_t s) {
    const int64_t gpp = ceil_div(a.groups, parts);
    dim3 grid((unsigned)ceil_div(parts, kWarps), (unsigned)ceil_div(a.nq, QT));
    size_t smem = (size_t)QT * a.m * 2 * sizeof(uint4);
    topk_prmt_kernel<QT, KPL><<<grid, kScanThreads, smem, s>>>(a, k, metric, index_base, parts, gpp,
                                                               part_keys);
    return cudaGetLastError();
}

template <int QT>
cudaError_t launch_topk_qt(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                           uint64_t* part_keys, cudaStream_t s) {
    switch (pick_kpl(k)) {
        case 1: return launch_topk_t<QT, 1>(a, k, metric, index_base, parts, part_keys, s);
        case 2: return launch_topk_t<QT, 2>(a, k, metric, index_base, parts, part_keys, s);
        default: return launch_topk_t<QT, 4>(a, k, metric, index_base, parts, part_keys, s);
    }
}

}  // namespace

cudaError_t launch_scan_full(const ScanArgs& a, uint16_t* out16, float* out32, int64_t ldo,
                             float inv_a, float b_sum, cudaStream_t s) {
    if (a.n == 0 || a.nq == 0) return cudaSuccess;
    switch (pick_qt(a.nq)) {
        case 8: return launch_full_qt<8>(a, out16, out32, ldo, inv_a, b_sum, s);
        case 4: return launch_full_qt<4>(a, out16, out32, ldo, inv_a, b_sum, s);
        case 2: return launch_full_qt<2>(a, out16, out32, ldo, inv_a, b_sum, s);
        default: return launch_full_qt<1>(a, out16, out32, ldo, inv_a, b_sum, s);
    }
}

// Split of the rows into `parts` contiguous partitions: enough warp tasks to
// fill the GPU (~32 per SM) while keeping >= 4 warp steps per task and the
// merge input parts*k <= 8192.
int topk_prmt_parts(int64_t n, int m, int64_t nq, int k, int num_sms) {
    (void)m;
    const int64_t groups = ceil_div(n, 8);
    int qt = pick_qt(nq);
    if (pick_kpl(k) == 2 && qt > 4) qt = 4;
    if (pick_kpl(k) == 4 && qt > 2) qt = 2;
    const int64_t tiles = ceil_div(nq, qt);
    int64_t parts = ceil_div((int64_t)num_sms * 32, tiles);
    const int64_t max_by_rows = groups / (32 * 4);
    parts = min64(parts, max64(1, max_by_rows));
    parts = min64(parts, max64(1, 8192 / k));
    parts = max64(1, parts);
    return (int)parts;
}

cudaError_t launch_topk_prmt(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                             uint64_t* part_keys, cudaStream_t s) {
    int qt = pick_qt(a.nq);
    const int kpl = pick_kpl(k);
    if (kpl == 2 && qt > 4) qt = 4;
    if (kpl == 4 && qt > 2) qt = 2;
    switch (qt) {
        case 8: return launch_topk_qt<8>(a, k, metric, index_base, parts, part_keys, s);
        case 4: return launch_topk_qt<4>(a, k, metric, index_base, parts, part_keys, s);
        case 2: return launch_topk_qt<2>(a, k, metric, index_base, parts, part_keys, s);
        default: return launch_topk_qt<1>(a, k, metric, index_base, parts, part_keys, s);
    }
}

}  // namespace bolt
