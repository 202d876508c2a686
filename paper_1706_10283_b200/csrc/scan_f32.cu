// scan_f32.cu -- "Bolt No Quantize": the scan
// with the unquantized fp32 tables, out[i][q] = sum_m D[q][m][code(i,m)].
//
// The paper keeps this variant only to show that table quantization costs no
// accuracy ("it sacrifices Bolt's high speed"); here it is the same layout-v1
// codes read against fp32 tables held in shared memory.  Sums run in fp32 in
// ascending m from 0.0f (R18), so a top-k decided by them is exact against the
// oracle given the same fp32 tables.  Lookups are LDS from a 16-word table:
// the 32 lanes of a warp (32 rows) read one (query, codebook) table, whose 16
// entries lie in 16 distinct banks -- conflict-free whatever the codes.
// Bound: shared-memory issue, one LDS (4 B) per lookup = M per distance.
//
// Keys (R18): the float's order-preserving code (negative: bits flipped, else
// the sign bit set; inverted for the dot product) << 32 | global index.
#include <cmath>

#include "common.cuh"

namespace bolt {
namespace {

constexpr int kF32Threads = 256;  // one row per thread, 32 layout-v1 groups per block
constexpr int kF32QT = 32;        // queries per block (128 B of output per row)

__device__ __forceinline__ uint64_t key_f32(float v, uint64_t gidx, int metric) {
    const uint32_t u = __float_as_uint(v);
    uint32_t ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    if (metric == BOLT_DOT) ord = ~ord;
    return ((uint64_t)ord << 32) | gidx;
}

// tables of queries [q0, q0 + QT) -> shared memory [QT][M][16] (zero past nq)
__device__ __forceinline__ void load_tables(const float* __restrict__ luts, int64_t nq, int m, int64_t q0,
                                            float* tab) {
    const int total = kF32QT * m * kK;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int64_t q = q0 + e / (m * kK);
        tab[e] = q < nq ? luts[q0 * m * kK + e] : 0.f;
    }
}

// sums of this thread's row against the QT tables (ascending m, fp32)
__device__ __forceinline__ void row_sums(const uint32_t* __restrict__ codes, int64_t row, int m, const float* tab,
                                         float (&acc)[kF32QT]) {
#pragma unroll
    for (int q = 0; q < kF32QT; ++q) acc[q] = 0.f;
    const uint32_t* wp = codes + (row >> 3) * m;
    const int sh = (int)(row & 7) * 4;
    for (int c = 0; c < m; ++c) {
        const int code = (int)((__ldg(wp + c) >> sh) & 0xFu);
        const float* t = tab + c * kK + code;
#pragma unroll
        for (int q = 0; q < kF32QT; ++q) acc[q] = __fadd_rn(acc[q], t[q * m * kK]);
    }
}

// Full output: block = 256 rows x 32 queries; each thread writes its row's
// 32 consecutive outputs (one 128-byte line when ldo allows).
__global__ void __launch_bounds__(kF32Threads)
scan_f32_kernel(const uint32_t* __restrict__ codes, int64_t n, int m, const float* __restrict__ luts, int64_t nq,
                float* __restrict__ out, int64_t ldo, int qtiles) {
    extern __shared__ float f32_tab[];
    const int64_t q0 = (int64_t)(blockIdx.x % qtiles) * kF32QT;
    const int64_t row = (int64_t)(blockIdx.x / qtiles) * kF32Threads + threadIdx.x;
    load_tables(luts, nq, m, q0, f32_tab);
    __syncthreads();
    if (row >= n) return;
    float acc[kF32QT];
    row_sums(codes, row, m, f32_tab, acc);
    float* dst = out + row * ldo + q0;
    const int nv = (int)min64(kF32QT, nq - q0);
    if (nv == kF32QT && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < kF32QT; q += 4)
            *reinterpret_cast<float4*>(dst + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
    } else {
#pragma unroll
        for (int q = 0; q < kF32QT; ++q)
            if (q < nv) dst[q] = acc[q];
    }
}

// Fused top-k: block = (query tile, row partition); warp w of the block scans
// rows (32 per step, one per lane) and keeps one sorted list of k keys per
// query in shared memory.  A lane's key enters the list only if it beats the
// list's k-th key; candidates of a step are inserted one at a time by the
// whole warp (lane l < k holds entry l; shift by shuffles).  Each warp's lists
// are one partial list per query: part index = partition * 8 + warp.
constexpr int kF32Warps = kF32Threads / 32;

__global__ void __launch_bounds__(kF32Threads)
topk_f32_kernel(const uint32_t* __restrict__ codes, int64_t n, int m, const float* __restrict__ luts, int64_t nq,
                int k, int metric, int64_t index_base, int qtiles, int64_t rows_per_warp,
                uint64_t* __restrict__ part_keys) {
    extern __shared__ float f32_tab[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t q0 = (int64_t)(blockIdx.x % qtiles) * kF32QT;
    const int64_t part = (int64_t)(blockIdx.x / qtiles) * kF32Warps + warp;
    uint64_t* lists = reinterpret_cast<uint64_t*>(f32_tab + kF32QT * m * kK) + (size_t)warp * kF32QT * k;
    load_tables(luts, nq, m, q0, f32_tab);
    for (int e = lane; e < kF32QT * k; e += 32) lists[e] = ~0ull;
    __syncthreads();
    const int64_t r0 = part * rows_per_warp;
    const int64_t r1 = min64(n, r0 + rows_per_warp);
    const int nv = (int)min64(kF32QT, nq - q0);
    // per-query threshold in registers (the same in every lane): the value of
    // the list's k-th key once the list is full; a lane's value is a
    // candidate if it is at least as good (ties are settled on the full key)
    const bool dot = metric == BOLT_DOT;
    float thr[kF32QT];
#pragma unroll
    for (int q = 0; q < kF32QT; ++q) thr[q] = dot ? -INFINITY : INFINITY;
    for (int64_t base = r0; base < r1; base += 32) {
        const int64_t row = base + lane;
        const bool valid = row < r1;
        float acc[kF32QT];
        row_sums(codes, valid ? row : r0, m, f32_tab, acc);
        uint32_t mask = 0;
#pragma unroll
        for (int q = 0; q < kF32QT; ++q) {
            const bool c = q < nv && valid && (dot ? acc[q] >= thr[q] : acc[q] <= thr[q]);
            mask |= (uint32_t)c << q;
        }
        uint32_t any = __reduce_or_sync(0xffffffffu, mask);
        while (any) {
            const int q = __ffs(any) - 1;
            any &= any - 1;
            uint64_t* list = lists + q * k;
            // this query's value of the lane (dynamic q: select from registers)
            float v = 0.f;
#pragma unroll
            for (int t = 0; t < kF32QT; ++t) v = t == q ? acc[t] : v;
            const uint64_t key = (mask >> q) & 1u ? key_f32(v, (uint64_t)(index_base + row), metric) : ~0ull;
            uint32_t cand = __ballot_sync(0xffffffffu, key < list[k - 1]);
            uint64_t kth = ~0ull;
            while (cand) {
                const int src = __ffs(cand) - 1;
                cand &= cand - 1;
                const uint64_t c = __shfl_sync(0xffffffffu, key, src);
                const uint64_t cur = lane < k ? list[lane] : ~0ull;
                if (c >= __shfl_sync(0xffffffffu, cur, k - 1)) continue;  // list tightened meanwhile
                const uint64_t prev = __shfl_up_sync(0xffffffffu, cur, 1);
                const uint32_t below = __ballot_sync(0xffffffffu, lane < k && cur < c);
                const int pos = __popc(below);  // entries ahead of c
                uint64_t nw = cur;
                if (lane == pos) nw = c;
                else if (lane > pos) nw = prev;
                __syncwarp();
                if (lane < k) list[lane] = nw;
                __syncwarp();
            }
            kth = list[k - 1];
            if (kth != ~0ull) {  // full: the k-th value bounds the list
                uint32_t ord = (uint32_t)(kth >> 32);
                if (dot) ord = ~ord;
                const float kv = __uint_as_float((ord & 0x80000000u) ? (ord & 0x7FFFFFFFu) : ~ord);
#pragma unroll
                for (int t = 0; t < kF32QT; ++t)
                    if (t == q) thr[t] = kv;
            }
        }
    }
    __syncwarp();
    for (int q = 0; q < nv; ++q)
        for (int e = lane; e < k; e += 32) part_keys[(part * nq + q0 + q) * k + e] = lists[q * k + e];
}

__global__ void keys_split_f32_kernel(const uint64_t* __restrict__ keys, int64_t count, int metric,
                                      float* __restrict__ vals, int64_t* __restrict__ idx) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const uint64_t key = keys[e];
    if (key == ~0ull) {
        if (vals) vals[e] = 0.f;
        if (idx) idx[e] = -1;
        return;
    }
    uint32_t ord = (uint32_t)(key >> 32);
    if (metric == BOLT_DOT) ord = ~ord;
    const uint32_t u = (ord & 0x80000000u) ? (ord & 0x7FFFFFFFu) : ~ord;
    if (vals) vals[e] = __uint_as_float(u);
    if (idx) idx[e] = (int64_t)(key & 0xFFFFFFFFull);
}

size_t tab_bytes(int m) { return (size_t)kF32QT * m * kK * sizeof(float); }

}  // namespace

int topk_f32_parts(int64_t n, int64_t nq, int num_sms) {
    // enough blocks for ~2 waves of 2 blocks per SM, at least 1024 rows per warp
    const int64_t qtiles = ceil_div(nq, kF32QT);
    const int64_t want = max64(1, ceil_div((int64_t)num_sms * 4, qtiles));
    const int64_t by_rows = max64(1, ceil_div(n, (int64_t)kF32Warps * 1024));
    return (int)(min64(want, by_rows) * kF32Warps);
}

cudaError_t launch_scan_f32(const uint32_t* codes, int64_t n, int m, const float* luts, int64_t nq, float* out,
                            int64_t ldo, cudaStream_t s) {
    if (n == 0 || nq == 0) return cudaSuccess;
    const int qtiles = (int)ceil_div(nq, kF32QT);
    const size_t smem = tab_bytes(m);
    cudaFuncSetAttribute(scan_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t blocks = ceil_div(n, kF32Threads) * qtiles;
    scan_f32_kernel<<<(unsigned)blocks, kF32Threads, smem, s>>>(codes, n, m, luts, nq, out, ldo, qtiles);
    return cudaGetLastError();
}

// part_keys [parts][nq][k] (parts = topk_f32_parts(...))
cudaError_t launch_topk_f32(const uint32_t* codes, int64_t n, int m, const float* luts, int64_t nq, int k,
                            int metric, int64_t index_base, int parts, uint64_t* part_keys, cudaStream_t s) {
    if (n == 0 || nq == 0) return cudaSuccess;
    const int qtiles = (int)ceil_div(nq, kF32QT);
    const int64_t rpw = ceil_div(ceil_div(n, (int64_t)parts), 32) * 32;
    const size_t smem = tab_bytes(m) + (size_t)kF32Warps * kF32QT * k * sizeof(uint64_t);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    cudaFuncSetAttribute(topk_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t blocks = (int64_t)(parts / kF32Warps) * qtiles;
    topk_f32_kernel<<<(unsigned)blocks, kF32Threads, smem, s>>>(codes, n, m, luts, nq, k, metric, index_base,
                                                                qtiles, rpw, part_keys);
    return cudaGetLastError();
}

cudaError_t launch_keys_split_f32(const uint64_t* keys, int64_t count, int metric, float* vals, int64_t* idx,
                                  cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    keys_split_f32_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, s>>>(keys, count, metric, vals, idx);
    return cudaGetLastError();
}

}  // namespace bolt
