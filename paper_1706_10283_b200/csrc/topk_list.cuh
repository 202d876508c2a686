// topk_list.cuh -- a warp-private sorted list of the k best keys in shared
// memory, used by the fused top-k epilogues of both scan variants.
//
// Keys are (kv << 48) | global index with kv = acc (squared L2) or
// 0xFFFF - acc (dot) (R13), so ascending keys = best first with ties to the
// lower index.  The scan filters candidates with the value part of the k-th
// key ("threshold"); a warp walks its rows in increasing index order, so a
// row whose kv equals the threshold can never displace the k-th key and the
// filter kv < threshold is exact.  Insertions are rare after the first rows
// (about k ln(rows/k) per list), so they run out of line.
#pragma once
#include "common.cuh"

namespace bolt {

constexpr uint32_t kNotFull = 0x10000u;  // threshold while fewer than k keys are held

__device__ __forceinline__ void wl_init(uint64_t* list, int k, int lane) {
    for (int p = lane; p < k; p += 32) list[p] = ~0ull;
}

__device__ __forceinline__ uint32_t wl_threshold(const uint64_t* list, int k) {
    const uint64_t kth = list[k - 1];
    return kth == ~0ull ? kNotFull : (uint32_t)(kth >> 48);
}

// Insert the warp-uniform key c into the sorted list [0, k) (k <= 128).
__device__ __forceinline__ void wl_insert(uint64_t* list, int k, uint64_t c, int lane) {
    uint64_t v[4];
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int p = j * 32 + lane;
        v[j] = p < k ? list[p] : ~0ull;
        cnt += __popc(__ballot_sync(0xffffffffu, v[j] < c));
    }
    if (cnt >= k) return;
    uint64_t prev[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int p = j * 32 + lane;
        prev[j] = (p >= 1 && p < k) ? list[p - 1] : 0ull;
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int p = j * 32 + lane;
        if (p == cnt) list[p] = c;
        else if (p > cnt && p < k) list[p] = prev[j];
    }
    __syncwarp();
}

// Candidate rows of one lane from packed u16 totals t0..t3 = rows (0,2),
// (1,3), (4,6), (5,7) of its 8-row group: kv = (acc ^ flip) & 0xFFFF, a
// candidate if r < nrows and kv < thr.  Inserts every candidate of the warp
// and returns the new threshold.  Arguments by value keep the caller's
// totals in registers.
static __device__ __noinline__ uint32_t wl_insert_group(uint64_t* list, int k, uint32_t t0, uint32_t t1,
                                                 uint32_t t2, uint32_t t3, uint32_t flip, int nrows,
                                                 uint32_t thr, uint64_t gbase, int lane) {
    const uint32_t tt[4] = {t0 ^ flip, t1 ^ flip, t2 ^ flip, t3 ^ flip};
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const uint32_t pair = tt[(r >> 2) * 2 + (r & 1)];
        const uint32_t kv = (r & 2) ? (pair >> 16) : (pair & 0xFFFFu);
        const bool ok = r < nrows;
        const uint64_t mine = make_key(kv, gbase + r);
        unsigned b = __ballot_sync(0xffffffffu, ok && kv <= thr);  // equal kv may still win on index
        while (b) {
            const int src = __ffs(b) - 1;
            wl_insert(list, k, __shfl_sync(0xffffffffu, mine, src), lane);
            thr = wl_threshold(list, k);  // re-filter the remaining lanes
            b &= __ballot_sync(0xffffffffu, ok && kv <= thr) & ~(1u << src) & ~((1u << src) - 1u);
        }
    }
    __syncwarp();
    return wl_threshold(list, k);
}

}  // namespace bolt
