// topk.cu -- merge of sorted per-partition / per-shard key lists and key split.
//
// Keys are (value << 48 | global index) (R13), a total order, so the k best
// of a union of lists are exactly the k smallest keys of the concatenation:
// the merge is exact however the rows were partitioned (split-N partials of
// one GPU or the row shards of several GPUs).
#include "common.cuh"

namespace bolt {
namespace {

constexpr int kMergeThreads = 256;

// One block per query: a k-round tournament over the heads of the w sorted
// lists (head keys and read positions in shared memory).  Each round the
// block finds the smallest head (ties impossible: keys are unique except
// the UINT64_MAX padding), emits it and advances that list.
// lists of lk keys ([w][nq][lk]) -> k outputs per query
__global__ void __launch_bounds__(kMergeThreads)
merge_kernel(const uint64_t* __restrict__ keys, int w, int64_t nq, int lk, int k, uint64_t* __restrict__ out) {
    extern __shared__ uint64_t mhead[];
    int* mpos = reinterpret_cast<int*>(mhead + w);
    __shared__ uint64_t wkey[kMergeThreads / 32];
    __shared__ int wlist[kMergeThreads / 32];
    const int64_t q = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    for (int p = threadIdx.x; p < w; p += blockDim.x) {
        mhead[p] = keys[((int64_t)p * nq + q) * lk];
        mpos[p] = 0;
    }
    __syncthreads();
    for (int r = 0; r < k; ++r) {
        uint64_t best = ~0ull;
        int bi = -1;
        for (int p = threadIdx.x; p < w; p += blockDim.x) {
            const uint64_t h = mhead[p];
            if (h < best) { best = h; bi = p; }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const uint64_t ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ob < best || (ob == best && (unsigned)oi < (unsigned)bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) { wkey[warp] = best; wlist[warp] = bi; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int t = 1; t < nwarps; ++t)
                if (wkey[t] < best || (wkey[t] == best && (unsigned)wlist[t] < (unsigned)bi)) {
                    best = wkey[t];
                    bi = wlist[t];
                }
            out[q * k + r] = best;
            if (bi >= 0 && best != ~0ull) {
                const int np = ++mpos[bi];
                mhead[bi] = np < lk ? keys[((int64_t)bi * nq + q) * lk + np] : ~0ull;
            }
        }
        __syncthreads();
    }
}

// Merge of many partial lists (the small-batch scan: one list per block).
// The k smallest list heads are k distinct keys, so the k-th smallest head H
// bounds the k-th key of the union; only keys <= H can be in the result, and
// they lie in the k lists whose heads are <= H: at most k*k survivors.
//   1. heads -> shared memory; k rounds of argmin give H (no global loads
//      inside the rounds)
//   2. one coalesced pass over all keys keeps those <= H
//   3. k rounds of argmin over the survivors
// Used for k <= kFilteredMaxK (k*k survivors fit in shared memory).
constexpr int kFilteredMaxK = 32;

// One block per query: all threads load the heads and scan the keys (many
// independent loads in flight), warp 0 alone runs the k-round selections
// (no block barrier inside a round).
__device__ __forceinline__ void warp_argmin(uint64_t& best, int& bi) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (o < best || (o == best && (unsigned)oi < (unsigned)bi)) { best = o; bi = oi; }
    }
}

__global__ void __launch_bounds__(kMergeThreads)
merge_many_kernel(const uint64_t* __restrict__ keys, int w, int64_t nq, int k, uint64_t* __restrict__ out) {
    extern __shared__ uint64_t heads[];  // [w] heads, then [k*k] survivors
    uint64_t* surv = heads + w;
    __shared__ uint64_t sbound;
    __shared__ int count;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t q = blockIdx.x;
    for (int p = threadIdx.x; p < w; p += blockDim.x) heads[p] = keys[((int64_t)p * nq + q) * k];
    if (threadIdx.x == 0) count = 0;
    __syncthreads();
    if (warp == 0) {
        uint64_t bound = ~0ull;
        for (int r = 0; r < k; ++r) {
            uint64_t best = ~0ull;
            int bi = -1;
            for (int p = lane; p < w; p += 32)
                if (heads[p] < best) { best = heads[p]; bi = p; }
            warp_argmin(best, bi);
            if (bi < 0 || best == ~0ull) break;  // fewer than k keys in all lists
            bound = best;
            if (lane == 0) heads[bi] = ~0ull;
            __syncwarp();
        }
        if (lane == 0) sbound = bound;
    }
    __syncthreads();
    const uint64_t bound = sbound;
    const int64_t total = (int64_t)w * k;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
        const int p = (int)(e / k), rr = (int)(e - (int64_t)p * k);
        const uint64_t key = keys[((int64_t)p * nq + q) * k + rr];
        if (key <= bound && key != ~0ull) {
            const int slot = atomicAdd(&count, 1);
            if (slot < k * k) surv[slot] = key;
        }
    }
    __syncthreads();
    if (warp != 0) return;
    const int n = min(count, k * k);
    for (int r = 0; r < k; ++r) {
        uint64_t best = ~0ull;
        int bi = -1;
        for (int i = lane; i < n; i += 32)
            if (surv[i] < best) { best = surv[i]; bi = i; }
        warp_argmin(best, bi);
        if (lane == 0) {
            out[q * k + r] = best;
            if (bi >= 0) surv[bi] = ~0ull;
        }
        __syncwarp();
    }
}

__global__ void keys_split_kernel(const uint64_t* __restrict__ keys, int64_t count, int metric,
                                  uint16_t* __restrict__ vals, int64_t* __restrict__ idx) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const uint64_t key = keys[e];
    if (key == ~0ull) {
        if (vals) vals[e] = 0;
        if (idx) idx[e] = -1;
        return;
    }
    uint32_t v = (uint32_t)(key >> 48);
    if (metric == BOLT_DOT) v = 0xFFFFu - v;
    if (vals) vals[e] = (uint16_t)v;
    if (idx) idx[e] = (int64_t)(key & ((1ull << 48) - 1));
}

// Shared-threshold seed from a prefix sample (scan_tc.cu): per query the k-th
// smallest key of the union of w sorted partial lists over the sample rows,
// converted to the tcgen05 epilogue's inverted threshold 0xFFFF - kv'
// (kv' = acc for L2, 255 M - acc for dot).  Every row of the sample is a row
// of the database, so at least k keys of the full top-k search have a value
// <= that one: a valid bound for the full scan (0 = no bound if the sample
// holds fewer than k keys).
__global__ void prefix_threshold_kernel(const uint64_t* __restrict__ keys, int w, int64_t nq, int k, int metric,
                                        uint32_t kvmax, uint32_t* __restrict__ gthr) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    int pos[32];
    for (int p = 0; p < w; ++p) pos[p] = 0;
    uint64_t kth = ~0ull;
    for (int r = 0; r < k; ++r) {
        uint64_t best = ~0ull;
        int bi = -1;
        for (int p = 0; p < w; ++p) {
            const uint64_t h = pos[p] < k ? keys[((int64_t)p * nq + q) * k + pos[p]] : ~0ull;
            if (h < best) { best = h; bi = p; }
        }
        if (bi < 0) break;
        ++pos[bi];
        kth = best;
    }
    uint32_t g = 0;
    if (kth != ~0ull) {
        const uint32_t v = (uint32_t)(kth >> 48);
        const uint32_t kvp = metric == BOLT_DOT ? kvmax - (0xFFFFu - v) : v;
        g = 0xFFFFu - kvp;
    }
    gthr[q] = g;
}

}  // namespace

cudaError_t launch_prefix_threshold(const uint64_t* keys, int w, int64_t nq, int k, int metric, uint32_t kvmax,
                                    uint32_t* gthr, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    if (w > 32) return cudaErrorInvalidValue;
    prefix_threshold_kernel<<<(unsigned)ceil_div(nq, 128), 128, 0, s>>>(keys, w, nq, k, metric, kvmax, gthr);
    return cudaGetLastError();
}

cudaError_t launch_merge(const uint64_t* keys, int w, int64_t nq, int k, uint64_t* out,
                         cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    const size_t smem = (size_t)w * (sizeof(uint64_t) + sizeof(int));
    const int threads = w >= kMergeThreads ? kMergeThreads : (int)(((w + 31) / 32) * 32);
    cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    merge_kernel<<<(unsigned)nq, threads, smem, s>>>(keys, w, nq, k, k, out);
    return cudaGetLastError();
}

// Large-k tcgen05 top-k (32 < k <= 128): the lists hold 32 keys; merge them
// into k and flag the queries where a list's 32nd key is below the merged k-th
// key (that list may have dropped keys of the top-k): flags[q] = 1, count++.
__global__ void verify_lists_kernel(const uint64_t* __restrict__ keys, int w, int64_t nq, int lk,
                                    const uint64_t* __restrict__ out, int k, uint32_t* __restrict__ flags,
                                    uint32_t* __restrict__ count) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint64_t kth = out[q * k + k - 1];
    uint32_t f = 0;
    for (int p = 0; p < w && !f; ++p) f = keys[((int64_t)p * nq + q) * lk + lk - 1] < kth;
    flags[q] = f;
    if (f) atomicAdd(count, 1u);
}

cudaError_t launch_merge_lists(const uint64_t* keys, int w, int64_t nq, int lk, int k, uint64_t* out,
                               uint32_t* flags, uint32_t* count, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    const size_t smem = (size_t)w * (sizeof(uint64_t) + sizeof(int));
    const int threads = w >= kMergeThreads ? kMergeThreads : (int)(((w + 31) / 32) * 32);
    cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    merge_kernel<<<(unsigned)nq, threads, smem, s>>>(keys, w, nq, lk, k, out);
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    verify_lists_kernel<<<(unsigned)ceil_div(nq, 128), 128, 0, s>>>(keys, w, nq, lk, out, k, flags, count);
    return cudaGetLastError();
}

cudaError_t launch_merge_many(const uint64_t* keys, int w, int64_t nq, int k, uint64_t* out, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    const size_t smem = (size_t)(w + k * k) * sizeof(uint64_t);
    if (k > kFilteredMaxK || smem > 200 * 1024) return launch_merge(keys, w, nq, k, out, s);
    cudaFuncSetAttribute(merge_many_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    merge_many_kernel<<<(unsigned)nq, kMergeThreads, smem, s>>>(keys, w, nq, k, out);
    return cudaGetLastError();
}

cudaError_t launch_keys_split(const uint64_t* keys, int64_t count, int metric, uint16_t* vals,
                              int64_t* idx, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    keys_split_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, s>>>(keys, count, metric, vals, idx);
    return cudaGetLastError();
}

}  // namespace bolt
