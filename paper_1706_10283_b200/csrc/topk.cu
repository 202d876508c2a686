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

// Merge of many partial lists ([w][nq][lk] sorted keys -> k per query), for
// the small-batch scan (one list per block) and the large-k tcgen05 lists.
// With r = ceil(k / w) leading keys of every list as candidates, the
// candidate of rank k-1 is the largest of k distinct keys, so it bounds the
// k-th key of the union (H); only keys <= H can be in the result.  If w > k
// (r = 1) they lie in the k lists whose heads are <= H, else w <= k lists
// hold them all: at most min(w, k) * lk survivors.
//   1. candidates -> shared memory; H = the candidate of rank k-1 (rank by
//      counting smaller candidates, all threads, no serial rounds)
//   2. one coalesced pass over all keys keeps those <= H
//   3. each survivor's rank among the survivors is its output slot
// Keys are distinct except the UINT64_MAX padding, which never survives.
constexpr int kMergeManySmem = 200 * 1024;

__global__ void __launch_bounds__(kMergeThreads)
merge_many_kernel(const uint64_t* __restrict__ keys, int w, int64_t nq, int lk, int k, int r,
                  uint64_t* __restrict__ out) {
    extern __shared__ uint64_t cand[];  // [w * r] candidates, then the survivors
    const int nc = w * r;
    uint64_t* surv = cand + nc;
    __shared__ uint64_t sbound;
    __shared__ int count;
    const int64_t q = blockIdx.x;
    for (int e = threadIdx.x; e < nc; e += blockDim.x) {
        const int p = e / r, t = e - p * r;
        cand[e] = t < lk ? keys[((int64_t)p * nq + q) * lk + t] : ~0ull;
    }
    if (threadIdx.x == 0) { count = 0; sbound = ~0ull; }
    __syncthreads();
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
        const uint64_t c = cand[i];
        if (c == ~0ull) continue;
        int below = 0;
        for (int j = 0; j < nc && below < k; ++j) below += cand[j] < c;
        if (below == k - 1) sbound = c;  // unique: candidates are distinct
    }
    __syncthreads();
    const uint64_t bound = sbound;  // UINT64_MAX if fewer than k keys: all keys survive
    const int64_t total = (int64_t)w * lk;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
        const int p = (int)(e / lk), t = (int)(e - (int64_t)p * lk);
        const uint64_t key = keys[((int64_t)p * nq + q) * lk + t];
        if (key <= bound && key != ~0ull) surv[atomicAdd(&count, 1)] = key;
    }
    __syncthreads();
    const int n = count;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t key = surv[i];
        int below = 0;
        for (int j = 0; j < n && below < k; ++j) below += surv[j] < key;
        if (below < k) out[q * k + below] = key;
    }
    for (int i = n + threadIdx.x; i < k; i += blockDim.x) out[q * k + i] = ~0ull;
}

size_t merge_many_smem(int w, int lk, int k) {
    const int r = (k + w - 1) / w;
    return ((size_t)w * r + (size_t)(w < k ? w : k) * lk) * sizeof(uint64_t);
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


}  // namespace


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
    cudaError_t e = launch_merge_many(keys, w, nq, lk, k, out, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(count, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    verify_lists_kernel<<<(unsigned)ceil_div(nq, 128), 128, 0, s>>>(keys, w, nq, lk, out, k, flags, count);
    return cudaGetLastError();
}

cudaError_t launch_merge_many(const uint64_t* keys, int w, int64_t nq, int lk, int k, uint64_t* out,
                              cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    const size_t smem = merge_many_smem(w, lk, k);
    if (smem > kMergeManySmem) {
        const size_t tsmem = (size_t)w * (sizeof(uint64_t) + sizeof(int));
        const int threads = w >= kMergeThreads ? kMergeThreads : (int)(((w + 31) / 32) * 32);
        cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
        merge_kernel<<<(unsigned)nq, threads, tsmem, s>>>(keys, w, nq, lk, k, out);
        return cudaGetLastError();
    }
    cudaFuncSetAttribute(merge_many_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    merge_many_kernel<<<(unsigned)nq, kMergeThreads, smem, s>>>(keys, w, nq, lk, k, (k + w - 1) / w, out);
    return cudaGetLastError();
}

cudaError_t launch_keys_split(const uint64_t* keys, int64_t count, int metric, uint16_t* vals,
                              int64_t* idx, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    keys_split_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, s>>>(keys, count, metric, vals, idx);
    return cudaGetLastError();
}

}  // namespace bolt
