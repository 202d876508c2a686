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

// One block per query: bitonic sort of the w*k candidates in shared memory.
__global__ void __launch_bounds__(kMergeThreads)
merge_kernel(const uint64_t* __restrict__ keys, int w, int64_t nq, int k, int pow2,
             uint64_t* __restrict__ out) {
    extern __shared__ uint64_t mbuf[];
    const int64_t q = blockIdx.x;
    const int total = w * k;
    for (int e = threadIdx.x; e < pow2; e += blockDim.x) {
        uint64_t v = ~0ull;
        if (e < total) {
            const int s = e / k, p = e - s * k;
            v = keys[((int64_t)s * nq + q) * k + p];
        }
        mbuf[e] = v;
    }
    __syncthreads();
    for (int size = 2; size <= pow2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int e = threadIdx.x; e < pow2 / 2; e += blockDim.x) {
                const int lo = 2 * e - (e & (stride - 1));
                const int hi = lo + stride;
                const bool asc = (lo & size) == 0;
                const uint64_t a = mbuf[lo], b = mbuf[hi];
                if ((a > b) == asc) {
                    mbuf[lo] = b;
                    mbuf[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    for (int p = threadIdx.x; p < k; p += blockDim.x) out[q * k + p] = mbuf[p];
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
    int pow2 = 1;
    while (pow2 < w * k) pow2 <<= 1;
    if (pow2 < 2) pow2 = 2;
    size_t smem = (size_t)pow2 * sizeof(uint64_t);
    cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    merge_kernel<<<(unsigned)nq, kMergeThreads, smem, s>>>(keys, w, nq, k, pow2, out);
    return cudaGetLastError();
}

cudaError_t launch_keys_split(const uint64_t* keys, int64_t count, int metric, uint16_t* vals,
                              int64_t* idx, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    keys_split_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, s>>>(keys, count, metric, vals, idx);
    return cudaGetLastError();
}

}  // namespace bolt
