// common.cuh -- shared device helpers of the sm_100a Bolt library.
// (No code here is shared with oracle/; the oracle has its own C file.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bolt.h"

namespace bolt {

constexpr int kK = 16;           // centroids per codebook
constexpr int kMaxM = 64;        // codebooks
constexpr int kRowsPerWord = 8;  // layout v1: 8 rows x 4 bits per u32 word
constexpr int kMaxK = 128;       // top-k

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

// PRMT (byte permute, default mode): result byte i = byte sel[4i+2:4i] of
// {hi, lo}; if sel bit 4i+3 is set the sign bit of that byte is replicated
// instead.  Only the low 16 bits of sel are used.
__device__ __forceinline__ uint32_t prmt(uint32_t lo, uint32_t hi, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(lo), "r"(hi), "r"(sel));
    return d;
}

__device__ __forceinline__ uint32_t vminu2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// 64-bit ranking key (R13): smaller is better; ties -> lower global index.
__device__ __forceinline__ uint64_t make_key(uint32_t kv, uint64_t gidx) {
    return (static_cast<uint64_t>(kv) << 48) | gidx;
}

// Number of row partitions for `tiles` query tiles over `groups` 8-row
// groups and W resident warps (one warp task = one tile x one partition,
// dealt round robin): at least 4 tasks per warp, at least
// `min_groups_per_task` groups per task, and the partition count in a small
// window that best fills the last round.
inline int choose_parts(int64_t tiles, int64_t groups, int64_t W, int64_t min_groups_per_task) {
    tiles = max64(tiles, 1);  // nq = 0: no work, one partition
    const int64_t max_parts = max64(1, min64(16384, groups / min_groups_per_task));
    int64_t lo = max64(1, ceil_div(4 * W, tiles));
    if (lo >= max_parts) return (int)max_parts;
    const int64_t hi = min64(max_parts, 2 * lo + 8);
    int64_t best = lo;
    double best_eff = 0.0;
    for (int64_t p = lo; p <= hi; ++p) {
        const int64_t tasks = tiles * p;
        const double eff = (double)tasks / (double)(ceil_div(tasks, W) * W);
        if (eff > best_eff + 1e-9) { best_eff = eff; best = p; }
        if (eff >= 0.97) break;
    }
    return (int)best;
}

// Diagnostic cycle counters (BOLT_PROFILE builds only).
constexpr int kNumCounters = 24;
#ifdef BOLT_PROFILE
// defined (per translation unit that uses it) by BOLT_DEFINE_COUNTERS
#define BOLT_PROF_ADD(i, v) atomicAdd(&g_counters[(i)], (unsigned long long)(v))
// warp-aggregated: one atomic per group of converged lanes; `lanes` != 0 adds
// the number of active lanes, else 1 per warp group
#define BOLT_PROF_WARP(i, lanes)                                                               \
    do {                                                                                       \
        const unsigned _am = __activemask();                                                   \
        if ((threadIdx.x & 31) == (unsigned)(__ffs(_am) - 1))                                  \
            atomicAdd(&g_counters[(i)], (unsigned long long)((lanes) ? __popc(_am) : 1));      \
    } while (0)
#define BOLT_CLOCK() clock64()
#else
#define BOLT_PROF_ADD(i, v) ((void)0)
#define BOLT_PROF_WARP(i, lanes) ((void)0)
#define BOLT_CLOCK() 0ll
#endif

// Per-launch argument block for the scan kernels.
struct ScanArgs {
    const uint32_t* codes;
    int64_t n;            // rows
    int64_t groups;       // ceil(n / 8)
    int m;
    const uint8_t* qluts;
    int64_t nq;
    int noshare = 0;      // tcgen05 top-k with lists of 32 for k > 32: G = ceil(k/32) threshold groups
};

}  // namespace bolt

// ---------------------------------------------------------------- launchers
// Implemented in the .cu files, called by api.cu after validation.  They
// return cudaGetLastError() of their launch.
namespace bolt {
// sms: the device's SM count (block-size heuristic), passed down from the ABI's device cache
// mode: 0 auto / 1 direct: the direct-difference kernels; 2 (J/M = 8): the
// TMA-staged expanded-distance kernel, the same codes by its bound + direct
// fallback (measured no faster: DESIGN.md 6.3)
cudaError_t launch_encode(const float* X, int64_t n, int j, int64_t ldx, const float* C, int m,
                          uint32_t* codes, int sms, cudaStream_t s, int mode = 0);
// Bolt No Quantize (scan_f32.cu): fp32 tables, fp32 sums, R18 keys
int topk_f32_parts(int64_t n, int64_t nq, int num_sms);
cudaError_t launch_scan_f32(const uint32_t* codes, int64_t n, int m, const float* luts, int64_t nq, float* out,
                            int64_t ldo, cudaStream_t s);
cudaError_t launch_topk_f32(const uint32_t* codes, int64_t n, int m, const float* luts, int64_t nq, int k,
                            int metric, int64_t index_base, int parts, uint64_t* part_keys, cudaStream_t s);
cudaError_t launch_keys_split_f32(const uint64_t* keys, int64_t count, int metric, float* vals, int64_t* idx,
                                  cudaStream_t s);
cudaError_t launch_encode_append(const float* X, int64_t n_new, int j, int64_t ldx, const float* C, int m,
                                 uint32_t* codes, int64_t n_old, int sms, cudaStream_t s);
cudaError_t launch_pack(const uint8_t* flat, int64_t n, int m, uint32_t* codes, cudaStream_t s);
cudaError_t launch_unpack(const uint32_t* codes, int64_t n, int m, uint8_t* flat, cudaStream_t s);

cudaError_t launch_build_luts(const float* Q, int64_t nq, int j, int64_t ldq, const float* C, int m,
                              int metric, float a, const float* b, uint8_t* qluts, float* luts32,
                              double* luts64, cudaStream_t s);
cudaError_t launch_quantize(const float* luts, int64_t nq, int m, float a, const float* b,
                            uint8_t* qluts, cudaStream_t s);

cudaError_t launch_scan_full(const ScanArgs& a, uint16_t* out16, float* out32, int64_t ldo,
                             float inv_a, float b_sum, cudaStream_t s);

// top-k (PRMT variant): partial lists [parts][nq][k] in ws, then merge
int topk_prmt_parts(int64_t n, int m, int64_t nq, int k, int num_sms);
cudaError_t launch_topk_prmt(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                             uint64_t* part_keys, int sms, cudaStream_t s);
// top-k (tcgen05 variant)
int topk_tc_supported(int64_t n, int m, int64_t nq, int k);
int scan_tc_supported(int64_t n, int m, int64_t nq);
cudaError_t launch_scan_tc(const ScanArgs& a, uint16_t* out16, float* out32, int64_t ldo, float inv_a, float b_sum,
                           int sms, cudaStream_t s);
int topk_tc_parts(int64_t n, int m, int64_t nq, int k, int num_sms);
// swapped tcgen05 top-k for small query batches (vectors on the MMA M side)
int topk_tcs_supported(int64_t n, int m, int64_t nq, int k);
int topk_tcs_parts(int64_t n, int m, int64_t nq, int k, int num_sms);
cudaError_t launch_topk_tcs(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                            uint64_t* part_keys, cudaStream_t s);
// 2:4-sparse tcgen05 top-k (scan_sp.cu): vectors on M, 224 queries per tile
int topk_sp_supported(int64_t n, int m, int64_t nq, int k);
int topk_sp_parts(int64_t n, int m, int64_t nq, int k, int num_sms);
cudaError_t launch_topk_sp(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                           uint64_t* part_keys, cudaStream_t s);
// part_keys: parts*nq*k keys followed by the shared threshold words (zeroed by the launch)
cudaError_t launch_topk_tc(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                           uint64_t* part_keys, int sms, cudaStream_t s);
// small query batches (scan_small.cu): one partial list per warp + shared thresholds
int topk_small_supported(int64_t n, int m, int64_t nq, int k);
int topk_small_parts(int64_t n, int m, int64_t nq, int k, int num_sms);
cudaError_t launch_topk_small(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                              uint64_t* part_keys, cudaStream_t s);
// merge of lk-key lists into k keys + exactness flags (large-k tcgen05 top-k)
cudaError_t launch_merge_lists(const uint64_t* keys, int w, int64_t nq, int lk, int k, uint64_t* out,
                               uint32_t* flags, uint32_t* count, cudaStream_t s);
// merge of many lists (k <= 32): bound by the k-th smallest head, then select
cudaError_t launch_merge_many(const uint64_t* keys, int w, int64_t nq, int lk, int k, uint64_t* out,
                              cudaStream_t s);
constexpr int kMaxParts = 16384;  // merge limit (shared memory of the tournament merge)

int tc_debug_counters(uint64_t* out, int n);  // scan_tc.cu (BOLT_PROFILE builds)
cudaError_t launch_merge(const uint64_t* keys, int w, int64_t nq, int k, uint64_t* out,
                         cudaStream_t s);
cudaError_t launch_keys_split(const uint64_t* keys, int64_t count, int metric, uint16_t* vals,
                              int64_t* idx, cudaStream_t s);

size_t kmeans_ws_bytes(int64_t n, int j, int m);
cudaError_t launch_kmeans(const float* train, int64_t n, int j, int64_t ldx, int m,
                          const int64_t* init, int iters, float* C_out, void* ws, cudaStream_t s);
size_t calibrate_ws_bytes(int64_t nq, int m);
cudaError_t launch_calibrate(const double* luts, int64_t nq, int m, float* a_out, float* b_out,
                             double* alpha_mse, void* ws, cudaStream_t s);
}  // namespace bolt
