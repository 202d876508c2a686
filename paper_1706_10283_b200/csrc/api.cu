// api.cu -- the extern "C" boundary (include/bolt.h): argument validation,
// status codes, thread-local error text, workspace sizing and dispatch to the
// sm_100a kernels.  No allocation, no synchronization, no torch types.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>

#include <cstdlib>

#include "common.cuh"

using namespace bolt;

namespace {

thread_local char g_err[512] = "";

bolt_status fail(bolt_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

bolt_status cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return BOLT_OK;
    return fail(BOLT_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

struct DevInfo {
    int ok;   // 1 = sm_100, 0 = unsupported
    int sms;
};
std::atomic<int> g_dev_cache[64];  // 0 unknown, else (sms << 2) | (ok << 1) | 1

bolt_status device_info(DevInfo* info) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    int cached = (dev >= 0 && dev < 64) ? g_dev_cache[dev].load(std::memory_order_relaxed) : 0;
    if (!cached) {
        int major = 0, minor = 0, sms = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
        const int ok = (major == 10 && minor == 0) ? 1 : 0;
        cached = (sms << 2) | (ok << 1) | 1;
        if (dev >= 0 && dev < 64) g_dev_cache[dev].store(cached, std::memory_order_relaxed);
    }
    info->ok = (cached >> 1) & 1;
    info->sms = cached >> 2;
    if (!info->ok) return fail(BOLT_E_DEVICE, "device %d is not sm_100 (B200); this library is sm_100a only", dev);
    return BOLT_OK;
}

int sms_or_default() {
    DevInfo d{};
    if (device_info(&d) != BOLT_OK) return 148;
    return d.sms;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

bolt_status check_m(int m) {
    if (m < 1 || m > kMaxM) return fail(BOLT_E_SHAPE, "m = %d outside 1..64", m);
    return BOLT_OK;
}

bolt_status check_jm(int j, int m) {
    if (bolt_status st = check_m(m)) return st;
    if (j < 1) return fail(BOLT_E_SHAPE, "j = %d < 1", j);
    if (j % m) return fail(BOLT_E_SHAPE, "j = %d not divisible by m = %d (zero-pad to a multiple)", j, m);
    return BOLT_OK;
}

#define TRY(x)                                \
    do {                                      \
        bolt_status _st = (x);                \
        if (_st != BOLT_OK) return _st;       \
    } while (0)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// ---- top-k plan shared by workspace sizing and execution
struct TopkPlan {
    int variant;     // resolved PRMT / TC
    int klist;       // TC: keys per partial list (k, or 32 when k > 32)
    size_t large_off;  // TC, k > 32: byte offset of flags | count | fallback area in ws
    bool small;      // PRMT: the small-batch kernel (scan_small.cu, nq < 64)
    int parts;
    size_t ws;
};


constexpr int kTcListMax = 32;      // register list capacity of the tcgen05 epilogue
constexpr int kFallbackBatch = 48;  // flagged queries per exact fallback batch (small-batch kernel)

TopkPlan topk_plan(int64_t n, int m, int64_t nq, int k, int variant, int sms) {
    TopkPlan p{};
    int v = variant;
    // auto: tensor cores above a per-M query count, else PRMT.  Crossovers measured on 10^8
    // rows: M = 16 TC 3.0 ms flat for Q <= 128 vs PRMT 2.57 (Q = 12) / 3.24
    // (Q = 13); M = 8 even at Q = 20; M = 32 (pair tiles) even at Q = 16.
    const int64_t tc_above = m == 16 ? 12 : (m == 8 ? 20 : 16);
    if (v == BOLT_VARIANT_AUTO) v = topk_tc_supported(n, m, nq, k) && nq > tc_above ? BOLT_VARIANT_TC : BOLT_VARIANT_PRMT;
    p.variant = v;
    p.small = v == BOLT_VARIANT_PRMT && topk_small_supported(n, m, nq, k);
    p.parts = v == BOLT_VARIANT_TC    ? topk_tc_parts(n, m, nq, k, sms)
              : v == BOLT_VARIANT_TCS ? topk_tcs_parts(n, m, nq, k, sms)
              : v == BOLT_VARIANT_SP  ? topk_sp_parts(n, m, nq, k, sms)
              : p.small               ? topk_small_parts(n, m, nq, k, sms)
                                      : topk_prmt_parts(n, m, nq, k, sms);
    p.klist = v == BOLT_VARIANT_TC && k > kTcListMax ? kTcListMax : k;
    p.ws = p.parts > 1 || p.small || v == BOLT_VARIANT_TCS || v == BOLT_VARIANT_SP
               ? (size_t)p.parts * nq * p.klist * sizeof(uint64_t) : 0;
    // shared per-query thresholds (u32) after the partial lists: PRMT one word,
    // TC 9 nq + 4 (k-th value words + 16 B aligned rows of 8 union-group words, scan_tc.cu;
    // k > 32: 4 nq group words), then rparts ceil(nq / 128) finished-partition counters,
    // small-batch PRMT 33 nq (k-th value word + 32 minima slots, scan_small.cu)
    if (p.ws > 0)
        p.ws += (size_t)(v == BOLT_VARIANT_TC ? (k > kTcListMax ? 4 * nq : 9 * nq + 4) + (p.parts / 2) * ceil_div(nq, 128)
                                              : p.small ? 33 * nq : nq) *
                sizeof(uint32_t);  // TCS, SP: nq words; TC also the finished-partition counters [rparts][tiles_q]
    if (v == BOLT_VARIANT_TC && k > kTcListMax) {
        // flags [nq] u32, count, then the exact fallback for flagged queries in
        // batches of kFallbackBatch: gathered tables, keys, small-batch workspace
        // -- sized for every batch size 1..kFallbackBatch (the last batch is
        // smaller, and fewer queries may take more row partitions)
        size_t fb_ws = 0;
        for (int nb = 1; nb <= kFallbackBatch; ++nb) {
            const size_t w = topk_plan(n, m, nb, k, BOLT_VARIANT_PRMT, sms).ws;
            fb_ws = w > fb_ws ? w : fb_ws;
        }
        p.large_off = align256(p.ws);
        p.ws = p.large_off + align256((size_t)nq * sizeof(uint32_t) + 16) + align256((size_t)kFallbackBatch * m * kK) +
               align256((size_t)kFallbackBatch * k * sizeof(uint64_t)) + align256(fb_ws);
    }
    return p;
}

}  // namespace

extern "C" {

int bolt_debug_counters(uint64_t* out, int n) {
    if (!out || n <= 0) return 0;
    return tc_debug_counters(out, n);  // counters, then (libbolt_x.so) the scan trace
}

const char* bolt_version(void) { return "bolt-b200 1.0 (abi 1, sm_100a)"; }

const char* bolt_last_error(void) { return g_err; }

int64_t bolt_codes_words(int64_t n, int m) {
    if (n < 0 || m < 1 || m > kMaxM) return -1;
    return ceil_div(n, kRowsPerWord) * m;
}

bolt_status bolt_encode(const float* X, int64_t n, int j, int64_t ldx, const float* C, int m,
                        uint32_t* codes, bolt_stream_t stream) {
    return bolt_encode_ex(X, n, j, ldx, C, m, codes, BOLT_ENCODE_AUTO, stream);
}

bolt_status bolt_encode_ex(const float* X, int64_t n, int j, int64_t ldx, const float* C, int m,
                           uint32_t* codes, int variant, bolt_stream_t stream) {
    if (variant != BOLT_ENCODE_AUTO && variant != BOLT_ENCODE_DIRECT && variant != BOLT_ENCODE_EXPANDED)
        return fail(BOLT_E_RANGE, "encode variant %d", variant);
    TRY(check_jm(j, m));
    if (n < 0) return fail(BOLT_E_SHAPE, "n = %lld < 0", (long long)n);
    if (ldx < j) return fail(BOLT_E_SHAPE, "ldx = %lld < j = %d", (long long)ldx, j);
    if (j > 2048) return fail(BOLT_E_SHAPE, "j = %d > 2048 (centroids must fit in shared memory)", j);
    if (n == 0) return BOLT_OK;
    if (!X || !C || !codes) return fail(BOLT_E_NULL, "bolt_encode: NULL pointer");
    if (!aligned(C, 16)) return fail(BOLT_E_ALIGN, "bolt_encode: C must be 16-byte aligned");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_encode(X, n, j, ldx, C, m, codes, d.sms, (cudaStream_t)stream,
                                     variant == BOLT_ENCODE_DIRECT ? 1 : variant == BOLT_ENCODE_EXPANDED ? 2 : 0),
                       "bolt_encode");
}

// ---- Bolt No Quantize (scan_f32.cu)
static bolt_status f32_common(const uint32_t* codes, int64_t n, int m, const float* luts, int64_t nq) {
    TRY(check_m(m));
    if (n < 0 || nq < 0) return fail(BOLT_E_SHAPE, "n or nq < 0");
    if (n > 0 && nq > 0) {
        if (!codes || !luts) return fail(BOLT_E_NULL, "codes/luts NULL");
        if (!aligned(codes, 16)) return fail(BOLT_E_ALIGN, "codes must be 16-byte aligned");
        if (!aligned(luts, 4)) return fail(BOLT_E_ALIGN, "luts must be 4-byte aligned");
    }
    return BOLT_OK;
}

bolt_status bolt_scan_f32(const uint32_t* codes, int64_t n, int m, const float* luts, int64_t nq, float* out,
                          int64_t ldo, bolt_stream_t stream) {
    TRY(f32_common(codes, n, m, luts, nq));
    if (ldo < nq) return fail(BOLT_E_SHAPE, "ldo < nq");
    if (n == 0 || nq == 0) return BOLT_OK;
    if (!out) return fail(BOLT_E_NULL, "out NULL");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_scan_f32(codes, n, m, luts, nq, out, ldo, (cudaStream_t)stream), "bolt_scan_f32");
}

size_t bolt_topk_f32_workspace_bytes(int64_t n, int m, int64_t nq, int k) {
    if (n <= 0 || nq <= 0 || k < 1 || k > 32 || m < 1 || m > kMaxM) return 0;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    return (size_t)topk_f32_parts(n, nq, sms) * nq * k * sizeof(uint64_t);
}

bolt_status bolt_topk_f32(const uint32_t* codes, int64_t n, int m, const float* luts, int64_t nq, int k,
                          bolt_metric metric, int64_t index_base, uint64_t* out_keys, void* ws, size_t ws_bytes,
                          bolt_stream_t stream) {
    TRY(f32_common(codes, n, m, luts, nq));
    if (k < 1 || k > 32) return fail(BOLT_E_SHAPE, "k = %d outside 1..32", k);
    if (metric != BOLT_L2SQ && metric != BOLT_DOT) return fail(BOLT_E_RANGE, "metric %d", (int)metric);
    if (index_base < 0 || index_base + n > (int64_t(1) << 32)) return fail(BOLT_E_RANGE, "index_base + n > 2^32");
    if (nq == 0) return BOLT_OK;
    if (!out_keys) return fail(BOLT_E_NULL, "out_keys NULL");
    DevInfo d;
    TRY(device_info(&d));
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0)
        return cuda_status(cudaMemsetAsync(out_keys, 0xFF, (size_t)nq * k * sizeof(uint64_t), s), "bolt_topk_f32");
    const int parts = topk_f32_parts(n, nq, d.sms);
    const size_t need = (size_t)parts * nq * k * sizeof(uint64_t);
    if (!ws || ws_bytes < need) return fail(BOLT_E_WORKSPACE, "workspace of %zu bytes required, %zu given", need, ws_bytes);
    if (!aligned(ws, 8)) return fail(BOLT_E_ALIGN, "workspace must be 8-byte aligned");
    uint64_t* pk = static_cast<uint64_t*>(ws);
    TRY(cuda_status(launch_topk_f32(codes, n, m, luts, nq, k, (int)metric, index_base, parts, pk, s),
                    "bolt_topk_f32 scan"));
    return cuda_status(launch_merge_many(pk, parts, nq, k, k, out_keys, s), "bolt_topk_f32 merge");
}

bolt_status bolt_keys_split_f32(const uint64_t* keys, int64_t count, bolt_metric metric, float* vals, int64_t* idx,
                                bolt_stream_t stream) {
    if (count < 0) return fail(BOLT_E_SHAPE, "count < 0");
    if (count == 0) return BOLT_OK;
    if (!keys) return fail(BOLT_E_NULL, "keys NULL");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_keys_split_f32(keys, count, (int)metric, vals, idx, (cudaStream_t)stream),
                       "bolt_keys_split_f32");
}

bolt_status bolt_encode_append(const float* X, int64_t n_new, int j, int64_t ldx, const float* C, int m,
                               uint32_t* codes, int64_t n_old, bolt_stream_t stream) {
    TRY(check_jm(j, m));
    if (n_new < 0 || n_old < 0) return fail(BOLT_E_SHAPE, "n_new = %lld, n_old = %lld", (long long)n_new,
                                            (long long)n_old);
    if (ldx < j) return fail(BOLT_E_SHAPE, "ldx = %lld < j = %d", (long long)ldx, j);
    if (j > 2048) return fail(BOLT_E_SHAPE, "j = %d > 2048 (centroids must fit in shared memory)", j);
    if (n_new == 0) return BOLT_OK;
    if (!X || !C || !codes) return fail(BOLT_E_NULL, "bolt_encode_append: NULL pointer");
    if (!aligned(C, 16)) return fail(BOLT_E_ALIGN, "bolt_encode_append: C must be 16-byte aligned");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_encode_append(X, n_new, j, ldx, C, m, codes, n_old, d.sms, (cudaStream_t)stream),
                       "bolt_encode_append");
}

bolt_status bolt_pack_codes(const uint8_t* flat, int64_t n, int m, uint32_t* codes,
                            bolt_stream_t stream) {
    TRY(check_m(m));
    if (n < 0) return fail(BOLT_E_SHAPE, "n < 0");
    if (n == 0) return BOLT_OK;
    if (!flat || !codes) return fail(BOLT_E_NULL, "bolt_pack_codes: NULL pointer");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_pack(flat, n, m, codes, (cudaStream_t)stream), "bolt_pack_codes");
}

bolt_status bolt_unpack_codes(const uint32_t* codes, int64_t n, int m, uint8_t* flat,
                              bolt_stream_t stream) {
    TRY(check_m(m));
    if (n < 0) return fail(BOLT_E_SHAPE, "n < 0");
    if (n == 0) return BOLT_OK;
    if (!flat || !codes) return fail(BOLT_E_NULL, "bolt_unpack_codes: NULL pointer");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_unpack(codes, n, m, flat, (cudaStream_t)stream), "bolt_unpack_codes");
}

static bolt_status lut_common(const float* Q, int64_t nq, int j, int64_t ldq, const float* C, int m,
                              bolt_metric metric) {
    TRY(check_jm(j, m));
    if (nq < 0) return fail(BOLT_E_SHAPE, "nq < 0");
    if (ldq < j) return fail(BOLT_E_SHAPE, "ldq = %lld < j = %d", (long long)ldq, j);
    if (metric != BOLT_L2SQ && metric != BOLT_DOT) return fail(BOLT_E_RANGE, "metric %d", (int)metric);
    if (nq > 0 && (!Q || !C)) return fail(BOLT_E_NULL, "NULL query/centroid pointer");
    return BOLT_OK;
}

bolt_status bolt_build_luts(const float* Q, int64_t nq, int j, int64_t ldq, const float* C, int m,
                            bolt_metric metric, float* luts, bolt_stream_t stream) {
    TRY(lut_common(Q, nq, j, ldq, C, m, metric));
    if (nq == 0) return BOLT_OK;
    if (!luts) return fail(BOLT_E_NULL, "luts NULL");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_build_luts(Q, nq, j, ldq, C, m, metric, 1.f, nullptr, nullptr, luts,
                                         nullptr, (cudaStream_t)stream), "bolt_build_luts");
}

bolt_status bolt_build_luts_f64(const float* Q, int64_t nq, int j, int64_t ldq, const float* C,
                                int m, bolt_metric metric, double* luts, bolt_stream_t stream) {
    TRY(lut_common(Q, nq, j, ldq, C, m, metric));
    if (nq == 0) return BOLT_OK;
    if (!luts) return fail(BOLT_E_NULL, "luts NULL");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_build_luts(Q, nq, j, ldq, C, m, metric, 1.f, nullptr, nullptr, nullptr,
                                         luts, (cudaStream_t)stream), "bolt_build_luts_f64");
}

bolt_status bolt_quantize_luts(const float* luts, int64_t nq, int m, float a, const float* b,
                               uint8_t* qluts, bolt_stream_t stream) {
    TRY(check_m(m));
    if (nq < 0) return fail(BOLT_E_SHAPE, "nq < 0");
    if (!(a > 0.f)) return fail(BOLT_E_RANGE, "a = %g must be > 0", (double)a);
    if (nq == 0) return BOLT_OK;
    if (!luts || !b || !qluts) return fail(BOLT_E_NULL, "bolt_quantize_luts: NULL pointer");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_quantize(luts, nq, m, a, b, qluts, (cudaStream_t)stream), "bolt_quantize_luts");
}

bolt_status bolt_build_quantized_luts(const float* Q, int64_t nq, int j, int64_t ldq, const float* C,
                                      int m, bolt_metric metric, float a, const float* b,
                                      uint8_t* qluts, float* luts_or_null, bolt_stream_t stream) {
    TRY(lut_common(Q, nq, j, ldq, C, m, metric));
    if (!(a > 0.f)) return fail(BOLT_E_RANGE, "a = %g must be > 0", (double)a);
    if (nq == 0) return BOLT_OK;
    if (!b || !qluts) return fail(BOLT_E_NULL, "bolt_build_quantized_luts: NULL pointer");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_build_luts(Q, nq, j, ldq, C, m, metric, a, b, qluts, luts_or_null,
                                         nullptr, (cudaStream_t)stream), "bolt_build_quantized_luts");
}

static bolt_status scan_common(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts,
                               int64_t nq) {
    TRY(check_m(m));
    if (n < 0 || nq < 0) return fail(BOLT_E_SHAPE, "n or nq < 0");
    if (n > 0 && nq > 0) {
        if (!codes || !qluts) return fail(BOLT_E_NULL, "codes/qluts NULL");
        if (!aligned(codes, 16)) return fail(BOLT_E_ALIGN, "codes must be 16-byte aligned");
        if (!aligned(qluts, 16)) return fail(BOLT_E_ALIGN, "qluts must be 16-byte aligned");
    }
    return BOLT_OK;
}

// Full-output scan dispatch: the tcgen05 contraction for batched queries
// (nq >= 64, m in {8, 16, 32}), else the PRMT kernel.
static int scan_variant(int64_t n, int m, int64_t nq, int variant) {
    if (variant == BOLT_VARIANT_AUTO) return scan_tc_supported(n, m, nq) && nq >= 64 ? BOLT_VARIANT_TC : BOLT_VARIANT_PRMT;
    return variant;
}

bolt_status bolt_scan_ex(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts, int64_t nq,
                         uint16_t* out, int64_t ldo, int variant, bolt_stream_t stream) {
    TRY(scan_common(codes, n, m, qluts, nq));
    if (ldo < nq) return fail(BOLT_E_SHAPE, "ldo = %lld < nq = %lld", (long long)ldo, (long long)nq);
    if (variant < BOLT_VARIANT_AUTO || variant > BOLT_VARIANT_TC) return fail(BOLT_E_RANGE, "variant %d", variant);
    if (variant == BOLT_VARIANT_TC && !scan_tc_supported(n, m, nq))
        return fail(BOLT_E_RANGE, "tcgen05 scan does not support m=%d", m);
    if (n == 0 || nq == 0) return BOLT_OK;
    if (!out) return fail(BOLT_E_NULL, "out NULL");
    DevInfo d;
    TRY(device_info(&d));
    ScanArgs a{codes, n, ceil_div(n, 8), m, qluts, nq};
    cudaStream_t s = (cudaStream_t)stream;
    return cuda_status(scan_variant(n, m, nq, variant) == BOLT_VARIANT_TC
                           ? launch_scan_tc(a, out, nullptr, ldo, 0.f, 0.f, d.sms, s)
                           : launch_scan_full(a, out, nullptr, ldo, 0.f, 0.f, s),
                       "bolt_scan");
}

bolt_status bolt_scan(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts, int64_t nq,
                      uint16_t* out, int64_t ldo, bolt_stream_t stream) {
    return bolt_scan_ex(codes, n, m, qluts, nq, out, ldo, BOLT_VARIANT_AUTO, stream);
}

bolt_status bolt_scan_dequant_ex(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts,
                                 int64_t nq, float a, float b_sum, float* out, int64_t ldo, int variant,
                                 bolt_stream_t stream) {
    TRY(scan_common(codes, n, m, qluts, nq));
    if (ldo < nq) return fail(BOLT_E_SHAPE, "ldo = %lld < nq = %lld", (long long)ldo, (long long)nq);
    if (!(a > 0.f)) return fail(BOLT_E_RANGE, "a = %g must be > 0", (double)a);
    if (variant < BOLT_VARIANT_AUTO || variant > BOLT_VARIANT_TC) return fail(BOLT_E_RANGE, "variant %d", variant);
    if (variant == BOLT_VARIANT_TC && !scan_tc_supported(n, m, nq))
        return fail(BOLT_E_RANGE, "tcgen05 scan does not support m=%d", m);
    if (n == 0 || nq == 0) return BOLT_OK;
    if (!out) return fail(BOLT_E_NULL, "out NULL");
    DevInfo d;
    TRY(device_info(&d));
    ScanArgs sa{codes, n, ceil_div(n, 8), m, qluts, nq};
    cudaStream_t s = (cudaStream_t)stream;
    return cuda_status(scan_variant(n, m, nq, variant) == BOLT_VARIANT_TC
                           ? launch_scan_tc(sa, nullptr, out, ldo, 1.0f / a, b_sum, d.sms, s)
                           : launch_scan_full(sa, nullptr, out, ldo, 1.0f / a, b_sum, s),
                       "bolt_scan_dequant");
}

bolt_status bolt_scan_dequant(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts,
                              int64_t nq, float a, float b_sum, float* out, int64_t ldo,
                              bolt_stream_t stream) {
    return bolt_scan_dequant_ex(codes, n, m, qluts, nq, a, b_sum, out, ldo, BOLT_VARIANT_AUTO, stream);
}

size_t bolt_topk_workspace_bytes_ex(int64_t n, int m, int64_t nq, int k, int variant) {
    if (n < 0 || nq <= 0 || k < 1 || k > kMaxK || m < 1 || m > kMaxM) return 0;
    return topk_plan(n, m, nq, k, variant, sms_or_default()).ws;
}

bolt_status bolt_topk_plan(int64_t n, int m, int64_t nq, int k, int variant, int* resolved_variant,
                           int* parts) {
    TRY(check_m(m));
    if (n < 0 || nq < 0 || k < 1 || k > kMaxK) return fail(BOLT_E_SHAPE, "bad n/nq/k");
    if (variant < BOLT_VARIANT_AUTO || variant > BOLT_VARIANT_SP) return fail(BOLT_E_RANGE, "variant %d", variant);
    TopkPlan p = topk_plan(n, m, nq, k, variant, sms_or_default());
    if (resolved_variant) *resolved_variant = p.variant;
    if (parts) *parts = p.parts;
    return BOLT_OK;
}

size_t bolt_topk_workspace_bytes(int64_t n, int m, int64_t nq, int k) {
    return bolt_topk_workspace_bytes_ex(n, m, nq, k, BOLT_VARIANT_AUTO);
}

bolt_status bolt_topk_ex(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts,
                         int64_t nq, int k, bolt_metric metric, int64_t index_base,
                         uint64_t* out_keys, void* ws, size_t ws_bytes, int variant,
                         bolt_stream_t stream) {
    TRY(scan_common(codes, n, m, qluts, nq));
    if (k < 1 || k > kMaxK) return fail(BOLT_E_SHAPE, "k = %d outside 1..128", k);
    if (metric != BOLT_L2SQ && metric != BOLT_DOT) return fail(BOLT_E_RANGE, "metric %d", (int)metric);
    if (variant < BOLT_VARIANT_AUTO || variant > BOLT_VARIANT_SP) return fail(BOLT_E_RANGE, "variant %d", variant);
    if (index_base < 0 || index_base + n >= (int64_t(1) << 48))
        return fail(BOLT_E_RANGE, "index_base + n must be < 2^48");
    if (nq == 0) return BOLT_OK;
    if (!out_keys) return fail(BOLT_E_NULL, "out_keys NULL");
    DevInfo d;
    TRY(device_info(&d));
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0)
        return cuda_status(cudaMemsetAsync(out_keys, 0xFF, (size_t)nq * k * sizeof(uint64_t), s), "bolt_topk");
    if (variant == BOLT_VARIANT_TC && !topk_tc_supported(n, m, nq, k))
        return fail(BOLT_E_RANGE, "tcgen05 variant does not support m=%d k=%d", m, k);
    if (variant == BOLT_VARIANT_TCS && !topk_tcs_supported(n, m, nq, k))
        return fail(BOLT_E_RANGE, "swapped tcgen05 variant needs m in {8,16,32}, nq <= 128, k <= 32");
    if (variant == BOLT_VARIANT_SP && !topk_sp_supported(n, m, nq, k))
        return fail(BOLT_E_RANGE, "sparse tcgen05 variant needs m in {8,16,32}, k <= 32 (k <= 16 for m = 32)");
    TopkPlan p = topk_plan(n, m, nq, k, variant, d.sms);
    if (p.ws > 0 && (!ws || ws_bytes < p.ws))
        return fail(BOLT_E_WORKSPACE, "workspace of %zu bytes required, %zu given", p.ws, ws_bytes);
    if (p.ws > 0 && !aligned(ws, 8)) return fail(BOLT_E_ALIGN, "workspace must be 8-byte aligned");
    ScanArgs a{codes, n, ceil_div(n, 8), m, qluts, nq};
    uint64_t* parts_out = p.parts > 1 ? static_cast<uint64_t*>(ws) : out_keys;
    cudaError_t e = cudaSuccess;
    if (p.variant == BOLT_VARIANT_SP) {
        e = launch_topk_sp(a, k, metric, index_base, p.parts, parts_out, s);
        if (e != cudaSuccess) return cuda_status(e, "bolt_topk scan");
        return cuda_status(launch_merge_many(parts_out, p.parts, nq, k, k, out_keys, s), "bolt_topk merge");
    }
    if (p.variant == BOLT_VARIANT_TCS) {
        e = launch_topk_tcs(a, k, metric, index_base, p.parts, parts_out, s);
        if (e != cudaSuccess) return cuda_status(e, "bolt_topk scan");
        return cuda_status(launch_merge_many(parts_out, p.parts, nq, k, k, out_keys, s), "bolt_topk merge");
    }
    if (p.variant == BOLT_VARIANT_TC && k > kTcListMax) {
        // lists of 32 per (query, partition), no shared thresholds; merged into
        // k keys; a query is exact unless some list's 32nd key lies below the
        // merged k-th key -- those queries (rare) are redone exactly by the
        // PRMT kernels.  One host synchronisation (the flag count).
        a.noshare = (k + kTcListMax - 1) / kTcListMax;  // group-shared thresholds (scan_tc.cu)
        e = launch_topk_tc(a, kTcListMax, metric, index_base, p.parts, parts_out, d.sms, s);
        if (e != cudaSuccess) return cuda_status(e, "bolt_topk scan");
        char* lp = static_cast<char*>(ws) + p.large_off;
        uint32_t* flags = reinterpret_cast<uint32_t*>(lp);
        uint32_t* count = flags + nq;
        lp += align256((size_t)nq * sizeof(uint32_t) + 16);
        uint8_t* fq = reinterpret_cast<uint8_t*>(lp); lp += align256((size_t)kFallbackBatch * m * kK);
        uint64_t* fk = reinterpret_cast<uint64_t*>(lp); lp += align256((size_t)kFallbackBatch * k * sizeof(uint64_t));
        void* fws = lp;
        const size_t fws_bytes = p.ws - (size_t)(lp - static_cast<char*>(ws));
        TRY(cuda_status(launch_merge_lists(parts_out, p.parts, nq, kTcListMax, k, out_keys, flags, count, s),
                        "bolt_topk merge"));
        uint32_t hcount = 0;
        TRY(cuda_status(cudaMemcpyAsync(&hcount, count, sizeof(uint32_t), cudaMemcpyDeviceToHost, s), "count"));
        TRY(cuda_status(cudaStreamSynchronize(s), "sync"));
        if (hcount == 0) return BOLT_OK;
        uint32_t* hflags = static_cast<uint32_t*>(malloc((size_t)nq * sizeof(uint32_t)));
        if (!hflags) return fail(BOLT_E_CUDA, "host allocation failed");
        cudaError_t ce = cudaMemcpy(hflags, flags, (size_t)nq * sizeof(uint32_t), cudaMemcpyDeviceToHost);
        if (ce != cudaSuccess) { free(hflags); return cuda_status(ce, "flags"); }
        int64_t qs[kFallbackBatch];
        int nb = 0;
        bolt_status st = BOLT_OK;
        for (int64_t q = 0; q <= nq && st == BOLT_OK; ++q) {
            if (q < nq && hflags[q]) {
                ce = cudaMemcpyAsync(fq + (size_t)nb * m * kK, qluts + (size_t)q * m * kK, (size_t)m * kK,
                                     cudaMemcpyDeviceToDevice, s);
                if (ce != cudaSuccess) { st = cuda_status(ce, "gather"); break; }
                qs[nb++] = q;
            }
            if (nb == kFallbackBatch || (q == nq && nb > 0)) {
                st = bolt_topk_ex(codes, n, m, fq, nb, k, metric, index_base, fk, fws, fws_bytes, BOLT_VARIANT_PRMT,
                                  stream);
                for (int i = 0; i < nb && st == BOLT_OK; ++i) {
                    ce = cudaMemcpyAsync(out_keys + qs[i] * k, fk + (size_t)i * k, (size_t)k * sizeof(uint64_t),
                                         cudaMemcpyDeviceToDevice, s);
                    if (ce != cudaSuccess) st = cuda_status(ce, "scatter");
                }
                nb = 0;
            }
        }
        free(hflags);
        return st;
    } else if (p.small) {
        if (p.parts == 1) {  // the kernel needs its threshold words: keep them in a 1-list workspace
            e = launch_topk_small(a, k, metric, index_base, 1, static_cast<uint64_t*>(ws), s);
            if (e != cudaSuccess) return cuda_status(e, "bolt_topk scan");
            return cuda_status(cudaMemcpyAsync(out_keys, ws, (size_t)nq * k * sizeof(uint64_t),
                                               cudaMemcpyDeviceToDevice, s), "bolt_topk copy");
        }
        e = launch_topk_small(a, k, metric, index_base, p.parts, parts_out, s);
    } else {
        e = p.variant == BOLT_VARIANT_TC ? launch_topk_tc(a, k, metric, index_base, p.parts, parts_out, d.sms, s)
                                         : launch_topk_prmt(a, k, metric, index_base, p.parts, parts_out, d.sms, s);
    }
    if (e != cudaSuccess) return cuda_status(e, "bolt_topk scan");
    if (p.small && p.parts > 64)
        return cuda_status(launch_merge_many(parts_out, p.parts, nq, k, k, out_keys, s), "bolt_topk merge");
    if (p.parts > 1) return cuda_status(launch_merge(parts_out, p.parts, nq, k, out_keys, s), "bolt_topk merge");
    return BOLT_OK;
}

bolt_status bolt_topk(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts, int64_t nq,
                      int k, bolt_metric metric, int64_t index_base, uint64_t* out_keys, void* ws,
                      size_t ws_bytes, bolt_stream_t stream) {
    return bolt_topk_ex(codes, n, m, qluts, nq, k, metric, index_base, out_keys, ws, ws_bytes,
                        BOLT_VARIANT_AUTO, stream);
}

bolt_status bolt_topk_merge(const uint64_t* keys, int w, int64_t nq, int k, uint64_t* out_keys,
                            bolt_stream_t stream) {
    if (w < 1 || k < 1 || nq < 0) return fail(BOLT_E_SHAPE, "w, k must be >= 1, nq >= 0");
    if (w > kMaxParts || k > kMaxK) return fail(BOLT_E_SHAPE, "w = %d > 16384 or k = %d > 128", w, k);
    if (nq == 0) return BOLT_OK;
    if (!keys || !out_keys) return fail(BOLT_E_NULL, "bolt_topk_merge: NULL pointer");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_merge(keys, w, nq, k, out_keys, (cudaStream_t)stream), "bolt_topk_merge");
}

bolt_status bolt_keys_split(const uint64_t* keys, int64_t count, bolt_metric metric,
                            uint16_t* vals, int64_t* idx, bolt_stream_t stream) {
    if (count < 0) return fail(BOLT_E_SHAPE, "count < 0");
    if (metric != BOLT_L2SQ && metric != BOLT_DOT) return fail(BOLT_E_RANGE, "metric %d", (int)metric);
    if (count == 0) return BOLT_OK;
    if (!keys || (!vals && !idx)) return fail(BOLT_E_NULL, "bolt_keys_split: NULL pointer");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_keys_split(keys, count, metric, vals, idx, (cudaStream_t)stream), "bolt_keys_split");
}

// ------------------------------------------------------------ host search
size_t bolt_search_host_workspace_bytes(int64_t n, int j, int m, int64_t nq, int k) {
    if (n < 0 || nq < 0 || j < 1 || m < 1 || m > kMaxM || k < 1 || k > kMaxK) return 0;
    size_t s = 0;
    s += align256((size_t)n * j * sizeof(float));
    s += align256((size_t)nq * j * sizeof(float));
    s += align256((size_t)ceil_div(n, 8) * m * sizeof(uint32_t));
    s += align256((size_t)nq * m * kK);
    s += align256((size_t)nq * k * sizeof(uint64_t));
    s += align256(bolt_topk_workspace_bytes(n, m, nq, k));
    return s;
}

bolt_status bolt_search_host(const float* X_host, int64_t n, int j, const float* Q_host,
                             int64_t nq, const float* C, int m, bolt_metric metric, float a,
                             const float* b, int k, uint64_t* keys_host, void* ws,
                             size_t ws_bytes, bolt_stream_t stream) {
    return bolt_search_host_ex(X_host, n, j, Q_host, nq, C, m, metric, a, b, k, 0, keys_host, ws, ws_bytes, stream);
}

bolt_status bolt_search_host_ex(const float* X_host, int64_t n, int j, const float* Q_host,
                                int64_t nq, const float* C, int m, bolt_metric metric, float a,
                                const float* b, int k, int64_t index_base, uint64_t* keys_host, void* ws,
                                size_t ws_bytes, bolt_stream_t stream) {
    TRY(check_jm(j, m));
    if (n < 1 || nq < 0) return fail(BOLT_E_SHAPE, "n must be >= 1, nq >= 0");
    if (k < 1 || k > kMaxK) return fail(BOLT_E_SHAPE, "k = %d outside 1..128", k);
    if (!(a > 0.f)) return fail(BOLT_E_RANGE, "a must be > 0");
    if (nq == 0) return BOLT_OK;
    if (!X_host || !Q_host || !C || !b || !keys_host || !ws) return fail(BOLT_E_NULL, "bolt_search_host: NULL pointer");
    const size_t need = bolt_search_host_workspace_bytes(n, j, m, nq, k);
    if (ws_bytes < need) return fail(BOLT_E_WORKSPACE, "workspace of %zu bytes required, %zu given", need, ws_bytes);
    if (!aligned(ws, 256)) return fail(BOLT_E_ALIGN, "workspace must be 256-byte aligned");
    DevInfo d;
    TRY(device_info(&d));
    cudaStream_t s = (cudaStream_t)stream;
    char* p = static_cast<char*>(ws);
    float* Xd = reinterpret_cast<float*>(p); p += align256((size_t)n * j * sizeof(float));
    float* Qd = reinterpret_cast<float*>(p); p += align256((size_t)nq * j * sizeof(float));
    uint32_t* codes = reinterpret_cast<uint32_t*>(p); p += align256((size_t)ceil_div(n, 8) * m * sizeof(uint32_t));
    uint8_t* ql = reinterpret_cast<uint8_t*>(p); p += align256((size_t)nq * m * kK);
    uint64_t* keys = reinterpret_cast<uint64_t*>(p); p += align256((size_t)nq * k * sizeof(uint64_t));
    void* tws = p;
    const size_t tws_bytes = bolt_topk_workspace_bytes(n, m, nq, k);
    TRY(cuda_status(cudaMemcpyAsync(Xd, X_host, (size_t)n * j * sizeof(float), cudaMemcpyHostToDevice, s), "H2D X"));
    TRY(cuda_status(cudaMemcpyAsync(Qd, Q_host, (size_t)nq * j * sizeof(float), cudaMemcpyHostToDevice, s), "H2D Q"));
    TRY(bolt_encode(Xd, n, j, j, C, m, codes, stream));
    TRY(bolt_build_quantized_luts(Qd, nq, j, j, C, m, metric, a, b, ql, nullptr, stream));
    TRY(bolt_topk(codes, n, m, ql, nq, k, metric, index_base, keys, tws, tws_bytes, stream));
    return cuda_status(cudaMemcpyAsync(keys_host, keys, (size_t)nq * k * sizeof(uint64_t), cudaMemcpyDeviceToHost, s), "D2H keys");
}

// ------------------------------------------------------------------- fit
// Pipelined host search: the database crosses PCIe in `chunks` row blocks on
// copy_stream while `stream` encodes and scans the blocks already resident
// (per-block top-k with the global index base), so the compute hides under the
// host->device copy; the block lists are merged at the end (exact: total key
// order).  Events are created per call and released after enqueueing.
static int64_t chunk_row(int64_t n, int chunks, int i) {
    // boundaries at multiples of 256 rows (whole layout-v1 groups and scan tiles)
    const int64_t per = ceil_div(ceil_div(n, chunks), 256) * 256;
    return min64(n, per * i);
}

size_t bolt_search_host_pipelined_workspace_bytes(int64_t n, int j, int m, int64_t nq, int k, int chunks) {
    if (n < 0 || nq < 0 || j < 1 || m < 1 || m > kMaxM || k < 1 || k > kMaxK || chunks < 1 || chunks > 64) return 0;
    size_t s = 0;
    s += align256((size_t)n * j * sizeof(float));
    s += align256((size_t)nq * j * sizeof(float));
    s += align256((size_t)ceil_div(n, 8) * m * sizeof(uint32_t));
    s += align256((size_t)nq * m * kK);
    s += align256((size_t)chunks * nq * k * sizeof(uint64_t));
    s += align256((size_t)nq * k * sizeof(uint64_t));
    size_t tws = 0;
    for (int i = 0; i < chunks; ++i) {
        const int64_t r = chunk_row(n, chunks, i + 1) - chunk_row(n, chunks, i);
        if (r > 0) tws = tws > bolt_topk_workspace_bytes(r, m, nq, k) ? tws : bolt_topk_workspace_bytes(r, m, nq, k);
    }
    return s + align256(tws);
}

bolt_status bolt_search_host_pipelined(const float* X_host, int64_t n, int j, const float* Q_host, int64_t nq,
                                       const float* C, int m, bolt_metric metric, float a, const float* b, int k,
                                       uint64_t* keys_host, void* ws, size_t ws_bytes, int chunks,
                                       bolt_stream_t stream, bolt_stream_t copy_stream) {
    return bolt_search_host_pipelined_ex(X_host, n, j, Q_host, nq, C, m, metric, a, b, k, 0, keys_host, ws, ws_bytes,
                                         chunks, stream, copy_stream);
}

bolt_status bolt_search_host_pipelined_ex(const float* X_host, int64_t n, int j, const float* Q_host, int64_t nq,
                                          const float* C, int m, bolt_metric metric, float a, const float* b, int k,
                                          int64_t index_base, uint64_t* keys_host, void* ws, size_t ws_bytes,
                                          int chunks, bolt_stream_t stream, bolt_stream_t copy_stream) {
    TRY(check_jm(j, m));
    if (n < 1 || nq < 0) return fail(BOLT_E_SHAPE, "n must be >= 1, nq >= 0");
    if (k < 1 || k > kMaxK) return fail(BOLT_E_SHAPE, "k = %d outside 1..128", k);
    if (chunks < 1 || chunks > 64) return fail(BOLT_E_RANGE, "chunks = %d outside 1..64", chunks);
    if (!(a > 0.f)) return fail(BOLT_E_RANGE, "a must be > 0");
    if (nq == 0) return BOLT_OK;
    if (!X_host || !Q_host || !C || !b || !keys_host || !ws) return fail(BOLT_E_NULL, "bolt_search_host_pipelined: NULL pointer");
    const size_t need = bolt_search_host_pipelined_workspace_bytes(n, j, m, nq, k, chunks);
    if (ws_bytes < need) return fail(BOLT_E_WORKSPACE, "workspace of %zu bytes required, %zu given", need, ws_bytes);
    if (!aligned(ws, 256)) return fail(BOLT_E_ALIGN, "workspace must be 256-byte aligned");
    DevInfo d;
    TRY(device_info(&d));
    cudaStream_t s = (cudaStream_t)stream, cs = (cudaStream_t)copy_stream;
    char* p = static_cast<char*>(ws);
    float* Xd = reinterpret_cast<float*>(p); p += align256((size_t)n * j * sizeof(float));
    float* Qd = reinterpret_cast<float*>(p); p += align256((size_t)nq * j * sizeof(float));
    uint32_t* codes = reinterpret_cast<uint32_t*>(p); p += align256((size_t)ceil_div(n, 8) * m * sizeof(uint32_t));
    uint8_t* ql = reinterpret_cast<uint8_t*>(p); p += align256((size_t)nq * m * kK);
    uint64_t* parts = reinterpret_cast<uint64_t*>(p); p += align256((size_t)chunks * nq * k * sizeof(uint64_t));
    uint64_t* keys = reinterpret_cast<uint64_t*>(p); p += align256((size_t)nq * k * sizeof(uint64_t));
    void* tws = p;
    const size_t tws_bytes = need - (size_t)(p - static_cast<char*>(ws));
    cudaEvent_t start, ev[64];
    TRY(cuda_status(cudaEventCreateWithFlags(&start, cudaEventDisableTiming), "event"));
    // the copies may only overwrite Xd once everything enqueued on `stream` before this call is done
    TRY(cuda_status(cudaEventRecord(start, s), "event record"));
    TRY(cuda_status(cudaStreamWaitEvent(cs, start, 0), "stream wait"));
    cudaEventDestroy(start);
    // Q first on the copy stream: host->device copies share one DMA queue, so a
    // Q copy behind the X blocks would hold the tables (and every block's scan)
    // until all of X had landed
    cudaEvent_t evq;
    TRY(cuda_status(cudaEventCreateWithFlags(&evq, cudaEventDisableTiming), "event"));
    TRY(cuda_status(cudaMemcpyAsync(Qd, Q_host, (size_t)nq * j * sizeof(float), cudaMemcpyHostToDevice, cs), "H2D Q"));
    TRY(cuda_status(cudaEventRecord(evq, cs), "event record"));
    int used = 0;
    for (int i = 0; i < chunks; ++i) {
        const int64_t r0 = chunk_row(n, chunks, i), r1 = chunk_row(n, chunks, i + 1);
        if (r1 <= r0) break;
        TRY(cuda_status(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event"));
        TRY(cuda_status(cudaMemcpyAsync(Xd + r0 * j, X_host + r0 * j, (size_t)(r1 - r0) * j * sizeof(float),
                                        cudaMemcpyHostToDevice, cs), "H2D X"));
        TRY(cuda_status(cudaEventRecord(ev[i], cs), "event record"));
        used = i + 1;
    }
    TRY(cuda_status(cudaStreamWaitEvent(s, evq, 0), "stream wait"));
    cudaEventDestroy(evq);
    TRY(bolt_build_quantized_luts(Qd, nq, j, j, C, m, metric, a, b, ql, nullptr, stream));
    for (int i = 0; i < used; ++i) {
        const int64_t r0 = chunk_row(n, chunks, i), r1 = chunk_row(n, chunks, i + 1);
        TRY(cuda_status(cudaStreamWaitEvent(s, ev[i], 0), "stream wait"));
        cudaEventDestroy(ev[i]);
        uint32_t* cw = codes + (r0 / 8) * m;
        TRY(bolt_encode(Xd + r0 * j, r1 - r0, j, j, C, m, cw, stream));
        TRY(bolt_topk(cw, r1 - r0, m, ql, nq, k, metric, index_base + r0, used == 1 ? keys : parts + (size_t)i * nq * k, tws,
                      tws_bytes, stream));
    }
    if (used > 1) TRY(bolt_topk_merge(parts, used, nq, k, keys, stream));
    return cuda_status(cudaMemcpyAsync(keys_host, keys, (size_t)nq * k * sizeof(uint64_t), cudaMemcpyDeviceToHost, s), "D2H keys");
}

size_t bolt_kmeans_workspace_bytes(int64_t n, int j, int m) {
    if (n < 1 || j < 1 || m < 1 || m > kMaxM || j % m) return 0;
    return kmeans_ws_bytes(n, j, m);
}

bolt_status bolt_kmeans(const float* train, int64_t n, int j, int64_t ldx, int m,
                        const int64_t* init, int iters, float* C_out, void* ws, size_t ws_bytes,
                        bolt_stream_t stream) {
    TRY(check_jm(j, m));
    if (n < kK) return fail(BOLT_E_SHAPE, "k-means needs n >= 16 rows, got %lld", (long long)n);
    if (ldx < j) return fail(BOLT_E_SHAPE, "ldx < j");
    if (iters < 0) return fail(BOLT_E_RANGE, "iters < 0");
    if (j / m > 64) return fail(BOLT_E_SHAPE, "sub-vector length j/m = %d > 64", j / m);
    if (!train || !init || !C_out) return fail(BOLT_E_NULL, "bolt_kmeans: NULL pointer");
    const size_t need = kmeans_ws_bytes(n, j, m);
    if (!ws || ws_bytes < need) return fail(BOLT_E_WORKSPACE, "workspace of %zu bytes required", need);
    if (!aligned(ws, 256)) return fail(BOLT_E_ALIGN, "workspace must be 256-byte aligned");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_kmeans(train, n, j, ldx, m, init, iters, C_out, ws, (cudaStream_t)stream), "bolt_kmeans");
}

size_t bolt_calibrate_workspace_bytes(int64_t nq, int m) {
    if (nq < 1 || m < 1 || m > kMaxM) return 0;
    return calibrate_ws_bytes(nq, m);
}

bolt_status bolt_calibrate(const double* luts, int64_t nq, int m, float* a_out, float* b_out,
                           double* alpha_mse_out, void* ws, size_t ws_bytes, bolt_stream_t stream) {
    TRY(check_m(m));
    if (nq < 1) return fail(BOLT_E_SHAPE, "nq must be >= 1");
    if (!luts || !a_out || !b_out) return fail(BOLT_E_NULL, "bolt_calibrate: NULL pointer");
    const size_t need = calibrate_ws_bytes(nq, m);
    if (!ws || ws_bytes < need) return fail(BOLT_E_WORKSPACE, "workspace of %zu bytes required", need);
    if (!aligned(ws, 256)) return fail(BOLT_E_ALIGN, "workspace must be 256-byte aligned");
    DevInfo d;
    TRY(device_info(&d));
    return cuda_status(launch_calibrate(luts, nq, m, a_out, b_out, alpha_mse_out, ws, (cudaStream_t)stream),
                       "bolt_calibrate");
}

}  // extern "C"
