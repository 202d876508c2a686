/*
 * bolt.h -- C ABI (v1) of the B200-native Bolt read-side hot path.
 *
 * Bolt (Blalock & Guttag, KDD'17, arXiv 1706.10283): 4-bit product
 * quantization (K = 16 centroids per codebook) with
 * learned 8-bit lookup tables (L262-291) scanned with vectorized in-register
 * lookups (L264).  "P:Lx" below = /root/reference/PAPER.md line x; "R<n>" =
 * reading n in DESIGN.md ("Readings of the paper").
 *
 * Conventions (every entry point):
 *  - Pointers are DEVICE pointers unless marked (host).  The caller allocates
 *    and frees everything; the library keeps no pointer after the call's
 *    enqueued work and allocates nothing (CUDA-graph capturable).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *    Calls validate their arguments synchronously, then enqueue kernels on
 *    `stream` and return without synchronizing.  Asynchronous device faults
 *    surface at the caller's next synchronization.
 *  - Return value: BOLT_OK, or an error code with nothing enqueued (argument
 *    errors) / a launch failure (BOLT_E_CUDA).  bolt_last_error() returns a
 *    thread-local message for the last non-OK status of the calling thread.
 *  - No C++ exception crosses the ABI; every function is thread-safe.
 *  - Device values (codes, tables) are not validated: codes are masked to 4
 *    bits where they are read.
 *
 * Shapes: n database vectors of dimension j; m codebooks (1 <= m <= 64,
 * j % m == 0; zero-pad otherwise, which is exact for both metrics since
 * delta(0,0) = 0); sub-vector length L = j / m, sub-vector p_m = dims
 * [m*L, (m+1)*L) (R10); nq queries.
 *
 * Code layout v1 (R12): u32 word codes[g*m + c] holds codebook c of rows
 * 8g .. 8g+7, row 8g+r in bits [4r, 4r+4).  bolt_codes_words(n, m) =
 * ceil(n/8)*m words; rows >= n in the last group are zero padding.  A row
 * shard [r0, r1) with r0 % 8 == 0 is the contiguous word range
 * [r0/8*m, ceil(r1/8)*m).
 *
 * Tables: fp32 / fp64 tables D[q][c][i] (i = centroid index, 16 contiguous
 * entries per codebook, row-major [nq][m][16]); quantized tables
 * beta[q][c][i] u8 with the same layout.
 */
#ifndef BOLT_H_
#define BOLT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BOLT_ABI_VERSION 1

#if defined(__GNUC__)
#define BOLT_API __attribute__((visibility("default")))
#else
#define BOLT_API
#endif

typedef void* bolt_stream_t; /* cudaStream_t */

typedef enum {
    BOLT_OK = 0,
    BOLT_E_NULL = 1,      /* a required pointer is NULL */
    BOLT_E_SHAPE = 2,     /* n/j/m/nq/k/ld out of range or inconsistent */
    BOLT_E_RANGE = 3,     /* scalar parameter out of range (metric, variant, a <= 0 ...) */
    BOLT_E_ALIGN = 4,     /* pointer misaligned for the documented access width */
    BOLT_E_DEVICE = 5,    /* current device is not sm_100 / no device */
    BOLT_E_CUDA = 6,      /* CUDA launch or runtime error (see bolt_last_error) */
    BOLT_E_WORKSPACE = 7  /* workspace NULL or smaller than *_workspace_bytes() */
} bolt_status;

/* delta of P:L114-122: squared L2 (delta = (q-x)^2, f = identity; smaller is
 * better) or dot product (delta = q*x, f = identity; larger is better). */
typedef enum { BOLT_L2SQ = 0, BOLT_DOT = 1 } bolt_metric;

/* Scan implementation for bolt_topk_ex / bolt_scan_ex. */
typedef enum {
    BOLT_VARIANT_AUTO = 0,  /* library picks (documented in DESIGN.md) */
    BOLT_VARIANT_PRMT = 1,  /* CUDA-core PRMT byte-permute lookups */
    BOLT_VARIANT_TC = 2,    /* tcgen05 one-hot(codes) x table, kind::i8 */
    BOLT_VARIANT_TCS = 3,   /* tcgen05 with the roles swapped for small query batches:
                               vectors on the MMA's M side, nq <= 128 queries on N
                               (top-k only, k <= 32, m in {8, 16, 32}) */
    BOLT_VARIANT_SP = 4     /* tcgen05.mma.sp (2:4 structured-sparse A = the one-hot
                               codes, compressed): vectors on M, 224
                               queries per tile on N; twice the dense int8 rate
                               (top-k only, m in {8, 16, 32}, k <= 32; k <= 16 for m = 32) */
} bolt_variant;

/* ------------------------------------------------------------------ info */
BOLT_API const char* bolt_version(void);                 /* (host) static string */
BOLT_API const char* bolt_last_error(void);              /* (host) thread-local, never NULL */
BOLT_API int64_t bolt_codes_words(int64_t n, int m);     /* (host) ceil(n/8)*m, -1 on bad args */

/* ------------------------------------------------------------ encode (h) */
/* h(x) = [i_1; ...; i_M], i_m = argmin_i ||x^(m) - c_i^(m)||^2 (
 * squared L2 for both metrics, R9; ties -> lowest i).  fp32 arithmetic.
 *   X     [n][ldx] fp32, row i's j values at X + i*ldx (ldx >= j, 16 B aligned
 *         rows when ldx % 4 == 0)
 *   C     [m][16][j/m] fp32 centroids (the model's codebooks)
 *   codes out, bolt_codes_words(n, m) u32 words, layout v1
 * Errors: NULL, SHAPE (n < 0, j < 1, m not in 1..64, j % m, ldx < j, j/m > 64). */
BOLT_API bolt_status bolt_encode(const float* X, int64_t n, int j, int64_t ldx, const float* C, int m,
                        uint32_t* codes, bolt_stream_t stream);
/* As bolt_encode with an explicit kernel.  BOLT_ENCODE_DIRECT: direct
 * differences, fp32 (x - c)^2 summed in ascending dimension (the arithmetic
 * whose argmin is returned).  BOLT_ENCODE_EXPANDED (j/m in {8, 16}, j % 32 == 0,
 * j <= 512, m % 8 == 0, rows 16 B aligned; else direct): the distances are
 * first ranked by the expansion ||c||^2 - 2 x.c (one FMA per dimension and
 * centroid) and a codebook whose two best centroids lie within that
 * computation's rounding bound is redone by direct differences, so the codes
 * equal BOLT_ENCODE_DIRECT's bit for bit.  BOLT_ENCODE_AUTO: EXPANDED where
 * it applies (measured faster on a B200), DIRECT otherwise.
 * Errors: as bolt_encode; RANGE for another variant. */
enum { BOLT_ENCODE_AUTO = 0, BOLT_ENCODE_DIRECT = 1, BOLT_ENCODE_EXPANDED = 2 };
BOLT_API bolt_status bolt_encode_ex(const float* X, int64_t n, int j, int64_t ldx, const float* C, int m,
                                    uint32_t* codes, int variant, bolt_stream_t stream);

/* Streaming encode-on-write (the write path T_h of P:L72-89,
 * P:L141): encode n_new rows and append them to a live code buffer holding
 * n_old rows, i.e. afterwards `codes` equals bolt_encode of the n_old + n_new
 * rows (bit for bit; same fp32 operations).  When n_old % 8 != 0 the first
 * layout-v1 group is partial: its existing nibbles are kept and the new rows
 * fill the rest (a read-modify-write of that group's m words).
 *   X, j, ldx, C, m as for bolt_encode (X = the n_new new rows)
 *   codes in/out: capacity bolt_codes_words(n_old + n_new, m) words; words of
 *         groups before n_old / 8 are not touched
 * Errors: as bolt_encode, plus SHAPE (n_old < 0). */
BOLT_API bolt_status bolt_encode_append(const float* X, int64_t n_new, int j, int64_t ldx, const float* C, int m,
                                        uint32_t* codes, int64_t n_old, bolt_stream_t stream);

/* Pack flat codes u8 [n][m] (values masked to 4 bits) into layout v1, and back. */
BOLT_API bolt_status bolt_pack_codes(const uint8_t* flat, int64_t n, int m, uint32_t* codes,
                            bolt_stream_t stream);
BOLT_API bolt_status bolt_unpack_codes(const uint32_t* codes, int64_t n, int m, uint8_t* flat,
                              bolt_stream_t stream);

/* -------------------------------------------------------- query tables (g) */
/* D_iq = delta(q^(m), c_i^(m)) summed over the sub-vector in ascending
 * dimension order, accumulated in fp64 from direct differences.
 *   Q [nq][ldq] fp32 queries; C as for bolt_encode.
 *   luts out [nq][m][16] fp32 (bolt_build_luts) or fp64 (bolt_build_luts_f64). */
BOLT_API bolt_status bolt_build_luts(const float* Q, int64_t nq, int j, int64_t ldq, const float* C, int m,
                            bolt_metric metric, float* luts, bolt_stream_t stream);
BOLT_API bolt_status bolt_build_luts_f64(const float* Q, int64_t nq, int j, int64_t ldq, const float* C,
                                int m, bolt_metric metric, double* luts, bolt_stream_t stream);

/* beta = clamp(floor(a * (y - b[c])), 0, 255) computed in fp64 from the fp32
 * inputs (R1: b in distance units).  a > 0 is the global
 * scale (host scalar), b [m] fp32 per-table offsets (device).
 *   luts [nq][m][16] fp32 -> qluts [nq][m][16] u8. */
BOLT_API bolt_status bolt_quantize_luts(const float* luts, int64_t nq, int m, float a, const float* b,
                               uint8_t* qluts, bolt_stream_t stream);

/* Fused g: build (fp64) and quantize from the fp64 value in one kernel.
 * luts_or_null optionally receives the fp32 tables. */
BOLT_API bolt_status bolt_build_quantized_luts(const float* Q, int64_t nq, int j, int64_t ldq, const float* C,
                                      int m, bolt_metric metric, float a, const float* b,
                                      uint8_t* qluts, float* luts_or_null, bolt_stream_t stream);

/* ------------------------------------------------------------ scan (d^) */
/* acc[i][q] = sum_c qluts[q][c][code(i,c)] exactly (<= 255*m <= 16320, R11),
 * the "running total" of P:L224-231 over 8-bit tables.
 *   codes layout v1 for n rows; qluts [nq][m][16] u8 (16 B aligned)
 *   out   u16, out[i*ldo + q] (row = database vector), ldo >= nq */
BOLT_API bolt_status bolt_scan(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts, int64_t nq,
                      uint16_t* out, int64_t ldo, bolt_stream_t stream);

/* Same scan with the affine correction of P:L286/L291 fused (R6, R7):
 * out[i*ldo + q] = (float)acc * (1/a) + b_sum (fp32), b_sum = sum_c b[c]. */
BOLT_API bolt_status bolt_scan_dequant(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts,
                              int64_t nq, float a, float b_sum, float* out, int64_t ldo,
                              bolt_stream_t stream);

/* As bolt_scan / bolt_scan_dequant with an explicit implementation:
 * BOLT_VARIANT_AUTO (tcgen05 when nq >= 64 and m is 8, 16 or 32, else
 * PRMT), BOLT_VARIANT_PRMT, or BOLT_VARIANT_TC (BOLT_E_RANGE for other m).
 * Both variants return the same integers bit for bit; the fp32 output is
 * fmaf((float)acc, 1/a, b_sum) in both. */
BOLT_API bolt_status bolt_scan_ex(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts, int64_t nq,
                                  uint16_t* out, int64_t ldo, int variant, bolt_stream_t stream);
BOLT_API bolt_status bolt_scan_dequant_ex(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts,
                                          int64_t nq, float a, float b_sum, float* out, int64_t ldo, int variant,
                                          bolt_stream_t stream);

/* --------------------------------------------------------------- top-k */
/* k best database vectors per query ("the k closest"; NN and MIPS,
 * P:L33) by the 64-bit key (R13)
 *   L2SQ: key = (acc << 48) | (index_base + i)
 *   DOT : key = ((0xFFFF - acc) << 48) | (index_base + i)
 * ascending, so best first and ties broken by the lower global index.
 *   out_keys [nq][k] u64, sorted ascending; UINT64_MAX padding when k > n.
 *   1 <= k <= 128; index_base + n < 2^48 (index 2^48 - 1 with value 0xFFFF would equal the padding key).
 *   ws: device scratch of at least bolt_topk_workspace_bytes(n, m, nq, k)
 *   bytes (8 B aligned).
 * Asynchronous on `stream`, except on the tcgen05 path with k > 32: lists of
 * 32 are merged and checked, and the call waits for one count of queries
 * that need the exact PRMT rescan (not CUDA-graph capturable). */
BOLT_API size_t bolt_topk_workspace_bytes(int64_t n, int m, int64_t nq, int k);
BOLT_API bolt_status bolt_topk(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts, int64_t nq,
                      int k, bolt_metric metric, int64_t index_base, uint64_t* out_keys, void* ws,
                      size_t ws_bytes, bolt_stream_t stream);
/* The plan bolt_topk_ex will use for these shapes (host): the resolved
 * variant (BOLT_VARIANT_PRMT / BOLT_VARIANT_TC) and the number of row
 * partitions whose partial lists are merged (1 = no merge).  AUTO picks
 * tcgen05 for m in {8, 16, 32}, k <= 128 and nq above 20 (m = 8), 12
 * (m = 16) or 16 (m = 32) — crossovers measured on 10^8 rows (DESIGN.md
 * §1) — else PRMT; the results are the same keys either way. */
BOLT_API bolt_status bolt_topk_plan(int64_t n, int m, int64_t nq, int k, int variant,
                                    int* resolved_variant, int* parts);
/* As bolt_topk with an explicit scan variant (tests, benchmarks). */
BOLT_API size_t bolt_topk_workspace_bytes_ex(int64_t n, int m, int64_t nq, int k, int variant);
BOLT_API bolt_status bolt_topk_ex(const uint32_t* codes, int64_t n, int m, const uint8_t* qluts,
                         int64_t nq, int k, bolt_metric metric, int64_t index_base,
                         uint64_t* out_keys, void* ws, size_t ws_bytes, int variant,
                         bolt_stream_t stream);

/* Merge w sorted key lists [w][nq][k] (indices already global) into the k
 * smallest keys per query [nq][k]; 1 <= w <= 16384, 1 <= k <= 128.  Equals bolt_topk over the
 * union of the shards bit for bit. */
BOLT_API bolt_status bolt_topk_merge(const uint64_t* keys, int w, int64_t nq, int k, uint64_t* out_keys,
                            bolt_stream_t stream);

/* Split keys into values (acc, u16) and global indices (int64, -1 for padding). */
BOLT_API bolt_status bolt_keys_split(const uint64_t* keys, int64_t count, bolt_metric metric,
                            uint16_t* vals, int64_t* idx, bolt_stream_t stream);

/* ------------------------------------------- Bolt No Quantize (fp32 tables) */
/* The variant of P:L390 that skips table quantization: the
 * running total of P:L224-231 over the fp32 tables D of bolt_build_luts,
 * summed in fp32 in ascending codebook order from 0 (R18).
 *   luts [nq][m][16] fp32 (4 B aligned); codes layout v1 for n rows (16 B aligned)
 *   out  fp32, out[i*ldo + q], ldo >= nq
 * Errors: NULL, SHAPE (m not in 1..64, n or nq < 0, ldo < nq), ALIGN. */
BOLT_API bolt_status bolt_scan_f32(const uint32_t* codes, int64_t n, int m, const float* luts, int64_t nq,
                                   float* out, int64_t ldo, bolt_stream_t stream);
/* k best per query of those fp32 totals by the 64-bit key (R18)
 *   key = (ord(v) << 32) | (index_base + i), ord = the float's order-preserving
 *   unsigned code (negative: bits flipped, else sign bit set), inverted for DOT;
 * ascending, best first, ties by the lower index.  1 <= k <= 32;
 * index_base + n <= 2^32.  ws >= bolt_topk_f32_workspace_bytes(n, m, nq, k). */
BOLT_API size_t bolt_topk_f32_workspace_bytes(int64_t n, int m, int64_t nq, int k);
BOLT_API bolt_status bolt_topk_f32(const uint32_t* codes, int64_t n, int m, const float* luts, int64_t nq, int k,
                                   bolt_metric metric, int64_t index_base, uint64_t* out_keys, void* ws,
                                   size_t ws_bytes, bolt_stream_t stream);
/* Split R18 keys into fp32 values and global indices (-1 for padding). */
BOLT_API bolt_status bolt_keys_split_f32(const uint64_t* keys, int64_t count, bolt_metric metric, float* vals,
                                         int64_t* idx, bolt_stream_t stream);

/* ------------------------------------------------- end-to-end (host buffers) */
/* One search from HOST inputs: copies X and Q host->device, encodes X (h),
 * builds quantized tables (g), runs the top-k scan, copies the keys
 * device->host.  Everything is enqueued on `stream`; pinned host buffers make
 * it asynchronous.  ws >= bolt_search_host_workspace_bytes(...) device bytes.
 *   X_host [n][j] fp32, Q_host [nq][j] fp32, keys_host [nq][k] u64 (host)
 *   C [m][16][j/m], b [m] device. */
BOLT_API size_t bolt_search_host_workspace_bytes(int64_t n, int j, int m, int64_t nq, int k);
BOLT_API bolt_status bolt_search_host(const float* X_host, int64_t n, int j, const float* Q_host,
                             int64_t nq, const float* C, int m, bolt_metric metric, float a,
                             const float* b, int k, uint64_t* keys_host, void* ws,
                             size_t ws_bytes, bolt_stream_t stream);
/* As bolt_search_host with the rows' global index base (a row shard
 * starting at row index_base of a larger database; index_base + n < 2^48). */
BOLT_API bolt_status bolt_search_host_ex(const float* X_host, int64_t n, int j, const float* Q_host,
                                         int64_t nq, const float* C, int m, bolt_metric metric, float a,
                                         const float* b, int k, int64_t index_base, uint64_t* keys_host, void* ws,
                                         size_t ws_bytes, bolt_stream_t stream);

/* Same search with the host->device copy of X overlapped with the compute:
 * X crosses in `chunks` row blocks (boundaries at multiples of 256 rows) on
 * copy_stream, while `stream` encodes each block as soon as it has landed and
 * runs its top-k (global indices); the block lists are then merged (the
 * result equals bolt_search_host bit for bit).  copy_stream first waits for
 * the work already enqueued on `stream`.  1 <= chunks <= 64.
 * ws >= bolt_search_host_pipelined_workspace_bytes(...) device bytes. */
BOLT_API size_t bolt_search_host_pipelined_workspace_bytes(int64_t n, int j, int m, int64_t nq, int k, int chunks);
BOLT_API bolt_status bolt_search_host_pipelined(const float* X_host, int64_t n, int j, const float* Q_host,
                                                int64_t nq, const float* C, int m, bolt_metric metric, float a,
                                                const float* b, int k, uint64_t* keys_host, void* ws,
                                                size_t ws_bytes, int chunks, bolt_stream_t stream,
                                                bolt_stream_t copy_stream);
/* As bolt_search_host_pipelined with the rows' global index base. */
BOLT_API bolt_status bolt_search_host_pipelined_ex(const float* X_host, int64_t n, int j, const float* Q_host,
                                                   int64_t nq, const float* C, int m, bolt_metric metric, float a,
                                                   const float* b, int k, int64_t index_base, uint64_t* keys_host,
                                                   void* ws, size_t ws_bytes, int chunks, bolt_stream_t stream,
                                                   bolt_stream_t copy_stream);

/* ----------------------------------------------- offline fit */
/* k-means codebooks (R8): per subspace, centroids start at rows
 * init[c][0..15] of train, exactly `iters` Lloyd iterations in fp64
 * (assignment ties -> lowest centroid; empty cluster -> farthest point, ties
 * -> lowest row, rows used once per iteration).  Deterministic.
 *   train [n][ldx] fp32, init [m][16] int64 (device), C_out [m][16][j/m] fp32. */
BOLT_API size_t bolt_kmeans_workspace_bytes(int64_t n, int j, int m);
BOLT_API bolt_status bolt_kmeans(const float* train, int64_t n, int j, int64_t ldx, int m,
                        const int64_t* init, int iters, float* C_out, void* ws, size_t ws_bytes,
                        bolt_stream_t stream);

/* LUT-quantizer learning (R1-R4) from fp64 tables of calibration
 * queries [nq][m][16]: alpha grid {0,.001,.002,.005,.01,.02,.05,.1},
 * nearest-rank quantiles, first strictly minimal MSE.  Outputs (device):
 * a_out [1] fp32, b_out [m] fp32, alpha_mse_out [9] fp64 = {alpha, mse[8]}. */
BOLT_API size_t bolt_calibrate_workspace_bytes(int64_t nq, int m);
BOLT_API bolt_status bolt_calibrate(const double* luts, int64_t nq, int m, float* a_out, float* b_out,
                           double* alpha_mse_out, void* ws, size_t ws_bytes, bolt_stream_t stream);

/* ------------------------------------------------------------ diagnostics */
/* (host) Copy up to n internal kernel cycle counters to host `out` and reset
 * them.  All zeros unless the library was built with -DBOLT_PROFILE
 * (python -m paper_1706_10283_b200.build --profile); used by tools/ only.
 * Returns the number of counters written. */
BOLT_API int bolt_debug_counters(uint64_t* out, int n);


#ifdef __cplusplus
}
#endif
#endif /* BOLT_H_ */
