/*
 * bolt_oracle.c -- plain, slow, obviously-correct CPU oracle for Bolt's
 * read-side hot path (Blalock & Guttag, KDD'17, arXiv 1706.10283).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_1706_10283_b200/csrc) and never includes anything from it.
 *
 * Citations: "P:Lx" = /root/reference/PAPER.md line x (LaTeX source),
 * "R<n>" = reading n of DESIGN.md section "Readings of the paper".
 *
 * Precision: every shared input is fp32 (data, queries, centroids C32, a32,
 * b32); all arithmetic here is fp64 (double), integers are int64, sums are
 * taken in ascending index order.  Compiled with -ffp-contract=off so that
 * a*b+c is never fused.  OpenMP only distributes independent outer
 * iterations (rows or queries); it never changes the arithmetic of one
 * output.
 *
 * Functions (O-numbers follow SURVEY.md §8(c)):
 *   O1 split          sub-vector p_m = [m*L, (m+1)*L), L = J/M         P:L204 (R10)
 *   O2 kmeans         per-subspace Lloyd iterations, fixed init/iters  P:L196,L234 (R8)
 *   O3 encode         i_m = argmin_i ||x^(m) - c_i^(m)||^2             P:L214-218 (R9)
 *   O4 luts           D_im = delta(q^(m), c_i^(m))
 *   O5 calibrate      alpha grid, b_m = F^-1(alpha), global a          P:L268-291 (R1-R4)
 *   O6 quantize       beta = clamp(floor(a (y - b_m)), 0, 255)         P:L279, L289 (R1)
 *   O7 scan           sum_m beta[m][i_m] as an exact integer           P:L224-231 (R11)
 *   O8 topk           k smallest (value, index) keys                   P:L143, L33 (R13)
 *   O9 merge          k smallest of the union of shard lists           (R13)
 *   O10 dequant       acc/a + sum_m b_m                                P:L286, L291 (R6, R7)
 *   O12 unpack v1     read the CUDA path's packed code layout          (R12)
 *
 * Parity pins for every function are in tests/test_oracle_*.py; O2 k-means is
 * pinned only by exact-structure cases and monotone inertia.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define K 16 /* centroids per codebook */

enum { ORACLE_L2SQ = 0, ORACLE_DOT = 1 };

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ---------------------------------------------------------------- O1 -- */
/* delta summed over one sub-vector: P:L206-210 ("boldsymbol delta sums the
 * delta functions applied to each dimension"); squared L2 delta=(q-x)^2,
 * dot delta=q*x. */
static double subspace_delta(const float* q, const float* c, int L, int metric) {
    double s = 0.0;
    for (int j = 0; j < L; ++j) {
        double qj = (double)q[j], cj = (double)c[j];
        double t;
        if (metric == ORACLE_L2SQ) {
            double d = qj - cj;
            t = d * d;
        } else {
            t = qj * cj;
        }
        s = s + t;
    }
    return s;
}

static double subspace_l2_f64c(const float* x, const double* c, int L) {
    double s = 0.0;
    for (int j = 0; j < L; ++j) {
        double d = (double)x[j] - c[j];
        s = s + d * d;
    }
    return s;
}

/* ---------------------------------------------------------------- O3 -- */
/* h(x) = [i_1; ...; i_M], i_m = argmin_i d(c_i^(m), x^(m)).
 * d is squared L2 for both metrics (R9); ties go to the lowest i.
 * gap (optional) = (d2 - d1) / max(d2, 1e-30) with d1 <= d2 the two smallest
 * distances -- the near-tie measure of the parity contract. */
void oracle_encode(const float* X, int64_t n, int J, const float* C, int M,
                   uint8_t* codes, double* gap) {
    const int L = J / M;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const float* x = X + i * (int64_t)J;
        for (int m = 0; m < M; ++m) {
            double best = INFINITY, second = INFINITY;
            int arg = 0;
            for (int k = 0; k < K; ++k) {
                double d = subspace_delta(x + m * L, C + ((int64_t)m * K + k) * L, L, ORACLE_L2SQ);
                if (d < best) {
                    second = best;
                    best = d;
                    arg = k;
                } else if (d < second) {
                    second = d;
                }
            }
            codes[i * M + m] = (uint8_t)arg;
            if (gap) gap[i * M + m] = (second - best) / (second > 1e-30 ? second : 1e-30);
        }
    }
}

/* ---------------------------------------------------------------- O4 -- */
/* D_im = delta(q^(m), c_i^(m)); stored D[q][m][i]. */
void oracle_luts(const float* Q, int64_t nq, int J, const float* C, int M, int metric,
                 double* D) {
    const int L = J / M;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nq; ++q)
        for (int m = 0; m < M; ++m)
            for (int k = 0; k < K; ++k)
                D[(q * M + m) * K + k] =
                    subspace_delta(Q + q * (int64_t)J + m * L, C + ((int64_t)m * K + k) * L, L, metric);
}

/* ---------------------------------------------------------------- O6 -- */
/* beta_m(y) = max(0, min(255, floor(a (y - b_m))))  (P:L279 with R1: b_m in
 * distance units, so the alpha quantile maps to 0 as P:L289 states).
 * a and b are the fp32 model parameters promoted to fp64.  t (optional)
 * receives the pre-floor value for the near-tie rule. */
void oracle_quantize(const double* D, int64_t nq, int M, float a32, const float* b32,
                     uint8_t* beta, double* t_out) {
    const double a = (double)a32;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nq; ++q)
        for (int m = 0; m < M; ++m)
            for (int k = 0; k < K; ++k) {
                int64_t e = (q * M + m) * K + k;
                double t = a * (D[e] - (double)b32[m]);
                double f = floor(t);
                if (f < 0.0) f = 0.0;
                if (f > 255.0) f = 255.0;
                beta[e] = (uint8_t)f;
                if (t_out) t_out[e] = t;
            }
}

/* ---------------------------------------------------------------- O5 -- */
static int cmp_double(const void* pa, const void* pb) {
    double a = *(const double*)pa, b = *(const double*)pb;
    return (a > b) - (a < b);
}

/* nearest-rank empirical inverse CDF on a sorted sample (R4) */
static double nearest_rank(const double* sorted, int64_t n, double p) {
    int64_t idx = (int64_t)ceil(p * (double)n) - 1;
    if (idx < 0) idx = 0;
    if (idx > n - 1) idx = n - 1;
    return sorted[idx];
}

static const double ALPHA_GRID[8] = {0.0, 0.001, 0.002, 0.005, 0.01, 0.02, 0.05, 0.1};

/* Learn (a, b_m) on the exact tables D of calibration queries:
 * for each alpha in the grid, b_m = F_m^-1(alpha) over table m's entries,
 * a = 255 / F^-1(1 - alpha) of the aggregated residuals y - b_m over all
 * tables (R2, R3), then the mean squared reconstruction error of
 * yhat = beta/a + b_m (R1).  The first alpha with the strictly
 * smallest error wins (R4).  Outputs are fp64; the model stores them as fp32.
 * mse_out (optional) receives the 8 grid errors; a_grid [8] and b_grid [8][M]
 * (optional) the (a, b_m) of every grid alpha, so that each quantile can be
 * checked on its own, not only the winner's. */
void oracle_calibrate_grid(const double* D, int64_t nq, int M, double* a_out, double* b_out,
                           double* alpha_out, double* mse_out, double* a_grid, double* b_grid) {
    const int64_t per_table = nq * K;
    const int64_t total = per_table * M;
    double* col = (double*)malloc(sizeof(double) * per_table);
    double* sorted_tables = (double*)malloc(sizeof(double) * total);
    double* pooled = (double*)malloc(sizeof(double) * total);
    double* b = (double*)malloc(sizeof(double) * M);
    /* sorted entries of each table m */
    for (int m = 0; m < M; ++m) {
        for (int64_t q = 0; q < nq; ++q)
            for (int k = 0; k < K; ++k) col[q * K + k] = D[(q * M + m) * K + k];
        qsort(col, per_table, sizeof(double), cmp_double);
        memcpy(sorted_tables + m * per_table, col, sizeof(double) * per_table);
    }
    double best_mse = INFINITY, best_a = 1.0, best_alpha = 0.0;
    double* best_b = (double*)malloc(sizeof(double) * M);
    for (int g = 0; g < 8; ++g) {
        double alpha = ALPHA_GRID[g];
        for (int m = 0; m < M; ++m) b[m] = nearest_rank(sorted_tables + m * per_table, per_table, alpha);
        int64_t p = 0;
        for (int64_t q = 0; q < nq; ++q)
            for (int m = 0; m < M; ++m)
                for (int k = 0; k < K; ++k) pooled[p++] = D[(q * M + m) * K + k] - b[m];
        qsort(pooled, total, sizeof(double), cmp_double);
        double hi = nearest_rank(pooled, total, 1.0 - alpha);
        double a = hi > 0.0 ? 255.0 / hi : 1.0;
        double sse = 0.0;
        for (int64_t q = 0; q < nq; ++q)
            for (int m = 0; m < M; ++m)
                for (int k = 0; k < K; ++k) {
                    double y = D[(q * M + m) * K + k];
                    double f = floor(a * (y - b[m]));
                    if (f < 0.0) f = 0.0;
                    if (f > 255.0) f = 255.0;
                    double yhat = f / a + b[m];
                    double e = yhat - y;
                    sse = sse + e * e;
                }
        double mse = sse / (double)total;
        if (mse_out) mse_out[g] = mse;
        if (a_grid) a_grid[g] = a;
        if (b_grid) memcpy(b_grid + (int64_t)g * M, b, sizeof(double) * M);
        if (mse < best_mse) {
            best_mse = mse;
            best_a = a;
            best_alpha = alpha;
            memcpy(best_b, b, sizeof(double) * M);
        }
    }
    *a_out = best_a;
    *alpha_out = best_alpha;
    memcpy(b_out, best_b, sizeof(double) * M);
    free(col);
    free(sorted_tables);
    free(pooled);
    free(b);
    free(best_b);
}

void oracle_calibrate(const double* D, int64_t nq, int M, double* a_out, double* b_out,
                      double* alpha_out, double* mse_out) {
    oracle_calibrate_grid(D, nq, M, a_out, b_out, alpha_out, mse_out, NULL, NULL);
}

/* ---------------------------------------------------------------- O2 -- */
/* k-means with K=16 on the sub-vectors of one subspace,
 * R8: centroids start at the rows `init` (given by the harness), exactly
 * `iters` Lloyd iterations, assignment ties to the lowest centroid, update =
 * mean of assigned points summed in row order; an empty cluster k (in
 * ascending k) takes the point with the largest current assignment distance
 * (ties to the lowest row), skipping rows already taken this iteration.
 * C64 receives [K][L] fp64 centroids; inertia (optional) [iters] the sum of
 * assignment distances at each iteration's assignment step. */
void oracle_kmeans_subspace(const float* train, int64_t n, int J, int col0, int L,
                            const int64_t* init, int iters, double* C64, double* inertia) {
    int* assign = (int*)malloc(sizeof(int) * n);
    double* dist = (double*)malloc(sizeof(double) * n);
    double* sums = (double*)malloc(sizeof(double) * K * L);
    int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * K);
    unsigned char* taken = (unsigned char*)malloc(n);
    for (int k = 0; k < K; ++k)
        for (int j = 0; j < L; ++j) C64[k * L + j] = (double)train[init[k] * (int64_t)J + col0 + j];
    for (int it = 0; it < iters; ++it) {
        double tot = 0.0;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            double best = INFINITY;
            int arg = 0;
            for (int k = 0; k < K; ++k) {
                double d = subspace_l2_f64c(train + i * (int64_t)J + col0, C64 + k * L, L);
                if (d < best) {
                    best = d;
                    arg = k;
                }
            }
            assign[i] = arg;
            dist[i] = best;
        }
        for (int64_t i = 0; i < n; ++i) tot = tot + dist[i];
        if (inertia) inertia[it] = tot;
        memset(sums, 0, sizeof(double) * K * L);
        memset(counts, 0, sizeof(int64_t) * K);
        for (int64_t i = 0; i < n; ++i) {
            int k = assign[i];
            counts[k] += 1;
            for (int j = 0; j < L; ++j) sums[k * L + j] = sums[k * L + j] + (double)train[i * (int64_t)J + col0 + j];
        }
        memset(taken, 0, n);
        for (int k = 0; k < K; ++k) {
            if (counts[k] > 0) {
                for (int j = 0; j < L; ++j) C64[k * L + j] = sums[k * L + j] / (double)counts[k];
            } else {
                int64_t far = -1;
                double fd = -1.0;
                for (int64_t i = 0; i < n; ++i)
                    if (!taken[i] && dist[i] > fd) {
                        fd = dist[i];
                        far = i;
                    }
                if (far >= 0) {
                    taken[far] = 1;
                    for (int j = 0; j < L; ++j) C64[k * L + j] = (double)train[far * (int64_t)J + col0 + j];
                }
            }
        }
    }
    free(assign);
    free(dist);
    free(sums);
    free(counts);
    free(taken);
}

/* ---------------------------------------------------------------- O7 -- */
/* running total sum_m D'[i_m][m] with the 8-bit tables,
 * as an exact integer (R11); out[i*nq + q] (row = database vector). */
void oracle_scan(const uint8_t* codes, int64_t n, int M, const uint8_t* qluts, int64_t nq,
                 uint16_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t q = 0; q < nq; ++q) {
            int64_t acc = 0;
            for (int m = 0; m < M; ++m) acc += qluts[(q * M + m) * K + codes[i * M + m]];
            out[i * nq + q] = (uint16_t)acc; /* acc <= 255*M <= 16320 for M <= 64 */
        }
}

/* ---------------------------------------------------------------- O8 -- */
/* key of one (query, vector) pair (R13): smaller key = better; squared L2
 * ranks ascending acc, dot ranks descending acc; ties by lower global index. */
static uint64_t make_key(int64_t acc, int64_t gidx, int metric) {
    uint64_t v = metric == ORACLE_L2SQ ? (uint64_t)acc : (uint64_t)(0xFFFF - acc);
    return (v << 48) | (uint64_t)gidx;
}

/* k smallest keys per query, ascending; padded with UINT64_MAX when k > n. */
void oracle_topk(const uint8_t* codes, int64_t n, int M, const uint8_t* qluts, int64_t nq,
                 int k, int metric, int64_t index_base, uint64_t* keys) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nq; ++q) {
        uint64_t* best = keys + q * k;
        for (int r = 0; r < k; ++r) best[r] = UINT64_MAX;
        for (int64_t i = 0; i < n; ++i) {
            int64_t acc = 0;
            for (int m = 0; m < M; ++m) acc += qluts[(q * M + m) * K + codes[i * M + m]];
            uint64_t key = make_key(acc, index_base + i, metric);
            if (key >= best[k - 1]) continue;
            int r = k - 1; /* insertion into the sorted list */
            while (r > 0 && best[r - 1] > key) {
                best[r] = best[r - 1];
                --r;
            }
            best[r] = key;
        }
    }
}

/* --------------------------------------------------------------- O13 -- */
/* "Bolt No Quantize": the scan with the unquantized
 * tables, out[i*nq + q] = sum_m D[q][m][i_m] with D the fp32 tables.  R18:
 * summed in fp32, in ascending m from 0.0f -- the paper fixes no precision for
 * this variant, so the oracle takes the kernel's, and a top-k decided by these
 * sums is then exact (the near-tie rule of the parity contract). */
void oracle_scan_f32(const uint8_t* codes, int64_t n, int M, const float* luts, int64_t nq, float* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t q = 0; q < nq; ++q) {
            float acc = 0.0f;
            for (int m = 0; m < M; ++m) acc = acc + luts[(q * M + m) * K + codes[i * M + m]];
            out[i * nq + q] = acc;
        }
}

/* O14: key of an fp32 distance (R18): the float's bits mapped to an unsigned
 * order-preserving code (negative: all bits flipped; else the sign bit set),
 * inverted for the dot product (larger is better), in the high 32 bits; the
 * global index (< 2^32) in the low 32: ties by lower index. */
static uint64_t make_key_f32(float v, int64_t gidx, int metric) {
    uint32_t u;
    memcpy(&u, &v, sizeof u);
    uint32_t ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    if (metric != ORACLE_L2SQ) ord = ~ord;
    return ((uint64_t)ord << 32) | (uint64_t)gidx;
}

/* k smallest fp32 keys per query, ascending; UINT64_MAX padding when k > n. */
void oracle_topk_f32(const uint8_t* codes, int64_t n, int M, const float* luts, int64_t nq, int k, int metric,
                     int64_t index_base, uint64_t* keys) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nq; ++q) {
        uint64_t* best = keys + q * k;
        for (int r = 0; r < k; ++r) best[r] = UINT64_MAX;
        for (int64_t i = 0; i < n; ++i) {
            float acc = 0.0f;
            for (int m = 0; m < M; ++m) acc = acc + luts[(q * M + m) * K + codes[i * M + m]];
            uint64_t key = make_key_f32(acc, index_base + i, metric);
            if (key >= best[k - 1]) continue;
            int r = k - 1;
            while (r > 0 && best[r - 1] > key) {
                best[r] = best[r - 1];
                --r;
            }
            best[r] = key;
        }
    }
}

/* ---------------------------------------------------------------- O9 -- */
static int cmp_u64(const void* pa, const void* pb) {
    uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    return (a > b) - (a < b);
}

/* union of W shard lists [W][nq][k] -> the k smallest keys per query */
void oracle_merge(const uint64_t* shard_keys, int W, int64_t nq, int k, uint64_t* out) {
#pragma omp parallel
    {
        uint64_t* buf = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)W * k);
#pragma omp for schedule(static)
        for (int64_t q = 0; q < nq; ++q) {
            for (int w = 0; w < W; ++w)
                memcpy(buf + (size_t)w * k, shard_keys + ((int64_t)w * nq + q) * k, sizeof(uint64_t) * k);
            qsort(buf, (size_t)W * k, sizeof(uint64_t), cmp_u64);
            memcpy(out + q * k, buf, sizeof(uint64_t) * k);
        }
        free(buf);
    }
}

/* --------------------------------------------------------------- O10 -- */
/* yhat sum: each entry reconstructs as beta/a + b_m, so the total is
 * acc/a + sum_m b_m -- the single overall bias "corrected for" (R7). */
void oracle_dequant(const uint16_t* acc, int64_t count, float a32, const float* b32, int M,
                    double* out) {
    double bsum = 0.0;
    for (int m = 0; m < M; ++m) bsum = bsum + (double)b32[m];
    const double a = (double)a32;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < count; ++e) out[e] = (double)acc[e] / a + bsum;
}

/* --------------------------------------------------------------- O12 -- */
/* Layout v1 (R12): u32 word g*M + m holds codebook m of rows 8g..8g+7, row
 * 8g+r in bits [4r, 4r+4).  Used only to read the CUDA path's output. */
void oracle_unpack_v1(const uint32_t* words, int64_t n, int M, uint8_t* flat) {
    for (int64_t i = 0; i < n; ++i)
        for (int m = 0; m < M; ++m) {
            uint32_t w = words[(i / 8) * M + m];
            flat[i * M + m] = (uint8_t)((w >> (4 * (i % 8))) & 0xFu);
        }
}
