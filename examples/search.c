/* search.c -- the Bolt hot path through the C ABI alone (no Python, no
 * torch): fit (GPU k-means + LUT quantizer), encode a database, build the
 * quantized query tables, top-k search, split the keys.
 *
 *   make -C examples          (needs paper_1706_10283_b200/libbolt.so)
 *   ./examples/search [n] [nq]
 *
 * Synthetic data: uniform integers in [0, 256) (a stand-in; see DESIGN.md for
 * the benchmark recipes).  Prints the first query's 5 best rows and the time
 * of the search calls. */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "bolt.h"

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)
#define BK(x)                                                                              \
    do {                                                                                   \
        if ((x) != BOLT_OK) {                                                              \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, bolt_last_error());          \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

static uint64_t rng = 0x9E3779B97F4A7C15ull;
static float next_value(void) {  /* xorshift64*: a fixed synthetic stream */
    rng ^= rng >> 12; rng ^= rng << 25; rng ^= rng >> 27;
    return (float)((rng * 0x2545F4914F6CDD1Dull) >> 56);
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 1000000, nq = argc > 2 ? atoll(argv[2]) : 1000;
    const int j = 128, m = 16, k = 10;
    const int64_t ntrain = 20000 < n ? 20000 : n;
    printf("%s: n=%lld nq=%lld j=%d m=%d k=%d\n", bolt_version(), (long long)n, (long long)nq, j, m, k);

    float* hX = (float*)malloc(sizeof(float) * n * j);
    float* hQ = (float*)malloc(sizeof(float) * nq * j);
    int64_t* hinit = (int64_t*)malloc(sizeof(int64_t) * m * 16);
    for (int64_t i = 0; i < n * j; ++i) hX[i] = next_value();
    for (int64_t i = 0; i < nq * j; ++i) hQ[i] = next_value();
    for (int i = 0; i < m * 16; ++i) hinit[i] = (i % 16) * (ntrain / 16);  /* distinct seed rows */

    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    float *X, *Q, *C, *b, *a;
    double *Dcal, *amse;
    int64_t* init;
    uint32_t* codes;
    uint8_t* ql;
    uint64_t* keys;
    CK(cudaMalloc((void**)&X, sizeof(float) * n * j));
    CK(cudaMalloc((void**)&Q, sizeof(float) * nq * j));
    CK(cudaMalloc((void**)&C, sizeof(float) * m * 16 * (j / m)));
    CK(cudaMalloc((void**)&b, sizeof(float) * m));
    CK(cudaMalloc((void**)&a, sizeof(float)));
    CK(cudaMalloc((void**)&amse, sizeof(double) * 9));
    CK(cudaMalloc((void**)&init, sizeof(int64_t) * m * 16));
    CK(cudaMalloc((void**)&codes, sizeof(uint32_t) * bolt_codes_words(n, m)));
    CK(cudaMalloc((void**)&ql, (size_t)nq * m * 16));
    CK(cudaMalloc((void**)&keys, sizeof(uint64_t) * nq * k));
    CK(cudaMemcpy(X, hX, sizeof(float) * n * j, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(Q, hQ, sizeof(float) * nq * j, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(init, hinit, sizeof(int64_t) * m * 16, cudaMemcpyHostToDevice));

    /* offline fit: k-means on the first rows, quantizer from 200 of them as queries */
    size_t wk = bolt_kmeans_workspace_bytes(ntrain, j, m);
    void* ws;
    CK(cudaMalloc(&ws, wk > 0 ? wk : 8));
    BK(bolt_kmeans(X, ntrain, j, j, m, init, 16, C, ws, wk, s));
    CK(cudaFree(ws));
    const int64_t ncal = 200;
    CK(cudaMalloc((void**)&Dcal, sizeof(double) * ncal * m * 16));
    BK(bolt_build_luts_f64(X, ncal, j, j, C, m, BOLT_L2SQ, Dcal, s));
    size_t wc = bolt_calibrate_workspace_bytes(ncal, m);
    CK(cudaMalloc(&ws, wc > 0 ? wc : 8));
    BK(bolt_calibrate(Dcal, ncal, m, a, b, amse, ws, wc, s));
    CK(cudaFree(ws));
    float ha;
    CK(cudaMemcpyAsync(&ha, a, sizeof(float), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));

    /* the hot path: encode, tables, top-k */
    size_t wt = bolt_topk_workspace_bytes(n, m, nq, k);
    CK(cudaMalloc(&ws, wt > 0 ? wt : 8));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int rep = 0; rep < 2; ++rep) {  /* the first pass loads the kernels; time the second */
        CK(cudaEventRecord(e0, s));
        BK(bolt_encode(X, n, j, j, C, m, codes, s));
        BK(bolt_build_quantized_luts(Q, nq, j, j, C, m, BOLT_L2SQ, ha, b, ql, NULL, s));
        BK(bolt_topk(codes, n, m, ql, nq, k, BOLT_L2SQ, 0, keys, ws, wt, s));
        CK(cudaEventRecord(e1, s));
    }
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));

    uint16_t* vals;
    int64_t* idx;
    CK(cudaMalloc((void**)&vals, sizeof(uint16_t) * nq * k));
    CK(cudaMalloc((void**)&idx, sizeof(int64_t) * nq * k));
    BK(bolt_keys_split(keys, nq * k, BOLT_L2SQ, vals, idx, s));
    uint16_t hv[10];
    int64_t hi[10];
    CK(cudaMemcpyAsync(hv, vals, sizeof(hv), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hi, idx, sizeof(hi), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    printf("encode + tables + top-%d: %.3f ms (%.1f Gdist/s)\n", k, ms, (double)n * nq / (ms * 1e-3) / 1e9);
    printf("query 0:");
    for (int r = 0; r < 5; ++r) printf("  row %lld (%u)", (long long)hi[r], hv[r]);
    printf("\n");
    return 0;
}
