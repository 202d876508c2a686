// lut.cu -- g(q): query lookup tables and their 8-bit
// quantization (L262, L277-291).
//
// One thread per table entry (q, c, i).  The entry is accumulated in fp64
// from direct differences in ascending dimension order with explicitly
// rounded operations (no FMA contraction): for squared L2
//   y = sum_d (q_d - c_d)^2,  for dot  y = sum_d q_d * c_d,
// then quantized from the fp64 value (R1):
//   beta = clamp(floor(a * (y - b_c)), 0, 255).
// The work is Q*16*J multiply-adds -- negligible next to the scan (P:L396:
// "unlikely to be a bottleneck") -- so fp64 is used to keep the quantized
// tables exact away from rounding boundaries.
#include "common.cuh"

#ifndef BOLT_LUT_QC
#define BOLT_LUT_QC 1  // 0: one thread per entry (A/B builds)
#endif

namespace bolt {
namespace {

__device__ __forceinline__ uint8_t quantize_one(double y, double a, double b) {
    double t = __dmul_rn(a, __dsub_rn(y, b));
    double f = floor(t);
    f = f < 0.0 ? 0.0 : f;
    f = f > 255.0 ? 255.0 : f;
    return (uint8_t)f;
}

__global__ void build_luts_kernel(const float* __restrict__ Q, int64_t nq, int j, int64_t ldq,
                                  const float* __restrict__ C, int m, int metric, double a,
                                  const float* __restrict__ b, uint8_t* __restrict__ qluts,
                                  float* __restrict__ luts32, double* __restrict__ luts64) {
    const int64_t total = nq * m * kK;
    const int L = j / m;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = e / (m * kK);
        const int r = (int)(e - q * m * kK);
        const int c = r / kK;
        const int i = r - c * kK;
        const float* qv = Q + q * ldq + (int64_t)c * L;
        const float* cv = C + ((int64_t)c * kK + i) * L;
        double y = 0.0;
        if (metric == BOLT_L2SQ) {
            for (int d = 0; d < L; ++d) {
                double diff = __dsub_rn((double)__ldg(qv + d), (double)__ldg(cv + d));
                y = __dadd_rn(y, __dmul_rn(diff, diff));
            }
        } else {
            for (int d = 0; d < L; ++d)
                y = __dadd_rn(y, __dmul_rn((double)__ldg(qv + d), (double)__ldg(cv + d)));
        }
        if (luts64) luts64[e] = y;
        if (luts32) luts32[e] = (float)y;
        if (qluts) qluts[e] = quantize_one(y, a, (double)__ldg(b + c));
    }
}

// One thread per (query, codebook), the 16 entries of its table in
// registers: lane = query (32 consecutive queries per warp), warp-uniform
// codebook, so the centroid loads are broadcasts; the same fp64 operations
// in the same order as build_luts_kernel (bit-identical), the 16 quantized
// entries written as one 16-byte store.
template <int L>
__global__ void __launch_bounds__(256)
build_luts_qc_kernel(const float* __restrict__ Q, int64_t nq, int64_t ldq, const float* __restrict__ C, int m,
                     int metric, double a, const float* __restrict__ b, uint8_t* __restrict__ qluts,
                     float* __restrict__ luts32, double* __restrict__ luts64) {
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // global warp
    const int lane = threadIdx.x & 31;
    const int c = (int)(wg % m);
    const int64_t q = (wg / m) * 32 + lane;
    if (q >= nq) return;
    double x[L];
    const float* qv = Q + q * ldq + (int64_t)c * L;
#pragma unroll
    for (int d = 0; d < L; ++d) x[d] = (double)__ldg(qv + d);
    const double bc = qluts ? (double)__ldg(b + c) : 0.0;  // b is only given for quantized tables
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < kK; ++i) {
        const float* cv = C + ((int64_t)c * kK + i) * L;
        double y = 0.0;
        if (metric == BOLT_L2SQ) {
#pragma unroll
            for (int d = 0; d < L; ++d) {
                const double diff = __dsub_rn(x[d], (double)__ldg(cv + d));
                y = __dadd_rn(y, __dmul_rn(diff, diff));
            }
        } else {
#pragma unroll
            for (int d = 0; d < L; ++d) y = __dadd_rn(y, __dmul_rn(x[d], (double)__ldg(cv + d)));
        }
        const int64_t e = (q * m + c) * kK + i;
        if (luts64) luts64[e] = y;
        if (luts32) luts32[e] = (float)y;
        w[i >> 2] |= (uint32_t)quantize_one(y, a, bc) << (8 * (i & 3));
    }
    if (qluts) *reinterpret_cast<uint4*>(qluts + (q * m + c) * kK) = make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void quantize_kernel(const float* __restrict__ luts, int64_t nq, int m, double a,
                                const float* __restrict__ b, uint8_t* __restrict__ qluts) {
    const int64_t total = nq * m * kK;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)((e / kK) % m);
        qluts[e] = quantize_one((double)luts[e], a, (double)__ldg(b + c));
    }
}

unsigned grid_for(int64_t total, int threads) {
    int64_t blocks = ceil_div(total, threads);
    return (unsigned)(blocks < 148 * 32 ? blocks : 148 * 32);
}

}  // namespace

cudaError_t launch_build_luts(const float* Q, int64_t nq, int j, int64_t ldq, const float* C, int m,
                              int metric, float a, const float* b, uint8_t* qluts, float* luts32,
                              double* luts64, cudaStream_t s) {
    const int64_t total = nq * m * kK;
    if (total == 0) return cudaSuccess;
    const int L = j / m;
    const bool q16 = qluts == nullptr || (reinterpret_cast<uintptr_t>(qluts) & 15) == 0;
    if (BOLT_LUT_QC && q16 && (L == 4 || L == 8 || L == 16)) {
        const int64_t threads = ceil_div(nq, (int64_t)32) * 32 * m;  // warps of 32 queries x codebooks
        const unsigned blocks = (unsigned)ceil_div(threads, (int64_t)256);
        auto kern = L == 4 ? build_luts_qc_kernel<4> : L == 8 ? build_luts_qc_kernel<8> : build_luts_qc_kernel<16>;
        kern<<<blocks, 256, 0, s>>>(Q, nq, ldq, C, m, metric, (double)a, b, qluts, luts32, luts64);
        return cudaGetLastError();
    }
    build_luts_kernel<<<grid_for(total, 256), 256, 0, s>>>(Q, nq, j, ldq, C, m, metric, (double)a, b,
                                                         qluts, luts32, luts64);
    return cudaGetLastError();
}

cudaError_t launch_quantize(const float* luts, int64_t nq, int m, float a, const float* b,
                            uint8_t* qluts, cudaStream_t s) {
    const int64_t total = nq * m * kK;
    if (total == 0) return cudaSuccess;
    quantize_kernel<<<grid_for(total, 256), 256, 0, s>>>(luts, nq, m, (double)a, b, qluts);
    return cudaGetLastError();
}

}  // namespace bolt
