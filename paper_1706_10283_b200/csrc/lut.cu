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
