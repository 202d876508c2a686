// probe_ffma2.cu -- issue cost of FFMA2 / FADD2 (packed fp32x2) vs FFMA on sm_100a.
#include <cstdio>
template <int OP>
__global__ void k(float* out, long long* cyc, int iters) {
    float2 x[8];
    for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    const float2 y = make_float2(0.999f, 1.001f);
    float s[16];
    for (int i = 0; i < 16; ++i) s[i] = threadIdx.x * 1e-3f + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (OP == 0) x[i] = __ffma2_rn(x[i], y, x[i]);
                if (OP == 1) x[i] = __fadd2_rn(x[i], y);
                if (OP == 2) { s[2 * i] = fmaf(s[2 * i], 0.999f, s[2 * i]); s[2 * i + 1] = fmaf(s[2 * i + 1], 1.001f, s[2 * i + 1]); }
            }
    }
    __syncthreads();
    long long t1 = clock64();
    float a = 0;
    for (int i = 0; i < 8; ++i) a += x[i].x + x[i].y + s[2 * i] + s[2 * i + 1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP>
void run(const char* nm, float* out, long long* cyc) {
    const int iters = 256, wps = 4;
    k<OP><<<148, 128 * wps>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double n = (double)iters * 16 * 8 * wps;  // packed ops (or scalar pairs) per SMSP
    printf("%-8s %.2f cycles per (warp, 2 fp32 ops) per SMSP\n", nm, h / n);
}
int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
    run<0>("ffma2", out, cyc); run<1>("fadd2", out, cyc); run<2>("2xffma", out, cyc);
}
