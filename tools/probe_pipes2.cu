// probe_pipes2.cu -- which pipe an instruction issues on: throughput of X alone
// and of X interleaved 1:1 with LOP3 (alu).  If X is on the fma pipe the mix
// runs at ~1 cycle/instr/SMSP, if on alu at ~2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_pipes2_bin tools/probe_pipes2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b) {
    uint32_t d;
    if (OP == 0) asm volatile("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 1) asm volatile("fma.rn.f16x2 %0, %1, %2, %1;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 2) asm volatile("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 3) asm volatile("mad.lo.u32 %0, %1, 3, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 4) asm volatile("add.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 5) asm volatile("min.f32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 6) asm volatile("shl.b32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 7) asm volatile("add.rn.f32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 8) asm volatile("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 9) asm volatile("prmt.b32 %0, %1, %2, 0x3210;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 10) asm volatile("add.u32 %0, %1, 1234;" : "=r"(d) : "r"(a));
    if (OP == 11) asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 12) asm volatile("mad.lo.u32 %0, %1, 8, -96;" : "=r"(d) : "r"(a));
    if (OP == 13) asm volatile("shl.b32 %0, %1, 3;" : "=r"(d) : "r"(a));
    if (OP == 14) asm volatile("fma.rn.f32 %0, %1, %2, %1;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 15) {
        float2 x = make_float2(__uint_as_float(a), __uint_as_float(a ^ 1));
        float2 y = make_float2(__uint_as_float(b), __uint_as_float(b));
        float2 z = __ffma2_rn(x, y, x);
        d = __float_as_uint(z.x) ^ __float_as_uint(z.y);
    }
    if (OP == 16) {
        float2 x = make_float2(__uint_as_float(a), __uint_as_float(a ^ 1));
        float2 y = make_float2(__uint_as_float(b), __uint_as_float(b));
        float2 z = __fadd2_rn(x, y);
        d = __float_as_uint(z.x) ^ __float_as_uint(z.y);
    }
    return d;
}
__device__ __forceinline__ uint32_t lop(uint32_t a, uint32_t b) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

template <int OP, bool MIX>
__global__ void k(uint32_t* out, long long* cyc, int iters) {
    uint32_t x[8], y[8];
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 7 + i; y[i] = x[i] * 3; }
    const uint32_t b = 0x12345678u ^ blockIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                x[i] = op<OP>(x[i], b + r);
                if (MIX) y[i] = lop(y[i], b ^ r);
            }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s ^= x[i] ^ y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, uint32_t* out, long long* cyc) {
    const int iters = 256, wps = 4, threads = 128 * wps;
    long long h[148];
    k<OP, false><<<148, threads>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double n = (double)iters * 16 * 8 * wps;
    double alone = h[0] / n;
    k<OP, true><<<148, threads>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-14s alone %.2f cyc/warp-instr/SMSP; 1:1 with LOP3 %.2f cyc per pair\n", name, alone, h[0] / n);
}

int main() {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&cyc, 148 * 8);
    run<0>("min.f16x2", out, cyc);
    run<8>("max.f16x2", out, cyc);
    run<1>("fma.f16x2", out, cyc);
    run<2>("min.u16x2", out, cyc);
    run<3>("mad.lo.u32", out, cyc);
    run<4>("add.u32", out, cyc);
    run<5>("min.f32", out, cyc);
    run<6>("shl.b32", out, cyc);
    run<7>("add.f32", out, cyc);
    run<9>("prmt", out, cyc);
    run<10>("add.u32 imm", out, cyc);
    run<11>("add.f16x2", out, cyc);
    run<12>("mad imm 8,-96", out, cyc);
    run<13>("shl imm", out, cyc);
    run<14>("fma.f32", out, cyc);
    run<15>("ffma2 (+lop)", out, cyc);
    run<16>("fadd2 (+lop)", out, cyc);
    return 0;
}
