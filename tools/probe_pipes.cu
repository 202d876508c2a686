// probe_pipes.cu -- issue throughput of the integer instructions the scan
// epilogues use (u16x2 min/max, 3-input u16x2 min, IADD3, LOP3, PRMT, IMAD),
// measured with clock64 over 8 independent chains per thread, 1..4 warps per
// SMSP.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_pipes tools/probe_pipes.cu
#include <cstdio>
#include <cstdint>

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    if (OP == 0) asm volatile("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 1) d = __vimin3_u16x2(a, b, c);
    if (OP == 2) asm volatile("add.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 3) asm volatile("lop3.b32 %0, %1, %2, %3, 0xFE;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    if (OP == 4) asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    if (OP == 5) asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    if (OP == 6) asm volatile("min.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    if (OP == 7) d = __vimax3_u16x2(a, b, c);
    return d;
}

template <int OP>
__global__ void k(uint32_t* out, long long* cyc, int iters) {
    uint32_t x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i;
    const uint32_t b = 0x12345678u ^ blockIdx.x, c = 0x0F0F0F0Fu;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = op<OP>(x[i], b + r, c);
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, uint32_t* out, long long* cyc) {
    const int iters = 256;
    for (int wps = 1; wps <= 4; wps *= 2) {
        int threads = 128 * wps;
        k<OP><<<148, threads>>>(out, cyc, iters);
        cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double instr_per_smsp = (double)iters * 16 * 8 * wps;  // warp-instructions per SMSP
        printf("%-12s warps/SMSP=%d  cycles/warp-instr/SMSP = %.2f\n", name, wps, (double)h[0] / instr_per_smsp);
    }
}

int main() {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&cyc, 148 * 8);
    run<0>("min.u16x2", out, cyc);
    run<1>("vimin3.u16x2", out, cyc);
    run<7>("vimax3.u16x2", out, cyc);
    run<2>("add.u32", out, cyc);
    run<3>("lop3", out, cyc);
    run<4>("prmt", out, cyc);
    run<5>("mad.lo.u32", out, cyc);
    run<6>("min.u32", out, cyc);
    return 0;
}
