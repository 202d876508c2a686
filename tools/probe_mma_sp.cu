// Probe: issue rate of tcgen05.mma.kind::i8, dense vs 2:4
// sparse (.sp, A = the sparse operand: one-hot codes compressed to K/2 with
// metadata in TMEM), for one CTA (cta_group::1, M = 128) and a CTA pair
// (cta_group::2, M = 256), N = 256, operands in shared memory (K-major,
// SWIZZLE_NONE, contents irrelevant: the probe times the tensor pipe).
//
// Each CTA (pair) issues TILES tiles of K = 256 bytes (dense: 8 instructions of
// K = 32; sparse: 4 of K = 64) into one TMEM accumulator back to back, commits
// once and waits; cycles / instruction and logical int8 ops / s are printed
// for one CTA (pair) alone and for a full grid (all SMs).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probe_mma_sp_bin tools/probe_mma_sp.cu
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int TILES = 512;
constexpr int KBYTES = 256;  // logical K per tile (M = 16 codebooks x 16)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <bool PAIR, bool SPARSE>
__global__ void __launch_bounds__(128, 1) probe(unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int MR = 128;                 // A rows per CTA
    constexpr int NB = PAIR ? 128 : 256;    // B rows per CTA (pair: each CTA holds half of N)
    constexpr int A_BYTES = MR * (SPARSE ? KBYTES / 2 : KBYTES);
    constexpr int B_BYTES = NB * KBYTES;
    uint8_t* sA = smem;
    uint8_t* sB = smem + A_BYTES;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + A_BYTES + B_BYTES);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t rank = 0;
    if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < (A_BYTES + B_BYTES) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *slot;
    // sparse metadata (columns 256..511): every 4-bit group = indices (0, 1), valid for any layout
    if (SPARSE) {
        const uint32_t t = tmem + ((uint32_t)(warp * 32) << 16) + 256;
        const uint32_t v = 0x44444444u;
        for (int c = 0; c < 256; c += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(t + c),
                         "r"(v));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // instruction descriptor: D s32, A/B u8, K-major, N = 256, M = 128 / 256, bit 2 = sparse
    const uint32_t idesc = (2u << 4) | ((256u >> 3) << 17) | ((uint32_t)((PAIR ? 256 : 128) >> 4) << 24) |
                           (SPARSE ? 4u : 0u);
    constexpr int KSTEP = SPARSE ? 64 : 32;       // logical K per instruction
    constexpr int NSTEP = KBYTES / KSTEP;
    constexpr int ACH = 2;                        // 16-byte A chunks per instruction (K/2 compressed for sparse)
    constexpr int BCH = KSTEP / 16;               // 16-byte B chunks per instruction
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        const long long t0 = clock64();
        for (int t = 0; t < TILES; ++t) {
#pragma unroll
            for (int ks = 0; ks < NSTEP; ++ks) {
                const uint64_t ad = desc(a0 + ks * ACH * MR * 16, MR * 16, 128);
                const uint64_t bd = desc(b0 + ks * BCH * NB * 16, NB * 16, 128);
                const uint32_t acc = ks > 0 ? 1u : 0u;
                if (SPARSE) {
                    const uint32_t e = tmem + 256 + ks * 8;
                    if (PAIR)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(tmem),
                                     "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(e));
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(tmem),
                                     "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(e));
                } else {
                    if (PAIR)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad),
                                     "l"(bd), "r"(idesc), "r"(acc));
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad),
                                     "l"(bd), "r"(idesc), "r"(acc));
                }
            }
        }
        if (PAIR)
            asm volatile("{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
                         "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}"
                         ::"r"(smem_u32(bar)));
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
        asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(
            smem_u32(bar)));
        cycles[blockIdx.x / (PAIR ? 2 : 1)] = clock64() - t0;
    } else if (PAIR && rank == 1 && threadIdx.x == 0) {
        asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(
            smem_u32(bar)));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
    else __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <bool PAIR, bool SPARSE>
void run(const char* name, int ctas, int clock_mhz) {
    constexpr int MR = 128, NB = PAIR ? 128 : 256;
    const int smem = MR * (SPARSE ? KBYTES / 2 : KBYTES) + NB * KBYTES + 64;
    auto k = probe<PAIR, SPARSE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* d;
    const int units = PAIR ? ctas / 2 : ctas;
    cudaMalloc(&d, units * sizeof(unsigned long long));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = PAIR ? 1 : 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, k, d);  // warm-up
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(units);
    cudaMemcpy(h.data(), d, units * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto c : h) mean += (double)c;
    mean /= units;
    const int nstep = KBYTES / (SPARSE ? 64 : 32);
    const double instr = (double)TILES * nstep;
    const double ops = 2.0 * (PAIR ? 256 : 128) * 256 * KBYTES * (double)TILES * units;  // logical int8 ops
    printf("%-34s ctas=%3d  %s  cycles/instr=%7.1f  cycles/tile(K=256)=%7.1f  kernel %.3f ms  %.0f TOP/s logical "
           "(at %d MHz from cycles: %.0f TOP/s)\n",
           name, ctas, cudaGetErrorString(err), mean / instr, mean / TILES, ms, ops / (ms * 1e-3) / 1e12, clock_mhz,
           ops / (mean / (clock_mhz * 1e6)) / 1e12);
    cudaFree(d);
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    clk /= 1000;
    printf("SMs %d, clock %d MHz; tile = M x 256 x K=256 (M = 128 per CTA, 256 per pair)\n", sms, clk);
    run<false, false>("dense  i8 cta_group::1 M=128", 1, clk);
    run<false, true>("sparse i8 cta_group::1 M=128", 1, clk);
    run<true, false>("dense  i8 cta_group::2 M=256", 2, clk);
    run<true, true>("sparse i8 cta_group::2 M=256", 2, clk);
    run<false, false>("dense  i8 cta_group::1 M=128", sms, clk);
    run<false, true>("sparse i8 cta_group::1 M=128", sms, clk);
    run<true, false>("dense  i8 cta_group::2 M=256", sms, clk);
    run<true, true>("sparse i8 cta_group::2 M=256", sms, clk);
    return 0;
}
