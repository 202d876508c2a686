// Probe: operand layout of tcgen05.mma.sp.kind::i8 (2:4 sparse A).
// One CTA, cta_group::1, M = 128, N = 64, K = 64 (one instruction).
// B = identity (B[n][k] = 1 iff k == n), so D[m][n] = A_logical[m][n]: the
// decompressed sparse row.  Compressed A (K/2 = 32 bytes per row, K-major,
// SWIZZLE_NONE: 16-byte chunk j of row r at j*(128*16) + (r/8)*128 + (r%8)*16)
// holds comp[m][e] = 1 + ((m * 7 + e) % 100); metadata (TMEM columns meta0,
// meta0 + 1 of lane m) is set per test:
//   test 0: every nibble 0x4 (indices 0, 1)
//   test 1: row m: nibble (m % 16) of the 64-bit pair = 0xE (indices 2, 3), others 0x4
//   test 2: row m: nibble (m % 16) = 0x9 (indices 1, 2), others 0x4
// Prints D for a few rows so the metadata-bit -> (row, K group) map can be read off.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probe_sp_layout_bin tools/probe_sp_layout.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

constexpr int MR = 128, NN = 64, KL = 64;

__global__ void probe(int test, int id2, int meta_col_off, int32_t* out) {
    __shared__ __align__(1024) uint8_t sA[MR * KL / 2];
    __shared__ __align__(1024) uint8_t sB[NN * KL];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = threadIdx.x;  // one thread per A row / TMEM lane
    // compressed A row m: 32 bytes = chunks 0, 1
    for (int e = 0; e < KL / 2; ++e) {
        const int j = e / 16, b = e % 16;
        sA[j * (MR * 16) + (m / 8) * 128 + (m % 8) * 16 + b] = (uint8_t)(1 + ((m * 7 + e) % 100));
    }
    // B identity: row n (< 64), K byte k: 4 chunks
    if (m < NN)
        for (int k = 0; k < KL; ++k) {
            const int j = k / 16, b = k % 16;
            sB[j * (NN * 16) + (m / 8) * 128 + (m % 8) * 16 + b] = (uint8_t)(k == m ? 1 : 0);
        }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    const uint32_t meta = tmem + 128 + meta_col_off;  // columns 128.. hold the metadata
    {
        uint32_t w[4] = {0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u};
        if (test == 1 || test == 2) {
            const int nib = m % 16;
            const uint32_t pat = test == 1 ? 0xEu : 0x9u;
            w[nib / 8] = (w[nib / 8] & ~(0xFu << (4 * (nib % 8)))) | (pat << (4 * (nib % 8)));
        }
        if (test == 3) {  // row m: nibble (m % 32) over 4 columns = 0xE
            const int nib = m % 32;
            w[nib / 8] = (w[nib / 8] & ~(0xFu << (4 * (nib % 8)))) | (0xEu << (4 * (nib % 8)));
        }
        const uint32_t t = meta + ((uint32_t)(warp * 32) << 16);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(t), "r"(w[0]), "r"(w[1]),
                     "r"(w[2]), "r"(w[3]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(MR >> 4) << 24) | 4u |
                               (uint32_t)(id2 & 3);
        const uint64_t ad = desc(smem_u32(sA), MR * 16, 128);
        const uint64_t bd = desc(smem_u32(sB), NN * 16, 128);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%4], %3, p;\n\t}" ::"r"(tmem), "l"(ad),
                     "l"(bd), "r"(idesc), "r"(meta));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(
        smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    // D row m = lane m: 64 columns
    for (int c = 0; c < NN; c += 8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int i = 0; i < 8; ++i) out[m * NN + c + i] = (int32_t)r[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main(int argc, char** argv) {
    int32_t* d;
    cudaMalloc(&d, MR * NN * 4);
    static int32_t h[MR * NN];
    const int rows[] = {0, 1, 2, 3, 5, 8, 15, 16, 17, 31, 32, 33, 64, 127};
    for (int test = 0; test < 4; ++test)
        for (int id2 = 0; id2 < 1; ++id2) {
            cudaMemset(d, 0xEE, MR * NN * 4);
            probe<<<1, 128>>>(test, id2, 0, d);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            printf("=== test %d id2 %d: %s\n", test, id2, cudaGetErrorString(e));
            if (e != cudaSuccess) return 1;
            for (int r : rows) {
                printf("row %3d comp[0..7]=", r);
                for (int k = 0; k < 8; ++k) printf("%d,", 1 + ((r * 7 + k) % 100));
                printf(" D:");
                for (int n = 0; n < NN; ++n) printf(" %d", h[r * NN + n]);
                printf("\n");
            }
        }
    return 0;
}
