// gen_gpu.cu -- device-side generator of BASELINE c5 rows:
// the c2 Gaussian mixture drawn from Philox4x32-10 so that a 1e8-row
// database never has to exist on the host.  Input synthesis only (no Bolt
// arithmetic); built into synth/libsynth_gpu.so, used by bench.py and the
// tests, never by the product library.
//
// Row i (global index): counter (i, block, 0, 0), key (S, 5).  Block 0's
// first word picks the component (u32 mod 1024); blocks 1..32 give 4
// uniforms each, turned into 4 normals by Box-Muller on (u + 1/2) / 2^32,
// so dims 4(b-1) .. 4(b-1)+3.  x = clip(rint(mu[c][d] + 20 z), 0, 255) as fp32.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ void philox_round(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
    const uint32_t m0 = 0xD2511F53u, m1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(m0, c[0]), lo0 = m0 * c[0];
    const uint32_t hi1 = __umulhi(m1, c[2]), lo1 = m1 * c[2];
    c[0] = hi1 ^ c[1] ^ k0;
    c[1] = lo1;
    c[2] = hi0 ^ c[3] ^ k1;
    c[3] = lo0;
}

__device__ __forceinline__ void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        philox_round(c, k0, k1);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// one thread per (row, 4-dim block)
__global__ void c5_rows_kernel(int64_t row0, int64_t n, const float* __restrict__ mu, uint32_t key0,
                               uint32_t key1, float* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * 32) return;
    const int64_t r = e >> 5;
    const int b = (int)(e & 31);
    const uint64_t gi = (uint64_t)(row0 + r);
    uint32_t c0[4] = {(uint32_t)gi, (uint32_t)(gi >> 32), 0u, 0u};
    philox4x32_10(c0, key0, key1);
    const int comp = (int)(c0[0] & 1023u);  // u32 mod 1024: exactly uniform
    uint32_t c[4] = {(uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)(b + 1), 0u};
    philox4x32_10(c, key0, key1);
    float u[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) u[t] = ((float)c[t] + 0.5f) * 2.3283064365386963e-10f;  // (u + 1/2) / 2^32
    float z[4];
    const float ra = sqrtf(-2.0f * logf(u[0])), rb = sqrtf(-2.0f * logf(u[2]));
    float sa, ca, sb, cb;
    sincospif(2.0f * u[1], &sa, &ca);
    sincospif(2.0f * u[3], &sb, &cb);
    z[0] = ra * ca; z[1] = ra * sa; z[2] = rb * cb; z[3] = rb * sb;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int d = 4 * b + t;
        float x = rintf(mu[comp * 128 + d] + 20.0f * z[t]);
        x = fminf(fmaxf(x, 0.0f), 255.0f);
        out[r * 128 + d] = x;
    }
}

}  // namespace

extern "C" __attribute__((visibility("default")))
int synth_c5_rows(int64_t row0, int64_t n, const float* mu, uint32_t key0, uint32_t key1, float* out, void* stream) {
    if (n <= 0) return 0;
    const int64_t threads = n * 32;
    c5_rows_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(row0, n, mu, key0, key1, out);
    return (int)cudaGetLastError();
}
