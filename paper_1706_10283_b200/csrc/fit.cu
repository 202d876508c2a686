// fit.cu -- the offline phase on the GPU: k-means codebooks
// (reading R8) and the LUT-quantizer learning of
// L289-291 (readings R1-R4).  Not on the timed hot path; written to be
// deterministic and to follow the same fp64 operation order as the
// definitions, so a fit is reproducible bit for bit.
//
// k-means, per iteration:
//   assign  : one thread per (row, subspace); distances to the 16 fp64
//             centroids in shared memory, sum_d ((double)x - c)^2 in ascending
//             d with explicitly rounded ops; ties -> lowest centroid.
//   sums    : one thread per (subspace, dimension) walks the rows in order and
//             adds x into the assigned centroid's running sum (a sequential
//             sum per (centroid, dimension): deterministic, row order).
//   update  : one block per subspace; mean = sum / count, or for an empty
//             cluster (ascending k) the row with the largest assignment
//             distance (ties -> lowest row), each row used once per iteration.
// calibration, per alpha of the grid {0,.001,.002,.005,.01,.02,.05,.1}:
//   b_m   = nearest-rank alpha quantile of table m's entries (block radix select)
//   a     = 255 / nearest-rank (1-alpha) quantile of the pooled y - b_m
//   mse   = mean over entries (sequential sum, entry order) of (beta/a + b_m - y)^2
// and the first alpha with the strictly smallest mse wins.
#include "common.cuh"

namespace bolt {
namespace {

constexpr int kFitThreads = 256;

struct KmWs {
    double* C64;     // [m][16][L]
    int* assign;     // [m][n]
    double* dist;    // [m][n]
    double* sums;    // [m][16][L]
    int64_t* counts; // [m][16]
};

size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

KmWs carve_km(void* ws, int64_t n, int j, int m) {
    char* p = static_cast<char*>(ws);
    KmWs w;
    w.C64 = reinterpret_cast<double*>(p); p += a256((size_t)j * kK * sizeof(double));
    w.assign = reinterpret_cast<int*>(p); p += a256((size_t)m * n * sizeof(int));
    w.dist = reinterpret_cast<double*>(p); p += a256((size_t)m * n * sizeof(double));
    w.sums = reinterpret_cast<double*>(p); p += a256((size_t)j * kK * sizeof(double));
    w.counts = reinterpret_cast<int64_t*>(p);
    return w;
}

__global__ void km_init(const float* __restrict__ X, int64_t ldx, int j, int m,
                        const int64_t* __restrict__ init, double* __restrict__ C64) {
    const int L = j / m;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < j * kK; e += gridDim.x * blockDim.x) {
        const int c = e / (kK * L);
        const int r = e - c * kK * L;
        const int k = r / L;
        const int d = r - k * L;
        C64[e] = (double)X[init[c * kK + k] * ldx + c * L + d];
    }
}

__global__ void km_assign(const float* __restrict__ X, int64_t n, int64_t ldx, int j, int m,
                          const double* __restrict__ C64, int* __restrict__ assign,
                          double* __restrict__ dist) {
    extern __shared__ double kc[];
    const int L = j / m;
    for (int e = threadIdx.x; e < j * kK; e += blockDim.x) kc[e] = C64[e];
    __syncthreads();
    const int64_t total = n * m;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e / n);
        const int64_t i = e - (int64_t)c * n;
        const float* x = X + i * ldx + c * L;
        double best = 0.0;
        int arg = 0;
        for (int k = 0; k < kK; ++k) {
            const double* cc = kc + ((size_t)c * kK + k) * L;
            double s = 0.0;
            for (int d = 0; d < L; ++d) {
                const double df = __dsub_rn((double)x[d], cc[d]);
                s = __dadd_rn(s, __dmul_rn(df, df));
            }
            if (k == 0 || s < best) {
                best = s;
                arg = k;
            }
        }
        assign[e] = arg;
        dist[e] = best;
    }
}

// one thread per (subspace c, dimension d): per-centroid running sums in smem
__global__ void km_sums(const float* __restrict__ X, int64_t n, int64_t ldx, int j, int m,
                        const int* __restrict__ assign, double* __restrict__ sums,
                        int64_t* __restrict__ counts) {
    extern __shared__ double ks[];  // [16][blockDim.x]
    const int e = blockIdx.x * blockDim.x + threadIdx.x;  // = c*L + d
    const int L = j / m;
    double* s = ks + threadIdx.x;
    for (int k = 0; k < kK; ++k) s[k * blockDim.x] = 0.0;
    if (e >= j) return;
    const int c = e / L;
    const int d = e - c * L;
    const int* as = assign + (int64_t)c * n;
    int64_t cnt[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) cnt[k] = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int k = __ldg(as + i);
        s[k * blockDim.x] = __dadd_rn(s[k * blockDim.x], (double)__ldg(X + i * ldx + e));
        if (d == 0) {
#pragma unroll
            for (int t = 0; t < kK; ++t) cnt[t] += (t == k);
        }
    }
    for (int k = 0; k < kK; ++k) sums[((int64_t)c * kK + k) * L + d] = s[k * blockDim.x];
    if (d == 0)
        for (int k = 0; k < kK; ++k) counts[c * kK + k] = cnt[k];
}

// one block per subspace
__global__ void km_update(const float* __restrict__ X, int64_t n, int64_t ldx, int j, int m,
                          const double* __restrict__ dist, const double* __restrict__ sums,
                          const int64_t* __restrict__ counts, double* __restrict__ C64) {
    __shared__ double rv[kFitThreads];
    __shared__ int64_t ri[kFitThreads];
    __shared__ int64_t taken[kK];
    __shared__ int ntaken;
    const int c = blockIdx.x;
    const int L = j / m;
    if (threadIdx.x == 0) ntaken = 0;
    __syncthreads();
    const double* dc = dist + (int64_t)c * n;
    for (int k = 0; k < kK; ++k) {
        const int64_t cnt = counts[c * kK + k];
        double* ck = C64 + ((int64_t)c * kK + k) * L;
        if (cnt > 0) {
            for (int d = threadIdx.x; d < L; d += blockDim.x)
                ck[d] = __ddiv_rn(sums[((int64_t)c * kK + k) * L + d], (double)cnt);
            continue;
        }
        // empty cluster: farthest row not yet taken (largest dist, lowest row on ties)
        double bv = -1.0;
        int64_t bi = -1;
        const int nt = ntaken;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            bool used = false;
            for (int t = 0; t < nt; ++t) used |= taken[t] == i;
            if (!used && dc[i] > bv) {
                bv = dc[i];
                bi = i;
            }
        }
        rv[threadIdx.x] = bv;
        ri[threadIdx.x] = bi;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) {
                const double ov = rv[threadIdx.x + s];
                const int64_t oi = ri[threadIdx.x + s];
                if (oi >= 0 && (ri[threadIdx.x] < 0 || ov > rv[threadIdx.x] ||
                                (ov == rv[threadIdx.x] && oi < ri[threadIdx.x]))) {
                    rv[threadIdx.x] = ov;
                    ri[threadIdx.x] = oi;
                }
            }
            __syncthreads();
        }
        const int64_t far = ri[0];
        if (far >= 0) {
            for (int d = threadIdx.x; d < L; d += blockDim.x) ck[d] = (double)X[far * ldx + c * L + d];
        }
        __syncthreads();
        if (threadIdx.x == 0 && far >= 0) taken[ntaken++] = far;
        __syncthreads();
    }
}

__global__ void km_finish(const double* __restrict__ C64, int total, float* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x)
        out[e] = (float)C64[e];
}

// ----------------------------------------------------------------- calibrate
__device__ __forceinline__ uint64_t dkey(double v) {
    const uint64_t u = (uint64_t)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(uint64_t k) {
    const uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)u);
}

// rank r (0-based) smallest of the values val(i), i < count, by block radix select
template <typename F>
__device__ double block_select(F val, int64_t count, int64_t r) {
    __shared__ unsigned hist[256];
    __shared__ uint64_t s_prefix;
    __shared__ int64_t s_r;
    uint64_t prefix = 0, mask = 0;
    if (threadIdx.x == 0) s_r = r;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int t = threadIdx.x; t < 256; t += blockDim.x) hist[t] = 0;
        __syncthreads();
        for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
            const uint64_t key = dkey(val(i));
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t rr = s_r;
            int bkt = 0;
            for (; bkt < 255; ++bkt) {
                if ((int64_t)hist[bkt] > rr) break;
                rr -= hist[bkt];
            }
            s_r = rr;
            s_prefix = prefix | ((uint64_t)bkt << shift);
        }
        __syncthreads();
        prefix = s_prefix;
        mask |= 0xFFull << shift;
        __syncthreads();
    }
    return dkey_inv(prefix);
}

__device__ __forceinline__ int64_t nearest_rank_index(double p, int64_t count) {
    int64_t idx = (int64_t)ceil(__dmul_rn(p, (double)count)) - 1;
    return idx < 0 ? 0 : (idx > count - 1 ? count - 1 : idx);
}

__constant__ double kAlphaGrid[8] = {0.0, 0.001, 0.002, 0.005, 0.01, 0.02, 0.05, 0.1};

// block c: b[g][c] = NR_alpha_g(entries of table c)
__global__ void cal_tables(const double* __restrict__ D, int64_t nq, int m, int g, double* __restrict__ b) {
    const int c = blockIdx.x;
    const int64_t cnt = nq * kK;
    auto val = [&](int64_t i) { return D[((i / kK) * m + c) * kK + (i % kK)]; };
    const double v = block_select(val, cnt, nearest_rank_index(kAlphaGrid[g], cnt));
    if (threadIdx.x == 0) b[g * m + c] = v;
}

// a[g] = 255 / NR_{1-alpha}(pooled y - b_m)  (1 if that quantile is <= 0)
__global__ void cal_pooled(const double* __restrict__ D, int64_t nq, int m, int g,
                           const double* __restrict__ b, double* __restrict__ a) {
    const int64_t cnt = nq * m * kK;
    const double* bg = b + g * m;
    auto val = [&](int64_t i) { return __dsub_rn(D[i], bg[(i / kK) % m]); };
    const double hi = block_select(val, cnt, nearest_rank_index(__dsub_rn(1.0, kAlphaGrid[g]), cnt));
    if (threadIdx.x == 0) a[g] = hi > 0.0 ? __ddiv_rn(255.0, hi) : 1.0;
}

__global__ void cal_err(const double* __restrict__ D, int64_t total, int m, int g,
                        const double* __restrict__ b, const double* __restrict__ a,
                        double* __restrict__ err) {
    const double ag = a[g];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const double bm = b[g * m + (e / kK) % m];
        const double y = D[e];
        double f = floor(__dmul_rn(ag, __dsub_rn(y, bm)));
        f = f < 0.0 ? 0.0 : (f > 255.0 ? 255.0 : f);
        const double ee = __dsub_rn(__dadd_rn(__ddiv_rn(f, ag), bm), y);
        err[e] = __dmul_rn(ee, ee);
    }
}

// sequential sum in entry order (the definition's order) -> mse[g]
__global__ void cal_sum(const double* __restrict__ err, int64_t total, int g, double* __restrict__ mse) {
    if (threadIdx.x != 0) return;
    double s = 0.0;
    for (int64_t e = 0; e < total; ++e) s = __dadd_rn(s, err[e]);
    mse[g] = __ddiv_rn(s, (double)total);
}

__global__ void cal_choose(const double* __restrict__ a, const double* __restrict__ b,
                           const double* __restrict__ mse, int m, float* __restrict__ a_out,
                           float* __restrict__ b_out, double* __restrict__ alpha_mse) {
    __shared__ int best;
    if (threadIdx.x == 0) {
        int bg = 0;
        for (int g = 1; g < 8; ++g)
            if (mse[g] < mse[bg]) bg = g;
        best = bg;
        a_out[0] = (float)a[bg];
        if (alpha_mse) {
            alpha_mse[0] = kAlphaGrid[bg];
            for (int g = 0; g < 8; ++g) alpha_mse[1 + g] = mse[g];
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < m; c += blockDim.x) b_out[c] = (float)b[best * m + c];
}

}  // namespace

size_t kmeans_ws_bytes(int64_t n, int j, int m) {
    return a256((size_t)j * kK * sizeof(double)) + a256((size_t)m * n * sizeof(int)) +
           a256((size_t)m * n * sizeof(double)) + a256((size_t)j * kK * sizeof(double)) +
           a256((size_t)m * kK * sizeof(int64_t));
}

cudaError_t launch_kmeans(const float* train, int64_t n, int j, int64_t ldx, int m,
                          const int64_t* init, int iters, float* C_out, void* ws, cudaStream_t s) {
    KmWs w = carve_km(ws, n, j, m);
    const size_t csmem = (size_t)j * kK * sizeof(double);
    if (csmem > 200 * 1024) return cudaErrorInvalidValue;
    cudaFuncSetAttribute(km_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem);
    km_init<<<(unsigned)ceil_div(j * kK, 256), 256, 0, s>>>(train, ldx, j, m, init, w.C64);
    const int sum_threads = 128;
    for (int it = 0; it < iters; ++it) {
        const int64_t total = n * m;
        const unsigned ablocks = (unsigned)min64(ceil_div(total, kFitThreads), 148 * 16);
        km_assign<<<ablocks, kFitThreads, csmem, s>>>(train, n, ldx, j, m, w.C64, w.assign, w.dist);
        km_sums<<<(unsigned)ceil_div(j, sum_threads), sum_threads, kK * sum_threads * sizeof(double), s>>>(
            train, n, ldx, j, m, w.assign, w.sums, w.counts);
        km_update<<<m, kFitThreads, 0, s>>>(train, n, ldx, j, m, w.dist, w.sums, w.counts, w.C64);
    }
    km_finish<<<(unsigned)ceil_div(j * kK, 256), 256, 0, s>>>(w.C64, j * kK, C_out);
    return cudaGetLastError();
}

size_t calibrate_ws_bytes(int64_t nq, int m) {
    return a256(8 * (size_t)m * sizeof(double)) + a256(8 * sizeof(double)) + a256(8 * sizeof(double)) +
           a256((size_t)nq * m * kK * sizeof(double));
}

cudaError_t launch_calibrate(const double* D, int64_t nq, int m, float* a_out, float* b_out,
                             double* alpha_mse, void* ws, cudaStream_t s) {
    char* p = static_cast<char*>(ws);
    double* b = reinterpret_cast<double*>(p); p += a256(8 * (size_t)m * sizeof(double));
    double* a = reinterpret_cast<double*>(p); p += a256(8 * sizeof(double));
    double* mse = reinterpret_cast<double*>(p); p += a256(8 * sizeof(double));
    double* err = reinterpret_cast<double*>(p);
    const int64_t total = nq * m * kK;
    for (int g = 0; g < 8; ++g) {
        cal_tables<<<m, 1024, 0, s>>>(D, nq, m, g, b);
        cal_pooled<<<1, 1024, 0, s>>>(D, nq, m, g, b, a);
        cal_err<<<(unsigned)min64(ceil_div(total, 256), 148 * 8), 256, 0, s>>>(D, total, m, g, b, a, err);
        cal_sum<<<1, 32, 0, s>>>(err, total, g, mse);
    }
    cal_choose<<<1, 64, 0, s>>>(a, b, mse, m, a_out, b_out, alpha_mse);
    return cudaGetLastError();
}

}  // namespace bolt
