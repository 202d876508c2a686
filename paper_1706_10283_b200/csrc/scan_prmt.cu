// scan_prmt.cu -- dispatch of the PRMT scan (kernels in scan_prmt.cuh,
// instantiated per QT in scan_prmt_q{1,2,4,8}.cu).
#include "scan_prmt.cuh"

namespace bolt {

cudaError_t launch_scan_full(const ScanArgs& a, uint16_t* out16, float* out32, int64_t ldo,
                             float inv_a, float b_sum, cudaStream_t s) {
    if (a.n == 0 || a.nq == 0) return cudaSuccess;
    switch (pscan::pick_qt(a.nq)) {
        case 8: return prmt_full_entry<8>(a, out16, out32, ldo, inv_a, b_sum, s);
        case 4: return prmt_full_entry<4>(a, out16, out32, ldo, inv_a, b_sum, s);
        case 2: return prmt_full_entry<2>(a, out16, out32, ldo, inv_a, b_sum, s);
        default: return prmt_full_entry<1>(a, out16, out32, ldo, inv_a, b_sum, s);
    }
}

int topk_prmt_parts(int64_t n, int m, int64_t nq, int k, int num_sms) {
    (void)m;
    (void)k;
    const int64_t tiles = ceil_div(nq, pscan::pick_qt(nq));
    return choose_parts(tiles, ceil_div(n, 8), (int64_t)num_sms * 4 * pscan::kWarps, 32 * 4);
}

cudaError_t launch_topk_prmt(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                             uint64_t* part_keys, int sms, cudaStream_t s) {
    switch (pscan::pick_qt(a.nq)) {
        case 8: return prmt_topk_entry<8>(a, k, metric, index_base, parts, part_keys, sms, s);
        case 4: return prmt_topk_entry<4>(a, k, metric, index_base, parts, part_keys, sms, s);
        case 2: return prmt_topk_entry<2>(a, k, metric, index_base, parts, part_keys, sms, s);
        default: return prmt_topk_entry<1>(a, k, metric, index_base, parts, part_keys, sms, s);
    }
}

}  // namespace bolt
