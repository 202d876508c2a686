// scan_prmt_q8.cu -- PRMT scan kernels instantiated for QT = 8 queries per thread
// (one translation unit per QT so the build compiles them in parallel).
#include "scan_prmt.cuh"

namespace bolt {
template <>
cudaError_t prmt_full_entry<8>(const ScanArgs& a, uint16_t* out16, float* out32, int64_t ldo, float inv_a,
                                 float b_sum, cudaStream_t s) {
    return pscan::launch_full_qt<8>(a, out16, out32, ldo, inv_a, b_sum, s);
}
template <>
cudaError_t prmt_topk_entry<8>(const ScanArgs& a, int k, int metric, int64_t index_base, int parts,
                                 uint64_t* part_keys, int sms, cudaStream_t s) {
    return pscan::launch_topk_qt<8>(a, k, metric, index_base, parts, part_keys, sms, s);
}
}  // namespace bolt
