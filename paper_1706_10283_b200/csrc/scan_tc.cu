// scan_tc.cu -- tcgen05 one-hot(codes) x table variant (placeholder until implemented).
#include "common.cuh"

namespace bolt {
int topk_tc_supported(int64_t, int, int64_t, int) { return 0; }
int topk_tc_parts(int64_t, int, int64_t, int, int) { return 1; }
cudaError_t launch_topk_tc(const ScanArgs&, int, int, int64_t, int, uint64_t*, cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace bolt
