// fit.cu -- offline fit on the GPU (placeholder until implemented).
#include "common.cuh"

namespace bolt {
size_t kmeans_ws_bytes(int64_t, int, int) { return 256; }
cudaError_t launch_kmeans(const float*, int64_t, int, int64_t, int, const int64_t*, int, float*, void*,
                          cudaStream_t) {
    return cudaErrorNotSupported;
}
size_t calibrate_ws_bytes(int64_t, int) { return 256; }
cudaError_t launch_calibrate(const double*, int64_t, int, float*, float*, double*, void*, cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace bolt
