// tc_wgrad.cu — placeholder, replaced by the tcgen05 backward-weight kernel.
#include "kernels.h"
namespace c1d {
bool tc_wgrad_supported(int64_t, int64_t, int64_t, int64_t, int64_t, int64_t) { return false; }
size_t tc_wgrad_workspace_bytes(int64_t, int64_t, int64_t, int64_t, int64_t, int64_t) { return 0; }
cudaError_t launch_tc_wgrad(const uint16_t*, const uint16_t*, float*, void*, int64_t, int64_t, int64_t, int64_t,
                            int64_t, int64_t, cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace c1d
