// tc_conv.cu — placeholder, replaced by the tcgen05 row-tap kernel.
#include "kernels.h"
namespace c1d {
bool tc_conv_supported(const ConvGeom&) { return false; }
size_t tc_conv_workspace_bytes(const ConvGeom&) { return 0; }
cudaError_t launch_tc_conv(const uint16_t*, const float*, float*, const ConvGeom&, void*, cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace c1d
