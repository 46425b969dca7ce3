// select_tc.cu -- placeholder until the tcgen05 scorer lands.
#include "kernels.h"
namespace msn {
bool select_tc_supported(const Shape&) { return false; }
cudaError_t launch_select_tc(const Shape&, const void*, const void*, float*, int32_t*, cudaStream_t,
                             int*) {
  return cudaErrorNotSupported;
}
}  // namespace msn
