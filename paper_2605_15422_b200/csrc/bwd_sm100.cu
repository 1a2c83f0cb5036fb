// bwd_sm100.cu -- tcgen05 backward (placeholder until the kernel lands).
#include "dkv_internal.h"
namespace dkv {
bool tc_bwd_supported(int, int, int, int) { return false; }
int launch_tc_bwd(const SimtArgs&, float*, const float2*, float*, int, int, bool, cudaStream_t) {
  set_error("tcgen05 backward not built");
  return DKV_ERR_UNSUPPORTED;
}
}  // namespace dkv
