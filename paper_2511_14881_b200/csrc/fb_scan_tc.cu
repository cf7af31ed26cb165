// tcgen05 (sm_100a) emit scan -- placeholder until the tensor-core path lands.
#include "fb_internal.cuh"

namespace fb {

bool scan_tc_supported(const ScanArgs&) { return false; }

int launch_scan_tc(const ScanArgs&, cudaStream_t) { return FB_ERR_UNSUPPORTED; }

}  // namespace fb
