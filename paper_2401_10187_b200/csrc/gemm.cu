// gemm.cu — large-P GEMM-style sliced multiply.  Placeholder: the planner
// does not select KIND_GEMM until the kernel lands, so large-P factors use generic.cu.
#include <cuda_runtime.h>

#include "kron_internal.h"

namespace kron {

bool gemm_supported(int, int64_t, int64_t, int, int) { return false; }

int launch_gemm(const PassPlan &, int, int64_t, const void *, void *, const void *, void *) {
  return (int)cudaErrorNotSupported;
}

}  // namespace kron
