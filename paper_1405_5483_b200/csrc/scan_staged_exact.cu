// Staged-machine instantiations for one gram mode (see scan_staged.cuh).
#include "scan_staged.cuh"

namespace magb {
cudaError_t launch_staged_exact(const ScanArgs& a, cudaStream_t stream, int grid) {
  return launch_e<kKExact>(a, stream, grid);
}
}  // namespace magb
