// K = 1 instantiations of the mma.sync SBVR GEMV kernel (gemv_mma.cuh), one TU per K for parallel builds.
#include "gemv_mma.cuh"

namespace sbvr {
namespace mma {
template cudaError_t launch_k<1>(const ImmaParams&, int, int, bool, bool, bool, cudaStream_t);
}  // namespace mma
}  // namespace sbvr
