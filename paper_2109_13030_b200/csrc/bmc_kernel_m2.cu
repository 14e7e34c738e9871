// Instantiation of the fused AM kernel for 2 footprint circle(s).
#include "bmc_kernel.cuh"
namespace bmc {
template cudaError_t launch_am_m<2>(const KernelArgs&, int, cudaStream_t);
}  // namespace bmc
