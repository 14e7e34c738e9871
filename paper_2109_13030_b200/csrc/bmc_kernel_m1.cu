// Instantiation of the fused AM kernel for 1 footprint circle(s).
#include "bmc_kernel.cuh"
namespace bmc {
template cudaError_t launch_am_m<1>(const KernelArgs&, int, cudaStream_t);
}  // namespace bmc
