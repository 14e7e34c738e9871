// Instantiation of the fused AM kernel for 5 footprint circle(s).
#include "bmc_kernel.cuh"
namespace bmc {
template cudaError_t launch_am_m<5>(const KernelArgs&, int, cudaStream_t);
}  // namespace bmc
