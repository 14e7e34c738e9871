// Instantiation of the fused AM kernel for 8 footprint circle(s).
#include "bmc_kernel.cuh"
namespace bmc {
template cudaError_t launch_am_m<8>(const KernelArgs&, int, cudaStream_t);
}  // namespace bmc
