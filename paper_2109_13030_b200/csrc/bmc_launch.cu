// Dispatch of the fused AM kernel on the circle count m (see bmc_kernel.cuh).
#include "bmc_kernel.cuh"

namespace bmc {

extern template cudaError_t launch_am_m<1>(const KernelArgs&, int, cudaStream_t);
extern template cudaError_t launch_am_m<2>(const KernelArgs&, int, cudaStream_t);
extern template cudaError_t launch_am_m<3>(const KernelArgs&, int, cudaStream_t);
extern template cudaError_t launch_am_m<4>(const KernelArgs&, int, cudaStream_t);
extern template cudaError_t launch_am_m<5>(const KernelArgs&, int, cudaStream_t);
extern template cudaError_t launch_am_m<6>(const KernelArgs&, int, cudaStream_t);
extern template cudaError_t launch_am_m<7>(const KernelArgs&, int, cudaStream_t);
extern template cudaError_t launch_am_m<8>(const KernelArgs&, int, cudaStream_t);

size_t kernel_smem_bytes(int /*QP: fixed Q_MAX*/, int n, int ipc, int team) { return smem_bytes(n, ipc, team); }

cudaError_t launch_am(const KernelArgs& a, int wpc, cudaStream_t s) {
  switch (a.m) {
    case 1: return launch_am_m<1>(a, wpc, s);
    case 2: return launch_am_m<2>(a, wpc, s);
    case 3: return launch_am_m<3>(a, wpc, s);
    case 4: return launch_am_m<4>(a, wpc, s);
    case 5: return launch_am_m<5>(a, wpc, s);
    case 6: return launch_am_m<6>(a, wpc, s);
    case 7: return launch_am_m<7>(a, wpc, s);
    case 8: return launch_am_m<8>(a, wpc, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace bmc
