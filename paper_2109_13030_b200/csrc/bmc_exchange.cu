// bmc_exchange.cu -- device side of the multi-GPU best-of-batch exchange.
//
// The batch argmin ("best cost trajectory"; rule G17) of a sharded
// solve is the minimum packed key over all ranks (keys carry the global
// index, so the minimum is unique and order-independent).  Each rank packs
// its shard's best {key, 55 coefficients} into a 256-byte record; the records
// are all-gathered over NCCL (torch.distributed, outside this library); every
// rank then selects the minimum record.  Both steps are one-warp kernels.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/bmc.h"
#include "bmc_internal.h"

namespace bmc {
namespace {

constexpr int REC = 32;   // int64 words per record: key, 55 floats packed, pad

__global__ void pack_best_kernel(const long long* __restrict__ best, const float* __restrict__ coeffs,
                                 const float* __restrict__ residual, const float* __restrict__ cost,
                                 long long index_base, long long* __restrict__ record) {
  const int lane = threadIdx.x;
  const long long key = best[1];
  const long long local = best[0] - index_base;   // instance within this shard
  const bool empty = key == -1ll;                 // empty shard: key ~0, no coefficients
  float* rf = reinterpret_cast<float*>(record + 1);
  if (lane == 0) record[0] = key;
  for (int k = lane; k < 5 * NV; k += 32) rf[k] = empty ? 0.f : coeffs[local * 5 * NV + k];
  for (int k = 5 * NV + lane; k < 2 * (REC - 1); k += 32) {
    float v = 0.f;   // floats 55, 56, 57: r1, r_psi, J of the instance
    if (!empty && residual && k < 5 * NV + 2) v = residual[local * 2 + (k - 5 * NV)];
    if (!empty && cost && k == 5 * NV + 2) v = cost[local];
    rf[k] = v;
  }
}

__global__ void select_best_kernel(const long long* __restrict__ records, int nranks,
                                   long long* __restrict__ best_out, float* __restrict__ coeffs_out) {
  const int lane = threadIdx.x;
  unsigned long long kmin = ~0ull;
  int rmin = 0;
  for (int r = lane; r < nranks; r += 32) {
    const unsigned long long k = (unsigned long long)records[(size_t)r * REC];
    if (k < kmin) { kmin = k; rmin = r; }
  }
  for (int o = 16; o >= 1; o >>= 1) {
    const unsigned long long ko = __shfl_xor_sync(0xffffffffu, kmin, o);
    const int ro = __shfl_xor_sync(0xffffffffu, rmin, o);
    if (ko < kmin || (ko == kmin && ro < rmin)) { kmin = ko; rmin = ro; }
  }
  const float* rf = reinterpret_cast<const float*>(records + (size_t)rmin * REC + 1);
  for (int k = lane; k < 5 * NV; k += 32) coeffs_out[k] = rf[k];
  if (lane == 0) {
    best_out[0] = (long long)(kmin & ((1ull << 30) - 1));
    best_out[1] = (long long)kmin;
  }
}

}  // namespace
}  // namespace bmc

namespace {
int32_t launch_status(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    bmc::set_last_error(BMC_OK, "");
    return BMC_OK;
  }
  return bmc::set_last_error(BMC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

extern "C" {

int32_t bmc_pack_best(const int64_t* best, const float* coeffs, const float* residual, const float* cost,
                      int64_t index_base, int64_t* record, bmc_stream_t stream) {
  if (!best || !coeffs || !record) return bmc::set_last_error(BMC_EINVAL, "bmc_pack_best: NULL pointer");
  bmc::pack_best_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const long long*>(best), coeffs, residual, cost, (long long)index_base,
      reinterpret_cast<long long*>(record));
  return launch_status("pack_best_kernel launch");
}

int32_t bmc_select_best(const int64_t* records, int32_t nranks, int64_t* best_out, float* coeffs_out,
                        bmc_stream_t stream) {
  if (!records || !best_out || !coeffs_out) return bmc::set_last_error(BMC_EINVAL, "bmc_select_best: NULL pointer");
  if (nranks < 1) return bmc::set_last_error(BMC_EINVAL, "bmc_select_best: nranks < 1");
  bmc::select_best_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const long long*>(records), nranks, reinterpret_cast<long long*>(best_out),
      coeffs_out);
  return launch_status("select_best_kernel launch");
}

}  // extern "C"
