// bmc_sample.cu -- STOMP-style initial samples on the device (
// contract and reading G28 in include/bmc.h).  One thread per instance: three
// Philox4x32-10 blocks (counter-based, so a sample depends only on (seed,
// stream, global index)), Box-Muller in fp64, the 5 x 5 STOMP factor applied
// to the control points 3..7 of the straight segment.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bmc_internal.h"

namespace bmc {

namespace {

// Philox4x32-10 (Salmon et al., SC'11): multipliers and Weyl key increments.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__global__ void __launch_bounds__(128) stomp_kernel(const SampleArgs a) {
  const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= a.B) return;
  const long long g = a.index_base + l;
  float* o = a.init + l * 3 * NV;
  double cx[NV], cy[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    cx[k] = a.x0 + (a.xT - a.x0) * k / (NV - 1);
    cy[k] = a.y0 + (a.yT - a.y0) * k / (NV - 1);
  }
  if (!(a.line_first && g == 0)) {
    const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
    double z[12];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint4 x = philox4x32_10(make_uint4((uint32_t)(unsigned long long)g,
                                               (uint32_t)((unsigned long long)g >> 32),
                                               (uint32_t)a.stream + (uint32_t)j, (uint32_t)(a.stream >> 32)),
                                    key);
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const double u1 = ((double)w[2 * p] + 0.5) * 2.3283064365386963e-10;   // 2^-32
        const double u2 = ((double)w[2 * p + 1] + 0.5) * 2.3283064365386963e-10;
        const double r = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincospi(2.0 * u2, &sn, &cs);
        z[4 * j + 2 * p] = r * cs;
        z[4 * j + 2 * p + 1] = r * sn;
      }
    }
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      double ex = 0.0, ey = 0.0;
#pragma unroll
      for (int b = 0; b <= i; ++b) {
        ex = fma(a.L[i][b], z[b], ex);
        ey = fma(a.L[i][b], z[5 + b], ey);
      }
      cx[3 + i] = fma(a.sigma_x, ex, cx[3 + i]);
      cy[3 + i] = fma(a.sigma_y, ey, cy[3 + i]);
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    o[k] = (float)cx[k];
    o[NV + k] = (float)cy[k];
    o[2 * NV + k] = 0.f;
  }
}

}  // namespace

cudaError_t launch_stomp(const SampleArgs& a, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((a.B + 127) / 128);
  stomp_kernel<<<grid, 128, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace bmc
