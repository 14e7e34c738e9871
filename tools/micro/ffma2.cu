// Microbenchmark: packed FFMA2 (fma.rn.ftz.f32x2, sm_100a) against scalar FFMA, register operands
// only (no immediates), throughput per SM at several warps/SM and dependent-chain latency.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2 ffma2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t f2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm volatile("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float f1(float a, float b, float c) {
  float d;
  asm volatile("fma.rn.ftz.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
template <int CH>
__global__ void k1(float* out, int iters, const float* in) {
  float v[CH], a = in[threadIdx.x & 7], b = in[8 + (threadIdx.x & 7)];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = in[16 + c];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = f1(v[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 1234.5f) out[0] = s;
}
template <int CH>
__global__ void k2(float* out, int iters, const float* in) {
  const uint64_t* p = reinterpret_cast<const uint64_t*>(in);
  uint64_t v[CH], a = p[threadIdx.x & 3], b = p[4 + (threadIdx.x & 3)];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = p[8 + c];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = f2(v[c], a, b);
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= v[c];
  if (s == 12345) out[0] = 1.f;
}
template <typename K> float timeit(K k) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k(); cudaDeviceSynchronize();
  cudaEventRecord(a); k(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  float *fo, *in;
  cudaMalloc(&fo, 64); cudaMalloc(&in, 4096);
  cudaMemset(in, 0, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  const double clk = 1.965e9;
  for (int warps : {1, 2, 4, 8, 16, 32}) {
    const int th = 32 * warps;
    const double lanes1 = (double)sms * th * iters * 8;   // scalar FMAs (8 chains)
    const float t1 = timeit([&] { k1<8><<<sms, th>>>(fo, iters, in); });
    const float t2 = timeit([&] { k2<8><<<sms, th>>>(fo, iters, in); });
    printf("warps/SM %2d: FFMA %6.1f lane-FMA/clk/SM   FFMA2 %6.1f lane-FMA/clk/SM (%.1f instr/clk/SM)\n", warps,
           lanes1 / (t1 * 1e-3) / sms / clk, 2 * lanes1 / (t2 * 1e-3) / sms / clk,
           lanes1 / 32 / (t2 * 1e-3) / sms / clk);
  }
  const float tl1 = timeit([&] { k1<1><<<1, 32>>>(fo, 1 << 16, in); });
  const float tl2 = timeit([&] { k2<1><<<1, 32>>>(fo, 1 << 16, in); });
  printf("dependent latency (cycles @1.965 GHz, incl. loop overhead): FFMA %.1f  FFMA2 %.1f\n",
         tl1 * 1e-3 * clk / 65536, tl2 * 1e-3 * clk / 65536);
  return 0;
}
