// Microbenchmark: FFMA / DFMA / MUFU.RSQ throughput and dependent latency on one SM and full chip.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T, int CH>
__global__ void thr(T* out, int iters, T a, T b) {
  T v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = v[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == (T)1234.5) out[0] = s;
}
__global__ void rsq(float* out, int iters) {
  float v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = 1.f + threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) { float y; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[c])); v[c] = y + 1.f; }
  }
  float s = 0; for (int c = 0; c < 8; ++c) s += v[c];
  if (s == 1234.5f) out[0] = s;
}
template <typename K> float timeit(K k) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k(); cudaDeviceSynchronize();
  cudaEventRecord(a); k(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  float* fo; double* dd; cudaMalloc(&fo, 64); cudaMalloc(&dd, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int warps : {1, 4, 8, 16, 32}) {
    int blocks = sms, th = 32 * warps;
    double nop = (double)blocks * th * iters * 8;
    float tf = timeit([&] { thr<float, 8><<<blocks, th>>>(fo, iters, 1.0001f, 0.5f); });
    float td = timeit([&] { thr<double, 8><<<blocks, th>>>(dd, iters, 1.0001, 0.5); });
    float tr = timeit([&] { rsq<<<blocks, th>>>(fo, iters); });
    printf("warps/SM %2d: FFMA %.2f Tlane-op/s (%.1f /clk/SM @1.965GHz)  DFMA %.3f T/s (%.2f /clk/SM)  RSQ %.2f T/s (%.1f /clk/SM)\n",
           warps, nop / tf * 1e-9, nop / tf * 1e3 / sms / 1.965e9, nop / td * 1e-9, nop / td * 1e3 / sms / 1.965e9,
           nop / tr * 1e-9, nop / tr * 1e3 / sms / 1.965e9);
  }
  // dependent-chain latency: 1 warp, 1 chain
  float tl = timeit([&] { thr<float, 1><<<1, 32>>>(fo, 1 << 16, 1.0001f, 0.5f); });
  float tdl = timeit([&] { thr<double, 1><<<1, 32>>>(dd, 1 << 16, 1.0001, 0.5); });
  printf("latency (cycles @1.965GHz, incl. loop overhead): FFMA %.1f  DFMA %.1f\n", tl * 1e-3 * 1.965e9 / 65536,
         tdl * 1e-3 * 1.965e9 / 65536);
  return 0;
}
