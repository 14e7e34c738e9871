// Microbenchmark: FP64 tensor-core MMA (mma.sync f64) throughput and latency on sm_100a,
// next to plain DFMA.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a dmma.cu -o dmma
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1688(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

template <int CH>
__global__ void k884(double* out, int iters) {
  double acc[CH][2];
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = threadIdx.x * 1e-3 + c;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) mma884(acc[c], a, b);
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1234.5) out[0] = s;
}
template <int CH>
__global__ void k1688(double* out, int iters) {
  double acc[CH][4];
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = threadIdx.x * 1e-3 + c;
  double a[4] = {1.0, 1.0, 1.0, 1.0 + threadIdx.x * 1e-9}, b[2] = {0.5, 0.25};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) mma1688(acc[c], a, b);
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 1234.5) out[0] = s;
}

template <typename K>
float timeit(K k) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k();
  cudaEventRecord(a);
  k();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ghz = clk * 1e-6;
  const int iters = 20000;
  // latency: one warp, one chain
  {
    float ms = timeit([&] { k884<1><<<1, 32>>>(out, iters); });
    printf("m8n8k4 latency: %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / iters);
    ms = timeit([&] { k1688<1><<<1, 32>>>(out, iters); });
    printf("m16n8k8 latency: %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / iters);
  }
  for (int warps : {1, 4, 8, 16}) {
    float ms = timeit([&] { k884<8><<<sms, 32 * warps>>>(out, iters); });
    const double inst = (double)sms * warps * iters * 8;
    printf("m8n8k4  %2d warps/SM x 8 chains: %.2f inst/clk/SM, %.1f TFLOP/s\n", warps,
           inst / (ms * 1e-3 * ghz * 1e9) / sms, inst * 512 / (ms * 1e-3) / 1e12);
    ms = timeit([&] { k1688<8><<<sms, 32 * warps>>>(out, iters); });
    printf("m16n8k8 %2d warps/SM x 8 chains: %.2f inst/clk/SM, %.1f TFLOP/s\n", warps,
           inst / (ms * 1e-3 * ghz * 1e9) / sms, inst * 2048 / (ms * 1e-3) / 1e12);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s (clock %.2f GHz nominal)\n", cudaGetErrorString(e), ghz);
  return 0;
}
