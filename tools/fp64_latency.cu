// Dependent-chain latency of FP64 DADD / DMUL / DFMA and of a shared-memory load feeding
// a DADD chain (the position-table running sums), one thread, clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_fp64lat tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double x, double y, long long* out, double* sink) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double a = x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) a = __dadd_rn(a, y);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) a = __dmul_rn(a, y);
  long long t2 = clock64();
  double acc = 0.0;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) acc = __dadd_rn(acc, __dmul_rn(s[i], s[(i * 7) & 1023]));
  long long t3 = clock64();
  double acc2 = 0.0;
#pragma unroll 8
  for (int i = 0; i < 1024; ++i) acc2 = __dadd_rn(acc2, __dmul_rn(s[i], s[(i * 7) & 1023]));
  long long t4 = clock64();
  out[0] = t1 - t0;
  out[1] = t2 - t1;
  out[2] = t3 - t2;
  out[3] = t4 - t3;
  sink[0] = a + acc + acc2;
}

int main() {
  long long* d;
  double* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 8);
  long long h[4];
  for (int r = 0; r < 2; ++r) k_lat<<<1, 32>>>(1.0, 1.0000001, d, sink);
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("cycles per op: dadd chain %.1f, dmul chain %.1f, lds+dmul+dadd (no unroll) %.1f, (unroll 8) %.1f\n",
         h[0] / 1024.0, h[1] / 1024.0, h[2] / 1024.0, h[3] / 1024.0);
  return 0;
}
