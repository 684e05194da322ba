// On-box peak of the FP64 CUDA-core pipe (SURVEY.md §8d asks for the K2 FP64 pipe
// utilisation against a DFMA peak measured on the box).  Independent DFMA chains,
// 8 per thread, enough CTAs to fill every SM; timed with CUDA events.
#include <cuda_runtime.h>

#include "atc_b200.h"
#include "capi_internal.h"

namespace atc {

__global__ void __launch_bounds__(256) k_dfma_chains(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

}  // namespace atc

extern "C" int atc_measure_dfma_peak(atc_ctx* ctx, double* gflops) {
  ATC_ENTER(ctx);
  if (!gflops) return ATC_ERR_ARG;
  cudaSetDevice(ctx->device);
  double* out = (double*)atc_ctx_scratch(ctx, 31, 64);
  if (!out) return ATC_ERR_CUDA;
  const int blocks = ctx->sm_count * 8, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  atc::k_dfma_chains<<<blocks, 256, 0, ctx->stream>>>(out, iters, 0.999999, 1e-7);  // warm-up
  cudaEventRecord(e0, ctx->stream);
  atc::k_dfma_chains<<<blocks, 256, 0, ctx->stream>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1, ctx->stream);
  const bool ok = atc_cuda_ok(ctx, cudaEventSynchronize(e1), "dfma peak");
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (!ok || ms <= 0) return ATC_ERR_CUDA;
  *gflops = 2.0 * 8.0 * iters * (double)blocks * 256 / (ms * 1e-3) / 1e9;
  return ATC_OK;
}
