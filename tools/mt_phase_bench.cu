// Microbenchmark of the generator's pieces (k_probe_regions): the mt19937_64 seeding
// (one thread, 311 serial steps) and the one-warp register twist of P phases, with no
// emission.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mtb tools/mt_phase_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kN = 312, kM = 156;
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ull;

__device__ __forceinline__ void tw(uint32_t ah, uint32_t al, uint32_t bl, uint32_t ch, uint32_t cl, uint32_t& rh,
                                   uint32_t& rl) {
  const uint32_t yl = (al & 0x80000000u) | (bl & 0x7FFFFFFFu);
  const uint32_t m = 0u - (yl & 1u);
  rl = cl ^ __funnelshift_r(yl, ah, 1) ^ (m & (uint32_t)kMatrixA);
  rh = ch ^ (ah >> 1) ^ (m & (uint32_t)(kMatrixA >> 32));
}

__global__ void k_seed(uint64_t* out) {
  __shared__ uint64_t z[kN];
  if (threadIdx.x == 0) {
    uint64_t x = 5489 + blockIdx.x;
    z[0] = x;
    for (int i = 1; i < kN; ++i) {
      x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
      z[i] = x;
    }
  }
  __syncthreads();
  out[blockIdx.x * 32 + threadIdx.x] = z[threadIdx.x * 9];
}

template <int kJ>
__global__ void k_twist(int phases, uint64_t* out) {
  const int L = threadIdx.x;
  const unsigned full = 0xffffffffu;
  const int nxt = (L + 1) & 31;
  const bool l31 = L == 31, l27 = L == 27;
  uint32_t Ah[kJ], Al[kJ], Bh[kJ], Bl[kJ];
  for (int j = 0; j < kJ; ++j) {
    Ah[j] = L * 7 + j + blockIdx.x;
    Al[j] = L * 13 + j;
    Bh[j] = L * 5 + j;
    Bl[j] = L * 3 + j;
  }
  for (int k = 0; k < phases; ++k) {
    uint32_t sa[kJ], sb[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      sa[j] = __shfl_sync(full, Al[j], nxt);
      sb[j] = __shfl_sync(full, Bl[j], nxt);
    }
    const uint32_t b0 = __shfl_sync(full, Bl[0], 0);
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      uint32_t n = j + 1 < kJ && l31 ? sa[j + 1 < kJ ? j + 1 : j] : sa[j];
      if (j == kJ - 1 && l27) n = b0;
      uint32_t rh, rl;
      tw(Ah[j], Al[j], n, Bh[j], Bl[j], rh, rl);
      Ah[j] = rh;
      Al[j] = rl;
    }
    const uint32_t a0 = __shfl_sync(full, Al[0], 0);
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      uint32_t n = j + 1 < kJ && l31 ? sb[j + 1 < kJ ? j + 1 : j] : sb[j];
      if (j == kJ - 1 && l27) n = a0;
      uint32_t rh, rl;
      tw(Bh[j], Bl[j], n, Ah[j], Al[j], rh, rl);
      Bh[j] = rh;
      Bl[j] = rl;
    }
  }
  uint64_t acc = 0;
  for (int j = 0; j < kJ; ++j) acc ^= (uint64_t)Ah[j] << 32 ^ Al[j] ^ (uint64_t)Bh[j] << 32 ^ Bl[j];
  out[blockIdx.x * 32 + L] = acc;
}

int main() {
  uint64_t* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_seed<<<16, 32>>>(out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep == 2) printf("seed: %.1f us\n", ms * 1e3);
    for (int P : {1, 442}) {
      cudaEventRecord(a);
      k_twist<5><<<16, 32>>>(P, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("twist kJ=5 P=%d: %.1f us (%.0f ns/phase)\n", P, ms * 1e3, ms * 1e6 / P);
    }
  }
  return 0;
}
