// probe SW128 descriptor conventions: A K-major SW128, B K-major or MN-major SW128, K=32 (4 MMAs)
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
constexpr int M = 128, N = 256, K = 32;
__global__ void probe(const float* A, const float* B, float* D, int mode, uint32_t lboB, uint32_t sboB) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  float* sA = (float*)sm;                   // 16 KB
  float* sB = (float*)(sm + M * K * 4);     // 32 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    int r = i / K, k = i % K;  // A row-major [M][K]
    sA[(r * 128 + (((k / 4) ^ (r % 8)) * 16) + (k % 4) * 4) / 4] = A[i];
  }
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) {
    int k = i / N, n = i % N;  // B row-major [K][N]
    int off;
    if (mode == 0) {  // K-major: row n holds 32 k values
      off = n * 128 + (((k / 4) ^ (n % 8)) * 16) + (k % 4) * 4;
    } else if (mode == 1) {          // MN-major: chunk j of 32 n, row k
      int j = n / 32, nn = n % 32;
      off = j * (K * 128) + k * 128 + (((nn / 4) ^ (k % 8)) * 16) + (nn % 4) * 4;
    } else {  // MN-major, 128B swizzle with 32B atomicity: granule ^= row % 4
      int j = n / 32, nn = n % 32;
      off = j * (K * 128) + k * 128 + (((nn / 8) ^ (k % 4)) * 32) + (nn % 8) * 4;
    }
    sB[off / 4] = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tm = tslot;
  if (warp == 1 && lane == 0) {
    uint32_t bmaj = mode == 0 ? 0u : 1u;
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (bmaj << 16) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    for (int kk = 0; kk < K / 8; ++kk) {
      uint64_t ad = desc(su(sA) + kk * 32, 16, 1024, 2);
      uint64_t bd = mode == 0 ? desc(su(sB) + kk * 32, 16, 1024, 2) : desc(su(sB) + kk * 1024, lboB, sboB, mode == 1 ? 2 : 1);
      uint32_t acc = kk > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp < 4) {
    for (int c = 0; c < N; ++c) {
      uint32_t r;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tm + ((warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      D[(warp * 32 + lane) * N + c] = __uint_as_float(r);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}
int main() {
  static float hA[M * K], hB[K * N], hD[M * N];
  for (int i = 0; i < M * K; ++i) hA[i] = (float)((i % 7) + 1);
  for (int i = 0; i < K * N; ++i) hB[i] = (float)((i % 5) + 1);
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  struct { int mode; uint32_t lbo, sbo; } cfg[] = {{0, 0, 0}, {2, 4096, 512}, {2, 512, 4096}, {2, 4096, 1024}};
  for (auto c : cfg) {
    cudaMemset(D, 0, sizeof hD);
    probe<<<1, 256, 100 * 1024>>>(A, B, D, c.mode, c.lbo, c.sbo);
    cudaError_t le = cudaGetLastError();
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    double maxerr = 0; int bad = 0;
    for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
      double ref = 0; for (int k = 0; k < K; ++k) ref += hA[i * K + k] * hB[k * N + j];
      double d = fabs(ref - hD[i * N + j]); if (d > maxerr) maxerr = d; if (d > 1e-3) ++bad;
    }
    printf("mode%d lbo=%u sbo=%u launch=%s sync=%s maxerr=%g bad=%d D00=%f ref00=%f\n", c.mode, c.lbo, c.sbo, cudaGetErrorString(le), cudaGetErrorString(e), maxerr, bad, hD[0], [&]{double r=0; for(int k=0;k<K;++k) r+=hA[k]*hB[k*N]; return r;}());
  }
  return 0;
}
