// Probe images generated on the device (atc_testsets_upload_seeded).
//
// verify_rewrite draws test t's inputs from one liftc::Rng stream
// (rewriter.cpp:236-245): Rng(seed) wraps std::mt19937_64 (rng.hpp:13-48), and
// analysis::build_probe_image (analysis.cpp:73-98) fills each pointer's region
// with uniform_real(-1, 1) draws — 53-bit mantissa (gen() >> 11) * 2^-53,
// lo + u * (hi - lo) — rounded through float for *f32 pointers.  The host sends
// the seed of the stream and the stream position of each region; a CTA per test
// replays the stream (std::mt19937_64 is fully specified by the C++ standard)
// and writes every region of that test, so no region crosses PCIe.
#include <cuda_runtime.h>

#include <cstdint>

namespace atc {

namespace {
constexpr int kN = 312, kM = 156;
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x000000007FFFFFFFull;

__device__ __forceinline__ uint64_t twist_word(uint64_t cur, uint64_t next, uint64_t mid) {
  const uint64_t y = (cur & kUpper) | (next & kLower);
  return mid ^ (y >> 1) ^ ((y & 1ull) ? kMatrixA : 0ull);
}
__device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}
}  // namespace

// One CTA (320 threads) per test t.  The twist runs in two parallel phases
// (words [0, 156) read only old words; [156, 312) read the phase-1 results at
// k - 156 and, for k = 311, the new word 0), then 312 outputs are tempered and
// written to whichever region's stream window holds them.
__global__ void __launch_bounds__(320) k_probe_regions(int T, int nP, const uint64_t* seeds, const uint64_t* skips,
                                                       const int64_t* region_len, const int32_t* is_f32,
                                                       const int64_t* region_off, double* init, double* fin) {
  __shared__ uint64_t mt[kN];
  const int t = blockIdx.x;
  if (t >= T) return;
  const int k = threadIdx.x;
  if (k == 0) {  // seeding: mt[i] = f * (mt[i-1] ^ (mt[i-1] >> 62)) + i
    uint64_t x = seeds[t];
    mt[0] = x;
    for (int i = 1; i < kN; ++i) {
      x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
      mt[i] = x;
    }
  }
  uint64_t lo[8], hi[8];
  uint64_t end = 0;
  for (int p = 0; p < nP && p < 8; ++p) {
    lo[p] = skips[(size_t)t * nP + p];
    hi[p] = lo[p] + (uint64_t)region_len[p];
    end = hi[p] > end ? hi[p] : end;
  }
  __syncthreads();
  // each twist: phase 1 (read, sync, write, sync), phase 2 (read, sync, write,
  // sync); the new word is tempered from the register it was just computed in
  auto emit = [&](uint64_t base, uint64_t word) {
    const uint64_t pos = base + (uint64_t)k;  // stream position of this output
    const uint64_t y = temper(word);
    for (int p = 0; p < nP && p < 8; ++p)
      if (pos >= lo[p] && pos < hi[p]) {
        const double u = (double)(y >> 11) * 0x1.0p-53;
        double x = __dadd_rn(-1.0, __dmul_rn(u, 2.0));  // lo + u * (hi - lo), not contracted
        if (is_f32[p]) x = (double)__double2float_rn(x);
        const int64_t o = region_off[(size_t)t * nP + p] + (int64_t)(pos - lo[p]);
        init[o] = x;
        fin[o] = x;
      }
  };
  for (uint64_t base = 0; base < end; base += kN) {
    uint64_t v = 0;
    if (k < kM) v = twist_word(mt[k], mt[k + 1], mt[k + kM]);
    __syncthreads();
    if (k < kM) mt[k] = v;
    __syncthreads();
    if (k < kM) emit(base, v);
    uint64_t w = 0;
    if (k >= kM && k < kN) w = twist_word(mt[k], mt[(k + 1) % kN], mt[k - kM]);
    __syncthreads();
    if (k >= kM && k < kN) {
      mt[k] = w;
      emit(base, w);
    }
    __syncthreads();
  }
}

// final = init with the original run's writes: entries [diff_off[i], diff_off[i+1])
// of (t, p) pair i.
__global__ void k_apply_diffs(int nP, const int64_t* region_len, const int64_t* region_off, const int64_t* diff_off,
                              const int32_t* diff_pos, const double* diff_val, double* fin) {
  const int i = blockIdx.x, p = i % nP;
  double* f = fin + region_off[i];
  for (int64_t e = diff_off[i] + threadIdx.x; e < diff_off[i + 1]; e += blockDim.x) {
    const int32_t pos = diff_pos[e];
    if (pos < region_len[p]) f[pos] = diff_val[e];
  }
}

}  // namespace atc
