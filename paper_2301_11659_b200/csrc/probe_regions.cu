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

#include "eval_common.cuh"

namespace atc {

namespace {
constexpr int kN = 312, kM = 156;
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x000000007FFFFFFFull;

__device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}
}  // namespace

// One CTA per test t.  As a sequence, std::mt19937_64 is z[0..311] = the seeded
// state and z[n + 312] = z[n + 156] ^ f(z[n], z[n + 1]) (f: the upper/lower-bit
// merge, shift and matrix-A step of the twist), draw i = temper(z[312 + i]) — the
// standard's twist computes exactly these words in place.  Step j computes the 156
// words z[312 + 156j + q] (q < 156) at once from words of earlier steps, in a
// 624-word ring (each step overwrites only words no later step reads), so one
// barrier per 156 draws; steps whose draws fall in no region are not tempered.
// need (optional, [T * nP]): generate only the first need[t * nP + p] elements of
// region (t, p) — the steps stop at the last of them — and then, in the same CTA,
// scatter test t's final-minus-init entries (k_apply_diffs) and build its dirty
// lists over those prefixes (k_build_dirty), diff_* and v's dirty arrays.
// pre / pre_off (atc_testsets_upload_prefix): the prefixes come from the caller
// (packed, entries [pre_off[i], pre_off[i+1]) for region i) instead of the stream.
__global__ void __launch_bounds__(160) k_probe_regions(int T, int nP, const uint64_t* seeds, const uint64_t* skips,
                                                       const int64_t* region_len, const int32_t* is_f32,
                                                       const int64_t* region_off, const int64_t* need, double* init,
                                                       double* fin, TestsetView v, const int64_t* diff_off,
                                                       const int32_t* diff_pos, const double* diff_val,
                                                       const double* pre, const int64_t* pre_off) {
  constexpr int kRing = 2 * kN;
  __shared__ uint64_t z[kRing];
  const int t = blockIdx.x;
  if (t >= T) return;
  const int q = threadIdx.x;
  if (pre) {  // atc_testsets_upload_prefix: the caller's own prefixes, no generator
    for (int p = 0; p < nP; ++p) {
      const size_t i = (size_t)t * nP + p;
      const double* src = pre + pre_off[i];
      const int64_t n = pre_off[i + 1] - pre_off[i], o = region_off[i];
      for (int64_t e = q; e < n; e += blockDim.x) {
        const double x = src[e];
        init[o + e] = x;
        fin[o + e] = x;
      }
    }
  } else if (q == 0) {  // seeding: mt[i] = f * (mt[i-1] ^ (mt[i-1] >> 62)) + i
    uint64_t x = seeds[t];
    z[0] = x;
    for (int i = 1; i < kN; ++i) {
      x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
      z[i] = x;
    }
  }
  uint64_t lo[8], hi[8];
  uint64_t end = 0;
  const int np = pre ? 0 : nP < 8 ? nP : 8;
  for (int p = 0; p < np; ++p) {
    lo[p] = skips[(size_t)t * nP + p];
    hi[p] = lo[p] + (uint64_t)(need ? need[(size_t)t * nP + p] : region_len[p]);
    end = hi[p] > end ? hi[p] : end;
  }
  __syncthreads();
  auto wrap = [](int i) { return i >= kRing ? i - kRing : i; };  // i < 2 * kRing
  auto twist = [](uint64_t a, uint64_t b, uint64_t c) {  // z[n + 312] from z[n], z[n + 1], z[n + 156]
    const uint64_t y = (a & kUpper) | (b & kLower);
    return c ^ (y >> 1) ^ ((y & 1ull) ? kMatrixA : 0ull);
  };
  auto emit = [&](uint64_t base, uint64_t w) {  // draw base + q of this step into the regions
    bool any = false;  // block-uniform: does this step's window meet a region?
    for (int p = 0; p < np; ++p) any = any || (base < hi[p] && base + kM > lo[p]);
    if (!any || q >= kM) return;
    const uint64_t pos = base + (uint64_t)q;
    const uint64_t y = temper(w);
    const double u = (double)(y >> 11) * 0x1.0p-53;
    const double x0 = __dadd_rn(-1.0, __dmul_rn(u, 2.0));  // lo + u * (hi - lo), not contracted
    for (int p = 0; p < np; ++p)
      if (pos >= lo[p] && pos < hi[p]) {
        const double x = is_f32[p] ? (double)__double2float_rn(x0) : x0;
        const int64_t o = region_off[(size_t)t * nP + p] + (int64_t)(pos - lo[p]);
        init[o] = x;
        fin[o] = x;
      }
  };
  // two steps per barrier: step B's thread q needs z[n + 156] and z[n + 157] (written two
  // steps back, visible since the last barrier) and z[n + 312] = its own step-A word;
  // only thread 155's z[n + 157] is step A's word of thread 0, which it recomputes
  int r = 0;  // base % kRing
  for (uint64_t base = 0; base < end; base += 2 * kM, r = wrap(r + 2 * kM)) {
    uint64_t wa = 0, wb = 0;
    if (q < kM) {
      const int n = r + q;
      const uint64_t zn156 = z[wrap(n + kM)];
      wa = twist(z[wrap(n)], z[wrap(n + 1)], zn156);
      const uint64_t zn157 = q == kM - 1 ? twist(z[wrap(r)], z[wrap(r + 1)], z[wrap(r + kM)]) : z[wrap(n + kM + 1)];
      wb = twist(zn156, zn157, wa);
      // the slots of z[n + 312] / z[n + 468] held z[n - 312] / z[n - 156]: read by
      // neither step of this pair
      z[wrap(n + kN)] = wa;
      z[wrap(n + kN + kM)] = wb;
    }
    emit(base, wa);
    emit(base + kM, wb);
    __syncthreads();  // this pair's words visible to the next pair
  }
  if (!need) return;
  for (int p = 0; p < nP; ++p) {  // final = init + the original run's writes
    const size_t i = (size_t)t * nP + p;
    double* f = fin + region_off[i];
    for (int64_t e = diff_off[i] + q; e < diff_off[i + 1]; e += blockDim.x) {
      const int32_t pos = diff_pos[e];
      if (pos < region_len[p]) f[pos] = diff_val[e];
    }
  }
  __syncthreads();
  const int lane = q & 31;
  for (int p = 0; p < nP; ++p) {  // dirty lists over the generated prefixes
    const size_t i = (size_t)t * nP + p;
    const int64_t len = need[i];
    const bool f32 = is_f32[p] != 0;
    const double* a = init + region_off[i];
    const double* f = fin + region_off[i];
    int32_t* out = const_cast<int32_t*>(v.dirty_pos) + v.dirty_off[i];
    constexpr int U = 4;  // four elements per thread in flight: the loads do not wait on the ballots
    for (int64_t b = 0; b < len; b += (int64_t)U * blockDim.x) {
      double av[U], fv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = b + (int64_t)u * blockDim.x + q;
        av[u] = e < len ? a[e] : 0.0;
        fv[u] = e < len ? f[e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = b + (int64_t)u * blockDim.x + q;
        const bool dirty = e < len && mismatch(av[u], fv[u], f32);
        const unsigned ball = __ballot_sync(0xffffffffu, dirty);
        if (ball == 0) continue;
        int slot = 0;
        if (lane == 0) slot = atomicAdd(const_cast<int32_t*>(v.dirty_cnt) + i, __popc(ball));
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (dirty) {
          out[slot + __popc(ball & ((1u << lane) - 1))] = (int32_t)e;
          atomicMax(const_cast<int32_t*>(v.dirty_max) + i, (int32_t)e);
        }
      }
    }
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
