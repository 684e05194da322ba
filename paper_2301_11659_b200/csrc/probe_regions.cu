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
// standard's twist computes exactly these words in place.  Phase k computes the 312
// words z[312 (k + 1) + q] from the previous phase's (156 threads, two words each:
// z[n + 312] and z[n + 468]) with the state in registers (neighbours' words by warp
// shuffles, warp-boundary words through shared memory, one barrier per phase); the draws
// of phases that meet a region (a per-CTA bitmap) are tempered and stored by the same
// threads.  (A variant with 312 more threads tempering the previous phase's draws
// measured slower: the extra warps' per-phase overhead outweighs the shorter chain.)
// need (optional, [T * nP]): generate only the first need[t * nP + p] elements of
// region (t, p) — the phases stop at the last of them — and then, in the same CTA,
// scatter test t's final-minus-init entries (k_apply_diffs) and build its dirty
// lists over those prefixes (k_build_dirty), diff_* and v's dirty arrays.
// pre / pre_off (atc_testsets_upload_prefix): the prefixes come from the caller
// (packed, entries [pre_off[i], pre_off[i+1]) for region i) instead of the stream.
__device__ __forceinline__ void probe_regions_cta(int t, int T, int nP, const uint64_t* seeds, const uint64_t* skips,
                                                  const int64_t* region_len, const int32_t* is_f32,
                                                  const int64_t* region_off, const int64_t* need, double* init,
                                                  double* fin, const TestsetView& v, const int64_t* diff_off,
                                                  const int32_t* diff_pos, const double* diff_val, const double* pre,
                                                  const int64_t* pre_off) {
  __shared__ uint64_t z[1024];
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
  // stream positions are < 2^32 (probe images of a few hundred thousand draws): 32-bit
  // region windows [lo, lo + len) tested as (pos - lo) < len, offsets and f32 flags in
  // registers
  uint32_t lo[8], len[8];
  int64_t off[8];
  uint32_t f32m = 0, end = 0;
  const int np = pre ? 0 : nP < 8 ? nP : 8;
  for (int p = 0; p < np; ++p) {
    lo[p] = (uint32_t)skips[(size_t)t * nP + p];
    len[p] = (uint32_t)(need ? need[(size_t)t * nP + p] : region_len[p]);
    off[p] = region_off[(size_t)t * nP + p];
    f32m |= (is_f32[p] ? 1u : 0u) << p;
    end = lo[p] + len[p] > end ? lo[p] + len[p] : end;
  }
  // phase k computes the words of draws [312 k, 312 k + 312) (z[312 (k + 1) + i]); a bit
  // per phase whose draws meet a region (block-uniform), so most phases only twist
  constexpr int kMaxPhases = 4096;
  __shared__ uint32_t s_emit[kMaxPhases / 32];
  const uint32_t n_phases = (end + kN - 1) / kN;
  const bool bitmap = n_phases <= (uint32_t)kMaxPhases;
  if (bitmap)
    for (uint32_t w = q; w < (n_phases + 31) / 32; w += blockDim.x) {
      uint32_t m = 0;
      for (int b = 0; b < 32; ++b) {
        const uint32_t k = w * 32 + b;
        if (k >= n_phases) continue;
        const uint32_t d0 = k * kN;
        bool any = false;
        for (int p = 0; p < np; ++p) any = any || (d0 < lo[p] + len[p] && d0 + kN > lo[p]);
        m |= (any ? 1u : 0u) << b;
      }
      s_emit[w] = m;
    }
  __syncthreads();
  auto emit = [&](uint32_t pos, uint64_t w) {  // draw pos -> its region element, if any
    for (int p = 0; p < np; ++p)
      if (pos - lo[p] < len[p]) {  // (regions of a test do not overlap: one hit)
        const uint64_t y = temper(w);
        const double u = (double)(y >> 11) * 0x1.0p-53;
        const double x0 = __dadd_rn(-1.0, __dmul_rn(u, 2.0));  // lo + u * (hi - lo), not contracted
        const double x = (f32m >> p) & 1u ? (double)__double2float_rn(x0) : x0;
        const int64_t o = off[p] + (int64_t)(pos - lo[p]);
        init[o] = x;
        fin[o] = x;
      }
  };
  // The state in registers: thread q < 156 holds A = z[base + q] and B = z[base + 156 + q]
  // of the previous phase, so z[n + 312] = twist(A, A', B) and z[n + 468] = twist(B, B',
  // z[n + 312]) with A', B' thread q + 1's — of which twist reads only the low 32 bits:
  // one shuffle each inside the warp, across a warp boundary a 32-bit exchange in shared
  // memory (one barrier per phase); thread 155's z[n + 157] = z[base + 312] is thread
  // 0's new word, recomputed from the exchange.  Twists in 32-bit halves.
  // The exchange: every thread stores its low A, low B and high A each phase (unconditional
  // stores, double-buffered by phase parity so that a fast warp's next write cannot
  // overtake a slow warp's read); a warp's last lane reads thread q + 1's, thread 155
  // thread 0's and 1's.
  __shared__ uint32_t xs[2][3][kM];  // [parity][low A, low B, high A][thread]
  auto tw = [](uint32_t ah, uint32_t al, uint32_t bl, uint32_t ch, uint32_t cl, uint32_t& rh, uint32_t& rl) {
    // y = (a & 0xFFFFFFFF80000000) | (b & 0x7FFFFFFF); z = c ^ (y >> 1) ^ (y odd ? matrix A : 0)
    const uint32_t yl = (al & 0x80000000u) | (bl & 0x7FFFFFFFu);
    const uint32_t m = 0u - (yl & 1u);
    rl = cl ^ __funnelshift_r(yl, ah, 1) ^ (m & (uint32_t)kMatrixA);
    rh = ch ^ (ah >> 1) ^ (m & (uint32_t)(kMatrixA >> 32));
  };
  uint32_t Ah = 0, Al = 0, Bh = 0, Bl = 0;
  const int qq = q < kM ? q : kM - 1;  // threads 156..159 shadow thread 155 (never stored)
  Ah = (uint32_t)(z[qq] >> 32);
  Al = (uint32_t)z[qq];
  Bh = (uint32_t)(z[kM + qq] >> 32);
  Bl = (uint32_t)z[kM + qq];
  const int wl = q & 31;
  const bool act = q < kM, edge = wl == 31 && q < kM - 1, last = q == kM - 1;
  const int nx = q + 1 < kM ? q + 1 : 0;
  uint32_t bits = 0;
  uint32_t k = 0;
  for (uint32_t base = 0; base < end; base += kN, ++k) {
    uint32_t(*x)[kM] = xs[k & 1];
    if (act) {
      x[0][q] = Al;
      x[1][q] = Bl;
      x[2][q] = Ah;
    }
    if ((k & 31) == 0) bits = bitmap ? s_emit[k >> 5] : 0xFFFFFFFFu;
    __syncthreads();  // the previous phase's words visible
    uint32_t A1 = __shfl_down_sync(0xffffffffu, Al, 1), B1 = __shfl_down_sync(0xffffffffu, Bl, 1);
    if (act) {
      if (last) {  // z[n + 1] = z[base + 156] (thread 0's B), z[n + 157] = thread 0's new word
        uint32_t a0h, a0l;
        tw(x[2][0], x[0][0], x[0][1], 0u, x[1][0], a0h, a0l);  // only its low half is read
        A1 = x[1][0];
        B1 = a0l;
      } else if (edge) {
        A1 = x[0][nx];
        B1 = x[1][nx];
      }
      uint32_t wah, wal, wbh, wbl;
      tw(Ah, Al, A1, Bh, Bl, wah, wal);
      tw(Bh, Bl, B1, wah, wal, wbh, wbl);
      Ah = wah;
      Al = wal;
      Bh = wbh;
      Bl = wbl;
      bool any = bits & 1u;
      if (!bitmap) {
        any = false;
        for (int p = 0; p < np; ++p) any = any || (base < lo[p] + len[p] && base + kN > lo[p]);
      }
      if (any) {
        emit(base + q, (uint64_t)Ah << 32 | Al);
        emit(base + kM + q, (uint64_t)Bh << 32 | Bl);
      }
    }
    bits >>= 1;
  }
  __syncthreads();
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

__global__ void __launch_bounds__(kProbeThreads) k_probe_regions(int T, int nP, const uint64_t* seeds,
                                                                 const uint64_t* skips, const int64_t* region_len,
                                                                 const int32_t* is_f32, const int64_t* region_off,
                                                                 const int64_t* need, double* init, double* fin,
                                                                 TestsetView v, const int64_t* diff_off,
                                                                 const int32_t* diff_pos, const double* diff_val,
                                                                 const double* pre, const int64_t* pre_off) {
  probe_regions_cta(blockIdx.x, T, nP, seeds, skips, region_len, is_f32, region_off, need, init, fin, v, diff_off,
                    diff_pos, diff_val, pre, pre_off);
}

// A group of the handles of a batched in-place update (atc_testsets_update_seeded_many):
// CTAs [jobs[j].cta0, jobs[j + 1].cta0) (relative to the group's first) are handle j's
// tests; its seeded block (seeds, stream positions, final-minus-init entries, needed
// prefixes) is read from the update's device staging.
__global__ void __launch_bounds__(kProbeThreads) k_probe_regions_many(const ProbeJob* __restrict__ jobs, int n_jobs) {
  const int g = jobs[0].cta0 + (int)blockIdx.x;
  int j = 0;
  while (j + 1 < n_jobs && g >= jobs[j + 1].cta0) ++j;
  const ProbeJob& b = jobs[j];
  const TestsetView& v = b.view;
  probe_regions_cta(g - b.cta0, v.T, v.nP, b.seeds, b.skips, v.region_len, v.is_f32, v.region_off, b.need,
                    const_cast<double*>(v.init), const_cast<double*>(v.fin), v, b.diff_off, b.diff_pos, b.diff_val,
                    nullptr, nullptr);
}

// Each handle's metadata block (the TestsetView arrays) from the update staging into
// place, before the generators (which build the dirty lists in it).
__global__ void k_copy_meta(const ProbeJob* __restrict__ jobs) {
  const ProbeJob& b = jobs[blockIdx.x];
  const uint8_t* src = b.meta_src;
  uint8_t* dst = b.meta_dst;
  const size_t n16 = b.meta_bytes / 16;
  for (size_t i = threadIdx.x; i < n16; i += blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  for (size_t i = n16 * 16 + threadIdx.x; i < b.meta_bytes; i += blockDim.x) dst[i] = src[i];
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
