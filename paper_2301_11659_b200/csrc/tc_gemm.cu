// K4/K5: tcgen05 tensor-core FP32-in / FP32-out contractions (kind::tf32).
//
// Replaces profitability::cpu_gemm / xpu_gemm (/root/reference/proj/src/
// profitability.cpp:14-63: row-major C[m][n] = sum_p A[m][p] * B[p][n], C
// overwritten) and reference_conv2d's semantics (equivalence.cpp:67-93; valid
// padding, unit stride, NCHW input, KCRS weights, NKOhOw output) on FP32 data.
//
// One persistent, warp-specialised kernel:
//   warp 0      TMA producer: A tile [128 x 32] K-major, B tile 8 x [32 x 32]
//               MN-major chunks, both 128B-swizzled, into a 4-stage smem ring
//   warp 1      MMA issuer: 4 x tcgen05.mma.cta_group::1.kind::tf32 (M=128,
//               N=256, K=8) per stage, accumulating in TMEM; tcgen05.commit
//               frees the smem stage / publishes the accumulator
//   warp 2      TMEM allocator (512 columns = 2 accumulators of 128 x 256 fp32)
//   warps 4-7   epilogue: tcgen05.ld 32x32b.x32 -> registers -> global
// The two TMEM accumulators let the epilogue of tile i overlap the MMAs of
// tile i+1.
//
// Precision: TF32 (1 pass; inputs truncated to 10-bit mantissas by the tensor
// core, FP32 accumulation) or 3xTF32 (A = Ah + Al, B = Bh + Bl split once by
// k_split_tf32; C = Ah*Bh + Al*Bh + Ah*Bl as one K' = 3K contraction), which
// recovers ~FP32 accuracy.  See DESIGN.md §4 for the measured error.
//
// Conv2d (NCHW, valid, unit stride) is the same kernel in implicit-GEMM form:
// M = filters, N = output pixels laid out on the INPUT grid (p = y*W + x),
// K' = (r, s, c).  The input is transposed once to NHWC (k_nchw_to_nhwc), so
// for a fixed (r, s) the B operand is rows p + r*W + s of the [N*H*W][C] view —
// an affine row shift, i.e. one plain K-major 2-D TMA box per stage, with no
// im2col buffer.  Pixels with x >= OW or y >= OH are computed and discarded by
// the epilogue (waste (R-1)/H + (S-1)/W), which writes NCHW directly.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "atc_b200.h"
#include "capi_internal.h"

namespace atc {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 32;  // BK = one 128B swizzle atom of fp32
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 4;        // 16 KB
constexpr int B_BYTES = BN * BK * 4;        // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EPI_WARPS = 4;  // one per TMEM lane quadrant (8 = two per quadrant, each half of the columns)
constexpr int NUM_THREADS = 128 + 32 * EPI_WARPS;
constexpr int TMEM_COLS = 512;
constexpr int kEpiStride = 1280;  // floats per epilogue warp: a 32x33 tile, rounded to 1 KB (TMA swizzle alignment)
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 1024 /*barriers*/ + EPI_WARPS * kEpiStride * 4;

// ------------------------------------------------------------ PTX helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
// 3-D box (MN-major B as [chunk][K row][32 columns]: all of a stage's chunks in one load)
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// smem matrix descriptor (tcgen05 "shared memory descriptor"): start >> 4 at
// [0,14), LBO >> 4 at [16,30), SBO >> 4 at [32,46), version 1 at [46,48),
// layout at [61,64): 2 = SWIZZLE_128B (16 B granules ^= row % 8), 1 =
// SWIZZLE_128B_BASE32B (32 B granules ^= row % 4).  32-bit MN-major operands
// need the BASE32B form (TMA: CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B); a plain
// 128B swizzle on an MN-major tf32 operand makes the MMA produce zeros
// (measured with tools/tc_probe_mn_major.cu).
constexpr uint32_t kSw128 = 2, kSw128Base32 = 1;
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// instruction descriptor, kind::tf32: D f32 [4,6)=1, A tf32 [7,10)=2,
// B tf32 [10,13)=2, A K-major [15]=0, B major [16] (1 = MN-major for the sgemm's
// row-major B, 0 = K-major for the conv's NHWC input), N>>3 [17,23), M>>4 [24,29)
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t b_mn_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (b_mn_major << 16) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

// M = 128 with the operand majors and N given (N a multiple of 16, <= 256)
__host__ __device__ constexpr uint32_t idesc_tf32_n(uint32_t a_mn_major, uint32_t b_mn_major, uint32_t n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn_major << 15) | (b_mn_major << 16) | ((n >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#define TMEM_LD_32x32b_x32(taddr, r)                                                                          \
  asm volatile(                                                                                               \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                          \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),       \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),          \
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),          \
        "=r"(r[30]), "=r"(r[31])                                                                              \
      : "r"(taddr))

// ------------------------------------------------------------ problem -------
struct Problem {
  // GEMM: C[M][N] (row-major, ldc) ; A map over [M][K] ; B map over [K][N]
  // CONV: out NCHW ; A map over W_krsc [Kf][R*S*C] ; B map over In [Nimg*C][H*W]
  int conv;
  int M, N, K;          // gemm sizes; conv: M = filters, N = H*W (pixels on the input grid), K = C (per r,s)
  int splits;           // 1 (TF32) or 3 (3xTF32: K' = 3K over hi/lo operand maps)
  float* C;
  int64_t ldc;
  // conv geometry
  int img, Cin, H, W, R, S, OH, OW;
  int tiles_m, tiles_n, tiles_img;
  int pair;  // 1: CTA pairs (cluster of 2) on adjacent M tiles share the B tile via TMA multicast
  int tma_store;  // 1: epilogue writes 32x32 sub-tiles with TMA bulk stores (modes 0, 2, 3)
  int umma2;      // 1: sgemm on k_tc_gemm2 (cta_group::2, M = 256 per CTA pair)
  int b3d;        // the MN-major operand's map is 3-D [chunks of 32][K][32] (one load per stage):
                  // sgemm (mode 0) B, 1x1 pixels-as-M (mode 5) A
  int bn;         // conv mode 5: filters per tile (N of the MMA, a multiple of 32, <= BN)
  int ksplit;     // k_tc_gemm2, conv mode 4: 2 = each tile's k-blocks in two halves on two
                  // pairs, both added into the zeroed output (two partial sums: the same
                  // result in either order)
};

struct Maps {
  CUtensorMap a[2];  // hi, lo
  CUtensorMap b[2];
  CUtensorMap c;     // output [rows][cols] fp32, 32x32 boxes, 128B swizzle (p.tma_store)
};

__device__ __forceinline__ void tile_coords(const Problem& p, int tile, int& tm, int& tn, int& ti, int G = 0) {
  // grouped raster: G m-tiles x all n-tiles per group, for L2 reuse of A/B panels.
  // With p.pair the unit is an M-tile pair: the caller maps tm -> 2*tm + rank.
  const int tiles_m = p.pair ? (p.tiles_m + 1) / 2 : p.tiles_m;
  const int per_img = tiles_m * p.tiles_n;
  ti = tile / per_img;
  int t = tile - ti * per_img;
  if (G == 0) G = p.pair ? 8 : 16;
  const int group = t / (G * p.tiles_n);
  const int first_m = group * G;
  const int gm = min(G, tiles_m - first_m);
  const int in_group = t - group * G * p.tiles_n;
  tm = first_m + in_group % gm;
  tn = in_group / gm;
}

// The producers' walk over a unit's k-blocks kb in [0, splits * kblocks), without
// divisions (the producer is one thread and a stage's MMAs last ~500 cycles, so its
// per-k-block integer work must stay far below that).  Coordinates of k-block k:
//   A (every mode): column k * BK of [M][K] / W_krsc [Kf][R*S*C] (= r*S*C + s*C + c0), row tm * BM
//   B sgemm: (tn * BN, k * BK) of [K][N]; mode 3 (B transposed): (k * BK, tn * BN) of [N][K]
//   B conv on the NHWC input grid (mode 1): channel c0, pixel row img*H*W + tn*BN + r*W + s
//   B 1x1 on NCHW (mode 2): pixel tn * BN, row img * C + c0 of [N*C][H*W]
//   B im2col (mode 4): channel c0 at the tile's first output pixel, tap offsets (s, r)
// 3xTF32 order of the splits: lo*hi, hi*lo, hi*hi (small terms first).
struct KbWalk {
  int split, k;   // operand split (3xTF32), k-block within the split
  int c0, r, s;   // conv: channel block start, filter tap
  __device__ __forceinline__ void start(const Problem& p, int kb, int kblocks) {
    split = kb / kblocks;
    k = kb - split * kblocks;
    c0 = r = s = 0;
    if (p.conv == 1 || p.conv == 2 || p.conv == 4 || p.conv == 5) {
      const int cblocks = p.K / BK, rs = k / cblocks;
      c0 = (k - rs * cblocks) * BK;
      r = rs / p.S;
      s = rs - r * p.S;
    }
  }
  __device__ __forceinline__ void next(const Problem& p, int kblocks) {
    if (++k == kblocks) {
      k = 0;
      ++split;
      c0 = r = s = 0;
      return;
    }
    c0 += BK;
    if (c0 == p.K) {
      c0 = 0;
      if (++s == p.S) {
        s = 0;
        ++r;
      }
    }
  }
  __device__ __forceinline__ int sel_a(const Problem& p) const { return split == 0 && p.splits == 3 ? 1 : 0; }
  __device__ __forceinline__ int sel_b() const { return split == 1 ? 1 : 0; }
};

__global__ void __launch_bounds__(NUM_THREADS, 1) k_tc_gemm(const __grid_constant__ Maps maps, const Problem p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kblocks = (p.conv == 1 || p.conv == 2 || p.conv == 5 ? p.R * p.S * (p.K / BK) : (p.K + BK - 1) / BK);
  const int total_kb = kblocks * p.splits;
  // work units: single tiles, or M-tile pairs processed by a 2-CTA cluster
  uint32_t rank = 0;
  if (p.pair) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int num_units = (p.pair ? (p.tiles_m + 1) / 2 : p.tiles_m) * p.tiles_n * p.tiles_img;
  const int unit0 = p.pair ? (int)(blockIdx.x / 2) : (int)blockIdx.x;
  const int unit_step = p.pair ? (int)(gridDim.x / 2) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], p.pair ? 2 : 1);  // pair: both CTAs' MMAs release the stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], EPI_WARPS);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (p.pair) cluster_sync();  // peer barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer =================
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = unit0; unit < num_units; unit += unit_step) {
        int tm, tn, ti;
        tile_coords(p, unit, tm, tn, ti);
        if (p.pair) tm = 2 * tm + (int)rank;
        KbWalk w;
        w.start(p, 0, kblocks);
        // per-unit parts of the B coordinates (kblock_coords)
        const int pix0 = ti * p.H * p.W + tn * BN, a1 = tm * BM;
        for (int kb = 0; kb < total_kb; ++kb, w.next(p, kblocks)) {
          mbar_wait(&empty[stage], phase ^ 1);
          const int sa = w.sel_a(p), sb = w.sel_b();
          const int a0 = w.k * BK;
          int b0, b1;
          if (p.conv == 0) {
            b0 = tn * BN;
            b1 = w.k * BK;
          } else if (p.conv == 3) {
            b0 = w.k * BK;
            b1 = tn * BN;
          } else if (p.conv == 1) {
            b0 = w.c0;
            b1 = pix0 + w.r * p.W + w.s;
          } else {
            b0 = tn * BN;
            b1 = ti * p.Cin + w.c0;
          }
          uint8_t* sA = smem + stage * STAGE_BYTES;
          uint8_t* sB = sA + A_BYTES;
          if (p.conv == 5) {
            // 1x1 with pixels as M: A = this tile's 128 pixels x 32 channels of the
            // [N*C][H*W] input (MN-major: 4 chunks of 32 pixels), B = bn filters x 32
            // channels of the [K][C] weights (K-major)
            mbar_expect_tx(&full[stage], A_BYTES + p.bn * BK * 4);
            if (p.b3d)
              tma_load_3d(sA, &maps.a[sa], &full[stage], 0, ti * p.Cin + w.c0, a1 >> 5);
            else
              for (int j = 0; j < BM / 32; ++j)
                tma_load_2d(sA + j * (BK * 128), &maps.a[sa], &full[stage], a1 + 32 * j, ti * p.Cin + w.c0);
            tma_load_2d(sB, &maps.b[sb], &full[stage], w.c0, tn * p.bn);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(sA, &maps.a[sa], &full[stage], a0, a1);
          if (p.conv == 1) {
            // K-major: 256 pixel rows x 32 channels (128 B) in one box
            tma_load_2d(sB, &maps.b[sb], &full[stage], b0, b1);
          } else if (p.conv == 3) {
            // K-major B in two boxes of 128 rows; a pair multicasts one half each
            if (p.pair)
              tma_load_2d_mc(sB + rank * (BN / 2) * 128, &maps.b[sb], &full[stage], b0, b1 + (int)rank * (BN / 2),
                             0x3);
            else
              for (int h = 0; h < 2; ++h)
                tma_load_2d(sB + h * (BN / 2) * 128, &maps.b[sb], &full[stage], b0, b1 + h * (BN / 2));
          } else if (p.b3d) {
            // MN-major B as one 3-D box of chunks (pair: this CTA's half, multicast)
            if (p.pair)
              tma_load_3d_mc(sB + rank * (BN / 64) * (BK * 128), &maps.b[sb], &full[stage], 0, b1,
                             (b0 >> 5) + (int)rank * (BN / 64), 0x3);
            else
              tma_load_3d(sB, &maps.b[sb], &full[stage], 0, b1, b0 >> 5);
          } else if (p.pair) {
            // MN-major B shared by the pair: this CTA loads half of the 8 chunks and
            // multicasts them into both CTAs' smem (each CTA's full barrier expects
            // its A plus all of B)
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) {
              const int jj = (int)rank * (BN / 64) + j;
              tma_load_2d_mc(sB + jj * (BK * 128), &maps.b[sb], &full[stage], b0 + 32 * jj, b1, 0x3);
            }
          } else {
            // MN-major: 8 chunks of [32 K rows x 32 N]
#pragma unroll
            for (int j = 0; j < BN / 32; ++j)
              tma_load_2d(sB + j * (BK * 128), &maps.b[sb], &full[stage], b0 + 32 * j, b1);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (p.pair) {
        // tail: wait until both CTAs' MMAs released every stage, so no remote
        // arrive is still in flight towards this CTA's barriers at exit
        for (int i = 0; i < STAGES; ++i) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer =================
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      // mode 5 swaps the majors: A (pixels) MN-major, B (filters) K-major, N = bn
      const bool a_mn = p.conv == 5, b_kmajor = p.conv == 1 || p.conv == 3 || p.conv == 5;
      const uint32_t a_base = smem_u32(smem);
      const uint64_t adesc0 = a_mn ? make_desc(a_base, BK * 128, 512, kSw128Base32) : make_desc(a_base, 16, 1024, kSw128);
      const uint64_t bdesc0 = b_kmajor ? make_desc(a_base + A_BYTES, 16, 1024, kSw128)
                                       : make_desc(a_base + A_BYTES, BK * 128, 512, kSw128Base32);
      const uint32_t astep = a_mn ? 64u : 2u, bstep = b_kmajor ? 2u : 64u;  // (32 B | 1 KB) >> 4 per K = 8
      const uint32_t idesc = a_mn ? idesc_tf32_n(1, 0, (uint32_t)p.bn) : b_kmajor ? idesc_tf32(0) : idesc_tf32(1);
      for (int unit = unit0; unit < num_units; unit += unit_step) {
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < total_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          // the stage's descriptors: the base descriptors plus the stage offset (>> 4)
          const uint64_t soff = (uint64_t)((stage * STAGE_BYTES) >> 4);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            // A: K-major SW128, +32 B per K=8 step inside the 128 B atom; SBO = 8 rows * 128 B
            // B (sgemm): MN-major SW128 with 32 B atoms: chunks of 32 N at LBO = 32 rows *
            // 128 B, 4-row K groups at SBO = 512 B; +8 rows (1 KB) per K step.
            // B (conv): K-major SW128 like A.
            mma_tf32(d_tmem, adesc0 + soff + (uint64_t)(kk * astep), bdesc0 + soff + (uint64_t)(kk * bstep),
                     idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          // smem stage free once these MMAs complete (pair: in both CTAs)
          if (p.pair)
            mma_commit_mc(&empty[stage], 0x3);
          else
            mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tmem_full[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue =================
    const int q = (warp - 4) % 4;        // TMEM lanes 32q .. 32q+31 (a warp reaches quadrant warp % 4)
    const int half = (warp - 4) / 4;     // columns [half * BN/2, (half + 1) * BN/2)
    // 1024-aligned per-warp staging (the TMA store buffer needs the 128B-swizzle alignment)
    float* stg = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 1024) + (warp - 4) * kEpiStride;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int unit = unit0; unit < num_units; unit += unit_step) {
      int tm, tn, ti;
      tile_coords(p, unit, tm, tn, ti);
      if (p.pair) tm = 2 * tm + (int)rank;
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      // gemm / 1x1: each lane stores its row's 32 contiguous columns as float4s.
      // conv on the input grid (gaps at x >= OW): each 32x32 sub-tile goes TMEM ->
      // registers (lane = row) -> shared memory -> registers (lane = column), so a
      // store instruction writes consecutive pixels of one output row
      const int row0 = tm * BM + q * 32;
      if (p.conv == 5) {
        // lane = output pixel, register v = filter: each store writes 32 consecutive
        // pixels of one filter's output plane (128 B)
        const int64_t ohw = p.N;
        const int px = row0 + lane, f0 = tn * p.bn;
        float* dst = p.C + ((int64_t)ti * p.M + f0) * ohw + px;
#pragma unroll 1
        for (int c0 = 0; c0 < p.bn && f0 + c0 < p.M; c0 += 32) {
          uint32_t r[32];
          TMEM_LD_32x32b_x32(tmem_base + acc * BN + c0 + ((uint32_t)(q * 32) << 16), r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (px < ohw) {
            float* d = dst + (int64_t)c0 * ohw;
            if (f0 + c0 + 32 <= p.M) {
#pragma unroll
              for (int v = 0; v < 32; ++v, d += ohw) *d = __uint_as_float(r[v]);
            } else {
              const int nv = p.M - f0 - c0;
#pragma unroll
              for (int v = 0; v < 32; ++v, d += ohw)
                if (v < nv) __stcs(d, __uint_as_float(r[v]));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tmem_empty[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
#pragma unroll 1
      constexpr int kColSpan = BN / (EPI_WARPS / 4);  // columns per epilogue warp
      for (int c0 = half * kColSpan; c0 < (half + 1) * kColSpan; c0 += 32) {
        // rows past M: nothing to store (a TMA store would clip only at the tensor's
        // edge, and in the 1x1 [N*K][OH*OW] view rows past M belong to the next image)
        if (row0 >= p.M) continue;
        uint32_t r[32];
        const uint32_t taddr = tmem_base + acc * BN + c0 + ((uint32_t)(q * 32) << 16);
        TMEM_LD_32x32b_x32(taddr, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (p.tma_store) {
          // registers -> this warp's 4 KB buffer in the TMA 128B-swizzle layout (16 B
          // chunk j of row `lane` at chunk j ^ (lane & 7): conflict-free STS.128) ->
          // one bulk tensor store of the 32x32 sub-tile (full-line writes; edges clipped)
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(stg + lane * 32 + ((j ^ (lane & 7)) * 4)) =
                make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                            __uint_as_float(r[4 * j + 3]));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            tma_store_2d(&maps.c, stg, tn * BN + c0, (p.conv == 2 ? ti * p.M : 0) + row0);
          continue;
        }
        if (p.conv != 1) {
          // gemm rows / 1x1 image rows: 128 contiguous bytes per lane, float4 stores
          const int row = row0 + lane;
          const int col0 = tn * BN + c0;
          const int64_t ncols = (p.conv == 2) ? (int64_t)p.OH * p.OW : p.N;
          const int64_t pitch = (p.conv == 2) ? ncols : p.ldc;
          float* dst = p.C + ((p.conv == 2) ? ((int64_t)ti * p.M + row) * ncols : (int64_t)row * pitch) + col0;
          if (row < p.M) {
            if (col0 + 32 <= ncols && (pitch & 3) == 0) {
#pragma unroll
              for (int v = 0; v < 32; v += 4)
                *reinterpret_cast<float4*>(dst + v) = make_float4(__uint_as_float(r[v]), __uint_as_float(r[v + 1]),
                                                                  __uint_as_float(r[v + 2]), __uint_as_float(r[v + 3]));
            } else {
              for (int v = 0; v < 32; ++v)
                if (col0 + v < ncols) dst[v] = __uint_as_float(r[v]);
            }
          }
          continue;
        }
#pragma unroll
        for (int v = 0; v < 32; ++v) stg[lane * 33 + v] = __uint_as_float(r[v]);
        __syncwarp();
        const int col = tn * BN + c0 + lane;  // this lane's output column
        bool ok;
        int64_t off, rstride;  // element of (row0, col), distance between rows
        if (p.conv == 0 || p.conv == 3) {
          ok = col < p.N;
          off = (int64_t)row0 * p.ldc + col;
          rstride = p.ldc;
        } else if (p.conv == 1) {
          // pixels of the whole batch back to back (P = img*H*W + y*W + x) on the input grid
          const int hw = p.H * p.W;
          const int img = col / hw, rem = col - img * hw, y = rem / p.W, x = rem - (rem / p.W) * p.W;
          rstride = (int64_t)p.OH * p.OW;
          ok = img < p.img && y < p.OH && x < p.OW;
          off = ((int64_t)img * p.M + row0) * rstride + (int64_t)y * p.OW + x;
        } else {
          // 1x1 on one image: every pixel is an output
          rstride = (int64_t)p.OH * p.OW;
          ok = col < rstride;
          off = ((int64_t)ti * p.M + row0) * rstride + col;
        }
        const int rows = min(32, p.M - row0);
        if (ok)
          for (int i = 0; i < rows; ++i) p.C[off + (int64_t)i * rstride] = stg[i * 33 + lane];
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  if (p.tma_store && warp >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (p.pair) cluster_sync();  // no multicast or remote arrive may still target this CTA
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
}

// One 32x32 accumulator sub-tile (lane = row row0 + lane, columns c0..c0+31 of
// tile column tn) from registers to global: TMA bulk store (p.tma_store), the
// smem-transposed path for conv on the input grid, or per-row stores.
__device__ __forceinline__ void epilogue_chunk(const Problem& p, const Maps& maps, const uint32_t (&r)[32], float* stg,
                                               int lane, int row0, int tn, int ti, int c0) {
  if (p.tma_store) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<float4*>(stg + lane * 32 + ((j ^ (lane & 7)) * 4)) =
          make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                      __uint_as_float(r[4 * j + 3]));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) tma_store_2d(&maps.c, stg, tn * BN + c0, (p.conv == 2 ? ti * p.M : 0) + row0);
    return;
  }
  if (p.conv == 4) {
    // compact output pixels q = n*OH*OW + oh*OW + ow: contiguous within an image
#pragma unroll
    for (int v = 0; v < 32; ++v) stg[lane * 33 + v] = __uint_as_float(r[v]);
    __syncwarp();
    const int q = tn * BN + c0 + lane;
    const int64_t ohw = (int64_t)p.OH * p.OW;
    const int n = (int)(q / ohw);
    const bool ok = n < p.img;
    const int64_t off = ((int64_t)n * p.M + row0) * ohw + (q - n * ohw);
    const int rows = min(32, p.M - row0);
    if (ok && p.ksplit > 1)
      for (int i = 0; i < rows; ++i) atomicAdd(p.C + off + (int64_t)i * ohw, stg[i * 33 + lane]);
    else if (ok)
      for (int i = 0; i < rows; ++i) p.C[off + (int64_t)i * ohw] = stg[i * 33 + lane];
    __syncwarp();
    return;
  }
  if (p.conv == 1) {
#pragma unroll
    for (int v = 0; v < 32; ++v) stg[lane * 33 + v] = __uint_as_float(r[v]);
    __syncwarp();
    const int col = tn * BN + c0 + lane;
    const int hw = p.H * p.W;
    const int img = col / hw, rem = col - img * hw, y = rem / p.W, x = rem - (rem / p.W) * p.W;
    const int64_t rstride = (int64_t)p.OH * p.OW;
    const bool ok = img < p.img && y < p.OH && x < p.OW;
    const int64_t off = ((int64_t)img * p.M + row0) * rstride + (int64_t)y * p.OW + x;
    const int rows = min(32, p.M - row0);
    if (ok)
      for (int i = 0; i < rows; ++i) p.C[off + (int64_t)i * rstride] = stg[i * 33 + lane];
    __syncwarp();
    return;
  }
  const int row = row0 + lane, col0 = tn * BN + c0;
  const int64_t ncols = (p.conv == 2) ? (int64_t)p.OH * p.OW : p.N;
  const int64_t pitch = (p.conv == 2) ? ncols : p.ldc;
  if (row < p.M) {
    float* dst = p.C + ((p.conv == 2) ? ((int64_t)ti * p.M + row) * ncols : (int64_t)row * pitch) + col0;
    for (int v = 0; v < 32; ++v)
      if (col0 + v < ncols) dst[v] = __uint_as_float(r[v]);
  }
}

// ---------------------------------------------------------------------------
// k_tc_gemm2: the sgemm on CTA pairs with tcgen05.mma.cta_group::2 (M = 256 per
// pair, N = 256).  Each CTA of the pair holds its 128 rows of A and its 128
// columns of B per stage (32 KB, 6 stages); the leader (rank 0) issues the MMAs,
// which read A from each CTA's own shared memory and B from both; each CTA's TMEM
// holds its 128 rows x 256 columns of the accumulator.  Both CTAs' TMA loads
// signal the leader's `full` barrier (.cta_group::2); MMA commits arrive on both
// CTAs' `empty` / `tmem_full` barriers (multicast); both CTAs' epilogue warps
// arrive on the leader's `tmem_empty`.
constexpr int STAGES2 = 6;
constexpr int B2_BYTES = (BN / 2) * BK * 4;  // 16 KB: this CTA's half of the B tile
constexpr int STAGE2_BYTES = A_BYTES + B2_BYTES;
constexpr int SMEM2_BYTES = STAGES2 * STAGE2_BYTES + 1024 /*align*/ + 1024 /*barriers*/ + EPI_WARPS * kEpiStride * 4;

__device__ __forceinline__ uint32_t peer_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
// im2col-mode TMA (conv, mode 4): pixelsPerColumn consecutive OUTPUT pixels starting
// at (n, oh, ow) — traversal clipped to the valid-output box of the map — each
// shifted by the filter tap (s, r), x 32 channels from c, into K-major rows.
__device__ __forceinline__ void tma_load_3d_2sm(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_im2col_2sm(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c,
                                                    int w, int h, int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w), "h"(off_h)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
__host__ __device__ constexpr uint32_t idesc_tf32_m256(uint32_t b_mn_major) {  // M = 256 (cta_group::2), N = 256
  return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (b_mn_major << 16) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(256 >> 4) << 24);
}

// 256-row units: 8 per raster group (~sqrt of the units in flight: the fewest
// distinct A + B panels per wave)
constexpr int kGroup2 = 8;

__global__ void __launch_bounds__(NUM_THREADS, 1) k_tc_gemm2(const __grid_constant__ Maps maps, const Problem p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES2 * STAGE2_BYTES);
  uint64_t* empty = full + STAGES2;
  uint64_t* tmem_full = empty + STAGES2;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kblocks = (p.conv == 1 || p.conv == 2 || p.conv == 4 ? p.R * p.S * (p.K / BK) : (p.K + BK - 1) / BK);
  const int total_kb = kblocks * p.splits;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tiles_m2 = (p.tiles_m + 1) / 2;  // 256-row tiles
  const int ks_n = p.ksplit > 1 ? p.ksplit : 1;  // unit = tile * ks_n + k-part
  const int kb_per = total_kb / ks_n;
  const int num_units = tiles_m2 * p.tiles_n * p.tiles_img * ks_n;
  const int unit0 = (int)(blockIdx.x / 2), unit_step = (int)(gridDim.x / 2);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's arrive + both CTAs' bytes
      mbar_init(&empty[s], 1);  // the leader's MMA commit (multicast)
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 2 * EPI_WARPS);  // leader: both CTAs' epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer (both CTAs) =================
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full_leader = peer_addr(smem_u32(&full[0]), 0);
      for (int unit = unit0; unit < num_units; unit += unit_step) {
        int tm2, tn, ti;
        {
          Problem q = p;
          q.tiles_m = tiles_m2;
          q.pair = 0;
          tile_coords(q, unit / ks_n, tm2, tn, ti, kGroup2);
        }
        const int tm = 2 * tm2 + (int)rank;  // this CTA's 128 rows
        const int kb0 = (unit % ks_n) * kb_per;
        // per-unit parts of the coordinates: im2col's first output pixel of this CTA's
        // 128 (compact, across images), the input-grid pixel row, the A row
        int n0 = 0, oh0 = 0, ow0 = 0;
        if (p.conv == 4) {
          const int ohw = p.OH * p.OW, q0 = tn * BN + (int)rank * (BN / 2);
          n0 = q0 / ohw;
          const int rem = q0 - n0 * ohw;
          oh0 = rem / p.OW;
          ow0 = rem - oh0 * p.OW;
        }
        const int pix0 = ti * p.H * p.W + tn * BN + (int)rank * (BN / 2), a1 = tm * BM;
        KbWalk w;
        w.start(p, kb0, kblocks);
        for (int kb = kb0; kb < kb0 + kb_per; ++kb, w.next(p, kblocks)) {
          mbar_wait(&empty[stage], phase ^ 1);
          const int sa = w.sel_a(p), sb = w.sel_b();
          uint8_t* sA = smem + stage * STAGE2_BYTES;
          uint8_t* sB = sA + A_BYTES;
          const uint32_t bar = full_leader + stage * 8;  // the leader's barrier
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * STAGE2_BYTES);
          tma_load_2d_2sm(sA, &maps.a[sa], bar, w.k * BK, a1);
          if (p.conv == 4) {
            // im2col: this CTA's 128 output pixels at tap (r, s), channels c0 .. c0 + 31
            tma_load_im2col_2sm(sB, &maps.b[sb], bar, w.c0, ow0, oh0, n0, (uint16_t)w.s, (uint16_t)w.r);
          } else if (p.conv == 1) {
            // K-major: this CTA's 128 pixel rows x 32 channels in one box
            tma_load_2d_2sm(sB, &maps.b[sb], bar, w.c0, pix0 + w.r * p.W + w.s);
          } else if (p.b3d) {
            // this CTA's 4 chunks of 32 columns in one 3-D box
            tma_load_3d_2sm(sB, &maps.b[sb], bar, 0, w.k * BK, (tn * BN + (int)rank * (BN / 2)) >> 5);
          } else {
            const int b0 = tn * BN + (int)rank * (BN / 2);
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)  // MN-major: this CTA's 4 chunks of 32 columns
              tma_load_2d_2sm(sB + j * (BK * 128), &maps.b[sb], bar, b0 + 32 * j, w.k * BK);
          }
          if (++stage == STAGES2) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // tail: every stage released by the MMAs before exit
      for (int i = 0; i < STAGES2; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (++stage == STAGES2) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ================= MMA issuer (leader) =================
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const bool b_kmajor = p.conv == 1 || p.conv == 4;
      const uint32_t a_base = smem_u32(smem);
      const uint64_t adesc0 = make_desc(a_base, 16, 1024, kSw128);
      const uint64_t bdesc0 = b_kmajor ? make_desc(a_base + A_BYTES, 16, 1024, kSw128)
                                       : make_desc(a_base + A_BYTES, BK * 128, 512, kSw128Base32);
      const uint32_t bstep = b_kmajor ? 2u : 64u;
      const uint32_t idesc = idesc_tf32_m256(b_kmajor ? 0u : 1u);
      for (int unit = unit0; unit < num_units; unit += unit_step) {
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int kb0 = (unit % ks_n) * kb_per;
        for (int kb = kb0; kb < kb0 + kb_per; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t soff = (uint64_t)((stage * STAGE2_BYTES) >> 4);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk)
            mma_tf32_2sm(d_tmem, adesc0 + soff + (uint64_t)(kk * 2), bdesc0 + soff + (uint64_t)(kk * bstep), idesc,
                         (kb > kb0 || kk > 0) ? 1u : 0u);
          mma_commit_2sm(&empty[stage]);  // both CTAs' stage buffers free once these complete
          if (++stage == STAGES2) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_2sm(&tmem_full[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue (both CTAs: own 128 rows) =================
    const int q = (warp - 4) % 4;
    float* stg = reinterpret_cast<float*>(smem + STAGES2 * STAGE2_BYTES + 1024) + (warp - 4) * kEpiStride;
    const uint32_t empty_leader = peer_addr(smem_u32(&tmem_empty[0]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int unit = unit0; unit < num_units; unit += unit_step) {
      int tm2, tn, ti;
      {
        Problem q2 = p;
        q2.tiles_m = tiles_m2;
        q2.pair = 0;
        tile_coords(q2, unit / ks_n, tm2, tn, ti, kGroup2);
      }
      const int tm = 2 * tm2 + (int)rank;
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const int row0 = tm * BM + q * 32;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        const uint32_t taddr = tmem_base + acc * BN + c0 + ((uint32_t)(q * 32) << 16);
        TMEM_LD_32x32b_x32(taddr, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        epilogue_chunk(p, maps, r, stg, lane, row0, tn, ti, c0);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(empty_leader + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  if (p.tma_store && warp >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
}

// hi/lo split for 3xTF32: hi = x with the 13 low mantissa bits cleared (exactly
// representable in TF32), lo = x - hi (exact in FP32).
__global__ void k_split_tf32(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    hi[i] = h;
    lo[i] = v - h;
  }
}

// KCRS -> K(RS)C weight reorder (tiny), optionally split into hi/lo.
__global__ void k_weights_krsc(const float* __restrict__ w, float* __restrict__ hi, float* __restrict__ lo, int K,
                               int C, int R, int S) {
  const int64_t n = (int64_t)K * C * R * S;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    // i indexes the destination [k][r][s][c]
    int64_t t = i;
    const int c = (int)(t % C); t /= C;
    const int s = (int)(t % S); t /= S;
    const int r = (int)(t % R);
    const int k = (int)(t / R);
    const float v = w[(((int64_t)k * C + c) * R + r) * S + s];
    if (lo) {
      const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
      hi[i] = h;
      lo[i] = v - h;
    } else {
      hi[i] = v;
    }
  }
}

// Copies a [rows][cols] fp32 matrix into a row pitch that TMA accepts (16 B).
__global__ void k_pitch_copy(const float* __restrict__ src, float* __restrict__ dst, int64_t rows, int64_t cols,
                             int64_t dpitch) {
  const int64_t n = rows * dpitch;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / dpitch, c = i - r * dpitch;
    dst[i] = c < cols ? src[r * cols + c] : 0.0f;
  }
}

// NCHW -> NHWC, optionally split into TF32 hi/lo (3xTF32).  Block (32, 8): a
// [32 channels x 128 pixels] slab through padded shared memory — 16 coalesced 128 B
// loads in flight per thread along pixels, then 128 B stores along channels.
constexpr int kTP = 128;  // pixels per transpose block
__global__ void __launch_bounds__(256) k_nchw_to_nhwc(const float* __restrict__ in, float* __restrict__ hi,
                                                      float* __restrict__ lo, int C, int64_t HW) {
  __shared__ float tile[32][kTP + 1];
  const int64_t p0 = (int64_t)blockIdx.x * kTP;
  const int c0 = blockIdx.y * 32;
  const int64_t img = blockIdx.z;
  const float* src = in + (img * C + c0) * HW + p0;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int np = HW - p0 < kTP ? (int)(HW - p0) : kTP;
  float v[4][kTP / 32];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < kTP / 32; ++j) {
      const int q = j * 32 + tx;
      v[i][j] = q < np ? __ldcs(src + (int64_t)(ty + 8 * i) * HW + q) : 0.0f;
    }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < kTP / 32; ++j) tile[ty + 8 * i][j * 32 + tx] = v[i][j];
  __syncthreads();
  float* dh = hi + (img * HW + p0) * C + c0 + tx;
  float* dl = lo ? lo + (img * HW + p0) * C + c0 + tx : nullptr;
#pragma unroll 4
  for (int py = ty; py < np; py += 8) {
    const float x = tile[tx][py];
    if (dl) {
      const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
      dh[(int64_t)py * C] = h;
      dl[(int64_t)py * C] = x - h;
    } else {
      dh[(int64_t)py * C] = x;
    }
  }
}

// KCRS -> KRSC: block (k*R*S + rs, c-chunk) gathers tap rs of filter k for 256
// channels (stride R*S reads inside the filter's contiguous weights, L2-resident) and
// writes them contiguously; optionally split into hi/lo.
__global__ void __launch_bounds__(256) k_weights_krsc_tap(const float* __restrict__ w, float* __restrict__ hi,
                                                          float* __restrict__ lo, int C, int RS) {
  const int k = blockIdx.x / RS, rs = blockIdx.x - (blockIdx.x / RS) * RS;
  const int c = blockIdx.y * 256 + threadIdx.x;
  if (c >= C) return;
  const float x = __ldg(w + ((int64_t)k * C + c) * RS + rs);
  const int64_t o = ((int64_t)k * RS + rs) * C + c;
  if (lo) {
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    hi[o] = h;
    lo[o] = x - h;
  } else {
    hi[o] = x;
  }
}

}  // namespace tc
}  // namespace atc

using namespace atc::tc;

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode(atc_ctx* ctx) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn) return fn;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p) {
    atc_set_error(ctx, "cuTensorMapEncodeTiled is unavailable");
    return nullptr;
  }
  fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  return fn;
}

// im2col map over an NHWC fp32 tensor [n][h][w][c]: boxes of `pixels` consecutive
// valid-output pixels (the traversal box excludes the last r-1 rows and s-1
// columns of each image) x 32 channels, 128B swizzle (K-major rows like make_map).
bool make_im2col_map(atc_ctx* ctx, CUtensorMap* m, const float* base, int64_t n, int64_t h, int64_t w, int64_t c,
                     int r, int s, uint32_t pixels) {
  static PFN_cuTensorMapEncodeIm2col_v12000 enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p) {
      atc_set_error(ctx, "cuTensorMapEncodeIm2col is unavailable");
      return false;
    }
    enc = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
  }
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)c * 4, (cuuint64_t)(w * c) * 4, (cuuint64_t)(h * w * c) * 4};
  int lower[2] = {0, 0};
  int upper[2] = {-(s - 1), -(r - 1)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult res = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, lower, upper,
                     (cuuint32_t)BK, pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (res != CUDA_SUCCESS) {
    atc_set_error(ctx, "cuTensorMapEncodeIm2col failed (%d)", (int)res);
    return false;
  }
  return true;
}

// 2-D fp32 tensor map over [rows][cols] with row pitch `pitch` elements.
bool make_map(atc_ctx* ctx, CUtensorMap* m, const float* base, uint64_t rows, uint64_t cols, uint64_t pitch,
              uint32_t box_cols, uint32_t box_rows, bool mn_major) {
  auto enc = get_encode(ctx);
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    atc_set_error(ctx, "cuTensorMapEncodeTiled failed (%d) for [%llu x %llu] pitch %llu", (int)r,
                  (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)pitch);
    return false;
  }
  return true;
}

// MN-major [rows][cols] fp32 (cols % 32 == 0) as a 3-D map {32 columns, rows, cols / 32
// chunks}: one box of `chunks` [box_rows x 32] chunks lands chunk-major in shared
// memory, the layout of `chunks` separate 2-D chunk loads.
bool make_map_mn3(atc_ctx* ctx, CUtensorMap* m, const float* base, uint64_t rows, uint64_t cols, uint64_t pitch,
                  uint32_t box_rows, uint32_t chunks) {
  auto enc = get_encode(ctx);
  if (!enc) return false;
  cuuint64_t dims[3] = {32, rows, cols / 32};
  cuuint64_t strides[2] = {pitch * 4, 128};
  cuuint32_t box[3] = {32, box_rows, chunks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    atc_set_error(ctx, "cuTensorMapEncodeTiled (3-D) failed (%d) for [%llu x %llu] pitch %llu", (int)r,
                  (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)pitch);
    return false;
  }
  return true;
}

// Kernel-variant switches (context option ATC_OPT_TC_FLAGS, A/B checks):
// ATC_TC_NO_KSPLIT never splits K, ATC_TC_NO_2SM disables the cta_group::2 kernel,
// ATC_TC_NO_TMA_STORE the TMA-store epilogue, ATC_TC_NO_PAIR the 1-SM kernel's
// B multicast across a CTA pair, ATC_TC_NO_IM2COL the im2col-mode conv B operand;
// ATC_TC_B_KMAJOR transposes the sgemm B to K-major once; ATC_TC_NO_B3D loads the
// sgemm's MN-major B as separate 2-D chunk boxes; ATC_TC_NO_SWAP1X1 keeps
// 1x1 convolutions in the filters-as-M form (mode 2).
bool tc_flag(const atc_ctx* ctx, int f) { return (ctx->opt_tc_flags & f) != 0; }

// CTA pairs need an MN-major B (loaded as chunks, half by each CTA) and >= 2
// M tiles
int use_pair(const atc_ctx* ctx, const Problem& p) {
  return !tc_flag(ctx, ATC_TC_NO_PAIR) && p.conv != 1 && p.conv != 5 && p.tiles_m >= 2 ? 1 : 0;
}

// the dynamic shared-memory opt-in of both GEMM kernels, once per context (the
// attribute is per device; every context of a device sets it)
bool configure_tc(atc_ctx* ctx) {
  if (ctx->tc_configured) return true;
  if (!atc_cuda_ok(ctx, cudaFuncSetAttribute(k_tc_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES),
                   "cudaFuncSetAttribute") ||
      !atc_cuda_ok(ctx, cudaFuncSetAttribute(k_tc_gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES),
                   "cudaFuncSetAttribute"))
    return false;
  ctx->tc_configured = true;
  return true;
}

bool launch(atc_ctx* ctx, const Maps& maps, const Problem& p, cudaStream_t st) {
  if (!configure_tc(ctx)) return false;
  if (p.umma2) {
    const int units = (p.tiles_m + 1) / 2 * p.tiles_n * (p.ksplit > 1 ? p.ksplit : 1);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(2 * std::min(units, ctx->sm_count / 2)));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = SMEM2_BYTES;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return atc_cuda_ok(ctx, cudaLaunchKernelEx(&cfg, k_tc_gemm2, maps, p), "k_tc_gemm2 cluster launch");
  }
  if (p.pair) {
    // 2-CTA clusters: one M-tile pair per cluster iteration, persistent over pairs
    const int units = (p.tiles_m + 1) / 2 * p.tiles_n * p.tiles_img;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(2 * std::min(units, ctx->sm_count / 2)));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return atc_cuda_ok(ctx, cudaLaunchKernelEx(&cfg, k_tc_gemm, maps, p), "k_tc_gemm cluster launch");
  }
  const int tiles = p.tiles_m * p.tiles_n * p.tiles_img;
  const int grid = std::min(tiles, ctx->sm_count);
  k_tc_gemm<<<grid, NUM_THREADS, SMEM_BYTES, st>>>(maps, p);
  return atc_cuda_ok(ctx, cudaGetLastError(), "k_tc_gemm launch");
}

int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 16); }

}  // namespace

extern "C" {

int atc_sgemm_rm_device(atc_ctx* ctx, const float* dA, const float* dB, float* dC, int64_t m, int64_t n, int64_t k,
                        int32_t precision, void* stream) {
  ATC_ENTER(ctx);
  if (m < 1 || n < 1 || k < 1 || m >= (1LL << 31) || n >= (1LL << 31) || k >= (1LL << 31) || !dA || !dB || !dC ||
      (precision != ATC_PREC_TF32 && precision != ATC_PREC_3XTF32)) {
    atc_set_error(ctx, "bad arguments to atc_sgemm_rm");
    return ATC_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
  // TMA needs 16-byte row pitches: repitch A ([m][k]) / B ([k][n]) when needed
  const int64_t kp = (k + 3) / 4 * 4, np = (n + 3) / 4 * 4;
  const float* A = dA;
  const float* B = dB;
  if (kp != k) {
    float* t = (float*)atc_ctx_scratch(ctx, 11, (size_t)m * kp * 4);
    if (!t) return ATC_ERR_CUDA;
    k_pitch_copy<<<grid_for(m * kp), 256, 0, st>>>(dA, t, m, k, kp);
    A = t;
  }
  if (np != n) {
    float* t = (float*)atc_ctx_scratch(ctx, 12, (size_t)k * np * 4);
    if (!t) return ATC_ERR_CUDA;
    k_pitch_copy<<<grid_for(k * np), 256, 0, st>>>(dB, t, k, n, np);
    B = t;
  }
  // ATC_TC_B_KMAJOR: B transposed once to [N][K] (K-major, like A) — A/B experiment
  const bool b_kmajor = tc_flag(ctx, ATC_TC_B_KMAJOR) && k % 32 == 0 && n % 32 == 0;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  Problem p{};
  p.conv = b_kmajor ? 3 : 0;
  p.M = (int)m;
  p.N = (int)n;
  p.K = (int)k;
  p.C = dC;
  p.ldc = n;
  p.tiles_m = (int)((m + BM - 1) / BM);
  p.tiles_n = (int)((n + BN - 1) / BN);
  p.tiles_img = 1;
  p.pair = use_pair(ctx, p);
  p.splits = precision == ATC_PREC_3XTF32 ? 3 : 1;
  // TMA-store epilogue when C's row pitch is a multiple of 16 bytes
  p.tma_store = !tc_flag(ctx, ATC_TC_NO_TMA_STORE) && (n % 4) == 0 ? 1 : 0;
  // cta_group::2 (M = 256 per CTA pair) for the MN-major sgemm
  p.umma2 = !tc_flag(ctx, ATC_TC_NO_2SM) && p.conv == 0 && p.tiles_m >= 2 ? 1 : 0;
  if (p.tma_store && !make_map(ctx, &maps.c, dC, m, n, n, 32, 32, false)) return ATC_ERR_CUDA;
  // one 3-D load per stage for B (4 chunks per CTA on the pair kernels, else 8)
  p.b3d = !b_kmajor && n % 32 == 0 && !tc_flag(ctx, ATC_TC_NO_B3D) ? 1 : 0;
  const uint32_t chunks = p.umma2 || p.pair ? BN / 64 : BN / 32;
  auto bmap = [&](CUtensorMap* mp, const float* base) {
    return p.b3d ? make_map_mn3(ctx, mp, base, k, n, np, BK, chunks) : make_map(ctx, mp, base, k, n, np, 32, BK, true);
  };
  if (b_kmajor) {
    float* bt = (float*)atc_ctx_scratch(ctx, 14, (size_t)k * n * 4 * (p.splits == 3 ? 2 : 1));
    if (!bt) return ATC_ERR_CUDA;
    float* btl = p.splits == 3 ? bt + k * n : nullptr;
    dim3 grid((unsigned)((n + kTP - 1) / kTP), (unsigned)(k / 32), 1u);
    k_nchw_to_nhwc<<<grid, dim3(32, 8), 0, st>>>(B, bt, btl, (int)k, n);  // [K][N] -> [N][K] (+ hi/lo)
    float* a_lo = nullptr;
    const float* a_hi = A;
    if (p.splits == 3) {
      float* ah = (float*)atc_ctx_scratch(ctx, 13, (size_t)m * kp * 4 * 2);
      if (!ah) return ATC_ERR_CUDA;
      a_lo = ah + m * kp;
      k_split_tf32<<<grid_for(m * kp), 256, 0, st>>>(A, ah, a_lo, m * kp);
      a_hi = ah;
    }
    if (!make_map(ctx, &maps.a[0], a_hi, m, k, kp, BK, BM, false) ||
        !make_map(ctx, &maps.b[0], bt, n, k, k, BK, BN / 2, false))
      return ATC_ERR_CUDA;
    maps.a[1] = maps.a[0];
    maps.b[1] = maps.b[0];
    if (p.splits == 3 && (!make_map(ctx, &maps.a[1], a_lo, m, k, kp, BK, BM, false) ||
                          !make_map(ctx, &maps.b[1], btl, n, k, k, BK, BN / 2, false)))
      return ATC_ERR_CUDA;
  } else if (p.splits == 3) {
    float* ah = (float*)atc_ctx_scratch(ctx, 13, (size_t)m * kp * 4 * 2);
    float* bh = (float*)atc_ctx_scratch(ctx, 14, (size_t)k * np * 4 * 2);
    if (!ah || !bh) return ATC_ERR_CUDA;
    float* al = ah + m * kp;
    float* bl = bh + k * np;
    k_split_tf32<<<grid_for(m * kp), 256, 0, st>>>(A, ah, al, m * kp);
    k_split_tf32<<<grid_for(k * np), 256, 0, st>>>(B, bh, bl, k * np);
    if (!make_map(ctx, &maps.a[0], ah, m, k, kp, BK, BM, false) || !make_map(ctx, &maps.a[1], al, m, k, kp, BK, BM, false) ||
        !bmap(&maps.b[0], bh) || !bmap(&maps.b[1], bl))
      return ATC_ERR_CUDA;
  } else {
    if (!make_map(ctx, &maps.a[0], A, m, k, kp, BK, BM, false) || !bmap(&maps.b[0], B))
      return ATC_ERR_CUDA;
    maps.a[1] = maps.a[0];
    maps.b[1] = maps.b[0];
  }
  return launch(ctx, maps, p, st) ? ATC_OK : ATC_ERR_CUDA;
}

int atc_sgemm_rm(atc_ctx* ctx, const float* A, const float* B, float* C, int64_t m, int64_t n, int64_t k,
                 int32_t precision) {
  ATC_ENTER(ctx);
  if (m < 1 || n < 1 || k < 1 || !A || !B || !C) {
    atc_set_error(ctx, "bad arguments to atc_sgemm_rm");
    return ATC_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  float* dA = (float*)atc_ctx_scratch(ctx, 8, (size_t)m * k * 4);
  float* dB = (float*)atc_ctx_scratch(ctx, 9, (size_t)k * n * 4);
  float* dC = (float*)atc_ctx_scratch(ctx, 10, (size_t)m * n * 4);
  if (!dA || !dB || !dC) {
    atc_set_error(ctx, "device allocation failed");
    return ATC_ERR_CUDA;
  }
  // large calls are pipelined over row chunks of A and C: B goes over first, then chunk
  // i's A rows (copy stream 1) -> its GEMM (the context's stream) -> its C rows (copy
  // stream 2), so the H2D of later chunks and the D2H of earlier ones overlap the
  // tensor-core work (and each other: the copy engines are full duplex).  With pageable
  // host buffers the copies serialise and the call behaves like the unchunked one.
  const size_t bytes = ((size_t)m * k + (size_t)k * n + (size_t)m * n) * 4;
  const int chunks = bytes >= (64u << 20) && m >= 4 * 256 ? 4 : 1;
  if (chunks == 1) {
    if (!atc_cuda_ok(ctx, cudaMemcpyAsync(dA, A, (size_t)m * k * 4, cudaMemcpyHostToDevice, st), "H2D A") ||
        !atc_cuda_ok(ctx, cudaMemcpyAsync(dB, B, (size_t)k * n * 4, cudaMemcpyHostToDevice, st), "H2D B"))
      return ATC_ERR_CUDA;
    int rc = atc_sgemm_rm_device(ctx, dA, dB, dC, m, n, k, precision, st);
    if (rc) return rc;
    if (!atc_cuda_ok(ctx, cudaMemcpyAsync(C, dC, (size_t)m * n * 4, cudaMemcpyDeviceToHost, st), "D2H C") ||
        !atc_cuda_ok(ctx, cudaStreamSynchronize(st), "sgemm sync"))
      return ATC_ERR_CUDA;
    return ATC_OK;
  }
  cudaStream_t cin = ctx->copy_stream[0], cout = ctx->copy_stream[1];
  cudaEvent_t ev[2 * 4 + 2] = {};
  for (auto& e : ev)
    if (!atc_cuda_ok(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate")) return ATC_ERR_CUDA;
  cudaEvent_t e_start = ev[8], e_b = ev[9];
  bool ok = atc_cuda_ok(ctx, cudaEventRecord(e_start, st), "cudaEventRecord");  // after earlier work on st
  ok = ok && atc_cuda_ok(ctx, cudaStreamWaitEvent(cin, e_start, 0), "wait") &&
       atc_cuda_ok(ctx, cudaMemcpyAsync(dB, B, (size_t)k * n * 4, cudaMemcpyHostToDevice, cin), "H2D B") &&
       atc_cuda_ok(ctx, cudaEventRecord(e_b, cin), "cudaEventRecord") &&
       atc_cuda_ok(ctx, cudaStreamWaitEvent(st, e_b, 0), "wait");
  const int64_t step = (m / chunks + 255) / 256 * 256;
  int rc = ATC_OK;
  for (int c = 0; c < chunks && ok && rc == ATC_OK; ++c) {
    const int64_t r0 = c * step, r1 = std::min<int64_t>(m, r0 + step);
    if (r1 <= r0) break;
    const int64_t mr = r1 - r0;
    ok = atc_cuda_ok(ctx, cudaMemcpyAsync(dA + r0 * k, A + r0 * k, (size_t)mr * k * 4, cudaMemcpyHostToDevice, cin),
                     "H2D A") &&
         atc_cuda_ok(ctx, cudaEventRecord(ev[2 * c], cin), "cudaEventRecord") &&
         atc_cuda_ok(ctx, cudaStreamWaitEvent(st, ev[2 * c], 0), "wait");
    if (!ok) break;
    rc = atc_sgemm_rm_device(ctx, dA + r0 * k, dB, dC + r0 * n, mr, n, k, precision, st);
    ok = ok && rc == ATC_OK && atc_cuda_ok(ctx, cudaEventRecord(ev[2 * c + 1], st), "cudaEventRecord") &&
         atc_cuda_ok(ctx, cudaStreamWaitEvent(cout, ev[2 * c + 1], 0), "wait") &&
         atc_cuda_ok(ctx, cudaMemcpyAsync(C + r0 * n, dC + r0 * n, (size_t)mr * n * 4, cudaMemcpyDeviceToHost, cout),
                     "D2H C");
  }
  ok = ok && atc_cuda_ok(ctx, cudaStreamSynchronize(cout), "sgemm sync") &&
       atc_cuda_ok(ctx, cudaStreamSynchronize(st), "sgemm sync");
  for (auto& e : ev) cudaEventDestroy(e);
  if (rc) return rc;
  return ok ? ATC_OK : ATC_ERR_CUDA;
}

int atc_conv2d_nchw_device(atc_ctx* ctx, const float* d_in, const float* d_w, float* d_out, int64_t n, int64_t c,
                           int64_t h, int64_t w_, int64_t k, int64_t r, int64_t s, int32_t precision, void* stream) {
  ATC_ENTER(ctx);
  const int64_t oh = h - r + 1, ow = w_ - s + 1;
  if (n < 1 || c < 1 || h < 1 || w_ < 1 || k < 1 || r < 1 || s < 1 || oh < 1 || ow < 1 || !d_in || !d_w || !d_out ||
      (precision != ATC_PREC_TF32 && precision != ATC_PREC_3XTF32)) {
    atc_set_error(ctx, "bad arguments to atc_conv2d_nchw");
    return ATC_ERR_ARG;
  }
  if (c % BK != 0 || n * c >= (1LL << 31) || n * h * w_ >= (1LL << 31) - (1LL << 20)) {
    atc_set_error(ctx, "atc_conv2d_nchw: C must be a multiple of %d (got %lld)", BK, (long long)c);
    return ATC_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
  const int64_t hw = h * w_;
  const int splits = precision == ATC_PREC_3XTF32 ? 3 : 1;
  // NCHW -> NHWC once per call (one read + one write of the input; fused with
  // the hi/lo split in 3xTF32 mode).  Channels-innermost makes the conv's B
  // operand K-major, so the (r, s) pixel shift is a row offset of a 2-D TMA box
  // (any offset is legal) instead of a sub-16-byte column offset (illegal for
  // swizzled TMA boxes).
  // 1x1 filters need no pixel shift: the NCHW input is used as is ([N*C][H*W]
  // view, MN-major B, like the sgemm), no transpose (conv mode 2)
  const int64_t in_elems = n * c * hw;
  const bool direct = r == 1 && s == 1 && hw % 4 == 0;
  const float* ih = d_in;
  const float* il = nullptr;
  if (!direct || splits == 3) {
    float* buf = (float*)atc_ctx_scratch(ctx, 16, (size_t)in_elems * 4 * (splits == 3 ? 2 : 1));
    if (!buf) return ATC_ERR_CUDA;
    float* lo = splits == 3 ? buf + in_elems : nullptr;
    if (direct) {
      k_split_tf32<<<grid_for(in_elems), 256, 0, st>>>(d_in, buf, lo, in_elems);
    } else {
      dim3 grid((unsigned)((hw + kTP - 1) / kTP), (unsigned)(c / 32), (unsigned)n);
      k_nchw_to_nhwc<<<grid, dim3(32, 8), 0, st>>>(d_in, buf, lo, (int)c, hw);
    }
    ih = buf;
    il = lo;
  }
  // 1x1 with the output pixels as M (mode 5): lane = pixel in TMEM, so the epilogue
  // stores 128 B runs of each filter's output plane straight from registers, and a
  // filter count below 128 is the MMA's N instead of a half-empty M tile.  Used where
  // the call is store-bound (few channels: 2-4 k-blocks per tile) or K < 128; with
  // many channels the filters-as-M form reads less of the weights per pixel
  // (tools/time_conv.py: conv2_x.a 64->64 0.068 vs 0.079 ms, conv2_x.c 64->256 0.198
  // vs 0.205, conv3_x.a 512->128 0.109 vs 0.095)
  const bool swap = direct && (k < BM || c <= 128) && !tc_flag(ctx, ATC_TC_NO_SWAP1X1);
  const int64_t wn = k * c * r * s;
  const float* wh = d_w;  // 1x1 KCRS is already [K][C]
  const float* wl = nullptr;
  if (!(direct && splits == 1)) {
    float* wbuf = (float*)atc_ctx_scratch(ctx, 15, (size_t)wn * 4 * 2);
    if (!wbuf) return ATC_ERR_CUDA;
    wl = splits == 3 ? wbuf + wn : nullptr;
    if (k * r * s < (1LL << 31))
      k_weights_krsc_tap<<<dim3((unsigned)(k * r * s), (unsigned)((c + 255) / 256)), 256, 0, st>>>(
          d_w, wbuf, const_cast<float*>(wl), (int)c, (int)(r * s));
    else
      k_weights_krsc<<<grid_for(wn), 256, 0, st>>>(d_w, wbuf, const_cast<float*>(wl), (int)k, (int)c, (int)r, (int)s);
    wh = wbuf;
  }
  if (swap) {
    Maps maps;
    std::memset(&maps, 0, sizeof maps);
    Problem p{};
    p.conv = 5;
    p.M = (int)k;
    p.N = (int)hw;
    p.K = (int)c;
    p.splits = splits;
    p.C = d_out;
    p.img = (int)n;
    p.Cin = (int)c;
    p.H = (int)h;
    p.W = (int)w_;
    p.R = p.S = 1;
    p.OH = (int)oh;
    p.OW = (int)ow;
    p.bn = (int)std::min<int64_t>(BN, (k + 31) / 32 * 32);
    p.tiles_m = (int)((hw + BM - 1) / BM);
    p.tiles_n = (int)((k + p.bn - 1) / p.bn);
    p.tiles_img = (int)n;
    p.b3d = hw % 32 == 0 && !tc_flag(ctx, ATC_TC_NO_B3D) ? 1 : 0;
    for (int i = 0; i < splits && i < 2; ++i) {
      const float* xi = i ? il : ih;
      const float* wi = i ? wl : wh;
      if (!(p.b3d ? make_map_mn3(ctx, &maps.a[i], xi, n * c, hw, hw, BK, BM / 32)
                  : make_map(ctx, &maps.a[i], xi, n * c, hw, hw, 32, BK, true)) ||
          !make_map(ctx, &maps.b[i], wi, k, c, c, BK, (uint32_t)p.bn, false))
        return ATC_ERR_CUDA;
    }
    if (splits == 1) {
      maps.a[1] = maps.a[0];
      maps.b[1] = maps.b[0];
    }
    // (bulk tensor stores of [32 filters x 32 pixels] boxes measured no faster than the
    // direct 128 B stores: conv2_x.c 0.203 vs 0.200 ms)
    return launch(ctx, maps, p, st) ? ATC_OK : ATC_ERR_CUDA;
  }
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  // cta_group::2 (M = 256 filters per CTA pair) when there are >= 2 filter tiles;
  // each CTA then loads half of the pixel rows (K-major box of BN/2 rows)
  const bool umma2 = !tc_flag(ctx, ATC_TC_NO_2SM) && k > BM && !direct;  // (1x1 direct: slower on the pair kernel)
  // im2col-mode TMA on the pair kernel: tiles of compact output pixels (no input-grid
  // waste); ATC_TC_NO_IM2COL keeps the input-grid formulation
  const bool im2col = umma2 && !tc_flag(ctx, ATC_TC_NO_IM2COL) && r <= 128 && s <= 128;
  auto bmap = [&](CUtensorMap* m, const float* base) {
    if (im2col) return make_im2col_map(ctx, m, base, n, h, w_, c, (int)r, (int)s, BN / 2);
    return direct ? make_map(ctx, m, base, n * c, hw, hw, 32, BK, true)   // [N*C][H*W], MN-major chunks
                  : make_map(ctx, m, base, n * hw, c, c, BK, umma2 ? BN / 2 : BN, false);  // NHWC, K-major
  };
  if (!make_map(ctx, &maps.a[0], wh, k, r * s * c, r * s * c, BK, BM, false) || !bmap(&maps.b[0], ih))
    return ATC_ERR_CUDA;
  maps.a[1] = maps.a[0];
  maps.b[1] = maps.b[0];
  if (splits == 3 && (!make_map(ctx, &maps.a[1], wl, k, r * s * c, r * s * c, BK, BM, false) || !bmap(&maps.b[1], il)))
    return ATC_ERR_CUDA;
  Problem p{};
  p.conv = direct ? 2 : (im2col ? 4 : 1);
  p.M = (int)k;
  p.N = (int)hw;
  p.K = (int)c;
  p.splits = splits;
  p.C = d_out;
  p.img = (int)n;
  p.Cin = (int)c;
  p.H = (int)h;
  p.W = (int)w_;
  p.R = (int)r;
  p.S = (int)s;
  p.OH = (int)oh;
  p.OW = (int)ow;
  p.tiles_m = (int)((k + BM - 1) / BM);
  if (direct) {
    // per image ([N*C][H*W] view); only pixels p < OH*W can be valid outputs
    p.tiles_n = (int)((oh * w_ + BN - 1) / BN);
    p.tiles_img = (int)n;
  } else if (im2col) {
    // compact output pixels of the whole batch
    p.tiles_n = (int)((n * oh * ow + BN - 1) / BN);
    p.tiles_img = 1;
  } else {
    // the batch's pixels back to back on the NHWC input: tiles run across image
    // boundaries (shifted rows of a valid output never leave its image)
    const int64_t last = (n - 1) * hw + (oh - 1) * w_ + (ow - 1);
    p.tiles_n = (int)((last + BN) / BN);
    p.tiles_img = 1;
  }
  p.pair = use_pair(ctx, p);
  p.umma2 = umma2 ? 1 : 0;
  // split-K over two CTA pairs when the pair tiles leave most of a second wave idle
  // (conv5: 98 tiles on 74 pair slots); the output is zeroed and both halves added
  if (im2col && splits == 1 && !tc_flag(ctx, ATC_TC_NO_KSPLIT)) {
    const int pairs = std::max(1, ctx->sm_count / 2);
    const int units = (p.tiles_m + 1) / 2 * p.tiles_n;
    const int kb = (int)(r * s * (c / BK));
    auto eff = [&](int u) { return (double)u / (double)(((u + pairs - 1) / pairs) * pairs); };
    if (kb % 2 == 0 && eff(2 * units) > eff(units) + 0.1) {
      p.ksplit = 2;
      if (!atc_cuda_ok(ctx, cudaMemsetAsync(d_out, 0, (size_t)(n * k * oh * ow) * 4, st), "memset out"))
        return ATC_ERR_CUDA;
    }
  }
  // 1x1 direct: the output is a [N*K][OH*OW] matrix (hw % 4 == 0): TMA-store epilogue
  // when every 32-row store box lies inside one image's K rows
  p.tma_store = direct && k % 32 == 0 && !tc_flag(ctx, ATC_TC_NO_TMA_STORE) ? 1 : 0;
  if (p.tma_store && !make_map(ctx, &maps.c, d_out, n * k, oh * ow, oh * ow, 32, 32, false)) return ATC_ERR_CUDA;
  return launch(ctx, maps, p, st) ? ATC_OK : ATC_ERR_CUDA;
}

int atc_conv2d_nchw(atc_ctx* ctx, const float* in, const float* w, float* out, int64_t n, int64_t c, int64_t h,
                    int64_t w_, int64_t k, int64_t r, int64_t s, int32_t precision) {
  ATC_ENTER(ctx);
  const int64_t oh = h - r + 1, ow = w_ - s + 1;
  if (n < 1 || c < 1 || h < 1 || w_ < 1 || k < 1 || r < 1 || s < 1 || oh < 1 || ow < 1 || !in || !w || !out) {
    atc_set_error(ctx, "bad arguments to atc_conv2d_nchw");
    return ATC_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t bi = (size_t)(n * c * h * w_) * 4, bw = (size_t)(k * c * r * s) * 4, bo = (size_t)(n * k * oh * ow) * 4;
  float* di = (float*)atc_ctx_scratch(ctx, 8, bi);
  float* dw = (float*)atc_ctx_scratch(ctx, 9, bw);
  float* dout = (float*)atc_ctx_scratch(ctx, 10, bo);
  if (!di || !dw || !dout) return ATC_ERR_CUDA;
  if (!atc_cuda_ok(ctx, cudaMemcpyAsync(di, in, bi, cudaMemcpyHostToDevice, st), "H2D in") ||
      !atc_cuda_ok(ctx, cudaMemcpyAsync(dw, w, bw, cudaMemcpyHostToDevice, st), "H2D w"))
    return ATC_ERR_CUDA;
  int rc = atc_conv2d_nchw_device(ctx, di, dw, dout, n, c, h, w_, k, r, s, precision, st);
  if (rc) return rc;
  if (!atc_cuda_ok(ctx, cudaMemcpyAsync(out, dout, bo, cudaMemcpyDeviceToHost, st), "D2H out") ||
      !atc_cuda_ok(ctx, cudaStreamSynchronize(st), "conv sync"))
    return ATC_ERR_CUDA;
  return ATC_OK;
}

}  // extern "C"
