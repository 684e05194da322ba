// Shared device-side decode / check routines of the binding evaluator.
//
// The predicate restated here is the binding-dependent half of
// rewriter::verify_rewrite (/root/reference/proj/src/rewriter.cpp:215-284) for
// one (binding b, recorded test t):
//   1. run_dispatch extent checks (rewriter.cpp:136-148): every API array's dims
//      >= 1 and  prod(dims) <= region length, else "dispatch failed" (reason 2);
//   2. run_reference (equivalence.cpp:40-93) over full-region copies, FP64,
//      acc = acc + a*b with NO fused multiply-add, reference loop order, later
//      writes overwrite earlier ones;
//   3. write-back rounding (double)(float) for f32 regions (rewriter.cpp:156-157);
//   4. full-region compare |have - want| > abs + rel*|want| (rewriter.cpp:270-272),
//      rel/abs = 1e-4/1e-6 (f32) or 1e-9/1e-12 (f64).
// Step 4 over 65,536 elements is evaluated in O(footprint): positions the API
// never writes keep their initial value, so they fail iff they are "dirty"
// (|init - final| > tol), precomputed once per (t, pointer) by atc_build_dirty;
// a binding passes t iff every dirty position is written by the API call and
// every written position (its last writer) matches `final` within tolerance.
#pragma once
#include <cstdint>

#include "atc_b200.h"

namespace atc {

// k_screen_conv_pairs CTA size: every CTA builds the plane tables once, so fewer,
// larger CTAs (one per SM) pay that prologue fewer times
constexpr int kPairThreads = 1024;

// k_probe_regions CTA size: 156 threads twist (5 warps)
constexpr int kProbeThreads = 160;

// the first digit whose int has the same value as digit d's (test 0's ints)
__device__ __forceinline__ int canon_digit(const int64_t* ints, int nI, int d) {
  const int64_t v = ints[d];
  for (int j = 0; j < d; ++j)
    if (ints[j] == v) return j;
  return d;
}


constexpr int kMaxT = 64;
constexpr int kMaxPtrs = 16;
constexpr int kMaxInts = 32;

// Device view of an uploaded test-set bundle (atc_testset_handle).
struct TestsetView {
  int32_t T, nI, nP;
  const int64_t* ints;        // [T][nI]
  const int32_t* is_f32;      // [nP]
  const int64_t* region_len;  // [nP]
  const int32_t* test_ok;     // [T]
  const double* init;         // pool; region (t,p) at init + region_off[t*nP+p]
  const double* fin;          // pool; same offsets
  const int64_t* region_off;  // [T*nP]
  const int32_t* dirty_pos;   // pool; list (t,p) at dirty_pos + dirty_off[t*nP+p]
  const int64_t* dirty_off;   // [T*nP]
  const int32_t* dirty_cnt;   // [T*nP]
  const int32_t* dirty_max;   // [T*nP]  (-1 when empty)
  int32_t nF;                 // user float params (extended semantics only; 0 otherwise)
  const double* floats;       // [T][nF]
  // floor(n / nI) = umulhi(n, nI_m) >> nI_sh for n < 2^31 (nI_m = 0: nI = 1), see
  // div_nI; set by the upload
  uint32_t nI_m, nI_sh;
};

// floor(n / ts.nI) for n < 2^31 (the digit decode of an enumerated binding index)
__device__ __forceinline__ uint32_t div_nI(const TestsetView& ts, uint32_t n) {
  return ts.nI_m ? __umulhi(n, ts.nI_m) >> ts.nI_sh : n;
}
// floor(g / d) for d >= 1 and a quotient below 2^22 (a permutation index): a float
// estimate (relative error < 2^-22, so off by at most one) corrected either way
__device__ __forceinline__ uint64_t div_small_q(uint64_t g, uint64_t d) {
  uint64_t q = (uint64_t)((float)g * __frcp_rn((float)d));
  if (q * d > g) --q;
  else if ((q + 1) * d <= g) ++q;
  return q;
}

// One handle of a batched seeded update (k_copy_meta + k_probe_regions_many).
struct ProbeJob {
  TestsetView view;          // the handle's view (its meta block, pools)
  int32_t cta0;              // the handle's first CTA within its launch group's numbering
  const uint64_t* seeds;     // [T]       (update staging, device)
  const uint64_t* skips;     // [T * nP]
  const int64_t* diff_off;   // [T * nP + 1]
  const int32_t* diff_pos;
  const double* diff_val;
  const int64_t* need;       // [T * nP]
  const uint8_t* meta_src;   // staged metadata block
  uint8_t* meta_dst;         // the handle's meta block
  uint64_t meta_bytes;
};

// Spec decode table in a device-friendly form (copied by value into kernels).
struct SpecView {
  int32_t sem, layout, nA, nS;
  int32_t role[ATC_MAX_ARRAYS];
  int32_t ndims[ATC_MAX_ARRAYS];
  int32_t dims[ATC_MAX_ARRAYS][ATC_MAX_DIMS];
  int32_t role_size[ATC_SZ_COUNT];
  int32_t arr_of_role[3];  // API array index of role A/B/C (IN/WEIGHTS/OUT)
};

// Where a launch takes its bindings from.
struct BindingSource {
  // explicit list
  const uint8_t* arr_map;   // [n][nA]
  const uint8_t* size_map;  // [n][nS]
  // enumerated space
  const uint8_t* perms;     // [n_perms][nA]
  uint64_t size_maps;       // nI^nS
  uint64_t begin;
  int enumerated;
};

// Position-0 verdict table of an enumerated space (k_pos0_table).
constexpr int kMaxPos0Roles = 5;
struct Pos0Table {
  int R;                 // number of roles the position-0 value depends on
  int q[kMaxPos0Roles];  // size-param index of each role
  uint64_t per_perm;     // nI^R
  const uint8_t* table;  // [n_perms][nI^R]: 0 match, 1 mismatch, 2 not tabulated
};

// Per-launch plan of the row-hoisted screen (k_screen_rows).
struct RowPlan {
  uint32_t dim_mask[ATC_MAX_ARRAYS];   // per API array: bitmask of its dims over size params
  int32_t role_q[ATC_SZ_COUNT];        // per role: size-param index (fallbacks resolved), -1 absent
  Pos0Table pt;
  uint64_t key_stride[ATC_MAX_SIZES];  // table-key contribution of each size-param digit
  // gemm: the written-set check as one lookup — need[(p*nI + ldc digit)*nI + m digit]
  // = the smallest n writing every dirty position of region p at t = 0 (k_gemm_need;
  // INT32_MAX: none does, -1: not tabulated, use the dirty list)
  const int32_t* gemm_need;
  // conv (k_screen_conv_pairs): verdict bits over the nI values of tc_c per
  // (perm, h, w, r, s) key — output position 0 in bits 0..15, position 1 (used when
  // tc_ow >= 2) in bits 16..31 (k_pos0_table_conv / k_cmask)
  const uint32_t* cmask;
  // conv, canonical key order (h the fastest digit of a cmask word index): per (perm, w,
  // r, s) the h digits whose every c row mismatches — bit h in bits 0..15 for position 0,
  // bit 16 + h for positions 0 or 1 (ow >= 2); index = cmask word index / nI
  const uint32_t* allbad;
};

// One small enumerated space of a sweep for k_sweep_small (eval_kernels.cu): its
// CTAs are [cta0, cta0 + ctas), each screening and confirming a contiguous slice
// of the job's n bindings; results go to the job's block of the batch.
struct SmallJob {
  TestsetView ts;
  SpecView sp;
  BindingSource src;         // enumerated: device permutations, size_maps, begin = the range start
  uint64_t n;                // bindings in the range
  uint64_t* res;             // [0] K1 survivors, [1] passing count, [2 ..) passing global indices
  unsigned long long* hist;  // reason histogram (8 words)
  uint32_t cta0, ctas;
};

enum : int32_t { kUndecided = -2 };

// Encoded per-binding result: t * 8 + reason; kPassKey when every test passed.
constexpr int32_t kPassKey = 0x7fffffff;
__host__ __device__ inline int32_t fail_key(int t, int reason) { return t * 8 + reason; }

// ---- exact FP64 primitives: never contracted into DFMA -----------------------
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// rewriter.cpp:270-272 (tolerance test, evaluated without contraction)
__device__ __forceinline__ bool mismatch(double have, double want, bool f32) {
  const double rel = f32 ? 1e-4 : 1e-9;
  const double abs_ = f32 ? 1e-6 : 1e-12;
  return fabs(dsub(have, want)) > dadd(abs_, dmul(rel, fabs(want)));
}

__device__ __forceinline__ double round_region(double v, bool f32) {
  return f32 ? (double)__double2float_rn(v) : v;  // rewriter.cpp:156-157
}

// Verdict of one output position (does the value the API call writes there
// mismatch the recorded `want`?).
//   ATC_MODE_FP64:        the reference arithmetic (dot64: FP64, non-fused).
//   ATC_MODE_FP32_SCREEN: first an FP32 FMA dot product (dot32) with a running
//     sum S = sum |a'b'| of the float-rounded operands; the reference result
//     acc64 is then known to lie in [acc32 - E, acc32 + E] with
//       E = 1.01 (n + 4) u S + 1e-30,   u = 2^-24, n = dot length (< 4096),
//     covering operand rounding to float (2u|ab| per term), FMA accumulation
//     (gamma_n = n u / (1 - n u)), the reference's own FP64 rounding (2^-53 n) and
//     subnormal slack.  If every value in that interval (after the f32
//     write-back rounding, widened by u|acc| for f32 regions) is beyond the
//     tolerance the position is a mismatch; if every value is within it, a match;
//     otherwise the FP64 reference arithmetic decides.  Verdicts are therefore
//     identical in both modes; FP32 only makes clear cases cheaper.
template <class Dot64, class Dot32>
__device__ __forceinline__ bool position_mismatch(int mode, int n, double want, bool f32, Dot64 dot64, Dot32 dot32) {
  if (mode == ATC_MODE_FP32_SCREEN && n < 4096) {
    float S = 0.0f;
    const float acc32 = dot32(S);
    const double u = 5.9604644775390625e-08;  // 2^-24
    double E = 1.01 * (n + 4) * u * (double)S + 1e-30;
    if (f32) E += u * (fabs((double)acc32) + E);
    const double rel = f32 ? 1e-4 : 1e-9;
    const double abs_ = f32 ? 1e-6 : 1e-12;
    const double tol = abs_ + rel * fabs(want);
    const double d = fabs((double)acc32 - want);
    if (d - E > tol * (1.0 + 1e-12)) return true;    // every candidate value mismatches
    if (d + E < tol * (1.0 - 1e-12)) return false;   // every candidate value matches
  }
  return mismatch(round_region(dot64(), f32), want, f32);
}

// reference_gemm's inner loop (equivalence.cpp:55-58) over strided operands (generic
// loads: operands may be staged in shared memory)
__device__ __forceinline__ double gemm_dot64(const double* a, int sa, const double* b, int sb, int k) {
  double acc = 0.0;
  for (int p = 0; p < k; ++p) acc = dadd(acc, dmul(a[p * sa], b[p * sb]));
  return acc;
}
__device__ __forceinline__ float gemm_dot32(const double* a, int sa, const double* b, int sb, int k, float& S) {
  float acc = 0.0f;
  for (int p = 0; p < k; ++p) {
    const float x = __double2float_rn(a[p * sa]), y = __double2float_rn(b[p * sb]);
    acc = fmaf(x, y, acc);
    S = fmaf(fabsf(x), fabsf(y), S);
  }
  return acc;
}
// reference_conv2d's inner loops (equivalence.cpp:85-90); `in` points at
// in[b][0][y][x], `wt` at wt[q][0][0][0]
// Taps are loaded four at a time ahead of their (in-order) additions, the blocks running
// across filter rows (z outer, then u, v: the reference's order): the loads do not depend
// on the running sum, so each block's loads are in flight together.
__device__ __forceinline__ double conv_dot64(const double* in, const double* wt, int C, int R, int S, int H, int W) {
  double acc = 0.0;
  const int RS = R * S;
  for (int z = 0; z < C; ++z) {
    const double* az = in + z * H * W;
    const double* bz = wt + z * RS;
    int u = 0, v = 0;
    for (int k0 = 0; k0 < RS; k0 += 4) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool ok = k0 + i < RS;
        av[i] = ok ? az[u * W + v] : 0.0;
        bv[i] = ok ? bz[k0 + i] : 0.0;
        if (++v == S) {
          v = 0;
          ++u;
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (k0 + i < RS) acc = dadd(acc, dmul(av[i], bv[i]));
    }
  }
  return acc;
}

// conv_dot64 with the taps loaded eight at a time in blocks that run across filter rows
// (same order: z, then u, v) — fewer exposed load latencies per output; faster in K2-pre
// (183 -> 140 us of the serialised step), slower in K2b (359 -> 420 us: more registers on
// its 126-register warps), so K2-pre alone uses it.
__device__ __forceinline__ double conv_dot64_b8(const double* in, const double* wt, int C, int R, int S, int H,
                                                int W) {
  double acc = 0.0;
  const int RS = R * S;
  for (int z = 0; z < C; ++z) {
    const double* az = in + z * H * W;
    const double* bz = wt + z * RS;
    int u = 0, v = 0;
    for (int k0 = 0; k0 < RS; k0 += 8) {
      double av[8], bv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool ok = k0 + i < RS;
        av[i] = ok ? az[u * W + v] : 0.0;
        bv[i] = ok ? bz[k0 + i] : 0.0;
        if (++v == S) {
          v = 0;
          ++u;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (k0 + i < RS) acc = dadd(acc, dmul(av[i], bv[i]));
    }
  }
  return acc;
}

// conv_dot64 for MO outputs at once (independent chains, each in conv_dot64's order).
template <int MO>
__device__ __forceinline__ void conv_dot64_multi(const double* const* in, const double* const* wt, int C, int R, int S,
                                                 int H, int W, double* acc) {
#pragma unroll
  for (int m = 0; m < MO; ++m) acc[m] = 0.0;
  for (int z = 0; z < C; ++z)
    for (int u = 0; u < R; ++u) {
      const int ia = (z * H + u) * W, iw = (z * R + u) * S;
      for (int v0 = 0; v0 < S; v0 += 4) {
        double av[4][MO], bv[4][MO];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int m = 0; m < MO; ++m) {
            av[i][m] = v0 + i < S ? in[m][ia + v0 + i] : 0.0;
            bv[i][m] = v0 + i < S ? wt[m][iw + v0 + i] : 0.0;
          }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (v0 + i < S) {
#pragma unroll
            for (int m = 0; m < MO; ++m) acc[m] = dadd(acc[m], dmul(av[i][m], bv[i][m]));
          }
      }
    }
}
__device__ __forceinline__ float conv_dot32(const double* in, const double* wt, int C, int R, int S, int H, int W,
                                            float& Sabs) {
  float acc = 0.0f;
  for (int z = 0; z < C; ++z)
    for (int u = 0; u < R; ++u)
      for (int v = 0; v < S; ++v) {
        const float x = __double2float_rn(in[(z * H + u) * W + v]);
        const float y = __double2float_rn(wt[(z * R + u) * S + v]);
        acc = fmaf(x, y, acc);
        Sabs = fmaf(fabsf(x), fabsf(y), Sabs);
      }
  return acc;
}

// Resolved sizes of one (binding, t), reference roles with their fallbacks.
struct Dims {
  // gemm (equivalence.cpp:42-48)
  int64_t m, n, k, lda, ldb, ldc;
  // conv (equivalence.cpp:69-77)
  int64_t cn, cc, ch, cw, ck, cr, cs, coh, cow;
};

__device__ __forceinline__ int64_t role_or(const SpecView& sp, const int64_t* sz, int role, int64_t fb) {
  int q = sp.role_size[role];
  return q < 0 ? fb : sz[q];
}

__device__ __forceinline__ void resolve_dims(const SpecView& sp, const int64_t* sz, Dims& d) {
  if (sp.sem == ATC_SEM_GEMM) {
    const bool row = sp.layout == ATC_LAYOUT_ROW;
    d.m = role_or(sp, sz, ATC_SZ_M, 0);
    d.n = role_or(sp, sz, ATC_SZ_N, 0);
    d.k = role_or(sp, sz, ATC_SZ_K, 0);
    d.lda = role_or(sp, sz, ATC_SZ_LDA, row ? d.k : d.m);
    d.ldb = role_or(sp, sz, ATC_SZ_LDB, row ? d.n : d.k);
    d.ldc = role_or(sp, sz, ATC_SZ_LDC, row ? d.n : d.m);
  } else {
    d.cn = role_or(sp, sz, ATC_SZ_CN, 0);
    d.cc = role_or(sp, sz, ATC_SZ_CC, 0);
    d.ch = role_or(sp, sz, ATC_SZ_CH, 0);
    d.cw = role_or(sp, sz, ATC_SZ_CW, 0);
    d.ck = role_or(sp, sz, ATC_SZ_CK, 0);
    d.cr = role_or(sp, sz, ATC_SZ_CR, 0);
    d.cs = role_or(sp, sz, ATC_SZ_CS, 0);
    d.coh = role_or(sp, sz, ATC_SZ_COH, d.ch - d.cr + 1);
    d.cow = role_or(sp, sz, ATC_SZ_COW, d.cw - d.cs + 1);
  }
}

// run_dispatch (rewriter.cpp:136-148): 0 when the call would proceed, else
// ATC_FAIL_DISPATCH.  ptr_of[a] = user pointer bound to API array a.
__device__ __forceinline__ int extent_check(const SpecView& sp, const int64_t* sz, const int* ptr_of,
                                            const int64_t* region_len) {
  for (int a = 0; a < sp.nA; ++a) {
    int64_t ext = 1;
    for (int d = 0; d < sp.ndims[a]; ++d) {
      int64_t v = sz[sp.dims[a][d]];
      if (v < 1) return ATC_FAIL_DISPATCH;
      ext *= v;
    }
    if (region_len[ptr_of[a]] < ext) return ATC_FAIL_DISPATCH;
  }
  return 0;
}

// Accesses outside [0, region) would be undefined behaviour in the reference
// (std::vector operator[]); never reached at P2 sizes, rejected if they occur.
// Also guarantees every index below fits in int32.
__device__ __forceinline__ int ub_check(const SpecView& sp, const Dims& d, const int* ptr_of,
                                        const int64_t* region_len) {
  const int64_t lenA = region_len[ptr_of[sp.arr_of_role[0]]];
  const int64_t lenB = region_len[ptr_of[sp.arr_of_role[1]]];
  const int64_t lenC = region_len[ptr_of[sp.arr_of_role[2]]];
  if (sp.sem == ATC_SEM_GEMM) {
    if (d.m < 1 || d.n < 1 || d.k < 1) return 0;  // loops empty: nothing accessed
    if (d.lda < 0 || d.ldb < 0 || d.ldc < 0) return ATC_FAIL_UB;
    const bool row = sp.layout == ATC_LAYOUT_ROW;
    const int64_t amax = row ? (d.m - 1) * d.lda + (d.k - 1) : (d.k - 1) * d.lda + (d.m - 1);
    const int64_t bmax = row ? (d.k - 1) * d.ldb + (d.n - 1) : (d.n - 1) * d.ldb + (d.k - 1);
    const int64_t cmax = row ? (d.m - 1) * d.ldc + (d.n - 1) : (d.n - 1) * d.ldc + (d.m - 1);
    if (amax >= lenA || bmax >= lenB || cmax >= lenC) return ATC_FAIL_UB;
  } else {
    if (d.cn < 1 || d.ck < 1 || d.coh < 1 || d.cow < 1) return 0;
    if (d.cc < 1 || d.cr < 1 || d.cs < 1) return 0;  // out written with acc = 0, no reads
    const int64_t imax = (((d.cn - 1) * d.cc + (d.cc - 1)) * d.ch + (d.coh - 1) + (d.cr - 1)) * d.cw +
                         (d.cow - 1) + (d.cs - 1);
    const int64_t wmax = (((d.ck - 1) * d.cc + (d.cc - 1)) * d.cr + (d.cr - 1)) * d.cs + (d.cs - 1);
    const int64_t omax = ((d.cn * d.ck) * d.coh) * d.cow - 1;
    if (imax >= lenA || wmax >= lenB || omax >= lenC || imax < 0) return ATC_FAIL_UB;
  }
  return 0;
}

// ---- GEMM write-set algebra (reference loop order i -> j, C[pos] = acc) -------
// Row-major writes pos = i*ldc + j; col-major pos = j*ldc + i.
// (i,j) is the LAST writer of its position iff no later (i',j') hits it:
//   row: i == m-1 || j < ldc        col: j == 0 || i + ldc >= m
__device__ __forceinline__ bool gemm_last_writer(bool row, int i, int j, int m, int ldc) {
  return row ? (i == m - 1 || j < ldc) : (j == 0 || i + ldc >= m);
}
// Is position p written at all?
__device__ __forceinline__ bool gemm_written(bool row, int p, int m, int n, int ldc) {
  if (row) {
    int i = p / ldc;
    if (i > m - 1) i = m - 1;
    return p - i * ldc < n;
  }
  int hi = p < m - 1 ? p : m - 1;
  int r = p % ldc;
  if (r > hi) return false;
  int i = r + ldc * ((hi - r) / ldc);
  return (p - i) / ldc < n;
}

}  // namespace atc
