// Binding-evaluator kernels (K0 dirty lists, K1 screen, K2 confirm).
//
// Work decomposition:
//   K0 atc_build_dirty    one pass over every recorded (t, pointer) region pair;
//                         appends {i : |init_i - final_i| > tol} (rewriter.cpp:270-272).
//   K1 atc_screen_*       one THREAD per candidate binding, test t = 0 only, with a
//                         bounded budget of output positions.  Nearly every wrong
//                         binding is rejected here after a handful of integer ops
//                         and at most `budget` dot products.  Bindings that pass
//                         what they checked are appended to a survivor queue.
//   K2 atc_confirm        one CTA per (survivor, t) for every t: the A/B operand
//                         prefixes are staged into shared memory with coalesced
//                         vector loads, output positions are split across the CTA,
//                         a mismatch flag in shared memory gives block-wide early
//                         exit, and the first failing test is reduced with atomicMin.
// Both halves evaluate exactly the predicate of eval_common.cuh.
#include <cuda_runtime.h>

#include "eval_common.cuh"

namespace atc {

// ------------------------------------------------------------------ K0 -------
__global__ void k_build_dirty(TestsetView ts, int32_t* dirty_pos, int32_t* dirty_cnt,
                              int32_t* dirty_max) {
  const int tp = blockIdx.y;  // (t, p) pair
  const int p = tp % ts.nP;
  const int64_t len = ts.region_len[p];
  const bool f32 = ts.is_f32[p] != 0;
  const double* init = ts.init + ts.region_off[tp];
  const double* fin = ts.fin + ts.region_off[tp];
  int32_t* out = dirty_pos + ts.dirty_off[tp];
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < len; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool dirty = false;
    if (i < len) dirty = mismatch(init[i], fin[i], f32);
    const unsigned ball = __ballot_sync(0xffffffffu, dirty);
    if (ball == 0) continue;
    int slot = 0;
    if (lane == 0) slot = atomicAdd(&dirty_cnt[tp], __popc(ball));
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (dirty) {
      out[slot + __popc(ball & ((1u << lane) - 1))] = (int32_t)i;
      atomicMax(&dirty_max[tp], (int32_t)i);
    }
  }
}

// ------------------------------------------------------------ binding decode --


__device__ __forceinline__ void decode_binding(const BindingSource& src, const SpecView& sp, int nI,
                                               uint64_t idx, int* ptr_of, int* int_of) {
  if (!src.enumerated) {
    for (int a = 0; a < sp.nA; ++a) ptr_of[a] = src.arr_map[idx * sp.nA + a];
    for (int q = 0; q < sp.nS; ++q) int_of[q] = src.size_map[idx * sp.nS + q];
    return;
  }
  const uint64_t g = src.begin + idx;
  const uint64_t perm = g / src.size_maps;
  uint64_t s = g - perm * src.size_maps;
  for (int a = 0; a < sp.nA; ++a) ptr_of[a] = src.perms[perm * sp.nA + a];
  if (s < (1ull << 32)) {
    uint32_t s32 = (uint32_t)s;
    for (int q = 0; q < sp.nS; ++q) {
      uint32_t d = s32 / (uint32_t)nI;
      int_of[q] = (int)(s32 - d * (uint32_t)nI);
      s32 = d;
    }
  } else {
    for (int q = 0; q < sp.nS; ++q) {
      uint64_t d = s / (uint64_t)nI;
      int_of[q] = (int)(s - d * (uint64_t)nI);
      s = d;
    }
  }
}

// ---------------------------------------------------- single-thread check ----
// Checks test t for one binding on one thread.  Returns 0 (passed everything it
// looked at), a reason code, or kUndecided when `budget` output positions were
// checked without reaching the end.
__device__ int thread_check(const TestsetView& ts, const SpecView& sp, const int* ptr_of,
                            const int64_t* sz, int t, int budget, bool* complete, int mode) {
  *complete = false;
  if (!ts.test_ok[t]) return ATC_FAIL_TESTSET;
  if (int r = extent_check(sp, sz, ptr_of, ts.region_len)) return r;
  Dims d;
  resolve_dims(sp, sz, d);
  if (int r = ub_check(sp, d, ptr_of, ts.region_len)) return r;
  const int pA = ptr_of[sp.arr_of_role[0]], pB = ptr_of[sp.arr_of_role[1]], pC = ptr_of[sp.arr_of_role[2]];
  const int tpA = t * ts.nP + pA, tpB = t * ts.nP + pB, tpC = t * ts.nP + pC;
  const double* __restrict__ A = ts.init + ts.region_off[tpA];
  const double* __restrict__ B = ts.init + ts.region_off[tpB];
  const double* __restrict__ F = ts.fin + ts.region_off[tpC];
  const bool f32 = ts.is_f32[pC] != 0;
  const int ndirty = ts.dirty_cnt[tpC];
  const int32_t* dirty = ts.dirty_pos + ts.dirty_off[tpC];

  if (sp.sem == ATC_SEM_GEMM) {
    const bool row = sp.layout == ATC_LAYOUT_ROW;
    const int m = (int)d.m, n = (int)d.n, k = (int)d.k;
    const int lda = (int)d.lda, ldb = (int)d.ldb, ldc = (int)d.ldc;
    if (m < 1 || n < 1) {  // no writes: every dirty position is a mismatch
      if (ndirty) return ATC_FAIL_MISMATCH;
      *complete = true;
      return 0;
    }
    // dirty positions must all be written (else the untouched value differs)
    for (int e = 0; e < ndirty; ++e)
      if (!gemm_written(row, __ldg(dirty + e), m, n, ldc)) return ATC_FAIL_MISMATCH;
    const bool overlap = row ? (ldc < n && m > 1) : (ldc < m && n > 1);
    int checked = 0;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) {
        if (overlap && !gemm_last_writer(row, i, j, m, ldc)) continue;
        if (checked == budget) return kUndecided;
        ++checked;
        const double* a = row ? A + i * lda : A + i;
        const double* b = row ? B + j : B + j * ldb;
        const int sa = row ? 1 : lda, sb = row ? ldb : 1;
        const int pos = row ? i * ldc + j : j * ldc + i;
        if (position_mismatch(
                mode, k, __ldg(F + pos), f32, [&] { return gemm_dot64(a, sa, b, sb, k); },
                [&](float& S) { return gemm_dot32(a, sa, b, sb, k, S); }))
          return ATC_FAIL_MISMATCH;
      }
    *complete = true;
    return 0;
  }
  // conv2d: the write set is exactly [0, n*k*oh*ow) (a bijection)
  const int N = (int)d.cn, C = (int)d.cc, H = (int)d.ch, W = (int)d.cw, K = (int)d.ck, R = (int)d.cr,
            S = (int)d.cs, OH = (int)d.coh, OW = (int)d.cow;
  const int64_t wext = (int64_t)N * K * OH * OW;
  if (ts.dirty_max[tpC] >= wext) return ATC_FAIL_MISMATCH;
  int checked = 0;
  for (int b = 0; b < N; ++b)
    for (int q = 0; q < K; ++q)
      for (int y = 0; y < OH; ++y)
        for (int x = 0; x < OW; ++x) {
          if (checked == budget) return kUndecided;
          ++checked;
          const double* in = A + ((b * C) * H + y) * W + x;
          const double* wt = B + (q * C) * R * S;
          const int pos = ((b * K + q) * OH + y) * OW + x;
          if (position_mismatch(
                  mode, C * R * S, __ldg(F + pos), f32, [&] { return conv_dot64(in, wt, C, R, S, H, W); },
                  [&](float& Sa) { return conv_dot32(in, wt, C, R, S, H, W, Sa); }))
            return ATC_FAIL_MISMATCH;
        }
  *complete = true;
  return 0;
}

// ------------------------------------------------------------------ K1 -------
// Explicit lists: keys[b] receives the t=0 failure or stays kPassKey; bindings
// that are not rejected at t=0 go to the survivor queue (for every t in K2).
// Enumerated spaces: rejected bindings only feed the reason histogram.
__global__ void __launch_bounds__(256) k_screen(TestsetView ts, SpecView sp, BindingSource src,
                                                 uint64_t n, int budget, int32_t* keys,
                                                 uint64_t* surv, uint64_t surv_cap,
                                                 unsigned long long* surv_cnt,
                                                 unsigned long long* reason_hist, int mode) {
  __shared__ int64_t s_ints0[kMaxInts];
  __shared__ unsigned long long s_hist[ATC_REASON_COUNT];
  if (threadIdx.x < ts.nI) s_ints0[threadIdx.x] = ts.ints[threadIdx.x];
  if (threadIdx.x < ATC_REASON_COUNT) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += stride) {
    int ptr_of[ATC_MAX_ARRAYS], int_of[ATC_MAX_SIZES];
    decode_binding(src, sp, ts.nI, idx, ptr_of, int_of);
    int64_t sz[ATC_MAX_SIZES];
    for (int q = 0; q < sp.nS; ++q) sz[q] = s_ints0[int_of[q]];
    bool complete;
    int r = thread_check(ts, sp, ptr_of, sz, 0, budget, &complete, mode);
    if (r > 0) {
      if (keys) keys[idx] = fail_key(0, r);
      if (reason_hist) atomicAdd(&s_hist[r], 1ull);
    } else {
      // passed t = 0 so far: every remaining t (and t = 0 when undecided)
      // is decided by K2
      unsigned long long slot = atomicAdd(surv_cnt, 1ull);
      if (slot < surv_cap) surv[slot] = idx;
    }
  }
  if (reason_hist) {
    __syncthreads();
    if (threadIdx.x < ATC_REASON_COUNT && s_hist[threadIdx.x])
      atomicAdd(&reason_hist[threadIdx.x], s_hist[threadIdx.x]);
  }
}

// --------------------------------------------- K1 for enumerated spaces ------
// Factorised screen.  Position 0 of the output is written by the first loop
// iteration of run_reference (gemm (i,j) = (0,0); conv (b,q,y,x) = 0) and is
// always its own last writer.  Its value depends only on the array permutation
// and a few size roles:
//   gemm row-major  sum_p A[p] * B[p*ldb]      roles (k, ldb)   [ldb falls back to n]
//   gemm col-major  sum_p A[p*lda] * B[p]      roles (k, lda)   [lda falls back to m]
//   conv2d          sum_{z,u,v} in[(z*h+u)*w+v] * wt[(z*r+u)*s+v]   roles (c, h, w, r, s)
// so the t = 0 verdict of position 0 is tabulated once per (permutation,
// user ints bound to those roles) — e.g. 6 x 9^5 entries for a 2.3e9-binding
// conv space — with exactly the FP64 non-fused arithmetic of thread_check.
// The per-binding screen is then integer-only: run_dispatch extent checks,
// access bounds, the dirty-set (write-set) check, one table lookup.  Bindings
// that pass all of it go to K2, which re-checks every test completely.

// Written-set table for the gemm screen (RowPlan::gemm_need).  For a region p,
// an ldc value L and an m value, position q of the dirty list is written by a
// binding iff n >= n_min(q) (gemm_written is monotone in n):
//   row-major: i = min(q / L, m - 1),  n_min = q - i*L + 1
//   col-major: hi = min(q, m - 1), r = q % L; never if r > hi, else
//              i = r + L*((hi - r) / L),  n_min = (q - i)/L + 1
// need = max over the dirty list.  One CTA per (p, L digit, m digit).
__global__ void k_gemm_need(TestsetView ts, int row_major, int32_t* need) {
  const int nI = ts.nI;
  const int e = blockIdx.x;
  const int dm = e % nI, dl = (e / nI) % nI, p = e / (nI * nI);
  const int64_t m = ts.ints[dm], L = ts.ints[dl];  // t = 0 values
  __shared__ int32_t s_max;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  if (m < 1 || L < 1) {
    if (threadIdx.x == 0) need[e] = -1;
    return;
  }
  const int32_t* dirty = ts.dirty_pos + ts.dirty_off[p];
  const int cnt = ts.dirty_cnt[p];
  int32_t local = 0;
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
    const int64_t q = dirty[k];
    int64_t nmin;
    if (row_major) {
      const int64_t i = min(q / L, m - 1);
      nmin = q - i * L + 1;
    } else {
      const int64_t hi = min(q, m - 1), r = q % L;
      nmin = r > hi ? (int64_t)INT32_MAX : (q - (r + L * ((hi - r) / L))) / L + 1;
    }
    local = max(local, (int32_t)(nmin < INT32_MAX ? nmin : INT32_MAX));
  }
  for (int o = 16; o > 0; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&s_max, local);
  __syncthreads();
  if (threadIdx.x == 0) need[e] = s_max;
}

// out1 (conv, optional): the same verdict at output position 1 for bindings with
// tc_ow >= 2, i.e. output (b, q, y, x) = (0, 0, 0, 1): the input window shifted by one.
// Conv position-0/1 tables with one accumulation per (perm, h, w, r, s): the
// reference sums z (channel) outermost, so the sum for c channels is the running
// sum after z = c - 1 — every value of tc_c is read off one pass (same order, same
// bits as k_pos0_table's per-entry loops).  Lanes of a warp share (r, s).
// cm (optional): the same verdicts as bit words over the c digits — word
// (perm, h, w, r, s) bit j = table entry (perm, c digit j, h, w, r, s) == 1 for
// output position 0, bit 16 + j the same for position 1 — which is what
// k_screen_conv_pairs reads (one thread owns exactly one word).
__global__ void k_pos0_table_conv(TestsetView ts, SpecView sp, const uint8_t* perms, int n_perms, Pos0Table pt,
                                  uint8_t* out, uint8_t* out1, uint32_t* cm, int stage_a, int stage_b,
                                  uint32_t* allbad) {
  // blockIdx.y = permutation; blockIdx.x strides over its (h, w, r, s) entries.
  // stage_a / stage_b > 0: the first stage_a / stage_b elements of the in / weights
  // regions (every element a tabulated sum can read) are staged in shared memory.
  extern __shared__ double s_stage[];
  const uint64_t nI = (uint64_t)ts.nI, nI2 = nI * nI;
  const uint64_t per = nI2 * nI2;  // (h, w) x (r, s)
  __shared__ int64_t s_ints[kMaxInts];
  __shared__ uint8_t s_cd[kMaxInts];  // the digits whose value no earlier digit has
  __shared__ int s_nc;
  if (threadIdx.x < ts.nI) s_ints[threadIdx.x] = ts.ints[threadIdx.x];
  if (threadIdx.x == 0) {
    int nc = 0;
    for (int d = 0; d < ts.nI; ++d)
      if (canon_digit(ts.ints, ts.nI, d) == d) s_cd[nc++] = (uint8_t)d;
    s_nc = nc;
  }
  const uint64_t perm = blockIdx.y;
  const int pA = perms[perm * sp.nA + sp.arr_of_role[0]];
  const int pB = perms[perm * sp.nA + sp.arr_of_role[1]];
  const int pC = perms[perm * sp.nA + sp.arr_of_role[2]];
  const int64_t lenA = ts.region_len[pA], lenB = ts.region_len[pB];
  const double* A = ts.init + ts.region_off[pA];
  const double* B = ts.init + ts.region_off[pB];
  if (stage_a > 0) {
    const int na = (int)(lenA < stage_a ? lenA : stage_a), nb = (int)(lenB < stage_b ? lenB : stage_b);
    for (int k = threadIdx.x; k < na; k += blockDim.x) s_stage[k] = A[k];
    for (int k = threadIdx.x; k < nb; k += blockDim.x) s_stage[stage_a + k] = B[k];
    A = s_stage;
    B = s_stage + stage_a;
  }
  __syncthreads();
  int64_t cmax_all = 0;
  for (int j = 0; j < ts.nI; ++j) cmax_all = max(cmax_all, s_ints[j]);
  const double want = ts.fin[ts.region_off[pC]];
  const bool f32 = ts.is_f32[pC] != 0;
  const bool pos1 = out1 && ts.region_len[pC] > 1;
  const double want1 = pos1 ? ts.fin[ts.region_off[pC] + 1] : 0.0;
  const uint8_t empty_res = mismatch(round_region(0.0, f32), want, f32) ? 1 : 0;
  // an entry depends on the digits' VALUES only: thread i takes the i-th tuple of
  // distinct values (each value's first digit; k_pos0_table_expand copies the tuples
  // with repeated values), (h, w) fastest
  const uint64_t nc = (uint64_t)s_nc, nc2 = nc * nc, per_c = nc2 * nc2;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per_c; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t rs_c = i / nc2, hw_c = i - rs_c * nc2;
    const uint64_t r_d = s_cd[rs_c % nc], s_d = s_cd[rs_c / nc], h_d = s_cd[hw_c % nc], w_d = s_cd[hw_c / nc];
    const int64_t h = s_ints[h_d], w = s_ints[w_d], r = s_ints[r_d], s = s_ints[s_d];
    const uint64_t base = perm * pt.per_perm + nI * (h_d + nI * (w_d + nI * (r_d + nI * s_d)));  // + c digit
    const bool shape_ok = r >= 1 && s >= 1 && h >= 0 && w >= 0;
    auto words = [&]() {  // this thread's entries as bit words (it wrote them itself)
      if (!cm) return;
      uint32_t m0 = 0, m1 = 0;
      for (uint64_t j = 0; j < nI; ++j) {
        m0 |= (out[base + j] == 1 ? 1u : 0u) << j;
        if (out1) m1 |= (out1[base + j] == 1 ? 1u : 0u) << j;
      }
      cm[base / nI] = m0 | (m0 | m1) << 16;  // position 0 in bits 0..15, positions 0 or 1 in bits 16..31
      if (allbad) {  // (zeroed by the host) this h digit in its (perm, w, r, s) group's mask
        const uint32_t all = (1u << nI) - 1u;
        const uint32_t bits = (m0 == all ? 1u << h_d : 0u) | ((m0 | m1) == all ? 1u << (16 + h_d) : 0u);
        if (bits) atomicOr(allbad + base / nI / nI, bits);
      }
    };
    // entries whose c digit is < 1 (or a bad shape): the empty sum; others: 2 until computed
    for (uint64_t j = 0; j < nI; ++j) {
      const bool empty_sum = !shape_ok || s_ints[j] < 1;
      out[base + j] = empty_sum ? empty_res : 2;
      if (out1) out1[base + j] = 2;
    }
    if (!shape_ok) {
      words();
      continue;
    }
    double acc = 0.0, acc1 = 0.0;
    bool v1_live = pos1;
    for (int64_t z = 0; z < cmax_all; ++z) {
      const int64_t c = z + 1;
      const int64_t imax = ((c - 1) * h + (r - 1)) * w + (s - 1), wmax = c * r * s - 1;
      const bool v0 = imax < lenA && wmax < lenB;  // imax >= 0 here
      v1_live = v1_live && imax + 1 < lenA && wmax < lenB;
      if (!v0) break;  // monotone in c: no larger c is tabulated either
      // indices below are < len(region) < 2^31 here (and < stage_a / stage_b when staged)
      const int hi = (int)h, wi = (int)w, ri = (int)r, si = (int)s, zi = (int)z;
      if (v1_live) {
        for (int u = 0; u < ri; ++u) {
          const double* __restrict__ a = A + (zi * hi + u) * wi;
          const double* __restrict__ b = B + (zi * ri + u) * si;
          double a0 = a[0];
          for (int t = 0; t < si; ++t) {
            const double bv = b[t], a1 = a[t + 1];
            acc = dadd(acc, dmul(a0, bv));
            acc1 = dadd(acc1, dmul(a1, bv));
            a0 = a1;
          }
        }
      } else {
        for (int u = 0; u < ri; ++u) {
          const double* __restrict__ a = A + (zi * hi + u) * wi;
          const double* __restrict__ b = B + (zi * ri + u) * si;
          for (int t = 0; t < si; ++t) acc = dadd(acc, dmul(a[t], b[t]));
        }
      }
      for (uint64_t j = 0; j < nI; ++j)
        if (s_ints[j] == c) {
          out[base + j] = mismatch(round_region(acc, f32), want, f32) ? 1 : 0;
          if (out1 && v1_live) out1[base + j] = mismatch(round_region(acc1, f32), want1, f32) ? 1 : 0;
        }
    }
    words();
  }
}

// The (h, w, r, s) tuples k_pos0_table_conv skipped (a digit whose value an earlier
// digit also has): each a copy of its canonical tuple's entries — table bytes at
// position 0 (and 1 when out1 is given), the bit word, and its h bit in the all-bad masks.  The ints of a
// test repeat values (nine ints over a few sizes), so the running sums run for a few
// hundred value tuples per permutation instead of nI^4.
__global__ void k_pos0_table_expand(TestsetView ts, int n_perms, Pos0Table pt, uint8_t* out, uint8_t* out1,
                                    uint32_t* cm, uint32_t* allbad) {
  __shared__ uint8_t s_canon[kMaxInts];
  if (threadIdx.x < ts.nI) s_canon[threadIdx.x] = (uint8_t)canon_digit(ts.ints, ts.nI, (int)threadIdx.x);
  __syncthreads();
  const uint64_t nI = (uint64_t)ts.nI, nI2 = nI * nI, per = nI2 * nI2;
  const uint64_t perm = blockIdx.y;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t rs_d = i / nI2, hw_d = i - rs_d * nI2;
    const uint64_t r_d = rs_d % nI, s_d = rs_d / nI, h_d = hw_d % nI, w_d = hw_d / nI;
    const uint64_t ch = s_canon[h_d], cw = s_canon[w_d], cr = s_canon[r_d], cs = s_canon[s_d];
    if (ch == h_d && cw == w_d && cr == r_d && cs == s_d) continue;  // computed in place
    const uint64_t base = perm * pt.per_perm + nI * (h_d + nI * (w_d + nI * (r_d + nI * s_d)));
    const uint64_t src = perm * pt.per_perm + nI * (ch + nI * (cw + nI * (cr + nI * cs)));
    for (uint64_t j = 0; j < nI; ++j) {
      out[base + j] = out[src + j];
      if (out1) out1[base + j] = out1[src + j];
    }
    if (cm) {
      const uint32_t wd = cm[src / nI];
      cm[base / nI] = wd;
      if (allbad) {
        const uint32_t all = (1u << nI) - 1u;
        const uint32_t bits = ((wd & 0xFFFFu) == all ? 1u << h_d : 0u) | ((wd >> 16) == all ? 1u << (16 + h_d) : 0u);
        if (bits) atomicOr(allbad + base / nI / nI, bits);
      }
    }
  }
}

__global__ void k_pos0_table(TestsetView ts, SpecView sp, const uint8_t* perms, int n_perms, Pos0Table pt,
                             uint8_t* out, uint8_t* out1) {
  const uint64_t total = (uint64_t)n_perms * pt.per_perm;
  // conv: thread i takes the entry whose (c, r, s) digits are its slowest-varying
  // part, so the lanes of a warp share the dot-product trip counts c*r*s and
  // differ in (h, w, permutation) only (no divergence in the loops below)
  const uint64_t nI = (uint64_t)ts.nI, nI2 = nI * nI;
  const uint64_t inner = nI2 * (uint64_t)n_perms;  // (h, w, perm) combinations
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t e = i;
    if (sp.sem == ATC_SEM_CONV2D && pt.R == 5) {
      const uint64_t crs = i / inner, hwp = i - crs * inner;  // crs = c + nI*(r + nI*s)
      const uint64_t perm_i = hwp / nI2, hw = hwp - perm_i * nI2;
      const uint64_t c = crs % nI, rs = crs / nI;               // rs = r + nI*s
      e = perm_i * pt.per_perm + c + nI * hw + nI2 * nI * rs;   // key: c + nI*(h + nI*(w + nI*(r + nI*s)))
    }
    const uint64_t perm = e / pt.per_perm;
    uint64_t rem = e - perm * pt.per_perm;
    int64_t v[kMaxPos0Roles];
    for (int r = 0; r < pt.R; ++r) {
      v[r] = ts.ints[rem % ts.nI];  // t = 0 values
      rem /= ts.nI;
    }
    const int pA = perms[perm * sp.nA + sp.arr_of_role[0]];
    const int pB = perms[perm * sp.nA + sp.arr_of_role[1]];
    const int pC = perms[perm * sp.nA + sp.arr_of_role[2]];
    const double* A = ts.init + ts.region_off[pA];
    const double* B = ts.init + ts.region_off[pB];
    const double want = ts.fin[ts.region_off[pC]];
    const bool f32 = ts.is_f32[pC] != 0;
    const int64_t lenA = ts.region_len[pA], lenB = ts.region_len[pB];
    uint8_t res = 2;
    double acc = 0.0;
    if (sp.sem == ATC_SEM_GEMM) {
      const int64_t k = v[0], ld = v[1];  // ld = ldb (row) or lda (col)
      const bool row = sp.layout == ATC_LAYOUT_ROW;
      if (k >= 1 && ld >= 0) {
        const int64_t amax = row ? k - 1 : (k - 1) * ld, bmax = row ? (k - 1) * ld : k - 1;
        if (amax < lenA && bmax < lenB) {
          for (int64_t p = 0; p < k; ++p) acc = dadd(acc, dmul(row ? A[p] : A[p * ld], row ? B[p * ld] : B[p]));
          res = mismatch(round_region(acc, f32), want, f32) ? 1 : 0;
        }
      } else if (k < 1) {
        res = mismatch(round_region(0.0, f32), want, f32) ? 1 : 0;
      }
    } else {
      const int64_t c = v[0], h = v[1], w = v[2], r = v[3], s = v[4];
      uint8_t res1 = 2;
      if (c >= 1 && r >= 1 && s >= 1 && h >= 0 && w >= 0) {
        const int64_t imax = ((c - 1) * h + (r - 1)) * w + (s - 1), wmax = c * r * s - 1;
        const bool ok0 = imax >= 0 && imax < lenA && wmax < lenB;
        const bool ok1 = out1 && imax >= 0 && imax + 1 < lenA && wmax < lenB && ts.region_len[pC] > 1;
        if (ok0 || ok1) {
          // positions 0 and 1 in one pass (each its own reference-order sum); the
          // indices are < len(region) < 2^31
          double acc1 = 0.0;
          const int ci = (int)c, hi = (int)h, wi = (int)w, ri = (int)r, si = (int)s;
          for (int z = 0; z < ci; ++z)
            for (int u = 0; u < ri; ++u) {
              const double* a = A + (z * hi + u) * wi;
              const double* b = B + (z * ri + u) * si;
              for (int t = 0; t < si; ++t) {
                const double bv = b[t];
                if (ok0) acc = dadd(acc, dmul(a[t], bv));
                if (ok1) acc1 = dadd(acc1, dmul(a[t + 1], bv));
              }
            }
          if (ok0) res = mismatch(round_region(acc, f32), want, f32) ? 1 : 0;
          if (ok1) res1 = mismatch(round_region(acc1, f32), ts.fin[ts.region_off[pC] + 1], f32) ? 1 : 0;
        }
      } else {
        res = mismatch(round_region(0.0, f32), want, f32) ? 1 : 0;
      }
      if (out1) out1[e] = res1;
    }
    out[e] = res;
  }
}

// Per-binding integer screen over [begin, begin + n) of the Appendix C space.
// Each thread walks a run of consecutive indices with an odometer over the
// size-map digits (no per-binding division).  Rejections are counted per reason
// in registers and reduced per warp / block; survivors are queued for K2.
constexpr int kRun = 16;

__global__ void __launch_bounds__(256) k_screen_enum(TestsetView ts, SpecView sp, BindingSource src, uint64_t n,
                                                      Pos0Table pt, uint64_t* surv, uint64_t surv_cap,
                                                      unsigned long long* surv_cnt,
                                                      unsigned long long* reason_hist) {
  __shared__ int64_t s_u0[kMaxInts];
  __shared__ unsigned int s_hist[ATC_REASON_COUNT];
  if (threadIdx.x < ts.nI) s_u0[threadIdx.x] = ts.ints[threadIdx.x];
  if (threadIdx.x < ATC_REASON_COUNT) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const int nI = ts.nI, nS = sp.nS;
  const int tpC_base = 0;  // t = 0
  unsigned int cnt[ATC_REASON_COUNT] = {0, 0, 0, 0, 0};
  const uint64_t runs = (n + kRun - 1) / kRun;
  for (uint64_t run = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; run < runs;
       run += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t lo = run * kRun;
    const int len = (int)min((uint64_t)kRun, n - lo);
    // decode the first index of the run
    const uint64_t g = src.begin + lo;
    uint64_t perm = g / src.size_maps;
    uint64_t s = g - perm * src.size_maps;
    int digit[ATC_MAX_SIZES];
#pragma unroll
    for (int q = 0; q < ATC_MAX_SIZES; ++q) {
      if (q < nS) {
        const uint64_t d = s / (uint64_t)nI;
        digit[q] = (int)(s - d * (uint64_t)nI);
        s = d;
      }
    }
    for (int j = 0; j < len; ++j) {
      int ptr_of[ATC_MAX_ARRAYS];
#pragma unroll
      for (int a = 0; a < ATC_MAX_ARRAYS; ++a)
        if (a < sp.nA) ptr_of[a] = src.perms[perm * sp.nA + a];
      int64_t sz[ATC_MAX_SIZES];
#pragma unroll
      for (int q = 0; q < ATC_MAX_SIZES; ++q)
        if (q < nS) sz[q] = s_u0[digit[q]];
      int r = 0;
      if (!ts.test_ok[0]) r = ATC_FAIL_TESTSET;
      if (!r) r = extent_check(sp, sz, ptr_of, ts.region_len);
      Dims d;
      if (!r) {
        resolve_dims(sp, sz, d);
        r = ub_check(sp, d, ptr_of, ts.region_len);
      }
      if (!r) {
        // write-set check: every dirty position must be written
        const int pC = ptr_of[sp.arr_of_role[2]];
        const int tpC = tpC_base + pC;
        if (sp.sem == ATC_SEM_GEMM) {
          const bool row = sp.layout == ATC_LAYOUT_ROW;
          const int m = (int)d.m, nn = (int)d.n, ldc = (int)d.ldc;
          const int nd = ts.dirty_cnt[tpC];
          const int32_t* dirty = ts.dirty_pos + ts.dirty_off[tpC];
          if (m < 1 || nn < 1) {
            if (nd) r = ATC_FAIL_MISMATCH;
          } else {
            for (int e = 0; e < nd; ++e)
              if (!gemm_written(row, __ldg(dirty + e), m, nn, ldc)) {
                r = ATC_FAIL_MISMATCH;
                break;
              }
          }
          if (!r && m >= 1 && nn >= 1) {
            uint64_t key = 0, mul = 1;
            for (int k = 0; k < pt.R; ++k) {
              key += (uint64_t)digit[pt.q[k]] * mul;
              mul *= (uint64_t)nI;
            }
            if (__ldg(pt.table + perm * pt.per_perm + key) == 1) r = ATC_FAIL_MISMATCH;
          }
        } else {
          const int64_t wext = d.cn * d.ck * d.coh * d.cow;
          if (ts.dirty_max[tpC] >= wext) r = ATC_FAIL_MISMATCH;
          if (!r && wext > 0) {
            uint64_t key = 0, mul = 1;
            for (int k = 0; k < pt.R; ++k) {
              key += (uint64_t)digit[pt.q[k]] * mul;
              mul *= (uint64_t)nI;
            }
            if (__ldg(pt.table + perm * pt.per_perm + key) == 1) r = ATC_FAIL_MISMATCH;
          }
        }
      }
      if (r > 0) {
#pragma unroll
        for (int rr = 1; rr < ATC_REASON_COUNT; ++rr) cnt[rr] += (r == rr);
      } else {
        const unsigned long long slot = atomicAdd(surv_cnt, 1ull);
        if (slot < surv_cap) surv[slot] = lo + j;
      }
      // odometer: next size map (digit 0 fastest), carrying into the permutation
      for (int q = 0; q < nS; ++q) {
        if (++digit[q] < nI) break;
        digit[q] = 0;
        if (q == nS - 1) ++perm;
      }
    }
  }
  // per-reason reduction: warp shuffle, one shared atomic per warp, one global per block
#pragma unroll
  for (int r = 1; r < ATC_REASON_COUNT; ++r) {
    unsigned int v = cnt[r];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_hist[r], v);
  }
  __syncthreads();
  if (threadIdx.x < ATC_REASON_COUNT && s_hist[threadIdx.x])
    atomicAdd(&reason_hist[threadIdx.x], (unsigned long long)s_hist[threadIdx.x]);
}


// ------------------------------------------------------------------ K2 -------

// The verdict of binding `idx` at test t computed by one warp (every lane returns
// it): the scalar checks of run_dispatch / bounds, then the dirty set and the
// written outputs 32 at a time (lanes split the write set, __any_sync early exit).
// screened: an enumerated conv space of the bundled conv2d layout (the pair
// screen's precondition: size params 0..8 = n, c, h, w, k, r, s, oh, ow; arrays
// in, weights, out = 0, 1, 2) — the same checks on sizes read straight off the
// nine digits, without the generic decode.
// stop (optional, with parts > 1): the binding's shared key — a part stops early once
// another part has folded a t = 0 failure into it.
__device__ int warp_verdict(const TestsetView& ts, const SpecView& sp, const BindingSource& src, uint64_t idx, int t,
                            int mode, int lane, bool screened = false, int part = 0, int parts = 1,
                            const int32_t* stop = nullptr) {
  int ptr_of[ATC_MAX_ARRAYS];
  int r = 0;
  Dims d;
  if (screened) {
    const uint64_t g = src.begin + idx;
    const uint64_t perm = div_small_q(g, src.size_maps);
    uint64_t s = g - perm * src.size_maps;
    int64_t v[9];
    const int64_t* tints = ts.ints + (size_t)t * ts.nI;
    if (s < (1ull << 31)) {
      uint32_t s32 = (uint32_t)s;
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const uint32_t dq = div_nI(ts, s32);
        v[q] = tints[s32 - dq * (uint32_t)ts.nI];
        s32 = dq;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const uint64_t dq = s / (uint64_t)ts.nI;
        v[q] = tints[s - dq * (uint64_t)ts.nI];
        s = dq;
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) ptr_of[a] = src.perms[perm * 3 + a];
    d.cn = v[0], d.cc = v[1], d.ch = v[2], d.cw = v[3], d.ck = v[4], d.cr = v[5], d.cs = v[6], d.coh = v[7],
    d.cow = v[8];
    if (!ts.test_ok[t]) r = ATC_FAIL_TESTSET;
    if (!r) {  // extent_check over in (n,c,h,w), weights (k,c,r,s), out (n,k,oh,ow)
      bool pos = true;
#pragma unroll
      for (int q = 0; q < 9; ++q) pos = pos && v[q] >= 1;
      if (!pos || ts.region_len[ptr_of[0]] < v[0] * v[1] * v[2] * v[3] ||
          ts.region_len[ptr_of[1]] < v[4] * v[1] * v[5] * v[6] || ts.region_len[ptr_of[2]] < v[0] * v[4] * v[7] * v[8])
        r = ATC_FAIL_DISPATCH;
    }
  } else {
    int int_of[ATC_MAX_SIZES];
    decode_binding(src, sp, ts.nI, idx, ptr_of, int_of);
    int64_t sz[ATC_MAX_SIZES];
    for (int q = 0; q < sp.nS; ++q) sz[q] = ts.ints[t * ts.nI + int_of[q]];
    if (!ts.test_ok[t]) r = ATC_FAIL_TESTSET;
    if (!r) r = extent_check(sp, sz, ptr_of, ts.region_len);
    resolve_dims(sp, sz, d);
  }
  if (!r) r = ub_check(sp, d, ptr_of, ts.region_len);
  if (r) return r;
  const int pA = ptr_of[sp.arr_of_role[0]], pB = ptr_of[sp.arr_of_role[1]], pC = ptr_of[sp.arr_of_role[2]];
  const int tpA = t * ts.nP + pA, tpB = t * ts.nP + pB, tpC = t * ts.nP + pC;
  const double* __restrict__ A = ts.init + ts.region_off[tpA];
  const double* __restrict__ B = ts.init + ts.region_off[tpB];
  const double* __restrict__ F = ts.fin + ts.region_off[tpC];
  const bool f32 = ts.is_f32[pC] != 0;
  const int ndirty = ts.dirty_cnt[tpC];
  const int32_t* dirty = ts.dirty_pos + ts.dirty_off[tpC];
  bool bad = false;
  if (sp.sem == ATC_SEM_GEMM) {
    const bool row = sp.layout == ATC_LAYOUT_ROW;
    const int m = (int)d.m, n = (int)d.n, k = (int)d.k, lda = (int)d.lda, ldb = (int)d.ldb, ldc = (int)d.ldc;
    if (m < 1 || n < 1) {
      bad = ndirty > 0;
    } else {
      for (int e = lane; e < ndirty && !bad; e += 32) bad = !gemm_written(row, __ldg(dirty + e), m, n, ldc);
      bad = __any_sync(0xffffffffu, bad);
      const bool overlap = row ? (ldc < n && m > 1) : (ldc < m && n > 1);
      const int outs = m * n;
      if (mode == ATC_MODE_FP64 && outs > 32) {
        // four outputs per lane per step: four independent accumulation chains (each in
        // the reference's p order), as the conv check does — long m*n*k checks (config 1's
        // 64^3) are latency bound on one dependent chain per lane
        constexpr int MO = 4;
        for (int o0 = part * 32 * MO; o0 < outs && !bad; o0 += parts * 32 * MO) {
          const double* ap[MO];
          const double* bp[MO];
          int pos[MO];
#pragma unroll
          for (int q = 0; q < MO; ++q) {
            const int o = o0 + q * 32 + lane;
            pos[q] = -1;
            ap[q] = A;
            bp[q] = B;
            if (o < outs) {
              const int i = o / n, j = o - (o / n) * n;
              if (!overlap || gemm_last_writer(row, i, j, m, ldc)) {
                pos[q] = row ? i * ldc + j : j * ldc + i;
                ap[q] = row ? A + i * lda : A + i;
                bp[q] = row ? B + j : B + j * ldb;
              }
            }
          }
          const int sa = row ? 1 : lda, sb = row ? ldb : 1;
          double acc[MO] = {0.0, 0.0, 0.0, 0.0};
          // operands of U consecutive p loaded ahead of their (in-order) multiply-adds:
          // the loads of a block are independent, so their latencies overlap
          constexpr int U = 8;
          int p = 0;
          for (; p + U <= k; p += U) {
            double av[U][MO], bv[U][MO];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
              for (int q = 0; q < MO; ++q) {
                av[u][q] = __ldg(ap[q] + (p + u) * sa);
                bv[u][q] = __ldg(bp[q] + (p + u) * sb);
              }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
              for (int q = 0; q < MO; ++q) acc[q] = dadd(acc[q], dmul(av[u][q], bv[u][q]));
          }
          for (; p < k; ++p) {
#pragma unroll
            for (int q = 0; q < MO; ++q) acc[q] = dadd(acc[q], dmul(ap[q][p * sa], bp[q][p * sb]));
          }
          bool mm = false;
#pragma unroll
          for (int q = 0; q < MO; ++q)
            if (pos[q] >= 0) mm = mm || mismatch(round_region(acc[q], f32), __ldg(F + pos[q]), f32);
          bad = __any_sync(0xffffffffu, mm);
        }
        return bad ? ATC_FAIL_MISMATCH : 0;
      }
      if (part > 0) return bad ? ATC_FAIL_MISMATCH : 0;  // short checks: part 0 alone
      for (int o0 = 0; o0 < outs && !bad; o0 += 32) {
        const int o = o0 + lane;
        bool mm = false;
        if (o < outs) {
          const int i = o / n, j = o - (o / n) * n;
          if (!overlap || gemm_last_writer(row, i, j, m, ldc)) {
            const double* a = row ? A + i * lda : A + i;
            const double* b = row ? B + j : B + j * ldb;
            const int sa = row ? 1 : lda, sb = row ? ldb : 1;
            mm = position_mismatch(
                mode, k, __ldg(F + (row ? i * ldc + j : j * ldc + i)), f32,
                [&] { return gemm_dot64(a, sa, b, sb, k); }, [&](float& S) { return gemm_dot32(a, sa, b, sb, k, S); });
          }
        }
        bad = __any_sync(0xffffffffu, mm);
      }
    }
  } else {
    const int N = (int)d.cn, C = (int)d.cc, H = (int)d.ch, W = (int)d.cw, K = (int)d.ck, R = (int)d.cr,
              S = (int)d.cs, OH = (int)d.coh, OW = (int)d.cow;
    const int64_t wext = (int64_t)N * K * OH * OW;
    bad = ts.dirty_max[tpC] >= wext;
    if (mode == ATC_MODE_FP64) {
      // four outputs per lane per step: four independent accumulation chains (each in
      // the reference's order) hide the dependent-add latency of long checks
      constexpr int MO = 4;
      // part / parts: this warp's share of the output steps (the others run in other warps)
      int steps = 0;
      for (int o0 = part * 32 * MO; o0 < (int)wext && !bad; o0 += parts * 32 * MO) {
        if (stop && (++steps & 3) == 0) {  // every fourth step: has another part decided it?
          int k = lane == 0 ? *(volatile const int32_t*)stop : kPassKey;
          k = __shfl_sync(0xffffffffu, k, 0);
          if (k < fail_key(t + 1, 0)) break;  // failed at test <= t: this part cannot lower it
        }
        const double* inp[MO];
        const double* wtp[MO];
        int oo[MO];
#pragma unroll
        for (int m = 0; m < MO; ++m) {
          const int o = o0 + m * 32 + lane;
          oo[m] = o < wext ? o : -1;
          int rem = o < wext ? o : 0;
          const int x = rem % OW; rem /= OW;
          const int y = rem % OH; rem /= OH;
          const int q = rem % K;
          const int b = rem / K;
          inp[m] = A + ((b * C) * H + y) * W + x;
          wtp[m] = B + (q * C) * R * S;
        }
        double acc[MO];
        conv_dot64_multi<MO>(inp, wtp, C, R, S, H, W, acc);
        bool mm = false;
#pragma unroll
        for (int m = 0; m < MO; ++m)
          if (oo[m] >= 0) mm = mm || mismatch(round_region(acc[m], f32), __ldg(F + oo[m]), f32);
        bad = __any_sync(0xffffffffu, mm);
      }
      return bad ? ATC_FAIL_MISMATCH : 0;
    }
    for (int o0 = 0; o0 < (int)wext && !bad; o0 += 32) {
      const int o = o0 + lane;
      bool mm = false;
      if (o < wext) {
        int rem = o;
        const int x = rem % OW; rem /= OW;
        const int y = rem % OH; rem /= OH;
        const int q = rem % K;
        const int b = rem / K;
        const double* in = A + ((b * C) * H + y) * W + x;
        const double* wt = B + (q * C) * R * S;
        mm = position_mismatch(
            mode, C * R * S, __ldg(F + o), f32, [&] { return conv_dot64(in, wt, C, R, S, H, W); },
            [&](float& Sa) { return conv_dot32(in, wt, C, R, S, H, W, Sa); });
      }
      bad = __any_sync(0xffffffffu, mm);
    }
  }
  return bad ? ATC_FAIL_MISMATCH : 0;
}

// K2a: one WARP per survivor, test t = 0 only.  Most K1 survivors agree with the
// user program at output positions 0 and 1 but not elsewhere.  Survivors of t = 0
// are appended to `next` for K2b.
// K2-pre (conv): one THREAD per survivor, test t = 0, a few probe outputs — where
// wrong bindings that agree at positions 0 and 1 first differ: position 2, the
// first output of row 1 / filter 1 / image 1, the one after the original's last
// write.  A mismatch there decides the binding (reason 1 at t = 0, as the full
// check would); the rest go to K2a through `pend`.  Gemm spaces pass everything.
// screened (enumerated conv survivors of k_screen_conv_pairs, bundled conv2d
// layout): K1 has already passed t = 0's test, extent, UB and written-set checks
// exactly, so only the probes run, on sizes read straight off the nine digits.
__global__ void __launch_bounds__(256) k_confirm_pre(TestsetView ts, SpecView sp, BindingSource src,
                                                     const uint64_t* surv, const unsigned long long* surv_cnt,
                                                     uint64_t surv_cap, int32_t* surv_keys, uint32_t* pend,
                                                     unsigned long long* pend_cnt, int mode, int screened) {
  unsigned long long cnt = *surv_cnt;
  if (cnt > surv_cap) cnt = surv_cap;
  for (uint64_t si = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; si < cnt;
       si += (uint64_t)gridDim.x * blockDim.x) {
    bool decided = false;
    if (screened) {
      const uint64_t g = src.begin + surv[si];
      const uint64_t perm = div_small_q(g, src.size_maps);
      uint64_t s = g - perm * src.size_maps;
      int32_t v[9];
      if (s < (1ull << 31)) {
        uint32_t s32 = (uint32_t)s;
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          const uint32_t dq = div_nI(ts, s32);
          v[q] = (int32_t)ts.ints[s32 - dq * (uint32_t)ts.nI];
          s32 = dq;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          const uint64_t dq = s / (uint64_t)ts.nI;
          v[q] = (int32_t)ts.ints[s - dq * (uint64_t)ts.nI];
          s = dq;
        }
      }
      const int N = v[0], C = v[1], H = v[2], W = v[3], K = v[4], R = v[5], S = v[6], OH = v[7], OW = v[8];
      const int pA = src.perms[perm * 3 + 0], pB = src.perms[perm * 3 + 1], pC = src.perms[perm * 3 + 2];
      const double* __restrict__ A = ts.init + ts.region_off[pA];
      const double* __restrict__ B = ts.init + ts.region_off[pB];
      const double* __restrict__ F = ts.fin + ts.region_off[pC];
      const bool f32 = ts.is_f32[pC] != 0;
      const int64_t wext = (int64_t)N * K * OH * OW;
      const int64_t probes[6] = {2, OW, (int64_t)OW * OH, (int64_t)OW * OH * K, (int64_t)ts.dirty_max[pC] + 1, 3};
      for (int i = 0; i < 6 && !decided; ++i) {
        const int64_t o = probes[i];
        if (o < 2 || o >= wext) continue;
        int rem = (int)o;
        const int x = rem % OW; rem /= OW;
        const int y = rem % OH; rem /= OH;
        const int q = rem % K;
        const int b = rem / K;
        const double* in = A + ((b * C) * H + y) * W + x;
        const double* wt = B + (q * C) * R * S;
        if (position_mismatch(
                mode, C * R * S, __ldg(F + o), f32, [&] { return conv_dot64_b8(in, wt, C, R, S, H, W); },
                [&](float& Sa) { return conv_dot32(in, wt, C, R, S, H, W, Sa); })) {
          surv_keys[si] = fail_key(0, ATC_FAIL_MISMATCH);
          decided = true;
        }
      }
    } else if (sp.sem == ATC_SEM_CONV2D) {
      int ptr_of[ATC_MAX_ARRAYS], int_of[ATC_MAX_SIZES];
      decode_binding(src, sp, ts.nI, surv[si], ptr_of, int_of);
      int64_t sz[ATC_MAX_SIZES];
      for (int q = 0; q < sp.nS; ++q) sz[q] = ts.ints[int_of[q]];
      int r = 0;
      if (!ts.test_ok[0]) r = ATC_FAIL_TESTSET;
      if (!r) r = extent_check(sp, sz, ptr_of, ts.region_len);
      Dims d;
      resolve_dims(sp, sz, d);
      if (!r) r = ub_check(sp, d, ptr_of, ts.region_len);
      if (r) {
        surv_keys[si] = fail_key(0, r);
        decided = true;
      } else {
        const int pA = ptr_of[sp.arr_of_role[0]], pB = ptr_of[sp.arr_of_role[1]], pC = ptr_of[sp.arr_of_role[2]];
        const double* __restrict__ A = ts.init + ts.region_off[pA];
        const double* __restrict__ B = ts.init + ts.region_off[pB];
        const double* __restrict__ F = ts.fin + ts.region_off[pC];
        const bool f32 = ts.is_f32[pC] != 0;
        const int N = (int)d.cn, C = (int)d.cc, H = (int)d.ch, W = (int)d.cw, K = (int)d.ck, R = (int)d.cr,
                  S = (int)d.cs, OH = (int)d.coh, OW = (int)d.cow;
        const int64_t wext = (int64_t)N * K * OH * OW;
        const int dmax = ts.dirty_max[pC];
        if (dmax >= wext) {
          surv_keys[si] = fail_key(0, ATC_FAIL_MISMATCH);
          decided = true;
        } else {
          const int64_t probes[6] = {2, OW, (int64_t)OW * OH, (int64_t)OW * OH * K, (int64_t)dmax + 1, 3};
          for (int i = 0; i < 6 && !decided; ++i) {
            const int64_t o = probes[i];
            if (o < 2 || o >= wext) continue;
            int rem = (int)o;
            const int x = rem % OW; rem /= OW;
            const int y = rem % OH; rem /= OH;
            const int q = rem % K;
            const int b = rem / K;
            const double* in = A + ((b * C) * H + y) * W + x;
            const double* wt = B + (q * C) * R * S;
            if (position_mismatch(
                    mode, C * R * S, __ldg(F + o), f32, [&] { return conv_dot64_b8(in, wt, C, R, S, H, W); },
                    [&](float& Sa) { return conv_dot32(in, wt, C, R, S, H, W, Sa); })) {
              surv_keys[si] = fail_key(0, ATC_FAIL_MISMATCH);
              decided = true;
            }
          }
        }
      }
    }
    if (!decided) {
      surv_keys[si] = kPassKey;  // lazy K2a / K2b fold failures in with atomicMin
      pend[atomicAdd(pend_cnt, 1ull)] = (uint32_t)si;
    }
  }
}

// K2a: one WARP per pending survivor (all survivors without K2-pre), test t = 0
// only: every written output, 32 per step.  Survivors of t = 0 are appended to
// `next` for K2b.
// lazy (enumerated ranges, which report reasons but not failing tests): K2b has
// already run over the pending list, and t = 0 is checked only where it can change
// the reason — a binding whose first failure at t >= 1 is a mismatch is a mismatch
// whatever t = 0 gives (K2-pre has passed t = 0's scalar checks).
__global__ void __launch_bounds__(256) k_confirm_t0(TestsetView ts, SpecView sp, BindingSource src,
                                                    const uint64_t* surv, const unsigned long long* surv_cnt,
                                                    uint64_t surv_cap, int32_t* surv_keys, const uint32_t* pend,
                                                    const unsigned long long* pend_cnt, uint32_t* next,
                                                    unsigned long long* next_cnt, int mode, int lazy, int screened,
                                                    int gemm_parts) {
  const int lane = threadIdx.x & 31;
  unsigned long long cnt = pend ? *pend_cnt : *surv_cnt;
  if (cnt > surv_cap) cnt = surv_cap;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  // warp-major numbering: consecutive items land in different CTAs (different SMs) —
  // the few long full-length checks do not share an SM
  // lazy conv (FP64): the few bindings still needing t = 0 are mostly full-length checks
  // — eight warps share one binding's outputs and fold failures in with atomicMin
  // heavy gemm spaces (gemm_parts > 1; keys initialised, K2b over every survivor): the
  // same split of one binding's outputs over warps
  const int parts = lazy && sp.sem == ATC_SEM_CONV2D && mode == ATC_MODE_FP64 ? 8 : gemm_parts > 1 ? gemm_parts : 1;
  if (parts > 1) {
    const uint64_t work = cnt * (uint64_t)parts;
    for (uint64_t w = (uint64_t)(threadIdx.x / 32) * gridDim.x + blockIdx.x; w < work; w += warps) {
      const uint64_t wi = w / (uint64_t)parts;
      const int part = (int)(w - wi * (uint64_t)parts);
      const uint64_t si = pend ? pend[wi] : wi;
      const int32_t k = *(volatile int32_t*)(surv_keys + si);
      if (k != kPassKey && ((k & 7) == ATC_FAIL_MISMATCH || k < fail_key(1, 0))) continue;  // decided
      const int r = warp_verdict(ts, sp, src, surv[si], 0, mode, lane, screened != 0, part, parts, surv_keys + si);
      if (lane == 0 && r) atomicMin(&surv_keys[si], fail_key(0, r));
    }
    return;
  }
  for (uint64_t wi = (uint64_t)(threadIdx.x / 32) * gridDim.x + blockIdx.x; wi < cnt; wi += warps) {
    const uint64_t si = pend ? pend[wi] : wi;
    if (lazy) {
      const int32_t k = surv_keys[si];
      if (k != kPassKey && (k & 7) == ATC_FAIL_MISMATCH) continue;
    }
    const int r = warp_verdict(ts, sp, src, surv[si], 0, mode, lane, screened != 0);
    if (lane == 0) {
      if (r) {
        surv_keys[si] = fail_key(0, r);
      } else if (!lazy) {
        surv_keys[si] = kPassKey;
        const unsigned long long slot = atomicAdd(next_cnt, 1ull);
        next[slot] = (uint32_t)si;
      }
    }
  }
}

// K2b: one WARP per (t = 0 passer, t >= 1) — many (binding, t) items in flight
// per SM, each with its own scalar prologue; an item is skipped once a lower t of
// the same binding has failed (the atomicMin result is unchanged by the skip).
// sel == nullptr: every survivor (keys initialised by k_init_keys, t = 0 failures
// already folded in by K2a); parts > 1: a (binding, t) item's outputs split over
// `parts` warps (long gemm checks), failures folded with atomicMin.
__global__ void __launch_bounds__(256) k_confirm_warp(TestsetView ts, SpecView sp, BindingSource src,
                                                      const uint64_t* surv, uint64_t surv_cap, int32_t* surv_keys,
                                                      const uint32_t* sel, const unsigned long long* sel_cnt,
                                                      int mode, int screened, int parts) {
  const int lane = threadIdx.x & 31;
  unsigned long long cnt = *sel_cnt;
  if (cnt > surv_cap) cnt = surv_cap;
  const int nt = ts.T - 1;
  if (nt <= 0 || cnt == 0) return;
  const uint64_t work = cnt * (uint64_t)nt * (uint64_t)parts;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  // t-major: every binding's t = 1 item is dispatched before any t = 2 item, so the
  // later items of bindings that fail early are mostly skipped
  for (uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; w < work; w += warps) {
    const uint64_t item = w / (uint64_t)parts;
    const int part = (int)(w - item * (uint64_t)parts);
    const uint64_t tt = item / cnt;
    const uint32_t si = sel ? sel[item - tt * cnt] : (uint32_t)(item - tt * cnt);
    const int t = 1 + (int)tt;
    if (*(volatile int32_t*)(surv_keys + si) < fail_key(t, 0)) continue;  // failed at a lower t already
    const int r = warp_verdict(ts, sp, src, surv[si], t, mode, lane, screened != 0, part, parts,
                               parts > 1 ? surv_keys + si : nullptr);
    if (lane == 0 && r) atomicMin(&surv_keys[si], fail_key(t, r));
  }
}

// kPassKey for every survivor K1 queued (the count is on the device).
__global__ void k_init_keys(int32_t* keys, const unsigned long long* cnt, uint64_t cap) {
  unsigned long long n = *cnt;
  if (n > cap) n = cap;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = kPassKey;
}

// Merge K2 results into the per-binding keys of an explicit list.
__global__ void k_merge_keys(const uint64_t* surv, const unsigned long long* surv_cnt, uint64_t cap,
                             const int32_t* surv_keys, int32_t* keys) {
  unsigned long long cnt = *surv_cnt;
  if (cnt > cap) cnt = cap;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x)
    keys[surv[i]] = surv_keys[i];
}

__global__ void k_keys_to_verdicts(const int32_t* keys, int64_t n, int8_t* fail_t, int8_t* reason) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = keys[i];
    fail_t[i] = k == kPassKey ? (int8_t)-1 : (int8_t)(k >> 3);
    reason[i] = k == kPassKey ? (int8_t)0 : (int8_t)(k & 7);
  }
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace atc

namespace atc {
// Enumerated spaces: fold the K2 outcome of every survivor into the passing list
// (global indices) and the reason histogram, so the host reads one small block.
__global__ void k_finalize(const uint64_t* surv, const unsigned long long* surv_cnt, uint64_t cap,
                           const int32_t* surv_keys, uint64_t base, uint64_t* res, uint64_t res_cap,
                           unsigned long long* hist) {
  __shared__ unsigned int s_hist[ATC_REASON_COUNT];
  if (threadIdx.x < ATC_REASON_COUNT) s_hist[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long cnt = *surv_cnt;
  if (blockIdx.x == 0 && threadIdx.x == 0) res[0] = cnt;
  if (cnt > cap) return;  // overflow: the host retries with smaller chunks
  unsigned int local[ATC_REASON_COUNT] = {0, 0, 0, 0, 0};
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t k = surv_keys[i];
    if (k == kPassKey) {
      const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(res + 1), 1ull);
      if (slot < res_cap) res[2 + slot] = base + surv[i];
    } else {
#pragma unroll
      for (int r = 1; r < ATC_REASON_COUNT; ++r) local[r] += (k & 7) == r;
    }
  }
#pragma unroll
  for (int r = 1; r < ATC_REASON_COUNT; ++r) {
    unsigned int v = local[r];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_hist[r], v);
  }
  __syncthreads();
  if (threadIdx.x < ATC_REASON_COUNT && s_hist[threadIdx.x])
    atomicAdd(&hist[threadIdx.x], (unsigned long long)s_hist[threadIdx.x]);
}
}  // namespace atc

namespace atc {
// ------------------------------------------------------- small-space sweep --
// Every small enumerated space of a sweep (the gemm spaces: 162 .. 279,936
// bindings) in three launches instead of a chain of six per space (written-set
// table, position-0 table, row screen, K2a, K2b, finalize — each mostly ramp-up
// and tail):
//   k_sweep_small     CTA slices of every job: thread per binding, t = 0 by
//                     thread_check (run_dispatch extents, access bounds, the written
//                     set, up to `budget` output positions, exact FP64); rejections
//                     go to the job's histogram, the rest to one global survivor
//                     list (job, index);
//   k_confirm_small   warp per (survivor, t) over the whole grid, t-major (K2b's
//                     order): warp_verdict, atomicMin of t*8 + reason;
//   k_finalize_small  thread per survivor: passing indices into the job's block
//                     ([1] count, [2 ..) global indices), failures into its
//                     histogram; [0] += the job's K1 survivors.
// On survivor-list overflow every job's [0] is marked and the host re-runs them
// through atc_eval_enumerated.
__global__ void __launch_bounds__(256) k_sweep_small(const SmallJob* __restrict__ jobs, int n_jobs, int budget,
                                                     int mode, uint2* surv, int32_t* keys, uint64_t surv_cap,
                                                     unsigned long long* surv_cnt) {
  __shared__ unsigned int s_hist[ATC_REASON_COUNT];
  __shared__ int64_t s_ints0[kMaxInts];
  __shared__ int s_job;
  if (threadIdx.x == 0) {  // the job owning this CTA (jobs sorted by cta0)
    int lo = 0, hi = n_jobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (jobs[mid].cta0 <= blockIdx.x) lo = mid;
      else hi = mid - 1;
    }
    s_job = lo;
  }
  if (threadIdx.x < ATC_REASON_COUNT) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const int j = s_job;
  const SmallJob& J = jobs[j];
  const TestsetView ts = J.ts;
  const SpecView sp = J.sp;
  const BindingSource src = J.src;
  if (threadIdx.x < ts.nI) s_ints0[threadIdx.x] = ts.ints[threadIdx.x];
  __syncthreads();
  const uint32_t c = blockIdx.x - J.cta0;
  const uint64_t lo = J.n * c / J.ctas, hi = J.n * (c + 1) / J.ctas;
  for (uint64_t idx = lo + threadIdx.x; idx < hi; idx += blockDim.x) {
    int ptr_of[ATC_MAX_ARRAYS], int_of[ATC_MAX_SIZES];
    decode_binding(src, sp, ts.nI, idx, ptr_of, int_of);
    int64_t sz[ATC_MAX_SIZES];
    for (int q = 0; q < sp.nS; ++q) sz[q] = s_ints0[int_of[q]];
    bool complete;
    const int r = thread_check(ts, sp, ptr_of, sz, 0, budget, &complete, mode);
    if (r > 0) {
      atomicAdd(&s_hist[r], 1u);
    } else {
      const unsigned long long slot = atomicAdd(surv_cnt, 1ull);
      if (slot < surv_cap) {
        surv[slot] = make_uint2((uint32_t)j, (uint32_t)idx);
        keys[slot] = kPassKey;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < ATC_REASON_COUNT && s_hist[threadIdx.x])
    atomicAdd(&J.hist[threadIdx.x], (unsigned long long)s_hist[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_confirm_small(const SmallJob* __restrict__ jobs, int T, int mode,
                                                       const uint2* surv, int32_t* keys, uint64_t surv_cap,
                                                       const unsigned long long* surv_cnt) {
  unsigned long long cnt = *surv_cnt;
  if (cnt > surv_cap) return;
  const int lane = threadIdx.x & 31;
  const uint64_t work = cnt * (uint64_t)T;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; w < work; w += warps) {
    const uint64_t t64 = w / cnt;
    const uint64_t si = w - t64 * cnt;
    const int t = (int)t64;
    const uint2 e = surv[si];
    const SmallJob& J = jobs[e.x];
    if (t >= J.ts.T) continue;
    if (*(volatile int32_t*)(keys + si) < fail_key(t, 0)) continue;  // failed at a lower t already
    const int r = warp_verdict(J.ts, J.sp, J.src, e.y, t, mode, lane);
    if (lane == 0 && r) atomicMin(&keys[si], fail_key(t, r));
  }
}

__global__ void k_finalize_small(const SmallJob* __restrict__ jobs, int n_jobs, uint64_t prefix, const uint2* surv,
                                 const int32_t* keys, uint64_t surv_cap, const unsigned long long* surv_cnt,
                                 uint64_t overflow_mark) {
  const unsigned long long cnt = *surv_cnt;
  if (cnt > surv_cap) {  // every small job is redone by the host
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_jobs; j += gridDim.x * blockDim.x)
      jobs[j].res[0] = overflow_mark;
    return;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 e = surv[i];
    const SmallJob& J = jobs[e.x];
    atomicAdd(reinterpret_cast<unsigned long long*>(J.res), 1ull);
    const int32_t k = keys[i];
    if (k == kPassKey) {
      const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(J.res + 1), 1ull);
      if (slot < prefix) J.res[2 + slot] = J.src.begin + e.y;
    } else {
      atomicAdd(&J.hist[k & 7], 1ull);
    }
  }
}
}  // namespace atc
