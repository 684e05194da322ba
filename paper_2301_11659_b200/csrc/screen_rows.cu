// K1 for enumerated spaces: the row-hoisted integer screen (k_screen_rows).
//
// Predicate: the t = 0 part of eval_common.cuh (run_dispatch extent checks,
// access bounds, write-set/dirty check) plus the tabulated position-0 verdict
// of k_pos0_table (eval_kernels.cu); bindings that pass go to K2, which
// re-checks every output of every test.  Equivalent to k_screen_enum, which it
// replaces for the bundled spec shapes (gemm with 3 or 6 size params, conv2d
// with 9).
//
// Organisation (SURVEY.md Appendix C order): a thread owns one "row" — a fixed
// array permutation and fixed size-map digits 1..NS-1 — and walks the nI values
// of digit 0, the fastest-varying size param.  Everything independent of digit
// 0 is computed once per row: the row decode (NS-1 divisions), the role values,
// extents of arrays that do not use it, the table key, the dirty maximum.  NS
// and the semantics are template parameters so the per-size arrays unroll into
// registers, and I32 selects 32-bit index arithmetic when the host has proven
// every product fits (max t=0 size <= 215, so any product of 4 sizes < 2^31).
#include <cuda_runtime.h>

#include <type_traits>

#include "eval_common.cuh"

namespace atc {

template <int NS>
__device__ __forceinline__ int64_t pick(const int64_t (&u)[NS], int q) {
  int64_t v = 0;
#pragma unroll
  for (int i = 0; i < NS; ++i)
    if (q == i) v = u[i];
  return v;
}

template <int NS>
__device__ __forceinline__ int pick_digit(const int (&d)[NS], int q) {
  int v = 0;
#pragma unroll
  for (int i = 1; i < NS; ++i)
    if (q == i) v = d[i];
  return v;
}

// Q0MASK: compile-time set of roles bound to digit 0 (bit per ATC_SZ_* role), so
// that every quantity not depending on digit 0 is loop-invariant and hoisted by
// the compiler; kQ0Dynamic takes the set from the plan at run time.
constexpr uint32_t kQ0Dynamic = 0xFFFFFFFFu;

template <int SEM, int NS, bool I32, uint32_t Q0MASK>
__global__ void __launch_bounds__(256) k_screen_rows(TestsetView ts, SpecView sp, const uint8_t* perms,
                                                      uint64_t size_maps, uint64_t begin, uint64_t end, RowPlan plan,
                                                      uint64_t* surv, uint64_t surv_cap, unsigned long long* surv_cnt,
                                                      unsigned long long* reason_hist) {
  using I = typename std::conditional<I32, int32_t, int64_t>::type;
  __shared__ int64_t s_u0[kMaxInts];
  __shared__ unsigned int s_hist[ATC_REASON_COUNT];
  if (threadIdx.x < ts.nI) s_u0[threadIdx.x] = ts.ints[threadIdx.x];
  if (threadIdx.x < ATC_REASON_COUNT) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const int nI = ts.nI;
  const bool test_ok0 = ts.test_ok[0] != 0;
  const bool row_major = sp.layout == ATC_LAYOUT_ROW;
  unsigned int cnt1 = 0, cnt2 = 0, cnt3 = 0, cnt4 = 0;
  const uint64_t row_lo = begin / nI, row_hi = (end + nI - 1) / nI;
  // each thread owns kRowBlock consecutive rows: one full decode, then an
  // odometer step (digit 1 upwards, carrying into the permutation) per row
  constexpr int kRowBlock = 4;
  const uint64_t blocks = (row_hi - row_lo + kRowBlock - 1) / kRowBlock;
  for (uint64_t rb = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; rb < blocks;
       rb += (uint64_t)gridDim.x * blockDim.x) {
  const uint64_t row0 = row_lo + rb * kRowBlock;
  uint64_t perm = (row0 * nI) / size_maps;
  int digit[NS];
  digit[0] = 0;
  {
    uint64_t s = (row0 * nI - perm * size_maps) / nI;
    if (s < (1ull << 32)) {
      uint32_t s32 = (uint32_t)s;
#pragma unroll
      for (int q = 1; q < NS; ++q) {
        const uint32_t dq = s32 / (uint32_t)nI;
        digit[q] = (int)(s32 - dq * (uint32_t)nI);
        s32 = dq;
      }
    } else {
#pragma unroll
      for (int q = 1; q < NS; ++q) {
        const uint64_t dq = s / (uint64_t)nI;
        digit[q] = (int)(s - dq * (uint64_t)nI);
        s = dq;
      }
    }
  }
  for (int rbi = 0; rbi < kRowBlock; ++rbi) {
    const uint64_t row = row0 + rbi;
    if (row >= row_hi) break;
    if (rbi > 0) {  // odometer: next row = next value of digits 1..NS-1
      bool carry = true;
#pragma unroll
      for (int q = 1; q < NS; ++q) {
        if (carry) {
          carry = ++digit[q] == nI;
          if (carry) digit[q] = 0;
        }
      }
      if (carry) ++perm;
    }
    // ---------------- per-row setup ----------------
    const uint64_t g0 = row * nI;
    int64_t u[NS];
    u[0] = 0;
#pragma unroll
    for (int q = 1; q < NS; ++q) u[q] = s_u0[digit[q]];
    int ptr_of[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) ptr_of[a] = perms[perm * 3 + a];
    const I len_a0 = (I)ts.region_len[ptr_of[0]], len_a1 = (I)ts.region_len[ptr_of[1]],
            len_a2 = (I)ts.region_len[ptr_of[2]];
    const int pC = ptr_of[sp.arr_of_role[2]];
    const I lenA = (I)ts.region_len[ptr_of[sp.arr_of_role[0]]];
    const I lenB = (I)ts.region_len[ptr_of[sp.arr_of_role[1]]];
    const I lenC = (I)ts.region_len[pC];
    // extents without digit 0; any non-digit-0 dim < 1 fails every binding of the row
    I ext_rest[3];
    bool bad_rest = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      I e = 1;
#pragma unroll
      for (int q = 1; q < NS; ++q)
        if (plan.dim_mask[a] & (1u << q)) {
          e *= (I)u[q];
          bad_rest |= u[q] < 1;
        }
      ext_rest[a] = e;
    }
    const bool use0_a0 = plan.dim_mask[0] & 1u, use0_a1 = plan.dim_mask[1] & 1u, use0_a2 = plan.dim_mask[2] & 1u;
    const bool use0_any = use0_a0 || use0_a1 || use0_a2;
    // role values not bound to digit 0
    I rv[ATC_SZ_COUNT];
    bool r0[ATC_SZ_COUNT];
    // only the roles of this semantics (gemm m..ldc, conv n..ow)
    constexpr int kRoleLo = SEM == ATC_SEM_GEMM ? ATC_SZ_M : ATC_SZ_CN;
    constexpr int kRoleHi = SEM == ATC_SEM_GEMM ? ATC_SZ_LDC + 1 : ATC_SZ_COUNT;
#pragma unroll
    for (int rr = 0; rr < ATC_SZ_COUNT; ++rr) {
      r0[rr] = false;
      rv[rr] = 0;
      if (rr < kRoleLo || rr >= kRoleHi) continue;
      const int q = plan.role_q[rr];
      r0[rr] = q == 0;
      rv[rr] = q <= 0 ? 0 : (I)pick<NS>(u, q);
    }
    uint64_t key_rest = perm * plan.pt.per_perm;
#pragma unroll
    for (int q = 1; q < NS; ++q) key_rest += (uint64_t)digit[q] * plan.key_stride[q];
    const uint64_t key0 = plan.key_stride[0];
    const int row_tab = key0 == 0 ? __ldg(plan.pt.table + key_rest) : -1;
    const I dmaxC = (I)ts.dirty_max[pC];
    const int ndirty = ts.dirty_cnt[pC];
    const int32_t* dirty = ts.dirty_pos + ts.dirty_off[pC];

    const int v_lo = g0 < begin ? (int)(begin - g0) : 0;
    const int v_hi = g0 + nI > end ? (int)(end - g0) : nI;
    // ---------------- digit-0 loop ----------------
    for (int v = v_lo; v < v_hi; ++v) {
      const I uv = (I)s_u0[v];
      auto role = [&](int rr) -> I {
        if (Q0MASK == kQ0Dynamic) return r0[rr] ? uv : rv[rr];
        return ((Q0MASK >> rr) & 1u) ? uv : rv[rr];
      };
      int r = test_ok0 ? 0 : ATC_FAIL_TESTSET;
      if (!r) {  // run_dispatch extent checks (rewriter.cpp:136-148)
        const I e0 = use0_a0 ? ext_rest[0] * uv : ext_rest[0];
        const I e1 = use0_a1 ? ext_rest[1] * uv : ext_rest[1];
        const I e2 = use0_a2 ? ext_rest[2] * uv : ext_rest[2];
        if (bad_rest || (use0_any && uv < 1) || e0 > len_a0 || e1 > len_a1 || e2 > len_a2) r = ATC_FAIL_DISPATCH;
      }
      if (!r) {
        int tv = -1;  // position-0 table verdict, when position 0 is written
        if (SEM == ATC_SEM_GEMM) {
          const I m = role(ATC_SZ_M), n = role(ATC_SZ_N), k = role(ATC_SZ_K);
          const I lda = role(ATC_SZ_LDA), ldb = role(ATC_SZ_LDB), ldc = role(ATC_SZ_LDC);
          if (m >= 1 && n >= 1 && k >= 1) {
            if (lda < 0 || ldb < 0 || ldc < 0) {
              r = ATC_FAIL_UB;
            } else {
              const I amax = row_major ? (m - 1) * lda + (k - 1) : (k - 1) * lda + (m - 1);
              const I bmax = row_major ? (k - 1) * ldb + (n - 1) : (n - 1) * ldb + (k - 1);
              const I cmax = row_major ? (m - 1) * ldc + (n - 1) : (n - 1) * ldc + (m - 1);
              if (amax >= lenA || bmax >= lenB || cmax >= lenC) r = ATC_FAIL_UB;
            }
          }
          if (!r) {
            if (m < 1 || n < 1) {
              if (ndirty) r = ATC_FAIL_MISMATCH;
            } else {
              int need = -1;
              if (plan.gemm_need) {  // digits of m and ldc -> tabulated minimum n
                const int qm = plan.role_q[ATC_SZ_M], ql = plan.role_q[ATC_SZ_LDC];
                const int dm = qm == 0 ? v : pick_digit<NS>(digit, qm);
                const int dl = ql == 0 ? v : pick_digit<NS>(digit, ql);
                need = __ldg(plan.gemm_need + ((size_t)pC * nI + dl) * nI + dm);
              }
              if (need >= 0) {
                if ((int64_t)n < need) r = ATC_FAIL_MISMATCH;
              } else {
                for (int e = 0; e < ndirty; ++e)
                  if (!gemm_written(row_major, __ldg(dirty + e), (int)m, (int)n, (int)ldc)) {
                    r = ATC_FAIL_MISMATCH;
                    break;
                  }
              }
              if (!r) tv = row_tab >= 0 ? row_tab : __ldg(plan.pt.table + key_rest + (uint64_t)v * key0);
            }
          }
        } else {
          const I cn = role(ATC_SZ_CN), cc = role(ATC_SZ_CC), ch = role(ATC_SZ_CH), cw = role(ATC_SZ_CW);
          const I ck = role(ATC_SZ_CK), cr = role(ATC_SZ_CR), cs = role(ATC_SZ_CS);
          const I coh = plan.role_q[ATC_SZ_COH] >= 0 ? role(ATC_SZ_COH) : ch - cr + 1;
          const I cow = plan.role_q[ATC_SZ_COW] >= 0 ? role(ATC_SZ_COW) : cw - cs + 1;
          // grouped so that, with tc_n on digit 0, the n-free factors are loop-invariant
          const I wext = cn * (ck * (coh * cow));
          if (cn >= 1 && ck >= 1 && coh >= 1 && cow >= 1 && cc >= 1 && cr >= 1 && cs >= 1) {
            // = (((cn-1)*cc + (cc-1))*ch + (coh-1) + (cr-1))*cw + (cow-1) + (cs-1), expanded
            const I imax = cn * (cc * (ch * cw)) - ch * cw + (coh + cr - 2) * cw + (cow + cs - 2);
            const I wmax = ck * cc * cr * cs - 1;
            if (imax >= lenA || imax < 0 || wmax >= lenB || wext - 1 >= lenC) r = ATC_FAIL_UB;
          }
          if (!r && dmaxC >= wext) r = ATC_FAIL_MISMATCH;
          if (!r && wext > 0) tv = row_tab >= 0 ? row_tab : __ldg(plan.pt.table + key_rest + (uint64_t)v * key0);
        }
        if (tv == 1) r = ATC_FAIL_MISMATCH;
      }
      cnt1 += r == ATC_FAIL_MISMATCH;
      cnt2 += r == ATC_FAIL_DISPATCH;
      cnt3 += r == ATC_FAIL_TESTSET;
      cnt4 += r == ATC_FAIL_UB;
      if (r == 0) {
        const unsigned long long slot = atomicAdd(surv_cnt, 1ull);
        if (slot < surv_cap) surv[slot] = g0 + v - begin;
      }
    }
  }
  }  // row block
  // per-reason reduction: warp shuffle, one shared atomic per warp, one global per block
  unsigned int cnt[ATC_REASON_COUNT] = {0, cnt1, cnt2, cnt3, cnt4};
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

// ----------------------------------------------------------------------------
// k_screen_conv_planes: k_screen_rows for the bundled conv2d spec shape, with
// the loops over digits 0 and 1 (tc_n, tc_c) replaced by thresholds.
//
// Preconditions (checked by the host, capi.cu conv_thresholds_ok): roles
// tc_n .. tc_ow bound to size params 0 .. 8 in order, array dims in = (n,c,h,w),
// weights = (c,k,r,s), out = (n,k,oh,ow) in any order, in/weights/out = API
// arrays 0/1/2, every digit value |u| <= 200 (every product below is exact in
// 32 bits), nI <= 32, a position-0 table key free of digit 0.
//
// A thread owns a "plane": the nI x nI bindings sharing the permutation and
// digits 2..8 (contiguous in Appendix C order).  With x = tc_n and c = tc_c,
// every t = 0 check of the screen is a threshold on x whose bound depends on
// the plane and on c only through one small division:
//   dispatch (rewriter.cpp:136-148)  fails iff x < 1, c < 1, a digit 2..8 < 1,
//                                    c > len(wt)/(k*r*s), x > (len(in)/(h*w))/c
//                                    or x > len(out)/(k*oh*ow)   [floors]
//   access bound (UB)                fails iff x*c*h*w + Q >= len(in), i.e.
//                                    x > ((len(in) - Q - 1)/(h*w))/c, Q = the
//                                    x-free part of the last input index; the
//                                    weights/out bounds equal the extents above
//   written set                      fails iff x*k*oh*ow <= dirty_max(out)
//   position 0                       the tabulated verdict of (perm, c,h,w,r,s)
// (floor(floor(a/b)/c) = floor(a/(b*c)) for positive integers).  A row's
// verdicts over its nI values of x are then bit masks: gt[T] = the digits whose
// value exceeds T, tabulated once per CTA for T in [0, 255].  Verdicts, reason
// counts and survivors are identical to k_screen_rows (tests/test_gpu_eval.py).
constexpr int kGtCap = 255;  // > every digit value in 32-bit mode (<= 200)

// min(floor(a / b), kGtCap) for a >= 0, b >= 1, rb ~= 1/b: float estimate, exact fix-up
__device__ __forceinline__ int div_cap(int64_t a, int64_t b, float rb) {
  if (a >= b * kGtCap) return kGtCap;
  int q = (int)((float)a * rb);  // |error| < 1 since q < 256
  if ((int64_t)q * b > a) --q;
  else if ((int64_t)(q + 1) * b <= a) ++q;
  return q;
}

// min(floor(a / c), kGtCap) for 0 <= a <= kDivClamp, 1 <= c <= 200, rc ~= 1/c (exact)
constexpr int32_t kDivClamp = kGtCap * 200;  // a >= this gives kGtCap for every c <= 200
__device__ __forceinline__ int div_small(int32_t a, int32_t c, float rc) {
  int q = __float2int_rz(__int2float_rn(a) * rc);  // a < 2^24: |error| < 1
  q -= q * c > a;
  q += (q + 1) * c <= a;
  return min(q, kGtCap);
}

// min(floor(a / b), kDivClamp) for a >= 0, b >= 1
__device__ __forceinline__ int32_t clamp_div(int64_t a, int32_t b) {
  if (a >= (int64_t)b * kDivClamp) return kDivClamp;
  return (int32_t)((uint32_t)a / (uint32_t)b);  // a < 200 * 255 * b < 2^32 here (b <= 200^2)
}

__global__ void __launch_bounds__(256) k_screen_conv_planes(TestsetView ts, const uint8_t* perms,
                                                             uint64_t size_maps, uint64_t begin, uint64_t end,
                                                             RowPlan plan, uint64_t* surv, uint64_t surv_cap,
                                                             unsigned long long* surv_cnt,
                                                             unsigned long long* reason_hist) {
  constexpr int NS = 9;
  __shared__ int32_t s_u[kMaxInts];
  __shared__ float s_rcp[kMaxInts];
  __shared__ uint32_t s_gt[kGtCap + 1];
  __shared__ unsigned int s_hist[ATC_REASON_COUNT];
  const int nI = ts.nI;
  if (threadIdx.x < nI) {
    const int32_t u = (int32_t)ts.ints[threadIdx.x];
    s_u[threadIdx.x] = u;
    s_rcp[threadIdx.x] = __frcp_rn((float)(u > 0 ? u : 1));
  }
  if (threadIdx.x < ATC_REASON_COUNT) s_hist[threadIdx.x] = 0;
  for (int t = threadIdx.x; t <= kGtCap; t += blockDim.x) {
    uint32_t m = 0;
    for (int i = 0; i < nI; ++i) m |= (ts.ints[i] > t ? 1u : 0u) << i;
    s_gt[t] = m;
  }
  __syncthreads();
  const bool test_ok0 = ts.test_ok[0] != 0;
  const uint32_t per_perm = (uint32_t)plan.pt.per_perm;  // table < 256 MB: 32-bit keys
  const uint32_t ks1 = (uint32_t)plan.key_stride[1];
  const uint32_t gt0 = s_gt[0];
  const uint64_t nI2 = (uint64_t)nI * nI;
  const uint64_t planes_per_perm = size_maps / nI2;
  const uint32_t all_rows = nI >= 32 ? 0xFFFFFFFFu : ((1u << nI) - 1u);
  const uint32_t magic = (uint32_t)(0xFFFFFFFFull / (uint32_t)nI) + 1u;  // n / nI = umulhi(n, magic), n < 2^27
  unsigned int cnt1 = 0, cnt2 = 0, cnt3 = 0, cnt4 = 0;
  const uint64_t plane_lo = begin / nI2, plane_hi = (end + nI2 - 1) / nI2;
  for (uint64_t pl = plane_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; pl < plane_hi;
       pl += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p0 = pl * nI2;
    const uint64_t lo = p0 < begin ? begin : p0, hi = p0 + nI2 > end ? end : p0 + nI2;
    const unsigned int n_here = (unsigned int)(hi - lo);
    if (!test_ok0) {
      cnt3 += n_here;
      continue;
    }
    const uint64_t perm = pl / planes_per_perm;
    int digit[NS];
    {
      uint64_t s = pl - perm * planes_per_perm;  // digits 2..8
      if (s < (1ull << 27)) {
        uint32_t s32 = (uint32_t)s;
#pragma unroll
        for (int q = 2; q < NS; ++q) {
          const uint32_t dq = __umulhi(s32, magic);
          digit[q] = (int)(s32 - dq * (uint32_t)nI);
          s32 = dq;
        }
      } else if (s < (1ull << 32)) {
        uint32_t s32 = (uint32_t)s;
#pragma unroll
        for (int q = 2; q < NS; ++q) {
          const uint32_t dq = s32 / (uint32_t)nI;
          digit[q] = (int)(s32 - dq * (uint32_t)nI);
          s32 = dq;
        }
      } else {
#pragma unroll
        for (int q = 2; q < NS; ++q) {
          const uint64_t dq = s / (uint64_t)nI;
          digit[q] = (int)(s - dq * (uint64_t)nI);
          s = dq;
        }
      }
    }
    const int32_t ch = s_u[digit[2]], cw = s_u[digit[3]], ck = s_u[digit[4]], cr = s_u[digit[5]];
    const int32_t cs = s_u[digit[6]], coh = s_u[digit[7]], cow = s_u[digit[8]];
    if (min(min(min(ch, cw), min(ck, cr)), min(min(cs, coh), cow)) < 1) {
      cnt2 += n_here;  // a dim of the plane < 1: "size is not positive" for every binding
      continue;
    }
    const int p_in = perms[perm * 3 + 0], p_w = perms[perm * 3 + 1], p_out = perms[perm * 3 + 2];
    const int64_t len_in = ts.region_len[p_in], len_w = ts.region_len[p_w], len_out = ts.region_len[p_out];
    const int32_t hw = ch * cw, krs = ck * cr * cs, ext_out = ck * coh * cow;
    const float r_out = __frcp_rn((float)ext_out);
    // plane-level bounds (exact floors)
    const int64_t c_max = len_w / krs;    // weights extent: c*k*r*s <= len(wt)
    // in extent: x*c <= a_in; clamped where every quotient saturates anyway
    const int32_t a_in = clamp_div(len_in, hw);
    const int32_t q_in = -hw + (coh + cr - 2) * cw + (cow + cs - 2);
    const int64_t alim = len_in - q_in;   // UB iff x*c*h*w >= alim
    const int32_t b_in = alim > 0 ? clamp_div(alim - 1, hw) : -1;
    const bool full = lo == p0 && hi == p0 + nI2;
    const uint32_t out_fail = s_gt[div_cap(len_out, ext_out, r_out)];
    const int dmax = ts.dirty_max[p_out];
    const uint32_t dirty_fail = ~s_gt[dmax < 0 ? 0 : div_cap(dmax, ext_out, r_out)];
    uint32_t key = (uint32_t)perm * per_perm;
#pragma unroll
    for (int q = 2; q < NS; ++q) key += (uint32_t)digit[q] * (uint32_t)plan.key_stride[q];
    for (int j = 0; j < nI; ++j) {  // digit 1: tc_c
      uint32_t range = all_rows;
      if (!full) {
        const uint64_t g0 = p0 + (uint64_t)j * nI;
        if (g0 + nI <= begin || g0 >= end) continue;
        const int v_lo = g0 < begin ? (int)(begin - g0) : 0;
        const int v_hi = g0 + nI > end ? (int)(end - g0) : nI;
        range = (v_hi >= 32 ? 0xFFFFFFFFu : ((1u << v_hi) - 1u)) & ~((1u << v_lo) - 1u);
      }
      const int32_t c = s_u[j];
      if (c < 1 || c > c_max) {
        cnt2 += __popc(range);
        continue;
      }
      const float rc = s_rcp[j];
      const uint32_t dm = range & (~gt0 | out_fail | s_gt[div_small(a_in, c, rc)]);
      uint32_t ok = range & ~dm, um = 0, mm = 0;
      if (ok) {
        um = b_in < 0 ? ok : (ok & s_gt[div_small(b_in, c, rc)]);
        ok &= ~um;
        if (ok) {
          const bool tab_fail = __ldg(plan.pt.table + key + (uint32_t)j * ks1) == 1;
          mm = tab_fail ? ok : (ok & dirty_fail);
          ok &= ~mm;
        }
      }
      cnt2 += __popc(dm);
      cnt4 += __popc(um);
      cnt1 += __popc(mm);
      if (ok) {
        unsigned long long slot = atomicAdd(surv_cnt, (unsigned long long)__popc(ok));
        for (; ok; ok &= ok - 1, ++slot)
          if (slot < surv_cap) surv[slot] = p0 + (uint64_t)j * nI + (__ffs(ok) - 1) - begin;
      }
    }
  }
  unsigned int cnt[ATC_REASON_COUNT] = {0, cnt1, cnt2, cnt3, cnt4};
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

// ----------------------------------------------------------------------------
// k_cmask: verdict bits of the nI values of tc_c (the first table role, key
// stride 1): cmask[i] bit j = table[i*nI + j] == 1 (position 0).
// shift 16: the upper half gets position 0's bits OR position 1's (the rows a binding
// with ow >= 2 fails), so a reader takes word >> (ow >= 2 ? 16 : 0).
__global__ void k_cmask(const uint8_t* table, uint64_t n_words, int nI, uint32_t* cmask, int shift) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_words; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t m = 0;
    for (int j = 0; j < nI; ++j) m |= (table[i * nI + j] == 1 ? 1u : 0u) << j;
    cmask[i] = shift ? (cmask[i] | (m | (cmask[i] & 0xFFFFu)) << shift) : m;
  }
}

// k_screen_conv_pairs: k_screen_conv_planes with the loop over tc_c removed too
// (nI <= 11, so a plane's nI x nI bindings fit one 128-bit mask; bit
// c_index*nI + x_index = the binding's offset in the plane, Appendix C order).
//
// The plane's checks as masks over (x, c) pairs, from CTA-wide tables:
//   gtx[T] / gtc[T]   pairs whose x (tc_n) / c (tc_c) value exceeds T, T in [0, 255]
//   gt_prod(T)        pairs whose product x*c exceeds T (sorted products + suffix masks)
//   dispatch  = x < 1 | c < 1 | c > len(wt)/(k*r*s) | x*c > len(in)/(h*w) | x > len(out)/(k*oh*ow)
//   UB        = x*c > (len(in) - Q - 1)/(h*w)               (all, if len(in) <= Q)
//   mismatch  = x <= dirty_max(out)/(k*oh*ow) | position-0 verdict of (perm, c, h, w, r, s)
// (floors; the same thresholds as k_screen_conv_planes, now applied to all nI
// values of c at once).  Verdicts, reason counts and survivors are identical.
struct M128 {
  uint64_t lo, hi;
};
__device__ __forceinline__ M128 operator|(M128 a, M128 b) { return {a.lo | b.lo, a.hi | b.hi}; }
__device__ __forceinline__ M128 operator&(M128 a, M128 b) { return {a.lo & b.lo, a.hi & b.hi}; }
__device__ __forceinline__ M128 operator~(M128 a) { return {~a.lo, ~a.hi}; }
__device__ __forceinline__ bool any(M128 a) { return (a.lo | a.hi) != 0; }
__device__ __forceinline__ unsigned popc(M128 a) { return __popcll(a.lo) + __popcll(a.hi); }
__device__ __forceinline__ M128 bit_range(int lo, int hi) {  // bits [lo, hi), 0 <= lo <= hi <= 128
  auto upto = [](int n) -> M128 {
    if (n <= 0) return {0, 0};
    if (n < 64) return {(1ull << n) - 1, 0};
    if (n == 64) return {~0ull, 0};
    if (n < 128) return {~0ull, (1ull << (n - 64)) - 1};
    return {~0ull, ~0ull};
  };
  return upto(hi) & ~upto(lo);
}
__device__ __forceinline__ void set_bit(M128& m, int b) {
  if (b < 64) m.lo |= 1ull << b;
  else m.hi |= 1ull << (b - 64);
}

constexpr int kPairMaxInts = 11;  // nI^2 <= 121 bits

// floor(n / d) for n < 2^31 and 1 <= d < 2^31 from (m, s): m = ceil(2^(31 + s) / d)
// with s = ceil(log2 d) is < 2^32 and leaves an error below 2^-s <= 1/d, so the
// floor is exact; d = 1 is m = 0
__device__ __forceinline__ uint32_t mdiv(uint32_t n, uint32_t m, uint32_t sh) { return m ? __umulhi(n, m) >> sh : n; }
__device__ __forceinline__ void mdiv_consts(uint32_t d, uint32_t& m, uint32_t& sh) {
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;
  m = d <= 1 ? 0u : (uint32_t)(((1ull << (31 + s)) + d - 1) / d);
  sh = s ? s - 1 : 0;
}

// min(floor(a / b), cap) for 0 <= a < 2^32, 1 <= b, cap <= 65536, rb ~= 1/b (exact)
__device__ __forceinline__ int div_capn(uint32_t a, uint32_t b, float rb, int cap) {
  if ((uint64_t)a >= (uint64_t)b * (uint32_t)cap) return cap;
  int q = (int)((float)a * rb);  // q < cap: |error| < 1
  if ((uint64_t)q * b > a) --q;
  else if ((uint64_t)(q + 1) * b <= a) ++q;
  return q;
}

// lut_n > 0: products are in [.., lut_n - 1] and the dynamic shared memory holds a
// rank table (count of pair products <= T, T in [0, lut_n)) after the row table
template <int NIc>
__global__ void __launch_bounds__(kPairThreads, 1024 / kPairThreads) k_screen_conv_pairs(TestsetView ts, const uint8_t* perms, uint64_t size_maps,
                                                            uint64_t begin, uint64_t end, RowPlan plan,
                                                            uint64_t* surv, uint64_t surv_cap,
                                                            unsigned long long* surv_cnt,
                                                            unsigned long long* reason_hist, int lut_n) {
  constexpr int NS = 9;
  extern __shared__ M128 s_rowx[];  // [2^nI]: rows j of the plane for every bit j of the index
  __shared__ int32_t s_u[kMaxInts];
  __shared__ M128 s_gtx[kGtCap + 1], s_gtc[kGtCap + 1];
  __shared__ int32_t s_prod[128];  // products x*c ascending, padded with INT32_MAX
  __shared__ int s_pidx[128];
  __shared__ M128 s_pgt[129];      // s_pgt[r] = pairs of product rank >= r
  __shared__ unsigned int s_hist[ATC_REASON_COUNT];
  __shared__ M128 s_row[kPairMaxInts];   // bits [j*nI, j*nI + nI): row j of the plane
  __shared__ int32_t s_pp[128];          // product of pair b = (c digit b / nI, x digit b % nI)
  __shared__ uint8_t s_rk[128];          // stable rank of pair b's product
  __shared__ uint64_t s_div[8];          // 64-bit quotients every thread needs (computed once)
  __shared__ uint32_t s_cks[NS];
  __shared__ M128 s_okm[129];            // pairs of product rank < r that pass x >= 1, c >= 1
  __shared__ uint8_t s_cnt[129];         // their number
  __shared__ uint16_t s_skipm[8 * kPairMaxInts];  // per (in region, w digit): the h digits of skip planes
  __shared__ int32_t s_vmax[8 * kPairMaxInts];    // and the largest plane-table v over h
  const int nI = NIc ? NIc : ts.nI, nI2 = nI * nI;
  // CTA tables: built once, from O(nI^2) work per thread at most (the per-CTA
  // prologue is paid by every one of the 4 x 148 CTAs)
  if (threadIdx.x < nI) {
    s_u[threadIdx.x] = (int32_t)ts.ints[threadIdx.x];
    s_row[threadIdx.x] = bit_range(threadIdx.x * nI, threadIdx.x * nI + nI);
  }
  if (threadIdx.x < ATC_REASON_COUNT) s_hist[threadIdx.x] = 0;
  if (threadIdx.x < 128) s_prod[threadIdx.x] = INT32_MAX;
  if (threadIdx.x == 32) {
    const uint64_t nI3 = (uint64_t)nI2 * nI, planes_per_perm = size_maps / (uint64_t)nI2;
    s_div[0] = plan.pt.per_perm / (uint64_t)nI;   // cperm
    s_div[1] = planes_per_perm;
    s_div[2] = planes_per_perm / (uint64_t)nI;    // cubes per permutation
    s_div[3] = begin / nI3;                       // first cube
    s_div[4] = (end + nI3 - 1) / nI3;             // one past the last cube
    uint32_t m = 0, sh = 0;
    if (s_div[2] < (1ull << 31)) mdiv_consts((uint32_t)s_div[2], m, sh);
    s_div[5] = m;
    s_div[6] = sh;
  }
  if (threadIdx.x >= 64 && threadIdx.x < 64 + NS) {
    const int q = threadIdx.x - 64;
    s_cks[q] = q >= 2 ? (uint32_t)(plan.key_stride[q] / (uint64_t)nI) : 0u;
  }
  __syncthreads();
  if (threadIdx.x < nI2) s_pp[threadIdx.x] = s_u[threadIdx.x % nI] * s_u[threadIdx.x / nI];
  for (int m = threadIdx.x; m < (1 << nI); m += blockDim.x) {  // rows j of the plane for every bit j of m
    M128 r{0, 0};
    for (uint32_t mm = (uint32_t)m; mm; mm &= mm - 1) r = r | s_row[__ffs(mm) - 1];
    s_rowx[m] = r;
  }
  __syncthreads();
  for (int t = threadIdx.x; t <= kGtCap; t += blockDim.x) {
    uint32_t xm = 0;  // digit indices whose value exceeds t
    for (int i = 0; i < nI; ++i) xm |= (s_u[i] > t ? 1u : 0u) << i;
    M128 gx{0, 0};    // the same x bits in every row
    for (int j = 0; j < nI; ++j) {
      const int b0 = j * nI;
      if (b0 < 64) gx.lo |= (uint64_t)xm << b0;
      if (b0 + nI > 64) gx.hi |= b0 >= 64 ? (uint64_t)xm << (b0 - 64) : (uint64_t)xm >> (64 - b0);
    }
    s_gtx[t] = gx;
    s_gtc[t] = s_rowx[xm];
  }
  if (threadIdx.x < nI2) {  // stable rank of the pair's product
    const int b = threadIdx.x;
    const int32_t pr = s_pp[b];
    int rank = 0;
    for (int i = 0; i < nI2; ++i) {
      const int32_t q = s_pp[i];
      rank += q < pr || (q == pr && i < b);
    }
    s_prod[rank] = pr;
    s_pidx[rank] = b;
    s_rk[b] = (uint8_t)rank;
  }
  __syncthreads();
  uint8_t* s_rank = reinterpret_cast<uint8_t*>(s_rowx + (1 << nI));
  {  // s_pgt[r] = pairs of rank >= r: one ballot per 32 pairs (warp w takes r = w, w + 8, ...)
    const int lane = threadIdx.x & 31;
    for (int r = threadIdx.x >> 5; r <= nI2; r += blockDim.x >> 5) {
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int b = k * 32 + lane;
        w[k] = __ballot_sync(0xffffffffu, b < nI2 && s_rk[b] >= r);
      }
      if (lane == 0) s_pgt[r] = M128{(uint64_t)w[0] | (uint64_t)w[1] << 32, (uint64_t)w[2] | (uint64_t)w[3] << 32};
    }
  }
  int p2 = 1;  // power of two > nI2: branch-free search over the padded products
  while (p2 <= nI2) p2 <<= 1;
  for (int t = threadIdx.x; t < lut_n; t += blockDim.x) {  // rank = number of products <= t
    int lo = 0;
    for (int step = p2 >> 1; step > 0; step >>= 1)
      if (s_prod[lo + step - 1] <= t) lo += step;
    s_rank[t] = (uint8_t)lo;
  }
  __syncthreads();
  // per (in region, w digit, h digit): the number of pair products <= len(in)/(h*w)
  // (the s_pgt index of the in-extent dispatch check), and 1/(h*w) for the UB bound
  const int nP = ts.nP;
  uint8_t* s_ainr = s_rank + (lut_n + 15) / 16 * 16;
  float* s_rhw = reinterpret_cast<float*>(s_ainr + (nP * nI2 + 15) / 16 * 16);
  // the rank-count fast path's plane table per (in region, w digit, h digit):
  // {h*w, v, ra, skip rows} and, per (in region, w digit), the dispatch failures of the cube's
  // planes summed over h.  v = h*w*(p - 1) with p the largest product of rank < ra
  // (clamped at 0): a plane has UB pairs only if v + Q' >= len(in) (below); planes
  // with h < 1 or no pair left get v = -2^30 (never) and every c row marked bad
  int4* s_pl = reinterpret_cast<int4*>(s_rhw + (nI2 + 3) / 4 * 4);
  uint32_t* s_f2sum = reinterpret_cast<uint32_t*>(s_pl + nP * nI2);
  // NIc instances: the cube's h-free dispatch bounds as tables over (region, k, r, s)
  // — c_max = min(len(wt) / (k*r*s), kGtCap) — and (region, k, oh, ow) — d_out =
  // min(len(out) / (k*oh*ow), kGtCap) | mth << 8, mth the same of dirty_max(out)
  const int nI3i = nI2 * nI;
  uint8_t* s_cmax = reinterpret_cast<uint8_t*>(s_f2sum + nP * nI);
  uint16_t* s_dout = reinterpret_cast<uint16_t*>(s_cmax + (NIc ? (nP * nI3i + 15) / 16 * 16 : 0));
  if (NIc) {
    for (int i = threadIdx.x; i < nP * nI3i; i += blockDim.x) {
      const int p = i / nI3i, r = i - p * nI3i, a = r / nI2, b = (r / nI) % nI, c = r % nI;  // digits (k, r|oh, s|ow)
      const int64_t e = (int64_t)s_u[a] * s_u[b] * s_u[c];
      uint8_t cm = 0;
      uint16_t dd = 0;
      if (s_u[a] >= 1 && s_u[b] >= 1 && s_u[c] >= 1) {
        const float re = __frcp_rn((float)e);
        cm = (uint8_t)div_cap((int64_t)ts.region_len[p], e, re);
        const int dmax = ts.dirty_max[p];
        dd = (uint16_t)(div_cap((int64_t)ts.region_len[p], e, re) | (dmax < 0 ? 0 : div_cap(dmax, e, re)) << 8);
      }
      s_cmax[i] = cm;
      s_dout[i] = dd;
    }
  }
  for (int i = threadIdx.x; i < nP * nI2; i += blockDim.x) {
    const int p = i / nI2, wh = i - p * nI2, wd = wh / nI, hd = wh - wd * nI;
    const int64_t hw = (int64_t)s_u[hd] * s_u[wd];
    int lo = 0;
    if (hw >= 1) {
      const int64_t a = ts.region_len[p] / hw;
      const int32_t tc = (int32_t)(a > INT32_MAX - 1 ? INT32_MAX - 1 : a);
      for (int step = p2 >> 1; step > 0; step >>= 1)
        if (s_prod[lo + step - 1] <= tc) lo += step;
    }
    s_ainr[i] = (uint8_t)lo;
  }
  for (int i = threadIdx.x; i < nI2; i += blockDim.x) {
    const int64_t hw = s_pp[i];
    s_rhw[i] = hw >= 1 ? __frcp_rn((float)hw) : 0.f;
  }
  __syncthreads();
  // pairs whose product x*c exceeds t (t >= 0; t >= lut_n: none when lut_n > 0)
  // the rank index of that set (pairs of rank >= it have a product > t)
  auto gt_rank = [&](int64_t t) -> int {
    if (lut_n) return t >= lut_n ? nI2 : s_rank[t];
    const int32_t tc = (int32_t)(t > INT32_MAX - 1 ? INT32_MAX - 1 : t);
    int lo = 0;
    for (int step = p2 >> 1; step > 0; step >>= 1)
      if (s_prod[lo + step - 1] <= tc) lo += step;
    return lo;
  };
  auto gt_prod = [&](int64_t t) -> M128 { return s_pgt[gt_rank(t)]; };
  const int qcap = lut_n ? lut_n : INT32_MAX;  // quotients at or above it select no pair
  const bool test_ok0 = ts.test_ok[0] != 0;
  // position-0 verdicts of a plane's nI values of c: one word of plan.cmask at
  // (table key without c) / nI — the key strides of the other roles are multiples of nI
  const uint32_t cperm = (uint32_t)s_div[0];
  uint32_t cks[NS];
#pragma unroll
  for (int q = 2; q < NS; ++q) cks[q] = s_cks[q];
  const M128 all = bit_range(0, nI2);
  const M128 x_lt1 = ~s_gtx[0] & all, c_lt1 = ~s_gtc[0] & all;
  // rank-count form of a plane's checks when the cube's h-free dispatch bounds
  // (c <= len(wt)/(k*r*s), x <= len(out)/(k*oh*ow)) hold for every digit value — the
  // usual case: the in-extent failures are the pairs of rank >= ra, the UB ones those
  // of rank in [ru, ra), so their counts are differences of s_cnt and the plane's
  // remaining pairs are the one mask s_okm[min(ra, ru)]
  for (int r = threadIdx.x; r <= nI2; r += blockDim.x) {
    const M128 m = all & ~s_pgt[r] & ~(x_lt1 | c_lt1);
    s_okm[r] = m;
    s_cnt[r] = (uint8_t)popc(m);
  }
  int32_t umax = 0, umin = INT32_MAX;
  for (int i = 0; i < nI; ++i) umax = max(umax, s_u[i]), umin = min(umin, s_u[i]);
  const bool all_pos = umin >= 1;                     // no plane has tc_h < 1
  const uint32_t rows_all = (1u << nI) - 1u;
  __syncthreads();
  const unsigned int n_base = (unsigned int)(nI2 - s_cnt[nI2]);  // pairs with x < 1 or c < 1
  for (int i = threadIdx.x; i < nP * nI2; i += blockDim.x) {
    const int wh = i % nI2, wd = wh / nI, hd = wh - wd * nI;
    const int ra = s_ainr[i];
    const bool skip = s_u[hd] < 1 || s_cnt[ra] == 0;
    const int32_t hw = s_u[hd] * s_u[wd], pm = ra >= 1 ? max(s_prod[ra - 1], 0) : 0;
    s_pl[i] = make_int4(hw, skip ? -(1 << 30) : hw * (pm - 1), ra, skip ? (1 << nI) - 1 : 0);
  }
  for (int i = threadIdx.x; i < nP * nI && i < 8 * kPairMaxInts; i += blockDim.x) {
    uint32_t m = 0;
    int32_t vm = INT32_MIN;
    for (int hd = 0; hd < nI; ++hd) {  // (the v of s_pl, recomputed: no barrier in between)
      const int ra = s_ainr[i * nI + hd];
      const bool skip = s_u[hd] < 1 || s_cnt[ra] == 0;
      const int32_t hw = s_u[hd] * s_u[i % nI], pm = ra >= 1 ? max(s_prod[ra - 1], 0) : 0;
      m |= (skip ? 1u : 0u) << hd;
      vm = max(vm, skip ? -(1 << 30) : hw * (pm - 1));
    }
    s_skipm[i] = (uint16_t)m;
    s_vmax[i] = vm;
  }
  for (int i = threadIdx.x; i < nP * nI; i += blockDim.x) {
    uint32_t f = 0;
    for (int hd = 0; hd < nI; ++hd)
      f += s_u[hd] < 1 ? (uint32_t)nI2 : n_base + (s_cnt[nI2] - s_cnt[s_ainr[i * nI + hd]]);
    s_f2sum[i] = f;
  }
  __syncthreads();
  const uint32_t magic = (uint32_t)(0xFFFFFFFFull / (uint32_t)nI) + 1u;  // n / nI = umulhi(n, magic), n < 2^27
  unsigned int cnt1 = 0, cnt2 = 0, cnt3 = 0, cnt4 = 0;
  // whole cubes inside [begin, end): mismatches are counted as the remainder
  unsigned int f_bind = 0, f2 = 0, f4 = 0, f_surv = 0;
  // a thread owns a "cube": the nI planes sharing the permutation and digits 3..8
  // (all values of tc_h, digit 2); everything free of h is computed once per cube
  const uint64_t nI3 = (uint64_t)nI2 * nI;
  const uint64_t cubes_per_perm = s_div[2];
  const uint64_t cube_lo = s_div[3], cube_hi = s_div[4];
  // cube / cubes_per_perm by multiply when both are < 2^31 (constants: s_div[5], [6])
  const bool pm_fast = cube_hi < (1ull << 31) && cubes_per_perm < (1ull << 31);
  const uint32_t pm_m = (uint32_t)s_div[5], pm_sh = (uint32_t)s_div[6];
  for (uint64_t cb = cube_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; cb < cube_hi;
       cb += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c0b = cb * nI3;
    if (!test_ok0) {
      const uint64_t lo = c0b < begin ? begin : c0b, hi = c0b + nI3 > end ? end : c0b + nI3;
      cnt3 += (unsigned int)(hi - lo);
      continue;
    }
    const uint64_t perm = pm_fast ? (uint64_t)mdiv((uint32_t)cb, pm_m, pm_sh) : cb / cubes_per_perm;
    int digit[NS];
    {
      uint64_t s = cb - perm * cubes_per_perm;  // digits 3..8
      if (s < (1ull << 27)) {
        uint32_t s32 = (uint32_t)s;
#pragma unroll
        for (int q = 3; q < NS; ++q) {
          const uint32_t dq = __umulhi(s32, magic);
          digit[q] = (int)(s32 - dq * (uint32_t)nI);
          s32 = dq;
        }
      } else {
#pragma unroll
        for (int q = 3; q < NS; ++q) {
          const uint64_t dq = s / (uint64_t)nI;
          digit[q] = (int)(s - dq * (uint64_t)nI);
          s = dq;
        }
      }
    }
    const int32_t cw = s_u[digit[3]], ck = s_u[digit[4]], cr = s_u[digit[5]];
    const int32_t cs = s_u[digit[6]], coh = s_u[digit[7]], cow = s_u[digit[8]];
    const bool cube_bad = min(min(min(cw, ck), min(cr, cs)), min(coh, cow)) < 1;
    const int p_in = perms[perm * 3 + 0], p_w = perms[perm * 3 + 1], p_out = perms[perm * 3 + 2];
    // region lengths are < 2^31 (atc_testsets_upload): 32-bit divisions
    const uint32_t len_in = (uint32_t)ts.region_len[p_in], len_w = (uint32_t)ts.region_len[p_w];
    const uint32_t len_out = (uint32_t)ts.region_len[p_out];
    int c_max = 0, d_out = 0, mth = 0;
    if (NIc) {  // tables (0 where a digit is < 1: cube_bad)
      const uint32_t k4 = (uint32_t)digit[4] * nI2;
      c_max = s_cmax[(uint32_t)p_w * nI3i + k4 + digit[5] * nI + digit[6]];
      const uint32_t dd = s_dout[(uint32_t)p_out * nI3i + k4 + digit[7] * nI + digit[8]];
      d_out = dd & 0xFF;
      mth = dd >> 8;
    } else if (!cube_bad) {
      const int32_t krs = ck * cr * cs, ext_out = ck * coh * cow;
      const float r_out = __frcp_rn((float)ext_out);
      c_max = div_cap(len_w, krs, __frcp_rn((float)krs));
      d_out = div_cap(len_out, ext_out, r_out);
      const int dmax = ts.dirty_max[p_out];
      mth = dmax < 0 ? 0 : div_cap(dmax, ext_out, r_out);
    }
    const int32_t q_rest = (coh + cr - 2) * cw + (cow + cs - 2);   // Q = -h*w + q_rest
    uint32_t ckey0 = (uint32_t)perm * cperm;
#pragma unroll
    for (int q = 3; q < NS; ++q) ckey0 += (uint32_t)digit[q] * cks[q];
    // the verdict word's upper half (positions 0 or 1) applies when ow >= 2: output
    // position 1 is (0, 0, 0, 1)
    const uint32_t wsh = cow >= 2 ? 16u : 0u;
    if (c0b >= begin && c0b + nI3 <= end) {  // the whole cube: no range masks
      f_bind += (unsigned int)nI3;
      if (cube_bad) {
        f2 += (unsigned int)nI3;
        continue;
      }
      const uint8_t* ainr = s_ainr + ((uint32_t)p_in * nI + digit[3]) * nI;
      const float* rhw = s_rhw + digit[3] * nI;
      if (c_max >= umax && d_out >= umax && lut_n) {  // cube_dm = x < 1 | c < 1: the rank-count form
        // the in-extent dispatch failures of every plane: one table sum; per plane the
        // table row {h*w, largest product of rank < ra, ra, skip} (skip: h < 1, or no
        // pair left), the UB test and the position-0/1 verdicts of the c rows
        const uint32_t tix = (uint32_t)p_in * nI + digit[3];
        f2 += s_f2sum[tix];
        const int4* pl = s_pl + tix * nI;
        const uint32_t* cm0 = plan.cmask + ckey0;
        const uint32_t ck2 = cks[2];  // 1 for the canonical key order: immediate offsets
        // branch-free pass over the planes: a bit per plane that needs a closer look —
        // UB pairs possible (v >= len(in) - Q': p*hw >= alim, see below) or a c row
        // without a position-0/1 mismatch (skip planes: t.w = every row, never)
        const int32_t lq = (int32_t)len_in - q_rest;
        uint32_t need = 0;
        if (plan.allbad && tix < 8 * kPairMaxInts) {
          // the h digits whose every c row mismatches, for the whole cube in one word
          // (built with the table), less the skip planes; then the UB test per plane
          need = ~((__ldg(plan.allbad + ckey0 / (uint32_t)nI) >> wsh) | s_skipm[tix]) & rows_all;
          if (s_vmax[tix] >= lq)  // some plane may have UB pairs (usually none does)
#pragma unroll
            for (int hd = 0; hd < nI; ++hd)  // digit 2: tc_h
              if (pl[hd].y >= lq) need |= 1u << hd;
        } else if (ck2 == 1) {
#pragma unroll
          for (int hd = 0; hd < nI; ++hd) {  // digit 2: tc_h
            const int4 t = pl[hd];
            const uint32_t rb = ((__ldg(cm0 + hd) >> wsh) | (uint32_t)t.w) & 0xFFFFu;
            if (t.y >= lq || rb != rows_all) need |= 1u << hd;
          }
        } else {
          const uint32_t* cm = cm0;
#pragma unroll
          for (int hd = 0; hd < nI; ++hd, cm += ck2) {
            const int4 t = pl[hd];
            const uint32_t rb = ((__ldg(cm) >> wsh) | (uint32_t)t.w) & 0xFFFFu;
            if (t.y >= lq || rb != rows_all) need |= 1u << hd;
          }
        }
        while (need) {
          const int hd = __ffs(need) - 1;
          need &= need - 1;
          const int4 t = pl[hd];
          int r_ok = t.z;
          // UB (see the general path below) takes pairs only if the largest remaining
          // product p exceeds floor((alim - 1) / hw), alim = len(in) + hw - Q', i.e. if
          // p*hw >= alim: v + Q' >= len(in) (32-bit: products < 4096 with lut_n; p*hw <=
          // len(in) by the in-extent check, so there is none when Q' < hw)
          if (t.y >= lq) {
            const int32_t hw = t.x;
            const int64_t alim = (int64_t)len_in + hw - q_rest;
            const uint32_t am1 = (uint32_t)(alim - 1);
            const int ru = alim <= 0 ? 0 : gt_rank(lut_n ? div_capn(am1, hw, rhw[hd], qcap) : (int)(am1 / (uint32_t)hw));
            if (ru < r_ok) {
              f4 += s_cnt[r_ok] - s_cnt[ru];
              r_ok = ru;
              if (!s_cnt[ru]) continue;
            }
          }
          const uint32_t rows_bad = (__ldg(cm0 + (uint32_t)hd * ck2) >> wsh) & 0xFFFFu;
          if (rows_bad == rows_all) continue;  // every c row mismatches at position 0 or 1
          const M128 ok = s_okm[r_ok] & ~(~s_gtx[mth] | s_rowx[rows_bad]);
          if (any(ok)) {
            const unsigned int k = popc(ok);
            f_surv += k;
            const uint64_t p0 = c0b + (uint64_t)hd * nI2;
            unsigned long long slot = atomicAdd(surv_cnt, (unsigned long long)k);
            for (uint64_t w = ok.lo; w; w &= w - 1, ++slot)
              if (slot < surv_cap) surv[slot] = p0 + (uint64_t)(__ffsll((long long)w) - 1) - begin;
            for (uint64_t w = ok.hi; w; w &= w - 1, ++slot)
              if (slot < surv_cap) surv[slot] = p0 + 64 + (uint64_t)(__ffsll((long long)w) - 1) - begin;
          }
        }
        continue;
      }
      const M128 cube_dm = x_lt1 | c_lt1 | s_gtc[c_max] | s_gtx[d_out];  // h-free dispatch failures
      const M128 dirty_fail = ~s_gtx[mth];
      for (int hd = 0; hd < nI; ++hd) {  // digit 2: tc_h
        const int32_t ch = s_u[hd];
        if (ch < 1) {
          f2 += (unsigned int)nI2;
          continue;
        }
        const M128 dm = cube_dm | s_pgt[ainr[hd]];
        M128 ok = all & ~dm;
        f2 += popc(dm);
        if (!any(ok)) continue;
        const int32_t hw = ch * cw;
        // UB needs (x*c - 1)*h*w + Q' >= len(in) with x*c*h*w <= len(in): only if Q' >= h*w
        if (q_rest >= hw) {
          const int64_t alim = (int64_t)len_in + hw - q_rest;
          const uint32_t am1 = (uint32_t)(alim - 1);
          const M128 um =
              alim <= 0 ? ok : (ok & gt_prod(lut_n ? div_capn(am1, hw, rhw[hd], qcap) : (int)(am1 / (uint32_t)hw)));
          f4 += popc(um);
          ok = ok & ~um;
          if (!any(ok)) continue;
        }
        const uint32_t cw2 = __ldg(plan.cmask + ckey0 + (uint32_t)hd * cks[2]) >> wsh;
        ok = ok & ~(dirty_fail | s_rowx[cw2 & 0xFFFFu]);
        if (any(ok)) {
          const unsigned int k = popc(ok);
          f_surv += k;
          const uint64_t p0 = c0b + (uint64_t)hd * nI2;
          unsigned long long slot = atomicAdd(surv_cnt, (unsigned long long)k);
          for (uint64_t w = ok.lo; w; w &= w - 1, ++slot)
            if (slot < surv_cap) surv[slot] = p0 + (uint64_t)(__ffsll((long long)w) - 1) - begin;
          for (uint64_t w = ok.hi; w; w &= w - 1, ++slot)
            if (slot < surv_cap) surv[slot] = p0 + 64 + (uint64_t)(__ffsll((long long)w) - 1) - begin;
        }
      }
      continue;
    }
    const M128 cube_dm = x_lt1 | c_lt1 | s_gtc[c_max] | s_gtx[d_out];  // h-free dispatch failures
    const M128 dirty_fail = ~s_gtx[mth];
    for (int hd = 0; hd < nI; ++hd) {  // digit 2: tc_h
      const uint64_t p0 = c0b + (uint64_t)hd * nI2;
      if (p0 + nI2 <= begin || p0 >= end) continue;
      const uint64_t lo = p0 < begin ? begin : p0, hi = p0 + nI2 > end ? end : p0 + nI2;
      const int32_t ch = s_u[hd];
      if (cube_bad || ch < 1) {
        cnt2 += (unsigned int)(hi - lo);  // a dim of the plane < 1: "size is not positive" for every binding
        continue;
      }
      const M128 range = (lo == p0 && hi == p0 + nI2) ? all : bit_range((int)(lo - p0), (int)(hi - p0));
      const int32_t hw = ch * cw;
      const float r_hw = __frcp_rn((float)hw);
      const int a_in = lut_n ? div_capn(len_in, hw, r_hw, qcap) : (int)(len_in / (uint32_t)hw);
      const M128 dm = range & (cube_dm | gt_prod(a_in));
      M128 ok = range & ~dm, um{0, 0}, mm{0, 0};
      if (any(ok)) {
        const int32_t q_in = -hw + q_rest;
        const int64_t alim = (int64_t)len_in - q_in;  // UB iff x*c*h*w >= alim (< 2^32)
        const uint32_t am1 = (uint32_t)(alim - 1);
        um = alim <= 0 ? ok : (ok & gt_prod(lut_n ? div_capn(am1, hw, r_hw, qcap) : (int)(am1 / (uint32_t)hw)));
        ok = ok & ~um;
        if (any(ok)) {
          const uint32_t cw2 = __ldg(plan.cmask + ckey0 + (uint32_t)hd * cks[2]) >> wsh;
          mm = ok & (dirty_fail | s_rowx[cw2 & 0xFFFFu]);
          ok = ok & ~mm;
        }
      }
      cnt2 += popc(dm);
      cnt4 += popc(um);
      cnt1 += popc(mm);
      if (any(ok)) {
        unsigned long long slot = atomicAdd(surv_cnt, (unsigned long long)popc(ok));
        for (uint64_t w = ok.lo; w; w &= w - 1, ++slot)
          if (slot < surv_cap) surv[slot] = p0 + (uint64_t)(__ffsll((long long)w) - 1) - begin;
        for (uint64_t w = ok.hi; w; w &= w - 1, ++slot)
          if (slot < surv_cap) surv[slot] = p0 + 64 + (uint64_t)(__ffsll((long long)w) - 1) - begin;
      }
    }
  }
  // whole cubes: every binding not counted as dispatch / UB / survivor is a mismatch
  cnt1 += f_bind - f2 - f4 - f_surv;
  cnt2 += f2;
  cnt4 += f4;
  unsigned int cnt[ATC_REASON_COUNT] = {0, cnt1, cnt2, cnt3, cnt4};
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

template __global__ void k_screen_conv_pairs<0>(TestsetView, const uint8_t*, uint64_t, uint64_t, uint64_t, RowPlan,
                                                uint64_t*, uint64_t, unsigned long long*, unsigned long long*, int);
template __global__ void k_screen_conv_pairs<9>(TestsetView, const uint8_t*, uint64_t, uint64_t, uint64_t, RowPlan,
                                                uint64_t*, uint64_t, unsigned long long*, unsigned long long*, int);

#define ATC_ROWS_INST(SEM, NS, I32, MASK)                                                                        \
  template __global__ void k_screen_rows<SEM, NS, I32, MASK>(TestsetView, SpecView, const uint8_t*, uint64_t,    \
                                                             uint64_t, uint64_t, RowPlan, uint64_t*, uint64_t,   \
                                                             unsigned long long*, unsigned long long*);
#define ATC_ROWS_INST2(SEM, NS, MASK) ATC_ROWS_INST(SEM, NS, true, MASK) ATC_ROWS_INST(SEM, NS, false, MASK)
ATC_ROWS_INST2(ATC_SEM_GEMM, 3, kQ0Dynamic)
ATC_ROWS_INST2(ATC_SEM_GEMM, 6, kQ0Dynamic)
ATC_ROWS_INST2(ATC_SEM_CONV2D, 9, kQ0Dynamic)
// the bundled specs: conv2d digit 0 = tc_n; gemm digit 0 = tc_m (col-major: lda/ldc fall back to m)
ATC_ROWS_INST2(ATC_SEM_CONV2D, 9, 1u << ATC_SZ_CN)
ATC_ROWS_INST2(ATC_SEM_GEMM, 3, 1u << ATC_SZ_M)
ATC_ROWS_INST2(ATC_SEM_GEMM, 3, (1u << ATC_SZ_M) | (1u << ATC_SZ_LDA) | (1u << ATC_SZ_LDC))
ATC_ROWS_INST2(ATC_SEM_GEMM, 6, 1u << ATC_SZ_M)

}  // namespace atc
