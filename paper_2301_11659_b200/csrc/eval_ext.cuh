// Extended semantics (include/atc_b200.h, "Extended semantics"): the decode and
// the dispatch checks, shared by the GPU kernels (eval_ext.cu) and the host (the
// messages of atc_run_reference_ext).  The CPU statement is oracle/ext_oracle.c.
#pragma once
#include <cstdint>

#include "atc_b200.h"

namespace atc {

constexpr int kMaxExtSizes = 16;

// Device-friendly copy of atc_spec_ext.
struct ExtView {
  int32_t sem, nA, nS, nF;
  int32_t arr_of_role[3];
  int32_t livein[ATC_MAX_ARRAYS];
  int32_t role_size[ATC_SZ_COUNT];
  int32_t ext_role[ATC_XR_COUNT];
  int32_t role_float[ATC_FR_COUNT];
  int64_t iconst[ATC_MAX_CONSTS];
  double fconst[ATC_MAX_CONSTS];
};

// Every quantity a call needs, resolved from the bound sizes and floats.
struct ExtCall {
  int64_t m, n, k, lda, ldb, ldc, ta, tb;
  double alpha, beta;
  int64_t N, C, H, W, K, R, S, OH, OW, sh, sw, ph, pw, dh, dw;
};

__host__ __device__ inline int64_t ext_base(const ExtView& e, const int64_t* sz, int role, int64_t fb) {
  return e.role_size[role] >= 0 ? sz[e.role_size[role]] : fb;
}
__host__ __device__ inline int64_t ext_xr(const ExtView& e, const int64_t* sz, int role, int64_t fb) {
  return e.ext_role[role] >= 0 ? sz[e.ext_role[role]] : fb;
}

// 0, or the index of the failed dispatch check (reason 2): see ext_check_text.
// lens[role] = length of the region bound to the array of that role.
__host__ __device__ inline int ext_resolve(const ExtView& e, const int64_t* sz, const double* fl, const int64_t* lens,
                                           ExtCall& c) {
  if (e.sem == ATC_SEM_GEMM_EXT) {
    c.m = ext_base(e, sz, ATC_SZ_M, 0), c.n = ext_base(e, sz, ATC_SZ_N, 0), c.k = ext_base(e, sz, ATC_SZ_K, 0);
    c.lda = ext_base(e, sz, ATC_SZ_LDA, 0), c.ldb = ext_base(e, sz, ATC_SZ_LDB, 0);
    c.ldc = ext_base(e, sz, ATC_SZ_LDC, 0);
    c.ta = ext_xr(e, sz, ATC_XR_TRANSA, 0), c.tb = ext_xr(e, sz, ATC_XR_TRANSB, 0);
    c.alpha = e.role_float[ATC_FR_ALPHA] >= 0 ? fl[e.role_float[ATC_FR_ALPHA]] : 1.0;
    c.beta = e.role_float[ATC_FR_BETA] >= 0 ? fl[e.role_float[ATC_FR_BETA]] : 0.0;
    if (c.m < 1 || c.n < 1 || c.k < 1 || c.lda < 1 || c.ldb < 1 || c.ldc < 1) return 1;
    if ((c.ta != 0 && c.ta != 1) || (c.tb != 0 && c.tb != 1)) return 2;
    if (c.lda < (c.ta ? c.m : c.k) || c.ldb < (c.tb ? c.k : c.n) || c.ldc < c.n) return 3;
    if (((c.ta ? c.k : c.m) - 1) * c.lda + (c.ta ? c.m : c.k) > lens[0]) return 4;
    if (((c.tb ? c.n : c.k) - 1) * c.ldb + (c.tb ? c.k : c.n) > lens[1]) return 5;
    if ((c.m - 1) * c.ldc + c.n > lens[2]) return 6;
    return 0;
  }
  c.N = ext_base(e, sz, ATC_SZ_CN, 0), c.C = ext_base(e, sz, ATC_SZ_CC, 0), c.H = ext_base(e, sz, ATC_SZ_CH, 0);
  c.W = ext_base(e, sz, ATC_SZ_CW, 0), c.K = ext_base(e, sz, ATC_SZ_CK, 0), c.R = ext_base(e, sz, ATC_SZ_CR, 0);
  c.S = ext_base(e, sz, ATC_SZ_CS, 0);
  c.sh = ext_xr(e, sz, ATC_XR_STRIDE_H, 1), c.sw = ext_xr(e, sz, ATC_XR_STRIDE_W, 1);
  c.ph = ext_xr(e, sz, ATC_XR_PAD_H, 0), c.pw = ext_xr(e, sz, ATC_XR_PAD_W, 0);
  c.dh = ext_xr(e, sz, ATC_XR_DIL_H, 1), c.dw = ext_xr(e, sz, ATC_XR_DIL_W, 1);
  if (c.N < 1 || c.C < 1 || c.H < 1 || c.W < 1 || c.K < 1 || c.R < 1 || c.S < 1) return 1;
  if (c.sh < 1 || c.sw < 1 || c.dh < 1 || c.dw < 1 || c.ph < 0 || c.pw < 0) return 7;
  const int64_t eh = c.H + 2 * c.ph - c.dh * (c.R - 1) - 1, ew = c.W + 2 * c.pw - c.dw * (c.S - 1) - 1;
  if (eh < 0 || ew < 0) return 8;
  const int64_t oh = eh / c.sh + 1, ow = ew / c.sw + 1;
  c.OH = ext_base(e, sz, ATC_SZ_COH, oh);
  c.OW = ext_base(e, sz, ATC_SZ_COW, ow);
  if (c.OH != oh || c.OW != ow) return 9;
  if (c.N * c.C * c.H * c.W > lens[0] || c.K * c.C * c.R * c.S > lens[1] || c.N * c.K * c.OH * c.OW > lens[2])
    return 10;
  return 0;
}

inline const char* ext_check_text(int k) {
  switch (k) {
    case 1: return "size is not positive";
    case 2: return "transpose flag is not 0 or 1";
    case 3: return "leading dimension too small";
    case 4: return "A footprint exceeds its region";
    case 5: return "B footprint exceeds its region";
    case 6: return "C footprint exceeds its region";
    case 7: return "bad stride / dilation / padding";
    case 8: return "filter larger than the padded image";
    case 9: return "output size does not match stride / padding / dilation";
    case 10: return "extent exceeds its region";
    default: return "ok";
  }
}

}  // namespace atc
