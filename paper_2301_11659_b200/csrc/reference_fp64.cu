// FP64 reference semantics on the GPU: equivalence::run_reference
// (/root/reference/proj/src/equivalence.cpp:131-139 -> reference_gemm :40-65,
// reference_conv2d :67-93) and the oracle dispatch handler body run_dispatch
// (rewriter.cpp:99-162).  One thread per output element; the reference's
// "later writes overwrite earlier ones" order for overlapping GEMM writes
// (ldc < n) is reproduced by letting only the last writer of a position store.
// Accumulation is acc = acc + a*b in IEEE double, never fused, in the
// reference's p (resp. z,u,v) order, so results are bit-identical to the
// reference built without FMA contraction.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "atc_b200.h"
#include "capi_internal.h"
#include "eval_common.cuh"

namespace atc {

__global__ void k_ref_gemm(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                           int m, int n, int k, int lda, int ldb, int ldc, int row) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= (int64_t)m * n) return;
  const int i = (int)(o / n), j = (int)(o % n);
  const bool overlap = row ? (ldc < n && m > 1) : (ldc < m && n > 1);
  if (overlap && !gemm_last_writer(row, i, j, m, ldc)) return;
  double acc = 0.0;
  if (row)
    for (int p = 0; p < k; ++p) acc = dadd(acc, dmul(A[(int64_t)i * lda + p], B[(int64_t)p * ldb + j]));
  else
    for (int p = 0; p < k; ++p) acc = dadd(acc, dmul(A[(int64_t)p * lda + i], B[(int64_t)j * ldb + p]));
  if (row)
    C[(int64_t)i * ldc + j] = acc;
  else
    C[(int64_t)j * ldc + i] = acc;
}

__global__ void k_ref_conv(const double* __restrict__ in, const double* __restrict__ wt, double* __restrict__ out,
                           int N, int C, int H, int W, int K, int R, int S, int OH, int OW) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= (int64_t)N * K * OH * OW) return;
  int64_t rem = o;
  const int x = (int)(rem % OW); rem /= OW;
  const int y = (int)(rem % OH); rem /= OH;
  const int q = (int)(rem % K);
  const int b = (int)(rem / K);
  double acc = 0.0;
  for (int z = 0; z < C; ++z)
    for (int u = 0; u < R; ++u)
      for (int v = 0; v < S; ++v)
        acc = dadd(acc, dmul(in[(((int64_t)b * C + z) * H + y + u) * W + x + v], wt[(((int64_t)q * C + z) * R + u) * S + v]));
  out[o] = acc;
}

__global__ void k_round_f32(double* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (double)__double2float_rn(p[i]);
}

}  // namespace atc

using namespace atc;

namespace {

bool spec_basic(atc_ctx* ctx, const atc_spec_desc* s) {
  if (!s || (s->semantics != ATC_SEM_GEMM && s->semantics != ATC_SEM_CONV2D) || s->n_arrays != 3 ||
      s->n_sizes < 1 || s->n_sizes > ATC_MAX_SIZES) {
    atc_set_error(ctx, "malformed spec descriptor");
    return false;
  }
  return true;
}

int64_t role_val(const atc_spec_desc* s, const int64_t* sizes, int role, int64_t fb) {
  int q = s->role_size[role];
  return q < 0 ? fb : sizes[q];
}

int arr_of(const atc_spec_desc* s, int role) {
  for (int a = 0; a < s->n_arrays; ++a)
    if (s->array_role[a] == role) return a;
  return -1;
}

// Device round trip of run_reference over host buffers.
int run_reference_impl(atc_ctx* ctx, const atc_spec_desc* s, const int64_t* sizes, double* const* bufs,
                       const int64_t* lens, const int32_t* round_f32) {
  const int ia = arr_of(s, 0), ib = arr_of(s, 1), ic = arr_of(s, 2);
  if (ia < 0 || ib < 0 || ic < 0) {
    atc_set_error(ctx, "spec lacks a/b/c roles");
    return ATC_ERR_ARG;
  }
  int64_t amax = -1, bmax = -1, cmax = -1, outs = 0;
  Dims d{};
  if (s->semantics == ATC_SEM_GEMM) {
    const bool row = s->layout == ATC_LAYOUT_ROW;
    d.m = role_val(s, sizes, ATC_SZ_M, 0);
    d.n = role_val(s, sizes, ATC_SZ_N, 0);
    d.k = role_val(s, sizes, ATC_SZ_K, 0);
    d.lda = role_val(s, sizes, ATC_SZ_LDA, row ? d.k : d.m);
    d.ldb = role_val(s, sizes, ATC_SZ_LDB, row ? d.n : d.k);
    d.ldc = role_val(s, sizes, ATC_SZ_LDC, row ? d.n : d.m);
    if (d.m > 0 && d.n > 0) {
      outs = d.m * d.n;
      cmax = row ? (d.m - 1) * d.ldc + d.n - 1 : (d.n - 1) * d.ldc + d.m - 1;
      if (d.k > 0) {
        amax = row ? (d.m - 1) * d.lda + d.k - 1 : (d.k - 1) * d.lda + d.m - 1;
        bmax = row ? (d.k - 1) * d.ldb + d.n - 1 : (d.n - 1) * d.ldb + d.k - 1;
      }
    }
    if (d.ldc < 1 && outs > 0) {
      atc_set_error(ctx, "ldc %lld < 1", (long long)d.ldc);
      return ATC_ERR_ARG;
    }
  } else {
    d.cn = role_val(s, sizes, ATC_SZ_CN, 0);
    d.cc = role_val(s, sizes, ATC_SZ_CC, 0);
    d.ch = role_val(s, sizes, ATC_SZ_CH, 0);
    d.cw = role_val(s, sizes, ATC_SZ_CW, 0);
    d.ck = role_val(s, sizes, ATC_SZ_CK, 0);
    d.cr = role_val(s, sizes, ATC_SZ_CR, 0);
    d.cs = role_val(s, sizes, ATC_SZ_CS, 0);
    d.coh = role_val(s, sizes, ATC_SZ_COH, d.ch - d.cr + 1);
    d.cow = role_val(s, sizes, ATC_SZ_COW, d.cw - d.cs + 1);
    if (d.cn > 0 && d.ck > 0 && d.coh > 0 && d.cow > 0) {
      outs = d.cn * d.ck * d.coh * d.cow;
      cmax = outs - 1;
      if (d.cc > 0 && d.cr > 0 && d.cs > 0) {
        amax = (((d.cn - 1) * d.cc + d.cc - 1) * d.ch + d.coh - 1 + d.cr - 1) * d.cw + d.cow - 1 + d.cs - 1;
        bmax = (((d.ck - 1) * d.cc + d.cc - 1) * d.cr + d.cr - 1) * d.cs + d.cs - 1;
      }
    }
  }
  if (amax >= lens[ia] || bmax >= lens[ib] || cmax >= lens[ic]) {
    atc_set_error(ctx, "access outside a buffer (max index a %lld/%lld, b %lld/%lld, c %lld/%lld)",
                  (long long)amax, (long long)lens[ia], (long long)bmax, (long long)lens[ib], (long long)cmax,
                  (long long)lens[ic]);
    return ATC_ERR_ARG;
  }
  if (outs == 0) {
    if (round_f32 && round_f32[ic])
      for (int64_t i = 0; i < lens[ic]; ++i) bufs[ic][i] = (double)(float)bufs[ic][i];
    return ATC_OK;
  }
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t ba = (size_t)lens[ia] * 8, bb = (size_t)lens[ib] * 8, bc = (size_t)lens[ic] * 8;
  double* dA = (double*)atc_ctx_scratch(ctx, 8, ba);
  double* dB = (double*)atc_ctx_scratch(ctx, 9, bb);
  double* dC = (double*)atc_ctx_scratch(ctx, 10, bc);
  if (!dA || !dB || !dC) {
    atc_set_error(ctx, "scratch allocation failed");
    return ATC_ERR_CUDA;
  }
  bool ok = atc_cuda_ok(ctx, cudaMemcpyAsync(dA, bufs[ia], ba, cudaMemcpyHostToDevice, st), "H2D") &&
            atc_cuda_ok(ctx, cudaMemcpyAsync(dB, bufs[ib], bb, cudaMemcpyHostToDevice, st), "H2D") &&
            atc_cuda_ok(ctx, cudaMemcpyAsync(dC, bufs[ic], bc, cudaMemcpyHostToDevice, st), "H2D");
  if (!ok) return ATC_ERR_CUDA;
  const unsigned grid = (unsigned)((outs + 255) / 256);
  if (s->semantics == ATC_SEM_GEMM)
    k_ref_gemm<<<grid, 256, 0, st>>>(dA, dB, dC, (int)d.m, (int)d.n, (int)d.k, (int)d.lda, (int)d.ldb, (int)d.ldc,
                                     s->layout == ATC_LAYOUT_ROW);
  else
    k_ref_conv<<<grid, 256, 0, st>>>(dA, dB, dC, (int)d.cn, (int)d.cc, (int)d.ch, (int)d.cw, (int)d.ck, (int)d.cr,
                                     (int)d.cs, (int)d.coh, (int)d.cow);
  if (round_f32 && round_f32[ic]) k_round_f32<<<64, 256, 0, st>>>(dC, lens[ic]);
  ok = atc_cuda_ok(ctx, cudaGetLastError(), "reference launch") &&
       atc_cuda_ok(ctx, cudaMemcpyAsync(bufs[ic], dC, bc, cudaMemcpyDeviceToHost, st), "D2H") &&
       atc_cuda_ok(ctx, cudaStreamSynchronize(st), "reference sync");
  return ok ? ATC_OK : ATC_ERR_CUDA;
}

}  // namespace

extern "C" {

int atc_run_reference(atc_ctx* ctx, const atc_spec_desc* spec, const int64_t* sizes, double* const* buffers,
                      const int64_t* buffer_len) {
  ATC_ENTER(ctx);
  if (!spec_basic(ctx, spec) || !sizes || !buffers || !buffer_len) {
    if (ctx->err.empty()) atc_set_error(ctx, "bad arguments to atc_run_reference");
    return ATC_ERR_ARG;
  }
  return run_reference_impl(ctx, spec, sizes, buffers, buffer_len, nullptr);
}

// run_dispatch (rewriter.cpp:136-161): extent checks with the reference's
// messages, the computation over the full regions, write-back of the output
// with (double)(float) rounding when the region is f32.
int atc_dispatch(atc_ctx* ctx, const atc_spec_desc* spec, const int64_t* sizes, double* const* regions,
                 const int64_t* region_len, const int32_t* region_is_f32) {
  ATC_ENTER(ctx);
  if (!spec_basic(ctx, spec) || !sizes || !regions || !region_len || !region_is_f32) {
    if (ctx->err.empty()) atc_set_error(ctx, "bad arguments to atc_dispatch");
    return ATC_ERR_ARG;
  }
  for (int a = 0; a < spec->n_arrays; ++a) {
    int64_t extent = 1;
    for (int d = 0; d < spec->array_ndims[a]; ++d) {
      int q = spec->array_dims[a][d];
      if (sizes[q] < 1) {
        atc_set_error(ctx, "dispatch size #%d is not positive", q);
        return ATC_ERR_DISPATCH;
      }
      extent *= sizes[q];
    }
    if (region_len[a] < extent) {
      atc_set_error(ctx, "region bound to array #%d holds %lld elements, call needs %lld", a,
                    (long long)region_len[a], (long long)extent);
      return ATC_ERR_DISPATCH;
    }
  }
  return run_reference_impl(ctx, spec, sizes, regions, region_len, region_is_f32);
}

}  // extern "C"
