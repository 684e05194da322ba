// Extended semantics on the GPU (include/atc_b200.h, "Extended semantics";
// SURVEY.md §8(f).4): explicit candidate lists under gemm_ext / conv2d_ext, and
// the semantics on caller buffers.  No reference counterpart; the CPU statement
// (oracle/ext_oracle.c, pinned by known answers) is the checker (tests/test_ext.py).
//
// k_eval_ext: one WARP per binding, tests in order until the first failure — the
// P2 predicate of the header: reason 3 for a failed test set, 2 from the dispatch
// checks (eval_ext.cuh), else every written output recomputed (FP64, no FMA,
// reference-style loop order; lanes split the outputs, __any_sync early exit) and
// compared with the recorded final image, and every dirty position (|init - final|
// above tolerance, k_build_dirty) checked to lie in the written set.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "atc_b200.h"
#include "capi_internal.h"
#include "eval_common.cuh"
#include "eval_ext.cuh"

namespace atc {

__device__ int ext_verdict(const TestsetView& ts, const ExtView& e, const uint8_t* am, const uint8_t* sm,
                           const uint8_t* fm, int t, int lane) {
  if (!ts.test_ok[t]) return ATC_FAIL_TESTSET;
  int64_t sz[kMaxExtSizes];
  double fl[ATC_MAX_FLOATS];
  for (int q = 0; q < e.nS; ++q)
    sz[q] = sm[q] < ts.nI ? ts.ints[(size_t)t * ts.nI + sm[q]] : e.iconst[sm[q] - ts.nI];
  for (int f = 0; f < e.nF; ++f) fl[f] = fm[f] < ts.nF ? ts.floats[(size_t)t * ts.nF + fm[f]] : e.fconst[fm[f] - ts.nF];
  const int pA = am[e.arr_of_role[0]], pB = am[e.arr_of_role[1]], pC = am[e.arr_of_role[2]];
  const int64_t lens[3] = {ts.region_len[pA], ts.region_len[pB], ts.region_len[pC]};
  ExtCall c;
  if (ext_resolve(e, sz, fl, lens, c)) return ATC_FAIL_DISPATCH;
  const int tpA = t * ts.nP + pA, tpB = t * ts.nP + pB, tpC = t * ts.nP + pC;
  const double* __restrict__ A = ts.init + ts.region_off[tpA];
  const double* __restrict__ B = ts.init + ts.region_off[tpB];
  const double* __restrict__ C0 = ts.init + ts.region_off[tpC];
  const double* __restrict__ F = ts.fin + ts.region_off[tpC];
  const bool f32 = ts.is_f32[pC] != 0;
  const int ndirty = ts.dirty_cnt[tpC];
  const int32_t* dirty = ts.dirty_pos + ts.dirty_off[tpC];
  bool bad = false;
  if (e.sem == ATC_SEM_GEMM_EXT) {
    for (int d = lane; d < ndirty && !bad; d += 32) {  // every dirty position is written
      const int64_t q = __ldg(dirty + d);
      bad = !(q / c.ldc < c.m && q % c.ldc < c.n);
    }
    bad = __any_sync(0xffffffffu, bad);
    const int64_t outs = c.m * c.n;
    for (int64_t o0 = 0; o0 < outs && !bad; o0 += 32) {
      const int64_t o = o0 + lane;
      bool mm = false;
      if (o < outs) {
        const int64_t i = o / c.n, j = o - i * c.n;
        double acc = 0.0;
        for (int64_t p = 0; p < c.k; ++p) {
          const double av = c.ta ? A[p * c.lda + i] : A[i * c.lda + p];
          const double bv = c.tb ? B[j * c.ldb + p] : B[p * c.ldb + j];
          acc = dadd(acc, dmul(av, bv));
        }
        const int64_t pos = i * c.ldc + j;
        const double v = c.beta == 0.0 ? dmul(c.alpha, acc) : dadd(dmul(c.alpha, acc), dmul(c.beta, C0[pos]));
        mm = mismatch(round_region(v, f32), __ldg(F + pos), f32);
      }
      bad = __any_sync(0xffffffffu, mm);
    }
  } else {
    const int64_t outs = c.N * c.K * c.OH * c.OW;
    bad = ts.dirty_max[tpC] >= outs;  // the written set is [0, outs)
    for (int64_t o0 = 0; o0 < outs && !bad; o0 += 32) {
      const int64_t o = o0 + lane;
      bool mm = false;
      if (o < outs) {
        int64_t rem = o;
        const int64_t x = rem % c.OW;
        rem /= c.OW;
        const int64_t y = rem % c.OH;
        rem /= c.OH;
        const int64_t q = rem % c.K, b = rem / c.K;
        double acc = 0.0;
        for (int64_t z = 0; z < c.C; ++z)
          for (int64_t u = 0; u < c.R; ++u) {
            const int64_t iy = y * c.sh - c.ph + u * c.dh;
            if (iy < 0 || iy >= c.H) continue;
            for (int64_t v = 0; v < c.S; ++v) {
              const int64_t ix = x * c.sw - c.pw + v * c.dw;
              if (ix < 0 || ix >= c.W) continue;
              acc = dadd(acc, dmul(A[((b * c.C + z) * c.H + iy) * c.W + ix], B[((q * c.C + z) * c.R + u) * c.S + v]));
            }
          }
        mm = mismatch(round_region(acc, f32), __ldg(F + o), f32);
      }
      bad = __any_sync(0xffffffffu, mm);
    }
  }
  return bad ? ATC_FAIL_MISMATCH : 0;
}

__global__ void __launch_bounds__(256) k_eval_ext(TestsetView ts, ExtView e, const uint8_t* arr_map,
                                                  const uint8_t* size_map, const uint8_t* float_map, int64_t n,
                                                  int8_t* fail_t, int8_t* reason) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t b = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; b < n; b += warps) {
    int r = 0, t = 0;
    for (; t < ts.T; ++t) {
      r = ext_verdict(ts, e, arr_map + b * e.nA, size_map + b * e.nS, float_map + b * (e.nF > 0 ? e.nF : 1), t,
                      lane);
      if (r) break;
    }
    if (lane == 0) {
      fail_t[b] = r ? (int8_t)t : (int8_t)-1;
      reason[b] = (int8_t)r;
    }
  }
}

// The semantics on caller buffers: thread per output (each written exactly once).
__global__ void k_ref_ext(ExtView e, ExtCall c, const double* A, const double* B, double* Cb, int f32) {
  if (e.sem == ATC_SEM_GEMM_EXT) {
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < c.m * c.n;
         o += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = o / c.n, j = o - i * c.n;
      double acc = 0.0;
      for (int64_t p = 0; p < c.k; ++p)
        acc = dadd(acc, dmul(c.ta ? A[p * c.lda + i] : A[i * c.lda + p], c.tb ? B[j * c.ldb + p] : B[p * c.ldb + j]));
      const int64_t pos = i * c.ldc + j;
      const double v = c.beta == 0.0 ? dmul(c.alpha, acc) : dadd(dmul(c.alpha, acc), dmul(c.beta, Cb[pos]));
      Cb[pos] = round_region(v, f32 != 0);
    }
    return;
  }
  const int64_t outs = c.N * c.K * c.OH * c.OW;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < outs; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = o;
    const int64_t x = rem % c.OW;
    rem /= c.OW;
    const int64_t y = rem % c.OH;
    rem /= c.OH;
    const int64_t q = rem % c.K, b = rem / c.K;
    double acc = 0.0;
    for (int64_t z = 0; z < c.C; ++z)
      for (int64_t u = 0; u < c.R; ++u) {
        const int64_t iy = y * c.sh - c.ph + u * c.dh;
        if (iy < 0 || iy >= c.H) continue;
        for (int64_t v = 0; v < c.S; ++v) {
          const int64_t ix = x * c.sw - c.pw + v * c.dw;
          if (ix < 0 || ix >= c.W) continue;
          acc = dadd(acc, dmul(A[((b * c.C + z) * c.H + iy) * c.W + ix], B[((q * c.C + z) * c.R + u) * c.S + v]));
        }
      }
    Cb[o] = round_region(acc, f32 != 0);
  }
}

}  // namespace atc

using namespace atc;

namespace {

bool ext_view(atc_ctx* ctx, const atc_spec_ext* s, ExtView& v) {
  if (!s || (s->base.semantics != ATC_SEM_GEMM_EXT && s->base.semantics != ATC_SEM_CONV2D_EXT) ||
      s->base.n_arrays != 3 || s->base.n_sizes < 1 || s->base.n_sizes > kMaxExtSizes || s->n_floats < 0 ||
      s->n_floats > ATC_MAX_FLOATS || s->n_iconst < 0 || s->n_iconst > ATC_MAX_CONSTS || s->n_fconst < 0 ||
      s->n_fconst > ATC_MAX_CONSTS || (s->base.semantics == ATC_SEM_GEMM_EXT && s->base.layout != ATC_LAYOUT_ROW)) {
    atc_set_error(ctx, "malformed extended spec descriptor");
    return false;
  }
  std::memset(&v, 0, sizeof v);
  v.sem = s->base.semantics;
  v.nA = s->base.n_arrays;
  v.nS = s->base.n_sizes;
  v.nF = s->n_floats;
  int seen[3] = {-1, -1, -1};
  for (int a = 0; a < 3; ++a) {
    const int r = s->base.array_role[a];
    if (r < 0 || r > 2 || seen[r] >= 0) {
      atc_set_error(ctx, "extended spec: bad or duplicate array role %d", r);
      return false;
    }
    seen[r] = a;
    v.livein[a] = s->base.array_livein[a];
  }
  for (int r = 0; r < 3; ++r) v.arr_of_role[r] = seen[r];
  for (int r = 0; r < ATC_SZ_COUNT; ++r) {
    v.role_size[r] = s->base.role_size[r];
    if (v.role_size[r] >= v.nS) {
      atc_set_error(ctx, "extended spec: role %d size index out of range", r);
      return false;
    }
  }
  for (int r = 0; r < ATC_XR_COUNT; ++r) {
    v.ext_role[r] = s->ext_role_size[r];
    if (v.ext_role[r] >= v.nS) {
      atc_set_error(ctx, "extended spec: extended role %d size index out of range", r);
      return false;
    }
  }
  for (int r = 0; r < ATC_FR_COUNT; ++r) {
    v.role_float[r] = s->role_float[r];
    if (v.role_float[r] >= v.nF) {
      atc_set_error(ctx, "extended spec: float role %d index out of range", r);
      return false;
    }
  }
  for (int i = 0; i < ATC_MAX_CONSTS; ++i) {
    v.iconst[i] = s->iconst[i];
    v.fconst[i] = s->fconst[i];
  }
  return true;
}

}  // namespace

extern "C" {

int atc_eval_bindings_ext(atc_ctx* ctx, const atc_spec_ext* spec, const atc_testset_handle* ts,
                          const uint8_t* arr_map, const uint8_t* size_map, const uint8_t* float_map,
                          int64_t n_bindings, int8_t* fail_t, int8_t* reason, int64_t* first_pass) {
  ATC_ENTER(ctx);
  if (first_pass) *first_pass = -1;
  ExtView e;
  if (!ext_view(ctx, spec, e)) return ATC_ERR_ARG;
  if (!ts || n_bindings < 0 ||
      (n_bindings > 0 && (!arr_map || !size_map || (e.nF > 0 && !float_map) || !fail_t || !reason))) {
    atc_set_error(ctx, "bad arguments to atc_eval_bindings_ext");
    return ATC_ERR_ARG;
  }
  if (n_bindings == 0) return ATC_OK;
  const size_t n = (size_t)n_bindings, nf = e.nF > 0 ? (size_t)e.nF : 1;
  // every map entry must name a user value or a constant of the spec
  for (size_t b = 0; b < n; ++b) {
    for (int a = 0; a < e.nA; ++a)
      if (arr_map[b * e.nA + a] >= ts->nP) {
        atc_set_error(ctx, "binding %zu: array %d maps to pointer %d of %d", b, a, arr_map[b * e.nA + a], ts->nP);
        return ATC_ERR_ARG;
      }
    for (int q = 0; q < e.nS; ++q)
      if (size_map[b * e.nS + q] >= ts->nI + spec->n_iconst) {
        atc_set_error(ctx, "binding %zu: size %d entry %d beyond %d ints + %d constants", b, q,
                      size_map[b * e.nS + q], ts->nI, spec->n_iconst);
        return ATC_ERR_ARG;
      }
    for (int f = 0; f < e.nF; ++f)
      if (float_map[b * e.nF + f] >= ts->nF + spec->n_fconst) {
        atc_set_error(ctx, "binding %zu: float %d entry %d beyond %d floats + %d constants", b, f,
                      float_map[b * e.nF + f], ts->nF, spec->n_fconst);
        return ATC_ERR_ARG;
      }
  }
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  ts_wait(ts, st);
  const size_t in_bytes = n * (e.nA + e.nS + nf);
  uint8_t* d_in = (uint8_t*)atc_ctx_scratch(ctx, 29, in_bytes + 16);
  int8_t* d_out = (int8_t*)atc_ctx_scratch(ctx, 30, n * 2 + 16);
  if (!d_in || !d_out) {
    atc_set_error(ctx, "scratch allocation failed");
    return ATC_ERR_CUDA;
  }
  std::vector<uint8_t> fz;
  const uint8_t* fmap = float_map;
  if (e.nF == 0) {
    fz.assign(n, 0);
    fmap = fz.data();
  }
  if (!atc_cuda_ok(ctx, cudaMemcpyAsync(d_in, arr_map, n * e.nA, cudaMemcpyHostToDevice, st), "H2D arr_map") ||
      !atc_cuda_ok(ctx, cudaMemcpyAsync(d_in + n * e.nA, size_map, n * e.nS, cudaMemcpyHostToDevice, st),
                   "H2D size_map") ||
      !atc_cuda_ok(ctx, cudaMemcpyAsync(d_in + n * (e.nA + e.nS), fmap, n * nf, cudaMemcpyHostToDevice, st),
                   "H2D float_map"))
    return ATC_ERR_CUDA;
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((n + 7) / 8, (size_t)ctx->sm_count * 8));
  k_eval_ext<<<grid, 256, 0, st>>>(ts->view, e, d_in, d_in + n * e.nA, d_in + n * (e.nA + e.nS), n_bindings, d_out,
                                   d_out + n);
  if (ctx->prof) ctx->prof_kernels += 1;
  if (!atc_cuda_ok(ctx, cudaGetLastError(), "k_eval_ext") ||
      !atc_cuda_ok(ctx, cudaMemcpyAsync(fail_t, d_out, n, cudaMemcpyDeviceToHost, st), "D2H") ||
      !atc_cuda_ok(ctx, cudaMemcpyAsync(reason, d_out + n, n, cudaMemcpyDeviceToHost, st), "D2H") ||
      !atc_cuda_ok(ctx, cudaStreamSynchronize(st), "eval sync"))
    return ATC_ERR_CUDA;
  if (first_pass)
    for (size_t b = 0; b < n; ++b)
      if (reason[b] == ATC_PASS) {
        *first_pass = (int64_t)b;
        break;
      }
  return ATC_OK;
}

int atc_run_reference_ext(atc_ctx* ctx, const atc_spec_ext* spec, const int64_t* sizes, const double* floats,
                          double* const* buffers, const int64_t* buffer_len, const int32_t* buffer_is_f32) {
  ATC_ENTER(ctx);
  ExtView e;
  if (!ext_view(ctx, spec, e)) return ATC_ERR_ARG;
  if (!sizes || !buffers || !buffer_len || (e.nF > 0 && !floats)) {
    atc_set_error(ctx, "bad arguments to atc_run_reference_ext");
    return ATC_ERR_ARG;
  }
  const int64_t lens[3] = {buffer_len[e.arr_of_role[0]], buffer_len[e.arr_of_role[1]], buffer_len[e.arr_of_role[2]]};
  ExtCall c;
  if (const int k = ext_resolve(e, sizes, floats, lens, c)) {
    atc_set_error(ctx, "dispatch failed: %s", ext_check_text(k));
    return ATC_ERR_DISPATCH;
  }
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  double* d[3] = {nullptr, nullptr, nullptr};
  bool ok = true;
  for (int r = 0; r < 3 && ok; ++r) {
    d[r] = (double*)atc_ctx_scratch(ctx, 29 + r, (size_t)lens[r] * 8 + 16);
    ok = d[r] && atc_cuda_ok(ctx, cudaMemcpyAsync(d[r], buffers[e.arr_of_role[r]], (size_t)lens[r] * 8,
                                                  cudaMemcpyHostToDevice, st), "H2D");
  }
  if (!ok) return ATC_ERR_CUDA;
  const int f32 = buffer_is_f32 ? buffer_is_f32[e.arr_of_role[2]] : 0;
  k_ref_ext<<<64, 256, 0, st>>>(e, c, d[0], d[1], d[2], f32);
  return atc_cuda_ok(ctx, cudaGetLastError(), "k_ref_ext") &&
                 atc_cuda_ok(ctx, cudaMemcpyAsync(buffers[e.arr_of_role[2]], d[2], (size_t)lens[2] * 8,
                                                  cudaMemcpyDeviceToHost, st), "D2H") &&
                 atc_cuda_ok(ctx, cudaStreamSynchronize(st), "sync")
             ? ATC_OK
             : ATC_ERR_CUDA;
}

}  // extern "C"
