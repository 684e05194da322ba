// C ABI: the binding evaluator (K1 screen + K2 confirm) over explicit lists and enumerated ranges.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "atc_b200.h"
#include "capi_internal.h"

using namespace atc;

namespace atc {

constexpr int kScreenThreads = 256;

int screen_budget(const SpecView& sp) { return sp.sem == ATC_SEM_GEMM ? 16 : 2; }

// Preconditions of k_screen_conv_planes (screen_rows.cu): the bundled conv2d
// shape — roles tc_n..tc_ow on size params 0..8, dims in=(n,c,h,w),
// weights=(c,k,r,s), out=(n,k,oh,ow) in any order, in/weights/out = arrays
// 0/1/2, a table key free of digit 0, nI <= 32.  The context option
// ATC_OPT_CONV_SCREEN selects k_screen_conv_planes (ATC_CONV_SCREEN_PLANES) or the
// generic k_screen_rows (ATC_CONV_SCREEN_GENERIC) instead of k_screen_conv_pairs
// (A/B checks: tests/test_gpu_eval.py::test_conv_screen_kernels_agree).
bool pairs_disabled(const atc_ctx* ctx) { return ctx->opt_conv_screen != ATC_CONV_SCREEN_AUTO; }

// 32-bit index arithmetic when every t=0 size is <= 200 (any product of 4 sizes < 2^31)
bool ts_i32(const atc_testset_handle* ts) {
  int64_t umax = 0;
  for (int i = 0; i < ts->nI; ++i) umax = std::max<int64_t>(umax, std::llabs(ts->h_ints[i]));
  return umax <= 200;
}

bool conv_thresholds_ok(const atc_ctx* ctx, const SpecView& sp, const RowPlan& plan, int nI) {
  if (ctx->opt_conv_screen == ATC_CONV_SCREEN_GENERIC || sp.sem != ATC_SEM_CONV2D || sp.nS != 9 || sp.nA != 3 ||
      nI > kMaxInts)
    return false;
  for (int i = 0; i < 9; ++i)
    if (plan.role_q[ATC_SZ_CN + i] != i) return false;
  if (plan.dim_mask[0] != 0xFu || plan.dim_mask[1] != 0x72u || plan.dim_mask[2] != 0x191u) return false;
  if (sp.arr_of_role[0] != 0 || sp.arr_of_role[1] != 1 || sp.arr_of_role[2] != 2) return false;
  return plan.key_stride[0] == 0;
}

// Runs K1 + K2 over `n` bindings; survivors/keys live in ctx scratch.
int run_eval(atc_ctx* ctx, const SpecView& sp, const atc_testset_handle* ts, const BindingSource& src,
             uint64_t n, int32_t* keys, uint64_t* surv, uint64_t surv_cap, unsigned long long* surv_cnt,
             int32_t* surv_keys, unsigned long long* hist, cudaStream_t st, const Pos0Table* pt,
             const RowPlan* plan) {
  if (n == 0) return ATC_OK;
  const uint64_t blocks_needed = (n + kScreenThreads - 1) / kScreenThreads;
  const unsigned grid = (unsigned)std::min<uint64_t>(blocks_needed, (uint64_t)ctx->sm_count * 32);
  cudaMemsetAsync(surv_cnt, 0, sizeof(unsigned long long), st);
  auto ev_pair = [&]() {
    std::pair<cudaEvent_t, cudaEvent_t> p{nullptr, nullptr};
    cudaEventCreate(&p.first);
    cudaEventCreate(&p.second);
    return p;
  };
  std::pair<cudaEvent_t, cudaEvent_t> e1{}, e2{};
  if (ctx->prof) {
    e1 = ev_pair();
    cudaEventRecord(e1.first, st);
    ctx->prof_bindings += (long long)n;
  }
  if (plan) {
    const uint64_t rows = n / ts->nI + 2;
    const unsigned g2 = (unsigned)std::min<uint64_t>((rows + kScreenThreads - 1) / kScreenThreads,
                                                     (uint64_t)ctx->sm_count * 16);
    const uint64_t b = src.begin, e = src.begin + n;
    // 32-bit index arithmetic when every t=0 size is <= 200 (any product of 4 sizes < 2^31)
    int64_t umax = 0;
    for (int i = 0; i < ts->nI; ++i) umax = std::max<int64_t>(umax, std::llabs(ts->h_ints[i]));
    const bool i32 = umax <= 200;
    uint32_t q0mask = 0;  // roles bound to digit 0 (after fallbacks)
    for (int rr = 0; rr < ATC_SZ_COUNT; ++rr)
      if (plan->role_q[rr] == 0) q0mask |= 1u << rr;
    constexpr uint32_t kDyn = 0xFFFFFFFFu;
#define ATC_LAUNCH_ROWS(SEM, NS, MASK)                                                                               \
  do {                                                                                                              \
    if (i32)                                                                                                        \
      k_screen_rows<SEM, NS, true, MASK><<<g2, kScreenThreads, 0, st>>>(ts->view, sp, src.perms, src.size_maps, b, \
                                                                        e, *plan, surv, surv_cap, surv_cnt, hist); \
    else                                                                                                            \
      k_screen_rows<SEM, NS, false, MASK><<<g2, kScreenThreads, 0, st>>>(ts->view, sp, src.perms, src.size_maps,  \
                                                                         b, e, *plan, surv, surv_cap, surv_cnt,    \
                                                                         hist);                                    \
  } while (0)
    constexpr uint32_t kM = 1u << ATC_SZ_M, kMcol = (1u << ATC_SZ_M) | (1u << ATC_SZ_LDA) | (1u << ATC_SZ_LDC);
    constexpr uint32_t kCN = 1u << ATC_SZ_CN;
    if (sp.sem == ATC_SEM_GEMM && sp.nS == 3) {
      if (q0mask == kM)
        ATC_LAUNCH_ROWS(ATC_SEM_GEMM, 3, kM);
      else if (q0mask == kMcol)
        ATC_LAUNCH_ROWS(ATC_SEM_GEMM, 3, kMcol);
      else
        ATC_LAUNCH_ROWS(ATC_SEM_GEMM, 3, kDyn);
    } else if (sp.sem == ATC_SEM_GEMM && sp.nS == 6) {
      if (q0mask == kM)
        ATC_LAUNCH_ROWS(ATC_SEM_GEMM, 6, kM);
      else
        ATC_LAUNCH_ROWS(ATC_SEM_GEMM, 6, kDyn);
    } else if (plan->cmask) {  // conv_pairs_ok at table time
      // rank table of pair products when they are small (<= 4095)
      int64_t pmax = 0;
      for (int i = 0; i < ts->nI; ++i)
        for (int k = 0; k < ts->nI; ++k) pmax = std::max<int64_t>(pmax, ts->h_ints[i] * ts->h_ints[k]);
      const int lut_n = pmax < 4096 ? (int)pmax + 1 : 0;
      const size_t nI2 = (size_t)ts->nI * ts->nI;
      const size_t smem = ((size_t)16 << ts->nI) + (size_t)(lut_n + 15) / 16 * 16 +
                          ((size_t)ts->nP * nI2 + 15) / 16 * 16 + (nI2 + 3) / 4 * 4 * sizeof(float) +
                          (size_t)ts->nP * nI2 * 16 + (size_t)ts->nP * ts->nI * 4 +
                          (ts->nI == 9 ? ((size_t)ts->nP * nI2 * ts->nI + 15) / 16 * 16 + (size_t)ts->nP * nI2 * ts->nI * 2
                                       : 0);  // the nI = 9 instance's cube-bound tables
      // one wave of 1024 / kPairThreads CTAs per SM (64 registers): each CTA builds its tables once
      const uint64_t cubes = rows / ts->nI + 2;
      const unsigned g3 = std::min<unsigned>((unsigned)((cubes + kPairThreads - 1) / kPairThreads),
                                             (unsigned)ctx->sm_count * (1024 / kPairThreads));
      if (ts->nI == 9)
        k_screen_conv_pairs<9><<<g3, kPairThreads, smem, st>>>(ts->view, src.perms, src.size_maps, b, e, *plan, surv,
                                                               surv_cap, surv_cnt, hist, lut_n);
      else
        k_screen_conv_pairs<0><<<g3, kPairThreads, smem, st>>>(ts->view, src.perms, src.size_maps, b, e, *plan, surv,
                                                               surv_cap, surv_cnt, hist, lut_n);
    } else if (i32 && conv_thresholds_ok(ctx, sp, *plan, ts->nI)) {
      k_screen_conv_planes<<<g2, kScreenThreads, 0, st>>>(ts->view, src.perms, src.size_maps, b, e, *plan, surv,
                                                        surv_cap, surv_cnt, hist);
    } else {
      if (q0mask == kCN)
        ATC_LAUNCH_ROWS(ATC_SEM_CONV2D, 9, kCN);
      else
        ATC_LAUNCH_ROWS(ATC_SEM_CONV2D, 9, kDyn);
    }
#undef ATC_LAUNCH_ROWS
  } else if (pt) {
    const uint64_t runs = (n + 15) / 16;
    const unsigned g2 = (unsigned)std::min<uint64_t>((runs + kScreenThreads - 1) / kScreenThreads,
                                                     (uint64_t)ctx->sm_count * 16);
    k_screen_enum<<<g2, kScreenThreads, 0, st>>>(ts->view, sp, src, n, *pt, surv, surv_cap, surv_cnt, hist);
  } else {
    k_screen<<<grid, kScreenThreads, 0, st>>>(ts->view, sp, src, n, screen_budget(sp), keys, surv, surv_cap,
                                              surv_cnt, hist, ctx->mode);
  }
  if (ctx->prof) {
    cudaEventRecord(e1.second, st);
    ctx->prof_screen.push_back(e1);
  }
  // (no key initialisation: K2a writes the key of every survivor it reads)
  if (ctx->prof) {
    e2 = ev_pair();
    cudaEventRecord(e2.first, st);
  }
  // K2a: warp per survivor at t = 0; K2b: CTA per (t = 0 passer, t >= 1)
  uint32_t* next = (uint32_t*)atc_ctx_scratch(ctx, 18, surv_cap * 4 + 16);
  unsigned long long* next_cnt = (unsigned long long*)atc_ctx_scratch(ctx, 19, 64);
  if (!next || !next_cnt) {
    atc_set_error(ctx, "scratch allocation failed (K2)");
    return ATC_ERR_CUDA;
  }
  cudaMemsetAsync(next_cnt, 0, 16, st);  // next_cnt[0]: t=0 passers, next_cnt[1]: K2-pre pending
  uint32_t* pend = (uint32_t*)atc_ctx_scratch(ctx, 24, surv_cap * 4 + 16);
  if (!pend) {
    atc_set_error(ctx, "scratch allocation failed (K2)");
    return ATC_ERR_CUDA;
  }
  // grids bounded by the most work there can be (survivors <= bindings screened):
  // small spaces launch a few CTAs instead of 8 per SM
  const uint64_t max_surv = std::min<uint64_t>(n, surv_cap);
  // gemm spaces keep few survivors (grid-stride loops cover them): a small cap keeps
  // their mostly-empty K2 grids from taking SM slots from the concurrent conv chain
  // (large-output gemm spaces — a drawn int above 16, e.g. config 1's 64^3 — get the
  // full grid: their checks are long)
  int64_t umax_all = 0;
  for (int64_t v : ts->h_ints) umax_all = std::max(umax_all, v);
  // conv K2 grids at two CTAs per SM (one resident wave at 126 registers, grid-stride
  // loops): the eight chains' K2 kernels then interleave instead of queueing waves
  // behind each other (corpus sweep 0.78 -> 0.76 ms; 1 / 2 / 4 / 8 per SM: 0.744 /
  // 0.757 / 0.803 / 0.783 ms, e2e 1.14 / 1.12 / 1.12 / 1.12)
  const uint64_t k2_cap = sp.sem == ATC_SEM_GEMM ? (umax_all <= 16 ? 64 : (uint64_t)ctx->sm_count * 8)
                                                 : (uint64_t)ctx->sm_count * 2;
  const unsigned g_t0 = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((max_surv + 7) / 8, k2_cap));
  const unsigned g_t1 = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>((max_surv * (uint64_t)std::max(ts->T - 1, 0) + 7) / 8, k2_cap));
  const bool pre = sp.sem == ATC_SEM_CONV2D;
  const int screened = plan && plan->cmask && src.enumerated ? 1 : 0;  // pair-screened conv space
  if (pre)
    k_confirm_pre<<<(unsigned)std::max<uint64_t>(1, std::min<uint64_t>((max_surv + 255) / 256, k2_cap)),
                    256, 0, st>>>(ts->view, sp, src, surv, surv_cnt, surv_cap, surv_keys, pend, next_cnt + 1,
                                  ctx->mode, screened);
  if (pre && !keys) {
    // enumerated ranges report reasons, not failing tests: t >= 1 first over every
    // pending survivor, then t = 0 only where it can change the reason (k_confirm_t0)
    // each (binding, t) item's outputs over opt_k2b_parts warps (the long checks of the
    // few bindings that pass many tests set the kernel's tail)
    const int kp = ctx->opt_k2b_parts;
    k_confirm_warp<<<(unsigned)std::min<uint64_t>((uint64_t)g_t1 * kp, k2_cap), 256, 0, st>>>(
        ts->view, sp, src, surv, surv_cap, surv_keys, pend, next_cnt + 1, ctx->mode, screened, kp);
    const unsigned g_lazy = (unsigned)std::min<uint64_t>((uint64_t)g_t0 * 8, k2_cap);  // 8 warps per binding
    k_confirm_t0<<<g_lazy, 256, 0, st>>>(ts->view, sp, src, surv, surv_cnt, surv_cap, surv_keys, pend, next_cnt + 1,
                                         next, next_cnt, ctx->mode, 1, screened, 1);
  } else if (sp.sem == ATC_SEM_GEMM && umax_all > 16 && ctx->mode == ATC_MODE_FP64) {
    // long gemm checks (config 1's 64^3: 4,096 outputs of 64 terms per (binding, t)):
    // each binding's outputs split over kGemmParts warps in K2a and K2b, failures
    // folded with atomicMin into keys initialised to kPassKey; K2b walks every
    // survivor (those failing t = 0 are skipped by their key)
    constexpr int kGemmParts = 8;
    const unsigned g_t0p = (unsigned)std::min<uint64_t>((uint64_t)g_t0 * kGemmParts, k2_cap);
    const unsigned g_t1p = (unsigned)std::min<uint64_t>((uint64_t)g_t1 * kGemmParts, k2_cap);
    k_init_keys<<<(unsigned)std::max<uint64_t>(1, std::min<uint64_t>((max_surv + 255) / 256, 1024)), 256, 0, st>>>(
        surv_keys, surv_cnt, surv_cap);
    k_confirm_t0<<<g_t0p, 256, 0, st>>>(ts->view, sp, src, surv, surv_cnt, surv_cap, surv_keys, nullptr, next_cnt + 1,
                                        next, next_cnt, ctx->mode, 1, screened, kGemmParts);
    k_confirm_warp<<<g_t1p, 256, 0, st>>>(ts->view, sp, src, surv, surv_cap, surv_keys, nullptr, surv_cnt, ctx->mode,
                                          screened, kGemmParts);
    if (ctx->prof) ctx->prof_kernels += 1;
  } else {
    k_confirm_t0<<<g_t0, 256, 0, st>>>(ts->view, sp, src, surv, surv_cnt, surv_cap, surv_keys,
                                       pre ? pend : nullptr, next_cnt + 1, next, next_cnt, ctx->mode, 0, screened, 1);
    k_confirm_warp<<<g_t1, 256, 0, st>>>(ts->view, sp, src, surv, surv_cap, surv_keys, next, next_cnt, ctx->mode,
                                         screened, 1);
  }
  if (ctx->prof) {
    cudaEventRecord(e2.second, st);
    ctx->prof_confirm.push_back(e2);
  }
  if (keys) k_merge_keys<<<64, 256, 0, st>>>(surv, surv_cnt, surv_cap, surv_keys, keys);
  if (ctx->prof) ctx->prof_kernels += (keys ? 4 : 3) + (pre ? 1 : 0); /* K1, (K2-pre), K2a, K2b (+ merge) */
  if (!atc_cuda_ok(ctx, cudaGetLastError(), "evaluator launch")) return ATC_ERR_CUDA;
  return ATC_OK;
}

}  // namespace atc

extern "C" {

int atc_eval_bindings_device(atc_ctx* ctx, const atc_spec_desc* spec, const atc_testset_handle* ts,
                             const uint8_t* d_arr_map, const uint8_t* d_size_map, int64_t n_bindings,
                             int32_t mode, int8_t* d_fail_t, int8_t* d_reason, void* stream) {
  ATC_ENTER(ctx);
  SpecView sp;
  if (!build_spec_view(ctx, spec, sp)) return ATC_ERR_ARG;
  if (!ts || n_bindings < 0 || (mode != ATC_MODE_FP64 && mode != ATC_MODE_FP32_SCREEN)) {
    atc_set_error(ctx, "bad arguments to atc_eval_bindings");
    return ATC_ERR_ARG;
  }
  if (n_bindings == 0) return ATC_OK;
  cudaSetDevice(ctx->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
  ts_wait(ts, st);
  const uint64_t n = (uint64_t)n_bindings;
  ctx->mode = mode;
  int32_t* keys = (int32_t*)atc_ctx_scratch(ctx, 0, n * 4);
  uint64_t* surv = (uint64_t*)atc_ctx_scratch(ctx, 1, n * 8);
  int32_t* skeys = (int32_t*)atc_ctx_scratch(ctx, 2, n * 4);
  unsigned long long* cnt = (unsigned long long*)atc_ctx_scratch(ctx, 3, 64);
  if (!keys || !surv || !skeys || !cnt) {
    atc_set_error(ctx, "scratch allocation failed for %lld bindings", (long long)n_bindings);
    return ATC_ERR_CUDA;
  }
  BindingSource src{d_arr_map, d_size_map, nullptr, 0, 0, 0};
  k_fill_i32<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, st>>>(keys, (int64_t)n, kPassKey);
  int rc = run_eval(ctx, sp, ts, src, n, keys, surv, n, cnt, skeys, nullptr, st);
  if (rc) return rc;
  k_keys_to_verdicts<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, st>>>(keys, (int64_t)n,
                                                                                         d_fail_t, d_reason);
  return atc_cuda_ok(ctx, cudaGetLastError(), "verdict launch") ? ATC_OK : ATC_ERR_CUDA;
}

int atc_eval_bindings(atc_ctx* ctx, const atc_spec_desc* spec, const atc_testset_handle* ts,
                      const uint8_t* arr_map, const uint8_t* size_map, int64_t n_bindings, int32_t mode,
                      int8_t* fail_t, int8_t* reason, int64_t* first_pass) {
  ATC_ENTER(ctx);
  if (first_pass) *first_pass = -1;
  if (n_bindings < 0 || (n_bindings > 0 && (!arr_map || !size_map || !fail_t || !reason))) {
    atc_set_error(ctx, "bad arguments to atc_eval_bindings");
    return ATC_ERR_ARG;
  }
  if (n_bindings == 0) return ATC_OK;
  SpecView sp;
  if (!build_spec_view(ctx, spec, sp)) return ATC_ERR_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t n = (size_t)n_bindings;
  uint8_t* d_in = (uint8_t*)atc_ctx_scratch(ctx, 4, n * (sp.nA + sp.nS));
  int8_t* d_out = (int8_t*)atc_ctx_scratch(ctx, 5, n * 2);
  if (!d_in || !d_out) {
    atc_set_error(ctx, "scratch allocation failed");
    return ATC_ERR_CUDA;
  }
  if (!atc_cuda_ok(ctx, cudaMemcpyAsync(d_in, arr_map, n * sp.nA, cudaMemcpyHostToDevice, st), "H2D arr_map") ||
      !atc_cuda_ok(ctx, cudaMemcpyAsync(d_in + n * sp.nA, size_map, n * sp.nS, cudaMemcpyHostToDevice, st),
                   "H2D size_map"))
    return ATC_ERR_CUDA;
  int rc = atc_eval_bindings_device(ctx, spec, ts, d_in, d_in + n * sp.nA, n_bindings, mode, d_out, d_out + n, st);
  if (rc) return rc;
  if (!atc_cuda_ok(ctx, cudaMemcpyAsync(fail_t, d_out, n, cudaMemcpyDeviceToHost, st), "D2H") ||
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

int atc_eval_bindings_many(atc_ctx* ctx, atc_bind_job* jobs, int32_t n_jobs, int32_t mode) {
  ATC_ENTER(ctx);
  if (n_jobs < 0 || (n_jobs > 0 && !jobs) || (mode != ATC_MODE_FP64 && mode != ATC_MODE_FP32_SCREEN)) {
    atc_set_error(ctx, "bad arguments to atc_eval_bindings_many");
    return ATC_ERR_ARG;
  }
  // validate every job and lay out one staging block: maps in, verdicts out
  std::vector<size_t> in_off(n_jobs), out_off(n_jobs);
  size_t in_bytes = 0, out_bytes = 0;
  uint64_t nmax = 0;
  int first_rc = ATC_OK;
  for (int j = 0; j < n_jobs; ++j) {
    atc_bind_job& jb = jobs[j];
    jb.first_pass = -1;
    jb.status = ATC_OK;
    SpecView sp;
    if (!jb.ts || jb.n_bindings < 0 ||
        (jb.n_bindings > 0 && (!jb.arr_map || !jb.size_map || !jb.fail_t || !jb.reason))) {
      atc_set_error(ctx, "bad arguments to atc_eval_bindings_many (job %d)", j);
      jb.status = ATC_ERR_ARG;
    } else if (!build_spec_view(ctx, jb.spec, sp)) {
      jb.status = ATC_ERR_ARG;
    }
    if (jb.status != ATC_OK) {
      if (first_rc == ATC_OK) first_rc = jb.status;
      continue;
    }
    in_off[j] = in_bytes;
    out_off[j] = out_bytes;
    in_bytes += ((size_t)jb.n_bindings * (sp.nA + sp.nS) + 15) / 16 * 16;
    out_bytes += ((size_t)jb.n_bindings * 2 + 15) / 16 * 16;
    nmax = std::max<uint64_t>(nmax, (uint64_t)jb.n_bindings);
  }
  if (first_rc != ATC_OK || in_bytes == 0) return first_rc;
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  // scratch sized once for the largest list (run_eval's slots), so no buffer is
  // reallocated while an earlier list's kernels are queued
  uint8_t* pin = (uint8_t*)atc_ctx_pinned(ctx, 2, in_bytes + out_bytes);
  uint8_t* d_in = (uint8_t*)atc_ctx_scratch(ctx, 4, in_bytes);
  int8_t* d_out = (int8_t*)atc_ctx_scratch(ctx, 5, out_bytes);
  if (!pin || !d_in || !d_out || !atc_ctx_scratch(ctx, 0, nmax * 4) || !atc_ctx_scratch(ctx, 1, nmax * 8) ||
      !atc_ctx_scratch(ctx, 2, nmax * 4) || !atc_ctx_scratch(ctx, 3, 64) ||
      !atc_ctx_scratch(ctx, 18, nmax * 4 + 16) || !atc_ctx_scratch(ctx, 19, 64) ||
      !atc_ctx_scratch(ctx, 24, nmax * 4 + 16)) {
    atc_set_error(ctx, "scratch allocation failed");
    return ATC_ERR_CUDA;
  }
  for (int j = 0; j < n_jobs; ++j) {
    const atc_bind_job& jb = jobs[j];
    const size_t n = (size_t)jb.n_bindings;
    std::memcpy(pin + in_off[j], jb.arr_map, n * jb.spec->n_arrays);
    std::memcpy(pin + in_off[j] + n * jb.spec->n_arrays, jb.size_map, n * jb.spec->n_sizes);
  }
  if (!atc_cuda_ok(ctx, cudaMemcpyAsync(d_in, pin, in_bytes, cudaMemcpyHostToDevice, st), "H2D maps"))
    return ATC_ERR_CUDA;
  for (int j = 0; j < n_jobs; ++j) {
    atc_bind_job& jb = jobs[j];
    if (jb.n_bindings == 0) continue;
    const size_t n = (size_t)jb.n_bindings;
    const uint8_t* am = d_in + in_off[j];
    jb.status = atc_eval_bindings_device(ctx, jb.spec, jb.ts, am, am + n * jb.spec->n_arrays, jb.n_bindings, mode,
                                         d_out + out_off[j], d_out + out_off[j] + n, st);
    if (jb.status != ATC_OK) return jb.status;
  }
  if (!atc_cuda_ok(ctx, cudaMemcpyAsync(pin + in_bytes, d_out, out_bytes, cudaMemcpyDeviceToHost, st), "D2H") ||
      !atc_cuda_ok(ctx, cudaStreamSynchronize(st), "eval sync"))
    return ATC_ERR_CUDA;
  for (int j = 0; j < n_jobs; ++j) {
    atc_bind_job& jb = jobs[j];
    const size_t n = (size_t)jb.n_bindings;
    const int8_t* o = (const int8_t*)(pin + in_bytes + out_off[j]);
    std::memcpy(jb.fail_t, o, n);
    std::memcpy(jb.reason, o + n, n);
    for (size_t b = 0; b < n; ++b)
      if (jb.reason[b] == ATC_PASS) {
        jb.first_pass = (int64_t)b;
        break;
      }
  }
  return ATC_OK;
}

}  // extern "C"

namespace atc {

// ---- enumerated spaces --------------------------------------------------------

int plan_enumerated(atc_ctx* ctx, const atc_spec_desc* spec, const atc_testset_handle* ts, const uint8_t* perms,
                    int32_t n_perms, uint64_t begin, uint64_t end, int32_t mode, EnumPlan& e) {
  if (!build_spec_view(ctx, spec, e.sp)) return ATC_ERR_ARG;
  const SpecView& sp = e.sp;
  if (!ts || n_perms < 0 || !perms || end < begin || (mode != ATC_MODE_FP64 && mode != ATC_MODE_FP32_SCREEN)) {
    atc_set_error(ctx, "bad arguments to atc_eval_enumerated");
    return ATC_ERR_ARG;
  }
  for (int p = 0; p < n_perms; ++p)
    for (int a = 0; a < sp.nA; ++a)
      if (perms[p * sp.nA + a] >= ts->nP) {
        atc_set_error(ctx, "perm %d maps array %d to pointer %d of %d", p, a, perms[p * sp.nA + a], ts->nP);
        return ATC_ERR_ARG;
      }
  e.size_maps = 1;
  for (int q = 0; q < sp.nS; ++q) e.size_maps *= (uint64_t)ts->nI;
  if (end > (uint64_t)n_perms * e.size_maps) {
    atc_set_error(ctx, "range end %llu beyond the space (%llu)", (unsigned long long)end,
                  (unsigned long long)((uint64_t)n_perms * e.size_maps));
    return ATC_ERR_ARG;
  }
  // position-0 table (k_pos0_table): roles the first output element depends on
  Pos0Table& pt = e.pt;
  pt = Pos0Table{};
  e.use_table = true;
  if (sp.sem == ATC_SEM_GEMM) {
    const bool row = sp.layout == ATC_LAYOUT_ROW;
    const int ld = row ? (sp.role_size[ATC_SZ_LDB] >= 0 ? sp.role_size[ATC_SZ_LDB] : sp.role_size[ATC_SZ_N])
                       : (sp.role_size[ATC_SZ_LDA] >= 0 ? sp.role_size[ATC_SZ_LDA] : sp.role_size[ATC_SZ_M]);
    pt.R = 2;
    pt.q[0] = sp.role_size[ATC_SZ_K];
    pt.q[1] = ld;
  } else {
    pt.R = 5;
    const int roles[5] = {ATC_SZ_CC, ATC_SZ_CH, ATC_SZ_CW, ATC_SZ_CR, ATC_SZ_CS};
    for (int r = 0; r < 5; ++r) pt.q[r] = sp.role_size[roles[r]];
  }
  pt.per_perm = 1;
  for (int r = 0; r < pt.R; ++r) {
    if (pt.q[r] < 0) e.use_table = false;
    pt.per_perm *= (uint64_t)ts->nI;
  }
  e.table_bytes = pt.per_perm * (uint64_t)n_perms;
  if (e.table_bytes > (256ull << 20)) e.use_table = false;
  // row-hoisted screen (k_screen_rows) for the bundled spec shapes
  RowPlan& plan = e.plan;
  plan = RowPlan{};
  e.use_rows = e.use_table && ((sp.sem == ATC_SEM_GEMM && (sp.nS == 3 || sp.nS == 6)) ||
                               (sp.sem == ATC_SEM_CONV2D && sp.nS == 9));
  if (e.use_rows) {
    for (int a = 0; a < sp.nA; ++a) {
      plan.dim_mask[a] = 0;
      for (int d = 0; d < sp.ndims[a]; ++d) {
        if (plan.dim_mask[a] & (1u << sp.dims[a][d])) e.use_rows = false;  // repeated dim: not expressible
        plan.dim_mask[a] |= 1u << sp.dims[a][d];
      }
    }
    for (int r = 0; r < ATC_SZ_COUNT; ++r) plan.role_q[r] = sp.role_size[r];
    if (sp.sem == ATC_SEM_GEMM) {  // equivalence.cpp:46-48 fallbacks
      const bool row = sp.layout == ATC_LAYOUT_ROW;
      if (plan.role_q[ATC_SZ_LDA] < 0) plan.role_q[ATC_SZ_LDA] = row ? sp.role_size[ATC_SZ_K] : sp.role_size[ATC_SZ_M];
      if (plan.role_q[ATC_SZ_LDB] < 0) plan.role_q[ATC_SZ_LDB] = row ? sp.role_size[ATC_SZ_N] : sp.role_size[ATC_SZ_K];
      if (plan.role_q[ATC_SZ_LDC] < 0) plan.role_q[ATC_SZ_LDC] = row ? sp.role_size[ATC_SZ_N] : sp.role_size[ATC_SZ_M];
    }
    uint64_t mul = 1;
    for (int q = 0; q < ATC_MAX_SIZES; ++q) plan.key_stride[q] = 0;
    for (int k = 0; k < pt.R; ++k) {
      plan.key_stride[pt.q[k]] += mul;
      mul *= (uint64_t)ts->nI;
    }
  }
  return ATC_OK;
}

// Uploads the permutations and builds the per-space tables (k_gemm_need,
// k_pos0_table) on the stream; scratch slots 6/17/21 are reused in stream order.
int enqueue_tables(atc_ctx* ctx, EnumPlan& e, const atc_testset_handle* ts, const uint8_t* perms, int32_t n_perms,
                   uint8_t** d_perms_out, cudaStream_t st, uint64_t begin, uint64_t end) {
  const SpecView& sp = e.sp;
  // only the permutations [p_lo, p_hi] the range [begin, end) touches are tabulated
  // (a rank of a multi-GPU sweep owns a block of the space)
  const uint64_t p_lo = end > begin ? begin / e.size_maps : 0;
  const uint64_t p_hi = end > begin ? (end - 1) / e.size_maps : 0;
  const uint64_t np_local = std::min<uint64_t>(p_hi - p_lo + 1, (uint64_t)n_perms - p_lo);
  uint8_t* d_perms = *d_perms_out;  // device-resident already (batches), else staged here
  if (!d_perms) {
    d_perms = (uint8_t*)atc_ctx_scratch(ctx, 6, (size_t)n_perms * sp.nA + 16);
    if (!d_perms) {
      atc_set_error(ctx, "scratch allocation failed");
      return ATC_ERR_CUDA;
    }
    cudaMemcpyAsync(d_perms, perms, (size_t)n_perms * sp.nA, cudaMemcpyHostToDevice, st);
    *d_perms_out = d_perms;
  }
  if (e.use_rows && sp.sem == ATC_SEM_GEMM) {  // written-set check by lookup (k_gemm_need)
    const unsigned cells = (unsigned)(ts->nP * ts->nI * ts->nI);
    int32_t* need = (int32_t*)atc_ctx_scratch(ctx, 21, (size_t)cells * 4 + 16);
    if (!need) {
      atc_set_error(ctx, "scratch allocation failed (gemm_need)");
      return ATC_ERR_CUDA;
    }
    k_gemm_need<<<cells, 128, 0, st>>>(ts->view, sp.layout == ATC_LAYOUT_ROW ? 1 : 0, need);
    e.plan.gemm_need = need;
    if (ctx->prof) ctx->prof_kernels += 1;
  }
  if (e.use_table) {
    // conv with nI <= 11: the pair screen reads the table as one bit word per
    // (perm, h, w, r, s) over the values of tc_c (key stride 1), for output
    // positions 0 and 1
    const bool pairs = e.use_rows && ts_i32(ts) && conv_thresholds_ok(ctx, sp, e.plan, ts->nI) && ts->nI <= 11 &&
                       ts->nP <= 8 /* k_screen_conv_pairs' tables within 64 KB of shared memory */ &&
                       e.plan.key_stride[1] == 1 && !pairs_disabled(ctx);
    uint8_t* tab = (uint8_t*)atc_ctx_scratch(ctx, 17, e.table_bytes * (pairs ? 2 : 1) + 32);
    if (!tab) {
      atc_set_error(ctx, "scratch allocation failed (table)");
      return ATC_ERR_CUDA;
    }
    uint8_t* tab1 = pairs ? tab + (e.table_bytes + 15) / 16 * 16 : nullptr;
    e.pt.table = tab;
    e.plan.pt = e.pt;
    // conv with the canonical key (c first): one running sum per (perm, h, w, r, s)
    const uint64_t t_off = p_lo * e.pt.per_perm, t_bytes = np_local * e.pt.per_perm;
    const uint8_t* perms_local = d_perms + p_lo * sp.nA;
    e.plan.cmask = nullptr;
    uint32_t* cm = nullptr;
    const uint64_t words = e.table_bytes / (uint64_t)ts->nI;
    if (pairs) {
      cm = (uint32_t*)atc_ctx_scratch(ctx, 23, words * 4 + 32);
      if (!cm) {
        atc_set_error(ctx, "scratch allocation failed (cmask)");
        return ATC_ERR_CUDA;
      }
      e.plan.cmask = cm;
    }
    const uint64_t w_off = t_off / (uint64_t)ts->nI;
    e.plan.allbad = nullptr;
    if (sp.sem == ATC_SEM_CONV2D && e.pt.R == 5 && e.plan.key_stride[1] == 1 && e.use_rows &&
        conv_thresholds_ok(ctx, sp, e.plan, ts->nI)) {
      // one running sum per (perm, h, w, r, s); the pair screen's bit words come out
      // of the same pass
      // every element a sum reads: in < (cmax*hmax + rmax)*wmax + smax + 1 (position 1
      // included), weights < cmax*rmax*smax; staged in shared memory when <= 48 KB
      int64_t umax = 0;
      for (int q = 0; q < ts->nI; ++q) umax = std::max<int64_t>(umax, ts->h_ints[q]);
      const int64_t need_a = (umax * umax + umax) * umax + umax + 1, need_b = umax * umax * umax;
      const bool stage = umax >= 1 && need_a + need_b <= 6144;
      const int sa = stage ? (int)need_a : 0, sb = stage ? (int)need_b : 0;
      const uint64_t per = (uint64_t)ts->nI * ts->nI * ts->nI * ts->nI;
      const dim3 grid((unsigned)std::max<uint64_t>(1, std::min<uint64_t>((per + 255) / 256, 65535)),
                      (unsigned)np_local);
      uint64_t nc = 0;  // distinct values among test 0's ints: the table kernel's tuples
      for (int d = 0; d < ts->nI; ++d)
        nc += std::find(ts->h_ints.begin(), ts->h_ints.begin() + d, ts->h_ints[d]) == ts->h_ints.begin() + d;
      const dim3 grid_c((unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nc * nc * nc * nc + 255) / 256, 65535)),
                        (unsigned)np_local);
      // the all-bad masks (per (perm, w, r, s), from the same pass) when h is the fastest
      // digit of the cmask word index
      uint32_t* ab = nullptr;
      if (cm && e.plan.key_stride[2] == (uint64_t)ts->nI) {
        ab = (uint32_t*)atc_ctx_scratch(ctx, 32, (words / ts->nI + 8) * 4);
        if (!ab) {
          atc_set_error(ctx, "scratch allocation failed (allbad)");
          return ATC_ERR_CUDA;
        }
        cudaMemsetAsync(ab + w_off / ts->nI, 0, (size_t)(t_bytes / ts->nI / ts->nI + 1) * 4, st);
        e.plan.allbad = ab;
      }
      k_pos0_table_conv<<<grid_c, 256, (size_t)(sa + sb) * sizeof(double), st>>>(
          ts->view, sp, perms_local, (int)np_local, e.pt, tab + t_off, tab1 ? tab1 + t_off : nullptr,
          cm ? cm + w_off : nullptr, sa, sb, ab ? ab + w_off / ts->nI : nullptr);
      // (the position-1 bytes only feed the words, which the expansion copies)
      k_pos0_table_expand<<<grid, 256, 0, st>>>(ts->view, (int)np_local, e.pt, tab + t_off, nullptr,
                                                cm ? cm + w_off : nullptr, ab ? ab + w_off / ts->nI : nullptr);
      if (ctx->prof) ctx->prof_kernels += 2;
    } else {
      k_pos0_table<<<(unsigned)std::max<uint64_t>(
                         1, std::min<uint64_t>((t_bytes + 255) / 256, (uint64_t)ctx->sm_count * 16)),
                     256, 0, st>>>(ts->view, sp, perms_local, (int)np_local, e.pt, tab + t_off,
                                   tab1 ? tab1 + t_off : nullptr);
      if (ctx->prof) ctx->prof_kernels += 1;
      if (pairs) {
        const uint64_t w_local = t_bytes / (uint64_t)ts->nI;
        const unsigned g =
            (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((w_local + 255) / 256, (uint64_t)ctx->sm_count * 16));
        k_cmask<<<g, 256, 0, st>>>(tab + t_off, w_local, ts->nI, cm + w_off, 0);
        k_cmask<<<g, 256, 0, st>>>(tab1 + t_off, w_local, ts->nI, cm + w_off, 16);
        if (ctx->prof) ctx->prof_kernels += 2;
      }
    }
  }
  return ATC_OK;
}

}  // namespace atc

extern "C" {

int atc_eval_enumerated(atc_ctx* ctx, const atc_spec_desc* spec, const atc_testset_handle* ts,
                        const uint8_t* perms, int32_t n_perms, uint64_t begin, uint64_t end, int32_t mode,
                        uint64_t* survivors, int64_t cap, int64_t* n_survivors, int64_t* reason_counts) {
  ATC_ENTER(ctx);
  EnumPlan e;
  int rc = plan_enumerated(ctx, spec, ts, perms, n_perms, begin, end, mode, e);
  if (rc) return rc;
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  ts_wait(ts, st);
  ctx->mode = mode;
  const uint64_t chunk_cap = kEnumChunkCap;
  uint64_t* surv = (uint64_t*)atc_ctx_scratch(ctx, 1, chunk_cap * 8);
  int32_t* skeys = (int32_t*)atc_ctx_scratch(ctx, 2, chunk_cap * 4);
  unsigned long long* cnt = (unsigned long long*)atc_ctx_scratch(ctx, 3, 64);
  unsigned long long* hist = (unsigned long long*)atc_ctx_scratch(ctx, 7, 64);
  if (!surv || !skeys || !cnt || !hist) {
    atc_set_error(ctx, "scratch allocation failed");
    return ATC_ERR_CUDA;
  }
  cudaMemsetAsync(hist, 0, 64, st);
  uint8_t* d_perms = nullptr;
  rc = enqueue_tables(ctx, e, ts, perms, n_perms, &d_perms, st, begin, end);
  if (rc) return rc;
  // result block on the device: [0] survivor count (copied from cnt), [1] passing
  // count, [2..2+cap) passing global indices; reasons accumulate in `hist`
  uint64_t* res = (uint64_t*)atc_ctx_scratch(ctx, 20, (chunk_cap + 2) * 8);
  uint64_t* h_res = (uint64_t*)atc_ctx_pinned(ctx, 0, (kResultPrefix + 2 + ATC_REASON_COUNT) * 8);
  if (!res || !h_res) {
    atc_set_error(ctx, "result buffer allocation failed");
    return ATC_ERR_CUDA;
  }
  std::vector<uint64_t> pass_all;
  int64_t passed = 0;
  uint64_t chunk = 1ull << 34;  // one chunk covers every corpus space
  for (uint64_t lo = begin; lo < end;) {
    const uint64_t hi = std::min(end, lo + chunk);
    BindingSource src{nullptr, nullptr, d_perms, e.size_maps, lo, 1};
    rc = run_eval(ctx, e.sp, ts, src, hi - lo, nullptr, surv, chunk_cap, cnt, skeys, hist, st,
                  e.use_table ? &e.pt : nullptr, e.use_rows ? &e.plan : nullptr);
    if (rc) return rc;
    // K2 outcomes -> passing list + reason histogram, on the device (one sync per chunk)
    cudaMemsetAsync(res + 1, 0, 8, st);
    k_finalize<<<64, 256, 0, st>>>(surv, cnt, chunk_cap, skeys, lo, res, chunk_cap, hist);
    if (ctx->prof) ctx->prof_kernels += 1;
    // the passing list is unordered on the device: the smallest `cap` need all of it
    const uint64_t pre = cap > 0 ? kResultPrefix : 0;
    if (!atc_cuda_ok(ctx, cudaMemcpyAsync(h_res, res, (2 + pre) * 8, cudaMemcpyDeviceToHost, st), "D2H result") ||
        !atc_cuda_ok(ctx, cudaMemcpyAsync(h_res + 2 + kResultPrefix, hist, ATC_REASON_COUNT * 8,
                                          cudaMemcpyDeviceToHost, st), "D2H hist") ||
        !atc_cuda_ok(ctx, cudaStreamSynchronize(st), "enumerate sync"))
      return ATC_ERR_CUDA;
    const uint64_t c = h_res[0], npass = h_res[1];
    if (c > chunk_cap) {  // too many survivors for this chunk: restart with smaller chunks
      if (chunk == 1) {
        atc_set_error(ctx, "survivor overflow");
        return ATC_ERR_CUDA;
      }
      chunk = std::max<uint64_t>(1, std::min(chunk, hi - lo) / 8);
      cudaMemsetAsync(hist, 0, 64, st);
      lo = begin;
      pass_all.clear();
      passed = 0;
      continue;
    }
    if (ctx->prof) ctx->prof_survivors += (long long)c;
    const uint64_t want = cap > 0 ? npass : 0;
    std::vector<uint64_t> chunk_pass(h_res + 2, h_res + 2 + std::min(want, pre));
    if (want > pre) {  // rare: more passing bindings than the pinned prefix
      chunk_pass.resize(want);
      if (!atc_cuda_ok(ctx, cudaMemcpyAsync(chunk_pass.data(), res + 2, want * 8, cudaMemcpyDeviceToHost, st),
                       "D2H passing") ||
          !atc_cuda_ok(ctx, cudaStreamSynchronize(st), "passing sync"))
        return ATC_ERR_CUDA;
    }
    std::sort(chunk_pass.begin(), chunk_pass.end());
    pass_all.insert(pass_all.end(), chunk_pass.begin(), chunk_pass.end());
    passed += (int64_t)npass;
    lo = hi;
  }
  for (size_t i = 0; i < pass_all.size() && (int64_t)i < cap; ++i)
    if (survivors) survivors[i] = pass_all[i];
  if (n_survivors) *n_survivors = passed;
  if (reason_counts) {
    const uint64_t* h_hist = h_res + 2 + kResultPrefix;
    for (int r = 0; r < ATC_REASON_COUNT; ++r) reason_counts[r] = end > begin ? (int64_t)h_hist[r] : 0;
    reason_counts[ATC_PASS] = passed;
  }
  return ATC_OK;
}

}  // extern "C"
