// C ABI (include/atc_b200.h): context, test-set upload, evaluator entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <atomic>
#include <string>
#include <vector>

#include "atc_b200.h"
#include "capi_internal.h"
#include "eval_common.cuh"

namespace atc {
__global__ void k_probe_regions(int T, int nP, const uint64_t* seeds, const uint64_t* skips, const int64_t* region_len,
                                const int32_t* is_f32, const int64_t* region_off, const int64_t* need, double* init,
                                double* fin, TestsetView v, const int64_t* diff_off, const int32_t* diff_pos,
                                const double* diff_val, const double* pre, const int64_t* pre_off);
__global__ void k_apply_diffs(int nP, const int64_t* region_len, const int64_t* region_off, const int64_t* diff_off,
                              const int32_t* diff_pos, const double* diff_val, double* fin);
__global__ void k_build_dirty(TestsetView ts, int32_t* dirty_pos, int32_t* dirty_cnt, int32_t* dirty_max);

__global__ void k_screen(TestsetView ts, SpecView sp, BindingSource src, uint64_t n, int budget,
                         int32_t* keys, uint64_t* surv, uint64_t surv_cap, unsigned long long* surv_cnt,
                         unsigned long long* reason_hist, int mode);
__global__ void k_pos0_table(TestsetView ts, SpecView sp, const uint8_t* perms, int n_perms, Pos0Table pt,
                             uint8_t* out, uint8_t* out1);
__global__ void k_pos0_table_conv(TestsetView ts, SpecView sp, const uint8_t* perms, int n_perms, Pos0Table pt,
                                  uint8_t* out, uint8_t* out1, uint32_t* cm, int stage_a, int stage_b);
__global__ void k_screen_enum(TestsetView ts, SpecView sp, BindingSource src, uint64_t n, Pos0Table pt,
                              uint64_t* surv, uint64_t surv_cap, unsigned long long* surv_cnt,
                              unsigned long long* reason_hist);
__global__ void k_gemm_need(TestsetView ts, int row_major, int32_t* need);
__global__ void k_cmask(const uint8_t* table, uint64_t n_words, int nI, uint32_t* cmask, int shift);
__global__ void k_screen_conv_pairs(TestsetView ts, const uint8_t* perms, uint64_t size_maps, uint64_t begin,
                                    uint64_t end, RowPlan plan, uint64_t* surv, uint64_t surv_cap,
                                    unsigned long long* surv_cnt, unsigned long long* reason_hist, int lut_n);
__global__ void k_screen_conv_planes(TestsetView ts, const uint8_t* perms, uint64_t size_maps, uint64_t begin,
                                   uint64_t end, RowPlan plan, uint64_t* surv, uint64_t surv_cap,
                                   unsigned long long* surv_cnt, unsigned long long* reason_hist);
template <int SEM, int NS, bool I32, uint32_t Q0MASK>
__global__ void k_screen_rows(TestsetView ts, SpecView sp, const uint8_t* perms, uint64_t size_maps, uint64_t begin,
                              uint64_t end, RowPlan plan, uint64_t* surv, uint64_t surv_cap,
                              unsigned long long* surv_cnt, unsigned long long* reason_hist);
__global__ void k_confirm_warp(TestsetView ts, SpecView sp, BindingSource src, const uint64_t* surv,
                               uint64_t surv_cap, int32_t* surv_keys, const uint32_t* sel,
                               const unsigned long long* sel_cnt, int mode, int screened);
__global__ void k_confirm_pre(TestsetView ts, SpecView sp, BindingSource src, const uint64_t* surv,
                              const unsigned long long* surv_cnt, uint64_t surv_cap, int32_t* surv_keys,
                              uint32_t* pend, unsigned long long* pend_cnt, int mode, int screened);
__global__ void k_confirm_t0(TestsetView ts, SpecView sp, BindingSource src, const uint64_t* surv,
                             const unsigned long long* surv_cnt, uint64_t surv_cap, int32_t* surv_keys,
                             const uint32_t* pend, const unsigned long long* pend_cnt, uint32_t* next,
                             unsigned long long* next_cnt, int mode, int lazy, int screened);
__global__ void k_merge_keys(const uint64_t* surv, const unsigned long long* surv_cnt, uint64_t cap,
                             const int32_t* surv_keys, int32_t* keys);
__global__ void k_keys_to_verdicts(const int32_t* keys, int64_t n, int8_t* fail_t, int8_t* reason);
__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v);
__global__ void k_finalize(const uint64_t* surv, const unsigned long long* surv_cnt, uint64_t cap,
                           const int32_t* surv_keys, uint64_t base, uint64_t* res, uint64_t res_cap,
                           unsigned long long* hist);
constexpr uint64_t kResultPrefix = 4096;  // passing indices returned with the first D2H
}  // namespace atc

using namespace atc;

struct atc_testset_handle {
  TestsetView view{};
  int32_t T = 0, nI = 0, nP = 0;
  std::vector<int64_t> h_ints;  // host copy of the int values
  std::vector<void*> allocations;
  cudaEvent_t ready = nullptr;  // uploads + dirty lists complete (recorded on the copy stream)
  // layout, kept for in-place updates (atc_testsets_update_seeded)
  int cs = 0;                   // the copy stream all of this handle's uploads use
  std::vector<int64_t> lens, off, doff;
  std::vector<int32_t> is_f32;
  uint8_t* meta = nullptr;      // the small arrays (TestsetView points into it)
  size_t meta_bytes = 0, o_ints = 0, o_rlen = 0, o_roff = 0, o_dof = 0, o_isf = 0, o_tok = 0, o_dcnt = 0,
         o_dmax = 0;
  uint8_t* seeded = nullptr;    // seeds, stream positions, final-minus-init entries
  size_t seeded_cap = 0;
  bool needed_only = false;     // seeded with needed_only: region prefixes only
  uint8_t* pin = nullptr;       // pinned staging of the metadata + seeded blocks (async DMA)
  size_t pin_bytes = 0;
};

// Makes `st` wait for the upload of `ts` (no-op once it has completed).
static void ts_wait(const atc_testset_handle* ts, cudaStream_t st) {
  if (ts && ts->ready) cudaStreamWaitEvent(st, ts->ready, 0);
}

// ------------------------------------------------------------ ctx helpers -----
void atc_set_error(atc_ctx* ctx, const char* fmt, ...) {
  if (!ctx) return;
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  ctx->err = buf;
}

bool atc_cuda_ok(atc_ctx* ctx, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  atc_set_error(ctx, "%s: %s", what, cudaGetErrorString(e));
  return false;
}

void* atc_ctx_scratch(atc_ctx* ctx, int slot, size_t bytes) {
  slot += ctx->slot_base;
  if (slot < 0 || slot >= atc_ctx::kSlots) {
    atc_set_error(ctx, "internal: scratch slot %d out of range", slot);
    return nullptr;
  }
  if (ctx->scratch_bytes[slot] >= bytes) return ctx->scratch[slot];
  if (ctx->scratch[slot]) cudaFree(ctx->scratch[slot]);
  ctx->scratch[slot] = nullptr;
  ctx->scratch_bytes[slot] = 0;
  size_t want = std::max(bytes, (size_t)4096);
  if (cudaMalloc(&ctx->scratch[slot], want) != cudaSuccess) return nullptr;
  ctx->scratch_bytes[slot] = want;
  return ctx->scratch[slot];
}

void* atc_ctx_pinned(atc_ctx* ctx, int slot, size_t bytes) {
  if (slot < 0 || slot >= 4) return nullptr;
  if (ctx->pinned_bytes[slot] >= bytes) return ctx->pinned[slot];
  if (ctx->pinned[slot]) cudaFreeHost(ctx->pinned[slot]);
  ctx->pinned[slot] = nullptr;
  ctx->pinned_bytes[slot] = 0;
  if (cudaMallocHost(&ctx->pinned[slot], bytes) != cudaSuccess) return nullptr;
  ctx->pinned_bytes[slot] = bytes;
  return ctx->pinned[slot];
}

// Device-memory pool for test-set uploads: freed blocks are kept per context and
// reused (best fit), so a per-function upload costs no cudaMalloc/cudaFree.
void* atc_pool_alloc(atc_ctx* ctx, size_t bytes) {
  bytes = (bytes + 255) / 256 * 256;
  size_t best = SIZE_MAX, bi = 0;
  for (size_t i = 0; i < ctx->pool_free.size(); ++i)
    if (ctx->pool_free[i].second >= bytes && ctx->pool_free[i].second < best) {
      best = ctx->pool_free[i].second;
      bi = i;
    }
  if (best != SIZE_MAX) {
    auto blk = ctx->pool_free[bi];
    ctx->pool_free.erase(ctx->pool_free.begin() + bi);
    ctx->pool_used[blk.first] = blk.second;
    return blk.first;
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  ctx->pool_used[p] = bytes;
  return p;
}

void atc_pool_free(atc_ctx* ctx, void* p) {
  auto it = ctx->pool_used.find(p);
  if (it == ctx->pool_used.end()) {
    cudaFree(p);
    return;
  }
  ctx->pool_free.emplace_back(p, it->second);
  ctx->pool_used.erase(it);
}

namespace {

bool build_spec_view(atc_ctx* ctx, const atc_spec_desc* s, SpecView& v) {
  if (!s) {
    atc_set_error(ctx, "null spec descriptor");
    return false;
  }
  if ((s->semantics != ATC_SEM_GEMM && s->semantics != ATC_SEM_CONV2D) ||
      (s->layout != ATC_LAYOUT_ROW && s->layout != ATC_LAYOUT_COL) || s->n_arrays != 3 ||
      s->n_sizes < 1 || s->n_sizes > ATC_MAX_SIZES) {
    atc_set_error(ctx, "malformed spec descriptor (semantics %d, layout %d, %d arrays, %d sizes)",
                  s->semantics, s->layout, s->n_arrays, s->n_sizes);
    return false;
  }
  std::memset(&v, 0, sizeof v);
  v.sem = s->semantics;
  v.layout = s->layout;
  v.nA = s->n_arrays;
  v.nS = s->n_sizes;
  int seen[3] = {-1, -1, -1};
  int outputs = 0;
  for (int a = 0; a < v.nA; ++a) {
    int r = s->array_role[a];
    if (r < 0 || r > 2 || seen[r] >= 0) {
      atc_set_error(ctx, "array %d: bad or duplicate role %d", a, r);
      return false;
    }
    seen[r] = a;
    v.role[a] = r;
    if (!s->array_livein[a]) {
      ++outputs;
      if (r != ATC_ROLE_C) {
        atc_set_error(ctx, "only the C/out array may be an output (array %d)", a);
        return false;
      }
    }
    if (s->array_ndims[a] < 1 || s->array_ndims[a] > ATC_MAX_DIMS) {
      atc_set_error(ctx, "array %d: bad dim count %d", a, s->array_ndims[a]);
      return false;
    }
    v.ndims[a] = s->array_ndims[a];
    for (int d = 0; d < v.ndims[a]; ++d) {
      int q = s->array_dims[a][d];
      if (q < 0 || q >= v.nS) {
        atc_set_error(ctx, "array %d dim %d: size index %d out of range", a, d, q);
        return false;
      }
      v.dims[a][d] = q;
    }
  }
  if (outputs != 1) {
    atc_set_error(ctx, "spec must have exactly one non-LiveIn array (has %d)", outputs);
    return false;
  }
  for (int r = 0; r < 3; ++r) v.arr_of_role[r] = seen[r];
  for (int r = 0; r < ATC_SZ_COUNT; ++r) {
    int q = s->role_size[r];
    if (q >= v.nS) {
      atc_set_error(ctx, "role %d: size index %d out of range", r, q);
      return false;
    }
    v.role_size[r] = q;
  }
  if (v.sem == ATC_SEM_GEMM) {
    for (int r : {ATC_SZ_M, ATC_SZ_N, ATC_SZ_K})
      if (v.role_size[r] < 0) {
        // the reference would use 0 (equivalence.cpp:42-44): loops never run
      }
  }
  return true;
}


}  // namespace

extern "C" {

int atc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

atc_ctx* atc_create(int device) {
  auto* ctx = new atc_ctx();
  ctx->device = device;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || device < 0 || device >= n) {
    atc_set_error(ctx, "no CUDA device %d (%s)", device, e == cudaSuccess ? "out of range" : cudaGetErrorString(e));
    ctx->broken = true;
    return ctx;
  }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  ctx->sm_count = prop.multiProcessorCount;
  if (prop.major != 10) {
    atc_set_error(ctx, "device %d is sm_%d%d; this library is built for sm_100a only", device, prop.major,
                  prop.minor);
    ctx->broken = true;
    return ctx;
  }
  cudaSetDevice(device);
  // k_screen_conv_pairs: up to 2^11 row masks + rank / in-extent tables (~40 KB dynamic)
  cudaFuncSetAttribute(k_screen_conv_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  if (!atc_cuda_ok(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate") ||

      !atc_cuda_ok(ctx, cudaEventCreateWithFlags(&ctx->free_ev, cudaEventDisableTiming), "cudaEventCreate") ||
      !atc_cuda_ok(ctx, cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming), "cudaEventCreate"))
    ctx->broken = true;
  for (int k = 0; k < atc_ctx::kSideStreams && !ctx->broken; ++k)
    if (!atc_cuda_ok(ctx, cudaStreamCreateWithFlags(&ctx->side_stream[k], cudaStreamNonBlocking), "cudaStreamCreate") ||
        !atc_cuda_ok(ctx, cudaEventCreateWithFlags(&ctx->join_ev[k], cudaEventDisableTiming), "cudaEventCreate"))
      ctx->broken = true;
  for (auto& cs : ctx->copy_stream)
    if (!ctx->broken && !atc_cuda_ok(ctx, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "cudaStreamCreate"))
      ctx->broken = true;
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (!ctx->broken &&
      (!atc_cuda_ok(ctx, cudaStreamCreateWithPriority(&ctx->conv_stream, cudaStreamNonBlocking, prio_hi),
                    "cudaStreamCreate") ||
       !atc_cuda_ok(ctx, cudaEventCreateWithFlags(&ctx->conv_join_ev, cudaEventDisableTiming), "cudaEventCreate")))
    ctx->broken = true;
  ctx->own_stream = ctx->stream;
  return ctx;
}

void atc_destroy(atc_ctx* ctx) {
  if (!ctx) return;
  if (!ctx->broken) {
    cudaSetDevice(ctx->device);
    for (auto& p : ctx->scratch)
      if (p) cudaFree(p);
    for (auto& b : ctx->pool_free) cudaFree(b.first);
    for (auto& b : ctx->pool_used) cudaFree(b.first);
    for (auto& p : ctx->pinned)
      if (p) cudaFreeHost(p);
    for (auto& e : ctx->prof_screen) cudaEventDestroy(e.first), cudaEventDestroy(e.second);
    for (auto& e : ctx->prof_confirm) cudaEventDestroy(e.first), cudaEventDestroy(e.second);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    for (auto& cs : ctx->copy_stream)
      if (cs) cudaStreamDestroy(cs);
    if (ctx->free_ev) cudaEventDestroy(ctx->free_ev);
    if (ctx->update_ev) cudaEventDestroy(ctx->update_ev);
    for (int k = 0; k < atc_ctx::kSideStreams; ++k) {
      if (ctx->side_stream[k]) cudaStreamDestroy(ctx->side_stream[k]);
      if (ctx->join_ev[k]) cudaEventDestroy(ctx->join_ev[k]);
    }
    if (ctx->conv_stream) cudaStreamDestroy(ctx->conv_stream);
    if (ctx->conv_join_ev) cudaEventDestroy(ctx->conv_join_ev);
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  }
  delete ctx;
}

const char* atc_last_error(const atc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int atc_set_stream(atc_ctx* ctx, void* stream) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  return ATC_OK;
}

static void prof_clear(atc_ctx* ctx) {
  for (auto& e : ctx->prof_screen) cudaEventDestroy(e.first), cudaEventDestroy(e.second);
  for (auto& e : ctx->prof_confirm) cudaEventDestroy(e.first), cudaEventDestroy(e.second);
  ctx->prof_screen.clear();
  ctx->prof_confirm.clear();
  ctx->prof_survivors = ctx->prof_bindings = ctx->prof_kernels = 0;
}

int atc_profile_start(atc_ctx* ctx) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
  cudaSetDevice(ctx->device);
  prof_clear(ctx);
  ctx->prof = true;
  return ATC_OK;
}

int atc_profile_read(atc_ctx* ctx, atc_profile* out) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
  if (!out) return ATC_ERR_ARG;
  cudaSetDevice(ctx->device);
  std::memset(out, 0, sizeof *out);
  for (auto* list : {&ctx->prof_screen, &ctx->prof_confirm}) {
    double ms = 0;
    for (auto& e : *list) {
      if (!atc_cuda_ok(ctx, cudaEventSynchronize(e.second), "profile sync")) return ATC_ERR_CUDA;
      float f = 0;
      cudaEventElapsedTime(&f, e.first, e.second);
      ms += f;
    }
    if (list == &ctx->prof_screen) {
      out->screen_ms = ms;
      out->screen_launches = (int64_t)list->size();
    } else {
      out->confirm_ms = ms;
      out->confirm_launches = (int64_t)list->size();
    }
  }
  out->survivors = ctx->prof_survivors;
  out->bindings = ctx->prof_bindings;
  out->kernels = ctx->prof_kernels;
  prof_clear(ctx);
  ctx->prof = false;
  return ATC_OK;
}

}  // extern "C"

// Fills an allocated handle from full host regions (`ts_full`) or from seeds +
// final-minus-init entries (`sd`, regions generated on the device), on the
// handle's copy stream, and records its ready event.
// needed_only bound of region (t, p): max(U^4 + 2U^2 + 2U + 1, last final-minus-init
// position + 1), U = test t's largest int (include/atc_b200.h), capped at the region
// length; the whole region without needed_only.
static std::vector<int64_t> region_need(const atc_testset_handle* h, const atc_seeded_testsets* sd) {
  const int T = h->T, nI = h->nI, nP = h->nP;
  std::vector<int64_t> need((size_t)T * nP);
  for (int t = 0; t < T; ++t) {
    int64_t u = 1;
    for (int q = 0; q < nI; ++q) u = std::max<int64_t>(u, sd->int_values[(size_t)t * nI + q]);
    const int64_t bound = u > 46340 ? INT64_MAX : u * u * u * u + 2 * u * u + 2 * u + 1;
    for (int p = 0; p < nP; ++p) {
      const size_t i = (size_t)t * nP + p;
      int64_t n = bound;
      for (int64_t e = sd->diff_off[i]; e < sd->diff_off[i + 1]; ++e) n = std::max<int64_t>(n, sd->diff_pos[e] + 1);
      need[i] = sd->needed_only ? std::min<int64_t>(n, h->lens[p]) : h->lens[p];
    }
  }
  return need;
}

// pre (optional, with sd): the caller's own init regions [T*nP] — only their needed
// prefixes are staged and copied, instead of generating them from the seeds.
static int testsets_fill(atc_ctx* ctx, atc_testset_handle* h, const atc_testsets* ts_full,
                         const atc_seeded_testsets* sd, bool sync, bool pinned_staging = false,
                         cudaEvent_t reuse = nullptr, const double* const* pre = nullptr) {
  const int T = h->T, nI = h->nI, nP = h->nP;
  const size_t TP = (size_t)T * nP;
  const int64_t* int_values = ts_full ? ts_full->int_values : sd->int_values;
  const int32_t* test_ok = ts_full ? ts_full->test_ok : sd->test_ok;
  h->h_ints.assign(int_values, int_values + (size_t)T * nI);
  // every small array in one block, built in pinned staging and copied once; the
  // seeded block follows it in the same staging buffer
  const int64_t nd_s = sd ? sd->diff_off[TP] : 0;
  std::vector<int64_t> need = sd ? region_need(h, sd) : std::vector<int64_t>();
  if (pre)  // a failed test has no region: every binding fails there (reason 3), nothing to stage
    for (size_t i = 0; i < TP; ++i)
      if (!pre[i] || (test_ok && !test_ok[i / nP])) need[i] = 0;
  std::vector<int64_t> pre_off(pre ? TP + 1 : 0, 0);
  for (size_t i = 0; pre && i < TP; ++i)
    pre_off[i + 1] = pre_off[i] + need[i];
  const size_t pre_bytes = pre ? ((size_t)pre_off[TP] * 8 + 15) / 16 * 16 + ((TP + 1) * 8 + 15) / 16 * 16 : 0;
  const size_t seeded_need =
      sd ? ((size_t)T * 8 + 15) / 16 * 16 + (TP * 8 + 15) / 16 * 16 + ((TP + 1) * 8 + 15) / 16 * 16 +
               ((size_t)nd_s * 8 + 15) / 16 * 16 + ((size_t)nd_s * 4 + 15) / 16 * 16 + (TP * 8 + 15) / 16 * 16 +
               pre_bytes
         : 0;
  // in-place updates stage through the handle's pinned buffer (true async DMA,
  // allocated once); a first upload stages through pageable memory (the driver
  // copies it before returning) and avoids a pinned allocation per handle
  std::vector<uint8_t> pageable;
  uint8_t* meta = nullptr;
  if (pinned_staging) {
    if (h->ready && !atc_cuda_ok(ctx, cudaEventSynchronize(h->ready), "staging reuse"))  // previous DMA done
      return ATC_ERR_CUDA;
    if (h->pin_bytes < h->meta_bytes + seeded_need) {
      if (h->pin) cudaFreeHost(h->pin);
      h->pin = nullptr;
      h->pin_bytes = 0;
      if (!atc_cuda_ok(ctx, cudaMallocHost(&h->pin, h->meta_bytes + seeded_need), "cudaMallocHost"))
        return ATC_ERR_CUDA;
      h->pin_bytes = h->meta_bytes + seeded_need;
    }
    meta = h->pin;
  } else {
    pageable.resize(h->meta_bytes + seeded_need);
    meta = pageable.data();
  }
  std::memset(meta, 0, h->meta_bytes);
  auto put = [&](size_t o, const void* src, size_t bytes) {
    if (bytes) std::memcpy(meta + o, src, bytes);
  };
  put(h->o_ints, int_values, (size_t)T * nI * 8);
  put(h->o_rlen, h->lens.data(), nP * 8);
  put(h->o_roff, h->off.data(), TP * 8);
  put(h->o_dof, h->doff.data(), TP * 8);
  put(h->o_isf, h->is_f32.data(), nP * 4);
  for (int t = 0; t < T; ++t) {
    const int32_t ok_t = test_ok ? (test_ok[t] ? 1 : 0) : 1;
    put(h->o_tok + t * 4, &ok_t, 4);
  }
  for (size_t i = 0; i < TP; ++i) {
    const int32_t neg = -1;
    put(h->o_dmax + i * 4, &neg, 4);  // dirty counts stay 0
  }
  cudaStream_t st = ctx->copy_stream[h->cs];
  if (ctx->free_pending & (1ull << h->cs)) {  // pool memory freed by earlier handles
    cudaStreamWaitEvent(st, ctx->free_ev, 0);
    ctx->free_pending &= ~(1ull << h->cs);
  }
  if (reuse) cudaStreamWaitEvent(st, reuse, 0);  // in-place update: earlier readers first
  bool ok = atc_cuda_ok(ctx, cudaMemcpyAsync(h->meta, meta, h->meta_bytes, cudaMemcpyHostToDevice, st),
                        "H2D metadata");
  double* init = const_cast<double*>(h->view.init);
  double* fin = const_cast<double*>(h->view.fin);
  bool fused = false;  // dirty lists built by k_probe_regions
  if (ts_full) {
    // host regions that lie back to back in the same order as the device pool are
    // copied as one run (one DMA instead of T*n_ptrs)
    struct Run {
      const double* src = nullptr;
      size_t dst = 0, bytes = 0;
    };
    Run run_i, run_f;
    auto flush = [&](Run& r, double* base, const char* what) {
      if (r.bytes)
        ok = ok && atc_cuda_ok(ctx, cudaMemcpyAsync(base + r.dst, r.src, r.bytes, cudaMemcpyHostToDevice, st), what);
      r = Run{};
    };
    auto add = [&](Run& r, double* base, const double* src, size_t dst, size_t bytes, const char* what) {
      if (r.bytes && r.src + r.bytes / 8 == src && r.dst + r.bytes / 8 == dst && r.bytes % 256 == 0) {
        r.bytes += bytes;
        return;
      }
      flush(r, base, what);
      r.src = src;
      r.dst = dst;
      r.bytes = bytes;
    };
    for (int t = 0; t < T && ok; ++t)
      for (int p = 0; p < nP && ok; ++p) {
        const size_t i = (size_t)t * nP + p;
        const size_t bytes = (size_t)h->lens[p] * 8;
        const double* hi = ts_full->init[i];
        const double* hf = ts_full->final_[i];
        if (!hi || !hf) {
          // a test whose original run failed has no final image; the region stays
          // unused because every binding fails at t (test_ok[t] == 0)
          if (test_ok && test_ok[t]) {
            atc_set_error(ctx, "test %d pointer %d: missing region", t, p);
            ok = false;
          }
          ok = ok && atc_cuda_ok(ctx, cudaMemsetAsync(init + h->off[i], 0, bytes, st), "memset") &&
               atc_cuda_ok(ctx, cudaMemsetAsync(fin + h->off[i], 0, bytes, st), "memset");
          continue;
        }
        add(run_i, init, hi, (size_t)h->off[i], bytes, "H2D init");
        add(run_f, fin, hf, (size_t)h->off[i], bytes, "H2D final");
      }
    flush(run_i, init, "H2D init");
    flush(run_f, fin, "H2D final");
  } else if (ok) {
    // regions from the tests' mt19937_64 streams (k_probe_regions), then the
    // final-minus-init entries scattered into the final images (k_apply_diffs)
    const int64_t nd = sd->diff_off[TP];
    for (int64_t i = 0; ok && i < nd; ++i)
      if (sd->diff_pos[i] < 0) {
        atc_set_error(ctx, "negative final-minus-init position");
        ok = false;
      }
    size_t so = 0;
    auto take = [&](size_t bytes) {
      const size_t o = so;
      so += (bytes + 15) / 16 * 16;
      return o;
    };
    const size_t o_seeds = take((size_t)T * 8), o_skips = take(TP * 8), o_doffs = take((TP + 1) * 8),
                 o_dvs = take((size_t)nd * 8), o_dps = take((size_t)nd * 4), o_need = take(TP * 8);
    const size_t o_pre = pre ? take((size_t)pre_off[TP] * 8) : 0, o_preoff = pre ? take((TP + 1) * 8) : 0;
    h->needed_only = sd->needed_only != 0;
    if (ok && so > h->seeded_cap) {  // grow (the old block stays owned by the handle)
      h->seeded = (uint8_t*)atc_pool_alloc(ctx, std::max(so, (size_t)256));
      if (h->seeded) h->allocations.push_back(h->seeded);
      h->seeded_cap = h->seeded ? so : 0;
      if (!h->seeded) {
        atc_set_error(ctx, "device allocation failed (seeded test sets)");
        ok = false;
      }
    }
    if (ok) {
      uint8_t* sb = meta + h->meta_bytes;  // so == seeded_need
      std::memcpy(sb + o_seeds, sd->stream_seed, (size_t)T * 8);
      std::memcpy(sb + o_skips, sd->stream_skip, TP * 8);
      std::memcpy(sb + o_doffs, sd->diff_off, (TP + 1) * 8);
      if (nd) {
        std::memcpy(sb + o_dvs, sd->diff_val, (size_t)nd * 8);
        std::memcpy(sb + o_dps, sd->diff_pos, (size_t)nd * 4);
      }
      std::memcpy(sb + o_need, need.data(), TP * 8);
      if (pre) {
        for (size_t i = 0; i < TP; ++i)
          if (pre_off[i + 1] > pre_off[i])
            std::memcpy(sb + o_pre + (size_t)pre_off[i] * 8, pre[i], (size_t)(pre_off[i + 1] - pre_off[i]) * 8);
        std::memcpy(sb + o_preoff, pre_off.data(), (TP + 1) * 8);
      }
      ok = atc_cuda_ok(ctx, cudaMemcpyAsync(h->seeded, sb, so, cudaMemcpyHostToDevice, st), "H2D seeds");
    }
    if (ok) {
      const TestsetView& v = h->view;
      // needed_only: one kernel generates the prefixes, applies the diffs and builds
      // the dirty lists; else whole regions, then k_apply_diffs and k_build_dirty
      const int64_t* dn = sd->needed_only ? (const int64_t*)(h->seeded + o_need) : nullptr;
      k_probe_regions<<<T, 160, 0, st>>>(T, nP, (const uint64_t*)(h->seeded + o_seeds),
                                         (const uint64_t*)(h->seeded + o_skips), v.region_len, v.is_f32,
                                         v.region_off, dn, init, fin, v, (const int64_t*)(h->seeded + o_doffs),
                                         (const int32_t*)(h->seeded + o_dps), (const double*)(h->seeded + o_dvs),
                                         pre ? (const double*)(h->seeded + o_pre) : nullptr,
                                         pre ? (const int64_t*)(h->seeded + o_preoff) : nullptr);
      if (!dn)
        k_apply_diffs<<<(unsigned)TP, 256, 0, st>>>(nP, v.region_len, v.region_off,
                                                    (const int64_t*)(h->seeded + o_doffs),
                                                    (const int32_t*)(h->seeded + o_dps),
                                                    (const double*)(h->seeded + o_dvs), fin);
      fused = dn != nullptr;
      ok = atc_cuda_ok(ctx, cudaGetLastError(), "k_probe_regions");
    }
  }
  if (ok) {
    if (!fused) {
      int64_t maxlen = 0;
      for (int p = 0; p < nP; ++p) maxlen = std::max<int64_t>(maxlen, h->lens[p]);
      dim3 grid((unsigned)std::min<int64_t>((maxlen + 255) / 256, 64), (unsigned)(T * nP));
      k_build_dirty<<<grid, 256, 0, st>>>(h->view, const_cast<int32_t*>(h->view.dirty_pos),
                                          const_cast<int32_t*>(h->view.dirty_cnt),
                                          const_cast<int32_t*>(h->view.dirty_max));
    }
    ok = atc_cuda_ok(ctx, cudaGetLastError(), "k_build_dirty") &&
         (h->ready || atc_cuda_ok(ctx, cudaEventCreateWithFlags(&h->ready, cudaEventDisableTiming), "cudaEventCreate")) &&
         atc_cuda_ok(ctx, cudaEventRecord(h->ready, st), "cudaEventRecord") &&
         (!sync || atc_cuda_ok(ctx, cudaEventSynchronize(h->ready), "upload sync"));
  }
  return ok ? ATC_OK : ATC_ERR_CUDA;
}

// Both upload forms: full host regions (`ts`) or seeds + final-minus-init entries
// (`sd`, regions generated on the device); the common header fields are equal.
static int testsets_upload(atc_ctx* ctx, const atc_testsets* ts_full, const atc_seeded_testsets* sd,
                           atc_testset_handle** out, bool sync, const double* const* pre = nullptr) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
  atc_testsets hdr{};
  if (ts_full) hdr = *ts_full;
  if (sd) {
    hdr.n_tests = sd->n_tests;
    hdr.n_ints = sd->n_ints;
    hdr.n_ptrs = sd->n_ptrs;
    hdr.int_values = sd->int_values;
    hdr.ptr_is_f32 = sd->ptr_is_f32;
    hdr.region_len = sd->region_len;
    hdr.test_ok = sd->test_ok;
  }
  const atc_testsets* ts = &hdr;
  if ((!ts_full && !sd) || !out || ts->n_tests < 1 || ts->n_tests > kMaxT || ts->n_ints < 1 ||
      ts->n_ints > kMaxInts || ts->n_ptrs < 1 || ts->n_ptrs > kMaxPtrs || !ts->int_values || !ts->region_len ||
      !ts->ptr_is_f32 || (sd && (!sd->stream_seed || !sd->stream_skip || !sd->diff_off || sd->diff_off[0] != 0))) {
    atc_set_error(ctx, "malformed test sets");
    return ATC_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  const int T = ts->n_tests, nI = ts->n_ints, nP = ts->n_ptrs;
  const size_t TP = (size_t)T * nP;
  auto* h = new atc_testset_handle();
  h->T = T;
  h->nI = nI;
  h->nP = nP;
  h->lens.assign(ts->region_len, ts->region_len + nP);
  h->is_f32.assign(ts->ptr_is_f32, ts->ptr_is_f32 + nP);
  // region pool layout: (t, p) regions back to back, each 32-element aligned
  h->off.resize(TP);
  h->doff.resize(TP);
  int64_t total = 0, dtotal = 0;
  for (int t = 0; t < T; ++t)
    for (int p = 0; p < nP; ++p) {
      int64_t len = ts->region_len[p];
      if (len < 4 || len >= (1LL << 31)) {
        atc_set_error(ctx, "region %d length %lld outside [4, 2^31)", p, (long long)len);
        delete h;
        return ATC_ERR_ARG;
      }
      h->off[(size_t)t * nP + p] = total;
      h->doff[(size_t)t * nP + p] = dtotal;
      total += (len + 31) / 32 * 32;
      dtotal += len;
    }
  size_t mo = 0;
  auto take = [&](size_t bytes) {
    const size_t o = mo;
    mo += (bytes + 15) / 16 * 16;
    return o;
  };
  h->o_ints = take((size_t)T * nI * 8);
  h->o_rlen = take(nP * 8);
  h->o_roff = take(TP * 8);
  h->o_dof = take(TP * 8);
  h->o_isf = take(nP * 4);
  h->o_tok = take(T * 4);
  h->o_dcnt = take(TP * 4);
  h->o_dmax = take(TP * 4);
  h->meta_bytes = mo;
  auto dmalloc = [&](size_t bytes) -> void* {
    void* p = atc_pool_alloc(ctx, std::max(bytes, (size_t)256));
    if (p) h->allocations.push_back(p);
    return p;
  };
  double* init = (double*)dmalloc(total * 8);
  double* fin = (double*)dmalloc(total * 8);
  int32_t* dpos = (int32_t*)dmalloc(dtotal * 4);
  h->meta = (uint8_t*)dmalloc(mo);
  if (!init || !fin || !dpos || !h->meta) {
    atc_set_error(ctx, "cudaMalloc failed for %lld region doubles", (long long)total);
    atc_testsets_free(ctx, h);
    return ATC_ERR_CUDA;
  }
  TestsetView& v = h->view;
  v.T = T;
  v.nI = nI;
  v.nP = nP;
  v.ints = (const int64_t*)(h->meta + h->o_ints);
  v.is_f32 = (const int32_t*)(h->meta + h->o_isf);
  v.region_len = (const int64_t*)(h->meta + h->o_rlen);
  v.test_ok = (const int32_t*)(h->meta + h->o_tok);
  v.init = init;
  v.fin = fin;
  v.region_off = (const int64_t*)(h->meta + h->o_roff);
  v.dirty_pos = dpos;
  v.dirty_off = (const int64_t*)(h->meta + h->o_dof);
  v.dirty_cnt = (const int32_t*)(h->meta + h->o_dcnt);
  v.dirty_max = (const int32_t*)(h->meta + h->o_dmax);
  h->cs = ctx->copy_next;  // round-robin over the copy streams
  ctx->copy_next = (h->cs + 1) % atc_ctx::kCopyStreams;
  const int rc = testsets_fill(ctx, h, ts_full, sd, sync, false, nullptr, pre);
  if (rc) {
    atc_testsets_free(ctx, h);
    return rc;
  }
  *out = h;
  return ATC_OK;
}

extern "C" {

int atc_testsets_upload(atc_ctx* ctx, const atc_testsets* ts, atc_testset_handle** out) {
  return testsets_upload(ctx, ts, nullptr, out, true);
}

int atc_testsets_upload_async(atc_ctx* ctx, const atc_testsets* ts, atc_testset_handle** out) {
  return testsets_upload(ctx, ts, nullptr, out, false);
}

int atc_testsets_upload_seeded(atc_ctx* ctx, const atc_seeded_testsets* ts, atc_testset_handle** out) {
  return testsets_upload(ctx, nullptr, ts, out, false);
}

int atc_testsets_upload_prefix(atc_ctx* ctx, const atc_prefix_testsets* ts, atc_testset_handle** out) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
  if (!ts || !ts->init || !ts->diff_off || ts->n_tests < 1 || ts->n_ptrs < 1 || ts->n_tests > kMaxT ||
      ts->n_ptrs > kMaxPtrs) {
    atc_set_error(ctx, "malformed test sets");
    return ATC_ERR_ARG;
  }
  const size_t TP = (size_t)ts->n_tests * ts->n_ptrs;
  for (size_t i = 0; i < TP; ++i)
    if (!ts->init[i] && (!ts->test_ok || ts->test_ok[i / ts->n_ptrs])) {
      atc_set_error(ctx, "test %d pointer %d: missing region", (int)(i / ts->n_ptrs), (int)(i % ts->n_ptrs));
      return ATC_ERR_ARG;
    }
  // the seeded form's header with unused stream fields: the prefixes replace the generator
  std::vector<uint64_t> zeros(TP, 0);
  atc_seeded_testsets sd{ts->n_tests, ts->n_ints,   ts->n_ptrs,   ts->int_values, ts->ptr_is_f32,
                         ts->region_len, ts->test_ok, zeros.data(), zeros.data(),  ts->diff_off,
                         ts->diff_pos,   ts->diff_val, /*needed_only=*/1};
  return testsets_upload(ctx, nullptr, &sd, out, false, ts->init);
}

static bool update_matches(atc_ctx* ctx, const atc_testset_handle* h, const atc_seeded_testsets* ts) {
  if (!h || !ts || ts->n_tests != h->T || ts->n_ints != h->nI || ts->n_ptrs != h->nP || !ts->int_values ||
      !ts->region_len || !ts->ptr_is_f32 || !ts->stream_seed || !ts->stream_skip || !ts->diff_off ||
      ts->diff_off[0] != 0) {
    atc_set_error(ctx, "atc_testsets_update_seeded: test sets do not match the handle");
    return false;
  }
  for (int p = 0; p < h->nP; ++p)
    if (ts->region_len[p] != h->lens[p] || (ts->ptr_is_f32[p] != 0) != (h->is_f32[p] != 0)) {
      atc_set_error(ctx, "atc_testsets_update_seeded: pointer %d differs from the handle's", p);
      return false;
    }
  return true;
}

int atc_testsets_update_seeded(atc_ctx* ctx, atc_testset_handle* h, const atc_seeded_testsets* ts) {
  return atc_testsets_update_seeded_many(ctx, &h, ts, 1);
}

int atc_testsets_update_seeded_many(atc_ctx* ctx, atc_testset_handle* const* handles, const atc_seeded_testsets* ts,
                                    int32_t n) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
  if (n < 0 || (n > 0 && (!handles || !ts))) {
    atc_set_error(ctx, "bad arguments to atc_testsets_update_seeded_many");
    return ATC_ERR_ARG;
  }
  for (int i = 0; i < n; ++i)
    if (!update_matches(ctx, handles[i], ts + i)) return ATC_ERR_ARG;
  if (n == 0) return ATC_OK;
  cudaSetDevice(ctx->device);
  // the new contents are written after everything queued so far on the compute
  // stream (evaluations of every sweep branch join it) has read the old ones: one
  // event for the whole set of updates
  if (!ctx->update_ev &&
      !atc_cuda_ok(ctx, cudaEventCreateWithFlags(&ctx->update_ev, cudaEventDisableTiming), "cudaEventCreate"))
    return ATC_ERR_CUDA;
  if (!atc_cuda_ok(ctx, cudaEventRecord(ctx->update_ev, ctx->stream), "cudaEventRecord")) return ATC_ERR_CUDA;
  // shared context state first, serially: pool growth of the seeded blocks and the
  // copy streams' waits on earlier frees; then the per-handle work (staging, H2D,
  // generator launch) on up to four host threads when the handles are distinct
  bool distinct = true;
  for (int i = 0; i < n && distinct; ++i) {
    atc_testset_handle* h = handles[i];
    for (int k = 0; k < i; ++k) distinct = distinct && handles[k] != h;
    const size_t TP = (size_t)h->T * h->nP;
    const int64_t nd = ts[i].diff_off[TP];
    const size_t so = ((size_t)h->T * 8 + 15) / 16 * 16 + (TP * 8 + 15) / 16 * 16 + ((TP + 1) * 8 + 15) / 16 * 16 +
                      ((size_t)nd * 8 + 15) / 16 * 16 + ((size_t)nd * 4 + 15) / 16 * 16 + (TP * 8 + 15) / 16 * 16;
    if (so > h->seeded_cap) {
      h->seeded = (uint8_t*)atc_pool_alloc(ctx, std::max(so, (size_t)256));
      if (!h->seeded) {
        h->seeded_cap = 0;
        atc_set_error(ctx, "device allocation failed (seeded test sets)");
        return ATC_ERR_CUDA;
      }
      h->allocations.push_back(h->seeded);
      h->seeded_cap = so;
    }
    if (ctx->free_pending & (1ull << h->cs)) {
      cudaStreamWaitEvent(ctx->copy_stream[h->cs], ctx->free_ev, 0);
      ctx->free_pending &= ~(1ull << h->cs);
    }
  }
  const int workers = distinct ? std::min(n, 4) : 1;
  std::atomic<int> first_rc{ATC_OK};
  auto work = [&](int w) {
    cudaSetDevice(ctx->device);
    for (int i = w; i < n; i += workers) {
      const int rc = testsets_fill(ctx, handles[i], nullptr, ts + i, false, true, ctx->update_ev);
      if (rc) {
        int expected = ATC_OK;
        first_rc.compare_exchange_strong(expected, rc);
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < workers; ++w) pool.emplace_back(work, w);
  work(0);
  for (auto& th : pool) th.join();
  return first_rc.load();
}

int atc_testsets_download(atc_ctx* ctx, const atc_testset_handle* h, double* init, double* final_) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
  if (!h || (!init && !final_)) {
    atc_set_error(ctx, "bad arguments to atc_testsets_download");
    return ATC_ERR_ARG;
  }
  if (h->needed_only) {
    atc_set_error(ctx, "atc_testsets_download: the handle holds only the needed region prefixes");
    return ATC_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  if (h->ready && !atc_cuda_ok(ctx, cudaEventSynchronize(h->ready), "upload wait")) return ATC_ERR_CUDA;
  std::vector<int64_t> off((size_t)h->T * h->nP), len(h->nP);
  if (!atc_cuda_ok(ctx, cudaMemcpy(off.data(), h->view.region_off, off.size() * 8, cudaMemcpyDeviceToHost), "D2H") ||
      !atc_cuda_ok(ctx, cudaMemcpy(len.data(), h->view.region_len, len.size() * 8, cudaMemcpyDeviceToHost), "D2H"))
    return ATC_ERR_CUDA;
  size_t o = 0;  // host layout: (t, p) regions back to back, unpadded
  for (int t = 0; t < h->T; ++t)
    for (int p = 0; p < h->nP; ++p) {
      const size_t i = (size_t)t * h->nP + p, bytes = (size_t)len[p] * 8;
      if ((init && !atc_cuda_ok(ctx, cudaMemcpy(init + o, h->view.init + off[i], bytes, cudaMemcpyDeviceToHost), "D2H")) ||
          (final_ && !atc_cuda_ok(ctx, cudaMemcpy(final_ + o, h->view.fin + off[i], bytes, cudaMemcpyDeviceToHost), "D2H")))
        return ATC_ERR_CUDA;
      o += (size_t)len[p];
    }
  return ATC_OK;
}

int atc_testsets_free(atc_ctx* ctx, atc_testset_handle* h) {
  if (!h) return ATC_OK;
  if (ctx && !ctx->broken) {
    cudaSetDevice(ctx->device);
    // the memory returns to the pool: later uploads wait until the compute
    // stream has passed this point (and this handle's own copies are done)
    ts_wait(h, ctx->stream);
    cudaEventRecord(ctx->free_ev, ctx->stream);
    ctx->free_pending = (atc_ctx::kCopyStreams >= 64) ? ~0ull : (1ull << atc_ctx::kCopyStreams) - 1;
  }
  if (h->ready) {
    cudaEventSynchronize(h->ready);  // the staging buffer may still be read by its DMA
    cudaEventDestroy(h->ready);
  }
  if (h->pin) cudaFreeHost(h->pin);
  for (void* p : h->allocations) {
    if (ctx && !ctx->broken)
      atc_pool_free(ctx, p);
    else
      cudaFree(p);
  }
  delete h;
  return ATC_OK;
}

}  // extern "C"

namespace {

constexpr int kScreenThreads = 256;

int screen_budget(const SpecView& sp) { return sp.sem == ATC_SEM_GEMM ? 16 : 2; }

// Preconditions of k_screen_conv_planes (screen_rows.cu): the bundled conv2d
// shape — roles tc_n..tc_ow on size params 0..8, dims in=(n,c,h,w),
// weights=(c,k,r,s), out=(n,k,oh,ow) in any order, in/weights/out = arrays
// 0/1/2, a table key free of digit 0, nI <= 32.  ATC_SCREEN_GENERIC=1 forces
// the generic k_screen_rows (A/B checks).
// ATC_SCREEN_PLANES=1: k_screen_conv_planes instead of k_screen_conv_pairs (A/B checks)
bool pairs_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("ATC_SCREEN_PLANES");
    return e && e[0] == '1';
  }();
  return off;
}

// 32-bit index arithmetic when every t=0 size is <= 200 (any product of 4 sizes < 2^31)
bool ts_i32(const atc_testset_handle* ts) {
  int64_t umax = 0;
  for (int i = 0; i < ts->nI; ++i) umax = std::max<int64_t>(umax, std::llabs(ts->h_ints[i]));
  return umax <= 200;
}

bool conv_thresholds_ok(const SpecView& sp, const RowPlan& plan, int nI) {
  static const bool generic = [] {
    const char* e = std::getenv("ATC_SCREEN_GENERIC");
    return e && e[0] == '1';
  }();
  if (generic || sp.sem != ATC_SEM_CONV2D || sp.nS != 9 || sp.nA != 3 || nI > kMaxInts) return false;
  for (int i = 0; i < 9; ++i)
    if (plan.role_q[ATC_SZ_CN + i] != i) return false;
  if (plan.dim_mask[0] != 0xFu || plan.dim_mask[1] != 0x72u || plan.dim_mask[2] != 0x191u) return false;
  if (sp.arr_of_role[0] != 0 || sp.arr_of_role[1] != 1 || sp.arr_of_role[2] != 2) return false;
  return plan.key_stride[0] == 0;
}

// Runs K1 + K2 over `n` bindings; survivors/keys live in ctx scratch.
int run_eval(atc_ctx* ctx, const SpecView& sp, const atc_testset_handle* ts, const BindingSource& src,
             uint64_t n, int32_t* keys, uint64_t* surv, uint64_t surv_cap, unsigned long long* surv_cnt,
             int32_t* surv_keys, unsigned long long* hist, cudaStream_t st, const Pos0Table* pt = nullptr,
             const RowPlan* plan = nullptr) {
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
                          ((size_t)ts->nP * nI2 + 15) / 16 * 16 + nI2 * sizeof(float);
      // one wave (3 CTAs per SM at 80 registers): each CTA builds its tables once
      const unsigned g3 = std::min<unsigned>(g2, (unsigned)ctx->sm_count * 4);
      k_screen_conv_pairs<<<g3, kScreenThreads, smem, st>>>(ts->view, src.perms, src.size_maps, b, e, *plan, surv,
                                                            surv_cap, surv_cnt, hist, lut_n);
    } else if (i32 && conv_thresholds_ok(sp, *plan, ts->nI)) {
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
  const uint64_t k2_cap = sp.sem == ATC_SEM_GEMM ? 64 : (uint64_t)ctx->sm_count * 8;
  const unsigned g_t0 = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((max_surv + 7) / 8, k2_cap));
  const unsigned g_t1 = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>((max_surv * (uint64_t)std::max(ts->T - 1, 0) + 7) / 8, k2_cap));
  const bool pre = sp.sem == ATC_SEM_CONV2D;
  const int screened = plan && plan->cmask && src.enumerated ? 1 : 0;  // pair-screened conv space
  if (pre)
    k_confirm_pre<<<(unsigned)std::max<uint64_t>(1, std::min<uint64_t>((max_surv + 255) / 256, ctx->sm_count * 8)),
                    256, 0, st>>>(ts->view, sp, src, surv, surv_cnt, surv_cap, surv_keys, pend, next_cnt + 1,
                                  ctx->mode, screened);
  if (pre && !keys) {
    // enumerated ranges report reasons, not failing tests: t >= 1 first over every
    // pending survivor, then t = 0 only where it can change the reason (k_confirm_t0)
    k_confirm_warp<<<g_t1, 256, 0, st>>>(ts->view, sp, src, surv, surv_cap, surv_keys, pend, next_cnt + 1,
                                         ctx->mode, screened);
    const unsigned g_lazy = (unsigned)std::min<uint64_t>((uint64_t)g_t0 * 8, k2_cap);  // 8 warps per binding
    k_confirm_t0<<<g_lazy, 256, 0, st>>>(ts->view, sp, src, surv, surv_cnt, surv_cap, surv_keys, pend, next_cnt + 1,
                                         next, next_cnt, ctx->mode, 1, screened);
  } else {
    k_confirm_t0<<<g_t0, 256, 0, st>>>(ts->view, sp, src, surv, surv_cnt, surv_cap, surv_keys,
                                       pre ? pend : nullptr, next_cnt + 1, next, next_cnt, ctx->mode, 0, screened);
    k_confirm_warp<<<g_t1, 256, 0, st>>>(ts->view, sp, src, surv, surv_cap, surv_keys, next, next_cnt, ctx->mode,
                                         screened);
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

}  // namespace

extern "C" {

int atc_eval_bindings_device(atc_ctx* ctx, const atc_spec_desc* spec, const atc_testset_handle* ts,
                             const uint8_t* d_arr_map, const uint8_t* d_size_map, int64_t n_bindings,
                             int32_t mode, int8_t* d_fail_t, int8_t* d_reason, void* stream) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
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
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
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
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
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

namespace {

// ---- enumerated spaces --------------------------------------------------------
// Per-space plan: the decode, the position-0 table shape and the row plan.
struct EnumPlan {
  SpecView sp;
  Pos0Table pt;
  RowPlan plan;
  bool use_table = false, use_rows = false;
  uint64_t size_maps = 1, table_bytes = 0;
};

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
    const bool pairs = e.use_rows && ts_i32(ts) && conv_thresholds_ok(sp, e.plan, ts->nI) && ts->nI <= 11 &&
                       e.plan.key_stride[1] == 1 && !pairs_disabled();
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
    if (sp.sem == ATC_SEM_CONV2D && e.pt.R == 5 && e.plan.key_stride[1] == 1 && e.use_rows &&
        conv_thresholds_ok(sp, e.plan, ts->nI)) {
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
      k_pos0_table_conv<<<grid, 256, (size_t)(sa + sb) * sizeof(double), st>>>(
          ts->view, sp, perms_local, (int)np_local, e.pt, tab + t_off, tab1 ? tab1 + t_off : nullptr,
          cm ? cm + w_off : nullptr, sa, sb);
      if (ctx->prof) ctx->prof_kernels += 1;
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

constexpr uint64_t kEnumChunkCap = 1ull << 22;  // survivors per K1 launch

}  // namespace

extern "C" {

int atc_eval_enumerated(atc_ctx* ctx, const atc_spec_desc* spec, const atc_testset_handle* ts,
                        const uint8_t* perms, int32_t n_perms, uint64_t begin, uint64_t end, int32_t mode,
                        uint64_t* survivors, int64_t cap, int64_t* n_survivors, int64_t* reason_counts) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
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

// A prepared sweep (atc_enum_batch_*): per-job plans, device-resident
// permutations, a result block per job; replayed as one CUDA graph after the
// first (eager) run has sized every scratch buffer.
struct atc_enum_batch {
  atc_enum_job* jobs = nullptr;
  int n = 0, mode = 0, runs = 0;
  std::vector<EnumPlan> plans;
  std::vector<uint8_t*> d_perms;
  std::vector<char> batched;
  uint64_t* res = nullptr;    // device: n blocks of kBatchStride, then n x 8 histogram words
  uint64_t* h_res = nullptr;  // pinned mirror
  cudaGraphExec_t exec = nullptr;
  bool graph_failed = false;
  std::vector<std::vector<int64_t>> captured_ints;  // per job: its test sets' ints when the graph was captured
  bool transient = false;  // one-shot (atc_eval_enumerated_many): buffers borrowed from the context
  uint8_t* perm_block = nullptr;  // owned permutation buffer (reusable batches)
};

namespace {

// per job of a batch: count, passing count, passing prefix (a job with more passing
// bindings than the prefix is redone alone by atc_eval_enumerated); small, because
// the whole block comes back every run
constexpr uint64_t kBatchPrefix = 256;
constexpr uint64_t kBatchStride = 2 + kBatchPrefix;

size_t batch_res_words(int n) { return (size_t)n * (kBatchStride + 8); }

// Concurrent branches: conv spaces (large K1 launches) on the caller's stream,
// gemm spaces (chains of small latency-bound kernels) round-robin on the side
// streams with their own scratch (slot + 32 * (k + 1)); they fork from and join
// back into `st`, so a captured graph has the same branches.
int enqueue_batch(atc_ctx* ctx, atc_enum_batch* b, cudaStream_t st, bool wait_uploads) {
  const uint64_t chunk_cap = kEnumChunkCap;
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(b->res + (size_t)b->n * kBatchStride);
  cudaMemsetAsync(b->res, 0, batch_res_words(b->n) * 8, st);
  int n_side = 0;
  // jobs with an empty range (a multi-GPU rank's share of nothing) take no stream,
  // event wait or graph node at all
  auto active = [&](int j) { return b->batched[j] && b->jobs[j].end > b->jobs[j].begin; };
  int n_active = 0;
  for (int j = 0; j < b->n; ++j) {
    n_active += active(j);
    n_side += active(j) && b->plans[j].sp.sem != ATC_SEM_CONV2D;
  }
  const bool split = n_side > 1 || (n_side == 1 && n_side < n_active);
  if (split) {
    cudaEventRecord(ctx->fork_ev, st);
    for (int k = 0; k < atc_ctx::kSideStreams; ++k) cudaStreamWaitEvent(ctx->side_stream[k], ctx->fork_ev, 0);
    cudaStreamWaitEvent(ctx->conv_stream, ctx->fork_ev, 0);
  }
  int side_next = 0, conv_next = 0;
  int rc = ATC_OK;
  for (int j = 0; j < b->n && rc == ATC_OK; ++j) {
    if (!active(j)) continue;
    atc_enum_job& job = b->jobs[j];
    EnumPlan& e = b->plans[j];
    // conv spaces on the caller's stream and side stream 0 alternately when they
    // are small (a multi-GPU rank's share: chains of short kernels), else the
    // caller's stream; gemm spaces round-robin over the side streams
    int sk = -1;
    if (split && e.sp.sem == ATC_SEM_CONV2D) {
      if (job.end - job.begin < (1ull << 30)) {
        sk = conv_next ? 0 : -1;
        conv_next ^= 1;
      }
    } else if (split) {
      sk = side_next;
      side_next = (side_next + 1) % atc_ctx::kSideStreams;
    }
    const bool side = sk >= 0;
    cudaStream_t js = side ? ctx->side_stream[sk] : split ? ctx->conv_stream : st;
    ctx->slot_base = side ? 32 * (sk + 1) : 0;
    uint64_t* surv = (uint64_t*)atc_ctx_scratch(ctx, 1, chunk_cap * 8);
    int32_t* skeys = (int32_t*)atc_ctx_scratch(ctx, 2, chunk_cap * 4);
    unsigned long long* cnt = (unsigned long long*)atc_ctx_scratch(ctx, 3, 64);
    if (!surv || !skeys || !cnt) {
      atc_set_error(ctx, "scratch allocation failed");
      rc = ATC_ERR_CUDA;
      break;
    }
    // job j starts as soon as its own test sets are resident; in a captured graph the
    // wait is an external event node on the handle's ready event, so a replay after
    // an in-place update (atc_testsets_update_seeded) waits for that update only
    if (wait_uploads)
      ts_wait(job.ts, js);
    else if (job.ts->ready)
      cudaStreamWaitEvent(js, job.ts->ready, cudaEventWaitExternal);
    rc = enqueue_tables(ctx, e, job.ts, job.perms, job.n_perms, &b->d_perms[j], js, job.begin, job.end);
    if (rc) break;
    if (job.end > job.begin) {
      BindingSource src{nullptr, nullptr, b->d_perms[j], e.size_maps, job.begin, 1};
      rc = run_eval(ctx, e.sp, job.ts, src, job.end - job.begin, nullptr, surv, chunk_cap, cnt, skeys,
                    hist + 8 * j, js, e.use_table ? &e.pt : nullptr, e.use_rows ? &e.plan : nullptr);
      if (rc) break;
      k_finalize<<<64, 256, 0, js>>>(surv, cnt, chunk_cap, skeys, job.begin, b->res + (size_t)j * kBatchStride,
                                     kBatchPrefix, hist + 8 * j);
      if (ctx->prof) ctx->prof_kernels += 1;
    }
  }
  ctx->slot_base = 0;
  if (split) {
    for (int k = 0; k < atc_ctx::kSideStreams; ++k) {
      cudaEventRecord(ctx->join_ev[k], ctx->side_stream[k]);
      cudaStreamWaitEvent(st, ctx->join_ev[k], 0);
    }
    cudaEventRecord(ctx->conv_join_ev, ctx->conv_stream);
    cudaStreamWaitEvent(st, ctx->conv_join_ev, 0);
  }
  if (rc) return rc;
  if (!atc_cuda_ok(ctx, cudaMemcpyAsync(b->h_res, b->res, batch_res_words(b->n) * 8, cudaMemcpyDeviceToHost, st),
                   "D2H results"))
    return ATC_ERR_CUDA;
  return atc_cuda_ok(ctx, cudaGetLastError(), "batch launch") ? ATC_OK : ATC_ERR_CUDA;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

atc_enum_batch* batch_create(atc_ctx* ctx, atc_enum_job* jobs, int32_t n_jobs, int32_t mode, bool transient) {
  if (!ctx || ctx->broken) return nullptr;
  if (n_jobs < 0 || (n_jobs > 0 && !jobs) || (mode != ATC_MODE_FP64 && mode != ATC_MODE_FP32_SCREEN)) {
    atc_set_error(ctx, "bad arguments to atc_enum_batch_create");
    return nullptr;
  }
  cudaSetDevice(ctx->device);
  auto* b = new atc_enum_batch;
  b->jobs = jobs;
  b->n = n_jobs;
  b->mode = mode;
  b->transient = transient;
  b->plans.resize(n_jobs);
  b->d_perms.assign(n_jobs, nullptr);
  b->batched.assign(n_jobs, 0);
  std::vector<size_t> off(n_jobs, 0);
  size_t total = 0;
  for (int j = 0; j < n_jobs; ++j) {
    atc_enum_job& job = jobs[j];
    job.status = plan_enumerated(ctx, job.spec, job.ts, job.perms, job.n_perms, job.begin, job.end, mode,
                                 b->plans[j]);
    if (job.status != ATC_OK || job.end - job.begin > (1ull << 34)) continue;  // errors / chunked: not batched
    off[j] = total;
    total += ((size_t)job.n_perms * b->plans[j].sp.nA + 15) / 16 * 16;
    b->batched[j] = 1;
  }
  // every job's permutations in one device buffer (the context's slot 6 for a
  // one-shot batch, an owned allocation for a reusable one)
  uint8_t* perms = nullptr;
  const size_t words = batch_res_words(n_jobs > 0 ? n_jobs : 1);
  bool ok = true;
  if (transient) {
    perms = (uint8_t*)atc_ctx_scratch(ctx, 6, total + 16);
    b->res = (uint64_t*)atc_ctx_scratch(ctx, 22, words * 8);
    b->h_res = (uint64_t*)atc_ctx_pinned(ctx, 1, words * 8);
    ok = perms && b->res && b->h_res;
  } else {
    ok = cudaMalloc(&perms, total + 16) == cudaSuccess && cudaMalloc(&b->res, words * 8) == cudaSuccess &&
         cudaMallocHost(&b->h_res, words * 8) == cudaSuccess;
    b->perm_block = perms;
  }
  if (!ok) {
    atc_set_error(ctx, "batch allocation failed");
    atc_enum_batch_destroy(ctx, b);
    return nullptr;
  }
  for (int j = 0; j < n_jobs; ++j) {
    if (!b->batched[j]) continue;
    b->d_perms[j] = perms + off[j];
    cudaMemcpyAsync(b->d_perms[j], jobs[j].perms, (size_t)jobs[j].n_perms * b->plans[j].sp.nA,
                    cudaMemcpyHostToDevice, ctx->stream);
  }
  return b;
}

}  // namespace

extern "C" {

atc_enum_batch* atc_enum_batch_create(atc_ctx* ctx, atc_enum_job* jobs, int32_t n_jobs, int32_t mode) {
  atc_enum_batch* b = batch_create(ctx, jobs, n_jobs, mode, false);
  if (b)
    for (int j = 0; j < n_jobs; ++j) ts_wait(jobs[j].ts, ctx->stream);
  if (b && !atc_cuda_ok(ctx, cudaStreamSynchronize(ctx->stream), "batch upload")) {
    atc_enum_batch_destroy(ctx, b);
    return nullptr;
  }
  return b;
}

void atc_enum_batch_destroy(atc_ctx* ctx, atc_enum_batch* b) {
  if (!b) return;
  if (ctx) cudaSetDevice(ctx->device);
  if (b->exec) cudaGraphExecDestroy(b->exec);
  if (!b->transient) {
    if (b->perm_block) cudaFree(b->perm_block);
    if (b->res) cudaFree(b->res);
    if (b->h_res) cudaFreeHost(b->h_res);
  }
  delete b;
}

int atc_enum_batch_run(atc_ctx* ctx, atc_enum_batch* b) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
  if (!b) {
    atc_set_error(ctx, "null batch");
    return ATC_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  ctx->mode = b->mode;
  for (int j = 0; j < b->n; ++j) {
    atc_enum_job& job = b->jobs[j];
    if (job.status != ATC_OK && b->batched[j]) job.status = ATC_OK;
    job.n_survivors = 0;
    for (int r = 0; r < ATC_REASON_COUNT; ++r) job.reason_counts[r] = 0;
  }
  // eager on the first run (sizes the scratch) and whenever profiling; a graph
  // replay afterwards (one launch for the whole sweep)
  int rc = ATC_OK;
  if (b->runs == 0 || ctx->prof || b->graph_failed) {
    rc = enqueue_batch(ctx, b, st, true);
  } else {
    // the graph bakes in choices made from the test sets' ints (index width, tables,
    // kernels): re-capture if an in-place update changed any of them
    bool stale = false;
    for (int j = 0; j < b->n && b->exec && !stale; ++j)
      stale = b->batched[j] && (size_t)j < b->captured_ints.size() && b->captured_ints[j] != b->jobs[j].ts->h_ints;
    if (stale) {
      cudaGraphExecDestroy(b->exec);
      b->exec = nullptr;
    }
    if (!b->exec) {
      b->captured_ints.assign(b->n, {});
      for (int j = 0; j < b->n; ++j)
        if (b->batched[j]) b->captured_ints[j] = b->jobs[j].ts->h_ints;
      cudaGraph_t g = nullptr;
      bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed) == cudaSuccess;
      if (ok) {
        const int erc = enqueue_batch(ctx, b, st, false);  // uploads completed at create
        ok = cudaStreamEndCapture(st, &g) == cudaSuccess && erc == ATC_OK;
        ok = ok && cudaGraphInstantiate(&b->exec, g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
      }
      if (!ok) {
        cudaGetLastError();
        b->exec = nullptr;
        b->graph_failed = true;
      }
    }
    rc = b->exec ? (atc_cuda_ok(ctx, cudaGraphLaunch(b->exec, st), "batch graph launch") ? ATC_OK : ATC_ERR_CUDA)
                 : enqueue_batch(ctx, b, st, true);
  }
  if (rc) return rc;
  if (!atc_cuda_ok(ctx, cudaStreamSynchronize(st), "batch sync")) return ATC_ERR_CUDA;
  ++b->runs;
  const uint64_t* h_hist = b->h_res + (size_t)b->n * kBatchStride;
  for (int j = 0; j < b->n; ++j) {
    atc_enum_job& job = b->jobs[j];
    if (job.status != ATC_OK) continue;
    const uint64_t* rj = b->h_res + (size_t)j * kBatchStride;
    const uint64_t c = rj[0], npass = rj[1];
    if (!b->batched[j] || c > kEnumChunkCap || npass > kBatchPrefix) {
      // overflow (or a very large range): the single-space path with its own chunking
      job.status = atc_eval_enumerated(ctx, job.spec, job.ts, job.perms, job.n_perms, job.begin, job.end, b->mode,
                                       job.survivors, job.cap, &job.n_survivors, job.reason_counts);
      continue;
    }
    if (ctx->prof) ctx->prof_survivors += (long long)c;
    std::vector<uint64_t> pass(rj + 2, rj + 2 + npass);
    std::sort(pass.begin(), pass.end());
    for (size_t i = 0; i < pass.size() && (int64_t)i < job.cap; ++i)
      if (job.survivors) job.survivors[i] = pass[i];
    job.n_survivors = (int64_t)npass;
    for (int r = 0; r < ATC_REASON_COUNT; ++r) job.reason_counts[r] = job.end > job.begin ? (int64_t)h_hist[8 * j + r] : 0;
    job.reason_counts[ATC_PASS] = (int64_t)npass;
  }
  return ATC_OK;
}

int atc_eval_enumerated_many(atc_ctx* ctx, atc_enum_job* jobs, int32_t n_jobs, int32_t mode) {
  if (!ctx || ctx->broken) return ATC_ERR_DEVICE;
  if (n_jobs == 0) return ATC_OK;
  atc_enum_batch* b = batch_create(ctx, jobs, n_jobs, mode, true);
  if (!b) return ATC_ERR_ARG;
  const int rc = atc_enum_batch_run(ctx, b);
  atc_enum_batch_destroy(ctx, b);
  return rc;
}

}  // extern "C"
