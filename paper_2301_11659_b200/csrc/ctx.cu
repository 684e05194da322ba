// C ABI (include/atc_b200.h): contexts, errors, scratch and pools, options, profiling.
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

// ------------------------------------------------------------ ctx helpers -----
void atc_set_error(atc_ctx* ctx, const char* fmt, ...) {
  if (!ctx) return;
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  std::lock_guard<std::mutex> lk(ctx->err_mu);
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

namespace atc {

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

}  // namespace atc

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
  if (!atc_cuda_ok(ctx, cudaFuncSetAttribute(k_screen_conv_pairs<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024),
                   "cudaFuncSetAttribute(k_screen_conv_pairs)") ||
      !atc_cuda_ok(ctx, cudaFuncSetAttribute(k_screen_conv_pairs<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024),
                   "cudaFuncSetAttribute(k_screen_conv_pairs)") ||
      !atc_cuda_ok(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate") ||

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
    if (ctx->upd_h2d_ev) cudaEventSynchronize(ctx->upd_h2d_ev), cudaEventDestroy(ctx->upd_h2d_ev);
    if (ctx->upd_meta_ev) cudaEventDestroy(ctx->upd_meta_ev);
    for (auto& e : ctx->upd_done_ev)
      if (e) cudaEventDestroy(e);
    if (ctx->upd_pin) cudaFreeHost(ctx->upd_pin);
    if (ctx->upd_dev) cudaFree(ctx->upd_dev);
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

int atc_set_option(atc_ctx* ctx, int32_t option, int32_t value) {
  ATC_ENTER(ctx);
  if (option == ATC_OPT_CONV_SCREEN && value >= ATC_CONV_SCREEN_AUTO && value <= ATC_CONV_SCREEN_GENERIC) {
    ctx->opt_conv_screen = value;
    return ATC_OK;
  }
  if (option == ATC_OPT_SMALL_LOG2 && value >= 0 && value <= 30) {
    ctx->opt_small_log2 = value;
    return ATC_OK;
  }
  if (option == ATC_OPT_K2B_PARTS && (value == 1 || value == 2 || value == 4 || value == 8)) {
    ctx->opt_k2b_parts = value;
    return ATC_OK;
  }
  if (option == ATC_OPT_CONV_STREAMS && value >= 1 && value <= atc_ctx::kSideStreams - 2) {
    ctx->opt_conv_streams = value;
    return ATC_OK;
  }
  if (option == ATC_OPT_TC_FLAGS && value >= 0 && value < 256) {
    ctx->opt_tc_flags = value;
    return ATC_OK;
  }
  atc_set_error(ctx, "atc_set_option: bad option %d / value %d", option, value);
  return ATC_ERR_ARG;
}

int atc_set_stream(atc_ctx* ctx, void* stream) {
  ATC_ENTER(ctx);
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
  ATC_ENTER(ctx);
  cudaSetDevice(ctx->device);
  prof_clear(ctx);
  ctx->prof = true;
  return ATC_OK;
}

int atc_profile_read(atc_ctx* ctx, atc_profile* out) {
  ATC_ENTER(ctx);
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
