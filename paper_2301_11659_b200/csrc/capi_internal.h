// Internal context shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include <map>
#include <string>
#include <utility>
#include <vector>

struct atc_ctx {
  int device = 0;
  int sm_count = 148;
  bool broken = false;
  std::string err;
  cudaStream_t stream = nullptr;
  // reusable device scratch, grown on demand (slot ids are per call site)
  // sweeps run conv spaces on the caller's stream and gemm spaces round-robin on
  // kSideStreams concurrent side streams; side stream k's evaluator scratch lives
  // at slot + 32 * (k + 1) (set while enqueueing it)
  static constexpr int kSideStreams = 4;
  static constexpr int kSlots = 32 * (kSideStreams + 1);
  int slot_base = 0;
  cudaStream_t side_stream[kSideStreams] = {};
  cudaEvent_t fork_ev = nullptr, join_ev[kSideStreams] = {};
  // conv spaces of a split batch (the critical path) run on a highest-priority
  // stream, so their CTAs are dispatched ahead of the gemm branches'
  cudaStream_t conv_stream = nullptr;
  cudaEvent_t conv_join_ev = nullptr;
  void* scratch[kSlots] = {};
  size_t scratch_bytes[kSlots] = {};
  void* pinned[4] = {};
  size_t pinned_bytes[4] = {};
  cudaStream_t own_stream = nullptr;
  // test-set uploads run on their own stream (copy engine) and publish a ready
  // event per handle; frees record free_ev on the compute stream, which the
  // next upload waits on before reusing pool memory
  static constexpr int kCopyStreams = 48;  // uploads round-robin over these (concurrent generators)
  cudaStream_t copy_stream[kCopyStreams] = {};
  int copy_next = 0;
  cudaEvent_t free_ev = nullptr;
  cudaEvent_t update_ev = nullptr;  // in-place updates wait for earlier readers (compute stream)
  uint64_t free_pending = 0;  // copy streams that have not waited on the latest free (bit per stream)
  int mode = 0;  // ATC_MODE_* of the evaluation in flight
  // instrumentation (atc_profile_*)
  bool prof = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_screen, prof_confirm;
  long long prof_survivors = 0, prof_bindings = 0, prof_kernels = 0;
  // device-memory pool for test-set uploads (atc_pool_alloc / atc_pool_free)
  std::vector<std::pair<void*, size_t>> pool_free;
  std::map<void*, size_t> pool_used;
};

void* atc_pool_alloc(atc_ctx* ctx, size_t bytes);
void atc_pool_free(atc_ctx* ctx, void* p);

void atc_set_error(atc_ctx* ctx, const char* fmt, ...);
bool atc_cuda_ok(atc_ctx* ctx, cudaError_t e, const char* what);
void* atc_ctx_scratch(atc_ctx* ctx, int slot, size_t bytes);
void* atc_ctx_pinned(atc_ctx* ctx, int slot, size_t bytes);
