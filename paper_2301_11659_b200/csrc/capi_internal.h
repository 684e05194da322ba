// Internal context and declarations shared by the C-ABI translation units
// (ctx.cu, testsets.cu, evaluate.cu, sweep.cu, group.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "atc_b200.h"
#include "eval_common.cuh"

struct atc_ctx {
  int device = 0;
  int sm_count = 148;
  bool broken = false;
  std::string err;
  cudaStream_t stream = nullptr;
  // reusable device scratch, grown on demand (slot ids are per call site)
  // sweeps run conv spaces on the caller's stream and gemm spaces round-robin on
  // kSideStreams concurrent side streams; side stream k's evaluator scratch lives
  // at slot + kSlotsPerStream * (k + 1) (set while enqueueing it)
  static constexpr int kSideStreams = 10;
  static constexpr int kSlotsPerStream = 40;  // evaluator scratch slots per (side) stream
  static constexpr int kSlots = kSlotsPerStream * (kSideStreams + 1);
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
  // batched seeded updates (atc_testsets_update_seeded_many): pinned + device staging
  uint8_t* upd_pin = nullptr;
  uint8_t* upd_dev = nullptr;
  size_t upd_cap = 0;
  cudaEvent_t upd_h2d_ev = nullptr, upd_meta_ev = nullptr, upd_done_ev[kCopyStreams] = {};
  uint64_t free_pending = 0;  // copy streams that have not waited on the latest free (bit per stream)
  int mode = 0;  // ATC_MODE_* of the evaluation in flight
  // instrumentation (atc_profile_*)
  bool prof = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_screen, prof_confirm;
  long long prof_survivors = 0, prof_bindings = 0, prof_kernels = 0;
  // device-memory pool for test-set uploads (atc_pool_alloc / atc_pool_free)
  std::vector<std::pair<void*, size_t>> pool_free;
  std::map<void*, size_t> pool_used;
  // per-context options (atc_set_option): kernel-variant selection for A/B checks
  int opt_conv_screen = ATC_CONV_SCREEN_AUTO;
  int opt_tc_flags = 0;
  int opt_small_log2 = 16;   // gemm spaces of <= 2^this bindings go to k_sweep_small (0: none;
                             // tools/small_threshold.py: 16 keeps config 4's 279,936 on its chain)
  int opt_conv_streams = 8;  // streams the conv chains of a sweep round-robin over (tools/sweep_streams.py)
  int opt_k2b_parts = 1;     // warps per (binding, t) item of the conv K2b (k_confirm_warp)
  bool tc_configured = false;  // k_tc_gemm* shared-memory attributes set on this context's device
  // every ABI entry point holds this for its whole call, so a context is
  // serialised (the pipeline's worker threads may share one)
  std::recursive_mutex mu;
  std::mutex err_mu;  // host worker threads of one call may report errors concurrently
};

void* atc_pool_alloc(atc_ctx* ctx, size_t bytes);
void atc_pool_free(atc_ctx* ctx, void* p);

void atc_set_error(atc_ctx* ctx, const char* fmt, ...);
bool atc_cuda_ok(atc_ctx* ctx, cudaError_t e, const char* what);
void* atc_ctx_scratch(atc_ctx* ctx, int slot, size_t bytes);
void* atc_ctx_pinned(atc_ctx* ctx, int slot, size_t bytes);

// Holds the context's lock for one ABI call; fails (returns false) on a null or
// broken context.
struct AtcLock {
  std::unique_lock<std::recursive_mutex> lk;
  explicit AtcLock(atc_ctx* ctx) {
    if (ctx) lk = std::unique_lock<std::recursive_mutex>(ctx->mu);
  }
};
#define ATC_ENTER(ctx)                          \
  if (!(ctx) || (ctx)->broken) return ATC_ERR_DEVICE; \
  AtcLock atc_lock_(ctx)

namespace atc {
__global__ void k_probe_regions(int T, int nP, const uint64_t* seeds, const uint64_t* skips, const int64_t* region_len,
                                const int32_t* is_f32, const int64_t* region_off, const int64_t* need, double* init,
                                double* fin, TestsetView v, const int64_t* diff_off, const int32_t* diff_pos,
                                const double* diff_val, const double* pre, const int64_t* pre_off);
__global__ void k_probe_regions_many(const ProbeJob* jobs, int n_jobs);
__global__ void k_copy_meta(const ProbeJob* jobs);
__global__ void k_apply_diffs(int nP, const int64_t* region_len, const int64_t* region_off, const int64_t* diff_off,
                              const int32_t* diff_pos, const double* diff_val, double* fin);
__global__ void k_build_dirty(TestsetView ts, int32_t* dirty_pos, int32_t* dirty_cnt, int32_t* dirty_max);

__global__ void k_screen(TestsetView ts, SpecView sp, BindingSource src, uint64_t n, int budget,
                         int32_t* keys, uint64_t* surv, uint64_t surv_cap, unsigned long long* surv_cnt,
                         unsigned long long* reason_hist, int mode);
__global__ void k_pos0_table(TestsetView ts, SpecView sp, const uint8_t* perms, int n_perms, Pos0Table pt,
                             uint8_t* out, uint8_t* out1);
__global__ void k_pos0_table_expand(TestsetView ts, int n_perms, Pos0Table pt, uint8_t* out, uint8_t* out1,
                                    uint32_t* cm, uint32_t* allbad);
__global__ void k_pos0_table_conv(TestsetView ts, SpecView sp, const uint8_t* perms, int n_perms, Pos0Table pt,
                                  uint8_t* out, uint8_t* out1, uint32_t* cm, int stage_a, int stage_b,
                                  uint32_t* allbad);
__global__ void k_screen_enum(TestsetView ts, SpecView sp, BindingSource src, uint64_t n, Pos0Table pt,
                              uint64_t* surv, uint64_t surv_cap, unsigned long long* surv_cnt,
                              unsigned long long* reason_hist);
__global__ void k_gemm_need(TestsetView ts, int row_major, int32_t* need);
__global__ void k_cmask(const uint8_t* table, uint64_t n_words, int nI, uint32_t* cmask, int shift);
template <int NIc>  // NIc: the number of user ints when fixed at compile time (9), else 0
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
                               const unsigned long long* sel_cnt, int mode, int screened, int parts);
__global__ void k_confirm_pre(TestsetView ts, SpecView sp, BindingSource src, const uint64_t* surv,
                              const unsigned long long* surv_cnt, uint64_t surv_cap, int32_t* surv_keys,
                              uint32_t* pend, unsigned long long* pend_cnt, int mode, int screened);
__global__ void k_confirm_t0(TestsetView ts, SpecView sp, BindingSource src, const uint64_t* surv,
                             const unsigned long long* surv_cnt, uint64_t surv_cap, int32_t* surv_keys,
                             const uint32_t* pend, const unsigned long long* pend_cnt, uint32_t* next,
                             unsigned long long* next_cnt, int mode, int lazy, int screened, int gemm_parts);
__global__ void k_merge_keys(const uint64_t* surv, const unsigned long long* surv_cnt, uint64_t cap,
                             const int32_t* surv_keys, int32_t* keys);
__global__ void k_keys_to_verdicts(const int32_t* keys, int64_t n, int8_t* fail_t, int8_t* reason);
__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v);
__global__ void k_init_keys(int32_t* keys, const unsigned long long* cnt, uint64_t cap);
__global__ void k_sweep_small(const SmallJob* jobs, int n_jobs, int budget, int mode, uint2* surv, int32_t* keys,
                              uint64_t surv_cap, unsigned long long* surv_cnt);
__global__ void k_confirm_small(const SmallJob* jobs, int T, int mode, const uint2* surv, int32_t* keys,
                                uint64_t surv_cap, const unsigned long long* surv_cnt);
__global__ void k_finalize_small(const SmallJob* jobs, int n_jobs, uint64_t prefix, const uint2* surv,
                                 const int32_t* keys, uint64_t surv_cap, const unsigned long long* surv_cnt,
                                 uint64_t overflow_mark);
__global__ void k_finalize(const uint64_t* surv, const unsigned long long* surv_cnt, uint64_t cap,
                           const int32_t* surv_keys, uint64_t base, uint64_t* res, uint64_t res_cap,
                           unsigned long long* hist);
}  // namespace atc

struct atc_testset_handle {
  atc::TestsetView view{};
  int32_t T = 0, nI = 0, nP = 0, nF = 0;
  std::vector<int64_t> h_ints;  // host copy of the int values
  std::vector<void*> allocations;
  cudaEvent_t ready = nullptr;  // uploads + dirty lists complete (recorded on the copy stream)
  // layout, kept for in-place updates (atc_testsets_update_seeded)
  int cs = 0;                   // the copy stream all of this handle's uploads use
  std::vector<int64_t> lens, off, doff;
  std::vector<int32_t> is_f32;
  uint8_t* meta = nullptr;      // the small arrays (TestsetView points into it)
  size_t meta_bytes = 0, o_ints = 0, o_rlen = 0, o_roff = 0, o_dof = 0, o_isf = 0, o_tok = 0, o_dcnt = 0,
         o_dmax = 0, o_flt = 0;
  uint8_t* seeded = nullptr;    // seeds, stream positions, final-minus-init entries
  size_t seeded_cap = 0;
  bool needed_only = false;     // seeded with needed_only: region prefixes only
  uint8_t* pin = nullptr;       // pinned staging of the metadata + seeded blocks (async DMA)
  size_t pin_bytes = 0;
};

// Makes `st` wait for the upload of `ts` (no-op once it has completed).
inline void ts_wait(const atc_testset_handle* ts, cudaStream_t st) {
  if (ts && ts->ready) cudaStreamWaitEvent(st, ts->ready, 0);
}

namespace atc {

constexpr uint64_t kResultPrefix = 4096;        // passing indices returned with the first D2H
constexpr uint64_t kEnumChunkCap = 1ull << 22;  // survivors per K1 launch

bool build_spec_view(atc_ctx* ctx, const atc_spec_desc* s, SpecView& v);

// Runs K1 + K2 over `n` bindings; survivors/keys live in ctx scratch.
int run_eval(atc_ctx* ctx, const SpecView& sp, const atc_testset_handle* ts, const BindingSource& src,
             uint64_t n, int32_t* keys, uint64_t* surv, uint64_t surv_cap, unsigned long long* surv_cnt,
             int32_t* surv_keys, unsigned long long* hist, cudaStream_t st, const Pos0Table* pt = nullptr,
             const RowPlan* plan = nullptr);

// Per-space plan of an enumerated range: the decode, the position-0 table shape and
// the row plan.
struct EnumPlan {
  SpecView sp;
  Pos0Table pt;
  RowPlan plan;
  bool use_table = false, use_rows = false;
  uint64_t size_maps = 1, table_bytes = 0;
};
int plan_enumerated(atc_ctx* ctx, const atc_spec_desc* spec, const atc_testset_handle* ts, const uint8_t* perms,
                    int32_t n_perms, uint64_t begin, uint64_t end, int32_t mode, EnumPlan& e);
int enqueue_tables(atc_ctx* ctx, EnumPlan& e, const atc_testset_handle* ts, const uint8_t* perms, int32_t n_perms,
                   uint8_t** d_perms_out, cudaStream_t st, uint64_t begin, uint64_t end);

}  // namespace atc
