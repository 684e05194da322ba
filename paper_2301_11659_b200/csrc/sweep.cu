// C ABI: prepared corpus sweeps (atc_enum_batch_*, atc_eval_enumerated_many), one CUDA graph per run.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "atc_b200.h"
#include "capi_internal.h"

using namespace atc;

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
  // small spaces (k_sweep_small: one launch for all of them)
  std::vector<char> small;       // per job
  std::vector<int> small_jobs;   // job indices, in SmallJob order
  SmallJob* d_small = nullptr;   // device job table
  uint32_t small_ctas = 0;
  int small_T = 0;                // largest T of the small jobs
  uint2* small_surv = nullptr;    // (job, index) survivors of k_sweep_small
  int32_t* small_keys = nullptr;
  unsigned long long* small_cnt = nullptr;
  std::vector<const atc_testset_handle*> small_ts;  // distinct handles the launch waits for
};

namespace {

// per job of a batch: count, passing count, passing prefix (a job with more passing
// bindings than the prefix is redone alone by atc_eval_enumerated); small, because
// the whole block comes back every run
constexpr uint64_t kBatchPrefix = 256;
constexpr uint64_t kBatchStride = 2 + kBatchPrefix;

size_t batch_res_words(int n) { return (size_t)n * (kBatchStride + 8); }

// Gemm spaces of at most 2^ctx->opt_small_log2 bindings run in k_sweep_small; each
// gets one CTA per kSmallSlice bindings.
constexpr uint64_t kSmallSlice = 1024;
constexpr int64_t kSmallMaxInt = 16;
constexpr int kSmallBudget = 16;  // output positions thread_check looks at (t = 0)
constexpr uint64_t kSmallSurvCap = 1ull << 20;  // survivors of all small jobs together

// Concurrent branches: the small (gemm) spaces as one k_sweep_small chain on side
// stream 0; the conv spaces' chains (tables, K1, K2, finalize) round-robin over
// ctx->opt_conv_streams streams (conv_stream, side streams 3, 2, 1: one space's
// latency-bound tables and K2 run beside another's K1; 4 streams: 3.00 -> 2.32 ms
// per corpus sweep, tools/sweep_streams.py; 8 streams, one per corpus conv space,
// after K1's instruction diet: 1.28 -> 1.06 ms); other large gemm ranges round-robin
// over side streams 1, 2, ... (in the corpus: one, on a stream of its own).  (Higher launch priority
// for the tables / K2 / finalize kernels was measured too: K2 then interleaves with
// the next K1s, 1.06 -> 1.11 ms — the step is K1-throughput bound.)  Side stream
// k's scratch lives at slot + kSlotsPerStream * (k + 1); every branch forks from and joins back
// into `st`, so a captured graph has the same branches.
int enqueue_batch(atc_ctx* ctx, atc_enum_batch* b, cudaStream_t st, bool wait_uploads) {
  const uint64_t chunk_cap = kEnumChunkCap;
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(b->res + (size_t)b->n * kBatchStride);
  cudaMemsetAsync(b->res, 0, batch_res_words(b->n) * 8, st);
  int n_side = 0;
  // jobs with an empty range (a multi-GPU rank's share of nothing) take no stream,
  // event wait or graph node at all; small spaces run in the one k_sweep_small launch
  auto active = [&](int j) { return b->batched[j] && !b->small[j] && b->jobs[j].end > b->jobs[j].begin; };
  int n_active = 0;
  for (int j = 0; j < b->n; ++j) {
    n_active += active(j);
    n_side += active(j) && b->plans[j].sp.sem != ATC_SEM_CONV2D;
  }
  const bool has_small = b->small_ctas > 0;
  const int n_conv = n_active - n_side;
  const bool split = (has_small && n_active > 0) || (ctx->opt_conv_streams > 1 && n_conv > 1) || n_side > 1 ||
                     (n_side == 1 && n_side < n_active);
  if (split) {
    cudaEventRecord(ctx->fork_ev, st);
    for (int k = 0; k < atc_ctx::kSideStreams; ++k) cudaStreamWaitEvent(ctx->side_stream[k], ctx->fork_ev, 0);
    cudaStreamWaitEvent(ctx->conv_stream, ctx->fork_ev, 0);
  }
  if (has_small) {  // every small space in one launch, on side stream 0 (or `st` alone)
    cudaStream_t ss = split ? ctx->side_stream[0] : st;
    for (const atc_testset_handle* h : b->small_ts) {
      if (wait_uploads)
        ts_wait(h, ss);
      else if (h->ready)
        cudaStreamWaitEvent(ss, h->ready, cudaEventWaitExternal);
    }
    const int nj = (int)b->small_jobs.size();
    cudaMemsetAsync(b->small_cnt, 0, 8, ss);
    k_sweep_small<<<b->small_ctas, 256, 0, ss>>>(b->d_small, nj, kSmallBudget, b->mode, b->small_surv, b->small_keys,
                                                 kSmallSurvCap, b->small_cnt);
    k_confirm_small<<<(unsigned)ctx->sm_count * 4, 256, 0, ss>>>(b->d_small, b->small_T, b->mode, b->small_surv,
                                                                 b->small_keys, kSmallSurvCap, b->small_cnt);
    k_finalize_small<<<64, 256, 0, ss>>>(b->d_small, nj, kBatchPrefix, b->small_surv, b->small_keys, kSmallSurvCap,
                                         b->small_cnt, (unsigned long long)kEnumChunkCap + 1);
    if (ctx->prof) ctx->prof_kernels += 3;
  }
  // large gemm chains on side streams 1, 2, ... (0: the small-space sweep); the conv
  // chains take side streams kSideStreams - 1, - 2, ... and conv_stream
  int side_next = has_small ? 1 : 0, conv_next = 0;
  int rc = ATC_OK;
  // gemm chains first: nodes are handed to the GPU in the order they were enqueued,
  // and a gemm chain enqueued after the conv chains only gets SMs once the K1 CTAs
  // (a whole SM each) have drained — its short latency-bound kernels then form the
  // step's tail; enqueued first, they run beside the conv tables
  std::vector<int> order;
  for (int pass = 0; pass < 2; ++pass)
    for (int j = 0; j < b->n; ++j)
      if (active(j) && (b->plans[j].sp.sem == ATC_SEM_CONV2D) == (pass == 1)) order.push_back(j);
  {  // conv chains longest first (estimated K1 + table time; timeline span 695 -> 678 us)
    auto est = [&](int j) { return (double)(b->jobs[j].end - b->jobs[j].begin) * 16e-9 + 2.0 * b->jobs[j].n_perms; };
    auto first_conv =
        std::find_if(order.begin(), order.end(), [&](int j) { return b->plans[j].sp.sem == ATC_SEM_CONV2D; });
    std::stable_sort(first_conv, order.end(), [&](int x, int y) { return est(x) > est(y); });
  }
  for (size_t oi = 0; oi < order.size() && rc == ATC_OK; ++oi) {
    const int j = order[oi];
    atc_enum_job& job = b->jobs[j];
    EnumPlan& e = b->plans[j];
    // conv spaces on the caller's stream and side stream 0 alternately when they
    // are small (a multi-GPU rank's share: chains of short kernels), else the
    // caller's stream; gemm spaces round-robin over the side streams
    int sk = -1;
    if (split && e.sp.sem == ATC_SEM_CONV2D) {
      if (ctx->opt_conv_streams > 1) {  // large conv chains round-robin over conv_stream + side streams 3, 2, 1
        const int k = conv_next++ % ctx->opt_conv_streams;
        sk = k == 0 ? -1 : atc_ctx::kSideStreams - k;
      } else if (job.end - job.begin < (1ull << 30)) {
        sk = conv_next ? 0 : -1;
        conv_next ^= 1;
      }
    } else if (split) {
      sk = side_next;
      side_next = side_next + 1 < atc_ctx::kSideStreams ? side_next + 1 : (has_small ? 1 : 0);
    }
    const bool side = sk >= 0;
    cudaStream_t js = side ? ctx->side_stream[sk] : split ? ctx->conv_stream : st;
    ctx->slot_base = side ? atc_ctx::kSlotsPerStream * (sk + 1) : 0;
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
  // the small (gemm) spaces: one k_sweep_small launch per run, CTAs in job order
  b->small.assign(n_jobs, 0);
  std::vector<SmallJob> small;
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(b->res + (size_t)n_jobs * kBatchStride);
  for (int j = 0; j < n_jobs; ++j) {
    const atc_enum_job& job = jobs[j];
    const uint64_t n = job.end - job.begin;
    if (!b->batched[j] || n == 0 || ctx->opt_small_log2 == 0 || n > (1ull << ctx->opt_small_log2) ||
        b->plans[j].sp.sem != ATC_SEM_GEMM)
      continue;
    // a warp per (survivor, test) suits short checks; spaces whose outputs can be
    // many (m*n up to U^2 for the largest drawn int U: config 1's 64^3) keep the
    // per-space chain, whose K2 spreads one binding's outputs over more warps
    int64_t umax = 0;
    for (int64_t v : job.ts->h_ints) umax = std::max(umax, v);
    if (umax > kSmallMaxInt) continue;
    b->small[j] = 1;
    b->small_jobs.push_back(j);
    SmallJob sj{};
    sj.ts = job.ts->view;
    sj.sp = b->plans[j].sp;
    sj.src = BindingSource{nullptr, nullptr, b->d_perms[j], b->plans[j].size_maps, job.begin, 1};
    sj.n = n;
    sj.res = b->res + (size_t)j * kBatchStride;
    sj.hist = hist + 8 * (size_t)j;
    sj.cta0 = b->small_ctas;
    sj.ctas = (uint32_t)((n + kSmallSlice - 1) / kSmallSlice);
    b->small_ctas += sj.ctas;
    b->small_T = std::max(b->small_T, (int)job.ts->T);
    small.push_back(sj);
    if (std::find(b->small_ts.begin(), b->small_ts.end(), job.ts) == b->small_ts.end()) b->small_ts.push_back(job.ts);
  }
  if (!small.empty()) {
    // survivor list and keys: context scratch (the same slots every batch; a graph
    // replays with them in place)
    b->small_surv = (uint2*)atc_ctx_scratch(ctx, 26, kSmallSurvCap * sizeof(uint2));
    b->small_keys = (int32_t*)atc_ctx_scratch(ctx, 27, kSmallSurvCap * 4);
    b->small_cnt = (unsigned long long*)atc_ctx_scratch(ctx, 28, 64);
    const size_t bytes = small.size() * sizeof(SmallJob);
    if (transient)
      b->d_small = (SmallJob*)atc_ctx_scratch(ctx, 25, bytes);
    else if (cudaMalloc(&b->d_small, bytes) != cudaSuccess)
      b->d_small = nullptr;
    if (!b->d_small || !b->small_surv || !b->small_keys || !b->small_cnt ||
        !atc_cuda_ok(ctx, cudaMemcpyAsync(b->d_small, small.data(), bytes, cudaMemcpyHostToDevice, ctx->stream),
                     "H2D small jobs")) {
      atc_set_error(ctx, "batch allocation failed (small jobs)");
      atc_enum_batch_destroy(ctx, b);
      return nullptr;
    }
  }
  return b;
}

}  // namespace

extern "C" {

atc_enum_batch* atc_enum_batch_create(atc_ctx* ctx, atc_enum_job* jobs, int32_t n_jobs, int32_t mode) {
  AtcLock lock(ctx);
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
  AtcLock lock(ctx);
  if (ctx) cudaSetDevice(ctx->device);
  if (b->exec) cudaGraphExecDestroy(b->exec);
  if (!b->transient) {
    if (b->d_small) cudaFree(b->d_small);
    if (b->perm_block) cudaFree(b->perm_block);
    if (b->res) cudaFree(b->res);
    if (b->h_res) cudaFreeHost(b->h_res);
  }
  delete b;
}

int atc_enum_batch_run(atc_ctx* ctx, atc_enum_batch* b) {
  ATC_ENTER(ctx);
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
  ATC_ENTER(ctx);
  if (n_jobs == 0) return ATC_OK;
  atc_enum_batch* b = batch_create(ctx, jobs, n_jobs, mode, true);
  if (!b) return ATC_ERR_ARG;
  const int rc = atc_enum_batch_run(ctx, b);
  atc_enum_batch_destroy(ctx, b);
  return rc;
}

}  // extern "C"
