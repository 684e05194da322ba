// atc_liftc_adapter — the reference-side glue a liftc maintainer adds to use
// libatc_b200 (include/atc_b200.h).  It is written against the reference's own
// headers (/root/reference/proj/include/liftc/*.hpp) and replaces exactly two
// things:
//
//   1. the per-candidate loop body of pipeline::lift_function
//      (src/pipeline.cpp:248-310) — first_accepted() runs P2 for every ranked
//      candidate of a spec in ONE GPU launch and P1 (check_equivalence) only on
//      the P2 survivors, in rank order;
//   2. the oracle DispatchContext (rewriter.cpp:176-181) — make_gpu_dispatch()
//      returns a handler with the same checks and messages that computes on the
//      GPU (FP64, bit-exact); make_gpu_routed_dispatch() is the routed one
//      (rewriter.cpp:183-213), with "xpu" f32 calls on the tcgen05 backends.
//
// Nothing in the reference changes otherwise; the binding-independent half of
// verify_rewrite (draw_sizes, build_probe_image, the original run) is recorded
// with the reference's own functions.
#pragma once

#include <chrono>
#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "atc_b200.h"
#include "liftc/analysis.hpp"
#include "liftc/api_spec.hpp"
#include "liftc/interp.hpp"
#include "liftc/matching.hpp"
#include "liftc/minilang.hpp"
#include "liftc/pipeline.hpp"
#include "liftc/profitability.hpp"
#include "liftc/rewriter.hpp"

namespace liftc::gpu {

// atc_spec_desc for a validated ApiSpec (canonical dims, api_spec.cpp:116-119).
atc_spec_desc encode_spec(const api::ApiSpec& spec);

// The binding-independent half of verify_rewrite (rewriter.cpp:235-251) for
// tests t = 0..tests-1, kept alive for the upload.
struct RecordedTests {
  std::vector<std::string> int_params, ptr_params;
  std::vector<int64_t> ints;                  // [T][nI]
  std::vector<int32_t> is_f32, test_ok;       // [nP], [T]
  std::vector<int64_t> region_len;            // [nP]
  std::vector<std::vector<double>> init, fin;  // [T*nP]
  int T = 0;
  // The original run's final-minus-init entries per (t, p) (positions and final
  // values): with them the upload sends only the region prefixes an evaluation
  // can read (atc_testsets_upload_prefix) and rebuilds the finals on the device.
  std::vector<int64_t> diff_off;  // [T*nP + 1]
  std::vector<int32_t> diff_pos;
  std::vector<double> diff_val;
  // verify_rewrite's detail for a test whose draw or original run failed
  // (rewriter.cpp:241-251); empty when test_ok[t]
  std::vector<std::string> test_detail;  // [T]
};
RecordedTests record_tests(const minilang::Program& prog, const std::string& function,
                           const api::SizeRules& rules, uint64_t p2seed, int tests);

struct LoopResult {
  std::optional<size_t> winner;  // rank of the accepted candidate
  std::vector<int8_t> p2_fail_t, p2_reason;
  int p1_calls = 0;
  double gpu_ms = 0.0, record_ms = 0.0, p1_ms = 0.0;
  std::vector<std::string> verdicts;  // report_parity: evaluated[] verdicts in rank order
};

// Replacement of pipeline.cpp:248-310 for one spec: P2 (GPU, batched) for all
// ranked candidates, then P1 (host) on the survivors in rank order.
// The P2 verdicts of every spec's ranked list of one function from ONE test-set
// upload (atc_testsets_upload_prefix: needed-only region prefixes) and ONE batched
// evaluation (atc_eval_bindings_many): lists[i] are the ranked candidates of
// specs[i].  fail_t/reason are filled per spec, in rank order.
struct SpecVerdicts {
  std::vector<int8_t> fail_t, reason;
};
std::vector<SpecVerdicts> p2_verdicts(atc_ctx* ctx, const RecordedTests& r,
                                      const std::vector<const api::ApiSpec*>& specs,
                                      const std::vector<const std::vector<matching::CandidateBinding>*>& lists);

LoopResult first_accepted(atc_ctx* ctx, const minilang::Program& prog, const analysis::AnalyzedFunction& fn,
                          const std::string& function, const api::ApiSpec& spec,
                          const std::vector<matching::CandidateBinding>& ranked, const api::SizeRules& rules,
                          uint64_t fseed, int p1_tests, int verify_tests, const RecordedTests* recorded = nullptr,
                          bool report_parity = false, const SpecVerdicts* p2 = nullptr);

// The unpruned binding space of one spec in SURVEY.md Appendix C order: array
// k-permutations of the user pointers (odometer order) x size maps over the user
// ints (digit 0 fastest) — the space matching::raw_candidate_count counts
// (matching.cpp:119-131) before any pruning.
struct UnprunedSpace {
  std::vector<std::vector<int>> perms;
  std::vector<std::string> ptrs, ints;
  size_t maps = 1;
  UnprunedSpace(const analysis::AnalyzedFunction& fn, const api::ApiSpec& spec);
  size_t count() const { return perms.size() * maps; }
  matching::CandidateBinding at(const api::ApiSpec& spec, size_t idx) const;
  std::vector<uint8_t> perm_table() const;  // [n_perms][n_arrays] for atc_group_job / atc_enum_job
};

// The unpruned space as the ranked list, on every GPU of a device group: P2 over
// the whole space (atc_group_eval_enumerated_many: the space sharded over the
// members, the per-device results combined), then P1 (host check_equivalence) on
// the P2 survivors in index order; the first P1-equivalent survivor wins.
struct UnprunedResult {
  int64_t winner = -1;                // index of the accepted binding, -1 if none
  int64_t p2_passed = 0;              // bindings passing every P2 test
  std::vector<uint64_t> p2_passing;   // their indices (ascending, at most `cap`)
  int64_t reason_counts[ATC_REASON_COUNT] = {};
  int p1_calls = 0;
  double record_ms = 0.0, gpu_ms = 0.0, p1_ms = 0.0;
};
UnprunedResult first_accepted_unpruned(atc_group* g, const minilang::Program& prog,
                                       const analysis::AnalyzedFunction& fn, const std::string& function,
                                       const api::ApiSpec& spec, const api::SizeRules& rules, uint64_t fseed,
                                       int p1_tests, int verify_tests, int64_t cap = 4096);

// run_dispatch's exception text (rewriter.cpp:141, :145-147) for an
// ATC_ERR_DISPATCH message of atc_dispatch, which names params by index.
std::string dispatch_error_text(const api::ApiSpec& spec, const std::string& abi_msg);

// verify_rewrite's failure detail (rewriter.cpp:238-279) for binding `b` that the
// GPU rejected at test t with `reason` (ATC_FAIL_*): the test-set failure text,
// "dispatch failed: " + run_dispatch's message, or the first mismatching element
// of the compared arrays in the reference's order ("mismatch on X[i]: original
// ..., lifted ...") — recomputed for that one (binding, t) with atc_dispatch on
// the recorded probe image.
std::string p2_detail(atc_ctx* ctx, const RecordedTests& r, const minilang::FunctionIR& f,
                      const api::ApiSpec& spec, const matching::CandidateBinding& b, int t, int reason);

// The whole candidate stage of pipeline::lift_function (pipeline.cpp:223-330):
// every spec's matching + ranking (host, unchanged), ONE recording of the P2 test
// sets, ONE GPU P2 evaluation of every spec's ranked list, then the reference's
// control flow — specs in order, truncated specs skipped (too_many), candidates
// in rank order under the time budget, P1 (host check_equivalence) and, for an
// Equivalent candidate, rewrite + the GPU's P2 verdict — so status, winner,
// by_spec and evaluated[] (verdicts and details) equal the reference's.  With
// cfg.report = false, P1 runs only on P2 survivors (same winner, fewer P1 calls,
// evaluated[] lists only the candidates P1 ran on).
struct LoopConfig {
  int tests = 30;              // PipelineConfig::tests (P1)
  int verify_tests = 10;       // PipelineConfig::verify_tests (P2)
  size_t max_candidates = 100;
  double budget_sec = 600.0;
  bool report = true;
  // at most this many ranked candidates over all specs: P2 on demand, after P1 said
  // Equivalent (the reference's order); more: one GPU P2 batch up front
  size_t lazy_p2_max = 4;
};
struct CandidateLoop {
  pipeline::FunctionStatus status = pipeline::FunctionStatus::NoMatch;
  std::string status_detail;
  const api::ApiSpec* winning_spec = nullptr;
  int winner_rank = -1;
  rewriter::RewriteResult rewrite;  // the winner's (manifest: arrays/sizes/scalars)
  std::vector<pipeline::SpecCandidates> by_spec;
  std::vector<pipeline::CandidateOutcome> evaluated;
  int p1_calls = 0;
  double record_ms = 0.0, gpu_ms = 0.0, p1_ms = 0.0, total_ms = 0.0;
};
CandidateLoop candidate_loop(atc_ctx* ctx, const minilang::Program& prog, const analysis::AnalyzedFunction& fn,
                             const std::string& function, const std::vector<const api::ApiSpec*>& specs,
                             const api::SizeRules& rules, uint64_t fseed, const LoopConfig& cfg,
                             std::chrono::steady_clock::time_point start = std::chrono::steady_clock::now());

// DispatchContext whose handler is run_dispatch on the GPU (atc_dispatch).
interp::DispatchContext make_gpu_dispatch(const api::ApiSpec& spec, atc_ctx* ctx);

// rewriter::make_routed_dispatch (rewriter.hpp, rewriter.cpp:183-213) on the GPU.
// Labels each call "cpu"/"xpu" with profitability::predict_backend on the same
// (m, n, k) features the reference uses and records it in *choices.  "cpu"
// calls, f64 regions, and calls the FP32 backends cannot express run the exact
// FP64 path (== make_gpu_dispatch, bit-identical to the reference).  "xpu" calls
// on f32 regions run on atc_sgemm_rm / atc_conv2d_nchw only when the caller opts
// in with `precision` = ATC_PREC_TF32 / ATC_PREC_3XTF32.  The default, kRouteExact,
// keeps every call on the exact path, which makes the handler a drop-in for the
// reference's routed dispatch (labels recorded, results unchanged).
constexpr int32_t kRouteExact = -1;
interp::DispatchContext make_gpu_routed_dispatch(const api::ApiSpec& spec, atc_ctx* ctx,
                                                 const profitability::SvmModel* model,
                                                 std::vector<std::string>* choices,
                                                 int32_t precision = kRouteExact);

// The predictor features of one call (rewriter.cpp:194-205).
std::vector<long long> routed_sizes(const api::ApiSpec& spec, const std::map<std::string, long long>& sizes);

// profitability::sample_one (profitability.cpp:65-109) with the accelerator side on
// the B200 backend the routed dispatch calls: the same inputs (the TF32/BF16-exact
// patterns of :73-74), the same verification pass against profitability::cpu_gemm
// (finite, |c_cpu - c_xpu| <= 1e-3 (1 + |c_cpu|), else BackendFailure), then the
// median of `reps` runs of each side.  t_xpu is atc_sgemm_rm on the host buffers —
// H2D, tcgen05 GEMM, D2H: everything a routed "xpu" call costs — plus
// `xpu_overhead_sec` (0 by default: the measured call already includes its launch;
// the reference charges its CPU stand-in a fixed 2 ms, kXpuLaunchOverheadSec).  The
// label is 1 iff the B200 call was faster.  Samples feed profitability::train_svm
// unchanged, so the routed dispatch's model is trained on the backend it dispatches to.
profitability::TimingSample sample_one_b200(atc_ctx* ctx, const std::vector<long long>& sizes, int reps = 5,
                                            int32_t precision = ATC_PREC_3XTF32, double xpu_overhead_sec = 0.0);
// sample_timings (profitability.cpp:111-118): sample_one_b200 over every grid point, in order.
std::vector<profitability::TimingSample> sample_timings_b200(atc_ctx* ctx,
                                                             const std::vector<std::vector<long long>>& grid,
                                                             int reps = 5, int32_t precision = ATC_PREC_3XTF32,
                                                             double xpu_overhead_sec = 0.0);

}  // namespace liftc::gpu
