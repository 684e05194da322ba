// See atc_liftc_adapter.hpp.  Reference anchors are cited per function.
#include "atc_liftc_adapter.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <stdexcept>
#include <thread>

#include "liftc/equivalence.hpp"
#include "liftc/rng.hpp"

namespace liftc::gpu {

namespace {

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int role_code(const std::string& semantics, const std::string& role) {
  static const std::map<std::string, int> gemm = {{"m", ATC_SZ_M},     {"n", ATC_SZ_N},     {"k", ATC_SZ_K},
                                                  {"lda", ATC_SZ_LDA}, {"ldb", ATC_SZ_LDB}, {"ldc", ATC_SZ_LDC}};
  static const std::map<std::string, int> conv = {{"n", ATC_SZ_CN}, {"c", ATC_SZ_CC},   {"h", ATC_SZ_CH},
                                                  {"w", ATC_SZ_CW}, {"k", ATC_SZ_CK},   {"r", ATC_SZ_CR},
                                                  {"s", ATC_SZ_CS}, {"oh", ATC_SZ_COH}, {"ow", ATC_SZ_COW}};
  const auto& t = semantics == "gemm" ? gemm : conv;
  auto it = t.find(role);
  return it == t.end() ? -1 : it->second;
}

}  // namespace

atc_spec_desc encode_spec(const api::ApiSpec& spec) {
  atc_spec_desc d;
  std::memset(&d, 0, sizeof d);
  d.semantics = spec.semantics == "gemm" ? ATC_SEM_GEMM : ATC_SEM_CONV2D;
  d.layout = spec.layout == api::Layout::RowMajor ? ATC_LAYOUT_ROW : ATC_LAYOUT_COL;
  const auto arrays = spec.arrays();
  const auto sizes = spec.size_params();
  d.n_arrays = (int32_t)arrays.size();
  d.n_sizes = (int32_t)sizes.size();
  for (int r = 0; r < ATC_SZ_COUNT; ++r) d.role_size[r] = -1;
  std::map<std::string, int> size_index;
  for (size_t q = 0; q < sizes.size(); ++q) {
    size_index[sizes[q]->name] = (int)q;
    int rc = role_code(spec.semantics, sizes[q]->role);
    if (rc >= 0) d.role_size[rc] = (int)q;
  }
  for (size_t a = 0; a < arrays.size(); ++a) {
    const std::string& role = arrays[a]->role;
    d.array_role[a] = (role == "a" || role == "in") ? 0 : (role == "b" || role == "weights") ? 1 : 2;
    d.array_livein[a] = arrays[a]->liveness == api::Liveness::LiveIn;
    d.array_ndims[a] = (int32_t)arrays[a]->dims.size();
    for (size_t k = 0; k < arrays[a]->dims.size(); ++k) d.array_dims[a][k] = size_index.at(arrays[a]->dims[k]);
  }
  return d;
}

// rewriter.cpp:226-251: the same draws, image and original run verify_rewrite does.
RecordedTests record_tests(const minilang::Program& prog, const std::string& function, const api::SizeRules& rules,
                           uint64_t p2seed, int tests) {
  RecordedTests r;
  r.T = tests;
  const auto* f = prog.find(function);
  if (!f) throw std::invalid_argument("no function " + function);
  for (const auto& p : f->params) {
    if (p.kind == minilang::ParamKind::IntScalar) r.int_params.push_back(p.name);
    if (p.kind == minilang::ParamKind::Pointer) {
      r.ptr_params.push_back(p.name);
      r.is_f32.push_back(p.elem == minilang::ScalarType::F32);
    }
  }
  const size_t nP = r.ptr_params.size(), nI = r.int_params.size();
  r.ints.assign((size_t)tests * nI, 0);
  r.test_ok.assign(tests, 0);
  r.region_len.assign(nP, 65536);
  r.init.resize((size_t)tests * nP);
  r.fin.resize((size_t)tests * nP);
  // the T tests are independent streams (rewriter.cpp:236) and interp::execute is
  // re-entrant, so they are recorded on parallel host threads
  auto record_one = [&](int t) {
    Rng rng(Rng::mix(p2seed, "verify:" + function + ":" + std::to_string(t)));
    std::map<std::string, long long> sizes;
    bool drawn = false;
    for (int tries = 0; tries < 20 && !drawn; ++tries) drawn = analysis::draw_sizes(r.int_params, rules, rng, sizes);
    if (!drawn) {
      for (size_t p = 0; p < nP; ++p) r.init[t * nP + p].assign(65536, 0.0);
      return;
    }
    interp::MemoryImage img = analysis::build_probe_image(*f, sizes, rng);
    for (size_t i = 0; i < nI; ++i) r.ints[t * nI + i] = sizes.at(r.int_params[i]);
    interp::InstrumentationPolicy plain;
    auto ref = interp::execute(prog, function, img, plain);
    for (size_t p = 0; p < nP; ++p) {
      r.init[t * nP + p] = img.regions.at(r.ptr_params[p]).data;
      if (ref.status == interp::ExecStatus::Normal) r.fin[t * nP + p] = ref.final.regions.at(r.ptr_params[p]).data;
    }
    r.test_ok[t] = ref.status == interp::ExecStatus::Normal;
  };
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int workers = (int)std::min<unsigned>(hw, (unsigned)tests);
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w)
    pool.emplace_back([&] {
      for (int t = next.fetch_add(1); t < tests; t = next.fetch_add(1)) record_one(t);
    });
  for (auto& th : pool) th.join();
  // probe regions are kProbeRegionLen (analysis.cpp:23) long for every pointer
  for (size_t p = 0; p < nP; ++p)
    for (int t = 0; t < tests; ++t)
      if (!r.init[t * nP + p].empty()) r.region_len[p] = (int64_t)r.init[t * nP + p].size();
  return r;
}

LoopResult first_accepted(atc_ctx* ctx, const minilang::Program& prog, const analysis::AnalyzedFunction& fn,
                          const std::string& function, const api::ApiSpec& spec,
                          const std::vector<matching::CandidateBinding>& ranked, const api::SizeRules& rules,
                          uint64_t fseed, int p1_tests, int verify_tests, const RecordedTests* recorded,
                          bool report_parity) {
  LoopResult out;
  if (ranked.empty()) return out;
  auto t0 = std::chrono::steady_clock::now();
  RecordedTests local;
  if (!recorded) {
    local = record_tests(prog, function, rules, Rng::mix(fseed, "post"), verify_tests);  // pipeline.cpp:277
    recorded = &local;
  }
  out.record_ms = ms_since(t0);
  const RecordedTests& r = *recorded;
  const size_t nP = r.ptr_params.size();

  t0 = std::chrono::steady_clock::now();
  std::vector<const double*> ip(r.init.size()), fp(r.fin.size());
  for (size_t i = 0; i < r.init.size(); ++i) {
    ip[i] = r.init[i].data();
    fp[i] = r.fin[i].empty() ? nullptr : r.fin[i].data();
  }
  atc_testsets ts{r.T, (int32_t)r.int_params.size(), (int32_t)nP, r.ints.data(), r.is_f32.data(),
                  r.region_len.data(), ip.data(), fp.data(), r.test_ok.data()};
  atc_testset_handle* h = nullptr;
  if (atc_testsets_upload(ctx, &ts, &h) != ATC_OK) throw std::runtime_error(atc_last_error(ctx));
  const atc_spec_desc desc = encode_spec(spec);
  const auto arrays = spec.arrays();
  const auto sizes = spec.size_params();
  std::vector<uint8_t> am(ranked.size() * arrays.size()), sm(ranked.size() * sizes.size());
  for (size_t b = 0; b < ranked.size(); ++b) {
    for (size_t a = 0; a < arrays.size(); ++a) {
      const std::string& u = ranked[b].arrays.at(arrays[a]->name);
      am[b * arrays.size() + a] = (uint8_t)(std::find(r.ptr_params.begin(), r.ptr_params.end(), u) - r.ptr_params.begin());
    }
    for (size_t q = 0; q < sizes.size(); ++q) {
      const std::string& u = ranked[b].sizes.at(sizes[q]->name);
      sm[b * sizes.size() + q] = (uint8_t)(std::find(r.int_params.begin(), r.int_params.end(), u) - r.int_params.begin());
    }
  }
  out.p2_fail_t.resize(ranked.size());
  out.p2_reason.resize(ranked.size());
  int64_t first = -1;
  int rc = atc_eval_bindings(ctx, &desc, h, am.data(), sm.data(), (int64_t)ranked.size(), ATC_MODE_FP64,
                             out.p2_fail_t.data(), out.p2_reason.data(), &first);
  atc_testsets_free(ctx, h);
  if (rc != ATC_OK) throw std::runtime_error(atc_last_error(ctx));
  out.gpu_ms = ms_since(t0);

  // P1 on P2 survivors in rank order (pipeline.cpp:257-261 + :271-307).  With
  // report_parity, P1 also runs on the P2-rejected candidates that precede the
  // winner, so `verdicts` reproduces the reference's evaluated[] entries exactly:
  // the P1 verdict name, or "VerificationFailed" when P1 said Equivalent but P2
  // failed (pipeline.cpp:279-283).
  t0 = std::chrono::steady_clock::now();
  for (size_t b = 0; b < ranked.size(); ++b) {
    const bool p2_ok = out.p2_reason[b] == ATC_PASS;
    if (!p2_ok && !report_parity) continue;
    equivalence::EquivalenceConfig ec;
    ec.tests = p1_tests;
    ec.seed = fseed;
    ++out.p1_calls;
    auto er = equivalence::check_equivalence(prog, fn, ranked[b], spec, rules, ec);
    const bool eq = er.verdict == equivalence::Verdict::Equivalent;
    if (report_parity)
      out.verdicts.push_back(eq && !p2_ok ? std::string("VerificationFailed")
                                          : std::string(equivalence::verdict_name(er.verdict)));
    if (eq && p2_ok) {
      out.winner = b;
      break;
    }
  }
  out.p1_ms = ms_since(t0);
  return out;
}

interp::DispatchContext make_gpu_dispatch(const api::ApiSpec& spec, atc_ctx* ctx) {
  interp::DispatchContext dc;
  const atc_spec_desc desc = encode_spec(spec);
  dc.handler = [spec, desc, ctx](const std::string& name, const std::vector<interp::DispatchArg>& args,
                                 interp::MemoryImage& mem) {
    // rewriter.cpp:101-134: name, arity and kinds, positional decode
    if (name != "atc_dispatch_" + spec.semantics)
      throw std::runtime_error("dispatch name '" + name + "' does not match api semantics '" + spec.semantics + "'");
    if (args.size() != spec.params.size())
      throw std::runtime_error("dispatch arity " + std::to_string(args.size()) + ", api expects " +
                               std::to_string(spec.params.size()));
    std::vector<int64_t> sizes;
    std::vector<std::string> regions;
    for (size_t i = 0; i < spec.params.size(); ++i) {
      const auto& ap = spec.params[i];
      const auto& a = args[i];
      if (ap.kind == api::ApiParamKind::Array) {
        if (a.kind != interp::DispatchArg::Kind::Ptr)
          throw std::runtime_error("dispatch arg for array '" + ap.name + "' is not a pointer");
        if (!mem.regions.count(a.region)) throw std::runtime_error("dispatch region '" + a.region + "' missing");
        regions.push_back(a.region);
      } else if (ap.kind == api::ApiParamKind::IntSize) {
        if (a.kind != interp::DispatchArg::Kind::Int)
          throw std::runtime_error("dispatch arg for size '" + ap.name + "' is not an int");
        sizes.push_back(a.i);
      }
    }
    // full-region copies (rewriter.cpp:121), computed and written back on the GPU
    std::vector<std::vector<double>> bufs;
    std::vector<double*> ptrs;
    std::vector<int64_t> lens;
    std::vector<int32_t> f32;
    for (const auto& rname : regions) bufs.push_back(mem.regions.at(rname).data);
    for (size_t a = 0; a < regions.size(); ++a) {
      ptrs.push_back(bufs[a].data());
      lens.push_back((int64_t)bufs[a].size());
      f32.push_back(mem.regions.at(regions[a]).elem == minilang::ScalarType::F32);
    }
    int rc = atc_dispatch(ctx, &desc, sizes.data(), ptrs.data(), lens.data(), f32.data());
    if (rc == ATC_ERR_DISPATCH) {
      // same wording as rewriter.cpp:141,145-147 ("... is not positive", "... elements ...")
      throw std::runtime_error(std::string("dispatch: ") + atc_last_error(ctx));
    }
    if (rc != ATC_OK) throw std::runtime_error(atc_last_error(ctx));
    const auto arrays = spec.arrays();
    for (size_t a = 0; a < arrays.size(); ++a)
      if (arrays[a]->liveness != api::Liveness::LiveIn) mem.regions.at(regions[a]).data = bufs[a];
  };
  return dc;
}

}  // namespace liftc::gpu
