// See atc_liftc_adapter.hpp.  Reference anchors are cited per function.
#include "atc_liftc_adapter.hpp"

#include <algorithm>
#include <functional>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <thread>

#include "host_phases.hpp"
#include "host_vm.hpp"
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
  r.test_detail.assign(tests, "");
  r.init.resize((size_t)tests * nP);
  r.fin.resize((size_t)tests * nP);
  // the T tests are independent streams (rewriter.cpp:236): recorded on parallel
  // host threads, each original run on the compiled host VM (the
  // reference interpreter's semantics, host_vm.hpp)
  const HostVm vm(prog);
  std::vector<std::vector<int32_t>> dpos((size_t)tests * nP);
  std::vector<std::vector<double>> dval((size_t)tests * nP);
  auto record_one = [&](int t) {
    Rng rng(Rng::mix(p2seed, "verify:" + function + ":" + std::to_string(t)));
    std::map<std::string, long long> sizes;
    bool drawn = false;
    for (int tries = 0; tries < 20 && !drawn; ++tries) drawn = analysis::draw_sizes(r.int_params, rules, rng, sizes);
    if (!drawn) {
      for (size_t p = 0; p < nP; ++p) r.init[t * nP + p].assign(65536, 0.0);
      r.test_detail[t] = "could not draw sizes under the declared rules";  // rewriter.cpp:240
      return;
    }
    interp::MemoryImage img = analysis::build_probe_image(*f, sizes, rng);
    for (size_t i = 0; i < nI; ++i) r.ints[t * nI + i] = sizes.at(r.int_params[i]);
    interp::InstrumentationPolicy plain;
    auto ref = vm.execute(function, img, plain);
    for (size_t p = 0; p < nP; ++p) {
      r.init[t * nP + p] = img.regions.at(r.ptr_params[p]).data;
      if (ref.status == interp::ExecStatus::Normal) {
        r.fin[t * nP + p] = ref.final.regions.at(r.ptr_params[p]).data;
        const auto& a = r.init[t * nP + p];
        const auto& b = r.fin[t * nP + p];
        for (size_t i = 0; i < a.size() && i < b.size(); ++i)
          if (std::memcmp(&a[i], &b[i], sizeof(double)) != 0) {  // bitwise: -0.0 / NaN entries travel too
            dpos[t * nP + p].push_back((int32_t)i);
            dval[t * nP + p].push_back(b[i]);
          }
      }
    }
    r.test_ok[t] = ref.status == interp::ExecStatus::Normal;
    if (!r.test_ok[t]) r.test_detail[t] = std::string("original run ended ") + interp::status_name(ref.status);
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
  r.diff_off.assign(1, 0);
  for (size_t i = 0; i < dpos.size(); ++i) {
    r.diff_pos.insert(r.diff_pos.end(), dpos[i].begin(), dpos[i].end());
    r.diff_val.insert(r.diff_val.end(), dval[i].begin(), dval[i].end());
    r.diff_off.push_back((int64_t)r.diff_pos.size());
  }
  // probe regions are kProbeRegionLen (analysis.cpp:23) long for every pointer
  for (size_t p = 0; p < nP; ++p)
    for (int t = 0; t < tests; ++t)
      if (!r.init[t * nP + p].empty()) r.region_len[p] = (int64_t)r.init[t * nP + p].size();
  return r;
}

namespace {

// The prefix-upload descriptor of r (pointers into r and `ip`).
atc_prefix_testsets prefix_desc(const RecordedTests& r, std::vector<const double*>& ip) {
  const size_t nP = r.ptr_params.size();
  ip.assign(r.init.size(), nullptr);
  for (size_t i = 0; i < r.init.size(); ++i) ip[i] = r.test_ok[i / nP] ? r.init[i].data() : nullptr;
  return atc_prefix_testsets{r.T,
                             (int32_t)r.int_params.size(),
                             (int32_t)nP,
                             r.ints.data(),
                             r.is_f32.data(),
                             r.region_len.data(),
                             r.test_ok.data(),
                             ip.data(),
                             r.diff_off.data(),
                             r.diff_pos.data(),
                             r.diff_val.data()};
}

// Uploads r (the needed region prefixes + final-minus-init entries when the diffs
// were recorded, else the full regions) and returns the handle.
atc_testset_handle* upload(atc_ctx* ctx, const RecordedTests& r) {
  const size_t nP = r.ptr_params.size();
  atc_testset_handle* h = nullptr;
  int rc;
  if (!r.diff_off.empty()) {
    std::vector<const double*> ip;
    const atc_prefix_testsets px = prefix_desc(r, ip);
    rc = atc_testsets_upload_prefix(ctx, &px, &h);
  } else {
    std::vector<const double*> ip(r.init.size()), fp(r.fin.size());
    for (size_t i = 0; i < r.init.size(); ++i) {
      ip[i] = r.init[i].data();
      fp[i] = r.fin[i].empty() ? nullptr : r.fin[i].data();
    }
    atc_testsets ts{r.T, (int32_t)r.int_params.size(), (int32_t)nP, r.ints.data(), r.is_f32.data(),
                    r.region_len.data(), ip.data(), fp.data(), r.test_ok.data()};
    rc = atc_testsets_upload(ctx, &ts, &h);
  }
  if (rc != ATC_OK) throw std::runtime_error(atc_last_error(ctx));
  return h;
}

}  // namespace

std::vector<SpecVerdicts> p2_verdicts(atc_ctx* ctx, const RecordedTests& r,
                                      const std::vector<const api::ApiSpec*>& specs,
                                      const std::vector<const std::vector<matching::CandidateBinding>*>& lists) {
  std::vector<SpecVerdicts> out(specs.size());
  std::vector<atc_spec_desc> descs(specs.size());
  std::vector<std::vector<uint8_t>> am(specs.size()), sm(specs.size());
  std::vector<atc_bind_job> jobs;
  size_t total = 0;
  for (size_t i = 0; i < specs.size(); ++i) total += lists[i]->size();
  if (total == 0) return out;
  atc_testset_handle* h = upload(ctx, r);
  for (size_t i = 0; i < specs.size(); ++i) {
    const auto& ranked = *lists[i];
    descs[i] = encode_spec(*specs[i]);
    const auto arrays = specs[i]->arrays();
    const auto sizes = specs[i]->size_params();
    am[i].resize(ranked.size() * arrays.size());
    sm[i].resize(ranked.size() * sizes.size());
    for (size_t b = 0; b < ranked.size(); ++b) {
      for (size_t a = 0; a < arrays.size(); ++a) {
        const std::string& u = ranked[b].arrays.at(arrays[a]->name);
        am[i][b * arrays.size() + a] =
            (uint8_t)(std::find(r.ptr_params.begin(), r.ptr_params.end(), u) - r.ptr_params.begin());
      }
      for (size_t q = 0; q < sizes.size(); ++q) {
        const std::string& u = ranked[b].sizes.at(sizes[q]->name);
        sm[i][b * sizes.size() + q] =
            (uint8_t)(std::find(r.int_params.begin(), r.int_params.end(), u) - r.int_params.begin());
      }
    }
    out[i].fail_t.resize(ranked.size());
    out[i].reason.resize(ranked.size());
    if (ranked.empty()) continue;
    atc_bind_job j{};
    j.spec = &descs[i];
    j.ts = h;
    j.arr_map = am[i].data();
    j.size_map = sm[i].data();
    j.n_bindings = (int64_t)ranked.size();
    j.fail_t = out[i].fail_t.data();
    j.reason = out[i].reason.data();
    jobs.push_back(j);
  }
  const int rc = atc_eval_bindings_many(ctx, jobs.data(), (int32_t)jobs.size(), ATC_MODE_FP64);
  const std::string err = rc != ATC_OK ? atc_last_error(ctx) : "";
  atc_testsets_free(ctx, h);
  if (rc != ATC_OK) throw std::runtime_error(err);
  return out;
}

LoopResult first_accepted(atc_ctx* ctx, const minilang::Program& prog, const analysis::AnalyzedFunction& fn,
                          const std::string& function, const api::ApiSpec& spec,
                          const std::vector<matching::CandidateBinding>& ranked, const api::SizeRules& rules,
                          uint64_t fseed, int p1_tests, int verify_tests, const RecordedTests* recorded,
                          bool report_parity, const SpecVerdicts* p2) {
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

  t0 = std::chrono::steady_clock::now();
  if (p2) {
    out.p2_fail_t = p2->fail_t;
    out.p2_reason = p2->reason;
  } else {
    auto v = p2_verdicts(ctx, r, {&spec}, {&ranked});
    out.p2_fail_t = std::move(v[0].fail_t);
    out.p2_reason = std::move(v[0].reason);
  }
  out.gpu_ms = ms_since(t0);

  const HostVm vm(prog);
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
    auto er = check_equivalence(vm, prog, fn, ranked[b], spec, rules, ec);
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

UnprunedSpace::UnprunedSpace(const analysis::AnalyzedFunction& fn, const api::ApiSpec& spec) : ints(fn.int_params) {
  for (const auto& a : fn.arrays) ptrs.push_back(a.name);
  const size_t nA = spec.arrays().size();
  std::vector<int> sel(nA);
  std::vector<bool> used(ptrs.size(), false);
  std::function<void(size_t)> rec = [&](size_t i) {
    if (i == nA) {
      perms.push_back(sel);
      return;
    }
    for (size_t j = 0; j < ptrs.size(); ++j)
      if (!used[j]) {
        used[j] = true;
        sel[i] = (int)j;
        rec(i + 1);
        used[j] = false;
      }
  };
  rec(0);
  for (size_t q = 0; q < spec.size_params().size(); ++q) maps *= ints.size();
}

matching::CandidateBinding UnprunedSpace::at(const api::ApiSpec& spec, size_t idx) const {
  matching::CandidateBinding b;
  const auto arrays = spec.arrays();
  const auto sizes = spec.size_params();
  const auto& perm = perms[idx / maps];
  for (size_t a = 0; a < arrays.size(); ++a) b.arrays[arrays[a]->name] = ptrs[perm[a]];
  size_t x = idx % maps;
  for (size_t q = 0; q < sizes.size(); ++q) {
    b.sizes[sizes[q]->name] = ints[x % ints.size()];
    x /= ints.size();
  }
  return b;
}

std::vector<uint8_t> UnprunedSpace::perm_table() const {
  std::vector<uint8_t> t;
  for (const auto& p : perms)
    for (int u : p) t.push_back((uint8_t)u);
  return t;
}

UnprunedResult first_accepted_unpruned(atc_group* g, const minilang::Program& prog,
                                       const analysis::AnalyzedFunction& fn, const std::string& function,
                                       const api::ApiSpec& spec, const api::SizeRules& rules, uint64_t fseed,
                                       int p1_tests, int verify_tests, int64_t cap) {
  UnprunedResult out;
  const UnprunedSpace space(fn, spec);
  if (space.count() == 0) return out;
  auto t0 = std::chrono::steady_clock::now();
  const RecordedTests r = record_tests(prog, function, rules, Rng::mix(fseed, "post"), verify_tests);
  out.record_ms = ms_since(t0);

  t0 = std::chrono::steady_clock::now();
  std::vector<const double*> ip;
  const atc_prefix_testsets px = prefix_desc(r, ip);
  atc_group_testsets* h = nullptr;
  if (atc_group_testsets_upload_prefix(g, &px, &h) != ATC_OK) throw std::runtime_error(atc_group_last_error(g));
  const atc_spec_desc desc = encode_spec(spec);
  const std::vector<uint8_t> perms = space.perm_table();
  out.p2_passing.resize((size_t)std::max<int64_t>(cap, 1));
  atc_group_job job{};
  job.spec = &desc;
  job.ts = h;
  job.perms = perms.data();
  job.n_perms = (int32_t)space.perms.size();
  job.begin = 0;
  job.end = space.count();
  job.survivors = out.p2_passing.data();
  job.cap = cap;
  const int rc = atc_group_eval_enumerated_many(g, &job, 1, ATC_MODE_FP64);
  const std::string err = rc != ATC_OK ? atc_group_last_error(g) : "";
  atc_group_testsets_free(g, h);
  if (rc != ATC_OK) throw std::runtime_error(err);
  out.p2_passed = job.n_survivors;
  for (int k = 0; k < ATC_REASON_COUNT; ++k) out.reason_counts[k] = job.reason_counts[k];
  out.p2_passing.resize((size_t)std::min<int64_t>(job.n_survivors, cap));
  out.gpu_ms = ms_since(t0);

  // P1 on the P2 survivors in index order (pipeline.cpp:257-261, :275-277 order of
  // the two phases swapped: P2 is the cheap screen here)
  t0 = std::chrono::steady_clock::now();
  const HostVm vm(prog);
  for (uint64_t idx : out.p2_passing) {
    equivalence::EquivalenceConfig ec;
    ec.tests = p1_tests;
    ec.seed = fseed;
    ++out.p1_calls;
    auto er = check_equivalence(vm, prog, fn, space.at(spec, idx), spec, rules, ec);
    if (er.verdict == equivalence::Verdict::Equivalent) {
      out.winner = (int64_t)idx;
      break;
    }
  }
  out.p1_ms = ms_since(t0);
  return out;
}

std::string dispatch_error_text(const api::ApiSpec& spec, const std::string& abi_msg) {
  // atc_dispatch names params by index (the C descriptor carries no names)
  int idx = -1;
  long long have = 0, need = 0;
  const auto sizes = spec.size_params();
  const auto arrays = spec.arrays();
  if (std::sscanf(abi_msg.c_str(), "dispatch size #%d is not positive", &idx) == 1 && idx >= 0 &&
      (size_t)idx < sizes.size())
    return "dispatch size '" + sizes[idx]->name + "' is not positive";  // rewriter.cpp:141
  if (std::sscanf(abi_msg.c_str(), "region bound to array #%d holds %lld elements, call needs %lld", &idx, &have,
                  &need) == 3 &&
      idx >= 0 && (size_t)idx < arrays.size())
    return "region bound to '" + arrays[idx]->name + "' holds " + std::to_string(have) +  // :145-147
           " elements, call needs " + std::to_string(need);
  return abi_msg;
}

namespace {

// One decoded dispatch call: rewriter.cpp:101-134's name/arity/kind checks and
// positional decode (messages verbatim).
struct DecodedCall {
  std::vector<int64_t> sizes;                 // spec.size_params() order
  std::map<std::string, long long> by_name;  // size name -> value
  std::vector<std::string> regions;           // spec.arrays() order
};

DecodedCall decode_call(const api::ApiSpec& spec, const std::string& name,
                        const std::vector<interp::DispatchArg>& args, const interp::MemoryImage& mem) {
  if (name != "atc_dispatch_" + spec.semantics)
    throw std::runtime_error("dispatch name '" + name + "' does not match api semantics '" + spec.semantics + "'");
  if (args.size() != spec.params.size())
    throw std::runtime_error("dispatch arity " + std::to_string(args.size()) + ", api expects " +
                             std::to_string(spec.params.size()));
  DecodedCall d;
  for (size_t i = 0; i < spec.params.size(); ++i) {
    const auto& ap = spec.params[i];
    const auto& a = args[i];
    if (ap.kind == api::ApiParamKind::Array) {
      if (a.kind != interp::DispatchArg::Kind::Ptr)
        throw std::runtime_error("dispatch arg for array '" + ap.name + "' is not a pointer");
      if (!mem.regions.count(a.region)) throw std::runtime_error("dispatch region '" + a.region + "' missing");
      d.regions.push_back(a.region);
    } else if (ap.kind == api::ApiParamKind::IntSize) {
      if (a.kind != interp::DispatchArg::Kind::Int)
        throw std::runtime_error("dispatch arg for size '" + ap.name + "' is not an int");
      d.sizes.push_back(a.i);
      d.by_name[ap.name] = a.i;
    }
  }
  return d;
}

// run_dispatch (rewriter.cpp:136-161) on the GPU in FP64: atc_dispatch does the
// extent checks, the reference arithmetic and the f32 write-back rounding.
void exact_dispatch(const api::ApiSpec& spec, const atc_spec_desc& desc, atc_ctx* ctx, const DecodedCall& d,
                    interp::MemoryImage& mem) {
  // full-region copies (rewriter.cpp:121), computed and written back on the GPU
  std::vector<std::vector<double>> bufs;
  std::vector<double*> ptrs;
  std::vector<int64_t> lens;
  std::vector<int32_t> f32;
  for (const auto& rname : d.regions) bufs.push_back(mem.regions.at(rname).data);
  for (size_t a = 0; a < d.regions.size(); ++a) {
    ptrs.push_back(bufs[a].data());
    lens.push_back((int64_t)bufs[a].size());
    f32.push_back(mem.regions.at(d.regions[a]).elem == minilang::ScalarType::F32);
  }
  int rc = atc_dispatch(ctx, &desc, d.sizes.data(), ptrs.data(), lens.data(), f32.data());
  if (rc == ATC_ERR_DISPATCH) throw std::runtime_error(dispatch_error_text(spec, atc_last_error(ctx)));
  if (rc != ATC_OK) throw std::runtime_error(atc_last_error(ctx));
  const auto arrays = spec.arrays();
  for (size_t a = 0; a < arrays.size(); ++a)
    if (arrays[a]->liveness != api::Liveness::LiveIn) mem.regions.at(d.regions[a]).data = bufs[a];
}

// rewriter.cpp:164-172: the value of the size parameter with `role`, else 1.
long long role_size(const api::ApiSpec& spec, const std::map<std::string, long long>& sizes, const std::string& role,
                    long long dflt = 1) {
  for (const auto& p : spec.params)
    if (p.kind == api::ApiParamKind::IntSize && p.role == role) {
      auto it = sizes.find(p.name);
      if (it != sizes.end()) return it->second;
    }
  return dflt;
}

// The array of `spec` with semantic `role` and its region index in d.regions.
int array_slot(const api::ApiSpec& spec, const std::string& role) {
  const auto arrays = spec.arrays();
  for (size_t a = 0; a < arrays.size(); ++a)
    if (arrays[a]->role == role) return (int)a;
  return -1;
}

// The "xpu" leg: the same call on the tcgen05 FP32 backends (atc_sgemm_rm /
// atc_conv2d_nchw) when every region is f32 and the call is one those backends
// express; returns false (caller runs the exact path) otherwise.  The checks
// mirror run_dispatch's (rewriter.cpp:136-148) so the exact path is left to
// raise the reference's errors.
bool tensor_dispatch(const api::ApiSpec& spec, atc_ctx* ctx, int32_t precision, const DecodedCall& d,
                     interp::MemoryImage& mem) {
  for (const auto& r : d.regions)
    if (mem.regions.at(r).elem != minilang::ScalarType::F32) return false;
  for (const auto* ap : spec.arrays()) {
    long double extent = 1;
    for (const auto& dim : ap->dims) {
      auto it = d.by_name.find(dim);
      if (it == d.by_name.end() || it->second < 1) return false;
      extent *= (long double)it->second;
    }
    if ((long double)mem.regions.at(d.regions[array_slot(spec, ap->role)]).data.size() < extent) return false;
  }
  const auto& S = d.by_name;
  if (spec.semantics == "gemm") {
    // equivalence.cpp:40-64 with lda/ldb/ldc; operands packed dense row-major
    const long long m = role_size(spec, S, "m", 0), n = role_size(spec, S, "n", 0), k = role_size(spec, S, "k", 0);
    const bool row = spec.layout == api::Layout::RowMajor;
    const long long lda = role_size(spec, S, "lda", row ? k : m), ldb = role_size(spec, S, "ldb", row ? n : k),
                    ldc = role_size(spec, S, "ldc", row ? n : m);
    if (m < 1 || n < 1 || k < 1 || lda < (row ? k : m) || ldb < (row ? n : k) || ldc < (row ? n : m)) return false;
    const int sa = array_slot(spec, "a"), sb = array_slot(spec, "b"), sc = array_slot(spec, "c");
    if (sa < 0 || sb < 0 || sc < 0) return false;
    const auto& A = mem.regions.at(d.regions[sa]).data;
    const auto& B = mem.regions.at(d.regions[sb]).data;
    auto& Cr = mem.regions.at(d.regions[sc]).data;
    // last element each operand touches (row: i*lda+p; col: p*lda+i)
    if ((size_t)((m - 1) * (row ? lda : 1) + (k - 1) * (row ? 1 : lda)) >= A.size() ||
        (size_t)((k - 1) * (row ? ldb : 1) + (n - 1) * (row ? 1 : ldb)) >= B.size() ||
        (size_t)((m - 1) * (row ? ldc : 1) + (n - 1) * (row ? 1 : ldc)) >= Cr.size())
      return false;
    std::vector<float> a((size_t)(m * k)), b((size_t)(k * n)), c((size_t)(m * n));
    for (long long i = 0; i < m; ++i)
      for (long long p = 0; p < k; ++p) a[(size_t)(i * k + p)] = (float)A[(size_t)(row ? i * lda + p : p * lda + i)];
    for (long long p = 0; p < k; ++p)
      for (long long j = 0; j < n; ++j) b[(size_t)(p * n + j)] = (float)B[(size_t)(row ? p * ldb + j : j * ldb + p)];
    if (atc_sgemm_rm(ctx, a.data(), b.data(), c.data(), m, n, k, precision) != ATC_OK)
      throw std::runtime_error(atc_last_error(ctx));
    for (long long i = 0; i < m; ++i)
      for (long long j = 0; j < n; ++j) Cr[(size_t)(row ? i * ldc + j : j * ldc + i)] = (double)c[(size_t)(i * n + j)];
    return true;
  }
  // equivalence.cpp:66-93; the backend takes valid padding, unit stride, C % 32 == 0
  const long long n = role_size(spec, S, "n", 0), c = role_size(spec, S, "c", 0), h = role_size(spec, S, "h", 0),
                  w = role_size(spec, S, "w", 0), k = role_size(spec, S, "k", 0), r = role_size(spec, S, "r", 0),
                  s = role_size(spec, S, "s", 0);
  const long long oh = role_size(spec, S, "oh", h - r + 1), ow = role_size(spec, S, "ow", w - s + 1);
  if (n < 1 || c < 1 || k < 1 || r < 1 || s < 1 || oh != h - r + 1 || ow != w - s + 1 || oh < 1 || ow < 1 ||
      c % 32 != 0)
    return false;
  const int si = array_slot(spec, "in"), sw = array_slot(spec, "weights"), so = array_slot(spec, "out");
  if (si < 0 || sw < 0 || so < 0) return false;
  const auto& In = mem.regions.at(d.regions[si]).data;
  const auto& Wt = mem.regions.at(d.regions[sw]).data;
  auto& Out = mem.regions.at(d.regions[so]).data;
  const size_t nin = (size_t)(n * c * h * w), nw = (size_t)(k * c * r * s), nout = (size_t)(n * k * oh * ow);
  if (In.size() < nin || Wt.size() < nw || Out.size() < nout) return false;
  std::vector<float> x(In.begin(), In.begin() + nin), wt(Wt.begin(), Wt.begin() + nw), out(nout);
  if (atc_conv2d_nchw(ctx, x.data(), wt.data(), out.data(), n, c, h, w, k, r, s, precision) != ATC_OK)
    throw std::runtime_error(atc_last_error(ctx));
  for (size_t i = 0; i < nout; ++i) Out[i] = (double)out[i];
  return true;
}

}  // namespace

std::string p2_detail(atc_ctx* ctx, const RecordedTests& r, const minilang::FunctionIR& f,
                      const api::ApiSpec& spec, const matching::CandidateBinding& b, int t, int reason) {
  if (reason == ATC_FAIL_TESTSET) return r.test_detail[t];
  if (reason == ATC_FAIL_UB) return "access outside a region at test " + std::to_string(t);  // no reference text (UB)
  const size_t nP = r.ptr_params.size(), nI = r.int_params.size();
  auto ptr_index = [&](const std::string& u) {
    return (size_t)(std::find(r.ptr_params.begin(), r.ptr_params.end(), u) - r.ptr_params.begin());
  };
  const auto arrays = spec.arrays();
  const auto sizes = spec.size_params();
  std::vector<int64_t> sz(sizes.size());
  for (size_t q = 0; q < sizes.size(); ++q) {
    const std::string& u = b.sizes.at(sizes[q]->name);
    const size_t i = (size_t)(std::find(r.int_params.begin(), r.int_params.end(), u) - r.int_params.begin());
    sz[q] = r.ints[(size_t)t * nI + i];
  }
  // the lifted run is the single dispatch call of rewriter::rewrite (rewriter.cpp:80-91)
  // on the probe image: full-region copies, run_reference, f32 write-back
  std::vector<std::vector<double>> bufs;
  std::vector<double*> ptrs;
  std::vector<int64_t> lens;
  std::vector<int32_t> f32;
  for (const auto* ap : arrays) bufs.push_back(r.init[(size_t)t * nP + ptr_index(b.arrays.at(ap->name))]);
  for (size_t a = 0; a < arrays.size(); ++a) {
    ptrs.push_back(bufs[a].data());
    lens.push_back((int64_t)bufs[a].size());
    f32.push_back(r.is_f32[ptr_index(b.arrays.at(arrays[a]->name))]);
  }
  const atc_spec_desc desc = encode_spec(spec);
  const int rc = atc_dispatch(ctx, &desc, sz.data(), ptrs.data(), lens.data(), f32.data());
  if (rc == ATC_ERR_DISPATCH) return "dispatch failed: " + dispatch_error_text(spec, atc_last_error(ctx));
  if (rc != ATC_OK) throw std::runtime_error(atc_last_error(ctx));
  // rewriter.cpp:264-279: bound arrays in binding order, LiveIn skipped, full regions
  for (const auto& [api_arr, user_arr] : b.arrays) {
    const api::ApiParam* ap = spec.find(api_arr);
    if (!ap || ap->liveness == api::Liveness::LiveIn) continue;
    size_t a = 0;
    while (a < arrays.size() && arrays[a]->name != api_arr) ++a;
    const auto& want = r.fin[(size_t)t * nP + ptr_index(user_arr)];
    const auto& have = bufs[a];
    const bool is32 = f.find_param(user_arr)->elem == minilang::ScalarType::F32;
    const double rel = is32 ? 1e-4 : 1e-9, abs = is32 ? 1e-6 : 1e-12;
    for (size_t i = 0; i < want.size(); ++i)
      if (std::fabs(have[i] - want[i]) > abs + rel * std::fabs(want[i]))
        return "mismatch on " + user_arr + "[" + std::to_string(i) + "]: original " + std::to_string(want[i]) +
               ", lifted " + std::to_string(have[i]);
  }
  return "";  // the GPU and this recomputation disagree: never expected
}

CandidateLoop candidate_loop(atc_ctx* ctx, const minilang::Program& prog, const analysis::AnalyzedFunction& fn,
                             const std::string& function, const std::vector<const api::ApiSpec*>& specs,
                             const api::SizeRules& rules, uint64_t fseed, const LoopConfig& cfg,
                             std::chrono::steady_clock::time_point start) {
  CandidateLoop out;
  const auto t_all = std::chrono::steady_clock::now();
  const minilang::FunctionIR* f = prog.find(function);
  if (!f) throw std::invalid_argument("no function " + function);
  // matching + ranking per spec (pipeline.cpp:228-240), all up front: their P2
  // verdicts come from one batched GPU evaluation
  std::vector<matching::RankResult> ranked(specs.size());
  std::vector<pipeline::SpecCandidates> sc(specs.size());
  const size_t user_ptrs = fn.arrays.size();
  for (size_t s = 0; s < specs.size(); ++s) {
    sc[s].api = specs[s]->name;
    sc[s].raw = matching::raw_candidate_count(user_ptrs, specs[s]->arrays().size(), fn.int_params.size(),
                                              specs[s]->size_params().size());
    auto found = matching::find_matchings(fn, *specs[s]);
    sc[s].filtered = found.size();
    ranked[s] = matching::rank_candidates(std::move(found), cfg.max_candidates);
    sc[s].kept = ranked[s].ranked.size();
    sc[s].truncated = ranked[s].truncated;
    for (size_t i = 0; i < ranked[s].ranked.size() && i < 10; ++i) sc[s].top.push_back(ranked[s].ranked[i]);
  }
  std::vector<const api::ApiSpec*> eval_specs;
  std::vector<const std::vector<matching::CandidateBinding>*> lists;
  std::vector<int> slot(specs.size(), -1);
  for (size_t s = 0; s < specs.size(); ++s)
    if (!ranked[s].truncated && !ranked[s].ranked.empty()) {
      slot[s] = (int)eval_specs.size();
      eval_specs.push_back(specs[s]);
      lists.push_back(&ranked[s].ranked);
    }
  RecordedTests rec;
  std::vector<SpecVerdicts> p2;
  size_t total = 0;
  for (const auto* l : lists) total += l->size();
  // P2 for every spec's list in one GPU batch: up front for long lists (P1 then runs
  // only on P2 survivors), on demand for short ones — there the reference's order (P1
  // first, P2 when P1 says Equivalent, pipeline.cpp:257-277) costs less, since a P1
  // rejection on the host VM is cheaper than recording the test sets
  const bool lazy = total <= cfg.lazy_p2_max;
  auto ensure_p2 = [&] {
    if (!p2.empty() || eval_specs.empty()) return;
    auto t0 = std::chrono::steady_clock::now();
    rec = record_tests(prog, function, rules, Rng::mix(fseed, "post"), cfg.verify_tests);  // pipeline.cpp:277
    out.record_ms = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    p2 = p2_verdicts(ctx, rec, eval_specs, lists);
    out.gpu_ms = ms_since(t0);
  };
  if (!lazy) ensure_p2();
  // pipeline.cpp:241-309 (P1 = check_equivalence on the host VM, host_phases.hpp)
  const HostVm vm(prog);
  bool too_many = false;
  const auto t_p1 = std::chrono::steady_clock::now();
  for (size_t s = 0; s < specs.size(); ++s) {
    out.by_spec.push_back(sc[s]);
    if (ranked[s].truncated) {
      too_many = true;
      continue;
    }
    const auto& list = ranked[s].ranked;
    for (size_t i = 0; i < list.size(); ++i) {
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count() > cfg.budget_sec) {
        too_many = true;
        out.status_detail = "per-function budget exhausted";
        break;
      }
      const auto& cand = list[i];
      if (!lazy && p2[slot[s]].reason[i] != ATC_PASS && !cfg.report) continue;  // P1 cannot make it the winner
      const auto t0 = std::chrono::steady_clock::now();
      equivalence::EquivalenceConfig ec;
      ec.tests = cfg.tests;
      ec.seed = fseed;
      auto er = check_equivalence(vm, prog, fn, cand, *specs[s], rules, ec);
      ++out.p1_calls;
      pipeline::CandidateOutcome co;
      co.api = specs[s]->name;
      co.rank = (int)i;
      co.binding = cand;
      co.verdict = equivalence::verdict_name(er.verdict);
      co.detail = er.detail;
      co.equiv_ms = ms_since(t0);
      if (er.verdict == equivalence::Verdict::Equivalent) {
        ensure_p2();
        const bool p2_ok = p2[slot[s]].reason[i] == ATC_PASS;
        try {
          out.rewrite = rewriter::rewrite(prog, function, cand, *specs[s]);
        } catch (const std::exception& e) {
          co.verdict = "VerificationFailed";
          co.detail = std::string("rewrite: ") + e.what();
          out.evaluated.push_back(std::move(co));
          continue;
        }
        if (!out.rewrite.manifest.warnings.empty()) {
          // rewrite skipped (already a single dispatch call, rewriter.cpp:75-79): the
          // "lifted" program is the original, so P2 is the reference's own check of it
          auto vr = rewriter::verify_rewrite(prog, out.rewrite.program, function, cand, *specs[s], rules,
                                             Rng::mix(fseed, "post"), cfg.verify_tests);
          if (!vr.ok) {
            co.verdict = "VerificationFailed";
            co.detail = vr.detail;
            out.evaluated.push_back(std::move(co));
            continue;
          }
        } else if (!p2_ok) {
          co.verdict = "VerificationFailed";
          co.detail = p2_detail(ctx, rec, *f, *specs[s], cand, p2[slot[s]].fail_t[i], p2[slot[s]].reason[i]);
          out.evaluated.push_back(std::move(co));
          continue;
        }
        out.status = pipeline::FunctionStatus::Lifted;
        out.winning_spec = specs[s];
        out.winner_rank = (int)i;
        out.evaluated.push_back(std::move(co));
        break;
      }
      out.evaluated.push_back(std::move(co));
    }
    if (out.status == pipeline::FunctionStatus::Lifted || too_many) break;
  }
  out.p1_ms = ms_since(t_p1);
  // pipeline.cpp:318-329
  if (out.status != pipeline::FunctionStatus::Lifted) {
    if (too_many) {
      out.status = pipeline::FunctionStatus::TooManyCandidates;
      if (out.status_detail.empty()) out.status_detail = "candidate cap exceeded";
    } else {
      bool any_filtered = false;
      for (const auto& b : out.by_spec) any_filtered |= b.filtered > 0;
      out.status_detail = any_filtered ? "no candidate proved equivalent" : "no candidate passed the constraints";
    }
  }
  out.total_ms = ms_since(t_all);
  return out;
}

interp::DispatchContext make_gpu_dispatch(const api::ApiSpec& spec, atc_ctx* ctx) {
  interp::DispatchContext dc;
  const atc_spec_desc desc = encode_spec(spec);
  dc.handler = [spec, desc, ctx](const std::string& name, const std::vector<interp::DispatchArg>& args,
                                 interp::MemoryImage& mem) {
    exact_dispatch(spec, desc, ctx, decode_call(spec, name, args, mem), mem);
  };
  return dc;
}

std::vector<long long> routed_sizes(const api::ApiSpec& spec, const std::map<std::string, long long>& sizes) {
  // rewriter.cpp:194-205: conv as its im2col GEMM (filters x batch*out positions, depth c*r*s)
  if (spec.semantics == "conv2d")
    return {role_size(spec, sizes, "k"),
            role_size(spec, sizes, "n") * role_size(spec, sizes, "oh") * role_size(spec, sizes, "ow"),
            role_size(spec, sizes, "c") * role_size(spec, sizes, "r") * role_size(spec, sizes, "s")};
  return {role_size(spec, sizes, "m"), role_size(spec, sizes, "n"), role_size(spec, sizes, "k")};
}

interp::DispatchContext make_gpu_routed_dispatch(const api::ApiSpec& spec, atc_ctx* ctx,
                                                 const profitability::SvmModel* model,
                                                 std::vector<std::string>* choices, int32_t precision) {
  interp::DispatchContext dc;
  const atc_spec_desc desc = encode_spec(spec);
  dc.handler = [spec, desc, ctx, model, choices, precision](const std::string& name,
                                                             const std::vector<interp::DispatchArg>& args,
                                                             interp::MemoryImage& mem) {
    // rewriter.cpp:190-209: the label comes first, from an arity-clipped decode of
    // the size slots (so a call run_dispatch then rejects is still labelled)
    bool xpu = false;
    if (model && choices) {
      std::map<std::string, long long> sizes;
      for (size_t i = 0; i < spec.params.size() && i < args.size(); ++i)
        if (spec.params[i].kind == api::ApiParamKind::IntSize) sizes[spec.params[i].name] = args[i].i;
      xpu = profitability::predict_backend(*model, routed_sizes(spec, sizes)) == 1;
      choices->push_back(xpu ? "xpu" : "cpu");
    } else if (choices) {
      choices->push_back("cpu");
    }
    const DecodedCall d = decode_call(spec, name, args, mem);
    if (xpu && precision != kRouteExact && tensor_dispatch(spec, ctx, precision, d, mem)) return;
    exact_dispatch(spec, desc, ctx, d, mem);
  };
  return dc;
}

profitability::TimingSample sample_one_b200(atc_ctx* ctx, const std::vector<long long>& sizes, int reps,
                                            int32_t precision, double xpu_overhead_sec) {
  if (sizes.size() != 3) throw std::invalid_argument("expected sizes m, n, k");  // profitability.cpp:66-69
  if (reps < 3) throw std::invalid_argument("need at least 3 repetitions");
  const long long m = sizes[0], n = sizes[1], k = sizes[2];
  if (m < 1 || n < 1 || k < 1) throw std::invalid_argument("sizes must be positive");
  std::vector<float> a((size_t)(m * k)), b((size_t)(k * n)), c_cpu((size_t)(m * n)), c_xpu((size_t)(m * n));
  for (size_t i = 0; i < a.size(); ++i) a[i] = 0.25f + (float)(i % 17) * 0.0625f;  // :73-74
  for (size_t i = 0; i < b.size(); ++i) b[i] = -0.5f + (float)(i % 23) * 0.0625f;
  auto xpu = [&](float* out) {
    if (atc_sgemm_rm(ctx, a.data(), b.data(), out, m, n, k, precision) != ATC_OK)
      throw profitability::BackendFailure(std::string("B200 backend: ") + atc_last_error(ctx));
  };
  profitability::cpu_gemm(a.data(), b.data(), c_cpu.data(), m, n, k);  // verification pass (:76-85)
  xpu(c_xpu.data());
  for (size_t i = 0; i < c_cpu.size(); ++i) {
    if (!std::isfinite(c_cpu[i]) || !std::isfinite(c_xpu[i]))
      throw profitability::BackendFailure("non-finite backend output");
    if (std::fabs((double)c_cpu[i] - (double)c_xpu[i]) > 1e-3 * (1.0 + std::fabs((double)c_cpu[i])))
      throw profitability::BackendFailure("backend results disagree");
  }
  auto median_sec = [&](auto&& fn, float* out) {  // :87-99
    std::vector<double> times;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      fn(out);
      times.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(times.begin(), times.end());
    return times[times.size() / 2];
  };
  profitability::TimingSample s;
  s.sizes = sizes;
  s.t_cpu = median_sec([&](float* out) { profitability::cpu_gemm(a.data(), b.data(), out, m, n, k); },
                       c_cpu.data());
  s.t_xpu = median_sec(xpu, c_xpu.data()) + xpu_overhead_sec;
  s.label = s.t_xpu < s.t_cpu ? 1 : 0;
  return s;
}

std::vector<profitability::TimingSample> sample_timings_b200(atc_ctx* ctx,
                                                             const std::vector<std::vector<long long>>& grid,
                                                             int reps, int32_t precision, double xpu_overhead_sec) {
  if (grid.empty()) throw std::invalid_argument("empty size grid");
  std::vector<profitability::TimingSample> out;
  for (const auto& sizes : grid) out.push_back(sample_one_b200(ctx, sizes, reps, precision, xpu_overhead_sec));
  return out;
}

}  // namespace liftc::gpu
