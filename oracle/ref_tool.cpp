// ref_tool — drives the UNMODIFIED reference (liftc_core, built into
// oracle/_ref/ by oracle/Makefile). TEST INFRASTRUCTURE ONLY: it generates the
// golden fixtures under tests/golden/ and times the reference's CPU path for
// bench.py's reference arm / cpu_baseline. It is never on the product path.
//
// Subcommands
//   golden <outdir>                 dump pipeline reports, P2 test sets, and per-binding
//                                   P1/P2 verdicts for every GEMM/conv corpus program
//   time-p2  <stem> <spec> <T> <budget_s> <threads> [rules64]
//   time-acc <stem> <spec> <T> <budget_s> <threads> [rules64]
//   svm-golden <out.json>           profitability::train_svm on rewriter_test.cpp:109-118's
//                                   volume-labelled set, save_svm's JSON, and
//                                   decision_value / predict_backend over a feature grid
//   time-xpu-gemm <m> <n> <k>       profitability::xpu_gemm (hardware_concurrency threads)
//   time-cpu-gemm <m> <n> <k> <rows> profitability::cpu_gemm over a `rows`-row M slice
//   time-conv <n> <c> <h> <w> <k> <r> <s>   equivalence::run_reference (conv2d, f64)
//
// Reference anchors: the per-function analysis replicates pipeline.cpp:131-221,
// the bench driver replicates tools/liftc.cpp:271-330, P1 is
// equivalence::check_equivalence (equivalence.cpp:141-379) called exactly as
// pipeline.cpp:257-261 does, and P2 is rewriter::verify_rewrite
// (rewriter.cpp:215-284) called as pipeline.cpp:274-277 does.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <mutex>
#include <set>
#include <sstream>
#include <thread>

#include <json.hpp>

#include "liftc/analysis.hpp"
#include "liftc/api_spec.hpp"
#include "liftc/classifier.hpp"
#include "liftc/equivalence.hpp"
#include "liftc/interp.hpp"
#include "liftc/matching.hpp"
#include "liftc/minilang.hpp"
#include "liftc/pipeline.hpp"
#include "liftc/profitability.hpp"
#include "liftc/rewriter.hpp"
#include "liftc/rng.hpp"

extern const std::map<std::string, std::string>& embedded_files();

using namespace liftc;
using json = nlohmann::json;

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

const std::string& file_text(const std::string& key) {
  auto it = embedded_files().find(key);
  if (it == embedded_files().end()) throw std::runtime_error("no embedded file " + key);
  return it->second;
}

std::vector<api::ApiSpec> default_specs() {  // tools/liftc.cpp:57-66 order
  std::vector<api::ApiSpec> specs;
  for (const char* n : {"gemm_rowmajor", "gemm_colmajor", "gemm_rowmajor_ld", "conv2d"})
    specs.push_back(api::parse_api_spec(file_text(std::string("specs/") + n + ".json")));
  return specs;
}

const api::ApiSpec& spec_named(const std::vector<api::ApiSpec>& specs, const std::string& n) {
  for (const auto& s : specs)
    if (s.name == n) return s;
  throw std::runtime_error("no spec " + n);
}

struct CorpusFile {
  std::string key;   // corpus/gemm/naive_ld.ml
  std::string tag;   // naive_ld.ml
  std::string stem;  // naive_ld
  std::string dir;   // gemm
  json sidecar;      // raw sidecar json (or null)
};

std::vector<CorpusFile> corpus_files() {
  std::vector<CorpusFile> out;
  for (const auto& [k, v] : embedded_files()) {
    if (k.rfind("corpus/", 0) != 0 || k.size() < 3 || k.substr(k.size() - 3) != ".ml") continue;
    CorpusFile f;
    f.key = k;
    f.tag = k.substr(k.rfind('/') + 1);
    f.stem = f.tag.substr(0, f.tag.size() - 3);
    f.dir = k.substr(7, k.rfind('/') - 7);
    std::string side = k.substr(0, k.size() - 3) + ".json";
    auto it = embedded_files().find(side);
    if (it != embedded_files().end()) f.sidecar = json::parse(it->second);
    out.push_back(std::move(f));
  }
  // tools/liftc.cpp:69-75 sorts full paths; embedded keys sort the same way
  // within one corpus root (conv < gemm < nonidiom).
  return out;
}

pipeline::FixtureMeta meta_of(const CorpusFile& f) {
  if (f.sidecar.is_null()) return {};
  return pipeline::parse_fixture_meta(f.sidecar.dump());
}

classifier::ClassifierModel corpus_classifier() {  // tools/liftc.cpp:92-106
  std::vector<std::pair<classifier::FeatureVector, std::string>> ex;
  for (const auto& f : corpus_files()) {
    auto meta = meta_of(f);
    if (meta.function.empty() || meta.label.empty()) continue;
    try {
      auto prog = minilang::parse_program(file_text(f.key));
      const auto* fn = prog.find(meta.function);
      if (fn) ex.emplace_back(classifier::extract_features(prog, *fn), meta.label);
    } catch (const std::exception&) {
    }
  }
  return classifier::train_classifier(ex);
}

// pipeline.cpp:164-221, for one function, against the specs of its label.
analysis::AnalyzedFunction analyze(const minilang::Program& prog, const std::string& function,
                                   const pipeline::FixtureMeta& meta, uint64_t fseed,
                                   const std::vector<const api::ApiSpec*>& specs) {
  const auto* f = prog.find(function);
  auto live = analysis::detect_liveness(prog, *f, fseed, meta.rules);
  analysis::AnalyzedFunction fn;
  fn.name = function;
  for (const auto& p : f->params) {
    if (p.kind == minilang::ParamKind::IntScalar) fn.int_params.push_back(p.name);
    if (p.kind == minilang::ParamKind::FloatScalar) fn.float_params.push_back(p.name);
  }
  int max_rank = meta.max_rank;
  for (const auto* s : specs)
    if (!meta.max_rank) max_rank = std::max(max_rank, s->max_rank());
  auto probe_values = analysis::assign_probe_values(fn.int_params, meta.rules, meta.probes, 0);
  for (const auto& p : f->params) {
    if (p.kind != minilang::ParamKind::Pointer) continue;
    analysis::ArrayInfo info;
    info.name = p.name;
    info.elem = p.elem;
    info.liveness = live.classes.at(p.name);
    try {
      auto d = analysis::detect_dims(prog, *f, p.name, fn.int_params, probe_values, max_rank);
      info.has_dims = true;
      info.dims = d.dims;
      info.slow_dim = d.slow_dim;
    } catch (const analysis::NoDimsFound&) {
      info.has_dims = false;
    }
    fn.arrays.push_back(std::move(info));
  }
  return fn;
}

// SURVEY.md Appendix C canonical enumeration of the unpruned binding space.
struct Space {
  std::vector<std::string> user_ptrs, user_ints, api_arrays, api_sizes;
  std::vector<std::vector<int>> perms;  // odometer (DFS) order, matching.cpp:141-194 unfiltered
  unsigned long long size_maps = 1;

  Space(const analysis::AnalyzedFunction& fn, const api::ApiSpec& spec) {
    for (const auto& a : fn.arrays) user_ptrs.push_back(a.name);
    user_ints = fn.int_params;
    for (const auto* p : spec.arrays()) api_arrays.push_back(p->name);
    for (const auto* p : spec.size_params()) api_sizes.push_back(p->name);
    std::vector<int> sel(api_arrays.size());
    std::vector<bool> used(user_ptrs.size(), false);
    std::function<void(size_t)> rec = [&](size_t i) {
      if (i == api_arrays.size()) {
        perms.push_back(sel);
        return;
      }
      for (size_t j = 0; j < user_ptrs.size(); ++j) {
        if (used[j]) continue;
        used[j] = true;
        sel[i] = (int)j;
        rec(i + 1);
        used[j] = false;
      }
    };
    if (api_arrays.size() <= user_ptrs.size()) rec(0);
    for (size_t q = 0; q < api_sizes.size(); ++q) size_maps *= user_ints.size();
  }
  unsigned long long count() const { return perms.size() * size_maps; }
  // inverse of binding(): global index of a complete binding
  unsigned long long index_of(const matching::CandidateBinding& b) const {
    std::vector<int> sel;
    for (const auto& a : api_arrays) {
      const std::string& u = b.arrays.at(a);
      sel.push_back((int)(std::find(user_ptrs.begin(), user_ptrs.end(), u) - user_ptrs.begin()));
    }
    unsigned long long p = (unsigned long long)(std::find(perms.begin(), perms.end(), sel) - perms.begin());
    unsigned long long s = 0, mul = 1;
    for (const auto& a : api_sizes) {
      const std::string& u = b.sizes.at(a);
      s += (unsigned long long)(std::find(user_ints.begin(), user_ints.end(), u) - user_ints.begin()) * mul;
      mul *= user_ints.size();
    }
    return p * size_maps + s;
  }
  matching::CandidateBinding binding(unsigned long long idx) const {
    matching::CandidateBinding b;
    const auto& perm = perms[idx / size_maps];
    unsigned long long s = idx % size_maps;
    for (size_t i = 0; i < api_arrays.size(); ++i) b.arrays[api_arrays[i]] = user_ptrs[perm[i]];
    for (size_t q = 0; q < api_sizes.size(); ++q) {
      b.sizes[api_sizes[q]] = user_ints[s % user_ints.size()];
      s /= user_ints.size();
    }
    return b;
  }
};

struct P2Out {
  int8_t fail_t = -1;  // -1 = passed every test
  int8_t reason = 0;   // 0 pass, 1 mismatch, 2 dispatch failed, 3 other
};

P2Out run_p2(const minilang::Program& prog, const std::string& function,
             const matching::CandidateBinding& b, const api::ApiSpec& spec,
             const api::SizeRules& rules, uint64_t p2seed, int tests) {
  P2Out o;
  rewriter::RewriteResult rr = rewriter::rewrite(prog, function, b, spec);
  auto vr = rewriter::verify_rewrite(prog, rr.program, function, b, spec, rules, p2seed, tests);
  if (vr.ok) return o;
  // rewriter.cpp:272-276 sets tests_run = t+1 on a mismatch; the dispatch
  // failure path (:255-257) returns with tests_run == t.
  if (vr.detail.rfind("mismatch", 0) == 0) {
    o.reason = 1;
    o.fail_t = (int8_t)(vr.tests_run - 1);
  } else if (vr.detail.rfind("dispatch failed", 0) == 0) {
    o.reason = 2;
    o.fail_t = (int8_t)vr.tests_run;
  } else {
    o.reason = 3;
    o.fail_t = (int8_t)vr.tests_run;
  }
  return o;
}

int8_t run_p1(const minilang::Program& prog, const analysis::AnalyzedFunction& fn,
              const matching::CandidateBinding& b, const api::ApiSpec& spec,
              const api::SizeRules& rules, uint64_t fseed, std::string* detail = nullptr) {
  equivalence::EquivalenceConfig ec;  // pipeline.cpp:257-259
  ec.tests = 30;
  ec.seed = fseed;
  auto er = equivalence::check_equivalence(prog, fn, b, spec, rules, ec);
  if (detail) *detail = er.detail;
  return er.verdict == equivalence::Verdict::Equivalent      ? 0
         : er.verdict == equivalence::Verdict::NotEquivalent ? 1
                                                             : 2;
}

void parallel_for(size_t n, int threads, const std::function<void(size_t)>& fn) {
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t i = next.fetch_add(1); i < n; i = next.fetch_add(1)) fn(i);
  };
  std::vector<std::thread> pool;
  for (int w = 0; w < threads; ++w) pool.emplace_back(work);
  for (auto& t : pool) t.join();
}

int hw_threads() {
  unsigned h = std::thread::hardware_concurrency();
  return h == 0 ? 1 : (int)h;
}

std::string hexbits(double v) {
  uint64_t u;
  std::memcpy(&u, &v, 8);
  char buf[32];
  std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)u);
  return buf;
}

uint64_t fnv1a(const std::vector<double>& v) {
  uint64_t h = 1469598103934665603ULL;
  const unsigned char* p = reinterpret_cast<const unsigned char*>(v.data());
  for (size_t i = 0; i < v.size() * 8; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

struct BinWriter {
  std::ofstream out;
  size_t off = 0;
  explicit BinWriter(const std::string& path) : out(path, std::ios::binary) {
    if (!out) throw std::runtime_error("cannot write " + path);
  }
  template <typename T>
  json put(const std::vector<T>& v) {
    json j = {{"offset", off}, {"count", v.size()}};
    out.write(reinterpret_cast<const char*>(v.data()), (std::streamsize)(v.size() * sizeof(T)));
    off += v.size() * sizeof(T);
    return j;
  }
};

// The binding-independent half of verify_rewrite (rewriter.cpp:235-251) for
// t = 0..tests-1: sizes, probe image, and the original run's final regions.
json dump_testsets(const minilang::Program& prog, const std::string& function,
                   const api::SizeRules& rules, uint64_t p2seed, int tests, BinWriter& bin) {
  const auto* f = prog.find(function);
  std::vector<std::string> int_params;
  for (const auto& p : f->params)
    if (p.kind == minilang::ParamKind::IntScalar) int_params.push_back(p.name);
  json sets = json::array();
  for (int t = 0; t < tests; ++t) {
    json js;
    js["t"] = t;
    Rng rng(Rng::mix(p2seed, "verify:" + function + ":" + std::to_string(t)));
    std::map<std::string, long long> sizes;
    bool drawn = false;
    int tries = 0;
    for (; tries < 20 && !drawn; ++tries) drawn = analysis::draw_sizes(int_params, rules, rng, sizes);
    js["draw_tries"] = tries;
    if (!drawn) {
      js["status"] = "draw_failed";
      sets.push_back(js);
      continue;
    }
    js["sizes"] = sizes;
    interp::MemoryImage img = analysis::build_probe_image(*f, sizes, rng);
    json fl = json::object();
    for (const auto& [k, v] : img.float_args) fl[k] = hexbits(v);
    js["floats"] = fl;
    interp::InstrumentationPolicy plain;
    auto ref = interp::execute(prog, function, img, plain);
    js["status"] = interp::status_name(ref.status);
    json regions = json::object();
    for (const auto& [name, reg] : img.regions) {
      json jr;
      jr["len"] = reg.data.size();
      jr["init_fnv"] = std::to_string(fnv1a(reg.data));
      jr["init_head"] = {hexbits(reg.data[0]), hexbits(reg.data[1]), hexbits(reg.data[2]),
                         hexbits(reg.data[3])};
      if (ref.status == interp::ExecStatus::Normal) {
        const auto& fin = ref.final.regions.at(name).data;
        std::vector<int64_t> pos;
        std::vector<double> val;
        for (size_t i = 0; i < fin.size(); ++i)
          if (std::memcmp(&fin[i], &reg.data[i], 8) != 0) {
            pos.push_back((int64_t)i);
            val.push_back(fin[i]);
          }
        jr["diff_pos"] = bin.put(pos);
        jr["diff_val"] = bin.put(val);
        jr["final_fnv"] = std::to_string(fnv1a(fin));
      }
      regions[name] = jr;
    }
    js["regions"] = regions;
    sets.push_back(js);
  }
  return sets;
}

json binding_json(const matching::CandidateBinding& b) {
  return {{"arrays", b.arrays}, {"sizes", b.sizes}, {"scalars", b.scalars},
          {"lex_score", b.lex_score}, {"provenance", b.provenance}};
}

std::string elem_name(minilang::ScalarType t) {
  return t == minilang::ScalarType::F32 ? "f32" : t == minilang::ScalarType::F64 ? "f64" : "i64";
}

// Indices sampled from spaces too large to sweep with the reference.
std::vector<unsigned long long> sample_indices(const Space& sp, uint64_t seed) {
  std::set<unsigned long long> s;
  Rng rng(seed);
  const unsigned long long n = sp.count();
  while (s.size() < 3000) s.insert(rng.next() % n);
  // the identity perm (if any) and every perm with the identity size map,
  // plus single- and double-slot perturbations of the identity size map.
  const size_t nI = sp.user_ints.size(), nS = sp.api_sizes.size();
  unsigned long long ident = 0, mul = 1;
  for (size_t q = 0; q < nS; ++q) {
    ident += (unsigned long long)(q % nI) * mul;
    mul *= nI;
  }
  for (size_t p = 0; p < sp.perms.size(); ++p) {
    s.insert(p * sp.size_maps + ident);
    if (p != 0) continue;
    unsigned long long pw_q = 1;
    for (size_t q = 0; q < nS; ++q, pw_q *= nI) {
      for (size_t v = 0; v < nI; ++v) {
        unsigned long long base = ident - (q % nI) * pw_q + v * pw_q;
        s.insert(base);
        unsigned long long pw_r = 1;
        for (size_t r = 0; r < q; ++r, pw_r *= nI)
          for (size_t w = 0; w < nI; ++w) s.insert(base - (r % nI) * pw_r + w * pw_r);
      }
    }
  }
  return {s.begin(), s.end()};
}

json spec_json(const api::ApiSpec& s) {
  json j;
  j["name"] = s.name;
  j["semantics"] = s.semantics;
  j["layout"] = s.layout == api::Layout::RowMajor ? "rowmajor" : "colmajor";
  j["affix"] = s.affix;
  json params = json::array();
  for (const auto& p : s.params) {
    json jp;
    jp["name"] = p.name;
    jp["kind"] = p.kind == api::ApiParamKind::Array     ? "array"
                 : p.kind == api::ApiParamKind::IntSize ? "int"
                                                        : "float";
    jp["liveness"] = api::liveness_name(p.liveness);
    jp["dims"] = p.dims;  // canonical order (api_spec.cpp:116-119)
    jp["element_type"] = p.element_type;
    jp["role"] = p.role;
    params.push_back(jp);
  }
  j["params"] = params;
  json ranges = json::object();
  for (const auto& [k, v] : s.ranges) ranges[k] = {v.first, v.second};
  j["ranges"] = ranges;
  json derived = json::object();
  for (const auto& [k, d] : s.derived) {
    json terms = json::array();
    for (const auto& [c, n] : d.terms) terms.push_back({c, n});
    derived[k] = {{"terms", terms}, {"constant", d.constant}, {"slack", d.slack_max}};
  }
  j["derived"] = derived;
  return j;
}

int cmd_golden(const std::string& outdir) {
  const int threads = hw_threads();
  auto specs = default_specs();
  auto model = corpus_classifier();

  json specs_out = json::object();
  for (const auto& s : specs) specs_out[s.name] = spec_json(s);
  std::ofstream(outdir + "/specs.json") << specs_out.dump(1) << "\n";

  // 1. the reference pipeline over the whole corpus, as `liftc bench` runs it
  pipeline::PipelineConfig cfg;
  cfg.specs = specs;
  cfg.classifier = &model;
  cfg.tests = 30;
  cfg.seed = 0;
  cfg.workers = 1;
  json reports = json::array();
  for (const auto& f : corpus_files()) {
    auto prog = minilang::parse_program(file_text(f.key));
    auto meta = meta_of(f);
    auto rep = pipeline::lift_program(prog, f.tag, meta, cfg, nullptr);
    json j = pipeline::mask_timings(pipeline::report_to_json(rep));
    j["corpus_dir"] = f.dir;
    j["function_of_interest"] = meta.function;
    j["expect_lift"] = meta.expect_lift;
    reports.push_back(j);
    std::fprintf(stderr, "[golden] pipeline %s\n", f.key.c_str());
  }
  std::ofstream(outdir + "/pipeline.json") << reports.dump(1) << "\n";

  // 2. per GEMM/conv program: test sets + per-binding verdicts
  json index = json::array();
  for (const auto& f : corpus_files()) {
    if (f.dir != "gemm" && f.dir != "conv") continue;
    auto prog = minilang::parse_program(file_text(f.key));
    auto meta = meta_of(f);
    std::string function = meta.function.empty() ? prog.functions[0].name : meta.function;
    const auto* fir = prog.find(function);
    const uint64_t fseed = Rng::mix(0, f.tag + ":" + function);
    const uint64_t p2seed = Rng::mix(fseed, "post");
    const std::string label = f.dir == "gemm" ? "gemm" : "conv2d";
    std::vector<const api::ApiSpec*> lspecs;
    for (const auto& s : specs)
      if (s.semantics == label) lspecs.push_back(&s);

    json jp;
    jp["file"] = f.tag;
    jp["stem"] = f.stem;
    jp["corpus_dir"] = f.dir;
    jp["function"] = function;
    jp["fseed"] = std::to_string(fseed);
    jp["p2seed"] = std::to_string(p2seed);
    jp["size_rules"] = f.sidecar.is_null() || !f.sidecar.contains("size_rules")
                           ? json::object()
                           : f.sidecar["size_rules"];
    json params = json::array();
    for (const auto& p : fir->params)
      params.push_back({{"name", p.name},
                        {"kind", p.kind == minilang::ParamKind::Pointer       ? "ptr"
                                 : p.kind == minilang::ParamKind::IntScalar   ? "int"
                                                                              : "float"},
                        {"elem", elem_name(p.elem)}});
    jp["params"] = params;

    analysis::AnalyzedFunction fn;
    try {
      fn = analyze(prog, function, meta, fseed, lspecs);
    } catch (const std::exception& e) {
      jp["analysis_error"] = e.what();
      std::ofstream(outdir + "/" + f.stem + ".json") << jp.dump(1) << "\n";
      index.push_back(f.stem);
      continue;
    }
    json arrays = json::array();
    for (const auto& a : fn.arrays)
      arrays.push_back({{"name", a.name}, {"elem", elem_name(a.elem)},
                        {"liveness", api::liveness_name(a.liveness)},
                        {"has_dims", a.has_dims}, {"dims", a.dims}});
    jp["analysis"] = {{"arrays", arrays}, {"int_params", fn.int_params},
                      {"float_params", fn.float_params}};

    BinWriter bin(outdir + "/" + f.stem + ".bin");
    const int T = 16;
    jp["testsets"] = dump_testsets(prog, function, meta.rules, p2seed, T, bin);

    // config 1 variant: P2 draws pinned to 64x64x64 (BASELINE.json configs[0])
    api::SizeRules rules64 = meta.rules;
    bool want64 = f.stem == "naive_f32" || f.stem == "naive_rowmajor";
    if (want64) {
      for (const auto& u : fn.int_params) rules64.ranges[u] = {64, 64};
      jp["testsets64"] = dump_testsets(prog, function, rules64, p2seed, T, bin);
    }

    json jspecs = json::object();
    for (const auto* spec : lspecs) {
      json js;
      auto found = matching::find_matchings(fn, *spec);
      auto ranked = matching::rank_candidates(found, 100);
      json pruned = json::array();
      for (const auto& c : ranked.ranked) {
        std::string d1;
        int8_t p1 = run_p1(prog, fn, c, *spec, meta.rules, fseed, &d1);
        P2Out p2 = run_p2(prog, function, c, *spec, meta.rules, p2seed, T);
        json jc = binding_json(c);
        jc["p1"] = p1;
        jc["p1_detail"] = d1;
        jc["p2_fail_t"] = p2.fail_t;
        jc["p2_reason"] = p2.reason;
        pruned.push_back(jc);
      }
      js["pruned"] = pruned;
      js["filtered"] = found.size();
      js["truncated"] = ranked.truncated;

      Space sp(fn, *spec);
      js["raw"] = matching::raw_candidate_count(fn.arrays.size(), spec->arrays().size(),
                                                fn.int_params.size(), spec->size_params().size());
      js["count"] = sp.count();
      std::vector<unsigned long long> idx;
      bool full = sp.count() <= 400000ULL;
      if (full) {
        idx.resize(sp.count());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
      } else {
        idx = sample_indices(sp, Rng::mix(fseed, "sample:" + spec->name));
        std::set<unsigned long long> all(idx.begin(), idx.end());
        for (const auto& c : ranked.ranked) all.insert(sp.index_of(c));
        idx.assign(all.begin(), all.end());
      }
      json pruned_idx = json::array();
      for (const auto& c : ranked.ranked) pruned_idx.push_back(sp.index_of(c));
      js["pruned_index"] = pruned_idx;
      js["enumerated"] = full ? "full" : "sampled";
      std::vector<int8_t> p2t(idx.size()), p2r(idx.size()), p1v(idx.size());
      double t0 = now_s();
      parallel_for(idx.size(), threads, [&](size_t i) {
        auto b = sp.binding(idx[i]);
        P2Out o = run_p2(prog, function, b, *spec, meta.rules, p2seed, T);
        p2t[i] = o.fail_t;
        p2r[i] = o.reason;
        p1v[i] = run_p1(prog, fn, b, *spec, meta.rules, fseed);
      });
      std::fprintf(stderr, "[golden] %s x %s: %zu bindings in %.1fs\n", f.stem.c_str(),
                   spec->name.c_str(), idx.size(), now_s() - t0);
      std::vector<uint64_t> idx64(idx.begin(), idx.end());
      js["idx"] = bin.put(idx64);
      js["p2_fail_t"] = bin.put(p2t);
      js["p2_reason"] = bin.put(p2r);
      js["p1"] = bin.put(p1v);
      if (want64 && sp.count() <= 400000ULL) {
        std::vector<int8_t> t64(idx.size()), r64(idx.size());
        parallel_for(idx.size(), threads, [&](size_t i) {
          P2Out o = run_p2(prog, function, sp.binding(idx[i]), *spec, rules64, p2seed, T);
          t64[i] = o.fail_t;
          r64[i] = o.reason;
        });
        js["p2_64_fail_t"] = bin.put(t64);
        js["p2_64_reason"] = bin.put(r64);
      }
      jspecs[spec->name] = js;
    }
    jp["specs"] = jspecs;
    std::ofstream(outdir + "/" + f.stem + ".json") << jp.dump(1) << "\n";
    index.push_back(f.stem);
  }
  std::ofstream(outdir + "/index.json") << index.dump(1) << "\n";
  return 0;
}

struct ProgCtx {
  minilang::Program prog;
  pipeline::FixtureMeta meta;
  std::string function, tag;
  uint64_t fseed = 0, p2seed = 0;
  analysis::AnalyzedFunction fn;
};

ProgCtx load_prog(const std::string& stem, const std::vector<api::ApiSpec>& specs) {
  for (const auto& f : corpus_files()) {
    if (f.stem != stem) continue;
    ProgCtx c;
    c.prog = minilang::parse_program(file_text(f.key));
    c.meta = meta_of(f);
    c.function = c.meta.function.empty() ? c.prog.functions[0].name : c.meta.function;
    c.tag = f.tag;
    c.fseed = Rng::mix(0, f.tag + ":" + c.function);
    c.p2seed = Rng::mix(c.fseed, "post");
    std::vector<const api::ApiSpec*> ls;
    const std::string label = f.dir == "gemm" ? "gemm" : "conv2d";
    for (const auto& s : specs)
      if (s.semantics == label) ls.push_back(&s);
    c.fn = analyze(c.prog, c.function, c.meta, c.fseed, ls);
    return c;
  }
  throw std::runtime_error("no corpus program " + stem);
}

// Times the reference over the unpruned space in index order (wrapping),
// sharded round-robin over `threads`, until `budget` seconds elapse.
// mode p2  : verify_rewrite only (the predicate the GPU evaluates)
// mode acc : the reference acceptance decision, P1 then P2 on Equivalent
int cmd_time(const std::string& mode, const std::string& stem, const std::string& spec_name,
             int tests, double budget, int threads, bool rules64) {
  auto specs = default_specs();
  const auto& spec = spec_named(specs, spec_name);
  ProgCtx c = load_prog(stem, specs);
  api::SizeRules rules = c.meta.rules;
  if (rules64)
    for (const auto& u : c.fn.int_params) rules.ranges[u] = {64, 64};
  Space sp(c.fn, spec);
  std::atomic<unsigned long long> next{0}, done{0}, passed{0};
  const double t0 = now_s();
  auto work = [&] {
    for (;;) {
      if (now_s() - t0 > budget) break;
      // pseudo-random walk over the space (a fixed odd multiplier mod count),
      // so the sample is not biased towards the first permutation block
      unsigned long long i =
          (unsigned long long)(((unsigned __int128)next.fetch_add(1) * 0x9E3779B97F4A7C15ULL) % sp.count());
      auto b = sp.binding(i);
      bool ok;
      if (mode == "p2") {
        ok = run_p2(c.prog, c.function, b, spec, rules, c.p2seed, tests).fail_t < 0;
      } else {
        ok = run_p1(c.prog, c.fn, b, spec, c.meta.rules, c.fseed) == 0 &&
             run_p2(c.prog, c.function, b, spec, rules, c.p2seed, tests).fail_t < 0;
      }
      done.fetch_add(1);
      if (ok) passed.fetch_add(1);
    }
  };
  std::vector<std::thread> pool;
  for (int w = 0; w < threads; ++w) pool.emplace_back(work);
  for (auto& t : pool) t.join();
  const double dt = now_s() - t0;
  json j = {{"mode", mode}, {"stem", stem}, {"spec", spec_name}, {"tests", tests},
            {"threads", threads}, {"bindings", done.load()}, {"passed", passed.load()},
            {"seconds", dt}, {"bindings_per_s", done.load() / dt}, {"space", sp.count()}};
  std::cout << j.dump() << std::endl;
  return 0;
}

// The reference's own P2 verdicts (verify_rewrite: first failing test + reason)
// for every binding within `radius` of each given index of one unpruned space —
// the neighbourhoods of the passing bindings the GPU reports in spaces too large
// to sweep with the reference (tests/golden/conv_neighbourhoods.npz, made by
// oracle/gen_neighbourhoods.py).  Output: one JSON line with the sorted indices
// and the verdict arrays.
int cmd_neighbourhood(const std::string& stem, const std::string& spec_name, int tests, long long radius,
                      const std::vector<unsigned long long>& centers, int threads) {
  auto specs = default_specs();
  const auto& spec = spec_named(specs, spec_name);
  ProgCtx c = load_prog(stem, specs);
  Space sp(c.fn, spec);
  std::set<unsigned long long> all;
  for (unsigned long long ctr : centers)
    for (long long d = -radius; d <= radius; ++d) {
      const long long i = (long long)ctr + d;
      if (i >= 0 && (unsigned long long)i < sp.count()) all.insert((unsigned long long)i);
    }
  std::vector<unsigned long long> idx(all.begin(), all.end());
  std::vector<int> ft(idx.size()), rs(idx.size());
  parallel_for(idx.size(), threads, [&](size_t i) {
    P2Out o = run_p2(c.prog, c.function, sp.binding(idx[i]), spec, c.meta.rules, c.p2seed, tests);
    ft[i] = o.fail_t;
    rs[i] = o.reason;
  });
  json j = {{"stem", stem}, {"spec", spec_name}, {"tests", tests}, {"radius", radius}, {"centers", centers},
            {"count", sp.count()}, {"idx", idx}, {"fail_t", ft}, {"reason", rs}};
  std::cout << j.dump() << std::endl;
  return 0;
}

int cmd_time_gemm(bool xpu, long long m, long long n, long long k, long long rows) {
  // inputs: uniform[-1,1] from Rng(mix(0,"bench:A"/"bench:B"))
  long long mm = xpu ? m : rows;
  std::vector<float> a((size_t)(mm * k)), b((size_t)(k * n)), c((size_t)(mm * n));
  Rng ra(Rng::mix(0, "bench:A")), rb(Rng::mix(0, "bench:B"));
  for (auto& v : a) v = (float)ra.uniform_real(-1.0, 1.0);
  for (auto& v : b) v = (float)rb.uniform_real(-1.0, 1.0);
  const double t0 = now_s();
  if (xpu)
    profitability::xpu_gemm(a.data(), b.data(), c.data(), mm, n, k);
  else
    profitability::cpu_gemm(a.data(), b.data(), c.data(), mm, n, k);
  const double dt = now_s() - t0;
  double flops = 2.0 * (double)mm * (double)n * (double)k;
  json j = {{"mode", xpu ? "xpu_gemm" : "cpu_gemm"}, {"m", mm}, {"n", n}, {"k", k},
            {"seconds", dt}, {"gflops", flops / dt / 1e9},
            {"threads", xpu ? hw_threads() : 1}, {"c0", c[0]}};
  std::cout << j.dump() << std::endl;
  return 0;
}

int cmd_time_conv(long long n, long long c, long long h, long long w, long long k, long long r,
                  long long s) {
  auto specs = default_specs();
  const auto& spec = spec_named(specs, "conv2d");
  std::map<std::string, long long> sizes = {{"tc_n", n}, {"tc_c", c}, {"tc_h", h},
                                            {"tc_w", w}, {"tc_k", k}, {"tc_r", r},
                                            {"tc_s", s}, {"tc_oh", h - r + 1},
                                            {"tc_ow", w - s + 1}};
  std::map<std::string, std::vector<double>> bufs;
  Rng ri(Rng::mix(0, "bench:in")), rw(Rng::mix(0, "bench:w"));
  bufs["tc_in"].resize((size_t)(n * c * h * w));
  bufs["tc_weights"].resize((size_t)(k * c * r * s));
  bufs["tc_out"].assign((size_t)(n * k * (h - r + 1) * (w - s + 1)), 0.0);
  for (auto& v : bufs["tc_in"]) v = (double)(float)ri.uniform_real(-1.0, 1.0);
  for (auto& v : bufs["tc_weights"]) v = (double)(float)rw.uniform_real(-1.0, 1.0);
  const double t0 = now_s();
  equivalence::run_reference(spec, sizes, bufs);
  const double dt = now_s() - t0;
  double flops = 2.0 * n * k * (h - r + 1) * (w - s + 1) * c * r * s;
  json j = {{"mode", "run_reference_conv2d"}, {"seconds", dt}, {"gflops", flops / dt / 1e9},
            {"threads", 1}};
  std::cout << j.dump() << std::endl;
  return 0;
}


int cmd_svm_golden(const std::string& out) {
  std::vector<profitability::TimingSample> data;
  for (long long m = 2; m <= 10; m += 2)
    for (long long n = 2; n <= 10; n += 2)
      for (long long k = 2; k <= 10; k += 2) {
        const long long v = m * n * k;
        if (v > 150 && v < 600) continue;
        profitability::TimingSample t;
        t.sizes = {m, n, k};
        t.t_cpu = 1.0;
        t.t_xpu = v >= 600 ? 0.5 : 2.0;
        t.label = v >= 600 ? 1 : 0;
        data.push_back(t);
      }
  const auto model = profitability::train_svm(data);
  profitability::save_svm(model, out + ".model");
  std::ifstream in(out + ".model");
  json j = {{"model", json::parse(in)}};
  std::remove((out + ".model").c_str());
  json cases = json::array();
  std::vector<std::vector<long long>> grid;
  for (long long m = 1; m <= 12; ++m)
    for (long long n = 1; n <= 12; n += 1)
      for (long long k = 1; k <= 12; k += 1) grid.push_back({m, n, k});
  for (long long v : {16LL, 64LL, 256LL, 1024LL, 8192LL}) grid.push_back({v, v, v});
  grid.push_back({48, 180, 576});  // a conv im2col feature (k, n*oh*ow, c*r*s)
  grid.push_back({1, 1000, 3});
  for (const auto& g : grid)
    cases.push_back({{"mnk", g},
                     {"decision", profitability::decision_value(model, g)},
                     {"backend", profitability::predict_backend(model, g)}});
  j["cases"] = cases;
  std::ofstream(out) << j.dump(1) << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw std::runtime_error("usage: ref_tool <cmd> ...");
    std::string cmd = argv[1];
    if (cmd == "golden" && argc == 3) return cmd_golden(argv[2]);
    if (cmd == "svm-golden" && argc == 3) return cmd_svm_golden(argv[2]);
    if ((cmd == "time-p2" || cmd == "time-acc") && argc >= 7)
      return cmd_time(cmd == "time-p2" ? "p2" : "acc", argv[2], argv[3], std::atoi(argv[4]),
                      std::atof(argv[5]), std::atoi(argv[6]),
                      argc >= 8 && std::string(argv[7]) == "rules64");
    if (cmd == "neighbourhood" && argc >= 8) {
      std::vector<unsigned long long> centers;
      for (int a = 7; a < argc; ++a) centers.push_back(std::strtoull(argv[a], nullptr, 10));
      return cmd_neighbourhood(argv[2], argv[3], std::atoi(argv[4]), std::atoll(argv[5]), centers,
                               std::atoi(argv[6]));
    }
    if (cmd == "time-xpu-gemm" && argc == 5)
      return cmd_time_gemm(true, std::atoll(argv[2]), std::atoll(argv[3]), std::atoll(argv[4]), 0);
    if (cmd == "time-cpu-gemm" && argc == 6)
      return cmd_time_gemm(false, std::atoll(argv[2]), std::atoll(argv[3]), std::atoll(argv[4]),
                           std::atoll(argv[5]));
    if (cmd == "time-conv" && argc == 9)
      return cmd_time_conv(std::atoll(argv[2]), std::atoll(argv[3]), std::atoll(argv[4]),
                           std::atoll(argv[5]), std::atoll(argv[6]), std::atoll(argv[7]),
                           std::atoll(argv[8]));
    throw std::runtime_error("bad arguments for '" + cmd + "'");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_tool: %s\n", e.what());
    return 1;
  }
}
