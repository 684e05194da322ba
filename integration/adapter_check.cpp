// adapter_check — end-to-end check of the reference-side adapter on the GPU box.
//
// Built by `make -C oracle adapter` against the UNMODIFIED reference (headers from
// /root/reference/proj/include, liftc_core from oracle/_ref) and libatc_b200.so;
// it is test infrastructure (oracle/_ref/adapter_check), run by
// tests/test_integration.py.
//
//   adapter_check corpus
//       for every GEMM/conv corpus program: the reference's own
//       pipeline::lift_program vs. the same analysis followed by
//       liftc::gpu::candidate_loop (one GPU P2 batch for every spec + host P1 in
//       rank order): byte-equal masked report_to_json, and the production
//       setting's (P1 on P2 survivors only) winner and timings.
//   adapter_check unpruned <stem> <spec> [tests]
//       the full unpruned binding space of one program in Appendix C order:
//       gpu::first_accepted_unpruned on the device group (every GPU, enumerated
//       P2 + host P1 on survivors), and — for spaces up to 2^20 — the same space
//       as an explicit ranked list through gpu::first_accepted on one context;
//       winners, passing counts and passing lists must agree.
//   adapter_check dispatch
//       the lifted program run with make_gpu_dispatch vs make_oracle_dispatch.
//   adapter_check details [per_space]
//       gpu::p2_detail vs rewriter::verify_rewrite's detail on P2-rejected bindings
//       of every corpus program x spec (report parity of VerificationFailed).
//   adapter_check sampler
//       the profitability sampler on the B200 backend (gpu::sample_timings_b200) over
//       the reference's training / holdout grids, the reference's train_svm on its
//       labels, holdout accuracy.
//   adapter_check routed
//       make_gpu_routed_dispatch vs rewriter::make_routed_dispatch: the same
//       cpu/xpu labels on every lifted corpus function (model trained by the
//       reference's train_svm on rewriter_test.cpp's volume-labelled set),
//       bit-identical results on the exact route; then f32 GEMM/conv calls
//       routed "xpu" onto the tcgen05 backends, within 3xTF32 / TF32 tolerance
//       of the reference's FP64 dispatch.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <json.hpp>

#include "atc_liftc_adapter.hpp"
#include "host_phases.hpp"
#include "host_vm.hpp"
#include "liftc/classifier.hpp"
#include "liftc/equivalence.hpp"
#include "liftc/pipeline.hpp"
#include "liftc/profitability.hpp"
#include "liftc/rewriter.hpp"
#include "liftc/rng.hpp"

extern const std::map<std::string, std::string>& embedded_files();

using namespace liftc;
using json = nlohmann::json;

namespace {

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

std::vector<api::ApiSpec> default_specs() {
  std::vector<api::ApiSpec> specs;
  for (const char* n : {"gemm_rowmajor", "gemm_colmajor", "gemm_rowmajor_ld", "conv2d"})
    specs.push_back(api::parse_api_spec(embedded_files().at(std::string("specs/") + n + ".json")));
  return specs;
}

struct Prog {
  std::string key, tag, stem, dir, function;
  minilang::Program prog;
  pipeline::FixtureMeta meta;
};

std::vector<Prog> corpus(bool every_dir = false) {
  std::vector<Prog> out;
  for (const auto& [k, v] : embedded_files()) {
    if (k.rfind("corpus/", 0) != 0 || k.substr(k.size() - 3) != ".ml") continue;
    Prog p;
    p.key = k;
    p.tag = k.substr(k.rfind('/') + 1);
    p.stem = p.tag.substr(0, p.tag.size() - 3);
    p.dir = k.substr(7, k.rfind('/') - 7);
    if (!every_dir && p.dir != "gemm" && p.dir != "conv") continue;
    p.prog = minilang::parse_program(v);
    auto side = embedded_files().find(k.substr(0, k.size() - 3) + ".json");
    if (side != embedded_files().end()) p.meta = pipeline::parse_fixture_meta(side->second);
    p.function = p.meta.function.empty() ? p.prog.functions[0].name : p.meta.function;
    out.push_back(std::move(p));
  }
  return out;
}

// the analysis half of pipeline.cpp:164-221 on the host VM (gpu::analyze_function:
// the same liveness, probe values and dims as the reference's calls — pinned by
// `adapter_check host`)
analysis::AnalyzedFunction analyze(const Prog& p, uint64_t fseed, const std::vector<const api::ApiSpec*>& specs,
                                   const std::string& function = "") {
  const auto* f = p.prog.find(function.empty() ? p.function : function);
  int max_rank = p.meta.max_rank;
  for (const auto* s : specs)
    if (!p.meta.max_rank) max_rank = std::max(max_rank, s->max_rank());
  const gpu::HostVm vm(p.prog);
  return gpu::analyze_function(vm, *f, fseed, p.meta.rules, p.meta.probes, max_rank);
}

int cmd_corpus(atc_ctx* ctx) {
  auto specs = default_specs();
  std::vector<std::pair<classifier::FeatureVector, std::string>> ex;
  for (const auto& [k, v] : embedded_files()) {  // tools/liftc.cpp:92-106 over the whole corpus
    if (k.rfind("corpus/", 0) != 0 || k.substr(k.size() - 3) != ".ml") continue;
    auto side = embedded_files().find(k.substr(0, k.size() - 3) + ".json");
    if (side == embedded_files().end()) continue;
    auto meta = pipeline::parse_fixture_meta(side->second);
    if (meta.function.empty() || meta.label.empty()) continue;
    auto prog = minilang::parse_program(v);
    if (const auto* fn = prog.find(meta.function)) ex.emplace_back(classifier::extract_features(prog, *fn), meta.label);
  }
  auto model = classifier::train_classifier(ex);
  pipeline::PipelineConfig cfg;
  cfg.specs = specs;
  cfg.classifier = &model;
  cfg.workers = 1;
  int mismatches = 0;
  // every function of every corpus file (gemm, conv, nonidiom): the reference's
  // lift_program report vs. the same report with the candidate stage replaced
  for (const auto& p : corpus(true)) {
    auto t0 = std::chrono::steady_clock::now();
    auto rep = pipeline::lift_program(p.prog, p.tag, p.meta, cfg, nullptr);
    const double ref_ms = ms_since(t0);
    for (const auto& fref : rep.functions) {
    const pipeline::FunctionReport* fr = &fref;
    const std::string function = fr->function;
    json j = {{"stem", p.stem}, {"function", function}, {"dir", p.dir},
              {"reference_status", pipeline::status_name(fr->status)}, {"reference_ms", ref_ms}};
    std::vector<const api::ApiSpec*> lspecs;
    for (const auto& s : specs)
      if (s.semantics == fr->class_label) lspecs.push_back(&s);
    if (fr->status == pipeline::FunctionStatus::Misclassified || lspecs.empty() ||
        fr->status == pipeline::FunctionStatus::AnalysisFailed) {
      // no candidate stage in the reference either (pipeline.cpp:141-162, :164-221):
      // the report is the host's, unchanged
      j["candidate_stage"] = false;
      std::cout << j.dump() << std::endl;
      continue;
    }
    const uint64_t fseed = Rng::mix(cfg.seed, p.tag + ":" + function);  // pipeline.cpp:131
    auto t_an = std::chrono::steady_clock::now();
    auto fn = analyze(p, fseed, lspecs, function);
    const double analysis_ms = ms_since(t_an);
    gpu::LoopConfig lc;
    lc.tests = cfg.tests;
    lc.verify_tests = cfg.verify_tests;
    lc.max_candidates = cfg.max_candidates;
    lc.budget_sec = cfg.budget_sec;
    lc.report = true;
    t0 = std::chrono::steady_clock::now();
    auto loop = gpu::candidate_loop(ctx, p.prog, fn, function, lspecs, p.meta.rules, fseed, lc);
    const double ours_ms = ms_since(t0);
    // the reference's report with every candidate-stage field replaced by ours
    // (pipeline.cpp:223-330); everything else is the unchanged host analysis
    pipeline::FunctionReport mine = *fr;
    mine.status = loop.status;
    mine.status_detail = loop.status_detail;
    mine.by_spec = loop.by_spec;
    mine.evaluated = loop.evaluated;
    mine.winning_api.clear();
    mine.manifest = rewriter::LiftManifest{};
    if (loop.status == pipeline::FunctionStatus::Lifted) {  // pipeline.cpp:285-298
      mine.winning_api = loop.winning_spec->name;
      mine.manifest = loop.rewrite.manifest;
      mine.manifest.verdict = "Equivalent";
      mine.manifest.class_label = fr->class_label;
      mine.manifest.class_score = fr->class_score;
      for (const auto& b : loop.by_spec)
        if (b.api == mine.winning_api) {
          mine.manifest.raw_candidates = b.raw;
          mine.manifest.pruned_candidates = b.filtered;
        }
      mine.manifest.winner_rank = loop.winner_rank;
    }
    pipeline::FileReport ref_file, our_file;
    ref_file.file = our_file.file = p.tag;
    ref_file.functions = {*fr};
    our_file.functions = {mine};
    const std::string ref_json = pipeline::mask_timings(pipeline::report_to_json(ref_file)).dump();
    const std::string our_json = pipeline::mask_timings(pipeline::report_to_json(our_file)).dump();
    const bool same_report = ref_json == our_json;
    std::string gpu_status = pipeline::status_name(loop.status), gpu_api = mine.winning_api;
    const int gpu_rank = loop.winner_rank;
    bool same = gpu_status == pipeline::status_name(fr->status);
    if (same && gpu_status == "Lifted")
      same = gpu_api == fr->winning_api && gpu_rank == fr->manifest.winner_rank &&
             loop.rewrite.manifest.arrays == fr->manifest.arrays && loop.rewrite.manifest.sizes == fr->manifest.sizes;
    j["same_report_json"] = same_report;
    if (!same_report) {
      j["ref_report"] = json::parse(ref_json);
      j["our_report"] = json::parse(our_json);
    }
    same = same && same_report;
    const int p1_calls = loop.p1_calls;
    const double gpu_ms = loop.gpu_ms;
    j["record_ms"] = loop.record_ms;
    j["p1_ms"] = loop.p1_ms;
    // the production setting (P1 only on P2 survivors) against the reference's own
    // candidate stage (its match + equivalence + rewrite/verify phases)
    lc.report = false;
    t0 = std::chrono::steady_clock::now();
    auto fast = gpu::candidate_loop(ctx, p.prog, fn, function, lspecs, p.meta.rules, fseed, lc);
    j["fast_loop_ms"] = ms_since(t0);
    // the whole lift of the function with the GPU candidate stage and the host-VM
    // analyses (liveness, dims, P1), against the reference's lift_program
    j["analysis_ms"] = analysis_ms;
    j["ours_lift_ms"] = analysis_ms + (double)j["fast_loop_ms"];
    j["fast_gpu_p2_ms"] = fast.gpu_ms;
    j["fast_record_ms"] = fast.record_ms;
    j["fast_p1_ms"] = fast.p1_ms;
    j["fast_same_winner"] = fast.status == loop.status && fast.winner_rank == loop.winner_rank &&
                            fast.winning_spec == loop.winning_spec;
    same = same && fast.status == loop.status && fast.winner_rank == loop.winner_rank &&
           fast.winning_spec == loop.winning_spec;
    double ref_loop = 0;
    for (const char* k : {"match_ms", "equivalence_ms", "rewrite_ms"})
      if (fr->phase_ms.count(k)) ref_loop += fr->phase_ms.at(k);
    j["reference_loop_ms"] = ref_loop;
    if (!same) ++mismatches;
    j["gpu_status"] = gpu_status;
    j["gpu_api"] = gpu_api;
    j["gpu_rank"] = gpu_rank;
    j["same_outcome"] = same;
    j["p1_calls"] = p1_calls;
    j["candidate_loop_ms"] = ours_ms;
    j["gpu_p2_ms"] = gpu_ms;
    j["candidate_stage"] = true;
    std::cout << j.dump() << std::endl;
    }
  }
  std::cout << json({{"mismatches", mismatches}}).dump() << std::endl;
  return mismatches == 0 ? 0 : 1;
}

int cmd_unpruned(atc_ctx* ctx, atc_group* g, const std::string& stem, const std::string& spec_name, int tests) {
  auto specs = default_specs();
  const api::ApiSpec* spec = nullptr;
  for (const auto& s : specs)
    if (s.name == spec_name) spec = &s;
  for (const auto& p : corpus()) {
    if (p.stem != stem || !spec) continue;
    const uint64_t fseed = Rng::mix(0, p.tag + ":" + p.function);
    auto fn = analyze(p, fseed, {spec});
    const gpu::UnprunedSpace sp(fn, *spec);
    json j = {{"stem", stem}, {"spec", spec_name}, {"bindings", sp.count()}, {"tests", tests},
              {"devices", atc_group_size(g)}};
    // the whole space on the device group (enumerated, sharded over the members)
    auto t0 = std::chrono::steady_clock::now();
    auto ur = gpu::first_accepted_unpruned(g, p.prog, fn, p.function, *spec, p.meta.rules, fseed, 30, tests);
    j["group"] = {{"winner", ur.winner}, {"p2_passed", ur.p2_passed}, {"p1_calls", ur.p1_calls},
                  {"record_ms", ur.record_ms}, {"gpu_p2_ms", ur.gpu_ms}, {"p1_ms", ur.p1_ms},
                  {"total_ms", ms_since(t0)},
                  {"reason_counts", std::vector<int64_t>(ur.reason_counts, ur.reason_counts + ATC_REASON_COUNT)}};
    bool ok = true;
    if (sp.count() <= (1u << 20)) {  // the same space as an explicit ranked list on one context
      std::vector<matching::CandidateBinding> space;
      for (size_t i = 0; i < sp.count(); ++i) space.push_back(sp.at(*spec, i));
      t0 = std::chrono::steady_clock::now();
      auto lr = gpu::first_accepted(ctx, p.prog, fn, p.function, *spec, space, p.meta.rules, fseed, 30, tests);
      const double total = ms_since(t0);
      int64_t passed = 0;
      std::vector<uint64_t> passing;
      for (size_t b = 0; b < lr.p2_reason.size(); ++b)
        if (lr.p2_reason[b] == ATC_PASS) {
          ++passed;
          if (passing.size() < ur.p2_passing.size()) passing.push_back(b);
        }
      const int64_t winner = lr.winner ? (int64_t)*lr.winner : -1;
      ok = winner == ur.winner && passed == ur.p2_passed && passing == ur.p2_passing;
      j["list"] = {{"winner", winner}, {"p2_passed", passed}, {"p1_calls", lr.p1_calls}, {"record_ms", lr.record_ms},
                   {"gpu_p2_ms", lr.gpu_ms}, {"p1_ms", lr.p1_ms}, {"total_ms", total}};
    }
    j["same"] = ok;
    std::cout << j.dump() << std::endl;
    return ok ? 0 : 1;
  }
  return 1;
}


// p2_detail vs the reference's own verify_rewrite detail (rewriter.cpp:215-284) on
// bindings of every corpus program x spec that P2 rejects: a strided sample of
// each unpruned space plus its first bindings (mismatch and dispatch-failure
// details; f32 and f64 regions; every program's recorded test sets).
int cmd_details(atc_ctx* ctx, int per_space) {
  auto specs = default_specs();
  int bad = 0, checked = 0;
  std::map<std::string, int> kinds;
  for (const auto& p : corpus()) {
    if (p.dir != "gemm" && p.dir != "conv") continue;
    const uint64_t fseed = Rng::mix(0, p.tag + ":" + p.function);
    const auto* f = p.prog.find(p.function);
    for (const auto& spec : specs) {
      if ((spec.semantics == "conv2d") != (p.dir == "conv")) continue;
      auto fn = analyze(p, fseed, {&spec});
      gpu::UnprunedSpace sp(fn, spec);
      if (sp.count() == 0) continue;
      // a wide strided sample screened on the GPU, then up to per_space rejected
      // bindings of each failure reason re-run through the reference
      std::vector<matching::CandidateBinding> list;
      const size_t wide = 64 * (size_t)per_space;
      const size_t stride = std::max<size_t>(1, sp.count() / wide);
      for (size_t i = 0; i < sp.count() && list.size() < wide + 16; i += (i < 16 ? 1 : stride))
        list.push_back(sp.at(spec, i));
      auto rec = gpu::record_tests(p.prog, p.function, p.meta.rules, Rng::mix(fseed, "post"), 10);
      auto v = gpu::p2_verdicts(ctx, rec, {&spec}, {&list});
      std::map<int, int> taken;
      for (size_t b = 0; b < list.size(); ++b) {
        if (v[0].reason[b] == ATC_PASS || taken[v[0].reason[b]]++ >= per_space) continue;
        auto rr = rewriter::rewrite(p.prog, p.function, list[b], spec);
        auto vr = rewriter::verify_rewrite(p.prog, rr.program, p.function, list[b], spec, p.meta.rules,
                                           Rng::mix(fseed, "post"), 10);
        const std::string ours =
            gpu::p2_detail(ctx, rec, *f, spec, list[b], v[0].fail_t[b], v[0].reason[b]);
        ++checked;
        ++kinds[vr.detail.rfind("mismatch", 0) == 0 ? "mismatch"
                : vr.detail.rfind("dispatch failed", 0) == 0 ? "dispatch failed"
                                                               : "other"];
        if (vr.ok || ours != vr.detail) {
          ++bad;
          std::cout << json({{"stem", p.stem}, {"spec", spec.name}, {"reference", vr.detail}, {"ours", ours},
                             {"reference_ok", vr.ok}})
                           .dump()
                    << std::endl;
        }
      }
    }
  }
  std::cout << json({{"checked", checked}, {"mismatches", bad}, {"kinds", kinds}}).dump() << std::endl;
  return bad == 0 ? 0 : 1;
}

// host_vm / host_phases against the reference interpreter and analyses on every
// function of every corpus file (no GPU needed): raw executions (status, fault
// message, steps, final images, write flags, return value), detect_liveness,
// detect_dims per pointer, and P1 check_equivalence (verdict, tests_run, detail,
// counterexample) on every ranked candidate plus a strided sample of each
// unpruned space; with the time each side took.
int cmd_host() {
  auto specs = default_specs();
  int bad = 0;
  long long runs = 0, p1 = 0, dims = 0, lives = 0;
  double t_ref[4] = {}, t_vm[4] = {};  // exec, liveness, dims, p1
  auto report = [&](const json& j) {
    ++bad;
    std::cout << j.dump() << std::endl;
  };
  for (const auto& [k, v] : embedded_files()) {
    if (k.rfind("corpus/", 0) != 0 || k.substr(k.size() - 3) != ".ml") continue;
    const std::string tag = k.substr(k.rfind('/') + 1);
    auto prog = minilang::parse_program(v);
    pipeline::FixtureMeta meta;
    auto side = embedded_files().find(k.substr(0, k.size() - 3) + ".json");
    if (side != embedded_files().end()) meta = pipeline::parse_fixture_meta(side->second);
    const gpu::HostVm vm(prog);
    for (const auto& f : prog.functions) {
      const uint64_t fseed = Rng::mix(0, tag + ":" + f.name);
      std::vector<std::string> ints;
      for (const auto& q : f.params)
        if (q.kind == minilang::ParamKind::IntScalar) ints.push_back(q.name);
      // raw executions on probe images (sizes per the sidecar rules, three seeds)
      for (int rep = 0; rep < 3; ++rep) {
        Rng rng(Rng::mix(fseed, "hostvm:" + std::to_string(rep)));
        std::map<std::string, long long> sizes;
        if (!analysis::draw_sizes(ints, meta.rules, rng, sizes)) continue;
        auto img = analysis::build_probe_image(f, sizes, rng);
        interp::InstrumentationPolicy pol;
        pol.track_writes = rep != 1;
        auto t0 = std::chrono::steady_clock::now();
        auto a = interp::execute(prog, f.name, img, pol);
        t_ref[0] += ms_since(t0);
        t0 = std::chrono::steady_clock::now();
        auto b = vm.execute(f.name, img, pol);
        t_vm[0] += ms_since(t0);
        ++runs;
        bool same = a.status == b.status && a.fault_msg == b.fault_msg && a.steps == b.steps &&
                    a.has_ret == b.has_ret && a.ret_is_int == b.ret_is_int && a.ret_int == b.ret_int &&
                    (a.ret_float == b.ret_float || (std::isnan(a.ret_float) && std::isnan(b.ret_float))) &&
                    a.writes == b.writes && a.final.regions.size() == b.final.regions.size();
        for (const auto& [name, r] : a.final.regions)
          same = same && b.final.regions.count(name) &&
                 std::memcmp(r.data.data(), b.final.regions.at(name).data.data(), r.data.size() * 8) == 0;
        if (!same)
          report({{"file", tag}, {"function", f.name}, {"what", "execute"}, {"status", {a.status, b.status}},
                  {"msg", {a.fault_msg, b.fault_msg}}, {"steps", {a.steps, b.steps}}});
      }
      // liveness
      std::string ra, rb;
      analysis::LivenessReport la, lb;
      auto t0 = std::chrono::steady_clock::now();
      try { la = analysis::detect_liveness(prog, f, fseed, meta.rules); } catch (const std::exception& e) { ra = e.what(); }
      t_ref[1] += ms_since(t0);
      t0 = std::chrono::steady_clock::now();
      try { lb = gpu::detect_liveness(vm, f, fseed, meta.rules); } catch (const std::exception& e) { rb = e.what(); }
      t_vm[1] += ms_since(t0);
      ++lives;
      if (ra != rb || la.classes != lb.classes)
        report({{"file", tag}, {"function", f.name}, {"what", "liveness"}, {"errors", {ra, rb}}});
      // dims (max rank: the sidecar's, else the bundled specs' largest)
      int max_rank = meta.max_rank;
      for (const auto& sp : specs)
        if (!meta.max_rank) max_rank = std::max(max_rank, sp.max_rank());
      std::map<std::string, long long> probe;
      try { probe = analysis::assign_probe_values(ints, meta.rules, meta.probes, 0); } catch (const std::exception&) { continue; }
      std::vector<gpu::DimsOutcome> ours;
      std::string eb;
      t0 = std::chrono::steady_clock::now();
      try { ours = gpu::detect_dims_all(vm, f, ints, probe, max_rank); } catch (const std::exception& e) { eb = e.what(); }
      t_vm[2] += ms_since(t0);
      size_t oi = 0;
      for (const auto& q : f.params) {
        if (q.kind != minilang::ParamKind::Pointer) continue;
        std::string ea;
        bool found = false;
        analysis::DimSpec d;
        t0 = std::chrono::steady_clock::now();
        try {
          d = analysis::detect_dims(prog, f, q.name, ints, probe, max_rank);
          found = true;
        } catch (const analysis::NoDimsFound&) {
        } catch (const std::exception& e) {
          ea = e.what();
        }
        t_ref[2] += ms_since(t0);
        ++dims;
        const bool same = ea == eb && (!eb.empty() || (oi < ours.size() && ours[oi].found == found &&
                                                       (!found || (ours[oi].spec.dims == d.dims &&
                                                                   ours[oi].spec.slow_dim == d.slow_dim))));
        if (!same) report({{"file", tag}, {"function", f.name}, {"what", "dims"}, {"array", q.name}, {"errors", {ea, eb}}});
        ++oi;
      }
      // P1 on gemm/conv functions: ranked candidates + a strided unpruned sample
      if (meta.function != f.name || meta.label.empty()) continue;
      for (const auto& spec : specs) {
        if (spec.semantics != meta.label) continue;
        analysis::AnalyzedFunction fn;
        try {
          fn = gpu::analyze_function(vm, f, fseed, meta.rules, meta.probes, max_rank);
        } catch (const std::exception&) {
          break;
        }
        std::vector<matching::CandidateBinding> cands;
        auto ranked = matching::rank_candidates(matching::find_matchings(fn, spec), 100);
        for (const auto& c : ranked.ranked) cands.push_back(c);
        gpu::UnprunedSpace sp(fn, spec);
        const size_t stride = std::max<size_t>(1, sp.count() / 24);
        for (size_t i = 0; i < sp.count() && cands.size() < 40; i += stride) cands.push_back(sp.at(spec, i));
        for (const auto& c : cands) {
          equivalence::EquivalenceConfig ec;
          ec.seed = fseed;
          t0 = std::chrono::steady_clock::now();
          auto a = equivalence::check_equivalence(prog, fn, c, spec, meta.rules, ec);
          t_ref[3] += ms_since(t0);
          t0 = std::chrono::steady_clock::now();
          auto b = gpu::check_equivalence(vm, prog, fn, c, spec, meta.rules, ec);
          t_vm[3] += ms_since(t0);
          ++p1;
          const bool same = a.verdict == b.verdict && a.tests_run == b.tests_run && a.detail == b.detail &&
                            a.cex.sizes == b.cex.sizes && a.cex.array == b.cex.array &&
                            a.cex.offset == b.cex.offset && a.cex.expected == b.cex.expected &&
                            a.cex.actual == b.cex.actual;
          if (!same)
            report({{"file", tag}, {"function", f.name}, {"what", "p1"}, {"spec", spec.name},
                    {"verdict", {equivalence::verdict_name(a.verdict), equivalence::verdict_name(b.verdict)}},
                    {"tests_run", {a.tests_run, b.tests_run}}, {"detail", {a.detail, b.detail}}});
        }
      }
    }
  }
  std::cout << json({{"mismatches", bad}, {"executions", runs}, {"liveness", lives}, {"dims", dims}, {"p1", p1},
                     {"reference_ms", {{"execute", t_ref[0]}, {"liveness", t_ref[1]}, {"dims", t_ref[2]}, {"p1", t_ref[3]}}},
                     {"host_vm_ms", {{"execute", t_vm[0]}, {"liveness", t_vm[1]}, {"dims", t_vm[2]}, {"p1", t_vm[3]}}}})
                   .dump()
            << std::endl;
  return bad == 0 ? 0 : 1;
}

int cmd_dispatch(atc_ctx* ctx) {
  auto specs = default_specs();
  int bad = 0;
  for (const auto& p : corpus()) {
    if (!p.meta.expect_lift) continue;
    const api::ApiSpec* spec = nullptr;
    for (const auto& s : specs)
      if (s.name == p.meta.api) spec = &s;
    if (!spec) continue;
    matching::CandidateBinding b;
    for (const auto& [k, v] : p.meta.binding_truth) {
      const auto* ap = spec->find(k);
      if (ap && ap->kind == api::ApiParamKind::Array) b.arrays[k] = v;
      if (ap && ap->kind == api::ApiParamKind::IntSize) b.sizes[k] = v;
    }
    auto rr = rewriter::rewrite(p.prog, p.function, b, *spec);
    const uint64_t fseed = Rng::mix(0, p.tag + ":" + p.function);
    Rng rng(Rng::mix(fseed, "dispatch-check"));
    std::vector<std::string> int_params;
    for (const auto& q : p.prog.find(p.function)->params)
      if (q.kind == minilang::ParamKind::IntScalar) int_params.push_back(q.name);
    std::map<std::string, long long> sizes;
    while (!analysis::draw_sizes(int_params, p.meta.rules, rng, sizes)) {
    }
    auto img = analysis::build_probe_image(*p.prog.find(p.function), sizes, rng);
    auto oracle = rewriter::make_oracle_dispatch(*spec);
    auto gpu_ctx = gpu::make_gpu_dispatch(*spec, ctx);
    interp::InstrumentationPolicy po, pg;
    po.dispatch = &oracle;
    pg.dispatch = &gpu_ctx;
    auto a = interp::execute(rr.program, p.function, img, po);
    auto g = interp::execute(rr.program, p.function, img, pg);
    bool same = a.status == g.status;
    for (const auto& [name, reg] : a.final.regions) same = same && reg.data == g.final.regions.at(name).data;
    bad += !same;
    std::cout << json({{"stem", p.stem}, {"api", spec->name}, {"bit_identical", same}}).dump() << std::endl;
  }
  std::cout << json({{"mismatches", bad}}).dump() << std::endl;
  return bad == 0 ? 0 : 1;
}


// rewriter_test.cpp:109-118's volume-thresholded training set.
profitability::SvmModel volume_model() {
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
  return profitability::train_svm(data);
}

// A model whose decision value is the constant b (no support vectors).
profitability::SvmModel constant_model(double b) {
  profitability::SvmModel m;
  m.feature_dim = 3;
  m.feat_min = {0, 0, 0};
  m.feat_max = {1, 1, 1};
  m.b = b;
  return m;
}

double max_rel_err(const std::vector<double>& got, const std::vector<double>& ref) {
  double e = 0;
  for (size_t i = 0; i < ref.size(); ++i) e = std::max(e, std::abs(got[i] - ref[i]) / (1.0 + std::abs(ref[i])));
  return e;
}

// The profitability sampler on the B200 backend (gpu::sample_timings_b200): the
// reference's training and holdout grids (profitability.cpp:120-136), every point
// cross-checked against cpu_gemm and timed; the reference's own train_svm on the
// B200 labels, its accuracy on the holdout grid.
int cmd_sampler(atc_ctx* ctx) {
  auto train = gpu::sample_timings_b200(ctx, profitability::training_grid(), 5);
  auto hold = gpu::sample_timings_b200(ctx, profitability::holdout_grid(), 5);
  auto model = profitability::train_svm(train);
  int right = 0, xpu = 0;
  json pts = json::array();
  for (const auto* set : {&train, &hold})
    for (const auto& t : *set) {
      pts.push_back({{"sizes", t.sizes}, {"t_cpu_ms", t.t_cpu * 1e3}, {"t_b200_ms", t.t_xpu * 1e3}, {"label", t.label},
                     {"holdout", set == &hold}});
      xpu += t.label;
    }
  for (const auto& h : hold) right += profitability::predict_backend(model, h.sizes) == h.label;
  std::cout << json({{"points", pts},
                     {"train_accuracy", model.train_accuracy},
                     {"holdout_accuracy", (double)right / (double)hold.size()},
                     {"xpu_labels", xpu},
                     {"samples", train.size() + hold.size()},
                     {"support_vectors", model.support.size()}})
                   .dump()
            << std::endl;
  return 0;
}

int cmd_routed(atc_ctx* ctx) {
  auto specs = default_specs();
  const auto model = volume_model();
  int bad = 0;
  for (const auto& p : corpus()) {
    if (!p.meta.expect_lift) continue;
    const api::ApiSpec* spec = nullptr;
    for (const auto& s : specs)
      if (s.name == p.meta.api) spec = &s;
    if (!spec) continue;
    matching::CandidateBinding b;
    for (const auto& [k, v] : p.meta.binding_truth) {
      const auto* ap = spec->find(k);
      if (ap && ap->kind == api::ApiParamKind::Array) b.arrays[k] = v;
      if (ap && ap->kind == api::ApiParamKind::IntSize) b.sizes[k] = v;
    }
    auto rr = rewriter::rewrite(p.prog, p.function, b, *spec);
    Rng rng(Rng::mix(Rng::mix(0, p.tag + ":" + p.function), "routed-check"));
    std::vector<std::string> int_params;
    for (const auto& q : p.prog.find(p.function)->params)
      if (q.kind == minilang::ParamKind::IntScalar) int_params.push_back(q.name);
    std::map<std::string, long long> sizes;
    while (!analysis::draw_sizes(int_params, p.meta.rules, rng, sizes)) {
    }
    auto img = analysis::build_probe_image(*p.prog.find(p.function), sizes, rng);
    std::vector<std::string> rc_, ge_, gt_;
    auto ref = rewriter::make_routed_dispatch(*spec, &model, &rc_);
    auto exact = gpu::make_gpu_routed_dispatch(*spec, ctx, &model, &ge_, gpu::kRouteExact);
    auto tens = gpu::make_gpu_routed_dispatch(*spec, ctx, &model, &gt_, ATC_PREC_3XTF32);
    interp::InstrumentationPolicy pr, pe, pt;
    pr.dispatch = &ref;
    pe.dispatch = &exact;
    pt.dispatch = &tens;
    auto a = interp::execute(rr.program, p.function, img, pr);
    auto e = interp::execute(rr.program, p.function, img, pe);
    auto t = interp::execute(rr.program, p.function, img, pt);
    bool same = a.status == e.status && rc_ == ge_ && rc_ == gt_ && a.status == t.status;
    double err = 0;
    for (const auto& [name, reg] : a.final.regions) {
      same = same && reg.data == e.final.regions.at(name).data;
      err = std::max(err, max_rel_err(t.final.regions.at(name).data, reg.data));
    }
    same = same && err <= 1e-3;
    bad += !same;
    std::cout << json({{"stem", p.stem}, {"api", spec->name}, {"choices", rc_}, {"ok", same}, {"tensor_err", err}})
                     .dump()
              << std::endl;
  }

  // f32 calls the predictor routes "xpu", straight through the handler
  const auto xpu = constant_model(1.0), cpu = constant_model(-1.0);
  auto call = [&](const api::ApiSpec& spec, const std::map<std::string, long long>& ints,
                  const std::map<std::string, size_t>& lens, const profitability::SvmModel& m, int32_t prec,
                  uint64_t seed, std::string& label, double& err) {
    Rng rng(seed);
    interp::MemoryImage mem;
    std::vector<interp::DispatchArg> args;
    for (const auto& ap : spec.params) {
      interp::DispatchArg a;
      if (ap.kind == api::ApiParamKind::Array) {
        interp::Region r;
        r.elem = minilang::ScalarType::F32;
        r.data.resize(lens.at(ap.role));
        for (auto& x : r.data) x = (double)(float)rng.uniform_real(-1.0, 1.0);
        mem.regions[ap.name] = r;
        a.kind = interp::DispatchArg::Kind::Ptr;
        a.region = ap.name;
      } else {
        a.kind = interp::DispatchArg::Kind::Int;
        a.i = ints.at(ap.role);
      }
      args.push_back(a);
    }
    auto mem_ref = mem;
    std::vector<std::string> ch, rch;
    gpu::make_gpu_routed_dispatch(spec, ctx, &m, &ch, prec).handler("atc_dispatch_" + spec.semantics, args, mem);
    rewriter::make_routed_dispatch(spec, &m, &rch).handler("atc_dispatch_" + spec.semantics, args, mem_ref);
    label = ch.at(0) == rch.at(0) ? ch.at(0) : "label-mismatch";
    err = 0;
    for (const auto& [name, reg] : mem_ref.regions) err = std::max(err, max_rel_err(mem.regions.at(name).data, reg.data));
  };
  struct Case {
    const char* spec;
    std::map<std::string, long long> ints;
    std::map<std::string, size_t> lens;
    double depth;  // reduction length (k, or c*r*s)
  };
  const std::vector<Case> cases = {
      {"gemm_rowmajor", {{"m", 256}, {"n", 192}, {"k", 320}}, {{"a", 256 * 320}, {"b", 320 * 192}, {"c", 256 * 192}}, 320},
      {"gemm_colmajor", {{"m", 130}, {"n", 70}, {"k", 200}}, {{"a", 130 * 200}, {"b", 200 * 70}, {"c", 130 * 70}}, 200},
      {"gemm_rowmajor_ld",
       {{"m", 200}, {"n", 96}, {"k", 160}, {"lda", 170}, {"ldb", 100}, {"ldc", 101}},
       {{"a", 200 * 170}, {"b", 160 * 100}, {"c", 200 * 101}}, 160},
      {"conv2d",
       {{"n", 2}, {"c", 64}, {"h", 12}, {"w", 11}, {"k", 48}, {"r", 3}, {"s", 3}, {"oh", 10}, {"ow", 9}},
       {{"in", 2 * 64 * 12 * 11}, {"weights", 48 * 64 * 9}, {"out", 2 * 48 * 10 * 9}}, 576},
  };
  for (const auto& c : cases) {
    const api::ApiSpec* spec = nullptr;
    for (const auto& s : specs)
      if (s.name == c.spec) spec = &s;
    for (int32_t prec : {ATC_PREC_3XTF32, ATC_PREC_TF32}) {
      std::string lx, lc;
      double ex, ec;
      call(*spec, c.ints, c.lens, xpu, prec, 7 + prec, lx, ex);
      call(*spec, c.ints, c.lens, cpu, prec, 7 + prec, lc, ec);
      // the backends' stated bounds (tests/test_gpu_backends.py TOLS): TOL * sqrt(depth)
      const double tol = (prec == ATC_PREC_3XTF32 ? 2e-5 : 5e-4) * std::sqrt(c.depth);
      const bool ok = lx == "xpu" && lc == "cpu" && ex > 0 && ex <= tol && ec == 0;
      bad += !ok;
      std::cout << json({{"direct", c.spec}, {"precision", prec == ATC_PREC_TF32 ? "tf32" : "3xtf32"},
                         {"xpu_err", ex}, {"cpu_err", ec}, {"labels", {lx, lc}}, {"ok", ok}})
                       .dump()
                << std::endl;
    }
  }
  std::cout << json({{"mismatches", bad}}).dump() << std::endl;
  return bad == 0 ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "host") {  // host-side checks: no GPU needed
    try {
      return cmd_host();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "adapter_check: %s\n", e.what());
      return 1;
    }
  }
  // every visible GPU as one device group; single-context work
  // (the candidate loop, dispatch) runs on member 0, as one pipeline worker would
  atc_group* g = atc_group_create(nullptr, 0);
  atc_ctx* ctx = g ? atc_group_member(g, 0) : nullptr;
  if (!g || atc_group_last_error(g)[0] || !ctx) {
    std::fprintf(stderr, "adapter_check: %s\n", g ? atc_group_last_error(g) : "no device group");
    return 2;
  }
  int rc = 1;
  try {
    std::string cmd = argc > 1 ? argv[1] : "corpus";
    if (cmd == "corpus") rc = cmd_corpus(ctx);
    if (cmd == "unpruned" && argc >= 4) rc = cmd_unpruned(ctx, g, argv[2], argv[3], argc > 4 ? std::atoi(argv[4]) : 10);
    if (cmd == "dispatch") rc = cmd_dispatch(ctx);
    if (cmd == "details") rc = cmd_details(ctx, argc > 2 ? std::atoi(argv[2]) : 24);
    if (cmd == "routed") rc = cmd_routed(ctx);
    if (cmd == "sampler") rc = cmd_sampler(ctx);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "adapter_check: %s\n", e.what());
    rc = 1;
  }
  atc_group_destroy(g);
  return rc;
}
