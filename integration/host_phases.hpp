// host_phases — the host analyses around candidate evaluation, on host_vm
// (SURVEY.md §8(f).1, §8(f).3).  Each function returns exactly what the
// reference function it names returns for the same inputs (tests:
// adapter_check host; tests/test_integration.py).
#pragma once

#include <map>
#include <string>
#include <vector>

#include "host_vm.hpp"
#include "liftc/analysis.hpp"
#include "liftc/api_spec.hpp"
#include "liftc/equivalence.hpp"
#include "liftc/matching.hpp"
#include "liftc/minilang.hpp"

namespace liftc::gpu {

// analysis::detect_dims (analysis.cpp:234-282) for EVERY pointer parameter of f
// from ONE survey run (HostVm::dim_survey): per pointer, in signature order,
// found = false where the reference throws NoDimsFound.  Argument errors (probe
// values < 5 or not distinct) throw std::invalid_argument like the reference.
struct DimsOutcome {
  std::string array;
  bool found = false;
  analysis::DimSpec spec;
};
std::vector<DimsOutcome> detect_dims_all(const HostVm& vm, const minilang::FunctionIR& f,
                                         const std::vector<std::string>& int_params,
                                         const std::map<std::string, long long>& probe_values, int max_rank);

// analysis::detect_liveness (analysis.cpp:106-167) with the probe runs on host_vm.
analysis::LivenessReport detect_liveness(const HostVm& vm, const minilang::FunctionIR& f, uint64_t seed,
                                         const api::SizeRules& rules);

// The analysis half of pipeline::lift_function (pipeline.cpp:164-221): liveness,
// probe values, dims of every pointer.  Throws what the reference's calls throw
// (the caller maps them to AnalysisFailed like pipeline.cpp does).
analysis::AnalyzedFunction analyze_function(const HostVm& vm, const minilang::FunctionIR& f, uint64_t fseed,
                                            const api::SizeRules& rules,
                                            const std::vector<std::map<std::string, long long>>& probes,
                                            int max_rank);

// equivalence::check_equivalence (equivalence.cpp:141-379) — P1 — with the user
// program run on host_vm; the same verdict, tests_run, detail and counterexample.
equivalence::EquivalenceResult check_equivalence(const HostVm& vm, const minilang::Program& prog,
                                                 const analysis::AnalyzedFunction& fn,
                                                 const matching::CandidateBinding& binding,
                                                 const api::ApiSpec& spec, const api::SizeRules& user_rules,
                                                 const equivalence::EquivalenceConfig& cfg);

}  // namespace liftc::gpu
