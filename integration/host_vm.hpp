// host_vm — a compiled executor for the mini-language with the exact semantics of
// the reference interpreter (src/interp.cpp:46-558), for the host-side phases that
// bound the pipeline's wall clock once candidate evaluation runs on the GPU
// (SURVEY.md §8(f).1 and §8(f).3): the DimProbe surveys of detect_dims
// (analysis.cpp:234-282), the P1 user-program runs of check_equivalence
// (equivalence.cpp:342-350) and the original runs the P2 test sets record
// (rewriter.cpp:242-247).
//
// The reference walks the IR with std::map scopes keyed by name and exceptions
// for `return`; here every name is resolved once to a frame slot, regions to an
// index, builtins to an opcode, and `return` is a status, so a statement costs a
// few dozen instructions.  Everything observable is unchanged: values (int/float
// promotion, f32 rounding on every write, the Value quirks of interp.cpp), step
// counting (one per executed statement plus one per while iteration), the fault
// statuses and their messages, the DimProbe rules (non-target loads yield the
// scratch value, stores are dropped, target accesses are traced and checked) and
// the write tracking of Plain runs.  Dispatch builtins are no-ops (no handler);
// a policy with a dispatch handler is refused — lifted programs keep the
// reference interpreter.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "liftc/interp.hpp"
#include "liftc/minilang.hpp"

namespace liftc::gpu {

struct VmProgram;  // compiled functions (host_vm.cpp)

class HostVm {
 public:
  explicit HostVm(const minilang::Program& prog);
  ~HostVm();
  HostVm(const HostVm&) = delete;
  HostVm& operator=(const HostVm&) = delete;

  // interp::execute (interp.hpp) for Plain and DimProbe policies without a
  // dispatch handler: the same ExecutionOutcome, field by field.
  interp::ExecutionOutcome execute(const std::string& function, const interp::MemoryImage& input,
                                   const interp::InstrumentationPolicy& policy,
                                   unsigned long long step_limit = interp::kDefaultStepLimit) const;

  // One DimProbe execution with EVERY pointer parameter of `function` as the
  // target at once, extent unbounded, trace recorded.  Loads yield the scratch
  // value whatever the target and stores are dropped, so the run is the same
  // for every target; a target's own run ends only where it sees a negative
  // offset (OutOfBounds), which is recorded per pointer.  Result per pointer:
  // what interp::execute with pol.target = that pointer returns (status,
  // fault_msg, max_target_offset, trace).
  struct Survey {
    interp::ExecStatus status = interp::ExecStatus::Normal;
    std::string fault_msg;
    long long max_target_offset = -1;
    std::vector<long long> trace;
  };
  std::map<std::string, Survey> dim_survey(const std::string& function, const interp::MemoryImage& input,
                                           unsigned long long step_limit = interp::kDefaultStepLimit) const;

 private:
  std::unique_ptr<VmProgram> prog_;
};

}  // namespace liftc::gpu
