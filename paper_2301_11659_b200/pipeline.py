"""The pipeline's candidate loop with the GPU P2 screen (host-side mirror).

Reference: pipeline::lift_function's per-spec candidate loop
(/root/reference/proj/src/pipeline.cpp:227-312).  The reference evaluates each
ranked candidate with P1 (equivalence::check_equivalence, :257-261) and, when
Equivalent, P2 (rewriter::verify_rewrite, :274-277); the first candidate passing
both wins (:285-307).  Here P2 for every ranked candidate of a spec runs as ONE
batched GPU launch, and the host's P1 runs only on P2 survivors in rank order —
the accepted candidate is the same because the acceptance rule is P1 AND P2 in
rank order (P2 is not a subset of P1, so P1 stays the final word).

Specs are tried in configuration order; a truncated spec (more candidates than
the cap) sets too_many and is skipped, and the loop stops after the spec that
lifted or once too_many is set (:243-246, :311).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .evaluator import Evaluator, RecordedTestsets, encode_bindings
from .spec import ApiSpec


@dataclass
class SpecCandidates:
    """What matching::find_matchings + rank_candidates produced for one spec."""

    spec: ApiSpec
    ranked: list  # CandidateBinding dicts in rank order (lex_score, provenance)
    truncated: bool = False


@dataclass
class LiftOutcome:
    status: str  # "Lifted" | "NoMatch" | "TooManyCandidates"
    winning_api: str = ""
    winner_rank: int = -1
    binding: Optional[dict] = None
    p1_calls: int = 0  # host P1 evaluations the GPU screen left to do
    evaluated: list = field(default_factory=list)  # (api, rank, verdict) of candidates decided before the winner
    status_detail: str = ""  # pipeline.cpp:314-325


def lift_function(specs: list, testsets: RecordedTestsets, user_ptrs: list, p1: Callable[[ApiSpec, dict], str],
                  evaluator: Optional[Evaluator] = None, p2_override: Optional[Callable] = None) -> LiftOutcome:
    """`p1(spec, binding)` returns the reference verdict name ("Equivalent",
    "NotEquivalent", "Inconclusive").  `p2_override(spec, arr_map, size_map)` may
    supply P2 verdicts (bool array) instead of the GPU (used by CPU-only tests)."""
    ev = evaluator
    out = LiftOutcome("NoMatch")
    too_many = False
    any_filtered = False
    for sc in specs:
        any_filtered |= len(sc.ranked) > 0
        if sc.truncated:
            too_many = True
            continue
        if sc.ranked:
            am, sm = encode_bindings(sc.ranked, sc.spec, user_ptrs, testsets.int_params)
            if p2_override is not None:
                p2_ok = np.asarray(p2_override(sc.spec, am, sm), dtype=bool)
            else:
                ev = ev or Evaluator()
                p2_ok = ev.eval_bindings(sc.spec, testsets, am, sm).ok
            for rank, cand in enumerate(sc.ranked):
                if not p2_ok[rank]:
                    # the reference would have run P1 here and, if Equivalent,
                    # recorded VerificationFailed; report the P2 outcome
                    out.evaluated.append((sc.spec.name, rank, "P2-rejected"))
                    continue
                out.p1_calls += 1
                verdict = p1(sc.spec, cand)
                out.evaluated.append((sc.spec.name, rank, verdict))
                if verdict == "Equivalent":
                    out.status, out.winning_api, out.winner_rank, out.binding = "Lifted", sc.spec.name, rank, cand
                    return out
        if too_many:
            break
    if too_many:
        out.status, out.status_detail = "TooManyCandidates", "candidate cap exceeded"
    else:  # pipeline.cpp:318-324
        out.status = "NoMatch"
        out.status_detail = "no candidate proved equivalent" if any_filtered else "no candidate passed the constraints"
    return out
