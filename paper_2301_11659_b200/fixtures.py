"""Recorded-corpus fixtures (tests/golden/) -> evaluator inputs.

A fixture holds what the reference host records for one corpus function: its
signature, size rules and seeds, and for every P2 test t the sizes plus the
positions/values the ORIGINAL run changed (the final-minus-init diff of
interp::execute, rewriter.cpp:247).  The initial probe regions are not stored;
they are regenerated bit-exactly from the seeds (probe.p2_test_inputs) and pinned
against the FNV-1a the reference dump recorded.  Fixtures are produced by
oracle/gen_golden.py from the compiled reference; this module only reads them.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .evaluator import BindingSpace, RecordedTestsets
from .probe import Param, SizeRules, p2_test_inputs
from .spec import ApiSpec, parse_api_spec

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


@lru_cache(maxsize=None)
def specs() -> dict:
    with open(os.path.join(GOLDEN, "specs.json")) as f:
        return {name: parse_api_spec(j) for name, j in json.load(f).items()}


def spec(name: str) -> ApiSpec:
    return specs()[name]


def stems() -> list:
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


@dataclass
class Program:
    stem: str
    meta: dict
    arrays: dict  # npz contents

    @property
    def function(self) -> str:
        return self.meta["function"]

    @property
    def params(self) -> list:
        return [Param(p["name"], p["kind"], p["elem"]) for p in self.meta["params"]]

    @property
    def user_ptrs(self) -> list:
        return [p["name"] for p in self.meta["params"] if p["kind"] == "ptr"]

    @property
    def user_ints(self) -> list:
        return [p["name"] for p in self.meta["params"] if p["kind"] == "int"]

    @property
    def rules(self) -> SizeRules:
        return SizeRules.from_json(self.meta.get("size_rules") or {})

    def rules64(self) -> SizeRules:
        r = self.rules
        for u in self.user_ints:
            r.ranges[u] = (64, 64)
        return r

    @property
    def p2seed(self) -> int:
        return int(self.meta["p2seed"])

    def spec_names(self) -> list:
        return list((self.meta.get("specs") or {}).keys())

    def space(self, spec_name: str) -> BindingSpace:
        return BindingSpace(self.user_ptrs, self.user_ints, spec(spec_name))

    def verdicts(self, spec_name: str, which: str = "p2") -> dict:
        s = self.meta["specs"][spec_name]
        out = {"idx": self.arrays[s["idx"]], "p1": self.arrays[s["p1"]]}
        if which == "p2_64":
            out["fail_t"] = self.arrays[s["p2_64_fail_t"]]
            out["reason"] = self.arrays[s["p2_64_reason"]]
        else:
            out["fail_t"] = self.arrays[s["p2_fail_t"]]
            out["reason"] = self.arrays[s["p2_reason"]]
        out["enumerated"] = s["enumerated"]
        out["count"] = s["count"]
        return out

    def testsets(self, T: int = 16, variant: str = "testsets", check=None) -> RecordedTestsets:
        """Rebuild the recorded test sets; `check(region, meta)` may pin each
        regenerated init region (tests pass an FNV-1a comparison)."""
        rules = self.rules64() if variant == "testsets64" else self.rules
        params = self.params
        ptrs = [p for p in params if p.kind == "ptr"]
        ints = np.zeros((T, len(self.user_ints)), dtype=np.int64)
        float_names = [p.name for p in params if p.kind == "float"]
        floats = np.zeros((T, len(float_names)), dtype=np.float64)
        init, final, ok = [], [], np.zeros(T, dtype=np.int32)
        seeds, skips = np.zeros(T, dtype=np.uint64), np.zeros((T, len(ptrs)), dtype=np.uint64)
        for rec in self.meta[variant][:T]:
            t = rec["t"]
            pt = p2_test_inputs(self.function, params, rules, self.p2seed, t)
            if pt.ok:
                floats[t] = [pt.floats[n] for n in float_names]
            if rec["status"] == "draw_failed" or not pt.ok:
                assert rec["status"] == "draw_failed" and not pt.ok, f"{self.stem} t={t}: draw mismatch"
                init.append([np.zeros(len(pt.regions.get(p.name, [0] * 65536))) for p in ptrs])
                final.append(None)
                continue
            assert {k: int(v) for k, v in rec["sizes"].items()} == pt.sizes, f"{self.stem} t={t}: sizes differ"
            ints[t] = [pt.sizes[u] for u in self.user_ints]
            seeds[t] = pt.seed
            skips[t] = [pt.streams[p.name] for p in ptrs]
            init.append([pt.regions[p.name] for p in ptrs])
            if check is not None:
                for p in ptrs:
                    check(pt.regions[p.name], rec["regions"][p.name])
            if rec["status"] != "Normal":
                final.append(None)
                continue
            fin = []
            for p in ptrs:
                f = pt.regions[p.name].copy()
                key = rec["regions"][p.name]["diff_key"]
                f[self.arrays[key + "_pos"]] = self.arrays[key + "_val"]
                fin.append(f)
            final.append(fin)
            ok[t] = 1
        return RecordedTestsets(params, ints, init, final, ok, seeds=seeds, skips=skips, floats=floats)


@lru_cache(maxsize=None)
def load(stem: str) -> Program:
    with open(os.path.join(GOLDEN, stem + ".json")) as f:
        meta = json.load(f)
    path = os.path.join(GOLDEN, stem + ".npz")
    arrays = dict(np.load(path)) if os.path.exists(path) else {}
    return Program(stem, meta, arrays)


def pipeline_reports() -> list:
    with open(os.path.join(GOLDEN, "pipeline.json")) as f:
        return json.load(f)


def conv_passing() -> dict:
    """tests/golden/conv_passing.json: every conv space's full passing list at T = 16
    and T = 10 as the GPU sweep reports it, keyed "<stem>x<spec>" (tools/conv_passing.py);
    pinned by the reference's verdicts on their neighbourhoods (conv_neighbourhoods)."""
    with open(os.path.join(GOLDEN, "conv_passing.json")) as f:
        return json.load(f)


def conv_neighbourhoods() -> dict:
    """tests/golden/conv_neighbourhoods.npz (oracle/gen_neighbourhoods.py): the
    reference's verify_rewrite verdicts (T = 16) of every binding within `radius` of
    each passing index and pruned candidate of each conv space:
    {key: {"idx", "fail_t", "reason", "centers"}}, plus "radius"."""
    z = np.load(os.path.join(GOLDEN, "conv_neighbourhoods.npz"))
    out = {"radius": int(z["radius"])}
    for name in z.files:
        if ":" in name:
            key, field = name.split(":")
            out.setdefault(key, {})[field] = z[name]
    return out
