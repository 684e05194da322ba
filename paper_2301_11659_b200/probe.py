"""P2 input-set builder: the binding-independent half of verify_rewrite.

Restates, for building the recorded test sets the GPU evaluator consumes:
  * liftc::Rng           include/liftc/rng.hpp:13-48  (mt19937_64 draws, mix())
  * api::SizeRules       include/liftc/api_spec.hpp:80-97, api_spec.cpp:178-222
  * analysis::draw_sizes          src/analysis.cpp:25-71
  * analysis::build_probe_image   src/analysis.cpp:73-98
  * the per-test seeding of verify_rewrite  src/rewriter.cpp:235-245
The mt19937_64 stream itself is produced by libatc_b200 (atc_mt64_*), which uses
std::mt19937_64 — fully specified by the C++ standard.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._lib import lib

MASK64 = (1 << 64) - 1
PROBE_REGION_LEN = 65536  # analysis.cpp:23


def rng_mix(seed: int, tag: str) -> int:
    """Rng::mix (rng.hpp:32-44): FNV-1a of the tag, xor seed, splitmix64 finalizer."""
    h = 1469598103934665603
    for c in tag.encode():
        h ^= c
        h = (h * 1099511628211) & MASK64
    x = (seed ^ h) & MASK64
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


class Rng:
    """liftc::Rng over a std::mt19937_64 stream; tracks the draw position."""

    def __init__(self, seed: int):
        self.seed = seed & MASK64
        self.pos = 0
        self._buf = np.empty(0, dtype=np.uint64)
        self._buf_start = 0

    def next(self) -> int:
        i = self.pos - self._buf_start
        if i < 0 or i >= len(self._buf):
            self._buf = np.empty(64, dtype=np.uint64)
            self._buf_start = self.pos
            lib().atc_mt64_raw(self.seed, self.pos, 64, self._buf.ctypes.data)
            i = 0
        self.pos += 1
        return int(self._buf[i])

    def uniform_int(self, lo: int, hi: int) -> int:  # rng.hpp:20-23
        span = ((hi - lo) & MASK64) + 1
        return lo + int(self.next() % span)

    def uniform_real(self, lo: float, hi: float) -> float:  # rng.hpp:25-28
        out = np.empty(1, dtype=np.float64)
        lib().atc_mt64_uniform(self.seed, self.pos, 1, lo, hi, 0, out.ctypes.data)
        self.pos += 1
        return float(out[0])

    def fill_uniform(self, n: int, lo: float, hi: float, round_f32: bool) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        lib().atc_mt64_uniform(self.seed, self.pos, n, lo, hi, 1 if round_f32 else 0, out.ctypes.data)
        self.pos += n
        return out


@dataclass
class UserDerived:  # api_spec.hpp:74-78
    is_product: bool = False
    terms: list = field(default_factory=list)  # [(coef, name)]
    constant: int = 0


@dataclass
class SizeRules:  # api_spec.hpp:80-91
    ranges: dict = field(default_factory=dict)
    equal_groups: list = field(default_factory=list)
    multiple_of: dict = field(default_factory=dict)
    power_of_two: set = field(default_factory=set)
    derived: dict = field(default_factory=dict)

    @staticmethod
    def from_json(j: dict) -> "SizeRules":  # api_spec.cpp:178-206
        r = SizeRules()
        for name, rg in (j.get("ranges") or {}).items():
            r.ranges[name] = (int(rg[0]), int(rg[1]))
        for g in j.get("equal") or []:
            r.equal_groups.append(list(g))
        for name, k in (j.get("multiple_of") or {}).items():
            r.multiple_of[name] = int(k)
        for name in j.get("power_of_two") or []:
            r.power_of_two.add(name)
        for name, dj in (j.get("derived") or {}).items():
            d = UserDerived()
            d.is_product = dj.get("kind", "affine") == "product"
            if d.is_product:
                d.terms = [(1, t) for t in dj["terms"]]
            else:
                d.terms = [(int(t[0]), t[1]) for t in dj["terms"]]
                d.constant = int(dj.get("constant", 0))
            r.derived[name] = d
        return r


def eval_derived(d: UserDerived, values: dict) -> int:  # api_spec.cpp:208-222
    if d.is_product:
        v = 1
        for _, name in d.terms:
            v *= values[name]
        return v
    v = d.constant
    for c, name in d.terms:
        v += c * values[name]
    return v


def _c_div(a: int, b: int) -> int:
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


def draw_sizes(int_params: list, rules: SizeRules, rng: Rng):
    """analysis::draw_sizes (analysis.cpp:25-71). Returns the size map or None."""
    out: dict = {}
    head = {}
    for g in rules.equal_groups:
        for m in g:
            if g:
                head[m] = g[0]
    for name in int_params:
        if name in rules.derived:
            continue
        h = head.get(name)
        if h is not None and h in out:
            out[name] = out[h]
            continue
        lo, hi = rules.ranges.get(name, (2, 8))
        v = rng.uniform_int(lo, hi)
        m = rules.multiple_of.get(name)
        if m is not None and m > 1:
            v = _c_div(v + m - 1, m) * m
            if v > hi:
                v = _c_div(lo + m - 1, m) * m
        out[name] = v
    # std::map iteration order = sorted names
    pending = len(rules.derived)
    while pending > 0:
        before = pending
        for name in sorted(rules.derived):
            if name in out:
                continue
            rule = rules.derived[name]
            if not all(t[1] in out for t in rule.terms):
                continue
            out[name] = eval_derived(rule, out)
            pending -= 1
        if pending == before:
            return None
    for name in int_params:
        if out[name] < 1:
            return None
    return out


@dataclass
class Param:
    name: str
    kind: str  # "ptr" | "int" | "float"
    elem: str  # "f32" | "f64" | "i64"


def build_probe_image(params: list, sizes: dict, rng: Rng, region_len: int = PROBE_REGION_LEN,
                      streams: dict | None = None):
    """analysis::build_probe_image (analysis.cpp:73-98): params in signature order.
    `streams`, when given, receives each region's first stream position."""
    regions, floats = {}, {}
    for p in params:
        if p.kind == "float":
            floats[p.name] = rng.uniform_real(-1.0, 1.0)
        elif p.kind == "ptr":
            if streams is not None:
                streams[p.name] = rng.pos
            regions[p.name] = rng.fill_uniform(region_len, -1.0, 1.0, p.elem == "f32")
    return regions, floats


@dataclass
class ProbeTest:
    t: int
    ok: bool
    sizes: dict
    regions: dict  # name -> np.float64[65536] (initial contents)
    floats: dict
    seed: int = 0  # the test's Rng seed
    streams: dict = field(default_factory=dict)  # name -> stream position of the region's first draw


def p2_test_inputs(function: str, params: list, rules: SizeRules, p2seed: int, t: int) -> ProbeTest:
    """verify_rewrite's per-test inputs (rewriter.cpp:236-245)."""
    rng = Rng(rng_mix(p2seed, f"verify:{function}:{t}"))
    int_params = [p.name for p in params if p.kind == "int"]
    sizes = None
    for _ in range(20):
        sizes = draw_sizes(int_params, rules, rng)
        if sizes is not None:
            break
    if sizes is None:
        return ProbeTest(t, False, {}, {}, {})
    streams: dict = {}
    regions, floats = build_probe_image(params, sizes, rng, streams=streams)
    return ProbeTest(t, True, sizes, regions, floats, rng.seed, streams)


def fnv1a_bytes(a: np.ndarray) -> int:
    """FNV-1a 64 over the raw bytes (used to pin regenerated regions)."""
    b = np.frombuffer(np.ascontiguousarray(a).tobytes(), dtype=np.uint8)
    h = np.uint64(1469598103934665603)
    prime = np.uint64(1099511628211)
    with np.errstate(over="ignore"):
        for x in b:
            h = (h ^ np.uint64(x)) * prime
    return int(h)

