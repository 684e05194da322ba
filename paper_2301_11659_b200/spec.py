"""API spec model (mirror of include/liftc/api_spec.hpp:26-66 / src/api_spec.cpp).

Loads the same JSON the reference loads from proj/specs/*.json, validates it like
api_spec.cpp:91-128 (including the canonical dim order of :116-119) and encodes
it into the atc_spec_desc decode table consumed by the GPU evaluator.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import _lib


class SpecError(RuntimeError):
    """api::SpecError (api_spec.hpp:42-44)."""


@dataclass
class ApiParam:
    name: str
    kind: str  # "array" | "int" | "float"
    liveness: str = "livein"  # "livein" | "liveout" | "liveinout"
    dims: list = field(default_factory=list)
    element_type: str = "any"
    role: str = ""
    domain: list = field(default_factory=list)  # extended specs: the constants this param may bind


@dataclass
class ApiSpec:
    name: str
    semantics: str
    layout: str = "rowmajor"
    affix: str = ""
    params: list = field(default_factory=list)
    ranges: dict = field(default_factory=dict)
    derived: dict = field(default_factory=dict)

    def find(self, n: str):
        for p in self.params:
            if p.name == n:
                return p
        return None

    def position(self, n: str) -> int:
        for i, p in enumerate(self.params):
            if p.name == n:
                return i
        return -1

    def arrays(self) -> list:
        return [p for p in self.params if p.kind == "array"]

    def size_params(self) -> list:
        return [p for p in self.params if p.kind == "int"]

    def float_scalars(self) -> list:
        return [p for p in self.params if p.kind == "float"]

    # ---- GPU decode table --------------------------------------------------
    def to_desc(self) -> "_lib.SpecDesc":
        d = _lib.SpecDesc()
        d.semantics = _lib.SEM_GEMM if self.semantics == "gemm" else _lib.SEM_CONV2D
        d.layout = _lib.LAYOUT_ROW if self.layout == "rowmajor" else _lib.LAYOUT_COL
        arrays, sizes = self.arrays(), self.size_params()
        if len(arrays) > _lib.ATC_MAX_ARRAYS or len(sizes) > _lib.ATC_MAX_SIZES:
            raise SpecError(f"{self.name}: too many params for the GPU decode table")
        d.n_arrays, d.n_sizes = len(arrays), len(sizes)
        size_index = {p.name: q for q, p in enumerate(sizes)}
        roles = _lib.ARRAY_ROLES[self.semantics]
        for a, p in enumerate(arrays):
            if p.role not in roles:
                raise SpecError(f"{self.name}: array '{p.name}' has no {self.semantics} role")
            d.array_role[a] = roles[p.role]
            d.array_livein[a] = 1 if p.liveness == "livein" else 0
            d.array_ndims[a] = len(p.dims)
            for k, dim in enumerate(p.dims):
                d.array_dims[a][k] = size_index[dim]
        for r in range(_lib.ATC_SZ_COUNT):
            d.role_size[r] = -1
        table = _lib.SIZE_ROLES if self.semantics == "gemm" else _lib.CONV_SIZE_ROLES
        base = 0 if self.semantics == "gemm" else len(_lib.SIZE_ROLES)
        for q, p in enumerate(sizes):
            if p.role in table:
                d.role_size[base + table.index(p.role)] = q
        return d


EXT_SEMANTICS = {"gemm_ext": "gemm", "conv2d_ext": "conv2d"}


def ext_desc(spec: ApiSpec) -> "_lib.SpecExt":
    """atc_spec_ext of an extended spec (include/atc_b200.h, "Extended semantics"):
    the base table of the underlying semantics, the extended size roles, the float
    roles and the constant tables (size_map entry n_ints + c -> iconst[c]; float_map
    entry n_user_floats + c -> fconst[c], c = the value's position in its table)."""
    if spec.semantics not in EXT_SEMANTICS:
        raise SpecError(f"{spec.name}: not an extended spec")
    base = ApiSpec(spec.name, EXT_SEMANTICS[spec.semantics], spec.layout, spec.affix,
                   [p for p in spec.params if not (p.kind == "int" and p.role in _lib.EXT_SIZE_ROLES)])
    d = _lib.SpecExt()
    b = base.to_desc()
    sizes = spec.size_params()
    size_index = {p.name: q for q, p in enumerate(sizes)}
    d.base = b
    d.base.semantics = _lib.SEM_GEMM_EXT if spec.semantics == "gemm_ext" else _lib.SEM_CONV2D_EXT
    # the base table was built without the extended params: re-index against every size param
    d.base.n_sizes = len(sizes)
    for a, p in enumerate(spec.arrays()):
        for k, dim in enumerate(p.dims):
            d.base.array_dims[a][k] = size_index[dim]
    table = _lib.SIZE_ROLES if EXT_SEMANTICS[spec.semantics] == "gemm" else _lib.CONV_SIZE_ROLES
    off = 0 if EXT_SEMANTICS[spec.semantics] == "gemm" else len(_lib.SIZE_ROLES)
    for r in range(_lib.ATC_SZ_COUNT):
        d.base.role_size[r] = -1
    for r in range(_lib.ATC_XR_COUNT):
        d.ext_role_size[r] = -1
    for q, p in enumerate(sizes):
        if p.role in table:
            d.base.role_size[off + table.index(p.role)] = q
        elif p.role in _lib.EXT_SIZE_ROLES:
            d.ext_role_size[_lib.EXT_SIZE_ROLES.index(p.role)] = q
    floats = spec.float_scalars()
    d.n_floats = len(floats)
    for r in range(_lib.ATC_FR_COUNT):
        d.role_float[r] = -1
    for f, p in enumerate(floats):
        if p.role in _lib.EXT_FLOAT_ROLES:
            d.role_float[_lib.EXT_FLOAT_ROLES.index(p.role)] = f
    ic, fc = ext_constants(spec)
    if len(ic) > _lib.ATC_MAX_CONSTS or len(fc) > _lib.ATC_MAX_CONSTS or len(floats) > _lib.ATC_MAX_FLOATS:
        raise SpecError(f"{spec.name}: too many constants / floats for the GPU decode table")
    d.n_iconst, d.n_fconst = len(ic), len(fc)
    for i, v in enumerate(ic):
        d.iconst[i] = v
    for i, v in enumerate(fc):
        d.fconst[i] = v
    return d


def ext_constants(spec: ApiSpec) -> tuple:
    """The constant tables of an extended spec: distinct int / float domain values in
    order of appearance."""
    ic, fc = [], []
    for p in spec.params:
        for v in p.domain:
            tab = ic if p.kind == "int" else fc
            v = int(v) if p.kind == "int" else float(v)
            if v not in tab:
                tab.append(v)
    return ic, fc


def _validate(spec: ApiSpec) -> None:  # api_spec.cpp:91-128
    if spec.semantics not in ("gemm", "conv2d", *EXT_SEMANTICS):
        raise SpecError(f"{spec.name}: semantics must be gemm, conv2d, gemm_ext or conv2d_ext")
    names = set()
    for p in spec.params:
        if p.name in names:
            raise SpecError(f"{spec.name}: duplicate param '{p.name}'")
        names.add(p.name)
    has_output = False
    for p in spec.params:
        if p.kind == "array":
            if not p.dims:
                raise SpecError(f"{spec.name}: array '{p.name}' has no dims")
            for d in p.dims:
                dp = spec.find(d)
                if dp is None or dp.kind != "int":
                    raise SpecError(f"{spec.name}: dim '{d}' of '{p.name}' is not an int size param")
            if p.liveness != "livein":
                has_output = True
            if p.element_type not in ("f32", "f64", "any"):
                raise SpecError(f"{spec.name}: bad element_type '{p.element_type}'")
        elif p.liveness != "livein":
            raise SpecError(f"{spec.name}: scalar '{p.name}' must be livein")
        p.dims = sorted(p.dims, key=spec.position)  # canonical dim order
    if not has_output:
        raise SpecError(f"{spec.name}: no output array")
    for name, d in spec.derived.items():
        if spec.find(name) is None:
            raise SpecError(f"{spec.name}: derived unknown param '{name}'")
        for _, t in d["terms"]:
            if spec.find(t) is None:
                raise SpecError(f"{spec.name}: derived term unknown param '{t}'")


def parse_api_spec(j: dict) -> ApiSpec:
    """api_spec.cpp:130-163 (from an already-parsed JSON object)."""
    layout = j.get("layout", "rowmajor")
    if layout not in ("rowmajor", "colmajor"):
        raise SpecError(f"{j['name']}: bad layout '{layout}'")
    kinds = {"array": "array", "int": "int", "float": "float"}
    spec = ApiSpec(name=j["name"], semantics=j["semantics"], layout=layout, affix=j.get("affix", ""))
    for pj in j["params"]:
        kind = kinds.get(pj["kind"])
        if kind is None:
            raise SpecError(f"bad param kind '{pj['kind']}'")
        spec.params.append(ApiParam(name=pj["name"], kind=kind, liveness=pj.get("liveness", "livein").lower(),
                                    dims=list(pj.get("dims", [])), element_type=pj.get("element_type", "any"),
                                    role=pj.get("role", ""), domain=list(pj.get("domain", []))))
    s = j.get("sampling") or {}
    for name, r in (s.get("ranges") or j.get("ranges") or {}).items():
        spec.ranges[name] = (int(r[0]), int(r[1]))
    for name, d in (s.get("derived") or j.get("derived") or {}).items():
        spec.derived[name] = {"terms": [(int(c), t) for c, t in d["terms"]], "constant": int(d.get("constant", 0)),
                              "slack": int(d.get("slack", 0))}
    _validate(spec)
    return spec
