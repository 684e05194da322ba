"""The reference-side adapter (integration/atc_liftc_adapter.cpp), compiled against
the unmodified reference into oracle/_ref/adapter_check, driving libatc_b200 from the
reference's own C++ (test infrastructure: it links the oracle build)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "oracle", "_ref", "adapter_check")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(TOOL), reason="oracle/_ref/adapter_check not built")]


def _run(*args, timeout=900):
    r = subprocess.run([TOOL, *args], capture_output=True, text=True, timeout=timeout)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    return r.returncode, lines, r.stderr


def test_adapter_reproduces_reference_pipeline():
    """Reference lift_program vs analysis + matching + ranking + GPU P2 batch + host
    P1 on survivors: same status, spec, rank and binding for every corpus program."""
    rc, lines, err = _run("corpus")
    assert rc == 0, err + json.dumps(lines[-3:])
    assert lines[-1]["mismatches"] == 0
    lifted = [x for x in lines[:-1] if x.get("gpu_status") == "Lifted"]
    assert len(lifted) == 29  # 23 GEMM + 6 conv


def test_adapter_gpu_dispatch_bit_identical():
    """make_gpu_dispatch vs make_oracle_dispatch on every lifted corpus function."""
    rc, lines, err = _run("dispatch")
    assert rc == 0, err
    assert lines[-1]["mismatches"] == 0


def test_adapter_unpruned_stress_space():
    """naive_ld x gemm_rowmajor_ld (279,936 bindings) as one ranked list: the GPU
    screen leaves one survivor, host P1 accepts it (index 44790, the identity)."""
    rc, lines, err = _run("unpruned", "naive_ld", "gemm_rowmajor_ld", "10")
    assert rc == 0, err
    j = lines[-1]
    assert j["bindings"] == 279936 and j["p2_passed"] == 1 and j["winner"] == 44790 and j["p1_calls"] == 1


def test_adapter_routed_dispatch():
    """make_gpu_routed_dispatch vs rewriter::make_routed_dispatch (rewriter.cpp:183-213):
    identical cpu/xpu labels on every lifted corpus function, bit-identical results on
    the exact route; f32 GEMM (row/col/ld) and conv calls labelled "xpu" run on the
    tcgen05 backends within their stated TF32 / 3xTF32 bounds; "cpu" stays exact."""
    rc, lines, err = _run("routed")
    assert rc == 0, err + json.dumps([x for x in lines if not x.get("ok", True)][:3])
    assert lines[-1]["mismatches"] == 0
    direct = [x for x in lines if "direct" in x]
    assert len(direct) == 8 and all(x["ok"] for x in direct)
