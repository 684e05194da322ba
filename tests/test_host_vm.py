"""The compiled host VM (integration/host_vm.cpp) and the host analyses on it
(integration/host_phases.cpp) against the reference interpreter and analyses
(SURVEY.md §8(f).1, §8(f).3), on every function of every corpus file — no GPU:
raw executions (status, fault message, step count, final images bit for bit,
write flags, return value), detect_liveness, detect_dims of every pointer (dims
and slow dim), and P1 check_equivalence (verdict, tests_run, detail,
counterexample) on every ranked candidate plus a strided sample of each unpruned
space.  oracle/_ref/adapter_check is built from the unmodified reference by
oracle/Makefile (test infrastructure)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


@pytest.mark.skipif(not os.path.exists(TOOL), reason="oracle/_ref/adapter_check not built")
def test_host_vm_matches_reference_interpreter_and_analyses():
    r = subprocess.run([TOOL, "host"], capture_output=True, text=True, timeout=1200)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert r.returncode == 0, r.stderr + json.dumps(lines[:5])[:4000]
    last = lines[-1]
    assert last["mismatches"] == 0
    assert last["executions"] >= 150 and last["liveness"] >= 55 and last["dims"] >= 150 and last["p1"] >= 2000
    # the surveys of every pointer share one run: far below the reference's time
    assert last["host_vm_ms"]["dims"] * 4 < last["reference_ms"]["dims"]
