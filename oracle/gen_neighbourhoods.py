"""Reference-verified neighbourhoods of the conv spaces' passing bindings
(TEST INFRASTRUCTURE — run in the build container, where the reference compiles).

The conv spaces (2.3e9 / 9.3e9 bindings) are too large to sweep with the
reference.  tests/golden/conv_passing.json holds every conv space's full passing
list at T = 16 and T = 10 as the GPU reports it (tools/conv_passing.py on a B200);
this script asks the UNMODIFIED reference (oracle/_ref/ref_tool neighbourhood:
rewriter::verify_rewrite per binding) for the verdict — first failing test and
reason at T = 16 — of every binding within RADIUS of each of those passing
indices and of each pruned candidate's index, and stores them in
tests/golden/conv_neighbourhoods.npz (keys "<stem>x<spec>:idx|fail_t|reason").

    python oracle/gen_neighbourhoods.py [radius]
"""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")
TOOL = os.path.join(HERE, "_ref", "ref_tool")


def main():
    radius = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    passing = json.load(open(os.path.join(GOLDEN, "conv_passing.json")))
    out = {}
    for key in sorted(passing):
        stem, spec = key.rsplit("x", 1)
        meta = json.load(open(os.path.join(GOLDEN, stem + ".json")))
        centers = set(passing[key]["16"]["passing"]) | set(meta["specs"][spec]["pruned_index"])
        if not centers:
            continue
        r = subprocess.run([TOOL, "neighbourhood", stem, spec, "16", str(radius), str(os.cpu_count() or 8),
                            *map(str, sorted(centers))], capture_output=True, text=True, check=True)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        out[f"{key}:idx"] = np.asarray(d["idx"], dtype=np.uint64)
        out[f"{key}:fail_t"] = np.asarray(d["fail_t"], dtype=np.int8)
        out[f"{key}:reason"] = np.asarray(d["reason"], dtype=np.int8)
        out[f"{key}:centers"] = np.asarray(sorted(centers), dtype=np.uint64)
        print(f"{key}: {len(d['idx'])} bindings, {int((out[f'{key}:reason'] == 0).sum())} passing", flush=True)
    np.savez_compressed(os.path.join(GOLDEN, "conv_neighbourhoods.npz"), radius=np.int64(radius), **out)


if __name__ == "__main__":
    main()
