"""Every conv corpus space swept whole on the GPU at T = 16 and T = 10: the full
passing lists (gpurun_out/conv_passing.json), the centres of the reference-verified
neighbourhoods in tests/golden/conv_neighbourhoods.npz (oracle/gen_neighbourhoods.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2301_11659_b200 import Evaluator, workloads  # noqa: E402


def main():
    ev = Evaluator()
    out = {}
    for T in (16, 10):
        jobs = workloads.corpus_jobs(T, ("conv",))
        res = ev.eval_enumerated_many([(j.spec, j.ts, j.space, 0, j.count) for j in jobs], cap=1 << 16)
        for j, (passing, n, hist) in zip(jobs, res):
            assert n == len(passing)
            out.setdefault(f"{j.stem}x{j.spec_name}", {})[str(T)] = {"passing": [int(x) for x in passing],
                                                                      "hist": [int(x) for x in hist]}
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/conv_passing.json", "w"), indent=1)
    print(json.dumps({k: v["16"]["passing"][:8] for k, v in out.items()}))


if __name__ == "__main__":
    main()
