"""Per-kernel shares of a step from an ncu launch list.

    python tools/launch_shares.py LAUNCHES.csv STEPS OUT.json [STEP_MS]

LAUNCHES.csv: `ncu --metrics gpu__time_duration.sum --csv` of tools/replay_step.py
(STEPS replayed steps, nothing else captured).  ncu serialises the launches and
runs them cold, so the absolute sum exceeds a concurrent step; the SHARE of each
kernel is what bench.py quotes (roofline.step_share).
"""
import csv
import json
import sys
from collections import defaultdict

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}


def shares(path: str, steps: int) -> dict:
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    per = defaultdict(float)
    count = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("<")[0]
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1.0)
        per[name] += v / steps
        count[name] += 1
    total = sum(per.values())
    return {"launches_per_step": sum(count.values()) / steps, "serialised_ms_per_step": total,
            "kernels": {k: {"ms_per_step": v, "share": v / total, "launches_per_step": count[k] / steps}
                        for k, v in sorted(per.items(), key=lambda kv: -kv[1])}}


if __name__ == "__main__":
    out = shares(sys.argv[1], int(sys.argv[2]))
    k1 = out["kernels"].get("k_screen_conv_pairs", {})
    out["k_screen_conv_pairs_share"] = k1.get("share")
    if len(sys.argv) > 4:
        out["step_ms_replayed"] = float(sys.argv[4])
    out["source"] = sys.argv[1]
    with open(sys.argv[3], "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "kernels"}, indent=1))
