"""Summarise ncu captures (gpurun_out/*.ncu-rep) into profiles/<round>_ncu_summary.json.

    python profiles/summarize.py r1 gpurun_out/prof_screen_rows_v3.ncu-rep gpurun_out/prof_tc_gemm_r1.ncu-rep ...
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_per_sm",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__grid_size": "grid_size",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "second": 1, "s": 1}


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:120], "report": os.path.basename(rep)}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if v != v:  # NaN: metric not collected for this launch
                    continue
                v *= SCALE.get(units[i], 1)
                d[name] = v
        if len(d) > 3:
            res.append(d)
    return res


if __name__ == "__main__":
    tag, reps = sys.argv[1], sys.argv[2:]
    allr = [x for rep in reps for x in summarize(rep)]
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{tag}_ncu_summary.json")
    with open(path, "w") as f:
        json.dump(allr, f, indent=1)
    print(json.dumps(allr, indent=1))
