#!/usr/bin/env python
"""Benchmark of the B200 candidate-evaluation stage (and the API backends).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload corpus|stress|naive64]
    python bench.py --impl reference ...     # the reference CPU path, same metric

One step = one pass of the batched IO-equivalence check (P2, rewriter.cpp:215-284)
over the workload: every binding of every unpruned corpus binding space against
16 recorded random input sets, each binding decided (all 16 pass, or the first
failing set found), plus — with N > 1 ranks — the one packed all-gather that
combines the ranks' results (shard.reduce_packed: first passing index, reason
histograms, passing lists).  Spaces are partitioned over ranks by
workloads.plan_shards; value = bindings decided per second (all ranks).

`--gpus N` without a torchrun environment re-launches itself under
`torch.distributed.run` with N ranks (one process per GPU).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate bindings IO-checked/sec (GEMM+conv corpus)"
UNIT = "bindings/s"
N_SM = 148


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return j.get("hbm_gbs", 6547.8), j.get("bf16_tflops", 1636.5), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def _lib_mapped() -> list:
    """In-tree product libraries mapped into this process (/proc/self/maps)."""
    try:
        with open("/proc/self/maps") as f:
            return sorted({ln.split()[-1] for ln in f if "libatc_b200" in ln})
    except OSError:
        return []


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(n: int) -> int:
    """Re-launch this command as n ranks (torch.distributed.run, one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.proc = device, None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ reference --
def reference_rates(seconds: float, threads: int) -> dict:
    """Times the unmodified reference (oracle/_ref/ref_tool: rewriter::verify_rewrite,
    T=16, all host threads) on bounded random samples of the GEMM and conv spaces."""
    tool = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    if not os.path.exists(tool):
        return {}
    out = {}
    for key, stem, spec in (("conv", "conv_direct", "conv2d"), ("gemm", "naive_ld", "gemm_rowmajor_ld")):
        r = subprocess.run([tool, "time-p2", stem, spec, "16", str(seconds), str(threads)], capture_output=True,
                           text=True, timeout=seconds * 10 + 120)
        if r.returncode == 0:
            out[key] = json.loads(r.stdout.strip().splitlines()[-1])
    return out


def weighted_rate(rates: dict, jobs) -> float:
    """Bindings/s of the reference on this workload: total / sum(count_i / rate_i)."""
    total = sum(j.count for j in jobs)
    t = 0.0
    for j in jobs:
        key = "conv" if j.spec.semantics == "conv2d" else "gemm"
        t += j.count / rates[key]["bindings_per_s"]
    return total / t


def run_reference_arm(args, spaces, rank):
    """The reference's own CPU path (oracle/_ref/ref_tool = the unmodified liftc
    sources) on this arm's metric.  `spaces` are counts only (workloads.
    corpus_spaces): this process never loads libatc_b200 — asserted below."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    per = max(2.0, 20.0 / max(1, args.steps))
    vals = []
    rates = {}
    for _ in range(max(1, args.steps)):
        rates = reference_rates(per / 2, threads)
        if not rates:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_tool not built"}))
            return
        vals.append(weighted_rate(rates, spaces))
    v = float(np.median(vals))
    mapped = _lib_mapped()
    assert not mapped, f"the reference arm must not load the product library: {mapped}"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "dtype": "f64",
            "data": "recorded corpus test sets (regenerated from seeds by the reference itself)",
            "config": _config(args, spaces),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"rewriter::verify_rewrite T=16 on random bindings of conv_direct x conv2d and "
                                       f"naive_ld x gemm_rowmajor_ld, {per / 2:.0f}s each per step, weighted by the "
                                       f"workload's binding counts",
                             "rates": {k: r["bindings_per_s"] for k, r in rates.items()}},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "native_libs_mapped": mapped}
    print(json.dumps(line))


def _backend_cpu_baseline() -> dict:
    """The reference's backend loop nests on the host: profitability::xpu_gemm (all
    host threads) on a 512-row M-slice of the 8192^3 sgemm, and run_reference's
    f64 conv2d on one image of the conv2_x 3x3 layer."""
    tool = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    out = {}
    if not os.path.exists(tool):
        return out
    try:
        r = subprocess.run([tool, "time-xpu-gemm", "512", "8192", "8192"], capture_output=True, text=True, timeout=300)
        j = json.loads(r.stdout.strip().splitlines()[-1])
        out["xpu_gemm_gflops"] = j["gflops"]
        out["xpu_gemm_threads"] = j["threads"]
        out["xpu_gemm_sample"] = "512 x 8192 x 8192 M-slice of the 8192^3 workload"
        r = subprocess.run([tool, "time-conv", "1", "64", "58", "58", "64", "3", "3"], capture_output=True, text=True,
                           timeout=300)
        j = json.loads(r.stdout.strip().splitlines()[-1])
        out["run_reference_conv_gflops"] = j["gflops"]
        out["run_reference_conv_sample"] = "N=1, 64->64, 3x3, 58x58 (one image of conv2_x.b), f64, 1 thread"
    except Exception as e:  # the baseline is reported, not required
        out["error"] = str(e)
    return out


def _profiles_json(suffix: str):
    """The newest committed profiles/<round><suffix> (e.g. _ncu_summary.json)."""
    d = os.path.join(ROOT, "profiles")
    try:
        files = sorted(f for f in os.listdir(d) if f.endswith(suffix))
        with open(os.path.join(d, files[-1])) as f:
            return files[-1], json.load(f)
    except Exception:
        return None, None


def _ncu(prefix: str) -> dict:
    """The committed ncu --set full summary of one kernel (newest round first)."""
    d = os.path.join(ROOT, "profiles")
    for name in sorted((f for f in os.listdir(d) if f.endswith("_ncu_summary.json")), reverse=True):
        with open(os.path.join(d, name)) as f:
            for row in json.load(f):
                if prefix in row["kernel"]:
                    return dict(row, summary=name)
    return {}


def _config(args, jobs):
    return {"workload": args.workload, "programs": len({j.stem for j in jobs}), "spaces": len(jobs),
            "bindings_per_step": int(sum(j.count for j in jobs)), "tests_per_binding": 16,
            "parallelism": f"dp{args.gpus}: spaces partitioned over ranks (workloads.plan_shards), one packed "
                           f"all-gather of the results per step",
            "l2": "flushed (256 MB write) between steps"}


def _jobs(workload: str):
    from paper_2301_11659_b200 import workloads

    if workload == "corpus":
        jobs = workloads.corpus_jobs()
    elif workload == "stress":
        jobs = workloads.stress_jobs()
    else:
        jobs = workloads.naive64_jobs()
    # conv spaces first: in the e2e pass their (long) evaluation overlaps the
    # uploads of the gemm programs' test sets
    jobs.sort(key=lambda j: j.spec.semantics != "conv2d")
    return jobs


def _spaces(workload: str):
    from paper_2301_11659_b200 import workloads

    if workload == "corpus":
        sp = workloads.corpus_spaces()
    elif workload == "stress":
        sp = [s for s in workloads.corpus_spaces(("gemm",)) if s.stem == "naive_ld" and s.spec_name == "gemm_rowmajor_ld"]
    else:
        sp = [s for s in workloads.corpus_spaces(("gemm",)) if s.stem == "naive_f32"]
    sp.sort(key=lambda j: j.spec.semantics != "conv2d")
    return sp


def _time_events(fn, stream, torch, reps: int, warm: int = 2) -> list:
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return ts


# ------------------------------------------------------------------ ours -------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="corpus", choices=["corpus", "stress", "naive64"])
    ap.add_argument("--no-sgemm", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the config sub-keys and e2e variants")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args.gpus))
    rank, world, local = _env_rank()
    args.gpus = world if world > 1 else args.gpus
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        # counts only: the reference arm never regenerates test sets, so it never
        # loads libatc_b200 (the probe-image generator lives there)
        run_reference_arm(args, _spaces(args.workload), rank)
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    from paper_2301_11659_b200 import _lib, shard, workloads
    from paper_2301_11659_b200.evaluator import Evaluator

    jobs = _jobs(args.workload)
    ctx = _lib.Context(local)
    # a real (non-legacy) stream: every library launch and every CUDA event of
    # the timed region go to this one stream
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    _lib.check(ctx.handle, _lib.lib().atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
    ev = Evaluator(ctx)
    shards = workloads.plan_shards(jobs, rank, world)
    for j, (b, e) in zip(jobs, shards):
        if e > b:
            j.ts.upload(ctx)  # device-resident recorded test sets for the kernel-level number
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    items = [(j.spec, j.ts, j.space, b, e) for j, (b, e) in zip(jobs, shards)]
    sweep = ev.sweep(items, cap=1 << 16)  # atc_enum_batch: one CUDA graph of every space after run 1

    last = {}

    def run_local():
        res = last["local"] = sweep.run()
        return res

    def step():
        # with N ranks the results meet in ONE packed all-gather inside the timed
        # step (shard.sharded_step; tests/test_multiproc.py runs the same flow on gloo)
        return shard.sharded_step(jobs, shards, run_local, dist, device="cuda") if dist else run_local()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    step_ms = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush between timed iterations (not timed)
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            results = step()
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    combined = results if dist else shard.reduce_packed(results, None)
    total_ms = _max_over_ranks(sum(step_ms), dist, torch)
    ms_per_step = total_ms / args.steps
    bindings = sum(j.count for j in jobs)
    value = bindings / (ms_per_step / 1e3)

    # one more step, profiled (eager launches with per-kernel events): the launch
    # count and the K1/K2 split of one step; not part of the timed region
    prof = _lib.Profile()
    _lib.check(ctx.handle, _lib.lib().atc_profile_start(ctx.handle))
    sweep.run()
    _lib.check(ctx.handle, _lib.lib().atc_profile_read(ctx.handle, C.byref(prof)))

    # ---- correctness of what was timed (the combined, all-rank results)
    correct, summary = _check(jobs, combined)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic: recorded corpus P2 test sets regenerated from the reference seeds",
        "config": _config(args, jobs), "correct": correct, "passing_sample": summary,
        # every library kernel of one step (counted by the profiled step) x timed steps;
        # the timed steps replay them as one CUDA graph per step
        "gpu_launches": int(prof.kernels) * args.steps,
        "launches_per_step": int(prof.kernels),
    }
    # ---- e2e through the C ABI with host buffers (pinned), uploads inside the region
    e2e_ms, h2d, d2h, e2e_ok = _e2e_prepared(args, ctx, ev, jobs, shards, stream, torch, dist, last["local"])
    line["correct"] = correct and e2e_ok
    line["e2e"] = {"value": bindings / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                   "inputs": "per program, every step: the P2 tests' Rng seeds + region stream positions + int "
                             "values + the original runs' final-minus-init entries, written into the program's "
                             "test-set handle (atc_testsets_update_seeded, needed_only: the GPU regenerates the "
                             "region prefixes an evaluation can read), then the prepared sweep "
                             "(atc_enum_batch_run: one CUDA-graph replay), its result block D2H"
                             + (" and the packed all-gather" if dist else "")}
    if not args.no_extras:
        e2e_once_ms, h2d_once, d2h_once = _e2e(args, ctx, jobs, shards, stream, torch, dist, seeded=True)
        e2e_full_ms, h2d_full, _ = _e2e(args, ctx, jobs, shards, stream, torch, dist, seeded=False)
        line["e2e"]["one_shot"] = {"value": bindings / (e2e_once_ms / 1e3), "ms_per_step": e2e_once_ms,
                                   "h2d_bytes_per_step": h2d_once, "d2h_bytes_per_step": d2h_once,
                                   "inputs": "handles created and freed every step (atc_testsets_upload_seeded) "
                                             "and one eager atc_eval_enumerated_many"}
        line["e2e"]["full_regions"] = {"value": bindings / (e2e_full_ms / 1e3), "ms_per_step": e2e_full_ms,
                                       "h2d_bytes_per_step": h2d_full,
                                       "inputs": "every 65,536-element init and final region "
                                                 "(atc_testsets_upload_async)"}

    line["roofline"] = _roofline(ctx, ev, jobs, stream, torch, prof, ms_per_step)
    line["k2_confirm"] = {"ms_per_step": prof.confirm_ms, "survivors_per_step": prof.survivors,
                          "note": "sum of K2 launch durations of one eager profiled step (concurrent streams "
                                  "overlap, so this is not a wall-clock share)",
                          "fp64_pipe": _fp64_pipe(ctx)}
    if not args.no_extras and args.workload == "corpus":
        line["configs"] = {"config1_naive_f32_64": _config1(ev, stream, torch, dist),
                           "config4_stress": _config4(ev, stream, torch, dist),
                           "config2_pruned": _config2_pruned(ctx, ev, stream, torch)}
    if not args.no_sgemm:
        # replaced-call backends: sgemm split along M, conv along batch, no collective
        # on the data path; the time of the slowest rank is the job time
        line["replaced_gemm"] = _sgemm_bench(ctx, stream, torch, dist, world)
        line["replaced_conv"] = _conv_bench(ctx, stream, torch, dist, world)
    if rank == 0:
        line["clocks"] = clocks.summary()
        if not args.no_cpu_baseline and world == 1:
            rates = reference_rates(6.0, os.cpu_count() or 1)
            if rates:
                line["cpu_baseline"] = {
                    "value": weighted_rate(rates, jobs), "unit": UNIT, "cores": os.cpu_count() or 1,
                    "kind": "reference",
                    "sample": "rewriter::verify_rewrite T=16, random bindings of conv_direct x conv2d and naive_ld x "
                              "gemm_rowmajor_ld, 6 s each, weighted by this workload's binding counts",
                    "rates": {k: r["bindings_per_s"] for k, r in rates.items()},
                    "backends": _backend_cpu_baseline()}
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def _check(jobs, combined):
    """Every full space's combined passing set must equal the reference dump; conv
    spaces (sampled dumps) must agree with every reference-decided index the dump
    holds (the pinned conv passing sets of tests/golden when present)."""
    correct, summary = True, {}
    for j, (pl, first, hist, complete) in zip(jobs, combined):
        ok = complete and (first if first >= 0 else None) == (pl[0] if pl else None)
        ok = ok and int(hist.sum()) == j.count
        if j.expected_pass is not None:
            ok = ok and pl == j.expected_pass
        else:
            ok = ok and _sampled_agree(j, pl)
        correct &= bool(ok)
        if pl:
            summary[f"{j.stem}x{j.spec_name}"] = pl[:4]
    return correct, summary


def _sampled_agree(j, passing) -> bool:
    """A sampled (conv) dump: the reference's verdict of every dumped index (the
    random sample and the +-4096 neighbourhoods of every passing index and pruned
    candidate, tests/golden/conv_neighbourhoods.npz) agrees with membership in
    `passing`, and `passing` is the pinned list (tests/golden/conv_passing.json)."""
    from paper_2301_11659_b200 import fixtures

    key = f"{j.stem}x{j.spec_name}"
    T = j.ts.n_tests
    v = fixtures.load(j.stem).verdicts(j.spec_name)
    nb = fixtures.conv_neighbourhoods().get(key)
    idx, ft = v["idx"].astype(np.int64), v["fail_t"]
    if nb is not None:
        idx, ft = np.concatenate([idx, nb["idx"].astype(np.int64)]), np.concatenate([ft, nb["fail_t"]])
    ref_ok = (ft < 0) | (ft >= T)
    got = np.isin(idx, np.asarray(passing, dtype=np.int64))
    pinned = fixtures.conv_passing().get(key, {}).get(str(T))
    return bool(np.array_equal(ref_ok, got)) and (pinned is None or list(passing) == pinned["passing"])


def _fp64_pipe(ctx):
    """K2's FP64-pipe utilisation (ncu) against a DFMA peak measured on
    this box (atc_measure_dfma_peak)."""
    from paper_2301_11659_b200 import _lib

    peak = C.c_double(0)
    rc = _lib.lib().atc_measure_dfma_peak(ctx.handle, C.byref(peak))
    k2a, k2b = _ncu("k_confirm_t0"), _ncu("k_confirm_warp")
    return {"dfma_peak_gflops_measured": peak.value if rc == 0 else None,
            "k2a_fp64_pipe_pct": k2a.get("fp64_pipe_pct"), "k2b_fp64_pipe_pct": k2b.get("fp64_pipe_pct"),
            "note": "ncu sm__inst_executed_pipe_fp64 (% of peak, active cycles) of the K2 launches in "
                    "profiles/<round>_ncu_summary.json; K2 is latency bound (short dependent FP64 chains "
                    "per output), not FP64-throughput bound"}


def _roofline(ctx, ev, jobs, stream, torch, prof, ms_per_step):
    """The dominant kernel, K1 k_screen_conv_pairs on conv_direct x conv2d
    (2,324,522,934 bindings in one launch).  It is integer-issue bound (its
    operands are L1/L2-resident tables; DRAM traffic is ~0.2 MB per launch), so
    the roofline is the SM issue rate: achieved = warp instructions of that launch
    (ncu smsp__inst_executed.sum, profiles/) / its duration measured live here
    with CUDA events on the launching stream; peak = 148 SMs x 4 schedulers x 1
    warp-instruction/cycle x the SM clock."""
    from paper_2301_11659_b200 import _lib

    j = next((j for j in jobs if j.stem == "conv_direct" and j.spec_name == "conv2d"), None)
    if j is None:
        return None
    sw = ev.sweep([(j.spec, j.ts, j.space, 0, j.count)])
    sw.run()
    k1 = []
    L = _lib.lib()
    for _ in range(7):
        p = _lib.Profile()
        _lib.check(ctx.handle, L.atc_profile_start(ctx.handle))
        sw.run()
        _lib.check(ctx.handle, L.atc_profile_read(ctx.handle, C.byref(p)))
        if p.screen_launches == 1:
            k1.append(p.screen_ms)
    sw.close()
    k1_ms = float(np.median(k1)) if k1 else None
    n = _ncu("k_screen_conv_pairs")
    clk = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            clk = json.load(f).get("sm_max_mhz")
    except Exception:
        pass
    clk = clk or 1965.0
    peak = N_SM * 4 * clk * 1e6 / 1e9  # G warp-instructions / s
    wi = n.get("warp_instructions")
    achieved = wi / (k1_ms / 1e3) / 1e9 if (wi and k1_ms) else None
    shares_name, shares = _profiles_json("_launch_shares.json")
    out = {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "G warp-instructions/s",
           "frac": achieved / peak if achieved else None,
           "traffic": (n.get("dram_read", 0) + n.get("dram_write", 0)) if n else None,
           "kernel": "k_screen_conv_pairs (K1) on conv_direct x conv2d, 2,324,522,934 bindings per launch",
           "kernel_ms": k1_ms, "kernel_ms_how": "CUDA events around the launch on its stream, median of 7",
           "peak_how": f"{N_SM} SMs x 4 warp schedulers x 1 issue/cycle x {clk:.0f} MHz (sm_max_mhz)",
           "ncu": {"summary": n.get("summary"), "warp_instructions": wi, "duration_ms": (n.get("duration") or 0) * 1e3,
                   "issue_slots_busy_pct": n.get("issue_slots_busy_pct"), "alu_pipe_pct": n.get("alu_pipe_pct"),
                   "dram_GBps": ((n.get("dram_read", 0) + n.get("dram_write", 0)) / n["duration"] / 1e9)
                   if n.get("duration") else None,
                   "thread_instructions_per_binding": wi * 32 / 2324522934 if wi else None},
           "k1_ms_per_step_eager": prof.screen_ms,
           "note": "SURVEY 8d's operand bytes (8 B x (extA+extB+extC) per binding) are never streamed by the "
                   "factorised screen, so no HBM fraction is claimed; see ncu.dram_GBps for the real traffic"}
    if shares:
        out["step_share"] = dict(shares, file=f"profiles/{shares_name}")
    return out


def _config1(ev, stream, torch, dist):
    """Config 1: naive_f32 at 64^3 x {gemm_rowmajor, gemm_colmajor} (162 bindings
    each, 16 sets): one prepared sweep of both spaces (latency bound)."""
    from paper_2301_11659_b200 import workloads

    jobs = workloads.naive64_jobs()
    sw = ev.sweep([(j.spec, j.ts, j.space, 0, j.count) for j in jobs])
    res = [None]

    def run():
        res[0] = sw.run()

    ts = _time_events(run, stream, torch, 20)
    sw.close()
    ms = _max_over_ranks(float(np.median(ts)), dist, torch)
    n = sum(j.count for j in jobs)
    ok = all(r[0].tolist() == j.expected_pass for r, j in zip(res[0], jobs))
    return {"value": n / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "bindings": n, "correct": ok,
            "passing": {j.spec_name: r[0].tolist() for r, j in zip(res[0], jobs)},
            "workload": "naive_f32.ml, m = n = k = 64 (P2 sets drawn with the [64,64] rule), T=16, both dense specs"}


def _config4(ev, stream, torch, dist):
    """Config 4 alone: naive_ld x gemm_rowmajor_ld, 279,936 bindings, 16 sets."""
    from paper_2301_11659_b200 import workloads

    j = workloads.stress_jobs()[0]
    sw = ev.sweep([(j.spec, j.ts, j.space, 0, j.count)])
    res = [None]

    def run():
        res[0] = sw.run()

    ts = _time_events(run, stream, torch, 20)
    sw.close()
    ms = _max_over_ranks(float(np.median(ts)), dist, torch)
    return {"value": j.count / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "bindings": j.count,
            "correct": res[0][0][0].tolist() == j.expected_pass == [44790],
            "workload": "naive_ld.ml x gemm_rowmajor_ld, full unpruned space, T=16"}


def _config2_pruned(ctx, ev, stream, torch):
    """Config 2 as the pipeline sees it: each (program, spec)'s ranked candidate
    list (1-2 bindings) checked at T=16 — the latency of one candidate-loop P2
    batch.  device: test sets resident; e2e: per program the seeded upload
    (needed-only regions generated on the GPU) + every spec's list + free."""
    from paper_2301_11659_b200 import workloads

    lists = workloads.pruned_lists()
    ok = True
    dev = []
    for stem, sname, spec, ts, am, sm, ref in lists:
        v = [None]

        def run():
            v[0] = ev.eval_bindings(spec, ts, am, sm)

        dev.append(float(np.median(_time_events(run, stream, torch, 5))))
        ok &= all(r is None or r == bool(g) for r, g in zip(ref, v[0].ok))
    by_prog = {}
    for item in lists:
        by_prog.setdefault(item[0], []).append(item)
    e2e = []
    for stem, items in by_prog.items():
        ts = items[0][3]

        def run():
            h = ts.upload_seeded(ctx, needed_only=True)
            for _, _, spec, _, am, sm, _ in items:
                ev.eval_bindings(spec, ts, am, sm, handle=h)
            h.free()

        e2e.append(float(np.median(_time_events(run, stream, torch, 5))))
    return {"lists": len(lists), "bindings": int(sum(x[4].shape[0] for x in lists)), "programs": len(by_prog),
            "device_ms_per_list_median": float(np.median(dev)), "device_ms_total": float(np.sum(dev)),
            "e2e_ms_per_program_median": float(np.median(e2e)), "e2e_ms_total": float(np.sum(e2e)),
            "correct": bool(ok),
            "workload": "every GEMM/conv corpus program's ranked (pruned) candidates per spec, T=16 "
                        "(atc_eval_bindings; e2e adds atc_testsets_upload_seeded per program)"}


def _e2e_prepared(args, ctx, ev, jobs, shards, stream, torch, dist, want):
    """The e2e metric through the prepared-sweep API: one test-set handle per program
    and one atc_enum_batch, created once; every timed step rewrites every handle from
    pinned host buffers (atc_testsets_update_seeded: seeds, stream positions, int
    values, final-minus-init entries -> H2D, probe images regenerated on the GPU),
    replays the sweep and reads its result block back (atc_enum_batch_run).  The
    passing lists of the last step must equal the device-resident run's."""
    import dataclasses

    from paper_2301_11659_b200 import _lib
    from paper_2301_11659_b200.evaluator import _TestsetHandle

    active = [(i, j, sh) for i, (j, sh) in enumerate(zip(jobs, shards)) if sh[1] > sh[0]]
    L = _lib.lib()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    progs, h2d = {}, 0
    for _, j, _ in active:
        if j.stem in progs:
            continue
        s, keep = j.ts.seeded_struct(needed_only=True)
        keep = [pin(a) for a in keep]  # same order as the struct's fields below
        (s.int_values, s.ptr_is_f32, s.region_len, s.test_ok, s.stream_seed, s.stream_skip, s.diff_off,
         s.diff_pos, s.diff_val) = [a.ctypes.data for a in keep]
        out = C.c_void_p()
        _lib.check(ctx.handle, L.atc_testsets_upload_seeded(ctx.handle, C.byref(s), C.byref(out)))
        h = _TestsetHandle(ctx, out.value)
        holder = dataclasses.replace(j.ts, _handles={id(ctx): h})
        progs[j.stem] = (s, keep, h, holder)
        h2d += sum(a.nbytes for a in keep)
    sweep = ev.sweep([(j.spec, progs[j.stem][3], j.space, b, e) for _, j, (b, e) in active], cap=1 << 16)
    d2h = len(active) * (2 + 256 + 8) * 8  # the batch's result block (atc_enum_batch_run)

    vals = list(progs.values())
    structs = (_lib.SeededTestsets * len(vals))(*[v[0] for v in vals])
    hptrs = (C.c_void_p * len(vals))(*[v[2].value for v in vals])

    from paper_2301_11659_b200 import shard

    empty = (np.zeros(0, np.uint64), 0, np.zeros(5, np.int64))

    def one():  # one C call rewrites every program's handle, then the graph replay
        _lib.check(ctx.handle, L.atc_testsets_update_seeded_many(ctx.handle, hptrs, structs, len(vals)))
        got = sweep.run()
        if dist:  # the same single packed all-gather as the device-resident step
            full = [empty] * len(jobs)
            for g, (i, _, _) in zip(got, active):
                full[i] = g
            shard.reduce_packed(full, dist, device="cuda")
        return got

    for _ in range(2):  # eager + capture
        one()
    times = []
    for _ in range(max(1, args.steps)):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        got = one()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ok = all(g[0].tolist() == want[i][0].tolist() and g[1] == want[i][1] for g, (i, _, _) in zip(got, active))
    sweep.close()
    for _, _, h, holder in progs.values():
        holder._handles.clear()
        h.free()
    ms = _max_over_ranks(float(np.mean(times)), dist, torch)
    return ms, h2d, d2h, ok


def _e2e(args, ctx, jobs, shards, stream, torch, dist, seeded=True):
    """Same metric through the C ABI from pinned host buffers, every program's test
    sets uploaded every step (copies inside the timed region), then
    atc_eval_enumerated_many.  seeded: atc_testsets_upload_seeded (the tests' Rng
    seeds + stream positions + the original runs' final-minus-init entries; the
    probe images are generated on the GPU); else atc_testsets_upload_async with the
    full 65,536-element regions."""
    from paper_2301_11659_b200 import _lib

    # only the spaces (and so the programs) this rank has work in
    active = [(j, sh) for j, sh in zip(jobs, shards) if sh[1] > sh[0]]
    jobs, shards = [a[0] for a in active], [a[1] for a in active]

    L = _lib.lib()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    progs, h2d = {}, 0
    for j in jobs:
        if j.stem in progs:
            continue
        ts = j.ts
        if seeded:
            s, keep = ts.seeded_struct(needed_only=True)
            keep = [pin(a) for a in keep]  # same order as the struct's fields below
            (s.int_values, s.ptr_is_f32, s.region_len, s.test_ok, s.stream_seed, s.stream_skip, s.diff_off,
             s.diff_pos, s.diff_val) = [a.ctypes.data for a in keep]
            progs[j.stem] = (s, keep, L.atc_testsets_upload_seeded)
            h2d += sum(a.nbytes for a in keep)
            continue
        # one pinned block per program for the initial regions and one for the
        # final regions, (t, pointer) back to back: one DMA each
        nP = len(ts.ptrs)
        lens = [len(ts.init[0][p]) for p in range(nP)]
        total = ts.n_tests * sum(lens)
        blk_i = torch.empty(total, dtype=torch.float64, pin_memory=True).numpy()
        blk_f = torch.zeros(total, dtype=torch.float64, pin_memory=True).numpy()
        pinned, o = [], 0
        for t in range(ts.n_tests):
            row_i, row_f = [], []
            for p in range(nP):
                a, f = blk_i[o:o + lens[p]], blk_f[o:o + lens[p]]
                a[:] = ts.init[t][p]
                row_i.append(a)
                if ts.final[t] is not None:
                    f[:] = ts.final[t][p]
                    row_f.append(f)
                else:
                    row_f.append(None)
                o += lens[p]
            pinned.append((row_i, row_f))
        from paper_2301_11659_b200.evaluator import RecordedTestsets

        pts = RecordedTestsets(ts.params, ts.ints, [r[0] for r in pinned],
                               [None if any(x is None for x in r[1]) else r[1] for r in pinned], ts.test_ok)
        s, keep = pts.c_struct()
        progs[j.stem] = (s, keep, L.atc_testsets_upload_async)
        h2d += 2 * s.n_tests * s.n_ptrs * 65536 * 8
    d2h = 0
    static = [(j.spec.to_desc(), np.ascontiguousarray(j.space.perms, dtype=np.uint8), np.zeros(1 << 16, np.uint64))
              for j in jobs]

    def one():
        nonlocal d2h
        d2h = 0
        handles = {}
        for stem, (s, _, upload) in progs.items():
            out = C.c_void_p()
            # copy stream; each space's kernels wait only for their own program's upload
            _lib.check(ctx.handle, upload(ctx.handle, C.byref(s), C.byref(out)))
            handles[stem] = out.value
        arr = (_lib.EnumJob * len(jobs))()
        for i, (j, (b, e)) in enumerate(zip(jobs, shards)):
            desc, perms, surv = static[i]
            jb = arr[i]
            jb.spec = C.cast(C.pointer(desc), C.c_void_p)
            jb.ts = handles[j.stem]
            jb.perms, jb.n_perms = perms.ctypes.data, perms.shape[0]
            jb.begin, jb.end = b, e
            jb.survivors, jb.cap = surv.ctypes.data, 1 << 16
        _lib.check(ctx.handle, L.atc_eval_enumerated_many(ctx.handle, arr, len(jobs), 0))
        for i in range(len(jobs)):
            d2h += 8 * min(arr[i].n_survivors, 1 << 16) + 8 + 40
        for h in handles.values():
            L.atc_testsets_free(ctx.handle, h)

    one()
    times = []
    for _ in range(max(1, args.steps)):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.mean(times))
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, h2d, d2h


# ResNet-50 conv layers expressible as valid, unit-stride NCHW (SURVEY.md §8d
# config 5; 3x3 layers on host-padded inputs): (name, C, K, R, H_in)
RESNET_LAYERS = [("conv2_x.a 1x1", 64, 64, 1, 56), ("conv2_x.b 3x3", 64, 64, 3, 58),
                 ("conv2_x.c 1x1", 64, 256, 1, 56), ("conv3_x.b 3x3", 128, 128, 3, 30),
                 ("conv3_x.a 1x1", 512, 128, 1, 28), ("conv4_x.b 3x3", 256, 256, 3, 16),
                 ("conv5_x.b 3x3", 512, 512, 3, 9)]


def _max_over_ranks(ms, dist, torch):
    if dist is None:
        return ms
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _time_ms(fn, stream, torch, reps=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def _library_tf32(torch):
    """A library comparison point (not on the product path): cuBLAS / cuDNN with TF32."""
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    torch.backends.cudnn.benchmark = True


def _conv_bench(ctx, stream, torch, dist=None, world=1, batch=256):
    """Replaced-call conv2d backend on tcgen05 (TF32): global batch `batch`,
    split across ranks (batch // world images each)."""
    from paper_2301_11659_b200 import _lib

    L = _lib.lib()
    out = {"batch": batch, "per_rank_batch": batch // world, "precision": "tf32", "layers": []}
    tot_flops = tot_ms = 0.0
    gb = batch
    batch = gb // world
    for name, c, k, r, h in RESNET_LAYERS:
        oh = h - r + 1
        x = torch.empty(batch, c, h, h, device="cuda").uniform_(-1, 1)
        w = torch.empty(k, c, r, r, device="cuda").uniform_(-1, 1)
        y = torch.empty(batch, k, oh, oh, device="cuda")

        def run():
            _lib.check(ctx.handle, L.atc_conv2d_nchw_device(ctx.handle, x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                                            batch, c, h, h, k, r, r, _lib.PREC_TF32,
                                                            C.c_void_p(stream.cuda_stream)))

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = _max_over_ranks(float(np.median(ts)), dist, torch)
        flops = 2.0 * gb * k * oh * oh * c * r * r
        # first, middle and last image (a tile's rows can reach into the next image)
        pick = [0, batch // 2, batch - 1]
        ref = torch.nn.functional.conv2d(x[pick].double(), w.double())
        err = ((y[pick].double() - ref).abs() / (1 + ref.abs())).max().item()
        _library_tf32(torch)
        lib_ms = _max_over_ranks(_time_ms(lambda: torch.nn.functional.conv2d(x, w), stream, torch), dist, torch)
        out["layers"].append({"layer": name, "C": c, "K": k, "RxS": f"{r}x{r}", "H": h, "ms": ms,
                              "tflops": flops / (ms / 1e3) / 1e12, "max_rel_err_vs_fp64": err,
                              "cudnn_tf32_tflops": flops / (lib_ms / 1e3) / 1e12})
        tot_flops += flops
        tot_ms += ms
        del x, w, y
    out["total_tflops"] = tot_flops / (tot_ms / 1e3) / 1e12
    out["note"] = ("includes the per-call NCHW->NHWC input transpose and KCRS->KRSC weight reorder; "
                   "cudnn_tf32_tflops = torch conv2d (cuDNN, TF32, benchmark mode) on the same tensors, "
                   "a library comparison point only")
    return out


def _sgemm_bench(ctx, stream, torch, dist=None, world=1):
    """Replaced-call backend: row-major FP32 sgemm 8192^3 (cpu_gemm contract) on
    tcgen05, split along M across ranks (8192/world rows each, B replicated)."""
    from paper_2301_11659_b200 import _lib

    L = _lib.lib()
    M = n = k = 8192
    m = M // world
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1, generator=g)
    b = torch.empty(k, n, device="cuda").uniform_(-1, 1, generator=g)
    c = torch.empty(m, n, device="cuda")
    out = {}
    for prec_name, prec in (("tf32", _lib.PREC_TF32), ("3xtf32", _lib.PREC_3XTF32)):
        def run():
            _lib.check(ctx.handle, L.atc_sgemm_rm_device(ctx.handle, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n,
                                                         k, prec, C.c_void_p(stream.cuda_stream)))

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        times = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = _max_over_ranks(float(np.median(times)), dist, torch)
        tflops = 2.0 * M * n * k / (ms / 1e3) / 1e12
        ref = (a[:256].double() @ b.double())
        err = ((c[:256].double() - ref).abs() / (1 + ref.abs())).max().item()
        out[prec_name] = {"ms": ms, "tflops": tflops, "max_rel_err_vs_fp64": err}
    # the cpu_gemm contract end to end: atc_sgemm_rm on pinned host buffers (H2D of A and
    # B, the tcgen05 GEMM, D2H of C inside the call), wall clock of the call
    ha, hb = a.cpu().pin_memory(), b.cpu().pin_memory()
    hc = torch.empty(m, n).pin_memory()
    host_ms = []
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(ctx.handle, L.atc_sgemm_rm(ctx.handle, ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k,
                                              _lib.PREC_TF32))
        if it:
            host_ms.append((time.perf_counter() - t0) * 1e3)
    hms = _max_over_ranks(float(np.median(host_ms)), dist, torch)
    out["e2e_host_buffers"] = {"ms": hms, "tflops": 2.0 * M * n * k / (hms / 1e3) / 1e12, "precision": "tf32",
                               "h2d_bytes": (m * k + k * n) * 4, "d2h_bytes": m * n * 4,
                               "call": "atc_sgemm_rm on pinned host A, B, C (wall clock of the call)"}
    del ha, hb, hc
    _library_tf32(torch)
    cublas_ms = _max_over_ranks(_time_ms(lambda: torch.matmul(a, b, out=c), stream, torch), dist, torch)
    out["cublas_tf32_tflops"] = 2.0 * M * n * k / (cublas_ms / 1e3) / 1e12
    # the TF32 dense peak, measured on this box: cuBLAS TF32 at 8192^3, best of 10
    # (one rank's full problem; the library's own best is the attainable ceiling)
    tf32_peak = _tf32_peak(torch, stream)
    out["shape"] = [M, n, k]
    out["per_rank_rows"] = m
    g = _ncu("k_tc_gemm2")
    out["roofline"] = {"bound": "tensor", "achieved": out["tf32"]["tflops"], "peak": tf32_peak, "unit": "TFLOP/s",
                       "frac": out["tf32"]["tflops"] / tf32_peak,
                       "traffic": (g.get("dram_read", 0) + g.get("dram_write", 0)) if g else None,
                       "algorithmic_bytes": (m * k + k * n + m * n) * 4,
                       "tensor_pipe_active_pct": g.get("tensor_pipe_active_pct"),
                       "ncu_summary": g.get("summary"),
                       "peak_kind": "measured: cuBLAS TF32 8192^3 (torch.matmul fp32, allow_tf32), best of 10, this box",
                       "fp32_contract": {"precision": "3xtf32", "tflops": out["3xtf32"]["tflops"],
                                         "frac_of_tf32_peak_over_3": out["3xtf32"]["tflops"] / (tf32_peak / 3),
                                         "note": "3xTF32 issues 3 TF32 MMAs per useful MAC and honours the "
                                                 "cpu_gemm 1e-3*(1+|c|) cross-check on random data"}}
    return out


def _tf32_peak(torch, stream) -> float:
    _library_tf32(torch)
    N = 8192
    a = torch.empty(N, N, device="cuda").uniform_(-1, 1)
    b = torch.empty(N, N, device="cuda").uniform_(-1, 1)
    c = torch.empty(N, N, device="cuda")
    ts = _time_events(lambda: torch.matmul(a, b, out=c), stream, torch, 10, warm=3)
    del a, b, c
    return 2.0 * N ** 3 / (min(ts) / 1e3) / 1e12


if __name__ == "__main__":
    main()
