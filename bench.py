#!/usr/bin/env python
"""Benchmark of the B200 candidate-evaluation stage (and the sgemm backend).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload corpus|stress]
    python bench.py --impl reference ...     # the reference CPU path, same metric

One step = one pass of the batched IO-equivalence check (P2, rewriter.cpp:215-284)
over the workload: every binding of every unpruned corpus binding space against
16 recorded random input sets, each binding decided (all 16 pass, or the first
failing set found).  Bindings are block-partitioned across ranks (one process per
GPU); the per-space passing sets are gathered and the first passing index reduced
with an NCCL all-reduce MIN.  value = bindings decided per second (all ranks).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate bindings IO-checked/sec (GEMM+conv corpus)"
UNIT = "bindings/s"


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return j.get("hbm_gbs", 6547.8), j.get("bf16_tflops", 1636.5), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


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


def run_reference_arm(args, jobs, rank):
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
        vals.append(weighted_rate(rates, jobs))
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "dtype": "f64",
            "data": "recorded corpus test sets (regenerated from seeds)", "config": _config(args, jobs),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"rewriter::verify_rewrite T=16 on random bindings of conv_direct x conv2d and "
                                       f"naive_ld x gemm_rowmajor_ld, {per / 2:.0f}s each per step, weighted by the "
                                       f"workload's binding counts",
                             "rates": {k: r["bindings_per_s"] for k, r in rates.items()}},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
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


def _ncu_summary():
    """The newest committed ncu summary (profiles/<round>_ncu_summary.json)."""
    d = os.path.join(ROOT, "profiles")
    try:
        files = sorted(f for f in os.listdir(d) if f.endswith("_ncu_summary.json"))
        with open(os.path.join(d, files[-1])) as f:
            return json.load(f)
    except Exception:
        return []


def _fp64_pipe(ctx, ncu):
    """K2's FP64-pipe utilisation (ncu) against a DFMA peak measured on
    this box (atc_measure_dfma_peak)."""
    from paper_2301_11659_b200 import _lib

    peak = C.c_double(0)
    rc = _lib.lib().atc_measure_dfma_peak(ctx.handle, C.byref(peak))
    get = lambda name: next((d for d in ncu if d["kernel"].startswith(name)), {})
    k2a, k2b = get("k_confirm_t0"), get("k_confirm_warp")
    return {"dfma_peak_gflops_measured": peak.value if rc == 0 else None,
            "k2a_fp64_pipe_pct": k2a.get("fp64_pipe_pct"), "k2b_fp64_pipe_pct": k2b.get("fp64_pipe_pct"),
            "note": "ncu sm__inst_executed_pipe_fp64 (% of peak, active cycles) of the K2 launches in "
                    "profiles/<round>_ncu_summary.json; K2 is latency bound (short dependent FP64 chains "
                    "per output), not FP64-throughput bound"}


def _config(args, jobs):
    return {"workload": args.workload, "programs": len({j.stem for j in jobs}), "spaces": len(jobs),
            "bindings_per_step": int(sum(j.count for j in jobs)), "tests_per_binding": 16,
            "parallelism": f"dp{args.gpus}: large spaces block-partitioned over ranks, small spaces dealt whole",
            "l2": "flushed (256 MB write) between steps"}


# ------------------------------------------------------------------ ours -------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="corpus", choices=["corpus", "stress"])
    ap.add_argument("--no-sgemm", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank, world, local = _env_rank()
    args.gpus = world if world > 1 else args.gpus

    from paper_2301_11659_b200 import workloads

    jobs = workloads.corpus_jobs() if args.workload == "corpus" else workloads.stress_jobs()
    # conv spaces first: in the e2e pass their (long) evaluation overlaps the
    # uploads of the gemm programs' test sets
    jobs.sort(key=lambda j: j.spec.semantics != "conv2d")
    if args.impl == "reference":
        run_reference_arm(args, jobs, rank)
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    from paper_2301_11659_b200 import _lib
    from paper_2301_11659_b200.evaluator import Evaluator

    ctx = _lib.Context(local)
    # a real (non-legacy) stream: every library launch and every CUDA event of
    # the timed region go to this one stream
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    _lib.check(ctx.handle, _lib.lib().atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
    ev = Evaluator(ctx)
    shards = workloads.plan_shards(jobs, rank, world)
    for j in jobs:
        j.ts.upload(ctx)  # device-resident recorded test sets for the kernel-level number
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    items = [(j.spec, j.ts, j.space, b, e) for j, (b, e) in zip(jobs, shards)]
    sweep = ev.sweep(items, cap=1 << 16)  # atc_enum_batch: one CUDA graph of every space after run 1

    def step():
        return sweep.run()

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
    # one more step, profiled (eager launches with per-kernel events): the K1/K2
    # split and the launch count of one step; not part of the timed region
    prof = _lib.Profile()
    _lib.check(ctx.handle, _lib.lib().atc_profile_start(ctx.handle))
    step()
    _lib.check(ctx.handle, _lib.lib().atc_profile_read(ctx.handle, C.byref(prof)))
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    bindings = sum(j.count for j in jobs)
    value = bindings / (ms_per_step / 1e3)

    # ---- correctness of what was timed: NCCL all-reduce MIN of the first passing
    # index and all-gather of the passing sets (paper_2301_11659_b200.shard)
    from paper_2301_11659_b200 import shard

    correct = True
    summary = {}
    for j, r in zip(jobs, results):
        pl, first, _ = shard.reduce_results(r[0].tolist(), r[2], dist, device="cuda")
        if j.expected_pass is not None and pl != j.expected_pass:
            correct = False
        if (first if first >= 0 else None) != (pl[0] if pl else None):
            correct = False
        if pl:
            summary[f"{j.stem}x{j.spec_name}"] = pl[:4]

    # ---- e2e through the C ABI with host buffers (pinned), uploads inside the region
    e2e_ms, h2d, d2h, e2e_ok = _e2e_prepared(args, ctx, ev, jobs, shards, stream, torch, dist, results)
    correct = correct and e2e_ok
    e2e_once_ms, h2d_once, d2h_once = _e2e(args, ctx, jobs, shards, stream, torch, dist, seeded=True)
    e2e_full_ms, h2d_full, _ = _e2e(args, ctx, jobs, shards, stream, torch, dist, seeded=False)

    # ---- roofline of the dominant kernel (K1: k_screen_conv_pairs on the conv
    # spaces, k_screen_rows on the gemm spaces), from the profiled step
    hbm, _, peak_kind = _peaks()
    ncu = _ncu_summary()
    k1 = next((d for d in ncu if d["kernel"].startswith("k_screen_conv_pairs")), {})
    screen_s = prof.screen_ms / 1e3
    # algorithmic bytes: the recorded data the factorised screen must read.  Per
    # conv plane (permutation + digits 2..8; nI x nI bindings): the permutation
    # (3 B), three region lengths (24 B), the output's dirty maximum (4 B) and the
    # position-0/1 verdict words (8 B).  Per gemm row (nI bindings): 3 + 24 + 4 + 1 B.
    alg_bytes = 0.0
    for j, (b, e) in zip(jobs, shards):
        nI = len(j.ts.int_params)
        if j.spec.semantics == "conv2d":
            alg_bytes += (e - b) / (nI * nI) * 39.0
        else:
            alg_bytes += (e - b) / nI * 32.0
    achieved = alg_bytes / screen_s / 1e9 if screen_s > 0 else None
    survey_bytes = sum(j.t0_bytes(b, e) for j, (b, e) in zip(jobs, shards))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic: recorded corpus P2 test sets regenerated from the reference seeds",
        "config": _config(args, jobs),
        "correct": correct, "passing_sample": summary,
        "e2e": {"value": bindings / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "inputs": "per program, every step: the P2 tests' Rng seeds + region stream positions + int "
                          "values + the original runs' final-minus-init entries, written into the program's "
                          "test-set handle (atc_testsets_update_seeded, needed_only: the GPU regenerates the "
                          "region prefixes an evaluation can read), then "
                          "the prepared sweep (atc_enum_batch_run: one CUDA-graph replay) and its result block D2H",
                "one_shot": {"value": bindings / (e2e_once_ms / 1e3), "ms_per_step": e2e_once_ms,
                             "h2d_bytes_per_step": h2d_once, "d2h_bytes_per_step": d2h_once,
                             "inputs": "handles created and freed every step (atc_testsets_upload_seeded) and "
                                       "one eager atc_eval_enumerated_many"},
                "full_regions": {"value": bindings / (e2e_full_ms / 1e3), "ms_per_step": e2e_full_ms,
                                 "h2d_bytes_per_step": h2d_full,
                                 "inputs": "every 65,536-element init and final region (atc_testsets_upload_async)"}},
        # every library kernel of one step (counted by the profiled step) x timed steps;
        # the timed steps replay them as one CUDA graph per step
        "gpu_launches": int(prof.kernels) * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": (achieved / hbm) if achieved else None,
                     "traffic": k1.get("dram_read", 0) + k1.get("dram_write", 0) if k1 else None,
                     "traffic_launch": "ncu --set full of the conv_direct x conv2d launch (2.3e9 bindings; "
                                       "profiles/r1_ncu_summary.json)",
                     "peak_kind": peak_kind, "kernel": "K1 screen (k_screen_conv_pairs + k_screen_rows)",
                     "kernel_ms_per_step": prof.screen_ms,
                     "kernel_ms_note": "sum of the K1 launch durations of one profiled step (CUDA events); the "
                                       "gemm and conv branches of a sweep run concurrently, so this exceeds their "
                                       "wall-clock share",
                     "limiter": "instruction issue (integer ALU); operands are L1/L2 resident",
                     "issue_slots_busy_pct": k1.get("issue_slots_busy_pct"), "ipc_per_sm": k1.get("ipc_per_sm"),
                     "alu_pipe_pct": k1.get("alu_pipe_pct"),
                     "survey_operand_GBps": survey_bytes / screen_s / 1e9 if screen_s > 0 else None,
                     "note": "achieved counts the recorded data the factorised screen reads (per conv plane / gemm "
                             "row, see bench.py); survey_operand_GBps is SURVEY 8d's 8 B x (extA+extB+extC) per "
                             "binding at t=0 — operand bytes the factorisation never streams, so it is not an HBM "
                             "utilisation.  The kernel is issue bound: see issue_slots_busy_pct (ncu)."},
        "k2_confirm": {"ms_per_step": prof.confirm_ms, "survivors_per_step": prof.survivors,
                       "note": "sum of K2 launch durations over the concurrent sweep streams (overlapping)",
                       "fp64_pipe": _fp64_pipe(ctx, ncu)},
    }
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

    def one():  # one C call rewrites every program's handle, then the graph replay
        _lib.check(ctx.handle, L.atc_testsets_update_seeded_many(ctx.handle, hptrs, structs, len(vals)))
        return sweep.run()

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
        ref = torch.nn.functional.conv2d(x[:1].double(), w.double())
        err = ((y[:1].double() - ref).abs() / (1 + ref.abs())).max().item()
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
    _library_tf32(torch)
    cublas_ms = _max_over_ranks(_time_ms(lambda: torch.matmul(a, b, out=c), stream, torch), dist, torch)
    out["cublas_tf32_tflops"] = 2.0 * M * n * k / (cublas_ms / 1e3) / 1e12
    _, bf16, kind = _peaks()
    tf32_peak = bf16 / 2
    out["shape"] = [M, n, k]
    out["per_rank_rows"] = m
    g = next((d for d in _ncu_summary() if d["kernel"].startswith("k_tc_gemm")), {})
    out["roofline"] = {"bound": "tensor", "achieved": out["tf32"]["tflops"], "peak": tf32_peak, "unit": "TFLOP/s",
                       "frac": out["tf32"]["tflops"] / tf32_peak,
                       "traffic": (g.get("dram_read", 0) + g.get("dram_write", 0)) if g else None,
                       "algorithmic_bytes": 3 * m * n * 4,
                       "tensor_pipe_active_pct": g.get("tensor_pipe_active_pct"),
                       "peak_kind": f"TF32 dense = 1/2 of the {kind} cuBLAS bf16 peak; cuBLAS TF32 on the same "
                                    f"operands measured {out['cublas_tf32_tflops']:.0f} TFLOP/s in this run"}
    return out


if __name__ == "__main__":
    main()
