#!/usr/bin/env python
"""bench.py — batched fp64 GFLOP/s vs n and % of roofline on B200
(BASELINE.json metric; SURVEY §8d definitions).

A "step" is one pass of the hot path over one batch of synthetic input per
size: by default configs[1] of BASELINE.json, the upper-Cholesky sweep over
n in {4, 8, ..., 128} with batch floor(2^28 / 8n^2) (256 MiB of A per n),
seed n.  The Lyapunov (configs[2]) and Sylvester (configs[3]) sweeps are
measured the same way and reported under "extra".

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload chol-sweep|lyap-sweep|sylv-sweep|c1|c5-chol|c5-lyap|c5-sylv]
                    [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU, NCCL only for the barrier and the
max-over-ranks time): every rank solves its own index range of problems
(weak scaling for the sweeps, strong scaling for c5), no data-path
collective.

Timing: W untimed warm-up steps, then K steps; the sweep is captured once
in a CUDA graph (one kernel per size) and replayed; CUDA events on the
launching stream, synchronize + barrier on both sides, max over ranks.
Inputs per size are >= 256 MiB per operand (larger than the 126 MB L2)
except c1, which flushes L2 between steps.
"""

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

SIZES = list(range(4, 129, 4))
EQS = {"chol": "cholesky", "lyap": "lyapunov", "sylv": "sylvester"}
NOMINAL_HBM_GBS = 8000.0        # BASELINE.md roofline (nominal)
NOMINAL_FP64_TFLOPS = 37.2      # 148 SM x 64 FMA/clk x 2 x 1.965 GHz
METRIC = "batched fp64 GFLOP/s vs n (n^3/3 chol; 2n^3 lyap/sylv); % of roofline"


def measured_peaks():
    peaks = {"hbm_gbs": None, "fp64_tflops": None, "source": {}}
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        peaks["hbm_gbs"] = d.get("hbm_gbs")
        peaks["source"]["hbm_gbs"] = "MEASURED_PEAKS.json (measured copy)"
    if peaks["hbm_gbs"] is None:
        peaks["hbm_gbs"] = 6650.0
        peaks["source"]["hbm_gbs"] = "fallback (B200_PROFILING.md)"
    f = REPO / "profiles" / "fp64_peaks.json"
    if f.exists():
        d = json.loads(f.read_text())
        peaks["fp64_tflops"] = max(d.get("dfma_tflops", 0), d.get("dmma_tflops", 0))
        peaks["source"]["fp64_tflops"] = "profiles/fp64_peaks.json (tools/fp64_peaks.cu, measured)"
    else:
        peaks["fp64_tflops"] = NOMINAL_FP64_TFLOPS
        peaks["source"]["fp64_tflops"] = "nominal"
    return peaks


def batch_for(n):
    return (1 << 28) // (8 * n * n)


def workload(name, world, rank=0):
    """(eq, [(n, batch_this_rank, seed, first_index)], scaling, description)."""
    from paper_1906_08613_b200.shard import shard_range, weak_range
    if name.endswith("-sweep"):
        eq = EQS[name.split("-")[0]]
        return eq, [(n, batch_for(n), n, weak_range(batch_for(n), rank)[0]) for n in SIZES], "weak", \
            f"{eq} sweep n=4..128 step 4, batch floor(2^28/8n^2) per GPU, seed n"
    if name == "c1":
        return "cholesky", [(16, 4096, 0, weak_range(4096, rank)[0])], "weak", \
            "cholesky n=16 batch 4096 seed 0 (L2 flushed between steps)"
    if name.startswith("c5-"):
        eq = EQS[name.split("-")[1]]
        first, count = shard_range(1 << 20, rank, world)
        return eq, [(64, count, 7, first)], "strong", f"{eq} n=64, 2^20 problems sharded over GPUs, seed 7"
    raise SystemExit(f"unknown workload {name}")


# ----------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ----------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, v in self.REASONS.items():
                    if mask & v and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.nvml:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.nvml:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------
def dist_setup(gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        torch.distributed.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM)
    return float(t.item())


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def run_sweep(eq, cases, rank, steps, warmup, peaks, flush_l2=False, per_n_reps=None, clocks=None):
    """Returns dict with per-step times, per-n kernel times and bookkeeping."""
    from paper_1906_08613_b200 import executor
    from paper_1906_08613_b200.variants import bytes_compulsory, flops_alg, flops_nominal

    stream = torch.cuda.Stream()
    plans = []
    with torch.cuda.stream(stream):
        for n, batch, seed, first in cases:
            ins = executor.generate(eq, n, seed, batch, first=first, stream=stream)
            plans.append(executor.Plan(eq, ins))
    stream.synchronize()
    # first launches (sets kernel attributes outside capture) + check
    for p in plans:
        p.launch(stream)
    stream.synchronize()
    for p in plans:
        bad = int((p.info != 0).sum())
        if bad:
            raise RuntimeError(f"{eq} n={p.n}: {bad} problems reported info != 0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if flush_l2 else None

    graph = None
    if not flush_l2:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for p in plans:
                p.launch(stream)
        stream.synchronize()

    def one_step():
        if graph is not None:
            graph.replay()
        else:
            for p in plans:
                p.launch(stream)

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            if flush is not None:
                flush.fill_(1)
            one_step()
    stream.synchronize()
    times = []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    with (clocks or _Null()):
        with torch.cuda.stream(stream):
            for i in range(steps):
                if flush is not None:
                    flush.fill_(1)
                ev[i][0].record(stream)
                one_step()
                ev[i][1].record(stream)
        stream.synchronize()
    times = [a.elapsed_time(b) for a, b in ev]

    # per-size kernel times (events around each launch; median of reps)
    reps = per_n_reps or max(3, min(steps, 10))
    per_n = []
    with torch.cuda.stream(stream):
        for p in plans:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(reps)]
            for a, b in evs:
                if flush is not None:
                    flush.fill_(1)
                a.record(stream)
                p.launch(stream)
                b.record(stream)
            stream.synchronize()
            ms = statistics.median(x.elapsed_time(y) for x, y in evs)
            n, batch = p.n, p.batch
            f_nom, f_alg, byt = flops_nominal(eq, n), flops_alg(eq, n), bytes_compulsory(eq, n)
            t = ms * 1e-3
            t_roof_nom = batch * max(f_alg / (NOMINAL_FP64_TFLOPS * 1e12), byt / (NOMINAL_HBM_GBS * 1e9))
            t_roof_meas = batch * max(f_alg / (peaks["fp64_tflops"] * 1e12), byt / (peaks["hbm_gbs"] * 1e9))
            per_n.append({
                "n": n, "batch": batch, "variant": p.variant, "b": p.b, "engine": p.engine, "ms": round(ms, 5),
                "gflops": round(batch * f_nom / t / 1e9, 1),
                "gflops_alg": round(batch * f_alg / t / 1e9, 1),
                "gbs": round(batch * byt / t / 1e9, 1),
                "bound": "hbm" if byt / (peaks["hbm_gbs"] * 1e9) >= f_alg / (peaks["fp64_tflops"] * 1e12) else "fp64",
                "roofline_frac_nominal": round(t_roof_nom / t, 4),
                "roofline_frac_measured": round(t_roof_meas / t, 4),
            })
    out = {"times_ms": times, "per_n": per_n, "plans": plans, "stream": stream,
           "flops_nominal": sum(p.batch * flops_nominal(eq, p.n) for p in plans),
           "flops_alg": sum(p.batch * flops_alg(eq, p.n) for p in plans),
           "bytes": sum(p.batch * bytes_compulsory(eq, p.n) for p in plans),
           "launches_per_step": len(plans)}
    return out


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def run_e2e(eq, plans, steps, world):
    """Same workload through the public host-buffer API (executor.solve_host):
    every step moves the inputs from pinned host memory to the GPU, solves,
    and moves X and info back.  Only the structurally needed part of each
    operand crosses PCIe where that wins (solve_host's default from n = 16
    on: the copy engines move the contiguous mostly-needed half of each
    triangular operand, zero-copy kernels the remaining small triangle; dense
    copies below); for Cholesky the host X is zeroed once at allocation — the
    reference's own contract for its kernels' outputs (codegen.py:4-7) — so
    only X's upper triangle comes back there (LAGEN_HOST_X_ZEROED)."""
    from paper_1906_08613_b200 import _lib, executor
    from paper_1906_08613_b200.variants import EQ_CODES
    zeroed = eq == "cholesky"
    hosts = []
    for p in plans:
        ins = [t.cpu().pin_memory() for t in p.inputs]
        out = torch.zeros(ins[0].shape, dtype=torch.float64).pin_memory()
        info = torch.empty(p.batch, dtype=torch.int32).pin_memory()
        hosts.append((p, ins, out, info))
    def flags_of(n):  # what solve_host's default picks (executor.solve_host, triangles=None)
        tri = executor.host_triangles_default(eq, n)
        return (_lib.HOST_TRIANGLES if tri else 0) | (_lib.HOST_X_ZEROED if zeroed else 0)
    moved = [_lib.host_bytes(EQ_CODES[eq], p.n, p.batch, flags_of(p.n)) for p, _, _, _ in hosts]
    h2d = sum(m[0] for m in moved)
    d2h = sum(m[1] for m in moved)

    def one_pass():
        # the sizes of a step are queued back to back (wait=False) and waited
        # for once: the four-stream pipeline fills and drains once per step,
        # not once per size
        for p, ins, out, info in hosts:
            executor.solve_host(eq, ins, variant=p.variant, b=p.b, out=out, info=info, engine=p.engine,
                                out_zeroed=zeroed, wait=False)
        executor.host_sync()
    one_pass()  # warm-up
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        one_pass()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    barrier(world)
    dt = max_over_ranks(dt, world)
    # correctness of what came back (smallest and largest size)
    for p, ins, out, info in (hosts[0], hosts[-1]):
        assert torch.equal(out, p.out.cpu()), "host pipeline result differs from device path"
        assert int(info.abs().sum()) == 0
    return dt / steps, h2d, d2h


# ----------------------------------------------------------------------------
# CPU baseline (reference's emitted C through oracle/_ref, else the port)
# ----------------------------------------------------------------------------
def cpu_baseline(eq, cases, budget_s=12.0, inputs_from=None, seed_first=0):
    """Time the reference CPU path on a bounded sample of each size; value is
    the throughput it would sustain on the full workload (problems are
    independent, so time scales linearly with the batch)."""
    from oracle import build_ref, oracle
    from paper_1906_08613_b200.variants import builtin_variants, default_blocks, flops_nominal

    cores = len(os.sched_getaffinity(0))
    use_ref = build_ref.available()
    ref = build_ref.RefLib() if use_ref else None
    per_size_budget = budget_s / len(cases)
    tot_flops, tot_time, detail = 0.0, 0.0, []
    for ci, (n, batch, seed, first) in enumerate(cases):
        # sample size: aim at ~per_size_budget/2 for the timed run
        est_ns = {"cholesky": 0.35, "lyapunov": 0.8, "sylvester": 1.1}[eq] * n ** 3 / cores
        s = int(max(cores, min(batch, per_size_budget * 0.5 / (est_ns * 1e-9))))
        if inputs_from is not None:
            ins = [t[:s].cpu().numpy() for t in inputs_from[ci]]
        else:
            ins = oracle.generate(eq, n, seed, first, s)
        if ref is not None:
            cands = ref.kernels(eq, n)
            best = None
            probe = [a[: max(cores, s // 8)] for a in ins]
            for idx, k in cands:
                ref.run(idx, probe)
                t0 = time.perf_counter()
                ref.run(idx, probe)
                dt = time.perf_counter() - t0
                if best is None or dt < best[0]:
                    best = (dt, idx, k)
            _, idx, k = best
            ref.run(idx, [a[:cores] for a in ins])
            t0 = time.perf_counter()
            ref.run(idx, ins)
            dt = time.perf_counter() - t0
            which = k["name"]
        else:
            v = builtin_variants(eq)[0]
            b = default_blocks(n)[0]
            t0 = time.perf_counter()
            oracle.execute(eq, v.statements, n, b, ins, nthreads=cores)
            dt = time.perf_counter() - t0
            which = f"oracle port v0 b{b}"
        t_full = dt * batch / s
        tot_flops += batch * flops_nominal(eq, n)
        tot_time += t_full
        detail.append({"n": n, "sample": s, "kernel": which, "gflops": round(s * flops_nominal(eq, n) / dt / 1e9, 2)})
    return {
        "value": round(tot_flops / tot_time / 1e9, 2), "unit": "GFLOP/s", "cores": cores,
        "kind": "reference" if use_ref else "port",
        "sample": (f"per size: the first s problems of the same workload (s sized for ~{per_size_budget:.2f} s), "
                   "throughput extrapolated to the full batch; kernel = fastest verified emitted variant "
                   "(lagen emit_function, scalar and nu=4 modes) compiled gcc -O3 -march=native -std=c99, OpenMP over problems")
        if use_ref else "oracle C port, OpenMP over problems",
        "sample_short": (f"first s problems of each size (~{per_size_budget:.2f} s per size), "
                         "extrapolated to the full batch"),
        "cpu_model": _cpu_model(), "per_n": detail,
    }


def _cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ----------------------------------------------------------------------------
def summarize(eq, res, steps, peaks, world):
    """(value, ms_per_step, roofline, per_n) for one sweep.

    roofline: aggregate over the step's launches — the algorithmic bytes (or
    flops) of every launch (SURVEY §8d per-problem figure x batch) over the
    sum of their event-timed durations, against the measured peak of the
    binding roof; "dominant" is the launch with the largest share of the
    step, with its own achieved / frac and its ncu DRAM traffic."""
    ms = statistics.mean(res["times_ms"])
    ms = max_over_ranks(ms, world)
    flops = sum_over_ranks(res["flops_nominal"], world)
    value = flops / (ms * 1e-3) / 1e9
    per_n = res["per_n"]
    t_kernels = sum(r["ms"] for r in per_n) * 1e-3
    achieved_gbs = res["bytes"] / t_kernels / 1e9
    achieved_tf = res["flops_alg"] / t_kernels / 1e12
    hbm_time = res["bytes"] / (peaks["hbm_gbs"] * 1e9)
    fp_time = res["flops_alg"] / (peaks["fp64_tflops"] * 1e12)
    if hbm_time >= fp_time:
        roof = {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved_gbs / peaks["hbm_gbs"], 4)}
    else:
        roof = {"bound": "fp64", "achieved": round(achieved_tf, 3), "peak": peaks["fp64_tflops"],
                "unit": "TFLOP/s", "frac": round(achieved_tf / peaks["fp64_tflops"], 4)}
    # per-n roofline (time at the binding measured roof / measured time),
    # aggregated as roof time over kernel time
    t_roof = sum(r["ms"] * r["roofline_frac_measured"] for r in per_n) * 1e-3
    roof["frac_roofline_time"] = round(t_roof / t_kernels, 4)
    roof["frac_min_n_ge_32"] = min((r["roofline_frac_measured"] for r in per_n if r["n"] >= 32), default=None)
    dom = max(per_n, key=lambda r: r["ms"])
    roof["dominant"] = {"n": dom["n"], "engine": dom["engine"], "share": round(dom["ms"] * 1e-3 / t_kernels, 3),
                        "gbs": dom["gbs"], "frac": dom["roofline_frac_measured"]}
    roof["scope"] = "all launches of one step (sum of algorithmic bytes / sum of launch times)"
    roof["traffic"] = None
    for tf in (REPO / "profiles" / "r02_traffic.json", REPO / "profiles" / "r01_traffic.json"):
        if tf.exists():
            t = json.loads(tf.read_text()).get(eq)
            if t:
                roof["traffic"] = t["dram_bytes_per_launch"]
                roof["traffic_ratio"] = t["ratio"]
                roof["traffic_of"] = f"n={t['n']} ({tf.name})"
                break
    return value, ms, roof, per_n


def cpu_compact(c):
    return {k: c[k] for k in ("value", "unit", "cores", "kind")} | {"sample": c["sample_short"]}


def run_one(wl, args, world, rank, peaks, warmup, clocks=None, want_e2e=True, want_cpu=True):
    eq, cases, scaling, desc = workload(wl, world, rank)
    res = run_sweep(eq, cases, rank, args.steps, warmup, peaks, flush_l2=(wl == "c1"), clocks=clocks)
    value, ms, roof, per_n = summarize(eq, res, args.steps, peaks, world)
    out = {"eq": eq, "value": value, "ms": ms, "roofline": roof, "per_n": per_n, "desc": desc,
           "scaling": scaling, "sizes": [c[0] for c in cases], "launches": res["launches_per_step"]}
    if want_e2e and not args.no_e2e:
        e2e_steps = max(1, min(2, args.steps))
        dt, h2d, d2h = run_e2e(eq, res["plans"], e2e_steps, world)
        out["e2e"] = {"value": round(sum_over_ranks(res["flops_nominal"], world) / dt / 1e9, 2),
                      "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                      "path": "solve_host, pinned" + (", X zeroed by caller (reference contract)" if eq == "cholesky" else "")}
    if want_cpu and rank == 0 and world == 1 and not args.no_cpu:
        out["cpu"] = cpu_baseline(eq, cases, budget_s=args.cpu_budget, inputs_from=[p.inputs for p in res["plans"]])
    del res
    torch.cuda.empty_cache()
    return out


def spawn_ranks(gpus):
    """--gpus N > 1 without a launcher: re-exec this script under
    torch.distributed.run with N processes (one per GPU)."""
    port = os.environ.get("MASTER_PORT", "29533")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", "--master-port", port, str(Path(__file__).resolve()), *sys.argv[1:]]
    import subprocess
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="chol-sweep")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sizes", default=None, help="comma-separated subset of n (debug)")
    ap.add_argument("--no-extra", action="store_true", help="skip the lyap/sylv sweeps")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=8.0)
    ap.add_argument("--json-out", default=None, help="full per-n detail (the printed line stays compact)")
    ap.add_argument("--stub", action="store_true",
                    help="CPU-only dry run of the distributed plumbing (gloo, no kernels); tests only")
    args = ap.parse_args()
    if args.sizes:
        global SIZES
        SIZES = [int(x) for x in args.sizes.split(",")]
    warmup = max(3, args.warmup)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return reference_arm(args, warmup)
    if args.stub:
        return stub_arm(args, warmup)

    world, rank, local = dist_setup(args.gpus)
    if args.gpus > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    peaks = measured_peaks()
    clocks = ClockSampler(local)
    barrier(world)
    head = run_one(args.workload, args, world, rank, peaks, warmup, clocks=clocks)
    extra = {}
    if args.workload == "chol-sweep" and not args.no_extra:
        for wl in ("lyap-sweep", "sylv-sweep"):
            extra[wl] = run_one(wl, args, world, rank, peaks, warmup)
    line = {
        "metric": METRIC, "value": round(head["value"], 2), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": warmup, "ms_per_step": round(head["ms"], 4), "higher_is_better": True,
        "scaling": head["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, BASELINE.json distributions)",
        "config": {"workload": args.workload, "description": head["desc"],
                   "sizes": _sizes_text(head["sizes"]),
                   "l2": "flush 256 MiB between steps" if args.workload == "c1" else
                   "inputs > L2 (>= 256 MiB per operand per size)",
                   "parallelism": f"shard by problem index x{world}, no collective"},
        "roofline": head["roofline"],
        "gpu_launches": head["launches"] * args.steps,
        "clocks": clocks.summary(),
    }
    if "e2e" in head:
        line["e2e"] = head["e2e"]
    if "cpu" in head:
        line["cpu_baseline"] = cpu_compact(head["cpu"])
    if extra:
        line["extra"] = {}
        for wl, r in extra.items():
            e = {"value": round(r["value"], 2), "ms_per_step": round(r["ms"], 3),
                 "roofline_frac": r["roofline"]["frac"], "roofline_bound": r["roofline"]["bound"],
                 "frac_roofline_time": r["roofline"]["frac_roofline_time"],
                 "frac_min_n_ge_32": r["roofline"]["frac_min_n_ge_32"]}
            if "e2e" in r:
                e["e2e"] = r["e2e"]["value"]
            if "cpu" in r:
                e["cpu_baseline"] = r["cpu"]["value"]
            line["extra"][r["eq"]] = e
    if rank == 0:
        print(json.dumps(line, separators=(",", ":")), flush=True)
        if args.json_out:
            detail = dict(line)
            detail["peaks"] = peaks
            detail["per_n"] = head["per_n"]
            if "cpu" in head:
                detail["cpu_baseline_detail"] = head["cpu"]
            detail["extra_detail"] = {r["eq"]: {"per_n": r["per_n"], "roofline": r["roofline"],
                                                "cpu": r.get("cpu"), "e2e": r.get("e2e")}
                                      for r in extra.values()}
            Path(args.json_out).write_text(json.dumps(detail, indent=1) + "\n")
    if world > 1:
        torch.distributed.destroy_process_group()


def _sizes_text(sizes):
    if len(sizes) > 3 and all(b - a == sizes[1] - sizes[0] for a, b in zip(sizes, sizes[1:])):
        return f"{sizes[0]}..{sizes[-1]} step {sizes[1] - sizes[0]}"
    return ",".join(map(str, sizes))


def stub_arm(args, warmup):
    """The distributed plumbing of the GPU arm (rank setup, barrier, per-rank
    shard, max-over-ranks time, whole-job sum, rank-0 line) with a CPU stub
    in place of the kernels, under gloo — exercised by tests/test_bench_dist.py."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        torch.distributed.init_process_group("gloo")
    eq, cases, scaling, desc = workload(args.workload, world, rank)
    flops = 0.0
    for n, batch, seed, first in cases:
        flops += batch * _nominal(eq, n)
    dts = []
    for i in range(warmup + args.steps):
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        time.sleep(0.001 * (rank + 1))  # rank-dependent "device time"
        dt = time.perf_counter() - t0
        if i >= warmup:
            dts.append(dt)
    ms = statistics.mean(dts) * 1e3
    t = torch.tensor([ms, flops], dtype=torch.float64)
    if world > 1:
        mx = t[:1].clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        sm = t[1:].clone()
        torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM)
        ms, flops = float(mx.item()), float(sm.item())
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                          "n_gpus": world, "steps": args.steps, "warmup": warmup, "ms_per_step": ms,
                          "scaling": scaling, "stub": True,
                          "config": {"workload": args.workload, "first_index": [c[3] for c in cases][:1]}}),
              flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def _nominal(eq, n):
    return n ** 3 / 3 if eq == "cholesky" else 2.0 * n ** 3


def reference_arm(args, warmup):
    """The reference's own CPU implementation of the path (oracle/_ref: the
    emitted kernels compiled with the reference's flags) on the host cores,
    same workload / metric; rank 0 only (other ranks exit 0 without work)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    eq, cases, scaling, desc = workload(args.workload, 1, 0)
    # each step: a bounded sample of every size, throughput extrapolated
    budget = max(1.0, 60.0 / (args.steps + warmup))
    for _ in range(warmup):
        cpu_baseline(eq, cases, budget_s=budget / 4)
    vals = []
    t0 = time.perf_counter()
    base = None
    for _ in range(args.steps):
        base = cpu_baseline(eq, cases, budget_s=budget)
        vals.append(base["value"])
    dt = time.perf_counter() - t0
    value = statistics.median(vals)
    base["value"] = value
    line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": warmup, "ms_per_step": round(dt / args.steps * 1e3, 2), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator CPU twin, BASELINE.json distributions)",
            "config": {"workload": args.workload, "description": desc, "sizes": _sizes_text([c[0] for c in cases])},
            "impl": "reference", "cpu_baseline": cpu_compact(base),
            "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line, separators=(",", ":")), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
