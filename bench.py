#!/usr/bin/env python
"""Benchmark: full branch-length-gradient evaluations per second (BJ:metric).

One step = one full evaluation of the hot path:
transition matrices from the eigensystem for new branch lengths, post-order
pruning, root likelihood, pre-order partials, per-edge gradient, the pattern
reduction and -- at N > 1 GPUs -- the NCCL allreduce of [logL, g].

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--precision fp64]
    torchrun --nproc-per-node N bench.py --gpus N ...      (patterns sharded, strong scaling)
    python bench.py --impl reference ...                    (the CPU oracle as the reference arm)

Timing: K device-timed steps (CUDA events on the instance stream), L2 flushed
between timed steps (outside the events), barrier + synchronize on both
sides, max over ranks.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import phylo_synth as ps  # noqa: E402

METRIC = "full BLS-gradient evals/sec"
UNIT = "evals/s"
CONFIG_NAMES = {0: "jc5_c200", 1: "dengue997_hky_g4_c10000", 2: "carnivore62_mmm16_c5000",
                3: "yeast49_gy94_g4_c4000", 4: "wnv104_gy94_g4_ucld_c3700",
                5: "yeast49_mmm2x61_c4000"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--no-flush", action="store_true", help="do not flush L2 between timed steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the baseline sample")
    ap.add_argument("--virtual-shard", type=int, default=0, metavar="G",
                    help="evidence runs only: time rank 0's pattern shard of a G-GPU run on this one GPU "
                         "(value = that shard's evals/s; not a bench line)")
    ap.add_argument("--patterns", type=int, default=0, metavar="C",
                    help="evidence runs only (pattern-count sweep, SURVEY §8(f) NEXT-3): the config's "
                         "workload with C unique patterns instead of its default; not a bench line")
    return ap.parse_args()


def workload_name(cfg: int, C: int) -> str:
    base = CONFIG_NAMES[cfg]
    return base if cfg == 0 else base[:base.rfind("_c")] + f"_c{C}"


def make_problem(cfg: int, precision: str, patterns: int = 0):
    kw = {"precision": precision} if cfg in (1, 2, 3, 4, 5) else {}
    if patterns > 0:
        kw["C"] = patterns
    return ps.make_config(cfg, **kw)


def dtype_name(precision: str) -> str:
    return "f64" if precision == "fp64" else "f32"


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------- roofline ----

def algorithmic_bytes(pb, C: int, precision: str) -> int:
    """Compulsory HBM bytes of one traversal launch:
    u = P p of every internal non-root node written once (post) and read once
    (pre): 2 (N-2) R C SP w; tip codes read once per pass: 2 N C; pattern
    weights 8 C.  SP = padded states."""
    N, S, R = pb.n_tips, pb.states, len(pb.cat_rates)
    SP = 4 if S <= 4 else 8 if S <= 8 else 16 if S <= 16 else 32 if S <= 32 else 64 if S <= 64 else 128
    w = 8 if precision == "fp64" else 4
    tips = 2 * N * C if pb.tip_partials is None else 2 * N * C * SP * w
    return 2 * (N - 2) * R * C * SP * w + tips + 8 * C


def algorithmic_flops(pb, C: int) -> int:
    """Minimal flops of one evaluation: 3 (N-2) matvecs of
    2 S^2 per (pattern, category) with unpadded S."""
    N, S, R = pb.n_tips, pb.states, len(pb.cat_rates)
    return 3 * (N - 2) * 2 * S * S * R * C


def alu_roofline(pb, C, trav_ms, peaks, precision, abytes, traffic):
    """S > 64 (and fp32 S > 16): the SIMT large-state kernel is bound by plain
    FP64 (FP32) FMA throughput, not HBM: achieved = minimal flops / launch time
    against the measured DFMA peak (derived FFMA peak for fp32)."""
    fl = algorithmic_flops(pb, C)
    ach = fl / (trav_ms * 1e-3) / 1e12
    pk, src = ((peaks["dfma_tflops"], peaks["dfma_src"]) if precision == "fp64"
               else (peaks["ffma_tflops"], peaks["ffma_src"]))
    return {"bound": "alu", "achieved": round(ach, 3), "peak": round(pk, 2), "unit": "TFLOP/s",
            "frac": round(ach / pk, 4), "traffic": traffic, "kernel": "traverse_large_kernel (SIMT)",
            "algorithmic_flops_per_eval": fl, "kernel_ms": round(trav_ms, 5), "hbm_algorithmic_bytes": abytes,
            "peak_source": src}


def load_peaks():
    """HBM: MEASURED_PEAKS.json (driver-written copy bandwidth).  FP64 tensor:
    our DMMA microbenchmark on this pool's B200 (scripts/fp64_peak.cu ->
    profiles/r01/fp64_peak.json); MEASURED_PEAKS.json has no FP64 entry."""
    out = {}
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out.update(hbm_gbs=float(d["hbm_gbs"]), hbm_src="measured (MEASURED_PEAKS.json hbm_gbs)")
    except Exception:
        out.update(hbm_gbs=6650.0, hbm_src="fallback (B200_PROFILING.md)")
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r01", "fp64_peak.json")))
        out.update(fp64_tflops=float(d["dmma_tflops"]),
                   fp64_src="measured (mma.sync f64 DMMA microbenchmark, profiles/r01/fp64_peak.json)")
    except Exception:
        out.update(fp64_tflops=37.0, fp64_src="fallback (B200 datasheet FP64 tensor ~37-40 TF/s)")
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r01", "fp64_peak.json")))
        out.update(dfma_tflops=float(d["dfma_tflops"]),
                   dfma_src="measured (DFMA microbenchmark, profiles/r01/fp64_peak.json)")
    except Exception:
        out.update(dfma_tflops=36.0, dfma_src="fallback (B200 FP64 ~37 TF/s)")
    # FP32 FFMA: 148 SMs x 128 lanes x 2 flops x 1.965 GHz (guide unit counts, max clock)
    out.update(ffma_tflops=148 * 128 * 2 * 1.965e9 / 1e12, ffma_src="derived: 148 SMs x 128 FP32 lanes x 2 x 1.965 GHz")
    return out


def load_traffic(cfg: int, precision: str):
    """DRAM bytes per traversal launch from a committed ncu --set full capture
    (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p)).get(f"config{cfg}_{precision}")
        return None if d is None else d["bytes"]
    except Exception:
        return None


# ------------------------------------------------------------ CPU oracle ----

def cpu_oracle_rate(pb, seconds: float):
    """Oracle evals/s on a bounded pattern sample, all host cores."""
    import oracle
    threads = os.cpu_count() or 1
    C = pb.patterns
    # calibrate on a small sample, then size the sample to ~`seconds`
    m0 = min(C, max(threads * 4, 64))
    t0 = time.perf_counter()
    oracle.loglik_grad(pb, 0, m0, threads=threads, block=max(1, m0 // threads))
    dt0 = time.perf_counter() - t0
    m = int(min(C, max(m0, m0 * seconds / max(dt0, 1e-6))))
    reps, dt = 0, 0.0
    while reps == 0 or (dt < 0.5 * seconds and reps < 50):     # whole workload faster than the budget: repeat
        t0 = time.perf_counter()
        oracle.loglik_grad(pb, 0, m, threads=threads, block=max(1, -(-m // (threads * 4))))
        dt += time.perf_counter() - t0
        reps += 1
    rate = reps * (m / C) / dt
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"patterns [0,{m}) of {C} (full tree) x {reps} evaluation(s), {dt:.1f} s, scaled by C/{m}"}


# ------------------------------------------------------------------ ours ----

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2303_04390_b200 as pg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    pb = make_problem(args.config, args.precision, args.patterns)
    C = pb.patterns
    lo, hi = pg.shard_range(C, world, rank)
    if args.virtual_shard > 1:
        assert world == 1, "--virtual-shard is a single-process emulation"
        lo, hi = pg.shard_range(C, args.virtual_shard, 0)
    inst = pg.from_problem(pb, precision=args.precision, device=local, lo=lo, hi=hi)
    stream = inst.stream
    B = 2 * pb.n_tips - 2
    out = torch.zeros(B + 1, dtype=torch.float64, device=dev)

    # seeded +-1% branch-length jitter per step, resident on the device
    rng = np.random.default_rng(ps.MASTER_SEED + 99)
    nvar = args.warmup + args.steps
    bls = pb.branch_lengths[None, :] * rng.uniform(0.99, 1.01, size=(nvar, B))
    bl_dev = torch.tensor(bls, dtype=torch.float64, device=dev)
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(i):
        inst.set_branch_lengths_device(bl_dev[i])
        inst.compute_device(out)
        if world > 1:
            pg.allreduce_evaluation(out)

    inst.set_kernel_timing(True)
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
        stream.synchronize()
        zp = inst.check_status()
        assert zp < 0, f"zero likelihood at pattern {zp}"
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        ktimes = {"pmat": 0.0, "traverse": 0.0, "reduce": 0.0}
        with ClockSampler(local) as clk:
            for k in range(args.steps):
                if flush is not None:
                    flush.zero_()
                evs[k][0].record(stream)
                step(args.warmup + k)
                evs[k][1].record(stream)
                if k % 16 == 0 or k == args.steps - 1:     # per-kernel split on a sample of steps
                    t = inst.kernel_times()
                    for n in ktimes:
                        ktimes[n] += t[n]
            stream.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    nsamp = len([k for k in range(args.steps) if k % 16 == 0 or k == args.steps - 1])
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms = float(t.item())
    ms_per_step = dev_ms / args.steps
    value = 1000.0 / ms_per_step            # whole-job evaluations per second
    kavg = {n: v / nsamp for n, v in ktimes.items()}

    # ---- end to end through the public API with host buffers ---------------
    inst.set_kernel_timing(False)
    e2e_steps = max(10, min(args.steps, 200))
    host_out = torch.empty(B + 1, dtype=torch.float64, pin_memory=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        inst.set_branch_lengths(bls[k % nvar])
        if world == 1:
            logl, g = inst.compute()
        else:
            with torch.cuda.stream(stream):
                inst.compute_device(out)
                pg.allreduce_evaluation(out)
                host_out.copy_(out, non_blocking=True)
            stream.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_rate = e2e_steps / float(te.item())

    # ---- parity spot check of this run's last evaluation (rank 0, N = 1) -----
    result = None
    if rank == 0:
        peaks = load_peaks()
        Cl = hi - lo
        abytes = algorithmic_bytes(pb, Cl, args.precision)
        trav_ms = kavg["traverse"]
        achieved = abytes / (trav_ms * 1e-3) / 1e9
        traffic = load_traffic(args.config, args.precision)
        info = inst.plan_info()
        tensor = info["kernel_variant"] == 2
        result = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": dtype_name(args.precision), "data": "synthetic",
            "config": {"workload": workload_name(args.config, C), "tips": pb.n_tips, "patterns": C,
                       "states": pb.states, "categories": len(pb.cat_rates),
                       "precision": args.precision,
                       "l2": "flushed (256 MiB write) between timed steps" if flush is not None else "not flushed",
                       "parallelism": f"pattern-shard x{world}" if args.virtual_shard <= 1 else
                                      f"virtual: rank 0's shard [{lo},{hi}) of x{args.virtual_shard}, on 1 GPU",
                       "branch_lengths": "seeded +-1% jitter per step, device resident"},
            "e2e": {"value": round(e2e_rate, 3), "unit": UNIT, "h2d_bytes_per_step": 8 * B,
                    "d2h_bytes_per_step": 8 * (B + 1) + (4 if world == 1 else 0)},
            "gpu_launches": args.steps * inst.kernels_per_eval(),
            "roofline": alu_roofline(pb, Cl, trav_ms, peaks, args.precision, abytes, traffic)
            if info["kernel_variant"] == 1 else
            ({"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                          "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                          "traffic": traffic,
                          "kernel": "traverse_small_kernel" if info["kernel_variant"] == 0 else "traverse_large_kernel",
                          "algorithmic_bytes_per_launch": abytes, "kernel_ms": round(trav_ms, 5),
                          "peak_source": peaks["hbm_src"]} if not tensor else
                         {"bound": "tensor",
                          "achieved": round(algorithmic_flops(pb, Cl) / (trav_ms * 1e-3) / 1e12, 3),
                          "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                          "frac": round(algorithmic_flops(pb, Cl) / (trav_ms * 1e-3) / 1e12 / peaks["fp64_tflops"], 4),
                          "traffic": traffic,
                          "kernel": ("codon_flow_kernel (post + pre order, one launch)" if info.get("flow_tiles", 0) > 0
                                     else "codon_post_kernel + codon_pre_kernel (all levels of one evaluation)"),
                          "algorithmic_flops_per_eval": algorithmic_flops(pb, Cl), "kernel_ms": round(trav_ms, 5),
                          "hbm_algorithmic_bytes": abytes, "peak_source": peaks["fp64_src"],
                          "dtype_note": "fp64 on the FP64 tensor path (DMMA)"}),
            "kernel_ms": {k: round(v, 5) for k, v in kavg.items()},
            "plan": info,
            "clocks": clk.summary(),
        }

    inst.close()
    return result, pb


def run_reference(args):
    """The CPU oracle as the reference arm, on our arm's config and metric."""
    import oracle
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    pb = make_problem(args.config, args.precision, args.patterns)
    C = pb.patterns
    threads = os.cpu_count() or 1
    # size the per-step sample so the whole run takes ~2-3 minutes
    m0 = min(C, threads * 4)
    t0 = time.perf_counter()
    oracle.loglik_grad(pb, 0, m0, threads=threads, block=max(1, m0 // threads))
    per_pat = (time.perf_counter() - t0) / m0
    budget = 150.0 / max(1, args.steps + min(args.warmup, 3))
    m = int(max(threads, min(C, budget / per_pat)))
    for _ in range(min(args.warmup, 3)):
        oracle.loglik_grad(pb, 0, m, threads=threads, block=max(1, -(-m // threads)))
    times = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        oracle.loglik_grad(pb, 0, m, threads=threads, block=max(1, -(-m // threads)))
        times.append(time.perf_counter() - t0)
    step_s = sum(times) / len(times)
    value = (m / C) / step_s
    sample = f"patterns [0,{m}) of {C} per step (full tree), scaled by C/{m}"
    return {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000.0 / value, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config, C), "tips": pb.n_tips, "patterns": C,
                       "states": pb.states, "categories": len(pb.cat_rates), "precision": "fp64"},
            "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": threads,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if args.impl == "reference":
        res = run_reference(args)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    res, pb = run_ours(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_oracle_rate(pb, args.cpu_seconds)
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
